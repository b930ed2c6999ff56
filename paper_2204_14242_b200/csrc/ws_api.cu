// ws_api.cu -- host side of libwsb200.so: the C ABI of include/ws.h.
// Validates and deep-copies descriptors, owns device scratch, enqueues the
// device path (ws_kernels.cu) on the context stream.  No arithmetic of the
// estimator runs here: every step a1-a8 is a kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX: ranges for nsys / ncu --nvtx (no cost without a tool)

#include "ws_internal.cuh"

using namespace wsb;

namespace {
struct NvtxRange {  // one NVTX range per ABI call
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct ws_ctx {
  int device = 0;
  int n_sm_dev = 148;
  cudaStream_t stream = nullptr;
  std::string err;
  std::vector<DKernel> hk;
  std::vector<DGpu> hg;
  std::vector<int64_t> chunk_bound;  // per kernel: max row chunks of one configuration
  DKernel* dk = nullptr;
  DGpu* dg = nullptr;
  size_t cap_k = 0, cap_g = 0;
  bool dirty = false;
  void* scratch = nullptr;
  size_t scratch_cap = 0;
  void* io = nullptr;  // host-path staging for configs + results
  wsb::SimCache sim_cache;  // ws_simulate's device buffers (until ws_sim_release / ws_destroy)
  size_t io_cap = 0;
  uint32_t last_launches = 0;
  unsigned long long* last_work = nullptr;
  // ws_rank: device scratch of the radix path and the host path's staging (grow-only)
  void* rank_buf = nullptr;
  size_t rank_cap = 0;
  void* rank_io = nullptr;
  size_t rank_io_cap = 0;
  uint32_t last_groups = 0; // ws_estimate_multi: integer-stage groups of the last call
  void* xcfg = nullptr;     // ws_estimate_multi: expanded configurations (grow-only)
  size_t xcfg_cap = 0;
  // tracing
  bool profiling = false;
  struct Rec {
    int first_kind, n;
    std::vector<cudaEvent_t> ev;
    uint32_t skip = 0;  // kinds (bit i = first_kind + i) whose events this call never records
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> free_ev;
  // aux streams + fork/join events for the concurrent worker chains
  cudaStream_t aux[2] = {nullptr, nullptr};
  cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr}, scanned = nullptr;
  // CUDA graph of the whole estimate launch sequence, captured on `cap` and replayed on
  // `stream` while the launch arguments (key) are unchanged
  struct GKey {
    const void *cfgs, *out, *scratch, *dk, *dg;
    size_t n;
    int nk, ng;
    uint64_t fan;       // ws_estimate_multi: hash of the fan-out descriptor (0 = plain estimate)
    const void* xcfg;   // its expanded-configuration buffer
    const void* top;    // ws_estimate_ranked_async: top-k buffer and k (rank_k = -1: no ranking tail)
    long long rank_k;
    bool operator==(const GKey& o) const {
      return cfgs == o.cfgs && out == o.out && scratch == o.scratch && dk == o.dk && dg == o.dg && n == o.n &&
             nk == o.nk && ng == o.ng && fan == o.fan && xcfg == o.xcfg && top == o.top && rank_k == o.rank_k;
    }
  };
  cudaStream_t cap = nullptr;
  // captured estimate graphs, keyed by everything a capture bakes in (buffers, scratch, descriptor
  // counts, fan-out, ranking): a few kept so that callers alternating buffers (double buffering)
  // replay instead of re-capturing; round-robin replacement
  struct GEntry {
    cudaGraphExec_t exec = nullptr;
    GKey key{};
    uint32_t launches = 0;
    int tail_done = 0;   // the captured graph's k_model also ranks (ws_estimate_ranked_async)
  };
  static constexpr int kGraphCache = 4;
  GEntry gcache[kGraphCache];
  int gnext = 0;
  void* wclean_ptr = nullptr;   // warp-class counter region known to be zero (ensure_scratch)
  size_t wclean_n = 0;
  bool graphs = true;
  // 2 events (start, end) per kernel kind, kinds [first_kind, first_kind + nk)
  cudaEvent_t* take_events(int first_kind, int nk) {
    Rec r;
    r.first_kind = first_kind;
    r.n = nk;
    for (int i = 0; i < 2 * nk; ++i) {
      cudaEvent_t e;
      if (!free_ev.empty()) {
        e = free_ev.back();
        free_ev.pop_back();
      } else if (cudaEventCreate(&e) != cudaSuccess) {
        for (cudaEvent_t x : r.ev) free_ev.push_back(x);
        return nullptr;
      }
      r.ev.push_back(e);
    }
    pending.push_back(std::move(r));
    return pending.back().ev.data();
  }
};

namespace {

ws_status fail(ws_ctx* c, ws_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}
ws_status cuda_fail(ws_ctx* c, cudaError_t e, const char* where) {
  return fail(c, WS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
int lg2(uint64_t v) {  // exact log2 or -1
  if (v == 0 || (v & (v - 1))) return -1;
  int l = 0;
  while ((1ull << l) < v) ++l;
  return l;
}

ws_status upload(ws_ctx* c) {
  if (!c->dirty) return WS_OK;
  cudaError_t e;
  if (c->hk.size() > c->cap_k) {
    if (c->dk) cudaFree(c->dk);
    c->cap_k = std::max<size_t>(c->hk.size() * 2, 4);
    if ((e = cudaMalloc(&c->dk, c->cap_k * sizeof(DKernel))) != cudaSuccess) return cuda_fail(c, e, "cudaMalloc kernels");
  }
  if (c->hg.size() > c->cap_g) {
    if (c->dg) cudaFree(c->dg);
    c->cap_g = std::max<size_t>(c->hg.size() * 2, 4);
    if ((e = cudaMalloc(&c->dg, c->cap_g * sizeof(DGpu))) != cudaSuccess) return cuda_fail(c, e, "cudaMalloc gpus");
  }
  if (!c->hk.empty() &&
      (e = cudaMemcpyAsync(c->dk, c->hk.data(), c->hk.size() * sizeof(DKernel), cudaMemcpyHostToDevice, c->stream)) !=
          cudaSuccess)
    return cuda_fail(c, e, "upload kernels");
  if (!c->hg.empty() &&
      (e = cudaMemcpyAsync(c->dg, c->hg.data(), c->hg.size() * sizeof(DGpu), cudaMemcpyHostToDevice, c->stream)) !=
          cudaSuccess)
    return cuda_fail(c, e, "upload gpus");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "upload sync");
  c->dirty = false;
  return WS_OK;
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }
constexpr size_t kMaxBatch = size_t(1) << 24;

// grow-only device buffer owned by the context (the old contents are not kept)
ws_status grow(ws_ctx* c, void*& p, size_t& cap, size_t need, const char* what) {
  if (need <= cap) return WS_OK;
  if (p) {
    cudaStreamSynchronize(c->stream);   // in-flight work may still read the old buffer
    cudaFree(p);
  }
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&p, need);
  if (e != cudaSuccess) return fail(c, WS_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
  cap = need;
  return WS_OK;
}

// Scratch layout for a batch of n configurations; with bytes_only, only its size.
ws_status ensure_scratch(ws_ctx* c, size_t n, Scratch& s, size_t* bytes_only = nullptr) {
  int64_t cb = 1;
  for (int64_t v : c->chunk_bound) cb = std::max(cb, v);
  const size_t max_chunks = n * (size_t)cb;
  size_t off = 0;
  // fixed offsets (survive re-layouts): plan_done, the call epoch, the a5/a6 sharing table
  const size_t o_pdone = off;   off = align_up(off + sizeof(unsigned int));
  const size_t o_epoch = off;   off = align_up(off + sizeof(unsigned long long));
  const size_t o_rctr = off;    off = align_up(off + 16 * sizeof(unsigned long long));
  const size_t o_rtab = off;    off = align_up(off + (size_t)kRowTab * 8 * sizeof(unsigned long long));
  const size_t o_plans = off;   off = align_up(off + n * sizeof(DPlan));
  const size_t o_instr = off;   off = align_up(off + n * (size_t)kMaxInstr * sizeof(DInstr));
  const size_t o_row = off;     off = align_up(off + n * (size_t)kMaxFields * sizeof(DRowInfo));
  const size_t o_acc = off;     off = align_up(off + n * (size_t)A_N * sizeof(unsigned long long));
  const size_t o_pre = off;     off = align_up(off + (n + 1) * sizeof(DPrefix));
  const size_t o_chunk = off;   off = align_up(off + max_chunks * (size_t)kNQ * 3 * sizeof(long long));
  const size_t o_wcnt = off;    off = align_up(off + n * (size_t)kWSlots * sizeof(unsigned int));
  const size_t o_wrep = off;    off = align_up(off + n * (size_t)kWSlots * sizeof(unsigned long long));
  const size_t o_scnt = off;    off = align_up(off + n * (size_t)kSSlots * sizeof(unsigned int));
  const size_t o_srep = off;    off = align_up(off + n * (size_t)kSSlots * sizeof(unsigned long long));
  size_t max_fields = 1;
  for (const DKernel& k : c->hk) max_fields = std::max<size_t>(max_fields, (size_t)k.n_fields);
  const size_t o_spart = off;   off = align_up(off + n * max_fields * kSectSeg * (size_t)kSectPartBytes);
  const size_t o_sdone = off;   off = align_up(off + n * max_fields * sizeof(unsigned int));
  const size_t o_skey = off;    off = align_up(off + (size_t)kShareTab * sizeof(unsigned long long));
  const size_t o_sval = off;    off = align_up(off + (size_t)kShareTab * 2 * sizeof(unsigned long long));
  const size_t o_work = off;    off = align_up(off + 16 * sizeof(unsigned long long));
  static_assert(K_NKINDS <= 16, "work slots");
  const size_t o_lists = off;   off = align_up(off + 8 * sizeof(unsigned long long));
  const size_t o_wlist = off;   off = align_up(off + n * (size_t)kWSlots * sizeof(unsigned long long));
  const size_t o_slist = off;   off = align_up(off + n * (size_t)kSSlots * sizeof(unsigned long long));
  size_t max_nsm = 1;
  for (const DGpu& g : c->hg) max_nsm = std::max<size_t>(max_nsm, g.g.n_sm);
  // direct SM-set items: one per set, or one per multi-member connected component (<= 16 per set)
  const size_t o_dlist = off;   off = align_up(off + n * max_nsm * 16 * sizeof(unsigned long long));
  const size_t o_dmask = off;   off = align_up(off + n * max_nsm * 16 * sizeof(unsigned int));
  const size_t o_gkey = off;    off = align_up(off + n * max_nsm * sizeof(unsigned long long));
  const size_t cdesc_cap = n * (size_t)kCDescPerConfig, cpool_cap = n * (size_t)kCPoolPerConfig;
  const size_t o_cdesc = off;   off = align_up(off + cdesc_cap * sizeof(CDesc));
  const size_t o_cpool = off;   off = align_up(off + cpool_cap * 2 * 24);   // Tri pairs (3 x i64 each)
  const size_t o_citems = off;  off = align_up(off + cpool_cap * sizeof(uint32_t));
  const size_t o_cfb = off;     off = align_up(off + n * (size_t)kSSlots * sizeof(uint32_t));
  const size_t o_clist = off;   off = align_up(off + max_chunks * sizeof(uint32_t));  // k_rows items per config
  const size_t o_ritems = off;  off = align_up(off + max_chunks * sizeof(unsigned long long));
  const size_t o_fitems = off;  off = align_up(off + n * max_fields * sizeof(uint32_t));
  if (bytes_only) {
    *bytes_only = off;
    return WS_OK;
  }
  if (off > c->scratch_cap) {
    if (c->scratch) cudaFree(c->scratch);
    c->scratch = nullptr;
    c->scratch_cap = 0;
    cudaError_t e = cudaMalloc(&c->scratch, off);
    if (e != cudaSuccess) return fail(c, WS_ENOMEM, std::string("device scratch: ") + cudaGetErrorString(e));
    c->scratch_cap = off;
    // counters (k_plan's plan_done) start at 0: zeroed on the context stream (ordered before
    // every later kernel of this context, whatever the stream's flags) and waited for
    e = cudaMemsetAsync(c->scratch, 0, off, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "scratch init");
  }
  char* b = (char*)c->scratch;
  // the warp-class counters are self-cleaning (k_wclass zeroes every slot it consumes): zero the
  // region only when this layout places it somewhere the previous call did not
  if ((void*)(b + o_wcnt) != c->wclean_ptr || n > c->wclean_n) {
    cudaError_t e = cudaMemsetAsync(b + o_wcnt, 0, n * (size_t)kWSlots * sizeof(unsigned int), c->stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "warp-class counters");
    c->wclean_ptr = (void*)(b + o_wcnt);
    c->wclean_n = n;
  }
  s.plans = (DPlan*)(b + o_plans);
  s.instr = (DInstr*)(b + o_instr);
  s.rowinfo = (DRowInfo*)(b + o_row);
  s.acc = (unsigned long long*)(b + o_acc);
  s.prefix = (DPrefix*)(b + o_pre);
  s.chunkres = (long long*)(b + o_chunk);
  s.max_chunks = (int64_t)max_chunks;
  s.wcnt = (unsigned int*)(b + o_wcnt);
  s.wrep = (unsigned long long*)(b + o_wrep);
  s.scnt = (unsigned int*)(b + o_scnt);
  s.srep = (unsigned long long*)(b + o_srep);
  s.skey = (unsigned long long*)(b + o_skey);
  s.spart = (void*)(b + o_spart);
  s.sdone = (unsigned int*)(b + o_sdone);
  s.max_fields = (int32_t)max_fields;
  s.sval = (unsigned long long*)(b + o_sval);
  s.work = (unsigned long long*)(b + o_work);
  s.lists = (unsigned long long*)(b + o_lists);
  s.wlist = (unsigned long long*)(b + o_wlist);
  s.slist = (unsigned long long*)(b + o_slist);
  s.dlist = (unsigned long long*)(b + o_dlist);
  s.dmask = (unsigned int*)(b + o_dmask);
  s.gkey = (unsigned long long*)(b + o_gkey);
  s.cdesc = (void*)(b + o_cdesc);
  s.cpool = (void*)(b + o_cpool);
  s.citems = (uint32_t*)(b + o_citems);
  s.cfbl = (uint32_t*)(b + o_cfb);
  s.cdesc_cap = (int64_t)cdesc_cap;
  s.cpool_cap = (int64_t)cpool_cap;
  s.plan_done = (unsigned int*)(b + o_pdone);
  s.clist = (uint32_t*)(b + o_clist);
  s.clist_stride = (int64_t)cb;
  s.epoch = (unsigned long long*)(b + o_epoch);
  s.rctr = (unsigned long long*)(b + o_rctr);
  s.ritems = (unsigned long long*)(b + o_ritems);
  s.fitems = (uint32_t*)(b + o_fitems);
  s.rowtab = (unsigned long long*)(b + o_rtab);
  c->last_work = s.work;
  return WS_OK;
}

}  // namespace

extern "C" {

ws_status ws_create(int cuda_device, void* cuda_stream, ws_ctx** out) {
  if (!out) return WS_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) return WS_ECUDA;  // no CPU fallback
  if (cuda_device < 0 || cuda_device >= ndev) return WS_EINVAL;
  if (cudaSetDevice(cuda_device) != cudaSuccess) return WS_ECUDA;
  ws_ctx* c = new (std::nothrow) ws_ctx();
  if (!c) return WS_ENOMEM;
  c->device = cuda_device;
  c->stream = (cudaStream_t)cuda_stream;
  c->graphs = !(getenv("WS_GRAPH") && getenv("WS_GRAPH")[0] == '0');
#ifdef WS_CHECK
  c->graphs = false;   // the bounds-check build uploads each call's capacities before its launches
#endif
  cudaDeviceGetAttribute(&c->n_sm_dev, cudaDevAttrMultiProcessorCount, cuda_device);
  if (c->n_sm_dev <= 0) c->n_sm_dev = 148;
  // stream priorities: the row chain (k_rows -> k_fold, the critical path) gets the highest, so
  // its CTAs are scheduled first whenever the concurrent chains compete for SM slots
  // (WS_PRIO=0 disables, diagnostics / A/B)
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  static const int prio_mode = getenv("WS_PRIO") ? atoi(getenv("WS_PRIO")) : 0;
  const int p_rows = prio_mode >= 1 ? prio_hi : prio_lo;
  const int p_set = prio_mode >= 2 ? (prio_hi + prio_lo) / 2 : prio_lo;
  if (cudaStreamCreateWithPriority(&c->aux[0], cudaStreamNonBlocking, p_set) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->aux[1], cudaStreamNonBlocking, p_rows) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->join[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->join[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->scanned, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess) {
    ws_destroy(c);
    return WS_ECUDA;
  }
  *out = c;
  return WS_OK;
}

void ws_destroy(ws_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->dk) cudaFree(c->dk);
  if (c->dg) cudaFree(c->dg);
  if (c->scratch) cudaFree(c->scratch);
  if (c->io) cudaFree(c->io);
  if (c->rank_buf) cudaFree(c->rank_buf);
  if (c->rank_io) cudaFree(c->rank_io);
  if (c->xcfg) cudaFree(c->xcfg);
  c->sim_cache.release();
  for (auto& r : c->pending)
    for (cudaEvent_t e : r.ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->free_ev) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (c->aux[i]) cudaStreamDestroy(c->aux[i]);
    if (c->join[i]) cudaEventDestroy(c->join[i]);
  }
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->scanned) cudaEventDestroy(c->scanned);
  for (auto& ge : c->gcache)
    if (ge.exec) cudaGraphExecDestroy(ge.exec);
  if (c->cap) cudaStreamDestroy(c->cap);
  delete c;
}

const char* ws_last_error(const ws_ctx* c) { return c ? c->err.c_str() : "null context"; }

ws_status ws_set_stream(ws_ctx* c, void* s) {
  if (!c) return WS_EINVAL;
  if ((cudaStream_t)s == c->stream) return WS_OK;
  cudaSetDevice(c->device);
  // the scratch, io buffers and graph are shared: work issued on the new stream is ordered
  // after everything already enqueued on the old one
  cudaEvent_t e = nullptr;
  cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (r == cudaSuccess) r = cudaEventRecord(e, c->stream);
  if (r == cudaSuccess) r = cudaStreamWaitEvent((cudaStream_t)s, e, 0);
  if (e) cudaEventDestroy(e);
  if (r != cudaSuccess) return cuda_fail(c, r, "set_stream");
  c->stream = (cudaStream_t)s;
  return WS_OK;
}

uint32_t ws_last_launch_count(const ws_ctx* c) { return c ? c->last_launches : 0; }

static const char* kKindNames[K_NKINDS] = {"k_plan",   "k_instr", "k_warp",  "k_wclass", "k_smset",
                                           "k_sclass", "k_rows",  "k_fold",  "k_sect",   "k_model",
                                           "k_rank",   "k_simgen", "k_simrun", "k_fit"};

const char* ws_kernel_name(uint32_t i) { return i < (uint32_t)K_NKINDS ? kKindNames[i] : nullptr; }

ws_status ws_profile_enable(ws_ctx* c, int on) {
  if (!c) return WS_EINVAL;
  c->profiling = on != 0;
  return WS_OK;
}

ws_status ws_profile_read(ws_ctx* c, double* ms, uint64_t* launches, uint32_t cap, uint32_t* n_kinds) {
  if (!c) return WS_EINVAL;
  cudaSetDevice(c->device);
  std::vector<double> acc(K_NKINDS, 0.0);
  std::vector<uint64_t> cnt(K_NKINDS, 0);
  ws_status st = WS_OK;
  for (auto& r : c->pending) {
    for (int i = 0; i < r.n; ++i) {
      if ((r.skip >> i) & 1u) continue;
      float t = 0.f;
      cudaError_t e = cudaEventSynchronize(r.ev[2 * i + 1]);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.ev[2 * i], r.ev[2 * i + 1]);
      if (e == cudaErrorInvalidResourceHandle) {  // kind not launched by this call (events never recorded)
        cudaGetLastError();
        continue;
      }
      if (e != cudaSuccess) st = cuda_fail(c, e, "profile read");
      acc[r.first_kind + i] += t;
      cnt[r.first_kind + i] += 1;
    }
    for (cudaEvent_t e : r.ev) c->free_ev.push_back(e);
  }
  c->pending.clear();
  for (uint32_t i = 0; i < cap && i < (uint32_t)K_NKINDS; ++i) {
    if (ms) ms[i] = acc[i];
    if (launches) launches[i] = cnt[i];
  }
  if (n_kinds) *n_kinds = K_NKINDS;
  return st;
}

ws_status ws_work_read(ws_ctx* c, uint64_t* units, uint32_t cap) {
  if (!c || !units) return WS_EINVAL;
  cudaSetDevice(c->device);
  unsigned long long h[16] = {0};
  if (c->last_work) {
    cudaError_t e = cudaMemcpyAsync(h, c->last_work, sizeof(h), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "work read");
  }
  for (uint32_t i = 0; i < cap && i < 16; ++i) units[i] = h[i];
  return WS_OK;
}

ws_status ws_describe_kernel(ws_ctx* c, const ws_kernel* k, uint32_t* id) {
  if (!c || !k || !id) return fail(c, WS_EINVAL, "null argument");
  if (k->n_fields < 1 || k->n_fields > (uint32_t)kMaxFields || k->n_accesses < 1 || k->n_accesses > (uint32_t)kMaxAcc ||
      !k->fields || !k->accesses)
    return fail(c, WS_EINVAL, "n_fields must be 1..64 and n_accesses 1..128");
  DKernel D;
  memset(&D, 0, sizeof(D));
  D.n_fields = (int)k->n_fields;
  D.n_acc = (int)k->n_accesses;
  D.regs = (int)k->regs_per_thread;
  D.flops = k->flops_per_lup;
  D.cells = 1.0;
  for (int d = 0; d < 3; ++d) {
    if (k->dom_lo[d] < 0 || k->dom_hi[d] <= k->dom_lo[d]) return fail(c, WS_EINVAL, "empty or negative domain");
    D.lo[d] = k->dom_lo[d];
    D.hi[d] = k->dom_hi[d];
    D.cells *= (double)(k->dom_hi[d] - k->dom_lo[d]);
  }
  for (uint32_t i = 0; i < k->n_fields; ++i) {
    const ws_field& F = k->fields[i];
    DField& G = D.f[i];
    const int le = lg2(F.elem_bytes);
    if (le < 0 || F.elem_bytes > 32) return fail(c, WS_EINVAL, "elem_bytes must be a power of two <= 32");
    // an element never straddles a sector, so the alignment is a multiple of elem_bytes
    if (F.align_bytes & (int64_t)(F.elem_bytes - 1))
      return fail(c, WS_EINVAL, "align_bytes must be a multiple of elem_bytes");
    for (int d = 0; d < 3; ++d)
      if (F.extent[d] < 1) return fail(c, WS_EINVAL, "field extent < 1");
    if (F.pitch[0] != 1 || F.pitch[1] < F.extent[0] || F.pitch[2] < F.pitch[1] * F.extent[1])
      return fail(c, WS_EINVAL, "layout: need pitch[0]==1, pitch[1]>=extent[0], pitch[2]>=pitch[1]*extent[1]");
    // plane-relative 32-bit unit arithmetic adds < 2 lines (<= 8 KiB) to in-plane offsets
    if ((F.pitch[2] * (int64_t)F.elem_bytes) > (int64_t(1) << 31) - (int64_t(1) << 14) || F.extent[2] >= (int64_t(1) << 31))
      return fail(c, WS_ELIMIT, "a z-plane of a field must be at most 2 GiB - 16 KiB");
    for (int d = 0; d < 3; ++d) {
      G.ext[d] = F.extent[d];
      G.pitch[d] = F.pitch[d];
    }
    G.align = F.align_bytes;
    G.lg_elem = le;
  }
  for (uint32_t i = 0; i < k->n_accesses; ++i) {
    const ws_access& A = k->accesses[i];
    if (A.field >= k->n_fields || A.is_store > 1) return fail(c, WS_EINVAL, "access: bad field index or kind");
    const ws_field& F = k->fields[A.field];
    for (int d = 0; d < 3; ++d)
      if (k->dom_lo[d] + A.off[d] < 0 || k->dom_hi[d] - 1 + A.off[d] >= F.extent[d])
        return fail(c, WS_EBOUNDS, "access leaves its field for an active cell");
    D.acc[i] = A;
  }
  // groups: (field, kind, oy, oz) -> maximal runs of consecutive ox
  int ng = 0;
  int64_t chunks = 0;
  for (int fi = 0; fi < D.n_fields; ++fi) {
    DField& G = D.f[fi];
    G.g_begin = ng;
    std::vector<std::pair<int, int>> runs;
    G.oy_min = G.oz_min = G.ld_oy_min = G.ld_oz_min = 1 << 30;
    G.oy_max = G.oz_max = G.ld_oy_max = G.ld_oz_max = -(1 << 30);
    for (int kind = 0; kind < 2; ++kind) {
      std::map<std::pair<int, int>, std::set<int>> byrow;
      for (int i = 0; i < D.n_acc; ++i)
        if ((int)D.acc[i].field == fi && (int)D.acc[i].is_store == kind)
          byrow[{D.acc[i].off[1], D.acc[i].off[2]}].insert(D.acc[i].off[0]);
      for (auto& kv : byrow) {
        std::vector<int> xs(kv.second.begin(), kv.second.end());
        size_t a = 0;
        while (a < xs.size()) {
          size_t b = a;
          while (b + 1 < xs.size() && xs[b + 1] == xs[b] + 1) ++b;
          std::pair<int, int> run(xs[a], xs[b]);
          int ri = -1;
          for (size_t q = 0; q < runs.size(); ++q)
            if (runs[q] == run) ri = (int)q;
          if (ri < 0) {
            if ((int)runs.size() >= kMaxRuns) return fail(c, WS_ELIMIT, "more than 16 distinct x-offset runs in a field");
            ri = (int)runs.size();
            runs.push_back(run);
          }
          DGroup gr;
          gr.field = fi;
          gr.kind = kind;
          gr.oy = kv.first.first;
          gr.oz = kv.first.second;
          gr.run = ri;
          gr.pad = 0;
          D.g[ng++] = gr;
          G.oy_min = std::min(G.oy_min, gr.oy);
          G.oy_max = std::max(G.oy_max, gr.oy);
          G.oz_min = std::min(G.oz_min, gr.oz);
          G.oz_max = std::max(G.oz_max, gr.oz);
          if (kind == 0) {
            G.n_ld_groups++;
            G.ld_oy_min = std::min(G.ld_oy_min, gr.oy);
            G.ld_oy_max = std::max(G.ld_oy_max, gr.oy);
            G.ld_oz_min = std::min(G.ld_oz_min, gr.oz);
            G.ld_oz_max = std::max(G.ld_oz_max, gr.oz);
          }
          G.kinds |= 1 << kind;
          a = b + 1;
        }
      }
    }
    G.g_end = ng;
    G.oz_mask = 0;
    if (G.g_end > G.g_begin && G.oz_max - G.oz_min < 64)
      for (int q = G.g_begin; q < G.g_end; ++q) G.oz_mask |= 1ull << (D.g[q].oz - G.oz_min);
    G.n_runs = (int)runs.size();
    for (size_t q = 0; q < runs.size(); ++q) {
      G.run_lo[q] = runs[q].first;
      G.run_hi[q] = runs[q].second;
    }
    // k_rows chunks: (z-plane, segment of kRowSeg rows) of the field's row box
    if (G.g_end > G.g_begin) chunks += G.ext[2] * ((G.ext[1] + kRowSeg - 1) / kRowSeg);
  }
  D.n_groups = ng;
  {
    DLoadEnv& E = D.env;
    E.spy = E.spz = 0;
    E.oy_min = E.ext1_min = E.row_bytes_min = E.plane_bytes_min = INT64_MAX;
    E.oy_max = INT64_MIN;
    E.has_load = 0;
    E.n_ld = 0;
    E.max_lg_elem = 0;
    E.same_layout = 1;
    E.pad2 = E.pad3 = 0;
    for (int fi = 0; fi < D.n_fields; ++fi) {
      E.max_lg_elem = std::max(E.max_lg_elem, D.f[fi].lg_elem);
      for (int d = 0; d < 3; ++d)
        if (D.f[fi].pitch[d] != D.f[0].pitch[d] || D.f[fi].lg_elem != D.f[0].lg_elem) E.same_layout = 0;
    }
    for (int fi = 0; fi < D.n_fields; ++fi) {
      const DField& F = D.f[fi];
      if (!(F.kinds & 1)) continue;
      E.has_load = 1;
      E.n_ld++;
      E.spy = std::max<int64_t>(E.spy, F.ld_oy_max - F.ld_oy_min);
      E.spz = std::max<int64_t>(E.spz, F.ld_oz_max - F.ld_oz_min);
      E.oy_min = std::min<int64_t>(E.oy_min, F.ld_oy_min);
      E.oy_max = std::max<int64_t>(E.oy_max, F.ld_oy_max);
      E.ext1_min = std::min<int64_t>(E.ext1_min, F.ext[1]);
      E.row_bytes_min = std::min<int64_t>(E.row_bytes_min, F.pitch[1] << F.lg_elem);
      E.plane_bytes_min = std::min<int64_t>(E.plane_bytes_min, F.pitch[2] << F.lg_elem);
    }
  }
  c->hk.push_back(D);
  c->chunk_bound.push_back(chunks);
  c->dirty = true;
  *id = (uint32_t)(c->hk.size() - 1);
  return WS_OK;
}

ws_status ws_describe_gpu(ws_ctx* c, const ws_gpu* g, uint32_t* id) {
  if (!c || !g || !id) return fail(c, WS_EINVAL, "null argument");
  DGpu D;
  memset(&D, 0, sizeof(D));
  D.g = *g;
  D.lg_sector = lg2(g->sector_bytes);
  D.lg_line = lg2(g->line_bytes);
  D.lg_bank = lg2(g->bank_bytes);
  D.lg_hw = lg2(g->half_warp);
  D.lg_nbanks = lg2(g->n_banks);
  if (g->n_sm < 1 || g->max_thr_sm < 1 || g->max_blk_sm < 1 || g->max_thr_blk < 1 || g->regs_sm < 1)
    return fail(c, WS_EINVAL, "occupancy limits must be >= 1");
  if (D.lg_sector < 0 || D.lg_line < 0 || D.lg_line < D.lg_sector || D.lg_bank < 0 || D.lg_hw < 0 || g->half_warp > 32 ||
      D.lg_nbanks < 0 || g->n_banks > 256)
    return fail(c, WS_EINVAL, "sector/line/bank/half-warp geometry must be powers of two (line >= sector, half_warp <= 32)");
  if (g->line_bytes > 4096) return fail(c, WS_ELIMIT, "line_bytes must be <= 4096");
  if (g->pair_window_bytes < 1 || g->l2_sections < 1 || g->l1_bytes < 1 || g->l2_bytes < 1)
    return fail(c, WS_EINVAL, "cache sizes / window must be >= 1");
  if (!(g->clock_hz > 0) || !(g->dram_bw > 0) || !(g->l2_bw > 0)) return fail(c, WS_EINVAL, "rates must be > 0");
  if (!(g->link_bw >= 0) || g->link_bw > 1e30) return fail(c, WS_EINVAL, "link_bw must be >= 0 and finite");
  D.lg_page = g->page_bytes ? lg2(g->page_bytes) : -1;
  if (g->page_bytes && (D.lg_page < 0 || g->page_bytes < g->line_bytes || D.lg_page > 40))
    return fail(c, WS_EINVAL, "page_bytes must be 0 or a power of two >= line_bytes (<= 2^40)");
  if (g->l2_sections > (uint32_t)kMaxSections) return fail(c, WS_ELIMIT, "l2_sections must be <= 4");
  c->hg.push_back(D);
  c->dirty = true;
  *id = (uint32_t)(c->hg.size() - 1);
  return WS_OK;
}

static ws_status estimate_launch(ws_ctx* c, const ws_config* d_cfgs, size_t n, ws_result* d_out, bool allow_graph,
                                 const FanOut* fan, TailRank* tail = nullptr);
static size_t chunk_configs(ws_ctx* c, size_t per_item_mult);

ws_status ws_estimate_async(ws_ctx* c, const ws_config* d_cfgs, size_t n, ws_result* d_out) {
  const NvtxRange range("ws_estimate_async");
  if (!c) return WS_EINVAL;
  if (n == 0) return WS_OK;
  if (!d_cfgs || !d_out) return fail(c, WS_EINVAL, "null argument");
  if (n > kMaxBatch) return fail(c, WS_ELIMIT, "batch larger than 2^24 configurations");
  if (c->hk.empty() || c->hg.empty()) return fail(c, WS_EUNKNOWN_ID, "describe a kernel and a gpu first");
  cudaSetDevice(c->device);
  ws_status s = upload(c);
  if (s != WS_OK) return s;
  const size_t chunk = chunk_configs(c, 1);   // bounded scratch (see chunk_configs)
  if (n <= chunk) return estimate_launch(c, d_cfgs, n, d_out, true, nullptr);
  uint32_t launches = 0;
  for (size_t off = 0; off < n; off += chunk) {
    s = estimate_launch(c, d_cfgs + off, std::min(chunk, n - off), d_out + off, false, nullptr);
    if (s != WS_OK) return s;
    launches += c->last_launches;
  }
  c->last_launches = launches;
  return WS_OK;
}

ws_status ws_estimate_ranked_async(ws_ctx* c, const ws_config* d_cfgs, size_t n, ws_result* d_out, size_t k,
                                   uint32_t* d_top) {
  const NvtxRange range("ws_estimate_ranked_async");
  if (!c) return WS_EINVAL;
  if (n == 0) return WS_OK;
  if (!d_cfgs || !d_out) return fail(c, WS_EINVAL, "null argument");
  if (n > kMaxBatch) return fail(c, WS_ELIMIT, "batch larger than 2^24 configurations");
  if (c->hk.empty() || c->hg.empty()) return fail(c, WS_EUNKNOWN_ID, "describe a kernel and a gpu first");
  cudaSetDevice(c->device);
  ws_status s = upload(c);
  if (s != WS_OK) return s;
  TailRank tail{(int)std::min(k, n), d_top, 0};
  if (n <= (size_t)kTailMax && n <= chunk_configs(c, 1)) {
    s = estimate_launch(c, d_cfgs, n, d_out, true, nullptr, &tail);
    if (s != WS_OK || tail.done) return s;
  } else {
    s = ws_estimate_async(c, d_cfgs, n, d_out);
    if (s != WS_OK) return s;
  }
  const uint32_t le = c->last_launches;
  s = ws_rank_async(c, d_out, n, k, d_top);
  c->last_launches += le;
  return s;
}

static uint64_t fan_hash(const FanOut* f) {  // FNV-1a over the fan-out descriptor (graph key)
  if (!f) return 0;
  uint64_t h = 1469598103934665603ull;
  const unsigned char* p = (const unsigned char*)f;
  for (size_t i = 0; i < sizeof(FanOut); ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h | 1;
}

// One launch sequence of the estimator over n configurations (fan == nullptr), or, for
// ws_estimate_multi, over fan->m configurations x fan->n_groups representative hardware sets
// with the model fanned out to fan->n_gpu sets (d_cfgs: the caller's configurations).
static ws_status estimate_launch(ws_ctx* c, const ws_config* d_cfgs, size_t n, ws_result* d_out, bool allow_graph,
                                 const FanOut* fan, TailRank* tail) {
  ws_status s;
  Scratch S;
  const size_t n_int = fan ? (size_t)fan->m * fan->n_groups : n;
  if ((s = ensure_scratch(c, n_int, S)) != WS_OK) return s;
  ws_config* xcfg = nullptr;
  if (fan) {
    if ((s = grow(c, c->xcfg, c->xcfg_cap, n_int * sizeof(ws_config), "expanded configurations")) != WS_OK) return s;
    xcfg = (ws_config*)c->xcfg;
  }
  const ws_config* icfg = fan ? xcfg : d_cfgs;
  cudaEvent_t* ev = c->profiling ? c->take_events(K_PLAN, kEstimateKernels) : nullptr;
  Streams st;
  st.main = c->stream;
  // WS_SERIAL=1 (diagnostics): every chain on the context stream -> uncontended kernel times
  static const bool serial = getenv("WS_SERIAL") && getenv("WS_SERIAL")[0] == '1';
  st.aux[0] = serial ? c->stream : c->aux[0];
  st.aux[1] = serial ? c->stream : c->aux[1];
  st.fork = c->fork;
  st.join[0] = c->join[0];
  st.join[1] = c->join[1];
  st.scanned = c->scanned;
  auto enqueue = [&](uint32_t* launches, cudaEvent_t* evs) -> int {
    uint32_t extra = 0;
    if (fan) {
      const int e0 = launch_expand(d_cfgs, *fan, xcfg, st.main);
      if (e0) return e0;
      extra = 1;
    }
    const int e1 = launch_estimate(icfg, (int)n_int, c->dk, (int)c->hk.size(), c->dg, (int)c->hg.size(), S, d_out, st,
                                   c->n_sm_dev, launches, evs, fan, tail);
    if (launches) *launches += extra;
    return e1;
  };
  // graph replay unless profiling (per-kernel events), serial diagnostics, or the caller's
  // stream is itself being captured (then the launches become part of the caller's graph)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  if (allow_graph && c->graphs && !ev && !serial && cs == cudaStreamCaptureStatusNone) {
    const ws_ctx::GKey key{d_cfgs, d_out, c->scratch, c->dk, c->dg, n, (int)c->hk.size(), (int)c->hg.size(),
                           fan_hash(fan), xcfg, tail ? (const void*)tail->top : nullptr,
                           tail ? (long long)tail->k : -1ll};
    int hit = -1;
    for (int i = 0; i < ws_ctx::kGraphCache; ++i)
      if (c->gcache[i].exec && c->gcache[i].key == key) hit = i;
    if (hit < 0) {
      hit = c->gnext;
      c->gnext = (c->gnext + 1) % ws_ctx::kGraphCache;
      ws_ctx::GEntry& ge = c->gcache[hit];
      if (ge.exec) {
        cudaGraphExecDestroy(ge.exec);
        ge.exec = nullptr;
      }
      st.main = c->cap;
      cudaError_t e = cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return cuda_fail(c, e, "graph capture");
      enqueue(&ge.launches, nullptr);
      cudaGraph_t g = nullptr;
      e = cudaStreamEndCapture(c->cap, &g);
      if (e == cudaSuccess) e = cudaGraphInstantiate(&ge.exec, g, 0);
      if (g) cudaGraphDestroy(g);
      if (e != cudaSuccess) {
        ge.exec = nullptr;
        return cuda_fail(c, e, "graph instantiate");
      }
      ge.key = key;
      ge.tail_done = tail ? tail->done : 0;
    }
    const ws_ctx::GEntry& ge = c->gcache[hit];
    if (tail) tail->done = ge.tail_done;
    cudaError_t e = cudaGraphLaunch(ge.exec, c->stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "graph launch");
    c->last_launches = ge.launches;
    return WS_OK;
  }
  int e = enqueue(&c->last_launches, ev);
  if (e) return cuda_fail(c, (cudaError_t)e, "launch");
  return WS_OK;
}

// Per-configuration scratch bytes and the chunk size that keeps the scratch within the budget
// (WS_SCRATCH_MB, default 4096): larger batches run as consecutive chunks on the same stream
// (results identical: configurations are independent; chunks use direct launches).
static size_t chunk_configs(ws_ctx* c, size_t per_item_mult) {
  Scratch S0;
  size_t b1 = 0, b2 = 0;
  ensure_scratch(c, 1, S0, &b1);
  ensure_scratch(c, 2, S0, &b2);
  const size_t per = std::max<size_t>(1, b2 - b1) * per_item_mult, fixed = b1 > per ? b1 - per : 0;
  static const size_t budget = (getenv("WS_SCRATCH_MB") ? (size_t)atoll(getenv("WS_SCRATCH_MB")) : 4096) << 20;
  return budget > fixed + per ? (budget - fixed) / per : 1;
}

// Integer-stage key of a hardware set: every ws_gpu parameter the kernels before the model read
// (occupancy limits, SM count, sector / line / bank geometry, sections, pages, link on/off).
static bool same_integer_stage(const DGpu& a, const DGpu& b) {
  const ws_gpu &x = a.g, &y = b.g;
  return x.n_sm == y.n_sm && x.max_thr_sm == y.max_thr_sm && x.max_blk_sm == y.max_blk_sm &&
         x.max_thr_blk == y.max_thr_blk && x.regs_sm == y.regs_sm && x.sector_bytes == y.sector_bytes &&
         x.line_bytes == y.line_bytes && x.n_banks == y.n_banks && x.bank_bytes == y.bank_bytes &&
         x.half_warp == y.half_warp && x.pair_window_bytes == y.pair_window_bytes && x.l2_sections == y.l2_sections &&
         x.page_bytes == y.page_bytes && (x.link_bw > 0) == (y.link_bw > 0);
}

ws_status ws_estimate(ws_ctx* c, const ws_config* cfgs, size_t n, ws_result* out) {
  if (!c) return WS_EINVAL;
  if (n == 0) return WS_OK;
  if (!cfgs || !out) return fail(c, WS_EINVAL, "null argument");
  cudaSetDevice(c->device);
  const size_t need = align_up(n * sizeof(ws_config)) + n * sizeof(ws_result);
  cudaError_t e;
  if (need > c->io_cap) {
    if (c->io) cudaFree(c->io);
    c->io = nullptr;
    c->io_cap = 0;
    if ((e = cudaMalloc(&c->io, need)) != cudaSuccess) return fail(c, WS_ENOMEM, "device io buffer");
    c->io_cap = need;
  }
  ws_config* dc = (ws_config*)c->io;
  ws_result* dr = (ws_result*)((char*)c->io + align_up(n * sizeof(ws_config)));
  if ((e = cudaMemcpyAsync(dc, cfgs, n * sizeof(ws_config), cudaMemcpyHostToDevice, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "H2D configs");
  ws_status s = ws_estimate_async(c, dc, n, dr);
  if (s != WS_OK) return s;
  if ((e = cudaMemcpyAsync(out, dr, n * sizeof(ws_result), cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "D2H results");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "estimate");
  return WS_OK;
}

ws_status ws_estimate_multi_async(ws_ctx* c, const ws_config* d_cfgs, size_t n, const uint32_t* gpu_ids,
                                  uint32_t n_gpu, ws_result* d_out) {
  const NvtxRange range("ws_estimate_multi_async");
  if (!c) return WS_EINVAL;
  if (n == 0 || n_gpu == 0) return WS_OK;
  if (!d_cfgs || !d_out || !gpu_ids) return fail(c, WS_EINVAL, "null argument");
  if (n_gpu > (uint32_t)kMaxFanGpus) return fail(c, WS_ELIMIT, "at most 256 hardware sets per call");
  if (n * n_gpu > kMaxBatch) return fail(c, WS_ELIMIT, "n * n_gpu larger than 2^24 records");
  if (c->hk.empty() || c->hg.empty()) return fail(c, WS_EUNKNOWN_ID, "describe a kernel and a gpu first");
  for (uint32_t g = 0; g < n_gpu; ++g)
    if (gpu_ids[g] >= c->hg.size()) return fail(c, WS_EUNKNOWN_ID, "gpu_ids: id not described in this context");
  cudaSetDevice(c->device);
  ws_status s = upload(c);
  if (s != WS_OK) return s;
  FanOut f;
  memset(&f, 0, sizeof(f));
  f.n = (int32_t)n;
  f.n_gpu = (int32_t)n_gpu;
  for (uint32_t g = 0; g < n_gpu; ++g) {
    int grp = -1;
    for (int j = 0; j < f.n_groups && grp < 0; ++j)
      if (same_integer_stage(c->hg[f.rep[j]], c->hg[gpu_ids[g]])) grp = j;
    if (grp < 0) {
      grp = f.n_groups++;
      f.rep[grp] = gpu_ids[g];
    }
    f.group[g] = (uint16_t)grp;
    f.gid[g] = (uint16_t)gpu_ids[g];
  }
  c->last_groups = (uint32_t)f.n_groups;
  const size_t chunk = chunk_configs(c, (size_t)f.n_groups);
  uint32_t launches = 0;
  for (size_t off = 0; off < n; off += chunk) {
    f.i0 = (int32_t)off;
    f.m = (int32_t)std::min(chunk, n - off);
    s = estimate_launch(c, d_cfgs, n, d_out, n <= chunk, &f);
    if (s != WS_OK) return s;
    launches += c->last_launches;
  }
  c->last_launches = launches;
  return WS_OK;
}

ws_status ws_estimate_multi(ws_ctx* c, const ws_config* cfgs, size_t n, const uint32_t* gpu_ids, uint32_t n_gpu,
                            ws_result* out) {
  if (!c) return WS_EINVAL;
  if (n == 0 || n_gpu == 0) return WS_OK;
  if (!cfgs || !out || !gpu_ids) return fail(c, WS_EINVAL, "null argument");
  if (n * n_gpu > kMaxBatch) return fail(c, WS_ELIMIT, "n * n_gpu larger than 2^24 records");
  cudaSetDevice(c->device);
  const size_t need = align_up(n * sizeof(ws_config)) + n * n_gpu * sizeof(ws_result);
  cudaError_t e;
  ws_status s = grow(c, c->io, c->io_cap, need, "device io buffer");
  if (s != WS_OK) return s;
  ws_config* dc = (ws_config*)c->io;
  ws_result* dr = (ws_result*)((char*)c->io + align_up(n * sizeof(ws_config)));
  if ((e = cudaMemcpyAsync(dc, cfgs, n * sizeof(ws_config), cudaMemcpyHostToDevice, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "H2D configs");
  s = ws_estimate_multi_async(c, dc, n, gpu_ids, n_gpu, dr);
  if (s != WS_OK) return s;
  if ((e = cudaMemcpyAsync(out, dr, n * n_gpu * sizeof(ws_result), cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "D2H results");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return cuda_fail(c, e, "estimate_multi");
  return WS_OK;
}

uint32_t ws_last_group_count(const ws_ctx* c) { return c ? c->last_groups : 0; }

ws_status ws_rank_async(ws_ctx* c, ws_result* d_res, size_t n, size_t k, uint32_t* d_top) {
  const NvtxRange range("ws_rank_async");
  if (!c) return WS_EINVAL;
  if (n == 0) return WS_OK;
  if (!d_res) return fail(c, WS_EINVAL, "null argument");
  if (n > (size_t)kMaxBatch) return fail(c, WS_ELIMIT, "rank: more than 2^24 records");
  cudaSetDevice(c->device);
  ws_status s = grow(c, c->rank_buf, c->rank_cap, rank_scratch_bytes((int)n), "rank scratch");
  if (s != WS_OK) return s;
  cudaEvent_t* ev = c->profiling ? c->take_events(K_RANK, 1) : nullptr;
  int e = launch_rank(d_res, (int)n, (int)std::min(k, n), d_top, c->rank_buf, c->stream, &c->last_launches, ev);
  if (e) return cuda_fail(c, (cudaError_t)e, "rank launch");
  return WS_OK;
}

ws_status ws_check_read(ws_ctx* c, uint64_t* out) {
  if (!c || !out) return WS_EINVAL;
  cudaSetDevice(c->device);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "check read");
  unsigned long long h[5];
  const int r = check_read(h);
  if (r) return cuda_fail(c, (cudaError_t)r, "check read");
  for (int i = 0; i < 5; ++i) out[i] = h[i];
  return WS_OK;
}

ws_status ws_rank(ws_ctx* c, ws_result* res, size_t n, size_t k, uint32_t* top) {
  if (!c) return WS_EINVAL;
  if (n == 0) return WS_OK;
  if (!res) return fail(c, WS_EINVAL, "null argument");
  if (n > (size_t)kMaxBatch) return fail(c, WS_ELIMIT, "rank: more than 2^24 records");
  cudaSetDevice(c->device);
  k = std::min(k, n);
  cudaError_t e;
  const size_t bytes = align_up(n * sizeof(ws_result)) + (k + 1) * sizeof(uint32_t);
  ws_status s0 = grow(c, c->rank_io, c->rank_io_cap, bytes, "rank buffer");   // kept by the context
  if (s0 != WS_OK) return s0;
  void* buf = c->rank_io;
  ws_result* dr = (ws_result*)buf;
  uint32_t* dt = (uint32_t*)((char*)buf + align_up(n * sizeof(ws_result)));
  ws_status s = WS_OK;
  if ((e = cudaMemcpyAsync(dr, res, n * sizeof(ws_result), cudaMemcpyHostToDevice, c->stream)) != cudaSuccess) {
    s = cuda_fail(c, e, "H2D results");
  } else if ((s = ws_rank_async(c, dr, n, k, k ? dt : nullptr)) == WS_OK) {
    if ((e = cudaMemcpyAsync(res, dr, n * sizeof(ws_result), cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
      s = cuda_fail(c, e, "D2H results");
    else if (k && top && (e = cudaMemcpyAsync(top, dt, k * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
      s = cuda_fail(c, e, "D2H top");
    else if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess)
      s = cuda_fail(c, e, "rank");
  }
  return s;
}

ws_status ws_simulate(ws_ctx* c, const ws_config* cfgs, size_t n, const uint64_t* caps, uint32_t n_cap,
                      ws_sim_result* out) {
  const NvtxRange range("ws_simulate");
  if (!c) return WS_EINVAL;
  if (n == 0 || n_cap == 0) return WS_OK;
  if (!cfgs || !caps || !out) return fail(c, WS_EINVAL, "null argument");
  if (n_cap > (uint32_t)kSimMaxCaps) return fail(c, WS_ELIMIT, "at most 64 capacities per call");
  if (n > (size_t)(1 << 20)) return fail(c, WS_ELIMIT, "batch larger than 2^20 configurations");
  if (c->hk.empty() || c->hg.empty()) return fail(c, WS_EUNKNOWN_ID, "describe a kernel and a gpu first");
  cudaSetDevice(c->device);
  ws_status s = upload(c);
  if (s != WS_OK) return s;
  Scratch S;
  if ((s = ensure_scratch(c, n, S)) != WS_OK) return s;
  const size_t need = align_up(n * sizeof(ws_config)) + n * sizeof(ws_result);
  cudaError_t e;
  if (need > c->io_cap) {
    if (c->io) cudaFree(c->io);
    c->io = nullptr;
    c->io_cap = 0;
    if ((e = cudaMalloc(&c->io, need)) != cudaSuccess) return fail(c, WS_ENOMEM, "device io buffer");
    c->io_cap = need;
  }
  ws_config* dc = (ws_config*)c->io;
  ws_result* dr = (ws_result*)((char*)c->io + align_up(n * sizeof(ws_config)));
  if ((e = cudaMemcpyAsync(dc, cfgs, n * sizeof(ws_config), cudaMemcpyHostToDevice, c->stream)) != cudaSuccess)
    return cuda_fail(c, e, "H2D configs");
  Streams st;
  st.main = c->stream;
  st.aux[0] = c->aux[0];
  st.aux[1] = c->aux[1];
  st.fork = c->fork;
  st.join[0] = c->join[0];
  st.join[1] = c->join[1];
  st.scanned = c->scanned;
  cudaEvent_t* ev = nullptr;
  if (c->profiling) {
    ev = c->take_events(K_SIMGEN, 2);
  }
  const int rc = run_simulate(dc, (int)n, c->dk, (int)c->hk.size(), c->dg, (int)c->hg.size(), c->hg, S, dr, st,
                              c->n_sm_dev, caps, (int)n_cap, out, &c->last_launches, ev, c->sim_cache);
  if (rc == -WS_ELIMIT) return fail(c, WS_ELIMIT, "a request stream of 2^31 or more requests");
  if (rc == -WS_EINVAL) return fail(c, WS_EINVAL, "all configurations of a ws_simulate call need one line_bytes");
  if (rc) return cuda_fail(c, (cudaError_t)rc, "simulate");
  return WS_OK;
}

ws_status ws_sim_release(ws_ctx* c) {
  if (!c) return WS_EINVAL;
  cudaSetDevice(c->device);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  c->sim_cache.release();
  return e == cudaSuccess ? WS_OK : cuda_fail(c, e, "sim_release");
}

ws_status ws_fit_gompertz(ws_ctx* c, const double* O, const double* R, size_t n, double abc[3], double* rss) {
  if (!c) return WS_EINVAL;
  if (!O || !R || !abc) return fail(c, WS_EINVAL, "null argument");
  if (n < 3 || n > (size_t)(1 << 20)) return fail(c, WS_EINVAL, "need 3 .. 2^20 samples");
  cudaSetDevice(c->device);
  cudaEvent_t* ev = c->profiling ? c->take_events(K_FIT, 1) : nullptr;
  double out[4];
  const int rc = run_fit(O, R, (int)n, out, c->stream, ev);
  if (rc) return cuda_fail(c, (cudaError_t)rc, "fit");
  abc[0] = out[0];
  abc[1] = out[1];
  abc[2] = out[2];
  if (rss) *rss = out[3];
  c->last_launches = 1;
  return WS_OK;
}

}  // extern "C"
