// ws_internal.cuh -- device-side descriptors shared by ws_api.cu and ws_kernels.cu
// (library-internal; the oracle never sees this file).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include "ws.h"

namespace wsb {

constexpr int kMaxFields = 64;
constexpr int kMaxAcc = 128;
constexpr int kMaxRuns = 16;       // distinct x-offset runs per field (bitmask width of k_rows)
constexpr int kMaxInstr = 1024;    // instructions per thread after fold dedupe
constexpr int kMaxFoldCube = 64;   // prod(fold)
constexpr int kRowThreads = 256;
constexpr int kRowsPerThread = 4;
constexpr int kRowsPerChunk = kRowThreads * kRowsPerThread;
constexpr int kNQ = 9;             // union triples per row chunk (see k_rows)

// x-offset run: all accesses of one (field, kind, oy, oz) whose ox values form a
// maximal run of consecutive integers [lo, hi] ("group").  The union of a
// row interval [x0,x1) shifted by every ox of a run is [x0+lo, x1+hi).
struct DField {
  int64_t ext[3], pitch[3], align;
  int32_t lg_elem, kinds;          // kinds: bit0 = has loads, bit1 = has stores
  int32_t g_begin, g_end;          // this field's groups in DKernel::g
  int32_t n_runs, n_ld_groups;
  int32_t oy_min, oy_max, oz_min, oz_max;  // over all groups of the field
  int32_t ld_oy_min, ld_oy_max, ld_oz_min, ld_oz_max;  // over load groups
  int32_t run_lo[kMaxRuns], run_hi[kMaxRuns];
  uint64_t oz_mask;                // distinct oz of all groups: bit oz - oz_min (0 if oz_max - oz_min > 63)
};

struct DGroup {
  int32_t field, kind, oy, oz, run, pad;
};

// load-offset envelope over the load fields (k_smset's quick separation test)
struct DLoadEnv {
  int64_t spy, spz;                   // max over load fields of ld_oy/oz_max - ld_oy/oz_min
  int64_t oy_min, oy_max, ext1_min;   // min / max load oy, min ext[1]
  int64_t row_bytes_min, plane_bytes_min;
  int32_t has_load, n_ld;             // n_ld: fields with loads
  int32_t max_lg_elem, same_layout;   // over all fields: largest lg_elem; one pitch and element size
  int32_t pad2, pad3;
};
struct DKernel {
  int32_t n_fields, n_acc, n_groups, regs;
  int64_t lo[3], hi[3];
  DLoadEnv env;
  double flops, cells;
  DField f[kMaxFields];
  ws_access acc[kMaxAcc];
  DGroup g[kMaxAcc];
};

struct DGpu {
  ws_gpu g;
  int32_t lg_sector, lg_line, lg_bank, lg_hw, lg_nbanks, lg_page;  // lg_page: -1 = no pages
};
constexpr int kMaxSections = 4;    // L2 sections (k_sect keeps 2 triples per section)

// One per-thread instruction after fold dedupe:
// address = C + (pitch . base) << lg_elem ; issued iff kmask & active_kappas != 0.
struct DInstr {
  int64_t C;
  uint64_t kmask;
  int32_t field, kind, lg_elem, pad;
};

// Row box (field-index rows (y,z), z-major) of the wave + layer-set footprint of one field.
// A chunk is `ppc` consecutive z-planes of the box (k_rows: one warp per chunk).
struct DRowInfo {
  int64_t y0, ny, z0, nz, chunk_begin, n_chunks, ppc, nseg;  // nseg: row segments per plane
};
// k_rows chunk = (plane, segment of kRowSeg rows).  A/B on B200 (configs[1], k_rows serial): 1024
// rows (one segment for every plane of the paper's grids) 78 us, 256: 117 us, 128: 176 us, 64:
// 286 us -- more, smaller items cost more per-item overhead than the runs they spread
#ifndef WS_ROW_SEG
#define WS_ROW_SEG 1024
#endif
constexpr int kRowSeg = WS_ROW_SEG;
constexpr int kPlaneRows = 8192;   // target rows per k_rows chunk

// One contiguous block-id range [a, b) seen per block row: first / last block row touched and the
// four cell x-intervals it can cover in a row (FULL, SUFFIX, PREFIX, MIDDLE).
struct RangeInfo {
  int64_t ra, rl;
  int64_t iv[4][2];
  int32_t nonempty, pad;
};

// n / d for 0 <= n < 2^31 by multiply-high (Granlund-Montgomery round-up method):
// q = (umulhi(n, m) + n) >> l with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1.
struct FDiv {
  uint32_t m, l;
};

struct DPlan {
  int32_t status, kid, gid, n_instr;
  int32_t b[3], f[3];
  int32_t T, nwarps, k, fcube;
  int64_t lo[3], hi[3], G[3], BF[3];
  int64_t N, W, s, nsets, Ly0, Lz0;
  // translation classes: 0 = disabled
  int32_t wcls_R, scls_R;        // residue slots per warp index / per SM set
  int64_t cls_pitch[3];          // the common pitch of every field when classes are enabled
  int32_t cls_lg_elem, wpow2;    // wpow2: power-of-two block dims and T % 32 == 0
  int64_t n_warp_items, n_wclass_items, n_set_items, n_sclass_items, n_chunks, n_fields;
  uint64_t addr_evals;
  FDiv fd_BF[3];                 // division by BF[d] (cell -> block coordinate)
  int64_t part[3];               // extent of a partial last block per dim (0 = none)
  // k_rows: ranges 0 = wave, 1 = L_y, 2 = L_z, 3 = L_y + wave, 4 = L_z + wave, and the sorted
  // distinct block rows where some range's classification zone starts
  RangeInfo rng[5];
  int64_t bnd[20];
  int32_t nb, pad3;
  // model variants (ws_config.variant) and the outlook metrics (NEXT-3 / NEXT-4)
  int32_t variant, mdim;         // mdim: wave / layer-set footprints in the multidimensional space
  int32_t want_pages, want_sect; // k_sect: TLB pages / L2-section footprints wanted
  int64_t n_sect_items;          // k_sect work items (fields) of this config
  int64_t rep_B, rep_mult;       // WS_VAR_REP_BLOCK: the representative block and W (0 = off)
  // a5/a6 sharing: configurations with identical wave / layer-set footprints (same kernel, sector
  // and line geometry, block footprint BF, W, s, L_y, L_z, address space) have identical row-scope
  // counts; the first to claim the key in the row table computes them, the others (row_owner !=
  // own index) have no k_rows / k_fold work and k_model reads the owner's accumulators
  int32_t row_owner, row_slot;
  int32_t istat, pad5;           // k_instr: WS_ELIMIT when the instruction table overflows (else 0)
  // k_rows items: the chunks of computed planes only (derived planes -- translates of their zone
  // segment's representative by whole lines -- are folded by k_fold from the representative)
  int64_t n_ritems, chunk_base;  // chunk_base: this configuration's first slot in chunkres (owners)
};
// row-sharing table (fixed offset in the scratch, survives re-layouts): entries of 8 u64 =
// state ((epoch << 32) | ready bit 31 | busy bit 30 | owner) + 6 key words; epoch = call counter,
// entries of other calls count as empty
constexpr int kRowTab = 4096;
constexpr int kRowTabProbe = 64;

// single-block SM-set class by computed planes: one descriptor per (class entry, load field)
struct CDesc {
  int32_t entry, c, field, per;
  int32_t z0, np, y0, ny;
  long long S0, off;  // the class block, the descriptor's first plane in the pool
  int32_t box[6];     // the block's cell box x0, x1, y0, y1, z0, z1 (k_cplanes' member box)
  int32_t pad[2];
};
constexpr int kCPoolPerConfig = 2048;   // plane pool (Tri pairs) per configuration
constexpr int kCDescPerConfig = 64;     // descriptors per configuration

// per-config accumulator slots (u64, atomically added by the worker kernels)
enum {
  A_LUP = 0, A_WF, A_REQ_LD, A_REQ_ST, A_SM_SEC, A_SM_LIN,
  A_WLD, A_WST, A_WLIN, A_LY, A_LZ, A_OVY, A_OVZ,
  A_PAGES, A_SECLD, A_SECLIN, A_ULD, A_ULIN,   // k_sect (linear address space)
  A_N = 24
};

struct DPrefix {
  int64_t warp, wclass, set, sclass, chunk, fold, sect, ritem;  // ritem: k_rows items (computed chunks)
};
constexpr int kNPrefix = 8;
constexpr int kWSlots = 32 * 64 * 8;  // per config: warp index (<32) x residue (<64) x clip pattern (<8)
constexpr int kSSlots = 64 * 8;       // per config: residue (<64) x clip pattern (<8)
constexpr int kShareTab = 8192;       // SM-set classes shared across configurations (k_smset)
#ifndef WS_SECT_SEG
#define WS_SECT_SEG 8
#endif
constexpr int kSectSeg = WS_SECT_SEG;  // k_sect: row segments (CTAs) per (config, field)
constexpr int kSectPartBytes = 11 * 24;  // k_sect: one segment's partial triples (kSectNQ x Tri)

// ---------------------------------------------------------------- launchers (ws_kernels.cu)
struct Scratch {
  DPlan* plans;
  DInstr* instr;
  DRowInfo* rowinfo;
  unsigned long long* acc;
  DPrefix* prefix;            // n + 1 entries
  long long* chunkres;        // max_chunks * kNQ * 3
  int64_t max_chunks;
  unsigned int* wcnt;         // n * kWSlots
  unsigned long long* wrep;   // n * kWSlots
  unsigned int* scnt;         // n * kSSlots
  unsigned long long* srep;   // n * kSSlots
  unsigned long long* skey;   // kShareTab: cross-configuration class keys (~0 = empty)
  unsigned long long* sval;   // kShareTab * 2: the owner's (sectors, lines)
  void* spart;                // k_sect: n * max_fields * kSectSeg partial triple sets
  unsigned int* sdone;        // k_sect: n * max_fields finished segments
  int32_t max_fields;
  unsigned long long* work;   // K_NKINDS algorithmic work units of the last call (ws_work_read)
  unsigned long long* lists;  // [0] # warp classes, [1] # SM-set classes, [2] # direct SM sets (zeroed by k_scan)
  unsigned long long* wlist;  // n * kWSlots entries (config << 32 | slot)
  unsigned long long* slist;  // n * kSSlots entries
  unsigned long long* dlist;  // multi-block SM sets evaluated directly: n * max n_sm * 16 entries
  unsigned int* dmask;        // per dlist entry: member mask of a connected component (0 = the set)
  unsigned long long* gkey;   // per SM set (pre.set order): k_spairs' translation-group key for k_smset
  // single-block SM-set classes by computed planes (k_cplan / k_cplanes / k_cfold)
  void* cdesc;                // CDesc[cdesc_cap]
  void* cpool;                // Tri pairs [cpool_cap]
  uint32_t* citems;           // computed-plane items [cpool_cap]
  uint32_t* cfbl;             // class entries k_cplan leaves to k_sclass (CTA path)
  int64_t cdesc_cap, cpool_cap;
  unsigned int* plan_done;    // k_plan CTAs finished (the last one scans; reset to 0 by it)
  unsigned long long* epoch;  // estimate calls so far (k_plan's last CTA increments it)
  unsigned long long* rowtab; // kRowTab x 8 u64: a5/a6 sharing keys (see DPlan::row_owner)
  uint32_t* clist;            // per config (stride clist_stride): its computed chunks, fi << 26 | chunk
  int64_t clist_stride;
  // the row chain's own work lists (no prefix scan): k_plan reserves each owner's ranges with atomics
  // on the counters of the call's epoch parity; rctr[p * 4 + 0] row items, + 1 chunks, + 2 fold items,
  // rctr[8] = p (written by k_plan)
  unsigned long long* rctr;
  unsigned long long* ritems;  // config << 32 | fi << 26 | chunk (max_chunks entries)
  uint32_t* fitems;            // config << 6 | fi (n * max_fields entries)
};

// kernel kinds, in launch order (ws_kernel_name)
enum { K_PLAN = 0, K_INSTR, K_WARP, K_WCLASS, K_SMSET, K_SCLASS, K_ROWS, K_FOLD, K_SECT, K_MODEL, K_RANK,
       K_SIMGEN, K_SIMRUN, K_FIT, K_NKINDS };
constexpr int kEstimateKernels = 10;

// Streams and fork/join events of one context: the three worker chains (warp scope, SM-set
// scope, row scope) run concurrently after k_scan.
struct Streams {
  cudaStream_t main, aux[2];
  cudaEvent_t fork, join[2], scanned;   // scanned: k_scan done (the warp chain waits for it)
};
// ws_estimate_multi (BJ configs[3]): one integer pass over m configurations x n_groups
// representative hardware sets, the model over m x n_gpu outputs (k_expand / k_model_fan).
constexpr int kMaxFanGpus = 256;
struct FanOut {
  int32_t n, i0, m, n_gpu, n_groups, pad;  // n: configurations of the call (output stride); [i0, i0+m): this chunk
  uint32_t rep[kMaxFanGpus];               // group -> representative gpu id (the integer pass runs with it)
  uint16_t group[kMaxFanGpus], gid[kMaxFanGpus];  // output hardware set g -> its group, its gpu id
};
// ev: nullptr, or 2 events per kernel (start, end) in K_* order, recorded on the kernel's stream.
// fan: nullptr (k_model writes d_out[0..n)) or the fan-out of ws_estimate_multi (n = m * n_groups).
// tail: nullptr, or the ranking of ws_estimate_ranked_async; for n <= kTailMax (no fan) the last
// CTA of k_model ranks the batch and tail->done is set, else the caller ranks.
constexpr int kTailMax = 1024;
struct TailRank {
  int k;
  uint32_t* top;
  int done;
};
int launch_estimate(const ws_config* d_cfgs, int n, const DKernel* d_k, int nk, const DGpu* d_g, int ng,
                    const Scratch& s, ws_result* d_out, const Streams& st, int n_sm_dev, uint32_t* launches,
                    cudaEvent_t* ev, const FanOut* fan = nullptr, TailRank* tail = nullptr);
int launch_expand(const ws_config* d_cfgs, const FanOut& f, ws_config* xcfg, cudaStream_t st);
// ---------------------------------------------------------------- NEXT-1: simulated hit rates
// Request encoding: bits 0..45 sector + 2^45, bit 46 store, bits 48..55 field.
constexpr int kSimSecBits = 46;
constexpr long long kSimSecBias = 1ll << 45;
constexpr int kSimMaxCaps = 64;
constexpr int kSimAcc = 8 + 4 * (kSimMaxCaps + 1);  // per-config u64 accumulators
// per-config accumulator layout
enum { SA_L1REQ = 0, SA_L1COMP, SA_STREQ, SA_STCOMP, SA_OVY, SA_OVZ, SA_L1H = 8 };
// SA_L1H + b: L1 misses histogram; +65: store; +130: y resident; +195: z resident (b = 0..64)
constexpr int kSimHist = kSimMaxCaps + 1;

struct DSimTrace {
  int64_t req_off, n, fen_off, slot_off, hcap, t_y, m_off;
  int32_t config, type;  // type 0 = SM-set loads, 1 = wave, 2 = layer set L_z
};

struct SimScratch {
  int64_t* item_pre;           // per config: exclusive prefix of block items (n + 1)
  int64_t* trace_pre;          // per config: first trace index (n + 1)
  int64_t* item_cnt;           // per block item: requests (then exclusive prefix, + total)
  uint32_t* order;             // n * kMaxInstr: canonical instruction order
  unsigned long long* req;     // requests
  DSimTrace* traces;
  int64_t n_traces;
  uint32_t* fen;               // Fenwick trees
  unsigned long long* keys;    // slot keys
  uint32_t* last;              // slot: last access of the line
  uint32_t* M;                 // slot x sector: max line distance since the sector's last access
  uint32_t* SL;                // slot x sector: last access of the sector
  unsigned long long* wld;     // per config WLD hash sets
  int64_t* wld_off;            // per config (offset, capacity) pairs
  unsigned long long* acc;     // n * kSimAcc
  unsigned long long* lines;   // capacities in lines, ascending (n_cap)
  unsigned long long* counter; // trace work counter
};

// ev: nullptr or 2 events (start, end)
// scratch: rank_scratch_bytes(n) bytes of device memory (none for n <= 16384)
int launch_rank(ws_result* d_res, int n, int k, uint32_t* d_top, void* scratch, cudaStream_t st, uint32_t* launches,
                cudaEvent_t* ev);
size_t rank_scratch_bytes(int n);
// WS_CHECK build: out[5] = {1, violations, first line, its index, its capacity} (and resets them);
// ordinary build: zeros
int check_read(unsigned long long* out);

// NEXT-1 (ws_kernels.cu): the whole ws_simulate device sequence (estimate, request streams,
// stack-distance simulation, sample records) on st.main, synchronous; returns 0, a
// cudaError_t, or -WS_ELIMIT / -WS_EINVAL.  ev: nullptr or 4 events (gen start/end, run start/end).
// ws_simulate's device buffers, kept by the context between calls (grow-only, one slot per
// allocation site in call order): cudaMalloc / cudaFree of tens of GB cost more than the kernels
struct SimCache {
  std::vector<void*> ptr;
  std::vector<size_t> bytes;
  void release() {
    for (void* p : ptr)
      if (p) cudaFree(p);
    ptr.clear();
    bytes.clear();
  }
};
int run_simulate(const ws_config* d_cfgs, int n, const DKernel* d_k, int nk, const DGpu* d_g, int ng,
                 const std::vector<DGpu>& hg, const Scratch& s, ws_result* d_est, const Streams& st, int n_sm_dev,
                 const uint64_t* h_caps, int ncap, ws_sim_result* h_out, uint32_t* launches, cudaEvent_t* ev,
                 SimCache& cache);
// ws_fit_gompertz on the device; out = (a, b, c, rss).  ev: nullptr or 2 events.
int run_fit(const double* h_O, const double* h_R, int n, double* h_out, cudaStream_t q, cudaEvent_t* ev);

}  // namespace wsb
