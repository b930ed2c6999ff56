// ws_kernels.cu -- sm_100a kernels of the Warpspeed hot path.
//
//   k_plan   (a1)  one CTA per configuration: geometry, wave, SM sets, layer sets,
//                  fold-deduplicated instruction table, row boxes, work counts.
//   (scan)         exclusive prefix of the per-config work counts: k_plan's last CTA.
//   k_warp   (a2+a3) one warp per (config, wave warp): addresses of every lane and
//                  instruction, unique sectors per warp instruction (lanes are
//                  address-sorted, so a shuffle against the previous issuing lane
//                  dedupes), half-warp wavefronts (__match_any_sync bank histogram
//                  per 1024 B cluster), lattice updates.
//   k_smset  (a4)  one CTA per configuration: SM-resident block sets into translation
//                  classes (per config, shared across configs with the same block
//                  footprint) or translation groups of directly evaluated sets;
//   k_sclass       one CTA per class representative / direct set: unique load
//                  sectors/lines of the set's footprint, plane by plane; k_sshare
//                  adds shared classes to their sharers.
//   k_rows   (a5+a6) one CTA per (config, field, chunk of 1024 address rows):
//                  unique sectors/lines of the wave, the layer sets and their unions,
//                  row by row, as ordered (first, last, count) triples.
//   k_fold         ordered fold of the chunk triples -> per-config counts.
//   k_model  (a7)  FP64 Eqs. 1-5 + max-limiter.
//   k_rank   (a8)  rank by (t_pred, index).
//
// Exactness: every count is an exact set cardinality.  Footprints of a set of
// threads are computed as unions of element intervals per address row: the
// footprint of blocks R for field phi is {addr(c+o) : c active cell of R,
// o an offset of phi} (every active cell c = base+kappa issues instruction
// r = kappa+o).  Rows are element-
// disjoint and address-ordered (validated layout), so the sector union of a
// sorted list of element intervals is sum(len) - #(adjacent pairs sharing a
// sector); the (first, last, count) triple is a monoid under that rule.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ws_internal.cuh"

// minimum resident CTAs per SM of the two heaviest kernels (register budget; A/B-tunable)
// (A/B on B200, BJ configs[1]: rows/sclass 2/1 -> 3/3 took the step from 0.283 to 0.207 ms,
// k_fold 4 resident CTAs to 0.206 ms; scripts/ab.sh)
#ifndef WS_ROWS_MINB
#define WS_ROWS_MINB 3
#endif
#ifndef WS_SCLASS_MINB
#define WS_SCLASS_MINB 3
#endif
#ifndef WS_SECT_CTAS
#define WS_SECT_CTAS 2  // k_sect CTAs per SM (launched even when no configuration wants outlook metrics)
#endif
#ifndef WS_SCLASS_THREADS
#define WS_SCLASS_THREADS 256  // threads per k_sclass CTA (<= 1024; shared arrays sized by it)
#endif
#ifndef WS_FOLD_MINB
#define WS_FOLD_MINB 4
#endif

namespace wsb {

#define FULL 0xffffffffu

// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic-serialization
// attribute starts while its predecessor in the stream finishes; griddepcontrol.wait blocks until
// the predecessor grid has completed and its memory is visible (a no-op for ordinary launches),
// launch_dependents lets this grid's own dependent start its prologue early.
#define PDL_PROLOGUE() asm volatile("griddepcontrol.wait;" ::: "memory")
#define PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")

// ------------------------------------------------------------------ bounds-check build (WS_CHECK)
// The GPU pool's compute-sanitizer is closed, so a -DWS_CHECK build checks every dynamically
// computed scratch index of the estimate chain against its capacity (WS_CHK) and records the
// first violation (source line, index, capacity) and the count; ws_check_read returns them.
#ifdef WS_CHECK
struct CheckCaps {
  long long max_chunks, clist_stride, wslots, sslots, cdesc, cpool, spart, rowinfo, instr, fitems;
};
__device__ CheckCaps g_caps;
__device__ unsigned long long g_check[4];   // violations, first line, its index, its capacity
__device__ __noinline__ void ws_check_fail(int line, long long i, long long cap) {
  if (atomicAdd(&g_check[0], 1ull) == 0ull) {
    g_check[1] = (unsigned long long)line;
    g_check[2] = (unsigned long long)i;
    g_check[3] = (unsigned long long)cap;
  }
}
#define WS_CHK(i, cap)                                                       \
  do {                                                                       \
    const long long _wi = (long long)(i), _wc = (long long)(cap);            \
    if (_wi < 0 || _wi >= _wc) ws_check_fail(__LINE__, _wi, _wc);           \
  } while (0)
#else
#define WS_CHK(i, cap) \
  do {                 \
  } while (0)
#endif

int check_read(unsigned long long* out) {   // {is check build, violations, line, index, capacity}
#ifdef WS_CHECK
  unsigned long long h[4] = {0, 0, 0, 0};
  cudaError_t e = cudaMemcpyFromSymbol(h, g_check, sizeof(h));
  if (e != cudaSuccess) return (int)e;
  const unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_check, z, sizeof(z));
  out[0] = 1;
  for (int i = 0; i < 4; ++i) out[1 + i] = h[i];
#else
  for (int i = 0; i < 5; ++i) out[i] = 0;
#endif
  return 0;
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ long long shfl64(long long v, int src) {
  int lo = __shfl_sync(FULL, (int)(v & 0xffffffffll), src);
  int hi = __shfl_sync(FULL, (int)(v >> 32), src);
  return ((long long)hi << 32) | (unsigned int)lo;
}
__device__ __forceinline__ long long shfl64_up(long long v, int d) {
  int lo = __shfl_up_sync(FULL, (int)(v & 0xffffffffll), d);
  int hi = __shfl_up_sync(FULL, (int)(v >> 32), d);
  return ((long long)hi << 32) | (unsigned int)lo;
}
__device__ __forceinline__ long long shfl64_down(long long v, int d) {
  int lo = __shfl_down_sync(FULL, (int)(v & 0xffffffffll), d);
  int hi = __shfl_down_sync(FULL, (int)(v >> 32), d);
  return ((long long)hi << 32) | (unsigned int)lo;
}

__device__ __forceinline__ FDiv make_fdiv(unsigned long long d) {
  unsigned l = 0;
  while ((1ull << l) < d) ++l;
  FDiv f;
  f.l = l;
  f.m = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1ull);
  return f;
}
// n / d for 0 <= n < 2^31
__device__ __forceinline__ long long fdiv(long long n, FDiv f) {
  return (long long)((__umulhi((unsigned)n, f.m) + (unsigned)n) >> f.l);
}

// Smallest power of two k <= 16 with k * plane_pitch_bytes a multiple of line_bytes (0: none):
// planes that far apart are translates by whole lines.
__device__ __forceinline__ int plane_period(long long pz, int le, int ll) {
  const long long pb = pz << le;
  const long long tz = pb == 0 ? 63 : __ffsll(pb) - 1;
  const long long need = ll > tz ? ll - tz : 0;
  return need <= 4 ? (1 << need) : 0;
}

// Row layout of field F seen by the wave / layer-set scopes: the field's own (linear address
// space), or under WS_VAR_MDIM the multidimensional address space realised as a
// virtual layout whose rows start on a line boundary and are padded to whole lines, with no
// alignment: (z, y, floor(x * elem / sector)) tuples never share a sector or line across
// rows, exactly the paper's "two multi dimensional addresses are distinct when their tuples
// differ"; floor(x * elem / sector) is unchanged by a line-aligned row start.
__device__ __forceinline__ void field_rows(const DField& F, const DPlan& P, int ll, long long& py, long long& pz,
                                           long long& align) {
  if (!P.mdim) {
    py = F.pitch[1];
    pz = F.pitch[2];
    align = F.align;
    return;
  }
  const long long rowb = (((F.ext[0] << F.lg_elem) + (1ll << ll) - 1) >> ll) << ll;
  py = rowb >> F.lg_elem;
  pz = py * F.ext[1];
  align = 0;
}

// Plane derivation (k_plan, k_fold): a plane whose every offset group of the field falls in the
// same block layer (or the same side outside the domain) as in the plane `per` before it has the
// same row structure, translated by whole lines.  Returns the plane's representative: the start
// of its zone segment (the largest zone start over the groups, at least the box start z0) plus
// (z - start) mod per; the plane itself when per == 0 (no period within 16 planes).
__device__ __forceinline__ int plane_rep(const DGroup* g, int ng, int z, int z0, int lo2, int hi2, int BF2, FDiv fdz,
                                         int per) {
  if (per <= 0) return z;
  int seg = z0;
  for (int i = 0; i < ng; ++i) {
    const int oz = g[i].oz, zz = z - oz;
    int st;
    if (zz < lo2) st = -0x7fffffff;
    else if (zz >= hi2) st = hi2 + oz;
    else st = lo2 + (int)fdiv(zz - lo2, fdz) * BF2 + oz;
    seg = st > seg ? st : seg;
  }
  return seg + ((z - seg) % per);
}
// the same over the field's distinct oz values (DField::oz_mask: groups sharing an oz give the
// same zone start), falling back to the group loop when the mask is unavailable
__device__ __forceinline__ int plane_rep_f(const DField& F, const DGroup* g, int z, int z0, int lo2, int hi2, int BF2,
                                           FDiv fdz, int per) {
  if (per <= 0) return z;
  unsigned long long m = F.oz_mask;
  if (m == 0ull) return plane_rep(g, F.g_end - F.g_begin, z, z0, lo2, hi2, BF2, fdz, per);
  int seg = z0;
  while (m) {
    const int oz = F.oz_min + __ffsll((long long)m) - 1, zz = z - oz;
    m &= m - 1;
    int st;
    if (zz < lo2) st = -0x7fffffff;
    else if (zz >= hi2) st = hi2 + oz;
    else st = lo2 + (int)fdiv(zz - lo2, fdz) * BF2 + oz;
    seg = st > seg ? st : seg;
  }
  return seg + ((z - seg) % per);
}

// The zone segment of plane z and where it ends: seg = plane_rep's segment start (the largest zone
// start over the field's distinct oz values, at least z0) and the next plane where some oz's zone
// start changes (INT_MAX: none).  plane_rep(z) == z  <=>  z - seg < per, constant on [z, next).
__device__ __forceinline__ int plane_seg(const DField& F, const DGroup* g, int z, int z0, int lo2, int hi2, int BF2,
                                         FDiv fdz, int& seg) {
  seg = z0;
  int nxt = 0x7fffffff;
  auto one = [&](int oz) {
    const int zz = z - oz;
    int st, nx;
    if (zz < lo2) {
      st = -0x7fffffff;
      nx = lo2 + oz;
    } else if (zz >= hi2) {
      st = hi2 + oz;
      nx = 0x7fffffff;
    } else {
      const int bl = lo2 + (int)fdiv(zz - lo2, fdz) * BF2;
      st = bl + oz;
      nx = (bl + BF2 < hi2 ? bl + BF2 : hi2) + oz;
    }
    seg = st > seg ? st : seg;
    nxt = nx < nxt ? nx : nxt;
  };
  unsigned long long m = F.oz_mask;
  if (m) {
    while (m) {
      const int oz = F.oz_min + __ffsll((long long)m) - 1;
      m &= m - 1;
      one(oz);
    }
  } else {
    for (int i = 0; i < F.g_end - F.g_begin; ++i) one(g[i].oz);
  }
  return nxt;
}

struct Tri {
  long long f, l, c;  // first, last, count; c == 0: empty
};
__device__ __forceinline__ Tri tri_empty() { return Tri{0, 0, 0}; }
// append the sorted range [s0, s1] (s0 >= last element appended so far)
__device__ __forceinline__ void tri_add(Tri& t, long long s0, long long s1) {
  if (t.c == 0) {
    t.f = s0;
    t.c = s1 - s0 + 1;
  } else {
    t.c += s1 - s0 + 1 - (t.l == s0 ? 1 : 0);
  }
  t.l = s1;
}
__device__ __forceinline__ Tri tri_combine(const Tri& a, const Tri& b) {  // branch-free (selects)
  const bool ea = a.c == 0, eb = b.c == 0;
  return Tri{ea ? b.f : a.f, eb ? a.l : b.l, a.c + b.c - ((!ea && !eb && a.l == b.f) ? 1 : 0)};
}

// Ordered warp reduction of NQ triples (lane order = address order), result in every lane.  The
// fold of sorted element runs is associative with the only overlap between consecutive non-empty
// triples (last == next first), so total count = sum of counts - #{consecutive non-empty pairs with
// l_prev == f}, first = the first non-empty lane's f, last = the last non-empty lane's l: a ballot,
// three shuffles and two sums per triple instead of a 5-level shuffle tree of whole triples.
template <int NQ>
__device__ __forceinline__ void warp_ordered_reduce(Tri (&t)[NQ]) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const bool ne = t[q].c != 0;
    const unsigned m = __ballot_sync(FULL, ne);
    if (m == 0u) {
      t[q] = tri_empty();
      continue;
    }
    const unsigned below = m & lt;
    const long long lprev = shfl64(t[q].l, below ? 31 - __clz(below) : lane);
    long long c = t[q].c - ((ne && below && lprev == t[q].f) ? 1 : 0);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) c += shfl64_down(c, o);
    t[q] = Tri{shfl64(t[q].f, __ffs(m) - 1), shfl64(t[q].l, 31 - __clz(m)), shfl64(c, 0)};
  }
}

// Ordered CTA reduction of NQ triples per thread (thread order = row order).
// Result valid in thread 0.  `sm` holds (blockDim/32)*NQ triples.
template <int NQ>
__device__ void cta_ordered_reduce(Tri (&t)[NQ], Tri* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  warp_ordered_reduce<NQ>(t);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) sm[warp * NQ + q] = t[q];
  __syncthreads();
  // the warps' partials in warp order, one triple slot per thread of warp 0 (NQ <= 32 in parallel)
  if (threadIdx.x < NQ) {
    const int q = threadIdx.x;
    Tri a = sm[q];
    for (int w = 1; w < nw; ++w) a = tri_combine(a, sm[w * NQ + q]);
    sm[q] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) t[q] = sm[q];
  __syncthreads();
}


// Union of the element intervals produced by `gen` (each [xs, xe), xs < xe) in one
// address row whose element 0 is at byte R0; appends the union's sectors/lines in
// increasing order to *ts / *tl.  Repeated extension: no sorting, no storage.
template <class Gen>
__device__ __forceinline__ void row_union(const Gen& gen, long long R0, int lg_elem, int lg_sec, int lg_line, Tri* ts,
                                          Tri* tl, Tri* ts2 = nullptr) {
  const long long INF = LLONG_MAX;
  long long start = INF, mx_s = LLONG_MIN, mn_e = INF, mx_e = LLONG_MIN;
  gen([&](long long xs, long long xe) {
    start = xs < start ? xs : start;
    mx_s = xs > mx_s ? xs : mx_s;
    mn_e = xe < mn_e ? xe : mn_e;
    mx_e = xe > mx_e ? xe : mx_e;
  });
  if (start == INF) return;
  if (mx_s <= mn_e) {  // every interval reaches the point mx_s: one component [start, mx_e)
    const long long a0 = R0 + (start << lg_elem), a1 = R0 + ((mx_e - 1) << lg_elem);
    if (ts) tri_add(*ts, a0 >> lg_sec, a1 >> lg_sec);
    if (ts2) tri_add(*ts2, a0 >> lg_sec, a1 >> lg_sec);
    if (tl) tri_add(*tl, a0 >> lg_line, a1 >> lg_line);
    return;
  }
  while (start != INF) {
    long long end = start, nxt;
    bool grew;
    do {
      grew = false;
      nxt = INF;
      gen([&](long long xs, long long xe) {
        if (xs <= end) {
          if (xe > end) {
            end = xe;
            grew = true;
          }
        } else if (xs < nxt) {
          nxt = xs;
        }
      });
    } while (grew);
    const long long a0 = R0 + (start << lg_elem), a1 = R0 + ((end - 1) << lg_elem);
    if (ts) tri_add(*ts, a0 >> lg_sec, a1 >> lg_sec);
    if (ts2) tri_add(*ts2, a0 >> lg_sec, a1 >> lg_sec);
    if (tl) tri_add(*tl, a0 >> lg_line, a1 >> lg_line);
    start = nxt;
  }
}

// Triple of `run` consecutive rows that are translates of each other by `step` bytes;
// row(r) returns row r's own triple in units of 2^sh bytes.  Rows r and r+P (P =
// 2^sh / gcd(step, 2^sh)) differ by exactly D = P*step >> sh units, so the run is nb full
// periods (each the translate of rows [0,P) by D) plus the translate of rows [0, rem):
// only the first P rows are evaluated.
template <class RowFn>
__device__ __forceinline__ Tri run_triple(const RowFn& row, long long step, int run, int sh) {
  const int tz = step == 0 ? 63 : __ffsll(step) - 1;
  const int P = sh > tz ? 1 << (sh - tz) : 1;
  if (run <= 2 * P) {
    Tri acc = tri_empty();
    for (int r = 0; r < run; ++r) acc = tri_combine(acc, row(r));
    return acc;
  }
  const int nb = run / P, rem = run % P;
  const long long D = ((long long)P * step) >> sh;
  Tri blk = tri_empty(), remb = tri_empty();
  for (int i = 0; i < P; ++i) {
    const Tri rt = row(i);
    blk = tri_combine(blk, rt);
    if (i < rem) remb = tri_combine(remb, rt);
  }
  if (blk.c == 0) return blk;  // every row empty
  const long long adj = blk.l == blk.f + D ? 1 : 0;
  Tri acc{blk.f, blk.l + (long long)(nb - 1) * D, (long long)nb * blk.c - (long long)(nb - 1) * adj};
  if (remb.c) acc = tri_combine(acc, Tri{remb.f + (long long)nb * D, remb.l + (long long)nb * D, remb.c});
  return acc;
}

template <int MEMBER>
__device__ __forceinline__ int find_config(const DPrefix* pre, int n, long long item) {
  // largest c in [0, n) with pre[c].member <= item (pre is an exclusive prefix)
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    const long long v = MEMBER == 0   ? pre[mid].warp
                        : MEMBER == 1 ? pre[mid].wclass
                        : MEMBER == 2 ? pre[mid].set
                        : MEMBER == 3 ? pre[mid].sclass
                        : MEMBER == 4 ? pre[mid].chunk
                        : MEMBER == 5 ? pre[mid].fold
                        : MEMBER == 6 ? pre[mid].sect
                                      : pre[mid].ritem;
    if (v <= item) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <int MEMBER>
__device__ __forceinline__ long long prefix_member(const DPrefix& p) {
  return MEMBER == 0   ? p.warp
         : MEMBER == 1 ? p.wclass
         : MEMBER == 2 ? p.set
         : MEMBER == 3 ? p.sclass
         : MEMBER == 4 ? p.chunk
         : MEMBER == 5 ? p.fold
         : MEMBER == 6 ? p.sect
                       : p.ritem;
}

// find_config by the whole warp (item warp-uniform): 32-ary search, one load round per
// factor 32 of n, starting from the hint c when item still lies in config c.
template <int MEMBER>
__device__ __forceinline__ int find_config_warp(const DPrefix* pre, int n, long long item, int hint) {
  const int lane = threadIdx.x & 31;
  if (hint >= 0 && item >= prefix_member<MEMBER>(pre[hint]) && item < prefix_member<MEMBER>(pre[hint + 1]))
    return hint;
  int lo = 0, hi = n - 1;  // invariant: member(pre[lo]) <= item
  while (hi > lo) {
    const int stride = (hi - lo + 32) >> 5;
    const int idx = lo + lane * stride;
    const bool le = idx <= hi && prefix_member<MEMBER>(pre[idx]) <= item;
    const unsigned b = __ballot_sync(FULL, le);
    lo += (31 - __clz(b)) * stride;
    hi = min(hi, lo + stride - 1);
  }
  return lo;
}

// ------------------------------------------------------------------ a1: plan
// P must be zeroed by the caller (k_plan zeroes its shared copy cooperatively)
__device__ void plan_geometry(const ws_config& cf, const DKernel* ks, int nk, const DGpu* gs, int ng, DPlan& P) {
  P.kid = (int)cf.kernel_id;
  P.gid = (int)cf.gpu_id;
  if (cf.kernel_id >= (uint32_t)nk || cf.gpu_id >= (uint32_t)ng) {
    P.status = WS_EUNKNOWN_ID;
    return;
  }
  const DKernel& K = ks[cf.kernel_id];
  const DGpu& G = gs[cf.gpu_id];
  for (int d = 0; d < 3; ++d) {
    if (cf.block[d] < 1 || cf.fold[d] < 1) {
      P.status = WS_EINVAL;
      return;
    }
  }
  if (K.env.max_lg_elem > G.lg_sector) {   // an element wider than a sector (describe-time maximum)
    P.status = WS_EINVAL;
    return;
  }
  if (cf.variant & ~15u) {  // unknown WS_VAR_* bits
    P.status = WS_EINVAL;
    return;
  }
  P.variant = (int)cf.variant;
  P.mdim = (cf.variant & WS_VAR_MDIM) != 0;
  if (P.mdim) {  // padded rows (whole lines) must keep a z-plane within the 32-bit plane arithmetic
    for (int i = 0; i < K.n_fields; ++i) {
      const long long rowb = (((K.f[i].ext[0] << K.f[i].lg_elem) + (1ll << G.lg_line) - 1) >> G.lg_line) << G.lg_line;
      if (rowb * K.f[i].ext[1] > (1ll << 31) - (1ll << 14)) {
        P.status = WS_ELIMIT;
        return;
      }
    }
  }
  const long long T = (long long)cf.block[0] * cf.block[1] * cf.block[2];
  if (T > (long long)G.g.max_thr_blk) {
    P.status = WS_ELIMIT;
    return;
  }
  const long long fc = (long long)cf.fold[0] * cf.fold[1] * cf.fold[2];
  if (fc > kMaxFoldCube) {
    P.status = WS_ELIMIT;
    return;
  }
  long long k;
  const long long Ta = (T + 31) / 32 * 32;
  if (cf.blocks_per_sm > 0) {
    k = cf.blocks_per_sm;
  } else {
    k = (long long)G.g.max_thr_sm / Ta;
    if ((long long)G.g.max_blk_sm < k) k = G.g.max_blk_sm;
    if (K.regs > 0) {
      long long kr = (long long)G.g.regs_sm / ((long long)K.regs * Ta);
      if (kr < k) k = kr;
    }
  }
  if (k < 1) {
    P.status = WS_ELIMIT;
    return;
  }
  for (int d = 0; d < 3; ++d) {
    P.b[d] = (int)cf.block[d];
    P.f[d] = (int)cf.fold[d];
    P.lo[d] = K.lo[d];
    P.hi[d] = K.hi[d];
    P.BF[d] = (long long)cf.block[d] * cf.fold[d];
    P.G[d] = (K.hi[d] - K.lo[d] + P.BF[d] - 1) / P.BF[d];
  }
  P.T = (int)T;
  P.fcube = (int)fc;
  P.nwarps = (int)((T + 31) / 32);
  P.k = (int)k;
  P.N = P.G[0] * P.G[1] * P.G[2];
  const long long cap = (long long)G.g.n_sm * k;
  P.W = P.N < cap ? P.N : cap;
  const long long cen = P.G[0] / 2 + P.G[0] * (P.G[1] / 2 + P.G[1] * (P.G[2] / 2));
  long long s = cen - P.W / 2;
  if (s < 0) s = 0;
  if (s > P.N - P.W) s = P.N - P.W;
  P.s = s;
  P.nsets = (long long)G.g.n_sm < P.W ? (long long)G.g.n_sm : P.W;
  P.Ly0 = s - P.G[0] > 0 ? s - P.G[0] : 0;
  P.Lz0 = s - P.G[0] * P.G[1] > 0 ? s - P.G[0] * P.G[1] : 0;
  // WS_VAR_PREV_WAVE (V100 / SBAC model): both look-back sets are the preceding wave
  if (cf.variant & WS_VAR_PREV_WAVE) P.Ly0 = P.Lz0 = s - P.W > 0 ? s - P.W : 0;
  // NEXT-4 outlook metrics: TLB pages (page size given) and L2-section footprints (several
  // sections and either the link limiter or the duplication-based capacity wanted)
  // WS_VAR_REP_BLOCK: the wave's middle block stands for all W blocks in the L1 scopes
  if (cf.variant & WS_VAR_REP_BLOCK) {
    P.rep_B = s + P.W / 2;
    P.rep_mult = P.W;
  }
  P.want_pages = G.lg_page >= 0;
  P.want_sect = G.g.l2_sections > 1 && (G.g.link_bw > 0 || (cf.variant & WS_VAR_L2_DUP));
  for (int d = 0; d < 3; ++d) {
    P.fd_BF[d] = make_fdiv((unsigned long long)P.BF[d]);
    const long long last = (K.hi[d] - K.lo[d]) - (P.G[d] - 1) * P.BF[d];
    P.part[d] = last < P.BF[d] ? last : 0;
  }
  // translation classes need one pitch and one element size for every field
  const bool same = K.env.same_layout != 0;   // (computed at describe time)
  // sector counts are invariant under translation by multiples of sector_bytes; bank words
  // shift uniformly under multiples of bank_bytes, which only relabels the banks cyclically
  // (the max multiplicity and the cluster split are unchanged): M = lcm = max (powers of two)
  const long long M = (long long)G.g.sector_bytes > (long long)G.g.bank_bytes ? (long long)G.g.sector_bytes
                                                                              : (long long)G.g.bank_bytes;
  const long long Rw = M >> K.f[0].lg_elem, Rs = (long long)G.g.line_bytes >> K.f[0].lg_elem;
  P.wcls_R = (same && Rw >= 1 && Rw <= 64 && P.nwarps <= 32 && !P.rep_mult) ? (int)Rw : 0;
  P.scls_R = (same && Rs >= 1 && Rs <= 64) ? (int)Rs : 0;
  for (int d = 0; d < 3; ++d) P.cls_pitch[d] = K.f[0].pitch[d];
  P.cls_lg_elem = K.f[0].lg_elem;
  P.wpow2 = (T % 32 == 0) && !(cf.block[0] & (cf.block[0] - 1)) && !(cf.block[1] & (cf.block[1] - 1)) &&
            !(cf.block[2] & (cf.block[2] - 1));
  P.status = WS_OK;
}

// k_rows range q of a plan: 0 = wave, 1 = L_y, 2 = L_z, 3 = L_y + wave, 4 = L_z + wave
__device__ void plan_range(DPlan& P, int q) {
  long long a, b;
  if (q == 0) { a = P.s; b = P.s + P.W; }
  else if (q == 1) { a = P.Ly0; b = P.s; }
  else if (q == 2) { a = P.Lz0; b = P.s; }
  else if (q == 3) { a = P.Ly0; b = P.s + P.W; }
  else { a = P.Lz0; b = P.s + P.W; }
  RangeInfo& R = P.rng[q];
  R.nonempty = a < b;
  R.pad = 0;
  const long long Gx = P.G[0], lx = P.lo[0], hx = P.hi[0], bf = P.BF[0];
  long long xa = 0, xl = Gx;
  if (a < b) {
    R.ra = a / Gx;
    xa = a % Gx;
    R.rl = (b - 1) / Gx;
    xl = (b - 1) % Gx + 1;
  } else {
    R.ra = R.rl = 0;
  }
  const long long xs_a = lx + xa * bf;
  long long xe_l = lx + xl * bf;
  if (xe_l > hx) xe_l = hx;
  R.iv[0][0] = lx;   R.iv[0][1] = hx;
  R.iv[1][0] = xs_a; R.iv[1][1] = hx;
  R.iv[2][0] = lx;   R.iv[2][1] = xe_l;
  R.iv[3][0] = xs_a; R.iv[3][1] = xe_l;
}

// the sorted distinct block rows where some range's classification zone starts, by one warp: lane 4q + k holds candidate k of range q, the first lane of each
// distinct value (match) writes it at its rank among the distinct values (shuffle count)
__device__ void plan_boundaries_warp(DPlan& P, int lane) {
  const unsigned long long INF = ~0ull;
  unsigned long long v = INF;
  if (lane < 20) {
    const RangeInfo& R = P.rng[lane >> 2];
    if (R.nonempty) {
      const int k = lane & 3;
      v = (unsigned long long)(k == 0 ? R.ra : (k == 1 ? R.ra + 1 : (k == 2 ? R.rl : R.rl + 1)));
    }
  }
  const unsigned peers = __match_any_sync(FULL, v);
  const bool first = v != INF && __ffs(peers) - 1 == lane;
  int rank = 0;
  for (int j = 0; j < 20; ++j) {
    const unsigned long long vj = __shfl_sync(FULL, v, j);
    const bool fj = __shfl_sync(FULL, first, j);
    rank += (fj && vj < v) ? 1 : 0;
  }
  if (first) P.bnd[rank] = (long long)v;
  const int nb = __popc(__ballot_sync(FULL, first));
  if (lane == 0) P.nb = nb;
  __syncwarp();
}

// a5/a6 sharing (DPlan::row_owner): claim this configuration's row-scope key in the row table, or
// find the configuration of this call that claimed it first.  The row-scope counts depend only on
// the kernel, the sector / line geometry, the address space, BF (with the domain: G, the block-row
// map), W, s and the look-back starts (the five k_rows ranges).  One thread per configuration.
__device__ void row_claim(DPlan& P, int c, const DGpu& G, unsigned long long cur_epoch,
                          unsigned long long* __restrict__ tab) {
  P.row_owner = c;
  P.row_slot = -1;
  unsigned long long key[6] = {
      (unsigned long long)P.kid | ((unsigned long long)G.lg_sector << 32) | ((unsigned long long)G.lg_line << 40) |
          ((unsigned long long)P.mdim << 48),
      (unsigned long long)P.BF[0] | ((unsigned long long)P.BF[1] << 21) | ((unsigned long long)P.BF[2] << 42),
      (unsigned long long)P.W, (unsigned long long)P.s, (unsigned long long)P.Ly0, (unsigned long long)P.Lz0};
  unsigned long long h = 0x9e3779b97f4a7c15ull;
  for (int i = 0; i < 6; ++i) h = (h ^ key[i]) * 0xff51afd7ed558ccdull, h ^= h >> 29;
  const unsigned long long ep = cur_epoch << 32;
  const unsigned long long READY = 1ull << 31, BUSY = 1ull << 30, OWNER = (1ull << 30) - 1ull;
  for (int probe = 0; probe < kRowTabProbe; ++probe) {
    unsigned long long* e = tab + ((h + probe) & (kRowTab - 1)) * 8;
    unsigned long long st = *(volatile unsigned long long*)e;
    if ((st >> 32) != cur_epoch) {  // empty for this call: try to claim it
      const unsigned long long old = atomicCAS(e, st, ep | BUSY);
      if (old == st) {
        for (int i = 0; i < 6; ++i) e[1 + i] = key[i];
        __threadfence();
        atomicExch(e, ep | READY | (unsigned long long)c);
        P.row_slot = (int)((h + probe) & (kRowTab - 1));
        return;
      }
      st = old;
      if ((st >> 32) != cur_epoch) {  // lost to a claimant of another epoch?  cannot happen; retry slot
        --probe;
        continue;
      }
    }
    while (!(st & READY)) st = *(volatile unsigned long long*)e;  // being written by its claimant
    __threadfence();
    bool eq = true;
    for (int i = 0; i < 6; ++i) eq = eq && ((volatile unsigned long long*)e)[1 + i] == key[i];
    if (eq) {
      P.row_owner = (int)(st & OWNER);
      return;
    }
  }
}

__device__ __forceinline__ void decode_kappa(int q, const int* f, int& kx, int& ky, int& kz) {
  kx = q % f[0];
  ky = (q / f[0]) % f[1];
  kz = q / (f[0] * f[1]);
}

__device__ __forceinline__ long long plan_count(const DPlan& P, int j) {
  switch (j) {
    case 0: return P.n_warp_items;
    case 1: return P.n_wclass_items;
    case 2: return P.n_set_items;
    case 3: return P.n_sclass_items;
    case 4: return P.n_chunks;
    case 5: return P.n_fields;
    case 6: return P.n_sect_items;
    default: return P.n_ritems;
  }
}

// exclusive prefix of the per-config work counts (one CTA of any size)
__device__ void scan_body(const DPlan* __restrict__ plans, int n, DPrefix* __restrict__ pre) {
  __shared__ long long s_w[32][kNPrefix];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int seg = (n + nt - 1) / nt;
  long long a[kNPrefix];
#pragma unroll
  for (int j = 0; j < kNPrefix; ++j) a[j] = 0;
  for (int c = tid * seg; c < n && c < (tid + 1) * seg; ++c) {
    const DPlan& P = plans[c];
    if (P.status != WS_OK) continue;
#pragma unroll
    for (int j = 0; j < kNPrefix; ++j) a[j] += plan_count(P, j);
  }
  // block exclusive scan of the per-thread sums: warp inclusive scans, then the warp totals
  long long inc[kNPrefix];
#pragma unroll
  for (int j = 0; j < kNPrefix; ++j) {
    long long v = a[j];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = shfl64_up(v, o);
      if (lane >= o) v += u;
    }
    inc[j] = v;
    if (lane == 31) s_w[wid][j] = v;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < kNPrefix; ++j) {
      long long v = lane < (nt >> 5) ? s_w[lane][j] : 0;
      const long long own = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long u = shfl64_up(v, o);
        if (lane >= o) v += u;
      }
      if (lane < (nt >> 5)) s_w[lane][j] = v - own;  // exclusive warp offsets
    }
  }
  __syncthreads();
  long long r[kNPrefix];
#pragma unroll
  for (int j = 0; j < kNPrefix; ++j) r[j] = s_w[wid][j] + inc[j] - a[j];
  for (int c = tid * seg; c < n && c < (tid + 1) * seg; ++c) {
    pre[c] = DPrefix{r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7]};
    const DPlan& P = plans[c];
    if (P.status != WS_OK) continue;
#pragma unroll
    for (int j = 0; j < kNPrefix; ++j) r[j] += plan_count(P, j);
  }
  if (tid == nt - 1) pre[n] = DPrefix{r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7]};
}


// the work-count prefix of the warp and SM-set chains (one CTA, at the head of the SM-set chain;
// the row chain has its own atomically reserved lists and does not wait for it); then the call's
// epoch advances (every k_plan CTA of this call has read it)
__global__ void __launch_bounds__(256) k_scan(const DPlan* __restrict__ plans, int n, DPrefix* __restrict__ pre,
                                              unsigned long long* __restrict__ epoch) {
  scan_body(plans, n, pre);
  if (threadIdx.x == 0) *epoch = *epoch + 1ull;
}

// a3 instruction table (O3), on the warp chain: k_plan's plan is complete; the row and SM-set
// chains never read the table, n_instr or addr_evals, so they start without waiting for it.  One
// CTA per configuration.  Pair p = (access a, kappa q) gives instruction (field, kind, kappa + o_a);
// keep the first occurrence of each key.  An earlier pair with the same key needs an earlier access
// a2 of the same field and kind with r - o_a2 inside the fold cube (for a2 == a only q2 == q gives
// the key).  More than kMaxInstr instructions: istat = WS_ELIMIT (k_model reports it).
__global__ void __launch_bounds__(128) k_instr(const DKernel* __restrict__ ks, DPlan* __restrict__ plans,
                                               DInstr* __restrict__ instr, unsigned int* __restrict__ wcnt, int n) {
  PDL_PROLOGUE();
  const int c = blockIdx.x, tid = threadIdx.x;
  // (the warp-class counters of k_warp are zero here: k_wclass returns every slot it reads to 0,
  // and the host zeroes the region whenever the scratch layout moves it)
  __shared__ unsigned char s_first[kMaxAcc * kMaxFoldCube];
  __shared__ int s_part[128];
  __shared__ int s_total;
  __shared__ ws_access s_acc[kMaxAcc];
  __shared__ int s_f[3], s_fc, s_ok;
  if (tid == 0) {
    const DPlan& Pg = plans[c];
    s_ok = Pg.status == WS_OK;
    for (int d = 0; d < 3; ++d) s_f[d] = Pg.f[d];
    s_fc = Pg.fcube;
  }
  __syncthreads();
  if (!s_ok) return;
  const DPlan& PG = plans[c];
  const DKernel& K = ks[PG.kid];
  for (int i = tid; i < K.n_acc; i += blockDim.x) s_acc[i] = K.acc[i];
  struct { int f[3]; } P{{s_f[0], s_f[1], s_f[2]}};
  const int fc = s_fc;
  const int np = K.n_acc * fc;
  __syncthreads();
  // ---- O3: fold-deduplicated instruction table.  Pair p = (access a, kappa q) gives
  // instruction (field, kind, kappa + o_a); keep the first occurrence of each key.  An earlier
  // pair with the same key needs an earlier access a2 of the same field and kind with
  // r - o_a2 inside the fold cube (for a2 == a only q2 == q gives the key).
  __shared__ int s_kap[kMaxFoldCube][3];
  for (int q = tid; q < fc; q += blockDim.x) decode_kappa(q, P.f, s_kap[q][0], s_kap[q][1], s_kap[q][2]);
  __syncthreads();
  for (int p = tid; p < np; p += blockDim.x) {
    const int a = p / fc, q = p - a * fc;
    const ws_access A = s_acc[a];
    const int rx = s_kap[q][0] + A.off[0], ry = s_kap[q][1] + A.off[1], rz = s_kap[q][2] + A.off[2];
    unsigned char first = 1;
    for (int a2 = 0; a2 < a && first; ++a2) {
      const ws_access B = s_acc[a2];
      if (B.field != A.field || B.is_store != A.is_store) continue;
      const int dx = rx - B.off[0], dy = ry - B.off[1], dz = rz - B.off[2];
      if (dx >= 0 && dx < P.f[0] && dy >= 0 && dy < P.f[1] && dz >= 0 && dz < P.f[2]) first = 0;
    }
    s_first[p] = first;
  }
  __syncthreads();
  // block-wide exclusive prefix of s_first (contiguous segments per thread)
  const int seg = (np + blockDim.x - 1) / blockDim.x;
  int mysum = 0;
  for (int p = tid * seg; p < np && p < (tid + 1) * seg; ++p) mysum += s_first[p];
  {  // exclusive scan over the 128 threads: warp shuffles, then the 4 warp totals
    const int lane = tid & 31, wid = tid >> 5;
    int v = mysum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULL, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) s_part[wid] = v;
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      const int x = s_part[w];
      if (w < wid) off += x;
      tot += x;
    }
    __syncthreads();
    s_part[tid] = off + v - mysum;
    if (tid == 0) s_total = tot;
  }
  __syncthreads();
  if (s_total > kMaxInstr) {   // the configuration fails (status WS_ELIMIT in k_model)
    if (tid == 0) {
      plans[c].istat = WS_ELIMIT;
      plans[c].n_instr = 0;
    }
    return;
  }
  {
    int pos = s_part[tid];
    for (int p = tid * seg; p < np && p < (tid + 1) * seg; ++p) {
      if (!s_first[p]) continue;
      const int a = p / fc, q = p - a * fc;
      const ws_access A = s_acc[a];
      const int r[3] = {s_kap[q][0] + A.off[0], s_kap[q][1] + A.off[1], s_kap[q][2] + A.off[2]};
      // kappas whose folded cell uses this instruction: r - kappa2 is an access offset (Q27)
      unsigned long long km = 0;
      for (int q2 = 0; q2 < fc; ++q2) {
        const int o0 = r[0] - s_kap[q2][0], o1 = r[1] - s_kap[q2][1], o2 = r[2] - s_kap[q2][2];
        for (int a2 = 0; a2 < K.n_acc; ++a2) {
          const ws_access B = s_acc[a2];
          if (B.field == A.field && B.is_store == A.is_store && B.off[0] == o0 && B.off[1] == o1 && B.off[2] == o2) {
            km |= 1ull << q2;
            break;
          }
        }
      }
      const DField& F = K.f[A.field];
      DInstr e;
      e.C = F.align + ((r[0] * F.pitch[0] + r[1] * F.pitch[1] + r[2] * F.pitch[2]) << F.lg_elem);
      e.kmask = km;
      e.field = (int)A.field;
      e.kind = (int)A.is_store;
      e.lg_elem = F.lg_elem;
      e.pad = 0;
      WS_CHK(pos, kMaxInstr);
      WS_CHK((long long)c * kMaxInstr + pos, g_caps.instr);
      instr[(long long)c * kMaxInstr + pos] = e;
      ++pos;
    }
  }
  __syncthreads();
  if (tid == 0) {
    DPlan& Q = plans[c];
    Q.n_instr = s_total;
    Q.addr_evals = (unsigned long long)((Q.W + Q.s - Q.Lz0) * (long long)Q.T * s_total);
  }
}

#ifndef WS_PLAN_THREADS
#define WS_PLAN_THREADS 160   // 4 worker warps + the row-claim warp
#endif
__global__ void __launch_bounds__(WS_PLAN_THREADS) k_plan(const ws_config* __restrict__ cfgs, int n,
                                              const DKernel* __restrict__ ks, int nk, const DGpu* __restrict__ gs,
                                              int ng, DPlan* __restrict__ plans, DInstr* __restrict__ instr,
                                              DRowInfo* __restrict__ rowinfo, unsigned long long* __restrict__ acc,
                                              unsigned int* __restrict__ wcnt, unsigned int* __restrict__ scnt,
                                              unsigned long long* __restrict__ rctr,
                                              unsigned long long* __restrict__ ritems, uint32_t* __restrict__ fitems,
                                              unsigned long long* __restrict__ work,
                                              unsigned long long* __restrict__ lists,
                                              unsigned long long* __restrict__ skey, unsigned int* __restrict__ sdone,
                                              int max_fields, unsigned long long* __restrict__ epoch,
                                              unsigned long long* __restrict__ rowtab, uint32_t* __restrict__ clist,
                                              long long clist_stride) {
  const int c = blockIdx.x;
  const int tid = threadIdx.x;
  // k_rows (the row chain, a programmatic dependent on the same stream) may launch now: its CTAs
  // wait in griddepcontrol.wait until this grid has completed, then start without a launch gap
  PDL_TRIGGER();
  const unsigned long long cur_epoch = *(volatile unsigned long long*)epoch + 1ull;  // this call
  const int par = (int)(cur_epoch & 1ull);   // the row chain's counters of this call: rctr[par * 4 ..]
  if (c == 0 && tid < 16) {   // the call's counters (every consumer runs after this grid)
    work[tid] = 0ull;         // K_NKINDS <= 16
    if (tid < 8) lists[tid] = 0ull;                 // class / direct / class-plane / model counters
    if (tid < 4) rctr[(par ^ 1) * 4 + tid] = 0ull;  // the next call's row-chain counters
    if (tid == 8) rctr[8] = (unsigned long long)par;
  }
#ifdef WS_PLAN_CLOCK
  long long clk[12];
  int nclk = 0;
#define PLAN_MARK() if (tid == 0) clk[nclk++] = clock64();
#else
#define PLAN_MARK()
#endif
  __shared__ __align__(16) DPlan P;
  __shared__ __align__(16) DKernel sK;   // this configuration's kernel and GPU descriptors, staged once: the
  __shared__ __align__(16) DGpu sG;      // serial plan work then reads shared memory, not dependent global loads

  if (tid < A_N) acc[(long long)c * A_N + tid] = 0ull;
  // this configuration's SM-set class counters and k_sect counters, and a share of the cross-config
  // class table: zeroed here instead of by memset nodes ahead of the graph's first kernel (the
  // warp-chain counters: k_instr)
  {
    uint4* sc = reinterpret_cast<uint4*>(scnt + (long long)c * kSSlots);
    for (int i = tid; i < kSSlots / 4; i += blockDim.x) sc[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < max_fields; i += blockDim.x) sdone[(long long)c * max_fields + i] = 0u;
    for (int i = c * blockDim.x + tid; i < kShareTab; i += n * blockDim.x) skey[i] = ~0ull;
  }
  static_assert(sizeof(DPlan) % 16 == 0 && sizeof(DKernel) % 16 == 0 && sizeof(DGpu) % 16 == 0, "uint4 copies");
  constexpr int kPlanVec = (int)(sizeof(DPlan) / 16);
  for (int i = tid; i < kPlanVec; i += blockDim.x) reinterpret_cast<uint4*>(&P)[i] = make_uint4(0u, 0u, 0u, 0u);
  PLAN_MARK()
  const ws_config cf = cfgs[c];
  const bool ids_ok = cf.kernel_id < (uint32_t)nk && cf.gpu_id < (uint32_t)ng;
  if (ids_ok) {
    // only the used parts of the kernel descriptor (21 KB in full): header, fields, accesses,
    // groups, each range widened to 16-byte units
    const uint4* srcK = reinterpret_cast<const uint4*>(ks + cf.kernel_id);
    uint4* dstK = reinterpret_cast<uint4*>(&sK);
    const DKernel* hk = ks + cf.kernel_id;
    const int nf = hk->n_fields, na = hk->n_acc, ngr = hk->n_groups;
    const size_t rl[4] = {0, offsetof(DKernel, f), offsetof(DKernel, acc), offsetof(DKernel, g)};
    const size_t rh[4] = {offsetof(DKernel, f), offsetof(DKernel, f) + nf * sizeof(DField),
                          offsetof(DKernel, acc) + na * sizeof(ws_access), offsetof(DKernel, g) + ngr * sizeof(DGroup)};
#pragma unroll
    for (int r = 0; r < 4; ++r)
      for (int i = (int)(rl[r] / 16) + tid; i < (int)((rh[r] + 15) / 16); i += blockDim.x) dstK[i] = srcK[i];
    const uint4* srcG = reinterpret_cast<const uint4*>(gs + cf.gpu_id);
    for (int i = tid; i < (int)(sizeof(DGpu) / 16); i += blockDim.x) reinterpret_cast<uint4*>(&sG)[i] = srcG[i];
  }
  PLAN_MARK()
  __syncthreads();
  if (tid == 0) {
    if (ids_ok) {
      ws_config c0 = cf;
      c0.kernel_id = c0.gpu_id = 0;
      plan_geometry(c0, &sK, 1, &sG, 1, P);
      P.kid = (int)cf.kernel_id;
      P.gid = (int)cf.gpu_id;
    } else {
      plan_geometry(cf, ks, nk, gs, ng, P);  // sets WS_EUNKNOWN_ID
    }
  }
  __syncthreads();
  PLAN_MARK()
  auto store_plan = [&]() {  // cooperative 16-byte copy of the shared plan
    uint4* dst = reinterpret_cast<uint4*>(plans + c);
    for (int i = tid; i < kPlanVec; i += blockDim.x) dst[i] = reinterpret_cast<const uint4*>(&P)[i];
  };
  if (P.status != WS_OK) {
    store_plan();
    return;
  }
  // the batch's split of directly evaluated SM sets by field (k_sclass): kernels with many load
  // fields are evaluated one (set, field) per CTA item
  if (tid == 0 && sK.env.n_ld > 4) atomicMax(rctr + par * 4 + 3, (unsigned long long)sK.n_fields);
  PLAN_MARK()
  // warp kPlanWork/32 alone claims the row-table key (global atomics, a few dependent round trips);
  // warps 0 .. kPlanWork/32-1 meanwhile compute the ranges, boundaries, row boxes and the computed-
  // plane lists as if this configuration owned its row scope (named barrier 1), and the join below
  // drops the lists of a sharer
  constexpr int kPlanWork = WS_PLAN_THREADS - 32;
  static_assert(kPlanWork >= 32 && kPlanWork % 32 == 0, "k_plan: worker warps + the claim warp");
  const int ll = sG.lg_line;
  const DKernel& K = sK;
  __shared__ DRowInfo s_ri[kMaxFields];   // row boxes staged here, written out once
  __shared__ int s_nri;
  __shared__ unsigned long long s_rb[2];   // reserved bases: row items, fold items
  __shared__ int s_zoff[kMaxFields + 1];   // prefix of the fields' window counts (fields with chunks)
  __shared__ int s_wsh;                    // listing window = 1 << s_wsh planes
  uint32_t* cl = clist + (long long)c * clist_stride;
#ifdef WS_PLAN_CLOCK
  __shared__ long long s_clk[4];   // phase start, claim end, workers end, join end
  __shared__ unsigned long long s_wclk[4];   // workers: ranges+boundaries, row boxes, chunk prefix, listing
  if (tid == 0) s_clk[0] = clock64();
  if (tid < 4) s_wclk[tid] = 0ull;
  __syncthreads();
#endif
  if (tid >= kPlanWork) {
    if (tid == kPlanWork) row_claim(P, c, sG, cur_epoch, rowtab);
#ifdef WS_PLAN_CLOCK
    if (tid == kPlanWork) s_clk[1] = clock64();
#endif
  } else {
    auto wbar = [] { asm volatile("bar.sync 1, %0;" ::"r"(kPlanWork) : "memory"); };
    if (tid < 5) plan_range(P, tid);
    __syncwarp();
    if (tid < 32) plan_boundaries_warp(P, tid);
#ifdef WS_PLAN_CLOCK
    if (tid == 0) atomicMax(&s_wclk[0], (unsigned long long)(clock64() - s_clk[0]));
#endif
    // ---- row boxes of the wave + layer-set footprint, per field
    for (int fi = tid; fi < K.n_fields; fi += kPlanWork) {
      const DField& F = K.f[fi];
      const long long rA = P.Lz0 / P.G[0], rB = (P.s + P.W - 1) / P.G[0];
      const long long byA = rA % P.G[1], bzA = rA / P.G[1], byB = rB % P.G[1], bzB = rB / P.G[1];
      long long ylo, yhi;
      if (bzA == bzB) {
        ylo = P.lo[1] + byA * P.BF[1];
        yhi = P.lo[1] + (byB + 1) * P.BF[1];
        if (yhi > P.hi[1]) yhi = P.hi[1];
      } else {
        ylo = P.lo[1];
        yhi = P.hi[1];
      }
      long long zlo = P.lo[2] + bzA * P.BF[2], zhi = P.lo[2] + (bzB + 1) * P.BF[2];
      if (zhi > P.hi[2]) zhi = P.hi[2];
      long long y0 = ylo + F.oy_min, y1 = yhi + F.oy_max, z0 = zlo + F.oz_min, z1 = zhi + F.oz_max;
      if (y0 < 0) y0 = 0;
      if (z0 < 0) z0 = 0;
      if (y1 > F.ext[1]) y1 = F.ext[1];
      if (z1 > F.ext[2]) z1 = F.ext[2];
      DRowInfo ri;
      ri.y0 = y0;
      ri.ny = y1 > y0 ? y1 - y0 : 0;
      ri.z0 = z0;
      ri.nz = z1 > z0 ? z1 - z0 : 0;
      if (F.g_end == F.g_begin) ri.ny = ri.nz = 0;
      ri.ppc = 1;
      ri.nseg = ri.ny > 0 ? (ri.ny + kRowSeg - 1) / kRowSeg : 1;
      ri.n_chunks = ri.ny > 0 ? ri.nz * ri.nseg : 0;   // as the owner (the join below drops a sharer's)
      ri.chunk_begin = 0;
      s_ri[fi] = ri;
    }
#ifdef WS_PLAN_CLOCK
    atomicMax(&s_wclk[1], (unsigned long long)(clock64() - s_clk[0]));
#endif
    wbar();
    if (tid == 0) {
      long long cb = 0, npl = 0;
      for (int fi = 0; fi < K.n_fields; ++fi)
        if (s_ri[fi].n_chunks > 0) npl += s_ri[fi].nz;
      // up to 8 planes per worker thread: one-plane windows, the direct plane_rep test (clock
      // probes: a window walk costs a thread more than 4-8 direct tests when the zone boundaries
      // cluster, BJ configs[1] (1,16,64)+2z: 18k vs 9k cycles); more (LBM: 32 fields x ~260
      // planes): 8-plane windows walked by zone segments (38k -> 10-20k cycles)
      const int wsh = npl <= 8 * kPlanWork ? 0 : 3;
      int zo = 0;
      for (int fi = 0; fi < K.n_fields; ++fi) {
        s_ri[fi].chunk_begin = cb;
        cb += s_ri[fi].n_chunks;
        s_zoff[fi] = zo;
        if (s_ri[fi].n_chunks > 0) zo += (int)((s_ri[fi].nz + (1 << wsh) - 1) >> wsh);
      }
      s_zoff[K.n_fields] = zo;
      s_wsh = wsh;
      s_nri = 0;
#ifdef WS_PLAN_CLOCK
      s_wclk[2] = (unsigned long long)(clock64() - s_clk[0]);
#endif
    }
    wbar();
    // k_rows items: the chunks of computed planes (plane_rep(z) == z), listed per configuration;
    // derived planes are folded from their representative by k_fold (same rule).  The (field,
    // 8-plane window) pairs of all fields are one flat range over the worker threads; a window is
    // walked by zone segments (plane_seg): the first `per` planes of a segment are computed, the
    // rest of it is skipped at once (LBM, deep blocks: most planes are derived)
    const int nzt = s_zoff[K.n_fields];
    int fi = 0;
    for (int t = tid; t < nzt; t += kPlanWork) {
      while (s_zoff[fi + 1] <= t) ++fi;   // t ascends per thread: the field index only advances
      const DRowInfo& ri = s_ri[fi];
      const DField& F = K.f[fi];
      long long py, pz, falign;
      field_rows(F, P, ll, py, pz, falign);
      const int per = plane_period(pz, F.lg_elem, ll);
      const int zw = (int)ri.z0 + ((t - s_zoff[fi]) << s_wsh), ze = min(zw + (1 << s_wsh), (int)(ri.z0 + ri.nz));
      unsigned cm = 0u;   // computed planes of the window (bit z - zw)
      if (per <= 0) {
        cm = (1u << (ze - zw)) - 1u;
      } else if (ze - zw == 1) {   // one plane: the direct test
        cm = plane_rep_f(F, K.g + F.g_begin, zw, (int)ri.z0, (int)P.lo[2], (int)P.hi[2], (int)P.BF[2], P.fd_BF[2],
                         per) == zw ? 1u : 0u;
      } else {
        for (int z = zw; z < ze;) {
          int seg;
          const int nb = plane_seg(F, K.g + F.g_begin, z, (int)ri.z0, (int)P.lo[2], (int)P.hi[2], (int)P.BF[2],
                                   P.fd_BF[2], seg);
          const int hi = nb < ze ? nb : ze;
          const int ce = seg + per < hi ? seg + per : hi;   // computed planes [z, ce)
          if (ce > z) cm |= ((1u << (ce - zw)) - 1u) & ~((1u << (z - zw)) - 1u);
          z = hi;
        }
      }
      if (cm == 0u) continue;
      const int ncp = __popc(cm);
      const int at = atomicAdd(&s_nri, ncp * (int)ri.nseg);
      for (int i = 0; i < ncp; ++i) {
        const int b = __fns(cm, 0, i + 1);
        const long long zi = zw + b - ri.z0;
        for (int sg = 0; sg < (int)ri.nseg; ++sg) {
          const int slot = at + i * (int)ri.nseg + sg;
          WS_CHK(slot, g_caps.clist_stride);
          WS_CHK((long long)c * clist_stride + slot, g_caps.max_chunks);
          cl[slot] = ((uint32_t)fi << 26) | (uint32_t)(ri.chunk_begin + zi * ri.nseg + sg);
        }
      }
    }
#ifdef WS_PLAN_CLOCK
    atomicMax(&s_wclk[3], (unsigned long long)(clock64() - s_clk[0]));
#endif
  }
#ifdef WS_PLAN_CLOCK
  if (tid == 0) s_clk[2] = clock64();
#endif
  __syncthreads();   // join: the claim's row_owner, the workers' boxes and lists
  if (tid == 0) {
    const bool owner = P.row_owner == c;
    long long cb = 0;
    for (int fi = 0; fi < K.n_fields; ++fi) {
      if (!owner) {   // sharer: the owner's rows (no k_rows / k_fold items)
        s_ri[fi].n_chunks = 0;
        s_ri[fi].chunk_begin = 0;
      }
      cb += s_ri[fi].n_chunks;
    }
    P.n_warp_items = (P.rep_mult ? 1 : P.W) * P.nwarps;
    P.n_wclass_items = 0;
    P.n_set_items = P.rep_mult ? 1 : P.nsets;
    // k_spairs items: the sets j < nsets of >= 2 members, i.e. j < W - n_sm (members j + m * n_sm < W)
    P.n_sclass_items = (P.scls_R > 0 && !P.rep_mult && P.W > P.nsets) ? min(P.nsets, P.W - P.nsets) : 0;
    P.n_chunks = cb;
    P.n_fields = owner ? K.n_fields : 0;   // k_fold items
    P.n_sect_items = (P.want_pages || P.want_sect) ? K.n_fields : 0;
    P.n_ritems = owner ? s_nri : 0;
    // the row chain's items: reserve this owner's ranges (row items, chunk slots, fold items)
    s_rb[0] = owner ? atomicAdd(rctr + par * 4 + 0, (unsigned long long)P.n_ritems) : 0ull;
    P.chunk_base = owner ? (long long)atomicAdd(rctr + par * 4 + 1, (unsigned long long)cb) : 0ll;
    s_rb[1] = owner ? atomicAdd(rctr + par * 4 + 2, (unsigned long long)P.n_fields) : 0ull;
#ifdef WS_PLAN_CLOCK
    s_clk[3] = clock64();
#endif
  }
  __syncthreads();
  for (int fi = tid; fi < K.n_fields; fi += blockDim.x) rowinfo[(long long)c * kMaxFields + fi] = s_ri[fi];
  for (long long i = tid; i < P.n_ritems; i += blockDim.x) {
    WS_CHK(s_rb[0] + i, g_caps.max_chunks);
    ritems[s_rb[0] + i] = ((unsigned long long)c << 32) | (unsigned long long)cl[i];
  }
  for (int fi = tid; fi < (int)P.n_fields; fi += blockDim.x) {
    WS_CHK(s_rb[1] + fi, g_caps.fitems);
    fitems[s_rb[1] + fi] = ((uint32_t)c << 6) | (uint32_t)fi;
  }
  PLAN_MARK()
  store_plan();
  PLAN_MARK()
#ifdef WS_PLAN_CLOCK
  if (tid == 0 && (c == 0 || c == n - 1)) {
    printf("PLANCLK c=%d claim %lld workers %lld (ranges %llu boxes %llu prefix %llu list %llu) join %lld owner %d "
           "nri %lld nf %d b=(%d,%d,%d) f=(%d,%d,%d) nz0 %lld nseg0 %lld wsh %d nzt %d |", c, s_clk[1] - s_clk[0],
           s_clk[2] - s_clk[0], s_wclk[0], s_wclk[1], s_wclk[2], s_wclk[3], s_clk[3] - s_clk[0],
           (int)(P.row_owner == c), (long long)P.n_ritems, K.n_fields, P.b[0], P.b[1], P.b[2], P.f[0], P.f[1], P.f[2],
           (long long)s_ri[0].nz, (long long)s_ri[0].nseg, s_wsh, s_zoff[K.n_fields]);
    for (int i = 1; i < nclk; ++i) printf(" %lld", clk[i] - clk[i - 1]);
    printf(" total %lld\n", clk[nclk - 1] - clk[0]);
  }
#endif
}

// ------------------------------------------------------------------ scan of work counts


// ------------------------------------------------------------------ a2 + a3: warp instructions
struct Lane {
  long long base[3];
  unsigned long long act;  // active folded cells (guard clipping)
  bool valid;              // thread index < T
};

__device__ __forceinline__ unsigned bm_all(bool p) { return __ballot_sync(FULL, p); }

__device__ __forceinline__ unsigned long long full_cube(int fc) { return fc == 64 ? ~0ull : ((1ull << fc) - 1ull); }

__device__ __forceinline__ Lane lane_setup(const DPlan& P, long long B, int w, int lane) {
  Lane L;
  const long long bc[3] = {B % P.G[0], (B / P.G[0]) % P.G[1], B / (P.G[0] * P.G[1])};
  const int t = w * 32 + lane;
  L.valid = t < P.T;
  const int tc[3] = {t % P.b[0], (t / P.b[0]) % P.b[1], t / (P.b[0] * P.b[1])};
  long long lim[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    L.base[d] = P.lo[d] + (bc[d] * P.b[d] + tc[d]) * P.f[d];
    lim[d] = P.hi[d] - L.base[d];
  }
  L.act = 0;
  if (L.valid && lim[0] > 0 && lim[1] > 0 && lim[2] > 0) {
    if (lim[0] >= P.f[0] && lim[1] >= P.f[1] && lim[2] >= P.f[2]) {
      L.act = full_cube(P.fcube);
    } else {
      for (int q = 0; q < P.fcube; ++q) {
        int kx, ky, kz;
        decode_kappa(q, P.f, kx, ky, kz);
        if (kx < lim[0] && ky < lim[1] && kz < lim[2]) L.act |= 1ull << q;
      }
    }
  }
  return L;
}

// Every instruction of one warp: unique sectors per warp instruction (the
// issuing lanes are address-sorted, so comparing with the previous issuing lane
// dedupes) and half-warp wavefronts (unique bank words, greedy 1024 B
// clusters, max bank multiplicity).  Wavefronts, loop-free when every run of
// unique words between gaps >= the pair window spans less than the window (then
// the greedy clusters are exactly those runs): sum over clusters of the max bank
// multiplicity = number of distinct (cluster, rank-within-bank) pairs.  Otherwise
// the greedy split is walked cluster by cluster.  Returns warp totals in lane 0.
__device__ void eval_warp(const DPlan& P, const DKernel& K, const DGpu& G, const DInstr* __restrict__ tab,
                          const Lane& L, int lane, long long& lup, long long& wf_out, long long& req_ld,
                          long long& req_st) {
  const unsigned lt_mask = (1u << lane) - 1u, le_mask = lt_mask | (1u << lane);
  const int lg_sec = G.lg_sector, lg_bank = G.lg_bank, lg_hw = G.lg_hw;
  const long long bank_bytes = G.g.bank_bytes, window = G.g.pair_window_bytes;
  const int nbm = (int)G.g.n_banks - 1;
  const unsigned hbits = (lg_hw == 5 ? FULL : ((1u << (1 << lg_hw)) - 1u)) << ((lane >> lg_hw) << lg_hw);
  const bool hleader = (lane & ((1 << lg_hw) - 1)) == 0;
  long long wf_u = 0, wf_l = 0;  // warp-uniform part / per half-warp-leader part
  req_ld = req_st = 0;
  int cur_field = -1;
  long long plane = 0;
  const int ni = P.n_instr;
  // the instruction table in chunks of 32 entries, one per lane (one coalesced load round per
  // chunk), broadcast by shuffles: no dependent global load per instruction
  long long mC = 0;
  unsigned long long mK = 0;
  int mF = 0;
  for (int i = 0; i < ni; ++i) {
    if ((i & 31) == 0) {
      if (i + lane < ni) {
        const DInstr me = tab[i + lane];
        mC = me.C;
        mK = me.kmask;
        mF = me.field | (me.kind << 8) | (me.lg_elem << 16);
      }
    }
    DInstr cur;
    cur.C = shfl64(mC, i & 31);
    cur.kmask = (unsigned long long)shfl64((long long)mK, i & 31);
    {
      const int pk = __shfl_sync(FULL, mF, i & 31);
      cur.field = pk & 255;
      cur.kind = (pk >> 8) & 255;
      cur.lg_elem = pk >> 16;
    }
    const bool iss = (cur.kmask & L.act) != 0ull;
    const unsigned m = __ballot_sync(FULL, iss);
    if (m == 0u) continue;
    if (cur.field != cur_field) {
      cur_field = cur.field;
      const DField& F = K.f[cur.field];
      plane = L.base[0] + F.pitch[1] * L.base[1] + F.pitch[2] * L.base[2];
    }
    const long long A = cur.C + (plane << cur.lg_elem);
    const long long sec = A >> lg_sec;
    const unsigned pm = m & lt_mask;
    const long long psec = shfl64(sec, pm ? 31 - __clz(pm) : lane);
    const bool us = iss && (pm == 0u || psec != sec);
    const int cnt = __popc(__ballot_sync(FULL, us));
    if (cur.kind) req_st += cnt;
    else req_ld += cnt;
    const long long word = A >> lg_bank;
    const unsigned pmh = m & hbits & lt_mask;
    const long long pword = shfl64(word, pmh ? 31 - __clz(pmh) : lane);
    const bool uw = iss && (pmh == 0u || pword != word);
    const bool bnd = uw && (pmh == 0u || (word - pword) * bank_bytes >= window);
    const unsigned bm = __ballot_sync(FULL, bnd) & hbits & le_mask;
    const int sl = bm ? 31 - __clz(bm) : lane;
    const long long sword = shfl64(word, sl);
    const bool longseg = uw && (word - sword) * bank_bytes >= window;
    if (!__any_sync(FULL, longseg)) {
      // a cluster spanning fewer than n_banks words has every bank at most once
      if (!__any_sync(FULL, uw && (word - sword) > (long long)nbm)) {
        wf_u += __popc(bm_all(bnd));
        continue;
      }
      const int bank = (int)(word & nbm);
      const unsigned peers = __match_any_sync(FULL, uw ? (unsigned)(bank | (sl << 8)) : (0x10000u | (unsigned)lane));
      const int rank = __popc(peers & le_mask);
      const unsigned p2 = __match_any_sync(FULL, uw ? (unsigned)(rank | (sl << 8)) : (0x10000u | (unsigned)lane));
      wf_u += __popc(__ballot_sync(FULL, uw && (p2 & lt_mask) == 0u));
      continue;
    }
    unsigned rem = __ballot_sync(FULL, uw) & hbits;
    while (__any_sync(FULL, rem != 0u)) {
      const int first = rem ? __ffs(rem) - 1 : lane;
      const long long cs = shfl64(word, first);
      const bool inC = ((rem >> lane) & 1u) && ((word - cs) * bank_bytes < window);
      const unsigned cm = __ballot_sync(FULL, inC) & hbits;
      const int bank = (int)(word & nbm);
      const unsigned key = inC ? (unsigned)(bank | ((lane >> lg_hw) << 8)) : (0x10000u | (unsigned)lane);
      const unsigned peers = __match_any_sync(FULL, key);
      int cb = inC ? __popc(peers) : 0;
      for (int o = (1 << lg_hw) >> 1; o >= 1; o >>= 1) cb = max(cb, __shfl_xor_sync(FULL, cb, o));
      if (hleader && rem != 0u) wf_l += cb;
      rem &= ~cm;
    }
  }
  lup = L.valid ? __popcll(L.act) : 0;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    lup += shfl64_down(lup, o);
    wf_l += shfl64_down(wf_l, o);
  }
  wf_out = wf_l + wf_u;
}

__device__ __forceinline__ void add_warp_stats(unsigned long long* a, long long mult, long long lup, long long wf,
                                               long long rl, long long rs) {
  if (lup) atomicAdd(a + A_LUP, (unsigned long long)(lup * mult));
  if (wf) atomicAdd(a + A_WF, (unsigned long long)(wf * mult));
  if (rl) atomicAdd(a + A_REQ_LD, (unsigned long long)(rl * mult));
  if (rs) atomicAdd(a + A_REQ_ST, (unsigned long long)(rs * mult));
}

// clip pattern of a block: bit d set when it is the partial last block along d
__device__ __forceinline__ int clip_pattern(const DPlan& P, const long long* bc) {
  int pat = 0;
#pragma unroll
  for (int d = 0; d < 3; ++d)
    if (P.part[d] != 0 && bc[d] == P.G[d] - 1) pat |= 1 << d;
  return pat;
}

// Pass 1 over every wave warp.  Two warps with the same warp index, the same clip
// pattern of their block (hence identical lane activity) and the same base address
// residue mod M = max(sector, bank_bytes*n_banks) are translates by a multiple of M:
// identical sector, bank and cluster statistics.
// With classes enabled the warp is only counted into its class (first member
// appends the class to a compact list); otherwise it is evaluated here.
__global__ void __launch_bounds__(256) k_warp(const DPlan* __restrict__ plans, const DPrefix* __restrict__ pre, int n,
                                              const DInstr* __restrict__ instr, const DKernel* __restrict__ ks,
                                              const DGpu* __restrict__ gs, unsigned long long* __restrict__ acc,
                                              unsigned int* __restrict__ wcnt, unsigned long long* __restrict__ wrep,
                                              unsigned long long* __restrict__ lists,
                                              unsigned long long* __restrict__ wlist,
                                              unsigned long long* __restrict__ work) {
  PDL_PROLOGUE();
  const long long total = pre[n].warp;
  const int lane = threadIdx.x & 31;
  unsigned long long my_units = 0;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  int c0 = -1;
  // each lane classifies one wave warp; warps of configs without classes are then
  // evaluated cooperatively by the whole warp
  for (long long base = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < total; base += nw * 32) {
    const long long item = base + lane;
    const bool have = item < total;
    int c = 0;
    bool direct = false;
    unsigned long long key = ~0ull;
    long long B = 0;
    int wrep_w = 0;
    // one search per warp (lanes hold consecutive items), then each lane advances
    c0 = find_config_warp<0>(pre, n, base, c0);
    if (have) {
      c = c0;
      while (c + 1 < n && pre[c + 1].warp <= item) ++c;
      const DPlan& P = plans[c];
      const long long wi = item - pre[c].warp;
      B = P.s + wi / P.nwarps;
      const int w = (int)(wi % P.nwarps);
      wrep_w = w;
      if (P.wcls_R > 0) {
        const long long bc[3] = {B % P.G[0], (B / P.G[0]) % P.G[1], B / (P.G[0] * P.G[1])};
        const int t0 = w * 32;
        const long long tc[3] = {t0 % P.b[0], (t0 / P.b[0]) % P.b[1], t0 / (P.b[0] * P.b[1])};
        long long pl = 0;
#pragma unroll
        for (int d = 0; d < 3; ++d) pl += P.cls_pitch[d] * (P.lo[d] + (bc[d] * P.b[d] + tc[d]) * P.f[d]);
        const int res = (int)(pl & (P.wcls_R - 1));  // (pl * elem) mod M, in elements
        int pat = clip_pattern(P, bc);
        // power-of-two blocks: every warp covers an aligned sub-box with the same relative lane
        // pattern, so in an unclipped block the warp index does not matter; in a clipped block a
        // warp whose every folded cell is inside the domain is such a warp too, and a warp with
        // no active cell contributes nothing
        bool skip = false;
        if (P.wpow2 && pat != 0) {
          long long ext[3];  // thread extent of the warp's aligned sub-box
          ext[0] = P.b[0] < 32 ? P.b[0] : 32;
          ext[1] = P.b[0] >= 32 ? 1 : (P.b[0] * P.b[1] >= 32 ? 32 / P.b[0] : P.b[1]);
          ext[2] = 32 / (ext[0] * ext[1]);
          bool full = true, none = false;
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const long long c0 = P.lo[d] + (bc[d] * P.b[d] + tc[d]) * P.f[d];
            if (c0 + ext[d] * P.f[d] > P.hi[d]) full = false;
            if (c0 >= P.hi[d]) none = true;
          }
          if (none) skip = true;
          else if (full) pat = 0;
        }
        const int wk = (P.wpow2 && pat == 0) ? 0 : w;
        const unsigned slot = (unsigned)(((wk * 64 + res) << 3) | pat);
        if (!skip) key = ((unsigned long long)c << 32) | slot;
        my_units += 32;
      } else {
        direct = true;
      }
    }
    // one atomic per distinct class among the lanes
    const unsigned peers = __match_any_sync(FULL, key);
    if (key != ~0ull && (peers & ((1u << lane) - 1u)) == 0u) {
      const int cc = (int)(key >> 32);
      const unsigned slot = (unsigned)(key & 0xffffffffu);
      const long long gslot = (long long)cc * kWSlots + slot;
      WS_CHK(slot, kWSlots);
      WS_CHK(gslot, g_caps.wslots);
      if (atomicAdd(wcnt + gslot, (unsigned)__popc(peers)) == 0u) {
        wrep[gslot] = ((unsigned long long)B << 5) | (unsigned long long)wrep_w;
        const unsigned long long idx = atomicAdd(lists + 0, 1ull);
        WS_CHK(idx, g_caps.wslots);
        wlist[idx] = key;
      }
    }
    unsigned dm = __ballot_sync(FULL, direct);
    while (dm) {
      const int src = __ffs(dm) - 1;
      dm &= dm - 1;
      const long long it = shfl64(item, src);
      const int cc = __shfl_sync(FULL, c, src);
      const DPlan& P = plans[cc];
      const long long wi = it - pre[cc].warp;
      const Lane L = lane_setup(P, P.rep_mult ? P.rep_B : P.s + wi / P.nwarps, (int)(wi % P.nwarps), lane);
      long long lup, wf, rl, rs;
      eval_warp(P, ks[P.kid], gs[P.gid], instr + (long long)cc * kMaxInstr, L, lane, lup, wf, rl, rs);
      if (lane == 0) {
        add_warp_stats(acc + (long long)cc * A_N, P.rep_mult ? P.rep_mult : 1, lup, wf, rl, rs);
        my_units += 32ull * (unsigned long long)P.n_instr;
      }
    }
  }
  // per-warp total of the units counted by the lanes
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) my_units += __shfl_down_sync(FULL, my_units, o);
  if (lane == 0 && my_units) atomicAdd(work + K_WARP, my_units);
}

// Pass 2: one representative warp per class, counted class-size times.
__global__ void __launch_bounds__(256) k_wclass(const DPlan* __restrict__ plans, const DInstr* __restrict__ instr,
                                                const DKernel* __restrict__ ks, const DGpu* __restrict__ gs,
                                                unsigned long long* __restrict__ acc,
                                                unsigned int* __restrict__ wcnt,
                                                const unsigned long long* __restrict__ wrep,
                                                const unsigned long long* __restrict__ lists,
                                                const unsigned long long* __restrict__ wlist,
                                                unsigned long long* __restrict__ work) {
  PDL_PROLOGUE();
  const long long total = (long long)lists[0];
  const int lane = threadIdx.x & 31;
  unsigned long long my_units = 0;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < total; item += nw) {
    const unsigned long long ent = wlist[item];
    const int c = (int)(ent >> 32);
    const unsigned slot = (unsigned)(ent & 0xffffffffu);
    const DPlan& P = plans[c];
    const long long gslot = (long long)c * kWSlots + slot;
    WS_CHK(gslot, g_caps.wslots);
    unsigned int cnt = 0;
    if (lane == 0) {  // the class size; the slot returns to 0 for the next call (k_instr no longer zeroes)
      cnt = wcnt[gslot];
      wcnt[gslot] = 0u;
    }
    const long long B = (long long)(wrep[gslot] >> 5);
    const int w = (int)(wrep[gslot] & 31ull);
    const Lane L = lane_setup(P, B, w, lane);
    long long lup, wf, rl, rs;
    eval_warp(P, ks[P.kid], gs[P.gid], instr + (long long)c * kMaxInstr, L, lane, lup, wf, rl, rs);
    if (lane == 0) add_warp_stats(acc + (long long)c * A_N, cnt, lup, wf, rl, rs);
    my_units += 32ull * (unsigned long long)P.n_instr;
  }
  if (lane == 0 && my_units) atomicAdd(work + K_WCLASS, my_units);
}

// ------------------------------------------------------------------ a4: SM-resident block sets
struct SmBox {
  long long x0, x1, y0, y1, z0, z1;  // active cell box of one member block (clipped to the domain)
};
constexpr int kMaxMembers = 32;

struct SmBox32 {
  int x0, x1, y0, y1, z0, z1;
};

// One block (single-block SM-set class of a kernel with many load fields, LBM): fields are
// independent (they never alias), so each warp takes whole fields -- the field's footprint box
// rows in contiguous lane chunks, per row the union of the load groups' x-intervals, an ordered
// warp reduction of (sectors, lines) -- and the per-field counts add up (shared atomics).  No
// CTA barrier per field (smset_eval's flat rows synchronise the CTA twice per field).
__device__ void smset_eval_warps(const DPlan& P, const DKernel& K, const DGpu& G, long long S0,
                                 unsigned long long* s_sum, unsigned long long& sum_s, unsigned long long& sum_l,
                                 unsigned long long& units) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int lg_sec = G.lg_sector, lg_line = G.lg_line;
  const long long bc[3] = {S0 % P.G[0], (S0 / P.G[0]) % P.G[1], S0 / (P.G[0] * P.G[1])};
  long long lo[3], hi[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    lo[d] = P.lo[d] + bc[d] * P.BF[d];
    hi[d] = lo[d] + P.BF[d];
    if (hi[d] > P.hi[d]) hi[d] = P.hi[d];
  }
  if (threadIdx.x < 3) s_sum[threadIdx.x] = 0ull;
  __syncthreads();
  unsigned long long my_s = 0, my_l = 0, my_u = 0;
  for (int fi = wid; fi < K.n_fields; fi += nw) {
    const DField& F = K.f[fi];
    if (!(F.kinds & 1)) continue;
    long long y0 = lo[1] + F.ld_oy_min, y1 = hi[1] + F.ld_oy_max, z0 = lo[2] + F.ld_oz_min, z1 = hi[2] + F.ld_oz_max;
    if (y0 < 0) y0 = 0;
    if (z0 < 0) z0 = 0;
    if (y1 > F.ext[1]) y1 = F.ext[1];
    if (z1 > F.ext[2]) z1 = F.ext[2];
    const long long ny = y1 > y0 ? y1 - y0 : 0, nz = z1 > z0 ? z1 - z0 : 0, rows = ny * nz;
    if (rows == 0) continue;
    my_u += (unsigned long long)rows;
    const long long align = F.align, py = F.pitch[1], pz = F.pitch[2];
    const int le = F.lg_elem;
    const long long step = py << le;
    // lanes take contiguous planes; in a plane the rows split into runs between the groups'
    // y edges (lo1 + oy, hi1 + oy), the rows of a run have the same candidates and are
    // translates by the row pitch: run_triple evaluates one period of them
    const long long pper = (nz + 31) / 32;
    Tri t[2] = {tri_empty(), tri_empty()};
    for (long long z = z0 + lane * pper; z < z1 && z < z0 + (lane + 1) * pper; ++z) {
      long long cur = y0;
      while (cur < y1) {
        unsigned mk = 0;   // runs whose group's cell row (y - oy, z - oz) lies in the block
        long long nxt = y1;
        for (int g = F.g_begin; g < F.g_end; ++g) {
          const DGroup gr = K.g[g];
          const long long zz = z - gr.oz;
          if (gr.kind != 0 || zz < lo[2] || zz >= hi[2]) continue;
          const long long ya = lo[1] + gr.oy, yb = hi[1] + gr.oy;
          if (cur >= ya && cur < yb) {
            mk |= 1u << gr.run;
            nxt = yb < nxt ? yb : nxt;
          } else if (ya > cur && ya < nxt) {
            nxt = ya;
          }
        }
        if (mk) {
          const long long R0 = align + ((py * cur + pz * z) << le);
          auto gen = [&](auto&& cb) {
            unsigned q = mk;
            while (q) {
              const int b = __ffs(q) - 1;
              q &= q - 1;
              cb(lo[0] + F.run_lo[b], hi[0] + F.run_hi[b]);
            }
          };
          const int run = (int)(nxt - cur);
          t[0] = tri_combine(t[0], run_triple([&](int r) {
            Tri x = tri_empty();
            row_union(gen, R0 + r * step, le, lg_sec, lg_line, &x, nullptr);
            return x;
          }, step, run, lg_sec));
          t[1] = tri_combine(t[1], run_triple([&](int r) {
            Tri x = tri_empty();
            row_union(gen, R0 + r * step, le, lg_sec, lg_line, nullptr, &x);
            return x;
          }, step, run, lg_line));
        }
        cur = nxt;
      }
    }
    warp_ordered_reduce<2>(t);
    if (lane == 0) {
      my_s += (unsigned long long)t[0].c;
      my_l += (unsigned long long)t[1].c;
    }
  }
  if (lane == 0) {
    if (my_s) atomicAdd(&s_sum[0], my_s);
    if (my_l) atomicAdd(&s_sum[1], my_l);
    if (my_u) atomicAdd(&s_sum[2], my_u);
  }
  __syncthreads();
  sum_s = s_sum[0];
  sum_l = s_sum[1];
  units = s_sum[2];
  __syncthreads();
}

// ---- 32-bit plane-relative arithmetic for k_rows ---------------------------------------------
// Every address of one z-plane of a field is R0p + rel with R0p the address of the plane's first
// box row and 0 <= rel < 2^31 (describe-time limit: pitch[2] * elem_bytes < 2^31).  Sectors and
// lines are counted relative to B = floor(R0p / line_bytes) * line_bytes, a multiple of both unit
// sizes: unit(R0p + rel) = (B >> sh) + ((off0 + rel) >> sh) with off0 = R0p - B < line_bytes.
struct T32 {
  int f, l, c;  // first, last, count; c == 0: empty
};
__device__ __forceinline__ T32 t32_empty() { return T32{0, 0, 0}; }
__device__ __forceinline__ void t32_add(T32& t, int s0, int s1) {
  if (t.c == 0) {
    t.f = s0;
    t.c = s1 - s0 + 1;
  } else {
    t.c += s1 - s0 + 1 - (t.l == s0 ? 1 : 0);
  }
  t.l = s1;
}
__device__ __forceinline__ T32 t32_combine(const T32& a, const T32& b) {
#ifndef WS_T32_BRANCHY
  // branch-free (selects): the lanes of a warp combine different triples without diverging
  const bool ea = a.c == 0, eb = b.c == 0;
  return T32{ea ? b.f : a.f, eb ? a.l : b.l, a.c + b.c - ((!ea && !eb && a.l == b.f) ? 1 : 0)};
#else
  if (a.c == 0) return b;
  if (b.c == 0) return a;
  return T32{a.f, b.l, a.c + b.c - (a.l == b.f ? 1 : 0)};
#endif
}

// union of the intervals [xs, xe) produced by gen, in the row starting at plane offset R
template <class Gen>
__device__ __forceinline__ void row_union32(const Gen& gen, int R, int le, int sh, T32& t) {
  const int INF = 0x7fffffff;
  int start = INF, mx_s = -INF, mn_e = INF, mx_e = -INF;
  gen([&](int xs, int xe) {
    start = xs < start ? xs : start;
    mx_s = xs > mx_s ? xs : mx_s;
    mn_e = xe < mn_e ? xe : mn_e;
    mx_e = xe > mx_e ? xe : mx_e;
  });
  if (start == INF) return;
  if (mx_s <= mn_e) {
    t32_add(t, (R + (start << le)) >> sh, (R + ((mx_e - 1) << le)) >> sh);
    return;
  }
  while (start != INF) {
    int end = start, nxt;
    bool grew;
    do {
      grew = false;
      nxt = INF;
      gen([&](int xs, int xe) {
        if (xs <= end) {
          if (xe > end) {
            end = xe;
            grew = true;
          }
        } else if (xs < nxt) {
          nxt = xs;
        }
      });
    } while (grew);
    t32_add(t, (R + (start << le)) >> sh, (R + ((end - 1) << le)) >> sh);
    start = nxt;
  }
}

// run_triple (above) in 32-bit: rows r and r+P are translates by D = P*step >> sh units
template <class RowFn>
__device__ __forceinline__ T32 run_triple32(const RowFn& row, int step, int run, int sh) {
  const int tz = step == 0 ? 31 : __ffs(step) - 1;
  const int P = sh > tz ? 1 << (sh - tz) : 1;
  if (run <= 2 * P) {
    T32 acc = t32_empty();
    for (int r = 0; r < run; ++r) acc = t32_combine(acc, row(r));
    return acc;
  }
  const int nb = run / P, rem = run % P;
  const int D = (P * step) >> sh;
  T32 blk = t32_empty(), remb = t32_empty();
  for (int i = 0; i < P; ++i) {
    const T32 rt = row(i);
    blk = t32_combine(blk, rt);
    if (i < rem) remb = t32_combine(remb, rt);
  }
  if (blk.c == 0) return blk;
  const int adj = blk.l == blk.f + D ? 1 : 0;
  T32 acc{blk.f, blk.l + (nb - 1) * D, nb * blk.c - (nb - 1) * adj};
  if (remb.c) acc = t32_combine(acc, T32{remb.f + nb * D, remb.l + nb * D, remb.c});
  return acc;
}

// lanes [0, cnt) hold data (lanes >= cnt empty): steps with offset >= cnt are no-ops
template <int NQ>
__device__ __forceinline__ void warp_ordered_reduce32(T32 (&t)[NQ], int cnt = 32) {
  // as warp_ordered_reduce (sum of counts minus the consecutive-pair overlaps), 32-bit sums in one
  // redux instruction each; cnt (lanes holding data) is no longer needed
  (void)cnt;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const bool ne = t[q].c != 0;
    const unsigned m = __ballot_sync(FULL, ne);
    if (m == 0u) {
      t[q] = t32_empty();
      continue;
    }
    const unsigned below = m & lt;
    const int lprev = __shfl_sync(FULL, t[q].l, below ? 31 - __clz(below) : lane);
    const unsigned dup = (ne && below && lprev == t[q].f) ? 1u : 0u;
    const unsigned cs = __reduce_add_sync(FULL, (unsigned)t[q].c) - __reduce_add_sync(FULL, dup);
    t[q] = T32{__shfl_sync(FULL, t[q].f, __ffs(m) - 1), __shfl_sync(FULL, t[q].l, 31 - __clz(m)), (int)cs};
  }
}


struct T32x2 {
  T32 s, l;
};

constexpr int kMaxPlanes = 256;   // planes per segment of the SM-set plane fold
// rows of a plane per SM-set run segment (per-warp shared arrays: fewer rows for wider CTAs)
constexpr int kSegRowsS = WS_SCLASS_THREADS <= 256 ? 1024 : (WS_SCLASS_THREADS <= 512 ? 512 : 256);

// One run of rows [y, y + run) of plane z (row y at plane offset R0): candidates of its first
// row (member boxes x offset groups), their union, the run's sector and line triples.
__device__ __noinline__ T32x2 smset_run(const SmBox32* mb, int nm, const DKernel& K, const DField& F, int g0, int ng,
                                        int y, int z, int R0, int step, int run, int le, int ls, int ll) {
  unsigned long long mk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int g = 0; g < ng; ++g) {
    const DGroup gr = K.g[g0 + g];
    if (gr.kind != 0) continue;
    const int yy = y - gr.oy, zz = z - gr.oz;
#pragma unroll 4
    for (int m = 0; m < nm; ++m) {
      const SmBox32& bx = mb[m];
      if (yy >= bx.y0 && yy < bx.y1 && zz >= bx.z0 && zz < bx.z1) mk[m >> 2] |= 1ull << ((m & 3) * 16 + gr.run);
    }
  }
  auto gen = [&](auto&& cb) {
    for (int w = 0; w < ((nm + 3) >> 2); ++w) {
      unsigned long long q = mk[w];
      while (q) {
        const int bb = __ffsll((long long)q) - 1;
        q &= q - 1;
        const SmBox32& bx = mb[w * 4 + (bb >> 4)];
        cb(bx.x0 + F.run_lo[bb & 15], bx.x1 + F.run_hi[bb & 15]);
      }
    }
  };
  const int INF = 0x7fffffff;
  int mn_s = INF, mx_s = -INF, mn_e = INF, mx_e = -INF;
  gen([&](int xs, int xe) {
    mn_s = xs < mn_s ? xs : mn_s;
    mx_s = xs > mx_s ? xs : mx_s;
    mn_e = xe < mn_e ? xe : mn_e;
    mx_e = xe > mx_e ? xe : mx_e;
  });
  T32x2 o{t32_empty(), t32_empty()};
  if (mn_s == INF) return o;
  if (mx_s <= mn_e) {
    const int a0 = R0 + (mn_s << le), a1 = R0 + ((mx_e - 1) << le);
    o.s = run_triple32([&](int r) {
      const int s0 = (a0 + r * step) >> ls, s1 = (a1 + r * step) >> ls;
      return T32{s0, s1, s1 - s0 + 1};
    }, step, run, ls);
    o.l = run_triple32([&](int r) {
      const int s0 = (a0 + r * step) >> ll, s1 = (a1 + r * step) >> ll;
      return T32{s0, s1, s1 - s0 + 1};
    }, step, run, ll);
  } else {
    o.s = run_triple32([&](int r) {
      T32 x = t32_empty();
      row_union32(gen, R0 + r * step, le, ls, x);
      return x;
    }, step, run, ls);
    o.l = run_triple32([&](int r) {
      T32 x = t32_empty();
      row_union32(gen, R0 + r * step, le, ll, x);
      return x;
    }, step, run, ll);
  }
  return o;
}
// smset_run over the plane's active (group, member) pairs only (SmWarp::gm / gl): a member box
// that the group's plane z - oz misses contributes nothing to any row of the plane
__device__ __noinline__ T32x2 smset_run_g(const SmBox32* mb, int nm, const unsigned* gm, const unsigned char* gl,
                                          int ngl, const DKernel& K, const DField& F, int g0, int y, int R0, int step,
                                          int run, int le, int ls, int ll) {
  unsigned long long mk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < ngl; ++i) {
    const DGroup gr = K.g[g0 + gl[i]];
    const int yy = y - gr.oy;
    unsigned q = gm[i];
    while (q) {
      const int m = __ffs(q) - 1;
      q &= q - 1;
      const SmBox32& bx = mb[m];
      if (yy >= bx.y0 && yy < bx.y1) mk[m >> 2] |= 1ull << ((m & 3) * 16 + gr.run);
    }
  }
  auto gen = [&](auto&& cb) {
    for (int w = 0; w < ((nm + 3) >> 2); ++w) {
      unsigned long long q = mk[w];
      while (q) {
        const int bb = __ffsll((long long)q) - 1;
        q &= q - 1;
        const SmBox32& bx = mb[w * 4 + (bb >> 4)];
        cb(bx.x0 + F.run_lo[bb & 15], bx.x1 + F.run_hi[bb & 15]);
      }
    }
  };
  const int INF = 0x7fffffff;
  int mn_s = INF, mx_s = -INF, mn_e = INF, mx_e = -INF;
  gen([&](int xs, int xe) {
    mn_s = xs < mn_s ? xs : mn_s;
    mx_s = xs > mx_s ? xs : mx_s;
    mn_e = xe < mn_e ? xe : mn_e;
    mx_e = xe > mx_e ? xe : mx_e;
  });
  T32x2 o{t32_empty(), t32_empty()};
  if (mn_s == INF) return o;
  if (mx_s <= mn_e) {
    const int a0 = R0 + (mn_s << le), a1 = R0 + ((mx_e - 1) << le);
    o.s = run_triple32([&](int r) {
      const int s0 = (a0 + r * step) >> ls, s1 = (a1 + r * step) >> ls;
      return T32{s0, s1, s1 - s0 + 1};
    }, step, run, ls);
    o.l = run_triple32([&](int r) {
      const int s0 = (a0 + r * step) >> ll, s1 = (a1 + r * step) >> ll;
      return T32{s0, s1, s1 - s0 + 1};
    }, step, run, ll);
  } else {
    o.s = run_triple32([&](int r) {
      T32 x = t32_empty();
      row_union32(gen, R0 + r * step, le, ls, x);
      return x;
    }, step, run, ls);
    o.l = run_triple32([&](int r) {
      T32 x = t32_empty();
      row_union32(gen, R0 + r * step, le, ll, x);
      return x;
    }, step, run, ll);
  }
  return o;
}
// Unique load sectors / lines of the blocks {S0 + m*nsm : m < kj} (one SM set, round-robin
// dispatch, Q9) by one CTA.  Row (y,z) of field phi holds element x iff some member box
// contains (x - ox, y - oy, z - oz) for a load offset o.  Per z-plane: if every
// (group, member) z-membership equals that of plane z - per, the plane is the translate of
// that plane by whole lines (derived); otherwise a warp computes it, lanes taking rows
// (per row: compares against the member boxes into a candidate mask, union, triple), with an
// ordered warp reduction.  Thread 0 folds the plane triples in z order.
struct SmWarp {
  unsigned bm[kSegRowsS / 32];
  short rs[kSegRowsS + 2];
  // the computed plane's active (load group, members) pairs: group gl[i] reaches the plane
  // z - oz inside exactly the members of gm[i] (ngl entries)
  unsigned gm[kMaxAcc];
  unsigned char gl[kMaxAcc];
};

// msk: 0 = every member S0 + m * nsm (m < kj); else only the members m whose bit is set (one
// connected component of the set, k_smset)
__device__ void smset_cta(const DPlan& P, const DKernel& K, const DGpu& G, long long S0, long long kj, long long nsm,
                          SmBox* mb, SmBox32* mb32, Tri* pt /* 2*kMaxPlanes */, unsigned char* pder /* kMaxPlanes */,
                          SmWarp* sw,
                          unsigned long long& sum_s, unsigned long long& sum_l, unsigned long long& units,
                          unsigned msk = 0u, int field_only = -1) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwp = blockDim.x >> 5;
  const int ls = G.lg_sector, ll = G.lg_line;
  const int nm = msk ? __popc(msk) : (int)(kj < kMaxMembers ? kj : kMaxMembers);
  sum_s = sum_l = 0;
  units = 0;
  __syncthreads();
  if (tid < nm) {
    const long long mi = msk ? (long long)__fns(msk, 0, tid + 1) : (long long)tid;  // tid-th member
    const long long Bm = S0 + mi * nsm;
    const long long bc[3] = {Bm % P.G[0], (Bm / P.G[0]) % P.G[1], Bm / (P.G[0] * P.G[1])};
    long long lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = P.lo[d] + bc[d] * P.BF[d];
      hi[d] = lo[d] + P.BF[d];
      if (hi[d] > P.hi[d]) hi[d] = P.hi[d];
    }
    mb[tid] = SmBox{lo[0], hi[0], lo[1], hi[1], lo[2], hi[2]};
    mb32[tid] = SmBox32{(int)lo[0], (int)hi[0], (int)lo[1], (int)hi[1], (int)lo[2], (int)hi[2]};
  }
  __syncthreads();
  long long ylo = LLONG_MAX, yhi = LLONG_MIN, zlo = LLONG_MAX, zhi = LLONG_MIN;
  for (int m = 0; m < nm; ++m) {
    ylo = min(ylo, mb[m].y0);
    yhi = max(yhi, mb[m].y1);
    zlo = min(zlo, mb[m].z0);
    zhi = max(zhi, mb[m].z1);
  }
  for (int fi = field_only < 0 ? 0 : field_only; fi < (field_only < 0 ? K.n_fields : field_only + 1); ++fi) {
    const DField& F = K.f[fi];
    if (!(F.kinds & 1)) continue;
    const int g0 = F.g_begin, ng = F.g_end - F.g_begin;
    const int le = F.lg_elem;
    long long y0 = ylo + F.ld_oy_min, y1 = yhi + F.ld_oy_max, z0 = zlo + F.ld_oz_min, z1 = zhi + F.ld_oz_max;
    if (y0 < 0) y0 = 0;
    if (z0 < 0) z0 = 0;
    if (y1 > F.ext[1]) y1 = F.ext[1];
    if (z1 > F.ext[2]) z1 = F.ext[2];
    if (y1 <= y0 || z1 <= z0) continue;
    const long long ny = y1 - y0;
    const long long align = F.align, py = F.pitch[1], pz = F.pitch[2];
    const long long pbytes = pz << le, pystep = py << le;
    const int per = plane_period(pz, le, ll);
    const int npairs = ng * nm;
    Tri cs_all = tri_empty(), cl_all = tri_empty();
    for (long long zs = z0; zs < z1; zs += kMaxPlanes) {
      const int np = (int)(z1 - zs < kMaxPlanes ? z1 - zs : kMaxPlanes);
      // (a) derived planes (relative to plane z - per of the whole box)
      for (int p = wid; p < np; p += nwp) {
        const long long z = zs + p;
        bool same = per > 0 && z - per >= zs;  // derive only within this segment
        if (same) {
          for (int k = lane; k < npairs; k += 32) {
            const DGroup gr = K.g[g0 + k / nm];
            if (gr.kind != 0) continue;
            const SmBox& bx = mb[k % nm];
            const long long za = z - gr.oz, zb = za - per;
            same = same && ((za >= bx.z0 && za < bx.z1) == (zb >= bx.z0 && zb < bx.z1));
          }
        }
        same = __all_sync(FULL, same);
        if (lane == 0) pder[p] = same ? 1 : 0;
      }
      __syncthreads();
      // (b) computed planes, dealt round-robin to the warps in order of their rank among the
      //     computed planes (balanced): one warp per plane.  A row's candidates change only
      //     where some y - oy crosses a member's y edge: lanes mark these breakpoints, then take
      //     one run each (smset_run), in 32-bit plane-relative arithmetic (see k_rows).
      int rank0 = 0;  // computed planes before the current 32-plane window
      for (int pb = 0; pb < np; pb += 32) {
        const int pw = pb + lane;
        const unsigned cm = __ballot_sync(FULL, pw < np && !pder[pw]);
        unsigned mine = 0;  // planes of this window whose rank % nwp == wid
        {
          unsigned q = cm;
          int rm = rank0 % nwp;  // rank mod nwp, advanced incrementally
          while (q) {
            const int b = __ffs(q) - 1;
            q &= q - 1;
            if (rm == wid) mine |= 1u << b;
            rm = rm + 1 == nwp ? 0 : rm + 1;
          }
        }
        rank0 += __popc(cm);
        while (mine) {
          const int p = pb + __ffs(mine) - 1;
          mine &= mine - 1;
          const int z = (int)(zs + p);
          SmWarp& Wp = sw[wid];
          const long long R0p = align + ((py * y0 + pz * (long long)z) << le);
          const long long Bp = (R0p >> ll) << ll;
          const int off0 = (int)(R0p - Bp), step = (int)pystep;
          T32 ps = t32_empty(), pl = t32_empty();
          // the plane's active (load group, members) pairs: one ballot over the members per group
          int ngl = 0;
          for (int g = 0; g < ng; ++g) {
            const DGroup gr = K.g[g0 + g];
            if (gr.kind != 0) continue;
            const int zz = z - gr.oz;
            const unsigned mm = __ballot_sync(FULL, lane < nm && zz >= mb32[lane].z0 && zz < mb32[lane].z1);
            if (mm) {
              if (lane == 0) {
                Wp.gm[ngl] = mm;
                Wp.gl[ngl] = (unsigned char)g;
              }
              ++ngl;
            }
          }
          __syncwarp();
          for (int ys = 0; ys < (int)ny; ys += kSegRowsS) {
            const int nseg = (int)ny - ys < kSegRowsS ? (int)ny - ys : kSegRowsS;
            const int nwd = (nseg + 31) >> 5;
            for (int w = lane; w < nwd; w += 32) Wp.bm[w] = 0u;
            __syncwarp();
            if (lane == 0) atomicOr(&Wp.bm[0], 1u);
            for (int i = 0; i < ngl; ++i) {   // lane m: member m's y edges shifted by the group's oy
              if (!((Wp.gm[i] >> lane) & 1u)) continue;
              const DGroup gr = K.g[g0 + Wp.gl[i]];
              const SmBox32& bx = mb32[lane];
              const int e0 = bx.y0 + gr.oy - (int)y0 - ys, e1 = bx.y1 + gr.oy - (int)y0 - ys;
              if (e0 > 0 && e0 < nseg) atomicOr(&Wp.bm[e0 >> 5], 1u << (e0 & 31));
              if (e1 > 0 && e1 < nseg) atomicOr(&Wp.bm[e1 >> 5], 1u << (e1 & 31));
            }
            __syncwarp();
            const int wpl = (nwd + 31) >> 5;
            int cnt = 0;
            for (int w = lane * wpl; w < nwd && w < (lane + 1) * wpl; ++w) cnt += __popc(Wp.bm[w]);
            int pos = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int v = __shfl_up_sync(FULL, pos, o);
              if (lane >= o) pos += v;
            }
            const int nruns = __shfl_sync(FULL, pos, 31);
            pos -= cnt;
            for (int w = lane * wpl; w < nwd && w < (lane + 1) * wpl; ++w) {
              unsigned bits = Wp.bm[w];
              while (bits) {
                const int bt = __ffs(bits) - 1;
                bits &= bits - 1;
                Wp.rs[pos++] = (short)(w * 32 + bt);
              }
            }
            if (lane == 0) Wp.rs[nruns] = (short)nseg;
            __syncwarp();
            for (int rb = 0; rb < nruns; rb += 32) {
              T32 tt[2] = {t32_empty(), t32_empty()};
              const int j = rb + lane;
              if (j < nruns) {
                const int yr = ys + Wp.rs[j];  // row index inside the box
                const T32x2 o = smset_run_g(mb32, nm, Wp.gm, Wp.gl, ngl, K, F, g0, (int)y0 + yr, off0 + yr * step,
                                            step, Wp.rs[j + 1] - Wp.rs[j], le, ls, ll);
                tt[0] = o.s;
                tt[1] = o.l;
              }
              warp_ordered_reduce32<2>(tt, nruns - rb);
              if (lane == 0) {  // ps, pl: lane 0 only
                ps = t32_combine(ps, tt[0]);
                pl = t32_combine(pl, tt[1]);
              }
            }
            __syncwarp();
          }
          if (lane == 0) {
            const long long bs = Bp >> ls, bl = Bp >> ll;
            pt[2 * p] = ps.c ? Tri{ps.f + bs, ps.l + bs, ps.c} : tri_empty();
            pt[2 * p + 1] = pl.c ? Tri{pl.f + bl, pl.l + bl, pl.c} : tri_empty();
            units += (unsigned long long)ny;
          }
        }
      }
      __syncthreads();
      // (c) ordered fold by the whole CTA: a derived plane is its computed source plane (p - m*per,
      //     the nearest non-derived one) translated by m*per planes; threads take contiguous planes,
      //     then an ordered CTA reduction
      // (few planes -- single blocks: warp 0 alone, no CTA barriers)
      const bool one_warp = np <= 64;
      if (!one_warp || wid == 0) {
        const int nthr = one_warp ? 32 : (int)blockDim.x;
        const int ppl = (np + nthr - 1) / nthr;
        Tri t2[2] = {tri_empty(), tri_empty()};
        for (int p = tid * ppl; p < np && p < (tid + 1) * ppl; ++p) {
          int q = p;
          while (pder[q]) q -= per;
          const long long dsh = (long long)(p - q) * pbytes;
          const Tri a = pt[2 * q], b = pt[2 * q + 1];
          t2[0] = tri_combine(t2[0], a.c ? Tri{a.f + (dsh >> ls), a.l + (dsh >> ls), a.c} : tri_empty());
          t2[1] = tri_combine(t2[1], b.c ? Tri{b.f + (dsh >> ll), b.l + (dsh >> ll), b.c} : tri_empty());
        }
        if (one_warp) {
          warp_ordered_reduce<2>(t2);
        } else {
          __shared__ Tri s_fold[(WS_SCLASS_THREADS / 32) * 2];
          cta_ordered_reduce<2>(t2, s_fold);
        }
        if (tid == 0) {
          cs_all = tri_combine(cs_all, t2[0]);
          cl_all = tri_combine(cl_all, t2[1]);
        }
      }
      __syncthreads();
    }
    if (tid == 0) {
      sum_s += (unsigned long long)cs_all.c;
      sum_l += (unsigned long long)cl_all.c;
    }
  }
}

// ---- single-block SM-set classes shared across configurations: the count of a class depends on
// the kernel, the GPU's sector / line geometry, the block footprint BF (which fixes the clipped
// extents) and the class slot (line residue, clip pattern) only, so configurations with the same
// (kernel, GPU, BF) -- e.g. (32,2,1)+2y and (32,4,1) -- share it.  Key: kid 8 | gid 8 | BF 3 x 13
// | slot 9 bits; 0 = not shareable.
__device__ __forceinline__ unsigned long long share_key(const DPlan& P, unsigned slot) {
  if (P.kid > 255 || P.gid > 255 || P.BF[0] >= 8192 || P.BF[1] >= 8192 || P.BF[2] >= 8192) return 0ull;
  const unsigned long long k = ((unsigned long long)P.kid << 56) | ((unsigned long long)P.gid << 48) |
                               ((unsigned long long)P.BF[0] << 35) | ((unsigned long long)P.BF[1] << 22) |
                               ((unsigned long long)P.BF[2] << 9) | (unsigned long long)slot;
  return k == ~0ull ? 0ull : k;
}
// owner (bit 30) or sharer (bit 31) of table entry t (bits 9..21) for a class slot; plain otherwise
__device__ __forceinline__ unsigned share_claim(unsigned long long* skey, unsigned long long key, unsigned slot) {
  if (!key) return slot;
  unsigned t = (unsigned)((key * 0x9e3779b97f4a7c15ull) >> 51) & (kShareTab - 1);
  for (int probe = 0; probe < 64; ++probe, t = (t + 1) & (kShareTab - 1)) {
    const unsigned long long old = atomicCAS(skey + t, ~0ull, key);
    if (old == ~0ull) return slot | (t << 9) | (1u << 30);
    if (old == key) return slot | (t << 9) | (1u << 31);
  }
  return slot;  // table crowded: evaluate without sharing
}

// ---- translation groups of directly evaluated multi-block SM sets (k_smset)
constexpr int kSetGrp = 1024;  // sets per config grouped in shared memory (more: no grouping)
__device__ __forceinline__ void block_coord(const DPlan& P, long long B, long long* bc) {
  bc[0] = B % P.G[0];
  bc[1] = (B / P.G[0]) % P.G[1];
  bc[2] = B / (P.G[0] * P.G[1]);
}
// load-offset envelope of a kernel's load fields (k_smset's quick separation test)
struct SetEnv {
  long long spy, spz, oy_min, oy_max, ext1_min;
  bool rows_ok, planes_ok;
};
__device__ __forceinline__ SetEnv set_env(const DKernel& K, long long lb) {
  const DLoadEnv& E = K.env;  // precomputed by ws_describe_kernel
  SetEnv e{E.spy, E.spz, E.oy_min, E.oy_max, E.ext1_min, E.has_load && E.row_bytes_min >= lb,
           E.has_load && E.plane_bytes_min >= lb};
  return e;
}
// block-coordinate walk over a set's members (B -> B + nsm): adds and carries only
struct MemberWalk {
  long long ax, ay, az;  // nsm as (x, y, z) digits of the grid (az: whole grid planes)
  __device__ __forceinline__ MemberWalk(const DPlan& P, long long nsm) {
    ax = nsm % P.G[0];
    ay = (nsm / P.G[0]) % P.G[1];
    az = nsm / (P.G[0] * P.G[1]);
  }
  __device__ __forceinline__ void step(const DPlan& P, long long* bc) const {
    bc[0] += ax;
    long long cy = 0;
    if (bc[0] >= P.G[0]) {
      bc[0] -= P.G[0];
      cy = 1;
    }
    bc[1] += ay + cy;
    long long cz = 0;
    if (bc[1] >= P.G[1]) {
      bc[1] -= P.G[1];
      cz = 1;
    }
    bc[2] += az + cz;
  }
};
__device__ __forceinline__ bool set_unclipped(const DPlan& P, long long S0, long long kj, long long nsm) {
  const MemberWalk mw(P, nsm);
  long long bc[3];
  block_coord(P, S0, bc);
  for (long long m = 0; m < kj; ++m) {
    if (m) mw.step(P, bc);
    if (clip_pattern(P, bc)) return false;
  }
  return true;
}
// line residue of the set's first block (translation by a multiple of a line keeps every count)
__device__ __forceinline__ long long set_residue(const DPlan& P, long long S0) {
  long long bc[3], pl = 0;
  block_coord(P, S0, bc);
#pragma unroll
  for (int d = 0; d < 3; ++d) pl += P.cls_pitch[d] * (P.lo[d] + bc[d] * P.BF[d]);
  return pl & (P.scls_R - 1);
}
// hash of (member count, residue, members' block offsets from the first member); never 0
__device__ __forceinline__ unsigned long long set_shape_key(const DPlan& P, long long S0, long long kj, long long nsm) {
  const MemberWalk mw(P, nsm);
  long long b0[3], bc[3];
  block_coord(P, S0, b0);
  bc[0] = b0[0], bc[1] = b0[1], bc[2] = b0[2];
  unsigned long long h = 0x9e3779b97f4a7c15ull ^ ((unsigned long long)kj << 8) ^ (unsigned long long)set_residue(P, S0);
  for (long long m = 1; m < kj; ++m) {
    mw.step(P, bc);
    for (int d = 0; d < 3; ++d) {
      h ^= (unsigned long long)(bc[d] - b0[d]) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 0xff51afd7ed558ccdull;
    }
  }
  return h | 1ull;
}
// exact check: every member of set S1 is the same block translate of S0's member (same count)
__device__ __forceinline__ bool set_translates(const DPlan& P, long long S0, long long S1, long long kj, long long nsm) {
  if (set_residue(P, S0) != set_residue(P, S1)) return false;
  const MemberWalk mw(P, nsm);
  long long a0[3], b0[3], a[3], b[3];
  block_coord(P, S0, a0);
  block_coord(P, S1, b0);
  for (int d = 0; d < 3; ++d) a[d] = a0[d], b[d] = b0[d];
  for (long long m = 1; m < kj; ++m) {
    mw.step(P, a);
    mw.step(P, b);
    for (int d = 0; d < 3; ++d)
      if (a[d] - a0[d] != b[d] - b0[d]) return false;
  }
  return true;
}


// Two members' load footprints (block box + the field's load-offset extremes) share no line when
// they are >= 2 planes apart in z, or >= 2 rows apart in y without touching the field's first or
// last row (rows / planes of >= one line), or >= one line of elements apart in x unless one reaches
// a row end and the other a row start (wrap-around adjacency of consecutive rows).  The load-offset
// envelope of all fields (one pitch for all fields under scls_R) decides most pairs at once.
// Boxes: {x0, x1, y0, y1, z0, z1}, inclusive ends.
__device__ bool set_pair_separated(const DKernel& K, const SetEnv& env, long long lb, const long long* A,
                                   const long long* B) {
  if (env.planes_ok && (B[4] - A[5] >= 2 + env.spz || A[4] - B[5] >= 2 + env.spz)) return true;
  if (env.rows_ok && min(A[2], B[2]) + env.oy_min >= 1 && max(A[3], B[3]) + env.oy_max <= env.ext1_min - 2 &&
      (B[2] - A[3] >= 2 + env.spy || A[2] - B[3] >= 2 + env.spy))
    return true;
  for (int fi = 0; fi < K.n_fields; ++fi) {
    const DField& F = K.f[fi];
    if (!(F.kinds & 1)) continue;
    int xlo = 0x7fffffff, xhi = -0x7fffffff;
    for (int r = 0; r < F.n_runs; ++r) {
      xlo = min(xlo, F.run_lo[r]);
      xhi = max(xhi, F.run_hi[r]);
    }
    const long long D = (lb >> F.lg_elem) + 1;  // elements per line, plus one
    const bool rows_ok = (F.pitch[1] << F.lg_elem) >= lb, planes_ok = (F.pitch[2] << F.lg_elem) >= lb;
    const long long ax0 = A[0] + xlo, ax1 = A[1] + xhi, bx0 = B[0] + xlo, bx1 = B[1] + xhi;
    const long long ay0 = A[2] + F.ld_oy_min, ay1 = A[3] + F.ld_oy_max;
    const long long by0 = B[2] + F.ld_oy_min, by1 = B[3] + F.ld_oy_max;
    const long long az0 = A[4] + F.ld_oz_min, az1 = A[5] + F.ld_oz_max;
    const long long bz0 = B[4] + F.ld_oz_min, bz1 = B[5] + F.ld_oz_max;
    // rows >= 2 apart share no line within a plane; across consecutive planes only if a box
    // reaches the field's first / last row (p2 >= p1 * ext1), hence the y-ends condition
    const bool y_inner = min(ay0, by0) >= 1 && max(ay1, by1) <= F.ext[1] - 2;
    const bool sep_y = rows_ok && y_inner && (ay1 + 2 <= by0 || by1 + 2 <= ay0);
    const bool sep_z = planes_ok && (az1 + 2 <= bz0 || bz1 + 2 <= az0);
    // consecutive rows in memory can share a line only between a box reaching the row end and one
    // reaching the row start
    const bool a_end = ax1 > F.pitch[1] - 1 - D, a_start = ax0 < D;
    const bool b_end = bx1 > F.pitch[1] - 1 - D, b_start = bx0 < D;
    const bool wrap = (a_end && b_start) || (b_end && a_start);
    const bool sep_x = rows_ok && !wrap && (ax1 + D <= bx0 || bx1 + D <= ax0);
    if (!(sep_y || sep_z || sep_x)) return false;
  }
  return true;
}

// block Bm of configuration c joins its single-block translation class (slot: line residue of its
// first cell, clip pattern); the first member of a class claims it (and the cross-configuration
// key).  Called by the whole warp (active lanes join): lanes of one slot are counted with one
// atomic by their leader (__match_any_sync), not one per block.
__device__ void smset_claim(const DPlan& P, int c, long long Bm, bool active, unsigned int* __restrict__ scnt,
                            unsigned long long* __restrict__ srep, unsigned long long* __restrict__ skey,
                            unsigned long long* __restrict__ slist, unsigned long long* __restrict__ lists) {
  const int lane = threadIdx.x & 31;
  unsigned slot = 0u;
  if (active) {
    const long long bc[3] = {Bm % P.G[0], (Bm / P.G[0]) % P.G[1], Bm / (P.G[0] * P.G[1])};
    long long pl = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) pl += P.cls_pitch[d] * (P.lo[d] + bc[d] * P.BF[d]);
    slot = (unsigned)(((pl & (P.scls_R - 1)) << 3) | clip_pattern(P, bc));
  }
  const unsigned peers = __match_any_sync(FULL, active ? slot : 0x80000000u + (unsigned)lane);
  if (!active || lane != __ffs(peers) - 1) return;
  const long long gslot = (long long)c * kSSlots + slot;
  if (atomicAdd(scnt + gslot, (unsigned)__popc(peers)) == 0u) {
    srep[gslot] = (unsigned long long)Bm;
    const unsigned low = share_claim(skey, share_key(P, slot), slot);
    {
      const unsigned long long si = atomicAdd(lists + 1, 1ull);
      WS_CHK(si, g_caps.sslots);
      slist[si] = ((unsigned long long)c << 32) | low;
    }
  }
}

// Pass 1 (one thread per SM set): single-block sets go to their translation class: clip
// pattern of the block x residue of its first cell's address mod line_bytes (identical
// active-cell boxes that are translates by a multiple of the line size have identical
// sector and line counts).  Multi-block sets are appended to the direct list.
constexpr int kSmsetThreads = 256;
__global__ void __launch_bounds__(kSmsetThreads) k_smset(const DPlan* __restrict__ plans, const DPrefix* __restrict__ pre, int n,
                                               const DKernel* __restrict__ ks,
                                               const DGpu* __restrict__ gs, unsigned int* __restrict__ scnt,
                                               unsigned long long* __restrict__ srep,
                                               unsigned long long* __restrict__ lists,
                                               unsigned long long* __restrict__ slist,
                                               unsigned long long* __restrict__ dlist,
                                               unsigned long long* __restrict__ skey,
                                               unsigned int* __restrict__ dmask,
                                               const unsigned long long* __restrict__ gkey) {
  PDL_PROLOGUE();
  __shared__ unsigned long long s_key[kSetGrp];  // directly evaluated sets: shape key (0: not grouped)
  __shared__ unsigned s_cnt[kSetGrp];            // group sizes (at the group's smallest member)
  __shared__ short s_rep[kSetGrp];               // smallest member of the set's group
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const DPlan& P = plans[c];
    const long long nset = pre[c + 1].set - pre[c].set;
    if (nset <= 0) continue;  // failed configuration (its kid / gid may be out of range): no sets
    const long long nsm = gs[P.gid].g.n_sm;
    const bool grp = nset <= kSetGrp && P.scls_R > 0 && !P.rep_mult;
    const SetEnv env = set_env(ks[P.kid], gs[P.gid].g.line_bytes);
    // A multi-block set whose members' load footprints cannot share a line is the disjoint union
    // of its members' footprints: every member is then counted like a single-block set, in its
    // translation class (members are n_sm blocks apart, usually far apart in the grid).  Members
    // that cannot share a line with any member of another group form connected components (union
    // of the non-separated pairs, set_pair_separated): the set's footprint is the disjoint union of
    // its components' footprints.  All singletons: the set splits into single-block classes; one
    // component: the set is evaluated directly (translation groups below); otherwise singletons
    // join the classes and each larger component is a direct item of its own (member mask).
    const bool pairs_on = P.scls_R > 0 && !P.rep_mult;
    // (1) one thread per set (sets of 2..32 members were analysed by k_spairs)
    for (long long j0 = threadIdx.x - (threadIdx.x & 31); j0 < nset; j0 += blockDim.x) {  // warp-uniform
      const long long j = j0 + (threadIdx.x & 31);
      const long long S0 = P.s + j;
      const long long kj = j < nset ? (P.W - j + nsm - 1) / nsm : 0;  // members S0 + m*nsm, m < kj
      smset_claim(P, c, S0, pairs_on && kj == 1, scnt, srep, skey, slist, lists);  // whole warp
      if (j >= nset) continue;
      if (pairs_on && kj > 1 && kj <= 32) {  // analysed by k_spairs: its translation-group key
        if (grp) s_key[j] = gkey[pre[c].set + j];
        continue;
      }
      if (pairs_on && kj == 1) {
        if (grp) s_key[j] = 0ull;
      } else if (grp && kj <= 32 && set_unclipped(P, S0, kj, nsm)) {
        s_key[j] = set_shape_key(P, S0, kj, nsm);
      } else {
        if (grp) s_key[j] = 0ull;
        const unsigned long long pos = atomicAdd(lists + 2, 1ull);
        dlist[pos] = ((unsigned long long)c << 32) | (unsigned long long)j;
        dmask[pos] = 0u;
      }
    }
    __syncthreads();
    if (grp) {
      // Multi-block sets evaluated directly, grouped by translation: two sets whose members are
      // the same translate of each other (same count, unclipped, same line residue) have equal
      // counts.  The smallest j of each group is evaluated, counted group-size times.
      __syncthreads();
      for (long long j = threadIdx.x; j < nset; j += blockDim.x) s_cnt[j] = 0u;
      __syncthreads();
      // every grouped set finds its group's smallest member (usually one verification) and
      // counts itself there
      for (long long j = threadIdx.x; j < nset; j += blockDim.x) {
        const unsigned long long kj_key = s_key[j];
        if (!kj_key) continue;
        const long long kj = (P.W - j + nsm - 1) / nsm;
        long long r = j;
        for (long long i = 0; i < j; ++i)
          if (s_key[i] == kj_key && (P.W - i + nsm - 1) / nsm == kj && set_translates(P, P.s + i, P.s + j, kj, nsm)) {
            r = i;
            break;
          }
        s_rep[j] = (short)r;
        atomicAdd(&s_cnt[r], 1u);
      }
      __syncthreads();
      for (long long j = threadIdx.x; j < nset; j += blockDim.x) {
        if (!s_key[j] || s_rep[j] != j) continue;
        const unsigned mult = s_cnt[j];
        const unsigned long long pos = atomicAdd(lists + 2, 1ull);
        dlist[pos] = ((unsigned long long)c << 32) | 0x80000000ull | ((unsigned long long)(mult - 1) << 20) |
                     (unsigned long long)j;
        dmask[pos] = 0u;
      }
      __syncthreads();
    }
  }
}

// SM sets of 2..32 members (k_smset's pair analysis), one warp per set over every configuration's
// sets (items: the pre.set prefix): lanes test the member pairs (set_pair_separated), lane 0 unites
// the connected components; all singletons -> the members' single-block classes, one component ->
// the set as a whole (its translation-group key for k_smset in gkey, or a direct item), several ->
// singletons to their classes, larger components to direct items with a member mask.
__global__ void __launch_bounds__(kSmsetThreads) k_spairs(const DPlan* __restrict__ plans,
                                                const DPrefix* __restrict__ pre, int n,
                                                const DKernel* __restrict__ ks, const DGpu* __restrict__ gs,
                                                unsigned int* __restrict__ scnt, unsigned long long* __restrict__ srep,
                                                unsigned long long* __restrict__ lists,
                                                unsigned long long* __restrict__ slist,
                                                unsigned long long* __restrict__ dlist,
                                                unsigned long long* __restrict__ skey, unsigned int* __restrict__ dmask,
                                                unsigned long long* __restrict__ gkey) {
  PDL_PROLOGUE();
  __shared__ long long s_mbox[kSmsetThreads / 32][32 * 6];  // member boxes of a warp's set
  __shared__ unsigned s_adj[kSmsetThreads / 32][32];        // non-separated pairs, row a1 bit b1
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long total = pre[n].sclass;   // sets of >= 2 members only (k_plan's n_sclass_items)
  const long long nwg = (long long)gridDim.x * (blockDim.x >> 5);
  int c = -1;
  for (long long item0 = (long long)blockIdx.x * (blockDim.x >> 5) + wid; item0 < total; item0 += nwg) {
    c = find_config_warp<3>(pre, n, item0, c);
    const DPlan& P = plans[c];
    const long long j = item0 - pre[c].sclass;
    const long long item = pre[c].set + j;  // the set's index in pre.set order (gkey)
    const long long nsm = gs[P.gid].g.n_sm;
    const long long kj = (P.W - j + nsm - 1) / nsm;
    if (!(P.scls_R > 0 && !P.rep_mult) || kj <= 1 || kj > 32) continue;
    const long long nset = pre[c + 1].set - pre[c].set;
    const bool grp = nset <= kSetGrp;
    const SetEnv env = set_env(ks[P.kid], gs[P.gid].g.line_bytes);
    const DKernel& K = ks[P.kid];
    const long long lb = gs[P.gid].g.line_bytes;
    const long long S0 = P.s + j;
    unsigned long long gk = 0ull;
    {
      {
        long long* bx = s_mbox[wid];
        if (lane < kj) {
          long long bc[3];
          block_coord(P, S0 + (long long)lane * nsm, bc);
          for (int d = 0; d < 3; ++d) {
            bx[lane * 6 + 2 * d] = P.lo[d] + bc[d] * P.BF[d];
            const long long hi = bx[lane * 6 + 2 * d] + P.BF[d];
            bx[lane * 6 + 2 * d + 1] = (hi > P.hi[d] ? P.hi[d] : hi) - 1;
          }
        }
        s_adj[wid][lane] = 0u;
        __syncwarp();
        const int k = (int)kj;
        // circulant pair assignment: lane a tests (a, a + d mod k) for d = 1 .. k/2, every unordered
        // pair once (d = k/2 with k even: lanes < d only); the adjacency is kept symmetric
        if (lane < k) {
          unsigned row = 0u;
          for (int d = 1; 2 * d <= k; ++d) {
            if (2 * d == k && lane >= d) break;
            const int b1 = lane + d < k ? lane + d : lane + d - k;
            if (!set_pair_separated(K, env, lb, bx + lane * 6, bx + b1 * 6)) {
              row |= 1u << b1;
              atomicOr(&s_adj[wid][b1], 1u << lane);
            }
          }
          atomicOr(&s_adj[wid][lane], row);
        }
        __syncwarp();
        // connected components: transitive closure of adjacency | self by repeated squaring (paths
        // of length <= 2^t after t rounds; stops when nothing changes)
        unsigned comp = lane < k ? (s_adj[wid][lane] | (1u << lane)) : 0u;
        for (int it = 0; it < 5; ++it) {
          unsigned nc = comp;
          for (int jj = 0; jj < k; ++jj) {
            const unsigned cj = __shfl_sync(FULL, comp, jj);
            if ((comp >> jj) & 1u) nc |= cj;
          }
          const bool changed = nc != comp;
          comp = nc;
          if (!__any_sync(FULL, changed)) break;
        }
        const bool leader = lane < k && __ffs(comp) - 1 == lane;
        const int ncomp = __popc(__ballot_sync(FULL, leader));
        // singletons join the single-block classes; one component: the set as a whole (translation
        // groups, k_smset); several: every larger component a direct item with its member mask
        const unsigned single = ncomp > 1 ? __ballot_sync(FULL, lane < k && comp == (1u << lane)) : 0u;
        if (ncomp == 1) {
          if (lane == 0) {
            if (grp && set_unclipped(P, S0, kj, nsm)) {
              gk = set_shape_key(P, S0, kj, nsm);
            } else {
              const unsigned long long pos = atomicAdd(lists + 2, 1ull);
              dlist[pos] = ((unsigned long long)c << 32) | (unsigned long long)j;
              dmask[pos] = 0u;
            }
          }
        } else if (leader && __popc(comp) > 1) {
          const unsigned long long pos = atomicAdd(lists + 2, 1ull);
          dlist[pos] = ((unsigned long long)c << 32) | (unsigned long long)j;
          dmask[pos] = comp;
        }
        smset_claim(P, c, S0 + (long long)lane * nsm, (single >> lane) & 1u, scnt, srep, skey, slist, lists);
        __syncwarp();
      }
    }
    if (lane == 0) gkey[item] = gk;
  }
}

// ---- single-block SM-set classes by computed planes (the class representatives' footprints,
// a4): one warp per (class, load field, computed plane) instead of one CTA per class.
//   k_cplan : one warp per class entry: per load field the footprint box (block box + the
//             field's load-offset extremes), plane derivation (a plane whose every (group,
//             block) membership equals the plane `per` below it is its translate by whole
//             lines), a descriptor, a slice of the plane pool (derived planes marked), and one
//             item per computed plane.  Entries the pool cannot hold, and blocks of kernels with
//             many load fields (LBM: flat rows, smset_eval), stay on the CTA path (k_sclass).
//   k_cplanes: one warp per item: the plane's runs (smset_run with the one block), its sector and
//             line triples into the pool.
//   k_cfold : one warp per descriptor: ordered fold over the box's planes (derived planes
//             translated from their source), counts x class size into the configuration's
//             accumulators; owners of shared classes accumulate the published counts.

__device__ __forceinline__ bool cplane_derived(const DKernel& K, const DField& F, const SmBox32& b, int z, int z0,
                                               int per) {
  if (per <= 0 || z - per < z0) return false;
  for (int g = F.g_begin; g < F.g_end; ++g) {
    const DGroup gr = K.g[g];
    if (gr.kind != 0) continue;
    const int za = z - gr.oz, zb = za - per;
    if ((za >= b.z0 && za < b.z1) != (zb >= b.z0 && zb < b.z1)) return false;
  }
  return true;
}

__device__ __forceinline__ SmBox32 block_box32(const DPlan& P, long long B) {
  const long long bc[3] = {B % P.G[0], (B / P.G[0]) % P.G[1], B / (P.G[0] * P.G[1])};
  long long lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = P.lo[d] + bc[d] * P.BF[d];
    hi[d] = lo[d] + P.BF[d];
    if (hi[d] > P.hi[d]) hi[d] = P.hi[d];
  }
  return SmBox32{(int)lo[0], (int)hi[0], (int)lo[1], (int)hi[1], (int)lo[2], (int)hi[2]};
}

// field fi's footprint box of block box b (rows y0..y1, planes z0..z1, clipped to the field)
__device__ __forceinline__ bool cfield_box(const DField& F, const SmBox32& b, int& y0, int& y1, int& z0, int& z1) {
  y0 = b.y0 + F.ld_oy_min;
  y1 = b.y1 + F.ld_oy_max;
  z0 = b.z0 + F.ld_oz_min;
  z1 = b.z1 + F.ld_oz_max;
  y0 = y0 < 0 ? 0 : y0;
  z0 = z0 < 0 ? 0 : z0;
  y1 = y1 > (int)F.ext[1] ? (int)F.ext[1] : y1;
  z1 = z1 > (int)F.ext[2] ? (int)F.ext[2] : z1;
  return y1 > y0 && z1 > z0 && (F.kinds & 1);
}

// cctr: [0] descriptors << 40 | pool planes (one atomic per class entry), [1] items, [2] CTA-path entries
__global__ void __launch_bounds__(256) k_cplan(const DPlan* __restrict__ plans, const DKernel* __restrict__ ks,
                                               const DGpu* __restrict__ gs, const unsigned long long* __restrict__ lists,
                                               const unsigned long long* __restrict__ slist,
                                               const unsigned long long* __restrict__ srep,
                                               unsigned long long* __restrict__ sval, uint32_t* __restrict__ cfbl,
                                               CDesc* __restrict__ cdesc, Tri* __restrict__ cpool,
                                               uint32_t* __restrict__ citems, unsigned long long* __restrict__ cctr,
                                               long long desc_cap, long long pool_cap) {
  PDL_PROLOGUE();
  const int lane = threadIdx.x & 31;
  const long long ncls = (long long)lists[1];
  const long long nwg = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < ncls; e += nwg) {
    const unsigned long long ent = slist[e];
    const int c = (int)(ent >> 32);
    const unsigned low = (unsigned)(ent & 0xffffffffu);
    if (low >> 31) continue;  // sharer: k_sshare adds the owner's counts
    const DPlan& P = plans[c];
    const DKernel& K = ks[P.kid];
    const DGpu& G = gs[P.gid];
    const long long S0 = (long long)srep[(long long)c * kSSlots + (low & 511u)];
    const SmBox32 b = block_box32(P, S0);
    const int ll = G.lg_line;
    // descriptors and pool planes of the entry: lanes over fields, one packed atomic
    int ndesc = 0, nplanes = 0, n_ld = 0;
    bool fits = true;
    for (int fi = lane; fi < K.n_fields; fi += 32) {
      const DField& F = K.f[fi];
      n_ld += F.kinds & 1;
      int y0, y1, z0, z1;
      if (!cfield_box(F, b, y0, y1, z0, z1)) continue;
      ++ndesc;
      nplanes += z1 - z0;
      if (z1 - z0 > 4096) fits = false;   // item code: plane index in 12 bits
    }
    ndesc = __reduce_add_sync(FULL, ndesc);
    nplanes = __reduce_add_sync(FULL, nplanes);
    n_ld = __reduce_add_sync(FULL, n_ld);
    fits = __all_sync(FULL, fits) && n_ld <= 4;   // many load fields: the CTA path's flat rows
    unsigned long long base = 0;
    if (fits && lane == 0) base = atomicAdd(cctr + 0, ((unsigned long long)ndesc << 40) | (unsigned long long)nplanes);
    base = __shfl_sync(FULL, base, 0);
    long long dbase = (long long)(base >> 40), pbase = (long long)(base & ((1ull << 40) - 1));
    fits = fits && dbase + ndesc <= desc_cap && dbase + ndesc <= (1 << 20) && pbase + nplanes <= pool_cap;
    if (!fits) {
      if (lane == 0) {
        const unsigned long long fb = atomicAdd(cctr + 2, 1ull);
        WS_CHK(fb, g_caps.sslots);
        cfbl[fb] = (uint32_t)e;
      }
      continue;
    }
    if (lane == 0 && ((low >> 30) & 1u)) {  // owner of a shared class: k_cfold accumulates the counts
      const unsigned t = (low >> 9) & (kShareTab - 1);
      sval[2 * t] = 0ull;
      sval[2 * t + 1] = 0ull;
    }
    // per load field: the descriptor, derived planes' sources, the computed-plane items
    for (int fi = 0; fi < K.n_fields; ++fi) {
      const DField& F = K.f[fi];
      int y0, y1, z0, z1;
      if (!cfield_box(F, b, y0, y1, z0, z1)) continue;
      const int per = plane_period(F.pitch[2], F.lg_elem, ll);
      const int np = z1 - z0;
      if (lane == 0) {
        CDesc d{(int)e, c, fi, per, z0, np, y0, y1 - y0, S0, pbase, {b.x0, b.x1, b.y0, b.y1, b.z0, b.z1}, {0, 0}};
        WS_CHK(dbase, g_caps.cdesc);
        cdesc[dbase] = d;
      }
      // windows of 32 planes (a multiple of per, a power of two <= 16): lane L's planes all have
      // the residue L mod per, so its derived planes' source -- the last computed plane of that
      // residue -- is carried across windows per lane
      const unsigned same_res = per > 0 ? (0xffffffffu / ((1u << per) - 1u)) << (lane % per) : 0u;
      // cplane_derived in O(1): plane z is computed iff some load group's z - oz lies in
      // [b.z0, b.z1) xor [b.z0 + per, b.z1 + per) = [L1, R1) u [L2, R2), i.e. iff the field's
      // load-offset mask (bit oz - ld_oz_min, lanes over the groups) has a bit in one of two ranges
      const int ozmin = F.ld_oz_min;
      const bool fast = F.ld_oz_max - ozmin < 64;
      unsigned long long ozm = 0;
      for (int g = F.g_begin + lane; g < F.g_end; g += 32) {
        const DGroup gr = K.g[g];
        if (gr.kind == 0) ozm |= 1ull << ((gr.oz - ozmin) & 63);
      }
      ozm = (unsigned long long)__reduce_or_sync(FULL, (unsigned)ozm) |
            ((unsigned long long)__reduce_or_sync(FULL, (unsigned)(ozm >> 32)) << 32);
      const int L1 = b.z0, R1 = min(b.z1, b.z0 + per), L2 = max(b.z1, b.z0 + per), R2 = b.z1 + per;
      auto any_bits = [&](int lo, int hi) {   // a bit of ozm in [lo, hi]
        lo = max(lo, 0);
        hi = min(hi, 63);
        if (hi < lo) return false;
        const int w = hi - lo + 1;
        return ((ozm >> lo) & (w == 64 ? ~0ull : ((1ull << w) - 1ull))) != 0ull;
      };
      auto derived = [&](int z) {
        if (!fast) return cplane_derived(K, F, b, z, z0, per);
        if (per <= 0 || z - per < z0) return false;
        return !(any_bits(z - R1 + 1 - ozmin, z - L1 - ozmin) || any_bits(z - R2 + 1 - ozmin, z - L2 - ozmin));
      };
      int ncomp = 0;
      for (int w0 = 0; w0 < np; w0 += 32) {  // count the computed planes (one item atomic per field)
        const int p = w0 + lane;
        ncomp += __popc(__ballot_sync(FULL, p < np && !derived(z0 + p)));
      }
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(cctr + 1, (unsigned long long)ncomp);
      at = __shfl_sync(FULL, at, 0);
      int carry = -1;
      for (int w0 = 0; w0 < np; w0 += 32) {
        const int p = w0 + lane;
        const bool in = p < np;
        const bool der = in && derived(z0 + p);
        const unsigned m = __ballot_sync(FULL, in && !der);   // computed planes of the window
        if (der) {
          const unsigned below = m & same_res & ((1u << lane) - 1u);
          const int src = below ? w0 + 31 - __clz(below) : carry;
          WS_CHK(pbase + p, g_caps.cpool);
          cpool[2 * (pbase + p)].c = -2 - (long long)src;  // derived: its computed source plane
        }
        if (in && !der) {
          WS_CHK(at + __popc(m & ((1u << lane) - 1u)), g_caps.cpool);
          citems[at + __popc(m & ((1u << lane) - 1u))] = (uint32_t)dbase | ((uint32_t)p << 20);
        }
        at += __popc(m);
        const unsigned mr = m & same_res;
        if (mr) carry = w0 + 31 - __clz(mr);
      }
      ++dbase;
      pbase += np;
    }
  }
}

// one warp per item (descriptor 20 bits | plane 12 bits): the computed plane's runs
__global__ void __launch_bounds__(256) k_cplanes(const DPlan* __restrict__ plans, const DKernel* __restrict__ ks,
                                                 const DGpu* __restrict__ gs, const CDesc* __restrict__ cdesc,
                                                 Tri* __restrict__ cpool, const uint32_t* __restrict__ citems,
                                                 const unsigned long long* __restrict__ cctr,
                                                 unsigned long long* __restrict__ work) {
  PDL_PROLOGUE();
  __shared__ SmWarp s_sw[8];
  __shared__ SmBox32 s_mb[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long total = (long long)cctr[1];
  const long long nwg = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned long long units = 0;
  for (long long it = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < total; it += nwg) {
    const uint32_t code = citems[it];
    const CDesc D = cdesc[code & 0xfffffu];
    const int p = (int)(code >> 20);
    const DPlan& P = plans[D.c];
    const DKernel& K = ks[P.kid];
    const DGpu& G = gs[P.gid];
    const DField& F = K.f[D.field];
    const int ls = G.lg_sector, ll = G.lg_line, le = F.lg_elem;
    const int g0 = F.g_begin, ng = F.g_end - F.g_begin;
    if (lane == 0) s_mb[wid] = SmBox32{D.box[0], D.box[1], D.box[2], D.box[3], D.box[4], D.box[5]};
    __syncwarp();
    SmWarp& Wp = s_sw[wid];
    const int z = D.z0 + p, y0 = D.y0, ny = D.ny;
    const long long py = F.pitch[1], pz = F.pitch[2];
    const long long R0p = F.align + ((py * y0 + pz * (long long)z) << le);
    const long long Bp = (R0p >> ll) << ll;
    const int off0 = (int)(R0p - Bp), step = (int)(py << le);
    T32 ps = t32_empty(), pl = t32_empty();
    for (int ys = 0; ys < ny; ys += kSegRowsS) {
      const int nseg = ny - ys < kSegRowsS ? ny - ys : kSegRowsS;
      const int nwd = (nseg + 31) >> 5;
      for (int w = lane; w < nwd; w += 32) Wp.bm[w] = 0u;
      __syncwarp();
      if (lane == 0) atomicOr(&Wp.bm[0], 1u);
      const SmBox32& bx = s_mb[wid];
      for (int k = lane; k < ng; k += 32) {  // breakpoints: rows where a group's row enters / leaves the block
        const DGroup gr = K.g[g0 + k];
        if (gr.kind != 0) continue;
        const int zz = z - gr.oz;
        if (zz < bx.z0 || zz >= bx.z1) continue;
        const int e0 = bx.y0 + gr.oy - y0 - ys, e1 = bx.y1 + gr.oy - y0 - ys;
        if (e0 > 0 && e0 < nseg) atomicOr(&Wp.bm[e0 >> 5], 1u << (e0 & 31));
        if (e1 > 0 && e1 < nseg) atomicOr(&Wp.bm[e1 >> 5], 1u << (e1 & 31));
      }
      __syncwarp();
      const int wpl = (nwd + 31) >> 5;
      int cnt = 0;
      for (int w = lane * wpl; w < nwd && w < (lane + 1) * wpl; ++w) cnt += __popc(Wp.bm[w]);
      int pos = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, pos, o);
        if (lane >= o) pos += v;
      }
      const int nruns = __shfl_sync(FULL, pos, 31);
      pos -= cnt;
      for (int w = lane * wpl; w < nwd && w < (lane + 1) * wpl; ++w) {
        unsigned bits = Wp.bm[w];
        while (bits) {
          const int bt = __ffs(bits) - 1;
          bits &= bits - 1;
          Wp.rs[pos++] = (short)(w * 32 + bt);
        }
      }
      if (lane == 0) Wp.rs[nruns] = (short)nseg;
      __syncwarp();
      for (int rb = 0; rb < nruns; rb += 32) {
        T32 tt[2] = {t32_empty(), t32_empty()};
        const int j = rb + lane;
        if (j < nruns) {
          const int yr = ys + Wp.rs[j];
          const T32x2 o = smset_run(&bx, 1, K, F, g0, ng, y0 + yr, z, off0 + yr * step, step, Wp.rs[j + 1] - Wp.rs[j],
                                    le, ls, ll);
          tt[0] = o.s;
          tt[1] = o.l;
        }
        warp_ordered_reduce32<2>(tt, nruns - rb);
        if (lane == 0) {
          ps = t32_combine(ps, tt[0]);
          pl = t32_combine(pl, tt[1]);
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
      const long long bs = Bp >> ls, bl = Bp >> ll;
      WS_CHK(D.off + p, g_caps.cpool);
      cpool[2 * (D.off + p)] = ps.c ? Tri{ps.f + bs, ps.l + bs, ps.c} : tri_empty();
      cpool[2 * (D.off + p) + 1] = pl.c ? Tri{pl.f + bl, pl.l + bl, pl.c} : tri_empty();
      units += (unsigned long long)ny;
    }
  }
  if (lane == 0 && units) atomicAdd(work + K_SCLASS, units);
}

// one warp per descriptor: ordered fold of the box's planes, counts x class size
__global__ void __launch_bounds__(256) k_cfold(const DPlan* __restrict__ plans, const DKernel* __restrict__ ks,
                                               const DGpu* __restrict__ gs, const unsigned long long* __restrict__ slist,
                                               const unsigned int* __restrict__ scnt, const CDesc* __restrict__ cdesc,
                                               const Tri* __restrict__ cpool, const unsigned long long* __restrict__ cctr,
                                               unsigned long long* __restrict__ acc, unsigned long long* __restrict__ sval) {
  PDL_PROLOGUE();
  const int lane = threadIdx.x & 31;
  const long long total = (long long)(cctr[0] >> 40);
  const long long nwg = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long d = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; d < total; d += nwg) {
    const CDesc D = cdesc[d];
    const DPlan& P = plans[D.c];
    const DField& F = ks[P.kid].f[D.field];
    const DGpu& G = gs[P.gid];
    const int ls = G.lg_sector, ll = G.lg_line;
    const long long pbytes = F.pitch[2] << F.lg_elem;
    const int ppl = (D.np + 31) / 32;
    Tri t[2] = {tri_empty(), tri_empty()};
    for (int p = lane * ppl; p < D.np && p < (lane + 1) * ppl; ++p) {
      int q = p;
      const long long mk = cpool[2 * (D.off + p)].c;
      if (mk < 0) q = (int)(-mk - 2);   // derived: its computed source plane (k_cplan)
      const long long dsh = (long long)(p - q) * pbytes;
      WS_CHK(D.off + q, g_caps.cpool);
      const Tri a = cpool[2 * (D.off + q)], bl = cpool[2 * (D.off + q) + 1];
      t[0] = tri_combine(t[0], a.c ? Tri{a.f + (dsh >> ls), a.l + (dsh >> ls), a.c} : tri_empty());
      t[1] = tri_combine(t[1], bl.c ? Tri{bl.f + (dsh >> ll), bl.l + (dsh >> ll), bl.c} : tri_empty());
    }
    warp_ordered_reduce<2>(t);
    if (lane == 0) {
      const unsigned long long ent = slist[D.entry];
      const unsigned low = (unsigned)(ent & 0xffffffffu);
      const unsigned long long mult = scnt[(long long)D.c * kSSlots + (low & 511u)];
      unsigned long long* a = acc + (long long)D.c * A_N;
      atomicAdd(a + A_SM_SEC, (unsigned long long)t[0].c * mult);
      atomicAdd(a + A_SM_LIN, (unsigned long long)t[1].c * mult);
      if ((low >> 30) & 1u) {  // owner of a shared class: the class's counts (over its load fields)
        const unsigned tt = (low >> 9) & (kShareTab - 1);
        atomicAdd(sval + 2 * tt, (unsigned long long)t[0].c);
        atomicAdd(sval + 2 * tt + 1, (unsigned long long)t[1].c);
      }
    }
  }
}

// Pass 2 (one CTA per entry): class representatives (counted class-size times), then the
// directly evaluated multi-block SM sets.
#ifdef WS_SCLASS_TRACE
__device__ unsigned long long g_sctrace[65536][2];  // diagnostics build: per-item cycles
#endif
__global__ void __launch_bounds__(WS_SCLASS_THREADS, WS_SCLASS_MINB) k_sclass(const DPlan* __restrict__ plans, const DKernel* __restrict__ ks,
                                                const DGpu* __restrict__ gs, unsigned long long* __restrict__ acc,
                                                const unsigned int* __restrict__ scnt,
                                                const unsigned long long* __restrict__ srep,
                                                unsigned long long* __restrict__ lists,
                                                const unsigned long long* __restrict__ slist,
                                                const unsigned long long* __restrict__ dlist,
                                                unsigned long long* __restrict__ work,
                                                unsigned long long* __restrict__ sval,
                                                const unsigned int* __restrict__ dmask,
                                                const uint32_t* __restrict__ cfbl,
                                                const unsigned long long* __restrict__ cctr,
                                                const unsigned long long* __restrict__ rctr) {
  PDL_PROLOGUE();
  __shared__ long long s_item;
  __shared__ SmBox s_mb[kMaxMembers];
  __shared__ SmBox32 s_mb32[kMaxMembers];
  __shared__ Tri s_pt[2 * kMaxPlanes];
  __shared__ unsigned char s_der[kMaxPlanes];
  __shared__ SmWarp s_sw[WS_SCLASS_THREADS / 32];
  __shared__ unsigned long long s_wsum[3];
  // class entries: all of them, or (class-plane path) only those k_cplan left to the CTA path
  const long long ncls = cfbl ? (long long)cctr[2] : (long long)lists[1], ndir = (long long)lists[2];
  // direct sets of kernels with many load fields split into (set, field) items: fs per set
  // (k_plan's batch maximum; 1 when no such kernel is in the batch)
  const unsigned long long fsr = rctr[rctr[8] * 4 + 3];
  const long long fs = fsr > 1 ? (long long)fsr : 1;
  const long long total = ncls + ndir * fs;
  if (total == 0) return;  // nothing for the CTA path (e.g. every SM set one block, classes by planes)
  // dynamic scheduling (lists[3], zeroed by the plan's scan): the directly evaluated sets --
  // the expensive, uneven entries -- first, then the single-block class representatives
  for (;;) {
    if (threadIdx.x == 0) s_item = (long long)atomicAdd(lists + 3, 1ull);
    __syncthreads();
    const long long item = s_item;
    __syncthreads();  // s_item is rewritten by the next fetch
    if (item >= total) break;
#ifdef WS_SCLASS_TRACE
    const long long t_item0 = clock64();
#endif
    const bool cls = item >= ndir * fs;
    const long long ce = cls ? (cfbl ? (long long)cfbl[item - ndir * fs] : item - ndir * fs) : 0;
    const long long ditem = cls ? 0 : item / fs;
    const int fsel = cls ? -1 : (int)(item - ditem * fs);
    const unsigned long long ent = cls ? slist[ce] : dlist[ditem];
    const int c = (int)(ent >> 32);
    const unsigned low = (unsigned)(ent & 0xffffffffu);
    const DPlan& P = plans[c];
    const DGpu& G = gs[P.gid];
    const long long nsm = G.g.n_sm;
    unsigned long long mult = 1;
    long long S0, kj;
    unsigned msk = 0u;  // direct item of one connected component of a set (k_smset)
    if (cls && (low >> 31)) continue;  // shared class: k_sshare adds the owner's counts
    if (cls) {
      const long long gslot = (long long)c * kSSlots + (low & 511u);
      mult = scnt[gslot];
      S0 = (long long)srep[gslot];
      kj = 1;
    } else if (P.rep_mult) {  // WS_VAR_REP_BLOCK: one block, counted for every wave block
      S0 = P.rep_B;
      kj = 1;
      mult = (unsigned long long)P.rep_mult;
    } else {  // directly evaluated set j (grouped: bit 31, group size - 1 in bits 20..30)
      const long long jj = (low & 0x80000000u) ? (long long)(low & 0xfffffu) : (long long)low;
      if (low & 0x80000000u) mult = 1ull + ((low >> 20) & 0x7ffu);
      S0 = P.s + jj;
      kj = (P.W - jj + nsm - 1) / nsm;
      msk = dmask[ditem];
    }
    unsigned long long ss, sl, un;
    const int n_ld = ks[P.kid].env.n_ld;
    int fonly = -1;   // (set, field) item of a many-field kernel's multi-block set; else the whole set
    if (!cls && fs > 1) {
      if (kj > 1 && n_ld > 4) {
        if (fsel >= ks[P.kid].n_fields) continue;
        fonly = fsel;
      } else if (fsel != 0) {
        continue;
      }
    }
    // one block of a kernel with many load fields (LBM): warps over whole fields, row runs per
    // plane (smset_eval_warps); otherwise the CTA's plane derivation + lane-per-run unions
    // (smset_cta; a many-field kernel's multi-block set one field per item).  A/B on B200 (LBM15):
    // multi-block LBM sets through a member-general smset_eval_warps made k_sclass 58 -> 85 us (a
    // lane walks every (group, member) pair per row run, and the one-block case slowed too)
    if (kj == 1 && n_ld > 4) {
      smset_eval_warps(P, ks[P.kid], G, S0, s_wsum, ss, sl, un);
      if (threadIdx.x == 0) atomicAdd(work + (cls ? K_SCLASS : K_SMSET), un);
    } else {        // several blocks: plane derivation + runs
      smset_cta(P, ks[P.kid], G, S0, kj, nsm, s_mb, s_mb32, s_pt, s_der, s_sw, ss, sl, un, msk, fonly);
      // every warp's lane 0 counted its planes' rows
      if ((threadIdx.x & 31) == 0 && un) atomicAdd(work + (cls ? K_SCLASS : K_SMSET), un);
    }
    if (threadIdx.x == 0) {
      unsigned long long* a = acc + (long long)c * A_N;
      atomicAdd(a + A_SM_SEC, ss * mult);
      atomicAdd(a + A_SM_LIN, sl * mult);
      if (cls && ((low >> 30) & 1u)) {  // owner of a shared class: publish the counts
        const unsigned t = (low >> 9) & (kShareTab - 1);
        sval[2 * t] = ss;
        sval[2 * t + 1] = sl;
      }
#ifdef WS_SCLASS_TRACE
      if (item < 65536) {
        g_sctrace[item][0] = ((unsigned long long)c << 32) | ((unsigned long long)kj << 1) | (cls ? 1u : 0u);
        g_sctrace[item][1] = (unsigned long long)(clock64() - t_item0) | ((unsigned long long)un << 40);
      }
#endif
    }
  }
}
#ifdef WS_SCLASS_TRACE
__global__ void k_sctrace_dump(const unsigned long long* __restrict__ lists, const DPlan* __restrict__ plans) {
  const long long total = (long long)lists[1] + (long long)lists[2];
  for (long long i = 0; i < total && i < 65536; ++i) {
    const unsigned long long a = g_sctrace[i][0], b = g_sctrace[i][1];
    const int c = (int)(a >> 32);
    if ((b & 0xffffffffffull) > WS_SCLASS_TRACE)
      printf("SCITEM c=%d b=(%d,%d,%d) f=(%d,%d,%d) kj=%d cls=%d rows=%llu cycles=%llu\n", c, plans[c].b[0], plans[c].b[1],
             plans[c].b[2], plans[c].f[0], plans[c].f[1], plans[c].f[2], (int)((a & 0xffffffffu) >> 1), (int)(a & 1),
             b >> 40, b & 0xffffffffffull);
    g_sctrace[i][1] = 0;
  }
}
#endif

// the shared classes' counts (owner evaluated in k_sclass) times each sharer's class size
__global__ void __launch_bounds__(256) k_sshare(const unsigned long long* __restrict__ lists,
                                                const unsigned long long* __restrict__ slist,
                                                const unsigned int* __restrict__ scnt,
                                                const unsigned long long* __restrict__ sval,
                                                unsigned long long* __restrict__ acc) {
  PDL_PROLOGUE();
  const long long ncls = (long long)lists[1];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ncls; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long ent = slist[i];
    const unsigned low = (unsigned)(ent & 0xffffffffu);
    if (!(low >> 31)) continue;
    const int c = (int)(ent >> 32);
    const unsigned t = (low >> 9) & (kShareTab - 1);
    const unsigned long long mult = scnt[(long long)c * kSSlots + (low & 511u)];
    unsigned long long* a = acc + (long long)c * A_N;
    atomicAdd(a + A_SM_SEC, sval[2 * t] * mult);
    atomicAdd(a + A_SM_LIN, sval[2 * t + 1] * mult);
  }
}

// ------------------------------------------------------------------ a5 + a6: wave and layer sets
// ranges: 0 = wave [s, s+W), 1 = L_y [Ly0, s), 2 = L_z [Lz0, s), 3 = L_y + wave, 4 = L_z + wave

__device__ __forceinline__ int classify(const RangeInfo& R, long long r) {
  if (!R.nonempty || r < R.ra || r > R.rl) return -1;
  if (R.ra == R.rl) return 3;
  if (r == R.ra) return 1;
  if (r == R.rl) return 2;
  return 0;
}

// Cached union of one row: a single component [x0, x1) (x0 >= x1: empty) or `multi`.
struct UC {
  long long x0, x1;
  int single;
};

template <class Gen>
__device__ __forceinline__ void row_union_c(const Gen& gen, long long R0, int le, int ls, int ll, Tri* ts, Tri* tl,
                                            Tri* ts2, UC& uc) {
  const long long INF = LLONG_MAX;
  long long start = INF, mx_s = LLONG_MIN, mn_e = INF, mx_e = LLONG_MIN;
  gen([&](long long xs, long long xe) {
    start = xs < start ? xs : start;
    mx_s = xs > mx_s ? xs : mx_s;
    mn_e = xe < mn_e ? xe : mn_e;
    mx_e = xe > mx_e ? xe : mx_e;
  });
  if (start == INF) {
    uc = UC{0, 0, 1};
    return;
  }
  if (mx_s <= mn_e) {
    uc = UC{start, mx_e, 1};
    const long long a0 = R0 + (start << le), a1 = R0 + ((mx_e - 1) << le);
    if (ts) tri_add(*ts, a0 >> ls, a1 >> ls);
    if (ts2) tri_add(*ts2, a0 >> ls, a1 >> ls);
    if (tl) tri_add(*tl, a0 >> ll, a1 >> ll);
    return;
  }
  uc.single = 0;
  row_union(gen, R0, le, ls, ll, ts, tl, ts2);
}

template <class Gen>
__device__ __forceinline__ void row_union_cached(const Gen& gen, bool first, long long R0, int le, int ls, int ll,
                                                 Tri* ts, Tri* tl, Tri* ts2, UC& uc) {
  if (first) {
    row_union_c(gen, R0, le, ls, ll, ts, tl, ts2, uc);
  } else if (uc.single) {
    if (uc.x0 < uc.x1) {
      const long long a0 = R0 + (uc.x0 << le), a1 = R0 + ((uc.x1 - 1) << le);
      if (ts) tri_add(*ts, a0 >> ls, a1 >> ls);
      if (ts2) tri_add(*ts2, a0 >> ls, a1 >> ls);
      if (tl) tri_add(*tl, a0 >> ll, a1 >> ll);
    }
  } else {
    row_union(gen, R0, le, ls, ll, ts, tl, ts2);
  }
}

#ifndef WS_ROW_WARPS
#define WS_ROW_WARPS 8
#endif
constexpr int kRowWarps = WS_ROW_WARPS;

constexpr int kSegRows = 1024;  // rows of a plane handled per k_rows segment

struct RI32 {
  int ra, rl;
  int iv[4][2];
  int nonempty, pad;
};

__device__ __forceinline__ int classify32(const RI32& R, int r) {
  if (!R.nonempty || r < R.ra || r > R.rl) return -1;
  if (R.ra == R.rl) return 3;
  if (r == R.ra) return 1;
  if (r == R.rl) return 2;
  return 0;
}

struct WarpRowCtx {
  RI32 r[5];
  int bnd[20];  // sorted distinct block rows where some range's classification zone starts
  int nb, pad;
  T32 pt[kNQ];                 // the plane's triples (lane 0)
  unsigned bm[kSegRows / 32];  // run-start bitmap of the current segment
  short rs[kSegRows + 2];      // run starts (ascending) + end
  // the field's offset groups whose cell plane z - oz lies in the domain, per computed plane:
  // x = Gy * block layer of z - oz (the block-row base), y = oy << 8 | run << 1 | kind
  int2 gv[kMaxAcc];
};

// Union of the candidates (range q1, mask m1) u (range q2, mask m2) over `run` consecutive rows
// (row 0 at plane offset R0, rows `step` bytes apart): sector triple (if want_s) and line
// triple (if want_l).  One out-of-line copy (instruction-cache footprint); the callers fold
// the triples into their compile-time targets.
__device__ __noinline__ T32x2 row_emit32(const WarpRowCtx& X, const DField& F, unsigned long long m1, int q1,
                                         unsigned long long m2, int q2, int R0, int step, int run, int le, int ls,
                                         int ll, bool want_s, bool want_l) {
  auto gen = [&](auto&& cb) {
    unsigned long long m = m1;
    while (m) {
      const int bb = __ffsll((long long)m) - 1;
      m &= m - 1;
      const int ty = bb >> 4, rr = bb & 15;
      cb(X.r[q1].iv[ty][0] + F.run_lo[rr], X.r[q1].iv[ty][1] + F.run_hi[rr]);
    }
    m = m2;
    while (m) {
      const int bb = __ffsll((long long)m) - 1;
      m &= m - 1;
      const int ty = bb >> 4, rr = bb & 15;
      cb(X.r[q2].iv[ty][0] + F.run_lo[rr], X.r[q2].iv[ty][1] + F.run_hi[rr]);
    }
  };
  const int INF = 0x7fffffff;
  int mn_s = INF, mx_s = -INF, mn_e = INF, mx_e = -INF;
  gen([&](int xs, int xe) {
    mn_s = xs < mn_s ? xs : mn_s;
    mx_s = xs > mx_s ? xs : mx_s;
    mn_e = xe < mn_e ? xe : mn_e;
    mx_e = xe > mx_e ? xe : mx_e;
  });
  T32x2 o{t32_empty(), t32_empty()};
  if (mn_s == INF) return o;
  if (mx_s <= mn_e) {  // one interval per row
    const int a0 = R0 + (mn_s << le), a1 = R0 + ((mx_e - 1) << le);
    if (want_s)
      o.s = run_triple32([&](int r) {
        const int s0 = (a0 + r * step) >> ls, s1 = (a1 + r * step) >> ls;
        return T32{s0, s1, s1 - s0 + 1};
      }, step, run, ls);
    if (want_l)
      o.l = run_triple32([&](int r) {
        const int s0 = (a0 + r * step) >> ll, s1 = (a1 + r * step) >> ll;
        return T32{s0, s1, s1 - s0 + 1};
      }, step, run, ll);
  } else {  // several intervals per row (the same components in every row of the run)
    if (want_s)
      o.s = run_triple32([&](int r) {
        T32 x = t32_empty();
        row_union32(gen, R0 + r * step, le, ls, x);
        return x;
      }, step, run, ls);
    if (want_l)
      o.l = run_triple32([&](int r) {
        T32 x = t32_empty();
        row_union32(gen, R0 + r * step, le, ll, x);
        return x;
      }, step, run, ll);
  }
  return o;
}

// compile-time targets t[TS] (sectors), t[TL] (lines), t[TS2] (sectors again); -1 = none
template <int TS, int TL, int TS2>
__device__ __forceinline__ void row_emit32(T32 (&t)[kNQ], const WarpRowCtx& X, const DField& F, unsigned long long m1,
                                           int q1, unsigned long long m2, int q2, int R0, int step, int run, int le,
                                           int ls, int ll) {
  const T32x2 o = row_emit32(X, F, m1, q1, m2, q2, R0, step, run, le, ls, ll, TS >= 0 || TS2 >= 0, TL >= 0);
  if (TS >= 0) t[TS >= 0 ? TS : 0] = t32_combine(t[TS >= 0 ? TS : 0], o.s);
  if (TS2 >= 0) t[TS2 >= 0 ? TS2 : 0] = t32_combine(t[TS2 >= 0 ? TS2 : 0], o.s);
  if (TL >= 0) t[TL >= 0 ? TL : 0] = t32_combine(t[TL >= 0 ? TL : 0], o.l);
}

__device__ __forceinline__ int fdiv32(int n, FDiv f) { return (int)((__umulhi((unsigned)n, f.m) + (unsigned)n) >> f.l); }

#ifdef WS_ROWS_TRACE
constexpr long long kRowTrace = 1 << 17;
__device__ unsigned long long g_rowtrace[kRowTrace][2];
// diagnostics build: print the computed planes of the last k_rows launch, slowest first is left to
// the reader (one line per computed plane with cycles > WS_ROWS_TRACE)
__global__ void k_rowtrace_dump(const unsigned long long* __restrict__ rctr) {
  const long long nit = (long long)rctr[rctr[8] * 4 + 0];
  const long long total = nit < kRowTrace ? nit : kRowTrace;
  for (long long i = 0; i < total; ++i) {
    const unsigned long long a = g_rowtrace[i][0], b = g_rowtrace[i][1];
    if ((b & 0xffffffffffull) > WS_ROWS_TRACE)
      printf("ROWITEM c=%d field=%d z=%d runs=%d cycles=%llu\n", (int)(a >> 40), (int)((a >> 32) & 255),
             (int)(a & 0xffffffffu), (int)(b >> 40), b & 0xffffffffffull);
    g_rowtrace[i][1] = 0;
  }
}
#endif

// One warp per (config, field, z-plane) of the row box of the wave + layer-set footprint.
//  * Plane derivation: a plane whose every offset group falls in the same block layer (or the
//    same side outside the domain) as its representative (start of that zone segment, aligned
//    to the reuse period per) is that plane's translate by whole lines: only marked here,
//    translated by k_fold.
//  * Computed planes: a row's candidate masks change only where some offset group's region row
//    enters another classification zone (the 5 ranges' first / second / last / after-last block
//    rows) or the domain.  Lanes mark these breakpoints in a bitmap, compact the run starts, then
//    take one run each: masks of its first row, the <= 7 unions, the run's triple in closed form
//    (rows of a run are translates).  An ordered warp reduction of the lanes' 9 triples gives the
//    plane's contribution.  All of it in 32-bit plane-relative arithmetic.
__global__ void __launch_bounds__(kRowWarps * 32, WS_ROWS_MINB) k_rows(const DPlan* __restrict__ plans,
                                                            const DKernel* __restrict__ ks,
                                                            const DGpu* __restrict__ gs,
                                                            const DRowInfo* __restrict__ rowinfo,
                                                            long long* __restrict__ chunkres,
                                                            unsigned long long* __restrict__ work,
                                                            const unsigned long long* __restrict__ rctr,
                                                            const unsigned long long* __restrict__ ritems) {
  PDL_PROLOGUE();
  __shared__ WarpRowCtx s_ctx[kRowWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpRowCtx& X = s_ctx[wid];
  // computed chunks only: k_plan's reserved item list (config << 32 | field << 26 | chunk)
  const long long total = (long long)rctr[rctr[8] * 4 + 0];
  const long long nwg = (long long)gridDim.x * kRowWarps;
  unsigned long long my_ops = 0;
  int ranges_c = -1;
  int c = -1;
  // block-row span of each range: r in range q iff (unsigned)(r - rra[q]) <= rsp[q] (empty: rra far
  // below every row, rsp 0); classification (r == rra) + 2 (r == rrl): 1 first, 2 last, 3 both, 0 inside
  int rra[5] = {0, 0, 0, 0, 0}, rrl[5] = {0, 0, 0, 0, 0};
  unsigned rsp[5] = {0, 0, 0, 0, 0};
#ifndef WS_ROWS_SPREAD
#define WS_ROWS_SPREAD 0
#endif
  // item order: consecutive items (neighbouring planes of one configuration) go to the 8 warps of
  // one CTA; WS_ROWS_SPREAD=1 spreads them over CTAs (A/B on B200: 0.193 vs 0.170 ms per configs[1]
  // step, k_rows 90.6 vs 79.6 us serial -- the shared per-configuration data stays in one SM's L1)
  const long long item0 = WS_ROWS_SPREAD ? (long long)wid * gridDim.x + blockIdx.x : (long long)blockIdx.x * kRowWarps + wid;
  for (long long item = item0; item < total; item += nwg) {
#ifdef WS_ROWS_TRACE
    const long long t_item0 = clock64();
    int tr_runs = 0;
#endif
    const unsigned long long ent = ritems[item];
    c = (int)(ent >> 32);
    const int fi = (int)((ent >> 26) & 63ull);
    const long long ci = (long long)(ent & ((1ull << 26) - 1ull));
    const DPlan& P = plans[c];
    const DKernel& K = ks[P.kid];
    const DGpu& G = gs[P.gid];
    WS_CHK((long long)c * kMaxFields + fi, g_caps.rowinfo);
    const DRowInfo RI = rowinfo[(long long)c * kMaxFields + fi];
    const DField& F = K.f[fi];
    const int g0 = F.g_begin, ng = F.g_end - F.g_begin;
    const int ls = G.lg_sector, ll = G.lg_line, le = F.lg_elem;
    const int lo1 = (int)P.lo[1], hi1 = (int)P.hi[1], lo2 = (int)P.lo[2], hi2 = (int)P.hi[2];
    const int Gy = (int)P.G[1], BF1 = (int)P.BF[1];
    const FDiv fdy = P.fd_BF[1], fdz = P.fd_BF[2];
    const int y0 = (int)RI.y0, ny = (int)RI.ny;
    // chunk = (plane, row segment of kRowSeg rows): a plane's runs spread over several warps
    const int nsg = (int)RI.nseg, pci = (int)(ci - RI.chunk_begin);
    const int z = (int)RI.z0 + pci / nsg, sg = pci % nsg;
    const int ys0 = y0 + sg * kRowSeg, ys1 = ys0 + kRowSeg < y0 + ny ? ys0 + kRowSeg : y0 + ny;
    long long py, pz, falign;
    field_rows(F, P, ll, py, pz, falign);
    if (ranges_c != c) {  // ranges and zone boundaries of this config (k_plan) -> warp smem, 32-bit
      __syncwarp();
      if (lane < 5) {
        const RangeInfo& R = P.rng[lane];
        RI32 r32;
        r32.ra = (int)R.ra;
        r32.rl = (int)R.rl;
        for (int a = 0; a < 4; ++a) {
          r32.iv[a][0] = (int)R.iv[a][0];
          r32.iv[a][1] = (int)R.iv[a][1];
        }
        r32.nonempty = R.nonempty;
        r32.pad = 0;
        X.r[lane] = r32;
      }
      if (lane < 20) X.bnd[lane] = (int)P.bnd[lane];
      __syncwarp();
      ranges_c = c;
#pragma unroll
      for (int q = 0; q < 5; ++q) {  // block-row span of each range in registers
        rra[q] = P.rng[q].nonempty ? (int)P.rng[q].ra : -0x40000000;
        rrl[q] = P.rng[q].nonempty ? (int)P.rng[q].rl : -0x40000000;
        rsp[q] = P.rng[q].nonempty ? (unsigned)(P.rng[q].rl - P.rng[q].ra) : 0u;
      }
    }
    const int nb = P.nb;
    const long long R0p = falign + ((py * y0 + pz * z) << le);
    const long long Bp = (R0p >> ll) << ll;
    const int off0 = (int)(R0p - Bp);
    const int pystep = (int)(py << le);
    if (lane < kNQ) X.pt[lane] = t32_empty();
    // this plane's valid groups and their block-row bases, once (lanes over the groups)
    int ngv = 0, ngl = 0;   // valid groups, loads first (ngl of them), then stores
    for (int kind = 0; kind < 2; ++kind) {
      for (int gb = 0; gb < ng; gb += 32) {
        const int g = gb + lane;
        bool v = false;
        int2 e = make_int2(0, 0);
        if (g < ng) {
          const DGroup gr = K.g[g0 + g];
          const int zz = z - gr.oz;
          v = gr.kind == kind && zz >= lo2 && zz < hi2;
          if (v) e = make_int2(Gy * fdiv32(zz - lo2, fdz), (gr.oy << 8) | (gr.run << 1) | (gr.kind & 1));
        }
        const unsigned bal = __ballot_sync(FULL, v);
        if (v) X.gv[ngv + __popc(bal & ((1u << lane) - 1u))] = e;
        ngv += __popc(bal);
      }
      if (kind == 0) ngl = ngv;
    }
    __syncwarp();
    for (int ys = ys0; ys < ys1; ys += kSegRows) {
      const int nseg = ys1 - ys < kSegRows ? ys1 - ys : kSegRows;
      const int nwd = (nseg + 31) >> 5;
      for (int w = lane; w < nwd; w += 32) X.bm[w] = 0u;
      __syncwarp();
      if (lane == 0) atomicOr(&X.bm[0], 1u);
      my_ops += (unsigned long long)(lane < ng ? 8 * (nb + 2) : 0);
      for (int g = lane; g < ngv; g += 32) {
        const int2 e = X.gv[g];
        const int C = e.x, oy = e.y >> 8;
        auto mark = [&](int yb) {
          const int i = yb - ys;
          if (i > 0 && i < nseg) atomicOr(&X.bm[i >> 5], 1u << (i & 31));
        };
        mark(lo1 + oy);
        mark(hi1 + oy);
        for (int k = 0; k < nb; ++k) {
          const int d = X.bnd[k] - C;
          if (d > 0 && d < Gy) mark(lo1 + d * BF1 + oy);
        }
      }
      __syncwarp();
      // compact the run starts (ascending) into X.rs
      const int wpl = (nwd + 31) >> 5;
      int cnt = 0;
      for (int w = lane * wpl; w < nwd && w < (lane + 1) * wpl; ++w) cnt += __popc(X.bm[w]);
      int pos = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, pos, o);
        if (lane >= o) pos += v;
      }
      const int nruns = __shfl_sync(FULL, pos, 31);
#ifdef WS_ROWS_TRACE
      tr_runs += nruns;
#endif
      pos -= cnt;
      for (int w = lane * wpl; w < nwd && w < (lane + 1) * wpl; ++w) {
        unsigned bits = X.bm[w];
        while (bits) {
          const int bt = __ffs(bits) - 1;
          bits &= bits - 1;
          X.rs[pos++] = (short)(w * 32 + bt);
        }
      }
      if (lane == 0) X.rs[nruns] = (short)nseg;
      __syncwarp();
#ifndef WS_ROWS_CONTIG   // 1: contiguous runs per lane, one reduction per segment (A/B on B200:
#define WS_ROWS_CONTIG 0 // k_rows 63 vs 51 us serial -- the longer per-lane loop; rounds kept)
#endif
#if WS_ROWS_CONTIG
      // lanes take contiguous runs (in row order): one ordered reduction per segment
      const int rpl = (nruns + 31) >> 5, nact = (nruns + rpl - 1) / rpl;
      {
        T32 t[kNQ];
#pragma unroll
        for (int q = 0; q < kNQ; ++q) t[q] = t32_empty();
        for (int j = lane * rpl; j < nruns && j < (lane + 1) * rpl; ++j) {
#else
      // rounds of 32 runs, a run per lane, an ordered reduction per round
      for (int rb = 0; rb < nruns; rb += 32) {
        const int nact = nruns - rb < 32 ? nruns - rb : 32;
        T32 t[kNQ];
#pragma unroll
        for (int q = 0; q < kNQ; ++q) t[q] = t32_empty();
        const int j = rb + lane;
        if (j < nruns) {
#endif
          const int y = ys + X.rs[j];
          const int run = X.rs[j + 1] - X.rs[j];
          my_ops += (unsigned long long)(30 * ng + 72 * run);
          unsigned long long mL[5] = {0, 0, 0, 0, 0}, mS[5] = {0, 0, 0, 0, 0};
          auto classify = [&](int g, unsigned long long (&m)[5]) {
            const int2 e = X.gv[g];
            const int yy = y - (e.y >> 8);
            if (yy < lo1 || yy >= hi1) return;
            const int r = fdiv32(yy - lo1, fdy) + e.x;
            const unsigned long long b0 = 1ull << ((e.y >> 1) & 15);
#pragma unroll
            for (int q = 0; q < 5; ++q) {  // classify32 from registers
              const int ty = (r == rra[q] ? 1 : 0) + (r == rrl[q] ? 2 : 0);
              m[q] |= (unsigned)(r - rra[q]) <= rsp[q] ? b0 << (ty * 16) : 0ull;
            }
          };
          for (int g = 0; g < ngl; ++g) classify(g, mL);
          for (int g = ngl; g < ngv; ++g) classify(g, mS);
          const int R0 = off0 + (y - y0) * pystep;
          const bool noS = mS[0] == 0ull, noL = mL[0] == 0ull;
          if (noS) {
            row_emit32<0, 2, -1>(t, X, F, mL[0], 0, 0ull, 0, R0, pystep, run, le, ls, ll);
          } else if (noL) {
            row_emit32<1, 2, -1>(t, X, F, mS[0], 0, 0ull, 0, R0, pystep, run, le, ls, ll);
          } else {
            row_emit32<0, -1, -1>(t, X, F, mL[0], 0, 0ull, 0, R0, pystep, run, le, ls, ll);
            row_emit32<1, -1, -1>(t, X, F, mS[0], 0, 0ull, 0, R0, pystep, run, le, ls, ll);
            row_emit32<-1, 2, -1>(t, X, F, mL[0] | mS[0], 0, 0ull, 0, R0, pystep, run, le, ls, ll);
          }
          if (!noL) {
            row_emit32<3, 4, -1>(t, X, F, mL[1] | mS[1], 1, 0ull, 1, R0, pystep, run, le, ls, ll);
            row_emit32<5, 6, -1>(t, X, F, mL[2] | mS[2], 2, 0ull, 2, R0, pystep, run, le, ls, ll);
            row_emit32<7, -1, -1>(t, X, F, mL[3], 3, mS[1], 1, R0, pystep, run, le, ls, ll);
            row_emit32<8, -1, -1>(t, X, F, mL[4], 4, mS[2], 2, R0, pystep, run, le, ls, ll);
          } else {
            row_emit32<3, 4, 7>(t, X, F, mL[1] | mS[1], 1, 0ull, 1, R0, pystep, run, le, ls, ll);
            row_emit32<5, 6, 8>(t, X, F, mL[2] | mS[2], 2, 0ull, 2, R0, pystep, run, le, ls, ll);
          }
        }
        warp_ordered_reduce32<kNQ>(t, nact);
        if (lane == 0)  // plane triples: lane 0 only
#pragma unroll
          for (int q = 0; q < kNQ; ++q) X.pt[q] = t32_combine(X.pt[q], t[q]);
      }
      __syncwarp();
    }
    if (lane < kNQ) {   // the plane's triples out, one per lane (X.pt written by lane 0 before the syncwarp)
      const int q = lane;
      WS_CHK(P.chunk_base + ci, g_caps.max_chunks);
      long long* out = chunkres + (P.chunk_base + ci) * (kNQ * 3);
      const long long b = (q == 2 || q == 4 || q == 6) ? (Bp >> ll) : (Bp >> ls);
      const T32 v = X.pt[q];
      out[q * 3 + 0] = v.c ? v.f + b : 0;
      out[q * 3 + 1] = v.c ? v.l + b : 0;
      out[q * 3 + 2] = v.c;
    }
#ifdef WS_ROWS_TRACE  // diagnostics build: per computed plane (config, field, z, runs, cycles)
    if (lane == 0 && item < kRowTrace) {
      g_rowtrace[item][0] = ((unsigned long long)c << 40) | ((unsigned long long)fi << 32) | (unsigned)z;
      g_rowtrace[item][1] = ((unsigned long long)tr_runs << 40) | (unsigned long long)(clock64() - t_item0);
    }
#endif
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) my_ops += __shfl_down_sync(FULL, my_ops, o);
  if (lane == 0 && my_ops) atomicAdd(work + K_ROWS, my_ops);
}

// one CTA per (config, field): threads take contiguous planes, ordered CTA reduction
__device__ void fold_cta(const DPlan* __restrict__ plans, long long total, const uint32_t* __restrict__ fitems,
                         const DKernel* __restrict__ ks, const DGpu* __restrict__ gs, const DRowInfo* __restrict__ rowinfo,
                         const long long* __restrict__ chunkres, unsigned long long* __restrict__ acc) {
  __shared__ Tri s_red[(256 / 32) * kNQ];
  const int tid = threadIdx.x;
  for (long long item = blockIdx.x; item < total; item += gridDim.x) {
    const uint32_t ent = fitems[item];   // k_plan's reserved fold items: config << 6 | field
    const int c = (int)(ent >> 6), fi = (int)(ent & 63u);
    const DPlan& P = plans[c];
    const DField& F = ks[P.kid].f[fi];
    const DGpu& G = gs[P.gid];
    const int ls = G.lg_sector, ll = G.lg_line;
    long long py, pz, falign;
    field_rows(F, P, ll, py, pz, falign);
    const long long pbytes = pz << F.lg_elem;
    const DRowInfo RI = rowinfo[(long long)c * kMaxFields + fi];
    const long long nch = RI.n_chunks;
    const long long per_l = (nch + blockDim.x - 1) / blockDim.x;
    const long long* base = chunkres + (P.chunk_base + RI.chunk_begin) * (kNQ * 3);
    Tri t[kNQ];
#pragma unroll
    for (int q = 0; q < kNQ; ++q) t[q] = tri_empty();
    const DGroup* gk = ks[P.kid].g + F.g_begin;
    const int per = plane_period(pz, F.lg_elem, ll);
#pragma unroll 2   // two planes' loads in flight
    for (long long k = tid * per_l; k < nch && k < (tid + 1) * per_l; ++k) {
      // derived plane: its representative's triple, translated (plane_rep, as in k_plan)
      const long long pi = k / RI.nseg;
      const int zr = plane_rep_f(F, gk, (int)(RI.z0 + pi), (int)RI.z0, (int)P.lo[2], (int)P.hi[2], (int)P.BF[2],
                               P.fd_BF[2], per);
      const long long src = (zr - RI.z0) * RI.nseg + (k - pi * RI.nseg);
      WS_CHK(P.chunk_base + RI.chunk_begin + src, g_caps.max_chunks);
      const long long* in = base + src * (kNQ * 3);
      const long long dbytes = ((k - src) / RI.nseg) * pbytes;   // same row segment, whole planes apart
#pragma unroll
      for (int q = 0; q < kNQ; ++q) {
        const long long d = dbytes >> ((q == 2 || q == 4 || q == 6) ? ll : ls);
        const long long cq = in[q * 3 + 2];
        t[q] = tri_combine(t[q], cq ? Tri{in[q * 3] + d, in[q * 3 + 1] + d, cq} : tri_empty());
      }
    }
    // the ordered CTA reduction in 32-bit item-relative indices when the item's span fits (half the
    // shuffles of the 64-bit triples); only the counts leave the fold
    const long long a0 = falign + ((py * RI.y0 + pz * RI.z0) << F.lg_elem);
    if (((RI.nz * pbytes) >> ls) < (1ll << 29)) {
      const long long bs = (a0 >> ls) - (1ll << 24), bl = (a0 >> ll) - (1ll << 24);
      T32 u[kNQ];
#pragma unroll
      for (int q = 0; q < kNQ; ++q) {
        const long long b = (q == 2 || q == 4 || q == 6) ? bl : bs;
        u[q] = t[q].c ? T32{(int)(t[q].f - b), (int)(t[q].l - b), (int)t[q].c} : t32_empty();
      }
      warp_ordered_reduce32<kNQ>(u);
      __shared__ T32 s_red32[(256 / 32) * kNQ];
      const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < kNQ; ++q) s_red32[warp * kNQ + q] = u[q];
      __syncthreads();
      if (tid < kNQ) {
        T32 a = s_red32[tid];
        for (int w = 1; w < nw; ++w) a = t32_combine(a, s_red32[w * kNQ + tid]);
        s_red32[tid] = a;
      }
      __syncthreads();
      if (tid == 0)
#pragma unroll
        for (int q = 0; q < kNQ; ++q) t[q].c = s_red32[q].c;
      __syncthreads();
    } else {
      cta_ordered_reduce<kNQ>(t, s_red);
    }
    if (tid == 0 && nch > 0) {
      unsigned long long* a = acc + (long long)c * A_N;
      atomicAdd(a + A_WLD, (unsigned long long)t[0].c);
      atomicAdd(a + A_WST, (unsigned long long)t[1].c);
      atomicAdd(a + A_WLIN, (unsigned long long)t[2].c);
      atomicAdd(a + A_LY, (unsigned long long)t[4].c);
      atomicAdd(a + A_LZ, (unsigned long long)t[6].c);
      atomicAdd(a + A_OVY, (unsigned long long)(t[0].c + t[3].c - t[7].c));
      atomicAdd(a + A_OVZ, (unsigned long long)(t[0].c + t[5].c - t[8].c));
    }
  }
}

// Ordered fold of the plane triples of one (config, field); one warp per item.  A derived
// plane (count slot = -(representative index) - 2) takes its representative's triple
// translated by the plane distance (a multiple of the reuse period: whole lines).
__global__ void __launch_bounds__(256, WS_FOLD_MINB) k_fold(const DPlan* __restrict__ plans,
                                              const unsigned long long* __restrict__ rctr,
                                              const uint32_t* __restrict__ fitems,
                                              const DKernel* __restrict__ ks, const DGpu* __restrict__ gs,
                                              const DRowInfo* __restrict__ rowinfo,
                                              const long long* __restrict__ chunkres,
                                              unsigned long long* __restrict__ acc, int mode) {
  PDL_PROLOGUE();
  const long long total = (long long)rctr[rctr[8] * 4 + 2];
  const int lane = threadIdx.x & 31;
  // items (config, field) <= CTAs (BJ configs[1]: 336 items x ~40 planes): one CTA per item (all
  // items at once, 256 threads each); more items (LBM: 58 fields per config): one warp per item.
  // (A/B on B200: 0.202 vs 0.212 ms per configs[1] step; LBM15 0.238 vs 0.284 ms the other way.)
  // mode: 0 = that choice, 1 = CTA, 2 = warp (WS_FOLD_MODE, diagnostics)
  if (mode == 1 || (mode == 0 && total <= gridDim.x)) {
    fold_cta(plans, total, fitems, ks, gs, rowinfo, chunkres, acc);
    return;
  }
  const long long nwg = ((long long)gridDim.x * blockDim.x) >> 5;
  // one warp per (config, field): lanes take contiguous planes, ordered warp reduction
  for (long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < total; item += nwg) {
    const uint32_t ent = fitems[item];
    const int c = (int)(ent >> 6), fi = (int)(ent & 63u);
    const DPlan& P = plans[c];
    const DField& F = ks[P.kid].f[fi];
    const DGpu& G = gs[P.gid];
    const int ls = G.lg_sector, ll = G.lg_line;
    long long py, pz, falign;
    field_rows(F, P, ll, py, pz, falign);
    const long long pbytes = pz << F.lg_elem;
    const DRowInfo RI = rowinfo[(long long)c * kMaxFields + fi];
    const long long nch = RI.n_chunks;
    const long long per_l = (nch + 31) / 32;
    const long long* base = chunkres + (P.chunk_base + RI.chunk_begin) * (kNQ * 3);
    Tri t[kNQ];
#pragma unroll
    for (int q = 0; q < kNQ; ++q) t[q] = tri_empty();
    const DGroup* gk = ks[P.kid].g + F.g_begin;
    const int per = plane_period(pz, F.lg_elem, ll);
#pragma unroll 2   // two planes' loads in flight
    for (long long k = lane * per_l; k < nch && k < (lane + 1) * per_l; ++k) {
      const long long pi = k / RI.nseg;   // derived plane: its representative's triple, translated
      const int zr = plane_rep_f(F, gk, (int)(RI.z0 + pi), (int)RI.z0, (int)P.lo[2], (int)P.hi[2], (int)P.BF[2],
                               P.fd_BF[2], per);
      const long long src = (zr - RI.z0) * RI.nseg + (k - pi * RI.nseg);
      WS_CHK(P.chunk_base + RI.chunk_begin + src, g_caps.max_chunks);
      const long long* in = base + src * (kNQ * 3);
      const long long dbytes = ((k - src) / RI.nseg) * pbytes;   // same row segment, whole planes apart
#pragma unroll
      for (int q = 0; q < kNQ; ++q) {
        const long long d = dbytes >> ((q == 2 || q == 4 || q == 6) ? ll : ls);
        const long long cq = in[q * 3 + 2];
        t[q] = tri_combine(t[q], cq ? Tri{in[q * 3] + d, in[q * 3 + 1] + d, cq} : tri_empty());
      }
    }
    warp_ordered_reduce<kNQ>(t);
    if (lane == 0 && nch > 0) {
      unsigned long long* a = acc + (long long)c * A_N;
      atomicAdd(a + A_WLD, (unsigned long long)t[0].c);
      atomicAdd(a + A_WST, (unsigned long long)t[1].c);
      atomicAdd(a + A_WLIN, (unsigned long long)t[2].c);
      atomicAdd(a + A_LY, (unsigned long long)t[4].c);
      atomicAdd(a + A_LZ, (unsigned long long)t[6].c);
      // |WLD n F_L| = |WLD| + |F_L| - |WLD u F_L|  (per field; fields never alias)
      atomicAdd(a + A_OVY, (unsigned long long)(t[0].c + t[3].c - t[7].c));
      atomicAdd(a + A_OVZ, (unsigned long long)(t[0].c + t[5].c - t[8].c));
    }
  }
}

// ------------------------------------------------------------------ NEXT-4: pages + L2 sections
// Union of the element intervals produced by gen(cb) in one address row (element 0 at byte
// R0): appends the union's sectors (ts), lines (tl) and pages (tp) in increasing order.
template <class Gen>
__device__ __forceinline__ void row_union_p(const Gen& gen, long long R0, int le, int ls, int ll, int lp, Tri* ts,
                                            Tri* tl, Tri* tp) {
  const long long INF = LLONG_MAX;
  long long start = INF;
  gen([&](long long xs, long long xe) { start = xs < start ? xs : start; });
  while (start != INF) {
    long long end = start, nxt;
    bool grew;
    do {
      grew = false;
      nxt = INF;
      gen([&](long long xs, long long xe) {
        if (xs <= end) {
          if (xe > end) {
            end = xe;
            grew = true;
          }
        } else if (xs < nxt) {
          nxt = xs;
        }
      });
    } while (grew);
    const long long a0 = R0 + (start << le), a1 = R0 + ((end - 1) << le);
    if (ts) tri_add(*ts, a0 >> ls, a1 >> ls);
    if (tl) tri_add(*tl, a0 >> ll, a1 >> ll);
    if (tp) tri_add(*tp, a0 >> lp, a1 >> lp);
    start = nxt;
  }
}

constexpr int kSectNQ = 2 * kMaxSections + 3;  // per section: load sectors, lines; union: load sectors, lines; pages
static_assert(kSectNQ * sizeof(Tri) == kSectPartBytes, "k_sect partial size");

// One CTA per (config, field) of the configs that want the outlook metrics.
// Linear address space.  The wave's rows (y, z) are walked in address order, threads taking
// contiguous row ranges; per row and offset group, the wave blocks of the group's block row
// are split into pieces of one L2 section (SM j = (B - s) mod n_sm belongs to section
// floor(j * S / n_sm)), each piece a cell x-interval shifted by the group's x-run.  Unions
// per section and over all sections give ordered triples; an ordered CTA reduction gives the
// field's counts.
// One CTA per (config, field, row segment): kSectSeg segments of the field's rows; the CTA that
// finishes an item's last segment folds the segments' partial triples in row order.
__global__ void __launch_bounds__(256) k_sect(const DPlan* __restrict__ plans, const DPrefix* __restrict__ pre, int n,
                                              const DKernel* __restrict__ ks, const DGpu* __restrict__ gs,
                                              unsigned long long* __restrict__ acc,
                                              unsigned long long* __restrict__ work, Tri* __restrict__ spart,
                                              unsigned int* __restrict__ sdone, int max_fields) {
  PDL_PROLOGUE();
  __shared__ Tri s_red[(256 / 32) * kSectNQ];
  __shared__ int s_last;
  const long long total = pre[n].sect * kSectSeg;
  const int tid = threadIdx.x, nt = blockDim.x;
  unsigned long long my_ops = 0;
  int c = -1;
  for (long long it2 = blockIdx.x; it2 < total; it2 += gridDim.x) {
    const long long item = it2 / kSectSeg;
    const int seg = (int)(it2 % kSectSeg);
    c = find_config_warp<6>(pre, n, item, c);
    const int fi = (int)(item - pre[c].sect);
    const DPlan& P = plans[c];
    const DKernel& K = ks[P.kid];
    const DGpu& G = gs[P.gid];
    const DField& F = K.f[fi];
    const int le = F.lg_elem, ls = G.lg_sector, ll = G.lg_line, lp = G.lg_page >= 0 ? G.lg_page : ll;
    const int S = (int)G.g.l2_sections;
    const long long nsm = G.g.n_sm, s = P.s, Wb = P.W, Gx = P.G[0], Gy = P.G[1];
    // cell box of the wave's block rows, then the field rows its accesses can touch
    const long long rA = s / Gx, rB = (s + Wb - 1) / Gx;
    const long long byA = rA % Gy, bzA = rA / Gy, byB = rB % Gy, bzB = rB / Gy;
    long long ylo = P.lo[1], yhi = P.hi[1];
    if (bzA == bzB) {
      ylo = P.lo[1] + byA * P.BF[1];
      yhi = P.lo[1] + (byB + 1) * P.BF[1];
      if (yhi > P.hi[1]) yhi = P.hi[1];
    }
    long long zlo = P.lo[2] + bzA * P.BF[2], zhi = P.lo[2] + (bzB + 1) * P.BF[2];
    if (zhi > P.hi[2]) zhi = P.hi[2];
    long long y0 = ylo + F.oy_min, y1 = yhi + F.oy_max, z0 = zlo + F.oz_min, z1 = zhi + F.oz_max;
    if (y0 < 0) y0 = 0;
    if (z0 < 0) z0 = 0;
    if (y1 > F.ext[1]) y1 = F.ext[1];
    if (z1 > F.ext[2]) z1 = F.ext[2];
    const long long ny = y1 > y0 ? y1 - y0 : 0, nz = z1 > z0 ? z1 - z0 : 0;
    const long long nrows = (F.g_end > F.g_begin) ? ny * nz : 0;
    const long long r_begin = nrows * seg / kSectSeg, r_end = nrows * (seg + 1) / kSectSeg;
    const long long per = (r_end - r_begin + nt - 1) / nt;
    Tri t[kSectNQ];
#pragma unroll
    for (int q = 0; q < kSectNQ; ++q) t[q] = tri_empty();
    // per row: each offset group's block row and its wave-block range, computed once (32-bit,
    // multiply-high divisions), then the unions scan the cached list
    int c_b0[kMaxAcc], c_b1[kMaxAcc], c_rx[kMaxAcc], c_g[kMaxAcc];
    const int lo0 = (int)P.lo[0], hi0 = (int)P.hi[0], lo1 = (int)P.lo[1], hi1 = (int)P.hi[1];
    const int lo2 = (int)P.lo[2], hi2 = (int)P.hi[2], BF0 = (int)P.BF[0];
    const unsigned nsm32 = (unsigned)nsm, S32 = (unsigned)S;
    const FDiv fd_nsm = make_fdiv((unsigned long long)nsm);
    int a_sec[kMaxSections + 1];  // first SM index of each section: ceil(i * n_sm / S)
#pragma unroll
    for (int i = 0; i <= kMaxSections; ++i) a_sec[i] = i <= S ? (int)((i * nsm + S - 1) / S) : (int)nsm;
    const int s32 = (int)s, e32 = (int)(s + Wb), Gx32 = (int)Gx, Gy32 = (int)Gy;
    for (long long ri = r_begin + tid * per; ri < r_end && ri < r_begin + (tid + 1) * per; ++ri) {
      const long long z = z0 + ri / ny, y = y0 + ri % ny;
      const long long R0 = F.align + ((F.pitch[1] * y + F.pitch[2] * z) << le);
      my_ops += (unsigned long long)(F.g_end - F.g_begin);
      int nc = 0;
      for (int g = F.g_begin; g < F.g_end; ++g) {
        const DGroup gr = K.g[g];
        const int yy = (int)y - gr.oy, zz = (int)z - gr.oz;
        if (yy < lo1 || yy >= hi1 || zz < lo2 || zz >= hi2) continue;
        const int r = fdiv32(yy - lo1, P.fd_BF[1]) + Gy32 * fdiv32(zz - lo2, P.fd_BF[2]);
        const int rx = r * Gx32;
        const int b0 = rx > s32 ? rx : s32, b1 = rx + Gx32 < e32 ? rx + Gx32 : e32;
        if (b0 >= b1) continue;
        c_b0[nc] = b0;
        c_b1[nc] = b1;
        c_rx[nc] = rx;
        c_g[nc] = g;
        ++nc;
      }
      if (nc == 0) continue;
      // intervals of (section sel or -1 = any, kind mask km: 1 = loads, 3 = loads + stores)
      auto pieces = [&](auto&& cb) {  // cb(section, kind, xs, xe)
        for (int q = 0; q < nc; ++q) {
          const DGroup gr = K.g[c_g[q]];
          int b0 = c_b0[q];
          const int b1 = c_b1[q], rx = c_rx[q];
          while (b0 < b1) {  // pieces of blocks on the SMs of one section
            const int x = b0 - s32;
            const int j = x - (int)nsm32 * fdiv32(x, fd_nsm);
            int sec = 0;
#pragma unroll
            for (int i = 1; i < kMaxSections; ++i) sec += (i < (int)S32 && a_sec[i] <= j) ? 1 : 0;
            const int jend = a_sec[sec + 1];
            int e = b0 + (jend - j);
            if (e > b1) e = b1;
            const int xs = lo0 + (b0 - rx) * BF0;
            int xe = lo0 + (e - rx) * BF0;
            if (xe > hi0) xe = hi0;
            if (xs < xe) cb((int)sec, gr.kind, xs + F.run_lo[gr.run], xe + F.run_hi[gr.run]);
            b0 = e;
          }
        }
      };
      auto gen_for = [&](int sel, int km) {
        return [&, sel, km](auto&& cb) {
          pieces([&](int sec, int kind, int xs, int xe) {
            if (((km >> kind) & 1) && (sel < 0 || sel == sec)) cb((long long)xs, (long long)xe);
          });
        };
      };
      // one scan: per target (section loads, section all, union loads, union all) the extreme
      // starts / ends; a target whose max start <= min end is one interval (the common case)
      constexpr int NT = 2 * kMaxSections + 2;
      int mns[NT], mxs[NT], mne[NT], mxe[NT];
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        mns[q] = mne[q] = 0x7fffffff;
        mxs[q] = mxe[q] = -0x7fffffff;
      }
      pieces([&](int sec, int kind, int xs, int xe) {
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          const bool hit = q < 2 * kMaxSections ? ((q >> 1) == sec && ((q & 1) || kind == 0))
                                                : ((q & 1) || kind == 0);
          if (hit) {
            mns[q] = min(mns[q], xs);
            mxs[q] = max(mxs[q], xs);
            mne[q] = min(mne[q], xe);
            mxe[q] = max(mxe[q], xe);
          }
        }
      });
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const bool need = q == NT - 1 || (P.want_sect && (q >= 2 * kMaxSections || (q >> 1) < S));
        if (!need || mns[q] == 0x7fffffff) continue;
        Tri* ts = (q & 1) ? nullptr : &t[q];
        Tri* tl = (q & 1) ? &t[q] : nullptr;
        Tri* tp = (q == NT - 1 && P.want_pages) ? &t[2 * kMaxSections + 2] : nullptr;
        if (mxs[q] <= mne[q]) {
          const long long a0 = R0 + ((long long)mns[q] << le), a1 = R0 + ((long long)(mxe[q] - 1) << le);
          if (ts) tri_add(*ts, a0 >> ls, a1 >> ls);
          if (tl) tri_add(*tl, a0 >> ll, a1 >> ll);
          if (tp) tri_add(*tp, a0 >> lp, a1 >> lp);
        } else {
          row_union_p(gen_for(q < 2 * kMaxSections ? (q >> 1) : -1, (q & 1) ? 3 : 1), R0, le, ls, ll, lp, ts, tl, tp);
        }
      }
    }
    cta_ordered_reduce<kSectNQ>(t, s_red);
    // publish this segment; the last segment of the item folds all of them in row order
    const long long pslot = ((long long)c * max_fields + fi) * kSectSeg;
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < kSectNQ; ++q) {
        WS_CHK((pslot + seg) * kSectNQ + q, g_caps.spart);
        spart[(pslot + seg) * kSectNQ + q] = t[q];
      }
      __threadfence();
      s_last = atomicAdd(sdone + (long long)c * max_fields + fi, 1u) == (unsigned)(kSectSeg - 1);
    }
    __syncthreads();
    const bool last = s_last;
    __syncthreads();
    if (tid == 0 && last) {
      __threadfence();
#pragma unroll
      for (int q = 0; q < kSectNQ; ++q) {
        Tri a = tri_empty();
        for (int k = 0; k < kSectSeg; ++k) {
          const long long* src = reinterpret_cast<const long long*>(spart + (pslot + k) * kSectNQ + q);
          a = tri_combine(a, Tri{__ldcg(src), __ldcg(src + 1), __ldcg(src + 2)});
        }
        t[q] = a;
      }
    }
    if (tid == 0 && last && nrows > 0) {
      unsigned long long* a = acc + (long long)c * A_N;
      long long sld = 0, slin = 0;
      for (int i = 0; i < kMaxSections; ++i) {
        sld += t[2 * i].c;
        slin += t[2 * i + 1].c;
      }
      atomicAdd(a + A_SECLD, (unsigned long long)sld);
      atomicAdd(a + A_SECLIN, (unsigned long long)slin);
      atomicAdd(a + A_ULD, (unsigned long long)t[2 * kMaxSections].c);
      atomicAdd(a + A_ULIN, (unsigned long long)t[2 * kMaxSections + 1].c);
      atomicAdd(a + A_PAGES, (unsigned long long)t[2 * kMaxSections + 2].c);
    }
  }
  if (my_ops) atomicAdd(work + K_SECT, my_ops);
}

// ------------------------------------------------------------------ a7: model (FP64)
__device__ __forceinline__ double gompertz(const double* abc, double O) { return abc[0] * exp(-abc[1] * exp(-abc[2] * O)); }

__device__ __noinline__ void model_one(const DPlan& P, const DKernel* __restrict__ ks, const DGpu& G,
                                       const unsigned long long* a, ws_result& R) {
  memset(&R, 0, sizeof(R));
  R.status = P.status != WS_OK ? P.status : P.istat;   // istat: k_instr's instruction-table limit
  if (R.status != WS_OK) return;
  const DKernel& K = ks[P.kid];
  for (int d = 0; d < 3; ++d) R.grid[d] = (uint32_t)P.G[d];
  R.k = (uint32_t)P.k;
  R.wave_blocks = (uint32_t)P.W;
  R.n_smsets = (uint32_t)P.nsets;
  R.n_instr = (uint32_t)P.n_instr;
  R.wave_first_block = (uint64_t)P.s;
  R.lup_wave = a[A_LUP];
  R.l1_wavefronts = a[A_WF];
  R.l1_req_ld_sectors = a[A_REQ_LD];
  R.l1_req_st_sectors = a[A_REQ_ST];
  R.sm_ld_sectors = a[A_SM_SEC];
  R.sm_ld_lines = a[A_SM_LIN];
  R.wave_ld_sectors = a[A_WLD];
  R.wave_st_sectors = a[A_WST];
  R.wave_lines = a[A_WLIN];
  R.ly_lines = a[A_LY];
  R.lz_lines = a[A_LZ];
  R.ov_y = a[A_OVY];
  R.ov_z = a[A_OVZ];
  R.addr_evals = P.addr_evals;
  const double sector = (double)G.g.sector_bytes, line = (double)G.g.line_bytes;
  const double lup = (double)R.lup_wave;
  // L1: capacity on the mean SM-set allocation (Eq. 4) and Eq. 5 on the redundant loads
  R.O_l1 = ((double)R.sm_ld_lines * line / (double)P.nsets) / (double)G.g.l1_bytes;
  R.R_l1 = gompertz(G.g.hit_abc[0], R.O_l1);
  const double red1 = (double)R.l1_req_ld_sectors > (double)R.sm_ld_sectors
                          ? (double)R.l1_req_ld_sectors - (double)R.sm_ld_sectors : 0.0;
  const double v_l2l1_ld = (double)R.sm_ld_sectors + (1.0 - R.R_l1) * red1;
  const double v_l1l2_st = (double)R.l1_req_st_sectors;
  // L2: split-L2 effective capacity; layer-set overlaps (Q13-Q16)
  // NEXT-4 outlook metrics (k_sect, linear address space)
  R.wave_pages = a[A_PAGES];
  R.l2_dup_lines = P.want_sect ? a[A_SECLIN] - a[A_ULIN] : 0ull;
  R.l2_link_sectors = P.want_sect ? a[A_SECLD] - a[A_ULD] : 0ull;
  double l2_eff = (double)G.g.l2_bytes / (double)G.g.l2_sections;
  // WS_VAR_L2_DUP: the capacity holds U + dup line copies for U distinct lines
  if ((P.variant & WS_VAR_L2_DUP) && P.want_sect && a[A_ULIN] > 0)
    l2_eff = (double)G.g.l2_bytes * (double)a[A_ULIN] / (double)(a[A_ULIN] + R.l2_dup_lines);
  R.l2_eff_bytes = l2_eff;
  R.O_y = (double)R.ly_lines * line / l2_eff;
  R.O_z = (double)R.lz_lines * line / l2_eff;
  R.R_y = gompertz(G.g.hit_abc[1], R.O_y);
  R.R_z = gompertz(G.g.hit_abc[2], R.O_z);
  const double hit = R.R_y * (double)R.ov_y + R.R_z * (double)(R.ov_z - R.ov_y);
  const double red_st = (double)R.l1_req_st_sectors > (double)R.wave_st_sectors
                            ? (double)R.l1_req_st_sectors - (double)R.wave_st_sectors : 0.0;
  R.O_st = (double)R.wave_lines * line / l2_eff;
  R.R_st = gompertz(G.g.hit_abc[3], R.O_st);
  const double v_dram_ld = (double)R.wave_ld_sectors - hit + (1.0 - R.R_st) * red_st;
  const double v_dram_st = (double)R.wave_st_sectors;
  R.l1_cyc_per_lup = (double)R.l1_wavefronts / lup;
  R.l2_ld_Bpl = sector * v_l2l1_ld / lup;
  R.l2_st_Bpl = sector * v_l1l2_st / lup;
  R.dram_ld_Bpl = sector * v_dram_ld / lup;
  R.dram_st_Bpl = sector * v_dram_st / lup;
  R.t_l1 = (double)R.l1_wavefronts / (lup * (double)G.g.n_sm * G.g.clock_hz);
  R.t_l2 = sector * (v_l2l1_ld + v_l1l2_st) / (lup * G.g.l2_bw);
  R.t_dram = sector * (v_dram_ld + v_dram_st) / (lup * G.g.dram_bw);
  // the inter-section link as an additional L2 limiter
  R.t_link = G.g.link_bw > 0 ? sector * (double)R.l2_link_sectors / (lup * G.g.link_bw) : 0.0;
  const double tm = fmax(fmax(R.t_l1, R.t_link), fmax(R.t_l2, R.t_dram));
  R.limiter = R.t_dram >= tm ? 2u : (R.t_l2 >= tm ? 1u : (R.t_link >= tm ? 3u : 0u));
  R.t_pred = tm * K.cells;
}

// a5/a6 sharing: a configuration whose row scope another one computed (DPlan::row_owner) takes
// the owner's wave / layer-set counts (the plan is already in shared memory; lanes A_WLD..A_OVZ)
__device__ __forceinline__ void shared_row_counts(const DPlan& P, long long c, const unsigned long long* __restrict__ acc,
                                                  unsigned long long* a, int lane) {
  if (P.status == WS_OK && P.row_owner != c && lane >= A_WLD && lane <= A_OVZ)
    a[lane] = acc[(long long)P.row_owner * A_N + lane];
}

// a8 rank key: 64-bit order-preserving (IEEE bits with the sign folded; failed configurations = +inf)
__device__ __forceinline__ unsigned long long rank_key(const ws_result& r) {
  if (r.status != WS_OK) return 0xfff0000000000000ull;     // +inf after the fold below
  const unsigned long long b = (unsigned long long)__double_as_longlong(r.t_pred);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// one warp per configuration: the accumulators in by the lanes, the model by lane 0, the
// 336-byte record out by the lanes (coalesced).  With rank_ctr (ws_estimate_ranked_async, n <=
// kTailMax) the last CTA to finish (threadfence + counter, lists[7], zeroed by k_plan's scan)
// also ranks the batch: keys of every record, bitonic sort of (key, index) in shared memory (the
// k_rank_smem network), ranks and top-k -- no separate rank launch.
__global__ void __launch_bounds__(128) k_model(const DPlan* __restrict__ plans, int n, const DKernel* __restrict__ ks,
                                               const DGpu* __restrict__ gs, const unsigned long long* __restrict__ acc,
                                               ws_result* __restrict__ out, int rank_k, uint32_t* __restrict__ top,
                                               unsigned long long* __restrict__ rank_ctr) {
  static_assert(sizeof(ws_result) % 8 == 0 && A_N <= 32, "record copy / accumulator lanes");
  PDL_PROLOGUE();   // (WS_MODELPDL: k_fold's programmatic dependent; a no-op otherwise)
  __shared__ unsigned long long s_a[4][A_N];
  __shared__ ws_result s_r[4];
  __shared__ __align__(16) DPlan s_p[4];  // plan and GPU descriptor staged by the lanes (one load round)
  __shared__ __align__(16) DGpu s_gp[4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 4 + w;
  if (c < n) {
    if (lane < A_N) s_a[w][lane] = acc[(long long)c * A_N + lane];
    {
      const uint4* sp = reinterpret_cast<const uint4*>(plans + c);
      uint4* dp = reinterpret_cast<uint4*>(&s_p[w]);
      for (int i = lane; i < (int)(sizeof(DPlan) / 16); i += 32) dp[i] = sp[i];
    }
    __syncwarp();
    {
      const int gid = s_p[w].status == WS_OK ? s_p[w].gid : 0;
      const uint4* sg = reinterpret_cast<const uint4*>(gs + gid);
      uint4* dg = reinterpret_cast<uint4*>(&s_gp[w]);
      for (int i = lane; i < (int)(sizeof(DGpu) / 16); i += 32) dg[i] = sg[i];
    }
    shared_row_counts(s_p[w], c, acc, s_a[w], lane);
    __syncwarp();
    if (lane == 0) model_one(s_p[w], ks, s_gp[w], s_a[w], s_r[w]);
    __syncwarp();
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&s_r[w]);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(out + c);
    for (int i = lane; i < (int)(sizeof(ws_result) / 8); i += 32) dst[i] = src[i];
  }
  if (!rank_ctr) return;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(rank_ctr, 1ull) == (unsigned long long)(gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ unsigned long long key[kTailMax];
  __shared__ uint32_t idx[kTailMax];
  int P = 32;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < n) {
      const ws_result* r = out + i;   // other CTAs' records: through L2
      ws_result t;
      t.status = __ldcg(&r->status);
      t.t_pred = __ldcg(&r->t_pred);
      key[i] = rank_key(t);
    } else {
      key[i] = ~0ull;
    }
    idx[i] = (uint32_t)i;
  }
  __syncthreads();
  if (n <= 256) {
    // small batch: each record's rank is the number of (key, index) pairs below its own -- one
    // pass over the keys per thread, no sorting network (36 barrier-separated stages at n = 168)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long ki = key[i];
      int r = 0;
      for (int j = 0; j < n; ++j) {
        const unsigned long long kj = key[j];
        r += (kj < ki || (kj == ki && j < i)) ? 1 : 0;
      }
      out[i].rank = (uint32_t)r;
      if (r < rank_k && top) top[r] = (uint32_t)i;
    }
    return;
  }
  const int half = P >> 1;
  for (int kk = 2; kk <= P; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < half; t += blockDim.x) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), l = i + j;
        const unsigned long long ki = key[i], kl = key[l];
        const uint32_t ii = idx[i], il = idx[l];
        const bool gt = ki > kl || (ki == kl && ii > il);
        if (gt == ((i & kk) == 0)) {
          key[i] = kl;
          key[l] = ki;
          idx[i] = il;
          idx[l] = ii;
        }
      }
      __syncthreads();
    }
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const uint32_t cc = idx[p];
    out[cc].rank = (uint32_t)p;
    if (p < rank_k && top) top[p] = cc;
  }
}

// BJ configs[3] architecture exploration (ws_estimate_multi): the integer stages ran once per
// group of hardware sets that agree in every parameter they read; the FP64 model fans out over
// the group's sets.  Expanded batch: xcfg[j * m + t] = cfgs[i0 + t] with the group's
// representative gpu id; output out[g * n + i0 + t] from the plan / accumulators of entry
// group[g] * m + t and the descriptor of gid[g].
__global__ void __launch_bounds__(256) k_expand(const ws_config* __restrict__ cfgs, FanOut f,
                                                ws_config* __restrict__ xcfg) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= (long long)f.m * f.n_groups) return;
  const int grp = (int)(j / f.m), t = (int)(j % f.m);
  ws_config c = cfgs[f.i0 + t];
  c.gpu_id = f.rep[grp];
  xcfg[j] = c;
}

__global__ void __launch_bounds__(128) k_model_fan(const DPlan* __restrict__ plans, const DKernel* __restrict__ ks,
                                                   const DGpu* __restrict__ gs, const unsigned long long* __restrict__ acc,
                                                   FanOut f, ws_result* __restrict__ out) {
  __shared__ unsigned long long s_a[4][A_N];
  __shared__ ws_result s_r[4];
  __shared__ __align__(16) DPlan s_p[4];
  __shared__ __align__(16) DGpu s_gp[4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long o = (long long)blockIdx.x * 4 + w;   // output entry (g, t)
  if (o >= (long long)f.m * f.n_gpu) return;
  const int g = (int)(o / f.m), t = (int)(o % f.m);
  const long long c = (long long)f.group[g] * f.m + t;  // integer entry
  if (lane < A_N) s_a[w][lane] = acc[c * A_N + lane];
  {
    const uint4* sp = reinterpret_cast<const uint4*>(plans + c);
    uint4* dp = reinterpret_cast<uint4*>(&s_p[w]);
    for (int i = lane; i < (int)(sizeof(DPlan) / 16); i += 32) dp[i] = sp[i];
    const uint4* sg = reinterpret_cast<const uint4*>(gs + f.gid[g]);
    uint4* dg = reinterpret_cast<uint4*>(&s_gp[w]);
    for (int i = lane; i < (int)(sizeof(DGpu) / 16); i += 32) dg[i] = sg[i];
  }
  __syncwarp();
  shared_row_counts(s_p[w], c, acc, s_a[w], lane);
  __syncwarp();
  if (lane == 0) model_one(s_p[w], ks, s_gp[w], s_a[w], s_r[w]);
  __syncwarp();
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&s_r[w]);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(out + (long long)g * f.n + f.i0 + t);
  for (int i = lane; i < (int)(sizeof(ws_result) / 8); i += 32) dst[i] = src[i];
}

int launch_expand(const ws_config* d_cfgs, const FanOut& f, ws_config* xcfg, cudaStream_t st) {
  const long long m = (long long)f.m * f.n_groups;
  k_expand<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(d_cfgs, f, xcfg);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ a8: rank
// Rank by (t_pred ascending, index ascending), failed configurations last:
// a sort of 64-bit order-preserving keys (IEEE bits with the sign folded; failed = +inf) carrying
// the configuration index; (key, index) pairs are unique, so every comparison is strict.
//   n <= kRankSmem: one CTA, bitonic sort in shared memory, ranks written directly;
//   n <= kRankMerge: tiles of 2048 (n <= 2^15) or 4096 sorted the same way by one CTA each, then every element's
//     rank = its position in its tile + the number of smaller pairs in every other tile (binary
//     searches of the sorted tiles);
//   larger n: a stable LSD radix sort, 8 passes of 8 bits (tile histogram -> one-CTA scan -> stable
//     tile scatter), whose stability over the index-ordered input gives the index tie-break.
constexpr int kRankSmem = 2048;    // one CTA (1024 threads, one pair per thread per stage)
constexpr int kRankTile = 4096;    // tile of the merge path (2048 below kRankSmall)
constexpr int kRankSmall = 1 << 15;
constexpr int kRankMerge = 1 << 18;
constexpr int kRkTile = 2048;
// CTA b sorts the P-element tile [b*P, b*P+P) of the records (padding: key ~0, sorts last); with
// skey == nullptr (a single tile) it writes ranks and top-k, else the sorted tile to skey / sidx.
__global__ void __launch_bounds__(1024) k_rank_smem(ws_result* __restrict__ res, int n, int P, int k,
                                                    uint32_t* __restrict__ top, unsigned long long* __restrict__ skey,
                                                    uint32_t* __restrict__ sidx) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(s_raw);
  uint32_t* idx = reinterpret_cast<uint32_t*>(s_raw + (size_t)P * 8);
  const int base = blockIdx.x * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const int g = base + i;
    key[i] = g < n ? rank_key(res[g]) : ~0ull;
    idx[i] = (uint32_t)g;
  }
  __syncthreads();
  const int half = P >> 1;
  for (int kk = 2; kk <= P; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < half; t += blockDim.x) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), l = i + j;
        const unsigned long long ki = key[i], kl = key[l];
        const uint32_t ii = idx[i], il = idx[l];
        const bool gt = ki > kl || (ki == kl && ii > il);
        if (gt == ((i & kk) == 0)) {
          key[i] = kl;
          key[l] = ki;
          idx[i] = il;
          idx[l] = ii;
        }
      }
      __syncthreads();
    }
  if (!skey) {
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const uint32_t c = idx[p];
      res[c].rank = (uint32_t)p;
      if (p < k && top) top[p] = c;
    }
    return;
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    skey[base + i] = key[i];
    sidx[base + i] = idx[i];
  }
}
// global rank of every element from the sorted tiles (one thread per sorted position)
__global__ void __launch_bounds__(256) k_rank_merge(ws_result* __restrict__ res, int n, int P, int ntiles, int k,
                                                    uint32_t* __restrict__ top, const unsigned long long* __restrict__ skey,
                                                    const uint32_t* __restrict__ sidx) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ntiles * P) return;
  const uint32_t c = sidx[q];
  if ((int)c >= n) return;                         // padding
  const unsigned long long x = skey[q];
  const int my = q / P;
  long long r = q - (long long)my * P;             // smaller pairs in its own tile
  // branchless lower bounds of the key alone (P a power of two) in 8 other tiles at once: each
  // halving step issues 8 independent loads, so the latency chain is log2(P) steps per group of
  // tiles.  Pairs of another tile smaller than (x, c): keys < x, plus keys == x with index < c
  // (rare: a walk over the equal keys, which the tile holds in index order).
  constexpr int kG = 8;
  for (int t0 = 0; t0 < ntiles; t0 += kG) {
    int pos[kG];
#pragma unroll
    for (int u = 0; u < kG; ++u) pos[u] = 0;
    for (int step = P >> 1; step > 0; step >>= 1) {
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        const int t = t0 + u;
        if (t < ntiles && t != my && skey[(long long)t * P + pos[u] + step - 1] < x) pos[u] += step;
      }
    }
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      const int t = t0 + u;
      if (t < ntiles && t != my) {   // pos = #keys < x among the first P - 1
        const unsigned long long* K = skey + (long long)t * P;
        int p = pos[u];
        if (p == P - 1 && K[p] < x) ++p;
        while (p < P && K[p] == x && sidx[(long long)t * P + p] < c) ++p;
        r += p;
      }
    }
  }
  res[c].rank = (uint32_t)r;
  if (r < k && top) top[r] = c;
}
__global__ void __launch_bounds__(256) k_rank_keys(const ws_result* __restrict__ res, int n,
                                                   unsigned long long* __restrict__ key, uint32_t* __restrict__ val) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    key[i] = rank_key(res[i]);
    val[i] = (uint32_t)i;
  }
}
__global__ void __launch_bounds__(256) k_rank_hist(const unsigned long long* __restrict__ key, int n, int shift,
                                                   uint32_t* __restrict__ hist, int ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int t0 = blockIdx.x * kRkTile;
  for (int r = 0; r < kRkTile / 256; ++r) {
    const int i = t0 + r * 256 + threadIdx.x;
    if (i < n) atomicAdd(&h[(unsigned)(key[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];   // digit-major
}
// one CTA: exclusive scan of m counts in place (each thread a contiguous segment)
__global__ void __launch_bounds__(1024) k_rank_scan(uint32_t* __restrict__ v, int m) {
  __shared__ uint32_t s_w[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int seg = (m + 1023) / 1024, a = tid * seg, b = min(m, a + seg);
  uint32_t sum = 0;
  for (int i = a; i < b; ++i) sum += v[i];
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = s_w[lane], z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, z, o);
      if (lane >= o) z += y;
    }
    s_w[lane] = z - w;
  }
  __syncthreads();
  uint32_t run = s_w[wid] + x - sum;
  for (int i = a; i < b; ++i) {
    const uint32_t t = v[i];
    v[i] = run;
    run += t;
  }
}
__global__ void __launch_bounds__(256) k_rank_scatter(const unsigned long long* __restrict__ key,
                                                      const uint32_t* __restrict__ val, int n, int shift,
                                                      const uint32_t* __restrict__ off, int ntiles,
                                                      unsigned long long* __restrict__ key2, uint32_t* __restrict__ val2) {
  __shared__ uint32_t run[256];
  __shared__ uint32_t wc[8][256];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  run[tid] = off[tid * ntiles + blockIdx.x];
  const int t0 = blockIdx.x * kRkTile;
  for (int r = 0; r < kRkTile / 256; ++r) {
#pragma unroll
    for (int w = 0; w < 8; ++w) wc[w][tid] = 0u;
    __syncthreads();
    const int i = t0 + r * 256 + tid;
    const bool ok = i < n;
    const unsigned long long kk = ok ? key[i] : 0ull;
    const uint32_t v = ok ? val[i] : 0u;
    const uint32_t d = (unsigned)(kk >> shift) & 255u;
    const unsigned peers = __match_any_sync(FULL, ok ? d : 0x100u + (unsigned)lane);
    const int rk = __popc(peers & ((1u << lane) - 1u));
    if (ok && rk == 0) wc[wid][d] = (uint32_t)__popc(peers);
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < wid; ++w) before += wc[w][d];
    if (ok) {
      const uint32_t pos = run[d] + before + (uint32_t)rk;
      key2[pos] = kk;
      val2[pos] = v;
    }
    __syncthreads();
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += wc[w][tid];
    run[tid] += tot;
    __syncthreads();
  }
}
__global__ void __launch_bounds__(256) k_rank_out(ws_result* __restrict__ res, const uint32_t* __restrict__ val, int n,
                                                  int k, uint32_t* __restrict__ top) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) {
    const uint32_t c = val[p];
    res[c].rank = (uint32_t)p;
    if (p < k && top) top[p] = c;
  }
}

size_t rank_scratch_bytes(int n) {
  if (n <= kRankSmem) return 0;
  if (n <= kRankMerge) return ((size_t)n + kRankTile) * 12 + 1024;
  const size_t nt = (size_t)(n + kRkTile - 1) / kRkTile;
  return 2 * (size_t)n * 8 + 2 * (size_t)n * 4 + 256 * nt * 4 + 1024;
}

// ------------------------------------------------------------------ launchers
static int check_launch() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

// launch `kern` on `q`, as a programmatic dependent of the stream's previous kernel when `pdl`
template <typename... P, typename... A>
static void launch_k(bool pdl, void (*kern)(P...), dim3 grid, dim3 block, cudaStream_t q, A... args) {
  if (!pdl) {
    kern<<<grid, block, 0, q>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = q;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

int launch_estimate(const ws_config* d_cfgs, int n, const DKernel* d_k, int nk, const DGpu* d_g, int ng,
                    const Scratch& s, ws_result* d_out, const Streams& st, int n_sm_dev, uint32_t* launches,
                    cudaEvent_t* ev, const FanOut* fan, TailRank* tail) {
  // programmatic dependent launches along each chain (not while per-kernel events are recorded
  // between the kernels; WS_PDL=0 disables, A/B)
  static const bool pdl_env = !(getenv("WS_PDL") && getenv("WS_PDL")[0] == '0');
  const bool pdl = pdl_env && !ev;
  uint32_t L = 0;
  auto beg = [&](int kind, cudaStream_t q) {
    if (ev) cudaEventRecord(ev[2 * kind], q);
  };
  auto end = [&](int kind, cudaStream_t q) {
    if (ev) cudaEventRecord(ev[2 * kind + 1], q);
    ++L;
  };
#ifndef WS_PERSIST
#define WS_PERSIST 8
#endif
#ifndef WS_PERSIST_ROWS
#define WS_PERSIST_ROWS 8
#endif
#ifndef WS_PERSIST_SCLASS
#define WS_PERSIST_SCLASS 16  // A/B: 0.182 vs 0.184 ms (dynamic item fetch; more CTAs fill the SMs sooner)
#endif
  // CTAs per SM of each chain's grid: build defaults, WS_GRID_<NAME> overrides at run time (A/B)
  auto knob = [](const char* name, int def) {
    const char* v = getenv(name);
    return v && atoi(v) > 0 ? atoi(v) : def;
  };
  static const int g_warp = knob("WS_GRID_WARP", WS_PERSIST), g_rows = knob("WS_GRID_ROWS", WS_PERSIST_ROWS),
                   g_sclass = knob("WS_GRID_SCLASS", WS_PERSIST_SCLASS), g_smset = knob("WS_GRID_SMSET", 8),
                   g_cplan = knob("WS_GRID_CPLAN", 4), g_cplanes = knob("WS_GRID_CPLANES", 8),
                   g_fold = knob("WS_GRID_FOLD", 4), g_cfold = knob("WS_GRID_CFOLD", 2);
  const int persist = n_sm_dev * g_warp;
  cudaStream_t m = st.main, a = st.aux[0], b = st.aux[1];
#ifdef WS_CHECK
  {  // capacities of this call's scratch layout (the check build never captures graphs)
    static CheckCaps hc;
    hc = CheckCaps{(long long)s.max_chunks, (long long)s.clist_stride, (long long)n * kWSlots, (long long)n * kSSlots,
                   (long long)s.cdesc_cap, (long long)s.cpool_cap, (long long)n * s.max_fields * kSectSeg * kSectNQ,
                   (long long)n * kMaxFields, (long long)n * kMaxInstr, (long long)n * s.max_fields};
    cudaMemcpyToSymbolAsync(g_caps, &hc, sizeof(hc), 0, cudaMemcpyHostToDevice, m);
    cudaStreamSynchronize(m);
  }
#endif
  beg(K_PLAN, m);
  k_plan<<<n, WS_PLAN_THREADS, 0, m>>>(d_cfgs, n, d_k, nk, d_g, ng, s.plans, s.instr, s.rowinfo, s.acc, s.wcnt, s.scnt,
                           s.rctr, s.ritems, s.fitems, s.work, s.lists, s.skey, s.sdone, s.max_fields, s.epoch,
                           s.rowtab, s.clist, s.clist_stride);
  end(K_PLAN, m);
  // fork: SM-set chain on aux[0], row chain on aux[1], warp chain on the main stream.  WS_ROWMAIN=1
  // swaps the row and warp chains so that k_rows is k_plan's programmatic dependent (its CTAs
  // launch while k_plan runs): A/B on B200, configs[1] 0.125 vs 0.123 ms -- the early k_rows CTAs
  // hold SM slots the other chains' first kernels need -- so off by default
  static const bool rowmain = getenv("WS_ROWMAIN") && getenv("WS_ROWMAIN")[0] == '1';
  cudaEventRecord(st.fork, m);
  cudaStreamWaitEvent(a, st.fork, 0);
  cudaStreamWaitEvent(b, st.fork, 0);
  {
    const cudaStream_t r = rowmain ? m : b;
    b = rowmain ? b : m;   // the warp chain's stream from here on
    m = r;                 // ... and the row chain's (joins on the caller's stream below)
  }
  beg(K_ROWS, m);
  launch_k(pdl && rowmain, k_rows, n_sm_dev * g_rows, kRowWarps * 32, m, (const DPlan*)s.plans, d_k, d_g,
           (const DRowInfo*)s.rowinfo, s.chunkres, s.work, (const unsigned long long*)s.rctr,
           (const unsigned long long*)s.ritems);
  end(K_ROWS, m);
#ifdef WS_ROWS_TRACE
  k_rowtrace_dump<<<1, 1, 0, m>>>(s.rctr);
#endif
  beg(K_FOLD, m);
  static const int fold_mode = getenv("WS_FOLD_MODE") ? atoi(getenv("WS_FOLD_MODE")) : 0;  // diagnostics
  launch_k(pdl, k_fold, n_sm_dev * g_fold, 256, m, (const DPlan*)s.plans, (const unsigned long long*)s.rctr,
           (const uint32_t*)s.fitems, d_k, d_g, (const DRowInfo*)s.rowinfo, (const long long*)s.chunkres, s.acc,
           (int)fold_mode);
  end(K_FOLD, m);
  beg(K_SMSET, a);
  // the work-count prefix for the SM-set and warp chains (the row chain does not need it)
  k_scan<<<1, 256, 0, a>>>(s.plans, n, s.prefix, s.epoch);
  ++L;
  cudaEventRecord(st.scanned, a);
  k_spairs<<<n_sm_dev * 4, kSmsetThreads, 0, a>>>(s.plans, s.prefix, n, d_k, d_g, s.scnt, s.srep, s.lists, s.slist,
                                                  s.dlist, s.skey, s.dmask, s.gkey);
  launch_k(pdl, k_smset, n_sm_dev * g_smset, kSmsetThreads, a, (const DPlan*)s.plans, (const DPrefix*)s.prefix, n, d_k, d_g,
           s.scnt, s.srep, s.lists, s.slist, s.dlist, s.skey, s.dmask, (const unsigned long long*)s.gkey);
  ++L;
  end(K_SMSET, a);
  beg(K_SCLASS, a);
  static const bool cplanes = !(getenv("WS_CPLANES") && getenv("WS_CPLANES")[0] == '0');  // A/B, diagnostics
  if (cplanes) {  // single-block classes by computed planes
    CDesc* cd = (CDesc*)s.cdesc;
    Tri* cp = (Tri*)s.cpool;
    unsigned long long* cctr = s.lists + 4;  // descriptors, pool planes, items (zeroed with the lists)
    launch_k(pdl, k_cplan, n_sm_dev * g_cplan, 256, a, (const DPlan*)s.plans, d_k, d_g, (const unsigned long long*)s.lists,
             (const unsigned long long*)s.slist, (const unsigned long long*)s.srep, s.sval, s.cfbl, cd, cp, s.citems,
             cctr, (long long)s.cdesc_cap, (long long)s.cpool_cap);
    launch_k(pdl, k_cplanes, n_sm_dev * g_cplanes, 256, a, (const DPlan*)s.plans, d_k, d_g, (const CDesc*)cd, cp,
             (const uint32_t*)s.citems, (const unsigned long long*)cctr, s.work);
    launch_k(pdl, k_cfold, n_sm_dev * g_cfold, 256, a, (const DPlan*)s.plans, d_k, d_g, (const unsigned long long*)s.slist,
             (const unsigned int*)s.scnt, (const CDesc*)cd, (const Tri*)cp, (const unsigned long long*)cctr, s.acc,
             s.sval);
    L += 3;
  }
  launch_k(pdl, k_sclass, n_sm_dev * g_sclass, WS_SCLASS_THREADS, a, (const DPlan*)s.plans, d_k, d_g, s.acc,
           (const unsigned int*)s.scnt, (const unsigned long long*)s.srep, s.lists, (const unsigned long long*)s.slist,
           (const unsigned long long*)s.dlist, s.work, s.sval, (const unsigned int*)s.dmask,
           (const uint32_t*)(cplanes ? s.cfbl : nullptr), (const unsigned long long*)(s.lists + 4),
           (const unsigned long long*)s.rctr);
  launch_k(pdl, k_sshare, n_sm_dev, 256, a, (const unsigned long long*)s.lists, (const unsigned long long*)s.slist,
           (const unsigned int*)s.scnt, (const unsigned long long*)s.sval, s.acc);
#ifdef WS_SCLASS_TRACE
  k_sctrace_dump<<<1, 1, 0, a>>>(s.lists, s.plans);
#endif
  ++L;
  end(K_SCLASS, a);
  beg(K_INSTR, b);
  k_instr<<<n, 128, 0, b>>>(d_k, s.plans, s.instr, s.wcnt, n);
  end(K_INSTR, b);
  cudaStreamWaitEvent(b, st.scanned, 0);
  beg(K_WARP, b);
  launch_k(pdl, k_warp, persist, 256, b, (const DPlan*)s.plans, (const DPrefix*)s.prefix, n, (const DInstr*)s.instr, d_k,
           d_g, s.acc, s.wcnt, s.wrep, s.lists, s.wlist, s.work);
  end(K_WARP, b);
  beg(K_WCLASS, b);
  launch_k(pdl, k_wclass, persist, 256, b, (const DPlan*)s.plans, (const DInstr*)s.instr, d_k, d_g, s.acc,
           s.wcnt, (const unsigned long long*)s.wrep, s.lists, (const unsigned long long*)s.wlist,
           s.work);
  end(K_WCLASS, b);
  beg(K_SECT, b);
  launch_k(pdl, k_sect, n_sm_dev * WS_SECT_CTAS, 256, b, (const DPlan*)s.plans, (const DPrefix*)s.prefix, n, d_k, d_g,
           s.acc, s.work, (Tri*)s.spart, s.sdone, (int)s.max_fields);
  end(K_SECT, b);
  // join
  // WS_MODELPDL=1 (A/B): the model runs on the row chain's stream as k_fold's programmatic dependent
  // (after waiting for the other two chains), then the caller's stream joins it
  static const bool model_pdl = getenv("WS_MODELPDL") && getenv("WS_MODELPDL")[0] == '1';
  const bool mpdl = model_pdl && pdl && m != st.main && !fan;
  if (mpdl) {
    cudaEventRecord(st.join[0], a);
    cudaEventRecord(st.join[1], b);
    cudaStreamWaitEvent(m, st.join[0], 0);
    cudaStreamWaitEvent(m, st.join[1], 0);
  } else {  // join the other two chains into the caller's stream, which runs the model
    const cudaStream_t other = m == st.main ? b : m;
    m = st.main;
    cudaEventRecord(st.join[0], a);
    cudaEventRecord(st.join[1], other);
    cudaStreamWaitEvent(m, st.join[0], 0);
    cudaStreamWaitEvent(m, st.join[1], 0);
  }
  beg(K_MODEL, m);
  if (tail && !fan && n <= kTailMax) {   // ws_estimate_ranked_async: the model's last CTA ranks
    launch_k(mpdl, k_model, (n + 3) / 4, 128, m, (const DPlan*)s.plans, n, d_k, d_g, (const unsigned long long*)s.acc,
             d_out, tail->k, tail->top, s.lists + 7);
    tail->done = 1;
  } else if (mpdl) {
    launch_k(true, k_model, (n + 3) / 4, 128, m, (const DPlan*)s.plans, n, d_k, d_g, (const unsigned long long*)s.acc,
             d_out, 0, (uint32_t*)nullptr, (unsigned long long*)nullptr);
  } else if (fan)
    k_model_fan<<<(unsigned)(((long long)fan->m * fan->n_gpu + 3) / 4), 128, 0, m>>>(s.plans, d_k, d_g, s.acc, *fan,
                                                                                    d_out);
  else
    k_model<<<(n + 3) / 4, 128, 0, m>>>(s.plans, n, d_k, d_g, s.acc, d_out, 0, nullptr, nullptr);
  end(K_MODEL, m);
  if (mpdl) {   // the caller's stream waits for the model (on the row stream)
    cudaEventRecord(st.fork, m);
    cudaStreamWaitEvent(st.main, st.fork, 0);
  }
  if (launches) *launches = L;
  return check_launch();
}

int launch_rank(ws_result* d_res, int n, int k, uint32_t* d_top, void* scratch, cudaStream_t st, uint32_t* launches,
                cudaEvent_t* ev) {
  if (ev) cudaEventRecord(ev[0], st);
  uint32_t L = 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_rank_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kRankTile * 12);
    attr = true;
  }
  if (n <= kRankSmem) {
    int P = 32;
    while (P < n) P <<= 1;
    k_rank_smem<<<1, P / 2 < 1024 ? P / 2 : 1024, (size_t)P * 12, st>>>(d_res, n, P, k, d_top, nullptr, nullptr);
    L = 1;
  } else if (n <= kRankMerge) {
    const int P = n <= kRankSmall ? 2048 : kRankTile;
    const int nt = (n + P - 1) / P;
    unsigned long long* skey = (unsigned long long*)scratch;
    uint32_t* sidx = (uint32_t*)(skey + (size_t)nt * P);
    k_rank_smem<<<nt, 1024, (size_t)P * 12, st>>>(d_res, n, P, k, d_top, skey, sidx);
    k_rank_merge<<<(nt * P + 255) / 256, 256, 0, st>>>(d_res, n, P, nt, k, d_top, skey, sidx);
    L = 2;
  } else {
    const int nt = (n + kRkTile - 1) / kRkTile;
    char* b = (char*)scratch;
    unsigned long long* k0 = (unsigned long long*)b;
    unsigned long long* k1 = k0 + n;
    uint32_t* v0 = (uint32_t*)(k1 + n);
    uint32_t* v1 = v0 + n;
    uint32_t* hist = v1 + n;
    k_rank_keys<<<(n + 255) / 256, 256, 0, st>>>(d_res, n, k0, v0);
    ++L;
    for (int pass = 0; pass < 8; ++pass) {
      k_rank_hist<<<nt, 256, 0, st>>>(k0, n, 8 * pass, hist, nt);
      k_rank_scan<<<1, 1024, 0, st>>>(hist, 256 * nt);
      k_rank_scatter<<<nt, 256, 0, st>>>(k0, v0, n, 8 * pass, hist, nt, k1, v1);
      L += 3;
      std::swap(k0, k1);
      std::swap(v0, v1);
    }
    k_rank_out<<<(n + 255) / 256, 256, 0, st>>>(d_res, v0, n, k, d_top);
    ++L;
  }
  if (ev) cudaEventRecord(ev[1], st);
  if (launches) *launches = L;
  return check_launch();
}


// ================================================================== NEXT-1: simulated hit rates
// SURVEY 8(f) NEXT-1 (include/ws.h ws_simulate): the configuration's request streams replayed
// through a sectored, fully associative LRU cache, answered for every capacity at once from
// exact LRU stack distances (Mattson): a line access at q hits a cache of L lines iff the
// number of distinct other lines accessed since its previous access, dist(q), is < L; a
// sector access i is valid iff no access of its line in (previous access of the sector, i]
// missed, i.e. iff D_i = max of those dist(q) is < L (an eviction re-allocates the line with
// only the requested sector valid).  One warp per stream, 32 requests per step: dist from a
// Fenwick tree over "latest access of its line" markers (state before the step) corrected for
// the step's own earlier lanes; D from per-(line, sector) running maxima.
// simulated: estimate ok, linear address space, at most 32 sectors per line (valid bits)
__device__ __forceinline__ int sim_status(const DPlan& P, const DGpu* gs) {
  if (P.status != WS_OK) return P.status;
  if (P.istat != WS_OK) return P.istat;
  if (P.mdim) return WS_EINVAL;
  if (gs[P.gid].lg_line - gs[P.gid].lg_sector > 5) return WS_ELIMIT;
  return WS_OK;
}
__device__ __forceinline__ bool sim_ok(const DPlan& P, const DGpu* gs) { return sim_status(P, gs) == WS_OK; }

__device__ __forceinline__ long long sim_items_of(const DPlan& P, const DGpu* gs) {
  return sim_ok(P, gs) ? 2 * P.W + (P.s - P.Lz0) : 0;
}
__device__ __forceinline__ long long sim_traces_of(const DPlan& P, const DGpu* gs) { return sim_ok(P, gs) ? P.nsets + 2 : 0; }

// canonical instruction order (field, kind, offset C): one CTA per configuration, rank sort
__global__ void __launch_bounds__(256) k_sim_order(const DPlan* __restrict__ plans, const DGpu* __restrict__ gs,
                                                   const DInstr* __restrict__ instr, uint32_t* __restrict__ order, int n) {
  const int c = blockIdx.x;
  const DPlan& P = plans[c];
  if (!sim_ok(P, gs)) return;
  const DInstr* tab = instr + (long long)c * kMaxInstr;
  const int ni = P.n_instr;
  for (int i = threadIdx.x; i < ni; i += blockDim.x) {
    const DInstr e = tab[i];
    int rank = 0;
    for (int j = 0; j < ni; ++j) {
      const DInstr f = tab[j];
      rank += (f.field < e.field || (f.field == e.field && (f.kind < e.kind || (f.kind == e.kind && f.C < e.C)))) ? 1 : 0;
    }
    order[(long long)c * kMaxInstr + rank] = (uint32_t)i;
  }
}

// exclusive prefix (single CTA) of per-config block items and streams
__global__ void __launch_bounds__(1024) k_sim_cscan(const DPlan* __restrict__ plans, const DGpu* __restrict__ gs, int n,
                                                    int64_t* __restrict__ ipre, int64_t* __restrict__ tpre) {
  __shared__ long long s_a[1024], s_b[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int seg = (n + nt - 1) / nt;
  long long a = 0, b = 0;
  for (int c = tid * seg; c < n && c < (tid + 1) * seg; ++c) {
    a += sim_items_of(plans[c], gs);
    b += sim_traces_of(plans[c], gs);
  }
  s_a[tid] = a;
  s_b[tid] = b;
  __syncthreads();
  if (tid == 0) {
    long long ra = 0, rb = 0;
    for (int i = 0; i < nt; ++i) {
      const long long va = s_a[i], vb = s_b[i];
      s_a[i] = ra;
      s_b[i] = rb;
      ra += va;
      rb += vb;
    }
    ipre[n] = ra;
    tpre[n] = rb;
  }
  __syncthreads();
  a = s_a[tid];
  b = s_b[tid];
  for (int c = tid * seg; c < n && c < (tid + 1) * seg; ++c) {
    ipre[c] = a;
    tpre[c] = b;
    a += sim_items_of(plans[c], gs);
    b += sim_traces_of(plans[c], gs);
  }
}

// exclusive prefix (single CTA) of v[0..m) in place; v[m] = total
__global__ void __launch_bounds__(1024) k_sim_scan(int64_t* __restrict__ v, long long m) {
  __shared__ long long s_a[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long seg = (m + nt - 1) / nt;
  long long a = 0;
  for (long long i = tid * seg; i < m && i < (tid + 1) * seg; ++i) a += v[i];
  s_a[tid] = a;
  __syncthreads();
  if (tid == 0) {
    long long r = 0;
    for (int i = 0; i < nt; ++i) {
      const long long x = s_a[i];
      s_a[i] = r;
      r += x;
    }
    v[m] = r;
  }
  __syncthreads();
  a = s_a[tid];
  for (long long i = tid * seg; i < m && i < (tid + 1) * seg; ++i) {
    const long long x = v[i];
    v[i] = a;
    a += x;
  }
}

__device__ __forceinline__ int find_c64(const int64_t* pre, int n, long long item) {
  int lo = 0, hi = n - 1;  // largest c with pre[c] <= item
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// block item q of a configuration -> (stream tl, block B).  Items: the SM sets' blocks set by
// set (set j: s + j + m * n_sm), then the wave's blocks, then L_z's blocks.
__device__ __forceinline__ void sim_item(const DPlan& P, long long nsm, long long q, int& tl, long long& B) {
  const long long W = P.W;
  if (q < W) {
    const long long h = W / nsm, r = W % nsm;
    long long j, m;
    if (q < r * (h + 1)) {
      j = q / (h + 1);
      m = q % (h + 1);
    } else {
      const long long q2 = q - r * (h + 1);
      j = r + q2 / h;
      m = q2 % h;
    }
    tl = (int)j;
    B = P.s + j + m * nsm;
  } else if (q < 2 * W) {
    tl = (int)P.nsets;
    B = P.s + (q - W);
  } else {
    tl = (int)P.nsets + 1;
    B = P.Lz0 + (q - 2 * W);
  }
}
// first block item of stream tl
__device__ __forceinline__ long long sim_first_item(const DPlan& P, long long nsm, int tl) {
  const long long W = P.W;
  if (tl < P.nsets) {
    const long long h = W / nsm, r = W % nsm;
    return tl < r ? tl * (h + 1) : r * (h + 1) + (tl - r) * h;
  }
  return tl == P.nsets ? W : 2 * W;
}

__device__ __forceinline__ unsigned long long sim_encode(int field, long long sec, int kind) {
  return ((unsigned long long)field << 48) | ((unsigned long long)kind << kSimSecBits) |
         ((unsigned long long)(sec + kSimSecBias) & ((1ull << kSimSecBits) - 1ull));
}

// Requests of one block item (one warp per item): count (GEN = false) or write them.
template <bool GEN>
__global__ void __launch_bounds__(256) k_sim_warp(const DPlan* __restrict__ plans, const DKernel* __restrict__ ks,
                                                  const DGpu* __restrict__ gs, const DInstr* __restrict__ instr,
                                                  const uint32_t* __restrict__ order,
                                                  const int64_t* __restrict__ ipre, int n, long long n_items,
                                                  int64_t* __restrict__ cnt, unsigned long long* __restrict__ req) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const long long nwg = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long item = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < n_items; item += nwg) {
    const int c = find_c64(ipre, n, item);
    const DPlan& P = plans[c];
    const DKernel& K = ks[P.kid];
    const DGpu& G = gs[P.gid];
    int tl;
    long long B;
    sim_item(P, (long long)G.g.n_sm, item - ipre[c], tl, B);
    const int kinds = tl < P.nsets ? 1 : 3;
    const DInstr* tab = instr + (long long)c * kMaxInstr;
    const uint32_t* ord = order + (long long)c * kMaxInstr;
    long long total = 0;
    unsigned long long* out = GEN ? req + cnt[item] : nullptr;
    for (int w = 0; w < P.nwarps; ++w) {
      const Lane L = lane_setup(P, B, w, lane);
      int cur_field = -1;
      long long plane = 0;
      for (int ii = 0; ii < P.n_instr; ++ii) {
        const DInstr e = tab[ord[ii]];
        if (!((kinds >> e.kind) & 1)) continue;
        const bool iss = (e.kmask & L.act) != 0ull;
        const unsigned m = __ballot_sync(FULL, iss);
        if (m == 0u) continue;
        if (e.field != cur_field) {
          cur_field = e.field;
          const DField& F = K.f[e.field];
          plane = L.base[0] + F.pitch[1] * L.base[1] + F.pitch[2] * L.base[2];
        }
        const long long A = e.C + (plane << e.lg_elem);
        const long long sec = A >> G.lg_sector;
        const unsigned pm = m & lt_mask;
        const long long psec = shfl64(sec, pm ? 31 - __clz(pm) : lane);
        const bool us = iss && (pm == 0u || psec != sec);
        const unsigned bm = __ballot_sync(FULL, us);
        if (GEN && us) out[total + __popc(bm & lt_mask)] = sim_encode(e.field, sec, e.kind);
        total += __popc(bm);
      }
    }
    if (!GEN && lane == 0) cnt[item] = total;
  }
}

// stream table: (config, type, request offset, length, L_y start)
__global__ void k_sim_traces(const DPlan* __restrict__ plans, const DGpu* __restrict__ gs, int n,
                             const int64_t* __restrict__ ipre, const int64_t* __restrict__ tpre,
                             const int64_t* __restrict__ cnt, DSimTrace* __restrict__ tr) {
  const int c = blockIdx.x;
  const DPlan& P = plans[c];
  if (!sim_ok(P, gs)) return;
  const long long nsm = gs[P.gid].g.n_sm;
  const int nt = (int)P.nsets + 2;
  for (int tl = threadIdx.x; tl < nt; tl += blockDim.x) {
    const long long a = ipre[c] + sim_first_item(P, nsm, tl);
    const long long b = tl + 1 < nt ? ipre[c] + sim_first_item(P, nsm, tl + 1) : ipre[c] + sim_items_of(P, gs);
    DSimTrace T;
    T.req_off = cnt[a];
    T.n = cnt[b] - cnt[a];
    T.fen_off = T.slot_off = T.hcap = T.m_off = 0;
    T.t_y = tl == nt - 1 ? cnt[a + (P.Ly0 - P.Lz0)] - cnt[a] : 0;
    T.config = c;
    T.type = tl < P.nsets ? 0 : (tl == P.nsets ? 1 : 2);
    tr[tpre[c] + tl] = T;
  }
}

__device__ __forceinline__ unsigned long long sim_hash(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
constexpr unsigned long long kEmpty = ~0ull;

// the wave's load sectors (WLD) of each configuration into its hash set
__global__ void k_sim_wld(const DSimTrace* __restrict__ tr, long long n_traces, const unsigned long long* __restrict__ req,
                          unsigned long long* __restrict__ wld, const int64_t* __restrict__ wld_off) {
  for (long long t = blockIdx.y; t < n_traces; t += gridDim.y) {
    const DSimTrace T = tr[t];
    if (T.type != 1) continue;
    unsigned long long* H = wld + wld_off[2 * T.config];
    const unsigned long long hm = (unsigned long long)wld_off[2 * T.config + 1] - 1ull;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < T.n; i += (long long)gridDim.x * blockDim.x) {
      const unsigned long long r = req[T.req_off + i];
      if ((r >> kSimSecBits) & 1ull) continue;  // stores
      unsigned long long h = sim_hash(r) & hm;
      for (;;) {
        const unsigned long long old = atomicCAS(&H[h], kEmpty, r);
        if (old == kEmpty || old == r) break;
        h = (h + 1) & hm;
      }
    }
  }
}

__device__ __forceinline__ bool wld_has(const unsigned long long* H, unsigned long long hm, unsigned long long k) {
  unsigned long long h = sim_hash(k) & hm;
  for (;;) {
    const unsigned long long v = H[h];
    if (v == k) return true;
    if (v == kEmpty) return false;
    h = (h + 1) & hm;
  }
}

// Fenwick tree over positions [0, n) (1-indexed storage, f[1..n]).  The prefix over [0, x)
// visits the nodes (x >> b) << b for every set bit b of x: independent loads, issued together.
__device__ __forceinline__ uint32_t fen_prefix(const uint32_t* f, long long x) {  // sum over [0, x)
  uint32_t s = 0;
#pragma unroll
  for (int b = 0; b < 31; ++b)
    if ((x >> b) & 1) s += __ldcg(&f[(x >> b) << b]);
  return s;
}
__device__ __forceinline__ void fen_add(uint32_t* f, long long n, long long pos, uint32_t d) {
  for (long long x = pos + 1; x <= n; x += x & -x) atomicAdd(&f[x], d);
}
__device__ __forceinline__ int cap_bin(const unsigned long long* lines, int ncap, uint32_t D) {
  if (D == 0xffffffffu) return ncap;  // compulsory: a miss at every capacity
  int b = 0;  // number of capacities (ascending, in lines) <= D
  while (b < ncap && lines[b] <= (unsigned long long)D) ++b;
  return b;
}

constexpr uint32_t kInf = 0xffffffffu;
constexpr int kSimWarps = 4;

__global__ void __launch_bounds__(kSimWarps * 32) k_sim_run(const DPlan* __restrict__ plans,
                                                             const DGpu* __restrict__ gs, SimScratch S, int ncap) {
  __shared__ unsigned s_hist[kSimWarps][2][kSimHist];
  __shared__ unsigned long long s_lines[kSimMaxCaps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u, gt = lane == 31 ? 0u : ~((2u << lane) - 1u);
  for (int k = threadIdx.x; k < ncap; k += blockDim.x) s_lines[k] = S.lines[k];
  __syncthreads();
  for (;;) {
    long long t = 0;
    if (lane == 0) t = (long long)atomicAdd(S.counter, 1ull);
    t = shfl64(t, 0);
    if (t >= S.n_traces) break;
    const DSimTrace T = S.traces[t];
    const DPlan& P = plans[T.config];
    const DGpu& G = gs[P.gid];
    const int lspl = G.lg_line - G.lg_sector, spl = 1 << lspl;
    const long long n = T.n;
    uint32_t* f = S.fen + T.fen_off;
    unsigned long long* keys = S.keys + T.slot_off;
    uint32_t* lastv = S.last + T.slot_off;
    uint32_t* Mv = S.M + T.m_off;
    uint32_t* SLv = S.SL + T.m_off;
    const unsigned long long hm = (unsigned long long)T.hcap - 1ull;
    for (int b = lane; b < 2 * kSimHist; b += 32) s_hist[wid][b / kSimHist][b % kSimHist] = 0u;
    unsigned long long comp = 0, counted_n = 0;
    __syncwarp();
    unsigned long long r_next = lane < n ? __ldcs(&S.req[T.req_off + lane]) : 0ull;
    for (long long c0 = 0; c0 < n; c0 += 32) {
      const long long i = c0 + lane;
      const bool valid = i < n;
      const unsigned long long r = r_next;
      r_next = (i + 32 < n) ? __ldcs(&S.req[T.req_off + i + 32]) : 0ull;  // prefetch the next step
      const unsigned long long sb = r & ((1ull << kSimSecBits) - 1ull);
      const int is_st = (int)((r >> kSimSecBits) & 1ull);
      const unsigned long long lkey = ((r >> 48) << 48) | (sb >> lspl);
      const int sidx = (int)(sb & (unsigned long long)(spl - 1));
      const unsigned m = __match_any_sync(FULL, valid ? lkey : ((1ull << 63) | (unsigned long long)lane));
      const unsigned pl = m & lt, ngm = m & gt;
      const int prev_lane = pl ? 31 - __clz(pl) : -1;
      const int next_lane = valid ? (ngm ? __ffs(ngm) - 1 : 32) : -1;
      const bool leader = valid && prev_lane < 0;
      long long slot = -1;
      int existed = 0;
      long long lastp = -1;
      if (leader) {
        unsigned long long h = sim_hash(lkey) & hm;
        for (;;) {
          const unsigned long long k = keys[h];
          if (k == lkey) {
            existed = 1;
            break;
          }
          if (k == kEmpty) {
            const unsigned long long old = atomicCAS(&keys[h], kEmpty, lkey);
            if (old == kEmpty) break;
            if (old == lkey) {
              existed = 1;
              break;
            }
          }
          h = (h + 1) & hm;
        }
        slot = (long long)h;
        if (existed) lastp = (long long)lastv[slot];
      }
      const int first = __ffs(m) - 1;
      slot = shfl64(slot, first);
      existed = __shfl_sync(FULL, existed, first);
      uint32_t msnap = (valid && existed) ? Mv[slot * spl + sidx] : kInf;
      // previous access of the line: an earlier lane of this step, or the stored last access
      const long long p = prev_lane >= 0 ? c0 + prev_lane : lastp;
      const long long psnap = (leader && lastp >= 0) ? lastp : -1;  // a marker of the state before the step
      // prefix over [0, c0) (the same for every lane): one tree node per set bit of c0, one lane each
      uint32_t fpart = 0u;
      if (lane < 31 && ((c0 >> lane) & 1)) fpart = __ldcg(&f[(c0 >> lane) << lane]);
      const uint32_t Fc0 = __reduce_add_sync(FULL, fpart);
      const uint32_t Fp = psnap >= 0 ? fen_prefix(f, psnap + 1) : 0u;
      // pass 1 (uniform): markers moved / set by the step's earlier lanes
      int sub = 0, add_all = 0, add_after_prev = 0;
      const int psnap32 = (int)psnap;  // positions < 2^31 (ws_simulate limit)
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const long long pj = __shfl_sync(FULL, psnap32, j);
        const int nj = __shfl_sync(FULL, next_lane, j);
        if (j < lane) {
          sub += (pj > p) ? 1 : 0;                 // old marker in (p, c0) moved into the step
          const int still = nj >= lane ? 1 : 0;    // lane j is the latest access of its line before me
          add_all += still;
          add_after_prev += (j > prev_lane) ? still : 0;
        }
      }
      uint32_t dist = kInf;
      if (valid && p >= 0)
        dist = p >= c0 ? (uint32_t)add_after_prev : (uint32_t)((long long)Fc0 - (long long)Fp - sub + add_all);
      // pass 2 (uniform): D = max line distance since the sector's previous access (own access
      // included); suffix maxima for the write-back
      uint32_t acc = msnap, suf = 0u, lmax = 0u;
      bool later_same = false;
      unsigned amask = 0u;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const uint32_t dj = __shfl_sync(FULL, dist, j);
        const int sj = __shfl_sync(FULL, sidx, j);
        if ((m >> j) & 1u) {
          lmax = max(lmax, dj);
          amask |= 1u << sj;
          if (j < lane) {
            if (sj == sidx) acc = 0u;
            else acc = max(acc, dj);
          } else if (j == lane) {
            acc = max(acc, dj);
          } else {
            suf = max(suf, dj);
            later_same |= sj == sidx;
          }
        }
      }
      if (valid) {
        const uint32_t D = acc;
        const bool counted = T.type == 0 || (T.type == 1 && is_st);
        if (counted) {
          atomicAdd(&s_hist[wid][0][cap_bin(s_lines, ncap, D)], 1u);
          counted_n += 1;
          comp += D == kInf ? 1ull : 0ull;
        }
        // the step's last access of each (line, sector): running max restarts at it
        if (!later_same) {
          Mv[slot * spl + sidx] = suf;
          SLv[slot * spl + sidx] = (uint32_t)i;
        }
        if (next_lane == 32) {  // last lane of the line: sectors the step did not touch
          for (int sg = 0; sg < spl; ++sg) {
            if ((amask >> sg) & 1u) continue;
            if (existed) {
              const uint32_t a2 = Mv[slot * spl + sg];
              Mv[slot * spl + sg] = max(a2, lmax);
            } else {
              Mv[slot * spl + sg] = kInf;
              SLv[slot * spl + sg] = kInf;
            }
          }
          lastv[slot] = (uint32_t)i;
        }
      }
      // the step's new markers (last access of each line in the step): the tree nodes inside the
      // step (c0 + 1 .. c0 + 31; untouched so far) are written directly, the node c0 + 32 and its
      // ancestors (which cover the whole step) get the step's total
      {
        const unsigned newm = __ballot_sync(FULL, valid && next_lane == 32);
        const int j1 = lane + 1;
        if (lane < 31 && c0 + j1 <= n) {
          const int lb = j1 & -j1;
          const unsigned msk = (lb >= 32 ? 0xffffffffu : ((1u << lb) - 1u)) << (j1 - lb);
          f[c0 + j1] = (uint32_t)__popc(newm & msk);
        }
        if (lane == 0 && c0 + 32 <= n) {
          const uint32_t tot = (uint32_t)__popc(newm);
          if (tot)
            for (long long x = c0 + 32; x <= n; x += x & -x) atomicAdd(&f[x], tot);
        }
      }
      if (psnap >= 0) fen_add(f, n, psnap, 0xffffffffu);
      __syncwarp();
    }
    // end state of L_z: the wave's overlap sectors still valid (y: touched by blocks >= Ly0)
    unsigned long long ovy = 0, ovz = 0;
    if (T.type == 2) {
      const uint32_t total = fen_prefix(f, n);
      const unsigned long long* H = S.wld + S.wld_off[2 * T.config];
      const unsigned long long whm = (unsigned long long)S.wld_off[2 * T.config + 1] - 1ull;
      for (long long sl = lane; sl < T.hcap; sl += 32) {
        const unsigned long long k = keys[sl];
        if (k == kEmpty) continue;
        const uint32_t dend = total - fen_prefix(f, (long long)lastv[sl] + 1);
        for (int sg = 0; sg < spl; ++sg) {
          const uint32_t lastsec = SLv[sl * spl + sg];
          if (lastsec == kInf) continue;
          const unsigned long long skey = ((k >> 48) << 48) | (((k & ((1ull << 48) - 1ull)) << lspl) | (unsigned)sg);
          if (!wld_has(H, whm, skey)) continue;
          const uint32_t De = max(Mv[sl * spl + sg], dend);
          const bool isy = (long long)lastsec >= T.t_y;
          atomicAdd(&s_hist[wid][isy ? 0 : 1][cap_bin(s_lines, ncap, De)], 1u);
          if (isy) ++ovy;
          else ++ovz;
        }
      }
    }
    __syncwarp();
    // per-configuration accumulators
    unsigned long long* A = S.acc + (long long)T.config * kSimAcc;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      comp += __shfl_down_sync(FULL, comp, o);
      counted_n += __shfl_down_sync(FULL, counted_n, o);
      ovy += __shfl_down_sync(FULL, ovy, o);
      ovz += __shfl_down_sync(FULL, ovz, o);
    }
    if (lane == 0) {
      if (T.type == 0) {
        atomicAdd(A + SA_L1REQ, counted_n);
        atomicAdd(A + SA_L1COMP, comp);
      } else if (T.type == 1) {
        atomicAdd(A + SA_STREQ, counted_n);
        atomicAdd(A + SA_STCOMP, comp);
      } else {
        atomicAdd(A + SA_OVY, ovy);
        atomicAdd(A + SA_OVZ, ovz);
      }
    }
    const int h0 = T.type == 0 ? SA_L1H : (T.type == 1 ? SA_L1H + kSimHist : SA_L1H + 2 * kSimHist);
    for (int b = lane; b <= ncap; b += 32) {
      if (s_hist[wid][0][b]) atomicAdd(A + h0 + b, (unsigned long long)s_hist[wid][0][b]);
      if (T.type == 2 && s_hist[wid][1][b]) atomicAdd(A + SA_L1H + 3 * kSimHist + b, (unsigned long long)s_hist[wid][1][b]);
    }
    __syncwarp();
  }
}

// sample records: one thread per (configuration, capacity)
__global__ void k_sim_out(const DPlan* __restrict__ plans, const DGpu* __restrict__ gs, const ws_result* __restrict__ est,
                          int n, const unsigned long long* __restrict__ acc, int ncap, const uint64_t* __restrict__ caps,
                          const int* __restrict__ cap_rank, ws_sim_result* __restrict__ out) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (long long)n * ncap) return;
  const int c = (int)(id / ncap), k = (int)(id % ncap);
  ws_sim_result o;
  memset(&o, 0, sizeof(o));
  const DPlan& P = plans[c];
  o.capacity_bytes = caps[k];
  o.status = sim_status(P, gs);
  if (o.status == WS_OK && caps[k] < 1) o.status = WS_EINVAL;
  if (o.status != WS_OK) {
    out[id] = o;
    return;
  }
  const DGpu& G = gs[P.gid];
  const ws_result& R = est[c];
  const unsigned long long* A = acc + (long long)c * kSimAcc;
  const int kr = cap_rank[k];  // position of this capacity in the ascending order
  unsigned long long l1m = 0, stm = 0, yr = 0, zr = 0;
  for (int b = 0; b <= ncap; ++b) {
    if (b > kr) {
      l1m += A[SA_L1H + b];
      stm += A[SA_L1H + kSimHist + b];
    } else {
      yr += A[SA_L1H + 2 * kSimHist + b];
      zr += A[SA_L1H + 3 * kSimHist + b];
    }
  }
  o.l1_requests = A[SA_L1REQ];
  o.l1_compulsory = A[SA_L1COMP];
  o.l1_misses = l1m;
  o.st_requests = A[SA_STREQ];
  o.st_compulsory = A[SA_STCOMP];
  o.st_misses = stm;
  o.ov_y = A[SA_OVY];
  o.y_resident = yr;
  o.ov_z_only = A[SA_OVZ];
  o.z_resident = zr;
  const double LB = (double)G.g.line_bytes, C = (double)caps[k];
  o.O_l1 = ((double)R.sm_ld_lines * LB / (double)P.nsets) / C;
  o.O_y = (double)R.ly_lines * LB / C;
  o.O_z = (double)R.lz_lines * LB / C;
  o.O_st = (double)R.wave_lines * LB / C;
  o.R_l1 = o.l1_requests > o.l1_compulsory
               ? (double)(o.l1_requests - o.l1_misses) / (double)(o.l1_requests - o.l1_compulsory) : 1.0;
  o.R_st = o.st_requests > o.st_compulsory
               ? (double)(o.st_requests - o.st_misses) / (double)(o.st_requests - o.st_compulsory) : 1.0;
  o.R_y = o.ov_y > 0 ? (double)o.y_resident / (double)o.ov_y : 1.0;
  o.R_z = o.ov_z_only > 0 ? (double)o.z_resident / (double)o.ov_z_only : 1.0;
  out[id] = o;
}

// Gompertz least squares (ws.h ws_fit_gompertz): grid search by the CTA, LM by thread 0
// (sequential sums, the oracle's order).  out = (a, b, c, rss).
__device__ __forceinline__ double gompertz_abc(double a, double b, double c, double O) { return a * exp(-b * exp(-c * O)); }

__device__ double fit_rss_d(const double* O, const double* R, int n, double a, double b, double c) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    const double e = gompertz_abc(a, b, c, O[i]) - R[i];
    s += e * e;
  }
  return s;
}

__global__ void __launch_bounds__(256) k_fit(const double* __restrict__ O, const double* __restrict__ R, int n,
                                             double* __restrict__ out) {
  __shared__ double s_v[256];
  __shared__ int s_i[256];
  const int tid = threadIdx.x;
  double best = __longlong_as_double(0x7ff0000000000000ll);
  int bi = 1 << 30;
  for (int idx = tid; idx < 6 * 23 * 32; idx += blockDim.x) {
    const int i = idx / (23 * 32), j = (idx / 32) % 23, k = idx % 32;
    const double v = fit_rss_d(O, R, n, 0.5 + 0.1 * i, exp(-8.0 + 0.5 * j), -8.0 + 0.25 * k);
    if (v < best) {  // ascending idx per thread: keeps the first minimum
      best = v;
      bi = idx;
    }
  }
  s_v[tid] = best;
  s_i[tid] = bi;
  __syncthreads();
  if (tid != 0) return;
  for (int t = 1; t < (int)blockDim.x; ++t)
    if (s_v[t] < best || (s_v[t] == best && s_i[t] < bi)) {
      best = s_v[t];
      bi = s_i[t];
    }
  double th[3] = {0.5 + 0.1 * (bi / (23 * 32)), exp(-8.0 + 0.5 * ((bi / 32) % 23)), -8.0 + 0.25 * (bi % 32)};
  double lambda = 1e-3;
  for (int it = 0; it < 200; ++it) {
    double A[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, gv[3] = {0, 0, 0};
    for (int m = 0; m < n; ++m) {
      const double E = exp(-th[2] * O[m]);
      const double F = exp(-th[1] * E);
      const double J[3] = {F, -th[0] * E * F, th[0] * F * th[1] * E * O[m]};
      const double res = th[0] * F - R[m];
      for (int a = 0; a < 3; ++a) {
        gv[a] += J[a] * res;
        for (int b = 0; b < 3; ++b) A[a][b] += J[a] * J[b];
      }
    }
    double Mx[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) Mx[a][b] = A[a][b] + (a == b ? lambda * A[a][a] : 0.0);
    const double det = Mx[0][0] * (Mx[1][1] * Mx[2][2] - Mx[1][2] * Mx[2][1]) -
                       Mx[0][1] * (Mx[1][0] * Mx[2][2] - Mx[1][2] * Mx[2][0]) +
                       Mx[0][2] * (Mx[1][0] * Mx[2][1] - Mx[1][1] * Mx[2][0]);
    if (!(fabs(det) > 0.0)) break;
    double d[3];
    for (int col = 0; col < 3; ++col) {
      double Mc[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Mc[a][b] = (b == col) ? -gv[a] : Mx[a][b];
      d[col] = (Mc[0][0] * (Mc[1][1] * Mc[2][2] - Mc[1][2] * Mc[2][1]) -
                Mc[0][1] * (Mc[1][0] * Mc[2][2] - Mc[1][2] * Mc[2][0]) +
                Mc[0][2] * (Mc[1][0] * Mc[2][1] - Mc[1][1] * Mc[2][0])) / det;
    }
    const double t2[3] = {th[0] + d[0], th[1] + d[1], th[2] + d[2]};
    const double v = fit_rss_d(O, R, n, t2[0], t2[1], t2[2]);
    if (v < best) {
      best = v;
      th[0] = t2[0];
      th[1] = t2[1];
      th[2] = t2[2];
      lambda = fmax(lambda / 10.0, 1e-15);
    } else {
      lambda *= 10.0;
    }
  }
  out[0] = th[0];
  out[1] = th[1];
  out[2] = th[2];
  out[3] = best;
}



// ================================================================== NEXT-1: long streams in parallel
// A stream of n >= kLongStream requests is not replayed by one warp but computed offline, fully
// parallel (same exact results): dense line ids (hash), a stable radix sort of the requests by
// line (time order kept inside each line), previous access p(i) of every request's line, the LRU
// stack distance dist(i) = #{j < i : p(j) <= p(i)} - p(i) - 1 (the distinct lines accessed in
// (p(i), i) are the accesses j there whose own previous access is <= p(i), and every j <= p(i)
// has p(j) < j) counted with a wavelet matrix over p(j) + 1, then one thread per line walks its
// accesses in time order with the per-sector running maxima D (as the warp path), histogramming
// the counted requests and, for the layer stream, the end state of the overlap sectors.
constexpr long long kLongStream = 1 << 16;
constexpr int kScanB = 1024;  // elements per block of the device-wide scans

__global__ void __launch_bounds__(256) k_ps_reduce(const uint32_t* __restrict__ in, long long m, uint32_t* __restrict__ bsum) {
  const long long b0 = (long long)blockIdx.x * kScanB;
  uint32_t v = 0;
  for (int r = 0; r < kScanB / 256; ++r) {
    const long long i = b0 + r * 256 + threadIdx.x;
    if (i < m) v += in[i];
  }
  v = __reduce_add_sync(FULL, v);
  __shared__ uint32_t s[8];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += s[w];
    bsum[blockIdx.x] = t;
  }
}
// single CTA: exclusive scan of nb block sums (in place), total to *total
__global__ void __launch_bounds__(1024) k_ps_bsum(uint32_t* __restrict__ bsum, long long nb, uint32_t* __restrict__ total) {
  __shared__ unsigned long long s[1024];
  const int tid = threadIdx.x;
  const long long seg = (nb + 1023) / 1024;
  unsigned long long a = 0;
  for (long long i = tid * seg; i < nb && i < (tid + 1) * seg; ++i) a += bsum[i];
  s[tid] = a;
  __syncthreads();
  if (tid == 0) {
    unsigned long long r = 0;
    for (int i = 0; i < 1024; ++i) {
      const unsigned long long x = s[i];
      s[i] = r;
      r += x;
    }
    *total = (uint32_t)r;
  }
  __syncthreads();
  a = s[tid];
  for (long long i = tid * seg; i < nb && i < (tid + 1) * seg; ++i) {
    const uint32_t x = bsum[i];
    bsum[i] = (uint32_t)a;
    a += x;
  }
}
// exclusive scan of io[0..m) given the scanned block sums
__global__ void __launch_bounds__(256) k_ps_apply(uint32_t* __restrict__ io, long long m, const uint32_t* __restrict__ bsum) {
  __shared__ uint32_t s_w[8];
  __shared__ uint32_t s_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long b0 = (long long)blockIdx.x * kScanB;
  if (threadIdx.x == 0) s_base = bsum[blockIdx.x];
  __syncthreads();
  for (int r = 0; r < kScanB / 256; ++r) {
    const long long i = b0 + r * 256 + threadIdx.x;
    const uint32_t v = i < m ? io[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    uint32_t wb = 0, tot = 0;
    for (int w = 0; w < 8; ++w) {
      const uint32_t t = s_w[w];
      if (w < wid) wb += t;
      tot += t;
    }
    if (i < m) io[i] = s_base + wb + x - v;
    __syncthreads();
    if (threadIdx.x == 0) s_base += tot;
    __syncthreads();
  }
}

// dense line ids: phase 1 insert the line keys, phase 2 (after a scan of the occupancy flags)
// look them up; ids follow slot order (deterministic)
__global__ void k_pl_occ(const unsigned long long* __restrict__ H, long long hcap, uint32_t* __restrict__ occ) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < hcap; i += (long long)gridDim.x * blockDim.x)
    occ[i] = H[i] != kEmpty ? 1u : 0u;
}

// stable LSD radix pass on 8 bits of key (tiles of 2048 = 256 threads x 8 rounds)
constexpr int kRsTile = 2048;
__global__ void __launch_bounds__(256) k_rs_hist(const uint32_t* __restrict__ key, long long n, int shift,
                                                 uint32_t* __restrict__ hist, long long ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const long long t0 = (long long)blockIdx.x * kRsTile;
  for (int r = 0; r < kRsTile / 256; ++r) {
    const long long i = t0 + r * 256 + threadIdx.x;
    if (i < n) atomicAdd(&h[(key[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(long long)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];   // digit-major
}
__global__ void __launch_bounds__(256) k_rs_scatter(const uint32_t* __restrict__ key, const uint32_t* __restrict__ val,
                                                    long long n, int shift, const uint32_t* __restrict__ off,
                                                    long long ntiles, uint32_t* __restrict__ key2,
                                                    uint32_t* __restrict__ val2) {
  __shared__ uint32_t run[256];           // elements of each digit already placed from this tile
  __shared__ uint32_t wc[8][256];         // per-warp digit counts of the current round
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  run[tid] = off[(long long)tid * ntiles + blockIdx.x];
  const long long t0 = (long long)blockIdx.x * kRsTile;
  for (int r = 0; r < kRsTile / 256; ++r) {
#pragma unroll
    for (int w = 0; w < 8; ++w) wc[w][tid] = 0u;
    __syncthreads();
    const long long i = t0 + r * 256 + tid;
    const bool ok = i < n;
    const uint32_t k = ok ? key[i] : 0u, v = ok ? val[i] : 0u;
    const uint32_t d = (k >> shift) & 255u;
    const unsigned peers = __match_any_sync(FULL, ok ? d : 0x100u + (unsigned)lane);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (ok && rank == 0) wc[wid][d] = (uint32_t)__popc(peers);
    __syncthreads();
    uint32_t before = 0;  // same digit in earlier warps of this round
    for (int w = 0; w < wid; ++w) before += wc[w][d];
    if (ok) {
      const uint32_t pos = run[d] + before + (uint32_t)rank;
      key2[pos] = k;
      val2[pos] = v;
    }
    __syncthreads();
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += wc[w][tid];
    run[tid] += tot;
    __syncthreads();
  }
}

// previous access of the line, last-access flags, line starts; V = prev + 1 for the wavelet matrix,
// the last-access flag in bit 31 (positions < 2^31 - 2): one scattered store per access
__global__ void k_pl_prev(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ sval, long long n,
                          uint32_t* __restrict__ V, uint32_t* __restrict__ lstart) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const uint32_t i = sval[k], l = skey[k];
    const bool first = k == 0 || skey[k - 1] != l;
    const bool last = k + 1 == n || skey[k + 1] != l;
    V[i] = (first ? 0u : sval[k - 1] + 1u) | (last ? 0x80000000u : 0u);
    if (first) lstart[l] = (uint32_t)k;
  }
}
// split the flags off (coalesced)
__global__ void k_pl_split(uint32_t* __restrict__ V, long long n, uint32_t* __restrict__ islast) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t v = V[i];
    islast[i] = v >> 31;
    V[i] = v & 0x7fffffffu;
  }
}
// one wavelet-matrix level, one entry per 64 positions: {bit word, zeros before the word} (one
// 16-byte load per rank query).  k_wm_bits writes the words and each word's zero count (wz);
// the exclusive scan of wz is the rank directory, which k_wm_next stores next to the words while
// it partitions the values stably by the bit (zeros first)
__global__ void k_wm_bits(const uint32_t* __restrict__ cur, long long n, int bit, ulonglong2* __restrict__ wr,
                          uint32_t* __restrict__ wz) {
  constexpr int kU = 4;  // words per warp iteration (loads in flight)
  const int lane = threadIdx.x & 31;
  const long long nw = (n + 63) / 64;
  for (long long w0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kU; w0 < nw;
       w0 += (((long long)gridDim.x * blockDim.x) >> 5) * kU) {
    uint32_t b[2 * kU];
#pragma unroll
    for (int u = 0; u < 2 * kU; ++u) {
      const long long i = w0 * 64 + u * 32 + lane;
      b[u] = i < n ? (cur[i] >> bit) & 1u : 2u;  // 2: past the end (neither bit)
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned lo = __ballot_sync(FULL, b[2 * u] == 1u), hi = __ballot_sync(FULL, b[2 * u + 1] == 1u);
      const unsigned z0 = __ballot_sync(FULL, b[2 * u] == 0u), z1 = __ballot_sync(FULL, b[2 * u + 1] == 0u);
      if (lane == u && w0 + u < nw) {
        wr[w0 + u].x = ((unsigned long long)hi << 32) | lo;
        wz[w0 + u] = (uint32_t)(__popc(z0) + __popc(z1));
      }
    }
  }
}
__global__ void k_wm_next(const uint32_t* __restrict__ cur, long long n, int bit, const uint32_t* __restrict__ wz,
                          const uint32_t* __restrict__ Z, uint32_t* __restrict__ nxt) {
  constexpr int kU = 4;  // words per warp iteration; the word's bits come from ballots
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t Zv = *Z;
  const long long nw = (n + 63) / 64;
  for (long long w0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kU; w0 < nw;
       w0 += (((long long)gridDim.x * blockDim.x) >> 5) * kU) {
    uint32_t v[2 * kU], zb[kU];
#pragma unroll
    for (int u = 0; u < 2 * kU; ++u) {
      const long long i = w0 * 64 + u * 32 + lane;
      v[u] = i < n ? cur[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) zb[u] = w0 + u < nw ? wz[w0 + u] : 0u;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long i0 = w0 * 64 + u * 64 + lane, i1 = i0 + 32;
      const bool one0 = (v[2 * u] >> bit) & 1u, one1 = (v[2 * u + 1] >> bit) & 1u;
      const unsigned z0 = __ballot_sync(FULL, i0 < n && !one0), z1 = __ballot_sync(FULL, i1 < n && !one1);
      const uint32_t zp0 = zb[u] + (uint32_t)__popc(z0 & lt);                        // zeros before i0
      const uint32_t zp1 = zb[u] + (uint32_t)__popc(z0) + (uint32_t)__popc(z1 & lt);  // zeros before i1
      if (i0 < n) nxt[one0 ? Zv + (uint32_t)i0 - zp0 : zp0] = v[2 * u];
      if (i1 < n) nxt[one1 ? Zv + (uint32_t)i1 - zp1 : zp1] = v[2 * u + 1];
    }
  }
}
// the rank directory next to the words (a separate pass: stores into the entries while k_wm_next
// reads their words would evict the words' L1 lines); the sentinel entry holds Z
__global__ void k_wm_rank(ulonglong2* __restrict__ wr, long long nw, const uint32_t* __restrict__ wz,
                          const uint32_t* __restrict__ Z) {
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (long long)gridDim.x * blockDim.x)
    wr[w].y = w + 1 < nw ? wz[w] : *Z;
}
__device__ __forceinline__ uint32_t wm_rank0(const ulonglong2* wr, long long pos) {
  const ulonglong2 e = wr[pos >> 6];
  const int r = (int)(pos & 63);
  return (uint32_t)e.y + (r ? (uint32_t)__popcll(~e.x & ((1ull << r) - 1ull)) : 0u);
}
// dist(i) = #{j < i : V[j] < p(i) + 2} - p(i) - 1 (kInf for a line's first access).  Only the
// capacity bin of a distance is ever used (cap_bin of running maxima; cap_bin is monotone), so a
// reuse window of i - p - 1 < lines[0] positions -- at most that many distinct lines, a hit at
// every capacity -- stores the window length, an upper bound in the same bin, without a query.
__global__ void k_pl_dist(const uint32_t* __restrict__ V, long long n, int LV, const ulonglong2* __restrict__ wr,
                          const uint32_t* __restrict__ Zs, long long wstride,
                          const unsigned long long* __restrict__ lines, uint32_t* __restrict__ dist) {
  const unsigned long long l0 = lines[0];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t v = V[i];
    if (v == 0u) {
      dist[i] = kInf;
      continue;
    }
    const uint32_t p = v - 1u, x = p + 2u;
    const uint32_t win = (uint32_t)i - p - 1u;
    if ((unsigned long long)win < l0) {
      dist[i] = win;
      continue;
    }
    long long a = 0, b = i;
    uint32_t cnt = 0;
    for (int lev = 0; lev < LV; ++lev) {
      const int bit = LV - 1 - lev;
      const ulonglong2* W = wr + (long long)lev * wstride;
      const uint32_t ra = wm_rank0(W, a), rb = wm_rank0(W, b);
      if ((x >> bit) & 1u) {
        cnt += rb - ra;
        a = Zs[lev] + (a - ra);
        b = Zs[lev] + (b - rb);
      } else {
        a = ra;
        b = rb;
      }
    }
    dist[i] = cnt - p - 1u;
  }
}

// ---- batched long streams: several long streams concatenated (positions are global; the stack
// distance formula is invariant under the shift, and every quantity that must stay per stream --
// line ids, the end state -- is keyed by the stream)
struct DPB {
  int64_t req_off, n, start, hoff, hcap, t_y_abs, wld_off, wld_cap;
  int32_t type, config, spl, lspl;
};

__global__ void k_pb_gather(const unsigned long long* __restrict__ req, const DPB* __restrict__ pb,
                            unsigned long long* __restrict__ cat, uint32_t* __restrict__ tid) {
  const DPB T = pb[blockIdx.y];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < T.n; i += (long long)gridDim.x * blockDim.x) {
    cat[T.start + i] = req[T.req_off + i];
    tid[T.start + i] = blockIdx.y;
  }
}
__global__ void k_pb_insert(const unsigned long long* __restrict__ cat, const uint32_t* __restrict__ tid, long long n,
                            const DPB* __restrict__ pb, unsigned long long* __restrict__ H) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const DPB& T = pb[tid[i]];
    const unsigned long long r = cat[i];
    const unsigned long long sb = r & ((1ull << kSimSecBits) - 1ull);
    const unsigned long long lkey = ((r >> 48) << 48) | (sb >> T.lspl);
    unsigned long long* R = H + T.hoff;
    const unsigned long long hm = (unsigned long long)T.hcap - 1ull;
    unsigned long long h = sim_hash(lkey) & hm;
    for (;;) {
      const unsigned long long old = atomicCAS(&R[h], kEmpty, lkey);
      if (old == kEmpty || old == lkey) break;
      h = (h + 1) & hm;
    }
  }
}
__global__ void k_pb_ids(const unsigned long long* __restrict__ cat, const uint32_t* __restrict__ tid, long long n,
                         const DPB* __restrict__ pb, const unsigned long long* __restrict__ H,
                         const uint32_t* __restrict__ occ, uint32_t* __restrict__ key, uint32_t* __restrict__ val,
                         unsigned char* __restrict__ sidx) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const DPB& T = pb[tid[i]];
    const unsigned long long r = cat[i];
    const unsigned long long sb = r & ((1ull << kSimSecBits) - 1ull);
    const unsigned long long lkey = ((r >> 48) << 48) | (sb >> T.lspl);
    const unsigned long long* R = H + T.hoff;
    const unsigned long long hm = (unsigned long long)T.hcap - 1ull;
    unsigned long long h = sim_hash(lkey) & hm;
    while (R[h] != lkey) h = (h + 1) & hm;
    key[i] = occ[T.hoff + h];  // dense id, grouped by stream (regions in stream order)
    val[i] = (uint32_t)i;
    sidx[i] = (unsigned char)(sb & (unsigned long long)(T.spl - 1));
  }
}
// one thread per line of the batch (ids grouped by stream): per-sector running maxima, the
// counted requests' histograms, the layer stream's end state.  Histograms of the CTA's first
// stream accumulate in shared memory, lines of other streams add to global memory directly.
__global__ void __launch_bounds__(128) k_pb_lines(const uint32_t* __restrict__ sval, const uint32_t* __restrict__ lstart,
                                                  const uint32_t* __restrict__ Uptr, long long n,
                                                  const unsigned char* __restrict__ sidx, const uint32_t* __restrict__ dist,
                                                  const unsigned long long* __restrict__ cat, const uint32_t* __restrict__ tid,
                                                  const uint32_t* __restrict__ cntlast, const DPB* __restrict__ pb,
                                                  const unsigned long long* __restrict__ wld,
                                                  const unsigned long long* __restrict__ lines, int ncap,
                                                  unsigned long long* __restrict__ acc) {
  __shared__ unsigned s_h[2][kSimHist];
  __shared__ unsigned long long s_c[4];
  __shared__ int s_t;
  const long long U = *Uptr;
  if ((long long)blockIdx.x * blockDim.x >= U) return;
  for (int b = threadIdx.x; b < 2 * kSimHist; b += blockDim.x) s_h[b / kSimHist][b % kSimHist] = 0u;
  if (threadIdx.x < 4) s_c[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) s_t = (int)tid[sval[lstart[(long long)blockIdx.x * blockDim.x]]];
  __syncthreads();
  const int ct = s_t;
  const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (l < U) {
    const long long k0 = lstart[l], k1 = l + 1 < U ? (long long)lstart[l + 1] : n;
    const int t = (int)tid[sval[k0]];
    const DPB& T = pb[t];
    const bool local = t == ct;
    unsigned long long* A = acc + (long long)T.config * kSimAcc;
    const int spl = T.spl, lspl = T.lspl, type = T.type;
    const int h0 = type == 0 ? SA_L1H : (type == 1 ? SA_L1H + kSimHist : SA_L1H + 2 * kSimHist);
    uint32_t M[32], SL[32];
    for (int s = 0; s < spl; ++s) {
      M[s] = kInf;
      SL[s] = kInf;
    }
    unsigned long long cnt = 0, comp = 0;
    uint32_t lasti = 0;
    for (long long k = k0; k < k1; ++k) {
      const uint32_t i = sval[k];
      const int s = sidx[i];
      const uint32_t d = dist[i];
      const uint32_t D = max(M[s], d);
      for (int s2 = 0; s2 < spl; ++s2) M[s2] = max(M[s2], d);
      M[s] = 0u;
      SL[s] = i;
      lasti = i;
      const bool st = (cat[i] >> kSimSecBits) & 1ull;
      if (type == 0 || (type == 1 && st)) {
        const int bin = cap_bin(lines, ncap, D);
        if (local) atomicAdd(&s_h[0][bin], 1u);
        else atomicAdd(A + h0 + bin, 1ull);
        ++cnt;
        comp += D == kInf ? 1ull : 0ull;
      }
    }
    if (cnt) {
      if (local) {
        atomicAdd(&s_c[0], cnt);
        atomicAdd(&s_c[1], comp);
      } else {
        atomicAdd(A + (type == 0 ? SA_L1REQ : SA_STREQ), cnt);
        atomicAdd(A + (type == 0 ? SA_L1COMP : SA_STCOMP), comp);
      }
    }
    if (type == 2) {
      // lines of this stream whose last access is after this line's
      const uint32_t dend = cntlast[T.start + T.n] - cntlast[lasti] - 1u;
      const unsigned long long r = cat[lasti];
      const unsigned long long lkey = ((r >> 48) << 48) | ((r & ((1ull << kSimSecBits) - 1ull)) >> lspl);
      const unsigned long long* Hw = wld + T.wld_off;
      const unsigned long long whm = (unsigned long long)T.wld_cap - 1ull;
      unsigned long long oy = 0, oz = 0;
      for (int s = 0; s < spl; ++s) {
        if (SL[s] == kInf) continue;
        const unsigned long long skey = ((lkey >> 48) << 48) | (((lkey & ((1ull << 48) - 1ull)) << lspl) | (unsigned)s);
        if (!wld_has(Hw, whm, skey)) continue;
        const uint32_t De = max(M[s], dend);
        const bool isy = (long long)SL[s] >= T.t_y_abs;
        const int bin = cap_bin(lines, ncap, De);
        if (local) atomicAdd(&s_h[isy ? 0 : 1][bin], 1u);
        else atomicAdd(A + SA_L1H + (isy ? 2 : 3) * kSimHist + bin, 1ull);
        if (isy) ++oy;
        else ++oz;
      }
      if (local) {
        if (oy) atomicAdd(&s_c[2], oy);
        if (oz) atomicAdd(&s_c[3], oz);
      } else {
        if (oy) atomicAdd(A + SA_OVY, oy);
        if (oz) atomicAdd(A + SA_OVZ, oz);
      }
    }
  }
  __syncthreads();
  const DPB& T = pb[ct];
  unsigned long long* A = acc + (long long)T.config * kSimAcc;
  const int type = T.type;
  const int h0 = type == 0 ? SA_L1H : (type == 1 ? SA_L1H + kSimHist : SA_L1H + 2 * kSimHist);
  for (int b = threadIdx.x; b <= ncap; b += blockDim.x) {
    if (s_h[0][b]) atomicAdd(A + h0 + b, (unsigned long long)s_h[0][b]);
    if (type == 2 && s_h[1][b]) atomicAdd(A + SA_L1H + 3 * kSimHist + b, (unsigned long long)s_h[1][b]);
  }
  if (threadIdx.x == 0) {
    if (type == 0) {
      if (s_c[0]) atomicAdd(A + SA_L1REQ, s_c[0]);
      if (s_c[1]) atomicAdd(A + SA_L1COMP, s_c[1]);
    } else if (type == 1) {
      if (s_c[0]) atomicAdd(A + SA_STREQ, s_c[0]);
      if (s_c[1]) atomicAdd(A + SA_STCOMP, s_c[1]);
    } else {
      if (s_c[2]) atomicAdd(A + SA_OVY, s_c[2]);
      if (s_c[3]) atomicAdd(A + SA_OVZ, s_c[3]);
    }
  }
}

// ------------------------------------------------------------------ NEXT-1 host orchestration
namespace {
// simulator scratch: the k-th allocation of a call reuses the cache's slot k when it is large
// enough; otherwise the slot grows (slots not yet handed out are dropped first when memory is short)
struct Owned {
  SimCache* cache;
  size_t next;
};
template <typename T>
int dmalloc(T** p, size_t count, Owned& o) {
  *p = nullptr;
  if (count == 0) count = 1;
  const size_t need = count * sizeof(T);
  SimCache& C = *o.cache;
  const size_t k = o.next++;
  if (k >= C.ptr.size()) {
    C.ptr.push_back(nullptr);
    C.bytes.push_back(0);
  }
  if (C.bytes[k] < need) {
    if (C.ptr[k]) cudaFree(C.ptr[k]);
    C.ptr[k] = nullptr;
    C.bytes[k] = 0;
    cudaError_t e = cudaMalloc(&C.ptr[k], need);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      for (size_t j = k + 1; j < C.ptr.size(); ++j) {
        if (C.ptr[j]) cudaFree(C.ptr[j]);
        C.ptr[j] = nullptr;
        C.bytes[j] = 0;
      }
      e = cudaMalloc(&C.ptr[k], need);
    }
    if (e != cudaSuccess) {
      C.ptr[k] = nullptr;
      return (int)e;
    }
    C.bytes[k] = need;
  }
  *p = (T*)C.ptr[k];
  return 0;
}
long long pow2_at_least(long long v) {
  long long p = 1;
  while (p < v) p <<= 1;
  return p;
}
}  // namespace

int run_simulate(const ws_config* d_cfgs, int n, const DKernel* d_k, int nk, const DGpu* d_g, int ng,
                 const std::vector<DGpu>& hg, const Scratch& s, ws_result* d_est, const Streams& st, int n_sm_dev,
                 const uint64_t* h_caps, int ncap, ws_sim_result* h_out, uint32_t* launches, cudaEvent_t* ev,
                 SimCache& cache) {
  cudaStream_t q = st.main;
  Owned owned{&cache, 0};
  // WS_SIM_HOSTTIME=1: synchronise and print the elapsed host time at each phase (diagnostics)
  static const bool htime = getenv("WS_SIM_HOSTTIME") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!htime) return;
    cudaStreamSynchronize(q);
    fprintf(stderr, "[ws_simulate] %-14s %9.2f ms\n", what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  };
  auto cleanup = [&](int rc) {
    cudaStreamSynchronize(q);
    mark("end");
    if (rc) cache.release();  // after an error nothing is kept
    return rc;
  };
  uint32_t L = 0;
  int rc = launch_estimate(d_cfgs, n, d_k, nk, d_g, ng, s, d_est, st, n_sm_dev, &L, nullptr);
  if (rc) return cleanup(rc);
  SimScratch S;
  memset(&S, 0, sizeof(S));
  uint64_t* d_caps;
  int* d_rank;
  if ((rc = dmalloc(&S.item_pre, n + 1, owned)) || (rc = dmalloc(&S.trace_pre, n + 1, owned)) ||
      (rc = dmalloc(&S.order, (size_t)n * kMaxInstr, owned)) || (rc = dmalloc(&S.acc, (size_t)n * kSimAcc, owned)) ||
      (rc = dmalloc(&S.lines, kSimMaxCaps, owned)) || (rc = dmalloc(&S.counter, 1, owned)) ||
      (rc = dmalloc(&d_caps, kSimMaxCaps, owned)) || (rc = dmalloc(&d_rank, kSimMaxCaps, owned)))
    return cleanup(rc);
  k_sim_order<<<n, 256, 0, q>>>(s.plans, d_g, s.instr, S.order, n);
  k_sim_cscan<<<1, 1024, 0, q>>>(s.plans, d_g, n, S.item_pre, S.trace_pre);
  L += 2;
  int64_t n_items = 0, n_traces = 0;
  cudaMemcpyAsync(&n_items, S.item_pre + n, sizeof(int64_t), cudaMemcpyDeviceToHost, q);
  cudaMemcpyAsync(&n_traces, S.trace_pre + n, sizeof(int64_t), cudaMemcpyDeviceToHost, q);
  if ((rc = (int)cudaStreamSynchronize(q))) return cleanup(rc);
  int64_t* d_cnt;
  DSimTrace* d_tr;
  mark("estimate");
  if ((rc = dmalloc(&d_cnt, (size_t)n_items + 1, owned)) || (rc = dmalloc(&d_tr, (size_t)n_traces, owned)))
    return cleanup(rc);
  S.item_cnt = d_cnt;
  const int grid = n_sm_dev * 8;
  if (ev) cudaEventRecord(ev[0], q);
  if (n_items > 0) {
    k_sim_warp<false><<<grid, 256, 0, q>>>(s.plans, d_k, d_g, s.instr, S.order, S.item_pre, n, n_items, d_cnt, nullptr);
    k_sim_scan<<<1, 1024, 0, q>>>(d_cnt, n_items);
    k_sim_traces<<<n, 128, 0, q>>>(s.plans, d_g, n, S.item_pre, S.trace_pre, d_cnt, d_tr);
    L += 3;
  }
  std::vector<DSimTrace> tr((size_t)n_traces);
  std::vector<ws_result> est((size_t)n);
  if (n_traces) cudaMemcpyAsync(tr.data(), d_tr, tr.size() * sizeof(DSimTrace), cudaMemcpyDeviceToHost, q);
  cudaMemcpyAsync(est.data(), d_est, est.size() * sizeof(ws_result), cudaMemcpyDeviceToHost, q);
  std::vector<ws_config> cf((size_t)n);
  cudaMemcpyAsync(cf.data(), d_cfgs, cf.size() * sizeof(ws_config), cudaMemcpyDeviceToHost, q);
  if ((rc = (int)cudaStreamSynchronize(q))) return cleanup(rc);
  // ---- host sizing of the per-stream state
  long long req_total = 0, fen_total = 0, slot_total = 0, m_total = 0;
  // streams of >= kLongStream requests take the parallel offline path (WS_SIM_PAR: "0" = never,
  // "all" = every stream; both paths are exact and give identical counts)
  const char* par_env = getenv("WS_SIM_PAR");
  const char* th_env = getenv("WS_SIM_LONG");  // threshold override (requests), for tuning
  const long long long_th = par_env && par_env[0] == '0' ? LLONG_MAX
                            : (par_env && par_env[0] == 'a' ? 0 : (th_env ? atoll(th_env) : kLongStream));
  std::vector<DSimTrace> longs;
  const std::vector<DSimTrace> all_tr = tr;  // every stream (the WLD sets need the wave streams)
  for (DSimTrace& T : tr) {
    if (T.n >= (1ll << 31) - 1) return cleanup(-WS_ELIMIT);
    const DGpu& G = hg[cf[T.config].gpu_id];
    const int spl = 1 << (G.lg_line - G.lg_sector);
    long long bound = T.n;
    if (T.type == 1) bound = std::min<long long>(bound, (long long)est[T.config].wave_lines);
    if (T.type == 2) bound = std::min<long long>(bound, (long long)est[T.config].lz_lines);
    T.hcap = pow2_at_least(std::max<long long>(2, 2 * bound));
    req_total = std::max<long long>(req_total, T.req_off + T.n);
    if (T.n >= long_th && T.n > 0) {
      longs.push_back(T);
      T.n = -1;  // marked: removed from the warp path below
      continue;
    }
    T.m_off = spl;  // sectors per line (the offsets are assigned per batch below)
  }
  tr.erase(std::remove_if(tr.begin(), tr.end(), [](const DSimTrace& T) { return T.n < 0; }), tr.end());
  // warp-path state in batches of bounded device memory (streams are independent)
  const long long kBatchBytes = 8ll << 30;
  std::vector<std::pair<size_t, size_t>> batches;  // [first, last) into tr (sorted by n below)
  std::vector<int64_t> wld_off(2 * (size_t)n, 0);
  long long wld_total = 0;
  for (int c = 0; c < n; ++c) {
    const long long cap = pow2_at_least(std::max<long long>(2, 2 * (long long)est[c].wave_ld_sectors));
    wld_off[2 * c] = wld_total;
    wld_off[2 * c + 1] = cap;
    wld_total += cap;
  }
  std::sort(tr.begin(), tr.end(), [](const DSimTrace& a, const DSimTrace& b) { return a.n > b.n; });
  {
    size_t first = 0;
    long long fen_b = 0, slot_b = 0, m_b = 0;
    for (size_t t = 0; t < tr.size(); ++t) {
      DSimTrace& T = tr[t];
      const long long spl = T.m_off;
      const long long bytes = (T.n + 1) * 4 + T.hcap * 12 + T.hcap * spl * 8;
      if (t > first && (fen_b + T.n + 1) * 4 + slot_b * 12 + m_b * 8 + bytes > kBatchBytes) {
        batches.push_back({first, t});
        first = t;
        fen_b = slot_b = m_b = 0;
      }
      T.fen_off = fen_b;
      fen_b += T.n + 1;
      T.slot_off = slot_b;
      slot_b += T.hcap;
      T.m_off = m_b;
      m_b += T.hcap * spl;
      fen_total = std::max(fen_total, fen_b);
      slot_total = std::max(slot_total, slot_b);
      m_total = std::max(m_total, m_b);
    }
    if (first < tr.size()) batches.push_back({first, tr.size()});
  }
  // capacities: ascending, in lines (every GPU of the batch shares line_bytes? no: per record below)
  std::vector<int> idx(ncap);
  for (int k = 0; k < ncap; ++k) idx[k] = k;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return h_caps[a] < h_caps[b]; });
  std::vector<int> rank(ncap);
  std::vector<unsigned long long> lines(ncap);
  int lb = -1;
  for (const ws_config& c : cf)
    if (c.gpu_id < hg.size()) {
      if (lb >= 0 && lb != hg[c.gpu_id].lg_line) return cleanup(-WS_EINVAL);  // one line size per call
      lb = hg[c.gpu_id].lg_line;
    }
  if (lb < 0) lb = 7;
  for (int k = 0; k < ncap; ++k) {
    rank[idx[k]] = k;
    lines[k] = std::max<unsigned long long>(1ull, h_caps[idx[k]] >> lb);
  }
  mark("sizing");
  if ((rc = dmalloc(&S.req, (size_t)req_total, owned)) || (rc = dmalloc(&S.fen, (size_t)fen_total, owned)) ||
      (rc = dmalloc(&S.keys, (size_t)slot_total, owned)) || (rc = dmalloc(&S.last, (size_t)slot_total, owned)) ||
      (rc = dmalloc(&S.M, (size_t)m_total, owned)) || (rc = dmalloc(&S.SL, (size_t)m_total, owned)) ||
      (rc = dmalloc(&S.wld, (size_t)wld_total, owned)) || (rc = dmalloc(&S.wld_off, 2 * (size_t)n, owned)))
    return cleanup(rc);
  S.traces = d_tr;
  S.n_traces = n_traces;
  ws_sim_result* d_out;
  if ((rc = dmalloc(&d_out, (size_t)n * ncap, owned))) return cleanup(rc);
  mark("alloc+gen");
  cudaMemsetAsync(S.wld, 0xff, (size_t)wld_total * sizeof(unsigned long long), q);
  cudaMemsetAsync(S.acc, 0, (size_t)n * kSimAcc * sizeof(unsigned long long), q);
  cudaMemsetAsync(S.counter, 0, sizeof(unsigned long long), q);
  if (n_traces) cudaMemcpyAsync(d_tr, all_tr.data(), all_tr.size() * sizeof(DSimTrace), cudaMemcpyHostToDevice, q);
  cudaMemcpyAsync(S.wld_off, wld_off.data(), wld_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice, q);
  cudaMemcpyAsync(S.lines, lines.data(), ncap * sizeof(unsigned long long), cudaMemcpyHostToDevice, q);
  cudaMemcpyAsync(d_caps, h_caps, ncap * sizeof(uint64_t), cudaMemcpyHostToDevice, q);
  cudaMemcpyAsync(d_rank, rank.data(), ncap * sizeof(int), cudaMemcpyHostToDevice, q);
  if (n_items > 0) {
    k_sim_warp<true><<<grid, 256, 0, q>>>(s.plans, d_k, d_g, s.instr, S.order, S.item_pre, n, n_items, d_cnt, S.req);
    k_sim_wld<<<dim3(64, (unsigned)std::min<long long>(n_traces, 4096)), 256, 0, q>>>(d_tr, n_traces, S.req, S.wld,
                                                                                   S.wld_off);
    L += 2;
  }
  if (ev) {
    cudaEventRecord(ev[1], q);
    cudaEventRecord(ev[2], q);
  }
  // warp path: the short streams, batch by batch
  for (const auto& bt : batches) {
    S.n_traces = (int64_t)(bt.second - bt.first);
    cudaMemsetAsync(S.fen, 0, (size_t)fen_total * sizeof(uint32_t), q);
    cudaMemsetAsync(S.keys, 0xff, (size_t)slot_total * sizeof(unsigned long long), q);
    cudaMemsetAsync(S.counter, 0, sizeof(unsigned long long), q);
    cudaMemcpyAsync(d_tr, tr.data() + bt.first, (size_t)S.n_traces * sizeof(DSimTrace), cudaMemcpyHostToDevice, q);
    k_sim_run<<<n_sm_dev * 4, kSimWarps * 32, 0, q>>>(s.plans, d_g, S, ncap);
    ++L;
    if ((rc = (int)cudaStreamSynchronize(q))) return cleanup(rc);  // the host copy of tr is reused
  }
  // parallel path: the long streams, concatenated in batches (positions < 2^31), device-wide kernels
  mark("warp path");
  if (!longs.empty()) {
    std::vector<std::pair<size_t, size_t>> pbat;
    {
      // positions per batch: < 2^31, and within 85 % of the free device memory at ~72 bytes
      // per position (request copy, ids, radix buffers, wavelet values and levels, distances,
      // flags) plus the streams' hash tables
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const long long kPosBytes = 72;
      const long long cap_mem = (long long)(0.85 * (double)free_b);
      size_t first = 0;
      long long tot_n = 0, tot_h = 0;
      for (size_t t = 0; t < longs.size(); ++t) {
        const long long n2 = tot_n + longs[t].n, h2 = tot_h + longs[t].hcap;
        if (t > first && (n2 >= (1ll << 31) - 2 || t - first >= 4096 || n2 * kPosBytes + h2 * 12 > cap_mem)) {
          pbat.push_back({first, t});
          first = t;
          tot_n = tot_h = 0;
        }
        tot_n += longs[t].n;
        tot_h += longs[t].hcap;
      }
      pbat.push_back({first, longs.size()});
    }
    long long nmax = 0, hmax = 0;
    size_t tmax = 0;
    for (const auto& bt : pbat) {
      long long nb = 0, hb = 0;
      for (size_t t = bt.first; t < bt.second; ++t) {
        nb += longs[t].n;
        hb += longs[t].hcap;
      }
      nmax = std::max<long long>(nmax, nb);
      hmax = std::max<long long>(hmax, hb);
      tmax = std::max<size_t>(tmax, bt.second - bt.first);
    }
    const long long nwmax = (nmax + 63) / 64 + 1;
    int LVmax = 1;
    while ((1ll << LVmax) <= nmax) ++LVmax;
    unsigned long long *H, *cat;
    ulonglong2* wr;
    uint32_t *occ, *key, *val, *key2, *val2, *V, *cur, *nxt, *wz, *bsum, *tot, *Zs, *dist, *isl, *lst, *hist, *tidv;
    unsigned char* sidx;
    DPB* d_pb;
    const long long ntmax = (nmax + kRsTile - 1) / kRsTile;
    const long long nbmax = (std::max(std::max(nmax + 1, hmax), 256 * ntmax) + kScanB - 1) / kScanB + 1;
    if ((rc = dmalloc(&H, (size_t)hmax, owned)) || (rc = dmalloc(&occ, (size_t)hmax, owned)) ||
        (rc = dmalloc(&key, (size_t)nmax, owned)) || (rc = dmalloc(&val, (size_t)nmax, owned)) ||
        (rc = dmalloc(&key2, (size_t)nmax, owned)) || (rc = dmalloc(&val2, (size_t)nmax, owned)) ||
        (rc = dmalloc(&V, (size_t)nmax, owned)) || (rc = dmalloc(&cur, (size_t)nmax, owned)) ||
        (rc = dmalloc(&nxt, (size_t)nmax, owned)) || (rc = dmalloc(&wz, (size_t)nwmax, owned)) ||
        (rc = dmalloc(&bsum, (size_t)nbmax, owned)) || (rc = dmalloc(&tot, 8, owned)) ||
        (rc = dmalloc(&wr, (size_t)(LVmax * nwmax), owned)) ||
        (rc = dmalloc(&Zs, (size_t)LVmax, owned)) || (rc = dmalloc(&dist, (size_t)nmax, owned)) ||
        (rc = dmalloc(&isl, (size_t)nmax + 1, owned)) || (rc = dmalloc(&lst, (size_t)hmax + 1, owned)) ||
        (rc = dmalloc(&hist, (size_t)(256 * ntmax), owned)) || (rc = dmalloc(&sidx, (size_t)nmax, owned)) ||
        (rc = dmalloc(&cat, (size_t)nmax, owned)) || (rc = dmalloc(&tidv, (size_t)nmax, owned)) ||
        (rc = dmalloc(&d_pb, tmax, owned)))
      return cleanup(rc);
    mark("long alloc");
    auto scan = [&](uint32_t* io, long long m, uint32_t* total) {
      const long long nb = (m + kScanB - 1) / kScanB;
      k_ps_reduce<<<(unsigned)nb, 256, 0, q>>>(io, m, bsum);
      k_ps_bsum<<<1, 1024, 0, q>>>(bsum, nb, total);
      k_ps_apply<<<(unsigned)nb, 256, 0, q>>>(io, m, bsum);
    };
    const unsigned gridN = (unsigned)(n_sm_dev * 8);
    for (const auto& bt : pbat) {
      std::vector<DPB> hp;
      long long nn = 0, hcap = 0, Ubound = 0, lmax = 0;
      for (size_t t = bt.first; t < bt.second; ++t) {
        const DSimTrace& T = longs[t];
        const DGpu& G = hg[cf[T.config].gpu_id];
        DPB P;
        P.req_off = T.req_off;
        P.n = T.n;
        P.start = nn;
        P.hoff = hcap;
        P.hcap = T.hcap;
        P.t_y_abs = nn + T.t_y;
        P.wld_off = wld_off[2 * T.config];
        P.wld_cap = wld_off[2 * T.config + 1];
        P.type = T.type;
        P.config = T.config;
        P.lspl = G.lg_line - G.lg_sector;
        P.spl = 1 << P.lspl;
        hp.push_back(P);
        nn += T.n;
        hcap += T.hcap;
        Ubound += T.hcap / 2;  // hcap >= 2 * (an upper bound of the stream's distinct lines)
        lmax = std::max<long long>(lmax, T.n);
      }
      const int ntr = (int)hp.size();
      // pageable host memory: the copy completes before the call returns, hp may go out of scope
      cudaMemcpyAsync(d_pb, hp.data(), hp.size() * sizeof(DPB), cudaMemcpyHostToDevice, q);
      k_pb_gather<<<dim3((unsigned)std::min<long long>((lmax + 255) / 256, 4096), (unsigned)ntr), 256, 0, q>>>(
          S.req, d_pb, cat, tidv);
      cudaMemsetAsync(H, 0xff, (size_t)hcap * sizeof(unsigned long long), q);
      k_pb_insert<<<gridN, 256, 0, q>>>(cat, tidv, nn, d_pb, H);
      k_pl_occ<<<gridN, 256, 0, q>>>(H, hcap, occ);
      scan(occ, hcap, tot);  // tot[0] = distinct (stream, line) pairs U
      k_pb_ids<<<gridN, 256, 0, q>>>(cat, tidv, nn, d_pb, H, occ, key, val, sidx);
      int bits = 1;
      while ((1ll << bits) < Ubound) ++bits;
      const long long ntiles = (nn + kRsTile - 1) / kRsTile;
      uint32_t *ka = key, *va = val, *kb = key2, *vb = val2;
      for (int sh = 0; sh < bits; sh += 8) {
        k_rs_hist<<<(unsigned)ntiles, 256, 0, q>>>(ka, nn, sh, hist, ntiles);
        scan(hist, 256 * ntiles, tot + 1);
        k_rs_scatter<<<(unsigned)ntiles, 256, 0, q>>>(ka, va, nn, sh, hist, ntiles, kb, vb);
        std::swap(ka, kb);
        std::swap(va, vb);
      }
      k_pl_prev<<<gridN, 256, 0, q>>>(ka, va, nn, V, lst);
      k_pl_split<<<gridN, 256, 0, q>>>(V, nn, isl);
      int LV = 1;
      while ((1ll << LV) <= nn) ++LV;
      const long long nw = (nn + 63) / 64 + 1;
      uint32_t *c1 = V, *c2 = cur;  // level 0 reads V (kept for k_pl_dist), then cur <-> nxt
      for (int lev = 0; lev < LV; ++lev) {
        const int bit = LV - 1 - lev;
        ulonglong2* Wl = wr + (long long)lev * nw;
        k_wm_bits<<<gridN, 256, 0, q>>>(c1, nn, bit, Wl, wz);
        scan(wz, nw - 1, Zs + lev);  // zeros before each word; Z = all zeros of the level
        k_wm_next<<<gridN, 256, 0, q>>>(c1, nn, bit, wz, Zs + lev, c2);
        k_wm_rank<<<gridN, 256, 0, q>>>(Wl, nw, wz, Zs + lev);
        c1 = c2;
        c2 = c2 == cur ? nxt : cur;
      }
      k_pl_dist<<<gridN, 256, 0, q>>>(V, nn, LV, wr, Zs, nw, S.lines, dist);
      scan(isl, nn, isl + nn);  // exclusive prefix of the last-access flags; isl[nn] = total
      k_pb_lines<<<(unsigned)((Ubound + 127) / 128), 128, 0, q>>>(va, lst, tot, nn, sidx, dist, cat, tidv, isl, d_pb,
                                                                   S.wld, S.lines, ncap, S.acc);
      if ((rc = check_launch())) return cleanup(rc);
      if ((rc = (int)cudaStreamSynchronize(q))) return cleanup(rc);  // d_pb / buffers reused by the next batch
    }
  }
  if (ev) cudaEventRecord(ev[3], q);
  k_sim_out<<<(unsigned)(((long long)n * ncap + 127) / 128), 128, 0, q>>>(s.plans, d_g, d_est, n, S.acc, ncap, d_caps,
                                                                          d_rank, d_out);
  ++L;
  if ((rc = check_launch())) return cleanup(rc);
  cudaMemcpyAsync(h_out, d_out, (size_t)n * ncap * sizeof(ws_sim_result), cudaMemcpyDeviceToHost, q);
  if (launches) *launches = L;
  return cleanup((int)cudaStreamSynchronize(q));
}

int run_fit(const double* h_O, const double* h_R, int n, double* h_out, cudaStream_t q, cudaEvent_t* ev) {
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, (2 * (size_t)n + 4) * sizeof(double));
  if (e != cudaSuccess) return (int)e;
  cudaMemcpyAsync(d, h_O, n * sizeof(double), cudaMemcpyHostToDevice, q);
  cudaMemcpyAsync(d + n, h_R, n * sizeof(double), cudaMemcpyHostToDevice, q);
  if (ev) cudaEventRecord(ev[0], q);
  k_fit<<<1, 256, 0, q>>>(d, d + n, n, d + 2 * n);
  if (ev) cudaEventRecord(ev[1], q);
  int rc = check_launch();
  cudaMemcpyAsync(h_out, d + 2 * n, 4 * sizeof(double), cudaMemcpyDeviceToHost, q);
  cudaError_t e2 = cudaStreamSynchronize(q);
  cudaFree(d);
  return rc ? rc : (int)e2;
}

}  // namespace wsb
