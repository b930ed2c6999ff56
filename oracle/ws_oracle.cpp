// oracle/ws_oracle.cpp -- plain, slow CPU oracle of the Warpspeed estimator.
//
// TEST INFRASTRUCTURE ONLY (see ws_oracle.h).  Nothing here is shared with
// the CUDA path.  Each function names the passage of PAPER.md (P:line) or the
// reading of SURVEY.md section 8(c) (Qnn) it writes out.  The structure
// follows SURVEY.md 8(c) "Specification of the integer core" steps O1..O10.
//
// Deliberately naive: every (thread, instruction) address of every scope is
// generated and inserted into std::set; counts are set sizes; overlaps are
// std::set_intersection sizes.
#include "ws_oracle.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <iterator>
#include <list>
#include <map>
#include <set>
#include <thread>
#include <utility>
#include <vector>

namespace {

typedef std::array<int64_t, 3> V3;
typedef std::pair<int64_t, int64_t> Key;  // (field, sector or line): fields never alias

int64_t floordiv(int64_t a, int64_t b) {  // floor(a / b), b > 0  ("floor divide")
  int64_t q = a / b;
  if ((a % b) != 0 && (a < 0)) q -= 1;
  return q;
}
int64_t floormod(int64_t a, int64_t b) { return a - floordiv(a, b) * b; }
int64_t ceildiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- O4: address map
// A = align + elem * sum_d pitch[d] * cell[d]   (P:157-161 with the base pointer
// replaced by the field alignment; worked example P:540-545).
int64_t address(const wso_field& f, const V3& cell) {
  return f.align_bytes + f.elem_bytes * (f.pitch[0] * cell[0] + f.pitch[1] * cell[1] + f.pitch[2] * cell[2]);
}

// ---------------------------------------------------------------- O5 pieces
// Number of distinct 32 B sectors among addresses (CL32Visitor).
int64_t unique_sectors(const std::vector<int64_t>& a, int64_t sector_bytes) {
  std::set<int64_t> s;
  for (int64_t x : a) s.insert(floordiv(x, sector_bytes));
  return (int64_t)s.size();
}

// Wavefronts of one half-warp instruction (Listing lst:griditeration
// BankConflictVisitor P:408-417 with the far-address rule P:393-395; Q2-Q4):
//   U = sorted unique bank words (A div bank_bytes)
//   split U greedily into clusters; a new cluster starts at u when
//   (u - cluster_start) * bank_bytes >= pair_window_bytes
//   cycles = sum over clusters of max over banks of |{u in cluster : u mod n_banks = bank}|
int64_t halfwarp_wavefronts(const std::vector<int64_t>& a, const wso_gpu& g) {
  std::set<int64_t> U;
  for (int64_t x : a) U.insert(floordiv(x, g.bank_bytes));
  int64_t cycles = 0;
  std::vector<int64_t> banks(g.n_banks, 0);
  bool open = false;
  int64_t start = 0;
  for (int64_t u : U) {
    if (open && (u - start) * g.bank_bytes >= g.pair_window_bytes) {
      cycles += *std::max_element(banks.begin(), banks.end());
      std::fill(banks.begin(), banks.end(), 0);
      open = false;
    }
    if (!open) { start = u; open = true; }
    banks[floormod(u, g.n_banks)] += 1;
  }
  if (open) cycles += *std::max_element(banks.begin(), banks.end());
  return cycles;
}

// Gompertz-form hit rate R(O) = a * exp(-b * exp(-c * O))
double hit_rate(const double abc[3], double O) { return abc[0] * std::exp(-abc[1] * std::exp(-abc[2] * O)); }

int64_t log2_exact(int64_t v) {
  int64_t l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return ((int64_t(1) << l) == v) ? l : -1;
}

// ---------------------------------------------------------------- O1: validation
int64_t check_kernel(const wso_kernel& K) {
  if (K.n_fields < 1 || K.n_fields > 64 || K.n_accesses < 1 || K.n_accesses > 128) return WSO_EINVAL;
  for (int64_t i = 0; i < K.n_fields; ++i) {
    const wso_field& f = K.fields[i];
    if (log2_exact(f.elem_bytes) < 0 || f.elem_bytes > 32) return WSO_EINVAL;
    // elements never straddle a sector: the alignment is a multiple of the element size
    // (WS_EINVAL otherwise; every sector count below keys an element by its first byte)
    if (floormod(f.align_bytes, f.elem_bytes) != 0) return WSO_EINVAL;
    for (int d = 0; d < 3; ++d)
      if (f.extent[d] < 1) return WSO_EINVAL;
    // x contiguous, rows and planes disjoint (row-major, padding allowed)
    if (f.pitch[0] != 1 || f.pitch[1] < f.extent[0] || f.pitch[2] < f.pitch[1] * f.extent[1]) return WSO_EINVAL;
  }
  for (int d = 0; d < 3; ++d)
    if (K.dom_lo[d] < 0 || K.dom_hi[d] <= K.dom_lo[d]) return WSO_EINVAL;
  for (int64_t i = 0; i < K.n_accesses; ++i) {
    const wso_access& a = K.accesses[i];
    if (a.field < 0 || a.field >= K.n_fields || (a.is_store != 0 && a.is_store != 1)) return WSO_EINVAL;
    const wso_field& f = K.fields[a.field];
    for (int d = 0; d < 3; ++d)  // every active cell + offset stays inside the field
      if (K.dom_lo[d] + a.off[d] < 0 || K.dom_hi[d] - 1 + a.off[d] >= f.extent[d]) return WSO_EBOUNDS;
  }
  return WSO_OK;
}

// ---------------------------------------------------------------- O3: instruction table
// One instruction per distinct (field, kind, kappa + o) over the fold cube
// kappa in [0,f) and the accesses o of that field and kind (Q7).
struct Instr {
  int64_t field, is_store;
  V3 r;
  std::vector<V3> kappas;  // {kappa in [0,f) : r - kappa is an access offset of (field, kind)}
};

struct Plan {
  V3 b, f, lo, hi, G;
  int64_t T, N, k, W, s, n_sets, Ly0, Lz0;
  bool mdim;  // multidimensional address space for the wave / layer-set footprints
  std::vector<Instr> instr;
};

bool in_offsets(const wso_kernel& K, int64_t field, int64_t is_store, const V3& o) {
  for (int64_t i = 0; i < K.n_accesses; ++i) {
    const wso_access& a = K.accesses[i];
    if (a.field == field && a.is_store == is_store && a.off[0] == o[0] && a.off[1] == o[1] && a.off[2] == o[2])
      return true;
  }
  return false;
}

// Block id -> block coordinates in X-Y-Z scheduling order.
V3 block_coord(const Plan& p, int64_t B) { return V3{B % p.G[0], (B / p.G[0]) % p.G[1], B / (p.G[0] * p.G[1])}; }
// Thread index -> thread coordinates, tid = tx + bx*(ty + by*tz).
V3 thread_coord(const Plan& p, int64_t t) { return V3{t % p.b[0], (t / p.b[0]) % p.b[1], t / (p.b[0] * p.b[1])}; }
// Base cell of a thread: lo + (blockcoord * b + threadcoord) * f; it computes cells base + kappa.
V3 base_cell(const Plan& p, int64_t B, int64_t t) {
  V3 bc = block_coord(p, B), tc = thread_coord(p, t), c;
  for (int d = 0; d < 3; ++d) c[d] = p.lo[d] + (bc[d] * p.b[d] + tc[d]) * p.f[d];
  return c;
}
bool active(const Plan& p, const V3& cell) {  // guard clipping by the domain
  for (int d = 0; d < 3; ++d)
    if (cell[d] >= p.hi[d]) return false;
  return true;
}
// Thread issues instruction r iff some active folded cell base+kappa has
// r - kappa among the accesses of that field and kind (Q27).  The kappas with
// r - kappa an access offset are listed once per instruction (I.kappas).
bool issues(const Plan& p, const V3& base, const Instr& I) {
  for (const V3& kap : I.kappas)
    if (active(p, V3{base[0] + kap[0], base[1] + kap[1], base[2] + kap[2]})) return true;
  return false;
}
int64_t instr_address(const wso_kernel& K, const V3& base, const Instr& I) {
  V3 cell{base[0] + I.r[0], base[1] + I.r[1], base[2] + I.r[2]};
  return address(K.fields[I.field], cell);
}

// ---------------------------------------------------------------- O2: geometry
int64_t make_plan(const wso_kernel& K, const wso_gpu& g, const wso_config& c, Plan& p, wso_result& r) {
  for (int d = 0; d < 3; ++d) {
    if (c.block[d] < 1 || c.fold[d] < 1) return WSO_EINVAL;
    p.b[d] = c.block[d];
    p.f[d] = c.fold[d];
    p.lo[d] = K.dom_lo[d];
    p.hi[d] = K.dom_hi[d];
  }
  for (int64_t i = 0; i < K.n_fields; ++i)
    if (K.fields[i].elem_bytes > g.sector_bytes) return WSO_EINVAL;
  p.T = p.b[0] * p.b[1] * p.b[2];
  if (p.T > g.max_thr_blk) return WSO_ELIMIT;
  if (p.f[0] * p.f[1] * p.f[2] > 64) return WSO_ELIMIT;
  for (int d = 0; d < 3; ++d) p.G[d] = ceildiv(p.hi[d] - p.lo[d], p.b[d] * p.f[d]);
  p.N = p.G[0] * p.G[1] * p.G[2];
  // Resident blocks per SM (Q10): threads, blocks and registers,
  // allocated at warp granularity.
  if (c.variant < 0 || c.variant > 15) return WSO_EINVAL;
  p.mdim = (c.variant & WSO_VAR_MDIM) != 0;
  if (c.blocks_per_sm > 0) {
    p.k = c.blocks_per_sm;
  } else {
    int64_t Ta = ceildiv(p.T, 32) * 32;
    p.k = std::min(g.max_thr_sm / Ta, g.max_blk_sm);
    if (K.regs_per_thread > 0) p.k = std::min(p.k, g.regs_sm / (K.regs_per_thread * Ta));
  }
  if (p.k < 1) return WSO_ELIMIT;
  // Wave: W resident blocks; representative wave centred on the grid's
  // central block (Q11).
  p.W = std::min(p.N, g.n_sm * p.k);
  int64_t cen = p.G[0] / 2 + p.G[0] * (p.G[1] / 2 + p.G[1] * (p.G[2] / 2));
  p.s = std::min(std::max(cen - p.W / 2, int64_t(0)), p.N - p.W);
  p.n_sets = std::min(g.n_sm, p.W);
  // Layer thread sets: everything scheduled since the wave's y-neighbour block
  // row / z-neighbour block layer (Q13).
  p.Ly0 = std::max(int64_t(0), p.s - p.G[0]);
  p.Lz0 = std::max(int64_t(0), p.s - p.G[0] * p.G[1]);
  // Variant (NEXT-3): the V100 / SBAC model looks back exactly one wave:
  // both look-back sets become the directly preceding wave [s - W, s).
  if (c.variant & WSO_VAR_PREV_WAVE) p.Ly0 = p.Lz0 = std::max(int64_t(0), p.s - p.W);
  // O3: instruction table
  for (int64_t fi = 0; fi < K.n_fields; ++fi)
    for (int64_t st = 0; st < 2; ++st) {
      std::set<V3> R;
      for (int64_t i = 0; i < K.n_accesses; ++i) {
        const wso_access& a = K.accesses[i];
        if (a.field != fi || a.is_store != st) continue;
        for (int64_t kz = 0; kz < p.f[2]; ++kz)
          for (int64_t ky = 0; ky < p.f[1]; ++ky)
            for (int64_t kx = 0; kx < p.f[0]; ++kx) R.insert(V3{kx + a.off[0], ky + a.off[1], kz + a.off[2]});
      }
      for (const V3& rr : R) {
        Instr I{fi, st, rr, {}};
        for (int64_t kz = 0; kz < p.f[2]; ++kz)
          for (int64_t ky = 0; ky < p.f[1]; ++ky)
            for (int64_t kx = 0; kx < p.f[0]; ++kx)
              if (in_offsets(K, fi, st, V3{rr[0] - kx, rr[1] - ky, rr[2] - kz})) I.kappas.push_back(V3{kx, ky, kz});
        p.instr.push_back(I);
      }
    }
  if (p.instr.size() > 1024) return WSO_ELIMIT;
  r.grid[0] = p.G[0];
  r.grid[1] = p.G[1];
  r.grid[2] = p.G[2];
  r.k = p.k;
  r.wave_blocks = p.W;
  r.n_smsets = p.n_sets;
  r.wave_first_block = p.s;
  r.n_instr = (int64_t)p.instr.size();
  return WSO_OK;
}

// Footprint key of the wave / layer-set scopes: (field, z, y, x-sector).  Linear address
// space: (field, 0, 0, A div sector_bytes).  Multidimensional address space:
// two addresses are distinct when their tuples differ; the innermost dimension keeps the
// floor division by the fetch granularity, the array alignment is not considered
// ("the alignment of arrays cannot be considered").
typedef std::array<int64_t, 4> K4;
K4 scope_key(const wso_kernel& K, const wso_gpu& g, const Plan& p, const V3& base, const Instr& I) {
  if (!p.mdim) return K4{I.field, 0, 0, floordiv(instr_address(K, base, I), g.sector_bytes)};
  V3 cell{base[0] + I.r[0], base[1] + I.r[1], base[2] + I.r[2]};
  return K4{I.field, cell[2], cell[1], floordiv(cell[0] * K.fields[I.field].elem_bytes, g.sector_bytes)};
}
// sector key -> line key (128 / 32 = 4 sectors per line, floor(floor(a/32)/4) = floor(a/128))
K4 line_of(const K4& k, int64_t sec_per_line) { return K4{k[0], k[1], k[2], floordiv(k[3], sec_per_line)}; }

template <class S>
size_t intersection_size(const S& a, const S& b) {
  std::vector<typename S::value_type> out;
  std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(out));
  return out.size();
}

// F_L: every sector touched by any instruction (loads and stores) of the
// blocks [B0, B1) (Q15: L2 is write-back, stored data can be hit).
std::set<K4> layer_footprint(const wso_kernel& K, const wso_gpu& g, const Plan& p, int64_t B0, int64_t B1) {
  std::set<K4> F;
  for (int64_t B = B0; B < B1; ++B)
    for (int64_t t = 0; t < p.T; ++t) {
      V3 base = base_cell(p, B, t);
      for (const Instr& I : p.instr)
        if (issues(p, base, I)) F.insert(scope_key(K, g, p, base, I));
    }
  return F;
}

int64_t estimate(const wso_kernel& K, const wso_gpu& g, const wso_config& c, wso_result& r) {
  r = wso_result();
  int64_t st = check_kernel(K);
  Plan p;
  if (st == WSO_OK) st = make_plan(K, g, c, p, r);
  if (st != WSO_OK) {
    wso_result z = wso_result();
    z.status = st;
    r = z;
    return st;
  }
  const int64_t sec_per_line = g.line_bytes / g.sector_bytes;

  // ------------------------------------------------------------ O5-O7 over the wave
  int64_t wf = 0, req_ld = 0, req_st = 0, lup = 0;
  std::vector<std::set<Key>> SMsec(p.n_sets), SMlin(p.n_sets);
  std::set<K4> WLD, WST, WLIN;
  // NEXT-4: TLB pages of the wave and the per-L2-section footprints
  // (P:322-329), always in the linear (physical) address space.  SM j is
  // attached to section floor(j * S / n_sm); block B runs on SM (B - s) mod n_sm (Q9).
  const int64_t S = g.l2_sections;
  std::set<Key> PAGES;
  std::vector<std::set<Key>> SECld(S), SEClin(S);
  const int64_t n_warps = ceildiv(p.T, 32);
  // Variant (NEXT-3): L1 scopes from one representative block (the wave's middle
  // block) standing for every wave block: no L1 sharing between co-resident blocks, volumes and
  // cycles = W x the block's, lattice updates = W x the block's.
  const bool rep = (c.variant & WSO_VAR_REP_BLOCK) != 0;
  const int64_t B_rep = p.s + p.W / 2;
  // a3 / a4 contributions of one warp instruction of block B (issuing lanes' addresses A)
  auto lanes_of = [&](int64_t B, int64_t w, const Instr& I, int64_t h0, int64_t h1) {
    std::vector<int64_t> A;
    for (int64_t lane = h0; lane < h1; ++lane) {
      int64_t t = w * 32 + lane;
      if (t >= p.T) break;
      V3 base = base_cell(p, B, t);
      if (issues(p, base, I)) A.push_back(instr_address(K, base, I));
    }
    return A;
  };
  auto l1_instr = [&](int64_t B, int64_t w, const Instr& I, const std::vector<int64_t>& A, int64_t j) {
    // warp instruction: unique sectors over issuing lanes (Q5);
    // stores are written through and counted per instruction
    if (I.is_store) req_st += unique_sectors(A, g.sector_bytes);
    else req_ld += unique_sectors(A, g.sector_bytes);
    // half-warps: wavefronts (Q6: loads and stores)
    for (int64_t h = 0; h < 32 / g.half_warp; ++h)
      wf += halfwarp_wavefronts(lanes_of(B, w, I, h * g.half_warp, (h + 1) * g.half_warp), g);
    if (!I.is_store)
      for (int64_t a : A) {
        SMsec[j].insert(Key(I.field, floordiv(a, g.sector_bytes)));  // L1: SM-resident set (Q8)
        SMlin[j].insert(Key(I.field, floordiv(a, g.line_bytes)));    // 128 B allocation (Q18)
      }
  };
  auto block_lup = [&](int64_t B) {  // active cells = lattice updates of the block
    int64_t n = 0;
    for (int64_t t = 0; t < p.T; ++t) {
      V3 base = base_cell(p, B, t);
      for (int64_t kz = 0; kz < p.f[2]; ++kz)
        for (int64_t ky = 0; ky < p.f[1]; ++ky)
          for (int64_t kx = 0; kx < p.f[0]; ++kx)
            if (active(p, V3{base[0] + kx, base[1] + ky, base[2] + kz})) ++n;
    }
    return n;
  };
  for (int64_t B = p.s; B < p.s + p.W; ++B) {
    const int64_t j = (B - p.s) % g.n_sm;  // round-robin SM assignment (Q9)
    const int64_t sec = j * S / g.n_sm;      // L2 section of that SM
    if (!rep) lup += block_lup(B);
    for (int64_t w = 0; w < n_warps; ++w) {
      for (const Instr& I : p.instr) {
        std::vector<int64_t> A = lanes_of(B, w, I, 0, 32);
        if (!rep) l1_instr(B, w, I, A, j);
        for (int64_t a : A) {
          Key ks(I.field, floordiv(a, g.sector_bytes)), kl(I.field, floordiv(a, g.line_bytes));
          if (!I.is_store) SECld[sec].insert(ks);
          SEClin[sec].insert(kl);
          if (g.page_bytes > 0) PAGES.insert(Key(I.field, floordiv(a, g.page_bytes)));
        }
        // wave scope keys (linear or multidimensional address space)
        for (int64_t lane = 0; lane < 32; ++lane) {
          int64_t t = w * 32 + lane;
          if (t >= p.T) break;
          V3 base = base_cell(p, B, t);
          if (!issues(p, base, I)) continue;
          K4 k4 = scope_key(K, g, p, base, I);
          if (!I.is_store) WLD.insert(k4);  // wave load footprint
          else WST.insert(k4);              // wave store footprint
          WLIN.insert(line_of(k4, sec_per_line));
        }
      }
    }
  }
  if (rep) {
    lup = p.W * block_lup(B_rep);
    for (int64_t w = 0; w < n_warps; ++w)
      for (const Instr& I : p.instr) l1_instr(B_rep, w, I, lanes_of(B_rep, w, I, 0, 32), 0);
    wf *= p.W;
    req_ld *= p.W;
    req_st *= p.W;
  }
  int64_t sm_sec = 0, sm_lin = 0;
  for (int64_t j = 0; j < p.n_sets; ++j) {
    sm_sec += (int64_t)SMsec[j].size();
    sm_lin += (int64_t)SMlin[j].size();
  }
  if (rep) {  // W blocks, each with the representative block's footprint (no sharing)
    sm_sec *= p.W;
    sm_lin *= p.W;
  }

  // ------------------------------------------------------------ O8 layer sets
  std::set<K4> Fy = layer_footprint(K, g, p, p.Ly0, p.s);
  std::set<K4> Fz = layer_footprint(K, g, p, p.Lz0, p.s);
  std::set<K4> Fy_lines, Fz_lines;
  for (const K4& k : Fy) Fy_lines.insert(line_of(k, sec_per_line));
  for (const K4& k : Fz) Fz_lines.insert(line_of(k, sec_per_line));

  // NEXT-4: duplication = copies beyond the first of a line held by several sections;
  // link volume = load sectors fetched by more than one section (one far-section copy each).
  std::set<Key> Uld, Ulin;
  int64_t sum_ld = 0, sum_lin = 0;
  for (int64_t i = 0; i < S; ++i) {
    sum_ld += (int64_t)SECld[i].size();
    sum_lin += (int64_t)SEClin[i].size();
    Uld.insert(SECld[i].begin(), SECld[i].end());
    Ulin.insert(SEClin[i].begin(), SEClin[i].end());
  }
  r.wave_pages = (int64_t)PAGES.size();
  // reported on request (ABI): several sections and the link limiter or WSO_VAR_L2_DUP
  const bool want_sect = S > 1 && (g.link_bw > 0 || (c.variant & WSO_VAR_L2_DUP));
  r.l2_dup_lines = want_sect ? sum_lin - (int64_t)Ulin.size() : 0;
  r.l2_link_sectors = want_sect ? sum_ld - (int64_t)Uld.size() : 0;

  r.lup_wave = lup;
  r.l1_wavefronts = wf;
  r.l1_req_ld_sectors = req_ld;
  r.l1_req_st_sectors = req_st;
  r.sm_ld_sectors = sm_sec;
  r.sm_ld_lines = sm_lin;
  r.wave_ld_sectors = (int64_t)WLD.size();
  r.wave_st_sectors = (int64_t)WST.size();
  r.wave_lines = (int64_t)WLIN.size();
  r.ly_lines = (int64_t)Fy_lines.size();
  r.lz_lines = (int64_t)Fz_lines.size();
  r.ov_y = (int64_t)intersection_size(WLD, Fy);
  r.ov_z = (int64_t)intersection_size(WLD, Fz);
  r.addr_evals = (p.W + (p.s - p.Lz0)) * p.T * (int64_t)p.instr.size();

  // ------------------------------------------------------------ O9 model (FP64)
  // Volumes in sectors; x sector_bytes gives bytes.
  const double SB = (double)g.sector_bytes, LB = (double)g.line_bytes;
  const double n = (double)lup;
  // L1 level: Eq.4 O = V_alloc / V_cache with V_alloc the mean SM-set line
  // footprint; Eq.2/3/5: V_down = V_comp + (1 - R) * (V_up - V_comp).
  r.O_l1 = ((double)sm_lin * LB / (double)p.n_sets) / (double)g.l1_bytes;
  r.R_l1 = hit_rate(g.hit_abc[0], r.O_l1);
  double v_red_l1 = std::max(0.0, (double)req_ld - (double)sm_sec);
  double l2l1_ld = (double)sm_sec + (1.0 - r.R_l1) * v_red_l1;
  double l1l2_st = (double)req_st;  // write-through
  // L2 level: effective capacity of one section (Q31)
  double l2eff = (double)g.l2_bytes / (double)g.l2_sections;
  // Variant (NEXT-4): instead of assuming full duplication (capacity / S),
  // the capacity holds |Ulin| + dup line copies for |Ulin| distinct lines.
  if ((c.variant & WSO_VAR_L2_DUP) && !Ulin.empty())
    l2eff = (double)g.l2_bytes * (double)Ulin.size() / (double)(Ulin.size() + r.l2_dup_lines);
  r.l2_eff_bytes = l2eff;
  r.O_y = (double)Fy_lines.size() * LB / l2eff;
  r.O_z = (double)Fz_lines.size() * LB / l2eff;
  r.R_y = hit_rate(g.hit_abc[1], r.O_y);
  r.R_z = hit_rate(g.hit_abc[2], r.O_z);
  double hits = r.R_y * (double)r.ov_y + r.R_z * (double)(r.ov_z - r.ov_y);  // Q16
  // stores: redundant partial stores missing in L2 are read back (Q19)
  double red_st = std::max(0.0, (double)req_st - (double)r.wave_st_sectors);
  r.O_st = (double)r.wave_lines * LB / l2eff;
  r.R_st = hit_rate(g.hit_abc[3], r.O_st);
  double cap_st = (1.0 - r.R_st) * red_st;
  double dram_ld = (double)r.wave_ld_sectors - hits + cap_st;
  double dram_st = (double)r.wave_st_sectors;
  // per lattice update
  r.l1_cyc_per_lup = (double)wf / n;
  r.l2_ld_Bpl = SB * l2l1_ld / n;
  r.l2_st_Bpl = SB * l1l2_st / n;
  r.dram_ld_Bpl = SB * dram_ld / n;
  r.dram_st_Bpl = SB * dram_st / n;
  // limiters (Q1): seconds per lattice update
  r.t_l1 = (double)wf / (n * (double)g.n_sm * g.clock_hz);
  r.t_l2 = SB * (l2l1_ld + l1l2_st) / (n * g.l2_bw);
  r.t_dram = SB * (dram_ld + dram_st) / (n * g.dram_bw);
  // inter-section link as an additional L2 limiter, when its bandwidth is given
  r.t_link = g.link_bw > 0 ? SB * (double)r.l2_link_sectors / (n * g.link_bw) : 0.0;
  double t = std::max(std::max(r.t_l1, r.t_link), std::max(r.t_l2, r.t_dram));
  // limiter: argmax, ties resolved DRAM > L2 > link > L1 (Q29)
  r.limiter = (r.t_dram >= t) ? 2 : (r.t_l2 >= t) ? 1 : (r.t_link >= t) ? 3 : 0;
  double cells = 1.0;
  for (int d = 0; d < 3; ++d) cells *= (double)(p.hi[d] - p.lo[d]);
  r.t_pred = t * cells;
  r.status = WSO_OK;
  return WSO_OK;
}

// ================================================================ NEXT-1: simulated hit rates
// replace the paper's counter-based curve fits by
// (O, R) samples from a sectored, fully associative LRU simulator (SPEC cachesim-oracle,
// S:507-555) replaying the configuration's own request streams, and a least-squares fit of
// the Gompertz form ("coarse grid search ... followed by local refinement").
//
// Request stream of a block B: warps in order; per warp the instructions in canonical order
// (field, kind [loads first], offset C = elem * (pitch . r)); per warp instruction its distinct
// sectors in ascending order (the coalesced requests).  Every request updates LRU
// recency; a request to a resident line with the sector invalid, or to an absent line, is a
// miss (the line is allocated with that sector valid, evicting the least recently used line).

struct SimReq {
  Key sector;
  bool is_store;
};

// Requests of blocks [B0, B1) in schedule order, only those of kind in `kinds` (bit mask).
std::vector<SimReq> block_trace(const wso_kernel& K, const wso_gpu& g, const Plan& p, const std::vector<int64_t>& blocks,
                                int kinds) {
  std::vector<const Instr*> order;
  for (const Instr& I : p.instr) order.push_back(&I);
  auto offs = [&](const Instr* I) {
    const wso_field& f = K.fields[I->field];
    return f.elem_bytes * (f.pitch[0] * I->r[0] + f.pitch[1] * I->r[1] + f.pitch[2] * I->r[2]);
  };
  std::stable_sort(order.begin(), order.end(), [&](const Instr* a, const Instr* b) {
    if (a->field != b->field) return a->field < b->field;
    if (a->is_store != b->is_store) return a->is_store < b->is_store;
    return offs(a) < offs(b);
  });
  std::vector<SimReq> out;
  const int64_t n_warps = ceildiv(p.T, 32);
  for (int64_t B : blocks)
    for (int64_t w = 0; w < n_warps; ++w)
      for (const Instr* I : order) {
        if (!((kinds >> I->is_store) & 1)) continue;
        std::set<int64_t> secs;
        for (int64_t lane = 0; lane < 32; ++lane) {
          int64_t t = w * 32 + lane;
          if (t >= p.T) break;
          V3 base = base_cell(p, B, t);
          if (issues(p, base, *I)) secs.insert(floordiv(instr_address(K, base, *I), g.sector_bytes));
        }
        for (int64_t sct : secs) out.push_back(SimReq{Key(I->field, sct), I->is_store != 0});
      }
  return out;
}

// Fully associative LRU cache over lines with per-sector valid bits.
struct SimCache {
  int64_t cap, spl;
  std::list<Key> lru;  // front = most recently used line
  std::map<Key, std::pair<std::list<Key>::iterator, std::set<int64_t>>> lines;
  SimCache(int64_t cap_lines, int64_t sectors_per_line) : cap(std::max<int64_t>(1, cap_lines)), spl(sectors_per_line) {}
  bool access(const Key& s) {  // returns hit
    Key ln(s.first, floordiv(s.second, spl));
    auto it = lines.find(ln);
    if (it != lines.end()) {
      lru.splice(lru.begin(), lru, it->second.first);
      bool hit = it->second.second.count(s.second) > 0;
      it->second.second.insert(s.second);
      return hit;
    }
    lru.push_front(ln);
    lines[ln] = std::make_pair(lru.begin(), std::set<int64_t>{s.second});
    if ((int64_t)lines.size() > cap) {
      lines.erase(lru.back());
      lru.pop_back();
    }
    return false;
  }
  bool valid(const Key& s) const {
    auto it = lines.find(Key(s.first, floordiv(s.second, spl)));
    return it != lines.end() && it->second.second.count(s.second) > 0;
  }
};

int64_t simulate(const wso_kernel& K, const wso_gpu& g, const wso_config& c, const int64_t* caps, int64_t ncap,
                 wso_sim_result* out) {
  wso_result r;
  int64_t st = estimate(K, g, c, r);
  if (st == WSO_OK && (c.variant & WSO_VAR_MDIM)) st = WSO_EINVAL;  // the simulator replays linear addresses
  if (st == WSO_OK && g.line_bytes / g.sector_bytes > 32) st = WSO_ELIMIT;
  for (int64_t k = 0; k < ncap; ++k) {
    out[k] = wso_sim_result();
    out[k].status = st;
    out[k].capacity_bytes = caps[k];
    if (caps[k] < 1) out[k].status = WSO_EINVAL;
  }
  if (st != WSO_OK) return st;
  Plan p;
  wso_result tmp;
  make_plan(K, g, c, p, tmp);
  const int64_t spl = g.line_bytes / g.sector_bytes;
  // ---- L1: each SM set's load requests through a fresh cache (Q8/Q9)
  int64_t l1_req = 0, l1_comp = 0;
  std::vector<int64_t> l1_miss(ncap, 0);
  for (int64_t j = 0; j < p.n_sets; ++j) {
    std::vector<int64_t> blocks;
    for (int64_t B = p.s + j; B < p.s + p.W; B += g.n_sm) blocks.push_back(B);
    std::vector<SimReq> tr = block_trace(K, g, p, blocks, 1);
    l1_req += (int64_t)tr.size();
    std::set<Key> distinct;
    for (const SimReq& q : tr) distinct.insert(q.sector);
    l1_comp += (int64_t)distinct.size();  // compulsory misses of the stream
    for (int64_t k = 0; k < ncap; ++k) {
      SimCache cache(caps[k] / g.line_bytes, spl);
      for (const SimReq& q : tr) l1_miss[k] += cache.access(q.sector) ? 0 : 1;
    }
  }
  // ---- stores: the wave's requests (loads and stores) in schedule order; misses among stores
  std::vector<int64_t> wave;
  for (int64_t B = p.s; B < p.s + p.W; ++B) wave.push_back(B);
  std::vector<SimReq> wtr = block_trace(K, g, p, wave, 3);
  int64_t st_req = 0, st_comp = 0;
  std::set<Key> WLD, seen;
  for (const SimReq& q : wtr) {
    if (q.is_store) {
      ++st_req;
      if (!seen.count(q.sector)) ++st_comp;
    } else {
      WLD.insert(q.sector);
    }
    seen.insert(q.sector);
  }
  std::vector<int64_t> st_miss(ncap, 0);
  for (int64_t k = 0; k < ncap; ++k) {
    SimCache cache(caps[k] / g.line_bytes, spl);
    for (const SimReq& q : wtr) {
      bool hit = cache.access(q.sector);
      if (q.is_store && !hit) ++st_miss[k];
    }
  }
  // ---- layer sets: replay L_z = [Lz0, s) (loads + stores, Q15), then count the wave's
  // overlap sectors still valid: those of F_Ly (touched by blocks >= Ly0) for the y curve,
  // the rest of WLD n F_Lz for the z curve (Q16: hits = R_y ov_y + R_z (ov_z - ov_y)).
  std::vector<int64_t> lz, ly;
  for (int64_t B = p.Lz0; B < p.s; ++B) lz.push_back(B);
  for (int64_t B = p.Ly0; B < p.s; ++B) ly.push_back(B);
  std::vector<SimReq> ltr = block_trace(K, g, p, lz, 3);
  std::set<Key> FY, FZ;
  for (const SimReq& q : block_trace(K, g, p, ly, 3)) FY.insert(q.sector);
  for (const SimReq& q : ltr) FZ.insert(q.sector);
  std::vector<Key> ovy, ovz;
  for (const Key& s : WLD)
    if (FY.count(s)) ovy.push_back(s);
    else if (FZ.count(s)) ovz.push_back(s);
  std::vector<int64_t> yres(ncap, 0), zres(ncap, 0);
  for (int64_t k = 0; k < ncap; ++k) {
    SimCache cache(caps[k] / g.line_bytes, spl);
    for (const SimReq& q : ltr) cache.access(q.sector);
    for (const Key& s : ovy) yres[k] += cache.valid(s) ? 1 : 0;
    for (const Key& s : ovz) zres[k] += cache.valid(s) ? 1 : 0;
  }
  // ---- samples: O as in the model (Eq. 4) at capacity C; R = hits / redundant requests
  // (Eq. 3: R_hit = 1 - V_cap / V_red) or resident / potential reuse
  const double LB = (double)g.line_bytes;
  for (int64_t k = 0; k < ncap; ++k) {
    if (out[k].status != WSO_OK) continue;
    wso_sim_result& o = out[k];
    const double C = (double)caps[k];
    o.l1_requests = l1_req;
    o.l1_compulsory = l1_comp;  // = sm_ld_sectors of the estimate unless WSO_VAR_REP_BLOCK
    o.l1_misses = l1_miss[k];
    o.st_requests = st_req;
    o.st_compulsory = st_comp;
    o.st_misses = st_miss[k];
    o.ov_y = (int64_t)ovy.size();
    o.y_resident = yres[k];
    o.ov_z_only = (int64_t)ovz.size();
    o.z_resident = zres[k];
    o.O_l1 = ((double)r.sm_ld_lines * LB / (double)p.n_sets) / C;
    o.O_y = (double)r.ly_lines * LB / C;
    o.O_z = (double)r.lz_lines * LB / C;
    o.O_st = (double)r.wave_lines * LB / C;
    o.R_l1 = l1_req > l1_comp ? (double)(l1_req - o.l1_misses) / (double)(l1_req - l1_comp) : 1.0;
    o.R_st = st_req > st_comp ? (double)(st_req - o.st_misses) / (double)(st_req - st_comp) : 1.0;
    o.R_y = o.ov_y > 0 ? (double)o.y_resident / (double)o.ov_y : 1.0;
    o.R_z = o.ov_z_only > 0 ? (double)o.z_resident / (double)o.ov_z_only : 1.0;
  }
  return WSO_OK;
}

// Least-squares fit of R(O) = a exp(-b exp(-c O)) to n samples:
// (1) grid search a in {0.5, 0.6, ..., 1.0}, b = exp(-8 + 0.5 j) (j = 0..22),
//     c = -8 + 0.25 k (k = 0..31); first minimum of the residual sum of squares in (a, b, c) order;
// (2) 200 Levenberg-Marquardt steps: (J^T J + lambda diag(J^T J)) d = -J^T res, Cramer's rule,
//     a step is taken only if it lowers the RSS (lambda / 10, floor 1e-15), else lambda * 10.
double fit_rss(const double* O, const double* R, int64_t n, const double th[3]) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double e = hit_rate(th, O[i]) - R[i];
    s += e * e;
  }
  return s;
}

double fit_gompertz(const double* O, const double* R, int64_t n, double th[3]) {
  double best = INFINITY;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 23; ++j)
      for (int k = 0; k < 32; ++k) {
        double t[3] = {0.5 + 0.1 * i, std::exp(-8.0 + 0.5 * j), -8.0 + 0.25 * k};
        double v = fit_rss(O, R, n, t);
        if (v < best) {
          best = v;
          th[0] = t[0];
          th[1] = t[1];
          th[2] = t[2];
        }
      }
  double lambda = 1e-3;
  for (int it = 0; it < 200; ++it) {
    double A[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, gv[3] = {0, 0, 0};
    for (int64_t m = 0; m < n; ++m) {
      const double E = std::exp(-th[2] * O[m]);
      const double F = std::exp(-th[1] * E);
      const double J[3] = {F, -th[0] * E * F, th[0] * F * th[1] * E * O[m]};
      const double res = th[0] * F - R[m];
      for (int a = 0; a < 3; ++a) {
        gv[a] += J[a] * res;
        for (int b = 0; b < 3; ++b) A[a][b] += J[a] * J[b];
      }
    }
    double M[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) M[a][b] = A[a][b] + (a == b ? lambda * A[a][a] : 0.0);
    const double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                       M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                       M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    if (!(std::fabs(det) > 0.0)) break;
    double d[3];
    for (int col = 0; col < 3; ++col) {  // Cramer: replace column col by -g
      double Mc[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Mc[a][b] = (b == col) ? -gv[a] : M[a][b];
      d[col] = (Mc[0][0] * (Mc[1][1] * Mc[2][2] - Mc[1][2] * Mc[2][1]) -
                Mc[0][1] * (Mc[1][0] * Mc[2][2] - Mc[1][2] * Mc[2][0]) +
                Mc[0][2] * (Mc[1][0] * Mc[2][1] - Mc[1][1] * Mc[2][0])) / det;
    }
    double t2[3] = {th[0] + d[0], th[1] + d[1], th[2] + d[2]};
    double v = fit_rss(O, R, n, t2);
    if (v < best) {
      best = v;
      th[0] = t2[0];
      th[1] = t2[1];
      th[2] = t2[2];
      lambda = std::max(lambda / 10.0, 1e-15);
    } else {
      lambda *= 10.0;
    }
  }
  return best;
}

}  // namespace

extern "C" {

int64_t wso_check_kernel(const wso_kernel* k) { return check_kernel(*k); }

int64_t wso_plan(const wso_kernel* k, const wso_gpu* g, const wso_config* c, wso_result* r) {
  *r = wso_result();
  int64_t st = check_kernel(*k);
  Plan p;
  if (st == WSO_OK) st = make_plan(*k, *g, *c, p, *r);
  r->status = st;
  if (st == WSO_OK) r->addr_evals = (p.W + (p.s - p.Lz0)) * p.T * (int64_t)p.instr.size();
  return st;
}

int64_t wso_estimate(const wso_kernel* k, const wso_gpu* g, const wso_config* c, wso_result* r) {
  return estimate(*k, *g, *c, *r);
}

void wso_estimate_batch(const wso_kernel* k, const wso_gpu* g, const wso_config* c, int64_t n, wso_result* r,
                        int64_t n_threads) {
  if (n_threads < 1) n_threads = 1;
  std::atomic<int64_t> next(0);
  auto work = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) break;
      estimate(*k, *g, c[i], r[i]);
    }
  };
  std::vector<std::thread> pool;
  for (int64_t i = 1; i < n_threads; ++i) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

int64_t wso_address(const wso_field* f, const int64_t cell[3]) { return address(*f, V3{cell[0], cell[1], cell[2]}); }

int64_t wso_unique_sectors(const int64_t* a, int64_t n, int64_t sector_bytes) {
  return unique_sectors(std::vector<int64_t>(a, a + n), sector_bytes);
}

int64_t wso_halfwarp_wavefronts(const int64_t* a, int64_t n, const wso_gpu* g) {
  return halfwarp_wavefronts(std::vector<int64_t>(a, a + n), *g);
}

double wso_hit_rate(const double abc[3], double O) { return hit_rate(abc, O); }

int64_t wso_simulate(const wso_kernel* k, const wso_gpu* g, const wso_config* c, const int64_t* caps, int64_t ncap,
                     wso_sim_result* out) {
  return simulate(*k, *g, *c, caps, ncap, out);
}

void wso_simulate_batch(const wso_kernel* k, const wso_gpu* g, const wso_config* c, int64_t n, const int64_t* caps,
                        int64_t ncap, wso_sim_result* out, int64_t n_threads) {
  if (n_threads < 1) n_threads = 1;
  std::atomic<int64_t> next(0);
  auto work = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) break;
      simulate(*k, *g, c[i], caps, ncap, out + i * ncap);
    }
  };
  std::vector<std::thread> pool;
  for (int64_t i = 1; i < n_threads; ++i) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

double wso_fit_gompertz(const double* O, const double* R, int64_t n, double abc[3]) {
  return fit_gompertz(O, R, n, abc);
}

}  // extern "C"
