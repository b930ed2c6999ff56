/* oracle/ws_oracle.h -- plain, slow CPU oracle of the Warpspeed data-volume
 * estimator (Ernst et al., arXiv 2204.14242).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2204_14242_b200/, include/ws.h) and neither side includes the other.
 *
 * Every quantity is defined by enumerating every (thread, instruction)
 * address into std::set, following PAPER.md section 4 in the
 * reading fixed by SURVEY.md section 8(c).
 * All integers are int64; all floating point is IEEE double.
 */
#ifndef WS_ORACLE_H
#define WS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t extent[3];   /* elements per dimension, x fastest                    */
  int64_t pitch[3];    /* elements; pitch[0] == 1                             */
  int64_t align_bytes; /* byte address of element (0,0,0)      */
  int64_t elem_bytes;  /* 8 for double                                        */
} wso_field;

typedef struct {
  int64_t field;
  int64_t is_store;
  int64_t off[3];      /* relative cell offset                    */
} wso_access;

typedef struct {
  int64_t n_fields, n_accesses;
  const wso_field*  fields;
  const wso_access* accesses;
  int64_t dom_lo[3], dom_hi[3];   /* iteration domain in field-index coords  */
  int64_t regs_per_thread;        /* 0 = no register limit                   */
  double  flops_per_lup;
} wso_kernel;

typedef struct {
  int64_t n_sm, max_thr_sm, max_blk_sm, max_thr_blk, regs_sm;
  int64_t sector_bytes, line_bytes, n_banks, bank_bytes, half_warp, pair_window_bytes;
  int64_t l2_sections;
  int64_t l1_bytes, l2_bytes;
  double  clock_hz, dram_bw, l2_bw;
  double  hit_abc[4][3];          /* L1, L2-over-y, L2-over-z, L2-store */
  int64_t page_bytes;             /* TLB page size; 0 = pages not counted */
  double  link_bw;                /* L2 inter-section link bytes/s; 0 = no link limiter */
} wso_gpu;

/* model variants, bit flags of wso_config.variant */
enum {
  WSO_VAR_MDIM = 1,       /* multidimensional address space for wave + layer sets */
  WSO_VAR_PREV_WAVE = 2,  /* warm reuse from the directly preceding wave only (SBAC) */
  WSO_VAR_L2_DUP = 4,     /* L2 capacity from the estimated line duplication */
  WSO_VAR_REP_BLOCK = 8   /* L1 scopes from one representative block */
};

typedef struct {
  int64_t block[3], fold[3], blocks_per_sm;
  int64_t variant;                /* WSO_VAR_* bits */
} wso_config;

typedef struct {
  int64_t status, limiter;
  int64_t grid[3], k, wave_blocks, n_smsets, wave_first_block, lup_wave, n_instr;
  int64_t l1_wavefronts, l1_req_ld_sectors, l1_req_st_sectors, sm_ld_sectors, sm_ld_lines;
  int64_t wave_ld_sectors, wave_st_sectors, wave_lines, ly_lines, lz_lines, ov_y, ov_z;
  double  O_l1, R_l1, O_y, R_y, O_z, R_z, O_st, R_st;
  double  l1_cyc_per_lup, l2_ld_Bpl, l2_st_Bpl, dram_ld_Bpl, dram_st_Bpl;
  double  t_l1, t_l2, t_dram, t_pred;
  int64_t addr_evals;             /* (thread, instruction) evaluations done   */
  int64_t wave_pages;             /* TLB pages touched by the wave (0 if page_bytes == 0) */
  int64_t l2_dup_lines;           /* sum over L2 sections of section lines - distinct wave lines */
  int64_t l2_link_sectors;        /* sum over sections of section load sectors - distinct ones */
  double  l2_eff_bytes, t_link;   /* effective L2 capacity used by the model; link time per LUP */
} wso_result;

/* NEXT-1: simulated hit-rate samples of one configuration at one cache capacity (see
 * ws_oracle.cpp "NEXT-1" for the request streams and the cache). */
typedef struct {
  int64_t status, capacity_bytes;
  int64_t l1_requests, l1_compulsory, l1_misses;   /* SM-set load request streams, summed over sets */
  int64_t st_requests, st_compulsory, st_misses;   /* store requests of the wave stream */
  int64_t ov_y, y_resident, ov_z_only, z_resident; /* wave load sectors of F_Ly / F_Lz minus F_Ly valid after L_z */
  double  O_l1, R_l1, O_y, R_y, O_z, R_z, O_st, R_st;
} wso_sim_result;

/* status codes (same meaning as the ABI's, defined independently) */
enum { WSO_OK = 0, WSO_EINVAL = 1, WSO_ELIMIT = 2, WSO_EBOUNDS = 3 };

/* Kernel descriptor check (ABI section (b) conventions). Returns a status. */
int64_t wso_check_kernel(const wso_kernel* k);

/* One configuration, single-threaded. Returns status (also in r->status). */
int64_t wso_estimate(const wso_kernel* k, const wso_gpu* g, const wso_config* c, wso_result* r);

/* Geometry only (O1-O3): status, grid, k, W, s, n_instr and addr_evals, no enumeration. */
int64_t wso_plan(const wso_kernel* k, const wso_gpu* g, const wso_config* c, wso_result* r);

/* n configurations on up to n_threads host threads (one config per thread). */
void wso_estimate_batch(const wso_kernel* k, const wso_gpu* g, const wso_config* c,
                        int64_t n, wso_result* r, int64_t n_threads);

/* Pieces exposed for the pins in tests/ (each is the definition, written out). */
int64_t wso_address(const wso_field* f, const int64_t cell[3]);
int64_t wso_unique_sectors(const int64_t* addr, int64_t n, int64_t sector_bytes);
int64_t wso_halfwarp_wavefronts(const int64_t* addr, int64_t n, const wso_gpu* g);
double  wso_hit_rate(const double abc[3], double O);

/* NEXT-1: LRU-simulated (O, R) samples at capacities caps[0..ncap) (out: ncap records per config),
 * and the least-squares Gompertz fit (returns the residual sum of squares). */
int64_t wso_simulate(const wso_kernel* k, const wso_gpu* g, const wso_config* c, const int64_t* caps,
                     int64_t ncap, wso_sim_result* out);
void    wso_simulate_batch(const wso_kernel* k, const wso_gpu* g, const wso_config* c, int64_t n,
                           const int64_t* caps, int64_t ncap, wso_sim_result* out, int64_t n_threads);
double  wso_fit_gompertz(const double* O, const double* R, int64_t n, double abc[3]);

#ifdef __cplusplus
}
#endif
#endif
