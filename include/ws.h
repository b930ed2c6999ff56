/* include/ws.h -- C ABI of libwsb200.so, the B200-native hot path of the
 * Warpspeed data-volume estimator (Ernst et al., arXiv 2204.14242,
 * "Analytical Performance Estimation during Code Generation on Modern GPUs").
 *
 * The estimator takes, per the paper's statement of the problem (PAPER.md
 * P:163-166), only address expressions (here: per-field constant relative
 * cell offsets), a launch configuration (block, folding; grid is
 * derived), field sizes and field alignments, plus
 * hardware parameters (Table tab:av100).  For every configuration
 * it counts distinct 32 B sectors / 128 B lines at the warp-instruction, SM-
 * resident-set, wave and layer-set scopes, evaluates the capacity
 * model (Eqs. 1-5) and the max-limiter performance model
 * (P:262-281), and ranks the configurations.  Exact semantics:
 * DESIGN.md ("Readings") and SURVEY.md section 8.
 *
 * Conventions (all functions):
 *  - Every function returns ws_status; WS_OK = 0.  On a call-level error the
 *    message is available from ws_last_error(ctx) until the next call on ctx.
 *  - The caller owns every array passed in or out; the library never keeps a
 *    pointer to caller memory after a call returns (describe calls deep-copy).
 *  - Per-configuration problems never fail a batch: they set ws_result.status
 *    (WS_EINVAL, WS_ELIMIT, WS_EUNKNOWN_ID) and leave that record's numbers 0.
 *  - A context is bound to one CUDA device and one stream and is not
 *    thread-safe.  Results are byte-identical for identical inputs.
 *  - There is no CPU fallback: a context cannot be created without a CUDA
 *    device (WS_ECUDA).
 */
#ifndef WS_H
#define WS_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WS_OK = 0,
  WS_EINVAL = 1,      /* malformed argument / descriptor                                    */
  WS_ELIMIT = 2,      /* a documented limit is exceeded (threads/block, occupancy k = 0, ...) */
  WS_EBOUNDS = 3,     /* an access of an active cell leaves its field              */
  WS_ENOMEM = 4,      /* device or host allocation failed                                   */
  WS_ECUDA = 5,       /* CUDA runtime error (no device, launch failure, ...)                */
  WS_EUNKNOWN_ID = 6  /* kernel_id / gpu_id not described in this context                   */
} ws_status;

typedef struct ws_ctx ws_ctx;

/* Create a context on CUDA device `cuda_device`; work is issued on
 * `cuda_stream` (a cudaStream_t; NULL = the legacy default stream). */
ws_status ws_create(int cuda_device, void* cuda_stream, ws_ctx** out);
void ws_destroy(ws_ctx* ctx);
const char* ws_last_error(const ws_ctx* ctx);
/* Change the stream later work is issued on (e.g. torch's current stream). */
ws_status ws_set_stream(ws_ctx* ctx, void* cuda_stream);

/* ------------------------------------------------------------------ kernels
 * Field: a row-major array, x fastest.  Byte address of element (x,y,z):
 *   align_bytes + elem_bytes * (x*pitch[0] + y*pitch[1] + z*pitch[2])
 * (P:157-161 with the unknown base pointer replaced by the alignment).
 * Requirements: pitch[0] == 1, pitch[1] >= extent[0], pitch[2] >= pitch[1]*extent[1]
 * (rows and planes never overlap); elem_bytes in {1,2,4,8,16,32}; one z-plane
 * (pitch[2] * elem_bytes) at most 2 GiB - 16 KiB (WS_ELIMIT).  */
typedef struct {
  int64_t extent[3];
  int64_t pitch[3];
  int64_t align_bytes;   /* may be negative (P:540 example uses -8); a multiple of elem_bytes */
  uint32_t elem_bytes;
  uint32_t pad;
} ws_field;

/* One access `field[cell + off]` (relative field access). */
typedef struct {
  uint32_t field;
  uint32_t is_store;     /* 0 = load, 1 = store */
  int32_t off[3];
} ws_access;

typedef struct {
  uint32_t n_fields;           /* 1..64  */
  uint32_t n_accesses;         /* 1..128 */
  const ws_field* fields;
  const ws_access* accesses;
  int64_t dom_lo[3], dom_hi[3];/* iteration domain (field-index coords); guard clipping P:171-172 */
  uint32_t regs_per_thread;    /* 0 = ignore the register limit on occupancy (Q10) */
  uint32_t pad;
  double flops_per_lup;        /* carried, not a limiter */
} ws_kernel;

/* Deep-copies the description.  Errors: WS_EINVAL (counts, layout, elem,
 * align_bytes not a multiple of elem_bytes, empty domain), WS_EBOUNDS (dom +- offsets leaves a field), WS_ELIMIT (a
 * field has more than 16 distinct x-offset runs, or a z-plane > 2 GiB - 16 KiB).
 * *kernel_id receives a new id. */
ws_status ws_describe_kernel(ws_ctx* ctx, const ws_kernel* k, uint32_t* kernel_id);

/* ------------------------------------------------------------------ hardware
 * Table tab:av100 plus the cache geometry of P:373-395. */
typedef struct {
  uint32_t n_sm;
  uint32_t max_thr_sm, max_blk_sm, max_thr_blk, regs_sm;   /* occupancy limits (Q10) */
  uint32_t sector_bytes;       /* 32  (power of two, >= every elem_bytes used)  */
  uint32_t line_bytes;         /* 128 (power of two, multiple of sector_bytes, <= 4096) */
  uint32_t n_banks;            /* 16  (power of two)                            */
  uint32_t bank_bytes;         /* 8   (power of two)                            */
  uint32_t half_warp;          /* 16  (power of two dividing 32)                */
  uint32_t pair_window_bytes;  /* 1024                                  */
  uint32_t l2_sections;        /* 2 for the split A100 L2: L2_eff = l2_bytes / l2_sections */
  uint64_t l1_bytes, l2_bytes;
  double clock_hz, dram_bw, l2_bw;   /* Hz, bytes/s, bytes/s */
  double hit_abc[4][3];        /* R(O) = a exp(-b exp(-c O)) for L1, L2-over-y, L2-over-z, L2-store */
  /* Outlook metrics: */
  uint64_t page_bytes;         /* TLB page size (power of two >= line_bytes); 0 = wave_pages not counted */
  double link_bw;              /* bytes/s of the link between L2 sections; 0 = not a limiter */
} ws_gpu;

/* Deep-copies.  Errors: WS_EINVAL (zero / non-power-of-two geometry, page_bytes not 0
 * or a power of two >= line_bytes, link_bw < 0, ...), WS_ELIMIT (line_bytes > 4096,
 * l2_sections > 4). */
ws_status ws_describe_gpu(ws_ctx* ctx, const ws_gpu* g, uint32_t* gpu_id);

/* ------------------------------------------------------------------ configurations */
/* Model variants (bit flags of ws_config.variant).  0 = the
 * model of DESIGN.md section 3. */
enum {
  /* Wave and layer-set footprints in the multidimensional address space: a
   * sector is (field, z, y, floor(x * elem_bytes / sector_bytes)); rows never share a
   * sector or line and the field alignment is not considered.  Warp and SM-set
   * scopes keep linear addresses (explicit grid iteration). */
  WS_VAR_MDIM = 1,
  /* Warm-cache reuse from the directly preceding wave only (the V100 / SBAC model,
   * P:583-587): both look-back sets become [max(0, s - W), s), so ov_z = ov_y and
   * ly_lines = lz_lines; the model uses the L2-over-y curve for it. */
  WS_VAR_PREV_WAVE = 2,
  /* Effective L2 capacity from the estimated line duplication between L2 sections
   * instead of l2_bytes / l2_sections: l2_bytes * U / (U + l2_dup_lines),
   * U = distinct wave lines. */
  WS_VAR_L2_DUP = 4,
  /* L1 scopes (warp instructions, SM sets) from one representative block, the wave's middle
   * block s + W/2, standing for all W wave blocks (per-block footprint, no
   * L1 sharing between co-resident blocks): l1_wavefronts, l1_req_*_sectors, sm_ld_*,
   * lup_wave = W x the block's.  Wave / layer-set scopes are unchanged. */
  WS_VAR_REP_BLOCK = 8
};

typedef struct {
  uint32_t kernel_id, gpu_id;
  uint32_t block[3];           /* threads per block (X,Y,Z)            */
  uint32_t fold[3];            /* thread folding factors; prod <= 64       */
  uint32_t blocks_per_sm;      /* 0 = derive the occupancy k (Q10)                */
  uint32_t variant;            /* WS_VAR_* bits; other bits -> status WS_EINVAL   */
} ws_config;                   /* 40 bytes */

typedef struct {
  int32_t status;              /* WS_OK or the per-config error                   */
  uint32_t limiter;            /* 0 = L1, 1 = L2, 2 = DRAM, 3 = L2 section link   */
  uint32_t grid[3];            /* blocks per dimension                            */
  uint32_t k;                  /* resident blocks per SM                          */
  uint32_t wave_blocks;        /* W                                               */
  uint32_t n_smsets;           /* min(n_sm, W)                                    */
  uint32_t n_instr;            /* instructions per thread after folding dedupe    */
  uint32_t rank;               /* filled by ws_rank                               */
  uint64_t wave_first_block;   /* s                                               */
  uint64_t lup_wave;           /* active cells (lattice updates) of the wave      */
  uint64_t l1_wavefronts;      /* a3: sum of half-warp wavefronts (loads+stores)  */
  uint64_t l1_req_ld_sectors;  /* a3: per-warp-instruction unique load sectors    */
  uint64_t l1_req_st_sectors;  /* a3: per-warp-instruction unique store sectors   */
  uint64_t sm_ld_sectors;      /* a4: sum over SM sets of unique load sectors     */
  uint64_t sm_ld_lines;        /* a4: sum over SM sets of unique load lines       */
  uint64_t wave_ld_sectors;    /* a5 */
  uint64_t wave_st_sectors;    /* a5 */
  uint64_t wave_lines;         /* a5: lines of all wave accesses                  */
  uint64_t ly_lines, lz_lines; /* a6: lines of the layer sets                     */
  uint64_t ov_y, ov_z;         /* a6: |wave load sectors  intersect  layer sectors| */
  uint64_t addr_evals;         /* (W + |L_z|) * T * n_instr: plain-definition work units */
  double O_l1, R_l1, O_y, R_y, O_z, R_z, O_st, R_st;
  double l1_cyc_per_lup, l2_ld_Bpl, l2_st_Bpl, dram_ld_Bpl, dram_st_Bpl;
  double t_l1, t_l2, t_dram;   /* seconds per lattice update                      */
  double t_pred;               /* seconds for the whole domain                    */
  /* Outlook metrics (NEXT-4), linear address space.  SM j belongs to L2 section
   * floor(j * l2_sections / n_sm); wave block B runs on SM (B - s) mod n_sm. */
  uint64_t wave_pages;         /* distinct (field, address / page_bytes) of the wave */
  uint64_t l2_dup_lines;       /* sum over sections of the section's lines - distinct wave lines   */
  uint64_t l2_link_sectors;    /* sum over sections of the section's load sectors - distinct ones  */
                               /* (both 0 unless l2_sections > 1 and (link_bw > 0 or WS_VAR_L2_DUP)) */
  double l2_eff_bytes;         /* L2 capacity the model used (l2_bytes / l2_sections or WS_VAR_L2_DUP) */
  double t_link;               /* seconds per LUP on the section link (0 if link_bw == 0)          */
} ws_result;                   /* 336 bytes */

/* Host pointers; synchronous.  Copies cfgs to the device, runs the whole
 * device path, copies n results back. */
ws_status ws_estimate(ws_ctx* ctx, const ws_config* cfgs, size_t n, ws_result* out);

/* Device pointers (cfgs: n ws_config, out: n ws_result in device memory);
 * enqueued on the context stream, returns without synchronising. */
ws_status ws_estimate_async(ws_ctx* ctx, const ws_config* d_cfgs, size_t n, ws_result* d_out);

/* One sweep step end to end on the device ("the best configurations are selected",
 * P:1025-1046): ws_estimate_async of d_cfgs followed by ws_rank_async of d_out (d_top: k
 * device uint32 indices, may be null), records and top-k byte-identical to those two calls.
 * For n <= 1024 the FP64 model kernel (a7) also ranks (a8): its last CTA to finish ranks the
 * batch's (t_pred, index) keys in shared memory (by counting for n <= 256, a sorting network
 * above), saving the rank launch and a kernel boundary on the critical path; larger batches call
 * the two paths in turn.
 * Device pointers, enqueued on the context stream; errors as ws_estimate_async / ws_rank_async. */
ws_status ws_estimate_ranked_async(ws_ctx* ctx, const ws_config* d_cfgs, size_t n, ws_result* d_out, size_t k,
                                   uint32_t* d_top_idx);

/* Architecture exploration (BJ configs[3]; hardware parameters P:307-320): every configuration
 * against every hardware set of gpu_ids (a host array of n_gpu <= 256 described gpu ids).
 *   out[g * n + i] = the record ws_estimate gives for cfgs[i] with gpu_id = gpu_ids[g]
 * (cfgs[i].gpu_id is ignored), byte-identical.  The integer stages a1-a6 read a hardware set
 * only through its occupancy limits, SM count, sector / line / bank geometry, half-warp, pair
 * window, section count, page size and whether link_bw > 0; they run once per group of gpu_ids
 * that agree in all of these, and the FP64 model (a7) fans out over each group's sets.
 * ws_estimate_multi: host cfgs / out, synchronous.  ws_estimate_multi_async: device d_cfgs (n) /
 * d_out (n * n_gpu), gpu_ids on the host, enqueued on the context stream.
 * Errors: WS_EUNKNOWN_ID (an id not described), WS_ELIMIT (n_gpu > 256, n * n_gpu > 2^24). */
ws_status ws_estimate_multi(ws_ctx* ctx, const ws_config* cfgs, size_t n, const uint32_t* gpu_ids, uint32_t n_gpu,
                            ws_result* out);
ws_status ws_estimate_multi_async(ws_ctx* ctx, const ws_config* d_cfgs, size_t n, const uint32_t* gpu_ids,
                                  uint32_t n_gpu, ws_result* d_out);
/* Integer-stage groups the last ws_estimate_multi[_async] call formed. */
uint32_t ws_last_group_count(const ws_ctx* ctx);

/* Rank by (t_pred ascending, index ascending); failed configs rank last.
 * Fills res[i].rank and top_idx[0..min(k,n)) with the indices of the best.
 * ws_rank: host pointers, synchronous.  ws_rank_async: device pointers, no sync.
 * n <= 2^24 (WS_ELIMIT).  Device work: one CTA sorting in shared memory up to 2048 records;
 * up to 2^18: sorted tiles of 2048 / 4096 records and a binary-search merge-rank; beyond: a
 * stable radix sort of 64-bit keys (scratch kept by the context, grow-only). */
ws_status ws_rank(ws_ctx* ctx, ws_result* res, size_t n, size_t k, uint32_t* top_idx);
ws_status ws_rank_async(ws_ctx* ctx, ws_result* d_res, size_t n, size_t k, uint32_t* d_top_idx);

/* Bounds checks (diagnostics; SURVEY 4 layer 5 in place of compute-sanitizer, which this GPU
 * pool does not run): a library built with -DWS_CHECK checks every dynamically computed scratch
 * index of the estimate chain against its capacity on the device and counts violations (no
 * graphs in that build).  out[5] = {1 if this is a bounds-check build else 0, violations since
 * the last read, first violation's source line, its index, its capacity}; reading resets them.
 * Synchronises the context stream.  Ordinary builds: all zeros, WS_OK. */
ws_status ws_check_read(ws_ctx* ctx, uint64_t* out);

/* ------------------------------------------------------------------ NEXT-1: simulated hit rates
 * (O, R) samples for the four hit-rate curves from a sectored,
 * fully associative LRU cache (line_bytes lines, sector valid bits; SPEC cachesim-oracle
 * S:507-555) replaying the configuration's own request streams, instead of the paper's
 * hardware-counter measurements.  Request stream of a block: warps in order; per
 * warp the instructions in canonical order (field, kind [loads first], offset elem*(pitch.r));
 * per warp instruction its distinct sectors ascending.  Every request updates recency; a
 * request whose sector is not valid (absent line or invalid sector) is a miss that validates it.
 *   L1:    each SM set's load requests (blocks s+j, s+j+n_sm, ...) through its own cache;
 *   store: the wave's requests (loads and stores, blocks s..s+W-1); misses among stores;
 *   layer: the requests of L_z = [Lz0, s); afterwards the wave's load sectors of F_Ly (ov_y)
 *          and of F_Lz minus F_Ly (ov_z_only) that are still valid.
 * R = hits / (requests - compulsory) (Eq. 3) for L1 and stores, resident / overlap for y and z;
 * O = the model's allocation (Eq. 4) over the capacity.  The GPU computes exact LRU stack
 * distances once per stream and answers every capacity from them. */
typedef struct {
  int32_t status;              /* WS_OK; WS_EINVAL for WS_VAR_MDIM configs or capacity 0;
                                  WS_ELIMIT: line_bytes/sector_bytes > 32 or a stream >= 2^31 */
  uint32_t pad;
  uint64_t capacity_bytes;
  uint64_t l1_requests, l1_compulsory, l1_misses;
  uint64_t st_requests, st_compulsory, st_misses;
  uint64_t ov_y, y_resident, ov_z_only, z_resident;
  double O_l1, R_l1, O_y, R_y, O_z, R_z, O_st, R_st;
} ws_sim_result;               /* 160 bytes */

/* Host arrays; synchronous.  out[i * n_cap + k] = configuration i at capacities[k];
 * n_cap <= 64.  Device memory grows with the streams (about 40 B per request); the context
 * keeps these buffers for later calls (grow-only) until ws_sim_release or ws_destroy, and
 * drops them after a failed call. */
ws_status ws_simulate(ws_ctx* ctx, const ws_config* cfgs, size_t n, const uint64_t* capacities, uint32_t n_cap,
                      ws_sim_result* out);
/* Free ws_simulate's kept device buffers (synchronises the context's stream). */
ws_status ws_sim_release(ws_ctx* ctx);

/* Least-squares fit of R(O) = a exp(-b exp(-c O)) to n >= 3 samples, on the device:
 * grid search a in {0.5,...,1.0}, b = exp(-8 + 0.5 j) (j < 23), c = -8 + 0.25 k (k < 32), then 200
 * Levenberg-Marquardt steps (accepted only when the residual sum of squares drops).  Host
 * arrays; abc receives (a, b, c), *rss the residual sum of squares. */
ws_status ws_fit_gompertz(ws_ctx* ctx, const double* O, const double* R, size_t n, double abc[3], double* rss);

/* ------------------------------------------------------------------ NEXT-2: on-box validation
 * The modelled workload itself: the 3D-25pt range-4 FP64 star stencil of
 * P:751-764 as an sm_100a kernel, dst = w0 src + sum_k w_k (six neighbours at distance k),
 * k = 1..4, over the domain [4, n+4)^3 of (n+8)^3 fields (x fastest, ghost 4, the K25
 * description).  block = threads per block (X,Y,Z), fold = (1,1,1), (1,2,1) or (1,1,2)
 * (thread folding P:754).  Runs `reps` launches on cuda_stream (a cudaStream_t) and writes the
 * average device milliseconds per launch to *ms_avg (CUDA events, synchronises).  d_src /
 * d_dst: device arrays of (n[0]+8)(n[1]+8)(n[2]+8) doubles owned by the caller.
 * Errors: WS_EINVAL (null, fold not one of the three), WS_ELIMIT (block > 1024 threads or
 * grid > 65535 in y/z), WS_ECUDA. */
ws_status ws_validate_stencil25(void* cuda_stream, const double* d_src, double* d_dst, const int64_t n[3],
                                const uint32_t block[3], const uint32_t fold[3], uint32_t reps, double* ms_avg);

/* The paper's second workload (the estimator's LBM15 description) as an
 * sm_100a kernel: D3Q15 pull (PDF q loaded at cell - c_q from d_src + q * array, stored at the
 * cell to d_dst + q * array), phase field d_phi loaded at the cell and its 6 neighbours, FD
 * result stored to d_fd; FP64; arrays of (n[0]+2)(n[1]+2)(n[2]+2) doubles (ghost 1, fzyx: the 15
 * PDFs of d_src / d_dst consecutive), domain [1, n+1)^3; velocities in workloads.D3Q15 order.
 * block = threads per block; reps launches; average device ms in *ms_avg.  Errors as
 * ws_validate_stencil25. */
ws_status ws_validate_lbm15(void* cuda_stream, const double* d_src, double* d_dst, const double* d_phi, double* d_fd,
                            const int64_t n[3], const uint32_t block[3], uint32_t reps, double* ms_avg);

/* Number of kernel launches the last ws_estimate[_async] / ws_rank[_async]
 * call enqueued (for the bench's gpu_launches count). */
uint32_t ws_last_launch_count(const ws_ctx* ctx);

/* Tracing.  While enabled, CUDA events are recorded on the context stream
 * around every kernel the library launches.  ws_profile_read synchronises on
 * them, writes the summed device milliseconds per kernel (in the order of
 * ws_kernel_name(0..)) and the number of launches per kernel, resets the
 * accumulators and returns the number of kernel kinds in *n_kinds. */
ws_status ws_profile_enable(ws_ctx* ctx, int on);
ws_status ws_profile_read(ws_ctx* ctx, double* ms, uint64_t* launches, uint32_t cap, uint32_t* n_kinds);
const char* ws_kernel_name(uint32_t i);   /* NULL past the last kind */

/* Algorithmic work units each kernel kind processed in the last
 * ws_estimate[_async] call (synchronises).  Units:
 * k_warp / k_wclass: lane-instructions evaluated (32 per warp and instruction,
 * 32 per warp only classified); k_smset / k_sclass: address rows evaluated;
 * k_rows: algorithmic integer operations (weighted per offset group, run and row);
 * k_plan: unused (0). */
ws_status ws_work_read(ws_ctx* ctx, uint64_t* units, uint32_t cap);

#ifdef __cplusplus
}
#endif
#endif
