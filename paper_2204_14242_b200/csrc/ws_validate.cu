// ws_validate.cu -- SURVEY 8(f) NEXT-2: the modelled workload itself, for on-box validation.
//
// The paper validates its predictions against hardware counters of the pystencils-generated
// 3D-25pt range-4 star stencil.  This is that kernel written for
// sm_100a: one thread per cell (x fastest), thread folding 2y / 2z (a thread updates
// consecutive cells; the loads the folded cells share are issued once), guard clipping
// by the domain, FP64.  Layout as the estimator's K25 description: double fields of
// (nx+8) x (ny+8) x (nz+8), ghost width 4, domain [4, n+4) per dimension.
// bench / scripts/validate_next2.py run it over the 168-config space under ncu and compare the
// counters with the estimator's per-level volumes.
#include <cuda_runtime.h>

#include <cstdint>

#include "ws.h"

namespace wsv {

__constant__ double c_w[5];  // centre + 4 ring weights

template <int FY, int FZ>
__global__ void k_st25(const double* __restrict__ src, double* __restrict__ dst, int nx, int ny, int nz,
                       long long py, long long pz) {
  const int x = 4 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  const int yb = 4 + (int)(blockIdx.y * blockDim.y + threadIdx.y) * FY;
  const int zb = 4 + (int)(blockIdx.z * blockDim.z + threadIdx.z) * FZ;
  if (x >= nx + 4 || yb >= ny + 4 || zb >= nz + 4) return;
  const long long c = x + py * yb + pz * zb;
  const double* p = src + c;
  // one folded cell at offset (fy, fz) from the thread's base cell; with every folded cell
  // active the cells share one straight-line block, so loads of the same address are issued
  // once (register reuse of folding: 2y / 2z -> 42 loads instead of 50)
  auto cell = [&](int fy, int fz) {
    const long long o = fy * py + fz * pz;
    double v = c_w[0] * p[o];
#pragma unroll
    for (int k = 1; k <= 4; ++k)
      v += c_w[k] * (p[o - k] + p[o + k] + p[(fy - k) * py + fz * pz] + p[(fy + k) * py + fz * pz] +
                     p[fy * py + (fz - k) * pz] + p[fy * py + (fz + k) * pz]);
    return v;
  };
  if (yb + FY <= ny + 4 && zb + FZ <= nz + 4) {
#pragma unroll
    for (int fz = 0; fz < FZ; ++fz)
#pragma unroll
      for (int fy = 0; fy < FY; ++fy) dst[c + fy * py + fz * pz] = cell(fy, fz);
  } else {  // partially outside the domain: every cell has its own guard (Q27)
#pragma unroll
    for (int fz = 0; fz < FZ; ++fz)
#pragma unroll
      for (int fy = 0; fy < FY; ++fy)
        if (yb + fy < ny + 4 && zb + fz < nz + 4) dst[c + fy * py + fz * pz] = cell(fy, fz);
  }
}

// D3Q15 velocities in the estimator's order (workloads.D3Q15): rest, 6 faces, 8 corners
__constant__ int c_q15[15][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0},  {0, 1, 0},  {0, -1, 0},
                                 {0, 0, 1},  {0, 0, -1},  {-1, -1, -1}, {-1, -1, 1}, {-1, 1, -1},
                                 {-1, 1, 1}, {1, -1, -1}, {1, -1, 1},  {1, 1, -1}, {1, 1, 1}};

// The paper's second workload (SURVEY Q23 "LBM15"): a pull-scheme D3Q15 update coupled
// to a 3D 7-point phase-field stencil, FP64, 32 arrays in fzyx layout (15 source PDFs, 15
// destination PDFs, phi, the finite-difference result), one thread per cell.  Memory accesses
// are exactly the estimator's LBM15 description: PDF q loaded at cell - c_q, stored at the
// cell; phi loaded at the cell and its 6 neighbours; one FD result stored.  The arithmetic is a
// BGK-style relaxation towards an equilibrium weighted by the phase-field Laplacian (the
// counters, not the physics, are what is validated).
__global__ void __launch_bounds__(512, 1) k_lbm15(const double* __restrict__ src, double* __restrict__ dst, const double* __restrict__ phi,
                        double* __restrict__ fd, int nx, int ny, int nz, long long py, long long pz, long long arr) {
  const int x = 1 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  const int y = 1 + (int)(blockIdx.y * blockDim.y + threadIdx.y);
  const int z = 1 + (int)(blockIdx.z * blockDim.z + threadIdx.z);
  if (x >= nx + 1 || y >= ny + 1 || z >= nz + 1) return;
  const long long c = x + py * y + pz * z;
  double f[15], rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
  for (int q = 0; q < 15; ++q) {
    f[q] = src[q * arr + c - c_q15[q][0] - py * c_q15[q][1] - pz * c_q15[q][2]];
    rho += f[q];
    jx += c_q15[q][0] * f[q];
    jy += c_q15[q][1] * f[q];
    jz += c_q15[q][2] * f[q];
  }
  const double p0 = phi[c];
  const double lap = phi[c + 1] + phi[c - 1] + phi[c + py] + phi[c - py] + phi[c + pz] + phi[c - pz] - 6.0 * p0;
  const double omega = 1.2 + 0.1 * p0, g = 0.05 * lap;
#pragma unroll
  for (int q = 0; q < 15; ++q) {
    const double w = q == 0 ? 2.0 / 9.0 : (q < 7 ? 1.0 / 9.0 : 1.0 / 72.0);
    const double cu = 3.0 * (c_q15[q][0] * jx + c_q15[q][1] * jy + c_q15[q][2] * jz);
    const double feq = w * (rho + cu) + w * g;
    dst[q * arr + c] = f[q] + omega * (feq - f[q]);
  }
  fd[c] = lap;
}

}  // namespace wsv

extern "C" ws_status ws_validate_stencil25(void* cuda_stream, const double* d_src, double* d_dst, const int64_t n[3],
                                           const uint32_t block[3], const uint32_t fold[3], uint32_t reps,
                                           double* ms_avg) {
  if (!d_src || !d_dst || !n || !block || !fold) return WS_EINVAL;
  if (fold[0] != 1 || fold[1] < 1 || fold[1] > 2 || fold[2] < 1 || fold[2] > 2 || fold[1] * fold[2] > 2) return WS_EINVAL;
  if (block[0] * block[1] * block[2] == 0 || block[0] * block[1] * block[2] > 1024 || block[2] > 64) return WS_ELIMIT;
  for (int d = 0; d < 3; ++d)
    if (n[d] < 1 || n[d] > (1 << 20)) return WS_EINVAL;
  static const double w[5] = {-7.5, 1.6, -0.2, 0.025, -0.0017857142857142857};
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (cudaMemcpyToSymbolAsync(wsv::c_w, w, sizeof(w), 0, cudaMemcpyHostToDevice, st) != cudaSuccess) return WS_ECUDA;
  const long long py = n[0] + 8, pz = py * (n[1] + 8);
  const dim3 b(block[0], block[1], block[2]);
  const dim3 g((unsigned)((n[0] + block[0] - 1) / block[0]), (unsigned)((n[1] + block[1] * fold[1] - 1) / (block[1] * fold[1])),
               (unsigned)((n[2] + block[2] * fold[2] - 1) / (block[2] * fold[2])));
  if (g.y > 65535 || g.z > 65535) return WS_ELIMIT;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (uint32_t r = 0; r < (reps ? reps : 1); ++r) {
    if (fold[1] == 2) wsv::k_st25<2, 1><<<g, b, 0, st>>>(d_src, d_dst, (int)n[0], (int)n[1], (int)n[2], py, pz);
    else if (fold[2] == 2) wsv::k_st25<1, 2><<<g, b, 0, st>>>(d_src, d_dst, (int)n[0], (int)n[1], (int)n[2], py, pz);
    else wsv::k_st25<1, 1><<<g, b, 0, st>>>(d_src, d_dst, (int)n[0], (int)n[1], (int)n[2], py, pz);
  }
  cudaEventRecord(e1, st);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) return WS_ECUDA;
  if (ms_avg) *ms_avg = (double)ms / (double)(reps ? reps : 1);
  return WS_OK;
}

extern "C" ws_status ws_validate_lbm15(void* cuda_stream, const double* d_src, double* d_dst, const double* d_phi,
                                       double* d_fd, const int64_t n[3], const uint32_t block[3], uint32_t reps,
                                       double* ms_avg) {
  if (!d_src || !d_dst || !d_phi || !d_fd || !n || !block) return WS_EINVAL;
  if (block[0] * block[1] * block[2] == 0 || block[0] * block[1] * block[2] > 1024 || block[2] > 64) return WS_ELIMIT;
  for (int d = 0; d < 3; ++d)
    if (n[d] < 1 || n[d] > (1 << 20)) return WS_EINVAL;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const long long py = n[0] + 2, pz = py * (n[1] + 2), arr = pz * (n[2] + 2);
  const dim3 b(block[0], block[1], block[2]);
  const dim3 g((unsigned)((n[0] + block[0] - 1) / block[0]), (unsigned)((n[1] + block[1] - 1) / block[1]),
               (unsigned)((n[2] + block[2] - 1) / block[2]));
  if (g.y > 65535 || g.z > 65535) return WS_ELIMIT;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (uint32_t r = 0; r < (reps ? reps : 1); ++r)
    wsv::k_lbm15<<<g, b, 0, st>>>(d_src, d_dst, d_phi, d_fd, (int)n[0], (int)n[1], (int)n[2], py, pz, arr);
  cudaEventRecord(e1, st);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) return WS_ECUDA;
  if (ms_avg) *ms_avg = (double)ms / (double)(reps ? reps : 1);
  return WS_OK;
}
