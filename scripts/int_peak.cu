// int_peak.cu -- measured integer-issue peak of this B200 (the roofline denominator of the
// integer-bound estimator kernels; VERDICT r01 "measure an integer-issue peak").
//
// Each thread runs ITER iterations of 8 independent dependency chains (ILP 8) of one op mix;
// the grid fills every SM (148 x 8 CTAs x 256 threads).  Lane-ops/s = threads x ITER x ops per
// iteration / CUDA-event time (best of 5, after a warm-up).  Mixes:
//   alu   : IADD3 + LOP3 (+ SHF)          -- the ALU pipe only
//   mix   : IADD3 + LOP3 + IMAD           -- ALU + FMA pipes (the estimator kernels' mix)
//   shfl  : mix + one SHFL per 8 ops      -- with warp shuffles (ordered reductions)
// Results are written so nothing is dead code; SASS: cuobjdump -sass scripts/int_peak | grep -c IADD3.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/int_peak scripts/int_peak.cu
//   scripts/int_peak > profiles/r02_int_peak.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

template <int MODE>
__global__ void __launch_bounds__(256) k_int(unsigned* out, unsigned seed) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u + blockIdx.x;
  const unsigned k1 = seed | 1u, k2 = seed ^ 0x5bd1e995u;
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {         // IADD3, LOP3, IADD3, SHF-free LOP3: 4 ops
        a[i] = a[i] + k1 + it;
        a[i] = (a[i] ^ k2) & (a[i] | k1);
        a[i] = a[i] + k2 + i;
        a[i] = (a[i] & k1) ^ (a[i] | k2);
      } else {                 // IADD3, LOP3, IMAD, IMAD: 4 ops
        a[i] = a[i] + k1 + it;
        a[i] = (a[i] ^ k2) & (a[i] | k1);
        a[i] = a[i] * k1 + k2;
        a[i] = a[i] * k2 + (unsigned)i;
      }
    }
    if (MODE == 2) {           // one shuffle per 8 chains (32 ops)
      a[it & 7] += __shfl_xor_sync(0xffffffffu, a[(it + 1) & 7], 1);
    }
  }
  unsigned r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r ^= a[i];
  if (r == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = r;  // keep the chains alive
}

template <int MODE>
double run(unsigned* d, int blocks, double* best_ms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_int<MODE><<<blocks, 256>>>(d, 7u);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_int<MODE><<<blocks, 256>>>(d, 7u + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  *best_ms = best;
  const double ops = (double)blocks * 256.0 * ITER * (8 * 4 + (MODE == 2 ? 1 : 0));
  return ops / (best * 1e-3);
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz (max boost)
  unsigned* d = nullptr;
  const int blocks = nsm * 8;
  cudaMalloc(&d, (size_t)blocks * 256 * sizeof(unsigned));
  double ms[3];
  const double alu = run<0>(d, blocks, &ms[0]);
  const double mix = run<1>(d, blocks, &ms[1]);
  const double shf = run<2>(d, blocks, &ms[2]);
  const double nominal = (double)nsm * 4 * 32 * clk * 1e3;  // 4 SMSPs x 1 warp-instruction/clk x 32 lanes
  printf("{\"what\": \"measured integer lane-op throughput (scripts/int_peak.cu), best of 5 CUDA-event timings\", "
         "\"n_sm\": %d, \"max_clock_mhz\": %.0f, \"ops_per_s_alu\": %.6e, \"ops_per_s_mix\": %.6e, "
         "\"ops_per_s_mix_shfl\": %.6e, \"ms\": [%.4f, %.4f, %.4f], \"nominal_issue_peak\": %.6e, "
         "\"frac_of_nominal\": {\"alu\": %.4f, \"mix\": %.4f, \"mix_shfl\": %.4f}, "
         "\"note\": \"alu: IADD3+LOP3 (ALU pipe only); mix: IADD3+LOP3+IMAD (ALU + FMA pipes); 8 independent chains per thread\"}\n",
         nsm, clk / 1e3, alu, mix, shf, ms[0], ms[1], ms[2], nominal, alu / nominal, mix / nominal, shf / nominal);
  cudaFree(d);
  return 0;
}
