// Measured fp64 issue peak of the GPU: independent DFMA / DADD / DMUL chains
// in registers, every SM filled, timed with CUDA events.  The result is the
// denominator of K_P's "fp64_frac" (bench.py): K_P is bound by the fp64 pipe
// and instruction issue, not by HBM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
//   ./fp64_peak > profiles/fp64_peak.json
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) chains(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = a + k * 1e-3 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (OP == 0) x[k] = __fma_rn(x[k], b, a);
        if (OP == 1) x[k] = __dadd_rn(x[k], b);
        if (OP == 2) x[k] = __dmul_rn(x[k], b);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;   // keeps the chains alive
}

template <int OP>
double run(double* out, int sms, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  chains<OP><<<blocks, threads>>>(out, iters / 10, 1.0000001, 0.9999999);   // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    chains<OP><<<blocks, threads>>>(out, iters, 1.0000001, 0.9999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double insts = (double)blocks * threads * iters * 32.0;   // thread-instructions
  return insts / (best * 1e-3);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000;
  const double fma = run<0>(out, p.multiProcessorCount, iters);
  const double add = run<1>(out, p.multiProcessorCount, iters);
  const double mul = run<2>(out, p.multiProcessorCount, iters);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_khz_max\": %d, "
         "\"dfma_per_s\": %.6e, \"dadd_per_s\": %.6e, \"dmul_per_s\": %.6e, "
         "\"tflops\": %.3f, \"fp64_inst_per_clk_per_sm\": %.2f, "
         "\"how\": \"8 independent chains per thread, 256 threads x 8 CTAs per SM, best of 5, "
         "CUDA events; tflops = 2 x DFMA/s; per-clock figure at the max SM clock\"}\n",
         p.name, p.multiProcessorCount, clk, fma, add, mul, 2.0 * fma / 1e12,
         fma / ((double)clk * 1e3) / p.multiProcessorCount);
  return 0;
}
