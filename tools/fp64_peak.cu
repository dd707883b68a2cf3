// fp64_peak.cu -- microbenchmark of the B200 FP64 pipe (no measured
// FP64 peak exists).  Each thread runs 8 independent DFMA chains; the kernel
// is sized to many waves.  Reports DFMA/s, FP64 TFLOP/s (FMA = 2 flops) and
// the SM clock implied by 64 FP64 lanes per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_chains(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void dmul_chains(double* out, int iters, double a) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k + 1.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = x[k] * a;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = prop.multiProcessorCount * 8, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int kind = 0; kind < 2; ++kind) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) dfma_chains<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
      else dmul_chains<<<blocks, threads>>>(out, iters, 0.9999999);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    const double ops = (double)blocks * threads * iters * 8;
    const double per_s = ops / (best * 1e-3);
    printf("{\"op\": \"%s\", \"sms\": %d, \"ms\": %.3f, \"ops_per_s\": %.4e, \"tflops\": %.3f, "
           "\"implied_clock_mhz_at_64_lanes\": %.1f}\n",
           kind == 0 ? "DFMA" : "DMUL", prop.multiProcessorCount, best, per_s,
           per_s * (kind == 0 ? 2.0 : 1.0) / 1e12, per_s / (prop.multiProcessorCount * 64.0) / 1e6);
  }
  return 0;
}
