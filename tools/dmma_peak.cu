// dmma_peak.cu -- does FP64 tensor-core MMA (mma.sync m8n8k4 f64, SASS DMMA)
// beat, or add to, CUDA-core DFMA on B200?  (BASELINE.json north star: "fp64
// DMMA tensor cores only if ncu shows they beat CUDA-core FMA".)
// Three kernels, each sized to many waves:
//   dfma  : 8 independent DFMA chains per thread
//   dmma  : 4 independent m8n8k4 accumulators per warp
//   mixed : even warps run the dmma loop, odd warps the dfma loop
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int MODE>  // 0 dfma, 1 dmma, 2 mixed
__global__ void bench(double* out, int iters, double a, double b) {
  const int warp = threadIdx.x >> 5;
  const bool do_mma = MODE == 1 || (MODE == 2 && (warp & 1) == 0);
  double s = 0.0;
  if (do_mma) {
    double c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = threadIdx.x * 1e-9 + k;
    const double av = a + threadIdx.x * 1e-12, bv = b - threadIdx.x * 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma(c[2 * k], c[2 * k + 1], av, bv);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k];
  } else {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
    // 2x the loop count so one dfma-warp iteration ~ one dmma-warp iteration in flops
    for (int i = 0; i < iters * (MODE == 2 ? 4 : 1); ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = prop.multiProcessorCount * 8, iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"dfma", "dmma", "mixed"};
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) bench<0><<<blocks, threads>>>(out, iters * 4, 0.9999999, 1e-7);
      if (mode == 1) bench<1><<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
      if (mode == 2) bench<2><<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    const double warps = (double)blocks * threads / 32;
    // flops: dfma thread-op = 2 flops; dmma m8n8k4 = 2*8*8*4 = 512 flops per warp-instr
    double flops = 0;
    if (mode == 0) flops = warps * 32 * 8.0 * iters * 4 * 2;
    if (mode == 1) flops = warps * 4.0 * iters * 512;
    if (mode == 2) flops = warps / 2 * 4.0 * iters * 512 + warps / 2 * 32 * 8.0 * iters * 4 * 2;
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"tflops\": %.3f}\n", names[mode], best,
           flops / (best * 1e-3) / 1e12);
  }
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
