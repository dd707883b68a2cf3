// k_krylov.cuh -- vector kernels of the GMRES solve of BIE 5.4 (NEXT-2).
// Dot products use a fixed grid and a fixed-order two-pass reduction, so
// every Krylov iterate is bitwise reproducible run to run.
#pragma once
#include "common.cuh"

namespace bie {

constexpr int kDotBlocks = 592;  // 4 x 148 SMs; fixed => deterministic
constexpr int kDotThreads = 256;

// y = a x + b y
__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b,
                        double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// part[b] = sum over the grid-stride slice of block b of x_i y_i
__global__ void __launch_bounds__(kDotThreads) k_dot_partial(int64_t n, const double* __restrict__ x,
                                                             const double* __restrict__ y,
                                                             double* __restrict__ part) {
  __shared__ double red[kDotThreads / 32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kDotThreads + threadIdx.x; i < n;
       i += (int64_t)kDotBlocks * kDotThreads)
    s = fma(x[i], y[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// out[0] = sum_b part[b] in fixed order
__global__ void __launch_bounds__(kDotThreads) k_dot_final(const double* __restrict__ part,
                                                           double* __restrict__ out) {
  __shared__ double red[kDotThreads / 32];
  double s = 0.0;
  for (int b = threadIdx.x; b < kDotBlocks; b += kDotThreads) s += part[b];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

}  // namespace bie

namespace bie {

// part[i][b] = block b's partial of  V_i . w,  i < nv   (fixed grid).  Four
// vectors per pass share the loads of w and one barrier; each partial is
// reduced exactly as block_sum does (per-thread fma chain, warp xor tree,
// then warp q's xor tree over the warp sums of vector q), so the values are
// those of one block_sum per vector.
__global__ void __launch_bounds__(kDotThreads) k_mdot_partial(int64_t n, int nv,
                                                              const double* __restrict__ V,
                                                              const double* __restrict__ w,
                                                              double* __restrict__ part) {
  constexpr int NW = kDotThreads / 32, G = 4;
  static_assert(NW >= G, "one warp per vector of a group");
  __shared__ double red[G][NW];
  const int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i0 = 0; i0 < nv; i0 += G) {
    const int g = min(G, nv - i0);
    double s[G] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t e = blockIdx.x * (int64_t)kDotThreads + threadIdx.x; e < n;
         e += (int64_t)kDotBlocks * kDotThreads) {
      const double we = w[e];
#pragma unroll
      for (int q = 0; q < G; ++q)
        if (q < g) s[q] = fma(V[(int64_t)(i0 + q) * n + e], we, s[q]);
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      double v = s[q];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (l == 0) red[q][wi] = v;
    }
    __syncthreads();
    if (wi < g) {
      double v = l < NW ? red[wi][l] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (l == 0) part[(int64_t)(i0 + wi) * kDotBlocks + blockIdx.x] = v;
    }
    __syncthreads();
  }
}

// out[i] (+)= sum_b part[i][b]   (one block per vector; accumulate: out[i] += ...)
__global__ void __launch_bounds__(kDotThreads) k_mdot_final(const double* __restrict__ part,
                                                            double* __restrict__ out, int accumulate) {
  __shared__ double red[kDotThreads / 32];
  double s = 0.0;
  for (int b = threadIdx.x; b < kDotBlocks; b += kDotThreads) s += part[(int64_t)blockIdx.x * kDotBlocks + b];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = accumulate ? out[blockIdx.x] + s : s;
}

// w -= sum_i h_i V_i   (h on the device; fixed order in i)
__global__ void k_maxpy(int64_t n, int nv, const double* __restrict__ h,
                        const double* __restrict__ V, double* __restrict__ w) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = w[e];
    for (int i = 0; i < nv; ++i) s = fma(-h[i], V[(int64_t)i * n + e], s);
    w[e] = s;
  }
}

}  // namespace bie
