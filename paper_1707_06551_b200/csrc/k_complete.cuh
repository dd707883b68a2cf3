// k_complete.cuh -- completion operator of the mobility BIE (eq 5.8,
// P:490-491), reading R22: for x on sphere s,
//   L[mu](x) = F_s + T_s x (x - c_s),
//   F_s = sum_{k in s} w_k mu_k,  T_s = sum_{k in s} w_k (x_k - c_s) x mu_k,
// one rank-6 block per sphere.  One CTA per sphere: the six moments are
// reduced in a fixed order (strided per-thread sums, fixed shuffle tree,
// warps summed in index order), so the result is bitwise reproducible; the
// second pass adds the rigid field to u.  HBM-bound and tiny (the nodes,
// weights and mu are read once, u read and written once).
#pragma once
#include "common.cuh"

namespace bie {

constexpr int kCompleteThreads = 128;

__global__ void __launch_bounds__(kCompleteThreads) k_completion(
    int nsn, const double* __restrict__ centres, const double* __restrict__ x,
    const double* __restrict__ w, const double* __restrict__ mu, double* __restrict__ u) {
  __shared__ double red[kCompleteThreads / 32][6];
  __shared__ double mom[6];
  const int s = blockIdx.x, tid = threadIdx.x;
  const double c0 = centres[3 * s], c1 = centres[3 * s + 1], c2 = centres[3 * s + 2];
  const int64_t base = (int64_t)s * nsn;
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int k = tid; k < nsn; k += kCompleteThreads) {
    const int64_t i = base + k;
    const double wk = w[i];
    const double d0 = x[3 * i] - c0, d1 = x[3 * i + 1] - c1, d2 = x[3 * i + 2] - c2;
    const double m0 = wk * mu[3 * i], m1 = wk * mu[3 * i + 1], m2 = wk * mu[3 * i + 2];
    acc[0] += m0;
    acc[1] += m1;
    acc[2] += m2;
    acc[3] += d1 * m2 - d2 * m1;
    acc[4] += d2 * m0 - d0 * m2;
    acc[5] += d0 * m1 - d1 * m0;
  }
#pragma unroll
  for (int e = 0; e < 6; ++e)
    for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  if ((tid & 31) == 0)
#pragma unroll
    for (int e = 0; e < 6; ++e) red[tid >> 5][e] = acc[e];
  __syncthreads();
  if (tid < 6) {
    double v = 0.0;
    for (int q = 0; q < kCompleteThreads / 32; ++q) v += red[q][tid];
    mom[tid] = v;
  }
  __syncthreads();
  const double F0 = mom[0], F1 = mom[1], F2 = mom[2], T0 = mom[3], T1 = mom[4], T2 = mom[5];
  for (int k = tid; k < nsn; k += kCompleteThreads) {
    const int64_t i = base + k;
    const double d0 = x[3 * i] - c0, d1 = x[3 * i + 1] - c1, d2 = x[3 * i + 2] - c2;
    u[3 * i] += F0 + (T1 * d2 - T2 * d1);
    u[3 * i + 1] += F1 + (T2 * d0 - T0 * d2);
    u[3 * i + 2] += F2 + (T0 * d1 - T1 * d0);
  }
}

}  // namespace bie
