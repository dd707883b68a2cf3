// nbody_const.cu -- measurement: the far-field S+D pair step with the source
// records read as CONSTANT-BANK operands (uniform datapath: the FP64
// instructions take the source coordinates, normal and densities from
// c[3][..] / uniform registers, so none needs three fresh 64-bit reads from
// the vector register file) against the shared-memory broadcast formulation
// of k_nbody (LDS.128 into vector registers), same arithmetic, same targets
// per thread.  The register-file read model caps k_nbody's
// FP64 pipe at ~0.90; DFMA with a constant operand measures 0.997
// (profiles/r02_fp64_peak.json, DFMA_CB).  Timing and a consistency check
// only; not part of the library.
//   u_i += y [f'_k + rho (rho.f'_k + (rho.n_k)(rho.q'_k) y^2) y^2],  rho = x_i - x_k
// Constant memory holds KC = 680 records (65,280 B); a launch processes all
// targets against one batch of KC sources (the probe repeats the same batch).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v \
//          -o tools/nbody_const tools/nbody_const.cu
// Run:   tools/nbody_const [waves] [reps]
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_1707_06551_b200/csrc/common.cuh"

using namespace bie;

constexpr int TPB = 64;
constexpr int KC = 680;  // records per constant batch (multiple of 8)

#ifndef BATCHED
__constant__ double2 c_src[KC * 6];
#endif

__device__ __forceinline__ double rsq(double r2) {
  const double y0 = rsqrt_seed(r2);
  const double e = fma(-r2, y0 * y0, 1.0);
  return y0 * fma(e, fma(e, 0.375, 0.5), 1.0);
}

template <int R>
__device__ __forceinline__ void pair_g(const double2 s0, const double2 s1, const double2 s2, const double2 s3,
                                       const double2 s4, const double2 s5, const double (*xt)[3],
                                       double (*acc)[3]) {
  // s0=(x0,x1) s1=(x2,n0) s2=(n1,n2) s3=(f0,f1) s4=(f2,q0) s5=(q1,q2)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double dx = xt[r][0] - s0.x, dy = xt[r][1] - s0.y, dz = xt[r][2] - s1.x;
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    const double y = rsq(r2);
    const double rn = fma(dz, s2.y, fma(dy, s2.x, dx * s1.y));
    const double rq = fma(dz, s5.y, fma(dy, s5.x, dx * s4.y));
    const double y2 = y * y;
#ifdef T2CHAIN  // rho.f' accumulated onto (rho.n)(rho.q') y^2: no DFMA with three register operands
    const double t2 = fma(dz, s4.x, fma(dy, s3.y, fma(dx, s3.x, (rn * rq) * y2)));
#else
    const double rf = fma(dz, s4.x, fma(dy, s3.y, dx * s3.x));
    const double t2 = fma(rn * rq, y2, rf);
#endif
    const double sp = t2 * y2;
    acc[r][0] = fma(y, fma(dx, sp, s3.x), acc[r][0]);
    acc[r][1] = fma(y, fma(dy, sp, s3.y), acc[r][1]);
    acc[r][2] = fma(y, fma(dz, sp, s4.x), acc[r][2]);
  }
}

#ifndef BATCHED
// sources from the constant bank
template <int R, int UNR>
__global__ void __launch_bounds__(TPB, 1) k_const(const double* __restrict__ tx, double* u, int nrep) {
  double xt[R][3], acc[R][3];
  const int64_t t0 = (int64_t)blockIdx.x * TPB * R + threadIdx.x;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xt[r][c] = tx[(t0 + r * TPB) * 3 + c];
      acc[r][c] = 0.0;
    }
  for (int rep = 0; rep < nrep; ++rep) {
#pragma unroll UNR
    for (int s = 0; s < KC; ++s) {
      const double2* sr = c_src + s * 6;
      pair_g<R>(sr[0], sr[1], sr[2], sr[3], sr[4], sr[5], xt, acc);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) u[(t0 + r * TPB) * 3 + c] = acc[r][c];
}

// sources staged in shared memory, broadcast LDS.128 (what k_nbody does)
template <int R, int UNR>
__global__ void __launch_bounds__(TPB, 1) k_smem(const double* __restrict__ rec, const double* __restrict__ tx,
                                                 double* u, int nrep) {
  extern __shared__ double2 srec[];  // KC * 6
  double xt[R][3], acc[R][3];
  const int64_t t0 = (int64_t)blockIdx.x * TPB * R + threadIdx.x;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xt[r][c] = tx[(t0 + r * TPB) * 3 + c];
      acc[r][c] = 0.0;
    }
  const double2* g2 = reinterpret_cast<const double2*>(rec);
  for (int e = threadIdx.x; e < KC * 6; e += TPB) srec[e] = g2[e];
  __syncthreads();
  for (int rep = 0; rep < nrep; ++rep) {
#pragma unroll UNR
    for (int s = 0; s < KC; ++s) {
      const double2* sr = srec + s * 6;
      pair_g<R>(sr[0], sr[1], sr[2], sr[3], sr[4], sr[5], xt, acc);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) u[(t0 + r * TPB) * 3 + c] = acc[r][c];
}

#endif

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

#ifndef BATCHED
template <int R, int UNR>
static int run(int waves, int reps, int nrep, const double* d_rec, const std::vector<double>& h_tx_all) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int occ_c = 0, occ_s = 0;
  constexpr int kSmem = KC * 96;
  CK(cudaFuncSetAttribute(k_smem<R, UNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, k_const<R, UNR>, TPB, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_smem<R, UNR>, TPB, kSmem));
  const int occ = occ_c < occ_s ? occ_c : occ_s;  // same grid for both
  const int grid = prop.multiProcessorCount * occ * waves;
  const int64_t M = (int64_t)grid * TPB * R;
  double *d_tx, *d_u1, *d_u2;
  CK(cudaMalloc(&d_tx, M * 3 * 8));
  CK(cudaMalloc(&d_u1, M * 3 * 8));
  CK(cudaMalloc(&d_u2, M * 3 * 8));
  std::vector<double> h_tx(M * 3);
  for (int64_t i = 0; i < M * 3; ++i) h_tx[i] = h_tx_all[i % h_tx_all.size()];
  CK(cudaMemcpy(d_tx, h_tx.data(), M * 3 * 8, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms_c = 1e30f, ms_s = 1e30f;
  for (int it = 0; it < reps + 1; ++it) {
    float ms;
    CK(cudaEventRecord(e0));
    k_const<R, UNR><<<grid, TPB>>>(d_tx, d_u1, nrep);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (it && ms < ms_c) ms_c = ms;
    CK(cudaEventRecord(e0));
    k_smem<R, UNR><<<grid, TPB, kSmem>>>(d_rec, d_tx, d_u2, nrep);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (it && ms < ms_s) ms_s = ms;
  }
  CK(cudaGetLastError());
  std::vector<double> u1(M * 3), u2(M * 3);
  CK(cudaMemcpy(u1.data(), d_u1, M * 3 * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(u2.data(), d_u2, M * 3 * 8, cudaMemcpyDeviceToHost));
  double md = 0, mx = 0;
  for (int64_t i = 0; i < M * 3; ++i) {
    const double d = u1[i] - u2[i];
    md = d * d > md ? d * d : md;
    mx = u2[i] * u2[i] > mx ? u2[i] * u2[i] : mx;
  }
  const double pairs = (double)M * KC * nrep;
  printf("{\"tool\": \"nbody_const\", \"R\": %d, \"UNR\": %d, \"occ_const\": %d, \"occ_smem\": %d, \"grid\": %d, "
         "\"targets\": %lld, \"pairs\": %.4g, \"ms_const\": %.4f, \"ms_smem\": %.4f, \"pairs_per_s_const\": %.4g, "
         "\"pairs_per_s_smem\": %.4g, \"ratio\": %.4f, \"max_abs_diff\": %.3g, \"max_abs\": %.3g}\n",
         R, UNR, occ_c, occ_s, grid, (long long)M, pairs, ms_c, ms_s, pairs / ms_c * 1e3, pairs / ms_s * 1e3,
         ms_s / ms_c, sqrt(md), sqrt(mx));
  cudaFree(d_tx);
  cudaFree(d_u1);
  cudaFree(d_u2);
  return 0;
}

#endif

#ifdef BATCHED
// ---- the schedule a library version would need: batches of KB = 340 records
// (32,640 B; the 64 KB constant bank holds two such buffers), even batches on
// stream 0 / buffer A / accumulator A, odd batches on stream 1 / buffer B /
// accumulator B, so that one launch's tail overlaps the other stream's launch;
// every launch adds its batch to its accumulator (read-modify-write).
#ifndef NBUF
#define NBUF 2  // constant buffers = streams (-DNBUF=3, 4: more, smaller batches)
#endif
constexpr int KB = (680 / NBUF) / 4 * 4;
__constant__ double2 c_buf[NBUF][KB * 6];

template <int R, int UNR, int BUF>
__global__ void __launch_bounds__(TPB, 1) k_constb(const double* __restrict__ tx, double* acc_io, int64_t M, int ks) {
  double xt[R][3], acc[R][3];
  const int64_t t0 = (int64_t)blockIdx.x * TPB * R + threadIdx.x;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t t = t0 + r * TPB < M ? t0 + r * TPB : M - 1;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xt[r][c] = tx[t * 3 + c];
      acc[r][c] = acc_io[t * 3 + c];
    }
  }
  const double2* cs = c_buf[BUF];
#pragma unroll UNR
  for (int s = 0; s < ks; ++s) {
    const double2* sr = cs + s * 6;
    pair_g<R>(sr[0], sr[1], sr[2], sr[3], sr[4], sr[5], xt, acc);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t t = t0 + r * TPB;
    if (t < M) {
#pragma unroll
      for (int c = 0; c < 3; ++c) acc_io[t * 3 + c] = acc[r][c];
    }
  }
}

template <int R, int UNR>
static int run_real(int64_t M, int64_t N, int reps) {
  std::mt19937_64 g(11);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> h_rec(N * 12), h_tx(M * 3);
  for (int64_t k = 0; k < N; ++k) {
    for (int c = 0; c < 3; ++c) h_rec[k * 12 + c] = 4.0 * U(g);
    for (int c = 3; c < 12; ++c) h_rec[k * 12 + c] = U(g);
  }
  for (int64_t i = 0; i < M * 3; ++i) h_tx[i] = 10.0 + 4.0 * U(g);
  double *d_rec, *d_tx, *d_acc[NBUF];
  CK(cudaMalloc(&d_rec, N * 96));
  CK(cudaMalloc(&d_tx, M * 24));
  for (int w = 0; w < NBUF; ++w) CK(cudaMalloc(&d_acc[w], M * 24));
  CK(cudaMemcpy(d_rec, h_rec.data(), N * 96, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tx, h_tx.data(), M * 24, cudaMemcpyHostToDevice));
  cudaStream_t st[NBUF];
  for (int w = 0; w < NBUF; ++w) CK(cudaStreamCreateWithFlags(&st[w], cudaStreamNonBlocking));
  cudaEvent_t e0, e1, ej;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
  const unsigned grid = (unsigned)((M + TPB * R - 1) / (TPB * R));
  const int64_t nb = (N + KB - 1) / KB;
  for (int nstream = 1; nstream <= NBUF; ++nstream) {
    float best = 1e30f;
    for (int it = 0; it < reps; ++it) {
      for (int w = 0; w < NBUF; ++w) CK(cudaMemsetAsync(d_acc[w], 0, M * 24, st[0]));
      CK(cudaEventRecord(e0, st[0]));
      CK(cudaEventRecord(ej, st[0]));
      for (int w = 1; w < NBUF; ++w) CK(cudaStreamWaitEvent(st[w], ej, 0));
      for (int64_t b = 0; b < nb; ++b) {
        const int w = (int)(b % nstream);
        const int ks = (int)std::min<int64_t>(KB, N - b * KB);
        CK(cudaMemcpyToSymbolAsync(c_buf, d_rec + b * KB * 12, (size_t)ks * 96, (size_t)w * KB * 96,
                                   cudaMemcpyDeviceToDevice, st[w]));
        switch (w) {
          case 0: k_constb<R, UNR, 0><<<grid, TPB, 0, st[0]>>>(d_tx, d_acc[0], M, ks); break;
          case 1: k_constb<R, UNR, 1><<<grid, TPB, 0, st[1]>>>(d_tx, d_acc[1], M, ks); break;
#if NBUF > 2
          case 2: k_constb<R, UNR, 2><<<grid, TPB, 0, st[2]>>>(d_tx, d_acc[2], M, ks); break;
#endif
#if NBUF > 3
          case 3: k_constb<R, UNR, 3><<<grid, TPB, 0, st[3]>>>(d_tx, d_acc[3], M, ks); break;
#endif
        }
      }
      for (int w = 1; w < NBUF; ++w) {
        CK(cudaEventRecord(ej, st[w]));
        CK(cudaStreamWaitEvent(st[0], ej, 0));
      }
      CK(cudaEventRecord(e1, st[0]));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    // consistency: a few targets against a host sum in the same arithmetic order is not
    // needed here (the single-batch run above checks the arithmetic); report checksums
    std::vector<double> a0(M * 3);
    double cs = 0;
    for (int w = 0; w < NBUF; ++w) {
      CK(cudaMemcpy(a0.data(), d_acc[w], M * 24, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < M * 3; ++i) cs += a0[i];
    }
    const double pairs = (double)M * (double)N;
    printf("{\"tool\": \"nbody_const\", \"mode\": \"batched\", \"R\": %d, \"UNR\": %d, \"streams\": %d, \"KB\": %d, "
           "\"targets\": %lld, \"sources\": %lld, \"launches\": %lld, \"grid\": %u, \"ms\": %.3f, "
           "\"pairs_per_s\": %.4g, \"checksum\": %.17g}\n",
           R, UNR, nstream, KB, (long long)M, (long long)N, (long long)nb, grid, best, pairs / best * 1e3, cs);
    fflush(stdout);
  }
  cudaFree(d_rec);
  cudaFree(d_tx);
  for (int w = 0; w < NBUF; ++w) cudaFree(d_acc[w]);
  return 0;
}

#endif

int main(int argc, char** argv) {
#ifdef BATCHED
  const int64_t M = argc > 1 ? atoll(argv[1]) : 980000;
  const int64_t N = argc > 2 ? atoll(argv[2]) : 980000;
  const int reps = argc > 3 ? atoi(argv[3]) : 2;
  if (run_real<8, 4>(M, N, reps)) return 1;
  if (run_real<8, 8>(M, N, reps)) return 1;
  return 0;
#else
  const int waves = argc > 1 ? atoi(argv[1]) : 2;
  const int reps = argc > 2 ? atoi(argv[2]) : 3;
  const int nrep = argc > 3 ? atoi(argv[3]) : 8;
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> h_rec(KC * 12), h_tx(3 * 65536);
  for (int k = 0; k < KC; ++k) {
    for (int c = 0; c < 3; ++c) h_rec[k * 12 + c] = 4.0 * U(g);                   // x in [-4, 4]^3
    for (int c = 3; c < 12; ++c) h_rec[k * 12 + c] = U(g);
  }
  for (size_t i = 0; i < h_tx.size(); ++i) h_tx[i] = 10.0 + 4.0 * U(g);           // targets away from the sources
  double* d_rec;
  CK(cudaMalloc(&d_rec, KC * 12 * 8));
  CK(cudaMemcpy(d_rec, h_rec.data(), KC * 12 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpyToSymbol(c_src, h_rec.data(), KC * 12 * 8));
  if (run<8, 2>(waves, reps, nrep, d_rec, h_tx)) return 1;
  if (run<8, 4>(waves, reps, nrep, d_rec, h_tx)) return 1;
  if (run<6, 2>(waves, reps, nrep, d_rec, h_tx)) return 1;
  if (run<4, 4>(waves, reps, nrep, d_rec, h_tx)) return 1;
  return 0;
#endif
}
