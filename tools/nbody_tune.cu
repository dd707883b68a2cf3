// nbody_tune.cu -- sweep launch/blocking variants of k_nbody on synthetic
// sphere-grouped sources (timing only; parity is the test suite's job).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v \
//          -o tools/nbody_tune tools/nbody_tune.cu
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_1707_06551_b200/csrc/k_nbody.cuh"

using namespace bie;

template <int R, int TPB, int TS, int NST, bool OFF, int MINB, int UNR, int MODE = 0>
void run(const char* name, const NbodyArgs& base, int sm, double pairs, int reps) {
  auto kern = k_nbody<R, TPB, TS, NST, OFF, MINB, UNR, MODE>;
  const int smem = NbodySmem<TS, NST, OFF>::kBytes;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TPB, smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  NbodyArgs A = base;
  const int tile = R * TPB;
  A.n_tt = (int)((A.M + tile - 1) / tile);
  const int64_t n_src_tiles = (A.N + TS - 1) / TS;
  int64_t S = (64LL * sm * occ + A.n_tt - 1) / A.n_tt;
  S = std::min<int64_t>(S, std::max<int64_t>(1, n_src_tiles / 4));
  A.tiles_per_chunk = (int)((n_src_tiles + S - 1) / S);
  A.n_chunks = (int)((n_src_tiles + A.tiles_per_chunk - 1) / A.tiles_per_chunk);
  double* part;
  cudaMalloc(&part, (size_t)A.n_chunks * 4 * A.M * sizeof(double));
  A.uout = part;
  A.pout = (OFF && MODE == 0) ? part + (size_t)A.n_chunks * 3 * A.M : nullptr;
  A.uinit = nullptr;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f, tot = 0.f;
  for (int r = 0; r < reps + 1; ++r) {
    cudaEventRecord(e0);
    kern<<<(unsigned)((int64_t)A.n_tt * A.n_chunks), TPB, smem>>>(A);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0) {
      best = std::min(best, ms);
      tot += ms;
    }
  }
  cudaError_t err = cudaGetLastError();
  const double ops = MODE == 1 ? 25.0 : (OFF ? 32.0 : 30.0);
  const double pps = pairs / (best * 1e-3);
  printf("{\"variant\": \"%s\", \"regs\": %d, \"occ\": %d, \"chunks\": %d, \"ms\": %.3f, \"ms_mean\": %.3f, "
         "\"pairs_per_s\": %.4e, \"pipe_frac_1965\": %.4f, \"err\": \"%s\"}\n",
         name, fa.numRegs, occ, A.n_chunks, best, tot / reps, pps,
         pps * ops / (sm * 64.0 * 1.965e9), cudaGetErrorString(err));
  fflush(stdout);
  cudaFree(part);
}

int main(int argc, char** argv) {
  const int nsn = 98;                       // p = 6
  const int64_t ns = argc > 1 ? atoll(argv[1]) : 2000;
  const int reps = argc > 2 ? atoi(argv[2]) : 3;
  const int64_t N = ns * nsn;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> rec(N * kRec + 2 * kRec), qn3(N + 2), tx(3 * N), tn(3 * N);
  for (int64_t s = 0; s < ns; ++s) {
    double c[3] = {U(g) * 30, U(g) * 30, U(g) * 30};
    for (int k = 0; k < nsn; ++k) {
      int64_t i = s * nsn + k;
      double n[3] = {U(g), U(g), U(g)};
      double r = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]) + 1e-3;
      for (int d = 0; d < 3; ++d) {
        rec[i * kRec + d] = c[d] + n[d] / r;
        rec[i * kRec + 3 + d] = n[d] / r;
        rec[i * kRec + 6 + d] = U(g) * 0.01;
        rec[i * kRec + 9 + d] = U(g) * 0.01;
        tx[3 * i + d] = c[d] + 1.7 * n[d] / r;
        tn[3 * i + d] = n[d] / r;
      }
      qn3[i] = U(g) * 0.01;
    }
  }
  double *drec, *dqn, *dtx, *dtn;
  cudaMalloc(&dtn, tn.size() * 8);
  cudaMemcpy(dtn, tn.data(), tn.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&drec, rec.size() * 8);
  cudaMalloc(&dqn, qn3.size() * 8);
  cudaMalloc(&dtx, tx.size() * 8);
  cudaMemcpy(drec, rec.data(), rec.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dqn, qn3.data(), qn3.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dtx, tx.data(), tx.size() * 8, cudaMemcpyHostToDevice);
  NbodyArgs A{};
  A.rec = drec;
  A.qn3 = dqn;
  A.tx = dtx;
  A.tn = dtn;
  A.N = N;
  A.M = N;
  A.nsn = nsn;
  A.pscale = 2.0;
  const double pairs_apply = (double)N * (N - nsn), pairs_off = (double)N * N;
  const int sm = prop.multiProcessorCount;
  printf("# N = %lld, SMs = %d\n", (long long)N, sm);
  const bool k_only = argc > 3 && argv[3][0] == 'K';  // "K": K variants only; "A": apply/off only
  if (!k_only) {
    run<8, 64, 64, 3, false, 1, 2>("apply R8 T64 u2 (library)", A, sm, pairs_apply, reps);
    run<8, 64, 64, 3, true, 1, 1>("off R8 T64 u1 (library)", A, sm, pairs_off, reps);
    run<8, 64, 64, 3, true, 1, 2>("off R8 T64 u2", A, sm, pairs_off, reps);
    run<8, 64, 128, 3, true, 1, 1>("off R8 T64 TS128 u1", A, sm, pairs_off, reps);
    run<8, 32, 64, 3, true, 1, 1>("off R8 T32 u1", A, sm, pairs_off, reps);
    run<7, 64, 64, 3, true, 1, 1>("off R7 T64 u1", A, sm, pairs_off, reps);
    run<6, 64, 64, 3, true, 1, 2>("off R6 T64 u2", A, sm, pairs_off, reps);
    run<7, 64, 64, 3, false, 1, 2>("apply R7 T64 u2", A, sm, pairs_apply, reps);
    run<7, 64, 64, 3, false, 1, 1>("apply R7 T64 u1", A, sm, pairs_apply, reps);
    run<7, 64, 64, 3, false, 1, 4>("apply R7 T64 u4", A, sm, pairs_apply, reps);
    run<8, 64, 64, 3, false, 1, 4>("apply R8 T64 u4", A, sm, pairs_apply, reps);
    run<7, 64, 64, 3, true, 1, 2>("off R7 T64 u2", A, sm, pairs_off, reps);
    run<8, 64, 64, 3, true, 1, 4>("off R8 T64 u4", A, sm, pairs_off, reps);
  }
  if (argc > 3 && argv[3][0] == 'A') return 0;
  if (argc > 3 && argv[3][0] == 'S') {  // small N (cfg 2 size): blocking vs tail/overheads
    run<8, 64, 64, 3, false, 1, 2>("apply R8 T64 (library)", A, sm, pairs_apply, reps);
    run<4, 64, 64, 3, false, 1, 2>("apply R4 T64", A, sm, pairs_apply, reps);
    run<4, 128, 64, 3, false, 1, 2>("apply R4 T128", A, sm, pairs_apply, reps);
    run<8, 32, 64, 3, false, 1, 2>("apply R8 T32", A, sm, pairs_apply, reps);
    run<6, 64, 64, 3, false, 1, 2>("apply R6 T64", A, sm, pairs_apply, reps);
    run<8, 64, 32, 3, false, 1, 2>("apply R8 T64 TS32", A, sm, pairs_apply, reps);
    return 0;
  }
  if (argc > 3 && argv[3][0] == 'P') {  // apply: pipeline depth / tile size / unroll
    run<8, 64, 64, 3, false, 1, 2>("apply R8 T64 TS64 NST3 u2 (library)", A, sm, pairs_apply, reps);
    run<8, 64, 64, 2, false, 1, 2>("apply R8 T64 TS64 NST2 u2", A, sm, pairs_apply, reps);
    run<8, 64, 64, 4, false, 1, 2>("apply R8 T64 TS64 NST4 u2", A, sm, pairs_apply, reps);
    run<8, 64, 32, 4, false, 1, 2>("apply R8 T64 TS32 NST4 u2", A, sm, pairs_apply, reps);
    run<8, 64, 128, 2, false, 1, 2>("apply R8 T64 TS128 NST2 u2", A, sm, pairs_apply, reps);
    run<8, 64, 128, 3, false, 1, 2>("apply R8 T64 TS128 NST3 u2", A, sm, pairs_apply, reps);
    run<8, 64, 64, 3, false, 1, 3>("apply R8 T64 TS64 NST3 u3", A, sm, pairs_apply, reps);
    run<8, 96, 64, 3, false, 1, 2>("apply R8 T96 TS64 NST3 u2", A, sm, pairs_apply, reps);
    run<8, 128, 64, 3, false, 1, 2>("apply R8 T128 TS64 NST3 u2", A, sm, pairs_apply, reps);
    run<7, 64, 64, 3, true, 1, 2>("off R7 T64 TS64 NST3 u2 (library)", A, sm, pairs_off, reps);
    run<7, 64, 64, 4, true, 1, 2>("off R7 T64 TS64 NST4 u2", A, sm, pairs_off, reps);
    run<7, 64, 128, 3, true, 1, 2>("off R7 T64 TS128 NST3 u2", A, sm, pairs_off, reps);
    run<7, 64, 64, 3, true, 1, 4>("off R7 T64 TS64 NST3 u4", A, sm, pairs_off, reps);
    return 0;
  }
  // traction operator K (MODE 1): apply (target normals from the records) and off-surface
  run<8, 64, 64, 3, false, 1, 2, 1>("K apply R8 T64 u2 (library)", A, sm, pairs_apply, reps);
  run<8, 64, 64, 3, false, 1, 1, 1>("K apply R8 T64 u1", A, sm, pairs_apply, reps);
  run<8, 64, 64, 3, false, 1, 4, 1>("K apply R8 T64 u4", A, sm, pairs_apply, reps);
  run<7, 64, 64, 3, false, 1, 1, 1>("K apply R7 T64 u1", A, sm, pairs_apply, reps);
  run<7, 64, 64, 3, false, 1, 4, 1>("K apply R7 T64 u4", A, sm, pairs_apply, reps);
  run<7, 64, 64, 3, false, 1, 2, 1>("K apply R7 T64 u2", A, sm, pairs_apply, reps);
  run<6, 64, 64, 3, false, 1, 2, 1>("K apply R6 T64 u2", A, sm, pairs_apply, reps);
  run<6, 64, 64, 3, false, 1, 1, 1>("K apply R6 T64 u1", A, sm, pairs_apply, reps);
  run<4, 128, 64, 3, false, 1, 2, 1>("K apply R4 T128 u2", A, sm, pairs_apply, reps);
  run<8, 32, 64, 3, false, 1, 2, 1>("K apply R8 T32 u2", A, sm, pairs_apply, reps);
  run<8, 64, 64, 3, true, 1, 1, 1>("K off R8 T64 u1 (library)", A, sm, pairs_off, reps);
  run<8, 64, 64, 3, true, 1, 2, 1>("K off R8 T64 u2", A, sm, pairs_off, reps);
  run<6, 64, 64, 3, true, 1, 2, 1>("K off R6 T64 u2", A, sm, pairs_off, reps);
  run<7, 64, 64, 3, true, 1, 2, 1>("K off R7 T64 u2", A, sm, pairs_off, reps);
  run<6, 64, 64, 3, true, 1, 1, 1>("K off R6 T64 u1", A, sm, pairs_off, reps);
  return 0;
}
