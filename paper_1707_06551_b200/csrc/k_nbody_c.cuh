// k_nbody_c.cuh -- the far-field pair sum of k_nbody.cuh (rows a3, a7; eqs
// 2.19-2.21 with R1 under the smooth rule eq 4.4; same pair_acc arithmetic)
// with the SOURCE records read as constant-bank operands.
//
// Why: k_nbody reads each source from shared memory into vector registers, and
// its FP64 pipe stops at ~88 % because a DFMA with three fresh 64-bit register
// operands needs three register-file read cycles.  A source
// is the same for every thread, so it can live on the uniform datapath instead:
// ptxas loads c[3][..] into uniform registers (SASS LDCU.64) and the
// DADD/DMUL/DFMA take them as UR operands, which cost no vector register-file
// read (tools/nbody_const.cu: 5.81e11 vs 5.45e11 pairs/s on the cfg 5 shape).
//
// Schedule (host side in bie.cu, run_const_pass): the sources
// are cut into batches of kCB records; a batch is copied device-to-device
// into one of two constant buffers (the 64 KB bank holds 2 x kCB x 104 B) and
// ONE launch adds its contribution at every target to an accumulator
// (read-modify-write, fixed batch order).  Even batches use buffer 0 /
// accumulator A on the caller's stream, odd batches buffer 1 / accumulator B
// on a side stream, so the ragged last wave of one launch overlaps the other
// stream's launch; a final pass adds B to A.  Deterministic: the batch ->
// accumulator assignment and the order within each are fixed.  A pass walks
// the targets in sub-ranges (<= 655,360 targets, each against every batch) so
// that positions + both accumulators of a sub-range stay L2-resident between
// launches (DRAM per launch 2.9 MB -> 45 KB at cfg 5).
// Self-sphere exclusion (reading R8): per-pair select, only in CTAs whose
// target spheres overlap the batch's source range.
#pragma once
#include "k_nbody.cuh"

namespace bie {

constexpr int kCB = 312;  // records per constant batch: 2 x 312 x (96 + 8) B = 64,896 B

__constant__ double2 c_nb_rec[2][kCB * 6];
__constant__ double c_nb_qn[2][kCB];

struct NbodyCArgs {
  const double* tx;  // [M][3] targets
  double* acc;       // [M][3] accumulator (in/out)
  double* pacc;      // [M] pressure accumulator (OFF; may be nullptr)
  int64_t M;
  int64_t k0;        // global index of the batch's first source (masking)
  int64_t tbase;     // global node index of target 0 of this launch (masking; apply only)
  int ks;            // sources in the batch (<= kCB)
  int nsn;           // nodes per sphere (masking; apply only)
};

template <int R, int TPB, int UNR, int BUF, bool OFF>
__global__ void __launch_bounds__(TPB, 1) k_nbody_c(const NbodyCArgs A) {
  double xt[R][3], acc[R][3], pacc[R];
  const int64_t tb = (int64_t)blockIdx.x * (TPB * R);
  const int64_t t0 = tb + threadIdx.x;
  const bool wp = OFF && A.pacc != nullptr;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t t = t0 + r * TPB < A.M ? t0 + r * TPB : A.M - 1;  // ragged tail: clamped, not stored
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xt[r][c] = A.tx[t * 3 + c];
      acc[r][c] = A.acc[t * 3 + c];
    }
    pacc[r] = wp ? A.pacc[t] : 0.0;
  }
  const double2* cs = c_nb_rec[BUF];
  const double* cq = c_nb_qn[BUF];
  const int ks = A.ks;
  bool masked = false;
  if (!OFF) {  // does the batch [k0, k0 + ks) meet the spheres of this CTA's targets?
    const int64_t te = (tb + TPB * R < A.M ? tb + TPB * R : A.M) - 1;
    const int64_t span_lo = ((A.tbase + tb) / A.nsn) * A.nsn, span_hi = ((A.tbase + te) / A.nsn + 1) * A.nsn;
    masked = A.k0 < span_hi && A.k0 + ks > span_lo;
  }
  if (!masked) {
#pragma unroll UNR
    for (int s = 0; s < ks; ++s) {
      const double2* sr = cs + s * 6;
      const double2 s0 = sr[0], s1 = sr[1], s2 = sr[2], s3 = sr[3], s4 = sr[4], s5 = sr[5];
      const double qn = OFF ? cq[s] : 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) pair_acc<false, OFF>(s0, s1, s2, s3, s4, s5, qn, xt[r], acc[r], pacc[r], 0, 0, 0);
    }
  } else {
    int lo[R];  // first node of each target's sphere, relative to the batch start
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t t = t0 + r * TPB < A.M ? t0 + r * TPB : A.M - 1;
      lo[r] = (int)(((A.tbase + t) / A.nsn) * A.nsn - A.k0);
    }
#pragma unroll 1
    for (int s = 0; s < ks; ++s) {
      const double2* sr = cs + s * 6;
      const double2 s0 = sr[0], s1 = sr[1], s2 = sr[2], s3 = sr[3], s4 = sr[4], s5 = sr[5];
#pragma unroll
      for (int r = 0; r < R; ++r)
        pair_acc<true, OFF>(s0, s1, s2, s3, s4, s5, 0.0, xt[r], acc[r], pacc[r], s, lo[r], A.nsn);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t t = t0 + r * TPB;
    if (t < A.M) {
#pragma unroll
      for (int c = 0; c < 3; ++c) A.acc[t * 3 + c] = acc[r][c];
      if (wp) A.pacc[t] = pacc[r];
    }
  }
}

// u += b (3M values); p = pscale (p + pb) (M values, when p != nullptr)
__global__ void k_nbody_c_join(int64_t M, double* __restrict__ u, const double* __restrict__ b, double* __restrict__ p,
                               const double* __restrict__ pb, double pscale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 3 * M) u[i] += b[i];
  if (p && i < M) p[i] = pscale * (p[i] + pb[i]);
}

}  // namespace bie
