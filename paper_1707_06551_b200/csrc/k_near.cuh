// k_near.cuh -- near-singular correction.
//
// PAPER §4.1 "Singular and near-singular integrands" and §4.3
// (P:436): for sphere pairs that are not well separated (eq 4.5)
//     dist(G_s, G_t) < eta max(diam G_s, diam G_t),
// the smooth-rule contribution of source sphere s at the nodes of target
// sphere t is replaced by the exact exterior field of s's degree-<=p vector
// spherical harmonic expansion (eqs 3.6-3.11 with sign reading R1, written as
// eq 4.7: coefficients kappa(x) = F(x) sigma^ with F depending on r only):
//     u_t += sum_{s near t} [ exterior_s(x) - smooth_s(x) ].
// The expansion coefficients come from k_self (phase C, written to `alpha`);
// the correction runs after the far-field sum, one CTA per target sphere,
// looping over its near neighbours in ascending index (deterministic).
#pragma once
#include <climits>
#include "common.cuh"
#include "k_nbody.cuh"
#include "k_setup.cuh"
#include "k_traction.cuh"

namespace bie {

struct NearArgs {
  int p, nsn;
  const double* tab;
  const double* centres;
  const double* radii;
  const double* rec;     // packed sources (x, n, f', q') of all nodes
  const double* coef;    // [ns][nlm][10] from k_near_coef
  const int* tgt;        // target spheres with >= 1 near neighbour
  const int* nb_off;     // [ns+1]
  const int* nb_idx;     // neighbour sphere indices
  double* u;             // [N][3], accumulated
};

__host__ __device__ inline int64_t near_smem_doubles(int p, bool stage) {
  const int nlm = (p + 1) * (p + 2) / 2, nsn = (p + 1) * (2 * p + 2);
  return 3LL * nsn + ((3LL * nlm + 1) & ~1LL) + (stage ? 12LL * nsn + 10LL * nlm : 0);
}

// stage the source sphere's records and coefficients in shared memory when they fit
__host__ __device__ inline bool near_stage(int p) { return near_smem_doubles(p, true) * 8 <= 160 * 1024; }

// PART 2 with staging: neighbours per batch -- as many coefficient blocks as
// the record region holds, capped so that their per-node results
// [batch][nsn][3] keep the CTA within 110 KB (two CTAs per SM, the register
// limit) where the rest allows it, else one neighbour per batch
__host__ __device__ inline int near2_batch(int p) {
  const int nlm = (p + 1) * (p + 2) / 2, nsn = (p + 1) * (2 * p + 2);
  const int b = (12 * nsn + 10 * nlm) / (10 * nlm);
  const int64_t room = (110LL * 1024 / 8 - near_smem_doubles(p, true)) / (3LL * nsn);
  return (int)(room < 1 ? 1 : (room < b ? room : b));
}
__host__ __device__ inline int64_t near2_smem_doubles(int p) {
  const int nsn = (p + 1) * (2 * p + 2);
  return near_smem_doubles(p, true) + 3LL * nsn * near2_batch(p);
}
__host__ __device__ inline bool near2_stage(int p) {
  return near_stage(p) && near2_smem_doubles(p) * 8 <= 227 * 1024;
}

template <bool PRESSURE>
__device__ __forceinline__ void exterior_field(int p, const double* __restrict__ cf,
                                               const double* rA, const double* rB,
                                               const double* rC, const double* c, double a,
                                               const double* x, double ex[3], double* pex);

// One CTA per target sphere t with near neighbours; for each neighbour s (in
// ascending index) every thread adds exterior_s(x) - smooth_s(x) at its nodes.
// STAGE: s's packed records and expansion coefficients are copied to shared
// memory first (broadcast reads in the O(n_s^2) smooth-rule subtraction).
// K = false: velocity of S + D (NEXT-1); K = true: traction of S with the
// target normal (NEXT-3, exterior_traction and the K pair kernel).
// PART (velocity, K = false): 0 exterior - smooth (NEXT-1); 1 smooth only
// (NEXT-4 mode: the exterior part arrives in coefficient space, k_n4); 2
// exterior only (measurement of the direct evaluation's cost; not an operator).
template <bool STAGE, bool K, int PART = 0>
__global__ void __launch_bounds__(128) k_near(const NearArgs A) {
  extern __shared__ __align__(16) double sm[];
  const int p = A.p, nsn = A.nsn;
  const TableLayout L(p);
  const int nlm = L.nlm;
  double* du = sm;              // [nsn][3]
  double* rt = du + 3 * nsn;    // rA, rB, rC [3][nlm]
  double* srec = rt + ((3 * nlm + 1) & ~1);  // STAGE: [nsn][12] (16-byte aligned)
  double* scf = srec + 12 * nsn;  // STAGE: [nlm][10]
  const int tid = threadIdx.x, nt = blockDim.x;
  const int t = A.tgt[blockIdx.x];
  for (int e = tid; e < 3 * nlm; e += nt) rt[e] = A.tab[L.rA + e];
  for (int e = tid; e < 3 * nsn; e += nt) du[e] = 0.0;
  if constexpr (PART == 2 && STAGE) {
    // Exterior part alone: only the neighbours' coefficients are read, so the
    // record region holds a batch of them -- two barriers per batch of B
    // neighbours instead of per neighbour (ncu r30: k_near<1,1,2> stalled on
    // barriers, 46 % FP64 pipe).  Same per-node accumulation order.
    const int B = near2_batch(p);
    double* res = scf + 10 * nlm;  // [B][nsn][3] per-neighbour results of the batch
    const int q0 = A.nb_off[t], q1 = A.nb_off[t + 1];
    for (int qb = q0; qb < q1; qb += B) {
      const int nb = min(B, q1 - qb);
      __syncthreads();  // previous batch no longer in use (and du / rt ready)
      for (int j = 0; j < nb; ++j) {
        const double2* c2 = reinterpret_cast<const double2*>(A.coef + (int64_t)A.nb_idx[qb + j] * nlm * 10);
        double2* d2 = reinterpret_cast<double2*>(srec + j * 10 * nlm);
        for (int e = tid; e < 5 * nlm; e += nt) d2[e] = c2[e];
      }
      __syncthreads();
      // (neighbour, node) items spread over the CTA -- nsn alone leaves lanes
      // idle (cfg 3: 162 nodes on 128 threads, 63 % of the thread slots) --
      // consecutive lanes on consecutive nodes of the same neighbour
      for (int item = tid; item < nb * nsn; item += nt) {
        const int j = item / nsn, kk = item - j * nsn;
        const int64_t i = (int64_t)t * nsn + kk;
        const double* ri = A.rec + i * kRec;
        const double xt[3] = {ri[0], ri[1], ri[2]};
        double nx[3] = {0.0, 0.0, 0.0};
        if constexpr (K) {
          nx[0] = ri[3];
          nx[1] = ri[4];
          nx[2] = ri[5];
        }
        const int s = A.nb_idx[qb + j];
        const double cs[3] = {A.centres[3 * s], A.centres[3 * s + 1], A.centres[3 * s + 2]};
        const double a = A.radii[s];
        const double* cfj = srec + j * 10 * nlm;
        double ex[3];
        if constexpr (K) exterior_traction(p, cfj, rt, rt + nlm, cs, a, xt, nx, ex);
        else exterior_field<false>(p, cfj, rt, rt + nlm, rt + 2 * nlm, cs, a, xt, ex, nullptr);
        double* r3 = res + 3 * item;
        r3[0] = ex[0];
        r3[1] = ex[1];
        r3[2] = ex[2];
      }
      __syncthreads();
      // per node, the batch's neighbours in ascending order (deterministic)
      for (int kk = tid; kk < nsn; kk += nt) {
        double d0 = du[3 * kk], d1 = du[3 * kk + 1], d2 = du[3 * kk + 2];
        for (int j = 0; j < nb; ++j) {
          const double* r3 = res + 3 * (j * nsn + kk);
          d0 += r3[0];
          d1 += r3[1];
          d2 += r3[2];
        }
        du[3 * kk] = d0;
        du[3 * kk + 1] = d1;
        du[3 * kk + 2] = d2;
      }
    }
    __syncthreads();
    for (int e = tid; e < 3 * nsn; e += nt) A.u[(int64_t)t * 3 * nsn + e] += du[e];
    return;
  } else {  // the general path (not compiled where the branch above returns)
    for (int qn = A.nb_off[t]; qn < A.nb_off[t + 1]; ++qn) {
      const int s = A.nb_idx[qn];
      const double cs[3] = {A.centres[3 * s], A.centres[3 * s + 1], A.centres[3 * s + 2]};
      const double a = A.radii[s];
      const double* cf = A.coef + (int64_t)s * nlm * 10;
      const double* rec_s = A.rec + (int64_t)s * nsn * kRec;
      if (STAGE) {
        __syncthreads();  // previous neighbour's staged data no longer in use
        if (PART != 2) {  // (the exterior part alone needs only the coefficients)
          const double2* g2 = reinterpret_cast<const double2*>(rec_s);
          double2* s2 = reinterpret_cast<double2*>(srec);
          for (int e = tid; e < 6 * nsn; e += nt) s2[e] = g2[e];
          rec_s = srec;
        }
        const double2* c2 = reinterpret_cast<const double2*>(cf);
        double2* d2 = reinterpret_cast<double2*>(scf);
        for (int e = tid; e < 5 * nlm; e += nt) d2[e] = c2[e];
        __syncthreads();
        cf = scf;
      } else if (qn == A.nb_off[t]) {
        __syncthreads();
      }
      const double2* sr = reinterpret_cast<const double2*>(rec_s);
      for (int kk = tid; kk < nsn; kk += nt) {
        const int64_t i = (int64_t)t * nsn + kk;
        const double* ri = A.rec + i * kRec;
        const double xt[3] = {ri[0], ri[1], ri[2]};
        double ex[3], acc[3] = {0.0, 0.0, 0.0};
        if constexpr (K) {
          const double nx[3] = {ri[3], ri[4], ri[5]};
          exterior_traction(p, cf, rt, rt + nlm, cs, a, xt, nx, ex);
          if (PART != 2)
            for (int k = 0; k < nsn; ++k) {
              const double2* q2 = sr + k * (kRec / 2);
              pair_K<false>(q2[0], q2[1], q2[4], q2[5], xt, nx, acc, 0, 0, 1);
            }
        } else {
          ex[0] = ex[1] = ex[2] = 0.0;
          if (PART != 1) exterior_field<false>(p, cf, rt, rt + nlm, rt + 2 * nlm, cs, a, xt, ex, nullptr);
          double pdummy = 0.0;
          if (PART != 2)
            for (int k = 0; k < nsn; ++k) {
              const double2* q2 = sr + k * (kRec / 2);
              pair_acc<false, false>(q2[0], q2[1], q2[2], q2[3], q2[4], q2[5], 0.0, xt, acc, pdummy, 0, 0, 1);
            }
        }
        du[3 * kk + 0] += ex[0] - acc[0];
        du[3 * kk + 1] += ex[1] - acc[1];
        du[3 * kk + 2] += ex[2] - acc[2];
      }
    }
    __syncthreads();
    for (int e = tid; e < 3 * nsn; e += nt) A.u[(int64_t)t * 3 * nsn + e] += du[e];
  }
}

}  // namespace bie

namespace bie {

// ------------------------------------------- per-sphere expansion coefficients
// coef[s][c][0..9]: c1, c2, c3, c4 (velocity, as in k_near) and cp (pressure)
// for sphere s and (n, m) column c, complex (re, im):
//   beta_V = c1 r^{-n-2} + c2 r^{-n}, beta_W = c3 r^{-n}, beta_X = c4 r^{-n-1},
//   p = sum cp Y_n^m r^{-n-1},  cp = (mu/a) [n aW_f + 2n(n-1) aW_q]
// (P:189 and reading R12 for the exterior pressures; R5/R6 scalings).
__global__ void k_near_coef(int p, int64_t ns, double mu, const double* __restrict__ radii,
                            const double* __restrict__ alpha, double* __restrict__ coef) {
  const TableLayout L(p);
  const int nlm = L.nlm;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ns * nlm) return;
  const int64_t s = e / nlm;
  const int c = (int)(e - s * nlm);
  int m = 0, off = 0;
  while (off + (p + 1 - m) <= c) { off += p + 1 - m; ++m; }
  const int n = m + (c - off);
  const double* af = alpha + ((int64_t)s * 2 * nlm + c) * 6;
  const double* aq = alpha + ((int64_t)s * 2 * nlm + nlm + c) * 6;
  const double inn = n ? 1.0 / ((double)n * (n + 1)) : 0.0;
  const double i2n = 1.0 / (2.0 * n + 1.0);
  const double lSV = n / ((2.0 * n + 1.0) * (2.0 * n + 3.0));
  const double lDV = (2.0 * n * n + 4.0 * n + 3.0) / ((2.0 * n + 1.0) * (2.0 * n + 3.0));
  const double xS = n / (4.0 * n + 2.0), xD = 2.0 * n * (n - 1.0) / (4.0 * n + 2.0);
  const double wS = n ? (n + 1.0) / ((2.0 * n + 1.0) * (2.0 * n - 1.0)) : 0.0;
  const double wD = n ? 2.0 * (n + 1.0) * (n - 1.0) / ((2.0 * n + 1.0) * (2.0 * n - 1.0)) : 0.0;
  const double kS = n ? 1.0 / (2.0 * n + 1.0) : 0.0, kD = n ? (n - 1.0) / (2.0 * n + 1.0) : 0.0;
  const double pm = mu / radii[s];
  double* o = coef + e * 10;
#pragma unroll
  for (int ri = 0; ri < 2; ++ri) {
    const double fV = (n * af[2 + ri] * inn - af[ri]) * i2n;
    const double fW = n ? ((n + 1) * af[2 + ri] * inn + af[ri]) * i2n : 0.0;
    const double fX = af[4 + ri] * inn;
    const double qV = (n * aq[2 + ri] * inn - aq[ri]) * i2n;
    const double qW = n ? ((n + 1) * aq[2 + ri] * inn + aq[ri]) * i2n : 0.0;
    const double qX = aq[4 + ri] * inn;
    o[0 + ri] = fV * lSV + fW * xS + qV * lDV + qW * xD;
    o[2 + ri] = -(fW * xS + qW * xD);
    o[4 + ri] = fW * wS + qW * wD;
    o[6 + ri] = fX * kS + qX * kD;
    o[8 + ri] = pm * (n * fW + 2.0 * n * (n - 1.0) * qW);
  }
}

// Exterior velocity (and pressure) of sphere (c, a) with coefficient block cf
// at point x: the expansion of eq 4.7 with eqs 3.6-3.11 (same algebra as k_near).
template <bool PRESSURE>
__device__ __forceinline__ void exterior_field(int p, const double* __restrict__ cf,
                                               const double* rA, const double* rB,
                                               const double* rC, const double* c, double a,
                                               const double* x, double ex[3], double* pex) {
  const double r0 = (x[0] - c[0]) / a, r1 = (x[1] - c[1]) / a, r2v = (x[2] - c[2]) / a;
  const double rxy = sqrt(r0 * r0 + r1 * r1);
  const double r = sqrt(rxy * rxy + r2v * r2v);
  const double rho = 1.0 / r;
  const double ct = r2v * rho, st = rxy * rho;
  const double cp = rxy > 0.0 ? r0 / rxy : 1.0, sp = rxy > 0.0 ? r1 / rxy : 0.0;
  const double inv_sqrt4pi = 0.28209479177387814347;
  double ur = 0.0, uth = 0.0, uph = 0.0, pr = 0.0;
  double e_re = 1.0, e_im = 0.0, rho_m = 1.0, pbar_mm = 0.0;
  for (int m = 0; m <= p; ++m) {
    double Ur0 = 0, Ur1 = 0, Ut0 = 0, Ut1 = 0, Up0 = 0, Up1 = 0, Pp0 = 0, Pp1 = 0;
    double Pp = 0.0, Pc, dPp = 0.0, dPc = 0.0;
    if (m == 0) {
      Pc = inv_sqrt4pi;
    } else {
      pbar_mm = (m == 1) ? inv_sqrt4pi * sqrt(1.5) : pbar_mm * st * sqrt((2.0 * m + 1.0) / (2.0 * m));
      Pc = pbar_mm;
    }
    double rn = rho_m;
    const int c0 = lm_index(p, m, m);
    for (int n = m; n <= p; ++n) {
      const int cc = c0 + (n - m);
      if (n > m) {
        const double nx = rA[cc] * (ct * Pc - rB[cc] * Pp);
        if (m == 0) {
          const double dnx = rA[cc] * (ct * dPc - st * Pc - rB[cc] * dPp);
          dPp = dPc;
          dPc = dnx;
        }
        Pp = Pc;
        Pc = nx;
      }
      double Pt, dPt, mPs;
      if (m == 0) {
        Pt = Pc;
        dPt = dPc;
        mPs = 0.0;
      } else {
        Pt = st * Pc;
        mPs = m * Pc;
        dPt = n * ct * Pc - rC[cc] * (n > m ? Pp : 0.0);
      }
      const double* o = cf + 10 * cc;
      const double bV0 = rn * fma(o[0], rho * rho, o[2]), bV1 = rn * fma(o[1], rho * rho, o[3]);
      const double bW0 = rn * o[4], bW1 = rn * o[5];
      const double bX0 = rn * rho * o[6], bX1 = rn * rho * o[7];
      const double gG0 = bV0 + bW0, gG1 = bV1 + bW1;
      const double gY0 = -(n + 1.0) * bV0 + n * bW0, gY1 = -(n + 1.0) * bV1 + n * bW1;
      Ur0 = fma(gY0, Pt, Ur0);
      Ur1 = fma(gY1, Pt, Ur1);
      Ut0 = fma(gG0, dPt, fma(bX1, mPs, Ut0));
      Ut1 = fma(gG1, dPt, fma(-bX0, mPs, Ut1));
      Up0 = fma(bX0, dPt, fma(-gG1, mPs, Up0));
      Up1 = fma(bX1, dPt, fma(gG0, mPs, Up1));
      if (PRESSURE) {
        Pp0 = fma(o[8] * rn * rho, Pt, Pp0);
        Pp1 = fma(o[9] * rn * rho, Pt, Pp1);
      }
      rn *= rho;
    }
    const double wm = m ? 2.0 : 1.0;
    ur += wm * (Ur0 * e_re - Ur1 * e_im);
    uth += wm * (Ut0 * e_re - Ut1 * e_im);
    uph += wm * (Up0 * e_re - Up1 * e_im);
    if (PRESSURE) pr += wm * (Pp0 * e_re - Pp1 * e_im);
    const double ne = e_re * cp - e_im * sp;
    e_im = e_re * sp + e_im * cp;
    e_re = ne;
    rho_m *= rho;
  }
  ex[0] = ur * st * cp + uth * ct * cp - uph * sp;
  ex[1] = ur * st * sp + uth * ct * sp + uph * cp;
  ex[2] = ur * ct - uth * st;
  if (PRESSURE) *pex = pr;
}

// ------------------------------------------- near correction at arbitrary targets
// One thread per target.  Near spheres (point-to-surface form of eq 4.5:
// |x - c_s| - a_s < eta 2 a_s) are found by scanning the sphere list through
// shared-memory tiles in ascending index, up to kNearList at a time, then each
// is evaluated (exterior expansion minus smooth rule) -- all lanes run the same
// code on different spheres, so the warp stays convergent.  u[t] += du,
// p[t] += dp after the smooth-sum kernels (deterministic).
constexpr int kNearList = 16;
constexpr int kSphTile = 256;

struct NearOffArgs {
  int p, nsn;
  int64_t ns, M;
  double mu, eta;
  const double* tab;
  const double* centres;
  const double* radii;
  const double* rec;
  const double* qn3;
  const double* coef;  // [ns][nlm][10]
  const double* tx;    // [M][3]
  double* u;           // [M][3] accumulated
  double* pres;        // [M] accumulated, nullable
  const double* tn = nullptr;  // [M][3] target normals (traction, K = true)
  const int* order = nullptr;  // [M] processing order (Morton-sorted target indices), or identity
  // uniform cell grid of the sphere centres (built by bie_set_near): a target
  // x and sphere s are near only if |x - c_s| < a_s (1 + 2 eta) <= h, so
  // every near sphere lies in the 27 cells around x's cell
  const int* cell_start = nullptr;  // [ncell + 1]
  const int* cell_items = nullptr;  // [ns] sphere indices, ascending within a cell
  double g0x = 0, g0y = 0, g0z = 0, gh = 1;  // grid origin and cell size
  int gnx = 1, gny = 1, gnz = 1;
};

__host__ __device__ inline int64_t near_off_smem_doubles(int p) {
  const int nlm = (p + 1) * (p + 2) / 2;
  return 3LL * nlm;
}

// 30-bit Morton key of a point's cell (10 bits per axis, clamped to the grid)
__device__ __forceinline__ uint32_t morton_spread(uint32_t v) {
  v &= 0x3FF;
  v = (v | (v << 16)) & 0x030000FF;
  v = (v | (v << 8)) & 0x0300F00F;
  v = (v | (v << 4)) & 0x030C30C3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}
__global__ void k_morton(int64_t M, const double* __restrict__ tx, double g0x, double g0y, double g0z,
                         double h, uint32_t* __restrict__ key, int* __restrict__ idx) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= M) return;
  auto q = [&](double v, double o) {
    const double c = floor((v - o) / h);
    return (uint32_t)(c < 0 ? 0 : (c > 1023 ? 1023 : c));
  };
  key[t] = morton_spread(q(tx[3 * t], g0x)) | (morton_spread(q(tx[3 * t + 1], g0y)) << 1) |
           (morton_spread(q(tx[3 * t + 2], g0z)) << 2);
  idx[t] = (int)t;
}

// K = true: traction with the target normals A.tn (bie_eval_traction, NEXT-3).
template <bool PRESSURE, bool K>
__global__ void __launch_bounds__(128) k_near_off(const NearOffArgs A) {
  extern __shared__ __align__(16) double sm[];
  const int p = A.p, nsn = A.nsn;
  const TableLayout L(p);
  const int nlm = L.nlm;
  double* rt = sm;                // rA, rB, rC
  for (int e = threadIdx.x; e < 3 * nlm; e += blockDim.x) rt[e] = A.tab[L.rA + e];
  __syncthreads();
  const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = it < A.M;
  const int64_t t = live ? (A.order ? (int64_t)A.order[it] : it) : A.M - 1;
  const int64_t tc = t;
  const double x[3] = {A.tx[3 * tc], A.tx[3 * tc + 1], A.tx[3 * tc + 2]};
  double nv[3] = {0.0, 0.0, 0.0};
  if constexpr (K) {
    nv[0] = A.tn[3 * tc];
    nv[1] = A.tn[3 * tc + 1];
    nv[2] = A.tn[3 * tc + 2];
  }
  double du[3] = {0.0, 0.0, 0.0}, dp = 0.0;
  int list[kNearList];
  int cnt = 0;
  auto eval = [&](int s) {
    const double cs[3] = {A.centres[3 * s], A.centres[3 * s + 1], A.centres[3 * s + 2]};
    const double* cf = A.coef + (int64_t)s * nlm * 10;
    const double2* sr = reinterpret_cast<const double2*>(A.rec + (int64_t)s * nsn * kRec);
    double ex[3], pe = 0.0, acc[3] = {0.0, 0.0, 0.0}, pacc = 0.0;
    if constexpr (K) {
      exterior_traction(p, cf, rt, rt + nlm, cs, A.radii[s], x, nv, ex);
      for (int k = 0; k < nsn; ++k) {
        const double2* q2 = sr + k * (kRec / 2);
        pair_K<false>(__ldg(q2), __ldg(q2 + 1), __ldg(q2 + 4), __ldg(q2 + 5), x, nv, acc, 0, 0, 1);
      }
    } else {
      exterior_field<PRESSURE>(p, cf, rt, rt + nlm, rt + 2 * nlm, cs, A.radii[s], x, ex, &pe);
      const double* sq = A.qn3 + (int64_t)s * nsn;
      for (int k = 0; k < nsn; ++k) {
        const double2* q2 = sr + k * (kRec / 2);
        pair_acc<false, PRESSURE>(__ldg(q2), __ldg(q2 + 1), __ldg(q2 + 2), __ldg(q2 + 3),
                                  __ldg(q2 + 4), __ldg(q2 + 5), PRESSURE ? __ldg(sq + k) : 0.0, x,
                                  acc, pacc, 0, 0, 1);
      }
    }
    du[0] += ex[0] - acc[0];
    du[1] += ex[1] - acc[1];
    du[2] += ex[2] - acc[2];
    if (PRESSURE) dp += pe - 2.0 * A.mu * pacc;
  };
  auto flush = [&]() {  // lane-local (a list overflow inside the scan)
    for (int j = 0; j < cnt; ++j) eval(list[j]);
    cnt = 0;
  };
  // candidates: the 27 cells around x's (clamped) cell; the exact test of eq 4.5
  // (point-to-surface form) in the oracle's evaluation order decides
  auto cell = [&](double v, double o, int n) {
    const double c = floor((v - o) / A.gh);
    return (int)(c < 0 ? 0 : (c > n - 1 ? n - 1 : c));
  };
  const int cx = cell(x[0], A.g0x, A.gnx), cy = cell(x[1], A.g0y, A.gny), cz = cell(x[2], A.g0z, A.gnz);
  for (int iz = max(cz - 1, 0); iz <= min(cz + 1, A.gnz - 1); ++iz)
    for (int iy = max(cy - 1, 0); iy <= min(cy + 1, A.gny - 1); ++iy)
      for (int ix = max(cx - 1, 0); ix <= min(cx + 1, A.gnx - 1); ++ix) {
        const int cid = (iz * A.gny + iy) * A.gnx + ix;
        for (int q = A.cell_start[cid]; q < A.cell_start[cid + 1]; ++q) {
          const int sidx = A.cell_items[q];
          const double dx = __dsub_rn(x[0], A.centres[3 * sidx]), dy = __dsub_rn(x[1], A.centres[3 * sidx + 1]),
                       dz = __dsub_rn(x[2], A.centres[3 * sidx + 2]);
          const double a = A.radii[sidx];
          const double r =
              __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
          const double dsurf = __dsub_rn(r, a);
          if (live && dsurf >= 0.0 && dsurf < __dmul_rn(A.eta, __dmul_rn(2.0, a))) {  // exterior only
            list[cnt++] = sidx;
            if (cnt == kNearList) flush();
          }
        }
      }
  // Final flush in ascending sphere order (the per-target accumulation order).
  // (A warp-cooperative variant -- the warp walking the union of its lanes'
  // lists so each sphere is read once per warp -- cut long-scoreboard stalls
  // 7.8 -> 2.8 per issue but idled the lanes not holding the current sphere:
  // 2.14 -> 3.33 ms on cfg 5, profiles/r02_ncu_nearoff_cfg5*.txt; reverted.)
  for (int i = 1; i < cnt; ++i) {
    const int v = list[i];
    int j = i - 1;
    while (j >= 0 && list[j] > v) { list[j + 1] = list[j]; --j; }
    list[j + 1] = v;
  }
  flush();
  if (!live) return;
  A.u[3 * t] += du[0];
  A.u[3 * t + 1] += du[1];
  A.u[3 * t + 2] += du[2];
  if (PRESSURE && A.pres) A.pres[t] += dp;
}

// ------------------------------------------- grouped schedule (default)
// The (target, near sphere) pairs of the off-surface correction grouped by
// sphere: one CTA takes up to kGrpChunk pairs of ONE sphere, whose records,
// qn3 and expansion coefficients are staged in shared memory once and read as
// broadcasts by every thread.  (The per-target schedule above makes each lane
// walk its own spheres' records through L1/L2: 33 % FP64 pipe, bound by long
// scoreboard stalls, profiles/r02_ncu_nearoff_cfg5.txt.)  Per-pair results go
// to a buffer; k_noff_sum adds them per target in ascending sphere order, so
// the result is deterministic and does not depend on the grouping.
constexpr int kGrpChunk = 128;

struct NearGrp {
  int* cnt;              // [M + 1] near spheres per target (count pass; cnt[M] = 0)
  const int* off;        // [M + 1] exclusive scan of cnt: pair range of each target
  int* pair_s;           // [P] sphere of pair j (target-major, ascending sphere in a target)
  int* pair_t;           // [P] target of pair j
  int* pair_j;           // [P] j (the values of the sphere sort)
  int* scount;           // [ns + 1] pairs per sphere (integer atomics: order-free)
  int* nch;              // [ns + 1] chunks per sphere
  const int* sorted_j;   // [P] pair indices grouped by sphere (stable: ascending target)
  const int* sfirst;     // [ns + 1] exclusive scan of scount
  const int* choff;      // [ns + 1] exclusive scan of nch
  double* res;           // [P][4] (du, dp) of each pair
};

// Near spheres of target x in the candidate order of k_near_off (27 cells).
template <typename F>
__device__ __forceinline__ void near_candidates(const NearOffArgs& A, const double* x, F&& take) {
  auto cell = [&](double v, double o, int n) {
    const double c = floor((v - o) / A.gh);
    return (int)(c < 0 ? 0 : (c > n - 1 ? n - 1 : c));
  };
  const int cx = cell(x[0], A.g0x, A.gnx), cy = cell(x[1], A.g0y, A.gny), cz = cell(x[2], A.g0z, A.gnz);
  for (int iz = max(cz - 1, 0); iz <= min(cz + 1, A.gnz - 1); ++iz)
    for (int iy = max(cy - 1, 0); iy <= min(cy + 1, A.gny - 1); ++iy)
      for (int ix = max(cx - 1, 0); ix <= min(cx + 1, A.gnx - 1); ++ix) {
        const int cid = (iz * A.gny + iy) * A.gnx + ix;
        for (int q = A.cell_start[cid]; q < A.cell_start[cid + 1]; ++q) {
          const int sidx = A.cell_items[q];
          const double dx = __dsub_rn(x[0], A.centres[3 * sidx]), dy = __dsub_rn(x[1], A.centres[3 * sidx + 1]),
                       dz = __dsub_rn(x[2], A.centres[3 * sidx + 2]);
          const double a = A.radii[sidx];
          const double r =
              __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
          const double dsurf = __dsub_rn(r, a);
          if (dsurf >= 0.0 && dsurf < __dmul_rn(A.eta, __dmul_rn(2.0, a))) take(sidx);  // exterior only
        }
      }
}

// WRITE = false: cnt[t] = number of near spheres of target t.  WRITE = true:
// the pairs of t at off[t].. in ascending sphere order, and the per-sphere counts.
template <bool WRITE>
__global__ void __launch_bounds__(128) k_noff_pairs(const NearOffArgs A, const NearGrp G) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= A.M) return;
  const double x[3] = {A.tx[3 * t], A.tx[3 * t + 1], A.tx[3 * t + 2]};
  const int base = WRITE ? G.off[t] : 0;
  int r = 0;
  near_candidates(A, x, [&](int sidx) {
    if (WRITE) G.pair_s[base + r] = sidx;
    ++r;
  });
  if (!WRITE) {
    G.cnt[t] = r;
    return;
  }
  int* ps = G.pair_s + base;
  for (int i = 1; i < r; ++i) {  // a handful of spheres: insertion sort
    const int v = ps[i];
    int j = i - 1;
    while (j >= 0 && ps[j] > v) { ps[j + 1] = ps[j]; --j; }
    ps[j + 1] = v;
  }
  for (int i = 0; i < r; ++i) {
    G.pair_t[base + i] = (int)t;
    G.pair_j[base + i] = base + i;
    atomicAdd(&G.scount[ps[i]], 1);
  }
}

__global__ void k_noff_nch(int64_t ns, const int* __restrict__ scount, int* __restrict__ nch) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < ns) nch[s] = (scount[s] + kGrpChunk - 1) / kGrpChunk;
}

__host__ __device__ inline int64_t noff_grp_smem_doubles(int p, bool stage) {
  const int nlm = (p + 1) * (p + 2) / 2, nsn = (p + 1) * (2 * p + 2);
  const int64_t head = (3LL * nlm + 10LL * nlm + 1) & ~1LL;  // rA rB rC, coefficients
  return head + (stage ? 12LL * nsn + nsn : 0);
}
__host__ __device__ inline bool noff_grp_stage(int p) { return noff_grp_smem_doubles(p, true) * 8 <= 100 * 1024; }

// One CTA per (sphere, chunk of <= kGrpChunk of its pairs); thread i takes one
// pair.  STAGE: the sphere's packed records and qn3 in shared memory (else
// read with warp-uniform addresses, which L1 serves as broadcasts).
template <bool PRESSURE, bool K, bool STAGE>
__global__ void __launch_bounds__(kGrpChunk) k_noff_grp(const NearOffArgs A, const NearGrp G) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const int ns = (int)A.ns;
  if (b >= G.choff[ns]) return;
  int lo = 0, hi = ns;  // largest s with choff[s] <= b
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (G.choff[mid] <= b) lo = mid;
    else hi = mid;
  }
  const int s = lo;
  const int i0 = G.sfirst[s] + (b - G.choff[s]) * kGrpChunk;
  const int i1 = min(i0 + kGrpChunk, G.sfirst[s + 1]);
  const int p = A.p, nsn = A.nsn;
  const TableLayout L(p);
  const int nlm = L.nlm;
  double* rt = sm;              // rA, rB, rC [3][nlm]
  double* cf = rt + 3 * nlm;    // [nlm][10]
  double* srec = sm + ((13 * nlm + 1) & ~1);  // STAGE: [nsn][12], then qn3 [nsn]
  const int tid = threadIdx.x;
  for (int e = tid; e < 3 * nlm; e += kGrpChunk) rt[e] = A.tab[L.rA + e];
  const double* gcf = A.coef + (int64_t)s * nlm * 10;
  for (int e = tid; e < 10 * nlm; e += kGrpChunk) cf[e] = gcf[e];
  const double2* sr = reinterpret_cast<const double2*>(A.rec + (int64_t)s * nsn * kRec);
  const double* sq = (PRESSURE && !K) ? A.qn3 + (int64_t)s * nsn : nullptr;
  if (STAGE) {
    double2* s2 = reinterpret_cast<double2*>(srec);
    for (int e = tid; e < 6 * nsn; e += kGrpChunk) s2[e] = sr[e];
    if (PRESSURE && !K)
      for (int e = tid; e < nsn; e += kGrpChunk) srec[12 * nsn + e] = sq[e];
    sr = s2;
    if (PRESSURE && !K) sq = srec + 12 * nsn;
  }
  __syncthreads();
  const int i = i0 + tid;
  if (i >= i1) return;
  const int j = G.sorted_j[i];
  const int t = G.pair_t[j];
  const double x[3] = {A.tx[3 * (int64_t)t], A.tx[3 * (int64_t)t + 1], A.tx[3 * (int64_t)t + 2]};
  const double cs[3] = {A.centres[3 * s], A.centres[3 * s + 1], A.centres[3 * s + 2]};
  const double a = A.radii[s];
  double ex[3], pe = 0.0, acc[3] = {0.0, 0.0, 0.0}, pacc = 0.0;
  if constexpr (K) {
    const double nv[3] = {A.tn[3 * (int64_t)t], A.tn[3 * (int64_t)t + 1], A.tn[3 * (int64_t)t + 2]};
    exterior_traction(p, cf, rt, rt + nlm, cs, a, x, nv, ex);
    for (int k = 0; k < nsn; ++k) {
      const double2* q2 = sr + k * (kRec / 2);
      pair_K<false>(q2[0], q2[1], q2[4], q2[5], x, nv, acc, 0, 0, 1);
    }
  } else {
    exterior_field<PRESSURE>(p, cf, rt, rt + nlm, rt + 2 * nlm, cs, a, x, ex, &pe);
    for (int k = 0; k < nsn; ++k) {
      const double2* q2 = sr + k * (kRec / 2);
      pair_acc<false, PRESSURE>(q2[0], q2[1], q2[2], q2[3], q2[4], q2[5], PRESSURE ? sq[k] : 0.0, x, acc,
                                pacc, 0, 0, 1);
    }
  }
  double4 o;
  o.x = ex[0] - acc[0];
  o.y = ex[1] - acc[1];
  o.z = ex[2] - acc[2];
  o.w = PRESSURE ? pe - 2.0 * A.mu * pacc : 0.0;
  reinterpret_cast<double4*>(G.res)[j] = o;
}

// u[t] += sum over t's pairs (ascending sphere) of du; p[t] likewise.
template <bool PRESSURE>
__global__ void k_noff_sum(const NearOffArgs A, const NearGrp G) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= A.M) return;
  const int j0 = G.off[t], j1 = G.off[t + 1];
  if (j0 == j1) return;
  const double4* r4 = reinterpret_cast<const double4*>(G.res);
  double du0 = 0.0, du1 = 0.0, du2 = 0.0, dp = 0.0;
  for (int j = j0; j < j1; ++j) {
    const double4 o = r4[j];
    du0 += o.x;
    du1 += o.y;
    du2 += o.z;
    dp += o.w;
  }
  A.u[3 * t] += du0;
  A.u[3 * t + 1] += du1;
  A.u[3 * t + 2] += du2;
  if (PRESSURE && A.pres) A.pres[t] += dp;
}

}  // namespace bie
