// k_self.cuh -- per-sphere spectral self term fused with source packing.
//
// One CTA per sphere (rows a2, a4, a5, a6 of SURVEY §8(a)):
//   A  load f, q of the sphere; write the packed far-field source records
//      (x, n, w f/(8 pi mu), (3/(4 pi)) w q); rotate (a/mu) f and q to
//      spherical components (e_r, e_theta, e_phi)
//   B  forward real DFT over the 2p+2 azimuthal nodes of every latitude
//      (the FFT stage of the paper's fast transform; a dense
//      26-point DFT at p = 12)
//   C  Legendre projection per (n, m) (eq 2.3 discretised, reading R9) onto
//      {Y e_r, G, X} (eq 2.12), conversion to {V, W, X} (eqs 2.13-2.14), and
//      the diagonal scale psi = lamS (a/mu) alpha[f] + lamD_pv alpha[q]
//      (Thm 2, readings R2/R3/R5/R6); back to {Y, G, X} (eqs 2.16-2.17)
//   D  inverse Legendre sum per (latitude, m)
//   E  inverse DFT, back to Cartesian, write u_self ("u may thus be
//      evaluated using a fast inverse transform")
// All intermediate spectra stay in shared memory; HBM sees f, q (48 B/node)
// in and u (24 B/node) + records (96 B/node) out.
#pragma once
#include "common.cuh"
#include "k_setup.cuh"

namespace bie {

struct SelfArgs {
  int p;
  int64_t ns;
  double mu;
  const double* tab;
  const double* centres;
  const double* radii;
  const double* f;  // nullable
  const double* q;  // nullable
  double* u;        // [N][3] out: self term (or 0 when !self)
  double* rec;      // [N][kRec] out: packed sources
  int self;         // compute the self term (else write zeros)
};

__host__ __device__ inline int64_t self_smem_doubles(int p) {
  const int P1 = p + 1, nphi = 2 * p + 2, nsn = P1 * nphi;
  const int64_t C = 6LL * nsn;                    // spherical components; reused as U
  const int64_t F = 12LL * P1 * P1;               // [2 dens][3 comp][j][m][re,im]
  const int64_t PSI = 6LL * (P1 * (P1 + 1) / 2);  // [(n,m)][Y,G,X][re,im]
  return C + F + PSI + 2LL * nphi;
}

__global__ void __launch_bounds__(256) k_self(SelfArgs A) {
  extern __shared__ __align__(16) double sm[];
  const int p = A.p, P1 = p + 1, nphi = 2 * p + 2, nsn = P1 * nphi;
  const TableLayout L(p);
  const int nlm = L.nlm;
  double* C = sm;                          // [2][3][nsn]
  double* F = C + 6 * nsn;                 // [2][3][P1][P1][2]
  double* PSI = F + 12 * P1 * P1;          // [nlm][3][2]
  double* cs = PSI + 6 * nlm;              // cos(2 pi k/nphi)
  double* sn = cs + nphi;                  // sin(2 pi k/nphi)
  double* U = C;                           // [3][P1][P1][2] (C is dead after B)
  const double* __restrict__ tab = A.tab;
  const int64_t s = blockIdx.x;
  const double a = A.radii[s];
  const double cx = A.centres[3 * s], cy = A.centres[3 * s + 1], cz = A.centres[3 * s + 2];
  const double aS = a / A.mu;
  const double cS = 1.0 / (8.0 * kPi * A.mu), cD = 3.0 / (4.0 * kPi);
  const int tid = threadIdx.x, nt = blockDim.x;

  for (int k = tid; k < nphi; k += nt) {
    cs[k] = tab[L.cph + k];
    sn[k] = tab[L.sph + k];
  }
  // ---------------------------------------------------------------- A
  for (int kk = tid; kk < nsn; kk += nt) {
    const int j = kk / nphi, k = kk - j * nphi;
    const int64_t i = s * nsn + kk;
    double f0 = 0, f1 = 0, f2 = 0, q0 = 0, q1 = 0, q2 = 0;
    if (A.f) { f0 = A.f[3 * i]; f1 = A.f[3 * i + 1]; f2 = A.f[3 * i + 2]; }
    if (A.q) { q0 = A.q[3 * i]; q1 = A.q[3 * i + 1]; q2 = A.q[3 * i + 2]; }
    const double ct = tab[L.t + j], st = tab[L.st + j];
    const double cp = tab[L.cph + k], sp = tab[L.sph + k];
    const double n0 = st * cp, n1 = st * sp, n2 = ct;
    const double w = a * a * tab[L.wu + j];
    // packed source record (row a2)
    double2* r2 = reinterpret_cast<double2*>(A.rec + i * kRec);
    const double ws = w * cS, wd = w * cD;
    r2[0] = make_double2(cx + a * n0, cy + a * n1);
    r2[1] = make_double2(cz + a * n2, n0);
    r2[2] = make_double2(n1, n2);
    r2[3] = make_double2(ws * f0, ws * f1);
    r2[4] = make_double2(ws * f2, wd * q0);
    r2[5] = make_double2(wd * q1, wd * q2);
    if (A.self) {
      // e_r = n, e_theta = (ct cp, ct sp, -st), e_phi = (-sp, cp, 0)
      C[0 * nsn + kk] = aS * (f0 * n0 + f1 * n1 + f2 * n2);
      C[1 * nsn + kk] = aS * (f0 * ct * cp + f1 * ct * sp - f2 * st);
      C[2 * nsn + kk] = aS * (-f0 * sp + f1 * cp);
      C[3 * nsn + kk] = q0 * n0 + q1 * n1 + q2 * n2;
      C[4 * nsn + kk] = q0 * ct * cp + q1 * ct * sp - q2 * st;
      C[5 * nsn + kk] = -q0 * sp + q1 * cp;
    }
  }
  if (!A.self) {
    for (int e = tid; e < 3 * nsn; e += nt) A.u[s * 3 * nsn + e] = 0.0;
    return;
  }
  __syncthreads();
  // ---------------------------------------------------------------- B
  // F[dc][j][m] = sum_k C[dc][j,k] e^{-i m phi_k}
  for (int it = tid; it < 6 * P1 * P1; it += nt) {
    const int m = it % P1, j = (it / P1) % P1, dc = it / (P1 * P1);
    const double* row = C + dc * nsn + j * nphi;
    double re = 0.0, im = 0.0;
    int idx = 0;
    for (int k = 0; k < nphi; ++k) {
      re = fma(row[k], cs[idx], re);
      im = fma(-row[k], sn[idx], im);
      idx += m;
      if (idx >= nphi) idx -= nphi;
    }
    F[2 * it] = re;
    F[2 * it + 1] = im;
  }
  __syncthreads();
  // ---------------------------------------------------------------- C
  for (int c = tid; c < nlm; c += nt) {
    int m = 0, off = 0;
    while (off + (P1 - m) <= c) { off += P1 - m; ++m; }
    const int n = m + (c - off);
    double acc[2][3][2];  // [dens][Y,<G>,<X>][re,im]
#pragma unroll
    for (int d = 0; d < 2; ++d)
#pragma unroll
      for (int z = 0; z < 3; ++z) acc[d][z][0] = acc[d][z][1] = 0.0;
    for (int j = 0; j < P1; ++j) {
      const double wj = tab[L.wu + j];
      const double Pv = wj * tab[L.P + (int64_t)j * nlm + c];
      const double dPv = wj * tab[L.dP + (int64_t)j * nlm + c];
      const double mPv = wj * tab[L.mPs + (int64_t)j * nlm + c];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const double* Fr = F + 2 * (((3 * d + 0) * P1 + j) * P1 + m);
        const double* Ft = F + 2 * (((3 * d + 1) * P1 + j) * P1 + m);
        const double* Fp = F + 2 * (((3 * d + 2) * P1 + j) * P1 + m);
        // <F, Y e_r>
        acc[d][0][0] = fma(Pv, Fr[0], acc[d][0][0]);
        acc[d][0][1] = fma(Pv, Fr[1], acc[d][0][1]);
        // <F, G> = dP F_t - i mP F_p
        acc[d][1][0] = fma(dPv, Ft[0], fma(mPv, Fp[1], acc[d][1][0]));
        acc[d][1][1] = fma(dPv, Ft[1], fma(-mPv, Fp[0], acc[d][1][1]));
        // <F, X> = dP F_p + i mP F_t
        acc[d][2][0] = fma(dPv, Fp[0], fma(-mPv, Ft[1], acc[d][2][0]));
        acc[d][2][1] = fma(dPv, Fp[1], fma(mPv, Ft[0], acc[d][2][1]));
      }
    }
    const double* lS = tab + L.lamS + 3 * n;
    const double* lD = tab + L.lamD + 3 * n;
    const double inn = n ? 1.0 / ((double)n * (n + 1)) : 0.0;
    const double i2n = 1.0 / (2.0 * n + 1.0);
    double psV[2], psW[2], psX[2];
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
      double aV[2], aW[2], aX[2];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const double phY = acc[d][0][ri], phG = acc[d][1][ri] * inn, phX = acc[d][2][ri] * inn;
        aV[d] = (n * phG - phY) * i2n;          // eq 2.13
        aW[d] = ((n + 1) * phG + phY) * i2n;    // eq 2.14
        aX[d] = phX;
      }
      psV[ri] = lS[0] * aV[0] + lD[0] * aV[1];
      psW[ri] = lS[1] * aW[0] + lD[1] * aW[1];
      psX[ri] = lS[2] * aX[0] + lD[2] * aX[1];
    }
    double* o = PSI + 6 * c;
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
      o[0 + ri] = -(n + 1.0) * psV[ri] + n * psW[ri];  // psi^Y (eq 2.17)
      o[2 + ri] = psV[ri] + psW[ri];                   // psi^G (eq 2.16)
      o[4 + ri] = psX[ri];                             // psi^X
    }
  }
  __syncthreads();
  // ---------------------------------------------------------------- D
  // U_r = sum_n psiY P, U_t = sum_n psiG dP - i psiX mP, U_p = sum_n i psiG mP + psiX dP
  for (int it = tid; it < P1 * P1; it += nt) {
    const int j = it / P1, m = it % P1;
    double ur0 = 0, ur1 = 0, ut0 = 0, ut1 = 0, up0 = 0, up1 = 0;
    const int c0 = lm_index(p, m, m);
    for (int n = m; n <= p; ++n) {
      const int c = c0 + (n - m);
      const double Pv = tab[L.P + (int64_t)j * nlm + c];
      const double dPv = tab[L.dP + (int64_t)j * nlm + c];
      const double mPv = tab[L.mPs + (int64_t)j * nlm + c];
      const double* ps = PSI + 6 * c;
      ur0 = fma(ps[0], Pv, ur0);
      ur1 = fma(ps[1], Pv, ur1);
      ut0 = fma(ps[2], dPv, fma(ps[5], mPv, ut0));
      ut1 = fma(ps[3], dPv, fma(-ps[4], mPv, ut1));
      up0 = fma(ps[4], dPv, fma(-ps[3], mPv, up0));
      up1 = fma(ps[5], dPv, fma(ps[2], mPv, up1));
    }
    U[2 * ((0 * P1 + j) * P1 + m)] = ur0;
    U[2 * ((0 * P1 + j) * P1 + m) + 1] = ur1;
    U[2 * ((1 * P1 + j) * P1 + m)] = ut0;
    U[2 * ((1 * P1 + j) * P1 + m) + 1] = ut1;
    U[2 * ((2 * P1 + j) * P1 + m)] = up0;
    U[2 * ((2 * P1 + j) * P1 + m) + 1] = up1;
  }
  __syncthreads();
  // ---------------------------------------------------------------- E
  for (int kk = tid; kk < nsn; kk += nt) {
    const int j = kk / nphi, k = kk - j * nphi;
    double v[3];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      const double* Uc = U + 2 * ((comp * P1 + j) * P1);
      double acc = 0.0;
      int idx = k;
      for (int m = 1; m <= p; ++m) {
        acc = fma(Uc[2 * m], cs[idx], fma(-Uc[2 * m + 1], sn[idx], acc));
        idx += k;
        if (idx >= nphi) idx -= nphi;
      }
      v[comp] = fma(2.0, acc, Uc[0]);
    }
    const double ct = tab[L.t + j], st = tab[L.st + j];
    const double cp = cs[k], sp = sn[k];
    const int64_t i = s * nsn + kk;
    A.u[3 * i + 0] = v[0] * st * cp + v[1] * ct * cp - v[2] * sp;
    A.u[3 * i + 1] = v[0] * st * sp + v[1] * ct * sp + v[2] * cp;
    A.u[3 * i + 2] = v[0] * ct - v[1] * st;
  }
}

// Source packing alone (row a2) for the off-surface evaluator; also writes
// qn3_k = (q'_k . n_k)/3 for the double-layer pressure.
__global__ void k_pack(int p, int64_t N, double mu, const double* __restrict__ tab,
                       const double* __restrict__ centres, const double* __restrict__ radii,
                       const double* __restrict__ f, const double* __restrict__ q,
                       double* __restrict__ rec, double* __restrict__ qn3) {
  const TableLayout L(p);
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int nsn = (p + 1) * L.nphi;
  const int64_t s = i / nsn;
  const int kk = (int)(i - s * nsn);
  const int j = kk / L.nphi, k = kk - j * L.nphi;
  const double st = tab[L.st + j];
  const double n0 = st * tab[L.cph + k], n1 = st * tab[L.sph + k], n2 = tab[L.t + j];
  const double a = radii[s];
  const double w = a * a * tab[L.wu + j];
  const double ws = w / (8.0 * kPi * mu), wd = w * (3.0 / (4.0 * kPi));
  double f0 = 0, f1 = 0, f2 = 0, q0 = 0, q1 = 0, q2 = 0;
  if (f) { f0 = f[3 * i]; f1 = f[3 * i + 1]; f2 = f[3 * i + 2]; }
  if (q) { q0 = q[3 * i]; q1 = q[3 * i + 1]; q2 = q[3 * i + 2]; }
  double2* r2 = reinterpret_cast<double2*>(rec + i * kRec);
  r2[0] = make_double2(centres[3 * s] + a * n0, centres[3 * s + 1] + a * n1);
  r2[1] = make_double2(centres[3 * s + 2] + a * n2, n0);
  r2[2] = make_double2(n1, n2);
  r2[3] = make_double2(ws * f0, ws * f1);
  r2[4] = make_double2(ws * f2, wd * q0);
  r2[5] = make_double2(wd * q1, wd * q2);
  qn3[i] = wd * (q0 * n0 + q1 * n1 + q2 * n2) * (1.0 / 3.0);
}

}  // namespace bie
