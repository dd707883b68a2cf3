// k_n4.cuh -- NEXT-4: FFT-accelerated near evaluation with rotations
// (PAPER §4.2 "General case", Fig 2; vector version P:394-404).
//
// For every target sphere t and each near source sphere s (eq 4.5), the exact
// exterior field of s's degree-<=p expansion (eqs 3.6-3.11, reading R1) is
// re-expanded in t's own vector spherical harmonics WITHOUT evaluating it at
// t's nodes:
//   (1) rotate s's exterior coefficients into the pair frame, whose pole points
//       from c_s to c_t: Q = Rz(alpha) Ry(beta) (reading R25), i.e.
//         c^R = Delta^H E(beta) Delta E(alpha) c,   E(g) = diag(e^{i m g}),
//       with Delta_n = the rotation operator of T = Rx(-pi/2) (T e_z = e_y,
//       so Ry(b) = T Rz(b) T^-1): a fixed (2n+1)^2 matrix per degree, built
//       once per context by quadrature (k_n4_delta);
//   (2) in the pair frame t's grid is pole-aligned: its nodes lie on p+1 discs
//       of constant (r_j, theta'_j) in s's spherical coordinates with the same
//       longitudes phi_k, so the field's m-th Fourier coefficient on disc j
//       is a Legendre sum over n (eq 4.8) -- the FFT of P:363 is not needed
//       at all, because the forward transform of stage (3) runs on the same
//       longitudes: the inverse and forward DFTs cancel mode by mode.  The
//       spherical components of s are turned into t's (a rotation by
//       theta_j - theta'_j in each meridian plane, eq 4.9's geometry);
//   (3) Legendre analysis over t's latitudes (the forward transform) gives t's
//       coefficients psi^{Y,G,X} in the pair frame; rotate them back,
//         b = E(-alpha) Delta^H E(-beta) Delta b^R,
//       and ACCUMULATE them ("add spherical harmonic coefficients from
//       itself and all its neighbors, and then perform one fast inverse
//       transform") -- the self-term kernel adds them to its own psi before
//       its single inverse transform.
// Cost per pair: O(p^3) (the Delta products), against O(p^4) for the direct
// evaluation at t's nodes (k_near).  The smooth-rule contribution of s at t's
// nodes is still subtracted pointwise (k_near, SMOOTH part only).
// Real fields: coefficients are stored for m >= 0 only (c_{n,-m} = conj
// c_{n,m} with eq 2.1's Y_n^{-m} = conj Y_n^m), and every stage keeps that
// symmetry, so only the m >= 0 rows are computed.
#pragma once
#include "common.cuh"
#include "k_setup.cuh"

namespace bie {

// offset (complex entries) of Delta_n in the packed table: sum_{n'<n} (2n'+1)^2
__host__ __device__ __forceinline__ int n4_doff(int n) { return n * (4 * n * n - 1) / 3; }
__host__ __device__ inline int64_t n4_delta_doubles(int p) { return 2LL * n4_doff(p + 1); }

// Normalised P~_n^m(t) (eq 2.1 without the Condon-Shortley phase, the
// normalisation of k_tables) for all n <= p, m >= 0, at t = cos th, s = sin th.
__device__ inline void n4_legendre_all(int p, double t, double s, double* out /* [nlm] */) {
  double pmm = 0.28209479177387814347;  // 1/sqrt(4 pi)
  for (int m = 0; m <= p; ++m) {
    if (m > 0) pmm *= s * sqrt((2.0 * m + 1.0) / (2.0 * m));
    double pprev = 0.0, pcur = pmm;
    for (int n = m; n <= p; ++n) {
      if (n == m + 1) {
        pprev = pcur;
        pcur = t * sqrt(2.0 * m + 3.0) * pmm;
      } else if (n > m + 1) {
        const double an = sqrt((4.0 * n * n - 1.0) / ((double)n * n - (double)m * m));
        const double bn = sqrt(((n - 1.0) * (n - 1.0) - (double)m * m) / (4.0 * (n - 1.0) * (n - 1.0) - 1.0));
        const double nx = an * (t * pcur - bn * pprev);
        pprev = pcur;
        pcur = nx;
      }
      out[lm_index(p, n, m)] = pcur;
    }
  }
}

// Setup 1: P~_n^m at the rotated unit-grid directions T n_k, T(x,y,z) = (x,z,-y)
// (one thread per node): rot[k][nlm] Legendre values, rphi[k] = longitude.
__global__ void k_n4_rotpts(int p, const double* __restrict__ tab, double* __restrict__ rot,
                            double* __restrict__ rphi) {
  const TableLayout L(p);
  const int nsn = (p + 1) * L.nphi;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nsn) return;
  const int j = k / L.nphi, kk = k - j * L.nphi;
  const double st = tab[L.st + j], ct = tab[L.t + j];
  const double x = st * tab[L.cph + kk], y = st * tab[L.sph + kk], z = ct;
  const double tx = x, ty = z, tz = -y;  // T n
  const double rs = sqrt(tx * tx + ty * ty);
  n4_legendre_all(p, tz, rs, rot + (int64_t)k * L.nlm);
  rphi[k] = atan2(ty, tx);
}

// Setup 2: Delta_n[m'][m] = <Y_n^m', Y_n^m o T> by the grid quadrature (exact:
// the integrand has degree 2n <= 2p), one block per degree n.
__global__ void k_n4_delta(int p, const double* __restrict__ tab, const double* __restrict__ rot,
                           const double* __restrict__ rphi, double* __restrict__ delta,
                           double* __restrict__ deltaT) {
  const TableLayout L(p);
  const int n = blockIdx.x, W = 2 * n + 1, nsn = (p + 1) * L.nphi;
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
    const int mp = e / W - n, m = e % W - n;
    const int amp = mp < 0 ? -mp : mp, am = m < 0 ? -m : m;
    double re = 0.0, im = 0.0;
    for (int k = 0; k < nsn; ++k) {
      const int j = k / L.nphi, kk = k - j * L.nphi;
      const double w = tab[L.wu + j];
      // conj Y_n^{m'}(n_k) = P~ e^{-i m' phi_k}
      const double a = tab[L.P + (int64_t)j * L.nlm + lm_index(p, n, amp)];
      double sa, ca;
      sincospi(-2.0 * mp * kk / L.nphi, &sa, &ca);
      // Y_n^m(T n_k) = P~(cos th') e^{i m phi'}
      const double b = rot[(int64_t)k * L.nlm + lm_index(p, n, am)];
      double sb, cb;
      sincos(m * rphi[k], &sb, &cb);
      const double pr = w * a * b;
      re += pr * (ca * cb - sa * sb);
      im += pr * (ca * sb + sa * cb);
    }
    delta[2 * (n4_doff(n) + e)] = re;
    delta[2 * (n4_doff(n) + e) + 1] = im;
    const int eT = (m + n) * W + (mp + n);  // transposed copy: rows over m
    deltaT[2 * (n4_doff(n) + eT)] = re;
    deltaT[2 * (n4_doff(n) + eT) + 1] = im;
  }
}

struct N4Args {
  int p, nsn;
  const double* tab;
  const double* centres;
  const double* radii;
  const double* coef;    // [ns][nlm][10] exterior coefficients (k_near_coef)
  const double* delta;   // packed Delta_n
  const double* deltaT;  // packed Delta_n^T (coalesced row products)
  const int* tgt;        // target spheres with >= 1 near neighbour
  const int* nb_off;     // [ns+1]
  const int* nb_idx;     // neighbour sphere indices (ascending)
  double* psi;           // [ns][nlm][6] out: accumulated psi^{Y,G,X} (re, im)
};

__host__ __device__ inline int64_t n4_smem_doubles(int p) {
  const int nlm = (p + 1) * (p + 2) / 2, P1 = p + 1;
  return 8LL * nlm + 8LL * nlm + 8LL * nlm + 6LL * P1 * P1 + 6LL * nlm + 3LL * nlm + nlm;
}

// complex helpers (re, im) in registers
struct Cx {
  double r, i;
};
__device__ __forceinline__ Cx cmul(Cx a, Cx b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
__device__ __forceinline__ Cx cfma(Cx a, Cx b, Cx c) {  // a b + c
  return {fma(a.r, b.r, fma(-a.i, b.i, c.r)), fma(a.r, b.i, fma(a.i, b.r, c.i))};
}
__device__ __forceinline__ Cx cfma_conj(Cx a, Cx b, Cx c) {  // conj(a) b + c
  return {fma(a.r, b.r, fma(a.i, b.i, c.r)), fma(a.r, b.i, fma(-a.i, b.r, c.i))};
}


// One CTA per target sphere with near neighbours; neighbours in ascending
// index (deterministic accumulation).
__global__ void __launch_bounds__(128) k_n4(const N4Args A) {
  extern __shared__ __align__(16) double sm[];
  const int p = A.p, P1 = p + 1, nphi = 2 * p + 2;
  const TableLayout L(p);
  const int nlm = L.nlm;
  double* R1 = sm;              // [4 fam][nlm][2]: c (m >= 0); later b^R [3][nlm][2]
  double* R2 = R1 + 8 * nlm;    // [4][nlm][2]: Delta E(alpha) c; later Delta b^R
  double* CR = R2 + 8 * nlm;    // [nlm][8]: rotated c1..c4 (pair frame)
  double* F = CR + 8 * nlm;     // [P1 j][P1 m][3 comp][2]
  double* ACC = F + 6 * P1 * P1;  // [nlm][6]
  double* rt = ACC + 6 * nlm;   // rA, rB, rC
  // item q (degree-major: q = n(n+1)/2 + m) -> (n, m, lm column); consecutive
  // threads then share n and walk m, so the rotation matrices are read in
  // consecutive addresses (Delta^T for the row products, Delta for the column ones)
  int* nmc = reinterpret_cast<int*>(rt + 3 * nlm);  // [nlm][2]: (n << 16 | m), column
  const int tid = threadIdx.x, nt = blockDim.x;
  const int t = A.tgt[blockIdx.x];
  const double ct_[3] = {A.centres[3 * t], A.centres[3 * t + 1], A.centres[3 * t + 2]};
  const double at = A.radii[t];
  for (int e = tid; e < 3 * nlm; e += nt) rt[e] = A.tab[L.rA + e];
  for (int e = tid; e < 6 * nlm; e += nt) ACC[e] = 0.0;
  for (int q = tid; q < nlm; q += nt) {
    int n = 0;
    while ((n + 1) * (n + 2) / 2 <= q) ++n;
    const int m = q - n * (n + 1) / 2;
    nmc[2 * q] = (n << 16) | m;
    nmc[2 * q + 1] = lm_index(p, n, m);
  }
  __syncthreads();
  const double* rA = rt;
  const double* rB = rt + nlm;
  const double* rC = rt + 2 * nlm;
  auto cofs = [&](int c) {  // (n, m) of coefficient column c (m-major)
    int m = 0, off = 0;
    while (off + (P1 - m) <= c) { off += P1 - m; ++m; }
    return make_int2(m + (c - off), m);
  };
  for (int qn = A.nb_off[t]; qn < A.nb_off[t + 1]; ++qn) {
    const int s = A.nb_idx[qn];
    const double as = A.radii[s];
    double d[3] = {ct_[0] - A.centres[3 * s], ct_[1] - A.centres[3 * s + 1], ct_[2] - A.centres[3 * s + 2]};
    const double Cz = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    const double beta = acos(fmin(1.0, fmax(-1.0, d[2] / Cz))), alpha = atan2(d[1], d[0]);
    __syncthreads();  // previous pair done with R1/R2/CR/F
    // ---- (1a) load c (families c1..c4) and apply E(alpha)
    const double* cf = A.coef + (int64_t)s * nlm * 10;
    for (int e = tid; e < 4 * nlm; e += nt) {
      const int f = e / nlm, c = e - f * nlm;
      const int m = cofs(c).y;
      double sa, ca;
      sincos(m * alpha, &sa, &ca);
      const Cx v = {cf[10 * c + 2 * f], cf[10 * c + 2 * f + 1]};
      const Cx r = cmul(v, Cx{ca, sa});
      R1[2 * e] = r.r;
      R1[2 * e + 1] = r.i;
    }
    __syncthreads();
    // ---- (1b) x = Delta (E(alpha) c), rows m' >= 0, then E(beta)
    for (int e = tid; e < 4 * nlm; e += nt) {
      const int f = e & 3, q = e >> 2;  // families fastest: 4 lanes share each matrix entry
      const int n = nmc[2 * q] >> 16, mp = nmc[2 * q] & 0xFFFF, c = nmc[2 * q + 1];
      Cx acc = {0.0, 0.0};
      const double* DT = A.deltaT + 2 * n4_doff(n);
      const int W = 2 * n + 1;
      for (int m = -n; m <= n; ++m) {
        const int am = m < 0 ? -m : m;
        const int cc = f * nlm + lm_index(p, n, am);
        Cx x = {R1[2 * cc], R1[2 * cc + 1]};
        if (m < 0) x.i = -x.i;
        const int de = (m + n) * W + (mp + n);  // Delta[mp][m] from the transpose
        acc = cfma(Cx{__ldg(DT + 2 * de), __ldg(DT + 2 * de + 1)}, x, acc);
      }
      double sb, cb;
      sincos(mp * beta, &sb, &cb);
      const Cx r = cmul(acc, Cx{cb, sb});
      R2[2 * (f * nlm + c)] = r.r;
      R2[2 * (f * nlm + c) + 1] = r.i;
    }
    __syncthreads();
    // ---- (1c) c^R = Delta^H (E(beta) Delta E(alpha) c), rows m >= 0 -> CR[c][2 f]
    for (int e = tid; e < 4 * nlm; e += nt) {
      const int f = e & 3, q = e >> 2;  // families fastest: 4 lanes share each matrix entry
      const int n = nmc[2 * q] >> 16, m = nmc[2 * q] & 0xFFFF, c = nmc[2 * q + 1];
      Cx acc = {0.0, 0.0};
      const double* D = A.delta + 2 * n4_doff(n);
      const int W = 2 * n + 1;
      for (int mp = -n; mp <= n; ++mp) {
        const int amp = mp < 0 ? -mp : mp;
        const int cc = f * nlm + lm_index(p, n, amp);
        Cx x = {R2[2 * cc], R2[2 * cc + 1]};
        if (mp < 0) x.i = -x.i;
        const int de = (mp + n) * W + (m + n);
        acc = cfma_conj(Cx{__ldg(D + 2 * de), __ldg(D + 2 * de + 1)}, x, acc);
      }
      CR[8 * c + 2 * f] = acc.r;
      CR[8 * c + 2 * f + 1] = acc.i;
    }
    __syncthreads();
    // ---- (2) pole-aligned discs: F[j][m] = t-frame components of the m-th mode
    for (int e = tid; e < P1 * P1; e += nt) {
      const int j = e / P1, m = e - j * P1;
      const double ctj = A.tab[L.t + j], stj = A.tab[L.st + j];
      const double X = at * stj, Z = Cz + at * ctj;  // disc point (rho, z) in the pair frame
      const double R = sqrt(X * X + Z * Z);
      const double cth = Z / R, sth = X / R;  // theta' of the disc (sin >= 0)
      const double rho = as / R;              // 1/r in units of a_s
      // Legendre chain at theta' for order m (normalised; Pc = P~/sin for m >= 1)
      double pbar = 0.28209479177387814347;
      for (int k = 1; k <= m; ++k) pbar *= (k == 1 ? sqrt(1.5) : sth * sqrt((2.0 * k + 1.0) / (2.0 * k)));
      double Pp = 0.0, Pc = pbar, dPp = 0.0, dPc = 0.0;
      double rn = 1.0;
      for (int k = 0; k < m; ++k) rn *= rho;
      double Ur0 = 0, Ur1 = 0, Ut0 = 0, Ut1 = 0, Up0 = 0, Up1 = 0;
      const int c0 = lm_index(p, m, m);
      for (int n = m; n <= p; ++n) {
        const int cc = c0 + (n - m);
        if (n > m) {
          const double nx = rA[cc] * (cth * Pc - rB[cc] * Pp);
          if (m == 0) {
            const double dnx = rA[cc] * (cth * dPc - sth * Pc - rB[cc] * dPp);
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
          Pt = sth * Pc;
          mPs = m * Pc;
          dPt = n * cth * Pc - rC[cc] * (n > m ? Pp : 0.0);
        }
        const double* o = CR + 8 * cc;  // c1 c2 c3 c4 (re, im)
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
        rn *= rho;
      }
      if (m == 0) { Ur1 = 0.0; Ut1 = 0.0; Up1 = 0.0; }  // real m = 0 mode
      // s-frame (e_r', e_th') -> t-frame (e_r, e_th): rotation by d = th_j - th'_j
      const double cd = ctj * cth + stj * sth, sd = stj * cth - ctj * sth;
      double* o = F + 6 * (j * P1 + m);
      o[0] = cd * Ur0 + sd * Ut0;
      o[1] = cd * Ur1 + sd * Ut1;
      o[2] = -sd * Ur0 + cd * Ut0;
      o[3] = -sd * Ur1 + cd * Ut1;
      o[4] = Up0;
      o[5] = Up1;
    }
    __syncthreads();
    // ---- (3a) analysis over t's latitudes: b^R = (Y, G/(n(n+1)), X/(n(n+1))) -> R1 [3][nlm]
    for (int c = tid; c < nlm; c += nt) {
      const int2 nm = cofs(c);
      const int n = nm.x, m = nm.y;
      double y0 = 0, y1 = 0, g0 = 0, g1 = 0, x0 = 0, x1 = 0;
      for (int j = 0; j < P1; ++j) {
        const double wj = A.tab[L.wu + j] * nphi;  // lambda_j 2 pi
        const double Pv = wj * A.tab[L.P + (int64_t)j * nlm + c];
        const double dPv = wj * A.tab[L.dP + (int64_t)j * nlm + c];
        const double mPv = wj * A.tab[L.mPs + (int64_t)j * nlm + c];
        const double* o = F + 6 * (j * P1 + m);
        y0 = fma(Pv, o[0], y0);
        y1 = fma(Pv, o[1], y1);
        g0 = fma(dPv, o[2], fma(mPv, o[5], g0));
        g1 = fma(dPv, o[3], fma(-mPv, o[4], g1));
        x0 = fma(dPv, o[4], fma(-mPv, o[3], x0));
        x1 = fma(dPv, o[5], fma(mPv, o[2], x1));
      }
      const double inn = n ? 1.0 / ((double)n * (n + 1)) : 0.0;
      R1[2 * c] = y0;
      R1[2 * c + 1] = y1;
      R1[2 * (nlm + c)] = g0 * inn;
      R1[2 * (nlm + c) + 1] = g1 * inn;
      R1[2 * (2 * nlm + c)] = x0 * inn;
      R1[2 * (2 * nlm + c) + 1] = x1 * inn;
    }
    __syncthreads();
    // ---- (3b) x = Delta b^R (rows m' >= 0), then E(-beta)
    for (int e = tid; e < 3 * nlm; e += nt) {
      const int q = e / 3, f = e - 3 * q;  // families fastest: 3 lanes share each matrix entry
      const int n = nmc[2 * q] >> 16, mp = nmc[2 * q] & 0xFFFF, c = nmc[2 * q + 1];
      Cx acc = {0.0, 0.0};
      const double* DT = A.deltaT + 2 * n4_doff(n);
      const int W = 2 * n + 1;
      for (int m = -n; m <= n; ++m) {
        const int am = m < 0 ? -m : m;
        const int cc = f * nlm + lm_index(p, n, am);
        Cx x = {R1[2 * cc], R1[2 * cc + 1]};
        if (m < 0) x.i = -x.i;
        const int de = (m + n) * W + (mp + n);
        acc = cfma(Cx{__ldg(DT + 2 * de), __ldg(DT + 2 * de + 1)}, x, acc);
      }
      double sb, cb;
      sincos(mp * beta, &sb, &cb);
      const Cx r = cmul(acc, Cx{cb, -sb});
      R2[2 * (f * nlm + c)] = r.r;
      R2[2 * (f * nlm + c) + 1] = r.i;
    }
    __syncthreads();
    // ---- (3c) b = E(-alpha) Delta^H (...), rows m >= 0; accumulate
    for (int e = tid; e < 3 * nlm; e += nt) {
      const int q = e / 3, f = e - 3 * q;  // families fastest: 3 lanes share each matrix entry
      const int n = nmc[2 * q] >> 16, m = nmc[2 * q] & 0xFFFF, c = nmc[2 * q + 1];
      Cx acc = {0.0, 0.0};
      const double* D = A.delta + 2 * n4_doff(n);
      const int W = 2 * n + 1;
      for (int mp = -n; mp <= n; ++mp) {
        const int amp = mp < 0 ? -mp : mp;
        const int cc = f * nlm + lm_index(p, n, amp);
        Cx x = {R2[2 * cc], R2[2 * cc + 1]};
        if (mp < 0) x.i = -x.i;
        const int de = (mp + n) * W + (m + n);
        acc = cfma_conj(Cx{__ldg(D + 2 * de), __ldg(D + 2 * de + 1)}, x, acc);
      }
      double sa, ca;
      sincos(m * alpha, &sa, &ca);
      const Cx r = cmul(acc, Cx{ca, -sa});
      ACC[6 * c + 2 * f] += r.r;
      ACC[6 * c + 2 * f + 1] += (m == 0) ? 0.0 : r.i;
    }
  }
  __syncthreads();
  for (int e = tid; e < 6 * nlm; e += nt) A.psi[(int64_t)t * 6 * nlm + e] = ACC[e];
}

}  // namespace bie
