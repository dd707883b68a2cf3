// k_traction.cuh -- exact traction of one sphere's single-layer expansion,
// used by the near-singular correction of the traction operator K
// (PAPER eqs 3.17-3.18, with the eq 4.5
// partition of NEXT-1).  For a target node x (normal n) on sphere t and a
// near source sphere s, the smooth-rule K sum over s's nodes is replaced by
// the exact traction of s's degree-<=p single-layer expansion:
//     K_t(x) += T_s(x; n) - smooth_K_s(x; n),
//     T_s = (grad u + grad u^T) n - p n,   u, p = exterior S field of s
// (mu- and a-free: the a/mu of S and the 1/a of grad cancel; reading R24 for
// the sign of the pressure term).
//
// Evaluation (different route from the oracle's spherical formulas of eq
// 3.18): everything is Cartesian and pole-safe.  With d = (x - c)/a,
// xh = d/|d|, zeta = xh_z, xi = xh_x + i xh_y,
//     Y_n^m(xh) = Q_n^m(zeta) xi^m          (Q: normalised Legendre / sin^m)
//     grad_g Y  = P_T (m Q xi^{m-1} (1, i, 0) + Q'(zeta) xi^m e_z),
// P_T = I - xh xh^T, and the velocity in the k_near coefficient form
//     u = Re sum wm [ gY Y xh + gG grad_g Y + bX xh x grad_g Y ].
// grad u comes from forward-mode dual numbers (value + d/dd_x, d/dd_y,
// d/dd_z) carried through every operation -- no theta/phi, no 1/sin theta,
// so targets on the source's polar axis are exact.
#pragma once
#include "common.cuh"
#include "k_setup.cuh"

namespace bie {

// ------------------------------------------------------------ dual numbers
struct D3 {
  double v, x, y, z;
};
__device__ __forceinline__ D3 d3(double v) { return {v, 0.0, 0.0, 0.0}; }
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return {a.v + b.v, a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return {a.v - b.v, a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 operator*(double s, D3 a) { return {s * a.v, s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ D3 operator*(D3 a, D3 b) {
  return {a.v * b.v, fma(a.v, b.x, a.x * b.v), fma(a.v, b.y, a.y * b.v), fma(a.v, b.z, a.z * b.v)};
}
// a + s * b
__device__ __forceinline__ D3 fmad(double s, D3 b, D3 a) {
  return {fma(s, b.v, a.v), fma(s, b.x, a.x), fma(s, b.y, a.y), fma(s, b.z, a.z)};
}
// a + b * c
__device__ __forceinline__ D3 fmad(D3 b, D3 c, D3 a) {
  return {fma(b.v, c.v, a.v), fma(b.v, c.x, fma(b.x, c.v, a.x)), fma(b.v, c.y, fma(b.y, c.v, a.y)),
          fma(b.v, c.z, fma(b.z, c.v, a.z))};
}

struct C3 {  // complex dual
  D3 re, im;
};
__device__ __forceinline__ C3 c3(D3 re) { return {re, d3(0.0)}; }
__device__ __forceinline__ C3 operator+(C3 a, C3 b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ C3 operator-(C3 a, C3 b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ C3 operator*(C3 a, C3 b) {
  return {a.re * b.re - a.im * b.im, fmad(a.re, b.im, a.im * b.re)};
}
__device__ __forceinline__ C3 operator*(D3 s, C3 a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ C3 operator*(double s, C3 a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ C3 mul_i(C3 a) { return {d3(0.0) - a.im, a.re}; }
// a + (cr + i ci) * q,  q real dual
__device__ __forceinline__ C3 cfma(double cr, double ci, D3 q, C3 a) {
  return {fmad(cr, q, a.re), fmad(ci, q, a.im)};
}

// -------------------------------------------- exterior traction of sphere s
// cf: k_near_coef_K block of sphere s ([nlm][10]: c1..c4 (re, im) of the S
// field, pressure coefficient cp); rA, rB: normalised Legendre recurrence.
__device__ __noinline__ void exterior_traction(int p, const double* __restrict__ cf,
                                               const double* __restrict__ rA,
                                               const double* __restrict__ rB, const double* c,
                                               double a, const double* x, const double* nv,
                                               double out[3]) {
  const double ia = 1.0 / a;
  const D3 dx = {(x[0] - c[0]) * ia, 1.0, 0.0, 0.0};
  const D3 dy = {(x[1] - c[1]) * ia, 0.0, 1.0, 0.0};
  const D3 dz = {(x[2] - c[2]) * ia, 0.0, 0.0, 1.0};
  const double r2v = fma(dz.v, dz.v, fma(dy.v, dy.v, dx.v * dx.v));
  const double rv = sqrt(r2v);
  const double rhov = 1.0 / rv;
  const double hx = dx.v * rhov, hy = dy.v * rhov, hz = dz.v * rhov;
  // rho = 1/r: d rho / dd_j = -rho^2 xh_j;  xh_i = d_i rho
  const D3 rho = {rhov, -rhov * rhov * hx, -rhov * rhov * hy, -rhov * rhov * hz};
  const D3 X = dx * rho, Yc = dy * rho, Z = dz * rho;  // xh as duals
  const D3 rho2 = rho * rho;
  const C3 xi = {X, Yc};
  const double inv_sqrt4pi = 0.28209479177387814347;
  C3 u[3] = {c3(d3(0.0)), c3(d3(0.0)), c3(d3(0.0))};
  double pr = 0.0;
  C3 Em = c3(d3(1.0)), Em1 = c3(d3(0.0));  // xi^m, xi^{m-1}
  D3 rho_m = d3(1.0);                      // r^{-m}
  double qmm = inv_sqrt4pi;                // Q_m^m
  for (int m = 0; m <= p; ++m) {
    if (m > 0) qmm *= sqrt((2.0 * m + 1.0) / (2.0 * m));
    C3 SY = c3(d3(0.0)), SG = SY, SGd = SY, SX = SY, SXd = SY;
    double Pp0 = 0.0, Pp1 = 0.0;
    D3 Qc = d3(qmm), Qp = d3(0.0), dQc = d3(0.0), dQp = d3(0.0);
    D3 rn = rho_m;  // r^{-n}
    const int c0 = lm_index(p, m, m);
    for (int n = m; n <= p; ++n) {
      const int cc = c0 + (n - m);
      if (n > m) {
        // Q_n = rA (zeta Q_{n-1} - rB Q_{n-2});  Q'_n = rA (Q_{n-1} + zeta Q'_{n-1} - rB Q'_{n-2})
        const D3 nq = rA[cc] * fmad(-rB[cc], Qp, Z * Qc);
        const D3 ndq = rA[cc] * fmad(-rB[cc], dQp, fmad(Z, dQc, Qc));
        Qp = Qc;
        Qc = nq;
        dQp = dQc;
        dQc = ndq;
      }
      const double* o = cf + 10 * cc;
      // bV = r^{-n} (c1 r^{-2} + c2), bW = r^{-n} c3, bX = r^{-n-1} c4
      const D3 rq = rn * Qc, rdq = rn * dQc;                  // r^{-n} Q, r^{-n} Q'
      const D3 r2q = rho2 * rq, r2dq = rho2 * rdq;            // r^{-n-2} Q, ...
      const D3 r1q = rho * rq, r1dq = rho * rdq;              // r^{-n-1} Q, ...
      // gG = bV + bW, gY = -(n+1) bV + n bW  (times Q or Q')
      const double gG2r = o[2] + o[4], gG2i = o[3] + o[5];    // r^{-n} part of gG
      const double gY2r = -(n + 1.0) * o[2] + n * o[4], gY2i = -(n + 1.0) * o[3] + n * o[5];
      const double gY0r = -(n + 1.0) * o[0], gY0i = -(n + 1.0) * o[1];
      SY = cfma(gY0r, gY0i, r2q, cfma(gY2r, gY2i, rq, SY));
      SG = cfma(o[0], o[1], r2q, cfma(gG2r, gG2i, rq, SG));
      SGd = cfma(o[0], o[1], r2dq, cfma(gG2r, gG2i, rdq, SGd));
      SX = cfma(o[6], o[7], r1q, SX);
      SXd = cfma(o[6], o[7], r1dq, SXd);
      Pp0 = fma(o[8], r1q.v, Pp0);
      Pp1 = fma(o[9], r1q.v, Pp1);
      rn = rn * rho;
    }
    // grad_g-type vectors before projection: v = m S xi^{m-1} (1, i, 0) + S' xi^m e_z
    const C3 gx = (double)m * (SG * Em1), gz = SGd * Em;
    const C3 gy = mul_i(gx);
    const C3 xx = (double)m * (SX * Em1), xz = SXd * Em;
    const C3 xy = mul_i(xx);
    // tangential projection of the G vector
    const C3 hg = X * gx + Yc * gy + Z * gz;
    const C3 TGx = gx - X * hg, TGy = gy - Yc * hg, TGz = gz - Z * hg;
    // xh x v_X
    const C3 CXx = Yc * xz - Z * xy, CXy = Z * xx - X * xz, CXz = X * xy - Yc * xx;
    const C3 YE = SY * Em;
    const double wm = m ? 2.0 : 1.0;
    const C3 um0 = X * YE + TGx + CXx, um1 = Yc * YE + TGy + CXy, um2 = Z * YE + TGz + CXz;
    u[0].re = fmad(wm, um0.re, u[0].re);
    u[1].re = fmad(wm, um1.re, u[1].re);
    u[2].re = fmad(wm, um2.re, u[2].re);
    // pressure Re(sum cp r^{-n-1} Q xi^m), values only
    pr += wm * (Pp0 * Em.re.v - Pp1 * Em.im.v);
    Em1 = Em;
    Em = Em * xi;
    rho_m = rho_m * rho;
  }
  // G_ij = d u_i / d d_j ; traction = (G + G^T) n - p n  (a-free)
  const double G[3][3] = {{u[0].re.x, u[0].re.y, u[0].re.z},
                          {u[1].re.x, u[1].re.y, u[1].re.z},
                          {u[2].re.x, u[2].re.y, u[2].re.z}};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double t = -pr * nv[i];
#pragma unroll
    for (int j = 0; j < 3; ++j) t = fma(G[i][j] + G[j][i], nv[j], t);
    out[i] = t;
  }
}

// Per-sphere coefficients of the exterior S field of sigma, from the k_self
// projections of sigma in the q slot (unscaled): same c1..c4 as k_near_coef
// with f := sigma, a/mu := 1, q := 0; pressure cp = n alpha_W.
__global__ void k_near_coef_K(int p, int64_t ns, const double* __restrict__ alpha,
                              double* __restrict__ coef) {
  const TableLayout L(p);
  const int nlm = L.nlm;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ns * nlm) return;
  const int64_t s = e / nlm;
  const int c = (int)(e - s * nlm);
  int m = 0, off = 0;
  while (off + (p + 1 - m) <= c) { off += p + 1 - m; ++m; }
  const int n = m + (c - off);
  const double* af = alpha + ((int64_t)s * 2 * nlm + nlm + c) * 6;  // q slot
  const double inn = n ? 1.0 / ((double)n * (n + 1)) : 0.0;
  const double i2n = 1.0 / (2.0 * n + 1.0);
  const double lSV = n / ((2.0 * n + 1.0) * (2.0 * n + 3.0));
  const double xS = n / (4.0 * n + 2.0);
  const double wS = n ? (n + 1.0) / ((2.0 * n + 1.0) * (2.0 * n - 1.0)) : 0.0;
  const double kS = n ? 1.0 / (2.0 * n + 1.0) : 0.0;
  double* o = coef + e * 10;
#pragma unroll
  for (int ri = 0; ri < 2; ++ri) {
    const double fV = (n * af[2 + ri] * inn - af[ri]) * i2n;
    const double fW = n ? ((n + 1) * af[2 + ri] * inn + af[ri]) * i2n : 0.0;
    const double fX = af[4 + ri] * inn;
    o[0 + ri] = fV * lSV + fW * xS;
    o[2 + ri] = -(fW * xS);
    o[4 + ri] = fW * wS;
    o[6 + ri] = fX * kS;
    o[8 + ri] = n * fW;
  }
}

}  // namespace bie
