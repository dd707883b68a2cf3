// =============================================================================
// oracle/oracle.cpp -- plain, slow, obviously-correct CPU oracle for the
// discretised Stokes boundary-integral-operator apply of Corona & Veerapaneni,
// arXiv 1707.06551.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  It
// shares no code, header, table or constant generator with the CUDA path in
// paper_1707_06551_b200/ and never calls it.
//
// Precision: IEEE fp64, compiled with -O2 -ffp-contract=off (no FMA
// contraction, no fast-math); far-field and off-surface sums use Neumaier
// compensated accumulation in ascending source order.
//
// Citations "P:n" are PAPER.md line numbers; "SURVEY" is /root/repo/SURVEY.md;
// readings of garbled/ambiguous passages are listed in DESIGN.md §3.
//
// Steps:
//   O-1 oracle_gl_rule      Gauss-Legendre rule, eq 4.2
//   O-2 oracle_nodes        nodes/normals/weights, eqs 4.2, 4.4,
//                           reading R4 (w = a^2 lambda_j 2pi/(2p+2))
//   O-3 oracle_far          smooth Nystrom sum of S and D, eqs 2.19-2.21, 4.4
//                           (P:121-132), stresslet sign reading R1,
//                           own sphere excluded (reading R8)
//   O-4 oracle_self         self term: discrete VSH projection (eqs 2.1, 2.3,
//                           2.4-2.6), diagonal scale by the r->1
//                           limits of eqs 3.6-3.11 (readings R2,R3),
//                           inverse expansion (eq 2.12)
//   O-6 oracle_offsurface   velocity + pressure at arbitrary targets (reading R12)
//   O-7 oracle_self_addthm  the same self operator built from the addition
//                           theorem, an internal cross-check
//   helpers for pins: oracle_ylm, oracle_vsh, oracle_eigen
// Beyond §8(a), each pinned in tests/test_oracle_*.py:
//   NEXT-1  oracle_exterior_eval, oracle_is_near, oracle_near,
//           oracle_exterior_pressure, oracle_near_offsurface
//   NEXT-3  oracle_far_K, oracle_K_at (eq 2.22, reading R21),
//           oracle_exterior_traction, oracle_near_K, oracle_near_K_offsurface
//           (eqs 3.17-3.18, reading R24), oracle_completion (eq 5.8, R22)
//   (NEXT-2's dense operator and LU solve are in oracle/__init__.py.)
// =============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <omp.h>

typedef std::complex<double> cplx;
static const double PI = 3.141592653589793238462643383279502884;

// ---------------------------------------------------------------- utilities
struct Neumaier {  // compensated summation (Neumaier's variant of Kahan)
  double s = 0.0, c = 0.0;
  void add(double v) {
    double t = s + v;
    if (std::fabs(s) >= std::fabs(v)) c += (s - t) + v;
    else c += (v - t) + s;
    s = t;
  }
  double get() const { return s + c; }
};

// Legendre polynomial P_n(x) and derivative via the three-term recurrence.
static void legendre_pn(int n, double x, double* Pn, double* dPn) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { *Pn = 1.0; *dPn = 0.0; return; }
  for (int k = 2; k <= n; ++k) {
    double pk = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1; p1 = pk;
  }
  *Pn = p1;
  *dPn = n * (x * p1 - p0) / (x * x - 1.0);
}

// ------------------------------------------------------------------ O-1
// (p+1)-point Gauss-Legendre rule on [-1,1], nodes ascending (eq 4.2).
extern "C" int oracle_gl_rule(int p, double* t, double* lam) {
  if (p < 0 || !t || !lam) return 1;
  const int n = p + 1;
  for (int j = 0; j < n; ++j) {
    double x = -std::cos(PI * (j + 0.75) / (n + 0.5));
    double P, dP;
    for (int it = 0; it < 100; ++it) {
      legendre_pn(n, x, &P, &dP);
      double dx = P / dP;
      x -= dx;
      if (std::fabs(dx) < 1e-15) break;
    }
    legendre_pn(n, x, &P, &dP);  // one extra step
    x -= P / dP;
    legendre_pn(n, x, &P, &dP);
    t[j] = x;
    lam[j] = 2.0 / ((1.0 - x * x) * dP * dP);
  }
  return 0;
}

// ------------------------------------------------------------------ O-2
// Node i = s*(p+1)(2p+2) + j*(2p+2) + k: n = (sin th_j cos ph_k,
// sin th_j sin ph_k, t_j), x = c_s + a_s n, w = a_s^2 lambda_j 2pi/(2p+2).
extern "C" int oracle_nodes(const double* centres, const double* radii, int64_t ns, int p,
                            double* x, double* nrm, double* w) {
  if (ns < 1 || p < 1 || !centres || !radii) return 1;
  const int nphi = 2 * p + 2, nsn = (p + 1) * nphi;
  std::vector<double> t(p + 1), lam(p + 1);
  oracle_gl_rule(p, t.data(), lam.data());
  for (int64_t s = 0; s < ns; ++s)
    for (int j = 0; j <= p; ++j)
      for (int k = 0; k < nphi; ++k) {
        int64_t i = s * nsn + (int64_t)j * nphi + k;
        double st = std::sqrt(1.0 - t[j] * t[j]);
        double ph = 2.0 * PI * k / nphi;
        double n3[3] = {st * std::cos(ph), st * std::sin(ph), t[j]};
        for (int c = 0; c < 3; ++c) {
          if (nrm) nrm[3 * i + c] = n3[c];
          if (x) x[3 * i + c] = centres[3 * s + c] + radii[s] * n3[c];
        }
        if (w) w[i] = radii[s] * radii[s] * lam[j] * 2.0 * PI / nphi;
      }
  return 0;
}

struct Geometry {
  int p, nphi, nsn;
  int64_t ns, N;
  std::vector<double> x, n, w;
  Geometry(const double* c, const double* a, int64_t ns_, int p_) : p(p_), ns(ns_) {
    nphi = 2 * p + 2;
    nsn = (p + 1) * nphi;
    N = ns * nsn;
    x.resize(3 * N); n.resize(3 * N); w.resize(N);
    oracle_nodes(c, a, ns, p, x.data(), n.data(), w.data());
  }
};

// Smooth-rule contribution of source k at point xt (eqs 2.19-2.21 with 4.4):
//   S: w_k (1/(8 pi mu)) (f/r + (rho.f) rho / r^3)            (eq 2.19)
//   D: w_k (3/(4 pi)) (rho.n)(rho.q) rho / r^5                 (eq 2.20, R1)
//   pressure (R12): w_k [ (1/(4pi)) (rho.f)/r^3
//                         + (mu/(2pi)) (-(q.n)/r^3 + 3 (rho.q)(rho.n)/r^5) ]
static inline void pair_terms(const double* xt, const double* y, const double* ny, double wk,
                              const double* f, const double* q, double mu, double u[3],
                              double* pr) {
  double rho[3] = {xt[0] - y[0], xt[1] - y[1], xt[2] - y[2]};
  double r2 = rho[0] * rho[0] + rho[1] * rho[1] + rho[2] * rho[2];
  double r = std::sqrt(r2);
  double r3 = r2 * r, r5 = r3 * r2;
  u[0] = u[1] = u[2] = 0.0;
  double pv = 0.0;
  if (f) {
    double rf = rho[0] * f[0] + rho[1] * f[1] + rho[2] * f[2];
    double cS = wk / (8.0 * PI * mu);
    for (int c = 0; c < 3; ++c) u[c] += cS * (f[c] / r + rf * rho[c] / r3);
    pv += wk * rf / (4.0 * PI * r3);
  }
  if (q) {
    double rn = rho[0] * ny[0] + rho[1] * ny[1] + rho[2] * ny[2];
    double rq = rho[0] * q[0] + rho[1] * q[1] + rho[2] * q[2];
    double qn = q[0] * ny[0] + q[1] * ny[1] + q[2] * ny[2];
    double cD = 3.0 * wk / (4.0 * PI);
    for (int c = 0; c < 3; ++c) u[c] += cD * rn * rq * rho[c] / r5;
    pv += wk * mu / (2.0 * PI) * (-qn / r3 + 3.0 * rq * rn / r5);
  }
  if (pr) *pr = pv;
}

// ------------------------------------------------------------------ O-3
// Far field at the subset of nodes tidx[0..nt): sum over every node of every
// OTHER sphere (reading R8), ascending source index, Neumaier per component.
extern "C" int oracle_far(const double* centres, const double* radii, int64_t ns, int p,
                          double mu, const double* f, const double* q, const int64_t* tidx,
                          int64_t nt, double* u) {
  if (ns < 1 || p < 1 || !(mu > 0) || !u || !tidx) return 1;
  Geometry G(centres, radii, ns, p);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t i = tidx[t];
    const int64_t si = i / G.nsn;
    Neumaier acc[3];
    for (int64_t k = 0; k < G.N; ++k) {
      if (k / G.nsn == si) continue;
      double v[3];
      pair_terms(&G.x[3 * i], &G.x[3 * k], &G.n[3 * k], G.w[k], f ? f + 3 * k : nullptr,
                 q ? q + 3 * k : nullptr, mu, v, nullptr);
      for (int c = 0; c < 3; ++c) acc[c].add(v[c]);
    }
    for (int c = 0; c < 3; ++c) u[3 * t + c] = acc[c].get();
  }
  return 0;
}

// ------------------------------------------------------------------ O-6
// Off-surface velocity and pressure: sum over ALL nodes (no exclusion).
extern "C" int oracle_offsurface(const double* centres, const double* radii, int64_t ns, int p,
                                 double mu, const double* f, const double* q,
                                 const double* targets, int64_t m, double* u, double* pres) {
  if (ns < 1 || p < 1 || !(mu > 0) || (m > 0 && (!targets || !u))) return 1;
  Geometry G(centres, radii, ns, p);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < m; ++t) {
    Neumaier acc[3], pacc;
    for (int64_t k = 0; k < G.N; ++k) {
      double v[3], pv;
      pair_terms(&targets[3 * t], &G.x[3 * k], &G.n[3 * k], G.w[k], f ? f + 3 * k : nullptr,
                 q ? q + 3 * k : nullptr, mu, v, &pv);
      for (int c = 0; c < 3; ++c) acc[c].add(v[c]);
      pacc.add(pv);
    }
    for (int c = 0; c < 3; ++c) u[3 * t + c] = acc[c].get();
    if (pres) pres[t] = pacc.get();
  }
  return 0;
}

// ---------------------------------------------------------- harmonics (eq 2.1)
// Unnormalised associated Legendre P_n^m(x), m >= 0, WITHOUT the
// Condon-Shortley phase (eq 2.1 writes P_n^{|m|} with no phase), and
// d/dtheta P_n^m(cos theta) = (n cos th P_n^m - (n+m) P_{n-1}^m) / sin th.
static void assoc_legendre(int n, int m, double x, double* P, double* dPdth) {
  double s = std::sqrt(1.0 - x * x);
  double pmm = 1.0;
  for (int k = 1; k <= m; ++k) pmm *= (2.0 * k - 1.0) * s;  // (2m-1)!! s^m
  double pprev = 0.0, pcur = pmm;                             // P_{m-1}^m = 0
  for (int l = m + 1; l <= n; ++l) {
    double pn = ((2.0 * l - 1.0) * x * pcur - (l + m - 1.0) * pprev) / (l - m);
    pprev = pcur;
    pcur = pn;
  }
  *P = pcur;  // P_n^m ; pprev = P_{n-1}^m (0 when n == m)
  *dPdth = (n * x * pcur - (n + m) * pprev) / s;
}

static double ynm_norm(int n, int m) {  // sqrt((2n+1)/(4pi) (n-|m|)!/(n+|m|)!)
  int am = std::abs(m);
  double ratio = 1.0;
  for (int k = n - am + 1; k <= n + am; ++k) ratio /= k;
  return std::sqrt((2.0 * n + 1.0) / (4.0 * PI) * ratio);
}

// Y_n^m(theta,phi), dY/dtheta and (1/sin theta) dY/dphi (eq 2.1).
static void ynm_all(int n, int m, double th, double ph, cplx* Y, cplx* dY, cplx* dYphi) {
  int am = std::abs(m);
  double P, dP;
  assoc_legendre(n, am, std::cos(th), &P, &dP);
  double N = ynm_norm(n, m);
  cplx e = std::polar(1.0, m * ph);
  *Y = N * P * e;
  *dY = N * dP * e;
  *dYphi = cplx(0.0, (double)m) * N * P * e / std::sin(th);
}

// Cartesian V, W, X (eqs 2.4-2.6) at (th, ph): out[0..2]=V, [3..5]=W, [6..8]=X.
static void vsh_cart(int n, int m, double th, double ph, cplx out[9]) {
  cplx Y, dY, dYp;
  ynm_all(n, m, th, ph, &Y, &dY, &dYp);
  double st = std::sin(th), ct = std::cos(th), sp = std::sin(ph), cp = std::cos(ph);
  double er[3] = {st * cp, st * sp, ct}, et[3] = {ct * cp, ct * sp, -st}, ep[3] = {-sp, cp, 0.0};
  for (int c = 0; c < 3; ++c) {
    cplx grad = dY * et[c] + dYp * ep[c];               // surface gradient
    out[c] = grad - (double)(n + 1) * Y * er[c];        // V  (2.4)
    out[3 + c] = grad + (double)n * Y * er[c];          // W  (2.5)
    out[6 + c] = dY * ep[c] - dYp * et[c];              // X = e_r x grad (2.6)
  }
}

extern "C" void oracle_ylm(int n, int m, double th, double ph, double* out6) {
  cplx Y, dY, dYp;
  ynm_all(n, m, th, ph, &Y, &dY, &dYp);
  out6[0] = Y.real(); out6[1] = Y.imag();
  out6[2] = dY.real(); out6[3] = dY.imag();
  out6[4] = dYp.real(); out6[5] = dYp.imag();
}

extern "C" void oracle_vsh(int n, int m, double th, double ph, double* out18) {
  cplx z[9];
  vsh_cart(n, m, th, ph, z);
  for (int c = 0; c < 9; ++c) { out18[2 * c] = z[c].real(); out18[2 * c + 1] = z[c].imag(); }
}

// ------------------------------------------------------- eigenvalues (Thm 2)
// Unit sphere, mu = 1.  Channel ch: 0=V, 1=W, 2=X.  The r->1 limits of the
// exterior/interior branches of eqs 3.6-3.8 (S) and 3.9-3.11 (D);
// at r = 1 the cross terms vanish.  S is continuous (reading R3); the on-surface
// D is the principal value, the mean of the two limits (reading R2).
extern "C" void oracle_eigen(int n, int ch, double* lamS, double* lamD_ext, double* lamD_int,
                             double* lamD_pv) {
  double a = 2.0 * n + 1.0;
  double S = 0, De = 0, Di = 0;
  if (ch == 0) {         // V_n
    S = n / (a * (2.0 * n + 3.0));
    De = (2.0 * n * n + 4.0 * n + 3.0) / (a * (2.0 * n + 3.0));
    Di = -2.0 * n * (n + 2.0) / (a * (2.0 * n + 3.0));
  } else if (ch == 1) {  // W_n
    S = (n + 1.0) / (a * (2.0 * n - 1.0));
    De = 2.0 * (n + 1.0) * (n - 1.0) / (a * (2.0 * n - 1.0));
    Di = -(2.0 * n * n + 1.0) / (a * (2.0 * n - 1.0));
  } else {               // X_n
    S = 1.0 / a;
    De = (n - 1.0) / a;
    Di = -(n + 2.0) / a;
  }
  if (lamS) *lamS = S;
  if (lamD_ext) *lamD_ext = De;
  if (lamD_int) *lamD_int = Di;
  if (lamD_pv) *lamD_pv = 0.5 * (De + Di);
}

// ||Z_n||^2 on the unit sphere: V (n+1)(2n+1), W n(2n+1), X n(n+1).
static double vsh_norm2(int n, int ch) {
  if (ch == 0) return (n + 1.0) * (2.0 * n + 1.0);
  if (ch == 1) return n * (2.0 * n + 1.0);
  return n * (n + 1.0);
}

// ------------------------------------------------------------------ O-4
// Self term at the subset nodes tidx[0..nt):
//   alpha^Z_nm[g] = (1/||Z_n||^2) sum_{k in sphere} w^_k g_k . conj Z_nm(k),
//     w^_k = lambda_j 2pi/(2p+2), g in {(a/mu) f, q}            (eq 2.3 discretised)
//   psi = lamS(n,Z) alpha[(a/mu) f] + lamD_pv(n,Z) alpha[q]      (Thm 2)
//   u_i = Re sum_{n<=p, m, Z} psi Z_nm(i)                         (eq 2.12)
extern "C" int oracle_self(const double* centres, const double* radii, int64_t ns, int p,
                           double mu, const double* f, const double* q, const int64_t* tidx,
                           int64_t nt, double* u) {
  if (ns < 1 || p < 1 || !(mu > 0) || !u || !tidx) return 1;
  (void)centres;
  const int nphi = 2 * p + 2, nsn = (p + 1) * nphi;
  std::vector<double> t(p + 1), lam(p + 1);
  oracle_gl_rule(p, t.data(), lam.data());
  // table of Z_nm at the unit-grid nodes: index ((k*(p+1)^2 + (n*n+n+m))*3 + ch)*3 + c
  const int nlm = (p + 1) * (p + 1);
  std::vector<cplx> Z((size_t)nsn * nlm * 9);
  std::vector<double> what(nsn);
  for (int j = 0; j <= p; ++j)
    for (int k = 0; k < nphi; ++k) {
      int kk = j * nphi + k;
      what[kk] = lam[j] * 2.0 * PI / nphi;
      double th = std::acos(t[j]), ph = 2.0 * PI * k / nphi;
      for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m) {
          cplx z[9];
          vsh_cart(n, m, th, ph, z);
          for (int c = 0; c < 9; ++c) Z[((size_t)kk * nlm + n * n + n + m) * 9 + c] = z[c];
        }
    }
  // group targets by sphere
  std::vector<int64_t> order(nt);
  for (int64_t a = 0; a < nt; ++a) order[a] = a;
  std::vector<int64_t> sph(nt);
  for (int64_t a = 0; a < nt; ++a) sph[a] = tidx[a] / nsn;
  std::vector<int64_t> uniq(sph);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t ui = 0; ui < (int64_t)uniq.size(); ++ui) {
    const int64_t s = uniq[ui];
    const double aS = radii[s] / mu;
    std::vector<cplx> psi((size_t)nlm * 3, cplx(0.0, 0.0));
    for (int n = 0; n <= p; ++n)
      for (int m = -n; m <= n; ++m)
        for (int ch = 0; ch < 3; ++ch) {
          if (n == 0 && ch > 0) continue;  // W_0 = X_0 = 0 (reading R7)
          cplx af(0.0, 0.0), aq(0.0, 0.0);
          for (int kk = 0; kk < nsn; ++kk) {
            const cplx* z = &Z[((size_t)kk * nlm + n * n + n + m) * 9 + 3 * ch];
            int64_t i = s * nsn + kk;
            for (int c = 0; c < 3; ++c) {
              if (f) af += what[kk] * aS * f[3 * i + c] * std::conj(z[c]);
              if (q) aq += what[kk] * q[3 * i + c] * std::conj(z[c]);
            }
          }
          double nn = vsh_norm2(n, ch);
          double lS, lD;
          oracle_eigen(n, ch, &lS, nullptr, nullptr, &lD);
          psi[(size_t)(n * n + n + m) * 3 + ch] = lS * af / nn + lD * aq / nn;
        }
    for (int64_t a = 0; a < nt; ++a) {
      if (sph[a] != s) continue;
      int kk = (int)(tidx[a] - s * nsn);
      cplx acc[3] = {0.0, 0.0, 0.0};
      for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m)
          for (int ch = 0; ch < 3; ++ch) {
            if (n == 0 && ch > 0) continue;
            cplx ps = psi[(size_t)(n * n + n + m) * 3 + ch];
            const cplx* z = &Z[((size_t)kk * nlm + n * n + n + m) * 9 + 3 * ch];
            for (int c = 0; c < 3; ++c) acc[c] += ps * z[c];
          }
      for (int c = 0; c < 3; ++c) u[3 * a + c] = acc[c].real();
    }
  }
  return 0;
}

// ------------------------------------------------------------------ O-7
// The same discrete self operator on ONE sphere (all its nodes), built from
// the addition theorem instead of explicit harmonics:
//   sum_m Y(x) conj Y(y)          = c_n P_n(t),                 t = x.y
//   sum_m gradY(x) conj Y(y)      = c_n P_n'(t) (y - t x)
//   sum_m Y(x) conj gradY(y)      = c_n P_n'(t) (x - t y)
//   sum_m gradY(x) (x) conj gradY(y) = c_n [P_n''(t)(y - t x)(x - t y)^T
//                                        + P_n'(t)(I - x x^T)(I - y y^T)]
// with c_n = (2n+1)/(4 pi), V = gradY - (n+1) Y x, W = gradY + n Y x,
// X = x cross gradY.  u_i = sum_k w^_k sum_n sum_Z lam_Z(n)/||Z_n||^2 K_n^ZZ(x_i,x_k) g_k.
extern "C" int oracle_self_addthm(int p, double mu, double a, const double* f, const double* q,
                                  double* u) {
  if (p < 1 || !(mu > 0) || !(a > 0) || !u) return 1;
  const int nphi = 2 * p + 2, nsn = (p + 1) * nphi;
  std::vector<double> t(p + 1), lam(p + 1);
  oracle_gl_rule(p, t.data(), lam.data());
  std::vector<double> X(3 * nsn), wh(nsn);
  for (int j = 0; j <= p; ++j)
    for (int k = 0; k < nphi; ++k) {
      int kk = j * nphi + k;
      double st = std::sqrt(1.0 - t[j] * t[j]), ph = 2.0 * PI * k / nphi;
      X[3 * kk] = st * std::cos(ph);
      X[3 * kk + 1] = st * std::sin(ph);
      X[3 * kk + 2] = t[j];
      wh[kk] = lam[j] * 2.0 * PI / nphi;
    }
#pragma omp parallel for schedule(dynamic, 4)
  for (int i = 0; i < nsn; ++i) {
    const double* x = &X[3 * i];
    double acc[3] = {0, 0, 0};
    for (int k = 0; k < nsn; ++k) {
      const double* y = &X[3 * k];
      double tt = x[0] * y[0] + x[1] * y[1] + x[2] * y[2];
      // P_n, P_n', P_n'' by upward recurrences valid at t = +-1
      std::vector<double> P(p + 1), dP(p + 1), ddP(p + 1);
      P[0] = 1; dP[0] = 0; ddP[0] = 0;
      if (p >= 1) { P[1] = tt; dP[1] = 1; ddP[1] = 0; }
      for (int n = 2; n <= p; ++n) {
        P[n] = ((2.0 * n - 1.0) * tt * P[n - 1] - (n - 1.0) * P[n - 2]) / n;
        dP[n] = dP[n - 2] + (2.0 * n - 1.0) * P[n - 1];
        ddP[n] = ddP[n - 2] + (2.0 * n - 1.0) * dP[n - 1];
      }
      double ytx[3], xty[3];
      for (int c = 0; c < 3; ++c) { ytx[c] = y[c] - tt * x[c]; xty[c] = x[c] - tt * y[c]; }
      double Px[9], Py[9];  // I - x x^T, I - y y^T
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          Px[3 * r + c] = (r == c) - x[r] * x[c];
          Py[3 * r + c] = (r == c) - y[r] * y[c];
        }
      double PxPy[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          double s = 0;
          for (int l = 0; l < 3; ++l) s += Px[3 * r + l] * Py[3 * l + c];
          PxPy[3 * r + c] = s;
        }
      double KS[9] = {0}, KD[9] = {0};
      for (int n = 0; n <= p; ++n) {
        double cn = (2.0 * n + 1.0) / (4.0 * PI);
        double A0 = cn * P[n];
        double A1[3], A1p[3], T[9];
        for (int c = 0; c < 3; ++c) { A1[c] = cn * dP[n] * ytx[c]; A1p[c] = cn * dP[n] * xty[c]; }
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c)
            T[3 * r + c] = cn * (ddP[n] * ytx[r] * xty[c] + dP[n] * PxPy[3 * r + c]);
        double KV[9], KW[9], KX[9];
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) {
            KV[3 * r + c] = T[3 * r + c] - (n + 1.0) * A1[r] * y[c] - (n + 1.0) * x[r] * A1p[c] +
                            (n + 1.0) * (n + 1.0) * A0 * x[r] * y[c];
            KW[3 * r + c] = T[3 * r + c] + n * A1[r] * y[c] + n * x[r] * A1p[c] +
                            (double)n * n * A0 * x[r] * y[c];
          }
        // KX = [x]_x T [y]_x^T ; [v]_x w = v cross w
        double Cx[9] = {0, -x[2], x[1], x[2], 0, -x[0], -x[1], x[0], 0};
        double Cy[9] = {0, -y[2], y[1], y[2], 0, -y[0], -y[1], y[0], 0};
        double tmp[9];
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) {
            double s = 0;
            for (int l = 0; l < 3; ++l) s += Cx[3 * r + l] * T[3 * l + c];
            tmp[3 * r + c] = s;
          }
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) {
            double s = 0;
            for (int l = 0; l < 3; ++l) s += tmp[3 * r + l] * Cy[3 * c + l];
            KX[3 * r + c] = s;
          }
        double lS[3], lD[3];
        for (int ch = 0; ch < 3; ++ch) oracle_eigen(n, ch, &lS[ch], nullptr, nullptr, &lD[ch]);
        for (int e = 0; e < 9; ++e) {
          KS[e] += lS[0] / vsh_norm2(n, 0) * KV[e];
          KD[e] += lD[0] / vsh_norm2(n, 0) * KV[e];
          if (n >= 1) {
            KS[e] += lS[1] / vsh_norm2(n, 1) * KW[e] + lS[2] / vsh_norm2(n, 2) * KX[e];
            KD[e] += lD[1] / vsh_norm2(n, 1) * KW[e] + lD[2] / vsh_norm2(n, 2) * KX[e];
          }
        }
      }
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          if (f) acc[r] += wh[k] * KS[3 * r + c] * (a / mu) * f[3 * k + c];
          if (q) acc[r] += wh[k] * KD[3 * r + c] * q[3 * k + c];
        }
    }
    for (int c = 0; c < 3; ++c) u[3 * i + c] = acc[c];
  }
  return 0;
}

extern "C" int oracle_num_threads(void) { return omp_get_max_threads(); }
extern "C" void oracle_set_num_threads(int n) { if (n > 0) omp_set_num_threads(n); }

// ============================================================ NEXT-1 (near)
// Near-singular correction (PAPER §4.1 "Singular and near-singular
// integrands"; composite scheme §4.3).  Sphere pairs that
// fail the well-separation test of eq 4.5,
//     dist(G_src, G_trg) >= eta max(diam(G_src), diam(G_trg)),
// with dist = |c_s - c_t| - a_s - a_t and diam = 2a, are not evaluated with
// the smooth rule: the source density is expanded in VSH of degree <= p
// (eq 4.6, the discrete projection of reading R9) and the exterior formulas
// of eqs 3.6-3.11 (sign reading R1) are evaluated at the targets (eq 4.7).

// VSH coefficients of one sphere: alpha[(n*n+n+m)*3 + ch] for the density
// g_k (node order of the sphere), alpha = (1/||Z_n||^2) sum_k w^_k g_k . conj Z.
static void project_sphere(int p, const double* g, std::vector<cplx>& alpha) {
  const int nphi = 2 * p + 2, nsn = (p + 1) * nphi, nlm = (p + 1) * (p + 1);
  std::vector<double> t(p + 1), lam(p + 1);
  oracle_gl_rule(p, t.data(), lam.data());
  alpha.assign((size_t)nlm * 3, cplx(0.0, 0.0));
  for (int j = 0; j <= p; ++j)
    for (int k = 0; k < nphi; ++k) {
      const int kk = j * nphi + k;
      const double wk = lam[j] * 2.0 * PI / nphi;
      const double th = std::acos(t[j]), ph = 2.0 * PI * k / nphi;
      for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m) {
          cplx z[9];
          vsh_cart(n, m, th, ph, z);
          for (int ch = 0; ch < 3; ++ch) {
            if (n == 0 && ch > 0) continue;
            cplx acc(0.0, 0.0);
            for (int c = 0; c < 3; ++c) acc += g[3 * kk + c] * std::conj(z[3 * ch + c]);
            alpha[(size_t)(n * n + n + m) * 3 + ch] += wk * acc;
          }
        }
    }
  for (int n = 0; n <= p; ++n)
    for (int m = -n; m <= n; ++m)
      for (int ch = 0; ch < 3; ++ch) alpha[(size_t)(n * n + n + m) * 3 + ch] /= (n == 0 && ch > 0) ? 1.0 : vsh_norm2(n, ch);
  (void)nsn;
}

// Exterior field (r >= 1, unit sphere) of a unit-coefficient density Z_n^m,
// channel ch, for S (kind 0) or D (kind 1): eqs 3.6-3.8 / 3.9-3.11.
// Zv, Zw, Zx: V_n^m, W_n^m, X_n^m at the target's angles (complex Cartesian).
static void exterior_unit(int kind, int ch, int n, double r, const cplx* Zv, const cplx* Zw,
                          const cplx* Zx, cplx out[3]) {
  const double a = 2.0 * n + 1.0;
  for (int c = 0; c < 3; ++c) out[c] = 0.0;
  if (kind == 0) {
    if (ch == 0) {
      for (int c = 0; c < 3; ++c) out[c] = n / (a * (2.0 * n + 3.0)) * Zv[c] * std::pow(r, -n - 2.0);
    } else if (ch == 1) {
      for (int c = 0; c < 3; ++c)
        out[c] = (n + 1.0) / (a * (2.0 * n - 1.0)) * Zw[c] * std::pow(r, -(double)n) +
                 n / (4.0 * n + 2.0) * Zv[c] * (std::pow(r, -n - 2.0) - std::pow(r, -(double)n));
    } else {
      for (int c = 0; c < 3; ++c) out[c] = 1.0 / a * Zx[c] * std::pow(r, -n - 1.0);
    }
  } else {
    if (ch == 0) {
      for (int c = 0; c < 3; ++c)
        out[c] = (2.0 * n * n + 4.0 * n + 3.0) / (a * (2.0 * n + 3.0)) * Zv[c] * std::pow(r, -n - 2.0);
    } else if (ch == 1) {
      for (int c = 0; c < 3; ++c)
        out[c] = 2.0 * (n + 1.0) * (n - 1.0) / (a * (2.0 * n - 1.0)) * Zw[c] * std::pow(r, -(double)n) +
                 2.0 * n * (n - 1.0) / (4.0 * n + 2.0) * Zv[c] * (std::pow(r, -n - 2.0) - std::pow(r, -(double)n));
    } else {
      for (int c = 0; c < 3; ++c) out[c] = (n - 1.0) / a * Zx[c] * std::pow(r, -n - 1.0);
    }
  }
}

// Field of sphere (c, a) carrying densities f (S) and q (D) [nsn][3] at an
// exterior point x: u = sum_{n<=p,m,Z} (a/mu) alpha_Z[f] S[Z](r) + alpha_Z[q] D[Z](r)
// with r = |x - c|/a (radius/viscosity scalings R5, R6).
static void exterior_eval(int p, const double* c, double a, double mu,
                          const std::vector<cplx>* af, const std::vector<cplx>* aq,
                          const double* x, double u[3]) {
  const double rv[3] = {(x[0] - c[0]) / a, (x[1] - c[1]) / a, (x[2] - c[2]) / a};
  const double r = std::sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
  const double th = std::acos(rv[2] / r), ph = std::atan2(rv[1], rv[0]);
  cplx acc[3] = {0.0, 0.0, 0.0};
  for (int n = 0; n <= p; ++n)
    for (int m = -n; m <= n; ++m) {
      cplx z[9];
      vsh_cart(n, m, th, ph, z);
      for (int ch = 0; ch < 3; ++ch) {
        if (n == 0 && ch > 0) continue;
        const size_t ix = (size_t)(n * n + n + m) * 3 + ch;
        cplx e[3];
        if (af) {
          exterior_unit(0, ch, n, r, z, z + 3, z + 6, e);
          for (int k = 0; k < 3; ++k) acc[k] += (a / mu) * (*af)[ix] * e[k];
        }
        if (aq) {
          exterior_unit(1, ch, n, r, z, z + 3, z + 6, e);
          for (int k = 0; k < 3; ++k) acc[k] += (*aq)[ix] * e[k];
        }
      }
    }
  for (int k = 0; k < 3; ++k) u[k] = acc[k].real();
}

// Velocity of the spectral (exact) layer potentials of ONE sphere at m
// exterior targets: f_s, q_s are that sphere's nodal densities [nsn][3] (either
// may be NULL).  Used by the near correction and pinned on its own.
extern "C" int oracle_exterior_eval(int p, const double* c, double a, double mu, const double* f_s,
                                    const double* q_s, const double* targets, int64_t m, double* u) {
  if (p < 1 || !(a > 0) || !(mu > 0) || !c || (m > 0 && (!targets || !u))) return 1;
  std::vector<cplx> af, aq;
  if (f_s) project_sphere(p, f_s, af);
  if (q_s) project_sphere(p, q_s, aq);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < m; ++t)
    exterior_eval(p, c, a, mu, f_s ? &af : nullptr, q_s ? &aq : nullptr, targets + 3 * t, u + 3 * t);
  return 0;
}

// eq 4.5: true when spheres s and t are NOT well separated (and s != t).
extern "C" int oracle_is_near(const double* cs, double as, const double* ct, double at, double eta) {
  const double d = std::sqrt((cs[0] - ct[0]) * (cs[0] - ct[0]) + (cs[1] - ct[1]) * (cs[1] - ct[1]) +
                             (cs[2] - ct[2]) * (cs[2] - ct[2])) - as - at;
  return d < eta * std::max(2.0 * as, 2.0 * at) ? 1 : 0;
}

// Near correction at the subset nodes tidx: du_i = sum over near spheres s of
// [ exterior_eval of sphere s at x_i  -  smooth-rule sum over s's nodes at x_i ].
// The corrected apply is oracle_far + oracle_self + oracle_near.
extern "C" int oracle_near(const double* centres, const double* radii, int64_t ns, int p, double mu,
                           const double* f, const double* q, double eta, const int64_t* tidx,
                           int64_t nt, double* du) {
  if (ns < 1 || p < 1 || !(mu > 0) || !(eta >= 0) || !du || !tidx) return 1;
  Geometry G(centres, radii, ns, p);
  const int nsn = G.nsn;
  // spheres whose expansion is needed
  std::vector<char> need(ns, 0);
  for (int64_t a = 0; a < nt; ++a) {
    const int64_t t = tidx[a] / nsn;
    for (int64_t s = 0; s < ns; ++s)
      if (s != t && oracle_is_near(centres + 3 * s, radii[s], centres + 3 * t, radii[t], eta)) need[s] = 1;
  }
  std::vector<std::vector<cplx>> AF(ns), AQ(ns);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < ns; ++s) {
    if (!need[s]) continue;
    if (f) project_sphere(p, f + 3 * s * nsn, AF[s]);
    if (q) project_sphere(p, q + 3 * s * nsn, AQ[s]);
  }
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t a = 0; a < nt; ++a) {
    const int64_t i = tidx[a], t = i / nsn;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t s = 0; s < ns; ++s) {
      if (s == t || !oracle_is_near(centres + 3 * s, radii[s], centres + 3 * t, radii[t], eta)) continue;
      double ue[3];
      exterior_eval(p, centres + 3 * s, radii[s], mu, f ? &AF[s] : nullptr, q ? &AQ[s] : nullptr,
                    &G.x[3 * i], ue);
      Neumaier sm[3];
      for (int64_t k = s * nsn; k < (s + 1) * nsn; ++k) {
        double v[3];
        pair_terms(&G.x[3 * i], &G.x[3 * k], &G.n[3 * k], G.w[k], f ? f + 3 * k : nullptr,
                   q ? q + 3 * k : nullptr, mu, v, nullptr);
        for (int c = 0; c < 3; ++c) sm[c].add(v[c]);
      }
      for (int c = 0; c < 3; ++c) acc[c] += ue[c] - sm[c].get();
    }
    for (int c = 0; c < 3; ++c) du[3 * a + c] = acc[c];
  }
  return 0;
}

// ============================================================ NEXT-3 (K)
// Traction of the single layer (eq 2.22):
//   K[s](x)_i = int T_ijk(x,y) n_k(x) s_j(y) dS_y,
// with the TARGET normal n(x).  The sign of T in eq 2.20 is ambiguous (reading
// R1 fixed it for D with the source normal); for K the reading is
//   K[s](x) = -(3/(4 pi)) int ((x-y).n(x)) ((x-y).s(y)) (x-y) / |x-y|^5 dS_y,
// i.e. the L2 adjoint of D, which is what P:219 ("the spectra of K+ matches
// that of D- and K- that of D+") requires: K_pv = D_pv on the sphere
// (reading R21, pinned by brute-force quadrature and the translating-sphere
// traction in tests/test_oracle_traction.py).
//
// One source node k of the smooth-rule K sum at point x with normal nx
// (eq 2.22 under the node rule of eq 4.4, reading R21):
//   out = -(3/(4 pi)) w_k ((x-y_k).nx) ((x-y_k).sigma_k) (x-y_k) / |x-y_k|^5.
static inline void k_pair(const double* x, const double* nx, const double* y, const double* sg,
                          double wk, double out[3]) {
  const double rho[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
  const double r2 = rho[0] * rho[0] + rho[1] * rho[1] + rho[2] * rho[2];
  const double r5 = r2 * r2 * std::sqrt(r2);
  const double rn = rho[0] * nx[0] + rho[1] * nx[1] + rho[2] * nx[2];
  const double rs = rho[0] * sg[0] + rho[1] * sg[1] + rho[2] * sg[2];
  const double cK = -3.0 * wk / (4.0 * PI);
  for (int c = 0; c < 3; ++c) out[c] = cK * rn * rs * rho[c] / r5;
}

// Far field of K at the subset nodes tidx (own sphere excluded, Neumaier).
extern "C" int oracle_far_K(const double* centres, const double* radii, int64_t ns, int p,
                            const double* sigma, const int64_t* tidx, int64_t nt, double* u) {
  if (ns < 1 || p < 1 || !sigma || !u || !tidx) return 1;
  Geometry G(centres, radii, ns, p);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t i = tidx[t];
    const int64_t si = i / G.nsn;
    const double* x = &G.x[3 * i];
    const double* nx = &G.n[3 * i];
    Neumaier acc[3];
    for (int64_t k = 0; k < G.N; ++k) {
      if (k / G.nsn == si) continue;
      double v[3];
      k_pair(x, nx, &G.x[3 * k], sigma + 3 * k, G.w[k], v);
      for (int c = 0; c < 3; ++c) acc[c].add(v[c]);
    }
    for (int c = 0; c < 3; ++c) u[3 * t + c] = acc[c].get();
  }
  return 0;
}

// Off-surface version with an explicit target normal (used by the pins).
extern "C" int oracle_K_at(const double* centres, const double* radii, int64_t ns, int p,
                           const double* sigma, const double* targets, const double* normals,
                           int64_t m, double* u) {
  if (ns < 1 || p < 1 || !sigma || (m > 0 && (!targets || !normals || !u))) return 1;
  Geometry G(centres, radii, ns, p);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < m; ++t) {
    const double* x = targets + 3 * t;
    const double* nx = normals + 3 * t;
    Neumaier acc[3];
    for (int64_t k = 0; k < G.N; ++k) {
      double v[3];
      k_pair(x, nx, &G.x[3 * k], sigma + 3 * k, G.w[k], v);
      for (int c = 0; c < 3; ++c) acc[c].add(v[c]);
    }
    for (int c = 0; c < 3; ++c) u[3 * t + c] = acc[c].get();
  }
  return 0;
}

// ----------------------------------------------- NEXT-3: near correction for K
// Traction of the exterior single-layer flow of ONE sphere: the
// field is the expansion of eqs 3.6-3.8 (eq 3.17: each term u = g(r) Z with Z
// in {V, W, X}); PAPER eq 3.18 gives the traction of one term,
//   (grad u + grad u^T - pI) n = g'(r) ((e_r.n) Z + (Z.n) e_r)
//                              + (g(r)/r) (grad_g Z + grad_g Z^T) n - q(r) Y n,
// with grad_g Z the surface gradient of Z's Cartesian components on the unit
// sphere (hence the 1/r at radius r) and p = q(r) Y_n^m the pressure of the
// S[W_n^m] term (n Y r^{-n-1}).  Eq 3.18 prints "+ q Y n"; the
// Newtonian stress -pI gives "- q Y n" (reading R24).  Unit sphere, mu = 1:
// K is a- and mu-free (the a/mu of S and the 1/a of grad cancel).  The
// surface derivatives are written out in spherical coordinates with the
// Legendre equation for Y_thth, so targets on the source's polar axis
// (sin theta = 0) are excluded from this routine (the tests avoid them).
static void exterior_traction(int p, const double* c, double a, const std::vector<cplx>& al,
                              const double* x, const double* nv, double out[3]) {
  const double rv[3] = {(x[0] - c[0]) / a, (x[1] - c[1]) / a, (x[2] - c[2]) / a};
  const double r = std::sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
  const double th = std::acos(rv[2] / r), ph = std::atan2(rv[1], rv[0]);
  const double st = std::sin(th), ct = std::cos(th), sp = std::sin(ph), cp = std::cos(ph);
  const double er[3] = {st * cp, st * sp, ct}, et[3] = {ct * cp, ct * sp, -st}, ep[3] = {-sp, cp, 0.0};
  const double nr = er[0] * nv[0] + er[1] * nv[1] + er[2] * nv[2];
  const double nt = et[0] * nv[0] + et[1] * nv[1] + et[2] * nv[2];
  const double np = ep[0] * nv[0] + ep[1] * nv[1] + ep[2] * nv[2];
  const double cot = ct / st;
  const cplx I(0.0, 1.0);
  cplx acc[3] = {0.0, 0.0, 0.0};
  // one term g Z (value Z, theta-derivative Zt, (1/sin th) phi-derivative Zp)
  auto term = [&](cplx coef, double g, double gp, const cplx* Z, const cplx* Zt, const cplx* Zp) {
    cplx Zn = 0.0, Ztn = 0.0, Zpn = 0.0;
    for (int k = 0; k < 3; ++k) {
      Zn += Z[k] * nv[k];
      Ztn += Zt[k] * nv[k];
      Zpn += Zp[k] * nv[k];
    }
    for (int k = 0; k < 3; ++k)
      acc[k] += coef * (gp * (nr * Z[k] + Zn * er[k]) +
                        (g / r) * (Zt[k] * nt + Zp[k] * np + et[k] * Ztn + ep[k] * Zpn));
  };
  for (int n = 1; n <= p; ++n)
    for (int m = -n; m <= n; ++m) {
      cplx Y, A, B;
      ynm_all(n, m, th, ph, &Y, &A, &B);  // Y, Y_th, (1/st) Y_ph
      const double mm = (double)m;
      const cplx At = -cot * A - (n * (n + 1.0) - mm * mm / (st * st)) * Y;  // Legendre eq.
      const cplx Bt = (I * mm / st) * (A - cot * Y);
      const cplx Ap = (I * mm / st) * A, Bp = (I * mm / st) * B;
      cplx V[3], Vt[3], Vp[3], W[3], Wt[3], Wp[3], X[3], Xt[3], Xp[3];
      for (int k = 0; k < 3; ++k) {
        const cplx Yr = Y * er[k], Yrt = A * er[k] + Y * et[k], Yrp = B * er[k] + Y * ep[k];
        const cplx G = A * et[k] + B * ep[k];
        const cplx Gt = At * et[k] - A * er[k] + Bt * ep[k];
        const cplx Gp = Ap * et[k] + A * cot * ep[k] + Bp * ep[k] - B * (er[k] + cot * et[k]);
        V[k] = G - (n + 1.0) * Yr;  Vt[k] = Gt - (n + 1.0) * Yrt;  Vp[k] = Gp - (n + 1.0) * Yrp;
        W[k] = G + (double)n * Yr;  Wt[k] = Gt + (double)n * Yrt;  Wp[k] = Gp + (double)n * Yrp;
        X[k] = A * ep[k] - B * et[k];
        Xt[k] = At * ep[k] - Bt * et[k] + B * er[k];
        Xp[k] = Ap * ep[k] - A * (er[k] + cot * et[k]) - Bp * et[k] - B * cot * ep[k];
      }
      const size_t ix = (size_t)(n * n + n + m) * 3;
      const double d = 2.0 * n + 1.0;
      const double rn2 = std::pow(r, -n - 2.0), rn = std::pow(r, -(double)n), rn1 = std::pow(r, -n - 1.0);
      // S[V] = n/(d(2n+3)) V r^{-n-2}                                  (eq 3.6)
      const double cV = n / (d * (2.0 * n + 3.0));
      term(al[ix], cV * rn2, -(n + 2.0) * cV * rn2 / r, V, Vt, Vp);
      // S[W] = (n+1)/(d(2n-1)) W r^{-n} + n/(4n+2) V (r^{-n-2} - r^{-n}) (eq 3.7)
      const double cW = (n + 1.0) / (d * (2.0 * n - 1.0)), cWV = n / (4.0 * n + 2.0);
      term(al[ix + 1], cW * rn, -n * cW * rn / r, W, Wt, Wp);
      term(al[ix + 1], cWV * (rn2 - rn), cWV * (-(n + 2.0) * rn2 + n * rn) / r, V, Vt, Vp);
      // S[X] = 1/d X r^{-n-1}                                          (eq 3.8)
      term(al[ix + 2], rn1 / d, -(n + 1.0) * rn1 / (d * r), X, Xt, Xp);
      // pressure of S[W]: n Y r^{-n-1}, traction -p n
      const cplx pq = al[ix + 1] * (double)n * Y * rn1;
      for (int k = 0; k < 3; ++k) acc[k] -= pq * nv[k];
    }
  for (int k = 0; k < 3; ++k) out[k] = acc[k].real();
}

extern "C" int oracle_exterior_traction(int p, const double* c, double a, const double* sigma_s,
                                        const double* targets, const double* normals, int64_t m,
                                        double* t) {
  if (p < 1 || !(a > 0) || !c || !sigma_s || (m > 0 && (!targets || !normals || !t))) return 1;
  std::vector<cplx> al;
  project_sphere(p, sigma_s, al);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < m; ++i) exterior_traction(p, c, a, al, targets + 3 * i, normals + 3 * i, t + 3 * i);
  return 0;
}

// Near correction of K at the subset nodes tidx (eq 4.5 partition, as
// oracle_near): dK_i = sum over near spheres s of [exterior traction of s at
// x_i with normal n_i  -  smooth-rule K sum over s's nodes].
extern "C" int oracle_near_K(const double* centres, const double* radii, int64_t ns, int p,
                             const double* sigma, double eta, const int64_t* tidx, int64_t nt,
                             double* du) {
  if (ns < 1 || p < 1 || !sigma || !(eta >= 0) || !du || !tidx) return 1;
  Geometry G(centres, radii, ns, p);
  const int nsn = G.nsn;
  std::vector<char> need(ns, 0);
  for (int64_t q = 0; q < nt; ++q) {
    const int64_t t = tidx[q] / nsn;
    for (int64_t s = 0; s < ns; ++s)
      if (s != t && oracle_is_near(centres + 3 * s, radii[s], centres + 3 * t, radii[t], eta)) need[s] = 1;
  }
  std::vector<std::vector<cplx>> AL(ns);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < ns; ++s)
    if (need[s]) project_sphere(p, sigma + 3 * s * nsn, AL[s]);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t q = 0; q < nt; ++q) {
    const int64_t i = tidx[q], t = i / nsn;
    const double* x = &G.x[3 * i];
    const double* nx = &G.n[3 * i];
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t s = 0; s < ns; ++s) {
      if (s == t || !oracle_is_near(centres + 3 * s, radii[s], centres + 3 * t, radii[t], eta)) continue;
      double te[3];
      exterior_traction(p, centres + 3 * s, radii[s], AL[s], x, nx, te);
      Neumaier sm[3];
      for (int64_t k = s * nsn; k < (s + 1) * nsn; ++k) {
        double v[3];
        k_pair(x, nx, &G.x[3 * k], sigma + 3 * k, G.w[k], v);
        for (int e = 0; e < 3; ++e) sm[e].add(v[e]);
      }
      for (int e = 0; e < 3; ++e) acc[e] += te[e] - sm[e].get();
    }
    for (int e = 0; e < 3; ++e) du[3 * q + e] = acc[e];
  }
  return 0;
}

// Near correction of K at arbitrary targets with given normals: target x and
// sphere s are near when 0 <= |x - c_s| - a_s < eta 2 a_s (as
// oracle_near_offsurface; exterior targets only).  dt = sum over near s of
// [exterior traction of s  -  smooth-rule K sum over s's nodes].  The
// corrected evaluator is oracle_K_at + this.
extern "C" int oracle_near_K_offsurface(const double* centres, const double* radii, int64_t ns,
                                        int p, const double* sigma, double eta,
                                        const double* targets, const double* normals, int64_t m,
                                        double* dt) {
  if (ns < 1 || p < 1 || !sigma || !(eta >= 0) || (m > 0 && (!targets || !normals || !dt))) return 1;
  Geometry G(centres, radii, ns, p);
  const int nsn = G.nsn;
  auto near_pt = [&](int64_t s, const double* x) {
    const double dx = x[0] - centres[3 * s], dy = x[1] - centres[3 * s + 1], dz = x[2] - centres[3 * s + 2];
    const double d = std::sqrt(dx * dx + dy * dy + dz * dz) - radii[s];
    return d >= 0.0 && d < eta * 2.0 * radii[s];
  };
  std::vector<char> need(ns, 0);
  for (int64_t t = 0; t < m; ++t)
    for (int64_t s = 0; s < ns; ++s)
      if (near_pt(s, targets + 3 * t)) need[s] = 1;
  std::vector<std::vector<cplx>> AL(ns);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < ns; ++s)
    if (need[s]) project_sphere(p, sigma + 3 * s * nsn, AL[s]);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < m; ++t) {
    const double* x = targets + 3 * t;
    const double* nx = normals + 3 * t;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t s = 0; s < ns; ++s) {
      if (!near_pt(s, x)) continue;
      double te[3];
      exterior_traction(p, centres + 3 * s, radii[s], AL[s], x, nx, te);
      Neumaier sm[3];
      for (int64_t k = s * nsn; k < (s + 1) * nsn; ++k) {
        double v[3];
        k_pair(x, nx, &G.x[3 * k], sigma + 3 * k, G.w[k], v);
        for (int e = 0; e < 3; ++e) sm[e].add(v[e]);
      }
      for (int e = 0; e < 3; ++e) acc[e] += te[e] - sm[e].get();
    }
    for (int e = 0; e < 3; ++e) dt[3 * t + e] = acc[e];
  }
  return 0;
}

// Completion operator of the mobility BIE (eq 5.8):
//   L_k[mu](x) = int_{Gamma_k} mu dGamma
//              + (int_{Gamma_k} (y - x_c) x mu(y) dGamma) x (x - x_c),
// "added ... to eliminate the 6n dimensional nullspace of 1/2 I + K".  The
// subscripts of eq 5.8 are garbled (x_i^c next to Gamma_k); reading R22: L_k
// acts on the targets of its own body only (x in Gamma_k, x_c = x_k^c), so
// sum_k L_k is block diagonal with one rank-6 block per sphere -- the only
// reading that removes a 6n-dimensional (per-body rigid motion) nullspace
// with per-body moments.  Integrals by the node rule (w of O-2), Neumaier.
extern "C" int oracle_completion(const double* centres, const double* radii, int64_t ns, int p,
                                 const double* mu, double* u) {
  if (ns < 1 || p < 1 || !mu || !u) return 1;
  Geometry G(centres, radii, ns, p);
  for (int64_t s = 0; s < ns; ++s) {
    const double* c = centres + 3 * s;
    Neumaier F[3], T[3];
    for (int64_t k = s * G.nsn; k < (s + 1) * G.nsn; ++k) {
      const double d[3] = {G.x[3 * k] - c[0], G.x[3 * k + 1] - c[1], G.x[3 * k + 2] - c[2]};
      const double* m = mu + 3 * k;
      const double cr[3] = {d[1] * m[2] - d[2] * m[1], d[2] * m[0] - d[0] * m[2],
                            d[0] * m[1] - d[1] * m[0]};
      for (int e = 0; e < 3; ++e) {
        F[e].add(G.w[k] * m[e]);
        T[e].add(G.w[k] * cr[e]);
      }
    }
    const double f[3] = {F[0].get(), F[1].get(), F[2].get()};
    const double t[3] = {T[0].get(), T[1].get(), T[2].get()};
    for (int64_t k = s * G.nsn; k < (s + 1) * G.nsn; ++k) {
      const double d[3] = {G.x[3 * k] - c[0], G.x[3 * k + 1] - c[1], G.x[3 * k + 2] - c[2]};
      u[3 * k + 0] = f[0] + (t[1] * d[2] - t[2] * d[1]);
      u[3 * k + 1] = f[1] + (t[2] * d[0] - t[0] * d[2]);
      u[3 * k + 2] = f[2] + (t[0] * d[1] - t[1] * d[0]);
    }
  }
  return 0;
}

// ============================================ NEXT-1 for off-surface targets
// Exterior pressure of a sphere's expansion: only the W_n channels carry
// pressure outside (P:189 for S: n Y_n r^{-n-1}; the D value 2n(n-1) Y_n
// r^{-n-1} replaces the inconsistent P:215 per reading R12).  Scalings
// (R5, R6): S pressure is a- and mu-free for the unscaled density, D pressure
// carries mu/a.  With alpha_f = projections of (a/mu) f:
//   p = sum_{n,m} (mu/a) [ n alpha_W[(a/mu) f] + 2n(n-1) alpha_W[q] ] Y_n^m r^{-n-1}.
static double exterior_pressure(int p, const double* c, double a, double mu,
                                const std::vector<cplx>* af, const std::vector<cplx>* aq,
                                const double* x) {
  const double rv[3] = {(x[0] - c[0]) / a, (x[1] - c[1]) / a, (x[2] - c[2]) / a};
  const double r = std::sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
  const double th = std::acos(rv[2] / r), ph = std::atan2(rv[1], rv[0]);
  cplx acc = 0.0;
  for (int n = 1; n <= p; ++n)
    for (int m = -n; m <= n; ++m) {
      cplx Y, dY, dYp;
      ynm_all(n, m, th, ph, &Y, &dY, &dYp);
      const size_t ix = (size_t)(n * n + n + m) * 3 + 1;  // W channel
      cplx coef = 0.0;
      if (af) coef += (double)n * (*af)[ix];
      if (aq) coef += 2.0 * n * (n - 1.0) * (*aq)[ix];
      acc += (mu / a) * coef * Y * std::pow(r, -n - 1.0);
    }
  return acc.real();
}

extern "C" int oracle_exterior_pressure(int p, const double* c, double a, double mu,
                                        const double* f_s, const double* q_s,
                                        const double* targets, int64_t m, double* pr) {
  if (p < 1 || !(a > 0) || !(mu > 0) || !c || (m > 0 && (!targets || !pr))) return 1;
  std::vector<cplx> af, aq;
  if (f_s) {  // projections of (a/mu) f, as in the velocity path
    std::vector<double> g(3 * (p + 1) * (2 * p + 2));
    for (size_t k = 0; k < g.size(); ++k) g[k] = (a / mu) * f_s[k];
    project_sphere(p, g.data(), af);
  }
  if (q_s) project_sphere(p, q_s, aq);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < m; ++t)
    pr[t] = exterior_pressure(p, c, a, mu, f_s ? &af : nullptr, q_s ? &aq : nullptr, targets + 3 * t);
  return 0;
}

// Near correction at arbitrary targets: target x and sphere s are near when
// the point-to-surface distance |x - c_s| - a_s < eta * 2 a_s (eq 4.5 with
// the target as a point: SPEC's "point-to-surface distance for target
// batches").  du, dp = sum over near s of [exterior - smooth] (velocity and
// pressure).  The corrected evaluator is oracle_offsurface + this.
extern "C" int oracle_near_offsurface(const double* centres, const double* radii, int64_t ns, int p,
                                      double mu, const double* f, const double* q, double eta,
                                      const double* targets, int64_t m, double* du, double* dp) {
  if (ns < 1 || p < 1 || !(mu > 0) || !(eta >= 0) || (m > 0 && (!targets || !du))) return 1;
  Geometry G(centres, radii, ns, p);
  const int nsn = G.nsn;
  auto near_pt = [&](int64_t s, const double* x) {
    const double dx = x[0] - centres[3 * s], dy = x[1] - centres[3 * s + 1], dz = x[2] - centres[3 * s + 2];
    const double d = std::sqrt(dx * dx + dy * dy + dz * dz) - radii[s];
    return d >= 0.0 && d < eta * 2.0 * radii[s];  // exterior targets only (eqs 3.6-3.11 r >= 1)
  };
  std::vector<char> need(ns, 0);
  for (int64_t t = 0; t < m; ++t)
    for (int64_t s = 0; s < ns; ++s)
      if (near_pt(s, targets + 3 * t)) need[s] = 1;
  std::vector<std::vector<cplx>> AF(ns), AQ(ns);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < ns; ++s) {
    if (!need[s]) continue;
    if (f) {
      std::vector<double> g(3 * nsn);
      for (int k = 0; k < 3 * nsn; ++k) g[k] = (radii[s] / mu) * f[3 * s * nsn + k];
      project_sphere(p, g.data(), AF[s]);
    }
    if (q) project_sphere(p, q + 3 * s * nsn, AQ[s]);
  }
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < m; ++t) {
    const double* x = targets + 3 * t;
    double acc[3] = {0.0, 0.0, 0.0}, pacc = 0.0;
    for (int64_t s = 0; s < ns; ++s) {
      if (!near_pt(s, x)) continue;
      double ue[3];
      // exterior_eval scales alpha_f by a/mu itself; pass unscaled projections
      std::vector<cplx> afu;
      if (f) {
        afu = AF[s];
        for (auto& v : afu) v *= mu / radii[s];
      }
      exterior_eval(p, centres + 3 * s, radii[s], mu, f ? &afu : nullptr, q ? &AQ[s] : nullptr, x, ue);
      const double pe = exterior_pressure(p, centres + 3 * s, radii[s], mu, f ? &AF[s] : nullptr,
                                          q ? &AQ[s] : nullptr, x);
      Neumaier sm[3], sp;
      for (int64_t k = s * nsn; k < (s + 1) * nsn; ++k) {
        double v[3], pv;
        pair_terms(x, &G.x[3 * k], &G.n[3 * k], G.w[k], f ? f + 3 * k : nullptr,
                   q ? q + 3 * k : nullptr, mu, v, &pv);
        for (int c = 0; c < 3; ++c) sm[c].add(v[c]);
        sp.add(pv);
      }
      for (int c = 0; c < 3; ++c) acc[c] += ue[c] - sm[c].get();
      pacc += pe - sp.get();
    }
    for (int c = 0; c < 3; ++c) du[3 * t + c] = acc[c];
    if (dp) dp[t] = pacc;
  }
  return 0;
}

// ============================================================ NEXT-4 (§4.2)
// FFT-accelerated near evaluation with rotations (PAPER §4.2 "General case",
// Fig 2), followed stage by stage and evaluated plainly -- no
// Wigner matrices, no FFT: every stage is a direct evaluation of a degree-<=p
// VSH expansion or a direct quadrature projection (eq 4.4 on the grid of eq
// 4.2), so a reader can check each against the paper:
//   (0) "Input: spherical harmonic coefficients of the density on the
//       original grid": project_sphere of the source's f and q (eq 4.6).
//   (1) "Density rotation: rotate the computational grid so that the north
//       pole points in the direction of target center C ... equivalent
//       coefficients for the rotated grid": Q = Rz(alpha) Ry(beta) with
//       Q e_z = d = (c_t - c_s)/|c_t - c_s| (Euler angles (alpha, beta, 0),
//       reading R25); the rotated-frame density sigma^R(y) = Q^T sigma(Q y) is
//       sampled on the source grid and projected (exact: it has degree <= p).
//   (2) "Fast evaluation at translated grid": the exterior formulas of eqs
//       3.6-3.11 (exterior_eval) of sigma^R at the target grid of the rotated
//       frame, x^R_jk = |c_t - c_s| e_z + a_t n_jk (discs of constant r, theta).
//   (3) "Rotate function samples": forward transform of those samples on the
//       target grid (project_sphere, the discrete projection of reading R9),
//       rotated back and evaluated at the original target nodes:
//       u(x_i) = Q u^R(Q^T n_i), with u^R the target-centred expansion.
// The result is the degree-p re-expansion of the exact near field on the
// target sphere (it equals the exterior field when that is band-limited and
// converges spectrally to it as p grows); P:392's delayed evaluation (add the
// neighbours' coefficients to the target's own, then one inverse transform)
// changes only the rounding order, not this value.

// Q = Rz(alpha) Ry(beta), Q e_z = d (row-major 3x3).
static void next4_rotation(const double* cs, const double* ct, double Q[9]) {
  double d[3] = {ct[0] - cs[0], ct[1] - cs[1], ct[2] - cs[2]};
  const double L = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  for (int k = 0; k < 3; ++k) d[k] /= L;
  const double beta = std::acos(std::max(-1.0, std::min(1.0, d[2])));
  const double alpha = std::atan2(d[1], d[0]);
  const double ca = std::cos(alpha), sa = std::sin(alpha), cb = std::cos(beta), sb = std::sin(beta);
  const double Rz[9] = {ca, -sa, 0.0, sa, ca, 0.0, 0.0, 0.0, 1.0};
  const double Ry[9] = {cb, 0.0, sb, 0.0, 1.0, 0.0, -sb, 0.0, cb};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += Rz[3 * i + k] * Ry[3 * k + j];
      Q[3 * i + j] = s;
    }
}

// Cartesian V, W, X (eqs 2.4-2.6) of degree n, order m at the unit direction
// u, pole-safe: with x = cos th = u_z, s = sin th = |(u_x, u_y)| (never from
// sqrt(1 - x^2)) and Pb = P_n^|m| / s^|m| (a polynomial in x; no
// Condon-Shortley phase, eq 2.1):
//   Pb_m^m = (2m-1)!!, Pb_{m+1}^m = (2m+1) x Pb_m^m,
//   (n-m) Pb_n^m = (2n-1) x Pb_{n-1}^m - (n+m-1) Pb_{n-2}^m   (and d/dx of it),
//   Y = N Pb s^m e^{i m ph},  (1/s) dY/dph = i m N Pb s^{m-1} e^{i m ph},
//   dY/dth = N s^{m-1} (m x Pb - s^2 dPb/dx) e^{i m ph};
// no division by s, so a direction on (or rounding onto) the polar axis is exact.
static void next4_vsh_dir(int n, int m, const double* u, cplx out[9]) {
  const int am = std::abs(m);
  const double x = u[2], s = std::sqrt(u[0] * u[0] + u[1] * u[1]);
  const double ph = std::atan2(u[1], u[0]);
  double pb = 1.0;
  for (int k = 1; k <= am; ++k) pb *= (2.0 * k - 1.0);  // (2m-1)!!
  double p0 = 0.0, p1 = pb, d0 = 0.0, d1 = 0.0;         // Pb_{m-1} = 0
  for (int l = am + 1; l <= n; ++l) {
    const double p2 = ((2.0 * l - 1.0) * x * p1 - (l + am - 1.0) * p0) / (l - am);
    const double d2 = ((2.0 * l - 1.0) * (p1 + x * d1) - (l + am - 1.0) * d0) / (l - am);
    p0 = p1; p1 = p2; d0 = d1; d1 = d2;
  }
  const double sm1 = am >= 1 ? std::pow(s, am - 1) : 0.0;  // s^{m-1} (unused for m = 0)
  const double N = ynm_norm(n, m);
  const cplx e = std::polar(1.0, m * ph);
  const cplx Y = N * p1 * std::pow(s, am) * e;
  cplx dY, dYp;
  if (am == 0) {
    dY = N * (-s * d1) * e;  // d/dth P_n(cos th) = -s P_n'(x)
    dYp = 0.0;
  } else {
    dY = N * sm1 * (am * x * p1 - s * s * d1) * e;
    dYp = cplx(0.0, (double)m) * N * p1 * sm1 * e;
  }
  const double cp = std::cos(ph), sp = std::sin(ph);
  const double er[3] = {s * cp, s * sp, x}, et[3] = {x * cp, x * sp, -s}, ep[3] = {-sp, cp, 0.0};
  for (int c = 0; c < 3; ++c) {
    const cplx grad = dY * et[c] + dYp * ep[c];
    out[c] = grad - (double)(n + 1) * Y * er[c];
    out[3 + c] = grad + (double)n * Y * er[c];
    out[6 + c] = dY * ep[c] - dYp * et[c];
  }
}

// Re sum_{n<=p, m, Z} alpha[(n n + n + m) 3 + ch] Z_nm(u), u a unit direction.
static void next4_expand(int p, const std::vector<cplx>& al, const double* u, double out[3]) {
  cplx acc[3] = {0.0, 0.0, 0.0};
  for (int n = 0; n <= p; ++n)
    for (int m = -n; m <= n; ++m) {
      cplx z[9];
      next4_vsh_dir(n, m, u, z);
      for (int ch = 0; ch < 3; ++ch) {
        if (n == 0 && ch > 0) continue;
        const cplx a = al[(size_t)(n * n + n + m) * 3 + ch];
        for (int k = 0; k < 3; ++k) acc[k] += a * z[3 * ch + k];
      }
    }
  for (int k = 0; k < 3; ++k) out[k] = acc[k].real();
}

// Unit-sphere grid directions n_k of order p (node order of eq 4.2).
static void next4_unit_grid(int p, std::vector<double>& nh) {
  const double c0[3] = {0.0, 0.0, 0.0}, a1 = 1.0;
  const int nsn = (p + 1) * (2 * p + 2);
  std::vector<double> nn(3 * nsn), w(nsn);
  nh.resize(3 * nsn);
  oracle_nodes(c0, &a1, 1, p, nh.data(), nn.data(), w.data());
}

// Stage (1) alone: the rotated-frame density at the source grid nodes,
// gR_k = Q^T g(Q n_k), g being the degree-<=p expansion of the nodal density g.
extern "C" int oracle_next4_rotate_density(int p, const double* Q, const double* g, double* gR) {
  if (p < 1 || !Q || !g || !gR) return 1;
  std::vector<cplx> al;
  project_sphere(p, g, al);
  std::vector<double> nh;
  next4_unit_grid(p, nh);
  const int nsn = (p + 1) * (2 * p + 2);
  for (int k = 0; k < nsn; ++k) {
    double y[3], v[3];
    for (int i = 0; i < 3; ++i) y[i] = Q[3 * i] * nh[3 * k] + Q[3 * i + 1] * nh[3 * k + 1] + Q[3 * i + 2] * nh[3 * k + 2];
    next4_expand(p, al, y, v);
    for (int i = 0; i < 3; ++i) gR[3 * k + i] = Q[i] * v[0] + Q[3 + i] * v[1] + Q[6 + i] * v[2];  // Q^T v
  }
  return 0;
}

// VSH coefficients of a nodal density (project_sphere), exposed for the pins:
// alpha[(n n + n + m) 3 + ch] as (re, im) pairs, (p+1)^2 * 3 complex values.
extern "C" int oracle_vsh_project(int p, const double* g, double* alpha_out) {
  if (p < 1 || !g || !alpha_out) return 1;
  std::vector<cplx> al;
  project_sphere(p, g, al);
  for (size_t i = 0; i < al.size(); ++i) {
    alpha_out[2 * i] = al[i].real();
    alpha_out[2 * i + 1] = al[i].imag();
  }
  return 0;
}

// Re sum alpha Z(u) at arbitrary unit directions (pole-safe), for the pins.
extern "C" int oracle_vsh_expand(int p, const double* alpha_in, const double* dirs, int64_t m, double* out) {
  if (p < 1 || !alpha_in || (m > 0 && (!dirs || !out))) return 1;
  std::vector<cplx> al((size_t)(p + 1) * (p + 1) * 3);
  for (size_t i = 0; i < al.size(); ++i) al[i] = cplx(alpha_in[2 * i], alpha_in[2 * i + 1]);
  for (int64_t t = 0; t < m; ++t) {
    const double* u = dirs + 3 * t;
    const double r = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    const double uh[3] = {u[0] / r, u[1] / r, u[2] / r};
    next4_expand(p, al, uh, out + 3 * t);
  }
  return 0;
}

// Stages (1)-(3) for one (source s, target t) pair: the NEXT-4 estimate of the
// exact exterior field S[f_s] + D[q_s] of sphere s at every node of sphere t
// (out [nsn][3]); f_s or q_s may be NULL.
extern "C" int oracle_next4_pair(int p, const double* cs, double as, const double* ct, double at,
                                 double mu, const double* f_s, const double* q_s, double* out) {
  if (p < 1 || !cs || !ct || !(as > 0) || !(at > 0) || !(mu > 0) || !out) return 1;
  const int nsn = (p + 1) * (2 * p + 2);
  double Q[9];
  next4_rotation(cs, ct, Q);
  // (1) rotated-frame densities on the source grid and their coefficients
  std::vector<double> fR, qR;
  std::vector<cplx> afR, aqR;
  if (f_s) {
    fR.resize(3 * nsn);
    oracle_next4_rotate_density(p, Q, f_s, fR.data());
    project_sphere(p, fR.data(), afR);
  }
  if (q_s) {
    qR.resize(3 * nsn);
    oracle_next4_rotate_density(p, Q, q_s, qR.data());
    project_sphere(p, qR.data(), aqR);
  }
  // (2) exterior field at the target grid of the rotated frame (source at the origin)
  std::vector<double> nh;
  next4_unit_grid(p, nh);
  const double Cz = std::sqrt((ct[0] - cs[0]) * (ct[0] - cs[0]) + (ct[1] - cs[1]) * (ct[1] - cs[1]) +
                              (ct[2] - cs[2]) * (ct[2] - cs[2]));
  const double origin[3] = {0.0, 0.0, 0.0};
  std::vector<double> uR(3 * nsn);
#pragma omp parallel for schedule(dynamic, 8)
  for (int k = 0; k < nsn; ++k) {
    const double x[3] = {at * nh[3 * k], at * nh[3 * k + 1], Cz + at * nh[3 * k + 2]};
    exterior_eval(p, origin, as, mu, f_s ? &afR : nullptr, q_s ? &aqR : nullptr, x, &uR[3 * k]);
  }
  // (3) forward transform on the target grid, rotate back, evaluate at the nodes
  std::vector<cplx> bR;
  project_sphere(p, uR.data(), bR);
  for (int k = 0; k < nsn; ++k) {
    const double* n = &nh[3 * k];
    double y[3], v[3];
    for (int i = 0; i < 3; ++i) y[i] = Q[i] * n[0] + Q[3 + i] * n[1] + Q[6 + i] * n[2];  // Q^T n
    next4_expand(p, bR, y, v);
    for (int i = 0; i < 3; ++i) out[3 * k + i] = Q[3 * i] * v[0] + Q[3 * i + 1] * v[1] + Q[3 * i + 2] * v[2];
  }
  return 0;
}

// NEXT-4 near correction at the subset nodes tidx: as oracle_near, with the
// exact exterior field of each near sphere replaced by its NEXT-4 estimate:
// du_i = sum_{s near t} [ next4_pair(s -> t)(x_i) - smooth_s(x_i) ].
extern "C" int oracle_near4(const double* centres, const double* radii, int64_t ns, int p, double mu,
                            const double* f, const double* q, double eta, const int64_t* tidx,
                            int64_t nt, double* du) {
  if (ns < 1 || p < 1 || !(mu > 0) || !(eta >= 0) || !du || !tidx) return 1;
  Geometry G(centres, radii, ns, p);
  const int nsn = G.nsn;
  // every (target sphere, near source) pair the subset touches, evaluated once
  std::vector<int64_t> tsph;
  for (int64_t a = 0; a < nt; ++a) tsph.push_back(tidx[a] / nsn);
  std::sort(tsph.begin(), tsph.end());
  tsph.erase(std::unique(tsph.begin(), tsph.end()), tsph.end());
  std::vector<std::vector<double>> corr(tsph.size());
  for (size_t ti = 0; ti < tsph.size(); ++ti) {
    const int64_t t = tsph[ti];
    corr[ti].assign(3 * nsn, 0.0);
    for (int64_t s = 0; s < ns; ++s) {
      if (s == t || !oracle_is_near(centres + 3 * s, radii[s], centres + 3 * t, radii[t], eta)) continue;
      std::vector<double> ue(3 * nsn);
      oracle_next4_pair(p, centres + 3 * s, radii[s], centres + 3 * t, radii[t], mu,
                        f ? f + 3 * s * nsn : nullptr, q ? q + 3 * s * nsn : nullptr, ue.data());
#pragma omp parallel for schedule(static)
      for (int kk = 0; kk < nsn; ++kk) {
        const int64_t i = t * nsn + kk;
        Neumaier sm[3];
        for (int64_t k = s * nsn; k < (s + 1) * nsn; ++k) {
          double v[3];
          pair_terms(&G.x[3 * i], &G.x[3 * k], &G.n[3 * k], G.w[k], f ? f + 3 * k : nullptr,
                     q ? q + 3 * k : nullptr, mu, v, nullptr);
          for (int c = 0; c < 3; ++c) sm[c].add(v[c]);
        }
        for (int c = 0; c < 3; ++c) corr[ti][3 * kk + c] += ue[3 * kk + c] - sm[c].get();
      }
    }
  }
  for (int64_t a = 0; a < nt; ++a) {
    const int64_t t = tidx[a] / nsn;
    const size_t ti = std::lower_bound(tsph.begin(), tsph.end(), t) - tsph.begin();
    for (int c = 0; c < 3; ++c) du[3 * a + c] = corr[ti][3 * (tidx[a] - t * nsn) + c];
  }
  return 0;
}
