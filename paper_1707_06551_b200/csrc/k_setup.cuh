// k_setup.cuh -- one-off kernels run by bie_create (row a1 of SURVEY §8(a)):
// Gauss-Legendre rule, unit-grid trig tables, normalised associated Legendre
// tables, the S / D_pv eigenvalue tables, and node/normal/weight generation.
#pragma once
#include "common.cuh"

namespace bie {

// Device-side tables for order p (one allocation, carved by TableLayout).
struct TableLayout {
  int p, nphi, nlm;  // nlm = (p+1)(p+2)/2 (n,m) pairs with m >= 0
  // offsets in doubles
  int64_t t, st, wu, cph, sph, P, dP, mPs, lamS, lamD, rA, rB, rC, cinv, total;
  __host__ __device__ explicit TableLayout(int p_) : p(p_) {
    nphi = 2 * p + 2;
    nlm = (p + 1) * (p + 2) / 2;
    int64_t o = 0;
    t = o;    o += p + 1;
    st = o;   o += p + 1;
    wu = o;   o += p + 1;
    cph = o;  o += nphi;
    sph = o;  o += nphi;
    o = (o + 1) & ~int64_t(1);
    P = o;    o += int64_t(p + 1) * nlm;
    dP = o;   o += int64_t(p + 1) * nlm;
    mPs = o;  o += int64_t(p + 1) * nlm;
    lamS = o; o += 3 * (p + 1);
    lamD = o; o += 3 * (p + 1);
    rA = o;   o += nlm;  // normalised-Legendre recurrence coefficients per (n, m):
    rB = o;   o += nlm;  //   P~_n = rA (t P~_{n-1} - rB P~_{n-2})
    rC = o;   o += nlm;  //   sin(th) dP~_n/dth = n t P~_n - rC P~_{n-1}
    cinv = o; o += 2 * (p + 1);  // per degree n: 1/(n(n+1)) (0 at n = 0), 1/(2n+1)
    total = o;
  }
};

// (n, m) -> column of the Legendre tables; m-major so that, for fixed m, the
// degrees n = m..p are contiguous.
__host__ __device__ __forceinline__ int lm_index(int p, int n, int m) {
  return m * (p + 1) - (m * (m - 1)) / 2 + (n - m);
}

// (p+1)-point Gauss-Legendre rule, nodes ascending (eq 4.2).  One
// thread per node: Tricomi's asymptotic guess, Newton on P_{p+1}.
__global__ void k_gl_rule(int p, double* tab) {
  const TableLayout L(p);
  const int j = threadIdx.x, n = p + 1;
  if (j >= n) return;
  const int i = n - j;  // i-th largest root
  double x = (1.0 - (n - 1.0) / (8.0 * n * n * n)) * cos(kPi * (4.0 * i - 1.0) / (4.0 * n + 2.0));
  double Pn = 0.0, Pm1 = 0.0;
  for (int it = 0; it < 12; ++it) {
    double a = 1.0, b = x;  // P_0, P_1
    for (int k = 2; k <= n; ++k) {
      double c = ((2.0 * k - 1.0) * x * b - (k - 1.0) * a) / k;
      a = b;
      b = c;
    }
    Pn = b;
    Pm1 = a;
    const double dP = n * (x * Pn - Pm1) / (x * x - 1.0);
    x -= Pn / dP;
  }
  double a = 1.0, b = x;
  for (int k = 2; k <= n; ++k) {
    double c = ((2.0 * k - 1.0) * x * b - (k - 1.0) * a) / k;
    a = b;
    b = c;
  }
  const double dP = n * (x * b - a) / (x * x - 1.0);
  tab[L.t + j] = x;
  tab[L.st + j] = sqrt((1.0 - x) * (1.0 + x));
  // unit-sphere weight: lambda_j * 2 pi/(2p+2)   (eq 4.4, reading R4)
  tab[L.wu + j] = 2.0 / ((1.0 - x * x) * dP * dP) * (2.0 * kPi / L.nphi);
}

// Trig tables cos/sin(2 pi k/(2p+2)), normalised associated Legendre
// functions P~_n^m(t_j) = sqrt((2n+1)/(4 pi) (n-m)!/(n+m)!) P_n^m(t_j) without
// the Condon-Shortley phase (eq 2.1), their theta-derivatives, m P~/sin(theta),
// and the eigenvalue tables.  Grid: one thread per (j, m).
__global__ void k_tables(int p, double* tab) {
  const TableLayout L(p);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid < L.nphi) {
    double s, c;
    sincospi(2.0 * tid / L.nphi, &s, &c);
    tab[L.cph + tid] = c;
    tab[L.sph + tid] = s;
  }
  if (tid <= p) {
    // Unit-sphere eigenvalues (Thm 2; App. A.1 of SURVEY: the r -> 1
    // limits of eqs 3.6-3.11, D as principal value = mean of the limits).
    const int n = tid;
    const double a = 2.0 * n + 1.0;
    double* lS = tab + L.lamS + 3 * n;
    double* lD = tab + L.lamD + 3 * n;
    lS[0] = n / (a * (2.0 * n + 3.0));          // V
    lD[0] = 1.5 / (a * (2.0 * n + 3.0));
    lS[1] = n ? (n + 1.0) / (a * (2.0 * n - 1.0)) : 0.0;  // W (W_0 = 0)
    lD[1] = n ? -1.5 / (a * (2.0 * n - 1.0)) : 0.0;
    lS[2] = n ? 1.0 / a : 0.0;                 // X (X_0 = 0)
    lD[2] = n ? -1.5 / a : 0.0;
    tab[L.cinv + 2 * n] = n ? 1.0 / ((double)n * (n + 1)) : 0.0;  // eqs 2.13-2.14 factors
    tab[L.cinv + 2 * n + 1] = 1.0 / (2.0 * n + 1.0);
  }
  if (tid >= (p + 1) * (p + 1)) return;
  const int j = tid / (p + 1), m = tid % (p + 1);
  const double t = tab[L.t + j], s = tab[L.st + j];
  // P~_m^m = sqrt((2m+1)/(4 pi (2m)!)) (2m-1)!! s^m via the ratio recurrence
  double pmm = 0.28209479177387814347;  // 1/sqrt(4 pi)
  for (int k = 1; k <= m; ++k) pmm *= s * sqrt((2.0 * k + 1.0) / (2.0 * k));
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
    // d/dtheta P~_n^m = (n t P~_n^m - sqrt((2n+1)(n^2-m^2)/(2n-1)) P~_{n-1}^m) / sin(theta)
    const double cnm = (n > m) ? sqrt((2.0 * n + 1.0) * ((double)n * n - (double)m * m) / (2.0 * n - 1.0)) : 0.0;
    const double prev = (n > m) ? pprev : 0.0;
    const int c = lm_index(p, n, m);
    if (j == 0) {
      tab[L.rA + c] = (n > m + 1) ? sqrt((4.0 * n * n - 1.0) / ((double)n * n - (double)m * m))
                                  : (n == m + 1 ? sqrt(2.0 * m + 3.0) : 0.0);
      tab[L.rB + c] = (n > m + 1) ? sqrt(((n - 1.0) * (n - 1.0) - (double)m * m) /
                                         (4.0 * (n - 1.0) * (n - 1.0) - 1.0))
                                  : 0.0;
      tab[L.rC + c] = cnm;
    }
    tab[L.P + (int64_t)j * L.nlm + c] = pcur;
    tab[L.dP + (int64_t)j * L.nlm + c] = (n * t * pcur - cnm * prev) / s;
    tab[L.mPs + (int64_t)j * L.nlm + c] = m * pcur / s;
  }
}

// Node positions, outward normals and weights (eqs 4.2, 4.4):
// n = (sin th_j cos ph_k, sin th_j sin ph_k, t_j), x = c + a n, w = a^2 w^_j.
__global__ void k_nodes(int p, int64_t N, const double* __restrict__ tab,
                        const double* __restrict__ centres, const double* __restrict__ radii,
                        double* __restrict__ x, double* __restrict__ nrm, double* __restrict__ w) {
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
  nrm[3 * i + 0] = n0;
  nrm[3 * i + 1] = n1;
  nrm[3 * i + 2] = n2;
  x[3 * i + 0] = centres[3 * s + 0] + a * n0;
  x[3 * i + 1] = centres[3 * s + 1] + a * n1;
  x[3 * i + 2] = centres[3 * s + 2] + a * n2;
  w[i] = a * a * tab[L.wu + j];
}

}  // namespace bie
