// k_self.cuh -- per-sphere spectral self term fused with source packing.
//
// One CTA per sphere (rows a2, a4, a5, a6 of SURVEY §8(a)):
//   A  load f, q of the sphere; write the packed far-field source records
//      (x, n, w f/(8 pi mu), (3/(4 pi)) w q); rotate (a/mu) f and q to
//      spherical components (e_r, e_theta, e_phi)
//   B  forward real DFT over the 2p+2 azimuthal nodes of every latitude
//      (the k <-> 2p+2-k symmetry is folded into phase A)
//      (the FFT stage of the paper's fast transform; a dense
//      26-point DFT at p = 12)
//   C  Legendre projection per (density, n, m) (eq 2.3 discretised, reading
//      R9) onto {Y e_r, G, X} (eq 2.12)
//   C2 conversion to {V, W, X} (eqs 2.13-2.14), the diagonal scale
//      psi = lamS (a/mu) alpha[f] + lamD_pv alpha[q] (Thm 2, readings
//      R2/R3/R5/R6), back to {Y, G, X} (eqs 2.16-2.17)
//   D  inverse Legendre sum per (component, latitude, m)
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
  double* alpha;    // nullable: [ns][2][nlm][3][2] projections <F,Y e_r>, <F,G>, <F,X>
                    // of (a/mu) f and q, for the near-singular correction (k_near)
  const double* psinear = nullptr;  // k_sht only: [ns][nlm][6] psi^{Y,G,X} added before the
                                    // inverse transform (NEXT-4 delayed evaluation)
  int precond;      // 1: u = P^{-1} q with P = 1/2 I + S_self + D_self (f ignored):
                    //    eigenvalue 1/(1/2 + lamS a/mu + lamD) on every VSH mode of
                    //    degree <= p and 2 on the rest (NEXT-2 preconditioner)
  double cS = 0.0;    // 1/(8 pi mu) (computed once on the host)
  int out_stage = 0;  // k_self_t: records (and u) staged in shared memory and written
                      // by TMA bulk stores (launch with self_smem_bytes(p, SPC, true))
};


// column c of the m-major (n, m) layout (lm_index) -> m and the column of
// (m, m): the root of off(m) = m P1 - m (m - 1) / 2 <= c in fp32, then one
// integer correction step each way (exact for every p <= BIE_P_MAX)
__device__ __forceinline__ void decode_col(int c, int P1, int& m, int& off) {
  const float b = 2.0f * P1 + 1.0f;
  m = (int)((b - sqrtf(b * b - 8.0f * c)) * 0.5f);
  m = max(0, min(m, P1 - 1));
  off = m * P1 - (m * (m - 1)) / 2;
  if (off > c) { --m; off -= P1 - m; }
  else if (off + (P1 - m) <= c) { off += P1 - m; ++m; }
}

__host__ __device__ inline int64_t self_smem_doubles(int p);
// Dynamic shared memory of k_self_t for SPC spheres per CTA; out_stage adds
// the SPC x 12 nsn-double record staging area.  (Staging the Legendre tables
// P, dP, mPs as well -- one more bulk copy -- measured slower at p = 6, 8, 12:
// profiles/r02_self_tune.jsonl, r34.)
inline size_t self_smem_bytes(int p, int spc, bool out_stage) {
  const int P1 = p + 1, nphi = 2 * p + 2, nsn = P1 * nphi;
  return (size_t)(spc * (6 * nsn + 12 * P1 * P1) + 2 * nphi + 2 + (out_stage ? spc * 12 * nsn : 0)) *
         sizeof(double);
}
__host__ __device__ inline int64_t self_smem_doubles(int p) {
  const int P1 = p + 1, nphi = 2 * p + 2, nsn = P1 * nphi;
  const int64_t C = 6LL * nsn;       // spherical components; reused as ALPHA, then U
  const int64_t F = 12LL * P1 * P1;  // [2 dens][3 comp][j][m][re,im]; reused as PSI
  // F first stages the sphere's f and q (6 nsn = 12 P1^2 doubles) for phase A.
  // PSI ([(n,m)][Y,G,X][re,im], 3 P1 (P1+1) <= F doubles) aliases F, dead after
  // phase C: 24 P1^2 + 4 P1 + 2 doubles = 210 KB at p = 32 (<= 227 KB opt-in).
  return C + F + 2LL * nphi + 2;  // + the staging mbarrier
}

// PT > 0: the order p is the compile-time constant PT (loop bounds, index
// decoding and strides fold away); PT = 0: generic runtime p.
// SPC: spheres per CTA.  Each phase's item loop handles the same item of all
// SPC spheres back to back -- independent work the scheduler interleaves
// (latency hiding within a thread) -- sharing the phase barriers.
template <int TPB, int MINB, int PT = 0, int SPC = 1>
__global__ void __launch_bounds__(TPB, MINB) k_self_t(SelfArgs A) {
  extern __shared__ __align__(16) double sm[];
  const int p = PT > 0 ? PT : A.p, P1 = p + 1, nphi = 2 * p + 2, nsn = P1 * nphi;
  const TableLayout L(p);
  const int nlm = L.nlm;
  const int SZ = 6 * nsn + 12 * P1 * P1;  // per sphere: C [2][3][nsn] + F [2][3][P1][P1][2]
  double2* tw = reinterpret_cast<double2*>(sm + SPC * SZ);  // (cos, sin)(2 pi q/nphi), shared
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SPC * SZ + 2 * nphi);
  // out_stage: per-sphere packed records [nsn][12], written by one TMA bulk store
  auto Rp = [&](int sp) { return sm + SPC * SZ + 2 * nphi + 2 + sp * 12 * nsn; };
  // per-sphere views: C; F (PSI aliases F, dead after phase C); U aliases C
  auto Cp = [&](int sp) { return sm + sp * SZ; };
  auto Fp_ = [&](int sp) { return sm + sp * SZ + 6 * nsn; };
  const double* __restrict__ tab = A.tab;
  int64_t sidx[SPC];
  bool valid[SPC];
  double ra[SPC], rcx[SPC], rcy[SPC], rcz[SPC], raS[SPC];
#pragma unroll
  for (int sp = 0; sp < SPC; ++sp) {
    sidx[sp] = (int64_t)blockIdx.x * SPC + sp;
    valid[sp] = sidx[sp] < A.ns;
  }
  const int tid = threadIdx.x, nt = blockDim.x;
  // f and q of the sphere (contiguous 24 nsn bytes each) land in F through the
  // TMA unit (cp.async.bulk, no LSU wavefronts); the strided per-node reads of
  // phase A and of the record writer then hit shared memory (ncu r18: the
  // kernel was bound by L1 wavefronts, 84 %, half of them strided global
  // accesses).  Unaligned user pointers fall back to cooperative loads.  The
  // copies are issued first so that their DRAM latency overlaps the rest of
  // the CTA's set-up; the other threads meet the mbarrier only after the
  // barrier below.
  const bool tma_f = A.f && !(reinterpret_cast<uintptr_t>(A.f) & 15);
  const bool tma_q = A.q && !(reinterpret_cast<uintptr_t>(A.q) & 15);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const uint32_t bytes = (uint32_t)(3 * nsn * sizeof(double));
    int nvalid = 0;
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp) nvalid += valid[sp] ? 1 : 0;
    mbar_arrive_expect_tx(bar, (uint32_t)nvalid * bytes * ((tma_f ? 1 : 0) + (tma_q ? 1 : 0)));
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp) {
      if (!valid[sp]) continue;
      if (tma_f) bulk_g2s(Fp_(sp), A.f + sidx[sp] * 3 * nsn, bytes, bar);
      if (tma_q) bulk_g2s(Fp_(sp) + 3 * nsn, A.q + sidx[sp] * 3 * nsn, bytes, bar);
    }
  }
#pragma unroll
  for (int sp = 0; sp < SPC; ++sp) {
    const int64_t sc = valid[sp] ? sidx[sp] : A.ns - 1;
    ra[sp] = A.radii[sc];
    rcx[sp] = A.centres[3 * sc];
    rcy[sp] = A.centres[3 * sc + 1];
    rcz[sp] = A.centres[3 * sc + 2];
    raS[sp] = ra[sp] / A.mu;
  }
  const double cS = A.cS, cD = 3.0 / (4.0 * kPi);  // cS = 1/(8 pi mu) from the host

  // ---------------------------------------------------------------- A (+ B0)
  // Node pairs (k, nphi-k) of a latitude are handled by one thread so that
  // the real-signal symmetry used by the DFT below is applied on the fly:
  //   C[k] = g(k) + g(nphi-k),  C[nphi-k] = g(k) - g(nphi-k)   (k = 1..p),
  //   C[0] = g(0),  C[P1] = g(P1)  -- halving the DFT's multiply-adds.
  const bool spec = A.self || A.alpha;
  auto node = [&](int sp, int j, int k, double* g) {
    const int kk = j * nphi + k;
    const double aS = raS[sp];
    const double* Fs = Fp_(sp);
    const double f0 = Fs[3 * kk], f1 = Fs[3 * kk + 1], f2 = Fs[3 * kk + 2];
    const double q0 = Fs[3 * nsn + 3 * kk], q1 = Fs[3 * nsn + 3 * kk + 1], q2 = Fs[3 * nsn + 3 * kk + 2];
    const double ct = tab[L.t + j], st = tab[L.st + j];
    const double cp = tw[k].x, sp_ = tw[k].y;
    const double n0 = st * cp, n1 = st * sp_, n2 = ct;
    if (A.out_stage) {  // packed source record (row a2) into the staging area
      const double a = ra[sp];
      const double w = a * a * tab[L.wu + j];
      const double ws = w * cS, wd = w * cD;
      double2* r2 = reinterpret_cast<double2*>(Rp(sp) + kk * kRec);
      r2[0] = make_double2(rcx[sp] + a * n0, rcy[sp] + a * n1);
      r2[1] = make_double2(rcz[sp] + a * n2, n0);
      r2[2] = make_double2(n1, n2);
      r2[3] = make_double2(ws * f0, ws * f1);
      r2[4] = make_double2(ws * f2, wd * q0);
      r2[5] = make_double2(wd * q1, wd * q2);
    }
    // e_r = n, e_theta = (ct cp, ct sp, -st), e_phi = (-sp, cp, 0)
    g[0] = aS * (f0 * n0 + f1 * n1 + f2 * n2);
    g[1] = aS * (f0 * ct * cp + f1 * ct * sp_ - f2 * st);
    g[2] = aS * (-f0 * sp_ + f1 * cp);
    g[3] = q0 * n0 + q1 * n1 + q2 * n2;
    g[4] = q0 * ct * cp + q1 * ct * sp_ - q2 * st;
    g[5] = -q0 * sp_ + q1 * cp;
  };
  // -------------------------------------------------------------- A0 staging
  for (int k = tid; k < nphi; k += nt) tw[k] = make_double2(tab[L.cph + k], tab[L.sph + k]);
#pragma unroll
  for (int sp = 0; sp < SPC; ++sp) {
    if (!valid[sp]) continue;
    double* Fs = Fp_(sp);
    for (int e = tid; e < 3 * nsn; e += nt) {
      if (!tma_f) Fs[e] = A.f ? A.f[sidx[sp] * 3 * nsn + e] : 0.0;
      if (!tma_q) Fs[3 * nsn + e] = A.q ? A.q[sidx[sp] * 3 * nsn + e] : 0.0;
    }
  }
  __syncthreads();  // tw, fallback staging and the mbarrier ready
  mbar_wait(bar, 0);
  // -------------------------------------------------------------- A1 records
  // Without out_stage (shared memory too small): packed source records (row
  // a2) written as consecutive 16-byte chunks so that a warp's stores cover
  // contiguous 512 bytes.
#pragma unroll
  for (int sp = 0; sp < SPC; ++sp) {
    if (!valid[sp] || A.out_stage) continue;
    const double* Fs = Fp_(sp);
    const double a = ra[sp];
    double2* out = reinterpret_cast<double2*>(A.rec + sidx[sp] * nsn * kRec);
    for (int e = tid; e < 6 * nsn; e += nt) {
      const int kk = e / 6, part = e - 6 * kk;
      const int j = kk / nphi, k = kk - j * nphi;
      double2 v;
      if (part < 3) {
        const double st = tab[L.st + j];
        const double2 t = tw[k];
        const double n0 = st * t.x, n1 = st * t.y, n2 = tab[L.t + j];
        v = part == 0 ? make_double2(rcx[sp] + a * n0, rcy[sp] + a * n1)
                      : (part == 1 ? make_double2(rcz[sp] + a * n2, n0) : make_double2(n1, n2));
      } else {
        const double w = a * a * tab[L.wu + j];
        // (f0 f1 | f2 q0 | q1 q2) scaled by (ws ws | ws wd | wd wd)
        const int u0 = 2 * (part - 3), u1 = u0 + 1;
        const double x0 = Fs[u0 < 3 ? 3 * kk + u0 : 3 * nsn + 3 * kk + u0 - 3];
        const double x1 = Fs[u1 < 3 ? 3 * kk + u1 : 3 * nsn + 3 * kk + u1 - 3];
        v = make_double2(x0 * w * (u0 < 3 ? cS : cD), x1 * w * (u1 < 3 ? cS : cD));
      }
      out[e] = v;
    }
  }
  for (int it = tid; it < P1 * (P1 + 1); it += nt) {
    const int j = it / (P1 + 1), k = it - j * (P1 + 1);
    const bool pair = k > 0 && k < P1;
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp) {
      if (!valid[sp]) continue;
      if (spec || A.out_stage) {
        double g1[6], g2[6];
        node(sp, j, k, g1);
        if (pair) node(sp, j, nphi - k, g2);
        if (!spec) continue;
        double* row = Cp(sp) + j * nphi;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          if (pair) {
            row[d * nsn + k] = g1[d] + g2[d];
            row[d * nsn + nphi - k] = g1[d] - g2[d];
          } else {
            row[d * nsn + k] = g1[d];
          }
        }
      }
    }
  }
  auto zero_u = [&]() {
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp)
      if (valid[sp] && A.u)
        for (int e = tid; e < 3 * nsn; e += nt) A.u[sidx[sp] * 3 * nsn + e] = 0.0;
  };
  // out_stage: the staged records leave through one TMA bulk store per sphere
  // (no LSU wavefronts; the issuing thread waits for its reads before exit)
  if (A.out_stage) fence_proxy_async_smem();
  __syncthreads();
  if (A.out_stage && tid == 0) {
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp)
      if (valid[sp]) bulk_s2g(A.rec + sidx[sp] * nsn * kRec, Rp(sp), (uint32_t)(nsn * kRec * sizeof(double)));
    bulk_commit();
  }
  if (!spec) {
    zero_u();
    if (A.out_stage && tid == 0) bulk_wait_read0();
    return;
  }
  // ---------------------------------------------------------------- B
  // F[dc][j][m] = sum_k g[k] e^{-i m phi_k}
  //   = g0 + (-1)^m g_{p+1} + sum_{k=1}^{p} S_k cos(m phi_k) - i sum_k D_k sin(m phi_k)
  // Two azimuthal orders per item (m and m + H, H = ceil(P1/2)) share the row
  // loads and give two independent accumulation chains.
  {
    const int H = (P1 + 1) / 2;
    for (int it = tid; it < 6 * P1 * H; it += nt) {
      const int mh = it % H, row = it / H;
      const int m1 = mh, m2 = mh + H;
      const bool two = m2 < P1;
#pragma unroll
      for (int sp = 0; sp < SPC; ++sp) {
        const double* g = Cp(sp) + row * nphi;
        double* F = Fp_(sp);
        double re1 = (m1 & 1) ? g[0] - g[P1] : g[0] + g[P1], im1 = 0.0;
        double re2 = (m2 & 1) ? g[0] - g[P1] : g[0] + g[P1], im2 = 0.0;
        // (cos, sin)(m phi_k) by the angle-addition recurrence from
        // (cos, sin)(m phi_1): no twiddle loads in the loop (rounding grows
        // like k eps, < 1e-14 at p = 32)
        const double2 w1 = tw[m1], w2 = tw[two ? m2 : 0];
        double2 t1 = w1, t2 = w2;
        for (int k = 1; k <= p; ++k) {
          const double gs = g[k], gd = g[nphi - k];
          re1 = fma(gs, t1.x, re1);
          im1 = fma(-gd, t1.y, im1);
          re2 = fma(gs, t2.x, re2);
          im2 = fma(-gd, t2.y, im2);
          t1 = make_double2(fma(t1.x, w1.x, -t1.y * w1.y), fma(t1.y, w1.x, t1.x * w1.y));
          t2 = make_double2(fma(t2.x, w2.x, -t2.y * w2.y), fma(t2.y, w2.x, t2.x * w2.y));
        }
        F[2 * (row * P1 + m1)] = re1;
        F[2 * (row * P1 + m1) + 1] = im1;
        if (two) {
          F[2 * (row * P1 + m2)] = re2;
          F[2 * (row * P1 + m2) + 1] = im2;
        }
      }
    }
  }
  __syncthreads();
  // ---------------------------------------------------------------- C
  // Projection per (density, n, m): ALPHA[d][c] = (<F,Y e_r>, <F,G>, <F,X>),
  // complex.  ALPHA aliases C, which is dead after phase B.
  for (int it = tid; it < 2 * nlm; it += nt) {
    const int d = it / nlm, c = it - d * nlm;
    int m, off;
    decode_col(c, P1, m, off);
    double y0[SPC], y1[SPC], g0[SPC], g1[SPC], x0[SPC], x1[SPC];
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp) y0[sp] = y1[sp] = g0[sp] = g1[sp] = x0[sp] = x1[sp] = 0.0;
    for (int j = 0; j < P1; ++j) {
      const double wj = tab[L.wu + j];
      const double Pv = wj * tab[L.P + (int64_t)j * nlm + c];
      const double dPv = wj * tab[L.dP + (int64_t)j * nlm + c];
      const double mPv = wj * tab[L.mPs + (int64_t)j * nlm + c];
#pragma unroll
      for (int sp = 0; sp < SPC; ++sp) {
        const double* F = Fp_(sp);
        const double* Fr = F + 2 * (((3 * d + 0) * P1 + j) * P1 + m);
        const double* Ft = F + 2 * (((3 * d + 1) * P1 + j) * P1 + m);
        const double* Fp = F + 2 * (((3 * d + 2) * P1 + j) * P1 + m);
        y0[sp] = fma(Pv, Fr[0], y0[sp]);                          // <F, Y e_r>
        y1[sp] = fma(Pv, Fr[1], y1[sp]);
        g0[sp] = fma(dPv, Ft[0], fma(mPv, Fp[1], g0[sp]));        // <F, G> = dP F_t - i mP F_p
        g1[sp] = fma(dPv, Ft[1], fma(-mPv, Fp[0], g1[sp]));
        x0[sp] = fma(dPv, Fp[0], fma(-mPv, Ft[1], x0[sp]));       // <F, X> = dP F_p + i mP F_t
        x1[sp] = fma(dPv, Fp[1], fma(mPv, Ft[0], x1[sp]));
      }
    }
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp) {
      double* o = Cp(sp) + 6 * it;  // ALPHA [2][nlm][3][2]
      o[0] = y0[sp]; o[1] = y1[sp]; o[2] = g0[sp]; o[3] = g1[sp]; o[4] = x0[sp]; o[5] = x1[sp];
      if (A.alpha && valid[sp]) {
        double2* g2 = reinterpret_cast<double2*>(A.alpha + (sidx[sp] * 2 * nlm + it) * 6);
        g2[0] = make_double2(y0[sp], y1[sp]);
        g2[1] = make_double2(g0[sp], g1[sp]);
        g2[2] = make_double2(x0[sp], x1[sp]);
      }
    }
  }
  if (!A.self) {
    zero_u();
    if (A.out_stage && tid == 0) bulk_wait_read0();
    return;
  }
  __syncthreads();
  // ---------------------------------------------------------------- C2
  // {Y,G,X} -> {V,W,X} (eqs 2.13-2.14), diagonal scale (Thm 2), back to
  // {Y,G,X} (eqs 2.16-2.17) for the inverse transform.
  // items (c, re/im): twice the column count, so that more threads have work
  for (int itc = tid; itc < 2 * nlm; itc += nt) {
    const int c = itc >> 1, ri = itc & 1;
    int m, off;
    decode_col(c, P1, m, off);
    const int n = m + (c - off);
    const double* lS = tab + L.lamS + 3 * n;
    const double* lD = tab + L.lamD + 3 * n;
    const double inn = tab[L.cinv + 2 * n], i2n = tab[L.cinv + 2 * n + 1];  // (table: no divisions)
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp) {
      const double* ALPHA = Cp(sp);
      const double* af = ALPHA + 6 * c;
      const double* aq = ALPHA + 6 * (nlm + c);
      double* o = Fp_(sp) + 6 * c;  // PSI
      const double aS = raS[sp];
      {
        double aV[2], aW[2], aX[2];
        const double* al[2] = {af, aq};
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          const double phY = al[d][ri], phG = al[d][2 + ri] * inn, phX = al[d][4 + ri] * inn;
          aV[d] = (n * phG - phY) * i2n;          // eq 2.13
          aW[d] = ((n + 1) * phG + phY) * i2n;    // eq 2.14
          aX[d] = phX;
        }
        double psV, psW, psX;
        if (A.precond) {  // (1/sigma - 2) on the degree-<=p modes; +2 x added in phase E
          psV = (1.0 / (0.5 + lS[0] * aS + lD[0]) - 2.0) * aV[1];
          psW = n ? (1.0 / (0.5 + lS[1] * aS + lD[1]) - 2.0) * aW[1] : 0.0;
          psX = n ? (1.0 / (0.5 + lS[2] * aS + lD[2]) - 2.0) * aX[1] : 0.0;
        } else {
          psV = lS[0] * aV[0] + lD[0] * aV[1];
          psW = lS[1] * aW[0] + lD[1] * aW[1];
          psX = lS[2] * aX[0] + lD[2] * aX[1];
        }
        o[0 + ri] = -(n + 1.0) * psV + n * psW;  // psi^Y (eq 2.17)
        o[2 + ri] = psV + psW;                   // psi^G (eq 2.16)
        o[4 + ri] = psX;                         // psi^X
      }
    }
  }
  __syncthreads();
  // ---------------------------------------------------------------- D
  // per (latitude, m): U_r from one item, U_theta and U_phi together from
  // another (they share the dP, mP and psi^G, psi^X loads):
  // U_r = sum_n psiY P, U_t = sum_n psiG dP - i psiX mP, U_p = sum_n i psiG mP + psiX dP
  for (int it = tid; it < 2 * P1 * P1; it += nt) {
    const int half = it / (P1 * P1);
    const int j = (it / P1) % P1, m = it % P1;
    const int c0 = lm_index(p, m, m);
    const double* Pj = tab + L.P + (int64_t)j * nlm;
    const double* dPj = tab + L.dP + (int64_t)j * nlm;
    const double* mPj = tab + L.mPs + (int64_t)j * nlm;
    const int o = j * P1 + m;
    if (half == 0) {
      double a0[SPC], a1[SPC];
#pragma unroll
      for (int sp = 0; sp < SPC; ++sp) a0[sp] = a1[sp] = 0.0;
      for (int c = c0; c < c0 + (P1 - m); ++c) {
        const double pv = __ldg(Pj + c);
#pragma unroll
        for (int sp = 0; sp < SPC; ++sp) {
          const double* ps = Fp_(sp) + 6 * c;
          a0[sp] = fma(ps[0], pv, a0[sp]);
          a1[sp] = fma(ps[1], pv, a1[sp]);
        }
      }
#pragma unroll
      for (int sp = 0; sp < SPC; ++sp) {
        double* U = Cp(sp);
        U[2 * o] = a0[sp];
        U[2 * o + 1] = a1[sp];
      }
    } else {
      double t0[SPC], t1[SPC], q0[SPC], q1[SPC];
#pragma unroll
      for (int sp = 0; sp < SPC; ++sp) t0[sp] = t1[sp] = q0[sp] = q1[sp] = 0.0;
      for (int c = c0; c < c0 + (P1 - m); ++c) {
        const double dp = __ldg(dPj + c), mp = __ldg(mPj + c);
#pragma unroll
        for (int sp = 0; sp < SPC; ++sp) {
          const double* ps = Fp_(sp) + 6 * c;
          t0[sp] = fma(ps[2], dp, fma(ps[5], mp, t0[sp]));
          t1[sp] = fma(ps[3], dp, fma(-ps[4], mp, t1[sp]));
          q0[sp] = fma(ps[4], dp, fma(-ps[3], mp, q0[sp]));
          q1[sp] = fma(ps[5], dp, fma(ps[2], mp, q1[sp]));
        }
      }
#pragma unroll
      for (int sp = 0; sp < SPC; ++sp) {
        double* U = Cp(sp);
        U[2 * (P1 * P1 + o)] = t0[sp];
        U[2 * (P1 * P1 + o) + 1] = t1[sp];
        U[2 * (2 * P1 * P1 + o)] = q0[sp];
        U[2 * (2 * P1 * P1 + o) + 1] = q1[sp];
      }
    }
  }
  __syncthreads();
  // ---------------------------------------------------------------- E
  // Inverse DFT for the node pair (k, nphi-k) of a latitude:
  //   u(k) = U0 + 2(c - s), u(nphi-k) = U0 + 2(c + s),
  //   c = sum_m Re U_m cos(m phi_k), s = sum_m Im U_m sin(m phi_k),
  // then spherical -> Cartesian components and the store of u_self (out_stage
  // with a 16-byte-aligned u: into F, dead after phase D, then one TMA bulk
  // store per sphere).
  const bool ustage = A.out_stage && !(reinterpret_cast<uintptr_t>(A.u) & 15);
  for (int it = tid; it < P1 * (P1 + 1); it += nt) {
    const int j = it / (P1 + 1), k = it % (P1 + 1);
    double c[SPC][3], sn_[SPC][3];
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp)
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) c[sp][comp] = sn_[sp][comp] = 0.0;
    const double2 wk = tw[k];  // (cos, sin)(m phi_k) by angle addition in m
    double2 t = wk;
    for (int m = 1; m <= p; ++m) {
#pragma unroll
      for (int sp = 0; sp < SPC; ++sp) {
        const double2* U2 = reinterpret_cast<const double2*>(Cp(sp));
#pragma unroll
        for (int comp = 0; comp < 3; ++comp) {
          const double2 Um = U2[(comp * P1 + j) * P1 + m];
          c[sp][comp] = fma(Um.x, t.x, c[sp][comp]);
          sn_[sp][comp] = fma(Um.y, t.y, sn_[sp][comp]);
        }
      }
      t = make_double2(fma(t.x, wk.x, -t.y * wk.y), fma(t.y, wk.x, t.x * wk.y));
    }
    const double ct = tab[L.t + j], st = tab[L.st + j];
#pragma unroll
    for (int sp = 0; sp < SPC; ++sp) {
      if (!valid[sp]) continue;
      const double* U = Cp(sp);
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        if (side == 1 && (k == 0 || k == P1)) break;
        const int kk = side ? nphi - k : k;
        double v[3];
#pragma unroll
        for (int comp = 0; comp < 3; ++comp) {
          const double U0 = U[2 * ((comp * P1 + j) * P1)];
          v[comp] = fma(2.0, side ? c[sp][comp] + sn_[sp][comp] : c[sp][comp] - sn_[sp][comp], U0);
        }
        const double2 t = tw[kk];
        const double cp = t.x, spn = t.y;
        const int64_t i = sidx[sp] * nsn + j * nphi + kk;
        double w0 = v[0] * st * cp + v[1] * ct * cp - v[2] * spn;
        double w1 = v[0] * st * spn + v[1] * ct * spn + v[2] * cp;
        double w2 = v[0] * ct - v[1] * st;
        if (A.precond) {
          w0 = fma(2.0, A.q[3 * i + 0], w0);
          w1 = fma(2.0, A.q[3 * i + 1], w1);
          w2 = fma(2.0, A.q[3 * i + 2], w2);
        }
        double* uo = ustage ? Fp_(sp) + 3 * (j * nphi + kk) : A.u + 3 * i;
        uo[0] = w0;
        uo[1] = w1;
        uo[2] = w2;
      }
    }
  }
  if (ustage) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int sp = 0; sp < SPC; ++sp)
        if (valid[sp]) bulk_s2g(A.u + sidx[sp] * 3 * nsn, Fp_(sp), (uint32_t)(3 * nsn * sizeof(double)));
      bulk_commit();
    }
  }
  if (A.out_stage && tid == 0) bulk_wait_read0();
}

// Launch configurations chosen by tools/self_tune.cu (profiles/r01_self_tune.txt,
// re-swept with the TMA staging in profiles/r02_self_tune.jsonl): p <= 8 many
// 64-thread CTAs, p = 12 128 threads.  The orders of the BASELINE
// configurations (4, 6, 8, 12) get compile-time-p instantiations; every other
// p runs the generic kernel.  Outputs are staged (out_stage) whenever the
// staging area fits the 227 KB opt-in (p <= 22 for one sphere per CTA).
inline bool self_out_stage(int p, int spc) { return self_smem_bytes(p, spc, true) <= 227 * 1024; }
inline void launch_self(const SelfArgs& A0, cudaStream_t s) {
  SelfArgs A = A0;
  A.out_stage = self_out_stage(A.p, 1) ? 1 : 0;
  const size_t smem = self_smem_bytes(A.p, 1, A.out_stage);
  const unsigned g = (unsigned)A.ns;
  switch (A.p) {
    case 4: k_self_t<64, 12, 4><<<g, 64, smem, s>>>(A); break;
    case 6: k_self_t<64, 12, 6><<<g, 64, smem, s>>>(A); break;
    case 8: k_self_t<64, 12, 8><<<g, 64, smem, s>>>(A); break;
    case 12: k_self_t<128, 5, 12><<<g, 128, smem, s>>>(A); break;
    default:
      if (A.p <= 8) k_self_t<64, 12><<<g, 64, smem, s>>>(A);
      else k_self_t<128, 4><<<g, 128, smem, s>>>(A);
  }
}
// Two spheres per CTA (SPC = 2): independent work per thread for the scheduler
// to interleave; same phases and barriers (measured against SPC = 1 in
// profiles/r02_self_bench.jsonl).
inline size_t self2_smem_bytes(int p) { return self_smem_bytes(p, 2, false); }
inline void launch_self2(const SelfArgs& A0, cudaStream_t s) {
  SelfArgs A = A0;
  A.out_stage = self_out_stage(A.p, 2) ? 1 : 0;
  const size_t smem = self_smem_bytes(A.p, 2, A.out_stage);
  const unsigned g = (unsigned)((A.ns + 1) / 2);
  switch (A.p) {
    case 4: k_self_t<64, 8, 4, 2><<<g, 64, smem, s>>>(A); break;
    case 6: k_self_t<64, 8, 6, 2><<<g, 64, smem, s>>>(A); break;
    case 8: k_self_t<64, 8, 8, 2><<<g, 64, smem, s>>>(A); break;
    case 12: k_self_t<128, 3, 12, 2><<<g, 128, smem, s>>>(A); break;
    default:
      if (A.p <= 8) k_self_t<64, 8, 0, 2><<<g, 64, smem, s>>>(A);
      else k_self_t<128, 3, 0, 2><<<g, 128, smem, s>>>(A);
  }
}

inline void set_self_smem(int p) {
  const int smem2 = (int)self_smem_bytes(p, 2, self_out_stage(p, 2));
  if (smem2 <= 227 * 1024) {
    cudaFuncSetAttribute(k_self_t<64, 8, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    cudaFuncSetAttribute(k_self_t<64, 8, 6, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    cudaFuncSetAttribute(k_self_t<64, 8, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    cudaFuncSetAttribute(k_self_t<128, 3, 12, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    cudaFuncSetAttribute(k_self_t<64, 8, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    cudaFuncSetAttribute(k_self_t<128, 3, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  }
  const int smem = (int)self_smem_bytes(p, 1, self_out_stage(p, 1));
  cudaFuncSetAttribute(k_self_t<64, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_self_t<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_self_t<64, 12, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_self_t<64, 12, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_self_t<64, 12, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_self_t<128, 5, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
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
