// k_sht.cuh -- the per-sphere spectral self term (rows a2, a4, a5, a6 of
// SURVEY §8(a)) as batched small dense contractions on the FP64 tensor cores.
//
// What it computes (PAPER §4.1; Thm 2; readings R2-R9 of
// DESIGN.md §3): for every sphere s and g in {(a_s/mu) f, q}, the discrete
// vector-spherical-harmonic projection alpha^Z_nm[g] (eqs 2.3, 2.12-2.14,
// reading R9), the diagonal scale psi = lamS(n) alpha[(a/mu) f] +
// lamD_pv(n) alpha[q] (Thm 2 via eqs 3.6-3.11 at r -> 1), and one inverse
// transform (eqs 2.15-2.17; "add coefficients ... then one inverse
// transform"), fused with the packing of the far-field source records (row a2).
// It is the same operator as the round-1 k_self (kept in k_self.cuh as the
// DFMA reference design); only the schedule differs.
//
// Schedule (one CTA processes SB spheres per iteration, persistent over the
// sphere batches; every separable stage is a GEMM whose M dimension runs over
// the batch's spheres x components x {re, im}, so the transform tables are the
// shared B operand):
//   A   load f, q; write the records; rotate to (e_r, e_th, e_ph); fold the
//       real-DFT symmetry: row (b, d, j) = [g_0, g_P1, S_1..S_p | D_1..D_p],
//       S_k = g_k + g_{2P1-k}, D_k = g_k - g_{2P1-k}
//   B   forward real DFT over longitude (the "FFT in longitude" of P:47/P:342):
//         Re F = [g0 gP1 S] x Tc      Im F = D x Ts           (two GEMMs)
//   C   Legendre projection per azimuthal order m (eq 2.3 discretised):
//         Y  = F_r(re, im rows) x (w P~_n^m)                    K = latitudes
//         GX = F_th,ph(re, im rows) x [w dP~ | w mP~/sin]        (one GEMM)
//   C2  {Y,G,X} -> {V,W,X} (eqs 2.13-2.14), diagonal scale (Thm 2), back to
//       {Y,G,X} (eqs 2.16-2.17), laid out as the next GEMM's A operand
//   D   inverse Legendre sum per m:  U = psi x [P~^T] and [psiG|psiX] x [dP~^T; mP~^T]
//   E   inverse real DFT:  c = ReU x Ec,  s = ImU x Es           (two GEMMs)
//   F   u(k) = c_k - s_k, u(2P1-k) = c_k + s_k; back to Cartesian; store u.
// The GEMMs run on mma.sync.m8n8k4.f64 (SASS DMMA) when MMA = true, else on a
// register-tiled DFMA micro-kernel with the same fragment layout (kept so the
// two can be measured in the kernel).  B operands (the tables)
// are pre-arranged in fragment order by k_sht_tables (one coalesced 256-byte
// warp load per fragment, L1-resident) and held in registers across the
// warp's M tiles; A operands are read from shared memory with row strides
// = 4 (mod 8) doubles, which makes every 8x4 fragment load conflict-free.
#pragma once
#include "common.cuh"
#include "k_setup.cuh"
#include "k_self.cuh"

namespace bie {

// ------------------------------------------------------------ sizes
__host__ __device__ constexpr int sht_rup(int x, int a) { return (x + a - 1) / a * a; }
// smallest stride >= x with stride = 4 (mod 8) doubles (conflict-free 8x4 fragments)
__host__ __device__ constexpr int sht_ld(int x) { return x % 8 <= 4 ? x - x % 8 + 4 : x - x % 8 + 12; }
// spheres per group iteration (one: every sphere is owned by one warp group)
__host__ __device__ constexpr int sht_sb(int) { return 1; }
// warps per group (one sphere at a time) and groups per CTA; groups are
// independent -- they synchronise with named barriers (or __syncwarp), never
// with the whole CTA -- so one group's load or barrier latency overlaps the
// others' work.
__host__ __device__ constexpr int sht_wps(int p) { return p <= 8 ? 1 : (p <= 16 ? 2 : 8); }
__host__ __device__ constexpr int sht_groups(int p) { return p <= 4 ? 16 : (p <= 7 ? 12 : (p == 8 ? 9 : 1)); }
// p <= 8: the fragment-order tables (<= 44 KB) are staged in shared memory once
// per CTA and shared by all its groups; above, they are read through L1/L2.
__host__ __device__ constexpr bool sht_tab_smem(int p) { return p <= 8; }

__host__ __device__ constexpr int64_t sht_max(int64_t a, int64_t b) { return a > b ? a : b; }

// doubles of the fragment-order tables of order p (== ShtTabLayout(p).total)
__host__ __device__ constexpr int64_t sht_tab_doubles(int p) {
  const int P1 = p + 1;
  int64_t o = 32LL * (((P1 + 4) / 4) * ((P1 + 7) / 8) + ((p + 3) / 4) * ((P1 + 7) / 8) +
                      ((P1 + 3) / 4) * ((P1 + 8) / 8) + ((p + 3) / 4) * ((p + 7) / 8)) +
              4 * P1;
  for (int m = 0; m <= p; ++m) {
    const int n = P1 - m;
    o += 32LL * (((P1 + 3) / 4) * ((n + 7) / 8) + ((P1 + 3) / 4) * ((2 * n + 7) / 8) +
                 ((n + 3) / 4) * ((P1 + 7) / 8) + ((2 * n + 3) / 4) * ((P1 + 7) / 8));
  }
  return o;
}

// Shared-memory carve-up of k_sht for order p (doubles).  Two big regions,
// each reused by the phases in turn (sizes are the max over their tenants):
//   region G : G (A -> B) | alpha partials AL (C -> C2) | U (D -> E)
//   region F : FT (B -> C) | AD (C2 -> D) | EO (E -> F)
// followed by the per-order constants (trig, latitude data, per-degree
// eigenvalue factors, the (m, c) decode of the coefficient index).
struct ShtDims {
  int p, P1, NP, SB, nlm, ldG, ldF, ldE, KY, KX, ADm;
  int64_t sizeG, sizeF, offG, offF, group, offTrig, offDeg, offMC, offTab, total;  // group = doubles per group
  __host__ __device__ constexpr ShtDims(int p_)
      : p(p_), P1(p_ + 1), NP(2 * p_ + 2), SB(sht_sb(p_)), nlm((p_ + 1) * (p_ + 2) / 2),
        ldG(sht_ld(p_ + 2 + sht_rup(p_, 4))),  // [g0 gP1 S | D] + K padding of the sin GEMM
        ldF(sht_ld(sht_rup(p_ + 1, 4))), ldE(2 * p_ + 3),
        KY(sht_ld(sht_rup(p_ + 1, 4))), KX(sht_ld(sht_rup(2 * p_ + 2, 4))),
        ADm(2 * sht_sb(p_) * sht_ld(sht_rup(p_ + 1, 4)) + 4 * sht_sb(p_) * sht_ld(sht_rup(2 * p_ + 2, 4))),
        // G region: G rows read up to the next multiple of 8 (last M tile)
        sizeG(sht_max((int64_t)sht_rup(6 * (p_ + 1) * sht_sb(p_), 8) * sht_ld(p_ + 2 + sht_rup(p_, 4)),
                      (int64_t)20 * sht_sb(p_) * ((p_ + 1) * (p_ + 2) / 2))),
        // F region: FT | AD (+ the pad rows of the last order's GX tile) | EO
        sizeF(sht_max(sht_max((int64_t)(12 * (p_ + 1) * sht_sb(p_)) * sht_ld(sht_rup(p_ + 1, 4)),
                              (int64_t)(p_ + 1) *
                                      (2 * sht_sb(p_) * sht_ld(sht_rup(p_ + 1, 4)) +
                                       4 * sht_sb(p_) * sht_ld(sht_rup(2 * p_ + 2, 4))) +
                                  8 * sht_ld(sht_rup(2 * p_ + 2, 4))),
                      (int64_t)3 * (p_ + 1) * sht_sb(p_) * (2 * p_ + 3))),
        offG(0), offF(sht_rup((int)sizeG, 2)),
        group(sht_rup((int)sizeG, 2) + sht_rup((int)sizeF, 2)),
        offTrig(sht_groups(p_) * (int64_t)(sht_rup((int)sizeG, 2) + sht_rup((int)sizeF, 2))),
        offDeg(offTrig + 2 * (2 * p_ + 2) + 3 * (p_ + 1)), offMC(offDeg + 8 * (p_ + 1)),
        offTab(sht_rup((int)(offMC + ((p_ + 1) * (p_ + 2) / 2 + 1) / 2 + 2), 2)),
        total(offTab + (sht_tab_smem(p_) ? sht_tab_doubles(p_) : 0)) {}
};

// Fragment-order table layout (built once per context by k_sht_tables).
// A B operand of K x N (padded to KS*4 x NT*8) is stored as
//   Bf[(nt * KS + ks) * 32 + lane] = B[ks*4 + lane%4][nt*8 + lane/4]   (0 in the pad).
// Per azimuthal order m the C and D tables have their own KS / NT.
struct ShtTabLayout {
  int p, P1;
  int KSc, NTc, KSs, NTs;   // forward DFT: cos (K = P1+1, N = P1), sin (K = p, N = P1)
  int KEc, NEc, KEs, NEs;   // inverse DFT: cos (K = P1, N = P1+1), sin (K = p, N = p)
  int64_t Tc, Ts, Ec, Es, mtab, total;  // doubles; mtab = per-m offsets (stored as doubles)
  __host__ __device__ explicit ShtTabLayout(int p_) : p(p_), P1(p_ + 1) {
    KSc = (P1 + 1 + 3) / 4; NTc = (P1 + 7) / 8;
    KSs = (p + 3) / 4;      NTs = (P1 + 7) / 8;
    KEc = (P1 + 3) / 4;     NEc = (P1 + 1 + 7) / 8;
    KEs = (p + 3) / 4;      NEs = (p + 7) / 8;
    int64_t o = 0;
    Tc = o; o += (int64_t)KSc * NTc * 32;
    Ts = o; o += (int64_t)KSs * NTs * 32;
    Ec = o; o += (int64_t)KEc * NEc * 32;
    Es = o; o += (int64_t)KEs * NEs * 32;
    mtab = o; o += 4 * P1;  // per m: offsets of CY, CGX, DY, DGX
    for (int m = 0; m <= p; ++m) {
      const int n = P1 - m;
      o += (int64_t)((P1 + 3) / 4) * ((n + 7) / 8) * 32;          // CY:  K = P1, N = n
      o += (int64_t)((P1 + 3) / 4) * ((2 * n + 7) / 8) * 32;      // CGX: K = P1, N = 2n
      o += (int64_t)((n + 3) / 4) * ((P1 + 7) / 8) * 32;          // DY:  K = n,  N = P1
      o += (int64_t)((2 * n + 3) / 4) * ((P1 + 7) / 8) * 32;      // DGX: K = 2n, N = P1
    }
    total = o;
  }
};

// One thread per table; the per-m blocks are filled by block m, the four DFT
// tables by the last four blocks.  Reads the normalised Legendre / trig /
// weight tables of k_tables (same context), so run after it.
__global__ void k_sht_tables(int p, const double* __restrict__ tab, double* __restrict__ st) {
  const TableLayout L(p);
  const ShtTabLayout S(p);
  const int P1 = p + 1, NP = 2 * p + 2;
  const int blk = blockIdx.x;
  auto cosk = [&](int m, int k) { return tab[L.cph + (m * k) % NP]; };
  auto sink = [&](int m, int k) { return tab[L.sph + (m * k) % NP]; };
  auto fill = [&](double* dst, int KS, int NT, auto val) {  // val(k, n) on the valid range, else 0
    for (int e = threadIdx.x; e < KS * NT * 32; e += blockDim.x) {
      const int lane = e % 32, ks = (e / 32) % KS, nt = e / 32 / KS;
      dst[e] = val(ks * 4 + lane % 4, nt * 8 + lane / 4);
    }
  };
  if (blk <= p) {  // per azimuthal order m
    const int m = blk, n = P1 - m;
    int64_t o = S.mtab + 4 * P1;
    for (int mm = 0; mm < m; ++mm) {
      const int nn = P1 - mm;
      o += (int64_t)((P1 + 3) / 4) * ((nn + 7) / 8) * 32 + (int64_t)((P1 + 3) / 4) * ((2 * nn + 7) / 8) * 32 +
           (int64_t)((nn + 3) / 4) * ((P1 + 7) / 8) * 32 + (int64_t)((2 * nn + 3) / 4) * ((P1 + 7) / 8) * 32;
    }
    const int64_t oCY = o;
    const int64_t oCGX = oCY + (int64_t)((P1 + 3) / 4) * ((n + 7) / 8) * 32;
    const int64_t oDY = oCGX + (int64_t)((P1 + 3) / 4) * ((2 * n + 7) / 8) * 32;
    const int64_t oDGX = oDY + (int64_t)((n + 3) / 4) * ((P1 + 7) / 8) * 32;
    if (threadIdx.x == 0) {
      st[S.mtab + 4 * m + 0] = (double)oCY;
      st[S.mtab + 4 * m + 1] = (double)oCGX;
      st[S.mtab + 4 * m + 2] = (double)oDY;
      st[S.mtab + 4 * m + 3] = (double)oDGX;
    }
    auto Pt = [&](int j, int deg) { return tab[L.P + (int64_t)j * L.nlm + lm_index(p, deg, m)]; };
    auto dPt = [&](int j, int deg) { return tab[L.dP + (int64_t)j * L.nlm + lm_index(p, deg, m)]; };
    auto mPt = [&](int j, int deg) { return tab[L.mPs + (int64_t)j * L.nlm + lm_index(p, deg, m)]; };
    // C: projection (weighted by the unit-sphere quadrature weight of latitude j)
    fill(st + oCY, (P1 + 3) / 4, (n + 7) / 8, [&](int j, int c) {
      return (j < P1 && c < n) ? tab[L.wu + j] * Pt(j, m + c) : 0.0;
    });
    fill(st + oCGX, (P1 + 3) / 4, (2 * n + 7) / 8, [&](int j, int c) {
      if (j >= P1 || c >= 2 * n) return 0.0;
      return c < n ? tab[L.wu + j] * dPt(j, m + c) : tab[L.wu + j] * mPt(j, m + c - n);
    });
    // D: synthesis (unweighted, transposed: K = degree, N = latitude)
    fill(st + oDY, (n + 3) / 4, (P1 + 7) / 8, [&](int c, int j) {
      return (j < P1 && c < n) ? Pt(j, m + c) : 0.0;
    });
    fill(st + oDGX, (2 * n + 3) / 4, (P1 + 7) / 8, [&](int c, int j) {
      if (j >= P1 || c >= 2 * n) return 0.0;
      return c < n ? dPt(j, m + c) : mPt(j, m + c - n);
    });
  } else if (blk == P1) {  // Tc: rows [g0, gP1, S_1..S_p] -> Re F_m
    fill(st + S.Tc, S.KSc, S.NTc, [&](int k, int m) {
      if (k > P1 || m >= P1) return 0.0;
      if (k == 0) return 1.0;
      if (k == 1) return (m & 1) ? -1.0 : 1.0;
      return cosk(m, k - 1);
    });
  } else if (blk == P1 + 1) {  // Ts: rows D_1..D_p -> Im F_m
    fill(st + S.Ts, S.KSs, S.NTs, [&](int k, int m) {
      return (k < p && m < P1) ? -sink(m, k + 1) : 0.0;
    });
  } else if (blk == P1 + 2) {  // Ec: Re U_m -> c_k, k = 0..P1 (weights 1, 2, 2, ...)
    fill(st + S.Ec, S.KEc, S.NEc, [&](int m, int k) {
      return (m < P1 && k <= P1) ? (m ? 2.0 : 1.0) * cosk(m, k) : 0.0;
    });
  } else if (blk == P1 + 3) {  // Es: Im U_m (m = 1..p) -> s_k (k = 1..p)
    fill(st + S.Es, S.KEs, S.NEs, [&](int m, int k) {
      return (m < p && k < p) ? 2.0 * sink(m + 1, k + 1) : 0.0;
    });
  }
}

// ------------------------------------------------------------ micro-kernel
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// C[M x N] = A[M x K] B[K x N] for one warp's share of the output tiles.
//   A: shared memory, row stride lda, first column a_k0 (K padded with finite
//      values up to KS*4 columns -- the B pad rows are zero);
//   B: fragment-order table (global, L1-resident) with KS x NT fragments;
//   store(row, col, v0, v1): output (row, col) and (row, col + 1), col even.
// Tiles are distributed over (nt, pair of M tiles); each warp keeps its B
// panel in registers (KMAX >= KS) and runs two independent accumulators.
// MMA = false: the same tiles on DFMA (the lane computes its two outputs with
// a K loop; the A row and B column are read from shared/L1 per k).
template <bool MMA, int KMAX, class Store>
__device__ __forceinline__ void sht_gemm(const double* __restrict__ A, int lda, int a_k0, int M, int K,
                                         const double* __restrict__ Bf, int KS, int NT, Store store,
                                         int item0, int nwarps) {
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) % nwarps;  // warp within the group
  const int MT = (M + 7) / 8, MP = (MT + 1) / 2;
  const int items = NT * MP;
  int w = warp - item0 % nwarps;
  if (w < 0) w += nwarps;
  for (int it = w; it < items; it += nwarps) {
    const int nt = it % NT, mp = it / NT;
    const int mt0 = 2 * mp, mt1 = 2 * mp + 1;
    const bool two = mt1 < MT;
    if (MMA) {
      double b[KMAX];
#pragma unroll
      for (int ks = 0; ks < KMAX; ++ks)
        if (ks < KS) b[ks] = Bf[(nt * KS + ks) * 32 + lane];
      const double* a0 = A + (mt0 * 8 + (lane >> 2)) * lda + a_k0 + (lane & 3);
      const double* a1 = a0 + 8 * lda;
      double c00 = 0, c01 = 0, c10 = 0, c11 = 0;
      // columns >= K of A are never read (their value would multiply a zero B
      // pad row, but stale shared memory may hold anything): masked to 0
#pragma unroll
      for (int ks = 0; ks < KMAX; ++ks) {
        if (ks < KS) {
          const bool kin = ks * 4 + (lane & 3) < K;
          dmma884(c00, c01, kin ? a0[ks * 4] : 0.0, b[ks]);
          if (two) dmma884(c10, c11, kin ? a1[ks * 4] : 0.0, b[ks]);
        }
      }
      const int col = nt * 8 + 2 * (lane & 3);
      store(mt0 * 8 + (lane >> 2), col, c00, c01);
      if (two) store(mt1 * 8 + (lane >> 2), col, c10, c11);
    } else {
      // DFMA: lane (r = lane/4, c = 2 (lane%4)) of each 8x8 tile accumulates
      // its two outputs; the B column pair comes from the fragment table
      // (element (k, n) of fragment (ks, nt) sits at lane' = (n%8)*4 + k%4).
      const int r = lane >> 2, cc = 2 * (lane & 3);
      const double* a0 = A + (mt0 * 8 + r) * lda + a_k0;
      const double* a1 = a0 + 8 * lda;
      double c00 = 0, c01 = 0, c10 = 0, c11 = 0;
      for (int ks = 0; ks < KS; ++ks) {
        const double* bf = Bf + (nt * KS + ks) * 32;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (ks * 4 + kk >= K) break;
          const double b0 = bf[cc * 4 + kk], b1 = bf[(cc + 1) * 4 + kk];
          const double x0 = a0[ks * 4 + kk];
          c00 = fma(x0, b0, c00);
          c01 = fma(x0, b1, c01);
          if (two) {
            const double x1 = a1[ks * 4 + kk];
            c10 = fma(x1, b0, c10);
            c11 = fma(x1, b1, c11);
          }
        }
      }
      store(mt0 * 8 + r, nt * 8 + cc, c00, c01);
      if (two) store(mt1 * 8 + r, nt * 8 + cc, c10, c11);
    }
  }
}

// ------------------------------------------------------------ the kernel
template <int P, int NWARP, bool MMA>
__global__ void __launch_bounds__(NWARP * 32, 1)
    k_sht(SelfArgs A, const double* __restrict__ sht_g) {
  constexpr ShtDims Dm(P);
  constexpr int P1 = P + 1, NP = 2 * P + 2, nsn = P1 * NP, SB = Dm.SB;
  constexpr int ldG = Dm.ldG, ldF = Dm.ldF, ldE = Dm.ldE;
  constexpr int nlm = P1 * (P1 + 1) / 2;
  constexpr int KMAX = (2 * P1 + 3) / 4 > 1 ? (2 * P1 + 3) / 4 : 1;
  constexpr int WPS = sht_wps(P), GROUPS = sht_groups(P), GT = WPS * 32;
  static_assert(NWARP == WPS * GROUPS, "launch geometry");
  extern __shared__ __align__(16) double sm[];
  const int group = (threadIdx.x >> 5) / WPS, gt = threadIdx.x % GT;  // group, thread in group
  double* G = sm + group * Dm.group + Dm.offG;   // [6 P1 SB (+8)][ldG]      phase A -> B
  double* FT = sm + group * Dm.group + Dm.offF;  // [P1][12 SB][ldF] (+8 rows)  B -> C
  double* AL = G;              // alpha partials (C -> C2), aliases G
  double* AD = FT;             // D-GEMM A operand (C2 -> D), aliases FT
  double* U = G;               // [3 P1 SB (+8)][ldG]       D -> E, aliases G
  double* EO = FT;             // [3 P1 SB][ldE] = [c_0..c_P1 | s_1..s_p]   E -> F
  double* trig = sm + Dm.offTrig;  // cos phi_k, sin phi_k (NP each), ct, st, wu (P1 each)
  double* degc = sm + Dm.offDeg;   // per degree n: lamS V W X, lamD V W X, 1/(n(n+1)), 1/(2n+1)
  int* mcode = reinterpret_cast<int*>(sm + Dm.offMC);  // coefficient c -> (m << 16) | (n - m)
  const ShtTabLayout TL(P);
  const int tid = threadIdx.x, nt = NWARP * 32;
  const double mu = A.mu;
  const double cS = 1.0 / (8.0 * kPi * mu), cD = 3.0 / (4.0 * kPi);
  const TableLayout L(P);
  const double* __restrict__ tab = A.tab;

  for (int e = tid; e < Dm.offTrig; e += nt) sm[e] = 0.0;  // every pad entry finite
  for (int k = tid; k < NP; k += nt) {
    trig[k] = tab[L.cph + k];
    trig[NP + k] = tab[L.sph + k];
  }
  for (int j = tid; j < P1; j += nt) {
    trig[2 * NP + j] = tab[L.t + j];
    trig[2 * NP + P1 + j] = tab[L.st + j];
    trig[2 * NP + 2 * P1 + j] = tab[L.wu + j];
    const int n = j;
    for (int q = 0; q < 3; ++q) {
      degc[8 * n + q] = tab[L.lamS + 3 * n + q];
      degc[8 * n + 3 + q] = tab[L.lamD + 3 * n + q];
    }
    degc[8 * n + 6] = n ? 1.0 / ((double)n * (n + 1)) : 0.0;
    degc[8 * n + 7] = 1.0 / (2.0 * n + 1.0);
  }
  for (int m = 0, c0 = 0; m <= P; c0 += P1 - m, ++m)
    for (int c = c0 + tid; c < c0 + P1 - m; c += nt) mcode[c] = (m << 16) | (c - c0);
  const double* sht = sht_g;
  if constexpr (sht_tab_smem(P)) {  // stage the transform tables once per CTA
    static_assert(sht_tab_doubles(P) % 2 == 0, "table size");
    double2* dst = reinterpret_cast<double2*>(sm + Dm.offTab);
    const double2* src = reinterpret_cast<const double2*>(sht_g);
    for (int e = tid; e < (int)(sht_tab_doubles(P) / 2); e += nt) dst[e] = src[e];
    sht = sm + Dm.offTab;
  }
  const double* cph = trig;
  const double* sph = trig + NP;
  const double* ctj = trig + 2 * NP;
  const double* stj = ctj + P1;
  const double* wuj = stj + P1;
  __syncthreads();

  // group barrier: the group's warps only (named barrier 1 + group)
  auto gsync = [&]() {
    if (WPS == 1) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(GT) : "memory");
  };
  const int64_t nbatch = (A.ns + SB - 1) / SB;
  const int64_t gstride = (int64_t)gridDim.x * GROUPS;
  for (int64_t bt = (int64_t)blockIdx.x * GROUPS + group; bt < nbatch; bt += gstride) {
    const int64_t s0 = bt * SB;
    const int nb = (int)min((int64_t)SB, A.ns - s0);
    if (gt == 0 && bt + gstride < nbatch) {  // this group's next sphere -> L2
      const int64_t s1 = (bt + gstride) * SB;
      const int n1 = (int)min((int64_t)SB, A.ns - s1);
      const uint32_t bytes = (uint32_t)(n1 * nsn * 24);
      if (A.f && !(reinterpret_cast<uintptr_t>(A.f) & 15)) bulk_prefetch_l2(A.f + s1 * nsn * 3, bytes);
      if (A.q && !(reinterpret_cast<uintptr_t>(A.q) & 15)) bulk_prefetch_l2(A.q + s1 * nsn * 3, bytes);
    }
    // ------------------------------------------------------------ A
    for (int it = gt; it < SB * P1 * (P1 + 1); it += GT) {
      const int b = it / (P1 * (P1 + 1));
      const int r = it - b * (P1 * (P1 + 1));
      const int j = r / (P1 + 1), k = r - j * (P1 + 1);
      const bool pair = k > 0 && k < P1;
      double g1[6], g2[6];
      if (b < nb) {
        const int64_t s = s0 + b;
        const double a = A.radii[s];
        const double cx = A.centres[3 * s], cy = A.centres[3 * s + 1], cz = A.centres[3 * s + 2];
        const double aS = a / mu, w = a * a * wuj[j];
        const double ws = w * cS, wd = w * cD;
        const double ct = ctj[j], stt = stj[j];
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          if (side == 1 && !pair) break;
          const int kk = side ? NP - k : k;
          const int64_t i = s * nsn + j * NP + kk;
          double f0 = 0, f1 = 0, f2 = 0, q0 = 0, q1 = 0, q2 = 0;
          if (A.f) { f0 = A.f[3 * i]; f1 = A.f[3 * i + 1]; f2 = A.f[3 * i + 2]; }
          if (A.q) { q0 = A.q[3 * i]; q1 = A.q[3 * i + 1]; q2 = A.q[3 * i + 2]; }
          const double cp = cph[kk], sp = sph[kk];
          const double n0 = stt * cp, n1 = stt * sp, n2 = ct;
          double2* r2 = reinterpret_cast<double2*>(A.rec + i * kRec);
          r2[0] = make_double2(cx + a * n0, cy + a * n1);
          r2[1] = make_double2(cz + a * n2, n0);
          r2[2] = make_double2(n1, n2);
          r2[3] = make_double2(ws * f0, ws * f1);
          r2[4] = make_double2(ws * f2, wd * q0);
          r2[5] = make_double2(wd * q1, wd * q2);
          double* g = side ? g2 : g1;
          g[0] = aS * (f0 * n0 + f1 * n1 + f2 * n2);
          g[1] = aS * (f0 * ct * cp + f1 * ct * sp - f2 * stt);
          g[2] = aS * (-f0 * sp + f1 * cp);
          g[3] = q0 * n0 + q1 * n1 + q2 * n2;
          g[4] = q0 * ct * cp + q1 * ct * sp - q2 * stt;
          g[5] = -q0 * sp + q1 * cp;
        }
      } else {
#pragma unroll
        for (int d = 0; d < 6; ++d) g1[d] = g2[d] = 0.0;
      }
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        double* row = G + ((b * 6 + d) * P1 + j) * ldG;
        if (k == 0) row[0] = g1[d];
        else if (k == P1) row[1] = g1[d];
        else {
          row[1 + k] = g1[d] + g2[d];   // S_k
          row[P1 + k] = g1[d] - g2[d];  // D_k
        }
      }
    }
    if (!A.self && !A.alpha) {  // pack only (+ zero u)
      if (A.u)
        for (int64_t e = gt; e < (int64_t)nb * 3 * nsn; e += GT) A.u[s0 * 3 * nsn + e] = 0.0;
      gsync();
      continue;
    }
    gsync();
    // ------------------------------------------------------------ B
    // rows (b, d, j) of G -> FT[m][row(b, dens, comp, ri)][j]
    {
      auto ftrow = [](int b, int d, int ri) {
        const int dens = d / 3, comp = d - 3 * dens;
        return comp == 0 ? (b * 2 + dens) * 2 + ri : 4 * SB + ((b * 2 + dens) * 2 + comp - 1) * 2 + ri;
      };
      constexpr int M = 6 * P1 * SB;
      auto st_re = [&](int row, int col, double v0, double v1) {
        if (row >= M) return;
        const int j = row % P1, bd = row / P1, b = bd / 6, d = bd - 6 * b;
        const int fr = ftrow(b, d, 0);
        if (col < P1) FT[(col * 12 * SB + fr) * ldF + j] = v0;
        if (col + 1 < P1) FT[((col + 1) * 12 * SB + fr) * ldF + j] = v1;
      };
      auto st_im = [&](int row, int col, double v0, double v1) {
        if (row >= M) return;
        const int j = row % P1, bd = row / P1, b = bd / 6, d = bd - 6 * b;
        const int fr = ftrow(b, d, 1);
        if (col < P1) FT[(col * 12 * SB + fr) * ldF + j] = v0;
        if (col + 1 < P1) FT[((col + 1) * 12 * SB + fr) * ldF + j] = v1;
      };
      sht_gemm<MMA, KMAX>(G, ldG, 0, M, P1 + 1, sht + TL.Tc, TL.KSc, TL.NTc, st_re, 0, WPS);
      sht_gemm<MMA, KMAX>(G, ldG, P1 + 1, M, P, sht + TL.Ts, TL.KSs, TL.NTs, st_im,
                          TL.NTc * ((M + 15) / 16), WPS);
    }
    gsync();
    // ------------------------------------------------------------ C
    // alpha block of order m (compact): Y [4 SB][n], then PD|PM [8 SB][2n]
    {
      int item0 = 0;
      int64_t aoff = 0;
      for (int m = 0; m <= P; ++m) {
        const int n = P1 - m;
        const int64_t oCY = (int64_t)sht[TL.mtab + 4 * m];
        const int64_t oCGX = (int64_t)sht[TL.mtab + 4 * m + 1];
        double* aY = AL + aoff;
        double* aX = aY + 4 * SB * n;
        const double* Fm = FT + m * 12 * SB * ldF;
        auto stY = [&](int row, int col, double v0, double v1) {
          if (row >= 4 * SB) return;
          if (col < n) aY[row * n + col] = v0;
          if (col + 1 < n) aY[row * n + col + 1] = v1;
        };
        auto stX = [&](int row, int col, double v0, double v1) {
          if (row >= 8 * SB) return;
          if (col < 2 * n) aX[row * 2 * n + col] = v0;
          if (col + 1 < 2 * n) aX[row * 2 * n + col + 1] = v1;
        };
        const int NTy = (n + 7) / 8, NTx = (2 * n + 7) / 8, KSc = (P1 + 3) / 4;
        sht_gemm<MMA, KMAX>(Fm, ldF, 0, 4 * SB, P1, sht + oCY, KSc, NTy, stY, item0, WPS);
        item0 += NTy * ((4 * SB + 15) / 16);
        sht_gemm<MMA, KMAX>(Fm + 4 * SB * ldF, ldF, 0, 8 * SB, P1, sht + oCGX, KSc, NTx, stX, item0, WPS);
        item0 += NTx * ((8 * SB + 15) / 16);
        aoff += 20 * SB * n;
      }
    }
    gsync();
    // ------------------------------------------------------------ C2
    // per (b, n, m): {Y, G, X} of both densities -> psi (Thm 2) -> D-GEMM A:
    //   AD[m] = [ Y rows (b, ri) [2 SB][KY] | GX rows (b, th re/im, ph re/im) [4 SB][KX] ]
    constexpr int KY = Dm.KY, KX = Dm.KX, ADm = Dm.ADm;  // row strides, doubles per m block
    for (int it = gt; it < SB * nlm; it += GT) {
      const int b = it / nlm;
      const int cidx = it - b * nlm;
      const int code = mcode[cidx];
      const int m = code >> 16, c = code & 0xFFFF;
      const int n = P1 - m, deg = m + c;
      const int aoff = 20 * SB * (m * P1 - m * (m - 1) / 2);  // 20 SB sum_{m' < m} (P1 - m')
      const double* aY = AL + aoff;
      const double* aX = aY + 4 * SB * n;
      double ph[2][6];  // [dens][Y re, Y im, G re, G im, X re, X im] (raw projections)
#pragma unroll
      for (int dens = 0; dens < 2; ++dens) {
        const int ry = (b * 2 + dens) * 2;
        const int rx = (b * 2 + dens) * 2 * 2;  // th re, th im, ph re, ph im rows
        const double Yre = aY[ry * n + c], Yim = aY[(ry + 1) * n + c];
        const double* thr = aX + (rx + 0) * 2 * n;
        const double* thi = aX + (rx + 1) * 2 * n;
        const double* phr = aX + (rx + 2) * 2 * n;
        const double* phi = aX + (rx + 3) * 2 * n;
        ph[dens][0] = Yre;
        ph[dens][1] = Yim;
        ph[dens][2] = thr[c] + phi[n + c];  // <F,G> re: dP F_th^re + mP F_ph^im
        ph[dens][3] = thi[c] - phr[n + c];  //        im: dP F_th^im - mP F_ph^re
        ph[dens][4] = phr[c] - thi[n + c];  // <F,X> re: dP F_ph^re - mP F_th^im
        ph[dens][5] = phi[c] + thr[n + c];  //        im: dP F_ph^im + mP F_th^re
      }
      const int64_t s = s0 + b;
      if (A.alpha && b < nb) {
        const int cc = lm_index(P, deg, m);
#pragma unroll
        for (int dens = 0; dens < 2; ++dens) {
          double2* g2 = reinterpret_cast<double2*>(A.alpha + (s * 2 * nlm + dens * nlm + cc) * 6);
          g2[0] = make_double2(ph[dens][0], ph[dens][1]);
          g2[1] = make_double2(ph[dens][2], ph[dens][3]);
          g2[2] = make_double2(ph[dens][4], ph[dens][5]);
        }
      }
      if (!A.self) continue;
      const double* lS = degc + 8 * deg;
      const double* lD = lS + 3;
      const double inn = lS[6], i2n = lS[7];
      double psi[6];
#pragma unroll
      for (int ri = 0; ri < 2; ++ri) {
        double aV[2], aW[2], aXx[2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          const double phY = ph[d][ri], phG = ph[d][2 + ri] * inn, phX = ph[d][4 + ri] * inn;
          aV[d] = (deg * phG - phY) * i2n;        // eq 2.13
          aW[d] = ((deg + 1) * phG + phY) * i2n;  // eq 2.14
          aXx[d] = phX;
        }
        double psV, psW, psX;
        if (A.precond) {  // (1/sigma - 2) on the degree-<=p modes; + 2 q added in phase F
          const double aS = b < nb ? A.radii[s] / mu : 0.0;
          psV = (1.0 / (0.5 + lS[0] * aS + lD[0]) - 2.0) * aV[1];
          psW = deg ? (1.0 / (0.5 + lS[1] * aS + lD[1]) - 2.0) * aW[1] : 0.0;
          psX = deg ? (1.0 / (0.5 + lS[2] * aS + lD[2]) - 2.0) * aXx[1] : 0.0;
        } else {
          // (a/mu) is already folded into the f channels in phase A
          psV = lS[0] * aV[0] + lD[0] * aV[1];
          psW = lS[1] * aW[0] + lD[1] * aW[1];
          psX = lS[2] * aXx[0] + lD[2] * aXx[1];
        }
        psi[0 + ri] = -(deg + 1.0) * psV + deg * psW;  // psi^Y (eq 2.17)
        psi[2 + ri] = psV + psW;                      // psi^G (eq 2.16)
        psi[4 + ri] = psX;                            // psi^X
      }
      if (A.self == 2)  // neighbours' coefficients alone (apply of the FAR part in NEXT-4 mode)
#pragma unroll
        for (int k = 0; k < 6; ++k) psi[k] = 0.0;
      if (A.psinear && b < nb) {  // NEXT-4: neighbours' coefficients
        const double* pn = A.psinear + (s * nlm + lm_index(P, deg, m)) * 6;
#pragma unroll
        for (int k = 0; k < 6; ++k) psi[k] += pn[k];
      }
      double* Am = AD + m * ADm;
      double* Ay = Am;                 // [2 SB][KY]
      double* Ax = Am + 2 * SB * KY;   // [4 SB][KX]
      Ay[(b * 2 + 0) * KY + c] = psi[0];
      Ay[(b * 2 + 1) * KY + c] = psi[1];
      // th re: [G re | X im]; th im: [G im | -X re]; ph re: [X re | -G im]; ph im: [X im | G re]
      Ax[(b * 4 + 0) * KX + c] = psi[2];
      Ax[(b * 4 + 0) * KX + n + c] = psi[5];
      Ax[(b * 4 + 1) * KX + c] = psi[3];
      Ax[(b * 4 + 1) * KX + n + c] = -psi[4];
      Ax[(b * 4 + 2) * KX + c] = psi[4];
      Ax[(b * 4 + 2) * KX + n + c] = -psi[3];
      Ax[(b * 4 + 3) * KX + c] = psi[5];
      Ax[(b * 4 + 3) * KX + n + c] = psi[2];
    }
    if (!A.self) {
      if (A.u)
        for (int64_t e = gt; e < (int64_t)nb * 3 * nsn; e += GT) A.u[s0 * 3 * nsn + e] = 0.0;
      gsync();
      continue;
    }
    gsync();
    // ------------------------------------------------------------ D
    // U rows (b, comp, j): [Re U_0..p | Im U_0..p]
    {
      int item0 = 0;
      for (int m = 0; m <= P; ++m) {
        const int n = P1 - m;
        const int64_t oDY = (int64_t)sht[TL.mtab + 4 * m + 2];
        const int64_t oDGX = (int64_t)sht[TL.mtab + 4 * m + 3];
        const double* Am = AD + m * ADm;
        auto stY = [&](int row, int col, double v0, double v1) {  // row = (b, ri), col = j
          if (row >= 2 * SB) return;
          const int b = row >> 1, ri = row & 1;
          if (col < P1) U[((b * 3 + 0) * P1 + col) * ldG + ri * P1 + m] = v0;
          if (col + 1 < P1) U[((b * 3 + 0) * P1 + col + 1) * ldG + ri * P1 + m] = v1;
        };
        auto stX = [&](int row, int col, double v0, double v1) {  // row = (b, th/ph re/im)
          if (row >= 4 * SB) return;
          const int b = row >> 2, kind = row & 3, comp = 1 + (kind >> 1), ri = kind & 1;
          if (col < P1) U[((b * 3 + comp) * P1 + col) * ldG + ri * P1 + m] = v0;
          if (col + 1 < P1) U[((b * 3 + comp) * P1 + col + 1) * ldG + ri * P1 + m] = v1;
        };
        const int NTj = (P1 + 7) / 8;
        sht_gemm<MMA, KMAX>(Am, KY, 0, 2 * SB, n, sht + oDY, (n + 3) / 4, NTj, stY, item0, WPS);
        item0 += NTj * ((2 * SB + 15) / 16);
        sht_gemm<MMA, KMAX>(Am + 2 * SB * KY, KX, 0, 4 * SB, 2 * n, sht + oDGX, (2 * n + 3) / 4, NTj, stX,
                            item0, WPS);
        item0 += NTj * ((4 * SB + 15) / 16);
      }
    }
    gsync();
    // ------------------------------------------------------------ E
    {
      constexpr int M = 3 * P1 * SB;
      auto stc = [&](int row, int col, double v0, double v1) {
        if (row >= M) return;
        if (col <= P1) EO[row * ldE + col] = v0;
        if (col + 1 <= P1) EO[row * ldE + col + 1] = v1;
      };
      auto sts = [&](int row, int col, double v0, double v1) {  // s_{col+1}
        if (row >= M) return;
        if (col < P) EO[row * ldE + P1 + 1 + col] = v0;
        if (col + 1 < P) EO[row * ldE + P1 + 2 + col] = v1;
      };
      sht_gemm<MMA, KMAX>(U, ldG, 0, M, P1, sht + TL.Ec, TL.KEc, TL.NEc, stc, 0, WPS);
      sht_gemm<MMA, KMAX>(U, ldG, P1 + 1, M, P, sht + TL.Es, TL.KEs, TL.NEs, sts,
                          TL.NEc * ((M + 15) / 16), WPS);
    }
    gsync();
    // ------------------------------------------------------------ F
    for (int it = gt; it < nb * nsn; it += GT) {
      const int b = it / nsn, r = it - b * nsn;
      const int j = r / NP, kk = r - j * NP;
      double v[3];
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) {
        const double* e = EO + ((b * 3 + comp) * P1 + j) * ldE;
        if (kk <= P1) v[comp] = e[kk] - ((kk >= 1 && kk <= P) ? e[P1 + kk] : 0.0);
        else v[comp] = e[NP - kk] + e[P1 + NP - kk];
      }
      const double cp = cph[kk], sp = sph[kk], ct = ctj[j], stt = stj[j];
      const int64_t i = (s0 + b) * nsn + r;
      double w0 = v[0] * stt * cp + v[1] * ct * cp - v[2] * sp;
      double w1 = v[0] * stt * sp + v[1] * ct * sp + v[2] * cp;
      double w2 = v[0] * ct - v[1] * stt;
      if (A.precond) {
        w0 = fma(2.0, A.q[3 * i + 0], w0);
        w1 = fma(2.0, A.q[3 * i + 1], w1);
        w2 = fma(2.0, A.q[3 * i + 2], w2);
      }
      A.u[3 * i + 0] = w0;
      A.u[3 * i + 1] = w1;
      A.u[3 * i + 2] = w2;
    }
    gsync();
  }
}

// ------------------------------------------------------------ launch
// variant: 0 = DMMA GEMMs (default), 1 = DFMA GEMMs (same schedule; compiled
// for the BASELINE orders p in {4, 6, 8, 12}, others use DMMA).
__host__ __device__ constexpr int sht_threads(int p) { return 32 * sht_wps(p) * sht_groups(p); }

template <int P, bool MMA>
struct ShtKernel {
  static constexpr int kWarps = sht_wps(P) * sht_groups(P);
  static void* fn() { return (void*)k_sht<P, kWarps, MMA>; }
  static size_t smem() { return (size_t)ShtDims(P).total * sizeof(double); }
};

inline void* sht_kernel(int p, int variant, size_t* smem) {
  const bool dfma = variant == 1 && (p == 4 || p == 6 || p == 8 || p == 12);
#define BIE_SHT_CASE(PP)                                   \
  case PP:                                                 \
    *smem = ShtKernel<PP, true>::smem();                   \
    return ShtKernel<PP, true>::fn();
#define BIE_SHT_CASE2(PP)                                  \
  case PP:                                                 \
    *smem = ShtKernel<PP, true>::smem();                   \
    return dfma ? ShtKernel<PP, false>::fn() : ShtKernel<PP, true>::fn();
  switch (p) {
    BIE_SHT_CASE(1) BIE_SHT_CASE(2) BIE_SHT_CASE(3) BIE_SHT_CASE2(4) BIE_SHT_CASE(5)
    BIE_SHT_CASE2(6) BIE_SHT_CASE(7) BIE_SHT_CASE2(8) BIE_SHT_CASE(9) BIE_SHT_CASE(10)
    BIE_SHT_CASE(11) BIE_SHT_CASE2(12) BIE_SHT_CASE(13) BIE_SHT_CASE(14) BIE_SHT_CASE(15)
    BIE_SHT_CASE(16) BIE_SHT_CASE(17) BIE_SHT_CASE(18) BIE_SHT_CASE(19) BIE_SHT_CASE(20)
    BIE_SHT_CASE(21) BIE_SHT_CASE(22) BIE_SHT_CASE(23) BIE_SHT_CASE(24) BIE_SHT_CASE(25)
    BIE_SHT_CASE(26) BIE_SHT_CASE(27) BIE_SHT_CASE(28) BIE_SHT_CASE(29) BIE_SHT_CASE(30)
    BIE_SHT_CASE(31) BIE_SHT_CASE(32)
    default: *smem = 0; return nullptr;
  }
#undef BIE_SHT_CASE
#undef BIE_SHT_CASE2
}

// Opt in to the dynamic shared memory of both variants for order p; returns
// the resident CTAs per SM of the DMMA variant (the grid is sized from it).
inline int sht_prepare(int p) {
  if (sht_tab_doubles(p) != ShtTabLayout(p).total) return 0;  // layouts must agree
  int occ = 1;
  for (int v = 1; v >= 0; --v) {
    size_t smem = 0;
    void* fn = sht_kernel(p, v, &smem);
    if (!fn) return 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (v == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, sht_threads(p), smem);
  }
  return occ > 0 ? occ : 1;
}

// grid: one persistent CTA per resident slot (or fewer when there are fewer batches)
inline cudaError_t launch_sht(const SelfArgs& A, const double* sht, int variant, int sm_count, int occ,
                              cudaStream_t s) {
  size_t smem = 0;
  void* fn = sht_kernel(A.p, variant, &smem);
  if (!fn) return cudaErrorInvalidValue;
  const int64_t nbatch = (A.ns + sht_sb(A.p) - 1) / sht_sb(A.p);
  const int64_t ngroups = (nbatch + sht_groups(A.p) - 1) / sht_groups(A.p);
  const unsigned grid = (unsigned)std::min<int64_t>(ngroups, (int64_t)sm_count * occ);
  SelfArgs a = A;
  const double* t = sht;
  void* args[] = {&a, &t};
  return cudaLaunchKernel(fn, dim3(grid), dim3(sht_threads(A.p)), args, smem, s);
}

}  // namespace bie
