// k_nbody.cuh -- fused Stokeslet + stresslet fp64 N-body sum (rows a3, a7).
//
// u_i += sum_k y_k [ f'_k + rho (rho.f'_k + (rho.n_k)(rho.q'_k) y_k^2) y_k^2 ],
//   rho = x_i - x_k, y_k = 1/|rho|, f' = w f/(8 pi mu), q' = (3/(4 pi)) w q,
// which is S[f] (eq 2.19) + D[q] (eq 2.20 with sign reading R1) under the
// smooth rule (eq 4.4).  30 FP64 pipe instructions per pair (18 DFMA, 9 DMUL,
// 3 DADD); the reciprocal square root is a MUFU seed plus one third-order
// fp64 refinement y = y0 + y0 e (1/2 + 3/8 e), e = 1 - r^2 y0^2.
// Off-surface (a7) adds the pressure p += (t2 - qn3_k) y^3 (2 more ops).
//
// Decomposition: CTA = (target tile of TPB*R targets, source chunk).  Source
// tiles of TS packed records (96 B each) stream global -> shared through the
// TMA bulk-copy unit into an NST-deep ring guarded by mbarriers; every thread
// holds R targets in registers and reads each source once from shared memory
// (broadcast LDS.128).  Self-sphere exclusion (reading R8) is a per-pair
// select applied only in source tiles that overlap the CTA's own spheres.
// Chunk partials are reduced in fixed order by k_reduce (deterministic).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"


namespace bie {

struct NbodyArgs {
  const double* rec;    // [N][kRec] sources
  const double* qn3;    // [N (+pad)] (off-surface pressure only)
  const double* tx;     // [M][3] targets (off-surface) or nullptr (targets = source nodes)
  const double* uinit;  // [M][3] added when n_chunks == 1 (self term), may be nullptr
  double* uout;         // n_chunks == 1: [M][3] final; else partial base [n_chunks][M][3]
  double* pout;         // off-surface: n_chunks == 1: [M]; else [n_chunks][M]; may be nullptr
  int64_t N;            // number of sources
  int64_t M;            // number of targets
  int nsn;              // nodes per sphere (masking)
  int n_tt;             // target tiles
  int n_chunks;         // source chunks
  int tiles_per_chunk;  // source tiles per chunk
  double pscale;        // 2 mu (pressure)
  const double* tn = nullptr;  // [M][3] target normals (off-surface traction, OFF && MODE 1)
  // NX (near exclusion, apply only): CSR eq-4.5 neighbour lists per sphere; the
  // smooth rule skips the pairs of near spheres, whose exact field the near
  // correction adds (so nothing has to be subtracted afterwards)
  const int* nb_off = nullptr;
  const int* nb_idx = nullptr;
  // Chained chunk reduction (CL 1, n_chunks > 1, chain != nullptr): CTAs take
  // their (chunk, target tile) from a ticket counter chain[n_tt] in chunk-major
  // order; chunk c of tile t waits until chain[t] == c, adds its partial to the
  // running sum cacc (c = 0 stores it), and releases chain[t] = c + 1; the last
  // chunk writes uout (+ uinit) and pout.  The sum order is k_reduce's (fixed:
  // chunk 0, 1, ...), so results are deterministic, and no chunk partials reach
  // HBM beyond one running sum per target.  chain[0 .. n_tt] zeroed per launch.
  int* chain = nullptr;
  double* cacc = nullptr;  // [M][3] running sums (+ [M] pressure after them, OFF)
  // apply kernels: targets (and, for K, their normals) read from these compact
  // [M][3] arrays instead of the 96-byte records (one sector per target instead
  // of two); nullptr: from the records
  const double* txa = nullptr;
  const double* tna = nullptr;
};

// shared memory of the NX variant beyond the ring: the CTA's excluded-sphere
// table -- (sphere, bitmask of the tile's target spheres that exclude it),
// sorted by sphere -- staging for it, a count and one masked flag per stage
constexpr int kNxCap = 256;     // table entries (overflow: per-pair neighbour-list lookups)
constexpr int kNxTiles = 4096;  // masked-tile bitmap of the CTA's source range (else search)
constexpr int kNxBytes = kNxCap * (4 + 8) * 2 + kNxTiles / 8 + 32;

// first index of the sorted table xs[0..n) with xs[i] >= v
__device__ __forceinline__ int nx_lower(const int* xs, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (xs[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int TS, int NST, bool OFF>
struct NbodySmem {
  static constexpr int kRecBytes = TS * kRec * 8;
  static constexpr int kQnBytes = OFF ? TS * 8 : 0;
  static constexpr int kStageBytes = kRecBytes + kQnBytes;
  static constexpr int kBytes = NST * kStageBytes + NST * 8;
};

template <bool MASK, bool OFF>
__device__ __forceinline__ void pair_acc(const double2 s0, const double2 s1, const double2 s2,
                                         const double2 s3, const double2 s4, const double2 s5,
                                         double qn, const double* xt, double* acc, double& pacc,
                                         int k, int lo, int nsn) {
  // s0=(x0,x1) s1=(x2,n0) s2=(n1,n2) s3=(f0,f1) s4=(f2,q0) s5=(q1,q2)
  const double dx = xt[0] - s0.x, dy = xt[1] - s0.y, dz = xt[2] - s1.x;
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double y0 = rsqrt_seed(r2);
  const double e = fma(-r2, y0 * y0, 1.0);
  // y = y0 (1 + e (1/2 + 3/8 e)): every DFMA here has an immediate operand, so
  // none needs three fresh 64-bit register reads (RF model).
  double y = y0 * fma(e, fma(e, 0.375, 0.5), 1.0);
  if (MASK) {
    if ((unsigned)(k - lo) < (unsigned)nsn) y = 0.0;  // own sphere: excluded (R8)
  }
  const double rf = fma(dz, s4.x, fma(dy, s3.y, dx * s3.x));
  const double rn = fma(dz, s2.y, fma(dy, s2.x, dx * s1.y));
  const double rq = fma(dz, s5.y, fma(dy, s5.x, dx * s4.y));
  const double y2 = y * y;
  const double t2 = fma(rn * rq, y2, rf);
  const double sp = t2 * y2;
  acc[0] = fma(y, fma(dx, sp, s3.x), acc[0]);
  acc[1] = fma(y, fma(dy, sp, s3.y), acc[1]);
  acc[2] = fma(y, fma(dz, sp, s4.x), acc[2]);
  if (OFF) pacc = fma(fma(-qn, y2, sp), y, pacc);
}


// pair_acc for G targets at once, written stage by stage (every target's
// differences, then |rho|^2, the reciprocal root, each dot product, ...).  Same
// arithmetic and rounding as G calls of pair_acc; the form gives ptxas a
// register allocation of the hot loop that measured 0.9 % faster after the
// chained reduction was added (tools/nbody_rf.py).
template <int G, bool OFF>
__device__ __forceinline__ void pair_acc_g(const double2 s0, const double2 s1, const double2 s2,
                                           const double2 s3, const double2 s4, const double2 s5,
                                           double qn, const double (*xt)[3], double (*acc)[3], double* pacc) {
  double dx[G], dy[G], dz[G], r2[G], y[G], rf[G], rn[G], rq[G], y2[G], sp[G];
#pragma unroll
  for (int g = 0; g < G; ++g) dx[g] = xt[g][0] - s0.x;
#pragma unroll
  for (int g = 0; g < G; ++g) dy[g] = xt[g][1] - s0.y;
#pragma unroll
  for (int g = 0; g < G; ++g) dz[g] = xt[g][2] - s1.x;
#pragma unroll
  for (int g = 0; g < G; ++g) r2[g] = fma(dz[g], dz[g], fma(dy[g], dy[g], dx[g] * dx[g]));
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const double y0 = rsqrt_seed(r2[g]);
    const double e = fma(-r2[g], y0 * y0, 1.0);
    y[g] = y0 * fma(e, fma(e, 0.375, 0.5), 1.0);
  }
#pragma unroll
  for (int g = 0; g < G; ++g) rf[g] = dx[g] * s3.x;
#pragma unroll
  for (int g = 0; g < G; ++g) rf[g] = fma(dy[g], s3.y, rf[g]);
#pragma unroll
  for (int g = 0; g < G; ++g) rf[g] = fma(dz[g], s4.x, rf[g]);
#pragma unroll
  for (int g = 0; g < G; ++g) rn[g] = dx[g] * s1.y;
#pragma unroll
  for (int g = 0; g < G; ++g) rn[g] = fma(dy[g], s2.x, rn[g]);
#pragma unroll
  for (int g = 0; g < G; ++g) rn[g] = fma(dz[g], s2.y, rn[g]);
#pragma unroll
  for (int g = 0; g < G; ++g) rq[g] = dx[g] * s4.y;
#pragma unroll
  for (int g = 0; g < G; ++g) rq[g] = fma(dy[g], s5.x, rq[g]);
#pragma unroll
  for (int g = 0; g < G; ++g) rq[g] = fma(dz[g], s5.y, rq[g]);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    y2[g] = y[g] * y[g];
    sp[g] = fma(rn[g] * rq[g], y2[g], rf[g]) * y2[g];
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    acc[g][0] = fma(y[g], fma(dx[g], sp[g], s3.x), acc[g][0]);
    acc[g][1] = fma(y[g], fma(dy[g], sp[g], s3.y), acc[g][1]);
    acc[g][2] = fma(y[g], fma(dz[g], sp[g], s4.x), acc[g][2]);
    if (OFF) pacc[g] = fma(fma(-qn, y2[g], sp[g]), y[g], pacc[g]);
  }
}

// Traction operator K (NEXT-3, eq 2.22 with reading R21): target normal nx,
//   u_i -= (rho.n_x)(rho.q'_k) rho y^5,  q' = (3/(4 pi)) w sigma  (25 FP64 ops).
template <bool MASK>
__device__ __forceinline__ void pair_K(const double2 s0, const double2 s1, const double2 s4,
                                       const double2 s5, const double* xt, const double* nx,
                                       double* acc, int k, int lo, int nsn) {
  const double dx = xt[0] - s0.x, dy = xt[1] - s0.y, dz = xt[2] - s1.x;
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double y0 = rsqrt_seed(r2);
  const double e = fma(-r2, y0 * y0, 1.0);
  double y = y0 * fma(e, fma(e, 0.375, 0.5), 1.0);
  if (MASK) {
    if ((unsigned)(k - lo) < (unsigned)nsn) y = 0.0;  // own sphere: excluded (R8)
  }
  const double rq = fma(dz, s5.y, fma(dy, s5.x, dx * s4.y));
  const double rn = fma(dz, nx[2], fma(dy, nx[1], dx * nx[0]));
  const double y2 = y * y;
  const double t = (rn * rq) * (y2 * y2);
  const double sm = -t * y;
  acc[0] = fma(dx, sm, acc[0]);
  acc[1] = fma(dy, sm, acc[1]);
  acc[2] = fma(dz, sm, acc[2]);
}

// MODE 0: S + D (rows a3, a7); MODE 1: traction operator K (apply, or off-surface
// targets with normals A.tn when OFF).
// CL > 1: the CL source chunks of one target tile form a thread-block cluster
// (launched with cluster dims (CL,1,1); chunk = cluster rank) and their partial
// sums are reduced on chip through distributed shared memory, in fixed rank
// order (deterministic), by the cluster itself -- no partials in HBM and no
// k_reduce launch.  CL = 1: chunk partials go to HBM for k_reduce.
// NX (apply only, MODE 0, CL 1): pairs whose source sphere is the target's own
// OR one of its eq-4.5 near neighbours are excluded from the smooth sum (the
// near correction then adds only the exact exterior field).
template <int R, int TPB, int TS, int NST, bool OFF, int MINB = 1, int UNR = 2, int MODE = 0, int CL = 1,
          bool NX = false>
__global__ void __launch_bounds__(TPB, MINB) k_nbody(const NbodyArgs A) {
  using SM = NbodySmem<TS, NST, OFF>;
  static_assert(!NX || (!OFF && CL == 1), "near exclusion: apply kernels (S+D, K) only");
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + NST * SM::kStageBytes);
  // NX tables (after the ring): sorted spheres xs, their target-sphere masks xm,
  // unsorted staging (us, um), [0] count (-1: overflow), per-stage masked flags
  uint64_t* xm = reinterpret_cast<uint64_t*>(smraw + SM::kBytes);
  uint64_t* um = xm + kNxCap;
  int* xs = reinterpret_cast<int*>(um + kNxCap);
  int* us = xs + kNxCap;
  int* xinfo = us + kNxCap;
  unsigned char* mflag = reinterpret_cast<unsigned char*>(xinfo + 2);
  uint32_t* tbits = reinterpret_cast<uint32_t*>(xinfo + 4);  // masked tiles of [tile0, tile0 + ntile)

  __shared__ int s_ticket;
  int unit = (int)blockIdx.x;
  if (CL == 1 && A.chain != nullptr && A.n_chunks > 1) {
    // chained reduction: ticket order (every lower ticket belongs to a CTA
    // already running); the epilogue re-reads the ticket from shared memory so
    // that nothing of it stays live in registers across the pair loop
    if (threadIdx.x == 0) s_ticket = atomicAdd(A.chain + A.n_tt, 1);
    __syncthreads();
    unit = s_ticket;
  }
  const int tt = CL > 1 ? (int)(blockIdx.x / CL) : unit % A.n_tt;
  const int chunk = CL > 1 ? (int)(blockIdx.x % CL) : unit / A.n_tt;
  const int64_t n_src_tiles = (A.N + TS - 1) / TS;
  const int64_t tile0 = (int64_t)chunk * A.tiles_per_chunk;
  int ntile = (int)min((int64_t)A.tiles_per_chunk, n_src_tiles - tile0);
  if (ntile < 0) ntile = 0;

  // ---- targets held in registers
  double xt[R][3], acc[R][3], pacc[R];
  double nx[MODE == 1 ? R : 1][3];
  int lo[R];
  int64_t tidx[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int64_t i = (int64_t)tt * TPB * R + r * TPB + threadIdx.x;
    tidx[r] = i;
    const int64_t ic = i < A.M ? i : A.M - 1;
    if (OFF) {
      xt[r][0] = A.tx[3 * ic];
      xt[r][1] = A.tx[3 * ic + 1];
      xt[r][2] = A.tx[3 * ic + 2];
      lo[r] = 0;
      if (MODE == 1) {
        nx[MODE == 1 ? r : 0][0] = A.tn[3 * ic];
        nx[MODE == 1 ? r : 0][1] = A.tn[3 * ic + 1];
        nx[MODE == 1 ? r : 0][2] = A.tn[3 * ic + 2];
      }
    } else if (A.txa) {
      xt[r][0] = A.txa[3 * ic];
      xt[r][1] = A.txa[3 * ic + 1];
      xt[r][2] = A.txa[3 * ic + 2];
      lo[r] = (int)((ic / A.nsn) * A.nsn);
      if (MODE == 1) {
        nx[MODE == 1 ? r : 0][0] = A.tna[3 * ic];
        nx[MODE == 1 ? r : 0][1] = A.tna[3 * ic + 1];
        nx[MODE == 1 ? r : 0][2] = A.tna[3 * ic + 2];
      }
    } else {
      xt[r][0] = A.rec[ic * kRec];
      xt[r][1] = A.rec[ic * kRec + 1];
      xt[r][2] = A.rec[ic * kRec + 2];
      lo[r] = (int)((ic / A.nsn) * A.nsn);
      if (MODE == 1) {
        nx[MODE == 1 ? r : 0][0] = A.rec[ic * kRec + 3];
        nx[MODE == 1 ? r : 0][1] = A.rec[ic * kRec + 4];
        nx[MODE == 1 ? r : 0][2] = A.rec[ic * kRec + 5];
      }
    }
    acc[r][0] = acc[r][1] = acc[r][2] = 0.0;
    pacc[r] = 0.0;
  }
  // CTA-uniform node range of the spheres owning this tile's targets
  int64_t first = (int64_t)tt * TPB * R;
  int64_t last = min(first + TPB * R, A.M) - 1;
  const int64_t cta_lo = (first / A.nsn) * A.nsn;
  const int64_t cta_hi = (last / A.nsn + 1) * A.nsn;

  const int t_lo = (int)(first / A.nsn);  // first target sphere of the tile
  if constexpr (NX) {
    // excluded-sphere table of the tile's targets (their own spheres and their
    // eq-4.5 neighbours), each entry tagged with the bit of the target sphere
    // that excludes it; rank-sorted by sphere (ties by position) by all threads
    if (threadIdx.x == 0) {
      int n = 0;
      bool over = false;
      for (int64_t t = t_lo; t <= last / A.nsn; ++t) {
        const uint64_t bit = 1ull << (t - t_lo);
        if (n < kNxCap) { us[n] = (int)t; um[n] = bit; ++n; } else over = true;
        for (int q = A.nb_off[t]; q < A.nb_off[t + 1]; ++q) {
          if (n < kNxCap) { us[n] = A.nb_idx[q]; um[n] = bit; ++n; } else over = true;
        }
      }
      xinfo[0] = over ? -1 : n;
    }
    __syncthreads();
    const int n = xinfo[0];
    for (int i = threadIdx.x; i < n; i += TPB) {
      const int v = us[i];
      int rank = 0;
      for (int j = 0; j < n; ++j) rank += (us[j] < v) || (us[j] == v && j < i);
      xs[rank] = v;
      xm[rank] = um[i];
    }
    // masked-tile bitmap of this CTA's source tiles (each thread one word)
    if (ntile <= kNxTiles) {
      for (int w = threadIdx.x; w < (ntile + 31) / 32; w += TPB) tbits[w] = 0u;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += TPB) {  // tiles of excluded sphere xs[i]
        const int64_t ta = (int64_t)xs[i] * A.nsn / TS - tile0;
        const int64_t tb = ((int64_t)(xs[i] + 1) * A.nsn - 1) / TS - tile0;
        for (int64_t t = max(ta, (int64_t)0); t <= min(tb, (int64_t)ntile - 1); ++t)
          atomicOr(&tbits[t >> 5], 1u << (t & 31));
      }
    }
    __syncthreads();
  }
  // Records: plain LRU.  In chunk-major order a chunk's records (4.7 MB on
  // cfg 5) are re-read by every target tile of the pass and stay hot anyway;
  // evict_last would pin all passes' records (94 MB) and push out the targets
  // and running sums, which are re-read once per pass (measured: off-surface
  // DRAM traffic 848 -> 330 MB per launch).
  const uint64_t pol = l2_evict_normal_policy();
  auto issue = [&](int it) {
    const int st = it % NST;
    const int64_t k0 = (tile0 + it) * TS;
    const int cnt = (int)min((int64_t)TS, A.N - k0);
    if constexpr (NX) {  // does the tile touch an excluded sphere?  (read after >= 1 barrier)
      const int n = xinfo[0];
      bool m = n < 0;
      if (!m && ntile <= kNxTiles) {
        m = (tbits[it >> 5] >> (it & 31)) & 1u;
      } else if (!m) {
        const int sa = (int)k0 / A.nsn, sb = ((int)k0 + cnt - 1) / A.nsn;
        const int i = nx_lower(xs, n, sa);
        m = i < n && xs[i] <= sb;
      }
      mflag[st] = m ? 1 : 0;
    }
    unsigned char* base = smraw + st * SM::kStageBytes;
    uint32_t bytes = cnt * kRec * 8;
    uint32_t qbytes = (OFF && MODE == 0) ? ((cnt + 1) & ~1) * 8 : 0;
    mbar_arrive_expect_tx(&bar[st], bytes + qbytes);
    bulk_g2s_hint(base, A.rec + k0 * kRec, bytes, &bar[st], pol);
    if (OFF && MODE == 0) bulk_g2s(base + SM::kRecBytes, A.qn3 + k0, qbytes, &bar[st]);
  };

  if (threadIdx.x == 0) {
    for (int st = 0; st < NST; ++st) mbar_init(&bar[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int it = 0; it < NST && it < ntile; ++it) issue(it);
  }
  if constexpr (NX) __syncthreads();  // the first stages' masked flags

  for (int it = 0; it < ntile; ++it) {
    const int st = it % NST;
    mbar_wait(&bar[st], (it / NST) & 1);
    const int64_t k0 = (tile0 + it) * TS;
    const int cnt = (int)min((int64_t)TS, A.N - k0);
    const double2* srec = reinterpret_cast<const double2*>(smraw + st * SM::kStageBytes);
    const double* sqn = reinterpret_cast<const double*>(smraw + st * SM::kStageBytes + SM::kRecBytes);
    const bool masked = NX ? mflag[st] != 0 : (!OFF && (k0 < cta_hi) && (k0 + cnt > cta_lo));
    if (!masked) {
#pragma unroll(UNR)
      for (int sidx = 0; sidx < cnt; ++sidx) {
        const double2* sr = srec + sidx * (kRec / 2);
        const double2 s0 = sr[0], s1 = sr[1], s2 = sr[2], s3 = sr[3], s4 = sr[4], s5 = sr[5];
        const double qn = (OFF && MODE == 0) ? sqn[sidx] : 0.0;
        if (MODE == 1) {
#pragma unroll
          for (int r = 0; r < R; ++r)
            pair_K<false>(s0, s1, s4, s5, xt[r], nx[MODE == 1 ? r : 0], acc[r], 0, 0, 1);
        } else if (!OFF) {
          pair_acc_g<R, false>(s0, s1, s2, s3, s4, s5, qn, xt, acc, pacc);
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r)
            pair_acc<false, OFF>(s0, s1, s2, s3, s4, s5, qn, xt[r], acc[r], pacc[r], 0, 0, 1);
        }
      }
    } else if (NX) {
      // Segments of one source sphere each.  A sphere excluded by every target
      // sphere of the tile is skipped, one excluded by none runs the unmasked
      // unrolled loop, and only a mixed one takes the per-pair mask (targets
      // of the same CTA on different spheres).
      const int n = xinfo[0];
      const int nts = (int)(last / A.nsn) - t_lo + 1;
      const uint64_t all = nts >= 64 ? ~0ull : ((1ull << nts) - 1);
      for (int seg = 0; seg < cnt;) {
        const int k = (int)k0 + seg;
        const int sk = k / A.nsn;
        const int seg_end = min(cnt, (sk + 1) * A.nsn - (int)k0);
        uint64_t mk = 0;
        bool ex[R];
        if (n >= 0) {  // target spheres excluding sk: OR of the table's masks
          for (int i = nx_lower(xs, n, sk); i < n && xs[i] == sk; ++i) mk |= xm[i];
#pragma unroll
          for (int r = 0; r < R; ++r) ex[r] = (mk >> (lo[r] / A.nsn - t_lo)) & 1;
        } else {  // table overflow: the neighbour lists themselves
          mk = 1;  // (forces the per-pair path)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int tr = lo[r] / A.nsn;
            bool e = tr == sk;
            for (int q = A.nb_off[tr]; q < A.nb_off[tr + 1] && !e; ++q) e = A.nb_idx[q] == sk;
            ex[r] = e;
          }
        }
        if (n >= 0 && (mk & all) == all) {
          seg = seg_end;  // excluded for every target of the tile
          continue;
        }
        if (mk == 0) {  // excluded for none: the unmasked loop
#pragma unroll(UNR)
          for (int sidx = seg; sidx < seg_end; ++sidx) {
            const double2* sr = srec + sidx * (kRec / 2);
            const double2 s0 = sr[0], s1 = sr[1], s2 = sr[2], s3 = sr[3], s4 = sr[4], s5 = sr[5];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if (MODE == 1)
                pair_K<false>(s0, s1, s4, s5, xt[r], nx[MODE == 1 ? r : 0], acc[r], 0, 0, 1);
              else
                pair_acc<false, false>(s0, s1, s2, s3, s4, s5, 0.0, xt[r], acc[r], pacc[r], 0, 0, 1);
            }
          }
        } else {
          // mixed: per target, a node range that masks the whole segment
          // (its sphere's start) or none (far below every index)
          int lx[R];
#pragma unroll
          for (int r = 0; r < R; ++r) lx[r] = ex[r] ? sk * A.nsn : -(1 << 30);
#pragma unroll(UNR)
          for (int sidx = seg; sidx < seg_end; ++sidx) {
            const int kk = (int)k0 + sidx;
            const double2* sr = srec + sidx * (kRec / 2);
            const double2 s0 = sr[0], s1 = sr[1], s2 = sr[2], s3 = sr[3], s4 = sr[4], s5 = sr[5];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if (MODE == 1)
                pair_K<true>(s0, s1, s4, s5, xt[r], nx[MODE == 1 ? r : 0], acc[r], kk, lx[r], A.nsn);
              else
                pair_acc<true, false>(s0, s1, s2, s3, s4, s5, 0.0, xt[r], acc[r], pacc[r], kk, lx[r],
                                      A.nsn);
            }
          }
        }
        seg = seg_end;
      }
    } else {
      for (int sidx = 0; sidx < cnt; ++sidx) {
        const double2* sr = srec + sidx * (kRec / 2);
        const double2 s0 = sr[0], s1 = sr[1], s2 = sr[2], s3 = sr[3], s4 = sr[4], s5 = sr[5];
        const int k = (int)(k0 + sidx);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (MODE == 1)
            pair_K<true>(s0, s1, s4, s5, xt[r], nx[MODE == 1 ? r : 0], acc[r], k, lo[r], A.nsn);
          else
            pair_acc<true, false>(s0, s1, s2, s3, s4, s5, 0.0, xt[r], acc[r], pacc[r], k, lo[r],
                                  A.nsn);
        }
      }
    }
    __syncthreads();  // every thread is done with stage st
    if (threadIdx.x == 0 && it + NST < ntile) issue(it + NST);
  }

  // ---- epilogue
  if constexpr (CL > 1) {
    // partials -> own shared memory (the ring is free: the loop ended with a
    // barrier), cluster barrier, then rank q reduces targets [q T/CL, (q+1) T/CL)
    // of the tile over ranks 0..CL-1 in order, reading the peers' shared memory.
    constexpr int T = TPB * R;
    constexpr int NC = OFF ? 4 : 3;
    static_assert(NC * T * 8 <= NST * SM::kStageBytes, "reduction buffer");
    double* red = reinterpret_cast<double*>(smraw);  // [NC][T]
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int li = r * TPB + threadIdx.x;
      red[li] = acc[r][0];
      red[T + li] = acc[r][1];
      red[2 * T + li] = acc[r][2];
      if (OFF) red[3 * T + li] = pacc[r];
    }
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int q = (int)cl.block_rank();
    const int lo_t = q * T / CL, hi_t = (q + 1) * T / CL;
    const int64_t base = (int64_t)tt * T;
    for (int li = lo_t + threadIdx.x; li < hi_t; li += TPB) {
      const int64_t i = base + li;
      if (i >= A.M) break;
      double sm3[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) sm3[c] = 0.0;
      for (int rk = 0; rk < CL; ++rk) {
        const double* rr = cl.map_shared_rank(red, rk);
#pragma unroll
        for (int c = 0; c < NC; ++c) sm3[c] += rr[c * T + li];
      }
      double u0 = sm3[0], u1 = sm3[1], u2 = sm3[2];
      if (A.uinit) {
        u0 = A.uinit[3 * i] + u0;
        u1 = A.uinit[3 * i + 1] + u1;
        u2 = A.uinit[3 * i + 2] + u2;
      }
      A.uout[3 * i] = u0;
      A.uout[3 * i + 1] = u1;
      A.uout[3 * i + 2] = u2;
      if (OFF && A.pout) A.pout[i] = A.pscale * sm3[NC - 1];
    }
    cl.sync();  // peers keep their shared memory until every rank has read it
    return;
  }
  if (CL == 1 && A.chain != nullptr && A.n_chunks > 1) {
    const int ticket = *reinterpret_cast<volatile int*>(&s_ticket);
    const int ctt = ticket % A.n_tt, cchunk = ticket / A.n_tt;
    const bool last_chunk = cchunk == A.n_chunks - 1;
    int* flag = A.chain + ctt;
    if (cchunk > 0) {
      // chunk - 1 of this tile holds a lower ticket, so it is running or done;
      // a wait that outlives any launch (60 s) traps instead of hanging
      if (threadIdx.x == 0) {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_gpu(flag) != cchunk) {
          __nanosleep(256);
          if (globaltimer_ns() - t0 > 60000000000ull) __trap();
        }
      }
      __syncthreads();
    }
    double* pacc_g = A.cacc + 3 * A.M;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = tidx[r];
      if (i >= A.M) continue;
      double s0 = acc[r][0], s1 = acc[r][1], s2 = acc[r][2], sp = pacc[r];
      if (cchunk > 0) {  // running sum (written by the previous chunk, read through L2) + own
        s0 = __ldcg(A.cacc + 3 * i) + s0;
        s1 = __ldcg(A.cacc + 3 * i + 1) + s1;
        s2 = __ldcg(A.cacc + 3 * i + 2) + s2;
        if (OFF && A.pout) sp = __ldcg(pacc_g + i) + sp;
      }
      if (last_chunk) {
        if (A.uinit) {
          s0 = A.uinit[3 * i] + s0;
          s1 = A.uinit[3 * i + 1] + s1;
          s2 = A.uinit[3 * i + 2] + s2;
        }
        A.uout[3 * i] = s0;
        A.uout[3 * i + 1] = s1;
        A.uout[3 * i + 2] = s2;
        if (OFF && A.pout) A.pout[i] = A.pscale * sp;
      } else {
        __stcg(A.cacc + 3 * i, s0);
        __stcg(A.cacc + 3 * i + 1, s1);
        __stcg(A.cacc + 3 * i + 2, s2);
        if (OFF && A.pout) __stcg(pacc_g + i, sp);
      }
    }
    if (!last_chunk) {
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release_gpu(flag, cchunk + 1);
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = tidx[r];
    if (i >= A.M) continue;
    const int64_t li = i;
    if (A.n_chunks == 1) {
      double u0 = acc[r][0], u1 = acc[r][1], u2 = acc[r][2];
      if (A.uinit) {
        u0 += A.uinit[3 * i];
        u1 += A.uinit[3 * i + 1];
        u2 += A.uinit[3 * i + 2];
      }
      A.uout[3 * li] = u0;
      A.uout[3 * li + 1] = u1;
      A.uout[3 * li + 2] = u2;
      if (OFF && A.pout) A.pout[li] = A.pscale * pacc[r];
    } else {
      const int64_t Mb = A.M;
      double* po = A.uout + ((int64_t)chunk * Mb + li) * 3;  // read once by k_reduce: streaming
      __stcs(po, acc[r][0]);
      __stcs(po + 1, acc[r][1]);
      __stcs(po + 2, acc[r][2]);
      if (OFF && A.pout) __stcs(A.pout + (int64_t)chunk * Mb + li, pacc[r]);
    }
  }
}

// u[i] = (uinit ? uinit[i] : 0) + sum_{c < n_chunks} part[c][i], fixed order;
// pressure likewise, scaled by pscale.  One thread per target component.
__global__ void k_reduce(int64_t Mb, int n_chunks, const double* __restrict__ part,
                         const double* __restrict__ uinit, double* __restrict__ u,
                         const double* __restrict__ ppart, double* __restrict__ p, double pscale) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < 3 * Mb) {
    double s = 0.0;
    for (int c = 0; c < n_chunks; ++c) s += part[(int64_t)c * 3 * Mb + e];
    u[e] = uinit ? uinit[e] + s : s;
  }
  if (ppart && p && e < Mb) {
    double s = 0.0;
    for (int c = 0; c < n_chunks; ++c) s += ppart[(int64_t)c * Mb + e];
    p[e] = pscale * s;
  }
}

}  // namespace bie

namespace bie {

// ---------------------------------------------------------------- stream-K
// Persistent far-field kernel (the default schedule): the work units
// (target tile tt, source tile st), flattened tt-major (u = tt S + st, S source
// tiles, T = n_tt S units), are split into G equal contiguous ranges, one per
// resident CTA slot, so every CTA does the same amount of work (no idle last
// wave).  A CTA walks its range as segments of one target tile each; a segment
// that covers all S source tiles of its tile writes the result directly, the
// (at most two) partial segments of a CTA -- its first and its last -- go to
// the partial buffer, slot 2c (first) / 2c+1 (last), and k_sk_fixup sums the
// partials of every split tile in CTA order (deterministic).  HBM traffic:
// targets once, records through L2, <= 2G partial tiles.
__host__ __device__ __forceinline__ int64_t sk_u0(int64_t c, int64_t T, int64_t G) { return c * T / G; }
// CTA whose range contains unit u: the largest c with sk_u0(c) <= u
__host__ __device__ __forceinline__ int64_t sk_owner(int64_t u, int64_t T, int64_t G) {
  return ((u + 1) * G + T - 1) / T - 1;
}

struct SkArgs {
  NbodyArgs A;
  int64_t S, T, G;   // source tiles, units, CTAs
  double* part;      // [2G][NC][TPB R] partial tiles
};

template <int R, int TPB, int TS, int NST, bool OFF, int MINB = 1, int UNR = 2, int MODE = 0>
__global__ void __launch_bounds__(TPB, MINB) k_nbody_sk(const SkArgs K) {
  using SM = NbodySmem<TS, NST, OFF>;
  constexpr int T_TILE = TPB * R;
  constexpr int NC = OFF ? 4 : 3;
  const NbodyArgs& A = K.A;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + NST * SM::kStageBytes);
  const int64_t c = blockIdx.x;
  const int64_t u_begin = sk_u0(c, K.T, K.G), u_end = sk_u0(c + 1, K.T, K.G);
  const int64_t tt_first = u_begin / K.S;
  const uint64_t pol = l2_evict_last_policy();

  if (threadIdx.x == 0) {
    for (int st = 0; st < NST; ++st) mbar_init(&bar[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int64_t g = 0;  // ring position over all of this CTA's source tiles (stage, parity)
  for (int64_t u = u_begin; u < u_end;) {
    const int64_t tt = u / K.S;
    const int64_t st0 = u - tt * K.S;
    const int64_t st1 = min(K.S, st0 + (u_end - u));
    const int ntile = (int)(st1 - st0);
    // ---- targets of tile tt in registers
    double xt[R][3], acc[R][3], pacc[R];
    double nx[MODE == 1 ? R : 1][3];
    int lo[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = tt * T_TILE + r * TPB + threadIdx.x;
      const int64_t ic = i < A.M ? i : A.M - 1;
      if (OFF) {
        xt[r][0] = A.tx[3 * ic];
        xt[r][1] = A.tx[3 * ic + 1];
        xt[r][2] = A.tx[3 * ic + 2];
        lo[r] = 0;
        if (MODE == 1) {
          nx[MODE == 1 ? r : 0][0] = A.tn[3 * ic];
          nx[MODE == 1 ? r : 0][1] = A.tn[3 * ic + 1];
          nx[MODE == 1 ? r : 0][2] = A.tn[3 * ic + 2];
        }
      } else {
        xt[r][0] = A.rec[ic * kRec];
        xt[r][1] = A.rec[ic * kRec + 1];
        xt[r][2] = A.rec[ic * kRec + 2];
        lo[r] = (int)((ic / A.nsn) * A.nsn);
        if (MODE == 1) {
          nx[MODE == 1 ? r : 0][0] = A.rec[ic * kRec + 3];
          nx[MODE == 1 ? r : 0][1] = A.rec[ic * kRec + 4];
          nx[MODE == 1 ? r : 0][2] = A.rec[ic * kRec + 5];
        }
      }
      acc[r][0] = acc[r][1] = acc[r][2] = 0.0;
      pacc[r] = 0.0;
    }
    const int64_t first = tt * T_TILE;
    const int64_t last = min(first + T_TILE, A.M) - 1;
    const int64_t cta_lo = (first / A.nsn) * A.nsn;
    const int64_t cta_hi = (last / A.nsn + 1) * A.nsn;
    auto issue = [&](int it) {
      const int st = (int)((g + it) % NST);
      const int64_t k0 = (st0 + it) * TS;
      const int cnt = (int)min((int64_t)TS, A.N - k0);
      unsigned char* base = smraw + st * SM::kStageBytes;
      const uint32_t bytes = cnt * kRec * 8;
      const uint32_t qbytes = (OFF && MODE == 0) ? ((cnt + 1) & ~1) * 8 : 0;
      mbar_arrive_expect_tx(&bar[st], bytes + qbytes);
      bulk_g2s_hint(base, A.rec + k0 * kRec, bytes, &bar[st], pol);
      if (OFF && MODE == 0) bulk_g2s(base + SM::kRecBytes, A.qn3 + k0, qbytes, &bar[st]);
    };
    if (threadIdx.x == 0)
      for (int it = 0; it < NST && it < ntile; ++it) issue(it);
    for (int it = 0; it < ntile; ++it) {
      const int st = (int)((g + it) % NST);
      mbar_wait(&bar[st], (uint32_t)(((g + it) / NST) & 1));
      const int64_t k0 = (st0 + it) * TS;
      const int cnt = (int)min((int64_t)TS, A.N - k0);
      const double2* srec = reinterpret_cast<const double2*>(smraw + st * SM::kStageBytes);
      const double* sqn = reinterpret_cast<const double*>(smraw + st * SM::kStageBytes + SM::kRecBytes);
      const bool masked = !OFF && (k0 < cta_hi) && (k0 + cnt > cta_lo);
      if (!masked) {
#pragma unroll(UNR)
        for (int sidx = 0; sidx < cnt; ++sidx) {
          const double2* sr = srec + sidx * (kRec / 2);
          const double2 s0 = sr[0], s1 = sr[1], s2 = sr[2], s3 = sr[3], s4 = sr[4], s5 = sr[5];
          const double qn = (OFF && MODE == 0) ? sqn[sidx] : 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (MODE == 1)
              pair_K<false>(s0, s1, s4, s5, xt[r], nx[MODE == 1 ? r : 0], acc[r], 0, 0, 1);
            else
              pair_acc<false, OFF>(s0, s1, s2, s3, s4, s5, qn, xt[r], acc[r], pacc[r], 0, 0, 1);
          }
        }
      } else {
        for (int sidx = 0; sidx < cnt; ++sidx) {
          const double2* sr = srec + sidx * (kRec / 2);
          const double2 s0 = sr[0], s1 = sr[1], s2 = sr[2], s3 = sr[3], s4 = sr[4], s5 = sr[5];
          const int k = (int)(k0 + sidx);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (MODE == 1)
              pair_K<true>(s0, s1, s4, s5, xt[r], nx[MODE == 1 ? r : 0], acc[r], k, lo[r], A.nsn);
            else
              pair_acc<true, false>(s0, s1, s2, s3, s4, s5, 0.0, xt[r], acc[r], pacc[r], k, lo[r],
                                    A.nsn);
          }
        }
      }
      __syncthreads();  // every thread is done with stage st
      if (threadIdx.x == 0 && it + NST < ntile) issue(it + NST);
    }
    g += ntile;
    // ---- epilogue of the segment
    const bool complete = st0 == 0 && st1 == K.S;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int li = r * TPB + threadIdx.x;
      const int64_t i = first + li;
      if (complete) {
        if (i >= A.M) continue;
        double u0 = acc[r][0], u1 = acc[r][1], u2 = acc[r][2];
        if (A.uinit) {
          u0 = A.uinit[3 * i] + u0;
          u1 = A.uinit[3 * i + 1] + u1;
          u2 = A.uinit[3 * i + 2] + u2;
        }
        A.uout[3 * i] = u0;
        A.uout[3 * i + 1] = u1;
        A.uout[3 * i + 2] = u2;
        if (OFF && A.pout) A.pout[i] = A.pscale * pacc[r];
      } else {
        const int64_t slot = 2 * c + (tt == tt_first ? 0 : 1);
        double* P = K.part + slot * NC * T_TILE;
        __stcs(P + li, acc[r][0]);
        __stcs(P + T_TILE + li, acc[r][1]);
        __stcs(P + 2 * T_TILE + li, acc[r][2]);
        if (OFF) __stcs(P + 3 * T_TILE + li, pacc[r]);
      }
    }
    u += ntile;
  }
}

// Sum the partial segments of every split target tile in CTA order: block b
// handles the tile containing boundary b+1 if that is the tile's first boundary.
template <int T_TILE, bool OFF>
__global__ void k_sk_fixup(const SkArgs K) {
  constexpr int NC = OFF ? 4 : 3;
  const NbodyArgs& A = K.A;
  const int64_t cb = blockIdx.x + 1;  // boundary between CTA cb-1 and cb
  const int64_t ub = sk_u0(cb, K.T, K.G);
  if (ub >= K.T || ub % K.S == 0) return;
  const int64_t tt = ub / K.S;
  const int64_t c_lo = sk_owner(tt * K.S, K.T, K.G);
  if (c_lo != cb - 1) return;  // an earlier boundary of this tile handles it
  const int64_t c_hi = sk_owner((tt + 1) * K.S - 1, K.T, K.G);
  for (int li = threadIdx.x; li < T_TILE; li += blockDim.x) {
    const int64_t i = tt * T_TILE + li;
    if (i >= A.M) break;
    double s[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) s[q] = 0.0;
    for (int64_t cc = c_lo; cc <= c_hi; ++cc) {
      if (sk_u0(cc, K.T, K.G) == sk_u0(cc + 1, K.T, K.G)) continue;  // empty range (T < G)
      const int64_t slot = 2 * cc + (sk_u0(cc, K.T, K.G) / K.S == tt ? 0 : 1);
      const double* P = K.part + slot * NC * T_TILE;
#pragma unroll
      for (int q = 0; q < NC; ++q) s[q] += P[q * T_TILE + li];
    }
    double u0 = s[0], u1 = s[1], u2 = s[2];
    if (A.uinit) {
      u0 = A.uinit[3 * i] + u0;
      u1 = A.uinit[3 * i + 1] + u1;
      u2 = A.uinit[3 * i + 2] + u2;
    }
    A.uout[3 * i] = u0;
    A.uout[3 * i + 1] = u1;
    A.uout[3 * i + 2] = u2;
    if (OFF && A.pout) A.pout[i] = A.pscale * s[NC - 1];
  }
}

}  // namespace bie
