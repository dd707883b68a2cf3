// bie.cu -- C ABI of libbie.so (declared and documented in include/bie.h).
//
// Host side: argument validation, device memory ownership, launch
// configuration and profiling events.  Every arithmetic step of the path runs
// in the kernels of k_setup.cuh, k_self.cuh and k_nbody.cuh.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <algorithm>
#include <unordered_map>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "../../include/bie.h"
#include "common.cuh"
#include "k_complete.cuh"
#include "k_krylov.cuh"
#include "k_nbody.cuh"
#include "k_nbody_c.cuh"
#include "k_n4.cuh"
#include "k_near.cuh"
#include "k_self.cuh"
#include "k_sht.cuh"
#include "k_setup.cuh"

using namespace bie;

namespace {

// Far-field kernel configurations: R targets per thread,
// TPB threads, TS sources per shared-memory tile, NST pipeline stages, source
// loop unroll.  Chosen per kernel by tools/nbody_tune.cu on B200
// (profiles/r01_nbody_tune.txt): 8 targets per thread for the SL+DL apply,
// 7 for the off-surface and traction kernels (their extra per-target
// registers -- pressure, normals -- make 8 spill-prone and RF-read bound).
constexpr int kTPB = 64, kTS = 64, kNST = 3;
constexpr int kR_APPLY = 8, kR_OFF = 7, kR_K = 7, kR_OFFK = 7;
constexpr int kR_APPLY_C = 8, kR_OFF_C = 8, kUNR_C = 4;  // constant-bank kernels (k_nbody_c.cuh)
#ifndef BIE_UNR_OFF_C
#define BIE_UNR_OFF_C 2
#endif
constexpr int kUNR_OFF_C = BIE_UNR_OFF_C;  // off-surface batch-loop unroll (2 measured: see DESIGN.md 5.2)
constexpr int64_t kOffBatch = 1 << 21;  // off-surface targets per batch (bounds scratch)
constexpr double kScratchBytes = 3.0e9;  // cap on chunk-partial scratch

#define NBODY_APPLY k_nbody<kR_APPLY, kTPB, kTS, kNST, false, 1, 2>
// near exclusion: the smooth rule skips eq-4.5 neighbour pairs (NEXT-1/4 on)
#define NBODY_APPLY_NX k_nbody<kR_APPLY, kTPB, kTS, kNST, false, 1, 2, 0, 1, true>
#define NBODY_K_NX k_nbody<kR_K, kTPB, kTS, kNST, false, 1, 2, 1, 1, true>
#define NBODY_OFF k_nbody<kR_OFF, kTPB, kTS, kNST, true, 1, 2>
#define NBODY_K k_nbody<kR_K, kTPB, kTS, kNST, false, 1, 2, 1>
#define NBODY_OFFK k_nbody<kR_OFFK, kTPB, kTS, kNST, true, 1, 2, 1>
// cluster-reduced variants (source chunks of a target tile = one cluster)
constexpr int kCL = 8;
#define NBODY_APPLY_CL k_nbody<kR_APPLY, kTPB, kTS, kNST, false, 1, 2, 0, kCL>
#define NBODY_APPLY_CL4 k_nbody<kR_APPLY, kTPB, kTS, kNST, false, 1, 2, 0, 4>
// stream-K persistent variants (the default schedule)
#define NBODY_APPLY_SK k_nbody_sk<kR_APPLY, kTPB, kTS, kNST, false, 1, 2, 0>
#define NBODY_OFF_SK k_nbody_sk<kR_OFF, kTPB, kTS, kNST, true, 1, 2, 0>
#define NBODY_K_SK k_nbody_sk<kR_K, kTPB, kTS, kNST, false, 1, 2, 1>
#define NBODY_OFFK_SK k_nbody_sk<kR_OFFK, kTPB, kTS, kNST, true, 1, 2, 1>
#define NBODY_APPLY_CL16 k_nbody<kR_APPLY, kTPB, kTS, kNST, false, 1, 2, 0, 16>
#define NBODY_OFF_CL k_nbody<kR_OFF, kTPB, kTS, kNST, true, 1, 2, 0, kCL>
#define NBODY_K_CL k_nbody<kR_K, kTPB, kTS, kNST, false, 1, 2, 1, kCL>
#define NBODY_OFFK_CL k_nbody<kR_OFFK, kTPB, kTS, kNST, true, 1, 2, 1, kCL>

struct Ev {
  int kind;
  cudaEvent_t a, b;
};

}  // namespace

struct bie_ctx {
  int dev = -1, sm_count = 0, occ_apply = 1, occ_off = 1, occ_K = 1, occ_offK = 1;
  int p = 0, nsn = 0;
  int64_t ns = 0, N = 0;
  double mu = 1.0;
  double* d_centres = nullptr;
  double* d_radii = nullptr;
  double* d_tab = nullptr;
  double* d_x = nullptr;
  double* d_n = nullptr;
  double* d_w = nullptr;
  double* d_rec = nullptr;
  double* d_qn3 = nullptr;
  double* d_part = nullptr;
  size_t part_cap = 0;  // doubles
  cudaStream_t st_side = nullptr;              // constant-bank far field: stream of the odd batches
  int64_t const_sub = 655360;                  // targets per sub-range of a constant-bank pass (0: all)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double* d_sht = nullptr;  // fragment-order transform tables of k_sht
  int sht_occ = 1;          // resident k_sht CTAs per SM
  int self_variant = -1;    // -1 auto (fastest measured per order), 0 k_sht DMMA, 1 k_sht DFMA,
                            // 2 round-1 k_self_t
  int chunks_override = 0;
  int far_red = 1;  // bie_set_far_reduction: 0 stream-K, 1 chunks (default; chained or k_reduce by
                    // size), 2/3/4 clusters, 5 chunks always chained, 6 chunks always + k_reduce
  double* d_cacc = nullptr;  // chained reduction: running sums [M][4]
  size_t cacc_cap = 0;       // doubles
  int* d_chain = nullptr;    // chained reduction: per-tile flags + ticket counter
  size_t chain_cap = 0;      // ints
  int occ_sk[4] = {1, 1, 1, 1};
  int occ_apply_nx = 1, occ_K_nx = 1;  // resident CTAs per SM of the near-exclusion kernels  // resident CTAs per SM of the stream-K kernels (apply, off, K, offK)
  // near-singular correction (NEXT-1)
  double eta = 0.0;
  int n_near_tgt = 0;
  int64_t n_near_pairs = 0;
  int* d_nb_off = nullptr;
  int* d_nb_idx = nullptr;
  int* d_near_tgt = nullptr;
  double* d_alpha = nullptr;
  double* d_ncoef = nullptr;
  // sphere cell grid for the off-surface near search (bie_set_near)
  int* d_cell_start = nullptr;
  int* d_cell_items = nullptr;
  double g0[3] = {0, 0, 0}, gh = 1.0;
  int gn[3] = {1, 1, 1};
  // Morton-sorted target order scratch (off-surface near correction)
  void* d_sort = nullptr;
  size_t sort_cap = 0;
  // off-surface near correction schedule (bie_set_near_off_schedule): 0 pairs
  // grouped by sphere (default), 1 one thread per Morton-sorted target
  int noff_sched = 0;
  void* d_grp1 = nullptr;  // per-target scratch of the grouped schedule
  size_t grp1_cap = 0;
  void* d_grp2 = nullptr;  // per-pair / per-sphere scratch
  size_t grp2_cap = 0;
  // NEXT-4 (bie_set_near_mode): 0 direct, 1 rotated (PAPER §4.2), 2/3 measurement
  int near_mode = 0;
  int near_excl = -1;  // bie_set_near_exclusion: -1 auto (cost model), 0 subtract, 1 exclude
  double* d_delta = nullptr;    // packed Delta_n (rotation operator of T = Rx(-pi/2))
  double* d_deltaT = nullptr;   // and its per-degree transpose
  double* d_psinear = nullptr;  // [ns][nlm][6] accumulated neighbour coefficients
  // staging for the _host entry points
  double *d_f = nullptr, *d_q = nullptr, *d_u = nullptr;
  double *d_tg = nullptr, *d_uo = nullptr, *d_po = nullptr;
  int64_t tg_cap = 0;
  // profiling
  bool prof = false;
  std::vector<Ev> pending;
  double ms[BIE_NUM_KINDS] = {0};
  int64_t launches[BIE_NUM_KINDS] = {0};
  std::string err;
};

static int fail(bie_ctx* c, int st, const char* fmt, const char* a = "") {
  if (c) {
    char buf[512];
    snprintf(buf, sizeof buf, fmt, a);
    c->err = buf;
  }
  return st;
}

static int cuda_fail(bie_ctx* c, cudaError_t e, const char* where) {
  if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e);
  return BIE_ERR_CUDA;
}

// ---------------------------------------------------------------- profiling
static void prof_begin(bie_ctx* c, int kind, cudaStream_t s, Ev* ev) {
  c->launches[kind]++;
  ev->kind = kind;
  ev->a = ev->b = nullptr;
  if (!c->prof) return;
  cudaEventCreate(&ev->a);
  cudaEventCreate(&ev->b);
  cudaEventRecord(ev->a, s);
}

static void prof_end(bie_ctx* c, cudaStream_t s, Ev* ev) {
  if (!c->prof || !ev->a) return;
  cudaEventRecord(ev->b, s);
  c->pending.push_back(*ev);
}

static void prof_drain(bie_ctx* c) {
  for (Ev& e : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(e.b);
    cudaEventElapsedTime(&ms, e.a, e.b);
    c->ms[e.kind] += ms;
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  c->pending.clear();
}

// ---------------------------------------------------------------- validation
// Device memory of the context's GPU (the device current at bie_create), or
// managed memory.  Memory of another GPU is rejected here: a kernel touching it
// would fault with a sticky error that kills the context.
static bool is_device_ptr(const bie_ctx* c, const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (at.type == cudaMemoryTypeManaged) return true;
  return at.type == cudaMemoryTypeDevice && at.device == c->dev;
}

static bool overlaps(const double* a, int64_t na, const double* b, int64_t nb) {
  if (!a || !b) return false;
  return a < b + nb && b < a + na;
}

static int check_device(bie_ctx* c) {
  int d = -1;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaGetDevice");
  if (d != c->dev) return fail(c, BIE_ERR_ARG, "current device differs from the device at bie_create%s");
  return BIE_OK;
}

// Overlap/contact test with a uniform cell list (cell = 2 max radius): O(n_spheres).
static bool spheres_overlap(const double* c, const double* a, int64_t n, int64_t* bad_i, int64_t* bad_j) {
  double amax = 0;
  for (int64_t i = 0; i < n; ++i) amax = std::max(amax, a[i]);
  const double h = 2.0 * amax;
  auto key = [](int64_t x, int64_t y, int64_t z) {
    return (uint64_t)((x & 0x1FFFFF) | ((y & 0x1FFFFF) << 21) | ((z & 0x1FFFFF) << 42));
  };
  std::unordered_map<uint64_t, std::vector<int64_t>> grid;
  grid.reserve(2 * n);
  std::vector<int64_t> cell(3 * n);
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < 3; ++d) cell[3 * i + d] = (int64_t)std::floor(c[3 * i + d] / h);
    grid[key(cell[3 * i], cell[3 * i + 1], cell[3 * i + 2])].push_back(i);
  }
  for (int64_t i = 0; i < n; ++i)
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          auto it = grid.find(key(cell[3 * i] + dx, cell[3 * i + 1] + dy, cell[3 * i + 2] + dz));
          if (it == grid.end()) continue;
          for (int64_t j : it->second) {
            if (j <= i) continue;
            double r2 = 0;
            for (int d = 0; d < 3; ++d) r2 += (c[3 * i + d] - c[3 * j + d]) * (c[3 * i + d] - c[3 * j + d]);
            double lim = a[i] + a[j];
            if (r2 <= lim * lim) {  // touching spheres can share a node (r = 0)
              *bad_i = i;
              *bad_j = j;
              return true;
            }
          }
        }
  return false;
}

// eq 4.5 for the sphere pair (s, t), evaluated in the oracle's
// order with IEEE round-to-nearest (host x86-64 SSE2: no contraction, no
// extended precision):  |c_s - c_t| - a_s - a_t < eta max(2 a_s, 2 a_t).
static bool near_pair_host(const double* cs, double as, const double* ct, double at, double eta) {
  const double dx = cs[0] - ct[0], dy = cs[1] - ct[1], dz = cs[2] - ct[2];
  const double r2 = (dx * dx + dy * dy) + dz * dz;
  const double d = (std::sqrt(r2) - as) - at;
  return d < eta * std::max(2.0 * as, 2.0 * at);
}

// CSR neighbour lists of eq 4.5 (NEXT-1) with a uniform cell list, O(n):
// a near pair has |c_s - c_t| < a_s + a_t + 2 eta a_max <= 2 a_max (1 + eta),
// so with cells of that size (padded) every near source of t lies in the 27
// cells around t's cell.  off is int64 (the caller bounds the total); each
// target's sources are ascending (the order k_near accumulates in).
static void near_lists_host(const double* c, const double* a, int64_t n, double eta,
                            std::vector<int64_t>& off, std::vector<int>& idx) {
  double amax = 0;
  for (int64_t i = 0; i < n; ++i) amax = std::max(amax, a[i]);
  const double h = 2.0 * amax * (1.0 + eta) * (1.0 + 1e-9) + 1e-300;
  auto key = [](int64_t x, int64_t y, int64_t z) {
    return (uint64_t)((x & 0x1FFFFF) | ((y & 0x1FFFFF) << 21) | ((z & 0x1FFFFF) << 42));
  };
  std::unordered_map<uint64_t, std::vector<int>> grid;
  grid.reserve(2 * n);
  std::vector<int64_t> cell(3 * n);
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < 3; ++d) cell[3 * i + d] = (int64_t)std::floor(c[3 * i + d] / h);
    grid[key(cell[3 * i], cell[3 * i + 1], cell[3 * i + 2])].push_back((int)i);
  }
  off.assign(n + 1, 0);
  idx.clear();
  std::vector<int> cand;
  for (int64_t t = 0; t < n; ++t) {
    cand.clear();
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          auto it = grid.find(key(cell[3 * t] + dx, cell[3 * t + 1] + dy, cell[3 * t + 2] + dz));
          if (it == grid.end()) continue;
          for (int s : it->second)
            if (s != t && near_pair_host(c + 3 * (int64_t)s, a[s], c + 3 * t, a[t], eta)) cand.push_back(s);
        }
    std::sort(cand.begin(), cand.end());
    idx.insert(idx.end(), cand.begin(), cand.end());
    off[t + 1] = (int64_t)idx.size();
  }
}

// ---------------------------------------------------------------- launches
struct ChunkPlan {
  int n_tt, n_chunks, tiles_per_chunk;
};

static ChunkPlan plan_chunks(const bie_ctx* c, int64_t M, int64_t N, int occ, int r) {
  ChunkPlan P;
  const int64_t tile = (int64_t)r * kTPB;  // targets per CTA
  P.n_tt = (int)((M + tile - 1) / tile);
  const int64_t n_src_tiles = (N + kTS - 1) / kTS;
  int64_t S;
  if (c->chunks_override > 0) {
    S = c->chunks_override;
  } else {
    // Units = target tiles x source chunks.  With many waves (>= 16 units per
    // resident CTA slot) the hardware's dynamic CTA dispatch keeps the tail
    // small; below that, pick the chunk count whose last wave is fullest.
    const int64_t slots = (int64_t)c->sm_count * std::max(occ, 1);
    const int64_t cap = (int64_t)(kScratchBytes / (32.0 * std::max<int64_t>(M, 1)));
    int64_t smax = (64 * slots + P.n_tt - 1) / P.n_tt;  // ~64 units per CTA slot
    smax = std::min<int64_t>(smax, std::max<int64_t>(1, n_src_tiles / 2));
    smax = std::max<int64_t>(1, std::min<int64_t>(smax, cap));
    if ((int64_t)P.n_tt * smax >= 16 * slots) {
      S = smax;
    } else {
      S = 1;
      double best = -1.0;
      for (int64_t s = 1; s <= smax; ++s) {
        const int64_t tpc = (n_src_tiles + s - 1) / s;
        const int64_t se = (n_src_tiles + tpc - 1) / tpc;
        const int64_t units = (int64_t)P.n_tt * se;
        const int64_t waves = (units + slots - 1) / slots;
        // busy fraction of the slot-time, with a per-unit start cost of ~1/20 tile
        const double eff = (double)units / (double)(waves * slots) * (double)tpc / (tpc + 0.05);
        if (eff > best + 1e-9) {
          best = eff;
          S = se;
        }
      }
    }
  }
  S = std::max<int64_t>(1, std::min<int64_t>(S, n_src_tiles));
  P.tiles_per_chunk = (int)((n_src_tiles + S - 1) / S);
  P.n_chunks = (int)((n_src_tiles + P.tiles_per_chunk - 1) / P.tiles_per_chunk);
  return P;
}

static int ensure_part(bie_ctx* c, size_t doubles) {
  if (doubles <= c->part_cap) return BIE_OK;
  if (c->d_part) cudaFree(c->d_part);
  c->d_part = nullptr;
  c->part_cap = 0;
  cudaError_t e = cudaMalloc(&c->d_part, doubles * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, BIE_ERR_ALLOC, "cannot allocate far-field scratch%s");
  }
  c->part_cap = doubles;
  return BIE_OK;
}

// Chained chunk reduction (bie_set_far_reduction 5): the running-sum buffer
// ([M][3] + [M] pressure) and the n_tt flags + ticket counter, zeroed on the
// stream before the launch (a launch that died mid-way cannot leave stale flags).
static int setup_chain(bie_ctx* c, NbodyArgs& A, int64_t M, cudaStream_t s) {
  const size_t nd = (size_t)4 * M, ni = (size_t)A.n_tt + 1;
  if (nd > c->cacc_cap) {
    cudaFree(c->d_cacc);
    c->d_cacc = nullptr;
    c->cacc_cap = 0;
    if (cudaMalloc(&c->d_cacc, nd * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, BIE_ERR_ALLOC, "cannot allocate the chained-reduction sums%s");
    }
    c->cacc_cap = nd;
  }
  if (ni > c->chain_cap) {
    cudaFree(c->d_chain);
    c->d_chain = nullptr;
    c->chain_cap = 0;
    if (cudaMalloc(&c->d_chain, ni * sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, BIE_ERR_ALLOC, "cannot allocate the chained-reduction flags%s");
    }
    c->chain_cap = ni;
  }
  cudaError_t e = cudaMemsetAsync(c->d_chain, 0, ni * sizeof(int), s);
  if (e != cudaSuccess) return cuda_fail(c, e, "chained reduction flags");
  A.chain = c->d_chain;
  A.cacc = c->d_cacc;
  return BIE_OK;
}

// Chained in-kernel reduction (5) or HBM partials + k_reduce (6) for a chunked
// launch; the default (1) chains when the launch has >= 16 units per resident
// CTA slot -- then chunk c - 1 of a tile finished long before chunk c does --
// and uses k_reduce below that, where the chunks of a tile run side by side
// and a chained CTA would idle waiting for its predecessor (cfg 2: 0.33 vs
// 0.24 ms, profiles/r02_far_reduction.jsonl).
static bool use_chain(const bie_ctx* c, const ChunkPlan& P, int occ) {
  if (c->far_red == 5) return true;
  if (c->far_red != 1) return false;
  const int64_t slots = (int64_t)c->sm_count * std::max(occ, 1);
  return (int64_t)P.n_tt * P.n_chunks >= 16 * slots;
}

static int launch_check(bie_ctx* c, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(c, e, what);
  return BIE_OK;
}

// The self-term kernel of this context's variant: k_sht (batched DMMA or DFMA
// contractions, default) or the round-1 per-sphere k_self_t (kept for
// comparison; bie_set_self_kernel).
static void self_launch(bie_ctx* c, const SelfArgs& SA, cudaStream_t s) {
  // auto: the per-sphere kernel up to p = 19, the DMMA contractions above
  // (profiles/r02_self_bench.jsonl: 1.37x at p = 24, 1.6x at p = 32)
  const int variant = c->self_variant >= 0 ? c->self_variant : (c->p <= 19 ? 2 : 0);
  if (variant == 2 && !SA.psinear) {
    launch_self(SA, s);
    return;
  }
  if (variant == 3 && !SA.psinear) {
    launch_self2(SA, s);
    return;
  }
  // (NEXT-4's coefficient accumulation exists only in k_sht)
  const cudaError_t e = launch_sht(SA, c->d_sht, variant >= 2 ? 0 : variant, c->sm_count, c->sht_occ, s);
  (void)e;  // surfaced by the caller's launch_check (cudaGetLastError)
}

// Arguments of the per-sphere self-term kernel (k_self) for this context.
static SelfArgs self_args(const bie_ctx* c, const double* f, const double* q, double* u, int self,
                          double* alpha, int precond) {
  SelfArgs SA;
  SA.p = c->p;
  SA.ns = c->ns;
  SA.mu = c->mu;
  SA.cS = 1.0 / (8.0 * kPi * c->mu);
  SA.tab = c->d_tab;
  SA.centres = c->d_centres;
  SA.radii = c->d_radii;
  SA.f = f;
  SA.q = q;
  SA.u = u;
  SA.rec = c->d_rec;
  SA.self = self;
  SA.alpha = alpha;
  SA.precond = precond;
  return SA;
}

static int run_far(bie_ctx* c, double* u, cudaStream_t s, int mode = 0, bool nx = false);

// per-sphere exterior-expansion coefficients from the k_self projections
static int run_near_coef(bie_ctx* c, cudaStream_t s) {
  const TableLayout L(c->p);
  const int64_t n = c->ns * L.nlm;
  Ev ev;
  prof_begin(c, BIE_KIND_NEAR, s, &ev);
  k_near_coef<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(c->p, c->ns, c->mu, c->d_radii, c->d_alpha,
                                                          c->d_ncoef);
  prof_end(c, s, &ev);
  return launch_check(c, "k_near_coef");
}

// Near correction at the nodes (NEXT-1 velocity, K = false; NEXT-3 traction,
// K = true), after the far field: one CTA per target sphere with neighbours.
static int run_near(bie_ctx* c, double* u, cudaStream_t s, bool K, int part = 0) {
  NearArgs NA;
  NA.p = c->p;
  NA.nsn = c->nsn;
  NA.tab = c->d_tab;
  NA.centres = c->d_centres;
  NA.radii = c->d_radii;
  NA.rec = c->d_rec;
  NA.coef = c->d_ncoef;
  NA.tgt = c->d_near_tgt;
  NA.nb_off = c->d_nb_off;
  NA.nb_idx = c->d_nb_idx;
  NA.u = u;
  Ev ev;
  prof_begin(c, BIE_KIND_NEAR, s, &ev);
  const bool stage = near_stage(c->p);
  const size_t nsm = near_smem_doubles(c->p, stage) * sizeof(double);
  const unsigned g = (unsigned)c->n_near_tgt;
  const size_t nsm2 = near2_smem_doubles(c->p) * sizeof(double);  // PART 2, staged
  if (K && part == 2) {  // exact traction only (the smooth K sum excluded these pairs)
    if (near2_stage(c->p)) k_near<true, true, 2><<<g, 128, nsm2, s>>>(NA);
    else k_near<false, true, 2><<<g, 128, nsm, s>>>(NA);
  } else if (K) {
    if (stage) k_near<true, true><<<g, 128, nsm, s>>>(NA);
    else k_near<false, true><<<g, 128, nsm, s>>>(NA);
  } else if (part == 1) {  // smooth-rule subtraction only (NEXT-4 mode)
    if (stage) k_near<true, false, 1><<<g, 128, nsm, s>>>(NA);
    else k_near<false, false, 1><<<g, 128, nsm, s>>>(NA);
  } else if (part == 2) {  // exterior part only (measurement)
    if (near2_stage(c->p)) k_near<true, false, 2><<<g, 128, nsm2, s>>>(NA);
    else k_near<false, false, 2><<<g, 128, nsm, s>>>(NA);
  } else {
    if (stage) k_near<true, false><<<g, 128, nsm, s>>>(NA);
    else k_near<false, false><<<g, 128, nsm, s>>>(NA);
  }
  prof_end(c, s, &ev);
  return launch_check(c, K ? "k_near<K>" : "k_near");
}

// Near correction at m arbitrary targets: velocity (+ pressure when p) or,
// with target normals tn, traction (K).  Accumulates onto u (and p).
// Carves 256-byte-aligned arrays out of one scratch buffer (base == nullptr:
// sizing pass).
struct Carve {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    T* r = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return r;
  }
};

static int grow(bie_ctx* c, void** buf, size_t* cap, size_t need, const char* what) {
  if (need <= *cap) return BIE_OK;
  cudaFree(*buf);
  *buf = nullptr;
  *cap = 0;
  if (cudaMalloc(buf, need) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, BIE_ERR_ALLOC, "%s scratch", what);
  }
  *cap = need;
  return BIE_OK;
}

// Grouped schedule of the off-surface near correction (k_near.cuh): pairs
// (target, near sphere) listed per target, grouped by sphere with a stable
// radix sort, evaluated one CTA per (sphere, chunk), summed per target.  One
// stream synchronisation reads the pair count (it sizes the pair arrays).
static int run_near_off_grp(bie_ctx* c, NearOffArgs NO, cudaStream_t s) {
  const int64_t m = NO.M, ns = c->ns;
  NearGrp G{};
  // per-target arrays and the scan of the counts
  size_t scan_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (const int*)nullptr, (int*)nullptr, (int)(m + 1), s);
  auto carve1 = [&](char* base, size_t* total) {
    Carve cv{base};
    G.cnt = cv.take<int>(m + 1);
    G.off = cv.take<int>(m + 1);
    void* tmp = cv.take<char>(scan_tmp);
    *total = cv.off;
    return tmp;
  };
  size_t need1 = 0;
  carve1(nullptr, &need1);
  int rc = grow(c, &c->d_grp1, &c->grp1_cap, need1, "near pair count");
  if (rc) return rc;
  void* scan1 = carve1(static_cast<char*>(c->d_grp1), &need1);
  Ev ev;
  prof_begin(c, BIE_KIND_NEAR, s, &ev);
  cudaMemsetAsync(G.cnt + m, 0, sizeof(int), s);
  const unsigned gt = (unsigned)((m + 127) / 128);
  k_noff_pairs<false><<<gt, 128, 0, s>>>(NO, G);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(scan1, scan_tmp, G.cnt, const_cast<int*>(G.off), (int)(m + 1), s);
  if (e != cudaSuccess) return cuda_fail(c, e, "near pair scan");
  int P = 0;
  e = cudaMemcpyAsync(&P, G.off + m, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(c, e, "near pair count");
  prof_end(c, s, &ev);
  c->launches[BIE_KIND_NEAR] += 2;  // k_noff_pairs + the scan's two kernels (one counted)
  if (P == 0) return BIE_OK;
  // per-pair and per-sphere arrays
  int bits = 1;
  while (bits < 31 && (1LL << bits) <= ns) ++bits;
  size_t sort_tmp = 0, sscan_tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (const int*)nullptr, (int*)nullptr, (const int*)nullptr,
                                  (int*)nullptr, P, 0, bits, s);
  cub::DeviceScan::ExclusiveSum(nullptr, sscan_tmp, (const int*)nullptr, (int*)nullptr, (int)(ns + 1), s);
  int* sorted_s = nullptr;
  void *stmp = nullptr, *sctmp = nullptr;
  auto carve2 = [&](char* base) {
    Carve cv{base};
    G.pair_s = cv.take<int>(P);
    G.pair_t = cv.take<int>(P);
    G.pair_j = cv.take<int>(P);
    sorted_s = cv.take<int>(P);
    G.sorted_j = cv.take<int>(P);
    G.res = cv.take<double>(4 * (size_t)P);
    G.scount = cv.take<int>(ns + 1);
    G.nch = cv.take<int>(ns + 1);
    G.sfirst = cv.take<int>(ns + 1);
    G.choff = cv.take<int>(ns + 1);
    stmp = cv.take<char>(sort_tmp);
    sctmp = cv.take<char>(sscan_tmp);
    return cv.off;
  };
  if ((rc = grow(c, &c->d_grp2, &c->grp2_cap, carve2(nullptr), "near pair"))) return rc;
  carve2(static_cast<char*>(c->d_grp2));
  prof_begin(c, BIE_KIND_NEAR, s, &ev);
  cudaMemsetAsync(G.scount, 0, (ns + 1) * sizeof(int), s);
  cudaMemsetAsync(G.nch, 0, (ns + 1) * sizeof(int), s);
  k_noff_pairs<true><<<gt, 128, 0, s>>>(NO, G);
  e = cub::DeviceRadixSort::SortPairs(stmp, sort_tmp, G.pair_s, sorted_s, G.pair_j, const_cast<int*>(G.sorted_j),
                                      P, 0, bits, s);
  if (e == cudaSuccess) {
    k_noff_nch<<<(unsigned)((ns + 255) / 256), 256, 0, s>>>(ns, G.scount, G.nch);
    e = cub::DeviceScan::ExclusiveSum(sctmp, sscan_tmp, G.scount, const_cast<int*>(G.sfirst), (int)(ns + 1), s);
  }
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(sctmp, sscan_tmp, G.nch, const_cast<int*>(G.choff), (int)(ns + 1), s);
  if (e != cudaSuccess) return cuda_fail(c, e, "near pair grouping");
  // chunks <= P / kGrpChunk + (spheres with pairs) <= P / kGrpChunk + min(ns, P)
  const unsigned gb = (unsigned)((P + kGrpChunk - 1) / kGrpChunk + std::min<int64_t>(ns, P));
  const bool stage = noff_grp_stage(c->p);
  const size_t sm = noff_grp_smem_doubles(c->p, stage) * sizeof(double);
  const bool K = NO.tn != nullptr, pr = !K && NO.pres;
#define NOFF_GRP(PR, KK)                                                                       \
  do {                                                                                         \
    if (stage) {                                                                               \
      cudaFuncSetAttribute(k_noff_grp<PR, KK, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
      k_noff_grp<PR, KK, true><<<gb, kGrpChunk, sm, s>>>(NO, G);                               \
    } else {                                                                                   \
      cudaFuncSetAttribute(k_noff_grp<PR, KK, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
      k_noff_grp<PR, KK, false><<<gb, kGrpChunk, sm, s>>>(NO, G);                              \
    }                                                                                          \
  } while (0)
  if (K) NOFF_GRP(false, true);
  else if (pr) NOFF_GRP(true, false);
  else NOFF_GRP(false, false);
#undef NOFF_GRP
  if (pr) k_noff_sum<true><<<gt, 128, 0, s>>>(NO, G);
  else k_noff_sum<false><<<gt, 128, 0, s>>>(NO, G);
  prof_end(c, s, &ev);
  // k_noff_pairs, radix sort (histogram, scan, 2 onesweep passes for <= 16 key
  // bits), k_noff_nch, two scans (2 kernels each), k_noff_grp, k_noff_sum
  c->launches[BIE_KIND_NEAR] += 11 + (bits > 16 ? 2 : 0);
  return launch_check(c, K ? "k_noff_grp<K>" : "k_noff_grp");
}

static int run_near_off(bie_ctx* c, const double* tg, const double* tn, int64_t m, double* u,
                        double* p, cudaStream_t s) {
  NearOffArgs NO;
  NO.p = c->p;
  NO.nsn = c->nsn;
  NO.ns = c->ns;
  NO.M = m;
  NO.mu = c->mu;
  NO.eta = c->eta;
  NO.tab = c->d_tab;
  NO.centres = c->d_centres;
  NO.radii = c->d_radii;
  NO.rec = c->d_rec;
  NO.qn3 = tn ? nullptr : c->d_qn3;
  NO.coef = c->d_ncoef;
  NO.tx = tg;
  NO.tn = tn;
  NO.u = u;
  NO.pres = tn ? nullptr : p;
  NO.cell_start = c->d_cell_start;
  NO.cell_items = c->d_cell_items;
  NO.g0x = c->g0[0];
  NO.g0y = c->g0[1];
  NO.g0z = c->g0[2];
  NO.gh = c->gh;
  NO.gnx = c->gn[0];
  NO.gny = c->gn[1];
  NO.gnz = c->gn[2];
  if (c->noff_sched == 0 && m < (int64_t)INT32_MAX) return run_near_off_grp(c, NO, s);
  // process the targets in Morton order of their grid cell: neighbouring lanes
  // then share near spheres (coefficients and records hit L1 instead of L2)
  if (m <= (int64_t)INT32_MAX) {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const int*)nullptr, (int*)nullptr, (int)m, 0, 30, s);
    const size_t need = 2 * m * sizeof(uint32_t) + 2 * m * sizeof(int) + tmp + 256;
    if (need > c->sort_cap) {
      cudaFree(c->d_sort);
      c->d_sort = nullptr;
      c->sort_cap = 0;
      if (cudaMalloc(&c->d_sort, need) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, BIE_ERR_ALLOC, "near target sort scratch%s");
      }
      c->sort_cap = need;
    }
    char* b = static_cast<char*>(c->d_sort);
    uint32_t* k_in = reinterpret_cast<uint32_t*>(b);
    uint32_t* k_out = k_in + m;
    int* i_in = reinterpret_cast<int*>(k_out + m);
    int* i_out = i_in + m;
    void* tmpb = reinterpret_cast<void*>(((uintptr_t)(i_out + m) + 255) & ~(uintptr_t)255);
    Ev ev0;
    prof_begin(c, BIE_KIND_NEAR, s, &ev0);
    k_morton<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, tg, c->g0[0], c->g0[1], c->g0[2], c->gh, k_in,
                                                        i_in);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(tmpb, tmp, k_in, k_out, i_in, i_out, (int)m, 0, 30, s);
    prof_end(c, s, &ev0);
    if (e != cudaSuccess) return cuda_fail(c, e, "near target sort");
    NO.order = i_out;
  }
  const size_t sm = near_off_smem_doubles(c->p) * sizeof(double);
  const unsigned g = (unsigned)((m + 127) / 128);
  Ev ev;
  prof_begin(c, BIE_KIND_NEAR, s, &ev);
  if (tn) k_near_off<false, true><<<g, 128, sm, s>>>(NO);
  else if (p) k_near_off<true, false><<<g, 128, sm, s>>>(NO);
  else k_near_off<false, false><<<g, 128, sm, s>>>(NO);
  prof_end(c, s, &ev);
  return launch_check(c, tn ? "k_near_off<K>" : "k_near_off");
}

// NEXT-4 (PAPER §4.2): neighbours' exact fields re-expanded on each target
// sphere through rotations (k_n4), accumulated in coefficient space.
static int run_n4(bie_ctx* c, cudaStream_t s) {
  const TableLayout L(c->p);
  if (cudaMemsetAsync(c->d_psinear, 0, (size_t)c->ns * L.nlm * 6 * sizeof(double), s) != cudaSuccess)
    return cuda_fail(c, cudaGetLastError(), "NEXT-4 psi reset");
  if (c->n_near_tgt == 0) return BIE_OK;
  N4Args NA;
  NA.p = c->p;
  NA.nsn = c->nsn;
  NA.tab = c->d_tab;
  NA.centres = c->d_centres;
  NA.radii = c->d_radii;
  NA.coef = c->d_ncoef;
  NA.delta = c->d_delta;
  NA.deltaT = c->d_deltaT;
  NA.tgt = c->d_near_tgt;
  NA.nb_off = c->d_nb_off;
  NA.nb_idx = c->d_nb_idx;
  NA.psi = c->d_psinear;
  Ev ev;
  prof_begin(c, BIE_KIND_NEAR4, s, &ev);
  k_n4<<<(unsigned)c->n_near_tgt, 128, n4_smem_doubles(c->p) * sizeof(double), s>>>(NA);
  prof_end(c, s, &ev);
  return launch_check(c, "k_n4");
}

// Near pairs in the far field: excluded inside k_nbody (NX; the correction then
// only adds the exact field) or kept and subtracted by k_near.  Exclusion
// costs ~1.5 % of the far field (masked-tile bookkeeping),
// subtraction one smooth-rule pass per near pair at k_near's lower efficiency
// (~3x per pair): auto picks the cheaper.
static bool use_near_exclusion(const bie_ctx* c) {
  if (c->near_excl >= 0) return c->near_excl == 1;
  const double far_pairs = (double)c->N * (double)(c->N - c->nsn);
  const double sub_pairs = (double)c->n_near_pairs * (double)c->nsn * (double)c->nsn;
  return 0.015 * far_pairs < 3.0 * sub_pairs;
}

static int run_apply(bie_ctx* c, const double* f, const double* q, double* u, int parts,
                     cudaStream_t s) {
  // rows a2 + a4-a6: self term (or zeros) into u, packed sources into d_rec
  const bool near = (parts & BIE_PART_FAR) && c->n_near_tgt > 0;
  const bool n4 = near && (c->near_mode == 1 || c->near_mode == 3);
  SelfArgs SA =
      self_args(c, f, q, u, (parts & BIE_PART_SELF) && !n4 ? 1 : 0, near ? c->d_alpha : nullptr, 0);
  Ev ev;
  prof_begin(c, BIE_KIND_SELF, s, &ev);
  self_launch(c, SA, s);
  prof_end(c, s, &ev);
  int rc = launch_check(c, "k_self");
  if (rc) return rc;
  if (!(parts & BIE_PART_FAR)) return BIE_OK;
  if (near) {
    rc = run_near_coef(c, s);
    if (rc) return rc;
  }
  if (n4) {
    // exact near fields as coefficients, then the self term's single inverse
    // transform evaluates self + neighbours together
    if ((rc = run_n4(c, s))) return rc;
    SA = self_args(c, f, q, u, 1, nullptr, 0);
    SA.psinear = c->d_psinear;
    if (!(parts & BIE_PART_SELF)) SA.self = 2;  // far only: synthesise the neighbours' psi alone
    prof_begin(c, BIE_KIND_SELF, s, &ev);
    self_launch(c, SA, s);
    prof_end(c, s, &ev);
    if ((rc = launch_check(c, "k_self(NEXT-4)"))) return rc;
  }
  // near pairs (modes 0, 1): excluded from the smooth rule (k_nbody NX) so the
  // correction only ADDS the exact exterior field, or kept and subtracted by
  // k_near (use_near_exclusion).  NEXT-1: k_near's exterior part (- smooth);
  // NEXT-4: the exterior part is already in u through the self term's
  // coefficients (k_near: - smooth only, when not excluded).  Modes 2/3
  // (measurement): the exterior part alone, smooth rule kept.
  const bool nx = near && (c->near_mode == 0 || c->near_mode == 1) && use_near_exclusion(c);
  rc = run_far(c, u, s, 0, nx);
  if (rc || !near) return rc;
  if (c->near_mode == 3 || (c->near_mode == 1 && nx)) return BIE_OK;
  const int part = c->near_mode == 2 || nx ? 2 : (c->near_mode == 1 ? 1 : 0);
  return run_near(c, u, s, false, part);
}

// Launch a cluster-reduced far-field kernel: n_tt clusters of cl CTAs.
template <class Kern>
static cudaError_t launch_cluster(Kern kern, int n_tt, size_t smem, cudaStream_t s, const NbodyArgs& A,
                                  int cl = kCL) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((int64_t)n_tt * cl));
  cfg.blockDim = dim3(kTPB);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, A);
}

// The cluster size of the on-chip (DSMEM) chunk reduction, or 0 for HBM
// partials + k_reduce: clusters only when selected (bie_set_far_reduction), the
// launch leaves >= 16 units per resident slot and no chunk count is forced.
// (Measured on cfg 5, profiles/r02_far_reduction.jsonl: see DESIGN.md §5.)
static int cluster_size(const bie_ctx* c, const ChunkPlan& P, int occ, int64_t n_src_tiles, bool apply) {
  if (c->chunks_override > 0 || c->far_red < 2 || c->far_red > 4) return 0;
  const int cl = !apply ? kCL : (c->far_red == 3 ? 4 : (c->far_red == 4 ? 16 : kCL));
  const int64_t slots = (int64_t)c->sm_count * std::max(occ, 1);
  return (P.n_chunks > 1 && n_src_tiles >= 2 * cl && (int64_t)P.n_tt * cl >= 16 * slots) ? cl : 0;
}

// Stream-K far field (default schedule; k_nbody_sk + k_sk_fixup): G = one
// persistent CTA per resident slot, equal contiguous ranges of (target tile,
// source tile) units.  `which`: 0 apply, 1 off-surface, 2 K, 3 off-surface K.
template <class Kern, class Fix>
static int run_sk(bie_ctx* c, Kern kern, Fix fix, int which, int r, int nc, NbodyArgs A, size_t smem,
                  int kind, cudaStream_t s) {
  SkArgs K;
  K.A = A;
  K.S = (A.N + kTS - 1) / kTS;
  K.A.n_tt = (int)((A.M + (int64_t)r * kTPB - 1) / ((int64_t)r * kTPB));
  K.T = (int64_t)K.A.n_tt * K.S;
  K.G = std::max<int64_t>(1, std::min<int64_t>((int64_t)c->sm_count * c->occ_sk[which], K.T));
  int rc = ensure_part(c, (size_t)2 * K.G * nc * r * kTPB);
  if (rc) return rc;
  K.part = c->d_part;
  Ev ev;
  prof_begin(c, kind, s, &ev);
  kern<<<(unsigned)K.G, kTPB, smem, s>>>(K);
  if (K.G > 1) fix<<<(unsigned)(K.G - 1), 256, 0, s>>>(K);
  prof_end(c, s, &ev);
  c->launches[kind] += K.G > 1 ? 1 : 0;
  return launch_check(c, "k_nbody_sk");
}

// row a3: far-field smooth sum over all other spheres, accumulated onto u

// Which launches take the constant-bank schedule: asked for (7), or by default
// (1) when one launch (all targets x one batch) nearly fills the GPU -- at
// least 0.8 waves of target tiles (242,483 targets on 148 SMs; the two streams
// keep two launches in flight) -- and there are at least 16 batches of
// sources.  Measured on lattices of unit spheres, p = 6 (tools/const_threshold.py,
// profiles/r02_const_threshold.jsonl), k_nbody / k_nbody_c time: 98,000 nodes
// 0.73, 196,000 1.01, 294,000 1.056, 392,000 1.052, 607,600 1.057, 980,000
// 1.054; cfg 3 (162,000 nodes) 0.94.
static bool use_const(const bie_ctx* c, int64_t M, int R) {
  if (c->chunks_override != 0) return false;
  if (c->far_red == 7) return true;
  if (c->far_red != 1) return false;
  return 5 * M >= (int64_t)4 * c->sm_count * 4 * kTPB * R && c->N >= (int64_t)16 * kCB;
}

// Constant-bank far field (bie_set_far_reduction 7; k_nbody_c.cuh): batches of
// kCB sources, even batches on the caller's stream into `acc` (which already
// holds the self term / zeros), odd batches on the context's side stream into
// the scratch accumulator, joined by k_nbody_c_join.  The two constant buffers
// belong to the process's CUDA module, not to a context: passes of different
// contexts on one device are ordered one after the other by an event (the
// enqueue runs under a mutex), so distinct contexts stay independent.
static std::mutex g_cb_mu;
static cudaEvent_t g_cb_done[64] = {};

template <bool OFF>
static int run_const_pass(bie_ctx* c, const double* tx, int64_t M, double* acc, double* pout, int kind,
                          cudaStream_t s) {
  constexpr int R = OFF ? kR_OFF_C : kR_APPLY_C;
  Ev ev;
  int rc;
  if (c->dev < 0 || c->dev >= 64) return fail(c, BIE_ERR_UNSUPPORTED, "constant-bank far field: device index%s");
  if (!c->st_side) {
    cudaError_t e = cudaStreamCreateWithFlags(&c->st_side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(c, e, "constant-bank far field: side stream");
  }
  const bool wp = OFF && pout != nullptr;
  // Target sub-ranges: every launch re-reads and re-writes the accumulators of
  // its targets, and they only stay in L2 between launches while targets + both
  // accumulators fit well inside it (measured DRAM per launch: 2.9 MB at 70 MB,
  // 23.7 MB at 88 MB) -- so a pass walks the targets in
  // sub-ranges of <= c->const_sub targets, each against every batch.
  const int64_t tile = (int64_t)kTPB * R;
  const int64_t nsub = c->const_sub > 0 ? (M + c->const_sub - 1) / c->const_sub : 1;
  const int64_t msub = ((M + nsub - 1) / nsub + tile - 1) / tile * tile;
  if ((rc = ensure_part(c, (size_t)(wp ? 4 : 3) * std::min(M, msub)))) return rc;
  const int64_t nb = (c->N + kCB - 1) / kCB;
  std::lock_guard<std::mutex> lk(g_cb_mu);
  cudaEvent_t& done = g_cb_done[c->dev];
  cudaError_t e = cudaSuccess;
  if (!done) e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
  else e = cudaStreamWaitEvent(s, done, 0);
  if (e != cudaSuccess) return cuda_fail(c, e, "constant-bank far field: ordering event");
  prof_begin(c, kind, s, &ev);
  for (int64_t m0 = 0; m0 < M && e == cudaSuccess; m0 += msub) {
    const int64_t Ms = std::min(msub, M - m0);
    double* accA = acc + 3 * m0;
    double* pA = wp ? pout + m0 : nullptr;
    double* accB = c->d_part;
    double* pB = wp ? c->d_part + 3 * Ms : nullptr;
    const unsigned grid = (unsigned)((Ms + tile - 1) / tile);
    cudaMemsetAsync(accB, 0, (size_t)(wp ? 4 : 3) * Ms * sizeof(double), s);
    cudaEventRecord(c->ev_fork, s);
    cudaStreamWaitEvent(c->st_side, c->ev_fork, 0);
    for (int64_t b = 0; b < nb && e == cudaSuccess; ++b) {
      const int w = (int)(b & 1);
      cudaStream_t sb = w ? c->st_side : s;
      NbodyCArgs A;
      A.tx = tx + 3 * m0;
      A.acc = w ? accB : accA;
      A.pacc = wp ? (w ? pB : pA) : nullptr;
      A.M = Ms;
      A.k0 = b * kCB;
      A.tbase = m0;
      A.ks = (int)std::min<int64_t>(kCB, c->N - A.k0);
      A.nsn = c->nsn;
      e = cudaMemcpyToSymbolAsync(c_nb_rec, c->d_rec + A.k0 * kRec, (size_t)A.ks * kRec * sizeof(double),
                                  (size_t)w * kCB * kRec * sizeof(double), cudaMemcpyDeviceToDevice, sb);
      if (e == cudaSuccess && OFF)
        e = cudaMemcpyToSymbolAsync(c_nb_qn, c->d_qn3 + A.k0, (size_t)A.ks * sizeof(double),
                                    (size_t)w * kCB * sizeof(double), cudaMemcpyDeviceToDevice, sb);
      if (e != cudaSuccess) break;
      constexpr int UNR = OFF ? kUNR_OFF_C : kUNR_C;
      if (w) k_nbody_c<R, kTPB, UNR, 1, OFF><<<grid, kTPB, 0, sb>>>(A);
      else k_nbody_c<R, kTPB, UNR, 0, OFF><<<grid, kTPB, 0, sb>>>(A);
    }
    cudaEventRecord(c->ev_join, c->st_side);
    cudaStreamWaitEvent(s, c->ev_join, 0);
    k_nbody_c_join<<<(unsigned)((3 * Ms + 255) / 256), 256, 0, s>>>(Ms, accA, accB, pA, pB, 2.0 * c->mu);
    c->launches[kind] += nb + (m0 ? 1 : 0);  // prof_begin counted the first join
  }
  prof_end(c, s, &ev);
  cudaEventRecord(done, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "constant-bank far field: batch copy");
  return launch_check(c, OFF ? "k_nbody_c (off-surface)" : "k_nbody_c");
}

static int run_far(bie_ctx* c, double* u, cudaStream_t s, int mode, bool nx) {
  if (mode == 0 && !nx && use_const(c, c->N, kR_APPLY_C))
    return run_const_pass<false>(c, c->d_x, c->N, u, nullptr, BIE_KIND_NBODY, s);
  Ev ev;
  int rc;
  const ChunkPlan P = plan_chunks(c, c->N, c->N,
                                  mode ? (nx ? c->occ_K_nx : c->occ_K) : (nx ? c->occ_apply_nx : c->occ_apply),
                                  mode ? kR_K : kR_APPLY);
  const int kind = mode ? BIE_KIND_KFAR : BIE_KIND_NBODY;
  NbodyArgs A;
  A.rec = c->d_rec;
  A.qn3 = nullptr;
  A.tx = nullptr;
  A.txa = c->d_x;  // compact target positions / normals (not the 96-byte records)
  A.tna = c->d_n;
  A.N = c->N;
  A.M = c->N;
  A.nsn = c->nsn;
  A.n_tt = P.n_tt;
  A.n_chunks = P.n_chunks;
  A.tiles_per_chunk = P.tiles_per_chunk;
  A.pscale = 2.0 * c->mu;
  A.pout = nullptr;
  const size_t nb_smem = NbodySmem<kTS, kNST, false>::kBytes;
  const int64_t n_src_tiles = (c->N + kTS - 1) / kTS;
  if (nx) {  // near exclusion (chunked schedule): neighbour pairs skipped by the smooth rule
    A.nb_off = c->d_nb_off;
    A.nb_idx = c->d_nb_idx;
    const size_t sm_nx = nb_smem + kNxBytes;
    if (P.n_chunks == 1) {
      A.uinit = u;
      A.uout = u;
      prof_begin(c, kind, s, &ev);
      if (mode) NBODY_K_NX<<<(unsigned)P.n_tt, kTPB, sm_nx, s>>>(A);
      else NBODY_APPLY_NX<<<(unsigned)P.n_tt, kTPB, sm_nx, s>>>(A);
      prof_end(c, s, &ev);
      return launch_check(c, "k_nbody (near exclusion)");
    }
    const bool chain = use_chain(c, P, mode ? c->occ_K_nx : c->occ_apply_nx);
    if (chain) {
      if ((rc = setup_chain(c, A, c->N, s))) return rc;
      A.uinit = u;
      A.uout = u;
    } else {
      if ((rc = ensure_part(c, (size_t)P.n_chunks * 3 * c->N))) return rc;
      A.uinit = nullptr;
      A.uout = c->d_part;
    }
    prof_begin(c, kind, s, &ev);
    if (mode) NBODY_K_NX<<<(unsigned)((int64_t)P.n_tt * P.n_chunks), kTPB, sm_nx, s>>>(A);
    else NBODY_APPLY_NX<<<(unsigned)((int64_t)P.n_tt * P.n_chunks), kTPB, sm_nx, s>>>(A);
    prof_end(c, s, &ev);
    if ((rc = launch_check(c, "k_nbody (near exclusion)"))) return rc;
    if (chain) return BIE_OK;
    prof_begin(c, BIE_KIND_REDUCE, s, &ev);
    k_reduce<<<(unsigned)((3 * c->N + 255) / 256), 256, 0, s>>>(c->N, P.n_chunks, c->d_part, u, u, nullptr,
                                                                 nullptr, 0.0);
    prof_end(c, s, &ev);
    return launch_check(c, "k_reduce");
  }
  if (c->far_red == 0 && c->chunks_override == 0) {
    A.uinit = u;
    A.uout = u;
    return mode ? run_sk(c, NBODY_K_SK, k_sk_fixup<kR_K * kTPB, false>, 2, kR_K, 3, A, nb_smem, kind, s)
                : run_sk(c, NBODY_APPLY_SK, k_sk_fixup<kR_APPLY * kTPB, false>, 0, kR_APPLY, 3, A, nb_smem,
                         kind, s);
  }
  if (const int cl = cluster_size(c, P, mode ? c->occ_K : c->occ_apply, n_src_tiles, mode == 0)) {
    A.n_chunks = cl;
    A.tiles_per_chunk = (int)((n_src_tiles + cl - 1) / cl);
    A.uinit = u;
    A.uout = u;
    prof_begin(c, kind, s, &ev);
    const cudaError_t e =
        mode ? launch_cluster(NBODY_K_CL, P.n_tt, nb_smem, s, A)
             : (cl == 4 ? launch_cluster(NBODY_APPLY_CL4, P.n_tt, nb_smem, s, A, 4)
                        : (cl == 16 ? launch_cluster(NBODY_APPLY_CL16, P.n_tt, nb_smem, s, A, 16)
                                    : launch_cluster(NBODY_APPLY_CL, P.n_tt, nb_smem, s, A)));
    prof_end(c, s, &ev);
    if (e != cudaSuccess) return cuda_fail(c, e, "k_nbody (cluster)");
    return launch_check(c, "k_nbody (cluster)");
  }
  if (P.n_chunks == 1) {
    A.uinit = u;
    A.uout = u;
    prof_begin(c, kind, s, &ev);
    if (mode) NBODY_K<<<(unsigned)P.n_tt, kTPB, nb_smem, s>>>(A);
    else NBODY_APPLY<<<(unsigned)P.n_tt, kTPB, nb_smem, s>>>(A);
    prof_end(c, s, &ev);
    return launch_check(c, "k_nbody");
  }
  const bool chain = use_chain(c, P, mode ? c->occ_K : c->occ_apply);
  if (chain) {
    if ((rc = setup_chain(c, A, c->N, s))) return rc;
    A.uinit = u;
    A.uout = u;
  } else {
    rc = ensure_part(c, (size_t)P.n_chunks * 3 * c->N);
    if (rc) return rc;
    A.uinit = nullptr;
    A.uout = c->d_part;
  }
  prof_begin(c, kind, s, &ev);
  if (mode) NBODY_K<<<(unsigned)((int64_t)P.n_tt * P.n_chunks), kTPB, nb_smem, s>>>(A);
  else NBODY_APPLY<<<(unsigned)((int64_t)P.n_tt * P.n_chunks), kTPB, nb_smem, s>>>(A);
  prof_end(c, s, &ev);
  rc = launch_check(c, "k_nbody");
  if (rc) return rc;
  if (chain) return BIE_OK;
  prof_begin(c, BIE_KIND_REDUCE, s, &ev);
  k_reduce<<<(unsigned)((3 * c->N + 255) / 256), 256, 0, s>>>(c->N, P.n_chunks, c->d_part, u, u,
                                                               nullptr, nullptr, 0.0);
  prof_end(c, s, &ev);
  return launch_check(c, "k_reduce");
}

static int run_offsurface(bie_ctx* c, const double* f, const double* q, const double* tg,
                          int64_t m, double* u, double* p, cudaStream_t s) {
  if (m == 0) return BIE_OK;
  Ev ev;
  const bool near = c->eta > 0.0 && c->d_alpha;
  int rc;
  if (near) {  // NEXT-1 at targets: VSH projections of every sphere, then coefficients
    const SelfArgs SA = self_args(c, f, q, nullptr, 0, c->d_alpha, 0);
    prof_begin(c, BIE_KIND_SELF, s, &ev);
    self_launch(c, SA, s);
    prof_end(c, s, &ev);
    if ((rc = launch_check(c, "k_self"))) return rc;
    if ((rc = run_near_coef(c, s))) return rc;
  }
  prof_begin(c, BIE_KIND_PACK, s, &ev);
  k_pack<<<(unsigned)((c->N + 255) / 256), 256, 0, s>>>(c->p, c->N, c->mu, c->d_tab, c->d_centres,
                                                        c->d_radii, f, q, c->d_rec, c->d_qn3);
  prof_end(c, s, &ev);
  rc = launch_check(c, "k_pack");
  if (rc) return rc;
  const size_t nb_smem = NbodySmem<kTS, kNST, true>::kBytes;
  for (int64_t b0 = 0; b0 < m; b0 += kOffBatch) {
    const int64_t Mb = std::min(kOffBatch, m - b0);
    if (use_const(c, Mb, kR_OFF_C)) {  // constant-bank batches (k_nbody_c.cuh)
      cudaMemsetAsync(u + 3 * b0, 0, (size_t)3 * Mb * sizeof(double), s);
      if (p) cudaMemsetAsync(p + b0, 0, (size_t)Mb * sizeof(double), s);
      if ((rc = run_const_pass<true>(c, tg + 3 * b0, Mb, u + 3 * b0, p ? p + b0 : nullptr, BIE_KIND_OFFSURF, s)))
        return rc;
      continue;
    }
    const ChunkPlan P = plan_chunks(c, Mb, c->N, c->occ_off, kR_OFF);
    NbodyArgs A;
    A.rec = c->d_rec;
    A.qn3 = c->d_qn3;
    A.tx = tg + 3 * b0;
    A.uinit = nullptr;
    A.N = c->N;
    A.M = Mb;
    A.nsn = c->nsn;
    A.n_tt = P.n_tt;
    A.n_chunks = P.n_chunks;
    A.tiles_per_chunk = P.tiles_per_chunk;
    A.pscale = 2.0 * c->mu;
    const int64_t n_src_tiles = (c->N + kTS - 1) / kTS;
    if (c->far_red == 0 && c->chunks_override == 0) {
      A.uout = u + 3 * b0;
      A.pout = p ? p + b0 : nullptr;
      if ((rc = run_sk(c, NBODY_OFF_SK, k_sk_fixup<kR_OFF * kTPB, true>, 1, kR_OFF, 4, A, nb_smem,
                       BIE_KIND_OFFSURF, s)))
        return rc;
      continue;
    }
    if (cluster_size(c, P, c->occ_off, n_src_tiles, false)) {
      A.n_chunks = kCL;
      A.tiles_per_chunk = (int)((n_src_tiles + kCL - 1) / kCL);
      A.uout = u + 3 * b0;
      A.pout = p ? p + b0 : nullptr;
      prof_begin(c, BIE_KIND_OFFSURF, s, &ev);
      const cudaError_t e = launch_cluster(NBODY_OFF_CL, P.n_tt, nb_smem, s, A);
      prof_end(c, s, &ev);
      if (e != cudaSuccess) return cuda_fail(c, e, "k_nbody_off (cluster)");
      if ((rc = launch_check(c, "k_nbody_off (cluster)"))) return rc;
      continue;
    }
    if (P.n_chunks == 1) {
      A.uout = u + 3 * b0;
      A.pout = p ? p + b0 : nullptr;
      prof_begin(c, BIE_KIND_OFFSURF, s, &ev);
      NBODY_OFF<<<(unsigned)P.n_tt, kTPB, nb_smem, s>>>(A);
      prof_end(c, s, &ev);
      rc = launch_check(c, "k_nbody_off");
      if (rc) return rc;
      continue;
    }
    const bool chain = use_chain(c, P, c->occ_off);
    if (chain) {
      if ((rc = setup_chain(c, A, Mb, s))) return rc;
      A.uout = u + 3 * b0;
      A.pout = p ? p + b0 : nullptr;
    } else {
      rc = ensure_part(c, (size_t)P.n_chunks * 4 * Mb);
      if (rc) return rc;
      A.uout = c->d_part;
      A.pout = p ? c->d_part + (size_t)P.n_chunks * 3 * Mb : nullptr;
    }
    prof_begin(c, BIE_KIND_OFFSURF, s, &ev);
    NBODY_OFF<<<(unsigned)((int64_t)P.n_tt * P.n_chunks), kTPB, nb_smem, s>>>(A);
    prof_end(c, s, &ev);
    rc = launch_check(c, "k_nbody_off");
    if (rc) return rc;
    if (chain) continue;
    prof_begin(c, BIE_KIND_REDUCE, s, &ev);
    k_reduce<<<(unsigned)((3 * Mb + 255) / 256), 256, 0, s>>>(
        Mb, P.n_chunks, c->d_part, nullptr, u + 3 * b0, A.pout, p ? p + b0 : nullptr, 2.0 * c->mu);
    prof_end(c, s, &ev);
    rc = launch_check(c, "k_reduce");
    if (rc) return rc;
  }
  if (!near) return BIE_OK;
  return run_near_off(c, tg, nullptr, m, u, p, s);
}

// NEXT-3 off the surface: traction K[sigma](x; n) at m targets with normals
static int run_traction(bie_ctx* c, const double* sigma, const double* tg, const double* tn,
                        int64_t m, double* t, cudaStream_t s) {
  Ev ev;
  int rc;
  const bool near = c->eta > 0.0 && c->d_alpha;
  if (near) {  // projections of sigma (q slot) -> exterior S coefficients
    const SelfArgs SA = self_args(c, nullptr, sigma, nullptr, 0, c->d_alpha, 0);
    prof_begin(c, BIE_KIND_SELF, s, &ev);
    self_launch(c, SA, s);
    prof_end(c, s, &ev);
    if ((rc = launch_check(c, "k_self"))) return rc;
    const TableLayout L(c->p);
    const int64_t n = c->ns * L.nlm;
    prof_begin(c, BIE_KIND_NEAR, s, &ev);
    k_near_coef_K<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(c->p, c->ns, c->d_alpha, c->d_ncoef);
    prof_end(c, s, &ev);
    if ((rc = launch_check(c, "k_near_coef_K"))) return rc;
  }
  prof_begin(c, BIE_KIND_PACK, s, &ev);  // q' = (3/4pi) w sigma
  k_pack<<<(unsigned)((c->N + 255) / 256), 256, 0, s>>>(c->p, c->N, c->mu, c->d_tab, c->d_centres,
                                                        c->d_radii, nullptr, sigma, c->d_rec, c->d_qn3);
  prof_end(c, s, &ev);
  if ((rc = launch_check(c, "k_pack"))) return rc;
  const size_t nb_smem = NbodySmem<kTS, kNST, true>::kBytes;
  for (int64_t b0 = 0; b0 < m; b0 += kOffBatch) {
    const int64_t Mb = std::min(kOffBatch, m - b0);
    const ChunkPlan P = plan_chunks(c, Mb, c->N, c->occ_offK, kR_OFFK);
    NbodyArgs A;
    A.rec = c->d_rec;
    A.qn3 = nullptr;
    A.tx = tg + 3 * b0;
    A.tn = tn + 3 * b0;
    A.uinit = nullptr;
    A.pout = nullptr;
    A.N = c->N;
    A.M = Mb;
    A.nsn = c->nsn;
    A.n_tt = P.n_tt;
    A.n_chunks = P.n_chunks;
    A.tiles_per_chunk = P.tiles_per_chunk;
    A.pscale = 0.0;
    const int64_t n_src_tiles = (c->N + kTS - 1) / kTS;
    if (c->far_red == 0 && c->chunks_override == 0) {
      A.uout = t + 3 * b0;
      if ((rc = run_sk(c, NBODY_OFFK_SK, k_sk_fixup<kR_OFFK * kTPB, true>, 3, kR_OFFK, 4, A, nb_smem,
                       BIE_KIND_KFAR, s)))
        return rc;
      continue;
    }
    if (cluster_size(c, P, c->occ_offK, n_src_tiles, false)) {
      A.n_chunks = kCL;
      A.tiles_per_chunk = (int)((n_src_tiles + kCL - 1) / kCL);
      A.uout = t + 3 * b0;
      prof_begin(c, BIE_KIND_KFAR, s, &ev);
      const cudaError_t e = launch_cluster(NBODY_OFFK_CL, P.n_tt, nb_smem, s, A);
      prof_end(c, s, &ev);
      if (e != cudaSuccess) return cuda_fail(c, e, "k_nbody_offK (cluster)");
      if ((rc = launch_check(c, "k_nbody_offK (cluster)"))) return rc;
      continue;
    }
    if (P.n_chunks == 1) {
      A.uout = t + 3 * b0;
      prof_begin(c, BIE_KIND_KFAR, s, &ev);
      NBODY_OFFK<<<(unsigned)P.n_tt, kTPB, nb_smem, s>>>(A);
      prof_end(c, s, &ev);
      if ((rc = launch_check(c, "k_nbody_offK"))) return rc;
      continue;
    }
    const bool chain = use_chain(c, P, c->occ_offK);
    if (chain) {
      if ((rc = setup_chain(c, A, Mb, s))) return rc;
      A.uout = t + 3 * b0;
    } else {
      if ((rc = ensure_part(c, (size_t)P.n_chunks * 4 * Mb))) return rc;
      A.uout = c->d_part;
    }
    prof_begin(c, BIE_KIND_KFAR, s, &ev);
    NBODY_OFFK<<<(unsigned)((int64_t)P.n_tt * P.n_chunks), kTPB, nb_smem, s>>>(A);
    prof_end(c, s, &ev);
    if ((rc = launch_check(c, "k_nbody_offK"))) return rc;
    if (chain) continue;
    prof_begin(c, BIE_KIND_REDUCE, s, &ev);
    k_reduce<<<(unsigned)((3 * Mb + 255) / 256), 256, 0, s>>>(Mb, P.n_chunks, c->d_part, nullptr,
                                                                t + 3 * b0, nullptr, nullptr, 0.0);
    prof_end(c, s, &ev);
    if ((rc = launch_check(c, "k_reduce"))) return rc;
  }
  if (!near) return BIE_OK;
  return run_near_off(c, tg, tn, m, t, nullptr, s);
}

// ================================================================ ABI
extern "C" {

const char* bie_status_string(int st) {
  switch (st) {
    case BIE_OK: return "ok";
    case BIE_ERR_ARG: return "invalid argument";
    case BIE_ERR_GEOMETRY: return "overlapping spheres";
    case BIE_ERR_ALLOC: return "device allocation failed";
    case BIE_ERR_CUDA: return "CUDA error";
    case BIE_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

const char* bie_last_error(const bie_ctx* c) { return c ? c->err.c_str() : "NULL context"; }

void bie_destroy(bie_ctx* c) {
  if (!c) return;
  prof_drain(c);
  double* ptrs[] = {c->d_centres, c->d_radii, c->d_tab, c->d_x, c->d_n, c->d_w, c->d_rec,
                    c->d_qn3, c->d_part, c->d_f, c->d_q, c->d_u, c->d_tg, c->d_uo, c->d_po, c->d_sht};
  for (double* p : ptrs)
    if (p) cudaFree(p);
  int* iptrs[] = {c->d_nb_off, c->d_nb_idx, c->d_near_tgt};
  for (int* p : iptrs)
    if (p) cudaFree(p);
  if (c->d_alpha) cudaFree(c->d_alpha);
  if (c->d_ncoef) cudaFree(c->d_ncoef);
  if (c->d_delta) cudaFree(c->d_delta);
  if (c->d_deltaT) cudaFree(c->d_deltaT);
  if (c->d_psinear) cudaFree(c->d_psinear);
  if (c->st_side) cudaStreamDestroy(c->st_side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  cudaFree(c->d_cacc);
  cudaFree(c->d_chain);
  cudaFree(c->d_cell_start);
  cudaFree(c->d_cell_items);
  cudaFree(c->d_sort);
  cudaFree(c->d_grp1);
  cudaFree(c->d_grp2);
  delete c;
}

int bie_create(const double* centres_h, const double* radii_h, int64_t n_spheres, int p, double mu,
               bie_ctx** out) {
  if (!out) return BIE_ERR_ARG;
  *out = nullptr;
  if (!centres_h || !radii_h || n_spheres < 1) return BIE_ERR_ARG;
  if (p < 1 || p > BIE_P_MAX) return BIE_ERR_UNSUPPORTED;
  if (!(mu > 0.0) || !std::isfinite(mu)) return BIE_ERR_ARG;
  for (int64_t i = 0; i < n_spheres; ++i) {
    if (!(radii_h[i] > 0.0) || !std::isfinite(radii_h[i])) return BIE_ERR_ARG;
    for (int d = 0; d < 3; ++d)
      if (!std::isfinite(centres_h[3 * i + d])) return BIE_ERR_ARG;
  }
  int64_t bi, bj;
  if (spheres_overlap(centres_h, radii_h, n_spheres, &bi, &bj)) return BIE_ERR_GEOMETRY;
  const int nsn = (p + 1) * (2 * p + 2);
  if (n_spheres > (int64_t)(INT32_MAX / nsn)) return BIE_ERR_UNSUPPORTED;  // int node indices

  bie_ctx* c = new bie_ctx();
  c->p = p;
  c->nsn = nsn;
  c->ns = n_spheres;
  c->N = n_spheres * nsn;
  c->mu = mu;
  cudaError_t e = cudaGetDevice(&c->dev);
  if (e != cudaSuccess) {
    delete c;
    cudaGetLastError();
    return BIE_ERR_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->dev) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return BIE_ERR_CUDA;
  }
  if (prop.major != 10 || prop.minor != 0) {
    delete c;
    return BIE_ERR_UNSUPPORTED;
  }
  c->sm_count = prop.multiProcessorCount;
  if (const char* ev_sub = std::getenv("BIE_CONST_SUB")) c->const_sub = std::atoll(ev_sub);  // tuning
  const TableLayout L(p);
  auto alloc = [&](double** ptr, size_t n) -> bool {
    return cudaMalloc(ptr, n * sizeof(double)) == cudaSuccess;
  };
  bool ok = alloc(&c->d_centres, 3 * n_spheres) && alloc(&c->d_radii, n_spheres) &&
            alloc(&c->d_tab, L.total) && alloc(&c->d_x, 3 * c->N) && alloc(&c->d_n, 3 * c->N) &&
            alloc(&c->d_w, c->N) && alloc(&c->d_rec, kRec * c->N + 2 * kRec) &&
            alloc(&c->d_qn3, c->N + 2) && alloc(&c->d_sht, ShtTabLayout(p).total);
  if (!ok) {
    cudaGetLastError();
    bie_destroy(c);
    return BIE_ERR_ALLOC;
  }
  if (cudaMemcpy(c->d_centres, centres_h, 3 * n_spheres * sizeof(double), cudaMemcpyHostToDevice) !=
          cudaSuccess ||
      cudaMemcpy(c->d_radii, radii_h, n_spheres * sizeof(double), cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    cudaGetLastError();
    bie_destroy(c);
    return BIE_ERR_CUDA;
  }
  // row a1: GL rule -> tables -> nodes (default stream, synchronous)
  Ev ev;
  prof_begin(c, BIE_KIND_SETUP, 0, &ev);
  k_gl_rule<<<1, 64>>>(p, c->d_tab);  // one thread per node, p + 1 <= 33
  k_tables<<<((p + 1) * (p + 1) + 127) / 128, 128>>>(p, c->d_tab);
  k_nodes<<<(unsigned)((c->N + 255) / 256), 256>>>(p, c->N, c->d_tab, c->d_centres, c->d_radii,
                                                  c->d_x, c->d_n, c->d_w);
  k_sht_tables<<<p + 5, 256>>>(p, c->d_tab, c->d_sht);
  c->launches[BIE_KIND_SETUP] += 3;  // prof_begin counted the first of the four
  prof_end(c, 0, &ev);
  set_self_smem(p);
  c->sht_occ = sht_prepare(p);
  if (c->sht_occ < 1) {  // table layouts disagree or no kernel for this order
    bie_destroy(c);
    return BIE_ERR_UNSUPPORTED;
  }
  // Dynamic shared memory opt-ins.  A staged near-correction variant whose
  // footprint exceeds the device limit is never launched (near_stage picks the
  // unstaged one), so it is skipped rather than requested.
  const size_t optin = (size_t)prop.sharedMemPerBlockOptin;
  cudaError_t se = cudaSuccess;
  auto smem = [&](const void* kern, size_t bytes) {
    if (bytes <= 48 * 1024 || bytes > optin) return;
    const cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (r != cudaSuccess && se == cudaSuccess) se = r;
  };
  const size_t near_st = near_smem_doubles(p, true) * sizeof(double);
  const size_t near_un = near_smem_doubles(p, false) * sizeof(double);
  const size_t near_off = near_off_smem_doubles(p) * sizeof(double);
  smem((const void*)k_near<true, false>, near_st);
  smem((const void*)k_near<false, false>, near_un);
  smem((const void*)k_near<true, false, 1>, near_st);
  smem((const void*)k_near<false, false, 1>, near_un);
  const size_t near_st2 = near2_smem_doubles(p) * sizeof(double);
  smem((const void*)k_near<true, false, 2>, near_st2);
  smem((const void*)k_near<false, false, 2>, near_un);
  smem((const void*)k_near<true, true, 2>, near_st2);
  smem((const void*)k_near<false, true, 2>, near_un);
  smem((const void*)k_near<true, true>, near_st);
  smem((const void*)k_near<false, true>, near_un);
  smem((const void*)k_near_off<true, false>, near_off);
  smem((const void*)k_near_off<false, false>, near_off);
  smem((const void*)k_near_off<false, true>, near_off);
  cudaFuncSetAttribute(NBODY_APPLY_CL16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_apply_nx, NBODY_APPLY_NX, kTPB,
                                                NbodySmem<kTS, kNST, false>::kBytes + kNxBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_K_nx, NBODY_K_NX, kTPB,
                                                NbodySmem<kTS, kNST, false>::kBytes + kNxBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_sk[0], NBODY_APPLY_SK, kTPB,
                                                NbodySmem<kTS, kNST, false>::kBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_sk[1], NBODY_OFF_SK, kTPB,
                                                NbodySmem<kTS, kNST, true>::kBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_sk[2], NBODY_K_SK, kTPB,
                                                NbodySmem<kTS, kNST, false>::kBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_sk[3], NBODY_OFFK_SK, kTPB,
                                                NbodySmem<kTS, kNST, true>::kBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_apply, NBODY_APPLY, kTPB,
                                                NbodySmem<kTS, kNST, false>::kBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_off, NBODY_OFF, kTPB,
                                                NbodySmem<kTS, kNST, true>::kBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_K, NBODY_K, kTPB,
                                                NbodySmem<kTS, kNST, false>::kBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_offK, NBODY_OFFK, kTPB,
                                                NbodySmem<kTS, kNST, true>::kBytes);
  if (se != cudaSuccess) {
    cudaGetLastError();
    bie_destroy(c);
    return BIE_ERR_CUDA;
  }
  e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    bie_destroy(c);
    return BIE_ERR_CUDA;
  }
  *out = c;
  return BIE_OK;
}

int64_t bie_num_nodes(const bie_ctx* c) { return c ? c->N : -1; }
int bie_order(const bie_ctx* c) { return c ? c->p : -1; }
int64_t bie_num_spheres(const bie_ctx* c) { return c ? c->ns : -1; }

int bie_get_nodes(const bie_ctx* cc, double* x, double* nrm, double* w, bie_stream_t s) {
  bie_ctx* c = const_cast<bie_ctx*>(cc);
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)s;
  const double* src[3] = {c->d_x, c->d_n, c->d_w};
  double* dst[3] = {x, nrm, w};
  const int64_t n[3] = {3 * c->N, 3 * c->N, c->N};
  for (int k = 0; k < 3; ++k) {
    if (!dst[k]) continue;
    if (!is_device_ptr(c, dst[k])) return fail(c, BIE_ERR_ARG, "bie_get_nodes: output %s is not a device pointer", k == 0 ? "x" : (k == 1 ? "normals" : "w"));
    cudaError_t e = cudaMemcpyAsync(dst[k], src[k], n[k] * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "bie_get_nodes");
  }
  return BIE_OK;
}

int bie_apply_parts(bie_ctx* c, const double* f, const double* q, double* u, int parts,
                    bie_stream_t s) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (parts <= 0 || parts > (BIE_PART_FAR | BIE_PART_SELF))
    return fail(c, BIE_ERR_ARG, "parts must be a non-empty subset of FAR|SELF%s");
  if (!u) return fail(c, BIE_ERR_ARG, "u is NULL%s");
  const int64_t n3 = 3 * c->N;
  if (!is_device_ptr(c, u)) return fail(c, BIE_ERR_ARG, "u is not a device pointer%s");
  if (f && !is_device_ptr(c, f)) return fail(c, BIE_ERR_ARG, "f is not a device pointer%s");
  if (q && !is_device_ptr(c, q)) return fail(c, BIE_ERR_ARG, "q is not a device pointer%s");
  if (overlaps(u, n3, f, n3) || overlaps(u, n3, q, n3))
    return fail(c, BIE_ERR_ARG, "output u overlaps an input%s");
  return run_apply(c, f, q, u, parts, (cudaStream_t)s);
}

int bie_apply_K(bie_ctx* c, const double* sigma, double* u, int parts, bie_stream_t st) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (parts <= 0 || parts > (BIE_PART_FAR | BIE_PART_SELF | BIE_PART_COMPLETION))
    return fail(c, BIE_ERR_ARG, "parts must be a non-empty subset of FAR|SELF|COMPLETION%s");
  const int64_t n3 = 3 * c->N;
  if (!sigma || !u || !is_device_ptr(c, sigma) || !is_device_ptr(c, u))
    return fail(c, BIE_ERR_ARG, "sigma and u must be device pointers%s");
  if (overlaps(u, n3, sigma, n3)) return fail(c, BIE_ERR_ARG, "output u overlaps sigma%s");
  cudaStream_t s = (cudaStream_t)st;
  // self term: K_pv has the D_pv spectrum; packs q' = (3/4pi) w sigma
  const bool near = (parts & BIE_PART_FAR) && c->n_near_tgt > 0;
  // projections of sigma land in the q slot of alpha (k_near_coef_K reads them there)
  const SelfArgs SA = self_args(c, nullptr, sigma, u, (parts & BIE_PART_SELF) ? 1 : 0,
                                near ? c->d_alpha : nullptr, 0);
  Ev ev;
  prof_begin(c, BIE_KIND_SELF, s, &ev);
  self_launch(c, SA, s);
  prof_end(c, s, &ev);
  rc = launch_check(c, "k_self");
  if (rc) return rc;
  if (parts & BIE_PART_FAR) {
    if (near) {
      const TableLayout L(c->p);
      const int64_t n = c->ns * L.nlm;
      prof_begin(c, BIE_KIND_NEAR, s, &ev);
      k_near_coef_K<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(c->p, c->ns, c->d_alpha, c->d_ncoef);
      prof_end(c, s, &ev);
      rc = launch_check(c, "k_near_coef_K");
      if (rc) return rc;
    }
    // near pairs excluded from the smooth K sum (or subtracted by k_near)
    const bool nx = near && use_near_exclusion(c);
    rc = run_far(c, u, s, 1, nx);
    if (rc) return rc;
    if (near) {  // traction of the exact exterior expansion for near pairs
      rc = run_near(c, u, s, true, nx ? 2 : 0);
      if (rc) return rc;
    }
  }
  if (parts & BIE_PART_COMPLETION) {
    prof_begin(c, BIE_KIND_COMPLETE, s, &ev);
    k_completion<<<(unsigned)c->ns, kCompleteThreads, 0, s>>>(c->nsn, c->d_centres, c->d_x, c->d_w,
                                                              sigma, u);
    prof_end(c, s, &ev);
    rc = launch_check(c, "k_completion");
  }
  return rc;
}

int bie_apply_SLDL(bie_ctx* c, const double* f, const double* q, double* u, bie_stream_t s) {
  if (!c) return BIE_ERR_ARG;
  if (!f || !q) return fail(c, BIE_ERR_ARG, "bie_apply_SLDL: f and q must be non-NULL%s");
  return bie_apply_parts(c, f, q, u, BIE_PART_FAR | BIE_PART_SELF, s);
}

int bie_apply_SL(bie_ctx* c, const double* f, double* u, bie_stream_t s) {
  if (!c) return BIE_ERR_ARG;
  if (!f) return fail(c, BIE_ERR_ARG, "bie_apply_SL: f is NULL%s");
  return bie_apply_parts(c, f, nullptr, u, BIE_PART_FAR | BIE_PART_SELF, s);
}

int bie_apply_DL(bie_ctx* c, const double* q, double* u, bie_stream_t s) {
  if (!c) return BIE_ERR_ARG;
  if (!q) return fail(c, BIE_ERR_ARG, "bie_apply_DL: q is NULL%s");
  return bie_apply_parts(c, nullptr, q, u, BIE_PART_FAR | BIE_PART_SELF, s);
}

int bie_eval_offsurface(bie_ctx* c, const double* f, const double* q, const double* tg, int64_t m,
                        double* u, double* p, bie_stream_t s) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (m < 0) return fail(c, BIE_ERR_ARG, "m < 0%s");
  if (m == 0) return BIE_OK;
  if (!tg || !u) return fail(c, BIE_ERR_ARG, "targets and u must be non-NULL%s");
  if (!is_device_ptr(c, tg) || !is_device_ptr(c, u) || (p && !is_device_ptr(c, p)) ||
      (f && !is_device_ptr(c, f)) || (q && !is_device_ptr(c, q)))
    return fail(c, BIE_ERR_ARG, "a buffer is not a device pointer%s");
  const int64_t n3 = 3 * c->N;
  if (overlaps(u, 3 * m, f, n3) || overlaps(u, 3 * m, q, n3) || overlaps(u, 3 * m, tg, 3 * m) ||
      overlaps(p, m, f, n3) || overlaps(p, m, q, n3) || overlaps(p, m, tg, 3 * m) ||
      overlaps(p, m, u, 3 * m))
    return fail(c, BIE_ERR_ARG, "an output overlaps an input or the other output%s");
  return run_offsurface(c, f, q, tg, m, u, p, (cudaStream_t)s);
}

int bie_eval_traction(bie_ctx* c, const double* sigma, const double* tg, const double* tn,
                      int64_t m, double* t, bie_stream_t s) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (m < 0) return fail(c, BIE_ERR_ARG, "m < 0%s");
  if (m == 0) return BIE_OK;
  if (!sigma || !tg || !tn || !t)
    return fail(c, BIE_ERR_ARG, "sigma, targets, normals and t must be non-NULL%s");
  if (!is_device_ptr(c, sigma) || !is_device_ptr(c, tg) || !is_device_ptr(c, tn) || !is_device_ptr(c, t))
    return fail(c, BIE_ERR_ARG, "a buffer is not a device pointer%s");
  if (overlaps(t, 3 * m, sigma, 3 * c->N) || overlaps(t, 3 * m, tg, 3 * m) ||
      overlaps(t, 3 * m, tn, 3 * m))
    return fail(c, BIE_ERR_ARG, "output t overlaps an input%s");
  return run_traction(c, sigma, tg, tn, m, t, (cudaStream_t)s);
}

static int stage(bie_ctx* c, double** d, size_t n) {
  if (*d) return BIE_OK;
  if (cudaMalloc(d, n * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, BIE_ERR_ALLOC, "cannot allocate staging buffers%s");
  }
  return BIE_OK;
}

int bie_apply_SLDL_host(bie_ctx* c, const double* f_h, const double* q_h, double* u_h,
                        bie_stream_t s) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (!f_h || !q_h || !u_h) return fail(c, BIE_ERR_ARG, "host buffers must be non-NULL%s");
  const size_t n3 = 3 * c->N;
  if ((rc = stage(c, &c->d_f, n3)) || (rc = stage(c, &c->d_q, n3)) || (rc = stage(c, &c->d_u, n3)))
    return rc;
  cudaStream_t st = (cudaStream_t)s;
  Ev ev;
  prof_begin(c, BIE_KIND_COPY, st, &ev);
  cudaError_t ce = cudaMemcpyAsync(c->d_f, f_h, n3 * sizeof(double), cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(c->d_q, q_h, n3 * sizeof(double), cudaMemcpyHostToDevice, st);
  prof_end(c, st, &ev);
  if (ce != cudaSuccess) return cuda_fail(c, ce, "bie_apply_SLDL_host: H2D");
  rc = run_apply(c, c->d_f, c->d_q, c->d_u, BIE_PART_FAR | BIE_PART_SELF, st);
  if (rc) return rc;
  prof_begin(c, BIE_KIND_COPY, st, &ev);
  ce = cudaMemcpyAsync(u_h, c->d_u, n3 * sizeof(double), cudaMemcpyDeviceToHost, st);
  prof_end(c, st, &ev);
  if (ce != cudaSuccess) return cuda_fail(c, ce, "bie_apply_SLDL_host: D2H");
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(c, e, "bie_apply_SLDL_host");
  return BIE_OK;
}

int bie_eval_offsurface_host(bie_ctx* c, const double* f_h, const double* q_h, const double* tg_h,
                             int64_t m, double* u_h, double* p_h, bie_stream_t s) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (m < 0) return fail(c, BIE_ERR_ARG, "m < 0%s");
  if (m == 0) return BIE_OK;
  if (!tg_h || !u_h) return fail(c, BIE_ERR_ARG, "targets and u must be non-NULL%s");
  const size_t n3 = 3 * c->N;
  if ((f_h && (rc = stage(c, &c->d_f, n3))) || (q_h && (rc = stage(c, &c->d_q, n3)))) return rc;
  if (m > c->tg_cap) {
    cudaFree(c->d_tg);
    cudaFree(c->d_uo);
    cudaFree(c->d_po);
    c->d_tg = c->d_uo = c->d_po = nullptr;
    c->tg_cap = 0;
    if ((rc = stage(c, &c->d_tg, 3 * m)) || (rc = stage(c, &c->d_uo, 3 * m)) ||
        (rc = stage(c, &c->d_po, m)))
      return rc;
    c->tg_cap = m;
  }
  cudaStream_t st = (cudaStream_t)s;
  Ev ev;
  prof_begin(c, BIE_KIND_COPY, st, &ev);
  cudaError_t ce = cudaSuccess;
  if (f_h) ce = cudaMemcpyAsync(c->d_f, f_h, n3 * sizeof(double), cudaMemcpyHostToDevice, st);
  if (q_h && ce == cudaSuccess)
    ce = cudaMemcpyAsync(c->d_q, q_h, n3 * sizeof(double), cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(c->d_tg, tg_h, 3 * m * sizeof(double), cudaMemcpyHostToDevice, st);
  prof_end(c, st, &ev);
  if (ce != cudaSuccess) return cuda_fail(c, ce, "bie_eval_offsurface_host: H2D");
  rc = run_offsurface(c, f_h ? c->d_f : nullptr, q_h ? c->d_q : nullptr, c->d_tg, m, c->d_uo,
                      p_h ? c->d_po : nullptr, st);
  if (rc) return rc;
  prof_begin(c, BIE_KIND_COPY, st, &ev);
  ce = cudaMemcpyAsync(u_h, c->d_uo, 3 * m * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (p_h && ce == cudaSuccess)
    ce = cudaMemcpyAsync(p_h, c->d_po, m * sizeof(double), cudaMemcpyDeviceToHost, st);
  prof_end(c, st, &ev);
  if (ce != cudaSuccess) return cuda_fail(c, ce, "bie_eval_offsurface_host: D2H");
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(c, e, "bie_eval_offsurface_host");
  return BIE_OK;
}

int bie_set_profiling(bie_ctx* c, int enable) {
  if (!c) return BIE_ERR_ARG;
  c->prof = enable != 0;
  return BIE_OK;
}

int bie_get_profile(bie_ctx* c, double* ms, int64_t* launches) {
  if (!c) return BIE_ERR_ARG;
  prof_drain(c);
  for (int k = 0; k < BIE_NUM_KINDS; ++k) {
    if (ms) ms[k] = c->ms[k];
    if (launches) launches[k] = c->launches[k];
  }
  return BIE_OK;
}

int bie_reset_profile(bie_ctx* c) {
  if (!c) return BIE_ERR_ARG;
  prof_drain(c);
  for (int k = 0; k < BIE_NUM_KINDS; ++k) {
    c->ms[k] = 0;
    c->launches[k] = 0;
  }
  return BIE_OK;
}

static void near_free(bie_ctx* c) {
  cudaFree(c->d_cell_start);
  cudaFree(c->d_cell_items);
  c->d_cell_start = c->d_cell_items = nullptr;
  cudaFree(c->d_nb_off);
  cudaFree(c->d_nb_idx);
  cudaFree(c->d_near_tgt);
  cudaFree(c->d_alpha);
  cudaFree(c->d_ncoef);
  c->d_nb_off = c->d_nb_idx = c->d_near_tgt = nullptr;
  c->d_alpha = c->d_ncoef = nullptr;
  c->n_near_tgt = 0;
  c->n_near_pairs = 0;
}

int bie_set_near(bie_ctx* c, double eta) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (!(eta >= 0.0) || !std::isfinite(eta)) return fail(c, BIE_ERR_ARG, "eta must be finite and >= 0%s");
  cudaDeviceSynchronize();
  near_free(c);
  c->eta = eta;
  if (eta == 0.0) return BIE_OK;
  const int64_t ns = c->ns;
  // Host-side copies of the geometry (bie_create keeps only device copies).
  std::vector<double> hc(3 * ns), ha(ns);
  if (cudaMemcpy(hc.data(), c->d_centres, 3 * ns * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(ha.data(), c->d_radii, ns * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaError_t e = cudaGetLastError();
    return cuda_fail(c, e, "bie_set_near: geometry");
  }
  std::vector<int64_t> off;
  std::vector<int> idx, tgt;
  near_lists_host(hc.data(), ha.data(), ns, eta, off, idx);
  // off-surface search grid: a target x is near sphere s only if
  // |x - c_s| < a_s (1 + 2 eta) <= a_max (1 + 2 eta) = cell size (padded)
  {
    double amax = 0, lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int64_t i = 0; i < ns; ++i) {
      amax = std::max(amax, ha[i]);
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], hc[3 * i + d]);
        hi[d] = std::max(hi[d], hc[3 * i + d]);
      }
    }
    double h = amax * (1.0 + 2.0 * eta) * (1.0 + 1e-9);
    auto dims = [&](double hh, int* n) {
      int64_t tot = 1;
      for (int d = 0; d < 3; ++d) {
        n[d] = (int)std::min<double>(1 << 20, std::floor((hi[d] - lo[d]) / hh) + 1.0);
        tot *= n[d];
      }
      return tot;
    };
    while (dims(h, c->gn) > 8 * ns + 4096) h *= 1.25;  // bounded grid for sparse geometries
    c->gh = h;
    for (int d = 0; d < 3; ++d) c->g0[d] = lo[d];
    const int64_t ncell = (int64_t)c->gn[0] * c->gn[1] * c->gn[2];
    std::vector<int> start(ncell + 1, 0), items(ns), cellof(ns);
    for (int64_t i = 0; i < ns; ++i) {
      int q[3];
      for (int d = 0; d < 3; ++d)
        q[d] = std::min(c->gn[d] - 1, std::max(0, (int)std::floor((hc[3 * i + d] - lo[d]) / h)));
      cellof[i] = (q[2] * c->gn[1] + q[1]) * c->gn[0] + q[0];
      start[cellof[i] + 1]++;
    }
    for (int64_t k = 0; k < ncell; ++k) start[k + 1] += start[k];
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int64_t i = 0; i < ns; ++i) items[fill[cellof[i]]++] = (int)i;  // ascending per cell
    if (cudaMalloc(&c->d_cell_start, (ncell + 1) * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&c->d_cell_items, ns * sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      near_free(c);
      return fail(c, BIE_ERR_ALLOC, "near search grid%s");
    }
    if (cudaMemcpy(c->d_cell_start, start.data(), (ncell + 1) * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_cell_items, items.data(), ns * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaError_t e = cudaGetLastError();
      near_free(c);
      return cuda_fail(c, e, "bie_set_near: grid");
    }
  }
  if (off[ns] > (int64_t)INT32_MAX)
    return fail(c, BIE_ERR_UNSUPPORTED, "bie_set_near: more than 2^31-1 near pairs%s");
  std::vector<int> off32(ns + 1);
  for (int64_t t = 0; t <= ns; ++t) off32[t] = (int)off[t];
  for (int64_t t = 0; t < ns; ++t)
    if (off[t + 1] > off[t]) tgt.push_back((int)t);
  c->n_near_pairs = off[ns];
  c->n_near_tgt = (int)tgt.size();
  const TableLayout L(c->p);
  if (cudaMalloc(&c->d_alpha, (size_t)ns * 12 * L.nlm * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->d_ncoef, (size_t)ns * 10 * L.nlm * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    near_free(c);
    return fail(c, BIE_ERR_ALLOC, "near coefficients%s");
  }
  if (c->n_near_pairs == 0) return BIE_OK;
  if (cudaMalloc(&c->d_nb_off, (ns + 1) * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->d_nb_idx, idx.size() * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->d_near_tgt, tgt.size() * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    near_free(c);
    return fail(c, BIE_ERR_ALLOC, "near lists%s");
  }
  if (cudaMemcpy(c->d_nb_off, off32.data(), (ns + 1) * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c->d_nb_idx, idx.data(), idx.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c->d_near_tgt, tgt.data(), tgt.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaError_t e = cudaGetLastError();
    near_free(c);
    return cuda_fail(c, e, "bie_set_near: lists");
  }
  return BIE_OK;
}

int64_t bie_near_pairs(const bie_ctx* c) { return c ? c->n_near_pairs : -1; }

int bie_near_lists(const double* centres_h, const double* radii_h, int64_t n_spheres, double eta,
                   int64_t* off_h, int* idx_h, int64_t cap, int64_t* total) {
  if (!centres_h || !radii_h || n_spheres < 1 || !off_h || !total || !(eta >= 0.0) || !std::isfinite(eta))
    return BIE_ERR_ARG;
  std::vector<int64_t> off;
  std::vector<int> idx;
  near_lists_host(centres_h, radii_h, n_spheres, eta, off, idx);
  *total = off[n_spheres];
  for (int64_t t = 0; t <= n_spheres; ++t) off_h[t] = off[t];
  if (idx_h) {
    if (cap < off[n_spheres]) return BIE_ERR_ARG;
    for (size_t k = 0; k < idx.size(); ++k) idx_h[k] = idx[k];
  }
  return BIE_OK;
}

int bie_set_near_exclusion(bie_ctx* c, int mode) {
  if (!c) return BIE_ERR_ARG;
  if (mode < -1 || mode > 1) return fail(c, BIE_ERR_ARG, "near exclusion must be -1, 0 or 1%s");
  c->near_excl = mode;
  return BIE_OK;
}

int bie_set_near_off_schedule(bie_ctx* c, int schedule) {
  if (!c) return BIE_ERR_ARG;
  if (schedule < 0 || schedule > 1) return fail(c, BIE_ERR_ARG, "near off-surface schedule must be 0 or 1%s");
  c->noff_sched = schedule;
  return BIE_OK;
}

int bie_set_near_mode(bie_ctx* c, int mode) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (mode < 0 || mode > 3) return fail(c, BIE_ERR_ARG, "near mode must be 0, 1, 2 or 3%s");
  if ((mode == 1 || mode == 3) && !c->d_delta) {
    // Delta_n by quadrature on this context's grid (exact for n <= p), once
    const TableLayout L(c->p);
    double *rot = nullptr, *rphi = nullptr;
    if (cudaMalloc(&c->d_delta, n4_delta_doubles(c->p) * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c->d_deltaT, n4_delta_doubles(c->p) * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c->d_psinear, (size_t)c->ns * L.nlm * 6 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&rot, (size_t)c->nsn * L.nlm * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&rphi, (size_t)c->nsn * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(rot);
      cudaFree(rphi);
      cudaFree(c->d_delta);
      cudaFree(c->d_deltaT);
      cudaFree(c->d_psinear);
      c->d_delta = c->d_deltaT = c->d_psinear = nullptr;
      return fail(c, BIE_ERR_ALLOC, "NEXT-4 tables%s");
    }
    Ev ev;
    prof_begin(c, BIE_KIND_SETUP, 0, &ev);
    k_n4_rotpts<<<(c->nsn + 127) / 128, 128>>>(c->p, c->d_tab, rot, rphi);
    k_n4_delta<<<c->p + 1, 256>>>(c->p, c->d_tab, rot, rphi, c->d_delta, c->d_deltaT);
    c->launches[BIE_KIND_SETUP] += 1;
    prof_end(c, 0, &ev);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaFree(rot);
    cudaFree(rphi);
    if (e != cudaSuccess) return cuda_fail(c, e, "bie_set_near_mode");
    const size_t sm = n4_smem_doubles(c->p) * sizeof(double);
    if (sm > 48 * 1024 &&
        cudaFuncSetAttribute((const void*)k_n4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
            cudaSuccess)
      return cuda_fail(c, cudaGetLastError(), "k_n4 shared memory");
  }
  c->near_mode = mode;
  return BIE_OK;
}

// ----------------------------------------------------------- NEXT-2 (GMRES)
namespace {
struct Krylov {
  bie_ctx* c;
  cudaStream_t s;
  int64_t n;
  double* part = nullptr;  // [kDotBlocks + 1]
  // First CUDA error seen by any Krylov step (launch, copy or synchronisation).
  // A failed step leaves its host-side result undefined, so every caller checks
  // `ok()` before using one (no false "converged" after a fault).
  cudaError_t err = cudaSuccess;
  void note(cudaError_t e) {
    if (e != cudaSuccess && err == cudaSuccess) err = e;
  }
  void note_launch() { note(cudaGetLastError()); }
  bool ok() const { return err == cudaSuccess; }
  double dot(const double* x, const double* y) {
    Ev ev;
    prof_begin(c, BIE_KIND_KRYLOV, s, &ev);
    k_dot_partial<<<kDotBlocks, kDotThreads, 0, s>>>(n, x, y, part);
    k_dot_final<<<1, kDotThreads, 0, s>>>(part, part + kDotBlocks);
    prof_end(c, s, &ev);
    note_launch();
    double h = 0.0;
    note(cudaMemcpyAsync(&h, part + kDotBlocks, sizeof(double), cudaMemcpyDeviceToHost, s));
    note(cudaStreamSynchronize(s));
    return ok() ? h : std::nan("");
  }
  // classical Gram-Schmidt twice against V[0..nv): on return hv[0..nv) holds
  // the projections (device), w is orthogonalised, and wnorm2 = w.w; one sync.
  void cgs2(const double* V, int nv, double* w, double* dh, double* hv, double* wnorm2) {
    Ev ev;
    prof_begin(c, BIE_KIND_KRYLOV, s, &ev);
    for (int pass = 0; pass < 2; ++pass) {
      k_mdot_partial<<<kDotBlocks, kDotThreads, 0, s>>>(n, nv, V, w, mpart);
      k_mdot_final<<<nv, kDotThreads, 0, s>>>(mpart, dh + pass * 512, 0);
      k_maxpy<<<kDotBlocks, kDotThreads, 0, s>>>(n, nv, dh + pass * 512, V, w);
    }
    k_dot_partial<<<kDotBlocks, kDotThreads, 0, s>>>(n, w, w, part);
    k_dot_final<<<1, kDotThreads, 0, s>>>(part, dh + 1024);
    prof_end(c, s, &ev);
    note_launch();
    std::vector<double> hh(1025, std::nan(""));
    note(cudaMemcpyAsync(hh.data(), dh, 1025 * sizeof(double), cudaMemcpyDeviceToHost, s));
    note(cudaStreamSynchronize(s));
    for (int i = 0; i < nv; ++i) hv[i] = hh[i] + hh[512 + i];
    *wnorm2 = hh[1024];
  }
  double* mpart = nullptr;  // [512][kDotBlocks]
  void axpby(double a, const double* x, double b, double* y) {
    Ev ev;
    prof_begin(c, BIE_KIND_KRYLOV, s, &ev);
    k_axpby<<<kDotBlocks, kDotThreads, 0, s>>>(n, a, x, b, y);
    prof_end(c, s, &ev);
    note_launch();
  }
  void copy(double* dst, const double* src) {
    note(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  void zero(double* dst) { note(cudaMemsetAsync(dst, 0, n * sizeof(double), s)); }
  // y = P^{-1} x, P = 1/2 I + S_self + D_self (block diagonal, exact via the spectra)
  int prec(const double* x, double* y) {
    const SelfArgs SA = self_args(c, nullptr, x, y, 1, nullptr, 1);
    Ev ev;
    prof_begin(c, BIE_KIND_KRYLOV, s, &ev);
    self_launch(c, SA, s);
    prof_end(c, s, &ev);
    return launch_check(c, "k_self(precond)");
  }
  // y = (1/2 I + S + D_pv (+ near correction)) x     (BIE 5.4)
  int op(const double* x, double* y) {
    int rc = run_apply(c, x, x, y, BIE_PART_FAR | BIE_PART_SELF, s);
    if (rc) return rc;
    axpby(0.5, x, 1.0, y);
    return ok() ? BIE_OK : cuda_fail(c, err, "bie_solve_porous: k_axpby");
  }
};
}  // namespace

int bie_solve_porous(bie_ctx* c, const double* uinf, double* mu_out, double tol, int max_iter,
                     int restart, int precond, int* iters_out, double* resid_out,
                     bie_stream_t st) {
  if (!c) return BIE_ERR_ARG;
  int rc = check_device(c);
  if (rc) return rc;
  if (!uinf || !mu_out || !is_device_ptr(c, uinf) || !is_device_ptr(c, mu_out))
    return fail(c, BIE_ERR_ARG, "uinf and mu must be device pointers%s");
  const int64_t n = 3 * c->N;
  if (overlaps(uinf, n, mu_out, n)) return fail(c, BIE_ERR_ARG, "mu overlaps uinf%s");
  if (!(tol > 0.0) || max_iter < 1 || restart < 1 || restart > 500)
    return fail(c, BIE_ERR_ARG, "need tol > 0, max_iter >= 1, 1 <= restart <= 500%s");
  // (restart + 1 <= 512 Krylov vectors: fits the batched Gram-Schmidt buffers)
  Krylov K{c, (cudaStream_t)st, n};
  const int m = restart;
  double *V = nullptr, *w = nullptr, *b = nullptr, *z = nullptr, *dh = nullptr;
  if (cudaMalloc(&V, (size_t)(m + 1) * n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&w, n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&b, n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&z, n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&dh, 1025 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&K.mpart, (size_t)512 * kDotBlocks * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&K.part, (kDotBlocks + 1) * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(V); cudaFree(w); cudaFree(b); cudaFree(z); cudaFree(dh); cudaFree(K.mpart);
    cudaFree(K.part);
    return fail(c, BIE_ERR_ALLOC, "GMRES workspace%s");
  }
  auto cleanup = [&]() {
    cudaFree(V); cudaFree(w); cudaFree(b); cudaFree(z); cudaFree(dh); cudaFree(K.mpart);
    cudaFree(K.part);
  };
  // b = -u_inf, x0 = 0
  K.zero(mu_out);
  K.zero(b);
  K.axpby(-1.0, uinf, 0.0, b);
  const double bnorm = std::sqrt(K.dot(b, b));
  int it = 0;
  double rel = 0.0;
  if (!K.ok()) {
    cleanup();
    return cuda_fail(c, K.err, "bie_solve_porous: setup");
  }
  if (bnorm == 0.0) {
    cleanup();
    if (iters_out) *iters_out = 0;
    if (resid_out) *resid_out = 0.0;
    return BIE_OK;
  }
  std::vector<double> H((size_t)(m + 1) * m), g(m + 1), cs(m), sn(m), y(m);
  bool done = false;
  while (!done) {
    // r = b - A x  -> V[0]
    double* v0 = V;
    if ((rc = K.op(mu_out, w))) { cleanup(); return rc; }
    K.copy(v0, b);
    K.axpby(-1.0, w, 1.0, v0);
    const double beta = std::sqrt(K.dot(v0, v0));
    if (!K.ok()) { cleanup(); return cuda_fail(c, K.err, "bie_solve_porous: residual"); }
    rel = beta / bnorm;
    if (rel <= tol || it >= max_iter) break;
    K.axpby(0.0, v0, 1.0 / beta, v0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    for (; j < m && it < max_iter; ++j, ++it) {
      double* vj = V + (size_t)j * n;
      double* vn = V + (size_t)(j + 1) * n;
      if (precond) {  // right preconditioning: A P^{-1} v_j
        if ((rc = K.prec(vj, z)) || (rc = K.op(z, vn))) { cleanup(); return rc; }
      } else if ((rc = K.op(vj, vn))) {
        cleanup();
        return rc;
      }
      // classical Gram-Schmidt applied twice (CGS2): batched, one host sync
      std::vector<double> hcol(j + 1);
      double wn2 = 0.0;
      K.cgs2(V, j + 1, vn, dh, hcol.data(), &wn2);
      if (!K.ok()) { cleanup(); return cuda_fail(c, K.err, "bie_solve_porous: Arnoldi"); }
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = hcol[i];
      const double hn = std::sqrt(wn2);
      H[(size_t)(j + 1) * m + j] = hn;
      if (hn > 0.0) K.axpby(0.0, vn, 1.0 / hn, vn);
      for (int i = 0; i < j; ++i) {  // apply previous Givens rotations
        const double a1 = H[(size_t)i * m + j], a2 = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a1 + sn[i] * a2;
        H[(size_t)(i + 1) * m + j] = -sn[i] * a1 + cs[i] * a2;
      }
      const double a1 = H[(size_t)j * m + j], a2 = H[(size_t)(j + 1) * m + j];
      const double den = std::hypot(a1, a2);
      cs[j] = den > 0.0 ? a1 / den : 1.0;
      sn[j] = den > 0.0 ? a2 / den : 0.0;
      H[(size_t)j * m + j] = den;
      H[(size_t)(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rel = std::fabs(g[j + 1]) / bnorm;
      if (rel <= tol || hn == 0.0) {
        ++j;
        ++it;
        done = true;
        break;
      }
    }
    // x += V y,  H[0:j,0:j] y = g[0:j]
    for (int i = j - 1; i >= 0; --i) {
      double sacc = g[i];
      for (int k = i + 1; k < j; ++k) sacc -= H[(size_t)i * m + k] * y[k];
      y[i] = sacc / H[(size_t)i * m + i];
    }
    if (precond) {  // mu += P^{-1} (V y)
      K.zero(w);
      for (int i = 0; i < j; ++i) K.axpby(y[i], V + (size_t)i * n, 1.0, w);
      if ((rc = K.prec(w, z))) { cleanup(); return rc; }
      K.axpby(1.0, z, 1.0, mu_out);
    } else {
      for (int i = 0; i < j; ++i) K.axpby(y[i], V + (size_t)i * n, 1.0, mu_out);
    }
    if (it >= max_iter) done = true;
  }
  // true relative residual of the returned iterate
  if ((rc = K.op(mu_out, w))) { cleanup(); return rc; }
  K.axpby(1.0, b, -1.0, w);
  rel = std::sqrt(K.dot(w, w)) / bnorm;
  cleanup();
  if (!K.ok()) return cuda_fail(c, K.err, "bie_solve_porous");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(c, e, "bie_solve_porous");
  if (iters_out) *iters_out = it;
  if (resid_out) *resid_out = rel;
  return BIE_OK;
}

int bie_set_far_reduction(bie_ctx* c, int mode) {
  if (!c) return BIE_ERR_ARG;
  if (mode < 0 || mode > 7) return fail(c, BIE_ERR_ARG, "far reduction mode must be 0..7%s");
  c->far_red = mode;
  return BIE_OK;
}

int bie_set_self_kernel(bie_ctx* c, int variant) {
  if (!c) return BIE_ERR_ARG;
  if (variant < -1 || variant > 3) return fail(c, BIE_ERR_ARG, "self kernel variant must be -1..3%s");
  if (variant == 3 && self2_smem_bytes(c->p) > 227 * 1024)
    return fail(c, BIE_ERR_UNSUPPORTED, "two spheres per CTA exceed shared memory at this order%s");
  c->self_variant = variant;
  return BIE_OK;
}

int bie_set_source_chunks(bie_ctx* c, int chunks) {
  if (!c) return BIE_ERR_ARG;
  if (chunks < 0 || chunks > 4096) return fail(c, BIE_ERR_ARG, "chunks must be in [0, 4096]%s");
  c->chunks_override = chunks;
  return BIE_OK;
}

}  // extern "C"
