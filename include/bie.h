/*
 * bie.h -- C ABI of libbie.so, the B200 (sm_100a) fp64 implementation of the
 * discretised Stokes boundary-integral-operator apply of Corona & Veerapaneni,
 * "Boundary integral equation analysis for suspension of spheres in Stokes
 * flow", arXiv 1707.06551.  P:n = PAPER.md line n; R<k> = reading k
 * in DESIGN.md §3 (where the paper is garbled or silent).
 *
 * Conventions (all entry points)
 *   - fp64 everywhere.  Vectors are [count][3] row-major, xyz interleaved.
 *   - Node order (eq 4.2; R11): node i = s*(p+1)*(2p+2) + j*(2p+2) + k
 *     for sphere s, polar index j (t_j = cos(theta_j) ascending Gauss-Legendre
 *     nodes) and azimuthal index k (phi_k = 2 pi k/(2p+2)).
 *   - Pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors on the
 *     device current at bie_create) unless the name ends in _h (host).
 *   - Streams: bie_stream_t is a cudaStream_t (NULL = legacy default stream).
 *     Device-pointer calls are stream-ordered and return after enqueue; the
 *     caller's buffers must stay valid until the stream reaches the work.
 *     Asynchronous faults surface at the next synchronisation.  A context
 *     holds scratch, so it must not be used from two streams concurrently;
 *     distinct contexts are independent.
 *   - Outputs are OVERWRITTEN, never accumulated.  An output that overlaps an
 *     input returns BIE_ERR_ARG.
 *   - Validation happens on the host at entry; kernels never check.  No C++
 *     exception crosses the ABI.  On error the context's message
 *     (bie_last_error) says which argument was wrong.
 *   - Viscosity: PAPER sets nu = 1; here mu > 0 is a parameter (R5):
 *     S velocity scales 1/mu, D velocity is mu-free, S pressure is mu-free,
 *     D pressure scales mu.
 */
#ifndef BIE_H
#define BIE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bie_ctx bie_ctx;
typedef void* bie_stream_t; /* cudaStream_t */

enum bie_status {
  BIE_OK = 0,
  BIE_ERR_ARG = 1,         /* bad pointer, size, value or aliasing          */
  BIE_ERR_GEOMETRY = 2,    /* overlapping/touching spheres (|c_i-c_j| <= a_i + a_j) */
  BIE_ERR_ALLOC = 3,       /* device allocation failed                      */
  BIE_ERR_CUDA = 4,        /* CUDA launch/runtime error                     */
  BIE_ERR_UNSUPPORTED = 5  /* p outside [1, BIE_P_MAX] or no sm_100a device  */
};

#define BIE_P_MAX 32 /* 1 <= p <= 32 */

/* Parts selector for bie_apply_parts (testing / measurement). */
#define BIE_PART_FAR 1  /* smooth Nystrom sum over all other spheres (a3)  */
#define BIE_PART_SELF 2 /* spectral self term (a4-a6)                     */
#define BIE_PART_COMPLETION 4 /* completion L of eq 5.8 (bie_apply_K only)  */

/* Kernel kinds reported by bie_get_profile. */
#define BIE_KIND_SETUP 0    /* GL rule, Legendre/eigen tables, node generation (a1) */
#define BIE_KIND_SELF 1     /* fused pack + forward VSHT + scale + inverse VSHT (a2, a4-a6) */
#define BIE_KIND_PACK 2     /* source packing for off-surface evaluation (a2)   */
#define BIE_KIND_NBODY 3    /* far-field SL+DL pair sum, self-sphere masked (a3) */
#define BIE_KIND_REDUCE 4   /* deterministic reduction of source-chunk partials */
#define BIE_KIND_OFFSURF 5  /* off-surface u,p pair sum (a7)                    */
#define BIE_KIND_COPY 6     /* host<->device copies of the _host entry points   */
#define BIE_KIND_NEAR 7     /* near-singular correction (NEXT-1)              */
#define BIE_KIND_KRYLOV 8   /* GMRES vector kernels (NEXT-2)                  */
#define BIE_KIND_KFAR 9     /* far-field traction operator K pair sum (NEXT-3) */
#define BIE_KIND_COMPLETE 10 /* completion operator L of eq 5.8 (NEXT-3)          */
#define BIE_KIND_NEAR4 11   /* rotated near evaluation of PAPER §4.2 (NEXT-4)    */
#define BIE_NUM_KINDS 12

/*
 * bie_create -- build nodes, weights, normals and spectral tables (row a1).
 *   centres_h [n_spheres][3], radii_h [n_spheres] : host, copied.
 *   p  : quadrature/expansion order, grid (p+1) x (2p+2) per sphere (eq 4.2,
 *        P:311), 1 <= p <= BIE_P_MAX.
 *   mu : viscosity, finite and > 0.
 *   Weights w = a^2 lambda_j 2 pi/(2p+2) (eq 4.4, reading R4);
 *   outward normals.  Synchronous.  Returns BIE_ERR_ARG on NULL or
 *   non-finite input, n_spheres < 1 or radii <= 0; BIE_ERR_GEOMETRY if two
 *   spheres overlap or touch (|c_i - c_j| <= a_i + a_j; SPEC's "pairwise
 *   center distance > sum of radii", R19 -- touching spheres can place a node
 *   of each at the contact point, r = 0); BIE_ERR_UNSUPPORTED
 *   for p out of range.  *out is NULL on failure.
 */
int bie_create(const double* centres_h, const double* radii_h, int64_t n_spheres, int p,
               double mu, bie_ctx** out);

/* bie_destroy -- frees everything the context owns.  NULL-safe. Synchronous. */
void bie_destroy(bie_ctx* ctx);

/* Number of nodes N = n_spheres (p+1)(2p+2); -1 for NULL. */
int64_t bie_num_nodes(const bie_ctx* ctx);
int bie_order(const bie_ctx* ctx);
int64_t bie_num_spheres(const bie_ctx* ctx);

/*
 * bie_get_nodes -- copy node positions x [N][3], outward normals [N][3] and
 * quadrature weights w [N] (device pointers; any may be NULL to skip) on s.
 */
int bie_get_nodes(const bie_ctx* ctx, double* x, double* normals, double* w, bie_stream_t s);

/*
 * bie_apply_SLDL -- u = S[f] + D_pv[q] at every node (rows a2-a6, the metric path).
 *   S[f] (eq 2.19, 2.21), D[q] with the stresslet of eq 2.20 taken
 *   with the sign fixed by the paper's spectra (reading R1): for node i of
 *   sphere s
 *     u_i = sum over nodes k of every OTHER sphere of
 *             w_k [ (1/(8 pi mu)) (f_k/r + (rho.f_k) rho/r^3)
 *                   + (3/(4 pi)) (rho.n_k)(rho.q_k) rho/r^5 ],  rho = x_i - x_k
 *           (smooth rule eq 4.4 for all non-self pairs, "far-interactions with
 *            the smooth quadrature" P:436; no near correction)
 *         + the self term of sphere s: forward vector spherical harmonic
 *           transform of (a_s/mu) f and q (discrete projection, R9), diagonal
 *           scale by the S and principal-value D eigenvalues (Thm 2, P:217,
 *           via eqs 3.6-3.11 at r -> 1, readings R2/R3), one inverse transform
 *           (P:342).
 *   No 1/2 I term is added (R14): D_pv is the principal value; the one-sided
 *   limits are D_pv +- q/2, formed by the caller.
 *   f, q, u : device [N][3].  u must not overlap f or q.
 */
int bie_apply_SLDL(bie_ctx* ctx, const double* f, const double* q, double* u, bie_stream_t s);

/* bie_apply_SL -- u = S[f] (as bie_apply_SLDL with q = 0). */
int bie_apply_SL(bie_ctx* ctx, const double* f, double* u, bie_stream_t s);

/* bie_apply_DL -- u = D_pv[q] (as bie_apply_SLDL with f = 0). */
int bie_apply_DL(bie_ctx* ctx, const double* q, double* u, bie_stream_t s);

/*
 * bie_apply_parts -- as bie_apply_SLDL restricted to `parts` (bitwise OR of
 * BIE_PART_FAR and BIE_PART_SELF; 0 is BIE_ERR_ARG).  f or q may be NULL
 * (zero density).  Used by the parity tests to check each row alone.
 */
int bie_apply_parts(bie_ctx* ctx, const double* f, const double* q, double* u, int parts,
                    bie_stream_t s);

/*
 * bie_apply_K -- u = K_pv[sigma] at every node: the traction
 * of the single layer (eq 2.22) with the target normal,
 *     K[s](x) = -(3/(4 pi)) int ((x-y).n(x)) ((x-y).s(y)) (x-y)/|x-y|^5 dS_y
 * (reading R21: the adjoint of the R1 double layer, as P:219 requires),
 * smooth rule over every other sphere + the principal-value self term, whose
 * spectrum is that of D_pv (K_+ = D_-, K_- = D_+).  The one-sided
 * tractions are K_pv -+ sigma/2 (exterior: minus).  `parts`: bitwise OR of
 * BIE_PART_FAR, BIE_PART_SELF and BIE_PART_COMPLETION (non-empty).  With
 * BIE_PART_COMPLETION the completion operator of the mobility BIE (eq 5.8,
 * P:490-491, "added ... to eliminate the 6n dimensional nullspace") is added:
 *     L[sigma](x) = int_{G_s} sigma dG + (int_{G_s} (y - c_s) x sigma dG) x (x - c_s)
 * for x on sphere s (reading R22: one rank-6 block per sphere, integrals by
 * the node rule), so (1/2) sigma + u is the operator of eq 5.8's left side.
 * With bie_set_near(eta > 0) and BIE_PART_FAR, sphere pairs failing eq 4.5
 * get the traction of the source sphere's exact degree-<=p single-layer
 * expansion instead of the smooth rule (eqs 3.17-3.18; reading
 * R24), evaluated at the target node with the target normal.
 * sigma, u: device [N][3]; u must not overlap sigma.
 */
int bie_apply_K(bie_ctx* ctx, const double* sigma, double* u, int parts, bie_stream_t s);

/*
 * bie_eval_offsurface -- velocity and pressure at m arbitrary targets (row a7).
 *   u(x) = the smooth sum of bie_apply_SLDL over ALL nodes (no exclusion);
 *   p(x) = sum_k w_k [ (1/(4 pi)) (rho.f_k)/r^3
 *                      + (mu/(2 pi)) ( -(q_k.n_k)/r^3 + 3 (rho.q_k)(rho.n_k)/r^5 ) ]
 *   (Stokeslet and stresslet pressures, reading R12; the paper's printed D
 *   pressures P:215 are not used).  f or q may be NULL (zero density), p may
 *   be NULL (not computed).  targets [m][3], u [m][3], p [m]: device.  Targets
 *   closer to a surface than the smooth rule resolves are the caller's
 *   contract (SPEC "garbage-in for non-separated targets"); a target that
 *   coincides with a node gives inf/NaN.  m = 0 is a no-op.
 */
int bie_eval_offsurface(bie_ctx* ctx, const double* f, const double* q, const double* targets,
                        int64_t m, double* u, double* p, bie_stream_t s);

/*
 * bie_eval_traction -- traction of the single-layer flow S[sigma] at m
 * arbitrary points with given normals (eq 2.22 off the
 * surface, whose one-sphere closed forms are eqs 3.19-3.21):
 *   t(x) = K[sigma](x; n) = (grad u + grad u^T - pI) n,  u = S[sigma],
 *        = -(3/(4 pi)) sum_k w_k ((x-y_k).n)((x-y_k).sigma_k)(x-y_k)/|x-y_k|^5
 * (smooth rule over ALL nodes; mu- and a-free).  With bie_set_near(eta > 0)
 * a target at point-to-surface distance 0 <= d < eta 2 a_s from sphere s
 * gets the traction of s's exact degree-<=p expansion instead of s's smooth
 * sum (eqs 3.17-3.18, reading R24; exterior targets only, as
 * bie_eval_offsurface).  sigma: device [N][3]; targets, normals, t: device
 * [m][3]; normals are used as given (unit length expected, not
 * renormalised).  m = 0 is a no-op; a target on a node gives inf/NaN.
 * Uses the context's packed-source scratch, like every apply.
 */
int bie_eval_traction(bie_ctx* ctx, const double* sigma, const double* targets,
                      const double* normals, int64_t m, double* t, bie_stream_t s);

/*
 * Host-buffer variants (end-to-end): identical results; the inputs are copied
 * host->device on s (pinned host memory makes the copies asynchronous), the
 * outputs device->host, and the call synchronises s before returning.
 */
int bie_apply_SLDL_host(bie_ctx* ctx, const double* f_h, const double* q_h, double* u_h,
                        bie_stream_t s);
int bie_eval_offsurface_host(bie_ctx* ctx, const double* f_h, const double* q_h,
                             const double* targets_h, int64_t m, double* u_h, double* p_h,
                             bie_stream_t s);

/*
 * Profiling: when enabled, every kernel the context launches is bracketed by
 * CUDA events recorded on the launching stream.  bie_get_profile synchronises
 * those events and returns, per kind (BIE_KIND_*), the cumulative device
 * milliseconds and launch counts since the last reset.  Arrays have
 * BIE_NUM_KINDS entries; either may be NULL.
 */
int bie_set_profiling(bie_ctx* ctx, int enable);
int bie_get_profile(bie_ctx* ctx, double* ms, int64_t* launches);
int bie_reset_profile(bie_ctx* ctx);

/*
 * bie_set_near -- near-singular correction (PAPER §4.1 "Singular and
 * near-singular integrands"; §4.3).  eta > 0 enables it:
 * every sphere pair that is not well separated by eq 4.5,
 *     |c_s - c_t| - a_s - a_t  <  eta * max(2 a_s, 2 a_t),
 * has its smooth-rule contribution in bie_apply_* replaced by the exact
 * exterior field of the source sphere's degree-<=p vector spherical harmonic
 * expansion (eqs 3.6-3.11 with reading R1, eq 4.7; the expansion is the
 * discrete projection of reading R9).  eta = 0 disables it (the default, and
 * the BASELINE.json metric path).  bie_eval_offsurface applies the same
 * correction to u and p at every EXTERIOR target x within eta * 2 a_s of the
 * surface of a sphere s (0 <= |x - c_s| - a_s < eta * 2 a_s, SPEC's
 * point-to-surface form of eq 4.5), using the exterior pressures of P:189 (S)
 * and reading R12 (D); targets inside a sphere keep the plain smooth sum.
 * The same partition drives the traction paths (NEXT-3): bie_apply_K and
 * bie_eval_traction use the exact traction of the source expansion (eqs
 * 3.17-3.18) for near pairs / near exterior targets.
 * In the applies (bie_apply_*, bie_apply_K) the far-field kernel may skip the
 * near pairs (as it skips a target's own sphere) so the correction only adds
 * the exact field, or keep them and subtract them (bie_set_near_exclusion).
 * Builds the neighbour lists (host cell list, O(n_spheres); int64 offsets,
 * BIE_ERR_UNSUPPORTED beyond 2^31 - 1 pairs) and the off-surface search grid,
 * and synchronises.  BIE_ERR_ARG for eta < 0 or non-finite.
 */
int bie_set_near(bie_ctx* ctx, double eta);

/*
 * Host utility (no GPU needed): the CSR neighbour lists bie_set_near builds --
 * for every target sphere t the source spheres s != t failing eq 4.5 (P:323-
 * 328) in the IEEE evaluation order |c_s - c_t| - a_s - a_t < eta max(2 a_s,
 * 2 a_t), ascending -- from a uniform cell list (cell = 2 a_max (1 + eta)).
 * off_h [n_spheres + 1] (int64) is always filled and *total set; idx_h (cap
 * entries, may be NULL) receives the lists.  BIE_ERR_ARG on bad arguments or
 * cap < *total (off_h and *total are still valid then).
 */
int bie_near_lists(const double* centres_h, const double* radii_h, int64_t n_spheres, double eta,
                   int64_t* off_h, int* idx_h, int64_t cap, int64_t* total);

/* Number of (target sphere, source sphere) near pairs of the current eta; -1 for NULL. */
int64_t bie_near_pairs(const bie_ctx* ctx);

/*
 * bie_solve_porous -- Problem 1 of PAPER §5 (porous media, eqs 5.3-5.4,
 * P:458-472): static spheres in an imposed flow u_inf; with the ansatz
 * u = u_inf + sum_k (S_k + D_k)[mu] (eq 5.3) and no slip, solve the
 * second-kind BIE (eq 5.4)
 *     (1/2 I + sum_k (S_k + D_k)) [mu] = -u_inf     at every node
 * by restarted GMRES(restart) with classical Gram-Schmidt applied twice
 * (batched, one host synchronisation per Arnoldi step; the paper names no
 * solver; SPEC picks GMRES).  The operator is bie_apply_SLDL with f = q = mu
 * (plus the near correction if bie_set_near is on) and the 1/2 I of the
 * exterior limit (reading R14).  Dot products are fixed-order reductions, so
 * the iterates are reproducible.
 *   uinf [N][3] (device): imposed flow at the nodes; mu [N][3] (device) out.
 *   Stops when the relative residual ||b - A mu|| / ||b|| <= tol or after
 *   max_iter operator applications; *iters gets the count, *rel_resid the TRUE
 *   relative residual of the returned mu (recomputed).  Not converging is
 *   not an error (check *rel_resid).  Synchronous; workspace of
 *   (restart + 4) x 3N doubles (Krylov basis V[restart + 1], w, b, z) plus
 *   512 x 592 + 1618 doubles of reduction partials is allocated per call and
 *   freed before return.  Any CUDA failure inside the solve (launch, copy,
 *   synchronisation) returns BIE_ERR_CUDA; *iters and *rel_resid are then
 *   left untouched.  1 <= restart <= 500;
 *   restarting costs iterations (cfg 3: restart 30/50/100 -> 114/94/80
 *   iterations; cfg 5: 50 -> 200, 300 -> 138), so a restart at least as
 *   long as the expected iteration count is the better use of HBM
 *   (cfg 5 at restart 300: 304 x 3N doubles = 7.2 GB).
 *   The force on sphere s is -sum_{k in s} w_k mu_k (Stokes drag; pinned in
 *   tests/test_oracle_porous.py).
 *   precond = 1: right preconditioning by the exact inverse of each sphere's
 *   own operator P = 1/2 I + S_self + D_self, which the spectra of Thm 2 make
 *   diagonal in the VSH basis (eigenvalue 1/(1/2 + lamS a/mu + lamD_pv) on
 *   every mode of degree <= p, 2 on the remainder); applied by the self-term
 *   kernel.  precond = 0: plain GMRES.
 */
int bie_solve_porous(bie_ctx* ctx, const double* uinf, double* mu, double tol, int max_iter,
                     int restart, int precond, int* iters, double* rel_resid, bie_stream_t s);

/*
 * bie_set_near_mode -- how the near-singular correction of bie_set_near
 * evaluates the exact exterior field of a near source sphere s at the nodes of
 * a target sphere t (velocity applies: bie_apply_SL/DL/SLDL/parts):
 *   0 (default) direct (NEXT-1): the exterior expansion of eqs 3.6-3.11
 *     evaluated at every node of t, O(p^4) per pair.
 *   1 rotated (NEXT-4, PAPER §4.2 "General case", Fig 2): s's
 *     coefficients are rotated into the frame whose pole points at c_t
 *     (Wigner-type rotation through a fixed per-degree matrix, reading R25),
 *     evaluated on t's pole-aligned discs (eq 4.8; eq 4.9's geometry),
 *     re-expanded in t's vector spherical harmonics, rotated back and
 *     accumulated with t's own coefficients before the self term's single
 *     inverse transform, O(p^3) per pair.  The result is the degree-p
 *     re-expansion of the exact near field on t (it differs from mode 0 by
 *     the degree > p tail of that field, which decays spectrally with p).
 *   2, 3: measurement only -- the exterior part alone (mode 0's and mode 1's
 *     respectively) with the far field's smooth rule NOT excluding the near
 *     pairs; not an operator.
 * Modes 1 and 3 build a (p+1)(2p+1)(2p+3)/3-entry complex table and an
 * [n_spheres][nlm][6] coefficient buffer on the first call (synchronous).
 * The traction operator and the off-surface evaluators always use mode 0.
 * Returns BIE_ERR_ARG for other modes.
 */
int bie_set_near_mode(bie_ctx* ctx, int mode);

/*
 * Measurement knob: schedule of the off-surface near correction (NEXT-1 in
 * bie_eval_offsurface / bie_eval_traction).  0 (default): the (target, near
 * sphere) pairs grouped by sphere, one CTA per sphere chunk with the sphere's
 * records in shared memory, per-pair results summed per target in ascending
 * sphere order; costs one stream synchronisation per call (the pair count
 * sizes the scratch).  1: one thread per Morton-sorted target walking its own
 * near spheres (round-2 schedule).  Same operator (parity-tested).
 * BIE_ERR_ARG outside 0..1.
 */
int bie_set_near_off_schedule(bie_ctx* ctx, int schedule);

/*
 * How the applies treat the smooth rule of near pairs: 1 the far-field kernel
 * skips them (the correction adds the exact field only); 0 the far field keeps
 * them and the correction subtracts them pointwise; -1 (default) the cheaper
 * by a cost model (skipping costs ~1.5 % of the far field, subtracting one
 * smooth-rule pass per near pair).  Same operator either way (parity-tested);
 * BIE_ERR_ARG outside -1..1.
 */
int bie_set_near_exclusion(bie_ctx* ctx, int mode);

/*
 * Measurement knob: which kernel computes the spectral self term (rows a2,
 * a4-a6).  -1 (default): the fastest measured for the context's order (2 for
 * p <= 19, 0 above).  0: k_sht, the separable transforms as
 * small dense contractions on the FP64 tensor cores (mma.sync m8n8k4 f64,
 * SASS DMMA), one sphere per warp group; 1: the same schedule with DFMA
 * micro-kernels (compiled for p in {4, 6, 8, 12}; other orders use 0); 2: the
 * one-CTA-per-sphere scalar kernel; 3: the same scalar kernel with two
 * spheres per CTA (BIE_ERR_UNSUPPORTED, previous setting kept, when two
 * spheres' staging exceeds 227 KB of shared memory, p >= 24).  All compute
 * the same operator (parity-tested); they differ only in schedule and speed.
 * NEXT-4's coefficient accumulation always runs on k_sht.  BIE_ERR_ARG
 * outside -1..3.
 */
int bie_set_self_kernel(bie_ctx* ctx, int variant);

/*
 * Measurement knob: the schedule of the far-field pair-sum kernels.
 * 1 (default): source chunks chosen by a wave-aware planner, one CTA per
 *   (target tile, chunk).  With >= 16 such units per resident CTA slot the
 *   chunks of a tile are summed inside the kernel (as 5), below that through
 *   HBM partials and a fixed-order reduction kernel (as 6).
 * 5: chained in-kernel reduction -- CTAs take (chunk, tile) from a ticket
 *   counter in chunk-major order; chunk c of a tile waits for chunk c - 1's
 *   release flag, adds its partial to the tile's running sum and releases c + 1;
 *   the last chunk writes u.  Same fixed summation order as 6 (bit-identical
 *   results), no chunk partials in HBM, no reduction launch.  A wait longer
 *   than 60 s traps (the launch then fails with BIE_ERR_CUDA) instead of hanging.
 * 6: chunk partials in HBM + the fixed-order reduction kernel.
 * 0: stream-K -- one persistent CTA per resident slot, each given an equal
 *   contiguous range of (target tile, source tile) units; a target tile whose
 *   units span several CTAs is finished by a fixed-order fix-up kernel from at
 *   most 2 partial tiles per CTA (no chunk partials; measured slower: the
 *   static split cannot absorb SM-to-SM speed differences).
 * 2 / 3 / 4: when the launch is large enough (>= 16 units per resident slot),
 *   the 8 / 4 / 16 source chunks of a target tile run as ONE thread-block
 *   cluster (16: apply only, non-portable size) and are summed on chip through
 *   distributed shared memory in fixed rank order; smaller launches use 1.
 * 7: constant-bank batches (SL+DL apply without near exclusion, off-surface
 *   u / p; other far-field operators keep schedule 1).  Schedule 1 (the
 *   default) takes this path by itself for large launches (>= 0.8 waves of
 *   512-target tiles, i.e. >= 242,483 targets on 148 SMs, and >= 4992 sources);
 *   5 and 6 never do.  The sources are cut
 *   into batches of 312 records that are copied device-to-device into one of
 *   two __constant__ buffers; one launch per batch adds the batch's
 *   contribution at every target of a sub-range (<= 655,360 targets, so that
 *   the accumulators stay in L2 between launches; environment variable
 *   BIE_CONST_SUB, read by bie_create, overrides the size, 0 = one range) to
 *   an accumulator.  The FP64 instructions
 *   then take the source operands from the uniform datapath instead of the
 *   vector register file, which lifts the register-file read limit of the
 *   shared-memory kernel.  Even batches run on the caller's
 *   stream into u, odd batches on a stream owned by the context into scratch
 *   ([M][3] (+ [M]) doubles), joined before the call's work on the caller's
 *   stream ends; the two partial sums are added at the end.  The constant
 *   buffers belong to the process: passes of different contexts on one device
 *   are ordered one after the other by an event.
 * bie_set_source_chunks > 0 forces the chunked schedules (1, 5 or 6).  All
 * schedules are deterministic; they differ only in fp64 summation grouping
 * (1, 5 and 6 not at all).  BIE_ERR_ARG outside 0..7.
 */
int bie_set_far_reduction(bie_ctx* ctx, int mode);

/*
 * Tuning knob: number of source chunks of the far-field kernel (0 = automatic;
 * otherwise 1..4096).  Results are deterministic for a given value; different
 * values change only the fp64 summation grouping.
 */
int bie_set_source_chunks(bie_ctx* ctx, int chunks);

const char* bie_status_string(int status);
const char* bie_last_error(const bie_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* BIE_H */
