/*
 * prgd.h — C-ABI of the B200 (sm_100a) PRGD hot path for low-TT-rank tensor
 * completion (arXiv 2501.13385, "Fast and Provable Tensor-Train Format Tensor
 * Completion via Preconditioned Riemannian Gradient Descent").
 *
 * Problem (`model: Low TT`):
 *     min_T  f(T) = 1/2 <T - T*, P_Omega(T - T*)>   s.t.  rank_tt(T) = r,
 * solved by Alg. 2.  One call of tt_prgd_step is one pass of
 * the loop body (lines 214-218) without trimming.
 *
 * Conventions (all functions):
 *  - d >= 2 modes, mode sizes n[0..d-1] (paper: d_1..d_m), TT ranks r[0..d] with
 *    r[0] = r[d] = 1 (paper: r_0..r_m).  Indices are 0-based.
 *  - Cores are float64, C-order [r[k]][n[k]][r[k+1]] (T_k in
 *    R^{r_{k-1} x d_k x r_k}).
 *  - Pointers named h_* are HOST pointers.  The library copies in/out; the caller
 *    keeps ownership of its buffers and may reuse them when the call returns.
 *    Device memory is owned by the context (allocated through the allocator hook
 *    when one is installed, else cudaMalloc) and released by tt_destroy.
 *  - Every function returns a tt_status.  On a non-OK status the context (if any)
 *    keeps a message readable with tt_last_error; the context stays usable
 *    unless the status is TT_ERR_CUDA.
 *  - Work is enqueued on the context's stream (tt_set_stream; default: a stream
 *    the library creates).  Calls that return data to the host synchronise that
 *    stream; tt_prgd_step does not (device-side numeric faults are reported by the
 *    next synchronising call as TT_ERR_NUMERIC).
 *  - A context is not thread-safe; distinct contexts are independent.
 *  - Device kernels only: there is no CPU fallback.  Without a usable sm_100
 *    device tt_create returns TT_ERR_CUDA.
 */
#ifndef PRGD_H
#define PRGD_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PRGD_API __attribute__((visibility("default")))
#else
#define PRGD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tt_status {
  TT_OK = 0,
  TT_ERR_ARG = -1,          /* bad argument (null pointer, size, enum, out of range k) */
  TT_ERR_RANK = -2,         /* infeasible TT ranks (see tt_create) */
  TT_ERR_INDEX = -3,        /* an observed or queried index outside [0, n_k) */
  TT_ERR_STATE = -4,        /* call needs observations / cores not set yet */
  TT_ERR_NUMERIC = -5,      /* NaN/Inf, or Cholesky breakdown of a right Gram P_k */
  TT_ERR_CUDA = -6,         /* CUDA runtime error (no device, launch failure) */
  TT_ERR_OOM = -7,          /* device allocation failed */
  TT_ERR_UNSUPPORTED = -8   /* valid but outside this build's limits (see tt_plan) */
} tt_status;

typedef struct tt_ctx tt_ctx;

/* eps rules of the data-driven metric G_{l,k} = eps I + diag(M_k(G) M_k(G)^T)
 * (PAPER.md:161-165):
 *   TT_EPS_VEE   eps_l = ||G_l||_vee^2 = max_{k,j} ||M_k(G_l)(j,:)||^2, per iteration
 *                (default).  eps_l = 0 (exact fit) makes the step a no-op.
 *   TT_EPS_FIXED eps given by tt_set_metric (> 0), constant.
 *   TT_EPS_NONE  W = I: the RGD iteration through the same path.
 * step rules (A12):
 *   TT_STEP_THEORY alpha_l = step_size * eps_l^{1/2} / p (Thm 4.1 with step_size =
 *                  1.001; with TT_EPS_NONE: step_size / p).  Default.
 *   TT_STEP_RAW    alpha_l = step_size.
 *   TT_STEP_ADAPTIVE  the steepest step along the search direction in the tangent space,
 *                  alpha_l = step_size * ||P~_T W^{-1} G||_W^2 / ||P_Omega P~_T W^{-1} G||_F^2
 *                  (eq. `PRGD stepsize`; with TT_EPS_NONE RGD's
 *                  ||P_T G||^2 / ||P_Omega P_T G||^2).  Costs one more pass
 *                  over Omega per step (the tangent vector evaluated at every sample);
 *                  alpha_l = 0 if that vanishes. */
enum { TT_EPS_VEE = 0, TT_EPS_FIXED = 1, TT_EPS_NONE = 2 };
enum { TT_STEP_THEORY = 0, TT_STEP_RAW = 1, TT_STEP_ADAPTIVE = 2 };

/* ------------------------------------------------------------------ lifecycle */

/* Create a context for order-d tensors of mode sizes n[d] and TT ranks r[d+1].
 * Ranks must satisfy r[0] = r[d] = 1, r[k] >= 1 and the feasibility bounds
 * r[k] <= min(prod_{i<k} n_i, prod_{i>=k} n_i), r[k] <= r[k-1] n[k-1],
 * r[k-1] <= n[k-1] r[k] (TT_ERR_RANK otherwise).  Build limits
 * (TT_ERR_UNSUPPORTED): r[k] <= 32, and some prefix split K with
 * prod(n[0..K-1]) and prod(n[K..d-1]) both <= 2^30 (see tt_plan), with the split-level
 * tables below 2^31 doubles (max(N_L, N_R) * pad(r_K) < 2^31; 32-bit table offsets).
 * Cores start at zero; observations unset.  *out receives the context. */
PRGD_API int tt_create(int d, const int64_t* n, const int64_t* r, tt_ctx** out);

/* Release all device memory and the context.  NULL is a no-op.  (Plumbing: the paper's
 * method is CPU-only and defines no resource calls; tt_destroy, tt_set_stream and
 * tt_set_allocator follow SURVEY.md §8(b).) */
PRGD_API int tt_destroy(tt_ctx* ctx);

/* Use `stream` (a cudaStream_t, e.g. PyTorch's current stream) for all work.
 * NULL restores the library's own stream.  Several contexts may share one stream:
 * each captures its step graphs on a private stream and only launches them on this
 * one.  tt_set_observations also uses a private side stream for the value upload. */
PRGD_API int tt_set_stream(tt_ctx* ctx, void* stream);

/* Route device allocations through alloc(bytes, user) / free(ptr, user) (e.g.
 * PyTorch's caching allocator).  Must be called before tt_set_observations and
 * before any core is set; otherwise TT_ERR_STATE. */
PRGD_API int tt_set_allocator(tt_ctx* ctx, void* (*alloc)(size_t bytes, void* user),
                     void (*release)(void* ptr, void* user), void* user);

/* Path over Omega.  Both compute the same iteration; they differ in how the
 * left / right parts T^{<=k-1}, T^{>=k+1} of every sample are formed:
 *   TT_PATH_TABLES  memoised prefix / suffix tables in HBM (one split K_L), passes over Omega
 *                   as sampled dense-dense / sparse-dense products (tables needed: see tt_create)
 *   TT_PATH_CHAINS  per-sample chains of r x r slice products ("fast recursive computations",
 *                   PAPER.md:146), interfaces materialised per sample (2 sum_k r_k doubles each),
 *                   per-mode buckets (A0) and a segmented contraction per slice (DMMA where a
 *                   piece holds >= 32 samples, rank-1 updates otherwise)
 *   TT_PATH_AUTO    tables when they fit, else chains (default)
 * Must be called before any core or observation is set (TT_ERR_STATE); TT_PATH_TABLES on a
 * shape whose tables do not fit returns TT_ERR_UNSUPPORTED.  tt_get_path reports the path in
 * use (resolved from AUTO). */
enum { TT_PATH_AUTO = 0, TT_PATH_TABLES = 1, TT_PATH_CHAINS = 2 };
PRGD_API int tt_set_path(tt_ctx* ctx, int path);
PRGD_API int tt_get_path(tt_ctx* ctx, int* path);

/* ------------------------------------------------------------------ data */

/* Set the observed set Omega: h_idx[m][d] sample-major int32
 * multi-indices (0-based), h_vals[m] the observed values y_s.  Omega is a set:
 * duplicate multi-indices are the caller's error (not detected).  Validates every
 * index (TT_ERR_INDEX), copies to the device and builds the one-time bucketing
 * (A0: stable LSD counting sorts -- into prefix and suffix order on the table path, by x_k
 * for every mode k on the chain path).  m = 0 is allowed (empty Omega).  m must be < 2^31.
 * Sets p = m / prod(n) (reading R3). */
PRGD_API int tt_set_observations(tt_ctx* ctx, const int32_t* h_idx, const double* h_vals, int64_t m);

/* The same call for compact multi-indices (the same Omega): h_idx[m][d]
 * sample-major uint8 (0-based), accepted when every n_k <= 256 (TT_ERR_ARG otherwise) -- true of
 * all of BASELINE.json's configs (n_k = 2 .. 256).  The indices are a quarter of the int32
 * bytes on the host link (config 5: 0.3 GB instead of 1.2 GB); they are widened to int32 on the
 * device and then bucketed exactly as in tt_set_observations (same validation, same errors,
 * same resulting state).  h_idx / h_vals are host pointers, read before the call returns. */
PRGD_API int tt_set_observations_u8(tt_ctx* ctx, const uint8_t* h_idx, const double* h_vals, int64_t m);

/* Copy core k (0 <= k < d) in/out, [r[k]][n[k]][r[k+1]] C-order float64.
 * Cores may be in any gauge; after tt_prgd_step cores 0..d-2 are left-orthogonal
 * (L(T_k)^T L(T_k) = I) and core d-1 carries the norm.
 * tt_get_core synchronises the stream. */
PRGD_API int tt_set_core(tt_ctx* ctx, int k, const double* h_core);
PRGD_API int tt_get_core(tt_ctx* ctx, int k, double* h_core_out);

/* Metric / step rules, see the enums above.  eps is used by TT_EPS_FIXED only
 * (must be > 0 then).  Defaults: TT_EPS_VEE, TT_STEP_THEORY.  TT_STEP_ADAPTIVE allocates
 * its buffers here (TT_ERR_OOM).  The denominator ||P_Omega D||^2 is evaluated through the
 * tables when 2 r_k <= 32 on the table path, else by per-sample chains of the rank-2r tangent
 * TT (the multi-indices of Omega stay on the device for this). */
PRGD_API int tt_set_metric(tt_ctx* ctx, int eps_rule, double eps, int step_rule);

/* Retraction (Alg. 2 line 5):
 *   TT_RETRACT_PLAIN     T_{l+1} = SVD_r^tt(W_l), Alg. 1 as TT-rounding of the rank-2r W_l (default;
 *                        reading R8).  Output cores 0..d-2 left-orthogonal.
 *   TT_RETRACT_WEIGHTED  T_{l+1} = W_l^{-1/2} SVD_r^tt(W_l^{1/2} W_l), the alternative of the Remark
 *                        at PAPER.md:365-367 (PRGD becomes "almost RGD on That"): the rounding acts on
 *                        the weighted blocks and the rounded cores' mode-2 slices are divided by
 *                        phi_{k,j} (Prop. 3.1).  Output cores are then not left-orthogonal.
 * Takes effect from the next tt_prgd_step. */
enum { TT_RETRACT_PLAIN = 0, TT_RETRACT_WEIGHTED = 1 };
PRGD_API int tt_set_retraction(tt_ctx* ctx, int kind);

/* Spectral initialisation at scale: set every core to
 * T_0 = SVD_r^tt(p^{-1} P_Omega(y)), Alg. 1 (TT-SVD) applied to the sparse
 * zero-filled, rescaled observations (the "TT-SVD spectral initialization" of PAPER.md:42;
 * BASELINE.json config 1) without densifying it: step k takes the top r_k eigenvectors of the
 * Gram of the projected unfolding, accumulated over the samples grouped by (x_{k+1..d}, x_k)
 * (DESIGN.md §2); an unfolding with r_{k-1} n_k > 1024 rows (config 3: 4096) is taken from the
 * other side when it has at most 1024 nonzero columns (the Gram M_k^T M_k, U = M_k V Lambda^{-1/2},
 * re-orthonormalised).  Gram-based, so the kept subspace is accurate to ~u ||G|| / eigen-gap.
 * Needs observations (TT_ERR_STATE otherwise, and in sharded mode), prod(n) < 2^62, per step
 * r_{k-1} n_k <= 1024 or at most 1024 distinct suffixes (x_{k+1}..x_d) in Omega (TT_ERR_ARG),
 * and the table path (TT_ERR_STATE on the chain path).  Synchronous.  Output cores 0..d-2 have
 * orthonormal columns L(T_k). */
PRGD_API int tt_spectral_init(tt_ctx* ctx);

/* ------------------------------------------------------------------ the hot path */

/* One PRGD iteration (Alg. 2; no Trim):
 *   G_l = P_Omega(T_l - y)                           A1-A2 (pass A over Omega)
 *   weights, eps_l, phi = (eps + h)^{1/(4d)}         A3
 *   That = W^{1/2} T_l left-orthogonalised, P_k      A4-A6
 *   Y_k = (That^{<=k-1} (x) I)^T (W^{-1/2}G)^{<k>} (That^{>=k+1})^T   A7-A9 (pass B)
 *   closed-form projection, unweighting              A10-A11
 *   alpha_l, rank-2r W_l, TT-rounding SVD_r^tt(W_l)  A12-A14
 * Enqueued asynchronously; step_size as in the step rule.  Returns TT_ERR_STATE
 * without observations (m = 0 included) or before any core was set.
 * With eps_l = 0 under TT_EPS_VEE the iterate is left unchanged (reading R4). */
PRGD_API int tt_prgd_step(tt_ctx* ctx, double step_size);

/* Evaluate the CURRENT iterate at h_idx[count][d] (A1) into
 * h_out[count].  Validates indices (TT_ERR_INDEX).  count = 0 is a no-op.
 * Synchronises. */
PRGD_API int tt_eval_at(tt_ctx* ctx, const int32_t* h_idx, int64_t count, double* h_out);

/* ||P_Omega(T_cur) - y||_2 at the CURRENT iterate (0 for empty Omega): the norm of the sparse
 * residual G_l = P_Omega(T_l - T*) of Alg. 2 line 1 (y replaces T*, reading R14),
 * i.e. sqrt(2 f(T_cur)) for the objective f(T) = 1/2 <T - T*, P_Omega(T - T*)> of PAPER.md:30-41.
 * Synchronises; reports pending TT_ERR_NUMERIC. */
PRGD_API int tt_residual_norm(tt_ctx* ctx, double* out);

/* Wait for all enqueued work; report pending device faults (TT_ERR_NUMERIC). */
PRGD_API int tt_sync(tt_ctx* ctx);

/* Message for the last non-OK status on ctx (static "..." string for NULL ctx). */
PRGD_API const char* tt_last_error(const tt_ctx* ctx);

/* ------------------------------------------------------------------ sharded (multi-GPU) */

/* Sharded mode: Omega is split over ranks, one context per
 * rank (one GPU each) holding the same cores and its own observations; every h_{k,j}
 * and every contraction Y_k is a sum over samples, so a step
 * all-reduces exactly two buffers -- h (sum_k n_k doubles) after pass A and Y (sum_k
 * r_k n_k r_{k+1} doubles) after pass B -- and replicates the small dense work, which keeps
 * the iterates identical on all ranks.  fn(buf, count, stream, user) must enqueue an in-place
 * fp64 sum over ranks of the DEVICE buffer buf[count] on `stream` (a cudaStream_t, e.g. NCCL
 * through torch.distributed) and return; it is called from the host thread inside
 * tt_prgd_step / tt_residual_norm.  m_global = |Omega| summed over ranks (p = m_global /
 * prod(n), reading R3).  Must be called before tt_set_observations (TT_ERR_STATE); fn = NULL
 * returns to the single-rank mode. */
typedef void (*tt_allreduce_fn)(double* buf, int64_t count, void* stream, void* user);
PRGD_API int tt_set_allreduce(tt_ctx* ctx, tt_allreduce_fn fn, void* user, int64_t m_global);

/* ------------------------------------------------------------------ introspection */

/* Host-only planning (no device needed): validates (d, n, r) like tt_create and
 * returns the prefix/suffix split K_L (1..d-1) used by the table path's bucketing and
 * partial-product tables: N_L = prod(n[0..K_L-1]), N_R = prod(n[K_L..d-1]).  For shapes
 * whose tables do not fit (TT_PATH_AUTO resolves to the chain path) K_L = 0, N_L = N_R = 0.
 * Any output pointer may be NULL. */
PRGD_API int tt_plan(int d, const int64_t* n, const int64_t* r, int* K_L, int64_t* N_L, int64_t* N_R);

/* Counters: launches = kernels this context launched since creation (graph nodes
 * counted per replay); steps = tt_prgd_step calls. */
typedef struct tt_stats {
  int64_t launches;
  int64_t steps;
  int64_t launches_per_step;
  int32_t K_L;
  int32_t graphs;           /* 1 when the step runs as a captured CUDA graph */
} tt_stats;
PRGD_API int tt_get_stats(tt_ctx* ctx, tt_stats* out);

/* Profiling: when on, steps run as direct launches with a CUDA-event pair around
 * every kernel group; tt_get_profile returns the accumulated milliseconds per
 * group (names via tt_profile_name) and the number of steps accumulated, then
 * resets.  Off by default (steps run as one captured graph). */
PRGD_API int tt_set_profiling(tt_ctx* ctx, int on);
PRGD_API int tt_get_profile(tt_ctx* ctx, double* h_ms, int cap, int* n_groups, int64_t* n_steps);
PRGD_API const char* tt_profile_name(int group);

/* Debug readback of internal device state into host memory (tests only):
 * what = TT_DBG_* below, k = mode where relevant, cap = capacity in elements.
 * Returns the element count in *count.  Synchronises. */
enum {
  TT_DBG_PERM_PRE = 1,   /* int32[m]   sample ids in prefix order (table path)  (A0) */
  TT_DBG_OFFS_L = 2,     /* int64[N_L+1] prefix bucket offsets (table path)     (A0) */
  TT_DBG_PERM_SUF = 3,   /* int32[m]   sample ids in suffix order (table path)  (A0) */
  TT_DBG_OFFS_R = 4,     /* int64[N_R+1] suffix bucket offsets (table path)     (A0) */
  TT_DBG_RESID = 5,      /* double[m]  g_s in ORIGINAL sample order          (A2) */
  TT_DBG_H = 6,          /* double[n_k] h_{k,j} of the last pass A           (A3) */
  TT_DBG_PHI = 7,        /* double[n_k] phi_{k,j} of the last step           (A3) */
  TT_DBG_EPS = 8,        /* double[13] or [29] (cap >= 29): eps, sum g^2, alpha, p, Jacobi sweeps,
                            then 8 (24) cumulative dense-phase cycle counters / counts */
  TT_DBG_U = 9,          /* double[core k] U_k of the last step              (A5) */
  TT_DBG_P = 10,         /* double[r_k+1 ^2] P_{k+1} (right Gram) of last step (A6) */
  TT_DBG_Y = 11,         /* double[core k] Y_k of the last step              (A9) */
  TT_DBG_AHAT = 12,      /* double[core k] Ahat_k of the last step           (A10) */
  TT_DBG_PERM_MODE = 13, /* int32[m]   sample ids bucketed by x_k (chain path) (A0) */
  TT_DBG_OFFS_MODE = 14  /* int64[n_k+1] mode-k bucket offsets (chain path)    (A0) */
};
PRGD_API int tt_debug_get(tt_ctx* ctx, int what, int k, void* h_out, int64_t cap, int64_t* count);

/* Test hook for A14 alone: upload a rank-2r block TT h_B (count doubles, the layout the step
 * assembles: core k is [R_k][n_k][R_{k+1}] with R_0 = R_d = 1 and R_k = 2 r_k otherwise, cores
 * concatenated) and run only the TT-rounding SVD_r^tt (Alg. 1 as TT-rounding)
 * into the context's cores (read them with tt_get_core).  Synchronous; TT_ERR_ARG on a count
 * mismatch, TT_ERR_NUMERIC if the rounding reports a fault. */
PRGD_API int tt_debug_round(tt_ctx* ctx, const double* h_B, int64_t count);

#ifdef __cplusplus
}
#endif
#endif /* PRGD_H */
