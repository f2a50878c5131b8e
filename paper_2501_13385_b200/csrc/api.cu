// api.cu — the C-ABI of include/prgd.h: context, planning, device memory, the
// per-iteration orchestration (two captured CUDA graphs) and debug readback.
//
// One iteration = G_B ("update": weights, orthogonalisation, pass B, backward
// recursions, projection + rounding) followed by G_A ("evaluate": C tables, pass A,
// marginals) of the new iterate, so tt_residual_norm after a step costs nothing and
// every step does exactly one pass A and one pass B over Omega.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/prgd.h"
#include "prgd_internal.cuh"

using namespace prgd;

namespace {

constexpr int kNumGroups = 12;
const char* kGroupNames[kNumGroups] = {
    "tables_C",   "passA_prefix", "passA_suffix", "marginals",   "weights_psi", "dense_orth",
    "tables_U",   "passB_prefix", "passB_suffix", "backward_Y", "dense_round", "adaptive_step"};

constexpr int64_t kSplit = 256;        // max samples per virtual row
constexpr int kVrowCost = 8;            // plan cost of a virtual row: samples + kVrowCost
constexpr int64_t kWarpCost = 320;      // plan cost per warp (about 8 rows of 30 samples)

int64_t sat_mul(int64_t a, int64_t b) {
  const int64_t cap = (int64_t)1 << 62;
  if (a == 0 || b == 0) return 0;
  if (a > cap / b) return cap;
  return a * b;
}

struct Plan {
  int KL = 0;             // table path: prefix/suffix split (0 on the chain path)
  int64_t NL = 0, NR = 0;
  bool chain = false;     // per-sample chain path (chains.cu) instead of the tables
};

// path: TT_PATH_AUTO (tables when they fit, else chains), TT_PATH_TABLES, TT_PATH_CHAINS.
int validate_and_plan(int d, const int64_t* n, const int64_t* r, Plan* pl, std::string* msg,
                      int path = TT_PATH_AUTO) {
  if (d < 2 || d > kMaxD || !n || !r) {
    *msg = "need 2 <= d <= 64 and non-null n, r";
    return TT_ERR_ARG;
  }
  for (int k = 0; k < d; ++k)
    if (n[k] < 1 || n[k] > (1 << 30)) {
      *msg = "mode sizes must be in [1, 2^30]";
      return TT_ERR_ARG;
    }
  if (r[0] != 1 || r[d] != 1) {
    *msg = "r[0] and r[d] must be 1";
    return TT_ERR_RANK;
  }
  for (int k = 1; k < d; ++k) {
    if (r[k] < 1) {
      *msg = "ranks must be >= 1";
      return TT_ERR_RANK;
    }
    int64_t left = 1, right = 1;
    for (int i = 0; i < k; ++i) left = sat_mul(left, n[i]);
    for (int i = k; i < d; ++i) right = sat_mul(right, n[i]);
    if (r[k] > std::min(left, right) || r[k] > sat_mul(r[k - 1], n[k - 1]) ||
        r[k] > sat_mul(r[k + 1], n[k])) {
      *msg = "infeasible TT rank r[" + std::to_string(k) + "]";
      return TT_ERR_RANK;
    }
  }
  for (int k = 1; k < d; ++k)
    if (r[k] > kMaxRank) {
      *msg = "TT ranks above 32 are not supported by this build";
      return TT_ERR_UNSUPPORTED;
    }
  int best = -1;
  int64_t bestv = 0, bNL = 0, bNR = 0;
  for (int kl = 1; kl < d; ++kl) {
    int64_t NL = 1, NR = 1;
    for (int i = 0; i < kl; ++i) NL = sat_mul(NL, n[i]);
    for (int i = kl; i < d; ++i) NR = sat_mul(NR, n[i]);
    int64_t v = std::max(NL, NR);
    if (best < 0 || v < bestv) {
      best = kl;
      bestv = v;
      bNL = NL;
      bNR = NR;
    }
  }
  bool tables_fit = bestv <= ((int64_t)1 << 30);
  if (tables_fit) {   // the pass kernels index the gathered split-level table with 32-bit offsets
    int pr = 2;
    while (pr < r[best]) pr <<= 1;
    tables_fit = bestv * pr < ((int64_t)1 << 31);
  }
  if (path == TT_PATH_TABLES && !tables_fit) {
    *msg = "table path: no prefix/suffix split with both table sizes <= 2^30 rows and split-level "
           "tables below 2^31 doubles";
    return TT_ERR_UNSUPPORTED;
  }
  *pl = Plan();
  if (path == TT_PATH_CHAINS || !tables_fit) {
    pl->chain = true;
    return TT_OK;
  }
  pl->KL = best;
  pl->NL = bNL;
  pl->NR = bNR;
  return TT_OK;
}

}  // namespace

struct tt_ctx {
  int d = 0;
  std::vector<int64_t> n, r;
  std::vector<int> n_i, ldr;
  Plan plan;
  std::vector<int64_t> NLk, NRk;   // NLk[k] = prod n[0..k-1] (k=0..KL), NRk[k] = prod n[k..d-1]
  std::string err;

  void* (*halloc)(size_t, void*) = nullptr;
  void (*hfree)(void*, void*) = nullptr;
  void* huser = nullptr;
  std::vector<void*> base_allocs, obs_allocs;

  cudaStream_t own_stream = nullptr, stream = nullptr;
  cudaStream_t side = nullptr;               // uploads overlapped with the bucketing sorts
  cudaStream_t cap = nullptr;                // private graph-capture stream
  cudaEvent_t ev_side[2] = {nullptr, nullptr};
  cudaStream_t ovl = nullptr;                // pass-B suffix branch beside the end of A5 / A6
  cudaEvent_t ev_ovl[2] = {nullptr, nullptr};

  bool base_ready = false;
  int* n_dev = nullptr;
  double *C = nullptr, *U = nullptr, *Y = nullptr, *Ahat = nullptr, *phi = nullptr, *h = nullptr;
  double *P = nullptr, *L = nullptr, *B = nullptr, *work = nullptr, *clw = nullptr;
  double* vwarm = nullptr;   // truncation Jacobi warm starts (k_round_cs), [2][d][32*32]
  int* wok = nullptr;
  int64_t clw_len = 0;
  int64_t work_len = 0;
  std::vector<int64_t> core_off, phi_off, b_off, p_off;
  Scalars* sc = nullptr;
  Scalars* sc_host = nullptr;
  std::vector<double*> LT, EL, RT, FR;
  double *HL = nullptr, *HR = nullptr, *psiL = nullptr, *psiR = nullptr, *Ypart = nullptr;
  double* margp = nullptr;      // marginal chunk partials, 32 * sum(n)
  double* g_suf = nullptr;      // residual in suffix order (written by pass A)
  // sliced pass A suffix (gsq_q >= 2 slices of g of gsq_slen samples): the sliced order's
  // prefix positions / suffix buckets, its index of every suffix-ordered sample, the staged g
  // (sliced order, read by pass B through sl_q) and the per-slice bucket sums
  int gsq_q = 0;
  int64_t gsq_slen = 0;
  int32_t *sl_pos = nullptr, *sl_row = nullptr, *sl_q = nullptr;
  double *stage = nullptr, *HRq = nullptr;
  int32_t* pre2suf = nullptr;   // suffix position of prefix position t
  int64_t Ypart_cap = 0;

  int path_req = TT_PATH_AUTO;  // tt_set_path
  // observed multi-indices, int32 [m][d] (the ABI layout), kept on the device: the chain path
  // reads them every pass; the table path uses them for the adaptive denominator when 2r > 32
  int32_t* idx_dev = nullptr;
  // chain path (chains.cu): values / residual / preconditioned residual in the original sample
  // order, interfaces IL_k / IR_k [k][s][r_k], per-mode buckets and their pieces
  double *yobs = nullptr, *ghat = nullptr, *IL = nullptr, *IR = nullptr;
  ChainPieces pcs;
  ChainTT ctt{};
  double* dval = nullptr;       // adaptive step by chains: D(x_s)^2
  double* Dblk = nullptr;       // adaptive step by chains: block cores of the tangent vector
  ChainTT dtt{};

  bool obs_set = false;
  int64_t m = 0;
  double p = 0.0;
  int32_t *Spre = nullptr, *sid_pre = nullptr, *pos_suf = nullptr, *Psuf = nullptr,
          *sid_suf = nullptr;
  double *ypre = nullptr, *g = nullptr;
  int32_t* Ppre = nullptr;    // bucket (prefix table row) of each sample, prefix order
  void* frec = nullptr;       // chunk records of the flat pass A
  int64_t *offsL = nullptr, *offsR = nullptr;
  SegPlan planL, planR;

  std::vector<char> core_set;
  bool evalValid = false, tablesC = false;
  int eps_rule = TT_EPS_VEE, step_rule = TT_STEP_THEORY;
  int retraction = TT_RETRACT_PLAIN;
  double eps_fixed = 0.0;

  cudaGraphExec_t gA = nullptr, gB = nullptr;
  // sharded (multi-rank) mode: Omega is split over ranks; h and Y are all-reduced
  cudaGraphExec_t gA1 = nullptr, gB1 = nullptr, gB2 = nullptr, gB3 = nullptr;
  int64_t nA1 = 0, nB1 = 0, nB2 = 0, nB3 = 0;
  // adaptive step (TT_STEP_ADAPTIVE): stacked cores, concatenated table inputs, den partials
  double *Dcore = nullptr, *dcatL = nullptr, *dcatR = nullptr, *dpart = nullptr;
  tt_allreduce_fn allreduce = nullptr;
  void* ar_user = nullptr;
  int64_t m_global = -1;
  int64_t nA = 0, nB = 0;
  int64_t launches = 0, steps = 0;

  bool profiling = false;
  cudaEvent_t ev[2 * kNumGroups] = {};
  bool ev_ready = false;
  double prof_ms[kNumGroups] = {};
  int64_t prof_steps = 0;
  bool capturing = false;
};

namespace {

int fail(tt_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(tt_ctx* c, cudaError_t e, const char* where) {
  return fail(c, TT_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                                  \
  do {                                                            \
    cudaError_t e_ = (call);                                      \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);      \
  } while (0)

void* dalloc(tt_ctx* ctx, size_t bytes, std::vector<void*>& list) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~(size_t)255;
  void* p = nullptr;
  if (ctx->halloc) {
    p = ctx->halloc(bytes, ctx->huser);
  } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
    p = nullptr;
  }
  if (p) list.push_back(p);
  return p;
}

void dfree_all(tt_ctx* ctx, std::vector<void*>& list) {
  for (void* p : list) {
    if (ctx->hfree) ctx->hfree(p, ctx->huser);
    else cudaFree(p);
  }
  list.clear();
}

// Diagnostic host wall-clock phases (env PRGD_TIMING=1): each mark synchronises the stream.
constexpr int64_t kGsqSliceBytes = 48ll << 20;   // g bytes per slice of the sliced pass A suffix

struct PhaseTimer {
  cudaStream_t s;
  const char* name;
  bool on;
  std::chrono::steady_clock::time_point t;
  std::string out;
  PhaseTimer(cudaStream_t st, const char* nm) : s(st), name(nm) {
    const char* e = std::getenv("PRGD_TIMING");
    on = e && *e == '1';
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    char buf[96];
    std::snprintf(buf, sizeof buf, " %s=%.2fms", what, std::chrono::duration<double, std::milli>(n - t).count());
    out += buf;
    t = n;
  }
  ~PhaseTimer() {
    if (on) std::fprintf(stderr, "[prgd] %s:%s\n", name, out.c_str());
  }
};

// Pinned host copies of the device scalars, recycled across contexts (cudaMallocHost costs about
// a millisecond per call; contexts are created per problem, e.g. every end-to-end run).
std::mutex g_pin_mu;
std::vector<Scalars*> g_pin_free;

Scalars* pinned_scalars_get() {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_free.empty()) {
      Scalars* p = g_pin_free.back();
      g_pin_free.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, sizeof(Scalars)) != cudaSuccess) return nullptr;
  return static_cast<Scalars*>(p);
}

void pinned_scalars_put(Scalars* p) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(p);
}

template <class T>
bool A(tt_ctx* ctx, T** out, int64_t count, std::vector<void*>& list) {
  *out = static_cast<T*>(dalloc(ctx, (size_t)std::max<int64_t>(count, 1) * sizeof(T), list));
  return *out != nullptr;
}

void drop_graphs(tt_ctx* ctx) {
  if (ctx->gA) cudaGraphExecDestroy(ctx->gA);
  if (ctx->gB) cudaGraphExecDestroy(ctx->gB);
  ctx->gA = ctx->gB = nullptr;
  for (cudaGraphExec_t* g : {&ctx->gA1, &ctx->gB1, &ctx->gB2, &ctx->gB3}) {
    if (*g) cudaGraphExecDestroy(*g);
    *g = nullptr;
  }
}

int ensure_base(tt_ctx* ctx) {
  if (ctx->base_ready) return TT_OK;
  const int d = ctx->d;
  auto& L = ctx->base_allocs;
  const int KL = ctx->plan.KL;
  // offsets
  ctx->core_off.assign(d + 1, 0);
  ctx->phi_off.assign(d + 1, 0);
  ctx->b_off.assign(d + 1, 0);
  ctx->p_off.assign(d + 1, 0);
  int64_t maxb = 1, maxcore = 1, maxgram = 1;
  for (int k = 0; k < d; ++k) {
    const int64_t sz = ctx->r[k] * ctx->n[k] * ctx->r[k + 1];
    ctx->core_off[k + 1] = ctx->core_off[k] + sz;
    ctx->phi_off[k + 1] = ctx->phi_off[k] + ctx->n[k];
    const int64_t rb0 = (k == 0) ? 1 : 2 * ctx->r[k];
    const int64_t rb1 = (k == d - 1) ? 1 : 2 * ctx->r[k + 1];
    ctx->b_off[k + 1] = ctx->b_off[k] + rb0 * ctx->n[k] * rb1;
    ctx->p_off[k + 1] = ctx->p_off[k] + ctx->r[k + 1] * ctx->r[k + 1];
    maxb = std::max(maxb, rb0 * ctx->n[k] * rb1);
    maxcore = std::max(maxcore, sz);
    maxgram = std::max(maxgram, ctx->r[k] * ctx->n[k] * ctx->r[k + 1]);
  }
  ctx->work_len = 2 * std::max(maxb, maxcore) + maxgram + 4096;
  {
    int64_t S = 2, nmax = 1;
    for (int k = 0; k <= d; ++k) S = std::max<int64_t>(S, 2 * ctx->r[k]);
    S = S <= 8 ? 8 : (S <= 16 ? 16 : std::max<int64_t>(S, 32));   // template sizes of k_round_cs
    for (int k = 0; k < d; ++k) nmax = std::max<int64_t>(nmax, ctx->n[k]);
    const int64_t nc = round_cluster_size();
    const int64_t lds = S <= 4 ? 4 : ((S + 11) / 16) * 16 + 4;
    ctx->clw_len = 8192 + nc * 2 * ((nmax + nc - 1) / nc) * S * lds;
  }
  bool ok = A(ctx, &ctx->n_dev, d, L) && A(ctx, &ctx->C, ctx->core_off[d], L) &&
            A(ctx, &ctx->U, ctx->core_off[d], L) && A(ctx, &ctx->Y, ctx->core_off[d], L) &&
            A(ctx, &ctx->Ahat, ctx->core_off[d], L) && A(ctx, &ctx->phi, ctx->phi_off[d], L) &&
            A(ctx, &ctx->h, ctx->phi_off[d], L) && A(ctx, &ctx->P, ctx->p_off[d], L) &&
            A(ctx, &ctx->L, ctx->p_off[d], L) && A(ctx, &ctx->B, ctx->b_off[d], L) &&
            A(ctx, &ctx->work, ctx->work_len, L) && A(ctx, &ctx->clw, ctx->clw_len, L) &&
            A(ctx, &ctx->sc, 1, L) && A(ctx, &ctx->vwarm, 2 * (int64_t)d * 1024, L) &&
            A(ctx, &ctx->wok, 2 * d, L);
  if (!ok) return fail(ctx, TT_ERR_OOM, "device allocation failed (base buffers)");
  // chain-path view of the cores (and of the rank-2r block cores for the adaptive step)
  ctx->ctt = ChainTT{};
  ctx->ctt.d = d;
  ctx->dtt = ChainTT{};
  ctx->dtt.d = d;
  for (int k = 0; k <= d; ++k) {
    ctx->ctt.r[k] = (int)ctx->r[k];
    ctx->ctt.off[k] = ctx->core_off[k];
    ctx->ctt.phi_off[k] = ctx->phi_off[k];
    ctx->dtt.r[k] = (k == 0 || k == d) ? 1 : 2 * (int)ctx->r[k];
    ctx->dtt.off[k] = ctx->b_off[k];
    ctx->dtt.phi_off[k] = ctx->phi_off[k];
  }
  for (int k = 0; k < d; ++k) ctx->ctt.n[k] = ctx->dtt.n[k] = (int)ctx->n[k];
  if (ctx->plan.chain) {
    if (!(ctx->sc_host = pinned_scalars_get()))
      return fail(ctx, TT_ERR_OOM, "pinned allocation failed");
    std::memset(ctx->sc_host, 0, sizeof(Scalars));
    CK(cudaMemcpyAsync(ctx->n_dev, ctx->n_i.data(), d * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->C, 0, ctx->core_off[d] * sizeof(double), ctx->stream));
    CK(cudaMemsetAsync(ctx->sc, 0, sizeof(Scalars), ctx->stream));
    CK(cudaMemsetAsync(ctx->h, 0, ctx->phi_off[d] * sizeof(double), ctx->stream));
    CK(cudaMemsetAsync(ctx->wok, 0, 2 * d * sizeof(int), ctx->stream));
    dense_init();
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->base_ready = true;
    return TT_OK;
  }
  // tables
  ctx->LT.assign(KL + 1, nullptr);
  ctx->EL.assign(KL + 1, nullptr);
  ctx->RT.assign(d + 1, nullptr);
  ctx->FR.assign(d + 1, nullptr);
  for (int k = 1; k <= KL; ++k) {
    const int64_t sz = ctx->NLk[k] * ctx->ldr[k];
    if (!A(ctx, &ctx->LT[k], sz, L) || !A(ctx, &ctx->EL[k], sz, L))
      return fail(ctx, TT_ERR_OOM, "device allocation failed (left tables)");
  }
  for (int k = KL; k < d; ++k) {
    const int64_t sz = ctx->NRk[k] * ctx->ldr[k];
    if (!A(ctx, &ctx->RT[k], sz, L) || !A(ctx, &ctx->FR[k], sz, L))
      return fail(ctx, TT_ERR_OOM, "device allocation failed (right tables)");
  }
  if (!A(ctx, &ctx->HL, ctx->plan.NL, L) || !A(ctx, &ctx->HR, ctx->plan.NR, L) ||
      !A(ctx, &ctx->psiL, ctx->plan.NL, L) || !A(ctx, &ctx->psiR, ctx->plan.NR, L) ||
      !A(ctx, &ctx->margp, 32 * ctx->phi_off[d], L))
    return fail(ctx, TT_ERR_OOM, "device allocation failed (H / psi)");
  int64_t ycap = 1;
  for (int k = 0; k < d; ++k) {
    const int64_t ng = k < KL ? ctx->NLk[k] : (k + 1 < d ? ctx->NRk[k + 1] : 1);
    const int r0 = (int)ctx->r[k], nk = (int)ctx->n[k], r1 = (int)ctx->r[k + 1];
    ycap = std::max(ycap, Y_partial_need(ng, r0, nk, r1));
    ycap = std::max(ycap, back_partial_need(ng, r0, nk, r1));
    ycap = std::max(ycap, level_back_partial_need(ng, r0, nk, r1, ctx->ldr[k < KL ? k + 1 : k]));
  }
  ctx->Ypart_cap = ycap;
  if (!A(ctx, &ctx->Ypart, ycap, L)) return fail(ctx, TT_ERR_OOM, "device allocation failed (Y)");
  if (!(ctx->sc_host = pinned_scalars_get()))
    return fail(ctx, TT_ERR_OOM, "pinned allocation failed");
  std::memset(ctx->sc_host, 0, sizeof(Scalars));
  CK(cudaMemcpyAsync(ctx->n_dev, ctx->n_i.data(), d * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(ctx->C, 0, ctx->core_off[d] * sizeof(double), ctx->stream));
  CK(cudaMemsetAsync(ctx->sc, 0, sizeof(Scalars), ctx->stream));
  CK(cudaMemsetAsync(ctx->h, 0, ctx->phi_off[d] * sizeof(double), ctx->stream));
  CK(cudaMemsetAsync(ctx->wok, 0, 2 * d * sizeof(int), ctx->stream));
  dense_init();
  tables_init();
  levels_init();
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->base_ready = true;
  return TT_OK;
}

DenseArgs dense_args(tt_ctx* ctx) {
  DenseArgs a;
  std::memset(&a, 0, sizeof(a));
  a.d = ctx->d;
  for (int k = 0; k < ctx->d; ++k) a.n[k] = (int)ctx->n[k];
  for (int k = 0; k <= ctx->d; ++k) {
    a.r[k] = (int)ctx->r[k];
    a.core_off[k] = ctx->core_off[k];
    a.phi_off[k] = ctx->phi_off[k];
    a.b_off[k] = ctx->b_off[k];
    a.p_off[k] = ctx->p_off[k];
  }
  a.C = ctx->C;
  a.U = ctx->U;
  a.Y = ctx->Y;
  a.Ahat = ctx->Ahat;
  a.phi = ctx->phi;
  a.P = ctx->P;
  a.L = ctx->L;
  a.B = ctx->B;
  a.work = ctx->work;
  a.work_len = ctx->work_len;
  // PRGD_NO_CLUSTER=1: the one-CTA dense kernels instead of the 8-CTA cluster ones (A/B only)
  static const bool no_cluster = [] {
    const char* e = getenv("PRGD_NO_CLUSTER");
    return e && e[0] == '1';
  }();
  a.clw = no_cluster ? nullptr : ctx->clw;
  a.clw_len = ctx->clw_len;
  a.sc = ctx->sc;
  a.smem_doubles = dense_smem_doubles();
  a.wretr = ctx->retraction == TT_RETRACT_WEIGHTED ? 1 : 0;
  a.vwarm = ctx->vwarm;
  a.wok = ctx->wok;
  return a;
}

// The adaptive denominator runs by chains on the chain path and when some 2 r_k exceeds the
// table kernels' rank limit.
bool adapt_by_chains(const tt_ctx* ctx) {
  if (ctx->plan.chain) return true;
  for (int k = 0; k <= ctx->d; ++k)
    if (2 * ctx->r[k] > kMaxRank) return true;
  return false;
}

// Buffers of the adaptive step (allocated once, before any graph capture).
int ensure_adaptive(tt_ctx* ctx) {
  int rc = ensure_base(ctx);
  if (rc) return rc;
  if (ctx->Dcore || ctx->Dblk) return TT_OK;
  const int d = ctx->d, KL = ctx->plan.KL;
  if (adapt_by_chains(ctx)) {   // D evaluated by per-sample chains of the rank-2r tangent TT
    if (!A(ctx, &ctx->Dblk, ctx->b_off[d], ctx->base_allocs) ||
        !A(ctx, &ctx->dpart, adapt_vsum_parts(), ctx->base_allocs))
      return fail(ctx, TT_ERR_OOM, "device allocation failed (adaptive step)");
    return TT_OK;
  }
  int64_t lenL = 1, lenR = 1;
  for (int k = 1; k < KL; ++k) lenL = std::max<int64_t>(lenL, ctx->NLk[k] * pad_rank(2 * (int)ctx->r[k]));
  for (int k = KL; k + 1 < d; ++k)
    lenR = std::max<int64_t>(lenR, ctx->NRk[k + 1] * pad_rank(2 * (int)ctx->r[k + 1]));
  auto& L = ctx->base_allocs;
  if (!A(ctx, &ctx->Dcore, 2 * ctx->core_off[d], L) || !A(ctx, &ctx->dcatL, lenL, L) ||
      !A(ctx, &ctx->dcatR, lenR, L) || !A(ctx, &ctx->dpart, adapt_vsum_parts(), L))
    return fail(ctx, TT_ERR_OOM, "device allocation failed (adaptive step)");
  return TT_OK;
}

// ------------------------------------------------------------------ profiling groups
void grp(tt_ctx* ctx, int id, bool begin) {
  if (!ctx->profiling || ctx->capturing || !ctx->ev_ready) return;
  cudaEventRecord(ctx->ev[2 * id + (begin ? 0 : 1)], ctx->stream);
}

// ------------------------------------------------------------------ enqueue pieces
// Tables of the left / right parts: left levels 1..K_L, right levels
// d-1..K_L (the U tables scaled by psi at the split level).
// `sides`: bit 0 the left levels, bit 1 the right levels; `st` the stream (default ctx->stream).
void enqueue_tables(tt_ctx* ctx, bool useU, int64_t* lc, int sides = 3, cudaStream_t st = nullptr) {
  const int d = ctx->d, KL = ctx->plan.KL;
  cudaStream_t s = st ? st : ctx->stream;
  const double* cores = useU ? ctx->U : ctx->C;
  const Scalars* sc = useU ? ctx->sc : nullptr;
  const int lmax = KL, rmin = KL;
  std::vector<TableLevel> L, R;
  bool ok = true;
  // left levels 1..lmax (A_{k+1} from A_k and core k), right levels d-1..rmin
  for (int k = 0; k < lmax && (sides & 1); ++k) {
    TableLevel t{true, k == 0 ? nullptr : ctx->LT[k], ctx->ldr[k], cores + ctx->core_off[k],
                 (int)ctx->r[k], (int)ctx->n[k], (int)ctx->r[k + 1], ctx->LT[k + 1], ctx->ldr[k + 1],
                 ctx->NLk[k + 1], (useU && k + 1 == KL) ? ctx->psiL : nullptr};
    ok = ok && level_tab_ok(t.r0, t.nk, t.r1, t.ld_out);
    L.push_back(t);
  }
  for (int k = d - 1; k >= rmin && (sides & 2); --k) {
    TableLevel t{false, k == d - 1 ? nullptr : ctx->RT[k + 1], ctx->ldr[k + 1],
                 cores + ctx->core_off[k], (int)ctx->r[k], (int)ctx->n[k], (int)ctx->r[k + 1],
                 ctx->RT[k], ctx->ldr[k], ctx->NRk[k], (useU && k == KL) ? ctx->psiR : nullptr};
    ok = ok && level_tab_ok(t.r0, t.nk, t.r1, t.ld_out);
    R.push_back(t);
  }
  if (ok) {
    launch_table_levels(s, L, R, sc, lc);
    return;
  }
  for (const TableLevel& t : L)
    launch_table_left(s, t.in, t.ld_in, t.core, t.r0, t.nk, t.r1, t.out, t.ld_out, t.rows_out,
                      t.rowscale, sc, lc);
  for (const TableLevel& t : R)
    launch_table_right(s, t.in, t.ld_in, t.core, t.r0, t.nk, t.r1, t.out, t.ld_out, t.rows_out,
                       t.rowscale, sc, lc);
}

void enqueue_evaluate(tt_ctx* ctx, int64_t* lc, bool with_sumsq = true) {
  const int d = ctx->d, KL = ctx->plan.KL;
  cudaStream_t s = ctx->stream;
  if (ctx->plan.chain) {   // pass A by per-sample chains (A1-A2), h by bucket pieces (A3)
    if (ctx->obs_set && (ctx->m > 0 || ctx->allreduce)) {
      grp(ctx, 1, true);
      launch_chain_eval(s, 1, ctx->idx_dev, ctx->m, ctx->ctt, ctx->C, ctx->yobs, ctx->g, nullptr, nullptr, lc);
      grp(ctx, 1, false);
      grp(ctx, 3, true);
      launch_chain_h(s, ctx->pcs, ctx->ctt, ctx->m, ctx->g, ctx->h, lc);
      if (with_sumsq) launch_gather_sq_sum(s, ctx->h, ctx->n_i[0], ctx->sc, lc);
      grp(ctx, 3, false);
    }
    return;
  }
  grp(ctx, 0, true);
  enqueue_tables(ctx, false, lc);
  grp(ctx, 0, false);
  if (ctx->obs_set && (ctx->m > 0 || ctx->allreduce)) {
    grp(ctx, 1, true);
    {   // flat sample-major SDDMM with the bucket sums H_L (passes_flat.cu)
      FlatArgs a;
      a.row = ctx->Ppre;
      a.col = ctx->Spre;
      a.x = ctx->ypre;
      a.g = ctx->g;
      a.m = ctx->m;
      a.nrows = ctx->plan.NL;
      a.ncols = ctx->plan.NR;
      a.ld = ctx->ldr[KL];
      a.rowtab = ctx->LT[KL];
      a.coltab = ctx->RT[KL];
      a.out = ctx->HL;
      a.rec = ctx->frec;
      launch_flat_sddmm(s, a, lc);
    }
    grp(ctx, 1, false);
    grp(ctx, 2, true);
    if (ctx->gsq_q >= 2) {
      for (int q = 0; q < ctx->gsq_q; ++q) {
        const int64_t off = q * ctx->gsq_slen;
        const int64_t mq = std::min<int64_t>(ctx->gsq_slen, ctx->m - off);
        launch_flat_gsq(s, ctx->sl_row + off, ctx->sl_pos + off, ctx->g, std::max<int64_t>(mq, 0),
                        ctx->plan.NR, ctx->stage + off, ctx->HRq + q * ctx->plan.NR, ctx->frec, lc);
      }
      launch_sum_slices(s, ctx->HRq, ctx->gsq_q, ctx->plan.NR, ctx->HR, lc);
    } else {
      SegArgs b{};
      b.plan = &ctx->planR;
      b.mode = kGSQ;
      b.ld = ctx->ldr[KL];
      b.perm = ctx->pos_suf;
      b.g = ctx->g;
      b.g2 = ctx->g_suf;      // the gathered g, stored in suffix order for pass B
      b.out = ctx->HR;
      launch_seg(s, b, nullptr, lc);
    }
    grp(ctx, 2, false);
    grp(ctx, 3, true);
    launch_marginals(s, ctx->HL, ctx->plan.NL, KL, ctx->n_i.data(), true, ctx->h,
                     ctx->margp, lc);
    launch_marginals(s, ctx->HR, ctx->plan.NR, d - KL, ctx->n_i.data() + KL, false,
                     ctx->h + ctx->phi_off[KL], ctx->margp + 32 * ctx->phi_off[KL], lc);
    if (with_sumsq) launch_gather_sq_sum(s, ctx->h, ctx->n_i[0], ctx->sc, lc);
    grp(ctx, 3, false);
  }
}

// part 0: the whole update; part 1: up to the contractions Y (pass B + backward);
// part 2: projection + rank-2r assembly + rounding (sharded mode all-reduces Y between).
// Adaptive step, front half: projection with the numerator terms, the
// one-Ahat chain tables LD / RD (in the E / F buffers, free after the backward recursions),
// the DPASS evaluation of D on Omega and the denominator.  The back half (alpha, assembly,
// rounding) is enqueue_adaptive_back; in sharded mode the denominator is all-reduced between.
void enqueue_adaptive_front(tt_ctx* ctx, int64_t* lc) {
  const int d = ctx->d, KL = ctx->plan.KL;
  cudaStream_t s = ctx->stream;
  DenseArgs da = dense_args(ctx);
  grp(ctx, 11, true);
  launch_project(s, da, 1, lc);
  if (adapt_by_chains(ctx)) {
    // D = sum_k [Ttil_1..A_k..Ttil_d] as a rank-2r block TT, evaluated by per-sample chains
    launch_tangent_cores(s, ctx->U, ctx->Ahat, ctx->phi, ctx->ctt, ctx->dtt, ctx->Dblk, ctx->sc, lc);
    if (ctx->m > 0) {
      launch_chain_eval(s, 2, ctx->idx_dev, ctx->m, ctx->dtt, ctx->Dblk, nullptr, ctx->dval, ctx->sc,
                        nullptr, lc);
      launch_adapt_den(s, ctx->dval, ctx->m, ctx->dpart, ctx->sc, lc);
    } else {
      cudaMemsetAsync(&ctx->sc->adapt_den, 0, sizeof(double), s);
    }
    grp(ctx, 11, false);
    return;
  }
  std::vector<int> ni(d), ri(d + 1);
  for (int k = 0; k < d; ++k) ni[k] = (int)ctx->n[k];
  for (int k = 0; k <= d; ++k) ri[k] = (int)ctx->r[k];
  launch_stack_cores(s, d, ni.data(), ri.data(), ctx->core_off.data(), KL, ctx->U, ctx->Ahat, ctx->Dcore,
                     ctx->sc, lc);
  const int nlev = std::max(KL, d - KL);
  for (int i = 0; i < nlev; ++i) {
    const bool hasL = i < KL, hasR = d - 1 - i >= KL;
    const int kR = d - 1 - i;
    const bool catL = hasL && i >= 1, catR = hasR && kR < d - 1;
    const int ldcL = catL ? pad_rank(2 * (int)ctx->r[i]) : 0;
    const int ldcR = catR ? pad_rank(2 * (int)ctx->r[kR + 1]) : 0;
    if (catL || catR)
      launch_concat2(s, catL ? ctx->dcatL : nullptr, ldcL, catL ? ctx->EL[i] : nullptr, ctx->ldr[i],
                     catL ? ctx->LT[i] : nullptr, ctx->ldr[i], catL ? ctx->NLk[i] : 0, (int)ctx->r[i],
                     catR ? ctx->dcatR : nullptr, ldcR, catR ? ctx->FR[kR + 1] : nullptr,
                     ctx->ldr[kR + 1], catR ? ctx->RT[kR + 1] : nullptr, ctx->ldr[kR + 1],
                     catR ? ctx->NRk[kR + 1] : 0, (int)ctx->r[kR + 1], ctx->sc, lc);
    std::vector<TableLevel> L, R;
    if (hasL) {
      TableLevel t{true, catL ? ctx->dcatL : nullptr, ldcL,
                   catL ? ctx->Dcore + 2 * ctx->core_off[i] : ctx->Ahat + ctx->core_off[i],
                   catL ? 2 * (int)ctx->r[i] : (int)ctx->r[i], (int)ctx->n[i], (int)ctx->r[i + 1],
                   ctx->EL[i + 1], ctx->ldr[i + 1], ctx->NLk[i + 1], i + 1 == KL ? ctx->psiL : nullptr};
      L.push_back(t);
    }
    if (hasR) {
      TableLevel t{false, catR ? ctx->dcatR : nullptr, ldcR,
                   catR ? ctx->Dcore + 2 * ctx->core_off[kR] : ctx->Ahat + ctx->core_off[kR],
                   (int)ctx->r[kR], (int)ctx->n[kR], catR ? 2 * (int)ctx->r[kR + 1] : (int)ctx->r[kR + 1],
                   ctx->FR[kR], ctx->ldr[kR], ctx->NRk[kR], kR == KL ? ctx->psiR : nullptr};
      R.push_back(t);
    }
    bool ok = true;
    for (const TableLevel& t : L) ok = ok && level_tab_ok(t.r0, t.nk, t.r1, t.ld_out);
    for (const TableLevel& t : R) ok = ok && level_tab_ok(t.r0, t.nk, t.r1, t.ld_out);
    if (ok) {
      launch_table_levels(s, L, R, ctx->sc, lc);
    } else {
      for (const TableLevel& t : L)
        launch_table_left(s, t.in, t.ld_in, t.core, t.r0, t.nk, t.r1, t.out, t.ld_out, t.rows_out,
                          t.rowscale, ctx->sc, lc);
      for (const TableLevel& t : R)
        launch_table_right(s, t.in, t.ld_in, t.core, t.r0, t.nk, t.r1, t.out, t.ld_out, t.rows_out,
                           t.rowscale, ctx->sc, lc);
    }
  }
  if (ctx->m > 0) {
    SegArgs a{};
    a.plan = &ctx->planL;
    a.mode = kDPASS;
    a.ld = ctx->ldr[KL];
    a.col = ctx->Spre;
    a.rowtab = ctx->EL[KL];     // LD (psi_L scaled)
    a.rowtab2 = ctx->LT[KL];    // LU (psi_L scaled)
    a.coltab = ctx->RT[KL];     // RU (psi_R scaled)
    a.coltab2 = ctx->FR[KL];    // RD (psi_R scaled)
    a.out = ctx->HL;
    launch_seg(s, a, ctx->sc, lc);
    launch_adapt_den(s, ctx->HL, ctx->plan.NL, ctx->dpart, ctx->sc, lc);
  } else {
    cudaMemsetAsync(&ctx->sc->adapt_den, 0, sizeof(double), s);
  }
  grp(ctx, 11, false);
}

void enqueue_adaptive_back(tt_ctx* ctx, int64_t* lc) {
  cudaStream_t s = ctx->stream;
  DenseArgs da = dense_args(ctx);
  grp(ctx, 10, true);
  launch_adapt_alpha(s, ctx->d, ctx->sc, lc);
  launch_project(s, da, 2, lc);
  launch_round_only(s, da, lc);
  grp(ctx, 10, false);
}

// part 0: the whole update; part 1: up to Y (sharded, before the Y all-reduce); part 2: after
// the Y all-reduce (rounding, or the adaptive front half); part 3: adaptive back half.
void enqueue_update(tt_ctx* ctx, int64_t* lc, int part = 0) {
  const int d = ctx->d, KL = ctx->plan.KL;
  cudaStream_t s = ctx->stream;
  const bool adaptive = ctx->step_rule == TT_STEP_ADAPTIVE;
  if (part == 2) {
    if (adaptive) {
      enqueue_adaptive_front(ctx, lc);
      return;
    }
    DenseArgs da = dense_args(ctx);
    grp(ctx, 10, true);
    launch_dense_round(ctx->stream, da, lc);
    grp(ctx, 10, false);
    return;
  }
  if (part == 3) {
    enqueue_adaptive_back(ctx, lc);
    return;
  }
  grp(ctx, 4, true);
  launch_weights(s, ctx->h, d, ctx->n_i.data(), ctx->phi_off[d], ctx->eps_rule, ctx->eps_fixed,
                 ctx->step_rule, ctx->phi, ctx->sc, lc);
  if (!ctx->plan.chain)
    launch_psi(s, ctx->phi, ctx->phi_off.data(), KL, d, ctx->n_i.data(), ctx->plan.NL,
               ctx->plan.NR, ctx->psiL, ctx->psiR, ctx->sc, lc);
  grp(ctx, 4, false);
  DenseArgs da = dense_args(ctx);
  // Overlap (table path, cluster A4-A6): the left tables of U and pass B's suffix-order SpMM
  // need only the cores < K_L, which the A5 sweep finishes first, so they run on a second
  // stream beside the rest of A5 and A6 (k_orth_cs split in two launches, identical
  // arithmetic).  Direct (profiling) runs keep the sequential order for the group timers.
  static const bool no_overlap = [] {
    const char* e = getenv("PRGD_NO_OVERLAP");
    return e && e[0] == '1';
  }();
  const bool ovl = !no_overlap && !ctx->profiling && !ctx->plan.chain && orth_cluster_ok(da) &&
                   ctx->obs_set;
  if (ovl && !ctx->ovl) {
    cudaStreamCreateWithFlags(&ctx->ovl, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ctx->ev_ovl[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_ovl[1], cudaEventDisableTiming);
  }
  DenseArgs da1 = da, da2 = da;
  da1.orth_part = 1;
  da2.orth_part = 2;
  da1.orth_split = da2.orth_split = KL;
  grp(ctx, 5, true);
  launch_dense_orth(s, ovl ? da1 : da, lc);
  grp(ctx, 5, false);
  if (ctx->plan.chain) {   // pass B by per-sample chains (A7-A8), segmented contraction (A9)
    grp(ctx, 7, true);
    launch_chain_iface(s, ctx->idx_dev, ctx->m, ctx->ctt, ctx->U, ctx->phi, ctx->g, ctx->ghat, ctx->IL,
                       ctx->IR, ctx->sc, lc);
    grp(ctx, 7, false);
    grp(ctx, 9, true);
    launch_chain_contract(s, ctx->pcs, ctx->ctt, ctx->m, ctx->ghat, ctx->IL, ctx->IR, ctx->Y, ctx->sc, lc);
    grp(ctx, 9, false);
  } else {
  if (!ovl) {
    grp(ctx, 6, true);
    enqueue_tables(ctx, true, lc);
    grp(ctx, 6, false);
  }
  grp(ctx, 7, true);
  {
  SegArgs a{};
  a.plan = &ctx->planL;
  a.mode = kSPMM;
  a.ld = ctx->ldr[KL];
  a.col = ctx->Spre;
  a.g = ctx->g;
  a.coltab = ctx->RT[KL];
  a.rowscale = ctx->psiL;
  a.out = ctx->EL[KL];
  SegArgs b{};
  b.plan = &ctx->planR;
  b.mode = kSPMM;
  b.ld = ctx->ldr[KL];
  b.col = ctx->Psuf;
  b.g = ctx->gsq_q >= 2 ? ctx->stage : ctx->g_suf;
  b.perm = ctx->gsq_q >= 2 ? ctx->sl_q : nullptr;
  b.coltab = ctx->LT[KL];
  b.rowscale = ctx->psiR;
  b.out = ctx->FR[KL];
  if (ovl) {
    // s: rest of A5 + A6 (launched first, highest priority), right tables, pass B prefix;
    // ctx->ovl: left tables, pass B suffix; joined before the backward recursions
    cudaEventRecord(ctx->ev_ovl[0], s);
    launch_dense_orth(s, da2, lc);
    cudaStreamWaitEvent(ctx->ovl, ctx->ev_ovl[0], 0);
    enqueue_tables(ctx, true, lc, 1, ctx->ovl);
    launch_seg(ctx->ovl, b, ctx->sc, lc);
    cudaEventRecord(ctx->ev_ovl[1], ctx->ovl);
    enqueue_tables(ctx, true, lc, 2, s);
    launch_seg(s, a, ctx->sc, lc);
    cudaStreamWaitEvent(s, ctx->ev_ovl[1], 0);
  } else {
    launch_seg(s, a, ctx->sc, lc);
    grp(ctx, 7, false);
    grp(ctx, 8, true);
    launch_seg(s, b, ctx->sc, lc);
  }
  grp(ctx, 8, false);
  }
  grp(ctx, 9, true);
  {
    std::vector<BackwardLevel> BL, BR;
    bool ok = true;
    for (int k = KL - 1; k >= 0; --k) {
      BackwardLevel t{true, ctx->EL[k + 1], ctx->ldr[k + 1], k >= 1 ? ctx->LT[k] : nullptr,
                      ctx->ldr[k], ctx->U + ctx->core_off[k], (int)ctx->r[k], (int)ctx->n[k],
                      (int)ctx->r[k + 1], k >= 1 ? ctx->EL[k] : nullptr, ctx->ldr[k], ctx->NLk[k],
                      ctx->Y + ctx->core_off[k]};
      ok = ok && level_back_ok(t.r0, t.nk, t.r1, t.wrow);
      BL.push_back(t);
    }
    for (int k = KL; k < d; ++k) {
      BackwardLevel t{false, ctx->FR[k], ctx->ldr[k], k + 1 < d ? ctx->RT[k + 1] : nullptr,
                      ctx->ldr[k + 1], ctx->U + ctx->core_off[k], (int)ctx->r[k], (int)ctx->n[k],
                      (int)ctx->r[k + 1], k + 1 < d ? ctx->FR[k + 1] : nullptr, ctx->ldr[k + 1],
                      k + 1 < d ? ctx->NRk[k + 1] : 1, ctx->Y + ctx->core_off[k]};
      ok = ok && level_back_ok(t.r0, t.nk, t.r1, t.wrow);
      BR.push_back(t);
    }
    if (ok) {
      launch_backward_levels(s, BL, BR, ctx->Ypart, ctx->Ypart_cap, ctx->sc, lc);
    } else {
      for (const BackwardLevel& t : BL) {
        if (back_fused_ok(t.r0, t.nk, t.r1)) {
          launch_back_level(s, true, t.X, t.wrow, t.V, t.ldV, t.core, t.r0, t.nk, t.r1, t.O, t.ldO,
                            t.ngroups, t.Y, ctx->Ypart, ctx->Ypart_cap, ctx->sc, lc);
          continue;
        }
        launch_Y(s, true, t.V, t.ldV, t.X, t.wrow, t.ngroups, t.r0, t.nk, t.r1, t.Y, ctx->Ypart,
                 ctx->Ypart_cap, ctx->sc, lc);
        if (t.O)
          launch_E_down(s, t.X, t.wrow, t.core, t.r0, t.nk, t.r1, t.O, t.ldO, t.ngroups, ctx->Ypart,
                        ctx->Ypart_cap, ctx->sc, lc);
      }
      for (const BackwardLevel& t : BR) {
        if (back_fused_ok(t.r0, t.nk, t.r1)) {
          launch_back_level(s, false, t.X, t.wrow, t.V, t.ldV, t.core, t.r0, t.nk, t.r1, t.O,
                            t.ldO, t.ngroups, t.Y, ctx->Ypart, ctx->Ypart_cap, ctx->sc, lc);
          continue;
        }
        launch_Y(s, false, t.V, t.ldV, t.X, t.wrow, t.ngroups, t.r0, t.nk, t.r1, t.Y, ctx->Ypart,
                 ctx->Ypart_cap, ctx->sc, lc);
        if (t.O)
          launch_F_up(s, t.X, t.wrow, t.core, t.r0, t.nk, t.r1, t.O, t.ldO, t.ngroups, ctx->Ypart,
                      ctx->Ypart_cap, ctx->sc, lc);
      }
    }
  }
  grp(ctx, 9, false);
  }   // table path
  if (part == 1) return;
  if (adaptive) {
    enqueue_adaptive_front(ctx, lc);
    enqueue_adaptive_back(ctx, lc);
    return;
  }
  grp(ctx, 10, true);
  launch_dense_round(s, da, lc);
  grp(ctx, 10, false);
}

// Run a piece either as a captured graph (cached) or directly (profiling).
// Pieces: 0 evaluate (+ sum g^2), 1 update, 2 evaluate without sum g^2, 3 update up to Y,
// 4 rounding.  Each runs as a captured CUDA graph (cached), or directly when profiling.
int run_piece(tt_ctx* ctx, int piece) {
  cudaGraphExec_t* slots[6] = {&ctx->gA, &ctx->gB, &ctx->gA1, &ctx->gB1, &ctx->gB2, &ctx->gB3};
  int64_t* counts[6] = {&ctx->nA, &ctx->nB, &ctx->nA1, &ctx->nB1, &ctx->nB2, &ctx->nB3};
  cudaGraphExec_t* ge = slots[piece];
  int64_t* nl = counts[piece];
  auto enqueue = [&](int64_t* lc) {
    switch (piece) {
      case 0: enqueue_evaluate(ctx, lc, true); break;
      case 1: enqueue_update(ctx, lc, 0); break;
      case 2: enqueue_evaluate(ctx, lc, false); break;
      case 3: enqueue_update(ctx, lc, 1); break;
      case 4: enqueue_update(ctx, lc, 2); break;
      default: enqueue_update(ctx, lc, 3); break;
    }
  };
  if (ctx->profiling) {
    int64_t lc = 0;
    enqueue(&lc);
    ctx->launches += lc;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    return TT_OK;
  }
  if (!*ge) {
    // First use: enqueue the piece directly (the GPU starts on it at once), then capture and
    // instantiate its graph on the host while the GPU runs it; later calls launch the graph.
    {
      int64_t lc = 0;
      enqueue(&lc);
      ctx->launches += lc;
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
    }
    // capture on a private stream (the launch stream may be shared with other contexts /
    // threads), launch on ctx->stream
    if (!ctx->cap) CK(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
    cudaGraph_t graph;
    int64_t lc = 0;
    cudaStream_t launch_stream = ctx->stream;
    ctx->stream = ctx->cap;
    ctx->capturing = true;
    cudaError_t e = cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      enqueue(&lc);
      e = cudaStreamEndCapture(ctx->cap, &graph);
    }
    ctx->capturing = false;
    ctx->stream = launch_stream;
    if (e != cudaSuccess) return cuda_fail(ctx, e, "graph capture");
    e = cudaGraphInstantiate(ge, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "graph instantiate");
    *nl = lc;
    return TT_OK;
  }
  CK(cudaGraphLaunch(*ge, ctx->stream));
  ctx->launches += *nl;
  return TT_OK;
}

// Evaluate the current iterate: tables + pass A + marginals; in sharded mode the per-rank
// marginals h (sum n_k doubles: every h_{k,j} is a sum over samples) are all-reduced before
// sum g^2 and the weights use them (exchange 1).
int run_evaluate(tt_ctx* ctx) {
  int rc;
  if (!ctx->allreduce) return run_piece(ctx, 0);
  if ((rc = run_piece(ctx, 2))) return rc;
  ctx->allreduce(ctx->h, ctx->phi_off[ctx->d], (void*)ctx->stream, ctx->ar_user);
  int64_t lc = 0;
  launch_gather_sq_sum(ctx->stream, ctx->h, ctx->n_i[0], ctx->sc, &lc);
  ctx->launches += lc;
  return TT_OK;
}

// Update: in sharded mode the contractions Y (sum_k r_k n_k r_{k+1} doubles, sums over
// samples) are all-reduced before the replicated projection and rounding (exchange 2).
int run_update(tt_ctx* ctx) {
  int rc;
  if (!ctx->allreduce) return run_piece(ctx, 1);
  if ((rc = run_piece(ctx, 3))) return rc;
  ctx->allreduce(ctx->Y, ctx->core_off[ctx->d], (void*)ctx->stream, ctx->ar_user);
  if ((rc = run_piece(ctx, 4))) return rc;
  if (ctx->step_rule != TT_STEP_ADAPTIVE) return TT_OK;
  ctx->allreduce(&ctx->sc->adapt_den, 1, (void*)ctx->stream, ctx->ar_user);   // sum over ranks
  return run_piece(ctx, 5);
}

int read_scalars(tt_ctx* ctx) {
  CK(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->sc_host->err) {
    int bits = ctx->sc_host->err;
    int zero = 0;
    CK(cudaMemcpyAsync(&ctx->sc->err, &zero, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::string what;
    if (bits & kErrNaN) what += " non-finite values;";
    if (bits & kErrChol) what += " Cholesky breakdown of a right Gram P_k;";
    if (bits & kErrSVD) what += " Jacobi SVD did not converge;";
    return fail(ctx, TT_ERR_NUMERIC, "numeric fault:" + what);
  }
  return TT_OK;
}

int collect_profile(tt_ctx* ctx, int g0, int g1) {
  if (!ctx->profiling || !ctx->ev_ready) return TT_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  for (int gi = g0; gi <= g1; ++gi) {
    float ms = 0.f;
    if (cudaEventQuery(ctx->ev[2 * gi + 1]) == cudaSuccess &&
        cudaEventElapsedTime(&ms, ctx->ev[2 * gi], ctx->ev[2 * gi + 1]) == cudaSuccess)
      ctx->prof_ms[gi] += ms;
  }
  cudaGetLastError();
  return TT_OK;
}

// Work plan of one pass side from the bucket offsets on the device (plan.cu): virtual rows
// (rows with > kSplit samples split into partial slots), split-row table, warp runs.  Two
// small device-to-host reads (totals, per-gather-block ranges); no per-row host work.
int make_plan(tt_ctx* ctx, const int64_t* offs_dev, int64_t nrow, int nblk, int ld, int64_t m,
              SegPlan* pl) {
  cudaStream_t s = ctx->stream;
  const int64_t nr = nrow * nblk;
  std::vector<void*> tmp;
  auto cleanup = [&]() { dfree_all(ctx, tmp); };
  int *nv = nullptr, *sp = nullptr, *np = nullptr, *cost = nullptr, *flag = nullptr;
  int64_t *vbase = nullptr, *sbase = nullptr, *pbase = nullptr, *C = nullptr, *wid = nullptr,
          *blk = nullptr;
  long long* bsum = nullptr;
  const int64_t vmax = nr + m / kSplit + 1;
  if (!(A(ctx, &nv, nr, tmp) && A(ctx, &sp, nr, tmp) && A(ctx, &np, nr, tmp) && A(ctx, &vbase, nr + 1, tmp) &&
        A(ctx, &sbase, nr + 1, tmp) && A(ctx, &pbase, nr + 1, tmp) &&
        A(ctx, &bsum, plan_scan_scratch(std::max(nr, vmax)), tmp) && A(ctx, &blk, 3 * (nblk + 1), tmp))) {
    cleanup();
    return fail(ctx, TT_ERR_OOM, "device allocation failed (plan)");
  }
  int64_t lc = 0;
  launch_plan_rows(s, offs_dev, nr, kSplit, nv, sp, np, vbase, sbase, pbase, bsum, &lc);
  int64_t tot[3] = {0, 0, 0};
  CK(cudaMemcpyAsync(&tot[0], vbase + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&tot[1], sbase + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&tot[2], pbase + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *pl = SegPlan();
  pl->nrows = nr;
  pl->nrow_real = nrow;
  pl->nblk = nblk;
  pl->nvrows = tot[0];
  pl->nsplit = tot[1];
  pl->npart = tot[2];
  const int64_t nvr = pl->nvrows;
  auto& OL = ctx->obs_allocs;
  if (!(A(ctx, &pl->vrow, nvr, OL) && A(ctx, &pl->warp_vbegin, nvr + 1, OL) &&
        A(ctx, &pl->split_row, pl->nsplit, OL) && A(ctx, &pl->split_first, pl->nsplit + 1, OL) &&
        A(ctx, &pl->part, std::max<int64_t>(pl->npart, 1) * ld, OL) && A(ctx, &cost, nvr, tmp) &&
        A(ctx, &C, nvr + 1, tmp) && A(ctx, &flag, nvr, tmp) && A(ctx, &wid, nvr + 1, tmp))) {
    cleanup();
    return fail(ctx, TT_ERR_OOM, "device allocation failed (plan)");
  }
  launch_plan_fill(s, offs_dev, nr, nrow, nblk, kSplit, vbase, sbase, pbase, nvr, pl->vrow,
                   pl->split_row, pl->split_first,
                   kVrowCost, kWarpCost, cost, C, flag, wid, bsum, blk, &lc);
  launch_plan_warps(s, flag, wid, nvr, pl->warp_vbegin, &lc);
  std::vector<int64_t> hb(3 * (nblk + 1));
  CK(cudaMemcpyAsync(hb.data(), blk, hb.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  ctx->launches += lc;
  cleanup();
  pl->blk_split.assign(hb.begin() + (nblk + 1), hb.begin() + 2 * (nblk + 1));
  pl->blk_warp.assign(hb.begin() + 2 * (nblk + 1), hb.end());
  pl->nwarps = pl->blk_warp[nblk];
  return TT_OK;
}

void apply_plan(tt_ctx* ctx, const Plan& pl) {
  ctx->plan = pl;
  ctx->NLk.assign(pl.KL + 1, 1);
  ctx->NRk.assign(ctx->d + 1, 1);
  if (pl.chain) return;
  for (int k = 1; k <= pl.KL; ++k) ctx->NLk[k] = ctx->NLk[k - 1] * ctx->n[k - 1];
  for (int k = ctx->d - 1; k >= pl.KL; --k) ctx->NRk[k] = ctx->NRk[k + 1] * ctx->n[k];
}

// Observations on the chain path: the multi-indices stay in the ABI layout,
// the values in the original order; A0 builds the per-mode buckets (stable radix sort of the
// sample ids by x_k, k = 0..d-1) and cuts them into pieces of <= P samples.
// Host multi-indices -> idx_dev (int32): copied as they are, or (ib = 1, tt_set_observations_u8)
// uploaded as bytes into `stage8` and widened on the device.
cudaError_t upload_idx(cudaStream_t s, const void* h_idx, int ib, int64_t count, uint8_t* stage8,
                       int32_t* idx_dev, int64_t* lc) {
  if (ib == 4)
    return cudaMemcpyAsync(idx_dev, h_idx, (size_t)count * sizeof(int32_t), cudaMemcpyHostToDevice, s);
  cudaError_t e = cudaMemcpyAsync(stage8, h_idx, (size_t)count, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  launch_widen_u8(s, stage8, count, idx_dev, lc);
  return cudaSuccess;
}

int set_obs_chain(tt_ctx* ctx, const void* h_idx, int ib, const double* h_vals, int64_t m) {
  const int d = ctx->d;
  auto& OL = ctx->obs_allocs;
  std::vector<void*> tmp;
  auto cleanup = [&]() { dfree_all(ctx, tmp); };
  ChainPieces& pc = ctx->pcs;
  pc = ChainPieces();
  int rmax = 1;
  for (int k = 0; k <= d; ++k) rmax = std::max<int>(rmax, (int)ctx->r[k]);
  pc.nbuckets = ctx->phi_off[d];
  pc.stride = 1;
  for (int k = 0; k < d; ++k) pc.stride = std::max<int>(pc.stride, (int)(ctx->r[k] * ctx->r[k + 1]));
  pc.P = chain_piece_size(m, d, rmax);
  int64_t iface = 0;                                  // interface doubles, m r_k for k = 1..d-1
  ctx->ctt.m = m;
  ctx->ctt.il_off[0] = ctx->ctt.il_off[1] = 0;
  for (int k = 1; k < d; ++k) {
    ctx->ctt.il_off[k] = iface;
    iface += m * ctx->r[k];
  }
  ctx->ctt.il_off[d] = iface;
  ctx->dtt.m = m;
  uint64_t *keys = nullptr, *ktmp = nullptr;
  uint32_t *vals = nullptr, *vtmp = nullptr;
  int* hist = nullptr;
  int* np = nullptr;
  long long* bsum = nullptr;
  const int64_t hl = radix_hist_len(m);
  const int64_t noffs = pc.nbuckets + d;
  uint8_t* stage8 = nullptr;
  bool ok = (ib == 4 || A(ctx, &stage8, m * d + 16, tmp)) &&
            A(ctx, &ctx->idx_dev, m * d, OL) && A(ctx, &ctx->yobs, m, OL) && A(ctx, &ctx->g, m, OL) &&
            A(ctx, &ctx->ghat, m, OL) && A(ctx, &ctx->IL, iface, OL) && A(ctx, &ctx->IR, iface, OL) &&
            A(ctx, &pc.perm, (int64_t)d * m, OL) && A(ctx, &pc.offs, noffs, OL) &&
            A(ctx, &pc.pbase, pc.nbuckets + 1, OL) && (!adapt_by_chains(ctx) || A(ctx, &ctx->dval, m, OL)) &&
            A(ctx, &keys, m, tmp) && A(ctx, &ktmp, m, tmp) && A(ctx, &vals, m, tmp) &&
            A(ctx, &vtmp, m, tmp) && A(ctx, &hist, hl, tmp) && A(ctx, &np, pc.nbuckets, tmp) &&
            A(ctx, &bsum, plan_scan_scratch(pc.nbuckets), tmp);
  if (!ok) {
    cleanup();
    dfree_all(ctx, OL);
    return fail(ctx, TT_ERR_OOM, "device allocation failed (observations, chain path)");
  }
  cudaStream_t s = ctx->stream;
  int64_t lc = 0;
  CK(cudaMemsetAsync(&ctx->sc->index_err, 0, sizeof(int), s));
  if (m > 0) {
    CK(upload_idx(s, h_idx, ib, m * d, stage8, ctx->idx_dev, &lc));
    CK(cudaMemcpyAsync(ctx->yobs, h_vals, (size_t)m * sizeof(double), cudaMemcpyHostToDevice, s));
    for (int k = 0; k < d; ++k) {
      int bits = 1;
      while (((int64_t)1 << bits) < ctx->n[k]) ++bits;
      launch_mode_keys(s, ctx->idx_dev, m, d, k, (int)ctx->n[k], keys, vals, &ctx->sc->index_err, &lc);
      uint64_t* ko;
      uint32_t* vo;
      radix_sort_pairs(s, keys, vals, ktmp, vtmp, m, bits, hist, hl, &ko, &vo, &lc);
      launch_mode_after_sort(s, ko, vo, m, ctx->n[k], pc.perm + (int64_t)k * m,
                             pc.offs + ctx->phi_off[k] + k, &lc);
    }
  } else {
    CK(cudaMemsetAsync(pc.offs, 0, noffs * sizeof(int64_t), s));
  }
  launch_piece_count(s, pc.offs, ctx->ctt, pc.nbuckets, pc.P, np, &lc);
  launch_scan_i32(s, np, pc.nbuckets, pc.pbase, bsum, &lc);
  CK(cudaMemcpyAsync(&pc.npieces, pc.pbase + pc.nbuckets, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (ctx->sc_host->index_err) {
    cleanup();
    dfree_all(ctx, OL);
    return fail(ctx, TT_ERR_INDEX, "an observed index is outside [0, n_k)");
  }
  if (!A(ctx, &pc.pieces, std::max<int64_t>(pc.npieces, 1), OL) ||
      !A(ctx, &pc.part, std::max<int64_t>(pc.npieces, 1) * pc.stride, OL)) {
    cleanup();
    dfree_all(ctx, OL);
    return fail(ctx, TT_ERR_OOM, "device allocation failed (bucket pieces)");
  }
  launch_piece_fill(s, pc.offs, pc.pbase, pc.nbuckets, ctx->ctt, pc.P, pc.pieces, &lc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(ctx, e, "bucketing kernels (chain path)");
  }
  CK(cudaStreamSynchronize(s));
  cleanup();
  ctx->launches += lc;
  ctx->m = m;
  double nstar = 1.0;
  for (int k = 0; k < d; ++k) nstar *= (double)ctx->n[k];
  ctx->p = (double)(ctx->allreduce ? ctx->m_global : m) / nstar;
  CK(cudaMemcpyAsync(&ctx->sc->p, &ctx->p, sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  ctx->obs_set = true;
  return TT_OK;
}

bool all_cores_set(tt_ctx* ctx) {
  for (char c : ctx->core_set)
    if (!c) return false;
  return true;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

int tt_plan(int d, const int64_t* n, const int64_t* r, int* K_L, int64_t* N_L, int64_t* N_R) {
  Plan pl;
  std::string msg;
  int rc = validate_and_plan(d, n, r, &pl, &msg);
  if (rc != TT_OK) return rc;
  if (K_L) *K_L = pl.KL;
  if (N_L) *N_L = pl.NL;
  if (N_R) *N_R = pl.NR;
  return TT_OK;
}

int tt_set_path(tt_ctx* ctx, int path) {
  if (!ctx) return TT_ERR_ARG;
  if (path < TT_PATH_AUTO || path > TT_PATH_CHAINS) return fail(ctx, TT_ERR_ARG, "unknown path");
  if (ctx->base_ready || ctx->obs_set)
    return fail(ctx, TT_ERR_STATE, "tt_set_path must precede any core or observation");
  Plan pl;
  std::string msg;
  int rc = validate_and_plan(ctx->d, ctx->n.data(), ctx->r.data(), &pl, &msg, path);
  if (rc != TT_OK) return fail(ctx, rc, msg);
  ctx->path_req = path;
  apply_plan(ctx, pl);
  return TT_OK;
}

int tt_get_path(tt_ctx* ctx, int* path) {
  if (!ctx || !path) return TT_ERR_ARG;
  *path = ctx->plan.chain ? TT_PATH_CHAINS : TT_PATH_TABLES;
  return TT_OK;
}

int tt_set_allreduce(tt_ctx* ctx, tt_allreduce_fn fn, void* user, int64_t m_global) {
  if (!ctx) return TT_ERR_ARG;
  if (fn && m_global < 0) return fail(ctx, TT_ERR_ARG, "m_global must be >= 0");
  if (ctx->obs_set) return fail(ctx, TT_ERR_STATE, "tt_set_allreduce must precede tt_set_observations");
  ctx->allreduce = fn;
  ctx->ar_user = user;
  ctx->m_global = fn ? m_global : -1;
  drop_graphs(ctx);
  ctx->evalValid = false;
  return TT_OK;
}

int tt_create(int d, const int64_t* n, const int64_t* r, tt_ctx** out) {
  if (!out) return TT_ERR_ARG;
  *out = nullptr;
  Plan pl;
  std::string msg;
  int rc = validate_and_plan(d, n, r, &pl, &msg);
  if (rc != TT_OK) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return TT_ERR_CUDA;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  int major = 0, minor = 0;   // (cudaGetDeviceProperties costs milliseconds per call)
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
      major != 10 || minor != 0)
    return TT_ERR_CUDA;
  tt_ctx* ctx = new tt_ctx();
  ctx->d = d;
  ctx->n.assign(n, n + d);
  ctx->r.assign(r, r + d + 1);
  ctx->n_i.resize(d);
  for (int k = 0; k < d; ++k) ctx->n_i[k] = (int)n[k];
  ctx->ldr.resize(d + 1);
  for (int k = 0; k <= d; ++k) ctx->ldr[k] = pad_rank((int)r[k]);
  apply_plan(ctx, pl);
  ctx->core_set.assign(d, 0);
  if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return TT_ERR_CUDA;
  }
  ctx->stream = ctx->own_stream;
  *out = ctx;
  return TT_OK;
}

int tt_destroy(tt_ctx* ctx) {
  if (!ctx) return TT_OK;
  cudaStreamSynchronize(ctx->stream);
  drop_graphs(ctx);
  dfree_all(ctx, ctx->obs_allocs);
  dfree_all(ctx, ctx->base_allocs);
  if (ctx->sc_host) pinned_scalars_put(ctx->sc_host);
  if (ctx->ev_ready)
    for (auto& e : ctx->ev) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->cap) cudaStreamDestroy(ctx->cap);
  for (cudaEvent_t e : ctx->ev_side)
    if (e) cudaEventDestroy(e);
  if (ctx->ovl) cudaStreamDestroy(ctx->ovl);
  for (cudaEvent_t e : ctx->ev_ovl)
    if (e) cudaEventDestroy(e);
  delete ctx;
  return TT_OK;
}

int tt_set_stream(tt_ctx* ctx, void* stream) {
  if (!ctx) return TT_ERR_ARG;
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  drop_graphs(ctx);
  return TT_OK;
}

int tt_set_allocator(tt_ctx* ctx, void* (*alloc)(size_t, void*), void (*release)(void*, void*),
                     void* user) {
  if (!ctx) return TT_ERR_ARG;
  if (ctx->base_ready || ctx->obs_set)
    return fail(ctx, TT_ERR_STATE, "allocator must be installed before any data is set");
  if ((alloc == nullptr) != (release == nullptr))
    return fail(ctx, TT_ERR_ARG, "alloc and release must both be set or both NULL");
  ctx->halloc = alloc;
  ctx->hfree = release;
  ctx->huser = user;
  return TT_OK;
}

int tt_set_metric(tt_ctx* ctx, int eps_rule, double eps, int step_rule) {
  if (!ctx) return TT_ERR_ARG;
  if (eps_rule < TT_EPS_VEE || eps_rule > TT_EPS_NONE || step_rule < TT_STEP_THEORY ||
      step_rule > TT_STEP_ADAPTIVE)
    return fail(ctx, TT_ERR_ARG, "unknown eps or step rule");
  if (eps_rule == TT_EPS_FIXED && !(eps > 0.0 && std::isfinite(eps)))
    return fail(ctx, TT_ERR_ARG, "TT_EPS_FIXED needs a finite eps > 0");
  if (step_rule == TT_STEP_ADAPTIVE) {
    int rc = ensure_adaptive(ctx);
    if (rc) return rc;
  }
  ctx->eps_rule = eps_rule;
  ctx->eps_fixed = eps;
  ctx->step_rule = step_rule;
  drop_graphs(ctx);   // rules are baked into the captured update graph
  return TT_OK;
}

int tt_set_retraction(tt_ctx* ctx, int kind) {
  if (!ctx) return TT_ERR_ARG;
  if (kind != TT_RETRACT_PLAIN && kind != TT_RETRACT_WEIGHTED)
    return fail(ctx, TT_ERR_ARG, "unknown retraction");
  ctx->retraction = kind;
  drop_graphs(ctx);   // baked into the captured update graph
  return TT_OK;
}

int tt_set_core(tt_ctx* ctx, int k, const double* h_core) {
  if (!ctx) return TT_ERR_ARG;
  if (k < 0 || k >= ctx->d || !h_core) return fail(ctx, TT_ERR_ARG, "bad core index or NULL");
  int rc = ensure_base(ctx);
  if (rc) return rc;
  const int64_t sz = ctx->core_off[k + 1] - ctx->core_off[k];
  CK(cudaMemcpyAsync(ctx->C + ctx->core_off[k], h_core, sz * sizeof(double), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->core_set[k] = 1;
  ctx->evalValid = false;
  ctx->tablesC = false;
  return TT_OK;
}

int tt_get_core(tt_ctx* ctx, int k, double* h_core_out) {
  if (!ctx) return TT_ERR_ARG;
  if (k < 0 || k >= ctx->d || !h_core_out) return fail(ctx, TT_ERR_ARG, "bad core index or NULL");
  int rc = ensure_base(ctx);
  if (rc) return rc;
  const int64_t sz = ctx->core_off[k + 1] - ctx->core_off[k];
  CK(cudaMemcpyAsync(h_core_out, ctx->C + ctx->core_off[k], sz * sizeof(double),
                     cudaMemcpyDeviceToHost, ctx->stream));
  return read_scalars(ctx);
}

static int set_observations_impl(tt_ctx* ctx, const void* h_idx, int ib, const double* h_vals, int64_t m);

int tt_set_observations(tt_ctx* ctx, const int32_t* h_idx, const double* h_vals, int64_t m) {
  if (!ctx) return TT_ERR_ARG;
  return set_observations_impl(ctx, h_idx, 4, h_vals, m);
}

int tt_set_observations_u8(tt_ctx* ctx, const uint8_t* h_idx, const double* h_vals, int64_t m) {
  if (!ctx) return TT_ERR_ARG;
  for (int k = 0; k < ctx->d; ++k)
    if (ctx->n[k] > 256) return fail(ctx, TT_ERR_ARG, "byte indices need every n_k <= 256");
  return set_observations_impl(ctx, h_idx, 1, h_vals, m);
}

static int set_observations_impl(tt_ctx* ctx, const void* h_idx, int ib, const double* h_vals, int64_t m) {
  PhaseTimer ptm(ctx->stream, "set_observations");
  if (m < 0 || m >= ((int64_t)1 << 31)) return fail(ctx, TT_ERR_ARG, "m must be in [0, 2^31)");
  if (m > 0 && (!h_idx || !h_vals)) return fail(ctx, TT_ERR_ARG, "NULL idx or vals");
  int rc = ensure_base(ctx);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  drop_graphs(ctx);
  dfree_all(ctx, ctx->obs_allocs);
  ctx->obs_set = false;
  ctx->evalValid = false;
  ctx->m = 0;
  ctx->idx_dev = nullptr;
  if (ctx->plan.chain) return set_obs_chain(ctx, h_idx, ib, h_vals, m);
  const int d = ctx->d, KL = ctx->plan.KL;
  const int64_t NL = ctx->plan.NL, NR = ctx->plan.NR;
  const int64_t NLv = NL, NRv = NR;
  auto& OL = ctx->obs_allocs;
  std::vector<void*> tmp;
  int32_t* idx_dev = nullptr;
  double* y_orig = nullptr;
  uint64_t *kpre = nullptr, *ksuf = nullptr, *ktmp = nullptr;
  uint32_t *vals = nullptr, *vals2 = nullptr, *vtmp = nullptr;
  int32_t* inv = nullptr;
  int* hist = nullptr;
  const int64_t hl = radix_hist_len(m);
  // pass A suffix by slices of g when g exceeds one slice (~48 MB, L2-resident gathers);
  // PRGD_GSQ_SLICES=Q forces Q slices (1: the row-plan gather), read per call (tests)
  {
    const char* e = getenv("PRGD_GSQ_SLICES");
    int64_t q = (m * 8 + kGsqSliceBytes - 1) / kGsqSliceBytes;
    if (e && *e) q = std::atoll(e);
    q = std::max<int64_t>(1, std::min<int64_t>(q, 256));
    if (m < 64 * q) q = 1;
    ctx->gsq_q = q >= 2 ? (int)q : 0;
    ctx->gsq_slen = ctx->gsq_q ? (m + q - 1) / q : 0;
  }
  const bool sliced = ctx->gsq_q >= 2;
  uint8_t* stage8 = nullptr;
  bool ok = (ib == 4 || A(ctx, &stage8, m * d + 16, tmp)) &&
            A(ctx, &idx_dev, m * d, OL) && A(ctx, &y_orig, m, tmp) && A(ctx, &kpre, m, tmp) &&
            A(ctx, &ksuf, m, tmp) && A(ctx, &ktmp, m, tmp) && A(ctx, &vals, m, tmp) &&
            A(ctx, &vals2, m, tmp) && A(ctx, &vtmp, m, tmp) && A(ctx, &inv, m, tmp) &&
            A(ctx, &hist, hl, tmp) && A(ctx, &ctx->Spre, m + 8, OL) && A(ctx, &ctx->ypre, m + 8, OL) &&
            A(ctx, &ctx->g, m + 8, OL) && A(ctx, &ctx->sid_pre, m, OL) && A(ctx, &ctx->pos_suf, m, OL) &&
            A(ctx, &ctx->Psuf, m + 8, OL) && A(ctx, &ctx->sid_suf, m, OL) &&
            (sliced || A(ctx, &ctx->g_suf, m + 8, OL)) && A(ctx, &ctx->pre2suf, m, OL) &&
            (!sliced || (A(ctx, &ctx->sl_pos, m, OL) && A(ctx, &ctx->sl_row, m, OL) &&
                         A(ctx, &ctx->sl_q, m, OL) && A(ctx, &ctx->stage, m + 8, OL) &&
                         A(ctx, &ctx->HRq, ctx->gsq_q * NRv, OL))) &&
            A(ctx, &ctx->offsL, NLv + 1 + 40, OL) && A(ctx, &ctx->offsR, NRv + 1 + 40, OL) &&
            A(ctx, &ctx->Ppre, m + 8, OL) &&
            A(ctx, reinterpret_cast<char**>(&ctx->frec), flat_rec_bytes(m), OL) &&
            (!adapt_by_chains(ctx) || A(ctx, &ctx->dval, m, OL));
  ctx->idx_dev = idx_dev;
  auto cleanup = [&]() { dfree_all(ctx, tmp); };
  if (!ok) {
    cleanup();
    dfree_all(ctx, OL);
    return fail(ctx, TT_ERR_OOM, "device allocation failed (observations)");
  }
  ptm.mark("alloc");
  int bitsP = 1, bitsS = 1, bitsVP = 1, bitsVS = 1;
  while (((int64_t)1 << bitsP) < NL) ++bitsP;
  while (((int64_t)1 << bitsS) < NR) ++bitsS;
  while (((int64_t)1 << bitsVP) < NLv) ++bitsVP;
  while (((int64_t)1 << bitsVS) < NRv) ++bitsVS;
  cudaStream_t s = ctx->stream;
  int64_t lc = 0;
  if (m > 0) {
    if (!ctx->side) {
      CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ctx->ev_side[0], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_side[1], cudaEventDisableTiming));
    }
    // idx first on the main stream; the values follow on the side stream (the link carries one
    // copy at a time) while the keys are built and sorted; after_sort_pre waits for them.
    CK(upload_idx(s, h_idx, ib, m * d, stage8, idx_dev, &lc));
    CK(cudaEventRecord(ctx->ev_side[0], s));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_side[0], 0));
    CK(cudaMemcpyAsync(y_orig, h_vals, (size_t)m * sizeof(double), cudaMemcpyHostToDevice, ctx->side));
    CK(cudaEventRecord(ctx->ev_side[1], ctx->side));
    CK(cudaMemsetAsync(&ctx->sc->index_err, 0, sizeof(int), s));
    launch_make_keys(s, idx_dev, m, d, ctx->n_dev, KL, bitsP, bitsS, kpre, ksuf, vals, ctx->sc, &lc);
    CK(cudaMemcpyAsync(vals2, vals, (size_t)m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ptm.mark("h2d+keys");
    if (ctx->sc_host->index_err) {
      cudaStreamSynchronize(ctx->side);   // the value upload still targets y_orig
      cleanup();
      dfree_all(ctx, OL);
      return fail(ctx, TT_ERR_INDEX, "an observed index is outside [0, n_k)");
    }
    // Both sorts run while the values are still on the link: the suffix sort takes as its
    // scratch the pair the prefix sort's result does not occupy, and only the two
    // after-sort kernels (which read y / the prefix inverse) wait for the value upload.
    uint64_t *ko, *ko2;
    uint32_t *vo, *vo2;
    radix_sort_pairs(s, kpre, vals, ktmp, vtmp, m, bitsVP + bitsS, hist, hl, &ko, &vo, &lc);
    ptm.mark("sort_pre");
    radix_sort_pairs(s, ksuf, vals2, ko == ktmp ? kpre : ktmp, vo == vtmp ? vals : vtmp, m,
                     bitsVS + bitsP, hist, hl, &ko2, &vo2, &lc);
    ptm.mark("sort_suf");
    CK(cudaStreamWaitEvent(s, ctx->ev_side[1], 0));
    launch_after_sort_pre(s, ko, vo, m, bitsS, NLv, y_orig, ctx->Spre, ctx->ypre, ctx->sid_pre, inv,
                          ctx->offsL, ctx->Ppre, &lc);
    launch_after_sort_suf(s, ko2, vo2, m, bitsP, NRv, inv, ctx->pos_suf, ctx->Psuf, ctx->sid_suf,
                          ctx->pre2suf, ctx->offsR, &lc);
    ptm.mark("after_sorts");
    if (sliced) {   // scratch: the key buffers other than ko2, all value buffers
      uint64_t* kf[2];
      int nf = 0;
      for (uint64_t* kb : {kpre, ktmp, ksuf})
        if (kb != ko2 && nf < 2) kf[nf++] = kb;
      launch_slice_setup(s, ctx->pos_suf, ko2, bitsP, m, ctx->gsq_slen, ctx->gsq_q, kf[0], vals, kf[1],
                         vtmp, hist, hl, ctx->sl_pos, ctx->sl_row, ctx->sl_q, &lc);
      ptm.mark("slices");
    }
  } else {
    CK(cudaMemsetAsync(ctx->offsL, 0, (NLv + 1) * sizeof(int64_t), s));
    CK(cudaMemsetAsync(ctx->offsR, 0, (NRv + 1) * sizeof(int64_t), s));
  }
  ctx->launches += lc;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(ctx, e, "bucketing kernels");
  }
  cleanup();
  ptm.mark("free_tmp");
  if ((rc = make_plan(ctx, ctx->offsL, NL, 1, ctx->ldr[KL], m, &ctx->planL))) return rc;
  ptm.mark("plan_L");
  if ((rc = make_plan(ctx, ctx->offsR, NR, 1, ctx->ldr[KL], m, &ctx->planR))) return rc;
  ptm.mark("plan_R");
  ctx->m = m;
  double nstar = 1.0;
  for (int k = 0; k < d; ++k) nstar *= (double)ctx->n[k];
  ctx->p = (double)(ctx->allreduce ? ctx->m_global : m) / nstar;
  CK(cudaMemcpyAsync(&ctx->sc->p, &ctx->p, sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  ctx->obs_set = true;
  return TT_OK;
}

int tt_spectral_init(tt_ctx* ctx) {
  if (!ctx) return TT_ERR_ARG;
  if (!ctx->obs_set || ctx->m <= 0) return fail(ctx, TT_ERR_STATE, "spectral init needs a nonempty Omega");
  if (ctx->allreduce) return fail(ctx, TT_ERR_STATE, "spectral init is single-rank (sharded mode set)");
  if (ctx->plan.chain) return fail(ctx, TT_ERR_STATE, "spectral init needs the table path (TT_PATH_TABLES)");
  const int d = ctx->d;
  long double nstar = 1;
  int Wmax = 1, cs = 1;
  for (int k = 0; k < d; ++k) {
    nstar *= (long double)ctx->n[k];
    Wmax = std::max<int>(Wmax, (int)(ctx->r[k] * ctx->n[k]));
    cs = std::max<int>(cs, (int)ctx->r[k + 1]);
  }
  if (nstar >= (long double)(1ull << 62)) return fail(ctx, TT_ERR_ARG, "spectral init needs prod(n) < 2^62");
  // step k < d-1 takes the left Gram (W = r_{k-1} n_k <= 1024 and the Gram kernel's shared
  // memory bound) or the right Gram (W > 1024; at most 1024 nonzero columns, checked at run time)
  int64_t Wuse = 1, Wr = 0;
  for (int k = 0; k + 1 < d; ++k) {
    const int64_t W = ctx->r[k] * ctx->n[k];
    if (W > kSpRightMax) {
      Wr = std::max<int64_t>(Wr, W);
      continue;
    }
    Wuse = std::max<int64_t>(Wuse, W);
    if ((ctx->r[k] <= 8 ? 64 : (ctx->r[k] <= 16 ? 256 : 1024)) * ctx->n[k] > 25 * 1024)
      return fail(ctx, TT_ERR_ARG, "spectral init needs pad(r_{k-1})^2 n_k <= 25600 where r_{k-1} n_k <= 1024");
  }
  if (Wr > ((int64_t)1 << 20)) return fail(ctx, TT_ERR_ARG, "spectral init needs r_{k-1} n_k <= 2^20");
  int rc = ensure_base(ctx);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  const int64_t m = ctx->m;
  SpectralArgs a{};
  a.d = d;
  a.KL = ctx->plan.KL;
  for (int k = 0; k < d; ++k) a.n[k] = (int)ctx->n[k];
  for (int k = 0; k <= d; ++k) {
    a.r[k] = (int)ctx->r[k];
    a.core_off[k] = ctx->core_off[k];
  }
  a.m = m;
  a.NL = ctx->plan.NL;
  a.nrows = ctx->plan.NL;
  a.p = ctx->p;
  a.offsL = ctx->offsL;
  a.Spre = ctx->Spre;
  a.y = ctx->ypre;
  a.C = ctx->C;
  a.cs = cs;
  a.hist_len = radix_hist_len(m);
  a.gram_parts_cap = std::max<int64_t>((int64_t)1 << 28, Wuse * Wuse);
  std::vector<void*> tmp;
  bool ok = A(ctx, &a.Ppos, m, tmp) && A(ctx, &a.z, m, tmp) && A(ctx, &a.chain, m * cs, tmp) &&
            A(ctx, &a.w, m * cs, tmp) && A(ctx, &a.keys, m, tmp) && A(ctx, &a.ktmp, m, tmp) &&
            A(ctx, &a.vals, m, tmp) && A(ctx, &a.vtmp, m, tmp) && A(ctx, &a.hist, a.hist_len, tmp) &&
            A(ctx, &a.flag, m, tmp) && A(ctx, &a.rx, m, tmp) && A(ctx, &a.gflag, m, tmp) &&
            A(ctx, &a.ridx, m + 1, tmp) && A(ctx, &a.rstart, m + 1, tmp) && A(ctx, &a.gidx, m + 1, tmp) &&
            A(ctx, &a.gstart, m + 1, tmp) && A(ctx, &a.rgroup, m + 1, tmp) && A(ctx, &a.byx, m + 1, tmp) &&
            A(ctx, &a.xoff, Wmax + 2, tmp) && A(ctx, &a.bsum, plan_scan_scratch(m + 1), tmp) &&
            A(ctx, &a.lflag, m, tmp) && A(ctx, &a.lnch, m, tmp) && A(ctx, &a.lidx, m + 1, tmp) &&
            A(ctx, &a.llist, m + 1, tmp) && A(ctx, &a.lchoff, m + 1, tmp) && A(ctx, &a.lchl, m + 1, tmp) &&
            A(ctx, &a.gparts, a.gram_parts_cap, tmp) && A(ctx, &a.G, Wuse * Wuse, tmp) &&
            A(ctx, &a.V, Wuse * Wuse, tmp);
  a.Wr_max = Wr;
  if (ok && Wr > 0)
    ok = A(ctx, &a.Md, Wr * kSpRightMax, tmp) && A(ctx, &a.Gr, (int64_t)kSpRightMax * kSpRightMax, tmp) &&
         A(ctx, &a.Vr, (int64_t)kSpRightMax * kSpRightMax, tmp) && A(ctx, &a.Vsel, (int64_t)kSpRightMax * kMaxRank, tmp) &&
         A(ctx, &a.lam, kMaxRank, tmp);
  if (!ok) {
    dfree_all(ctx, tmp);
    return fail(ctx, TT_ERR_OOM, "device allocation failed (spectral init)");
  }
  std::string msg;
  int64_t lc = 0;
  rc = spectral_init_run(ctx->stream, a, &msg, &lc);
  ctx->launches += lc;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  dfree_all(ctx, tmp);
  if (rc) return fail(ctx, rc, msg);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "spectral init");
  for (auto& c : ctx->core_set) c = 1;
  ctx->evalValid = false;
  ctx->tablesC = false;
  return TT_OK;
}

int tt_prgd_step(tt_ctx* ctx, double step_size) {
  if (!ctx) return TT_ERR_ARG;
  const int64_t mtot = ctx->allreduce ? ctx->m_global : ctx->m;
  if (!ctx->obs_set || mtot <= 0) return fail(ctx, TT_ERR_STATE, "no observations set (nonempty Omega required)");
  if (!all_cores_set(ctx)) return fail(ctx, TT_ERR_STATE, "all cores must be set before stepping");
  if (!std::isfinite(step_size)) return fail(ctx, TT_ERR_ARG, "step_size must be finite");
  if (ctx->profiling && !ctx->ev_ready) {
    for (auto& e : ctx->ev) cudaEventCreate(&e);
    ctx->ev_ready = true;
  }
  int64_t lc = 0;
  launch_set_step(ctx->stream, ctx->sc, step_size, &lc);
  ctx->launches += lc;
  int rc;
  if (!ctx->evalValid) {
    if ((rc = run_evaluate(ctx))) return rc;
    if (ctx->profiling) collect_profile(ctx, 0, 3);
  }
  if ((rc = run_update(ctx))) return rc;
  if (ctx->profiling) collect_profile(ctx, 4, 11);
  if ((rc = run_evaluate(ctx))) return rc;
  if (ctx->profiling) {
    collect_profile(ctx, 0, 3);
    ++ctx->prof_steps;
  }
  ctx->evalValid = true;
  ctx->tablesC = !ctx->plan.chain;
  ++ctx->steps;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "step");
  return TT_OK;
}

int tt_eval_at(tt_ctx* ctx, const int32_t* h_idx, int64_t count, double* h_out) {
  if (!ctx) return TT_ERR_ARG;
  if (count < 0) return fail(ctx, TT_ERR_ARG, "count < 0");
  if (count == 0) return TT_OK;
  if (!h_idx || !h_out) return fail(ctx, TT_ERR_ARG, "NULL idx or out");
  int rc = ensure_base(ctx);
  if (rc) return rc;
  int64_t lc = 0;
  if (!ctx->plan.chain && !ctx->tablesC) {
    enqueue_tables(ctx, false, &lc);
    ctx->tablesC = true;
  }
  std::vector<void*> tmp;
  int32_t* qidx = nullptr;
  double* qout = nullptr;
  if (!A(ctx, &qidx, count * ctx->d, tmp) || !A(ctx, &qout, count, tmp)) {
    dfree_all(ctx, tmp);
    return fail(ctx, TT_ERR_OOM, "device allocation failed (queries)");
  }
  cudaStream_t s = ctx->stream;
  CK(cudaMemsetAsync(&ctx->sc->index_err, 0, sizeof(int), s));
  CK(cudaMemcpyAsync(qidx, h_idx, (size_t)count * ctx->d * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  const int KL = ctx->plan.KL;
  if (ctx->plan.chain)
    launch_chain_eval(s, 0, qidx, count, ctx->ctt, ctx->C, nullptr, qout, nullptr, &ctx->sc->index_err, &lc);
  else
    launch_eval_queries(s, qidx, count, ctx->d, ctx->n_i.data(), KL, ctx->LT[KL], ctx->RT[KL],
                        ctx->ldr[KL], (int)ctx->r[KL], qout, ctx->sc, &lc);
  ctx->launches += lc;
  CK(cudaMemcpyAsync(h_out, qout, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, s));
  rc = read_scalars(ctx);
  dfree_all(ctx, tmp);
  if (rc) return rc;
  if (ctx->sc_host->index_err) return fail(ctx, TT_ERR_INDEX, "a queried index is outside [0, n_k)");
  return TT_OK;
}

int tt_residual_norm(tt_ctx* ctx, double* out) {
  if (!ctx || !out) return TT_ERR_ARG;
  if (!ctx->obs_set || (ctx->allreduce ? ctx->m_global : ctx->m) <= 0) {
    *out = 0.0;
    return TT_OK;
  }
  int rc;
  if (!ctx->evalValid) {
    if ((rc = run_evaluate(ctx))) return rc;
    ctx->evalValid = true;
    ctx->tablesC = !ctx->plan.chain;
  }
  if ((rc = read_scalars(ctx))) return rc;
  *out = std::sqrt(ctx->sc_host->sumsq);
  return TT_OK;
}

int tt_sync(tt_ctx* ctx) {
  if (!ctx) return TT_ERR_ARG;
  if (!ctx->base_ready) {
    CK(cudaStreamSynchronize(ctx->stream));
    return TT_OK;
  }
  return read_scalars(ctx);
}

const char* tt_last_error(const tt_ctx* ctx) {
  if (!ctx) return "no context";
  return ctx->err.c_str();
}

int tt_get_stats(tt_ctx* ctx, tt_stats* out) {
  if (!ctx || !out) return TT_ERR_ARG;
  out->launches = ctx->launches;
  out->steps = ctx->steps;
  out->launches_per_step = ctx->nA + ctx->nB + 1;
  out->K_L = ctx->plan.KL;
  out->graphs = ctx->profiling ? 0 : 1;
  return TT_OK;
}

int tt_set_profiling(tt_ctx* ctx, int on) {
  if (!ctx) return TT_ERR_ARG;
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->profiling = on != 0;
  for (double& v : ctx->prof_ms) v = 0.0;
  ctx->prof_steps = 0;
  return TT_OK;
}

int tt_get_profile(tt_ctx* ctx, double* h_ms, int cap, int* n_groups, int64_t* n_steps) {
  if (!ctx) return TT_ERR_ARG;
  CK(cudaStreamSynchronize(ctx->stream));
  if (n_groups) *n_groups = kNumGroups;
  if (n_steps) *n_steps = ctx->prof_steps;
  if (h_ms)
    for (int i = 0; i < kNumGroups && i < cap; ++i) h_ms[i] = ctx->prof_ms[i];
  for (double& v : ctx->prof_ms) v = 0.0;
  ctx->prof_steps = 0;
  return TT_OK;
}

const char* tt_profile_name(int group) {
  if (group < 0 || group >= kNumGroups) return "";
  return kGroupNames[group];
}

int tt_debug_round(tt_ctx* ctx, const double* h_B, int64_t count) {
  if (!ctx || !h_B) return TT_ERR_ARG;
  int rc = ensure_base(ctx);
  if (rc) return rc;
  if (count != ctx->b_off[ctx->d]) return fail(ctx, TT_ERR_ARG, "count must equal the rank-2r block size");
  cudaStream_t s = ctx->stream;
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpyAsync(ctx->B, h_B, (size_t)count * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(&ctx->sc->noop, 0, sizeof(int), s));
  DenseArgs da = dense_args(ctx);
  da.wretr = 0;
  int64_t lc = 0;
  launch_round_only(s, da, &lc);
  ctx->launches += lc;
  CK(cudaGetLastError());
  for (auto& c : ctx->core_set) c = 1;
  ctx->evalValid = false;
  ctx->tablesC = false;
  return read_scalars(ctx);
}

int tt_debug_get(tt_ctx* ctx, int what, int k, void* h_out, int64_t cap, int64_t* count) {
  if (!ctx || !h_out || !count) return TT_ERR_ARG;
  int rc = ensure_base(ctx);
  if (rc) return rc;
  cudaStream_t s = ctx->stream;
  const int d = ctx->d;
  auto need_k = [&]() { return k >= 0 && k < d; };
  const void* src = nullptr;
  int64_t cnt = 0;
  size_t esz = sizeof(double);
  switch (what) {
    case TT_DBG_PERM_PRE:
    case TT_DBG_PERM_SUF:
    case TT_DBG_OFFS_L:
    case TT_DBG_OFFS_R:
      if (ctx->plan.chain) return fail(ctx, TT_ERR_STATE, "prefix / suffix buckets exist on the table path");
      break;
    default:
      break;
  }
  switch (what) {
    case TT_DBG_PERM_PRE: src = ctx->sid_pre; cnt = ctx->m; esz = 4; break;
    case TT_DBG_PERM_SUF: src = ctx->sid_suf; cnt = ctx->m; esz = 4; break;
    case TT_DBG_OFFS_L: src = ctx->offsL; cnt = ctx->obs_set ? ctx->plan.NL + 1 : 0; esz = 8; break;
    case TT_DBG_OFFS_R: src = ctx->offsR; cnt = ctx->obs_set ? ctx->plan.NR + 1 : 0; esz = 8; break;
    case TT_DBG_PERM_MODE:
    case TT_DBG_OFFS_MODE:
      if (!need_k()) return fail(ctx, TT_ERR_ARG, "bad k");
      if (!ctx->plan.chain) return fail(ctx, TT_ERR_STATE, "per-mode buckets exist on the chain path");
      if (what == TT_DBG_PERM_MODE) {
        src = ctx->pcs.perm + (int64_t)k * ctx->m;
        cnt = ctx->obs_set ? ctx->m : 0;
        esz = 4;
      } else {
        src = ctx->pcs.offs + ctx->phi_off[k] + k;
        cnt = ctx->obs_set ? ctx->n[k] + 1 : 0;
        esz = 8;
      }
      break;
    case TT_DBG_H:
    case TT_DBG_PHI:
      if (!need_k()) return fail(ctx, TT_ERR_ARG, "bad k");
      src = (what == TT_DBG_H ? ctx->h : ctx->phi) + ctx->phi_off[k];
      cnt = ctx->n[k];
      break;
    case TT_DBG_U:
    case TT_DBG_Y:
    case TT_DBG_AHAT: {
      if (!need_k()) return fail(ctx, TT_ERR_ARG, "bad k");
      const double* base = what == TT_DBG_U ? ctx->U : (what == TT_DBG_Y ? ctx->Y : ctx->Ahat);
      src = base + ctx->core_off[k];
      cnt = ctx->core_off[k + 1] - ctx->core_off[k];
      break;
    }
    case TT_DBG_P:
      if (!need_k()) return fail(ctx, TT_ERR_ARG, "bad k");
      src = ctx->P + ctx->p_off[k];
      cnt = ctx->r[k + 1] * ctx->r[k + 1];
      break;
    case TT_DBG_EPS: {
      if ((rc = read_scalars(ctx))) return rc;
      if (cap < 13) return fail(ctx, TT_ERR_ARG, "capacity too small");
      double* o = static_cast<double*>(h_out);
      o[0] = ctx->sc_host->eps;
      o[1] = ctx->sc_host->sumsq;
      o[2] = ctx->sc_host->alpha;
      o[3] = ctx->sc_host->p;
      o[4] = (double)ctx->sc_host->pad;   // cumulative Jacobi sweeps (diagnostic)
      const int nc = cap >= 29 ? 24 : 8;
      for (int i = 0; i < nc; ++i) o[5 + i] = (double)ctx->sc_host->cyc[i];
      *count = 5 + nc;
      return TT_OK;
    }
    case TT_DBG_RESID: {
      if (!ctx->obs_set) return fail(ctx, TT_ERR_STATE, "no observations");
      if (cap < ctx->m) return fail(ctx, TT_ERR_ARG, "capacity too small");
      if (!ctx->evalValid && ctx->m > 0) {
        if ((rc = run_evaluate(ctx))) return rc;
        ctx->evalValid = true;
        ctx->tablesC = !ctx->plan.chain;
      }
      std::vector<double> gp(ctx->m);
      std::vector<int32_t> sp(ctx->m);
      if (ctx->plan.chain) {   // original sample order already
        if (ctx->m > 0)
          CK(cudaMemcpyAsync(h_out, ctx->g, ctx->m * sizeof(double), cudaMemcpyDeviceToHost, s));
        if ((rc = read_scalars(ctx))) return rc;
        *count = ctx->m;
        return TT_OK;
      }
      if (ctx->m > 0) {
        CK(cudaMemcpyAsync(gp.data(), ctx->g, ctx->m * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(sp.data(), ctx->sid_pre, ctx->m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      }
      if ((rc = read_scalars(ctx))) return rc;
      double* o = static_cast<double*>(h_out);
      for (int64_t t = 0; t < ctx->m; ++t) o[sp[t]] = gp[t];
      *count = ctx->m;
      return TT_OK;
    }
    default:
      return fail(ctx, TT_ERR_ARG, "unknown debug item");
  }
  if (cnt > cap) return fail(ctx, TT_ERR_ARG, "capacity too small");
  if (cnt > 0 && src) CK(cudaMemcpyAsync(h_out, src, cnt * esz, cudaMemcpyDeviceToHost, s));
  *count = cnt;
  CK(cudaStreamSynchronize(s));
  return TT_OK;
}

}  // extern "C"
