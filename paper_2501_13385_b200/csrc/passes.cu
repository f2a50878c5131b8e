// passes.cu — the two passes over Omega and the weight computation.
//
// Pass A, prefix side (A1-A2, SDDMM; passes_flat.cu): for every bucket P and sample s in it,
//   v_s = T^{<=KL-1}(P) . T^{>=KL}(:, S(s)),  g_s = v_s - y_s,  H_L[P] = sum g_s^2
// Pass A, suffix side (A3 input, k_seg GSQ): H_R[S] = sum_{s in S} g_s^2.
// Marginals (A3): h_{k,j} = sum of H over table rows whose k-th digit is j
//   (= ||M_k(G)(j,:)||^2).
// Weights (A3, A12): eps, w = eps + h, phi = w^{1/(4d)}, alpha.
// Pass B (A7-A9 boundary, SpMM):
//   E_KL[P] = psi_L[P] sum_{s in P} g_s Ttil^{>=KL}(:, S(s))
//   F_KL[S] = psi_R[S] sum_{s in S} g_s Ttil^{<=KL-1}(P(s))
// with psi = prod phi^{-1} over the prefix (suffix) digits, so that
// psi_L psi_R g_s = ghat_s = (W^{-1/2} G)_s.
//
// Work decomposition: a warp owns a run of "virtual rows" (<= kSplit samples of one
// bucket); results of split buckets go to partial slots reduced in order by k_seg_fix, so
// every sum has a fixed order (deterministic).  k_seg (GSQ, and the adaptive step's DPASS)
// walks the virtual rows one by one with LPS lanes per sample gathering one table row (2 fp64
// per lane, 16-byte loads); the SpMM passes run as k_spmm_pipe, which streams the warp's whole
// sample range through a cp.async gather pipeline in shared memory.
#include "prgd_internal.cuh"

namespace prgd {
namespace {

constexpr unsigned kFull = 0xffffffffu;

struct SegDev {
  int64_t nwarps;
  int64_t warp_off;       // first plan warp of this launch
  const int4* vrow;       // {row, count, first sample, partial slot} per virtual row
  const int64_t* warp_vbegin;
  double* part;
  int ld;
  const int32_t* col;
  const int32_t* perm;
  double* g;
  double* g2;             // GSQ: the gathered g stored to g2[s] (suffix order)
  const double* rowtab;
  const double* coltab;
  const double* rowtab2;  // DPASS second row / gathered tables
  const double* coltab2;
  const double* rowscale;
  double* out;
};

__device__ __forceinline__ double2 ld2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// Minimum resident CTAs per SM (register cap), measured on B200 at config 5: the dot-product
// (DPASS) pass is fastest at 4 (64 registers; 5 spills and is 10 % slower), the row-plan SpMM
// at 5 (48 registers).
#ifndef PRGD_SEG_OCC_SPMM
#define PRGD_SEG_OCC_SPMM 5
#endif
#ifndef PRGD_SEG_OCC_SDDMM
#define PRGD_SEG_OCC_SDDMM 4
#endif
#ifndef PRGD_SEG_UNR
#define PRGD_SEG_UNR 4
#endif
template <int MODE>
struct SegOcc {
  static constexpr int v = MODE == kDPASS ? PRGD_SEG_OCC_SDDMM : (MODE == kSPMM ? PRGD_SEG_OCC_SPMM : 8);
};

// LPS lanes per sample, each holding V double2 of the row (ld = 2 LPS V)
template <int LPS, int MODE, int V = 1>
__global__ void __launch_bounds__(256, SegOcc<MODE>::v) k_seg(SegDev a, const Scalars* sc) {
  static_assert(V == 1 || MODE != kGSQ, "vector lanes: not for the scalar GSQ pass");
  if (sc && sc->noop) return;
  constexpr int G = 32 / LPS;        // samples per warp step
  constexpr int STEPS = 32 / G;      // steps per 32-sample chunk (= LPS)
  constexpr int UNR = STEPS < PRGD_SEG_UNR ? STEPS : PRGD_SEG_UNR;
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPS, sub = lane - grp * LPS;
  const int64_t wl = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (wl >= a.nwarps) return;
  const int64_t warp = wl + a.warp_off;
  constexpr int ld = 2 * LPS * V;      // table row stride (the launcher picks LPS V = a.ld / 2)
  const int64_t v0 = a.warp_vbegin[warp], v1 = a.warp_vbegin[warp + 1];
  for (int64_t v = v0; v < v1; ++v) {
    const int4 vr = a.vrow[v];
    const int32_t row = vr.x;
    const int64_t trow = row;
    const int64_t beg = vr.z;
    const int cnt = vr.y;
    double2 rv[V], rv2[V];
#pragma unroll
    for (int q = 0; q < V; ++q) {
      rv[q] = rv2[q] = make_double2(0.0, 0.0);
      if (MODE == kDPASS) rv[q] = ld2(a.rowtab + trow * ld + 2 * (V * sub + q));
      if (MODE == kDPASS) rv2[q] = ld2(a.rowtab2 + trow * ld + 2 * (V * sub + q));
    }
    double accs = 0.0;
    double2 accv[V];
#pragma unroll
    for (int q = 0; q < V; ++q) accv[q] = make_double2(0.0, 0.0);
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int nc = cnt - c0 < 32 ? cnt - c0 : 32;
      const int64_t s = beg + c0 + lane;
      const bool have = lane < nc;
      // lane-parallel loads of this chunk's per-sample data (coalesced / independent)
      int colv = 0;
      double xv = 0.0;    // g (GSQ)
      if (have) {
        if (MODE != kGSQ) colv = a.col[s];
        if (MODE != kDPASS) xv = a.perm ? a.g[a.perm[s]] : a.g[s];
      }
      if constexpr (MODE == kGSQ) {
        if (have && a.g2) a.g2[s] = xv;
        accs = fma(xv, xv, accs);
        continue;
      } else if constexpr (MODE == kDPASS) {
        // partial dot products of the chunk's STEPS samples of this lane group, then a
        // transpose-reduction over the group's LPS lanes (LPS - 1 shuffles for LPS samples
        // instead of log2(LPS) per sample): afterwards lane `sub` holds the dot product of
        // sample t = sub * G + grp, which it finishes and stores (coalesced over the warp)
        double pd[STEPS];
#pragma unroll
        for (int st0 = 0; st0 < STEPS; st0 += UNR) {
          double2 b[UNR][V], b2[MODE == kDPASS ? UNR : 1][V];
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            // lanes past the chunk hold colv = 0: their loads read table row 0 (valid) and
            // their dot products are never finished (t >= nc below), so no predicate is needed
            const int t = (st0 + u) * G + grp;
            const int cidx = __shfl_sync(kFull, colv, t & 31);
            const int off = cidx * ld + 2 * V * sub;   // < 2^31: table size checked by the planner
#pragma unroll
            for (int q = 0; q < V; ++q) {
              b[u][q] = ld2(a.coltab + off + 2 * q);
              if constexpr (MODE == kDPASS) b2[u][q] = ld2(a.coltab2 + off + 2 * q);
            }
          }
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            double part = fma(rv[0].x, b[u][0].x, rv[0].y * b[u][0].y);
#pragma unroll
            for (int q = 1; q < V; ++q) part = fma(rv[q].y, b[u][q].y, fma(rv[q].x, b[u][q].x, part));
            if constexpr (MODE == kDPASS) {
#pragma unroll
              for (int q = 0; q < V; ++q) part = fma(rv2[q].y, b2[u][q].y, fma(rv2[q].x, b2[u][q].x, part));
            }
            pd[st0 + u] = part;
          }
        }
#pragma unroll
        for (int o = LPS / 2; o > 0; o >>= 1) {
          const bool up = (sub & o) != 0;
#pragma unroll
          for (int j = 0; j < o; ++j) {
            const double send = up ? pd[j] : pd[j + o];
            const double keep = up ? pd[j + o] : pd[j];
            pd[j] = keep + __shfl_xor_sync(kFull, send, o);
          }
        }
        const int t = sub * G + grp;
        {
          if (t < nc) accs = fma(pd[0], pd[0], accs);
        }
      } else {
#pragma unroll
      for (int st0 = 0; st0 < STEPS; st0 += UNR) {
        double2 b[UNR][V];
        double xs[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          // lanes past the chunk hold colv = 0 and xv = 0: they read table row 0 and add
          // 0 x row (finite tables), so no predicate is needed
          const int t = (st0 + u) * G + grp;
          const int cidx = __shfl_sync(kFull, colv, t & 31);
          xs[u] = __shfl_sync(kFull, xv, t & 31);
          const int off = cidx * ld + 2 * V * sub;   // < 2^31 (planner)
#pragma unroll
          for (int q = 0; q < V; ++q) b[u][q] = ld2(a.coltab + off + 2 * q);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < V; ++q) {
            accv[q].x = fma(xs[u], b[u][q].x, accv[q].x);
            accv[q].y = fma(xs[u], b[u][q].y, accv[q].y);
          }
      }
      }
    }
    const int32_t pslot = vr.w;
    if (MODE == kGSQ) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) accs += __shfl_xor_sync(kFull, accs, o);
      if (lane == 0) {
        if (pslot < 0) a.out[row] = accs;
        else a.part[pslot] = accs;
      }
    } else if (MODE == kDPASS) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) accs += __shfl_xor_sync(kFull, accs, o);   // every lane holds samples
      if (lane == 0) {
        if (pslot < 0) a.out[row] = accs;
        else a.part[pslot] = accs;
      }
    } else {
#pragma unroll
      for (int o = LPS; o < 32; o <<= 1)
#pragma unroll
        for (int q = 0; q < V; ++q) {
          accv[q].x += __shfl_xor_sync(kFull, accv[q].x, o);
          accv[q].y += __shfl_xor_sync(kFull, accv[q].y, o);
        }
      if (grp == 0) {
        double* dst;
        if (pslot < 0) {
          const double f = a.rowscale ? a.rowscale[trow] : 1.0;
          dst = a.out + trow * ld + 2 * V * sub;
#pragma unroll
          for (int q = 0; q < V; ++q) {
            accv[q].x *= f;
            accv[q].y *= f;
          }
        } else {
          dst = a.part + (int64_t)pslot * ld + 2 * V * sub;
        }
#pragma unroll
        for (int q = 0; q < V; ++q) *reinterpret_cast<double2*>(dst + 2 * q) = accv[q];
      }
    }
  }
}

// Sum the partial slots of split buckets in slot order.
__global__ void k_seg_fix(int vec, int64_t nsplit, const int32_t* __restrict__ split_row,
                          const int64_t* __restrict__ split_first, const double* __restrict__ part,
                          int ld, const double* __restrict__ rowscale, double* __restrict__ out,
                          const Scalars* sc) {
  if (sc && sc->noop) return;
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int w = vec ? ld : 1;
  int64_t i = e / w;
  int c = (int)(e - i * w);
  if (i >= nsplit) return;
  const int32_t row = split_row[i];
  double acc = 0.0;
  for (int64_t sl = split_first[i]; sl < split_first[i + 1]; ++sl)
    acc += vec ? part[sl * ld + c] : part[sl];
  if (vec) {
    if (rowscale) acc *= rowscale[row];
    out[(int64_t)row * ld + c] = acc;
  } else {
    out[row] = acc;
  }
}

struct MargArgs {
  int nm;
  int n[kMaxD];
  int64_t stride[kMaxD];
  int64_t out_off[kMaxD];
  int64_t blk_off[kMaxD + 1];
  int64_t N;
};

// Marginals in two deterministic stages.  Block (bin = (mode, j), chunk) sums its chunk of
// the (hi, lo) index space of H[(hi*n + j)*stride + lo] (fixed thread order + tree), then
// one warp per bin adds the chunk partials in chunk order.
constexpr int kMargChunks = 32;
__global__ void k_marg_partial(const double* __restrict__ H, MargArgs ma, double* __restrict__ part) {
  __shared__ double red[256];
  const int bin = blockIdx.x, chunk = blockIdx.y;
  int m = 0;
  while (m + 1 < ma.nm && ma.blk_off[m + 1] <= bin) ++m;
  const int j = bin - (int)ma.blk_off[m];
  const int64_t st = ma.stride[m];
  const int64_t span = (int64_t)ma.n[m] * st;
  const int64_t total = (ma.N / span) * st;
  const int64_t per = (total + kMargChunks - 1) / kMargChunks;
  const int64_t e0 = chunk * per, e1 = e0 + per < total ? e0 + per : total;
  double acc = 0.0;
  // table rows N <= 2^30 (planner): 32-bit index arithmetic (a 64-bit division per element
  // made this kernel issue-bound)
  const uint32_t st32 = (uint32_t)st, span32 = (uint32_t)span, off32 = (uint32_t)j * st32;
  for (uint32_t e = (uint32_t)e0 + threadIdx.x; e < (uint32_t)e1; e += blockDim.x) {
    const uint32_t hi = e / st32, lo = e - hi * st32;
    acc += H[hi * span32 + off32 + lo];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)bin * kMargChunks + chunk] = red[0];
}

__global__ void k_marg_final(const double* __restrict__ part, int nbins, const int64_t* __restrict__ dummy,
                             MargArgs ma, double* __restrict__ h) {
  const int bin = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (bin >= nbins) return;
  double v = lane < kMargChunks ? part[(int64_t)bin * kMargChunks + lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int m = 0;
  while (m + 1 < ma.nm && ma.blk_off[m + 1] <= bin) ++m;
  if (lane == 0) h[ma.out_off[m] + (bin - ma.blk_off[m])] = v;
  (void)dummy;
}

__global__ void k_weights(const double* __restrict__ h, int d, int64_t nsum, int n0, int eps_rule,
                          double eps_fixed, int step_rule, double* __restrict__ phi, Scalars* sc) {
  __shared__ double rs[256], rm[256];
  double s = 0.0, mx = 0.0;
  for (int64_t e = threadIdx.x; e < n0; e += blockDim.x) s += h[e];   // mode-0 marginal: sum g^2
  for (int64_t e = threadIdx.x; e < nsum; e += blockDim.x) mx = fmax(mx, h[e]);
  rs[threadIdx.x] = s;
  rm[threadIdx.x] = mx;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      rs[threadIdx.x] += rs[threadIdx.x + o];
      rm[threadIdx.x] = fmax(rm[threadIdx.x], rm[threadIdx.x + o]);
    }
    __syncthreads();
  }
  const double sumsq = rs[0];
  double eps = 0.0;
  if (eps_rule == 0) eps = rm[0];          // ||G||_vee^2
  else if (eps_rule == 1) eps = eps_fixed;
  const bool bad = !isfinite(sumsq) || !isfinite(eps);
  const bool noop = bad || (eps_rule == 0 && eps == 0.0);
  const double ex = 1.0 / (4.0 * d);
  if (!noop) {
    for (int64_t e = threadIdx.x; e < nsum; e += blockDim.x)
      phi[e] = eps_rule == 2 ? 1.0 : pow(eps + h[e], ex);
  }
  if (threadIdx.x == 0) {
    sc->sumsq = sumsq;
    sc->eps = eps;
    double alpha = sc->step_size;
    if (step_rule == 0) alpha = eps_rule == 2 ? sc->step_size / sc->p : sc->step_size * sqrt(eps) / sc->p;
    sc->alpha = alpha;
    sc->noop = noop ? 1 : 0;
    if (bad) atomicOr(&sc->err, (int)kErrNaN);
  }
}

struct PsiArgs {
  int d, KL;
  int n[kMaxD];
  int64_t phi_off[kMaxD];
  int64_t NL, NR;
};

__global__ void k_psi(const double* __restrict__ phi, PsiArgs pa, double* __restrict__ psiL,
                      double* __restrict__ psiR, const Scalars* sc) {
  if (sc && sc->noop) return;
  // table rows N_L, N_R <= 2^30 (planner): 32-bit digit extraction
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < pa.NL) {
    uint32_t P = (uint32_t)e;
    double v = 1.0;
    for (int k = pa.KL - 1; k >= 0; --k) {
      const uint32_t q = P / (uint32_t)pa.n[k];
      const int xk = (int)(P - q * (uint32_t)pa.n[k]);
      P = q;
      v /= phi[pa.phi_off[k] + xk];
    }
    psiL[e] = v;
  } else if (e < pa.NL + pa.NR) {
    uint32_t S = (uint32_t)(e - pa.NL);
    const int64_t S0 = e - pa.NL;
    double v = 1.0;
    for (int k = pa.KL; k < pa.d; ++k) {
      const uint32_t q = S / (uint32_t)pa.n[k];
      const int xk = (int)(S - q * (uint32_t)pa.n[k]);
      S = q;
      v /= phi[pa.phi_off[k] + xk];
    }
    psiR[S0] = v;
  }
}

struct QArgs {
  int d, KL, ld, rb;
  int n[kMaxD];
};

__global__ void k_eval_queries(const int32_t* __restrict__ idx, int64_t count, QArgs q,
                               const double* __restrict__ tabL, const double* __restrict__ tabR,
                               double* __restrict__ out, Scalars* sc) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= count) return;
  const int32_t* x = idx + s * q.d;
  int64_t P = 0, S = 0;
  bool bad = false;
  for (int k = 0; k < q.KL; ++k) {
    int xk = x[k];
    bad |= (xk < 0) | (xk >= q.n[k]);
    P = P * q.n[k] + (xk < 0 ? 0 : xk);
  }
  for (int k = q.d - 1; k >= q.KL; --k) {
    int xk = x[k];
    bad |= (xk < 0) | (xk >= q.n[k]);
    S = S * q.n[k] + (xk < 0 ? 0 : xk);
  }
  if (bad) {
    atomicOr(&sc->index_err, 1);
    out[s] = 0.0;
    return;
  }
  const double* a = tabL + P * q.ld;
  const double* b = tabR + S * q.ld;
  double v = 0.0;
  for (int i = 0; i < q.rb; ++i) v = fma(a[i], b[i], v);
  out[s] = v;
}

__global__ void k_set_step(Scalars* sc, double step) { sc->step_size = step; }

// sum g^2 = sum_j h_{0,j} (the mode-0 marginal), fixed-order block reduction.
__global__ void k_sumsq(const double* __restrict__ h0, int n0, Scalars* sc) {
  __shared__ double red[256];
  double s = 0.0;
  for (int e = threadIdx.x; e < n0; e += blockDim.x) s += h0[e];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) sc->sumsq = red[0];
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// ------------------------------------------------------------------ pipelined SpMM (pass B)
// Same sums as k_seg<SPMM> (out[row] = rowscale[row] sum_{s in vrow} g_s coltab[col_s], split
// rows to partial slots), same plan, different schedule: a warp walks the contiguous sample
// range of its virtual rows in 32-sample chunks.  The gathered table rows of chunk c + 1 land
// in shared memory by cp.async while chunk c is accumulated, and the per-sample streams (col,
// g) are loaded one to two chunks ahead, so a warp keeps one chunk of row gathers in flight and
// has no dependent load chain per row (k_seg: plan record -> col / g -> gathers, per row).
// Within a chunk, sample i is accumulated by lane group i mod G (LPS lanes, one double2 of the
// row each); a virtual row ending in the chunk is reduced over the groups and written.  Fixed
// order throughout (deterministic).
constexpr int kPipeWarps = 8;

__device__ __forceinline__ void pipe_cp16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void pipe_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void pipe_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int LPS, int NB>
__global__ void __launch_bounds__(32 * kPipeWarps) k_spmm_pipe(SegDev a, const Scalars* sc) {
  if (sc && sc->noop) return;
  constexpr int G = 32 / LPS, STEPS = LPS, LD = 2 * LPS, CH = 32 * LD;
  extern __shared__ double pipe_smem[];
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPS, sub = lane - grp * LPS;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (warp >= a.nwarps) return;
  // per warp: NB chunk buffers of gathered rows, then NB x 32 staged g values
  double* buf = pipe_smem + (size_t)(threadIdx.x >> 5) * NB * (CH + 32);
  double* gsm = buf + NB * CH;
  const int64_t v0 = a.warp_vbegin[warp], v1 = a.warp_vbegin[warp + 1];
  // sample positions fit in 32 bits (m < 2^31: the planner's int4 records)
  const int S0 = a.vrow[v0].z;
  const int4 lastv = a.vrow[v1 - 1];
  const int S1 = lastv.z + lastv.y;
  const int nch = S1 > S0 ? (S1 - S0 + 31) >> 5 : 1;
  auto ld_col = [&](int c) -> int {
    const int t = S0 + 32 * c + lane;
    return (c < nch && t < S1) ? a.col[t] : 0;   // past the end: row 0 (valid), weight 0
  };
  auto ld_g = [&](int c) -> double {
    const int t = S0 + 32 * c + lane;
    if (c >= nch || t >= S1) return 0.0;
    return a.perm ? a.g[a.perm[t]] : a.g[t];
  };
  const double* src0 = a.coltab + 2 * (lane % (LD / 2));
  auto issue = [&](int c, int colv) {   // chunk c's table rows -> buf[c % NB] (LD / 2 x 16 B per lane)
    double* dst = buf + (c % NB) * CH + 2 * (lane % (LD / 2));
#pragma unroll
    for (int j = 0; j < LD / 2; ++j) {
      const int i = (j * 32 + lane) / (LD / 2);   // sample; lane % (LD / 2) is its 16-byte part
      const int ci = __shfl_sync(kFull, colv, i);
      pipe_cp16(dst + i * LD, src0 + ci * LD);    // ci * LD < 2^31 (planner)
    }
  };
  // current virtual row (warp-uniform); records cached 32 at a time
  int64_t vb = v0, cur = v0;
  int4 rec = vb + lane < v1 ? a.vrow[vb + lane] : make_int4(0, 0, 0, -1);
  int row = __shfl_sync(kFull, rec.x, 0), cnt = __shfl_sync(kFull, rec.y, 0);
  int beg = __shfl_sync(kFull, rec.z, 0);
  int slot = __shfl_sync(kFull, rec.w, 0);
  double2 acc = make_double2(0.0, 0.0);

  // with a permutation (the staged g of the sliced pass A suffix) the index of chunk c + 2 is
  // loaded while chunk c runs, so the dependent g load of chunk c + 1 issues without waiting on it
  auto ld_p = [&](int c) -> int {
    const int t = S0 + 32 * c + lane;
    return (c < nch && t < S1) ? a.perm[t] : -1;
  };
  int pN = a.perm ? ld_p(1) : -1;
  double gC = ld_g(0);
#pragma unroll
  for (int j = 0; j + 1 < NB; ++j) {   // chunks 0 .. NB-2 in flight
    if (j < nch) issue(j, ld_col(j));
    pipe_commit();
  }
  int colN = ld_col(NB - 1);
  for (int c = 0; c < nch; ++c) {
    const int colNN = ld_col(c + NB);
    double gN;
    if (a.perm) {
      gN = pN >= 0 ? a.g[pN] : 0.0;
      pN = ld_p(c + 2);
    } else {
      gN = ld_g(c + 1);
    }
    if (c + NB - 1 < nch) issue(c + NB - 1, colN);
    pipe_commit();
    double* gc = gsm + (c % NB) * 32;
    gc[lane] = gC;
    pipe_wait<NB - 1>();
    __syncwarp();
    const double* cb = buf + (c % NB) * CH + 2 * sub;
    const int c0 = S0 + 32 * c;
    while (cur < v1) {
      const int e = beg + cnt;
      const int lo = beg > c0 ? beg - c0 : 0;
      const int hi = e < c0 + 32 ? e - c0 : 32;
      // samples outside the virtual row weigh 0 (every slot holds a finite gathered row), so
      // the accumulation runs unpredicated
#pragma unroll
      for (int st = 0; st < STEPS; ++st) {
        const int i = st * G + grp;
        const double w = (unsigned)(i - lo) < (unsigned)(hi - lo) ? gc[i] : 0.0;
        const double2 r = *reinterpret_cast<const double2*>(cb + i * LD);
        acc.x = fma(w, r.x, acc.x);
        acc.y = fma(w, r.y, acc.y);
      }
      if (e > c0 + 32) break;   // the virtual row continues in the next chunk
#pragma unroll
      for (int o = LPS; o < 32; o <<= 1) {
        acc.x += __shfl_xor_sync(kFull, acc.x, o);
        acc.y += __shfl_xor_sync(kFull, acc.y, o);
      }
      if (grp == 0) {
        double* dst;
        if (slot < 0) {
          const double f = a.rowscale ? a.rowscale[row] : 1.0;
          acc.x *= f;
          acc.y *= f;
          dst = a.out + (int64_t)row * LD + 2 * sub;
        } else {
          dst = a.part + (int64_t)slot * LD + 2 * sub;
        }
        *reinterpret_cast<double2*>(dst) = acc;
      }
      acc = make_double2(0.0, 0.0);
      if (++cur >= v1) break;
      if (cur - vb >= 32) {   // warp-uniform
        vb += 32;
        rec = vb + lane < v1 ? a.vrow[vb + lane] : make_int4(0, 0, 0, -1);
      }
      const int sl = (int)(cur - vb);
      row = __shfl_sync(kFull, rec.x, sl);
      cnt = __shfl_sync(kFull, rec.y, sl);
      beg = __shfl_sync(kFull, rec.z, sl);
      slot = __shfl_sync(kFull, rec.w, sl);
    }
    __syncwarp();   // every lane is done with buf / gsm[c % NB] before chunk c + NB lands there
    colN = colNN;
    gC = gN;
  }
}

template <int LPS, int NB>
void spmm_pipe_launch_nb(cudaStream_t s, const SegDev& dv, const Scalars* sc) {
  const size_t smem = (size_t)kPipeWarps * NB * 32 * (2 * LPS + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmm_pipe<LPS, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const unsigned grid = blocks_for(dv.nwarps, kPipeWarps);
  k_spmm_pipe<LPS, NB><<<grid, 32 * kPipeWarps, smem, s>>>(dv, sc);
}

// Two chunk buffers per warp (64 KB per CTA at 16-wide rows, 3 CTAs = 24 warps per SM).
// Measured at config 5: three buffers (2 CTAs per SM) 0.79 ms per pass vs 0.65 ms; L2
// evict_last hints on the gathers with evict-first streams / outputs: no change.
template <int LPS>
void spmm_pipe_launch(cudaStream_t s, const SegDev& dv, const Scalars* sc) {
  spmm_pipe_launch_nb<LPS, 2>(s, dv, sc);
}

// PRGD_SPMM_PIPE=0 / 1 forces the row-plan / pipelined SpMM (A/B measurements)
inline int spmm_pipe_env() {
  static const int v = [] {
    const char* e = getenv("PRGD_SPMM_PIPE");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return v;
}

template <int LPS>
void seg_dispatch_mode(cudaStream_t s, int mode, const SegDev& dv, unsigned grid,
                       const Scalars* sc) {
  // DPASS: from 16-wide rows on, 4 columns per lane (half the lanes per sample, half the
  // transpose-reduction and index shuffles per sample).  (Pass A's SDDMM runs as the flat
  // sample-major kernel of passes_flat.cu.)
  if constexpr (LPS >= 8) {
    if (mode == kDPASS) { k_seg<LPS / 2, kDPASS, 2><<<grid, 256, 0, s>>>(dv, sc); return; }
  }
  if (mode == kDPASS) k_seg<LPS, kDPASS><<<grid, 256, 0, s>>>(dv, sc);
  else if (mode == kGSQ) k_seg<1, kGSQ><<<grid, 256, 0, s>>>(dv, sc);
  else if (spmm_pipe_env() == 1 || (spmm_pipe_env() < 0 && LPS >= 8)) spmm_pipe_launch<LPS>(s, dv, sc);
  else k_seg<LPS, kSPMM><<<grid, 256, 0, s>>>(dv, sc);
}

}  // namespace

void launch_seg(cudaStream_t s, const SegArgs& a, const Scalars* sc, int64_t* launches) {
  const SegPlan& p = *a.plan;
  if (p.nwarps == 0) return;
  SegDev dv;
  dv.nwarps = p.nwarps;
  dv.warp_off = 0;
  dv.vrow = p.vrow;
  dv.warp_vbegin = p.warp_vbegin;
  dv.part = p.part;
  dv.ld = a.ld;
  dv.col = a.col;
  dv.perm = a.perm;
  dv.g = a.g;
  dv.g2 = a.g2;
  dv.rowtab = a.rowtab;
  dv.coltab = a.coltab;
  dv.rowtab2 = a.rowtab2;
  dv.coltab2 = a.coltab2;
  dv.rowscale = a.rowscale;
  dv.out = a.out;
  const int vec = a.mode == kSPMM ? 1 : 0;
  const unsigned grid = blocks_for(dv.nwarps * 32, 256);
  switch (a.ld / 2) {
    case 1: seg_dispatch_mode<1>(s, a.mode, dv, grid, sc); break;
    case 2: seg_dispatch_mode<2>(s, a.mode, dv, grid, sc); break;
    case 4: seg_dispatch_mode<4>(s, a.mode, dv, grid, sc); break;
    case 8: seg_dispatch_mode<8>(s, a.mode, dv, grid, sc); break;
    default: seg_dispatch_mode<16>(s, a.mode, dv, grid, sc); break;
  }
  ++*launches;
  if (p.nsplit > 0) {
    const int64_t n = p.nsplit * (vec ? a.ld : 1);
    k_seg_fix<<<blocks_for(n, 256), 256, 0, s>>>(vec, p.nsplit, p.split_row, p.split_first, p.part, a.ld,
                                                 a.rowscale, a.out, sc);
    ++*launches;
  }
}

// n_modes / strides are passed in n_dev_modes as host pointer to an int array of
// [nm] sizes (host!), msd_first: left side (first mode most significant).
void launch_marginals(cudaStream_t s, const double* H, int64_t N, int nm, const int* n_host,
                      bool msd_first, double* h_out, double* scratch, int64_t* launches) {
  MargArgs ma;
  ma.nm = nm;
  ma.N = N;
  int64_t off = 0;
  ma.blk_off[0] = 0;
  for (int m = 0; m < nm; ++m) {
    ma.n[m] = n_host[m];
    int64_t st = 1;
    if (msd_first) {
      for (int i = m + 1; i < nm; ++i) st *= n_host[i];
    } else {
      for (int i = 0; i < m; ++i) st *= n_host[i];
    }
    ma.stride[m] = st;
    ma.out_off[m] = off;
    off += n_host[m];
    ma.blk_off[m + 1] = off;
  }
  static_assert(kMargChunks <= 32, "one warp per bin");
  k_marg_partial<<<dim3((unsigned)off, kMargChunks), 256, 0, s>>>(H, ma, scratch);
  k_marg_final<<<(unsigned)((off * 32 + 255) / 256), 256, 0, s>>>(scratch, (int)off, nullptr, ma,
                                                                  h_out);
  *launches += 2;
}

void launch_weights(cudaStream_t s, const double* h, int d, const int* n_host, int64_t nsum,
                    int eps_rule, double eps_fixed, int step_rule, double* phi, Scalars* sc,
                    int64_t* launches) {
  k_weights<<<1, 256, 0, s>>>(h, d, nsum, n_host[0], eps_rule, eps_fixed, step_rule, phi, sc);
  ++*launches;
}

void launch_psi(cudaStream_t s, const double* phi, const int64_t* phi_off_host, int KL, int d,
                const int* n_host, int64_t NL, int64_t NR, double* psiL, double* psiR,
                const Scalars* sc, int64_t* launches) {
  PsiArgs pa;
  pa.d = d;
  pa.KL = KL;
  for (int k = 0; k < d; ++k) {
    pa.n[k] = n_host[k];
    pa.phi_off[k] = phi_off_host[k];
  }
  pa.NL = NL;
  pa.NR = NR;
  k_psi<<<blocks_for(NL + NR, 256), 256, 0, s>>>(phi, pa, psiL, psiR, sc);
  ++*launches;
}

void launch_eval_queries(cudaStream_t s, const int32_t* idx, int64_t count, int d,
                         const int* n_host, int KL, const double* tabL, const double* tabR,
                         int ld, int rb, double* out, Scalars* sc, int64_t* launches) {
  if (count <= 0) return;
  QArgs q;
  q.d = d;
  q.KL = KL;
  q.ld = ld;
  q.rb = rb;
  for (int k = 0; k < d; ++k) q.n[k] = n_host[k];
  k_eval_queries<<<blocks_for(count, 256), 256, 0, s>>>(idx, count, q, tabL, tabR, out, sc);
  ++*launches;
}

void launch_set_step(cudaStream_t s, Scalars* sc, double step, int64_t* launches) {
  k_set_step<<<1, 1, 0, s>>>(sc, step);
  ++*launches;
}

void launch_gather_sq_sum(cudaStream_t s, const double* h0, int n0, Scalars* sc, int64_t* launches) {
  k_sumsq<<<1, 256, 0, s>>>(h0, n0, sc);
  ++*launches;
}

}  // namespace prgd
