// passes_mid.cu — the passes over Omega re-associated through the middle cores
// ("middle split").  K = K_L (0-based split), j = x_K, i = x_{K-1}.
//
// Pass A (A1-A2, SDDMM), prefix rows P, samples ordered (P, j, S') with S = j + n_K S':
//   v_s = T^{<=K-1}(P) C_K(:, j, :) T^{>=K+1}(:, S')
// Per 32-row tile, W[P][(j, c)] = sum_a A_K[P][a] C_K[a][j][c] is one FP64 tensor-core GEMM
// (32 x r_K) . (r_K x n_K r_{K+1}); each sample then needs one row of the level-(K+1) right
// table (n_K times fewer rows than level K: 8 MB at config 5, L2 resident) and a length-r dot.
//
// Pass B (A7-A9 boundary, SpMM), prefix rows:
//   E_K[P] = psi_L[P] sum_s g_s psi_R[S] U^{>=K}(:, S)
//          = psi_L[P] sum_j U_K(:, j, :) Z[P][j],   Z[P][j] = sum_{s in P, x_K = j} w_s U^{>=K+1}(:, S')
// with w_s = g_s phi_K(j)^{-1} psi'_R[S'] (psi'_R = prod_{k > K} phi_k^{-1}):
// the samples of a row form one run per j, so each 8-lane group accumulates its row's runs
// in a fixed order (deterministic), and E = Z . Ust is a tile GEMM (32 x n_K r_{K+1}) .
// (n_K r_{K+1} x r_K) on DMMA.  The suffix side is the mirror image (rows S, runs of i =
// x_{K-1}, table level K-1 of the left part, F_K[S] = psi_R[S] sum_i Z'[S][i] U_{K-1}(:, i, :)).
// Compared with gathering the level-K tables (128 B random DRAM reads per sample, 134 MB
// tables at config 5), this trades ~286 FP64 flops per sample on the tensor cores for
// L2-resident gathers.
#include <algorithm>

#include "prgd_internal.cuh"

namespace prgd {
namespace {

constexpr int kMT = 256;          // threads per CTA
constexpr int kTR = 32;           // rows per tile = 8-lane groups per CTA

__host__ __device__ inline int mmald(int w) { return ((w + 15) / 16) * 16 + 4; }

__device__ __forceinline__ void dmma_m(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

struct MidA {                 // pass A, prefix rows
  const int64_t* offs;        // [N+1]
  const int32_t* key;         // j * N1 + S'
  const double* y;
  double* g;
  double* H;                  // [N] sum g^2 per row
  const double* A;            // left table level K, rows P (lda)
  const double* core;         // C_K [rK][nK][rK1]
  const double* Bt;           // right table level K+1, rows S' (ldb)
  int64_t N, N1;
  int lda, rK, nK, rK1, ldb;
  int shift;                  // key = (j << shift) | S'
};

struct MidB {                 // pass B, either side
  const int64_t* offs;
  const int32_t* key;         // j * N1 + r'
  const double* x;            // g in this side's order
  const double* T;            // gathered table (rows r', ldt), pre-scaled by psi' over r'
  const double* phij;         // phi of the middle mode (n_mid values)
  const double* rowscale;     // psi over the rows
  const double* core;         // middle core
  double* out;                // E_K or F_K rows (ldo)
  int64_t N, N1;
  int left;                   // 1: out[i] = sum U[i][j][c] Z[j][c]; 0: out[c] = sum U[a][i][c] Z[i][a]
  int nmid, rt, ldt, rout, ldo, r0, r1;   // core dims r0 x nmid x r1
  int shift;                  // key = (j << shift) | r'
};

// ---------------------------------------------------------------- tile staging (TMA bulk)
// Each CTA walks its 32-row tiles with a two-stage pipeline: while the groups process tile t
// from shared memory, thread 0 has already issued the bulk copies (cp.async.bulk, completion
// on an mbarrier) of tile t+1's row offsets, its samples' keys and values, and (pass A) its 32
// left-table rows.  Copies start at 16-byte aligned addresses below the wanted ranges
// (arrays are padded on the host); a tile with more than kCap samples is read from global.
constexpr int kCap = 1536;            // samples per staged tile
constexpr int kOffsN = 36;            // staged offsets (33 used, 16-byte multiple)

__device__ __forceinline__ unsigned saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra "
      "WAIT%=;\n}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}

struct Stage {            // one pipeline stage in shared memory
  int64_t* offs;          // [kOffsN]  offs[P0 ..]
  int32_t* key;           // [kCap + 8]
  double* val;            // [kCap + 4]
  double* A;              // [kTR * lda] (pass A only)
  int64_t a0k, a0v;       // first staged sample index of key / val
  int direct;             // 1: tile too large, read from global
};

// Issue the copies of tile `tile` into stage st (thread 0 only).  b, e: sample range.
__device__ void stage_issue(Stage& st, uint64_t* bar, const int64_t* offs, const int32_t* key,
                            const double* val, const double* A, int lda, int64_t P0, int64_t b,
                            int64_t e) {
  unsigned bytes = kOffsN * 8;
  const bool fits = (e - b) <= kCap;
  const int64_t a0k = b & ~(int64_t)3, e1k = (e + 3) & ~(int64_t)3;
  const int64_t a0v = b & ~(int64_t)1, e1v = (e + 1) & ~(int64_t)1;
  if (fits) bytes += (unsigned)((e1k - a0k) * 4 + (e1v - a0v) * 8);
  if (A) bytes += (unsigned)(kTR * lda * 8);
  mbar_expect(bar, bytes);
  bulk_g2s(st.offs, offs + P0, kOffsN * 8, bar);
  if (fits) {
    if (e1k > a0k) bulk_g2s(st.key, key + a0k, (unsigned)((e1k - a0k) * 4), bar);
    if (e1v > a0v) bulk_g2s(st.val, val + a0v, (unsigned)((e1v - a0v) * 8), bar);
  }
  if (A) bulk_g2s(st.A, A + P0 * lda, (unsigned)(kTR * lda * 8), bar);
  st.a0k = a0k;
  st.a0v = a0v;
  st.direct = fits ? 0 : 1;
}

// Pass A (SDDMM).  Shared memory: Cst (4 KS x ldw), Ws (32 x ldw), As (32 x ldaS), 2 stages.
__global__ void __launch_bounds__(kMT, 1) k_mid_sddmm(MidA p, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ Stage stg[2];
  __shared__ int64_t nxt[2];
  const int W = p.nK * p.ldb;
  const int ldw = mmald(W);
  const int K = p.rK, KS = (K + 3) >> 2, K4 = 4 * KS;
  const int ldaS = mmald(K4);
  double* Cst = sm;
  double* Ws = Cst + (int64_t)K4 * ldw;
  double* As = Ws + (int64_t)kTR * ldw;
  double* sbase = As + (int64_t)kTR * ldaS;
  const int stA = kTR * p.lda;                              // staged A doubles
  const int stride = kOffsN + (kCap + 8) / 2 + (kCap + 4) + stA;   // doubles per stage
  if (threadIdx.x < 2) {
    Stage& st = stg[threadIdx.x];
    double* base = sbase + (int64_t)threadIdx.x * stride;
    st.offs = reinterpret_cast<int64_t*>(base);
    st.key = reinterpret_cast<int32_t*>(base + kOffsN);
    st.val = base + kOffsN + (kCap + 8) / 2;
    st.A = st.val + (kCap + 4);
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  for (int t = threadIdx.x; t < K4 * W; t += blockDim.x) {
    const int k = t / W, q = t - k * W;
    const int j = q / p.ldb, c = q - j * p.ldb;
    Cst[k * ldw + q] = (k < K && c < p.rK1) ? p.core[((int64_t)k * p.nK + j) * p.rK1 + c] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tq = lane & 3;
  const int grp = threadIdx.x >> 3, sub = lane & 7, gbase = lane & 24;
  const unsigned gmask = 0xffu << gbase;
  const int nJ = W >> 3;
  const int sh = p.shift, smask = (1 << sh) - 1;
  const bool act = 2 * sub < p.ldb;
  const int64_t ntiles = (p.N + kTR - 1) / kTR;
  auto range = [&](int64_t tile, int64_t& b, int64_t& e) {
    const int64_t P0 = tile * kTR;
    b = p.offs[P0];
    e = p.offs[min(P0 + kTR, p.N)];
  };
  if (threadIdx.x == 0 && (int64_t)blockIdx.x < ntiles) {
    int64_t b, e;
    range(blockIdx.x, b, e);
    stage_issue(stg[0], &bars[0], p.offs, p.key, p.y, p.A, p.lda, blockIdx.x * (int64_t)kTR, b, e);
    const int64_t t1 = blockIdx.x + gridDim.x;
    if (t1 < ntiles) {
      nxt[0] = p.offs[t1 * kTR];
      nxt[1] = p.offs[min(t1 * kTR + kTR, p.N)];
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int sidx = it & 1;
    const int64_t P0 = tile * kTR;
    const int nrow = (int)(p.N - P0 < kTR ? p.N - P0 : kTR);
    if (threadIdx.x == 0) {
      const int64_t t1 = tile + gridDim.x;
      if (t1 < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_issue(stg[sidx ^ 1], &bars[sidx ^ 1], p.offs, p.key, p.y, p.A, p.lda, t1 * kTR, nxt[0],
                    nxt[1]);
        const int64_t t2 = t1 + gridDim.x;
        if (t2 < ntiles) {
          nxt[0] = p.offs[t2 * kTR];
          nxt[1] = p.offs[min(t2 * kTR + kTR, p.N)];
        }
      }
    }
    mbar_wait(&bars[sidx], (unsigned)((it >> 1) & 1));
    const Stage& st = stg[sidx];
    // As (padded) from the staged rows, then W = As . Cst with 16 independent tiles per warp
    for (int t = threadIdx.x; t < kTR * K4; t += blockDim.x) {
      const int r = t / K4, k = t - r * K4;
      As[r * ldaS + k] = (r < nrow && k < K) ? st.A[r * p.lda + k] : 0.0;
    }
    __syncthreads();
    for (int t = warp; t < 4 * nJ; t += kMT / 32) {
      const int I = t / nJ, J = t - I * nJ;
      double d0 = 0.0, d1 = 0.0;
      for (int k = 0; k < K4; k += 4)
        dmma_m(d0, d1, As[(I * 8 + gid) * ldaS + k + tq], Cst[(k + tq) * ldw + J * 8 + gid]);
      double* w = Ws + (I * 8 + gid) * ldw + J * 8 + 2 * tq;
      w[0] = d0;
      w[1] = d1;
    }
    __syncthreads();
    double acc = 0.0;
    if (grp < nrow) {
      const int64_t b = st.offs[grp], e = st.offs[grp + 1];
      const double* wrow = Ws + grp * ldw + 2 * sub;
      const int32_t* kb = st.direct ? p.key : st.key - st.a0k;
      const double* yb = st.direct ? p.y : st.val - st.a0v;
      for (int64_t c0 = b; c0 < e; c0 += 8) {
        const int nc = (int)(e - c0 < 8 ? e - c0 : 8);
        const int kv = sub < nc ? kb[c0 + sub] : 0;
        const double yv = sub < nc ? yb[c0 + sub] : 0.0;
        double2 bv[8];
        int jj[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int ku = __shfl_sync(gmask, kv, gbase + u);
          jj[u] = ku >> sh;
          bv[u] = make_double2(0.0, 0.0);
          if (u < nc && act)
            bv[u] = __ldg(reinterpret_cast<const double2*>(p.Bt + (int64_t)(ku & smask) * p.ldb) + sub);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          double part = 0.0;
          if (act) {
            const double* w = wrow + jj[u] * p.ldb;
            part = fma(w[0], bv[u].x, w[1] * bv[u].y);
          }
          part += __shfl_xor_sync(gmask, part, 4);
          part += __shfl_xor_sync(gmask, part, 2);
          part += __shfl_xor_sync(gmask, part, 1);
          const double yu = __shfl_sync(gmask, yv, gbase + u);
          if (u < nc) {
            const double gv = part - yu;
            if (sub == 0) p.g[c0 + u] = gv;
            acc = fma(gv, gv, acc);
          }
        }
      }
      if (sub == 0) p.H[P0 + grp] = acc;
    }
    __syncthreads();
  }
}

// Pass B (SpMM).  Shared memory: Ust (W x ldu), Zs (32 x ldz), 1/phi (nmid), 2 stages.
__global__ void __launch_bounds__(kMT, 1) k_mid_spmm(MidB p, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ Stage stg[2];
  __shared__ int64_t nxt[2];
  const int W = p.nmid * p.ldt;
  const int ldz = mmald(W);
  const int ro8 = (p.ldo + 7) & ~7;
  const int ldu = mmald(ro8);
  double* Us = sm;                          // W x ldu
  double* Zs = Us + (int64_t)W * ldu;       // kTR x ldz
  double* phinv = Zs + (int64_t)kTR * ldz;  // [nmid], padded to even
  double* sbase = phinv + ((p.nmid + 1) & ~1);
  const int stride = kOffsN + (kCap + 8) / 2 + (kCap + 4);
  if (threadIdx.x < 2) {
    Stage& st = stg[threadIdx.x];
    double* base = sbase + (int64_t)threadIdx.x * stride;
    st.offs = reinterpret_cast<int64_t*>(base);
    st.key = reinterpret_cast<int32_t*>(base + kOffsN);
    st.val = base + kOffsN + (kCap + 8) / 2;
    st.A = nullptr;
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  for (int t = threadIdx.x; t < W * ro8; t += blockDim.x) {
    const int q = t / ro8, o = t - q * ro8;
    const int j = q / p.ldt, x = q - j * p.ldt;
    double v = 0.0;
    if (o < p.rout && x < p.rt) {
      if (p.left) v = p.core[((int64_t)o * p.nmid + j) * p.r1 + x];   // U[o][j][x]
      else v = p.core[((int64_t)x * p.nmid + j) * p.r1 + o];          // U[x][j][o]
    }
    Us[q * ldu + o] = v;
  }
  for (int t = threadIdx.x; t < p.nmid; t += blockDim.x) phinv[t] = 1.0 / p.phij[t];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tq = lane & 3;
  const int grp = threadIdx.x >> 3, sub = lane & 7, gbase = lane & 24;
  const unsigned gmask = 0xffu << gbase;
  const bool act = 2 * sub < p.ldt;
  const int smask = (1 << p.shift) - 1;
  const int64_t ntiles = (p.N + kTR - 1) / kTR;
  if (threadIdx.x == 0 && (int64_t)blockIdx.x < ntiles) {
    const int64_t P0 = blockIdx.x * (int64_t)kTR;
    stage_issue(stg[0], &bars[0], p.offs, p.key, p.x, nullptr, 0, P0, p.offs[P0],
                p.offs[min(P0 + kTR, p.N)]);
    const int64_t t1 = blockIdx.x + gridDim.x;
    if (t1 < ntiles) {
      nxt[0] = p.offs[t1 * kTR];
      nxt[1] = p.offs[min(t1 * kTR + kTR, p.N)];
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int sidx = it & 1;
    const int64_t R0 = tile * kTR;
    const int nrow = (int)(p.N - R0 < kTR ? p.N - R0 : kTR);
    if (threadIdx.x == 0) {
      const int64_t t1 = tile + gridDim.x;
      if (t1 < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_issue(stg[sidx ^ 1], &bars[sidx ^ 1], p.offs, p.key, p.x, nullptr, 0, t1 * kTR, nxt[0],
                    nxt[1]);
        const int64_t t2 = t1 + gridDim.x;
        if (t2 < ntiles) {
          nxt[0] = p.offs[t2 * kTR];
          nxt[1] = p.offs[min(t2 * kTR + kTR, p.N)];
        }
      }
    }
    for (int t = threadIdx.x; t < kTR * W; t += blockDim.x) Zs[(t / W) * ldz + (t % W)] = 0.0;
    mbar_wait(&bars[sidx], (unsigned)((it >> 1) & 1));
    __syncthreads();
    const Stage& st = stg[sidx];
    if (grp < nrow) {
      const int64_t b = st.offs[grp], e = st.offs[grp + 1];
      const int32_t* kb = st.direct ? p.key : st.key - st.a0k;
      const double* xb = st.direct ? p.x : st.val - st.a0v;
      double* zrow = Zs + grp * ldz + 2 * sub;
      int jcur = -1;
      double2 acc = make_double2(0.0, 0.0);
      for (int64_t c0 = b; c0 < e; c0 += 8) {
        const int nc = (int)(e - c0 < 8 ? e - c0 : 8);
        const int kv = sub < nc ? kb[c0 + sub] : 0;
        const double xv = sub < nc ? xb[c0 + sub] : 0.0;
        double2 tv[8];
        int jj[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int ku = __shfl_sync(gmask, kv, gbase + u);
          jj[u] = u < nc ? (ku >> p.shift) : -1;
          tv[u] = make_double2(0.0, 0.0);
          if (u < nc && act)
            tv[u] = __ldg(reinterpret_cast<const double2*>(p.T + (int64_t)(ku & smask) * p.ldt) + sub);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (jj[u] < 0) break;
          const double wu = __shfl_sync(gmask, xv, gbase + u) * phinv[jj[u]];
          if (jj[u] != jcur) {
            if (jcur >= 0 && act) *reinterpret_cast<double2*>(zrow + jcur * p.ldt) = acc;
            jcur = jj[u];
            acc = make_double2(0.0, 0.0);
          }
          acc.x = fma(wu, tv[u].x, acc.x);
          acc.y = fma(wu, tv[u].y, acc.y);
        }
      }
      if (jcur >= 0 && act) *reinterpret_cast<double2*>(zrow + jcur * p.ldt) = acc;
    }
    __syncthreads();
    // out tile = Zs . Us  (4 row blocks x ro8/8 column blocks, K = W)
    const int ocb = ro8 >> 3;
    for (int t = warp; t < 4 * ocb; t += kMT / 32) {
      const int I = t / ocb, J = t - I * ocb;
      const double* zr = Zs + (I * 8 + gid) * ldz + tq;
      const double* ur = Us + tq * ldu + J * 8 + gid;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0, g0 = 0.0, g1 = 0.0;
      int q = 0;
      for (; q + 16 <= W; q += 16) {
        dmma_m(d0, d1, zr[q], ur[q * ldu]);
        dmma_m(e0, e1, zr[q + 4], ur[(q + 4) * ldu]);
        dmma_m(f0, f1, zr[q + 8], ur[(q + 8) * ldu]);
        dmma_m(g0, g1, zr[q + 12], ur[(q + 12) * ldu]);
      }
      for (; q < W; q += 4) dmma_m(d0, d1, zr[q], ur[q * ldu]);
      const int64_t r = R0 + I * 8 + gid;
      const int o = J * 8 + 2 * tq;
      if (r < p.N) {
        const double f = p.rowscale ? p.rowscale[r] : 1.0;
        if (o < p.ldo) p.out[r * p.ldo + o] = o < p.rout ? ((d0 + e0) + (f0 + g0)) * f : 0.0;
        if (o + 1 < p.ldo) p.out[r * p.ldo + o + 1] = o + 1 < p.rout ? ((d1 + e1) + (f1 + g1)) * f : 0.0;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- register-only variants
// The per-row state stays in registers (no shared-memory W / Z rows), so the number of rows
// in flight is bounded by registers, not by shared memory: an 8-lane group owns a row (lane
// l holds entries 2l, 2l+1 of every r-vector), W[P][j] = A_K[P] C_K(:, j, :) is formed once
// per run of equal j (16 x 16 matvec from the core staged in shared memory) and, for pass B,
// the run sum Z_j is folded into the row's output at the run's end, E += U_K(:, j, :) Z_j.

// Pass A: shared memory holds Cs[a][j][c] (c fastest, ldb wide).
__global__ void __launch_bounds__(kMT, 2) k_mid_sddmm_r(MidA p, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ __align__(16) double sm[];
  const int K = p.rK, nK = p.nK, ldb = p.ldb;
  double* Cs = sm;                                        // [K][nK][ldb]
  for (int t = threadIdx.x; t < K * nK * ldb; t += blockDim.x) {
    const int c = t % ldb, aj = t / ldb;
    const int j = aj % nK, a = aj / nK;
    Cs[t] = c < p.rK1 ? p.core[((int64_t)a * nK + j) * p.rK1 + c] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane & 7, gbase = lane & 24;
  const unsigned gmask = 0xffu << gbase;
  const bool act = 2 * sub < ldb;
  const int sh = p.shift, smask = (1 << sh) - 1;
  const int64_t ngrp = (int64_t)gridDim.x * (kMT / 8);
  for (int64_t P = (int64_t)blockIdx.x * (kMT / 8) + (threadIdx.x >> 3); P < p.N; P += ngrp) {
    // A_K[P] replicated in the group's registers
    double av[16];
    {
      const double2 mine = (2 * sub < p.lda && 2 * sub < 16)
                               ? __ldg(reinterpret_cast<const double2*>(p.A + P * p.lda) + sub)
                               : make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        av[2 * q] = __shfl_sync(gmask, mine.x, gbase + q);
        av[2 * q + 1] = __shfl_sync(gmask, mine.y, gbase + q);
      }
    }
    const int64_t b = p.offs[P], e = p.offs[P + 1];
    int jcur = -1;
    double2 wv = make_double2(0.0, 0.0);
    double acc = 0.0;
    for (int64_t c0 = b; c0 < e; c0 += 8) {
      const int nc = (int)(e - c0 < 8 ? e - c0 : 8);
      const int kv = sub < nc ? p.key[c0 + sub] : 0;
      const double yv = sub < nc ? p.y[c0 + sub] : 0.0;
      double2 bv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int ku = __shfl_sync(gmask, kv, gbase + u);
        bv[u] = make_double2(0.0, 0.0);
        if (u < nc && act)
          bv[u] = __ldg(reinterpret_cast<const double2*>(p.Bt + (int64_t)(ku & smask) * ldb) + sub);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u >= nc) break;
        const int j = __shfl_sync(gmask, kv, gbase + u) >> sh;
        if (j != jcur) {
          jcur = j;
          double wx = 0.0, wy = 0.0;
          if (act) {
            const double* cj = Cs + (int64_t)j * ldb + 2 * sub;
#pragma unroll
            for (int a = 0; a < 16; ++a)
              if (a < K) {
                const double2 c = *reinterpret_cast<const double2*>(cj + (int64_t)a * nK * ldb);
                wx = fma(av[a], c.x, wx);
                wy = fma(av[a], c.y, wy);
              }
          }
          wv = make_double2(wx, wy);
        }
        double part = fma(wv.x, bv[u].x, wv.y * bv[u].y);
        part += __shfl_xor_sync(gmask, part, 4);
        part += __shfl_xor_sync(gmask, part, 2);
        part += __shfl_xor_sync(gmask, part, 1);
        const double gv = part - __shfl_sync(gmask, yv, gbase + u);
        if (sub == 0) p.g[c0 + u] = gv;
        acc = fma(gv, gv, acc);
      }
    }
    if (sub == 0) p.H[P] = acc;
  }
}

// Pass B: shared memory holds the core as Us[j][x][o] (o fastest, ro wide): left
// Us[j][c][i] = U[i][j][c], right Us[i][a][c] = U[a][i][c], and 1/phi of the middle mode.
__global__ void __launch_bounds__(kMT, 2) k_mid_spmm_r(MidB p, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ __align__(16) double sm[];
  const int nmid = p.nmid, ldt = p.ldt;
  const int ro = (p.ldo + 1) & ~1;
  double* Us = sm;                                  // [nmid][ldt][ro]
  double* phinv = Us + (int64_t)nmid * ldt * ro;
  for (int t = threadIdx.x; t < nmid * ldt * ro; t += blockDim.x) {
    const int o = t % ro, jx = t / ro;
    const int x = jx % ldt, j = jx / ldt;
    double v = 0.0;
    if (o < p.rout && x < p.rt) {
      if (p.left) v = p.core[((int64_t)o * nmid + j) * p.r1 + x];   // U[o][j][x]
      else v = p.core[((int64_t)x * nmid + j) * p.r1 + o];          // U[x][j][o]
    }
    Us[t] = v;
  }
  for (int t = threadIdx.x; t < nmid; t += blockDim.x) phinv[t] = 1.0 / p.phij[t];
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane & 7, gbase = lane & 24;
  const unsigned gmask = 0xffu << gbase;
  const bool act = 2 * sub < ldt;          // this lane holds table entries 2 sub, 2 sub + 1
  const bool oact = 2 * sub < ro;          // ... and output entries 2 sub, 2 sub + 1
  const int smask = (1 << p.shift) - 1;
  const int64_t ngrp = (int64_t)gridDim.x * (kMT / 8);
  for (int64_t row = (int64_t)blockIdx.x * (kMT / 8) + (threadIdx.x >> 3); row < p.N; row += ngrp) {
    const int64_t b = p.offs[row], e = p.offs[row + 1];
    int jcur = -1;
    double2 z = make_double2(0.0, 0.0), eo = make_double2(0.0, 0.0);
    auto fold = [&](int j) {           // eo += U(:, j, :) z  (z: the run sum, 2 per lane)
      double zv[16];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        zv[2 * q] = __shfl_sync(gmask, z.x, gbase + q);
        zv[2 * q + 1] = __shfl_sync(gmask, z.y, gbase + q);
      }
      if (oact) {
        const double* uj = Us + (int64_t)j * ldt * ro + 2 * sub;
#pragma unroll
        for (int x = 0; x < 16; ++x)
          if (x < ldt) {
            const double2 u = *reinterpret_cast<const double2*>(uj + x * ro);
            eo.x = fma(u.x, zv[x], eo.x);
            eo.y = fma(u.y, zv[x], eo.y);
          }
      }
    };
    for (int64_t c0 = b; c0 < e; c0 += 8) {
      const int nc = (int)(e - c0 < 8 ? e - c0 : 8);
      const int kv = sub < nc ? p.key[c0 + sub] : 0;
      const double xv = sub < nc ? p.x[c0 + sub] : 0.0;
      double2 tv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int ku = __shfl_sync(gmask, kv, gbase + u);
        tv[u] = make_double2(0.0, 0.0);
        if (u < nc && act)
          tv[u] = __ldg(reinterpret_cast<const double2*>(p.T + (int64_t)(ku & smask) * ldt) + sub);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u >= nc) break;
        const int j = __shfl_sync(gmask, kv, gbase + u) >> p.shift;
        if (j != jcur) {
          if (jcur >= 0) fold(jcur);
          jcur = j;
          z = make_double2(0.0, 0.0);
        }
        const double w = __shfl_sync(gmask, xv, gbase + u) * phinv[j];
        z.x = fma(w, tv[u].x, z.x);
        z.y = fma(w, tv[u].y, z.y);
      }
    }
    if (jcur >= 0) fold(jcur);
    if (oact) {
      const double f = p.rowscale ? p.rowscale[row] : 1.0;
      const int o = 2 * sub;
      if (o < p.ldo) p.out[row * p.ldo + o] = o < p.rout ? eo.x * f : 0.0;
      if (o + 1 < p.ldo) p.out[row * p.ldo + o + 1] = o + 1 < p.rout ? eo.y * f : 0.0;
    }
  }
}

__global__ void k_scale_rows(const double* __restrict__ in, const double* __restrict__ f, int64_t rows,
                             int ld, double* __restrict__ out, const Scalars* sc) {
  if (sc && sc->noop) return;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rows * ld) return;
  out[e] = in[e] * f[e / ld];
}

int g_sms_mid = 0;
int sms_mid() {
  if (!g_sms_mid) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_mid, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms_mid <= 0) g_sms_mid = 148;
  }
  return g_sms_mid;
}

}  // namespace

void launch_mid_passA(cudaStream_t s, const int64_t* offs, const int32_t* key, const double* y,
                      double* g, double* H, const double* A, int lda, const double* core, int rK,
                      int nK, int rK1, const double* Bt, int ldb, int64_t N, int64_t N1,
                      const Scalars* sc, int64_t* launches) {
  int sh = 0;
  while (((int64_t)1 << sh) < N1) ++sh;
  MidA p{offs, key, y, g, H, A, core, Bt, N, N1, lda, rK, nK, rK1, ldb, sh};
  const int W = nK * ldb, K4 = 4 * ((rK + 3) / 4);
  const size_t stage = kOffsN + (kCap + 8) / 2 + (kCap + 4) + (size_t)kTR * lda;
  const size_t smem = ((size_t)K4 * mmald(W) + (size_t)kTR * mmald(W) + (size_t)kTR * mmald(K4) +
                       2 * stage) * sizeof(double);
  const int64_t ntiles = (N + kTR - 1) / kTR;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms_mid());
  const size_t smem_r = (size_t)rK * nK * ldb * sizeof(double);
  const int64_t ngr = (N + kMT / 8 - 1) / (kMT / 8);
  const int grid_r = (int)std::min<int64_t>(ngr, (int64_t)sms_mid() * 2);
  if (rK <= 16 && ldb <= 16 && lda <= 16) {
    k_mid_sddmm_r<<<std::max(grid_r, 1), kMT, smem_r, s>>>(p, sc);
    ++*launches;
    return;
  }
  k_mid_sddmm<<<std::max(grid, 1), kMT, smem, s>>>(p, sc);
  ++*launches;
}

void launch_mid_passB(cudaStream_t s, bool left, const int64_t* offs, const int32_t* key,
                      const double* x, const double* T, int rt, int ldt, const double* wr,
                      const double* phij, const double* rowscale, const double* core, int r0,
                      int nmid, int r1, double* out, int rout, int ldo, int64_t N, int64_t N1,
                      const Scalars* sc, int64_t* launches) {
  int sh = 0;
  while (((int64_t)1 << sh) < N1) ++sh;
  MidB p{offs, key, x, T, phij, rowscale, core, out, N, N1, left ? 1 : 0, nmid, rt, ldt, rout,
         ldo, r0, r1, sh};
  (void)wr;
  const int W = nmid * ldt, ro8 = (ldo + 7) & ~7;
  const size_t stage = kOffsN + (kCap + 8) / 2 + (kCap + 4);
  const size_t smem = ((size_t)W * mmald(ro8) + (size_t)kTR * mmald(W) + ((nmid + 1) & ~1) +
                       2 * stage) * sizeof(double);
  const int64_t ntiles = (N + kTR - 1) / kTR;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms_mid());
  const int ro = (ldo + 1) & ~1;
  const size_t smem_r = ((size_t)nmid * ldt * ro + nmid) * sizeof(double);
  const int64_t ngr = (N + kMT / 8 - 1) / (kMT / 8);
  const int grid_r = (int)std::min<int64_t>(ngr, (int64_t)sms_mid() * 2);
  if (ldt <= 16 && ro <= 16) {
    k_mid_spmm_r<<<std::max(grid_r, 1), kMT, smem_r, s>>>(p, sc);
    ++*launches;
    return;
  }
  k_mid_spmm<<<std::max(grid, 1), kMT, smem, s>>>(p, sc);
  ++*launches;
}

void launch_scale_rows(cudaStream_t s, const double* in, const double* f, int64_t rows, int ld,
                       double* out, const Scalars* sc, int64_t* launches) {
  k_scale_rows<<<(unsigned)((rows * ld + 255) / 256), 256, 0, s>>>(in, f, rows, ld, out, sc);
  ++*launches;
}

void passes_mid_init() {
  cudaFuncSetAttribute(k_mid_sddmm, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_mid_sddmm_r, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_mid_spmm_r, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_mid_spmm, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace prgd
