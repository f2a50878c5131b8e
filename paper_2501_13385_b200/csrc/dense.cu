// dense.cu — the small dense work of one PRGD iteration.
//
//   k_orth_cs      (one 8-CTA thread-block cluster, round_cs.inc) A4 That = W^{1/2} T
//                  (Prop. 3.1), A5 left-orthogonal U by distributed
//                  CholeskyQR, A6 right Grams P_k = That^{>=k+1}
//                  That^{>=k+1 T} and their Cholesky factors.
//   k_project      (d CTAs, one per core, independent) A10 closed-form projection
//                  (PAPER.md:356-360), A11 unweighting and A13 the
//                  rank-2r cores B_k of W_l = T_l - alpha grad.
//   k_round_cs     (one 8-CTA cluster, round_cs.inc) A14 TT-rounding = Alg. 1 on W_l
//                  (PAPER.md:114-131): right-to-left CholeskyQR, then left-to-right
//                  CholeskyQR + truncation of the small R factor by one-sided Jacobi.
//   k_dense_orth / k_dense_round (1 CTA, Householder below) are the fallbacks for bonds the
//                  cluster kernels do not take (2 r > 32) and for rank-deficient unfoldings.
//
// Householder QR (LAPACK dgeqr2 / dorg2r conventions: beta = -sign(alpha)||x||,
// tau = (beta - alpha)/beta, v_j = 1, tau = 0 for a zero sub-column) with rows owned
// by threads (row i by thread i mod blockDim) and two block barriers per column:
// per-thread column partials are reduced across the warp by a transpose-reduction
// (31 shuffles for 32 columns) and across warps through shared memory.  Matrices are
// staged in shared memory (odd row stride: conflict-free column access) when they
// fit, else processed in a global scratch area by the same code.
#include <cooperative_groups.h>

#include "prgd_internal.cuh"

namespace cg = cooperative_groups;

namespace prgd {
namespace {

constexpr int kNW = kDenseThreads / 32;
constexpr int kMaxCols = 2 * kMaxRank;   // 64
constexpr int kProjThreads = 512;        // k_project: one CTA per core, latency-bound phases

__device__ __forceinline__ double shx(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }

// Warp transpose-reduction of NM per-lane values: afterwards lane l holds the warp
// total of index (l & (NM-1)) in o0 (NM <= 32), or of indices l and l+32 (NM = 64).
template <int NM>
__device__ __forceinline__ void warp_treduce(double (&v)[NM], int lane, double& o0, double& o1) {
  if constexpr (NM == 64) {
    double a[32], b[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      a[i] = v[i];
      b[i] = v[i + 32];
    }
    double t;
    warp_treduce<32>(a, lane, o0, t);
    warp_treduce<32>(b, lane, o1, t);
  } else {
#pragma unroll
    for (int off = 16; off >= NM; off >>= 1) {
#pragma unroll
      for (int i = 0; i < NM; ++i) v[i] += shx(v[i], off);
    }
#pragma unroll
    for (int off = NM / 2; off >= 1; off >>= 1) {
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < off; ++i) {
        const double send = up ? v[i] : v[i + off];
        const double keep = up ? v[i + off] : v[i];
        v[i] = keep + shx(send, off);
      }
    }
    o0 = v[0];
    o1 = 0.0;
  }
}

// ---------------------------------------------------------------- FP64 tensor-core tiles
// D(8x8) += A(8x4) B(4x8), mma.sync m8n8k4 f64 (SASS DMMA.8x8x4).  Fragments:
// a = A[gid][tq], b = B[tq][gid], d0/d1 = D[gid][2tq], D[gid][2tq+1]; gid = lane/4, tq = lane%4.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Block GEMM C[M x N] = sum_k fa(i, k) fb(k, j) on DMMA tiles, warps round-robin over the
// 8x8 output tiles; the accessors must return 0 outside [0,M) x [0,K) / [0,K) x [0,N),
// fs(i, j, v) must ignore i >= M or j >= N.  No barrier inside.
template <class FA, class FB, class FS>
__device__ __forceinline__ void mma_gemm(int M, int N, int K, FA fa, FB fb, FS fs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gid = lane >> 2, tq = lane & 3;
  const int mt = (M + 7) >> 3, nt = (N + 7) >> 3;
  for (int t = warp; t < mt * nt; t += nw) {
    const int I = t / nt, J = t - I * nt;
    const int i = I * 8 + gid, j = J * 8 + gid;
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
    int k = 0;
    for (; k + 8 <= K; k += 8) {
      dmma(d0, d1, fa(i, k + tq), fb(k + tq, j));
      dmma(e0, e1, fa(i, k + 4 + tq), fb(k + 4 + tq, j));
    }
    for (; k < K; k += 4) {
      const int kk = k + tq;
      dmma(d0, d1, kk < K ? fa(i, kk) : 0.0, kk < K ? fb(kk, j) : 0.0);
    }
    fs(I * 8 + gid, J * 8 + 2 * tq, d0 + e0);
    fs(I * 8 + gid, J * 8 + 2 * tq + 1, d1 + e1);
  }
}

// In place A[m x n] <- A T^T (T: n x n, stride tl); each warp owns 8-row blocks and loads
// their fragments before writing.  n <= 32.
__device__ void mma_mul_rt_inplace(double* A, int ld, int m, int n, const double* T, int tl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gid = lane >> 2, tq = lane & 3;
  const int nk = (n + 3) >> 2, nt = (n + 7) >> 3;
  for (int I = warp; I * 8 < m; I += nw) {
    const int i = I * 8 + gid;
    double af[8];
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) {
      const int c = 4 * s2 + tq;
      af[s2] = (s2 < nk && i < m && c < n) ? A[(int64_t)i * ld + c] : 0.0;
    }
    for (int J = 0; J < nt; ++J) {
      const int j = J * 8 + gid;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        if (s2 < nk) {
          const int c = 4 * s2 + tq;
          dmma(d0, d1, af[s2], (j < n && c < n) ? T[j * tl + c] : 0.0);
        }
      }
      const int jc = J * 8 + 2 * tq;
      if (i < m && jc < n) A[(int64_t)i * ld + jc] = d0;
      if (i < m && jc + 1 < n) A[(int64_t)i * ld + jc + 1] = d1;
    }
  }
}

// Cholesky G = L L^T (n <= 64) by the whole CTA, in place (stride gl, upper zeroed).
// Step j: every thread reads the pivot itself (no broadcast barrier), r_j = rsqrt(pivot);
// the trailing update G[i][k] -= G[i][j] G[k][j] r_j^2 (j < k <= i) is spread over all
// threads; column j is scaled at the end from the saved r_j.  One barrier per step.
// Returns false (CTA-uniform) on a non-positive or non-finite pivot.
__device__ bool chol_cta(double* G, int gl, int n, double* rinv) {
  bool ok = true;
  for (int j = 0; j < n; ++j) {
    const double djj = G[j * gl + j];
    const bool good = djj > 0.0 && isfinite(djj);
    ok = ok && good;
    const double rj = good ? rsqrt(djj) : 1.0;
    const double rj2 = rj * rj;
    if (threadIdx.x == 0) rinv[j] = rj;
    const int nr = n - 1 - j;                       // rows/cols j+1..n-1
    for (int t = threadIdx.x; t < nr * nr; t += blockDim.x) {
      const int i = t / nr, k = t - i * nr;         // (i, k) over the square, k <= i kept
      if (k <= i) {
        const int gi = j + 1 + i, gk = j + 1 + k;
        G[gi * gl + gk] = fma(-G[gi * gl + j] * rj2, G[gk * gl + j], G[gi * gl + gk]);
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, c = e - i * n;
    double v;
    if (c > i) v = 0.0;
    else if (c == i) v = G[i * gl + i] * rinv[i];   // sqrt(pivot) = pivot * rsqrt(pivot)
    else v = G[i * gl + c] * rinv[c];
    G[i * gl + c] = v;
  }
  __syncthreads();
  return ok;
}

// Li = L^{-1} (lower, n <= 64): thread c < n computes column c by forward substitution
// directly into Li (shared memory), x_i = (delta_ic - sum_{c<=k<i} L[i][k] x_k) / L[i][i].
__device__ void trinv_cta(const double* L, int gl, int n, double* Li, int il) {
  const int c = threadIdx.x;
  if (c < n) {
    for (int i = 0; i < c; ++i) Li[i * il + c] = 0.0;
    for (int i = c; i < n; ++i) {
      double s0 = (i == c) ? 1.0 : 0.0, s1 = 0.0;
      int k = c;
      for (; k + 1 < i; k += 2) {
        s0 = fma(-L[i * gl + k], Li[k * il + c], s0);
        s1 = fma(-L[i * gl + k + 1], Li[(k + 1) * il + c], s1);
      }
      if (k < i) s0 = fma(-L[i * gl + k], Li[k * il + c], s0);
      Li[i * il + c] = (s0 + s1) / L[i * gl + i];
    }
  }
  __syncthreads();
}

struct Work {
  double* red;   // [kNW][kMaxCols] warp partials
  double* vec;   // [kMaxCols] per-column coefficients
  double* sc3;   // [4] tau, denom, beta
  double* tau;   // [kMaxCols]
  double* S1;    // S x S
  double* S2;
  double* S3;
  double* S4;    // S x S (QR scratch: Gram / Cholesky factor)
  double* S5;    // S x S (QR scratch: accumulated R)
  int* perm;     // [S]
  int* ptab;     // Jacobi pair table, [S][S/2] x 2 ints
  long long* diag;  // diagnostic counters (Scalars::cyc) or null
  double* mat;   // staging area
  int64_t mat_cap;
};

__device__ Work carve(double* sm, int smem_doubles, int S) {
  Work w;
  double* p = sm;
  w.red = p; p += kNW * kMaxCols;
  w.vec = p; p += kMaxCols;
  w.sc3 = p; p += 4 + kMaxCols;   // [0..3] scalars, [4..] per-column scratch (dinv)
  w.tau = p; p += kMaxCols;
  w.S1 = p; p += S * S;
  w.S2 = p; p += S * S;
  w.S3 = p; p += S * S;
  w.S4 = p; p += S * (S + 1);
  w.S5 = p; p += S * S;
  w.perm = reinterpret_cast<int*>(p); p += (S + 1) / 2 + 1;
  w.ptab = reinterpret_cast<int*>(p); p += (S * S) / 2 + 1;
  w.mat = p;
  w.mat_cap = smem_doubles - (int64_t)(p - sm);
  w.diag = nullptr;
  return w;
}

// Householder QR in place of the m x n row-major matrix A (row stride ld).
template <int NM>
__device__ void qr_rows(double* A, int ld, int m, int n, const Work& w) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x;
  const int kmin = m < n ? m : n;
  for (int j = 0; j < kmin; ++j) {
    double p[NM];
#pragma unroll
    for (int c = 0; c < NM; ++c) p[c] = 0.0;
    for (int i = tid; i < m; i += T) {
      if (i <= j) continue;
      const double* row = A + (int64_t)i * ld;
      const double aij = row[j];
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c >= j && c < n) p[c] = fma(aij, row[c], p[c]);
    }
    double o0, o1;
    warp_treduce<NM>(p, lane, o0, o1);
    if (lane < NM) w.red[warp * kMaxCols + lane] = o0;
    if (NM == 64) w.red[warp * kMaxCols + 32 + lane] = o1;
    __syncthreads();
    if (warp == 0) {
      double cs0 = 0.0, cs1 = 0.0;
      for (int ww = 0; ww < kNW; ++ww) {
        if (lane < NM) cs0 += w.red[ww * kMaxCols + lane];
        if (NM == 64) cs1 += w.red[ww * kMaxCols + 32 + lane];
      }
      const double xb2 = (j < 32) ? __shfl_sync(0xffffffffu, cs0, j & 31)
                                  : __shfl_sync(0xffffffffu, cs1, j & 31);
      const double alpha = A[(int64_t)j * ld + j];
      double tau = 0.0, denom = 0.0, beta = alpha;
      if (xb2 != 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xb2), alpha);
        tau = (beta - alpha) / beta;
        denom = 1.0 / (alpha - beta);
      }
      const double* rj = A + (int64_t)j * ld;
      if (lane > j && lane < n) w.vec[lane] = tau * (rj[lane] + cs0 * denom);
      if (NM == 64 && lane + 32 > j && lane + 32 < n) w.vec[lane + 32] = tau * (rj[lane + 32] + cs1 * denom);
      if (lane == 0) {
        w.sc3[0] = tau;
        w.sc3[1] = denom;
        w.sc3[2] = beta;
        w.tau[j] = tau;
      }
    }
    __syncthreads();
    const double tau = w.sc3[0];
    if (tau != 0.0) {
      const double denom = w.sc3[1], beta = w.sc3[2];
      for (int i = tid; i < m; i += T) {
        if (i < j) continue;
        double* row = A + (int64_t)i * ld;
        const double v = (i == j) ? 1.0 : row[j] * denom;
        for (int c = j + 1; c < n; ++c) row[c] = fma(-v, w.vec[c], row[c]);
        row[j] = (i == j) ? beta : v;
      }
    }
  }
  __syncthreads();
}

// Form Q (m x k, k = min(m, n) reflectors) in place over the first k columns (dorg2r).
template <int NM>
__device__ void orgqr_rows(double* A, int ld, int m, int k, const Work& w) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x;
  for (int j = k - 1; j >= 0; --j) {
    const double tj = w.tau[j];
    if (j < k - 1 && tj != 0.0) {
      double p[NM];
#pragma unroll
      for (int c = 0; c < NM; ++c) p[c] = 0.0;
      for (int i = tid; i < m; i += T) {
        if (i <= j) continue;
        const double* row = A + (int64_t)i * ld;
        const double aij = row[j];
#pragma unroll
        for (int c = 0; c < NM; ++c)
          if (c > j && c < k) p[c] = fma(aij, row[c], p[c]);
      }
      double o0, o1;
      warp_treduce<NM>(p, lane, o0, o1);
      if (lane < NM) w.red[warp * kMaxCols + lane] = o0;
      if (NM == 64) w.red[warp * kMaxCols + 32 + lane] = o1;
      __syncthreads();
      if (warp == 0) {
        double cs0 = 0.0, cs1 = 0.0;
        for (int ww = 0; ww < kNW; ++ww) {
          if (lane < NM) cs0 += w.red[ww * kMaxCols + lane];
          if (NM == 64) cs1 += w.red[ww * kMaxCols + 32 + lane];
        }
        const double* rj = A + (int64_t)j * ld;
        if (lane > j && lane < k) w.vec[lane] = (rj[lane] + cs0) * tj;
        if (NM == 64 && lane + 32 > j && lane + 32 < k) w.vec[lane + 32] = (rj[lane + 32] + cs1) * tj;
      }
      __syncthreads();
      for (int i = tid; i < m; i += T) {
        if (i < j) continue;
        double* row = A + (int64_t)i * ld;
        const double v = (i == j) ? 1.0 : row[j];
        for (int c = j + 1; c < k; ++c) row[c] = fma(-v, w.vec[c], row[c]);
      }
    }
    for (int i = tid; i < m; i += T) {
      double* row = A + (int64_t)i * ld;
      if (i > j) row[j] *= -tj;
      else if (i == j) row[j] = 1.0 - tj;
      else row[j] = 0.0;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- CholeskyQR2
// G = A^T A (n x n, full, row stride gl) for the m x n matrix A (stride ld).  Warp w
// owns the G rows {w, n-1-w, w+nw, n-1-w-nw, ...} (balanced triangle); lane l owns the
// columns j = i + l, i + l + 32 (j >= i); 4-way unrolled over the rows of A.
__device__ void blk_gram(const double* A, int ld, int m, int n, double* G, int gl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = warp; t < n; t += nw) {
    const int i = (t & 1) ? n - 1 - (t >> 1) : (t >> 1);
    for (int j = i + lane; j < n; j += 32) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int r = 0;
      for (; r + 3 < m; r += 4) {
        const double* a0 = A + (int64_t)r * ld;
        s0 = fma(a0[i], a0[j], s0);
        s1 = fma(a0[ld + i], a0[ld + j], s1);
        s2 = fma(a0[2 * ld + i], a0[2 * ld + j], s2);
        s3 = fma(a0[3 * ld + i], a0[3 * ld + j], s3);
      }
      for (; r < m; ++r) s0 = fma(A[(int64_t)r * ld + i], A[(int64_t)r * ld + j], s0);
      const double sv = (s0 + s1) + (s2 + s3);
      G[i * gl + j] = sv;
      G[j * gl + i] = sv;
    }
  }
  __syncthreads();
}

// In-place Cholesky G = L L^T by warp 0 (lower factor, upper zeroed).  A pivot below
// 1e-14 of its original diagonal counts as breakdown (the block is too ill-conditioned
// for CholeskyQR2 and goes to Householder).  Block-uniform result.
__device__ bool blk_chol_warp(double* G, int n, int gl) {
  __shared__ int s_ok;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    bool ok = true;
    for (int j = 0; j < n; ++j) {
      const double djj = G[j * gl + j];
      __syncwarp();
      double d = 1.0;
      if (djj > 0.0 && isfinite(djj)) d = sqrt(djj);
      else ok = false;
      const double dinv = 1.0 / d;
      for (int i = j + 1 + lane; i < n; i += 32) G[i * gl + j] *= dinv;
      if (lane == 0) G[j * gl + j] = d;
      __syncwarp();
      for (int i = j + 1 + lane; i < n; i += 32) {
        const double lij = G[i * gl + j];
        for (int k = j + 1; k <= i; ++k) G[i * gl + k] = fma(-lij, G[k * gl + j], G[i * gl + k]);
      }
      __syncwarp();
    }
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, c = e - i * n;
      if (c > i) G[i * gl + c] = 0.0;
    }
    if (lane == 0) s_ok = ok ? 1 : 0;
  }
  __syncthreads();
  return s_ok != 0;
}

// A <- A L^{-T} row by row (forward substitution with the lower factor L, stride gl).
__device__ void blk_solve_rows(double* A, int ld, int m, int n, const double* L, int gl,
                               double* dinv) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) dinv[j] = 1.0 / L[j * gl + j];
  __syncthreads();
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    double* row = A + (int64_t)r * ld;
    for (int j = 0; j < n; ++j) {
      double s = row[j];
      for (int i = 0; i < j; ++i) s = fma(-row[i], L[j * gl + i], s);
      row[j] = s * dinv[j];
    }
  }
  __syncthreads();
}

// CholeskyQR2 with an orthogonality check: on success Q in A, R (n x n upper) in R.
// Returns 0 on success, 1 if the first Cholesky failed (A untouched), 2 if it failed
// later (A holds Q1 = A R1^{-1}, R holds R1): the caller finishes with Householder.
__device__ int blk_cholqr2_smem(double* A, int ld, int m, int n, double* R, const Work& w) {
  double* G = w.S4;            // n x gl, gl odd (conflict-free column walks)
  const int gl = n | 1;
  double* dinv = w.sc3 + 4;
  double* diag0 = w.vec;
  for (int pass = 0; pass < 2; ++pass) {
    blk_gram(A, ld, m, n, G, gl);
    for (int j = threadIdx.x; j < n; j += blockDim.x) diag0[j] = G[j * gl + j];
    __syncthreads();
    bool ok = blk_chol_warp(G, n, gl);
    if (ok) {
      __shared__ int s_ok2;
      if (threadIdx.x == 0) {
        int o = 1;
        for (int j = 0; j < n; ++j)
          if (!(G[j * gl + j] * G[j * gl + j] > 1e-14 * diag0[j])) o = 0;
        s_ok2 = o;
      }
      __syncthreads();
      ok = s_ok2 != 0;
    }
    if (!ok) return pass == 0 ? 1 : 2;
    blk_solve_rows(A, ld, m, n, G, gl, dinv);
    if (pass == 0) {
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e - i * n;
        R[e] = j >= i ? G[j * gl + i] : 0.0;
      }
    } else {
      double* T = w.S5;
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e - i * n;
        double acc = 0.0;
        for (int q = i; q <= j; ++q) acc = fma(G[q * gl + i], R[q * n + j], acc);
        T[e] = j >= i ? acc : 0.0;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) R[e] = T[e];
    }
    __syncthreads();
  }
  blk_gram(A, ld, m, n, G, gl);
  __shared__ int s_orth;
  if (threadIdx.x == 0) s_orth = 1;
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    const double v = G[i * gl + j] - (i == j ? 1.0 : 0.0);
    if (!(fabs(v) <= 1e-13)) s_orth = 0;
  }
  __syncthreads();
  return s_orth ? 0 : 2;
}

// max_{i,j} |G[i][j] - delta_ij| over the n x n block (stride gl); CTA-uniform result.
__device__ __noinline__ double blk_max_dev_identity(const double* G, int gl, int n, double* red) {
  double mx = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    const double v = fabs(G[i * gl + j] - (i == j ? 1.0 : 0.0));
    mx = (v > mx || v != v) ? v : mx;                       // NaN propagates
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (t > mx || t != t) ? t : mx;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  double r = 0.0;
  for (int wv = 0; wv < (int)(blockDim.x >> 5); ++wv) r = (red[wv] > r || red[wv] != red[wv]) ? red[wv] : r;
  __syncthreads();
  return r;
}

// Adaptive shifted CholeskyQR on FP64 tensor cores (n <= 32).  Pass p: G = A^T A (DMMA);
// for p >= 1, if |G - I| <= 1e-8 finish with the first-order factor (exact to rounding,
// see below) and return; else factor G + s_p I = L L^T (CTA Cholesky; s_0 =
// 11 (mn + n(n+1)) u ||A||_F^2 makes pass 0 succeed for any condition number up to 1/u
// [shifted CholeskyQR3, Fukaya et al. 2020], s_p = 0 afterwards), Li = L^{-1},
// A <- A Li^T (DMMA), R <- L^T R.  Returns 0 on success, 1 on a breakdown (A untouched
// only if it happened in pass 0), 2 if not certified after 4 passes (caller finishes
// with Householder from the partial result).
__device__ int blk_cholqr2(double* A, int ld, int m, int n, double* R, const Work& w) {
  if (n > 32) return blk_cholqr2_smem(A, ld, m, n, R, w);   // (mma_mul_rt_inplace: n <= 32)
  double* G = w.S4;
  const int gl = n | 1;
  double* Li = w.S5;            // n x il
  const int il = n | 1;
  for (int pass = 0; pass < 4; ++pass) {
    mma_gemm(n, n, m,
             [&](int i, int k) { return i < n ? A[(int64_t)k * ld + i] : 0.0; },
             [&](int k, int j) { return j < n ? A[(int64_t)k * ld + j] : 0.0; },
             [&](int i, int j, double v) { if (i < n && j < n) G[i * gl + j] = v; });
    __syncthreads();
    if (pass > 0) {
      const double dev = blk_max_dev_identity(G, gl, n, w.red);
      if (dev <= 1e-8) {
        // G = Q^T Q = I + E, |E| <= 1e-8: chol(G) = I + L1 + O(E^2), L1 = tril(E,-1) +
        // diag(E)/2, inverse I - L1 + O(E^2); O(E^2) <= 1e-16 is below rounding.
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
          const int i = e / n, j = e - i * n;
          double l1 = 0.0;
          if (j < i) l1 = G[i * gl + j];
          else if (j == i) l1 = 0.5 * (G[i * gl + i] - 1.0);
          Li[i * il + j] = (i == j ? 1.0 : 0.0) - l1;
          w.S3[e] = (i == j ? 1.0 : 0.0) + l1;
        }
        __syncthreads();
        mma_mul_rt_inplace(A, ld, m, n, Li, il);
        double* T = w.S4;
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
          const int i = e / n, j = e - i * n;
          double acc = 0.0;
          for (int q = i; q <= j; ++q) acc = fma(w.S3[q * n + i], R[q * n + j], acc);
          T[e] = j >= i ? acc : 0.0;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) R[e] = T[e];
        __syncthreads();
        return 0;
      }
      if (!(dev <= 1e6)) return 2;
    }
    if (pass == 0) {
      __shared__ double s_shift;
      if (threadIdx.x == 0) {
        double tr = 0.0;
        for (int j = 0; j < n; ++j) tr += G[j * gl + j];
        s_shift = 11.0 * ((double)m * n + (double)n * (n + 1)) * 1.1102230246251565e-16 * tr;
      }
      __syncthreads();
      for (int j = threadIdx.x; j < n; j += blockDim.x) G[j * gl + j] += s_shift;
      __syncthreads();
    }
    const bool ok = chol_cta(G, gl, n, w.sc3 + 4);
    if (!ok) return pass == 0 ? 1 : 2;
    trinv_cta(G, gl, n, Li, il);
    mma_mul_rt_inplace(A, ld, m, n, Li, il);
    if (pass == 0) {
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e - i * n;
        R[e] = j >= i ? G[j * gl + i] : 0.0;
      }
    } else {
      double* T = w.S3;
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e - i * n;
        double acc = 0.0;
        for (int q = i; q <= j; ++q) acc = fma(G[q * gl + i], R[q * n + j], acc);
        T[e] = j >= i ? acc : 0.0;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) R[e] = T[e];
    }
    __syncthreads();
  }
  return 2;
}

// QR of the m x n matrix staged at A (stride ld): R (kmin x n, row-major, zeros below
// the diagonal) into Rout, Q in place over the first kmin columns.  Returns kmin.
// Tall blocks (m >= n) try CholeskyQR2 first (O(1) barriers); ill-conditioned or wide
// blocks use Householder (LAPACK conventions), continuing from CholeskyQR2's partial
// result when it failed late (A = Q1, R = R1  =>  A_orig = Q (R_h R1)).
__device__ __noinline__ void householder_explicit(double* A, int ld, int m, int n, double* Rout, const Work& w) {
  const int kmin = m < n ? m : n;
  if (n <= 8) qr_rows<8>(A, ld, m, n, w);
  else if (n <= 16) qr_rows<16>(A, ld, m, n, w);
  else if (n <= 32) qr_rows<32>(A, ld, m, n, w);
  else qr_rows<64>(A, ld, m, n, w);
  for (int e = threadIdx.x; e < kmin * n; e += blockDim.x) {
    const int a = e / n, b = e - a * n;
    Rout[e] = b >= a ? A[(int64_t)a * ld + b] : 0.0;
  }
  __syncthreads();
  if (kmin <= 8) orgqr_rows<8>(A, ld, m, kmin, w);
  else if (kmin <= 16) orgqr_rows<16>(A, ld, m, kmin, w);
  else if (kmin <= 32) orgqr_rows<32>(A, ld, m, kmin, w);
  else orgqr_rows<64>(A, ld, m, kmin, w);
}

__device__ int qr_explicit(double* A, int ld, int m, int n, double* Rout, const Work& w) {
  const int kmin = m < n ? m : n;
  if (m >= n) {
    const int st = blk_cholqr2(A, ld, m, n, Rout, w);
    if (threadIdx.x == 0 && w.diag) w.diag[st == 0 ? 6 : (st == 1 ? 7 : 5)] += 1;   // diagnostic
    if (st == 0) return kmin;
    if (st == 2) {
      // finish: Q1 = Q_h R_h  =>  A_orig = Q_h (R_h R1)
      double* R1 = w.S5;
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) R1[e] = Rout[e];
      __syncthreads();
      double* Rh = w.S4;
      householder_explicit(A, ld, m, n, Rh, w);
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e - i * n;
        double acc = 0.0;
        for (int q = i; q <= j; ++q) acc = fma(Rh[i * n + q], R1[q * n + j], acc);
        Rout[e] = j >= i ? acc : 0.0;
      }
      __syncthreads();
      return kmin;
    }
  }
  householder_explicit(A, ld, m, n, Rout, w);
  return kmin;
}

// In-place Cholesky of the R x R SPD matrix P (row-major), lower factor; false on
// breakdown (block-uniform).
__device__ bool blk_chol(double* P, int R) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  for (int j = 0; j < R; ++j) {
    if (threadIdx.x == 0) {
      double dd = P[j * R + j];
      for (int c = 0; c < j; ++c) dd -= P[j * R + c] * P[j * R + c];
      if (!(dd > 0.0) || !isfinite(dd)) {
        s_ok = 0;
        dd = 1.0;
      }
      P[j * R + j] = sqrt(dd);
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < R; i += blockDim.x) {
      double v = P[i * R + j];
      for (int c = 0; c < j; ++c) v -= P[i * R + c] * P[j * R + c];
      P[i * R + j] = v / P[j * R + j];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, c = e - i * R;
    if (c > i) P[e] = 0.0;
  }
  __syncthreads();
  return s_ok != 0;
}

// One-sided Jacobi on the columns of X (rows x kc, column-major X[c*rows + i]),
// accumulating V (kc x kc, column-major).  Round-robin ordering from a precomputed
// pair table, one warp per pair; column norms are kept in shared memory and updated
// by the exact rotation identities (a' = a - t g, b' = b + t g), recomputed per sweep.
__device__ __noinline__ bool blk_jacobi(double* X, int rows, int kc, double* V, int* sweeps, double* nrm,
                           int* ptab) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __shared__ int s_rot;
  for (int e = tid; e < kc * kc; e += blockDim.x) V[e] = (e / kc == e % kc) ? 1.0 : 0.0;
  if (kc < 2) {
    __syncthreads();
    return true;
  }
  const int kp = kc + (kc & 1);
  const int npairs = kp / 2;
  for (int e = tid; e < (kp - 1) * npairs; e += blockDim.x) {
    const int round = e / npairs, pr = e - round * npairs;
    int a = pr == 0 ? 0 : ((pr - 1 + round) % (kp - 1)) + 1;
    const int q = kp - 1 - pr;
    int b = q == 0 ? 0 : ((q - 1 + round) % (kp - 1)) + 1;
    if (a > b) { const int t = a; a = b; b = t; }
    ptab[2 * e] = a;
    ptab[2 * e + 1] = b;
  }
  const double tol = 2.3e-16 * sqrt((double)(rows > 1 ? rows : 1));
  const double tol2 = tol * tol;
  __shared__ unsigned long long s_maxoff;   // max (gamma^2 / (alpha beta)) of the sweep, as bits
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) {
      s_rot = 0;
      s_maxoff = 0ull;
      if (sweeps) atomicAdd(sweeps, 1);
    }
    __syncthreads();
    for (int c = warp; c < kc; c += nw) {
      double s = 0.0;
      for (int i = lane; i < rows; i += 32) s = fma(X[c * rows + i], X[c * rows + i], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += shx(s, o);
      if (lane == 0) nrm[c] = s;
    }
    __syncthreads();
    for (int round = 0; round < kp - 1; ++round) {
      const int* pt = ptab + 2 * round * npairs;
      const int hw = tid >> 4, hl = tid & 15, nhw = blockDim.x >> 4;   // half-warp per pair
      for (int pr0 = 0; pr0 < npairs; pr0 += nhw) {
        const int pr = pr0 + hw;
        const bool act = pr < npairs;
        int a = 0, b = 0;
        if (act) {
          a = pt[2 * pr];
          b = pt[2 * pr + 1];
        }
        const bool live = act && b < kc;
        double* xa = X + (int64_t)a * rows;
        double* xb = X + (int64_t)b * rows;
        double ga = 0.0;
        if (live)
          for (int i = hl; i < rows; i += 16) ga = fma(xa[i], xb[i], ga);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
        if (live) {
          const double al = nrm[a], be = nrm[b];
          if (hl == 0 && ga != 0.0) {
            const double rel = (ga * ga) / (al * be);
            atomicMax(&s_maxoff, __double_as_longlong(rel > 0.0 ? rel : 0.0));
          }
          if (ga != 0.0 && ga * ga > tol2 * (al * be)) {
            const double dlt = be - al;
            const double sg = (dlt > 0.0 || (dlt == 0.0 && !signbit(dlt))) ? 1.0 : -1.0;
            const double t = (2.0 * ga * sg) / (fabs(dlt) + sqrt(fma(dlt, dlt, 4.0 * ga * ga)));
            const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
            for (int i = hl; i < rows; i += 16) {
              const double u = xa[i], v = xb[i];
              xa[i] = c * u - sn * v;
              xb[i] = sn * u + c * v;
            }
            double* va = V + (int64_t)a * kc;
            double* vb = V + (int64_t)b * kc;
            for (int i = hl; i < kc; i += 16) {
              const double u = va[i], v = vb[i];
              va[i] = c * u - sn * v;
              vb[i] = sn * u + c * v;
            }
            if (hl == 0) {
              nrm[a] = al - t * ga;
              nrm[b] = be + t * ga;
              s_rot = 1;
            }
          }
        }
      }
      __syncthreads();
    }
    const int rot = s_rot;
    const double maxoff = __longlong_as_double((long long)s_maxoff);
    __syncthreads();
    // Converged when no rotation was needed, or when the largest relative off-diagonal
    // of this sweep was <= 1e-10: cyclic Jacobi converges quadratically, so after such a
    // sweep the residual is ~1e-20, far below tol (no verification sweep needed).
    if (!rot || maxoff <= 1e-20) return true;
  }
  return false;
}

// Norms of the kc columns of X (rows x kc col-major) into nrm, and the permutation
// perm sorting them by norm (descending, ties by index).  Ends with a barrier.
__device__ __noinline__ void col_norms_sorted(const double* X, int rows, int kc, double* nrm, int* perm) {
  __builtin_assume(__isShared(X));
  __builtin_assume(__isShared(nrm));
  __builtin_assume(__isShared(perm));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < kc; c += nw) {
    double s = 0.0;
    for (int i = lane; i < rows; i += 32) s = fma(X[c * rows + i], X[c * rows + i], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += shx(s, o);
    if (lane == 0) nrm[c] = s;
  }
  __syncthreads();
  if (threadIdx.x < kc) {
    const int c = threadIdx.x;
    const double v = nrm[c];
    int rank = 0;
    for (int c2 = 0; c2 < kc; ++c2) rank += (nrm[c2] > v) || (nrm[c2] == v && c2 < c);
    perm[rank] = c;
  }
  __syncthreads();
}

__device__ void blk_copy(double* dst, const double* src, int64_t n) {
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) dst[e] = src[e];
}

// Row stride of staged matrices: >= n and = 4 (mod 16).  DMMA fragment loads read 4 rows
// x 8 consecutive columns per half-warp; (4 tq + gid) mod 16 is then distinct for all 16
// lanes of a half-warp, i.e. bank-conflict free.
__device__ __forceinline__ int odd_ld(int n) { return n <= 4 ? 4 : ((n + 11) / 16) * 16 + 4; }

// Phase timer (thread 0): cyc[ph] += clock64() - t0.  Diagnostic only.
struct PhaseClock {
  long long t0;
  __device__ void start() { t0 = clock64(); }
  __device__ void stop(Scalars* sc, int ph) {
    if (threadIdx.x == 0) sc->cyc[ph] += clock64() - t0;
  }
};

__global__ void __launch_bounds__(kDenseThreads) k_dense_orth(DenseArgs a) {
  extern __shared__ double smraw[];
  Scalars* sc = a.sc;
  if (sc->noop) return;
  const int d = a.d;
  int S = 2;
  for (int k = 0; k <= d; ++k) S = a.r[k] > S ? a.r[k] : S;
  Work w = carve(smraw, a.smem_doubles, S);
  w.diag = sc->cyc;
  // A4: U_k = phi_k (.)_2 C_k
  for (int k = 0; k < d; ++k) {
    const int r0 = a.r[k], nk = a.n[k], r1 = a.r[k + 1];
    const int tot = r0 * nk * r1;
    const double* C = a.C + a.core_off[k];
    double* U = a.U + a.core_off[k];
    const double* ph = a.phi + a.phi_off[k];
    for (int e = threadIdx.x; e < tot; e += blockDim.x) U[e] = C[e] * ph[(e / r1) % nk];
  }
  __syncthreads();
  // A5: U_k <- Q, U_{k+1} <- R U_{k+1}
  double* gw = a.work;
  PhaseClock pc;
  pc.start();
  for (int k = 0; k + 1 < d; ++k) {
    const int r0 = a.r[k], nk = a.n[k], r1 = a.r[k + 1];
    const int m = r0 * nk;
    double* U = a.U + a.core_off[k];
    int ld = odd_ld(r1);
    double* A = w.mat;
    if ((int64_t)m * ld > w.mat_cap) {
      A = gw;
      ld = r1;
    }
    for (int e = threadIdx.x; e < m * r1; e += blockDim.x) {
      const int i = e / r1, c = e - i * r1;
      A[(int64_t)i * ld + c] = U[e];
    }
    __syncthreads();
    qr_explicit(A, ld, m, r1, w.S1, w);   // kmin = r1 (feasible ranks)
    for (int e = threadIdx.x; e < m * r1; e += blockDim.x) {
      const int i = e / r1, c = e - i * r1;
      U[e] = A[(int64_t)i * ld + c];
    }
    double* Un = a.U + a.core_off[k + 1];
    const int rest = a.n[k + 1] * a.r[k + 2];
    __syncthreads();
    double* st = ((int64_t)r1 * rest <= w.mat_cap) ? w.mat : gw + (int64_t)m * ld;
    blk_copy(st, Un, (int64_t)r1 * rest);        // stage U_{k+1} (coalesced)
    __syncthreads();
    {
      const double* Rr = w.S1;
      mma_gemm(r1, rest, r1,                         // U_{k+1} <- R U_{k+1}
               [&](int i, int q) { return i < r1 ? Rr[i * r1 + q] : 0.0; },
               [&](int q, int j) { return j < rest ? st[(int64_t)q * rest + j] : 0.0; },
               [&](int i, int j, double v) { if (i < r1 && j < rest) Un[(int64_t)i * rest + j] = v; });
    }
    __syncthreads();
  }
  pc.stop(sc, 5);
  pc.start();
  // A6: P_{d-1} = [1]; P_k = sum_j U_{k+1}(:,j,:) P_{k+1} U_{k+1}(:,j,:)^T; Cholesky.
  if (threadIdx.x == 0) {
    a.P[a.p_off[d - 1]] = 1.0;
    a.L[a.p_off[d - 1]] = 1.0;
  }
  __syncthreads();
  bool ok = true;
  for (int k = d - 2; k >= 0; --k) {
    const int R1 = a.r[k + 1], nk = a.n[k + 1], R2 = a.r[k + 2];
    const int t1 = R1 * nk * R2;
    const bool fits = 2 * (int64_t)t1 + R2 * R2 <= w.mat_cap;
    double* Un = fits ? w.mat : a.U + a.core_off[k + 1];
    double* T1 = fits ? w.mat + t1 : gw;
    double* Pn = fits ? w.mat + 2 * t1 : a.P + a.p_off[k + 1];
    if (fits) {
      blk_copy(Un, a.U + a.core_off[k + 1], t1);
      blk_copy(Pn, a.P + a.p_off[k + 1], R2 * R2);
      __syncthreads();
    }
    for (int e = threadIdx.x; e < t1; e += blockDim.x) {
      const int aj = e / R2, ee = e - aj * R2;
      double acc = 0.0;
      for (int c = 0; c < R2; ++c) acc = fma(Un[aj * R2 + c], Pn[c * R2 + ee], acc);
      T1[e] = acc;
    }
    __syncthreads();
    double* P = a.P + a.p_off[k];
    const int len = nk * R2;
    {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      for (int aa = warp; aa < R1; aa += kNW) {
        double pv[32];
#pragma unroll
        for (int bb = 0; bb < 32; ++bb) pv[bb] = 0.0;
        for (int q = lane; q < len; q += 32) {
          const double t = T1[aa * len + q];
#pragma unroll
          for (int bb = 0; bb < 32; ++bb)
            if (bb < R1) pv[bb] = fma(t, Un[bb * len + q], pv[bb]);
        }
        double o0, o1;
        warp_treduce<32>(pv, lane, o0, o1);
        if (lane < R1) P[aa * R1 + lane] = o0;
      }
    }
    __syncthreads();
    double* Ls = w.S1;
    for (int e = threadIdx.x; e < R1 * R1; e += blockDim.x) {
      const int aa = e / R1, bb = e - aa * R1;
      Ls[e] = 0.5 * (P[aa * R1 + bb] + P[bb * R1 + aa]);
    }
    __syncthreads();
    ok = blk_chol(Ls, R1) && ok;
    blk_copy(a.L + a.p_off[k], Ls, (int64_t)R1 * R1);
    __syncthreads();
  }
  pc.stop(sc, 4);
  if (!ok && threadIdx.x == 0) {
    atomicOr(&sc->err, (int)kErrChol);
    sc->noop = 1;
  }
}

// z = (L L^T)^{-1} y for one row (r1 <= R): forward then back substitution in registers.
template <int R>
__device__ __forceinline__ void proj_solve_row(const double* y, double* z, const double* Ls, int r1) {
  double zv[R];
#pragma unroll
  for (int i = 0; i < R; ++i) zv[i] = i < r1 ? y[i] : 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (i < r1) {
      double sacc = zv[i];
#pragma unroll
      for (int c = 0; c < i; ++c) sacc = fma(-Ls[i * r1 + c], zv[c], sacc);
      zv[i] = sacc / Ls[i * r1 + i];
    }
  }
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    if (i < r1) {
      double sacc = zv[i];
#pragma unroll
      for (int c = i + 1; c < R; ++c)
        if (c < r1) sacc = fma(-Ls[c * r1 + i], zv[c], sacc);
      zv[i] = sacc / Ls[i * r1 + i];
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (i < r1) z[i] = zv[i];
}

// One CTA per core k: projection (A10), unweighting (A11), assembly of B_k (A13).
__global__ void __launch_bounds__(kProjThreads) k_project(DenseArgs a) {
  extern __shared__ double smraw[];
  Scalars* sc = a.sc;
  if (sc->noop) return;
  const int d = a.d, k = blockIdx.x;
  const double alpha = sc->alpha;
  const int r0 = a.r[k], nk = a.n[k], r1 = a.r[k + 1];
  const int m = r0 * nk;
  const double* Y = a.Y + a.core_off[k];
  const double* U = a.U + a.core_off[k];
  double* Ah = a.Ahat + a.core_off[k];
  if (a.proj_mode == 2) {
    // assembly only: Ahat from the projection launch, alpha from the adaptive step
  } else if (k == d - 1) {
    blk_copy(Ah, Y, (int64_t)m * r1);
    __syncthreads();
  } else {
    double* Ls = smraw;                       // r1 x r1
    double* W = Ls + r1 * r1;                 // r1 x r1
    double* Z = W + r1 * r1;                  // m x ld (staged) or Ah
    const int ld = r1 | 1;                    // odd: row-per-thread substitutions below
    const bool stage = (int64_t)m * ld * 2 + 2 * r1 * r1 + kProjThreads <= a.smem_doubles;
    double* Us = stage ? Z + (int64_t)m * ld : nullptr;
    const int zld = stage ? ld : r1;
    if (!stage) Z = Ah;
    blk_copy(Ls, a.L + a.p_off[k], (int64_t)r1 * r1);
    if (stage)
      for (int e = threadIdx.x; e < m * r1; e += blockDim.x) {
        const int i = e / r1, c = e - i * r1;
        Us[(int64_t)i * ld + c] = U[e];
      }
    __syncthreads();
    // Z = L(Y_k) P_k^{-1}: per row, forward then back substitution with L L^T
    if (stage) {
      for (int e = threadIdx.x; e < m * r1; e += blockDim.x) {
        const int i = e / r1, c = e - i * r1;
        Z[(int64_t)i * ld + c] = Y[e];          // stage Y (coalesced); solve in place
      }
      __syncthreads();
    }
    // per row, in registers (the same operation order as a textbook forward / back solve)
    for (int row = threadIdx.x; row < m; row += blockDim.x) {
      const double* y = stage ? Z + (int64_t)row * zld : Y + (int64_t)row * r1;
      double* z = Z + (int64_t)row * zld;
      if (r1 <= 16) proj_solve_row<16>(y, z, Ls, r1);
      else proj_solve_row<kMaxRank>(y, z, Ls, r1);
    }
    __syncthreads();
    // W = L(U_k)^T Z  (r1 x r1): thread groups take interleaved rows, partials summed in
    // group order (fixed)
    const double* Uv = stage ? Us : U;
    const int uld = stage ? ld : r1;
    const int rr = r1 * r1;
    const int ngrp = (int)blockDim.x / rr > 0 ? (int)blockDim.x / rr : 1;
    double* Wp = smraw + 2 * rr + (stage ? 2 * (int64_t)m * ld : 0);   // ngrp x rr partials
    for (int e = threadIdx.x; e < ngrp * rr; e += blockDim.x) {
      const int gi = e / rr, el = e - gi * rr;
      const int aa = el / r1, bb = el - aa * r1;
      // four interleaved accumulators, eight rows' loads in flight (a single dependent chain
      // over m / ngrp rows of L2 loads was 0.66 ms at config 3's 4096-row core)
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int row = gi;
      for (; row + 7 * ngrp < m; row += 8 * ngrp) {
        double u[8], z[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          u[q] = Uv[(int64_t)(row + q * ngrp) * uld + aa];
          z[q] = Z[(int64_t)(row + q * ngrp) * zld + bb];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q & 3] = fma(u[q], z[q], acc[q & 3]);
      }
      for (int q = 0; row < m; row += ngrp, ++q)
        acc[q & 3] = fma(Uv[(int64_t)row * uld + aa], Z[(int64_t)row * zld + bb], acc[q & 3]);
      Wp[e] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rr; e += blockDim.x) {
      double acc = 0.0;
      for (int gi = 0; gi < ngrp; ++gi) acc += Wp[gi * rr + e];
      W[e] = acc;
    }
    __syncthreads();
    // Ahat = Z - L(U_k) W   (when Z aliases Ah each thread reads/writes only its slot)
    for (int e = threadIdx.x; e < m * r1; e += blockDim.x) {
      const int row = e / r1, bb = e - row * r1;
      double acc = 0.0;
      for (int aa = 0; aa < r1; ++aa) acc = fma(Uv[(int64_t)row * uld + aa], W[aa * r1 + bb], acc);
      Ah[e] = Z[(int64_t)row * zld + bb] - acc;
    }
    __syncthreads();
  }
  if (a.proj_mode == 1) {
    // adaptive step numerator: the W-norm of component k of the tangent
    // vector, ||[U_1..Ahat_k..U_d]||_F^2 = tr(L(Ahat_k) P_k L(Ahat_k)^T) = ||L(Ahat_k) chol(P_k)||^2
    // (left part orthonormal; P_d = [1]); fixed-order CTA reduction
    double acc = 0.0;
    const double* Lk = a.L + a.p_off[k];
    for (int row = threadIdx.x; row < m; row += blockDim.x) {
      const double* ar = Ah + (int64_t)row * r1;
      if (k == d - 1) {
        for (int c = 0; c < r1; ++c) acc = fma(ar[c], ar[c], acc);
      } else {
        for (int c = 0; c < r1; ++c) {
          double v = 0.0;
          for (int i = c; i < r1; ++i) v = fma(ar[i], Lk[i * r1 + c], v);
          acc = fma(v, v, acc);
        }
      }
    }
    double* red = smraw;
    __syncthreads();
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) sc->adapt_num[k] = red[0];
    return;
  }
  // A11 + A13: B_k from Ttil = U/phi and X = -alpha Ahat/phi.  With the weighted retraction
  // the rounding acts on W^{1/2} W_l, i.e. on the same blocks without the
  // 1/phi slice scaling (Prop. 3.1: W^{1/2} scales mode-k slices by phi); k_unweight_out
  // applies W^{-1/2} to the rounded cores.
  const double* ph = a.phi + a.phi_off[k];
  const bool wr = a.wretr != 0;
  double* B = a.B + a.b_off[k];
  // 1 / phi_{k,x} once per slice (a reciprocal per element was the assembly's cost at config 3)
  double* invp = smraw;
  const bool inv_sm = nk <= a.smem_doubles;
  if (inv_sm)
    for (int x = threadIdx.x; x < nk; x += blockDim.x) invp[x] = wr ? 1.0 : 1.0 / ph[x];
  __syncthreads();
  auto inv_of = [&](int x) { return inv_sm ? invp[x] : (wr ? 1.0 : 1.0 / ph[x]); };
  if (k == 0) {
    const int Rb1 = 2 * r1;
    for (int e = threadIdx.x; e < nk * Rb1; e += blockDim.x) {
      const int x = e / Rb1, c = e - x * Rb1;
      const double inv = inv_of(x);
      B[e] = c < r1 ? -alpha * Ah[x * r1 + c] * inv : U[x * r1 + (c - r1)] * inv;
    }
  } else if (k == d - 1) {
    for (int e = threadIdx.x; e < 2 * r0 * nk; e += blockDim.x) {
      const int aa = e / nk, x = e - aa * nk;
      const double inv = inv_of(x);
      B[e] = aa < r0 ? U[aa * nk + x] * inv
                     : (U[(aa - r0) * nk + x] - alpha * Ah[(aa - r0) * nk + x]) * inv;
    }
  } else {
    // one thread per source entry (a, x, c) of U / Ahat writes its four B_k entries
    // [[U, 0], [-alpha Ahat, U]] / phi; four entries per thread in flight (one CTA per core:
    // the 16 x 256 x 16 core of config 3 was latency-bound here)
    const int Rb1 = 2 * r1;
    const int tot = r0 * nk * r1;
    const int64_t half = (int64_t)r0 * nk * Rb1;   // offset of the bottom block row
    for (int e0 = threadIdx.x; e0 < tot; e0 += 4 * blockDim.x) {
      double u[4], h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = e0 + q * blockDim.x;
        u[q] = e < tot ? U[e] : 0.0;
        h[q] = e < tot ? Ah[e] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = e0 + q * blockDim.x;
        if (e >= tot) break;
        const int c = e % r1, ax = e / r1, x = ax % nk;
        const double inv = inv_of(x);
        const int64_t o = (int64_t)ax * Rb1 + c;     // (a, x, c) in the top block row
        B[o] = u[q] * inv;
        B[o + r1] = 0.0;
        B[half + o] = -alpha * h[q] * inv;
        B[half + o + r1] = u[q] * inv;
      }
    }
  }
}

__global__ void __launch_bounds__(kDenseThreads) k_dense_round(DenseArgs a) {
  extern __shared__ double smraw[];
  Scalars* sc = a.sc;
  if (sc->noop) return;
  const int d = a.d;
  int S = 2;
  for (int k = 0; k <= d; ++k) S = 2 * a.r[k] > S ? 2 * a.r[k] : S;
  Work w = carve(smraw, a.smem_doubles, S);
  w.diag = sc->cyc;
  double* gw = a.work;
  __shared__ int curR[kMaxD + 1];
  if (threadIdx.x == 0) {
    curR[0] = 1;
    for (int k = 1; k < d; ++k) curR[k] = 2 * a.r[k];
    curR[d] = 1;
  }
  __syncthreads();
  // ---- (i) right-to-left: R(B_k)^T = Q R, B_k <- Q^T, B_{k-1} <- B_{k-1} x_3 R^T
  for (int k = d - 1; k >= 1; --k) {
    const int R0 = curR[k], nk = a.n[k], R1 = curR[k + 1];
    const int rows = nk * R1, cols = R0;
    double* B = a.B + a.b_off[k];
    int ld = odd_ld(cols);
    double* A = w.mat;
    if ((int64_t)rows * ld > w.mat_cap) {
      A = gw;
      ld = cols;
    }
    for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
      const int aa = e / rows, i = e - aa * rows;      // B[aa][i], coalesced read
      A[(int64_t)i * ld + aa] = B[e];
    }
    __syncthreads();
    PhaseClock pc;
    pc.start();
    const int kmin = qr_explicit(A, ld, rows, cols, w.S1, w);
    pc.stop(sc, 0);
    pc.start();
    for (int e = threadIdx.x; e < kmin * rows; e += blockDim.x) {
      const int aa = e / rows, i = e - aa * rows;
      B[e] = A[(int64_t)i * ld + aa];
    }
    double* Bp = a.B + a.b_off[k - 1];
    const int prow = curR[k - 1] * a.n[k - 1];
    __syncthreads();
    double* st = ((int64_t)prow * R0 <= w.mat_cap) ? w.mat : gw + (int64_t)rows * ld;
    blk_copy(st, Bp, (int64_t)prow * R0);           // stage B_{k-1} (coalesced)
    __syncthreads();
    {
      const double* Rr = w.S1;                      // R: kmin x R0 row-major
      mma_gemm(prow, kmin, R0,                      // B_{k-1} <- B_{k-1} x_3 R^T
               [&](int i, int q) { return i < prow ? st[(int64_t)i * R0 + q] : 0.0; },
               [&](int q, int j) { return j < kmin ? Rr[j * R0 + q] : 0.0; },
               [&](int i, int j, double v) { if (i < prow && j < kmin) Bp[(int64_t)i * kmin + j] = v; });
    }
    if (threadIdx.x == 0) curR[k] = kmin;
    __syncthreads();
    pc.stop(sc, 1);
  }
  // ---- (ii) left-to-right truncated SVD sweep
  bool ok = true;
  for (int k = 0; k + 1 < d; ++k) {
    const int R0 = curR[k], nk = a.n[k], R1 = curR[k + 1];
    const int m = R0 * nk;
    const int rk = a.r[k + 1];
    double* B = a.B + a.b_off[k];
    int ld = odd_ld(R1);
    double* A = w.mat;
    if ((int64_t)m * ld > w.mat_cap) {
      A = gw;
      ld = R1;
    }
    for (int e = threadIdx.x; e < m * R1; e += blockDim.x) {
      const int i = e / R1, c = e - i * R1;
      A[(int64_t)i * ld + c] = B[e];
    }
    __syncthreads();
    double* X = w.S2;
    PhaseClock pc;
    pc.start();
    const int kmin = qr_explicit(A, ld, m, R1, X, w);   // X <- R (kmin x R1) row-major
    pc.stop(sc, 2);
    // the same storage read column-major (R1 x kmin) is X = R^T
    double* V = w.S3;
    pc.start();
    ok = blk_jacobi(X, R1, kmin, V, &sc->pad, w.red, w.ptab) && ok;
    col_norms_sorted(X, R1, kmin, w.red, w.perm);     // kept columns: perm[0..rk)
    pc.stop(sc, 3);
    pc.start();
    // C'_k = Q V[:, perm[:rk]]  (m x rk) on DMMA
    double* Cout = a.C + a.core_off[k];
    {
      const int* perm = w.perm;
      mma_gemm(m, rk, kmin,
               [&](int i, int q) { return i < m ? A[(int64_t)i * ld + q] : 0.0; },
               [&](int q, int j) { return j < rk && j < kmin ? V[perm[j] * kmin + q] : 0.0; },
               [&](int i, int j, double v) { if (i < m && j < rk) Cout[(int64_t)i * rk + j] = v; });
    }
    double* SV = w.S1;                              // (S V^T)_r: row a' = X[:, perm[a']]^T
    for (int e = threadIdx.x; e < rk * R1; e += blockDim.x) {
      const int ap = e / R1, i = e - ap * R1;
      SV[e] = ap < kmin ? X[w.perm[ap] * R1 + i] : 0.0;
    }
    __syncthreads();
    double* Bn = a.B + a.b_off[k + 1];
    const int rest = a.n[k + 1] * curR[k + 2];
    double* st = ((int64_t)R1 * rest <= w.mat_cap) ? w.mat : gw + (int64_t)m * ld;
    blk_copy(st, Bn, (int64_t)R1 * rest);           // stage B_{k+1} (coalesced)
    __syncthreads();
    mma_gemm(rk, rest, R1,                          // B_{k+1} <- (S V^T)_r x_1 B_{k+1}
             [&](int i, int q) { return i < rk ? SV[i * R1 + q] : 0.0; },
             [&](int q, int j) { return j < rest ? st[(int64_t)q * rest + j] : 0.0; },
             [&](int i, int j, double v) { if (i < rk && j < rest) Bn[(int64_t)i * rest + j] = v; });
    if (threadIdx.x == 0) curR[k + 1] = rk;
    __syncthreads();
    pc.stop(sc, 4);
  }
  blk_copy(a.C + a.core_off[d - 1], a.B + a.b_off[d - 1], (int64_t)curR[d - 1] * a.n[d - 1]);
  __syncthreads();
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int64_t e = threadIdx.x; e < a.core_off[d]; e += blockDim.x)
    if (!isfinite(a.C[e])) s_bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_bad) atomicOr(&sc->err, (int)kErrNaN);
    if (!ok) atomicOr(&sc->err, (int)kErrSVD);
  }
}

#include "round_cs.inc"

// Weighted retraction, last step: T_{l+1} = W^{-1/2} SVD_r^tt(W^{1/2} W_l),
// the rounded cores' mode-2 slices divided by phi (Prop. 3.1).  One CTA per core.
__global__ void k_unweight_out(DenseArgs a) {
  if (a.sc->noop) return;
  const int k = blockIdx.x;
  const int r0 = a.r[k], nk = a.n[k], r1 = a.r[k + 1];
  double* C = a.C + a.core_off[k];
  const double* ph = a.phi + a.phi_off[k];
  for (int64_t e = threadIdx.x; e < (int64_t)r0 * nk * r1; e += blockDim.x) {
    const int64_t x = (e / r1) % nk;
    C[e] = C[e] / ph[x];
  }
}

}  // namespace

int dense_smem_doubles() { return (200 * 1024) / 8; }

void dense_init() {
  const int bytes = dense_smem_doubles() * (int)sizeof(double);
  cudaFuncSetAttribute(k_dense_orth, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_dense_round, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_project, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  round_cs_init(bytes);
}

int round_cluster_size() { return kNC; }

bool round_cluster_ok(int d, const int* r) {
  int S = 2;
  for (int k = 0; k <= d; ++k) S = 2 * r[k] > S ? 2 * r[k] : S;
  return S <= 32;
}

// A4-A6 on one CTA (Householder sweep) when every unfolding is tiny: measured faster than the
// 8-CTA cluster (cluster barriers per stage) for configs 1, 4 and 6 (dense_orth 0.041 / 0.382 /
// 0.139 ms -> 0.028 / 0.336 / 0.103), equal for config 2 (r_{k-1} n_k = 250).
bool orth_one_cta(const DenseArgs& a) {
  int mx = 0;
  for (int k = 0; k < a.d; ++k) mx = a.r[k] * a.n[k] > mx ? a.r[k] * a.n[k] : mx;
  return mx <= 64;
}

// True when A4-A6 run on the cluster kernel, the only one that takes a split launch
// (DenseArgs::orth_part).
bool orth_cluster_ok(const DenseArgs& a) {
  int S = 2;
  for (int k = 0; k <= a.d; ++k) S = a.r[k] > S ? a.r[k] : S;
  return a.clw != nullptr && S <= 32 && !orth_one_cta(a);
}

void launch_dense_orth(cudaStream_t s, const DenseArgs& a, int64_t* launches) {
  const size_t bytes = (size_t)a.smem_doubles * sizeof(double);
  if (a.orth_part != 0) {   // caller checked orth_cluster_ok
    launch_orth_cs(s, a, bytes);
  } else if (orth_one_cta(a) || !(a.clw && launch_orth_cs(s, a, bytes))) {
    k_dense_orth<<<1, kDenseThreads, bytes, s>>>(a);
  }
  ++*launches;
}

void launch_dense_round(cudaStream_t s, const DenseArgs& a, int64_t* launches) {
  const size_t bytes = (size_t)a.smem_doubles * sizeof(double);
  k_project<<<a.d, kProjThreads, bytes, s>>>(a);
  if (!(a.clw && launch_round_cs(s, a, bytes))) k_dense_round<<<1, kDenseThreads, bytes, s>>>(a);
  *launches += 2;
  if (a.wretr) {
    k_unweight_out<<<a.d, 256, 0, s>>>(a);
    ++*launches;
  }
}

void launch_project(cudaStream_t s, const DenseArgs& a, int mode, int64_t* launches) {
  DenseArgs b = a;
  b.proj_mode = mode;
  k_project<<<b.d, kProjThreads, (size_t)b.smem_doubles * sizeof(double), s>>>(b);
  ++*launches;
}

void launch_round_only(cudaStream_t s, const DenseArgs& a, int64_t* launches) {
  const size_t bytes = (size_t)a.smem_doubles * sizeof(double);
  if (!(a.clw && launch_round_cs(s, a, bytes))) k_dense_round<<<1, kDenseThreads, bytes, s>>>(a);
  ++*launches;
  if (a.wretr) {
    k_unweight_out<<<a.d, 256, 0, s>>>(a);
    ++*launches;
  }
}

}  // namespace prgd
