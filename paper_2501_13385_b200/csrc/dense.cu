// dense.cu — the small, sequential dense work of one PRGD iteration, each sweep in a
// single persistent CTA (no host round trips, graph-capturable):
//
//   k_dense_orth   A4 That = W^{1/2} T (Prop. 3.1),
//                  A5 left-orthogonal U by a Householder QR sweep,
//                  A6 right Grams P_k = That^{>=k+1} That^{>=k+1 T} + Cholesky.
//   k_dense_round  A10 closed-form projection, A11 unweighting
//                  (PAPER.md:293, 360), A13 rank-2r TT of W_l,
//                  A14 TT-rounding = Alg. 1 on W_l: right-to-left
//                  Householder QR, then left-to-right QR + one-sided Jacobi SVD.
//
// Householder reflectors follow LAPACK dgeqr2/dorg2r conventions (beta = -sign(alpha)
// ||x||, tau = (beta - alpha)/beta, v_j = 1; tau = 0 when the sub-column is zero).
// Matrices are staged in shared memory when they fit, else processed in the global
// scratch area (same code through MatView).
#include "prgd_internal.cuh"

namespace prgd {
namespace {

struct MatView {
  double* p;
  int64_t rs, cs;
  __device__ __forceinline__ double& at(int i, int j) const { return p[i * rs + j * cs]; }
};

// Householder QR in place; tau[kmin].  red: >= blockDim.x doubles; colv: >= 2*n doubles.
__device__ void blk_geqr2(MatView A, int m, int n, double* tau, double* red, double* colv) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int kmin = m < n ? m : n;
  double* colsum = colv;        // [n]
  double* wv = colv + n;        // [n]
  __shared__ double s_tau, s_denom, s_beta;
  for (int j = 0; j < kmin; ++j) {
    const int nc = n - j;
    const int G = T / nc;
    const int q = tid % nc, g = tid / nc;
    double s = 0.0;
    if (g < G)
      for (int i = j + 1 + g; i < m; i += G) s = fma(A.at(i, j), A.at(i, j + q), s);
    red[tid] = (g < G) ? s : 0.0;
    __syncthreads();
    if (tid < nc) {
      double acc = 0.0;
      for (int gg = 0; gg < G; ++gg) acc += red[gg * nc + tid];
      colsum[tid] = acc;
    }
    __syncthreads();
    if (tid == 0) {
      const double alpha = A.at(j, j);
      const double xb2 = colsum[0];
      if (xb2 == 0.0) {
        s_tau = 0.0;
        s_denom = 0.0;
        s_beta = alpha;
      } else {
        const double beta = -copysign(sqrt(alpha * alpha + xb2), alpha);
        s_tau = (beta - alpha) / beta;
        s_denom = 1.0 / (alpha - beta);
        s_beta = beta;
      }
      tau[j] = s_tau;
    }
    __syncthreads();
    const double tj = s_tau, dn = s_denom;
    if (tj != 0.0) {
      if (tid < nc - 1) {
        const int c = j + 1 + tid;
        wv[c] = A.at(j, c) + colsum[1 + tid] * dn;
      }
      __syncthreads();
      const int ncr = nc - 1;
      if (ncr > 0) {
        const int64_t tot = (int64_t)(m - j) * ncr;
        for (int64_t e = tid; e < tot; e += T) {
          const int i = j + (int)(e / ncr);
          const int c = j + 1 + (int)(e % ncr);
          const double vi = (i == j) ? 1.0 : A.at(i, j) * dn;
          A.at(i, c) -= tj * vi * wv[c];
        }
      }
      __syncthreads();
      for (int i = j + 1 + tid; i < m; i += T) A.at(i, j) *= dn;
      if (tid == 0) A.at(j, j) = s_beta;
      __syncthreads();
    }
  }
}

// Form the m x k Q (k = #reflectors) in place over the first k columns (dorg2r).
__device__ void blk_org2r(MatView A, int m, int k, const double* tau, double* red, double* colv) {
  const int T = blockDim.x, tid = threadIdx.x;
  double* colsum = colv;
  for (int j = k - 1; j >= 0; --j) {
    const double tj = tau[j];
    const int nc = k - 1 - j;  // columns j+1..k-1
    if (nc > 0 && tj != 0.0) {
      const int G = T / nc;
      const int q = tid % nc, g = tid / nc;
      double s = 0.0;
      if (g < G)
        for (int i = j + 1 + g; i < m; i += G) s = fma(A.at(i, j), A.at(i, j + 1 + q), s);
      red[tid] = (g < G) ? s : 0.0;
      __syncthreads();
      if (tid < nc) {
        double acc = 0.0;
        for (int gg = 0; gg < G; ++gg) acc += red[gg * nc + tid];
        colsum[tid] = (A.at(j, j + 1 + tid) + acc) * tj;   // tau * w_c
      }
      __syncthreads();
      const int64_t tot = (int64_t)(m - j) * nc;
      for (int64_t e = tid; e < tot; e += T) {
        const int i = j + (int)(e / nc);
        const int c = j + 1 + (int)(e % nc);
        const double vi = (i == j) ? 1.0 : A.at(i, j);
        A.at(i, c) -= vi * colsum[c - j - 1];
      }
      __syncthreads();
    }
    for (int i = j + 1 + tid; i < m; i += T) A.at(i, j) *= -tj;
    for (int i = tid; i < j; i += T) A.at(i, j) = 0.0;
    if (tid == 0) A.at(j, j) = 1.0 - tj;
    __syncthreads();
  }
}

// In-place Cholesky of the R x R SPD matrix P (row-major), lower factor; returns false on
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
    int i = e / R, c = e % R;
    if (c > i) P[e] = 0.0;
  }
  __syncthreads();
  return s_ok != 0;
}

// One-sided Jacobi on the columns of X (rows x kc, column-major: X[c*rows + i]),
// accumulating V (kc x kc, column-major).  Round-robin parallel ordering, one warp
// per pair.  Returns false if not converged.
__device__ bool blk_jacobi(double* X, int rows, int kc, double* V) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __shared__ int s_rot;
  for (int e = tid; e < kc * kc; e += blockDim.x) V[e] = (e / kc == e % kc) ? 1.0 : 0.0;
  __syncthreads();
  if (kc < 2) return true;
  const int kp = kc + (kc & 1);
  const int npairs = kp / 2;
  const double tol = 2.3e-16 * sqrt((double)(rows > 1 ? rows : 1));
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < kp - 1; ++round) {
      for (int pr = warp; pr < npairs; pr += nw) {
        auto pos = [&](int i) { return i == 0 ? 0 : ((i - 1 + round) % (kp - 1)) + 1; };
        int a = pos(pr), b = pos(kp - 1 - pr);
        if (a > b) { int t = a; a = b; b = t; }
        if (b >= kc) continue;
        double* xa = X + (int64_t)a * rows;
        double* xb = X + (int64_t)b * rows;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < rows; i += 32) {
          const double u = xa[i], w = xb[i];
          al = fma(u, u, al);
          be = fma(w, w, be);
          ga = fma(u, w, ga);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = lane; i < rows; i += 32) {
            const double u = xa[i], w = xb[i];
            xa[i] = c * u - s * w;
            xb[i] = s * u + c * w;
          }
          double* va = V + (int64_t)a * kc;
          double* vb = V + (int64_t)b * kc;
          for (int i = lane; i < kc; i += 32) {
            const double u = va[i], w = vb[i];
            va[i] = c * u - s * w;
            vb[i] = s * u + c * w;
          }
          if (lane == 0) s_rot = 1;
        }
      }
      __syncthreads();
    }
    const int rot = s_rot;
    __syncthreads();
    if (!rot) return true;
  }
  return false;
}

struct Smem {
  double* red;    // blockDim
  double* colv;   // 2*kMaxCols
  double* tau;    // kMaxCols
  double* small1; // S x S
  double* small2; // S x S
  double* small3; // S x S
  int* perm;      // S
  double* mat;    // staging area
  int64_t mat_cap;
};

constexpr int kMaxCols = 2 * kMaxRank;

__device__ Smem carve(double* sm, int smem_doubles, int S) {
  Smem s;
  double* p = sm;
  s.red = p; p += kDenseThreads;
  s.colv = p; p += 2 * kMaxCols;
  s.tau = p; p += kMaxCols;
  s.small1 = p; p += S * S;
  s.small2 = p; p += S * S;
  s.small3 = p; p += S * S;
  s.perm = reinterpret_cast<int*>(p); p += (S + 1) / 2 + 1;
  s.mat = p;
  s.mat_cap = smem_doubles - (int64_t)(p - sm);
  return s;
}

// Copy a (rows x cols) strided view into a compact row-major destination.
__device__ void blk_copy_in(double* dst, const double* src, int rows, int cols, int64_t rs,
                            int64_t cs) {
  const int64_t tot = (int64_t)rows * cols;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    int i = (int)(e / cols), j = (int)(e % cols);
    dst[e] = src[i * rs + j * cs];
  }
}

__device__ void blk_copy(double* dst, const double* src, int64_t n) {
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) dst[e] = src[e];
}

// Mode-1 product: out[a', rest] = sum_b M[a', b] in[b, rest]; M (ra x rb) row-major.
__device__ void blk_mode1(double* out, const double* M, int ra, int rb, const double* in,
                          int64_t rest) {
  const int64_t tot = (int64_t)ra * rest;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int a = (int)(e / rest);
    const int64_t x = e - (int64_t)a * rest;
    double acc = 0.0;
    for (int b = 0; b < rb; ++b) acc = fma(M[a * rb + b], in[(int64_t)b * rest + x], acc);
    out[e] = acc;
  }
}

// Mode-3 product with M^T: out[row, c'] = sum_b in[row, b] M[c', b]; M (rc x rb) row-major.
__device__ void blk_mode3t(double* out, const double* in, int64_t rows, int rb, const double* M,
                           int rc) {
  const int64_t tot = rows * rc;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t row = e / rc;
    const int c = (int)(e - row * rc);
    double acc = 0.0;
    for (int b = 0; b < rb; ++b) acc = fma(in[row * rb + b], M[c * rb + b], acc);
    out[e] = acc;
  }
}

// QR of a compact row-major (m x n) matrix at `g` (global).  Stages into smem when it
// fits.  On return: R (kmin x n, row-major, zero below diag) in Rout, Q (m x kmin,
// row-major compact) at Qout (may alias g).  Returns kmin.
__device__ int blk_qr_explicit(const Smem& sm, double* g, int m, int n, double* Rout,
                               double* Qout, double* gwork) {
  const int kmin = m < n ? m : n;
  const int64_t sz = (int64_t)m * n;
  double* A = (sz <= sm.mat_cap) ? sm.mat : gwork;
  if (A != g) {
    blk_copy(A, g, sz);
    __syncthreads();
  }
  MatView V{A, n, 1};
  blk_geqr2(V, m, n, sm.tau, sm.red, sm.colv);
  for (int64_t e = threadIdx.x; e < (int64_t)kmin * n; e += blockDim.x) {
    int a = (int)(e / n), b = (int)(e % n);
    Rout[e] = b >= a ? V.at(a, b) : 0.0;
  }
  __syncthreads();
  blk_org2r(V, m, kmin, sm.tau, sm.red, sm.colv);
  // compact Q (m x kmin) from the leading columns
  if (Qout != A || kmin != n) {
    // write row-major m x kmin; when Qout aliases A and kmin < n, rows shrink: do it in
    // increasing order after a barrier-separated copy through the red buffer per row.
    if (Qout == A) {
      for (int i = 0; i < m; ++i) {
        double v = threadIdx.x < kmin ? A[(int64_t)i * n + threadIdx.x] : 0.0;
        __syncthreads();
        if (threadIdx.x < kmin) Qout[(int64_t)i * kmin + threadIdx.x] = v;
        __syncthreads();
      }
    } else {
      for (int64_t e = threadIdx.x; e < (int64_t)m * kmin; e += blockDim.x) {
        int i = (int)(e / kmin), c = (int)(e % kmin);
        Qout[e] = A[(int64_t)i * n + c];
      }
    }
  }
  __syncthreads();
  return kmin;
}

__global__ void __launch_bounds__(kDenseThreads) k_dense_orth(DenseArgs a) {
  extern __shared__ double smraw[];
  Scalars* sc = a.sc;
  if (sc->noop) return;
  const int d = a.d;
  int S = 2;
  for (int k = 0; k <= d; ++k) S = a.r[k] > S ? a.r[k] : S;
  Smem sm = carve(smraw, a.smem_doubles, S);
  // A4: U_k = phi_k (.)_2 C_k
  for (int k = 0; k < d; ++k) {
    const int r0 = a.r[k], nk = a.n[k], r1 = a.r[k + 1];
    const int64_t tot = (int64_t)r0 * nk * r1;
    const double* C = a.C + a.core_off[k];
    double* U = a.U + a.core_off[k];
    const double* ph = a.phi + a.phi_off[k];
    for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
      const int j = (int)((e / r1) % nk);
      U[e] = C[e] * ph[j];
    }
  }
  __syncthreads();
  // A5: Householder QR sweep, U_k <- Q, U_{k+1} <- R U_{k+1}
  double* gw = a.work;
  for (int k = 0; k + 1 < d; ++k) {
    const int r0 = a.r[k], nk = a.n[k], r1 = a.r[k + 1];
    const int m = r0 * nk;
    double* U = a.U + a.core_off[k];
    double* R = sm.small1;
    blk_qr_explicit(sm, U, m, r1, R, U, gw);   // kmin = r1 (feasible ranks); Q -> U
    double* Un = a.U + a.core_off[k + 1];
    const int64_t rest = (int64_t)a.n[k + 1] * a.r[k + 2];
    blk_mode1(gw, R, r1, r1, Un, rest);
    __syncthreads();
    blk_copy(Un, gw, (int64_t)r1 * rest);
    __syncthreads();
  }
  // A6: P_{d-1} = [1]; P_k = sum_j U_{k+1}(:,j,:) P_{k+1} U_{k+1}(:,j,:)^T, Cholesky.
  {
    double* P = a.P + a.p_off[d - 1];
    double* L = a.L + a.p_off[d - 1];
    if (threadIdx.x == 0) {
      P[0] = 1.0;
      L[0] = 1.0;
    }
    __syncthreads();
  }
  bool ok = true;
  for (int k = d - 2; k >= 0; --k) {
    const int R1 = a.r[k + 1], nk = a.n[k + 1], R2 = a.r[k + 2];
    const double* Un = a.U + a.core_off[k + 1];
    const double* Pn = a.P + a.p_off[k + 1];
    // T1[a, j, e] = sum_c U[a, j, c] Pn[c, e]  (into gw)
    const int64_t t1 = (int64_t)R1 * nk * R2;
    for (int64_t e = threadIdx.x; e < t1; e += blockDim.x) {
      const int ee = (int)(e % R2);
      const int64_t aj = e / R2;
      double acc = 0.0;
      for (int c = 0; c < R2; ++c) acc = fma(Un[aj * R2 + c], Pn[c * R2 + ee], acc);
      gw[e] = acc;
    }
    __syncthreads();
    double* P = a.P + a.p_off[k];
    for (int e = threadIdx.x; e < R1 * R1; e += blockDim.x) {
      const int aa = e / R1, bb = e % R1;
      double acc = 0.0;
      const int64_t len = (int64_t)nk * R2;
      for (int64_t q = 0; q < len; ++q) acc = fma(gw[aa * len + q], Un[bb * len + q], acc);
      P[e] = acc;
    }
    __syncthreads();
    // symmetrise (exact symmetry for the Cholesky input)
    double* Ls = sm.small1;
    for (int e = threadIdx.x; e < R1 * R1; e += blockDim.x) {
      const int aa = e / R1, bb = e % R1;
      Ls[e] = 0.5 * (P[aa * R1 + bb] + P[bb * R1 + aa]);
    }
    __syncthreads();
    ok = blk_chol(Ls, R1) && ok;
    double* L = a.L + a.p_off[k];
    blk_copy(L, Ls, (int64_t)R1 * R1);
    __syncthreads();
  }
  if (!ok && threadIdx.x == 0) {
    atomicOr(&sc->err, (int)kErrChol);
    sc->noop = 1;
  }
}

__global__ void __launch_bounds__(kDenseThreads) k_dense_round(DenseArgs a) {
  extern __shared__ double smraw[];
  Scalars* sc = a.sc;
  if (sc->noop) return;
  const int d = a.d;
  const double alpha = sc->alpha;
  int S = 2;
  for (int k = 0; k <= d; ++k) S = 2 * a.r[k] > S ? 2 * a.r[k] : S;
  Smem sm = carve(smraw, a.smem_doubles, S);
  double* gw = a.work;
  // ---- A10: projection, A11 + A13 assembly into B
  for (int k = 0; k < d; ++k) {
    const int r0 = a.r[k], nk = a.n[k], r1 = a.r[k + 1];
    const int m = r0 * nk;
    const double* Y = a.Y + a.core_off[k];
    double* Ah = a.Ahat + a.core_off[k];
    const double* U = a.U + a.core_off[k];
    if (k == d - 1) {
      blk_copy(Ah, Y, (int64_t)m * r1);
      __syncthreads();
    } else {
      const double* L = a.L + a.p_off[k];
      double* Ls = sm.small1;
      blk_copy(Ls, L, (int64_t)r1 * r1);
      __syncthreads();
      for (int row = threadIdx.x; row < m; row += blockDim.x) {
        const double* y = Y + (int64_t)row * r1;
        double* z = Ah + (int64_t)row * r1;
        for (int i = 0; i < r1; ++i) {
          double s = y[i];
          for (int c = 0; c < i; ++c) s -= Ls[i * r1 + c] * z[c];
          z[i] = s / Ls[i * r1 + i];
        }
        for (int i = r1 - 1; i >= 0; --i) {
          double s = z[i];
          for (int c = i + 1; c < r1; ++c) s -= Ls[c * r1 + i] * z[c];
          z[i] = s / Ls[i * r1 + i];
        }
      }
      __syncthreads();
      double* W = sm.small2;
      for (int e = threadIdx.x; e < r1 * r1; e += blockDim.x) {
        const int aa = e / r1, bb = e % r1;
        double acc = 0.0;
        for (int row = 0; row < m; ++row) acc = fma(U[(int64_t)row * r1 + aa], Ah[(int64_t)row * r1 + bb], acc);
        W[e] = acc;
      }
      __syncthreads();
      for (int64_t e = threadIdx.x; e < (int64_t)m * r1; e += blockDim.x) {
        const int64_t row = e / r1;
        const int bb = (int)(e - row * r1);
        double acc = 0.0;
        for (int aa = 0; aa < r1; ++aa) acc = fma(U[row * r1 + aa], W[aa * r1 + bb], acc);
        Ah[e] -= acc;
      }
      __syncthreads();
    }
    // assembly of B_k (ranks Rb[k] x n x Rb[k+1])
    const double* ph = a.phi + a.phi_off[k];
    double* B = a.B + a.b_off[k];
    if (d == 1) {
      // not reachable (d >= 2)
    } else if (k == 0) {
      const int Rb1 = 2 * r1;
      for (int64_t e = threadIdx.x; e < (int64_t)nk * Rb1; e += blockDim.x) {
        const int x = (int)(e / Rb1), c = (int)(e % Rb1);
        const double inv = 1.0 / ph[x];
        B[e] = c < r1 ? -alpha * Ah[x * r1 + c] * inv : U[x * r1 + (c - r1)] * inv;
      }
    } else if (k == d - 1) {
      for (int64_t e = threadIdx.x; e < (int64_t)2 * r0 * nk; e += blockDim.x) {
        const int aa = (int)(e / nk), x = (int)(e % nk);
        const double inv = 1.0 / ph[x];
        if (aa < r0) B[e] = U[aa * nk + x] * inv;
        else B[e] = (U[(aa - r0) * nk + x] - alpha * Ah[(aa - r0) * nk + x]) * inv;
      }
    } else {
      const int Rb0 = 2 * r0, Rb1 = 2 * r1;
      for (int64_t e = threadIdx.x; e < (int64_t)Rb0 * nk * Rb1; e += blockDim.x) {
        const int c = (int)(e % Rb1);
        const int x = (int)((e / Rb1) % nk);
        const int aa = (int)(e / ((int64_t)Rb1 * nk));
        const double inv = 1.0 / ph[x];
        double v;
        if (aa < r0) v = c < r1 ? U[((int64_t)aa * nk + x) * r1 + c] * inv : 0.0;
        else if (c < r1) v = -alpha * Ah[((int64_t)(aa - r0) * nk + x) * r1 + c] * inv;
        else v = U[((int64_t)(aa - r0) * nk + x) * r1 + (c - r1)] * inv;
        B[e] = v;
      }
    }
    __syncthreads();
  }
  // ---- A14 (i): right-to-left orthogonalisation
  __shared__ int curR[kMaxD + 1];
  if (threadIdx.x == 0) {
    curR[0] = 1;
    for (int k = 1; k < d; ++k) curR[k] = 2 * a.r[k];
    curR[d] = 1;
  }
  __syncthreads();
  for (int k = d - 1; k >= 1; --k) {
    const int R0 = curR[k], nk = a.n[k], R1 = curR[k + 1];
    const int rows = nk * R1, cols = R0;
    double* B = a.B + a.b_off[k];
    // stage M^T (rows x cols) compact: Mt[i, a] = B[a*rows + i]
    const int64_t sz = (int64_t)rows * cols;
    double* A = sz <= sm.mat_cap ? sm.mat : gw;
    for (int64_t e = threadIdx.x; e < sz; e += blockDim.x) {
      const int i = (int)(e / cols), aa = (int)(e % cols);
      A[e] = B[(int64_t)aa * rows + i];
    }
    __syncthreads();
    double* R = sm.small1;
    const int kmin = blk_qr_explicit(sm, A, rows, cols, R, A, A);
    double* tmp = (A == gw) ? gw + sz : gw;
    // new B_k = Q^T (kmin x rows)
    for (int64_t e = threadIdx.x; e < (int64_t)kmin * rows; e += blockDim.x) {
      const int aa = (int)(e / rows), i = (int)(e % rows);
      B[e] = A[(int64_t)i * kmin + aa];
    }
    __syncthreads();
    // B_{k-1} <- B_{k-1} x_3 R^T  (R: kmin x R0)
    double* Bp = a.B + a.b_off[k - 1];
    const int64_t prow = (int64_t)curR[k - 1] * a.n[k - 1];
    blk_mode3t(tmp, Bp, prow, R0, R, kmin);
    __syncthreads();
    blk_copy(Bp, tmp, prow * kmin);
    __syncthreads();
    if (threadIdx.x == 0) curR[k] = kmin;
    __syncthreads();
  }
  // ---- A14 (ii): left-to-right truncated SVD sweep
  bool ok = true;
  for (int k = 0; k + 1 < d; ++k) {
    const int R0 = curR[k], nk = a.n[k], R1 = curR[k + 1];
    const int m = R0 * nk;
    const int rk = a.r[k + 1];
    double* B = a.B + a.b_off[k];
    const int64_t sz = (int64_t)m * R1;
    double* A = sz <= sm.mat_cap ? sm.mat : gw;
    blk_copy(A, B, sz);
    __syncthreads();
    double* R = sm.small1;
    const int kmin = blk_qr_explicit(sm, A, m, R1, R, A, A);
    double* tmp = (A == gw) ? gw + sz : gw;
    // X = R^T (R1 x kmin), column-major: X[c*R1 + i] = R[c, i]
    double* X = sm.small2;
    double* V = sm.small3;
    for (int e = threadIdx.x; e < kmin * R1; e += blockDim.x) X[e] = R[e];
    __syncthreads();
    ok = blk_jacobi(X, R1, kmin, V) && ok;
    // sort columns by norm, descending (ties by index)
    double* nrm = sm.red;
    if (threadIdx.x < kmin) {
      double s = 0.0;
      for (int i = 0; i < R1; ++i) s = fma(X[threadIdx.x * R1 + i], X[threadIdx.x * R1 + i], s);
      nrm[threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x < kmin) {
      const int c = threadIdx.x;
      int rank = 0;
      for (int c2 = 0; c2 < kmin; ++c2)
        rank += (nrm[c2] > nrm[c]) || (nrm[c2] == nrm[c] && c2 < c);
      sm.perm[rank] = c;
    }
    __syncthreads();
    // C'_k = Q V[:, perm[:rk]]  (m x rk), written to the output core k
    double* Cout = a.C + a.core_off[k];
    for (int64_t e = threadIdx.x; e < (int64_t)m * rk; e += blockDim.x) {
      const int64_t row = e / rk;
      const int c = (int)(e - row * rk);
      double acc = 0.0;
      if (c < kmin) {
        const int pc = sm.perm[c];
        for (int q = 0; q < kmin; ++q) acc = fma(A[row * kmin + q], V[pc * kmin + q], acc);
      }
      tmp[e] = acc;
    }
    __syncthreads();
    blk_copy(Cout, tmp, (int64_t)m * rk);
    // SVt (rk x R1): row a' = X[:, perm[a']]^T
    double* SV = sm.small1;
    for (int e = threadIdx.x; e < rk * R1; e += blockDim.x) {
      const int ap = e / R1, i = e % R1;
      SV[e] = ap < kmin ? X[sm.perm[ap] * R1 + i] : 0.0;
    }
    __syncthreads();
    double* Bn = a.B + a.b_off[k + 1];
    const int64_t rest = (int64_t)a.n[k + 1] * curR[k + 2];
    blk_mode1(tmp, SV, rk, R1, Bn, rest);
    __syncthreads();
    blk_copy(Bn, tmp, (int64_t)rk * rest);
    __syncthreads();
    if (threadIdx.x == 0) curR[k + 1] = rk;
    __syncthreads();
  }
  {
    const int k = d - 1;
    const int64_t sz = (int64_t)curR[k] * a.n[k];
    blk_copy(a.C + a.core_off[k], a.B + a.b_off[k], sz);
  }
  __syncthreads();
  // finite check of the new iterate
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

}  // namespace

int dense_smem_doubles() { return (200 * 1024) / 8; }

void dense_init() {
  const int bytes = dense_smem_doubles() * (int)sizeof(double);
  cudaFuncSetAttribute(k_dense_orth, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_dense_round, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

void launch_dense_orth(cudaStream_t s, const DenseArgs& a, int64_t* launches) {
  const size_t bytes = (size_t)a.smem_doubles * sizeof(double);
  k_dense_orth<<<1, kDenseThreads, bytes, s>>>(a);
  ++*launches;
}

void launch_dense_round(cudaStream_t s, const DenseArgs& a, int64_t* launches) {
  const size_t bytes = (size_t)a.smem_doubles * sizeof(double);
  k_dense_round<<<1, kDenseThreads, bytes, s>>>(a);
  ++*launches;
}

}  // namespace prgd
