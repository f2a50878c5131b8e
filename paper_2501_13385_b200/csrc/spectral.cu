// spectral.cu — spectral initialisation at scale: T_0 = SVD_r^tt(Z),
// Alg. 1 (TT-SVD) applied to the sparse tensor Z = p^{-1} P_Omega(y) without
// densifying it (the "TT-SVD spectral initialization"; BASELINE.json config 1).
//
// Step k of Alg. 1 needs the top r_k left singular vectors of the projected unfolding
//   M_k[(a, x), q] = sum_{s: x_{s,k} = x, suffix_k(s) = q} a_s[a] z_s,
// a_s = the left chain U_1(x_{s,1}) ... U_{k-1}(x_{s,k-1}) of the cores already chosen
// (r_{k-1}-vector per sample), q = (x_{k+1}, ..., x_d).  Its rows number W = r_{k-1} n_k (<= 1024),
// its nonzero columns are the distinct suffixes in Omega.  Here:
//   * the samples (prefix order) are sorted by key (q, x_k) (the library's radix sort);
//   * runs of equal key give w_{q,x} = sum z_s a_s (thread per run, fixed order);
//   * the Gram G_k = M_k M_k^T = sum_q sum_{j, j' in q} w_j w_j'^T (blocks (x_j, x_j')) is
//     accumulated by warps over contiguous group ranges into private partials, summed in a
//     fixed order (deterministic);
//   * the symmetric eigenproblem of G_k by cyclic Jacobi (round-robin parallel ordering, one
//     CTA); U_k = the eigenvectors of the r_k largest eigenvalues (ties: lower index);
//   * a_s <- a_s U_k(:, x_{s,k}, :).
// The last core is M_d itself: C_d[a, x] = sum_{s: x_{s,d} = x} a_s[a] z_s.
// Gram-based: the kept subspace is accurate to ~u ||G|| / gap (the singular values squared).
// When W > 1024 (config 3's 16 x 256 = 4096 rows at k = 2) but M_k has at most 1024 nonzero
// columns (the distinct suffixes q present in Omega; 128 there), the same subspace comes from
// the other side: M_k is formed densely (W x Q, one entry per run), the Q x Q Gram M_k^T M_k is
// diagonalised by the same Jacobi kernel, U = M_k V_r Lambda_r^{-1/2}, and U's columns are
// re-orthonormalised (two modified Gram-Schmidt passes) so that the core is left-orthogonal to
// rounding.
#include <algorithm>
#include <vector>

#include "../../include/prgd.h"
#include "prgd_internal.cuh"

namespace prgd {
namespace {

constexpr int kT = 256;
constexpr int kLong = 32, kChunk = 8192;   // runs longer than kLong: chunked CTA sums
inline unsigned bl(int64_t n, int t = kT) { return (unsigned)((n + t - 1) / t); }

struct SpDims {
  int d, KL;
  int n[kMaxD];
  int64_t pstride[kMaxD];   // k < KL: prod_{j = k+1}^{KL-1} n_j  (x_0 most significant in P)
  int64_t sstride[kMaxD];   // k >= KL: prod_{j = KL}^{k-1} n_j   (x_KL least significant in S)
};

__device__ __forceinline__ int digit(const SpDims& D, int k, int64_t P, int64_t S) {
  if (k < D.KL) return (int)((P / D.pstride[k]) % D.n[k]);
  return (int)((S / D.sstride[k]) % D.n[k]);
}

// prefix row of every prefix position (virtual rows v = b N_L + P)
__global__ void k_sp_rows(const int64_t* __restrict__ offs, int64_t nrows, int64_t NL,
                          int32_t* __restrict__ Ppos) {
  const int64_t v = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (v >= nrows) return;
  const int32_t P = (int32_t)(v % NL);
  for (int64_t t = offs[v]; t < offs[v + 1]; ++t) Ppos[t] = P;
}

__global__ void k_sp_init(const double* __restrict__ y, int64_t m, double invp, double* __restrict__ z,
                          double* __restrict__ chain, int cs) {
  const int64_t t = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (t >= m) return;
  z[t] = y[t] * invp;
  chain[t * cs] = 1.0;   // r_0 = 1
}

// key = q n_k + x_k with q the code of (x_{k+1}, ..., x_{d-1}); value = prefix position
__global__ void k_sp_keys(const int32_t* __restrict__ Ppos, const int32_t* __restrict__ Spre, int64_t m,
                          SpDims D, int k, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t t = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (t >= m) return;
  const int64_t P = Ppos[t], S = Spre[t];
  uint64_t key;
  if (k < D.KL) {
    const uint64_t q = (uint64_t)(P % D.pstride[k]) + (uint64_t)D.pstride[k] * (uint64_t)S;
    key = q * (uint64_t)D.n[k] + (uint64_t)digit(D, k, P, S);
  } else {
    key = (uint64_t)(S / D.sstride[k]);
  }
  keys[t] = key;
  vals[t] = (uint32_t)t;
}

// run (equal key) and group (equal q) start flags of the sorted keys
__global__ void k_sp_flags(const uint64_t* __restrict__ ko, int64_t m, int nk, int* __restrict__ fr) {
  const int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (i >= m) return;
  fr[i] = (i == 0 || ko[i] != ko[i - 1]) ? 1 : 0;
  (void)nk;
}

// per run: start, x, group-start flag
__global__ void k_sp_runs(const uint64_t* __restrict__ ko, const int* __restrict__ fr,
                          const int64_t* __restrict__ ridx, int64_t m, int nk, int64_t* __restrict__ rstart,
                          int* __restrict__ rx, int* __restrict__ gflag) {
  const int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (i == 0) rstart[ridx[m]] = m;
  if (i >= m || !fr[i]) return;
  const int64_t r = ridx[i];
  rstart[r] = i;
  rx[r] = (int)(ko[i] % (uint64_t)nk);
  gflag[r] = (i == 0 || ko[i] / (uint64_t)nk != ko[i - 1] / (uint64_t)nk) ? 1 : 0;
}

// per run of <= kLong samples: w = sum z_t a_t by one thread, in order (longer runs below)
__global__ void k_sp_entries(const int64_t* __restrict__ rstart, int64_t nruns, const uint32_t* __restrict__ vo,
                             const double* __restrict__ z, const double* __restrict__ chain, int cs, int r0,
                             double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)kT + threadIdx.x;
  const int64_t rbase = r - lane;
  if (rbase >= nruns) return;
  int64_t b0 = 0, b1 = 0;
  if (r < nruns) {
    b0 = rstart[r];
    b1 = rstart[r + 1];
  }
  const bool longrun = b1 - b0 > kLong;
  if (r < nruns && !longrun) {
    double acc[kMaxRank];
#pragma unroll
    for (int a = 0; a < kMaxRank; ++a) acc[a] = 0.0;
    for (int64_t i = b0; i < b1; ++i) {
      const int64_t t = vo[i];
      const double zt = z[t];
      const double* ct = chain + t * cs;
#pragma unroll
      for (int a = 0; a < kMaxRank; ++a)
        if (a < r0) acc[a] = fma(zt, ct[a], acc[a]);
    }
#pragma unroll
    for (int a = 0; a < kMaxRank; ++a)
      if (a < r0) w[r * cs + a] = acc[a];
  }
}

// runs longer than kLong samples: CTA (run, chunk) sums a chunk of kChunk samples (thread-
// strided, fixed-order tree over the threads), then k_sp_long_combine adds the chunk partials in
// chunk order
__global__ void k_sp_long_flag(const int64_t* __restrict__ rstart, int64_t nruns, int* __restrict__ f) {
  const int64_t r = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (r >= nruns) return;
  f[r] = rstart[r + 1] - rstart[r] > kLong ? 1 : 0;
}
// long run l (list[l] = run), its chunk count and the chunk -> (run, index) map
__global__ void k_sp_long_list(const int* __restrict__ f, const int64_t* __restrict__ fidx, int64_t nruns,
                               const int64_t* __restrict__ rstart, int64_t* __restrict__ list,
                               int* __restrict__ nch) {
  const int64_t r = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (r >= nruns || !f[r]) return;
  const int64_t l = fidx[r];
  list[l] = r;
  nch[l] = (int)((rstart[r + 1] - rstart[r] + kChunk - 1) / kChunk);
}
__global__ void k_sp_chunk_map(const int64_t* __restrict__ choff, int64_t nlong, int64_t* __restrict__ chl) {
  const int64_t l = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (l >= nlong) return;
  for (int64_t c = choff[l]; c < choff[l + 1]; ++c) chl[c] = l;
}
__global__ void k_sp_long_chunks(const int64_t* __restrict__ chl, const int64_t* __restrict__ choff,
                                 const int64_t* __restrict__ list, const int64_t* __restrict__ rstart,
                                 const uint32_t* __restrict__ vo, const double* __restrict__ z,
                                 const double* __restrict__ chain, int cs, int r0, double* __restrict__ cpart) {
  __shared__ double red[kT];
  const int64_t ch = blockIdx.x;
  const int64_t l = chl[ch];
  const int64_t r = list[l];
  const int64_t b0 = rstart[r] + (ch - choff[l]) * kChunk, e = rstart[r + 1];
  const int64_t b1 = b0 + kChunk < e ? b0 + kChunk : e;
  double acc[kMaxRank];
#pragma unroll
  for (int a = 0; a < kMaxRank; ++a) acc[a] = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += kT) {
    const int64_t t = vo[i];
    const double zt = z[t];
    const double* ct = chain + t * cs;
#pragma unroll
    for (int a = 0; a < kMaxRank; ++a)
      if (a < r0) acc[a] = fma(zt, ct[a], acc[a]);
  }
#pragma unroll
  for (int a = 0; a < kMaxRank; ++a) {
    if (a >= r0) break;
    red[threadIdx.x] = acc[a];
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) cpart[ch * cs + a] = red[0];
    __syncthreads();
  }
}
__global__ void k_sp_long_combine(const int64_t* __restrict__ list, const int64_t* __restrict__ choff,
                                  int64_t nlong, const double* __restrict__ cpart, int cs, int r0,
                                  double* __restrict__ w) {
  const int64_t e = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (e >= nlong * r0) return;
  const int64_t l = e / r0;
  const int a = (int)(e - l * r0);
  double s = 0.0;
  for (int64_t c = choff[l]; c < choff[l + 1]; ++c) s += cpart[c * cs + a];
  w[list[l] * cs + a] = s;
}

__global__ void k_sp_gstart(const int* __restrict__ gflag, const int64_t* __restrict__ gidx, int64_t nruns,
                            int64_t* __restrict__ gstart) {
  const int64_t r = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (r == 0) gstart[gidx[nruns]] = nruns;
  if (r >= nruns || !gflag[r]) return;
  gstart[gidx[r]] = r;
}

// runs keyed by x (stable radix sort keeps the group order within each x)
__global__ void k_sp_xkeys(const int* __restrict__ rx, int64_t nruns, uint64_t* __restrict__ keys,
                           uint32_t* __restrict__ vals) {
  const int64_t r = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (r >= nruns) return;
  keys[r] = (uint64_t)rx[r];
  vals[r] = (uint32_t)r;
}
__global__ void k_sp_xoffs(const uint64_t* __restrict__ kx, const uint32_t* __restrict__ vx, int64_t nruns,
                           int nk, int64_t* __restrict__ xoff, int64_t* __restrict__ byx) {
  const int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (i >= nruns) return;
  byx[i] = vx[i];
  const int64_t x = (int64_t)kx[i], xp = i == 0 ? -1 : (int64_t)kx[i - 1];
  for (int64_t q = xp + 1; q <= x; ++q) xoff[q] = i;
  if (i == nruns - 1)
    for (int64_t q = x + 1; q <= nk; ++q) xoff[q] = nruns;
}

// CTA (x, part): block row x of G (rows (a, x), all columns (b, x')) over its slice of the runs
// of x: for each such run j (group q) and every run j' of q, G[(a,x), (b,x_j')] += w_j[a] w_j'[b].
// The CTA's warps each own an accumulator copy in shared memory (warp w takes the batch entries
// e = w mod nwarps; lane owns products (a, b) = lane, lane + 32, ...), the batch indices are
// prefetched into shared memory, and the copies are summed in warp order at the end, so every
// sum has a fixed order.  part[p] holds the block rows of slice p, reduced over p in order.
constexpr int kGB = 128;   // batch of runs whose indices are prefetched together
template <int R>            // products (a, b) laid out as a R x R grid (R >= r0, power of two)
__global__ void k_sp_gram(const int64_t* __restrict__ byx, const int64_t* __restrict__ xoff,
                          const int64_t* __restrict__ gstart, const int64_t* __restrict__ rgroup,
                          const int* __restrict__ rx, const double* __restrict__ w, int cs, int r0, int nk,
                          int nparts, double* __restrict__ part) {
  extern __shared__ double smg[];
  const int x = blockIdx.x, p = blockIdx.y;
  constexpr int rr = R * R, NU = (rr + 31) / 32;
  const int W = r0 * nk, len = rr * nk;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* acc = smg + (int64_t)warp * len;
  int64_t* Jb = reinterpret_cast<int64_t*>(smg + (int64_t)nw * len);
  int64_t* S0 = Jb + kGB;
  int64_t* S1 = S0 + kGB;
  for (int e = threadIdx.x; e < nw * len; e += blockDim.x) smg[e] = 0.0;
  const int64_t n = xoff[x + 1] - xoff[x];
  const int64_t i0 = xoff[x] + p * n / nparts, i1 = xoff[x] + (p + 1) * n / nparts;
  for (int64_t ib = i0; ib < i1; ib += kGB) {
    __syncthreads();
    for (int t = threadIdx.x; t < kGB; t += blockDim.x)
      if (ib + t < i1) {
        const int64_t j = byx[ib + t];
        const int64_t g = rgroup[j];
        Jb[t] = j;
        S0[t] = gstart[g];
        S1[t] = gstart[g + 1];
      }
    __syncthreads();
    const int nb = (int)(i1 - ib < kGB ? i1 - ib : kGB);
    for (int e = warp; e < nb; e += nw) {
      const int64_t j = Jb[e];
      const double* wj = w + j * cs;
      double wa[NU];       // w_j[a] of the lane's products (a = ab / R, b = ab % R)
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const int ab = lane + 32 * u, a = ab / R;
        wa[u] = (ab < rr && a < r0) ? wj[a] : 0.0;
      }
      for (int64_t jp = S0[e]; jp < S1[e]; ++jp) {
        const int xq = rx[jp];
        const double* wq = w + jp * cs;
        double* ax = acc + (int64_t)xq * rr;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const int ab = lane + 32 * u, b = ab % R;
          if (ab < rr && b < r0) ax[ab] = fma(wa[u], wq[b], ax[ab]);
        }
      }
    }
  }
  __syncthreads();
  double* out = part + (int64_t)p * W * W;
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    double v = 0.0;
    for (int c = 0; c < nw; ++c) v += smg[(int64_t)c * len + e];
    const int xq = e / rr, ab = e - xq * rr;
    const int a = ab / R, b = ab % R;
    if (a < r0 && b < r0) out[(int64_t)(a * nk + x) * W + (b * nk + xq)] = v;
  }
}

// group of every run
__global__ void k_sp_rgroup(const int64_t* __restrict__ gidx, const int* __restrict__ gflag, int64_t nruns,
                            int64_t* __restrict__ rgroup) {
  const int64_t r = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (r >= nruns) return;
  rgroup[r] = gidx[r] + gflag[r] - 1;   // exclusive scan of the group-start flags
}

__global__ void k_sp_gram_reduce(const double* __restrict__ part, int64_t nparts, int64_t WW,
                                 double* __restrict__ G) {
  const int64_t e = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (e >= WW) return;
  double s = 0.0;
  for (int64_t p = 0; p < nparts; ++p) s += part[p * WW + e];
  G[e] = s;
}

// Cyclic Jacobi for the symmetric W x W matrix G (global, in place) with eigenvectors V; round-
// robin parallel ordering (W' = W rounded up to even; index W is a dummy).  Then the eigenvectors
// of the r1 largest eigenvalues (ties: lower index) become core k: C[a][x][c] = V[(a nk + x), sel_c].
#ifndef PRGD_SP_DEBUG
#define PRGD_SP_DEBUG 0
#endif
constexpr int kJT = 512;
constexpr int kJU = 4;       // element pairs per thread per batch
__global__ void __launch_bounds__(kJT) k_sp_jacobi(double* __restrict__ G, double* __restrict__ V, int W,
                                                   int r0, int nk, int r1, double* __restrict__ core,
                                                   int max_sweeps, double* __restrict__ lam = nullptr) {
  __shared__ double cs_c[512], cs_s[512];
  __shared__ int pp[512], qq[512];
  __shared__ int rot_any;
  __shared__ int sel[kMaxRank];
  __shared__ double dmax;
  const int tid = threadIdx.x;
  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < W; ++i) mx = fmax(mx, fabs(G[(int64_t)i * W + i]));
    dmax = mx;
  }
  const int Wp = W + (W & 1);
  const int np = Wp / 2;
  for (int64_t e = tid; e < (int64_t)W * W; e += kJT) {
    const int i = (int)(e / W), j = (int)(e - (int64_t)i * W);
    V[e] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rot_any = 0;
    __syncthreads();
    for (int round = 0; round < Wp - 1; ++round) {
      for (int k = tid; k < np; k += kJT) {
        const int i1 = k, i2 = Wp - 1 - k;
        const int a1 = i1 == 0 ? 0 : ((i1 - 1 + round) % (Wp - 1)) + 1;
        const int a2 = i2 == 0 ? 0 : ((i2 - 1 + round) % (Wp - 1)) + 1;
        const int p = min(a1, a2), q = max(a1, a2);
        double c = 1.0, s = 0.0;
        if (q < W) {
          const double gpp = G[(int64_t)p * W + p], gqq = G[(int64_t)q * W + q], gpq = G[(int64_t)p * W + q];
          // rotate unless negligible at the matrix scale (the rounding level of a converged
          // sweep grows like sqrt(W) u ||G||)
          if (fabs(gpq) > 4e-16 * sqrt((double)W) * dmax) {
            const double tau = (gqq - gpp) / (2.0 * gpq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            rot_any = 1;
          }
        }
        pp[k] = p;
        qq[k] = q < W ? q : p;
        cs_c[k] = c;
        cs_s[k] = s;
      }
      __syncthreads();
      // rows: G <- J^T G (batches of kJU element pairs per thread: loads issued together)
      const int64_t tot = (int64_t)np * W;
      for (int64_t e0 = tid; e0 < tot; e0 += (int64_t)kJT * kJU) {
        double gp[kJU], gq[kJU];
        int64_t ip[kJU], iq[kJU];
        bool on[kJU];
#pragma unroll
        for (int u = 0; u < kJU; ++u) {
          const int64_t e = e0 + (int64_t)u * kJT;
          on[u] = false;
          if (e < tot) {
            const int k = (int)(e / W), j = (int)(e - (int64_t)k * W);
            on[u] = cs_s[k] != 0.0;
            ip[u] = (int64_t)pp[k] * W + j;
            iq[u] = (int64_t)qq[k] * W + j;
            if (on[u]) {
              gp[u] = G[ip[u]];
              gq[u] = G[iq[u]];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kJU; ++u)
          if (on[u]) {
            const int k = (int)((e0 + (int64_t)u * kJT) / W);
            const double c = cs_c[k], sn = cs_s[k];
            G[ip[u]] = c * gp[u] - sn * gq[u];
            G[iq[u]] = sn * gp[u] + c * gq[u];
          }
      }
      __syncthreads();
      // columns: G <- G J, V <- V J
      for (int64_t e0 = tid; e0 < tot; e0 += (int64_t)kJT * kJU) {
        double gp[kJU], gq[kJU], vp[kJU], vq[kJU];
        int64_t ip[kJU], iq[kJU];
        bool on[kJU];
#pragma unroll
        for (int u = 0; u < kJU; ++u) {
          const int64_t e = e0 + (int64_t)u * kJT;
          on[u] = false;
          if (e < tot) {   // row-major over (j, k): a warp touches one row j of G / V
            const int j = (int)(e / np), k = (int)(e - (int64_t)j * np);
            on[u] = cs_s[k] != 0.0;
            ip[u] = (int64_t)j * W + pp[k];
            iq[u] = (int64_t)j * W + qq[k];
            if (on[u]) {
              gp[u] = G[ip[u]];
              gq[u] = G[iq[u]];
              vp[u] = V[ip[u]];
              vq[u] = V[iq[u]];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kJU; ++u)
          if (on[u]) {
            const int k = (int)((e0 + (int64_t)u * kJT) % np);
            const double c = cs_c[k], sn = cs_s[k];
            G[ip[u]] = c * gp[u] - sn * gq[u];
            G[iq[u]] = sn * gp[u] + c * gq[u];
            V[ip[u]] = c * vp[u] - sn * vq[u];
            V[iq[u]] = sn * vp[u] + c * vq[u];
          }
      }
      __syncthreads();
    }
    if (!rot_any) { if (PRGD_SP_DEBUG && tid == 0) printf("jacobi W=%d sweeps=%d\n", W, sweep + 1); break; }
    __syncthreads();
  }
  if (tid == 0) {
    for (int c = 0; c < r1; ++c) {
      int best = -1;
      for (int i = 0; i < W; ++i) {
        bool used = false;
        for (int u = 0; u < c; ++u) used = used || sel[u] == i;
        if (used) continue;
        if (best < 0 || G[(int64_t)i * W + i] > G[(int64_t)best * W + best]) best = i;
      }
      sel[c] = best;
    }
  }
  __syncthreads();
  for (int64_t e = tid; e < (int64_t)W * r1; e += kJT) {
    const int row = (int)(e / r1), c = (int)(e - (int64_t)row * r1);
    const int a = row / nk, x = row - a * nk;
    core[((int64_t)a * nk + x) * r1 + c] = V[(int64_t)row * W + sel[c]];
  }
  if (lam && tid < r1) lam[tid] = G[(int64_t)sel[tid] * W + sel[tid]];
}

// ---- right Gram path (W > 1024): M_k dense, row (a nk + x), column = group of the run
__global__ void k_sp_dense_M(const int* __restrict__ rx, const int64_t* __restrict__ rgroup,
                             const double* __restrict__ w, int64_t nruns, int cs, int r0, int nk, int64_t Q,
                             double* __restrict__ M) {
  const int64_t r = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (r >= nruns) return;
  const int x = rx[r];
  const int64_t q = rgroup[r];
  for (int a = 0; a < r0; ++a) M[((int64_t)a * nk + x) * Q + q] = w[r * cs + a];
}

// G = M^T M (Q x Q), thread per entry, rows in order (fixed)
__global__ void k_sp_gram_right(const double* __restrict__ M, int64_t W, int64_t Q, double* __restrict__ G) {
  const int64_t e = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (e >= Q * Q) return;
  const int64_t i = e / Q, j = e - i * Q;
  double s = 0.0;
  for (int64_t row = 0; row < W; ++row) s = fma(M[row * Q + i], M[row * Q + j], s);
  G[e] = s;
}

// core[row][c] = sum_q M[row][q] Vsel[q][c] / sqrt(lam[c])   (U = M V_r Lambda_r^{-1/2})
__global__ void k_sp_right_core(const double* __restrict__ M, const double* __restrict__ Vsel,
                                const double* __restrict__ lam, int64_t W, int64_t Q, int r1,
                                double* __restrict__ core) {
  const int64_t e = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (e >= W * r1) return;
  const int64_t row = e / r1;
  const int c = (int)(e - row * r1);
  double s = 0.0;
  for (int64_t q = 0; q < Q; ++q) s = fma(M[row * Q + q], Vsel[q * r1 + c], s);
  core[e] = lam[c] > 0.0 ? s / sqrt(lam[c]) : 0.0;
}

// two passes of modified Gram-Schmidt on the r1 columns (length W) of core [W][r1]; one CTA
__global__ void __launch_bounds__(512) k_sp_mgs(double* __restrict__ core, int64_t W, int r1) {
  __shared__ double red[512 / 32];
  __shared__ double bc;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  auto dot = [&](int a, int b) {
    double s = 0.0;
    for (int64_t i = tid; i < W; i += 512) s = fma(core[i * r1 + a], core[i * r1 + b], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __syncthreads();
    if (lane == 0) red[wid] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int i = 0; i < 512 / 32; ++i) t += red[i];
      bc = t;
    }
    __syncthreads();
    return bc;
  };
  for (int pass = 0; pass < 2; ++pass)
    for (int c = 0; c < r1; ++c) {
      for (int c2 = 0; c2 < c; ++c2) {
        const double h = dot(c2, c);
        for (int64_t i = tid; i < W; i += 512) core[i * r1 + c] = fma(-h, core[i * r1 + c2], core[i * r1 + c]);
        __syncthreads();
      }
      const double nn = dot(c, c);
      const double f = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
      for (int64_t i = tid; i < W; i += 512) core[i * r1 + c] *= f;
      __syncthreads();
    }
}

// a_t <- a_t U_k(:, x_{t,k}, :)
__global__ void k_sp_chain(const int32_t* __restrict__ Ppos, const int32_t* __restrict__ Spre, int64_t m,
                           SpDims D, int k, const double* __restrict__ core, int r0, int r1,
                           double* __restrict__ chain, int cs) {
  const int64_t t = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (t >= m) return;
  const int x = digit(D, k, Ppos[t], Spre[t]);
  const int nk = D.n[k];
  double a[kMaxRank];
  double* ct = chain + t * cs;
#pragma unroll
  for (int i = 0; i < kMaxRank; ++i) a[i] = i < r0 ? ct[i] : 0.0;
  for (int c = 0; c < r1; ++c) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kMaxRank; ++i)
      if (i < r0) s = fma(a[i], core[((int64_t)i * nk + x) * r1 + c], s);
    ct[c] = s;
  }
}

// last core: C_d[a][x][0] = w of the run with key x (the core is zeroed first: absent x)
__global__ void k_sp_last_fill(const int* __restrict__ rx, const double* __restrict__ w, int64_t nruns, int cs,
                               int r0, int nk, double* __restrict__ core) {
  const int64_t r = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (r >= nruns) return;
  const int x = rx[r];
  for (int a = 0; a < r0; ++a) core[(int64_t)a * nk + x] = w[r * cs + a];
}

}  // namespace

// Host driver.  All buffers are allocated by the caller (api.cu) through `alloc`; returns 0 or
// a TT_ERR code (message in *msg).
int spectral_init_run(cudaStream_t s, const SpectralArgs& A, std::string* msg, int64_t* launches) {
  const int d = A.d, KL = A.KL;
  const int64_t m = A.m;
  SpDims D{};
  D.d = d;
  D.KL = KL;
  for (int k = 0; k < d; ++k) D.n[k] = A.n[k];
  for (int k = 0; k < KL; ++k) {
    int64_t p = 1;
    for (int j = k + 1; j < KL; ++j) p *= A.n[j];
    D.pstride[k] = p;
  }
  for (int k = KL; k < d; ++k) {
    int64_t p = 1;
    for (int j = KL; j < k; ++j) p *= A.n[j];
    D.sstride[k] = p;
  }
  const int cs = A.cs;
  int64_t lc = 0;
  cudaFuncSetAttribute(k_sp_gram<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 3 * kGB * 8);
  cudaFuncSetAttribute(k_sp_gram<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 3 * kGB * 8);
  cudaFuncSetAttribute(k_sp_gram<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 3 * kGB * 8);
  k_sp_rows<<<bl(A.nrows), kT, 0, s>>>(A.offsL, A.nrows, A.NL, A.Ppos);
  k_sp_init<<<bl(m), kT, 0, s>>>(A.y, m, 1.0 / A.p, A.z, A.chain, cs);
  lc += 2;
  for (int k = 0; k < d; ++k) {
    const int r0 = A.r[k], nk = A.n[k], r1 = A.r[k + 1];
    const int W = r0 * nk;
    // sort the samples by (suffix after k, x_k)
    long double range = 1;
    for (int j = k; j < d; ++j) range *= A.n[j];
    int bits = 1;
    while ((long double)(1ull << std::min(bits, 62)) < range && bits < 63) ++bits;
    k_sp_keys<<<bl(m), kT, 0, s>>>(A.Ppos, A.Spre, m, D, k, A.keys, A.vals);
    ++lc;
    uint64_t* ko;
    uint32_t* vo;
    radix_sort_pairs(s, A.keys, A.vals, A.ktmp, A.vtmp, m, bits, A.hist, A.hist_len, &ko, &vo, &lc);
    k_sp_flags<<<bl(m), kT, 0, s>>>(ko, m, nk, A.flag);
    launch_scan_i32(s, A.flag, m, A.ridx, A.bsum, &lc);
    int64_t nruns = 0;
    cudaMemcpyAsync(&nruns, A.ridx + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    k_sp_runs<<<bl(m), kT, 0, s>>>(ko, A.flag, A.ridx, m, nk, A.rstart, A.rx, A.gflag);
    k_sp_entries<<<bl(nruns), kT, 0, s>>>(A.rstart, nruns, vo, A.z, A.chain, cs, r0, A.w);
    lc += 3;
    {   // runs longer than kLong: chunked CTA sums, combined in chunk order
      k_sp_long_flag<<<bl(nruns), kT, 0, s>>>(A.rstart, nruns, A.lflag);
      launch_scan_i32(s, A.lflag, nruns, A.lidx, A.bsum, &lc);
      int64_t nlong = 0;
      cudaMemcpyAsync(&nlong, A.lidx + nruns, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (nlong > 0) {
        k_sp_long_list<<<bl(nruns), kT, 0, s>>>(A.lflag, A.lidx, nruns, A.rstart, A.llist, A.lnch);
        launch_scan_i32(s, A.lnch, nlong, A.lchoff, A.bsum, &lc);
        int64_t nchunks = 0;
        cudaMemcpyAsync(&nchunks, A.lchoff + nlong, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        k_sp_chunk_map<<<bl(nlong), kT, 0, s>>>(A.lchoff, nlong, A.lchl);
        k_sp_long_chunks<<<(unsigned)nchunks, kT, 0, s>>>(A.lchl, A.lchoff, A.llist, A.rstart, vo, A.z, A.chain,
                                                          cs, r0, A.gparts);
        k_sp_long_combine<<<bl(nlong * r0), kT, 0, s>>>(A.llist, A.lchoff, nlong, A.gparts, cs, r0, A.w);
        lc += 5;
      }
      lc += 1;
    }
    double* core = A.C + A.core_off[k];
    if (k == d - 1) {
      cudaMemsetAsync(core, 0, (size_t)r0 * nk * sizeof(double), s);
      k_sp_last_fill<<<bl(nruns), kT, 0, s>>>(A.rx, A.w, nruns, cs, r0, nk, core);
      ++lc;
      break;
    }
    launch_scan_i32(s, A.gflag, nruns, A.gidx, A.bsum, &lc);
    int64_t ngroups = 0;
    cudaMemcpyAsync(&ngroups, A.gidx + nruns, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    k_sp_gstart<<<bl(nruns), kT, 0, s>>>(A.gflag, A.gidx, nruns, A.gstart);
    k_sp_rgroup<<<bl(nruns), kT, 0, s>>>(A.gidx, A.gflag, nruns, A.rgroup);
    if (W > kSpRightMax) {   // right Gram path
      if (ngroups > kSpRightMax || W > A.Wr_max || !A.Md) {
        *msg = "spectral init: step " + std::to_string(k) + " has r_{k-1} n_k = " + std::to_string(W) +
               " > 1024 rows and " + std::to_string(ngroups) + " nonzero columns (both above 1024)";
        return TT_ERR_ARG;
      }
      const int64_t Q = ngroups;
      cudaMemsetAsync(A.Md, 0, (size_t)W * Q * sizeof(double), s);
      k_sp_dense_M<<<bl(nruns), kT, 0, s>>>(A.rx, A.rgroup, A.w, nruns, cs, r0, nk, Q, A.Md);
      k_sp_gram_right<<<bl(Q * Q), kT, 0, s>>>(A.Md, W, Q, A.Gr);
      k_sp_jacobi<<<1, kJT, 0, s>>>(A.Gr, A.Vr, (int)Q, 1, (int)Q, r1, A.Vsel, 40, A.lam);
      k_sp_right_core<<<bl((int64_t)W * r1), kT, 0, s>>>(A.Md, A.Vsel, A.lam, W, Q, r1, core);
      k_sp_mgs<<<1, 512, 0, s>>>(core, W, r1);
      k_sp_chain<<<bl(m), kT, 0, s>>>(A.Ppos, A.Spre, m, D, k, core, r0, r1, A.chain, cs);
      lc += 8;
      continue;
    }
    // runs of each x in group order: stable radix sort of the run indices by x, offsets by x
    k_sp_xkeys<<<bl(nruns), kT, 0, s>>>(A.rx, nruns, A.keys, A.vals);
    {
      int xb = 1;
      while ((1 << xb) < nk) ++xb;
      uint64_t* kx;
      uint32_t* vx;
      radix_sort_pairs(s, A.keys, A.vals, A.ktmp, A.vtmp, nruns, xb, A.hist, A.hist_len, &kx, &vx, &lc);
      k_sp_xoffs<<<bl(nruns), kT, 0, s>>>(kx, vx, nruns, nk, A.xoff, A.byx);
      lc += 2;
    }
    const int64_t WW = (int64_t)W * W;
    int nparts = (int)std::max<int64_t>(1, std::min<int64_t>((4 * 148 + nk - 1) / nk, A.gram_parts_cap / WW));
    const int R = r0 <= 8 ? 8 : (r0 <= 16 ? 16 : 32);
    const size_t len = (size_t)R * R * nk;
    const int nwg = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024 - 3 * kGB * 8) / (len * 8)));
    const size_t smem = len * nwg * sizeof(double) + 3 * kGB * sizeof(int64_t);
    dim3 grid(nk, nparts);
    if (R == 8)
      k_sp_gram<8><<<grid, 32 * nwg, smem, s>>>(A.byx, A.xoff, A.gstart, A.rgroup, A.rx, A.w, cs, r0, nk,
                                                nparts, A.gparts);
    else if (R == 16)
      k_sp_gram<16><<<grid, 32 * nwg, smem, s>>>(A.byx, A.xoff, A.gstart, A.rgroup, A.rx, A.w, cs, r0, nk,
                                                 nparts, A.gparts);
    else
      k_sp_gram<32><<<grid, 32 * nwg, smem, s>>>(A.byx, A.xoff, A.gstart, A.rgroup, A.rx, A.w, cs, r0, nk,
                                                 nparts, A.gparts);
    k_sp_gram_reduce<<<bl(WW), kT, 0, s>>>(A.gparts, nparts, WW, A.G);
    lc += 7;
    k_sp_jacobi<<<1, kJT, 0, s>>>(A.G, A.V, W, r0, nk, r1, core, 40);
    k_sp_chain<<<bl(m), kT, 0, s>>>(A.Ppos, A.Spre, m, D, k, core, r0, r1, A.chain, cs);
    lc += 5;
  }
  *launches += lc;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *msg = std::string("spectral init kernels: ") + cudaGetErrorString(e);
    return TT_ERR_CUDA;
  }
  return TT_OK;
}

}  // namespace prgd
