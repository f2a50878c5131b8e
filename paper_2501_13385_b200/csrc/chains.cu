// chains.cu — the per-sample chain path over Omega: the paper's "fast
// recursive computations" as hand-written kernels, used for shapes whose
// prefix / suffix tables would not fit (the planner's table limits) and selectable with
// tt_set_path.  Every sample's entry is a chain of slice products, its left
// and right interface vectors are the rows of T^{<=k-1} and columns of T^{>=k+1}
// (PAPER.md:99-110), and the gradient contraction of `equ: tsp in nm` is, per
// mode k and slice j, the segmented product  L_{k,j}^T diag(ghat) R_{k,j}  over the samples of
// the per-mode bucket (k, j) (A0).
//
//   A0  per-mode buckets: stable LSD radix sort of the sample ids by x_{s,k} (sort.cu) -> perm_k,
//       offs_k; buckets cut into pieces of <= P samples (fixed order, deterministic sums).
//   A1-A2  k_chain_eval<MODE 1>: g_s = T(x_s) - y_s, G lanes per sample, lane j holds entry j of
//       the running row vector, r_{k-1} shuffles + FMAs per mode against the coalesced row
//       C_k(i, x_k, :) (the ABI core layout [r][n][r'] keeps that row contiguous).
//   A3  k_piece_sumsq + k_piece_reduce: h_{k,j} = sum over bucket (k, j) of g_s^2.
//   A7-A8  k_chain_iface: ghat_s = g_s prod_k phi_{k,x_k}^{-1} and the interfaces of the
//       left-orthogonal U: IL_k(s) = U^{<=k-1}(x_s) (k = 1..d-1), IR_k(s) = U^{>=k}(:, x_s)
//       (k = 1..d-1), materialised in HBM [k][s][r_k].
//   A9  k_piece_contract: per piece of bucket (k, j), the r_k x r_{k+1} block
//       sum_s ghat_s IL_k(s) IR_{k+1}(s)^T — on the FP64 tensor cores (DMMA m8n8k4) when the piece
//       holds >= kDmmaMin samples, as warp-level rank-1 updates otherwise — then k_piece_reduce
//       sums each bucket's pieces in order into Y_k(:, j, :).
//   Adaptive step denominator: k_tangent_cores builds the block TT of the tangent vector
//       D = sum_k [Ttil_1 .. A_k .. Ttil_d] and k_chain_eval<MODE 2> sums
//       D(x_s)^2 (ranks 2r <= 64: 32 lanes x 2 entries).
#include "prgd_internal.cuh"

namespace prgd {
namespace {

constexpr int kT = 256;
constexpr int kPieceThreads = 128;
constexpr int kBatch = 32;       // samples staged per contraction batch
constexpr int kDmmaMin = 32;     // piece size from which the contraction runs on DMMA

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Buckets e = phi_off[k] + j of all modes; per-mode offsets concatenated: mode k's n_k + 1
// entries start at offs_cat[phi_off[k] + k], so bucket e spans [offs_cat[e + k], offs_cat[e + k + 1]).
__device__ __forceinline__ int bucket_mode(const ChainTT& tt, int64_t e) {
  int k = 0;
  while (k + 1 < tt.d && tt.phi_off[k + 1] <= e) ++k;
  return k;
}

// One chain step for a group of G lanes holding a row vector a (entry j = lane + G w in slot w):
// out(j) = sum_{i < r0} a(i) core[(i n + x) r1 + j],  j < r1.  Fully unrolled over the
// compile-time group rank G V with predication on the runtime ranks: the rows are loaded in
// chunks of up to 8 (all loads of a chunk in flight together, each a coalesced 8 r1-byte row
// of the slice), then a(i) is broadcast by shuffle and accumulated.  All lanes of the warp
// execute it (warp-uniform shapes), so full-mask shuffles are safe.
template <int G, int V>
__device__ __forceinline__ void chain_step(const double (&a)[V], double (&o)[V], const double* __restrict__ core,
                                           int r0, int64_t n, int r1, int64_t x, int lane) {
  constexpr int R = G * V, CH = R < 8 ? R : 8;
#pragma unroll
  for (int w = 0; w < V; ++w) o[w] = 0.0;
#pragma unroll
  for (int i0 = 0; i0 < R; i0 += CH) {
    double c[CH][V];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int i = i0 + u;
      const double* row = core + ((int64_t)i * n + x) * r1;
#pragma unroll
      for (int w = 0; w < V; ++w) {
        const int j = lane + G * w;
        c[u][w] = (i < r0 && j < r1) ? __ldg(row + j) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int i = i0 + u;
      const double ai = __shfl_sync(0xffffffffu, a[i / G], i % G, G);
#pragma unroll
      for (int w = 0; w < V; ++w) o[w] = fma(ai, c[u][w], o[w]);
    }
  }
}

// out(i) = sum_{c < r1} core[(i n + x) r1 + c] b(c),  i < r0 (right-part recursion,
// PAPER.md:102-105), b held like a (one entry per lane, G >= r): lane c forms the products
// core(i, x, c) b(c) for every i (loads coalesced over c), then a transpose-reduction over the
// group (G - 1 shuffles) leaves out(lane) in lane `lane`.
template <int G>
__device__ __forceinline__ double chain_step_right(double b, const double* __restrict__ core, int r0,
                                                   int64_t n, int r1, int64_t x, int lane) {
  double p[G];
#pragma unroll
  for (int i = 0; i < G; ++i)
    p[i] = (i < r0 && lane < r1) ? __ldg(core + ((int64_t)i * n + x) * r1 + lane) * b : 0.0;
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < o; ++j) {
      const double send = up ? p[j] : p[j + o];
      const double keep = up ? p[j + o] : p[j];
      p[j] = keep + __shfl_xor_sync(0xffffffffu, send, o, G);
    }
  }
  return p[0];
}

// MODE 0: out[s] = T(x_s); MODE 1: out[s] = T(x_s) - y[s] (pass A residual g); MODE 2:
// out[s] = T(x_s)^2 (adaptive denominator terms).  idx: int32 [m][d] sample-major (the ABI
// layout).  Out-of-range indices set *index_err and evaluate as 0.
template <int G, int V, int MODE>
__global__ void __launch_bounds__(kT) k_chain_eval(const int32_t* __restrict__ idx, int64_t m, ChainTT tt,
                                                   const double* __restrict__ cores,
                                                   const double* __restrict__ y, double* __restrict__ out,
                                                   const Scalars* sc, int* index_err) {
  if (MODE == 2 && sc && sc->noop) return;
  const int lane = threadIdx.x & (G - 1);
  const int64_t grp0 = (blockIdx.x * (int64_t)kT + threadIdx.x) / G;
  const int64_t ngrp = (gridDim.x * (int64_t)kT) / G;
  // warp-uniform trip count: every group of the warp runs the same number of iterations
  const int64_t wgrp0 = grp0 - (threadIdx.x & 31) / G;
  for (int64_t base = wgrp0; base < m; base += ngrp) {
    const int64_t s = grp0 + (base - wgrp0);
    const bool act = s < m;
    const int32_t* xs = idx + (act ? s : 0) * tt.d;
    double a[V], o[V];
    bool bad = false;
    for (int k = 0; k < tt.d; ++k) {
      int64_t x = act ? (int64_t)__ldg(xs + k) : 0;
      if (x < 0 || x >= tt.n[k]) {
        bad = true;
        x = 0;
      }
      const double* core = cores + tt.off[k];
      if (k == 0) {
#pragma unroll
        for (int w = 0; w < V; ++w) {
          const int j = lane + G * w;
          a[w] = j < tt.r[1] ? __ldg(core + x * tt.r[1] + j) : 0.0;
        }
      } else {
        chain_step<G, V>(a, o, core, tt.r[k], tt.n[k], tt.r[k + 1], x, lane);
#pragma unroll
        for (int w = 0; w < V; ++w) a[w] = o[w];
      }
    }
    const double v = __shfl_sync(0xffffffffu, a[0], 0, G);
    if (act && lane == 0) {
      if (bad && index_err) atomicOr(index_err, 1);
      out[s] = MODE == 0 ? v : (MODE == 1 ? v - y[s] : v * v);
    }
  }
}

// A7-A8: ghat_s and the interfaces of U at sample s.
template <int G>
__global__ void __launch_bounds__(kT) k_chain_iface(const int32_t* __restrict__ idx, int64_t m, ChainTT tt,
                                                    const double* __restrict__ U,
                                                    const double* __restrict__ phi,
                                                    const double* __restrict__ g, double* __restrict__ ghat,
                                                    double* __restrict__ IL, double* __restrict__ IR,
                                                    const Scalars* sc) {
  if (sc->noop) return;
  const int lane = threadIdx.x & (G - 1);
  const int64_t grp0 = (blockIdx.x * (int64_t)kT + threadIdx.x) / G;
  const int64_t ngrp = (gridDim.x * (int64_t)kT) / G;
  const int64_t wgrp0 = grp0 - (threadIdx.x & 31) / G;
  const int d = tt.d;
  for (int64_t base = wgrp0; base < m; base += ngrp) {
    const int64_t s = grp0 + (base - wgrp0);
    const bool act = s < m;
    const int32_t* xs = idx + (act ? s : 0) * d;
    double wprod = 1.0;
    for (int k = 0; k < d; ++k) wprod *= __ldg(phi + tt.phi_off[k] + __ldg(xs + k));
    if (act && lane == 0) ghat[s] = g[s] / wprod;          // prod_k phi^{-1}: one division
    double a[1], o[1];
    // left interfaces IL_k = U^{<=k-1}(x_s), k = 1..d-1 (row vectors of length r_k)
    for (int k = 0; k + 1 < d; ++k) {
      const int64_t x = __ldg(xs + k);
      const double* core = U + tt.off[k];
      if (k == 0) {
        a[0] = lane < tt.r[1] ? __ldg(core + x * tt.r[1] + lane) : 0.0;
      } else {
        chain_step<G, 1>(a, o, core, tt.r[k], tt.n[k], tt.r[k + 1], x, lane);
        a[0] = o[0];
      }
      if (act && lane < tt.r[k + 1]) IL[tt.il_off[k + 1] + s * tt.r[k + 1] + lane] = a[0];
    }
    // right interfaces IR_k = U^{>=k}(:, x_s), k = d-1..1 (column vectors of length r_k)
    for (int k = d - 1; k >= 1; --k) {
      const int64_t x = __ldg(xs + k);
      const double* core = U + tt.off[k];
      if (k == d - 1) {
        a[0] = lane < tt.r[k] ? __ldg(core + (int64_t)lane * tt.n[k] + x) : 0.0;   // r_d = 1
      } else {
        a[0] = chain_step_right<G>(a[0], core, tt.r[k], tt.n[k], tt.r[k + 1], x, lane);
      }
      if (act && lane < tt.r[k]) IR[tt.il_off[k] + s * tt.r[k] + lane] = a[0];
    }
  }
}

// A3: per piece, sum of g^2 over its samples (one warp per piece, fixed order).
__global__ void k_piece_sumsq(const int4* __restrict__ pieces, int64_t npieces, const int32_t* __restrict__ perm,
                              int64_t m, const double* __restrict__ g, double* __restrict__ part) {
  const int64_t p = (blockIdx.x * (int64_t)kT + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= npieces) return;
  const int4 pc = pieces[p];
  const int32_t* pk = perm + (int64_t)pc.y * m;
  double sacc = 0.0;
  for (int t = pc.z + lane; t < pc.w; t += 32) {
    const double v = g[pk[t]];
    sacc = fma(v, v, sacc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
  if (lane == 0) part[p] = sacc;
}

// A9: per piece of bucket (k, j), the block sum_s ghat_s IL_k(s) IR_{k+1}(s)^T (r0 x r1),
// written to part[p * stride ..].
__global__ void __launch_bounds__(kPieceThreads) k_piece_contract(const int4* __restrict__ pieces,
                                                                  const int32_t* __restrict__ perm,
                                                                  int64_t m, ChainTT tt,
                                                                  const double* __restrict__ ghat,
                                                                  const double* __restrict__ IL,
                                                                  const double* __restrict__ IR,
                                                                  double* __restrict__ part, int stride,
                                                                  const Scalars* sc) {
  __shared__ double Ls[kBatch][kMaxRank + 1];
  __shared__ double Rs[kBatch][kMaxRank + 1];
  if (sc->noop) return;
  const int4 pc = pieces[blockIdx.x];
  const int k = pc.y, t0 = pc.z, t1 = pc.w;
  const int r0 = tt.r[k], r1 = tt.r[k + 1], d = tt.d;
  const int32_t* pk = perm + (int64_t)k * m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool use_mma = (t1 - t0) >= kDmmaMin;
  const int gid = lane >> 2, tq = lane & 3;
  const int mt = (r0 + 7) >> 3, nt = (r1 + 7) >> 3, ntile = mt * nt;   // <= 16 tiles
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  for (int b0 = t0; b0 < t1; b0 += kBatch) {
    const int nb = min(kBatch, t1 - b0);
    __syncthreads();
    for (int e = tid; e < kBatch * (kMaxRank + 1); e += kPieceThreads) {
      const int t = e / (kMaxRank + 1), c = e - t * (kMaxRank + 1);
      double lv = 0.0, rv = 0.0;
      if (t < nb) {
        const int64_t s = pk[b0 + t];
        if (c < r0) lv = k == 0 ? 1.0 : IL[tt.il_off[k] + s * r0 + c];
        if (c < r1) rv = ghat[s] * (k == d - 1 ? 1.0 : IR[tt.il_off[k + 1] + s * r1 + c]);
      }
      Ls[t][c] = lv;
      Rs[t][c] = rv;
    }
    __syncthreads();
    if (use_mma) {
      // warp w owns tiles w, w+4, ...; acc[2q], acc[2q+1] = D[gid][2tq], D[gid][2tq+1] of its q-th tile
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tile = warp + 4 * q;
        if (tile < ntile) {
          const int I = tile / nt, J = tile - I * nt;
          for (int kk = 0; kk < nb; kk += 4) {
            const int t = kk + tq;   // rows >= nb are zero-filled
            dmma_c(acc[2 * q], acc[2 * q + 1], Ls[t][I * 8 + gid < kMaxRank ? I * 8 + gid : kMaxRank],
                   Rs[t][J * 8 + gid < kMaxRank ? J * 8 + gid : kMaxRank]);
          }
        }
      }
    } else {
      // rank-1 updates, thread per output element (<= 8 per thread)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = tid + q * kPieceThreads;
        if (e < r0 * r1) {
          const int i = e / r1, c = e - i * r1;
          double sacc = acc[q];
          for (int t = 0; t < nb; ++t) sacc = fma(Ls[t][i], Rs[t][c], sacc);
          acc[q] = sacc;
        }
      }
    }
  }
  double* out = part + (int64_t)blockIdx.x * stride;
  if (use_mma) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int tile = warp + 4 * q;
      if (tile < ntile) {
        const int I = tile / nt, J = tile - I * nt;
        const int i = I * 8 + gid, c = J * 8 + 2 * tq;
        if (i < r0 && c < r1) out[i * r1 + c] = acc[2 * q];
        if (i < r0 && c + 1 < r1) out[i * r1 + c + 1] = acc[2 * q + 1];
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * kPieceThreads;
      if (e < r0 * r1) out[e] = acc[q];
    }
  }
}

// Sum each bucket's pieces in order: bucket e = phi_off[k] + j.  width 1: h[e] (A3); else
// Y_k(i, j, c) with i < r_k, c < r_{k+1} (A9).
__global__ void k_piece_reduce(const int64_t* __restrict__ pbase, int64_t nbuckets, ChainTT tt,
                               const double* __restrict__ part, int stride, bool ymode,
                               double* __restrict__ out, const Scalars* sc) {
  if (ymode && sc->noop) return;
  const int64_t e = blockIdx.x;
  if (e >= nbuckets) return;
  const int k = bucket_mode(tt, e);
  const int64_t j = e - tt.phi_off[k];
  const int64_t p0 = pbase[e], p1 = pbase[e + 1];
  if (!ymode) {
    if (threadIdx.x == 0) {
      double sacc = 0.0;
      for (int64_t p = p0; p < p1; ++p) sacc += part[p];
      out[e] = sacc;
    }
    return;
  }
  const int r0 = tt.r[k], r1 = tt.r[k + 1];
  for (int c = threadIdx.x; c < r0 * r1; c += blockDim.x) {
    double sacc = 0.0;
    for (int64_t p = p0; p < p1; ++p) sacc += part[p * stride + c];
    const int i = c / r1, cc = c - i * r1;
    out[tt.off[k] + ((int64_t)i * tt.n[k] + j) * r1 + cc] = sacc;
  }
}

// pieces of every bucket: npieces(e) = ceil(cnt(e) / P)
__global__ void k_piece_count(const int64_t* __restrict__ offs_cat, int64_t nb, ChainTT tt, int P,
                              int* __restrict__ np) {
  const int64_t e = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (e >= nb) return;
  const int k = bucket_mode(tt, e);
  const int64_t c = offs_cat[e + k + 1] - offs_cat[e + k];
  np[e] = (int)((c + P - 1) / P);
}

__global__ void k_piece_fill(const int64_t* __restrict__ offs_cat, const int64_t* __restrict__ pbase,
                             int64_t nb, ChainTT tt, int P, int4* __restrict__ pieces) {
  const int64_t e = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (e >= nb) return;
  const int k = bucket_mode(tt, e);
  const int64_t lo = offs_cat[e + k], hi = offs_cat[e + k + 1];
  int64_t q = pbase[e];
  for (int64_t t = lo; t < hi; t += P, ++q) pieces[q] = make_int4((int)e, k, (int)t, (int)min(hi, t + P));
}

// per-mode keys: key = x_{s,k}, val = s; flags out-of-range indices
__global__ void k_mode_keys(const int32_t* __restrict__ idx, int64_t m, int d, int k, int nk,
                            uint64_t* __restrict__ keys, uint32_t* __restrict__ vals, int* index_err) {
  const int64_t s = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (s >= m) return;
  const int x = idx[s * d + k];
  if (x < 0 || x >= nk) atomicOr(index_err, 1);
  keys[s] = (uint64_t)(x < 0 ? 0 : (x >= nk ? nk - 1 : x));
  vals[s] = (uint32_t)s;
}

// sorted keys/values -> perm_k and bucket offsets offs_k[0..nk]
__global__ void k_mode_after_sort(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t m,
                                  int64_t nk, int32_t* __restrict__ perm, int64_t* __restrict__ offs) {
  const int64_t t = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (t >= m) return;
  perm[t] = (int32_t)vals[t];
  const int64_t x = (int64_t)keys[t];
  const int64_t xp = t == 0 ? -1 : (int64_t)keys[t - 1];
  for (int64_t q = xp + 1; q <= x; ++q) offs[q] = t;
  if (t == m - 1)
    for (int64_t q = x + 1; q <= nk; ++q) offs[q] = m;
}

// Block TT of the tangent vector D = sum_k [Ttil_1 .. A_k .. Ttil_d] with
// Ttil = U / phi, A = Ahat / phi (A11): first [A_1, Ttil_1], middle [[Ttil_k, 0], [A_k, Ttil_k]],
// last [[Ttil_d], [A_d]].  One CTA per core; output offsets b_off (ranks 2 r).
__global__ void k_tangent_cores(const double* __restrict__ U, const double* __restrict__ Ah,
                                const double* __restrict__ phi, ChainTT tt, ChainTT bt,
                                double* __restrict__ out, const Scalars* sc) {
  if (sc->noop) return;
  const int k = blockIdx.x, d = tt.d;
  const int r0 = tt.r[k], nk = tt.n[k], r1 = tt.r[k + 1];
  const int R0 = bt.r[k], R1 = bt.r[k + 1];
  const double* u = U + tt.off[k];
  const double* a = Ah + tt.off[k];
  const double* ph = phi + tt.phi_off[k];
  double* o = out + bt.off[k];
  const int64_t tot = (int64_t)R0 * nk * R1;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t row = e / ((int64_t)nk * R1);
    const int64_t rem = e - row * nk * R1;
    const int64_t j = rem / R1;
    const int col = (int)(rem - j * R1);
    const double iv = 1.0 / ph[j];
    double v = 0.0;
    if (k == 0) {                               // [A | Ttil], 1 x n x 2 r1
      v = col < r1 ? a[j * r1 + col] : u[j * r1 + (col - r1)];
    } else if (k == d - 1) {                    // [[Ttil], [A]], 2 r0 x n x 1
      v = row < r0 ? u[row * nk + j] : a[(row - r0) * nk + j];
    } else {
      if (row < r0) v = col < r1 ? u[(row * nk + j) * r1 + col] : 0.0;
      else v = col < r1 ? a[((row - r0) * nk + j) * r1 + col] : u[((row - r0) * nk + j) * r1 + (col - r1)];
    }
    o[e] = v * iv;
  }
}

template <int G, int V, int MODE>
void eval_launch(cudaStream_t s, const int32_t* idx, int64_t m, const ChainTT& tt, const double* cores,
                 const double* y, double* out, const Scalars* sc, int* index_err) {
  const int64_t thr = m * G;
  const unsigned grid = (unsigned)std::min<int64_t>(blocks_for(thr, kT), 148 * 16);
  k_chain_eval<G, V, MODE><<<grid, kT, 0, s>>>(idx, m, tt, cores, y, out, sc, index_err);
}

template <int MODE>
void eval_dispatch(cudaStream_t s, const int32_t* idx, int64_t m, const ChainTT& tt, const double* cores,
                   const double* y, double* out, const Scalars* sc, int* index_err) {
  int rmax = 1;
  for (int k = 0; k <= tt.d; ++k) rmax = std::max(rmax, tt.r[k]);
  if (rmax <= 4) eval_launch<4, 1, MODE>(s, idx, m, tt, cores, y, out, sc, index_err);
  else if (rmax <= 8) eval_launch<8, 1, MODE>(s, idx, m, tt, cores, y, out, sc, index_err);
  else if (rmax <= 16) eval_launch<16, 1, MODE>(s, idx, m, tt, cores, y, out, sc, index_err);
  else if (rmax <= 32) eval_launch<32, 1, MODE>(s, idx, m, tt, cores, y, out, sc, index_err);
  else eval_launch<32, 2, MODE>(s, idx, m, tt, cores, y, out, sc, index_err);
}

}  // namespace

int chain_piece_size(int64_t m, int d, int rmax) {
  // partial blocks bounded by ~2^25 doubles (256 MB): P >= d m r^2 / 2^25, at least 256
  const int64_t need = (int64_t)d * m * rmax * rmax / ((int64_t)1 << 25) + 1;
  int64_t P = 256;
  while (P < need) P <<= 1;
  return (int)std::min<int64_t>(P, (int64_t)1 << 30);
}

void launch_chain_eval(cudaStream_t s, int mode, const int32_t* idx, int64_t m, const ChainTT& tt,
                       const double* cores, const double* y, double* out, const Scalars* sc,
                       int* index_err, int64_t* launches) {
  if (m <= 0) return;
  if (mode == 0) eval_dispatch<0>(s, idx, m, tt, cores, y, out, sc, index_err);
  else if (mode == 1) eval_dispatch<1>(s, idx, m, tt, cores, y, out, sc, index_err);
  else eval_dispatch<2>(s, idx, m, tt, cores, y, out, sc, index_err);
  ++*launches;
}

void launch_chain_iface(cudaStream_t s, const int32_t* idx, int64_t m, const ChainTT& tt, const double* U,
                        const double* phi, const double* g, double* ghat, double* IL, double* IR,
                        const Scalars* sc, int64_t* launches) {
  if (m <= 0) return;
  int rmax = 1;
  for (int k = 0; k <= tt.d; ++k) rmax = std::max(rmax, tt.r[k]);
  const int G = rmax <= 4 ? 4 : (rmax <= 8 ? 8 : (rmax <= 16 ? 16 : 32));
  const unsigned grid = (unsigned)std::min<int64_t>(blocks_for(m * G, kT), 148 * 16);
  if (G == 4) k_chain_iface<4><<<grid, kT, 0, s>>>(idx, m, tt, U, phi, g, ghat, IL, IR, sc);
  else if (G == 8) k_chain_iface<8><<<grid, kT, 0, s>>>(idx, m, tt, U, phi, g, ghat, IL, IR, sc);
  else if (G == 16) k_chain_iface<16><<<grid, kT, 0, s>>>(idx, m, tt, U, phi, g, ghat, IL, IR, sc);
  else k_chain_iface<32><<<grid, kT, 0, s>>>(idx, m, tt, U, phi, g, ghat, IL, IR, sc);
  ++*launches;
}

void launch_chain_h(cudaStream_t s, const ChainPieces& pc, const ChainTT& tt, int64_t m, const double* g,
                    double* h, int64_t* launches) {
  if (pc.npieces > 0) {
    k_piece_sumsq<<<blocks_for(pc.npieces * 32, kT), kT, 0, s>>>(pc.pieces, pc.npieces, pc.perm, m, g, pc.part);
    ++*launches;
  }
  k_piece_reduce<<<(unsigned)pc.nbuckets, 32, 0, s>>>(pc.pbase, pc.nbuckets, tt, pc.part, 1, false, h, nullptr);
  ++*launches;
}

void launch_chain_contract(cudaStream_t s, const ChainPieces& pc, const ChainTT& tt, int64_t m,
                           const double* ghat, const double* IL, const double* IR, double* Y,
                           const Scalars* sc, int64_t* launches) {
  if (pc.npieces > 0) {
    k_piece_contract<<<(unsigned)pc.npieces, kPieceThreads, 0, s>>>(pc.pieces, pc.perm, m, tt, ghat, IL, IR,
                                                                    pc.part, pc.stride, sc);
    ++*launches;
  }
  k_piece_reduce<<<(unsigned)pc.nbuckets, 128, 0, s>>>(pc.pbase, pc.nbuckets, tt, pc.part, pc.stride, true, Y, sc);
  ++*launches;
}

void launch_mode_keys(cudaStream_t s, const int32_t* idx, int64_t m, int d, int k, int nk, uint64_t* keys,
                      uint32_t* vals, int* index_err, int64_t* launches) {
  if (m <= 0) return;
  k_mode_keys<<<blocks_for(m, kT), kT, 0, s>>>(idx, m, d, k, nk, keys, vals, index_err);
  ++*launches;
}

void launch_mode_after_sort(cudaStream_t s, const uint64_t* keys, const uint32_t* vals, int64_t m, int64_t nk,
                            int32_t* perm, int64_t* offs, int64_t* launches) {
  if (m <= 0) return;
  k_mode_after_sort<<<blocks_for(m, kT), kT, 0, s>>>(keys, vals, m, nk, perm, offs);
  ++*launches;
}

void launch_piece_count(cudaStream_t s, const int64_t* offs_cat, const ChainTT& tt, int64_t nb, int P,
                        int* np, int64_t* launches) {
  k_piece_count<<<blocks_for(nb, kT), kT, 0, s>>>(offs_cat, nb, tt, P, np);
  ++*launches;
}

void launch_piece_fill(cudaStream_t s, const int64_t* offs_cat, const int64_t* pbase, int64_t nb,
                       const ChainTT& tt, int P, int4* pieces, int64_t* launches) {
  k_piece_fill<<<blocks_for(nb, kT), kT, 0, s>>>(offs_cat, pbase, nb, tt, P, pieces);
  ++*launches;
}

void launch_tangent_cores(cudaStream_t s, const double* U, const double* Ahat, const double* phi,
                          const ChainTT& tt, const ChainTT& bt, double* out, const Scalars* sc,
                          int64_t* launches) {
  k_tangent_cores<<<tt.d, kT, 0, s>>>(U, Ahat, phi, tt, bt, out, sc);
  ++*launches;
}

}  // namespace prgd
