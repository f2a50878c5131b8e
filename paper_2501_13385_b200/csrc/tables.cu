// tables.cu — dense left/right partial-product tables and the backward recursions
// that turn the two per-sample accumulations of pass B into every Y_k.
//
// Left table level k (prefix length k, 0-based cores 0..k-1):
//   A_k[(p, j), c] = sum_i A_{k-1}[p, i] C_{k-1}[i, j, c]
// i.e. A_k = A_{k-1} R(C_{k-1}) reshaped; row index p*n + j (x_0 most significant).
// Right table level k (suffix from core k):
//   B_k[(j + n q), i] = sum_c C_k[i, j, c] B_{k+1}[q, c]
// Backward recursions (`equ: tsp in nm`):
//   E_k[p, i]   = sum_j sum_c U_k[i, j, c] E_{k+1}[p n_k + j, c]
//   F_{k+1}[q,c]= sum_j sum_i F_k[j + n_k q, i] U_k[i, j, c]
//   Y_k[i,j,c]  = sum_p A_k[p, i] E_{k+1}[p n_k + j, c]     (left modes, k < KL)
//   Y_k[i,j,c]  = sum_q F_k[j + n_k q, i] B_{k+1}[q, c]     (right modes, k >= KL)
#include <algorithm>

#include "prgd_internal.cuh"

namespace prgd {
namespace {

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

constexpr int kTabThreads = 256;
constexpr int kRowsPerBlock = 64;      // parent rows per (slice, block) of a table level
constexpr int kRecRows = 128;          // output rows per block of the E/F recursions

// Left table level: block (j, parent-row range).  out[(p n_k + j), c] =
// scale * sum_i in[p, i] C(i, j, c); slice C(:, j, :) staged in shared memory.
__global__ void __launch_bounds__(kTabThreads) k_table_left(
    const double* __restrict__ in, int ld_in, const double* __restrict__ core, int r0, int nk,
    int r1, double* __restrict__ out, int ld_out, int64_t nparent,
    const double* __restrict__ rowscale, const Scalars* sc) {
  if (sc && sc->noop) return;
  __shared__ double cs[kMaxRank * kMaxRank];
  const int j = blockIdx.x;
  for (int t = threadIdx.x; t < r0 * r1; t += blockDim.x) {
    const int i = t / r1, c = t - i * r1;
    cs[t] = core[((int64_t)i * nk + j) * r1 + c];
  }
  __syncthreads();
  const int lanes = ld_out, per = blockDim.x / lanes;
  const int pl = threadIdx.x / lanes, c = threadIdx.x - pl * lanes;
  if (pl >= per) return;
  const int64_t p0 = (int64_t)blockIdx.y * kRowsPerBlock;
  for (int64_t p = p0 + pl; p < p0 + kRowsPerBlock && p < nparent; p += per) {
    const int64_t row = p * nk + j;
    double acc = 0.0;
    if (c < r1) {
      if (in == nullptr) {
        acc = cs[c];
      } else {
        const double* a = in + p * ld_in;
        for (int i = 0; i < r0; ++i) acc = fma(a[i], cs[i * r1 + c], acc);
      }
      if (rowscale) acc *= rowscale[row];
    }
    out[row * ld_out + c] = acc;
  }
}

// Right table level: block (j, parent-row range).  out[(j + n_k q), i] =
// scale * sum_c C(i, j, c) in[q, c]; slice staged transposed ([c][i]).
__global__ void __launch_bounds__(kTabThreads) k_table_right(
    const double* __restrict__ in, int ld_in, const double* __restrict__ core, int r0, int nk,
    int r1, double* __restrict__ out, int ld_out, int64_t nparent,
    const double* __restrict__ rowscale, const Scalars* sc) {
  if (sc && sc->noop) return;
  __shared__ double ct[kMaxRank * kMaxRank];
  const int j = blockIdx.x;
  for (int t = threadIdx.x; t < r0 * r1; t += blockDim.x) {
    const int i = t / r1, c = t - i * r1;
    ct[c * r0 + i] = core[((int64_t)i * nk + j) * r1 + c];
  }
  __syncthreads();
  const int lanes = ld_out, per = blockDim.x / lanes;
  const int ql = threadIdx.x / lanes, i = threadIdx.x - ql * lanes;
  if (ql >= per) return;
  const int64_t q0 = (int64_t)blockIdx.y * kRowsPerBlock;
  for (int64_t q = q0 + ql; q < q0 + kRowsPerBlock && q < nparent; q += per) {
    const int64_t row = (int64_t)j + (int64_t)nk * q;
    double acc = 0.0;
    if (i < r0) {
      if (in == nullptr) {
        acc = ct[i];
      } else {
        const double* b = in + q * ld_in;
        for (int c = 0; c < r1; ++c) acc = fma(ct[c * r0 + i], b[c], acc);
      }
      if (rowscale) acc *= rowscale[row];
    }
    out[row * ld_out + i] = acc;
  }
}

// E_k[p, i] = sum_{j,c} U_k(i, j, c) E_{k+1}[p n_k + j, c]; the core is staged
// transposed ([j][c][i]) once per block (in chunks of slices) for kRecRows rows.
// (grid.y > 1: block y takes the slices j in [y nk / grid.y, (y+1) nk / grid.y) and writes a
// partial output to part[y], summed in y order by k_jsplit_reduce)
__global__ void __launch_bounds__(kTabThreads) k_E_down(
    const double* __restrict__ Ein, int ld_in, const double* __restrict__ core, int r0, int nk,
    int r1, double* __restrict__ Eout, int ld_out, int64_t rows, int jchunk, double* __restrict__ part,
    const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ double sm[];
  const int lanes = ld_out, per = blockDim.x / lanes;
  const int pl = threadIdx.x / lanes, i = threadIdx.x - pl * lanes;
  const int64_t p0 = (int64_t)blockIdx.x * kRecRows;
  double acc[kRecRows / (kTabThreads / kMaxRank) + 1];
  const int nloc = (kRecRows + per - 1) / per;
  for (int t = 0; t < nloc; ++t) acc[t] = 0.0;
  const int psz = r1 * r0;
  const int jbeg = (int)((int64_t)blockIdx.y * nk / gridDim.y), jend = (int)((int64_t)(blockIdx.y + 1) * nk / gridDim.y);
  for (int j0 = jbeg; j0 < jend; j0 += jchunk) {
    const int jn = jend - j0 < jchunk ? jend - j0 : jchunk;
    __syncthreads();
    for (int t = threadIdx.x; t < jn * psz; t += blockDim.x) {
      const int jj = t / psz, rem = t - jj * psz;
      const int ii = rem / r1, c = rem - ii * r1;
      sm[(jj * r1 + c) * r0 + ii] = core[((int64_t)ii * nk + j0 + jj) * r1 + c];
    }
    __syncthreads();
    if (pl < per && i < r0) {
      for (int t = 0; t < nloc; ++t) {
        const int64_t p = p0 + pl + (int64_t)t * per;
        if (p >= rows || p >= p0 + kRecRows) break;
        double a = acc[t];
        for (int jj = 0; jj < jn; ++jj) {
          const double* ein = Ein + (p * nk + j0 + jj) * ld_in;
          const double* sl = sm + jj * psz + i;
          for (int c = 0; c < r1; ++c) a = fma(sl[c * r0], ein[c], a);
        }
        acc[t] = a;
      }
    }
  }
  if (pl < per)
    for (int t = 0; t < nloc; ++t) {
      const int64_t p = p0 + pl + (int64_t)t * per;
      if (p >= rows || p >= p0 + kRecRows) break;
      double* dst = gridDim.y > 1 ? part + (int64_t)blockIdx.y * rows * ld_out : Eout;
      dst[p * ld_out + i] = i < r0 ? acc[t] : 0.0;
    }
}

// F_{k+1}[q, c] = sum_{j,i} F_k[j + n_k q, i] U_k(i, j, c); core staged as [j][i][c].
__global__ void __launch_bounds__(kTabThreads) k_F_up(
    const double* __restrict__ Fin, int ld_in, const double* __restrict__ core, int r0, int nk,
    int r1, double* __restrict__ Fout, int ld_out, int64_t rows, int jchunk, double* __restrict__ part,
    const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ double sm[];
  const int lanes = ld_out, per = blockDim.x / lanes;
  const int ql = threadIdx.x / lanes, c = threadIdx.x - ql * lanes;
  const int64_t q0 = (int64_t)blockIdx.x * kRecRows;
  double acc[kRecRows / (kTabThreads / kMaxRank) + 1];
  const int nloc = (kRecRows + per - 1) / per;
  for (int t = 0; t < nloc; ++t) acc[t] = 0.0;
  const int psz = r0 * r1;
  const int jbeg = (int)((int64_t)blockIdx.y * nk / gridDim.y), jend = (int)((int64_t)(blockIdx.y + 1) * nk / gridDim.y);
  for (int j0 = jbeg; j0 < jend; j0 += jchunk) {
    const int jn = jend - j0 < jchunk ? jend - j0 : jchunk;
    __syncthreads();
    for (int t = threadIdx.x; t < jn * psz; t += blockDim.x) {
      const int jj = t / psz, rem = t - jj * psz;
      const int ii = rem / r1, cc = rem - ii * r1;
      sm[t] = core[((int64_t)ii * nk + j0 + jj) * r1 + cc];   // [jj][ii][cc]
    }
    __syncthreads();
    if (ql < per && c < r1) {
      for (int t = 0; t < nloc; ++t) {
        const int64_t q = q0 + ql + (int64_t)t * per;
        if (q >= rows || q >= q0 + kRecRows) break;
        double a = acc[t];
        for (int jj = 0; jj < jn; ++jj) {
          const double* f = Fin + ((int64_t)(j0 + jj) + (int64_t)nk * q) * ld_in;
          const double* sl = sm + jj * psz + c;
          for (int ii = 0; ii < r0; ++ii) a = fma(f[ii], sl[ii * r1], a);
        }
        acc[t] = a;
      }
    }
  }
  if (ql < per)
    for (int t = 0; t < nloc; ++t) {
      const int64_t q = q0 + ql + (int64_t)t * per;
      if (q >= rows || q >= q0 + kRecRows) break;
      double* dst = gridDim.y > 1 ? part + (int64_t)blockIdx.y * rows * ld_out : Fout;
      dst[q * ld_out + c] = c < r1 ? acc[t] : 0.0;
    }
}

constexpr int kYThreads = 128;
constexpr int64_t kTableSmemDoubles = 12288;   // 96 KB of staged slices

// One thread per (j, c) of Y_k and a chunk of the summation index; all r0 values of
// i live in registers.  partial[chunk][i][j][c].
__global__ void __launch_bounds__(kYThreads) k_Y_partial(
    int left, const double* __restrict__ A, int ldA, const double* __restrict__ E, int ldE,
    int64_t nsum, int64_t chunk, int r0, int nk, int r1, double* __restrict__ partial,
    const Scalars* sc) {
  if (sc && sc->noop) return;
  const int64_t njc = (int64_t)nk * r1;
  int64_t jc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (jc >= njc) return;
  const int j = (int)(jc / r1), c = (int)(jc - (int64_t)j * r1);
  int64_t p0 = blockIdx.y * chunk;
  int64_t p1 = p0 + chunk < nsum ? p0 + chunk : nsum;
  double acc[kMaxRank];
#pragma unroll
  for (int i = 0; i < kMaxRank; ++i) acc[i] = 0.0;
  if (left) {
    // Y[i,j,c] += A[p,i] * E[p*nk + j, c]   (A == null: [1], r0 == 1, nsum == 1)
    for (int64_t p = p0; p < p1; ++p) {
      double x = E[(p * nk + j) * ldE + c];
      if (A == nullptr) {
        acc[0] += x;
      } else {
        const double* a = A + p * ldA;
#pragma unroll
        for (int i = 0; i < kMaxRank; ++i)
          if (i < r0) acc[i] = fma(a[i], x, acc[i]);
      }
    }
  } else {
    // Y[i,j,c] += F[j + nk*q, i] * B[q, c]   (B == null: [1], r1 == 1, nsum == 1)
    for (int64_t q = p0; q < p1; ++q) {
      double x = (A == nullptr) ? 1.0 : A[q * ldA + c];
      const double* f = E + ((int64_t)j + (int64_t)nk * q) * ldE;
#pragma unroll
      for (int i = 0; i < kMaxRank; ++i)
        if (i < r0) acc[i] = fma(f[i], x, acc[i]);
    }
  }
  double* out = partial + (int64_t)blockIdx.y * r0 * njc;
#pragma unroll
  for (int i = 0; i < kMaxRank; ++i)
    if (i < r0) out[(int64_t)i * njc + jc] = acc[i];
}

// Fused backward step of one mode k, for r_k n_k r_{k+1} <= 4096:
//  left  (k < K_L): group p, X_p[j][c] = E_{k+1}[p n_k + j, c], v = A_k[p, :]
//        E_k[p, i] = sum_{j,c} U_k(i,j,c) X_p[j][c];   Y_k(i,j,c) += v[i] X_p[j][c]
//  right (k >= K_L): group q, X_q[j][i] = F_k[j + n_k q, i], v = B_{k+1}[q, :]
//        F_{k+1}[q, c] = sum_{j,i} X_q[j][i] U_k(i,j,c); Y_k(i,j,c) += X_q[j][i] v[c]
// G groups are staged per sub-batch; the core is staged once in the order the output
// rows read it; each block writes one split-K partial of Y_k (reduced in chunk order).
constexpr int kBackThreads = 256;
constexpr int kBackNY = 16;
__global__ void __launch_bounds__(kBackThreads) k_back_level(
    int left, const double* __restrict__ X, int ldX, const double* __restrict__ V, int ldV,
    const double* __restrict__ core, int r0, int nk, int r1, double* __restrict__ O, int ldO,
    int64_t ngroups, int64_t chunk, int G, double* __restrict__ partial, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ double sm[];
  const int w = left ? r1 : r0;
  const int vlen = left ? r0 : r1;
  const int olen = left ? r0 : r1;
  const int blk = nk * w;
  const int count = r0 * nk * r1;
  const int njc = nk * r1;
  double* Us = sm;
  double* Xs = Us + count;
  double* Vs = Xs + (int64_t)G * blk;
  for (int t = threadIdx.x; t < count; t += blockDim.x) {
    const int i = t / njc, rem = t - i * njc;
    const int j = rem / r1, c = rem - j * r1;
    const double u = core[t];
    if (left) Us[(j * r1 + c) * r0 + i] = u;
    else Us[(j * r0 + i) * r1 + c] = u;
  }
  double acc[kBackNY];
#pragma unroll
  for (int u = 0; u < kBackNY; ++u) acc[u] = 0.0;
  const int64_t g0 = (int64_t)blockIdx.x * chunk;
  const int64_t g1 = g0 + chunk < ngroups ? g0 + chunk : ngroups;
  for (int64_t gb = g0; gb < g1; gb += G) {
    const int gn = (int)(g1 - gb < G ? g1 - gb : G);
    __syncthreads();
    for (int t = threadIdx.x; t < gn * blk; t += blockDim.x) {
      const int g = t / blk, rem = t - g * blk;
      const int j = rem / w, x = rem - j * w;
      Xs[t] = X[((gb + g) * nk + j) * ldX + x];
    }
    for (int t = threadIdx.x; t < gn * vlen; t += blockDim.x) {
      const int g = t / vlen, x = t - g * vlen;
      Vs[t] = V ? V[(gb + g) * ldV + x] : 1.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kBackNY; ++u) {
      const int o = threadIdx.x + u * kBackThreads;
      if (o < count) {
        const int i = o / njc, jc = o - i * njc;
        const int j = jc / r1, c = jc - j * r1;
        double a = acc[u];
        if (left) {
          for (int g = 0; g < gn; ++g) a = fma(Vs[g * vlen + i], Xs[g * blk + jc], a);
        } else {
          for (int g = 0; g < gn; ++g) a = fma(Xs[g * blk + j * w + i], Vs[g * vlen + c], a);
        }
        acc[u] = a;
      }
    }
    if (O) {
      const int len = nk * w;
      for (int pr = threadIdx.x; pr < gn * olen; pr += blockDim.x) {
        const int g = pr / olen, oo = pr - g * olen;
        const double* xg = Xs + g * blk;
        double s = 0.0;
        for (int q = 0; q < len; ++q) s = fma(Us[q * olen + oo], xg[q], s);
        O[(gb + g) * ldO + oo] = s;
      }
    }
  }
  double* out = partial + (int64_t)blockIdx.x * count;
#pragma unroll
  for (int u = 0; u < kBackNY; ++u) {
    const int o = threadIdx.x + u * kBackThreads;
    if (o < count) out[o] = acc[u];
  }
}

__global__ void k_Y_reduce(const double* __restrict__ partial, int64_t nchunks, int64_t count,
                           double* __restrict__ Y, const Scalars* sc) {
  if (sc && sc->noop) return;
  int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= count) return;
  double acc = 0.0;
  for (int64_t ch = 0; ch < nchunks; ++ch) acc += partial[ch * count + o];
  Y[o] = acc;
}

}  // namespace

void tables_init() {
  cudaFuncSetAttribute(k_E_down, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(k_F_up, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(k_back_level, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
}

namespace {

int64_t y_chunks(int64_t nsum, int nk, int r1) {
  int64_t njc = (int64_t)nk * r1;
  int64_t want = (160000 + njc - 1) / njc;     // enough threads to fill 148 SMs
  int64_t byrows = (nsum + 31) / 32;           // at least 32 summands per chunk
  int64_t ch = want < byrows ? want : byrows;
  if (ch < 1) ch = 1;
  if (ch > 65535) ch = 65535;
  return ch;
}

}  // namespace

void launch_table_left(cudaStream_t s, const double* in, int ld_in, const double* core, int r0,
                       int nk, int r1, double* out, int ld_out, int64_t rows_out,
                       const double* rowscale, const Scalars* sc, int64_t* launches) {
  const int64_t nparent = rows_out / nk;
  dim3 grid(nk, blocks_for(nparent, kRowsPerBlock));
  k_table_left<<<grid, kTabThreads, 0, s>>>(in, ld_in, core, r0, nk, r1, out, ld_out, nparent,
                                             rowscale, sc);
  ++*launches;
}

void launch_table_right(cudaStream_t s, const double* in, int ld_in, const double* core, int r0,
                        int nk, int r1, double* out, int ld_out, int64_t rows_out,
                        const double* rowscale, const Scalars* sc, int64_t* launches) {
  const int64_t nparent = rows_out / nk;
  dim3 grid(nk, blocks_for(nparent, kRowsPerBlock));
  k_table_right<<<grid, kTabThreads, 0, s>>>(in, ld_in, core, r0, nk, r1, out, ld_out, nparent,
                                              rowscale, sc);
  ++*launches;
}

static int rec_jchunk(int r0, int nk, int r1) {
  int jc = (int)(kTableSmemDoubles / ((int64_t)r0 * r1));
  if (jc > nk) jc = nk;
  if (jc < 1) jc = 1;
  return jc;
}

namespace {
__global__ void k_jsplit_reduce(const double* __restrict__ part, int nsplit, int64_t n, double* __restrict__ out,
                                const Scalars* sc) {
  if (sc && sc->noop) return;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  double acc = 0.0;
  for (int y = 0; y < nsplit; ++y) acc += part[(int64_t)y * n + e];
  out[e] = acc;
}

// slice splits for levels with few output rows (enough CTAs for the GPU), bounded by scratch
int rec_jsplit(int64_t rows_out, int nk, int jc, int ld_out, int64_t scratch_cap) {
  const int64_t rb = (rows_out + kRecRows - 1) / kRecRows;
  int64_t js = rb >= 148 ? 1 : (296 + rb - 1) / rb;
  js = std::min<int64_t>(js, nk);   // a CTA may cover fewer slices than one staged chunk jc
  (void)jc;
  if (scratch_cap > 0) js = std::min<int64_t>(js, scratch_cap / std::max<int64_t>(1, rows_out * ld_out));
  else js = 1;
  return (int)std::max<int64_t>(1, js);
}
}  // namespace

void launch_E_down(cudaStream_t s, const double* Ein, int ld_in, const double* core, int r0,
                   int nk, int r1, double* Eout, int ld_out, int64_t rows_out, double* scratch,
                   int64_t scratch_cap, const Scalars* sc, int64_t* launches) {
  const int jc = rec_jchunk(r0, nk, r1);
  const size_t smem = (size_t)jc * r0 * r1 * sizeof(double);
  const int js = rec_jsplit(rows_out, nk, jc, ld_out, scratch_cap);
  dim3 grid(blocks_for(rows_out, kRecRows), js);
  k_E_down<<<grid, kTabThreads, smem, s>>>(Ein, ld_in, core, r0, nk, r1, Eout, ld_out, rows_out, jc, scratch, sc);
  ++*launches;
  if (js > 1) {
    k_jsplit_reduce<<<blocks_for(rows_out * ld_out, 256), 256, 0, s>>>(scratch, js, rows_out * ld_out, Eout, sc);
    ++*launches;
  }
}

void launch_F_up(cudaStream_t s, const double* Fin, int ld_in, const double* core, int r0, int nk,
                 int r1, double* Fout, int ld_out, int64_t rows_out, double* scratch,
                 int64_t scratch_cap, const Scalars* sc, int64_t* launches) {
  const int jc = rec_jchunk(r0, nk, r1);
  const size_t smem = (size_t)jc * r0 * r1 * sizeof(double);
  const int js = rec_jsplit(rows_out, nk, jc, ld_out, scratch_cap);
  dim3 grid(blocks_for(rows_out, kRecRows), js);
  k_F_up<<<grid, kTabThreads, smem, s>>>(Fin, ld_in, core, r0, nk, r1, Fout, ld_out, rows_out, jc, scratch, sc);
  ++*launches;
  if (js > 1) {
    k_jsplit_reduce<<<blocks_for(rows_out * ld_out, 256), 256, 0, s>>>(scratch, js, rows_out * ld_out, Fout, sc);
    ++*launches;
  }
}

int64_t Y_partial_need(int64_t nsum, int r0, int nk, int r1) {
  return y_chunks(nsum, nk, r1) * (int64_t)r0 * nk * r1;
}

void launch_Y(cudaStream_t s, bool left, const double* A, int ldA, const double* E, int ldE,
              int64_t nsum, int r0, int nk, int r1, double* Y, double* partial,
              int64_t partial_cap, const Scalars* sc, int64_t* launches) {
  int64_t nch = y_chunks(nsum, nk, r1);
  int64_t count = (int64_t)r0 * nk * r1;
  if (nch * count > partial_cap) nch = partial_cap / count;
  if (nch < 1) nch = 1;
  int64_t chunk = (nsum + nch - 1) / nch;
  nch = (nsum + chunk - 1) / chunk;
  dim3 grid(blocks_for((int64_t)nk * r1, kYThreads), (unsigned)nch);
  k_Y_partial<<<grid, kYThreads, 0, s>>>(left ? 1 : 0, A, ldA, E, ldE, nsum, chunk, r0, nk, r1,
                                         partial, sc);
  k_Y_reduce<<<blocks_for(count, 256), 256, 0, s>>>(partial, nch, count, Y, sc);
  *launches += 2;
}

bool back_fused_ok(int r0, int nk, int r1) {
  return (int64_t)r0 * nk * r1 <= (int64_t)kBackNY * kBackThreads;
}

int64_t back_partial_need(int64_t ngroups, int r0, int nk, int r1) {
  const int64_t count = (int64_t)r0 * nk * r1;
  int64_t nb = (ngroups + 15) / 16;
  if (nb > 296) nb = 296;
  if (nb < 1) nb = 1;
  return nb * count;
}

void launch_back_level(cudaStream_t s, bool left, const double* X, int ldX, const double* V,
                       int ldV, const double* core, int r0, int nk, int r1, double* O, int ldO,
                       int64_t ngroups, double* Y, double* partial, int64_t partial_cap,
                       const Scalars* sc, int64_t* launches) {
  const int w = left ? r1 : r0;
  const int blk = nk * w;
  int G = (int)(8192 / blk);
  if (G > 16) G = 16;
  if (G < 1) G = 1;
  const int64_t count = (int64_t)r0 * nk * r1;
  int64_t nb = (ngroups + G - 1) / G;
  if (nb > 296) nb = 296;
  if (nb * count > partial_cap) nb = partial_cap / count;
  if (nb < 1) nb = 1;
  int64_t chunk = (ngroups + nb - 1) / nb;
  chunk = ((chunk + G - 1) / G) * G;
  nb = (ngroups + chunk - 1) / chunk;
  const size_t smem = ((size_t)count + (size_t)G * blk + (size_t)G * kMaxRank) * sizeof(double);
  k_back_level<<<(unsigned)nb, kBackThreads, smem, s>>>(left ? 1 : 0, X, ldX, V, ldV, core, r0, nk,
                                                       r1, O, ldO, ngroups, chunk, G, partial, sc);
  k_Y_reduce<<<blocks_for(count, 256), 256, 0, s>>>(partial, nb, count, Y, sc);
  *launches += 2;
}

}  // namespace prgd
