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
#include "prgd_internal.cuh"

namespace prgd {
namespace {

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__global__ void k_table_left(const double* __restrict__ in, int ld_in,
                             const double* __restrict__ core, int r0, int nk, int r1,
                             double* __restrict__ out, int ld_out, int64_t rows,
                             const double* __restrict__ rowscale, const Scalars* sc) {
  if (sc && sc->noop) return;
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t row = e / ld_out;
  int c = (int)(e - row * ld_out);
  if (row >= rows) return;
  double acc = 0.0;
  if (c < r1) {
    int64_t p = row / nk;
    int j = (int)(row - p * nk);
    const double* cp = core + (int64_t)j * r1 + c;
    if (in == nullptr) {
      acc = cp[0];
    } else {
      const double* a = in + p * ld_in;
      const int64_t cs = (int64_t)nk * r1;
      for (int i = 0; i < r0; ++i) acc = fma(a[i], cp[i * cs], acc);
    }
    if (rowscale) acc *= rowscale[row];
  }
  out[row * ld_out + c] = acc;
}

// Right table level: block = R rows x ld_out lanes; the R core slices C_k(:, j, :) the
// block needs are staged transposed ([c][i], i fastest) so lanes i read consecutive
// shared-memory words; the R input rows B_{k+1}[q, :] are staged too.
__global__ void k_table_right(const double* __restrict__ in, int ld_in,
                              const double* __restrict__ core, int r0, int nk, int r1,
                              double* __restrict__ out, int ld_out, int64_t rows,
                              const double* __restrict__ rowscale, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ double sm[];
  const int R = blockDim.x / ld_out;
  const int64_t row0 = (int64_t)blockIdx.x * R;
  double* slices = sm;                       // [R][r1][r0]
  double* vin = sm + (int64_t)R * r1 * r0;   // [R][r1]
  const int per = r1 * r0;
  for (int t = threadIdx.x; t < R * per; t += blockDim.x) {
    const int lr = t / per, rem = t - lr * per;
    const int i = rem / r1, c = rem - i * r1;  // c fastest: coalesced global reads
    const int64_t row = row0 + lr;
    double v = 0.0;
    if (row < rows) {
      const int j = (int)(row % nk);
      v = core[((int64_t)i * nk + j) * r1 + c];
    }
    slices[(lr * r1 + c) * r0 + i] = v;
  }
  for (int t = threadIdx.x; t < R * r1; t += blockDim.x) {
    const int lr = t / r1, c = t - lr * r1;
    const int64_t row = row0 + lr;
    double v = 0.0;
    if (row < rows) v = in == nullptr ? 1.0 : in[(row / nk) * ld_in + c];
    vin[t] = v;
  }
  __syncthreads();
  const int lr = threadIdx.x / ld_out, i = threadIdx.x - lr * ld_out;
  const int64_t row = row0 + lr;
  if (lr >= R || row >= rows) return;
  double acc = 0.0;
  if (i < r0) {
    const double* sl = slices + (int64_t)lr * r1 * r0 + i;
    const double* vv = vin + lr * r1;
    for (int c = 0; c < r1; ++c) acc = fma(sl[c * r0], vv[c], acc);
    if (rowscale) acc *= rowscale[row];
  }
  out[row * ld_out + i] = acc;
}

// E_k[p, i] = sum_{j,c} U_k[i, j, c] E_{k+1}[p n_k + j, c]: block = R rows p x ld_out
// lanes i; the core is staged transposed ([j][c][i]) in chunks of slices.
__global__ void k_E_down(const double* __restrict__ Ein, int ld_in, const double* __restrict__ core,
                         int r0, int nk, int r1, double* __restrict__ Eout, int ld_out,
                         int64_t rows, int jchunk, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ double sm[];
  const int R = blockDim.x / ld_out;
  const int lr = threadIdx.x / ld_out, i = threadIdx.x - lr * ld_out;
  const int64_t p = (int64_t)blockIdx.x * R + lr;
  const bool active = lr < R && p < rows && i < r0;
  double acc = 0.0;
  const int per = r1 * r0;
  for (int j0 = 0; j0 < nk; j0 += jchunk) {
    const int jn = nk - j0 < jchunk ? nk - j0 : jchunk;
    __syncthreads();
    for (int t = threadIdx.x; t < jn * per; t += blockDim.x) {
      const int jj = t / per, rem = t - jj * per;
      const int ii = rem / r1, c = rem - ii * r1;
      sm[(jj * r1 + c) * r0 + ii] = core[((int64_t)ii * nk + j0 + jj) * r1 + c];
    }
    __syncthreads();
    if (active) {
      for (int jj = 0; jj < jn; ++jj) {
        const double* ein = Ein + (p * nk + j0 + jj) * ld_in;
        const double* sl = sm + jj * per + i;
        for (int c = 0; c < r1; ++c) acc = fma(sl[c * r0], ein[c], acc);
      }
    }
  }
  if (lr < R && p < rows) Eout[p * ld_out + i] = acc;
}

__global__ void k_F_up(const double* __restrict__ Fin, int ld_in, const double* __restrict__ core,
                       int r0, int nk, int r1, double* __restrict__ Fout, int ld_out, int64_t rows,
                       const Scalars* sc) {
  if (sc && sc->noop) return;
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t q = e / ld_out;
  int c = (int)(e - q * ld_out);
  if (q >= rows) return;
  double acc = 0.0;
  if (c < r1) {
    const int64_t cs = (int64_t)nk * r1;
    for (int j = 0; j < nk; ++j) {
      const double* f = Fin + ((int64_t)j + (int64_t)nk * q) * ld_in;
      const double* cp = core + (int64_t)j * r1 + c;
      for (int i = 0; i < r0; ++i) acc = fma(f[i], cp[i * cs], acc);
    }
  }
  Fout[q * ld_out + c] = acc;
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
  cudaFuncSetAttribute(k_table_right, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(k_E_down, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
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
  int64_t n = rows_out * ld_out;
  k_table_left<<<blocks_for(n, 256), 256, 0, s>>>(in, ld_in, core, r0, nk, r1, out, ld_out,
                                                  rows_out, rowscale, sc);
  ++*launches;
}

void launch_table_right(cudaStream_t s, const double* in, int ld_in, const double* core, int r0,
                        int nk, int r1, double* out, int ld_out, int64_t rows_out,
                        const double* rowscale, const Scalars* sc, int64_t* launches) {
  const int threads = 256;
  const int R = threads / ld_out;
  const size_t smem = ((size_t)R * r1 * r0 + (size_t)R * r1) * sizeof(double);
  k_table_right<<<blocks_for(rows_out, R), threads, smem, s>>>(in, ld_in, core, r0, nk, r1, out,
                                                              ld_out, rows_out, rowscale, sc);
  ++*launches;
}

void launch_E_down(cudaStream_t s, const double* Ein, int ld_in, const double* core, int r0,
                   int nk, int r1, double* Eout, int ld_out, int64_t rows_out,
                   const Scalars* sc, int64_t* launches) {
  const int threads = 256;
  const int R = threads / ld_out;
  const int per = r0 * r1;
  int jchunk = (int)(kTableSmemDoubles / per);
  if (jchunk > nk) jchunk = nk;
  if (jchunk < 1) jchunk = 1;
  const size_t smem = (size_t)jchunk * per * sizeof(double);
  k_E_down<<<blocks_for(rows_out, R), threads, smem, s>>>(Ein, ld_in, core, r0, nk, r1, Eout,
                                                         ld_out, rows_out, jchunk, sc);
  ++*launches;
}

void launch_F_up(cudaStream_t s, const double* Fin, int ld_in, const double* core, int r0, int nk,
                 int r1, double* Fout, int ld_out, int64_t rows_out, const Scalars* sc,
                 int64_t* launches) {
  int64_t n = rows_out * ld_out;
  k_F_up<<<blocks_for(n, 256), 256, 0, s>>>(Fin, ld_in, core, r0, nk, r1, Fout, ld_out, rows_out,
                                            sc);
  ++*launches;
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

}  // namespace prgd
