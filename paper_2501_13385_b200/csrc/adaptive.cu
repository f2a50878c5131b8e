// adaptive.cu — the adaptive (steepest) step of PRGD / RGD (eq. `PRGD
// stepsize`; RGD's form PAPER.md:150-152):
//   alpha_l = step_size * ||D||_W^2 / ||P_Omega D||_F^2,   D = P~_T W^{-1} G = sum_k dA_k.
// Numerator: sum_k ||[U_1..Ahat_k..U_d]||_F^2 (k_project, proj_mode 1).  Denominator: D at
// every observed index through the prefix / suffix split,
//   D(x_s) = psi(x_s) ( LD(P) . RU(S) + LU(P) . RD(S) ),
// with LU / RU the U tables of pass B and LD / RD the tables of the chains that carry exactly
// one Ahat core:  LD_{k+1} = [LD_k | LU_k] . [U_k ; Ahat_k],  RD_k = [U_k | Ahat_k] . [RD_{k+1} ; RU_{k+1}]
// (block-triangular TT of the tangent vector), built as ordinary table levels
// over a concatenated input and a stacked core (this file), evaluated by k_seg in DPASS mode.
#include "prgd_internal.cuh"

namespace prgd {
namespace {

constexpr int kT = 256;
constexpr int kVsumBlocks = 256;

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + kT - 1) / kT); }

struct StackArgs {
  int d;
  int r[kMaxD + 1];
  int n[kMaxD];
  int64_t core_off[kMaxD + 1];
  int64_t st_off[kMaxD + 1];   // offsets of the stacked cores (2 x core size each)
  int left[kMaxD];             // 1: [U_k ; Ahat_k] along mode 1, 0: [U_k | Ahat_k] along mode 3
};

// one CTA per core k
__global__ void k_stack_cores(const double* __restrict__ U, const double* __restrict__ Ah, StackArgs sa,
                              double* __restrict__ st, const Scalars* sc) {
  if (sc && sc->noop) return;
  const int k = blockIdx.x;
  const int r0 = sa.r[k], nk = sa.n[k], r1 = sa.r[k + 1];
  const double* u = U + sa.core_off[k];
  const double* a = Ah + sa.core_off[k];
  double* o = st + sa.st_off[k];
  const int64_t sz = (int64_t)r0 * nk * r1;
  if (sa.left[k]) {            // (2 r0) x nk x r1: rows < r0 from U, rows >= r0 from Ahat
    for (int64_t e = threadIdx.x; e < 2 * sz; e += blockDim.x) o[e] = e < sz ? u[e] : a[e - sz];
  } else {                     // r0 x nk x (2 r1): cols < r1 from U, cols >= r1 from Ahat
    for (int64_t e = threadIdx.x; e < 2 * sz; e += blockDim.x) {
      const int64_t row = e / (2 * r1);
      const int c = (int)(e - row * 2 * r1);
      o[e] = c < r1 ? u[row * r1 + c] : a[row * r1 + (c - r1)];
    }
  }
}

struct CatJob {
  double* out;
  const double* x;   // first half  (LD_k / RD_{k+1})
  const double* y;   // second half (LU_k / RU_{k+1})
  int64_t rows;
  int ldo, ldx, ldy, w;
};

// out[p] = [x[p, 0:w] | y[p, 0:w] | 0 ...]  (up to two independent jobs, one per side)
__global__ void k_concat2(CatJob j0, CatJob j1, int64_t n0, const Scalars* sc) {
  if (sc && sc->noop) return;
  int64_t e = blockIdx.x * (int64_t)kT + threadIdx.x;
  const CatJob& j = e < n0 ? j0 : j1;
  if (e >= n0) e -= n0;
  const int64_t p = e / j.ldo;
  const int c = (int)(e - p * j.ldo);
  if (p >= j.rows) return;
  double v = 0.0;
  if (c < j.w) v = j.x[p * j.ldx + c];
  else if (c < 2 * j.w) v = j.y[p * j.ldy + (c - j.w)];
  j.out[e] = v;
}

// den partials: block b sums its contiguous chunk of x in a fixed order
__global__ void k_vsum_partial(const double* __restrict__ x, int64_t n, double* __restrict__ part,
                               const Scalars* sc) {
  __shared__ double red[kT];
  if (sc && sc->noop) return;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * chunk, b1 = b0 + chunk < n ? b0 + chunk : n;
  double s = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += kT) s += x[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_vsum_final(const double* __restrict__ part, int nparts, Scalars* sc) {
  if (sc->noop) return;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nparts; ++i) s += part[i];
    sc->adapt_den = s;
  }
}

// alpha = step_size * sum_k num_k / den (den = 0: no move, reading R20)
__global__ void k_adapt_alpha(int d, Scalars* sc) {
  if (sc->noop) return;
  if (threadIdx.x == 0) {
    double num = 0.0;
    for (int k = 0; k < d; ++k) num += sc->adapt_num[k];
    const double den = sc->adapt_den;
    const double alpha = den > 0.0 ? sc->step_size * num / den : 0.0;
    if (!isfinite(alpha)) atomicOr(&sc->err, (int)kErrNaN);
    sc->alpha = isfinite(alpha) ? alpha : 0.0;
  }
}

}  // namespace

int64_t stacked_cores_len(int d, const int64_t* core_off) { return 2 * core_off[d]; }

void launch_stack_cores(cudaStream_t s, int d, const int* n, const int* r, const int64_t* core_off,
                        int KL, const double* U, const double* Ahat, double* st, const Scalars* sc,
                        int64_t* launches) {
  StackArgs sa{};
  sa.d = d;
  for (int k = 0; k <= d; ++k) {
    sa.r[k] = r[k];
    sa.core_off[k] = core_off[k];
    sa.st_off[k] = 2 * core_off[k];
  }
  for (int k = 0; k < d; ++k) {
    sa.n[k] = n[k];
    sa.left[k] = k < KL ? 1 : 0;
  }
  k_stack_cores<<<d, kT, 0, s>>>(U, Ahat, sa, st, sc);
  ++*launches;
}

void launch_concat2(cudaStream_t s, double* o0, int ldo0, const double* x0, int ldx0, const double* y0,
                    int ldy0, int64_t rows0, int w0, double* o1, int ldo1, const double* x1, int ldx1,
                    const double* y1, int ldy1, int64_t rows1, int w1, const Scalars* sc,
                    int64_t* launches) {
  CatJob j0{o0, x0, y0, o0 ? rows0 : 0, ldo0, ldx0, ldy0, w0};
  CatJob j1{o1, x1, y1, o1 ? rows1 : 0, ldo1, ldx1, ldy1, w1};
  const int64_t n0 = j0.rows * (int64_t)ldo0, n1 = j1.rows * (int64_t)ldo1;
  if (n0 + n1 == 0) return;
  if (n0 == 0) {
    k_concat2<<<blocks_for(n1), kT, 0, s>>>(j1, j1, n1, sc);
  } else {
    k_concat2<<<blocks_for(n0 + n1), kT, 0, s>>>(j0, j1, n0, sc);
  }
  ++*launches;
}

int adapt_vsum_parts() { return kVsumBlocks; }

void launch_adapt_den(cudaStream_t s, const double* x, int64_t n, double* part, Scalars* sc,
                      int64_t* launches) {
  k_vsum_partial<<<kVsumBlocks, kT, 0, s>>>(x, n, part, sc);
  k_vsum_final<<<1, 32, 0, s>>>(part, kVsumBlocks, sc);
  *launches += 2;
}

void launch_adapt_alpha(cudaStream_t s, int d, Scalars* sc, int64_t* launches) {
  k_adapt_alpha<<<1, 32, 0, s>>>(d, sc);
  ++*launches;
}

}  // namespace prgd
