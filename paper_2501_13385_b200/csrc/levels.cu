// levels.cu — the dense table levels and backward recursions as FP64 tensor-core GEMMs,
// scheduled with few launches.
//
// Every level is a skinny GEMM over the "flat" rows of a table level: for a parent row p the
// n_k child rows (ld columns each) are contiguous, i.e. one row of W = n_k ld doubles
// (PAPER.md:99-105 recursion):
//   forward   out[p, :] = in[p, 0:K] . Cst[0:K, 0:W]          (tables; K = rank <= 32)
//     left  Cst[i][(j,c)] = C[i][j][c]      right Cst[c][(j,i)] = C[i][j][c]
//   backward  O[p, 0:olen] = X[p, :] . Ust[:, 0:olen]           (next E_k / F_{k+1} level)
//             Z[v, :]     += sum_p V[p, v] X[p, :]               (Y_k)
//     left  X = E_{k+1}, V = A_k, Ust[(j,c)][i] = U[i][j][c], Y[i][j][c] = Z[i][j ld + c]
//     right X = F_k, V = B_{k+1}, Ust[(j,i)][c] = U[i][j][c], Y[i][j][c] = Z[c][j ld + i]
// FP64 tensor-core tiles (mma.sync m8n8k4 f64 = SASS DMMA; B200's FP64 peak is the same
// through DFMA and DMMA, the tiles cut the shared-memory traffic per flop).  Operand strides
// are = 4 (mod 16) doubles, so fragment loads are bank-conflict free.
//
// Scheduling: the left and right sides are independent, so each launch carries up to two
// levels.  Large levels run as a grid (CTAs split between the two levels; backward levels
// write one Z partial per CTA, reduced in fixed chunk order => deterministic); the small
// tail levels of both sides run as one "chain" launch with one CTA per side executing its
// levels back to back (a level's output is the next level's input; __syncthreads orders the
// global writes within the CTA), which removes ~70% of the launches.
#include <algorithm>
#include <vector>

#include "prgd_internal.cuh"

namespace prgd {
namespace {

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ void dmma_l(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__host__ __device__ inline int mma_ld(int w) { return ((w + 15) / 16) * 16 + 4; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

constexpr int kT = 256;          // threads per CTA
constexpr int kNW = kT / 32;
constexpr int kFwdRows = 32;     // parent rows per forward tile
constexpr int kBackRows = 32;    // parent rows per backward tile
constexpr int kMaxLv = 8;

struct TabLv {
  const double* in;        // [nparent][ld_in] or null (the one parent row [1])
  const double* core;
  double* out;             // flat rows [nparent][W]
  const double* rowscale;  // child-row scale (psi) or null
  int64_t nparent;
  int left, ld_in, r0, nk, r1, ld_out;
};

struct TabLaunch {
  TabLv lv[kMaxLv];
  int split[kMaxLv + 1];   // grid mode: CTA range of level i; chain mode: level range of CTA i
  int nlv, chain;
};

// One forward level: CTA `cta` of `ncta` walks its 32-parent tiles.  Warp w owns the column
// blocks J = w, w+8, ...; A fragments are loaded straight from global per tile, each 8x8
// output tile leaves as double2 streaming stores.
template <int KSM>
__device__ void tab_level(const TabLv L, int cta, int ncta, double* Cs) {   // by value: fields in registers
  const int K = L.in ? (L.left ? L.r0 : L.r1) : 1;
  const int KS = (K + 3) >> 2;
  const int W = L.nk * L.ld_out;
  const int ldc = mma_ld(W);
  const int lg = __ffs(L.ld_out) - 1;                 // ld_out is a power of two
  for (int t = threadIdx.x; t < 4 * KS * W; t += blockDim.x) {
    const int k = t / W, q = t - k * W;
    const int j = q >> lg, o = q & (L.ld_out - 1);
    double v = 0.0;
    if (k < K) {
      if (L.left) v = o < L.r1 ? L.core[((int64_t)k * L.nk + j) * L.r1 + o] : 0.0;
      else v = o < L.r0 ? L.core[((int64_t)o * L.nk + j) * L.r1 + k] : 0.0;
    }
    Cs[k * ldc + q] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tq = lane & 3;
  const int nJ = W >> 3;
  const int64_t ntiles = (L.nparent + kFwdRows - 1) / kFwdRows;
  double* Fs = Cs + (int64_t)4 * KS * ldc;            // child-row scales of the tile
  for (int64_t tile = cta; tile < ntiles; tile += ncta) {
    const int64_t p0 = tile * kFwdRows;
    if (L.rowscale) {                                   // stage the tile's psi once (coalesced)
      __syncthreads();
      for (int t = threadIdx.x; t < kFwdRows * L.nk; t += blockDim.x) {
        const int64_t e = p0 * L.nk + t;
        Fs[t] = e < L.nparent * L.nk ? __ldg(L.rowscale + e) : 0.0;
      }
      __syncthreads();
    }
    // fragments beyond K are zero (the staged Cs rows k >= K are zero too), so the DMMA loop
    // runs unpredicated over KSM k-steps
    double af[4][KSM];
#pragma unroll
    for (int I = 0; I < 4; ++I) {
      const int64_t p = p0 + I * 8 + gid;
#pragma unroll
      for (int ks = 0; ks < KSM; ++ks) {
        const int k = 4 * ks + tq;
        double v = 0.0;
        if (k < K && p < L.nparent) v = L.in ? __ldg(L.in + p * L.ld_in + k) : 1.0;
        af[I][ks] = v;
      }
    }
    for (int J = warp; J < nJ; J += kNW) {
      const int q = J * 8 + 2 * tq;
      const int j = q >> lg;
      double bf[KSM];
#pragma unroll
      for (int ks = 0; ks < KSM; ++ks) bf[ks] = ks < KS ? Cs[(4 * ks + tq) * ldc + J * 8 + gid] : 0.0;
#pragma unroll
      for (int I = 0; I < 4; ++I) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KSM; ++ks) dmma_l(d0, d1, af[I][ks], bf[ks]);
        const int64_t p = p0 + I * 8 + gid;
        if (p < L.nparent) {
          const double f = L.rowscale ? Fs[(I * 8 + gid) * L.nk + j] : 1.0;
          __stcs(reinterpret_cast<double2*>(L.out + p * W + q), make_double2(d0 * f, d1 * f));
        }
      }
    }
  }
  __syncthreads();
}

template <int KSM>
__global__ void __launch_bounds__(kT, KSM <= 4 ? 3 : 2) k_tab_levels(TabLaunch La, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ double sm[];
  const int b = blockIdx.x;
  if (La.chain) {
    for (int i = La.split[b]; i < La.split[b + 1]; ++i) tab_level<KSM>(La.lv[i], 0, 1, sm);
  } else {
    int i = 0;
    while (i + 1 < La.nlv && b >= La.split[i + 1]) ++i;
    tab_level<KSM>(La.lv[i], b - La.split[i], La.split[i + 1] - La.split[i], sm);
  }
}

struct BackLv {
  const double* X;     // flat rows [ngroups][W]
  const double* V;     // [ngroups][ldV] or null (ones)
  const double* core;  // U_k
  double* O;           // [ngroups][ldO] or null
  double* part;        // grid mode: Z partials [ncta][vlen][W]
  double* Y;           // chain mode: Y_k written directly
  int64_t ngroups;
  int left, wrow, ldV, vlen, r0, nk, r1, ldO, olen;
};

struct BackLaunch {
  BackLv lv[kMaxLv];
  int split[kMaxLv + 1];
  int nlv, chain;
};

// One backward level, CTA `cta` of `ncta`.  Warp w owns the Z tiles (vb, qb = w + 8m); per
// 4-row k-step it loads NVB A- and <= 8 B-fragments and issues NVB x 8 independent DMMAs.
// The next tile's X / V rows land by cp.async while the current tile computes.
template <int NVB>
__device__ void back_level(const BackLv L, int cta, int ncta, double* sm, bool direct) {   // by value: fields in registers
  const int W = L.nk * L.wrow;
  const int ldx = mma_ld(W);
  const int olen8 = L.O ? max((L.olen + 7) & ~7, (L.ldO + 7) & ~7) : 0;
  const int vlen8 = (L.vlen + 7) & ~7;
  const int ldv = mma_ld(vlen8);
  const int ldu = mma_ld(olen8);
  double* Us = sm;                                     // W x ldu
  double* Xs0 = Us + (int64_t)W * ldu;                 // 2 x (kBackRows x ldx)
  double* Vs0 = Xs0 + 2 * (int64_t)kBackRows * ldx;    // 2 x (kBackRows x ldv)
  if (L.O) {
    for (int t = threadIdx.x; t < W * olen8; t += blockDim.x) {
      const int q = t / olen8, o = t - q * olen8;
      const int j = q / L.wrow, x = q - j * L.wrow;
      double v = 0.0;
      if (o < L.olen) {
        if (L.left) v = x < L.r1 ? L.core[((int64_t)o * L.nk + j) * L.r1 + x] : 0.0;
        else v = x < L.r0 ? L.core[((int64_t)x * L.nk + j) * L.r1 + o] : 0.0;
      }
      Us[q * ldu + o] = v;
    }
  }
  if (!L.V)
    for (int t = threadIdx.x; t < 2 * kBackRows * ldv; t += blockDim.x)
      Vs0[t] = (t % ldv) < L.vlen ? 1.0 : 0.0;
  const int w2 = W >> 1;
  const int64_t ngroups = L.ngroups;
  auto prefetch = [&](int64_t tile, int buf) {
    const int64_t p0 = tile * kBackRows;
    double* Xs = Xs0 + (int64_t)buf * kBackRows * ldx;
    for (int t = threadIdx.x; t < kBackRows * w2; t += blockDim.x) {
      const int r = t / w2, q2 = t - r * w2;
      const int64_t p = p0 + r;
      const bool ok = p < ngroups;
      cp_async16(Xs + r * ldx + 2 * q2, L.X + (ok ? p * W + 2 * q2 : 0), ok);
    }
    if (L.V) {
      double* Vs = Vs0 + (int64_t)buf * kBackRows * ldv;
      for (int t = threadIdx.x; t < kBackRows * vlen8; t += blockDim.x) {
        const int r = t / vlen8, v = t - r * vlen8;
        const int64_t p = p0 + r;
        const bool ok = p < ngroups && v < L.vlen;
        cp_async8(Vs + r * ldv + v, L.V + (ok ? p * L.ldV + v : 0), ok);
      }
    }
  };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tq = lane & 3;
  const int nqb = W >> 3;                              // column blocks of Z
  double z0[NVB][8], z1[NVB][8];
#pragma unroll
  for (int a = 0; a < NVB; ++a)
#pragma unroll
    for (int m = 0; m < 8; ++m) z0[a][m] = z1[a][m] = 0.0;
  const int64_t ntiles = (ngroups + kBackRows - 1) / kBackRows;
  int buf = 0;
  __syncthreads();
  if (cta < ntiles) prefetch(cta, 0);
  cp_commit();
  for (int64_t tile = cta; tile < ntiles; tile += ncta) {
    const int64_t p0 = tile * kBackRows;
    if (tile + ncta < ntiles) prefetch(tile + ncta, buf ^ 1);
    cp_commit();
    cp_wait1();
    __syncthreads();
    const double* Xs = Xs0 + (int64_t)buf * kBackRows * ldx;
    const double* Vs = Vs0 + (int64_t)buf * kBackRows * ldv;
    // Z[v][q] += sum_r Vs[r][v] Xs[r][q]
#pragma unroll
    for (int k = 0; k < kBackRows; k += 4) {
      double af[NVB];
#pragma unroll
      for (int a = 0; a < NVB; ++a) af[a] = Vs[(k + tq) * ldv + a * 8 + gid];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int qb = warp + kNW * m;
        if (qb < nqb) {
          const double bfr = Xs[(k + tq) * ldx + qb * 8 + gid];
#pragma unroll
          for (int a = 0; a < NVB; ++a) dmma_l(z0[a][m], z1[a][m], af[a], bfr);
        }
      }
    }
    // O[p][o] = sum_q Xs[r][q] Us[q][o]
    if (L.O) {
      const int ot_n = olen8 >> 3, ot = (kBackRows / 8) * ot_n;
      for (int t = warp; t < ot; t += kNW) {
        const int rb = t / ot_n, ob = t - rb * ot_n;
        const double* xr = Xs + (rb * 8 + gid) * ldx + tq;
        const double* ur = Us + tq * ldu + ob * 8 + gid;
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0, g0 = 0.0, g1 = 0.0;
        int q = 0;
        for (; q + 16 <= W; q += 16) {
          dmma_l(d0, d1, xr[q], ur[q * ldu]);
          dmma_l(e0, e1, xr[q + 4], ur[(q + 4) * ldu]);
          dmma_l(f0, f1, xr[q + 8], ur[(q + 8) * ldu]);
          dmma_l(g0, g1, xr[q + 12], ur[(q + 12) * ldu]);
        }
        for (; q < W; q += 4) dmma_l(d0, d1, xr[q], ur[q * ldu]);
        const int64_t p = p0 + rb * 8 + gid;
        const int o = ob * 8 + 2 * tq;
        if (p < ngroups) {
          if (o < L.ldO) L.O[p * L.ldO + o] = (o < L.olen) ? (d0 + e0) + (f0 + g0) : 0.0;
          if (o + 1 < L.ldO) L.O[p * L.ldO + o + 1] = (o + 1 < L.olen) ? (d1 + e1) + (f1 + g1) : 0.0;
        }
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  cp_wait0();
  // Z out: partial slice of this CTA, or Y directly (single CTA)
#pragma unroll
  for (int a = 0; a < NVB; ++a)
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int qb = warp + kNW * m;
      const int v = a * 8 + gid, q = qb * 8 + 2 * tq;
      if (qb < nqb && v < L.vlen) {
        if (!direct) {
          double* out = L.part + (int64_t)cta * L.vlen * W;
          out[(int64_t)v * W + q] = z0[a][m];
          out[(int64_t)v * W + q + 1] = z1[a][m];
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int qq = q + h, j = qq / L.wrow, x = qq - j * L.wrow;
            const double val = h ? z1[a][m] : z0[a][m];
            if (L.left) {
              if (x < L.r1) L.Y[((int64_t)v * L.nk + j) * L.r1 + x] = val;   // Y[i=v][j][c=x]
            } else {
              if (x < L.r0) L.Y[((int64_t)x * L.nk + j) * L.r1 + v] = val;   // Y[i=x][j][c=v]
            }
          }
        }
      }
    }
  __syncthreads();
}

template <int NVB>
__global__ void __launch_bounds__(kT) k_back_levels(BackLaunch La, const Scalars* sc) {
  if (sc && sc->noop) return;
  extern __shared__ double sm[];
  const int b = blockIdx.x;
  if (La.chain) {
    for (int i = La.split[b]; i < La.split[b + 1]; ++i) back_level<NVB>(La.lv[i], 0, 1, sm, true);
  } else {
    int i = 0;
    while (i + 1 < La.nlv && b >= La.split[i + 1]) ++i;
    back_level<NVB>(La.lv[i], b - La.split[i], La.split[i + 1] - La.split[i], sm, false);
  }
}

// Y of up to two grid-mode levels from their Z partials: one warp per output, lane l sums
// chunks l, l+32, ... then a fixed shuffle tree (deterministic).
struct ZRed {
  const double* part[2];
  double* Y[2];
  int64_t nchunks[2], count[2];
  int left[2], vlen[2], W[2], wrow[2], r0[2], nk[2], r1[2];
  int n;
};

__global__ void k_zreduce(ZRed R, const Scalars* sc) {
  if (sc && sc->noop) return;
  int64_t o = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int s = 0;
  if (o >= R.count[0]) {
    o -= R.count[0];
    s = 1;
    if (R.n < 2 || o >= R.count[1]) return;
  }
  const int nk = R.nk[s], r1 = R.r1[s], W = R.W[s], wrow = R.wrow[s];
  const int i = (int)(o / ((int64_t)nk * r1));
  const int rem = (int)(o - (int64_t)i * nk * r1);
  const int j = rem / r1, c = rem - j * r1;
  const int64_t zi = R.left[s] ? (int64_t)i * W + j * wrow + c : (int64_t)c * W + j * wrow + i;
  double acc = 0.0;
  const int64_t stride = (int64_t)R.vlen[s] * W;
  for (int64_t ch = lane; ch < R.nchunks[s]; ch += 32) acc += R.part[s][ch * stride + zi];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) R.Y[s][o] = acc;
}

int g_sms = 0;
int sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

constexpr int64_t kSmallOut = 1 << 13;   // doubles of output below which a level is "small"
constexpr int kMaxBackCtas = 160;

size_t tab_smem(const TabLv& L) {
  const int K = L.in ? (L.left ? L.r0 : L.r1) : 1;
  return ((size_t)(4 * ((K + 3) >> 2)) * mma_ld(L.nk * L.ld_out) + (L.rowscale ? kFwdRows * L.nk : 0)) *
         sizeof(double);
}

size_t back_smem(const BackLv& L) {
  const int W = L.nk * L.wrow;
  const int olen8 = L.O ? std::max((L.olen + 7) & ~7, (L.ldO + 7) & ~7) : 0;
  return ((size_t)W * mma_ld(olen8) + 2 * (size_t)kBackRows * mma_ld(W) +
          2 * (size_t)kBackRows * mma_ld((L.vlen + 7) & ~7)) * sizeof(double);
}

void launch_tab(cudaStream_t s, TabLaunch& La, int grid, size_t smem, int kmax, const Scalars* sc,
                int64_t* lc) {
  if (kmax <= 16) k_tab_levels<4><<<grid, kT, smem, s>>>(La, sc);
  else k_tab_levels<8><<<grid, kT, smem, s>>>(La, sc);
  ++*lc;
}

void launch_back(cudaStream_t s, BackLaunch& La, int grid, size_t smem, int vmax, const Scalars* sc,
                 int64_t* lc) {
  if (vmax <= 8) k_back_levels<1><<<grid, kT, smem, s>>>(La, sc);
  else if (vmax <= 16) k_back_levels<2><<<grid, kT, smem, s>>>(La, sc);
  else k_back_levels<4><<<grid, kT, smem, s>>>(La, sc);
  ++*lc;
}

}  // namespace

bool level_tab_ok(int r0, int nk, int r1, int ld_out) {
  const int W = nk * ld_out;
  return W <= 1024 && W % 8 == 0 && r0 <= kMaxRank && r1 <= kMaxRank;
}

bool level_back_ok(int r0, int nk, int r1, int wrow) {
  const int W = nk * wrow;
  if (W > 512 || W % 8 != 0 || W / 8 > 8 * kNW || r0 > kMaxRank || r1 > kMaxRank) return false;
  BackLv L{};
  L.nk = nk;
  L.wrow = wrow;
  L.vlen = std::max(r0, r1);
  L.olen = std::max(r0, r1);
  L.ldO = pad_rank(L.olen);
  L.O = reinterpret_cast<double*>(8);
  return back_smem(L) <= 200 * 1024;
}

int64_t level_back_partial_need(int64_t ngroups, int r0, int nk, int r1, int wrow) {
  return (int64_t)kMaxBackCtas * std::max(r0, r1) * nk * wrow;
}

// Forward table levels of both sides.  Each list is in dependency order (small first).
void launch_table_levels(cudaStream_t s, const std::vector<TableLevel>& left,
                         const std::vector<TableLevel>& right, const Scalars* sc, int64_t* lc) {
  auto mk = [](const TableLevel& t) {
    TabLv L{};
    L.in = t.in;
    L.core = t.core;
    L.out = t.out;
    L.rowscale = t.rowscale;
    L.nparent = t.rows_out / t.nk;
    L.left = t.left ? 1 : 0;
    L.ld_in = t.ld_in;
    L.r0 = t.r0;
    L.nk = t.nk;
    L.r1 = t.r1;
    L.ld_out = t.ld_out;
    return L;
  };
  const std::vector<TableLevel>* side[2] = {&left, &right};
  size_t nsmall[2] = {0, 0};
  for (int sd = 0; sd < 2; ++sd)
    while (nsmall[sd] < side[sd]->size() &&
           (*side[sd])[nsmall[sd]].rows_out * (*side[sd])[nsmall[sd]].ld_out <= kSmallOut &&
           nsmall[sd] < (size_t)kMaxLv / 2)
      ++nsmall[sd];
  // chain launch of the small prefixes (one CTA per side)
  if (nsmall[0] + nsmall[1] > 0) {
    TabLaunch La{};
    La.chain = 1;
    int n = 0, g = 0;
    size_t smem = 0;
    int kmax = 1;
    La.split[0] = 0;
    for (int sd = 0; sd < 2; ++sd) {
      if (!nsmall[sd]) continue;
      for (size_t i = 0; i < nsmall[sd]; ++i) {
        La.lv[n] = mk((*side[sd])[i]);
        smem = std::max(smem, tab_smem(La.lv[n]));
        kmax = std::max(kmax, std::max(La.lv[n].r0, La.lv[n].r1));
        ++n;
      }
      La.split[++g] = n;
    }
    La.nlv = n;
    launch_tab(s, La, g, smem, kmax, sc, lc);
  }
  // the large levels, left i-th with right i-th
  const size_t nb = std::max(left.size() - nsmall[0], right.size() - nsmall[1]);
  for (size_t i = 0; i < nb; ++i) {
    TabLaunch La{};
    La.chain = 0;
    int n = 0;
    size_t smem = 0;
    int kmax = 1;
    int64_t tiles[2] = {0, 0};
    for (int sd = 0; sd < 2; ++sd) {
      const size_t idx = nsmall[sd] + i;
      if (idx >= side[sd]->size()) continue;
      La.lv[n] = mk((*side[sd])[idx]);
      smem = std::max(smem, tab_smem(La.lv[n]));
      kmax = std::max(kmax, std::max(La.lv[n].r0, La.lv[n].r1));
      tiles[n] = (La.lv[n].nparent + kFwdRows - 1) / kFwdRows;
      ++n;
    }
    La.nlv = n;
    const int64_t tot = tiles[0] + tiles[1];
    const int64_t budget = (int64_t)sms() * 3;
    La.split[0] = 0;
    for (int q = 0; q < n; ++q) {
      int64_t c = tot <= budget ? tiles[q] : std::max<int64_t>(1, budget * tiles[q] / tot);
      La.split[q + 1] = La.split[q] + (int)c;
    }
    launch_tab(s, La, La.split[n], smem, kmax, sc, lc);
  }
}

// Backward levels of both sides.  Each list is in dependency order (large first).
void launch_backward_levels(cudaStream_t s, const std::vector<BackwardLevel>& left,
                            const std::vector<BackwardLevel>& right, double* part, int64_t part_cap,
                            const Scalars* sc, int64_t* lc) {
  auto mk = [](const BackwardLevel& t) {
    BackLv L{};
    L.X = t.X;
    L.V = t.V;
    L.core = t.core;
    L.O = t.O;
    L.Y = t.Y;
    L.ngroups = t.ngroups;
    L.left = t.left ? 1 : 0;
    L.wrow = t.wrow;
    L.ldV = t.ldV;
    L.r0 = t.r0;
    L.nk = t.nk;
    L.r1 = t.r1;
    L.vlen = t.left ? t.r0 : t.r1;
    L.olen = t.left ? t.r0 : t.r1;
    L.ldO = t.ldO;
    return L;
  };
  const std::vector<BackwardLevel>* side[2] = {&left, &right};
  size_t nbig[2];
  for (int sd = 0; sd < 2; ++sd) {
    size_t nb = side[sd]->size();
    size_t ns = 0;
    while (ns < nb && ns < (size_t)kMaxLv / 2) {
      const BackwardLevel& t = (*side[sd])[nb - 1 - ns];
      if (t.ngroups * (int64_t)t.nk * t.wrow > kSmallOut) break;
      ++ns;
    }
    nbig[sd] = nb - ns;
  }
  const size_t nb = std::max(nbig[0], nbig[1]);
  for (size_t i = 0; i < nb; ++i) {
    BackLaunch La{};
    La.chain = 0;
    ZRed R{};
    int n = 0;
    size_t smem = 0;
    int vmax = 1;
    int64_t tiles[2] = {0, 0};
    for (int sd = 0; sd < 2; ++sd) {
      if (i >= nbig[sd]) continue;
      La.lv[n] = mk((*side[sd])[i]);
      smem = std::max(smem, back_smem(La.lv[n]));
      vmax = std::max(vmax, La.lv[n].vlen);
      tiles[n] = (La.lv[n].ngroups + kBackRows - 1) / kBackRows;
      ++n;
    }
    La.nlv = n;
    const int64_t tot = tiles[0] + tiles[1];
    const int64_t budget = std::min<int64_t>(sms(), kMaxBackCtas);
    La.split[0] = 0;
    double* p = part;
    for (int q = 0; q < n; ++q) {
      int64_t c = tot <= budget ? tiles[q] : std::max<int64_t>(1, budget * tiles[q] / tot);
      const int64_t per = (int64_t)La.lv[q].vlen * La.lv[q].nk * La.lv[q].wrow;
      La.split[q + 1] = La.split[q] + (int)c;
      La.lv[q].part = p;
      p += c * per;
      R.part[q] = La.lv[q].part;
      R.Y[q] = La.lv[q].Y;
      R.nchunks[q] = c;
      R.count[q] = (int64_t)La.lv[q].r0 * La.lv[q].nk * La.lv[q].r1;
      R.left[q] = La.lv[q].left;
      R.vlen[q] = La.lv[q].vlen;
      R.W[q] = La.lv[q].nk * La.lv[q].wrow;
      R.wrow[q] = La.lv[q].wrow;
      R.r0[q] = La.lv[q].r0;
      R.nk[q] = La.lv[q].nk;
      R.r1[q] = La.lv[q].r1;
    }
    R.n = n;
    (void)part_cap;
    launch_back(s, La, La.split[n], smem, vmax, sc, lc);
    const int64_t outs = R.count[0] + (n > 1 ? R.count[1] : 0);
    k_zreduce<<<blocks_for(outs * 32, 256), 256, 0, s>>>(R, sc);
    ++*lc;
  }
  // chain launch of the small tails (one CTA per side)
  if (nbig[0] < left.size() || nbig[1] < right.size()) {
    BackLaunch La{};
    La.chain = 1;
    int n = 0, g = 0;
    size_t smem = 0;
    int vmax = 1;
    La.split[0] = 0;
    for (int sd = 0; sd < 2; ++sd) {
      if (nbig[sd] >= side[sd]->size()) continue;
      for (size_t i = nbig[sd]; i < side[sd]->size(); ++i) {
        La.lv[n] = mk((*side[sd])[i]);
        smem = std::max(smem, back_smem(La.lv[n]));
        vmax = std::max(vmax, La.lv[n].vlen);
        ++n;
      }
      La.split[++g] = n;
    }
    La.nlv = n;
    launch_back(s, La, g, smem, vmax, sc, lc);
  }
}

int64_t level_partial_need(int64_t per_level_max) { return 2 * per_level_max; }

void levels_init() {
  const int bytes = 200 * 1024;
  cudaFuncSetAttribute(k_tab_levels<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_tab_levels<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_back_levels<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_back_levels<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_back_levels<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace prgd
