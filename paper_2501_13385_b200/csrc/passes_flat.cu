// passes_flat.cu — pass A over Omega (prefix order) as a flat, sample-major SDDMM.
//
// Same arithmetic as the row-plan kernel k_seg<SDDMM> of passes.cu (A1-A2 and the prefix
// bucket sums of A3), different work split: a warp owns 32 consecutive
// samples (in bucket order) per iteration and loads every per-sample array it needs (bucket
// row P, gathered column S, value y) lane-parallel up front, so the chunk's loads and both
// row gathers are independent and in flight together (the row-plan kernel waits on a chain of
// dependent loads per bucket: plan record -> row vector / samples -> gathers).  Measured on
// B200 at config 5: DRAM-bound (ncu: 5.4 TB/s of gathered-table traffic).
//
// The bucket sums H_L[P] = sum g_s^2 are a segmented reduction over the chunk (a warp scan on
// the sorted bucket index); a bucket the chunk holds completely is written directly, the bucket
// it shares with the previous chunk is left as a head record and the one it shares with the next
// chunk as a tail record (a chunk inside one bucket: a "full" head record); k_flat_fix adds
// tail(c) + head(c+1) + ... in chunk order.  Every sum has a fixed order (deterministic).  Empty
// buckets are written as zeros by the chunk holding the next bucket start (or the last sample).
#include "prgd_internal.cuh"

namespace prgd {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kFT = 256;            // threads per CTA

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// Per-chunk records of the bucket sums (chunk c = samples [32 c, 32 c + 32)).
struct Rec {
  double* head;        // [nchunks] sum over the chunk's first bucket when it began before the chunk
  double* tail;        // [nchunks] sum over the chunk's last bucket when it continues after it
  int32_t* head_row;   // bucket of the head record or -1
  int32_t* tail_row;   // bucket of the tail record or -1
  int8_t* full;        // the chunk lies inside one bucket that began before and continues after it
};

// Segmented bucket sums of one 32-sample chunk (lane = sample, v its g^2, rv its bucket; buckets
// nondecreasing): a segmented warp scan, complete buckets written, straddling ones left as chunk
// records for k_flat_fix, empty buckets written as zeros.
__device__ __forceinline__ void seg_bucket_sums(int lane, bool have, double v, int rv, int prev, int next,
                                                int64_t c, int64_t t, int64_t m, int64_t nrows,
                                                double* __restrict__ H, const Rec& rec) {
  const int key = have ? rv : -2;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {            // segmented inclusive scan (buckets contiguous)
    const double yo = __shfl_up_sync(kFull, v, o);
    const int ko = __shfl_up_sync(kFull, key, o);
    if (lane >= o && ko == key) v += yo;
  }
  const int kup = __shfl_up_sync(kFull, key, 1), kdn = __shfl_down_sync(kFull, key, 1);
  const int kprev = lane == 0 ? prev : kup;
  const int knext = lane == 31 ? next : (kdn == -2 ? -1 : kdn);
  const unsigned valid = __ballot_sync(kFull, have);
  const int last = 31 - __clz(valid);                          // last valid lane of the chunk
  const unsigned ends = __ballot_sync(kFull, have && (key != knext || lane == last));
  const int first_end = __ffs(ends) - 1;                       // end lane of the first segment
  if (have) {
    if (key != kprev)                                          // empty buckets before this one
      for (int bb = kprev + 1; bb < key; ++bb) H[bb] = 0.0;
    if ((ends >> lane) & 1u) {
      // the segment ending here began in the chunk unless it is the first one and continued
      const bool began = lane != first_end || key != prev;
      const bool finishes = key != knext;
      if (began && finishes) H[key] = v;
      if (lane == first_end) {
        rec.head_row[c] = began ? -1 : key;
        rec.head[c] = began ? 0.0 : v;
        rec.full[c] = (!began && !finishes) ? 1 : 0;
      }
      if (lane == last) {
        const bool tl = began && !finishes;
        rec.tail_row[c] = tl ? key : -1;
        rec.tail[c] = tl ? v : 0.0;
      }
      if (t == m - 1)                                          // empty buckets after the last sample
        for (int64_t bb = (int64_t)key + 1; bb < nrows; ++bb) H[bb] = 0.0;
    }
  }
}

// ------------------------------------------------------------------ SDDMM (A1-A2) + H_L (A3)
// g[t] = rowtab[row[t]] . coltab[col[t]] - y[t],  H[b] = sum_{row[t] = b} g[t]^2.  LPS lanes per
// sample, V double2 per lane (ld = 2 LPS V); per 32-sample chunk: lane-parallel loads of
// row / col / y, LPS steps of 32 / LPS samples (one per lane group), partial dot products finished
// by a transpose-reduction over the group (LPS - 1 shuffles), g back to natural order by one
// shuffle, then a segmented warp scan of g^2 by bucket.
template <int LPS, int V>
__global__ void __launch_bounds__(kFT, 4) k_flat_sddmm(const int32_t* __restrict__ row,
                                                      const int32_t* __restrict__ col,
                                                      const double* __restrict__ y, int64_t m,
                                                      int64_t nrows, const double* __restrict__ rowtab,
                                                      const double* __restrict__ coltab,
                                                      double* __restrict__ g, double* __restrict__ H,
                                                      Rec rec, bool pf) {
  constexpr int G = 32 / LPS, STEPS = LPS, ld = 2 * LPS * V;
  constexpr int UNR = STEPS < 4 ? STEPS : 4;
  const int lane = threadIdx.x & 31, grp = lane / LPS, sub = lane - grp * LPS;
  const int64_t w0 = (blockIdx.x * (int64_t)kFT + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)kFT) >> 5;
  for (int64_t c = w0; c * 32 < m; c += nw) {
    const int64_t t = c * 32 + lane;
    const bool have = t < m;
    // samples past the end gather row / column 0 (valid table rows); never stored
    const int rv = have ? row[t] : 0, cv = have ? col[t] : 0;
    const double yv = have ? y[t] : 0.0;
    const int prev = c == 0 ? -1 : row[c * 32 - 1];                      // bucket before the chunk
    const int next = c * 32 + 32 < m ? row[c * 32 + 32] : -1;            // bucket after it
    // the gathered rows of this warp's next chunk are prefetched into L2 when this one is done
    // (measured at config 5: 0.716 -> 0.636 ms; two chunks ahead 0.703 ms, the row-table rows as
    // well 0.653 ms; the same prefetch in k_spmm_pipe, whose rows already travel a chunk ahead by
    // cp.async, made pass B 2 % slower).  Only for tables that do not stay in L2 by themselves
    // (pf): on config 5's Omega at r = 1, a 16 MB table, the prefetch costs 0.295 -> 0.355 ms.
    const int64_t tn = (c + nw) * 32 + lane;
    const int cvn = (pf && tn < m) ? col[tn] : -1;
    double pd[STEPS];
#pragma unroll
    for (int s0 = 0; s0 < STEPS; s0 += UNR) {
      double2 a[UNR][V], b[UNR][V];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int tt = (s0 + u) * G + grp;
        const int ri = __shfl_sync(kFull, rv, tt), ci = __shfl_sync(kFull, cv, tt);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          a[u][q] = ldg2(rowtab + (int64_t)ri * ld + 2 * (V * sub + q));
          b[u][q] = ldg2(coltab + (int64_t)ci * ld + 2 * (V * sub + q));
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        double p = fma(a[u][0].x, b[u][0].x, a[u][0].y * b[u][0].y);
#pragma unroll
        for (int q = 1; q < V; ++q) p = fma(a[u][q].y, b[u][q].y, fma(a[u][q].x, b[u][q].x, p));
        pd[s0 + u] = p;
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
    const int tt = sub * G + grp;   // the sample this lane finished
    const double gv = pd[0] - __shfl_sync(kFull, yv, tt);
    if (c * 32 + tt < m) g[c * 32 + tt] = gv;
    // natural order: sample `lane` was finished by lane (lane % G) * LPS + lane / G
    const double gn = __shfl_sync(kFull, gv, (lane % G) * LPS + lane / G);
    seg_bucket_sums(lane, have, have ? gn * gn : 0.0, rv, prev, next, c, t, m, nrows, H, rec);
    if (cvn >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(coltab + (int64_t)cvn * ld));
  }
}

// ------------------------------------------------------------------ pass A suffix, one slice
// Suffix-order residuals by slices of g ("pass A suffix"): over one slice's
// samples (suffix order restricted to the samples whose prefix position lies in the slice, so
// every gather hits a ~48 MB window of g that stays in L2) stage[t] = g[pos[t]] and the slice's
// bucket sums H[b] = sum_{row[t] = b} stage[t]^2 (rows nondecreasing within a slice).
__global__ void __launch_bounds__(kFT) k_flat_gsq(const int32_t* __restrict__ row,
                                                 const int32_t* __restrict__ pos,
                                                 const double* __restrict__ g, int64_t m, int64_t nrows,
                                                 double* __restrict__ stage, double* __restrict__ H,
                                                 Rec rec) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kFT + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)kFT) >> 5;
  for (int64_t c = w0; c * 32 < m; c += nw) {
    const int64_t t = c * 32 + lane;
    const bool have = t < m;
    const int rv = have ? row[t] : 0;
    const double gv = have ? __ldg(g + pos[t]) : 0.0;
    if (have) stage[t] = gv;
    const int prev = c == 0 ? -1 : row[c * 32 - 1];
    const int next = c * 32 + 32 < m ? row[c * 32 + 32] : -1;
    seg_bucket_sums(lane, have, gv * gv, rv, prev, next, c, t, m, nrows, H, rec);
  }
}

// For every chunk whose tail record starts a bucket that continues: tail(c) + head(c+1) + ...
// (through the "full" chunks) in chunk order.
__global__ void k_flat_fix(Rec rec, int64_t nchunks, double* __restrict__ H) {
  const int64_t c = blockIdx.x * (int64_t)kFT + threadIdx.x;
  if (c >= nchunks) return;
  const int32_t b = rec.tail_row[c];
  if (b < 0) return;
  double s = rec.tail[c];
  for (int64_t c2 = c + 1; c2 < nchunks; ++c2) {
    s += rec.head[c2];
    if (!rec.full[c2]) break;
  }
  H[b] = s;
}

Rec make_rec(void* base, int64_t nchunks) {
  Rec r;
  r.head = reinterpret_cast<double*>(base);
  r.tail = r.head + nchunks;
  r.head_row = reinterpret_cast<int32_t*>(r.tail + nchunks);
  r.tail_row = r.head_row + nchunks;
  r.full = reinterpret_cast<int8_t*>(r.tail_row + nchunks);
  return r;
}

template <int LPS, int V>
void sddmm_launch(cudaStream_t s, const FlatArgs& a, const Rec& rec, unsigned grid) {
  // L2 prefetch of the gathered rows when the gathered table exceeds ~40 MB
  const bool pf = a.ncols * (int64_t)a.ld * 8 > (40ll << 20);
  k_flat_sddmm<LPS, V><<<grid, kFT, 0, s>>>(a.row, a.col, a.x, a.m, a.nrows, a.rowtab, a.coltab, a.g,
                                            a.out, rec, pf);
}

// H[b] = sum_q Hq[q][b] in slice order (deterministic).
__global__ void k_sum_slices(const double* __restrict__ Hq, int nq, int64_t n, double* __restrict__ H) {
  const int64_t b = blockIdx.x * (int64_t)kFT + threadIdx.x;
  if (b >= n) return;
  double acc = Hq[b];
  for (int q = 1; q < nq; ++q) acc += Hq[(int64_t)q * n + b];
  H[b] = acc;
}

}  // namespace

void launch_sum_slices(cudaStream_t s, const double* Hq, int nq, int64_t n, double* H, int64_t* launches) {
  k_sum_slices<<<cdiv(n, kFT), kFT, 0, s>>>(Hq, nq, n, H);
  ++*launches;
}

void launch_flat_gsq(cudaStream_t s, const int32_t* row, const int32_t* pos, const double* g, int64_t m,
                     int64_t nrows, double* stage, double* H, void* recbuf, int64_t* launches) {
  if (m <= 0) {
    cudaMemsetAsync(H, 0, (size_t)nrows * sizeof(double), s);
    return;
  }
  const int64_t nc = (m + 31) / 32;
  const Rec rec = make_rec(recbuf, nc);
  const int64_t cap = 148 * 8 * (kFT / 32) * 4;
  const unsigned grid = cdiv((nc < cap ? nc : cap) * 32, kFT);
  k_flat_gsq<<<grid, kFT, 0, s>>>(row, pos, g, m, nrows, stage, H, rec);
  k_flat_fix<<<cdiv(nc, kFT), kFT, 0, s>>>(rec, nc, H);
  *launches += 2;
}

int64_t flat_rec_bytes(int64_t m) {
  const int64_t nc = (m + 31) / 32 + 1;
  return nc * (2 * 8 + 2 * 4 + 1) + 64;
}

void launch_flat_sddmm(cudaStream_t s, const FlatArgs& a, int64_t* launches) {
  if (a.m <= 0) {
    cudaMemsetAsync(a.out, 0, (size_t)a.nrows * sizeof(double), s);
    return;
  }
  const int64_t nc = (a.m + 31) / 32;
  const Rec rec = make_rec(a.rec, nc);
  const int64_t cap = 148 * 4 * (kFT / 32) * 4;   // a few waves of resident warps, grid-stride
  const unsigned grid = cdiv((nc < cap ? nc : cap) * 32, kFT);
  switch (a.ld) {
    case 2: sddmm_launch<1, 1>(s, a, rec, grid); break;
    case 4: sddmm_launch<2, 1>(s, a, rec, grid); break;
    case 8: sddmm_launch<4, 1>(s, a, rec, grid); break;
    case 16: sddmm_launch<4, 2>(s, a, rec, grid); break;
    default: sddmm_launch<8, 2>(s, a, rec, grid); break;   // 32
  }
  k_flat_fix<<<cdiv(nc, kFT), kFT, 0, s>>>(rec, nc, a.out);
  *launches += 2;
}

}  // namespace prgd
