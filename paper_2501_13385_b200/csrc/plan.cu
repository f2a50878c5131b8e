// plan.cu — device-side construction of the pass work plans (SegPlan) from the bucket
// offsets left on the device by the bucketing sorts (A0), so tt_set_observations moves no
// per-row data between host and device.
//
// A plan over nr = nblk * nrow buckets (rows):
//   * virtual rows: a row with cnt <= kSplit samples is one virtual row; a longer row is split
//     into ceil(cnt / kSplit) consecutive virtual rows whose results go to partial slots,
//     summed in slot order by k_seg_fix (so every sum keeps a fixed order);
//   * warps: a warp owns a run of consecutive virtual rows of one gather block; a new warp
//     starts where the running cost sum_{v' < v} (cnt_v' + kVrowCost) within the block
//     crosses a multiple of kWarpCost.  (Any run decomposition gives identical results;
//     only the balance changes.)
// Every step is a per-element kernel or an exclusive scan (three-pass, int64 sums).
#include "prgd_internal.cuh"

namespace prgd {
namespace {

constexpr int kPT = 256;                 // threads per block
constexpr int kSeg = 4096;               // scan segment per block
constexpr int kPer = kSeg / kPT;         // contiguous elements per thread

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + kPT - 1) / kPT); }

// per row: virtual-row count, split flag, partial-slot count
__global__ void k_plan_rows(const int64_t* __restrict__ offs, int64_t nr, int64_t split,
                            int* __restrict__ nv, int* __restrict__ sp, int* __restrict__ np) {
  const int64_t P = blockIdx.x * (int64_t)kPT + threadIdx.x;
  if (P >= nr) return;
  const int64_t cnt = offs[P + 1] - offs[P];
  const int v = cnt <= split ? 1 : (int)((cnt + split - 1) / split);
  nv[P] = v;
  sp[P] = cnt > split ? 1 : 0;
  np[P] = cnt > split ? v : 0;
}

// exclusive scan, int32 in -> int64 out[0..len] (out[len] = total): segment sums, one-block
// scan of the sums, in-order segment scans.
__global__ void k_pscan_sums(const int* __restrict__ in, int64_t len, long long* __restrict__ bsum) {
  __shared__ long long red[kPT];
  const int64_t base = (int64_t)blockIdx.x * kSeg;
  long long s = 0;
  for (int i = threadIdx.x; i < kSeg; i += kPT)
    if (base + i < len) s += in[base + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kPT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = red[0];
}

__global__ void k_pscan_top(long long* __restrict__ bsum, int nb) {
  // one block: chunked serial scan by thread 0 is enough (nb <= a few hundred)
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int i = 0; i < nb; ++i) {
      const long long t = bsum[i];
      bsum[i] = run;
      run += t;
    }
    bsum[nb] = run;
  }
}

__global__ void k_pscan_apply(const int* __restrict__ in, int64_t len, const long long* __restrict__ bsum,
                              int nb, int64_t* __restrict__ out) {
  __shared__ long long tot[kPT];
  const int64_t base = (int64_t)blockIdx.x * kSeg + (int64_t)threadIdx.x * kPer;
  int v[kPer];
  long long s = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    v[k] = base + k < len ? in[base + k] : 0;
    s += v[k];
  }
  tot[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = bsum[blockIdx.x];
    for (int i = 0; i < kPT; ++i) {
      const long long t = tot[i];
      tot[i] = run;
      run += t;
    }
  }
  __syncthreads();
  long long run = tot[threadIdx.x];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (base + k < len) out[base + k] = run;
    run += v[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[len] = bsum[nb];
}

// fill the virtual rows of every row and the split-row table; cost per virtual row
__global__ void k_plan_fill(const int64_t* __restrict__ offs, int64_t nr, int64_t split,
                            const int64_t* __restrict__ vbase, const int64_t* __restrict__ sbase,
                            const int64_t* __restrict__ pbase, int4* __restrict__ vrow,
                            int32_t* __restrict__ split_row,
                            int64_t* __restrict__ split_first, int* __restrict__ cost, int vcost) {
  const int64_t P = blockIdx.x * (int64_t)kPT + threadIdx.x;
  if (P == 0) split_first[sbase[nr]] = pbase[nr];
  if (P >= nr) return;
  const int64_t beg = offs[P], cnt = offs[P + 1] - beg;
  const int64_t v0 = vbase[P];
  if (cnt <= split) {
    vrow[v0] = make_int4((int)P, (int)cnt, (int)beg, -1);
    cost[v0] = (int)cnt + vcost;
    return;
  }
  const int64_t sidx = sbase[P], p0 = pbase[P];
  split_row[sidx] = (int32_t)P;
  split_first[sidx] = p0;
  const int64_t nv = vbase[P + 1] - v0;
  for (int64_t t = 0; t < nv; ++t) {
    const int64_t o = t * split;
    const int c = (int)(cnt - o < split ? cnt - o : split);
    vrow[v0 + t] = make_int4((int)P, c, (int)(beg + o), (int)(p0 + t));
    cost[v0 + t] = c + vcost;
  }
}

// warp-start flags: first virtual row of a gather block, or the block-relative running cost
// crosses a multiple of wcost
__global__ void k_plan_flags(const int64_t* __restrict__ C, const int4* __restrict__ vrow,
                             int64_t nvrows, int64_t nrow, const int64_t* __restrict__ vbase,
                             int64_t wcost, int* __restrict__ flag) {
  const int64_t v = blockIdx.x * (int64_t)kPT + threadIdx.x;
  if (v >= nvrows) return;
  const int64_t b = vrow[v].x / nrow;
  const int64_t v0 = vbase[b * nrow];
  int f = v == v0;
  if (!f) {
    const int64_t base = C[v0];
    f = (C[v] - base) / wcost != (C[v - 1] - base) / wcost;
  }
  flag[v] = f;
}

__global__ void k_plan_warps(const int* __restrict__ flag, const int64_t* __restrict__ wid,
                             int64_t nvrows, int64_t* __restrict__ warp_vbegin) {
  const int64_t v = blockIdx.x * (int64_t)kPT + threadIdx.x;
  if (v == 0) warp_vbegin[wid[nvrows]] = nvrows;
  if (v >= nvrows) return;
  if (flag[v]) warp_vbegin[wid[v]] = v;
}

// per gather block b: first virtual row, first split row, first warp (+ the totals at nblk)
__global__ void k_plan_blocks(const int64_t* __restrict__ vbase, const int64_t* __restrict__ sbase,
                              const int64_t* __restrict__ wid, int64_t nrow, int nblk,
                              int64_t* __restrict__ out) {
  const int b = threadIdx.x;
  if (b > nblk) return;
  const int64_t P = (int64_t)b * nrow;   // b == nblk: the totals
  const int64_t v = vbase[P];
  out[b] = v;
  out[(nblk + 1) + b] = sbase[P];
  out[2 * (nblk + 1) + b] = wid[v];
}

void scan_i32(cudaStream_t s, const int* in, int64_t len, int64_t* out, long long* bsum,
              int64_t* launches) {
  const int nb = (int)((len + kSeg - 1) / kSeg);
  if (nb > 0) k_pscan_sums<<<nb, kPT, 0, s>>>(in, len, bsum);
  k_pscan_top<<<1, 32, 0, s>>>(bsum, nb);
  k_pscan_apply<<<nb > 0 ? nb : 1, kPT, 0, s>>>(in, len, bsum, nb, out);
  *launches += nb > 0 ? 3 : 2;
}

}  // namespace

int64_t plan_scan_scratch(int64_t len) { return (len + kSeg - 1) / kSeg + 2; }

void launch_scan_i32(cudaStream_t s, const int* in, int64_t len, int64_t* out, long long* bsum,
                     int64_t* launches) {
  scan_i32(s, in, len, out, bsum, launches);
}

void launch_plan_rows(cudaStream_t s, const int64_t* offs, int64_t nr, int64_t split, int* nv, int* sp,
                      int* np, int64_t* vbase, int64_t* sbase, int64_t* pbase, long long* bsum,
                      int64_t* launches) {
  if (nr > 0) {
    k_plan_rows<<<blocks_for(nr), kPT, 0, s>>>(offs, nr, split, nv, sp, np);
    ++*launches;
  }
  scan_i32(s, nv, nr, vbase, bsum, launches);
  scan_i32(s, sp, nr, sbase, bsum, launches);
  scan_i32(s, np, nr, pbase, bsum, launches);
}

void launch_plan_fill(cudaStream_t s, const int64_t* offs, int64_t nr, int64_t nrow, int nblk,
                      int64_t split, const int64_t* vbase, const int64_t* sbase, const int64_t* pbase,
                      int64_t nvrows, int4* vrow, int32_t* split_row, int64_t* split_first, int vcost,
                      int64_t wcost, int* cost, int64_t* C, int* flag, int64_t* wid,
                      long long* bsum, int64_t* blk_out, int64_t* launches) {
  k_plan_fill<<<blocks_for(nr > 0 ? nr : 1), kPT, 0, s>>>(offs, nr, split, vbase, sbase, pbase, vrow,
                                                          split_row, split_first, cost, vcost);
  ++*launches;
  scan_i32(s, cost, nvrows, C, bsum, launches);
  if (nvrows > 0) {
    k_plan_flags<<<blocks_for(nvrows), kPT, 0, s>>>(C, vrow, nvrows, nrow, vbase, wcost, flag);
    ++*launches;
  }
  scan_i32(s, flag, nvrows, wid, bsum, launches);
  k_plan_blocks<<<1, 64, 0, s>>>(vbase, sbase, wid, nrow, nblk, blk_out);
  ++*launches;
}

void launch_plan_warps(cudaStream_t s, const int* flag, const int64_t* wid, int64_t nvrows,
                       int64_t* warp_vbegin, int64_t* launches) {
  k_plan_warps<<<blocks_for(nvrows > 0 ? nvrows : 1), kPT, 0, s>>>(flag, wid, nvrows, warp_vbegin);
  ++*launches;
}

}  // namespace prgd
