// sort.cu — A0: one-time bucketing of Omega ("A0").
//
// Each sample s gets a prefix index P(s) (mixed radix of x_0..x_{KL-1}, x_0 most
// significant) and a suffix index S(s) (mixed radix of x_KL..x_{d-1}, x_{d-1} most
// significant).  Prefix order = stable sort by key (P << bitsS) | S, suffix order = stable
// sort by (S << bitsP) | P: an LSD radix sort whose passes are stable counting sorts of 8-bit
// digits (histogram -> exclusive scan -> stable scatter).  The chain path sorts by x_k alone
// for every mode (chains.cu), the per-mode buckets of SURVEY §8(a) A0.
// The result is unique (stable sorts are), so it is compared bit-exactly with the
// oracle's numpy argsort(kind="stable") on the same keys.
#include "prgd_internal.cuh"

namespace prgd {

namespace {
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsSub = 512;                     // items per warp per tile
constexpr int kRsTile = kRsSub * kRsWarps;      // 4096 items per block

__global__ void k_make_keys(const int32_t* __restrict__ idx, int64_t m, int d,
                            const int* __restrict__ n, int KL, int bitsP, int bitsS,
                            uint64_t* __restrict__ kpre,
                            uint64_t* __restrict__ ksuf, uint32_t* __restrict__ vals, Scalars* sc) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= m) return;
  const int32_t* x = idx + s * d;
  uint64_t P = 0, S = 0;
  bool bad = false;
  for (int k = 0; k < KL; ++k) {
    int xk = x[k];
    bad |= (xk < 0) | (xk >= n[k]);
    P = P * (uint64_t)n[k] + (uint64_t)(xk < 0 ? 0 : xk);
  }
  for (int k = d - 1; k >= KL; --k) {
    int xk = x[k];
    bad |= (xk < 0) | (xk >= n[k]);
    S = S * (uint64_t)n[k] + (uint64_t)(xk < 0 ? 0 : xk);
  }
  if (bad) {
    atomicOr(&sc->index_err, 1);
    P = 0;
    S = 0;
  }
  kpre[s] = (P << bitsS) | S;
  ksuf[s] = (S << bitsP) | P;
  vals[s] = (uint32_t)s;
}

__global__ void k_rs_hist(const uint64_t* __restrict__ keys, int64_t m, int shift,
                          int* __restrict__ hist, int64_t nblocks) {
  __shared__ int cnt[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kRsTile;
  for (int i = threadIdx.x; i < kRsTile; i += blockDim.x) {
    int64_t t = base + i;
    if (t < m) atomicAdd(&cnt[(keys[t] >> shift) & 255u], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    hist[(int64_t)i * nblocks + blockIdx.x] = cnt[i];
}

// Exclusive scan of hist[0..len) in (digit, block) order, in three passes: segment sums
// (kScanSeg elements per block, coalesced), a one-block scan of the segment sums, and the
// in-order scan of each segment staged in shared memory.
constexpr int kScanSeg = 8192;
constexpr int kScanThreads = 256;
constexpr int kScanPer = kScanSeg / kScanThreads;   // 32 contiguous elements per thread

__global__ void k_scan_sums(const int* __restrict__ hist, int64_t len, long long* __restrict__ bsum) {
  __shared__ long long red[kScanThreads];
  const int64_t base = (int64_t)blockIdx.x * kScanSeg;
  long long s = 0;
  for (int i = threadIdx.x; i < kScanSeg; i += kScanThreads)
    if (base + i < len) s += hist[base + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kScanThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = red[0];
}

__global__ void k_scan_top(long long* __restrict__ bsum, int nb) {
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int i = 0; i < nb; ++i) {
      const long long t = bsum[i];
      bsum[i] = run;
      run += t;
    }
  }
}

__global__ void k_scan_apply(int* __restrict__ hist, int64_t len, const long long* __restrict__ bsum) {
  __shared__ int seg[kScanSeg];
  __shared__ long long tot[kScanThreads];
  const int64_t base = (int64_t)blockIdx.x * kScanSeg;
  for (int i = threadIdx.x; i < kScanSeg; i += kScanThreads)
    seg[i] = base + i < len ? hist[base + i] : 0;
  __syncthreads();
  long long s = 0;
  for (int k = 0; k < kScanPer; ++k) s += seg[threadIdx.x * kScanPer + k];
  tot[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = bsum[blockIdx.x];
    for (int i = 0; i < kScanThreads; ++i) {
      const long long t = tot[i];
      tot[i] = run;
      run += t;
    }
  }
  __syncthreads();
  long long run = tot[threadIdx.x];
  for (int k = 0; k < kScanPer; ++k) {
    const int v = seg[threadIdx.x * kScanPer + k];
    seg[threadIdx.x * kScanPer + k] = (int)run;
    run += v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kScanSeg; i += kScanThreads)
    if (base + i < len) hist[base + i] = seg[i];
}

// Stable scatter through shared memory: the tile's items are first placed in digit order in
// shared memory (warp w owns items [w*512, (w+1)*512) and walks them 32 at a time in order;
// __match_any_sync ranks equal digits by lane), then written out in that order, so consecutive
// threads write consecutive positions of each digit's output run (coalesced).
constexpr size_t kRsScatterSmem = (size_t)kRsTile * (sizeof(uint64_t) + sizeof(uint32_t));
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const uint64_t* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin,
                                                           uint64_t* __restrict__ kout,
                                                           uint32_t* __restrict__ vout, int64_t m,
                                                           int shift, const int* __restrict__ hist,
                                                           int64_t nblocks) {
  extern __shared__ uint64_t rs_sk[];                 // [kRsTile] keys, then [kRsTile] values
  uint32_t* rs_sv = reinterpret_cast<uint32_t*>(rs_sk + kRsTile);
  __shared__ int wcnt[kRsWarps][257];
  __shared__ int lstart[257], gbase[256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kRsWarps * 257; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile0 = (int64_t)blockIdx.x * kRsTile;
  const int64_t base = tile0 + (int64_t)w * kRsSub;
  for (int step = 0; step < kRsSub / 32; ++step) {
    int64_t t = base + step * 32 + lane;
    if (t < m) atomicAdd(&wcnt[w][(kin[t] >> shift) & 255u], 1);
  }
  __syncthreads();
  // per digit: tile total, then per-warp offsets inside the tile's digit run
  if (threadIdx.x < 256) {
    const int dg = threadIdx.x;
    int tot = 0;
    for (int w2 = 0; w2 < kRsWarps; ++w2) tot += wcnt[w2][dg];
    lstart[dg + 1] = tot;
    gbase[dg] = hist[(int64_t)dg * nblocks + blockIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    lstart[0] = 0;
    for (int dg = 0; dg < 256; ++dg) lstart[dg + 1] += lstart[dg];
  }
  __syncthreads();
  if (threadIdx.x < 256) {
    const int dg = threadIdx.x;
    int run = lstart[dg];
    for (int w2 = 0; w2 < kRsWarps; ++w2) {
      const int c = wcnt[w2][dg];
      wcnt[w2][dg] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int step = 0; step < kRsSub / 32; ++step) {
    int64_t t = base + step * 32 + lane;
    bool valid = t < m;
    uint64_t key = valid ? kin[t] : 0ull;
    uint32_t val = valid ? vin[t] : 0u;
    int dg = valid ? (int)((key >> shift) & 255u) : 256;
    unsigned peers = __match_any_sync(0xffffffffu, dg);
    int rank = __popc(peers & ((1u << lane) - 1u));
    int leader = __ffs(peers) - 1;
    int pos = wcnt[w][dg];
    if (valid) {
      rs_sk[pos + rank] = key;
      rs_sv[pos + rank] = val;
    }
    __syncwarp();
    if (lane == leader) wcnt[w][dg] = pos + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const int n = (int)(m - tile0 < kRsTile ? m - tile0 : kRsTile);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t key = rs_sk[i];
    const int dg = (int)((key >> shift) & 255u);
    const int64_t g = (int64_t)gbase[dg] + (i - lstart[dg]);
    kout[g] = key;
    vout[g] = rs_sv[i];
  }
}

__global__ void k_after_pre(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ sids,
                            int64_t m, int bitsS, int64_t NL, const double* __restrict__ y_orig,
                            int32_t* __restrict__ Spre, double* __restrict__ ypre,
                            int32_t* __restrict__ sid_pre, int32_t* __restrict__ inv,
                            int64_t* __restrict__ offsL, int32_t* __restrict__ Ppre) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= m) return;
  const uint64_t mask = (1ull << bitsS) - 1ull;
  uint64_t key = keys[t];
  int64_t P = (int64_t)(key >> bitsS);
  uint32_t sid = sids[t];
  Spre[t] = (int32_t)(key & mask);
  Ppre[t] = (int32_t)P;
  ypre[t] = y_orig[sid];
  sid_pre[t] = (int32_t)sid;
  inv[sid] = (int32_t)t;
  int64_t Pprev = t == 0 ? -1 : (int64_t)(keys[t - 1] >> bitsS);
  for (int64_t q = Pprev + 1; q <= P; ++q) offsL[q] = t;
  if (t == m - 1)
    for (int64_t q = P + 1; q <= NL; ++q) offsL[q] = m;
}

__global__ void k_after_suf(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ sids,
                            int64_t m, int bitsP, int64_t NR, const int32_t* __restrict__ inv,
                            int32_t* __restrict__ pos_suf, int32_t* __restrict__ Psuf,
                            int32_t* __restrict__ sid_suf, int32_t* __restrict__ pre2suf,
                            int64_t* __restrict__ offsR) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= m) return;
  const uint64_t mask = (1ull << bitsP) - 1ull;
  uint64_t key = keys[u];
  int64_t S = (int64_t)(key >> bitsP);
  uint32_t sid = sids[u];
  Psuf[u] = (int32_t)(key & mask);
  pos_suf[u] = inv[sid];
  pre2suf[inv[sid]] = (int32_t)u;
  sid_suf[u] = (int32_t)sid;
  int64_t Sprev = u == 0 ? -1 : (int64_t)(keys[u - 1] >> bitsP);
  for (int64_t q = Sprev + 1; q <= S; ++q) offsR[q] = u;
  if (u == m - 1)
    for (int64_t q = S + 1; q <= NR; ++q) offsR[q] = m;
}

// Slices of the suffix order for the sliced pass A suffix (passes_flat.cu k_flat_gsq): slice of
// a suffix-ordered sample u = its prefix position / slen.
__global__ void k_slice_keys(const int32_t* __restrict__ pos_suf, int64_t m, int64_t slen,
                             uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= m) return;
  keys[u] = (uint64_t)(pos_suf[u] / slen);
  vals[u] = (uint32_t)u;
}

// j-th sample of the sliced order (slice-major, suffix order within a slice) = suffix-ordered
// sample u = vo[j]: its prefix position, its suffix bucket, and u -> j.
__global__ void k_slice_order(const uint32_t* __restrict__ vo, const uint64_t* __restrict__ keys_suf,
                              int bitsP, const int32_t* __restrict__ pos_suf, int64_t m,
                              int32_t* __restrict__ sl_pos, int32_t* __restrict__ sl_row,
                              int32_t* __restrict__ sl_q) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const uint32_t u = vo[j];
  sl_pos[j] = pos_suf[u];
  sl_row[j] = (int32_t)(keys_suf[u] >> bitsP);
  sl_q[u] = (int32_t)j;
}

inline unsigned grid_for(int64_t n, int threads) {
  return (unsigned)((n + threads - 1) / threads);
}
}  // namespace

void launch_slice_setup(cudaStream_t s, const int32_t* pos_suf, const uint64_t* keys_suf, int bitsP,
                        int64_t m, int64_t slen, int nslices, uint64_t* kbuf, uint32_t* vbuf,
                        uint64_t* ktmp, uint32_t* vtmp, int* hist, int64_t hist_len, int32_t* sl_pos,
                        int32_t* sl_row, int32_t* sl_q, int64_t* launches) {
  if (m <= 0) return;
  k_slice_keys<<<grid_for(m, 256), 256, 0, s>>>(pos_suf, m, slen, kbuf, vbuf);
  int bits = 1;
  while ((1 << bits) < nslices) ++bits;
  uint64_t* ko;
  uint32_t* vo;
  radix_sort_pairs(s, kbuf, vbuf, ktmp, vtmp, m, bits, hist, hist_len, &ko, &vo, launches);
  k_slice_order<<<grid_for(m, 256), 256, 0, s>>>(vo, keys_suf, bitsP, pos_suf, m, sl_pos, sl_row, sl_q);
  *launches += 2;
}

int64_t radix_hist_len(int64_t m) {
  int64_t nb = (m + kRsTile - 1) / kRsTile;
  if (nb < 1) nb = 1;
  const int64_t len = 256 * nb;
  return len + 2 + 2 * ((len + kScanSeg - 1) / kScanSeg + 1);   // + segment sums (int64)
}

// Compact multi-indices (tt_set_observations_u8): one byte per index widened to the int32
// layout every consumer reads; 16 indices per thread (one 16-byte load, four 16-byte stores).
__global__ void k_widen_u8(const uint8_t* __restrict__ in, int64_t count, int32_t* __restrict__ out) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 16;
  if (i + 16 <= count) {
    const uint4 v = *reinterpret_cast<const uint4*>(in + i);
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<int4*>(out + i + 4 * q) =
          make_int4(w[q] & 255u, (w[q] >> 8) & 255u, (w[q] >> 16) & 255u, w[q] >> 24);
  } else {
    for (int64_t j = i; j < count; ++j) out[j] = in[j];
  }
}

void launch_widen_u8(cudaStream_t s, const uint8_t* in, int64_t count, int32_t* out, int64_t* launches) {
  if (count <= 0) return;
  k_widen_u8<<<grid_for((count + 15) / 16, 256), 256, 0, s>>>(in, count, out);
  ++*launches;
}

void launch_make_keys(cudaStream_t s, const int32_t* idx, int64_t m, int d, const int* n_dev,
                      int KL, int bitsP, int bitsS, uint64_t* kpre, uint64_t* ksuf, uint32_t* vals,
                      Scalars* sc, int64_t* launches) {
  if (m <= 0) return;
  k_make_keys<<<grid_for(m, 256), 256, 0, s>>>(idx, m, d, n_dev, KL, bitsP, bitsS, kpre, ksuf, vals, sc);
  ++*launches;
}

void radix_sort_pairs(cudaStream_t s, uint64_t* keys, uint32_t* vals, uint64_t* keys_tmp,
                      uint32_t* vals_tmp, int64_t m, int bits, int* hist, int64_t hist_len,
                      uint64_t** keys_out, uint32_t** vals_out, int64_t* launches) {
  uint64_t* kin = keys;
  uint32_t* vin = vals;
  uint64_t* ko = keys_tmp;
  uint32_t* vo = vals_tmp;
  if (m > 0) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_rs_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRsScatterSmem);
      attr = true;
    }
    int64_t nblocks = (m + kRsTile - 1) / kRsTile;
    (void)hist_len;
    for (int shift = 0; shift < bits; shift += 8) {
      k_rs_hist<<<(unsigned)nblocks, kRsThreads, 0, s>>>(kin, m, shift, hist, nblocks);
      {
        const int64_t len = 256 * nblocks;
        const int nb = (int)((len + kScanSeg - 1) / kScanSeg);
        long long* bsum = reinterpret_cast<long long*>(hist + len + (len & 1));
        k_scan_sums<<<nb, kScanThreads, 0, s>>>(hist, len, bsum);
        k_scan_top<<<1, 32, 0, s>>>(bsum, nb);
        k_scan_apply<<<nb, kScanThreads, 0, s>>>(hist, len, bsum);
        *launches += 2;
      }
      k_rs_scatter<<<(unsigned)nblocks, kRsThreads, kRsScatterSmem, s>>>(kin, vin, ko, vo, m, shift,
                                                                         hist, nblocks);
      *launches += 3;
      uint64_t* tk = kin;
      kin = ko;
      ko = tk;
      uint32_t* tv = vin;
      vin = vo;
      vo = tv;
    }
  }
  *keys_out = kin;
  *vals_out = vin;
}

void launch_after_sort_pre(cudaStream_t s, const uint64_t* keys, const uint32_t* sids, int64_t m,
                           int bitsS, int64_t NL, const double* y_orig, int32_t* Spre,
                           double* ypre, int32_t* sid_pre, int32_t* inv, int64_t* offsL,
                           int32_t* Ppre, int64_t* launches) {
  if (m <= 0) return;
  k_after_pre<<<grid_for(m, 256), 256, 0, s>>>(keys, sids, m, bitsS, NL, y_orig, Spre, ypre,
                                                sid_pre, inv, offsL, Ppre);
  ++*launches;
}

void launch_after_sort_suf(cudaStream_t s, const uint64_t* keys, const uint32_t* sids, int64_t m,
                           int bitsP, int64_t NR, const int32_t* inv, int32_t* pos_suf,
                           int32_t* Psuf, int32_t* sid_suf, int32_t* pre2suf, int64_t* offsR,
                           int64_t* launches) {
  if (m <= 0) return;
  k_after_suf<<<grid_for(m, 256), 256, 0, s>>>(keys, sids, m, bitsP, NR, inv, pos_suf, Psuf,
                                                sid_suf, pre2suf, offsR);
  ++*launches;
}

}  // namespace prgd
