// Diagnostic: pass-A-shaped traffic (30M random 128-B gathers from a 134 MB table, plus
// sequential streams: 4-B gather index, 8-B y read, 8-B g write, 134 MB prefix rows) under
// different L2 policies.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ double2 ld2(const double* p, uint64_t pol) {
  double2 v; asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol)); return v; }
__device__ __forceinline__ double ld1(const double* p, uint64_t pol) {
  double v; asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol)); return v; }
__device__ __forceinline__ int ldi(const int* p, uint64_t pol) {
  int v; asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol)); return v; }
__device__ __forceinline__ void st1(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(p), "d"(v), "l"(pol)); }

__global__ void k_init(double* t, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) t[i] = (double)(i & 1023);
}
__global__ void k_idx(int* idx, int64_t m, int64_t rows, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed; x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    idx[i] = (int)(x % rows);
  }
}
// one warp per "row" of ~29 samples: reads the prefix row A (128 B), then for each sample
// gathers T[idx] (128 B), dot with A, g = dot - y.  MODE 0 plain, 1 hints.
template <int MODE>
__global__ void k_pass(const double* __restrict__ T, const double* __restrict__ A, const int* __restrict__ idx,
                       const double* __restrict__ y, double* __restrict__ g, int64_t m, int64_t nrows) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t pf = 0, pl = 0;
  if (MODE) { pf = pol_first(); pl = pol_last(); }
  for (int64_t row = w; row < nrows; row += nw) {
    const int64_t s0 = row * m / nrows, s1 = (row + 1) * m / nrows;
    double2 a = MODE ? ld2(A + row * 16 + sub * 2, pf) : __ldg(reinterpret_cast<const double2*>(A + row * 16) + sub);
    for (int64_t base = s0; base < s1; base += 16) {
      double2 v[4]; int64_t ss[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int64_t s = base + u * 4 + grp; ss[u] = s;
        if (s < s1) {
          int j = MODE ? ldi(idx + s, pf) : __ldg(idx + s);
          v[u] = MODE ? ld2(T + (int64_t)j * 16 + sub * 2, pl) : __ldg(reinterpret_cast<const double2*>(T + (int64_t)j * 16) + sub);
        } else v[u] = make_double2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double dsum = v[u].x * a.x + v[u].y * a.y;
        dsum += __shfl_xor_sync(0xffffffffu, dsum, 1); dsum += __shfl_xor_sync(0xffffffffu, dsum, 2); dsum += __shfl_xor_sync(0xffffffffu, dsum, 4);
        if (sub == 0 && ss[u] < s1) {
          double yy = MODE ? ld1(y + ss[u], pf) : __ldg(y + ss[u]);
          if (MODE) st1(g + ss[u], dsum - yy, pf); else g[ss[u]] = dsum - yy;
        }
      }
    }
  }
}
int main() {
  const int64_t rows = 1 << 20, m = 30000000, nrows = 1 << 20;
  double *T, *A, *y, *g; int* idx;
  cudaMalloc(&T, rows * 128); cudaMalloc(&A, nrows * 128); cudaMalloc(&idx, m * 4); cudaMalloc(&y, m * 8); cudaMalloc(&g, m * 8);
  k_init<<<1024, 256>>>(T, rows * 16); k_init<<<1024, 256>>>(A, nrows * 16); k_init<<<1024, 256>>>(y, m);
  k_idx<<<1024, 256>>>(idx, m, rows, 777);
  cudaDeviceSynchronize();
  int dev = 0; cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  printf("L2 %d MB, persisting max %d MB, accessPolicyMaxWindow %d MB\n", pr.l2CacheSize >> 20, pr.persistingL2CacheMaxSize >> 20, pr.accessPolicyMaxWindowSize >> 20);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](int mode, const char* name) {
    for (int blocks : {148 * 8, 148 * 16}) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, st);
        if (mode) k_pass<1><<<blocks, 256, 0, st>>>(T, A, idx, y, g, m, nrows);
        else k_pass<0><<<blocks, 256, 0, st>>>(T, A, idx, y, g, m, nrows);
        cudaEventRecord(e1, st); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("%-28s blocks %5d: %.3f ms (gathers %.0f GB/s)\n", name, blocks, best, m * 128.0 / best / 1e6);
    }
  };
  run(0, "plain");
  run(1, "evict_first streams/last T");
  // persisting access-policy window over the gathered table
  size_t lim = pr.persistingL2CacheMaxSize;
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
  for (float frac : {0.5f, 1.0f}) {
    cudaStreamAttrValue at = {};
    at.accessPolicyWindow.base_ptr = T;
    at.accessPolicyWindow.num_bytes = (size_t)(rows * 128) < (size_t)pr.accessPolicyMaxWindowSize ? rows * 128 : pr.accessPolicyMaxWindowSize;
    at.accessPolicyWindow.hitRatio = frac * (float)lim / (float)at.accessPolicyWindow.num_bytes > 1.f ? 1.f : frac * (float)lim / (float)at.accessPolicyWindow.num_bytes;
    at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &at);
    printf("window %zu MB hitRatio %.2f\n", at.accessPolicyWindow.num_bytes >> 20, at.accessPolicyWindow.hitRatio);
    run(0, "plain + window");
    run(1, "hints + window");
    cudaCtxResetPersistingL2Cache();
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
