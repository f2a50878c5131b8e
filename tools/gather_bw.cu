// Microbenchmark (diagnostic): random 128-byte row gathers from a large table, the access
// pattern of the pass kernels.  Reports useful GB/s (rows x 128 B / time).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__global__ void k_init(double* t, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) t[i] = (double)(i & 1023);
}
__global__ void k_idx(int* idx, int64_t m, int64_t rows, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed; x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    idx[i] = (int)(x % rows);
  }
}
// 8 lanes per row (double2 each), each warp handles 4 rows per step, UNR steps in flight
template <int UNR>
__global__ void k_gather(const double* __restrict__ t, const int* __restrict__ idx, int64_t m, double* out) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  for (int64_t base = w * 4 * UNR; base < m; base += nw * 4 * UNR) {
    double2 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int64_t s = base + u * 4 + grp;
      v[u] = s < m ? __ldg(reinterpret_cast<const double2*>(t + (int64_t)idx[s] * 16) + sub) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 1234.5) out[0] = acc;
}
int main() {
  for (int64_t rows : {(int64_t)1 << 20, (int64_t)1 << 23, (int64_t)1 << 26}) {
    const int64_t m = 30000000;
    double* t; int* idx; double* out;
    cudaMalloc(&t, rows * 16 * 8); cudaMalloc(&idx, m * 4); cudaMalloc(&out, 8);
    k_init<<<1024, 256>>>(t, rows * 16); k_idx<<<1024, 256>>>(idx, m, rows, 12345);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
      k_gather<8><<<blocks, 256>>>(t, idx, m, out);
      cudaEventRecord(e0);
      k_gather<8><<<blocks, 256>>>(t, idx, m, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("table %6.0f MB  blocks %5d  UNR 8: %.3f ms  %.0f GB/s useful (+idx %.0f GB/s)\n", rows * 128.0 / 1e6, blocks, ms,
             m * 128.0 / ms / 1e6, m * 4.0 / ms / 1e6);
    }
    for (int blocks : {148 * 8}) {
      k_gather<16><<<blocks, 256>>>(t, idx, m, out);
      cudaEventRecord(e0);
      k_gather<16><<<blocks, 256>>>(t, idx, m, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("table %6.0f MB  blocks %5d  UNR16: %.3f ms  %.0f GB/s useful\n", rows * 128.0 / 1e6, blocks, ms, m * 128.0 / ms / 1e6);
    }
    cudaFree(t); cudaFree(idx); cudaFree(out);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
