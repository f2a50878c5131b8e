// Latency of dependent fp64 ops on one thread (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0) {
  double x = x0; long long t0, t1;
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = fma(x, 1.0000001, 1e-9); t1 = clock64(); cyc[0] = (t1 - t0) / 1000;
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = 1.0 / (x + 1e-3) + 0.5; t1 = clock64(); cyc[1] = (t1 - t0) / 1000;
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = sqrt(x + 1e-3) + 0.5; t1 = clock64(); cyc[2] = (t1 - t0) / 1000;
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = rsqrt(x + 1e-3) + 0.5; t1 = clock64(); cyc[3] = (t1 - t0) / 1000;
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = (x + 1e-3) / (x + 2.0) + 0.5; t1 = clock64(); cyc[4] = (t1 - t0) / 1000;
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * 1.0000001; t1 = clock64(); cyc[5] = (t1 - t0) / 1000;
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = (double)__frcp_rn((float)x) + 0.5; t1 = clock64(); cyc[6] = (t1 - t0) / 1000;
  {
    double d0 = x, d1 = 0.0, a = x * 1e-3, b = 1.0;
    t0 = clock64();
    for (int i = 0; i < 1000; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    t1 = clock64(); cyc[7] = (t1 - t0) / 1000;
    x += d0 + d1;
  }
  __shared__ double sm[64];
  sm[threadIdx.x] = x; __syncwarp();
  t0 = clock64(); for (int i = 0; i < 1000; ++i) { x = sm[(int)x & 31] + 1.0; } t1 = clock64(); cyc[8] = (t1 - t0) / 1000;
  out[threadIdx.x] = x;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 256 * 8); cudaMallocManaged(&c, 16 * 8);
  k<<<1, 32>>>(d, c, 1.5); cudaDeviceSynchronize();
  const char* nm[] = {"dfma", "1/x", "sqrt", "rsqrt", "x/y", "shfl.f64", "frcp_rn f32", "dmma chain", "lds chain"};
  for (int i = 0; i < 9; ++i) printf("%-12s %lld cycles (dependent)\n", nm[i], c[i]);
}
