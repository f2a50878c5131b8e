// FP64 peak microbenchmark (diagnostic): DFMA chains and DMMA m8n8k4 on all SMs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 20000, blocks = sms * 4, threads = 256;
    k_dfma<<<blocks, threads>>>(d, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s (%d SMs)\n", fl / ms / 1e9, sms);
    k_dmma<<<blocks, threads>>>(d, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dmma<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 8 * 4 * 4 * iters * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s\n", fl / ms / 1e9);
    // single SM
    cudaEventRecord(e0); k_dfma<<<1, 1024>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA 1 CTA x1024: %.1f GFLOP/s\n", 2.0 * 8 * iters * 1024 / ms / 1e6);
    cudaEventRecord(e0); k_dmma<<<1, 1024>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA 1 CTA x1024: %.1f GFLOP/s\n", 2.0 * 8 * 8 * 4 * 4 * iters * 32 / ms / 1e6);
  }
  return 0;
}
