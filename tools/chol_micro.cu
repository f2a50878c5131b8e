// Microbenchmark (diagnostic): cycles of the warp Cholesky + inverse of the cluster rounding
// in isolation (1 CTA).
#include "../paper_2501_13385_b200/csrc/dense.cu"
#include <cstdio>

namespace prgd {
namespace {
__global__ void k_chol_micro(long long* cyc, double* out, int n) {
  __shared__ double G[32 * 33], Lo[32 * 33], Li[32 * 36], rinv[32];
  __shared__ int flag;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e / n, j = e % n;
    G[i * 33 + j] = (i == j ? n + 1.0 : 0.0) + 1.0 / (1.0 + i + j);
  }
  __syncthreads();
  long long t0 = clock64();
  bool ok = true;
  for (int rep = 0; rep < 10; ++rep) ok = warp_chol_any(G, 33, n, 0.0, Lo, 33, Li, 36, rinv, &flag) && ok;
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 10; out[0] = Li[n - 1] + (ok ? 0 : 1); }
  if (threadIdx.x == 0) {
    long long s0, s1;
    double* Bs = Lo; double* Bis = Li;
    for (int e = 0; e < 64; ++e) Bs[e] = G[(e / 8) * 33 + e % 8];
    s0 = clock64();
    for (int rep = 0; rep < 10; ++rep) { ok = chol8_thread(Bs, 8, 8, Bis, 8, rinv) && ok; }
    s1 = clock64();
    cyc[6] = (s1 - s0) / 10; cyc[5] = 0;
  }
  __syncthreads();
  t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) ok = warp_chol_any(G, 33, n, 0.0, Lo, 33, nullptr, 36, rinv, &flag) && ok;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / 10;
  double x = 1.5;
  t0 = clock64();
  for (int rep = 0; rep < 100; ++rep) x = fast_rsqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) { cyc[2] = (t1 - t0) / 100; out[1] = x; }
  t0 = clock64();
  for (int rep = 0; rep < 100; ++rep) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / 100;
  t0 = clock64();
  double dv = 0;
  for (int rep = 0; rep < 10; ++rep) dv += blk_max_dev_identity(G, 33, n, Lo);
  t1 = clock64();
  if (threadIdx.x == 0) { cyc[4] = (t1 - t0) / 10; out[2] = dv; }
}
}  // namespace
}  // namespace prgd

int main() {
  long long* c; double* o;
  cudaMallocManaged(&c, 64 * 8); cudaMallocManaged(&o, 64 * 8);
  for (int n : {16, 32}) {
    prgd::k_chol_micro<<<1, 256>>>(c, o, n);
    cudaDeviceSynchronize();
    printf("n=%d chol+inv %lld cyc, chol %lld cyc, fast_rsqrt %lld cyc, syncthreads %lld cyc, maxdev %lld cyc, chol8 local %lld smem %lld (%s)\n",
           n, c[0], c[1], c[2], c[3], c[4], c[5], c[6], cudaGetErrorString(cudaGetLastError()));
  }
}
