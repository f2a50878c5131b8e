// Microbenchmark of the single-CTA dense primitives (diagnostic tool, not product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2501_13385_b200/csrc tools/dense_micro.cu -o /tmp/dm
#include "../paper_2501_13385_b200/csrc/dense.cu"
#include <cstdio>
#include <vector>

namespace prgd {
namespace {
__global__ void __launch_bounds__(kDenseThreads) k_micro(int which, int m, int n, int reps, long long* out) {
  extern __shared__ double smraw[];
  Work w = carve(smraw, (200 * 1024) / 8, 32);
  const int ld = n | 1;
  double* A = w.mat;
  for (int e = threadIdx.x; e < m * ld; e += blockDim.x) {
    const int i = e / ld, c = e % ld;
    A[e] = (c == i % n ? 3.0 : 0.0) + 0.01 * ((i * 7 + c * 13) % 17) / 17.0;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (which == 0) {
      double* G = w.S4; const int gl = n | 1;
      mma_gemm(n, n, m, [&](int i, int k) { return i < n ? A[(int64_t)k * ld + i] : 0.0; },
               [&](int k, int j) { return j < n ? A[(int64_t)k * ld + j] : 0.0; },
               [&](int i, int j, double v) { if (i < n && j < n) G[i * gl + j] = v; });
      __syncthreads();
    }
    else if (which == 1) {
      for (int e = threadIdx.x; e < n * (n | 1); e += blockDim.x) {
        const int i = e / (n | 1), c = e % (n | 1);
        w.S4[e] = (i == c ? 100.0 : 0.0) + 0.5 / (1 + i + c);
      }
      __syncthreads();
      chol_cta(w.S4, n | 1, n, w.sc3 + 4);
    } else if (which == 2) blk_solve_rows(A, ld, m, n, w.S4, n | 1, w.sc3 + 4);
    else if (which == 3) { if (n <= 16) qr_rows<16>(A, ld, m, n, w); else qr_rows<32>(A, ld, m, n, w); }
    else if (which == 4) { int k = m < n ? m : n; if (k <= 16) orgqr_rows<16>(A, ld, m, k, w); else orgqr_rows<32>(A, ld, m, k, w); }
    else if (which == 5) blk_cholqr2(A, ld, m, n, w.S1, w);
    else if (which == 6) {
      double* X = w.S2;
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) X[e] = (e % (n + 1) == 0 ? 2.0 + e * 0.001 : 0.1 / (1 + e % 7));
      __syncthreads();
      blk_jacobi(X, n, n, w.S3, nullptr, w.red, w.ptab);
    } else if (which == 7) { __syncthreads(); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / reps;
}
}  // namespace
}  // namespace prgd

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const int bytes = prgd::dense_smem_doubles() * 8;
  cudaFuncSetAttribute(prgd::k_micro, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  const char* names[] = {"gram_dmma", "chol_cta", "trinv+mul_rt", "householder_qr", "orgqr", "cholqr2", "jacobi(n x n)", "syncthreads"};
  int shapes[][2] = {{512, 32}, {256, 32}, {256, 16}};
  for (auto& sh : shapes) {
    for (int wch = 0; wch < 8; ++wch) {
      prgd::k_micro<<<1, prgd::kDenseThreads, bytes>>>(wch, sh[0], sh[1], 5, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long cyc = 0;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      printf("m=%4d n=%2d %-16s %9lld cycles  (%7.1f us @1.9GHz) %s\n", sh[0], sh[1], names[wch], cyc,
             cyc / 1900.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
