// Microbenchmark (diagnostic): register-resident one-warp Cholesky + inverse of a 32 x 32 SPD
// matrix versus the blocked CTA version of the cluster rounding.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double frsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y * y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x, y * y, 1.0);
  return fma(0.5 * y, e, y);
}

// lane i holds row i of G (n = 32); on return g = row i of L, rinv = 1/L_ii; Li (smem,
// stride 33) = L^{-1} (column c computed by lane c).
__device__ __noinline__ bool warp_chol32(const double* G, double* Lsm, double* Li) {
  const int lane = threadIdx.x & 31;
  double g[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) g[c] = G[lane * 33 + c];
  bool ok = true;
  double rmine = 1.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double piv = __shfl_sync(0xffffffffu, g[j], j);
    ok = ok && piv > 0.0;
    const double rs = frsqrt(piv);
    const double lij = g[j] * rs;
    g[j] = lij;
    if (lane == j) rmine = rs;
#pragma unroll
    for (int k = j + 1; k < 32; ++k) g[k] = fma(-lij, __shfl_sync(0xffffffffu, lij, k), g[k]);
  }
  // store L to smem (row lane), then column-wise inverse from smem broadcasts
#pragma unroll
  for (int c = 0; c < 32; ++c) Lsm[lane * 33 + c] = c <= lane ? g[c] : 0.0;
  __syncwarp();
  double s[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) s[i] = (i == lane) ? 1.0 : 0.0;
  const double rl[1] = {rmine};
  (void)rl;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double rk = __shfl_sync(0xffffffffu, rmine, k);
    const double xk = s[k] * rk;
    s[k] = xk;
#pragma unroll
    for (int i = k + 1; i < 32; ++i) s[i] = fma(-Lsm[i * 33 + k], xk, s[i]);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) Li[i * 33 + lane] = s[i];
  return __all_sync(0xffffffffu, ok);
}

__global__ void k(long long* cyc, double* out) {
  __shared__ double G[32 * 33], L[32 * 33], Li[32 * 33];
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    int i = e / 32, j = e % 32;
    G[i * 33 + j] = (i == j ? 33.0 : 0.0) + 1.0 / (1.0 + i + j);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    bool ok = true;
    long long t0 = clock64();
    for (int rep = 0; rep < 10; ++rep) ok = warp_chol32(G, L, Li) && ok;
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 10; out[0] = Li[31 * 33] + (ok ? 0 : 1); }
  }
  __syncthreads();
  // check: L * Li = I
  if (threadIdx.x == 0) {
    double err = 0;
    for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) {
      double s = 0; for (int k = 0; k < 32; ++k) s += L[i * 33 + k] * Li[k * 33 + j];
      err = fmax(err, fabs(s - (i == j)));
    }
    out[1] = err;
  }
}

int main() {
  long long* c; double* o;
  cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 64);
  k<<<1, 256>>>(c, o);
  cudaDeviceSynchronize();
  printf("warp register chol+inv 32: %lld cycles, |L Li - I| = %.2e (%s)\n", c[0], o[1], cudaGetErrorString(cudaGetLastError()));
}
