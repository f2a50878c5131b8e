// Microbenchmark (diagnostic): Cholesky + triangular inverse of a 32 x 32 SPD Gram in shared
// memory: the blocked CTA version of the cluster rounding vs a one-warp shared-memory version
// (row per lane, dynamic loops, one pivot broadcast per column).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ll = 33, li = 36, LX = 33;

__device__ __forceinline__ double frsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y * y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x, y * y, 1.0);
  return fma(0.5 * y, e, y);
}

// ---------------- current blocked CTA version (copy of cl_chol) ----------------
__device__ __noinline__ bool chol8_thread(double* B, int ld, int m, double* Bi, int ldi, double* rinv) {
  __builtin_assume(__isShared(B)); __builtin_assume(__isShared(Bi)); __builtin_assume(__isShared(rinv));
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c <= i; ++c) a[i][c] = (i < m && c < m) ? B[i * ld + c] : (i == c ? 1.0 : 0.0);
  bool ok = true; double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double d = a[j][j]; const bool good = d > 0.0 && d < 1.0e300; ok = ok && good;
    const double rs = good ? frsqrt(d) : 1.0; r[j] = rs; a[j][j] = d * rs;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) a[i][j] *= rs;
#pragma unroll
    for (int i = j + 1; i < 8; ++i)
#pragma unroll
      for (int k = j + 1; k <= i; ++k) a[i][k] = fma(-a[i][j], a[k][j], a[i][k]);
  }
  double x[8][8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    x[c][c] = r[c];
#pragma unroll
    for (int i = c + 1; i < 8; ++i) { double s = 0.0;
#pragma unroll
      for (int k = c; k < i; ++k) s = fma(-a[i][k], x[k][c], s);
      x[i][c] = s * r[i]; }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) if (i < m) { rinv[i] = r[i];
#pragma unroll
      for (int c = 0; c < 8; ++c) if (c < m) { B[i * ld + c] = c <= i ? a[i][c] : 0.0; Bi[i * ldi + c] = c <= i ? x[i][c] : 0.0; } }
  return ok;
}
__device__ __noinline__ bool blk_chol(const double* G, double* Lo, double* LI, double* rinv, int* flag, double* Tb, int n, double shift) {
  const int tid = threadIdx.x, T = blockDim.x;
  for (int e = tid; e < n * n; e += T) { const int i = e / n, c = e - i * n;
    Lo[i * ll + c] = c <= i ? G[i * ll + c] + (c == i ? shift : 0.0) : 0.0; LI[i * li + c] = 0.0; }
  if (tid == 0) *flag = 1;
  __syncthreads();
  const int nb = (n + 7) >> 3;
  for (int b = 0; b < nb; ++b) {
    const int b0 = 8 * b, m = min(8, n - b0);
    if (tid == 0) { if (!chol8_thread(Lo + b0 * ll + b0, ll, m, LI + b0 * li + b0, li, rinv + b0)) *flag = 0; }
    __syncthreads();
    const int r0 = b0 + m;
    for (int r = r0 + tid; r < n; r += T) { double g[8];
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) g[qq] = qq < m ? Lo[r * ll + b0 + qq] : 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) if (c < m) { double acc = 0.0;
#pragma unroll
          for (int qq = 0; qq <= c; ++qq) acc = fma(g[qq], LI[(b0 + c) * li + b0 + qq], acc);
          Lo[r * ll + b0 + c] = acc; } }
    __syncthreads();
    const int sz = n - r0;
    for (int e = tid; e < sz * sz; e += T) { const int i = r0 + e / sz, k = r0 + (e - (e / sz) * sz);
      if (k <= i) { double acc = Lo[i * ll + k];
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) if (qq < m) acc = fma(-Lo[i * ll + b0 + qq], Lo[k * ll + b0 + qq], acc);
        Lo[i * ll + k] = acc; } }
    __syncthreads();
  }
  for (int I = 1; I < nb; ++I) { const int i0 = 8 * I, mi = min(8, n - i0);
    for (int e = tid; e < mi * i0; e += T) { const int r = e / i0, c = e - r * i0; double acc = 0.0;
      for (int k = c; k < i0; ++k) acc = fma(Lo[(i0 + r) * ll + k], LI[k * li + c], acc);
      Tb[c * 9 + r] = acc; }
    __syncthreads();
    for (int e = tid; e < mi * i0; e += T) { const int r = e / i0, c = e - r * i0; double acc = 0.0;
      for (int qq = 0; qq <= r; ++qq) acc = fma(LI[(i0 + r) * li + i0 + qq], Tb[c * 9 + qq], acc);
      LI[(i0 + r) * li + c] = -acc; }
    __syncthreads();
  }
  __syncthreads();
  return *flag != 0;
}

// ---------------- one-warp shared-memory factor ----------------
// lane i owns row i; column j's entries are broadcast through Cb (double-buffered).
__device__ __noinline__ bool w_fac(const double* G, double* Lo, double* rinv, double* Cb, int n, double shift) {
  __builtin_assume(__isShared(G)); __builtin_assume(__isShared(Lo)); __builtin_assume(__isShared(rinv)); __builtin_assume(__isShared(Cb));
  const int lane = threadIdx.x & 31;
  double dg = 1.0, nxt = 0.0;
  if (lane < n) {
    for (int c = 0; c < n; ++c) Lo[lane * ll + c] = c <= lane ? G[lane * ll + c] : 0.0;
    dg = G[lane * ll + lane] + shift;
    nxt = G[lane * ll];
  }
  bool okme = true;
  for (int j = 0; j < n; ++j) {
    const double myr = frsqrt(dg);
    const double rs = __shfl_sync(0xffffffffu, myr, j);
    double* C = Cb + (j & 1) * 32;
    double l = 0.0;
    if (lane == j) { okme = dg > 0.0 && dg < 1.0e300; rinv[j] = rs; Lo[j * ll + j] = dg * rs; }
    if (lane > j && lane < n) { l = nxt * rs; Lo[lane * ll + j] = l; C[lane] = l; dg = fma(-l, l, dg); }
    __syncwarp();
    if (lane > j + 1 && lane < n) {
      nxt = fma(-l, C[j + 1], Lo[lane * ll + j + 1]);
      double* row = Lo + lane * ll;
      int k = j + 2;
      for (; k + 3 < lane; k += 4) {
        const double c0 = C[k], c1 = C[k + 1], c2 = C[k + 2], c3 = C[k + 3];
        const double r0 = row[k], r1 = row[k + 1], r2 = row[k + 2], r3 = row[k + 3];
        row[k] = fma(-l, c0, r0); row[k + 1] = fma(-l, c1, r1); row[k + 2] = fma(-l, c2, r2); row[k + 3] = fma(-l, c3, r3);
      }
      for (; k < lane; ++k) row[k] = fma(-l, C[k], row[k]);
    }
  }
  __syncwarp();
  return __all_sync(0xffffffffu, okme);
}
// one-warp inverse: lane c builds column c of X = L^{-1} (XT row c), lockstep over k.
__device__ __noinline__ void w_inv(const double* Lo, const double* rinv, double* XT, double* LI, int n) {
  __builtin_assume(__isShared(Lo)); __builtin_assume(__isShared(rinv)); __builtin_assume(__isShared(XT)); __builtin_assume(__isShared(LI));
  const int c = threadIdx.x & 31;
  if (c < n) for (int i = 0; i < n; ++i) XT[c * LX + i] = i == c ? 1.0 : 0.0;
  for (int k = 0; k < n; ++k) {
    if (c <= k && c < n) {
      const double xk = XT[c * LX + k] * rinv[k];
      XT[c * LX + k] = xk;
      double* xr = XT + c * LX;
      int i = k + 1;
      for (; i + 3 < n; i += 4) {
        const double l0 = Lo[i * ll + k], l1 = Lo[(i + 1) * ll + k], l2 = Lo[(i + 2) * ll + k], l3 = Lo[(i + 3) * ll + k];
        const double x0 = xr[i], x1 = xr[i + 1], x2 = xr[i + 2], x3 = xr[i + 3];
        xr[i] = fma(-l0, xk, x0); xr[i + 1] = fma(-l1, xk, x1); xr[i + 2] = fma(-l2, xk, x2); xr[i + 3] = fma(-l3, xk, x3);
      }
      for (; i < n; ++i) xr[i] = fma(-Lo[i * ll + k], xk, xr[i]);
    }
  }
  __syncwarp();
  if (c < n) for (int i = 0; i < n; ++i) LI[i * li + c] = i >= c ? XT[c * LX + i] : 0.0;
  __syncwarp();
}


// ---------------- one-warp register fraction-free Cholesky (power-of-two scaled) ----------------
// lane i holds row i of (G + shift I) (identity padded to NM).  Step j eliminates with
//   a_i[k] <- (P_j a_i[k] - a_i[j] a_k[j]) * 2^-e(P_j)     (P_j = current pivot a_j[j])
// so the pivot recursion has no division / square root on its dependency chain; the rows hold
// sigma_{j-1} x the Schur complement (sigma_j = sigma_{j-1} P_j 2^-e(P_j) in [1, 2^j)), and
// L_ij = a_i[j] / sqrt(sigma_{j-1} P_j).  Column entries a_k[j] (k > j+1) are broadcast through
// shared memory, a_{j+1}[j] by a shuffle.  Then X = L^{-1}: lane c forms column c (right-looking).
__device__ __forceinline__ double pow2_inv_exp(double p) {
  // 2^-e with e the unbiased exponent of p (p normal, > 0): exact power of two
  const int hi = __double2hiint(p);
  const int be = (hi >> 20) & 0x7ff;              // biased exponent
  return __hiloint2double((2046 - be) << 20, 0);  // biased exponent of 2^-(be-1023) is 2046-be
}
__device__ long long dbg[4];
template <int NM>
__device__ __noinline__ bool ff_chol(const double* G, double* Lo, double* LI, double* rinv, double* cb, double* LT, int n, double shift) {
  __builtin_assume(__isShared(G)); __builtin_assume(__isShared(Lo)); __builtin_assume(__isShared(LI));
  __builtin_assume(__isShared(rinv)); __builtin_assume(__isShared(cb)); __builtin_assume(__isShared(LT));
  constexpr int ldt = NM + 2;
  const int lane = threadIdx.x & 31;
  double a[NM];
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    double v = (lane < n && k < n) ? G[lane * ll + k] : (lane == k ? 1.0 : 0.0);
    if (k == lane && lane < n) v += shift;
    a[k] = v;
  }
  bool ok = true;
  double sig = 1.0, rme = 1.0;
  long long q0 = clock64();
#pragma unroll
  for (int j = 0; j < NM; ++j) {
    const double P = __shfl_sync(0xffffffffu, a[j], j);
    ok = ok && P > 0.0 && P < 1.0e300;
    const double s = pow2_inv_exp(P);
    const double t = frsqrt(sig * P);
    if (lane == j) rme = sig * t;
    if (j + 1 < NM) {
      double* C = cb + (j & 1) * NM;
      C[lane] = a[j];
      const double c1 = __shfl_sync(0xffffffffu, a[j], j + 1);
      __syncwarp();
      const double b = a[j] * s, Ps = P * s;
      a[j + 1] = fma(-b, c1, Ps * a[j + 1]);
      if ((j + 2) & 1) { if (j + 2 < NM) a[j + 2] = fma(-b, C[j + 2], Ps * a[j + 2]); }
#pragma unroll
      for (int k = ((j + 2) & 1) ? j + 3 : j + 2; k < NM; k += 2) {
        if (k + 1 < NM) {
          const double2 c = *reinterpret_cast<const double2*>(C + k);
          a[k] = fma(-b, c.x, Ps * a[k]);
          a[k + 1] = fma(-b, c.y, Ps * a[k + 1]);
        } else {
          a[k] = fma(-b, C[k], Ps * a[k]);
        }
      }
      sig = sig * Ps;
    }
    a[j] = a[j] * t;   // column j of L (rows >= j; rows < j hold upper garbage)
  }
  long long q1 = clock64();
  // L rows to Lo and transposed to LT
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    const double v = k <= lane ? a[k] : 0.0;
    if (lane < n && k < n) Lo[lane * ll + k] = v;
    LT[k * ldt + lane] = v;
  }
  rinv[lane] = rme;
  __syncwarp();
  long long q2 = clock64();
  if (lane == 0) { dbg[0] = q1 - q0; dbg[1] = q2 - q1; }
  return __all_sync(0xffffffffu, ok);
}
template <int NM>
__device__ __noinline__ void ff_inv(double* LI, const double* rinv, const double* LT, int n) {
  __builtin_assume(__isShared(LI)); __builtin_assume(__isShared(rinv)); __builtin_assume(__isShared(LT));
  constexpr int ldt = NM + 2;
  const int lane = threadIdx.x & 31;
  long long q2 = clock64();
  // inverse: lane c, x_k = (delta_kc - sum_{q<k} L_kq x_q) / L_kk, right-looking accumulation
  double sacc[NM];
#pragma unroll
  for (int i = 0; i < NM; ++i) sacc[i] = 0.0;
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    const double rk = rinv[k];
    const double xk = (k == lane ? 1.0 - sacc[k] : -sacc[k]) * rk;   // sacc[k] = 0 for k < lane
    sacc[k] = k >= lane ? xk : 0.0;
    if ((k + 1) & 1) { if (k + 1 < NM) sacc[k + 1] = fma(LT[k * ldt + k + 1], xk, sacc[k + 1]); }
#pragma unroll
    for (int i = ((k + 1) & 1) ? k + 2 : k + 1; i < NM; i += 2) {
      if (i + 1 < NM) {
        const double2 l = *reinterpret_cast<const double2*>(LT + k * ldt + i);
        sacc[i] = fma(l.x, xk, sacc[i]);
        sacc[i + 1] = fma(l.y, xk, sacc[i + 1]);
      } else {
        sacc[i] = fma(LT[k * ldt + i], xk, sacc[i]);
      }
    }
  }
  if (lane < n) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      if (i < n) LI[i * li + lane] = sacc[i];
  }
  __syncwarp();
  long long q3 = clock64();
  if (lane == 0) { dbg[2] = q3 - q2; }
}

__global__ void k(long long* cyc, double* out, int n) {
  __shared__ double A[40 * 33], G[32 * ll], Lo[32 * ll], LI[32 * li], rinv[32], Cb[64], XT[32 * LX], Tb[32 * 9];
  double* LTs = A;
  __shared__ int flag;
  for (int e = threadIdx.x; e < 40 * 32; e += blockDim.x) {
    int i = e / 32, c = e % 32;
    unsigned x = (unsigned)(e * 2654435761u) ^ 0x9e3779b9u; x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12;
    A[i * 33 + c] = ((double)(x & 0xffffff) / 16777216.0 - 0.5) * exp2(-0.4 * c);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e / n, j = e % n; double s = 0;
    for (int r = 0; r < 40; ++r) s += A[r * 33 + i] * A[r * 33 + j];
    G[i * ll + j] = s;
  }
  __syncthreads();
  const double shift = 1e-14 * G[0];
  for (int variant = 0; variant < 3; ++variant) {
    long long t0 = 0, t1 = 0; bool ok = true;
    for (int rep = 0; rep < 11; ++rep) {
      __syncthreads();
      if (rep == 1) t0 = clock64();
      if (variant == 0) ok = blk_chol(G, Lo, LI, rinv, &flag, Tb, n, shift);
      else if (variant == 2) {
        if (threadIdx.x < 32) { long long a0 = clock64(); bool o = ff_chol<32>(G, Lo, LI, rinv, Cb, LTs, n, shift); ff_inv<32>(LI, rinv, LTs, n); long long a1 = clock64();
          if (threadIdx.x == 0) { flag = o; cyc[4] = a1 - a0; cyc[5] = dbg[0]; cyc[6] = dbg[1]; cyc[7] = dbg[2]; } }
        __syncthreads();
        ok = flag;
      } else {
        if (threadIdx.x < 32) { long long a0 = clock64(); bool o = w_fac(G, Lo, rinv, Cb, n, shift); long long a1 = clock64(); w_inv(Lo, rinv, XT, LI, n);
          long long a2 = clock64(); if (threadIdx.x == 0) { flag = o; cyc[2] = a1 - a0; cyc[3] = a2 - a1; } }
        __syncthreads();
        ok = flag;
      }
    }
    __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) {
      double e1 = 0, e2 = 0, gn = 0;
      for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
        double s = 0, t = 0;
        for (int q = 0; q < n; ++q) { s += Lo[i * ll + q] * Lo[j * ll + q]; t += Lo[i * ll + q] * LI[q * li + j]; }
        e1 = fmax(e1, fabs(s - G[i * ll + j] - (i == j ? shift : 0))); e2 = fmax(e2, fabs(t - (i == j)));
        gn = fmax(gn, fabs(G[i * ll + j]));
        if (j > i && (Lo[i * ll + j] != 0 || LI[i * li + j] != 0)) e2 = 1e9;
      }
      cyc[variant] = (t1 - t0) / 10; out[2 * variant] = e1 / gn; out[2 * variant + 1] = e2 + (ok ? 0 : 1);
    }
    __syncthreads();
  }
}

int main() {
  long long* c; double* o;
  cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
  for (int n : {32, 24, 16}) {
    k<<<1, 256>>>(c, o, n);
    cudaDeviceSynchronize();
    printf("fac %lld inv %lld | n=%d blocked: %lld cyc |LL^T-G|/|G| %.2e |LX-I| %.2e   warp-smem: %lld cyc %.2e %.2e | ff-reg: %lld (%lld) cyc %.2e %.2e [fac %lld st %lld inv %lld] (%s)\n", c[2], c[3], n, c[0], o[0], o[1], c[1], o[2], o[3], c[2+0*0], c[4], o[4], o[5], c[5], c[6], c[7],
           cudaGetErrorString(cudaGetLastError()));
  }
}
