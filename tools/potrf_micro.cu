// Latency microbenchmark of 8x8 Cholesky + inverse variants on one warp
// (the per-step critical chain of the basis and coarse factorizations).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq_fast(double d) {
  // float seed + two Newton steps in double (rel. error ~1e-16 after 2 steps)
  double y = (double)rsqrtf((float)d);
  double h = 0.5 * d;
  y = y * (1.5 - h * y * y);
  y = y * (1.5 - h * y * y);
  return y;
}

template <int V, int C>
__device__ __forceinline__ void step(double (&x)[8], double& invd, int r) {
  if constexpr (C < 8) {
    double d = __shfl_sync(0xffffffffu, x[C], C);
    const double inv = V == 0 ? rsqrt(d) : rsq_fast(d);
    if (r > C) x[C] *= inv;
    if (r == C) { x[C] = d * inv; invd = inv; }
    const double lrc = x[C];
#pragma unroll
    for (int q = C + 1; q < 8; ++q) {
      const double lqc = __shfl_sync(0xffffffffu, lrc, q);
      if (r >= q) x[q] -= lrc * lqc;
    }
    step<V, C + 1>(x, invd, r);
  }
}
template <int R>
__device__ __forceinline__ void inv_step(double (&d)[8], int c, const double* Ds, const double* invd) {
  if constexpr (R < 8) {
    double acc = (R == c) ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < R; ++m) acc -= Ds[R * 8 + m] * d[m];
    d[R] = (R < c) ? 0.0 : acc * invd[R];
    inv_step<R + 1>(d, c, Ds, invd);
  }
}

// V2: every lane factors and inverts the whole 8x8 block redundantly (no
// shuffles); lane 0 publishes L^{-1}.
__global__ void k2(const double* A, double* out, long long* cyc, int reps) {
  __shared__ double Ds[64], Is[72];
  const int lane = threadIdx.x;
  double2 t = reinterpret_cast<const double2*>(A)[lane];
  long long c0 = 0, c1 = 0;
  double sink = 0.0;
  for (int it = 0; it < reps; ++it) {
    long long s0 = clock64();
    *reinterpret_cast<double2*>(Ds + lane * 2) = t;
    __syncwarp();
    double a[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) a[i][j] = Ds[i * 8 + j];
    double inv[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      inv[c] = rsqrt(a[c][c]);
#pragma unroll
      for (int i = c + 1; i < 8; ++i) a[i][c] *= inv[c];
#pragma unroll
      for (int j = c + 1; j < 8; ++j)
#pragma unroll
        for (int i = j; i < 8; ++i) a[i][j] -= a[i][c] * a[j][c];
    }
    long long s1 = clock64();
    // L^{-1}: z[i][j], lower; z[i][i] = inv[i]; z[i][j] = -inv[i] sum_{k=j}^{i-1} a[i][k] z[k][j]
    double z[8][8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      z[j][j] = inv[j];
#pragma unroll
      for (int i = j + 1; i < 8; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int k = j; k < i; ++k) acc += a[i][k] * z[k][j];
        z[i][j] = -inv[i] * acc;
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) Is[i * 8 + j] = j <= i ? z[i][j] : 0.0;
    }
    __syncwarp();
    double2 li = *reinterpret_cast<double2*>(Is + lane * 2);
    __syncwarp();
    long long s2 = clock64();
    c0 += s1 - s0;
    c1 += s2 - s1;
    sink += li.x + li.y;
    t.x += sink * 1e-300;
  }
  if (lane == 0) { cyc[0] = c0 / reps; cyc[1] = c1 / reps; }
  out[lane] = sink;
}

template <int V>
__global__ void k(const double* A, double* out, long long* cyc, int reps) {
  __shared__ double Ds[64], Is[72];
  const int lane = threadIdx.x;
  double2 t = reinterpret_cast<const double2*>(A)[lane];
  long long c0 = 0, c1 = 0, c2 = 0;
  double sink = 0.0;
  for (int it = 0; it < reps; ++it) {
    long long s0 = clock64();
    *reinterpret_cast<double2*>(Ds + lane * 2) = t;
    __syncwarp();
    const int r = lane & 7;
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = Ds[r * 8 + q];
    double invd = 1.0;
    step<V, 0>(x, invd, r);
    __syncwarp();
    if (lane < 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) Ds[r * 8 + q] = x[q];
      Is[64 + r] = invd;
    }
    __syncwarp();
    long long s1 = clock64();
    if (lane < 8) {
      double d[8];
      inv_step<0>(d, lane, Ds, Is + 64);
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) Is[rr * 8 + lane] = d[rr];
    }
    __syncwarp();
    double2 li = *reinterpret_cast<double2*>(Is + lane * 2);
    __syncwarp();
    long long s2 = clock64();
    c0 += s1 - s0;
    c1 += s2 - s1;
    sink += li.x + li.y;
    t.x += sink * 1e-300;   // keep the loop honest
  }
  if (lane == 0) { cyc[0] = c0 / reps; cyc[1] = c1 / reps; }
  out[lane] = sink;
}

int main() {
  double hA[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) hA[i * 8 + j] = (i == j ? 10.0 : 1.0 / (1 + i + j));
  double *A, *out; long long* cyc;
  cudaMalloc(&A, 512); cudaMalloc(&out, 256); cudaMalloc(&cyc, 16);
  cudaMemcpy(A, hA, 512, cudaMemcpyHostToDevice);
  long long h[2];
  k<0><<<1, 32>>>(A, out, cyc, 100); cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  printf("V0 rsqrt:      factor %lld cyc, inverse %lld cyc\n", h[0], h[1]);
  k<1><<<1, 32>>>(A, out, cyc, 100); cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  printf("V1 rsqrtf+NR:  factor %lld cyc, inverse %lld cyc\n", h[0], h[1]);
  k2<<<1, 32>>>(A, out, cyc, 100); cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  printf("V2 redundant:  factor %lld cyc, inverse %lld cyc\n", h[0], h[1]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
