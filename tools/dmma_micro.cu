// DMMA (mma.sync m8n8k4 f64) latency / throughput micro-benchmark: cycles per
// instruction for CH independent accumulator chains per warp at W warps per
// SM (W/4 per scheduler).  Used to size the ILP the basis kernel must expose.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double c0[CH], c1[CH];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < CH; ++i) c0[i] = c1[i] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) mma884(c0[i], c1[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// dependent-chain latencies of the scalar ops of the diagonal-tile POTRF
template <int MODE>
__global__ void klat(double* out, long long* cyc, int iters) {
  double d = 1.5 + threadIdx.x;
  float f = 1.5f + threadIdx.x;
  int i = threadIdx.x;
  __shared__ double sm[64];
  sm[threadIdx.x] = d;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0) d = rsqrt(d) + 1.0;
      else if (MODE == 1) {
        double y = (double)rsqrtf((float)d);
        const double h = 0.5 * d;
        y = y * fma(-h, y * y, 1.5);
        y = y * fma(-h, y * y, 1.5);
        d = y + 1.0;
      } else if (MODE == 2) d = __shfl_sync(0xffffffffu, d, (threadIdx.x + 1) & 31);
      else if (MODE == 3) d = fma(d, 0.999, 1e-3);
      else if (MODE == 4) d = d * 0.999;
      else if (MODE == 5) f = fmaf(f, 0.999f, 1e-3f);
      else if (MODE == 6) i = i * 3 + 1;
      else if (MODE == 7) d = sm[((int)d) & 31];
      else if (MODE == 8) d = 1.0 / d;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = d + f + i;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE>
void lat(const char* nm, double* out, long long* cyc) {
  klat<MODE><<<1, 32>>>(out, cyc, 256);
  cudaDeviceSynchronize();
  klat<MODE><<<1, 32>>>(out, cyc, 256);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-24s %.1f cycles per dependent op\n", nm, c / 2048.0);
}

template <int CH>
void run(int warps, double* out, long long* cyc) {
  const int iters = 4096;
  k<CH><<<148, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<148, warps * 32>>>(out, cyc, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double n = (double)iters * CH;
  const double tf = 148.0 * warps * n * 512 / (ms * 1e-3) / 1e12;
  printf("warps/SM %2d chains %2d: %.1f cycles per DMMA per warp (%.1f per DMMA per SMSP), %.1f TFLOP/s\n", warps,
         CH, c / n, c / n / (warps / 4.0 > 1 ? warps / 4.0 : 1), tf);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 148 * 8);
  for (int w : {4, 8, 16}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<4>(w, out, cyc);
    run<8>(w, out, cyc);
    run<16>(w, out, cyc);
  }
  lat<0>("rsqrt(double)", out, cyc);
  lat<1>("rsqrtf + 2 Newton", out, cyc);
  lat<2>("shfl", out, cyc);
  lat<3>("dfma", out, cyc);
  lat<4>("dmul", out, cyc);
  lat<5>("ffma", out, cyc);
  lat<6>("imad", out, cyc);
  lat<7>("lds.64 (dep. addr)", out, cyc);
  lat<8>("1/x double", out, cyc);
  return 0;
}
