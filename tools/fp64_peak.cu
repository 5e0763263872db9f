// Microbenchmark: FP64 FMA pipe, FP64 DMMA (mma.sync m8n8k4) and HBM copy
// bandwidth on the box.  Prints one JSON line.  Used to fill the FP64
// roofline denominator that MEASURED_PEAKS.json does not carry.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345) out[0] = x0;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0.0; c[k][1] = 0.0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // FMA
  int iters = 4096, blocks = sms * 8, threads = 256;
  fma_kernel<<<blocks, threads>>>(d, 16, 1.0000001, 1e-9);
  double best_fma = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    if (fl / (ms * 1e-3) > best_fma) best_fma = fl / (ms * 1e-3);
  }
  // DMMA
  int diters = 4096;
  dmma_kernel<<<blocks, threads>>>(d, 16);
  double best_dmma = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(d, diters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8 * (double)diters * blocks * (threads / 32);
    if (fl / (ms * 1e-3) > best_dmma) best_dmma = fl / (ms * 1e-3);
  }
  // copy
  size_t n = (size_t)1 << 28;  // 2^28 double2 = 4 GiB each
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  copy_kernel<<<sms * 16, 512>>>(a, b, n);
  double best_bw = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 16, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double by = 2.0 * n * 16;
    if (by / (ms * 1e-3) > best_bw) best_bw = by / (ms * 1e-3);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"fp64_fma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f, \"copy_gbs\": %.1f, \"err\": \"%s\"}\n",
         sms, best_fma / 1e12, best_dmma / 1e12, best_bw / 1e9, cudaGetErrorString(err));
  return 0;
}
