// grid.sync() cost with one CTA per SM (cooperative launch) and a hand-rolled
// flag barrier, to size the per-step overhead of the coarse factorization.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int n, int* dummy) {
  cg::grid_group grid = cg::this_grid();
  for (int i = 0; i < n; ++i) grid.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) dummy[0] = n;
}
// sense-reversing barrier on one counter (thread 0 of each CTA)
__global__ void k_flag(int n, unsigned* bar, int* dummy) {
  volatile unsigned* vgen = bar + 1;
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned gen = *vgen;
      __threadfence();
      if (atomicAdd(bar, 1u) == gridDim.x - 1) { bar[0] = 0; __threadfence(); atomicAdd(bar + 1, 1u); }
      else { while (*vgen == gen) { } }
      __threadfence();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) dummy[0] = n;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* d; cudaMalloc(&d, 4); unsigned* bar; cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {sms, 64, 16}) {
    int n = 1000;
    void* args[] = {&n, &d};
    cudaLaunchCooperativeKernel((void*)k_sync, grid, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_sync, grid, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    void* args2[] = {&n, &bar, &d};
    cudaLaunchCooperativeKernel((void*)k_flag, grid, 256, args2, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_flag, grid, 256, args2, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms2; cudaEventElapsedTime(&ms2, a, b);
    printf("grid %d: cg grid.sync %.3f us, flag barrier %.3f us (%s)\n", grid, ms * 1000 / n, ms2 * 1000 / n,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
