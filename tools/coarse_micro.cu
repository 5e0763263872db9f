// Microbenchmark of the coarse factorization building blocks: per-call
// latency of the blocked diagonal POTRF + inverse (with a phase breakdown) and
// of one trailing-update task, on a synthetic SPD band of the config-4 size.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1707_07598_b200/csrc/msfv_coarse.cu"
namespace msfv {
void count_launches(long long) {}
__device__ long long g_tprof[16];
__global__ void k_probe(Band B, int* flags, int which, int reps) {
  __shared__ FactorSmem sm;
  load_tile(sm.D, B.Dinv);
  __syncthreads();
  for (int i = 0; i < reps; ++i) {
    if (which == 0) coarse_potrf(B, 0, flags, sm, false, g_tprof);
    else coarse_task(B, 0, which - 1, sm);
  }
}
}  // namespace msfv
using namespace msfv;
int main() {
  size_t off = 0;
  Band probe = make_band(nullptr, off, 154 * 32 - 15, 10);
  double* base;
  cudaMalloc(&base, off * 8);
  cudaMemset(base, 0, off * 8);
  off = 0;
  Band B = make_band(base, off, 154 * 32 - 15, 10);
  (void)probe;
  // SPD-ish band: 100 I on the diagonal tiles, Dinv = 0.1 I
  std::vector<double> h((size_t)B.NT * (B.PT + 1) * TT, 0.0), hd((size_t)B.NT * TT, 0.0);
  for (int J = 0; J < B.NT; ++J)
    for (int r = 0; r < 32; ++r) {
      h[((size_t)J * (B.PT + 1)) * TT + r * 33] = 100.0;
      hd[(size_t)J * TT + r * 33] = 0.1;
    }
  cudaMemcpy(B.A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B.Dinv, hd.data(), hd.size() * 8, cudaMemcpyHostToDevice);
  int* flags;
  cudaMalloc(&flags, 4);
  cudaMemset(flags, 0, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"potrf+inv", "pair(1,1)", "pair(2,1)"};
  for (int which = 0; which < 3; ++which) {
    const int reps = 100;
    k_probe<<<1, 256>>>(B, flags, which, 2);
    cudaEventRecord(a);
    k_probe<<<1, 256>>>(B, flags, which, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-10s %.3f us per call (%s)\n", names[which], ms * 1000 / reps, cudaGetErrorString(cudaGetLastError()));
    if (which == 0) {
      long long tp[16];
      cudaMemcpyFromSymbol(tp, g_tprof, sizeof(tp));
      printf("  potrf phases (cycles, avg):");
      for (int k = 1; k <= 14; ++k) printf(" %lld", (tp[k] - tp[k - 1]) / (reps + 2));
      printf("\n");
    }
  }
  return 0;
}
