// Microbenchmark of the coarse factorization building blocks (per-step
#include <cstdio>
#include <cstdlib>
// latency of the panel POTRF+inverse and of one trailing-update task).
#include "../paper_1707_07598_b200/csrc/msfv_coarse.cu"
namespace msfv {
void count_launches(long long) {}
__device__ long long g_tprof[16];
__global__ void k_probe(Geo g, double* base, int* flags, int which, int reps) {
  __shared__ FactorSmem sm;
  const CoarseBufs B = coarse_bufs(g, base);
  load_tile(sm.D, B.Dinv);
  __syncthreads();
  for (int i = 0; i < reps; ++i) {
    if (which == 0) coarse_potrf(g, 0, B, flags, sm, false, g_tprof);
    else coarse_task(g, 0, which - 1, B, sm);
  }
}
}  // namespace msfv
using namespace msfv;
int main1() {
  Geo g{};
  g.NT = 154; g.PT = 10; g.kc = 154 * 32 - 15; g.TB = 32;
  size_t n = coarse_doubles(g);
  double* base; cudaMalloc(&base, n * 8);
  // SPD-ish band: identity diag tiles * 100, zero elsewhere
  double* h = (double*)calloc(n, 8);
  for (int J = 0; J < g.NT; ++J) for (int r = 0; r < 32; ++r) h[((size_t)J * (g.PT + 1)) * 1024 + r * 33] = 100.0;
  for (int J = 0; J < g.NT; ++J) for (int r = 0; r < 32; ++r) h[band_tiles(g) * 1024 + (size_t)J * 1024 + r * 33] = 0.1;
  cudaMemcpy(base, h, n * 8, cudaMemcpyHostToDevice);
  int* flags; cudaMalloc(&flags, 4); cudaMemset(flags, 0, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"potrf+inv", "pair(1,1)", "pair(2,1)"};
  for (int which = 0; which < 3; ++which) {
    int reps = 100;
    k_probe<<<1, 256>>>(g, base, flags, which, 2);
    cudaEventRecord(a);
    k_probe<<<1, 256>>>(g, base, flags, which, reps);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
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
// (appended) instrumented copy of the cooperative factor loop
namespace msfv {
__global__ void __launch_bounds__(256, 1) k_factor_timed(Geo g, double* __restrict__ base, int* __restrict__ flags,
                                                      unsigned long long* ts) {
  __shared__ FactorSmem sm;
  cg::grid_group grid = cg::this_grid();
  const CoarseBufs B = coarse_bufs(g, base);
  auto now = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
  if (blockIdx.x == 0) coarse_potrf(g, 0, B, flags, sm);
  grid.sync();
  for (int J = 0; J < g.NT; ++J) {
    unsigned long long t0 = now();
    const int pt = min(g.PT, g.NT - 1 - J);
    const int npairs = pt * (pt + 1) / 2;
    const int ntasks = npairs;
    if (blockIdx.x != 0) load_tile(sm.D, B.Dinv + (size_t)J * TT);
    __syncthreads();
    unsigned long long t1 = now(), t2 = t1, t3 = t1;
    if (blockIdx.x == 0 && pt >= 1) {
      coarse_task(g, J, 0, B, sm, true);
      t2 = now();
      coarse_potrf(g, J + 1, B, flags, sm, true);
      t3 = now();
    }
    const int first = (pt >= 1) ? 1 : 0;
    const int nw = gridDim.x > 1 ? gridDim.x - 1 : 1;
    if (gridDim.x == 1 || blockIdx.x > 0) {
      const int me = gridDim.x > 1 ? blockIdx.x - 1 : 0;
      for (int f = first + me; f < ntasks; f += nw) coarse_task(g, J, f, B, sm);
    }
    unsigned long long t4 = now();
    grid.sync();
    unsigned long long t5 = now();
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0) { ts[J * 8 + 0] = t1 - t0; ts[J * 8 + 1] = t2 - t1; ts[J * 8 + 2] = t3 - t2; ts[J * 8 + 5] = t5 - t0; }
      else atomicMax(&ts[J * 8 + 3], t4 - t0);
      if (blockIdx.x == 1) ts[J * 8 + 4] = t5 - t4;
    }
  }
}
}  // namespace msfv
int main2() {
  using namespace msfv;
  Geo g{};
  g.NT = 154; g.PT = 10; g.kc = 154 * 32 - 15; g.TB = 32;
  size_t n = coarse_doubles(g);
  double* base; cudaMalloc(&base, n * 8); cudaMemset(base, 0, n * 8);
  double* h = (double*)calloc(band_tiles(g) * 1024, 8);
  for (int J = 0; J < g.NT; ++J) for (int r = 0; r < 32; ++r) h[((size_t)J * (g.PT + 1)) * 1024 + r * 33] = 100.0;
  cudaMemcpy(base, h, band_tiles(g) * 1024 * 8, cudaMemcpyHostToDevice);
  int* flags; cudaMalloc(&flags, 4); cudaMemset(flags, 0, 4);
  unsigned long long* ts; cudaMalloc(&ts, 154 * 8 * 8); cudaMemset(ts, 0, 154 * 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* args[] = {&g, &base, &flags, &ts};
  cudaLaunchCooperativeKernel((void*)k_factor_timed, sms, 256, args, 0, 0);
  cudaDeviceSynchronize();
  unsigned long long hts[154 * 8];
  cudaMemcpy(hts, ts, sizeof(hts), cudaMemcpyDeviceToHost);
  double s[6] = {0};
  for (int J = 0; J < 154; ++J) for (int q = 0; q < 6; ++q) s[q] += hts[J * 8 + q];
  printf("per step avg (us): loadD %.2f task0 %.2f potrf %.2f maxworker %.2f barrier(cta1) %.2f total(cta0) %.2f  err %s\n",
         s[0] / 154e3, s[1] / 154e3, s[2] / 154e3, s[3] / 154e3, s[4] / 154e3, s[5] / 154e3,
         cudaGetErrorString(cudaGetLastError()));
  for (int J : {0, 50, 100, 150}) printf("  J=%d: %llu %llu %llu %llu %llu %llu\n", J, hts[J*8], hts[J*8+1], hts[J*8+2], hts[J*8+3], hts[J*8+4], hts[J*8+5]);
  return 0;
}
int main() { main1(); return main2(); }
