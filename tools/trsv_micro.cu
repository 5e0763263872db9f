// Per-step phase timing of the bulk coarse solve (k_coarse_trsv_bulk) on a
// synthetic SPD band of the config-4 coarse size.
#include <cstdio>
#include <cstdlib>
#include "../paper_1707_07598_b200/csrc/msfv_coarse.cu"
namespace msfv {
void count_launches(long long) {}
}
using namespace msfv;
int main() {
  Geo g{};
  g.NT = 154; g.PT = 10; g.kc = 154 * 32 - 15; g.TB = 32;
  size_t n = coarse_doubles(g);
  double* base; cudaMalloc(&base, n * 8); cudaMemset(base, 0, n * 8);
  CoarseBufs B = coarse_bufs(g, base);
  // Dinv = 0.1 I, off-diagonal factor tiles small random
  size_t nt = band_tiles(g) * TT;
  double* h = (double*)calloc(nt, 8);
  for (size_t i = 0; i < nt; ++i) h[i] = 1e-3 * ((i * 2654435761u) % 1000) / 1000.0;
  cudaMemcpy(B.Lo, h, nt * 8, cudaMemcpyHostToDevice);
  double* hd = (double*)calloc((size_t)g.NT * TT, 8);
  for (int J = 0; J < g.NT; ++J) for (int r = 0; r < 32; ++r) hd[(size_t)J * TT + r * 33] = 0.1;
  cudaMemcpy(B.Dinv, hd, (size_t)g.NT * TT * 8, cudaMemcpyHostToDevice);
  k_coarse_pack<<<(unsigned)band_tiles(g), 256>>>(g, B.Lo, B.Dinv, B.LF, B.LB);
  const int nrhs = 16;
  double* X; cudaMalloc(&X, (size_t)g.kc * nrhs * 8); cudaMemset(X, 0, (size_t)g.kc * nrhs * 8);
  int cht, ns; size_t smem;
  trsv_bulk_shape(g, cht, ns, smem);
  cudaFuncSetAttribute(k_coarse_trsv_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long* tp; cudaMalloc(&tp, 64); cudaMemset(tp, 0, 64);
  k_coarse_trsv_bulk<<<2, 256, smem>>>(g, B.LF, B.LB, X, nrhs, cht, ns, nullptr);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_coarse_trsv_bulk<<<2, 256, smem>>>(g, B.LF, B.LB, X, nrhs, cht, ns, nullptr);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  k_coarse_trsv_bulk<<<2, 256, smem>>>(g, B.LF, B.LB, X, nrhs, cht, ns, tp);
  cudaDeviceSynchronize();
  long long t[8]; cudaMemcpy(t, tp, 64, cudaMemcpyDeviceToHost);
  printf("solve %.3f ms (%s); per step cycles: fwd wait %lld diag %lld total %lld | bwd wait %lld total %lld\n", ms,
         cudaGetErrorString(cudaGetLastError()), t[0] / g.NT, t[1] / g.NT, t[2] / g.NT, t[3] / g.NT, t[5] / g.NT);
  return 0;
}
