// Per-step phase timing of the bulk coarse band sweep (k_coarse_trsv_bulk) on
// a synthetic band of the config-4 single-band size (154 tile columns).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1707_07598_b200/csrc/msfv_coarse.cu"
namespace msfv {
void count_launches(long long) {}
}
using namespace msfv;
int main(int argc, char** argv) {
  const int NTa = argc > 1 ? atoi(argv[1]) : 154, PTa = argc > 2 ? atoi(argv[2]) : 10;
  const int nrhs = argc > 3 ? atoi(argv[3]) : 16;
  size_t off = 0;
  make_band(nullptr, off, NTa * 32 - 15, PTa);
  double* base;
  cudaMalloc(&base, off * 8);
  cudaMemset(base, 0, off * 8);
  off = 0;
  Band B = make_band(base, off, NTa * 32 - 15, PTa);
  const size_t nt = (size_t)B.NT * (B.PT + 1) * TT;
  std::vector<double> h(nt), hd((size_t)B.NT * TT, 0.0);
  for (size_t i = 0; i < nt; ++i) h[i] = 1e-3 * ((i * 2654435761u) % 1000) / 1000.0;
  for (int J = 0; J < B.NT; ++J)
    for (int r = 0; r < 32; ++r) hd[(size_t)J * TT + r * 33] = 0.1;
  cudaMemcpy(B.Lo, h.data(), nt * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B.Dinv, hd.data(), hd.size() * 8, cudaMemcpyHostToDevice);
  k_coarse_pack<<<(unsigned)(B.NT * (B.PT + 1)), 256>>>(B);
  double* X;
  cudaMalloc(&X, (size_t)B.n * nrhs * 8);
  cudaMemset(X, 0, (size_t)B.n * nrhs * 8);
  int cht, ns;
  size_t smem;
  trsv_bulk_shape(B.PT, cht, ns, smem);
  cudaFuncSetAttribute(k_coarse_trsv_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  SweepJobs J{};
  J.j[0] = SweepJob{B.LF, B.LB, X, B.NT, B.PT, B.n, nrhs, 0, 3};
  J.groups = (nrhs + 7) / 8;
  long long* tp;
  cudaMalloc(&tp, 64);
  cudaMemset(tp, 0, 64);
  k_coarse_trsv_bulk<<<J.groups, 256, smem>>>(J, cht, ns, nullptr);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_coarse_trsv_bulk<<<J.groups, 256, smem>>>(J, cht, ns, nullptr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  k_coarse_trsv_bulk<<<J.groups, 256, smem>>>(J, cht, ns, tp);
  cudaDeviceSynchronize();
  long long t[8];
  cudaMemcpy(t, tp, 64, cudaMemcpyDeviceToHost);
  printf("NT %d PT %d nrhs %d: solve %.3f ms (%s); per step cycles: fwd wait %lld diag %lld total %lld | bwd wait %lld total %lld\n", B.NT, B.PT, nrhs, ms,
         cudaGetErrorString(cudaGetLastError()), t[0] / B.NT, t[1] / B.NT, t[2] / B.NT, t[3] / B.NT, t[5] / B.NT);
  return 0;
}
