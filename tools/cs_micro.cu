// Timing of the cluster-parallel coarse sweep (k_coarse_sweep_cluster) against
// the one-CTA bulk sweep on a synthetic band: cs_micro NT PT nrhs
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1707_07598_b200/csrc/msfv_coarse.cu"
namespace msfv {
void count_launches(long long) {}
}
using namespace msfv;
int main(int argc, char** argv) {
  const int NTa = argc > 1 ? atoi(argv[1]) : 73, PTa = argc > 2 ? atoi(argv[2]) : 10;
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
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  cudaEventRecord(a);
  k_coarse_pack<<<(unsigned)(B.NT * (B.PT + 1)), 256>>>(B);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("pack %.3f ms\n", ms);
  cudaEventRecord(a);
  k_coarse_pack_scaled<<<(unsigned)(B.NT * (B.PT + 1)), 256>>>(B);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("pack_scaled %.3f ms\n", ms);
  double* X;
  cudaMalloc(&X, (size_t)B.n * nrhs * 8);
  std::vector<double> hx((size_t)B.n * nrhs);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = 1.0 + 1e-3 * (i % 7);
  long long* prof;
  cudaMalloc(&prof, 64 * 8 * 8);
  cudaMemset(prof, 0, 64 * 64);
  for (int mode = 1; mode <= 3; ++mode) {
    for (int impl = 0; impl < 2; ++impl) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemcpy(X, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
        cudaEventRecord(a);
        cudaError_t e;
        if (impl == 0) {
          SweepJobs J{};
          J.j[0] = sweep_job(B, X, nrhs, 0, mode);
          e = launch_sweeps(J, 1, nrhs, 0);
        } else {
          CsJobs J{};
          J.j[0] = cs_job(B, X, nrhs, 0, mode);
          e = launch_cluster_sweeps(J, 1, nrhs, 0);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
        best = std::min(best, ms);
      }
      std::vector<double> hy(hx.size());
      cudaMemcpy(hy.data(), X, hy.size() * 8, cudaMemcpyDeviceToHost);
      double s = 0;
      for (double v : hy) s += v;
      printf("mode %d %s: %.3f ms (%.2f us/step) checksum %.12e\n", mode, impl ? "cluster" : "bulk   ", best,
             1e3 * best / (B.NT * (mode == 3 ? 2 : 1)), s);
    }
  }
  return 0;
}
