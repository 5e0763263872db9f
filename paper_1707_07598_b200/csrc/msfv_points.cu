// Survey point sets: products of the sparse receiver matrix P and source
// matrix Q (pinned node space, forward.py:23-51) with the basis S.
//
//   receive   out[col][s] = sum_{t in col} val_t (Xf(node_t,s) + S(node_t,:) Y[:,s])
//             D = P^T S T (forward.py:143), J v = P^T (ydm + S dt) (forward.py:268)
//   restrict  out[c][s]   = sum_{(t,cc) -> c} val_t S(node_t,cc) Z[col_t][s]
//             F = S^T Q (forward.py:115), S^T P W (forward.py:275-276)
//   scatter   field(node,s) = sum_{t at node} val_t Z[col_t][s]   (dense Q / P W)
// Every output element is one thread summing a host-sorted list, so results are
// deterministic.
#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace msfv {

__device__ __forceinline__ void decode_loc(int packed, int& x, int& y, int& z) {
  x = packed & 1023; y = (packed >> 10) & 1023; z = (packed >> 20) & 1023;
}

__device__ __forceinline__ double point_s(const Geo& g, const PointsDev& P, const double* Sint, long long t, int cc,
                                          int& corner) {
  int jb = P.blk[t];
  int x, y, z;
  decode_loc(P.loc[t], x, y, z);
  int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  corner = corner_col(g, bi, bj, bk, cc);
  return s_value(g, Sint + (size_t)jb * 8 * g.nI, jb, cc, x, y, z, false);
}

__global__ void k_points_receive(Geo g, PointsDev P, const double* __restrict__ Sint, const double* __restrict__ Y,
                                 const double* __restrict__ Xf, int nrhs, double* __restrict__ out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)P.ncol * nrhs) return;
  int s = (int)(i % nrhs), col = (int)(i / nrhs);
  double v = 0.0;
  for (long long t = P.colptr[col]; t < P.colptr[col + 1]; ++t) {
    double u = 0.0;
    if (Xf) u += Xf[P.node[t] * nrhs + s];
    if (Y) {
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        int corner;
        double sv = point_s(g, P, Sint, t, cc, corner);
        u += sv * Y[(size_t)corner * nrhs + s];
      }
    }
    v += P.val[t] * u;
  }
  out[i] = v;
}

__global__ void k_points_restrict(Geo g, PointsDev P, const double* __restrict__ Sint, const double* __restrict__ Z,
                                  int nrhs, double* __restrict__ out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)g.kc * nrhs) return;
  int s = (int)(i % nrhs), c = (int)(i / nrhs);
  double v = 0.0;
  for (long long e = P.cptr[c]; e < P.cptr[c + 1]; ++e) {
    long long packed = P.cent[e];
    long long t = packed >> 3;
    int cc = (int)(packed & 7);
    int col = P.col[t];
    double z = Z ? Z[(size_t)col * nrhs + s] : (col == s ? 1.0 : 0.0);
    if (z == 0.0) continue;
    int corner;
    double sv = point_s(g, P, Sint, t, cc, corner);
    v += P.val[t] * sv * z;
  }
  out[i] = v;
}

// Warp per coarse node: the lanes evaluate 32 entries' point factors
// val_t S(node_t, cc) and columns at once (the dependent index loads of
// different entries overlap), then each lane sums its right-hand sides over
// the staged entries in entry order: the same products and summation order as
// k_points_restrict.
constexpr int PR_WARPS = 4;
__global__ void __launch_bounds__(32 * PR_WARPS) k_points_restrict_w(Geo g, PointsDev P, const double* __restrict__ Sint,
                                                                  const double* __restrict__ Z, int nrhs,
                                                                  double* __restrict__ out) {
  __shared__ double pe[PR_WARPS][32];
  __shared__ int ce[PR_WARPS][32];
  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  const int c = blockIdx.x * PR_WARPS + wv;
  if (c >= g.kc) return;
  const long long e0 = P.cptr[c], e1 = P.cptr[c + 1];
  double acc[2] = {0.0, 0.0};                   // s = lane, lane + 32 (nrhs <= 64)
  for (long long eb = e0; eb < e1; eb += 32) {
    const int cnt = (int)min((long long)32, e1 - eb);
    if (lane < cnt) {
      const long long packed = P.cent[eb + lane];
      const long long t = packed >> 3;
      int corner;
      const double sv = point_s(g, P, Sint, t, (int)(packed & 7), corner);
      pe[wv][lane] = P.val[t] * sv;
      ce[wv][lane] = P.col[t];
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sidx = lane + 32 * h;
      if (sidx >= nrhs) continue;
      double v = acc[h];
      for (int j = 0; j < cnt; ++j) {
        const int col = ce[wv][j];
        const double z = Z ? Z[(size_t)col * nrhs + sidx] : (col == sidx ? 1.0 : 0.0);
        if (z != 0.0) v += pe[wv][j] * z;
      }
      acc[h] = v;
    }
    __syncwarp();
  }
  for (int h = 0; h < 2; ++h) {
    const int sidx = lane + 32 * h;
    if (sidx < nrhs) out[(size_t)c * nrhs + sidx] = acc[h];
  }
}

__global__ void k_points_scatter(Geo g, PointsDev P, const double* __restrict__ Z, int nrhs, double* __restrict__ field) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.nu * nrhs) return;
  int s = (int)(i % nrhs);
  long long u = i / nrhs;
  double v = 0.0;
  for (long long e = P.uptr[u]; e < P.uptr[u + 1]; ++e) {
    long long t = P.uent[e];
    int col = P.col[t];
    double z = Z ? Z[(size_t)col * nrhs + s] : (col == s ? 1.0 : 0.0);
    v += P.val[t] * z;
  }
  field[P.unode[u] * nrhs + s] = v;
}

// rhs_c[urow(node)][s] = sum_{t at node} val_t Z[col_t][s] for the interior nodes
__global__ void k_points_scatter_interior(Geo g, PointsDev P, const double* __restrict__ Z, int nrhs,
                                          double* __restrict__ rhs_c) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.nu * nrhs) return;
  int s = (int)(i % nrhs);
  long long u = i / nrhs;
  const long long row = P.urow[u];
  if (row < 0) return;
  double v = 0.0;
  for (long long e = P.uptr[u]; e < P.uptr[u + 1]; ++e) {
    long long t = P.uent[e];
    int col = P.col[t];
    double z = Z ? Z[(size_t)col * nrhs + s] : (col == s ? 1.0 : 0.0);
    v += P.val[t] * z;
  }
  rhs_c[row * nrhs + s] = v;
}

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_points_receive(const Geo& g, const PointsDev& P, const double* Sint, const double* Y,
                                  const double* Xf, int nrhs, double* out, cudaStream_t st) {
  long long tot = (long long)P.ncol * nrhs;
  if (tot == 0) return cudaSuccess;
  k_points_receive<<<nblk(tot, 128), 128, 0, st>>>(g, P, Sint, Y, Xf, nrhs, out);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_points_restrict(const Geo& g, const PointsDev& P, const double* Sint, const double* Z,
                                   int nrhs, double* out, cudaStream_t st) {
  long long tot = (long long)g.kc * nrhs;
  if (tot == 0) return cudaSuccess;
  if (nrhs <= 64)
    k_points_restrict_w<<<nblk(g.kc, PR_WARPS), 32 * PR_WARPS, 0, st>>>(g, P, Sint, Z, nrhs, out);
  else
    k_points_restrict<<<nblk(tot, 128), 128, 0, st>>>(g, P, Sint, Z, nrhs, out);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_points_scatter(const Geo& g, const PointsDev& P, const double* Z, int nrhs, double* field,
                                  cudaStream_t st) {
  long long tot = P.nu * nrhs;
  if (tot == 0) return cudaSuccess;
  k_points_scatter<<<nblk(tot, 128), 128, 0, st>>>(g, P, Z, nrhs, field);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_points_scatter_interior(const Geo& g, const PointsDev& P, const double* Z, int nrhs, double* rhs_c,
                                           cudaStream_t st) {
  if (P.nib == 0 || nrhs == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(rhs_c, 0, (size_t)P.nib * g.nI * nrhs * sizeof(double), st);
  if (e != cudaSuccess) return e;
  k_points_scatter_interior<<<nblk(P.nu * nrhs, 128), 128, 0, st>>>(g, P, Z, nrhs, rhs_c);
  count_launches(1);
  return cudaGetLastError();
}

// misfit_ssd on the device (inversion.py:22-29): resid = D - D_obs and phi = 0.5 sum resid^2 in one
// launch.  One CTA; every thread sums its strided elements in index order, the 512 partial sums are
// combined by a fixed tree: the value is reproducible bit for bit.
constexpr int MISFIT_THREADS = 512;
__global__ void __launch_bounds__(MISFIT_THREADS) k_misfit(const double* __restrict__ D, const double* __restrict__ Dobs,
                                                           long long n, double* __restrict__ resid,
                                                           double* __restrict__ phi) {
  __shared__ double part[MISFIT_THREADS];
  double a = 0.0;
  for (long long i = threadIdx.x; i < n; i += MISFIT_THREADS) {
    const double r = D[i] - Dobs[i];
    resid[i] = r;
    a = fma(r, r, a);
  }
  part[threadIdx.x] = a;
  __syncthreads();
  for (int s = MISFIT_THREADS / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) phi[0] = 0.5 * part[0];
}
cudaError_t launch_misfit(const double* D, const double* Dobs, long long n, double* resid, double* phi,
                          cudaStream_t st) {
  k_misfit<<<1, MISFIT_THREADS, 0, st>>>(D, Dobs, n, resid, phi);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
