// Fused per-block gradient of the adaptive rapply (forward.py:270-281):
//
//   g_c  = -sigma_c (V/4) sum_{e in c} xi_e                     (-Csig^T xi)
//   xi_e = sum_s [dU_s (dZ_s + dY_s) + dR_s dY_s] / h_e^2       (d = difference along e)
//
// with U = S T (forward fields), Y = S y (adjoint coarse solution y),
// Z = A_II^{-1}(p - A S y)_I and R = A_II^{-1}(q - A S T)_I.  The Lagrange
// columns solve their local problems, (A S)_I = 0 (basis.py:548), so
// Z = A_II^{-1} p_I and R = A_II^{-1} q_I: both vanish outside the few blocks
// whose interiors hold receiver / source nodes (compact per-block fields of
// the survey's interior slots, msfv_points_interior_solve).  Everywhere else
//   sum_s dU_s dY_s = dS_e^T M_j dS_e,   M_j = T_j y_j^T  (8 x 8 per block),
// where dS_e is the difference of the block's 8 basis columns along e.  One
// CTA per block: the block's closure basis values are staged in shared
// memory (interior from Sint, skeleton from the hats), xi is formed for the
// closure edges and the block's own cells gather their 12 edges, so the
// gradient is one pass over Sint with no node-field traffic.
#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace msfv {

size_t grad_smem_doubles(const Geo& g, int nrhs) {
  const size_t B1 = g.b1 + 1, B2 = g.b2 + 1, B3 = g.b3 + 1;
  const size_t ne = (size_t)g.b1 * B2 * B3 + B1 * g.b2 * B3 + B1 * B2 * g.b3;
  return B1 * B2 * B3 * 8 + ne + 16 * (size_t)nrhs + 64;
}

__global__ void __launch_bounds__(GRAD_THREADS)
k_grad_block(Geo g, const double* __restrict__ Sint, const double* __restrict__ T, const double* __restrict__ Y,
             int nrhs, const double* __restrict__ sigma, const int* __restrict__ zslot, const double* __restrict__ Zc,
             const int* __restrict__ rslot, const double* __restrict__ Rc, double* __restrict__ gout) {
  extern __shared__ __align__(16) double gsm[];
  const int jb = blockIdx.x, tid = threadIdx.x;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int B1 = g.b1 + 1, B2 = g.b2 + 1, B3 = g.b3 + 1, NN = B1 * B2 * B3;
  const int NEx = g.b1 * B2 * B3, NEy = B1 * g.b2 * B3, NEz = B1 * B2 * g.b3;
  double* Sn = gsm;                       // [NN][8] basis values on the block closure
  double* xi = Sn + (size_t)NN * 8;       // [NEx | NEy | NEz]
  double* Tj = xi + NEx + NEy + NEz;      // [8][nrhs]
  double* Yj = Tj + 8 * nrhs;             // [8][nrhs]
  double* M = Yj + 8 * nrhs;              // [8][8]

  for (int i = tid; i < 8 * nrhs; i += blockDim.x) {
    const int cc = i / nrhs, s = i - cc * nrhs;
    const size_t col = (size_t)corner_col(g, bi, bj, bk, cc);
    Tj[i] = T[col * nrhs + s];
    Yj[i] = Y[col * nrhs + s];
  }
  const double* Sb = Sint + (size_t)jb * 8 * g.nI;
  for (int i = tid; i < 8 * g.nI; i += blockDim.x) {
    const int cc = i / g.nI, a = i - cc * g.nI;
    int x, y, z;
    decode3f(a, g.ni1, g.r_ni1, g.ni2, g.r_ni2, x, y, z);
    Sn[((x + 1) + B1 * ((y + 1) + B2 * (z + 1))) * 8 + cc] = __ldg(Sb + i);
  }
  for (int n = tid; n < NN; n += blockDim.x) {
    const int x = n % B1, r = n / B1, y = r % B2, z = r / B2;
    if (x > 0 && x < g.b1 && y > 0 && y < g.b2 && z > 0 && z < g.b3) continue;
    const bool node0 = jb == 0 && n == 0;     // pinned node: no row of S
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) Sn[n * 8 + cc] = node0 ? 0.0 : hatf(g, cc, x, y, z);
  }
  __syncthreads();
  if (tid < 64) {
    const int c = tid >> 3, c2 = tid & 7;
    double v = 0.0;
    for (int s = 0; s < nrhs; ++s) v += Tj[c * nrhs + s] * Yj[c2 * nrhs + s];
    M[tid] = v;
  }
  __syncthreads();
  const int zs = zslot ? zslot[jb] : -1, rs = rslot ? rslot[jb] : -1;
  const int NE = NEx + NEy + NEz;
  for (int e = tid; e < NE; e += blockDim.x) {
    int x, y, z, step;
    double ihs;
    if (e < NEx) {
      x = e % g.b1; const int r = e / g.b1; y = r % B2; z = r / B2; step = 1; ihs = g.ih1 * g.ih1;
    } else if (e < NEx + NEy) {
      const int f = e - NEx;
      x = f % B1; const int r = f / B1; y = r % g.b2; z = r / g.b2; step = B1; ihs = g.ih2 * g.ih2;
    } else {
      const int f = e - NEx - NEy;
      x = f % B1; const int r = f / B1; y = r % B2; z = r / B2; step = B1 * B2; ihs = g.ih3 * g.ih3;
    }
    const int na = x + B1 * (y + B2 * z), nb = na + step;
    double d[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) d[cc] = Sn[nb * 8 + cc] - Sn[na * 8 + cc];
    double v = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double t = 0.0;
#pragma unroll
      for (int c2 = 0; c2 < 8; ++c2) t += M[c * 8 + c2] * d[c2];
      v += d[c] * t;
    }
    if (zs >= 0 || rs >= 0) {
      // interior-source / receiver blocks: dU dZ + dR dY per source
      const int xb = x + (step == 1), yb = y + (step == B1), zb = z + (step == B1 * B2);
      const int ia = interior_index(g, x, y, z), ib = interior_index(g, xb, yb, zb);
      for (int s = 0; s < nrhs; ++s) {
        double du = 0.0, dy = 0.0;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          du += d[cc] * Tj[cc * nrhs + s];
          dy += d[cc] * Yj[cc * nrhs + s];
        }
        double dz = 0.0, dr = 0.0;
        if (zs >= 0) {
          const double* Zb = Zc + (size_t)zs * g.nI * nrhs;
          dz = (ib >= 0 ? Zb[(size_t)ib * nrhs + s] : 0.0) - (ia >= 0 ? Zb[(size_t)ia * nrhs + s] : 0.0);
        }
        if (rs >= 0) {
          const double* Rb = Rc + (size_t)rs * g.nI * nrhs;
          dr = (ib >= 0 ? Rb[(size_t)ib * nrhs + s] : 0.0) - (ia >= 0 ? Rb[(size_t)ia * nrhs + s] : 0.0);
        }
        v += du * dz + dr * dy;
      }
    }
    xi[e] = v * ihs;
  }
  __syncthreads();
  const double* xx = xi;
  const double* xy = xi + NEx;
  const double* xz = xi + NEx + NEy;
  const int ncell = g.b1 * g.b2 * g.b3;
  for (int c = tid; c < ncell; c += blockDim.x) {
    const int x = c % g.b1, r = c / g.b1, y = r % g.b2, z = r / g.b2;
    auto ex = [&](int i, int j, int k) { return xx[i + g.b1 * (j + B2 * k)]; };
    auto ey = [&](int i, int j, int k) { return xy[i + B1 * (j + g.b2 * k)]; };
    auto ez = [&](int i, int j, int k) { return xz[i + B1 * (j + B2 * k)]; };
    double tot = 0.0;
    tot += ex(x, y, z) + ex(x, y + 1, z) + ex(x, y, z + 1) + ex(x, y + 1, z + 1);
    tot += ey(x, y, z) + ey(x + 1, y, z) + ey(x, y, z + 1) + ey(x + 1, y, z + 1);
    tot += ez(x, y, z) + ez(x + 1, y, z) + ez(x, y + 1, z) + ez(x + 1, y + 1, z);
    const long long cid = cell_id(g, X0 + x, Y0 + y, Z0 + z);
    gout[cid] = -sigma[cid] * (g.qv * tot);
  }
}

bool grad_supported(const Geo& g, int nrhs) { return grad_smem_doubles(g, nrhs) * sizeof(double) <= 200 * 1024; }

cudaError_t launch_grad_block(const Geo& g, const double* Sint, const double* T, const double* Y, int nrhs,
                              const double* sigma, const int* zslot, const double* Zc, const int* rslot,
                              const double* Rc, double* gout, cudaStream_t st) {
  const size_t smem = grad_smem_doubles(g, nrhs) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_grad_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_grad_block<<<g.nbl, GRAD_THREADS, smem, st>>>(g, Sint, T, Y, nrhs, sigma, zslot, Zc, rslot, Rc, gout);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
