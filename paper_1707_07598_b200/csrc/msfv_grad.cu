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
#include <algorithm>
#include <cstdlib>
#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace msfv {

// Basis values of block jb's 8 columns on its closure nodes (x fastest,
// (b1+1)(b2+1)(b3+1) nodes x 8): interior from Sint, skeleton from the hats,
// 0 at the pinned node.
// BB > 0: cubic blocks of BB cells per axis known at compile time (every
// index decode folds to multiply/shift); BB == 0: sizes from the Geo.
template <int BB>
__device__ __forceinline__ void stage_closure(const Geo& g, int jb, const double* __restrict__ Sint, double* Sn) {
  const int b1 = BB ? BB : g.b1, b2 = BB ? BB : g.b2, b3 = BB ? BB : g.b3;
  const int B1 = b1 + 1, B2 = b2 + 1, B3 = b3 + 1, NN = B1 * B2 * B3;
  const int ni1 = b1 - 1, ni2 = b2 - 1, nI = ni1 * ni2 * (b3 - 1);
  const double* Sb = Sint + (size_t)jb * 8 * nI;
  // interior: one coordinate decode per node, the 8 corner loads in flight together
  for (int a = threadIdx.x; a < nI; a += blockDim.x) {
    double v[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) v[cc] = __ldg(Sb + (size_t)cc * nI + a);
    int x, y, z;
    if (BB) {
      x = a % ni1; const int r = a / ni1; y = r % ni2; z = r / ni2;
    } else {
      decode3f(a, g.ni1, g.r_ni1, g.ni2, g.r_ni2, x, y, z);
    }
    double* d = Sn + ((x + 1) + B1 * ((y + 1) + B2 * (z + 1))) * 8;
#pragma unroll
    for (int cc = 0; cc < 8; cc += 2) *reinterpret_cast<double2*>(d + cc) = make_double2(v[cc], v[cc + 1]);
  }
  // skeleton: separable hats (6 one-dimensional values per node)
  for (int n = threadIdx.x; n < NN; n += blockDim.x) {
    const int x = n % B1, r = n / B1, y = r % B2, z = r / B2;
    if (x > 0 && x < b1 && y > 0 && y < b2 && z > 0 && z < b3) continue;
    const bool node0 = jb == 0 && n == 0;     // pinned node: no row of S
    const double hx[2] = {hatf1(x, g.ib1), hatf1(x - b1, g.ib1)};
    const double hy[2] = {hatf1(y, g.ib2), hatf1(y - b2, g.ib2)};
    const double hz[2] = {hatf1(z, g.ib3), hatf1(z - b3, g.ib3)};
    double h[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) h[cc] = node0 ? 0.0 : (hx[cc & 1] * hy[(cc >> 1) & 1]) * hz[cc >> 2];
#pragma unroll
    for (int cc = 0; cc < 8; cc += 2) *reinterpret_cast<double2*>(Sn + n * 8 + cc) = make_double2(h[cc], h[cc + 1]);
  }
}

// 8^3 blocks: the skeleton part of the closure (hats, identical for every
// block but the pinned node of block 0) and the closure edge table are one
// device-resident template; each CTA bulk-copies it into shared memory (TMA,
// L2-resident after the first CTAs) while its threads fetch the interior
// values, instead of recomputing 386 hat products and 1944 edge decodes.
constexpr int TPL_NN = 9 * 9 * 9, TPL_NE = 3 * 8 * 9 * 9, TPL_NEP = 2048;   // edge table padded to 16 warps x 16 steps x 8
__device__ __align__(16) double g_tpl8_sn[TPL_NN * 8];
__device__ __align__(16) int g_tpl8_et[TPL_NEP];

bool grad_template_init(const Geo& g) {
  if (!(g.b1 == 8 && g.b2 == 8 && g.b3 == 8)) return false;
  static double sn[TPL_NN * 8];
  static int et[TPL_NEP];   // padding entries: node 0, x axis (results discarded)
  const double ib = 1.0 / 8;
  auto hat = [&](int d) { const double v = 1.0 - fabs((double)d) * ib; return v > 0.0 ? v : 0.0; };
  for (int n = 0; n < TPL_NN; ++n) {
    const int x = n % 9, y = (n / 9) % 9, z = n / 81;
    const bool inner = x > 0 && x < 8 && y > 0 && y < 8 && z > 0 && z < 8;
    const double hx[2] = {hat(x), hat(x - 8)}, hy[2] = {hat(y), hat(y - 8)}, hz[2] = {hat(z), hat(z - 8)};
    for (int cc = 0; cc < 8; ++cc) sn[n * 8 + cc] = inner ? 0.0 : (hx[cc & 1] * hy[(cc >> 1) & 1]) * hz[cc >> 2];
  }
  const int NEx = 8 * 81, NEy = 8 * 81;
  for (int e = 0; e < TPL_NE; ++e) {
    int x, y, z, ax;
    if (e < NEx) { x = e % 8; y = (e / 8) % 9; z = e / 72; ax = 0; }
    else if (e < NEx + NEy) { const int f = e - NEx; x = f % 9; y = (f / 9) % 8; z = f / 72; ax = 1; }
    else { const int f = e - NEx - NEy; x = f % 9; y = (f / 9) % 9; z = f / 81; ax = 2; }
    et[e] = (x + 9 * (y + 9 * z)) | (ax << 24);
  }
  return cudaMemcpyToSymbol(g_tpl8_sn, sn, sizeof(sn)) == cudaSuccess &&
         cudaMemcpyToSymbol(g_tpl8_et, et, sizeof(et)) == cudaSuccess;
}

namespace {
__device__ __forceinline__ unsigned g_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
}

// Closure staging from the template: thread 0 bulk-copies the hats (into Sn)
// and, when Et != nullptr, the edge table; every thread loads its interior
// values into registers meanwhile, waits on the copy, then overwrites the
// interior nodes.  NT = blockDim.x.
template <int NT>
__device__ __forceinline__ void stage_closure_tpl8(int jb, const double* __restrict__ Sint, double* Sn, int* Et,
                                                   unsigned long long* bar) {
  constexpr int nI = 343;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(g_smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    const unsigned bsn = TPL_NN * 8 * sizeof(double), bet = Et ? TPL_NEP * sizeof(int) : 0;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(g_smem_u32(bar)), "r"(bsn + bet)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     g_smem_u32(Sn)), "l"(g_tpl8_sn), "r"(bsn), "r"(g_smem_u32(bar))
                 : "memory");
    if (Et)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       g_smem_u32(Et)), "l"(g_tpl8_et), "r"(bet), "r"(g_smem_u32(bar))
                   : "memory");
  }
  const double* Sb = Sint + (size_t)jb * 8 * nI;
  constexpr int NIT = (nI + NT - 1) / NT;
  double v[NIT][8];
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int a = tid + it * NT;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) v[it][cc] = a < nI ? __ldg(Sb + (size_t)cc * nI + a) : 0.0;
  }
  {
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(g_smem_u32(bar)), "r"(0u)
          : "memory");
    }
  }
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int a = tid + it * NT;
    if (a < nI) {
      const int x = a % 7, r = a / 7, y = r % 7, z = r / 7;
      double* d = Sn + ((x + 1) + 9 * ((y + 1) + 9 * (z + 1))) * 8;
#pragma unroll
      for (int cc = 0; cc < 8; cc += 2) *reinterpret_cast<double2*>(d + cc) = make_double2(v[it][cc], v[it][cc + 1]);
    }
  }
  if (jb == 0 && tid < 8) Sn[tid] = 0.0;     // pinned node: no row of S
}

size_t grad_smem_doubles(const Geo& g, int nrhs) {
  const size_t B1 = g.b1 + 1, B2 = g.b2 + 1, B3 = g.b3 + 1;
  const size_t ne = (size_t)g.b1 * B2 * B3 + B1 * g.b2 * B3 + B1 * B2 * g.b3;
  return B1 * B2 * B3 * 8 + ne + 16 * (size_t)nrhs + 64 + (ne + 1) / 2 + 64;   // + packed edge table (ints, padded)
}

// 8^3 blocks run 16 warps per CTA (two CTAs per SM, 64 registers): twice the
// warps of the 256-thread form at the same shared-memory occupancy.
constexpr int GRAD_T8 = 512;

template <int BB>
__global__ void __launch_bounds__(BB == 8 ? GRAD_T8 : GRAD_THREADS, BB == 8 ? 2 : 3)
k_grad_block(Geo g, const double* __restrict__ Sint, const double* __restrict__ T, const double* __restrict__ Y,
             int nrhs, const double* __restrict__ sigma, const int* __restrict__ zslot, const double* __restrict__ Zc,
             const int* __restrict__ rslot, const double* __restrict__ Rc, double* __restrict__ gout, int jb0) {
  extern __shared__ __align__(16) double gsm[];
  const int b1 = BB ? BB : g.b1, b2 = BB ? BB : g.b2, b3 = BB ? BB : g.b3;
  const int jb = jb0 + blockIdx.x, tid = threadIdx.x;
  int bi, bj, bk;
  decode3f(jb, g.nb1, g.r_nb1, g.nb2, g.r_nb2, bi, bj, bk);
  const int X0 = bi * b1, Y0 = bj * b2, Z0 = bk * b3;
  const int B1 = b1 + 1, B2 = b2 + 1, B3 = b3 + 1, NN = B1 * B2 * B3;
  const int NEx = b1 * B2 * B3, NEy = B1 * b2 * B3, NEz = B1 * B2 * b3;
  double* Sn = gsm;                       // [NN][8] basis values on the block closure
  double* xi = Sn + (size_t)NN * 8;       // [NEx | NEy | NEz]
  double* Tj = xi + NEx + NEy + NEz;      // [8][nrhs]
  double* Yj = Tj + 8 * nrhs;             // [8][nrhs]
  double* M = Yj + 8 * nrhs;              // [8][8]
  int* Et = reinterpret_cast<int*>(M + 64);  // [NE] lower closure node | axis << 24

  for (int i = tid; i < 8 * nrhs; i += blockDim.x) {
    const int cc = i & 7, s = i >> 3;
    const size_t col = (size_t)corner_col(g, bi, bj, bk, cc);
    Tj[cc * nrhs + s] = T[col * nrhs + s];
    Yj[cc * nrhs + s] = Y[col * nrhs + s];
  }
  if (BB == 8) {
    __shared__ unsigned long long tbar;
    stage_closure_tpl8<GRAD_T8>(jb, Sint, Sn, Et, &tbar);
  } else {
    stage_closure<BB>(g, jb, Sint, Sn);
  }
  __syncthreads();
  if (tid < 32) {   // M = Tj Yj^T on the DMMA, 4 sources per step (one warp)
    const int m = tid >> 2, k = tid & 3;
    double c0 = 0.0, c1 = 0.0;
    for (int s0 = 0; s0 < nrhs; s0 += 4) {
      const bool ok = s0 + k < nrhs;
      const double a = ok ? Tj[m * nrhs + s0 + k] : 0.0, b = ok ? Yj[m * nrhs + s0 + k] : 0.0;
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    }
    M[m * 8 + 2 * k] = c0;
    M[m * 8 + 2 * k + 1] = c1;
  }
  __syncthreads();
  const int zs = zslot ? zslot[jb] : -1, rs = rslot ? rslot[jb] : -1;
  const int NE = NEx + NEy + NEz;
  // edge e -> lower closure node, step to the upper node, 1/h^2
  auto edge = [&](int e, int& na, int& step, double& ihs) {
    int x, y, z;
    if (e < NEx) {
      x = e % b1; const int r = e / b1; y = r % B2; z = r / B2; step = 1; ihs = g.ih1 * g.ih1;
    } else if (e < NEx + NEy) {
      const int f = e - NEx;
      x = f % B1; const int r = f / B1; y = r % b2; z = r / b2; step = B1; ihs = g.ih2 * g.ih2;
    } else {
      const int f = e - NEx - NEy;
      x = f % B1; const int r = f / B1; y = r % B2; z = r / B2; step = B1 * B2; ihs = g.ih3 * g.ih3;
    }
    na = x + B1 * (y + B2 * z);
  };
  if (zs < 0 && rs < 0) {
    if (BB != 8) {   // no template: decode each edge once into a table
      for (int e = tid; e < NE; e += blockDim.x) {
        int na, step;
        double ihs;
        edge(e, na, step, ihs);
        Et[e] = na | ((e < NEx ? 0 : (e < NEx + NEy ? 1 : 2)) << 24);
      }
      __syncthreads();
    }
    const double ihx[3] = {g.ih1 * g.ih1, g.ih2 * g.ih2, g.ih3 * g.ih3};
    // xi_e = dS_e^T M dS_e for 8 edges per warp step: D (8 edges x 8 corners,
    // accumulator layout) times M on the DMMA (D += X Y^T with Y = M^T), then
    // the row-wise product with D and a 4-lane reduction.
    const int lane = tid & 31, wv = tid >> 5, m = lane >> 2, q = lane & 3;
    const double mt0 = M[(2 * q) * 8 + m], mt1 = M[(2 * q + 1) * 8 + m];   // C layout of M^T
    if (BB == 8) {
      // padded template table: fixed trip count, no bounds test but on the store
#pragma unroll 4
      for (int it = 0; it < TPL_NEP / (8 * (GRAD_T8 / 32)); ++it) {
        const int e = (it * (GRAD_T8 / 32) + wv) * 8 + m;
        const int pk = Et[e], ax = pk >> 24, na = pk & 0xFFFFFF;
        const int nb = na + (ax == 0 ? 1 : (ax == 1 ? 9 : 81));
        const double ihs = ax == 0 ? ihx[0] : (ax == 1 ? ihx[1] : ihx[2]);
        const double2 sb = *reinterpret_cast<const double2*>(Sn + nb * 8 + 2 * q);
        const double2 sa = *reinterpret_cast<const double2*>(Sn + na * 8 + 2 * q);
        const double d0 = sb.x - sa.x, d1 = sb.y - sa.y;
        double c0 = 0.0, c1 = 0.0;
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
            : "+d"(c0), "+d"(c1) : "d"(d0), "d"(mt0));
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
            : "+d"(c0), "+d"(c1) : "d"(d1), "d"(mt1));
        double v = c0 * d0 + c1 * d1;
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (q == 0 && e < NE) xi[e] = v * ihs;
      }
    } else
#pragma unroll 2
    for (int e0 = 8 * wv; e0 < NE; e0 += 8 * (blockDim.x >> 5)) {
      const int e = e0 + m;
      double d0 = 0.0, d1 = 0.0, ihs = 0.0;
      if (e < NE) {
        const int pk = Et[e], ax = pk >> 24, na = pk & 0xFFFFFF;
        const int nb = na + (ax == 0 ? 1 : (ax == 1 ? B1 : B1 * B2));
        ihs = ax == 0 ? ihx[0] : (ax == 1 ? ihx[1] : ihx[2]);
        const double2 sb = *reinterpret_cast<const double2*>(Sn + nb * 8 + 2 * q);
        const double2 sa = *reinterpret_cast<const double2*>(Sn + na * 8 + 2 * q);
        d0 = sb.x - sa.x;
        d1 = sb.y - sa.y;
      }
      double c0 = 0.0, c1 = 0.0;
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c0), "+d"(c1) : "d"(d0), "d"(mt0));
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c0), "+d"(c1) : "d"(d1), "d"(mt1));
      double v = c0 * d0 + c1 * d1;
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      if (q == 0 && e < NE) xi[e] = v * ihs;
    }
  } else {
    // interior-source / receiver blocks: scalar path with dU dZ + dR dY per source
    for (int e = tid; e < NE; e += blockDim.x) {
      int na, step;
      double ihs;
      edge(e, na, step, ihs);
      const int nb = na + step;
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
      const int x = na % B1, r = na / B1, y = r % B2, z = r / B2;
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
      xi[e] = v * ihs;
    }
  }
  __syncthreads();
  const double* xx = xi;
  const double* xy = xi + NEx;
  const double* xz = xi + NEx + NEy;
  const int ncell = b1 * b2 * b3;
  for (int c = tid; c < ncell; c += blockDim.x) {
    const int x = c % b1, r = c / b1, y = r % b2, z = r / b2;
    auto ex = [&](int i, int j, int k) { return xx[i + b1 * (j + B2 * k)]; };
    auto ey = [&](int i, int j, int k) { return xy[i + B1 * (j + b2 * k)]; };
    auto ez = [&](int i, int j, int k) { return xz[i + B1 * (j + B2 * k)]; };
    const double tx = (ex(x, y, z) + ex(x, y + 1, z)) + (ex(x, y, z + 1) + ex(x, y + 1, z + 1));
    const double ty = (ey(x, y, z) + ey(x + 1, y, z)) + (ey(x, y, z + 1) + ey(x + 1, y, z + 1));
    const double tz = (ez(x, y, z) + ez(x + 1, y, z)) + (ez(x, y + 1, z) + ez(x + 1, y + 1, z));
    const double tot = (tx + ty) + tz;
    const long long cid = cell_id(g, X0 + x, Y0 + y, Z0 + z);
    gout[cid] = -sigma[cid] * (g.qv * tot);
  }
}

// Coarse right-hand side of J v (forward.py:258-269) for surveys without
// interior receivers.  With c = Csig dm, U = S T and R = interior_solve(Q - A U):
//   rhs = xdm - S^T(gdm + A ydm) = -EP^T((G U + G R) o c)       (S^T A ydm = (A S)^T ydm = 0)
// and EP^T diag(c) G S T = sum_j  K_c(j) T_j,  K_c(j) = sum_{e owned by j} (c_e/h_e^2) dS_e dS_e^T,
// i.e. the Galerkin block of the conductances c.  part[j][cc][s] holds block
// j's share (gathered to coarse nodes by k_gather_corners with scale -1).
// Edge ownership: the edge's lower node is owned by j (node ownership of
// k_restrict_op).  K_c is a DMMA reduction (lane = corner cc, edge slot).
template <int BB>
__global__ void __launch_bounds__(GRAD_THREADS)
k_jv_block(Geo g, const double* __restrict__ Sint, const double* __restrict__ cvec, const double* __restrict__ T,
           int nrhs, const int* __restrict__ rslot, const double* __restrict__ Rc, double* __restrict__ part) {
  extern __shared__ __align__(16) double gsm[];
  const int b1 = BB ? BB : g.b1, b2 = BB ? BB : g.b2, b3 = BB ? BB : g.b3;
  const int jb = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int bi, bj, bk;
  decode3f(jb, g.nb1, g.r_nb1, g.nb2, g.r_nb2, bi, bj, bk);
  const int X0 = bi * b1, Y0 = bj * b2, Z0 = bk * b3;
  const int B1 = b1 + 1, B2 = b2 + 1, B3 = b3 + 1, NN = B1 * B2 * B3;
  const int ox = b1 + (bi == g.nb1 - 1), oy = b2 + (bj == g.nb2 - 1), oz = b3 + (bk == g.nb3 - 1);
  const int NOx = b1 * oy * oz, NOy = ox * b2 * oz, NOz = ox * oy * b3, NO = NOx + NOy + NOz;
  double* Sn = gsm;                       // [NN][8]
  double* Kw = Sn + (size_t)NN * 8;       // [8 warps][64]
  double* Tj = Kw + 8 * 64;               // [8][nrhs]
  if (BB == 8) {
    __shared__ unsigned long long tbar;
    stage_closure_tpl8<GRAD_THREADS>(jb, Sint, Sn, nullptr, &tbar);
  } else {
    stage_closure<BB>(g, jb, Sint, Sn);
  }
  for (int i = tid; i < 8 * nrhs; i += blockDim.x) {
    const int cc = i & 7, s = i >> 3;
    Tj[cc * nrhs + s] = T[(size_t)corner_col(g, bi, bj, bk, cc) * nrhs + s];
  }
  __syncthreads();
  // owned edge f -> (local lower node, step, global edge id, 1/h^2)
  auto edge = [&](int f, int& na, int& step, long long& eid, double& ihs) {
    int x, y, z;
    if (f < NOx) {
      x = f % b1; const int r = f / b1; y = r % oy; z = r / oy;
      step = 1; ihs = g.ih1 * g.ih1; eid = ex_id(g, X0 + x, Y0 + y, Z0 + z);
    } else if (f < NOx + NOy) {
      const int h = f - NOx;
      x = h % ox; const int r = h / ox; y = r % b2; z = r / b2;
      step = B1; ihs = g.ih2 * g.ih2; eid = ey_id(g, X0 + x, Y0 + y, Z0 + z);
    } else {
      const int h = f - NOx - NOy;
      x = h % ox; const int r = h / ox; y = r % oy; z = r / oy;
      step = B1 * B2; ihs = g.ih3 * g.ih3; eid = ez_id(g, X0 + x, Y0 + y, Z0 + z);
    }
    na = x + B1 * (y + B2 * z);
  };
  // owned-edge table: lower node | step code << 24 and c_e / h_e^2 (one decode
  // and one load of c per edge)
  int* Et = reinterpret_cast<int*>(Tj + 8 * nrhs);
  double* Ce = reinterpret_cast<double*>(Et + ((NO + 1) & ~1));
  for (int f = tid; f < NO; f += blockDim.x) {
    int na, step;
    long long eid;
    double ihs;
    edge(f, na, step, eid, ihs);
    Et[f] = na | ((step == 1 ? 0 : (step == B1 ? 1 : 2)) << 24);
    Ce[f] = __ldg(cvec + eid) * ihs;
  }
  __syncthreads();
  const int cc = lane >> 2, slot = lane & 3;
  double k0 = 0.0, k1 = 0.0;
  for (int base = 4 * wid; base < NO; base += 32) {
    const int f = base + slot;
    double a = 0.0, b = 0.0;
    if (f < NO) {
      const int pk = Et[f], sc = pk >> 24, na = pk & 0xFFFFFF;
      const int nb = na + (sc == 0 ? 1 : (sc == 1 ? B1 : B1 * B2));
      b = Sn[nb * 8 + cc] - Sn[na * 8 + cc];
      a = Ce[f] * b;
    }
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(k0), "+d"(k1)
        : "d"(a), "d"(b));
  }
  Kw[wid * 64 + 2 * lane] = k0;
  Kw[wid * 64 + 2 * lane + 1] = k1;
  __syncthreads();
  if (tid < 64) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += Kw[w * 64 + tid];
    Kw[tid] = v;                         // warp 0's slot now holds K_c (row-major 8x8)
  }
  __syncthreads();
  const int rs = rslot ? rslot[jb] : -1;
  const double* Rb = rs >= 0 ? Rc + (size_t)rs * g.nI * nrhs : nullptr;
  for (int i = tid; i < 8 * nrhs; i += blockDim.x) {
    const int c1 = i / nrhs, s = i - c1 * nrhs;
    double v = 0.0;
#pragma unroll
    for (int c2 = 0; c2 < 8; ++c2) v += Kw[c1 * 8 + c2] * Tj[c2 * nrhs + s];
    if (Rb) {
      // source blocks: + sum_e (c_e/h^2) dS_c1(e) dR_s(e), R interior-only
      for (int f = 0; f < NO; ++f) {
        int na, step;
        long long eid;
        double ihs;
        edge(f, na, step, eid, ihs);
        const int nb = na + step;
        const int xa = na % B1, ya = (na / B1) % B2, za = na / (B1 * B2);
        const int xb = nb % B1, yb = (nb / B1) % B2, zb = nb / (B1 * B2);
        const int ia = interior_index(g, xa, ya, za), ib = interior_index(g, xb, yb, zb);
        const double dr = (ib >= 0 ? Rb[(size_t)ib * nrhs + s] : 0.0) - (ia >= 0 ? Rb[(size_t)ia * nrhs + s] : 0.0);
        if (dr == 0.0) continue;
        v += (__ldg(cvec + eid) * ihs) * (Sn[nb * 8 + c1] - Sn[na * 8 + c1]) * dr;
      }
    }
    part[((size_t)jb * 8 + c1) * nrhs + s] = v;
  }
}

size_t jv_smem_doubles(const Geo& g, int nrhs) {
  const size_t B1 = g.b1 + 1, B2 = g.b2 + 1, B3 = g.b3 + 1;
  const size_t ne = (size_t)g.b1 * B2 * B3 + B1 * g.b2 * B3 + B1 * B2 * g.b3;   // >= owned edges
  return B1 * B2 * B3 * 8 + 8 * 64 + 8 * (size_t)nrhs + (ne + 2) / 2 + ne;
}

cudaError_t launch_jv_block(const Geo& g, const double* Sint, const double* cvec, const double* T, int nrhs,
                            const int* rslot, const double* Rc, double* part, cudaStream_t st) {
  const size_t smem = jv_smem_doubles(g, nrhs) * sizeof(double);
  auto kern = g.gtab8 ? k_jv_block<8> : k_jv_block<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<g.nbl, GRAD_THREADS, smem, st>>>(g, Sint, cvec, T, nrhs, rslot, Rc, part);
  count_launches(1);
  return cudaGetLastError();
}

bool grad_supported(const Geo& g, int nrhs) { return grad_smem_doubles(g, nrhs) * sizeof(double) <= 200 * 1024; }

// ---------------------------------------------------------------------------
// 8^3 blocks without interior survey nodes (every BASELINE 3D config): a
// persistent form.  Each CTA (16 warps, two per SM) keeps the closure hats and
// the edge table in shared memory for all its blocks (one template copy per
// CTA instead of per block) and streams the blocks: the next block's interior
// basis values (8 x 343 doubles, one contiguous 21 952-byte run of Sint) and
// its 512 cell conductivities arrive by bulk / cp.async copies while the
// current block's xi and cell gather run, so the HBM reads overlap compute.
namespace {
constexpr int GP_NI = 343, GP_SINT = 8 * GP_NI;
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(g_smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   g_smem_u32(dst)), "l"(src), "r"(bytes), "r"(g_smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(g_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(g_smem_u32(smem)), "l"(gmem));
}
}  // namespace

size_t grad8p_smem_bytes(int nrhs) {
  return ((size_t)TPL_NN * 8 + TPL_NE + GP_SINT + 512 + 16 * (size_t)nrhs + 64) * sizeof(double) +
         TPL_NEP * sizeof(int) + 64;
}

__global__ void __launch_bounds__(GRAD_T8, 2)
k_grad_block8p(Geo g, const double* __restrict__ Sint, const double* __restrict__ T, const double* __restrict__ Y,
               int nrhs, const double* __restrict__ sigma, double* __restrict__ gout, int jb0, int nb) {
  extern __shared__ __align__(16) double gsm[];
  __shared__ __align__(8) unsigned long long bars[2];   // 0: template, 1: next block's Sint
  constexpr int B1 = 9, B2 = 9, NEx = 8 * 81, NEy = 8 * 81, NE = TPL_NE;
  double* Sn = gsm;                               // [729][8] closure basis values (hats + interior)
  double* xi = Sn + TPL_NN * 8;                   // [1944]
  double* St = xi + NE;                           // [8][343] staged Sint of the next block
  double* Sg = St + GP_SINT;                      // [512] staged sigma of the next block (x fastest)
  double* Tj = Sg + 512;                          // [8][nrhs]
  double* Yj = Tj + 8 * nrhs;                     // [8][nrhs]
  double* M = Yj + 8 * nrhs;                      // [64]
  int* Et = reinterpret_cast<int*>(M + 64);       // [TPL_NEP]
  const int tid = threadIdx.x, lane = tid & 31, wv = tid >> 5, m = lane >> 2, q = lane & 3;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(g_smem_u32(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(g_smem_u32(&bars[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  int k = blockIdx.x;                             // local block index: jb = jb0 + k
  if (k >= nb) return;
  auto stage_next = [&](int kk) {                 // thread 0: Sint run; all threads: sigma rows (cp.async)
    const int jb = jb0 + kk;
    if (tid == 0) {
      expect_tx(&bars[1], GP_SINT * sizeof(double));
      bulk_g2s(St, Sint + (size_t)jb * GP_SINT, GP_SINT * sizeof(double), &bars[1]);
    }
    int bi, bj, bk;
    decode3f(jb, g.nb1, g.r_nb1, g.nb2, g.r_nb2, bi, bj, bk);
    if (tid < 256) {                              // 64 rows of 8 cells, 4 x 16 bytes each
      const int row = tid >> 2, part = tid & 3, y = row & 7, z = row >> 3;
      const long long cid = cell_id(g, bi * 8, bj * 8 + y, bk * 8 + z);
      cp_async16(Sg + row * 8 + part * 2, sigma + cid + part * 2);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  if (tid == 0) {
    expect_tx(&bars[0], TPL_NN * 8 * sizeof(double) + TPL_NEP * sizeof(int));
    bulk_g2s(Sn, g_tpl8_sn, TPL_NN * 8 * sizeof(double), &bars[0]);
    bulk_g2s(Et, g_tpl8_et, TPL_NEP * sizeof(int), &bars[0]);
  }
  stage_next(k);
  mbar_wait(&bars[0], 0);
  const double ihx[3] = {g.ih1 * g.ih1, g.ih2 * g.ih2, g.ih3 * g.ih3};
  unsigned par = 0;
  for (; k < nb; k += gridDim.x) {
    const int jb = jb0 + k;
    int bi, bj, bk;
    decode3f(jb, g.nb1, g.r_nb1, g.nb2, g.r_nb2, bi, bj, bk);
    for (int i = tid; i < 8 * nrhs; i += blockDim.x) {
      const int cc = i & 7, s = i >> 3;
      const size_t col = (size_t)corner_col(g, bi, bj, bk, cc);
      Tj[cc * nrhs + s] = T[col * nrhs + s];
      Yj[cc * nrhs + s] = Y[col * nrhs + s];
    }
    mbar_wait(&bars[1], par);
    par ^= 1u;
    // interior basis values into the closure (the hats stay from the template)
    for (int a = tid; a < GP_NI; a += blockDim.x) {
      const int x = a % 7, r = a / 7, y = r % 7, z = r / 7;
      double* d = Sn + ((x + 1) + 9 * ((y + 1) + 9 * (z + 1))) * 8;
#pragma unroll
      for (int cc = 0; cc < 8; cc += 2) *reinterpret_cast<double2*>(d + cc) = make_double2(St[cc * GP_NI + a], St[(cc + 1) * GP_NI + a]);
    }
    if (jb == 0 && tid < 8) Sn[tid] = 0.0;        // pinned node: no row of S
    __syncthreads();                              // St consumed; Tj/Yj/Sn ready
    const int knext = k + gridDim.x;
    // M = Tj Yj^T (warp 0) while the next block's copies start
    if (tid < 32) {
      double c0 = 0.0, c1 = 0.0;
      for (int s0 = 0; s0 < nrhs; s0 += 4) {
        const bool ok = s0 + q < nrhs;
        const double a = ok ? Tj[m * nrhs + s0 + q] : 0.0, b = ok ? Yj[m * nrhs + s0 + q] : 0.0;
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
            : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
      }
      M[m * 8 + 2 * q] = c0;
      M[m * 8 + 2 * q + 1] = c1;
    }
    __syncthreads();
    // sigma of this block (cp.async group of the previous stage) is needed by the
    // gather below; the next block's Sint bulk copy goes out now
    asm volatile("cp.async.wait_group 0;\n" ::);
    double sg = 0.0;
    {
      const int x = tid & 7, y = (tid >> 3) & 7, z = tid >> 6;
      sg = Sg[(y + 8 * z) * 8 + x];
    }
    __syncthreads();                              // everyone has its sigma: Sg may be refilled
    if (knext < nb) stage_next(knext);
    const double mt0 = M[(2 * q) * 8 + m], mt1 = M[(2 * q + 1) * 8 + m];
#pragma unroll 4
    for (int it = 0; it < TPL_NEP / (8 * (GRAD_T8 / 32)); ++it) {
      const int e = (it * (GRAD_T8 / 32) + wv) * 8 + m;
      const int pk = Et[e], ax = pk >> 24, na = pk & 0xFFFFFF;
      const int nbn = na + (ax == 0 ? 1 : (ax == 1 ? 9 : 81));
      const double ihs = ax == 0 ? ihx[0] : (ax == 1 ? ihx[1] : ihx[2]);
      const double2 sb = *reinterpret_cast<const double2*>(Sn + nbn * 8 + 2 * q);
      const double2 sa = *reinterpret_cast<const double2*>(Sn + na * 8 + 2 * q);
      const double d0 = sb.x - sa.x, d1 = sb.y - sa.y;
      double c0 = 0.0, c1 = 0.0;
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c0), "+d"(c1) : "d"(d0), "d"(mt0));
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c0), "+d"(c1) : "d"(d1), "d"(mt1));
      double v = c0 * d0 + c1 * d1;
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      if (q == 0 && e < NE) xi[e] = v * ihs;
    }
    __syncthreads();
    if (jb == 0 && tid < 8) Sn[tid] = g_tpl8_sn[tid];   // restore the template's node-0 hats
    {
      const int x = tid & 7, y = (tid >> 3) & 7, z = tid >> 6;
      const double* xx = xi;
      const double* xy = xi + NEx;
      const double* xz = xi + NEx + NEy;
      auto ex = [&](int i, int j, int kk) { return xx[i + 8 * (j + B2 * kk)]; };
      auto ey = [&](int i, int j, int kk) { return xy[i + B1 * (j + 8 * kk)]; };
      auto ez = [&](int i, int j, int kk) { return xz[i + B1 * (j + B2 * kk)]; };
      const double tx = (ex(x, y, z) + ex(x, y + 1, z)) + (ex(x, y, z + 1) + ex(x, y + 1, z + 1));
      const double ty = (ey(x, y, z) + ey(x + 1, y, z)) + (ey(x, y, z + 1) + ey(x + 1, y, z + 1));
      const double tz = (ez(x, y, z) + ez(x + 1, y, z)) + (ez(x, y + 1, z) + ez(x + 1, y + 1, z));
      const double tot = (tx + ty) + tz;
      const long long cid = cell_id(g, bi * 8 + x, bj * 8 + y, bk * 8 + z);
      gout[cid] = -sg * (g.qv * tot);
    }
    __syncthreads();                              // xi / Tj / Yj reused by the next block
  }
}

cudaError_t launch_grad_block(const Geo& g, const double* Sint, const double* T, const double* Y, int nrhs,
                              const double* sigma, const int* zslot, const double* Zc, const int* rslot,
                              const double* Rc, double* gout, cudaStream_t st, int jb0, int nb) {
  if (nb < 0) nb = g.nbl - jb0;
  if (nb <= 0) return cudaSuccess;
  if (g.gtab8 && !zslot && !rslot && !getenv("MSFV_GRAD_NONPERSISTENT")) {
    const size_t sm8 = grad8p_smem_bytes(nrhs);
    static PerDevice<int> sms_cache;
    const int sms = sms_cache.get([] {
      int dev = 0, n = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      return n;
    });
    cudaError_t e8 = cudaFuncSetAttribute(k_grad_block8p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm8);
    if (e8 != cudaSuccess) return e8;
    const int grid = std::min(nb, 2 * sms);
    k_grad_block8p<<<grid, GRAD_T8, sm8, st>>>(g, Sint, T, Y, nrhs, sigma, gout, jb0, nb);
    count_launches(1);
    return cudaGetLastError();
  }
  const size_t smem = grad_smem_doubles(g, nrhs) * sizeof(double);
  auto kern = g.gtab8 ? k_grad_block<8> : k_grad_block<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<nb, g.gtab8 ? GRAD_T8 : GRAD_THREADS, smem, st>>>(g, Sint, T, Y, nrhs, sigma, zslot, Zc, rslot, Rc, gout, jb0);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
