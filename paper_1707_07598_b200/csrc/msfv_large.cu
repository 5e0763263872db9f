// Local solver for blocks whose interior band does not fit the register-tile
// kernels (msfv_tc.cu, half bandwidth p = ni1*ni2 <= 56): 12^3 and 16^3-cell
// blocks -- the paper's Table-3 geometry -- and any block
// up to p = 8 * LG_MAX_PT.  The reference factors these A_II densely
// (n_I <= 2000) or with SuperLU (basis.py:258-298); here all fill lives in the
// band, so the band Cholesky is exact and the same tile algorithm serves every
// size.
//
// Factor ("LT", the msfv_tc.cu layout with a runtime band): per block, per 8-row
// tile column J, PT+1 row-major 8x8 tiles: slot 0 = L_JJ^{-1}, slot t =
// L_{J+t,J} (PT = ceil(p/8)).  One CTA per block factors its band in place in
// global memory; a block's active window is (PT+1)^2/2 tiles (~230 KB at 16^3),
// so the working set of the resident CTAs stays in the 126 MB L2.  Per tile
// column: one warp factors the diagonal tile and inverts it, all warps form
// the panel X_t = A_t L_JJ^{-T} on the DMMA, then the trailing window
// A_{J+a,J+b} -= X_a X_b^T is spread over the warps in batches of 8 tiles
// (loads of a batch in flight together).  The 8 Lagrange right-hand sides ride
// along transposed (y_J^T = r_J^T L_JJ^{-T}, r_{J+t}^T -= y_J^T X_t^T) in the
// block's Sint rows, and k_lg_solve finishes the backward sweep.
//
// k_lg_solve: blockdiag(A_II^{-1}) for any right-hand-side layout: one CTA per
// block, one warp per 8 right-hand sides; each tile column of the factor is
// staged once per CTA in shared memory (double-buffered cp.async) and shared
// by the warps; each warp keeps its window of PT+1 right-hand-side tiles in
// shared memory.
#include <algorithm>
#include "msfv_common.cuh"
#include "msfv_kernels.h"
#include "msfv_dmma.cuh"

namespace msfv {
namespace {

using namespace dmma;

constexpr int LGF_WARPS = 16;
constexpr int LGF_BATCH = 8;
constexpr int LGS_MAX_WARPS = 16;
constexpr int LGG_THREADS = 128;

__device__ __forceinline__ F2 lds2(const double* p) { return {p[0], p[1]}; }
__device__ __forceinline__ void sts2(double* p, const F2& f) { p[0] = f.x; p[1] = f.y; }
// C layout of the transpose of the row-major shared-memory tile at p
__device__ __forceinline__ F2 lds_t(const double* p, int lane) {
  const int m = lane >> 2, q = lane & 3;
  return {p[16 * q + m], p[16 * q + 8 + m]};
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// ------------------------------------------------------------------ factor

__global__ void __launch_bounds__(LGF_WARPS * 32)
k_lg_factor(Geo g, const double* __restrict__ w, double* __restrict__ LT, double* __restrict__ Sint,
            int* __restrict__ flags, int PT) {
  extern __shared__ __align__(16) double lsm[];
  const int jb = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int nI = g.nI, NTI = (nI + 7) >> 3;
  if (NTI == 0) return;
  double* Xs = lsm;                     // PT tiles: panel L_{J+t,J}
  double* Ys = Xs + (size_t)PT * 64;    // y_J^T
  double* Dg = Ys + 64;                 // diagonal tile
  double* Li = Dg + 64;                 // L_JJ^{-1}
  int* pairs = reinterpret_cast<int*>(Li + 64);   // (a << 16) | b, ordered by a then b
  const int npair = PT * (PT + 1) / 2;
  for (int k = tid; k < npair; k += nt) {
    int a = (int)((1.0 + sqrt(1.0 + 8.0 * k)) * 0.5);
    while (a * (a - 1) / 2 > k) --a;
    while ((a + 1) * a / 2 <= k) ++a;
    pairs[k] = (a << 16) | (k - a * (a - 1) / 2 + 1);
  }
  const size_t cstride = (size_t)(PT + 1) * 64;
  double* LTb = LT + (size_t)jb * NTI * cstride;
  double* Sb = Sint + (size_t)jb * 8 * nI;
  {
    double2* z2 = reinterpret_cast<double2*>(LTb);
    const size_t n2 = (size_t)NTI * cstride / 2;
    for (size_t i = tid; i < n2; i += nt) __stcg(z2 + i, make_double2(0.0, 0.0));
  }
  __syncthreads();
  // A_II band entries and the Lagrange right-hand sides -A_IB x_B (basis.py:537-551)
  {
    const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
    const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
    const bool has0 = jb == 0;
    const double s1 = g.ih1 * g.ih1, s2 = g.ih2 * g.ih2, s3 = g.ih3 * g.ih3;
    auto put = [&](int r, int c, double v) {
      __stcg(LTb + ((size_t)(c >> 3) * (PT + 1) + ((r >> 3) - (c >> 3))) * 64 + (r & 7) * 8 + (c & 7), v);
    };
    for (int a = tid; a < 8 * NTI; a += nt) {
      if (a >= nI) {
        put(a, a, 1.0);
        continue;
      }
      const int x = 1 + a % g.ni1, y = 1 + (a / g.ni1) % g.ni2, z = 1 + a / (g.ni1 * g.ni2);
      const long long I = X0 + x, J = Y0 + y, K = Z0 + z;
      const double kxm = w[ex_id(g, I - 1, J, K)] * s1, kxp = w[ex_id(g, I, J, K)] * s1;
      const double kym = w[ey_id(g, I, J - 1, K)] * s2, kyp = w[ey_id(g, I, J, K)] * s2;
      const double kzm = w[ez_id(g, I, J, K - 1)] * s3, kzp = w[ez_id(g, I, J, K)] * s3;
      put(a, a, ((((kxm + kxp) + kym) + kyp) + kzm) + kzp);
      if (x > 1) put(a, a - 1, -kxm);
      if (y > 1) put(a, a - g.ni1, -kym);
      if (z > 1) put(a, a - g.p, -kzm);
      double rhs[8];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) rhs[cc] = 0.0;
      auto add_nb = [&](int xx, int yy, int zz, double kc) {
        if (interior_index(g, xx, yy, zz) >= 0) return;
        if (has0 && xx == 0 && yy == 0 && zz == 0) return;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          rhs[cc] += kc * (g.bx ? skel_value(g, jb, cc, xx, yy, zz) : hat_corner(cc, xx, yy, zz, g.b1, g.b2, g.b3));
      };
      add_nb(x - 1, y, z, kxm); add_nb(x + 1, y, z, kxp);
      add_nb(x, y - 1, z, kym); add_nb(x, y + 1, z, kyp);
      add_nb(x, y, z - 1, kzm); add_nb(x, y, z + 1, kzp);
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) __stcg(Sb + (size_t)cc * nI + a, rhs[cc]);
    }
  }
  __syncthreads();

  const int m = lane >> 2, q2 = 2 * (lane & 3);
  // transposed right-hand-side tile I: element (corner m, row 8I + q2 + s)
  auto load_rt = [&](int I) -> F2 {
    const int a0 = 8 * I + q2;
    F2 v{0.0, 0.0};
    if (a0 < nI) v.x = __ldcg(Sb + (size_t)m * nI + a0);
    if (a0 + 1 < nI) v.y = __ldcg(Sb + (size_t)m * nI + a0 + 1);
    return v;
  };
  auto store_rt = [&](int I, const F2& v) {
    const int a0 = 8 * I + q2;
    if (a0 < nI) __stcg(Sb + (size_t)m * nI + a0, v.x);
    if (a0 + 1 < nI) __stcg(Sb + (size_t)m * nI + a0 + 1, v.y);
  };

  for (int J = 0; J < NTI; ++J) {
    const int ntj = min(PT, NTI - 1 - J);
    double* colJ = LTb + (size_t)J * cstride;
    // (a) diagonal tile: L_JJ (lanes = rows) and its inverse (lanes = columns)
    if (wid == 0) {
      for (int e = lane; e < 64; e += 32) Dg[e] = __ldcg(colJ + e);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (lane == k) {
          double d = Dg[k * 9];
          if (!(d > 0.0)) {
            atomicOr(flags, FLAG_LOCAL_NOT_SPD);
            d = 1.0;
          }
          Dg[k * 9] = sqrt(d);
        }
        __syncwarp();
        if (lane > k && lane < 8) Dg[lane * 8 + k] /= Dg[k * 9];
        __syncwarp();
        if (lane > k && lane < 8)
          for (int j = k + 1; j <= lane; ++j) Dg[lane * 8 + j] -= Dg[lane * 8 + k] * Dg[j * 8 + k];
        __syncwarp();
      }
      if (lane < 8) {
        const int j = lane;
        double xc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
          for (int k = 0; k < i; ++k)
            if (k >= j) s -= Dg[i * 8 + k] * xc[k];
          xc[i] = i < j ? 0.0 : s / Dg[i * 9];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) Li[i * 8 + j] = xc[i];
      }
      __syncwarp();
      for (int e = lane; e < 64; e += 32) __stcg(colJ + e, Li[e]);
    }
    __syncthreads();
    // (b) panel X_t = A_{J+t,J} L_JJ^{-T}; y_J^T = r_J^T L_JJ^{-T}
    {
      const F2 li = lds2(Li + lane * 2);
      for (int t = 1 + wid; t <= ntj; t += LGF_WARPS) {
        double* tp = colJ + (size_t)t * 64 + lane * 2;
        F2 x{0.0, 0.0};
        mma(x, ld2cg(tp), li);
        st2cg(tp, x);
        sts2(Xs + (t - 1) * 64 + lane * 2, x);
      }
      if (wid == LGF_WARPS - 1) {
        F2 y{0.0, 0.0};
        mma(y, load_rt(J), li);
        store_rt(J, y);
        sts2(Ys + lane * 2, y);
      }
    }
    __syncthreads();
    // (c) trailing window A_{J+a,J+b} -= X_a X_b^T and r_{J+t}^T -= y_J^T X_t^T
    {
      const int np = ntj * (ntj + 1) / 2;
      const int nwork = np + ntj;
      const F2 ny = neg(lds2(Ys + lane * 2));
      for (int k0 = wid * LGF_BATCH; k0 < nwork; k0 += LGF_WARPS * LGF_BATCH) {
        F2 c[LGF_BATCH];
        double* cp[LGF_BATCH];
        int ta[LGF_BATCH], tb[LGF_BATCH];
#pragma unroll
        for (int u = 0; u < LGF_BATCH; ++u) {
          const int k = k0 + u;
          cp[u] = nullptr;
          ta[u] = tb[u] = 0;
          if (k < np) {
            const int pr = pairs[k];
            ta[u] = pr >> 16;
            tb[u] = pr & 0xffff;
            cp[u] = LTb + ((size_t)(J + tb[u]) * (PT + 1) + (ta[u] - tb[u])) * 64 + lane * 2;
            c[u] = ld2cg(cp[u]);
          } else if (k < nwork) {
            ta[u] = k - np + 1;
            c[u] = load_rt(J + ta[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < LGF_BATCH; ++u) {
          const int k = k0 + u;
          if (k < np) {
            mma(c[u], neg(lds2(Xs + (ta[u] - 1) * 64 + lane * 2)), lds2(Xs + (tb[u] - 1) * 64 + lane * 2));
            st2cg(cp[u], c[u]);
          } else if (k < nwork) {
            mma(c[u], ny, lds2(Xs + (ta[u] - 1) * 64 + lane * 2));
            store_rt(J + ta[u], c[u]);
          }
        }
      }
    }
    __syncthreads();
  }
}

size_t lg_factor_smem(int PT) {
  return ((size_t)PT * 64 + 3 * 64) * sizeof(double) + (size_t)PT * (PT + 1) / 2 * sizeof(int) + 16;
}

// ------------------------------------------------------------------- solve

// MODE 0: node fields F[node][nrhs]; 1: compact interior fields
// [slot][a][nrhs] (blist[slot] = block, or slot itself); 2: the block's Sint
// rows [corner][a] (8 right-hand sides).  fwd = 0: the input already holds
// y = L^{-1} r (backward sweep only).  out may alias rhs.
template <int MODE>
__global__ void __launch_bounds__(LGS_MAX_WARPS * 32) k_lg_solve(Geo g, const double* __restrict__ LT, const double* rhs, double* out, int nrhs,
                           const int* __restrict__ blist, int PT, int fwd) {
  extern __shared__ __align__(16) double ssm[];
  const int slot = blockIdx.x;
  const int jb = (MODE == 1 && blist) ? blist[slot] : slot;
  const int nw = blockDim.x >> 5;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nI = g.nI, NTI = (nI + 7) >> 3;
  if (NTI == 0) return;
  const int cs = (PT + 1) * 64;
  double* Lb = ssm;                           // 2 tile columns
  double* win = Lb + 2 * cs + (size_t)wid * cs;
  const int s0 = (blockIdx.y * nw + wid) * 8;
  const bool active = s0 < nrhs;
  const double* LTb = LT + (size_t)jb * NTI * cs;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int m = lane >> 2, q2 = 2 * (lane & 3);
  const int col = s0 + m;
  auto addr = [&](int a) -> long long {
    if (a >= nI || col >= nrhs) return -1;
    if (MODE == 2) return ((long long)jb * 8 + col) * nI + a;
    if (MODE == 1) return ((long long)slot * nI + a) * nrhs + col;
    const int x = 1 + a % g.ni1, y = 1 + (a / g.ni1) % g.ni2, z = 1 + a / (g.ni1 * g.ni2);
    return node_id(g, X0 + x, Y0 + y, Z0 + z) * nrhs + col;
  };
  auto load_t = [&](const double* src, int I) -> F2 {
    F2 v{0.0, 0.0};
    const long long p0 = addr(8 * I + q2), p1 = addr(8 * I + q2 + 1);
    if (p0 >= 0) v.x = src[p0];
    if (p1 >= 0) v.y = src[p1];
    return v;
  };
  auto store_t = [&](int I, const F2& v) {
    const long long p0 = addr(8 * I + q2), p1 = addr(8 * I + q2 + 1);
    if (p0 >= 0) out[p0] = v.x;
    if (p1 >= 0) out[p1] = v.y;
  };
  auto fetch_col = [&](int J, int buf) {
    const double* src = LTb + (size_t)J * cs;
    double* dst = Lb + buf * cs;
    const int nv = (J + PT < NTI ? PT + 1 : NTI - J) * 32;   // 16-byte chunks of the valid tiles
    for (int i = tid; i < nv; i += blockDim.x) cp16(dst + 2 * i, src + 2 * i);
    cp_commit();
  };
  if (fwd) {
    if (active)
      for (int I = 0; I <= PT && I < NTI; ++I) sts2(win + (size_t)I * 64 + lane * 2, load_t(rhs, I));
    fetch_col(0, 0);
    for (int J = 0; J < NTI; ++J) {
      cp_wait_all();
      __syncthreads();
      if (J + 1 < NTI) fetch_col(J + 1, (J + 1) & 1);
      const double* L = Lb + (J & 1) * cs;
      if (active) {
        const int ntj = min(PT, NTI - 1 - J);
        double* wJ = win + (size_t)(J % (PT + 1)) * 64 + lane * 2;
        F2 y{0.0, 0.0};
        mma(y, lds2(wJ), lds2(L + lane * 2));          // y_J^T = r_J^T L_JJ^{-T}
        store_t(J, y);
        const F2 ny = neg(y);
        for (int t = 1; t <= ntj; ++t) {
          double* wt = win + (size_t)((J + t) % (PT + 1)) * 64 + lane * 2;
          F2 r = lds2(wt);
          mma(r, ny, lds2(L + t * 64 + lane * 2));    // r_{J+t}^T -= y_J^T X_t^T
          sts2(wt, r);
        }
        if (J + PT + 1 < NTI) sts2(wJ, load_t(rhs, J + PT + 1));
      }
    }
    cp_wait_all();
    __syncthreads();
    // make the y tiles written through `out` visible to the backward reads
    __threadfence_block();
  }
  const double* ysrc = fwd ? out : rhs;
  fetch_col(NTI - 1, (NTI - 1) & 1);
  for (int J = NTI - 1; J >= 0; --J) {
    cp_wait_all();
    __syncthreads();
    if (J > 0) fetch_col(J - 1, (J - 1) & 1);
    const double* L = Lb + (J & 1) * cs;
    if (active) {
      const int ntj = min(PT, NTI - 1 - J);
      F2 acc = load_t(ysrc, J);
      for (int t = 1; t <= ntj; ++t)
        mma(acc, neg(lds2(win + (size_t)((J + t) % (PT + 1)) * 64 + lane * 2)), lds_t(L + t * 64, lane));
      F2 x{0.0, 0.0};
      mma(x, acc, lds_t(L, lane));                     // x_J^T = (.) L_JJ^{-1}
      sts2(win + (size_t)(J % (PT + 1)) * 64 + lane * 2, x);
      store_t(J, x);
    }
  }
  cp_wait_all();
}

// ------------------------------------------------------- local Galerkin block

// Kloc[jb] = sum over the block's owned edges of (w_e/h^2) dS_e dS_e^T
// (forward.py:101-102 restricted to the block), fixed-order reduction.
__global__ void __launch_bounds__(LGG_THREADS)
k_lg_galerkin(Geo g, const double* __restrict__ w, const double* __restrict__ Sint, double* __restrict__ Kloc) {
  __shared__ double red[36][LGG_THREADS];
  const int jb = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const bool has0 = jb == 0;
  const double* Sb = Sint + (size_t)jb * 8 * g.nI;
  const int lx = (bi == g.nb1 - 1), ly = (bj == g.nb2 - 1), lz = (bk == g.nb3 - 1);
  const int ox = g.b1 * (g.b2 + ly) * (g.b3 + lz);
  const int oy = (g.b1 + lx) * g.b2 * (g.b3 + lz);
  const int oz = (g.b1 + lx) * (g.b2 + ly) * g.b3;
  double acc[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) acc[k] = 0.0;
  for (int f = tid; f < ox + oy + oz; f += nt) {
    int ax, x, y, z;
    double kc;
    if (f < ox) {
      ax = 0; x = f % g.b1; const int r = f / g.b1; y = r % (g.b2 + ly); z = r / (g.b2 + ly);
      kc = w[ex_id(g, X0 + x, Y0 + y, Z0 + z)] * g.ih1 * g.ih1;
    } else if (f < ox + oy) {
      ax = 1; const int qq = f - ox; x = qq % (g.b1 + lx); const int r = qq / (g.b1 + lx); y = r % g.b2; z = r / g.b2;
      kc = w[ey_id(g, X0 + x, Y0 + y, Z0 + z)] * g.ih2 * g.ih2;
    } else {
      ax = 2; const int qq = f - ox - oy; x = qq % (g.b1 + lx); const int r = qq / (g.b1 + lx); y = r % (g.b2 + ly);
      z = r / (g.b2 + ly);
      kc = w[ez_id(g, X0 + x, Y0 + y, Z0 + z)] * g.ih3 * g.ih3;
    }
    const int x1 = x + (ax == 0), y1 = y + (ax == 1), z1 = z + (ax == 2);
    const bool n0 = has0 && x == 0 && y == 0 && z == 0;
    double ds[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc)
      ds[cc] = s_value(g, Sb, jb, cc, x1, y1, z1, false) - s_value(g, Sb, jb, cc, x, y, z, n0);
#pragma unroll
    for (int c1 = 0; c1 < 8; ++c1) {
      const double kd = kc * ds[c1];
#pragma unroll
      for (int c2 = 0; c2 <= c1; ++c2) acc[c1 * (c1 + 1) / 2 + c2] += kd * ds[c2];
    }
  }
#pragma unroll
  for (int k = 0; k < 36; ++k) red[k][tid] = acc[k];
  __syncthreads();
  for (int width = nt / 2; width > 0; width >>= 1) {
    if (tid < width)
#pragma unroll
      for (int k = 0; k < 36; ++k) red[k][tid] += red[k][tid + width];
    __syncthreads();
  }
  if (tid < 36) {
    int c1 = 0;
    while ((c1 + 1) * (c1 + 2) / 2 <= tid) ++c1;
    const int c2 = tid - c1 * (c1 + 1) / 2;
    Kloc[(size_t)jb * 64 + c1 * 8 + c2] = red[tid][0];
    Kloc[(size_t)jb * 64 + c2 * 8 + c1] = red[tid][0];
  }
}

template <int MODE>
cudaError_t launch_solve_mode(const Geo& g, const double* LT, const double* rhs, double* out, int nrhs,
                              const int* blist, int nslots, int fwd, cudaStream_t st) {
  const int PT = lg_band(g);
  const size_t cs = (size_t)(PT + 1) * 64 * sizeof(double);
  const int chunks = (nrhs + 7) / 8;
  int nw = (int)std::min<size_t>(LGS_MAX_WARPS, (227 * 1024 - 2 * cs) / cs);
  nw = std::max(1, std::min(nw, chunks));
  const size_t smem = (2 + (size_t)nw) * cs;
  cudaError_t e = cudaFuncSetAttribute(k_lg_solve<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)nslots, (unsigned)((chunks + nw - 1) / nw));
  k_lg_solve<MODE><<<grid, nw * 32, smem, st>>>(g, LT, rhs, out, nrhs, blist, PT, fwd);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

// same as tc_band: the two paths share the factor layout, so either solve
// kernel can consume either factor
int lg_band(const Geo& g) {
  const int nti = (g.nI + 7) / 8;
  if (nti == 0) return 0;
  return std::min((g.p + 7) / 8, nti - 1);
}

bool lg_supported(const Geo& g) {
  const int PT = lg_band(g);
  const size_t cs = (size_t)(PT + 1) * 64 * sizeof(double);
  return PT <= LG_MAX_PT && lg_factor_smem(PT) <= 200 * 1024 && 3 * cs <= 227 * 1024;
}

size_t lg_factor_doubles(const Geo& g) {
  const size_t NTI = (g.nI + 7) / 8;
  return (size_t)g.nbl * NTI * (lg_band(g) + 1) * 64;
}

cudaError_t launch_basis_lg(const Geo& g, const double* w, double* LT, double* Sint, double* Kloc, int* flags,
                            cudaStream_t st) {
  if (g.nbl == 0) return cudaSuccess;
  const int PT = lg_band(g);
  const size_t smem = lg_factor_smem(PT);
  cudaError_t e = cudaFuncSetAttribute(k_lg_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_lg_factor<<<g.nbl, LGF_WARPS * 32, smem, st>>>(g, w, LT, Sint, flags, PT);
  count_launches(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // backward sweeps: Sint holds y = L^{-1} R transposed
  if ((e = launch_solve_mode<2>(g, LT, Sint, Sint, 8, nullptr, g.nbl, 0, st)) != cudaSuccess) return e;
  k_lg_galerkin<<<g.nbl, LGG_THREADS, 0, st>>>(g, w, Sint, Kloc);
  count_launches(1);
  return cudaGetLastError();
}

// Local Galerkin blocks from the edge weights and the basis values (hats or
// the bound reduced-boundary table on the skeleton), any local solver.
cudaError_t launch_lg_galerkin(const Geo& g, const double* w, const double* Sint, double* Kloc, cudaStream_t st) {
  if (g.nbl == 0) return cudaSuccess;
  k_lg_galerkin<<<g.nbl, LGG_THREADS, 0, st>>>(g, w, Sint, Kloc);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_block_solve_lg(const Geo& g, const double* LT, const double* rhs, double* out, int nrhs,
                                  cudaStream_t st, const int* blist, int nlist, int compact) {
  if (g.nI == 0 || nrhs == 0 || (compact && nlist == 0)) return cudaSuccess;
  if (compact) return launch_solve_mode<1>(g, LT, rhs, out, nrhs, blist, nlist, 1, st);
  return launch_solve_mode<0>(g, LT, rhs, out, nrhs, nullptr, g.nbl, 1, st);
}

}  // namespace msfv
