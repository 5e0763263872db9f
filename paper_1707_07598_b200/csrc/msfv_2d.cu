// 2D adaptive MSFV path (BASELINE.json configs 1-2: 64^2 / 256^2 cells,
// 8^2 / 16^2-cell blocks).  The reference package is 3D only;
// this is the same algorithm with d = 2: bilinear Lagrange
// hats, 5-point fine stencil A = G^T diag(C sigma) G with C = V/2 per touching
// cell, 9-point Galerkin coarse operator, node 0 pinned.
//
// The 2D problems are small (<= 66k nodes, 256 blocks, k <= 289 coarse
// unknowns), so the kernels are plain CUDA with block-level parallelism:
//  * k2_basis: one CTA per coarse block factors its interior operator A_II
//    ((b-1)^2 nodes, half band b-1) as a band Cholesky in shared memory and
//    solves the 4 Lagrange right-hand sides (basis.py:537-563);
//  * k2_galerkin: one warp per block reduces K_j = sum_owned (w/h^2) dS dS^T
//    (4x4) with a fixed-order butterfly; k2_assemble gathers the 9-point
//    coarse band in block order (deterministic, no atomics);
//  * k2_coarse_factor / k2_coarse_solve: one CTA band Cholesky of A_k in
//    shared memory (forward.py:117-131, dpotrf) and the banded solves;
//  * node/edge/cell field kernels for the sensitivity products
//    (forward.py:224-281): prolong S Y, restrict S^T X, A X, G X, G^T (a o c),
//    C sigma dm, C^T sigma e, blockdiag(A_II^-1) X, and a CSR SpMM for the
//    survey matrices.
// Fields are row-major [pinned node][rhs], pinned node id = full id - 1.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "msfv.h"
#include "msfv_kernels.h"

namespace msfv2 {

struct G2 {
  int n1, n2, b1, b2, nb1, nb2, ni1, ni2, nI, p, nbl, kx, ky, kc, pc;
  long long Nn, n, Nm, Ex, E;
  double h1, h2, ih1, ih2, ih1s, ih2s, hv, ib1, ib2;
};

__device__ __forceinline__ double hat1(int d, double ib) {
  const double v = 1.0 - fabs((double)d) * ib;
  return v > 0.0 ? v : 0.0;
}
__device__ __forceinline__ long long xe(const G2& g, int i, int j) { return i + (long long)g.n1 * j; }
__device__ __forceinline__ long long ye(const G2& g, int i, int j) { return g.Ex + i + (long long)(g.n1 + 1) * j; }
__device__ __forceinline__ long long nid(const G2& g, int i, int j) { return i + (long long)(g.n1 + 1) * j; }

// value of coarse column `c` (corner cx, cy of block (bi, bj)) at full node (i, j)
// of the block's closure: S_I on the interior, hats on the block boundary, 0 at
// the pinned node
__device__ __forceinline__ double sval(const G2& g, const double* __restrict__ Sb, int bi, int bj, int c, int i,
                                       int j) {
  if (i == 0 && j == 0) return 0.0;
  const int x = i - bi * g.b1, y = j - bj * g.b2;
  if (x > 0 && x < g.b1 && y > 0 && y < g.b2) {
    const int blk = bi + g.nb1 * bj;
    return Sb[((size_t)blk * 4 + c) * g.nI + (x - 1) + g.ni1 * (y - 1)];
  }
  return hat1(x - (c & 1) * g.b1, g.ib1) * hat1(y - (c >> 1) * g.b2, g.ib2);
}

// ------------------------------------------------------------- operator

__global__ void k2_sigma(G2 g, const double* __restrict__ m, double* __restrict__ sigma, int* flags) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.Nm) return;
  const double v = m[c];
  if (!isfinite(v)) atomicOr(flags, MSFV_FLAG_NONFINITE);
  sigma[c] = exp(v);
}
// w = C sigma (operators.py:136): V/2 per touching cell, ascending cell order
__global__ void k2_edges(G2 g, const double* __restrict__ s, double* __restrict__ w) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= g.E) return;
  double acc = 0.0;
  if (e < g.Ex) {
    const int i = (int)(e % g.n1), j = (int)(e / g.n1);
    if (j > 0) acc += g.hv * s[i + (long long)g.n1 * (j - 1)];
    if (j < g.n2) acc += g.hv * s[i + (long long)g.n1 * j];
  } else {
    const long long f = e - g.Ex;
    const int i = (int)(f % (g.n1 + 1)), j = (int)(f / (g.n1 + 1));
    if (i > 0) acc += g.hv * s[(i - 1) + (long long)g.n1 * j];
    if (i < g.n1) acc += g.hv * s[i + (long long)g.n1 * j];
  }
  w[e] = acc;
}

// ---------------------------------------------------------------- basis

constexpr int B2_THREADS = 128;

// band Cholesky of the nI x nI band (row-major, P1 = p + 1 entries per row,
// L[i][d] = A(i, i - d)) in shared memory; tab holds the (r, c) pairs of the
// trailing triangle.  Returns with L in place.
__device__ void band_potrf(double* L, int nI, int p, const short2* tab, int* flags, double* sinv) {
  const int P1 = p + 1, npair = p * (p + 1) / 2;
  for (int j = 0; j < nI; ++j) {
    if (threadIdx.x == 0) {
      double d = L[j * P1];
      if (!(d > 0.0)) {
        atomicOr(flags, MSFV_FLAG_LOCAL_NOT_SPD);
        d = 1.0;
      }
      const double l = sqrt(d);
      L[j * P1] = l;
      *sinv = 1.0 / l;
    }
    __syncthreads();
    const double inv = *sinv;
    for (int t = threadIdx.x; t < p; t += blockDim.x) {
      const int i = j + 1 + t;
      if (i < nI) L[i * P1 + t + 1] *= inv;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < npair; t += blockDim.x) {
      const int r = tab[t].x, c = tab[t].y;   // i = j + r, k = j + c, 1 <= c <= r <= p
      const int i = j + r;
      if (i < nI) L[i * P1 + (r - c)] -= L[i * P1 + r] * L[(j + c) * P1 + c];
    }
    __syncthreads();
  }
}
// X (nI x nr, row-major, in shared memory) <- L^-T L^-1 X
__device__ void band_solve(const double* L, int nI, int p, double* X, int nr) {
  const int P1 = p + 1;
  for (int j = 0; j < nI; ++j) {
    for (int s = threadIdx.x; s < nr; s += blockDim.x) X[j * nr + s] /= L[j * P1];
    __syncthreads();
    for (int t = threadIdx.x; t < p * nr; t += blockDim.x) {
      const int r = 1 + t / nr, s = t % nr, i = j + r;
      if (i < nI) X[i * nr + s] -= L[i * P1 + r] * X[j * nr + s];
    }
    __syncthreads();
  }
  for (int j = nI - 1; j >= 0; --j) {
    for (int s = threadIdx.x; s < nr; s += blockDim.x) X[j * nr + s] /= L[j * P1];
    __syncthreads();
    for (int t = threadIdx.x; t < p * nr; t += blockDim.x) {
      const int r = 1 + t / nr, s = t % nr, i = j - r;
      if (i >= 0) X[i * nr + s] -= L[j * P1 + r] * X[j * nr + s];
    }
    __syncthreads();
  }
}
// Same solve, one warp per right-hand-side column (half band p <= 31): lane r
// keeps row j + r (forward) / j - r (backward) of the column in a register
// window that slides by one shuffle per pivot, so a pivot costs one
// broadcast, one FMA and one shift instead of two CTA barriers.
// rinv[j] = 1 / L(j, j).
__device__ void band_solve_warp(const double* __restrict__ L, const double* __restrict__ rinv, int nI, int p,
                                double* __restrict__ X, int nr) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int P1 = p + 1;
  for (int s = wid; s < nr; s += nw) {
    // forward: the entering row and 1/L(j,j) are prefetched one pivot ahead
    double v = (lane <= p && lane < nI) ? X[lane * nr + s] : 0.0;
    double nx = (lane == p && p + 1 < nI) ? X[(p + 1) * nr + s] : 0.0;
    double ri = rinv[0];
    for (int j = 0; j < nI; ++j) {
      const double nx2 = (lane == p && j + 2 + p < nI) ? X[(j + 2 + p) * nr + s] : 0.0;
      const double ri2 = j + 1 < nI ? rinv[j + 1] : 0.0;
      const double lv = (lane >= 1 && lane <= p && j + lane < nI) ? L[(j + lane) * P1 + lane] : 0.0;
      const double x = __shfl_sync(FULL, v, 0) * ri;
      if (lane == 0) X[j * nr + s] = x;
      v = fma(-lv, x, v);
      v = __shfl_down_sync(FULL, v, 1);
      if (lane == p) v = nx;
      nx = nx2;
      ri = ri2;
    }
    __syncwarp();
    v = (lane <= p && nI - 1 - lane >= 0) ? X[(nI - 1 - lane) * nr + s] : 0.0;
    nx = (lane == p && nI - 2 - p >= 0) ? X[(nI - 2 - p) * nr + s] : 0.0;
    ri = rinv[nI - 1];
    for (int j = nI - 1; j >= 0; --j) {
      const double nx2 = (lane == p && j - 2 - p >= 0) ? X[(j - 2 - p) * nr + s] : 0.0;
      const double ri2 = j >= 1 ? rinv[j - 1] : 0.0;
      const double lv = (lane >= 1 && lane <= p && j - lane >= 0) ? L[j * P1 + lane] : 0.0;
      const double x = __shfl_sync(FULL, v, 0) * ri;
      if (lane == 0) X[j * nr + s] = x;
      v = fma(-lv, x, v);
      v = __shfl_down_sync(FULL, v, 1);
      if (lane == p) v = nx;
      nx = nx2;
      ri = ri2;
    }
    __syncwarp();
  }
  __syncthreads();
}
__device__ void fill_pairs(short2* tab, int p) {
  for (int t = threadIdx.x; t < p * (p + 1) / 2; t += blockDim.x) {
    int r = 1, rem = t;
    while (rem >= r) {
      rem -= r;
      ++r;
    }
    tab[t] = make_short2((short)r, (short)(rem + 1));
  }
}

// One CTA per block: A_II band + Lagrange rhs, band Cholesky, 4 solves.
// Factor -> fac[block][nI][P1]; S_I -> Sb[block][corner][nI].
__global__ void __launch_bounds__(B2_THREADS) k2_basis(G2 g, const double* __restrict__ w, double* __restrict__ fac,
                                                      double* __restrict__ Sb, int* flags) {
  extern __shared__ __align__(16) double sm2[];
  const int blk = blockIdx.x;
  const int nI = g.nI, p = g.p, P1 = p + 1;
  double* L = sm2;                    // nI * P1
  double* X = L + nI * P1;            // nI * 4
  double* rinv = X + nI * 4;          // nI
  double* sinv = rinv + nI;
  short2* tab = reinterpret_cast<short2*>(sinv + 2);
  const int bi = blk % g.nb1, bj = blk / g.nb1, X0 = bi * g.b1, Y0 = bj * g.b2;
  fill_pairs(tab, p);
  for (int a = threadIdx.x; a < nI; a += blockDim.x) {
    const int x = 1 + a % g.ni1, y = 1 + a / g.ni1, i = X0 + x, j = Y0 + y;
    const double kxm = w[xe(g, i - 1, j)] * g.ih1s, kxp = w[xe(g, i, j)] * g.ih1s;
    const double kym = w[ye(g, i, j - 1)] * g.ih2s, kyp = w[ye(g, i, j)] * g.ih2s;
    double* row = L + a * P1;
    for (int d = 0; d < P1; ++d) row[d] = 0.0;
    row[0] = ((kxm + kxp) + kym) + kyp;
    if (x > 1) row[1] = -kxm;
    if (y > 1) row[p] += -kym;          // p == ni1 (p == 1 merges with the x neighbour)
    // rhs = -A_IB x_B: boundary neighbours carry the hats (basis.py:548)
    for (int c = 0; c < 4; ++c) {
      const int cx = (c & 1) * g.b1, cy = (c >> 1) * g.b2;
      double v = 0.0;
      if (x == 1) v += kxm * (hat1(x - 1 - cx, g.ib1) * hat1(y - cy, g.ib2));
      if (x == g.ni1) v += kxp * (hat1(x + 1 - cx, g.ib1) * hat1(y - cy, g.ib2));
      if (y == 1) v += kym * (hat1(x - cx, g.ib1) * hat1(y - 1 - cy, g.ib2));
      if (y == g.ni2) v += kyp * (hat1(x - cx, g.ib1) * hat1(y + 1 - cy, g.ib2));
      X[a * 4 + c] = v;
    }
  }
  __syncthreads();
  band_potrf(L, nI, p, tab, flags, sinv);
  for (int a = threadIdx.x; a < nI; a += blockDim.x) rinv[a] = 1.0 / L[a * P1];
  __syncthreads();
  if (p <= 31)
    band_solve_warp(L, rinv, nI, p, X, 4);
  else
    band_solve(L, nI, p, X, 4);
  for (int t = threadIdx.x; t < nI * P1; t += blockDim.x) fac[(size_t)blk * nI * P1 + t] = L[t];
  for (int t = threadIdx.x; t < nI * 4; t += blockDim.x) {
    const int a = t >> 2, c = t & 3;
    Sb[((size_t)blk * 4 + c) * nI + a] = X[t];
  }
}

// blockdiag(A_II^-1) on the interior rows of a node field (nr columns);
// skeleton rows of `out` are zeroed (basis.py:339-353)
__global__ void __launch_bounds__(512) k2_interior_solve(G2 g, const double* __restrict__ fac,
                                                               const double* __restrict__ rhs,
                                                               double* __restrict__ out, int nr) {
  extern __shared__ __align__(16) double sm2[];
  const int blk = blockIdx.x;
  const int nI = g.nI, P1 = g.p + 1;
  double* L = sm2;
  double* X = L + nI * P1;
  double* rinv = X + nI * nr;
  const int bi = blk % g.nb1, bj = blk / g.nb1, X0 = bi * g.b1, Y0 = bj * g.b2;
  for (int t = threadIdx.x; t < nI * P1; t += blockDim.x) L[t] = fac[(size_t)blk * nI * P1 + t];
  for (int t = threadIdx.x; t < nI * nr; t += blockDim.x) {
    const int a = t / nr, s = t % nr;
    const long long node = nid(g, X0 + 1 + a % g.ni1, Y0 + 1 + a / g.ni1) - 1;
    X[t] = rhs[node * nr + s];
  }
  __syncthreads();
  for (int a = threadIdx.x; a < nI; a += blockDim.x) rinv[a] = 1.0 / L[a * P1];
  __syncthreads();
  if (g.p <= 31)
    band_solve_warp(L, rinv, nI, g.p, X, nr);
  else
    band_solve(L, nI, g.p, X, nr);
  for (int t = threadIdx.x; t < nI * nr; t += blockDim.x) {
    const int a = t / nr, s = t % nr;
    const long long node = nid(g, X0 + 1 + a % g.ni1, Y0 + 1 + a / g.ni1) - 1;
    out[node * nr + s] = X[t];
  }
}
__global__ void k2_zero_skeleton(G2 g, double* __restrict__ out, int nr) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.n * nr) return;
  const long long node = t / nr + 1;
  const int i = (int)(node % (g.n1 + 1)), j = (int)(node / (g.n1 + 1));
  if (i % g.b1 == 0 || j % g.b2 == 0) out[t] = 0.0;
}

// ------------------------------------------------------------- Galerkin

// Edge ownership: x-edges (i, j) with X0 <= i < X0 + b1, Y0 <= j < Y0 + b2
// (+ the top row for the last block row); y-edges with X0 <= i < X0 + b1
// (+ the right column for the last block column), Y0 <= j < Y0 + b2.
__global__ void k2_galerkin(G2 g, const double* __restrict__ w, const double* __restrict__ Sb,
                            double* __restrict__ Kloc) {
  const int lane = threadIdx.x & 31;
  const int blk = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (blk >= g.nbl) return;
  const int bi = blk % g.nb1, bj = blk / g.nb1, X0 = bi * g.b1, Y0 = bj * g.b2;
  const int nyx = g.b2 + (bj == g.nb2 - 1), nxy = g.b1 + (bi == g.nb1 - 1);
  const int nxe = g.b1 * nyx, nye = nxy * g.b2;
  double K[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) K[t] = 0.0;
  for (int e = lane; e < nxe + nye; e += 32) {
    int i0, j0, i1, j1;
    double k;
    if (e < nxe) {
      i0 = X0 + e % g.b1;
      j0 = Y0 + e / g.b1;
      i1 = i0 + 1;
      j1 = j0;
      k = w[xe(g, i0, j0)] * g.ih1s;
    } else {
      const int f = e - nxe;
      i0 = X0 + f % nxy;
      j0 = Y0 + f / nxy;
      i1 = i0;
      j1 = j0 + 1;
      k = w[ye(g, i0, j0)] * g.ih2s;
    }
    double d[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) d[c] = sval(g, Sb, bi, bj, c, i1, j1) - sval(g, Sb, bi, bj, c, i0, j0);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) K[a * 4 + b] += k * d[a] * d[b];
  }
#pragma unroll
  for (int t = 0; t < 16; ++t)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) K[t] += __shfl_xor_sync(0xffffffffu, K[t], o);
  if (lane < 16) {
    double v = K[0];
#pragma unroll
    for (int t = 1; t < 16; ++t)
      if (lane == t) v = K[t];
    Kloc[(size_t)blk * 16 + lane] = v;
  }
}

// Lower band of A_k in coarse lexicographic order: Ab[c][d] = A_k(c, c - d),
// d = 0..pc (pc = kx + 1); block contributions summed in ascending block order;
// `shift` is added on the diagonal (forward.py:119-129 fallback)
__global__ void k2_assemble(G2 g, const double* __restrict__ Kloc, double shift, double* __restrict__ Ab) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int P1 = g.pc + 1;
  if (t >= (long long)g.kc * P1) return;
  const int c1 = (int)(t / P1), d = (int)(t % P1), c2 = c1 - d;
  double v = 0.0;
  if (c2 >= 0) {
    const int x1 = c1 % g.kx, y1 = c1 / g.kx, x2 = c2 % g.kx, y2 = c2 / g.kx;
    if (abs(x1 - x2) <= 1 && abs(y1 - y2) <= 1) {
      for (int bj = max(y1, y2) - 1; bj <= min(y1, y2); ++bj)
        for (int bi = max(x1, x2) - 1; bi <= min(x1, x2); ++bi) {
          if (bi < 0 || bj < 0 || bi >= g.nb1 || bj >= g.nb2) continue;
          const int l1 = (x1 - bi) + 2 * (y1 - bj), l2 = (x2 - bi) + 2 * (y2 - bj);
          v += Kloc[(size_t)(bi + g.nb1 * bj) * 16 + l1 * 4 + l2];
        }
    }
    if (d == 0) v += shift;
  }
  Ab[t] = v;
}

// one CTA: band Cholesky of A_k (k x (pc+1)) in shared memory -> Lk
__global__ void k2_coarse_factor(G2 g, const double* __restrict__ Ab, double* __restrict__ Lk, int* flags) {
  extern __shared__ __align__(16) double sm2[];
  const int P1 = g.pc + 1;
  double* L = sm2;
  double* sinv = L + (size_t)g.kc * P1;
  short2* tab = reinterpret_cast<short2*>(sinv + 2);
  fill_pairs(tab, g.pc);
  for (int t = threadIdx.x; t < g.kc * P1; t += blockDim.x) L[t] = Ab[t];
  __syncthreads();
  const int npair = g.pc * (g.pc + 1) / 2;
  for (int j = 0; j < g.kc; ++j) {
    if (threadIdx.x == 0) {
      double d = L[j * P1];
      if (!(d > 0.0)) {
        atomicOr(flags, MSFV_FLAG_COARSE_NOT_SPD);
        d = 1.0;
      }
      const double l = sqrt(d);
      L[j * P1] = l;
      *sinv = 1.0 / l;
    }
    __syncthreads();
    const double inv = *sinv;
    for (int t = threadIdx.x; t < g.pc; t += blockDim.x) {
      const int i = j + 1 + t;
      if (i < g.kc) L[i * P1 + t + 1] *= inv;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < npair; t += blockDim.x) {
      const int r = tab[t].x, c = tab[t].y, i = j + r;
      if (i < g.kc) L[i * P1 + (r - c)] -= L[i * P1 + r] * L[(j + c) * P1 + c];
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < g.kc * P1; t += blockDim.x) Lk[t] = L[t];
}
// one CTA: X (k x nr, global) <- A_k^-1 X
__global__ void k2_coarse_solve(G2 g, const double* __restrict__ Lk, double* __restrict__ X, int nr) {
  extern __shared__ __align__(16) double sm2[];
  const int P1 = g.pc + 1;
  double* L = sm2;
  double* Y = L + (size_t)g.kc * P1;
  double* rinv = Y + (size_t)g.kc * nr;
  for (int t = threadIdx.x; t < g.kc * P1; t += blockDim.x) L[t] = Lk[t];
  for (int t = threadIdx.x; t < g.kc * nr; t += blockDim.x) Y[t] = X[t];
  __syncthreads();
  for (int a = threadIdx.x; a < g.kc; a += blockDim.x) rinv[a] = 1.0 / L[a * P1];
  __syncthreads();
  if (g.pc <= 31)
    band_solve_warp(L, rinv, g.kc, g.pc, Y, nr);
  else
    band_solve(L, g.kc, g.pc, Y, nr);
  for (int t = threadIdx.x; t < g.kc * nr; t += blockDim.x) X[t] = Y[t];
}

// ------------------------------------------------------ node/edge fields

// out = S Y (n x nr) from Y (k x nr)
__global__ void k2_prolong(G2 g, const double* __restrict__ Sb, const double* __restrict__ Y, double* __restrict__ out,
                           int nr) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.n * nr) return;
  const long long node = t / nr + 1;
  const int s = (int)(t % nr);
  const int i = (int)(node % (g.n1 + 1)), j = (int)(node / (g.n1 + 1));
  const int bi = min(i / g.b1, g.nb1 - 1), bj = min(j / g.b2, g.nb2 - 1);
  double v = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int cidx = (bi + (c & 1)) + g.kx * (bj + (c >> 1));
    v += sval(g, Sb, bi, bj, c, i, j) * Y[(size_t)cidx * nr + s];
  }
  out[t] = v;
}
// out[c][s] = sum_i S(i, c) X[i][s] over the support of column c, ascending node order
__global__ void k2_restrict(G2 g, const double* __restrict__ Sb, const double* __restrict__ X,
                            double* __restrict__ out, int nr) {
  const long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= (long long)g.kc * nr) return;
  const int c = (int)(t / nr), s = (int)(t % nr);
  const int cx = c % g.kx, cy = c / g.kx;
  const int i0 = max(cx * g.b1 - g.b1 + 1, 0), i1 = min(cx * g.b1 + g.b1 - 1, g.n1);
  const int j0 = max(cy * g.b2 - g.b2 + 1, 0), j1 = min(cy * g.b2 + g.b2 - 1, g.n2);
  const int wi = i1 - i0 + 1, tot = wi * (j1 - j0 + 1);
  double v = 0.0;
  for (int q = lane; q < tot; q += 32) {
    const int i = i0 + q % wi, j = j0 + q / wi;
    {
      if (i == 0 && j == 0) continue;
      // the block of c's support holding (i, j) (on a shared line either works)
      const int bi = i < cx * g.b1 ? cx - 1 : (i > cx * g.b1 ? cx : (cx < g.nb1 ? cx : cx - 1));
      const int bj = j < cy * g.b2 ? cy - 1 : (j > cy * g.b2 ? cy : (cy < g.nb2 ? cy : cy - 1));
      const int lc = (cx - bi) + 2 * (cy - bj);
      const double sv = sval(g, Sb, bi, bj, lc, i, j);
      if (sv != 0.0) v += sv * X[(nid(g, i, j) - 1) * nr + s];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) out[t] = v;
}
// out = A X (pinned node fields): sum over the 4 incident edges of k (x_n - x_m)
__global__ void k2_apply_A(G2 g, const double* __restrict__ w, const double* __restrict__ X, double* __restrict__ out,
                           int nr) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.n * nr) return;
  const long long node = t / nr + 1;
  const int s = (int)(t % nr);
  const int i = (int)(node % (g.n1 + 1)), j = (int)(node / (g.n1 + 1));
  const double xc = X[t];
  auto xv = [&](int a, int b) -> double {
    const long long q = nid(g, a, b);
    return q == 0 ? 0.0 : X[(q - 1) * nr + s];
  };
  double v = 0.0;
  if (i > 0) v += w[xe(g, i - 1, j)] * g.ih1s * (xc - xv(i - 1, j));
  if (i < g.n1) v += w[xe(g, i, j)] * g.ih1s * (xc - xv(i + 1, j));
  if (j > 0) v += w[ye(g, i, j - 1)] * g.ih2s * (xc - xv(i, j - 1));
  if (j < g.n2) v += w[ye(g, i, j)] * g.ih2s * (xc - xv(i, j + 1));
  out[t] = v;
}
// out (E x nr) = G_p X (forward differences / h, node 0 = 0)
__global__ void k2_grad(G2 g, const double* __restrict__ X, double* __restrict__ out, int nr) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.E * nr) return;
  const long long e = t / nr;
  const int s = (int)(t % nr);
  long long a, b;
  double ih;
  if (e < g.Ex) {
    const int i = (int)(e % g.n1), j = (int)(e / g.n1);
    a = nid(g, i, j);
    b = nid(g, i + 1, j);
    ih = g.ih1;
  } else {
    const long long f = e - g.Ex;
    const int i = (int)(f % (g.n1 + 1)), j = (int)(f / (g.n1 + 1));
    a = nid(g, i, j);
    b = nid(g, i, j + 1);
    ih = g.ih2;
  }
  const double xa = a == 0 ? 0.0 : X[(a - 1) * nr + s], xb = b == 0 ? 0.0 : X[(b - 1) * nr + s];
  out[t] = (xb - xa) * ih;
}
// out (n x nr) = G_p^T (a o c): a (E x nr), c (E) or null
__global__ void k2_gradT(G2 g, const double* __restrict__ a, const double* __restrict__ c, double* __restrict__ out,
                         int nr) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.n * nr) return;
  const long long node = t / nr + 1;
  const int s = (int)(t % nr);
  const int i = (int)(node % (g.n1 + 1)), j = (int)(node / (g.n1 + 1));
  auto term = [&](long long e) -> double { return a[e * nr + s] * (c ? c[e] : 1.0); };
  double v = 0.0;
  if (i > 0) v += term(xe(g, i - 1, j)) * g.ih1;
  if (i < g.n1) v -= term(xe(g, i, j)) * g.ih1;
  if (j > 0) v += term(ye(g, i, j - 1)) * g.ih2;
  if (j < g.n2) v -= term(ye(g, i, j)) * g.ih2;
  out[t] = v;
}
// c = C (sigma o dm) (the J v edge conductance change, forward.py:259)
__global__ void k2_edge_avg(G2 g, const double* __restrict__ sigma, const double* __restrict__ dm,
                            double* __restrict__ c) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= g.E) return;
  double acc = 0.0;
  if (e < g.Ex) {
    const int i = (int)(e % g.n1), j = (int)(e / g.n1);
    if (j > 0) { const long long q = i + (long long)g.n1 * (j - 1); acc += g.hv * (sigma[q] * dm[q]); }
    if (j < g.n2) { const long long q = i + (long long)g.n1 * j; acc += g.hv * (sigma[q] * dm[q]); }
  } else {
    const long long f = e - g.Ex;
    const int i = (int)(f % (g.n1 + 1)), j = (int)(f / (g.n1 + 1));
    if (i > 0) { const long long q = (i - 1) + (long long)g.n1 * j; acc += g.hv * (sigma[q] * dm[q]); }
    if (i < g.n1) { const long long q = i + (long long)g.n1 * j; acc += g.hv * (sigma[q] * dm[q]); }
  }
  c[e] = acc;
}
// g = -(C diag(sigma))^T sum_s e[:, s]  (forward.py:281)
__global__ void k2_cell_adj(G2 g, const double* __restrict__ sigma, const double* __restrict__ e,
                            double* __restrict__ out, int nr) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= g.Nm) return;
  const int i = (int)(q % g.n1), j = (int)(q / g.n1);
  const long long es[4] = {xe(g, i, j), xe(g, i, j + 1), ye(g, i, j), ye(g, i + 1, j)};
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    double se = 0.0;
    for (int s = 0; s < nr; ++s) se += e[es[t] * nr + s];
    acc += g.hv * se;
  }
  out[q] = -(sigma[q] * acc);
}
// out[r][s] = beta * out[r][s] + sum_k val[k] X[col[k]][s]  (CSR rows)
__global__ void k2_spmm(long long nrows, const long long* __restrict__ ptr, const int* __restrict__ col,
                        const double* __restrict__ val, const double* __restrict__ X, int nr, double beta,
                        double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nrows * nr) return;
  const long long r = t / nr;
  const int s = (int)(t % nr);
  double v = 0.0;
  for (long long k = ptr[r]; k < ptr[r + 1]; ++k) v += val[k] * X[(long long)col[k] * nr + s];
  out[t] = beta == 0.0 ? v : beta * out[t] + v;
}
// out = alpha * a + b (elementwise), b may be null
__global__ void k2_axpby(long long N, double alpha, const double* __restrict__ a, const double* __restrict__ b,
                         double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= N) return;
  out[t] = alpha * a[t] + (b ? b[t] : 0.0);
}
// out = a o b + c o d + e o f (elementwise, c..f may be null)
__global__ void k2_fma3(long long N, const double* __restrict__ a, const double* __restrict__ b,
                        const double* __restrict__ c, const double* __restrict__ d, const double* __restrict__ e,
                        const double* __restrict__ f, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= N) return;
  double v = a[t] * b[t];
  if (c) v += c[t] * d[t];
  if (e) v += e[t] * f[t];
  out[t] = v;
}

}  // namespace msfv2

// ================================================================ C-ABI

using namespace msfv2;

struct msfv2d_plan {
  G2 g;
};

namespace {
inline unsigned nblk(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }
size_t basis_smem(const G2& g) {
  return ((size_t)g.nI * (g.p + 1) + (size_t)g.nI * 5 + 2) * sizeof(double) +
         (size_t)(g.p * (g.p + 1) / 2 + 2) * sizeof(short2);
}
size_t coarse_smem(const G2& g, int nr) {
  const size_t band = (size_t)g.kc * (g.pc + 1);
  const size_t a = (band + 2) * sizeof(double) + (size_t)(g.pc * (g.pc + 1) / 2 + 2) * sizeof(short2);
  const size_t b = (band + (size_t)g.kc * nr) * sizeof(double);
  return a > b ? a : b;
}
int cuda_rc(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return MSFV_OK;
  return msfv::set_error(MSFV_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
int launched(const char* what, long long n = 1) {
  msfv::count_launches(n);
  return cuda_rc(cudaGetLastError(), what);
}
int smem_attr(const void* fn, size_t bytes, const char* what) {
  if (bytes > 227 * 1024)
    return msfv::set_error(MSFV_UNSUPPORTED, std::string(what) + ": working set exceeds shared memory");
  return cuda_rc(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), what);
}
}  // namespace

extern "C" {

MSFV_API int msfv2d_plan_create(const int32_t* cells, const double* h, const int32_t* blocks, msfv2d_plan** out) {
  if (!cells || !h || !blocks || !out) return msfv::set_error(MSFV_SHAPE, "null argument");
  G2 g{};
  g.n1 = cells[0];
  g.n2 = cells[1];
  g.b1 = blocks[0];
  g.b2 = blocks[1];
  if (g.n1 < 1 || g.n2 < 1 || g.b1 < 2 || g.b2 < 2 || g.n1 % g.b1 || g.n2 % g.b2)
    return msfv::set_error(MSFV_SHAPE, "block size must divide the cell count (blocks >= 2 cells)");
  g.nb1 = g.n1 / g.b1;
  g.nb2 = g.n2 / g.b2;
  g.ni1 = g.b1 - 1;
  g.ni2 = g.b2 - 1;
  g.nI = g.ni1 * g.ni2;
  g.p = g.ni1;
  g.nbl = g.nb1 * g.nb2;
  g.kx = g.nb1 + 1;
  g.ky = g.nb2 + 1;
  g.kc = g.kx * g.ky;
  g.pc = g.kx + 1;
  g.Nn = (long long)(g.n1 + 1) * (g.n2 + 1);
  g.n = g.Nn - 1;
  g.Nm = (long long)g.n1 * g.n2;
  g.Ex = (long long)g.n1 * (g.n2 + 1);
  g.E = g.Ex + (long long)(g.n1 + 1) * g.n2;
  g.h1 = h[0];
  g.h2 = h[1];
  g.ih1 = 1.0 / g.h1;
  g.ih2 = 1.0 / g.h2;
  g.ih1s = g.ih1 * g.ih1;
  g.ih2s = g.ih2 * g.ih2;
  g.hv = 0.5 * (g.h1 * g.h2);
  g.ib1 = 1.0 / g.b1;
  g.ib2 = 1.0 / g.b2;
  if (basis_smem(g) > 227 * 1024 || coarse_smem(g, 1) > 227 * 1024)
    return msfv::set_error(MSFV_UNSUPPORTED, "2D block or coarse band exceeds shared memory");
  auto* p = new msfv2d_plan{g};
  *out = p;
  return MSFV_OK;
}
MSFV_API void msfv2d_plan_destroy(msfv2d_plan* p) { delete p; }
MSFV_API int msfv2d_plan_info(const msfv2d_plan* p, int64_t* info, int32_t n) {
  if (!p || !info || n < MSFV2D_INFO_COUNT) return msfv::set_error(MSFV_SHAPE, "info buffer");
  const G2& g = p->g;
  info[MSFV2D_INFO_NN] = g.Nn;
  info[MSFV2D_INFO_N] = g.n;
  info[MSFV2D_INFO_NCELLS] = g.Nm;
  info[MSFV2D_INFO_NEDGES] = g.E;
  info[MSFV2D_INFO_NBLOCKS] = g.nbl;
  info[MSFV2D_INFO_NI] = g.nI;
  info[MSFV2D_INFO_K] = g.kc;
  info[MSFV2D_INFO_FACTOR_DOUBLES] = (int64_t)g.nbl * g.nI * (g.p + 1);
  info[MSFV2D_INFO_BAND_DOUBLES] = (int64_t)g.kc * (g.pc + 1);
  return MSFV_OK;
}
MSFV_API int msfv2d_operator(const msfv2d_plan* p, const double* m, double* sigma, double* w, int32_t* flags,
                             void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  const G2& g = p->g;
  auto st = (cudaStream_t)stream;
  k2_sigma<<<nblk(g.Nm), 256, 0, st>>>(g, m, sigma, flags);
  k2_edges<<<nblk(g.E), 256, 0, st>>>(g, sigma, w);
  return launched("2d operator", 2);
}
MSFV_API int msfv2d_basis(const msfv2d_plan* p, const double* w, double* factor, double* Sb, double* Kloc,
                          int32_t* flags, void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  const G2& g = p->g;
  auto st = (cudaStream_t)stream;
  const size_t sm = basis_smem(g);
  int rc = smem_attr((const void*)k2_basis, sm, "2d basis");
  if (rc) return rc;
  k2_basis<<<g.nbl, B2_THREADS, sm, st>>>(g, w, factor, Sb, flags);
  k2_galerkin<<<nblk(g.nbl, 4), 128, 0, st>>>(g, w, Sb, Kloc);
  return launched("2d basis", 2);
}
MSFV_API int msfv2d_galerkin(const msfv2d_plan* p, const double* Kloc, double shift, double* Ab, void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  const G2& g = p->g;
  k2_assemble<<<nblk((long long)g.kc * (g.pc + 1)), 256, 0, (cudaStream_t)stream>>>(g, Kloc, shift, Ab);
  return launched("2d galerkin");
}
MSFV_API int msfv2d_coarse_factor(const msfv2d_plan* p, const double* Ab, double* Lk, int32_t* flags, void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  const G2& g = p->g;
  const size_t sm = ((size_t)g.kc * (g.pc + 1) + 2) * sizeof(double) + (size_t)(g.pc * (g.pc + 1) / 2 + 2) * sizeof(short2);
  int rc = smem_attr((const void*)k2_coarse_factor, sm, "2d coarse factor");
  if (rc) return rc;
  k2_coarse_factor<<<1, 256, sm, (cudaStream_t)stream>>>(g, Ab, Lk, flags);
  return launched("2d coarse factor");
}
MSFV_API int msfv2d_coarse_solve(const msfv2d_plan* p, const double* Lk, double* X, int32_t nrhs, void* stream) {
  if (!p || nrhs < 1) return msfv::set_error(MSFV_SHAPE, "null plan / nrhs");
  const G2& g = p->g;
  const size_t sm = ((size_t)g.kc * (g.pc + 2) + (size_t)g.kc * nrhs) * sizeof(double);
  int rc = smem_attr((const void*)k2_coarse_solve, sm, "2d coarse solve");
  if (rc) return rc;
  k2_coarse_solve<<<1, 512, sm, (cudaStream_t)stream>>>(g, Lk, X, nrhs);
  return launched("2d coarse solve");
}
MSFV_API int msfv2d_interior_solve(const msfv2d_plan* p, const double* factor, const double* rhs, double* out,
                                   int32_t nrhs, void* stream) {
  if (!p || nrhs < 1) return msfv::set_error(MSFV_SHAPE, "null plan / nrhs");
  const G2& g = p->g;
  auto st = (cudaStream_t)stream;
  const size_t sm = ((size_t)g.nI * (g.p + 2) + (size_t)g.nI * nrhs) * sizeof(double);
  int rc = smem_attr((const void*)k2_interior_solve, sm, "2d interior solve");
  if (rc) return rc;
  k2_zero_skeleton<<<nblk(g.n * nrhs), 256, 0, st>>>(g, out, nrhs);
  k2_interior_solve<<<g.nbl, 512, sm, st>>>(g, factor, rhs, out, nrhs);
  return launched("2d interior solve", 2);
}
MSFV_API int msfv2d_prolong(const msfv2d_plan* p, const double* Sb, const double* Y, double* out, int32_t nrhs,
                            void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  k2_prolong<<<nblk(p->g.n * nrhs), 256, 0, (cudaStream_t)stream>>>(p->g, Sb, Y, out, nrhs);
  return launched("2d prolong");
}
MSFV_API int msfv2d_restrict(const msfv2d_plan* p, const double* Sb, const double* X, double* out, int32_t nrhs,
                             void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  k2_restrict<<<nblk((long long)p->g.kc * nrhs * 32, 128), 128, 0, (cudaStream_t)stream>>>(p->g, Sb, X, out, nrhs);
  return launched("2d restrict");
}
MSFV_API int msfv2d_apply_A(const msfv2d_plan* p, const double* w, const double* X, double* out, int32_t nrhs,
                            void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  k2_apply_A<<<nblk(p->g.n * nrhs), 256, 0, (cudaStream_t)stream>>>(p->g, w, X, out, nrhs);
  return launched("2d apply A");
}
MSFV_API int msfv2d_grad(const msfv2d_plan* p, const double* X, double* out, int32_t nrhs, void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  k2_grad<<<nblk(p->g.E * nrhs), 256, 0, (cudaStream_t)stream>>>(p->g, X, out, nrhs);
  return launched("2d grad");
}
MSFV_API int msfv2d_gradT(const msfv2d_plan* p, const double* a, const double* c, double* out, int32_t nrhs,
                          void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  k2_gradT<<<nblk(p->g.n * nrhs), 256, 0, (cudaStream_t)stream>>>(p->g, a, c, out, nrhs);
  return launched("2d gradT");
}
MSFV_API int msfv2d_edge_average(const msfv2d_plan* p, const double* sigma, const double* dm, double* c,
                                 void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  k2_edge_avg<<<nblk(p->g.E), 256, 0, (cudaStream_t)stream>>>(p->g, sigma, dm, c);
  return launched("2d edge average");
}
MSFV_API int msfv2d_cell_adjoint(const msfv2d_plan* p, const double* sigma, const double* e, double* out,
                                 int32_t nrhs, void* stream) {
  if (!p) return msfv::set_error(MSFV_SHAPE, "null plan");
  k2_cell_adj<<<nblk(p->g.Nm), 256, 0, (cudaStream_t)stream>>>(p->g, sigma, e, out, nrhs);
  return launched("2d cell adjoint");
}
MSFV_API int msfv2d_spmm(int64_t nrows, const int64_t* ptr, const int32_t* col, const double* val, const double* X,
                         int32_t nrhs, double beta, double* out, void* stream) {
  k2_spmm<<<nblk(nrows * nrhs), 256, 0, (cudaStream_t)stream>>>(nrows, (const long long*)ptr, col, val, X, nrhs, beta,
                                                                 out);
  return launched("2d spmm");
}
MSFV_API int msfv2d_axpby(int64_t n, double alpha, const double* a, const double* b, double* out, void* stream) {
  k2_axpby<<<nblk(n), 256, 0, (cudaStream_t)stream>>>(n, alpha, a, b, out);
  return launched("2d axpby");
}
MSFV_API int msfv2d_fma3(int64_t n, const double* a, const double* b, const double* c, const double* d,
                         const double* e, const double* f, double* out, void* stream) {
  k2_fma3<<<nblk(n), 256, 0, (cudaStream_t)stream>>>(n, a, b, c, d, e, f, out);
  return launched("2d fma3");
}

}  // extern "C"
