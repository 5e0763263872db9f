// Coarse (Galerkin) system: assembly of A_k = P^T A P from the per-block 8x8
// contributions, banded tiled Cholesky and multi-RHS triangular solves.
//
// Reference: forward.py:101-142 forms A_k densely and calls LAPACK dpotrf
// (cho_factor) for k <= 5000, SuperLU above.  A_k couples coarse nodes only
// within a 27-point stencil, so in lexicographic coarse order its half
// bandwidth is pc = (nb1+1)(nb2+1) + (nb1+1) + 1 and Cholesky fill stays
// inside that band: the banded factorization below is the same Cholesky
// factor as the reference's dense one, computed without the zero blocks.
//
// Layout: lower band in TB x TB tiles, tile column J holds tiles (J+t, J),
// t = 0..PT, each row-major:  Ak[((J*(PT+1) + t)*TB + r)*TB + q].
// Rows >= kc (padding) are identity.  Dinv[J] = inverse of the diagonal tile
// of L (computed after the factorization) turns the triangular solves into
// tile products.
#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace msfv {

constexpr int TB = COARSE_TB;

__device__ __forceinline__ double* tile(double* A, const Geo& g, int J, int t) {
  return A + ((size_t)J * (g.PT + 1) + t) * TB * TB;
}
__device__ __forceinline__ const double* tile(const double* A, const Geo& g, int J, int t) {
  return A + ((size_t)J * (g.PT + 1) + t) * TB * TB;
}

// Thread per (coarse row c, lower neighbour o): A_k[c][c'] = sum over blocks
// having both as corners (fixed order) of Kloc, + shift on the diagonal.
__global__ void k_coarse_assemble(Geo g, const double* __restrict__ Kloc, double shift, double* __restrict__ Ak) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long tot = (long long)g.NT * TB * 14;
  if (t >= tot) return;
  int o = (int)(t % 14);
  int c = (int)(t / 14);
  if (c >= g.kc) {
    if (o == 0) {
      int J = c / TB, r = c % TB;
      tile(Ak, g, J, 0)[r * TB + r] = 1.0;    // padding rows: identity
    }
    return;
  }
  // enumerate the 14 lexicographically-lower offsets (dz, dy, dx) <= 0
  int dz, dy, dx;
  if (o < 9) { dz = -1; dy = o / 3 - 1; dx = o % 3 - 1; }
  else if (o < 12) { dz = 0; dy = -1; dx = (o - 9) - 1; }
  else { dz = 0; dy = 0; dx = (o - 12) - 1; }
  int ci = c % (g.nb1 + 1), r = c / (g.nb1 + 1), cj = r % (g.nb2 + 1), ck = r / (g.nb2 + 1);
  int di = ci + dx, dj = cj + dy, dk = ck + dz;
  if (di < 0 || dj < 0 || dk < 0 || di > g.nb1 || dj > g.nb2 || dk > g.nb3) return;
  int c2 = coarse_of(g, di, dj, dk);
  double v = 0.0;
  for (int bk = max(ck, dk) - 1; bk <= min(ck, dk); ++bk) {
    if (bk < 0 || bk >= g.nb3) continue;
    for (int bj = max(cj, dj) - 1; bj <= min(cj, dj); ++bj) {
      if (bj < 0 || bj >= g.nb2) continue;
      for (int bi = max(ci, di) - 1; bi <= min(ci, di); ++bi) {
        if (bi < 0 || bi >= g.nb1) continue;
        int l1 = (ci - bi) + 2 * (cj - bj) + 4 * (ck - bk);
        int l2 = (di - bi) + 2 * (dj - bj) + 4 * (dk - bk);
        v += Kloc[(size_t)block_of(g, bi, bj, bk) * 64 + l1 * 8 + l2];
      }
    }
  }
  if (c2 == c) v += shift;
  int I = c / TB, J = c2 / TB;
  tile(Ak, g, J, I - J)[(c % TB) * TB + (c2 % TB)] = v;
}

__global__ void k_coarse_diag(Geo g, const double* __restrict__ Ak, double* __restrict__ diag) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.kc) return;
  diag[c] = tile(Ak, g, c / TB, 0)[(c % TB) * TB + (c % TB)];
}

// Panel of tile column J: Cholesky of the diagonal tile, its inverse Dinv_J,
// then L_{J+t,J} = A_{J+t,J} Dinv_J^T for the tiles below it.
__global__ void __launch_bounds__(256) k_coarse_panel(Geo g, int J, double* __restrict__ Ak, double* __restrict__ Dinv,
                                                      int* __restrict__ flags) {
  __shared__ double D[TB][TB + 1];
  __shared__ double Di[TB][TB + 1];
  __shared__ double As[TB][TB + 1];
  const int tid = threadIdx.x, nt = blockDim.x;
  double* Dg = tile(Ak, g, J, 0);
  for (int t = tid; t < TB * TB; t += nt) D[t / TB][t % TB] = Dg[t];
  __syncthreads();
  for (int jc = 0; jc < TB; ++jc) {
    double d = D[jc][jc];
    if (!(d > 0.0)) {
      if (tid == 0) atomicOr(flags, FLAG_COARSE_NOT_SPD);
      d = 1.0;
    }
    const double piv = sqrt(d), inv = 1.0 / piv;
    for (int r = jc + 1 + tid; r < TB; r += nt) D[r][jc] *= inv;
    __syncthreads();
    if (tid == 0) D[jc][jc] = piv;
    const int m = TB - 1 - jc;
    for (int f = tid; f < m * m; f += nt) {
      int r = jc + 1 + f / m, q = jc + 1 + f % m;
      if (q <= r) D[r][q] -= D[r][jc] * D[q][jc];
    }
    __syncthreads();
  }
  for (int t = tid; t < TB * TB; t += nt) {
    int r = t / TB, q = t % TB;
    Dg[t] = q <= r ? D[r][q] : 0.0;
  }
  // inverse of the lower-triangular diagonal tile, thread per column
  if (tid < TB) {
    const int c = tid;
    double x[TB];
#pragma unroll
    for (int r = 0; r < TB; ++r) {
      double v = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int m2 = 0; m2 < r; ++m2) v -= D[r][m2] * x[m2];
      x[r] = (r < c) ? 0.0 : v / D[r][r];
    }
#pragma unroll
    for (int r = 0; r < TB; ++r) Di[r][c] = x[r];
  }
  __syncthreads();
  {
    double* out = Dinv + (size_t)J * TB * TB;
    for (int t = tid; t < TB * TB; t += nt) out[t] = Di[t / TB][t % TB];
  }
  const int pt = min(g.PT, g.NT - 1 - J);
  for (int tt = 1; tt <= pt; ++tt) {
    double* A = tile(Ak, g, J, tt);
    for (int t = tid; t < TB * TB; t += nt) As[t / TB][t % TB] = A[t];
    __syncthreads();
    for (int t = tid; t < TB * TB; t += nt) {
      int r = t / TB, q = t % TB;
      double v = 0.0;
      for (int m2 = 0; m2 <= q; ++m2) v += As[r][m2] * Di[q][m2];
      A[t] = v;
    }
    __syncthreads();
  }
}

// Trailing update of tile column J: A_{J+t1, J+t2} -= L_{J+t1,J} L_{J+t2,J}^T.
__global__ void __launch_bounds__(256) k_coarse_update(Geo g, int J, double* __restrict__ Ak) {
  __shared__ double As[TB][TB + 1], Bs[TB][TB + 1];
  int f = blockIdx.x;
  int t1 = (int)((1.0 + sqrt(1.0 + 8.0 * f)) * 0.5);
  while (t1 * (t1 - 1) / 2 > f) --t1;
  while ((t1 + 1) * t1 / 2 <= f) ++t1;
  int t2 = f - t1 * (t1 - 1) / 2 + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double* A = tile(Ak, g, J, t1);
  const double* B = tile(Ak, g, J, t2);
  for (int t = tid; t < TB * TB; t += nt) { As[t / TB][t % TB] = A[t]; Bs[t / TB][t % TB] = B[t]; }
  __syncthreads();
  double* C = tile(Ak, g, J + t2, t1 - t2);
  for (int t = tid; t < TB * TB; t += nt) {
    int r = t / TB, q = t % TB;
    double v = 0.0;
#pragma unroll 8
    for (int m2 = 0; m2 < TB; ++m2) v += As[r][m2] * Bs[q][m2];
    C[t] -= v;
  }
}

// Forward then backward substitution with the banded tiled factor for RC
// right-hand sides per CTA.  X is [kc][nrhs] row-major.  Forward is
// right-looking (X_{J+t} -= L_{J+t,J} y_J straight in global memory, read back
// by the same CTA); backward keeps the last PT+1 solved tiles of x in a
// shared-memory ring so the transposed tile products read only L from L2.
template <int RC>
__global__ void __launch_bounds__(256) k_coarse_trsv(Geo g, const double* __restrict__ Lk, const double* __restrict__ Dinv,
                                                     double* __restrict__ X, int nrhs) {
  extern __shared__ double tsm[];
  double* Xs = tsm;                        // [TB][RC]
  double* acc = Xs + TB * RC;              // [TB][RC]
  double* win = acc + TB * RC;             // [PT+1][TB][RC]
  const int tid = threadIdx.x, nt = blockDim.x;
  const int s0 = blockIdx.x * RC;
  const int ns = min(RC, nrhs - s0);
  const int W = g.PT + 1;
  // ---------------- forward
  for (int J = 0; J < g.NT; ++J) {
    for (int t = tid; t < TB * RC; t += nt) {
      int r = t / RC, s = t % RC, row = J * TB + r;
      Xs[t] = (s < ns && row < g.kc) ? X[(size_t)row * nrhs + s0 + s] : 0.0;
    }
    __syncthreads();
    const double* Di = Dinv + (size_t)J * TB * TB;
    for (int t = tid; t < TB * RC; t += nt) {
      int r = t / RC, s = t % RC;
      const double* drow = Di + r * TB;
      double v = 0.0;
#pragma unroll 8
      for (int q = 0; q < TB; ++q) v += drow[q] * Xs[q * RC + s];   // Dinv upper part is zero
      acc[t] = v;
      int row = J * TB + r;
      if (s < ns && row < g.kc) X[(size_t)row * nrhs + s0 + s] = v;
    }
    __syncthreads();
    const int pt = min(g.PT, g.NT - 1 - J);
    for (int t = tid; t < pt * TB * RC; t += nt) {
      int tt = 1 + t / (TB * RC), rem = t % (TB * RC), r = rem / RC, s = rem % RC;
      int row = (J + tt) * TB + r;
      if (s >= ns || row >= g.kc) continue;
      const double* L = tile(Lk, g, J, tt) + r * TB;
      double v = 0.0;
#pragma unroll 8
      for (int q = 0; q < TB; ++q) v += L[q] * acc[q * RC + s];
      X[(size_t)row * nrhs + s0 + s] -= v;
    }
    __syncthreads();
  }
  // ---------------- backward
  for (int J = g.NT - 1; J >= 0; --J) {
    const int pt = min(g.PT, g.NT - 1 - J);
    for (int t = tid; t < TB * RC; t += nt) {
      int q = t / RC, s = t % RC, row = J * TB + q;
      double v = (s < ns && row < g.kc) ? X[(size_t)row * nrhs + s0 + s] : 0.0;
      for (int tt = 1; tt <= pt; ++tt) {
        const double* L = tile(Lk, g, J, tt);
        const double* xw = win + (size_t)((J + tt) % W) * TB * RC;
#pragma unroll 8
        for (int r = 0; r < TB; ++r) v -= L[r * TB + q] * xw[r * RC + s];
      }
      acc[t] = v;
    }
    __syncthreads();
    const double* Di = Dinv + (size_t)J * TB * TB;
    double* xo = win + (size_t)(J % W) * TB * RC;
    for (int t = tid; t < TB * RC; t += nt) {
      int r = t / RC, s = t % RC, row = J * TB + r;
      double v = 0.0;
      for (int q = r; q < TB; ++q) v += Di[q * TB + r] * acc[q * RC + s];
      if (row >= g.kc || s >= ns) v = 0.0;
      xo[t] = v;
      if (s < ns && row < g.kc) X[(size_t)row * nrhs + s0 + s] = v;
    }
    __syncthreads();
  }
}

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_coarse_assemble(const Geo& g, const double* Kloc, double shift, double* Ak, cudaStream_t st) {
  size_t bytes = (size_t)g.NT * (g.PT + 1) * TB * TB * sizeof(double);
  cudaError_t e = cudaMemsetAsync(Ak, 0, bytes, st);
  if (e != cudaSuccess) return e;
  long long tot = (long long)g.NT * TB * 14;
  k_coarse_assemble<<<nblk(tot, 256), 256, 0, st>>>(g, Kloc, shift, Ak);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_coarse_diag(const Geo& g, const double* Ak, double* diag, cudaStream_t st) {
  k_coarse_diag<<<nblk(g.kc, 256), 256, 0, st>>>(g, Ak, diag);
  count_launches(1);
  return cudaGetLastError();
}

// Dinv lives right after the tiles in the same allocation.
cudaError_t launch_coarse_factor(const Geo& g, double* Ak, int* flags, cudaStream_t st) {
  double* Dinv = Ak + (size_t)g.NT * (g.PT + 1) * TB * TB;
  for (int J = 0; J < g.NT; ++J) {
    k_coarse_panel<<<1, 256, 0, st>>>(g, J, Ak, Dinv, flags);
    count_launches(1);
    int pt = g.PT < g.NT - 1 - J ? g.PT : g.NT - 1 - J;
    int npairs = pt * (pt + 1) / 2;
    if (npairs > 0) {
      k_coarse_update<<<npairs, 256, 0, st>>>(g, J, Ak);
      count_launches(1);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_coarse_solve(const Geo& g, const double* Lk, double* X, int nrhs, cudaStream_t st) {
  if (nrhs == 0) return cudaSuccess;
  const double* Dinv = Lk + (size_t)g.NT * (g.PT + 1) * TB * TB;
  constexpr int RC = 4;
  size_t smem = ((size_t)2 + g.PT + 1) * TB * RC * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_coarse_trsv<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_coarse_trsv<RC><<<nblk(nrhs, RC), 256, smem, st>>>(g, Lk, Dinv, X, nrhs);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
