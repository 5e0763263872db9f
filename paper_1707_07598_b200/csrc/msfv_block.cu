// Fine-grid and per-block kernels of the MSFV forward + gradient path.
//
//   k_sigma / k_edge_weights   sigma = exp(m), w = C sigma        operators.py:23-28,136
//   k_basis                    per-block A_II band Cholesky, 8 hat RHS, local
//                              Galerkin block of P^T A P         basis.py:511-563, forward.py:101-102
//   k_block_solve              blockdiag(A_II^-1) on interiors   basis.py:339-353
//   k_residual                 alpha*src + beta*(A_wt X) on interiors  forward.py:243,278
//   k_prolong                  S Y on every node                 forward.py:143,241,277
//   k_restrict_op / gather     S^T (A_w1 X1 + A_w2 X2)           forward.py:266
//   k_cell_gradient            -sigma C^T sum_s(...)             forward.py:271-281 (compact form)
#include "msfv_common.cuh"
#include "msfv_kernels.h"

#include <atomic>

namespace msfv {

// ----------------------------------------------------------------- operator

__global__ void k_sigma(long long Nm, const double* __restrict__ m, const double* __restrict__ mul,
                        double* __restrict__ out, int* __restrict__ flags) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= Nm) return;
  double mc = m[c];
  double s = exp(mc);
  if (!isfinite(mc)) atomicOr(flags, FLAG_NONFINITE);
  else if (!(s > 0.0)) atomicOr(flags, FLAG_NONPOSITIVE);
  out[c] = mul ? s * mul[c] : s;
}

__global__ void k_mul(long long n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] * b[i];
}

// w_e = sum over touching cells of (V/4) * cv_c, cells in ascending cell
// index order exactly like the CSR product C @ sigma (operators.py:77-109,136).
__global__ void k_edge_weights(Geo g, const double* __restrict__ cv, double* __restrict__ w) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= g.E) return;
  int ax;
  int i, j, k;
  if (e < g.Ex) {
    ax = 0; decode3f(e, g.n1, g.r_n1, g.n2 + 1, g.r_n2p, i, j, k);
  } else if (e < g.Ex + g.Ey) {
    ax = 1; decode3f(e - g.Ex, g.n1 + 1, g.r_n1p, g.n2, g.r_n2, i, j, k);
  } else {
    ax = 2; decode3f(e - g.Ex - g.Ey, g.n1 + 1, g.r_n1p, g.n2 + 1, g.r_n2p, i, j, k);
  }
  double sum = 0.0;
  // transverse axes t1 < t2; outer loop on t2 (higher stride) gives ascending cell ids
  for (int d2 = -1; d2 <= 0; ++d2) {
    for (int d1 = -1; d1 <= 0; ++d1) {
      long long ci = i, cj = j, ck = k;
      if (ax == 0) { cj += d1; ck += d2; }
      else if (ax == 1) { ci += d1; ck += d2; }
      else { ci += d1; cj += d2; }
      if (ci < 0 || cj < 0 || ck < 0 || ci >= g.n1 || cj >= g.n2 || ck >= g.n3) continue;
      sum = __dadd_rn(sum, __dmul_rn(g.qv, cv[cell_id(g, ci, cj, ck)]));
    }
  }
  w[e] = sum;
}

// Same sums on a line grid: blockIdx.z = axis, blockIdx.y = the edge line
// (the two transverse indices), threads along x, so there is no index
// division and the four cell loads of a warp are coalesced rows.
constexpr int EW_THREADS = 128;
constexpr int EW_LINES = 4;
__global__ void __launch_bounds__(EW_THREADS * EW_LINES) k_edge_weights_lines(Geo g, const double* __restrict__ cv,
                                                                  double* __restrict__ w, int k0, int k1) {
  // planes k0 <= k <= k1 for x- and y-edges (node planes), k0 <= k < k1 for z-edges (cell planes)
  // EW_LINES lines per CTA (blockIdx.y * EW_LINES + threadIdx.y), threads along x
  const int ax = blockIdx.z;
  const int nx = ax == 0 ? g.n1 : g.n1 + 1;                  // edges along x in a line
  const int ny = ax == 1 ? g.n2 : g.n2 + 1;                  // lines per z plane
  const int line = blockIdx.y * EW_LINES + threadIdx.y;
  const int j = line % ny, k = k0 + line / ny;
  if (k > (ax == 2 ? k1 - 1 : k1) || k >= (ax == 2 ? g.n3 : g.n3 + 1)) return;
  const long long e0 = (ax == 0 ? 0 : (ax == 1 ? g.Ex : g.Ex + g.Ey)) + (long long)nx * (j + (long long)ny * k);
  for (int i = threadIdx.x; i < nx; i += EW_THREADS) {
    double sum = 0.0;
#pragma unroll
    for (int d2 = -1; d2 <= 0; ++d2) {
#pragma unroll
      for (int d1 = -1; d1 <= 0; ++d1) {
        int ci = i, cj = j, ck = k;
        if (ax == 0) { cj += d1; ck += d2; }
        else if (ax == 1) { ci += d1; ck += d2; }
        else { ci += d1; cj += d2; }
        if (ci < 0 || cj < 0 || ck < 0 || ci >= g.n1 || cj >= g.n2 || ck >= g.n3) continue;
        sum = __dadd_rn(sum, __dmul_rn(g.qv, __ldg(cv + cell_id(g, ci, cj, ck))));
      }
    }
    w[e0 + i] = sum;
  }
}

// Plane-tile form: CTA (tile of EWT_TY edge lines, node plane k) stages the
// premultiplied cell values (V/4) cv of cell planes k-1 and k, rows
// j0-1 .. j0+EWT_TY-1, columns -1 .. n1 (zero outside the mesh) in shared
// memory once, then forms the x- and y-edges of node plane k and the z-edges
// of cell plane k from it.  Same products and the same ascending-cell
// summation order as k_edge_weights (a skipped cell adds +0.0, which leaves
// the sum bit-identical).
constexpr int EWT_TY = 8, EWT_THREADS = 128, EWT_MAXW = 1024;
__global__ void __launch_bounds__(EWT_THREADS) k_edge_weights_tile(Geo g, const double* __restrict__ cv,
                                                                   double* __restrict__ w, int k0, int k1) {
  constexpr int NR = 2 * (EWT_TY + 1);         // staged rows: (cell plane k-1 | k) x (rows j0-1 .. j0+TY-1)
  extern __shared__ double q[];                 // [NR][W]
  const int n1 = g.n1, W = n1 + 2, RW = (EWT_TY + 1) * W;
  const int j0 = blockIdx.x * EWT_TY, k = k0 + blockIdx.y;
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    // all NR loads of a column in flight before the stores
    const int ci = c - 1;
    double v[NR];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
      const int dz = rr / (EWT_TY + 1), cj = j0 - 1 + rr - dz * (EWT_TY + 1), ck = k - 1 + dz;
      v[rr] = (ci >= 0 && ci < n1 && cj >= 0 && cj < g.n2 && ck >= 0 && ck < g.n3)
                  ? __ldg(cv + cell_id(g, ci, cj, ck)) : 0.0;
    }
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) q[rr * W + c] = __dmul_rn(g.qv, v[rr]);   // (V/4) * 0 = +0 outside
  }
  __syncthreads();
  auto Q = [&](int dz, int cj, int ci) { return q[dz * RW + (cj - j0 + 1) * W + ci + 1]; };
  // x-edges of node plane k: lines j in [j0, j0 + TY) ∩ [0, n2]
  {
    const int nl = min(EWT_TY, g.n2 + 1 - j0);
    double* out = w + (long long)n1 * (j0 + (long long)(g.n2 + 1) * k);
    for (int jj = 0; jj < nl; ++jj) {
      const int j = j0 + jj;
      for (int i = threadIdx.x; i < n1; i += blockDim.x) {
        double sum = 0.0;
        sum = __dadd_rn(sum, Q(0, j - 1, i));
        sum = __dadd_rn(sum, Q(0, j, i));
        sum = __dadd_rn(sum, Q(1, j - 1, i));
        sum = __dadd_rn(sum, Q(1, j, i));
        out[jj * n1 + i] = sum;
      }
    }
  }
  // y-edges of node plane k: lines j in [j0, j0 + TY) ∩ [0, n2)
  {
    const int nl = min(EWT_TY, g.n2 - j0);
    double* out = w + g.Ex + (long long)(n1 + 1) * (j0 + (long long)g.n2 * k);
    for (int jj = 0; jj < nl; ++jj) {
      const int j = j0 + jj;
      for (int i = threadIdx.x; i <= n1; i += blockDim.x) {
        double sum = 0.0;
        sum = __dadd_rn(sum, Q(0, j, i - 1));
        sum = __dadd_rn(sum, Q(0, j, i));
        sum = __dadd_rn(sum, Q(1, j, i - 1));
        sum = __dadd_rn(sum, Q(1, j, i));
        out[jj * (n1 + 1) + i] = sum;
      }
    }
  }
  // z-edges of cell plane k (k < k1, k < n3): lines j in [j0, j0 + TY) ∩ [0, n2]
  if (k < k1 && k < g.n3) {
    const int nl = min(EWT_TY, g.n2 + 1 - j0);
    double* out = w + g.Ex + g.Ey + (long long)(n1 + 1) * (j0 + (long long)(g.n2 + 1) * k);
    for (int jj = 0; jj < nl; ++jj) {
      const int j = j0 + jj;
      for (int i = threadIdx.x; i <= n1; i += blockDim.x) {
        double sum = 0.0;
        sum = __dadd_rn(sum, Q(1, j - 1, i - 1));
        sum = __dadd_rn(sum, Q(1, j - 1, i));
        sum = __dadd_rn(sum, Q(1, j, i - 1));
        sum = __dadd_rn(sum, Q(1, j, i));
        out[jj * (n1 + 1) + i] = sum;
      }
    }
  }
}

// ------------------------------------------------------------------ basis

// Closed-box edge weights of a block, staged in shared memory.
struct BoxW {
  double* wx; double* wy; double* wz;
  int b1, b2, b3;
  __device__ __forceinline__ double x(int i, int j, int k) const { return wx[i + b1 * (j + (b2 + 1) * k)]; }
  __device__ __forceinline__ double y(int i, int j, int k) const { return wy[i + (b1 + 1) * (j + b2 * k)]; }
  __device__ __forceinline__ double z(int i, int j, int k) const { return wz[i + (b1 + 1) * (j + (b2 + 1) * k)]; }
};

__device__ void load_box_weights(const Geo& g, const double* __restrict__ w, int X0, int Y0, int Z0,
                                 BoxW& bw) {
  for (int t = threadIdx.x; t < g.nwx; t += blockDim.x) {
    int i = t % g.b1, r = t / g.b1, j = r % (g.b2 + 1), k = r / (g.b2 + 1);
    bw.wx[t] = w[ex_id(g, X0 + i, Y0 + j, Z0 + k)];
  }
  for (int t = threadIdx.x; t < g.nwy; t += blockDim.x) {
    int i = t % (g.b1 + 1), r = t / (g.b1 + 1), j = r % g.b2, k = r / g.b2;
    bw.wy[t] = w[ey_id(g, X0 + i, Y0 + j, Z0 + k)];
  }
  for (int t = threadIdx.x; t < g.nwz; t += blockDim.x) {
    int i = t % (g.b1 + 1), r = t / (g.b1 + 1), j = r % (g.b2 + 1), k = r / (g.b2 + 1);
    bw.wz[t] = w[ez_id(g, X0 + i, Y0 + j, Z0 + k)];
  }
}

// One CTA per block: assemble the band of A_II and the 8 Lagrange right-hand
// sides (rhs = -A_IB x_B, basis.py:548), factor A_II = L L^T in shared memory
// (the reference's dense cho_factor, basis.py:275, restricted to the band where
// all fill lives), solve, write the interior basis values and both band forms
// of the factor, then accumulate this block's 8x8 Galerkin contribution
// sum_e w_e/h^2 dS_e dS_e^T over the edges it owns.
__global__ void __launch_bounds__(BASIS_THREADS)
k_basis(Geo g, const double* __restrict__ w, double* __restrict__ Lc, double* __restrict__ Lr,
        double* __restrict__ Sint, double* __restrict__ Kloc, int* __restrict__ flags) {
  extern __shared__ double sm[];
  const int jb = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int nI = g.nI, p = g.p, P1 = g.P1;
  const int ntri = p * (p + 1) / 2;
  const int cbsz = max(nI * P1, BASIS_THREADS * 36);

  double* Cb = sm;                      // column band  Cb[col][r] = A[col+r][col]
  double* Xs = Cb + cbsz;               // rhs / solution, [a][8]
  double* invd = Xs + nI * 8;           // 1 / L[a][a]
  BoxW bw;
  bw.wx = invd + nI; bw.wy = bw.wx + g.nwx; bw.wz = bw.wy + g.nwy;
  bw.b1 = g.b1; bw.b2 = g.b2; bw.b3 = g.b3;
  int* tri = (int*)(bw.wz + g.nwz);     // packed (r << 16 | q) for 1 <= q <= r <= p

  load_box_weights(g, w, X0, Y0, Z0, bw);
  for (int f = tid; f < ntri; f += nt) {
    int r = (int)((1.0 + sqrt(1.0 + 8.0 * f)) * 0.5);
    while (r * (r - 1) / 2 > f) --r;
    while ((r + 1) * r / 2 <= f) ++r;
    int q = f - r * (r - 1) / 2 + 1;
    tri[f] = (r << 16) | q;
  }
  __syncthreads();

  const double c1 = g.ih1 * g.ih1, c2 = g.ih2 * g.ih2, c3 = g.ih3 * g.ih3;
  const bool has0 = (jb == 0);   // block 0 holds the pinned corner node 0
  // band + rhs
  for (int a = tid; a < nI; a += nt) {
    int x = 1 + a % g.ni1, y = 1 + (a / g.ni1) % g.ni2, z = 1 + a / (g.ni1 * g.ni2);
    double kxm = bw.x(x - 1, y, z) * g.ih1 * g.ih1;
    double kxp = bw.x(x, y, z) * g.ih1 * g.ih1;
    double kym = bw.y(x, y - 1, z) * g.ih2 * g.ih2;
    double kyp = bw.y(x, y, z) * g.ih2 * g.ih2;
    double kzm = bw.z(x, y, z - 1) * g.ih3 * g.ih3;
    double kzp = bw.z(x, y, z) * g.ih3 * g.ih3;
    double* col = Cb + (size_t)a * P1;
    for (int r = 0; r < P1; ++r) col[r] = 0.0;
    col[0] = ((((kxm + kxp) + kym) + kyp) + kzm) + kzp;
    if (x + 1 <= g.ni1) col[1] = -kxp;
    if (y + 1 <= g.ni2) col[g.ni1] = -kyp;
    if (z + 1 <= g.ni3) col[p] = -kzp;
    double rhs[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) rhs[cc] = 0.0;
    // boundary neighbours contribute -A_IB x_B = + k_e * hat(nb)
    auto add_nb = [&](int xx, int yy, int zz, double kc) {
      if (interior_index(g, xx, yy, zz) >= 0) return;
      if (has0 && xx == 0 && yy == 0 && zz == 0) return;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) rhs[cc] += kc * hat_corner(cc, xx, yy, zz, g.b1, g.b2, g.b3);
    };
    add_nb(x - 1, y, z, kxm); add_nb(x + 1, y, z, kxp);
    add_nb(x, y - 1, z, kym); add_nb(x, y + 1, z, kyp);
    add_nb(x, y, z - 1, kzm); add_nb(x, y, z + 1, kzp);
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) Xs[a * 8 + cc] = rhs[cc];
  }
  (void)c1; (void)c2; (void)c3;
  __syncthreads();

  // right-looking band Cholesky
  for (int jc = 0; jc < nI; ++jc) {
    double* col = Cb + (size_t)jc * P1;
    const int rmax = min(p, nI - 1 - jc);
    double d = col[0];
    if (!(d > 0.0)) {
      if (tid == 0) atomicOr(flags, FLAG_LOCAL_NOT_SPD);
      d = 1.0;
    }
    const double piv = sqrt(d);
    const double inv = 1.0 / piv;
    for (int r = 1 + tid; r <= rmax; r += nt) col[r] *= inv;
    __syncthreads();
    if (tid == 0) { col[0] = piv; invd[jc] = inv; }
    const int nup = rmax * (rmax + 1) / 2;
    for (int f = tid; f < nup; f += nt) {
      int rq = tri[f];
      int r = rq >> 16, q = rq & 0xffff;
      Cb[(size_t)(jc + q) * P1 + (r - q)] -= col[r] * col[q];
    }
    __syncthreads();
  }

  // factor to global, both band forms, slot 0 holds the inverse diagonal
  {
    const size_t base = (size_t)jb * nI * g.P1s;
    for (int t = tid; t < nI * P1; t += nt) {
      int a = t / P1, r = t - a * P1;
      double v = (r == 0) ? invd[a] : Cb[(size_t)a * P1 + r];
      Lc[base + (size_t)a * g.P1s + r] = v;
      // row form: Lr[i][d] = L[i][i-d]
      int i = a, dd = r;
      double u;
      if (dd == 0) u = invd[i];
      else u = (i - dd >= 0) ? Cb[(size_t)(i - dd) * P1 + dd] : 0.0;
      Lr[base + (size_t)i * g.P1s + dd] = u;
    }
  }

  // forward substitution L y = rhs (column axpy, deferred row scaling)
  for (int i = 0; i < nI; ++i) {
    const int rmax = min(p, nI - 1 - i);
    const double inv = invd[i];
    const double* col = Cb + (size_t)i * P1;
    for (int t = tid; t < (rmax + 1) * 8; t += nt) {
      int r = t >> 3, s = t & 7;
      if (r == 0) { if (i > 0) Xs[(i - 1) * 8 + s] *= invd[i - 1]; }
      else Xs[(i + r) * 8 + s] -= col[r] * (Xs[i * 8 + s] * inv);
    }
    __syncthreads();
  }
  if (nI > 0) {
    if (tid < 8) Xs[(nI - 1) * 8 + tid] *= invd[nI - 1];
    __syncthreads();
  }
  // backward substitution L^T x = y (row axpy)
  for (int i = nI - 1; i >= 0; --i) {
    const int dmax = min(p, i);
    const double inv = invd[i];
    for (int t = tid; t < (dmax + 1) * 8; t += nt) {
      int d = t >> 3, s = t & 7;
      if (d == 0) { if (i < nI - 1) Xs[(i + 1) * 8 + s] *= invd[i + 1]; }
      else Xs[(i - d) * 8 + s] -= Cb[(size_t)(i - d) * P1 + d] * (Xs[i * 8 + s] * inv);
    }
    __syncthreads();
  }
  if (nI > 0) {
    if (tid < 8) Xs[tid] *= invd[0];
    __syncthreads();
  }
  for (int t = tid; t < nI * 8; t += nt) {
    int a = t >> 3, cc = t & 7;
    Sint[((size_t)jb * 8 + cc) * nI + a] = Xs[t];
  }

  // local Galerkin block over owned edges
  const int lx = (bi == g.nb1 - 1), ly = (bj == g.nb2 - 1), lz = (bk == g.nb3 - 1);
  const int ox = g.b1 * (g.b2 + ly) * (g.b3 + lz);
  const int oy = (g.b1 + lx) * g.b2 * (g.b3 + lz);
  const int oz = (g.b1 + lx) * (g.b2 + ly) * g.b3;
  double acc[36];
#pragma unroll
  for (int q = 0; q < 36; ++q) acc[q] = 0.0;
  for (int f = tid; f < ox + oy + oz; f += nt) {
    int ax, x, y, z;
    double kc;
    if (f < ox) {
      ax = 0; x = f % g.b1; int r = f / g.b1; y = r % (g.b2 + ly); z = r / (g.b2 + ly);
      kc = bw.x(x, y, z) * g.ih1 * g.ih1;
    } else if (f < ox + oy) {
      ax = 1; int q = f - ox; x = q % (g.b1 + lx); int r = q / (g.b1 + lx); y = r % g.b2; z = r / g.b2;
      kc = bw.y(x, y, z) * g.ih2 * g.ih2;
    } else {
      ax = 2; int q = f - ox - oy; x = q % (g.b1 + lx); int r = q / (g.b1 + lx); y = r % (g.b2 + ly); z = r / (g.b2 + ly);
      kc = bw.z(x, y, z) * g.ih3 * g.ih3;
    }
    int x1 = x + (ax == 0), y1 = y + (ax == 1), z1 = z + (ax == 2);
    bool n0 = has0 && x == 0 && y == 0 && z == 0;
    int a0 = interior_index(g, x, y, z), a1 = interior_index(g, x1, y1, z1);
    double ds[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      double s0 = a0 >= 0 ? Xs[a0 * 8 + cc] : (n0 ? 0.0 : hat_corner(cc, x, y, z, g.b1, g.b2, g.b3));
      double s1 = a1 >= 0 ? Xs[a1 * 8 + cc] : hat_corner(cc, x1, y1, z1, g.b1, g.b2, g.b3);
      ds[cc] = s1 - s0;
    }
#pragma unroll
    for (int c1i = 0; c1i < 8; ++c1i) {
      double kd = kc * ds[c1i];
#pragma unroll
      for (int c2i = 0; c2i <= c1i; ++c2i) acc[c1i * (c1i + 1) / 2 + c2i] += kd * ds[c2i];
    }
  }
  __syncthreads();           // Cb no longer needed: reuse for the reduction
  double* red = Cb;
#pragma unroll
  for (int q = 0; q < 36; ++q) red[q * nt + tid] = acc[q];
  __syncthreads();
  if (tid < 36) {
    double s = 0.0;
    for (int t = 0; t < nt; ++t) s += red[tid * nt + t];
    int c1i = (int)((sqrt(8.0 * tid + 1.0) - 1.0) * 0.5);
    while (c1i * (c1i + 1) / 2 > tid) --c1i;
    while ((c1i + 1) * (c1i + 2) / 2 <= tid) ++c1i;
    int c2i = tid - c1i * (c1i + 1) / 2;
    Kloc[(size_t)jb * 64 + c1i * 8 + c2i] = s;
    Kloc[(size_t)jb * 64 + c2i * 8 + c1i] = s;
  }
}

size_t basis_smem_bytes(const Geo& g) {
  size_t cbsz = (size_t)g.nI * g.P1;
  if (cbsz < (size_t)BASIS_THREADS * 36) cbsz = (size_t)BASIS_THREADS * 36;
  size_t d = cbsz + (size_t)g.nI * 8 + g.nI + g.nwx + g.nwy + g.nwz;
  size_t ntri = (size_t)g.p * (g.p + 1) / 2;
  return d * 8 + ntri * 4 + 16;
}

// ----------------------------------------------------- block-diagonal solve

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// One CTA per block.  The factor columns (forward) and rows (backward) stream
// through a RING-deep cp.async pipeline in shared memory; the right-hand sides
// of NSC sources at a time live in shared memory.  out may alias rhs.
template <int NSC>
__global__ void __launch_bounds__(SOLVE_THREADS)
k_block_solve(Geo g, const double* __restrict__ Lc, const double* __restrict__ Lr,
              const double* rhs, double* out, int nrhs) {
  constexpr int RING = SOLVE_RING;
  extern __shared__ double sm[];
  const int jb = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nI = g.nI, p = g.p, P1 = g.P1, P1s = g.P1s;
  if (nI == 0) return;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  double* Xs = sm;                        // [nI][NSC]
  double* ring = Xs + (size_t)nI * NSC;   // [RING][P1s]
  double* invd = ring + RING * P1s;       // [nI]
  const double* Lcb = Lc + (size_t)jb * nI * P1s;
  const double* Lrb = Lr + (size_t)jb * nI * P1s;

  for (int s0 = 0; s0 < nrhs; s0 += NSC) {
    const int ns = min(NSC, nrhs - s0);
    for (int t = tid; t < nI * NSC; t += nt) {
      int a = t / NSC, s = t - a * NSC;
      int x = 1 + a % g.ni1, y = 1 + (a / g.ni1) % g.ni2, z = 1 + a / (g.ni1 * g.ni2);
      long long node = node_id(g, X0 + x, Y0 + y, Z0 + z);
      Xs[t] = s < ns ? rhs[node * nrhs + s0 + s] : 0.0;
    }
    // ---- forward: columns of L
    for (int q = 0; q < RING - 1; ++q) {
      if (q < nI)
        for (int r = tid; r < P1; r += nt) cp_async8(ring + (q % RING) * P1s + r, Lcb + (size_t)q * P1s + r);
      cp_async_commit();
    }
    for (int i = 0; i < nI; ++i) {
      cp_async_wait<RING - 2>();
      __syncthreads();
      {
        int q = i + RING - 1;
        if (q < nI)
          for (int r = tid; r < P1; r += nt) cp_async8(ring + (q % RING) * P1s + r, Lcb + (size_t)q * P1s + r);
        cp_async_commit();
      }
      const double* col = ring + (i % RING) * P1s;
      const double inv = col[0];
      if (tid == 0) invd[i] = inv;
      const int rmax = min(p, nI - 1 - i);
      for (int t = tid; t < (rmax + 1) * NSC; t += nt) {
        int r = t / NSC, s = t - r * NSC;
        if (r == 0) { if (i > 0) Xs[(i - 1) * NSC + s] *= invd[i - 1]; }
        else Xs[(i + r) * NSC + s] -= col[r] * (Xs[i * NSC + s] * inv);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int t = tid; t < NSC; t += nt) Xs[(nI - 1) * NSC + t] *= invd[nI - 1];
    // ---- backward: rows of L, descending
    for (int q = 0; q < RING - 1; ++q) {
      int row = nI - 1 - q;
      if (row >= 0)
        for (int r = tid; r < P1; r += nt) cp_async8(ring + (q % RING) * P1s + r, Lrb + (size_t)row * P1s + r);
      cp_async_commit();
    }
    for (int it = 0; it < nI; ++it) {
      const int i = nI - 1 - it;
      cp_async_wait<RING - 2>();
      __syncthreads();
      {
        int q = it + RING - 1, row = nI - 1 - q;
        if (row >= 0)
          for (int r = tid; r < P1; r += nt) cp_async8(ring + (q % RING) * P1s + r, Lrb + (size_t)row * P1s + r);
        cp_async_commit();
      }
      const double* rw = ring + (it % RING) * P1s;
      const double inv = invd[i];
      const int dmax = min(p, i);
      for (int t = tid; t < (dmax + 1) * NSC; t += nt) {
        int d = t / NSC, s = t - d * NSC;
        if (d == 0) { if (i < nI - 1) Xs[(i + 1) * NSC + s] *= invd[i + 1]; }
        else Xs[(i - d) * NSC + s] -= rw[d] * (Xs[i * NSC + s] * inv);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int t = tid; t < NSC; t += nt) Xs[t] *= invd[0];
    __syncthreads();
    for (int t = tid; t < nI * NSC; t += nt) {
      int a = t / NSC, s = t - a * NSC;
      if (s >= ns) continue;
      int x = 1 + a % g.ni1, y = 1 + (a / g.ni1) % g.ni2, z = 1 + a / (g.ni1 * g.ni2);
      long long node = node_id(g, X0 + x, Y0 + y, Z0 + z);
      out[node * nrhs + s0 + s] = Xs[t];
    }
    __syncthreads();
  }
}

size_t solve_smem_bytes(const Geo& g) {
  return ((size_t)g.nI * SOLVE_NSC + SOLVE_RING * g.P1s + g.nI) * 8 + 16;
}

// ------------------------------------------------------- fine-grid helpers

// (A_wt X)(node) = sum_e wt_e/h^2 (X(node) - X(nb)) over the node's edges.
// X is a full node field with X[0] == 0, so this is the pinned operator row.
__device__ __forceinline__ double apply_A_row(const Geo& g, const double* __restrict__ wt,
                                              const double* __restrict__ X, int nrhs, int s,
                                              long long I, long long J, long long K) {
  const long long nd = node_id(g, I, J, K);
  const double xc = X[nd * nrhs + s];
  double v = 0.0;
  const double c1 = g.ih1 * g.ih1, c2 = g.ih2 * g.ih2, c3 = g.ih3 * g.ih3;
  if (I > 0) v += wt[ex_id(g, I - 1, J, K)] * c1 * (xc - X[node_id(g, I - 1, J, K) * nrhs + s]);
  if (I < g.n1) v += wt[ex_id(g, I, J, K)] * c1 * (xc - X[node_id(g, I + 1, J, K) * nrhs + s]);
  if (J > 0) v += wt[ey_id(g, I, J - 1, K)] * c2 * (xc - X[node_id(g, I, J - 1, K) * nrhs + s]);
  if (J < g.n2) v += wt[ey_id(g, I, J, K)] * c2 * (xc - X[node_id(g, I, J + 1, K) * nrhs + s]);
  if (K > 0) v += wt[ez_id(g, I, J, K - 1)] * c3 * (xc - X[node_id(g, I, J, K - 1) * nrhs + s]);
  if (K < g.n3) v += wt[ez_id(g, I, J, K)] * c3 * (xc - X[node_id(g, I, J, K + 1) * nrhs + s]);
  return v;
}

// Lane groups: a group of G = 2^lg lanes (G >= nrhs up to 32) shares one node
// and strides over the sources, so loads and stores of [node][s] fields are
// contiguous across the group.
__host__ __forceinline__ int group_log2(int nrhs) {
  int lg = 0;
  while ((1 << lg) < nrhs && lg < 5) ++lg;
  return lg;
}

// out(x) = alpha * src(x) + beta * (A_wt X)(x) on every block-interior node.
__global__ void k_residual(Geo g, const double* __restrict__ src, double alpha,
                           const double* __restrict__ wt, const double* __restrict__ X, double beta,
                           int nrhs, int lg, double* __restrict__ out) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long ii = t >> lg;
  const int j = (int)(t & ((1 << lg) - 1));
  if (ii >= (long long)g.nbl * g.nI) return;
  const int jb = fdiv(ii, g.nI, g.r_nI), a = (int)(ii - (long long)jb * g.nI);
  int bi, bj, bk, x, y, z;
  decode3f(jb, g.nb1, g.r_nb1, g.nb2, g.r_nb2, bi, bj, bk);
  decode3f(a, g.ni1, g.r_ni1, g.ni2, g.r_ni2, x, y, z);
  x += 1; y += 1; z += 1;
  long long I = (long long)bi * g.b1 + x, J = (long long)bj * g.b2 + y, K = (long long)bk * g.b3 + z;
  long long nd = node_id(g, I, J, K);
  const double c1 = g.ih1 * g.ih1, c2 = g.ih2 * g.ih2, c3 = g.ih3 * g.ih3;
  const double kxm = wt[ex_id(g, I - 1, J, K)] * c1, kxp = wt[ex_id(g, I, J, K)] * c1;
  const double kym = wt[ey_id(g, I, J - 1, K)] * c2, kyp = wt[ey_id(g, I, J, K)] * c2;
  const double kzm = wt[ez_id(g, I, J, K - 1)] * c3, kzp = wt[ez_id(g, I, J, K)] * c3;
  const long long sx = 1, sy = g.n1 + 1, sz = (long long)(g.n1 + 1) * (g.n2 + 1);
  for (int s = j; s < nrhs; s += (1 << lg)) {
    const double* Xn = X + s;
    const double xc = Xn[nd * nrhs];
    double v = 0.0;
    if (beta != 0.0) {
      double av = kxm * (xc - Xn[(nd - sx) * nrhs]);
      av += kxp * (xc - Xn[(nd + sx) * nrhs]);
      av += kym * (xc - Xn[(nd - sy) * nrhs]);
      av += kyp * (xc - Xn[(nd + sy) * nrhs]);
      av += kzm * (xc - Xn[(nd - sz) * nrhs]);
      av += kzp * (xc - Xn[(nd + sz) * nrhs]);
      v = beta * av;
    }
    if (src) v += alpha * src[nd * nrhs + s];
    out[nd * nrhs + s] = v;
  }
}

// field(node, s) = sum_cc S(node, cc) Y[col(cc), s]  (node 0 -> 0).  A lane
// group per node strides over the sources; with groups of >= 8 lanes each of
// the first 8 lanes evaluates one corner of the node's S row and the group
// shares them by shuffles.
__global__ void k_prolong(Geo g, const double* __restrict__ Sint, const double* __restrict__ Y,
                          int nrhs, int lg, double* __restrict__ out) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nd = t >> lg;
  const int G = 1 << lg;
  const int j = (int)(t & (G - 1));
  const bool valid = nd < g.Nn && nd > 0;
  int bi = 0, bj = 0, bk = 0, x = 0, y = 0, z = 0;
  if (valid) {
    int I, J, K;
    decode3f(nd, g.n1 + 1, g.r_n1p, g.n2 + 1, g.r_n2p, I, J, K);
    bi = min(fdiv(I, g.b1, g.r_b1), g.nb1 - 1); bj = min(fdiv(J, g.b2, g.r_b2), g.nb2 - 1);
    bk = min(fdiv(K, g.b3, g.r_b3), g.nb3 - 1);
    x = I - bi * g.b1; y = J - bj * g.b2; z = K - bk * g.b3;
  }
  const double* Sb = Sint + (size_t)block_of(g, bi, bj, bk) * 8 * g.nI;
  double sv[8];
  int col[8];
  if (G >= 8) {
    const int my = j & 7;
    const double s1 = valid ? s_value(g, Sb, my, x, y, z, false) : 0.0;
    const int c1 = corner_col(g, bi, bj, bk, my);
    const int base = (threadIdx.x & 31) & ~(G - 1);
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      sv[cc] = __shfl_sync(0xffffffffu, s1, base + cc);
      col[cc] = __shfl_sync(0xffffffffu, c1, base + cc);
    }
  } else {
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      sv[cc] = valid ? s_value(g, Sb, cc, x, y, z, false) : 0.0;
      col[cc] = corner_col(g, bi, bj, bk, cc);
    }
  }
  if (nd >= g.Nn) return;
  double* o = out + nd * nrhs;
  for (int s = j; s < nrhs; s += G) {
    double v = 0.0;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) v += sv[cc] * __ldg(Y + (size_t)col[cc] * nrhs + s);
    o[s] = v;
  }
}

// Per-block partial restriction: part[jb][cc][s] = sum over nodes owned by jb
// of S(node, cc) * h(node, s), h = A_w1 X1 + A_w2 X2 (either term optional).
__global__ void __launch_bounds__(RESTRICT_THREADS)
k_restrict_op(Geo g, const double* __restrict__ Sint, const double* __restrict__ w1,
              const double* __restrict__ X1, const double* __restrict__ w2,
              const double* __restrict__ X2, int nrhs, double* __restrict__ part) {
  __shared__ double red[RESTRICT_THREADS * 8];
  const int jb = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int lx = (bi == g.nb1 - 1), ly = (bj == g.nb2 - 1), lz = (bk == g.nb3 - 1);
  const int ox = g.b1 + lx, oy = g.b2 + ly, oz = g.b3 + lz;
  const int nown = ox * oy * oz;
  const double* Sb = Sint + (size_t)jb * 8 * g.nI;
  for (int s = 0; s < nrhs; ++s) {
    double acc[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) acc[cc] = 0.0;
    for (int f = tid; f < nown; f += nt) {
      int x = f % ox, r = f / ox, y = r % oy, z = r / oy;
      long long I = (long long)bi * g.b1 + x, J = (long long)bj * g.b2 + y, K = (long long)bk * g.b3 + z;
      if (I == 0 && J == 0 && K == 0) continue;   // pinned node has no row
      double h = 0.0;
      if (X1) h += apply_A_row(g, w1, X1, nrhs, s, I, J, K);
      if (X2) h += apply_A_row(g, w2, X2, nrhs, s, I, J, K);
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) acc[cc] += s_value(g, Sb, cc, x, y, z, false) * h;
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) red[cc * nt + tid] = acc[cc];
    __syncthreads();
    for (int width = nt / 2; width > 0; width >>= 1) {
      if (tid < width)
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) red[cc * nt + tid] += red[cc * nt + tid + width];
      __syncthreads();
    }
    if (tid < 8) part[((size_t)jb * 8 + tid) * nrhs + s] = red[tid * nt];
    __syncthreads();
  }
}

// out[c][s] = scale * sum over blocks having coarse node c as a corner (fixed
// order) of part[block][local corner][s].
__global__ void k_gather_corners(Geo g, const double* __restrict__ part, int nrhs, double scale,
                                 double* __restrict__ out) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)g.kc * nrhs) return;
  int s = (int)(t % nrhs);
  int c = (int)(t / nrhs);
  int ci = c % (g.nb1 + 1), r = c / (g.nb1 + 1), cj = r % (g.nb2 + 1), ck = r / (g.nb2 + 1);
  double v = 0.0;
  for (int bk = ck - 1; bk <= ck; ++bk) {
    if (bk < 0 || bk >= g.nb3) continue;
    for (int bj = cj - 1; bj <= cj; ++bj) {
      if (bj < 0 || bj >= g.nb2) continue;
      for (int bi = ci - 1; bi <= ci; ++bi) {
        if (bi < 0 || bi >= g.nb1) continue;
        int lc = (ci - bi) + 2 * (cj - bj) + 4 * (ck - bk);
        v += part[((size_t)block_of(g, bi, bj, bk) * 8 + lc) * nrhs + s];
      }
    }
  }
  out[t] = scale * v;
}

// Edge products of the compact rapply form (forward.py:271-281):
//   xi_e = sum_s [dU (dZ + dY) + dR dY] / h_e^2      (d = difference along e)
// A lane group per node computes the node's (up to) three forward edges; the
// group's lanes stride over sources (coalesced) and reduce with shuffles.
__global__ void k_edge_xi(Geo g, const double* __restrict__ U, const double* __restrict__ Z,
                          const double* __restrict__ Y, const double* __restrict__ R, int nrhs, int lg,
                          double* __restrict__ xi) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nd = t >> lg;
  const int j = (int)(t & ((1 << lg) - 1));
  const bool valid = nd < g.Nn;
  int i = 0, jj = 0, k = 0;
  if (valid) decode3f(nd, g.n1 + 1, g.r_n1p, g.n2 + 1, g.r_n2p, i, jj, k);
  const bool hx = valid && i < g.n1, hy = valid && jj < g.n2, hz = valid && k < g.n3;
  const long long nx = nd + 1, ny = nd + (g.n1 + 1), nz = nd + (long long)(g.n1 + 1) * (g.n2 + 1);
  double ax = 0.0, ay = 0.0, az = 0.0;
  if (valid) {
    for (int s = j; s < nrhs; s += (1 << lg)) {
      const long long o = nd * nrhs + s;
      const double u = __ldg(U + o), zz = __ldg(Z + o), yy = __ldg(Y + o), rr = __ldg(R + o);
      if (hx) {
        const long long q = nx * nrhs + s;
        const double du = __ldg(U + q) - u, dz = __ldg(Z + q) - zz, dy = __ldg(Y + q) - yy, dr = __ldg(R + q) - rr;
        ax += du * (dz + dy) + dr * dy;
      }
      if (hy) {
        const long long q = ny * nrhs + s;
        const double du = __ldg(U + q) - u, dz = __ldg(Z + q) - zz, dy = __ldg(Y + q) - yy, dr = __ldg(R + q) - rr;
        ay += du * (dz + dy) + dr * dy;
      }
      if (hz) {
        const long long q = nz * nrhs + s;
        const double du = __ldg(U + q) - u, dz = __ldg(Z + q) - zz, dy = __ldg(Y + q) - yy, dr = __ldg(R + q) - rr;
        az += du * (dz + dy) + dr * dy;
      }
    }
  }
  for (int off = (1 << lg) >> 1; off > 0; off >>= 1) {
    ax += __shfl_xor_sync(0xffffffffu, ax, off);
    ay += __shfl_xor_sync(0xffffffffu, ay, off);
    az += __shfl_xor_sync(0xffffffffu, az, off);
  }
  if (j == 0) {
    if (hx) xi[ex_id(g, i, jj, k)] = ax * (g.ih1 * g.ih1);
    if (hy) xi[ey_id(g, i, jj, k)] = ay * (g.ih2 * g.ih2);
    if (hz) xi[ez_id(g, i, jj, k)] = az * (g.ih3 * g.ih3);
  }
}

// g_c = -sigma_c (V/4) sum over the cell's 12 edges of xi_e  (= -Csig^T xi)
__global__ void k_cell_gather(Geo g, const double* __restrict__ sigma, const double* __restrict__ xi,
                              double* __restrict__ gout) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.Nm) return;
  int i, j, k;
  decode3f(c, g.n1, g.r_n1, g.n2, g.r_n2, i, j, k);
  double tot = 0.0;
  tot += xi[ex_id(g, i, j, k)] + xi[ex_id(g, i, j + 1, k)] + xi[ex_id(g, i, j, k + 1)] + xi[ex_id(g, i, j + 1, k + 1)];
  tot += xi[ey_id(g, i, j, k)] + xi[ey_id(g, i + 1, j, k)] + xi[ey_id(g, i, j, k + 1)] + xi[ey_id(g, i + 1, j, k + 1)];
  tot += xi[ez_id(g, i, j, k)] + xi[ez_id(g, i + 1, j, k)] + xi[ez_id(g, i, j + 1, k)] + xi[ez_id(g, i + 1, j + 1, k)];
  gout[c] = -sigma[c] * (g.qv * tot);
}

// CSC materialization of S in the reference pattern: vals[t] = Sint[src[t]] or
// the precomputed skeleton hat value.
__global__ void k_basis_csc(long long nnz, const double* __restrict__ Sint, const long long* __restrict__ src,
                            const double* __restrict__ hatv, double* __restrict__ vals) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  long long s = src[t];
  vals[t] = s >= 0 ? Sint[s] : hatv[t];
}

// ----------------------------------------------------------- launchers

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

static std::atomic<long long> g_launches{0};
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

cudaError_t launch_sigma(long long Nm, const double* m, const double* mul, double* out, int* flags, cudaStream_t st) {
  if (Nm == 0) return cudaSuccess;
  k_sigma<<<nblk(Nm, 256), 256, 0, st>>>(Nm, m, mul, out, flags);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_mul(long long n, const double* a, const double* b, double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_mul<<<nblk(n, 256), 256, 0, st>>>(n, a, b, out);
  count_launches(1);
  return cudaGetLastError();
}
static bool edge_tile_ok(const Geo& g) {
  return g.n1 + 2 <= EWT_MAXW && (g.n2 + 1 + EWT_TY - 1) / EWT_TY < 65535 && g.n3 + 1 < 65535 && !getenv("MSFV_EW_LINES");
}
static cudaError_t launch_edge_tile(const Geo& g, const double* cv, double* w, int k0, int k1, cudaStream_t st) {
  const size_t smem = (size_t)2 * (EWT_TY + 1) * (g.n1 + 2) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_edge_weights_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)((size_t)2 * (EWT_TY + 1) * EWT_MAXW * sizeof(double)));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const dim3 grid((g.n2 + 1 + EWT_TY - 1) / EWT_TY, k1 - k0 + 1);
  k_edge_weights_tile<<<grid, EWT_THREADS, smem, st>>>(g, cv, w, k0, k1);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_edge_weights(const Geo& g, const double* cv, double* w, cudaStream_t st) {
  if (edge_tile_ok(g)) return launch_edge_tile(g, cv, w, 0, g.n3, st);
  const unsigned lines = (unsigned)(((long long)(g.n2 + 1) * (g.n3 + 1) + EW_LINES - 1) / EW_LINES);
  if (lines < 65535u) {
    const dim3 grid(1, lines, 3);
    k_edge_weights_lines<<<grid, dim3(EW_THREADS, EW_LINES), 0, st>>>(g, cv, w, 0, g.n3);
  } else {
    k_edge_weights<<<nblk(g.E, 256), 256, 0, st>>>(g, cv, w);
  }
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_edge_weights_planes(const Geo& g, const double* cv, double* w, int k0, int k1, cudaStream_t st) {
  const unsigned lines = (unsigned)(((long long)(g.n2 + 1) * (k1 - k0 + 1) + EW_LINES - 1) / EW_LINES);
  if (k1 < k0 || lines >= 65535u) return cudaErrorInvalidValue;
  if (edge_tile_ok(g)) return launch_edge_tile(g, cv, w, k0, k1, st);
  const dim3 grid(1, lines, 3);
  k_edge_weights_lines<<<grid, dim3(EW_THREADS, EW_LINES), 0, st>>>(g, cv, w, k0, k1);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_basis(const Geo& g, const double* w, double* Lc, double* Lr, double* Sint, double* Kloc,
                         int* flags, cudaStream_t st) {
  size_t smem = basis_smem_bytes(g);
  cudaError_t e = cudaFuncSetAttribute(k_basis, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_basis<<<g.nbl, BASIS_THREADS, smem, st>>>(g, w, Lc, Lr, Sint, Kloc, flags);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_block_solve(const Geo& g, const double* Lc, const double* Lr, const double* rhs, double* out,
                               int nrhs, cudaStream_t st) {
  if (g.nI == 0 || nrhs == 0) return cudaSuccess;
  size_t smem = solve_smem_bytes(g);
  cudaError_t e = cudaFuncSetAttribute(k_block_solve<SOLVE_NSC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_block_solve<SOLVE_NSC><<<g.nbl, SOLVE_THREADS, smem, st>>>(g, Lc, Lr, rhs, out, nrhs);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_residual(const Geo& g, const double* src, double alpha, const double* wt, const double* X,
                            double beta, int nrhs, double* out, cudaStream_t st) {
  const int lg = group_log2(nrhs);
  long long tot = ((long long)g.nbl * g.nI) << lg;
  if (tot == 0 || nrhs == 0) return cudaSuccess;
  k_residual<<<nblk(tot, 256), 256, 0, st>>>(g, src, alpha, wt, X, beta, nrhs, lg, out);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_prolong(const Geo& g, const double* Sint, const double* Y, int nrhs, double* out, cudaStream_t st) {
  const int lg = group_log2(nrhs);
  k_prolong<<<nblk(g.Nn << lg, 256), 256, 0, st>>>(g, Sint, Y, nrhs, lg, out);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_restrict_op(const Geo& g, const double* Sint, const double* w1, const double* X1,
                               const double* w2, const double* X2, int nrhs, double* part, double scale,
                               double* out, cudaStream_t st) {
  k_restrict_op<<<g.nbl, RESTRICT_THREADS, 0, st>>>(g, Sint, w1, X1, w2, X2, nrhs, part);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_gather_corners<<<nblk((long long)g.kc * nrhs, 256), 256, 0, st>>>(g, part, nrhs, scale, out);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_gather_corners(const Geo& g, const double* part, int nrhs, double scale, double* out,
                                  cudaStream_t st) {
  k_gather_corners<<<nblk((long long)g.kc * nrhs, 256), 256, 0, st>>>(g, part, nrhs, scale, out);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_cell_gradient(const Geo& g, const double* sigma, const double* U, const double* Z,
                                 const double* Y, const double* R, int nrhs, double* xi, double* gout,
                                 cudaStream_t st) {
  const int lg = group_log2(nrhs);
  k_edge_xi<<<nblk(g.Nn << lg, 256), 256, 0, st>>>(g, U, Z, Y, R, nrhs, lg, xi);
  count_launches(1);
  k_cell_gather<<<nblk(g.Nm, 256), 256, 0, st>>>(g, sigma, xi, gout);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_basis_csc(long long nnz, const double* Sint, const long long* src, const double* hatv,
                             double* vals, cudaStream_t st) {
  if (nnz == 0) return cudaSuccess;
  k_basis_csc<<<nblk(nnz, 256), 256, 0, st>>>(nnz, Sint, src, hatv, vals);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
