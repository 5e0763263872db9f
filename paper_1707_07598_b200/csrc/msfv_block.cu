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
  const int jbk = block_of(g, bi, bj, bk);
  const double* Sb = Sint + (size_t)jbk * 8 * g.nI;
  double sv[8];
  int col[8];
  if (G >= 8) {
    const int my = j & 7;
    const double s1 = valid ? s_value(g, Sb, jbk, my, x, y, z, false) : 0.0;
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
      sv[cc] = valid ? s_value(g, Sb, jbk, cc, x, y, z, false) : 0.0;
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
      // w == nullptr: the field itself (S^T X, the coarse restriction of a node field)
      if (X1) h += w1 ? apply_A_row(g, w1, X1, nrhs, s, I, J, K) : X1[node_id(g, I, J, K) * nrhs + s];
      if (X2) h += w2 ? apply_A_row(g, w2, X2, nrhs, s, I, J, K) : X2[node_id(g, I, J, K) * nrhs + s];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) acc[cc] += s_value(g, Sb, jb, cc, x, y, z, false) * h;
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

// part[jb][cc][s] = sum over the nodes owned by jb of S(node, cc) X(node, s):
// the plain restriction S^T X of a node field (no operator), all right-hand
// sides at once.  Thread (group, s): s = tid % nrhs, the node groups stride
// the block's owned nodes; the groups' partial sums are reduced in a fixed
// order in shared memory.
__global__ void __launch_bounds__(RESTRICT_THREADS)
k_restrict_field(Geo g, const double* __restrict__ Sint, const double* __restrict__ X, int nrhs,
                 double* __restrict__ part) {
  __shared__ double red[RESTRICT_THREADS * 8];
  const int jb = blockIdx.x, tid = threadIdx.x;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int ox = g.b1 + (bi == g.nb1 - 1), oy = g.b2 + (bj == g.nb2 - 1), oz = g.b3 + (bk == g.nb3 - 1);
  const int nown = ox * oy * oz;
  const double* Sb = Sint + (size_t)jb * 8 * g.nI;
  const int ns_t = nrhs < RESTRICT_THREADS ? nrhs : RESTRICT_THREADS;
  const int ngroups = RESTRICT_THREADS / ns_t;
  for (int s0 = 0; s0 < nrhs; s0 += ns_t) {
    const int s = s0 + tid % ns_t, grp = tid / ns_t;
    double acc[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) acc[cc] = 0.0;
    if (grp < ngroups && s < nrhs) {
      for (int f = grp; f < nown; f += ngroups) {
        const int x = f % ox, r = f / ox, y = r % oy, z = r / oy;
        const long long I = (long long)bi * g.b1 + x, J = (long long)bj * g.b2 + y, K = (long long)bk * g.b3 + z;
        if (I == 0 && J == 0 && K == 0) continue;     // pinned node has no row
        const double h = X[node_id(g, I, J, K) * nrhs + s];
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) acc[cc] += s_value(g, Sb, jb, cc, x, y, z, false) * h;
      }
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) red[cc * RESTRICT_THREADS + tid] = acc[cc];
    __syncthreads();
    for (int t = tid; t < 8 * ns_t; t += blockDim.x) {
      const int cc = t / ns_t, sl = t % ns_t;
      double v = 0.0;
      for (int q = 0; q < ngroups; ++q) v += red[cc * RESTRICT_THREADS + q * ns_t + sl];
      if (s0 + sl < nrhs) part[((size_t)jb * 8 + cc) * nrhs + s0 + sl] = v;
    }
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
  static PerDevice<cudaError_t> attr;
  const cudaError_t ea = attr.get([] {
    return cudaFuncSetAttribute(k_edge_weights_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)((size_t)2 * (EWT_TY + 1) * EWT_MAXW * sizeof(double)));
  });
  if (ea != cudaSuccess) return ea;
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
  if (!w1 && X1 && !X2)
    k_restrict_field<<<g.nbl, RESTRICT_THREADS, 0, st>>>(g, Sint, X1, nrhs, part);
  else
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
cudaError_t launch_cell_gather(const Geo& g, const double* sigma, const double* xi, double* gout, cudaStream_t st) {
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
