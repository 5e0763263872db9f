// Materialized basis derivatives of the paper's Table 3 (basis.py:684-800):
//
//   apply_Yk(v):  d(S v)/dm = -blockdiag(A_II^{-1}) [G_p^T diag(G_p S v) Csig]_I   (n x N_m CSR)
//   apply_Xk(w):  d(S^T w)/dm:  row c, cell x of block j:
//                 -sum_{e in x} (G_p S)[e][c] (G_p z)_e Csig[e][x],  z = interior_solve(w)   (k x N_m CSR)
//
// The per-block right-hand sides of Y_k (8 non-zeros per interior row) are
// formed on the device, solved with the block factors (compact multi-RHS
// k_block_solve_tc, 512 right-hand sides per block), and scattered into a CSR
// whose pattern equals the reference's (rows: block interiors; columns: the
// block's cells whose right-hand-side column is non-zero, ascending).  X_k is
// one block-local pass; its rows collect the cells of up to 8 blocks, written
// straight to their sorted positions.
#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace msfv {

namespace {
__device__ __forceinline__ int ncell_b(const Geo& g) { return g.b1 * g.b2 * g.b3; }
__device__ __forceinline__ int mask_words(const Geo& g) { return (ncell_b(g) + 31) / 32; }
}  // namespace

// rhs_c[(jb*nI + a)*ncb + c] = W[I_a][cell c] (zeroed beforehand); mask bit c of block jb set when non-zero.
__global__ void k_yk_rhs(Geo g, const double* __restrict__ sigma, const double* __restrict__ Sv, double* __restrict__ rhs,
                         unsigned* __restrict__ mask) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)g.nbl * g.nI) return;
  const int jb = (int)(t / g.nI), a = (int)(t - (long long)jb * g.nI);
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  int x, y, z;
  decode3f(a, g.ni1, g.r_ni1, g.ni2, g.r_ni2, x, y, z);
  ++x; ++y; ++z;
  const long long I = (long long)bi * g.b1 + x, J = (long long)bj * g.b2 + y, K = (long long)bk * g.b3 + z;
  const double s0 = Sv[node_id(g, I, J, K)];
  // edge gradients gv_e = (Sv(upper) - Sv(lower)) / h, lower (-) / upper (+) side of the node
  const double gxm = (s0 - Sv[node_id(g, I - 1, J, K)]) * g.ih1, gxp = (Sv[node_id(g, I + 1, J, K)] - s0) * g.ih1;
  const double gym = (s0 - Sv[node_id(g, I, J - 1, K)]) * g.ih2, gyp = (Sv[node_id(g, I, J + 1, K)] - s0) * g.ih2;
  const double gzm = (s0 - Sv[node_id(g, I, J, K - 1)]) * g.ih3, gzp = (Sv[node_id(g, I, J, K + 1)] - s0) * g.ih3;
  // G_p^T diag(gv): +1/h on the edge below the node, -1/h on the edge above
  const double tx[2] = {g.ih1 * gxm, -g.ih1 * gxp}, ty[2] = {g.ih2 * gym, -g.ih2 * gyp},
               tz[2] = {g.ih3 * gzm, -g.ih3 * gzp};
  double* row = rhs + ((size_t)jb * g.nI + a) * ncell_b(g);
  unsigned* mk = mask + (size_t)jb * mask_words(g);
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    const int dx = d & 1, dy = (d >> 1) & 1, dz = d >> 2;
    const int cx = x - 1 + dx, cy = y - 1 + dy, cz = z - 1 + dz;
    const double sc = g.qv * sigma[cell_id(g, (long long)bi * g.b1 + cx, (long long)bj * g.b2 + cy,
                                           (long long)bk * g.b3 + cz)];
    const double v = ((tx[dx] * sc + ty[dy] * sc) + tz[dz] * sc);
    const int lc = cx + g.b1 * (cy + g.b2 * cz);
    row[lc] = v;
    if (v != 0.0) atomicOr(mk + (lc >> 5), 1u << (lc & 31));
  }
}

// counts[r] = number of Y_k entries of pinned row r
__global__ void k_yk_rowcount(Geo g, const unsigned* __restrict__ mask, long long* __restrict__ counts) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= g.Nn - 1) return;
  const long long nd = r + 1;
  int I, J, K;
  decode3f(nd, g.n1 + 1, g.r_n1p, g.n2 + 1, g.r_n2p, I, J, K);
  long long c = 0;
  if (I % g.b1 != 0 && J % g.b2 != 0 && K % g.b3 != 0) {
    const int jb = block_of(g, I / g.b1, J / g.b2, K / g.b3);
    const unsigned* mk = mask + (size_t)jb * mask_words(g);
    for (int w = 0; w < mask_words(g); ++w) c += __popc(mk[w]);
  }
  counts[r] = c;
}

// CSR scatter of -sol: one warp per (block, interior node) row; the lanes take
// 32 consecutive cells at a time and place the masked ones with a ballot
// prefix count, so the row's entries (ascending columns) are written by
// consecutive lanes to consecutive addresses.
constexpr int YKS_WARPS = 4;
__global__ void __launch_bounds__(YKS_WARPS * 32)
k_yk_scatter(Geo g, const unsigned* __restrict__ mask, const double* __restrict__ sol,
             const long long* __restrict__ indptr, int* __restrict__ indices, double* __restrict__ vals) {
  const long long t = (long long)blockIdx.x * YKS_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= (long long)g.nbl * g.nI) return;
  const int jb = (int)(t / g.nI), a = (int)(t - (long long)jb * g.nI);
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  int x, y, z;
  decode3f(a, g.ni1, g.r_ni1, g.ni2, g.r_ni2, x, y, z);
  const long long r = node_id(g, (long long)bi * g.b1 + x + 1, (long long)bj * g.b2 + y + 1,
                              (long long)bk * g.b3 + z + 1) - 1;
  long long p = indptr[r];
  const unsigned* mk = mask + (size_t)jb * mask_words(g);
  const double* srow = sol + ((size_t)jb * g.nI + a) * ncell_b(g);
  const int ncb = ncell_b(g);
  const unsigned below = (1u << lane) - 1u;
  for (int base = 0; base < ncb; base += 32) {
    const int lc = base + lane;
    const bool on = lc < ncb && ((mk[lc >> 5] >> (lc & 31)) & 1u);
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (on) {
      const long long q = p + __popc(bal & below);
      const int cx = lc % g.b1, qq = lc / g.b1, cy = qq % g.b2, cz = qq / g.b2;
      indices[q] = (int)cell_id(g, (long long)bi * g.b1 + cx, (long long)bj * g.b2 + cy, (long long)bk * g.b3 + cz);
      vals[q] = -srow[lc];
    }
    p += __popc(bal);
  }
}

// present[jb] = 1 when z (interior-only) is non-zero somewhere in block jb
__global__ void k_xk_present(Geo g, const double* __restrict__ zf, int* __restrict__ present) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)g.nbl * g.nI) return;
  const int jb = (int)(t / g.nI), a = (int)(t - (long long)jb * g.nI);
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  int x, y, z;
  decode3f(a, g.ni1, g.r_ni1, g.ni2, g.r_ni2, x, y, z);
  const double v = zf[node_id(g, (long long)bi * g.b1 + x + 1, (long long)bj * g.b2 + y + 1, (long long)bk * g.b3 + z + 1)];
  if (v != 0.0) present[jb] = 1;
}

namespace {
// cells of block B' = (pi, pj, pk) lexicographically (z, y, x) before global cell (X, Y, Z)
__device__ __forceinline__ long long cells_before(const Geo& g, int pi, int pj, int pk, long long X, long long Y,
                                                  long long Z) {
  const long long x0 = (long long)pi * g.b1, y0 = (long long)pj * g.b2, z0 = (long long)pk * g.b3;
  auto clampd = [](long long v, long long lo, long long n) { return v < lo ? 0 : (v - lo > n ? n : v - lo); };
  const long long nzb = clampd(Z, z0, g.b3);
  long long c = nzb * g.b1 * g.b2;
  if (Z >= z0 && Z < z0 + g.b3) {
    const long long nyb = clampd(Y, y0, g.b2);
    c += nyb * g.b1;
    if (Y >= y0 && Y < y0 + g.b2) c += clampd(X, x0, g.b1);
  }
  return c;
}
}  // namespace

// counts[c] = cells of the present blocks adjacent to coarse node c
__global__ void k_xk_rowcount(Geo g, const int* __restrict__ present, long long* __restrict__ counts) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.kc) return;
  const int ci = c % (g.nb1 + 1), r = c / (g.nb1 + 1), cj = r % (g.nb2 + 1), ck = r / (g.nb2 + 1);
  long long n = 0;
  for (int pk = ck - 1; pk <= ck; ++pk)
    for (int pj = cj - 1; pj <= cj; ++pj)
      for (int pi = ci - 1; pi <= ci; ++pi) {
        if (pi < 0 || pj < 0 || pk < 0 || pi >= g.nb1 || pj >= g.nb2 || pk >= g.nb3) continue;
        if (present[block_of(g, pi, pj, pk)]) n += (long long)g.b1 * g.b2 * g.b3;
      }
  counts[c] = n;
}

// X_k values: CTA per present block; closure basis values and z staged in
// shared memory; each thread owns cells, all 8 corner rows.
// STAGED = false (closures larger than shared memory, e.g. 16^3-cell blocks):
// the same arithmetic with the basis values and z read from global memory.
template <bool STAGED>
__global__ void __launch_bounds__(256) k_xk_values(Geo g, const double* __restrict__ sigma,
                                                   const double* __restrict__ Sint, const double* __restrict__ zf,
                                                   const int* __restrict__ present, const long long* __restrict__ indptr,
                                                   int* __restrict__ indices, double* __restrict__ vals) {
  extern __shared__ __align__(16) double xsm[];
  const int jb = blockIdx.x;
  if (!present[jb]) return;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int B1 = g.b1 + 1, B2 = g.b2 + 1, B3 = g.b3 + 1, NN = B1 * B2 * B3;
  double* Sn = xsm;                 // [NN][8]
  double* Zn = Sn + (size_t)NN * 8;  // [NN]
  const double* Sb = Sint + (size_t)jb * 8 * g.nI;
  auto S_at = [&](int n, int cc) -> double {
    if (STAGED) return Sn[n * 8 + cc];
    const int x = n % B1, r = n / B1, y = r % B2, z = r / B2;
    return s_value(g, Sb, jb, cc, x, y, z, jb == 0 && n == 0);
  };
  auto Z_at = [&](int n) -> double {
    if (STAGED) return Zn[n];
    const int x = n % B1, r = n / B1, y = r % B2, z = r / B2;
    const bool in = x > 0 && x < g.b1 && y > 0 && y < g.b2 && z > 0 && z < g.b3;
    return in ? zf[node_id(g, (long long)bi * g.b1 + x, (long long)bj * g.b2 + y, (long long)bk * g.b3 + z)] : 0.0;
  };
  if (STAGED) for (int n = threadIdx.x; n < NN; n += blockDim.x) {
    const int x = n % B1, r = n / B1, y = r % B2, z = r / B2;
    const bool in = x > 0 && x < g.b1 && y > 0 && y < g.b2 && z > 0 && z < g.b3;
    const bool node0 = jb == 0 && n == 0;
    const int a = in ? interior_index(g, x, y, z) : -1;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc)
      Sn[n * 8 + cc] = in ? Sb[(size_t)cc * g.nI + a] : (node0 ? 0.0 : hatf(g, cc, x, y, z));
    Zn[n] = in ? zf[node_id(g, (long long)bi * g.b1 + x, (long long)bj * g.b2 + y, (long long)bk * g.b3 + z)] : 0.0;
  }
  __syncthreads();
  const int ncb = g.b1 * g.b2 * g.b3;
  for (int lc = threadIdx.x; lc < ncb; lc += blockDim.x) {
    const int cx = lc % g.b1, q = lc / g.b1, cy = q % g.b2, cz = q / g.b2;
    const long long X = (long long)bi * g.b1 + cx, Y = (long long)bj * g.b2 + cy, Z = (long long)bk * g.b3 + cz;
    const long long cid = cell_id(g, X, Y, Z);
    const double sc = g.qv * sigma[cid];
    double acc[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) acc[cc] = 0.0;
    // the cell's 12 edges: (axis, lower-node offsets)
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double ih = ax == 0 ? g.ih1 : (ax == 1 ? g.ih2 : g.ih3);
      const int step = ax == 0 ? 1 : (ax == 1 ? B1 : B1 * B2);
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          int ox = cx, oy = cy, oz = cz;
          if (ax == 0) { oy += u; oz += v; }
          else if (ax == 1) { ox += u; oz += v; }
          else { ox += u; oy += v; }
          const int na = ox + B1 * (oy + B2 * oz), nb = na + step;
          const double ae = (Z_at(nb) - Z_at(na)) * ih;
          if (ae == 0.0) continue;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) acc[cc] += ((S_at(nb, cc) - S_at(na, cc)) * ih * ae) * sc;
        }
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int row = corner_col(g, bi, bj, bk, cc);
      const int ci = bi + (cc & 1), cj = bj + ((cc >> 1) & 1), ck = bk + ((cc >> 2) & 1);
      long long rank = 0;
      for (int pk = ck - 1; pk <= ck; ++pk)
        for (int pj = cj - 1; pj <= cj; ++pj)
          for (int pi = ci - 1; pi <= ci; ++pi) {
            if (pi < 0 || pj < 0 || pk < 0 || pi >= g.nb1 || pj >= g.nb2 || pk >= g.nb3) continue;
            if (present[block_of(g, pi, pj, pk)]) rank += cells_before(g, pi, pj, pk, X, Y, Z);
          }
      const long long p = indptr[row] + rank;
      indices[p] = (int)cid;
      vals[p] = -acc[cc];
    }
  }
}

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_yk_rhs(const Geo& g, const double* sigma, const double* Sv, double* rhs, unsigned* mask,
                          cudaStream_t st) {
  const long long tot = (long long)g.nbl * g.nI;
  if (tot == 0) return cudaSuccess;
  k_yk_rhs<<<nblk(tot, 128), 128, 0, st>>>(g, sigma, Sv, rhs, mask);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_yk_rowcount(const Geo& g, const unsigned* mask, long long* counts, cudaStream_t st) {
  k_yk_rowcount<<<nblk(g.Nn - 1, 256), 256, 0, st>>>(g, mask, counts);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_yk_scatter(const Geo& g, const unsigned* mask, const double* sol, const long long* indptr,
                              int* indices, double* vals, cudaStream_t st) {
  const long long tot = (long long)g.nbl * g.nI;
  if (tot == 0) return cudaSuccess;
  k_yk_scatter<<<nblk(tot, YKS_WARPS), YKS_WARPS * 32, 0, st>>>(g, mask, sol, indptr, indices, vals);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_xk_present(const Geo& g, const double* zf, int* present, cudaStream_t st) {
  const long long tot = (long long)g.nbl * g.nI;
  if (tot == 0) return cudaSuccess;
  k_xk_present<<<nblk(tot, 256), 256, 0, st>>>(g, zf, present);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_xk_rowcount(const Geo& g, const int* present, long long* counts, cudaStream_t st) {
  k_xk_rowcount<<<nblk(g.kc, 256), 256, 0, st>>>(g, present, counts);
  count_launches(1);
  return cudaGetLastError();
}
size_t xk_smem_bytes(const Geo& g) { return (size_t)(g.b1 + 1) * (g.b2 + 1) * (g.b3 + 1) * 9 * sizeof(double); }
cudaError_t launch_xk_values(const Geo& g, const double* sigma, const double* Sint, const double* zf, const int* present,
                             const long long* indptr, int* indices, double* vals, cudaStream_t st) {
  const size_t smem = xk_smem_bytes(g);
  if (smem > 200 * 1024) {
    k_xk_values<false><<<g.nbl, 256, 0, st>>>(g, sigma, Sint, zf, present, indptr, indices, vals);
  } else {
    cudaError_t e = cudaFuncSetAttribute(k_xk_values<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_xk_values<true><<<g.nbl, 256, smem, st>>>(g, sigma, Sint, zf, present, indptr, indices, vals);
  }
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
