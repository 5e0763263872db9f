// C-ABI entry points (include/msfv.h): argument checking, plan/point-set
// construction on the host, and kernel launches on the caller's stream.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/msfv.h"
#include "msfv_common.cuh"
#include "msfv_kernels.h"

using namespace msfv;

struct msfv_plan {
  Geo g;
  SkelEdge* skel_dev = nullptr;   // uploaded on first basis build (plan creation needs no GPU)
  bool mesh_only = false;         // msfv_plan_create_mesh: no coarse partition (fine-mesh entry points only)
};

// Skeleton-only owned edges of a block in the "last along every axis" case;
// k_skel_galerkin skips entries whose req bits the block does not have.
static std::vector<SkelEdge> skeleton_edges(const Geo& g) {
  std::vector<SkelEdge> out;
  const int b[3] = {g.b1, g.b2, g.b3};
  auto hat = [&](int c, int x, int y, int z) {
    const int cx = (c & 1) ? g.b1 : 0, cy = (c & 2) ? g.b2 : 0, cz = (c & 4) ? g.b3 : 0;
    auto h1 = [](int d, double ib) { double v = 1.0 - std::fabs((double)d) * ib; return v > 0.0 ? v : 0.0; };
    double w = h1(x - cx, g.ib1);
    w = w * h1(y - cy, g.ib2);
    w = w * h1(z - cz, g.ib3);
    return w;
  };
  for (int ax = 0; ax < 3; ++ax) {
    const int pa = ax == 0 ? 1 : 0, qa = ax == 2 ? 1 : 2;     // transverse axes (u, v)
    for (int v = 0; v <= b[qa]; ++v)
      for (int u = 0; u <= b[pa]; ++u) {
        const bool perim = u == 0 || u == b[pa] || v == 0 || v == b[qa];
        if (!(perim || b[ax] == 1)) continue;
        for (int xa = 0; xa < b[ax]; ++xa) {
          int c[3];
          c[ax] = xa; c[pa] = u; c[qa] = v;
          SkelEdge e{};
          e.ax = ax; e.x = c[0]; e.y = c[1]; e.z = c[2];
          e.req = (u == b[pa] ? (1 << pa) : 0) | (v == b[qa] ? (1 << qa) : 0);
          e.origin = (c[0] == 0 && c[1] == 0 && c[2] == 0);
          const int x1 = c[0] + (ax == 0), y1 = c[1] + (ax == 1), z1 = c[2] + (ax == 2);
          for (int cc = 0; cc < 8; ++cc) {
            e.h1[cc] = hat(cc, x1, y1, z1);
            e.h0[cc] = hat(cc, c[0], c[1], c[2]);
          }
          out.push_back(e);
        }
      }
  }
  return out;
}

struct msfv_points {
  PointsDev d;
  void* mem = nullptr;
};

// the register-window DMMA band path (msfv_tc.cu); plans with reduced
// boundary conditions always take the L2-resident band path (msfv_large.cu),
// whose kernels read the bound skeleton-value table
static inline bool use_tc(const Geo& g) { return tc_supported(g) && !g.reduced; }
// Local factor layout and interior solves: the register-window path whenever
// the band fits, reduced boundary conditions included (their right-hand sides
// come from the bound box table, msfv_tc.cu stencil_table; their Galerkin
// blocks from launch_lg_galerkin).
static inline bool tc_solver(const Geo& g) { return tc_supported(g); }

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
namespace msfv {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace msfv
static int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return MSFV_OK;
  return fail(MSFV_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CHECK_PLAN(p) \
  if (!(p)) return fail(MSFV_SHAPE, "null plan")
#define CHECK_PARTITION(p)                                                                               \
  do {                                                                                                   \
    CHECK_PLAN(p);                                                                                       \
    if ((p)->mesh_only) return fail(MSFV_UNSUPPORTED, "geometry-only plan (msfv_plan_create_mesh) has no coarse partition"); \
  } while (0)

extern "C" {

int msfv_abi_version(void) { return MSFV_ABI_VERSION; }
const char* msfv_last_error(void) { return g_err.c_str(); }
int64_t msfv_launch_count(void) { return launch_count(); }

static int plan_create(const int32_t cells[3], const double h[3], const int32_t blocks[3], bool mesh_only,
                       msfv_plan** out) {
  if (!cells || !h || !blocks || !out) return fail(MSFV_SHAPE, "null argument");
  for (int a = 0; a < 3; ++a) {
    if (cells[a] < 1) return fail(MSFV_SHAPE, "cell counts must be integers >= 1");
    if (!(h[a] > 0)) return fail(MSFV_SHAPE, "cell widths must be > 0");
    if (blocks[a] < 1) return fail(MSFV_SHAPE, "block size must be an integer >= 1");
    if (cells[a] % blocks[a]) return fail(MSFV_SHAPE, "block size does not divide cell count; partial blocks are not supported");
    if (cells[a] > 1000000 || blocks[a] > 1000) return fail(MSFV_SHAPE, "geometry too large");
  }
  Geo g{};
  g.n1 = cells[0]; g.n2 = cells[1]; g.n3 = cells[2];
  g.b1 = blocks[0]; g.b2 = blocks[1]; g.b3 = blocks[2];
  g.nb1 = g.n1 / g.b1; g.nb2 = g.n2 / g.b2; g.nb3 = g.n3 / g.b3;
  g.ni1 = g.b1 - 1; g.ni2 = g.b2 - 1; g.ni3 = g.b3 - 1;
  g.nI = g.ni1 * g.ni2 * g.ni3;
  g.p = g.ni1 * g.ni2;
  g.P1 = g.p + 1;
  g.P1s = (g.P1 + 1) & ~1;
  g.nbl = g.nb1 * g.nb2 * g.nb3;
  g.kc = (g.nb1 + 1) * (g.nb2 + 1) * (g.nb3 + 1);
  g.pc = (g.nb1 + 1) * (g.nb2 + 1) + (g.nb1 + 1) + 1;
  g.TB = COARSE_TB;
  g.NT = (g.kc + g.TB - 1) / g.TB;
  g.PT = std::min((g.pc + g.TB - 1) / g.TB, g.NT - 1);
  g.nwx = g.b1 * (g.b2 + 1) * (g.b3 + 1);
  g.nwy = (g.b1 + 1) * g.b2 * (g.b3 + 1);
  g.nwz = (g.b1 + 1) * (g.b2 + 1) * g.b3;
  g.Nn = (long long)(g.n1 + 1) * (g.n2 + 1) * (g.n3 + 1);
  g.nbox = (g.b1 + 1) * (g.b2 + 1) * (g.b3 + 1);
  g.Nm = (long long)g.n1 * g.n2 * g.n3;
  g.Ex = (long long)g.n1 * (g.n2 + 1) * (g.n3 + 1);
  g.Ey = (long long)(g.n1 + 1) * g.n2 * (g.n3 + 1);
  g.Ez = (long long)(g.n1 + 1) * (g.n2 + 1) * g.n3;
  g.E = g.Ex + g.Ey + g.Ez;
  g.h1 = h[0]; g.h2 = h[1]; g.h3 = h[2];
  g.ih1 = 1.0 / h[0]; g.ih2 = 1.0 / h[1]; g.ih3 = 1.0 / h[2];
  g.qv = 0.25 * (h[0] * h[1] * h[2]);
  g.ib1 = 1.0 / g.b1; g.ib2 = 1.0 / g.b2; g.ib3 = 1.0 / g.b3;
  g.r_n1 = 1.0f / g.n1; g.r_n2 = 1.0f / g.n2; g.r_n1p = 1.0f / (g.n1 + 1); g.r_n2p = 1.0f / (g.n2 + 1);
  g.r_b1 = 1.0f / g.b1; g.r_b2 = 1.0f / g.b2; g.r_b3 = 1.0f / g.b3;
  g.r_ni1 = g.ni1 > 0 ? 1.0f / g.ni1 : 0.0f; g.r_ni2 = g.ni2 > 0 ? 1.0f / g.ni2 : 0.0f;
  g.r_nI = g.nI > 0 ? 1.0f / g.nI : 0.0f; g.r_nb1 = 1.0f / g.nb1; g.r_nb2 = 1.0f / g.nb2;
  {
    // coarse nested dissection: on for k >= 1000 (MSFV_COARSE_ND=0/1 overrides)
    // coarse solver: one band below 1000 unknowns, multifrontal nested
    // dissection above (z-plane nested dissection of the band if the tree has
    // more fronts per level than the cooperative kernels take);
    // MSFV_COARSE_ND=0/1/2 overrides
    const char* ev = getenv("MSFV_COARSE_ND");
    g.coarse_nd = ev ? std::min(2, std::max(0, atoi(ev))) : (g.kc >= 1000 ? 2 : 0);
    if (mesh_only) g.coarse_nd = 0;
    g.mf = nullptr;
    g.skel = nullptr;
    g.nskel = 0;
  }
  if (!mesh_only && !tc_supported(g) && !lg_supported(g))
    return fail(MSFV_UNSUPPORTED, "block interior half bandwidth ni1*ni2 exceeds 512 (largest supported band)");
  if (!mesh_only && g.p >= 65535) return fail(MSFV_UNSUPPORTED, "block too large");
  if (g.Nn >= (1LL << 31) || g.E >= (1LL << 31)) return fail(MSFV_UNSUPPORTED, "mesh too large for 32-bit node/edge indices");
  if (g.coarse_nd == 2 && !mf_attach(g)) g.coarse_nd = g.kc >= 1000 ? 1 : 0;
  g.gtab8 = !mesh_only && grad_template_init(g) ? 1 : 0;
  msfv_plan* pl = new msfv_plan;
  pl->g = g;
  pl->mesh_only = mesh_only;
  *out = pl;
  return MSFV_OK;
}

int msfv_plan_create(const int32_t cells[3], const double h[3], const int32_t blocks[3], msfv_plan** out) {
  return plan_create(cells, h, blocks, false, out);
}

int msfv_plan_create_mesh(const int32_t cells[3], const double h[3], msfv_plan** out) {
  if (!cells) return fail(MSFV_SHAPE, "null argument");
  if (cells[0] > 1023 || cells[1] > 1023 || cells[2] > 1023)
    return fail(MSFV_UNSUPPORTED, "geometry-only plans take at most 1023 cells per axis");
  return plan_create(cells, h, cells, true, out);
}

void msfv_plan_destroy(msfv_plan* plan) {
  if (!plan) return;
  if (plan->skel_dev) cudaFree(plan->skel_dev);
  mf_release(plan->g);
  delete plan;
}

int msfv_plan_info(const msfv_plan* plan, int64_t* info, int32_t n) {
  CHECK_PLAN(plan);
  const Geo& g = plan->g;
  int64_t v[MSFV_INFO_COUNT];
  v[MSFV_INFO_NN] = g.Nn;
  v[MSFV_INFO_N] = g.Nn - 1;
  v[MSFV_INFO_NCELLS] = g.Nm;
  v[MSFV_INFO_NEDGES] = g.E;
  v[MSFV_INFO_NBLOCKS] = g.nbl;
  v[MSFV_INFO_NI] = g.nI;
  v[MSFV_INFO_P1S] = g.P1s;
  v[MSFV_INFO_K] = g.kc;
  v[MSFV_INFO_AK_DOUBLES] = (int64_t)coarse_doubles(g);
  v[MSFV_INFO_BASIS_SMEM] = 0;
  v[MSFV_INFO_NT] = coarse_tile_rows(g);
  v[MSFV_INFO_PT] = g.PT;
  v[MSFV_INFO_TB] = g.TB;
  v[MSFV_INFO_PC] = g.pc;
  const bool tc = use_tc(g), tcs = tc_solver(g);
  v[MSFV_INFO_FACTOR_DOUBLES] = tcs ? (int64_t)tc_factor_doubles(g) : (int64_t)lg_factor_doubles(g);
  v[MSFV_INFO_SCRATCH_DOUBLES] = tcs ? (int64_t)tc_scratch_doubles(g) : 0;
  v[MSFV_INFO_TC] = tc ? 1 : 2;
  v[MSFV_INFO_COARSE] = g.coarse_nd;
  v[MSFV_INFO_RED_FACE_DOUBLES] = g.reduced ? (int64_t)red_face_doubles(g) : 0;
  v[MSFV_INFO_RED_BOX_DOUBLES] = g.reduced ? (int64_t)red_box_doubles(g) : 0;
  for (int i = 0; i < n && i < MSFV_INFO_COUNT; ++i) info[i] = v[i];
  return MSFV_OK;
}

int msfv_points_create(const msfv_plan* plan, int64_t nnz, int32_t ncol, const int64_t* colptr, const int64_t* rows,
                       const double* vals, msfv_points** out) {
  CHECK_PLAN(plan);
  if (!out || ncol < 0 || nnz < 0 || (nnz > 0 && (!rows || !vals)) || !colptr)
    return fail(MSFV_SHAPE, "bad survey matrix arguments");
  const Geo& g = plan->g;
  if (colptr[0] != 0 || colptr[ncol] != nnz) return fail(MSFV_SHAPE, "colptr does not match nnz");
  std::vector<long long> node(nnz), cptr(g.kc + 1, 0), cent, uptr, unode, uent(nnz);
  std::vector<int> col(nnz), blk(nnz), loc(nnz);
  std::vector<double> val(vals, vals + nnz);
  for (int c = 0; c < ncol; ++c) {
    if (colptr[c + 1] < colptr[c]) return fail(MSFV_SHAPE, "colptr not monotone");
    for (int64_t t = colptr[c]; t < colptr[c + 1]; ++t) col[t] = c;
  }
  for (int64_t t = 0; t < nnz; ++t) {
    if (rows[t] < 0 || rows[t] >= g.Nn - 1) return fail(MSFV_SHAPE, "survey row out of range");
    long long nd = rows[t] + 1;   // pinned -> full id
    node[t] = nd;
    long long I = nd % (g.n1 + 1), r = nd / (g.n1 + 1), J = r % (g.n2 + 1), K = r / (g.n2 + 1);
    int bi = own1(I, g.b1, g.nb1), bj = own1(J, g.b2, g.nb2), bk = own1(K, g.b3, g.nb3);
    int x = (int)(I - (long long)bi * g.b1), y = (int)(J - (long long)bj * g.b2), z = (int)(K - (long long)bk * g.b3);
    blk[t] = block_of(g, bi, bj, bk);
    loc[t] = x | (y << 10) | (z << 20);
    for (int cc = 0; cc < 8; ++cc) cptr[corner_col(g, bi, bj, bk, cc) + 1]++;
  }
  for (int c = 0; c < g.kc; ++c) cptr[c + 1] += cptr[c];
  cent.resize(cptr[g.kc]);
  {
    std::vector<long long> fill(cptr.begin(), cptr.end() - 1);
    for (int64_t t = 0; t < nnz; ++t) {
      int jb = blk[t];
      int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
      for (int cc = 0; cc < 8; ++cc) cent[fill[corner_col(g, bi, bj, bk, cc)]++] = ((long long)t << 3) | cc;
    }
  }
  std::vector<long long> ord(nnz);
  for (int64_t t = 0; t < nnz; ++t) ord[t] = t;
  std::stable_sort(ord.begin(), ord.end(), [&](long long a, long long b) { return node[a] < node[b]; });
  for (int64_t i = 0; i < nnz; ++i) {
    if (i == 0 || node[ord[i]] != node[ord[i - 1]]) {
      uptr.push_back(i);
      unode.push_back(node[ord[i]]);
    }
    uent[i] = ord[i];
  }
  uptr.push_back(nnz);
  long long nu = (long long)unode.size();
  // blocks with survey entries on interior nodes (compact per-block fields of
  // the interior-only solves): slot per block, compact row per unique node
  std::vector<int> islot(g.nbl, -1), iblk;
  std::vector<long long> urow(nu, -1);
  for (long long u = 0; u < nu; ++u) {
    const long long nd = unode[u];
    const long long t = uent[uptr[u]];
    int x, y, z;
    x = loc[t] & 1023; y = (loc[t] >> 10) & 1023; z = (loc[t] >> 20) & 1023;
    (void)nd;
    const int a = interior_index(g, x, y, z);
    if (a < 0) continue;
    const int jb = blk[t];
    if (islot[jb] < 0) {
      islot[jb] = (int)iblk.size();
      iblk.push_back(jb);
    }
    urow[u] = (long long)islot[jb] * g.nI + a;
  }
  const int nib = (int)iblk.size();

  // one device allocation for all tables
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  size_t o_colptr = 0;
  size_t o_node = o_colptr + al((ncol + 1) * 8);
  size_t o_col = o_node + al(nnz * 8);
  size_t o_val = o_col + al(nnz * 4);
  size_t o_blk = o_val + al(nnz * 8);
  size_t o_loc = o_blk + al(nnz * 4);
  size_t o_cptr = o_loc + al(nnz * 4);
  size_t o_cent = o_cptr + al((g.kc + 1) * 8);
  size_t o_uptr = o_cent + al(cent.size() * 8);
  size_t o_unode = o_uptr + al((nu + 1) * 8);
  size_t o_uent = o_unode + al(nu * 8);
  size_t o_islot = o_uent + al(nnz * 8);
  size_t o_iblk = o_islot + al((size_t)g.nbl * 4);
  size_t o_urow = o_iblk + al((size_t)nib * 4);
  size_t total = o_urow + al(nu * 8) + 256;
  char* mem = nullptr;
  cudaError_t e = cudaMalloc(&mem, total);
  if (e != cudaSuccess) return cuda_check(e, "cudaMalloc(points)");
  auto up = [&](size_t off, const void* src, size_t bytes) {
    if (bytes) return cudaMemcpy(mem + off, src, bytes, cudaMemcpyHostToDevice);
    return cudaSuccess;
  };
  std::vector<long long> cp(colptr, colptr + ncol + 1);
  cudaError_t es[] = {up(o_colptr, cp.data(), (ncol + 1) * 8), up(o_node, node.data(), nnz * 8),
                      up(o_col, col.data(), nnz * 4),          up(o_val, val.data(), nnz * 8),
                      up(o_blk, blk.data(), nnz * 4),          up(o_loc, loc.data(), nnz * 4),
                      up(o_cptr, cptr.data(), (g.kc + 1) * 8), up(o_cent, cent.data(), cent.size() * 8),
                      up(o_uptr, uptr.data(), (nu + 1) * 8),   up(o_unode, unode.data(), nu * 8),
                      up(o_uent, uent.data(), nnz * 8),        up(o_islot, islot.data(), (size_t)g.nbl * 4),
                      up(o_iblk, iblk.data(), (size_t)nib * 4), up(o_urow, urow.data(), nu * 8)};
  for (cudaError_t x : es)
    if (x != cudaSuccess) {
      cudaFree(mem);
      return cuda_check(x, "cudaMemcpy(points)");
    }
  msfv_points* P = new msfv_points;
  P->mem = mem;
  P->d.nnz = nnz;
  P->d.ncol = ncol;
  P->d.colptr = (const long long*)(mem + o_colptr);
  P->d.node = (const long long*)(mem + o_node);
  P->d.col = (const int*)(mem + o_col);
  P->d.val = (const double*)(mem + o_val);
  P->d.blk = (const int*)(mem + o_blk);
  P->d.loc = (const int*)(mem + o_loc);
  P->d.cptr = (const long long*)(mem + o_cptr);
  P->d.cent = (const long long*)(mem + o_cent);
  P->d.nu = nu;
  P->d.uptr = (const long long*)(mem + o_uptr);
  P->d.unode = (const long long*)(mem + o_unode);
  P->d.uent = (const long long*)(mem + o_uent);
  P->d.nib = nib;
  P->d.islot = (const int*)(mem + o_islot);
  P->d.iblk = (const int*)(mem + o_iblk);
  P->d.urow = (const long long*)(mem + o_urow);
  *out = P;
  return MSFV_OK;
}

void msfv_points_destroy(msfv_points* pts) {
  if (!pts) return;
  cudaFree(pts->mem);
  delete pts;
}

int msfv_operator(const msfv_plan* plan, const double* m, double* sigma, double* w, int32_t* flags, void* stream) {
  CHECK_PLAN(plan);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = cuda_check(launch_sigma(plan->g.Nm, m, nullptr, sigma, flags, st), "sigma");
  if (rc) return rc;
  return cuda_check(launch_edge_weights(plan->g, sigma, w, st), "edge_weights");
}

int msfv_operator_slab(const msfv_plan* plan, const double* m, double* sigma, double* w, int32_t* flags, int32_t k0,
                       int32_t k1, void* stream) {
  CHECK_PLAN(plan);
  const Geo& g = plan->g;
  if (k0 < 0 || k1 > g.n3 || k0 >= k1) return fail(MSFV_SHAPE, "bad operator slab");
  cudaStream_t st = (cudaStream_t)stream;
  // sigma on cell planes k0 .. min(k1, n3 - 1) (plane k1 feeds the slab's top x/y edges)
  const long long plane = (long long)g.n1 * g.n2;
  const int kc1 = std::min(k1 + 1, g.n3);
  int rc = cuda_check(launch_sigma(plane * (kc1 - k0), m + plane * k0, nullptr, sigma + plane * k0, flags, st), "sigma");
  if (rc) return rc;
  return cuda_check(launch_edge_weights_planes(g, sigma, w, k0, k1, st), "edge_weights");
}

int msfv_edge_average(const msfv_plan* plan, const double* sigma, const double* dm, double* tmp, double* c,
                      void* stream) {
  CHECK_PLAN(plan);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = cuda_check(launch_mul(plan->g.Nm, sigma, dm, tmp, st), "mul");
  if (rc) return rc;
  return cuda_check(launch_edge_weights(plan->g, tmp, c, st), "edge_average");
}

static int ensure_skel(msfv_plan* pl) {
  if (pl->skel_dev) return MSFV_OK;
  const std::vector<SkelEdge> tab = skeleton_edges(pl->g);
  cudaError_t e = cudaMalloc(&pl->skel_dev, std::max<size_t>(tab.size(), 1) * sizeof(SkelEdge));
  if (e == cudaSuccess && !tab.empty())
    e = cudaMemcpy(pl->skel_dev, tab.data(), tab.size() * sizeof(SkelEdge), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_check(e, "skeleton edge table");
  pl->g.skel = pl->skel_dev;
  pl->g.nskel = (int)tab.size();
  return MSFV_OK;
}

static int basis_build(const msfv_plan* plan, const double* w, double* factor, double* Sint, double* Kloc,
                       double* scratch, int32_t* flags, void* stream, bool bwd) {
  CHECK_PARTITION(plan);
  const Geo& g = plan->g;
  cudaStream_t st = (cudaStream_t)stream;
  if (tc_solver(g)) {
    msfv_plan* pl = const_cast<msfv_plan*>(plan);
    int rc = ensure_skel(pl);
    if (rc) return rc;
    if (!g.reduced) return cuda_check(launch_basis_tc(pl->g, w, factor, Sint, Kloc, flags, st, bwd), "basis_build");
    // reduced boundary conditions: factor + both sweeps on the register-window kernel (right-hand sides
    // from the bound box table), then the Galerkin blocks from the actual skeleton values
    if (!g.bx) return fail(MSFV_SHAPE, "reduced plan without a bound boundary table");
    cudaError_t e = launch_basis_tc(pl->g, w, factor, Sint, Kloc, flags, st, true);
    if (e == cudaSuccess) e = launch_lg_galerkin(g, w, Sint, Kloc, st);
    return cuda_check(e, "basis_build");
  }
  return cuda_check(launch_basis_lg(g, w, factor, Sint, Kloc, flags, st), "basis_build");
}

int msfv_basis_build(const msfv_plan* plan, const double* w, double* factor, double* Sint, double* Kloc,
                     double* scratch, int32_t* flags, void* stream) {
  return basis_build(plan, w, factor, Sint, Kloc, scratch, flags, stream, true);
}

int msfv_basis_forward(const msfv_plan* plan, const double* w, double* factor, double* Sint, double* Kloc,
                       int32_t* flags, void* stream) {
  CHECK_PARTITION(plan);
  if (!use_tc(plan->g)) return fail(MSFV_UNSUPPORTED, "split basis build needs the tensor-core band path");
  return basis_build(plan, w, factor, Sint, Kloc, nullptr, flags, stream, false);
}

int msfv_basis_forward_slab(const msfv_plan* plan, const double* w, double* factor, double* Sint, double* Kloc,
                            int32_t* flags, int32_t bk0, int32_t bk1, void* stream) {
  CHECK_PARTITION(plan);
  const Geo& g = plan->g;
  if (!use_tc(g)) return fail(MSFV_UNSUPPORTED, "split basis build needs the tensor-core band path");
  if (bk0 < 0 || bk1 > g.nb3 || bk0 >= bk1) return fail(MSFV_SHAPE, "bad basis slab");
  msfv_plan* pl = const_cast<msfv_plan*>(plan);
  int rc = ensure_skel(pl);
  if (rc) return rc;
  const int per = g.nb1 * g.nb2;
  return cuda_check(launch_basis_tc(pl->g, w, factor, Sint, Kloc, flags, (cudaStream_t)stream, false, bk0 * per,
                                    bk1 * per),
                    "basis_forward_slab");
}

int msfv_basis_backward(const msfv_plan* plan, const double* factor, double* Sint, void* stream) {
  CHECK_PARTITION(plan);
  if (!use_tc(plan->g)) return fail(MSFV_UNSUPPORTED, "split basis build needs the tensor-core band path");
  return cuda_check(launch_basis_bwd(plan->g, factor, Sint, (cudaStream_t)stream), "basis_backward");
}

int msfv_basis_csc(int64_t nnz, const double* Sint, const int64_t* src, const double* hatv, double* vals,
                   void* stream) {
  return cuda_check(launch_basis_csc(nnz, Sint, (const long long*)src, hatv, vals, (cudaStream_t)stream),
                    "basis_csc");
}

int msfv_galerkin(const msfv_plan* plan, const double* Kloc, double shift, double* Ak, void* stream) {
  CHECK_PARTITION(plan);
  return cuda_check(launch_coarse_assemble(plan->g, Kloc, shift, Ak, (cudaStream_t)stream), "galerkin");
}

int msfv_coarse_diag(const msfv_plan* plan, const double* Ak, double* diag, void* stream) {
  CHECK_PARTITION(plan);
  return cuda_check(launch_coarse_diag(plan->g, Ak, diag, (cudaStream_t)stream), "coarse_diag");
}

int msfv_coarse_factor(const msfv_plan* plan, double* Ak, int32_t* flags, void* stream) {
  CHECK_PARTITION(plan);
  return cuda_check(launch_coarse_factor(plan->g, Ak, flags, (cudaStream_t)stream), "coarse_factor");
}

int msfv_coarse_solve(const msfv_plan* plan, const double* Lk, double* X, double* scratch, int32_t nrhs,
                      void* stream) {
  CHECK_PARTITION(plan);
  if (nrhs < 0) return fail(MSFV_SHAPE, "nrhs < 0");
  return cuda_check(launch_coarse_solve(plan->g, Lk, X, scratch, nrhs, (cudaStream_t)stream), "coarse_solve");
}

int msfv_survey_receive(const msfv_plan* plan, const msfv_points* pts, const double* Sint, const double* Y,
                        const double* Xfield, int32_t nrhs, double* out, void* stream) {
  CHECK_PLAN(plan);
  if (!pts) return fail(MSFV_SHAPE, "null points");
  return cuda_check(launch_points_receive(plan->g, pts->d, Sint, Y, Xfield, nrhs, out, (cudaStream_t)stream),
                    "survey_receive");
}

int msfv_misfit(const double* D, const double* Dobs, int64_t n, double* resid, double* phi, void* stream) {
  if (n < 0 || !D || !Dobs || !resid || !phi) return fail(MSFV_SHAPE, "bad misfit arguments");
  return cuda_check(launch_misfit(D, Dobs, (long long)n, resid, phi, (cudaStream_t)stream), "misfit");
}

int msfv_survey_restrict(const msfv_plan* plan, const msfv_points* pts, const double* Sint, const double* Z,
                         int32_t nrhs, double* out, void* stream) {
  CHECK_PLAN(plan);
  if (!pts) return fail(MSFV_SHAPE, "null points");
  return cuda_check(launch_points_restrict(plan->g, pts->d, Sint, Z, nrhs, out, (cudaStream_t)stream),
                    "survey_restrict");
}

int msfv_survey_scatter(const msfv_plan* plan, const msfv_points* pts, const double* Z, int32_t nrhs, double* field,
                        void* stream) {
  CHECK_PLAN(plan);
  if (!pts) return fail(MSFV_SHAPE, "null points");
  return cuda_check(launch_points_scatter(plan->g, pts->d, Z, nrhs, field, (cudaStream_t)stream), "survey_scatter");
}

int msfv_prolong(const msfv_plan* plan, const double* Sint, const double* Y, int32_t nrhs, double* field,
                 void* stream) {
  CHECK_PARTITION(plan);
  return cuda_check(launch_prolong(plan->g, Sint, Y, nrhs, field, (cudaStream_t)stream), "prolong");
}

int msfv_residual(const msfv_plan* plan, const double* src, double alpha, const double* wt, const double* X,
                  double beta, int32_t nrhs, double* out, void* stream) {
  CHECK_PARTITION(plan);
  return cuda_check(launch_residual(plan->g, src, alpha, wt, X, beta, nrhs, out, (cudaStream_t)stream), "residual");
}

int msfv_interior_solve(const msfv_plan* plan, const double* factor, const double* rhs, double* out, int32_t nrhs,
                        void* stream) {
  CHECK_PARTITION(plan);
  const Geo& g = plan->g;
  cudaStream_t st = (cudaStream_t)stream;
  if (tc_solver(g)) return cuda_check(launch_block_solve_tc(g, factor, rhs, out, nrhs, st), "interior_solve");
  return cuda_check(launch_block_solve_lg(g, factor, rhs, out, nrhs, st), "interior_solve");
}

int msfv_restrict_op(const msfv_plan* plan, const double* Sint, const double* w1, const double* X1,
                     const double* w2, const double* X2, int32_t nrhs, double scale, double* part, double* out,
                     void* stream) {
  CHECK_PARTITION(plan);
  return cuda_check(launch_restrict_op(plan->g, Sint, w1, X1, w2, X2, nrhs, part, scale, out, (cudaStream_t)stream),
                    "restrict_op");
}

int msfv_cell_gradient(const msfv_plan* plan, const double* sigma, const double* U, const double* Z,
                       const double* Y, const double* R, int32_t nrhs, double* xi, double* g, void* stream) {
  CHECK_PARTITION(plan);
  return cuda_check(launch_cell_gradient(plan->g, sigma, U, Z, Y, R, nrhs, xi, g, (cudaStream_t)stream),
                    "cell_gradient");
}

int msfv_points_interior_blocks(const msfv_points* pts, int64_t* nblocks) {
  if (!pts || !nblocks) return fail(MSFV_SHAPE, "null points");
  *nblocks = pts->d.nib;
  return MSFV_OK;
}

int msfv_points_interior_scatter(const msfv_plan* plan, const msfv_points* pts, const double* Z, int32_t nrhs,
                                 double* rhs_c, void* stream) {
  CHECK_PLAN(plan);
  if (!pts || nrhs < 0) return fail(MSFV_SHAPE, "bad interior scatter arguments");
  return cuda_check(launch_points_scatter_interior(plan->g, pts->d, Z, nrhs, rhs_c, (cudaStream_t)stream),
                    "points_interior_scatter");
}

int msfv_points_interior_solve(const msfv_plan* plan, const msfv_points* pts, const double* factor,
                               const double* rhs_c, double* out_c, int32_t nrhs, void* stream) {
  CHECK_PARTITION(plan);
  if (!pts || nrhs < 0) return fail(MSFV_SHAPE, "bad interior solve arguments");
  const Geo& g = plan->g;
  if (!tc_solver(g))
    return cuda_check(launch_block_solve_lg(g, factor, rhs_c, out_c, nrhs, (cudaStream_t)stream, pts->d.iblk,
                                            pts->d.nib, 1),
                      "points_interior_solve");
  return cuda_check(launch_block_solve_tc(g, factor, rhs_c, out_c, nrhs, (cudaStream_t)stream, pts->d.iblk, pts->d.nib, 1),
                    "points_interior_solve");
}

int msfv_block_gradient(const msfv_plan* plan, const double* sigma, const double* Sint, const double* T,
                        const double* y, int32_t nrhs, const msfv_points* pz, const double* Zc,
                        const msfv_points* pr, const double* Rc, double* g, void* stream) {
  CHECK_PARTITION(plan);
  if (nrhs < 0) return fail(MSFV_SHAPE, "bad gradient arguments");
  const Geo& gg = plan->g;
  if (gg.reduced) return fail(MSFV_UNSUPPORTED, "derivatives of reduced boundary conditions are not built");
  if (!grad_supported(gg, nrhs)) return fail(MSFV_UNSUPPORTED, "block closure exceeds shared memory");
  const bool hz = pz && pz->d.nib > 0 && Zc, hr = pr && pr->d.nib > 0 && Rc;
  return cuda_check(launch_grad_block(gg, Sint, T, y, nrhs, sigma, hz ? pz->d.islot : nullptr, Zc,
                                      hr ? pr->d.islot : nullptr, Rc, g, (cudaStream_t)stream),
                    "block_gradient");
}

int msfv_block_gradient_slab(const msfv_plan* plan, const double* sigma, const double* Sint, const double* T,
                             const double* y, int32_t nrhs, const msfv_points* pz, const double* Zc,
                             const msfv_points* pr, const double* Rc, int32_t bk0, int32_t bk1, double* g,
                             void* stream) {
  CHECK_PARTITION(plan);
  const Geo& gg = plan->g;
  if (nrhs < 0 || bk0 < 0 || bk1 > gg.nb3 || bk0 > bk1) return fail(MSFV_SHAPE, "bad gradient slab arguments");
  if (!grad_supported(gg, nrhs)) return fail(MSFV_UNSUPPORTED, "block closure exceeds shared memory");
  const bool hz = pz && pz->d.nib > 0 && Zc, hr = pr && pr->d.nib > 0 && Rc;
  const int per = gg.nb1 * gg.nb2;
  return cuda_check(launch_grad_block(gg, Sint, T, y, nrhs, sigma, hz ? pz->d.islot : nullptr, Zc,
                                      hr ? pr->d.islot : nullptr, Rc, g, (cudaStream_t)stream, bk0 * per,
                                      (bk1 - bk0) * per),
                    "block_gradient_slab");
}

int msfv_jv_coarse_rhs(const msfv_plan* plan, const double* Sint, const double* c, const double* T, int32_t nrhs,
                       const msfv_points* pr, const double* Rc, double* part, double* out, void* stream) {
  CHECK_PARTITION(plan);
  if (nrhs < 0) return fail(MSFV_SHAPE, "bad J v arguments");
  const Geo& g = plan->g;
  if (jv_smem_doubles(g, nrhs) * sizeof(double) > 200 * 1024)
    return fail(MSFV_UNSUPPORTED, "block closure exceeds shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  const bool hr = pr && pr->d.nib > 0 && Rc;
  int rc = cuda_check(launch_jv_block(g, Sint, c, T, nrhs, hr ? pr->d.islot : nullptr, Rc, part, st), "jv_block");
  if (rc) return rc;
  return cuda_check(launch_gather_corners(g, part, nrhs, -1.0, out, st), "jv_gather");
}

int msfv_yk_rhs(const msfv_plan* plan, const double* sigma, const double* Sv, double* rhs_c, uint32_t* mask,
                void* stream) {
  CHECK_PARTITION(plan);
  const Geo& g = plan->g;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t ncb = (size_t)g.b1 * g.b2 * g.b3, words = (ncb + 31) / 32;
  cudaError_t e = cudaMemsetAsync(rhs_c, 0, (size_t)g.nbl * g.nI * ncb * sizeof(double), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(mask, 0, (size_t)g.nbl * words * sizeof(uint32_t), st);
  if (e != cudaSuccess) return cuda_check(e, "yk_rhs memset");
  return cuda_check(launch_yk_rhs(g, sigma, Sv, rhs_c, mask, st), "yk_rhs");
}

int msfv_block_solve_compact(const msfv_plan* plan, const double* factor, const double* rhs_c, double* out_c,
                             int32_t nrhs, void* stream) {
  CHECK_PARTITION(plan);
  const Geo& g = plan->g;
  // wide solves (apply_Yk: one right-hand side per block cell) take the
  // CTA-per-block kernel that stages each factor tile column once for up to
  // 128 right-hand sides (the register-window kernel re-reads the factor per 16)
  if (!tc_solver(g) || nrhs >= 64)
    return cuda_check(launch_block_solve_lg(g, factor, rhs_c, out_c, nrhs, (cudaStream_t)stream, nullptr, g.nbl, 1),
                      "block_solve_compact");
  return cuda_check(launch_block_solve_tc(g, factor, rhs_c, out_c, nrhs, (cudaStream_t)stream, nullptr, g.nbl, 1),
                    "block_solve_compact");
}

int msfv_yk_rowcount(const msfv_plan* plan, const uint32_t* mask, int64_t* counts, void* stream) {
  CHECK_PLAN(plan);
  return cuda_check(launch_yk_rowcount(plan->g, mask, (long long*)counts, (cudaStream_t)stream), "yk_rowcount");
}

int msfv_yk_scatter(const msfv_plan* plan, const uint32_t* mask, const double* sol_c, const int64_t* indptr,
                    int32_t* indices, double* vals, void* stream) {
  CHECK_PLAN(plan);
  return cuda_check(launch_yk_scatter(plan->g, mask, sol_c, (const long long*)indptr, indices, vals,
                                      (cudaStream_t)stream), "yk_scatter");
}

int msfv_xk_present(const msfv_plan* plan, const double* z, int32_t* present, void* stream) {
  CHECK_PLAN(plan);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(present, 0, (size_t)plan->g.nbl * sizeof(int32_t), st);
  if (e != cudaSuccess) return cuda_check(e, "xk_present memset");
  return cuda_check(launch_xk_present(plan->g, z, present, st), "xk_present");
}

int msfv_xk_rowcount(const msfv_plan* plan, const int32_t* present, int64_t* counts, void* stream) {
  CHECK_PLAN(plan);
  return cuda_check(launch_xk_rowcount(plan->g, present, (long long*)counts, (cudaStream_t)stream), "xk_rowcount");
}

int msfv_plan_set_reduced(msfv_plan* plan, int32_t on) {
  CHECK_PARTITION(plan);
  if (on && !lg_supported(plan->g)) return fail(MSFV_UNSUPPORTED, "reduced boundary conditions need the L2 band solver");
  plan->g.reduced = on ? 1 : 0;
  plan->g.bx = nullptr;
  return MSFV_OK;
}

int msfv_boundary_reduced(const msfv_plan* plan, const double* w, double* faces, double* bx, int32_t* flags,
                          void* stream) {
  CHECK_PARTITION(plan);
  if (!plan->g.reduced) return fail(MSFV_SHAPE, "plan is not set up for reduced boundary conditions");
  if (!w || !faces || !bx || !flags) return fail(MSFV_SHAPE, "bad reduced boundary arguments");
  return cuda_check(launch_reduced_boundary(plan->g, w, faces, bx, flags, (cudaStream_t)stream), "boundary_reduced");
}

int msfv_plan_bind_boundary(msfv_plan* plan, const double* bx) {
  CHECK_PARTITION(plan);
  if (!plan->g.reduced) return fail(MSFV_SHAPE, "plan is not set up for reduced boundary conditions");
  plan->g.bx = bx;
  return MSFV_OK;
}

int msfv_basis_csc_box(int64_t nnz, const double* Sint, const int64_t* src, const int64_t* bsrc, const double* bx,
                       double* vals, void* stream) {
  return cuda_check(launch_basis_csc_box(nnz, Sint, (const long long*)src, (const long long*)bsrc, bx, vals,
                                         (cudaStream_t)stream),
                    "basis_csc_box");
}

int msfv_fine_apply(const msfv_plan* plan, const double* w, const double* X, int32_t nrhs, double* out,
                    void* stream) {
  CHECK_PLAN(plan);
  if (nrhs < 0 || !w || !X || !out) return fail(MSFV_SHAPE, "bad fine apply arguments");
  return cuda_check(launch_apply_full(plan->g, w, X, nrhs, out, (cudaStream_t)stream), "fine_apply");
}

int msfv_full_gradient(const msfv_plan* plan, const double* sigma, const double* U, const double* V, int32_t nrhs,
                       double* xi, double* g, void* stream) {
  CHECK_PLAN(plan);
  if (nrhs < 0 || !sigma || !U || !V || !xi || !g) return fail(MSFV_SHAPE, "bad full gradient arguments");
  return cuda_check(launch_full_gradient(plan->g, sigma, U, V, nrhs, xi, g, (cudaStream_t)stream), "full_gradient");
}

int msfv_edge_grad(const msfv_plan* plan, const double* X, int32_t ncol, double* out, void* stream) {
  CHECK_PLAN(plan);
  if (ncol < 0 || !X || !out) return fail(MSFV_SHAPE, "bad edge gradient arguments");
  return cuda_check(launch_edge_grad(plan->g, X, ncol, out, (cudaStream_t)stream), "edge_grad");
}

int msfv_edge_div(const msfv_plan* plan, const double* F, int32_t ncol, double* out, void* stream) {
  CHECK_PLAN(plan);
  if (ncol < 0 || !F || !out) return fail(MSFV_SHAPE, "bad edge divergence arguments");
  return cuda_check(launch_edge_div(plan->g, F, ncol, out, (cudaStream_t)stream), "edge_div");
}

int msfv_cell_gather(const msfv_plan* plan, const double* sigma, const double* xi, double* g, void* stream) {
  CHECK_PLAN(plan);
  if (!sigma || !xi || !g) return fail(MSFV_SHAPE, "bad cell gather arguments");
  return cuda_check(launch_cell_gather(plan->g, sigma, xi, g, (cudaStream_t)stream), "cell_gather");
}

int msfv_reg_apply(const msfv_plan* plan, double alpha, const double* v, double* out, void* stream) {
  CHECK_PLAN(plan);
  if (!v || !out) return fail(MSFV_SHAPE, "bad regularizer arguments");
  return cuda_check(launch_reg_apply(plan->g, alpha, v, out, (cudaStream_t)stream), "reg_apply");
}

int msfv_reg_faces(const msfv_plan* plan, const double* d, double* out, void* stream) {
  CHECK_PLAN(plan);
  if (!d || !out) return fail(MSFV_SHAPE, "bad regularizer arguments");
  return cuda_check(launch_reg_faces(plan->g, d, out, (cudaStream_t)stream), "reg_faces");
}

int msfv_xk_values(const msfv_plan* plan, const double* sigma, const double* Sint, const double* z,
                   const int32_t* present, const int64_t* indptr, int32_t* indices, double* vals, void* stream) {
  CHECK_PARTITION(plan);
  const Geo& g = plan->g;
  return cuda_check(launch_xk_values(g, sigma, Sint, z, present, (const long long*)indptr, indices, vals,
                                     (cudaStream_t)stream), "xk_values");
}

int msfv_coarse_dense(const msfv_plan* plan, const double* Kloc, double shift, double* out, void* stream) {
  CHECK_PARTITION(plan);
  return cuda_check(launch_coarse_dense(plan->g, Kloc, shift, out, (cudaStream_t)stream), "coarse_dense");
}

}  // extern "C"
