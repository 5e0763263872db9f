// Internal launcher declarations (not part of the public C-ABI).
#pragma once
#include <mutex>
#include <string>
#include <unordered_map>
#include <cuda_runtime.h>
#include "msfv_common.cuh"

namespace msfv {

// A lazily initialised per-device value (function attributes, occupancy-
// derived grid sizes, helper allocations): keyed by the current device and
// initialised once under a mutex, so several devices or host threads in one
// process each get their own, race-free.
template <class T>
struct PerDevice {
  std::mutex mu;
  std::unordered_map<int, T> vals;
  template <class F>
  T get(F&& init) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = vals.find(dev);
    if (it != vals.end()) return it->second;
    T v = init();
    vals.emplace(dev, v);
    return v;
  }
};

constexpr int RESTRICT_THREADS = 128;
constexpr int COARSE_TB = 32;
constexpr int TC_WARPS = 2;      // warps (= coarse blocks) per CTA in the DMMA kernels
constexpr int TC_MAX_PT = 7;     // largest tile band handled by the DMMA kernels (p <= 56)

constexpr int FLAG_NONFINITE = 1;
constexpr int FLAG_NONPOSITIVE = 2;
constexpr int FLAG_LOCAL_NOT_SPD = 4;
constexpr int FLAG_COARSE_NOT_SPD = 8;

void count_launches(long long n);
// record msg as msfv_last_error() and return code (msfv_capi.cu)
int set_error(int code, const std::string& msg);
// multifrontal coarse plan (msfv_coarse.cu): built at plan creation when coarse_nd == 2
bool mf_attach(Geo& g);
int mf_reserved_sms();   // SMs the multifrontal kernels leave to the backward basis sweeps   // false (and g.mf = nullptr) when the fronts exceed the kernels' shared memory
void mf_release(Geo& g);
long long launch_count();


cudaError_t launch_sigma(long long Nm, const double* m, const double* mul, double* out, int* flags, cudaStream_t st);
cudaError_t launch_mul(long long n, const double* a, const double* b, double* out, cudaStream_t st);
cudaError_t launch_edge_weights(const Geo& g, const double* cv, double* w, cudaStream_t st);
cudaError_t launch_residual(const Geo& g, const double* src, double alpha, const double* wt, const double* X,
                            double beta, int nrhs, double* out, cudaStream_t st);
cudaError_t launch_prolong(const Geo& g, const double* Sint, const double* Y, int nrhs, double* out, cudaStream_t st);
cudaError_t launch_restrict_op(const Geo& g, const double* Sint, const double* w1, const double* X1,
                               const double* w2, const double* X2, int nrhs, double* part, double scale,
                               double* out, cudaStream_t st);
cudaError_t launch_cell_gradient(const Geo& g, const double* sigma, const double* U, const double* Z,
                                 const double* Y, const double* R, int nrhs, double* xi, double* gout,
                                 cudaStream_t st);
// g_c = -sigma_c (V/4) sum over the cell's 12 edges of xi_e (msfv_block.cu)
cudaError_t launch_cell_gather(const Geo& g, const double* sigma, const double* xi, double* gout, cudaStream_t st);
// fine mesh and Gauss-Newton objective (msfv_fine.cu)
cudaError_t launch_apply_full(const Geo& g, const double* w, const double* X, int nrhs, double* out, cudaStream_t st);
cudaError_t launch_full_gradient(const Geo& g, const double* sigma, const double* U, const double* V, int nrhs,
                                 double* xi, double* gout, cudaStream_t st);
cudaError_t launch_edge_grad(const Geo& g, const double* X, int ncol, double* out, cudaStream_t st);
cudaError_t launch_edge_div(const Geo& g, const double* F, int ncol, double* out, cudaStream_t st);
cudaError_t launch_reg_apply(const Geo& g, double alpha, const double* v, double* out, cudaStream_t st);
cudaError_t launch_reg_faces(const Geo& g, const double* d, double* out, cudaStream_t st);
cudaError_t launch_basis_csc(long long nnz, const double* Sint, const long long* src, const double* hatv,
                             double* vals, cudaStream_t st);

// DMMA tile-band path (msfv_tc.cu)
int tc_band(const Geo& g);
bool tc_supported(const Geo& g);
size_t tc_factor_doubles(const Geo& g);
size_t tc_scratch_doubles(const Geo& g);
cudaError_t launch_misfit(const double* D, const double* Dobs, long long n, double* resid, double* phi,
                          cudaStream_t st);
cudaError_t launch_lg_galerkin(const Geo& g, const double* w, const double* Sint, double* Kloc, cudaStream_t st);
cudaError_t launch_basis_tc(const Geo& g, const double* w, double* LT, double* Sint, double* Kloc,
                            int* flags, cudaStream_t st, bool bwd = true, int jb0 = 0, int jb1 = -1);
cudaError_t launch_edge_weights_planes(const Geo& g, const double* cv, double* w, int k0, int k1, cudaStream_t st);
cudaError_t launch_basis_bwd(const Geo& g, const double* LT, double* Sint, cudaStream_t st);
cudaError_t launch_block_solve_tc(const Geo& g, const double* LT, const double* rhs, double* out, int nrhs,
                                  cudaStream_t st, const int* blist = nullptr, int nlist = 0, int compact = 0);

// L2-resident DMMA band path for larger blocks (msfv_large.cu)
constexpr int LG_MAX_PT = 64;    // half bandwidth p <= 512
int lg_band(const Geo& g);
bool lg_supported(const Geo& g);
size_t lg_factor_doubles(const Geo& g);
cudaError_t launch_basis_lg(const Geo& g, const double* w, double* LT, double* Sint, double* Kloc, int* flags,
                            cudaStream_t st);
cudaError_t launch_block_solve_lg(const Geo& g, const double* LT, const double* rhs, double* out, int nrhs,
                                  cudaStream_t st, const int* blist = nullptr, int nlist = 0, int compact = 0);

// reduced-dimension boundary conditions (msfv_reduced.cu)
size_t red_face_doubles(const Geo& g);
size_t red_box_doubles(const Geo& g);
cudaError_t launch_reduced_boundary(const Geo& g, const double* w, double* fv, double* bx, int* flags,
                                    cudaStream_t st);
cudaError_t launch_basis_csc_box(long long nnz, const double* Sint, const long long* src, const long long* bsrc,
                                 const double* bx, double* vals, cudaStream_t st);

// coarse (msfv_coarse.cu)
cudaError_t launch_coarse_assemble(const Geo& g, const double* Kloc, double shift, double* Ak, cudaStream_t st);
cudaError_t launch_coarse_factor(const Geo& g, double* Ak, int* flags, cudaStream_t st);
cudaError_t launch_coarse_solve(const Geo& g, const double* Lk, double* X, double* scratch, int nrhs, cudaStream_t st);
size_t coarse_doubles(const Geo& g);
size_t coarse_scratch_doubles(const Geo& g, int nrhs);
cudaError_t launch_coarse_diag(const Geo& g, const double* Ak, double* diag, cudaStream_t st);
cudaError_t launch_coarse_dense(const Geo& g, const double* Kloc, double shift, double* out, cudaStream_t st);
int coarse_tile_rows(const Geo& g);

// survey point sets (msfv_points.cu)
struct PointsDev {
  long long nnz;
  int ncol;
  const long long* colptr;   // [ncol+1]
  const long long* node;     // [nnz] full node id
  const int* col;            // [nnz]
  const double* val;         // [nnz]
  const int* blk;            // [nnz] owner block
  const int* loc;            // [nnz] packed local coords x | y<<10 | z<<20
  const long long* cptr;     // [kc+1] coarse -> entries
  const long long* cent;     // [..] packed (t << 3) | cc
  long long nu;              // unique nodes
  const long long* uptr;     // [nu+1]
  const long long* unode;    // [nu]
  const long long* uent;     // [nnz] entry ids grouped by node
  int nib;                   // blocks with entries on interior nodes
  const int* islot;          // [nbl] compact slot of a block or -1
  const int* iblk;           // [nib] block of a slot
  const long long* urow;     // [nu] compact row slot*nI + a of a unique node or -1
};
cudaError_t launch_points_receive(const Geo& g, const PointsDev& P, const double* Sint, const double* Y,
                                  const double* Xf, int nrhs, double* out, cudaStream_t st);
cudaError_t launch_points_restrict(const Geo& g, const PointsDev& P, const double* Sint, const double* Z,
                                   int nrhs, double* out, cudaStream_t st);
cudaError_t launch_points_scatter(const Geo& g, const PointsDev& P, const double* Z, int nrhs, double* field,
                                  cudaStream_t st);
// compact interior fields of the survey's interior blocks (zeroed, then scattered)
cudaError_t launch_points_scatter_interior(const Geo& g, const PointsDev& P, const double* Z, int nrhs, double* rhs_c,
                                           cudaStream_t st);

// fused per-block gradient (msfv_grad.cu)
constexpr int GRAD_THREADS = 256;
size_t grad_smem_doubles(const Geo& g, int nrhs);
bool grad_supported(const Geo& g, int nrhs);
bool grad_template_init(const Geo& g);   // 8^3 blocks: upload the closure template to the current device
cudaError_t launch_grad_block(const Geo& g, const double* Sint, const double* T, const double* Y, int nrhs,
                              const double* sigma, const int* zslot, const double* Zc, const int* rslot,
                              const double* Rc, double* gout, cudaStream_t st, int jb0 = 0, int nb = -1);
size_t jv_smem_doubles(const Geo& g, int nrhs);
cudaError_t launch_jv_block(const Geo& g, const double* Sint, const double* cvec, const double* T, int nrhs,
                            const int* rslot, const double* Rc, double* part, cudaStream_t st);
// Table-3 operators (msfv_table3.cu)
cudaError_t launch_yk_rhs(const Geo& g, const double* sigma, const double* Sv, double* rhs, unsigned* mask,
                          cudaStream_t st);
cudaError_t launch_yk_rowcount(const Geo& g, const unsigned* mask, long long* counts, cudaStream_t st);
cudaError_t launch_yk_scatter(const Geo& g, const unsigned* mask, const double* sol, const long long* indptr,
                              int* indices, double* vals, cudaStream_t st);
cudaError_t launch_xk_present(const Geo& g, const double* zf, int* present, cudaStream_t st);
cudaError_t launch_xk_rowcount(const Geo& g, const int* present, long long* counts, cudaStream_t st);
size_t xk_smem_bytes(const Geo& g);
cudaError_t launch_xk_values(const Geo& g, const double* sigma, const double* Sint, const double* zf, const int* present,
                             const long long* indptr, int* indices, double* vals, cudaStream_t st);
cudaError_t launch_gather_corners(const Geo& g, const double* part, int nrhs, double scale, double* out,
                                  cudaStream_t st);

}  // namespace msfv
