/*
 * msfv.h -- C-ABI of the B200-native adaptive MSFV forward + gradient path.
 *
 * This is the drop-in boundary.  The reference package (msinv, pure Python,
 * /root/reference/pkg/src/msinv) has no native interface; each entry point
 * below replaces the reference function cited next to it, and the Python
 * mirror package (paper_1707_07598_b200) binds them with ctypes exactly as a
 * maintainer would bind them from the reference.
 *
 * Conventions
 *  - All array arguments marked "device" are CUDA device pointers to float64
 *    (or int32 flags) owned by the caller (PyTorch tensors in the shim); the
 *    library allocates nothing per call.  Host arrays are only read.
 *  - `stream` is a cudaStream_t passed as void*; every call only enqueues work.
 *  - Index conventions are the reference's (x-fastest nodes/cells, edges
 *    x-then-y-then-z, pinned node 0 dropped, coarse columns in node order).
 *  - "Full node field" F: F[node * nrhs + s] over all (n1+1)(n2+1)(n3+1)
 *    nodes including the pinned node 0, whose entries are kept at zero.
 *  - Return value: MSFV_OK or an error code; msfv_last_error() describes it.
 *    The shim maps codes onto the reference exception types (errors.py:4-28).
 */
#ifndef MSFV_H
#define MSFV_H

#include <stdint.h>

#if defined(__GNUC__)
#define MSFV_API __attribute__((visibility("default")))
#else
#define MSFV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MSFV_ABI_VERSION 2

enum msfv_status {
  MSFV_OK = 0,
  MSFV_INVALID_MODEL = 1,     /* InvalidModelError   operators.py:26-27,128-129 */
  MSFV_STALE_BASIS = 2,       /* StaleBasisError     basis.py:333-337          */
  MSFV_REDUCED_SINGULAR = 3,  /* ReducedSingularError forward.py:126-129       */
  MSFV_SHAPE = 4,             /* ValueError (shapes / unsupported geometry)     */
  MSFV_CUDA = 5,              /* RuntimeError (CUDA failure)                    */
  MSFV_FACTORIZATION = 6,     /* FactorizationError  solvers.py:34-38           */
  MSFV_UNSUPPORTED = 7
};

/* Device flag bits written by msfv_operator / msfv_basis_build / msfv_coarse_factor. */
#define MSFV_FLAG_NONFINITE 1
#define MSFV_FLAG_NONPOSITIVE 2
#define MSFV_FLAG_LOCAL_NOT_SPD 4
#define MSFV_FLAG_COARSE_NOT_SPD 8

/* msfv_plan_info indices */
enum msfv_info {
  MSFV_INFO_NN = 0,          /* nodes incl. pinned                          */
  MSFV_INFO_N = 1,           /* pinned dimension n = NN - 1                 */
  MSFV_INFO_NCELLS = 2,
  MSFV_INFO_NEDGES = 3,
  MSFV_INFO_NBLOCKS = 4,
  MSFV_INFO_NI = 5,          /* interior nodes per block                    */
  MSFV_INFO_P1S = 6,         /* row stride of the per-block factor bands    */
  MSFV_INFO_K = 7,           /* coarse columns (Lagrange: coarse nodes)     */
  MSFV_INFO_AK_DOUBLES = 8,  /* size of the coarse factor buffer            */
  MSFV_INFO_BASIS_SMEM = 9,
  MSFV_INFO_NT = 10,
  MSFV_INFO_PT = 11,
  MSFV_INFO_TB = 12,
  MSFV_INFO_PC = 13,
  MSFV_INFO_FACTOR_DOUBLES = 14,  /* size of the per-model local factor buffer  */
  MSFV_INFO_SCRATCH_DOUBLES = 15, /* scratch needed by msfv_basis_build         */
  MSFV_INFO_TC = 16,              /* local solver: 1 DMMA register-window band (p <= 56, split build),
                                     2 DMMA L2-resident band (larger blocks)     */
  MSFV_INFO_COARSE = 17,          /* coarse solver: 0 band, 1 z-plane ND band, 2 multifrontal ND */
  MSFV_INFO_RED_FACE_DOUBLES = 18, /* msfv_boundary_reduced face scratch (reduced plans)        */
  MSFV_INFO_RED_BOX_DOUBLES = 19,  /* msfv_boundary_reduced box table [nblocks][8][(b+1)^3]      */
  MSFV_INFO_COUNT = 20
};

typedef struct msfv_plan msfv_plan;      /* geometry; model-independent        */
typedef struct msfv_points msfv_points;  /* one survey matrix (P or Q) on device */

MSFV_API int msfv_abi_version(void);
MSFV_API const char* msfv_last_error(void);
/* Number of kernels this library has launched so far (process-wide counter). */
MSFV_API int64_t msfv_launch_count(void);

/* TensorMesh + CoarsePartition (mesh.py:12-182).  blocks must divide cells. */
MSFV_API int msfv_plan_create(const int32_t cells[3], const double h[3], const int32_t blocks[3], msfv_plan** out);
/* Geometry-only plan (no coarse partition) for the fine-mesh entry points
 * (msfv_operator, msfv_edge_average, msfv_fine_apply, msfv_full_gradient,
 * msfv_reg_*, survey scatter/receive without basis); every basis or coarse
 * entry point returns MSFV_UNSUPPORTED on it.  At most 1023 cells per axis. */
MSFV_API int msfv_plan_create_mesh(const int32_t cells[3], const double h[3], msfv_plan** out);
MSFV_API void msfv_plan_destroy(msfv_plan* plan);
MSFV_API int msfv_plan_info(const msfv_plan* plan, int64_t* info, int32_t n);

/* A sparse pinned-space survey matrix in CSC form (Survey.P / Survey.Q,
 * forward.py:23-51; models.py:54-83).  Host arrays; uploaded once. */
MSFV_API int msfv_points_create(const msfv_plan* plan, int64_t nnz, int32_t ncol, const int64_t* colptr,
                       const int64_t* rows, const double* vals, msfv_points** out);
MSFV_API void msfv_points_destroy(msfv_points* pts);

/* sigma = exp(m), w = C sigma (operators.py:23-28,123-136).  flags |= NONFINITE/NONPOSITIVE. */
MSFV_API int msfv_operator(const msfv_plan* plan, const double* m, double* sigma, double* w, int32_t* flags, void* stream);
/* c = C (sigma .* dm)   (Csig @ dm, forward.py:237,259); tmp: ncells doubles */
MSFV_API int msfv_edge_average(const msfv_plan* plan, const double* sigma, const double* dm, double* tmp, double* c,
                      void* stream);

/* Lagrange basis at w (assemble_basis, basis.py:511-616 with _BlockFactor
 * basis.py:258-298; every block size the reference accepts up to a half
 * bandwidth ni1*ni2 <= 512, e.g. 16^3-cell blocks): per-block banded Cholesky factors (factor buffer of
 * MSFV_INFO_FACTOR_DOUBLES; opaque layout), interior basis values Sint
 * [nblocks][8][nI] and the per-block 8x8 Galerkin blocks Kloc [nblocks][64].
 * scratch: MSFV_INFO_SCRATCH_DOUBLES doubles.  flags |= LOCAL_NOT_SPD. */
MSFV_API int msfv_basis_build(const msfv_plan* plan, const double* w, double* factor, double* Sint, double* Kloc,
                     double* scratch, int32_t* flags, void* stream);
/* The same build in two launches (tensor-core geometries only): the forward
 * part (factors, Galerkin blocks, and y = L^{-1} R parked in Sint) and the
 * backward sweeps (Sint = S_I).  The Galerkin blocks do not need the backward
 * sweeps, so the coarse factorization can run while msfv_basis_backward
 * executes on another stream (a small persistent grid that leaves a CTA slot
 * per SM for the cooperative factorization). */
MSFV_API int msfv_basis_forward(const msfv_plan* plan, const double* w, double* factor, double* Sint, double* Kloc,
                       int32_t* flags, void* stream);
MSFV_API int msfv_basis_backward(const msfv_plan* plan, const double* factor, double* Sint, void* stream);
/* Values of S in the reference CSC pattern (basis.py:574-594):
 * vals[t] = src[t] >= 0 ? Sint[src[t]] : hatv[t]  (src, hatv device arrays). */
MSFV_API int msfv_basis_csc(int64_t nnz, const double* Sint, const int64_t* src, const double* hatv, double* vals,
                   void* stream);

/* A_k = S^T A S (+ shift I) into the tiled band buffer (forward.py:101-102,117-125). */
MSFV_API int msfv_galerkin(const msfv_plan* plan, const double* Kloc, double shift, double* Ak, void* stream);
/* diag(A_k) (for the shift 1e-12 tr(A_k)/k, forward.py:123) */
MSFV_API int msfv_coarse_diag(const msfv_plan* plan, const double* Ak, double* diag, void* stream);
/* In-place banded Cholesky of A_k (cho_factor, forward.py:121). flags |= COARSE_NOT_SPD. */
MSFV_API int msfv_coarse_factor(const msfv_plan* plan, double* Ak, int32_t* flags, void* stream);
/* X <- A_k^{-1} X, X [k][nrhs] (cho_solve, forward.py:72-75); scratch: k*nrhs doubles. */
MSFV_API int msfv_coarse_solve(const msfv_plan* plan, const double* Lk, double* X, double* scratch, int32_t nrhs,
                               void* stream);

/* out[col][s] = sum_t val_t (Xfield(node_t,s) + S(node_t,:) Y[:,s]); Y or Xfield may be NULL.
 * (P^T S T forward.py:143; P^T (ydm + S dt) forward.py:268) */
MSFV_API int msfv_survey_receive(const msfv_plan* plan, const msfv_points* pts, const double* Sint, const double* Y,
                        const double* Xfield, int32_t nrhs, double* out, void* stream);

/* misfit_ssd on the device (inversion.py:22-29): resid[i] = D[i] - D_obs[i] (n = receivers x sources
 * entries) and phi[0] = 0.5 sum resid^2, one launch, fixed summation order. */
MSFV_API int msfv_misfit(const double* D, const double* D_obs, int64_t n, double* resid, double* phi, void* stream);
/* out[c][s] = (S^T M Z)[c][s]; Z [ncol][nrhs] or NULL for the identity (S^T Q, forward.py:115). */
MSFV_API int msfv_survey_restrict(const msfv_plan* plan, const msfv_points* pts, const double* Sint, const double* Z,
                         int32_t nrhs, double* out, void* stream);
/* field(node,s) = (M Z)(node,s) on the survey's nodes (other entries untouched). */
MSFV_API int msfv_survey_scatter(const msfv_plan* plan, const msfv_points* pts, const double* Z, int32_t nrhs,
                        double* field, void* stream);

/* field = S Y on every node (basis.S @ T, forward.py:143,241). */
MSFV_API int msfv_prolong(const msfv_plan* plan, const double* Sint, const double* Y, int32_t nrhs, double* field,
                 void* stream);
/* out = alpha*src + beta*(A_wt X) on block-interior nodes (forward.py:243,278). src may be NULL. */
MSFV_API int msfv_residual(const msfv_plan* plan, const double* src, double alpha, const double* wt, const double* X,
                  double beta, int32_t nrhs, double* out, void* stream);
/* out = blockdiag(A_II^{-1}) rhs on interiors (MultiscaleBasis.interior_solve, basis.py:339-353). */
MSFV_API int msfv_interior_solve(const msfv_plan* plan, const double* factor, const double* rhs, double* out,
                        int32_t nrhs, void* stream);
/* out[k][nrhs] = scale * S^T (A_w1 X1 + A_w2 X2); part: nblocks*8*nrhs scratch (forward.py:266).
 * A null w_i takes the field X_i itself (S^T X: restriction of a node field). */
MSFV_API int msfv_restrict_op(const msfv_plan* plan, const double* Sint, const double* w1, const double* X1,
                     const double* w2, const double* X2, int32_t nrhs, double scale, double* part, double* out,
                     void* stream);
/* g = -sigma C^T sum_s [G U (G Z + G Y) + G R G Y]  (rapply compact form, forward.py:271-281).
 * xi: nedges doubles of scratch (the per-edge sums). */
MSFV_API int msfv_cell_gradient(const msfv_plan* plan, const double* sigma, const double* U, const double* Z,
                       const double* Y, const double* R, int32_t nrhs, double* xi, double* g, void* stream);

/* Interior-only survey fields.  The Lagrange columns solve their local
 * problems, (A S)_I = 0, so interior_solve(Q - A S T) = blockdiag(A_II^-1) Q_I
 * and interior_solve(P W - A S y) = blockdiag(A_II^-1) (P W)_I
 * (forward.py:240-246,278): nonzero only on the blocks whose interiors hold
 * survey nodes.  Compact fields hold nblocks x nI x nrhs doubles (slot-major).
 * msfv_points_interior_blocks: number of such blocks of a point set. */
MSFV_API int msfv_points_interior_blocks(const msfv_points* pts, int64_t* nblocks);
/* rhs_c = (M Z)_I on the interior slots (Z = NULL: the identity, i.e. M itself) */
MSFV_API int msfv_points_interior_scatter(const msfv_plan* plan, const msfv_points* pts, const double* Z, int32_t nrhs,
                                 double* rhs_c, void* stream);
/* out_c = blockdiag(A_II^-1) rhs_c on the interior slots (out_c may alias rhs_c) */
MSFV_API int msfv_points_interior_solve(const msfv_plan* plan, const msfv_points* pts, const double* factor,
                               const double* rhs_c, double* out_c, int32_t nrhs, void* stream);
/* Fused per-block rapply gradient (forward.py:270-281, the msfv_cell_gradient
 * sum without node fields): g = -sigma C^T xi with
 *   xi_e = sum_s [dU (dZ + dY) + dR dY] / h_e^2,  U = S T, Y = S y,
 * Z / R the compact interior fields of pz / pr (NULL when the point set has no
 * interior blocks).  MSFV_UNSUPPORTED when the block closure does not fit in
 * shared memory. */
MSFV_API int msfv_block_gradient(const msfv_plan* plan, const double* sigma, const double* Sint, const double* T,
                        const double* y, int32_t nrhs, const msfv_points* pz, const double* Zc,
                        const msfv_points* pr, const double* Rc, double* g, void* stream);
/* Slab forms of msfv_operator / msfv_basis_forward for pipelining the model
 * upload: msfv_operator_slab computes sigma on cell planes k0 .. min(k1, n3-1)
 * and the edge weights of node planes k0..k1 (x-, y-edges) and cell planes
 * k0..k1-1 (z-edges) -- the edges of the blocks with bk0*b3 = k0, bk1*b3 = k1;
 * it reads m on cell planes k0 .. min(k1, n3-1) only.  msfv_basis_forward_slab
 * builds the blocks bk0 <= bk < bk1 (their w must be complete). */
MSFV_API int msfv_operator_slab(const msfv_plan* plan, const double* m, double* sigma, double* w, int32_t* flags,
                                int32_t k0, int32_t k1, void* stream);
MSFV_API int msfv_basis_forward_slab(const msfv_plan* plan, const double* w, double* factor, double* Sint,
                                     double* Kloc, int32_t* flags, int32_t bk0, int32_t bk1, void* stream);
/* Same, for the blocks of the z-slab bk0 <= bk < bk1 only (they own the cells
 * with bk0*b3 <= k < bk1*b3, a contiguous range of g): lets the host copy
 * finished slabs of g back while the next slab is computed. */
MSFV_API int msfv_block_gradient_slab(const msfv_plan* plan, const double* sigma, const double* Sint, const double* T,
                             const double* y, int32_t nrhs, const msfv_points* pz, const double* Zc,
                             const msfv_points* pr, const double* Rc, int32_t bk0, int32_t bk1, double* g,
                             void* stream);
/* Coarse right-hand side of J v for surveys without interior receivers
 * (forward.py:258-269): out = xdm - S^T(gdm + A ydm) = -EP^T((G U + G R) o c)
 * with U = S T, R the compact interior field of pr (NULL: none) and c = Csig dm
 * (msfv_edge_average).  The S^T A ydm term vanishes because (A S)_I = 0 and
 * ydm lives on block interiors.  part: nblocks*8*nrhs doubles of scratch;
 * out: k x nrhs. */
MSFV_API int msfv_jv_coarse_rhs(const msfv_plan* plan, const double* Sint, const double* c, const double* T, int32_t nrhs,
                       const msfv_points* pr, const double* Rc, double* part, double* out, void* stream);
/* Dense natural-order A_k (+ shift I), both triangles, k x k doubles: the
 * reference's `ReducedState.A_k` attribute (forward.py:62-75,101-102). */
MSFV_API int msfv_coarse_dense(const msfv_plan* plan, const double* Kloc, double shift, double* out, void* stream);

/* ---- Table-3 operators: materialized basis derivatives (basis.py:684-800) ----
 * apply_Yk: W = G_p^T diag(G_p S v) Csig restricted to block interiors and the
 * block's cells; Y_k = -blockdiag(A_II^-1) W as an n x N_m CSR.
 *   msfv_yk_rhs: rhs_c[nblocks][nI][b1*b2*b3] = W (zeroed first) from Sv = S v
 *     (a node field, msfv_prolong) and sigma; mask[nblocks][ceil(b1b2b3/32)]
 *     marks the non-zero columns (the reference's Wd.any(axis=0)).
 *   msfv_block_solve_compact: out_c = blockdiag(A_II^-1) rhs_c for all blocks
 *     (compact layout, block-major).
 *   msfv_yk_rowcount: entries per pinned row; msfv_yk_scatter: CSR (int32
 *     indices, ascending) of -out_c with the row pointer from the counts.
 * apply_Xk: z = interior_solve(w) (msfv_interior_solve, node field).
 *   msfv_xk_present: blocks with z != 0 (the reference's np.any(a_j));
 *   msfv_xk_rowcount: entries per coarse row; msfv_xk_values: CSR values and
 *   ascending column indices. */
MSFV_API int msfv_yk_rhs(const msfv_plan* plan, const double* sigma, const double* Sv, double* rhs_c, uint32_t* mask,
                void* stream);
MSFV_API int msfv_block_solve_compact(const msfv_plan* plan, const double* factor, const double* rhs_c, double* out_c,
                             int32_t nrhs, void* stream);
MSFV_API int msfv_yk_rowcount(const msfv_plan* plan, const uint32_t* mask, int64_t* counts, void* stream);
MSFV_API int msfv_yk_scatter(const msfv_plan* plan, const uint32_t* mask, const double* sol_c, const int64_t* indptr,
                    int32_t* indices, double* vals, void* stream);
MSFV_API int msfv_xk_present(const msfv_plan* plan, const double* z, int32_t* present, void* stream);
MSFV_API int msfv_xk_rowcount(const msfv_plan* plan, const int32_t* present, int64_t* counts, void* stream);
MSFV_API int msfv_xk_values(const msfv_plan* plan, const double* sigma, const double* Sint, const double* z,
                   const int32_t* present, const int64_t* indptr, int32_t* indices, double* vals, void* stream);

/* ---- Reduced-dimension boundary conditions (an extension:
 * the reference uses the trilinear hats, basis.py:84-116) ----
 * msfv_plan_set_reduced(plan, 1): the plan's basis entry points use skeleton
 *   values from 1D line problems (normalized cumulative resistance along each
 *   skeleton segment) and 2D face-patch problems (5-point, in-plane edge
 *   weights w_e/h_e^2) instead of the hats; local solves take the L2 band path.
 * msfv_boundary_reduced: computes them from the edge weights w into the box
 *   table bx [nblocks][8][(b1+1)(b2+1)(b3+1)] (faces: scratch of
 *   MSFV_INFO_RED_FACE_DOUBLES); flags |= LOCAL_NOT_SPD on a failed face solve.
 * msfv_plan_bind_boundary: the table the following launches read (one model
 *   at a time, like the basis it belongs to).
 * msfv_basis_csc_box: S values in the reference CSC pattern, skeleton entries
 *   from the table (bsrc: flat index into bx).
 * The fused block gradient and the Y_k / X_k operators refuse reduced plans
 * (MSFV_UNSUPPORTED): the sensitivities through the boundary problems run on
 * node and edge fields (msfv_prolong, msfv_restrict_op, msfv_fine_apply,
 * msfv_interior_solve, msfv_edge_grad / msfv_edge_div, msfv_cell_gather read
 * the bound table), composed by the host (reduced_sens.py). */
MSFV_API int msfv_plan_set_reduced(msfv_plan* plan, int32_t on);
MSFV_API int msfv_boundary_reduced(const msfv_plan* plan, const double* w, double* faces, double* bx, int32_t* flags,
                                   void* stream);
MSFV_API int msfv_plan_bind_boundary(msfv_plan* plan, const double* bx);
MSFV_API int msfv_basis_csc_box(int64_t nnz, const double* Sint, const int64_t* src, const int64_t* bsrc,
                                const double* bx, double* vals, void* stream);

/* ---- Fine mesh (forward_full, FullSensitivity, block_cg) ----
 * msfv_fine_apply: out = A(w) X on every pinned node (the operator product
 *   op.A @ X of forward.py:84-90 and solvers.py:105; operators.py:138-141),
 *   X and out full node fields [node][nrhs] (row 0, the pinned node, is 0).
 * msfv_full_gradient: g = -sigma C^T sum_s (G U_s) o (G V_s) -- the adjoint
 *   product sum_j G_j^T v_j of FullSensitivity.rapply (forward.py:170-175)
 *   with G_j = d(A u_j)/dm = G^T diag(G u_j) C diag(sigma)
 *   (grad_A_u, operators.py:168-194); xi: nedges doubles of scratch. */
MSFV_API int msfv_fine_apply(const msfv_plan* plan, const double* w, const double* X, int32_t nrhs, double* out,
                             void* stream);
MSFV_API int msfv_full_gradient(const msfv_plan* plan, const double* sigma, const double* U, const double* V,
                                int32_t nrhs, double* xi, double* g, void* stream);
/* ---- edge-space pieces for the enriched basis families ----
 * The reference's AdaptiveSensitivity works on per-edge vectors
 * (forward.py:224-281: gprof, gu, a; basis.edge_profiles, basis.py:596-608).
 * msfv_edge_grad: out[e][c] = (G_p X)(e, c), the pinned nodal gradient
 *   (operators.py:36-74, G[:, 1:]) of ncol node fields X[node][ncol];
 * msfv_edge_div:  out[node][c] = (G_p^T F)(node, c) for edge fields
 *   F[e][ncol] (row 0, the pinned node, is 0);
 * msfv_cell_gather: g = -sigma o (C^T xi), the Csig^T products of
 *   forward.py:254-256,278-280 (C = edge_cell_map, operators.py:77-109). */
MSFV_API int msfv_edge_grad(const msfv_plan* plan, const double* X, int32_t ncol, double* out, void* stream);
MSFV_API int msfv_edge_div(const msfv_plan* plan, const double* F, int32_t ncol, double* out, void* stream);
MSFV_API int msfv_cell_gather(const msfv_plan* plan, const double* sigma, const double* xi, double* g, void* stream);
/* ---- Gauss-Newton objective (Objective, inversion.py:32-88) ----
 * L = cell_gradient(mesh): cell-centre differences across interior faces, +-1/h.
 * msfv_reg_apply: out = alpha L^T L v (Objective.hess_apply, inversion.py:87-88);
 * msfv_reg_faces: out_c = sum of (L d)_f^2 over the faces (c, c + e_axis), so
 *   ||L d||^2 = sum_c out_c (Objective.value_grad, inversion.py:82-85). */
MSFV_API int msfv_reg_apply(const msfv_plan* plan, double alpha, const double* v, double* out, void* stream);
MSFV_API int msfv_reg_faces(const msfv_plan* plan, const double* d, double* out, void* stream);

/* ==== 2D path (BASELINE.json configs 1-2) =================================
 * The reference package is 3D only; these entry points run the
 * same adaptive MSFV algorithm with d = 2: cells n1 x n2,
 * blocks b1 x b2 (>= 2 cells each), bilinear Lagrange hats, x- then y-edges,
 * C = V/2 per touching cell, node 0 pinned.  Fields are row-major
 * [pinned node][nrhs] (n = (n1+1)(n2+1) - 1 rows); coarse fields [k][nrhs] in
 * coarse-node order; edge fields [E][nrhs]; cell fields [n1 n2].
 *   Sb      [blocks][4 corners][nI]      interior basis values S_I
 *   factor  [blocks][nI][b1]             band Cholesky of A_II (row, offset)
 *   Kloc    [blocks][16]                 local Galerkin blocks
 *   Ab, Lk  [k][k_x + 2]                 lower band of A_k / its factor
 * Replaces: assemble_operator (operators.py:123-141), assemble_basis
 * (basis.py:511-616), forward_reduced (forward.py:105-144),
 * MultiscaleBasis.interior_solve (basis.py:339-353) and the products of
 * AdaptiveSensitivity (forward.py:224-281). */
typedef struct msfv2d_plan msfv2d_plan;
enum msfv2d_info {
  MSFV2D_INFO_NN = 0,
  MSFV2D_INFO_N = 1,
  MSFV2D_INFO_NCELLS = 2,
  MSFV2D_INFO_NEDGES = 3,
  MSFV2D_INFO_NBLOCKS = 4,
  MSFV2D_INFO_NI = 5,
  MSFV2D_INFO_K = 6,
  MSFV2D_INFO_FACTOR_DOUBLES = 7,
  MSFV2D_INFO_BAND_DOUBLES = 8,
  MSFV2D_INFO_COUNT = 9
};
MSFV_API int msfv2d_plan_create(const int32_t* cells, const double* h, const int32_t* blocks, msfv2d_plan** out);
MSFV_API void msfv2d_plan_destroy(msfv2d_plan* plan);
MSFV_API int msfv2d_plan_info(const msfv2d_plan* plan, int64_t* info, int32_t n);
/* sigma = exp(m) (flags |= NONFINITE on non-finite m), w = C sigma   operators.py:23-28,136 */
MSFV_API int msfv2d_operator(const msfv2d_plan* plan, const double* m, double* sigma, double* w, int32_t* flags,
                             void* stream);
/* per-block band Cholesky + 4 Lagrange solves, local Galerkin blocks   basis.py:537-563 */
MSFV_API int msfv2d_basis(const msfv2d_plan* plan, const double* w, double* factor, double* Sb, double* Kloc,
                          int32_t* flags, void* stream);
/* A_k band (+ shift on the diagonal)   forward.py:117-118,123 */
MSFV_API int msfv2d_galerkin(const msfv2d_plan* plan, const double* Kloc, double shift, double* Ab, void* stream);
/* band Cholesky of A_k (flags |= COARSE_NOT_SPD)   forward.py:119-129 */
MSFV_API int msfv2d_coarse_factor(const msfv2d_plan* plan, const double* Ab, double* Lk, int32_t* flags,
                                  void* stream);
/* X <- A_k^-1 X (k x nrhs, in place)   forward.py:72-75 */
MSFV_API int msfv2d_coarse_solve(const msfv2d_plan* plan, const double* Lk, double* X, int32_t nrhs, void* stream);
/* out = blockdiag(A_II^-1) rhs on interiors, 0 on the skeleton   basis.py:339-353 */
MSFV_API int msfv2d_interior_solve(const msfv2d_plan* plan, const double* factor, const double* rhs, double* out,
                                   int32_t nrhs, void* stream);
/* out = S Y ; out = S^T X ; out = A X ; out = G_p X ; out = G_p^T (a o c) */
MSFV_API int msfv2d_prolong(const msfv2d_plan* plan, const double* Sb, const double* Y, double* out, int32_t nrhs,
                            void* stream);
MSFV_API int msfv2d_restrict(const msfv2d_plan* plan, const double* Sb, const double* X, double* out, int32_t nrhs,
                             void* stream);
MSFV_API int msfv2d_apply_A(const msfv2d_plan* plan, const double* w, const double* X, double* out, int32_t nrhs,
                            void* stream);
MSFV_API int msfv2d_grad(const msfv2d_plan* plan, const double* X, double* out, int32_t nrhs, void* stream);
MSFV_API int msfv2d_gradT(const msfv2d_plan* plan, const double* a, const double* c, double* out, int32_t nrhs,
                          void* stream);
/* c = C (sigma o dm) ; out = -(C diag sigma)^T sum_s e[:, s]   forward.py:259,281 */
MSFV_API int msfv2d_edge_average(const msfv2d_plan* plan, const double* sigma, const double* dm, double* c,
                                 void* stream);
MSFV_API int msfv2d_cell_adjoint(const msfv2d_plan* plan, const double* sigma, const double* e, double* out,
                                 int32_t nrhs, void* stream);
/* out = beta out + M X for a CSR M (int64 row pointer, int32 columns): survey products */
MSFV_API int msfv2d_spmm(int64_t nrows, const int64_t* ptr, const int32_t* col, const double* val, const double* X,
                         int32_t nrhs, double beta, double* out, void* stream);
/* out = alpha a + b ; out = a o b + c o d + e o f (elementwise; b, c..f nullable) */
MSFV_API int msfv2d_axpby(int64_t n, double alpha, const double* a, const double* b, double* out, void* stream);
MSFV_API int msfv2d_fma3(int64_t n, const double* a, const double* b, const double* c, const double* d,
                         const double* e, const double* f, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MSFV_H */
