"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``msinv`` from /root/reference/pkg/src (read-only, never copied)
and writes one small ``.npz`` per case next to this script.  The fixtures
pin the CPU oracle (tests/test_oracle_golden.py) and the GPU path
(tests/test_gpu_parity.py); neither reads /root/reference at run time.
"""

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import numpy as np                                    # noqa: E402
import scipy.ndimage as ndi                           # noqa: E402
import scipy.sparse as sp                             # noqa: E402

from msinv.basis import BasisBuilder, BasisSpec, apply_Xk, apply_Yk  # noqa: E402
from msinv.forward import Survey, forward_reduced, sensitivity_adaptive  # noqa: E402
from msinv.inversion import misfit_ssd                # noqa: E402
from msinv.mesh import create_mesh, create_partition  # noqa: E402
from msinv.models import build_survey                 # noqa: E402
from msinv.operators import assemble_operator         # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def random_survey(mesh, n_rec, n_src, rng):
    """Random receivers/dipoles anywhere (interior and skeleton nodes)."""
    n = mesh.n_nodes - 1
    rec = rng.choice(n, size=n_rec, replace=False)
    P = sp.csc_matrix((np.ones(n_rec), (rec, np.arange(n_rec))), shape=(n, n_rec))
    a = rng.choice(n - 1, size=n_src, replace=False)
    rows = np.concatenate([a, a + 1])
    cols = np.tile(np.arange(n_src), 2)
    vals = np.concatenate([np.ones(n_src), -np.ones(n_src)])
    Q = sp.csc_matrix((vals, (rows, cols)), shape=(n, n_src))
    return Survey(P=P, Q=Q)


def top_random_survey(mesh, n_rec, n_src, rng):
    """Random receivers and x-dipoles on the top node plane (models.py:54-83 layout, random positions)."""
    n = mesh.n_nodes - 1
    kt = mesh.n3
    top = mesh.node_index(*np.meshgrid(np.arange(mesh.n1 + 1), np.arange(mesh.n2 + 1), indexing="ij"), kt)
    top = np.sort(top.ravel()) - 1
    rec = np.sort(rng.choice(top, size=n_rec, replace=False))
    P = sp.csc_matrix((np.ones(n_rec), (rec, np.arange(n_rec))), shape=(n, n_rec))
    i = rng.choice(mesh.n1, size=n_src, replace=False)
    j = rng.integers(0, mesh.n2 + 1, size=n_src)
    a = mesh.node_index(i, j, kt) - 1
    rows = np.concatenate([a, a + 1])
    cols = np.tile(np.arange(n_src), 2)
    vals = np.concatenate([np.ones(n_src), -np.ones(n_src)])
    return Survey(P=P, Q=sp.csc_matrix((vals, (rows, cols)), shape=(n, n_src)))


def pattern_digest(M):
    """sha256 of a CSR/CSC matrix's int32 index arrays (bit-exact pattern check)."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(M.indptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(M.indices, dtype=np.int64).tobytes())
    return np.frombuffer(h.digest(), dtype=np.uint8).copy()


def smooth_field(mesh, rng, sigma_cells, std):
    g = rng.standard_normal((mesh.n3, mesh.n2, mesh.n1))
    g = ndi.gaussian_filter(g, sigma_cells, mode="reflect")
    g = std * (g - g.mean()) / g.std()
    return g.ravel()


CASES = {
    # name: (cells, h, blocks, model kind, survey kind, yk)
    "c444_b222": ((4, 4, 4), (1.0, 1.0, 1.0), (2, 2, 2), ("normal", 0.3), ("random", 6, 3), True),
    "c664_b332": ((6, 6, 4), (1.0, 1.0, 1.0), (3, 3, 2), ("normal", 0.5), ("random", 8, 2), True),
    "c888_b444_h": ((8, 8, 8), (0.5, 1.0, 2.0), (4, 4, 4), ("uniform", 2.0), ("random", 10, 4), True),
    "c16_b844": ((16, 8, 8), (1.0, 1.0, 1.0), (8, 4, 4), ("smooth", 2.0, 1.0), ("random", 12, 3), True),
    "c16_b8": ((16, 16, 16), (1.0, 1.0, 1.0), (8, 8, 8), ("smooth", 2.0, 1.0), ("top", (2, 2), (4, 4)), False),
    "c32_b8": ((32, 32, 32), (1.0, 1.0, 1.0), (8, 8, 8), ("smooth", 3.0, 1.5), ("top", (2, 2), (8, 8)), False),
    # round 2: 8^3 blocks with receivers and dipoles inside block interiors
    "c32_b8_int": ((32, 32, 16), (1.0, 1.0, 1.0), (8, 8, 8), ("smooth", 3.0, 1.5), ("random", 40, 6), False),
    # blocks beyond the register-tile band: 16x16x4 (n_I 675, half band 225; Y_k as a digest)
    "c32_b16x4": ((32, 32, 8), (1.0, 1.0, 1.0), (16, 16, 4), ("smooth", 3.0, 1.0), ("random", 24, 4), "digest"),
    # 16^3 blocks: n_I = 3375 > 2000, the reference factors them with SuperLU (basis.py:276-278)
    "c32_b16": ((32, 32, 32), (1.0, 1.0, 1.0), (16, 16, 16), ("smooth", 4.0, 1.5), ("random", 30, 5), False),
    # the paper's Table-3 geometry: 64x64x32 cells, 16^3 blocks, top survey
    "c64_b16_t3": ((64, 64, 32), (1 / 64, 1 / 64, 1 / 64), (16, 16, 16), ("smooth", 4.0, 1.0), ("toprandom", 64, 6),
                   "xonly"),
}
# edge cases: blocks one cell thick along z (empty interiors, S = hats only)
# and a single block along x (nb1 = 1)
CASES["c884_b441"] = ((8, 8, 4), (1.0, 1.0, 1.0), (4, 4, 1), ("normal", 0.5), ("random", 8, 3), True)
CASES["c1688_b1644"] = ((16, 8, 8), (1.0, 1.0, 1.0), (16, 4, 4), ("smooth", 2.0, 1.0), ("random", 10, 3), True)
PERTURB = {"c64_b16_t3": 1.0}
# fixtures whose large arrays are stored as projections / digests
COMPACT = {"c32_b16x4", "c32_b16", "c64_b16_t3"}


def make_case(name, spec, seed=20240615):
    cells, h, blocks, mkind, skind, do_yk = spec
    rng = np.random.default_rng(seed)
    mesh = create_mesh(*cells, *h)
    part = create_partition(mesh, *blocks)
    if mkind[0] == "normal":
        m = mkind[1] * rng.normal(size=mesh.n_cells)
    elif mkind[0] == "uniform":
        m = rng.uniform(-mkind[1], mkind[1], size=mesh.n_cells)
    else:
        m = smooth_field(mesh, rng, mkind[1], mkind[2])
    if skind[0] == "random":
        survey = random_survey(mesh, skind[1], skind[2], rng)
    elif skind[0] == "toprandom":
        survey = top_random_survey(mesh, skind[1], skind[2], rng)
    else:
        survey = build_survey(mesh, n_src=skind[1], n_rec=skind[2])
    builder = BasisBuilder(part, BasisSpec(families=("lagrange",)))
    # observed data: reduced forward at a perturbed model.  The Table-3 case
    # uses a larger perturbation: with 0.2 its residual is 1.6% of D, which
    # amplifies the forward rounding into the gradient 64x (two valid
    # reference evaluation orders, dense vs SuperLU block factors, then differ
    # by 8e-11 on g)
    m_true = m + PERTURB.get(name, 0.2) * rng.normal(size=mesh.n_cells)
    op_t = assemble_operator(mesh, m_true)
    d_obs, _ = forward_reduced(op_t, survey, builder.assemble(op_t))

    op = assemble_operator(mesh, m)
    basis = builder.assemble(op)
    D, state = forward_reduced(op, survey, basis)
    phi, resid = misfit_ssd(D, d_obs)
    J = sensitivity_adaptive(state, survey)
    g = J.rapply(resid)
    dm = rng.normal(size=mesh.n_cells)
    Jv = J.apply(dm)
    W = rng.normal(size=(survey.n_receivers, survey.n_sources))
    JtW = J.rapply(W)
    out = dict(
        cells=np.array(cells), h=np.array(h), blocks=np.array(blocks), m=m,
        P_data=survey.P.data, P_indices=survey.P.indices, P_indptr=survey.P.indptr,
        P_shape=np.array(survey.P.shape),
        Q_data=survey.Q.data, Q_indices=survey.Q.indices, Q_indptr=survey.Q.indptr,
        Q_shape=np.array(survey.Q.shape),
        d_obs=d_obs, dm=dm, W=W,
        w=op.edge_weights,
        S_data=basis.S.data, S_indices=basis.S.indices, S_indptr=basis.S.indptr,
        T=state.T, D=D, phi=np.array(phi), resid=resid, g=g, Jv=Jv, JtW=JtW,
        US=basis.S @ state.T, shift=np.array(state.shift),
    )
    if op.n < 10000:
        out.update(A_data=op.A.data, A_indices=op.A.indices, A_indptr=op.A.indptr)
    if basis.k <= 200:
        out["A_k"] = np.asarray(state.A_k)
    if name in COMPACT:
        prj = np.random.default_rng(7)
        rn, rk = prj.standard_normal(basis.n), prj.standard_normal(basis.k)
        for key in ("S_data", "S_indices", "S_indptr", "US", "w"):
            out.pop(key)
        out.update(S_digest=pattern_digest(basis.S), S_nnz=np.array(basis.S.nnz), S_rn=basis.S.T @ rn,
                   S_rk=basis.S @ rk, S_norm=np.array(np.linalg.norm(basis.S.data)),
                   US_rs=(basis.S @ state.T).T @ rn, w_norm=np.array(np.linalg.norm(op.edge_weights)),
                   w_sum=np.array(op.edge_weights.sum()))
    if do_yk in ("digest", "xonly"):
        prj = np.random.default_rng(11)
        v = rng.normal(size=basis.k)
        wv = rng.normal(size=basis.n)
        rm = prj.standard_normal(mesh.n_cells)
        out.update(v=v, wv=wv, rm=rm)
        X = apply_Xk(basis, wv, m)
        xk = prj.standard_normal(basis.k)
        out.update(X_digest=pattern_digest(X), X_nnz=np.array(X.nnz), X_rm=X @ rm, X_rk=xk,
                   X_rt=X.T @ xk, X_norm=np.array(np.linalg.norm(X.data)))
        if do_yk == "digest":
            Y = apply_Yk(basis, v, m)
            rq = prj.standard_normal(basis.n)
            out.update(Y_rq=rq, Y_digest=pattern_digest(Y), Y_nnz=np.array(Y.nnz), Y_rm=Y @ rm, Y_rt=Y.T @ rq,
                       Y_norm=np.array(np.linalg.norm(Y.data)))
    elif do_yk:
        v = rng.normal(size=basis.k)
        wv = rng.normal(size=basis.n)
        Y = apply_Yk(basis, v, m)
        X = apply_Xk(basis, wv, m)
        out.update(v=v, wv=wv, Y_data=Y.data, Y_indices=Y.indices, Y_indptr=Y.indptr,
                   X_data=X.data, X_indices=X.indices, X_indptr=X.indptr)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "k", basis.k, "nnzS", basis.S.nnz, "phi", phi)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        make_case(nm, CASES[nm])
