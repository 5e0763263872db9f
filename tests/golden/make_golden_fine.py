"""Golden vectors for the fine-mesh path from the UNMODIFIED
reference: forward_full with SuperLU ("direct") and with block CG, the full
sensitivity products, and block_cg on a random right-hand side.

    python tests/golden/make_golden_fine.py

Imports msinv from /root/reference/pkg/src (read-only); writes fine_*.npz here.
"""
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import numpy as np                                    # noqa: E402

from msinv.forward import forward_full, sensitivity_full  # noqa: E402
from msinv.mesh import create_mesh                    # noqa: E402
from msinv.operators import assemble_operator         # noqa: E402
from msinv.solvers import block_cg                    # noqa: E402

sys.path.insert(0, os.path.dirname(__file__))
from make_golden import random_survey, smooth_field  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (cells, h, model (sigma_cells, std), receivers, sources)
    "fine_c16": ((16, 16, 16), (1 / 16, 1 / 16, 1 / 16), (2.0, 1.0), 20, 4, 1e-9, 400),
    "fine_c1288": ((12, 8, 8), (1.0, 0.5, 2.0), (1.5, 0.5), 12, 3, 1e-7, 150),
}


def make(name, spec, seed=20240615):
    cells, h, (sc, std), nrec, nsrc, btol, bmax = spec
    rng = np.random.default_rng(seed)
    mesh = create_mesh(*cells, *h)
    m = smooth_field(mesh, rng, sc, std)
    survey = random_survey(mesh, nrec, nsrc, rng)
    op = assemble_operator(mesh, m)
    D, st = forward_full(op, survey, solver="direct")
    J = sensitivity_full(st, survey)
    dm = rng.normal(size=mesh.n_cells)
    W = rng.normal(size=(survey.n_receivers, survey.n_sources))
    out = dict(cells=np.array(cells), h=np.array(h), m=m,
               P_data=survey.P.data, P_indices=survey.P.indices, P_indptr=survey.P.indptr,
               P_shape=np.array(survey.P.shape),
               Q_data=survey.Q.data, Q_indices=survey.Q.indices, Q_indptr=survey.Q.indptr,
               Q_shape=np.array(survey.Q.shape),
               D=D, U=st.U, dm=dm, W=W, Jv=J.apply(dm), JtW=J.rapply(W))
    # block CG mode (forward.py:88-93) at the reference defaults and a tight run
    Dc, stc = forward_full(op, survey, solver="blockcg", cg_tol=1e-6, cg_maxit=100)
    out.update(D_cg=Dc, cg_iterations=np.array(stc.solver_info["iterations"]),
               cg_relres=np.array(stc.solver_info["relres"]), cg_converged=np.array(stc.solver_info["converged"]))
    Jc = sensitivity_full(stc, survey)
    out.update(Jv_cg=Jc.apply(dm), JtW_cg=Jc.rapply(W))
    # the reference's own drift on the same non-converged problem with the
    # source columns reversed (only the summation order of the block products
    # changes): the scale any other implementation's iterates differ by
    from msinv.forward import Survey
    rev = np.arange(survey.n_sources)[::-1]
    srv_r = Survey(P=survey.P, Q=survey.Q[:, rev])
    Dr, str_ = forward_full(op, srv_r, solver="blockcg", cg_tol=1e-6, cg_maxit=100)
    Jr = sensitivity_full(str_, srv_r)
    out.update(D_cg_rev=Dr[:, rev], Jv_cg_rev=Jr.apply(dm)[:, rev], JtW_cg_rev=Jr.rapply(W[:, rev]))
    B = rng.normal(size=(op.A.shape[0], 5))
    B[:, 2] = 0.0                                        # a zero column counts as converged
    res = block_cg(op.A, B, tol=btol, maxit=bmax)
    rb = np.arange(B.shape[1])[::-1]
    res_r = block_cg(op.A, B[:, rb], tol=btol, maxit=bmax)
    out.update(X_bcg_rev=res_r.X[:, rb], bcg_history_rev=np.array(res_r.history))
    out.update(B=B, bcg_tol=np.array(btol), bcg_maxit=np.array(bmax), X_bcg=res.X, bcg_iterations=np.array(res.iterations), bcg_relres=np.array(res.relres),
               bcg_history=np.array(res.history))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "n", op.A.shape[0], "cg its", stc.solver_info["iterations"], "bcg its", res.iterations)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(CASES):
        make(nm, CASES[nm])
