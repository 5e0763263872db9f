"""Golden vectors for the enriched basis families from the
UNMODIFIED reference package.

    python tests/golden/make_golden_enriched.py

Imports ``msinv`` from /root/reference/pkg/src (read-only, never copied) and
writes ``enr_*.npz`` next to this script: boundary-condition data of the
``source`` / ``skeleton`` / ``local_pca`` families (basis.py:119-245), the
assembled basis, the reduced forward map and the adaptive sensitivity
products.  The fixtures pin tests/test_enriched_host.py (host logic on a numpy
engine) and tests/test_gpu_enriched.py (the CUDA path).
"""

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.dont_write_bytecode = True

import numpy as np                                    # noqa: E402

from msinv.basis import BasisBuilder, BasisSpec       # noqa: E402
from msinv.forward import forward_reduced, sensitivity_adaptive  # noqa: E402
from msinv.inversion import misfit_ssd                # noqa: E402
from msinv.mesh import create_mesh, create_partition  # noqa: E402
from msinv.models import build_survey                 # noqa: E402
from msinv.operators import assemble_operator         # noqa: E402

from make_golden import random_survey, smooth_field   # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (cells, h, blocks, families, pca (rank, total), survey, model std)
    "enr_c1212_all": ((12, 12, 6), (1.0, 1.0, 1.0), (6, 6, 3), ("lagrange", "source", "skeleton", "local_pca"),
                      (2, 0), ("random", 10, 4), 0.8),
    "enr_c1688_tot": ((16, 8, 8), (1.0, 0.5, 2.0), (8, 4, 4), ("lagrange", "skeleton", "local_pca"),
                      (2, 9), ("random", 12, 3), 1.0),
    "enr_c24_b8": ((24, 24, 8), (1.0, 1.0, 1.0), (8, 8, 8), ("lagrange", "skeleton", "local_pca"),
                   (3, 0), ("top", (2, 2), (6, 6)), 1.0),
    "enr_c1212_src": ((12, 12, 6), (1.0, 1.0, 1.0), (6, 6, 3), ("lagrange", "source"),
                      (0, 0), ("random", 10, 5), 0.8),
    "enr_c888_nolag": ((8, 8, 8), (1.0, 1.0, 1.0), (4, 4, 4), ("source", "skeleton", "local_pca"),
                       (1, 0), ("random", 9, 3), 0.5),
}


def make_case(name, spec, seed=20241021):
    cells, h, blocks, families, (rank, total), skind, std = spec
    rng = np.random.default_rng(seed)
    mesh = create_mesh(*cells, *h)
    part = create_partition(mesh, *blocks)
    m_ref = 0.3 * smooth_field(mesh, rng, 2.0, 1.0) + np.log(0.05)
    m = m_ref + smooth_field(mesh, rng, 1.5, std)
    if skind[0] == "random":
        survey = random_survey(mesh, skind[1], skind[2], rng)
    else:
        survey = build_survey(mesh, n_src=skind[1], n_rec=skind[2])
    bspec = BasisSpec(families=families, pca_rank=rank, pca_total=total)
    builder = BasisBuilder(part, bspec, Q=survey.Q, m_ref=m_ref)
    m_true = m + 0.3 * rng.normal(size=mesh.n_cells)
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
    wv = rng.normal(size=basis.n)
    out = dict(
        cells=np.array(cells), h=np.array(h), blocks=np.array(blocks),
        families=np.array(families), pca_rank=np.array(rank), pca_total=np.array(total),
        m=m, m_ref=m_ref,
        P_data=survey.P.data, P_indices=survey.P.indices, P_indptr=survey.P.indptr, P_shape=np.array(survey.P.shape),
        Q_data=survey.Q.data, Q_indices=survey.Q.indices, Q_indptr=survey.Q.indptr, Q_shape=np.array(survey.Q.shape),
        d_obs=d_obs, dm=dm, W=W, wv=wv,
        col_family=np.asarray(basis.families), labels=np.array([repr(lab) for lab in basis.labels]),
        S_data=basis.S.data, S_indices=basis.S.indices, S_indptr=basis.S.indptr,
        EP_data=basis.edge_profiles.data, EP_indices=basis.edge_profiles.indices,
        EP_indptr=basis.edge_profiles.indptr,
        A_k=np.asarray(state.A_k), T=state.T, D=D, phi=np.array(phi), resid=resid, g=g, Jv=Jv, JtW=JtW,
        shift=np.array(state.shift), isolve=basis.interior_solve(wv), gedge=basis.grad_edge(state.T[:, 0]),
    )
    for bc in builder.bc_sets:
        V = bc.values.tocsc()
        F = bc.forcing.tocsc()
        out[f"bc_{bc.family}_V_data"] = V.data
        out[f"bc_{bc.family}_V_indices"] = V.indices
        out[f"bc_{bc.family}_V_indptr"] = V.indptr
        out[f"bc_{bc.family}_F_data"] = F.data
        out[f"bc_{bc.family}_F_indices"] = F.indices
        out[f"bc_{bc.family}_F_indptr"] = F.indptr
        if bc.block_restrict is not None:
            out[f"bc_{bc.family}_restrict"] = np.asarray(bc.block_restrict)
        if bc.dropped:
            out[f"bc_{bc.family}_dropped"] = np.asarray(bc.dropped)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    fam, cnt = np.unique(np.asarray(basis.families), return_counts=True)
    print(name, "k", basis.k, dict(zip(fam, cnt)), "nnzS", basis.S.nnz, "phi", phi, "shift", state.shift)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        make_case(nm, CASES[nm])
