"""Pin the enriched-family oracle (oracle/msfv_enriched.py) against goldens of
the unmodified reference (tests/golden/make_golden_enriched.py)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import load_golden, rel
from oracle import msfv_enriched as oen
from oracle import msfv_oracle as orc

ENR_CASES = ["enr_c1212_all", "enr_c1688_tot", "enr_c24_b8", "enr_c1212_src", "enr_c888_nolag"]


def csc(g, key, shape):
    return sp.csc_matrix((g[key + "_data"], g[key + "_indices"], g[key + "_indptr"]), shape=shape)


@pytest.mark.parametrize("name", ENR_CASES)
def test_enriched_oracle_matches_reference(name):
    g = load_golden(name)
    mesh = orc.Mesh(*[int(x) for x in g["cells"]], *[float(x) for x in g["h"]])
    part = orc.make_partition(mesh, *[int(x) for x in g["blocks"]])
    n = mesh.n_nodes - 1
    survey = orc.Survey(csc(g, "P", tuple(g["P_shape"])), csc(g, "Q", tuple(g["Q_shape"])))
    names = tuple(str(f) for f in g["families"])
    fams = oen.families(part, names, Q=survey.Q, m_ref=g["m_ref"], rank=int(g["pca_rank"]),
                        total=int(g["pca_total"]))
    for f in fams:
        if f.name == "lagrange":
            continue
        V = csc(g, f"bc_{f.name}_V", (n, f.count))
        assert np.array_equal(f.values.indptr, V.indptr) and np.array_equal(f.values.indices, V.indices)
        assert rel(f.values.data, V.data) <= 1e-12 if V.nnz else True
        Fg = csc(g, f"bc_{f.name}_F", (n, f.count))
        assert (f.forcing - Fg).nnz == 0
        if f.restrict is not None:
            assert np.array_equal(f.restrict, g[f"bc_{f.name}_restrict"])
    op = orc.assemble(mesh, g["m"])
    basis = oen.build_basis(op, part, fams)
    assert list(basis.families) == [str(x) for x in g["col_family"]]
    assert [repr(x) for x in basis.labels] == [str(x) for x in g["labels"]]
    S_ref = csc(g, "S", (n, basis.k))
    assert np.array_equal(basis.S.indptr, S_ref.indptr) and np.array_equal(basis.S.indices, S_ref.indices)
    assert rel(basis.S.data, S_ref.data) <= 1e-12
    EP_ref = csc(g, "EP", basis.EP.shape)
    d = (basis.EP - EP_ref).tocsc()
    assert (np.linalg.norm(d.data) if d.nnz else 0.0) <= 1e-12 * np.linalg.norm(EP_ref.data)
    D, st = orc.forward_reduced(op, survey, basis)
    assert rel(st.A_k, g["A_k"]) <= 1e-12
    assert rel(D, g["D"]) <= 1e-11
    assert rel(g["A_k"] @ st.T, g["A_k"] @ g["T"]) <= 1e-10
    phi, resid = orc.misfit(D, g["d_obs"])
    assert abs(phi - float(g["phi"])) <= 1e-10 * float(g["phi"])
    J = orc.Sensitivity(st, survey)
    assert rel(J.rapply(resid), g["g"]) <= 1e-10
    assert rel(J.apply(g["dm"]), g["Jv"]) <= 1e-10
    assert rel(J.rapply(g["W"]), g["JtW"]) <= 1e-10
    assert rel(basis.interior_solve(g["wv"]), g["isolve"]) <= 1e-12
