"""Pin the CPU oracle against golden vectors from the unmodified reference."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN_CASES, LARGE_CASES, basis_errors, load_golden, rel, table3_errors
from oracle import msfv_oracle as orc


def golden_problem(g):
    cells, h, b = g["cells"], g["h"], g["blocks"]
    mesh = orc.Mesh(*[int(x) for x in cells], *[float(x) for x in h])
    part = orc.make_partition(mesh, *[int(x) for x in b])
    P = sp.csc_matrix((g["P_data"], g["P_indices"], g["P_indptr"]), shape=tuple(g["P_shape"]))
    Q = sp.csc_matrix((g["Q_data"], g["Q_indices"], g["Q_indptr"]), shape=tuple(g["Q_shape"]))
    return mesh, part, orc.Survey(P, Q)


@pytest.mark.parametrize("name", GOLDEN_CASES + LARGE_CASES)
def test_oracle_matches_reference(name):
    g = load_golden(name)
    mesh, part, survey = golden_problem(g)
    prob = orc.AdaptiveProblem(part, survey)
    D, st = prob.simulate(g["m"])
    op, basis = st.op, st.basis
    if "A_data" in g:
        assert np.array_equal(op.A.indptr, g["A_indptr"])
        assert np.array_equal(op.A.indices, g["A_indices"])
        assert rel(op.A.data, g["A_data"]) <= 1e-14
    # integer pattern of S is bit-exact (asserted inside), values tight
    errs = basis_errors(g, basis.S, st.T, op.w)
    assert errs.pop("w") <= 1e-14
    assert max(errs.values()) <= 1e-12, errs
    assert rel(st.T, g["T"]) <= 1e-12
    assert rel(D, g["D"]) <= 1e-12
    phi, resid = orc.misfit(D, g["d_obs"])
    assert abs(phi - float(g["phi"])) <= 1e-11 * abs(float(g["phi"]))
    J = prob.jacobian(st)
    assert rel(J.rapply(resid), g["g"]) <= 1e-11
    assert rel(J.apply(g["dm"]), g["Jv"]) <= 1e-11
    assert rel(J.rapply(g["W"]), g["JtW"]) <= 1e-11
    if "v" in g:
        Y = orc.apply_Yk(basis, g["v"], g["m"]) if ("Y_data" in g or "Y_digest" in g) else None
        X = orc.apply_Xk(basis, g["wv"], g["m"])
        errs = table3_errors(g, Y, X)
        assert max(errs.values()) <= 1e-12, errs
