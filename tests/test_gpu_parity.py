"""GPU parity: the CUDA path (through the C-ABI) against golden vectors from the
unmodified reference and against the CPU oracle.

Tolerances (north_star): relative error <= 1e-10 on S, T (u_c), S T (P u_c),
D, misfit and gradient (and J v / J^T w); integer patterns bit-exact.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN_CASES, LARGE_CASES, basis_errors, load_golden, rel, table3_errors

pytestmark = pytest.mark.gpu

TOL = 1e-10


def build_gpu(g):
    import paper_1707_07598_b200 as gp
    cells = [int(x) for x in g["cells"]]
    h = [float(x) for x in g["h"]]
    b = [int(x) for x in g["blocks"]]
    mesh = gp.create_mesh(*cells, *h)
    part = gp.create_partition(mesh, *b)
    P = sp.csc_matrix((g["P_data"], g["P_indices"], g["P_indptr"]), shape=tuple(g["P_shape"]))
    Q = sp.csc_matrix((g["Q_data"], g["Q_indices"], g["Q_indptr"]), shape=tuple(g["Q_shape"]))
    survey = gp.Survey(P=P, Q=Q)
    builder = gp.BasisBuilder(part, gp.BasisSpec(families=("lagrange",)))
    return gp, mesh, part, survey, builder


@pytest.mark.parametrize("name", GOLDEN_CASES + LARGE_CASES)
def test_forward_gradient_matches_reference(name):
    """Every golden case, including blocks beyond the register-tile band
    (16x16x4, 16^3 with n_I = 3375 > 2000 where the reference uses SuperLU,
    and the paper's Table-3 geometry 64x64x32 / 16^3)."""
    g = load_golden(name)
    gp, mesh, part, survey, builder = build_gpu(g)
    op = gp.assemble_operator(mesh, g["m"])
    basis = builder.assemble(op)
    D, state = gp.forward_reduced(op, survey, basis)
    errs = basis_errors(g, basis.S, state.T, op.edge_weights)
    errs["T"] = rel(state.T, g["T"])
    errs["D"] = rel(D, g["D"])
    phi, resid = gp.misfit_ssd(D, g["d_obs"])
    errs["phi"] = abs(phi - float(g["phi"])) / abs(float(g["phi"]))
    J = gp.sensitivity_adaptive(state, survey)
    errs["g"] = rel(J.rapply(resid), g["g"])
    errs["Jv"] = rel(J.apply(g["dm"]), g["Jv"])
    errs["JtW"] = rel(J.rapply(g["W"]), g["JtW"])
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, f"{name}: {errs}"


def test_skeleton_values_bit_exact():
    g = load_golden("c16_b8")
    gp, mesh, part, survey, builder = build_gpu(g)
    op = gp.assemble_operator(mesh, g["m"])
    S = builder.assemble(op).S
    # entries on skeleton rows are the model-independent hats: bit-exact
    skel = part.skeleton[part.skeleton != 0] - 1
    mask = np.isin(S.indices, skel)
    assert np.array_equal(S.data[mask], g["S_data"][mask])


def test_edge_weights_last_ulp():
    # w = C exp(m) in the reference's summation order; exp() itself is not
    # correctly rounded on either side, so allow a few ulps per entry.
    g = load_golden("c32_b8")
    gp, mesh, part, survey, builder = build_gpu(g)
    op = gp.assemble_operator(mesh, g["m"])
    builder.assemble(op)
    w = op.edge_weights
    assert np.max(np.abs(w - g["w"]) / np.abs(g["w"])) <= 1e-15


@pytest.mark.parametrize("name", [n for n in GOLDEN_CASES + LARGE_CASES
                                  if n not in ("c16_b8", "c32_b8", "c32_b8_int", "c32_b16")])
def test_table3_operators_match_reference(name):
    """apply_Yk / apply_Xk (basis.py:684-800): CSR pattern bit-exact, values <= 1e-10
    (full arrays, or digests + projections for the large fixtures)."""
    g = load_golden(name)
    gp, mesh, part, survey, builder = build_gpu(g)
    op = gp.assemble_operator(mesh, g["m"])
    basis = builder.assemble(op)
    has_y = "Y_data" in g or "Y_digest" in g
    Y = gp.apply_Yk(basis, g["v"], g["m"]) if has_y else None
    X = gp.apply_Xk(basis, g["wv"], g["m"])
    errs = table3_errors(g, Y, X)
    assert max(errs.values()) <= TOL, errs
    # stale-model contract (basis.py:333-337)
    with pytest.raises(gp.StaleBasisError):
        gp.apply_Yk(basis, g["v"], g["m"] + 1.0)


def test_table3_operators_match_oracle(rng):
    """apply_Yk / apply_Xk at 8^3-cell blocks (the BASELINE block size) against the oracle."""
    from oracle import msfv_oracle as oracle
    g = load_golden("c16_b8")
    gp, mesh, part, survey, builder = build_gpu(g)
    m = g["m"]
    op = gp.assemble_operator(mesh, m)
    basis = builder.assemble(op)
    omesh = oracle.Mesh(*[int(x) for x in g["cells"]], *[float(x) for x in g["h"]])
    obasis = oracle.build_basis(oracle.assemble(omesh, m), oracle.make_partition(omesh, *[int(x) for x in g["blocks"]]))
    v = rng.standard_normal(basis.k)
    w = rng.standard_normal(basis.n)
    for got, ref in ((gp.apply_Yk(basis, v, m), oracle.apply_Yk(obasis, v, m)),
                     (gp.apply_Xk(basis, w, m), oracle.apply_Xk(obasis, w, m))):
        assert np.array_equal(got.indptr, ref.indptr)
        assert np.array_equal(got.indices, ref.indices)
        assert rel(got.data, ref.data) <= TOL


@pytest.mark.parametrize("name", ["c16_b8", "c32_b8"])
def test_coarse_nested_dissection_matches_reference(name, monkeypatch):
    """The z-plane nested-dissection coarse solver (default for k >= 1000)
    forced on small golden cases: same T, D, misfit, gradient, J v, J^T w."""
    import paper_1707_07598_b200.engine as E
    monkeypatch.setenv("MSFV_COARSE_ND", "1")
    saved = dict(E._ENGINES)
    E._ENGINES.clear()
    try:
        g = load_golden(name)
        gp, mesh, part, survey, builder = build_gpu(g)
        op = gp.assemble_operator(mesh, g["m"])
        basis = builder.assemble(op)
        D, state = gp.forward_reduced(op, survey, basis)
        J = gp.sensitivity_adaptive(state, survey)
        errs = {"T": rel(state.T, g["T"]), "D": rel(D, g["D"]), "g": rel(J.rapply(g["resid"]), g["g"]),
                "Jv": rel(J.apply(g["dm"]), g["Jv"]), "JtW": rel(J.rapply(g["W"]), g["JtW"]),
                "A_k": rel(state.A_k, g["A_k"])}
        bad = {k: v for k, v in errs.items() if not v <= TOL}
        assert not bad, f"{name}: {errs}"
    finally:
        E._ENGINES.clear()
        E._ENGINES.update(saved)
