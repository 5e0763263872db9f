"""Reduced-dimension boundary conditions on the GPU against
the CPU oracle (oracle/msfv_reduced.py; parity unpinned by the reference,
which has no such code): S (values 1e-10, CSC pattern identical
to the hat basis), partition of unity, sigma == 1 reproducing the hat basis,
the reduced forward map T, D at 1e-10, and the sensitivities through the
reduced boundary problems (adjoint identity, central differences of the
oracle's forward map, Gauss-Newton trace)."""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu
TOL = 1e-10
GEOMS = [((8, 8, 8), (4, 4, 4), (1.0, 1.0, 1.0)), ((12, 8, 8), (4, 4, 2), (0.5, 1.0, 2.0)),
         ((16, 16, 16), (8, 8, 8), (1 / 16, 1 / 16, 1 / 16)), ((32, 32, 32), (16, 16, 16), (1.0, 1.0, 1.0))]


def _survey(mesh, rng):
    import scipy.sparse as sp
    import paper_1707_07598_b200 as gp
    n = mesh.n_nodes - 1
    rec = rng.choice(n, size=10, replace=False)
    P = sp.csc_matrix((np.ones(10), (rec, np.arange(10))), shape=(n, 10))
    a = rng.choice(n - 1, size=3, replace=False)
    Q = sp.csc_matrix((np.r_[np.ones(3), -np.ones(3)], (np.r_[a, a + 1], np.r_[0:3, 0:3])), shape=(n, 3))
    return gp.Survey(P=P, Q=Q)


@pytest.mark.parametrize("cells,b,h", GEOMS)
def test_reduced_basis_and_forward_match_oracle(cells, b, h, rng):
    import paper_1707_07598_b200 as gp
    from oracle import msfv_oracle as orc
    from oracle import msfv_reduced as red
    mesh = gp.create_mesh(*cells, *h)
    part = gp.create_partition(mesh, *b)
    survey = _survey(mesh, rng)
    m = 1.2 * rng.normal(size=mesh.n_cells)
    builder = gp.BasisBuilder(part, gp.BasisSpec(boundary="reduced"))
    op = gp.assemble_operator(mesh, m)
    basis = builder.assemble(op)
    D, st = gp.forward_reduced(op, survey, basis)

    om = orc.Mesh(*cells, *h)
    opart = orc.make_partition(om, *b)
    oop = orc.assemble(om, m)
    D0, st0 = red.forward_reduced(oop, orc.Survey(survey.P, survey.Q), opart)
    S, S0 = basis.S, st0.basis.S
    assert np.array_equal(S.indptr, S0.indptr) and np.array_equal(S.indices, S0.indices)
    rows = np.asarray(S.sum(axis=1)).ravel()
    errs = {"S": rel(S.data, S0.data), "T": rel(st.T, st0.T), "D": rel(D, D0),
            "unity": float(np.max(np.abs(rows - 1.0)))}
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, errs


@pytest.mark.parametrize("cells,b,h", GEOMS[:3])
def test_reduced_sensitivity(cells, b, h, rng):
    """J v and J^T W through the reduced boundary problems (reduced_sens.py):
    the adjoint identity ties the two (independent: forward- and reverse-mode
    skeleton derivatives, different kernel chains) to 1e-10; J v and the
    misfit gradient agree with central differences of the ORACLE's reduced
    forward map (oracle/msfv_reduced.py) to 1e-6."""
    import paper_1707_07598_b200 as gp
    from oracle import msfv_oracle as orc
    from oracle import msfv_reduced as red
    mesh = gp.create_mesh(*cells, *h)
    part = gp.create_partition(mesh, *b)
    survey = _survey(mesh, rng)
    m = 0.8 * rng.normal(size=mesh.n_cells)
    builder = gp.BasisBuilder(part, gp.BasisSpec(boundary="reduced"))
    op = gp.assemble_operator(mesh, m)
    D, st = gp.forward_reduced(op, survey, builder.assemble(op))
    J = gp.sensitivity_adaptive(st, survey)
    v = rng.normal(size=mesh.n_cells)
    W = rng.normal(size=D.shape)
    jv, jtw = J.apply(v), J.rapply(W)
    lhs, rhs = float(np.sum(jv * W)), float(np.dot(v, jtw))
    assert abs(lhs - rhs) <= 1e-10 * abs(lhs), (lhs, rhs)

    om = orc.Mesh(*cells, *h)
    opart = orc.make_partition(om, *b)
    osurvey = orc.Survey(survey.P, survey.Q)
    fwd = lambda mm: red.forward_reduced(orc.assemble(om, mm), osurvey, opart)[0]   # noqa: E731
    eps = 1e-5
    Dp, Dm = fwd(m + eps * v), fwd(m - eps * v)
    fd = (Dp - Dm) / (2 * eps)
    assert rel(jv, fd) <= 1e-6, rel(jv, fd)
    d_obs = fwd(m + 0.3 * rng.normal(size=m.size))
    g = J.rapply(D - d_obs)
    dphi = 0.5 * (np.sum((Dp - d_obs) ** 2) - np.sum((Dm - d_obs) ** 2)) / (2 * eps)
    assert abs(np.dot(g, v) - dphi) <= 1e-6 * abs(dphi), (np.dot(g, v), dphi)


def test_reduced_gauss_newton_decreases_objective(rng):
    """The device Gauss-Newton loop (inversion.py:187-263) on a problem whose
    basis uses the reduced boundary conditions: monotone trace."""
    import paper_1707_07598_b200 as gp
    mesh = gp.create_mesh(8, 8, 8)
    part = gp.create_partition(mesh, 4, 4, 4)
    survey = _survey(mesh, rng)
    prob = gp.AdaptiveReducedProblem(gp.BasisBuilder(part, gp.BasisSpec(boundary="reduced")), survey)
    d_obs = prob.simulate(0.4 * rng.normal(size=mesh.n_cells))[0]
    obj = gp.DeviceObjective(mesh, 1e-3, np.zeros(mesh.n_cells))
    m, trace = gp.gauss_newton_dev(prob, np.zeros(mesh.n_cells), d_obs, obj, gp.GNSettings(max_gn=3, max_cg=5))
    tot = trace.totals()
    assert np.all(np.diff(tot) <= 1e-15 * abs(tot[0])) and tot[-1] < 0.5 * tot[0]


@pytest.mark.parametrize("cells,b,h", GEOMS[:3])
def test_unit_conductivity_reproduces_hat_basis(cells, b, h):
    import paper_1707_07598_b200 as gp
    mesh = gp.create_mesh(*cells, *h)
    part = gp.create_partition(mesh, *b)
    m = np.zeros(mesh.n_cells)
    Sr = gp.BasisBuilder(part, gp.BasisSpec(boundary="reduced")).assemble(gp.assemble_operator(mesh, m)).S
    Sh = gp.BasisBuilder(part).assemble(gp.assemble_operator(mesh, m)).S
    assert np.array_equal(Sr.indices, Sh.indices)
    assert np.max(np.abs(Sr.data - Sh.data)) <= 1e-12
