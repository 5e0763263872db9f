"""2D path (BASELINE configs 1-2) on the B200 against the 2D oracle
(oracle/msfv_oracle2d.py).  Tolerance: 1e-10 relative (north_star) on T (u_c),
S T (P u_c), D, misfit, gradient, J v and J^T w."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import rel

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _oracle(mesh, part, survey):
    from oracle import msfv_oracle2d as o
    om = o.Mesh2D(mesh.n1, mesh.n2, mesh.h1, mesh.h2)
    return o, o.AdaptiveProblem(o.make_partition(om, part.b1, part.b2), o.Survey(survey.P, survey.Q))


def _compare(mesh, part, survey, m, d_obs, rng, n_products=1):
    import paper_1707_07598_b200 as gp
    prob = gp.AdaptiveReducedProblem2D(part, survey)
    D, st = prob.simulate(m)
    phi, r = gp.misfit_ssd(D, d_obs)
    J = prob.jacobian(st)
    g = J.rapply(r)
    o, oprob = _oracle(mesh, part, survey)
    D0, st0 = oprob.simulate(m)
    phi0, r0 = o.misfit(D0, d_obs)
    J0 = oprob.jacobian(st0)
    g0 = J0.rapply(r0)
    assert rel(st.T, st0.T) <= TOL
    U = st.U.cpu().numpy()
    assert rel(U, (st0.basis.S @ st0.T)) <= TOL
    assert rel(D, D0) <= TOL
    assert abs(phi - phi0) <= TOL * abs(phi0)
    assert rel(g, g0) <= TOL
    for _ in range(n_products):
        v = rng.standard_normal(m.size)
        w = rng.standard_normal(D.shape)
        assert rel(J.apply(v), J0.apply(v)) <= TOL
        assert rel(J.rapply(w), J0.rapply(w)) <= TOL


def test_small_anisotropic_nonsquare_blocks():
    import paper_1707_07598_b200 as gp
    rng = np.random.default_rng(11)
    mesh = gp.create_mesh_2d(24, 18, 1.0 / 24, 1.5 / 18)
    part = gp.create_partition_2d(mesh, 4, 3)
    n = mesh.n_nodes - 1
    P = sp.csc_matrix((np.ones(9), (rng.choice(n, 9, replace=False), np.arange(9))), shape=(n, 9))
    a = rng.choice(n - 1, 3, replace=False)
    Q = sp.csc_matrix((np.r_[np.ones(3), -np.ones(3)], (np.r_[a, a + 1], np.r_[0:3, 0:3])), shape=(n, 3))
    survey = gp.Survey(P=P, Q=Q)
    m = 0.9 * rng.standard_normal(mesh.n_cells)
    _compare(mesh, part, survey, m, 1e-3 * rng.standard_normal((9, 3)), rng, n_products=2)


@pytest.mark.parametrize("cfg", [1, 2])
def test_baseline_config(cfg):
    import paper_1707_07598_b200 as gp
    mesh, part, survey, m, d_obs = gp.config_problem_2d(cfg)
    _compare(mesh, part, survey, m, d_obs, np.random.default_rng(1), n_products=2 if cfg == 2 else 1)


def test_model_errors_and_determinism():
    import paper_1707_07598_b200 as gp
    mesh, part, survey, m, d_obs = gp.config_problem_2d(1)
    prob = gp.AdaptiveReducedProblem2D(part, survey)
    bad = m.copy()
    bad[5] = np.nan
    with pytest.raises(gp.InvalidModelError):
        prob.simulate(bad)
    with pytest.raises(ValueError):
        prob.simulate(m[:-1])
    D1, st1 = prob.simulate(m + 0.3)
    D2, st2 = prob.simulate(m + 0.3)
    assert np.array_equal(D1, D2)
    r = D1 - d_obs
    assert np.array_equal(prob.jacobian(st1).rapply(r), prob.jacobian(st2).rapply(r))
