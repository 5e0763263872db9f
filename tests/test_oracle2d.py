"""2D oracle (configs 1-2) validated by 2D ports of the reference's own test
oracles -- the reference is 3D only, so these properties are the
pin.  CPU only."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from oracle import msfv_oracle2d as o


def _case(n=(16, 12), b=(4, 3), seed=0, scale=0.8):
    mesh = o.Mesh2D(n[0], n[1], 1.0 / n[0], 1.5 / n[1])
    part = o.make_partition(mesh, *b)
    rng = np.random.default_rng(seed)
    m = scale * rng.normal(size=mesh.n_cells)
    return mesh, part, m, rng


def test_partition_sizes():
    # mesh.py:143-182 in 2D: interior (b-1)^2, boundary (b+1)^2 - (b-1)^2
    mesh = o.Mesh2D(16, 16)
    part = o.make_partition(mesh, 4, 4)
    assert all(I.size == 9 for I in part.interiors)
    assert all(B.size == 25 - 9 for B in part.boundaries)
    assert part.n_coarse == 25 and part.coarse_nodes.size == 25


def test_sigma_one_rows_are_five_point():
    # operators.py:77-109 with d = 2: C = V/2 per touching cell
    mesh = o.Mesh2D(6, 5, 0.5, 0.25)
    op = o.assemble(mesh, np.zeros(mesh.n_cells))
    r = mesh.node(3, 2) - 1
    row = op.A[r].toarray().ravel()
    V = mesh.volume
    assert row[r] == pytest.approx(2 * V / mesh.h1 ** 2 + 2 * V / mesh.h2 ** 2, rel=1e-14)
    assert row[mesh.node(2, 2) - 1] == pytest.approx(-V / mesh.h1 ** 2, rel=1e-14)
    assert row[mesh.node(3, 1) - 1] == pytest.approx(-V / mesh.h2 ** 2, rel=1e-14)
    assert np.count_nonzero(row) == 5


def test_local_solve_matches_dense_and_partition_of_unity():
    # test_basis.py:118-131 (local solve vs np.linalg.solve), test_acceptance.py:48-73 (unity)
    mesh, part, m, _ = _case()
    op = o.assemble(mesh, m)
    basis = o.build_basis(op, part)
    S = basis.S.toarray()
    cache = basis.cache
    for j in (0, 5, part.n_blocks - 1):
        I, B = cache.I[j], cache.B[j]
        A = op.A.toarray()
        x = np.linalg.solve(A[np.ix_(I, I)], -A[np.ix_(I, B)] @ cache.xb[j])
        assert np.allclose(S[np.ix_(I, cache.cols[j])], x, rtol=0, atol=1e-12)
    assert np.abs(S.sum(axis=1) - 1.0).max() <= 1e-10


def test_sigma_one_basis_is_bilinear():
    # test_acceptance.py:48-73: sigma = 1 reproduces the hats (bilinear here)
    mesh = o.Mesh2D(12, 12, 1 / 12, 1 / 12)
    part = o.make_partition(mesh, 4, 4)
    op = o.assemble(mesh, np.zeros(mesh.n_cells))
    S = o.build_basis(op, part).S.toarray()
    ids = np.arange(1, mesh.n_nodes)
    for c, cn in enumerate(part.coarse_nodes):
        assert np.abs(S[:, c] - o.hat(part, cn, ids)).max() <= 1e-10


def test_galerkin_identity_and_adjoint():
    # test_acceptance.py:252-268 (A_k = S^T A S), test_forward.py:228-258 (adjoint)
    mesh, part, m, rng = _case(seed=3)
    n = mesh.n_nodes - 1
    P = sp.csc_matrix((np.ones(7), (rng.choice(n, 7, replace=False), np.arange(7))), shape=(n, 7))
    a = rng.choice(n - 1, 3, replace=False)
    Q = sp.csc_matrix((np.r_[np.ones(3), -np.ones(3)], (np.r_[a, a + 1], np.r_[0:3, 0:3])), shape=(n, 3))
    prob = o.AdaptiveProblem(part, o.Survey(P, Q))
    D, st = prob.simulate(m)
    S = st.basis.S
    assert np.abs(st.A_k - (S.T @ st.op.A @ S).toarray()).max() <= 1e-12 * np.abs(st.A_k).max()
    J = prob.jacobian(st)
    v, W = rng.normal(size=m.size), rng.normal(size=D.shape)
    lhs, rhs = np.sum(W * J.apply(v)), np.sum(v * J.rapply(W))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_taylor_second_order():
    # test_basis.py:320-388 / test_forward.py:183-226: D(m + t v) - D(m) - t J v = O(t^2)
    mesh, part, m, rng = _case(seed=5, scale=0.5)
    n = mesh.n_nodes - 1
    P = sp.csc_matrix((np.ones(5), (rng.choice(n, 5, replace=False), np.arange(5))), shape=(n, 5))
    a = rng.choice(n - 1, 2, replace=False)
    Q = sp.csc_matrix((np.r_[1.0, 1, -1, -1], (np.r_[a, a + 1], np.r_[0, 1, 0, 1])), shape=(n, 2))
    prob = o.AdaptiveProblem(part, o.Survey(P, Q))
    D0, st = prob.simulate(m)
    Jv = prob.jacobian(st).apply(v := rng.normal(size=m.size))
    errs = []
    for t in (1e-2, 5e-3, 2.5e-3):
        errs.append(np.linalg.norm(prob.simulate(m + t * v)[0] - D0 - t * Jv))
    rate = np.log2(errs[0] / errs[1]), np.log2(errs[1] / errs[2])
    assert min(rate) > 1.8


def test_config1_inputs():
    from paper_1707_07598_b200.planar import config_problem_2d
    mesh, part, survey, m, d_obs = config_problem_2d(1)
    assert (mesh.n1, part.b1, part.n_blocks, part.n_coarse) == (64, 8, 64, 81)
    assert survey.Q.shape[1] == 1 and survey.P.shape[1] == 32 and d_obs.shape == (32, 1)
    assert np.isclose(survey.Q.sum(), 0.0) and np.all(np.isfinite(d_obs))
