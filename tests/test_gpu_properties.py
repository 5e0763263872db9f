"""GPU property tests restated from the reference suite (pkg/tests), run
through the drop-in API on the CUDA path: partition of unity, homogeneous
reduction to trilinear hats, Galerkin exactness, Taylor and adjoint tests of
the adaptive sensitivity with a rebuilt basis, objective-gradient finite
differences, determinism and the error contract."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import assert_quadratic, rel

pytestmark = pytest.mark.gpu

gp = pytest.importorskip("paper_1707_07598_b200")


def point_survey(mesh, n_rec=6, n_src=3, seed=0, dipoles=False):
    """pkg/tests/test_forward.py:17-31 (random receivers / sources, pinned ids)."""
    rng = np.random.default_rng(seed)
    n = mesh.n_nodes - 1
    rec = rng.choice(n, size=n_rec, replace=False)
    P = sp.csc_matrix((np.ones(n_rec), (rec, np.arange(n_rec))), shape=(n, n_rec))
    if dipoles:
        a = rng.choice(n - 1, size=n_src, replace=False)
        Q = sp.csc_matrix((np.r_[np.ones(n_src), -np.ones(n_src)], (np.r_[a, a + 1], np.r_[0:n_src, 0:n_src])),
                          shape=(n, n_src))
    else:
        s = rng.choice(n, size=n_src, replace=False)
        Q = sp.csc_matrix((np.ones(n_src), (s, np.arange(n_src))), shape=(n, n_src))
    return gp.Survey(P=P, Q=Q)


def build(cells, blocks, m, h=(1.0, 1.0, 1.0)):
    mesh = gp.create_mesh(*cells, *h)
    part = gp.create_partition(mesh, *blocks)
    op = gp.assemble_operator(mesh, m)
    basis = gp.BasisBuilder(part).assemble(op)
    return mesh, part, op, basis


def test_partition_of_unity_random_model():
    # test_basis.py:104-110 and acceptance criterion 1 (16x16x8 / 4^3, <= 1e-10)
    for cells, blocks, seed in (((8, 8, 4), (2, 2, 2), 77), ((16, 16, 8), (4, 4, 4), 101), ((32, 32, 32), (8, 8, 8), 5)):
        m = np.random.default_rng(seed).uniform(-3, 3, int(np.prod(cells)))
        _, _, _, basis = build(cells, blocks, m)
        total = np.asarray(basis.S.sum(axis=1)).ravel()
        assert np.max(np.abs(total - 1.0)) <= 1e-10


def test_homogeneous_basis_is_trilinear_hats():
    # test_basis.py:113-118, acceptance criterion 2
    mesh, part, _, basis = build((16, 16, 8), (4, 4, 4), np.zeros(16 * 16 * 8))
    S = basis.S.tocsc()
    ids = np.arange(1, mesh.n_nodes)
    worst = 0.0
    for c, cn in enumerate(part.coarse_nodes):
        col = S[:, c].toarray().ravel()
        worst = max(worst, float(np.max(np.abs(col - gp.coarse_hat_values(part, cn, ids)))))
    assert worst <= 1e-10


def test_interior_solve_matches_dense(rng):
    # test_basis.py:165-178 (dense local-solve oracle)
    cells, blocks = (8, 8, 8), (4, 4, 4)
    m = 0.5 * rng.normal(size=512)
    mesh, part, op, basis = build(cells, blocks, m)
    A = op.A.toarray()
    w = rng.normal(size=op.n)
    z = basis.interior_solve(w)
    for j in range(part.n_blocks):
        I = part.interiors[j] - 1
        ref = np.linalg.solve(A[np.ix_(I, I)], w[I])
        assert np.allclose(z[I], ref, rtol=1e-12, atol=1e-14)
    skel = part.skeleton[part.skeleton != 0] - 1
    assert np.all(z[skel] == 0.0)


def test_galerkin_exactness(rng):
    # test_forward.py:114-128: q in range(A S) is reproduced exactly
    mesh, part, op, basis = build((6, 6, 4), (3, 3, 2), 0.2 * rng.normal(size=144))
    t_star = rng.normal(size=basis.k)
    q = op.A @ (basis.S @ t_star)
    n = op.n
    rec = rng.choice(n, size=8, replace=False)
    P = sp.csc_matrix((np.ones(8), (rec, np.arange(8))), shape=(n, 8))
    D, st = gp.forward_reduced(op, gp.Survey(P=P, Q=sp.csc_matrix(q[:, None])), basis)
    U = np.linalg.solve(op.A.toarray(), q)
    D_full = P.T @ U
    assert np.linalg.norm(D[:, 0] - D_full) / np.linalg.norm(D_full) <= 1e-8


def test_homogeneous_coarse_galerkin_oracle():
    # test_forward.py:131-147
    mesh, part, op, basis = build((6, 6, 6), (3, 3, 3), np.zeros(216))
    survey = point_survey(mesh, n_rec=5, n_src=2, seed=3)
    ids = np.arange(1, mesh.n_nodes)
    H = np.column_stack([gp.coarse_hat_values(part, cn, ids) for cn in part.coarse_nodes])
    K = H.T @ op.A @ H
    F = H.T @ survey.Q.toarray()
    D_oracle = (survey.P.T @ H) @ np.linalg.solve(K, F)
    D, _ = gp.forward_reduced(op, survey, basis)
    assert np.allclose(D, D_oracle, rtol=1e-9, atol=1e-12)


def _problem(cells, blocks, survey_seed, m):
    mesh = gp.create_mesh(*cells)
    part = gp.create_partition(mesh, *blocks)
    survey = point_survey(mesh, n_rec=8, n_src=3, seed=survey_seed, dipoles=True)
    return mesh, gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey), survey


def test_adaptive_sensitivity_taylor(rng):
    # test_forward.py:228-243 (Taylor with rebuilt basis: quadratic remainders)
    m = 0.2 * rng.normal(size=8 * 8 * 8)
    mesh, prob, survey = _problem((8, 8, 8), (4, 4, 4), 9, m)
    D0, st = prob.simulate(m)
    J = prob.jacobian(st)
    dm = rng.normal(size=m.size)
    assert np.allclose(J.apply(np.zeros(m.size)), 0.0)
    rem, eps = [], 1e-2
    Jdm = J.apply(dm)
    for _ in range(6):
        rem.append(np.linalg.norm(prob.simulate(m + eps * dm)[0] - D0 - eps * Jdm))
        eps *= 0.5
    assert_quadratic(rem)


def test_adaptive_sensitivity_adjoint(rng):
    # test_forward.py:246-258 (<= 1e-12)
    m = 0.25 * rng.normal(size=8 * 8 * 8)
    mesh, prob, survey = _problem((8, 8, 8), (4, 4, 4), 13, m)
    _, st = prob.simulate(m)
    J = prob.jacobian(st)
    dm = rng.normal(size=m.size)
    W = rng.normal(size=(survey.n_receivers, survey.n_sources))
    lhs = np.sum(J.apply(dm) * W)
    rhs = np.dot(dm, J.rapply(W))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), abs(rhs))


def test_objective_gradient_central_difference(rng):
    # test_inversion.py:192-219 (ms_adaptive mode, rel 1e-5)
    m0 = np.log(0.05) + 0.05 * rng.normal(size=8 * 8 * 4)
    mesh = gp.create_mesh(8, 8, 4)
    part = gp.create_partition(mesh, 2, 2, 2)
    survey = point_survey(mesh, n_rec=10, n_src=3, seed=4, dipoles=True)
    prob = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
    d_obs = prob.simulate(m0 + 0.3)[0]
    import torch
    obj = gp.DeviceObjective(mesh, 1e-4, np.full(m0.size, np.log(0.05)))

    def reg(mm):
        r, gr = obj.value_grad(torch.from_numpy(mm).cuda())
        return float(r), gr.cpu().numpy()

    def total(mm):
        D, _ = prob.simulate(mm)
        return gp.misfit_ssd(D, d_obs)[0] + reg(mm)[0]

    D, st = prob.simulate(m0)
    _, resid = gp.misfit_ssd(D, d_obs)
    g = prob.jacobian(st).rapply(resid) + reg(m0)[1]
    dm = rng.normal(size=m0.size)
    eps = 1e-6
    fd = (total(m0 + eps * dm) - total(m0 - eps * dm)) / (2 * eps)
    assert fd == pytest.approx(float(g @ dm), rel=1e-5)


def test_runs_are_bitwise_deterministic(rng):
    # test_basis.py:411-425 / cli.py:186-210 (bitwise identical reruns)
    m = rng.normal(size=16 * 16 * 16)
    mesh, prob, survey = _problem((16, 16, 16), (8, 8, 8), 21, m)
    outs = []
    for _ in range(2):
        D, st = prob.simulate(m)
        J = prob.jacobian(st)
        outs.append((D, J.rapply(D), J.apply(m), st.basis.S.data))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_error_contract(rng):
    mesh = gp.create_mesh(8, 8, 4)
    part = gp.create_partition(mesh, 2, 2, 2)
    builder = gp.BasisBuilder(part)
    m = np.zeros(mesh.n_cells)
    survey = point_survey(mesh, n_rec=4, n_src=2, seed=1, dipoles=True)
    m2 = m.copy()
    m2[0] = np.inf
    for bad in (m2, m - 800.0):                                       # non-finite / exp underflow
        with pytest.raises(gp.InvalidModelError):
            op = gp.assemble_operator(mesh, bad)
            gp.forward_reduced(op, survey, builder.assemble(op))
    basis = builder.assemble(gp.assemble_operator(mesh, m))
    with pytest.raises(gp.StaleBasisError):
        basis.check_model(m + 1e-3)
    basis.check_model(m.copy())
    with pytest.raises(ValueError):                                   # basis.py:631 (needs Q and m_ref)
        gp.BasisBuilder(part, gp.BasisSpec(families=("lagrange", "skeleton")))
    with pytest.raises(ValueError):                                   # basis.py:47-49
        gp.BasisSpec(families=("lagrange", "wavelet"))
    with pytest.raises(NotImplementedError):                          # reduced BCs are Lagrange-only
        gp.BasisBuilder(part, gp.BasisSpec(families=("lagrange", "source"), boundary="reduced"))
    with pytest.raises(ValueError):
        gp.misfit_ssd(np.zeros((2, 2)), np.zeros((2, 3)))


def test_gauss_newton_decreases_objective(rng):
    # the method of inversion.py:187-263, device-resident (trace monotone)
    mesh = gp.create_mesh(8, 8, 4)
    part = gp.create_partition(mesh, 2, 2, 2)
    survey = point_survey(mesh, n_rec=12, n_src=3, seed=2, dipoles=True)
    prob = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
    m_true = 0.4 * rng.normal(size=mesh.n_cells)
    d_obs = prob.simulate(m_true)[0]
    obj = gp.DeviceObjective(mesh, 1e-3, np.zeros(mesh.n_cells))
    m, trace = gp.gauss_newton_dev(prob, np.zeros(mesh.n_cells), d_obs, obj, gp.GNSettings(max_gn=3, max_cg=5))
    tot = trace.totals()
    assert np.all(np.diff(tot) <= 1e-15 * abs(tot[0]))
    assert tot[-1] < tot[0]


def test_device_misfit_matches_host(rng):
    """msfv_misfit (misfit_ssd on the device, inversion.py:22-29): residual bitwise, phi to rounding,
    reruns bitwise."""
    import torch
    D, Dobs = rng.normal(size=(1024, 16)), rng.normal(size=(1024, 16))
    phi0, r0 = gp.misfit_ssd(D, Dobs)
    Dd, Do = torch.from_numpy(D).cuda(), torch.from_numpy(Dobs).cuda()
    phi, r = gp.misfit_ssd_dev(Dd, Do)
    phi2, _ = gp.misfit_ssd_dev(Dd, Do)
    assert np.array_equal(r.cpu().numpy(), r0)
    assert abs(float(phi) - phi0) <= 1e-13 * phi0 and float(phi) == float(phi2)
    with pytest.raises(ValueError):
        gp.misfit_ssd_dev(Dd, Do[:, :3])
