"""Gauss-Newton on the GPU problem (SURVEY 8(b) boundary, 8(f) N3).

* The reference's own outer loop, msinv.projected_gauss_newton
  (inversion.py:187-263), imported unmodified from baseline/_ref, drives
  paper_1707_07598_b200.AdaptiveReducedProblem: its trace and final model
  match the same loop driving the reference's CPU AdaptiveReducedProblem.
* gauss_newton_dev (device-resident) reproduces that trace too.
* DeviceObjective matches the reference Objective (value, gradient, Hessian).
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import import_reference, load_golden, rel

pytestmark = pytest.mark.gpu

msinv = import_reference()
needs_ref = pytest.mark.skipif(msinv is None, reason="reference not installed under baseline/_ref")


def _setup(name="c16_b844", bounds=False):
    import paper_1707_07598_b200 as gp
    g = load_golden(name)
    cells, h, b = [int(x) for x in g["cells"]], [float(x) for x in g["h"]], [int(x) for x in g["blocks"]]
    P = sp.csc_matrix((g["P_data"], g["P_indices"], g["P_indptr"]), shape=tuple(g["P_shape"]))
    Q = sp.csc_matrix((g["Q_data"], g["Q_indices"], g["Q_indptr"]), shape=tuple(g["Q_shape"]))
    mesh = gp.create_mesh(*cells, *h)
    gprob = gp.AdaptiveReducedProblem(gp.BasisBuilder(gp.create_partition(mesh, *b)), gp.Survey(P=P, Q=Q))
    from msinv.basis import BasisBuilder, BasisSpec
    from msinv.forward import Survey
    from msinv.inversion import AdaptiveReducedProblem, GNConfig, Objective
    from msinv.mesh import create_mesh, create_partition
    rmesh = create_mesh(*cells, *h)
    rprob = AdaptiveReducedProblem(BasisBuilder(create_partition(rmesh, *b), BasisSpec(families=("lagrange",))),
                                   Survey(P=P, Q=Q))
    m0 = np.zeros(rmesh.n_cells)
    obj = Objective(mesh=rmesh, alpha=1e-3, m_ref=np.zeros(rmesh.n_cells))
    kw = dict(max_gn=3, max_cg=6)
    if bounds:
        kw.update(lower=-0.15, upper=0.15)
    return g, gprob, rprob, m0, obj, GNConfig(**kw)


def _compare(tr_a, tr_b, m_a, m_b):
    assert len(tr_a.rows) == len(tr_b.rows)
    for ra, rb in zip(tr_a.rows, tr_b.rows):
        for c in ("iter", "cg_iters", "active", "rebuilt"):
            assert ra[c] == rb[c], (c, ra, rb)
        assert ra["step"] == rb["step"]
        for c in ("phi", "reg", "total", "pgnorm"):
            assert abs(ra[c] - rb[c]) <= 1e-8 * max(abs(rb[c]), 1e-300), (c, ra, rb)
    assert tr_a.line_search_failed == tr_b.line_search_failed
    assert rel(m_a, m_b) <= 1e-8


@needs_ref
@pytest.mark.parametrize("bounds", [False, True])
def test_reference_gn_loop_drives_gpu_problem(bounds):
    from msinv.inversion import projected_gauss_newton
    g, gprob, rprob, m0, obj, cfg = _setup(bounds=bounds)
    m_gpu, tr_gpu = projected_gauss_newton(gprob, m0, g["d_obs"], obj, cfg)
    m_ref, tr_ref = projected_gauss_newton(rprob, m0, g["d_obs"], obj, cfg)
    assert tr_ref.totals()[-1] < tr_ref.totals()[0]
    _compare(tr_gpu, tr_ref, m_gpu, m_ref)


@needs_ref
@pytest.mark.parametrize("bounds", [False, True])
def test_device_gn_matches_reference_loop(bounds):
    import paper_1707_07598_b200 as gp
    from msinv.inversion import projected_gauss_newton
    g, gprob, rprob, m0, obj, cfg = _setup(bounds=bounds)
    m_dev, tr_dev = gp.gauss_newton_dev(gprob, m0, g["d_obs"], obj, cfg)
    m_ref, tr_ref = projected_gauss_newton(rprob, m0, g["d_obs"], obj, cfg)
    _compare(tr_dev, tr_ref, m_dev, m_ref)


@needs_ref
def test_device_objective_matches_reference(rng):
    import torch
    import paper_1707_07598_b200 as gp
    from msinv.inversion import Objective
    from msinv.mesh import create_mesh
    for cells, h in (((7, 5, 4), (1.0, 0.5, 2.0)), ((16, 16, 8), (1 / 16, 1 / 16, 1 / 8))):
        rmesh = create_mesh(*cells, *h)
        m_ref = rng.normal(size=rmesh.n_cells)
        obj = Objective(mesh=rmesh, alpha=0.37, m_ref=m_ref)
        dobj = gp.DeviceObjective(gp.create_mesh(*cells, *h), 0.37, m_ref)
        m = rng.normal(size=rmesh.n_cells)
        v = rng.normal(size=rmesh.n_cells)
        r0, g0 = obj.value_grad(m)
        r1, g1 = dobj.value_grad(torch.from_numpy(m).cuda())
        assert abs(float(r1) - r0) <= 1e-13 * abs(r0)
        assert rel(g1.cpu().numpy(), g0) <= 1e-13
        assert rel(dobj.hess_apply(torch.from_numpy(v).cuda()).cpu().numpy(), obj.hess_apply(v)) <= 1e-14
