"""Reduced-dimension boundary conditions: the CPU oracle
(oracle/msfv_reduced.py) against the reference's own basis properties.  The
reference has no reduced-boundary code, so parity is unpinned;
these are the properties its tests hold the hat basis to
(test_basis.py:57-71, test_acceptance.py:48-73)."""

import numpy as np
import pytest

from oracle import msfv_oracle as orc
from oracle import msfv_reduced as red

GEOMS = [((8, 8, 8), (4, 4, 4), (1.0, 1.0, 1.0)), ((12, 8, 8), (4, 4, 2), (0.5, 1.0, 2.0)),
         ((16, 16, 8), (8, 8, 4), (1.0, 1.0, 1.0))]


@pytest.mark.parametrize("cells,b,h", GEOMS)
def test_unit_conductivity_reproduces_hats(cells, b, h):
    mesh = orc.Mesh(*cells, *h)
    part = orc.make_partition(mesh, *b)
    V = red.reduced_values(part, orc.assemble(mesh, np.zeros(mesh.n_cells)).w)
    H = orc.lagrange_values(part)
    assert np.array_equal(V.indptr, H.indptr) and np.array_equal(V.indices, H.indices)
    assert np.max(np.abs(V.data - H.data)) <= 1e-14


@pytest.mark.parametrize("cells,b,h", GEOMS)
def test_partition_of_unity_and_pattern(cells, b, h, rng):
    mesh = orc.Mesh(*cells, *h)
    part = orc.make_partition(mesh, *b)
    op = orc.assemble(mesh, 1.5 * rng.normal(size=mesh.n_cells))
    basis = red.build_basis_reduced(op, part)
    rows = np.asarray(basis.S.sum(axis=1)).ravel()
    assert np.max(np.abs(rows - 1.0)) <= 1e-12
    H = orc.build_basis(orc.assemble(mesh, np.zeros(mesh.n_cells)), part).S
    assert np.array_equal(basis.S.indptr, H.indptr) and np.array_equal(basis.S.indices, H.indices)
    # the skeleton data adapt to the model: they differ from the hats
    assert np.max(np.abs(basis.S.data - H.data)) > 1e-3


@pytest.mark.parametrize("cells,b,h", GEOMS + [((8, 4, 2), (4, 2, 1), (1.0, 1.0, 1.0))])
def test_skeleton_map_matches_oracle_and_differentiates(cells, b, h, rng):
    """paper_1707_07598_b200.skeleton (the differentiable skeleton map behind
    the reduced-boundary sensitivities) on the CPU: its entries equal the
    oracle's reduced_values, its J v matches central differences and its
    vector-Jacobian product satisfies the adjoint identity."""
    import torch
    import paper_1707_07598_b200 as gp
    from paper_1707_07598_b200.skeleton import SkeletonMap
    mesh = orc.Mesh(*cells, *h)
    part = orc.make_partition(mesh, *b)
    w = np.asarray(orc.assemble(mesh, 1.2 * rng.normal(size=mesh.n_cells)).w)
    B = red.reduced_values(part, w).tocsc()
    gmesh = gp.create_mesh(*cells, *h)
    sk = SkeletonMap(gp.create_partition(gmesh, *b), "cpu")
    wt = torch.from_numpy(w)
    vals = sk.values(wt)
    nodes, cols = (t.numpy().copy() for t in sk.entries())
    assert len(vals) == B.nnz - (part.n_coarse - 1)          # all but the coarse nodes' own unit entries (node 0 pinned)
    assert np.max(np.abs(vals.numpy() - np.asarray(B[nodes - 1, cols]).ravel())) <= 1e-13
    lam = torch.from_numpy(rng.normal(size=len(vals)))
    dw = torch.from_numpy(0.1 * w * rng.normal(size=len(w)))
    jv, g = sk.jvp(wt, dw), sk.vjp(wt, lam)
    eps = 1e-6
    fd = (sk.values(wt + eps * dw) - sk.values(wt - eps * dw)) / (2 * eps)
    assert float((jv - fd).abs().max() / jv.abs().max()) <= 1e-7
    a, c = float(torch.dot(g, dw)), float(torch.dot(lam, jv))
    assert abs(a - c) <= 1e-12 * abs(c)
