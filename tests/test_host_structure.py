"""CPU tests of the host-side integer structure of the drop-in package:
partition index sets, CSC pattern of S and the survey matrices must be
bit-exact with the reference (golden vectors) and with the oracle."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.basis import csc_pattern, generate_bc_lagrange
from paper_1707_07598_b200.models import build_survey
from conftest import GOLDEN_CASES, load_golden
from oracle import msfv_oracle as orc

GEOMS = [((4, 4, 4), (2, 2, 2)), ((6, 6, 4), (3, 3, 2)), ((8, 8, 8), (4, 4, 4)),
         ((16, 8, 8), (8, 4, 4)), ((12, 8, 4), (4, 2, 1)), ((3, 3, 2), (1, 1, 1)), ((16, 16, 16), (8, 8, 8))]


@pytest.mark.parametrize("cells,blocks", GEOMS)
def test_partition_matches_oracle(cells, blocks):
    mesh = gp.create_mesh(*cells)
    part = gp.create_partition(mesh, *blocks)
    om = orc.Mesh(*cells)
    op = orc.make_partition(om, *blocks)
    assert part.n_blocks == op.n_blocks
    assert np.array_equal(part.skeleton, op.skeleton)
    assert np.array_equal(part.coarse_nodes, op.coarse_nodes)
    for j in range(part.n_blocks):
        assert np.array_equal(part.interiors[j], op.interiors[j])
        assert np.array_equal(part.boundaries[j], op.boundaries[j])


def test_partition_set_sizes():
    # mesh.py semantics: interiors disjoint and covering the non-skeleton nodes
    mesh = gp.create_mesh(12, 8, 8)
    part = gp.create_partition(mesh, 4, 4, 4)
    inter = np.concatenate(part.interiors)
    assert inter.size == np.unique(inter).size
    assert np.array_equal(np.sort(np.concatenate([inter, part.skeleton])), np.arange(mesh.n_nodes))
    assert all(b.size == 5 ** 3 - 3 ** 3 for b in part.boundaries)


def test_partition_rejects_bad_blocks():
    mesh = gp.create_mesh(6, 6, 6)
    with pytest.raises(ValueError):
        gp.create_partition(mesh, 4, 3, 3)
    with pytest.raises(ValueError):
        gp.create_mesh(0, 2, 2)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_csc_pattern_bit_exact_with_reference(name):
    g = load_golden(name)
    mesh = gp.create_mesh(*[int(x) for x in g["cells"]], *[float(x) for x in g["h"]])
    part = gp.create_partition(mesh, *[int(x) for x in g["blocks"]])
    indices, indptr, src, hatv = csc_pattern(part)
    assert np.array_equal(indptr, g["S_indptr"])
    assert np.array_equal(indices, g["S_indices"])
    skel = src < 0
    assert np.array_equal(hatv[skel], g["S_data"][skel])     # skeleton values are exact hats
    # interior entries map one-to-one onto the device block layout
    inner = src[~skel]
    assert inner.size == np.unique(inner).size


@pytest.mark.parametrize("cells,blocks", GEOMS[:5])
def test_lagrange_bc_matches_oracle(cells, blocks):
    mesh = gp.create_mesh(*cells)
    part = gp.create_partition(mesh, *blocks)
    V = generate_bc_lagrange(part).values
    Vo = orc.lagrange_values(orc.make_partition(orc.Mesh(*cells), *blocks))
    assert (V != Vo).nnz == 0
    # hats sum to one at every skeleton node (test_basis.py:80-94)
    skel = part.skeleton[part.skeleton != 0] - 1
    assert np.max(np.abs(np.asarray(V[skel].sum(axis=1)).ravel() - 1.0)) < 1e-12


@pytest.mark.parametrize("n,src,rec", [(16, (2, 2), (4, 4)), (32, (4, 4), (8, 8)), (128, (4, 4), (32, 32))])
def test_survey_matches_reference_layout(n, src, rec):
    mesh = gp.create_mesh(n, n, n, 1 / n, 1 / n, 1 / n)
    s = build_survey(mesh, src, rec)
    o = orc.top_survey(orc.Mesh(n, n, n, 1 / n, 1 / n, 1 / n), src, rec)
    assert (s.P != o.P).nnz == 0 and (s.Q != o.Q).nnz == 0
    assert s.P.shape == (mesh.n_nodes - 1, rec[0] * rec[1])


def test_survey_validation():
    mesh = gp.create_mesh(4, 4, 4)
    n = mesh.n_nodes - 1
    P = sp.csc_matrix((np.ones(2), ([3, 5], [0, 1])), shape=(n, 2))
    Q = sp.csc_matrix((n, 1))
    with pytest.raises(ValueError):
        gp.Survey(P=P, Q=Q)          # empty source column (forward.py:38-39)
    with pytest.raises(ValueError):
        gp.Survey(P=P, Q=sp.csc_matrix((np.ones(1), ([1], [0])), shape=(n - 1, 1)))


def test_operator_host_pieces_match_oracle():
    mesh = gp.create_mesh(5, 4, 3, 0.5, 1.0, 2.0)
    om = orc.Mesh(5, 4, 3, 0.5, 1.0, 2.0)
    G, C = gp.nodal_gradient(mesh), gp.edge_cell_map(mesh)
    Go, Co = orc.gradient_matrix(om), orc.cell_average_matrix(om)
    assert (G != Go).nnz == 0 and (C != Co).nnz == 0


def test_invalid_model_shape_raises_on_host():
    mesh = gp.create_mesh(4, 4, 4)
    with pytest.raises(ValueError):
        gp.assemble_operator(mesh, np.zeros(5))
    m = np.zeros(mesh.n_cells)
    m[3] = np.nan
    with pytest.raises(gp.InvalidModelError):
        gp.sigma_map(m)
