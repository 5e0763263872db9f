"""Host logic of the enriched basis families (enriched.py) on a numpy engine
against goldens of the unmodified reference (make_golden_enriched.py):
boundary-condition data (basis.py:119-245), the CSC pattern of the extra
columns, the block-eliminated bordered coarse solve, the masked edge profiles
and the edge-space sensitivity (forward.py:209-281)."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1707_07598_b200 as gp
from paper_1707_07598_b200 import enriched as en
from conftest import load_golden, rel
from numpy_engine import NumpyEngine, NumpyOperator

ENR_CASES = ["enr_c1212_all", "enr_c1688_tot", "enr_c24_b8", "enr_c1212_src", "enr_c888_nolag"]


def csc(g, key, shape):
    return sp.csc_matrix((g[key + "_data"], g[key + "_indices"], g[key + "_indptr"]), shape=shape)


def setup(g):
    cells, h, blocks = tuple(int(x) for x in g["cells"]), tuple(float(x) for x in g["h"]), tuple(int(x) for x in g["blocks"])
    mesh = gp.create_mesh(*cells, *h)
    part = gp.create_partition(mesh, *blocks)
    eng = NumpyEngine(cells, h, blocks)
    survey = gp.Survey(P=csc(g, "P", tuple(g["P_shape"])), Q=csc(g, "Q", tuple(g["Q_shape"])))
    fams = tuple(str(f) for f in g["families"])
    spec = gp.BasisSpec(families=fams, pca_rank=int(g["pca_rank"]), pca_total=int(g["pca_total"]))
    builder = gp.BasisBuilder(part, spec, Q=survey.Q, m_ref=g["m_ref"])
    builder._engine = lambda: eng
    return mesh, part, eng, survey, builder


@pytest.mark.parametrize("name", ENR_CASES)
def test_bc_families_match_reference(name):
    g = load_golden(name)
    mesh, part, eng, survey, builder = setup(g)
    n = mesh.n_nodes - 1
    for bc in builder.bc_sets:
        if bc.family == "lagrange":
            continue
        V = csc(g, f"bc_{bc.family}_V", (n, bc.count))
        F = csc(g, f"bc_{bc.family}_F", (n, bc.count))
        mine = sp.csc_matrix(bc.values)
        assert np.array_equal(mine.indptr, V.indptr) and np.array_equal(mine.indices, V.indices), bc.family
        assert rel(mine.data, V.data) <= 1e-10 if V.nnz else True
        fm = sp.csc_matrix(bc.forcing)
        assert np.array_equal(fm.indptr, F.indptr) and np.array_equal(fm.indices, F.indices)
        assert np.array_equal(fm.data, F.data)
        if bc.block_restrict is not None:
            assert np.array_equal(bc.block_restrict, g[f"bc_{bc.family}_restrict"])


@pytest.mark.parametrize("name", ENR_CASES)
def test_enriched_host_logic_matches_reference(name):
    g = load_golden(name)
    mesh, part, eng, survey, builder = setup(g)
    n = mesh.n_nodes - 1
    op = NumpyOperator(eng, g["m"])
    basis = builder.assemble(op)
    assert basis.k == g["A_k"].shape[0]
    assert list(basis.families) == [str(f) for f in g["col_family"]]
    assert [repr(lab) for lab in basis.labels] == [str(x) for x in g["labels"]]
    S_ref = csc(g, "S", (n, basis.k))
    SE_ref = S_ref[:, basis.kL:]
    SE = basis.S_extra
    assert np.array_equal(SE.indptr, SE_ref.indptr) and np.array_equal(SE.indices, SE_ref.indices)
    assert rel(SE.data, SE_ref.data) <= 1e-10
    D, state = en.forward_enriched(op, survey, basis)
    assert rel(state.A_k, g["A_k"]) <= 1e-10
    assert rel(state.T, g["T"]) <= 1e-9          # coefficient split between near-dependent columns
    assert rel(D, g["D"]) <= 1e-10
    assert state.shift == float(g["shift"])
    J = en.EnrichedSensitivity(state, survey)
    assert rel(J.rapply(g["resid"]), g["g"]) <= 1e-9
    assert rel(J.rapply(g["W"]), g["JtW"]) <= 1e-10
    assert rel(J.apply(g["dm"]), g["Jv"]) <= 1e-10
    rng = np.random.default_rng(3)
    B = rng.normal(size=(basis.k, 2))
    assert rel(g["A_k"] @ state.solve_reduced(B), B) <= 1e-9
