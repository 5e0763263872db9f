"""GPU parity of the enriched basis families (source,
skeleton, local_pca; basis.py:119-245, forward.py:105-144, 209-281) against
goldens of the unmodified reference (tests/golden/make_golden_enriched.py).

Two layers: (1) with the reference's own boundary-condition data injected,
the model-dependent path (local solves of the extra columns, bordered coarse
solve, masked edge profiles, J v, J^T w) must match to 1e-10; (2) with the
boundary-condition data generated here from a device fine solve at m_ref,
the data itself and everything downstream must match to the accuracy of that
solve (PCG to 1e-13 vs the reference's SuperLU)."""

from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1707_07598_b200 as gp
from paper_1707_07598_b200 import enriched as en
from conftest import load_golden, rel

pytestmark = pytest.mark.gpu

ENR_CASES = ["enr_c1212_all", "enr_c1688_tot", "enr_c24_b8", "enr_c1212_src", "enr_c888_nolag"]
TOL = 1e-10


def csc(g, key, shape):
    return sp.csc_matrix((g[key + "_data"], g[key + "_indices"], g[key + "_indptr"]), shape=shape)


def setup(g):
    cells, h = tuple(int(x) for x in g["cells"]), tuple(float(x) for x in g["h"])
    blocks = tuple(int(x) for x in g["blocks"])
    mesh = gp.create_mesh(*cells, *h)
    part = gp.create_partition(mesh, *blocks)
    survey = gp.Survey(P=csc(g, "P", tuple(g["P_shape"])), Q=csc(g, "Q", tuple(g["Q_shape"])))
    fams = tuple(str(f) for f in g["families"])
    spec = gp.BasisSpec(families=fams, pca_rank=int(g["pca_rank"]), pca_total=int(g["pca_total"]))
    builder = gp.BasisBuilder(part, spec, Q=survey.Q, m_ref=g["m_ref"])
    return mesh, part, survey, builder


def golden_bc_sets(g, part, fams):
    """The reference's boundary-condition data (values, forcing, restriction)."""
    from paper_1707_07598_b200.basis import generate_bc_lagrange
    n = part.mesh.n_nodes - 1
    col_family = [str(f) for f in g["col_family"]]
    labels = [eval(str(x)) for x in g["labels"]]
    sets = []
    for fam in fams:
        if fam == "lagrange":
            sets.append(generate_bc_lagrange(part))
            continue
        cnt = col_family.count(fam)
        off = col_family.index(fam) if cnt else 0
        rst = g[f"bc_{fam}_restrict"] if f"bc_{fam}_restrict" in g else None
        sets.append(SimpleNamespace(family=fam, values=csc(g, f"bc_{fam}_V", (n, cnt)),
                                    forcing=csc(g, f"bc_{fam}_F", (n, cnt)), block_restrict=rst,
                                    labels=labels[off:off + cnt], dropped=[], count=cnt))
    return sets


def run_chain(g, mesh, survey, builder):
    op = gp.assemble_operator(mesh, g["m"])
    basis = builder.assemble(op)
    D, state = gp.forward_reduced(op, survey, basis)
    J = gp.sensitivity_adaptive(state, survey)
    phi, resid = gp.misfit_ssd(D, g["d_obs"])
    return op, basis, D, state, J, phi, resid


@pytest.mark.parametrize("name", ENR_CASES)
def test_enriched_matches_reference_with_reference_bc(name):
    g = load_golden(name)
    mesh, part, survey, builder = setup(g)
    builder._bc_sets = golden_bc_sets(g, part, builder.spec.families)
    op, basis, D, state, J, phi, resid = run_chain(g, mesh, survey, builder)
    n = mesh.n_nodes - 1
    assert basis.k == g["A_k"].shape[0]
    assert list(basis.families) == [str(f) for f in g["col_family"]]
    S_ref = csc(g, "S", (n, basis.k))
    S = basis.S
    assert np.array_equal(S.indptr, S_ref.indptr) and np.array_equal(S.indices, S_ref.indices), "S pattern"
    errs = {"S": rel(S.data, S_ref.data), "A_k": rel(state.A_k, g["A_k"]), "D": rel(D, g["D"]),
            "ST": rel(S @ state.T, S_ref @ g["T"]), "phi": abs(phi - float(g["phi"])) / float(g["phi"]),
            "g": rel(J.rapply(resid), g["g"]), "JtW": rel(J.rapply(g["W"]), g["JtW"]),
            "Jv": rel(J.apply(g["dm"]), g["Jv"]), "isolve": rel(basis.interior_solve(g["wv"]), g["isolve"])}
    EP = basis.edge_profiles
    EP_ref = csc(g, "EP", EP.shape)
    dEP = (EP - EP_ref).tocsc()
    errs["EP"] = float(np.linalg.norm(dEP.data) / np.linalg.norm(EP_ref.data)) if dEP.nnz else 0.0
    errs["gedge"] = rel(basis.grad_edge(g["T"][:, 0]), g["gedge"])
    assert state.shift == float(g["shift"])
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, (bad, errs)
    # T itself: split between near-dependent columns, compare through A_k
    assert rel(g["A_k"] @ state.T, g["A_k"] @ g["T"]) <= 1e-9
    # adjoint identity <J dm, W> = <dm, J^T W> (test_forward.py adjoint oracle)
    lhs = float(np.sum(J.apply(g["dm"]) * g["W"]))
    rhs = float(np.dot(g["dm"], J.rapply(g["W"])))
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), abs(rhs), 1e-300) * 100


@pytest.mark.parametrize("name", ENR_CASES)
def test_enriched_end_to_end_with_device_reference_fields(name):
    g = load_golden(name)
    mesh, part, survey, builder = setup(g)
    n = mesh.n_nodes - 1
    for bc in builder.bc_sets:
        if bc.family == "lagrange":
            continue
        V = csc(g, f"bc_{bc.family}_V", (n, bc.count))
        mine = sp.csc_matrix(bc.values)
        assert np.array_equal(mine.indptr, V.indptr) and np.array_equal(mine.indices, V.indices), bc.family
        if V.nnz:
            assert rel(mine.data, V.data) <= 1e-7, (bc.family, rel(mine.data, V.data))
        if bc.block_restrict is not None:
            assert np.array_equal(bc.block_restrict, g[f"bc_{bc.family}_restrict"])
    op, basis, D, state, J, phi, resid = run_chain(g, mesh, survey, builder)
    errs = {"D": rel(D, g["D"]), "g": rel(J.rapply(resid), g["g"]), "JtW": rel(J.rapply(g["W"]), g["JtW"]),
            "Jv": rel(J.apply(g["dm"]), g["Jv"])}
    bad = {k: v for k, v in errs.items() if not v <= 1e-6}
    assert not bad, (bad, errs)


def test_problem_protocol_and_dropped_sources():
    """AdaptiveReducedProblem with enriched families (inversion.py:307-323);
    a source family whose sources all sit on the skeleton adds no column and
    falls back to the Lagrange path (basis.py:131-137)."""
    g = load_golden("enr_c24_b8")
    mesh, part, survey, builder = setup(g)
    builder._bc_sets = golden_bc_sets(g, part, builder.spec.families)
    prob = gp.AdaptiveReducedProblem(builder, survey)
    D, state = prob.simulate(g["m"])
    assert rel(D, g["D"]) <= TOL
    assert rel(prob.jacobian(state).rapply(g["W"]), g["JtW"]) <= TOL
    b2 = gp.BasisBuilder(part, gp.BasisSpec(families=("lagrange", "source")), Q=survey.Q)
    assert b2.bc_sets[1].count == 0 and len(b2.bc_sets[1].dropped) == survey.n_sources
    op = gp.assemble_operator(mesh, g["m"])
    basis = b2.assemble(op)
    assert basis.k == part.n_coarse_nodes
    D2, _ = gp.forward_reduced(op, survey, basis)
    b1 = gp.BasisBuilder(part)
    op1 = gp.assemble_operator(mesh, g["m"])
    D1, _ = gp.forward_reduced(op1, survey, b1.assemble(op1))
    assert rel(D2, D1) <= 1e-13


def test_acceptance_criterion_8_sizes_and_oracle_parity():
    """test_acceptance.py:333-349 (k = 150 with 12^3 blocks, k = 572 with 6^3
    blocks on a 36x36x12 mesh, 25 sources), then forward + gradient + J v of
    those bases against the enriched oracle fed the same boundary data."""
    from oracle import msfv_enriched as oen
    from oracle import msfv_oracle as orc
    mesh = gp.create_mesh(36, 36, 12)
    survey = gp.build_survey(mesh, n_src=(5, 5), n_rec=(8, 8))
    assert survey.n_sources == 25
    m_ref = np.full(mesh.n_cells, np.log(0.01))
    rng = np.random.default_rng(5)
    m = m_ref + 0.5 * rng.normal(size=mesh.n_cells)
    omesh = orc.Mesh(36, 36, 12)
    oop = orc.assemble(omesh, m)
    osurvey = orc.Survey(survey.P, survey.Q)
    for blocks, rank, total, k in ((12, 11, 93, 150), (6, 6, 400, 572)):
        part = gp.create_partition(mesh, blocks, blocks, blocks)
        spec = gp.BasisSpec(families=("lagrange", "skeleton", "local_pca"), pca_rank=rank, pca_total=total)
        builder = gp.BasisBuilder(part, spec, Q=survey.Q, m_ref=m_ref)
        op = gp.assemble_operator(mesh, m)
        basis = builder.assemble(op)
        assert basis.k == k
        D, state = gp.forward_reduced(op, survey, basis)
        J = gp.sensitivity_adaptive(state, survey)
        W = rng.normal(size=D.shape)
        dm = rng.normal(size=mesh.n_cells)
        opart = orc.make_partition(omesh, blocks, blocks, blocks)
        fams = [oen.Family(s.family, sp.csc_matrix(s.values), sp.csc_matrix(s.forcing), s.block_restrict, s.labels)
                for s in builder.bc_sets]
        ob = oen.build_basis(oop, opart, fams)
        D0, st0 = orc.forward_reduced(oop, osurvey, ob)
        J0 = orc.Sensitivity(st0, osurvey)
        errs = {"D": rel(D, D0), "JtW": rel(J.rapply(W), J0.rapply(W)), "Jv": rel(J.apply(dm), J0.apply(dm)),
                "S": rel(basis.S.data, ob.S.data)}
        assert np.array_equal(basis.S.indices, ob.S.indices) and np.array_equal(basis.S.indptr, ob.S.indptr)
        bad = {kk: v for kk, v in errs.items() if not v <= 1e-9}
        assert not bad, (blocks, errs)
