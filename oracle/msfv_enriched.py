"""CPU oracle for the enriched basis families (source, skeleton, local_pca).

TEST INFRASTRUCTURE ONLY (same rule as msfv_oracle.py: imported by ``tests/``
and the bench's CPU legs, never by the product).

Numpy/scipy restatement of the reference's family generators
(basis.py:119-245), the stacked boundary-condition block and per-block column
support (basis.py:379-450), the general basis assembly with forcing and
block-restricted columns (basis.py:511-616) and the masked edge profiles
(basis.py:596-608).  The projected solve and the adaptive sensitivity of
msfv_oracle.py are written for any S / EP and are reused unchanged
(forward.py:105-144, 209-281).

Parity is pinned: tests/test_oracle_enriched.py checks this module against
goldens of the unmodified reference (tests/golden/make_golden_enriched.py).
"""

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import msfv_oracle as orc

ORDER = ("lagrange", "source", "skeleton", "local_pca")      # basis.py:25


@dataclass
class Family:
    """BoundaryConditionSet (basis.py:56-76)."""

    name: str
    values: sp.csc_matrix
    forcing: sp.csc_matrix
    restrict: np.ndarray = None
    labels: list = None

    @property
    def count(self):
        return self.values.shape[1]


def lagrange(part):
    v = orc.lagrange_values(part)
    n = part.mesh.n_nodes - 1
    return Family("lagrange", v, sp.csc_matrix((n, v.shape[1])), None,
                  [("coarse_node", int(c)) for c in part.coarse_nodes])


def source(part, Q):
    """basis.py:119-138."""
    n = part.mesh.n_nodes - 1
    inside = np.zeros(n)
    for ids in part.interiors:
        inside[orc.pin(ids)] = 1.0
    R = (sp.diags(inside) @ sp.csc_matrix(Q)).tocsc()
    R.eliminate_zeros()
    keep = np.flatnonzero(np.diff(R.indptr) > 0)
    F = R[:, keep] if keep.size else sp.csc_matrix((n, 0))
    return Family("source", sp.csc_matrix((n, F.shape[1])), F, None, [("source", int(j)) for j in keep])


def reference_fields(part, m_ref, Q):
    """basis.py:141-149 (direct_factorize = SuperLU, solvers.py:30-40)."""
    op = orc.assemble(part.mesh, m_ref)
    return spla.splu(sp.csc_matrix(op.A)).solve(np.asarray(sp.csc_matrix(Q).todense(), dtype=float))


def skeleton(part, u_ref):
    """basis.py:162-181."""
    n = part.mesh.n_nodes - 1
    on = np.zeros(n)
    on[orc.pin(part.skeleton)] = 1.0
    V = sp.csc_matrix(np.asarray(u_ref, dtype=float) * (on[:, None] > 0))
    return Family("skeleton", V, sp.csc_matrix((n, V.shape[1])), None, [("skeleton", j) for j in range(V.shape[1])])


def local_pca(part, u_ref, rank, total=0, drop_tol=1e-10):
    """basis.py:184-245: mean trace first, then singular directions of the
    centred traces, Gram-Schmidt-ed by a QR; ``rank`` per block, ``total``
    overall by singular weight."""
    u = np.asarray(u_ref, dtype=float)
    ns = u.shape[1]
    n = part.mesh.n_nodes - 1
    got = []
    for j in range(part.n_blocks):
        b = orc.pin(part.boundaries[j])
        tr = u[b]
        mu = tr.mean(axis=1)
        Us, s, _ = sla.svd(tr - mu[:, None], full_matrices=False)
        nm = float(np.linalg.norm(mu))
        vecs = ([mu / nm] if nm > 0 else []) + [Us[:, r] for r in range(s.size)]
        wts = ([nm * np.sqrt(ns)] if nm > 0 else []) + [float(x) for x in s]
        if not vecs or max(wts) == 0.0:
            continue
        Qm, Rm = np.linalg.qr(np.column_stack(vecs))
        kept = 0
        for r, w in enumerate(wts):
            if kept >= rank or w < drop_tol * max(wts):
                break
            if abs(Rm[r, r]) < 1e-10:
                continue
            got.append((j, kept, w, b, Qm[:, r].copy()))
            kept += 1
    if total and len(got) > total:
        sel = np.sort(np.argsort([-t[2] for t in got], kind="stable")[:total])
        got = [got[i] for i in sel]
    if got:
        V = sp.coo_matrix((np.concatenate([t[4] for t in got]),
                           (np.concatenate([t[3] for t in got]),
                            np.concatenate([np.full(t[3].size, c) for c, t in enumerate(got)]))),
                          shape=(n, len(got))).tocsc()
    else:
        V = sp.csc_matrix((n, 0))
    return Family("local_pca", V, sp.csc_matrix((n, len(got))), np.array([t[0] for t in got], dtype=int),
                  [("local_pca", t[0], t[1]) for t in got])


def families(part, names, Q=None, m_ref=None, rank=0, total=0, drop_tol=1e-10):
    """BasisBuilder.__init__ (basis.py:623-652)."""
    u_ref = reference_fields(part, m_ref, Q) if {"skeleton", "local_pca"} & set(names) else None
    out = []
    for f in ORDER:
        if f not in names:
            continue
        out.append(lagrange(part) if f == "lagrange" else source(part, Q) if f == "source"
                   else skeleton(part, u_ref) if f == "skeleton" else local_pca(part, u_ref, rank, total, drop_tol))
    return out


def build_basis(op, part, fams):
    """assemble_basis for stacked families (basis.py:379-397, 445-450, 511-616)."""
    n = part.mesh.n_nodes - 1
    fams = sorted(fams, key=lambda f: ORDER.index(f.name))
    V = sp.hstack([f.values for f in fams], format="csc")
    F = sp.hstack([f.forcing for f in fams], format="csc")
    k = V.shape[1]
    restrict = np.concatenate([np.full(f.count, -1) if f.restrict is None else f.restrict for f in fams]).astype(int)
    Vr, Fr = V.tocsr(), F.tocsr()
    A = op.A
    cache = orc.build_cache(part, op.G, op.C, values=V)          # I, B, edge owners (basis.py:463-476)
    vcoo = V.tocoo()
    rows, cols, vals = [vcoo.row], [vcoo.col], [vcoo.data]
    factors = []
    for j in range(part.n_blocks):
        I, B = cache.I[j], cache.B[j]
        if I.size == 0:
            factors.append(None)
            continue
        hit = np.zeros(k, dtype=bool)
        if Vr.nnz and B.size:
            hit |= np.diff(Vr[B].tocsc().indptr) > 0
        if Fr.nnz:
            hit |= np.diff(Fr[I].tocsc().indptr) > 0
        cj = np.flatnonzero((hit & (restrict < 0)) | (restrict == j))          # basis.py:445-450
        AI = A[I]
        f = orc.BlockFactor(AI[:, I])
        factors.append(f)
        if cj.size:
            rhs = Fr[I][:, cj].toarray() - AI[:, B] @ Vr[B][:, cj].toarray()    # basis.py:548
            sol = f.solve(np.asarray(rhs))
            rows.append(np.repeat(I, cj.size))
            cols.append(np.tile(cj, I.size))
            vals.append(sol.ravel())
    S = sp.coo_matrix((np.arange(1, sum(v.size for v in vals) + 1, dtype=float),
                       (np.concatenate(rows), np.concatenate(cols))), shape=(n, k)).tocsc()
    flat = np.concatenate(vals)
    if S.nnz != flat.size:
        raise orc.OracleError("basis entries are not disjoint")
    S = sp.csc_matrix((flat[S.data.astype(np.int64) - 1], S.indices, S.indptr), shape=(n, k))
    prof = (op.G[:, 1:] @ S).tocoo()                                            # basis.py:596-608
    rc = restrict[prof.col]
    keep = (rc < 0) | (cache.edge_owner[prof.row] == rc)
    EP = sp.coo_matrix((prof.data[keep], (prof.row[keep], prof.col[keep])), shape=prof.shape).tocsc()

    class _F:                                                                   # empty interiors solve nothing
        def solve(self, B):
            return B
    factors = [f if f is not None else _F() for f in factors]
    basis = orc.Basis(part, op.m.copy(), S, factors, cache.I, EP, cache, op.G, op.C)
    basis.families = np.concatenate([np.full(f.count, f.name) for f in fams])
    basis.labels = [lab for f in fams for lab in f.labels]
    return basis
