"""CPU oracle for the 2D adaptive MSFV path (BASELINE.json configs 1-2).

TEST INFRASTRUCTURE ONLY (same rule as msfv_oracle.py: only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import it).

The reference package is 3D only, so there is no reference
output to pin 2D against: PARITY UNPINNED by the reference.  This module
restates the reference algorithm with d = 2 as SURVEY.md 8(c) prescribes:
  * mesh / partition: mesh.py:12-75, 143-182 with two axes (x fastest;
    block interior (b-1)^2 nodes, boundary (b+1)^2 - (b-1)^2);
  * operator: operators.py:36-141 with x- then y-edges (i fastest) and the
    edge<-cell average C = V/2 per touching cell (V = h1 h2), so sigma = 1
    interior rows are the 5-point stencil; node 0 pinned;
  * Lagrange basis: bilinear hats (basis.py:84-116);
  * basis build, Galerkin, coarse solve, sensitivity: the 3D oracle's
    functions (basis.py:511-616, forward.py:105-144, 224-281), which are
    dimension-free once the mesh pieces above are supplied.
It is validated by 2D ports of the reference's own test oracles
(tests/test_oracle2d.py: partition of unity, local solve vs dense solve,
sigma = 1 bilinear reproduction, Galerkin identity, adjoint and Taylor tests).
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import msfv_oracle as o3


@dataclass(frozen=True)
class Mesh2D:
    n1: int
    n2: int
    h1: float = 1.0
    h2: float = 1.0

    @property
    def n_cells(self):
        return self.n1 * self.n2

    @property
    def n_nodes(self):
        return (self.n1 + 1) * (self.n2 + 1)

    @property
    def volume(self):
        return self.h1 * self.h2

    def node(self, i, j):
        return np.asarray(i) + (self.n1 + 1) * np.asarray(j)

    def node_ij(self, idx):
        idx = np.asarray(idx)
        return idx % (self.n1 + 1), idx // (self.n1 + 1)

    def cell(self, i, j):
        return np.asarray(i) + self.n1 * np.asarray(j)


@dataclass
class Partition2D:
    mesh: Mesh2D
    b: tuple
    interiors: list
    boundaries: list
    skeleton: np.ndarray
    coarse_nodes: np.ndarray

    @property
    def nb(self):
        return (self.mesh.n1 // self.b[0], self.mesh.n2 // self.b[1])

    @property
    def n_blocks(self):
        a, b = self.nb
        return a * b

    @property
    def n_coarse(self):
        a, b = self.nb
        return (a + 1) * (b + 1)


def make_partition(mesh, b1, b2):
    """create_partition (mesh.py:143-182) with two axes."""
    for n, b in ((mesh.n1, b1), (mesh.n2, b2)):
        if b < 1 or n % b:
            raise ValueError("block size must divide the cell count")
    i, j = mesh.node_ij(np.arange(mesh.n_nodes))
    skeleton = np.flatnonzero((i % b1 == 0) | (j % b2 == 0))
    coarse = np.flatnonzero((i % b1 == 0) & (j % b2 == 0))
    lx, ly = np.meshgrid(np.arange(b1 + 1), np.arange(b2 + 1), indexing="ij")
    lx, ly = lx.ravel(order="F"), ly.ravel(order="F")
    inner = (lx > 0) & (lx < b1) & (ly > 0) & (ly < b2)
    interiors, boundaries = [], []
    for bj in range(mesh.n2 // b2):
        for bi in range(mesh.n1 // b1):
            ids = mesh.node(bi * b1 + lx, bj * b2 + ly)
            interiors.append(ids[inner])
            boundaries.append(ids[~inner])
    return Partition2D(mesh, (b1, b2), interiors, boundaries, skeleton, coarse)


def gradient_matrix(mesh):
    """Node->edge differences, x-edges then y-edges, i fastest (operators.py:36-74)."""
    rows, cols, vals, off = [], [], [], 0
    for ax, (s1, s2, h) in enumerate(((mesh.n1, mesh.n2 + 1, mesh.h1), (mesh.n1 + 1, mesh.n2, mesh.h2))):
        i, j = np.meshgrid(np.arange(s1), np.arange(s2), indexing="ij")
        i, j = i.ravel(order="F"), j.ravel(order="F")
        a = mesh.node(i, j)
        b = mesh.node(i + (ax == 0), j + (ax == 1))
        r = off + np.arange(a.size)
        rows += [r, r]
        cols += [a, b]
        vals += [np.full(a.size, -1.0 / h), np.full(a.size, 1.0 / h)]
        off += a.size
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(off, mesh.n_nodes)).tocsr()


def cell_average_matrix(mesh):
    """Edge<-cell map, V/2 per touching cell (operators.py:77-109 with d = 2)."""
    rows, cols, off = [], [], 0
    for ax, (s1, s2) in enumerate(((mesh.n1, mesh.n2 + 1), (mesh.n1 + 1, mesh.n2))):
        i, j = np.meshgrid(np.arange(s1), np.arange(s2), indexing="ij")
        i, j = i.ravel(order="F"), j.ravel(order="F")
        r = off + np.arange(i.size)
        for d in (-1, 0):
            ci, cj = (i, j + d) if ax == 0 else (i + d, j)
            ok = (ci >= 0) & (ci < mesh.n1) & (cj >= 0) & (cj < mesh.n2)
            rows.append(r[ok])
            cols.append(mesh.cell(ci[ok], cj[ok]))
        off += i.size
    rows = np.concatenate(rows)
    return sp.coo_matrix((np.full(rows.size, 0.5 * mesh.volume), (rows, np.concatenate(cols))),
                         shape=(off, mesh.n_cells)).tocsr()


def hat(part, coarse_node, node_ids):
    """Bilinear coarse hat (basis.py:84-92 with two axes)."""
    mesh = part.mesh
    ci, cj = mesh.node_ij(coarse_node)
    i, j = mesh.node_ij(np.asarray(node_ids))
    w = np.ones(np.atleast_1d(i).shape, dtype=float)
    for x, c, b in ((i, ci, part.b[0]), (j, cj, part.b[1])):
        w = w * np.maximum(0.0, 1.0 - np.abs(np.asarray(x, dtype=float) - c) / b)
    return w


def lagrange_values(part):
    """Skeleton hat data, one column per coarse node, pinned node dropped (basis.py:95-116)."""
    mesh = part.mesh
    n = mesh.n_nodes - 1
    is_skel = np.zeros(mesh.n_nodes, dtype=bool)
    is_skel[part.skeleton] = True
    is_skel[0] = False
    b1, b2 = part.b
    rows, cols, vals = [], [], []
    for c, cn in enumerate(part.coarse_nodes):
        ci, cj = mesh.node_ij(cn)
        ii = np.arange(max(ci - b1 + 1, 0), min(ci + b1 - 1, mesh.n1) + 1)
        jj = np.arange(max(cj - b2 + 1, 0), min(cj + b2 - 1, mesh.n2) + 1)
        J, I = np.meshgrid(jj, ii, indexing="ij")
        ids = mesh.node(I.ravel(), J.ravel())
        ids = ids[is_skel[ids]]
        w = hat(part, cn, ids)
        nz = np.flatnonzero(w)
        rows.append(ids[nz] - 1)
        cols.append(np.full(nz.size, c))
        vals.append(w[nz])
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, part.n_coarse)).tocsc()


def assemble(mesh, m, pieces=None):
    pieces = pieces if pieces is not None else (gradient_matrix(mesh), cell_average_matrix(mesh))
    return o3.assemble(mesh, m, pieces=pieces)


def build_cache(part, G, C):
    return o3.build_cache(part, G, C, values=lagrange_values(part))


def build_basis(op, part, cache=None):
    return o3.build_basis(op, part, cache if cache is not None else build_cache(part, op.G, op.C))


forward_reduced = o3.forward_reduced
misfit = o3.misfit
Survey = o3.Survey
Sensitivity = o3.Sensitivity


def fine_solve(op, Q):
    """Fine-grid forward u = A^-1 Q, the d_obs generator of config 1 (forward.py:78-98)."""
    return spla.splu(op.A.tocsc()).solve(np.asarray(Q.toarray() if sp.issparse(Q) else Q, dtype=float))


class AdaptiveProblem:
    """2D twin of the oracle's AdaptiveProblem (inversion.py:307-323)."""

    mode = "ms_adaptive"

    def __init__(self, part, survey):
        self.part = part
        self.survey = survey
        self.pieces = (gradient_matrix(part.mesh), cell_average_matrix(part.mesh))
        self.cache = build_cache(part, *self.pieces)

    def simulate(self, m):
        op = assemble(self.part.mesh, m, pieces=self.pieces)
        basis = build_basis(op, self.part, self.cache)
        return forward_reduced(op, self.survey, basis)

    def jacobian(self, state):
        return Sensitivity(state, self.survey)
