"""CPU oracle for the adaptive MSFV forward + gradient path.

TEST INFRASTRUCTURE ONLY.  This module is the checker: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_1707_07598_b200``) never imports or calls it.

It is a numpy/scipy restatement of the reference package ``msinv``
(``/root/reference/pkg/src/msinv``) for the Lagrange-family adaptive path.
Each function cites the reference file:line it follows.  The arithmetic the
reference delegates to LAPACK (``dpotrf``/``dpotrs`` via
``scipy.linalg.cho_factor``/``cho_solve``) and SuperLU (``splu``) is called
through the same scipy entry points here (numpy>=1.24, scipy>=1.10 per
``pkg/pyproject.toml:9-13``; this image: numpy 2.3.5, scipy 1.18.1).
Per-source loops of the reference are batched over the source axis; the
algebra is unchanged.

Parity is pinned: ``tests/test_oracle_golden.py`` checks this module against
golden vectors produced by running the unmodified reference
(``tests/golden/make_golden.py``).
"""

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

DENSE_REDUCED_LIMIT = 5000      # forward.py:20


class OracleError(RuntimeError):
    pass


# Thread count of the per-block loops (the reference's `workers`,
# parallel.py:21-49).  LAPACK releases the GIL, so blocks run concurrently;
# results are collected in block order, hence bitwise independent of WORKERS.
WORKERS = 1


def run_indexed(fn, n):
    if WORKERS <= 1 or n <= 1:
        return [fn(j) for j in range(n)]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=WORKERS) as ex:
        return list(ex.map(fn, range(n), chunksize=max(1, n // (4 * WORKERS))))


# --------------------------------------------------------------------- mesh

@dataclass(frozen=True)
class Mesh:
    """Uniform tensor mesh, x-fastest numbering (mesh.py:12-75)."""

    n1: int
    n2: int
    n3: int
    h1: float = 1.0
    h2: float = 1.0
    h3: float = 1.0

    @property
    def n_cells(self):
        return self.n1 * self.n2 * self.n3

    @property
    def n_nodes(self):
        return (self.n1 + 1) * (self.n2 + 1) * (self.n3 + 1)

    @property
    def volume(self):
        return self.h1 * self.h2 * self.h3

    def node(self, i, j, k):                       # mesh.py:51-54
        return np.asarray(i) + (self.n1 + 1) * (np.asarray(j) + (self.n2 + 1) * np.asarray(k))

    def node_ijk(self, idx):                       # mesh.py:56-60
        idx = np.asarray(idx)
        i = idx % (self.n1 + 1)
        r = idx // (self.n1 + 1)
        return i, r % (self.n2 + 1), r // (self.n2 + 1)

    def cell(self, i, j, k):                       # mesh.py:62-64
        return np.asarray(i) + self.n1 * (np.asarray(j) + self.n2 * np.asarray(k))


@dataclass
class Partition:
    """Nested coarse partition (mesh.py:79-182)."""

    mesh: Mesh
    b: tuple
    interiors: list
    boundaries: list
    skeleton: np.ndarray
    coarse_nodes: np.ndarray

    @property
    def nb(self):
        m = self.mesh
        return (m.n1 // self.b[0], m.n2 // self.b[1], m.n3 // self.b[2])

    @property
    def n_blocks(self):
        a, b, c = self.nb
        return a * b * c

    @property
    def n_coarse(self):
        a, b, c = self.nb
        return (a + 1) * (b + 1) * (c + 1)


def make_partition(mesh, b1, b2, b3):
    """Vectorized restatement of create_partition (mesh.py:143-182)."""
    for n, b in ((mesh.n1, b1), (mesh.n2, b2), (mesh.n3, b3)):
        if b < 1 or n % b:
            raise ValueError("block size must divide the cell count")
    i, j, k = mesh.node_ijk(np.arange(mesh.n_nodes))
    skeleton = np.flatnonzero((i % b1 == 0) | (j % b2 == 0) | (k % b3 == 0))
    coarse = np.flatnonzero((i % b1 == 0) & (j % b2 == 0) & (k % b3 == 0))
    nb1, nb2, nb3 = mesh.n1 // b1, mesh.n2 // b2, mesh.n3 // b3
    # local node box of one block, x fastest -> sorted global order
    lx, ly, lz = np.meshgrid(np.arange(b1 + 1), np.arange(b2 + 1), np.arange(b3 + 1),
                             indexing="ij")
    lx, ly, lz = lx.ravel(order="F"), ly.ravel(order="F"), lz.ravel(order="F")
    inner = ((lx > 0) & (lx < b1) & (ly > 0) & (ly < b2) & (lz > 0) & (lz < b3))
    interiors, boundaries = [], []
    for bk in range(nb3):
        for bj in range(nb2):
            for bi in range(nb1):
                ids = mesh.node(bi * b1 + lx, bj * b2 + ly, bk * b3 + lz)
                interiors.append(ids[inner])          # already ascending
                boundaries.append(ids[~inner])
    return Partition(mesh, (b1, b2, b3), interiors, boundaries, skeleton, coarse)


def pin(ids):
    """Full ids -> pinned ids, dropping node 0 (basis.py:78-81)."""
    ids = np.asarray(ids)
    return ids[ids != 0] - 1


# ---------------------------------------------------------------- operators

def sigma_of(m):
    """exp(m) with the finite check (operators.py:23-28)."""
    m = np.asarray(m, dtype=float)
    if not np.all(np.isfinite(m)):
        raise ValueError("model vector contains non-finite entries")
    return np.exp(m)


def _edge_axes(mesh):
    n1, n2, n3 = mesh.n1, mesh.n2, mesh.n3
    return ((n1, n2 + 1, n3 + 1), (n1 + 1, n2, n3 + 1), (n1 + 1, n2 + 1, n3))


def _edge_ijk(shape):
    i, j, k = np.meshgrid(*(np.arange(s) for s in shape), indexing="ij")
    return i.ravel(order="F"), j.ravel(order="F"), k.ravel(order="F")


def gradient_matrix(mesh):
    """Node->edge difference G, rows x-, y-, z-edges (operators.py:36-74)."""
    h = (mesh.h1, mesh.h2, mesh.h3)
    rows, cols, vals, off = [], [], [], 0
    for ax, shape in enumerate(_edge_axes(mesh)):
        i, j, k = _edge_ijk(shape)
        a = mesh.node(i, j, k)
        d = [0, 0, 0]
        d[ax] = 1
        b = mesh.node(i + d[0], j + d[1], k + d[2])
        r = off + np.arange(a.size)
        rows += [r, r]
        cols += [a, b]
        vals += [np.full(a.size, -1.0 / h[ax]), np.full(a.size, 1.0 / h[ax])]
        off += a.size
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(off, mesh.n_nodes)).tocsr()


def cell_average_matrix(mesh):
    """Edge<-cell map with V/4 per touching cell (operators.py:77-109)."""
    nmax = (mesh.n1, mesh.n2, mesh.n3)
    rows, cols, off = [], [], 0
    for ax, shape in enumerate(_edge_axes(mesh)):
        ijk = list(_edge_ijk(shape))
        r = off + np.arange(ijk[0].size)
        t1, t2 = [a for a in range(3) if a != ax]
        for d1 in (-1, 0):
            for d2 in (-1, 0):
                c = [x.copy() for x in ijk]
                c[t1] += d1
                c[t2] += d2
                ok = (c[t1] >= 0) & (c[t1] < nmax[t1]) & (c[t2] >= 0) & (c[t2] < nmax[t2])
                rows.append(r[ok])
                cols.append(mesh.cell(c[0][ok], c[1][ok], c[2][ok]))
        off += ijk[0].size
    rows = np.concatenate(rows)
    return sp.coo_matrix((np.full(rows.size, 0.25 * mesh.volume), (rows, np.concatenate(cols))),
                         shape=(off, mesh.n_cells)).tocsr()


@dataclass
class Operator:
    mesh: Mesh
    m: np.ndarray
    sigma: np.ndarray
    G: sp.csr_matrix
    C: sp.csr_matrix
    w: np.ndarray
    A: sp.csr_matrix


def assemble(mesh, m, pieces=None):
    """A(m) = G^T diag(C sigma) G with node 0 eliminated (operators.py:123-141)."""
    m = np.asarray(m, dtype=float)
    if m.shape != (mesh.n_cells,):
        raise ValueError("model length mismatch")
    sigma = sigma_of(m)
    G, C = pieces if pieces is not None else (gradient_matrix(mesh), cell_average_matrix(mesh))
    w = C @ sigma
    A = (G.T @ sp.diags(w) @ G).tocsr()[1:, 1:].tocsr()
    return Operator(mesh, m.copy(), sigma, G, C, w, A)


# -------------------------------------------------------------------- basis

def hat(part, coarse_node, node_ids):
    """Trilinear coarse hat at full node ids (basis.py:84-92)."""
    mesh = part.mesh
    ci, cj, ck = mesh.node_ijk(coarse_node)
    i, j, k = mesh.node_ijk(np.asarray(node_ids))
    w = np.ones(np.atleast_1d(i).shape, dtype=float)
    for x, c, b in ((i, ci, part.b[0]), (j, cj, part.b[1]), (k, ck, part.b[2])):
        w = w * np.maximum(0.0, 1.0 - np.abs(np.asarray(x, dtype=float) - c) / b)
    return w


def lagrange_values(part):
    """Skeleton hat data, one column per coarse node (basis.py:95-116).

    Same entries as the reference; the hat of each coarse node is evaluated
    only on the skeleton nodes of its support box instead of the whole
    skeleton (values outside the box are exactly zero there too)."""
    mesh = part.mesh
    n = mesh.n_nodes - 1
    is_skel = np.zeros(mesh.n_nodes, dtype=bool)
    is_skel[part.skeleton] = True
    is_skel[0] = False                                   # pinned node dropped (basis.py:100)
    b1, b2, b3 = part.b
    rows, cols, vals = [], [], []
    for c, cn in enumerate(part.coarse_nodes):
        ci, cj, ck = mesh.node_ijk(cn)
        ii = np.arange(max(ci - b1 + 1, 0), min(ci + b1 - 1, mesh.n1) + 1)
        jj = np.arange(max(cj - b2 + 1, 0), min(cj + b2 - 1, mesh.n2) + 1)
        kk = np.arange(max(ck - b3 + 1, 0), min(ck + b3 - 1, mesh.n3) + 1)
        K, J, I = np.meshgrid(kk, jj, ii, indexing="ij")
        ids = mesh.node(I.ravel(), J.ravel(), K.ravel())
        ids = ids[is_skel[ids]]
        w = hat(part, cn, ids)
        nz = np.flatnonzero(w)
        rows.append(ids[nz] - 1)
        cols.append(np.full(nz.size, c))
        vals.append(w[nz])
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, part.n_coarse)).tocsc()


@dataclass
class Cache:
    """Model-independent per-block data (basis.py:421-492), Lagrange family."""

    values: sp.csc_matrix
    I: list
    B: list
    cols: list
    xb: list
    edge_owner: np.ndarray
    block_edges: list
    cells: list
    s_indices: np.ndarray = None
    s_indptr: np.ndarray = None
    s_perm: np.ndarray = None


def build_cache(part, G, C, values=None):
    values = lagrange_values(part) if values is None else values
    vcsr = values.tocsr()
    n = part.mesh.n_nodes - 1
    I_l, B_l, cols_l, xb_l = [], [], [], []
    for j in range(part.n_blocks):
        I = pin(part.interiors[j])
        B = pin(part.boundaries[j])
        if I.size:
            sub = vcsr[B]
            cols = np.flatnonzero(np.diff(sub.tocsc().indptr) > 0)    # basis.py:445-450
            xb = sub[:, cols].toarray()
        else:
            cols = np.empty(0, dtype=np.int64)
            xb = np.zeros((B.size, 0))
        I_l.append(I)
        B_l.append(B)
        cols_l.append(cols)
        xb_l.append(xb)
    # edge ownership: max over endpoint interior owners (basis.py:467-476)
    node_owner = np.full(n, -1, dtype=np.int64)
    for j, I in enumerate(I_l):
        node_owner[I] = j
    Gc = G.tocoo()
    end_owner = np.where(Gc.col == 0, -1, node_owner[np.maximum(Gc.col - 1, 0)])
    owner = np.full(G.shape[0], -1, dtype=np.int64)
    np.maximum.at(owner, Gc.row, end_owner)
    order = np.argsort(owner, kind="stable")
    counts = np.bincount(owner[owner >= 0], minlength=part.n_blocks)
    start = np.searchsorted(owner[order], 0)
    bounds = start + np.concatenate([[0], np.cumsum(counts)])
    block_edges = [np.sort(order[bounds[j]:bounds[j + 1]]) for j in range(part.n_blocks)]
    Ccsr = C.tocsr()
    cells = []
    for e in block_edges:                                           # basis.py:480-492
        if e.size == 0:
            cells.append(np.empty(0, dtype=np.int64))
        else:
            cells.append(np.unique(Ccsr[e].indices))
    return Cache(values, I_l, B_l, cols_l, xb_l, owner, block_edges, cells)


@dataclass
class Basis:
    part: Partition
    model: np.ndarray
    S: sp.csc_matrix
    factors: list
    I: list
    EP: sp.csc_matrix
    cache: Cache
    G: sp.csr_matrix
    C: sp.csr_matrix

    @property
    def k(self):
        return self.S.shape[1]

    @property
    def n(self):
        return self.S.shape[0]

    def interior_solve(self, w):
        """blockdiag(A_II^-1) on interiors, zero on the skeleton (basis.py:339-353)."""
        w = np.asarray(w, dtype=float)
        out = np.zeros_like(w)

        def task(j):
            I = self.I[j]
            return self.factors[j].solve(w[I]) if I.size else None

        for I, sol in zip(self.I, run_indexed(task, len(self.I))):
            if sol is not None:
                out[I] = sol
        return out


DENSE_BLOCK_LIMIT = 2000        # basis.py (DENSE_BLOCK_LIMIT)


class BlockFactor:
    """One block's A_II factor (_BlockFactor, basis.py:258-298): dense lower
    Cholesky up to DENSE_BLOCK_LIMIT unknowns, SuperLU beyond (the explicit
    inverse the reference switches to for wide solves only changes rounding)."""

    def __init__(self, A_II_sparse):
        self.n = A_II_sparse.shape[0]
        self.chol = self.lu = None
        if self.n <= DENSE_BLOCK_LIMIT:
            self.chol = sla.cho_factor(A_II_sparse.toarray(), lower=True, check_finite=False)   # basis.py:271-275
        else:
            self.lu = spla.splu(sp.csc_matrix(A_II_sparse))                                    # basis.py:276-278

    def solve(self, B):
        if self.chol is not None:
            return sla.cho_solve(self.chol, B, check_finite=False)
        return self.lu.solve(np.asarray(B, dtype=float))


def build_basis(op, part, cache=None):
    """Per-block Cholesky + solve, scatter into reference CSC order
    (basis.py:511-616; _BlockFactor basis.py:258-298, dense path).  The
    per-block factor/solve runs on WORKERS threads (ordered, like
    parallel.run_indexed, parallel.py:21-49)."""
    n = part.mesh.n_nodes - 1
    if cache is None:
        cache = build_cache(part, op.G, op.C)
    A = op.A

    def task(j):
        I, B, cols = cache.I[j], cache.B[j], cache.cols[j]
        if I.size == 0:
            return None, np.zeros((0, cols.size))
        AI = A[I]
        rhs = -(AI[:, B] @ cache.xb[j])                           # basis.py:548 (rhs0 = 0)
        f = BlockFactor(AI[:, I])                                   # basis.py:553-563
        return f, (f.solve(np.asarray(rhs)) if cols.size else np.zeros((I.size, 0)))

    res = run_indexed(task, part.n_blocks)
    factors = [r[0] for r in res]
    sols = [r[1] for r in res]
    vcoo = cache.values.tocoo()
    flat = np.concatenate([vcoo.data] + [s.ravel() for s in sols])
    if cache.s_perm is None:                                         # basis.py:576-592
        rows = [vcoo.row] + [np.repeat(cache.I[j], cache.cols[j].size)
                             for j in range(part.n_blocks) if cache.cols[j].size]
        cols = [vcoo.col] + [np.tile(cache.cols[j], cache.I[j].size)
                             for j in range(part.n_blocks) if cache.cols[j].size]
        probe = sp.coo_matrix((np.arange(1, flat.size + 1, dtype=np.float64),
                               (np.concatenate(rows), np.concatenate(cols))),
                              shape=(n, part.n_coarse)).tocsc()
        if probe.nnz != flat.size:
            raise OracleError("basis entries are not disjoint")
        cache.s_indices, cache.s_indptr = probe.indices, probe.indptr
        cache.s_perm = probe.data.astype(np.int64) - 1
    S = sp.csc_matrix((flat[cache.s_perm], cache.s_indices, cache.s_indptr),
                      shape=(n, part.n_coarse))
    EP = (op.G[:, 1:] @ S).tocsc()                                   # basis.py:601
    return Basis(part, op.m.copy(), S, factors, cache.I, EP, cache, op.G, op.C)


# ------------------------------------------------------------------ forward

@dataclass
class Survey:
    P: sp.csc_matrix
    Q: sp.csc_matrix


@dataclass
class Reduced:
    op: Operator
    basis: Basis
    A_k: object
    T: np.ndarray
    shift: float
    chol: object = None
    lu: object = None

    def solve(self, B):                                  # forward.py:72-75
        if self.chol is not None:
            return sla.cho_solve(self.chol, B)
        return self.lu.solve(np.asarray(B, dtype=float))


def forward_reduced(op, survey, basis, force_shift=False):
    """F = S^T Q, A_k = S^T A S, T = A_k^-1 F, D = P^T S T (forward.py:105-144).

    ``force_shift`` (test hook) takes the reference's except-branch as if the
    first factorization had failed: the shifted operator A_k + 1e-12 tr(A_k)/k I
    (forward.py:122-129, 136-139)."""
    k = basis.k
    S = basis.S
    F = np.asarray((S.T @ survey.Q).todense())
    if k <= DENSE_REDUCED_LIMIT:
        A_k = (S.T @ (op.A @ S)).toarray()
        shift = 0.0
        try:
            if force_shift:
                raise sla.LinAlgError("forced")
            chol = sla.cho_factor(A_k, lower=True)
        except sla.LinAlgError:
            shift = 1e-12 * np.trace(A_k) / k                # forward.py:123
            chol = sla.cho_factor(A_k + shift * np.eye(k), lower=True)
        st = Reduced(op, basis, A_k, None, shift, chol=chol)
    else:
        A_k = (S.T @ (op.A @ S)).tocsc()
        shift = 0.0
        try:
            if force_shift:
                raise RuntimeError("forced")
            lu = spla.splu(A_k)
        except RuntimeError:
            shift = 1e-12 * A_k.diagonal().sum() / k
            lu = spla.splu((A_k + shift * sp.eye(k, format="csc")).tocsc())
        st = Reduced(op, basis, A_k, None, shift, lu=lu)
    st.T = st.solve(F)
    D = np.asarray(survey.P.T @ (S @ st.T))
    return D, st


def misfit(D, D_obs):
    """0.5 ||D - D_obs||_F^2 and the residual (inversion.py:22-29)."""
    r = np.asarray(D, dtype=float) - np.asarray(D_obs, dtype=float)
    return 0.5 * float(np.sum(r * r)), r


class Sensitivity:
    """Adaptive sensitivity J, J^T (forward.py:209-281), sources batched."""

    def __init__(self, state, survey):
        op, basis = state.op, state.basis
        if not np.array_equal(basis.model, op.m):
            raise OracleError("stale basis")
        self.state, self.survey, self.basis = state, survey, basis
        self.A = op.A
        self.S = basis.S
        self.Gp = op.G[:, 1:].tocsr()
        self.Csig = (op.C @ sp.diags(op.sigma)).tocsr()
        self.EP = basis.EP.tocsr()
        T = state.T
        U = basis.S @ T                                      # forward.py:241
        R = survey.Q.toarray() - op.A @ U                     # forward.py:243
        self.gprof = self.EP @ T                              # forward.py:244
        self.gu = self.Gp @ U                                 # forward.py:245
        self.a = self.Gp @ basis.interior_solve(R)            # forward.py:246

    def apply(self, dm):                                      # forward.py:258-269
        c = self.Csig @ np.asarray(dm, dtype=float)
        ydm = -self.basis.interior_solve(self.Gp.T @ (self.gprof * c[:, None]))
        xdm = -(self.EP.T @ (self.a * c[:, None]))
        gdm = self.Gp.T @ (self.gu * c[:, None])
        rhs = xdm - self.S.T @ (gdm + self.A @ ydm)
        dt = self.state.solve(rhs)
        return np.asarray(self.survey.P.T @ (ydm + self.S @ dt))

    def rapply(self, W):                                      # forward.py:271-281
        W = np.asarray(W, dtype=float)
        p = np.asarray(self.survey.P @ W)
        y = self.state.solve(np.asarray(self.S.T @ p))
        sy = self.S @ y
        z = self.basis.interior_solve(p - self.A @ sy)
        e = (self.gprof * (self.Gp @ z) + self.a * (self.EP @ y)
             + self.gu * (self.Gp @ sy))
        return -(self.Csig.T @ e.sum(axis=1))


# ------------------------------------------------------------- Yk / Xk (Table 3)

def apply_Yk(basis, v, m):
    """Materialized d(S v)/dm, n x N_m CSR (basis.py:684-751)."""
    if not np.array_equal(basis.model, np.asarray(m, dtype=float)):
        raise OracleError("stale basis")
    Gp = basis.G[:, 1:]
    Csig = (basis.C @ sp.diags(sigma_of(m))).tocsr()
    gv = basis.EP @ np.asarray(v, dtype=float)
    W = (Gp.T @ sp.diags(gv) @ Csig).tocsr()
    rows, cols, vals = [], [], []
    for j, I in enumerate(basis.I):
        if I.size == 0:
            continue
        cells = basis.cache.cells[j]
        Wd = W[I][:, cells].toarray()
        nz = np.flatnonzero(Wd.any(axis=0))
        if nz.size == 0:
            continue
        sol = -basis.factors[j].solve(Wd[:, nz])
        rows.append(np.repeat(I, nz.size))
        cols.append(np.tile(cells[nz], I.size))
        vals.append(sol.ravel())
    shape = (basis.n, Csig.shape[1])
    if not rows:
        return sp.csr_matrix(shape)
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=shape).tocsr()


def apply_Xk(basis, w, m):
    """Materialized d(S^T w)/dm, k x N_m CSR (basis.py:754-800)."""
    if not np.array_equal(basis.model, np.asarray(m, dtype=float)):
        raise OracleError("stale basis")
    Gp = basis.G[:, 1:]
    Csig = (basis.C @ sp.diags(sigma_of(m))).tocsr()
    a = Gp @ basis.interior_solve(w)
    EPr = basis.EP.tocsr()
    rows, cols, vals = [], [], []
    for j, edges in enumerate(basis.cache.block_edges):
        if edges.size == 0:
            continue
        V = EPr[edges].tocsc()
        sup = np.flatnonzero(np.diff(V.indptr))
        if sup.size == 0:
            continue
        aj = a[edges]
        if not np.any(aj):
            continue
        Vd = V[:, sup].toarray()
        used = basis.cache.cells[j]
        Cjd = Csig[edges][:, used].toarray()
        contrib = -((Vd * aj[:, None]).T @ Cjd)
        rows.append(np.repeat(sup, used.size))
        cols.append(np.tile(used, sup.size))
        vals.append(contrib.ravel())
    shape = (basis.k, Csig.shape[1])
    if not rows:
        return sp.csr_matrix(shape)
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=shape).tocsr()


# ------------------------------------------------------------------- inputs

def surface_positions(count, n):
    """models.py:46-51."""
    return np.unique(np.round(np.linspace(0, n, count + 2))[1:-1].astype(int))


def top_survey(mesh, n_src, n_rec):
    """Top-plane dipoles and point receivers, pinned ids (models.py:54-83)."""
    n = mesh.n_nodes - 1
    kt = mesh.n3
    sx = surface_positions(n_src[0], mesh.n1 - 1)
    sy = surface_positions(n_src[1], mesh.n2)
    rows, cols, vals, col = [], [], [], 0
    for j in sy:
        for i in sx:
            rows += [mesh.node(i, j, kt) - 1, mesh.node(i + 1, j, kt) - 1]
            cols += [col, col]
            vals += [1.0, -1.0]
            col += 1
    Q = sp.csc_matrix((vals, (rows, cols)), shape=(n, col))
    rx = surface_positions(n_rec[0], mesh.n1)
    ry = surface_positions(n_rec[1], mesh.n2)
    rec = [mesh.node(i, j, kt) - 1 for j in ry for i in rx]
    P = sp.csc_matrix((np.ones(len(rec)), (rec, np.arange(len(rec)))), shape=(n, len(rec)))
    return Survey(P, Q)


# --------------------------------------------------------------- full path

class AdaptiveProblem:
    """Oracle twin of AdaptiveReducedProblem (inversion.py:307-323)."""

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
