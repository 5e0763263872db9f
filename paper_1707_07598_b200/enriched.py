"""Enriched basis families on the GPU: ``source``, ``skeleton``, ``local_pca``
(reference basis.py:119-245, 379-616, forward.py:105-144,
209-281).

The Lagrange columns keep their block layout and the structured coarse solver
(basis.py / forward.py here).  The extra columns -- a few per source, or a few
per block -- are dense node fields ``E[node][column]`` on the device:

  build     E = V + blockdiag(A_II^-1) M o (F - A V)       (basis.py:537-563)
            V Dirichlet values, F interior forcing, M the block restriction of
            the local_pca columns (only their own block solves, basis.py:445-450)
  project   A_k = [[A_LL, A_LE], [A_LE^T, A_EE]],  A_LE = S_L^T (A E),
            A_EE = E^T (A E)                                (forward.py:101-102)
  solve     block elimination: the multifrontal/banded Cholesky of A_LL (the
            Lagrange Galerkin operator) and a dense Cholesky of the Schur
            complement A_EE - A_LE^T A_LL^-1 A_LE         (forward.py:117-142)

The sensitivities follow forward.py:224-281 in edge space (msfv_edge_grad /
msfv_edge_div / msfv_cell_gather).  The reference masks the edge profiles of
block-restricted columns to the edges their block owns (basis.py:602-608):
with Delta = (1 - mask) o (G_p E_pca),

  EP v   = G_p (S v) - Delta v_pca,      EP^T f = S^T G_p^T f - [0; Delta^T f].

Dense products with E are plain GEMMs (torch.matmul); every stencil, local
solve and coarse solve is a libmsfv kernel.  There is no CPU path.
"""

from types import SimpleNamespace

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import torch

from .errors import ReducedSingularError

FAMILY_ORDER = ("lagrange", "source", "skeleton", "local_pca")
DENSE_FIELD_LIMIT = 48 << 30       # bytes of E we are willing to hold (dense node fields)


def _pin(ids):
    ids = np.asarray(ids)
    return ids[ids != 0] - 1


# ------------------------------------------------------- boundary-condition data

def source_family(partition, Q):
    """generate_bc_source (basis.py:119-138): the sources restricted to block
    interiors as forcing, zero Dirichlet data; empty restrictions dropped."""
    n = partition.mesh.n_nodes - 1
    Q = sp.csc_matrix(Q)
    inside = np.zeros(n, dtype=bool)
    for ids in partition.interiors:
        inside[_pin(ids)] = True
    R = sp.csc_matrix(sp.diags(inside.astype(float)) @ Q)
    R.eliminate_zeros()
    nz = np.diff(R.indptr)
    keep = np.flatnonzero(nz > 0)
    forcing = R[:, keep] if keep.size else sp.csc_matrix((n, 0))
    return SimpleNamespace(family="source", values=sp.csc_matrix((n, forcing.shape[1])), forcing=forcing,
                           block_restrict=None, labels=[("source", int(j)) for j in keep],
                           dropped=np.flatnonzero(nz == 0).tolist(), count=forcing.shape[1])


def skeleton_family(partition, u_ref):
    """generate_bc_skeleton (basis.py:162-181): skeleton trace of every
    reference field as Dirichlet data."""
    u = np.asarray(u_ref, dtype=float)
    u = u[:, None] if u.ndim == 1 else u
    n = partition.mesh.n_nodes - 1
    on = np.zeros(n, dtype=bool)
    on[_pin(partition.skeleton)] = True
    values = sp.csc_matrix(u * on[:, None])
    return SimpleNamespace(family="skeleton", values=values, forcing=sp.csc_matrix((n, values.shape[1])),
                           block_restrict=None, labels=[("skeleton", j) for j in range(values.shape[1])],
                           dropped=[], count=values.shape[1])


def local_pca_family(partition, u_ref, rank=1, total=0, drop_tol=1e-10):
    """generate_bc_local_pca (basis.py:184-245): per block, the mean boundary
    trace followed by the principal directions of the centred traces,
    orthonormalised (QR), at most ``rank`` per block and ``total`` overall."""
    u = np.asarray(u_ref, dtype=float)
    u = u[:, None] if u.ndim == 1 else u
    ns = u.shape[1]
    if rank < 1:
        raise ValueError(f"rank must be >= 1, got {rank}")
    if rank > ns:
        raise ValueError(f"rank {rank} exceeds number of reference fields {ns}")
    n = partition.mesh.n_nodes - 1
    picked = []                                     # (block, component, weight, rows, vector)
    for j in range(partition.n_blocks):
        rows = _pin(partition.boundaries[j])
        tr = u[rows, :]
        mean = tr.mean(axis=1)
        Uc, sv, _ = sla.svd(tr - mean[:, None], full_matrices=False)
        mnorm = float(np.linalg.norm(mean))
        cand, wts = [], []
        if mnorm > 0:
            cand.append(mean / mnorm)
            wts.append(mnorm * np.sqrt(ns))
        for r in range(sv.size):
            cand.append(Uc[:, r])
            wts.append(float(sv[r]))
        if not cand:
            continue
        Qb, Rb = np.linalg.qr(np.column_stack(cand))
        top = max(wts)
        if top == 0.0:
            continue
        have = 0
        for r, wt in enumerate(wts):
            if have >= rank or wt < drop_tol * top:
                break
            if abs(Rb[r, r]) < 1e-10:
                continue
            picked.append((j, have, wt, rows, Qb[:, r].copy()))
            have += 1
    if total and len(picked) > total:
        rankd = np.argsort([-p[2] for p in picked], kind="stable")
        picked = [picked[i] for i in np.sort(rankd[:total])]
    cnt = len(picked)
    if cnt:
        rr = np.concatenate([p[3] for p in picked])
        cc = np.concatenate([np.full(p[3].size, c) for c, p in enumerate(picked)])
        vv = np.concatenate([p[4] for p in picked])
        values = sp.coo_matrix((vv, (rr, cc)), shape=(n, cnt)).tocsc()
    else:
        values = sp.csc_matrix((n, 0))
    return SimpleNamespace(family="local_pca", values=values, forcing=sp.csc_matrix((n, cnt)),
                           block_restrict=np.asarray([p[0] for p in picked], dtype=int),
                           labels=[("local_pca", p[0], p[1]) for p in picked], dropped=[], count=cnt)


def reference_fields(partition, m_ref, Q, engine=None):
    """Pinned fine-mesh fields of every source at the reference model
    (basis.py:141-149), solved on the device (fine.py: PCG to 1e-13 with the
    two-level MSFV preconditioner).  Returns a host array (n, n_sources)."""
    if engine is not None and hasattr(engine, "reference_fields"):
        return engine.reference_fields(m_ref, Q)
    from .fine import _DeviceSolve, _bind
    from .operators import assemble_operator
    op = assemble_operator(partition.mesh, np.asarray(m_ref, dtype=float))
    eng, _, w = _bind(op)
    Qd = np.asarray(sp.csc_matrix(Q).todense(), dtype=float)
    Qf = eng.zeros(eng.Nn, Qd.shape[1])
    Qf[1:] = eng.to_device(Qd)
    U = _DeviceSolve(eng, w, op).solve_dev(Qf)
    return U[1:].cpu().numpy()


# ------------------------------------------------------------ model-independent

class EnrichedLayout:
    """What the reference's BlockSystemCache holds for the extra columns
    (basis.py:421-492), uploaded once per builder: Dirichlet values V and
    forcing F as dense node fields, the block restriction, the edge-ownership
    mask of the restricted columns and the CSC pattern of their part of S."""

    def __init__(self, partition, engine, bc_sets, pieces):
        self.partition, self.engine = partition, engine
        extra = [s for s in sorted(bc_sets, key=lambda s: FAMILY_ORDER.index(s.family)) if s.family != "lagrange"]
        self.has_lagrange = any(s.family == "lagrange" for s in bc_sets)
        self.kL = partition.n_coarse_nodes if self.has_lagrange else 0
        n = partition.mesh.n_nodes - 1
        self.nE = int(sum(s.count for s in extra))
        if self.kL + self.nE == 0:
            raise ValueError("no basis columns: all bc sets are empty")
        if (n + 1) * self.nE * 8 > DENSE_FIELD_LIMIT:
            raise NotImplementedError(
                f"{self.nE} enriched columns on {n} nodes exceed the dense node-field budget of the GPU path")
        values = sp.hstack([s.values for s in extra], format="csc") if extra else sp.csc_matrix((n, 0))
        forcing = sp.hstack([s.forcing for s in extra], format="csc") if extra else sp.csc_matrix((n, 0))
        restrict = np.full(self.nE, -1, dtype=np.int64)
        off = 0
        for s in extra:
            if s.block_restrict is not None:
                restrict[off:off + s.count] = s.block_restrict
            off += s.count
        self.restrict = restrict
        self.families = np.concatenate([np.full(self.kL, "lagrange")] + [np.full(s.count, s.family) for s in extra])
        self.labels = ([("coarse_node", int(c)) for c in partition.coarse_nodes] if self.has_lagrange else []) + \
            [lab for s in extra for lab in s.labels]
        self.values, self.forcing = values, forcing

        # node and edge owners (basis.py:463-476)
        owner_n = np.full(n, -1, dtype=np.int64)
        for j, ids in enumerate(partition.interiors):
            owner_n[_pin(ids)] = j
        G = pieces[0].tocsr()
        ends = G.indices.reshape(-1, 2).astype(np.int64)             # full node ids of each edge
        eo = np.where(ends == 0, -1, owner_n[np.maximum(ends - 1, 0)])
        self.edge_owner = eo.max(axis=1)
        self.node_owner = owner_n

        # per block: supported columns, and the CSC pattern of S_E (basis.py:445-450, 574-594)
        vcsr, fcsr = values.tocsr(), forcing.tocsr()
        free = restrict < 0
        vcoo = values.tocoo()
        rows, cols = [vcoo.row.astype(np.int64)], [vcoo.col.astype(np.int64)]
        self.block_cols = []
        for j in range(partition.n_blocks):
            I, B = _pin(partition.interiors[j]), _pin(partition.boundaries[j])
            if I.size == 0:
                self.block_cols.append(np.empty(0, dtype=np.int64))
                continue
            touched = np.zeros(self.nE, dtype=bool)
            if vcsr.nnz and B.size:
                touched |= np.diff(vcsr[B].tocsc().indptr) > 0
            if fcsr.nnz:
                touched |= np.diff(fcsr[I].tocsc().indptr) > 0
            cj = np.flatnonzero((touched & free) | (restrict == j))
            self.block_cols.append(cj)
            if cj.size:
                rows.append(np.repeat(I, cj.size))
                cols.append(np.tile(cj, I.size))
        rows, cols = np.concatenate(rows), np.concatenate(cols)
        order = np.lexsort((rows, cols))
        rows, cols = rows[order], cols[order]
        if rows.size > 1 and np.any((np.diff(rows) == 0) & (np.diff(cols) == 0)):
            raise AssertionError("basis entries are not disjoint")
        self.s_rows = rows.astype(np.int32)
        self.s_indptr = np.searchsorted(cols, np.arange(self.nE + 1)).astype(np.int64)
        self._s_gather = None

        # device copies
        dev = engine.device
        Vd = np.zeros((n + 1, self.nE))
        Vd[1:] = values.toarray()
        Fd = np.zeros((n + 1, self.nE))
        Fd[1:] = forcing.toarray()
        self.V = engine.to_device(Vd)
        self.F = engine.to_device(Fd)
        self.pcols = np.flatnonzero(restrict >= 0)
        self.colmask = self.edge_keep = None
        if self.pcols.size:
            own = torch.from_numpy(np.concatenate([[-2], owner_n])).to(dev)
            rst = torch.from_numpy(np.where(restrict >= 0, restrict, -1)).to(dev)
            # restricted columns are solved in their own block only; free ones everywhere
            self.colmask = ((own[:, None] == rst[None, :]) | (rst[None, :] < 0)).to(torch.float64)
            eo_d = torch.from_numpy(self.edge_owner).to(dev)
            self.edge_keep = (eo_d[:, None] == rst[self.pcols][None, :]).to(torch.float64)   # (E, n_p)
            self.pcols_dev = torch.from_numpy(self.pcols).to(dev)

    def s_gather(self):
        if self._s_gather is None:
            dev = self.engine.device
            cols = np.repeat(np.arange(self.nE), np.diff(self.s_indptr))
            self._s_gather = (torch.from_numpy(self.s_rows.astype(np.int64) + 1).to(dev),
                              torch.from_numpy(cols).to(dev))
        return self._s_gather


# ------------------------------------------------------------------------ basis

class EnrichedBasis:
    """MultiscaleBasis surface (basis.py:301-376) for S = [S_L | E]."""

    def __init__(self, layout, lag, op, E):
        self.layout, self.lag, self.op, self.E = layout, lag, op, E
        self.partition, self.engine = layout.partition, layout.engine
        self.kL, self.nE = layout.kL, layout.nE
        self.factor, self.flags = lag.factor, lag.flags
        self.families, self.labels = layout.families, layout.labels
        self.cache = None
        self.bx = None
        self._S = self._EP = None
        self._m_dev = lag._m_dev

    k = property(lambda self: self.kL + self.nE)
    n = property(lambda self: self.engine.n)
    model = property(lambda self: self.lag.model)
    pieces = property(lambda self: self.op.pieces)
    Sint = property(lambda self: self.lag.Sint)
    Kloc = property(lambda self: self.lag.Kloc)

    def check_model(self, m):
        return self.lag.check_model(m)

    def raise_on_flags(self, f=None):
        return self.lag.raise_on_flags(f)

    def interior_solve(self, w, workers=1):
        return self.lag.interior_solve(w, workers=workers)

    # S x for coefficient matrices x (k, ncol): node fields (Nn, ncol)
    def prolong(self, X):
        eng = self.engine
        out = self.E @ X[self.kL:] if self.nE else None
        if self.kL:
            lagp = eng.prolong(self.Sint, X[:self.kL].contiguous())
            out = lagp if out is None else out + lagp
        return out

    # S^T X for node fields X (Nn, ncol): (k, ncol)
    def restrict(self, X):
        eng = self.engine
        parts = []
        if self.kL:
            parts.append(eng.restrict_op(self.Sint, None, X.contiguous(), None, None, X.shape[1]))
        if self.nE:
            parts.append(self.E.T @ X)
        return torch.cat(parts, dim=0)

    @property
    def S_extra(self):
        """The extra columns of S in the reference's CSC pattern."""
        lay = self.layout
        r, c = lay.s_gather()
        ev = self.E[r, c].cpu().numpy() if lay.nE else np.zeros(0)
        return sp.csc_matrix((ev, lay.s_rows, lay.s_indptr), shape=(self.n, lay.nE))

    @property
    def S(self):
        """The reference's CSC matrix (same indices/indptr, basis.py:574-594)."""
        if self._S is None:
            self._S = sp.hstack([self.lag.S, self.S_extra], format="csc") if self.kL else self.S_extra
        return self._S

    @property
    def edge_profiles(self):
        """G_p S with the restricted columns masked to their block's edges
        (basis.py:596-608); host, off the hot path."""
        if self._EP is None:
            prof = (self.op.grad[:, 1:] @ self.S).tocoo()
            rst = np.concatenate([np.full(self.kL, -1), self.layout.restrict])[prof.col]
            keep = (rst < 0) | (self.layout.edge_owner[prof.row] == rst)
            self._EP = sp.coo_matrix((prof.data[keep], (prof.row[keep], prof.col[keep])), shape=prof.shape).tocsc()
        return self._EP

    def grad_edge(self, v):
        return self.edge_profiles @ np.asarray(v, dtype=float)


def assemble_enriched(op, layout):
    """assemble_basis (basis.py:511-616) for Lagrange + extra columns."""
    from .basis import MultiscaleBasis
    eng, part = layout.engine, layout.partition
    _, m_dev, sigma, w = op.device_state(eng)
    factor, Sint, Kloc, fl = eng.basis(w, op.flags)          # block factors (+ the Lagrange columns)
    lag = MultiscaleBasis(part, eng, op, factor, Sint, Kloc, fl)
    if layout.nE:
        rhs = layout.F - eng.fine_apply(w, layout.V)          # rhs0 - A_IB xb on interior rows (basis.py:548)
        if layout.colmask is not None:
            rhs = rhs * layout.colmask
        Z = eng.zeros(eng.Nn, layout.nE)
        eng.interior_solve(factor, rhs.contiguous(), Z)
        E = layout.V + Z
    else:
        E = eng.zeros(eng.Nn, 0)
    return EnrichedBasis(layout, lag, op, E)


# ---------------------------------------------------------------------- forward

def _survey_dev(eng, survey):
    return eng.survey_device(survey) if hasattr(eng, "survey_device") else survey.device(eng)


def _host(t):
    return t.detach().cpu().numpy()


class EnrichedState:
    """ReducedState (forward.py:62-75) with the block-eliminated factorization."""

    def __init__(self, op, basis, survey):
        self.op, self.basis, self.survey = op, basis, survey
        self.shift = 0.0
        self.chol = None
        self._A_k = None
        eng, b = basis.engine, basis
        _, _, self.sigma, self.w = op.device_state(eng)
        self.AE = eng.fine_apply(self.w, b.E) if b.nE else None                        # A E
        self.A_EE = b.E.T @ self.AE if b.nE else None
        self.A_LE = (eng.restrict_op(b.Sint, None, self.AE, None, None, b.nE)
                     if (b.nE and b.kL) else None)                                      # S_L^T A E
        self._factor(0.0)

    def _trace(self):
        eng, b = self.basis.engine, self.basis
        tr = 0.0
        if b.kL:
            tr += float(eng.coarse_trace(eng.galerkin(b.Kloc, 0.0)).sum().item())
        if b.nE:
            tr += float(torch.diagonal(self.A_EE).sum().item())
        return tr

    def _try_factor(self, shift):
        eng, b = self.basis.engine, self.basis
        fl = eng.flags()
        self.Lk = self.Z = self.Lc = None
        if b.kL:
            self.Lk = eng.galerkin(b.Kloc, shift)
            eng.coarse_factor(self.Lk, fl)
            if int(fl.item()) & 8:
                return False
        if b.nE:
            Sc = self.A_EE.clone()
            if shift:
                Sc.diagonal().add_(shift)
            if b.kL:
                self.Z = self.A_LE.clone()
                eng.coarse_solve(self.Lk, self.Z)                                       # A_LL^-1 A_LE
                Sc = Sc - self.A_LE.T @ self.Z
            Sc = 0.5 * (Sc + Sc.T)
            Lc, info = torch.linalg.cholesky_ex(Sc)
            if int(info.item()) != 0:
                return False
            self.Lc = Lc
        return True

    def _factor(self, shift):
        """cho_factor with the diagonal-shift fallback (forward.py:119-131)."""
        from .basis import raise_status
        raise_status(int(self.op.flags.item()) & 7)
        if self._try_factor(0.0):
            return
        k = self.basis.k
        self.shift = 1e-12 * self._trace() / k
        if not self._try_factor(self.shift):
            raise ReducedSingularError("projected operator is singular even after diagonal shift")

    def solve_dev(self, B):
        """A_k^-1 B for B (k, ncol) on the device."""
        eng, b = self.basis.engine, self.basis
        kL = b.kL
        if not b.nE:
            X = B.clone().contiguous()
            return eng.coarse_solve(self.Lk, X)
        bE = B[kL:]
        if not kL:
            return torch.cholesky_solve(bE, self.Lc)
        t = B[:kL].clone().contiguous()
        eng.coarse_solve(self.Lk, t)
        xE = torch.cholesky_solve(bE - self.A_LE.T @ t, self.Lc)
        return torch.cat([t - self.Z @ xE, xE], dim=0)

    def solve_reduced(self, B):
        B = np.asarray(B, dtype=float)
        single = B.ndim == 1
        X = self.basis.engine.to_device(B[:, None] if single else B)
        out = _host(self.solve_dev(X))
        return out[:, 0] if single else out

    @property
    def T(self):
        return _host(self.T_dev)

    @property
    def A_k(self):
        """Dense unshifted S^T A S (forward.py:102)."""
        if self._A_k is None:
            eng, b = self.basis.engine, self.basis
            blocks = []
            if b.kL:
                ALL = eng.coarse_dense(b.Kloc, 0.0)
                blocks.append(torch.cat([ALL, self.A_LE], dim=1) if b.nE else ALL)
            if b.nE:
                blocks.append(torch.cat([self.A_LE.T, self.A_EE], dim=1) if b.kL else self.A_EE)
            self._A_k = _host(torch.cat(blocks, dim=0))
        return self._A_k

    def check(self, host_flags=None):
        return None


def forward_enriched_dev(op, survey, basis):
    """forward_reduced (forward.py:105-144) for an enriched basis; device D."""
    eng = basis.engine
    state = EnrichedState(op, basis, survey)
    Pp, Qp, Qf = _survey_dev(eng, survey)
    ns = survey.n_sources
    parts = []
    if basis.kL:
        parts.append(eng.restrict_points(Qp, basis.Sint, None, ns))                     # S_L^T Q
    if basis.nE:
        parts.append(basis.E.T @ Qf)                                                    # E^T Q
    F = torch.cat(parts, dim=0)                                                         # forward.py:115
    T = state.solve_dev(F)                                                              # forward.py:142
    state.T_dev = T
    xf = basis.E @ T[basis.kL:] if basis.nE else None
    if basis.kL:
        D = eng.receive(Pp, basis.Sint, Y=T[:basis.kL].contiguous(), Xfield=xf)         # P^T S T (forward.py:143)
    else:
        D = eng.receive(Pp, None, Xfield=xf, nrhs=ns)
    state.D_dev = D
    return D, state


def forward_enriched(op, survey, basis):
    D, state = forward_enriched_dev(op, survey, basis)
    return _host(D), state


# ------------------------------------------------------------------ sensitivity

class EnrichedSensitivity:
    """AdaptiveSensitivity (forward.py:209-281) for S = [S_L | E], edge space."""

    mode = "ms_adaptive"

    def __init__(self, state, survey, workers=1):
        op, b = state.op, state.basis
        eng = b.engine
        if not _same_model(op, b):
            b.check_model(op.m)
        self.state, self.survey, self.basis, self.engine = state, survey, b, eng
        self.sigma, self.w = state.sigma, state.w
        self.Pp, self.Qp, self.Qf = _survey_dev(eng, survey)
        ns = survey.n_sources
        T = state.T_dev
        lay = b.layout
        self.U = b.prolong(T)                                                          # S T (forward.py:241)
        self.gu = eng.edge_grad(self.U)                                                # G_p S T (forward.py:245)
        self.Delta = None
        self.gprof = self.gu
        if lay.pcols.size:
            GEp = eng.edge_grad(b.E[:, lay.pcols_dev].contiguous())
            self.Delta = GEp * (1.0 - lay.edge_keep)                                   # masked-out profiles
            self.prow = lay.pcols_dev + b.kL                                           # their rows of T / y
            self.gprof = self.gu - self.Delta @ T[self.prow]                           # EP T (forward.py:244)
        R = self.Qf - eng.fine_apply(self.w, self.U)                                   # Q - A S T (forward.py:243)
        ZR = eng.zeros(eng.Nn, ns)
        eng.interior_solve(b.factor, R.contiguous(), ZR)
        self.a = eng.edge_grad(ZR)                                                     # forward.py:246

    def _EP(self, v, sv=None):
        """EP v for coefficients v (k, ns): edge fields."""
        sv = self.basis.prolong(v) if sv is None else sv
        out = self.engine.edge_grad(sv)
        if self.Delta is not None:
            out = out - self.Delta @ v[self.prow]
        return out

    def _EPt(self, f):
        """EP^T f for edge fields f (E, ns): (k, ns)."""
        out = self.basis.restrict(self.engine.edge_div(f))
        if self.Delta is not None:
            out[self.prow] -= self.Delta.T @ f
        return out

    def rapply_dev(self, W):
        eng, b = self.engine, self.basis
        ns = self.survey.n_sources
        W = eng.to_device(W)
        p = eng.scatter_points(self.Pp, W, ns)                                         # P W (forward.py:275)
        y = self.state.solve_dev(b.restrict(p))                                        # forward.py:276
        sy = b.prolong(y)                                                              # forward.py:277
        r = p - eng.fine_apply(self.w, sy)
        z = eng.zeros(eng.Nn, ns)
        eng.interior_solve(b.factor, r.contiguous(), z)                                # _Yt_w (forward.py:254-256)
        gsy = eng.edge_grad(sy)
        epy = gsy if self.Delta is None else gsy - self.Delta @ y[self.prow]
        xi = (self.gprof * eng.edge_grad(z) + self.a * epy + self.gu * gsy).sum(dim=1)  # forward.py:278-280
        return eng.cell_gather(self.sigma, xi)

    def apply_dev(self, dm):
        eng, b = self.engine, self.basis
        ns = self.survey.n_sources
        dm = eng.to_device(dm).reshape(-1)
        c = eng.edge_average(self.sigma, dm)[:, None]                                  # Csig dm (forward.py:259)
        rhs_y = eng.edge_div((self.gprof * c).contiguous())
        ydm = eng.zeros(eng.Nn, ns)
        eng.interior_solve(b.factor, rhs_y, ydm)
        ydm = -ydm                                                                     # _Y_dm (forward.py:250-252)
        xdm = -self._EPt((self.a * c).contiguous())                                    # forward.py:264
        gdm = eng.edge_div((self.gu * c).contiguous())                                 # forward.py:265
        rhs = xdm - b.restrict(gdm + eng.fine_apply(self.w, ydm))                      # forward.py:266
        dt = self.state.solve_dev(rhs)                                                 # forward.py:267
        field = ydm + (b.E @ dt[b.kL:] if b.nE else 0.0)
        if b.kL:
            return eng.receive(self.Pp, b.Sint, Y=dt[:b.kL].contiguous(), Xfield=field.contiguous())
        return eng.receive(self.Pp, None, Xfield=field.contiguous(), nrhs=ns)          # forward.py:268

    def apply(self, dm):
        return _host(self.apply_dev(dm))

    def rapply(self, W):
        return _host(self.rapply_dev(np.asarray(W, dtype=float) if not hasattr(W, "detach") else W))


def _same_model(op, basis):
    return op._dev is not None and op._dev[1] is basis._m_dev
