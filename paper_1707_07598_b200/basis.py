"""Model-adapted Lagrange multiscale basis built on the GPU.

Drop-in for the Lagrange family of the reference's basis.py.  The per-block
interior problems (basis.py:511-563) are factored and solved by ``k_basis``
(one CTA per coarse block, banded Cholesky in shared memory); the basis is
kept on the device in block layout (``Sint[block][corner][interior]`` plus
analytic skeleton hats).  ``MultiscaleBasis.S`` materialises the reference's
CSC matrix (same indices/indptr, basis.py:574-594) on demand.
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .engine import engine_for
from .errors import FactorizationError, InvalidModelError, StaleBasisError
from .operators import edge_cell_map, nodal_gradient

FAMILIES = ("lagrange", "source", "skeleton", "local_pca")


def raise_status(f):
    """Map device status bits onto the reference exception types."""
    if f & 1:
        raise InvalidModelError("model vector contains non-finite entries")
    if f & 2:
        raise InvalidModelError("conductivity must be positive")
    if f & 4:
        raise FactorizationError("local interior operator is not positive definite")


@dataclass(frozen=True)
class BasisSpec:
    """Boundary-condition families (basis.py:37-53): ``lagrange`` takes the
    block-layout path (basis.py / forward.py here), the enriched families
    (``source``, ``skeleton``, ``local_pca``) take enriched.py."""

    families: tuple = ("lagrange",)
    pca_rank: int = 0
    pca_total: int = 0
    pca_drop_tol: float = 1e-10
    # extension: "hats" = the reference's trilinear skeleton
    # data (basis.py:84-116); "reduced" = 1D line / 2D face problems with the
    # model's edge weights (msfv_reduced.cu; sensitivities: reduced_sens.py)
    boundary: str = "hats"

    def __post_init__(self):
        unknown = set(self.families) - set(FAMILIES)
        if unknown:
            raise ValueError(f"unknown basis families: {sorted(unknown)}")
        if not self.families:
            raise ValueError("at least one basis family must be enabled")
        if "local_pca" in self.families and self.pca_rank < 1:
            raise ValueError("local_pca requires pca_rank >= 1")
        if self.boundary not in ("hats", "reduced"):
            raise ValueError(f"unknown boundary condition kind {self.boundary!r}")


def coarse_hat_values(partition, coarse_node, node_ids):
    """Trilinear hat of a coarse node at full-space node ids (basis.py:84-92)."""
    mesh = partition.mesh
    ci, cj, ck = mesh.node_triple(coarse_node)
    i, j, k = mesh.node_triple(np.asarray(node_ids))
    w = np.ones(np.atleast_1d(i).shape, dtype=float)
    for x, c, b in ((i, ci, partition.b1), (j, cj, partition.b2), (k, ck, partition.b3)):
        w = w * np.maximum(0.0, 1.0 - np.abs(np.asarray(x, dtype=float) - c) / b)
    return w


def _skeleton_hat_entries(partition):
    """(pinned row, coarse column, hat value) of every nonzero skeleton hat
    entry -- the ``values`` block of generate_bc_lagrange (basis.py:95-116)."""
    mesh = partition.mesh
    b = (partition.b1, partition.b2, partition.b3)
    nbp = (partition.nb[0] + 1, partition.nb[1] + 1, partition.nb[2] + 1)
    skel = partition.skeleton[partition.skeleton != 0]
    ijk = mesh.node_triple(skel)
    # per axis: candidate coarse coordinates floor(x/b) and floor(x/b)+1
    cand, fac = [], []
    for ax in range(3):
        x = ijk[ax]
        c0 = x // b[ax]
        opts = []
        for c in (c0, c0 + 1):
            f = np.maximum(0.0, 1.0 - np.abs(x.astype(float) - c * b[ax]) / b[ax])
            f = np.where(c < nbp[ax], f, 0.0)
            opts.append((np.minimum(c, nbp[ax] - 1), f))
        cand.append(opts)
    rows, cols, vals = [], [], []
    for oz in range(2):
        for oy in range(2):
            for ox in range(2):
                w = np.ones(skel.size)
                w = w * cand[0][ox][1]
                w = w * cand[1][oy][1]
                w = w * cand[2][oz][1]
                col = cand[0][ox][0] + nbp[0] * (cand[1][oy][0] + nbp[1] * cand[2][oz][0])
                nz = np.flatnonzero(w)
                rows.append(skel[nz] - 1)
                cols.append(col[nz])
                vals.append(w[nz])
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def generate_bc_lagrange(partition):
    """Lagrange boundary data as a scipy CSC (basis.py:95-116), host side."""
    from types import SimpleNamespace
    n = partition.mesh.n_nodes - 1
    r, c, v = _skeleton_hat_entries(partition)
    values = sp.csc_matrix((v, (r, c)), shape=(n, partition.n_coarse_nodes))
    forcing = sp.csc_matrix((n, partition.n_coarse_nodes))
    return SimpleNamespace(family="lagrange", values=values, forcing=forcing, block_restrict=None,
                           labels=[("coarse_node", int(cn)) for cn in partition.coarse_nodes], dropped=[],
                           count=partition.n_coarse_nodes)


def csc_pattern(partition):
    """Model-independent CSC pattern of S and the gather map from the device
    block layout into it (basis.py:574-594), host side.

    Returns (indices, indptr, src, hatv): src[t] >= 0 indexes the device
    array Sint[block][corner][interior]; src[t] == -1 marks a skeleton entry
    whose value is the hat hatv[t] (bit-exact with the reference)."""
    n = partition.mesh.n_nodes - 1
    k = partition.n_coarse_nodes
    r_s, c_s, v_s = _skeleton_hat_entries(partition)
    nI = (partition.b1 - 1) * (partition.b2 - 1) * (partition.b3 - 1)
    rows, cols = [r_s], [c_s]
    src = [np.full(r_s.size, -1, dtype=np.int64)]
    hv = [v_s]
    if nI > 0:
        nb1, nb2, _ = partition.nb
        inter = np.stack(partition.interiors) - 1             # [block, a] pinned ids
        nbl = inter.shape[0]
        blk = np.arange(nbl)
        bi, bj, bk = blk % nb1, (blk // nb1) % nb2, blk // (nb1 * nb2)
        for cc in range(8):
            col = (bi + (cc & 1)) + (nb1 + 1) * ((bj + ((cc >> 1) & 1)) + (nb2 + 1) * (bk + ((cc >> 2) & 1)))
            rows.append(inter.ravel())
            cols.append(np.repeat(col, nI))
            src.append(((blk[:, None] * 8 + cc) * nI + np.arange(nI)[None, :]).ravel())
            hv.append(np.zeros(nbl * nI))
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    src, hv = np.concatenate(src), np.concatenate(hv)
    order = np.argsort(cols.astype(np.int64) * n + rows, kind="stable")
    indices = rows[order].astype(np.int32)
    indptr = np.searchsorted(cols[order], np.arange(k + 1)).astype(np.int32)
    return indices, indptr, src[order], hv[order]


def box_sources(partition, indices, indptr, src):
    """For the skeleton entries (src < 0) of the CSC pattern: flat index into
    the reduced-boundary box table bx[block][corner][(b1+1)(b2+1)(b3+1)] of a
    block having the entry's coarse node as a corner (msfv_reduced.cu)."""
    mesh = partition.mesh
    b = (partition.b1, partition.b2, partition.b3)
    nb = partition.nb
    k = partition.n_coarse_nodes
    cols = np.repeat(np.arange(k), np.diff(indptr))
    node = indices.astype(np.int64) + 1
    ijk = mesh.node_triple(node)
    nbp = (nb[0] + 1, nb[1] + 1)
    cijk = (cols % nbp[0], (cols // nbp[0]) % nbp[1], cols // (nbp[0] * nbp[1]))
    blk, loc, bit = [], [], []
    for ax in range(3):
        x, c = ijk[ax], cijk[ax]
        lower = (x < c * b[ax]) | ((x == c * b[ax]) & (c == nb[ax]))
        bi = np.where(lower, c - 1, c)
        blk.append(bi)
        loc.append(x - bi * b[ax])
        bit.append(lower.astype(np.int64))
    jb = blk[0] + nb[0] * (blk[1] + nb[1] * blk[2])
    cc = bit[0] + 2 * bit[1] + 4 * bit[2]
    nbox = (b[0] + 1) * (b[1] + 1) * (b[2] + 1)
    flat = (jb * 8 + cc) * nbox + loc[0] + (b[0] + 1) * (loc[1] + (b[1] + 1) * loc[2])
    return np.where(src < 0, flat, -1).astype(np.int64)


class _CscTemplate:
    """csc_pattern uploaded for one engine."""

    def __init__(self, partition, engine):
        import torch
        self.indices, self.indptr, src, hv = csc_pattern(partition)
        self.shape = (partition.mesh.n_nodes - 1, partition.n_coarse_nodes)
        self.src = torch.from_numpy(src).to(engine.device)
        self.hatv = torch.from_numpy(hv).to(engine.device)
        self.bsrc = None
        if engine.reduced:
            self.bsrc = torch.from_numpy(box_sources(partition, self.indices, self.indptr, src)).to(engine.device)


class MultiscaleBasis:
    """Assembled basis on the device (basis.py:301-376 surface)."""

    def __init__(self, partition, engine, op, factor, Sint, Kloc, flags):
        self.partition = partition
        self.engine = engine
        self.op = op
        self._model = None
        self._m_dev = op._dev[1]
        self.factor, self._Sint, self.Kloc, self.flags = factor, Sint, Kloc, flags
        self._sint_event = None          # set when the backward sweeps run on the side stream
        self._bwd_pending = False        # split build: backward sweeps not launched yet
        self._families = None
        self._labels = None
        self.cache = None
        self._S = None
        self._EP = None
        self._checked = False
        self.bx = None                   # reduced-boundary box table (spec.boundary == "reduced")

    def start_backward(self):
        """Launch the deferred backward sweeps (split build) on the side stream,
        ordered after everything already queued on the current stream."""
        if not self._bwd_pending:
            return
        import torch
        eng = self.engine
        self._bwd_pending = False
        main, side = torch.cuda.current_stream(), eng.side_stream
        ready = torch.cuda.Event()
        ready.record(main)
        side.wait_event(ready)
        with torch.cuda.stream(side):
            eng.basis_backward(self.factor, self._Sint)
        self.factor.record_stream(side)
        self._Sint.record_stream(side)
        done = torch.cuda.Event()
        done.record(side)
        self._sint_event = done

    @property
    def Sint(self):
        """Interior basis values; orders the current stream after the backward
        sweeps (split build)."""
        if self._bwd_pending:
            self.start_backward()
        if self._sint_event is not None:
            import torch
            torch.cuda.current_stream().wait_event(self._sint_event)
        return self._Sint

    def sint_for(self, pts):
        """Sint for a survey-point kernel: the backward sweeps are awaited only
        when the point set has interior nodes (skeleton values are hats)."""
        return self.Sint if pts.interior_blocks else self._Sint

    @property
    def families(self):
        if self._families is None:
            self._families = np.full(self.partition.n_coarse_nodes, "lagrange")
        return self._families

    @property
    def labels(self):
        if self._labels is None:
            self._labels = [("coarse_node", int(cn)) for cn in self.partition.coarse_nodes]
        return self._labels

    @property
    def model(self):
        if self._model is None:
            self._model = self._m_dev.cpu().numpy()
        return self._model

    @property
    def k(self):
        return self.engine.k

    @property
    def n(self):
        return self.engine.n

    def raise_on_flags(self, f=None):
        if f is None:
            f = int(self.flags.item())
        raise_status(f & 7)
        self._checked = True

    def check_model(self, m):
        """Bitwise model check (basis.py:333-337)."""
        if hasattr(m, "detach"):
            import torch
            mt = m.detach().to(self._m_dev.device, torch.float64).reshape(-1)
            same = mt.shape == self._m_dev.shape and bool(torch.equal(mt, self._m_dev))
        else:
            same = np.array_equal(self.model, np.asarray(m, dtype=float))
        if not same:
            raise StaleBasisError("basis was built at a different model; rebuild before applying")

    @property
    def S(self):
        if self._S is None:
            tpl = _template(self.partition, self.engine)
            if self.bx is not None:
                self.engine.bind_boundary(self.bx)
                vals = self.engine.basis_csc_box(self.Sint, tpl.src, tpl.bsrc, self.bx).cpu().numpy()
            else:
                vals = self.engine.basis_csc(self.Sint, tpl.src, tpl.hatv).cpu().numpy()
            self._S = sp.csc_matrix((vals, tpl.indices, tpl.indptr), shape=tpl.shape)
        return self._S

    @property
    def pieces(self):
        return self.op.pieces

    @property
    def edge_profiles(self):
        if self._EP is None:
            self._EP = (self.op.grad[:, 1:] @ self.S).tocsc()
        return self._EP

    def grad_edge(self, v):
        return self.edge_profiles @ np.asarray(v, dtype=float)

    def interior_solve(self, w, workers=1):
        """blockdiag(A_II^-1) on interiors, zero on the skeleton (basis.py:339-353)."""
        w = np.asarray(w, dtype=float)
        single = w.ndim == 1
        W = w[:, None] if single else w
        eng = self.engine
        F = eng.zeros(eng.Nn, W.shape[1])
        F[1:] = eng.to_device(W)
        out = eng.zeros(eng.Nn, W.shape[1])
        eng.interior_solve(self.factor, F, out)
        res = out[1:].cpu().numpy()
        return res[:, 0] if single else res


_TEMPLATES = {}


def _template(partition, engine):
    # keyed by what the template depends on (geometry, boundary kind, device), not by id(engine):
    # ids are reused after garbage collection
    m = partition.mesh
    key = (m.n1, m.n2, m.n3, partition.b1, partition.b2, partition.b3, bool(engine.reduced), str(engine.device))
    t = _TEMPLATES.get(key)
    if t is None:
        t = _CscTemplate(partition, engine)
        _TEMPLATES[key] = t
    return t


def _check_families(spec):
    """Lagrange alone takes the block-layout path; the enriched families
    (source, skeleton, local_pca) take enriched.py; both need the hat
    boundary data (the reduced boundary problems are Lagrange-only)."""
    if tuple(spec.families) != ("lagrange",) and spec.boundary != "hats":
        raise NotImplementedError("reduced boundary conditions are built for the Lagrange family only")


def assemble_basis(op, partition, bc_sets=None, workers=1, cache=None, spec=None):
    """Build the Lagrange basis at the operator's model (basis.py:511-616).
    ``spec.boundary == "reduced"``: skeleton data from the reduced 1D/2D
    problems at this model instead of the hats (extension)."""
    if bc_sets is not None:
        fams = [getattr(s, "family", "lagrange") for s in bc_sets]
        if fams != ["lagrange"]:
            raise NotImplementedError("the GPU path builds the Lagrange family only")
    if spec is not None and spec.boundary == "reduced":
        eng = engine_for(partition, reduced=True)
        _, m_dev, sigma, w = op.device_state(eng)
        bx = eng.boundary_reduced(w, op.flags)
        eng.bind_boundary(bx)
        factor, Sint, Kloc, fl = eng.basis(w, op.flags)
        basis = MultiscaleBasis(partition, eng, op, factor, Sint, Kloc, fl)
        basis.bx = bx
        return basis
    eng = engine_for(partition)
    _, m_dev, sigma, w = op.device_state(eng)
    if eng.tensor_core:
        # forward part (factor, forward sweep, Galerkin) now; the backward
        # sweeps that complete S_I are deferred to start_backward(), which the
        # forward chain calls after the coarse factorization so they overlap
        # the latency-bound coarse sweeps on the engine's side stream
        factor, Sint, Kloc, fl = eng.basis_forward(w, op.flags)
        basis = MultiscaleBasis(partition, eng, op, factor, Sint, Kloc, fl)
        basis._bwd_pending = True
        return basis
    factor, Sint, Kloc, fl = eng.basis(w, op.flags)
    return MultiscaleBasis(partition, eng, op, factor, Sint, Kloc, fl)


class BasisBuilder:
    """Re-assembles the basis at any model (basis.py:619-660).  The
    boundary-condition data of every family is generated once (reference
    fields for ``skeleton`` / ``local_pca`` come from a device fine solve at
    ``m_ref``) and never depends on the current model."""

    def __init__(self, partition, spec=None, Q=None, m_ref=None, workers=1):
        spec = spec if spec is not None else BasisSpec()
        _check_families(spec)
        self.partition = partition
        self.spec = spec
        self.default_workers = workers
        self._pieces = None
        self._bc_sets = None
        self._layout = None
        self.enriched = tuple(spec.families) != ("lagrange",)
        if self.enriched:
            fams = set(spec.families)
            if {"skeleton", "local_pca"} & fams and (Q is None or m_ref is None):
                raise ValueError("skeleton/local_pca families need Q and m_ref")
            if "source" in fams and Q is None:
                raise ValueError("source family needs Q")
            self._Q, self._m_ref = Q, m_ref

    @property
    def pieces(self):
        if self._pieces is None:
            self._pieces = (nodal_gradient(self.partition.mesh), edge_cell_map(self.partition.mesh))
        return self._pieces

    def _engine(self):
        return engine_for(self.partition)

    @property
    def bc_sets(self):
        if self._bc_sets is None:
            if not self.enriched:
                self._bc_sets = [generate_bc_lagrange(self.partition)]
            else:
                from . import enriched as en
                fams, spec, part = set(self.spec.families), self.spec, self.partition
                u_ref = None
                if {"skeleton", "local_pca"} & fams:
                    u_ref = en.reference_fields(part, self._m_ref, self._Q, engine=self._engine())
                sets = []
                for fam in FAMILIES:                       # canonical order (basis.py:638-652)
                    if fam not in fams:
                        continue
                    if fam == "lagrange":
                        sets.append(generate_bc_lagrange(part))
                    elif fam == "source":
                        sets.append(en.source_family(part, self._Q))
                    elif fam == "skeleton":
                        sets.append(en.skeleton_family(part, u_ref))
                    else:
                        sets.append(en.local_pca_family(part, u_ref, rank=spec.pca_rank, total=spec.pca_total,
                                                        drop_tol=spec.pca_drop_tol))
                self._bc_sets = sets
        return self._bc_sets

    def assemble(self, op, workers=None):
        if not self.enriched:
            return assemble_basis(op, self.partition, workers=workers, spec=self.spec)
        from . import enriched as en
        if self._layout is None:
            self._layout = en.EnrichedLayout(self.partition, self._engine(), self.bc_sets, op.pieces)
        if self._layout.nE == 0 and self._layout.has_lagrange:
            return assemble_basis(op, self.partition, workers=workers, spec=self.spec)   # every extra column dropped
        return en.assemble_enriched(op, self._layout)
