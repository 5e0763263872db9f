"""A numpy stand-in for ``paper_1707_07598_b200.engine.Engine`` (test
infrastructure): every device primitive the enriched-family host logic
(enriched.py) calls, restated with the CPU oracle's matrices.  It lets the
``-m "not gpu"`` suite run that host logic -- block elimination of the
bordered coarse system, the masked edge profiles, the edge-space sensitivity
-- against the reference goldens without a GPU.  Never imported by the
product."""

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import torch

from oracle import msfv_oracle as orc

F64 = torch.float64


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))


def _pad(a):
    a = np.asarray(a, dtype=float)
    return np.concatenate([np.zeros((1,) + a.shape[1:]), a], axis=0)


class _Points:
    def __init__(self, M):
        self.M = sp.csc_matrix(M)
        self.ncol = self.M.shape[1]


class NumpyEngine:
    def __init__(self, cells, h, blocks):
        self.mesh = orc.Mesh(*cells, *h)
        self.part = orc.make_partition(self.mesh, *blocks)
        self.G = orc.gradient_matrix(self.mesh)
        self.C = orc.cell_average_matrix(self.mesh)
        self.Gp = self.G[:, 1:].tocsr()
        self.Nn = self.mesh.n_nodes
        self.n = self.Nn - 1
        self.E = self.G.shape[0]
        self.Nm = self.mesh.n_cells
        self.k = self.part.n_coarse
        self.nbl = self.part.n_blocks
        self.device = torch.device("cpu")
        self.cache = orc.build_cache(self.part, self.G, self.C)

    # buffers
    def zeros(self, *shape):
        return torch.zeros(shape, dtype=F64)

    def empty(self, *shape):
        return torch.zeros(shape, dtype=F64)

    def flags(self):
        return torch.zeros(1, dtype=torch.int32)

    def to_device(self, a, n=None):
        return (a.to(F64) if isinstance(a, torch.Tensor) else _t(a)).contiguous()

    # operator / basis
    def operator_state(self, m):
        op = orc.assemble(self.mesh, m, pieces=(self.G, self.C))
        return op

    def A_of(self, w):
        w = w.numpy()
        return (self.Gp.T @ sp.diags(w) @ self.Gp).tocsr()

    def basis(self, w, fl=None):
        op = self._op
        basis = orc.build_basis(op, self.part, cache=self.cache)
        fl = fl if fl is not None else self.flags()
        return basis, basis.S, ("Kloc", basis), fl      # factor, Sint, Kloc stand-ins

    def fine_apply(self, w, X, out=None):
        return _t(_pad(self.A_of(w) @ X.numpy()[1:]))

    def interior_solve(self, factor, rhs, out=None):
        sol = _t(_pad(factor.interior_solve(rhs.numpy()[1:])))
        o = out if out is not None else rhs
        o.copy_(sol)
        return o

    def restrict_op(self, Sint, w1, X1, w2, X2, nrhs, scale=1.0):
        assert w1 is None and X2 is None
        return _t(scale * (Sint.T @ X1.numpy()[1:]))

    def prolong(self, Sint, Y):
        return _t(_pad(Sint @ Y.numpy()))

    def galerkin(self, Kloc, shift=0.0, out=None):
        b = Kloc[1]
        A = (b.S.T @ (self._op.A @ b.S)).toarray()
        return {"A": A + shift * np.eye(A.shape[0])}

    def coarse_dense(self, Kloc, shift=0.0):
        return _t(self.galerkin(Kloc, shift)["A"])

    def coarse_trace(self, Ak):
        return _t(np.diag(Ak["A"]))

    def coarse_factor(self, Ak, fl):
        try:
            Ak["chol"] = sla.cho_factor(Ak["A"], lower=True)
        except sla.LinAlgError:
            fl |= 8

    def coarse_solve(self, Lk, X):
        X.copy_(_t(sla.cho_solve(Lk["chol"], X.numpy())))
        return X

    # survey
    def survey_device(self, survey):
        Qf = _t(_pad(np.asarray(survey.Q.todense())))
        return _Points(survey.P), _Points(survey.Q), Qf

    def scatter_points(self, pts, Z=None, nrhs=None, field=None):
        M = pts.M
        return _t(_pad(M @ Z.numpy() if Z is not None else np.asarray(M.todense())))

    def restrict_points(self, pts, Sint, Z=None, nrhs=None):
        M = pts.M if Z is None else pts.M @ Z.numpy()
        M = np.asarray(M.todense()) if sp.issparse(M) else M
        return _t(Sint.T @ M)

    def receive(self, pts, Sint, Y=None, Xfield=None, nrhs=None):
        f = 0.0
        if Y is not None:
            f = f + Sint @ Y.numpy()
        if Xfield is not None:
            f = f + Xfield.numpy()[1:]
        return _t(pts.M.T @ f)

    # edge space
    def edge_grad(self, X):
        return _t(self.Gp @ X.numpy()[1:])

    def edge_div(self, F):
        return _t(_pad(self.Gp.T @ F.numpy()))

    def edge_average(self, sigma, dm):
        return _t(self.C @ (sigma.numpy() * dm.numpy()))

    def cell_gather(self, sigma, xi):
        return _t(-sigma.numpy() * (self.C.T @ xi.numpy()))

    # reference fields (basis.py:141-149), SuperLU like the reference
    def reference_fields(self, m_ref, Q):
        import scipy.sparse.linalg as spla
        op = orc.assemble(self.mesh, np.asarray(m_ref, dtype=float), pieces=(self.G, self.C))
        return spla.splu(sp.csc_matrix(op.A)).solve(np.asarray(sp.csc_matrix(Q).todense(), dtype=float))


class NumpyOperator:
    """DiffusionOperator stand-in bound to a NumpyEngine."""

    def __init__(self, engine, m):
        self.engine = engine
        self.mesh = engine.mesh
        self.m = np.asarray(m, dtype=float)
        self._o = engine.operator_state(self.m)
        engine._op = self._o
        self.flags = engine.flags()
        self._dev = (engine, _t(self.m), _t(self._o.sigma), _t(self._o.w))
        self.pieces = (engine.G, engine.C)
        self.grad = engine.G

    def device_state(self, engine):
        return self._dev
