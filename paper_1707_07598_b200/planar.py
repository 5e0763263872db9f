"""2D adaptive MSFV path (BASELINE.json configs 1-2) on the msfv2d_* C-ABI.

The reference package is 3D only, so there is no reference 2D
API to mirror literally; this module keeps the reference's Problem protocol
(``mode``, ``simulate(m) -> (D, state)``, ``jacobian(state)`` with
``apply``/``rapply``, inversion.py:196-230) and its algebra with d = 2
(SURVEY.md 8(c)):

  * mesh / partition: mesh.py:12-75, 143-182 with two axes (x fastest);
  * operator: A = G^T diag(C sigma) G, x- then y-edges, C = V/2 per touching
    cell, node 0 pinned (operators.py:36-141);
  * bilinear Lagrange basis: per-block band Cholesky + 4 solves
    (basis.py:84-116, 511-616);
  * forward_reduced: F = S^T Q, A_k = S^T A S (shift fallback), T = A_k^-1 F,
    D = P^T S T (forward.py:105-144);
  * sensitivity: the AdaptiveSensitivity products (forward.py:224-281).

Everything runs in libmsfv.so on the current CUDA stream; there is no CPU
fallback.  ``ReducedState2D``, ``Sensitivity2D`` keep their device tensors.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .engine import ptr, require_cuda, stream
from .errors import FactorizationError, ReducedSingularError
from .forward import Survey

F64 = torch.float64
INFO_NN, INFO_N, INFO_NCELLS, INFO_NEDGES, INFO_NBLOCKS, INFO_NI, INFO_K, INFO_FACTOR, INFO_BAND = range(9)


@dataclass(frozen=True)
class Mesh2D:
    """Uniform 2D tensor mesh, x-fastest numbering (mesh.py:12-75 with two axes)."""

    n1: int
    n2: int
    h1: float = 1.0
    h2: float = 1.0

    @property
    def dim(self):
        return 2

    @property
    def n_cells(self):
        return self.n1 * self.n2

    @property
    def n_nodes(self):
        return (self.n1 + 1) * (self.n2 + 1)

    @property
    def n_edges(self):
        return self.n1 * (self.n2 + 1) + (self.n1 + 1) * self.n2

    @property
    def volume(self):
        return self.h1 * self.h2

    def node_index(self, i, j):
        return np.asarray(i) + (self.n1 + 1) * np.asarray(j)

    def cell_index(self, i, j):
        return np.asarray(i) + self.n1 * np.asarray(j)


@dataclass(frozen=True)
class Partition2D:
    mesh: Mesh2D
    b1: int
    b2: int

    @property
    def nb(self):
        return (self.mesh.n1 // self.b1, self.mesh.n2 // self.b2)

    @property
    def n_blocks(self):
        return self.nb[0] * self.nb[1]

    @property
    def n_coarse(self):
        return (self.nb[0] + 1) * (self.nb[1] + 1)


def create_mesh_2d(n1, n2, h1=None, h2=None):
    if n1 < 1 or n2 < 1:
        raise ValueError("cell counts must be positive")
    return Mesh2D(int(n1), int(n2), 1.0 / n1 if h1 is None else float(h1), 1.0 / n2 if h2 is None else float(h2))


def create_partition_2d(mesh, b1, b2):
    """create_partition (mesh.py:143-182) with two axes; blocks need >= 2 cells."""
    if b1 < 2 or b2 < 2 or mesh.n1 % b1 or mesh.n2 % b2:
        raise ValueError("block size must divide the cell count (and be >= 2)")
    return Partition2D(mesh, int(b1), int(b2))


class Engine2D:
    """One msfv2d_plan per partition; typed wrappers on the current stream."""

    _cache = {}

    def __init__(self, part):
        require_cuda()
        self.L = _lib.load()
        m = part.mesh
        plan = ctypes.c_void_p()
        cells = (ctypes.c_int32 * 2)(m.n1, m.n2)
        h = (ctypes.c_double * 2)(m.h1, m.h2)
        blocks = (ctypes.c_int32 * 2)(part.b1, part.b2)
        _lib.check(self.L.msfv2d_plan_create(cells, h, blocks, ctypes.byref(plan)), "msfv2d_plan_create")
        self.plan = plan
        info = (ctypes.c_int64 * 9)()
        _lib.check(self.L.msfv2d_plan_info(plan, info, 9), "msfv2d_plan_info")
        self.NN, self.n, self.Nm, self.E, self.nbl, self.nI, self.k, self.factor_doubles, self.band_doubles = \
            [int(v) for v in info]
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.part = part

    def __del__(self):
        try:
            if getattr(self, "plan", None) is not None:
                self.L.msfv2d_plan_destroy(self.plan)
        except Exception:
            pass

    @classmethod
    def get(cls, part):
        key = (part, torch.cuda.current_device())
        e = cls._cache.get(key)
        if e is None:
            e = cls._cache[key] = Engine2D(part)
        return e

    def empty(self, *shape):
        return torch.empty(*shape, dtype=F64, device=self.device)

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=F64, device=self.device)

    # --- wrappers
    def operator(self, m):
        sigma, w = self.empty(self.Nm), self.empty(self.E)
        fl = torch.zeros(1, dtype=torch.int32, device=self.device)
        _lib.check(self.L.msfv2d_operator(self.plan, ptr(m), ptr(sigma), ptr(w), ptr(fl), stream()), "operator")
        return sigma, w, fl

    def basis(self, w, fl):
        factor, Sb, Kloc = self.empty(self.factor_doubles), self.empty(self.nbl * 4 * self.nI), self.empty(self.nbl * 16)
        _lib.check(self.L.msfv2d_basis(self.plan, ptr(w), ptr(factor), ptr(Sb), ptr(Kloc), ptr(fl), stream()), "basis")
        return factor, Sb, Kloc

    def galerkin(self, Kloc, shift):
        Ab = self.empty(self.band_doubles)
        _lib.check(self.L.msfv2d_galerkin(self.plan, ptr(Kloc), ctypes.c_double(shift), ptr(Ab), stream()), "galerkin")
        return Ab

    def coarse_factor(self, Ab, fl):
        Lk = self.empty(self.band_doubles)
        _lib.check(self.L.msfv2d_coarse_factor(self.plan, ptr(Ab), ptr(Lk), ptr(fl), stream()), "coarse_factor")
        return Lk

    def coarse_solve(self, Lk, X):
        X = X.contiguous().clone()
        _lib.check(self.L.msfv2d_coarse_solve(self.plan, ptr(Lk), ptr(X), X.shape[1], stream()), "coarse_solve")
        return X

    def interior_solve(self, factor, R):
        out = self.empty(*R.shape)
        _lib.check(self.L.msfv2d_interior_solve(self.plan, ptr(factor), ptr(R), ptr(out), R.shape[1], stream()),
                   "interior_solve")
        return out

    def prolong(self, Sb, Y):
        out = self.empty(self.n, Y.shape[1])
        _lib.check(self.L.msfv2d_prolong(self.plan, ptr(Sb), ptr(Y), ptr(out), Y.shape[1], stream()), "prolong")
        return out

    def restrict(self, Sb, X):
        out = self.empty(self.k, X.shape[1])
        _lib.check(self.L.msfv2d_restrict(self.plan, ptr(Sb), ptr(X), ptr(out), X.shape[1], stream()), "restrict")
        return out

    def apply_A(self, w, X):
        out = self.empty(*X.shape)
        _lib.check(self.L.msfv2d_apply_A(self.plan, ptr(w), ptr(X), ptr(out), X.shape[1], stream()), "apply_A")
        return out

    def grad(self, X):
        out = self.empty(self.E, X.shape[1])
        _lib.check(self.L.msfv2d_grad(self.plan, ptr(X), ptr(out), X.shape[1], stream()), "grad")
        return out

    def gradT(self, a, c=None):
        out = self.empty(self.n, a.shape[1])
        _lib.check(self.L.msfv2d_gradT(self.plan, ptr(a), ptr(c), ptr(out), a.shape[1], stream()), "gradT")
        return out

    def edge_average(self, sigma, dm):
        c = self.empty(self.E)
        _lib.check(self.L.msfv2d_edge_average(self.plan, ptr(sigma), ptr(dm), ptr(c), stream()), "edge_average")
        return c

    def cell_adjoint(self, sigma, e):
        out = self.empty(self.Nm)
        _lib.check(self.L.msfv2d_cell_adjoint(self.plan, ptr(sigma), ptr(e), ptr(out), e.shape[1], stream()),
                   "cell_adjoint")
        return out

    def axpby(self, alpha, a, b=None):
        out = self.empty(*a.shape)
        _lib.check(self.L.msfv2d_axpby(a.numel(), ctypes.c_double(alpha), ptr(a), ptr(b), ptr(out), stream()), "axpby")
        return out

    def fma3(self, a, b, c=None, d=None, e=None, f=None):
        out = self.empty(*a.shape)
        _lib.check(self.L.msfv2d_fma3(a.numel(), ptr(a), ptr(b), ptr(c), ptr(d), ptr(e), ptr(f), ptr(out), stream()),
                   "fma3")
        return out


class _Csr:
    """A host CSR matrix uploaded for msfv2d_spmm."""

    def __init__(self, eng, M):
        M = sp.csr_matrix(M)
        M.sort_indices()
        self.shape = M.shape
        self.ptr = torch.from_numpy(M.indptr.astype(np.int64)).to(eng.device)
        self.col = torch.from_numpy(M.indices.astype(np.int32)).to(eng.device)
        self.val = torch.from_numpy(M.data.astype(np.float64)).to(eng.device)
        self.L = eng.L
        self.eng = eng

    def mm(self, X, out=None, beta=0.0):
        nr = X.shape[1]
        if out is None:
            out = self.eng.empty(self.shape[0], nr)
        _lib.check(self.L.msfv2d_spmm(self.shape[0], ptr(self.ptr), ptr(self.col), ptr(self.val), ptr(X), nr,
                                      ctypes.c_double(beta), ptr(out), stream()), "spmm")
        return out


class SurveyDev2D:
    def __init__(self, eng, survey):
        self.P = _Csr(eng, survey.P)          # n x N_r: P W
        self.PT = _Csr(eng, survey.P.T)       # N_r x n: P^T X
        self.Qd = torch.from_numpy(np.ascontiguousarray(survey.Q.toarray(), dtype=np.float64)).to(eng.device)
        self.ns = survey.Q.shape[1]
        self.nr = survey.P.shape[1]


def _flags_check(fl, what):
    from .errors import InvalidModelError
    f = int(fl.item())
    if f & _lib.FLAG_NONFINITE:
        raise InvalidModelError("model vector contains non-finite entries")
    if f & _lib.FLAG_LOCAL_NOT_SPD:
        raise FactorizationError(f"{what}: a local interior operator is not SPD")
    return f


class ReducedState2D:
    """forward.py:62-75 ReducedState for the 2D path (device-resident)."""

    def __init__(self, eng, sdev, m_dev, sigma, w, factor, Sb, Lk, shift, T, U):
        self.eng, self.sdev = eng, sdev
        self.m_dev, self.sigma, self.w = m_dev, sigma, w
        self.factor, self.Sb, self.Lk, self.shift = factor, Sb, Lk, shift
        self.T_dev, self.U = T, U

    @property
    def T(self):
        return self.T_dev.cpu().numpy()

    def solve_reduced(self, B):
        B = torch.as_tensor(np.asarray(B, dtype=np.float64)).reshape(self.eng.k, -1).to(self.eng.device)
        return self.eng.coarse_solve(self.Lk, B).cpu().numpy()


class Sensitivity2D:
    """AdaptiveSensitivity (forward.py:224-281) for the 2D path.

    Init: U = S T, R = Q - A U, gprof = EP T = G_p (S T), gu = G_p U,
    a = G_p interior_solve(R).  EP = G_p S is never formed: EP^T x = S^T G_p^T x
    and EP y = G_p (S y)."""

    def __init__(self, state):
        e = self.eng = state.eng
        self.st = state
        sd = state.sdev
        R = e.axpby(-1.0, e.apply_A(state.w, state.U), sd.Qd)             # forward.py:243
        self.gu = e.grad(state.U)                                          # forward.py:245 (= EP T, :244)
        self.a = e.grad(e.interior_solve(state.factor, R))                 # forward.py:246

    def rapply_dev(self, W):                                               # forward.py:271-281
        e, st = self.eng, self.st
        p = st.sdev.P.mm(W.contiguous())
        y = e.coarse_solve(st.Lk, e.restrict(st.Sb, p))
        sy = e.prolong(st.Sb, y)
        z = e.interior_solve(st.factor, e.axpby(-1.0, e.apply_A(st.w, sy), p))
        gsy = e.grad(sy)
        ev = e.fma3(self.gu, e.grad(z), self.a, gsy, self.gu, gsy)
        return e.cell_adjoint(st.sigma, ev)

    def apply_dev(self, dm):                                               # forward.py:258-269
        e, st = self.eng, self.st
        c = e.edge_average(st.sigma, dm.contiguous())
        ydm = e.axpby(-1.0, e.interior_solve(st.factor, e.gradT(self.gu, c)))
        t = e.gradT(self.a, c)                                             # EP^T (a o c) = S^T t
        gdm = e.gradT(self.gu, c)
        rhs = e.axpby(-1.0, e.restrict(st.Sb, e.axpby(1.0, t, e.axpby(1.0, gdm, e.apply_A(st.w, ydm)))))
        dt = e.coarse_solve(st.Lk, rhs)
        return st.sdev.PT.mm(e.axpby(1.0, ydm, e.prolong(st.Sb, dt)))

    def apply(self, dm):
        dm = torch.as_tensor(np.asarray(dm, dtype=np.float64)).to(self.eng.device)
        return self.apply_dev(dm).cpu().numpy()

    def rapply(self, W):
        W = torch.as_tensor(np.asarray(W, dtype=np.float64)).to(self.eng.device)
        return self.rapply_dev(W).cpu().numpy()


class AdaptiveReducedProblem2D:
    """Problem protocol of inversion.py:307-323 for the 2D path."""

    mode = "ms_adaptive"

    def __init__(self, partition, survey, workers=1):
        self.partition = partition
        self.survey = survey
        self.workers = workers
        self._sdev = None

    @property
    def engine(self):
        return Engine2D.get(self.partition)

    def simulate_dev(self, m):
        e = self.engine
        if self._sdev is None:
            self._sdev = SurveyDev2D(e, self.survey)
        sd = self._sdev
        if torch.is_tensor(m):
            m_dev = m.to(device=e.device, dtype=F64).reshape(-1).contiguous()
        else:
            m = np.asarray(m, dtype=np.float64).reshape(-1)
            m_dev = torch.from_numpy(m).to(e.device)
        if m_dev.numel() != e.Nm:
            raise ValueError("model length does not match the mesh")
        sigma, w, fl = e.operator(m_dev)
        factor, Sb, Kloc = e.basis(w, fl)
        shift = 0.0
        Lk = e.coarse_factor(e.galerkin(Kloc, 0.0), fl)
        f = _flags_check(fl, "basis")
        if f & _lib.FLAG_COARSE_NOT_SPD:                                   # forward.py:122-129
            Ab = e.galerkin(Kloc, 0.0)
            diag = Ab.reshape(e.k, -1)[:, 0]
            shift = 1e-12 * float(diag.sum()) / e.k
            fl.zero_()
            Lk = e.coarse_factor(e.galerkin(Kloc, shift), fl)
            if int(fl.item()) & _lib.FLAG_COARSE_NOT_SPD:
                raise ReducedSingularError("reduced operator is singular even after the diagonal shift")
        T = e.coarse_solve(Lk, e.restrict(Sb, sd.Qd))                      # forward.py:115-116,142
        U = e.prolong(Sb, T)
        D = sd.PT.mm(U)                                                    # forward.py:143
        return D, ReducedState2D(e, sd, m_dev, sigma, w, factor, Sb, Lk, shift, T, U)

    def simulate(self, m):
        D, st = self.simulate_dev(m)
        return D.cpu().numpy(), st

    def jacobian(self, state):
        return Sensitivity2D(state)


# ----------------------------------------------------------- BASELINE configs 1-2

def _cell_nodes(mesh, i, j):
    """Pinned ids of the 4 corner nodes of cell (i, j) (node 0 dropped)."""
    ids = [mesh.node_index(i + a, j + b) for b in (0, 1) for a in (0, 1)]
    return [int(q) - 1 for q in ids if q != 0]


def cell_survey_2d(mesh, src_pairs, rec_cells):
    """Sources / receivers at cells: 1/4 on each corner node of the cell
    (SURVEY.md 8(d) cell->node mapping), pinned ids."""
    n = mesh.n_nodes - 1
    rows, cols, vals = [], [], []
    for s, (plus, minus) in enumerate(src_pairs):
        for cell, sgn in ((plus, 1.0), (minus, -1.0)):
            for q in _cell_nodes(mesh, *cell):
                rows.append(q)
                cols.append(s)
                vals.append(0.25 * sgn)
    Q = sp.csc_matrix((vals, (rows, cols)), shape=(n, len(src_pairs)))
    rows, cols, vals = [], [], []
    for r, cell in enumerate(rec_cells):
        for q in _cell_nodes(mesh, *cell):
            rows.append(q)
            cols.append(r)
            vals.append(0.25)
    P = sp.csc_matrix((vals, (rows, cols)), shape=(n, len(rec_cells)))
    return Survey(P=P, Q=Q)


def fine_operator_2d(mesh, m):
    """Host assembly of the fine 2D operator (pinned) for synthetic data only."""
    n1, n2 = mesh.n1, mesh.n2
    sig = np.exp(np.asarray(m, dtype=float)).reshape(n2, n1)
    hv = 0.5 * mesh.volume
    wx = np.zeros((n2 + 1, n1))
    wx[:-1] += hv * sig
    wx[1:] += hv * sig
    wy = np.zeros((n2, n1 + 1))
    wy[:, :-1] += hv * sig
    wy[:, 1:] += hv * sig
    I, J = np.meshgrid(np.arange(n1), np.arange(n2 + 1))
    a, b = mesh.node_index(I, J).ravel(), mesh.node_index(I + 1, J).ravel()
    kx = wx.ravel() / mesh.h1 ** 2
    I, J = np.meshgrid(np.arange(n1 + 1), np.arange(n2))
    c, d = mesh.node_index(I, J).ravel(), mesh.node_index(I, J + 1).ravel()
    ky = wy.ravel() / mesh.h2 ** 2
    r = np.concatenate([a, b, a, b, c, d, c, d])
    s = np.concatenate([a, b, b, a, c, d, d, c])
    v = np.concatenate([kx, kx, -kx, -kx, ky, ky, -ky, -ky])
    A = sp.coo_matrix((v, (r, s)), shape=(mesh.n_nodes,) * 2).tocsr()
    return A[1:, 1:].tocsc()


def fine_data_2d(mesh, m, survey):
    """D = P^T A^-1 Q on the fine grid (the d_obs generator of config 1)."""
    import scipy.sparse.linalg as spla
    u = spla.splu(fine_operator_2d(mesh, m)).solve(survey.Q.toarray())
    return np.asarray(survey.P.T @ u)


def config_problem_2d(cfg_id, seed=0):
    """(mesh, partition, survey, m_eval, d_obs) for BASELINE.json configs 1-2."""
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(seed)
    if cfg_id == 1:
        n, b = 64, 8
        mesh = create_mesh_2d(n, n)
        ci, cj = np.meshgrid(np.arange(n), np.arange(n))
        x, y = ((ci + 0.5) / n).ravel(), ((cj + 0.5) / n).ravel()
        m_true = (1.0 * ((x >= 0.2) & (x <= 0.4) & (y >= 0.5) & (y <= 0.7))
                  - 1.0 * ((x >= 0.6) & (x <= 0.8) & (y >= 0.2) & (y <= 0.4)))
        m_true = m_true + 0.1 * rng.standard_normal(n * n)
        survey = cell_survey_2d(mesh, [((8, 32), (56, 32))], [(i, 60) for i in range(1, 64, 2)])
        d_obs = fine_data_2d(mesh, m_true, survey)
        return mesh, create_partition_2d(mesh, b, b), survey, np.zeros(n * n), d_obs
    if cfg_id == 2:
        n, b = 256, 16
        mesh = create_mesh_2d(n, n)
        g = gaussian_filter(rng.standard_normal((n, n)), 8.0, mode="reflect")
        m = ((g - g.mean()) / g.std()).ravel()
        js = range(8, 256, 16)
        survey = cell_survey_2d(mesh, [((0, j), (255, j)) for j in js], [(i, 255) for i in range(1, 256, 2)])
        d_obs = fine_data_2d(mesh, m, survey)
        return mesh, create_partition_2d(mesh, b, b), survey, m, d_obs
    raise ValueError("2D configs are 1 and 2")
