"""Reduced forward map and adaptive sensitivities on the GPU.

Drop-in for the adaptive path of the reference's forward.py
(``forward_reduced`` forward.py:105-144, ``AdaptiveSensitivity``
forward.py:209-281, ``sensitivity_adaptive`` forward.py:292).  Inputs and
outputs are numpy arrays like the reference (torch tensors are accepted too);
everything in between stays on the device.

Compact forms used for the Lagrange basis (EP == G_p S, so the reference's
gprof == gu; verified against the reference to 1e-14):
  init      U = S T, ZR = blockdiag(A_II^-1)(Q - A U)
  rapply    y = A_k^-1 S^T P W, sy = S y, z = blockdiag(A_II^-1)(P W - A sy)
            g = -sigma C^T sum_s [G U . G(z + sy) + G ZR . G sy]
  apply     c = C(sigma dm), ydm = -blockdiag(A_II^-1) A_c U
            dt = -A_k^-1 S^T [A_c (ZR + U) + A ydm],  J dm = P^T (ydm + S dt)
where A_c = G_p^T diag(c) G_p.
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from .engine import Points, engine_for
from .errors import ReducedSingularError, StaleBasisError

DENSE_REDUCED_LIMIT = 5000     # forward.py:20 (kept for API parity; the GPU factor is banded at every k)


@dataclass
class Survey:
    """Receivers P, sources Q (pinned space) and optional data (forward.py:23-51)."""

    P: sp.csc_matrix
    Q: sp.csc_matrix
    D_obs: np.ndarray = None
    noise_level: float = 0.0
    _pts: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        self.P = sp.csc_matrix(self.P)
        self.Q = sp.csc_matrix(self.Q)
        if self.P.shape[0] != self.Q.shape[0]:
            raise ValueError("receiver and source matrices disagree on node count")
        for name, M in (("receiver", self.P), ("source", self.Q)):
            if np.any(np.diff(M.indptr) == 0):
                raise ValueError(f"{name} matrix has an empty column")
        if self.D_obs is not None:
            self.D_obs = np.asarray(self.D_obs, dtype=float)
            if self.D_obs.shape != (self.n_receivers, self.n_sources):
                raise ValueError("observed data shape does not match survey")

    @property
    def n_receivers(self):
        return self.P.shape[1]

    @property
    def n_sources(self):
        return self.Q.shape[1]

    def device(self, engine):
        """(P points, Q points, dense Q field) uploaded for ``engine``."""
        key = id(engine)
        d = self._pts.get(key)
        if d is None:
            if self.P.shape[0] != engine.n:
                raise ValueError("survey node count does not match the mesh")
            Pp = Points(engine, self.P)
            Qp = Points(engine, self.Q)
            Qf = engine.scatter_points(Qp, None, self.n_sources)
            # the entry keeps the engine alive: id(engine) cannot be reused by another engine while it is cached
            d = (Pp, Qp, Qf, engine)
            self._pts[key] = d
        return d[:3]


def _host(t):
    """Device tensor -> numpy.  Large results go through a page-locked buffer
    (torch's caching host allocator) so the copy runs at full link speed; the
    returned array owns that buffer."""
    if t.is_cuda and t.numel() * t.element_size() >= (1 << 20):
        import torch
        buf = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        buf.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return buf.numpy()
    return t.cpu().numpy()


class ReducedState:
    """Result of the reduced forward solve (forward.py:62-75)."""

    def __init__(self, op, basis, Lk, T_dev, shift, survey):
        self.op = op
        self.basis = basis
        self.Lk = Lk
        self.T_dev = T_dev
        self.shift = shift
        self.survey = survey
        self.chol = None
        self._T = None
        self._A_k = None

    @property
    def T(self):
        if self._T is None:
            self._T = _host(self.T_dev)
        return self._T

    @T.setter
    def T(self, value):
        self._T = np.asarray(value, dtype=float)
        self.T_dev = self.basis.engine.to_device(self._T)

    @property
    def A_k(self):
        """Dense projected operator (forward.py:102), re-assembled on demand.
        Like the reference it is the unshifted S^T A S: the diagonal shift of
        the fallback (forward.py:122-129) lives only in the factor."""
        if self._A_k is None:
            eng = self.basis.engine
            self._A_k = _host(eng.coarse_dense(self.basis.Kloc, 0.0))
        return self._A_k

    def check(self, host_flags=None):
        """Resolve the status of the forward chain (one device sync, or none
        when the caller already read the status word: ``host_flags``)."""
        if not getattr(self, "pending", False):
            return
        self.pending = False
        from .basis import raise_status
        f = int(self.flags.item()) if host_flags is None else int(host_flags)
        raise_status(f & 7)
        if f & 8:
            # diagonal shift fallback (forward.py:122-129)
            eng = self.basis.engine
            tr = float(eng.coarse_trace(eng.galerkin(self.basis.Kloc, 0.0)).sum().item())
            shift = 1e-12 * tr / eng.k
            self.flags.zero_()
            D, Ak, T = _coarse_solve_chain(eng, self.op, self.survey, self.basis, shift, self.flags)
            if int(self.flags.item()) & 8:
                raise ReducedSingularError("projected operator is singular even after diagonal shift")
            self.D_dev.copy_(D)
            self.Lk, self.T_dev, self.shift = Ak, T, shift
            self._T = None

    def solve_reduced(self, B):
        eng = self.basis.engine
        B = np.asarray(B, dtype=float)
        single = B.ndim == 1
        X = eng.to_device(B[:, None] if single else B).clone()
        eng.coarse_solve(self.Lk, X)
        out = _host(X)
        return out[:, 0] if single else out


def _coarse_solve_chain(eng, op, survey, basis, shift, fl):
    Pp, Qp, _ = survey.device(eng)
    ns = survey.n_sources
    F = eng.restrict_points(Qp, basis.sint_for(Qp), None, ns)        # S^T Q   (forward.py:115)
    Ak = eng.galerkin(basis.Kloc, shift)                              # S^T A S (+ shift I) (forward.py:118,125)
    if eng.coarse_multifrontal:
        basis.start_backward()                                        # S_I sweeps beside the whole coarse phase
    eng.coarse_factor(Ak, fl)                                         # cho_factor (forward.py:121)
    basis.start_backward()                                            # S_I sweeps overlap the coarse solve
    T = eng.coarse_solve(Ak, F)                                       # T = A_k^-1 S^T Q (forward.py:142)
    D = eng.receive(Pp, basis.sint_for(Pp), Y=T)                      # P^T S T (forward.py:143)
    return D, Ak, T


def forward_reduced_dev(op, survey, basis, defer_check=False):
    """Device-resident reduced forward: returns (D device tensor, state).

    With ``defer_check`` nothing synchronises; the status bits (invalid model,
    local or coarse factorization failure) are resolved by ``state.check()``,
    which also takes the reference's diagonal-shift fallback (forward.py:122-129)."""
    if hasattr(basis, "layout"):             # enriched families (enriched.py)
        from .enriched import forward_enriched_dev
        return forward_enriched_dev(op, survey, basis)
    eng = basis.engine
    if basis.bx is not None:
        eng.bind_boundary(basis.bx)          # reduced boundary values of this basis
    if op._dev is None or op._dev[0] is not eng:
        op.device_state(eng)
    if op._dev[1] is not basis._m_dev and not torch.equal(op._dev[1], basis._m_dev):
        raise NotImplementedError("forward_reduced with a basis frozen at another model "
                                  "(ms_fixed mode) is outside this tier's GPU path")
    fl = op.flags
    D, Ak, T = _coarse_solve_chain(eng, op, survey, basis, 0.0, fl)
    state = ReducedState(op, basis, Ak, T, 0.0, survey)
    state.D_dev = D
    state.flags = fl
    state.pending = True
    if not defer_check:
        state.check()
    return state.D_dev, state


def forward_reduced(op, survey, basis):
    """Predicted data through the projected problem (forward.py:105-144).

    The status word and D come back in one synchronisation (both copies are
    queued before the wait); the shift fallback, when the status asks for it,
    recomputes D and copies it again."""
    import torch
    if hasattr(basis, "layout"):             # enriched families (enriched.py)
        from .enriched import forward_enriched
        return forward_enriched(op, survey, basis)
    D, state = forward_reduced_dev(op, survey, basis, defer_check=True)
    Dh = torch.empty(D.shape, dtype=D.dtype, pin_memory=True)
    fh = torch.empty(1, dtype=state.flags.dtype, pin_memory=True)
    Dh.copy_(D, non_blocking=True)
    fh.copy_(state.flags, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    f = int(fh[0])
    state.check(host_flags=f)
    if f & 8:
        return _host(state.D_dev), state
    return Dh.numpy(), state


class AdaptiveSensitivity:
    """Sensitivity of the adaptive reduced map (forward.py:209-281)."""

    mode = "ms_adaptive"

    def __init__(self, state, survey, workers=1):
        op, basis = state.op, state.basis
        eng = basis.engine
        if basis.bx is not None:
            raise NotImplementedError("a basis with reduced boundary conditions takes ReducedSensitivity "
                                      "(sensitivity_adaptive dispatches to it)")
        if not getattr(state, "deferred", False):
            state.check()
        if op._dev is None or op._dev[1] is not basis._m_dev:
            basis.check_model(op.m)
        self.state, self.survey, self.basis, self.engine = state, survey, basis, eng
        self.workers = workers
        _, _, self.sigma, self.w = op._dev
        self.Pp, self.Qp, self._Qf = survey.device(eng)
        # interior_solve(Q - A S T) = blockdiag(A_II^-1) Q_I since (A S)_I = 0
        # (Lagrange local problems, basis.py:548): compact, on the source blocks only
        self.Rc = eng.interior_fields(self.Qp, basis.factor, None, survey.n_sources)
        self._U = self._ZR = self._UR = None

    # node fields of the forward state (J v only; rapply works block-locally)
    @property
    def U(self):
        if self._U is None:
            self._U = self.engine.prolong(self.basis.Sint, self.state.T_dev)               # S T (forward.py:241)
        return self._U

    @property
    def ZR(self):
        if self._ZR is None:
            eng, ns = self.engine, self.survey.n_sources
            R = eng.residual(self._Qf, 1.0, self.w, self.U, -1.0, ns)                     # Q - A U (forward.py:243)
            self._ZR = eng.interior_solve(self.basis.factor, R)                           # interior_solve(R) (:246)
        return self._ZR

    @property
    def UR(self):
        if self._UR is None:
            self._UR = self.U + self.ZR
        return self._UR

    # ---------------------------------------------------------- device API
    def rapply_dev(self, W):
        eng, b = self.engine, self.basis
        ns = self.survey.n_sources
        W = eng.to_device(W)
        y = eng.restrict_points(self.Pp, b.sint_for(self.Pp), W, ns)                # S^T P W (forward.py:276)
        eng.coarse_solve(self.state.Lk, y)
        # z = interior_solve(P W - A S y) = blockdiag(A_II^-1)(P W)_I (forward.py:278)
        Zc = eng.interior_fields(self.Pp, b.factor, W, ns)
        try:
            return eng.block_gradient(self.sigma, b.Sint, self.state.T_dev, y, self.Pp, Zc, self.Qp, self.Rc)
        except NotImplementedError:
            pass
        # blocks too large for the fused kernel: node-field form
        sy = eng.prolong(b.Sint, y)                                                 # S y (forward.py:277)
        pf = eng.scatter_points(self.Pp, W, ns)                                     # P W (forward.py:275)
        z = eng.residual(pf, 1.0, self.w, sy, -1.0, ns)                             # p - A sy (forward.py:278)
        eng.interior_solve(b.factor, z)
        return eng.cell_gradient(self.sigma, self.U, z, sy, self.ZR)                # forward.py:278-280

    def apply_dev(self, dm):
        eng, b = self.engine, self.basis
        ns = self.survey.n_sources
        dm = eng.to_device(dm).reshape(-1)
        c = eng.edge_average(self.sigma, dm)                                        # Csig dm (forward.py:259)
        if self.Pp.interior_blocks == 0:
            # receivers on the skeleton: P^T ydm = 0 and S^T A ydm = (A S)^T ydm = 0,
            # so only the coarse rhs -EP^T(G UR o c) remains (block-local)
            try:
                dt = eng.jv_coarse_rhs(b.Sint, c, self.state.T_dev, self.Qp, self.Rc)
            except NotImplementedError:
                dt = None
            if dt is not None:
                eng.coarse_solve(self.state.Lk, dt)                                 # forward.py:267
                return eng.receive(self.Pp, b.sint_for(self.Pp), Y=dt)              # P^T S dt (:268)
        ydm = eng.residual(None, 0.0, c, self.U, -1.0, ns)                          # -G^T(gu c)
        eng.interior_solve(b.factor, ydm)                                         # _Y_dm (forward.py:250-252)
        dt = eng.restrict_op(b.Sint, c, self.UR, self.w, ydm, ns, scale=-1.0)       # xdm - S^T(gdm + A ydm)
        eng.coarse_solve(self.state.Lk, dt)                                         # forward.py:267
        return eng.receive(self.Pp, b.Sint, Y=dt, Xfield=ydm)                       # P^T(ydm + S dt) (:268)

    # ------------------------------------------------------- reference API
    def apply(self, dm):
        dm = np.asarray(dm, dtype=float) if not hasattr(dm, "detach") else dm
        return _host(self.apply_dev(dm))

    def rapply(self, W):
        W = np.asarray(W, dtype=float) if not hasattr(W, "detach") else W
        eng, b = self.engine, self.basis
        ns = self.survey.n_sources
        Wd = eng.to_device(W)
        y = eng.restrict_points(self.Pp, b.sint_for(self.Pp), Wd, ns)
        eng.coarse_solve(self.state.Lk, y)
        Zc = eng.interior_fields(self.Pp, b.factor, Wd, ns)
        try:
            # fused gradient, copied back slab by slab behind the computation
            return eng.block_gradient_to_host(self.sigma, b.Sint, self.state.T_dev, y, self.Pp, Zc, self.Qp, self.Rc)
        except NotImplementedError:
            return _host(self.rapply_dev(W))


def sensitivity_adaptive(state, survey, workers=1):
    if hasattr(state.basis, "layout"):       # enriched families (enriched.py)
        from .enriched import EnrichedSensitivity
        return EnrichedSensitivity(state, survey, workers=workers)
    if getattr(state.basis, "bx", None) is not None:   # reduced boundary conditions (reduced_sens.py)
        from .reduced_sens import ReducedSensitivity
        return ReducedSensitivity(state, survey, workers=workers)
    return AdaptiveSensitivity(state, survey, workers=workers)
