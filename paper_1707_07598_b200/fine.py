"""Fine-mesh forward model, full-mesh sensitivities and block CG on the GPU
(SURVEY.md 8(f) row N1).

Drop-in for the reference's ``forward_full`` / ``FullState`` /
``FullSensitivity`` / ``sensitivity_full`` (forward.py:54-98, 147-175, 284)
and ``block_cg`` / ``IterativeResult`` (solvers.py:45-136).  The operator
products run in libmsfv.so (``msfv_fine_apply``: A(w) X over every pinned node
from the device edge weights; ``msfv_full_gradient``: the adjoint products
sum_j G_j^T v_j); the block recurrences keep the reference's algorithm, with
the tall-skinny block products (P^T Q, P alpha) as library GEMMs on the device
and the s x s Cholesky / solves on the host exactly as solvers.py does them.

``solver="direct"``: the reference factors A with SuperLU (solvers.py:30-40),
which does not finish at 64^3 in 20 min; the GPU path has no
sparse direct factorization and solves to a tight residual instead
(CG per column, relative residual <= DIRECT_TOL, preconditioned by the
two-level MSFV method itself: the adaptive basis, its Galerkin coarse solve
and the block interior solves), the role the factorization plays for every
later solve of the same state.
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from .engine import engine_for_mesh
from .errors import SolverBreakdown

DIRECT_TOL = 1e-13       # relative residual of the "direct" GPU solves
DIRECT_MAXIT = 100000


@dataclass
class IterativeResult:
    """solvers.py:45-52."""

    X: object
    iterations: int
    relres: float
    converged: bool
    history: list = field(default_factory=list)


def _cholesky_solve(c, B):
    # np.linalg.solve(c.T, np.linalg.solve(c, B)) as solvers.py:106,128
    return np.linalg.solve(c.T, np.linalg.solve(c, B))


def block_cg_dev(apply, B, tol=1e-6, maxit=100, precond=None):
    """Block CG on device tensors (solvers.py:57-136, same recurrence, restart
    and stopping rule).  ``apply(X)`` returns A X for an (N, s) device tensor;
    ``precond`` (optional) returns M^{-1} R, giving block PCG (the directions
    use Z = M^{-1} R; precond=None is exactly the reference's algorithm).
    Returns IterativeResult with X an (N, ns) device tensor."""
    if tol <= 0:
        raise ValueError(f"tolerance must be > 0, got {tol}")
    if maxit < 1:
        raise ValueError(f"maxit must be >= 1, got {maxit}")
    single = B.dim() == 1
    if single:
        B = B[:, None]
    B = B.contiguous()
    ns = B.shape[1]
    X = torch.zeros_like(B)
    bnorm = torch.linalg.vector_norm(B, dim=0).cpu().numpy()
    relres = np.zeros(ns)
    history = []
    active = np.flatnonzero(bnorm > 0)
    pz = precond if precond is not None else (lambda R: R)
    R = B[:, active].clone()
    P = pz(R).clone()
    it = 0
    converged = not active.size

    def finish(flag):
        return IterativeResult(X=X[:, 0] if single else X, iterations=it, relres=float(relres.max(initial=0.0)),
                               converged=flag, history=history)

    while it < maxit and active.size:
        Q = apply(P)
        G = torch.stack((P.T @ Q, P.T @ R)).cpu().numpy()         # P^T Q, P^T R in one transfer
        try:
            c = np.linalg.cholesky(G[0])
            alpha = _cholesky_solve(c, G[1])
        except np.linalg.LinAlgError:
            raise SolverBreakdown(f"direction block lost rank at iteration {it}", result=finish(False)) from None
        a_dev = torch.from_numpy(alpha).to(B.device)
        idx = torch.from_numpy(active).to(B.device)
        X[:, idx] += P @ a_dev
        R = R - Q @ a_dev
        it += 1
        relres[active] = torch.linalg.vector_norm(R, dim=0).cpu().numpy() / bnorm[active]
        history.append(float(relres.max(initial=0.0)))
        done = relres[active] <= tol
        if done.any():
            active = active[~done]
            if not active.size:
                converged = True
                break
            idx = torch.from_numpy(active).to(B.device)
            Xa = X[:, idx].contiguous()
            R = B[:, idx] - apply(Xa)                             # restart on the surviving columns
            P = pz(R).clone()
            continue
        Z = pz(R)
        beta = _cholesky_solve(c, -(Q.T @ Z).cpu().numpy())
        P = Z + P @ torch.from_numpy(beta).to(B.device)
    if active.size:
        idx = torch.from_numpy(active).to(B.device)
        Xa = X[:, idx].contiguous()
        relres[active] = torch.linalg.vector_norm(B[:, idx] - apply(Xa), dim=0).cpu().numpy() / bnorm[active]
        converged = bool(np.all(relres <= tol))
    return finish(converged)


def pcg_columns_dev(apply, B, tol, maxit, precond, check_every=8):
    """Independent preconditioned CG per column, all columns advanced together
    (one multi-column operator product per iteration; per-column step
    lengths, so no block Gram matrix can lose rank).  Converged columns are
    frozen; the residual test runs every ``check_every`` iterations.  Returns
    IterativeResult with X an (N, s) device tensor."""
    B = B.contiguous()
    ns = B.shape[1]
    X = torch.zeros_like(B)
    bnorm = torch.linalg.vector_norm(B, dim=0)
    live = (bnorm > 0).to(B.dtype)
    R = B.clone()
    Z = precond(R)
    P = Z.clone()
    rz = torch.sum(R * Z, dim=0)
    it = 0
    history = []
    relres = np.zeros(ns)
    while it < maxit:
        Q = apply(P)
        pq = torch.sum(P * Q, dim=0)
        a = torch.where(pq > 0, rz / torch.where(pq > 0, pq, torch.ones_like(pq)), torch.zeros_like(pq)) * live
        X += P * a
        R -= Q * a
        it += 1
        if it % check_every == 0 or it == maxit:
            rr = (torch.linalg.vector_norm(R, dim=0) / torch.where(bnorm > 0, bnorm, torch.ones_like(bnorm)))
            relres = (rr * live).cpu().numpy()
            history.append(float(relres.max(initial=0.0)))
            live = live * (rr > tol).to(B.dtype)
            if not bool(live.any()):
                break
        Z = precond(R)
        rz_new = torch.sum(R * Z, dim=0)
        b = torch.where(rz > 0, rz_new / torch.where(rz > 0, rz, torch.ones_like(rz)), torch.zeros_like(rz))
        P = Z + P * b
        rz = rz_new
    res = IterativeResult(X=X, iterations=it, relres=float(relres.max(initial=0.0)),
                          converged=bool(np.all(relres <= tol)), history=history)
    return res


def _csr_apply(A, device):
    """Device CSR SpMM for a scipy sparse matrix (pinned-space rows)."""
    from . import _lib
    from .engine import ptr, stream
    A = sp.csr_matrix(A)
    A.sort_indices()
    ip = torch.from_numpy(A.indptr.astype(np.int64)).to(device)
    ix = torch.from_numpy(A.indices.astype(np.int32)).to(device)
    vv = torch.from_numpy(A.data.astype(np.float64)).to(device)
    L = _lib.load()
    n = A.shape[0]

    def apply(X):
        X = X.contiguous()
        out = torch.empty((n, X.shape[1]), dtype=torch.float64, device=device)
        _lib.check(L.msfv2d_spmm(n, ptr(ip), ptr(ix), ptr(vv), ptr(X), X.shape[1], 0.0, ptr(out), stream()), "spmm")
        return out
    return apply


def _jacobi_inverse(eng, w):
    """1 / diag(A) as a full node field column (0 on the pinned node): the
    7-point stencil couples only nodes of opposite (i + j + k) parity, so
    A applied to the indicator of one parity class returns the diagonal on
    that class (two stencil sweeps)."""
    n1, n2 = eng.cells[0] + 1, eng.cells[1] + 1
    idx = torch.arange(eng.Nn, device=eng.device)
    par = ((idx % n1) + (idx // n1) % n2 + idx // (n1 * n2)) % 2
    red = (par == 0).to(torch.float64)[:, None]
    red[0] = 0.0
    black = (par == 1).to(torch.float64)[:, None]
    d = eng.fine_apply(w, red) * red + eng.fine_apply(w, black) * black
    dinv = torch.where(d > 0, 1.0 / d, torch.zeros_like(d))
    dinv[0] = 0.0
    return dinv


def block_cg(A, B, tol=1e-6, maxit=100):
    """Reference-named block CG (solvers.py:57-136): ``A`` is a scipy sparse
    SPD matrix (device CSR SpMM) or a DiffusionOperator (device stencil over
    the pinned space); ``B`` (n,) or (n, s) numpy or torch.  Returns an
    IterativeResult whose X is a numpy array (a device tensor when B is one)."""
    on_dev = isinstance(B, torch.Tensor) and B.is_cuda
    Bt = B if isinstance(B, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(B, dtype=np.float64))
    dev = torch.device("cuda", torch.cuda.current_device())
    Bt = Bt.to(dev, dtype=torch.float64)
    single = Bt.dim() == 1
    if single:
        Bt = Bt[:, None]
    if hasattr(A, "device_state"):
        eng = engine_for_mesh(A.mesh)
        _, _, _, w = A.device_state(eng)
        n = eng.n
        if Bt.shape[0] != n:
            raise ValueError(f"right-hand side has {Bt.shape[0]} rows, operator {n}")
        Bf = torch.zeros((eng.Nn, Bt.shape[1]), dtype=torch.float64, device=dev)
        Bf[1:] = Bt
        res = block_cg_dev(lambda X: eng.fine_apply(w, X), Bf, tol, maxit)
        X = res.X[1:]
    else:
        if Bt.shape[0] != A.shape[0]:
            raise ValueError(f"right-hand side has {Bt.shape[0]} rows, operator {A.shape[0]}")
        res = block_cg_dev(_csr_apply(A, dev), Bt, tol, maxit)
        X = res.X
    if single:
        X = X[:, 0]
    res.X = X if on_dev else X.cpu().numpy()
    return res


# ------------------------------------------------------------ forward model

@dataclass
class FullState:
    """forward.py:54-59; U is the (n, N_s) fine field, kept on the device."""

    op: object
    factor: object
    U_dev: object
    solver_info: dict = field(default_factory=dict)
    survey: object = None

    @property
    def U(self):
        return self.U_dev[1:].cpu().numpy()


def _coarse_blocks(n):
    """Coarse block size along one axis for the two-level preconditioner:
    the largest divisor of n up to 8 (8 on the BASELINE meshes)."""
    return max(d for d in range(1, 9) if n % d == 0)


class _TwoLevel:
    """Two-level additive Schwarz preconditioner built from this package's own
    MSFV machinery at the operator's model:

        M^{-1} r = S A_k^{-1} S^T r + blockdiag(A_II^{-1}) r_I + D_skel^{-1} r_skel

    (the adaptive Lagrange basis S, the Galerkin coarse operator and its
    factorization, the per-block interior solves, Jacobi on the skeleton).
    Symmetric positive definite (the three parts cover every node), so PCG
    applies; the coarse space removes the mesh- and contrast-dependent
    low modes the Jacobi preconditioner leaves (2992 -> tens of iterations at
    128^3)."""

    def __init__(self, op, dinv):
        from .basis import BasisBuilder
        from .mesh import create_partition
        mesh = op.mesh
        part = create_partition(mesh, _coarse_blocks(mesh.n1), _coarse_blocks(mesh.n2), _coarse_blocks(mesh.n3))
        self.basis = BasisBuilder(part).assemble(op)
        eng = self.eng = self.basis.engine
        self.Sint = self.basis.Sint
        self.Ak = eng.galerkin(self.basis.Kloc, 0.0)
        fl = eng.flags()
        eng.coarse_factor(self.Ak, fl)
        self.ok = int(fl.item()) == 0 and int(op.flags.item()) & 7 == 0
        # Jacobi on the skeleton only (interiors get the block solves)
        n1, n2, n3 = mesh.n1 + 1, mesh.n2 + 1, mesh.n3 + 1
        b = (part.b1, part.b2, part.b3)
        idx = torch.arange(eng.Nn, device=eng.device)
        i, j, k = idx % n1, (idx // n1) % n2, idx // (n1 * n2)
        skel = ((i % b[0]) == 0) | ((j % b[1]) == 0) | ((k % b[2]) == 0)
        self.dskel = dinv * skel.to(torch.float64)[:, None]

    def __call__(self, R):
        eng, ns = self.eng, R.shape[1]
        y = eng.restrict_op(self.Sint, None, R, None, None, ns)       # S^T r
        eng.coarse_solve(self.Ak, y)                                   # A_k^{-1} S^T r
        out = eng.prolong(self.Sint, y)                                # S (.)
        Z = eng.zeros(eng.Nn, ns)
        eng.interior_solve(self.basis.factor, R, Z)                    # blockdiag(A_II^{-1}) r_I
        return out + Z + self.dskel * R


class _DeviceSolve:
    """The solve a factorization would provide (solvers.py:16-27): PCG per
    column to a tight residual on the device, full node fields, with the
    two-level MSFV preconditioner (Jacobi when the mesh admits no coarse
    partition or the coarse factorization fails)."""

    def __init__(self, eng, w, op=None):
        self.eng, self.w = eng, w
        self.dinv = _jacobi_inverse(eng, w)
        self.n = eng.n
        self.pre = None
        if op is not None:
            try:
                pre = _TwoLevel(op, self.dinv)
                self.pre = pre if pre.ok else None
            except (NotImplementedError, ValueError):
                self.pre = None

    def solve_dev(self, Bf):
        pz = self.pre if self.pre is not None else (lambda R: R * self.dinv)
        res = pcg_columns_dev(lambda X: self.eng.fine_apply(self.w, X), Bf, DIRECT_TOL, DIRECT_MAXIT,
                              precond=pz)
        if not res.converged:
            from .errors import FactorizationError
            raise FactorizationError(f"fine solve stalled at relative residual {res.relres:.2e}")
        self.last = res
        return res.X


def _bind(op):
    eng = engine_for_mesh(op.mesh)
    _, _, sigma, w = op.device_state(eng)
    from .basis import raise_status
    raise_status(int(op.flags.item()) & 3)      # InvalidModelError (operators.py:26-27)
    return eng, sigma, w


def forward_full(op, survey, solver="direct", cg_tol=1e-6, cg_maxit=100):
    """Predicted data and fields of the fine-mesh problem (forward.py:78-98)."""
    eng, sigma, w = _bind(op)
    Pp, Qp, Qf = survey.device(eng)
    if solver == "direct":
        factor = _DeviceSolve(eng, w, op)
        U = factor.solve_dev(Qf)
        info = {}
    elif solver == "blockcg":
        res = block_cg_dev(lambda X: eng.fine_apply(w, X), Qf, tol=cg_tol, maxit=cg_maxit)
        factor = None
        U = res.X
        info = {"iterations": res.iterations, "relres": res.relres, "converged": res.converged}
    else:
        raise ValueError(f"unknown solver {solver!r}")
    D = eng.receive(Pp, None, Xfield=U, nrhs=U.shape[1])                      # P^T U (forward.py:97)
    return D.cpu().numpy(), FullState(op=op, factor=factor, U_dev=U, solver_info=info, survey=survey)


class FullSensitivity:
    """Sensitivity of the fine-mesh forward map (forward.py:147-175).

    apply:  J dm = -P^T A^{-1} [G_j dm]_j,  G_j dm = A_c u_j with c = C(sigma dm)
    rapply: J^T W = -sum_j G_j^T v_j,  V = A^{-1} P W,
            sum_j G_j^T v_j = sigma C^T sum_j (G u_j)(G v_j)   (msfv_full_gradient)"""

    mode = "full"

    def __init__(self, state, survey, cg_tol=1e-6, cg_maxit=100):
        op = state.op
        self.survey = survey
        self.eng, self.sigma, self.w = _bind(op)
        self.Pp, self.Qp, _ = survey.device(self.eng)
        self.U = state.U_dev
        if state.factor is not None:
            self._solve = state.factor.solve_dev
        else:
            eng, w = self.eng, self.w
            self._solve = lambda B: block_cg_dev(lambda X: eng.fine_apply(w, X), B, tol=cg_tol, maxit=cg_maxit).X

    def apply_dev(self, dm):
        eng = self.eng
        dm = eng.to_device(dm).reshape(-1)
        c = eng.edge_average(self.sigma, dm)                                  # C (sigma o dm)
        W = eng.fine_apply(c, self.U)                                         # [G_j dm]_j
        return -eng.receive(self.Pp, None, Xfield=self._solve(W), nrhs=W.shape[1])

    def rapply_dev(self, W):
        eng = self.eng
        Wd = eng.to_device(W)
        V = self._solve(eng.scatter_points(self.Pp, Wd, Wd.shape[1]))        # A^{-1} P W
        return eng.full_gradient(self.sigma, self.U, V)                       # -sum_j G_j^T v_j

    def apply(self, dm):
        return self.apply_dev(dm).cpu().numpy()

    def rapply(self, W):
        return self.rapply_dev(np.asarray(W, dtype=float) if not hasattr(W, "detach") else W).cpu().numpy()


def sensitivity_full(state, survey):
    """forward.py:284-285."""
    return FullSensitivity(state, survey)


class FullProblem:
    """Fine-mesh forward/sensitivity pair (inversion.py:266-285)."""

    mode = "full"

    def __init__(self, mesh, survey, solver="direct", cg_tol=1e-6, cg_maxit=100):
        self.mesh = mesh
        self.survey = survey
        self.solver = solver
        self.cg_tol = cg_tol
        self.cg_maxit = cg_maxit

    def simulate(self, m):
        from .operators import assemble_operator
        op = assemble_operator(self.mesh, m)
        return forward_full(op, self.survey, solver=self.solver, cg_tol=self.cg_tol, cg_maxit=self.cg_maxit)

    def jacobian(self, state):
        return sensitivity_full(state, self.survey)
