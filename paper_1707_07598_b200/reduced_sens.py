"""Sensitivity of the adaptive reduced map with reduced-dimension boundary
conditions (extension N4; the reference has no such basis,
SPEC.md:328 -- its AdaptiveSensitivity, forward.py:209-281, is the B-fixed
part of what follows).

With the skeleton data B(w) depending on the model, S = [B ; -A_II^-1 A_IB B]
changes through A (the reference's terms) and through B.  For a data-space
vector W, with T = A_k^-1 S^T Q, y = A_k^-1 S^T P W, U = S T, R = Q - A U,
Rw = P W - A S y, z_R = interior_solve(R), z = interior_solve(Rw):

  J^T W = -Csig^T [ sum_s G U o G z + G z_R o G S y + G U o G S y ]       (forward.py:270-281)
          + Csig^T d<B(w), Lam>/dw,
  Lam = (R - A z_R)_B y^T + (Rw - A z)_B T^T       on the pattern of B,

since <dS|_A, R y^T + Rw T^T> = <dB, Z_B - A_BI A_II^-1 Z_I>.  For J v, with
dw = Csig v and dB = B'(w) dw, the node field f = dB T (skeleton rows) extends
to delta = f - interior_solve(A f), and

  A_k dT = [reference terms] + dB^T (R - A z_R)_B - S^T A delta,
  J v    = P^T (S dT + y_dm + delta).

The skeleton map and its two derivatives are paper_1707_07598_b200.skeleton
(batched tensor formulas); every mesh-sized operation is a libmsfv kernel
(edge_grad / edge_div / fine_apply / interior_solve / restrict / prolong /
coarse solve / cell_gather) on node and edge fields.  There is no CPU path.
"""

import numpy as np
import torch

from .skeleton import SkeletonMap


def _host(t):
    return t.detach().cpu().numpy()


class ReducedSensitivity:
    """AdaptiveSensitivity for a basis built with BasisSpec(boundary="reduced")."""

    mode = "ms_adaptive"

    def __init__(self, state, survey, workers=1):
        op, basis = state.op, state.basis
        eng = basis.engine
        if not getattr(state, "deferred", False):
            state.check()
        if op._dev is None or op._dev[1] is not basis._m_dev:
            basis.check_model(op.m)
        self.state, self.survey, self.basis, self.engine = state, survey, basis, eng
        self.workers = workers
        _, _, self.sigma, self.w = op.device_state(eng)
        self.Pp, self.Qp, self.Qf = survey.device(eng)
        self.skel = SkeletonMap.get(basis.partition, eng.device)
        self.nodes, self.cols = self.skel.entries()
        eng.bind_boundary(basis.bx)
        self.T = state.T_dev
        self.U = eng.prolong(basis.Sint, self.T.contiguous())                           # S T
        self.gu = eng.edge_grad(self.U)                                                  # G_p S T
        R = self.Qf - eng.fine_apply(self.w, self.U)                                     # Q - A S T
        ZR = self._interior(R)
        self.a = eng.edge_grad(ZR)                                                       # G_p interior_solve(R)
        self.Rt = R - eng.fine_apply(self.w, ZR)                                         # (R - A z_R): skeleton rows used

    def _interior(self, X):
        out = self.engine.zeros(*X.shape)
        self.engine.interior_solve(self.basis.factor, X.contiguous(), out)
        return out

    def _restrict(self, X):
        return self.engine.restrict_op(self.basis.Sint, None, X.contiguous(), None, None, X.shape[1])

    def _solve(self, X):
        X = X.contiguous().clone()
        self.engine.coarse_solve(self.state.Lk, X)
        return X

    # ------------------------------------------------------------------ J^T W
    def rapply_dev(self, W):
        eng, b = self.engine, self.basis
        ns = self.survey.n_sources
        eng.bind_boundary(b.bx)
        W = eng.to_device(W)
        p = eng.scatter_points(self.Pp, W, ns)                                           # P W
        y = self._solve(self._restrict(p))
        sy = eng.prolong(b.Sint, y)
        rw = p - eng.fine_apply(self.w, sy)                                              # P W - A S y
        z = self._interior(rw)
        gsy = eng.edge_grad(sy)
        xi = (self.gu * eng.edge_grad(z) + self.a * gsy + self.gu * gsy).sum(dim=1)     # forward.py:278-280
        # boundary term: Lam = (R - A z_R)_B y^T + (Rw - A z)_B T^T on the entries of B
        rwt = rw - eng.fine_apply(self.w, z)
        lam = self.skel.contract(self.Rt, y) + self.skel.contract(rwt, self.T)
        xi = xi - self.skel.vjp(self.w, lam)
        return eng.cell_gather(self.sigma, xi)

    # -------------------------------------------------------------------- J v
    def apply_dev(self, dm):
        eng, b = self.engine, self.basis
        ns = self.survey.n_sources
        eng.bind_boundary(b.bx)
        dm = eng.to_device(dm).reshape(-1)
        dw = eng.edge_average(self.sigma, dm)                                            # Csig dm (forward.py:259)
        c = dw[:, None]
        ydm = -self._interior(eng.edge_div((self.gu * c).contiguous()))                  # dS_I T at fixed B
        xdm = -self._restrict(eng.edge_div((self.a * c).contiguous()))
        gdm = eng.edge_div((self.gu * c).contiguous())
        rhs = xdm - self._restrict(gdm + eng.fine_apply(self.w, ydm))
        # boundary term
        dB = self.skel.jvp(self.w, dw)
        f = self.skel.spread_nodes(dB, self.T, eng.Nn)                                   # dB T on the skeleton
        delta = f - self._interior(eng.fine_apply(self.w, f))
        extra = self.skel.spread_cols(dB, self.Rt, eng.k)                                # dB^T (R - A z_R)_B
        rhs = rhs + extra - self._restrict(eng.fine_apply(self.w, delta))
        dt = self._solve(rhs)
        field = (ydm + delta).contiguous()
        return eng.receive(self.Pp, b.Sint, Y=dt.contiguous(), Xfield=field)

    def apply(self, dm):
        return _host(self.apply_dev(dm))

    def rapply(self, W):
        return _host(self.rapply_dev(np.asarray(W, dtype=float) if not hasattr(W, "detach") else W))
