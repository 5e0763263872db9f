"""Stage-by-stage comparison of the 2D GPU path with the 2D oracle (debug helper)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from oracle import msfv_oracle2d as o  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


rng = np.random.default_rng(11)
n1, n2, b1, b2 = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (24, 18, 4, 3))]
mesh = gp.create_mesh_2d(n1, n2, 1.0 / n1, 1.5 / n2)
part = gp.create_partition_2d(mesh, b1, b2)
n = mesh.n_nodes - 1
m = 0.9 * rng.standard_normal(mesh.n_cells)
a = rng.choice(n - 1, 3, replace=False)
Q = sp.csc_matrix((np.r_[np.ones(3), -np.ones(3)], (np.r_[a, a + 1], np.r_[0:3, 0:3])), shape=(n, 3))
P = sp.csc_matrix((np.ones(9), (rng.choice(n, 9, replace=False), np.arange(9))), shape=(n, 9))
om = o.Mesh2D(n1, n2, mesh.h1, mesh.h2)
opart = o.make_partition(om, b1, b2)
op = o.assemble(om, m)
ob = o.build_basis(op, opart)
prob = gp.AdaptiveReducedProblem2D(part, gp.Survey(P=P, Q=Q))
e = prob.engine
D, st = prob.simulate(m)
print("w", rel(st.w.cpu().numpy(), op.w))
k = e.k
S = e.prolong(st.Sb, torch.eye(k, dtype=torch.float64, device="cuda")).cpu().numpy()
So = ob.S.toarray()
print("S", rel(S, So), "per-col max err", np.abs(S - So).max(axis=0)[:6])
bad = np.argwhere(np.abs(S - So) > 1e-8)
print("bad entries", len(bad), bad[:8])
Ak = (So.T @ (op.A @ So))
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
factor, Sb, Kloc = e.basis(st.w, fl)
Ab = e.galerkin(Kloc, 0.0).reshape(k, -1).cpu().numpy()
Akd = np.zeros((k, k))
for c in range(k):
    for d in range(Ab.shape[1]):
        if c - d >= 0:
            Akd[c, c - d] = Akd[c - d, c] = Ab[c, d]
print("A_k", rel(Akd, Ak))
F = e.restrict(st.Sb, torch.from_numpy(np.ascontiguousarray(Q.toarray())).cuda()).cpu().numpy()
print("F", rel(F, So.T @ Q.toarray()))
print("T", rel(st.T, np.linalg.solve(Ak, So.T @ Q.toarray())))
