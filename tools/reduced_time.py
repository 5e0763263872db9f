"""Event-timed forward + gradient with the reduced boundary conditions at a
BASELINE config (extension N4): forward (basis with reduced skeleton data,
coarse solve), ReducedSensitivity set-up, J^T W, J v."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.forward import forward_reduced_dev  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh, part, survey, m = config_problem(cfg)
builder = gp.BasisBuilder(part, gp.BasisSpec(boundary="reduced"))
m_dev = torch.from_numpy(m).cuda()
rng = np.random.default_rng(0)
v = torch.from_numpy(rng.normal(size=m.size)).cuda()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2], out


def fwd():
    op = gp.assemble_operator(mesh, m_dev)
    basis = builder.assemble(op)
    return forward_reduced_dev(op, survey, basis)


t_f, (D, st) = timed(fwd)
t_s, J = timed(lambda: gp.sensitivity_adaptive(st, survey))
W = torch.randn_like(D)
t_r, g = timed(lambda: J.rapply_dev(W))
t_a, jv = timed(lambda: J.apply_dev(v))
lhs, rhs = float((jv * W).sum()), float(torch.dot(v, g))
print(f"config {cfg} reduced BCs: forward {t_f:.2f} ms, sensitivity set-up {t_s:.2f} ms, J^T W {t_r:.2f} ms, "
      f"J v {t_a:.2f} ms; adjoint identity {abs(lhs - rhs) / abs(lhs):.1e}")
