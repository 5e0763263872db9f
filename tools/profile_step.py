"""One warm-up + one measured forward+gradient step at a BASELINE config
(target for ncu; no timing of its own)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.forward import forward_reduced_dev, sensitivity_adaptive  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mesh, part, survey, m = config_problem(cfg)
builder = gp.BasisBuilder(part)
m_dev = torch.from_numpy(m).cuda()
with_jv = len(sys.argv) > 3 and sys.argv[3] == "jv"
for _ in range(steps):
    op = gp.assemble_operator(mesh, m_dev)
    basis = builder.assemble(op)
    D, st = forward_reduced_dev(op, survey, basis)
    J = sensitivity_adaptive(st, survey)
    g = J.rapply_dev(D)
    if with_jv:                     # one CG-step pair of the config-4 GN iteration
        jv = J.apply_dev(g)
        g = J.rapply_dev(jv)
torch.cuda.synchronize()
print("profile_step done", float(g.norm()))
