"""Time forward_full(direct) at a BASELINE config (two-level preconditioned PCG)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh, part, survey, m = config_problem(cfg)
prob = gp.FullProblem(mesh, survey)
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D, st = prob.simulate(m)
    torch.cuda.synchronize()
    print(f"fine forward {time.perf_counter() - t0:.3f} s, iterations {st.factor.last.iterations}")
