"""Host-side cost of the e2e leg's pieces (no device sync inside): where the
GPU waits on Python between simulate() and rapply()."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

mesh, part, survey, m = config_problem(4)
problem = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
d_obs = problem.simulate(m + 0.1)[0]
m_pin = torch.from_numpy(m).pin_memory()
for _ in range(6):
    D, st = problem.simulate(m_pin)
    problem.jacobian(st).rapply(gp.misfit_ssd(D, d_obs)[1])
gc.collect()
gc.freeze()
torch.cuda.synchronize()
T = {}
n = 20
for _ in range(n):
    t0 = time.perf_counter()
    D, st = problem.simulate(m_pin)           # ends with a host copy of D (sync)
    t1 = time.perf_counter()
    phi, r = gp.misfit_ssd(D, d_obs)
    t2 = time.perf_counter()
    J = problem.jacobian(st)
    t3 = time.perf_counter()
    g = J.rapply(r)
    t4 = time.perf_counter()
    for k, v in (("simulate", t1 - t0), ("misfit", t2 - t1), ("jacobian()", t3 - t2), ("rapply", t4 - t3)):
        T[k] = T.get(k, 0.0) + v
print({k: round(1e3 * v / n, 3) for k, v in T.items()}, "total", round(1e3 * sum(T.values()) / n, 3))
# enqueue-only cost of simulate's launches (device busy: no waiting)
torch.cuda.synchronize()
t0 = time.perf_counter()
from paper_1707_07598_b200.inversion import _pipelined_build  # noqa: E402
op, basis = _pipelined_build(part, m_pin)
t1 = time.perf_counter()
from paper_1707_07598_b200.forward import forward_reduced_dev  # noqa: E402
Dd, st2 = forward_reduced_dev(op, survey, basis, defer_check=True)
t2 = time.perf_counter()
torch.cuda.synchronize()
t3 = time.perf_counter()
print("enqueue ms: pipelined build %.3f, forward chain %.3f, drain %.3f" % (1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)))
