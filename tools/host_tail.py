"""Host time between the end of one e2e step and the first model copy of
the next (patches the engine entry points with perf_counter stamps)."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200 import engine as E  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

st = {}
orig_bp, orig_bg = E.Engine.build_pipelined, E.Engine.block_gradient_to_host


def bp(self, *a, **k):
    st["bp_in"] = time.perf_counter()
    return orig_bp(self, *a, **k)


def bg(self, *a, **k):
    r = orig_bg(self, *a, **k)
    st["bg_out"] = time.perf_counter()
    return r


E.Engine.build_pipelined, E.Engine.block_gradient_to_host = bp, bg
mesh, part, survey, m = config_problem(4)
problem = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
d_obs = problem.simulate(m + 0.1)[0]
m_pin = torch.from_numpy(m).pin_memory()
for _ in range(6):
    D, s = problem.simulate(m_pin)
    problem.jacobian(s).rapply(gp.misfit_ssd(D, d_obs)[1])
gc.collect()
gc.freeze()
acc = {"rapply tail -> loop": 0.0, "simulate entry -> build_pipelined": 0.0, "simulate": 0.0,
       "misfit+jacobian()": 0.0, "rapply (incl. wait)": 0.0}
n = 20
for _ in range(n):
    t0 = time.perf_counter()
    D, s = problem.simulate(m_pin)
    t1 = time.perf_counter()
    acc["simulate entry -> build_pipelined"] += st["bp_in"] - t0
    acc["simulate"] += t1 - t0
    phi, r = gp.misfit_ssd(D, d_obs)
    J = problem.jacobian(s)
    t2 = time.perf_counter()
    acc["misfit+jacobian()"] += t2 - t1
    g = J.rapply(r)
    t3 = time.perf_counter()
    acc["rapply (incl. wait)"] += t3 - t2
    acc["rapply tail -> loop"] += t3 - st["bg_out"]
print({k: round(1e6 * v / n, 1) for k, v in acc.items()}, "us")
