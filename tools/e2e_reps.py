"""Distribution of the bench e2e leg (K-step repetitions through the public API)."""
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
for _ in range(5):
    D, st = problem.simulate(m_pin)
    problem.jacobian(st).rapply(gp.misfit_ssd(D, d_obs)[1])
gc.collect()
gc.freeze()
torch.cuda.synchronize()
reps = []
for r in range(8):
    t0 = time.perf_counter()
    for _ in range(10):
        D, st = problem.simulate(m_pin)
        phi, res = gp.misfit_ssd(D, d_obs)
        g = problem.jacobian(st).rapply(res)
    reps.append(1e3 * (time.perf_counter() - t0) / 10)
print("e2e ms per step over 8 repetitions:", [round(x, 3) for x in reps], "median", round(float(np.median(reps)), 3))
