"""cProfile of the host side of the e2e step (simulate -> misfit_ssd ->
jacobian().rapply with pinned host m): where the Python time between the
device activities goes."""
import cProfile
import io
import os
import pstats
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

mesh, part, survey, m = config_problem(4)
problem = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
d_obs = problem.simulate(m + 0.1)[0]
m_pin = torch.from_numpy(m).pin_memory()


def step():
    D, st = problem.simulate(m_pin)
    phi, res = gp.misfit_ssd(D, d_obs)
    return problem.jacobian(st).rapply(res)


for _ in range(6):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
pr.disable()
torch.cuda.synchronize()
for key in ("tottime", "cumtime"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(key).print_stats(28)
    print(s.getvalue()[:6000])
