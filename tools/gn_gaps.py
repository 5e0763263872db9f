"""GPU timeline of one device-resident Gauss-Newton iteration at config 4
(torch.profiler / CUPTI): busy time, idle gaps, per-kernel totals."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

mesh, part, survey, m = config_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
problem = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
d_obs = problem.simulate(m + 0.1)[0]
obj = gp.DeviceObjective(mesh, 1e-3, np.zeros(mesh.n_cells))
cfg = gp.GNSettings(max_gn=1, max_cg=5)


def it():
    return gp.gauss_newton_dev(problem, m, d_obs, obj, cfg)


for _ in range(3):
    it()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    it()
    torch.cuda.synchronize()
ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start)
t0, t1 = ev[0][0], ev[-1][1]
busy, cur_s, cur_e, last = 0.0, ev[0][0], ev[0][1], ev[0][2]
gaps = []
for s, e, n in ev[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, last, n))
        cur_s, cur_e = s, e
    elif e > cur_e:
        cur_e = e
    if e >= cur_e:
        last = n
busy += cur_e - cur_s
print(f"span {(t1 - t0):.1f} us, busy {busy:.1f} us, {len(ev)} device activities, gaps > 20 us: "
      f"{sum(1 for g in gaps if g[0] > 20)} totalling {sum(g[0] for g in gaps if g[0] > 20):.0f} us")
for g, a, b in sorted(gaps, reverse=True)[:12]:
    print(f"gap {g:7.1f} us  after {a[:50]!r}  before {b[:50]!r}")
tot = {}
for s, e, n in ev:
    k = n[:50]
    tot[k] = tot.get(k, (0, 0))
    tot[k] = (tot[k][0] + (e - s), tot[k][1] + 1)
for k, v in sorted(tot.items(), key=lambda x: -x[1][0])[:22]:
    print(f"{v[0]:8.1f} us  x{v[1]:3d}  {k}")
