"""GPU timeline of e2e steps (torch.profiler / CUPTI): busy time, idle gaps
between device activities and the activities on either side of each gap."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

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
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
        ev.append((e.time_range.start, e.time_range.end, e.name))
ev.sort()
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
print(f"span {(t1 - t0) / 3:.1f} us/step, busy {busy / 3:.1f} us/step")
for g, a, b in sorted(gaps, reverse=True)[:15]:
    print(f"gap {g:7.1f} us  after {a[:60]!r}  before {b[:60]!r}")
tot = {}
for s, e, n in ev:
    k = n[:50]
    tot[k] = tot.get(k, 0) + (e - s) / 3
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    print(f"{v:8.1f} us/step  {k}")
