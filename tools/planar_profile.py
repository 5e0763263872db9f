"""Per-kernel device times of the 2D path (BASELINE config 1 or 2): one
forward + gradient and one J v / J^T w pair (torch.profiler / CUPTI)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mesh, part, survey, m, d_obs = gp.config_problem_2d(cfg, seed=0)
prob = gp.AdaptiveReducedProblem2D(part, survey)
dev = torch.device("cuda")
m_dev, dobs = torch.from_numpy(m).to(dev), torch.from_numpy(d_obs).to(dev)
rng = np.random.default_rng(1)
V = torch.from_numpy(rng.standard_normal(m.size)).to(dev)
W = torch.from_numpy(rng.standard_normal(d_obs.shape)).to(dev)


def step(products):
    D, st = prob.simulate_dev(m_dev)
    J = prob.jacobian(st)
    g = J.rapply_dev(D - dobs)
    for _ in range(products):
        J.apply_dev(V)
        J.rapply_dev(W)
    return g


for _ in range(3):
    step(1)
torch.cuda.synchronize()
for products, label in ((0, "forward + gradient"), (1, "forward + gradient + one J v + one J^T w")):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step(products)
        torch.cuda.synchronize()
    ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start)
    tot = {}
    for s, e, n in ev:
        k = n[:48]
        tot[k] = tot.get(k, (0.0, 0))
        tot[k] = (tot[k][0] + (e - s), tot[k][1] + 1)
    busy = sum(v[0] for v in tot.values())
    print(f"config {cfg}, {label}: span {ev[-1][1] - ev[0][0]:.0f} us, device busy {busy:.0f} us, {len(ev)} activities")
    for k, v in sorted(tot.items(), key=lambda x: -x[1][0])[:10]:
        print(f"  {v[0]:8.1f} us  x{v[1]:3d}  {k}")
