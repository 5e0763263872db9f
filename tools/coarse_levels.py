import os, sys
sys.path.insert(0, "/root/repo")
import torch
from torch.profiler import ProfilerActivity, profile
import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.models import config_problem
cfg = int(sys.argv[1])
mesh, part, survey, m = config_problem(cfg)
b = gp.BasisBuilder(part); op = gp.assemble_operator(mesh, m); basis = b.assemble(op); eng = basis.engine
for _ in range(2):
    Ak = eng.galerkin(basis.Kloc, 0.0); fl = eng.flags(); eng.coarse_factor(Ak, fl)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    Ak = eng.galerkin(basis.Kloc, 0.0); fl = eng.flags(); eng.coarse_factor(Ak, fl); torch.cuda.synchronize()
ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start)
for s, e, n in ev: print(f"{e - s:9.1f} us  {n[:50]}")
