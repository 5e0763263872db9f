import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.forward import forward_reduced_dev
from paper_1707_07598_b200.models import config_problem
mesh, part, survey, m = config_problem(4)
builder = gp.BasisBuilder(part, gp.BasisSpec(boundary="reduced"))
m_dev = torch.from_numpy(m).cuda()
op = gp.assemble_operator(mesh, m_dev)
D, st = forward_reduced_dev(op, survey, builder.assemble(op))
J = gp.sensitivity_adaptive(st, survey)
W = torch.randn_like(D)
for _ in range(2): J.rapply_dev(W)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    J.rapply_dev(W); torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
        tot[e.name[:70]] = tot.get(e.name[:70], (0,0)); tot[e.name[:70]] = (tot[e.name[:70]][0] + e.time_range.end - e.time_range.start, tot[e.name[:70]][1]+1)
for k, v in sorted(tot.items(), key=lambda x: -x[1][0])[:18]: print(f"{v[0]/1e3:8.3f} ms x{v[1]:3d} {k}")
print("total device", sum(v[0] for v in tot.values())/1e3)
