import os, sys, cProfile, pstats, io
sys.path.insert(0, os.getcwd())
import torch
import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.models import config_problem
mesh, part, survey, m = config_problem(4)
builder = gp.BasisBuilder(part)
m_dev = torch.from_numpy(m).cuda()
for _ in range(3):
    op = gp.assemble_operator(mesh, m_dev); basis = builder.assemble(op)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(50):
    op = gp.assemble_operator(mesh, m_dev); basis = builder.assemble(op)
pr.disable()
torch.cuda.synchronize()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats('tottime').print_stats(15); print(s.getvalue()[:3500])
