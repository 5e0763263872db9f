"""Build the basis at a BASELINE config and check flags / finiteness (debug helper)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.models import config_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh, part, survey, m = config_problem(cfg)
b = gp.BasisBuilder(part)
op = gp.assemble_operator(mesh, m)
basis = b.assemble(op)
torch.cuda.synchronize()
print("basis ok", cfg, "flags", int(basis.flags.item()), "Sint finite", bool(torch.isfinite(basis.Sint).all()))
