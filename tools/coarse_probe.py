"""Time the coarse factor / solve alone at a BASELINE config (debug helper)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.models import config_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh, part, survey, m = config_problem(cfg)
b = gp.BasisBuilder(part)
op = gp.assemble_operator(mesh, m)
basis = b.assemble(op)
eng = basis.engine
print("k", eng.k, "NT", eng.NT, "PT", eng.PT, "ak_doubles", eng.ak_doubles, flush=True)
for it in range(3):
    Ak = eng.galerkin(basis.Kloc, 0.0)
    fl = eng.flags()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); c = torch.cuda.Event(enable_timing=True)
    a.record(); eng.coarse_factor(Ak, fl); c.record(); torch.cuda.synchronize()
    X = torch.randn(eng.k, 16, dtype=torch.float64, device="cuda")
    d = torch.cuda.Event(enable_timing=True); d.record(); eng.coarse_solve(Ak, X); e = torch.cuda.Event(enable_timing=True); e.record()
    torch.cuda.synchronize()
    print(f"factor {a.elapsed_time(c):.3f} ms  solve {d.elapsed_time(e):.3f} ms flags {int(fl.item())}", flush=True)
