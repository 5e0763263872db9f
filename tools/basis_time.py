"""Event-timed basis_forward (k_basis_tc + k_skel_galerkin) at a BASELINE
config, for each MSFV_BASIS_VARIANT given on the command line (the variant is
read at every launch).  Checks that every variant reproduces variant 1's
Galerkin blocks and parked y bit-for-bit or to 1e-13.

usage: python tools/basis_time.py [CFG] [VARIANTS e.g. 0,1,2,3]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
variants = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,3").split(",")]
mesh, part, survey, m = config_problem(cfg)
builder = gp.BasisBuilder(part)
op = gp.assemble_operator(mesh, torch.from_numpy(m).cuda())
eng = builder.assemble(op).engine
w = op.device_state(eng)[3]
ref = None
for v in variants:
    os.environ["MSFV_BASIS_VARIANT"] = str(v)
    for _ in range(3):
        out = eng.basis_forward(w)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = eng.basis_forward(w)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    factor, Sint, Kloc, fl = out
    if ref is None:
        ref = (Sint.clone(), Kloc.clone())
    eS = float((Sint - ref[0]).norm() / ref[0].norm())
    eK = float((Kloc - ref[1]).norm() / ref[1].norm())
    print(f"variant {v}: basis_forward median {ts[len(ts) // 2]:.4f} ms  min {ts[0]:.4f} ms  "
          f"flags {int(fl.item())}  rel diff vs first: y {eS:.1e} K {eK:.1e}")
