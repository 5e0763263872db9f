"""Time the Table-3 operators (apply_Yk / apply_Xk, device CSR) at a BASELINE config."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh, part, survey, m = config_problem(cfg)
builder = gp.BasisBuilder(part)
m_dev = torch.from_numpy(m).cuda()
op = gp.assemble_operator(mesh, m_dev)
basis = builder.assemble(op)
rng = np.random.default_rng(0)
v = torch.from_numpy(rng.standard_normal(basis.engine.k)).cuda()
w = torch.from_numpy(rng.standard_normal(basis.engine.n)).cuda()
for name, fn, arg in (("apply_Yk", gp.apply_Yk_dev, v), ("apply_Xk", gp.apply_Xk_dev, w)):
    out = fn(basis, arg, m_dev)
    torch.cuda.synchronize()
    del out
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn(basis, arg, m_dev)
    b.record()
    torch.cuda.synchronize()
    nnz = out[1].numel()
    print(f"{name}: {a.elapsed_time(b):.3f} ms, nnz {nnz}, shape {out[3]}, "
          f"CSR bytes {nnz * 12 + out[0].numel() * 8:,}")
    del out
    torch.cuda.synchronize()
