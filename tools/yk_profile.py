"""Per-kernel device times of apply_Yk_dev / apply_Xk_dev at a BASELINE config
(torch.profiler / CUPTI) with the algorithmic bytes each kernel moves."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402
from paper_1707_07598_b200.table3 import apply_Xk_dev, apply_Yk_dev  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh, part, survey, m = config_problem(cfg)
op = gp.assemble_operator(mesh, m)
basis = gp.BasisBuilder(part).assemble(op)
eng = basis.engine
rng = np.random.default_rng(0)
v = rng.normal(size=eng.k)
w = rng.normal(size=eng.n)
for _ in range(2):
    Y = apply_Yk_dev(basis, v, m)
    X = apply_Xk_dev(basis, w, m)
    del Y, X
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    Y = apply_Yk_dev(basis, v, m)
    torch.cuda.synchronize()
nnz = Y[2].numel()
ncb = part.b1 * part.b2 * part.b3
wide = eng.nbl * eng.nI * ncb * 8
fac = eng.factor_doubles * 8
alg = {"k_yk_rhs": wide, "k_lg_solve": 2 * wide + fac * ((ncb + 127) // 128), "k_yk_scatter": wide + nnz * 12,
       "k_yk_rowcount": eng.Nn * 8}
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
        tot[e.name] = tot.get(e.name, 0.0) + (e.time_range.end - e.time_range.start)
print(f"config {cfg}: Y_k nnz {nnz} ({nnz * 12 / 1e9:.2f} GB of CSR), wide right-hand sides {wide / 1e9:.2f} GB, "
      f"factor {fac / 1e9:.2f} GB")
print("| kernel | ms | algorithmic GB | GB/s |")
print("|---|---|---|---|")
for k, us in sorted(tot.items(), key=lambda x: -x[1])[:8]:
    key = next((a for a in alg if a in k), None)
    gb = alg[key] / 1e9 if key else float("nan")
    print(f"| `{k[:60]}` | {us / 1e3:.3f} | {gb:.2f} | {gb / (us / 1e6):.0f} |")
print(f"total device time {sum(tot.values()) / 1e3:.2f} ms")
