"""Time S_k, Y_k and X_k at the paper's Table-3 geometry:
64x64x32 cells, 16^3-cell coarse blocks (32 blocks, n_I = 3375), 72 sources,
3698 receivers.  Prints one JSON object (device and host-CSR times in ms)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import table3_problem  # noqa: E402


def dev_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
        del out
    return best


def host_ms(fn, reps=2):
    fn()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best


mesh, part, survey, m = table3_problem()
builder = gp.BasisBuilder(part)
m_dev = torch.from_numpy(m).cuda()
op = gp.assemble_operator(mesh, m_dev)
basis = builder.assemble(op)
eng = basis.engine
rng = np.random.default_rng(0)
v = torch.from_numpy(rng.standard_normal(eng.k)).cuda()
w = torch.from_numpy(rng.standard_normal(eng.n)).cuda()
res = {"geometry": "64x64x32 cells, 16^3 blocks (32), n_I 3375, k %d, 72 sources, 3698 receivers" % eng.k}
res["S_k_ms"] = dev_ms(lambda: builder.assemble(gp.assemble_operator(mesh, m_dev)).Sint)
res["Y_k_ms"] = dev_ms(lambda: gp.apply_Yk_dev(basis, v, m_dev))
res["X_k_ms"] = dev_ms(lambda: gp.apply_Xk_dev(basis, w, m_dev))
res["Y_k_nnz"] = int(gp.apply_Yk_dev(basis, v, m_dev)[1].numel())
vh, wh = v.cpu().numpy(), w.cpu().numpy()
res["S_k_host_ms"] = host_ms(lambda: builder.assemble(gp.assemble_operator(mesh, m)).S)
res["Y_k_host_ms"] = host_ms(lambda: gp.apply_Yk(basis, vh, m_dev))
res["X_k_host_ms"] = host_ms(lambda: gp.apply_Xk(basis, wh, m_dev))
prob = gp.AdaptiveReducedProblem(builder, survey)
D, st = prob.simulate(m)
res["forward_gradient_host_ms"] = host_ms(lambda: prob.jacobian(prob.simulate(m)[1]).rapply(D * 0.01))
res["paper_1_worker_s"] = {"S_k": 3.8595, "Y_k": 2.7380, "X_k": 2.9933}
res["paper_8_workers_s"] = {"S_k": 1.4150, "Y_k": 1.0658, "X_k": 1.3818}
print(json.dumps(res))
