"""Break down the end-to-end step (host copies, syncs) of bench.py's e2e leg."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

mesh, part, survey, m = config_problem(4)
builder = gp.BasisBuilder(part)
problem = gp.AdaptiveReducedProblem(builder, survey)
d_obs = problem.simulate(m + 0.1)[0]
m_pin = torch.from_numpy(m).pin_memory()
x = torch.empty(m.size, dtype=torch.float64, device="cuda")
buf = torch.empty(m.size, dtype=torch.float64, pin_memory=True)
for name, fn in (("H2D 16.8 MB pinned", lambda: x.copy_(m_pin, non_blocking=True)),
                 ("D2H 16.8 MB pinned", lambda: buf.copy_(x, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"{name}: {ms:.3f} ms ({m.nbytes / ms / 1e6:.1f} GB/s)")
for _ in range(3):
    D, st = problem.simulate(m_pin)
    phi, r = gp.misfit_ssd(D, d_obs)
    problem.jacobian(st).rapply(r)
gc.collect(); gc.freeze()
torch.cuda.synchronize()
T = {"simulate": 0.0, "misfit": 0.0, "jac+rapply": 0.0}
n = 20
t_all = time.perf_counter()
for _ in range(n):
    t0 = time.perf_counter()
    D, st = problem.simulate(m_pin)
    t1 = time.perf_counter()
    phi, r = gp.misfit_ssd(D, d_obs)
    t2 = time.perf_counter()
    g = problem.jacobian(st).rapply(r)
    t3 = time.perf_counter()
    T["simulate"] += t1 - t0; T["misfit"] += t2 - t1; T["jac+rapply"] += t3 - t2
print("wall per step %.3f ms" % (1e3 * (time.perf_counter() - t_all) / n), {k: round(1e3 * v / n, 3) for k, v in T.items()})

# host-side enqueue cost of the pieces (no sync inside)
from paper_1707_07598_b200.forward import forward_reduced_dev, sensitivity_adaptive  # noqa: E402
m_dev = torch.from_numpy(m).cuda()
for _ in range(3):
    op = gp.assemble_operator(mesh, m_dev); basis = builder.assemble(op)
    Dd, st = forward_reduced_dev(op, survey, basis, defer_check=True); st.deferred = True
    J = sensitivity_adaptive(st, survey); J.rapply_dev(Dd)
torch.cuda.synchronize()
H = {}
for _ in range(20):
    t0 = time.perf_counter(); op = gp.assemble_operator(mesh, m_dev); basis = builder.assemble(op)
    t1 = time.perf_counter(); Dd, st = forward_reduced_dev(op, survey, basis, defer_check=True); st.deferred = True
    t2 = time.perf_counter(); J = sensitivity_adaptive(st, survey)
    t3 = time.perf_counter(); gg = J.rapply_dev(Dd)
    t4 = time.perf_counter(); torch.cuda.synchronize(); t5 = time.perf_counter()
    for k, v in (("operator+basis", t1 - t0), ("forward", t2 - t1), ("sens init", t3 - t2), ("rapply", t4 - t3), ("drain", t5 - t4)):
        H[k] = H.get(k, 0.0) + v
print("host enqueue ms:", {k: round(1e3 * v / 20, 3) for k, v in H.items()})
