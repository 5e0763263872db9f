"""Host timeline of the host-returning rapply (where its wall time goes)."""
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
problem = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
d_obs = problem.simulate(m + 0.1)[0]
m_pin = torch.from_numpy(m).pin_memory()
for _ in range(5):
    D, st = problem.simulate(m_pin)
    problem.jacobian(st).rapply(gp.misfit_ssd(D, d_obs)[1])
gc.collect()
gc.freeze()
T = {}
n = 20
for _ in range(n):
    D, st = problem.simulate(m_pin)
    phi, r = gp.misfit_ssd(D, d_obs)
    J = problem.jacobian(st)
    torch.cuda.synchronize()
    eng, b = J.engine, J.basis
    t0 = time.perf_counter()
    Wd = eng.to_device(np.asarray(r, dtype=float))
    t1 = time.perf_counter()
    y = eng.restrict_points(J.Pp, b.sint_for(J.Pp), Wd, J.survey.n_sources)
    eng.coarse_solve(J.state.Lk, y)
    Zc = eng.interior_fields(J.Pp, b.factor, Wd, J.survey.n_sources)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    g = eng.block_gradient_to_host(J.sigma, b.Sint, J.state.T_dev, y, J.Pp, Zc, J.Qp, J.Rc)
    t4 = time.perf_counter()
    for k, v in (("H2D W", t1 - t0), ("enqueue restrict+solve", t2 - t1), ("drain restrict+solve", t3 - t2),
                 ("gradient+D2H", t4 - t3)):
        T[k] = T.get(k, 0.0) + v
print({k: round(1e3 * v / n, 3) for k, v in T.items()})

# variants of the gradient + copy-back
from paper_1707_07598_b200.forward import _host  # noqa: E402
def timed(name, fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name:36s} median {1e3 * sorted(ts)[n // 2]:.3f} ms")
D, st = problem.simulate(m_pin)
phi, r = gp.misfit_ssd(D, d_obs)
J = problem.jacobian(st)
eng, b = J.engine, J.basis
Wd = eng.to_device(np.asarray(r, dtype=float))
y = eng.restrict_points(J.Pp, b.sint_for(J.Pp), Wd, J.survey.n_sources)
eng.coarse_solve(J.state.Lk, y)
Zc = eng.interior_fields(J.Pp, b.factor, Wd, J.survey.n_sources)
torch.cuda.synchronize()
def dev_only():
    g = eng.block_gradient(J.sigma, b.Sint, J.state.T_dev, y, J.Pp, Zc, J.Qp, J.Rc)
    torch.cuda.synchronize()
    return g
timed("gradient kernel only (+sync)", dev_only)
timed("gradient + _host (one copy)", lambda: _host(eng.block_gradient(J.sigma, b.Sint, J.state.T_dev, y, J.Pp, Zc, J.Qp, J.Rc)))
for c in (1, 2, 4, 8):
    timed(f"slab copies, {c} chunks", lambda c=c: eng.block_gradient_to_host(J.sigma, b.Sint, J.state.T_dev, y, J.Pp, Zc, J.Qp, J.Rc, chunks=c))
