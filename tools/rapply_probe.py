"""Wall time of the host-returning rapply variants (e2e gradient leg)."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
from paper_1707_07598_b200.forward import _host  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

mesh, part, survey, m = config_problem(4)
problem = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
D, st = problem.simulate(m)
J = problem.jacobian(st)
r = D * 0.01
eng = J.engine
gc.collect()
gc.freeze()


def variant(name, fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        out = fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {1e3 * (time.perf_counter() - t0) / n:.3f} ms")
    return out


ref = variant("rapply (current)", lambda: J.rapply(r))
old = variant("_host(rapply_dev)", lambda: _host(J.rapply_dev(r)))
dev = variant("rapply_dev + sync", lambda: J.rapply_dev(r))
for c in (1, 2, 4, 8):
    b = J.basis
    def f(c=c):
        Wd = eng.to_device(r)
        y = eng.restrict_points(J.Pp, b.sint_for(J.Pp), Wd, J.survey.n_sources)
        eng.coarse_solve(J.state.Lk, y)
        Zc = eng.interior_fields(J.Pp, b.factor, Wd, J.survey.n_sources)
        return eng.block_gradient_to_host(J.sigma, b.Sint, J.state.T_dev, y, J.Pp, Zc, J.Qp, J.Rc, chunks=c)
    o = variant(f"slab copies, {c} chunks", f)
    print("  max diff", float(np.abs(o - old).max()))
