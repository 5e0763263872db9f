"""Host-side time of each piece of the e2e step (perf_counter stamps, no
extra synchronisation): where the GPU idles between simulate and rapply."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_07598_b200 as gp  # noqa: E402
import paper_1707_07598_b200.forward as F  # noqa: E402
from paper_1707_07598_b200.models import config_problem  # noqa: E402

mesh, part, survey, m = config_problem(4)
problem = gp.AdaptiveReducedProblem(gp.BasisBuilder(part), survey)
d_obs = problem.simulate(m + 0.1)[0]
m_pin = torch.from_numpy(m).pin_memory()
T = {}


def stamp(k, t0):
    T.setdefault(k, []).append((time.perf_counter() - t0) * 1e6)


orig_to_device = gp.engine.Engine.to_device
for it in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D, st = problem.simulate(m_pin)
    stamp("a simulate returned", t0)
    phi, res = gp.misfit_ssd(D, d_obs)
    stamp("b misfit", t0)
    J = problem.jacobian(st)
    stamp("c jacobian", t0)
    eng, b = J.engine, J.basis
    Wd = eng.to_device(res)
    stamp("d W to device", t0)
    y = eng.restrict_points(J.Pp, b.sint_for(J.Pp), Wd, res.shape[1])
    stamp("e restrict launched", t0)
    eng.coarse_solve(st.Lk, y)
    stamp("f coarse solve launched", t0)
    Zc = eng.interior_fields(J.Pp, b.factor, Wd, res.shape[1])
    g = eng.block_gradient_to_host(J.sigma, b.Sint, st.T_dev, y, J.Pp, Zc, J.Qp, J.Rc)
    stamp("g gradient on host", t0)
for k, v in T.items():
    v = np.array(v[10:])
    print(f"{k:28s} median {np.median(v):8.1f} us")
