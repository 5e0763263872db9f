"""Print per-quantity relative errors of the GPU path vs the golden vectors."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402

from conftest import GOLDEN_CASES, load_golden, rel  # noqa: E402
from test_gpu_parity import build_gpu  # noqa: E402

for name in GOLDEN_CASES:
    g = load_golden(name)
    try:
        gp, mesh, part, survey, builder = build_gpu(g)
        t0 = time.time()
        op = gp.assemble_operator(mesh, g["m"])
        basis = builder.assemble(op)
        D, state = gp.forward_reduced(op, survey, basis)
        e = {"w": rel(op.edge_weights, g["w"])}
        S = basis.S
        e["Spat"] = bool(np.array_equal(S.indptr, g["S_indptr"]) and np.array_equal(S.indices, g["S_indices"]))
        if e["Spat"]:
            e["S"] = rel(S.data, g["S_data"])
        e["T"] = rel(state.T, g["T"])
        e["D"] = rel(D, g["D"])
        if "A_k" in g:
            e["Ak"] = rel(state.A_k, g["A_k"])
        phi, resid = gp.misfit_ssd(D, g["d_obs"])
        J = gp.sensitivity_adaptive(state, survey)
        e["g"] = rel(J.rapply(resid), g["g"])
        e["Jv"] = rel(J.apply(g["dm"]), g["Jv"])
        e["JtW"] = rel(J.rapply(g["W"]), g["JtW"])
        print(name, {k: (f"{v:.2e}" if isinstance(v, float) else v) for k, v in e.items()},
              f"{time.time() - t0:.2f}s", flush=True)
    except Exception as ex:  # noqa: BLE001
        import traceback
        traceback.print_exc()
        print(name, "FAILED", repr(ex), flush=True)
