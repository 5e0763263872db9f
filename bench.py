#!/usr/bin/env python
"""Benchmark: adaptive MSFV forward + gradient on BASELINE.json config 4.

Contract (one JSON line from rank 0):
  step   = one forward + misfit + gradient (J^T r) of the adaptive MSFV reduced
           model: A(m), basis P(m) (all local block solves), Galerkin A_k,
           coarse factor + solve, D = P^T S T, misfit, sensitivity init and
           rapply.  Metric "MSFV forward+gradient s/iter" (lower is better).
  value  = device-timed seconds per step (CUDA events, inputs resident in HBM)
           divided by the number of replicas (whole-job aggregate).
  e2e    = same step through the public drop-in API with host buffers
           (pinned m in, D and g back to host), H2D/D2H inside the timed region.
Workload: 128^3 cells, 8^3-cell blocks (4096 local solves), 16 dipoles,
1024 receivers, m = 1.5 * smoothed GRF (sigma 6 cells), seed 0.  Every buffer
of the step (factors ~1.1 GB) exceeds the 126 MB L2, so no flush is needed.

--impl reference runs the CPU oracle port (oracle/, a numpy/scipy
restatement of the reference msinv path) on the full workload, every step
(config 4: about 15-20 s per step on the GPU box's host cores).
"""

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MSFV forward+gradient s/iter"
UNIT = "s/iter"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (1-2: the 2D path, 3-5: 3D)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gn", action="store_true", help="skip the Gauss-Newton iteration timing")
    ap.add_argument("--no-table3", action="store_true", help="skip the Table-3 geometry timings")
    ap.add_argument("--ncu", action="store_true",
                    help="profiling mode: device-resident setup, then only the guard, warm-up and timed steps "
                         "(no extra legs), so an ncu launch list ends with the last timed step")
    return ap.parse_args()


def workload_config_2d(cfg_id):
    if cfg_id == 1:
        return {"workload": "BASELINE config 1: 2D 64^2 cells, 8^2-cell blocks (64 local block solves), 1 dipole, "
                            "32 receivers on row 60, adaptive Lagrange MSFV forward+misfit+gradient at m = 0, "
                            "d_obs from the fine-grid solve at m_true",
                "mesh": [64, 64], "blocks": [8, 8], "n_blocks": 64, "k_coarse": 81, "n_sources": 1,
                "n_receivers": 32, "model": "two +-1 rectangles + N(0, 0.1^2), seed 0 (m_true); m = 0",
                "l2": "working set < L2 (2D config is small); no flush", "parallelism": "replicas"}
    return {"workload": "BASELINE config 2: 2D 256^2 cells, 16^2-cell blocks (256 local block solves), 16 dipoles, "
                        "128 receivers on row 255, adaptive Lagrange MSFV forward+misfit+gradient "
                        "+ 10 J v + 10 J^T v (v ~ N(0,1), seed+1)",
            "mesh": [256, 256], "blocks": [16, 16], "n_blocks": 256, "k_coarse": 289, "n_sources": 16,
            "n_receivers": 128, "model": "GRF(sigma=8 cells, std 1), seed 0; d_obs from the fine-grid solve",
            "l2": "working set < L2 (2D config is small); no flush", "parallelism": "replicas"}


def oracle2d_time(cfg_id, seed, reps=1, warm=1, log=None, workers=1):
    """CPU 2D oracle (oracle/msfv_oracle2d.py) on the full config-1/2 step."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    from oracle import msfv_oracle as o3
    from oracle import msfv_oracle2d as o
    from paper_1707_07598_b200.planar import config_problem_2d
    o3.WORKERS = workers
    mesh, part, survey, m, d_obs = config_problem_2d(cfg_id, seed)
    om = o.Mesh2D(mesh.n1, mesh.n2, mesh.h1, mesh.h2)
    prob = o.AdaptiveProblem(o.make_partition(om, part.b1, part.b2), o.Survey(survey.P, survey.Q))
    rng = np.random.default_rng(seed + 1)
    n_prod = 10 if cfg_id == 2 else 0
    V = rng.standard_normal((n_prod, m.size))
    W = rng.standard_normal((n_prod,) + d_obs.shape)
    ts = []
    for it in range(warm + reps):
        t0 = time.perf_counter()
        D, st = prob.simulate(m)
        phi, r = o.misfit(D, d_obs)
        J = prob.jacobian(st)
        J.rapply(r)
        for i in range(n_prod):
            J.apply(V[i])
            J.rapply(W[i])
        dt = time.perf_counter() - t0
        if it >= warm:
            ts.append(dt)
        if log:
            log(f"2D oracle iteration {it}: {dt:.3f} s")
    desc = (f"2D oracle (numpy/scipy restatement of the msinv algorithm with d = 2; the reference is 3D only), "
            f"{workers} worker thread(s) over blocks, OPENBLAS_NUM_THREADS=1, full config {cfg_id} step")
    return float(np.median(ts)), desc


def run_2d(args, log):
    """BASELINE configs 1-2 on the 2D path (paper_1707_07598_b200.planar)."""
    import numpy as np
    import torch
    import paper_1707_07598_b200 as gp
    from paper_1707_07598_b200 import _lib
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    mesh, part, survey, m, d_obs = gp.config_problem_2d(args.config, seed=args.seed)
    prob = gp.AdaptiveReducedProblem2D(part, survey)
    dev = torch.device("cuda")
    rng = np.random.default_rng(args.seed + 1)
    n_prod = 10 if args.config == 2 else 0
    Vh = rng.standard_normal((n_prod, m.size))
    Wh = rng.standard_normal((n_prod,) + d_obs.shape)
    m_dev, dobs = torch.from_numpy(m).to(dev), torch.from_numpy(d_obs).to(dev)
    V, W = torch.from_numpy(Vh).to(dev), torch.from_numpy(Wh).to(dev)
    L = _lib.load()

    def step_dev():
        D, st = prob.simulate_dev(m_dev)
        r = D - dobs
        phi = 0.5 * torch.sum(r * r)
        J = prob.jacobian(st)
        g = J.rapply_dev(r)
        for i in range(n_prod):
            J.apply_dev(V[i])
            J.rapply_dev(W[i])
        return phi, g

    phi0, g0 = step_dev()
    assert torch.isfinite(phi0).item() and torch.isfinite(g0).all().item()
    for _ in range(args.warmup):
        step_dev()
    torch.cuda.synchronize()
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", 0)))
    clocks.start()
    time.sleep(0.3)
    n0 = L.msfv_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step_dev()
    e1.record()
    torch.cuda.synchronize()
    launches = L.msfv_launch_count() - n0
    ms = e0.elapsed_time(e1) / args.steps
    clk = clocks.stop()
    log(f"2D device step {ms:.3f} ms")
    # e2e through the public API with host arrays
    m_pin = torch.from_numpy(m).pin_memory()

    def step_host():
        D, st = prob.simulate(m_pin)
        phi, r = gp.misfit_ssd(D, d_obs)
        J = prob.jacobian(st)
        g = J.rapply(r)
        for i in range(n_prod):
            J.apply(Vh[i])
            J.rapply(Wh[i])
        return D, g

    for _ in range(max(1, args.warmup)):
        step_host()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        D, g = step_host()
    b.record()
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / args.steps
    h2d = m.nbytes + d_obs.nbytes + Vh.nbytes + Wh.nbytes
    d2h = D.nbytes + g.nbytes + n_prod * (D.nbytes + g.nbytes)
    # dominant kernel: the per-block basis build (band Cholesky + 4 solves)
    PhaseT = torch.cuda.Event
    e = prob.engine
    sig, w, fl = e.operator(m_dev)
    for _ in range(3):
        e.basis(w, fl)
    ta, tb = PhaseT(enable_timing=True), PhaseT(enable_timing=True)
    ta.record()
    for _ in range(10):
        e.basis(w, fl)
    tb.record()
    torch.cuda.synchronize()
    t_basis = ta.elapsed_time(tb) / 10 / 1e3
    nI, p = e.nI, part.b1 - 1
    fl_block = basis_flops(nI, p, r=4, n_edges=0, sweeps=2)
    peak, peak_src = fp64_peak()
    achieved = fl_block * e.nbl / t_basis / 1e12
    roof = {"kernel": "k2_basis + k2_galerkin (one CTA per block: band Cholesky of A_II in shared memory, "
                      "4 Lagrange solves; local Galerkin)", "bound": "fp64", "achieved": round(achieved, 5),
            "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 6), "traffic": None,
            "flops_per_block": fl_block, "blocks_per_launch": e.nbl, "launch_ms": round(t_basis * 1e3, 4),
            "peak_source": peak_src,
            "note": "2D configs are latency-bound (64/256 blocks, one barrier chain per pivot); reported for completeness"}
    e2e = {"value": e2e_ms / 1e3, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "ms_per_step": round(e2e_ms, 4),
           "path": "AdaptiveReducedProblem2D.simulate -> misfit_ssd -> jacobian(state).rapply/apply (numpy)"}
    return {"ms": ms, "launches": launches, "clocks": clk, "e2e": e2e, "roofline": roof,
            "block_solves_per_s": e.nbl / t_basis}


def workload_config(cfg_id):
    from paper_1707_07598_b200.models import CONFIGS
    c = CONFIGS[cfg_id]
    n, b = c["n"], c["b"]
    nb = n // b
    return {
        "workload": f"BASELINE config {cfg_id}: 3D {n}^3 cells, {b}^3-cell blocks "
                    f"({nb ** 3} local block solves), {c['n_src'][0] * c['n_src'][1]} dipole sources, "
                    f"{c['n_rec'][0] * c['n_rec'][1]} receivers, adaptive Lagrange MSFV forward+misfit+gradient",
        "mesh": [n, n, n], "blocks": [b, b, b], "n_blocks": nb ** 3, "k_coarse": (nb + 1) ** 3,
        "n_sources": c["n_src"][0] * c["n_src"][1], "n_receivers": c["n_rec"][0] * c["n_rec"][1],
        "model": f"{c['field'][1]} * GRF(sigma={c['field'][0]} cells), seed 0",
        "l2": "inputs larger than L2 (per-step factors/fields >> 126 MB); no flush",
        "parallelism": "replicas",
    }


# ----------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline

def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_full_time(cfg_id, seed, reps=1, warm=1, log=None, workers=1):
    """Time the CPU oracle (oracle/msfv_oracle.py, the reference msinv
    algorithm restated in numpy/scipy) on the FULL config's forward + misfit +
    gradient step, the same seeded inputs as the GPU arm.  Returns (median
    seconds per step, description); the one-time setup (partition, pattern
    cache) is excluded like the reference's BlockSystemCache."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    from oracle import msfv_oracle as orc
    from paper_1707_07598_b200.models import CONFIGS, config_model
    import paper_1707_07598_b200.mesh as gmesh
    orc.WORKERS = workers             # per-block loops on `workers` threads (reference: workers=os.cpu_count())
    c = CONFIGS[cfg_id]
    n, b = c["n"], c["b"]
    mesh = orc.Mesh(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n)
    part = orc.make_partition(mesh, b, b, b)
    srv = orc.top_survey(mesh, c["n_src"], c["n_rec"])
    m = config_model(gmesh.create_mesh(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n), c, seed)
    t0 = time.perf_counter()
    prob = orc.AdaptiveProblem(part, srv)
    setup = time.perf_counter() - t0
    d_obs = None
    ts = []
    for it in range(warm + reps):
        t0 = time.perf_counter()
        D, st = prob.simulate(m)
        if d_obs is None:
            d_obs = D * 1.05
        phi, r = orc.misfit(D, d_obs)
        prob.jacobian(st).rapply(r)
        dt = time.perf_counter() - t0
        if it >= warm:
            ts.append(dt)
        if log:
            log(f"oracle full-config iteration {it}: {dt:.2f} s")
    desc = (f"oracle port (numpy/scipy restatement of msinv; the per-block loops on {workers} thread(s), "
            f"OPENBLAS_NUM_THREADS=1) forward+misfit+gradient on the full config {cfg_id} ({part.n_blocks} blocks, "
            f"same seeded m and survey), median of {reps} after {warm} warm-up; one-time setup {setup:.1f} s "
            f"excluded; CPU: {cpu_model()}")
    return float(np.median(ts)), desc


# --------------------------------------------------------------- GPU arm

def fp64_peak():
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    if os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
            d = json.loads(out.strip().splitlines()[-1])
            return max(d["fp64_fma_tflops"], d["fp64_dmma_tflops"]), "measured live (tools/fp64_peak: max of FP64 FMA and DMMA)"
        except Exception:  # noqa: BLE001
            pass
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        return max(d["fp64_fma_tflops"], d["fp64_dmma_tflops"]), "profiles/fp64_peak.json (tools/fp64_peak on B200)"
    except Exception:  # noqa: BLE001
        return 37.1, "fallback: earlier tools/fp64_peak DMMA measurement"


def basis_flops(nI, p, r=8, n_edges=0, sweeps=2):
    """Algorithmic FP64 flops of one block in k_basis (banded algorithm as
    executed): factor, `sweeps` 8-rhs substitution sweeps, local Galerkin."""
    f = 0
    for j in range(nI):
        rm = min(p, nI - 1 - j)
        f += rm + rm * (rm + 1)            # column scale + rank-1 update (FMA = 2)
    for i in range(nI):
        f += sweeps * 2 * min(p, nI - 1 - i) * r  # substitution sweeps
    f += n_edges * (r + 2 * 36 + 1)        # local Galerkin
    return f


def solve_flops(nI, p, nrhs):
    f = 0
    for i in range(nI):
        f += 2 * 2 * min(p, nI - 1 - i) * nrhs
    return f


def reduced_bc_times(args, log):
    """Extension N4 at the bench config: forward map and the two sensitivity
    products with BasisSpec(boundary="reduced") (node-field kernel chains +
    the tensor-level skeleton map), device-timed; the adjoint identity of the
    two products as a self-check."""
    import numpy as np
    import torch
    import paper_1707_07598_b200 as gp
    from paper_1707_07598_b200.forward import forward_reduced_dev
    from paper_1707_07598_b200.models import config_problem
    try:
        mesh, part, survey, m = config_problem(args.config, seed=args.seed)
        builder = gp.BasisBuilder(part, gp.BasisSpec(boundary="reduced"))
        m_dev = torch.from_numpy(m).cuda()
        v = torch.from_numpy(np.random.default_rng(args.seed + 3).normal(size=m.size)).cuda()

        def timed(fn, reps=3):
            fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                out = fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            return sorted(ts)[len(ts) // 2], out

        def fwd():
            op = gp.assemble_operator(mesh, m_dev)
            return forward_reduced_dev(op, survey, builder.assemble(op))

        t_f, (D, st) = timed(fwd)
        t_s, J = timed(lambda: gp.sensitivity_adaptive(st, survey))
        W = torch.randn_like(D)
        t_r, g = timed(lambda: J.rapply_dev(W))
        t_a, jv = timed(lambda: J.apply_dev(v))
        lhs, rhs = float((jv * W).sum()), float(torch.dot(v, g))
        res = {"forward_ms": round(t_f, 3), "sensitivity_setup_ms": round(t_s, 3), "JTw_ms": round(t_r, 3),
               "Jv_ms": round(t_a, 3), "adjoint_identity_rel": abs(lhs - rhs) / abs(lhs),
               "what": "BasisSpec(boundary='reduced') at the bench config: reduced 1D line / 2D face-patch boundary "
                       "problems, forward map and sensitivities through them (extension N4, no reference)"}
    except Exception as e:                                   # the headline numbers do not depend on the extension
        res = {"error": f"{type(e).__name__}: {e}"}
    log("reduced_bc: " + json.dumps(res))
    return res


def table3_times(log):
    """S_k, Y_k, X_k at the paper's Table-3 geometry (
    BASELINE.md section 1): 64x64x32 cells, 16^3 blocks (n_I = 3375, the
    L2-resident band solver), 72 sources, 3698 receivers.  Device times (CUDA
    events, best of 3 after a warm-up) and the host-CSR time of Y_k through
    the reference-named API, next to the paper's Julia numbers."""
    import numpy as np
    import torch
    import paper_1707_07598_b200 as gp
    from paper_1707_07598_b200.models import table3_problem
    mesh, part, survey, m = table3_problem()
    builder = gp.BasisBuilder(part)
    m_dev = torch.from_numpy(m).cuda()
    basis = builder.assemble(gp.assemble_operator(mesh, m_dev))
    eng = basis.engine
    rng = np.random.default_rng(0)
    v = torch.from_numpy(rng.standard_normal(eng.k)).cuda()
    w = torch.from_numpy(rng.standard_normal(eng.n)).cuda()

    def best(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        out = 1e30
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = fn()
            b.record()
            torch.cuda.synchronize()
            out = min(out, a.elapsed_time(b))
            del r
        return round(out, 3)

    res = {"geometry": f"64x64x32 cells, 16^3 blocks ({eng.nbl}), n_I {eng.nI}, k {eng.k}, 72 sources, 3698 receivers",
           "S_k_ms": best(lambda: builder.assemble(gp.assemble_operator(mesh, m_dev)).Sint),
           "Y_k_ms": best(lambda: gp.apply_Yk_dev(basis, v, m_dev)),
           "X_k_ms": best(lambda: gp.apply_Xk_dev(basis, w, m_dev))}
    t0 = time.perf_counter()
    Y = gp.apply_Yk(basis, v.cpu().numpy(), m_dev)
    res["Y_k_host_csr_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
    res["Y_k_nnz"] = int(Y.nnz)
    del Y
    res["paper_julia_s"] = {"workers_1": {"S_k": 3.8595, "Y_k": 2.7380, "X_k": 2.9933},
                            "workers_8": {"S_k": 1.4150, "Y_k": 1.0658, "X_k": 1.3818},
                            "hardware": "4x Xeon E5-4627 (40 cores), PAPER.md:576"}
    log("table3: " + json.dumps(res))
    return res


def run_gpu(args, rank, world, log):
    import numpy as np
    import torch
    import paper_1707_07598_b200 as gp
    from paper_1707_07598_b200 import _lib
    from paper_1707_07598_b200.engine import PhaseTimer
    from paper_1707_07598_b200.forward import forward_reduced_dev, sensitivity_adaptive
    from paper_1707_07598_b200.models import config_problem

    from paper_1707_07598_b200 import dist
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    mesh, part, survey, m = config_problem(args.config, seed=dist.replica_seed(args.seed, rank))
    m_obs = m + 0.25 * gp.models.gaussian_field(mesh, 6.0, 1.0, args.seed + 1)
    builder = gp.BasisBuilder(part, gp.BasisSpec())
    problem = gp.AdaptiveReducedProblem(builder, survey)
    dev = torch.device("cuda")
    if args.ncu:
        op_obs = gp.assemble_operator(mesh, torch.from_numpy(m_obs).to(dev))
        d_obs = forward_reduced_dev(op_obs, survey, builder.assemble(op_obs))[0].cpu().numpy()
    else:
        d_obs = problem.simulate(m_obs)[0]
    m_dev = torch.from_numpy(m).to(dev)
    dobs_dev = torch.from_numpy(d_obs).to(dev)
    L = _lib.load()

    def step_dev():
        # device-resident step: no host synchronisation until the status check
        op = gp.assemble_operator(mesh, m_dev)
        basis = builder.assemble(op)
        D, st = forward_reduced_dev(op, survey, basis, defer_check=True)
        st.deferred = True
        phi, resid = gp.misfit_ssd_dev(D, dobs_dev)
        g = sensitivity_adaptive(st, survey).rapply_dev(resid)
        st.check()
        return phi, g

    # correctness guard of the timed configuration: misfit and gradient finite
    phi0, g0 = step_dev()
    # long-lived setup objects (modules, survey, problem) move to the permanent
    # generation so a periodic full GC pass does not stall the host launch
    # stream for ~35 ms every ~10 steps
    gc.collect()
    gc.freeze()
    assert torch.isfinite(phi0).item() and torch.isfinite(g0).all().item()

    for _ in range(args.warmup):
        step_dev()
    # extra untimed steps until the per-step device time is stable (the first
    # ~10 steps after allocation run slower; see profiles/README)
    prev = None
    for _ in range(0 if args.ncu else 12):
        a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        step_dev()
        b0.record()
        torch.cuda.synchronize()
        t = a0.elapsed_time(b0)
        if prev is not None and abs(t - prev) <= 0.01 * prev:
            break
        prev = t
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", 0)))
    clocks.start()
    time.sleep(0.3)
    n0 = L.msfv_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        step_dev()
    e1.record()
    torch.cuda.synchronize()
    launches = L.msfv_launch_count() - n0
    ms = e0.elapsed_time(e1) / args.steps
    clk = clocks.stop()
    ms = dist.max_over_ranks(ms, dev)
    log(f"device step {ms:.3f} ms")
    if args.ncu:
        return None

    # end to end through the public API: pinned host m in, D and g out
    e2e = None
    if not args.no_e2e:
        m_pin = torch.from_numpy(m).pin_memory()
        # measured right after the device-timed steps (before the Gauss-Newton,
        # fine-mesh and Table-3 legs, whose large allocations leave the caching
        # allocators in a state the e2e warm-up takes tens of steps to leave);
        # release the device-resident leg's blocks so the warm-up settles its own
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        for _ in range(max(5, args.warmup)):
            D, st = problem.simulate(m_pin)
            phi, resid = gp.misfit_ssd(D, d_obs)
            problem.jacobian(st).rapply(resid)
        torch.cuda.synchronize()
        dist.barrier()
        # five back-to-back repetitions of the K-step loop, median reported
        # (the first repetition after the device-resident legs is ~25% slower:
        # host allocator / page-locked buffer warm-up)
        reps = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.steps):
                D, st = problem.simulate(m_pin)
                phi, resid = gp.misfit_ssd(D, d_obs)
                g_host = problem.jacobian(st).rapply(resid)
            b.record()
            torch.cuda.synchronize()
            reps.append(a.elapsed_time(b) / args.steps)
        log("e2e repetitions (ms/step): " + ", ".join(f"{x:.3f}" for x in reps))
        e2e_ms = dist.max_over_ranks(sorted(reps)[2], dev)
        h2d = m.nbytes + resid.nbytes
        d2h = D.nbytes + g_host.nbytes
        e2e = {"value": dist.aggregate_seconds_per_iter(e2e_ms / 1e3, world), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_ms, 4),
               "path": "AdaptiveReducedProblem.simulate -> misfit_ssd -> jacobian(state).rapply (numpy out)"}
        log(f"e2e step {e2e_ms:.3f} ms")

    # config-4 Gauss-Newton iteration (BASELINE configs[3]): one iteration of
    # the device-resident projected Gauss-Newton method (inversion.py:187-263;
    # GNConfig(max_gn=1, max_cg=5), Objective(alpha=1e-3, m_ref=0)): forward,
    # gradient with the Tikhonov term, 5 masked-CG steps on J^T J + alpha L^T L
    # (each one J v and one J^T (J v)), and the Armijo line search (forward
    # solves at the trial models)
    gn = None
    if not args.no_gn:
        gobj = gp.DeviceObjective(mesh, 1e-3, np.zeros(mesh.n_cells))
        gcfg = gp.GNSettings(max_gn=1, max_cg=5)
        for _ in range(min(args.warmup, 2)):
            gp.gauss_newton_dev(problem, m_dev, dobs_dev, gobj, gcfg)
        torch.cuda.synchronize()
        dist.barrier()
        trials = []
        g0e, g1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0e.record()
        nrep = max(1, min(args.steps, 5))
        for _ in range(nrep):
            _, tr = gp.gauss_newton_dev(problem, m_dev, dobs_dev, gobj, gcfg)
            trials.append(tr.rows[-1])
        g1e.record()
        torch.cuda.synchronize()
        gn_ms = dist.max_over_ranks(g0e.elapsed_time(g1e) / nrep, dev)
        last = trials[-1]
        gn = {"ms_per_iter": round(gn_ms, 4), "cg_steps": int(last["cg_iters"]), "step": last["step"],
              "what": "one projected Gauss-Newton iteration (gauss_newton_dev, max_gn=1, max_cg=5, alpha=1e-3): "
                      "forward + gradient + regularizer, masked CG (J v, J^T J v, alpha L^T L v per step), "
                      "Armijo line search with forward solves; device-resident, scalars synced per CG step"}
        log(f"GN iteration {gn_ms:.3f} ms (cg {last['cg_iters']}, step {last['step']})")

    # fine-mesh forward: d_obs generation at the config's
    # model with the fine operator (forward_full(solver="direct"): tight
    # Jacobi-PCG on the device, relative residual 1e-13)
    fine = None
    if not args.no_gn and args.config == 4:
        fprob = gp.FullProblem(mesh, survey)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Dfull, fst = fprob.simulate(m_obs)
        fine = {"seconds": round(time.perf_counter() - t0, 4), "iterations": int(fst.factor.last.iterations),
                "relres": fst.factor.last.relres,
                "what": "forward_full(direct) at 128^3 with 16 sources: PCG per column to relres 1e-13, preconditioned by the two-level MSFV method (adaptive basis + Galerkin coarse solve + block interior solves + skeleton Jacobi)",
                "n_sources": int(Dfull.shape[1])}
        log("fine forward: " + json.dumps(fine))
        del fprob, fst

    # per-phase breakdown (one extra instrumented step)
    PhaseTimer.start()
    step_dev()
    phases = PhaseTimer.stop()
    log("phases (ms): " + json.dumps({k: round(v, 4) for k, v in phases.items()}))

    eng = builder.assemble(gp.assemble_operator(mesh, m_dev)).engine
    nI = eng.nI
    p = (part.b1 - 1) * (part.b2 - 1)
    own_edges = 3 * part.b1 * part.b2 * part.b3
    # the tensor-core build runs as two launches: the forward part (factor,
    # forward sweep, Galerkin; the "basis" phase on the critical path) and the
    # backward sweeps on a side stream, overlapped with the coarse factorization
    fl_fwd = basis_flops(nI, p, 8, own_edges, sweeps=1)
    fl_whole = basis_flops(nI, p, 8, own_edges, sweeps=2)
    t_basis = phases.get("basis", float("nan")) / 1e3
    # whole build (forward part + backward sweeps, serial on one stream:
    # msfv_basis_build) timed on its own
    _, w_dev, fl_dev = eng.operator(m_dev)
    for _ in range(3):
        eng.basis(w_dev, fl_dev)
    wa, wb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wa.record()
    for _ in range(10):
        eng.basis(w_dev, fl_dev)
    wb.record()
    torch.cuda.synchronize()
    t_whole = wa.elapsed_time(wb) / 10 / 1e3
    peak, peak_src = fp64_peak()
    achieved = fl_fwd * eng.nbl / t_basis / 1e12
    # compulsory bytes of the basis construction: read the edge
    # weights, write S_I and the local Galerkin blocks
    compulsory = int(eng.E * 8 + eng.nbl * 8 * nI * 8 + eng.nbl * 64 * 8)
    traffic, traffic_src, dmma_pct = None, None, None
    for prof_name in ("r02_ncu.json", "r01c_ncu.json"):
        try:
            # dram__bytes_read.sum + dram__bytes_write.sum of k_basis_tc from the
            # committed ncu --set full capture of this configuration
            prof = json.load(open(os.path.join(ROOT, "profiles", prof_name)))["full"]
            kb = next(v for k, v in prof.items() if "k_basis_tc" in k)
            if args.config == 4:
                traffic = int(kb["dram_read_B"] + kb["dram_write_B"])
                traffic_src = f"profiles/{prof_name} (ncu --set full, k_basis_tc, bytes per launch)"
                if "dmma_pipe_pct" in kb:
                    dmma_pct = round(kb["dmma_pipe_pct"], 1)
            break
        except Exception:  # noqa: BLE001
            continue
    roof = {"kernel": "k_basis_tc<PT,false> + k_skel_lines (per-block A_II band Cholesky, 8-RHS forward sweep, "
                      "local Galerkin; skeleton line sums on a side stream beside it; the backward sweeps run "
                      "concurrently in k_basis_bwd)",
            "bound": "fp64", "achieved": round(achieved, 3), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_unit": "bytes", "traffic_source": traffic_src,
            "algorithmic_bytes": compulsory,
            "algorithmic_bytes_what": "compulsory: edge weights in, S_I and Kloc out (SURVEY 8d)",
            "flops_per_block": fl_fwd, "blocks_per_launch": eng.nbl, "launch_ms": round(t_basis * 1e3, 4),
            "peak_source": peak_src,
            "dmma_pipe_active_pct": dmma_pct,
            "dmma_pipe_note": "ncu sm__pipe_tensor_subpipe_dmma_cycles_active / cycles of the same capture: the FP64 "
                              "tensor pipe's occupancy including the tile padding of the band (useful flops are "
                              "the frac above)",
            "whole_build": {"ms": round(t_whole * 1e3, 4), "flops_per_block": fl_whole,
                            "achieved": round(fl_whole * eng.nbl / t_whole / 1e12, 3),
                            "frac": round(fl_whole * eng.nbl / t_whole / 1e12 / peak, 4),
                            "what": "forward part + backward sweeps on one stream (msfv_basis_build)"},
            "note": "FP64 bound: tcgen05 has no f64 kind; the kernel runs on DMMA (mma.sync m8n8k4 f64); "
                    "useful banded flops only (tile padding not counted)"}
    return {
        "ms": ms, "launches": launches, "clocks": clk, "phases": phases, "e2e": e2e, "roofline": roof,
        "block_solves_per_s": eng.nbl / t_whole, "nbl": eng.nbl,
        "interior_solve_ms": phases.get("interior_solve"), "gn": gn, "fine": fine,
    }


def main_2d(args, rank, world, log):
    cfg = workload_config_2d(args.config)
    if args.impl == "reference":
        if rank != 0:
            return 0
        workers = os.cpu_count() or 1
        t, desc = oracle2d_time(args.config, args.seed, reps=args.steps, warm=args.warmup, log=log, workers=workers)
        line = {"impl": "reference", "metric": METRIC, "value": t, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
                "cpu_baseline": {"value": t, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc},
                "e2e": {"value": t, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    import torch
    from paper_1707_07598_b200 import dist
    dist.init("nccl")
    res = run_2d(args, log)
    ms = dist.max_over_ranks(res["ms"], torch.device("cuda"))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t, desc = oracle2d_time(args.config, args.seed, reps=1, warm=1, log=log)
        cpu = {"value": t, "unit": UNIT, "cores": 1, "kind": "port", "sample": desc}
    if rank == 0:
        line = {"metric": METRIC, "value": dist.aggregate_seconds_per_iter(ms / 1e3, world), "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": cfg, "roofline": res["roofline"], "cpu_baseline": cpu,
                "e2e": res["e2e"], "gpu_launches": int(res["launches"]),
                "gpu_launches_per_step": res["launches"] / args.steps, "clocks": res["clocks"],
                "local_block_solves_per_s": round(res["block_solves_per_s"], 1)}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))

    def log(msg):
        if rank == 0:
            print(f"[bench] {msg}", file=sys.stderr, flush=True)

    if args.config in (1, 2):
        return main_2d(args, rank, world, log)
    cfg = workload_config(args.config)
    if args.impl == "reference":
        if rank != 0:
            return 0
        workers = os.cpu_count() or 1
        # every step is the full workload; warm-up capped at 2 full steps
        # (the oracle has no JIT or allocator state to settle beyond the first)
        warm = min(args.warmup, 2)
        v, desc = oracle_full_time(args.config, args.seed, reps=args.steps, warm=warm, log=log, workers=workers)
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "warmup_done": warm, "ms_per_step": v * 1e3,
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": cfg,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc,
                                 "cpu_model": cpu_model(), "extrapolated": False},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    from paper_1707_07598_b200 import dist
    dist.init("nccl")
    res = run_gpu(args, rank, world, log)
    if res is None:
        return 0
    t3 = None
    # side legs (Table-3 geometry, reduced boundary conditions): single-GPU runs only, so the ranks of a
    # scaling run leave the process group together
    if rank == 0 and world == 1 and args.config == 4 and not args.no_table3:
        t3 = table3_times(log)
    red = None
    if rank == 0 and world == 1 and args.config == 4 and not args.no_table3:
        red = reduced_bc_times(args, log)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        t, desc = oracle_full_time(args.config, args.seed, reps=1, warm=1, log=log, workers=workers)
        cpu = {"value": t, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc, "cpu_model": cpu_model(),
               "extrapolated": False}
    if rank == 0:
        line = {
            "metric": METRIC, "value": dist.aggregate_seconds_per_iter(res["ms"] / 1e3, world), "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms"], 4),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg, "roofline": res["roofline"], "cpu_baseline": cpu,
            "e2e": res["e2e"], "gpu_launches": int(res["launches"]),
            "gpu_launches_per_step": res["launches"] / args.steps, "clocks": res["clocks"],
            "local_block_solves_per_s": round(res["block_solves_per_s"], 1),
            "phases_ms": {k: round(v, 4) for k, v in res["phases"].items()},
            "gn_iteration": res["gn"],
            "fine_forward": res.get("fine"),
            "table3": t3,
            "reduced_bc": red,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
