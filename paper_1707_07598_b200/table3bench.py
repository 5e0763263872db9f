"""Table-3 style benchmark of the per-block operations on the GPU
(the reference's ``scaling_benchmark`` / ``msinv bench``,
cli.py:170-261, and the paper's Table 3).

    python -m paper_1707_07598_b200.table3bench [--geometry table3|config4]
                                                [--repeats 5] [--out DIR]

Like the reference it first checks that repeated evaluations are bitwise
identical (the reference compares worker counts against serial; the GPU path
has one schedule, fixed-order reductions and no atomics), then reports the
median time of ``basis`` (S_k(m): operator + all local block solves),
``dSv`` (apply_Yk) and ``dStw`` (apply_Xk).  Times are taken two ways:
device (CUDA events around the device-resident call) and host (wall clock of
the reference-named call returning scipy matrices).  Writes bench.csv with
the reference's columns, the worker column reading "gpu".
"""

import argparse
import json
import os
import time

import numpy as np
import torch

from .basis import BasisBuilder
from .operators import assemble_operator
from .table3 import apply_Xk, apply_Xk_dev, apply_Yk, apply_Yk_dev


def _problem(name):
    from .models import config_problem, table3_problem
    if name == "table3":
        return table3_problem()
    return config_problem(4)


def _same(a, b):
    return (a.shape == b.shape and np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
            and np.array_equal(a.data, b.data))


def run(geometry="table3", repeats=5, seed=0):
    mesh, part, survey, m = _problem(geometry)
    builder = BasisBuilder(part)
    m_dev = torch.from_numpy(m).cuda()
    op = assemble_operator(mesh, m_dev)
    basis = builder.assemble(op)
    eng = basis.engine
    rng = np.random.default_rng(seed)
    v = rng.normal(size=eng.k)
    w = rng.normal(size=eng.n)
    # determinism check (cli.py:186-210 compares against serial bitwise)
    S0, Y0, X0 = basis.S, apply_Yk(basis, v, m_dev), apply_Xk(basis, w, m_dev)
    b2 = builder.assemble(assemble_operator(mesh, m_dev))
    if not _same(b2.S.tocsr(), S0.tocsr()):
        raise RuntimeError("basis differs between two evaluations")
    if not _same(apply_Yk(b2, v, m_dev), Y0):
        raise RuntimeError("dSv differs between two evaluations")
    if not _same(apply_Xk(b2, w, m_dev), X0):
        raise RuntimeError("dStw differs between two evaluations")
    nnz = {"basis": int(S0.nnz), "dSv": int(Y0.nnz), "dStw": int(X0.nnz)}
    del S0, Y0, X0, b2
    vd, wd = torch.from_numpy(v).cuda(), torch.from_numpy(w).cuda()
    dev_ops = {
        "basis": lambda: builder.assemble(assemble_operator(mesh, m_dev)).Sint,
        "dSv": lambda: apply_Yk_dev(basis, vd, m_dev),
        "dStw": lambda: apply_Xk_dev(basis, wd, m_dev),
    }
    host_ops = {
        "basis": lambda: builder.assemble(assemble_operator(mesh, m)).S,
        "dSv": lambda: apply_Yk(basis, v, m_dev),
        "dStw": lambda: apply_Xk(basis, w, m_dev),
    }
    dev, host = {}, {}
    for name, fn in dev_ops.items():
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(repeats):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
            del out
        dev[name] = float(np.median(ts))
    for name, fn in host_ops.items():
        fn()
        ts = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            out = fn()
            ts.append(time.perf_counter() - t0)
            del out
        host[name] = float(np.median(ts))
    return {"geometry": geometry, "cells": list(eng.cells), "blocks": list(eng.blocks), "n_blocks": eng.nbl,
            "n_I": eng.nI, "k": eng.k, "nnz": nnz, "device_seconds": dev, "host_seconds": host,
            "bitwise_repeatable": True}


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--geometry", default="table3", choices=["table3", "config4"])
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    r = run(args.geometry, args.repeats)
    lines = ["workers,basis_seconds,dSv_seconds,dStw_seconds,speedup_basis,speedup_dSv,speedup_dStw"]
    for label, t in (("gpu", r["device_seconds"]), ("gpu_host_api", r["host_seconds"])):
        lines.append(f"{label},{t['basis']:.6f},{t['dSv']:.6f},{t['dStw']:.6f},1.00,1.00,1.00")
    if args.out:
        os.makedirs(args.out, exist_ok=True)
        with open(os.path.join(args.out, "bench.csv"), "w") as f:
            f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    print(json.dumps(r))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
