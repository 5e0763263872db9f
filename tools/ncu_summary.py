"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) and a
--set full report into profiles/ (markdown rows + JSON).

usage: python tools/ncu_summary.py LAUNCHES.csv REPORT.ncu-rep[,REPORT2.ncu-rep...] OUT_PREFIX
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path, steps=2):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    seq = [(r[ki], float(r[vi])) for r in rows[hdr + 1:] if r[mi] == "gpu__time_duration.sum"]
    # last step only: the kernels after the final k_sigma launch
    start = max(i for i, (k, _) in enumerate(seq) if k.startswith("msfv::k_sigma") or "k_sigma" in k)
    agg = collections.OrderedDict()
    for k, ns in seq[start:]:
        name = k.split("(")[0]
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + ns)
    return agg


WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "fp64_pipe_pct",
    "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg": "dmma_cycles",
    "smsp__cycles_elapsed.avg": "smsp_cycles",
    "sm__inst_executed.sum": "inst",
    "launch__registers_per_thread": "regs",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}
SCALE = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "nsecond": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "cycle": 1.0, "Kcycle": 1e3, "Mcycle": 1e6, "inst": 1.0, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    res = collections.OrderedDict()
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0]
        m = {}
        for k, nk in WANT.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    m[nk] = float(d[k].replace(",", "")) * SCALE.get(units.get(k, ""), 1.0)
                except ValueError:
                    pass
        if "dmma_cycles" in m and m.get("smsp_cycles"):
            m["dmma_pipe_pct"] = 100.0 * m["dmma_cycles"] / m["smsp_cycles"]
        if name not in res or m.get("duration_ns", 0) > res[name].get("duration_ns", 0):
            res[name] = m      # the longest instance of each kernel (its dominant launch)
    return res


def main():
    lp, rp, pre = sys.argv[1:4]
    L = launches(lp)
    F = collections.OrderedDict()
    for r in rp.split(","):
        F.update(full(r))
    tot = sum(t for _, t in L.values())
    md = ["| kernel | launches | ms (cold, serialized) | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(L.items(), key=lambda kv: -kv[1][1]):
        md.append(f"| `{k}` | {n} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    md.append(f"| **total** | | **{tot / 1e6:.3f}** | |")
    md.append("")
    md.append("| kernel | duration | DRAM read + write / launch | warps active | FP64 pipe | DMMA subpipe | regs |")
    md.append("|---|---|---|---|---|---|---|")
    for k, m in F.items():
        md.append(f"| `{k}` | {m.get('duration_ns', 0) / 1e6:.3f} ms | {m.get('dram_read_B', 0) / 1e9:.3f} + "
                  f"{m.get('dram_write_B', 0) / 1e9:.3f} GB | {m.get('warps_active_pct', 0):.1f}% | "
                  f"{m.get('fp64_pipe_pct', 0):.1f}% | {m.get('dmma_pipe_pct', 0):.1f}% | {m.get('regs', 0):.0f} |")
    open(pre + ".md", "w").write("\n".join(md) + "\n")
    json.dump({"launches": {k: {"n": n, "ns": t} for k, (n, t) in L.items()}, "full": F},
              open(pre + ".json", "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
