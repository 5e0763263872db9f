"""Aggregate an `ncu --page source --csv --print-source sass` export: stall
reasons, per-opcode samples / executed counts, and the hottest instructions
of the main loop (the most frequent execution count).

usage: python tools/sass_stalls.py EXPORT.csv [N_TOP]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = next(r for r in rows if "Address" in r and "Source" in r)
data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
S = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
tot = collections.Counter()
byop = collections.Counter()
cnt = collections.Counter()
execs = collections.Counter()
for r in data:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = float(r[ix["Instructions Executed"]] or 0)
    toks = r[ix["Source"]].split()
    op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "")).split(".")[0]
    byop[op] += s
    cnt[op] += ex
    execs[ex] += 1
    for h in stalls:
        tot[h] += float(r[ix[h]] or 0)
print(f"samples {S:.0f}, warp instructions executed {sum(cnt.values()):.4g}")
print("stalls: " + ", ".join(f"{h[6:]} {v / S * 100:.1f}%" for h, v in tot.most_common(9)))
print("by opcode (samples %, executed):")
for op, v in byop.most_common(18):
    print(f"  {op:10s} {v / S * 100:5.1f}%  {cnt[op]:.3g}")
loop_ex = max((e for e in execs if e > 0), key=lambda e: execs[e] * e)
print(f"main loop: {execs[loop_ex]} instructions executed {loop_ex:.0f} times")
