"""Group an `ncu --page source --csv --print-source sass` export into runs of
instructions with equal execution counts (basic blocks / loop bodies) and
print the heaviest runs: per-CTA executions, instruction share, samples and
opcode mix.  usage: python tools/sass_segments.py EXPORT.csv N_CTAS [N_TOP]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ncta = float(sys.argv[2])
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = next(r for r in rows if "Address" in r and "Source" in r)
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
segs = []
for r in data:
    ex = float(r[ix["Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    src = r[ix["Source"]].strip()
    if segs and segs[-1][0] == ex:
        segs[-1][1] += 1
        segs[-1][2] += s
        segs[-1][4].append(src)
    else:
        segs.append([ex, 1, s, r[ix["Address"]], [src]])
tot = sum(x[0] * x[1] for x in segs)
for ex, n, s, a, src in sorted(segs, key=lambda x: -x[0] * x[1])[:ntop]:
    ops = collections.Counter((t.split()[1] if t.startswith("@") else t.split()[0]).split(".")[0] for t in src if t)
    print(f"{a[-5:]} exec/CTA {ex / ncta:8.1f} n={n:4d} instr%={100 * ex * n / tot:5.1f} samples={s:6.0f}",
          dict(ops.most_common(6)))
