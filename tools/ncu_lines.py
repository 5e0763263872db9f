"""Aggregate an ncu --page source --csv dump by source line (debug helper)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None; fname = None; out = []
for r in rows:
    if r and r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if len(r) >= 5 and r[0].isdigit() and hdr:
        out.append((fname, int(r[0]), dict(zip(hdr, r))))
def gi(d, k):
    try: return int(d[k] or 0)
    except Exception: return 0
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
T = sum(gi(d, 'Warp Stall Sampling (All Samples)') for f, l, d in out)
TI = sum(gi(d, 'Instructions Executed') for f, l, d in out)
print('total samples', T, 'total inst', TI)
tot = collections.Counter()
for f, l, d in out:
    for s in stalls: tot[s] += gi(d, s)
print(' '.join(f"{s[6:]}={100*v/T:.1f}" for s, v in tot.most_common(10)))
for f, l, d in sorted(out, key=lambda x: -gi(x[2], 'Warp Stall Sampling (All Samples)'))[:n]:
    st = sorted(((gi(d, s), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{f[:16]:16s}:{l:4d} samp={100*gi(d,'Warp Stall Sampling (All Samples)')/T:5.2f}% inst={100*gi(d,'Instructions Executed')/TI:5.2f}% {st}")
