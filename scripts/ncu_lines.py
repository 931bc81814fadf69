"""Per-source-line instruction and stall-sample shares from an ncu cuda,sass
source export (development helper)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
def f(x):
    try: return float(x)
    except: return 0.0
ie = hdr.index('Instructions Executed'); sm = hdr.index('Warp Stall Sampling (All Samples)')
by = collections.defaultdict(lambda: [0, 0, ''])
for r in rows[hi + 1:]:
    if len(r) <= sm or not r[0]: continue
    try: ln = int(r[0])
    except: continue
    by[ln][0] += f(r[ie]); by[ln][1] += f(r[sm]); by[ln][2] = r[1]
tot = sum(v[0] for v in by.values()) or 1; st = sum(v[1] for v in by.values()) or 1
for ln, v in sorted(by.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"L{ln:4d} inst {v[0]/tot*100:5.1f}% stall {v[1]/st*100:5.1f}%  {v[2].strip()[:90]}")
