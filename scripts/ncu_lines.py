"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA source line:
warp-stall samples and the top stall reasons, per function.  usage: ncu_lines.py src.csv [topN]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
fn, fpath, hdr = None, None, None
agg = defaultdict(lambda: defaultdict(lambda: [0, defaultdict(int), ""]))
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] and r[0] != "":
        line = (fpath, int(r[0]))
        cur = agg[fn][line]
        cur[2] = r[1].strip()
        try:
            cur[0] += int(r[4])
        except ValueError:
            pass
        for k, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    cur[1][h[6:]] += int(r[k])
                except ValueError:
                    pass
for f, lines in agg.items():
    tot = sum(v[0] for v in lines.values())
    print(f"== {f}  samples {tot}")
    for (fp, ln), (s, st, src) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
        reasons = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{s:7d} {100*s/max(tot,1):5.1f}% {fp}:{ln:<5d} {src[:70]:70s} | {reasons}")
