"""Summarise an ncu launch list (gpu__time_duration per launch) into a per-kernel table."""
import csv
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag, path, steps = sys.argv[1], sys.argv[2], int(sys.argv[3])
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
        k = r[ki].split("(")[0].replace("void ", "").strip()
        tot[k] += v
        cnt[k] += 1
    all_t = sum(tot.values())
    lines = [f"# ncu launch list ({tag})", "",
             f"`ncu --metrics gpu__time_duration.sum --clock-control none` over the whole bench command "
             f"(warm-up + {steps} timed steps; cold-cache, serialised launches: compare SHARES).", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / all_t:.3f} |")
    out = os.path.join(ROOT, "profiles", f"{tag}_launches.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
