"""Summarise ncu reports (gpurun_out/*.ncu-rep) into profiles/: key metrics per kernel as
markdown + the per-launch DRAM traffic that bench.py reports as roofline.traffic."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, k in METRICS.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    v = float(v)
                    u = units[hdr.index(m)]
                    if u in ("Kbyte",): v *= 1e3
                    if u in ("Mbyte",): v *= 1e6
                    if u in ("Gbyte",): v *= 1e9
                    if u in ("usecond", "us"): v *= 1e3   # -> ns
                    if u in ("msecond", "ms"): v *= 1e6
                    if u in ("second", "s"): v *= 1e9
                except ValueError:
                    pass
                d[k] = v
        res.append(d)
    return res


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summaries ({tag})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 (gpurun).",
             "Per launch; bytes in B; duration in ns (ncu replays are cold-cache and serialised).", ""]
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for rep in reps:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        cfg = name.split("_")[-1].upper()
        lines.append(f"## {name}")
        lines.append("")
        keys = list(METRICS.values())
        lines.append("| kernel | " + " | ".join(keys) + " |")
        lines.append("|---|" + "---|" * len(keys))
        for d in raw(rep):
            k = d["kernel"].split("(")[0].replace("void ", "")
            lines.append(f"| {k} | " + " | ".join(f"{d.get(x, ''):.4g}" if isinstance(d.get(x), float) else str(d.get(x, "")) for x in keys) + " |")
            stage = {"k_line_top2": "passA_rows", "k_top2_cells": "passA_rows", "k_emit": "emit",
                     "k_sparse_fwd": "sparse_fwd", "k_sparse_bwd": "sparse_bwd"}
            for pre, st in stage.items():
                if pre in k and isinstance(d.get("dram_read"), float):
                    traffic.setdefault(cfg, {})[st] = d["dram_read"] + d.get("dram_write", 0.0)
                    if st == "passA_rows":
                        traffic[cfg]["passA_cols"] = traffic[cfg][st]
        lines.append("")
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
