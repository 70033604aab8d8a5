#!/bin/bash
# Source-level ncu stall tables (one gpurun call): the C2 sparse kernels and the full-sweep
# emit, the C4 cell-grid sweeps.  The .ncu-rep files are summarised on the box (per CUDA line:
# warp-stall samples and top reasons, scripts/ncu_lines.py) and removed (gpurun pulls <= 64 MiB).
mkdir -p gpurun_out
B="python bench.py --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
ncu --set full --clock-control none --import-source on -k regex:"k_sparse_fwd2|k_sparse_bwd2|k_emit" -s 3 -c 3 -o gpurun_out/src_c2 $B --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_top2_cells|k_emit_cells" -s 2 -c 2 -o gpurun_out/src_c4 $B --steps 1 --config C4 > /dev/null 2>&1
for pair in c2:k_sparse_fwd2 c2:k_sparse_bwd2 c2:k_emit c4:k_top2_cells c4:k_emit_cells; do
  rep=${pair%%:*}; k=${pair##*:}
  ncu -i gpurun_out/src_$rep.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > /tmp/src.csv 2>/dev/null
  python scripts/ncu_lines.py /tmp/src.csv 40 > gpurun_out/lines_${rep}_$k.txt 2>&1
done
rm -f gpurun_out/src_*.ncu-rep
