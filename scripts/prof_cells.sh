#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-graph --config C4"
ncu --set full --clock-control none --import-source on -k regex:"k_top2_cells|k_emit_cells" -s 2 -c 2 -o gpurun_out/src_cells $B > gpurun_out/ncu_src_cells.log 2>&1
for k in k_top2_cells k_emit_cells; do
  ncu -i gpurun_out/src_cells.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > gpurun_out/src_$k.csv 2>/dev/null
  python scripts/ncu_lines.py gpurun_out/src_$k.csv 40 > gpurun_out/lines_$k.txt 2>&1
done
ncu -i gpurun_out/src_cells.ncu-rep --page details --csv > gpurun_out/details_cells.csv 2>/dev/null
rm -f gpurun_out/src_*.csv
