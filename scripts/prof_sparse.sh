#!/bin/bash
# ncu source-level capture of the C2 sparse kernels (+ emit) and the phase split (one gpurun call).
mkdir -p gpurun_out
python scripts/phases.py C2 > gpurun_out/phases_c2.txt 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
ncu --set full --clock-control none --import-source on -k regex:"k_sparse_fwd2|k_sparse_bwd2|k_emit" -s 3 -c 3 -o gpurun_out/src_c2 $B > gpurun_out/ncu_src_c2.log 2>&1
for k in k_sparse_fwd2 k_sparse_bwd2 k_emit; do
  ncu -i gpurun_out/src_c2.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > gpurun_out/src_$k.csv 2>/dev/null
  python scripts/ncu_lines.py gpurun_out/src_$k.csv 45 > gpurun_out/lines_$k.txt 2>&1
done
rm -f gpurun_out/src_*.csv
