#!/bin/bash
# ncu evidence for profiles/ (one gpurun call): launch lists of the bench commands (C2 default,
# C4, C5) + full captures of the hot kernels (C2: full sweeps + cluster sparse kernels; C4: the
# grid sparse stage; C5: culled sweeps), the Fig. 2 sweep (nnz and memory per sample).
# Summaries are written back here with scripts/launch_summary.py / ncu_summary.py.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
for c in C2 C4 C5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c,,}.csv $B --config $c > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_line_top2|k_emit|k_sparse" -s 7 -c 6 -o gpurun_out/full_c2 $B --no-graph > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_rs_colsum_bstep|k_rs_bwd_rowrev2_rowrev" -s 20 -c 2 -o gpurun_out/full_c4 $B --no-graph --config C4 > gpurun_out/ncu_full_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_top2_cells|k_emit_cells" -s 2 -c 2 -o gpurun_out/full_c4cells python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --config C4 > gpurun_out/ncu_full_c4cells.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_top2_cells|k_emit_cells" -s 2 -c 2 -o gpurun_out/full_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --config C5 > gpurun_out/ncu_full_c5.log 2>&1
timeout 900 python scripts/fig2.py --trials 500 --all-large > gpurun_out/fig2.log 2>&1
cp profiles/fig2_nnz.csv profiles/fig2_nnz.md gpurun_out/ 2>/dev/null
