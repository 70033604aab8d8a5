#!/bin/bash
# ncu evidence for profiles/: launch list (C2 bench command) + full captures of the kernels.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B --config C4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_line_top2|k_emit|k_sparse" -s 7 -c 6 -o gpurun_out/full_c2 $B > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_line_top2|k_emit|k_sparse" -s 7 -c 6 -o gpurun_out/full_c4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --config C4 > gpurun_out/ncu_full_c4.log 2>&1
