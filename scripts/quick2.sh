#!/bin/bash
bash scripts/quick.sh "$@"
ncu --set full --clock-control none --import-source on -k regex:"k_sparse" -s 2 -c 2 -o gpurun_out/sp_q python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
