#!/bin/bash
mkdir -p gpurun_out
for c in C5 C4; do python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c,,}.json 2>&1; done
python scripts/summ.py c5 c4 > gpurun_out/summary_cells.txt 2>&1
