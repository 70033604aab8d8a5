#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fallback_paths or C4 or rowshard or grad_gt_every" 2>&1 | tail -2 > gpurun_out/pytest_grid.txt
for c in C4 C5; do python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c,,}.json 2>&1; done
python scripts/summ.py c4 c5 > gpurun_out/summary_grid.txt 2>&1
