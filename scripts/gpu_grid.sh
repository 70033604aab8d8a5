#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "fallback_paths or C4 or C5 or rowshard or grad_gt or nccl or ragged or plan or cell_sweeps or uniform" 2>&1 | tail -2 > gpurun_out/pytest_grid.txt
for c in C4 C5; do python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c,,}.json 2>&1; done
python scripts/summ.py c4 c5 > gpurun_out/summary_grid.txt 2>&1
python scripts/fig2.py --trials 20 --min-n 65536 --max-n 65536 --no-write > gpurun_out/fig2_65k.txt 2>&1
