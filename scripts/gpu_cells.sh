#!/bin/bash
mkdir -p gpurun_out
APML_CELL_STATS=1 python scripts/cell_stats.py C5:7 C5:6 C5:5 C4:5 C4:4 C2:3 C2:4 > gpurun_out/cell_stats.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "fallback_paths or C4 or C5 or rowshard or grad_gt_every" 2>&1 | tail -15 > gpurun_out/pytest_cells.txt
for b in 5 6 7; do APML_CELL_BITS=$b python bench.py --config C5 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5b$b.json 2>&1; done
for b in 4 5; do APML_CELL_BITS=$b python bench.py --config C4 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4b$b.json 2>&1; done
for b in 3 4; do APML_CULL=1 APML_CELL_BITS=$b python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2b$b.json 2>&1; done
python scripts/summ.py c5b5 c5b6 c5b7 c4b4 c4b5 c2b3 c2b4 > gpurun_out/summary_cells.txt 2>&1
