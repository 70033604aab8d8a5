#!/bin/bash
# One gpurun call for iteration: selected GPU tests and bench lines.
# usage: scripts/gpu_quick.sh "<pytest -k expr>" [configs...]   (configs default: C2)
mkdir -p gpurun_out
if [ -n "$1" ]; then timeout 1500 python -m pytest tests -m gpu -q -k "$1" 2>&1 | tail -3 > gpurun_out/pytest_quick.txt; fi
shift
for c in ${@:-C2}; do python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c,,}.json 2>&1; done
python scripts/summ.py $(for c in ${@:-C2}; do echo ${c,,}; done) > gpurun_out/summary_quick.txt 2>&1
