#!/bin/bash
# One gpurun call: GPU parity tests + bench lines (C2 default, C3, C4) into gpurun_out/.
# usage: scripts/gpu_check.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
timeout 1500 python -m pytest tests -m gpu -q -x "${KARG[@]}" 2>&1 | tail -25 > gpurun_out/pytest_gpu.txt
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1
python bench.py --config C4 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2>&1
