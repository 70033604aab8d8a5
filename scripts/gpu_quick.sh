#!/bin/bash
# One gpurun call for iteration: fp32 peak micro, parity diagnostics, selected GPU tests, C2 bench.
# usage: scripts/gpu_quick.sh "<pytest -k expr>"
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak scripts/micro/fp32_peak.cu && /tmp/fp32_peak > gpurun_out/fp32_peak.json 2>&1
timeout 600 python scripts/parity_diag.py > gpurun_out/parity_diag.txt 2>&1
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -q -k "$1" 2>&1 | tail -25 > gpurun_out/pytest_quick.txt; fi
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
