#!/bin/bash
# quick GPU iteration: parity tests (-k filter optional), phase breakdown, C2/C3 bench lines
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
timeout 900 python -m pytest tests -m gpu -q -x "${KARG[@]}" 2>&1 | tail -15 > gpurun_out/q_pytest.txt
python scripts/phases.py C2 C3 > gpurun_out/q_phases.txt 2>&1
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_c2.json 2>&1
python bench.py --config C3 --no-cpu-baseline --no-e2e > gpurun_out/q_c3.json 2>&1
