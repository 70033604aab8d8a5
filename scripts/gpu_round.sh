#!/bin/bash
bash scripts/gpu_check.sh
python bench.py --config C5 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
