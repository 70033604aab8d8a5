#!/bin/bash
# parity (the cluster-path / full-sweep variants), smoke, and the C2 / C3 / C3R bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowshard.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_q2.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2>&1
python bench.py --config C3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>&1
python bench.py --config C3R --no-cpu-baseline --no-e2e > gpurun_out/bench_c3r.json 2>&1
python scripts/summ.py c2 c3 c3r > gpurun_out/summary_q2.txt 2>&1
