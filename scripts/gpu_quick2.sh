#!/bin/bash
# parity (the cluster-path variants + smoke-size cases) and the C2 / C3 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_q2.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1
python bench.py --config C3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>&1
APML_ENTRY_SIM=0 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2n.json 2>&1
python scripts/phases.py C2 > gpurun_out/phases_c2.txt 2>&1
python scripts/summ.py c2 c2n c3 > gpurun_out/summary_q2.txt 2>&1
