#!/bin/bash
# Full GPU suite + smoke + bench lines of every config (one gpurun call).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_all.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in C3 C3R C4 C5; do python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/bench_${c,,}.json 2>&1; done
python scripts/summ.py c2 c3 c3r c4 c5 > gpurun_out/bench_summary.txt 2>&1
