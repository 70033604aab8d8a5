#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/w_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/w_smoke.txt 2>&1
python bench.py > gpurun_out/w_c2.json 2> gpurun_out/w_c2.err
for c in C3 C3R; do python bench.py --config $c --no-cpu-baseline > gpurun_out/w_${c,,}.json 2>&1; done
python bench.py --config C4 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/w_c4.json 2>&1
