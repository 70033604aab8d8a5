#!/bin/bash
# culled-sweep iteration: parity tests of the culled paths + C4/C5 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fallback or C4 or rowshard or fig2" 2>&1 | tail -3 > gpurun_out/qc_pytest.txt
for c in C4 C5; do python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/qc_$c.json 2>&1; done
