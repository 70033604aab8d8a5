#!/bin/bash
# A/B of the fused culled Pass A (APML_CULL_BOTH) on C4/C5 + the culled parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fallback or C4 or rowshard or fig2 or cull" 2>&1 | tail -3 > gpurun_out/cb_pytest.txt
for c in C4 C5; do for v in 1 0 1 0; do
  APML_CULL_BOTH=$v python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$c','both=$v',d['value'],d['ms_per_step'])" >> gpurun_out/cb_bench.txt
done; done
