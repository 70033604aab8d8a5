#!/bin/bash
# A/B of R = 1 (finer work units) for the culled Pass A (APML_CULL_RA) and Pass B (APML_CULL_RB)
mkdir -p gpurun_out; rm -f gpurun_out/cr_bench.txt
timeout 600 python -m pytest tests -m gpu -q -x -k "C4 or cull" 2>&1 | tail -2 > gpurun_out/cr_pytest.txt
APML_CULL_RA=1 APML_CULL_RB=1 timeout 600 python -m pytest tests -m gpu -q -x -k "C4 or cull" 2>&1 | tail -2 >> gpurun_out/cr_pytest.txt
for c in C4 C5; do for v in "2 2" "1 2" "2 1" "1 1" "2 2"; do set -- $v
  APML_CULL_RA=$1 APML_CULL_RB=$2 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$c','RA=$1 RB=$2',d['value'],d['ms_per_step'], d.get('stages_ms',''))" >> gpurun_out/cr_bench.txt
done; done
