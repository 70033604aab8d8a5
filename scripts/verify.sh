#!/bin/bash
# full GPU parity suite + smoke + bench lines for C2/C4/C5
mkdir -p gpurun_out; rm -f gpurun_out/v_bench.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/v_pytest.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/v_pytest.txt 2>&1
for c in C2 C4 C5; do python bench.py --config $c --steps 10 --no-cpu-baseline 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$c',d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline'])" >> gpurun_out/v_bench.txt
done
