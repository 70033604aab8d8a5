#!/bin/bash
# culled emit: 1 vs kRc groups per warp at C4 / C5 (APML_EMIT_R), + the culled parity variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "CULL or cull" 2>&1 | tail -3 > gpurun_out/e_pytest.txt
for c in C5 C4; do for r in 1 2; do
  APML_EMIT_R=$r python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/e_${c,,}_r$r.json 2>&1
done; done
python bench.py --config C5 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/e_c5_def.json 2>&1
