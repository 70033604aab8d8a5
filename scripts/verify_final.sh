#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/v_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.txt 2>&1
python bench.py > gpurun_out/v_c2.json 2> gpurun_out/v_c2.err
