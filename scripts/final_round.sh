#!/bin/bash
# Round-end evidence: full GPU tests, smoke, bench lines for every config, phase split, ncu.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/f_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1
python bench.py > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
for c in C3 C3R; do python bench.py --config $c --no-cpu-baseline > gpurun_out/f_${c,,}.json 2>&1; done
for c in C4 C5; do python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/f_${c,,}.json 2>&1; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref_c2.json 2>&1
python scripts/phases.py C2 C3 > gpurun_out/f_phases.txt 2>&1
bash scripts/profile_round.sh
