#!/bin/bash
# Round-end evidence (one gpurun call): the full GPU suite, smoke, bench lines of every config,
# the reference arm at C2, the phase split, then scripts/profile_round.sh (ncu + Fig. 2).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/f_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in C3 C3R; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c,,}.json 2>&1; done
for c in C4 C5; do python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/bench_${c,,}.json 2>&1; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref_c2.json 2>&1
python scripts/summ.py c2 c3 c3r c4 c5 > gpurun_out/bench_summary.txt 2>&1
python scripts/phases.py C2 C3 > gpurun_out/f_phases.txt 2>&1
bash scripts/profile_round.sh
