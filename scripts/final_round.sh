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
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB pull limit)
mkdir -p gpurun_out/profiles
for c in c2 c4 c5; do python scripts/launch_summary.py r02_$c gpurun_out/launches_$c.csv 2 > /dev/null 2>&1; done
python scripts/ncu_summary.py r02 gpurun_out/full_c2.ncu-rep gpurun_out/full_c4.ncu-rep gpurun_out/full_c4cells.ncu-rep gpurun_out/full_c5.ncu-rep > /dev/null 2>&1
for rep in full_c2 full_c4cells full_c5; do
  ncu -i gpurun_out/$rep.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src.csv 2>/dev/null
  python scripts/ncu_lines.py /tmp/src.csv 30 > gpurun_out/profiles/r02_${rep}_lines.txt 2>&1
done
cp profiles/r02_c*_launches.md profiles/r02_ncu.md profiles/ncu_traffic.json profiles/fig2_nnz.* gpurun_out/profiles/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
