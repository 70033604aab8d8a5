#!/bin/bash
mkdir -p gpurun_out
for mb in 64 125 216 343 512; do
  for c in C4 C5; do APML_CELL_MAXBLOCK=$mb python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c,,}m$mb.json 2>&1; done
done
python scripts/summ.py c4m64 c4m125 c4m216 c4m343 c4m512 c5m64 c5m125 c5m216 c5m343 c5m512 > gpurun_out/summary_sweep.txt 2>&1
