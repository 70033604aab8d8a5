#!/bin/bash
# split-target sweep at C3 / C3R (the full-sweep Pass A + emit split of the streamed cloud)
mkdir -p gpurun_out
B="python bench.py --steps 20 --no-cpu-baseline --no-e2e"
for st in 2368 4736 9472 18944; do APML_SPLIT_TARGET=$st $B --config C3 > gpurun_out/k2_c3_st$st.json 2>&1; done
for st in 2368 4736 9472; do APML_SPLIT_TARGET=$st $B --config C3R > gpurun_out/k2_c3r_st$st.json 2>&1; done
for st in 2368 4736 9472; do APML_SPLIT_TARGET=$st $B --config C4 --steps 5 > gpurun_out/k2_c4_st$st.json 2>&1; done
