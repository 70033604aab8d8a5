#!/bin/bash
# C2 knob sweep: cluster size and the Pass A split target (bench stages_ms per setting)
mkdir -p gpurun_out
B="python bench.py --steps 20 --no-cpu-baseline --no-e2e"
for cl in 2 4 8; do APML_CL=$cl $B > gpurun_out/k_c2_cl$cl.json 2>&1; done
for st in 1184 2368 4736 9472; do APML_SPLIT_TARGET=$st $B > gpurun_out/k_c2_st$st.json 2>&1; done
for st in 1184 2368 4736; do APML_SPLIT_TARGET=$st $B --config C3 > gpurun_out/k_c3_st$st.json 2>&1; done
