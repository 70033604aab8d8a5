#!/bin/bash
# Fig. 2 with the paper's 500 trials at every N (64 ... 262,144)
mkdir -p gpurun_out/profiles
timeout 3000 python scripts/fig2.py --trials 500 --all-large > gpurun_out/fig2_full.log 2>&1
cp profiles/fig2_nnz.csv profiles/fig2_nnz.md gpurun_out/profiles/ 2>/dev/null
