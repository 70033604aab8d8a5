#!/bin/bash
# Compare sweep variants: bench C2/C4 stage times for each libapml_*.so
mkdir -p gpurun_out
for lib in paper_2512_19743_b200/libapml.so paper_2512_19743_b200/libapml_r*.so; do
  n=$(basename $lib .so)
  APML_LIB=$PWD/$lib python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_${n}_c4.json 2>&1
  APML_LIB=$PWD/$lib python bench.py --config C2 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/var_${n}_c2.json 2>&1
done
