mkdir -p gpurun_out
for b in "" 4 5; do echo "bits=$b"; APML_CELL_BITS=$b python scripts/fig2.py --trials 4 --min-n 8192 --max-n 65536 --no-write; done > gpurun_out/fig2_quick.txt 2>&1
