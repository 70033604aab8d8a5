#!/bin/bash
# The cell-grid sweeps with in-kernel bounds checks (a -DAPML_CELL_CHECKS=1 build shipped in
# place of the default library): the culled parity tests and the full-size C4 / C5 checks.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "cell_sweeps or fallback_paths or C4 or C5 or rowshard or grad_gt_every or uniform_fallback" 2>&1 | tail -4 > gpurun_out/cell_checks.txt
