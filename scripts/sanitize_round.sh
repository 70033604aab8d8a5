#!/bin/bash
# compute-sanitizer memcheck (and racecheck on shared memory) over the current default paths:
# fwd2/bwd2 cluster kernels (C2-like, CL = 4), single-CTA clusters (C3-like), ragged, culled
# sweeps + grid sparse stage, the plan + grad w.r.t. gt.  Small sizes (sanitizer is slow).
mkdir -p gpurun_out
cat > /tmp/san2.py <<'PY'
import os, sys; sys.path.insert(0, os.environ['REPO'])
import torch
from paper_2512_19743_b200 import Config, forward, Plan
from synth import clouds
kind, B, N, M = os.environ["KIND"], int(os.environ["B"]), int(os.environ["NN"]), int(os.environ["MM"])
x, y = clouds.batch(kind, B, N, M, 5)
p, g = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
ns = ms = None
if os.environ.get("RAGGED"):
    ns = [N - 37 * b for b in range(B)]; ms = [M - 11 * b for b in range(B)]
cfg = Config(stability="uniform") if os.environ.get("UNIFORM") else Config()
if os.environ.get("UNIFORM"):
    y[:, 5:15] = y[:, 20:30]; g = torch.tensor(y, device="cuda")  # duplicated gt points
loss, ctx = forward(p, g, cfg, n_sizes=ns, m_sizes=ms)
gp, gg = ctx.backward(torch.ones(B, device="cuda"), want_gt=True)
if os.environ.get("PLAN"):
    pl = Plan(B, N, M, Config(sync_check=False))
    pl.forward(p, g); pl.backward(torch.ones(B, device="cuda"))
torch.cuda.synchronize()
print("ok", float(loss.sum()), float(gp.abs().sum()), float(gg.abs().sum()))
PY
run() { echo "== $*"; env REPO=$PWD "$@" compute-sanitizer --tool memcheck --show-backtrace no --print-limit 5 python /tmp/san2.py 2>&1 | tail -4; }
run KIND=shapenet B=4 NN=1024 MM=1024 PLAN=1
run KIND=mmfi B=2 NN=1024 MM=512 APML_CL=1
run KIND=mmfi B=3 NN=700 MM=520 RAGGED=1
run KIND=uniform B=2 NN=4500 MM=4200 APML_CULL=1
run KIND=scene B=1 NN=9000 MM=8000
run KIND=uniform B=2 NN=4500 MM=4200 APML_CULL=1 APML_CULL_MODE=0
run KIND=uniform B=1 NN=5000 MM=5000 APML_CELL_BITS=6
run KIND=uniform B=2 NN=700 MM=650 APML_FWD2=0
run KIND=uniform B=2 NN=700 MM=650 UNIFORM=1
run KIND=uniform B=2 NN=700 MM=650 APML_GRID=1 APML_RS_COLLECTIVES=1
echo "== racecheck (shared memory), fwd2/bwd2 CL=1"
env REPO=$PWD KIND=mmfi B=1 NN=512 MM=256 APML_CL=1 compute-sanitizer --tool racecheck --print-limit 5 python /tmp/san2.py 2>&1 | tail -6
echo "== racecheck (shared memory), the cell-grid sweeps (k_cells.cuh) + grid sparse stage"
env REPO=$PWD KIND=scene B=1 NN=5000 MM=5000 compute-sanitizer --tool racecheck --print-limit 5 python /tmp/san2.py 2>&1 | tail -6
echo "== synccheck (barrier / cluster-barrier divergence), fwd2/bwd2 CL=4 and the grid path"
env REPO=$PWD KIND=shapenet B=2 NN=1024 MM=1024 APML_CL=4 compute-sanitizer --tool synccheck --print-limit 5 python /tmp/san2.py 2>&1 | tail -4
env REPO=$PWD KIND=uniform B=2 NN=700 MM=650 APML_GRID=1 compute-sanitizer --tool synccheck --print-limit 5 python /tmp/san2.py 2>&1 | tail -4
echo "== initcheck (reads of uninitialised device memory), default path + plan"
env REPO=$PWD KIND=shapenet B=2 NN=1024 MM=1024 PLAN=1 compute-sanitizer --tool initcheck --print-limit 5 python /tmp/san2.py 2>&1 | tail -4
env REPO=$PWD KIND=scene B=1 NN=5000 MM=5000 compute-sanitizer --tool initcheck --print-limit 5 python /tmp/san2.py 2>&1 | tail -4
