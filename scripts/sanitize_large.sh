#!/bin/bash
# compute-sanitizer memcheck on the global-memory fallbacks (32-bit indices, no shared-memory
# replicas / slices) at a size the oracle can check.
cat > /tmp/san.py <<'PY'
import os, sys; sys.path.insert(0, os.environ['REPO'])
import torch, numpy as np
from paper_2512_19743_b200 import Config, forward
from synth import clouds
x, y = clouds.batch(os.environ.get("KIND", "uniform"), 1, int(os.environ.get("NN", 3000)), int(os.environ.get("MM", 2500)), 3)
p, g = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
loss, ctx = forward(p, g, Config())
gr = ctx.backward(torch.ones(1, device="cuda"))
torch.cuda.synchronize()
print("loss", loss.item(), float(gr.abs().sum()))
PY
REPO=$PWD APML_FORCE_IDX32=1 APML_SMEM_LIMIT=40000 APML_CL=8 compute-sanitizer --tool memcheck --show-backtrace no python /tmp/san.py 2>&1 | head -40
REPO=$PWD KIND=scene NN=${NN2:-40000} MM=${NN2:-40000} APML_FORCE_IDX32=1 APML_SMEM_LIMIT=40000 APML_CL=8 compute-sanitizer --tool memcheck --show-backtrace no python /tmp/san.py 2>&1 | head -40
REPO=$PWD KIND=scene NN=262144 MM=262144 CUDA_LAUNCH_BLOCKING=1 python /tmp/san.py 2>&1 | tail -5
