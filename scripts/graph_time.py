"""Step time of a CUDA-graph replay of a plan's forward + backward WITHOUT stage events (the
stage-timing event records sit between the kernels and can hide launch-overlap effects).
usage: graph_time.py [config] [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS
from paper_2512_19743_b200 import Config, Plan
from synth import clouds
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
c = CONFIGS[name]
x, y = clouds.batch(c["kind"], c["B"], c["N"], c["M"], 0)
pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
ones = torch.ones(c["B"], device="cuda")
loss = torch.empty(c["B"], device="cuda"); grad = torch.empty_like(pred)
for timing in (False, True):
    plan = Plan(c["B"], c["N"], c["M"], Config(sync_check=False, stage_timing=timing))
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            plan.forward(pred, gt, loss); plan.backward(ones, out=grad)
    torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.forward(pred, gt, loss); plan.backward(ones, out=grad)
    for _ in range(5): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): g.replay()
    e1.record(); torch.cuda.synchronize()
    print(f"{name} stage_timing={timing} PDL={os.environ.get('APML_PDL', '1')}: {e0.elapsed_time(e1) / steps * 1e3:.1f} us/step (back-to-back replays, L2 warm)")
    plan.close()
