import sys, os; sys.path.insert(0, os.getcwd())
import torch
from bench import CONFIGS
from paper_2512_19743_b200 import Config, Plan, forward
from synth import clouds
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
B, N, M = c["B"], c["N"], c["M"]
x, y = clouds.batch(c["kind"], B, N, M, 0)
pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
ones = torch.ones(B, device="cuda"); loss_buf = torch.empty(B, device="cuda"); grad_buf = torch.empty_like(pred)
def make_graph(cfg):
    p = Plan(B, N, M, cfg)
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            p.forward(pred, gt, loss_buf); p.backward(ones, out=grad_buf)
    torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
    print(" warm", loss_buf.sum().item(), p.stats()["nnz_total"])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        p.forward(pred, gt, loss_buf); p.backward(ones, out=grad_buf)
    return p, g
for name, cfg in (("all", Config(sync_check=False, stage_timing=True)), ("none", Config(sync_check=False)),
                  ("m10", Config(sync_check=False, stage_timing=True, stage_marks=10))):
    p, g = make_graph(cfg)
    for k in range(3):
        g.replay(); torch.cuda.synchronize()
        print(name, k, loss_buf.sum().item(), p.stats()["nnz_total"])
    p.close(); del g
