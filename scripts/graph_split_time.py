"""Cost of timing the backward kernel live: one graph with no marks vs two graphs (forward,
backward) with eager CUDA events between them vs one graph with two in-graph marks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS
from paper_2512_19743_b200 import Config, Plan
from synth import clouds
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = CONFIGS[name]
x, y = clouds.batch(c["kind"], c["B"], c["N"], c["M"], 0)
pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
ones = torch.ones(c["B"], device="cuda")
loss = torch.empty(c["B"], device="cuda"); grad = torch.empty_like(pred)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def cap(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g
def warm(p):
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            p.forward(pred, gt, loss); p.backward(ones, out=grad)
    torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
def timeit(run, n=30):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for k in range(n + 3):
        flush.fill_(k & 0xFF)
        if k >= 3: ev[k - 3][0].record()
        run()
        if k >= 3: ev[k - 3][1].record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return t[len(t) // 2] * 1e3
p = Plan(c["B"], c["N"], c["M"], Config(sync_check=False)); warm(p)
g1 = cap(lambda: (p.forward(pred, gt, loss), p.backward(ones, out=grad)))
print(name, "one graph, no marks: %.1f us" % timeit(g1.replay))
gf = cap(lambda: p.forward(pred, gt, loss)); gb = cap(lambda: p.backward(ones, out=grad))
e = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
def two():
    gf.replay(); e[0].record(); gb.replay(); e[1].record()
print(name, "two graphs + eager events: %.1f us" % timeit(two), " bwd %.1f us" % (e[0].elapsed_time(e[1]) * 1e3))
p.close()
p2 = Plan(c["B"], c["N"], c["M"], Config(sync_check=False, stage_timing=True, stage_marks=(1 << 7) | (1 << 8))); warm(p2)
g2 = cap(lambda: (p2.forward(pred, gt, loss), p2.backward(ones, out=grad)))
print(name, "one graph, 2 marks: %.1f us" % timeit(g2.replay), " bwd %.1f us" % (p2.stage_times()["sparse_bwd"] * 1e3))
