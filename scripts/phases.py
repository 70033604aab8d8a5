"""Per-phase breakdown of the sparse megakernels (APML_PHASES=1) for a bench config."""
import os, sys
os.environ["APML_PHASES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS
from paper_2512_19743_b200 import Config, forward
from synth import clouds
for name in sys.argv[1:] or ["C2"]:
    c = CONFIGS[name]
    x, y = clouds.batch(c["kind"], c["B"], c["N"], c["M"], 0)
    p, g = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    for _ in range(3):
        print(name, flush=True)
        loss, ctx = forward(p, g, Config(sync_check=False))
        ctx.backward(torch.ones(c["B"], device="cuda"))
        torch.cuda.synchronize()
