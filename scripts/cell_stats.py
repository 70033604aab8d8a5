"""Diagnostics of the cell sweeps: counters of one forward per (config, bits).  Needs a build with
APML_CELL_DIAG: python -c "from paper_2512_19743_b200.build import build; build(True, defines=['APML_CELL_DIAG=1'])"
then APML_CELL_STATS=1 python scripts/cell_stats.py C5 C4:4 ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS
from paper_2512_19743_b200 import Config, forward
from synth import clouds
for arg in sys.argv[1:]:
    name, bits = (arg.split(":") + [""])[:2]
    c = CONFIGS[name]
    if bits: os.environ["APML_CELL_BITS"] = bits
    else: os.environ.pop("APML_CELL_BITS", None)
    os.environ["APML_CULL"] = "1"
    x, y = clouds.batch(c["kind"], c["B"], c["N"], c["M"], 0)
    p, g = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    print(name, bits, flush=True)
    loss, ctx = forward(p, g, Config(sync_check=False))
    torch.cuda.synchronize()
