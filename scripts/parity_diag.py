"""Diagnostic (test infrastructure): per-entry P0 / v errors of the GPU path against the oracle,
with the derived per-entry P0 bound, on a few cases.  Prints a table."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import SparsePlan, OracleConfig
from synth import clouds
from paper_2512_19743_b200 import Config, forward

U = 2.0 ** -24
def lam(K, p): return math.log((K - 1) * p / (1 - p)) if K > 1 else 0.0

for kind, B, N, M, seed, env in [("shapenet", 2, 2048, 2048, 100, {}), ("mmfi", 2, 1024, 512, 200, {}),
                                  ("uniform", 2, 700, 650, 17, {}), ("scene", 1, 1500, 1200, 10, {})]:
    x, y = clouds.batch(kind, B, N, M, seed)
    cfg = Config()
    loss, ctx = forward(torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda"), cfg)
    torch.cuda.synchronize()
    oc = OracleConfig()
    for b in range(B):
        pl = SparsePlan(x[b], y[b], oc)
        o = pl.support(); g = ctx.support(b)
        rows, cols = pl.lines(0), pl.lines(1)
        key_o = {(int(i), int(j)): k for k, (i, j) in enumerate(zip(o["i"], o["j"]))}
        idx = [(k, key_o.get((int(i), int(j)))) for k, (i, j, f) in enumerate(zip(g["i"], g["j"], g["flags"])) if f]
        idx = [(a, c) for a, c in idx if c is not None]
        ga = np.array([a for a, _ in idx]); oa = np.array([c for _, c in idx])
        p0g, p0o = g["p0"][ga].astype(np.float64), o["p0"][oa]
        vg, vo = g["v"][ga].astype(np.float64), o["v"][oa]
        i_, j_ = o["i"][oa], o["j"][oa]
        def bound(ln, k, K):
            m, c2, gg = ln["m"][k], ln["c2"][k], ln["g"][k]
            return U * ((74 * (c2 + m) + 8 * lam(K, 0.9) * m) / gg + 110)
        bd = np.maximum(np.where(o["flags"][oa] & 1, bound(rows, i_, M), 0), np.where(o["flags"][oa] & 2, bound(cols, j_, N), 0))
        rel = np.abs(p0g - p0o) / p0o
        relv = np.abs(vg - vo) / np.maximum(vo, 1e-30)
        nv = np.linalg.norm(vg - vo) / np.linalg.norm(vo)
        print(f"{kind} {N}x{M} b{b}: nnz {len(oa)} P0 rel med {np.median(rel):.2e} p99 {np.percentile(rel,99):.2e} max {rel.max():.2e}; "
              f"rel/bound max {np.max(rel/bd):.3f}; bound med {np.median(bd):.2e}; v normwise {nv:.2e} rel med {np.median(relv):.2e} max {relv.max():.2e} "
              f"(max at v={vo[np.argmax(relv)]:.2e})")
