"""Host-side model of the culled sweeps (k_cull.cuh) to choose culling strategies without a GPU.

For one synthetic pair it reproduces the Morton order, the 128-point tiles and the bounds of
k_line_top2_cull / k_emit_cull and counts the (warp, tile) pairs each strategy evaluates,
as a fraction of the brute-force sweep.  Exact nearest neighbours come from scipy's KD-tree
(this script is a design aid; it is not part of the product or the tests).

    python scripts/cull_sim.py --kind shapenet --n 16384 [--order ring|sorted]
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np
from scipy.spatial import cKDTree

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TQ = 128
WARP_PTS = 128  # R * 32 points per warp
CTA_PTS = 512


def morton_sort(p, bb, bits):
    ext = np.maximum(bb[1] - bb[0], 1e-30)
    c = np.clip(((p - bb[0]) / ext * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    key = np.zeros(len(p), np.int64)
    for b in range(bits):
        for d in range(3):
            key |= ((c[:, d] >> b) & 1) << (3 * b + d)
    return np.argsort(key, kind="stable")


def boxes(p, size):
    n = len(p)
    nb = (n + size - 1) // size
    lo = np.full((nb, 3), np.inf)
    hi = np.full((nb, 3), -np.inf)
    for t in range(nb):
        q = p[t * size:(t + 1) * size]
        lo[t] = q.min(0)
        hi[t] = q.max(0)
    return lo, hi


def lb2(alo, ahi, blo, bhi):
    """squared box distance, a [na] x b [nb]"""
    g = np.maximum(0, np.maximum(alo[:, None, :] - bhi[None, :, :], blo[None, :, :] - ahi[:, None, :]))
    return (g * g).sum(-1)


def line_stats(own, other, lam, rho, delta=1e-6, eps_g=1e-8):
    d, _ = cKDTree(other).query(own, k=2)
    m, c2 = d[:, 0], d[:, 1]
    g = np.maximum(c2 - m + delta, eps_g)
    R = m + rho * g
    R2 = np.maximum(R * R, m * m)
    s2 = c2 * c2
    return s2, np.maximum(R2, s2)


def sim(x, y, order="ring", warp_pts=WARP_PTS, tq=TQ, progressive=True):
    N, M = len(x), len(y)
    K = M
    p = 0.9
    lam = -math.log((1 - p) / ((K - 1) * p))
    rho = math.log(1e8) / lam
    bb = np.stack([np.minimum(x.min(0), y.min(0)), np.maximum(x.max(0), y.max(0))])
    bits = min(7, max(2, (int(math.ceil(math.log2(max(N, M)))) + 2) // 3))
    xs = x[morton_sort(x, bb, bits)]
    ys = y[morton_sort(y, bb, bits)]
    s2x, e2x = line_stats(xs, ys, lam, rho)
    s2y, e2y = line_stats(ys, xs, lam, rho)
    wlo, whi = boxes(xs, warp_pts)
    tlo, thi = boxes(ys, tq)
    nw, nt = len(wlo), len(tlo)
    L = lb2(wlo, whi, tlo, thi) * (1 - 1e-5)
    # final per-warp bounds
    wmax_s = np.array([s2x[w * warp_pts:(w + 1) * warp_pts].max() for w in range(nw)])
    wmax_e = np.array([e2x[w * warp_pts:(w + 1) * warp_pts].max() for w in range(nw)])
    tmax_e = np.array([e2y[t * tq:(t + 1) * tq].max() for t in range(nt)])
    ideal_A = (L <= wmax_s[:, None]).mean()
    emit = (L <= np.maximum(wmax_e[:, None], tmax_e[None, :])).mean()
    emit_row_only = (L <= wmax_e[:, None]).mean()
    emit_col_only = (L <= tmax_e[None, :]).mean()
    out = dict(nw=nw, nt=nt, passA_ideal=ideal_A, emit=emit, emit_rowside=emit_row_only,
               emit_colside=emit_col_only)
    if progressive:
        # simulate the progressive bound in ring or sorted order (per warp, ignoring CTA grouping)
        evals = 0
        wpc = CTA_PTS // warp_pts
        for w in range(nw):
            pts = xs[w * warp_pts:(w + 1) * warp_pts]
            cta = w // wpc
            if order == "ring":
                t0 = min(nt - 1, (cta * CTA_PTS * nt * tq // max(N, 1)) // tq)
                seq = [t0]
                for dd in range(1, nt):
                    for t in (t0 + dd, t0 - dd):
                        if 0 <= t < nt:
                            seq.append(t)
            else:
                seq = list(np.argsort(L[w], kind="stable"))
            m = np.full(len(pts), np.inf)
            s = np.full(len(pts), np.inf)
            for t in seq:
                if L[w, t] > s.max():
                    if order == "sorted":
                        break
                    continue
                evals += 1
                q = ys[t * tq:(t + 1) * tq]
                d = ((pts[:, None, :] - q[None, :, :]) ** 2).sum(-1)
                both = np.concatenate([np.stack([m, s], 1), d], 1)
                both.sort(1)
                m, s = both[:, 0], both[:, 1]
        out["passA_" + order] = evals / (nw * nt)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="shapenet")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--order", default="ring")
    ap.add_argument("--warp-pts", type=int, default=WARP_PTS)
    ap.add_argument("--tq", type=int, default=TQ)
    ap.add_argument("--no-progressive", action="store_true")
    a = ap.parse_args()
    from synth import clouds
    x, y = clouds.pair(a.kind, a.n, a.n, seed=a.seed)
    r = sim(x.astype(np.float64), y.astype(np.float64), a.order, a.warp_pts, a.tq, not a.no_progressive)
    print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})


if __name__ == "__main__":
    main()
