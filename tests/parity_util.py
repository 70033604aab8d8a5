"""Comparison helpers for GPU-vs-oracle parity (test code).

* boundary band: an entry whose keep decision (s >= tau) is not determined by
  the fp32 inputs to within 4 ulps of c, m and c2 -- the GPU decides d2 <= R^2 in fp32, the
  oracle decides exp(-T (c - m)) >= tau in fp64; outside the band they must agree exactly.
* well-conditioned set: pred points none of whose gap-defining lines has
  Lambda * s^2 / g^2 >= 1e6 (s = median row-NN distance of the pair); on near-tie lines the
  T-path amplifies fp32 rounding by ~Lambda/g^2.
"""
from __future__ import annotations

import math

import numpy as np

U = 2.0 ** -24  # fp32 unit roundoff


def _lam(K: int, p: float) -> float:
    return math.log((K - 1) * p / (1 - p)) if K > 1 else 0.0


def _exp_interval(c, m, c2, K, p, delta, eps_g, ulps=4):
    """Interval of e = Lambda (c - m) / g over c, m, c2 widened by +-ulps fp32 ulps."""
    w = ulps * U
    lam = _lam(K, p)
    clo, chi = c * (1 - w), c * (1 + w)
    mlo, mhi = m * (1 - w), m * (1 + w)
    c2lo, c2hi = c2 * (1 - w), c2 * (1 + w)
    glo = max(c2lo - mhi + delta, eps_g)
    ghi = max(c2hi - mlo + delta, eps_g)
    nlo, nhi = clo - mhi, chi - mlo
    cands = [lam * n / g for n in (nlo, nhi) for g in (glo, ghi)]
    return min(cands), max(cands)


def boundary(x, y, plan, i, j, cfg) -> bool:
    """Is (i, j) in the boundary band of either direction?"""
    if cfg.tau <= 0.0:
        return False
    lt = math.log(1.0 / cfg.tau)
    c = float(np.linalg.norm(x[i].astype(np.float64) - y[j].astype(np.float64)))
    N, M = x.shape[0], y.shape[0]
    rows, cols = plan.lines(0), plan.lines(1)
    for K, ln, k in ((M, rows, i), (N, cols, j)):
        if K <= 1:
            continue
        lo, hi = _exp_interval(c, ln["m"][k], ln["c2"][k], K, cfg.p_min, cfg.delta, cfg.eps_g)
        if lo <= lt <= hi:
            return True
    return False


def support_diff(gpu_sup, orc_sup, keep_only=True):
    """Sets of (i, j) (flags != 0) present on one side only."""
    g = {(int(a), int(b)) for a, b, f in zip(gpu_sup["i"], gpu_sup["j"], gpu_sup["flags"]) if f or not keep_only}
    o = {(int(a), int(b)) for a, b in zip(orc_sup["i"], orc_sup["j"])}
    return g - o, o - g


def flags_map(sup) -> dict:
    return {(int(a), int(b)): int(f) for a, b, f in zip(sup["i"], sup["j"], sup["flags"])}


def well_conditioned(x, y, plan, cfg, thresh=1e6, skip_clamped=False) -> np.ndarray:
    """Boolean mask over pred points (see module doc).  skip_clamped: lines whose gap clamp is
    active are not excluded -- the clamp zeroes their T-path gradient (g-bar = 0), the
    path through which near-tie lines amplify rounding."""
    N, M = x.shape[0], y.shape[0]
    rows, cols = plan.lines(0), plan.lines(1)
    s = float(np.median(rows["m"]))
    ok = np.ones(N, bool)
    if M > 1:
        bad_r = _lam(M, cfg.p_min) * s * s / np.maximum(rows["g"], 1e-300) ** 2 >= thresh
        if skip_clamped:  # (and uniform-fallback lines: T = 0, no T-path gradient either)
            bad_r &= (rows["clamped"] == 0) & (rows["uniform"] == 0)
        ok &= ~bad_r
    if N > 1:
        bad_c = _lam(N, cfg.p_min) * s * s / np.maximum(cols["g"], 1e-300) ** 2 >= thresh
        if skip_clamped:
            bad_c &= (cols["clamped"] == 0) & (cols["uniform"] == 0)
        for j in np.nonzero(bad_c)[0]:
            for i in (cols["a"][j], cols["b"][j]):
                if i >= 0:
                    ok[i] = False
    return ok


def normwise(a, b) -> float:
    d = np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64))
    n = np.linalg.norm(np.asarray(b, np.float64))
    return d / n if n > 0 else d


def well_conditioned_gt(x, y, plan, cfg, thresh=1e6) -> np.ndarray:
    """Boolean mask over gt points: the gt analogue of well_conditioned (column j's own line
    and every row whose argmin / second argmin is j)."""
    N, M = x.shape[0], y.shape[0]
    rows, cols = plan.lines(0), plan.lines(1)
    s = float(np.median(rows["m"]))
    ok = np.ones(M, bool)
    if N > 1:
        ok &= ~(_lam(N, cfg.p_min) * s * s / np.maximum(cols["g"], 1e-300) ** 2 >= thresh)
    if M > 1:
        bad_r = _lam(M, cfg.p_min) * s * s / np.maximum(rows["g"], 1e-300) ** 2 >= thresh
        for i in np.nonzero(bad_r)[0]:
            for j in (rows["a"][i], rows["b"][i]):
                if j >= 0:
                    ok[j] = False
    return ok


def p0_bound(plan, cfg, oi, oj, oflags) -> np.ndarray:
    """Derived per-entry relative bound on the fp32 P0.  Per direction,
    with u the fp32 unit roundoff and the GPU evaluating c = sqrt(d2) (rel. err ~2u),
    g = c2 - m + delta (abs. err ~2u (c2 + m)), T = Lambda / g (rel. err ~2u (c2 + m) / g + u),
    e = T (c - m) <= ln(1/tau) on kept entries (abs. err <= e relT + 2u T (c + m)), s = exp(-e)
    (+2u), Z = sum s and P = s / Z (each at most the worst s error of the line):
        eps_dir <= u [ (74 (c2 + m) + 8 Lambda m) / g + 110 ]     (ln(1/tau) = 18.4 folded in)
    and P0 = (P_row + P_col) / 2 takes the larger of its directions."""
    rows, cols = plan.lines(0), plan.lines(1)
    N, M = plan.N, plan.M

    def line_bound(ln, k, K):
        m, c2, g = ln["m"][k], ln["c2"][k], ln["g"][k]
        c2 = np.where(np.isfinite(c2), c2, m)
        return U * ((74.0 * (c2 + m) + 8.0 * _lam(K, cfg.p_min) * m) / np.maximum(g, 1e-300) + 110.0)

    br = np.where(oflags & 1, line_bound(rows, oi, M), 0.0) if M > 1 else np.zeros(len(oi))
    bc = np.where(oflags & 2, line_bound(cols, oj, N), 0.0) if N > 1 else np.zeros(len(oi))
    return np.maximum(np.maximum(br, bc), 4 * U)


def match_support(gpu_sup, orc_sup):
    """Index arrays (gpu positions, oracle positions) of the entries both sides keep (flags != 0)."""
    key_o = {(int(i), int(j)): k for k, (i, j) in enumerate(zip(orc_sup["i"], orc_sup["j"]))}
    ga, oa = [], []
    for k, (i, j, f) in enumerate(zip(gpu_sup["i"], gpu_sup["j"], gpu_sup["flags"])):
        if f:
            o = key_o.get((int(i), int(j)))
            if o is not None:
                ga.append(k)
                oa.append(o)
    return np.asarray(ga, np.int64), np.asarray(oa, np.int64)
