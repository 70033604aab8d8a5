"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Every test here checks the oracle against something other than itself: hand-derived closed
forms (tests/golden/closed_forms.json), special cases that reduce to textbook quantities,
brute force on tiny inputs, finite differences, invariants, and torch-CPU-fp64 autograd of an
independently written dense masked formulation.  PAPER.md citations as P:<line>.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import OracleConfig, dense_forward, sparse_forward, temperature
from synth import clouds

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def _cost(x, y):
    x = np.asarray(x, np.float64); y = np.asarray(y, np.float64)
    return np.sqrt(((x[:, None, :] - y[None, :, :]) ** 2).sum(-1))


# ---------------------------------------------------------------- Eq. (1)
@pytest.mark.parametrize("case", GOLD["temperature"])
def test_temperature_hand_values(case):
    """Eq. (1), evaluated by hand."""
    assert temperature(case["g"], case["K"], case["p_min"]) == pytest.approx(case["T"], abs=1e-12)


@pytest.mark.parametrize("K", [2, 3, 10])
@pytest.mark.parametrize("p", [0.5, 0.8, 0.9])
def test_pmin_identity(K, p):
    """Eq. (1) is constructed so that a line {m, m+g, ..., m+g} (delta = 0) puts
    exactly p_min on its minimum.  Geometry: x at the origin, one gt point at distance 1, the
    rest at distance 1 + g on the axes (exact in fp32)."""
    g = 0.5
    y = [[1.0, 0, 0]]
    dirs = [[0, 1, 0], [0, 0, 1], [-1, 0, 0], [0, -1, 0], [0, 0, -1], [1, 0, 0]]
    for k in range(K - 1):
        d = dirs[k % len(dirs)]
        y.append([(1 + g) * c for c in d] if k % len(dirs) != 5 else [1 + g, 0, 0])
    cfg = OracleConfig(p_min=p, delta=0.0, tau=0.0, l_iter=0)
    P = sparse_forward([[0, 0, 0]], y, cfg)
    s = P.support()
    row = dict(zip(s["j"].tolist(), s["prow"].tolist()))
    assert row[0] == pytest.approx(p, abs=1e-12)
    for j in range(1, K):
        assert row[j] == pytest.approx((1 - p) / (K - 1), abs=1e-12)


# ---------------------------------------------------------------- whole forward closed forms
@pytest.mark.parametrize("case", GOLD["simplex"]["cases"])
@pytest.mark.parametrize("p", [0.5, 0.8, 0.9])
@pytest.mark.parametrize("tau", [0.0, 1e-8])
def test_regular_simplex_closed_form(case, p, tau):
    """X = Y regular simplex, delta = 0, eps_stab = 0: loss = N (1 - p_min) D (golden file)."""
    pts = np.array(case["points"], np.float32)
    N, D = len(pts), case["D"]
    cfg = OracleConfig(p_min=p, tau=tau, delta=0.0, eps_stab=0.0)
    want = N * (1 - p) * D
    assert sparse_forward(pts, pts, cfg).loss == pytest.approx(want, rel=1e-12, abs=1e-12)
    assert dense_forward(pts, pts, cfg) == pytest.approx(want, rel=1e-12, abs=1e-12)


def test_single_pair():
    g = GOLD["single_pair"]
    P = sparse_forward(g["x"], g["y"])
    assert P.loss == pytest.approx(g["loss"], rel=1e-7)
    gx, gy = P.backward()
    np.testing.assert_allclose(gx, g["grad_x"], rtol=1e-7)
    np.testing.assert_allclose(gy, -np.asarray(g["grad_x"]), rtol=1e-7)


def test_threshold_hand_case():
    """P:80, P:90, P:97 hand case: only the argmin survives tau = 0.2, renormalised to 1."""
    g = GOLD["threshold_hand_case"]
    cfg = OracleConfig(p_min=g["p_min"], delta=g["delta"], tau=g["tau"], l_iter=0)
    P = sparse_forward(g["x"], g["y"], cfg)
    s = P.support()
    rowkept = sorted(s["j"][(s["flags"] & 1) > 0].tolist())
    assert rowkept == g["row_kept"]
    assert s["prow"][s["j"] == 0][0] == pytest.approx(1.0, abs=1e-15)
    ln = P.lines(0)
    assert ln["T"][0] == pytest.approx(math.log(8.0), abs=1e-12)


@pytest.mark.parametrize("case", GOLD["gap_clamp"]["cases"])
def test_gap_clamp_hand_case(case):
    """P:140 (section III-D): CUDA-APML clamps the gap, g = max(gap, eps_g) (reading R17),
    hand-derived temperature and row similarities (golden file)."""
    cfg = OracleConfig(p_min=case["p_min"], delta=case["delta"], eps_g=case["eps_g"],
                       tau=case["tau"], l_iter=0)
    P = sparse_forward(case["x"], case["y"], cfg)
    ln = P.lines(0)
    assert ln["clamped"][0] == 1
    assert ln["g"][0] == case["eps_g"]
    assert ln["T"][0] == pytest.approx(case["T"], rel=1e-12)
    s = P.support()
    rowmask = (s["flags"] & 1) > 0
    want = np.asarray(case["row_s"])
    kept = case.get("row_kept", list(range(len(want))))
    assert sorted(s["j"][rowmask].tolist()) == kept
    want_p = want[kept] / want[kept].sum()
    got = dict(zip(s["j"][rowmask].tolist(), s["prow"][rowmask].tolist()))
    for j, p in zip(kept, want_p):
        assert got[j] == pytest.approx(p, rel=1e-12)


def test_gap_clamp_inactive_above_eps_g():
    """The clamp only acts below eps_g: the same line with eps_g = 0.1 < gap = 0.125 keeps
    g = 0.125 and T = 8 ln 18 (Eq. (1)), clamped flag 0."""
    case = GOLD["gap_clamp"]["cases"][0]
    cfg = OracleConfig(p_min=0.9, delta=0.0, eps_g=0.1, tau=0.0, l_iter=0)
    ln = sparse_forward(case["x"], case["y"], cfg).lines(0)
    assert ln["clamped"][0] == 0
    assert ln["T"][0] == pytest.approx(8 * math.log(18.0), rel=1e-12)


def test_k1_lines():
    """Eq. (1) needs K > 1; single-entry lines carry P = 1 (R4).
    N = 1: every column is a K = 1 line, so after Sinkhorn the row spreads evenly: loss =
    mean_j c_1j.  M = 1: loss = sum_i c_i1.  N = M = 1: loss = c."""
    x, y = clouds.pair("uniform", 1, 9, seed=3)
    c = _cost(x, y)
    assert sparse_forward(x, y).loss == pytest.approx(c.mean(), rel=1e-6)
    x, y = clouds.pair("uniform", 7, 1, seed=4)
    c = _cost(x, y)
    assert sparse_forward(x, y).loss == pytest.approx(c.sum(), rel=1e-6)
    x, y = clouds.pair("uniform", 1, 1, seed=5)
    assert sparse_forward(x, y).loss == pytest.approx(_cost(x, y)[0, 0], rel=1e-7)


# ---------------------------------------------------------------- threshold / sparse pipeline
@pytest.mark.parametrize("NM", [(16, 16), (64, 64), (40, 30), (25, 60)])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tau0_sparse_equals_dense(NM, seed):
    """tau = 0 keeps every entry, so the sparse pipeline must equal dense APML
    up to fp64 reassociation, loss and plan entrywise."""
    N, M = NM
    x, y = clouds.pair("uniform", N, M, seed)
    cfg = OracleConfig(tau=0.0)
    P = sparse_forward(x, y, cfg)
    ld, Pd = dense_forward(x, y, cfg, want_plan=True)
    assert P.nnz == N * M
    assert P.loss == pytest.approx(ld, rel=1e-12)
    s = P.support()
    Ps = np.zeros((N, M)); Ps[s["i"], s["j"]] = s["v"]
    np.testing.assert_allclose(Ps, Pd, rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("kind", ["uniform", "shapenet"])
def test_support_properties(kind):
    """Coverage (every line keeps its argmin, s = 1 >= tau), nnz monotone in tau, row
    marginals after the final row step = R/(R + eps_stab) (Eq. (4))."""
    x, y = clouds.pair(kind, 96, 80, 7)
    prev = None
    for tau in [0.0, 1e-12, 1e-8, 1e-4, 1e-2, 0.5, 1.0]:
        P = sparse_forward(x, y, OracleConfig(tau=tau))
        s = P.support()
        assert set(s["i"].tolist()) == set(range(96))
        assert set(s["j"].tolist()) == set(range(80))
        if prev is not None:
            assert P.nnz <= prev
        prev = P.nnz
        rs = np.bincount(s["i"], weights=s["v"], minlength=96)
        np.testing.assert_allclose(rs, 1.0, atol=2e-8)
        assert np.all(s["v"] >= 0)


def test_symmetrization_halves_singletons_near_converged():
    """R8: P0 = (P_row + P_col)/2 with a missing direction counting as 0.  For a
    near-converged pair the tau = 1e-8 plan then stays within ~1e-4 of dense APML; the literal
    "average of the present values" reading is ~1e-3 away."""
    for seed in range(3):
        x, y = clouds.pair("near", 256, 256, seed)
        ls = sparse_forward(x, y).loss
        ld = dense_forward(x, y)
        assert abs(ls - ld) / ld < 1e-4


def test_sinkhorn_marginals_converge_at_tau0():
    """Sinkhorn (Eqs. (3)-(4)) on a full support with N = M drives both marginals to the
    uniform targets; the column defect shrinks with L_iter."""
    x, y = clouds.pair("uniform", 16, 16, 1)
    errs = []
    for L in (10, 100, 1000):
        s = sparse_forward(x, y, OracleConfig(tau=0.0, l_iter=L)).support()
        cs = np.bincount(s["j"], weights=s["v"], minlength=16)
        errs.append(np.abs(cs - 1).max())
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-6


def test_sinkhorn_hand_fixed_point():
    """2x2 identity support (tau keeps only the argmins) is a Sinkhorn fixed point with
    eps_stab = 0 (Eqs. (3)-(4)); loss 0 since the matched points coincide."""
    pts = np.array([[0, 0, 0], [10, 0, 0]], np.float32)
    P = sparse_forward(pts, pts, OracleConfig(tau=0.5, eps_stab=0.0))
    s = P.support()
    assert P.nnz == 2 and np.all(s["i"] == s["j"])
    np.testing.assert_allclose(s["v"], 1.0, rtol=0, atol=0)
    assert P.loss == 0.0


@pytest.mark.parametrize("seed", range(5))
def test_birkhoff_bound_brute_force(seed):
    """tau = 0, N = M = 6, L = 2000: the plan is doubly stochastic to ~1e-8, hence a convex
    combination of permutations (Birkhoff), so <P, C> >= min over the 720 permutations."""
    x, y = clouds.pair("uniform", 6, 6, seed)
    P = sparse_forward(x, y, OracleConfig(tau=0.0, l_iter=2000))
    C = _cost(x, y)
    best = min(sum(C[i, pi[i]] for i in range(6)) for pi in itertools.permutations(range(6)))
    assert P.loss >= best - 1e-7


@pytest.mark.parametrize("seed", range(3))
def test_recovers_brute_force_assignment(seed):
    """Well separated, slightly perturbed copies with p_min = 0.999: the plan's row argmax is
    the brute-force optimal permutation."""
    rng = np.random.default_rng(seed)
    x = (rng.uniform(size=(6, 3)) * 10).astype(np.float32)
    pi = rng.permutation(6)
    y = (x[pi] + rng.normal(scale=0.01, size=(6, 3))).astype(np.float32)
    C = _cost(x, y)
    best = min(itertools.permutations(range(6)), key=lambda q: sum(C[i, q[i]] for i in range(6)))
    s = sparse_forward(x, y, OracleConfig(p_min=0.999)).support()
    Pd = np.zeros((6, 6)); Pd[s["i"], s["j"]] = s["v"]
    assert Pd.argmax(axis=1).tolist() == list(best)


def test_swap_identity():
    """Orientation pin: swapping X and Y swaps the roles of rows and columns, so
    loss(Y, X) = loss_rowfirst(X, Y) exactly; the two orders agree only when L_iter = 0."""
    x, y = clouds.pair("uniform", 30, 22, 2)
    a = sparse_forward(y, x).loss
    b = sparse_forward(x, y, OracleConfig(row_first=1)).loss
    assert a == pytest.approx(b, rel=1e-13)
    assert abs(sparse_forward(x, y).loss - a) / a > 1e-6
    l0 = OracleConfig(l_iter=0)
    assert sparse_forward(x, y, l0).loss == pytest.approx(sparse_forward(y, x, l0).loss, rel=1e-13)


def test_uniform_fallback_mode():
    """P:64 / P:97: with the uniform fallback, a line whose gap is below eps_g is written as
    1/K over all K entries.  Duplicate gt points make every row's c~(2) = 0."""
    x = np.array([[0, 0, 0], [3, 0, 0]], np.float32)
    y = np.array([[1, 0, 0], [1, 0, 0], [5, 5, 5]], np.float32)
    s = sparse_forward(x, y, OracleConfig(stability=1, l_iter=0)).support()
    r0 = {j: p for i, j, p, f in zip(s["i"], s["j"], s["prow"], s["flags"]) if i == 0 and f & 1}
    assert r0 == pytest.approx({0: 1 / 3, 1: 1 / 3, 2: 1 / 3})


# ---------------------------------------------------------------- backward
def _torch_dense_masked(x, y, cfg: OracleConfig, detach_plan: bool):
    """Independent dense formulation (test-only) in torch fp64 with the same frozen choices:
    argmin / second argmin (lowest index), support mask (s >= tau), gap clamp."""
    N, M = x.shape[0], y.shape[0]
    C = torch.sqrt(((x[:, None, :] - y[None, :, :]) ** 2).sum(-1))

    def direction(Cl, K):
        Cn = Cl.detach().numpy()
        order = np.argsort(Cn, axis=1, kind="stable")
        a = torch.as_tensor(order[:, 0]); b = torch.as_tensor(order[:, 1])
        m = Cl.gather(1, a[:, None]); c2 = Cl.gather(1, b[:, None])
        g = c2 - m + cfg.delta
        clamp = (g < cfg.eps_g).detach()
        g = torch.where(clamp, torch.full_like(g, cfg.eps_g), g)
        lam = math.log((K - 1) * cfg.p_min / (1 - cfg.p_min))
        T = lam / g
        s = torch.exp(-T * (Cl - m))
        mask = (s >= cfg.tau).detach().to(s.dtype)
        return mask * s / (mask * s).sum(1, keepdim=True)

    P = 0.5 * (direction(C, M) + direction(C.t(), N).t())
    for _ in range(cfg.l_iter):
        P = P / (P.sum(0, keepdim=True) + cfg.eps_stab)
        P = P / (P.sum(1, keepdim=True) + cfg.eps_stab)
    if detach_plan:
        P = P.detach()
    return (P * C).sum()


@pytest.mark.parametrize("NM", [(12, 10), (20, 20), (7, 15)])
@pytest.mark.parametrize("tau", [0.0, 1e-8, 1e-2])
@pytest.mark.parametrize("p", [0.5, 0.9])
@pytest.mark.parametrize("mode", [0, 1])
def test_backward_vs_torch_autograd(NM, tau, p, mode):
    """The hand-written reverse pass (oracle) equals torch autograd of an independent dense
    masked formulation; eps_dist = 0 so Eq. (5) is the exact norm derivative."""
    N, M = NM
    x, y = clouds.pair("uniform", N, M, seed=N * 31 + M)
    cfg = OracleConfig(p_min=p, tau=tau, eps_dist=0.0, grad_mode=mode)
    P = sparse_forward(x, y, cfg)
    gx, gy = P.backward(1.0)
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    yt = torch.tensor(y, dtype=torch.float64, requires_grad=True)
    lt = _torch_dense_masked(xt, yt, cfg, detach_plan=(mode == 1))
    lt.backward()
    assert P.loss == pytest.approx(lt.item(), rel=1e-12)
    np.testing.assert_allclose(gx, xt.grad.numpy(), rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(gy, yt.grad.numpy(), rtol=1e-8, atol=1e-10)


def _median_gap(x, y, delta):
    """Median over all rows and columns of c~(2) + delta, from the distance matrix (test-only)."""
    C = _cost(x, y)
    gaps = []
    for A in (C, C.T):
        s = np.sort(A, axis=1)
        gaps.append(s[:, 1] - s[:, 0] + delta)
    return float(np.median(np.concatenate(gaps)))


@pytest.mark.parametrize("NM", [(12, 10), (20, 20)])
@pytest.mark.parametrize("mode", [0, 1])
def test_backward_gap_clamp_vs_torch_autograd(NM, mode):
    """P:140 clamp in the reverse pass: with eps_g at the median gap, about half of the lines
    are clamped; a clamped g is a constant, so no gradient flows through it (the torch
    formulation clamps with torch.where and differentiates).  Loss and both gradients must
    agree; the test asserts that clamped and unclamped lines both occur."""
    N, M = NM
    x, y = clouds.pair("uniform", N, M, seed=N * 7 + M)
    eg = _median_gap(x.astype(np.float32), y.astype(np.float32), 1e-6)
    cfg = OracleConfig(eps_g=eg, eps_dist=0.0, tau=1e-8, grad_mode=mode)
    P = sparse_forward(x, y, cfg)
    cl = np.concatenate([P.lines(0)["clamped"], P.lines(1)["clamped"]])
    assert 0 < cl.sum() < len(cl)
    gx, gy = P.backward(1.0)
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    yt = torch.tensor(y, dtype=torch.float64, requires_grad=True)
    lt = _torch_dense_masked(xt, yt, cfg, detach_plan=(mode == 1))
    lt.backward()
    assert P.loss == pytest.approx(lt.item(), rel=1e-12)
    np.testing.assert_allclose(gx, xt.grad.numpy(), rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(gy, yt.grad.numpy(), rtol=1e-8, atol=1e-10)


def test_backward_gap_clamp_finite_differences():
    """Central differences with half of the lines clamped: where g is clamped the loss
    does not depend on the gap, so the FD derivative sees no T-path term for those lines."""
    x, y = clouds.pair("uniform", 9, 8, 5)
    x = x.astype(np.float64); y = y.astype(np.float64)
    eg = _median_gap(x, y, 1e-6)
    cfg = OracleConfig(eps_g=eg, eps_dist=0.0, tau=1e-8)
    P = sparse_forward(x, y, cfg, f64=True)
    cl0 = (P.lines(0)["clamped"].copy(), P.lines(1)["clamped"].copy())
    assert 0 < cl0[0].sum() + cl0[1].sum() < 17
    gx, _ = P.backward()
    key = lambda Q: (Q.nnz, tuple(Q.support()["i"] * 1000 + Q.support()["j"]),
                     tuple(Q.lines(0)["clamped"]), tuple(Q.lines(1)["clamped"]))
    k0 = key(P)
    h = 1e-6
    checked = 0
    for i in range(x.shape[0]):
        for d in range(3):
            xp = x.copy(); xp[i, d] += h
            xm = x.copy(); xm[i, d] -= h
            Pp = sparse_forward(xp, y, cfg, f64=True); Pm = sparse_forward(xm, y, cfg, f64=True)
            if key(Pp) != k0 or key(Pm) != k0:
                continue
            fd = (Pp.loss - Pm.loss) / (2 * h)
            assert fd == pytest.approx(gx[i, d], rel=1e-5, abs=1e-7)
            checked += 1
    assert checked >= 15


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("tau", [1e-8, 0.0])
def test_backward_finite_differences(seed, tau):
    """Central differences of the fp64 oracle loss (h = 1e-6) vs the reverse pass, skipping
    coordinates whose perturbation changes the support (mask is piecewise constant)."""
    x, y = clouds.pair("uniform", 9, 8, seed)
    x = x.astype(np.float64); y = y.astype(np.float64)
    cfg = OracleConfig(tau=tau, eps_dist=0.0)
    P = sparse_forward(x, y, cfg, f64=True)
    gx, _ = P.backward()
    key = lambda Q: (Q.nnz, tuple(Q.support()["i"] * 1000 + Q.support()["j"]))
    k0 = key(P)
    h = 1e-6
    checked = 0
    for i in range(x.shape[0]):
        for d in range(3):
            xp = x.copy(); xp[i, d] += h
            xm = x.copy(); xm[i, d] -= h
            Pp = sparse_forward(xp, y, cfg, f64=True); Pm = sparse_forward(xm, y, cfg, f64=True)
            if key(Pp) != k0 or key(Pm) != k0:
                continue
            fd = (Pp.loss - Pm.loss) / (2 * h)
            assert fd == pytest.approx(gx[i, d], rel=1e-5, abs=1e-7)
            checked += 1
    assert checked >= 20


@pytest.mark.parametrize("mode", [0, 1])
def test_backward_invariants(mode):
    """Translation: sum xbar + sum ybar = 0.  Rotation: sum x x xbar + y x ybar = 0.  Euler
    (delta = 0, eps_dist = 0, no clamp; the loss is 1-homogeneous in the coordinates because
    T scales as 1/g): sum x.xbar + y.ybar = loss."""
    x, y = clouds.pair("shapenet", 50, 40, 11)
    x = x.astype(np.float64); y = y.astype(np.float64)
    cfg = OracleConfig(delta=0.0, eps_dist=0.0, grad_mode=mode)
    P = sparse_forward(x, y, cfg, f64=True)
    gx, gy = P.backward()
    scale = np.abs(gx).max()
    np.testing.assert_allclose(gx.sum(0) + gy.sum(0), 0, atol=1e-10 * scale * 90)
    rot = np.cross(x, gx).sum(0) + np.cross(y, gy).sum(0)
    np.testing.assert_allclose(rot, 0, atol=1e-9 * scale * 90)
    euler = (x * gx).sum() + (y * gy).sum()
    assert euler == pytest.approx(P.loss, rel=1e-9)


def test_gradient_readings_differ():
    """R11: full and plan-detached gradients are different readings."""
    x, y = clouds.pair("uniform", 64, 64, 0)
    gf, _ = sparse_forward(x, y, OracleConfig(grad_mode=0)).backward()
    gd, _ = sparse_forward(x, y, OracleConfig(grad_mode=1)).backward()
    assert np.linalg.norm(gf - gd) / np.linalg.norm(gf) > 0.2


# ---------------------------------------------------------------- single-line entry point
def test_single_line_matches_plan_and_pmin_identity():
    """oracle.line (one row / column of Algorithm 1 on its own, used by the sampled C5 GPU
    check) is the plan's line: same m, c2, g, T, argmin, kept set and P_row / P_col as the
    pinned sparse plan; and on a line of costs {m, m+g, ..., m+g} with delta = 0 it puts
    exactly p_min on the argmin (Eq. (1) + softmax)."""
    from oracle import line
    x, y = clouds.pair("shapenet", 60, 45, 3)
    P = sparse_forward(x, y, OracleConfig())
    rows, cols = P.lines(0), P.lines(1)
    s = P.support()
    for i in (0, 7, 59):
        L = line(x[i], y, OracleConfig())
        for k in ("m", "c2", "g", "T"):
            assert L[k] == rows[k][i]
        assert L["a"] == rows["a"][i] and L["b"] == rows["b"][i]
        sel = (s["i"] == i) & ((s["flags"] & 1) != 0)
        np.testing.assert_array_equal(L["idx"], s["j"][sel])
        np.testing.assert_array_equal(L["p"], s["prow"][sel])
    for j in (0, 44):
        L = line(y[j], x, OracleConfig())
        assert L["T"] == cols["T"][j] and L["a"] == cols["a"][j]
        sel = (s["j"] == j) & ((s["flags"] & 2) != 0)
        np.testing.assert_array_equal(L["idx"], s["i"][sel])
        np.testing.assert_array_equal(L["p"], s["pcol"][sel])
    # p_min identity: other points on the axes at distances 2 (the minimum) and 2.5 (K - 1 ties)
    for K, p in ((5, 0.9), (12, 0.8)):
        pts = np.zeros((K, 3), np.float32)
        pts[0] = (2.0, 0, 0)
        for k in range(1, K):
            pts[k] = (0, 2.5, 0) if k % 2 else (0, 0, -2.5)
        L = line(np.zeros(3, np.float32), pts, OracleConfig(p_min=p, delta=0.0, tau=0.0))
        assert L["a"] == 0 and abs(L["g"] - 0.5) < 1e-15
        assert abs(L["p"][0] - p) < 1e-12
