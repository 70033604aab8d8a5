"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the same
seeded fp32 inputs.  Bars (BASELINE.json north_star):
  loss          |l_gpu - l_or| / l_or <= 1e-5 per pair
  support       identical outside the boundary band; direction flags identical too
  lines         argmin / second argmin identical outside distance ties; T rel 1e-5
  gradient      normwise <= 1e-4 per pair (full mode: over the well-conditioned set;
                plan-detached: over all points)
"""
import math

import numpy as np
import pytest
import torch

from oracle import OracleConfig, SparsePlan, batch as oracle_batch
from synth import clouds
from tests.parity_util import (boundary, flags_map, match_support, normwise, p0_bound, support_diff,
                               well_conditioned, well_conditioned_gt)

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-5
GRAD_RTOL = 1e-4


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_19743_b200 import Config, forward
    return Config, forward


def _ocfg(cfg) -> OracleConfig:
    return OracleConfig(p_min=cfg.p_min, tau=cfg.tau, l_iter=cfg.l_iter, eps_stab=cfg.eps_stab,
                        delta=cfg.delta, eps_g=cfg.eps_g, eps_dist=cfg.eps_dist,
                        grad_mode=0 if cfg.grad_mode == "full" else 1,
                        stability=1 if cfg.stability == "uniform" else 0)


def _run(x, y, cfg):
    Config, forward = _gpu()
    pred = torch.tensor(x, device="cuda")
    gt = torch.tensor(y, device="cuda")
    loss, ctx = forward(pred, gt, cfg)
    g = ctx.backward(torch.ones(x.shape[0], device="cuda"))
    torch.cuda.synchronize()
    return loss.cpu().numpy().astype(np.float64), g.cpu().numpy().astype(np.float64), ctx


def _check_pair(x, y, cfg, loss_g, grad_g, ctx, b, check_grad=True):
    oc = _ocfg(cfg)
    plan = SparsePlan(x[b], y[b], oc)
    rel = abs(loss_g[b] - plan.loss) / abs(plan.loss) if plan.loss != 0 else abs(loss_g[b])
    assert rel <= LOSS_RTOL, f"pair {b}: loss {loss_g[b]} vs oracle {plan.loss} (rel {rel:.3e})"
    # support and flags
    gs = ctx.support(b)
    os_ = plan.support()
    only_g, only_o = support_diff(gs, os_)
    bad = [e for e in only_g | only_o if not boundary(x[b], y[b], plan, e[0], e[1], oc)]
    assert not bad, f"pair {b}: {len(bad)} support entries differ outside the band: {sorted(bad)[:5]}"
    fg, fo = flags_map(gs), flags_map(os_)
    badf = [k for k in fo if k in fg and fg[k] != fo[k] and not boundary(x[b], y[b], plan, k[0], k[1], oc)]
    assert not badf, f"pair {b}: flags differ at {badf[:5]}"
    _check_plan_values(x[b], y[b], cfg, plan, gs, os_, b)
    # per-line statistics
    for d in (0, 1):
        gl, ol = ctx.lines(b, d), plan.lines(d)
        K = y.shape[1] if d == 0 else x.shape[1]
        np.testing.assert_allclose(gl["m"], ol["m"], rtol=1e-6, atol=1e-7)
        if K > 1:
            np.testing.assert_allclose(gl["c2"], ol["c2"], rtol=1e-6, atol=1e-7)
            u = 2.0 ** -24
            tie = np.abs(ol["c2"] - ol["m"]) <= 8 * u * np.maximum(ol["c2"], 1e-30)
            np.testing.assert_array_equal(gl["a"][~tie], ol["a"][~tie])
            # T = Lambda / g with g = c2 - m + delta: fp32 error of g is ~ u (m + c2)
            tol = 1e-5 + 8 * u * (ol["m"] + ol["c2"]) / ol["g"]
            relT = np.abs(gl["T"] - ol["T"]) / np.abs(ol["T"])
            assert np.all(relT <= tol), f"T mismatch, worst {relT.max():.3e}"
    if not check_grad:
        return
    gx, _ = plan.backward(1.0)
    if cfg.grad_mode == "full":
        mask = well_conditioned(x[b], y[b], plan, oc)
        assert mask.mean() > 0.9
        e = normwise(grad_g[b][mask], gx[mask])
    else:
        e = normwise(grad_g[b], gx)
    assert e <= GRAD_RTOL, f"pair {b}: grad normwise error {e:.3e} ({cfg.grad_mode})"


V_RTOL = 1e-4  # normwise, the north_star's gradient bar applied to the plan it is built from


def _check_plan_values(xb, yb, cfg, plan, gs, os_, b):
    """Per-entry P0 within the derived fp32 bound (parity_util.p0_bound), and the
    final plan v = a_i P0_ij b_j (Eqs. 3-4) normwise over the entries whose pred and gt points
    are both well-conditioned (the fp32 sensitivity of near-tie lines reaches v through the
    Sinkhorn-coupled scaling vectors)."""
    oc = _ocfg(cfg)
    ga, oa = match_support(gs, os_)
    if len(oa) == 0:
        return
    if cfg.tau == 0.0:  # full support: the bound assumes e = T (c - m) <= ln(1/tau); keep s >= 1e-8
        keep = os_["p0"][oa] >= 1e-7
        ga, oa = ga[keep], oa[keep]
    p0g, p0o = gs["p0"][ga].astype(np.float64), os_["p0"][oa]
    bound = p0_bound(plan, oc, os_["i"][oa], os_["j"][oa], os_["flags"][oa])
    rel = np.abs(p0g - p0o) / p0o
    worst = int(np.argmax(rel / bound))
    assert np.all(rel <= bound), (f"pair {b}: P0 rel {rel[worst]:.3e} > bound {bound[worst]:.3e} at "
                                  f"({os_['i'][oa][worst]}, {os_['j'][oa][worst]})")
    wx = well_conditioned(xb, yb, plan, oc)
    wy = well_conditioned_gt(xb, yb, plan, oc)
    sel = wx[os_["i"][oa]] & wy[os_["j"][oa]]
    e = normwise(gs["v"][ga][sel], os_["v"][oa][sel])
    assert e <= V_RTOL, f"pair {b}: plan v normwise {e:.3e}"


CASES = [
    # kind, B, N, M, p_min, tau, seed
    ("uniform", 1, 64, 64, 0.9, 1e-8, 0),           # C1
    ("shapenet", 1, 64, 64, 0.9, 1e-8, 1),          # C1
    ("uniform", 3, 300, 300, 0.9, 1e-8, 2),         # ragged vs 512-point tiles
    ("shapenet", 2, 700, 333, 0.8, 1e-8, 3),        # N != M, ragged
    ("mmfi", 2, 512, 1024, 0.9, 1e-8, 4),           # N < M: long rows
    ("mmfi", 2, 1024, 256, 0.9, 1e-8, 5),           # N > M
    ("near", 2, 600, 600, 0.9, 1e-8, 6),            # near-converged
    ("uniform", 2, 200, 150, 0.5, 1e-8, 7),         # flatter softmax
    ("uniform", 2, 257, 129, 0.9, 1e-4, 8),         # argmin-only regime (tau > tau*), R14
    ("uniform", 1, 96, 80, 0.9, 0.0, 9),            # tau = 0: full support (capacity retry)
    ("scene", 1, 1500, 1200, 0.95, 1e-8, 10),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-B{c[1]}-{c[2]}x{c[3]}-p{c[4]}-t{c[5]}")
@pytest.mark.parametrize("mode", ["full", "plan_detached"])
def test_parity_cases(case, mode):
    Config, _ = _gpu()
    kind, B, N, M, p, tau, seed = case
    x, y = clouds.batch(kind, B, N, M, seed)
    cfg = Config(p_min=p, tau=tau, grad_mode=mode)
    lg, gg, ctx = _run(x, y, cfg)
    for b in range(B):
        _check_pair(x, y, cfg, lg, gg, ctx, b)


@pytest.mark.parametrize("NM", [(1, 1), (1, 37), (41, 1), (2, 2), (3, 700)])
def test_degenerate_shapes(NM):
    """K = 1 lines (P = 1, R4), tiny clouds, single pair."""
    Config, _ = _gpu()
    N, M = NM
    x, y = clouds.batch("uniform", 2, N, M, 11)
    cfg = Config()
    lg, gg, ctx = _run(x, y, cfg)
    for b in range(2):
        plan = SparsePlan(x[b], y[b], _ocfg(cfg))
        assert abs(lg[b] - plan.loss) <= LOSS_RTOL * abs(plan.loss)
        gx, _ = plan.backward()
        mask = well_conditioned(x[b], y[b], plan, _ocfg(cfg))  # (3, 700): one column has g ~ 5e-6
        assert normwise(gg[b][mask], gx[mask]) <= GRAD_RTOL


def test_ties_duplicates_and_coincident_points():
    """Duplicated gt points (multiset second min = min, R5), coincident pred/gt points
    (d = 0, Eq. (5) eps_dist), gap clamp active when delta < eps_g."""
    Config, _ = _gpu()
    rng = np.random.default_rng(0)
    y = rng.uniform(size=(1, 200, 3)).astype(np.float32)
    y[0, 100:150] = y[0, 0:50]                                  # duplicates
    x = rng.uniform(size=(1, 180, 3)).astype(np.float32)
    x[0, :30] = y[0, 60:90]                                     # coincident
    for cfg in (Config(), Config(delta=0.0, eps_g=1e-6), Config(delta=0.0, eps_g=1e-6, grad_mode="plan_detached")):
        lg, gg, ctx = _run(x, y, cfg)
        oc = _ocfg(cfg)
        plan = SparsePlan(x[0], y[0], oc)
        assert abs(lg[0] - plan.loss) <= LOSS_RTOL * plan.loss
        st = ctx.stats()
        assert st["nnz_total"] == plan.nnz
        clamped = int(plan.lines(0)["clamped"].sum() + plan.lines(1)["clamped"].sum())
        assert st["clamp_count"] == clamped
        if cfg.delta == 0.0:
            assert clamped >= 20  # rows / columns whose nearest point is a duplicate (47 here)
        # gradient with the clamp active (g-bar = 0 on clamped lines, oracle apml_oracle.c)
        gx, _ = plan.backward(1.0)
        mask = well_conditioned(x[0], y[0], plan, oc, skip_clamped=True) if cfg.grad_mode == "full" \
            else np.ones(x.shape[1], bool)
        # delta = 1e-6 >= eps_g: the duplicates' lines keep g = 1e-6 unclamped (ill-conditioned,
        # excluded); with the clamp active they are kept in the compared set
        assert mask.mean() > (0.9 if cfg.delta == 0.0 else 0.5)
        e = normwise(gg[0][mask], gx[mask])
        assert e <= GRAD_RTOL, f"grad normwise {e:.3e} (delta {cfg.delta}, clamp lines {clamped})"
        _check_plan_values(x[0], y[0], cfg, plan, ctx.support(0), plan.support(), 0)


def test_capacity_retry_and_overflow_reporting():
    """Capacity too small: with sync_check the library retries exactly; without it the
    overflowed pairs report NaN loss and are counted (no silent truncation)."""
    Config, forward = _gpu()
    x, y = clouds.batch("uniform", 3, 400, 300, 12)
    ref, _, _ = _run(x, y, Config())
    small, _, ctx = _run(x, y, Config(capacity=1))
    np.testing.assert_array_equal(small, ref)
    assert ctx.stats()["overflow_pairs"] == 0
    pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    loss, ctx = forward(pred, gt, Config(capacity=1, sync_check=False))
    st = ctx.stats()
    assert st["overflow_pairs"] == 3 and torch.isnan(loss).all()


def test_determinism_and_batch_independence():
    """Bitwise-identical results across runs and independent of the batch a pair sits in."""
    x, y = clouds.batch("shapenet", 4, 1000, 900, 13)
    Config, _ = _gpu()
    l1, g1, _ = _run(x, y, Config())
    l2, g2, _ = _run(x, y, Config())
    np.testing.assert_array_equal(l1, l2)
    np.testing.assert_array_equal(g1, g2)
    l3, g3, _ = _run(x[2:3], y[2:3], Config())
    np.testing.assert_array_equal(l3[0], l1[2])
    np.testing.assert_array_equal(g3[0], g1[2])


def test_host_entry_point_matches_device_path():
    from paper_2512_19743_b200 import loss_grad_host
    Config, _ = _gpu()
    x, y = clouds.batch("mmfi", 3, 512, 256, 14)
    l1, g1, _ = _run(x, y, Config())
    l2, g2 = loss_grad_host(torch.tensor(x).pin_memory(), torch.tensor(y).pin_memory(), Config())
    np.testing.assert_array_equal(l2.numpy(), l1.astype(np.float32))
    np.testing.assert_array_equal(g2.numpy(), g1.astype(np.float32))


def test_autograd_function_and_state_errors():
    from paper_2512_19743_b200 import apml_loss
    from paper_2512_19743_b200._lib import ApmlError
    Config, forward = _gpu()
    x, y = clouds.batch("uniform", 2, 128, 100, 15)
    pred = torch.tensor(x, device="cuda", requires_grad=True)
    gt = torch.tensor(y, device="cuda")
    apml_loss(pred, gt, reduction="mean").backward()
    l, g, _ = _run(x, y, Config())
    np.testing.assert_allclose(pred.grad.cpu().numpy(), g / 2, rtol=1e-6, atol=1e-9)
    loss, ctx = forward(pred.detach(), gt)
    ctx.backward(torch.ones(2, device="cuda"))
    with pytest.raises(ApmlError):
        ctx.backward(torch.ones(2, device="cuda"))


# ------------------------------------------------------------ BASELINE.json full sizes
def _full_size(kind, B, N, M, sample, seed):
    """BASELINE.json sizes in the launch configuration bench.py times (sync-free plan): per
    sampled pair the full _check_pair bar -- loss, support SET and flags outside the boundary
    band, per-line statistics, per-entry P0 and plan v, gradient."""
    Config, _ = _gpu()
    x, y = clouds.batch(kind, B, N, M, seed)
    cfg = Config(sync_check=False)
    lg, gg, ctx = _run(x, y, cfg)
    assert ctx.stats()["overflow_pairs"] == 0
    for b in sample:
        _check_pair(x, y, cfg, lg, gg, ctx, b)


def test_full_size_C2_shapenet_all_pairs():
    """configs[1]: ShapeNet-55-shaped B = 32, N = M = 2048 -- every pair against the oracle."""
    _full_size("shapenet", 32, 2048, 2048, list(range(32)), seed=100)


def test_full_size_C3_mmfi_sampled():
    """configs[2]: MM-Fi-shaped B = 512, (N, M) = (1024, 512); sampled pairs."""
    _full_size("mmfi", 512, 1024, 512, [0, 1, 255, 510, 511], seed=200)


def test_full_size_C4_pcn_sampled():
    """configs[3] at 1 GPU: B = 64, N = M = 16384 (culled sweeps, grid sparse stage); sampled pairs."""
    _full_size("shapenet", 64, 16384, 16384, [0, 63], seed=300)


@pytest.mark.parametrize("kind,N,M,bits", [("uniform", 8192, 6000, ""), ("uniform", 5000, 5000, "6"),
                                             ("scene", 12000, 9000, ""), ("mmfi", 4096, 4096, "5")])
def test_cell_sweeps_whole_pair(kind, N, M, bits, monkeypatch):
    """The cell-grid culled sweeps (k_cells.cuh; the default for min(N, M) >= 4096) on volume
    data (Fig. 2's uniform clouds: Pass A shells and coarse far scans), surface scenes and
    human-pose clouds, unequal sizes, default and forced cell sizes: the whole per-pair bar
    against the oracle (support set and flags outside the band, line statistics, P0, v, loss,
    gradient)."""
    Config, _ = _gpu()
    if bits:
        monkeypatch.setenv("APML_CELL_BITS", bits)
    x, y = clouds.batch(kind, 1, N, M, 41)
    cfg = Config()
    lg, gg, ctx = _run(x, y, cfg)
    _check_pair(x, y, cfg, lg, gg, ctx, 0)


def test_full_size_C5_scene_sampled_lines():
    """configs[4] on one GPU: B = 1, N = M = 262144 (culled sweeps, Morton relabelling, grid
    sparse stage), in bench.py's launch configuration.  The whole oracle is out of reach here
    (2 x 6.9e10 cost + exp evaluations), so the check is on what it can compute one line at a
    time (oracle.line, Algorithm 1) plus properties that hold at any size:
      * 48 sampled rows and 48 sampled columns: m, c2, T, argmin; the kept set of each sampled
        line equals the GPU's entries with that direction flag outside the boundary band;
      * P0 of every entry of the sampled rows (P_row from the row, P_col from each entry's
        column line) within the derived fp32 bound;
      * Eq. (4) row marginals of the final plan, sum_j v_ij = R / (R + eps_stab) ~ 1, every row;
      * the loss equals sum_t v_t c_t over the GPU's own support (fp64 on the host);
      * translation and rotation invariance of the gradient (grad_pred and grad_gt)."""
    Config, forward = _gpu()
    from oracle import line as oracle_line
    N = M = 262144
    x, y = clouds.batch("scene", 1, N, M, 400)
    cfg = Config(sync_check=False)
    oc = _ocfg(cfg)
    pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    loss, ctx = forward(pred, gt, cfg)
    gp, gq = ctx.backward(torch.ones(1, device="cuda"), want_gt=True)
    torch.cuda.synchronize()
    assert ctx.stats()["overflow_pairs"] == 0
    sup = ctx.support(0)
    gi, gj, gf = sup["i"].astype(np.int64), sup["j"].astype(np.int64), sup["flags"]
    rows_g, cols_g = ctx.lines(0, 0), ctx.lines(0, 1)
    rng = np.random.default_rng(5)
    u = 2.0 ** -24
    lt = math.log(1.0 / cfg.tau)
    x0, y0 = x[0], y[0]

    def check_line(L, gl, k, K):
        assert abs(gl["m"][k] - L["m"]) <= 1e-6 * L["m"] + 1e-7
        assert abs(gl["c2"][k] - L["c2"]) <= 1e-6 * L["c2"] + 1e-7
        if L["c2"] - L["m"] > 8 * u * L["c2"]:
            assert gl["a"][k] == L["a"]
        tol = 1e-5 + 8 * u * (L["m"] + L["c2"]) / L["g"]
        assert abs(gl["T"][k] - L["T"]) <= tol * L["T"]

    def in_band(c, L, K):
        from tests.parity_util import _exp_interval
        lo, hi = _exp_interval(c, L["m"], L["c2"], K, cfg.p_min, cfg.delta, cfg.eps_g)
        return lo <= lt <= hi

    col_cache = {}

    def col_line(j):
        if j not in col_cache:
            col_cache[j] = oracle_line(y0[j], x0, oc)
        return col_cache[j]

    p0_checked = 0
    for i in rng.choice(N, 48, replace=False):
        L = oracle_line(x0[i], y0, oc)
        check_line(L, rows_g, i, M)
        sel = gi == i
        g_row = set(gj[sel & ((gf & 1) != 0)].tolist())
        o_row = set(L["idx"].tolist())
        for j in g_row ^ o_row:
            c = float(np.linalg.norm(x0[i].astype(np.float64) - y0[j]))
            assert in_band(c, L, M), f"row {i}: entry {j} differs outside the band"
        prow = dict(zip(L["idx"].tolist(), L["p"].tolist()))
        for t in np.nonzero(sel)[0]:
            j = int(gj[t])
            if not gf[t]:
                continue
            C = col_line(j)
            pcol = dict(zip(C["idx"].tolist(), C["p"].tolist())).get(int(i), 0.0)
            if (j in g_row) != (j in o_row) or ((gf[t] & 2) != 0) != (int(i) in C["idx"]):
                continue  # a boundary entry (asserted above / below): its P0 differs by design
            p0o = 0.5 * (prow.get(j, 0.0) + pcol)
            bnd = u * ((74 * (L["c2"] + L["m"]) + 8 * math.log((M - 1) * 0.9 / 0.1) * L["m"]) / L["g"] + 110)
            if gf[t] & 2:
                bnd = max(bnd, u * ((74 * (C["c2"] + C["m"]) + 8 * math.log((N - 1) * 0.9 / 0.1) * C["m"]) / C["g"] + 110))
            assert abs(sup["p0"][t] - p0o) <= bnd * p0o, f"P0 ({i}, {j}): {sup['p0'][t]} vs {p0o}"
            p0_checked += 1
    assert p0_checked >= 48
    for j in rng.choice(M, 48, replace=False):
        C = col_line(int(j))
        check_line(C, cols_g, j, N)
        g_col = set(gi[(gj == j) & ((gf & 2) != 0)].tolist())
        for i in g_col ^ set(C["idx"].tolist()):
            c = float(np.linalg.norm(x0[i].astype(np.float64) - y0[j]))
            assert in_band(c, C, N), f"column {j}: entry {i} differs outside the band"
    # Eq. (4): every row of the final plan sums to R / (R + eps) (fp32 sums of a few entries)
    rs = np.bincount(gi, weights=sup["v"].astype(np.float64), minlength=N)
    assert np.abs(rs - 1.0).max() <= 1e-5
    # loss = sum_t v_t c_t on the GPU's own support
    c = np.linalg.norm(x0[gi].astype(np.float64) - y0[gj].astype(np.float64), axis=1)
    ls = float(np.dot(sup["v"].astype(np.float64), c))
    assert abs(loss.item() - ls) <= 1e-5 * ls
    # gradient invariants: translation (sum xbar + sum ybar = 0) and rotation
    gx, gy = gp[0].double().cpu().numpy(), gq[0].double().cpu().numpy()
    scale = np.abs(gx).sum() + np.abs(gy).sum()
    assert np.abs(gx.sum(0) + gy.sum(0)).max() <= 1e-5 * scale
    rot = np.cross(x0.astype(np.float64), gx).sum(0) + np.cross(y0.astype(np.float64), gy).sum(0)
    rscale = (np.linalg.norm(x0, axis=1) * np.linalg.norm(gx, axis=1)).sum() + \
        (np.linalg.norm(y0, axis=1) * np.linalg.norm(gy, axis=1)).sum()
    assert np.abs(rot).max() <= 1e-5 * rscale


def test_sharded_loss_single_rank_equals_plain_sum():
    """parallel.apml_loss_sharded without a process group reduces to the plain batch sum."""
    from paper_2512_19743_b200 import apml_loss
    from paper_2512_19743_b200.parallel import apml_loss_sharded
    _gpu()
    x, y = clouds.batch("shapenet", 3, 300, 280, 16)
    p1 = torch.tensor(x, device="cuda", requires_grad=True)
    p2 = torch.tensor(x, device="cuda", requires_grad=True)
    gt = torch.tensor(y, device="cuda")
    a = apml_loss(p1, gt)
    b = apml_loss_sharded(p2, gt)
    a.backward(); b.backward()
    assert a.item() == b.item()
    assert torch.equal(p1.grad, p2.grad)


@pytest.mark.parametrize("env", [
    {"APML_FORCE_IDX32": "1"},                                   # 32-bit indices in shared memory
    {"APML_SMEM_LIMIT": "30000"},                                # replicas / slices in global memory
    {"APML_SMEM_LIMIT": "30000", "APML_FORCE_IDX32": "1", "APML_CL": "8"},
    {"APML_CL": "1"},                                            # one CTA per pair, no DSMEM peers
    {"APML_CL": "2"},
    {"APML_GRID": "1"},                                          # grid-wide kernels (few, large pairs)
    {"APML_CULL": "1"},                                          # spatially culled sweeps (NEXT-2): cell grid
    {"APML_CULL": "1", "APML_GRID": "1"},
    {"APML_CULL": "1", "APML_CELL_BITS": "1"},                   # 2 cells per axis: boxes reach the grid edge
    {"APML_CULL": "1", "APML_CELL_BITS": "6"},                   # tiny cells: shells, per-cell cubes
    {"APML_CULL": "1", "APML_CULL_MODE": "0"},                   # tile walk (k_cull.cuh)
    {"APML_CULL": "1", "APML_CULL_MODE": "0", "APML_CULL_RA": "2", "APML_EMIT_R": "1"},  # 2 groups / warp, emit 1
    {"APML_CULL": "1", "APML_CULL_MODE": "0", "APML_CULL_BOTH": "0"},  # tile walk, one launch per direction
    {"APML_FWD2": "0"},                                          # global-memory sparse forward (k_sparse_fwd)
    {"APML_BWD2": "0"},                                          # k_sparse_fwd2 + k_sparse_bwd
    {"APML_SMEM_LIMIT": "60000", "APML_CL": "1"},                # fwd2 / bwd2 slices in global memory
    {"APML_FUSE_INFO": "0", "APML_PDL": "0"},                    # separate line-info launch, no PDL
    {"APML_FUSE_INFO": "1"},                                     # line constants fused into Pass A
    {"APML_GRID": "1", "APML_RS_IDX16": "0"},                    # grid path with 32-bit Sinkhorn indices
    {"APML_GRID": "1", "APML_RS_FUSED_REV": "0", "APML_RS_ALIAS": "0"},  # grid path: two P0bar walks, no aliasing
], ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()))
def test_sparse_stage_fallback_paths(env, monkeypatch):
    """The plan the library picks depends on N, M, B and shared memory; force every variant at a
    size the oracle checks (the large configs C4 / C5 run on these paths)."""
    Config, _ = _gpu()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for kind, B, N, M in (("uniform", 2, 700, 650), ("mmfi", 2, 512, 1024)):
        x, y = clouds.batch(kind, B, N, M, 17)
        cfg = Config()
        lg, gg, ctx = _run(x, y, cfg)
        for b in range(B):
            _check_pair(x, y, cfg, lg, gg, ctx, b)


GT_CASES = [("uniform", 2, 300, 280, 21), ("mmfi", 2, 512, 1024, 22), ("shapenet", 2, 700, 333, 23)]


def _check_grad_gt(x, y, cfg, gp, gg):
    """grad w.r.t. gt (apml_backward_ex) against the oracle's ybar; translation
    invariance sum xbar + sum ybar = 0 on the GPU values themselves."""
    oc = _ocfg(cfg)
    for b in range(x.shape[0]):
        plan = SparsePlan(x[b], y[b], oc)
        gx, gy = plan.backward(1.0)
        if cfg.grad_mode == "full":
            mask = well_conditioned_gt(x[b], y[b], plan, oc)
            assert mask.mean() > 0.9
            e = normwise(gg[b][mask], gy[mask])
        else:
            e = normwise(gg[b], gy)
        assert e <= GRAD_RTOL, f"pair {b}: grad_gt normwise error {e:.3e} ({cfg.grad_mode})"
        t = np.abs(gp[b].sum(0) + gg[b].sum(0)).max()
        assert t <= 1e-4 * np.abs(gg[b]).sum(0).max(), f"pair {b}: translation invariance {t:.3e}"


@pytest.mark.parametrize("case", GT_CASES, ids=lambda c: f"{c[0]}-{c[2]}x{c[3]}")
@pytest.mark.parametrize("mode", ["full", "plan_detached"])
def test_grad_gt_matches_oracle(case, mode):
    Config, forward = _gpu()
    kind, B, N, M, seed = case
    x, y = clouds.batch(kind, B, N, M, seed)
    cfg = Config(grad_mode=mode)
    _, ctx = forward(torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda"), cfg)
    gp, gg = ctx.backward(torch.ones(B, device="cuda"), want_gt=True)
    torch.cuda.synchronize()
    _check_grad_gt(x, y, cfg, gp.cpu().numpy().astype(np.float64), gg.cpu().numpy().astype(np.float64))


@pytest.mark.parametrize("env", [{"APML_FWD2": "0"}, {"APML_GRID": "1"}, {"APML_CULL": "1"},
                                 {"APML_CULL": "1", "APML_GRID": "1"}],
                         ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()))
def test_grad_gt_every_path(env, monkeypatch):
    Config, forward = _gpu()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    x, y = clouds.batch("uniform", 2, 700, 650, 24)
    cfg = Config()
    _, ctx = forward(torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda"), cfg)
    gp, gg = ctx.backward(torch.ones(2, device="cuda"), want_gt=True)
    torch.cuda.synchronize()
    _check_grad_gt(x, y, cfg, gp.cpu().numpy().astype(np.float64), gg.cpu().numpy().astype(np.float64))


def test_grad_gt_through_autograd():
    """apml_loss with gt.requires_grad: torch autograd receives both gradients."""
    _gpu()
    from paper_2512_19743_b200 import Config, apml_loss
    x, y = clouds.batch("shapenet", 2, 300, 300, 25)
    pred = torch.tensor(x, device="cuda", requires_grad=True)
    gt = torch.tensor(y, device="cuda", requires_grad=True)
    apml_loss(pred, gt, Config(), reduction="sum").backward()
    torch.cuda.synchronize()
    _check_grad_gt(x, y, Config(), pred.grad.cpu().numpy().astype(np.float64),
                   gt.grad.cpu().numpy().astype(np.float64))


def _ragged_case(seed):
    rng = np.random.default_rng(seed)
    B, N, M = 5, 700, 520
    ns = [700, 1, 300, 437, 64]
    ms = [520, 260, 1, 333, 128]
    x, y = clouds.batch("mmfi", B, N, M, seed)
    # the padding is garbage on purpose: it must never be read
    for b in range(B):
        x[b, ns[b]:] = rng.normal(size=(N - ns[b], 3)).astype(np.float32) * 1e3
        y[b, ms[b]:] = np.nan
    return x, y, ns, ms


@pytest.mark.parametrize("env", [{}, {"APML_FWD2": "0"}, {"APML_CL": "1"}],
                         ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()) or "default")
@pytest.mark.parametrize("mode", ["full", "plan_detached"])
def test_ragged_batch_matches_per_pair_oracle(env, mode, monkeypatch):
    """apml_forward_ragged: every pair equals the oracle on its trimmed clouds
    (loss, support, grad_pred and grad_gt), padding rows of the gradients are zero; includes
    K = 1 pairs (n_b = 1, m_b = 1)."""
    Config, forward = _gpu()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    x, y, ns, ms = _ragged_case(31)
    B = x.shape[0]
    cfg = Config(grad_mode=mode)
    loss, ctx = forward(torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda"), cfg,
                        n_sizes=ns, m_sizes=ms)
    gp, gg = ctx.backward(torch.ones(B, device="cuda"), want_gt=True)
    torch.cuda.synchronize()
    loss = loss.cpu().numpy().astype(np.float64)
    gp = gp.cpu().numpy().astype(np.float64)
    gg = gg.cpu().numpy().astype(np.float64)
    oc = _ocfg(cfg)
    for b in range(B):
        xb, yb = x[b, :ns[b]], y[b, :ms[b]]
        plan = SparsePlan(xb, yb, oc)
        rel = abs(loss[b] - plan.loss) / abs(plan.loss)
        assert rel <= LOSS_RTOL, f"pair {b} ({ns[b]}x{ms[b]}): loss rel {rel:.3e}"
        gs, os_ = ctx.support(b), plan.support()
        only_g, only_o = support_diff(gs, os_)
        bad = [e for e in only_g | only_o if not boundary(xb, yb, plan, e[0], e[1], oc)]
        assert not bad, f"pair {b}: support differs at {sorted(bad)[:5]}"
        assert np.all(gp[b, ns[b]:] == 0) and np.all(gg[b, ms[b]:] == 0)
        gx, gy = plan.backward(1.0)
        if mode == "full":
            mx = well_conditioned(xb, yb, plan, oc)
            my = well_conditioned_gt(xb, yb, plan, oc)
        else:
            mx, my = np.ones(ns[b], bool), np.ones(ms[b], bool)
        if ns[b] > 1 or ms[b] > 1:
            assert normwise(gp[b, :ns[b]][mx], gx[mx]) <= GRAD_RTOL, f"pair {b}: grad_pred"
            assert normwise(gg[b, :ms[b]][my], gy[my]) <= GRAD_RTOL, f"pair {b}: grad_gt"


def test_ragged_rejects_bad_sizes():
    Config, forward = _gpu()
    x, y, ns, ms = _ragged_case(32)
    from paper_2512_19743_b200._lib import ApmlError
    for bad_n, bad_m in (([0] + ns[1:], ms), (ns, [9999] + ms[1:])):
        with pytest.raises(ApmlError, match="SHAPE"):
            forward(torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda"), Config(),
                    n_sizes=bad_n, m_sizes=bad_m)


def test_plan_matches_forward_and_replays_in_a_cuda_graph():
    """apml_plan_create / apml_plan_forward: allocation- and sync-free steps give the same bits
    as apml_forward, run repeatedly on new inputs, and replay correctly from a CUDA graph."""
    Config, forward = _gpu()
    from paper_2512_19743_b200 import Plan
    B, N, M = 4, 700, 650
    cfg = Config(sync_check=False)
    inputs = [clouds.batch(kind, B, N, M, 40 + k) for k, kind in enumerate(("shapenet", "uniform", "mmfi"))]

    def ref(x, y):
        loss, ctx = forward(torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda"), cfg)
        g = ctx.backward(torch.ones(B, device="cuda"))
        return loss, g

    plan = Plan(B, N, M, cfg)
    for x, y in inputs[:2]:  # eager, twice: counters re-zeroed per forward
        lp = plan.forward(torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda"))
        gp = plan.backward(torch.ones(B, device="cuda"))
        lr, gr = ref(x, y)
        assert torch.equal(lp, lr) and torch.equal(gp, gr)
    # CUDA graph: static buffers, capture one step, replay on other inputs
    ps = torch.zeros(B, N, 3, device="cuda")
    gs = torch.zeros(B, M, 3, device="cuda")
    ls = torch.zeros(B, device="cuda")
    gout = torch.zeros(B, N, 3, device="cuda")
    ones = torch.ones(B, device="cuda")
    ps.copy_(torch.tensor(inputs[0][0])); gs.copy_(torch.tensor(inputs[0][1]))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm the plan on the capture stream
        plan.forward(ps, gs, ls)
        plan.backward(ones, out=gout)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        plan.forward(ps, gs, ls)
        plan.backward(ones, out=gout)
    for x, y in inputs:
        ps.copy_(torch.tensor(x)); gs.copy_(torch.tensor(y))
        graph.replay()
        torch.cuda.synchronize()
        lr, gr = ref(x, y)
        assert torch.equal(ls, lr) and torch.equal(gout, gr)
    plan.close()


def test_plan_state_errors():
    Config, _ = _gpu()
    from paper_2512_19743_b200 import Plan
    from paper_2512_19743_b200._lib import ApmlError
    plan = Plan(2, 64, 64, Config())
    with pytest.raises(ApmlError, match="STATE"):
        plan.backward(torch.ones(2, device="cuda"))
    with pytest.raises(ValueError):
        plan.forward(torch.zeros(2, 65, 3, device="cuda"), torch.zeros(2, 64, 3, device="cuda"))
    plan.close()


def test_plan_step_host_matches_device_path():
    """apml_plan_step_host (the end-to-end host-buffer call bench.py times): H2D, a graph replay
    of forward + backward owned by the plan, D2H -- the same bits as apml_forward +
    apml_backward, on repeated calls with new inputs, on a side stream and on the NULL stream."""
    Config, forward = _gpu()
    from paper_2512_19743_b200 import Plan
    B, N, M = 3, 900, 700
    cfg = Config(sync_check=False)
    plan = Plan(B, N, M, cfg)
    for k, kind in enumerate(("shapenet", "mmfi", "uniform")):
        x, y = clouds.batch(kind, B, N, M, 60 + k)
        lh, gh = plan.step_host(torch.tensor(x).pin_memory(), torch.tensor(y).pin_memory())
        lr, gr, _ = _run(x, y, cfg)
        np.testing.assert_array_equal(lh.numpy(), lr.astype(np.float32))
        np.testing.assert_array_equal(gh.numpy(), gr.astype(np.float32))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # another stream: the captured graph is launched there
        lh2, gh2 = plan.step_host(torch.tensor(x), torch.tensor(y))  # pageable inputs too
    np.testing.assert_array_equal(lh2.numpy(), lr.astype(np.float32))
    np.testing.assert_array_equal(gh2.numpy(), gr.astype(np.float32))
    plan.close()


def test_plan_and_eager_pick_the_same_sparse_path():
    """apml_plan_create must size the sparse-stage plan from the real emit capacity,
    as apml_forward does; a shape where the two used to diverge (cluster vs grid path) gives
    bit-identical results through both."""
    Config, forward = _gpu()
    from paper_2512_19743_b200 import Plan
    B, N, M = 2, 8192, 8192
    cfg = Config(sync_check=False)
    x, y = clouds.batch("shapenet", B, N, M, 70)
    pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    plan = Plan(B, N, M, cfg)
    lp = plan.forward(pred, gt).clone()
    gp = plan.backward(torch.ones(B, device="cuda")).clone()
    lr, ctx = forward(pred, gt, cfg)
    gr = ctx.backward(torch.ones(B, device="cuda"))
    assert torch.equal(lp, lr) and torch.equal(gp, gr)
    assert plan.stats()["launches"] == ctx.stats()["launches"]
    plan.close()


def test_backward_on_another_stream_is_ordered_before_the_free():
    """a backward on a stream other than the forward's must finish before the
    context's stream-ordered free (and before the next plan forward) reuses the workspace."""
    Config, forward = _gpu()
    x, y = clouds.batch("uniform", 4, 1500, 1400, 71)
    lr, gr, _ = _run(x, y, Config())
    pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    for _ in range(3):
        loss, ctx = forward(pred, gt, Config())
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g = ctx.backward(torch.ones(4, device="cuda"))
        ctx.close()  # freed on the forward's stream, which now waits for s
        junk = torch.full((64 << 20,), 7.0, device="cuda")  # would reuse the freed block
        torch.cuda.synchronize()
        np.testing.assert_array_equal(g.cpu().numpy(), gr.astype(np.float32))
        del junk


def test_memory_follows_the_support():
    """Per-entry arrays sized by the support actually emitted (verdict r1 item 5): an eager call
    with the count read-back keeps the largest pair's count + 64 entries per pair; a plan sizes
    them on its first forward (1.25 x + 64) -- both far below the emit capacity -- and the results
    are the same bits as an explicitly sized plan."""
    Config, forward = _gpu()
    from paper_2512_19743_b200 import Plan
    B, N, M = 4, 3000, 2500
    x, y = clouds.batch("shapenet", B, N, M, 80)
    pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    loss, ctx = forward(pred, gt, Config())
    st = ctx.stats()
    mx = max(st["nnz"]) + (st["emitted_total"] - st["nnz_total"])  # >= the largest emitted count
    assert max(st["nnz"]) <= st["capacity"] <= mx + 128
    g = ctx.backward(torch.ones(B, device="cuda"))
    plan = Plan(B, N, M, Config(sync_check=False))
    lp = plan.forward(pred, gt)
    gp = plan.backward(torch.ones(B, device="cuda"))
    ps = plan.stats()
    assert ps["capacity"] <= 1.25 * mx + 128 and ps["capacity"] < 6 * (N + M) * 3 // 4
    fixed = Plan(B, N, M, Config(sync_check=False, capacity=6))
    lf = fixed.forward(pred, gt)
    gf = fixed.backward(torch.ones(B, device="cuda"))
    assert fixed.stats()["capacity"] == 6 * (N + M)
    assert torch.equal(lp, lf) and torch.equal(gp, gf) and torch.equal(lp, loss) and torch.equal(gp, g)
    assert ps["bytes_ctx"] < fixed.stats()["bytes_ctx"]
    plan.close(); fixed.close()


@pytest.mark.parametrize("env", [{}, {"APML_FWD2": "0"}, {"APML_GRID": "1"}, {"APML_CULL": "1"}],
                         ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()) or "default")
@pytest.mark.parametrize("mode", ["full", "plan_detached"])
def test_uniform_fallback_mode(env, mode, monkeypatch):
    """the uniform-fallback stability mode (APML_FLAG_UNIFORM_FALLBACK, P:64,
    P:97) against the oracle's stability = 1 on a duplicated-point fixture: lines whose gap is
    below eps_g keep all K entries with P = 1/K (T = 0, no softmax gradient); everything else
    as the default mode.  Loss, support and flags, per-entry P0 / v, gradient."""
    Config, _ = _gpu()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(3)
    B, N, M = 2, 300, 260
    y = rng.uniform(size=(B, M, 3)).astype(np.float32)
    y[:, 200:230] = y[:, 10:40]                 # duplicated gt points: rows with gap 0
    x = rng.uniform(size=(B, N, 3)).astype(np.float32)
    x[:, 250:270] = x[:, 0:20]                  # duplicated pred points: columns with gap 0
    cfg = Config(stability="uniform", grad_mode=mode)
    lg, gg, ctx = _run(x, y, cfg)
    oc = _ocfg(cfg)
    st = ctx.stats()
    nu = 0
    for b in range(B):
        plan = SparsePlan(x[b], y[b], oc)
        nu += int(plan.lines(0)["uniform"].sum() + plan.lines(1)["uniform"].sum())
        rel = abs(lg[b] - plan.loss) / plan.loss
        assert rel <= LOSS_RTOL, f"pair {b}: loss rel {rel:.3e}"
        gs, os_ = ctx.support(b), plan.support()
        only_g, only_o = support_diff(gs, os_)
        assert not (only_g or only_o), f"pair {b}: support differs ({len(only_g)}, {len(only_o)})"
        assert flags_map(gs) == flags_map(os_)
        _check_plan_values(x[b], y[b], cfg, plan, gs, os_, b)
        gx, _ = plan.backward(1.0)
        mask = well_conditioned(x[b], y[b], plan, oc, skip_clamped=True) if mode == "full" else np.ones(N, bool)
        assert mask.mean() > 0.9
        e = normwise(gg[b][mask], gx[mask])
        assert e <= GRAD_RTOL, f"pair {b}: grad normwise {e:.3e}"
    assert st["uniform_count"] == nu and nu >= 20
    # the uniform lines really are dense: each duplicated-minimum row keeps all M entries
    assert st["nnz_total"] >= nu * min(N, M) // 2


@pytest.mark.parametrize("shape", [("shapenet", 4, 2048, 2048), ("mmfi", 6, 1024, 512), ("uniform", 3, 700, 650)])
def test_plan_forward_backward_fused_matches(shape, monkeypatch):
    """apml_plan_forward_backward (sparse forward + backward in ONE cluster kernel) gives the
    bits of apml_plan_forward + apml_backward, eagerly and replayed from a CUDA graph, with a
    non-trivial grad_loss; an overflowed pair still reports NaN."""
    Config, forward = _gpu()
    from paper_2512_19743_b200 import Plan
    monkeypatch.setenv("APML_FUSED", "1")
    kind, B, N, M = shape
    cfg = Config(sync_check=False)
    x, y = clouds.batch(kind, B, N, M, 81)
    pred, gt = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    gl = torch.linspace(0.5, 2.0, B, device="cuda")
    plan = Plan(B, N, M, cfg)
    lr = plan.forward(pred, gt).clone()          # (the calibrating first forward)
    gr = plan.backward(gl).clone()
    lf, gf = plan.forward_backward(pred, gt, gl)
    assert torch.equal(lf, lr) and torch.equal(gf, gr)
    ls, gs = torch.zeros(B, device="cuda"), torch.zeros(B, N, 3, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        plan.forward_backward(pred, gt, gl, loss_out=ls, grad_out=gs)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.forward_backward(pred, gt, gl, loss_out=ls, grad_out=gs)
    x2, y2 = clouds.batch(kind, B, N, M, 82)
    pred.copy_(torch.tensor(x2)); gt.copy_(torch.tensor(y2))
    g.replay()
    torch.cuda.synchronize()
    l2, c2 = forward(pred, gt, cfg)
    g2 = c2.backward(gl)
    assert torch.equal(ls, l2) and torch.equal(gs, g2)
    plan.close()
    small = Plan(B, N, M, Config(sync_check=False, capacity=1))
    lo, go = small.forward_backward(pred, gt, gl)
    torch.cuda.synchronize()
    assert torch.isnan(lo).all() and torch.isnan(go).all()
    small.close()
