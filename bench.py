#!/usr/bin/env python
"""Benchmark of the sparse APML hot path (fwd + bwd) -- driver contract in DESIGN.md "Bench".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the whole hot path over one batch: forward (S0-S7) + full-mode
backward (S8) through the C ABI, plus (N > 1) the NCCL all-reduce of the loss.  Batch
sharding is weak scaling: every rank owns its own B pairs (seed offset by rank).  The JSON
line reports pairs/s of the whole job, per-stage device times, the roofline of the dominant
kernel, the oracle on the host cores (cpu_baseline), an end-to-end number through the host
entry point (apml_loss_grad_host, copies included) and the SM clocks seen while timing.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (tau = 1e-8, L_iter = 10 for all)
CONFIGS = {
    "C1": dict(B=1, N=64, M=64, kind="uniform", workload="C1 parity: B=1, N=M=64"),
    "C2": dict(B=32, N=2048, M=2048, kind="shapenet",
               workload="C2 ShapeNet-55-shaped: B=32, N=M=2048 (FoldingNet-style step)"),
    "C3": dict(B=512, N=1024, M=512, kind="mmfi",
               workload="C3 MM-Fi-shaped: B=512, N=1024, M=512 (N != M)"),
    "C3R": dict(B=512, N=1024, M=1024, kind="mmfi", ragged=(256, 1024),
                workload="C3 MM-Fi-shaped ragged: B=512, per-pair N_b, M_b ~ U[256, 1024], N_b != M_b"),
    "C4": dict(B=64, N=16384, M=16384, kind="shapenet",
               workload="C4 PCN-shaped: B=64, N=M=16384 (global batch; split over the ranks at N > 1)"),
    "C5": dict(B=1, N=262144, M=262144, kind="scene",
               workload="C5 scene: B=1, N=M=262144 (single GPU, unsharded)"),
}
METRIC = "point-cloud pairs/sec fwd+bwd"
LANE_OPS_PER_EVAL = 6  # d2 = 3 sub + 1 mul + 2 fma FP32 lane-ops per (i, j) per sweep


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML thread polling
    every ~1 ms (the C2 timed region is only ~10 ms, too short for nvidia-smi's 200 ms
    period), falling back to `nvidia-smi -lms 20`."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, pci_bus_id: str | None = None):
        self.index, self.pci = index, pci_bus_id
        self.rows, self.mode, self.p, self.th = [], None, None, None
        self.stop_flag = False

    def _nvml_loop(self, nv, h):
        names = [("hw_slowdown", nv.nvmlClocksEventReasonHwSlowdown),
                 ("hw_thermal_slowdown", nv.nvmlClocksEventReasonHwThermalSlowdown),
                 ("sw_thermal_slowdown", nv.nvmlClocksEventReasonSwThermalSlowdown),
                 ("sw_power_cap", nv.nvmlClocksEventReasonSwPowerCap)]
        smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while True:
            done = self.stop_flag
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1e3 if (done or not self.rows) else 0.0
                self.rows.append((float(sm), float(smax), pw, [n for n, bit in names if rs & bit]))
            except Exception:
                pass
            if done:
                return
            time.sleep(0.0002)

    def start(self):
        # the timed region can be ~10 ms: let the sampler thread take the GIL every 0.1 ms
        self.switch = sys.getswitchinterval()
        sys.setswitchinterval(1e-4)
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            h = None
            if self.pci:
                try:
                    h = nv.nvmlDeviceGetHandleByPciBusId(self.pci)
                except Exception:
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mode = "nvml"
            self.th = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.th.start()
            return
        except Exception:
            self.mode = None
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
            self.mode = "nvidia-smi"
        except Exception:
            self.p = None

    def stop(self) -> dict:
        sys.setswitchinterval(getattr(self, "switch", 0.005))
        if self.mode == "nvml":
            self.stop_flag = True
            self.th.join()
        elif self.mode == "nvidia-smi" and self.p is not None:
            time.sleep(0.05)
            self.p.terminate()
            self.p.wait()
            self.f.flush()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in open(self.f.name):
                r = [x.strip() for x in line.split(",")]
                if len(r) >= 8:
                    pw = float(r[2]) if r[2] not in ("", "[N/A]") else 0.0
                    self.rows.append((float(r[0]), float(r[1]), pw,
                                      [n for n, v in zip(names, r[4:8]) if v.lower() == "active"]))
            os.unlink(self.f.name)
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock sampler available"]}
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "source": self.mode}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({n for r in self.rows for n in r[3]})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.rows[0][1], "reasons": reasons,
                "samples": len(self.rows), "sm_mhz_min": sm[0], "power_w_max": max(r[2] for r in self.rows),
                "source": self.mode}


def _pci_bus_id(dev) -> str | None:
    try:
        p = __import__("torch").cuda.get_device_properties(dev)
        return f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
    except Exception:
        return None


def _host_cpu() -> dict:
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        avail = len(os.sched_getaffinity(0))
    except Exception:
        avail = os.cpu_count() or 1
    return {"cpu_model": model, "nproc": avail, "cpu_count": os.cpu_count()}


# Largest pair the oracle is timed on directly; bigger pairs (C5) are timed at this size and
# scaled by the O(N M) cost of its line passes (stated in the JSON "sample").
ORACLE_MAX_NM = 16384 * 16384


def _oracle_sample(c):
    N, M = c["N"], c["M"]
    if N * M <= ORACLE_MAX_NM:
        return N, M, 1.0
    return 16384, 16384, ORACLE_MAX_NM / (N * M)


def cpu_baseline(cfg_name: str, seed: int, budget_s: float = 15.0) -> dict:
    """The fp64 oracle as it stands (OpenMP over pairs) on a bounded sample of the workload."""
    from oracle import OracleConfig, batch as oracle_batch
    from synth import clouds
    c = CONFIGS[cfg_name]
    cores = os.cpu_count() or 1
    n = max(1, min(c["B"], cores))
    sN, sM, scale = _oracle_sample(c)
    x, y = clouds.batch(c["kind"], n, sN, sM, seed)
    t0 = time.perf_counter()
    _, _, _, used = oracle_batch(x, y, OracleConfig(), want_grad=True, nthreads=cores)
    dt = time.perf_counter() - t0
    done, reps = n, 1
    while time.perf_counter() - t0 + dt < budget_s and reps < 64:
        oracle_batch(x, y, OracleConfig(), want_grad=True, nthreads=cores)
        done += n
        reps += 1
    el = time.perf_counter() - t0
    note = "" if scale == 1.0 else f" at N=M={sN}, scaled by the O(NM) cost x{scale:.3g}"
    return {"value": done / el * scale, "unit": "pairs/s", "cores": used, "kind": "oracle", **_host_cpu(),
            "sample": f"{reps} x {n} pairs of {cfg_name} ({c['kind']}, N={c['N']}, M={c['M']}){note}, fwd+full bwd, fp64, {el:.1f} s"}


def _ragged_reference(args, c) -> None:
    """--impl reference for a ragged config: the oracle per pair (SparsePlan + backward, one
    core) on the first pairs of the same seeded ragged batch."""
    import numpy as np
    from oracle import OracleConfig, SparsePlan
    from synth import clouds
    lo, hi = c["ragged"]
    rng = np.random.default_rng(args.seed)
    sizes = []
    for _ in range(8):
        nb, mb = int(rng.integers(lo, hi + 1)), int(rng.integers(lo, hi + 1))
        while mb == nb:
            mb = int(rng.integers(lo, hi + 1))
        sizes.append((nb, mb))
    pairs = [clouds.pair(c["kind"], nb, mb, args.seed, b) for b, (nb, mb) in enumerate(sizes)]
    def step():
        for xb, yb in pairs:
            SparsePlan(xb, yb, OracleConfig()).backward()
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    val = len(pairs) * args.steps / el
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "pairs/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": c["workload"], "B": c["B"], "kind": c["kind"],
                                           "step_sample_pairs": len(pairs)},
           "cpu_baseline": {"value": val, "unit": "pairs/s", "cores": 1, "kind": "oracle", **_host_cpu(),
                            "sample": f"{len(pairs)} ragged pairs of {args.config} per step, fwd+full bwd, fp64"},
           "e2e": {"value": val, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_reference(args) -> None:
    """--impl reference: the oracle timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import OracleConfig, batch as oracle_batch
    from synth import clouds
    c = CONFIGS[args.config]
    if "ragged" in c:
        _ragged_reference(args, c)
        return
    cores = os.cpu_count() or 1
    n = max(1, min(c["B"], cores))
    sN, sM, scale = _oracle_sample(c)
    x, y = clouds.batch(c["kind"], n, sN, sM, args.seed)
    for _ in range(args.warmup):
        oracle_batch(x, y, OracleConfig(), want_grad=True, nthreads=cores)
    t0 = time.perf_counter()
    used = 1
    for _ in range(args.steps):
        _, _, _, used = oracle_batch(x, y, OracleConfig(), want_grad=True, nthreads=cores)
    el = time.perf_counter() - t0
    val = n * args.steps / el * scale
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "pairs/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": c["workload"], "B": c["B"], "N": c["N"], "M": c["M"],
                                           "kind": c["kind"], "step_sample_pairs": n},
           "cpu_baseline": {"value": val, "unit": "pairs/s", "cores": used, "kind": "oracle", **_host_cpu(),
                            "sample": f"{n} pairs of {args.config} per step (bounded sample)"
                            + ("" if scale == 1.0 else f" at N=M={sN}, scaled by the O(NM) cost x{scale:.3g}")
                            + ", fwd+full bwd, fp64"},
           "e2e": {"value": val, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--grad-mode", default="full", choices=["full", "plan_detached"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="N > 1 batch sharding: weak = B pairs per rank; strong = the config's B split "
                         "over the ranks (auto: strong for C3/C3R/C4, whose BASELINE configs fix the "
                         "global batch; weak for C2)")
    ap.add_argument("--force-dist", action="store_true",
                    help="initialise NCCL and take the multi-GPU code paths even at world size 1")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager calls instead of a CUDA-graph replay of a reusable plan")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2512_19743_b200 import Config, Plan, forward, loss_grad_host
    from paper_2512_19743_b200.parallel import Collectives, forward_rowsharded, shard_rows, sharded_reduce
    from synth import clouds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    # --force-dist: the N > 1 code paths (NCCL process group, loss all-reduce, row-sharded C5
    # with every collective through NCCL) even at world 1 -- the one-GPU test of the data plane
    dist_on = world > 1 or args.force_dist
    if args.force_dist:
        os.environ["APML_RS_COLLECTIVES"] = "1"
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if dist_on:
        dist.init_process_group("nccl", device_id=dev)
    c = CONFIGS[args.config]
    B, N, M = c["B"], c["N"], c["M"]
    scaling = args.scaling if args.scaling != "auto" else ("strong" if args.config in ("C3", "C3R", "C4") else "weak")
    B_global = B
    if world > 1 and scaling == "strong" and args.config != "C5":
        if B % world:
            raise SystemExit(f"strong scaling needs B={B} divisible by the {world} ranks")
        B = B // world  # this rank's share of the fixed global batch
    # C5 on several GPUs: one cloud, pred rows sharded (X2 all-gather + X3 column-sum
    # all-reduces inside the call); every other config: batch sharding (weak scaling)
    rowshard = args.config == "C5" and dist_on
    if rowshard:
        x, y = clouds.batch(c["kind"], B, N, M, args.seed)
        r0, r1 = shard_rows(N, rank, world)
        x = np.ascontiguousarray(x[:, r0:r1])
        # X3 (the per-iteration column sums) over an NVLS team when the box builds one (in-kernel
        # multimem reduction), else through the NCCL callbacks
        x3 = "nccl all-reduce callbacks"
        try:
            comm = Collectives(device=dev, nvls_bytes=8 * B * M + 256)
            x3 = "in-kernel NVLS " + ("multicast" if comm.nvls_multicast else "team in plain memory (one device)")
        except Exception as e:
            comm = Collectives(device=dev)
            x3 += f" (NVLS unavailable: {str(e)[:80]})"
    else:
        x, y = clouds.batch(c["kind"], B, N, M, args.seed + 1000 * rank) if "ragged" not in c else (None, None)
    ns = ms = None
    if "ragged" in c:  # per-pair sizes (seeded), clouds padded to N, M (apml_forward_ragged)
        lo, hi = c["ragged"]
        rng = np.random.default_rng(args.seed + 1000 * rank)
        ns, ms = [], []
        x = np.zeros((B, N, 3), np.float32)
        y = np.zeros((B, M, 3), np.float32)
        for b in range(B):
            nb, mb = int(rng.integers(lo, hi + 1)), int(rng.integers(lo, hi + 1))
            while mb == nb:
                mb = int(rng.integers(lo, hi + 1))
            xb, yb = clouds.pair(c["kind"], nb, mb, args.seed + 1000 * rank, b)
            x[b, :nb], y[b, :mb] = xb, yb
            ns.append(nb)
            ms.append(mb)
    pred = torch.tensor(x, device=dev)
    gt = torch.tensor(y, device=dev)
    ones = torch.ones(B, device=dev)
    loss_buf = torch.empty(B, device=dev)
    grad_buf = torch.empty(B, pred.shape[1], 3, device=dev)
    cfg = Config(grad_mode=args.grad_mode, sync_check=False, stage_timing=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # Default: a reusable plan (apml_plan_create: all memory allocated once, sync-free and
    # allocation-free steps) whose forward + backward are captured in ONE CUDA graph and
    # replayed per step (the NCCL loss all-reduce of batch sharding stays eager).
    use_graph = not args.no_graph and not rowshard and ns is None
    graph = plan = None
    launches_per_step = 0
    pre = None  # the instrumented pre-pass (graph mode)

    def make_graph(cfg_g):
        p_ = Plan(B, pred.shape[1], M, cfg_g, device=dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        nl = 0
        def one_step():
            p_.forward(pred, gt, loss_buf)
            p_.backward(ones, out=grad_buf)
        with torch.cuda.stream(side):
            for _ in range(2):
                l0 = p_.stats()["launches"]
                one_step()
                nl = p_.stats()["launches"] - l0
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize()
        g_ = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_):
            one_step()
        return p_, g_, nl

    if use_graph:
        # Every stage mark inside a graph is an event-record node that drains the launch
        # pipeline (all nine: ~40 us on a 318 us C2 step; even the two around one kernel: ~10 us,
        # as do eager events between two graphs).  So: (1) an instrumented pre-pass (all marks)
        # gives the stage breakdown and picks the dominant kernel; (2) the TIMED region replays
        # the step with no mark (value, ms_per_step); (3) right after it, a second K-step region
        # replays the step with only the two marks around the dominant kernel, whose live
        # duration the roofline uses (ms_per_step_instrumented reported beside).
        STAGE_MARKS = {"staging": (0, 1), "passA_rows": (1, 3), "line_info": (3, 4), "emit": (4, 5),
                       "sparse_fwd": (5, 6), "sparse_bwd": (7, 8)}
        p_i, g_i, _ = make_graph(cfg)
        pre_st = []
        for k in range(max(5, args.warmup)):
            flush.fill_(k & 0xFF)
            g_i.replay()
            pre_st.append(p_i.stage_times())
        pre_med = {k: float(np.median([st[k] for st in pre_st])) for k in pre_st[0]}
        dom_pre = max(STAGE_MARKS, key=lambda k: pre_med.get(k, 0.0))
        p_i.close()
        del g_i
        pre = {"stages_ms": pre_med, "dominant": dom_pre}
        pre["marks"] = STAGE_MARKS[dom_pre]
        plan, graph, launches_per_step = make_graph(Config(grad_mode=args.grad_mode, sync_check=False))

    class _GraphStep:  # the per-step handle the timing loop reads (stage times, stats)
        def stage_times(self):
            return plan.stage_times()

        def stats(self):
            st = dict(plan.stats())
            st["launches"] = launches_per_step
            return st

        def close(self):
            pass

    def step():
        if use_graph:
            graph.replay()
            if dist_on:
                sharded_reduce(loss_buf)  # X1: NCCL all-reduce of the loss (batch sharding)
            return _GraphStep()
        if rowshard:
            loss, ctx = forward_rowsharded(pred, gt, r0, N, cfg, comm, loss_out=loss_buf)
            ctx.backward(ones, out=grad_buf)
            return ctx
        loss, ctx = forward(pred, gt, cfg, loss_out=loss_buf, n_sizes=ns, m_sizes=ms)
        ctx.backward(ones, out=grad_buf)
        if dist_on:
            sharded_reduce(loss)  # X1: NCCL all-reduce of the loss (batch sharding)
        return ctx

    # warm-up with the timed loop's lifetime pattern (two contexts alive at a time), so the
    # caching allocator already holds every block the timed steps need
    prev = None
    for _ in range(args.warmup):
        ctx = step()
        if prev is not None:
            prev.close()
        prev = ctx
    prev.close()
    torch.cuda.synchronize()
    st0 = None
    if dist_on:
        dist.barrier()
    torch.cuda.reset_peak_memory_stats(dev)
    sampler = ClockSampler(local, _pci_bus_id(dev))
    sampler.start()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stages, launches, prev = [], 0, None
    t_wall = time.perf_counter()
    for k in range(args.steps):
        flush.fill_(k & 0xFF)  # evict L2 between timed steps (not inside the step bracket)
        evs[k][0].record()
        ctx = step()
        evs[k][1].record()
        if use_graph:
            launches += launches_per_step
            continue
        if prev is not None:
            stages.append(prev.stage_times()); launches += prev.stats()["launches"]; prev.close()
        prev = ctx
    if use_graph:
        # (the replays run on the current stream, the plan's own stream is the capture stream:
        # order the counter read after the last replay)
        torch.cuda.synchronize()
        st0 = _GraphStep().stats()
    else:
        stages.append(prev.stage_times()); st0 = prev.stats(); launches += st0["launches"]; prev.close()
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    step_ms = [a.elapsed_time(b) for a, b in evs]
    peak_gb = (torch.cuda.max_memory_allocated(dev) - flush.numel()) / 1e9  # without the L2-flush buffer
    if use_graph:  # (3): the dominant kernel live, K more steps with its two marks only
        a_, b_ = pre["marks"]
        plan_t, graph_t, _ = make_graph(Config(grad_mode=args.grad_mode, sync_check=False, stage_timing=True,
                                               stage_marks=(1 << a_) | (1 << b_)))
        evi = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            evi[k][0].record()
            graph_t.replay()
            evi[k][1].record()
            stages.append(plan_t.stage_times())  # (synchronises on the stage's last mark)
        torch.cuda.synchronize()
        pre["instrumented_ms_per_step"] = float(np.mean([a.elapsed_time(b) for a, b in evi]))
    clocks = sampler.stop()
    tot_ms = float(sum(step_ms))
    if dist_on:
        t = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    pairs_per_step = B if rowshard else B * world  # = B_global under strong scaling
    value = pairs_per_step / (ms_per_step / 1e3)

    # per-stage medians and the roofline of the dominant kernel (graph mode: the dominant
    # kernel live from the timed region, the other stages from the instrumented pre-pass)
    keys = list(stages[0].keys())
    med = {k: float(np.median([s[k] for s in stages])) for k in keys}
    if pre is not None:
        live = med[pre["dominant"]]
        med = dict(pre["stages_ms"])
        med[pre["dominant"]] = live
    fused = use_graph and os.environ.get("APML_FUSED") == "1" and med.get("sparse_fwd", 1.0) < 0.01
    if fused:  # apml_plan_forward_backward: one cluster kernel for the sparse forward + backward
        med["sparse_fwdbwd"] = med.pop("sparse_bwd")
        med.pop("sparse_fwd", None)
    peaks = _peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    alu_peak = sms * 128 * f_max / 1e12  # FP32 lane-ops/s (FMA = 1), DESIGN.md "Roofline"
    dist_stages = ("passA_rows", "passA_cols", "emit")
    # algorithmic (i, j) evaluations per sweep on this rank: B N M for the full sweeps; the
    # spatially culled sweeps (C4, C5) count on the device the (own point, other point) pairs they
    # evaluate (k_cells.cuh: staged points x active lanes; the tile walk: 32 x 32 blocks)
    # (apml_stats.sweep_evals), capped at B N M
    full_evals = B * pred.shape[1] * M if ns is None else int(sum(a * b for a, b in zip(ns, ms)))
    evals_by = {k: min(int(e), full_evals) for k, e in zip(dist_stages, st0["sweep_evals"])}
    culled = any(e < full_evals for e in evals_by.values())
    if med.get("passA_cols", 0.0) == 0.0:  # both Pass A directions in one launch (full sweeps)
        evals_by["passA_rows"] += evals_by["passA_cols"]
        evals_by["passA_cols"] = 0
    nnz = st0["nnz_total"]
    L = cfg.l_iter
    sparse_bytes = {  # algorithmic bytes per launch (SURVEY 8(d) per-entry totals x nnz)
        "sparse_fwd": nnz * (8 + 20 + 48 + 16 * L + 12),   # CSR/CSC + normalise + Sinkhorn + loss
        "sparse_bwd": nnz * (16 * L + 12 + 44 + 12),        # reverse Sinkhorn + P0bar + softmax rev + Eq. 5
    }
    sparse_bytes["sparse_fwdbwd"] = sparse_bytes["sparse_fwd"] + sparse_bytes["sparse_bwd"]
    dom = max(med, key=med.get)
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(args.config, {}).get(dom)
    except Exception:
        pass
    # the method's distance work is 2 sweeps (Pass A, emit) x B N M evaluations x 6
    # lane-ops.  This implementation's Pass A visits every (i, j) once per direction (rows and
    # columns), so its executed evaluations are counted once for the algorithmic figure; the
    # executed figure is reported beside it.  Culled sweeps: evaluations counted on the device.
    alg_by = dict(evals_by)
    alg_by["passA_rows"] = (evals_by["passA_rows"] + evals_by["passA_cols"]) // 2
    alg_by["passA_cols"] = 0
    fp32_meas = None
    try:
        fp32_meas = json.load(open(os.path.join(ROOT, "profiles", "fp32_peak.json")))
    except Exception:
        pass
    meas_note = ("" if not fp32_meas else
                 f"; measured (scripts/micro/fp32_peak.cu): FFMA2 {fp32_meas.get('ffma2_lane_tops', 0):.1f}, "
                 f"FFMA {fp32_meas.get('ffma_lane_tops', 0):.1f} T lane-op/s")
    if dom in dist_stages:
        ach = LANE_OPS_PER_EVAL * alg_by[dom] / (med[dom] / 1e3) / 1e12
        cells = os.environ.get("APML_CULL_MODE", "1") != "0"
        kname = (("k_top2_cells/k_emit_cells" if cells else "k_line_top2_cull/k_emit_cull") if culled
                 else "k_line_top2/k_emit") + f" ({dom})"
        roof = {"bound": "alu", "kernel": kname, "achieved": ach, "peak": alu_peak,
                "unit": "TFLOP/s", "frac": ach / alu_peak, "traffic": traffic, "evals": alg_by[dom],
                "executed_evals": evals_by[dom],
                "note": "FP32 lane-op roofline (FMA counted once): 148 SM x 128 lanes x sm_max clock"
                        + meas_note + "; " + ("evaluations counted by the culled kernels" if culled
                                              else "B N M evaluations per sweep")}
    else:
        byt = sparse_bytes.get(dom, 0)
        ach = byt / (med[dom] / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "frac": ach / peaks.get("hbm_gbs", 6544.7), "traffic": traffic,
                "note": "algorithmic bytes = SURVEY 8(d) per-entry figure x nnz; the per-pair working set "
                        "is shared-memory / L2 resident (see traffic), the stage is bound by dependent "
                        "gathers and 2 L_iter DSMEM exchange rounds (~0.6 us each, "
                        "scripts/micro/xchg_bench.cu), not by HBM bandwidth"}
    dist_ms = sum(med[k] for k in dist_stages)
    alg_evals, exe_evals = sum(alg_by.values()), sum(evals_by.values())
    roof_dist = {"bound": "alu", "achieved": LANE_OPS_PER_EVAL * alg_evals / (dist_ms / 1e3) / 1e12,
                 "peak": alu_peak, "unit": "TFLOP/s", "sweeps": 2, "ms": dist_ms, "evals": alg_evals,
                 "executed_evals": exe_evals,
                 "executed_achieved": LANE_OPS_PER_EVAL * exe_evals / (dist_ms / 1e3) / 1e12,
                 "culled": culled, "dense_equivalent_evals": 2 * full_evals,
                 "definition": "SURVEY 8(d): 6 lane-ops x 2 sweeps x evaluations / t(Pass A + emit)"}
    roof_dist["frac"] = roof_dist["achieved"] / alu_peak
    roof_dist["executed_frac"] = roof_dist["executed_achieved"] / alu_peak
    sm_load = (clocks or {}).get("sm_mhz")
    if sm_load:  # the same fractions against the peak at the clock measured under load
        roof_dist["frac_at_measured_clock"] = roof_dist["frac"] * f_max / (sm_load * 1e6)
        if roof["bound"] == "alu":
            roof["frac_at_measured_clock"] = roof["frac"] * f_max / (sm_load * 1e6)

    # end to end through the C ABI on HOST buffers: pinned host pred / gt in, host loss AND
    # gradient out, every copy inside the timed call.  Plans: apml_plan_step_host (H2D, a graph
    # replay of forward + backward owned by the plan, D2H, sync).  Ragged / row-sharded: the
    # public forward + backward with the same copies around them.
    e2e = None
    if not args.no_e2e:
        ph = torch.tensor(x).pin_memory()
        gh = torch.tensor(y).pin_memory()
        lo = torch.empty(B, pin_memory=True)
        go = torch.empty(B, pred.shape[1], 3, pin_memory=True)
        lred = torch.empty(B, device=dev)
        hplan = None
        if use_graph:
            hplan = Plan(B, pred.shape[1], M, Config(grad_mode=args.grad_mode, sync_check=False), device=dev)

        def e2e_step():
            if hplan is not None:
                hplan.step_host(ph, gh, lo, go)  # synchronises before returning
            else:
                pred.copy_(ph, non_blocking=True)
                gt.copy_(gh, non_blocking=True)
                if rowshard:
                    _, ctx = forward_rowsharded(pred, gt, r0, N, cfg, comm, loss_out=loss_buf)
                else:
                    _, ctx = forward(pred, gt, cfg, loss_out=loss_buf, n_sizes=ns, m_sizes=ms)
                ctx.backward(ones, out=grad_buf)
                lo.copy_(loss_buf, non_blocking=True)
                go.copy_(grad_buf, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
                ctx.close()
            if dist_on and not rowshard:  # X1 on the step's result
                lred.copy_(lo, non_blocking=True)
                sharded_reduce(lred)
                lo.copy_(lred)
        for _ in range(3):
            e2e_step()
        ke = max(5, min(args.steps, 20))
        e2e_list = []
        for _ in range(ke):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            e2e_list.append((time.perf_counter() - t0) * 1e3)
        e2e_ms = float(np.mean(e2e_list))
        if dist_on:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": pairs_per_step / (e2e_ms / 1e3), "unit": "pairs/s", "ms_per_step": e2e_ms,
               "ms_p10": float(np.percentile(e2e_list, 10)), "ms_p50": float(np.median(e2e_list)),
               "ms_p90": float(np.percentile(e2e_list, 90)), "steps": ke,
               "h2d_bytes_per_step": ph.numel() * 4 + gh.numel() * 4,
               "d2h_bytes_per_step": lo.numel() * 4 + go.numel() * 4,
               "api": ("apml_plan_step_host (C ABI, host fp32 in, host loss + grad out; graph replay "
                       "of forward + backward inside the call)" if hplan is not None else
                       "forward + backward (C ABI) with pinned H2D inputs and D2H loss + grad in the bracket"),
               "clock": "host wall clock around the synchronous call (max over ranks)"}
        if hplan is not None:
            hplan.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and ns is None:
        cpu = cpu_baseline(args.config, args.seed)

    if dist_on:
        dist.barrier()
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if (rowshard or (world > 1 and scaling == "strong")) else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": c["workload"], "B": B_global, "N": N, "M": M, "kind": c["kind"], "tau": cfg.tau,
                       **({} if ns is None else {"ragged_mean_N": float(np.mean(ns)), "ragged_mean_M": float(np.mean(ms))}),
                       "l_iter": cfg.l_iter, "p_min": cfg.p_min, "grad_mode": args.grad_mode,
                       "global_batch": pairs_per_step, "pairs_per_rank": B,
                       **({"x3_column_sums": x3} if rowshard else {}),
                       "parallelism": (f"row-shard x{world} (NCCL all-gather + per-iteration column-sum all-reduce)"
                                       if rowshard else f"batch-shard dp{world}" +
                                       (" + NCCL loss all-reduce" if dist_on else "")),
                       "l2": "flushed between timed steps (256 MiB write outside the step bracket)",
                       "cuda_graph": bool(use_graph)},
            "roofline": roof, "roofline_distance_pass": roof_dist,
            "stages_ms": med, "nnz_per_pair": nnz / B, "peak_gb": peak_gb,
            **({} if pre is None else {
                "stages_note": (f"{pre['dominant']} timed live over K steps replayed right after the "
                                "timed region with its two event marks in the graph (ms_per_step_instrumented); "
                                "the other stages from an instrumented pre-pass with all nine marks; the timed "
                                "region itself carries no mark (each drains the launch pipeline)"),
                "ms_per_step_instrumented": pre["instrumented_ms_per_step"]}),
            "dense_lower_bound_gb": 8 * B * N * M / 1e9,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": launches,
            "wall_s_timed": t_wall, "step_ms_min": min(step_ms), "step_ms_max": max(step_ms),
            "step_ms_p10": float(np.percentile(step_ms, 10)), "step_ms_p50": float(np.median(step_ms)),
            "step_ms_p90": float(np.percentile(step_ms, 90)),
        }
        print(json.dumps(out), flush=True)
    if dist_on:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
