"""Row-sharded mode (apml_forward_rowsharded) on one B200: world = 1 through the
same collectives, and world = 2 as two processes sharing cuda:0 over gloo -- the column
statistics all-gather, the column-sum all-reduces and the loss all-reduce all run for real.
Compared with the fp64 oracle on the whole cloud (loss rel 1e-5, gradient normwise 1e-4 on
the well-conditioned set)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import OracleConfig, SparsePlan
from synth import clouds
from tests.parity_util import normwise, well_conditioned, well_conditioned_gt

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_rank(rank, world, port, kind, B, N, M, mode, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_19743_b200 import Config
    from paper_2512_19743_b200.parallel import Collectives, apml_loss_rowsharded, shard_rows
    x, y = clouds.batch(kind, B, N, M, seed=41)
    a, b = shard_rows(N, rank, world)
    pred = torch.tensor(x[:, a:b], device="cuda", requires_grad=True)
    gt = torch.tensor(y, device="cuda", requires_grad=True)
    comm = Collectives(device="cuda")
    loss = apml_loss_rowsharded(pred, gt, a, N, Config(grad_mode=mode), comm, reduction="none")
    loss.sum().backward()
    torch.cuda.synchronize()
    out[rank] = (loss.detach().cpu().numpy().tolist(), a, b, pred.grad.cpu().numpy().tolist(), comm.errors,
                 gt.grad.cpu().numpy().tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(params=["0", "1"], ids=["brute", "culled"])
def cull_env(request, monkeypatch):
    monkeypatch.setenv("APML_CULL", request.param)
    return request.param


@pytest.mark.parametrize("world", [1, 2])
@pytest.mark.parametrize("mode", ["full", "plan_detached"])
@pytest.mark.parametrize("case", [("shapenet", 2, 700, 650), ("uniform", 1, 333, 1000)])
def test_rowsharded_matches_oracle(world, mode, case, cull_env):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    kind, B, N, M = case
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_run_rank, args=(world, _free_port(), kind, B, N, M, mode, out), nprocs=world, join=True)
    x, y = clouds.batch(kind, B, N, M, seed=41)
    oc = OracleConfig(grad_mode=0 if mode == "full" else 1)
    grad = np.zeros((B, N, 3))
    for r in range(world):
        loss, a, b, g, errs, _ = out[r]
        assert not errs
        grad[:, a:b] = np.asarray(g)
    for bb in range(B):
        plan = SparsePlan(x[bb], y[bb], oc)
        for r in range(world):
            assert abs(out[r][0][bb] - plan.loss) <= 1e-5 * plan.loss
        gx, gy = plan.backward()
        mask = well_conditioned(x[bb], y[bb], plan, oc) if mode == "full" else np.ones(N, bool)
        assert normwise(grad[bb][mask], gx[mask]) <= 1e-4
        # grad w.r.t. gt: every rank holds the sum over ranks (apml_backward_ex all-reduce)
        mg = well_conditioned_gt(x[bb], y[bb], plan, oc) if mode == "full" else np.ones(M, bool)
        for r in range(world):
            ggr = np.asarray(out[r][5])[bb]
            assert normwise(ggr[mg], gy[mg]) <= 1e-4
