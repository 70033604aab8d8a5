"""Host-side logic of the batch-sharded path (paper_2512_19743_b200/parallel.py) with the
gloo backend, world_size 2, on CPU.  The per-pair losses come from the CPU oracle (this is a
test of the sharding and the reduction, not of the kernels; the kernels' parity is in
tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_19743_b200.parallel import shard, sharded_reduce


@pytest.mark.parametrize("B,world", [(32, 1), (32, 2), (33, 2), (7, 4), (3, 8), (512, 8)])
def test_shard_partitions_the_batch(B, world):
    got = [shard(B, r, world) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == B
    for (a, b), (c, d) in zip(got, got[1:]):
        assert b == c
    sizes = [b - a for a, b in got]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import OracleConfig, batch as oracle_batch
    from synth import clouds
    B = 5
    x, y = clouds.batch("uniform", B, 40, 30, seed=9)
    a, b = shard(B, rank, world)
    loss, grad, _, _ = oracle_batch(x[a:b], y[a:b], OracleConfig(), want_grad=True)
    # stand-in for the per-pair CUDA losses: a differentiable function of a local tensor
    w = torch.ones(b - a, dtype=torch.float64, requires_grad=True)
    per_pair = w * torch.tensor(loss)
    total = sharded_reduce(per_pair, reduction="sum")
    mean = sharded_reduce(per_pair, reduction="mean")
    total.backward()
    out[rank] = (float(total.item()), float(mean.item()), w.grad.numpy().tolist(), loss.tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_reduce_gloo_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from oracle import OracleConfig, batch as oracle_batch
    from synth import clouds
    x, y = clouds.batch("uniform", 5, 40, 30, seed=9)
    full, _, _, _ = oracle_batch(x, y, OracleConfig(), want_grad=False)
    for r in range(world):
        total, mean, g, local = out[r]
        assert total == pytest.approx(full.sum(), rel=1e-12)      # value = global sum
        assert mean == pytest.approx(full.mean(), rel=1e-12)
        np.testing.assert_allclose(g, local)                        # gradient = local term only


# ---------------------------------------------------------------- row-sharding collectives

def _coll_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_19743_b200.parallel import Collectives, shard_rows
    coll = Collectives(device="cpu")
    assert (coll.rank, coll.world) == (rank, world)
    buf = np.arange(6, dtype=np.float32) * (rank + 1)
    st = coll.allreduce(buf.ctypes.data, 6, None, None)
    send = np.array([rank, rank + 0.5, -1.0], np.float32)
    recv = np.zeros(3 * world, np.float32)
    st2 = coll.allgather(send.ctypes.data, recv.ctypes.data, 3, None, None)
    # int32 bit patterns (argmin candidates, -1 = none) must survive the gather bit-exactly
    ints = np.array([-1, 7 + rank, 2 ** 30 - 1], np.int32)
    irecv = np.zeros(3 * world, np.int32)
    st3 = coll.allgather(ints.ctypes.data, irecv.ctypes.data, 3, None, None)
    out[rank] = (st, st2, st3, buf.tolist(), recv.tolist(), irecv.tolist(), shard_rows(10, rank, world))
    dist.barrier()
    dist.destroy_process_group()


def test_row_shard_collectives_gloo_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_coll_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        st, st2, st3, buf, recv, irecv, rows = out[r]
        assert (st, st2, st3) == (0, 0, 0)
        np.testing.assert_array_equal(buf, np.arange(6) * 3.0)            # 1x + 2x
        np.testing.assert_array_equal(recv, [0, 0.5, -1, 1, 1.5, -1])
        np.testing.assert_array_equal(irecv, [-1, 7, 2 ** 30 - 1, -1, 8, 2 ** 30 - 1])
    assert out[0][6] == (0, 5) and out[1][6] == (5, 10)
