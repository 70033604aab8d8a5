"""The multi-GPU data plane on the one-GPU box (verdict r1 item 7): NCCL collectives for real on
device buffers at world 1 (tests/helpers/nccl_world1.py), and bench.py's N > 1 code paths
(batch-shard loss all-reduce, row-sharded C5 with its per-iteration column-sum all-reduces)
under torchrun with --force-dist."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_world1_collectives_match_oracle():
    _need_gpu()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "helpers", "nccl_world1.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["backend"] == "nccl" and out["batchshard"] == "ok"
    assert out["rowshard_cull0_calls"] >= 20 and out["rowshard_cull1_calls"] >= 20
    # the NVLS team ran (a multicast object where the driver builds one for a
    # one-device team, else the plain-memory team with the same kernels) and matched bitwise
    assert out["nvls"] == "ok", out["nvls"]
    print("NVLS multicast object:", out["nvls_multicast"], "host collective calls (NVLS, callbacks):",
          out["nvls_calls"])


@pytest.mark.parametrize("config", ["C2", "C5"])
def test_bench_distributed_paths_under_torchrun(config):
    _need_gpu()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--force-dist", "--config", config, "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == 1 and out["value"] > 0 and out["e2e"]["value"] > 0
    assert "NCCL" in out["config"]["parallelism"]
