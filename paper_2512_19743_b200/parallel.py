"""Batch sharding over GPUs: pairs are independent units, so each rank runs
the whole hot path on its own contiguous slice of the batch; the only collective is the
all-reduce of the loss (NCCL over NVLink / NVSwitch; any torch.distributed backend works).

No gradient communication is needed for the loss itself: with loss = sum_r loss_r, the
gradient of the global loss w.r.t. rank r's predictions is the gradient of loss_r.
(Model-parameter gradient sync belongs to the caller's DDP.)
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) slice of B pairs for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    base, extra = divmod(B, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def sharded_reduce(local_losses: torch.Tensor, group=None, reduction: str = "sum",
                   global_batch: int | None = None) -> torch.Tensor:
    """Reduce per-pair losses of this rank's shard to the global loss.

    Value: all-reduce(sum of local per-pair losses) (divided by the global batch for
    "mean").  Gradient: that of the LOCAL reduction (straight-through), which is exactly the
    gradient of the global loss w.r.t. this rank's inputs."""
    local = local_losses.sum()
    glob = local.detach().clone()
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(glob, op=dist.ReduceOp.SUM, group=group)
    out = local + (glob - local).detach()
    if reduction == "sum":
        return out
    if reduction == "mean":
        if global_batch is None:
            n = torch.tensor([local_losses.numel()], dtype=torch.float64, device=local_losses.device)
            if dist.is_available() and dist.is_initialized():
                dist.all_reduce(n, group=group)
            global_batch = int(n.item())
        return out / global_batch
    raise ValueError(f"unknown reduction {reduction!r}")


def apml_loss_sharded(pred_local: torch.Tensor, gt_local: torch.Tensor, cfg=None, group=None,
                      reduction: str = "sum", global_batch: int | None = None) -> torch.Tensor:
    """Batch-sharded sparse APML: this rank's pairs through the CUDA path, loss all-reduced."""
    from .apml import apml_loss
    per_pair = apml_loss(pred_local, gt_local, cfg, reduction="none")
    return sharded_reduce(per_pair, group, reduction, global_batch)
