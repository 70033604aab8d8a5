"""Multi-GPU modes of the hot path.

1. Batch sharding: pairs are independent units, so each rank runs the whole hot path on its
   own contiguous slice of the batch; the only collective is the all-reduce of the loss
   (NCCL over NVLink / NVSwitch).  With loss = sum_r loss_r, the gradient of the global loss
   w.r.t. rank r's predictions is the gradient of loss_r: no gradient communication.
2. Row sharding (one cloud too large for one GPU): rank r owns a contiguous block of every
   pair's pred rows and the whole gt; the library (apml_forward_rowsharded) calls back into
   the collectives below for the column statistics (all-gather, X2) and every column sum
   (all-reduce, X3).  The callbacks wrap device pointers as zero-copy torch tensors
   (__cuda_array_interface__) and run torch.distributed on the current stream.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
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


# ---------------------------------------------------------------- row sharding

def shard_rows(N: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of a cloud's N pred rows owned by `rank`."""
    return shard(N, rank, world)


class _CudaBuf:
    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _view(ptr: int, n: int, device) -> torch.Tensor:
    """Zero-copy float32 tensor over n elements at ptr (device pointer, or host when device is cpu)."""
    if torch.device(device).type == "cuda":
        return torch.as_tensor(_CudaBuf(ptr, n), device=device)
    arr = np.ctypeslib.as_array((C.c_float * n).from_address(ptr))
    return torch.from_numpy(arr)


class Collectives:
    """The apml_comm callbacks over a torch.distributed group (NCCL for CUDA tensors; with
    gloo the all-gather goes through host memory because gloo gathers CPU tensors only).

    nvls_bytes > 0: also an NVLS team (apml_nvls_create, collective): the per-iteration
    Sinkhorn column sums are then reduced inside the library's kernels over NVSwitch multicast
    memory (no callback per iteration); needs 8 B M + 256 bytes for B pairs of M gt points."""

    def __init__(self, group=None, device="cuda", nvls_bytes: int = 0):
        from . import _lib as A
        self.group = group
        self.device = torch.device(device)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.backend = dist.get_backend(group) if dist.is_initialized() else "none"
        self.errors = []
        self.calls = 0  # collective invocations made on behalf of the library
        self._ar = A.ALLREDUCE_FN(self.allreduce)
        self._ag = A.ALLGATHER_FN(self.allgather)
        self._gb = A.GATHER_BYTES_FN(self.allgather_bytes)
        self.c = A.ApmlComm(self.rank, self.world, self._ar, self._ag, None, self._gb, None)
        self.nvls = None
        if nvls_bytes > 0:
            h = C.c_void_p()
            with torch.cuda.device(self.device):
                A.check(A.lib().apml_nvls_create(C.byref(self.c), int(nvls_bytes), C.byref(h)))
            self.nvls = h.value
            self.c.nvls = h.value
            self.nvls_multicast = bool(A.lib().apml_nvls_is_multicast(h.value))

    def allgather_bytes(self, send, recv, n, user) -> int:
        """Host all-gather of n bytes per rank (the NVLS handle rendezvous)."""
        try:
            mine = C.string_at(send, n)
            if self.world == 1:
                parts = [mine]
            else:
                parts = [None] * self.world
                dist.all_gather_object(parts, mine, group=self.group)
            C.memmove(recv, b"".join(parts), n * self.world)
            return 0
        except Exception as e:
            self.errors.append(repr(e))
            return 1

    def close(self):
        """Release the NVLS team (collective)."""
        if self.nvls:
            from . import _lib as A
            A.lib().apml_nvls_destroy(self.nvls)
            self.nvls = None
            self.c.nvls = None

    def allreduce(self, buf, n, stream, user) -> int:
        self.calls += 1
        try:  # (a world-1 NCCL group still runs the collective: the one-GPU test of the data plane)
            if self.world > 1 or self.backend == "nccl":
                dist.all_reduce(_view(buf, n, self.device), op=dist.ReduceOp.SUM, group=self.group)
            return 0
        except Exception as e:  # reported to the library as a non-zero status
            self.errors.append(repr(e))
            return 1

    def allgather(self, send, recv, n, stream, user) -> int:
        self.calls += 1
        try:
            s = _view(send, n, self.device)
            r = _view(recv, n * self.world, self.device)
            if self.backend == "nccl":
                dist.all_gather_into_tensor(r, s, group=self.group)
            elif self.world == 1:
                r.copy_(s)
            else:
                parts = [torch.empty(n, dtype=torch.float32) for _ in range(self.world)]
                dist.all_gather(parts, s.cpu(), group=self.group)
                r.copy_(torch.cat(parts).to(r.device))
            return 0
        except Exception as e:
            self.errors.append(repr(e))
            return 1


def forward_rowsharded(pred_local: torch.Tensor, gt: torch.Tensor, row_offset: int, n_global: int,
                       cfg=None, comm: "Collectives | None" = None, loss_out: torch.Tensor | None = None):
    """apml_forward_rowsharded: GLOBAL per-pair losses [B] (every rank) and the Context whose
    backward yields the gradient w.r.t. this rank's rows."""
    from .apml import Context, _check_points, _ALLOC, Config
    from . import _lib as A
    cfg = cfg or Config()
    comm = comm or Collectives(device=pred_local.device)
    pred_local = _check_points(pred_local, "pred")
    gt = _check_points(gt, "gt")
    B, N, M = pred_local.shape[0], pred_local.shape[1], gt.shape[1]
    loss = loss_out if loss_out is not None else torch.empty(B, device=pred_local.device, dtype=torch.float32)
    h = C.c_void_p()
    c = cfg.to_c()
    s = torch.cuda.current_stream(pred_local.device).cuda_stream
    A.check(A.lib().apml_forward_rowsharded(pred_local.data_ptr(), gt.data_ptr(), B, N, row_offset,
                                            n_global, M, C.byref(c), C.byref(_ALLOC), C.byref(comm.c),
                                            s, loss.data_ptr(), C.byref(h)))
    ctx = Context(h.value, B, N, M, pred_local.device)
    ctx.comm = comm  # keep the callbacks alive as long as the context
    return loss, ctx


class _RowShardedFunction(torch.autograd.Function):
    @staticmethod
    def forward(fctx, pred_local, gt, row_offset, n_global, cfg, comm):
        loss, fctx.apml = forward_rowsharded(pred_local, gt, row_offset, n_global, cfg, comm)
        return loss

    @staticmethod
    def backward(fctx, grad_loss):
        gg = None
        if fctx.needs_input_grad[1]:  # d global loss / d gt, summed over ranks (every rank)
            g, gg = fctx.apml.backward(grad_loss, want_gt=True)
        else:
            g = fctx.apml.backward(grad_loss)
        fctx.apml.close()
        return g, gg, None, None, None, None


def apml_loss_rowsharded(pred_local: torch.Tensor, gt: torch.Tensor, row_offset: int, n_global: int,
                         cfg=None, comm: Collectives | None = None, reduction: str = "sum") -> torch.Tensor:
    """Sparse APML with every pair's pred rows sharded over the ranks of `comm` (this rank's
    rows [row_offset, row_offset + N_local)); returns the GLOBAL loss on every rank and the
    gradient w.r.t. this rank's rows."""
    comm = comm or Collectives(device=pred_local.device)
    loss = _RowShardedFunction.apply(pred_local, gt, row_offset, n_global, cfg, comm)
    if reduction == "sum":
        return loss.sum()
    if reduction == "mean":
        return loss.mean()
    if reduction == "none":
        return loss
    raise ValueError(f"unknown reduction {reduction!r}")
