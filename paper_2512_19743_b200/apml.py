"""Python binding of libapml.so (include/apml.h) -- argument marshalling only.

Every step of the method runs in the CUDA kernels behind the C ABI; this module passes
device pointers, sizes and the current torch stream, and lets torch's caching allocator
back the library's workspace (so ``torch.cuda.max_memory_allocated`` sees it).

    loss = apml_loss(pred, gt)                 # [B,N,3], [B,M,3] fp32 CUDA -> scalar (sum)
    loss.backward()                            # grad w.r.t. pred
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as A


@dataclass
class Config:
    """Hyper-parameters, defaults per PAPER.md P:176 and DESIGN.md R2/R3."""
    p_min: float = 0.9
    tau: float = 1e-8
    l_iter: int = 10
    eps_stab: float = 1e-8
    delta: float = 1e-6
    eps_g: float = 1e-8
    eps_dist: float = 1e-8
    grad_mode: str = "full"          # "full" | "plan_detached"
    capacity: int = 0                # entries per point per pair; 0 = library default
    sync_check: bool = True          # read back support counts and retry on overflow
    check_finite: bool = False
    stage_timing: bool = False       # CUDA events between stages (apml_ctx_stage_times)
    stability: str = "clamp"         # "clamp" (CUDA-APML) | "uniform" (P:64 / P:97 fallback)
    stage_marks: int = 0             # with stage_timing: bit k records stage mark k only (0 = all)

    def to_c(self) -> A.ApmlConfig:
        if self.grad_mode not in ("full", "plan_detached"):
            raise ValueError(f"grad_mode must be 'full' or 'plan_detached', got {self.grad_mode!r}")
        if self.stability not in ("clamp", "uniform"):
            raise ValueError(f"stability must be 'clamp' or 'uniform', got {self.stability!r}")
        flags = (A.APML_FLAG_UNIFORM_FALLBACK if self.stability == "uniform" else 0) | \
            (A.APML_FLAG_SYNC_CHECK if self.sync_check else 0) | \
            (A.APML_FLAG_CHECK_FINITE if self.check_finite else 0) | \
            (A.APML_FLAG_STAGE_TIMING if self.stage_timing else 0) | ((int(self.stage_marks) & 0x1FF) << 8)
        return A.ApmlConfig(self.p_min, self.tau, self.l_iter, self.eps_stab, self.delta, self.eps_g,
                            self.eps_dist, A.APML_GRAD_FULL if self.grad_mode == "full"
                            else A.APML_GRAD_PLAN_DETACHED, self.capacity, flags)


def _torch_alloc(nbytes, stream, user):
    return torch.cuda.caching_allocator_alloc(int(nbytes), stream=int(stream or 0))


def _torch_free(ptr, nbytes, stream, user):
    torch.cuda.caching_allocator_delete(int(ptr))


_ALLOC = A.ApmlAllocator(A.ALLOC_FN(_torch_alloc), A.FREE_FN(_torch_free), None)


def _check_points(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != torch.float32 or t.dim() != 3 or t.shape[-1] != 3:
        raise ValueError(f"{name} must be float32 [B, n, 3], got {tuple(t.shape)} {t.dtype}")
    return t.contiguous()


class Context:
    """Saved forward state (opaque apml_ctx*) for one backward."""

    def __init__(self, handle: int, B: int, N: int, M: int, device: torch.device):
        self._h = handle
        self.B, self.N, self.M, self.device = B, N, M, device

    def stats(self) -> dict:
        """apml_ctx_stats (synchronises the stream)."""
        nnz = (C.c_int64 * self.B)()
        st = A.ApmlStats()
        A.check(A.lib().apml_ctx_stats(self._h, C.cast(nnz, C.c_void_p), C.byref(st)))
        return dict(nnz=list(nnz), nnz_total=st.nnz_total, emitted_total=st.emitted_total,
                    clamp_count=st.clamp_count, capacity=st.capacity,
                    overflow_pairs=st.overflow_pairs, bytes_ctx=st.bytes_ctx, launches=st.launches,
                    sweep_evals=list(st.sweep_evals), uniform_count=st.uniform_count)

    def stage_times(self) -> dict:
        """Per-stage device milliseconds (needs Config(stage_timing=True)); synchronises."""
        ms = (C.c_float * len(A.STAGES))()
        A.check(A.lib().apml_ctx_stage_times(self._h, C.cast(ms, C.c_void_p), len(A.STAGES)))
        return dict(zip(A.STAGES, list(ms)))

    def support(self, b: int) -> dict:
        """apml_ctx_support for pair b (synchronises): CSR-ordered i, j, flags, P0, v."""
        import numpy as np
        n = C.c_int64(0)
        st = A.lib().apml_ctx_support(self._h, b, C.byref(n), None, None, None, None, None)
        if st not in (A.APML_OK, A.APML_ERR_CAPACITY) or (st != A.APML_OK and n.value == 0):
            A.check(st)
        k = n.value
        i = np.zeros(max(k, 1), np.int32); j = np.zeros_like(i); fl = np.zeros_like(i)
        p0 = np.zeros(max(k, 1), np.float32); v = np.zeros_like(p0)
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)
        A.check(A.lib().apml_ctx_support(self._h, b, C.byref(n), ptr(i), ptr(j), ptr(fl), ptr(p0), ptr(v)))
        return dict(i=i[:k], j=j[:k], flags=fl[:k], p0=p0[:k], v=v[:k])

    def lines(self, b: int, direction: int) -> dict:
        """apml_ctx_lines for pair b (synchronises): m, c2, T, argmin, second."""
        import numpy as np
        n = self.M if direction else self.N
        m = np.zeros(n, np.float32); c2 = np.zeros_like(m); T = np.zeros_like(m)
        a = np.zeros(n, np.int32); s = np.zeros_like(a)
        ptr = lambda x: x.ctypes.data_as(C.c_void_p)
        A.check(A.lib().apml_ctx_lines(self._h, b, direction, ptr(m), ptr(c2), ptr(T), ptr(a), ptr(s)))
        return dict(m=m, c2=c2, T=T, a=a, b=s)

    def backward(self, grad_loss: torch.Tensor, out: torch.Tensor | None = None,
                 want_gt: bool = False, gt_out: torch.Tensor | None = None):
        """d loss / d pred [B,N,3]; with want_gt (or gt_out) also d loss / d gt [B,M,3]
        (apml_backward_ex) and returns (grad_pred, grad_gt)."""
        gl = grad_loss.to(device=self.device, dtype=torch.float32).contiguous().reshape(self.B)
        g = out if out is not None else torch.empty(self.B, self.N, 3, device=self.device)
        s = torch.cuda.current_stream(self.device).cuda_stream
        if not (want_gt or gt_out is not None):
            A.check(A.lib().apml_backward(self._h, gl.data_ptr(), g.data_ptr(), s))
            return g
        gg = gt_out if gt_out is not None else torch.empty(self.B, self.M, 3, device=self.device)
        A.check(A.lib().apml_backward_ex(self._h, gl.data_ptr(), g.data_ptr(), gg.data_ptr(), s))
        return g, gg

    def close(self):
        if self._h:
            A.lib().apml_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def forward(pred: torch.Tensor, gt: torch.Tensor, cfg: Config | None = None,
            keep_ctx: bool = True, loss_out: torch.Tensor | None = None,
            n_sizes=None, m_sizes=None):
    """Per-pair losses [B] (fp32, device) and a Context for backward (or None).

    Ragged batches (apml_forward_ragged): n_sizes / m_sizes (length B, host integers) give the
    real cloud sizes of each pair inside the padded [B, N, 3] / [B, M, 3] tensors."""
    cfg = cfg or Config()
    pred = _check_points(pred, "pred")
    gt = _check_points(gt, "gt")
    if pred.shape[0] != gt.shape[0] or pred.device != gt.device:
        raise ValueError("pred and gt must share batch size and device (BatchShapeMismatch)")
    B, N, M = pred.shape[0], pred.shape[1], gt.shape[1]
    loss = loss_out if loss_out is not None else torch.empty(B, device=pred.device, dtype=torch.float32)
    h = C.c_void_p()
    c = cfg.to_c()
    with torch.cuda.device(pred.device):
        s = torch.cuda.current_stream(pred.device).cuda_stream
        if n_sizes is None and m_sizes is None:
            A.check(A.lib().apml_forward(pred.data_ptr(), gt.data_ptr(), B, N, M, C.byref(c),
                                         C.byref(_ALLOC), s, loss.data_ptr(),
                                         C.byref(h) if keep_ctx else None))
        else:
            nb = (C.c_int64 * B)(*[int(v) for v in n_sizes])
            mb = (C.c_int64 * B)(*[int(v) for v in m_sizes])
            A.check(A.lib().apml_forward_ragged(pred.data_ptr(), gt.data_ptr(), B, N, M,
                                                C.cast(nb, C.c_void_p), C.cast(mb, C.c_void_p), C.byref(c),
                                                C.byref(_ALLOC), s, loss.data_ptr(),
                                                C.byref(h) if keep_ctx else None))
    ctx = Context(h.value, B, N, M, pred.device) if keep_ctx else None
    return loss, ctx


class Plan(Context):
    """A reusable forward/backward plan (apml_plan_create): all device memory allocated once,
    every forward sync-free and allocation-free, so `plan.forward` + `plan.backward` can be
    captured into a torch.cuda.CUDAGraph and replayed (static input / output tensors)."""

    def __init__(self, B: int, N: int, M: int, cfg: Config | None = None, device=None):
        cfg = cfg or Config()
        device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        h = C.c_void_p()
        c = cfg.to_c()
        with torch.cuda.device(device):
            s = torch.cuda.current_stream(device).cuda_stream
            A.check(A.lib().apml_plan_create(B, N, M, C.byref(c), C.byref(_ALLOC), s, C.byref(h)))
        super().__init__(h.value, B, N, M, device)

    def forward(self, pred: torch.Tensor, gt: torch.Tensor, loss_out: torch.Tensor | None = None) -> torch.Tensor:
        pred = _check_points(pred, "pred")
        gt = _check_points(gt, "gt")
        if tuple(pred.shape) != (self.B, self.N, 3) or tuple(gt.shape) != (self.B, self.M, 3):
            raise ValueError("pred / gt shapes differ from the plan's")
        loss = loss_out if loss_out is not None else torch.empty(self.B, device=self.device, dtype=torch.float32)
        s = torch.cuda.current_stream(self.device).cuda_stream
        A.check(A.lib().apml_plan_forward(self._h, pred.data_ptr(), gt.data_ptr(), s, loss.data_ptr()))
        return loss


    def forward_backward(self, pred: torch.Tensor, gt: torch.Tensor, grad_loss: torch.Tensor,
                         loss_out: torch.Tensor | None = None, grad_out: torch.Tensor | None = None):
        """apml_plan_forward_backward: per-pair losses and d(sum_b grad_loss[b] loss_b)/d pred in one
        call (sparse forward + backward fused in one cluster kernel); capturable in a graph."""
        pred = _check_points(pred, "pred")
        gt = _check_points(gt, "gt")
        if tuple(pred.shape) != (self.B, self.N, 3) or tuple(gt.shape) != (self.B, self.M, 3):
            raise ValueError("pred / gt shapes differ from the plan's")
        gl = grad_loss.to(device=self.device, dtype=torch.float32).contiguous().reshape(self.B)
        loss = loss_out if loss_out is not None else torch.empty(self.B, device=self.device, dtype=torch.float32)
        g = grad_out if grad_out is not None else torch.empty(self.B, self.N, 3, device=self.device)
        s = torch.cuda.current_stream(self.device).cuda_stream
        A.check(A.lib().apml_plan_forward_backward(self._h, pred.data_ptr(), gt.data_ptr(), gl.data_ptr(), s,
                                                   loss.data_ptr(), g.data_ptr()))
        return loss, g

    def step_host(self, pred_host: torch.Tensor, gt_host: torch.Tensor, loss_out: torch.Tensor | None = None,
                  grad_out: torch.Tensor | None = None):
        """apml_plan_step_host: host fp32 [B,N,3] / [B,M,3] in, host loss [B] and grad [B,N,3] out
        (sum reduction); copies both ways and a graph replay of forward + backward inside the call."""
        for t, n, k in ((pred_host, "pred", self.N), (gt_host, "gt", self.M)):
            if t.is_cuda or t.dtype != torch.float32 or tuple(t.shape) != (self.B, k, 3) or not t.is_contiguous():
                raise ValueError(f"{n} must be a contiguous float32 host tensor [{self.B}, {k}, 3]")
        loss = loss_out if loss_out is not None else torch.empty(self.B, dtype=torch.float32, pin_memory=True)
        grad = grad_out if grad_out is not None else torch.empty(self.B, self.N, 3, dtype=torch.float32,
                                                                 pin_memory=True)
        s = torch.cuda.current_stream(self.device).cuda_stream
        A.check(A.lib().apml_plan_step_host(self._h, pred_host.data_ptr(), gt_host.data_ptr(), s,
                                            loss.data_ptr(), grad.data_ptr()))
        return loss, grad


class _APMLFunction(torch.autograd.Function):
    @staticmethod
    def forward(fctx, pred, gt, cfg, n_sizes=None, m_sizes=None):
        loss, ctx = forward(pred, gt, cfg, keep_ctx=True, n_sizes=n_sizes, m_sizes=m_sizes)
        fctx.apml = ctx
        return loss

    @staticmethod
    def backward(fctx, grad_loss):
        ctx = fctx.apml
        if fctx.needs_input_grad[1]:  # gt is itself predicted: apml_backward_ex
            g, gg = ctx.backward(grad_loss, want_gt=True)
        else:
            g, gg = ctx.backward(grad_loss), None
        ctx.close()
        return g, gg, None, None, None


def apml_loss(pred: torch.Tensor, gt: torch.Tensor, cfg: Config | None = None,
              reduction: str = "sum", n_sizes=None, m_sizes=None) -> torch.Tensor:
    """Batched sparse APML (Alg. 1) with autograd w.r.t. pred (and gt when it requires
    grad).  n_sizes / m_sizes: per-pair real sizes of a ragged batch (padded tensors)."""
    loss = _APMLFunction.apply(pred, gt, cfg or Config(), n_sizes, m_sizes)
    if reduction == "sum":
        return loss.sum()
    if reduction == "mean":
        return loss.mean()
    if reduction == "none":
        return loss
    raise ValueError(f"unknown reduction {reduction!r}")


def loss_grad_host(pred_host: torch.Tensor, gt_host: torch.Tensor, cfg: Config | None = None,
                   loss_out: torch.Tensor | None = None, grad_out: torch.Tensor | None = None,
                   device: int | None = None, torch_allocator: bool = False):
    """apml_loss_grad_host: host fp32 buffers in, host loss [B] and grad [B,N,3] out (sum
    reduction), host<->device copies included.  Pinned inputs give async copies.  The library's
    device workspace comes from the CUDA stream-ordered pool (no Python callbacks inside the
    call) unless torch_allocator=True."""
    cfg = cfg or Config()
    for t, n in ((pred_host, "pred"), (gt_host, "gt")):
        if t.is_cuda or t.dtype != torch.float32 or t.dim() != 3 or not t.is_contiguous():
            raise ValueError(f"{n} must be a contiguous float32 host tensor [B, n, 3]")
    B, N, M = pred_host.shape[0], pred_host.shape[1], gt_host.shape[1]
    loss = loss_out if loss_out is not None else torch.empty(B, dtype=torch.float32, pin_memory=True)
    grad = grad_out if grad_out is not None else torch.empty(B, N, 3, dtype=torch.float32, pin_memory=True)
    c = cfg.to_c()
    dev = torch.cuda.current_device() if device is None else device
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream().cuda_stream
        A.check(A.lib().apml_loss_grad_host(pred_host.data_ptr(), gt_host.data_ptr(), B, N, M,
                                            C.byref(c), C.byref(_ALLOC) if torch_allocator else None, s,
                                            loss.data_ptr(), grad.data_ptr()))
    return loss, grad
