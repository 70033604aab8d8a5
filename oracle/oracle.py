"""ctypes binding of oracle/liboracle.so (TEST INFRASTRUCTURE ONLY).

Thin marshalling over apml_oracle.c; no arithmetic of the method lives here.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "apml_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build_oracle(force: bool = False) -> str:
    """Compile the C oracle (gcc, fp64, OpenMP over pairs).  Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Cfg(C.Structure):
    _fields_ = [("p_min", C.c_double), ("tau", C.c_double), ("eps_stab", C.c_double),
                ("delta", C.c_double), ("eps_g", C.c_double), ("eps_dist", C.c_double),
                ("l_iter", C.c_int32), ("stability", C.c_int32), ("grad_mode", C.c_int32),
                ("row_first", C.c_int32)]


@dataclass
class OracleConfig:
    """Hyper-parameters; defaults per PAPER.md P:176 (tau, L_iter, eps_stab) and DESIGN.md R2/R3."""
    p_min: float = 0.9
    tau: float = 1e-8
    eps_stab: float = 1e-8
    delta: float = 1e-6
    eps_g: float = 1e-8
    eps_dist: float = 1e-8
    l_iter: int = 10
    stability: int = 0      # 0 gap clamp, 1 uniform fallback
    grad_mode: int = 0      # 0 full, 1 plan-detached
    row_first: int = 0      # 0 column-then-row (Eqs. 3-4); 1 test-only variant

    def _c(self) -> _Cfg:
        return _Cfg(self.p_min, self.tau, self.eps_stab, self.delta, self.eps_g, self.eps_dist,
                    self.l_iter, self.stability, self.grad_mode, self.row_first)


_lib = None


def _L():
    global _lib
    if _lib is None:
        lib = C.CDLL(build_oracle())
        P = C.c_void_p
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        lib.oracle_temperature.restype = C.c_double
        lib.oracle_temperature.argtypes = [C.c_double, C.c_int64, C.c_double]
        lib.oracle_sparse_forward.restype = P
        lib.oracle_sparse_forward.argtypes = [f32p, f32p, C.c_int64, C.c_int64, C.POINTER(_Cfg)]
        lib.oracle_sparse_forward64.restype = P
        lib.oracle_sparse_forward64.argtypes = [f64p, f64p, C.c_int64, C.c_int64, C.POINTER(_Cfg)]
        lib.oracle_dense_forward64.restype = C.c_double
        lib.oracle_dense_forward64.argtypes = [f64p, f64p, C.c_int64, C.c_int64, C.POINTER(_Cfg), P]
        lib.oracle_plan_loss.restype = C.c_double
        lib.oracle_plan_loss.argtypes = [P]
        lib.oracle_plan_nnz.restype = C.c_int64
        lib.oracle_plan_nnz.argtypes = [P]
        lib.oracle_plan_support.restype = None
        lib.oracle_plan_support.argtypes = [P, i64p, i64p, i32p, f64p, f64p, f64p, f64p, f64p]
        lib.oracle_plan_lines.restype = None
        lib.oracle_plan_lines.argtypes = [P, C.c_int32, i64p, f64p]
        lib.oracle_plan_backward.restype = None
        lib.oracle_plan_backward.argtypes = [P, C.c_double, f64p, f64p]
        lib.oracle_plan_free.restype = None
        lib.oracle_plan_free.argtypes = [P]
        lib.oracle_dense_forward.restype = C.c_double
        lib.oracle_dense_forward.argtypes = [f32p, f32p, C.c_int64, C.c_int64, C.POINTER(_Cfg), P]
        lib.oracle_line.restype = C.c_int64
        lib.oracle_line.argtypes = [f32p, f32p, C.c_int64, C.POINTER(_Cfg), i64p, f64p, i64p, f64p]
        lib.oracle_batch.restype = C.c_int
        lib.oracle_batch.argtypes = [f32p, f32p, C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Cfg),
                                     P, f64p, P, P, C.c_int]
        _lib = lib
    return _lib


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def temperature(g: float, K: int, p_min: float) -> float:
    """Eq. (1) as evaluated by the oracle."""
    return _L().oracle_temperature(g, K, p_min)


class SparsePlan:
    """Sparse oracle forward for one pair (Algorithm 1); exposes support, lines, backward."""

    def __init__(self, x, y, cfg: OracleConfig | None = None, f64: bool = False):
        """f64=False: inputs rounded to fp32 (the bytes the GPU sees); f64=True: fp64 inputs
        (finite-difference tests)."""
        self.cfg = cfg or OracleConfig()
        conv = (lambda a: np.ascontiguousarray(np.asarray(a, np.float64))) if f64 else _f32
        self.x = conv(x).reshape(-1, 3)
        self.y = conv(y).reshape(-1, 3)
        self.N, self.M = self.x.shape[0], self.y.shape[0]
        c = self.cfg._c()
        fwd = _L().oracle_sparse_forward64 if f64 else _L().oracle_sparse_forward
        self._h = fwd(self.x, self.y, self.N, self.M, C.byref(c))
        if not self._h:
            raise ValueError("oracle rejected the input")
        self.loss = _L().oracle_plan_loss(self._h)
        self.nnz = _L().oracle_plan_nnz(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L().oracle_plan_free(h)
            self._h = None

    def support(self) -> dict:
        n = max(self.nnz, 1)
        i = np.zeros(n, np.int64); j = np.zeros(n, np.int64); fl = np.zeros(n, np.int32)
        p0, v, c, pr, pc = (np.zeros(n) for _ in range(5))
        _L().oracle_plan_support(self._h, i, j, fl, p0, v, c, pr, pc)
        k = self.nnz
        return dict(i=i[:k], j=j[:k], flags=fl[:k], p0=p0[:k], v=v[:k], c=c[:k], prow=pr[:k], pcol=pc[:k])

    def lines(self, direction: int) -> dict:
        n = self.M if direction else self.N
        ints = np.zeros(6 * n, np.int64); dbl = np.zeros(4 * n)
        _L().oracle_plan_lines(self._h, direction, ints, dbl)
        ints = ints.reshape(n, 6); dbl = dbl.reshape(n, 4)
        return dict(a=ints[:, 0], b=ints[:, 1], clamped=ints[:, 2], uniform=ints[:, 3], k1=ints[:, 4],
                    kept=ints[:, 5], m=dbl[:, 0], c2=dbl[:, 1], g=dbl[:, 2], T=dbl[:, 3])

    def backward(self, gbar: float = 1.0):
        gx = np.zeros(3 * self.N); gy = np.zeros(3 * self.M)
        _L().oracle_plan_backward(self._h, gbar, gx, gy)
        return gx.reshape(self.N, 3), gy.reshape(self.M, 3)


def sparse_forward(x, y, cfg: OracleConfig | None = None, f64: bool = False) -> SparsePlan:
    return SparsePlan(x, y, cfg, f64=f64)


def dense_forward(x, y, cfg: OracleConfig | None = None, want_plan: bool = False, f64: bool = False):
    cfg = cfg or OracleConfig()
    conv = (lambda a: np.ascontiguousarray(np.asarray(a, np.float64))) if f64 else _f32
    x = conv(x).reshape(-1, 3); y = conv(y).reshape(-1, 3)
    N, M = x.shape[0], y.shape[0]
    c = cfg._c()
    fn = _L().oracle_dense_forward64 if f64 else _L().oracle_dense_forward
    if want_plan:
        P = np.zeros((N, M))
        loss = fn(x, y, N, M, C.byref(c), P.ctypes.data_as(C.c_void_p))
        return loss, P
    return fn(x, y, N, M, C.byref(c), None)


def batch(x, y, cfg: OracleConfig | None = None, gbar=None, want_grad: bool = True, nthreads: int = 0):
    """Per-pair losses (and d loss_b / d pred_b) over a batch, OpenMP over pairs.

    Returns (loss[B], grad[B,N,3] or None, nnz[B], threads_used)."""
    cfg = cfg or OracleConfig()
    x = _f32(x); y = _f32(y)
    B, N, M = x.shape[0], x.shape[1], y.shape[1]
    loss = np.zeros(B)
    nnz = np.zeros(B, np.int64)
    grad = np.zeros((B, N, 3)) if want_grad else None
    g = None if gbar is None else np.ascontiguousarray(np.asarray(gbar, np.float64))
    c = cfg._c()
    used = _L().oracle_batch(x.reshape(-1), y.reshape(-1), B, N, M, C.byref(c),
                             None if g is None else g.ctypes.data_as(C.c_void_p), loss,
                             None if grad is None else grad.ctypes.data_as(C.c_void_p),
                             nnz.ctypes.data_as(C.c_void_p), nthreads)
    return loss, grad, nnz, used


def line(own_point, others, cfg: OracleConfig | None = None) -> dict:
    """One line of Algorithm 1 (P:161 / P:162) on its own: point `own_point` [3] against
    `others` [K, 3] -- m, c2, g, T, argmin a, second b, clamped, and the kept (index, P)."""
    cfg = cfg or OracleConfig()
    o = _f32(own_point).reshape(3)
    y = _f32(others).reshape(-1, 3)
    K = y.shape[0]
    ints = np.zeros(6, np.int64); dbl = np.zeros(4)
    idx = np.zeros(K, np.int64); p = np.zeros(K)
    c = cfg._c()
    n = _L().oracle_line(o, y.reshape(-1), K, C.byref(c), ints, dbl, idx, p)
    return dict(a=int(ints[0]), b=int(ints[1]), clamped=int(ints[2]), uniform=int(ints[3]), k1=int(ints[4]),
                kept=int(ints[5]), m=dbl[0], c2=dbl[1], g=dbl[2], T=dbl[3], idx=idx[:n].copy(), p=p[:n].copy())
