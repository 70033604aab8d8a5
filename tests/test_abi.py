"""C-ABI checks that need no GPU: the library loads, exports every symbol include/apml.h
declares, reports the ABI version, fills the documented defaults, and rejects invalid
arguments on the host (before any CUDA call) with the documented status codes."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2512_19743_b200 import _lib as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "apml.h")).read()
    return sorted(set(re.findall(r"APML_API\s+[\w\s\*]+?\b(apml_\w+)\s*\(", src)))


def test_header_declares_the_binding_exports():
    assert _declared() == sorted(A.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", A.LIB_PATH], capture_output=True, text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in _declared():
        assert name in syms, name
    # nothing else leaks out of the shared object (visibility=hidden)
    assert {s for s in syms if s.startswith("apml_")} == set(_declared())


def test_abi_version_and_defaults():
    L = A.lib()
    assert L.apml_abi_version() == 3
    c = A.ApmlConfig()
    L.apml_config_default(C.byref(c))
    assert c.p_min == pytest.approx(0.9) and c.tau == pytest.approx(1e-8)      # R2
    assert c.l_iter == 10 and c.eps_stab == pytest.approx(1e-8)
    assert c.delta == pytest.approx(1e-6) and c.eps_g == pytest.approx(1e-8)   # R3
    assert c.eps_dist == pytest.approx(1e-8) and c.grad_mode == A.APML_GRAD_FULL
    assert c.flags == A.APML_FLAG_SYNC_CHECK


def _fwd(B=1, N=4, M=4, **kw):
    L = A.lib()
    c = A.ApmlConfig()
    L.apml_config_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    fake = C.c_void_p(0x1000)  # never dereferenced: validation fails first
    h = C.c_void_p()
    st = L.apml_forward(fake, fake, B, N, M, C.byref(c), None, None, fake, C.byref(h))
    return st, h.value


@pytest.mark.parametrize("kw,status", [
    (dict(B=0), A.APML_ERR_SHAPE), (dict(N=0), A.APML_ERR_SHAPE), (dict(M=0), A.APML_ERR_SHAPE),
    (dict(N=1 << 30), A.APML_ERR_SHAPE),
    (dict(p_min=0.0), A.APML_ERR_INVALID_ARG), (dict(p_min=1.0), A.APML_ERR_INVALID_ARG),
    (dict(p_min=0.2, N=4), A.APML_ERR_INVALID_ARG),      # p_min <= 1/K: T <= 0 (dense line)
    (dict(tau=-1e-3), A.APML_ERR_INVALID_ARG), (dict(tau=1.5), A.APML_ERR_INVALID_ARG),
    (dict(l_iter=-1), A.APML_ERR_INVALID_ARG), (dict(eps_stab=0.0), A.APML_ERR_INVALID_ARG),
    (dict(eps_g=0.0), A.APML_ERR_INVALID_ARG), (dict(eps_dist=-1.0), A.APML_ERR_INVALID_ARG),
    (dict(delta=-1e-6), A.APML_ERR_INVALID_ARG), (dict(grad_mode=7), A.APML_ERR_INVALID_ARG),
    (dict(capacity=-1), A.APML_ERR_INVALID_ARG),
])
def test_invalid_arguments_rejected_on_host(kw, status):
    st, h = _fwd(**kw)
    assert st == status
    assert h is None
    assert A.lib().apml_last_error()


def test_null_pointers_and_state_errors():
    L = A.lib()
    st = L.apml_forward(None, None, 1, 4, 4, None, None, None, None, None)
    assert st == A.APML_ERR_INVALID_ARG
    assert L.apml_backward(None, None, None, None) == A.APML_ERR_STATE
    assert L.apml_ctx_stats(None, None, None) == A.APML_ERR_STATE
    L.apml_ctx_destroy(None)  # no-op


def test_binding_refuses_cpu_tensors():
    import torch
    from paper_2512_19743_b200 import forward
    with pytest.raises(TypeError):
        forward(torch.zeros(1, 4, 3), torch.zeros(1, 4, 3))


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2512_19743_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(^|\s)(from|import)\s+oracle\b|liboracle|apml_oracle", txt), f


def test_round2_entry_points_validate_on_host():
    """ABI 3 entry points reject bad arguments before touching the device: NVLS teams need
    rank < world and, for world > 1, the host all-gather used for the handle rendezvous; plan
    calls need a plan; the stage-mark mask travels in the config flags."""
    import ctypes as C
    L = A.lib()
    h = C.c_void_p()
    comm = A.ApmlComm(0, 2, A.ALLREDUCE_FN(lambda *a: 0), A.ALLGATHER_FN(lambda *a: 0), None,
                      A.GATHER_BYTES_FN(), None)  # world 2, no allgather_bytes
    assert L.apml_nvls_create(C.byref(comm), 4096, C.byref(h)) == A.APML_ERR_INVALID_ARG
    assert h.value is None
    bad = A.ApmlComm(3, 2, A.ALLREDUCE_FN(lambda *a: 0), A.ALLGATHER_FN(lambda *a: 0), None,
                     A.GATHER_BYTES_FN(), None)  # rank >= world
    assert L.apml_nvls_create(C.byref(bad), 4096, C.byref(h)) == A.APML_ERR_INVALID_ARG
    assert L.apml_nvls_is_multicast(None) == 0
    L.apml_nvls_destroy(None)  # no-op
    assert L.apml_plan_forward_backward(None, None, None, None, None, None, None) == A.APML_ERR_STATE
    assert L.apml_plan_step_host(None, None, None, None, None, None) == A.APML_ERR_STATE
    from paper_2512_19743_b200 import Config
    c = Config(stage_timing=True, stage_marks=(1 << 7) | (1 << 8)).to_c()
    assert (c.flags >> 8) & 0x1FF == (1 << 7) | (1 << 8)
    assert Config(stability="uniform").to_c().flags & A.APML_FLAG_UNIFORM_FALLBACK
    with pytest.raises(ValueError):
        Config(stability="dense").to_c()
