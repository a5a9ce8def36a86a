"""The C-ABI library loads on a CPU-only box and exports every symbol include/*.h declares
(no device calls here)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("slm.h", "slm_debug.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(slm_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    from paper_1604_06174_b200 import _lib
    names = _declared()
    assert len(names) >= 29
    missing = [n for n in sorted(names) if not hasattr(_lib.lib, n)]
    assert not missing, missing


def test_version_and_errors():
    import ctypes as C
    from paper_1604_06174_b200 import _lib
    assert b"sm_100a" in _lib.lib.slm_version()
    u, d = C.c_int64(), C.c_int64()
    assert _lib.lib.slm_recursion_estimate(0, 1, C.byref(u), C.byref(d)) == -6   # SLM_E_DOMAIN
    assert b"DomainError" in _lib.lib.slm_last_error()


def test_step_without_device_fails_loudly():
    # no CPU fallback: a step on a box without an sm_100a device returns an error
    import torch
    if torch.cuda.is_available():
        return
    import paper_1604_06174_b200 as slm
    import ctypes as C
    g = slm.Graph.chain(2, 64, 128)
    p = slm.Plan(g, "sqrt")
    desc = slm._lib.ChainDesc(1, 2, 64, 128, 0, *([C.c_void_p(256)] * 8))
    h = C.c_void_p()
    assert slm.lib.slm_model_chain(C.byref(desc), C.byref(h)) == 0
    rc = slm.lib.slm_step(p._h, h, C.c_void_p(256), C.c_void_p(256), C.c_void_p(256), 1 << 30,
                          C.c_void_p(256), 1 << 30, C.c_void_p(256), None, None)
    assert rc in (-20, -11)
    slm.lib.slm_model_destroy(h)
