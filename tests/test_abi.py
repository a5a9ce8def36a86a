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


def _fake_chain_model(slm, n, B, d):
    import ctypes as C
    desc = slm._lib.ChainDesc(1, n, B, d, 0, *([C.c_void_p(256)] * 8))
    h = C.c_void_p()
    assert slm.lib.slm_model_chain(C.byref(desc), C.byref(h)) == 0
    return h


def test_step_argument_errors_are_synchronous():
    """Shape / size / alignment errors are reported before any device work (include/slm.h
    conventions), so they are checkable on a CPU-only box."""
    import ctypes as C
    import paper_1604_06174_b200 as slm
    V = C.c_void_p
    h = _fake_chain_model(slm, 4, 64, 256)
    try:
        # plan built for other dims -> E_SHAPE
        p_other = slm.Plan(slm.Graph.chain(5, 64, 256), "sqrt")
        assert slm.lib.slm_step(p_other._h, h, V(256), V(256), V(256), 1 << 30, V(256), 1 << 30, V(256), None,
                                None) == -9
        # an LSTM plan on a chain model -> E_SHAPE
        p_lstm = slm.Plan(slm.Graph.lstm(1, 2, 64, 128, 50), "none")
        assert slm.lib.slm_step(p_lstm._h, h, V(256), V(256), V(256), 1 << 30, V(256), 1 << 30, V(256), None,
                                None) == -9
        p = slm.Plan(slm.Graph.chain(4, 64, 256), "sqrt")
        # pool smaller than the plan -> E_BUFFER_TOO_SMALL
        assert slm.lib.slm_step(p._h, h, V(256), V(256), V(256), p.pool_bytes - 1, V(256), 1 << 30, V(256), None,
                                None) == -10
        # workspace smaller than slm_workspace_bytes -> E_BUFFER_TOO_SMALL
        ws = C.c_size_t()
        assert slm.lib.slm_workspace_bytes(p._h, h, C.byref(ws)) == 0 and ws.value > 0
        assert slm.lib.slm_step(p._h, h, V(256), V(256), V(256), 1 << 30, V(256), ws.value - 1, V(256), None,
                                None) == -10
        # misaligned pool -> E_ARG; null buffers -> E_ARG
        assert slm.lib.slm_step(p._h, h, V(256), V(256), V(4096 + 8), 1 << 30, V(256), 1 << 30, V(256), None,
                                None) == -1
        assert slm.lib.slm_step(p._h, h, None, V(256), V(256), 1 << 30, V(256), 1 << 30, V(256), None, None) == -1
        assert b"aligned" in slm.lib.slm_last_error() or b"null" in slm.lib.slm_last_error()
    finally:
        slm.lib.slm_model_destroy(h)


def test_lstm_model_argument_checks():
    import ctypes as C
    import paper_1604_06174_b200 as slm
    V = C.c_void_p

    def make(L, T, B, H, I, Cn, ptr=V(256)):
        desc = slm._lib.LstmDesc(L, T, B, H, I, Cn, *([ptr] * 8))
        h = C.c_void_p()
        rc = slm.lib.slm_model_lstm(C.byref(desc), C.byref(h))
        if rc == 0:
            slm.lib.slm_model_destroy(h)
        return rc

    assert make(2, 8, 64, 128, 50, 300) == 0
    assert make(2, 8, 48, 128, 50, 300) == -1      # batch not in {64, 128, 256}
    assert make(2, 8, 64, 100, 50, 300) == -1      # hidden % 128
    assert make(0, 8, 64, 128, 50, 300) == -1
    assert make(2, 8, 64, 128, 50, 300, ptr=None) == -1
    # the workspace of an LSTM model is sized from its dims and the plan must match them
    desc = slm._lib.LstmDesc(2, 8, 64, 128, 50, 300, *([V(256)] * 8))
    h = C.c_void_p()
    assert slm.lib.slm_model_lstm(C.byref(desc), C.byref(h)) == 0
    try:
        ws = C.c_size_t()
        p = slm.Plan(slm.Graph.lstm(2, 8, 64, 128, 50), "none")
        assert slm.lib.slm_workspace_bytes(p._h, h, C.byref(ws)) == 0 and ws.value > 0
        p_bad = slm.Plan(slm.Graph.lstm(2, 9, 64, 128, 50), "none")
        assert slm.lib.slm_workspace_bytes(p_bad._h, h, C.byref(ws)) == -9
        # the LSTM runs replicas-only: a communicator is refused before any device work
        assert slm.lib.slm_step(p._h, h, V(256), V(256), V(256), 1 << 30, V(256), 1 << 30, V(256), None,
                                V(4096)) == -11
    finally:
        slm.lib.slm_model_destroy(h)


def test_lstm_segment_mirrors_shape():
    import paper_1604_06174_b200 as slm
    g = slm.Graph.lstm(2, 6, 64, 128, 50)
    m = g.lstm_segment_mirrors(3)
    per_t = 2 * 2 + 2
    kept = [v for v in range(len(m)) if m[v] == 0 and v % per_t in (2, 4)]   # S nodes kept
    assert [v // per_t for v in kept] == [2, 2, 5, 5]                        # t = 2 and t = 5
    assert all(m[v] == 0 for v in range(0, len(m) - 1, per_t))               # inputs never mirrored


def test_lstm_pack_unpack_roundtrip():
    """LstmModel.pack_w pads layer 0 to Kin0 = round_up(I, 128) zero columns between W_ih and
    W_hh (the C-ABI layout, reading A21); unpack_w recovers the true-width per-layer arrays."""
    import numpy as np
    import torch

    import paper_1604_06174_b200 as slm
    L, H, I = 3, 8, 5
    rng = np.random.default_rng(0)
    W = [rng.standard_normal((4 * H, (I if l == 0 else H) + H)) for l in range(L)]
    flat = slm.LstmModel.pack_w([torch.tensor(w) for w in W], I)
    k0 = slm.LstmModel.kin0(I)
    assert flat.numel() == 4 * H * (k0 + H) + (L - 1) * 4 * H * 2 * H
    w0 = flat[:4 * H * (k0 + H)].reshape(4 * H, k0 + H).numpy()
    assert np.array_equal(w0[:, :I], W[0][:, :I]) and not w0[:, I:k0].any() and np.array_equal(w0[:, k0:], W[0][:, I:])
    back = slm.LstmModel.unpack_w(flat.numpy(), L, H, I)
    for a, b in zip(back, W):
        assert np.array_equal(a, b)
