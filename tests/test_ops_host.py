"""Host-side checks of the op-granularity model (slm_model_ops): what it accepts
and rejects.  No GPU: model creation only records device pointers."""
import ctypes as C

import pytest

import paper_1604_06174_b200 as slm
from paper_1604_06174_b200 import _lib


def _desc(n, B, fc=(), bn=()):
    arrs = {k: (C.c_void_p * n)() for k in ("W", "b", "gamma", "beta", "dW", "db", "dgamma", "dbeta")}
    for v in fc:
        for k in ("W", "b", "dW", "db"):
            arrs[k][v] = 0x1000 + v
    for v in bn:
        for k in ("gamma", "beta", "dgamma", "dbeta"):
            arrs[k][v] = 0x2000 + v
    vpp = C.POINTER(C.c_void_p)
    d = _lib.OpsDesc(B, 0, n, *(C.cast(arrs[k], vpp) for k in ("W", "b", "gamma", "beta", "dW", "db", "dgamma", "dbeta")))
    return d, arrs


def _create(nodes, B, fc, bn):
    g = slm.Graph.from_nodes(nodes, [len(nodes) - 1])
    d, keep = _desc(len(nodes), B, fc, bn)
    h = C.c_void_p()
    rc = slm.lib.slm_model_ops(g._h, C.byref(d), C.byref(h))
    if rc == 0:
        slm.lib.slm_model_destroy(h)
    return rc


def test_preact_graph_accepted():
    B = 64
    nodes = slm.OpsModel.preact_nodes([2, 1], [128, 256], B)
    fc = [v for v, n in enumerate(nodes) if n[0] == slm.OP["fc"]]
    bn = [v for v, n in enumerate(nodes) if n[0] == slm.OP["bn"]]
    assert _create(nodes, B, fc, bn) == 0


def test_rejections():
    B = 64
    nodes = slm.OpsModel.preact_nodes([1], [128], B)
    fc = [v for v, n in enumerate(nodes) if n[0] == slm.OP["fc"]]
    bn = [v for v, n in enumerate(nodes) if n[0] == slm.OP["bn"]]
    assert _create(nodes, B, fc[:0], bn) != 0            # FC without parameters
    assert _create(nodes, B, fc, bn[:0]) != 0            # BN without parameters
    assert _create(nodes, 96, fc, bn) != 0               # batch not a multiple of 64
    bad = slm.OpsModel.preact_nodes([1], [192], B)       # width not a multiple of 128
    assert _create(bad, B, fc, bn) != 0
    sig = [(0, [], B * 128 * 4, 0), (slm.OP["sigmoid"], [0], B * 128 * 4, 0), (slm.OP["softmax_ce"], [1], 4, 1)]
    assert _create(sig, B, [], []) != 0                  # unsupported op


def _create_shaped(nodes, shapes, B):
    """Conv graphs: every Conv / FC node gets W, b; BN gamma, beta; per-node shapes."""
    g = slm.Graph.from_nodes(nodes, [len(nodes) - 1])
    wn = [v for v, n in enumerate(nodes) if n[0] in (slm.OP["fc"], slm.OP["conv"])]
    bn = [v for v, n in enumerate(nodes) if n[0] == slm.OP["bn"]]
    d, keep = _desc(len(nodes), B, wn, bn)
    flat = [int(x) for sh in shapes for x in sh]
    sh = (C.c_int32 * len(flat))(*flat)
    d.shape = C.cast(sh, C.POINTER(C.c_int32))
    h = C.c_void_p()
    rc = slm.lib.slm_model_ops(g._h, C.byref(d), C.byref(h))
    if rc == 0:
        slm.lib.slm_model_destroy(h)
    return rc


def test_conv_resnet_accepted_and_rejections():
    B = 64
    nodes, shapes = slm.OpsModel.preact_conv_nodes(B, 8, [(128, 1), (256, 1)], 128)
    assert _create_shaped(nodes, shapes, B) == 0
    conv = [v for v, n in enumerate(nodes) if n[0] == slm.OP["conv"]]
    # without shapes a Conv node is rejected
    g = slm.Graph.from_nodes(nodes, [len(nodes) - 1])
    d, keep = _desc(len(nodes), B, conv, [])
    h = C.c_void_p()
    assert slm.lib.slm_model_ops(g._h, C.byref(d), C.byref(h)) != 0

    def mutate(v, sh):
        s2 = list(shapes)
        s2[v] = sh
        return _create_shaped(nodes, s2, B)

    H, W, Cc, k, s = shapes[conv[0]]
    assert mutate(conv[0], (H, W, Cc, 5, s)) != 0          # kernel 5 unsupported
    assert mutate(conv[0], (H, W, Cc, k, 3)) != 0          # stride 3 unsupported
    proj = [v for v in conv if shapes[v][3] == 1][0]
    Hp, Wp, Cp, kp, sp = shapes[proj]
    assert mutate(proj, (Hp + 1, Wp + 1, Cp, kp, sp)) != 0  # output size inconsistent with the stride
    pool = [v for v, n in enumerate(nodes) if n[0] == slm.OP["pool"]][0]
    assert mutate(pool, (2, 1, shapes[pool][2], 0, 0)) != 0  # pool output must be 1 x 1
    # FC on a spatial input: drop the pool (FC reads the ReLU output directly)
    fc = [v for v, n in enumerate(nodes) if n[0] == slm.OP["fc"]][0]
    n2 = list(nodes)
    n2[fc] = (slm.OP["fc"], [pool - 1], nodes[fc][2], 0)
    assert _create_shaped(n2, shapes, B) != 0


def test_rows_beyond_int32_rejected():
    """The op kernels index rows (batch H W) in 32 bits: a value with >= 2^31 rows is refused at
    model creation (runtime.cu), not overflowed at run time."""
    B, C_ = 64, 128
    big = 8192                                           # 64 * 8192 * 8192 = 2^32 rows
    nodes = [(slm.OP["input"], [], B * big * big * C_ * 4, 0), (slm.OP["pool"], [0], B * C_ * 4, 0),
             (slm.OP["fc"], [1], B * 128 * 4, 0), (slm.OP["softmax_ce"], [2], 4, 1)]
    shapes = [(big, big, C_, 0, 0), (1, 1, C_, 0, 0), (1, 1, 128, 0, 0), (1, 1, 1, 0, 0)]
    assert _create_shaped(nodes, shapes, B) != 0
    small = [(slm.OP["input"], [], B * 8 * 8 * C_ * 4, 0)] + nodes[1:]
    assert _create_shaped(small, [(8, 8, C_, 0, 0)] + shapes[1:], B) == 0
