"""Pins for the oracle's fp64 chain numerics (CPU).

Independent references: torch.autograd in fp64 (a separate implementation of the forward
through library ops and of reverse mode), central finite differences, closed forms and
batch-norm identities.  The paper's safety claim ("all the memory
optimizations ... gives equivalent weight gradient") is checked bit for bit inside the
oracle for every planner strategy."""
import numpy as np
import pytest
import torch

import synth
from oracle import chain as C
from oracle import graph as G
from oracle import planner as P


def _params(n, B, d, dtype="f32", seed=7):
    inp = synth.chain_inputs(n, B, d, dtype=dtype, seed=seed)
    return C.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"]), inp


def _torch_step(Pm, x0, labels, batch_global=None):
    """Reference written with torch library ops (batch_norm, relu, linear, cross_entropy)."""
    W = torch.tensor(Pm.W, requires_grad=True)
    b = torch.tensor(Pm.b, requires_grad=True)
    ga = torch.tensor(Pm.gamma, requires_grad=True)
    be = torch.tensor(Pm.beta, requires_grad=True)
    x = torch.tensor(np.asarray(x0, np.float64))
    for l in range(Pm.n):
        h = torch.nn.functional.batch_norm(x, None, None, ga[l], be[l], training=True, eps=1e-5)
        x = x + torch.nn.functional.linear(torch.relu(h), W[l], b[l])
    Bg = batch_global or x.shape[0]
    loss = torch.nn.functional.cross_entropy(x, torch.tensor(labels, dtype=torch.long),
                                             reduction="sum") / Bg
    loss.backward()
    return loss.item(), dict(W=W.grad.numpy(), b=b.grad.numpy(), gamma=ga.grad.numpy(),
                             beta=be.grad.numpy())


@pytest.mark.parametrize("n,B,d", [(1, 4, 3), (3, 8, 5), (16, 8, 64)])
def test_chain_matches_torch_autograd_fp64(n, B, d):
    Pm, inp = _params(n, B, d)
    loss, grads, _ = C.step_plain(Pm, inp["x0"], inp["labels"])
    tl, tg = _torch_step(Pm, inp["x0"], inp["labels"])
    assert abs(loss - tl) <= 1e-12 * max(1, abs(tl))
    for k in grads:
        np.testing.assert_allclose(grads[k], tg[k], rtol=1e-9, atol=1e-12)


def test_finite_differences():
    # central differences in fp64: relative error < 1e-6
    n, B, d = 3, 6, 4
    Pm, inp = _params(n, B, d, seed=1)
    x0, y = inp["x0"].astype(np.float64), inp["labels"]
    _, grads, dx0 = C.step_plain(Pm, x0, y)
    rng = np.random.default_rng(0)
    h = 1e-6
    for name in ("W", "b", "gamma", "beta", "x0"):
        for _ in range(6):
            if name == "x0":
                arr = x0
            else:
                arr = getattr(Pm, name)
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            old = arr[idx]
            arr[idx] = old + h
            lp = C.step_plain(Pm, x0, y)[0]
            arr[idx] = old - h
            lm = C.step_plain(Pm, x0, y)[0]
            arr[idx] = old
            num = (lp - lm) / (2 * h)
            ana = dx0[idx] if name == "x0" else grads[name][idx]
            assert abs(num - ana) <= 1e-6 * max(1e-3, abs(ana)) + 1e-9, (name, idx, num, ana)


def test_closed_form_zero_weights():
    # W == 0: x_n = x_0 + sum_l b_l, and dx_l = dx_n for every l (only the residual path)
    n, B, d = 5, 4, 6
    Pm, inp = _params(n, B, d)
    Pm.W[:] = 0.0
    x0 = inp["x0"].astype(np.float64)
    xn = x0.copy()
    for l in range(n):
        xn = C.block_forward(xn, Pm, l)
    np.testing.assert_allclose(xn, x0 + Pm.b.sum(axis=0), rtol=0, atol=1e-12)
    _, grads, dx0 = C.step_plain(Pm, x0, inp["labels"])
    xlast = x0 + Pm.b.sum(axis=0)
    e = np.exp(xlast - xlast.max(axis=1, keepdims=True))
    sm = e / e.sum(axis=1, keepdims=True)
    onehot = np.eye(d)[inp["labels"]]
    np.testing.assert_allclose(dx0, (sm - onehot) / B, atol=1e-14)
    np.testing.assert_allclose(grads["gamma"], 0, atol=1e-14)


def test_closed_form_zero_layers():
    B, d = 5, 7
    x = np.random.default_rng(2).standard_normal((B, d))
    y = np.arange(B) % d
    Pm = C.Params(np.zeros((0, d, d)), np.zeros((0, d)), np.zeros((0, d)), np.zeros((0, d)))
    loss, _, dx0 = C.step_plain(Pm, x, y)
    ref = -np.log(np.exp(x[np.arange(B), y]) / np.exp(x).sum(axis=1)).mean()
    assert abs(loss - ref) < 1e-13
    sm = np.exp(x) / np.exp(x).sum(axis=1, keepdims=True)
    np.testing.assert_allclose(dx0, (sm - np.eye(d)[y]) / B, atol=1e-15)


def test_bn_backward_identities():
    # per feature: sum_b (dx_l - dx_{l+1}) = 0 and sum_b (dx_l - dx_{l+1}) * xhat = 0
    n, B, d = 1, 16, 8
    Pm, inp = _params(n, B, d)
    x = inp["x0"].astype(np.float64)
    g = np.random.default_rng(3).standard_normal((B, d))
    dx, (_, _, dgamma, _) = C.block_backward(g, x, Pm, 0)
    rstd = 1 / np.sqrt(x.var(0) + 1e-5)
    xhat = (x - x.mean(0)) * rstd
    np.testing.assert_allclose((dx - g).sum(0), 0, atol=1e-12)
    # with eps > 0, sum_b xhat^2 = B var rstd^2 = B (1 - eps rstd^2), so the second identity
    # is sum_b (dx - g) xhat = eps rstd^3 gamma dgamma
    np.testing.assert_allclose(((dx - g) * xhat).sum(0),
                               1e-5 * rstd ** 3 * Pm.gamma[0] * dgamma, rtol=1e-6, atol=1e-13)


@pytest.mark.parametrize("strategy,kw", [(P.S_NONE, {}), (P.S_SQRT, {}), (P.S_SEARCH, {}),
                                         (P.S_BUDGET, {"budget": 3 * 8 * 16 * 4}),
                                         (P.S_RECURSIVE, {"k": 1}), (P.S_RECURSIVE, {"k": 2})])
@pytest.mark.parametrize("mode", ["f64", "bf16"])
def test_plan_invariance_bitwise(strategy, kw, mode):
    # every plan gives the same gradients; the oracle reaches them bit for bit
    n, B, d = 16, 8, 16
    Pm, inp = _params(n, B, d, dtype="bf16" if mode == "bf16" else "f32")
    loss, grads, dx0 = C.step_plain(Pm, inp["x0"], inp["labels"], mode)
    p = P.plan(G.chain_graph(n, B, d), strategy, **kw)
    l2, g2, dx2, st = C.step_planned(p, Pm, inp["x0"], inp["labels"], mode)
    assert loss == l2
    for k in grads:
        assert np.array_equal(grads[k], g2[k]), k
    assert np.array_equal(dx0, dx2)
    # the interpreter's liveness peak (values still to be read, in-place outputs replacing their
    # input) never exceeds the planned pool, and Fig. 2's sharing allocator is tight on a chain
    assert st["peak_live_bytes"] <= p.alloc.exact_peak
    assert st["peak_live_bytes"] == p.alloc.exact_peak
    assert st["op_evaluations"] == (n + 1) + (n + 1) + p.extra_forward


@pytest.mark.parametrize("strategy", [P.S_NONE, P.S_SQRT, P.S_RECURSIVE])
def test_liveness_peak_vs_allocator(strategy):
    """Without sharing (PAPER.md:165-172 'memory sharing' off) the pool holds every tag (Sigma of
    the sizes) while the values' liveness peak stays the same: the gap is what sharing saves."""
    n, B, d = 16, 8, 16
    Pm, inp = _params(n, B, d)
    shared = P.plan(G.chain_graph(n, B, d), strategy, alloc_flags=P.A_INPLACE | P.A_SHARING)
    unshared = P.plan(G.chain_graph(n, B, d), strategy, alloc_flags=0)
    l1 = C.step_planned(shared, Pm, inp["x0"], inp["labels"])[3]["peak_live_bytes"]
    l0 = C.step_planned(unshared, Pm, inp["x0"], inp["labels"])[3]["peak_live_bytes"]
    assert l1 == shared.alloc.exact_peak
    # without in-place an op's input and output coexist: at most one more value than with it
    assert l1 <= l0 <= l1 + B * d * 4 < unshared.alloc.exact_peak


def test_planned_detects_clobber():
    n, B, d = 8, 4, 4
    Pm, inp = _params(n, B, d)
    p = P.plan(G.chain_graph(n, B, d), P.S_SQRT)
    # corrupt the plan: put a mirror in the tag of a kept segment boundary
    mirror = next(v for v in p.gg.order if p.gg.nodes[v].kind == "mirror")
    p.alloc.tag_of[mirror] = p.alloc.tag_of[4]
    with pytest.raises(C.TagClobber):
        C.step_planned(p, Pm, inp["x0"], inp["labels"])


def test_bf16_round_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(10000) * 10.0 ** rng.integers(-8, 8, 10000),
                        # exact ties: 1 + 2^-8 (tie -> even) and 1 + 3*2^-8
                        [1 + 2 ** -8, 1 + 3 * 2 ** -8, -1 - 2 ** -8, 0.0, -0.0]]).astype(np.float32)
    want = torch.tensor(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(C.bf16_round(x), want)
    np.testing.assert_array_equal(synth.bf16_values(x).astype(np.float64), want)


def test_bf16_emulation_close_to_fp64():
    n, B, d = 8, 16, 32
    Pm, inp = _params(n, B, d, dtype="bf16")
    l64, g64, _ = C.step_plain(Pm, inp["x0"], inp["labels"], "f64")
    l16, g16, _ = C.step_plain(Pm, inp["x0"], inp["labels"], "bf16")
    assert abs(l64 - l16) / abs(l64) < 1e-2
    for k in g64:
        assert np.linalg.norm(g16[k] - g64[k]) / np.linalg.norm(g64[k]) < 3e-2, k


def test_dp_emulation():
    # world = 1 is the single-GPU oracle; world = 2 equals the mean over shards of
    # shard-local grads (per-shard BN, reading A14), checked against torch per shard
    n, B, d = 3, 8, 6
    Pm, inp = _params(n, B, d)
    l1, g1 = C.step_dp(Pm, inp["x0"], inp["labels"], 1)
    l0, g0, _ = C.step_plain(Pm, inp["x0"], inp["labels"])
    assert l1 == l0 and all(np.array_equal(g1[k], g0[k]) for k in g0)
    l2, g2 = C.step_dp(Pm, inp["x0"], inp["labels"], 2)
    ta, ga = _torch_step(Pm, inp["x0"][:4], inp["labels"][:4], batch_global=8)
    tb, gb = _torch_step(Pm, inp["x0"][4:], inp["labels"][4:], batch_global=8)
    assert abs(l2 - (ta + tb)) < 1e-12
    for k in g2:
        np.testing.assert_allclose(g2[k], ga[k] + gb[k], rtol=1e-9, atol=1e-12)
