"""Pins for the op-granularity oracle (oracle.opgraph), each against something
other than itself:
  * a one-stage pre-activation graph (BN -> ReLU -> FC -> Add per layer) with the chain's
    parameters IS the residual chain of reading A10: loss and gradients equal oracle.chain's
    step_plain bit for bit (fp64, and the bf16 operand rounding);
  * central finite differences on a two-stage graph with an FC projection between widths;
  * every plan (none, sqrt, drop-cheap = drop bn-relu, App. A search) interpreted through its tags
    gives step_plain's result bit for bit, with the interference check on."""
import numpy as np
import pytest

import synth
from oracle import chain as OC
from oracle import graph as G
from oracle import opgraph as OG
from oracle import planner as P


def _params_from_chain(inp, n):
    # node ids of preact_resnet_graph([n], ...): 0 Input, then 4 per layer (BN, ReLU, FC, Add)
    W, b, gam, bet = {}, {}, {}, {}
    for l in range(n):
        bn, fc = 1 + 4 * l, 3 + 4 * l
        gam[bn], bet[bn] = inp["gamma"][l], inp["beta"][l]
        W[fc], b[fc] = inp["W"][l], inp["b"][l]
    return OG.OpParams(W, b, gam, bet)


@pytest.mark.parametrize("mode", ["f64", "bf16"])
def test_one_stage_graph_is_the_chain(mode):
    n, B, d = 5, 16, 32
    inp = synth.chain_inputs(n, B, d, dtype="bf16" if mode == "bf16" else "f32", seed=4)
    g = G.preact_resnet_graph([n], [B * d * 4])
    loss, grads = OG.step_plain(g, _params_from_chain(inp, n), inp["x0"], inp["labels"], mode)
    cl, cg, _ = OC.step_plain(OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"]), inp["x0"], inp["labels"], mode)
    assert loss == cl
    for l in range(n):
        assert np.array_equal(grads["W"][3 + 4 * l], cg["W"][l])
        assert np.array_equal(grads["b"][3 + 4 * l], cg["b"][l])
        assert np.array_equal(grads["gamma"][1 + 4 * l], cg["gamma"][l])
        assert np.array_equal(grads["beta"][1 + 4 * l], cg["beta"][l])


def _two_stage(B=6, d0=8, d1=12, seed=3):
    rng = np.random.default_rng(seed)
    g = G.preact_resnet_graph([2, 2], [B * d0 * 4, B * d1 * 4])
    W, b, gam, bet = {}, {}, {}, {}
    for v, nd in enumerate(g.nodes):
        if nd.op == G.FC:
            dout, din = nd.out_bytes // (4 * B), g.nodes[nd.preds[0]].out_bytes // (4 * B)
            W[v] = rng.standard_normal((dout, din)) / np.sqrt(din)
            b[v] = 0.1 * rng.standard_normal(dout)
        elif nd.op == G.BN:
            dd = nd.out_bytes // (4 * B)
            gam[v], bet[v] = 1 + 0.1 * rng.standard_normal(dd), 0.1 * rng.standard_normal(dd)
    x0 = rng.standard_normal((B, d0))
    y = rng.integers(0, d1, size=B)
    return g, OG.OpParams(W, b, gam, bet), x0, y


def test_finite_differences_two_stages_with_projection():
    g, Pm, x0, y = _two_stage()
    loss, grads = OG.step_plain(g, Pm, x0, y)
    rng = np.random.default_rng(0)
    for kind in ("W", "b", "gamma", "beta"):
        table = getattr(Pm, kind)
        for v in list(table)[:3]:
            a = table[v]
            for _ in range(3):
                idx = tuple(int(rng.integers(0, s)) for s in a.shape)
                h = 1e-6
                old = a[idx]
                a[idx] = old + h
                lp, _ = OG.step_plain(g, Pm, x0, y)
                a[idx] = old - h
                lm, _ = OG.step_plain(g, Pm, x0, y)
                a[idx] = old
                fd = (lp - lm) / (2 * h)
                an = grads[kind][v][idx]
                assert abs(fd - an) <= 1e-5 * max(1.0, abs(an)), (kind, v, idx, fd, an)


@pytest.mark.parametrize("strategy", [P.S_NONE, P.S_SQRT, P.S_DROP_CHEAP, P.S_SEARCH])
@pytest.mark.parametrize("mode", ["f64", "bf16"])
def test_plan_invariance_bitwise(strategy, mode):
    g, Pm, x0, y = _two_stage()
    loss, grads = OG.step_plain(g, Pm, x0, y, mode)
    plan = P.plan(g, strategy)
    l2, g2 = OG.step_planned(plan, g, Pm, x0, y, mode)
    assert l2 == loss
    for kind in grads:
        for v in grads[kind]:
            assert np.array_equal(grads[kind][v], g2[kind][v]), (strategy, kind, v)
    if strategy == P.S_DROP_CHEAP:
        assert plan.extra_forward > 0   # BN / ReLU outputs are re-computed
