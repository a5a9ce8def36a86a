"""Pins for the convolutional op-graph oracle (oracle.opgraph Conv / GlobalAvgPool),
each against something other than itself:
  * Conv forward / backward == torch.nn.functional.conv2d and its autograd in fp64 (a library
    routine; NHWC <-> NCHW permutes), for 3x3 stride 1 / 2 and the 1x1 stride-2 projection, on
    odd and even spatial sizes ("same" zero padding, PAPER.md:431-446's ResNet convolutions);
  * a 1x1 stride-1 Conv is the FC node applied row by row (closed form);
  * GlobalAvgPool == the mean over positions, its backward the uniform spread (closed form);
  * central finite differences of the loss of a two-stage conv ResNet w.r.t. conv, BN and FC
    parameters;
  * every plan (none, sqrt, drop bn-relu, App. A search) interpreted through its tags gives
    step_plain's result bit for bit, fp64 and bf16 operand rounding."""
import numpy as np
import pytest
import torch

import synth
from oracle import graph as G
from oracle import opgraph as OG
from oracle import planner as P
from oracle.chain import bf16_round


def _torch_conv(x, W, b, B, H, Wd, Cin, k, s):
    Cout = W.shape[0]
    xt = torch.tensor(x.reshape(B, H, Wd, Cin)).permute(0, 3, 1, 2).requires_grad_(True)
    wt = torch.tensor(W.reshape(Cout, k, k, Cin)).permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    bt = torch.tensor(b).requires_grad_(True)
    y = torch.nn.functional.conv2d(xt, wt, bt, stride=s, padding=k // 2)
    return xt, wt, bt, y


@pytest.mark.parametrize("H,k,s", [(5, 3, 1), (6, 3, 2), (5, 3, 2), (6, 1, 2), (4, 1, 1)])
def test_conv_matches_torch_fp64(H, k, s):
    rng = np.random.default_rng(H * 10 + k + s)
    B, Cin, Cout = 2, 3, 4
    x = rng.standard_normal((B * H * H, Cin))
    W = rng.standard_normal((Cout, k * k * Cin))
    b = rng.standard_normal(Cout)
    y = OG.conv_forward(x, W, b, (H, H, Cin), k, s, "f64")
    xt, wt, bt, yt = _torch_conv(x, W, b, B, H, H, Cin, k, s)
    ref = yt.permute(0, 2, 3, 1).reshape(-1, Cout).detach().numpy()
    assert y.shape == ref.shape
    assert np.allclose(y, ref, rtol=1e-12, atol=1e-12)
    dy = rng.standard_normal(y.shape)
    yt.backward(torch.tensor(dy.reshape(yt.shape[0], yt.shape[2], yt.shape[3], Cout)).permute(0, 3, 1, 2))
    dx, dW, db = OG.conv_backward(dy, x, W, (H, H, Cin), k, s, "f64")
    assert np.allclose(dx, xt.grad.permute(0, 2, 3, 1).reshape(-1, Cin).numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(dW, wt.grad.permute(0, 2, 3, 1).reshape(Cout, -1).numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(db, bt.grad.numpy(), rtol=1e-12, atol=1e-12)


def test_conv_bf16_rounds_exactly_the_operands():
    rng = np.random.default_rng(7)
    B, H, Cin, Cout, k, s = 2, 4, 3, 5, 3, 2
    x = rng.standard_normal((B * H * H, Cin))
    W = rng.standard_normal((Cout, k * k * Cin))
    b = rng.standard_normal(Cout)
    y = OG.conv_forward(x, W, b, (H, H, Cin), k, s, "bf16")
    _, _, _, yt = _torch_conv(bf16_round(x), bf16_round(W), b, B, H, H, Cin, k, s)
    assert np.allclose(y, yt.permute(0, 2, 3, 1).reshape(-1, Cout).detach().numpy(), rtol=1e-12, atol=1e-12)
    dy = rng.standard_normal(y.shape)
    dx, dW, _ = OG.conv_backward(dy, x, W, (H, H, Cin), k, s, "bf16")
    dx64, dW64, _ = OG.conv_backward(bf16_round(dy), bf16_round(x), bf16_round(W), (H, H, Cin), k, s, "f64")
    assert np.array_equal(dx, dx64)
    assert np.array_equal(dW, bf16_round(dW64))


def test_conv_1x1_stride1_is_fc_per_row():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2 * 3 * 3, 6))
    W = rng.standard_normal((4, 6))
    b = rng.standard_normal(4)
    assert np.allclose(OG.conv_forward(x, W, b, (3, 3, 6), 1, 1, "f64"), x @ W.T + b, rtol=1e-13, atol=1e-13)


def test_pool_closed_form():
    g = G.Graph([G.Node(G.INPUT, [], 4), G.Node(G.POOL, [0], 4)], [1])
    Pm = OG.OpParams(shapes=[(3, 2, 4, 0, 0), (1, 1, 4, 0, 0)], graph=g)
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2 * 6, 4))
    y = OG.forward_node(G.POOL, 1, [x], Pm, "f64")
    assert np.allclose(y, x.reshape(2, 6, 4).mean(axis=1))
    dy = rng.standard_normal((2, 4))
    (dx,) = OG.backward_node(G.POOL, 1, dy, [x], y, Pm, "f64", {})
    assert np.allclose(dx.reshape(2, 6, 4), np.broadcast_to(dy[:, None, :] / 6, (2, 6, 4)))


def _conv_net(B=2, hw=4, stages=((4, 1), (6, 1)), classes=5, seed=5):
    g, shapes = G.preact_resnet_conv_graph(B, hw, stages, classes)
    nodes = [(nd.op, nd.preds, nd.out_bytes, nd.flags) for nd in g.nodes]
    inp = synth.opgraph_inputs(nodes, B, seed=seed, shapes=shapes)
    pr = inp["params"]
    Pm = OG.OpParams({v: p["W"] for v, p in pr.items() if "W" in p}, {v: p["b"] for v, p in pr.items() if "b" in p},
                     {v: p["gamma"] for v, p in pr.items() if "gamma" in p},
                     {v: p["beta"] for v, p in pr.items() if "beta" in p}, shapes=shapes, graph=g)
    return g, shapes, Pm, inp["x0"].astype(np.float64), inp["labels"]


def test_conv_graph_structure():
    g, shapes = G.preact_resnet_conv_graph(8, 16, [(128, 2), (256, 2)], 128)
    ops = [nd.op for nd in g.nodes]
    assert ops.count(G.CONV) == 2 * 4 + 1    # two 3x3 per block, one 1x1 projection
    assert ops.count(G.POOL) == 1 and ops[-1] == G.SOFTMAX_CE
    assert shapes[ops.index(G.POOL)] == (1, 1, 256, 0, 0)
    for v, nd in enumerate(g.nodes[:-1]):   # sizes follow the shapes
        H, W, C = shapes[v][:3]
        assert nd.out_bytes == 8 * H * W * C * 4
    proj = [v for v, nd in enumerate(g.nodes) if nd.op == G.CONV and shapes[v][3] == 1]
    assert len(proj) == 1 and shapes[proj[0]][4] == 2 and shapes[proj[0]][:3] == (8, 8, 256)
    assert G.validate(g) == []


def test_conv_graph_finite_differences():
    g, shapes, Pm, x0, y = _conv_net()
    loss, grads = OG.step_plain(g, Pm, x0, y)
    rng = np.random.default_rng(0)
    for kind in ("W", "b", "gamma", "beta"):
        table = getattr(Pm, kind)
        for v in list(table)[:4]:
            a = table[v]
            for _ in range(2):
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
def test_conv_plan_invariance_bitwise(strategy, mode):
    g, shapes, Pm, x0, y = _conv_net()
    loss, grads = OG.step_plain(g, Pm, x0, y, mode)
    plan = P.plan(g, strategy)
    l2, g2 = OG.step_planned(plan, g, Pm, x0, y, mode)
    assert l2 == loss
    for kind in grads:
        for v in grads[kind]:
            assert np.array_equal(grads[kind][v], g2[kind][v]), (strategy, kind, v)
    if strategy == P.S_DROP_CHEAP:
        assert plan.extra_forward > 0


@pytest.mark.parametrize("H", [5, 6])
def test_stride1_input_gradient_is_flipped_kernel_convolution(H):
    """The identity the device's 3x3 stride-1 input gradient uses (op_wflip_kernel):
    dx = conv(dy, Wt) with Wt[c][(u' k + v') C_out + o] = W[o][((k-1-u') k + (k-1-v')) C_in + c],
    stride 1, "same" padding -- checked on the oracle's conv_backward (itself pinned to torch above)."""
    rng = np.random.default_rng(H)
    B, Cin, Cout, k = 2, 3, 4, 3
    x = rng.standard_normal((B * H * H, Cin))
    W = rng.standard_normal((Cout, k * k * Cin))
    dy = rng.standard_normal((B * H * H, Cout))
    dx, _, _ = OG.conv_backward(dy, x, W, (H, H, Cin), k, 1, "f64")
    Wr = W.reshape(Cout, k * k, Cin)
    Wt = np.transpose(Wr[:, ::-1, :], (2, 1, 0)).reshape(Cin, k * k * Cout)   # [c][t'][o], t' = 8 - t
    dx2 = OG.conv_forward(dy, Wt, np.zeros(Cin), (H, H, Cout), k, 1, "f64")
    assert np.allclose(dx, dx2, rtol=1e-12, atol=1e-12)
