"""Pins for the oracle's fp64 LSTM (CPU): torch.nn.LSTM in fp64 (an independent
implementation of the recurrence and of BPTT), finite differences, and bitwise plan
invariance of the V' interpreter for time-segment and budget plans."""
import numpy as np
import pytest
import torch

import synth
from oracle import graph as G
from oracle import lstm as OL
from oracle import planner as P


def _params(L, T, B, H, I, C, dtype="f32", seed=0):
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype=dtype, seed=seed)
    return OL.LstmParams(inp["W"], inp["b"], inp["W_o"], inp["b_o"], I), inp


def _torch(Pm, inp):
    L, H, I = Pm.L, Pm.H, Pm.n_in
    lstm = torch.nn.LSTM(I, H, num_layers=L, dtype=torch.float64)
    head = torch.nn.Linear(H, Pm.W_o.shape[0], dtype=torch.float64)
    with torch.no_grad():
        for l in range(L):
            kin = Pm.kin(l)
            w_ih = Pm.W[l][:, : (I if l == 0 else H)]
            getattr(lstm, f"weight_ih_l{l}").copy_(torch.tensor(w_ih))
            getattr(lstm, f"weight_hh_l{l}").copy_(torch.tensor(Pm.W[l][:, kin:]))
            getattr(lstm, f"bias_ih_l{l}").copy_(torch.tensor(Pm.b[l]))
            getattr(lstm, f"bias_hh_l{l}").zero_()
        head.weight.copy_(torch.tensor(Pm.W_o))
        head.bias.copy_(torch.tensor(Pm.b_o))
    x = torch.tensor(inp["x"], dtype=torch.float64)
    y, _ = lstm(x)
    logits = head(y)
    T, B = inp["labels"].shape
    loss = torch.nn.functional.cross_entropy(logits.reshape(T * B, -1),
                                             torch.tensor(inp["labels"].reshape(-1), dtype=torch.long))
    loss.backward()
    grads = dict(W_o=head.weight.grad.numpy(), b_o=head.bias.grad.numpy(), W=[], b=[])
    for l in range(L):
        kin = Pm.kin(l)
        gw = np.zeros_like(Pm.W[l])
        gw[:, : (I if l == 0 else H)] = getattr(lstm, f"weight_ih_l{l}").grad.numpy()
        gw[:, kin:] = getattr(lstm, f"weight_hh_l{l}").grad.numpy()
        grads["W"].append(gw)
        grads["b"].append(getattr(lstm, f"bias_ih_l{l}").grad.numpy())
    return loss.item(), grads


@pytest.mark.parametrize("L,T,B,H,I,C", [(1, 3, 2, 4, 3, 5), (2, 5, 3, 8, 5, 7), (3, 4, 2, 6, 50, 11)])
def test_lstm_matches_torch_fp64(L, T, B, H, I, C):
    Pm, inp = _params(L, T, B, H, I, C)
    loss, g = OL.step_plain(Pm, inp["x"], inp["labels"])
    tl, tg = _torch(Pm, inp)
    assert abs(loss - tl) < 1e-12 * max(1, abs(tl))
    np.testing.assert_allclose(g["W_o"], tg["W_o"], rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(g["b_o"], tg["b_o"], rtol=1e-9, atol=1e-13)
    for l in range(L):
        np.testing.assert_allclose(g["W"][l], tg["W"][l], rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(g["b"][l], tg["b"][l], rtol=1e-9, atol=1e-13)


def test_lstm_finite_differences():
    Pm, inp = _params(2, 3, 2, 3, 2, 4, seed=4)
    _, g = OL.step_plain(Pm, inp["x"], inp["labels"])
    rng = np.random.default_rng(1)
    h = 1e-6
    for name in ("W", "b"):
        for _ in range(6):
            l = int(rng.integers(0, Pm.L))
            arr = getattr(Pm, name)[l]
            idx = tuple(int(rng.integers(0, s)) for s in arr.shape)
            old = arr[idx]
            arr[idx] = old + h
            lp = OL.step_plain(Pm, inp["x"], inp["labels"])[0]
            arr[idx] = old - h
            lm = OL.step_plain(Pm, inp["x"], inp["labels"])[0]
            arr[idx] = old
            num = (lp - lm) / (2 * h)
            ana = g[name][l][idx]
            assert abs(num - ana) <= 1e-6 * max(1e-3, abs(ana)) + 1e-10, (name, l, idx, num, ana)


@pytest.mark.parametrize("plan_kind", ["none", "seg2", "seg3", "sqrt", "search"])
@pytest.mark.parametrize("mode", ["f64", "bf16"])
@pytest.mark.parametrize("flags", [P.A_INPLACE | P.A_SHARING, P.A_INPLACE | P.A_SHARING | P.A_GROUPED,
                                   P.A_INPLACE | P.A_SHARING | P.A_GROUPED | P.A_GROUP_MIRRORS])
def test_lstm_plan_invariance_bitwise(plan_kind, mode, flags):
    L, T, B, H, I, C = 2, 6, 3, 4, 3, 5
    Pm, inp = _params(L, T, B, H, I, C, dtype="bf16" if mode == "bf16" else "f32", seed=2)
    loss, g = OL.step_plain(Pm, inp["x"], inp["labels"], mode)
    gr = G.lstm_graph(L, T, B, H, Pm.kin(0))
    if plan_kind.startswith("seg"):
        p = P.plan(gr, P.S_EXPLICIT, m=OL.time_segment_plan(gr, int(plan_kind[3:])), alloc_flags=flags)
    else:
        p = P.plan(gr, {"none": P.S_NONE, "sqrt": P.S_SQRT, "search": P.S_SEARCH}[plan_kind], alloc_flags=flags)
    l2, g2 = OL.step_planned(p, Pm, inp["x"], inp["labels"], mode)
    assert loss == l2
    assert np.array_equal(g["W_o"], g2["W_o"]) and np.array_equal(g["b_o"], g2["b_o"])
    for l in range(L):
        assert np.array_equal(g["W"][l], g2["W"][l]), l
        assert np.array_equal(g["b"][l], g2["b"][l]), l


def test_lstm_time_segments_save_memory():
    # PAPER.md:490 "The sub-linear plan gives more than 4x reduction over the optimized memory
    # plan" (the paper's unroll length is garbled; here T = 64, segments of 8 = sqrt(T))
    gr = G.lstm_graph(4, 64, 64, 1024, 64)
    none = P.plan(gr, P.S_NONE).alloc.exact_peak
    seg = P.plan(gr, P.S_EXPLICIT, m=OL.time_segment_plan(gr, 8)).alloc.exact_peak
    assert seg * 4 < none, (seg, none)


def test_grouped_allocation_invariants():
    """Reading A22: with A_GROUPED every tag is only ever used by nodes of one allocation group
    (the LSTM layer, or the head); on a single-group graph it is the plain Fig. 2 allocator."""
    gr = G.lstm_graph(3, 10, 4, 8, 3)
    p = P.plan(gr, P.S_EXPLICIT, m=OL.time_segment_plan(gr, 3),
               alloc_flags=P.A_INPLACE | P.A_SHARING | P.A_GROUPED)
    users = {}
    for v in p.gg.order:
        users.setdefault(p.alloc.tag_of[v], set()).add(gr.nodes[p.gg.nodes[v].orig].group)
    assert all(len(s) == 1 for s in users.values())
    p2 = P.plan(gr, P.S_EXPLICIT, m=OL.time_segment_plan(gr, 3),
                alloc_flags=P.A_INPLACE | P.A_SHARING | P.A_GROUPED | P.A_GROUP_MIRRORS)
    kinds = {}
    for v in p2.gg.order:
        kinds.setdefault(p2.alloc.tag_of[v], set()).add(p2.gg.nodes[v].kind == "mirror")
    assert all(len(s) == 1 for s in kinds.values())    # mirrors never share with other nodes
    ch = G.chain_graph(40, 8, 64)
    a = P.plan(ch, P.S_SQRT, alloc_flags=P.A_INPLACE | P.A_SHARING).alloc
    b = P.plan(ch, P.S_SQRT, alloc_flags=P.A_INPLACE | P.A_SHARING | P.A_GROUPED).alloc
    assert a.tag_of == b.tag_of and a.offsets == b.offsets
