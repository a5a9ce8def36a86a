"""Device parity of the unrolled-LSTM training step (C3) through the C ABI (slm_step).

  * GPU vs the bf16-operand-emulating fp64 oracle (oracle.lstm.step_plain): loss and every
    gradient element by element, |g - ref| <= 2e-2 (|ref| + rms(ref)), and within 2e-2 relative
    norm (reading A12) — including the C3 shapes (L = 4, H = 1024, I = 50, C = 5000) with the
    bench's plan.
  * checkpointed GPU step == non-checkpointed GPU step, bit for bit, for the generic
    strategies and the time-segment plan of PAPER.md:486-490.
"""
import numpy as np
import pytest
import torch

import synth
from _util import assert_close
from oracle import lstm as OL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slm():
    import paper_1604_06174_b200 as m
    return m


def _dev(inp, L, H, C):
    """synth.lstm_inputs (bf16-valued, true widths) -> device tensors in the slm_lstm_desc layout
    (layer 0 padded to Kin0 by the binding's LstmModel.pack_w)."""
    import paper_1604_06174_b200 as slm
    Cp = -(-C // 128) * 128
    W = slm.LstmModel.pack_w(inp["W"], inp["n_in"]).to(torch.bfloat16).cuda()
    Wo = torch.zeros(Cp, H)
    Wo[:C] = torch.tensor(inp["W_o"])
    bo = torch.zeros(Cp)
    bo[:C] = torch.tensor(inp["b_o"])
    p = dict(W=W, b=torch.tensor(inp["b"]).cuda(), W_o=Wo.to(torch.bfloat16).cuda(), b_o=bo.cuda())
    g = dict(W=torch.empty(W.numel(), device="cuda"), b=torch.empty_like(p["b"]),
             W_o=torch.empty(Cp, H, device="cuda"), b_o=torch.empty(Cp, device="cuda"))
    return p, g, torch.tensor(inp["x"]).cuda(), torch.tensor(inp["labels"]).cuda()


def _run(slm, cfg, inp, strategy="none", m=None, alloc_flags=3, state_candidates=False, **opt):
    L, T, B, H, I, C = cfg
    p, g, x, y = _dev(inp, L, H, C)
    model = slm.LstmModel(p, g, L, T, B, H, I, C, **opt)
    graph = slm.Graph.lstm(L, T, B, H, I)
    if state_candidates:   # reading A25: only cell states are Alg. 3 split points
        graph.mark_not_candidate(slm.OP["lstm_gates"])
    plan = slm.Plan(graph, "explicit" if m is not None else strategy, m=m, alloc_flags=alloc_flags)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        loss = model.step(plan, x, y, stream=s)
        loss = model.step(plan, x, y, stream=s)   # graph replay (first call is eager + capture)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy().astype(np.float64) for k, v in g.items()}
    return float(loss.item()), out, plan


def _split_w(flat, inp):
    import paper_1604_06174_b200 as slm
    H = inp["W"][0].shape[0] // 4
    return slm.LstmModel.unpack_w(flat, len(inp["W"]), H, inp["n_in"])


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


# (L, T, B, H, I, C); T = 37 spans two weight-gradient chunks (32 + a ragged 5)
CFGS = [(2, 6, 64, 128, 50, 300), (1, 3, 128, 256, 50, 129), (3, 4, 64, 128, 200, 500), (1, 37, 64, 128, 50, 129)]


@pytest.mark.parametrize("cfg", CFGS)
def test_lstm_vs_oracle(slm, cfg):
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=sum(cfg))
    loss, g, _ = _run(slm, cfg, inp, "sqrt")
    P = OL.LstmParams(inp["W"], inp["b"], inp["W_o"], inp["b_o"], I)
    ol, og = OL.step_plain(P, inp["x"], inp["labels"], mode="bf16")
    _lstm_parity(loss, g, ol, og, inp, L, C)


def _lstm_parity(loss, g, ol, og, inp, L, C, tag="", max_frac=0.0):
    """loss, every W_l, b_l, W_o, b_o element by element (padded classes get no gradient)"""
    assert abs(loss - ol) / abs(ol) <= 2e-2, (tag, loss, ol)
    stats = {}
    for l, w in enumerate(_split_w(g["W"], inp)):
        stats[f"W{l}"] = assert_close(w, og["W"][l], 2e-2, f"{tag} W{l}", max_frac)
        stats[f"b{l}"] = assert_close(g["b"][l], og["b"][l], 2e-2, f"{tag} b{l}", max_frac)
    stats["W_o"] = assert_close(g["W_o"][:C], og["W_o"], 2e-2, f"{tag} W_o", max_frac)
    stats["b_o"] = assert_close(g["b_o"][:C], og["b_o"], 2e-2, f"{tag} b_o", max_frac)
    assert not np.any(g["W_o"][C:]) and not np.any(g["b_o"][C:])   # padded classes get no gradient
    return stats


@pytest.mark.slow
def test_lstm_c3_shapes_bench_plan_vs_oracle(slm):
    """C3's layer shapes (L = 4, H = 1024, I = 50 padded to 128, C = 5000 padded to 5120 — the head's
    class loops run 5 times) over T = 40 steps (one 32-step weight-gradient chunk plus a ragged 8),
    with the bench's plan: time segments, grouped allocation and recompute phases (A22, A24),
    the layer wavefront with mirror streams (lstm_streams = 2); element-wise against the oracle,
    all but 0.1 % of each tensor's elements (the bf16 rounding decisions of 160 dependent steps
    drift apart at the smallest elements of W_0: 0.02 % measured, relative L2 2.2e-3)."""
    cfg = (4, 40, 64, 1024, 50, 5000)
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=40)
    graph = slm.Graph.lstm(L, T, B, H, I)
    af = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_GROUPED | slm.ALLOC_MIRROR_PARITY
    m = graph.lstm_segment_mirrors(8)
    loss, g, plan = _run(slm, cfg, inp, m=m, alloc_flags=af, lstm_streams=2)
    assert plan.extra_forward > 0
    P = OL.LstmParams(inp["W"], inp["b"], inp["W_o"], inp["b_o"], I)
    ol, og = OL.step_plain(P, inp["x"], inp["labels"], mode="bf16")
    stats = _lstm_parity(loss, g, ol, og, inp, L, C, "C3 shapes", max_frac=1e-3)
    print("C3-shape parity (max_abs, rms_ref, rel_l2):", {k: tuple(f"{x:.2e}" for x in v) for k, v in stats.items()})


@pytest.mark.parametrize("cfg", [(2, 8, 64, 128, 50, 300), (1, 40, 64, 128, 50, 129)])
def test_lstm_ckpt_equals_nockpt_bitwise(slm, cfg):
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=7)
    ref_loss, ref, _ = _run(slm, cfg, inp, "none")
    runs = {s: _run(slm, cfg, inp, s) for s in ("sqrt", "search", "drop_cheap")}
    for seg in (2, 4):
        runs[f"seg{seg}"] = _run(slm, cfg, inp, m=slm.Graph.lstm(L, T, B, H, I).lstm_segment_mirrors(seg))
    for s, (loss, g, plan) in runs.items():
        assert loss == ref_loss, s
        for k in ref:
            assert np.array_equal(g[k], ref[k]), (s, k)
    # the time-segment plan re-computes and saves memory
    assert runs["seg4"][2].extra_forward > 0


def test_lstm_launch_count(slm):
    cfg = (2, 4, 64, 128, 50, 300)
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16")
    p, g, x, y = _dev(inp, L, H, C)
    model = slm.LstmModel(p, g, L, T, B, H, I, C, use_graph=0)
    plan = slm.Plan(slm.Graph.lstm(L, T, B, H, I), "none")
    # forward (one fused phase, lstm_run.cuh): per layer one run of the T = 4 steps (the input
    # projection GEMM and the persistent run kernel; layer 0 also packs its input); the heads run
    # batched per 32-step chunk (logits GEMM, CE rows, per-step losses); Sum 1.
    # backward: fill 1; the head gradients batched per 32-step chunk (pack, logits GEMM, CE,
    # dh GEMM, dh + db_o, dW_o GEMM); per t and layer 2 (fused cell / d_pre / pack, dX GEMM whose
    # partials the next cell gradients read in place); per chunk one weight-gradient GEMM + db
    # column sum per layer (T = 4: one chunk); the input gradient of a layer above 0 is a split-K
    # GEMM plus the slice-order sum of its partials (executor_lstm.cuh kDxSplit)
    assert model.launches(plan) == 2 * L + 1 + 3 + 1 + 1 + 6 + (1 + 5) * (L - 1) + (1 + 3)


@pytest.mark.parametrize("cfg", [(1, 1, 64, 128, 50, 129), (1, 2, 256, 128, 7, 128), (2, 33, 64, 128, 50, 200)])
def test_lstm_edge_sizes(slm, cfg):
    """T = 1 (no recurrence), batch 256 with a 7-wide input, a 33-step unroll (chunk + 1)."""
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=T + B)
    loss, g, _ = _run(slm, cfg, inp, "sqrt")
    P = OL.LstmParams(inp["W"], inp["b"], inp["W_o"], inp["b_o"], I)
    ol, og = OL.step_plain(P, inp["x"], inp["labels"], mode="bf16")
    _lstm_parity(loss, g, ol, og, inp, L, C, "edge")
    loss0, g0, _ = _run(slm, cfg, inp, "none")
    assert loss0 == loss
    for k in g0:
        assert np.array_equal(g0[k], g[k]), k


@pytest.mark.parametrize("cfg", [(1, 2, 256, 128, 7, 128), (3, 9, 64, 128, 50, 300)])
def test_lstm_wavefront_matches_single_stream(slm, cfg):
    """Race detection for the layer wavefront (lstm_streams=1): repeated steps must reproduce
    the single-stream step bit for bit (a missing happens-before edge shows up as a changed
    loss or gradient, e.g. a head reading a stale operand)."""
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=5)
    ref_loss, ref, _ = _run(slm, cfg, inp, m=slm.Graph.lstm(L, T, B, H, I).lstm_segment_mirrors(3),
                            lstm_streams=0)
    for rep in range(4):
        for pdl, af, ns in ((1, 3, 1), (0, 3, 1), (1, 7, 1), (1, 7, 2), (0, 3, 2), (1, 23, 2), (0, 19, 2)):
            loss, g, _ = _run(slm, cfg, inp, m=slm.Graph.lstm(L, T, B, H, I).lstm_segment_mirrors(3),
                              alloc_flags=af, lstm_streams=ns, pdl=pdl)
            assert loss == ref_loss, (rep, pdl, af)
            for k in ref:
                assert np.array_equal(g[k], ref[k]), (rep, pdl, af, k)


def test_lstm_sgd_training_reduces_loss(slm):
    L, T, B, H, I, C = 2, 16, 64, 128, 50, 200
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=13)
    p, g, x, y = _dev(inp, L, H, C)
    model = slm.LstmModel(p, g, L, T, B, H, I, C)
    graph = slm.Graph.lstm(L, T, B, H, I)
    plan = slm.Plan(graph, "explicit", m=graph.lstm_segment_mirrors(4), alloc_flags=7)
    losses = []
    for _ in range(6):
        losses.append(float(model.step(plan, x, y).item()))
        with torch.no_grad():
            for k in ("W", "W_o"):
                p[k].copy_((p[k].float() - 2.0 * g[k]).to(torch.bfloat16))
            for k in ("b", "b_o"):
                p[k].sub_(2.0 * g[k])
    assert all(b < a for a, b in zip(losses, losses[1:])), losses


def test_lstm_alternating_plans_share_buffers(slm):
    """Two plans stepped alternately on the same model and the same pool / workspace: every
    captured graph must keep reproducing its own step (no per-plan state left in the buffers)."""
    cfg = (2, 8, 64, 128, 50, 300)
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=17)
    p, g, x, y = _dev(inp, L, H, C)
    model = slm.LstmModel(p, g, L, T, B, H, I, C)
    graph = slm.Graph.lstm(L, T, B, H, I)
    pa = slm.Plan(graph, "explicit", m=graph.lstm_segment_mirrors(2), alloc_flags=7)
    pb = slm.Plan(graph, "none", alloc_flags=7)
    nbytes = max(pa.pool_bytes, pb.pool_bytes)
    pool = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ws = torch.empty(model.workspace_bytes(pa), dtype=torch.uint8, device="cuda")
    loss = torch.zeros(1, device="cuda")
    s = torch.cuda.Stream()
    out = []
    with torch.cuda.stream(s):
        for plan in (pa, pb, pa, pb, pa):
            model.step(plan, x, y, stream=s, bufs=(pool, ws, loss))
            torch.cuda.synchronize()
            out.append((float(loss.item()), g["W"].clone()))
    for a, b in zip(out, out[1:]):
        assert a[0] == b[0]
        assert torch.equal(a[1], b[1])



@pytest.mark.parametrize("cfg", [(2, 40, 64, 128, 50, 300), (3, 24, 64, 128, 50, 200)])
def test_lstm_search_plans_bitwise(slm, cfg):
    """The paper's App. A search over the LSTM grid graph, over all nodes and
    over cell states only (reading A25), with and without the A24 recompute phases: the
    checkpointed step equals the non-checkpointed one bit for bit, repeatedly."""
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=8)
    ref_loss, ref, _ = _run(slm, cfg, inp)
    for sc in (False, True):
        for af in (7, 23):
            for _ in range(2):
                loss, g, plan = _run(slm, cfg, inp, strategy="search", alloc_flags=af, state_candidates=sc)
                assert plan.extra_forward > 0
                assert loss == ref_loss, (sc, af)
                for k in ref:
                    assert np.array_equal(g[k], ref[k]), (sc, af, k)


def test_lstm_overlapped_recompute_race_midsize(slm):
    """Race detection for the overlapped recompute at a mid size (4 layers, 130 steps, 32-step
    segments: 4 recompute phases running under the next segment's backward on the mirror
    streams): repeated steps reproduce the non-checkpointed step bit for bit."""
    cfg = (4, 130, 64, 256, 50, 300)
    L, T, B, H, I, C = cfg
    inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=12)
    ref_loss, ref, _ = _run(slm, cfg, inp, alloc_flags=23)
    m = slm.Graph.lstm(L, T, B, H, I).lstm_segment_mirrors(32)
    for rep in range(3):
        loss, g, plan = _run(slm, cfg, inp, m=m, alloc_flags=23, lstm_streams=2)
        assert loss == ref_loss, rep
        for k in ref:
            assert np.array_equal(g[k], ref[k]), (rep, k)
