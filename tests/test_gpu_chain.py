"""Device parity of the checkpointed training step through the C ABI (slm_step).

  * GPU vs the fp64 oracle, element by element (reading A12): |g - ref| <= tol (|ref| + rms(ref))
    for every element of the loss and of every gradient tensor, and the relative L2 error <= tol;
    tol = 1e-4 (f32, C1) and 2e-2 (bf16, against the bf16-operand-emulating oracle).
  * checkpointed GPU step == non-checkpointed GPU step, bit for bit, for every strategy.
  * full C2 size (n=1024, d=2048, B=256): the same bit-exactness plus closed forms.
Inputs with a ReLU-margin screen (reading A20) are used where the 1e-4 f32 bar needs it and at
small bf16 sizes; the C2-width tests use plain seeded inputs (a rare flipped ReLU mask bit moves
one term of one batch sum, far inside the bf16 bound).
"""
import numpy as np
import pytest
import torch

import synth
from _util import assert_close, assert_close_chain, margin_inputs
from oracle import chain as OC
from oracle import graph as OG
from oracle import planner as OP

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slm():
    import paper_1604_06174_b200 as m
    return m


def _dev(inp, dtype):
    wdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    p = dict(W=torch.tensor(inp["W"]).to(wdt).cuda(), b=torch.tensor(inp["b"]).cuda(),
             gamma=torch.tensor(inp["gamma"]).cuda(), beta=torch.tensor(inp["beta"]).cuda())
    g = dict(W=torch.empty_like(p["W"]), b=torch.empty_like(p["b"]), gamma=torch.empty_like(p["gamma"]),
             beta=torch.empty_like(p["beta"]))
    return p, g, torch.tensor(inp["x0"]).cuda(), torch.tensor(inp["labels"]).cuda()


def _run(slm, n, B, d, dtype, strategy, inp=None, **opt):
    inp = inp or synth.chain_inputs(n, B, d, dtype=dtype)
    p, g, x0, y = _dev(inp, dtype)
    model = slm.ChainModel(p, g, dtype=dtype, batch=B, **opt)
    plan = slm.Plan(slm.Graph.chain(n, B, d), strategy)
    loss = model.step(plan, x0, y)
    torch.cuda.synchronize()
    return float(loss.item()), {k: v.float().cpu().numpy().astype(np.float64) for k, v in g.items()}, \
        (model, plan, p, g, x0, y)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _parity(loss, grads, ol, og, tol, tag="", inp=None):
    """loss and every gradient tensor element by element; returns {name: (max_abs, rms_ref, rel, ...)}.
    bf16 (inp given): the positions a decision-ambiguous ReLU can move (reading A20,
    _util.ambiguous_features) are held to the relative-L2 bound only."""
    assert abs(loss - ol) <= tol * abs(ol), (tag, loss, ol)
    if inp is not None:
        P = OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"])
        return assert_close_chain(grads, og, P, inp["x0"], tol, tag)
    return {k: assert_close(grads[k], og[k], tol, f"{tag} {k}") for k in og}


def _oracle(n, B, d, dtype, inp):
    Pm = OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"])
    return OC.step_plain(Pm, inp["x0"], inp["labels"], "bf16" if dtype == "bf16" else "f64")


@pytest.mark.parametrize("strategy", ["none", "sqrt", "search", "recursive"])
def test_c1_f32_vs_oracle(slm, strategy):
    n, B, d = 16, 8, 64
    inp = margin_inputs(n, B, d, "f32")
    loss, grads, _ = _run(slm, n, B, d, "f32", strategy, inp)
    ol, og, _ = _oracle(n, B, d, "f32", inp)
    _parity(loss, grads, ol, og, 1e-4, strategy)


@pytest.mark.parametrize("n,B,d", [(3, 64, 256), (2, 64, 128), (2, 128, 384), (2, 128, 512), (2, 256, 512),
                                   (2, 256, 640), (2, 256, 2048)])
@pytest.mark.parametrize("impl", [0, 1])
def test_bf16_vs_oracle(slm, n, B, d, impl):
    """The fused Block kernel (impl 0) at every cluster split it dispatches (block_split: S = 4 at
    d % 256 == 0, S = 2 at B <= 128 with d = 128 / 384) and the SIMT path (impl 1), element by
    element against the oracle.  Shallow chains: deeper ones drift from the oracle through
    decision chaos for every implementation alike (test_bf16_depth_vs_oracle, reading A20)."""
    inp = (margin_inputs(n, B, d, "bf16", seed=n + B + d) if n * B * d <= 300_000
           else synth.chain_inputs(n, B, d, dtype="bf16", seed=n + B + d))
    loss, grads, (model, *_rest) = _run(slm, n, B, d, "bf16", "sqrt", inp, gemm_impl=impl)
    if impl == 0:
        assert model.get_option("block_split") == (4 if d % 256 == 0 else 2)
    ol, og, _ = _oracle(n, B, d, "bf16", inp)
    _parity(loss, grads, ol, og, 2e-2, f"impl{impl}", inp)


@pytest.mark.parametrize("dtype,n,B,d", [("f32", 16, 8, 64), ("bf16", 24, 64, 256), ("bf16", 9, 256, 512)])
def test_ckpt_equals_nockpt_bitwise(slm, dtype, n, B, d):
    inp = synth.chain_inputs(n, B, d, dtype=dtype, seed=3)
    ref_loss, ref, _ = _run(slm, n, B, d, dtype, "none", inp)
    for s in ["sqrt", "search", "recursive"]:
        loss, grads, _ = _run(slm, n, B, d, dtype, s, inp)
        assert loss == ref_loss, s
        for k in ref:
            assert np.array_equal(grads[k], ref[k]), (s, k)


def test_graph_replay_and_no_allocation(slm):
    n, B, d = 12, 64, 256
    loss0, g0, (model, plan, p, g, x0, y) = _run(slm, n, B, d, "bf16", "sqrt", use_graph=0)
    model2 = slm.ChainModel(p, g, dtype="bf16", batch=B, use_graph=1)
    bufs = model2.buffers(plan)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):   # eager + capture, then two replays
            loss = model2.step(plan, x0, y, stream=s, bufs=bufs)
    torch.cuda.synchronize()
    assert torch.cuda.max_memory_allocated() == base          # slm_step never allocates
    assert float(loss.item()) == loss0
    for k in g0:
        assert np.array_equal(g[k].float().cpu().numpy().astype(np.float64), g0[k])


def test_pool_is_plan_sized(slm):
    n, B, d = 16, 64, 256
    plan = slm.Plan(slm.Graph.chain(n, B, d), "sqrt")
    u = B * d * 4
    assert plan.exact_peak == 8 * u + 4                  # tests/golden/sqrt_peaks.txt
    assert plan.pool_bytes == 7 * u                      # X_0 and the loss are caller buffers


@pytest.mark.slow
def test_c2_full_size_bitwise_and_closed_form(slm):
    # BASELINE.json configs[1] at full size: n=1024, d=2048, B=256, bf16 — in the bench's launch
    # configuration (tcgen05 path, CUDA graph)
    n, B, d = 1024, 256, 2048
    t = synth.chain_inputs_torch(n, B, d, dtype="bf16", seed=5)
    p = {k: t[k] for k in ("W", "b", "gamma", "beta")}
    out = {}
    par = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_MIRROR_PARITY
    for s in ("none", "sqrt", "sqrt+A24"):   # sqrt+A24 = the bench's plan (overlapped recompute)
        g = dict(W=torch.empty_like(p["W"]), b=torch.empty_like(p["b"]), gamma=torch.empty_like(p["gamma"]),
                 beta=torch.empty_like(p["beta"]))
        model = slm.ChainModel(p, g, dtype="bf16", batch=B)
        plan = slm.Plan(slm.Graph.chain(n, B, d), s.split("+")[0], alloc_flags=par if "A24" in s else 3)
        strm = torch.cuda.Stream()
        with torch.cuda.stream(strm):
            loss = model.step(plan, t["x0"], t["labels"], stream=strm)
            loss = model.step(plan, t["x0"], t["labels"], stream=strm)   # graph replay
        torch.cuda.synchronize()
        out[s] = (loss.item(), {k: v.clone() for k, v in g.items()})
        del model, g
    for s in ("sqrt", "sqrt+A24"):
        assert out["none"][0] == out[s][0], s
        for k in out["none"][1]:
            assert torch.equal(out["none"][1][k], out[s][1][k]), (s, k)
    # property that holds at any size: db_l = sum_b dx_{l+1} and BN backward conserves the
    # per-feature sum, so db is identical for every layer up to fp32 rounding
    db = out["sqrt"][1]["b"]
    assert torch.allclose(db[0], db[-1], rtol=1e-3, atol=1e-6)
    assert np.isfinite(out["sqrt"][0])


def _norm_parity(loss, grads, ol, og, tol, tag):
    """per-tensor relative L2 <= tol (north_star's bf16 bar) at depth; the element-wise statistics
    are reported (a deep bf16 chain's rare decision flips make individual elements drift)"""
    assert abs(loss - ol) <= tol * abs(ol), (tag, loss, ol)
    out = {}
    for k in og:
        rel = _rel(grads[k], og[k])
        err = np.abs(grads[k] - og[k])
        frac = float((err > tol * (np.abs(og[k]) + np.sqrt(np.mean(og[k] ** 2)))).mean())
        out[k] = (rel, float(err.max()), frac)
        assert rel <= tol, (tag, k, rel)
    print(tag, {k: f"rel {v[0]:.2e} max_abs {v[1]:.2e} frac_outside_elementwise {v[2]:.1e}" for k, v in out.items()})
    return out


@pytest.mark.parametrize("n,B,d", [(8, 64, 256), (8, 256, 2048)])
def test_bf16_depth_vs_oracle(slm, n, B, d):
    """Depth 8 (the C2 width and batch included): per-tensor relative L2 within 2e-2 of the oracle.
    Element-wise agreement is checked per Block (test_gpu_block.py) and on shallow chains."""
    inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=16)
    loss, grads, _ = _run(slm, n, B, d, "bf16", "sqrt", inp)
    ol, og, _ = _oracle(n, B, d, "bf16", inp)
    _norm_parity(loss, grads, ol, og, 2e-2, f"depth n={n} B={B} d={d}")


@pytest.mark.slow
def test_c2_width_bench_plan_vs_oracle(slm):
    """The bench's exact plan and launch configuration at C2 width and batch: sqrt(n) segments with
    mirror-run parity (A24), the recompute overlapped with the backward on its own stream
    (asserted through last_overlap), CUDA graph replay; against the oracle (n = 9: three segments
    of three, so two recompute runs overlap the backward)."""
    n, B, d = 9, 256, 2048
    inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=16)
    p, g, x0, y = _dev(inp, "bf16")
    model = slm.ChainModel(p, g, dtype="bf16", batch=B)
    par = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_MIRROR_PARITY
    plan = slm.Plan(slm.Graph.chain(n, B, d), "sqrt", alloc_flags=par)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):   # eager + capture, then a replay
            loss = model.step(plan, x0, y, stream=s)
    torch.cuda.synchronize()
    assert model.get_option("last_overlap") == 1
    grads = {k: v.float().cpu().numpy().astype(np.float64) for k, v in g.items()}
    ol, og, _ = _oracle(n, B, d, "bf16", inp)
    _norm_parity(float(loss.item()), grads, ol, og, 2e-2, "bench plan")


def test_zero_weights_closed_form(slm):
    # W == 0: x_n = x_0 + sum_l b_l and dx_l = dx_n; then dgamma = 0 and db_l is the column sum
    n, B, d = 6, 64, 256
    inp = synth.chain_inputs(n, B, d, dtype="bf16")
    inp["W"][:] = 0
    loss, grads, _ = _run(slm, n, B, d, "bf16", "sqrt", inp)
    x = inp["x0"].astype(np.float64) + inp["b"].astype(np.float64).sum(0)
    e = np.exp(x - x.max(1, keepdims=True))
    sm = e / e.sum(1, keepdims=True)
    ref = -np.log(sm[np.arange(B), inp["labels"]]).mean()
    assert abs(loss - ref) < 1e-5
    dxn = (sm - np.eye(d)[inp["labels"]]) / B
    for l in range(n):
        np.testing.assert_allclose(grads["b"][l], dxn.sum(0), atol=1e-6)
    assert np.abs(grads["gamma"]).max() == 0.0


def test_comm_world1_equals_no_comm(slm):
    """The data-parallel path (NCCL communicator, bucketed all-reduce on the comm stream,
    batch_global scaling) at world size 1 must reproduce the single-GPU step bit for bit."""
    n, B, d = 12, 64, 256
    inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=4)
    ref_loss, ref, _ = _run(slm, n, B, d, "bf16", "sqrt", inp)
    p, g, x0, y = _dev(inp, "bf16")
    model = slm.ChainModel(p, g, dtype="bf16", batch=B, batch_global=B)
    comm = slm.Comm(0, 1, bucket_bytes=2 * d * d * 2)   # several buckets
    par = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_MIRROR_PARITY
    for af in (3, par):   # sequential recompute, and the bench's overlapped recompute (A24)
        plan = slm.Plan(slm.Graph.chain(n, B, d), "sqrt", alloc_flags=af)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(2):
                loss = model.step(plan, x0, y, stream=s, comm=comm)
        torch.cuda.synchronize()
        assert model.get_option("last_overlap") == (af == par)
        assert float(loss.item()) == ref_loss, af
        for k in ref:
            assert np.array_equal(g[k].float().cpu().numpy().astype(np.float64), ref[k]), (af, k)


@pytest.mark.parametrize("dtype,n,B,d", [("f32", 1, 8, 64), ("f32", 2, 5, 48), ("f32", 3, 33, 80),
                                         ("bf16", 1, 64, 256), ("bf16", 2, 64, 128), ("bf16", 3, 128, 384)])
def test_edge_sizes_vs_oracle(slm, dtype, n, B, d):
    """Degenerate and ragged shapes: a single block, batch/width that are not tile multiples
    (f32 SIMT path), width not a multiple of 256 (bf16 basic lowering)."""
    tol = 1e-4 if dtype == "f32" else 2e-2
    inp = margin_inputs(n, B, d, dtype, seed=n * 100 + B + d)
    for strategy in ("none", "sqrt"):
        loss, grads, _ = _run(slm, n, B, d, dtype, strategy, inp)
        ol, og, _ = _oracle(n, B, d, dtype, inp)
        _parity(loss, grads, ol, og, tol, strategy, inp if dtype == "bf16" else None)


@pytest.mark.parametrize("strategy,kw", [("budget", {"budget": 3 * 64 * 256 * 4}), ("recursive", {"k": 2}),
                                         ("recursive", {"k": 3}), ("drop_cheap", {})])
def test_other_plans_bitwise(slm, strategy, kw):
    n, B, d = 20, 64, 256
    inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=9)
    ref_loss, ref, _ = _run(slm, n, B, d, "bf16", "none", inp)
    p, g, x0, y = _dev(inp, "bf16")
    model = slm.ChainModel(p, g, dtype="bf16", batch=B)
    plan = slm.Plan(slm.Graph.chain(n, B, d), strategy, **kw)
    loss = model.step(plan, x0, y)
    torch.cuda.synchronize()
    assert float(loss.item()) == ref_loss
    for k in ref:
        assert np.array_equal(g[k].float().cpu().numpy().astype(np.float64), ref[k]), k


def test_sgd_training_reduces_loss(slm):
    """End to end: the checkpointed step's gradients train the chain (plain SGD on the device
    parameters; the same batch) -- the loss falls monotonically over a few steps."""
    n, B, d = 16, 64, 256
    inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=31)
    p, g, x0, y = _dev(inp, "bf16")
    model = slm.ChainModel(p, g, dtype="bf16", batch=B)
    plan = slm.Plan(slm.Graph.chain(n, B, d), "sqrt")
    losses = []
    for _ in range(6):
        losses.append(float(model.step(plan, x0, y).item()))
        with torch.no_grad():
            W32 = p["W"].float() - 0.5 * g["W"].float()
            p["W"].copy_(W32.to(torch.bfloat16))
            for k in ("b", "gamma", "beta"):
                p[k].sub_(0.5 * g[k])
    assert all(b < a for a, b in zip(losses, losses[1:])), losses


@pytest.mark.parametrize("n,B,d,opt", [(40, 64, 256, {}), (100, 128, 512, {}), (40, 256, 512, {}),
                                       (33, 128, 384, {}), (40, 256, 2048, {}), (40, 256, 512, dict(pdl=0))])
def test_overlapped_recompute_bitwise(slm, n, B, d, opt):
    """Option overlap (reading A24): with a SLM_ALLOC_MIRROR_PARITY plan each segment's recompute
    runs on its own stream, concurrent with the backward of the next segment.  The step must
    really overlap (last_overlap), and give the non-checkpointed step's loss and gradients bit
    for bit, repeatedly (a race on a recycled pool slot would show up as a mismatch); plans
    without the flag fall back to the sequential schedule with the same bits."""
    inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=7)
    ref_loss, ref, _ = _run(slm, n, B, d, "bf16", "none", inp, **opt)
    par = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_MIRROR_PARITY
    p, g, x0, y = _dev(inp, "bf16")
    model = slm.ChainModel(p, g, dtype="bf16", batch=B, **opt)
    for strategy in ("sqrt", "search"):
        plan = slm.Plan(slm.Graph.chain(n, B, d), strategy, alloc_flags=par)
        for it in range(4):
            loss = model.step(plan, x0, y)
            torch.cuda.synchronize()
            assert model.get_option("last_overlap") == 1, strategy
            assert float(loss.item()) == ref_loss, (strategy, it)
            for k in ref:
                assert np.array_equal(g[k].float().cpu().numpy().astype(np.float64), ref[k]), (strategy, it, k)
    plan = slm.Plan(slm.Graph.chain(n, B, d), "sqrt")
    loss = model.step(plan, x0, y)
    torch.cuda.synchronize()
    assert model.get_option("last_overlap") == 0
    assert float(loss.item()) == ref_loss


@pytest.mark.parametrize("strategy,kw", [("recursive", dict(k=1)), ("recursive", dict(k=2)), ("budget", dict(budget=0)),
                                         ("sqrt", {})])
def test_overlap_soundness_check_other_plans(slm, strategy, kw):
    """The executor re-checks A24's disjointness on every plan: recursive / budget plans built
    with SLM_ALLOC_MIRROR_PARITY run overlapped only when the check holds, sequentially
    otherwise, and give the non-checkpointed bits either way (n = 2: a single mirror run, no
    overlap possible)."""
    for n in (2, 33):
        B, d = 64, 256
        inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=17)
        ref_loss, ref, _ = _run(slm, n, B, d, "bf16", "none", inp)
        p, g, x0, y = _dev(inp, "bf16")
        model = slm.ChainModel(p, g, dtype="bf16", batch=B)
        par = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_MIRROR_PARITY
        plan = slm.Plan(slm.Graph.chain(n, B, d), strategy, alloc_flags=par, **kw)
        for _ in range(2):
            loss = model.step(plan, x0, y)
            torch.cuda.synchronize()
            assert float(loss.item()) == ref_loss, (n, strategy)
            for k in ref:
                assert np.array_equal(g[k].float().cpu().numpy().astype(np.float64), ref[k]), (n, strategy, k)
        if n == 2:
            assert model.get_option("last_overlap") == 0


def test_poison_turns_a_clobbering_plan_into_nan(slm):
    """Debug option poison: every pool tag is filled with NaN once its value is
    dead.  On an intact plan nothing changes (the step's bits equal the plain run's); on a plan
    corrupted through slm_debug_plan_alias (the first gradient node written into x_1's slot, which
    Block_1's backward still reads) the silent corruption becomes NaN."""
    n, B, d = 6, 64, 256
    inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=2)
    ref_loss, ref, _ = _run(slm, n, B, d, "bf16", "none", inp)
    for strategy in ("none", "sqrt"):
        loss_p, gp, _ = _run(slm, n, B, d, "bf16", strategy, inp, poison=1)
        assert loss_p == ref_loss, strategy
        for k in ref:
            assert np.array_equal(gp[k], ref[k]), (strategy, k)

    def corrupted(poison):
        p, g, x0, y = _dev(inp, "bf16")
        model = slm.ChainModel(p, g, dtype="bf16", batch=B, poison=poison)
        plan = slm.Plan(slm.Graph.chain(n, B, d), "none")
        nodes = plan.nodes
        x1 = next(i for i, nd in enumerate(nodes) if nd["kind"] == 0 and nd["op"] == slm.OP["block"] and nd["orig"] == 1)
        gn = next(i for i, nd in enumerate(nodes) if nd["kind"] == 2 and nd["op"] == slm.OP["block"] and nd["orig"] == n)
        slm.check(slm.lib.slm_debug_plan_alias(plan._h, gn, x1), "slm_debug_plan_alias")
        loss = model.step(plan, x0, y)
        torch.cuda.synchronize()
        return float(loss.item()), {k: v.float().cpu().numpy() for k, v in g.items()}

    _, g0 = corrupted(0)
    assert all(np.isfinite(g0[k]).all() for k in g0)                       # silent ...
    assert not all(np.array_equal(g0[k], ref[k].astype(np.float32)) for k in g0)   # ... but wrong
    _, g1 = corrupted(1)
    assert np.isnan(g1["W"][0]).any() and np.isnan(g1["gamma"][0]).any()   # poisoned: NaN reaches layer 0
