"""GPU op-granularity executor: the pre-activation
network with BN, ReLU, FC and Add as separate nodes, executed on the device node by node through
the plan's tags -- element-wise parity with the op-graph oracle (oracle.opgraph, bf16 mode), the
checkpointed plans (sqrt, drop bn-relu, App. A search) bit-identical to the plain one, and the
drop-bn-relu plan's memory below the sharing plan's."""
import numpy as np
import pytest

import synth
from oracle import graph as OGR
from oracle import opgraph as OG
from _util import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slm():
    import paper_1604_06174_b200 as m
    return m


def _setup(slm, depths, widths, B, seed=5):
    import torch
    nodes = slm.OpsModel.preact_nodes(depths, widths, B)
    inp = synth.opgraph_inputs(nodes, B, seed=seed)
    dev = torch.device("cuda", 0)
    params, grads = {}, {}
    for v, pv in inp["params"].items():
        params[v] = {k: torch.tensor(a, device=dev, dtype=torch.bfloat16 if k == "W" else torch.float32)
                     for k, a in pv.items()}
        grads[v] = {k: torch.zeros_like(t) for k, t in params[v].items()}
    x = torch.tensor(inp["x0"], device=dev)
    y = torch.tensor(inp["labels"], device=dev)
    return nodes, inp, params, grads, x, y


def _run(slm, nodes, params, grads, x, y, B, strategy, af=3):
    import torch
    graph = slm.Graph.from_nodes(nodes, [len(nodes) - 1])
    model = slm.OpsModel(graph, params, grads, B)
    plan = slm.Plan(graph, strategy, alloc_flags=af)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        loss = model.step(plan, x, y, stream=s)
        loss = model.step(plan, x, y, stream=s)   # CUDA-graph replay
    torch.cuda.synchronize()
    g = {(v, k): t.float().cpu().numpy().astype(np.float64) for v, gv in grads.items() for k, t in gv.items()}
    return float(loss.item()), g, plan, model


@pytest.mark.parametrize("depths,widths,B", [([2, 2], [128, 256], 64), ([3], [256], 128)])
def test_ops_vs_oracle(slm, depths, widths, B):
    nodes, inp, params, grads, x, y = _setup(slm, depths, widths, B)
    loss, g, _, _ = _run(slm, nodes, params, grads, x, y, B, "sqrt")
    og = OGR.preact_resnet_graph(depths, [B * w * 4 for w in widths])
    P = OG.OpParams({v: p["W"] for v, p in inp["params"].items() if "W" in p},
                    {v: p["b"] for v, p in inp["params"].items() if "b" in p},
                    {v: p["gamma"] for v, p in inp["params"].items() if "gamma" in p},
                    {v: p["beta"] for v, p in inp["params"].items() if "beta" in p})
    ol, ogr = OG.step_plain(og, P, inp["x0"], inp["labels"], "bf16")
    assert abs(loss - ol) <= 2e-2 * abs(ol), (loss, ol)
    for (v, k), a in g.items():
        assert_close(a, ogr[k][v], 2e-2, f"node {v} d{k}")


def test_ops_plans_bitwise_and_drop_saves_memory(slm):
    depths, widths, B = [4, 4], [128, 256], 64
    nodes, inp, params, grads, x, y = _setup(slm, depths, widths, B, seed=9)
    ref_loss, ref, share, _ = _run(slm, nodes, params, grads, x, y, B, "none")
    runs = {s: _run(slm, nodes, params, grads, x, y, B, s) for s in ("sqrt", "drop_cheap", "search")}
    for s, (loss, g, plan, _) in runs.items():
        assert loss == ref_loss, s
        for k in ref:
            assert np.array_equal(g[k], ref[k]), (s, k)
    drop = runs["drop_cheap"][2]
    assert drop.extra_forward > 0          # BN and ReLU outputs are re-computed
    assert drop.exact_peak < share.exact_peak


def test_ops_launch_count(slm):
    depths, widths, B = [1], [128], 64
    nodes, inp, params, grads, x, y = _setup(slm, depths, widths, B)
    graph = slm.Graph.from_nodes(nodes, [len(nodes) - 1])
    model = slm.OpsModel(graph, params, grads, B)
    plan = slm.Plan(graph, "none", alloc_flags=3)
    # forward: BN, ReLU, FC (operand pack + GEMM), Add, CE (rows + reduce) = 7; backward: CE 1,
    # Add 1 (its upstream is the loss gradient, one whole slice), FC 6 (its upstream is the second
    # slice of Add's gradient -> one gather; dy and x packs, db column sums, dW and dX GEMMs),
    # ReLU 1, BN 1 (the Input gets no gradient)
    n = model.launches(plan)
    assert n == 7 + 1 + 1 + 6 + 1 + 1, n
