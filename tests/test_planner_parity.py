"""C++ planner (libslm) vs the independent Python oracle: plans, checkpoint sets, V', tags
and pool offsets must match byte for byte (north_star; SURVEY 8(c) parity contract)."""
import random

import pytest

import paper_1604_06174_b200 as slm
from oracle import graph as G
from oracle import planner as P

KIND = {"fwd": 0, "mirror": 1, "grad": 2}


def _cxx_graph(g):
    if g.kind == "chain" and "batch" in g.dims:
        return slm.Graph.chain(g.dims["n_layers"], g.dims["batch"], g.dims["width"])
    if g.kind == "lstm":
        d = g.dims
        return slm.Graph.lstm(d["n_layers"], d["steps"], d["batch"], d["hidden"], d["n_in"])
    return slm.Graph.from_nodes([(nd.op, nd.preds, nd.out_bytes, nd.flags) for nd in g.nodes], g.outputs)


def assert_same_plan(g, strategy, **kw):
    po = P.plan(g, strategy, **kw)
    cg = _cxx_graph(g)
    pc = slm.Plan(cg, strategy, **kw)
    assert pc.m == po.m
    assert pc.order == po.gg.order
    nodes = pc.nodes
    assert len(nodes) == len(po.gg.nodes)
    for a, b in zip(nodes, po.gg.nodes):
        assert (a["kind"], a["op"], a["orig"], a["level"], a["out_bytes"], a["inplace_slot"], a["preds"]) == \
               (KIND[b.kind], b.op, b.orig, b.level, b.out_bytes, b.inplace_slot, b.preds)
    node_tag, tsize, toff = pc.tags
    for v in po.gg.order:
        assert node_tag[v] == po.alloc.tag_of[v]
    assert tsize == po.alloc.tag_size
    assert toff == po.alloc.offsets
    assert pc.exact_peak == po.alloc.exact_peak
    assert pc.pool_bytes == po.alloc.pool_bytes
    assert pc.extra_forward == po.extra_forward
    assert (pc.x, pc.y, pc.budget) == (po.x, po.y, po.B)
    assert pc.trace == [tuple(r) for r in po.trace]
    return pc, po


@pytest.mark.parametrize("strategy,kw", [("none", {}), ("sqrt", {}), ("search", {}),
                                         ("budget", {"budget": 5 * 2048}),
                                         ("recursive", {"k": 1}), ("recursive", {"k": 3}),
                                         ("drop_cheap", {})])
def test_c1_chain(strategy, kw):
    assert_same_plan(G.chain_graph(16, 8, 64), P.__dict__["S_" + strategy.upper()], **kw)


@pytest.mark.parametrize("strategy", [P.S_NONE, P.S_SQRT, P.S_SEARCH])
def test_c2_chain(strategy):
    pc, po = assert_same_plan(G.chain_graph(1024, 256, 2048), strategy)
    if strategy == P.S_SQRT:
        assert pc.exact_peak == 64 * 256 * 2048 * 4 + 4


@pytest.mark.parametrize("strategy,kw", [(P.S_SEARCH, {}), (P.S_RECURSIVE, {"k": 1}),
                                         (P.S_RECURSIVE, {"k": 2}), (P.S_SQRT, {}),
                                         (P.S_BUDGET, {"budget": 40 * 2 ** 21})])
def test_c4_chain_1000(strategy, kw):
    assert_same_plan(G.chain_graph(1000, 256, 2048), strategy, **kw)


def test_c4_resnet_shaped_budget_sweep():
    # ResNet-shaped 1000-layer chain (4 stages x 250 layers, bottleneck output bytes at batch 32)
    sizes = [102760448] * 250 + [51380224] * 250 + [25690112] * 250 + [12845056] * 250
    nodes = [G.Node(G.INPUT, [], sizes[0])]
    for i, s in enumerate(sizes):
        nodes.append(G.Node(G.FC, [i], s))
    nodes.append(G.Node(G.SOFTMAX_CE, [len(sizes)], 4, G.F_NOT_CANDIDATE))
    g = G.Graph(nodes, [len(nodes) - 1])
    assert_same_plan(g, P.S_SEARCH)
    tot = sum(sizes)
    for i in range(0, 64, 9):
        B = int(max(sizes) * (tot / max(sizes)) ** (i / 63))
        assert_same_plan(g, P.S_BUDGET, budget=B)


def test_lstm_graph_plan():
    g = G.lstm_graph(2, 24, 4, 8, 3)
    m = [0] * len(g)
    t = -1
    for v, nd in enumerate(g.nodes):
        if nd.op == G.INPUT:
            t += 1
        if nd.op in (G.LSTM_GATES, G.LSTM_CELL) and not (nd.op == G.LSTM_CELL and t % 5 == 4):
            m[v] = 1
    assert_same_plan(g, P.S_EXPLICIT, m=m)
    assert_same_plan(g, P.S_SEARCH)
    assert_same_plan(g, P.S_NONE)
    grouped = P.A_INPLACE | P.A_SHARING | P.A_GROUPED
    assert_same_plan(g, P.S_EXPLICIT, m=m, alloc_flags=grouped)
    assert_same_plan(g, P.S_EXPLICIT, m=m, alloc_flags=grouped | P.A_GROUP_MIRRORS)
    assert_same_plan(G.chain_graph(40, 8, 64), P.S_SQRT, alloc_flags=P.A_INPLACE | P.A_SHARING | P.A_GROUP_MIRRORS)
    par = P.A_INPLACE | P.A_SHARING | P.A_MIRROR_PARITY
    for strat, kw in ((P.S_SQRT, {}), (P.S_SEARCH, {}), (P.S_RECURSIVE, dict(k=1)), (P.S_RECURSIVE, dict(k=2))):
        assert_same_plan(G.chain_graph(40, 8, 64), strat, alloc_flags=par, **kw)
    assert_same_plan(g, P.S_SQRT, alloc_flags=grouped | P.A_MIRROR_PARITY)
    rg = G.preact_resnet_graph([3, 5, 4, 2], [4096, 2048, 1024, 512])   # op-granularity ResNet (8(f) f1)
    for strat, fl in ((P.S_NONE, 0), (P.S_NONE, P.A_INPLACE), (P.S_NONE, 3), (P.S_DROP_CHEAP, 3), (P.S_SEARCH, 3),
                      (P.S_SQRT, 3), (P.S_SQRT, 3 | P.A_MIRROR_PARITY)):
        assert_same_plan(rg, strat, alloc_flags=fl)
    cg, _ = G.preact_resnet_conv_graph(16, 16, [(128, 3), (256, 3), (512, 2)], 128)   # conv ResNet (8(f) f4)
    for strat, fl in ((P.S_NONE, 0), (P.S_NONE, 3), (P.S_DROP_CHEAP, 3), (P.S_SEARCH, 3), (P.S_SQRT, 3),
                      (P.S_SQRT, 3 | P.A_MIRROR_PARITY)):
        assert_same_plan(cg, strat, alloc_flags=fl)
    assert_same_plan(g, P.S_SEARCH, alloc_flags=grouped)
    assert_same_plan(g, P.S_SQRT, alloc_flags=grouped)
    assert_same_plan(G.lstm_graph(4, 64, 64, 1024, 50), P.S_EXPLICIT,
                     m=[1 if (nd.op in (G.LSTM_GATES, G.LSTM_CELL)) else 0 for nd in G.lstm_graph(4, 64, 64, 1024, 50).nodes],
                     alloc_flags=grouped)


@pytest.mark.parametrize("L,T,seg", [(2, 24, 5), (4, 64, 8), (1, 7, 1), (3, 10, 64)])
def test_lstm_segment_mirrors(L, T, seg):
    from oracle.lstm import time_segment_plan
    dg = slm.Graph.lstm(L, T, 64, 128, 50)
    assert dg.lstm_segment_mirrors(seg) == time_segment_plan(G.lstm_graph(L, T, 64, 128, 50), seg)
    with pytest.raises(slm.SlmError if hasattr(slm, "SlmError") else Exception):
        slm.Graph.chain(4, 8, 64).lstm_segment_mirrors(seg)


def _random_dag(rnd, n):
    nodes = [G.Node(G.INPUT, [], rnd.randint(1, 5) * 64)]
    for i in range(1, n):
        if rnd.random() < 0.1:
            nodes.append(G.Node(G.INPUT, [], rnd.randint(1, 5) * 64))
            continue
        op = rnd.choice([G.FC, G.SIGMOID, G.RELU, G.BN, G.IDENTITY, G.ADD, G.MUL, G.BLOCK])
        preds = [rnd.randrange(0, i) for _ in range(G.OPS[op].arity_min)]
        size = rnd.randint(1, 5) * 64 + rnd.choice([0, 0, 7])
        if G.OPS[op].fwd_inplace == 0 and rnd.random() < 0.7:
            size = nodes[preds[0]].out_bytes
        flags = G.F_NOT_CANDIDATE if rnd.random() < 0.1 else 0
        nodes.append(G.Node(op, preds, size, flags))
    nodes.append(G.Node(G.SOFTMAX_CE, [n - 1], 4, G.F_NOT_CANDIDATE))
    return G.Graph(nodes, [len(nodes) - 1])


def test_random_dags():
    rnd = random.Random(1234)
    for it in range(300):
        g = _random_dag(rnd, rnd.randint(2, 60))
        s = rnd.choice([P.S_NONE, P.S_SQRT, P.S_BUDGET, P.S_SEARCH, P.S_DROP_CHEAP, P.S_EXPLICIT])
        kw = {}
        if s == P.S_BUDGET:
            kw["budget"] = rnd.randint(0, 3000)
        if s == P.S_EXPLICIT:
            kw["m"] = [0 if nd.op == G.INPUT else rnd.randint(0, 3) for nd in g.nodes]
        flags = rnd.choice([3, 3, 1, 2, 0, 19])
        assert_same_plan(g, s, alloc_flags=flags, **kw)


def test_random_chains_all_strategies():
    rnd = random.Random(99)
    for it in range(60):
        n = rnd.randint(1, 300)
        g = G.chain_graph(n, rnd.choice([1, 8, 64]), rnd.choice([3, 64]))
        for s, kw in [(P.S_SQRT, {}), (P.S_SEARCH, {}), (P.S_RECURSIVE, {"k": rnd.randint(1, 4)}),
                      (P.S_BUDGET, {"budget": rnd.randint(0, 10 ** 6)})]:
            assert_same_plan(g, s, **kw)


def test_validate_and_errors_match():
    d = [(G.RELU, [0], 1, 0)]
    assert slm.Graph.validate(d, [0]) == [(G.CYCLE, 0)]
    assert slm.Graph.validate([(G.FC, [], 1, 0)], [0]) == [(G.ARITY, 0)]
    assert slm.Graph.validate([(G.INPUT, [], 1, 0), (G.RELU, [7], 1, 0)], [1]) == [(G.DANGLING, 1)]
    assert slm.Graph.validate([(G.INPUT, [], 0, 0)], [0]) == [(G.ZERO_SIZE, 0)]
    g = slm.Graph.chain(3, 1, 1)
    with pytest.raises(slm._lib.SlmError) as e:
        slm.Plan(g, "explicit", m=[1, 0, 0, 0, 0])
    assert e.value.code == -4
    dg = slm.Graph.from_nodes([(G.INPUT, [], 1, 0), (G.RELU, [0], 1, 0), (G.RELU, [0], 1, 0),
                               (G.ADD, [1, 2], 1, 0)], [3])
    with pytest.raises(slm._lib.SlmError) as e:
        slm.Plan(dg, "recursive", k=1)
    assert e.value.code == -5
    for n, k in [(1024, 1), (81, 2), (1, 3), (10 ** 12, 1)]:
        assert slm.recursion_estimate(n, k) == P.recursion_estimate(n, k)


def test_lstm_state_candidates_search():
    """Reading A25: slm_graph_mark_not_candidate(LSTM_GATES) leaves the cell
    states as Alg. 3's only split points on the LSTM grid; the C++ plan equals the oracle's on
    the same flags (byte for byte), and no gates node is ever kept (m = 0)."""
    import copy
    g = G.lstm_graph(2, 24, 4, 8, 3)
    go = copy.deepcopy(g)
    for nd in go.nodes:
        if nd.op == G.LSTM_GATES:
            nd.flags |= G.F_NOT_CANDIDATE
    cg = slm.Graph.lstm(2, 24, 4, 8, 3)
    assert cg.mark_not_candidate(slm.OP["lstm_gates"]) == 48
    assert cg.mark_not_candidate(slm.OP["lstm_gates"]) == 0
    for strat, kw in ((P.S_SEARCH, {}), (P.S_BUDGET, dict(budget=4 * 8 * 4 * 6))):
        for fl in (3, 7, 23):
            po = P.plan(go, strat, alloc_flags=fl, **kw)
            pc = slm.Plan(cg, {P.S_SEARCH: "search", P.S_BUDGET: "budget"}[strat], alloc_flags=fl, **kw)
            assert po.m == pc.m and po.alloc.exact_peak == pc.exact_peak and po.alloc.offsets == pc.tags[2]
            assert all(po.m[v] >= 1 for v, nd in enumerate(go.nodes) if nd.op == G.LSTM_GATES)
    with pytest.raises(RuntimeError):
        cg.mark_not_candidate(999)


def test_binding_conv_builder_matches_oracle():
    """The binding's node list for the conv ResNet is oracle.graph's graph."""
    for B, hw, stages in ((64, 8, [(128, 1), (256, 2)]), (16, 16, [(128, 3), (256, 3), (512, 2)])):
        nodes, shapes = slm.OpsModel.preact_conv_nodes(B, hw, stages, 128)
        og, osh = G.preact_resnet_conv_graph(B, hw, stages, 128)
        assert [(nd.op, list(nd.preds), nd.out_bytes, nd.flags) for nd in og.nodes] == \
            [(o, list(p), ob, f) for o, p, ob, f in nodes]
        assert [tuple(s) for s in osh] == [tuple(s) for s in shapes]
