"""Computation graph G=(V, pred) and operator metadata (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md:125-131 — "A computation graph consists of operational nodes and edges that
represent the dependencies between the operations."  PAPER.md:261 — Alg. 2 input
"G=(V, pred) ... pred[v] gives the predecessors array of node v".
PAPER.md:174-186 — "Declare the dependency requirements of gradient operators in
minimum manner": the per-op backward dependency table below (reading A6).
PAPER.md:142, 156-160 — in-place operation (output written into an input's buffer).

Node ids are dense 0..N-1.  Each node has exactly one output of ``out_bytes`` bytes.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

# ---- op kinds (numbering is part of the C ABI, include/slm.h mirrors it independently) ----
INPUT, BLOCK, SOFTMAX_CE, FC, SIGMOID, RELU, BN, ADD, MUL, IDENTITY = range(10)
LSTM_GATES, LSTM_CELL, HEAD_CE, SUM = 10, 11, 12, 13
CONV, POOL = 14, 15   # convolution (NHWC, "same" padding) and global average pool

OP_NAMES = {
    INPUT: "Input", BLOCK: "Block", SOFTMAX_CE: "SoftmaxCE", FC: "FullyConnected",
    SIGMOID: "Sigmoid", RELU: "ReLU", BN: "BatchNormLite", ADD: "Add", MUL: "ElemMul",
    IDENTITY: "Identity", LSTM_GATES: "LstmGates", LSTM_CELL: "LstmCell",
    HEAD_CE: "HeadCE", SUM: "Sum", CONV: "Convolution", POOL: "GlobalAvgPool",
}


@dataclass(frozen=True)
class OpMeta:
    """Per-op metadata (reading A6/A18 in DESIGN.md).

    arity_min/max   number of predecessors.
    fwd_inplace     predecessor slot whose buffer the forward may overwrite, -1 none.
    grad_needs_out  the backward reads the op's own output (e.g. sigmoid).
    grad_needs_in   bitmask over predecessor slots the backward reads.
    grad_inplace    which input of the gradient node the backward may overwrite:
                    G_NONE, G_SUCC0 (the first successor gradient), G_OUT (the op's own
                    output a[v], as the sigmoid of Fig. 1) or G_IN0 (the
                    first declared input dependency).  Resolved to a slot by Alg. 2.
    low_cost        "low cost operations" of Sec. 4.2.
    """
    arity_min: int
    arity_max: int
    fwd_inplace: int
    grad_needs_out: bool
    grad_needs_in: int
    grad_inplace: int
    low_cost: bool


ANY = 1 << 30
G_NONE, G_SUCC0, G_OUT, G_IN0 = -1, 0, 1, 2
OPS = {
    #                    amin amax fwd_ip out   in_mask g_ip low
    INPUT:      OpMeta(0, 0, -1, False, 0b00, G_NONE, False),
    # residual pre-activation block x + ReLU(BN(x)) W^T + b (A10); backward needs its input only
    BLOCK:      OpMeta(1, 1, 0, False, 0b01, G_SUCC0, False),
    # mean softmax cross-entropy; backward needs its input (and the labels, which are not a node)
    SOFTMAX_CE: OpMeta(1, 1, -1, False, 0b01, G_IN0, False),
    FC:         OpMeta(1, 1, -1, False, 0b01, G_NONE, False),   # FC <- input
    SIGMOID:    OpMeta(1, 1, 0, True, 0b00, G_OUT, True),       # sigmoid <- output
    RELU:       OpMeta(1, 1, 0, True, 0b00, G_OUT, True),
    BN:         OpMeta(1, 1, 0, False, 0b01, G_SUCC0, True),
    ADD:        OpMeta(2, 2, 0, False, 0b00, G_NONE, False),
    MUL:        OpMeta(2, 2, 0, False, 0b11, G_NONE, False),
    IDENTITY:   OpMeta(1, 1, 0, False, 0b00, G_SUCC0, True),
    # LSTM (A13): gates G_t = act(x W_ih^T + h_{t-1} W_hh^T + b); preds (x_or_lower_S, S_{t-1})
    LSTM_GATES: OpMeta(1, 2, -1, True, 0b11, G_NONE, False),
    # cell S_t = (h_t, c_t) from (G_t, S_{t-1}); backward needs G_t and S_{t-1} (A6)
    LSTM_CELL:  OpMeta(1, 2, -1, False, 0b11, G_NONE, False),
    HEAD_CE:    OpMeta(1, 1, -1, False, 0b01, G_NONE, False),
    SUM:        OpMeta(1, ANY, -1, False, 0b00, G_NONE, False),
    # convolution y = conv(x, W) + b: like FC, the backward reads its input only
    CONV:       OpMeta(1, 1, -1, False, 0b01, G_NONE, False),
    # global average pool over the spatial positions: the backward needs only the shapes
    POOL:       OpMeta(1, 1, -1, False, 0b00, G_NONE, False),
}

# node flags (mirrored in include/slm.h)
F_NOT_CANDIDATE = 1  # exclude from Alg. 3's candidate set C; default C = non-Input
F_PIN = 2            # never recycle this node's tag
F_REQUEST_GRAD = 4   # (Input nodes) the gradient flowing into this input is retained


@dataclass
class Node:
    op: int
    preds: list
    out_bytes: int
    flags: int = 0
    group: int = 0     # allocation group (A_GROUPED, reading A22): the LSTM layer


@dataclass
class Graph:
    nodes: list
    outputs: list
    # informational (set by the builders)
    kind: str = "dag"
    dims: dict = field(default_factory=dict)

    def __len__(self):
        return len(self.nodes)


# ---------------------------------------------------------------- validation
CYCLE, ARITY, DANGLING, ZERO_SIZE, BAD_OUTPUT, BAD_OP = range(1, 7)


def validate(g: Graph):
    """Return a list of (code, node) diagnostics; empty iff valid (artifact plumbing)."""
    diags = []
    n = len(g.nodes)
    for i, nd in enumerate(g.nodes):
        if nd.op not in OPS:
            diags.append((BAD_OP, i))
            continue
        meta = OPS[nd.op]
        if not (meta.arity_min <= len(nd.preds) <= meta.arity_max):
            diags.append((ARITY, i))
        for p in nd.preds:
            if not (0 <= p < n):
                diags.append((DANGLING, i))
                break
        if nd.out_bytes <= 0:
            diags.append((ZERO_SIZE, i))
    if not g.outputs:
        diags.append((BAD_OUTPUT, -1))
    for o in g.outputs:
        if not (0 <= o < n):
            diags.append((BAD_OUTPUT, o))
    if not any(c == DANGLING for c, _ in diags):
        order = _kahn(g, range(n), lambda v: g.nodes[v].preds)
        if len(order) != n:
            placed = set(order)
            for i in range(n):
                if i not in placed:
                    diags.append((CYCLE, i))
    return diags


def _kahn(g, vertices, preds_of):
    """Kahn's algorithm, among ready vertices the lowest id first (reading: SPEC S:64)."""
    vs = list(vertices)
    vset = set(vs)
    indeg = {v: 0 for v in vs}
    succ = {v: [] for v in vs}
    for v in vs:
        for p in preds_of(v):
            if p in vset:
                indeg[v] += 1
                succ[p].append(v)
    heap = [v for v in vs if indeg[v] == 0]
    heapq.heapify(heap)
    out = []
    while heap:
        v = heapq.heappop(heap)
        out.append(v)
        for s in succ[v]:
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(heap, s)
    return out


def topo_order(g: Graph):
    """topological-order(V) of Alg. 2; lowest id first among ready nodes."""
    order = _kahn(g, range(len(g.nodes)), lambda v: g.nodes[v].preds)
    if len(order) != len(g.nodes):
        raise ValueError("CyclicGraph")
    return order


def successors(g: Graph):
    succ = [[] for _ in g.nodes]
    for v, nd in enumerate(g.nodes):
        for p in nd.preds:
            if v not in succ[p]:
                succ[p].append(v)
    for s in succ:
        s.sort()
    return succ


# ---------------------------------------------------------------- builders
def chain_graph(n_layers: int, batch: int, width: int, elem_bytes: int = 4) -> Graph:
    """Residual chain X_0 -> Block_0 -> ... -> Block_{n-1} -> SoftmaxCE.

    Node 0 = Input X_0, node l+1 = Block_l (output X_{l+1}), node n+1 = SoftmaxCE (scalar
    fp32 loss, 4 bytes).  Every X is stored fp32 (reading A11), so u = B*d*4 bytes.
    """
    u = batch * width * elem_bytes
    nodes = [Node(INPUT, [], u)]
    for l in range(n_layers):
        nodes.append(Node(BLOCK, [l], u))
    # the loss is pinned (a graph output) and never a split point
    nodes.append(Node(SOFTMAX_CE, [n_layers], 4, F_NOT_CANDIDATE))
    return Graph(nodes, [n_layers + 1], kind="chain",
                 dims=dict(n_layers=n_layers, batch=batch, width=width))


def preact_resnet_graph(depths, sizes) -> Graph:
    """Op-granularity pre-activation residual network for the paper's strategy comparison
    (Sec. 5.1 / Fig. 5): stage s has depths[s] layers whose
    feature maps are sizes[s] bytes; a layer ("conv-bn-relu counted as one layer") is
    BN(x) -> ReLU -> FC (the conv / GEMM stand-in) -> Add(x, .) = the next x.  Node 0 = Input
    (sizes[0]); the last x feeds a SoftmaxCE (4-byte loss).  Stage transitions are a plain FC
    to the next size (a projection)."""
    nodes = [Node(INPUT, [], sizes[0])]
    x = 0
    for st, (dep, sz) in enumerate(zip(depths, sizes)):
        if nodes[x].out_bytes != sz:
            nodes.append(Node(FC, [x], sz))
            x = len(nodes) - 1
        for _ in range(dep):
            nodes.append(Node(BN, [x], sz))
            nodes.append(Node(RELU, [len(nodes) - 1], sz))
            nodes.append(Node(FC, [len(nodes) - 1], sz))
            nodes.append(Node(ADD, [x, len(nodes) - 1], sz))
            x = len(nodes) - 1
    nodes.append(Node(SOFTMAX_CE, [x], 4, F_NOT_CANDIDATE))
    return Graph(nodes, [len(nodes) - 1], kind="dag", dims=dict(depths=list(depths)))


def preact_resnet_conv_graph(batch, hw, stages, classes):
    """Convolutional pre-activation ResNet (the network of the
    paper's Fig. 5/6 experiments at synthetic size).  Values are NHWC fp32, stored as
    [batch*H*W][C] rows; ``shapes[v] = (H, W, C, k, s)`` (k, s: kernel and stride of a CONV node,
    0 otherwise).  The Input is the stem output [batch, hw, hw, C_0].  Stage i (C_i, depth_i) has
    depth_i basic pre-activation blocks (He et al. 2016 "identity mappings"):
        r = ReLU(BN(x));  y = Conv3x3(ReLU(BN(Conv3x3_s(r)))) ;  x' = Add(y, x)
    where the first block of every stage after the first has stride 2 and a projection shortcut
    Conv1x1_s2(r) in place of x (the stage transitions of P:437-441).  Head: ReLU(BN(x)) ->
    GlobalAvgPool -> FC(classes) -> SoftmaxCE (4-byte loss)."""
    c0 = stages[0][0]
    nodes = [Node(INPUT, [], batch * hw * hw * c0 * 4)]
    shapes = [(hw, hw, c0, 0, 0)]

    def add(op, preds, H, W, C, k=0, s=0, flags=0):
        nodes.append(Node(op, list(preds), (batch * H * W * C * 4) if op != SOFTMAX_CE else 4, flags))
        shapes.append((H, W, C, k, s))
        return len(nodes) - 1

    x, H = 0, hw
    for i, (C, depth) in enumerate(stages):
        for j in range(depth):
            s = 2 if (i > 0 and j == 0) else 1
            Cin = shapes[x][2]
            Ho = (H - 1) // s + 1
            bn = add(BN, [x], H, H, Cin)
            r = add(RELU, [bn], H, H, Cin)
            c1 = add(CONV, [r], Ho, Ho, C, 3, s)
            bn2 = add(BN, [c1], Ho, Ho, C)
            r2 = add(RELU, [bn2], Ho, Ho, C)
            c2 = add(CONV, [r2], Ho, Ho, C, 3, 1)
            short = add(CONV, [r], Ho, Ho, C, 1, s) if (s != 1 or Cin != C) else x
            x = add(ADD, [c2, short], Ho, Ho, C)
            H = Ho
    C = shapes[x][2]
    bn = add(BN, [x], H, H, C)
    r = add(RELU, [bn], H, H, C)
    gp = add(POOL, [r], 1, 1, C)
    fc = add(FC, [gp], 1, 1, classes)
    add(SOFTMAX_CE, [fc], 1, 1, 1, flags=F_NOT_CANDIDATE)
    g = Graph(nodes, [len(nodes) - 1], kind="dag",
              dims=dict(batch=batch, hw=hw, stages=[list(t) for t in stages], classes=classes))
    return g, shapes


def unit_chain(n: int, unit: int = 1) -> Graph:
    """n Block nodes of size ``unit`` after an Input of size ``unit`` — no loss node.

    Used for the planner pins of SPEC S:264-266 (the 9-node unit chain = Input + 8 blocks,
    the output is the last block)."""
    nodes = [Node(INPUT, [], unit)]
    for l in range(n):
        nodes.append(Node(BLOCK, [l], unit))
    return Graph(nodes, [n], kind="chain", dims=dict(n_layers=n))


def lstm_graph(n_layers: int, steps: int, batch: int, hidden: int, n_in: int,
               elem_bytes: int = 4) -> Graph:
    """Unrolled LSTM (reading A13), time-major ids.

    For each t: Input X_t, then for l = 0..L-1: G^l_t (gates, B*4H) and S^l_t (h and c,
    B*2H), then H_t (per-step head CE, scalar).  Final node: Sum of all H_t (the loss).
    G^l_t preds = [X_t or S^{l-1}_t] + [S^l_{t-1} if t>0]; S^l_t preds = [G^l_t] + [S^l_{t-1}].
    """
    nodes = []
    s_prev = [None] * n_layers
    heads = []
    for t in range(steps):
        x = len(nodes)
        nodes.append(Node(INPUT, [], batch * n_in * elem_bytes))
        below = x
        for l in range(n_layers):
            gid = len(nodes)
            preds = [below] + ([s_prev[l]] if s_prev[l] is not None else [])
            nodes.append(Node(LSTM_GATES, preds, batch * 4 * hidden * elem_bytes, group=l))
            sid = len(nodes)
            preds = [gid] + ([s_prev[l]] if s_prev[l] is not None else [])
            nodes.append(Node(LSTM_CELL, preds, batch * 2 * hidden * elem_bytes, group=l))
            s_prev[l] = sid
            below = sid
        heads.append(len(nodes))
        nodes.append(Node(HEAD_CE, [below], 4, F_NOT_CANDIDATE, group=n_layers))
    nodes.append(Node(SUM, heads, 4, F_NOT_CANDIDATE, group=n_layers))
    return Graph(nodes, [len(nodes) - 1], kind="lstm",
                 dims=dict(n_layers=n_layers, steps=steps, batch=batch, hidden=hidden,
                           n_in=n_in))
