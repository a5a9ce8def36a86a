"""fp64 unrolled multi-layer LSTM training step (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md:480-485: "a four layer LSTM with 1024 hidden states ... unrolled over time ... The
input of each timestamp is a continuous 50 dimension vector and the output is softmax over
5000 class."  Reading A13: PyTorch gate order (i, f, g, o), no peepholes,
h_0 = c_0 = 0, a softmax head at every step, loss = mean over (t, b).

Parameter layout (PyTorch's, at the true widths; the device path pads layer 0 in its binding):
  W[l]   [4H, Kin_l + H]  = [W_ih | W_hh], Kin_0 = the input width I, Kin_l = H for l > 0
  b[l]   [4H]             = b_ih + b_hh
  W_o    [C, H], b_o [C]  the per-step softmax head

Forward, per step t and layer l (x^0_t = input, x^l_t = h^{l-1}_t):
  pre = [x^l_t | h^l_{t-1}] W[l]^T + b[l];  i, f, o = sigmoid, g = tanh (blocks of H)
  c^l_t = f c^l_{t-1} + i g;   h^l_t = o tanh(c^l_t)
  loss += sum_b CE(h^{L-1}_t W_o^T + b_o, y_t[b]) / (T B)

Two executors, as for the chain:
  * step_plain   — ordinary back-propagation through time (the definition);
  * step_planned — interprets V' of a plan on oracle.graph.lstm_graph node by node through the
                   allocator's tags with the interference check.
bf16 mode rounds exactly the GEMM operands the device rounds: W, the [x | h] operand, the
head operand h, and the gradient operands (d_pre, dlogits).
"""
from __future__ import annotations

import numpy as np

from .chain import TagClobber, _q, bf16_round
from .graph import HEAD_CE, INPUT, LSTM_CELL, LSTM_GATES, SUM


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


class LstmParams:
    def __init__(self, W, b, W_o, b_o, n_in):
        self.W = [np.asarray(w, dtype=np.float64) for w in W]
        self.b = [np.asarray(v, dtype=np.float64) for v in b]
        self.W_o = np.asarray(W_o, dtype=np.float64)
        self.b_o = np.asarray(b_o, dtype=np.float64)
        self.n_in = n_in                       # the input width I (= Kin_0)

    @property
    def L(self):
        return len(self.W)

    @property
    def H(self):
        return self.W[0].shape[0] // 4

    def kin(self, l):
        return self.W[l].shape[1] - self.H


def as_input(x):
    return np.asarray(x, dtype=np.float64)


# ------------------------------------------------------------------ node functions
def gates_forward(xin, h_prev, P: LstmParams, l, mode):
    """G^l_t: gate activations [B, 4H] from the layer input and h_{t-1}."""
    H = P.H
    op = _q(np.concatenate([xin, h_prev], axis=1), mode)
    pre = op @ _q(P.W[l], mode).T + P.b[l]
    act = np.empty_like(pre)
    act[:, :2 * H] = sigmoid(pre[:, :2 * H])
    act[:, 2 * H:3 * H] = np.tanh(pre[:, 2 * H:3 * H])
    act[:, 3 * H:] = sigmoid(pre[:, 3 * H:])
    return act


def cell_forward(act, c_prev):
    """S^l_t: (h, c) from the gate activations and c_{t-1}; returned as [B, 2H] = [h | c]."""
    H = act.shape[1] // 4
    i, f, g, o = act[:, :H], act[:, H:2 * H], act[:, 2 * H:3 * H], act[:, 3 * H:]
    c = f * c_prev + i * g
    h = o * np.tanh(c)
    return np.concatenate([h, c], axis=1)


def head_forward(h, labels, P: LstmParams, scale, mode):
    """Per-step softmax head: returns (loss contribution, dlogits)."""
    logits = _q(h, mode) @ _q(P.W_o, mode).T + P.b_o
    mx = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - mx)
    s = e.sum(axis=1, keepdims=True)
    lse = np.log(s[:, 0]) + mx[:, 0]
    loss = float((lse - logits[np.arange(len(labels)), labels]).sum() * scale)
    p = e / s
    p[np.arange(len(labels)), labels] -= 1.0
    return loss, p * scale


def head_backward(h, labels, P, scale, mode):
    """dL/dh (from this step's head) and the head's parameter gradients."""
    _, dlog = head_forward(h, labels, P, scale, mode)
    dq = _q(dlog, mode)
    dh = dq @ _q(P.W_o, mode)
    return dh, dq.T @ _q(h, mode), dlog.sum(axis=0)


def cell_backward(dh, dc_in, act, c_prev):
    """Back through S: returns (d act [B,4H], dc_prev)."""
    H = act.shape[1] // 4
    i, f, g, o = act[:, :H], act[:, H:2 * H], act[:, 2 * H:3 * H], act[:, 3 * H:]
    c = f * c_prev + i * g
    tc = np.tanh(c)
    do = dh * tc
    dc = dc_in + dh * o * (1.0 - tc * tc)
    dact = np.concatenate([dc * g, dc * c_prev, dc * i, do], axis=1)
    return dact, dc * f


def gates_backward(dact, act, xin, h_prev, P, l, mode):
    """Back through G: returns (dx [B, Kin], dh_prev [B, H], dW [4H, Kin+H], db [4H])."""
    H = P.H
    dpre = np.empty_like(dact)
    dpre[:, :2 * H] = dact[:, :2 * H] * act[:, :2 * H] * (1.0 - act[:, :2 * H])
    dpre[:, 2 * H:3 * H] = dact[:, 2 * H:3 * H] * (1.0 - act[:, 2 * H:3 * H] ** 2)
    dpre[:, 3 * H:] = dact[:, 3 * H:] * act[:, 3 * H:] * (1.0 - act[:, 3 * H:])
    dq = _q(dpre, mode)
    dop = dq @ _q(P.W[l], mode)
    kin = P.kin(l)
    op = _q(np.concatenate([xin, h_prev], axis=1), mode)
    return dop[:, :kin], dop[:, kin:], dq.T @ op, dpre.sum(axis=0)


# ------------------------------------------------------------------ plain BPTT (definition)
def step_plain(P: LstmParams, x, labels, mode="f64"):
    """x [T, B, n_in], labels [T, B] -> (loss, grads dict)."""
    T, B = labels.shape
    L, H = P.L, P.H
    xs = as_input(x)
    scale = 1.0 / (T * B)
    h = [[np.zeros((B, H)) for _ in range(T + 1)] for _ in range(L)]   # h[l][t+1]
    c = [[np.zeros((B, H)) for _ in range(T + 1)] for _ in range(L)]
    acts = [[None] * T for _ in range(L)]
    loss = 0.0
    for t in range(T):
        xin = xs[t]
        for l in range(L):
            acts[l][t] = gates_forward(xin, h[l][t], P, l, mode)
            s = cell_forward(acts[l][t], c[l][t])
            h[l][t + 1], c[l][t + 1] = s[:, :H], s[:, H:]
            xin = h[l][t + 1]
        loss += head_forward(h[L - 1][t + 1], labels[t], P, scale, mode)[0]
    dW = [np.zeros_like(w) for w in P.W]
    db = [np.zeros_like(v) for v in P.b]
    dWo = np.zeros_like(P.W_o)
    dbo = np.zeros_like(P.b_o)
    dh_next = [np.zeros((B, H)) for _ in range(L)]   # dh flowing back from step t+1
    dc_next = [np.zeros((B, H)) for _ in range(L)]
    for t in reversed(range(T)):
        dh_top, gwo, gbo = head_backward(h[L - 1][t + 1], labels[t], P, scale, mode)
        dWo += gwo
        dbo += gbo
        dh_from_above = dh_top
        for l in reversed(range(L)):
            xin = xs[t] if l == 0 else h[l - 1][t + 1]
            dact, dc_prev = cell_backward(dh_from_above + dh_next[l], dc_next[l], acts[l][t], c[l][t])
            dx, dhp, gw, gb = gates_backward(dact, acts[l][t], xin, h[l][t], P, l, mode)
            dW[l] += gw
            db[l] += gb
            dh_next[l], dc_next[l] = dhp, dc_prev
            dh_from_above = dx
    return loss, dict(W=dW, b=db, W_o=dWo, b_o=dbo)


def _round_grads(g, mode):
    return g


# ------------------------------------------------------------------ V' interpreter
def step_planned(plan, P: LstmParams, x, labels, mode="f64"):
    """Execute V' of ``plan`` (oracle.planner.Plan on oracle.graph.lstm_graph) through its tags.

    Gradient node g[v] holds the gradient w.r.t. all of v's inputs, concatenated in pred
    order (reading A17); a node's output gradient is the sum of the matching slices of its
    successors' gradient nodes.  Weight gradients accumulate in place across time steps
    (PAPER.md:488-489), in the same per-step order as step_plain."""
    T, B = labels.shape
    L, H = P.L, P.H
    xs = as_input(x)
    scale = 1.0 / (T * B)
    gg, al = plan.gg, plan.alloc
    nodes = gg.nodes
    # forward node -> (time, layer) from the builder's id pattern
    N = len(plan.m)
    info = {}
    t = -1
    for v in range(N):
        op = nodes[v].op
        if op == INPUT:
            t += 1
            layer = -1
        elif op == LSTM_GATES:
            layer = (info[nodes[v].preds[0]][1] + 1) if nodes[nodes[v].preds[0]].op == LSTM_CELL else 0
        elif op == LSTM_CELL:
            layer = info[nodes[v].preds[0]][1]
        else:
            layer = L
        info[v] = (t, layer)
    succ = {}
    for v in range(N):
        for j, p in enumerate(nodes[v].preds):
            succ.setdefault(p, []).append((v, j))
    sizes = {v: nodes[v].out_bytes // 8 for v in range(N)}  # not used for math
    store = {}
    dW = [np.zeros_like(w) for w in P.W]
    db = [np.zeros_like(v) for v in P.b]
    dWo = np.zeros_like(P.W_o)
    dbo = np.zeros_like(P.b_o)
    loss_parts = {}

    def read(p):
        tg = al.tag_of[p]
        if tg not in store or store[tg][0] != p:
            raise TagClobber(f"node {p}: tag {tg} holds {store.get(tg, (None,))[0]}")
        return store[tg][1]

    def out_grad(v_orig, want_width):
        """sum over original successors s of v of the slice of g[s] for v's slot."""
        acc = None
        for s, j in succ.get(v_orig, []):
            gs = gg.g.get(s)
            if gs is None:
                continue
            val = read(gs)
            widths = [_width(nodes[p], H, P) for p in nodes[s].preds]
            off = sum(widths[:j])
            part = val[:, off:off + widths[j]] if val.ndim == 2 else val
            acc = part if acc is None else acc + part
        if acc is None:
            acc = np.zeros((B, want_width))
        return acc

    for v in gg.order:
        nd = nodes[v]
        op = nd.op
        if nd.kind in ("fwd", "mirror"):
            t, l = info[nd.orig]
            if op == INPUT:
                val = xs[t]
            elif op == LSTM_GATES:
                xin = read(nd.preds[0])
                xin = xin[:, :H] if nodes[nodes[nd.orig].preds[0]].op == LSTM_CELL else xin
                h_prev = read(nd.preds[1])[:, :H] if len(nd.preds) > 1 else np.zeros((B, H))
                val = gates_forward(xin, h_prev, P, l, mode)
            elif op == LSTM_CELL:
                act = read(nd.preds[0])
                c_prev = read(nd.preds[1])[:, H:] if len(nd.preds) > 1 else np.zeros((B, H))
                val = cell_forward(act, c_prev)
            elif op == HEAD_CE:
                val = head_forward(read(nd.preds[0])[:, :H], labels[t], P, scale, mode)[0]
                loss_parts[t] = val
            elif op == SUM:
                val = 0.0
                for p in nd.preds:
                    val += read(p)
            else:
                raise NotImplementedError(op)
        else:
            vo = nd.orig
            t, l = info[vo]
            fpreds = nodes[vo].preds
            if op == SUM:
                val = np.ones(len(fpreds))
            elif op == HEAD_CE:
                h = read(nd.preds[-1])[:, :H]
                dh, gwo, gbo = head_backward(h, labels[t], P, scale, mode)
                dWo += gwo
                dbo += gbo
                val = np.concatenate([dh, np.zeros((B, H))], axis=1)
            elif op == LSTM_CELL:
                dS = out_grad(vo, 2 * H)
                act = read(nd.preds[-2] if len(fpreds) > 1 else nd.preds[-1])
                c_prev = read(nd.preds[-1])[:, H:] if len(fpreds) > 1 else np.zeros((B, H))
                dact, dc_prev = cell_backward(dS[:, :H], dS[:, H:], act, c_prev)
                parts = [dact]
                if len(fpreds) > 1:
                    parts.append(np.concatenate([np.zeros((B, H)), dc_prev], axis=1))
                val = np.concatenate(parts, axis=1)
            elif op == LSTM_GATES:
                dact = out_grad(vo, 4 * H)
                ndeps = len(nd.preds)
                act = read(nd.preds[ndeps - len(fpreds) - 1])
                xin = read(nd.preds[ndeps - len(fpreds)])
                xin = xin[:, :H] if nodes[fpreds[0]].op == LSTM_CELL else xin
                h_prev = read(nd.preds[-1])[:, :H] if len(fpreds) > 1 else np.zeros((B, H))
                dx, dhp, gw, gb = gates_backward(dact, act, xin, h_prev, P, l, mode)
                dW[l] += gw
                db[l] += gb
                if nodes[fpreds[0]].op == LSTM_CELL:
                    dx = np.concatenate([dx, np.zeros((B, H))], axis=1)
                parts = [dx]
                if len(fpreds) > 1:
                    parts.append(np.concatenate([dhp, np.zeros((B, H))], axis=1))
                val = np.concatenate(parts, axis=1)
            else:
                raise NotImplementedError(op)
        store[al.tag_of[v]] = (v, val)
    loss = 0.0
    for t in sorted(loss_parts):   # plain left-to-right adds (Python's sum() is compensated)
        loss += loss_parts[t]
    return loss, dict(W=dW, b=db, W_o=dWo, b_o=dbo)


def _width(node, H, P):
    if node.op == INPUT:
        return P.kin(0)
    if node.op == LSTM_CELL:
        return 2 * H
    if node.op == LSTM_GATES:
        return 4 * H
    return 1


def time_segment_plan(g, seg):
    """Explicit mirror plan for time-axis checkpointing: every gates/cell
    node is dropped (m = 1) except the cell states S^l_t at segment ends (t % seg == seg-1)."""
    m = [0] * len(g.nodes)
    t = -1
    for v, nd in enumerate(g.nodes):
        if nd.op == INPUT:
            t += 1
        if nd.op in (LSTM_GATES, LSTM_CELL):
            m[v] = 0 if (nd.op == LSTM_CELL and t % seg == seg - 1) else 1
    return m
