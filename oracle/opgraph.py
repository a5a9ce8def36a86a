"""fp64 training step of an op-granularity graph (oracle; TEST INFRASTRUCTURE ONLY).

SURVEY 8(f) f1 — the paper's strategy comparison (Sec. 5.1) is made on
networks whose "conv-bn-relu" layer is several graph nodes, so that "drop the results of low cost
operations" (Sec. 4.2) can drop the BN and ReLU outputs and recompute them.
The graphs are oracle.graph.preact_resnet_graph's: per layer BN(x) -> ReLU -> FC -> Add(x, .),
FC projections between stages of different widths, a SoftmaxCE loss.

Node semantics (every value is [B, width] with width = out_bytes / (4 B); reading A10 for BN):
  Input       the batch x_0
  BN          per-feature batch statistics (biased variance, eps = 1e-5), gamma xhat + beta
  ReLU        max(x, 0); ReLU'(0) = 0
  FC          x W^T + b, W [d_out, d_in]   (the conv / GEMM stand-in)
  Add         a + b
  SoftmaxCE   (1/B_global) sum_b [logsumexp(x_b) - x_b[y_b]]
bf16 mode (reading A11) rounds exactly the GEMM operands the device rounds: the FC input x and W
(forward), the upstream gradient dy (both backward GEMMs), and the dW output; the rest is fp64.

Convolutional graphs (oracle.graph.preact_resnet_conv_graph) carry per-node shapes
(H, W, C, k, s); a value is then the NHWC tensor [B, H, W, C] stored as [B*H*W, C] rows (BN's
statistics run over all B*H*W rows of a channel: per-channel batch norm):
  Conv        y[b,i,j,o] = b_o + sum_{u,v,c} W[o, (u k + v) C_in + c] x[b, i s + u - p, j s + v - p, c]
              ("same" zero padding p = k // 2, stride s, W [C_out, k*k*C_in]) -- the definition,
              summed tap by tap; bf16 mode rounds x, W, dy and dW like FC
  GlobalAvgPool  y[b,c] = (1 / (H W)) sum_{h,w} x[b,h,w,c]

Two executors, as for the chain: step_plain (ordinary back-propagation: the definition) and
step_planned (interprets V' of a plan node by node through the allocator's tags with the
interference check; gradient nodes hold the gradient w.r.t. all of v's inputs, concatenated in
pred order, a node's upstream gradient is the sum of its successors' slices in successor order,
reading A17).
"""
from __future__ import annotations

import numpy as np

from .chain import EPS, TagClobber, _q, bf16_round
from .graph import ADD, BN, CONV, FC, INPUT, POOL, RELU, SOFTMAX_CE, Graph


class OpParams:
    """Per-node parameters: FC / Conv -> (W, b), BN -> (gamma, beta); float64 arrays.
    Convolutional graphs also give ``shapes`` (node -> (H, W, C, k, s)) and the graph, from which
    every Conv / Pool node's input shape is taken (in_shape)."""

    def __init__(self, W=None, b=None, gamma=None, beta=None, shapes=None, graph=None):
        self.W = {k: np.asarray(v, np.float64) for k, v in (W or {}).items()}
        self.b = {k: np.asarray(v, np.float64) for k, v in (b or {}).items()}
        self.gamma = {k: np.asarray(v, np.float64) for k, v in (gamma or {}).items()}
        self.beta = {k: np.asarray(v, np.float64) for k, v in (beta or {}).items()}
        self.shapes = shapes
        self.in_shape = {}
        if shapes is not None and graph is not None:
            for v, nd in enumerate(graph.nodes):
                if nd.preds:
                    self.in_shape[v] = shapes[nd.preds[0]]

    def width(self, v, out_bytes, batch):
        """Row width of node v's value: C of its shape, else out_bytes / (4 batch)."""
        if self.shapes is not None:
            return self.shapes[v][2]
        return out_bytes // (4 * batch)


def conv_forward(x, W, b, in_shape, k, s, mode):
    """Conv (definition above) of x [B*H*W, C_in] -> [B*Ho*Wo, C_out]."""
    H, Wd, Cin = in_shape[0], in_shape[1], in_shape[2]
    B = x.shape[0] // (H * Wd)
    p = k // 2
    Ho, Wo = (H + 2 * p - k) // s + 1, (Wd + 2 * p - k) // s + 1
    Cout = W.shape[0]
    xp = np.pad(_q(x, mode).reshape(B, H, Wd, Cin), ((0, 0), (p, p), (p, p), (0, 0)))
    Wt = _q(W, mode).reshape(Cout, k, k, Cin)
    y = np.zeros((B, Ho, Wo, Cout)) + b
    for u in range(k):
        for v in range(k):
            xs = xp[:, u:u + s * (Ho - 1) + 1:s, v:v + s * (Wo - 1) + 1:s, :]
            y += xs @ Wt[:, u, v, :].T
    return y.reshape(B * Ho * Wo, Cout)


def conv_backward(dy, x, W, in_shape, k, s, mode):
    """(dx, dW, db) of the Conv: dW[o, (u,v,c)] = sum_{b,i,j} dy[b,i,j,o] x[b, i s+u-p, j s+v-p, c],
    dx[b,h,w,c] = sum over the taps that read x[b,h,w] of dy[b,i,j,:] . W[:, (u,v,c)]."""
    H, Wd, Cin = in_shape[0], in_shape[1], in_shape[2]
    B = x.shape[0] // (H * Wd)
    p = k // 2
    Ho, Wo = (H + 2 * p - k) // s + 1, (Wd + 2 * p - k) // s + 1
    Cout = W.shape[0]
    dq = _q(dy, mode).reshape(B, Ho, Wo, Cout)
    xp = np.pad(_q(x, mode).reshape(B, H, Wd, Cin), ((0, 0), (p, p), (p, p), (0, 0)))
    Wt = _q(W, mode).reshape(Cout, k, k, Cin)
    dW = np.zeros((Cout, k, k, Cin))
    dxp = np.zeros_like(xp)
    for u in range(k):
        for v in range(k):
            sl = (slice(None), slice(u, u + s * (Ho - 1) + 1, s), slice(v, v + s * (Wo - 1) + 1, s), slice(None))
            dW[:, u, v, :] = dq.reshape(-1, Cout).T @ xp[sl].reshape(-1, Cin)
            dxp[sl] += dq @ Wt[:, u, v, :]
    dx = dxp[:, p:p + H, p:p + Wd, :].reshape(B * H * Wd, Cin)
    return dx, _q(dW.reshape(Cout, k * k * Cin), mode), dy.sum(axis=0)


def forward_node(op, v, ins, P: OpParams, mode, labels=None, Bg=None):
    if op == BN:
        x = ins[0]
        mu = x.mean(axis=0)
        rstd = 1.0 / np.sqrt(((x - mu) ** 2).mean(axis=0) + EPS)
        return P.gamma[v] * ((x - mu) * rstd) + P.beta[v]
    if op == RELU:
        return np.maximum(ins[0], 0.0)
    if op == FC:
        return _q(ins[0], mode) @ _q(P.W[v], mode).T + P.b[v]
    if op == ADD:
        return ins[0] + ins[1]
    if op == CONV:
        return conv_forward(ins[0], P.W[v], P.b[v], P.in_shape[v], P.shapes[v][3], P.shapes[v][4], mode)
    if op == POOL:
        H, Wd, C = P.in_shape[v][:3]
        return ins[0].reshape(-1, H * Wd, C).mean(axis=1)
    if op == SOFTMAX_CE:
        x = ins[0]
        mx = x.max(axis=1, keepdims=True)
        lse = np.log(np.exp(x - mx).sum(axis=1)) + mx[:, 0]
        return float((lse - x[np.arange(x.shape[0]), labels]).sum() / (Bg or x.shape[0]))
    raise NotImplementedError(op)


def backward_node(op, v, dy, ins, out, P: OpParams, mode, grads, labels=None, Bg=None):
    """Gradients w.r.t. v's inputs (list, pred order); parameter gradients into `grads`."""
    if op == BN:
        x = ins[0]
        Bn = x.shape[0]
        mu = x.mean(axis=0)
        rstd = 1.0 / np.sqrt(((x - mu) ** 2).mean(axis=0) + EPS)
        xh = (x - mu) * rstd
        grads["gamma"][v] = (dy * xh).sum(axis=0)
        grads["beta"][v] = dy.sum(axis=0)
        dxh = dy * P.gamma[v]
        return [rstd * (dxh - dxh.sum(axis=0) / Bn - xh * (dxh * xh).sum(axis=0) / Bn)]
    if op == RELU:
        return [dy * (out > 0)]
    if op == FC:
        dq = _q(dy, mode)
        grads["W"][v] = _q(dq.T @ _q(ins[0], mode), mode)
        grads["b"][v] = dy.sum(axis=0)
        return [dq @ _q(P.W[v], mode)]
    if op == ADD:
        return [dy, dy]
    if op == CONV:
        dx, grads["W"][v], grads["b"][v] = conv_backward(dy, ins[0], P.W[v], P.in_shape[v], P.shapes[v][3],
                                                          P.shapes[v][4], mode)
        return [dx]
    if op == POOL:
        H, Wd, C = P.in_shape[v][:3]
        return [np.repeat(dy[:, None, :] / (H * Wd), H * Wd, axis=1).reshape(-1, C)]
    if op == SOFTMAX_CE:
        x = ins[0]
        mx = x.max(axis=1, keepdims=True)
        e = np.exp(x - mx)
        p = e / e.sum(axis=1, keepdims=True)
        p[np.arange(x.shape[0]), labels] -= 1.0
        return [p / (Bg or x.shape[0])]
    raise NotImplementedError(op)


def _empty_grads():
    return dict(W={}, b={}, gamma={}, beta={})


def step_plain(g: Graph, P: OpParams, x0, labels, mode="f64", batch_global=None):
    """Ordinary back-propagation over the graph (the definition the plans must reproduce)."""
    x0 = np.asarray(x0, np.float64)
    Bg = batch_global   # None: the loss input's rows (the batch)
    val = {}
    for v, nd in enumerate(g.nodes):
        val[v] = x0 if nd.op == INPUT else forward_node(nd.op, v, [val[u] for u in nd.preds], P, mode, labels, Bg)
    out = g.outputs[0]
    grads = _empty_grads()
    dval = {}
    for v in reversed(range(len(g.nodes))):
        nd = g.nodes[v]
        if nd.op == INPUT:
            continue
        if v == out:
            dy = None
        elif v not in dval:
            continue
        else:
            dy = dval[v]
        dins = backward_node(nd.op, v, dy, [val[u] for u in nd.preds], val[v], P, mode, grads, labels, Bg)
        for u, du in zip(nd.preds, dins):
            dval[u] = du if u not in dval else dval[u] + du
    return val[out], grads


def step_planned(plan, g: Graph, P: OpParams, x0, labels, mode="f64", batch_global=None):
    """Interpret V' of `plan` (oracle.planner.plan on g) node by node through the tags."""
    x0 = np.asarray(x0, np.float64)
    Bg = batch_global   # None: the loss input's rows (the batch)
    gg, al = plan.gg, plan.alloc
    store = {}
    grads = _empty_grads()
    loss = None

    def read(p):
        t = al.tag_of[p]
        if t not in store or store[t][0] != p:
            raise TagClobber(f"node {p}: tag {t} holds {store.get(t, (None,))[0]}")
        return store[t][1]

    for v in gg.order:
        nd = gg.nodes[v]
        if nd.kind in ("fwd", "mirror"):
            if nd.op == INPUT:
                val = x0
            else:
                val = forward_node(nd.op, nd.orig, [read(u) for u in nd.preds], P, mode, labels, Bg)
                if nd.op == SOFTMAX_CE:
                    loss = val
        else:
            orig = nd.orig
            onode = g.nodes[orig]
            # successor gradient nodes come first in the preds (Alg. 2, reading A17): the upstream
            # gradient of orig is the sum of their slices for orig, in successor order
            dy = None
            k = 0
            while k < len(nd.preds) and gg.nodes[nd.preds[k]].kind == "grad":
                s = gg.nodes[nd.preds[k]]
                sg = read(nd.preds[k])
                spreds = g.nodes[s.orig].preds
                off = 0
                for u in spreds:
                    w = P.width(u, g.nodes[u].out_bytes, x0.shape[0])
                    if u == orig:
                        sl = sg[:, off:off + w]
                        dy = sl if dy is None else dy + sl
                    off += w
                k += 1
            rest = [read(u) for u in nd.preds[k:]]
            out = rest.pop(0) if onode.op in (RELU,) else None
            ins = rest if rest else [None] * len(onode.preds)
            dins = backward_node(onode.op, orig, dy, ins, out, P, mode, grads, labels, Bg)
            val = np.concatenate(dins, axis=1)
        store[al.tag_of[v]] = (v, val)
    return loss, grads
