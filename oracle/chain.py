"""fp64 residual-chain training step (oracle; TEST INFRASTRUCTURE ONLY).

The chain is the paper's linear-chain network (Alg. 1) with the
ResNet "conv-bn-relu = one layer" block replaced by a dense
pre-activation residual block (reading A10):

    x_{l+1} = x_l + ReLU(gamma_l * (x_l - mu_l) * rstd_l + beta_l) @ W_l^T + b_l

mu_l, var_l = per-feature batch mean / biased variance, rstd = 1/sqrt(var + 1e-5); no
running statistics.  Loss = (1/B_global) * sum_b [logsumexp(x_n[b]) - x_n[b, y_b]]
(softmax cross-entropy over the d features).

Two executors:
  * ``step_plain``  — ordinary reverse-mode backprop, no planning: the *definition* the
    method must reproduce ("all the memory optimizations ... give equivalent weight
    gradient").
  * ``step_planned`` — interprets V' of a plan (Alg. 2 output) node by node, storing each
    value in its allocator tag and asserting every read sees the node it expects (the
    interference check; "ad hoc application ... can lead to errors").

Precision modes (reading A11):
  * "f64":  everything fp64.
  * "bf16": GEMM operands rounded to bf16 (round-to-nearest-even) exactly where the
            device path rounds them (W, a_l, dx_{l+1} copy; dW output); the rest fp64.
"""
from __future__ import annotations

import numpy as np

from .graph import BLOCK, SOFTMAX_CE, INPUT

EPS = 1e-5


def bf16_round(x):
    """Round-to-nearest-even to bfloat16, returned as float64 (via the fp32 bit pattern)."""
    f = np.asarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    b = (b + 0x7FFF + lsb) & 0xFFFF0000
    out = b.astype(np.uint32).view(np.float32).astype(np.float64)
    # NaN/inf are not produced by this model; keep them unchanged if they appear
    bad = ~np.isfinite(f)
    if bad.any():
        out[bad] = f[bad]
    return out


class Params:
    """W [n, d, d] (out, in), b/gamma/beta [n, d] as float64 arrays."""

    def __init__(self, W, b, gamma, beta):
        self.W = np.asarray(W, dtype=np.float64)
        self.b = np.asarray(b, dtype=np.float64)
        self.gamma = np.asarray(gamma, dtype=np.float64)
        self.beta = np.asarray(beta, dtype=np.float64)

    @property
    def n(self):
        return self.W.shape[0]


def _q(x, mode):
    return bf16_round(x) if mode == "bf16" else x


def block_forward(x, P: Params, l, mode="f64"):
    """Forward of Block_l (A10).  Returns x_{l+1}."""
    mu = x.mean(axis=0)
    var = ((x - mu) ** 2).mean(axis=0)
    rstd = 1.0 / np.sqrt(var + EPS)
    xhat = (x - mu) * rstd
    u = P.gamma[l] * xhat + P.beta[l]
    a = _q(np.maximum(u, 0.0), mode)
    z = a @ P.W[l].T + P.b[l]
    return x + z


def block_backward(g, x, P: Params, l, mode="f64"):
    """Backward of Block_l given g = dL/dx_{l+1} and its input x = x_l.

    Returns dx_l and (dW_l, db_l, dgamma_l, dbeta_l).  Standard BN backward with batch
    statistics; ReLU'(0) = 0 (A10)."""
    Bn = x.shape[0]
    mu = x.mean(axis=0)
    var = ((x - mu) ** 2).mean(axis=0)
    rstd = 1.0 / np.sqrt(var + EPS)
    xhat = (x - mu) * rstd
    u = P.gamma[l] * xhat + P.beta[l]
    a = _q(np.maximum(u, 0.0), mode)
    gq = _q(g, mode)
    db = g.sum(axis=0)
    dW = _q(gq.T @ a, mode)
    da = gq @ P.W[l]
    du = da * (u > 0)
    dgamma = (du * xhat).sum(axis=0)
    dbeta = du.sum(axis=0)
    dxhat = du * P.gamma[l]
    dxbn = rstd * (dxhat - dxhat.sum(axis=0) / Bn - xhat * (dxhat * xhat).sum(axis=0) / Bn)
    return g + dxbn, (dW, db, dgamma, dbeta)


def ce_loss(x, labels, batch_global):
    """Softmax cross-entropy summed over the local rows, divided by the global batch."""
    mx = x.max(axis=1, keepdims=True)
    lse = np.log(np.exp(x - mx).sum(axis=1)) + mx[:, 0]
    return float((lse - x[np.arange(x.shape[0]), labels]).sum() / batch_global)


def ce_backward(x, labels, batch_global):
    mx = x.max(axis=1, keepdims=True)
    e = np.exp(x - mx)
    p = e / e.sum(axis=1, keepdims=True)
    p[np.arange(x.shape[0]), labels] -= 1.0
    return p / batch_global


def step_plain(P: Params, x0, labels, mode="f64", batch_global=None):
    """Plain backprop: forward storing every x_l, then reverse."""
    x0 = np.asarray(x0, dtype=np.float64)
    Bg = batch_global or x0.shape[0]
    xs = [x0]
    for l in range(P.n):
        xs.append(block_forward(xs[-1], P, l, mode))
    loss = ce_loss(xs[-1], labels, Bg)
    g = ce_backward(xs[-1], labels, Bg)
    grads = [None] * P.n
    for l in reversed(range(P.n)):
        g, grads[l] = block_backward(g, xs[l], P, l, mode)
    return loss, _stack(grads), g


def _stack(grads):
    if not grads:
        return dict(W=None, b=None, gamma=None, beta=None)
    return dict(W=np.stack([t[0] for t in grads]), b=np.stack([t[1] for t in grads]),
                gamma=np.stack([t[2] for t in grads]), beta=np.stack([t[3] for t in grads]))


class TagClobber(AssertionError):
    pass


def step_planned(plan, P: Params, x0, labels, mode="f64", batch_global=None):
    """Execute V' of ``plan`` (oracle.planner.Plan on oracle.graph.chain_graph) through its
    tags: "gradient calculation ... just a forward pass on the entire computation graph"
    (PAPER.md:135).  Each node's value is stored under its tag; a read of predecessor p
    asserts the tag still holds p (interference check).  Returns (loss, grads, dx0, stats)
    with stats = dict(peak_live_bytes = the peak over V' of the bytes of values still to be read
    (Input values count throughout), op_evaluations)."""
    x0 = np.asarray(x0, dtype=np.float64)
    Bg = batch_global or x0.shape[0]
    gg, al = plan.gg, plan.alloc
    store = {}            # tag -> (node, value)
    grads = [None] * P.n
    evals = 0
    # liveness of the values (not the tags): a node's value is live from its evaluation until its
    # last reader in V' has run; the peak of the live bytes is what any allocator must hold at once
    last_read = {}
    for i, v in enumerate(gg.order):
        for p in gg.nodes[v].preds:
            last_read[p] = i
    live = {}             # node -> bytes
    peak = 0
    dx0 = None
    loss = None

    def read(p):
        t = al.tag_of[p]
        if t not in store or store[t][0] != p:
            raise TagClobber(f"node {p}: tag {t} holds {store.get(t, (None,))[0]}")
        return store[t][1]

    # Inputs and the loss (the graph output) stay live for the whole step (A8 pins them)
    pinned = {v for v, nd in enumerate(gg.nodes) if nd.op == INPUT or (nd.op == SOFTMAX_CE and nd.kind == "fwd")}
    for i, v in enumerate(gg.order):
        nd = gg.nodes[v]
        if nd.kind in ("fwd", "mirror"):
            if nd.op == INPUT:
                val = x0
            elif nd.op == BLOCK:
                val = block_forward(read(nd.preds[0]), P, nd.orig - 1, mode)
                evals += 1
            elif nd.op == SOFTMAX_CE:
                loss = ce_loss(read(nd.preds[0]), labels, Bg)
                val = loss
                evals += 1
            else:
                raise NotImplementedError(nd.op)
        else:  # gradient node
            if nd.op == SOFTMAX_CE:
                val = ce_backward(read(nd.preds[0]), labels, Bg)
            elif nd.op == BLOCK:
                gsucc, xin = read(nd.preds[0]), read(nd.preds[1])
                l = nd.orig - 1
                val, grads[l] = block_backward(gsucc, xin, P, l, mode)
                if l == 0:
                    dx0 = val
            else:
                raise NotImplementedError(nd.op)
            evals += 1
        # an in-place node (A8) overwrites the value of the predecessor whose tag it takes
        for p in nd.preds:
            if al.tag_of[p] == al.tag_of[v]:
                live.pop(p, None)
        store[al.tag_of[v]] = (v, val)
        live[v] = nd.out_bytes
        peak = max(peak, sum(live.values()))
        for p in [u for u in live if last_read.get(u, -1) <= i and u not in pinned]:
            del live[p]
    return loss, _stack(grads), dx0, dict(peak_live_bytes=peak, op_evaluations=evals)


def relu_margin(P: Params, x0, mode="f64"):
    """Smallest relative distance of a ReLU input from its decision point 0 over the forward
    pass: min |u| / (|gamma xhat| + |beta|).  Reading A20: ReLU'(0) = 0 is a discrete
    decision taken on fp32 u by the device and on fp64 u here; inputs whose margin is
    within the rounding of the fp32 batch statistics (< 1e-5) would let the two sides take
    different (equally valid) decisions, so parity tests draw seeds with a larger margin."""
    x = np.asarray(x0, dtype=np.float64)
    worst = np.inf
    for l in range(P.n):
        mu = x.mean(axis=0)
        rstd = 1.0 / np.sqrt(((x - mu) ** 2).mean(axis=0) + EPS)
        gx = P.gamma[l] * (x - mu) * rstd
        u = gx + P.beta[l]
        worst = min(worst, float((np.abs(u) / (np.abs(gx) + np.abs(P.beta[l]) + 1e-30)).min()))
        x = block_forward(x, P, l, mode)
    return worst


def step_dp(P: Params, x0, labels, world, mode="f64"):
    """Data-parallel emulation (reading A14): rank r holds rows [r*Bl, (r+1)*Bl); BN stats
    are local; loss = mean over the global batch; grads = sum over ranks of the locally
    1/B_global-scaled grads (what an all-reduce(sum) produces)."""
    x0 = np.asarray(x0, dtype=np.float64)
    Bg = x0.shape[0]
    Bl = Bg // world
    loss, tot = 0.0, None
    for r in range(world):
        sl = slice(r * Bl, (r + 1) * Bl)
        lr, gr, _ = step_plain(P, x0[sl], labels[sl], mode, batch_global=Bg)
        loss += lr
        tot = gr if tot is None else {k: tot[k] + gr[k] for k in tot}
    return loss, tot
