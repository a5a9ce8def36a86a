"""Memory planning of arXiv 1604.06174 (oracle; TEST INFRASTRUCTURE ONLY).

Transcribes, step by step and in the paper's order:
  * Alg. 3 "Memory Planning with Budget"
  * App. A "Search over Budget B"
  * Sec. 4.3 sqrt(n) segmentation, Eq. 1
  * Sec. 4.4 recursion, Eqs. 2-3
  * Sec. 4.2 drop results of low-cost operations
  * Alg. 2 "Memory Optimized Gradient Graph Construction"
  * Fig. 2 liveness-counter / temporal-tag static allocator
Readings A1..A20 are cited where the paper is silent.

Plans are deterministic functions of (graph, options): every tie has a total order, every
budget is an integer number of bytes, so the C++ planner can be compared byte for byte.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from .graph import (OPS, INPUT, F_NOT_CANDIDATE, F_PIN, F_REQUEST_GRAD, Graph,
                    topo_order, successors, _kahn, G_NONE, G_SUCC0, G_OUT, G_IN0)

# strategies (values mirrored independently in include/slm.h)
S_NONE, S_SQRT, S_BUDGET, S_SEARCH, S_RECURSIVE, S_EXPLICIT, S_DROP_CHEAP = range(7)
# allocator switches (the paper's compared strategies)
A_INPLACE, A_SHARING, A_GROUPED, A_GROUP_MIRRORS, A_MIRROR_PARITY = 1, 2, 4, 8, 16

# App. A grid, reading A3: 6 geometric points 2^((2i-5)/10), i=0..5, spanning [B/sqrt2, sqrt2 B]
GRID = (0.7071067811865476, 0.8122523963562356, 0.9330329915368074,
        1.0717734625362931, 1.2311444133449163, 1.4142135623730951)


class PlanError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


E_ARG, E_GRAPH_INVALID, E_MULTIPLE_ROOTS, E_INVALID_PLAN, E_NOT_A_CHAIN, E_DOMAIN = \
    -1, -2, -3, -4, -5, -6


# ================================================================== strategies -> m
def candidates(g: Graph):
    """Alg. 3's candidate set C, reading A19: every non-Input node not flagged."""
    return [g.nodes[v].op != INPUT and not (g.nodes[v].flags & F_NOT_CANDIDATE)
            for v in range(len(g))]


def alg3(g: Graph, B: int, topo=None):
    """Alg. 3, literally, with readings A1 (Input adds 0, m=0) and
    A2 (y = max(y, temp) after the loop).  Returns (x, y, m)."""
    topo = topo if topo is not None else topo_order(g)
    C = candidates(g)
    temp, x, y = 0, 0, 0
    m = [0] * len(g)
    for v in topo:
        if g.nodes[v].op == INPUT:                        # A1
            m[v] = 0
            continue
        temp = temp + g.nodes[v].out_bytes
        if C[v] and temp > B:
            x = x + g.nodes[v].out_bytes
            y = max(y, temp)
            m[v] = 0
            temp = 0
        else:
            m[v] = 1
    y = max(y, temp)                                      # A2
    return x, y, m


def sqrt_plan(g: Graph, topo=None):
    """Sec. 4.3: k = ceil(sqrt(n)) equal segments; keep segment outputs.

    Reading A4: S = candidates in topo order (n = |S|), k = isqrt(n-1)+1, kept S[s_j]
    with 1-based s_j = floor(j*n/k), j=1..k; every other member of S gets m=1."""
    topo = topo if topo is not None else topo_order(g)
    C = candidates(g)
    S = [v for v in topo if C[v]]
    m = [0] * len(g)
    n = len(S)
    if n == 0:
        return m
    k = math.isqrt(n - 1) + 1
    kept = {(j * n) // k for j in range(1, k + 1)}
    for i, v in enumerate(S, start=1):
        m[v] = 0 if i in kept else 1
    return m


def chain_positions(g: Graph, topo=None):
    """Chain check for the recursive plan: returns the path [X_0 .. X_n]
    (Input, then candidates) or raises NotAChain."""
    topo = topo if topo is not None else topo_order(g)
    succ = successors(g)
    if not topo or g.nodes[topo[0]].op != INPUT:
        raise PlanError(E_NOT_A_CHAIN, "NotAChain")
    for i, v in enumerate(topo):
        nd = g.nodes[v]
        if i > 0 and nd.preds != [topo[i - 1]]:
            raise PlanError(E_NOT_A_CHAIN, "NotAChain")
        if len(succ[v]) > 1:
            raise PlanError(E_NOT_A_CHAIN, "NotAChain")
    C = candidates(g)
    last = max([i for i, v in enumerate(topo) if C[v]], default=0)
    return topo[: last + 1]


def recursive_plan(g: Graph, k: int, topo=None):
    """Sec. 4.4: a segment is a bulk operator whose backward re-runs the
    same scheme on its sub-path.  Reading A5: interval (lo, hi), split points
    lo + floor(j*(hi-lo)/(k+1)), j=1..k, strictly inside, deduplicated; m(split) = level;
    recurse into each sub-interval at level+1; X_0 and X_n have m=0."""
    if k < 1:
        raise PlanError(E_DOMAIN, "DomainError")
    path = chain_positions(g, topo)
    n = len(path) - 1
    m = [0] * len(g)

    def rec(lo, hi, level):
        if hi - lo < 2:
            return
        splits = sorted({lo + (j * (hi - lo)) // (k + 1) for j in range(1, k + 1)})
        splits = [s for s in splits if lo < s < hi]
        for s in splits:
            m[path[s]] = level
        pts = [lo] + splits + [hi]
        for a, b in zip(pts[:-1], pts[1:]):
            rec(a, b, level + 1)

    rec(0, n, 0)
    return m


def drop_cheap_plan(g: Graph):
    """Sec. 4.2: drop (m=1) results of low-cost ops (BN, activation),
    keep the rest; graph outputs are kept."""
    outs = set(g.outputs)
    return [1 if (OPS[nd.op].low_cost and v not in outs and nd.op != INPUT) else 0
            for v, nd in enumerate(g.nodes)]


def recursion_estimate(n: int, k: int):
    """Eq. 2 g(n) = k + g(n/(k+1)) iterated with ceiling division until n <= 1
    (PAPER.md:366-367); returns (units, depth).  Eq. 3: g(n) = k log_{k+1} n."""
    if n < 1 or k < 1:
        raise PlanError(E_DOMAIN, "DomainError")
    units = depth = 0
    while n > 1:
        units += k
        n = -(-n // (k + 1))
        depth += 1
    return units, depth


# ================================================================== Alg. 2
@dataclass
class GNode:
    kind: str          # 'fwd' | 'mirror' | 'grad'
    op: int
    orig: int          # forward node it mirrors / differentiates (itself for 'fwd')
    level: int         # mirror level k (0 for fwd / grad)
    preds: list
    out_bytes: int
    inplace_slot: int


@dataclass
class GradGraph:
    nodes: list
    order: list            # V': the logical execution order
    a: list                # final a[v] (deepest mirror)
    g: dict                # forward node -> gradient node
    pinned: set = field(default_factory=set)
    external: set = field(default_factory=set)


def build_mirrored(g: Graph, m, topo=None) -> GradGraph:
    """Alg. 2, literally.  Readings: A6 (minimal deps), A7 (dead mirrors
    are not in V'), A17 (gradient nodes only for non-Input nodes that reach the loss; a
    gradient node's output is the gradient w.r.t. all of v's inputs, sum of their sizes)."""
    N = len(g)
    if len(g.outputs) != 1:
        raise PlanError(E_MULTIPLE_ROOTS, "MultipleRoots")
    if len(m) != N or any(x < 0 for x in m):
        raise PlanError(E_INVALID_PLAN, "InvalidPlan")
    for v in range(N):
        if g.nodes[v].op == INPUT and m[v] != 0:
            raise PlanError(E_INVALID_PLAN, "InvalidPlan")
    topo = topo if topo is not None else topo_order(g)
    nodes = [GNode('fwd', nd.op, v, 0, list(nd.preds), nd.out_bytes, OPS[nd.op].fwd_inplace)
             for v, nd in enumerate(g.nodes)]
    a = list(range(N))
    for k in range(1, max(m, default=0) + 1):
        for v in topo:
            if k <= m[v]:
                nd = g.nodes[v]
                nid = len(nodes)
                nodes.append(GNode('mirror', nd.op, v, k, [a[u] for u in nd.preds],  # :269
                                   nd.out_bytes, OPS[nd.op].fwd_inplace))
                a[v] = nid
    succ = successors(g)
    reaches = [False] * N
    for v in reversed(topo):
        reaches[v] = v in g.outputs or any(reaches[s] for s in succ[v])
    order = list(topo)
    in_order = set(order)
    gnode = {}
    for v in reversed(topo):
        nd = g.nodes[v]
        if nd.op == INPUT or not reaches[v]:
            continue
        meta = OPS[nd.op]
        preds = [gnode[s] for s in succ[v] if s in gnode]         # successor gradients
        n_succ = len(preds)
        slot = {G_SUCC0: 0 if n_succ else -1, G_NONE: -1}.get(meta.grad_inplace, -1)
        if meta.grad_needs_out:
            if meta.grad_inplace == G_OUT:
                slot = len(preds)
            preds.append(a[v])                                    # a[v]
        first_in = True
        for i, u in enumerate(nd.preds):                          # [a[u] for u in pred[v]]
            if (meta.grad_needs_in >> i) & 1:
                if meta.grad_inplace == G_IN0 and first_in:
                    slot = len(preds)
                first_in = False
                preds.append(a[u])
        size = sum(g.nodes[u].out_bytes for u in nd.preds)
        gid = len(nodes)
        nodes.append(GNode('grad', nd.op, v, 0, preds, size, slot))
        gnode[v] = gid
        # PAPER.md:276 V' <- append(V', topological-order(ancestors(g[v])) - V')
        new, stack = set(), [gid]
        while stack:
            w = stack.pop()
            if w in in_order or w in new:
                continue
            new.add(w)
            stack.extend(nodes[w].preds)
        app = _kahn(None, sorted(new), lambda w: nodes[w].preds)
        order.extend(app)
        in_order.update(app)
    pinned = set()
    external = set()
    for v, nd in enumerate(g.nodes):
        if nd.op == INPUT:
            pinned.add(v)
            external.add(v)
            if nd.flags & F_REQUEST_GRAD:
                for s in succ[v]:
                    if s in gnode:
                        pinned.add(gnode[s])
        if nd.flags & F_PIN:
            pinned.add(v)
    for o in g.outputs:
        pinned.add(o)
        external.add(o)
    return GradGraph(nodes, order, a, gnode, pinned, external)


def extra_forward(gg: GradGraph):
    """Reading A7: number of mirror nodes in V' (re-computed forward ops)."""
    return sum(1 for v in gg.order if gg.nodes[v].kind == 'mirror')


# ================================================================== Fig. 2 allocator
@dataclass
class Allocation:
    tag_of: dict           # node -> tag
    tag_size: list
    tag_external: list
    inplace_pairs: list
    offsets: list          # per tag; -1 for external tags
    pool_bytes: int
    exact_peak: int


def allocate(gg: GradGraph, flags=A_INPLACE | A_SHARING, align=256, groups=None) -> Allocation:
    """Fig. 2 over V' with reading A8:
    counter = pending consumers; (1) in place iff the op declares a slot, that input's
    counter is 1, sizes are equal and the input is not pinned; (2) else the smallest free
    tag with size >= request (ties: lowest tag id); (3) else a fresh tag of exactly that
    size; (4) only then decrement input counters and release tags that reach 0.  Nodes
    with no consumers are released right after they run.  Pinned tags never recycle.
    Offsets: reading A9.  A_GROUPED (reading A22, an extension): step (2) only considers free
    tags created by a node of the same allocation group (groups[orig]); A_GROUP_MIRRORS further
    separates mirror nodes from the others; A_MIRROR_PARITY (reading A24) separates them too and
    lets a mirror reuse only tags of mirrors whose recompute phase has the same parity."""
    nodes = gg.nodes
    mpar = {}
    if flags & A_MIRROR_PARITY:
        # recompute phase of each mirror (reading A24): a maximal run of consecutive mirrors in V'
        # joins the latest phase one of its mirrors reads a mirror of; otherwise it starts a new one
        phase, n_phase, order, i = {}, 0, gg.order, 0
        while i < len(order):
            if nodes[order[i]].kind != "mirror":
                i += 1
                continue
            j = i
            while j < len(order) and nodes[order[j]].kind == "mirror":
                j += 1
            ph = max((phase[u] for k in range(i, j) for u in nodes[order[k]].preds if u in phase), default=-1)
            if ph < 0:
                ph, n_phase = n_phase, n_phase + 1
            for k in range(i, j):
                phase[order[k]] = ph
                mpar[order[k]] = ph % 2
            i = j

    def grp(v):
        g = groups[nodes[v].orig] if (flags & A_GROUPED) and groups is not None else 0
        im = nodes[v].kind == "mirror"
        if flags & A_MIRROR_PARITY:
            return 3 * g + (1 + mpar[v] if im else 0)
        return 2 * g + im if flags & A_GROUP_MIRRORS else g
    tag_group = []
    cnt = {}
    for v in gg.order:
        cnt.setdefault(v, 0)
        for p in nodes[v].preds:
            cnt[p] = cnt.get(p, 0) + 1
    tag_of, tag_size, tag_ext, pairs, free = {}, [], [], [], []
    for v in gg.order:
        nd = nodes[v]
        t = None
        if v in gg.external:
            t = len(tag_size)
            tag_size.append(nd.out_bytes)
            tag_ext.append(True)
            tag_group.append(grp(v))
        else:
            s = nd.inplace_slot
            if (flags & A_INPLACE) and 0 <= s < len(nd.preds):
                u = nd.preds[s]
                if cnt[u] == 1 and nodes[u].out_bytes == nd.out_bytes and u not in gg.pinned:
                    t = tag_of[u]
                    pairs.append((u, v))
            if t is None and (flags & A_SHARING):
                best = None
                for f in free:
                    if tag_size[f] >= nd.out_bytes and tag_group[f] == grp(v):
                        if best is None or (tag_size[f], f) < (tag_size[best], best):
                            best = f
                if best is not None:
                    free.remove(best)
                    t = best
            if t is None:
                t = len(tag_size)
                tag_size.append(nd.out_bytes)
                tag_ext.append(False)
                tag_group.append(grp(v))
        tag_of[v] = t
        for u in nd.preds:
            cnt[u] -= 1
            if cnt[u] == 0 and u not in gg.pinned and tag_of[u] != t:
                free.append(tag_of[u])
        if cnt[v] == 0 and v not in gg.pinned:
            free.append(t)
    offsets, run = [], 0
    for t, sz in enumerate(tag_size):
        if tag_ext[t]:
            offsets.append(-1)
        else:
            off = (run + align - 1) // align * align
            offsets.append(off)
            run = off + sz
    return Allocation(tag_of, tag_size, tag_ext, pairs, offsets, run, sum(tag_size))


# ================================================================== full plan
@dataclass
class Plan:
    m: list
    gg: GradGraph
    alloc: Allocation
    extra_forward: int
    x: int = 0
    y: int = 0
    B: int = 0
    trace: list = field(default_factory=list)   # App. A rows (B, x, y, exact_peak, extra)


def _make(g, m, topo, flags, align):
    gg = build_mirrored(g, m, topo)
    al = allocate(gg, flags, align, [nd.group for nd in g.nodes])
    return Plan(list(m), gg, al, extra_forward(gg))


def plan(g: Graph, strategy=S_SQRT, budget=0, k=1, m=None, alloc_flags=A_INPLACE | A_SHARING,
         align=256) -> Plan:
    """plan(graph, budget) -> checkpoint set + memory plan (the C-ABI slm_plan_create)."""
    topo = topo_order(g)
    if strategy == S_NONE:
        return _make(g, [0] * len(g), topo, alloc_flags, align)
    if strategy == S_SQRT:
        return _make(g, sqrt_plan(g, topo), topo, alloc_flags, align)
    if strategy == S_BUDGET:
        if budget < 0:
            raise PlanError(E_ARG, "negative budget")
        x, y, mm = alg3(g, budget, topo)
        p = _make(g, mm, topo, alloc_flags, align)
        p.x, p.y, p.B = x, y, budget
        return p
    if strategy == S_SEARCH:
        return search(g, topo, alloc_flags, align)
    if strategy == S_RECURSIVE:
        return _make(g, recursive_plan(g, k, topo), topo, alloc_flags, align)
    if strategy == S_EXPLICIT:
        if m is None:
            raise PlanError(E_ARG, "explicit plan needs m")
        return _make(g, list(m), topo, alloc_flags, align)
    if strategy == S_DROP_CHEAP:
        return _make(g, drop_cheap_plan(g), topo, alloc_flags, align)
    raise PlanError(E_ARG, "unknown strategy")


def search(g: Graph, topo=None, alloc_flags=A_INPLACE | A_SHARING, align=256) -> Plan:
    """App. A, reading A3: run Alg. 3 with B=0 -> (x0, y0);
    B1 = isqrt(x0*y0); then the 6-point grid floor(B1*f_i).  Every budget's plan goes
    through Alg. 2 + the allocator for its exact cost.  Best = min
    exact peak, then min extra forward, then min B.  Trace = 8 rows."""
    topo = topo if topo is not None else topo_order(g)
    rows, plans = [], []

    def run(B):
        x, y, mm = alg3(g, B, topo)
        p = _make(g, mm, topo, alloc_flags, align)
        p.x, p.y, p.B = x, y, B
        rows.append((B, x, y, p.alloc.exact_peak, p.extra_forward))
        plans.append(p)
        return x, y

    x0, y0 = run(0)                                      # PAPER.md:532 "first ... with B=0"
    B1 = math.isqrt(x0 * y0)                             # PAPER.md:533 "B = sqrt(x y)"
    run(B1)
    for f in GRID:                                       # PAPER.md:537 "size 6 grid"
        run(math.floor(float(B1) * f))
    best = min(range(len(plans)), key=lambda i: (rows[i][3], rows[i][4], rows[i][0]))
    p = plans[best]
    p.trace = rows
    return p
