#!/usr/bin/env python
"""C4 planner report (BASELINE configs[3]): memory vs re-computation of the
paper's plans on 1,000-layer chains, C++ planner (libslm) vs the fp64 Python oracle.

For each graph: a 64-point geometric budget sweep of Alg. 3 (max node size .. sum of sizes),
the App. A search with its trace, recursive k = 1, 2, 3, sqrt(n) and no re-computation.
Every point reports exact peak bytes, extra forward count and re-computed bytes (mirror node
sizes, the FLOP-weighting of SURVEY 8(d)), the C++ wall time (µs) and the oracle's (s), and
asserts that both planners agree byte for byte.

    python scripts/planner_report.py [--out profiles/r1_planner_c4] [--no-oracle-sweep]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1604_06174_b200 as slm  # noqa: E402
from oracle import graph as G  # noqa: E402
from oracle import planner as P  # noqa: E402

MIB = 1 << 20


def resnet_chain(depths, sizes):
    """ResNet-shaped chain: stages of Blocks whose outputs shrink stage by stage (C4 (ii))."""
    nodes = [G.Node(G.INPUT, [], sizes[0])]
    for st, (dep, sz) in enumerate(zip(depths, sizes)):
        for _ in range(dep):
            nodes.append(G.Node(G.BLOCK, [len(nodes) - 1], sz))
    nodes.append(G.Node(G.SOFTMAX_CE, [len(nodes) - 1], 4, G.F_NOT_CANDIDATE))
    return G.Graph(nodes, [len(nodes) - 1], kind="dag", dims=dict(depths=depths))


def cxx_graph(g):
    if g.kind == "chain":
        return slm.Graph.chain(g.dims["n_layers"], g.dims["batch"], g.dims["width"])
    return slm.Graph.from_nodes([(nd.op, nd.preds, nd.out_bytes, nd.flags) for nd in g.nodes], g.outputs)


def recompute_bytes(plan_nodes, order):
    return sum(plan_nodes[v]["out_bytes"] for v in order if plan_nodes[v]["kind"] == 1)


def point(g, cg, label, strategy, oracle=True, **kw):
    t0 = time.perf_counter()
    pc = slm.Plan(cg, strategy, **kw)
    t_c = time.perf_counter() - t0
    nodes, order = pc.nodes, pc.order
    row = dict(plan=label, exact_peak=pc.exact_peak, pool_bytes=pc.pool_bytes, extra_forward=pc.extra_forward,
               recompute_bytes=recompute_bytes(nodes, order), x=pc.x, y=pc.y, budget=pc.budget,
               cxx_us=round(t_c * 1e6, 1))
    if oracle:
        t0 = time.perf_counter()
        po = P.plan(g, P.__dict__["S_" + strategy.upper()], **kw)
        row["oracle_s"] = round(time.perf_counter() - t0, 4)
        same = (po.m == pc.m and po.alloc.exact_peak == pc.exact_peak and po.extra_forward == pc.extra_forward
                and po.alloc.offsets == pc.tags[2])
        row["cxx_equals_oracle"] = bool(same)
        assert same, label
    if strategy == "search":
        row["trace"] = [dict(B=r[0], x=r[1], y=r[2], exact_peak=r[3], extra=r[4]) for r in pc.trace]
    return row


def report(name, g, oracle_sweep=True):
    cg = cxx_graph(g)
    sizes = [nd.out_bytes for nd in g.nodes]
    lo, hi = max(sizes), sum(sizes)
    rows = [point(g, cg, "none", "none"), point(g, cg, "sqrt", "sqrt"), point(g, cg, "search", "search")]
    if g.kind == "chain" or True:
        for k in (1, 2, 3):
            rows.append(point(g, cg, f"recursive k={k}", "recursive", k=k))
    for i in range(64):
        B = int(lo * (hi / lo) ** (i / 63))
        rows.append(point(g, cg, f"budget {i}", "budget", oracle=oracle_sweep or i % 8 == 0, budget=B))
    return dict(graph=name, n_nodes=len(g), sum_bytes=hi, max_node_bytes=lo, rows=rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_planner_c4"))
    ap.add_argument("--no-oracle-sweep", action="store_true")
    a = ap.parse_args()
    graphs = [
        ("uniform chain n=1000, u=2 MiB (B=256, d=2048 fp32)", G.chain_graph(1000, 256, 2048)),
        ("ResNet-shaped chain 4x250 (102.8/51.4/25.7/12.8 MB stages)",
         resnet_chain([250] * 4, [102_760_448, 51_380_224, 25_690_112, 12_845_056])),
        ("ResNet-shaped chain 60/160/720/60 (3:8:36:3 depths)",
         resnet_chain([60, 160, 720, 60], [102_760_448, 51_380_224, 25_690_112, 12_845_056])),
    ]
    out = dict(host=os.uname().nodename, cpus=os.cpu_count(),
               note="host planner only; C++ = libslm slm_plan_create wall time, oracle = oracle.planner.plan",
               reports=[report(n, g, not a.no_oracle_sweep) for n, g in graphs])
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump(out, f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("# C4 planner report: exact peak vs re-computation (C++ == oracle byte for byte)\n\n")
        for r in out["reports"]:
            f.write(f"## {r['graph']}\n\nnodes {r['n_nodes']}, sum of sizes {r['sum_bytes'] / MIB:.1f} MiB, "
                    f"max node {r['max_node_bytes'] / MIB:.1f} MiB\n\n")
            f.write("| plan | exact peak MiB | extra fwd | recompute MiB | C++ µs | oracle s |\n|---|---|---|---|---|---|\n")
            for row in r["rows"]:
                if row["plan"].startswith("budget") and int(row["plan"].split()[1]) % 8:
                    continue
                f.write(f"| {row['plan']}{' (B=%.1f MiB)' % (row['budget'] / MIB) if row['plan'].startswith('budget') else ''}"
                        f" | {row['exact_peak'] / MIB:.1f} | {row['extra_forward']} | {row['recompute_bytes'] / MIB:.1f}"
                        f" | {row['cxx_us']} | {row.get('oracle_s', '')} |\n")
            srch = next(x for x in r["rows"] if x["plan"] == "search")
            f.write("\nApp. A trace (B, x, y, exact peak, extra): " +
                    "; ".join(f"({t['B'] / MIB:.1f} MiB, {t['x'] / MIB:.0f}, {t['y'] / MIB:.0f}, "
                              f"{t['exact_peak'] / MIB:.1f}, {t['extra']})" for t in srch["trace"]) + "\n\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
