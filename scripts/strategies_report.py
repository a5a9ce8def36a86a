#!/usr/bin/env python
"""The paper's five-strategy memory comparison (Sec. 5 / Fig. 5(a) and 6(a), PAPER.md:409-446;
SURVEY 8(f) f1) on op-granularity graphs, host planner only: feature-map memory (the plan's
exact peak) of no optimization / inplace / sharing / drop bn-relu / sublinear plan (App. A
search over Alg. 3) versus depth, for a pre-activation ResNet (stage feature maps of batch 32
at 224x224: 102.8/51.4/25.7/12.8 MB, BN -> ReLU -> FC -> Add per layer) and for the unrolled
LSTM (4 layers, hidden 1024, batch 64; no drop bn-relu, as in the paper).  Every point is
planned by the C++ library and by the fp64 oracle, which must agree byte for byte; the slope of
log(memory) vs log(depth) is reported per strategy (the paper: linear for the system
optimizations, sub-linear for the plan).

    python scripts/strategies_report.py [--out profiles/r1_strategies]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1604_06174_b200 as slm  # noqa: E402
from oracle import graph as G  # noqa: E402
from oracle import planner as P  # noqa: E402

MB = 1 << 20
RESNET_SIZES = [102_760_448, 51_380_224, 25_690_112, 12_845_056]
STRATEGIES = [("no optimization", "none", 0), ("inplace", "none", slm.ALLOC_INPLACE),
              ("sharing", "none", slm.ALLOC_INPLACE | slm.ALLOC_SHARING),
              ("drop bn-relu", "drop_cheap", slm.ALLOC_INPLACE | slm.ALLOC_SHARING),
              ("sublinear plan", "search", slm.ALLOC_INPLACE | slm.ALLOC_SHARING)]


def plan_both(g, strategy, flags):
    cg = slm.Graph.from_nodes([(nd.op, nd.preds, nd.out_bytes, nd.flags) for nd in g.nodes], g.outputs)
    t0 = time.perf_counter()
    pc = slm.Plan(cg, strategy, alloc_flags=flags)
    t_c = time.perf_counter() - t0
    po = P.plan(g, P.__dict__["S_" + strategy.upper()], alloc_flags=flags)
    same = po.m == pc.m and po.alloc.exact_peak == pc.exact_peak and po.alloc.offsets == pc.tags[2]
    assert same, (strategy, flags)
    return dict(exact_peak=pc.exact_peak, extra_forward=pc.extra_forward, cxx_us=round(t_c * 1e6, 1))


def slope(xs, ys):
    lx, ly = [math.log(x) for x in xs], [math.log(y) for y in ys]
    mx, my = sum(lx) / len(lx), sum(ly) / len(ly)
    return sum((a - mx) * (b - my) for a, b in zip(lx, ly)) / sum((a - mx) ** 2 for a in lx)


def sweep(name, graphs, strategies):
    rows = []
    for depth, g in graphs:
        row = dict(depth=depth, nodes=len(g))
        for label, strat, fl in strategies:
            row[label] = plan_both(g, strat, fl)
        rows.append(row)
        print(name, depth, {k: round(v["exact_peak"] / MB) for k, v in row.items() if isinstance(v, dict)}, flush=True)
    slopes = {label: round(slope([r["depth"] for r in rows], [r[label]["exact_peak"] for r in rows]), 3)
              for label, _, _ in strategies}
    return dict(graph=name, rows=rows, slopes=slopes)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_strategies"))
    a = ap.parse_args()
    resnet = sweep("pre-activation ResNet, batch 32 (4 equal stages)",
                   [(4 * L, G.preact_resnet_graph([L] * 4, RESNET_SIZES)) for L in (8, 16, 32, 64, 128, 250)],
                   STRATEGIES)
    lstm = sweep("LSTM L=4 H=1024 B=64 I=50 (5000-way head per step)",
                 [(T, G.lstm_graph(4, T, 64, 1024, 50)) for T in (16, 32, 64, 128, 256)],
                 [s for s in STRATEGIES if s[0] != "drop bn-relu"])
    out = dict(note="exact peak = the static plan's feature-map memory (PAPER.md:397); C++ == oracle byte for byte",
               reports=[resnet, lstm])
    with open(a.out + ".json", "w") as f:
        json.dump(out, f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("# Memory allocation strategies vs depth (Fig. 5(a) / 6(a) structure, PAPER.md:409-446)\n\n")
        f.write("Host planner only; every number is the plan's exact peak in MiB, planned by the C++ library and the "
                "fp64 oracle (byte-for-byte equal). Sublinear plan = App. A search over Alg. 3 candidates = every "
                "non-Input node.\n\n")
        for r in out["reports"]:
            labels = list(r["slopes"])
            f.write(f"## {r['graph']}\n\n| depth | nodes | " + " | ".join(labels) + " |\n|---|---|" +
                    "---|" * len(labels) + "\n")
            for row in r["rows"]:
                f.write(f"| {row['depth']} | {row['nodes']} | " +
                        " | ".join(f"{row[k]['exact_peak'] / MB:.0f}" + (f" (+{row[k]['extra_forward']})"
                                                                          if row[k]['extra_forward'] else "")
                                   for k in labels) + " |\n")
            f.write("| log-log slope | | " + " | ".join(str(r["slopes"][k]) for k in labels) + " |\n\n")
        f.write("(+k) = re-computed nodes per step.\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
