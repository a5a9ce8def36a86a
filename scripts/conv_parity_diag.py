"""Conv ResNet parity diagnostics: per parameter gradient, the device vs the
oracle's bf16 mode and the oracle's bf16 vs fp64 modes (max_abs / rms_ref, rel_l2, fraction of
elements outside 2e-2 (|ref| + rms))."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402
from oracle import graph as OGR  # noqa: E402
from oracle import opgraph as OG  # noqa: E402

B, hw = int(os.environ.get("B", 64)), int(os.environ.get("HW", 8))
stages = [(128, 1), (256, 1)]
nodes, shapes = slm.OpsModel.preact_conv_nodes(B, hw, stages, 128)
inp = synth.opgraph_inputs(nodes, B, seed=int(os.environ.get("SEED", 5)), shapes=shapes)
dev = torch.device("cuda", 0)
params, grads = {}, {}
for v, pv in inp["params"].items():
    params[v] = {k: torch.tensor(a, device=dev, dtype=torch.bfloat16 if k == "W" else torch.float32) for k, a in pv.items()}
    grads[v] = {k: torch.zeros_like(t) for k, t in params[v].items()}
x = torch.tensor(inp["x0"], device=dev)
y = torch.tensor(inp["labels"], device=dev)
graph = slm.Graph.from_nodes(nodes, [len(nodes) - 1])
model = slm.OpsModel(graph, params, grads, B, shapes=shapes)
plan = slm.Plan(graph, os.environ.get("STRATEGY", "none"), alloc_flags=3)
loss = model.step(plan, x, y)
torch.cuda.synchronize()
og, osh = OGR.preact_resnet_conv_graph(B, hw, stages, 128)
pr = inp["params"]
P = OG.OpParams({v: p["W"] for v, p in pr.items() if "W" in p}, {v: p["b"] for v, p in pr.items() if "b" in p},
                {v: p["gamma"] for v, p in pr.items() if "gamma" in p},
                {v: p["beta"] for v, p in pr.items() if "beta" in p}, shapes=osh, graph=og)
lb, gb = OG.step_plain(og, P, inp["x0"].astype(np.float64), inp["labels"], "bf16")
lf, gf = OG.step_plain(og, P, inp["x0"].astype(np.float64), inp["labels"], "f64")
print(f"loss device {loss.item():.6f} oracle bf16 {lb:.6f} f64 {lf:.6f}")


def st(a, r):
    rms = float(np.sqrt(np.mean(r * r)))
    e = np.abs(a - r)
    return f"max/rms {e.max() / rms:.2e} rel {np.linalg.norm(a - r) / np.linalg.norm(r):.2e} out {(e > 2e-2 * (np.abs(r) + rms)).mean():.3f}"


for v in sorted(grads):
    for k, t in grads[v].items():
        a = t.float().cpu().numpy().astype(np.float64)
        print(f"node {v:3d} {OGR.OP_NAMES[og.nodes[v].op]:12s} d{k:5s} dev-vs-bf16: {st(a, gb[k][v])} | bf16-vs-f64: {st(gb[k][v], gf[k][v])}")
