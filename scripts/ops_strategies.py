"""SURVEY 8(f) f1 on the GPU: the paper's strategy comparison (Sec. 5.1, Fig. 5/6)
on the op-granularity pre-activation network (BN, ReLU, FC, Add nodes), executed by the op-graph
executor: per strategy the plan's exact activation memory, the measured pool, the re-computed
forward ops and the step time (CUDA graph replays, device events), with the loss bit-identical
across plans.  Prints one JSON object."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402

depths = [int(x) for x in os.environ.get("DEPTHS", "16,16,16").split(",")]
widths = [int(x) for x in os.environ.get("WIDTHS", "512,1024,2048").split(",")]
B = int(os.environ.get("B", 256))
steps = int(os.environ.get("STEPS", 10))
CONV = int(os.environ.get("CONV", 0))   # 1: the convolutional ResNet of SURVEY 8(f) f4 (HW, DEPTHS, WIDTHS)
HW = int(os.environ.get("HW", 32))
dev = torch.device("cuda", 0)
shapes = None
if CONV:
    nodes, shapes = slm.OpsModel.preact_conv_nodes(B, HW, list(zip(widths, depths)), 128)
else:
    nodes = slm.OpsModel.preact_nodes(depths, widths, B)
inp = synth.opgraph_inputs(nodes, B, seed=11, shapes=shapes)
params, grads = {}, {}
for v, pv in inp["params"].items():
    params[v] = {k: torch.tensor(a, device=dev, dtype=torch.bfloat16 if k == "W" else torch.float32) for k, a in pv.items()}
    grads[v] = {k: torch.zeros_like(t) for k, t in params[v].items()}
x = torch.tensor(inp["x0"], device=dev)
y = torch.tensor(inp["labels"], device=dev)
graph = slm.Graph.from_nodes(nodes, [len(nodes) - 1])
model = slm.OpsModel(graph, params, grads, B, shapes=shapes)
# the paper's five strategies (Fig. 5): no optimisation, in-place, sharing, drop bn-relu, sublinear
strategies = [("no-opt", "none", 0), ("inplace", "none", 1), ("sharing", "none", 3),
              ("drop bn-relu", "drop_cheap", 3), ("sublinear (sqrt)", "sqrt", 3), ("sublinear (search)", "search", 3)]
out = dict(graph=dict(depths=depths, widths=widths, batch=B, nodes=len(nodes), conv=CONV, hw=HW if CONV else None),
           strategies={})
ref = None
for name, strat, af in strategies:
    plan = slm.Plan(graph, strat, alloc_flags=af)
    pool, ws, loss = model.buffers(plan, dev)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            model.step(plan, x, y, stream=st, bufs=(pool, ws, loss))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        for _ in range(steps):
            model.step(plan, x, y, stream=st, bufs=(pool, ws, loss))
    e1.record(st)
    torch.cuda.synchronize()
    lv = float(loss.item())
    if ref is None:
        ref = lv
    out["strategies"][name] = dict(plan=strat, alloc_flags=af, exact_peak_mb=round(plan.exact_peak / 2**20, 2),
                                   pool_mb=round(plan.pool_bytes / 2**20, 2), extra_forward=plan.extra_forward,
                                   ms_per_step=round(e0.elapsed_time(e1) / steps, 3), loss=lv,
                                   loss_equal_to_no_opt=lv == ref)
print(json.dumps(out, indent=1))
