"""A lowering option against the default on the same chain and inputs (usage: opt_ab_check.py KEY=V):
prints whether the loss and every gradient are bit-identical (the option changes data movement only)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402

key, val = sys.argv[1].split("=")
n, B, d = int(os.environ.get("N", 12)), 256, int(os.environ.get("D", 2048))
dev = torch.device("cuda", 0)
inp = synth.chain_inputs_torch(n, B, d, dtype="bf16", device=dev)
params = {k: inp[k] for k in ("W", "b", "gamma", "beta")}
res = {}
for v in (0, int(val)):
    grads = {k: torch.empty_like(p) for k, p in params.items()}
    model = slm.ChainModel(params, grads, dtype="bf16", batch=B, **{key: v})
    plan = slm.Plan(slm.Graph.chain(n, B, d), "sqrt", alloc_flags=slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_MIRROR_PARITY)
    for _ in range(3):
        loss = model.step(plan, inp["x0"], inp["labels"])
    torch.cuda.synchronize()
    res[v] = (loss.item(), {k: g.float().cpu().numpy() for k, g in grads.items()})
a, b = res[0], res[int(val)]
print(key, val, "loss", a[0], b[0], "bitwise" if a[0] == b[0] else "DIFF")
for k in a[1]:
    print(" ", k, "bitwise" if np.array_equal(a[1][k], b[1][k]) else f"rel {np.linalg.norm(a[1][k] - b[1][k]) / np.linalg.norm(a[1][k]):.3e}")
