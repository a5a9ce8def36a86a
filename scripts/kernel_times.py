"""Event-timed per-kind kernel durations of the chain step (profile_events=1: an event pair
around every kernel, eager launches, no CUDA graph) at the bench configuration."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402

n, B, d = int(sys.argv[1]) if len(sys.argv) > 1 else 256, 256, 2048
opts = dict(kv.split("=") for kv in sys.argv[2:])
t = synth.chain_inputs_torch(n, B, d, dtype="bf16")
p = {k: t[k] for k in ("W", "b", "gamma", "beta")}
g = {k: torch.empty_like(v) for k, v in p.items()}
m = slm.ChainModel(p, g, dtype="bf16", batch=B, **{k: int(v) for k, v in opts.items()})
plan = slm.Plan(slm.Graph.chain(n, B, d), "sqrt")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    m.step(plan, t["x0"], t["labels"], stream=s)
torch.cuda.synchronize()
m.set_option("profile_events", 1)
m.kernel_times(reset=True)
with torch.cuda.stream(s):
    for _ in range(3):
        m.step(plan, t["x0"], t["labels"], stream=s)
torch.cuda.synchronize()
kt = m.kernel_times(reset=True)
for k, (ms, c) in kt.items():
    if c:
        print(f"{k:10s} n={c:6d} avg={1e3 * ms / c:8.2f} us total/step={ms / 3:8.2f} ms")
