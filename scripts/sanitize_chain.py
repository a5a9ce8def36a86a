"""One small checkpointed step of the chain for compute-sanitizer (memcheck / racecheck /
synccheck): C1 (f32, SIMT path) or a bf16 chain with the bench's plan (sqrt + A24 overlapped
recompute, fused Block kernels, dW stream), eager (no CUDA graph) so every launch is checked."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
n, B, d, dt = (16, 8, 64, "f32") if cfg == "c1" else (40, 256, 512, "bf16")
inp = synth.chain_inputs(n, B, d, dtype=dt, seed=3)
wdt = torch.bfloat16 if dt == "bf16" else torch.float32
p = dict(W=torch.tensor(inp["W"]).to(wdt).cuda(), b=torch.tensor(inp["b"]).cuda(),
         gamma=torch.tensor(inp["gamma"]).cuda(), beta=torch.tensor(inp["beta"]).cuda())
g = {k: torch.empty_like(v) for k, v in p.items()}
model = slm.ChainModel(p, g, dtype=dt, batch=B, use_graph=0)
af = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | (slm.ALLOC_MIRROR_PARITY if dt == "bf16" else 0)
plan = slm.Plan(slm.Graph.chain(n, B, d), "sqrt", alloc_flags=af)
loss = model.step(plan, torch.tensor(inp["x0"]).cuda(), torch.tensor(inp["labels"]).cuda())
torch.cuda.synchronize()
print(cfg, "loss", float(loss.item()), "overlap", model.get_option("last_overlap"))
