"""Per-layer error breakdown of the GPU chain step vs the oracle and a torch fp32 reference."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402
from oracle import chain as OC  # noqa: E402


def run(n, B, d, dtype, strategy="none", **opt):
    inp = synth.chain_inputs(n, B, d, dtype=dtype)
    wdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    p = dict(W=torch.tensor(inp["W"]).to(wdt).cuda(), b=torch.tensor(inp["b"]).cuda(),
             gamma=torch.tensor(inp["gamma"]).cuda(), beta=torch.tensor(inp["beta"]).cuda())
    g = {k: torch.zeros_like(v) for k, v in p.items()}
    m = slm.ChainModel(p, g, dtype=dtype, batch=B, **opt)
    plan = slm.Plan(slm.Graph.chain(n, B, d), strategy)
    loss = m.step(plan, torch.tensor(inp["x0"]).cuda(), torch.tensor(inp["labels"]).cuda())
    torch.cuda.synchronize()
    ol, og, odx = OC.step_plain(OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"]), inp["x0"],
                                inp["labels"], "bf16" if dtype == "bf16" else "f64")
    print(f"== {dtype} n={n} B={B} d={d} {strategy} {opt}: loss gpu {loss.item():.8f} oracle {ol:.8f}")
    for k in og:
        gg = g[k].float().cpu().numpy().astype(np.float64)
        per = [np.linalg.norm(gg[l] - og[k][l]) / max(np.linalg.norm(og[k][l]), 1e-30) for l in range(n)]
        print(f"  {k:6s} total {np.linalg.norm(gg - og[k]) / np.linalg.norm(og[k]):.2e}  per-layer",
              " ".join(f"{x:.1e}" for x in per))


if __name__ == "__main__":
    run(16, 8, 64, "f32")
    run(4, 8, 64, "f32")
    run(2, 64, 128, "f32")
    run(8, 64, 256, "bf16")
    run(8, 64, 256, "bf16", gemm_impl=1)
