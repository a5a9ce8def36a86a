"""Diagnostics for the fused Block kernel (blk_fused.cuh), run on the GPU box:
  parity  per-layer / per-tensor error breakdown vs the oracle (relative L2, element-wise
          violations of |g - r| <= tol (|r| + rms r), and where they sit), for the fused path
          (impl 0) and the SIMT path (impl 1) on the same inputs
  prof    one eager step (no CUDA graph) of a C2-width chain, for `ncu -k regex:blk_kernel`
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402
from oracle import chain as OC  # noqa: E402


def run(inp, n, B, d, strategy="sqrt", **opt):
    p = dict(W=torch.tensor(inp["W"]).bfloat16().cuda(), b=torch.tensor(inp["b"]).cuda(),
             gamma=torch.tensor(inp["gamma"]).cuda(), beta=torch.tensor(inp["beta"]).cuda())
    g = {k: torch.zeros_like(v) for k, v in p.items()}
    m = slm.ChainModel(p, g, dtype="bf16", batch=B, **opt)
    plan = slm.Plan(slm.Graph.chain(n, B, d), strategy)
    loss = m.step(plan, torch.tensor(inp["x0"]).cuda(), torch.tensor(inp["labels"]).cuda())
    torch.cuda.synchronize()
    return loss.item(), {k: v.float().cpu().numpy().astype(np.float64) for k, v in g.items()}


def parity(n, B, d, seed):
    from _util import margin_inputs
    inp = margin_inputs(n, B, d, "bf16", seed=seed)
    ol, og, _ = OC.step_plain(OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"]), inp["x0"], inp["labels"],
                              "bf16")
    res = {}
    for impl in (0, 1):
        loss, g = run(inp, n, B, d, gemm_impl=impl)
        res[impl] = g
        print(f"== n={n} B={B} d={d} impl {impl}: loss {loss:.8f} oracle {ol:.8f}")
        for k in og:
            r = og[k]
            rms = np.sqrt(np.mean(r * r))
            for l in range(n):
                e = np.abs(g[k][l] - r[l])
                bad = e > 2e-2 * (np.abs(r[l]) + rms)
                rel = np.linalg.norm(g[k][l] - r[l]) / max(np.linalg.norm(r[l]), 1e-30)
                line = f"  {k:5s} l={l} rel {rel:.2e} bad {int(bad.sum()):6d} max_ratio {np.max(e / (2e-2 * (np.abs(r[l]) + rms))):.2f}"
                if k == "W" and bad.any():
                    rows, cols = np.nonzero(bad)
                    line += (f" rows {np.unique(rows // 32)} (blk32) cols {np.unique(cols // 32)} (blk32)"
                             f" rowmod {np.bincount(rows % 8, minlength=8)}")
                print(line)
    for k in og:
        print(f"impl0 vs impl1 {k}: rel {np.linalg.norm(res[0][k] - res[1][k]) / np.linalg.norm(res[1][k]):.2e}")


def prof(n, B, d):
    inp_t = synth.chain_inputs_torch(n, B, d, dtype="bf16", seed=1)
    p = {k: inp_t[k] for k in ("W", "b", "gamma", "beta")}
    g = {k: torch.zeros_like(v) for k, v in p.items()}
    m = slm.ChainModel(p, g, dtype="bf16", batch=B, use_graph=0)
    plan = slm.Plan(slm.Graph.chain(n, B, d), "none")
    for _ in range(2):
        m.step(plan, inp_t["x0"], inp_t["labels"])
    torch.cuda.synchronize()
    print("prof done")


def depth(B, d, *ns):
    """relative L2 error of the loss / grads vs depth n for the fused path (impl 0), the SIMT path
    (impl 1) and between them: separates a kernel bug (one path off) from the decision chaos of
    a bf16 chain with ReLU (both paths drifting from the oracle alike)."""
    for n in ns:
        inp = synth.chain_inputs(n, B, d, dtype="bf16", seed=16)
        ol, og, _ = OC.step_plain(OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"]), inp["x0"], inp["labels"],
                                  "bf16")
        r = {}
        for impl in (0, 1):
            r[impl] = run(inp, n, B, d, "none", gemm_impl=impl)
        line = f"n={n:3d} B={B} d={d}:"
        for k in ("W", "gamma", "beta", "b"):
            e0 = np.linalg.norm(r[0][1][k] - og[k]) / np.linalg.norm(og[k])
            e1 = np.linalg.norm(r[1][1][k] - og[k]) / np.linalg.norm(og[k])
            e01 = np.linalg.norm(r[0][1][k] - r[1][1][k]) / np.linalg.norm(og[k])
            line += f"  {k}: fused {e0:.1e} simt {e1:.1e} fused-simt {e01:.1e}"
        print(line, flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "parity":
        parity(*[int(a) for a in sys.argv[2:6]])
    elif sys.argv[1] == "depth":
        depth(*[int(a) for a in sys.argv[2:]])
    else:
        prof(*[int(a) for a in sys.argv[2:5]])
