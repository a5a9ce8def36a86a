#!/usr/bin/env python
"""The metric's "vs n" axis (BASELINE.json: samples/sec + peak activation GB vs n, ckpt vs
no-ckpt) and the C4 points executed on the GPU: the C2 chain (d=2048, B=256, bf16) at
n in {64, 256, 1024, 4096} with the sqrt(n) plan and without checkpointing, plus, at n=1024,
the App. A search, the recursive k=1,2 plans and Alg. 3 budget points -- measured step time
and activation memory next to the plan's exact peak and re-computation count.

    python scripts/sweep_n.py [--out profiles/r1_vs_n]      (GPU box)
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402

B, D = 256, 2048


def measure(model, plan, x0, y, steps=5, warmup=3):
    dev = x0.device
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    bufs = model.buffers(plan, dev)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(warmup):
            model.step(plan, x0, y, stream=st, bufs=bufs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        for _ in range(steps):
            loss = model.step(plan, x0, y, stream=st, bufs=bufs)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    act = torch.cuda.max_memory_allocated(dev) - base
    model._bufs.clear()
    del bufs
    torch.cuda.empty_cache()
    return dict(ms_per_step=round(ms, 3), samples_per_s=round(B / (ms / 1e3), 1),
                plan_exact_peak_gb=round(plan.exact_peak / 1e9, 4), pool_gb=round(plan.pool_bytes / 1e9, 4),
                measured_activation_gb=round(act / 1e9, 4), extra_forward=plan.extra_forward,
                loss=float(loss.item()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_vs_n"))
    ap.add_argument("--ns", default="64,256,1024,4096")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    rows = []
    for n in [int(v) for v in a.ns.split(",")]:
        t = synth.chain_inputs_torch(n, B, D, dtype="bf16", device=dev)
        p = {k: t[k] for k in ("W", "b", "gamma", "beta")}
        g = {k: torch.empty_like(v) for k, v in p.items()}
        model = slm.ChainModel(p, g, dtype="bf16", batch=B)
        graph = slm.Graph.chain(n, B, D)
        par = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_MIRROR_PARITY
        plans = [("none", slm.Plan(graph, "none")), ("sqrt", slm.Plan(graph, "sqrt")),
                 ("sqrt + A24 (overlapped recompute)", slm.Plan(graph, "sqrt", alloc_flags=par))]
        if n == 1024:
            plans += [("search (App. A) + A24", slm.Plan(graph, "search", alloc_flags=par)),
                      ("search (App. A)", slm.Plan(graph, "search")),
                      ("recursive k=1", slm.Plan(graph, "recursive", k=1)),
                      ("recursive k=2", slm.Plan(graph, "recursive", k=2))]
            u = B * D * 4
            for mult in (16, 48, 128):
                plans.append((f"budget {mult}u", slm.Plan(graph, "budget", budget=mult * u)))
        for name, plan in plans:
            r = dict(n=n, plan=name, **measure(model, plan, t["x0"], t["labels"]))
            print(json.dumps(r), flush=True)
            rows.append(r)
        del model, g, p, t
        torch.cuda.empty_cache()
    with open(a.out + ".json", "w") as f:
        json.dump(dict(config=f"chain d={D} B={B} bf16, one B200", rows=rows), f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# samples/s and activation memory vs n (chain d={D}, B={B}, bf16, one B200)\n\n")
        f.write("| n | plan | ms/step | samples/s | plan exact peak GB | measured activation GB | extra fwd | ckpt/no-ckpt time |\n")
        f.write("|---|---|---|---|---|---|---|---|\n")
        base = {r["n"]: r["ms_per_step"] for r in rows if r["plan"] == "none"}
        for r in rows:
            f.write(f"| {r['n']} | {r['plan']} | {r['ms_per_step']} | {r['samples_per_s']} | {r['plan_exact_peak_gb']} | "
                    f"{r['measured_activation_gb']} | {r['extra_forward']} | {r['ms_per_step'] / base[r['n']]:.3f} |\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
