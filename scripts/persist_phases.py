"""Phase breakdown of the persistent forward kernel (fwd_persist.cuh) from per-layer, per-CTA
%globaltimer stamps (model option persist_dbg): one no-checkpoint step of an n-layer chain, the
forward run of n <= 64 Blocks is one launch.  Prints the median over layers of
(phase k stamp, min/median/max over CTAs) relative to the layer's earliest start."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402

PH = ["start", "accum", "epi_done", "bar1", "bn_done", "bar2"]

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=64)
ap.add_argument("--width", type=int, default=2048)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--opt", action="append", default=[])
a = ap.parse_args()
n, B, d = a.layers, a.batch, a.width
dev = torch.device("cuda", 0)
inp = synth.chain_inputs_torch(n, B, d, dtype="bf16", device=dev)
params = {k: inp[k] for k in ("W", "b", "gamma", "beta")}
grads = {k: torch.empty_like(v) for k, v in params.items()}
opts = dict(kv.split("=") for kv in a.opt)
model = slm.ChainModel(params, grads, dtype="bf16", batch=B, use_graph=0, **{k: int(v) for k, v in opts.items()})
plan = slm.Plan(slm.Graph.chain(n, B, d), "none")
ts = torch.zeros(n * 160 * 8, dtype=torch.int64, device=dev)
model.set_option("profile_ts_buffer", ts.data_ptr())
for _ in range(3):
    model.step(plan, inp["x0"], inp["labels"])
torch.cuda.synchronize()
model.set_option("persist_dbg", 1)
model.step(plan, inp["x0"], inp["labels"])
torch.cuda.synchronize()
model.set_option("persist_dbg", 0)
model.set_option("profile_ts_buffer", 0)
S = next(s for s in (16, 8, 4) if (d // 128) * s <= 148 and d % (s * 64) == 0 and 64 <= d // s <= 256)
ncta = d // 128 * S
t = ts[:n * ncta * 8].view(n, ncta, 8).cpu().double()[:, :, :6]
rows = []
for j in range(1, n - 1):
    t0 = t[j, :, 0].min()
    rows.append((t[j] - t0) / 1e3)
r = torch.stack(rows)   # [layers, cta, phase] us
print(f"n={n} d={d} B={B} CTAs={ncta}; per-layer us relative to the layer's first CTA start (median over layers)")
for k, name in enumerate(PH):
    mn = r[:, :, k].min(1).values.median().item()
    md = r[:, :, k].median(1).values.median().item()
    mx = r[:, :, k].max(1).values.median().item()
    print(f"  {name:9s} min {mn:7.3f}  med {md:7.3f}  max {mx:7.3f}")
lay = (t[2:n - 1, :, 0].min(1).values - t[1:n - 2, :, 0].min(1).values) / 1e3
print(f"layer period: median {lay.median().item():.3f} us")
