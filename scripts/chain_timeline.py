"""Device-clock timeline of the chain step's GEMM launches (profile_ts + slm_debug_ts_meta):
forward-phase / backward-phase spans, per-kind busy time, and the gap between consecutive
GEMMs of the same kind (the BN kernel + launch share of each Block on that chain)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402

n, B, d = int(os.environ.get("N", 1024)), 256, 2048
mp = int(os.environ.get("MP", 1))
dev = torch.device("cuda", 0)
inp = synth.chain_inputs_torch(n, B, d, dtype="bf16", device=dev)
params = {k: inp[k] for k in ("W", "b", "gamma", "beta")}
grads = {k: torch.empty_like(v) for k, v in params.items()}
opts = {k: int(v) for k, v in (kv.split("=") for kv in sys.argv[1:])}
model = slm.ChainModel(params, grads, dtype="bf16", batch=B, **opts)
af = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | (slm.ALLOC_MIRROR_PARITY if mp else 0)
plan = slm.Plan(slm.Graph.chain(n, B, d), os.environ.get("STRATEGY", "sqrt"), alloc_flags=af)
ngemm = 3 * n + plan.extra_forward
PH = int(os.environ.get("PHASES", 0))   # 1: all 8 phase stamps of every CTA (profile_ts_dep = 2)
W8 = 8 if PH else 2
ts = torch.zeros(ngemm * 1024 * W8, dtype=torch.int64, device=dev)
model.set_option("profile_ts", ngemm)
model.set_option("profile_ts_buffer", ts.data_ptr())
if PH:
    model.set_option("profile_ts_dep", 2)
st = torch.cuda.Stream()
bufs = model.buffers(plan, dev)
with torch.cuda.stream(st):
    for _ in range(3):
        model.step(plan, inp["x0"], inp["labels"], stream=st, bufs=bufs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
with torch.cuda.stream(st):
    model.step(plan, inp["x0"], inp["labels"], stream=st, bufs=bufs)
e1.record(st)
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1)
kind = (C.c_int32 * ngemm)()
aux = (C.c_int32 * ngemm)()
nn = C.c_int32()
slm.check(slm.lib.slm_debug_ts_meta(model._h, kind, aux, ngemm, C.byref(nn)))
t = ts.view(ngemm, 1024, W8).cpu().numpy()[:nn.value].astype(np.float64)
t[t == 0] = np.nan
s0 = np.nanmin(t[:, :, 0], axis=1)
s1 = np.nanmax(t[:, :, W8 - 1], axis=1)
if PH:   # per kind: median over launches of the median over CTAs of (phase_i - the launch's first start)
    kk_ = np.array(kind[:nn.value])
    for kv, nm in ((1, "fwd Block"), (2, "dX Block"), (3, "dW GEMM")):
        sel = np.where(kk_ == kv)[0]
        if not len(sel):
            continue
        rel = (t[sel] - s0[sel, None, None]) / 1e3
        med = np.nanmedian(np.nanmedian(rel, axis=1), axis=0)
        print(f"  phases {nm:10s} (us from launch start): " + " ".join(f"{i}:{med[i]:.2f}" for i in range(8)))
T0 = np.nanmin(s0)
s0, s1 = (s0 - T0) / 1e3, (s1 - T0) / 1e3
k = np.array(kind[:nn.value])
names = {1: "fwd", 2: "dx", 3: "dw"}
print(f"n={n} plan={os.environ.get('STRATEGY', 'sqrt')} mirror_parity={mp} opts={opts}: step {step_ms:.2f} ms (event), "
      f"last GEMM end {np.nanmax(s1) / 1e3:.2f} ms after the first start")
fwd = np.where(k == 1)[0]
nf = n   # the first n forward GEMMs are the forward pass
print(f"  forward pass: {s1[fwd[nf - 1]] / 1e3:.2f} ms ({(s1[fwd[nf - 1]] - s0[fwd[0]]) / nf:.2f} us/Block)")
dx = np.where(k == 2)[0]
print(f"  backward phase: {(s1[dx[-1]] - s0[dx[0]]) / 1e3:.2f} ms ({(s1[dx[-1]] - s0[dx[0]]) / len(dx):.2f} us/Block)")
for kk, nm in names.items():
    idx = np.where(k == kk)[0]
    if nm == "fwd":
        for part, sel in (("fwd (forward pass)", idx[:nf]), ("fwd (mirrors)", idx[nf:])):
            if len(sel) < 2:
                continue
            dur = s1[sel] - s0[sel]
            gap = s0[sel[1:]] - s1[sel[:-1]]
            print(f"  {part:20s} n={len(sel):5d} span med {np.median(dur):6.2f} us  gap to next med {np.median(gap):6.2f} us"
                  f"  period med {np.median(np.diff(s0[sel])):6.2f} us")
        continue
    dur = s1[idx] - s0[idx]
    gap = s0[idx[1:]] - s1[idx[:-1]]
    print(f"  {nm:20s} n={len(idx):5d} span med {np.median(dur):6.2f} us  gap to next med {np.median(gap):6.2f} us"
          f"  period med {np.median(np.diff(s0[idx])):6.2f} us")
