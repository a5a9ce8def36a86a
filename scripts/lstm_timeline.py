"""Device-clock timeline of the LSTM step's GEMM and persistent-run launches (profile_ts +
slm_debug_ts_meta): per stream busy time, concurrency and the gaps between consecutive launches."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1604_06174_b200 as slm  # noqa: E402

L, T, B, H, I, Cn = 4, int(os.environ.get("T", 1024)), 64, 1024, 50, 5000
dev = torch.device("cuda", 0)
p, g, x, y = bench.lstm_inputs_dev(L, T, B, H, I, Cn, dev)
graph = slm.Graph.lstm(L, T, B, H, I)
if os.environ.get("PLAN") == "none":
    plan = slm.Plan(graph, "none", alloc_flags=int(os.environ.get("AF", 7)))
else:
    plan = slm.Plan(graph, "explicit", m=graph.lstm_segment_mirrors(int(os.environ.get("SEG", 32))),
                    alloc_flags=int(os.environ.get("AF", 7)))
opts = {k: int(v) for k, v in (kv.split("=") for kv in sys.argv[1:])}
model = slm.LstmModel(p, g, L, T, B, H, I, Cn, **opts)
ngemm = 4 * T * (L + 2) + 64
KIND = {0: 'fwd run', 1: 'gemm fwd', 2: 'gemm dx', 3: 'gemm dw', 4: 'bwd run'}
ts = torch.zeros(ngemm * 1024 * 2, dtype=torch.int64, device=dev)
model.set_option("profile_ts", ngemm)
model.set_option("profile_ts_buffer", ts.data_ptr())
st = torch.cuda.Stream()
bufs = model.buffers(plan, dev)
with torch.cuda.stream(st):
    for _ in range(3):
        model.step(plan, x, y, stream=st, bufs=bufs)
torch.cuda.synchronize()
ts.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
with torch.cuda.stream(st):
    model.step(plan, x, y, stream=st, bufs=bufs)
e1.record(st)
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1)
n = C.c_int32()
slm.lib.slm_debug_ts_meta(model._h, None, None, 0, C.byref(n))
kind = (C.c_int32 * n.value)()
aux = (C.c_int32 * n.value)()
slm.check(slm.lib.slm_debug_ts_meta(model._h, kind, aux, n.value, C.byref(n)))
model.set_option("profile_ts", 0)
t = ts.view(ngemm, 1024, 2)[: n.value].cpu().numpy().astype(np.float64)
starts = np.where(t[:, :, 0] > 0, t[:, :, 0], np.inf).min(1)
ends = t[:, :, 1].max(1)
t0 = starts.min()
s_us, e_us = (starts - t0) / 1e3, (ends - t0) / 1e3
aux = np.array(aux[:])
kinds = np.array(kind[:])
for kd in sorted(set(kinds.tolist())):
    sel = kinds == kd
    print(f"{KIND.get(kd, kd):9s}: {sel.sum():6d} launches, busy {(e_us - s_us)[sel].sum() / 1e3:8.2f} ms, mean {(e_us - s_us)[sel].mean():8.2f} us")
print(f"T={T} step {step_ms:.2f} ms, {n.value} GEMM launches, first..last GEMM {e_us.max() / 1e3:.2f} ms")
streams = sorted(set(aux // 4))
for s in streams:
    sel = aux // 4 == s
    dur = (e_us - s_us)[sel]
    order = np.argsort(s_us[sel])
    ss, ee = s_us[sel][order], e_us[sel][order]
    gaps = ss[1:] - ee[:-1]
    print(f"stream {s}: {sel.sum():6d} GEMMs  busy {dur.sum() / 1e3:8.2f} ms  mean {dur.mean():6.2f} us  "
          f"median gap to next {np.median(gaps):6.2f} us  mean gap {gaps.mean():6.2f} us")
# concurrency: number of GEMMs in flight over time
ev = sorted([(a, 1) for a in s_us] + [(b, -1) for b in e_us])
cur, last, acc = 0, 0.0, np.zeros(16)
for tt, d in ev:
    acc[min(cur, 15)] += tt - last
    cur += d
    last = tt
tot = acc.sum()
print("GEMMs in flight (fraction of time):", {i: round(acc[i] / tot, 3) for i in range(8) if acc[i] > 0})
# phases: forward (kind 0), recompute (1), backward (2): first start .. last end and GEMM busy union
for kd, name in ((0, "forward"), (1, "recompute"), (2, "backward")):
    sel = aux % 4 == kd
    if not sel.any():
        continue
    ss, ee = s_us[sel], e_us[sel]
    order = np.argsort(ss)
    busy, cur_s, cur_e = 0.0, None, None
    for i in order:
        if cur_e is None or ss[i] > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = ss[i], ee[i]
        else:
            cur_e = max(cur_e, ee[i])
    busy += cur_e - cur_s
    print(f"{name:9s}: {sel.sum():6d} GEMMs, first {ss.min() / 1e3:8.2f} ms  last end {ee.max() / 1e3:8.2f} ms  "
          f"GEMM-busy union {busy / 1e3:8.2f} ms")
if os.environ.get("DUMP"):
    # a window of the launch list: start, end (us), stream, kind
    order = np.argsort(s_us)
    lo = float(os.environ.get("DUMP"))
    rows = [(s_us[i], e_us[i], aux[i] // 4, aux[i] % 4, KIND.get(kinds[i], kinds[i])) for i in order if s_us[i] >= lo * 1e3][:int(os.environ.get("DUMPN", 120))]
    for r in rows:
        print(f"{r[0]:10.1f} {r[1]:10.1f} {r[1] - r[0]:8.1f}  stream {r[2]} k{r[3]}  {r[4]}")
