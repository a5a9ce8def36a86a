"""Which gradients differ between the plain and a checkpointed LSTM step (debug), per option set;
and the per-step device-clock phases of the forward run kernels (option lstm_run_ts)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1604_06174_b200 as slm  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)


def run(cfg, strategy, m=None, **opt):
    L, T, B, H, I, C = cfg
    p, g, x, y = bench.lstm_inputs_dev(L, T, B, H, I, C, dev)
    model = slm.LstmModel(p, g, L, T, B, H, I, C, **opt)
    graph = slm.Graph.lstm(L, T, B, H, I)
    plan = slm.Plan(graph, "explicit" if m is not None else strategy, m=m, alloc_flags=3)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        loss = model.step(plan, x, y, stream=s)
        loss = model.step(plan, x, y, stream=s)
    torch.cuda.synchronize()
    return float(loss.item()), {k: v.cpu().numpy().astype(np.float64) for k, v in g.items()}


if os.environ.get("BITDIFF", "1") == "1":
    cfg = (2, 8, 64, 128, 50, 300)
    for opts in ({}, {"lstm_fuse_runs": 0}, {"lstm_streams": 0}, {"lstm_fuse_runs": 0, "lstm_streams": 0}):
        l0, g0 = run(cfg, "none", **opts)
        for st in ("sqrt", "search", "drop_cheap"):
            l1, g1 = run(cfg, st, **opts)
            bad = {k: float(np.abs(g1[k] - g0[k]).max()) for k in g0 if not np.array_equal(g0[k], g1[k])}
            print(opts, st, "loss eq", l0 == l1, "differs:", bad, flush=True)
# forward run phases at C3 widths
L, T, B, H, I, C = 4, 64, 64, 1024, 50, 5000
p, g, x, y = bench.lstm_inputs_dev(L, T, B, H, I, C, dev)
model = slm.LstmModel(p, g, L, T, B, H, I, C, use_graph=0)
plan = slm.Plan(slm.Graph.lstm(L, T, B, H, I), "none", alloc_flags=7)
nr = 64
ts = torch.zeros(nr * 16 * 16, dtype=torch.int64, device=dev)
model.set_option("lstm_run_ts", ts.data_ptr())
model.set_option("lstm_run_ts_n", nr)
bufs = model.buffers(plan, dev)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(2):
        model.step(plan, x, y, stream=s, bufs=bufs)
torch.cuda.synchronize()
t = ts.view(nr, 16, 16).cpu().numpy().astype(np.float64)
names = {1: "mma issued", 2: "accum", 4: "tmem ld", 5: "x ready", 6: "acts", 7: "bar1", 8: "cell", 9: "fence", 10: "bar2", 3: "released"}
bnames = {2: "accum", 4: "exchanged", 8: "cell", 3: "released"}
for r in range(nr):
    v = t[r]
    ok = v[:, 3] > 0
    v = v[ok]
    if len(v) < 2:
        continue
    bwd = v[0, 1] == 0   # the forward run stamps k = 1 (MMA issued), the backward run does not
    step = np.abs(np.diff(v[:, 3])).mean()
    ref = v[:, 0]
    if bwd:
        if r % 4 == 0 or r > nr - 5:
            print(f"bwd run {r}: steps {ok.sum()} period {step / 1e3:.2f} us; from the barrier: " +
                  "  ".join(f"{bnames[k]} {np.mean(v[1:, k] - ref[1:]) / 1e3:.2f}" for k in (2, 4, 8, 3)))
    elif r < 4:
        print(f"fwd run {r}: steps {ok.sum()} period {step / 1e3:.2f} us; from the barrier: " +
              "  ".join(f"{names[k]} {np.mean(v[:, k] - ref) / 1e3:.2f}" for k in (1, 2, 4, 5, 6, 7, 8, 9, 10, 3)))
