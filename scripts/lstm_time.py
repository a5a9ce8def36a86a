"""Time the C3 LSTM step for several plans and options (CUDA graph replays, events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1604_06174_b200 as slm  # noqa: E402

L, T, B, H, I, C = 4, int(os.environ.get("T", 4096)), 64, 1024, 50, int(os.environ.get("C", 5000))
dev = torch.device("cuda", 0)
p, g, x, y = bench.lstm_inputs_dev(L, T, B, H, I, C, dev)
graph = slm.Graph.lstm(L, T, B, H, I)
AF = int(os.environ.get("ALLOC", 7))
plans = {"seg64": slm.Plan(graph, "explicit", m=graph.lstm_segment_mirrors(64), alloc_flags=AF),
         "none": slm.Plan(graph, "none", alloc_flags=AF)}
for optstr in sys.argv[1:] or ["lstm_streams=1"]:
    opts = dict(kv.split("=") for kv in optstr.split(","))
    model = slm.LstmModel(p, g, L, T, B, H, I, C, **{k: int(v) for k, v in opts.items()})
    for name, plan in plans.items():
        st = torch.cuda.Stream()
        bufs = model.buffers(plan, dev)
        with torch.cuda.stream(st):
            for _ in range(3):
                model.step(plan, x, y, stream=st, bufs=bufs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            for _ in range(3):
                model.step(plan, x, y, stream=st, bufs=bufs)
        e1.record(st)
        torch.cuda.synchronize()
        print(f"{optstr:40s} {name:6s} {e0.elapsed_time(e1) / 3:9.2f} ms", flush=True)
        model._bufs.clear()
    del model
    torch.cuda.empty_cache()
