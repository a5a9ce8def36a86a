"""One eager LSTM step (no CUDA graph) at C3 widths and a short unroll: under ncu, the duration
of every forward run kernel launch (16-step runs) and of the input projections."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1604_06174_b200 as slm  # noqa: E402

L, T, B, H, I, C = int(os.environ.get("L", 4)), int(os.environ.get("T", 64)), 64, 1024, 50, 5000
dev = torch.device("cuda", 0)
p, g, x, y = bench.lstm_inputs_dev(L, T, B, H, I, C, dev)
graph = slm.Graph.lstm(L, T, B, H, I)
plan = slm.Plan(graph, "none", alloc_flags=7)
opts = {k: int(v) for k, v in (kv.split("=") for kv in sys.argv[1:])}
model = slm.LstmModel(p, g, L, T, B, H, I, C, use_graph=0, **opts)
bufs = model.buffers(plan, dev)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(2):
        loss = model.step(plan, x, y, stream=st, bufs=bufs)
torch.cuda.synchronize()
print("loss", float(loss))
