"""One LSTM training step at a small unroll for profiling: W untimed steps then one step
(CUDA graph off so ncu sees every launch).  usage: python scripts/lstm_step.py T W"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1604_06174_b200 as slm  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
L, B, H, I, C = 4, 64, 1024, 50, 5000
dev = torch.device("cuda", 0)
p, g, x, y = bench.lstm_inputs_dev(L, T, B, H, I, C, dev)
graph = slm.Graph.lstm(L, T, B, H, I)
plan = slm.Plan(graph, "explicit", m=graph.lstm_segment_mirrors(min(32, T)), alloc_flags=7)
model = slm.LstmModel(p, g, L, T, B, H, I, C, use_graph=0)
print("launches per step", model.launches(plan), flush=True)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(W + 1):
        model.step(plan, x, y, stream=st)
torch.cuda.synchronize()
print("done", flush=True)
