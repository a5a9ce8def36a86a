import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1604_06174_b200 as slm
import synth
from test_gpu_lstm import _dev

cfg = tuple(int(x) for x in os.environ.get("CFG", "1,2,256,128,7,128").split(","))
L, T, B, H, I, C = cfg
inp = synth.lstm_inputs(L, T, B, H, I, C, dtype="bf16", seed=T + B)
for optstr in sys.argv[1:]:
    opts = {k: int(v) for k, v in (kv.split("=") for kv in optstr.split(","))} if optstr else {}
    vals = []
    for rep in range(8):
        p, g, x, y = _dev(inp, L, H, C)
        model = slm.LstmModel(p, g, L, T, B, H, I, C, **opts)
        plan = slm.Plan(slm.Graph.lstm(L, T, B, H, I), "none")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            loss = model.step(plan, x, y, stream=s)
            l1 = loss.clone()
            loss = model.step(plan, x, y, stream=s)
        torch.cuda.synchronize()
        vals.append((round(l1.item(), 7), round(loss.item(), 7)))
    print(optstr, len(set(vals)), vals[:4], flush=True)
