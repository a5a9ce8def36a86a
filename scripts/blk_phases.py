"""Per-phase device-clock breakdown of the fused Block kernel (slm_debug_block with per-CTA
%globaltimer stamps): phase 0 start, 1 griddepcontrol.wait returned (producer), 2 accumulator ready,
3 own quarter-slices staged and stored (all warps), 4 incoming slices + x landed, 5 first BN pass
done, 7 end.  Prints the median and max over CTAs of each phase's time since the earliest start."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1604_06174_b200 as slm  # noqa: E402


def run(bwd, B, d, reps=5, cfg=0):
    S = 4 if d % 256 == 0 else 2
    W = (torch.randn(d, d, device="cuda") / d ** 0.5).bfloat16()
    opnd = torch.randn(B, d, device="cuda").bfloat16()
    x, g = torch.randn(B, d, device="cuda"), torch.randn(B, d, device="cuda")
    vec = [torch.randn(d, device="cuda") for _ in range(3)]
    out = torch.empty(B, d, device="cuda")
    a, gq = torch.empty(B, d, device="cuda", dtype=torch.bfloat16), torch.empty(B, d, device="cuda", dtype=torch.bfloat16)
    dd = [torch.empty(d, device="cuda") for _ in range(3)]
    P = torch.empty(4 * B * d, device="cuda")
    BM = 128 if (B == 256 and cfg in (0, 2, 4)) else 64
    if cfg == 3:
        S = 2
    ncta = d // BM * S
    ts = torch.zeros(ncta * 8, dtype=torch.int64, device="cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    slm.check(slm.lib.slm_debug_timestamps(p(ts)))
    res = []
    for r in range(reps):
        ts.zero_()
        # flush L2 so W comes from HBM as in the chain (8.6 GB of weights)
        torch.empty(256 << 20, dtype=torch.uint8, device="cuda").fill_(1)
        slm.check(slm.lib.slm_debug_block(bwd, B, d, p(W), p(opnd), p(x), p(g), p(vec[0]), p(vec[1]), p(vec[2]),
                                          p(out), p(a), p(gq), p(dd[0]), p(dd[1]), p(dd[2]), p(P), 1 | (cfg << 4), st))
        torch.cuda.synchronize()
        t = ts.view(ncta, 8).cpu().numpy().astype(np.float64)
        t0 = t[:, 0].min()
        res.append((t - t0) / 1000.0)
    slm.check(slm.lib.slm_debug_timestamps(None))
    r = np.median(np.stack(res[1:]), axis=0)
    print(f"{os.environ.get('SLM_LIB', 'libslm.so')} cfg={cfg} {'bwd' if bwd else 'fwd'} B={B} d={d} S={S} ({ncta} CTAs): phase median / max us:",
          " | ".join(f"{i}:{np.median(r[:, i]):.2f}/{r[:, i].max():.2f}" for i in range(8)))


if __name__ == "__main__":
    cfgs = [int(c) for c in sys.argv[1:]] or [0]
    for cfg in cfgs:
        for bwd in (0, 1):
            run(bwd, 256, 2048, cfg=cfg)
