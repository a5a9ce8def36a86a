"""Micro-benchmark of the block GEMMs at the C2 shape through slm_debug_gemm.

Each configuration is captured into a CUDA graph of `reps` launches cycling over `nw`
distinct weight matrices (nw * 8 MiB > L2, so W streams from HBM as in the step) and timed
with CUDA events.  Prints us/launch and TFLOP/s."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402


def bench(kind, impl, bn, split=1, M=2048, N=256, K=2048, nw=48, reps=96, check=True):
    dev = "cuda"
    if kind == 0:      # A = W [M][K], B = act [N][K]
        As = [torch.randn(M, K, device=dev).bfloat16() for _ in range(nw)]
        B = torch.randn(N, K, device=dev).bfloat16()
        out = torch.empty(split, N, M, device=dev)
        resid = torch.randn(N, M, device=dev)
        bias = torch.randn(M, device=dev)
    elif kind == 1:    # A = W [K][M], B = g [N][K]
        As = [torch.randn(K, M, device=dev).bfloat16() for _ in range(nw)]
        B = torch.randn(N, K, device=dev).bfloat16()
        out = torch.empty(split, N, M, device=dev)
        resid = bias = None
    else:              # dW: A = act [K][M], B = g [K][N], out [N][M]
        M, N, K = 2048, 2048, 256
        As = [torch.randn(K, M, device=dev).bfloat16() for _ in range(nw)]
        B = torch.randn(K, N, device=dev).bfloat16()
        out = torch.empty(N, M, device=dev, dtype=torch.bfloat16)
        resid = bias = None
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(2):
            slm.debug_gemm(kind, impl, bn, M, N, K, As[i], B, out, resid, bias, stream=s, split=split)
    torch.cuda.synchronize()
    err = None
    if check and impl in (0, 4):
        # correctness of this configuration against torch (fp32 reference)
        i = 1
        if kind == 0:
            ref = B.float() @ As[i].float().T + (resid + bias if split == 1 else 0)
        elif kind == 1:
            ref = B.float() @ As[i].float()
        else:
            ref = B.float().T @ As[i].float()
        o = out.float().sum(0) if kind < 2 else out.float()
        err = ((o - ref).norm() / ref.norm()).item()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            slm.debug_gemm(kind, impl, bn, M, N, K, As[i % nw], B, out, resid, bias, stream=s, split=split)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (3 * reps)
    tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
    return us, tf, err


if __name__ == "__main__":
    cfgs = [(0, 0, 32, 1), (0, 0, 64, 1), (0, 0, 64, 2), (0, 0, 128, 2), (0, 0, 128, 4), (0, 0, 256, 4),
            (0, 0, 256, 8), (1, 0, 64, 2), (1, 0, 128, 4), (1, 0, 256, 8), (2, 0, 256, 1),
            (0, 2, 128, 4), (0, 2, 256, 8)]
    if len(sys.argv) > 1:
        cfgs = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
    for c in cfgs:
        kind, impl, bn = c[:3]
        split = c[3] if len(c) > 3 else 1
        kw = {}
        if len(c) > 4:
            kw["K"] = c[4]
        us, tf, err = bench(kind, impl, bn, split, **kw)
        print(f"kind={kind} impl={impl} bn={bn:3d} split={split} {kw}: {us:8.2f} us/launch  {tf:7.1f} TFLOP/s  "
              f"relerr={err}", flush=True)
