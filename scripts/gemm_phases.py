"""Phase breakdown of one tcgen05 GEMM launch from per-CTA %globaltimer stamps."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_06174_b200 as slm  # noqa: E402

PH = ["start", "prologue", "accum", "staged", "csync1", "recv", "final", "end"]


def run(kind, bn, split, K=2048, impl=0, M=2048, N=256):
    dev = "cuda"
    if kind == 0:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        out = torch.empty(split, N, M, device=dev)
        resid, bias = torch.randn(N, M, device=dev), torch.randn(M, device=dev)
    elif kind == 1:
        A = torch.randn(K, M, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        out = torch.empty(split, N, M, device=dev)
        resid = bias = None
    else:   # dW: A = act [K][M], B = g [K][N] (both MN-major), out bf16 [N][M]
        A = torch.randn(K, M, device=dev).bfloat16()
        B = torch.randn(K, N, device=dev).bfloat16()
        out = torch.empty(N, M, device=dev).bfloat16()
        resid = bias = None
    ncta = (M // 128) * (N // bn) * split
    ts = torch.zeros(ncta * 8, dtype=torch.int64, device=dev)
    for _ in range(3):
        slm.debug_gemm(kind, impl, bn, M, N, K, A, B, out, resid, bias, split=split)
    torch.cuda.synchronize()
    slm.check(slm.lib.slm_debug_timestamps(C.c_void_p(ts.data_ptr())))
    # flush L2 so W comes from HBM like in the step
    junk = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    junk.fill_(1)
    torch.cuda.synchronize()
    slm.debug_gemm(kind, impl, bn, M, N, K, A, B, out, resid, bias, split=split)
    torch.cuda.synchronize()
    slm.check(slm.lib.slm_debug_timestamps(None))
    t = ts.view(ncta, 8).cpu().double()
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0  # us
    used = [i for i in range(8) if (t[:, i] > 0).all()]
    line = " ".join(f"{PH[i]}={rel[:, i].median():.2f}/{rel[:, i].max():.2f}" for i in used)
    print(f"kind={kind} bn={bn} split={split} K={K} impl={impl} ctas={ncta}: span={rel.max():.2f}us  {line}",
          flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        v = [int(x) for x in a.split(",")]
        run(*v)
