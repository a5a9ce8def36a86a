"""cuBLAS (torch.matmul) timing of the chain layer GEMM shapes on one B200 (reference point
for the fused Block; not part of the library): forward D[2048x256] = W[2048x2048] a^T, and the
weight-gradient shape [2048x2048] = g^T a with K = 256.  CUDA graph of 200 launches over 64
distinct weight matrices (512 MiB > L2, as in the real chain)."""
import torch

def timeit(fn, reps=200):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                fn(i)
        g.replay(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / (5 * reps)

d, B, L = 2048, 256, 64
W = torch.randn(L, d, d, device="cuda").bfloat16()
a = torch.randn(B, d, device="cuda").bfloat16()
out = torch.empty(d, B, device="cuda", dtype=torch.bfloat16)
outf = torch.empty(B, d, device="cuda", dtype=torch.float32)
g = torch.randn(B, d, device="cuda").bfloat16()
dW = torch.empty(d, d, device="cuda", dtype=torch.bfloat16)
fl = 2 * B * d * d
for name, fn in (
    ("fwd  W a^T (bf16 out)", lambda i: torch.mm(W[i % L], a.t(), out=out)),
    ("fwd  a W^T (fp32 out)", lambda i: torch.mm(a, W[i % L].t(), out=outf) if False else torch.matmul(a, W[i % L].t())),
    ("dX   g W", lambda i: torch.matmul(g, W[i % L])),
    ("dW   g^T a (K=256)", lambda i: torch.mm(g.t(), a, out=dW)),
):
    us = timeit(fn)
    print(f"cublas {name:24s}: {us:7.2f} us  {fl / us / 1e6:7.1f} TFLOP/s")
