"""tcgen05/TMA GEMM kernels vs a plain PyTorch fp32 reference and vs the SIMT kernel
(device tests; through the C ABI test hook slm_debug_gemm)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(128, 64, 64), (256, 128, 192), (512, 256, 1024), (2048, 256, 2048), (384, 64, 320)]


def _rel(a, b):
    return ((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30)).item()


@pytest.fixture(scope="module")
def slm():
    import paper_1604_06174_b200 as m
    return m


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("bn", [32, 64, 128, 256])
def test_fwd_gemm(slm, M, N, K, bn):
    if N % bn:
        pytest.skip("N % bn")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    W = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    a = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    resid = torch.randn(N, M, device="cuda", generator=g)
    bias = torch.randn(M, device="cuda", generator=g)
    ref = resid + a.float() @ W.float().T + bias
    out = torch.empty(N, M, device="cuda")
    slm.debug_gemm(0, 0, bn, M, N, K, W, a, out, resid, bias)
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-5
    out2 = torch.empty_like(out)
    slm.debug_gemm(0, 1, bn, M, N, K, W, a, out2, resid, bias)
    torch.cuda.synchronize()
    assert _rel(out2, ref) < 1e-5
    # in place over the residual, as the plan does for Block nodes
    r2 = resid.clone()
    slm.debug_gemm(0, 0, bn, M, N, K, W, a, r2, r2, bias)
    torch.cuda.synchronize()
    assert torch.equal(r2, out)


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("bn", [32, 64, 256])
def test_dx_gemm(slm, M, N, K, bn):
    if N % bn:
        pytest.skip("N % bn")
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + K)
    A = torch.randn(K, M, device="cuda", generator=g).bfloat16()      # W [d_out=K][d_in=M]
    B = torch.randn(N, K, device="cuda", generator=g).bfloat16()      # g [batch][d_out]
    ref = B.float() @ A.float()
    out = torch.empty(N, M, device="cuda")
    slm.debug_gemm(1, 0, bn, M, N, K, A, B, out)
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-5


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (256, 128, 128), (2048, 256, 256), (512, 512, 64)])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_dw_gemm(slm, M, N, K, bn):
    if N % bn:
        pytest.skip("N % bn")
    g = torch.Generator(device="cuda").manual_seed(M + N + 5 * K)
    A = torch.randn(K, M, device="cuda", generator=g).bfloat16()      # a [batch][d_in]
    B = torch.randn(K, N, device="cuda", generator=g).bfloat16()      # g [batch][d_out]
    ref = (B.float().T @ A.float())                                   # [d_out][d_in]
    out = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
    slm.debug_gemm(2, 0, bn, M, N, K, A, B, out)
    torch.cuda.synchronize()
    assert _rel(out.float(), ref) < 5e-3
    # rounding of the same fp32 sums: at most one bf16 ulp apart from torch's rounding
    diff = (out.float() - ref.bfloat16().float()).abs()
    ulp = ref.abs().clamp_min(1e-30) * 2 ** -7
    assert (diff <= ulp * 1.01 + 1e-30).float().mean() > 0.999


# ---- CTA-pair (cta_group::2) GEMM: impl 4 of slm_debug_gemm
PAIR_SHAPES = [(256, 128, 64), (512, 256, 1024), (2048, 256, 2048), (768, 128, 320)]


@pytest.mark.parametrize("M,N,K", PAIR_SHAPES)
@pytest.mark.parametrize("bn", [128, 256])
def test_pair_fwd_gemm(slm, M, N, K, bn):
    if N % bn:
        pytest.skip("N % bn")
    g = torch.Generator(device="cuda").manual_seed(M * 5 + N + K)
    W = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    a = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    resid = torch.randn(N, M, device="cuda", generator=g)
    bias = torch.randn(M, device="cuda", generator=g)
    ref = resid + a.float() @ W.float().T + bias
    out = torch.empty(N, M, device="cuda")
    slm.debug_gemm(0, 4, bn, M, N, K, W, a, out, resid, bias)
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-5
    # same fp32 accumulation order as the single-CTA kernel: identical bits
    out1 = torch.empty_like(out)
    slm.debug_gemm(0, 0, bn, M, N, K, W, a, out1, resid, bias)
    torch.cuda.synchronize()
    assert torch.equal(out, out1)


@pytest.mark.parametrize("M,N,K,split", [(2048, 256, 2048, 4), (2048, 256, 2048, 8), (512, 128, 1024, 2)])
@pytest.mark.parametrize("kind", [0, 1])
def test_pair_splitk_partials(slm, M, N, K, split, kind):
    g = torch.Generator(device="cuda").manual_seed(M + N + K + split)
    if kind == 0:
        A = torch.randn(M, K, device="cuda", generator=g).bfloat16()   # W [M][K]
        B = torch.randn(N, K, device="cuda", generator=g).bfloat16()
        ref = B.float() @ A.float().T
    else:
        A = torch.randn(K, M, device="cuda", generator=g).bfloat16()   # W [K][M] (MN)
        B = torch.randn(N, K, device="cuda", generator=g).bfloat16()
        ref = B.float() @ A.float()
    out = torch.empty(split, N, M, device="cuda")
    slm.debug_gemm(kind, 4, N, M, N, K, A, B, out, split=split)
    torch.cuda.synchronize()
    assert _rel(out.sum(0), ref) < 1e-5
    out1 = torch.empty_like(out)
    slm.debug_gemm(kind, 0, N, M, N, K, A, B, out1, split=split)
    torch.cuda.synchronize()
    assert torch.equal(out, out1)


@pytest.mark.parametrize("M,N,K", [(256, 128, 64), (2048, 256, 256), (512, 512, 128)])
@pytest.mark.parametrize("bn", [128, 256])
def test_pair_dw_gemm(slm, M, N, K, bn):
    if N % bn:
        pytest.skip("N % bn")
    g = torch.Generator(device="cuda").manual_seed(M + 2 * N + 5 * K)
    A = torch.randn(K, M, device="cuda", generator=g).bfloat16()
    B = torch.randn(K, N, device="cuda", generator=g).bfloat16()
    out = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
    slm.debug_gemm(2, 4, bn, M, N, K, A, B, out)
    out1 = torch.empty_like(out)
    slm.debug_gemm(2, 0, bn, M, N, K, A, B, out1)
    torch.cuda.synchronize()
    assert _rel(out.float(), (B.float().T @ A.float())) < 5e-3
    assert torch.equal(out, out1)
