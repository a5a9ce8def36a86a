"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

Holds none of the method's arithmetic: only random draws with the shapes and value
distributions of the paper's workloads.  The paper's data
(ImageNet, speech) is out of scope; PAPER.md:436 (ResNet, batch 32) and PAPER.md:481-483
(LSTM: batch 64, 50-d input, 5000-way softmax) fix the shapes we imitate.

Chain (reading A10):  x0 ~ N(0,1); W_l ~ N(0, 1/d); b_l ~ N(0, 0.01^2);
                      gamma_l ~ 1 + N(0, 0.1^2); beta_l ~ N(0, 0.1^2); labels ~ U{0..d-1}.
LSTM (reading A13):   x_t ~ N(0,1); W_ih, W_hh, b_ih, b_hh ~ U(+-1/sqrt(H)) (PyTorch
                      default); W_o ~ N(0, 1/H); b_o = 0; labels ~ U{0..C-1}.

Each tensor gets its own child stream of ``np.random.SeedSequence(seed)`` (spawn order is
fixed), values are drawn in fp64 and rounded to the working dtype on the host; the oracle
consumes the same rounded values.  For full-size GPU benches (8 GiB of weights) a device
generator (torch, seeded) is used instead — a different stream, documented as such.
"""
from __future__ import annotations

import numpy as np

SEED = 1604_06174


def bf16_values(a):
    """Round fp64 values to the nearest bf16 (RNE); returns float32 carrying bf16 values."""
    f = np.asarray(a, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def _streams(seed, k):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(k)]


def chain_inputs(n_layers, batch, width, dtype="f32", seed=SEED):
    """Returns dict(W [n,d,d] f32 (bf16-valued when dtype='bf16'), b, gamma, beta [n,d] f32,
    x0 [B,d] f32, labels [B] int32)."""
    r = _streams(seed, 6)
    d = width
    W = r[0].standard_normal((n_layers, d, d)) / np.sqrt(d)
    b = r[1].standard_normal((n_layers, d)) * 0.01
    gamma = 1.0 + r[2].standard_normal((n_layers, d)) * 0.1
    beta = r[3].standard_normal((n_layers, d)) * 0.1
    x0 = r[4].standard_normal((batch, d))
    labels = r[5].integers(0, d, size=batch).astype(np.int32)
    W = bf16_values(W) if dtype == "bf16" else W.astype(np.float32)
    return dict(W=W, b=b.astype(np.float32), gamma=gamma.astype(np.float32),
                beta=beta.astype(np.float32), x0=x0.astype(np.float32), labels=labels)


def chain_inputs_torch(n_layers, batch, width, dtype="bf16", seed=SEED, device="cuda"):
    """Device-side generator with the same distributions (a torch.Generator stream, not the
    NumPy one).  Returns torch tensors; W is bf16 (or f32), the rest f32, labels int32."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    d = width
    wdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    W = torch.empty((n_layers, d, d), dtype=wdt, device=device)
    for l in range(n_layers):  # layer by layer keeps the fp32 temporary small
        W[l].copy_(torch.randn((d, d), generator=gen, device=device) / d ** 0.5)
    b = torch.randn((n_layers, d), generator=gen, device=device) * 0.01
    gamma = 1.0 + torch.randn((n_layers, d), generator=gen, device=device) * 0.1
    beta = torch.randn((n_layers, d), generator=gen, device=device) * 0.1
    x0 = torch.randn((batch, d), generator=gen, device=device)
    labels = torch.randint(0, d, (batch,), generator=gen, device=device, dtype=torch.int32)
    return dict(W=W, b=b, gamma=gamma, beta=beta, x0=x0, labels=labels)


def lstm_inputs(n_layers, steps, batch, hidden, n_in, n_classes, dtype="f32", seed=SEED):
    """Unrolled LSTM inputs at the true widths: W[l] = [W_ih | W_hh] as [4H, Kin_l + H] with
    Kin_0 = n_in, Kin_l = H (the device layout pads layer 0 in the binding, LstmModel.pack_w),
    b[l] = b_ih + b_hh [4H], W_o [C, H], b_o [C] (zeros), x [T, B, n_in], labels [T, B]."""
    r = _streams(seed + 1, 8)
    H = hidden
    k = 1.0 / np.sqrt(H)
    W = []
    for l in range(n_layers):
        kin = n_in if l == 0 else H
        w = np.zeros((4 * H, kin + H))
        w[:, :kin] = r[0].uniform(-k, k, (4 * H, kin))
        w[:, kin:] = r[1].uniform(-k, k, (4 * H, H))
        W.append(w)
    b = r[2].uniform(-k, k, (n_layers, 4 * H)) + r[3].uniform(-k, k, (n_layers, 4 * H))
    W_o = r[4].standard_normal((n_classes, H)) / np.sqrt(H)
    x = r[5].standard_normal((steps, batch, n_in))
    labels = r[6].integers(0, n_classes, size=(steps, batch)).astype(np.int32)
    cast = bf16_values if dtype == "bf16" else (lambda a: np.asarray(a, np.float32))
    return dict(W=[cast(w) for w in W], b=b.astype(np.float32), W_o=cast(W_o),
                b_o=np.zeros(n_classes, np.float32), x=x.astype(np.float32), labels=labels,
                n_in=n_in)


def opgraph_inputs(nodes, batch, seed=SEED, shapes=None):
    """Inputs of an op-granularity graph: nodes = [(op, preds, out_bytes, flags)]
    with the slm op codes (FC = 3, BN = 6).  Per FC node W [dout, din] ~ N(0, 1/din) (bf16-valued
    f32) and b ~ N(0, 0.01^2); per BN node gamma ~ 1 + N(0, 0.1^2), beta ~ N(0, 0.1^2) (the chain's
    recipe); x0 [B, w_in] ~ N(0, 1); labels ~ U{0 .. w_out - 1} (w_out = the width of the
    loss's input).  Returns dict(params={node: {..}}, x0, labels).
    Convolutional graphs pass shapes[v] = (H, W, C, k, s): widths are the channel
    counts, x0 is [B*H*W, C_0] (NHWC rows), and a Conv node (op 14) gets W [C_out, k*k*C_in] ~
    N(0, 1/(k*k*C_in)) (fan-in scaling, as FC) and b ~ N(0, 0.01^2)."""
    r = _streams(seed, 2 + 2 * len(nodes))
    if shapes is not None:
        width = [sh[2] for sh in shapes]
        rows0 = batch * shapes[0][0] * shapes[0][1]
    else:
        width = [ob // (4 * batch) for (_, _, ob, _) in nodes]
        rows0 = batch
    params = {}
    for v, (op, preds, ob, _) in enumerate(nodes):
        ra, rb = r[2 + 2 * v], r[3 + 2 * v]
        if op == 14:
            k, cin, cout = shapes[v][3], width[preds[0]], width[v]
            fan = k * k * cin
            params[v] = dict(W=bf16_values(ra.standard_normal((cout, fan)) / np.sqrt(fan)),
                             b=(0.01 * rb.standard_normal(cout)).astype(np.float32))
        elif op == 3:
            din, dout = width[preds[0]], width[v]
            params[v] = dict(W=bf16_values(ra.standard_normal((dout, din)) / np.sqrt(din)),
                             b=(0.01 * rb.standard_normal(dout)).astype(np.float32))
        elif op == 6:
            params[v] = dict(gamma=(1.0 + 0.1 * ra.standard_normal(width[v])).astype(np.float32),
                             beta=(0.1 * rb.standard_normal(width[v])).astype(np.float32))
    x0 = r[0].standard_normal((rows0, width[0])).astype(np.float32)
    loss_in = nodes[-1][1][0]
    labels = r[1].integers(0, width[loss_in], size=batch).astype(np.int32)
    return dict(params=params, x0=x0, labels=labels)
