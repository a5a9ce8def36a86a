"""Data-parallel semantics of the library on the device (reading A14).

  * 1 GPU, shard emulation: two half-batch ChainModels with batch_global = 2 B (each scales its
    loss by 1 / B_global, batch statistics local to the shard) summed on the host equal the
    oracle's data-parallel definition oracle.chain.step_dp(world = 2) — the library's DP
    arithmetic without NCCL;
  * >= 2 GPUs: the real NCCL path (bucketed all-reduce inside slm_step, NCCL_ALGO / NCCL_PROTO
    pinned) at world 2 against the same definition, and checkpointed == non-checkpointed bit for
    bit on every rank.  Skipped where only one GPU is visible.
"""
import os
import socket

import numpy as np
import pytest
import torch

import synth
from _util import margin_inputs
from oracle import chain as OC

pytestmark = pytest.mark.gpu


def _dev(inp):
    p = dict(W=torch.tensor(inp["W"]).to(torch.bfloat16).cuda(), b=torch.tensor(inp["b"]).cuda(),
             gamma=torch.tensor(inp["gamma"]).cuda(), beta=torch.tensor(inp["beta"]).cuda())
    return p


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_dp_shard_emulation_matches_step_dp():
    import paper_1604_06174_b200 as slm
    n, Bl, d, world = 3, 64, 256, 2
    Bg = Bl * world
    inp = margin_inputs(n, Bg, d, "bf16", seed=23)
    p = _dev(inp)
    tot, loss = None, 0.0
    for r in range(world):
        g = {k: torch.empty_like(v) for k, v in p.items()}
        model = slm.ChainModel(p, g, dtype="bf16", batch=Bl, batch_global=Bg)
        plan = slm.Plan(slm.Graph.chain(n, Bl, d), "sqrt")
        sl = slice(r * Bl, (r + 1) * Bl)
        lr = model.step(plan, torch.tensor(inp["x0"][sl]).cuda(), torch.tensor(inp["labels"][sl]).cuda())
        torch.cuda.synchronize()
        loss += float(lr.item())
        gr = {k: v.float().cpu().numpy().astype(np.float64) for k, v in g.items()}
        tot = gr if tot is None else {k: tot[k] + gr[k] for k in tot}
    P = OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"])
    ol, og = OC.step_dp(P, inp["x0"], inp["labels"], world, mode="bf16")
    assert abs(loss - ol) <= 2e-2 * abs(ol), (loss, ol)
    for k in og:
        assert _rel(tot[k], og[k]) <= 2e-2, (k, _rel(tot[k], og[k]))
    # and the emulation is not the single-batch step: BN statistics are per shard (A14)
    ol1, og1, _ = OC.step_plain(P, inp["x0"], inp["labels"], "bf16")
    assert _rel(og1["gamma"], og["gamma"]) > 1e-3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _nccl_worker(rank, world, port, n, Bl, d, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_ALGO="Ring", NCCL_PROTO="Simple")
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)   # bootstrap only (the unique id)
    import paper_1604_06174_b200 as slm
    Bg = Bl * world
    inp = synth.chain_inputs(n, Bg, d, dtype="bf16", seed=29)
    p = _dev(inp)
    comm = slm.Comm(rank, world, bucket_bytes=2 * d * d * 2)
    res = {}
    for strategy in ("none", "sqrt"):
        g = {k: torch.empty_like(v) for k, v in p.items()}
        model = slm.ChainModel(p, g, dtype="bf16", batch=Bl, batch_global=Bg)
        par = slm.ALLOC_INPLACE | slm.ALLOC_SHARING | slm.ALLOC_MIRROR_PARITY
        plan = slm.Plan(slm.Graph.chain(n, Bl, d), strategy, alloc_flags=par)
        sl = slice(rank * Bl, (rank + 1) * Bl)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(2):
                loss = model.step(plan, torch.tensor(inp["x0"][sl]).cuda(), torch.tensor(inp["labels"][sl]).cuda(),
                                  stream=s, comm=comm)
        torch.cuda.synchronize()
        res[strategy] = (float(loss.item()), {k: v.float().cpu().numpy().astype(np.float64) for k, v in g.items()})
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_dp_nccl_world2():
    import torch.multiprocessing as mp
    n, Bl, d, world = 12, 64, 256, 2
    out = mp.Manager().dict()
    mp.spawn(_nccl_worker, args=(world, _free_port(), n, Bl, d, out), nprocs=world, join=True)
    inp = synth.chain_inputs(n, Bl * world, d, dtype="bf16", seed=29)
    P = OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"])
    ol, og = OC.step_dp(P, inp["x0"], inp["labels"], world, mode="bf16")
    for r in range(world):
        l0, g0 = out[r]["none"]
        l1, g1 = out[r]["sqrt"]
        assert l0 == l1
        for k in g0:
            assert np.array_equal(g0[k], g1[k]), (r, k)   # ckpt == no-ckpt bit for bit at world 2
            assert np.array_equal(g0[k], out[0]["none"][1][k]), (r, k)   # every rank holds the same sum
        assert abs(l0 - ol) <= 2e-2 * abs(ol)
        for k in og:
            assert _rel(g0[k], og[k]) <= 2e-2, (k, _rel(g0[k], og[k]))
