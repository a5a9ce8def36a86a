"""World-size-2 data-parallel host logic on CPU (gloo), SURVEY 8(e) / reading A14.

  * the NCCL unique id drawn by rank 0 through the C ABI reaches every rank unchanged
    (Comm.broadcast_unique_id, the bootstrap slm_comm_init consumes);
  * the DP step semantics: each rank runs the oracle on its row shard with the loss scaled by
    1/B_global, a real all-reduce(sum) over the process group combines loss and gradients, and
    the result equals oracle.chain.step_dp (the definition) on every rank;
  * world 1 reduces to the single-process oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import chain as OC


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _uid_worker(rank, world, port, out):
    _init(rank, world, port)
    import paper_1604_06174_b200 as slm
    uid = slm.Comm.broadcast_unique_id(rank, world)
    out[rank] = bytes(uid)
    dist.barrier()
    dist.destroy_process_group()


def _dp_worker(rank, world, port, n, Bg, d, out):
    _init(rank, world, port)
    inp = synth.chain_inputs(n, Bg, d, dtype="f32", seed=11)
    P = OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"])
    Bl = Bg // world
    sl = slice(rank * Bl, (rank + 1) * Bl)       # rows [r*Bl, (r+1)*Bl) as bench.py shards x0
    loss, g, _ = OC.step_plain(P, inp["x0"][sl], inp["labels"][sl], "f64", batch_global=Bg)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in g.items()}
    t["loss"] = torch.tensor([loss], dtype=torch.float64)
    for k in sorted(t):
        dist.all_reduce(t[k], op=dist.ReduceOp.SUM)
    out[rank] = {k: v.numpy().copy() for k, v in t.items()}
    dist.barrier()
    dist.destroy_process_group()


def test_unique_id_broadcast_world2():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_uid_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        ids = [out[r] for r in range(world)]
    assert len(ids[0]) == 128 and any(ids[0])
    assert ids[0] == ids[1]


@pytest.mark.parametrize("world", [1, 2])
def test_dp_allreduce_matches_step_dp(world):
    n, Bg, d = 4, 16, 64
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_dp_worker, args=(world, _free_port(), n, Bg, d, out), nprocs=world, join=True)
        res = [dict(out[r]) for r in range(world)]
    inp = synth.chain_inputs(n, Bg, d, dtype="f32", seed=11)
    P = OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"])
    ref_loss, ref = OC.step_dp(P, inp["x0"], inp["labels"], world)
    for r in range(world):
        assert np.allclose(res[r]["loss"][0], ref_loss, rtol=1e-13, atol=0)
        for k in ref:
            np.testing.assert_allclose(res[r][k], ref[k], rtol=1e-12, atol=1e-15)
    if world == 1:   # world 1 == the single-process definition
        l1, g1, _ = OC.step_plain(P, inp["x0"], inp["labels"], "f64")
        assert np.isclose(l1, ref_loss, rtol=1e-14)
        for k in g1:
            np.testing.assert_allclose(g1[k], ref[k], rtol=1e-12, atol=1e-15)


def test_dp_differs_from_full_batch_bn():
    """A14: BN statistics are local per rank, so world 2 is NOT the full-batch step (the
    test would pass vacuously if the shards were not actually normalised separately)."""
    n, Bg, d = 3, 16, 64
    inp = synth.chain_inputs(n, Bg, d, dtype="f32", seed=11)
    P = OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"])
    l2, g2 = OC.step_dp(P, inp["x0"], inp["labels"], 2)
    l1, g1, _ = OC.step_plain(P, inp["x0"], inp["labels"], "f64")
    assert not np.allclose(g2["W"], g1["W"], rtol=1e-6)
