"""Host-side logic of the sharded (N > 1) path on CPU with world_size 2 gloo:
request sharding, the rank-ordered all-gather of exchange records, the id broadcast, and the
fp64 oracle's batch-global selection being independent of how the batch is split
(the same property the GPU path is tested for in test_gpu_sharding.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_09731_b200 import dist as D


def test_shard_ranges():
    s = [D.shard(32, 4, r) for r in range(4)]
    assert [x.offset for x in s] == [0, 8, 16, 24] and all(x.b_loc == 8 for x in s)
    with pytest.raises(ValueError):
        D.shard(30, 4, 0)
    with pytest.raises(ValueError):
        D.shard(32, 4, 4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # exchange records: rank-ordered concatenation
        nbytes = 64
        send = torch.full((nbytes,), rank + 1, dtype=torch.uint8)
        recv = torch.zeros(world * nbytes, dtype=torch.uint8)
        D.exchange(send, recv)
        ok_gather = all(int(recv[g * nbytes]) == g + 1 and int(recv[(g + 1) * nbytes - 1]) == g + 1
                        for g in range(world))
        # id broadcast
        payload = bytes(range(128)) if rank == 0 else None
        got = D.broadcast_bytes(payload)
        q.put((rank, ok_gather, got == bytes(range(128))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_and_broadcast():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] and r[2] for r in res)


def _oracle_worker(rank, world, port, q):
    """Each rank runs the fp64 oracle on the FULL batch (the oracle is batch-global by
    construction) but keeps only its shard; gathered shards must equal the single-process run."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from inputs import synth
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, V = 8, 3000
        cfg = O.Config(V=V, k=4, d=4, W=4, b=b, B_verify=48, alpha=0.8, omega=1, dtype=O.FP32)
        cost = O.Cost(lam=0.02, gamma=0.05, delta=0.01, rho=1.2, eta=1.0, c_T=1.0)
        sh = D.shard(b, world, rank)
        # rows are keyed by global request id: each rank can build its own slice
        mine = synth.draft_pool(5, sh.b_loc, cfg.tmax(), V, r_offset=sh.offset, dtype="fp32", a_lo=4, a_hi=10)
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        full = np.concatenate(parts)
        res = O.step(cfg, cost, full)
        tok = torch.from_numpy(res.tok[sh.offset:sh.offset + sh.b_loc].copy())
        gathered = [torch.zeros_like(tok) for _ in range(world)]
        dist.all_gather(gathered, tok)
        ref = O.step(cfg, cost, synth.draft_pool(5, b, cfg.tmax(), V, dtype="fp32", a_lo=4, a_hi=10))
        q.put((rank, bool(np.array_equal(torch.cat(gathered).numpy(), ref.tok))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partition_invariant_inputs_and_oracle():
    """Input rows keyed by global request id + the batch-global oracle: shards reassemble the
    single-process tree exactly (the reference the GPU sharding test compares against)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_oracle_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] for r in res)
