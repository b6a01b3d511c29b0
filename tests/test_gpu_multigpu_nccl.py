"""Multi-GPU path through the library's own NCCL communicator (smart_attach_nccl): G = 2 processes,
one per GPU, each owning half of the requests; the per-layer exchange is ncclAllGather on the
step's stream and the end-of-step C2 all-reduce (ncclAllReduce of the accept-length and node
sums) gives the global acceptance counts.  The sharded step, captured in a CUDA
graph (what bench.py --gpus N replays), must reproduce the G = 1 trees, masks and walks bit for
bit, and the C2 sums must equal the G = 1 totals.

Needs >= 2 GPUs: skipped on single-GPU boxes (the host-side exchange logic is covered on one GPU
by test_gpu_sharding.py and on CPU by test_dist_gloo.py)."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _need_two():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 CUDA devices")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASE = dict(V=30000, k=6, d=5, W=6, b=8, B_verify=96, seed=31, cost=(0.002, 0.0, 0.03, 0.01, 1.2, 1.5, 1.0))


def _config(S, b_loc, b_glob, off):
    lam, beta, gamma, delta, rho, eta, c_T = CASE["cost"]
    cfg = S.Config(vocab=CASE["V"], top_k=CASE["k"], max_depth=CASE["d"], max_frontier=CASE["W"], batch_local=b_loc,
                   batch_global=b_glob, batch_offset=off, budget_verify=CASE["B_verify"], row_mode=S.ROWS_NODE)
    return cfg, S.Cost(lam=lam, beta=beta, gamma=gamma, delta=delta, rho=rho, eta=eta, c_T=c_T)


def _inputs(T):
    sys.path.insert(0, ROOT)
    from inputs import synth
    draft = synth.draft_pool(CASE["seed"], CASE["b"], T, CASE["V"], a_lo=5.0, a_hi=12.0)
    target = synth.target_pool(draft, CASE["seed"] + 1000, 1.0)
    rng = np.random.default_rng(CASE["seed"])
    return draft, target, rng.integers(0, CASE["V"], CASE["b"]).astype(np.int32), np.full(CASE["b"], 7, np.int32)


def _dev(a, device):
    import torch
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(a).to(device)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2604_09731_b200 import smart as S
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        b = CASE["b"] // world
        cfg, cost = _config(S, b, CASE["b"], rank * b)
        ctx = S.Smart(cfg, cost, rank)
        uid = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.attach_nccl(uid[0], rank, world)
        T = ctx.sizes["T"]
        draft, target, rt, rp = _inputs(T)
        sl = slice(rank * b, (rank + 1) * b)
        dd, tt = _dev(np.ascontiguousarray(draft[sl]), dev), _dev(np.ascontiguousarray(target[sl]), dev)
        rtd, rpd = _dev(rt[sl].copy(), dev), _dev(rp[sl].copy(), dev)
        out = ctx.alloc_outputs()
        s = torch.cuda.Stream(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            ctx.run_step(dd, tt, out, root_tok=rtd, root_pos=rpd, stream=s)  # eager, then captured
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            ctx.run_step(dd, tt, out, root_tok=rtd, root_pos=rpd, stream=s)
        for v in out.values():
            v.zero_()
        g.replay()
        torch.cuda.synchronize()
        st = ctx.stats()
        q.put((rank, {k: v.cpu().numpy() for k, v in out.items()}, st["accepted_global"], st["nodes_global"]))
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_nccl_two_ranks_match_one_rank_in_a_graph():
    _need_two()
    import torch
    import torch.multiprocessing as mp
    sys.path.insert(0, ROOT)
    from paper_2604_09731_b200 import _build
    from paper_2604_09731_b200 import smart as S
    _build.build()
    # G = 1 on device 0
    cfg, cost = _config(S, CASE["b"], CASE["b"], 0)
    ctx = S.Smart(cfg, cost, 0)
    T = ctx.sizes["T"]
    draft, target, rt, rp = _inputs(T)
    out1 = ctx.alloc_outputs()
    dev0 = torch.device("cuda", 0)
    ctx.run_step(_dev(draft, dev0), _dev(target, dev0), out1, root_tok=_dev(rt, dev0), root_pos=_dev(rp, dev0))
    torch.cuda.synchronize()
    ref = {k: v.cpu().numpy() for k, v in out1.items()}
    st1 = ctx.stats()
    assert st1["nodes_local"] >= CASE["b"], "the case must grow non-trivial trees"
    ctx.close()
    # G = 2, one process per GPU
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (o, a, n)) for r, o, a, n in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    b = CASE["b"] // 2
    for key in ("tree_len", "tok", "parent", "pos", "mask", "accept_len", "accept_path", "bonus"):
        got = np.concatenate([res[0][0][key], res[1][0][key]])
        np.testing.assert_array_equal(got, ref[key][: 2 * b], err_msg=key)
    # C2: every rank holds the global sums, equal to the G = 1 totals
    for r in range(2):
        assert res[r][1] == st1["accepted_local"] and res[r][2] == st1["nodes_local"]
