"""The peer exchange (NEXT #4; smart_attach_peer_exchange): each rank's local
selection record is written straight into every rank's receive buffer with a tagged release, and
the global phase polls the tags -- no collective call.  Checked against G = 1 bit for bit (trees,
scores, masks, verify), as the all-gather path is in test_gpu_sharding.py:
* in one process, G contexts on one GPU, every local phase before any global phase (stream order);
* across two processes on one GPU, the receive buffers mapped with CUDA IPC, the processes in
  lockstep through host barriers (no kernel waits on another process's kernel)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from smart_gpu_cases import Case, make_inputs, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_09731_b200 import _build
    _build.build()


def _T(case):
    from oracle import oracle as O
    return O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify).tmax()


def _ctx(case, g, G):
    from paper_2604_09731_b200 import smart as S
    lam, beta, gamma, delta, rho, eta, c_T = case.cost
    bl = case.b // G
    cfg = S.Config(vocab=case.V, top_k=case.k, max_depth=case.d, max_frontier=case.W, batch_local=bl,
                   batch_global=case.b, batch_offset=g * bl, budget_verify=case.B_verify, alpha=case.alpha,
                   bonus=case.omega, selection=case.selection, accept_model=case.accept_model,
                   marginal=case.marginal, logits_dtype=S.BF16 if case.dtype == "bf16" else S.FP32,
                   row_mode=S.ROWS_NODE)
    return S.Smart(cfg, S.Cost(lam=lam, beta=beta, gamma=gamma, delta=delta, rho=rho, eta=eta, c_T=c_T))


def run_peer(case, G, draft, target, rt, rp, steps=2):
    import torch
    bl = case.b // G
    ctxs = [_ctx(case, g, G) for g in range(G)]
    nbytes = ctxs[0].peer_exchange_bytes(G)
    bufs = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(G)]
    for g, c in enumerate(ctxs):
        c.attach_peer_exchange(g, G, [b.data_ptr() for b in bufs], keep=bufs)
    dd = [to_dev(np.ascontiguousarray(draft[g * bl:(g + 1) * bl])) for g in range(G)]
    tt = [to_dev(np.ascontiguousarray(target[g * bl:(g + 1) * bl])) for g in range(G)]
    for step in range(steps):  # a second step: the tags of the first may not be taken for the second
        for g, c in enumerate(ctxs):
            c.begin_step(to_dev(rt[g * bl:(g + 1) * bl].copy()), to_dev(rp[g * bl:(g + 1) * bl].copy()))
        for layer in range(1, case.d + 1):
            for g, c in enumerate(ctxs):
                c.expand_step(layer, dd[g])
                c.select(layer)
            for c in ctxs:
                c.select_finish(layer)
        outs = []
        for g, c in enumerate(ctxs):
            out = c.alloc_outputs()
            c.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"])
            c.verify_accept(tt[g], out["accept_len"], out["accept_path"], out["bonus"])
            outs.append(out)
        torch.cuda.synchronize()
    res = []
    for g, c in enumerate(ctxs):
        r = {k: v.cpu().numpy() for k, v in outs[g].items()}
        r["tree"] = c.tree()
        r["stats"] = c.stats()
        res.append(r)
    cat = {k: np.concatenate([r[k] for r in res]) for k in res[0] if k not in ("tree", "stats")}
    cat["cum"] = np.concatenate([r["tree"]["cum"] for r in res])
    cat["p"] = np.concatenate([r["tree"]["p"] for r in res])
    cat["stats"] = [r["stats"] for r in res]
    return cat


CASES = [
    Case(V=40000, k=6, d=5, W=6, b=8, B_verify=80, seed=31, cost=(0.02, 0.0, 0.05, 0.01, 1.2, 1.0, 1.0)),
    Case(V=128256, k=8, d=6, W=8, b=32, B_verify=200, seed=32, cost=(0.0084, 0.0, 6.69, 6.3e-7, 2.23, 2.47, 2.47)),
]


@pytest.mark.parametrize("case", CASES, ids=["b8", "cfg3"])
@pytest.mark.parametrize("G", [2, 4])
def test_peer_exchange_equals_single(case, G):
    from smart_gpu_cases import run_gpu
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    one = run_gpu(case, draft, target, rt, rp)
    many = run_peer(case, G, draft, target, rt, rp)
    for key in ("tree_len", "tok", "parent", "mask", "pos", "accept_len", "accept_path", "bonus"):
        np.testing.assert_array_equal(many[key], one[key], err_msg=key)
    np.testing.assert_array_equal(many["cum"].view(np.uint32), one["tree"]["cum"].view(np.uint32))
    for st in many["stats"]:
        assert st["error_flags"] == 0
        for l in range(case.d):
            a, b = st["layers"][l], one["stats"]["layers"][l]
            if b["executed"]:
                assert a["n_admit"] == b["n_admit"] and a["N0"] == b["N0"] and a["E0"] == b["E0"], (l, a, b)


_WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"]); sys.path.insert(0, os.path.join(os.environ["REPO"], "tests"))
from test_gpu_peer_exchange import _ctx, _T
from smart_gpu_cases import Case, make_inputs, to_dev
from paper_2604_09731_b200 import smart as S
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["PORT"],
                        rank=int(os.environ["RANK"]), world_size=2)
g, G = dist.get_rank(), 2
case = Case(V=40000, k=6, d=5, W=6, b=8, B_verify=80, seed=31, cost=(0.02, 0.0, 0.05, 0.01, 1.2, 1.0, 1.0))
T = _T(case)
draft, target, rt, rp = make_inputs(case, T)
bl = case.b // G
c = _ctx(case, g, G)
buf = torch.zeros(c.peer_exchange_bytes(G), dtype=torch.uint8, device="cuda")
handles = [None, None]
dist.all_gather_object(handles, S.ipc_handle(buf.data_ptr()))
ptrs = [buf.data_ptr() if h == g else S.ipc_open(handles[h]) for h in range(G)]
c.attach_peer_exchange(g, G, ptrs, keep=buf)
dd = to_dev(np.ascontiguousarray(draft[g * bl:(g + 1) * bl]))
tt = to_dev(np.ascontiguousarray(target[g * bl:(g + 1) * bl]))
c.begin_step(to_dev(rt[g * bl:(g + 1) * bl].copy()), to_dev(rp[g * bl:(g + 1) * bl].copy()))
for layer in range(1, case.d + 1):
    c.expand_step(layer, dd)
    c.select(layer)
    torch.cuda.synchronize(); dist.barrier()   # every rank's record pushed before any global phase
    c.select_finish(layer)
    torch.cuda.synchronize(); dist.barrier()
out = c.alloc_outputs()
c.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"])
c.verify_accept(tt, out["accept_len"], out["accept_path"], out["bonus"])
torch.cuda.synchronize()
res = {k: v.cpu().numpy() for k, v in out.items()}
allres = [None, None]
dist.all_gather_object(allres, res)
dist.barrier()
for h in range(G):
    if h != g:
        S.ipc_close(ptrs[h])
if g == 0:
    np.savez(os.environ["OUT"], **{k: np.concatenate([allres[0][k], allres[1][k]]) for k in res})
dist.destroy_process_group()
'''


def test_peer_exchange_two_processes_ipc(tmp_path):
    """Two processes (gloo for the handles and barriers), their receive buffers mapped with CUDA IPC."""
    from smart_gpu_cases import run_gpu
    import socket
    case = Case(V=40000, k=6, d=5, W=6, b=8, B_verify=80, seed=31, cost=(0.02, 0.0, 0.05, 0.01, 1.2, 1.0, 1.0))
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    one = run_gpu(case, draft, target, rt, rp)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "peer.npz")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    procs = [subprocess.Popen([sys.executable, "-c", _WORKER],
                              env=dict(os.environ, REPO=repo, PORT=str(port), RANK=str(r), OUT=out),
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(2)]
    logs = [p.communicate(timeout=600) for p in procs]
    assert all(p.returncode == 0 for p in procs), [l[1][-2000:] for l in logs]
    got = np.load(out)
    for key in ("tree_len", "tok", "parent", "mask", "pos", "accept_len", "accept_path", "bonus"):
        np.testing.assert_array_equal(got[key], one[key], err_msg=key)
