"""GPU parity of NEXT #4's second tree source: DFLASH position rows through the
C-ABI (row_mode = SMART_ROWS_POSITION) against the fp64 oracle (ROWS_POSITION) on the same seeded
inputs.  DFLASH+SMART (PREFIX / FROZEN): per-layer decisions, candidates, trees, masks and walks
bit-exact, scores within 1e-5 (smart_gpu_cases.compare).  DFLASH baseline (selection BASELINE
with max_frontier = g): the paper's Cartesian product pruned to the top-g by cum, bit-exact on the
final tree and the walk.
"""
import numpy as np
import pytest

from inputs import synth
from smart_gpu_cases import Case, REL_TOL, compare, gpu_ctx, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_09731_b200 import _build
    _build.build()
    from oracle import oracle as O
    O.build()


SMART_CASES = {
    "small_bf16": Case(V=3000, k=4, d=4, W=4, b=3, B_verify=60, seed=11),
    "small_fp32_frozen": Case(V=2500, k=3, d=3, W=3, b=2, B_verify=40, seed=12, dtype="fp32", selection=1,
                              accept_model=1, omega=0, cost=(0.02, 0.0, 0.05, 0.01, 1.2, 0.0, 1.0)),
    # cfg2-shaped DFLASH+SMART: Llama-3.1-8B vocab, b = 1, d = 6, k = 10, W = 10, 60 verified tokens
    "cfg2_dflash": Case(V=128256, k=10, d=6, W=10, b=1, B_verify=60, seed=13),
    "b16_ragged": Case(V=32001, k=8, d=5, W=8, b=16, B_verify=320, seed=14, ld_pad=7),
}
BASE_CASES = {
    "base_small": Case(V=4000, k=4, d=3, W=12, b=4, B_verify=48, seed=21, selection=2),
    "base_cfg2": Case(V=128256, k=10, d=6, W=60, b=1, B_verify=60, seed=22, selection=2),
}


def _pos_pool(case):
    # d independent position rows per request (the shape of one non-autoregressive DFLASH forward)
    return synth.draft_pool(case.seed, case.b, case.d, case.V, ld=case.V + case.ld_pad, dtype=case.dtype,
                            a_lo=case.a_lo, a_hi=case.a_hi, sigma_bg=case.sigma_bg)


def _target(case, pos, depth, T):
    # target row of node u = the position row of the token after u (+ noise), so the walk accepts
    node = np.zeros((case.b, T) + pos.shape[2:], pos.dtype)
    for r in range(case.b):
        for u in range(T):
            node[r, u] = pos[r, min(int(depth[r, u]), case.d - 1)]
    return synth.target_pool(node, case.seed + 1000, case.sigma_m, V=case.V)


def _roots(case):
    rng = np.random.default_rng(case.seed)
    return rng.integers(0, case.V, case.b).astype(np.int32), rng.integers(0, 4000, case.b).astype(np.int32)


def _ocfg(case, O):
    return O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify, alpha=case.alpha,
                    omega=case.omega, selection=case.selection if case.selection != 2 else 0,
                    accept_model=case.accept_model, marginal=case.marginal,
                    dtype=O.BF16 if case.dtype == "bf16" else O.FP32, row_mode=O.ROWS_POSITION)


def _run_gpu(case, pos, target, rt, rp):
    import torch
    from paper_2604_09731_b200 import smart as S
    ctx = gpu_ctx(case, row_mode=S.ROWS_POSITION)
    pd, td = to_dev(pos), to_dev(target)
    out = ctx.alloc_outputs()
    ctx.begin_step(to_dev(rt), to_dev(rp))
    for l in range(1, case.d + 1):
        ctx.expand_step(l, pd)
        ctx.select(l)
    ctx.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"])
    ctx.verify_accept(td, out["accept_len"], out["accept_path"], out["bonus"])
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["stats"] = ctx.stats()
    res["tree"] = ctx.tree()
    res["cands"] = {l: ctx.candidates(l) for l in range(1, case.d + 1) if res["stats"]["layers"][l - 1]["executed"]}
    res["ctx"] = ctx
    return res


@pytest.mark.parametrize("name", list(SMART_CASES))
def test_dflash_smart_parity(name):
    from oracle import oracle as O
    case = SMART_CASES[name]
    lam, beta, gamma, delta, rho, eta, c_T = case.cost
    cost = O.Cost(lam=lam, beta=beta, gamma=gamma, delta=delta, rho=rho, eta=eta, c_T=c_T)
    cfg = _ocfg(case, O)
    pos = _pos_pool(case)
    rt, rp = _roots(case)
    T = cfg.tmax()
    shape = O.step(cfg, cost, pos, None, root_tok=rt, root_pos=rp)  # tree shape for the target rows
    target = _target(case, pos, shape.depth, T)
    orc = O.step(cfg, cost, pos, target, root_tok=rt, root_pos=rp)
    gpu = _run_gpu(case, pos, target, rt, rp)
    assert gpu["ctx"].sizes["T"] == T
    L = compare(case, orc, gpu)
    assert L >= 1
    assert orc.n_nodes.sum() > case.b  # something was drafted


@pytest.mark.parametrize("name", list(BASE_CASES))
def test_dflash_baseline_parity(name):
    from oracle import oracle as O
    case = BASE_CASES[name]
    cfg = _ocfg(case, O)
    pos = _pos_pool(case)
    rt, rp = _roots(case)
    T = O.baseline_T(cfg)
    shape = O.baseline_step(cfg, pos, None, root_tok=rt, root_pos=rp)
    target = _target(case, pos, shape.depth, T)
    orc = O.baseline_step(cfg, pos, target, root_tok=rt, root_pos=rp)
    gpu = _run_gpu(case, pos, target, rt, rp)
    assert gpu["ctx"].sizes["T"] == T
    assert gpu["stats"]["error_flags"] & 3 == 0
    for key in ("tree_len", "tok", "parent", "pos", "accept_len", "accept_path", "bonus"):
        np.testing.assert_array_equal(gpu[key], orc.n_nodes if key == "tree_len" else getattr(orc, key), err_msg=key)
    np.testing.assert_array_equal(gpu["mask"].view(np.uint32), orc.mask)
    tree = gpu["tree"]
    for r in range(case.b):
        n = int(orc.n_nodes[r])
        np.testing.assert_allclose(tree["cum"][r, :n], orc.cum[r, :n], rtol=REL_TOL)
    g = case.B_verify // case.b
    assert (orc.n_nodes == g + 1).all()  # k + k^2 + ... >= g: exactly the top-g of the product
