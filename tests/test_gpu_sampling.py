"""GPU parity of A8 at temperature > 0 (NEXT #1, reading Q31): smart_verify_sample
against the oracle's orc_verify_sample on the same tree and the same counter-based stream.

The sampled token at a node is an argmax of perturbed logits x / tau + G; the GPU evaluates G
in fp32 and the oracle in fp64, so a request whose walk passes a node where the best and
second-best perturbed logits are within 1e-4 is tie-ambiguous (Q24 style) and skipped; every
other request must match bit for bit (accept length, accepted node path, bonus token).
"""
import numpy as np
import pytest

from smart_gpu_cases import Case, gpu_ctx, make_inputs, run_oracle, to_dev

pytestmark = pytest.mark.gpu

MARGIN = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_09731_b200 import _build
    _build.build()
    from oracle import oracle as O
    O.build()


def _T(case):
    from oracle import oracle as O
    return O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify).tmax()


def _gpu_tree_and_sample(case, draft, target, rt, rp, taus_seeds):
    import torch
    ctx = gpu_ctx(case)
    dd, tt = to_dev(draft), to_dev(target)
    out = ctx.alloc_outputs()
    ctx.begin_step(to_dev(rt), to_dev(rp))
    for l in range(1, case.d + 1):
        ctx.expand_step(l, dd)
        ctx.select(l)
    ctx.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"])
    res = []
    for tau, seed in taus_seeds:
        ctx.verify_sample(tt, tau, seed, out["accept_len"], out["accept_path"], out["bonus"])
        torch.cuda.synchronize()
        res.append({k: out[k].cpu().numpy().copy() for k in ("accept_len", "accept_path", "bonus")})
    torch.cuda.synchronize()
    return res


CASES = {
    "small_bf16": Case(V=30000, k=6, d=5, W=6, b=8, B_verify=80, seed=51, sigma_m=1.0),
    "small_fp32_ragged": Case(V=20011, k=4, d=4, W=4, b=6, B_verify=48, seed=52, dtype="fp32", sigma_m=2.0),
    "cfg3_full": Case(V=128256, k=8, d=6, W=8, b=32, B_verify=200, seed=53, sigma_m=2.0,
                      cost=(0.0117, 0.0, 0.05, 0.02, 1.3, 2.4631, 2.4631)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_sample_walk_matches_oracle(name):
    from oracle import oracle as O
    case = CASES[name]
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    orc = run_oracle(case, draft, target, rt, rp)
    taus_seeds = [(1.0, 1234), (0.7, 99), (1.0, 2 ** 63 + 17)]
    gpu = _gpu_tree_and_sample(case, draft, target, rt, rp, taus_seeds)
    compared = 0
    for (tau, seed), g in zip(taus_seeds, gpu):
        a, path, bonus, mg = O.verify_sample(target, orc.n_nodes, orc.parent, orc.tok, tau, seed, case.d, V=case.V)
        ok = mg >= MARGIN
        assert ok.mean() > 0.9, f"too many tie-ambiguous walks: {(~ok).sum()}"
        np.testing.assert_array_equal(g["accept_len"][ok], a[ok])
        np.testing.assert_array_equal(g["accept_path"][ok], path[ok])
        np.testing.assert_array_equal(g["bonus"][ok], bonus[ok])
        compared += int(ok.sum())
    assert compared > 0


def test_low_temperature_equals_greedy():
    case = Case(V=40000, k=6, d=5, W=6, b=8, B_verify=80, seed=54, dtype="fp32")
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    orc = run_oracle(case, draft, target, rt, rp)
    g = _gpu_tree_and_sample(case, draft, target, rt, rp, [(1e-5, 5)])[0]
    np.testing.assert_array_equal(g["accept_len"], orc.accept_len)
    np.testing.assert_array_equal(g["accept_path"], orc.accept_path)
    np.testing.assert_array_equal(g["bonus"], orc.bonus)


def test_bad_temperature_rejected():
    from paper_2604_09731_b200 import smart as S
    case = CASES["small_bf16"]
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    ctx = gpu_ctx(case)
    ctx.begin_step()
    for l in range(1, case.d + 1):
        ctx.expand_step(l, to_dev(draft))
        ctx.select(l)
    out = ctx.alloc_outputs()
    ctx.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"])
    with pytest.raises(S.SmartError):
        ctx.verify_sample(to_dev(target), 0.0, 1, out["accept_len"], out["accept_path"], out["bonus"])
