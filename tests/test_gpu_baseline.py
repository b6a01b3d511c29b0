"""GPU parity of NEXT #3 (Q32): the two-stage likelihood-maximising baseline
(EAGLE-3 / MSD, Fig. 2(a)(b)) run through the C-ABI with selection = BASELINE against
oracle.baseline_step on the same seeded inputs.  Bit-exact on the final tree (tree_len, tokens,
parents, masks, positions) and the greedy walk; 1e-5 relative on p / cum.
"""
import numpy as np
import pytest

from smart_gpu_cases import Case, make_inputs, run_gpu, REL_TOL

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


CASES = {
    "tiny_fp32": Case(V=1000, k=4, d=3, W=4, b=3, B_verify=30, dtype="fp32", seed=1, selection=2),
    "d1_w1": Case(V=3000, k=5, d=1, W=1, b=2, B_verify=8, seed=2, selection=2),
    "keep_all": Case(V=2000, k=3, d=2, W=2, b=2, B_verify=200, seed=3, selection=2),
    "mid_bf16": Case(V=50000, k=8, d=6, W=8, b=4, B_verify=160, seed=4, selection=2),
    # cfg2-shaped EAGLE default: Llama-3.1-8B vocab, b=1, d=6, k=10, W=10, 60 verified tokens
    "cfg2_eagle": Case(V=128256, k=10, d=6, W=10, b=1, B_verify=60, seed=5, selection=2),
    "b32_ragged": Case(V=32001, k=8, d=5, W=16, b=32, B_verify=2048, seed=6, selection=2, dtype="fp32"),
}


def _oracle(case, draft, target, rt, rp):
    from oracle import oracle as O
    cfg = O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify,
                   dtype=O.BF16 if case.dtype == "bf16" else O.FP32)
    return O.baseline_step(cfg, draft, target, root_tok=rt, root_pos=rp)


def _T(case):
    from oracle import oracle as O
    return O.baseline_T(O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify))


@pytest.mark.parametrize("name", list(CASES))
def test_baseline_parity(name):
    case = CASES[name]
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    orc = _oracle(case, draft, target, rt, rp)
    gpu = run_gpu(case, draft, target, rt, rp)
    assert gpu["ctx"].sizes["T"] == T
    st = gpu["stats"]
    assert st["error_flags"] & 3 == 0, st["error_flags"]
    # stage 1: every layer expands min(W, candidates) nodes per request
    n_adm = sum(st["layers"][l]["n_admit"] for l in range(case.d) if st["layers"][l]["executed"])
    assert n_adm == int((orc.extra["n_exp"] - 1).sum())
    # stage 2 + A7 + A8: the final tree and the walk
    np.testing.assert_array_equal(gpu["tree_len"], orc.n_nodes)
    np.testing.assert_array_equal(gpu["tok"], orc.tok)
    np.testing.assert_array_equal(gpu["parent"], orc.parent)
    np.testing.assert_array_equal(gpu["mask"].view(np.uint32), orc.mask)
    np.testing.assert_array_equal(gpu["pos"], orc.pos)
    np.testing.assert_array_equal(gpu["accept_len"], orc.accept_len)
    np.testing.assert_array_equal(gpu["accept_path"], orc.accept_path)
    np.testing.assert_array_equal(gpu["bonus"], orc.bonus)
    tree = gpu["tree"]
    for r in range(case.b):
        n = int(orc.n_nodes[r])
        np.testing.assert_array_equal(tree["depth"][r, :n], orc.depth[r, :n])
        np.testing.assert_allclose(tree["p"][r, :n], orc.p[r, :n], rtol=REL_TOL)
        np.testing.assert_allclose(tree["cum"][r, :n], orc.cum[r, :n], rtol=REL_TOL)
    # the tree is exactly min(g, #generated) + 1 nodes
    g = case.B_verify // case.b
    assert (orc.n_nodes <= g + 1).all()


def test_baseline_run_step_equals_separate_calls():
    case = CASES["mid_bf16"]
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    a = run_gpu(case, draft, target, rt, rp)
    b = run_gpu(case, draft, target, rt, rp, use_run_step=True)
    for key in ("mask", "pos", "parent", "tok", "tree_len", "accept_len", "accept_path", "bonus"):
        np.testing.assert_array_equal(a[key], b[key])

