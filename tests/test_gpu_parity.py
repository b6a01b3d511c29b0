"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle, element by element,
on the same seeded inputs.  Bit-exact on node sets, tokens, parents, masks,
positions, accept lengths/paths and bonus tokens; 1e-5 relative on p, cum, b, E and S.
"""
import json
import os

import numpy as np
import pytest

from smart_gpu_cases import Case, compare, make_inputs, run_gpu, run_oracle, to_dev

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


def _T(case):
    from oracle import oracle as O
    return O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify).tmax()


def _run(case, **kw):
    """The oracle against BOTH CUDA paths on the same inputs: the per-layer C-ABI calls (the
    layer kernels a real draft model interleaves with) and smart_run_step (the persistent
    whole-step kernel, step.cu)."""
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    orc = run_oracle(case, draft, target, rt, rp)
    gpu = run_gpu(case, draft, target, rt, rp, **kw)
    layers = compare(case, orc, gpu)
    if not kw:
        step = run_gpu(case, draft, target, rt, rp, use_run_step=True)
        assert compare(case, orc, step) == layers
    return orc, gpu, layers


# ---- the toy worked example (cfg1) ----------------------------------------------------------

def test_toy_cfg1_gpu():
    """SURVEY §8(c) toy: GPU reproduces the hand-traced HOTPATH/PAPER trees and the walk."""
    import torch
    from smart_toy import toy_pool, toy_target
    from paper_2604_09731_b200 import smart as S
    toy = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "toy_cfg1.json")))
    for preset in ("hotpath", "paper", "budget3"):
        P = toy["hotpath"] if preset != "paper" else toy["paper"]
        B_verify = toy["hotpath_budget3"]["B_verify"] if preset == "budget3" else P["B_verify"]
        hot = preset != "paper"
        cfg = S.Config(vocab=32, top_k=2, max_depth=3, max_frontier=0, batch_local=1, budget_verify=B_verify,
                       alpha=P["alpha"], bonus=1 if hot else 0, selection=S.PREFIX if hot else S.FROZEN,
                       accept_model=S.NODE_SUM if hot else S.PATH_MEAN, logits_dtype=S.FP32)
        cost = S.Cost(lam=1.0, eta=10.0 if hot else 0.0, c_T=10.0)
        ctx = S.Smart(cfg, cost)
        T = ctx.sizes["T"]
        draft = to_dev(toy_pool(toy, T))
        target = to_dev(toy_target(toy, T))
        out = ctx.alloc_outputs()
        ctx.run_step(draft, target, out, root_tok=torch.tensor([-1], dtype=torch.int32, device="cuda"),
                     root_pos=torch.tensor([100], dtype=torch.int32, device="cuda"))
        torch.cuda.synchronize()
        n = int(out["tree_len"][0])
        want = toy["hotpath"] if preset == "hotpath" else (toy["hotpath_budget3"] if preset == "budget3" else toy["paper"])
        assert out["tok"][0, :n].tolist() == want["tokens"], preset
        assert out["parent"][0, :n].tolist() == want["parent"], preset
        st = ctx.stats()
        if preset == "hotpath":
            assert out["mask"][0, :n, 0].tolist() == want["mask_words"]
            assert out["pos"][0, :n].tolist() == [100 + d for d in want["depth"]]
            assert [st["layers"][l]["n_admit"] for l in range(3)] == want["layer_admits"]
            np.testing.assert_allclose([st["layers"][l]["S_after"] for l in range(3)], want["layer_S_after"], rtol=1e-5)
            assert st["layers"][1]["argmax_j"] == want["layer2_argmax_j"]
            np.testing.assert_allclose(st["S_final"], want["S"], rtol=1e-5)
            v = toy["verify"]
            assert int(out["accept_len"][0]) == v["accept_len"]
            assert out["accept_path"][0, :2].tolist() == v["accept_path"]
            assert int(out["bonus"][0]) == v["bonus"]
        if preset == "paper":
            np.testing.assert_allclose(st["S_final"], want["S"], rtol=1e-5)


# ---- every selection x acceptance-model x marginal mode, W in {0, k}: seeded small configs that
# build multi-node, multi-layer trees (found by tools/find_parity_cases.py, which runs only the
# oracle): several 16 KiB chunks per row with ragged tails, both dtypes ---------------------------

MODES = [
    Case(V=40001, k=6, d=5, W=0, b=2, B_verify=30, alpha=0.8, omega=1, selection=0, accept_model=0, marginal=0, dtype='bf16', seed=116, cost=(0.010689, 0.0, 0.045507, 0.018745, 1.063907, 1.528943, 1.0), sigma_m=0.5, a_lo=7.357, a_hi=13.908),
    Case(V=9001, k=7, d=3, W=7, b=4, B_verify=92, alpha=0.8, omega=1, selection=0, accept_model=0, marginal=0, dtype='fp32', seed=287, cost=(0.003776, 0.0, 0.038439, 0.003287, 1.239743, 1.652726, 1.0), sigma_m=0.5, a_lo=7.514, a_hi=10.546),
    Case(V=9001, k=7, d=4, W=0, b=6, B_verify=84, alpha=1.0, omega=1, selection=0, accept_model=0, marginal=1, dtype='bf16', seed=308, cost=(0.003681, 0.0, 0.035029, 0.006724, 1.214171, 1.985393, 1.0), sigma_m=0.5, a_lo=4.829, a_hi=12.830),
    Case(V=9001, k=4, d=5, W=4, b=3, B_verify=33, alpha=1.0, omega=1, selection=0, accept_model=0, marginal=1, dtype='bf16', seed=488, cost=(0.013383, 0.0, 0.019334, 0.013011, 1.157557, 1.896736, 1.0), sigma_m=0.5, a_lo=6.876, a_hi=11.179),
    Case(V=40001, k=6, d=5, W=0, b=5, B_verify=60, alpha=1.0, omega=0, selection=0, accept_model=1, marginal=0, dtype='bf16', seed=490, cost=(0.004193, 0.0, 0.029212, 0.003996, 1.319183, 1.792375, 1.0), sigma_m=0.5, a_lo=4.939, a_hi=13.236),
    Case(V=20000, k=3, d=3, W=3, b=4, B_verify=32, alpha=0.8, omega=0, selection=0, accept_model=1, marginal=0, dtype='bf16', seed=588, cost=(0.028471, 0.0, 0.030318, 0.016611, 1.265421, 1.356562, 1.0), sigma_m=0.5, a_lo=6.062, a_hi=11.722),
    Case(V=9001, k=8, d=3, W=0, b=4, B_verify=40, alpha=0.8, omega=0, selection=0, accept_model=1, marginal=1, dtype='bf16', seed=686, cost=(0.006061, 0.0, 0.020802, 0.018138, 1.228884, 0.801365, 1.0), sigma_m=0.5, a_lo=7.033, a_hi=13.770),
    Case(V=9001, k=3, d=3, W=3, b=3, B_verify=18, alpha=0.8, omega=0, selection=0, accept_model=1, marginal=1, dtype='bf16', seed=780, cost=(0.005371, 0.0, 0.041229, 0.01346, 1.370219, 1.914697, 1.0), sigma_m=0.5, a_lo=7.305, a_hi=13.801),
    Case(V=9001, k=6, d=3, W=0, b=4, B_verify=80, alpha=1.0, omega=1, selection=1, accept_model=0, marginal=0, dtype='fp32', seed=923, cost=(0.010057, 0.0, 0.040986, 0.007588, 1.275317, 1.719908, 1.0), sigma_m=0.5, a_lo=7.926, a_hi=11.342),
    Case(V=20000, k=3, d=4, W=3, b=3, B_verify=27, alpha=1.0, omega=1, selection=1, accept_model=0, marginal=0, dtype='bf16', seed=1008, cost=(0.002231, 0.0, 0.04857, 0.003145, 1.266795, 1.42984, 1.0), sigma_m=0.5, a_lo=3.239, a_hi=13.834),
    Case(V=9001, k=5, d=4, W=0, b=4, B_verify=56, alpha=1.0, omega=1, selection=1, accept_model=0, marginal=1, dtype='bf16', seed=1074, cost=(0.003233, 0.0, 0.00134, 0.017097, 1.179637, 1.402959, 1.0), sigma_m=0.5, a_lo=7.529, a_hi=12.748),
    Case(V=40001, k=4, d=5, W=4, b=2, B_verify=10, alpha=1.0, omega=1, selection=1, accept_model=0, marginal=1, dtype='fp32', seed=191, cost=(0.004373, 0.0, 0.026322, 0.014431, 1.173766, 1.556655, 1.0), sigma_m=0.5, a_lo=5.664, a_hi=13.026),
    Case(V=9001, k=4, d=4, W=0, b=3, B_verify=24, alpha=1.0, omega=0, selection=1, accept_model=1, marginal=0, dtype='fp32', seed=267, cost=(0.010978, 0.0, 0.001829, 0.015514, 1.295275, 1.009407, 1.0), sigma_m=0.5, a_lo=6.212, a_hi=13.698),
    Case(V=20000, k=5, d=5, W=5, b=5, B_verify=70, alpha=1.0, omega=0, selection=1, accept_model=1, marginal=0, dtype='fp32', seed=381, cost=(0.003111, 0.0, 0.014269, 0.019977, 1.1975, 1.52077, 1.0), sigma_m=0.5, a_lo=7.490, a_hi=10.455),
    Case(V=9001, k=7, d=4, W=0, b=5, B_verify=115, alpha=1.0, omega=0, selection=1, accept_model=1, marginal=1, dtype='bf16', seed=458, cost=(0.006692, 0.0, 0.02317, 0.012523, 1.286867, 1.65413, 1.0), sigma_m=0.5, a_lo=5.633, a_hi=11.772),
    Case(V=9001, k=6, d=4, W=6, b=6, B_verify=96, alpha=1.0, omega=0, selection=1, accept_model=1, marginal=1, dtype='bf16', seed=560, cost=(0.022093, 0.0, 0.040561, 0.00997, 1.077764, 0.980571, 1.0), sigma_m=0.5, a_lo=5.283, a_hi=9.776),
]
MODE_IDS = [f"{['PREFIX', 'FROZEN'][c.selection]}-{['NODE_SUM', 'PATH_MEAN'][c.accept_model]}-"
            f"{['DERIV', 'DIFF'][c.marginal]}-W{'k' if c.W else '0'}" for c in MODES]


@pytest.mark.parametrize("case", MODES, ids=MODE_IDS)
def test_every_mode_nontrivial(case):
    orc, gpu, layers = _run(case)
    admitting = sum(1 for l in range(case.d) if orc.trace[l, 3] > 0)
    assert orc.N >= 2 * case.b and admitting >= 3, (orc.N, admitting)  # a real multi-admit cut
    assert layers == case.d


def test_local_cost_scope_replica():
    """cost_scope LOCAL (Q13, Q34): a context owning requests [off, off + b_loc) of a b_glob batch
    costs its share as its own batch (independent target replica) with B = floor(B_verify / b_glob);
    compared with the oracle run on that slice with b_budget = b_glob."""
    from inputs import synth
    from oracle import oracle as O
    from paper_2604_09731_b200 import smart as S
    import torch
    V, k, d, W, b_glob, Bv = 20000, 5, 4, 5, 8, 96
    cost = (0.002, 0.0, 0.03, 0.01, 1.2, 1.5, 1.0)
    for off, b_loc in ((0, 3), (3, 5)):
        case = Case(V=V, k=k, d=d, W=W, b=b_loc, B_verify=Bv, seed=77, cost=cost, a_lo=5.0, a_hi=12.0)
        ocfg = O.Config(V=V, k=k, d=d, W=W, b=b_loc, B_verify=Bv, alpha=case.alpha, omega=1, b_budget=b_glob)
        T = ocfg.tmax()
        draft = synth.draft_pool(77, b_loc, T, V, r_offset=off, a_lo=5.0, a_hi=12.0)
        target = synth.target_pool(draft, 1077, 1.0, r_offset=off)
        rt = np.arange(b_loc, dtype=np.int32) + off
        rp = np.full(b_loc, 10, np.int32)
        lam, beta, gamma, delta, rho, eta, c_T = cost
        orc = O.step(ocfg, O.Cost(lam=lam, beta=beta, gamma=gamma, delta=delta, rho=rho, eta=eta, c_T=c_T),
                     draft, target, root_tok=rt, root_pos=rp)
        assert orc.N >= 2 * b_loc
        cfg = S.Config(vocab=V, top_k=k, max_depth=d, max_frontier=W, batch_local=b_loc, batch_global=b_glob,
                       batch_offset=off, budget_verify=Bv, alpha=case.alpha, bonus=1, cost_scope=S.COST_LOCAL,
                       row_mode=S.ROWS_NODE)
        ctx = S.Smart(cfg, S.Cost(lam=lam, beta=beta, gamma=gamma, delta=delta, rho=rho, eta=eta, c_T=c_T))
        assert ctx.sizes["T"] == T
        out = ctx.alloc_outputs()
        ctx.begin_step(to_dev(rt), to_dev(rp))
        for l in range(1, d + 1):
            ctx.expand_step(l, to_dev(draft))
            ctx.select(l)
        ctx.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"])
        ctx.verify_accept(to_dev(target), out["accept_len"], out["accept_path"], out["bonus"])
        torch.cuda.synchronize()
        gpu = {kk: v.cpu().numpy() for kk, v in out.items()}
        gpu["stats"], gpu["tree"] = ctx.stats(), ctx.tree()
        gpu["cands"] = {l: ctx.candidates(l) for l in range(1, d + 1) if gpu["stats"]["layers"][l - 1]["executed"]}
        # the oracle numbers requests of the slice 0..b_loc-1; the GPU reports local indices too
        compare(case, orc, gpu)


def test_run_step_equals_separate_calls():
    case = Case(V=50000, k=6, d=5, W=6, b=5, B_verify=60, seed=3)
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    a = run_gpu(case, draft, target, rt, rp)
    b = run_gpu(case, draft, target, rt, rp, use_run_step=True)
    for key in ("mask", "pos", "parent", "tok", "tree_len", "accept_len", "accept_path", "bonus"):
        np.testing.assert_array_equal(a[key], b[key])


# ---- the step kernel's small-batch selection (select_small) and its hand-overs:
# each case is compared with the oracle on both paths (_run) and the step kernel's per-layer
# select_path trace shows the branch taken: 1 the one-warp threshold path, 2 the same with the full
# sorted list rebuilt for argmax_j (non-convex cost window), 3 handed over to the block selection
# (more than 64 candidates above the threshold / a long eligible list, or theta unusable) -------

SMALL = {
    "convex_cfg3like": (Case(V=30000, k=8, d=5, W=8, b=32, B_verify=200, seed=90, a_lo=8.0, a_hi=14.0, sigma_m=0.5,
                             cost=(0.0117, 0.0, 0.05, 0.02, 1.3, 2.4631, 2.4631)), {1}),
    "concave_cost": (Case(V=30000, k=6, d=5, W=6, b=8, B_verify=96, seed=48, a_lo=6.0, a_hi=12.0, sigma_m=0.5,
                          cost=(0.001, 0.0, 0.2, 0.05, 0.7, 1.5, 1.0)), {2}),
    "many_above": (Case(V=20000, k=8, d=4, W=8, b=32, B_verify=2048, seed=60,
                        cost=(0.0001, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0)), {3}),  # 63-77 admitted per layer
    "omega0_node_sum": (Case(V=30000, k=5, d=5, W=5, b=6, B_verify=60, omega=0, seed=72, a_lo=6.0, a_hi=12.0,
                             sigma_m=0.5, cost=(0.01, 0.0, 0.05, 0.02, 1.2, 1.5, 1.0)), {3}),
}


# full-mantissa fp32 logits (the fp32 path otherwise only sees bf16-representable values)
FP32_FULL = {
    "cfg3_fp32full": Case(V=128256, k=8, d=6, W=8, b=32, B_verify=200, seed=12, dtype="fp32full",
                          cost=(0.0117, 0.0, 0.05, 0.02, 1.3, 2.4631, 2.4631)),
    "mid_fp32full_frozen": Case(V=30000, k=6, d=5, W=6, b=8, B_verify=96, seed=48, dtype="fp32full", selection=1,
                                a_lo=6.0, a_hi=12.0, sigma_m=0.5, cost=(0.001, 0.0, 0.2, 0.05, 0.7, 1.5, 1.0)),
}


@pytest.mark.parametrize("name", list(FP32_FULL))
def test_fp32_full_mantissa(name):
    case = FP32_FULL[name]
    orc, gpu, layers = _run(case)
    assert sum(1 for l in range(case.d) if orc.trace[l, 3] > 0) >= 3 and layers == case.d


@pytest.mark.parametrize("name", list(SMALL))
def test_small_selection_paths(name):
    case, want = SMALL[name]
    orc, gpu, layers = _run(case)
    assert sum(1 for l in range(case.d) if orc.trace[l, 3] > 0) >= 2, "the case must admit in >= 2 layers"
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    step = run_gpu(case, draft, target, rt, rp, use_run_step=True)
    paths = [step["stats"]["layers"][l]["select_path"] for l in range(case.d) if step["stats"]["layers"][l]["executed"]]
    assert want & set(paths), paths
    assert set(paths) <= {1, 2, 3}, paths


# ---- BASELINE.json configs at full size ------------------------------------------------------

FULL = {
    # cfg2: Llama-3.1-8B-shaped, b=1, d=6, k=10, EAGLE-style W=10, B_verify=60
    "cfg2_llama8b_b1": Case(V=128256, k=10, d=6, W=10, b=1, B_verify=60, seed=11,
                            cost=(0.0117, 0.0, 0.0, 0.0, 1.0, 2.4631, 2.4631)),
    # cfg3: Llama-3.1-8B-shaped compute-bound regime, b=32, d=6, k=8, B_verify=200
    "cfg3_llama8b_b32": Case(V=128256, k=8, d=6, W=8, b=32, B_verify=200, seed=12,
                             cost=(0.0117, 0.0, 0.05, 0.02, 1.3, 2.4631, 2.4631)),
    # cfg4: Qwen2-VL-7B-shaped MSD-style, b=12, d=8, k=10
    "cfg4_qwen2vl_b12": Case(V=152064, k=10, d=8, W=10, b=12, B_verify=200, seed=13,
                             cost=(0.0105, 0.0, 0.04, 0.02, 1.3, 2.20, 2.20)),
}


@pytest.mark.parametrize("name", list(FULL))
def test_full_size_configs(name):
    _run(FULL[name])


# cfg5-sized batches: b = 256 (standalone 1024-thread select, bitonic global sort over up to
# 2048 eligible keys) and b = 64 with the PATH_MEAN model (fused select); a cost model cheap
# enough per node that trees still grow at these batch sizes
LARGE_B = {
    "b256_node_sum": Case(V=20000, k=8, d=4, W=8, b=256, B_verify=2048, seed=41,
                          cost=(0.0005, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0)),
    "b64_path_mean": Case(V=30000, k=6, d=5, W=6, b=64, B_verify=512, seed=42, accept_model=1, omega=0,
                          selection=1, cost=(0.0005, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0)),
    # cfg5 at full size (BASELINE.json configs[4] on one GPU): V = 152064, b = 256, d = 6, k = 8,
    # B_verify = 2048 (B = 8) -- the bench's roofline_hbm_regime shape, element by element
    "cfg5_full": Case(V=152064, k=8, d=6, W=8, b=256, B_verify=2048, seed=43,
                      cost=(0.0005, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0)),
}


@pytest.mark.parametrize("name", list(LARGE_B))
def test_large_batch(name):
    orc, gpu, layers = _run(LARGE_B[name])
    assert orc.N > LARGE_B[name].b and layers >= 2  # non-trivial trees were compared


def test_full_size_fp32_logits():
    c = FULL["cfg3_llama8b_b32"]
    _run(Case(**{**c.__dict__, "dtype": "fp32", "b": 8, "seed": 21}))


# ---- edge cases ----------------------------------------------------------------------------

def test_unaligned_rows_scalar_path():
    """ld*esz not a multiple of 16 -> the scalar (non-vector) load path."""
    _run(Case(V=9999, k=5, d=4, W=5, b=3, B_verify=30, dtype="bf16", ld_pad=3, seed=5))
    _run(Case(V=9999, k=5, d=4, W=5, b=3, B_verify=30, dtype="fp32", ld_pad=1, seed=6))


def test_tiny_vocab_single_chunk():
    _run(Case(V=37, k=3, d=4, W=0, b=2, B_verify=20, dtype="fp32", seed=7, a_lo=1, a_hi=3, sigma_bg=1.0))


def test_depth_zero_and_budget_one():
    _run(Case(V=3000, k=4, d=0, W=4, b=2, B_verify=8, seed=8))
    _run(Case(V=3000, k=4, d=5, W=4, b=4, B_verify=4, seed=9))   # B = 1


def test_edge_rows_ties_and_neg_inf():
    """all-equal rows, -inf entries, k-th/(k+1)-th ties: exact top-k order (Q9, Q23)."""
    import torch
    from inputs import synth
    from oracle import oracle as O
    for kind in ("all_equal", "neg_inf", "kth_tie"):
        V, k = 20000, 6
        case = Case(V=V, k=k, d=3, W=0, b=2, B_verify=40, dtype="bf16", seed=1)
        T = _T(case)
        draft, target, rt, rp = make_inputs(case, T)
        row = synth.f32_to_bf16_bits(synth.edge_rows(kind, V, k, seed=3))
        draft[:, :, :] = row[None, None, :]
        orc = run_oracle(case, draft, target, rt, rp)
        gpu = run_gpu(case, draft, target, rt, rp)
        compare(case, orc, gpu, allow_ambiguous=True)


def test_nan_row_sets_device_flag():
    from inputs import synth
    from paper_2604_09731_b200 import smart as S
    case = Case(V=5000, k=4, d=2, W=4, b=2, B_verify=20, seed=2)
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    draft[1, 0, :] = synth.f32_to_bf16_bits(synth.edge_rows("nan", 5000, 4))
    gpu = run_gpu(case, draft, target, rt, rp)
    assert gpu["stats"]["error_flags"] & 1
    with pytest.raises(S.SmartError) as e:
        gpu["ctx"].stats(raise_on_device_flag=True)
    assert e.value.status == S.EDEVICE
    with pytest.raises(ValueError):
        run_oracle(case, draft, target, rt, rp)


def test_frontier_row_mode_matches_node_mode():
    """ROWS_FRONTIER (what a real draft forward produces) gives the same tree as ROWS_NODE."""
    import torch
    from paper_2604_09731_b200 import smart as S
    from smart_gpu_cases import gpu_ctx
    case = Case(V=30000, k=5, d=5, W=5, b=4, B_verify=60, seed=4)
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    ref = run_gpu(case, draft, target, rt, rp)
    ctx = gpu_ctx(case, row_mode=S.ROWS_FRONTIER)
    dd = to_dev(draft)
    cap = ctx.sizes["frontier_cap"]
    fr = torch.zeros((cap, 2), dtype=torch.int32, device="cuda")
    cnt = torch.zeros((1,), dtype=torch.int32, device="cuda")
    ctx.begin_step(to_dev(rt), to_dev(rp))
    rows = dd[:, 0, :].contiguous()  # layer 1: the roots, one row per request
    for l in range(1, case.d + 1):
        ctx.expand_step(l, rows)
        ctx.select(l, fr, cnt)
        n = int(cnt.item())
        if n == 0:
            break
        f = fr[:n].long()
        rows = dd[f[:, 0], f[:, 1], :].contiguous()  # the "draft forward" over the frontier
    out = ctx.alloc_outputs()
    ctx.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out["tok"].cpu().numpy(), ref["tok"])
    np.testing.assert_array_equal(out["parent"].cpu().numpy(), ref["parent"])
    np.testing.assert_array_equal(out["mask"].cpu().numpy(), ref["mask"])


def test_verify_draft_equals_target_accepts_top1_chain():
    """sigma_m = 0 (target == draft): the walk accepts the longest top-1 chain."""
    case = Case(V=40000, k=4, d=6, W=4, b=6, B_verify=120, seed=10, sigma_m=0.0)
    orc, gpu, _ = _run(case)
    assert gpu["accept_len"].sum() > 0


def test_step_is_repeatable_and_graph_capturable():
    """Same inputs -> bit-identical outputs; the step replays from a captured CUDA graph."""
    import torch
    case = FULL["cfg3_llama8b_b32"]
    T = _T(case)
    draft, target, rt, rp = make_inputs(case, T)
    from smart_gpu_cases import gpu_ctx
    ctx = gpu_ctx(case)
    dd, tt, rtd, rpd = to_dev(draft), to_dev(target), to_dev(rt), to_dev(rp)
    out = ctx.alloc_outputs()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx.run_step(dd, tt, out, root_tok=rtd, root_pos=rpd, stream=s)
    s.synchronize()
    ref = {k: v.clone() for k, v in out.items()}
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.run_step(dd, tt, out, root_tok=rtd, root_pos=rpd, stream=s)
    for _ in range(3):
        for v in out.values():
            v.zero_()
        g.replay()
        torch.cuda.synchronize()
        for k in ref:
            assert torch.equal(ref[k], out[k]), k
