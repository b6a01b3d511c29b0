"""NEXT #1 pins (reading Q31): tree verification at temperature tau > 0.

The oracle draws one target token per visited node by Gumbel-max over the target row with a
counter-based uniform keyed by (seed, request, node, token), follows the child holding it, else
stops with that token as the bonus.  What the method fixes, and what is checked here:
  * losslessness: on a single-child chain the first emitted token is distributed as
    the target conditional softmax(logits / tau) -- total variation < 0.01 over 100k trials;
  * acceptance frequency of a node with several children = sum of the children's target
    probabilities (SPEC S:392 analytic sum), within 2% over 100k trials;
  * tau -> 0 reduces to the greedy walk of A8 (orc_step's verification) on random trees;
  * the uniform stream is uniform (moments) and keyed (distinct keys, distinct values).
"""
import numpy as np

from oracle import oracle as O


def softmax(x, tau=1.0):
    z = np.exp((x - x.max()) / tau)
    return z / z.sum()


def _batch_rows(rows, n):
    """target [n, T, V] float32 with the same rows for every request (requests differ in keys)."""
    return np.ascontiguousarray(np.broadcast_to(rows.astype(np.float32), (n,) + rows.shape))


def test_uniform_moments_and_keys():
    u = np.array([O.uniform(7, r, n, v) for r in range(20) for n in range(10) for v in range(1000)])
    assert 0.0 < u.min() and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.003
    assert abs(u.var() - 1.0 / 12.0) < 0.002
    assert len(np.unique(u)) > 0.97 * len(u)  # 23-bit values, 200k draws: nearly all distinct
    assert O.uniform(7, 0, 0, 0) != O.uniform(8, 0, 0, 0)


def test_lossless_single_child_chain():
    rng = np.random.default_rng(0)
    V, n = 6, 100_000
    root_row = rng.normal(0, 1.5, V)
    child_row = rng.normal(0, 1.5, V)
    t_child = int(np.argsort(-root_row)[1])  # the child is the target's 2nd choice
    target = _batch_rows(np.stack([root_row, child_row]), n)
    nn = np.full(n, 2)
    parent = np.tile(np.array([-1, 0]), (n, 1))
    tok = np.tile(np.array([-1, t_child]), (n, 1))
    a, path, bonus, _ = O.verify_sample(target, nn, parent, tok, 1.0, seed=123, d=1)
    first = np.where(a >= 1, t_child, bonus)
    freq = np.bincount(first, minlength=V) / n
    tv = 0.5 * np.abs(freq - softmax(root_row)).sum()
    assert tv < 0.01, tv
    # after an accepted child the walk continues at the child (its bonus is a sample of its row)
    acc = a >= 1
    f2 = np.bincount(bonus[acc], minlength=V) / acc.sum()
    assert 0.5 * np.abs(f2 - softmax(child_row)).sum() < 0.02


def test_multi_child_acceptance_frequency():
    rng = np.random.default_rng(1)
    V, n = 10, 100_000
    row = rng.normal(0, 1.0, V)
    kids = [3, 7, 1]
    T = 1 + len(kids)
    rows = np.stack([row] + [rng.normal(0, 1, V) for _ in kids])
    target = _batch_rows(rows, n)
    nn = np.full(n, T)
    parent = np.tile(np.array([-1] + [0] * len(kids)), (n, 1))
    tok = np.tile(np.array([-1] + kids), (n, 1))
    a, path, bonus, _ = O.verify_sample(target, nn, parent, tok, 1.0, seed=5, d=1)
    p = softmax(row)
    assert abs((a >= 1).mean() - p[kids].sum()) < 0.02 * p[kids].sum() + 0.002
    # the accepted child is the one holding the sampled token, with probability p(t)
    for j, t in enumerate(kids):
        assert abs((path[:, 0] == j + 1).mean() - p[t]) < 0.01


def test_temperature_scales_the_target():
    rng = np.random.default_rng(2)
    V, n, tau = 5, 100_000, 0.5
    row = rng.normal(0, 1.0, V)
    target = _batch_rows(row[None, :], n)
    a, _, bonus, _ = O.verify_sample(target, np.ones(n), np.full((n, 1), -1), np.full((n, 1), -1), tau,
                                     seed=9, d=1)
    assert (a == 0).all()  # empty tree: zero accepted, bonus = a target sample
    freq = np.bincount(bonus, minlength=V) / n
    assert 0.5 * np.abs(freq - softmax(row, tau)).sum() < 0.01


def test_low_temperature_equals_greedy_walk():
    from inputs import synth
    cfg = O.Config(V=3000, k=4, d=4, W=4, b=6, B_verify=60, alpha=0.8, omega=1, dtype=O.FP32)
    cost = O.Cost(lam=0.02, gamma=0.05, delta=0.01, rho=1.2, eta=1.0, c_T=1.0)
    T = cfg.tmax()
    draft = synth.draft_pool(3, cfg.b, T, cfg.V, dtype="fp32", a_lo=10, a_hi=18)
    target = synth.target_pool(draft, 4, 1.0, V=cfg.V)
    res = O.step(cfg, cost, draft, target)
    assert res.N > cfg.b
    a, path, bonus, mg = O.verify_sample(target, res.n_nodes, res.parent, res.tok, 1e-4, seed=77, d=cfg.d)
    np.testing.assert_array_equal(a, res.accept_len)
    np.testing.assert_array_equal(path, res.accept_path)
    np.testing.assert_array_equal(bonus, res.bonus)
    assert (mg > 0).all()
