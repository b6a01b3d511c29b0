"""Oracle pins for NEXT #4 (second tree source): DFLASH position rows.

DFLASH "generates all draft tokens in a single non-autoregressive forward pass ... produces
independent top-k candidates at each position; we construct an EAGLE-2 style tree by taking the
Cartesian product of candidates across positions and pruning to the top-g tokens by cumulative
probability".  In the oracle this is row_mode = ROWS_POSITION: every frontier node of
request r at layer l expands with the request's position-l row.  Pins:

* baseline (selection BASELINE, W >= g): the kept node set equals the top-g of an explicit
  enumeration of the Cartesian product (all k + k^2 + ... + k^d token paths) by cum, with cum the
  product of independently computed per-position softmax probabilities (numpy fp64);
* SMART on position rows equals SMART on a k-ary pool whose every node row at depth l-1 is a copy
  of position row l (the ROWS_KARY addressing, pinned elsewhere);
* every node of a SMART tree carries its position's top-k token and p = softmax(position)[token].
"""
import itertools

import numpy as np
import pytest

from oracle import oracle as O


@pytest.fixture(scope="module", autouse=True)
def _build():
    O.build()


def _pos_pool(rng, b, d, V):
    x = (rng.standard_normal((b, d, V)) * 1.5).astype(np.float32)
    heads = rng.integers(0, V, size=(b, d, 3))
    for r in range(b):
        for l in range(d):
            x[r, l, heads[r, l]] += rng.uniform(1, 4, 3).astype(np.float32)
    return x


def _softmax_topk(row, k):
    x = row.astype(np.float64)
    p = np.exp(x - x.max())
    p /= p.sum()
    order = np.lexsort((np.arange(len(x)), -x))[:k]  # value desc, id asc (Q9)
    return order, p


def _paths(res, r):
    """token path (tuple) of every drafted node of request r, with its cum"""
    n = int(res.n_nodes[r])
    out = {}
    for u in range(1, n):
        path, v = [], u
        while v > 0:
            path.append(int(res.tok[r, v]))
            v = int(res.parent[r, v])
        out[tuple(reversed(path))] = float(res.cum[r, u])
    return out


@pytest.mark.parametrize("seed", range(6))
def test_baseline_is_top_g_of_cartesian_product(seed):
    rng = np.random.default_rng(100 + seed)
    b, d, k, V = 2, 3, 3, 40
    g = int(rng.integers(4, 20))
    pool = _pos_pool(rng, b, d, V)
    cfg = O.Config(V=V, k=k, d=d, W=g, b=b, B_verify=g * b, dtype=O.FP32,
                   row_mode=O.ROWS_POSITION)
    res = O.baseline_step(cfg, pool)
    for r in range(b):
        tops = [_softmax_topk(pool[r, l], k) for l in range(d)]
        prod = {}
        for depth in range(1, d + 1):
            for ranks in itertools.product(range(k), repeat=depth):
                toks = tuple(int(tops[l][0][j]) for l, j in enumerate(ranks))
                prod[toks] = float(np.prod([tops[l][1][tops[l][0][j]] for l, j in enumerate(ranks)]))
        want = sorted(prod, key=lambda t: -prod[t])[:g]
        got = _paths(res, r)
        assert set(got) == set(want), (r, sorted(got), sorted(want))
        for t in got:
            assert abs(got[t] - prod[t]) <= 1e-12 * prod[t]


@pytest.mark.parametrize("seed", range(4))
def test_smart_position_rows_equal_replicated_kary_rows(seed):
    rng = np.random.default_rng(200 + seed)
    b, d, k, V = 2, 3, 2, 24
    pool = _pos_pool(rng, b, d, V)
    n = sum(k ** l for l in range(d + 1))
    depth_of = np.zeros(n, np.int64)
    for f in range(1, n):
        depth_of[f] = depth_of[(f - 1) // k] + 1
    kary = np.zeros((b, n, V), np.float32)
    for f in range(n):
        kary[:, f] = pool[:, min(depth_of[f], d - 1)]  # node at depth l-1 expands with position l
    cost = O.Cost(lam=0.1, gamma=0.05, delta=0.05, rho=1.2, eta=1.0, c_T=1.0)
    common = dict(V=V, k=k, d=d, W=0, b=b, B_verify=40 * b, dtype=O.FP32)
    a = O.step(O.Config(row_mode=O.ROWS_POSITION, **common), cost, pool)
    c = O.step(O.Config(row_mode=O.ROWS_KARY, **common), cost, kary)
    np.testing.assert_array_equal(a.n_nodes, c.n_nodes)
    np.testing.assert_array_equal(a.tok, c.tok)
    np.testing.assert_array_equal(a.parent, c.parent)
    np.testing.assert_array_equal(a.cum, c.cum)
    np.testing.assert_array_equal(a.trace, c.trace)


@pytest.mark.parametrize("seed", range(4))
def test_smart_tree_nodes_carry_position_topk(seed):
    rng = np.random.default_rng(300 + seed)
    b, d, k, V = 3, 4, 4, 64
    pool = _pos_pool(rng, b, d, V)
    cost = O.Cost(lam=0.05, gamma=0.02, delta=0.02, rho=1.3, eta=1.0, c_T=1.0)
    res = O.step(O.Config(V=V, k=k, d=d, W=k, b=b, B_verify=16 * b, dtype=O.FP32, row_mode=O.ROWS_POSITION),
                 cost, pool)
    assert res.n_nodes.sum() > b  # the step drafted something
    for r in range(b):
        for u in range(1, int(res.n_nodes[r])):
            l = int(res.depth[r, u])
            top, p = _softmax_topk(pool[r, l - 1], k)
            t = int(res.tok[r, u])
            assert t in set(int(x) for x in top)
            assert abs(res.p[r, u] - p[t]) <= 1e-12 * p[t]
            par = int(res.parent[r, u])
            assert abs(res.cum[r, u] - res.cum[r, par] * res.p[r, u]) <= 1e-15
