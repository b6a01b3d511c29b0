"""Pins of the oracle's closed-form pieces against values the paper/SPEC fix.

Each test names the passage it follows.  These are `-m "not gpu"` tests: they pin
oracle/smart_oracle.c to something other than itself (worked values, closed forms,
library routines, finite differences, brute-force enumeration).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_fixtures.json")


@pytest.fixture(scope="module")
def spec():
    with open(GOLD) as f:
        return json.load(f)


def test_draft_cost_spec_values(orc, spec):
    """Eq.(4)."""
    for ex in spec["draft_cost"]:
        c = orc.Cost(lam=ex["lam"], beta=ex["beta"])
        assert orc.cost_draft(c, ex["x"]) == pytest.approx(ex["value"], rel=1e-12, abs=1e-12), ex["cite"]


def test_verify_cost_spec_values(orc, spec):
    """Eq.(5); SPEC S:135-137 (delta=0 -> eta; e-1 closed form; origin)."""
    for ex in spec["verify_cost"]:
        c = orc.Cost(lam=0, gamma=ex["gamma"], delta=ex["delta"], rho=ex["rho"], eta=ex["eta"])
        v, sat = orc.cost_verify(c, ex["x"])
        assert not sat
        assert v == pytest.approx(ex["value"], rel=1e-12, abs=1e-15), ex["cite"]


def test_verify_cost_saturates(orc):
    """S:133 / S:184 / Q17: exponent > 700 saturates (finite) and flags."""
    c = orc.Cost(lam=0, gamma=1.0, delta=10.0, rho=2.0)
    v, sat = orc.cost_verify(c, 100)
    assert sat and math.isfinite(v) and v == pytest.approx(math.exp(700) - 1)
    v, sat = orc.cost_verify(c, 1)
    assert not sat and v == pytest.approx(math.exp(10) - 1)


def test_marginal_cost_closed_forms(orc):
    """Eq.(15) P:334-342 special cases: rho=1 -> lam + gamma*delta*e^(delta x);
    gamma=0 -> lam."""
    for lam, g, dl, x in [(0.3, 2.0, 0.05, 7), (1.0, 0.5, 0.01, 40), (0.0, 1.0, 0.2, 3)]:
        c = orc.Cost(lam=lam, gamma=g, delta=dl, rho=1.0)
        v, _ = orc.dc(c, x)
        assert v == pytest.approx(lam + g * dl * math.exp(dl * x), rel=1e-13)
    c = orc.Cost(lam=0.7, gamma=0.0, delta=0.3, rho=1.4)
    assert orc.dc(c, 12)[0] == pytest.approx(0.7, rel=1e-15)


def test_marginal_cost_matches_central_difference(orc):
    """Eq.(15) derivative within 2% of the central difference C(x+.5)-C(x-.5), x in [2,60],
    over a parameter grid — pins the derivative against the cost function itself."""
    for lam, g, dl, rho in itertools.product([0.0, 0.4], [0.5, 2.0], [0.002, 0.02], [0.8, 1.0, 1.3]):
        c = orc.Cost(lam=lam, gamma=g, delta=dl, rho=rho)
        for x in range(2, 61):
            if dl * (x + 1) ** rho > 5:
                continue
            fd = orc.cost_spec(c, x + 0.5) - orc.cost_spec(c, x - 0.5)
            der, _ = orc.dc(c, x)
            assert der == pytest.approx(fd, rel=0.02), (lam, g, dl, rho, x)


def test_difference_mode_telescopes(orc):
    """Q5: DIFFERENCE = cost(N+1)-cost(N), so summing 0..n-1 gives cost(n)-cost(0) exactly
    (up to rounding); the derivative mode telescopes within 5%."""
    c = orc.Cost(lam=0.3, gamma=0.8, delta=0.03, rho=1.2, eta=2.0)
    for n in (1, 5, 20, 60):
        s_diff = sum(orc.dc(c, N, orc.DIFFERENCE)[0] for N in range(n))
        assert s_diff == pytest.approx(orc.cost_spec(c, n) - orc.cost_spec(c, 0), rel=1e-12)
        if n >= 5:
            s_der = sum(orc.dc(c, N)[0] for N in range(1, n + 1))
            assert s_der == pytest.approx(orc.cost_spec(c, n) - orc.cost_spec(c, 0), rel=0.05)


def test_cost_monotone_and_positive_marginal(orc):
    """C_verify nondecreasing in |T|; marginal > 0 when lam > 0 or gamma*delta*rho > 0."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        c = orc.Cost(lam=rng.uniform(0, 1), gamma=rng.uniform(0, 3), delta=rng.uniform(0, 0.05),
                     rho=rng.uniform(0.3, 2.0))
        vals = [orc.cost_verify(c, x)[0] for x in range(0, 129)]
        assert all(b >= a for a, b in zip(vals, vals[1:]))
        assert all(orc.dc(c, x)[0] > 0 for x in (1, 7, 64))


def test_rule_spec_values(orc, spec):
    """Eq.(12)/(16) P:294-300."""
    for ex in spec["rule"]:
        dj = orc.delta_j(ex["alpha"], ex["ratio"], 1.0, ex["global"], 1.0)
        assert dj == pytest.approx(ex["delta_j"], abs=1e-12), ex["cite"]
        assert (dj > 0) == ex["admitted"]
    # empty-tree seed: c_spec = 0 -> global term 0
    assert orc.delta_j(0.8, 0.3, 2.0, 0.0, 0.0) == pytest.approx(0.12)


def test_acceptance_spec_values(orc, spec):
    """Eq.(2)."""
    for ex in spec["acceptance"]:
        assert orc.l_tree_path_mean(ex["parent"], ex["cum"]) == pytest.approx(ex["path_mean"], abs=1e-15)


def test_reward_spec_value(orc, spec):
    """Eq.(1)/(9) P:139-145; S:234 (chain (.5,.5), c_T=10, lam=1, gamma=0 ->
    C_target 7.5, C_spec 2, R 3.75).  PAPER preset: b=1, omega=0."""
    ex = spec["reward"][0]
    c = orc.Cost(lam=ex["lam"], gamma=ex["gamma"], c_T=ex["c_T"])
    L = orc.l_tree_path_mean(ex["parent"], ex["cum"])
    n = len(ex["parent"]) - 1
    assert ex["c_T"] * L == pytest.approx(ex["c_target"])
    assert orc.cost_spec(c, n) == pytest.approx(ex["c_spec"])
    assert orc.speedup(c, 0, 1, L, n) == pytest.approx(ex["R"], rel=1e-14)
    # empty tree: 0/0 := 0 (Q4); HOTPATH seed omega=1, eta=c_T -> S(empty) = 1 (Q19)
    assert orc.speedup(c, 0, 1, 0.0, 0) == 0.0
    c2 = orc.Cost(lam=1.0, eta=10.0, c_T=10.0)
    for b in (1, 4, 32):
        assert orc.speedup(c2, 1, b, 0.0, 0) == pytest.approx(1.0)
    # S scales linearly in c_T
    c3 = orc.Cost(lam=ex["lam"], gamma=ex["gamma"], c_T=2 * ex["c_T"])
    assert orc.speedup(c3, 0, 1, L, n) == pytest.approx(2 * ex["R"])


def _random_tree(rng, n):
    parent = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
    p = [1.0] + list(rng.uniform(0.05, 1.0, n - 1))
    cum = [1.0]
    for i in range(1, n):
        cum.append(cum[parent[i]] * p[i])
    return parent, cum


def test_path_mean_invariants(orc):
    """Eq.(2): invariant under child reordering; equals the node sum on chains;
    brute-force leaf enumeration via an explicit path list."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 12))
        parent, cum = _random_tree(rng, n)
        # explicit path enumeration
        kids = {i: [j for j in range(n) if parent[j] == i] for i in range(n)}
        paths = []

        def walk(u, acc):
            if not kids[u]:
                paths.append(acc)
            for v in kids[u]:
                walk(v, acc + cum[v])
        walk(0, 0.0)
        ref = sum(paths) / len(paths)
        assert orc.l_tree_path_mean(parent, cum) == pytest.approx(ref, rel=1e-12, abs=1e-15)
        # relabel nodes by a random topological permutation -> same value
        perm = [0] + list(1 + rng.permutation(n - 1)) if n > 1 else [0]
        order = sorted(range(n), key=lambda i: (_depth(parent, i), perm[i]))
        newid = {old: new for new, old in enumerate(order)}
        par2 = [-1 if parent[o] < 0 else newid[parent[o]] for o in order]
        cum2 = [cum[o] for o in order]
        assert orc.l_tree_path_mean(par2, cum2) == pytest.approx(ref, rel=1e-12, abs=1e-15)
    # chain: path mean == node sum
    cum = [1.0, 0.9, 0.45, 0.3]
    assert orc.l_tree_path_mean([-1, 0, 1, 2], cum) == pytest.approx(orc.l_tree_node_sum(cum))


def _depth(parent, i):
    d = 0
    while parent[i] >= 0:
        i = parent[i]
        d += 1
    return d


def test_node_sum_is_exact_expected_acceptance(orc):
    """P:160 ("expected number of consecutively accepted tokens equals the sum of the
    probabilities that each prefix is accepted"): with draft == target, the expected greedy-walk
    acceptance of a tree equals sum(cum) (Q11).  Brute force over every target outcome."""
    rng = np.random.default_rng(5)
    V, depth = 4, 3
    for _ in range(40):
        # a draft distribution per context (tuple of tokens)
        dist = {}

        def q(ctx):
            if ctx not in dist:
                dist[ctx] = rng.dirichlet(np.ones(V))
            return dist[ctx]
        # random tree over tokens: each node keeps a random subset of its children
        tok, parent, cum, ctx_of = [-1], [-1], [1.0], [()]
        frontier = [0]
        for _l in range(depth):
            nxt = []
            for u in frontier:
                for t in rng.permutation(V)[: int(rng.integers(0, 3))]:
                    tok.append(int(t)); parent.append(u)
                    cum.append(cum[u] * q(ctx_of[u])[t]); ctx_of.append(ctx_of[u] + (int(t),))
                    nxt.append(len(tok) - 1)
            frontier = nxt
        # enumerate all target token sequences of length `depth`
        expect = 0.0
        for seq in itertools.product(range(V), repeat=depth):
            pr, ctx, cur, acc = 1.0, (), 0, 0
            for t in seq:
                pr *= q(ctx)[t]
                ctx = ctx + (t,)
            ctx, cur = (), 0
            for t in seq:
                kid = [j for j in range(len(tok)) if parent[j] == cur and tok[j] == t]
                if not kid:
                    break
                cur = kid[0]
                acc += 1
            expect += pr * acc
        assert orc.l_tree_node_sum(cum) == pytest.approx(expect, rel=1e-10, abs=1e-14)


def test_topk_softmax_matches_library(orc):
    """A1 reduces to a textbook routine: fp64 softmax + stable lexsort on (-x, id) (Q9, Q10)."""
    from inputs import synth
    rng = np.random.default_rng(1)
    for V, k in [(32, 2), (1000, 8), (128256, 10), (152064, 10)]:
        for dt in ("bf16", "fp32"):
            x = rng.standard_normal(V).astype(np.float32) * 3
            x[rng.choice(V, 5, replace=False)] += 12
            row = synth.f32_to_bf16_bits(x) if dt == "bf16" else x
            xv = synth.bf16_bits_to_f32(row).astype(np.float64) if dt == "bf16" else x.astype(np.float64)
            tok, p, m, Z = orc.topk_softmax(row, k)
            ref = np.lexsort((np.arange(V), -xv))[:k]
            e = np.exp(xv - xv.max())
            assert (tok == ref).all()
            np.testing.assert_allclose(p, e[ref] / e.sum(), rtol=1e-12)
            assert m == xv.max()
    # edge rows
    for kind in ("all_equal", "neg_inf", "kth_tie"):
        x = synth.edge_rows(kind, 257, 4)
        tok, p, _, _ = orc.topk_softmax(x, 4)
        ref = np.lexsort((np.arange(257), -x.astype(np.float64)))[:4]
        assert (tok == ref).all(), kind
    with pytest.raises(ValueError):
        orc.topk_softmax(synth.edge_rows("nan", 257, 4), 4)
