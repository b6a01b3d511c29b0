"""NEXT #3 pins (reading Q32): the likelihood-maximising two-stage baseline of EAGLE-3 /
MSD (Fig. 2(a)(b)) in the oracle.

  * Fig. 2 configuration (2 nodes expanded per layer, top-2 children, rerank to 8): exactly 8
    retained drafted nodes (SPEC S:303 example);
  * a deterministic draft (top-1 probability ~1 everywhere) gives the chain of length d;
  * rerank budget >= generated nodes: the rerank is the identity (every generated node kept);
  * on random inputs: the final set is the top-g of ALL generated candidates by cum (checked
    against an independent enumeration of the generated candidates from the draft rows), it is
    ancestor-closed, the node order is (depth, canonical index) and A7/A8 hold on it.
"""
import numpy as np

from inputs import synth
from oracle import oracle as O


def _cfg(**kw):
    base = dict(V=50, k=2, d=4, W=2, b=1, B_verify=8, dtype=O.FP32, row_mode=O.ROWS_NODE)
    base.update(kw)
    return O.Config(**base)


def _random_pool(cfg, seed, peaked=False):
    T = O.baseline_T(cfg)
    rng = np.random.default_rng(seed)
    x = rng.normal(0, 1.0, (cfg.b, T, cfg.V)).astype(np.float32)
    if peaked:
        x[..., 0] += 40.0  # token 0 takes (almost) all the probability everywhere
    return x


def test_fig2_rerank_to_8():
    cfg = _cfg(V=50, k=2, W=2, d=4, B_verify=8)
    res = O.baseline_step(cfg, _random_pool(cfg, 1))
    # generated: 2 + 4 + 4 + 4 = 14 candidates; top-8 retained (closure already satisfied)
    assert res.n_nodes[0] == 1 + 8
    assert res.extra["n_exp"][0] == 1 + 2 * 4


def test_deterministic_draft_gives_the_chain():
    cfg = _cfg(V=30, k=2, W=2, d=5, B_verify=5)
    res = O.baseline_step(cfg, _random_pool(cfg, 2, peaked=True))
    n = res.n_nodes[0]
    assert n == 1 + 5
    # a chain: node i's parent is i-1 in depth order, all token 0
    depths = res.depth[0, 1:n]
    assert list(depths) == [1, 2, 3, 4, 5]
    assert (res.tok[0, 1:n] == 0).all()
    for i in range(1, n):
        assert res.parent[0, i] == i - 1


def test_rerank_identity_when_budget_covers_everything():
    cfg = _cfg(V=40, k=3, W=2, d=3, B_verify=100)
    res = O.baseline_step(cfg, _random_pool(cfg, 3))
    assert res.n_nodes[0] == 1 + 3 + 6 + 6  # every generated candidate kept


def _generated(cfg, draft, r):
    """independent enumeration: expand top-W of each layer (by cum desc, c asc), collect all."""
    def topk(row):
        x = row[:cfg.V].astype(np.float64)
        m = x.max()
        z = np.exp(x - m)
        p = z / z.sum()
        order = np.lexsort((np.arange(cfg.V), -x))[:cfg.k]
        return order, p[order]
    gen = []  # (cum, layer, c, tok, parent_gen_index or -1)
    front = [(-1, 1.0, 0)]  # (gen index, cum, expanded node index)
    ne = 1
    for l in range(1, cfg.d + 1):
        layer = []
        for i, (gi, pc, u) in enumerate(front):
            toks, ps = topk(draft[r, u])
            for j in range(cfg.k):
                layer.append((pc * ps[j], l, i * cfg.k + j, int(toks[j]), gi))
        base = len(gen)
        gen.extend(layer)
        order = sorted(range(len(layer)), key=lambda q: (-layer[q][0], layer[q][2]))[:cfg.W]
        front = []
        for q in sorted(order, key=lambda q: layer[q][2]):
            front.append((base + q, layer[q][0], ne))
            ne += 1
    return gen


def test_random_top_g_closure_and_order():
    for seed in range(8):
        cfg = _cfg(V=64, k=3, W=3, d=4, b=3, B_verify=3 * 10)
        draft = _random_pool(cfg, 100 + seed)
        target = _random_pool(cfg, 200 + seed)
        res = O.baseline_step(cfg, draft, target)
        g = cfg.B_verify // cfg.b
        for r in range(cfg.b):
            gen = _generated(cfg, draft, r)
            ranked = sorted(range(len(gen)), key=lambda q: (-gen[q][0], gen[q][1], gen[q][2]))
            keep = sorted(ranked[:g], key=lambda q: (gen[q][1], gen[q][2]))
            n = res.n_nodes[r]
            assert n == 1 + len(keep)
            np.testing.assert_array_equal(res.tok[r, 1:n], [gen[q][3] for q in keep])
            np.testing.assert_allclose(res.cum[r, 1:n], [gen[q][0] for q in keep], rtol=1e-12)
            # ancestor closure and parent mapping
            newidx = {q: i + 1 for i, q in enumerate(keep)}
            for i, q in enumerate(keep):
                pg = gen[q][4]
                assert res.parent[r, i + 1] == (0 if pg < 0 else newidx[pg])
            # A7: mask bit j of row i iff j is an ancestor-or-self of i
            for i in range(n):
                anc = set()
                j = i
                while j >= 0:
                    anc.add(j)
                    j = res.parent[r, j] if j > 0 else -1
                for j in range(n):
                    assert bool(res.mask[r, i, j // 32] >> (j % 32) & 1) == (j in anc)
        assert (res.accept_len >= 0).all() and (res.bonus >= 0).all()
