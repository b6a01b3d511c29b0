"""Pins of the two facts the step kernel's small-batch selection (select_small)
relies on, checked on the fp64 oracle (which does not use them) over random instances:

1. Screening threshold.  Eq.(16) (Algorithm 1 lines 5-9) admits the
   candidate at sorted position j only if alpha c_T b_j C(N0+j) > (rhs0 + c_T before_j) dc(N0+j)
   with before_j >= 0, so every admitted candidate has b > theta = min_j rhs0 dc(N0+j) /
   (alpha c_T C(N0+j)) -- for PREFIX and FROZEN alike.
2. Argmax certificate.  On a convex cost window the prefix speedups S_j of the sorted eligible
   list are unimodal and cannot rise past a benefit <= th2 = s_0 min dC (s = S / c_T), so
   argmax_j S_j (the A5 report) lies within the prefix of eligible benefits above th2.

Test infrastructure only (calls oracle/ and the closed-form cost of the oracle wrapper)."""
import math

import numpy as np

from inputs import synth


def _instance(orc, rng, concave=False, linear=False):
    b = int(rng.integers(1, 6))
    k = int(rng.integers(2, 7))
    d = int(rng.integers(2, 6))
    W = int(rng.choice([0, k, 3]))
    cfg = orc.Config(V=96, k=k, d=d, W=W, b=b, B_verify=int(rng.integers(2 * b, 30 * b)),
                     alpha=float(rng.choice([0.6, 0.8, 1.0])), omega=int(rng.integers(0, 2)),
                     selection=int(rng.integers(0, 2)), accept_model=orc.NODE_SUM,
                     marginal=int(rng.integers(0, 2)), dtype=orc.FP32)
    cost = orc.Cost(lam=float(rng.uniform(0.005, 0.2)), gamma=0.0 if linear else float(rng.uniform(0, 0.3)),
                    delta=float(rng.uniform(0.005, 0.1)),
                    rho=float(rng.uniform(0.4, 0.9) if concave else rng.uniform(1.0, 1.6)),
                    eta=float(rng.uniform(0.5, 2.0)) if cfg.omega else 0.0, c_T=1.0)
    pool = synth.draft_pool(int(rng.integers(1 << 30)), b, cfg.tmax(), cfg.V, dtype="fp32", a_lo=2, a_hi=8, sigma_bg=1.0)
    return cfg, cost, pool


def _layer_terms(orc, cfg, cost, res, l):
    tr = res.trace[l - 1]
    N0, E0, ne = int(tr[4]), float(tr[5]), int(tr[2])
    C = np.array([orc.cost_spec(cost, N0 + j) for j in range(ne + 2)])
    dc = np.array([orc.dc(cost, N0 + j, cfg.marginal)[0] for j in range(ne + 2)])
    return N0, E0, ne, C, dc


def _eligible(orc, cfg, res, l, cands):
    """A3 (Eq.(8)): per request the first min(B - n_r, W, |U_r|) candidates by
    (b desc, c asc); n_r = the request's drafted nodes before layer l (from the final tree)."""
    W = cfg.W if cfg.W > 0 else 1 << 30
    elig = np.zeros(len(cands["b"]), bool)
    for r in range(cfg.b):
        n = int(res.n_nodes[r])
        nd = int(np.sum(res.depth[r, 1:n] < l))
        idx = np.where(cands["r"] == r)[0]
        e = max(0, min(cfg.B - nd, W, len(idx)))
        order = sorted(idx, key=lambda q: (-cands["b"][q], cands["c"][q]))
        elig[order[:e]] = True
    return elig


def test_admitted_benefits_exceed_theta(orc):
    rng = np.random.default_rng(2024)
    checked = 0
    for concave in (False, True):
        for it in range(60):
            cfg, cost, pool = _instance(orc, rng, concave)
            res = orc.step(cfg, cost, pool)
            for l in range(1, cfg.d + 1):
                if not res.trace[l - 1, 12]:
                    continue
                cands = res.layer_cands(l)
                N0, E0, ne, C, dc = _layer_terms(orc, cfg, cost, res, l)
                rhs0 = cost.c_T * (cfg.omega * cfg.b + E0)
                ac = cfg.alpha * cost.c_T
                theta = min((rhs0 * dc[j] / (ac * C[j]) if C[j] > 0 else 0.0) for j in range(ne + 1))
                adm = cands["admitted"]
                assert np.all(cands["b"][adm] > theta * (1 - 1e-12)), (l, theta, cands["b"][adm].min())
                # the cut lies inside the above-theta prefix: no more admits than eligible above it
                elig = _eligible(orc, cfg, res, l, cands)
                assert int(tr_admit := res.trace[l - 1, 3]) <= int(np.sum(elig & (cands["b"] > theta * (1 - 1e-12)))), tr_admit
                assert int(np.sum(elig)) == ne  # the eligibility reconstruction matches the trace
                checked += int(adm.sum())
    assert checked > 100


def test_argmax_within_th2_prefix_on_convex_windows(orc):
    rng = np.random.default_rng(7)
    certified = 0
    for it in range(160):
        cfg, cost, pool = _instance(orc, rng, concave=False, linear=it % 4 == 0)  # linear: convex up to rounding
        res = orc.step(cfg, cost, pool)
        for l in range(1, cfg.d + 1):
            if not res.trace[l - 1, 12]:
                continue
            cands = res.layer_cands(l)
            N0, E0, ne, C, dc = _layer_terms(orc, cfg, cost, res, l)
            dC = np.diff(C[: ne + 2])
            if not (C[0] > 0 and np.all(np.diff(dC) >= -1e-9 * np.abs(dC[:-1])) and dC.min() > 0):
                continue
            th2 = (cfg.omega * cfg.b + E0) / C[0] * dC.min() * (1 - 1e-6)
            elig = _eligible(orc, cfg, res, l, cands)
            bs = np.sort(cands["b"][elig])[::-1]
            narg = int(np.sum(bs > th2))
            # S_j over every prefix of the sorted eligible list (fp64, the oracle's own report)
            assert int(res.trace[l - 1, 8]) <= narg, (int(res.trace[l - 1, 8]), narg, ne)
            # and the sequence really is unimodal past narg
            P = np.concatenate([[0.0], np.cumsum(bs)])
            S = cost.c_T * (cfg.omega * cfg.b + E0 + P) / C[: ne + 1]
            assert np.all(np.diff(S[narg:]) <= 1e-12 * np.abs(S[narg:-1]) + 0.0)
            certified += 1
    assert certified > 50
