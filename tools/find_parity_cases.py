"""Search seeded small configurations whose oracle trees are non-trivial in every mode.

For each combination selection (PREFIX / FROZEN) x acceptance model (NODE_SUM / PATH_MEAN) x
marginal (DERIVATIVE / DIFFERENCE) x W in {0 (unlimited), k}, draw random small configs (seeded)
and keep the first whose fp64 ORACLE run (the only thing this script executes) builds at least
2b drafted nodes, admits in at least 2 layers and has no tie-ambiguous decision (Q24, 1e-5).
Prints the Case(...) lines pasted into tests/test_gpu_parity.py (MODES).
"""
import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from smart_gpu_cases import Case, make_inputs, run_oracle  # noqa: E402
from oracle import oracle as O  # noqa: E402


def draw(i, sel, acc, mar, wmode):
    rng = np.random.default_rng(1000 * i + 7)
    i = i % 1000
    k = int(rng.integers(2, 9))
    b = int(rng.integers(2, 7))
    d = int(rng.integers(3, 6))
    V = int(rng.choice([9001, 20000, 40001, 70000]))
    W = 0 if wmode == 0 else k
    omega = int(rng.integers(0, 2)) if acc == 1 else 1
    lam = float(rng.uniform(0.002, 0.03))
    eta = float(rng.uniform(0.5, 2.0)) if omega or acc == 1 else float(rng.uniform(0.0, 1.0))
    cost = (lam, 0.0, float(rng.uniform(0.0, 0.05)), float(rng.uniform(0.001, 0.02)),
            float(rng.uniform(1.0, 1.4)), eta, 1.0)
    return Case(V=V, k=k, d=d, W=W, b=b, B_verify=int(b * rng.integers(k + 1, 3 * k + 4)),
                alpha=float(rng.choice([0.8, 1.0])), omega=omega, selection=sel, accept_model=acc,
                marginal=mar, dtype=["bf16", "fp32"][i % 2], seed=int(100 + i), cost=cost,
                sigma_m=0.5, a_lo=float(rng.uniform(3, 8)), a_hi=float(rng.uniform(9, 14)))


def ok(case):
    T = O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify).tmax()
    draft, target, rt, rp = make_inputs(case, T)
    orc = run_oracle(case, draft, target, rt, rp)
    adm = [int(orc.trace[l, 3]) for l in range(case.d)]
    adm_layers = sum(1 for a in adm if a > 0)
    later_multi = any(a >= 2 for a in adm[1:])
    return (orc.first_ambiguous_layer == 0 and orc.N >= 2 * case.b and adm_layers >= 3 and later_multi), orc


def main():
    for sel, acc, mar, wmode in itertools.product((0, 1), (0, 1), (0, 1), (0, 1)):
        off = 97 * (8 * sel + 4 * acc + 2 * mar + wmode)
        for i in range(off, off + 3000):
            c = draw(i, sel, acc, mar, wmode)
            good, orc = ok(c)
            if good:
                adm = [int(orc.trace[l, 3]) for l in range(c.d)]
                print(f"    Case(V={c.V}, k={c.k}, d={c.d}, W={c.W}, b={c.b}, B_verify={c.B_verify}, "
                      f"alpha={c.alpha}, omega={c.omega}, selection={sel}, accept_model={acc}, marginal={mar}, "
                      f"dtype={c.dtype!r}, seed={c.seed}, cost={tuple(round(x, 6) for x in c.cost)}, "
                      f"sigma_m=0.5, a_lo={c.a_lo:.3f}, a_hi={c.a_hi:.3f}),  # N={orc.N} admits={adm}")
                break
        else:
            print(f"    # no case found for sel={sel} acc={acc} mar={mar} W={'k' if wmode else 0}")


if __name__ == "__main__":
    main()
