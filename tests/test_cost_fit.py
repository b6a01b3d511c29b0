"""NEXT #2 pins: the cost-model fit (SPEC S:159 scheme, tools/make_cost_fixture.fit_verify) used for
both the roofline fixtures and the on-box measurements (tools/measure_cost_model.py).

Exact samples of gamma*(exp(delta N^rho) - 1) are refitted: the recovered curve reproduces the
samples (and a held-out point) to 1e-3 relative; the least-squares lambda of a line through the
origin is exact on exact data; the committed measured fixtures parse and are in the model's
domain (positive c_T, marginal cost > 0 at N >= 1).
"""
import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import make_cost_fixture as mcf  # noqa: E402


@pytest.mark.parametrize("gamma,delta,rho", [(0.05, 0.003, 1.3), (2.0, 0.0002, 1.8), (0.3, 0.05, 0.8)])
def test_fit_verify_recovers_exact_curve(gamma, delta, rho):
    xs = np.array([20, 80, 140, 200, 300], float)
    ys = gamma * np.expm1(delta * xs ** rho)
    g, d, r, rmse = mcf.fit_verify(xs, ys)
    fit = lambda x: g * math.expm1(d * x ** r)
    for x, y in zip(xs, ys):
        assert abs(fit(x) - y) <= 1e-3 * abs(y) + 1e-9
    x_mid = 110.0
    assert abs(fit(x_mid) - gamma * math.expm1(delta * x_mid ** rho)) <= 2e-3 * gamma * math.expm1(delta * x_mid ** rho)


@pytest.mark.parametrize("name", ["measured_llama8b_b32", "measured_llama8b_b1"])
def test_measured_fixtures_in_domain(name):
    fx = mcf.load(name)
    assert fx["c_T"] > 0 and fx["eta"] == fx["c_T"] and fx["beta"] == 0.0
    assert fx["lam"] > 0 and fx["gamma"] >= 0 and fx["delta"] >= 0 and fx["rho"] > 0
    path = os.path.join(mcf.ROOT, "fixtures", f"cost_b200_{name}.txt")
    assert "MEASURED" in open(path).readline()
