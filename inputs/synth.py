"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the SMART method (no softmax, top-k, cost model,
selection, mask or verify logic).  It only draws numbers: logit pools shaped like the
paper's workloads (DESIGN.md §5 "input recipe") and hand-specified toy rows.

Recipe:
  * draft row: x_v = sigma_bg * z_v, z ~ N(0,1), sigma_bg = 2, plus H = 8 "head" tokens at
    distinct uniform positions with amplitude A_h = A1 * h^-0.7, A1 ~ U(a_lo, a_hi);
  * target row for tree node u = draft row of u + sigma_m * z' (fresh noise), so that
    greedy verification accepts a fraction of the draft's top-1 chain;
  * rows are keyed by (seed, global request) with numpy's counter-based Philox, so a
    request's rows do not depend on how the batch is sharded across ranks;
  * logits are rounded to bf16 (round-to-nearest-even) and returned as uint16 bit
    patterns; the fp32 variant is the same values upcast, and "fp32full" keeps the full fp32
    mantissa (no bf16 rounding) for the fp32 path's own tests.
"""
from __future__ import annotations

import numpy as np


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit pattern (uint16). NaN stays NaN."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        r[nan] = 0x7FC0
    return r


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(h, np.uint16).astype(np.uint32) << 16).view(np.float32)


def _rng(seed: int, stream: int, sub: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[(seed & 0xFFFFFFFF) | (sub << 32), stream]))


def draft_rows(seed: int, r_glob: int, n_rows: int, V: int, ld: int | None = None,
               sigma_bg: float = 2.0, H: int = 8, a_lo: float = 10.0, a_hi: float = 18.0,
               sub: int = 0) -> np.ndarray:
    """float32 [n_rows, ld] draft logits of one request (padding columns = -inf)."""
    ld = ld or V
    g = _rng(seed, r_glob, sub)
    x = np.full((n_rows, ld), -np.inf, np.float32)
    x[:, :V] = g.standard_normal((n_rows, V), dtype=np.float32) * np.float32(sigma_bg)
    a1 = g.uniform(a_lo, a_hi, size=n_rows).astype(np.float32)
    h = np.arange(1, H + 1, dtype=np.float32)
    for i in range(n_rows):
        pos = g.choice(V, size=H, replace=False)
        x[i, pos] += a1[i] * h ** np.float32(-0.7)
    return x


def draft_pool(seed: int, b: int, T: int, V: int, ld: int | None = None, r_offset: int = 0,
               dtype: str = "bf16", **kw) -> np.ndarray:
    """[b, T, ld] pool, row (r, u) = draft logits used to expand node u of request r."""
    ld = ld or V
    out = np.empty((b, T, ld), np.uint16 if dtype == "bf16" else np.float32)
    for r in range(b):
        x = draft_rows(seed, r_offset + r, T, V, ld, **kw)
        if dtype == "fp32full":
            out[r] = x
        else:
            out[r] = f32_to_bf16_bits(x) if dtype == "bf16" else bf16_bits_to_f32(f32_to_bf16_bits(x))
    return out


def target_pool(draft: np.ndarray, seed: int, sigma_m: float, r_offset: int = 0,
                V: int | None = None, full: bool = False) -> np.ndarray:
    """target(r, u) = draft(r, u) + sigma_m * z' (fresh keyed noise); same dtype as draft."""
    bf = draft.dtype == np.uint16
    out = np.empty_like(draft)
    V = V or draft.shape[-1]
    for r in range(draft.shape[0]):
        base = bf16_bits_to_f32(draft[r]) if bf else draft[r].astype(np.float32)
        if sigma_m > 0:
            g = _rng(seed, r_offset + r, sub=7)
            noise = g.standard_normal((draft.shape[1], V), dtype=np.float32) * np.float32(sigma_m)
            base = base.copy()
            base[:, :V] += noise
        out[r] = f32_to_bf16_bits(base) if bf else (base if full else bf16_bits_to_f32(f32_to_bf16_bits(base)))
    return out


def logits_from_probs(V: int, listed: dict[int, float]) -> np.ndarray:
    """float32 row with logit ln p for the listed tokens and the remaining mass spread evenly
    over the other tokens (SURVEY.md §8(c) toy example recipe)."""
    rest = 1.0 - sum(listed.values())
    others = V - len(listed)
    x = np.full(V, np.log(rest / others) if rest > 0 else -np.inf, np.float64)
    for t, pr in listed.items():
        x[t] = np.log(pr)
    return x.astype(np.float32)


# ---- edge-case rows (SURVEY.md §8(d) "edge suites") ----------------------------

def edge_rows(kind: str, V: int, k: int, seed: int = 0) -> np.ndarray:
    g = _rng(seed, 0, sub=11)
    if kind == "all_equal":
        return np.zeros(V, np.float32)
    if kind == "neg_inf":
        x = g.standard_normal(V, dtype=np.float32) * 2
        x[g.choice(V, size=V // 2, replace=False)] = -np.inf
        return x
    if kind == "kth_tie":  # k-th and (k+1)-th (and more) largest logits tie exactly
        x = g.standard_normal(V, dtype=np.float32)
        top = g.choice(V, size=k + 3, replace=False)
        x[top[: k - 1]] = 20.0 + np.arange(k - 1, 0, -1, dtype=np.float32)
        x[top[k - 1:]] = 15.0
        return x
    if kind == "nan":
        x = g.standard_normal(V, dtype=np.float32)
        x[V // 3] = np.nan
        return x
    raise KeyError(kind)
