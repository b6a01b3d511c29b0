"""Pins of the pruning bounds the T > 0 verify kernel relies on (verify_core.cuh: sample_chunk).

The kernel evaluates the Gumbel perturbation only for tokens that can still reach the row's best
perturbed value, using G = -ln(-ln U) <= 16.64 for every 23-bit U, <= 6.92 unless U >= ~0.999,
and it decides "U >= 0.999" from the counter-based hash BEFORE its last xor-shift (a superset
test).  These are integer / closed-form facts about the generator, checked here exhaustively or
on large samples with numpy (no GPU, no oracle code involved)."""
import numpy as np

K_U999 = 8380000          # (h >> 9) >= this  <=>  U >= ~0.99898   (verify_core.cuh kU999)
K_U999_PRE = 0xFFBC0000   # the pre-shift threshold                  (verify_core.cuh kU999Pre)
M32 = np.uint64(0xFFFFFFFF)


def _mix_pre(h):
    h = h.astype(np.uint64)
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x7FEB352D)) & M32
    h ^= h >> np.uint64(15)
    h = (h * np.uint64(0x846CA68B)) & M32
    return h


def _final(hpre):
    return hpre ^ (hpre >> np.uint64(16))


def test_pre_shift_threshold_is_a_superset():
    # every 32-bit value whose final hash passes the U >= 0.999 test passes the pre-shift test.
    # The last xor-shift keeps bits 31..16, so a final value >= 0xFFBCC000 has a high half >= 0xFFBC
    # (checked on a sample of the other high halves), and every value with such a high half is
    # checked exhaustively (68 x 65536 values)
    assert K_U999 << 9 == 0xFFBCC000
    lo = np.arange(0x10000, dtype=np.uint64)
    rng = np.random.default_rng(3)
    for h16 in rng.integers(0, 0xFFBC, size=64):
        hpre = (np.uint64(h16) << np.uint64(16)) | lo
        assert not np.any((_final(hpre) >> np.uint64(9)) >= np.uint64(K_U999))
    extra = 0
    for h16 in range(0xFFBC, 0x10000):
        hpre = (np.uint64(h16) << np.uint64(16)) | lo
        passes_final = (_final(hpre) >> np.uint64(9)) >= np.uint64(K_U999)
        passes_pre = hpre >= np.uint64(K_U999_PRE)
        assert not np.any(passes_final & ~passes_pre)
        extra += int(np.sum(passes_pre & ~passes_final))
    assert extra <= 0x10000  # the superset adds at most the 0xFFBC high half (1 / 65536 of values)


def test_gumbel_bounds_over_all_23_bit_uniforms():
    # U = ((h >> 9) + 0.5) * 2^-23 for every 23-bit value: G = -ln(-ln U)
    u = (np.arange(1 << 23, dtype=np.float64) + 0.5) * 2.0 ** -23
    g = -np.log(-np.log(u))
    assert g.max() <= 16.64 - 3e-5  # the kernel's fast log is within 3e-5 of the exact G
    below = np.arange(1 << 23) < K_U999
    assert g[below].max() <= 6.92 - 3e-5


def test_pre_shift_test_on_hashed_counters():
    # the same implication on the generator's actual inputs: rowkey + v * golden, v over a row
    rng = np.random.default_rng(7)
    for rowkey in rng.integers(0, 2 ** 32, size=4, dtype=np.uint64):
        v = np.arange(152064, dtype=np.uint64)
        h0 = (rowkey + v * np.uint64(0x9E3779B9)) & M32
        hpre = _mix_pre(h0)
        big = (_final(hpre) >> np.uint64(9)) >= np.uint64(K_U999)
        assert np.all(hpre[big] >= np.uint64(K_U999_PRE))
