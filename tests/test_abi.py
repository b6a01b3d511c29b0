"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol that
include/smart.h declares, and host-side validation behaves (no compute calls)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sm():
    from paper_2604_09731_b200 import _build
    _build.build()
    from paper_2604_09731_b200 import smart
    return smart


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "smart.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(smart_[a-z_]+)\s*\(", txt)))


def test_every_declared_symbol_is_exported(sm):
    L = sm.lib()
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(sm.EXPORTED)


def test_header_compiles_as_plain_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "smart.h"\nint main(void){smart_sizes s; smart_config c = {0};'
                   ' return (int)smart_query_sizes(&c, &s) == 0;}\n')
    import subprocess
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-c", str(src), "-o", str(tmp_path / "t.o")])


def test_query_sizes(sm):
    cfg = sm.Config(vocab=128256, top_k=8, max_depth=6, max_frontier=8, batch_local=32,
                    budget_verify=200)
    s = sm.query_sizes(cfg)
    assert s["B"] == 6 and s["T"] == 7 and s["mask_words"] == 1
    assert s["frontier_cap"] == 32 * 6 and s["chunk_elems"] == 8192
    cfg2 = sm.Config(vocab=128256, top_k=10, max_depth=6, max_frontier=10, batch_local=1, budget_verify=60)
    assert sm.query_sizes(cfg2)["T"] == 61 and sm.query_sizes(cfg2)["mask_words"] == 2


def test_query_sizes_baseline(sm):
    """NEXT #3 (Q32): the baseline pool holds the expanded tree (1 + W d) and the final top-g tree."""
    from oracle import oracle as O
    for (V, k, d, W, b, Bv) in ((128256, 10, 6, 10, 1, 60), (32001, 8, 5, 16, 32, 2048), (2000, 3, 2, 2, 2, 200)):
        cfg = sm.Config(vocab=V, top_k=k, max_depth=d, max_frontier=W, batch_local=b, budget_verify=Bv,
                        selection=sm.BASELINE)
        s = sm.query_sizes(cfg)
        assert s["T"] == O.baseline_T(O.Config(V=V, k=k, d=d, W=W, b=b, B_verify=Bv))
        assert s["frontier_cap"] == b * W
    bad = [dict(max_frontier=0, batch_local=2),                       # no expansion width
           dict(max_frontier=4, batch_local=1, batch_global=2),      # multi-rank
           dict(max_frontier=4, batch_local=2, tree_capacity=8)]     # pool below 1 + d W
    for kw in bad:
        cfg = sm.Config(vocab=1000, top_k=4, max_depth=3, budget_verify=40, selection=sm.BASELINE, **kw)
        with pytest.raises(sm.SmartError):
            sm.query_sizes(cfg)


@pytest.mark.parametrize("field,value", [("top_k", 0), ("top_k", 33), ("max_depth", 17), ("alpha", 0.0),
                                         ("alpha", 1.5), ("budget_verify", 0), ("vocab", 1),
                                         ("selection", 3), ("bonus", 2), ("row_mode", 3), ("row_mode", -1)])
def test_validation_rejects(sm, field, value):
    cfg = sm.Config(vocab=1000, top_k=4, max_depth=4, batch_local=2, budget_verify=16)
    setattr(cfg, field, value)
    with pytest.raises(sm.SmartError) as e:
        sm.query_sizes(cfg)
    assert e.value.status == sm.EINVAL


def test_create_without_gpu_fails_cleanly(sm):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = sm.Config(vocab=1000, top_k=4, max_depth=4, batch_local=2, budget_verify=16)
    with pytest.raises(sm.SmartError) as e:
        sm.Smart(cfg, sm.Cost(lam=1.0, eta=1.0, c_T=1.0))
    assert e.value.status in (sm.ECUDA, sm.EINVAL)


def test_bad_cost_rejected(sm):
    cfg = sm.Config(vocab=1000, top_k=4, max_depth=4, batch_local=2, budget_verify=16)
    h = C.c_void_p()
    for cost in (sm.Cost(lam=0.0, c_T=1.0, eta=1.0), sm.Cost(lam=1.0, c_T=0.0, eta=1.0),
                 sm.Cost(lam=1.0, c_T=1.0)):  # bonus=1 with beta+eta = 0
        c, k = cfg.c(), cost.c()
        assert sm.lib().smart_create(C.byref(c), C.byref(k), 0, C.byref(h)) == sm.EINVAL


def test_product_does_not_import_oracle():
    """The product path never references the oracle."""
    pkg = os.path.join(ROOT, "paper_2604_09731_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(//|#).*", "", txt).lower() or f == "smart_internal.cuh", f


def test_position_row_mode_accepted(sm):
    """NEXT #4 DFLASH rows: SMART_ROWS_POSITION is a valid row mode for SMART and BASELINE."""
    for sel in (sm.PREFIX, sm.BASELINE):
        cfg = sm.Config(vocab=1000, top_k=4, max_depth=3, max_frontier=4, batch_local=2, budget_verify=16,
                        selection=sel, row_mode=sm.ROWS_POSITION)
        assert sm.query_sizes(cfg)["T"] >= 1


def test_bench_reference_arm_contract():
    """bench.py --impl reference prints one JSON line with the contract's keys (the fp64 oracle on
    the host cores; CPU only)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--workload", "cfg2_llama8b_b1"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_tree_capacity_below_reachable_size_is_rejected(sm):
    """A SMART tree can reach 1 + min(B, d * W) nodes; a smaller user-set tree_capacity would let
    the commit write past the request's arrays, so validation rejects it (EINVAL)."""
    base = dict(vocab=5000, top_k=4, max_depth=3, max_frontier=3, batch_local=2, budget_verify=20)
    assert sm.query_sizes(sm.Config(**base))["T"] == 1 + min(10, 9)
    with pytest.raises(sm.SmartError) as e:
        sm.query_sizes(sm.Config(**base, tree_capacity=4))
    assert e.value.status == sm.EINVAL
    assert sm.query_sizes(sm.Config(**base, tree_capacity=10))["T"] == 10
    assert sm.query_sizes(sm.Config(**base, tree_capacity=64))["T"] == 64
