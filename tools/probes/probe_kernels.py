"""Kernel timeline of one graph-captured step of the per-layer path (SMART_NO_STEP=1) for a bench
workload (probe build: SMART_PROBES=1 SMART_TIMING=1).  python tools/probes/probe_kernels.py [workload]"""
import ctypes as C
import os
import sys

os.environ["SMART_TIMING"] = "1"
os.environ.setdefault("SMART_PROBES", "1")
os.environ["SMART_NO_STEP"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_09731_b200 import _build  # noqa: E402
_build.build()
import bench  # noqa: E402
import make_cost_fixture as mcf  # noqa: E402
from paper_2604_09731_b200 import smart as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_r1distill_b256"
wl = bench.WORKLOADS[name]
fx = mcf.load(wl["fixture"])
cfg = S.Config(vocab=wl["V"], top_k=wl["k"], max_depth=wl["d"], max_frontier=wl["W"], batch_local=wl["b"],
               budget_verify=wl["B_verify"], alpha=0.8, bonus=1, logits_dtype=S.BF16, row_mode=S.ROWS_NODE)
ctx = S.Smart(cfg, S.Cost(lam=fx["lam"], beta=fx["beta"], gamma=fx["gamma"], delta=fx["delta"], rho=fx["rho"],
                          eta=fx["eta"], c_T=fx["c_T"]))
T = ctx.sizes["T"]
d, tg, rt, rp = bench.make_set(0, wl, T, wl["b"], 0)
dev = torch.device("cuda")
dd, tt = bench.bf16_dev(d, dev), bench.bf16_dev(tg, dev)
out = ctx.alloc_outputs()
L = S.lib()
L.smart_debug_probes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(4096, np.uint64)
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    ctx.run_step(dd, tt, out, stream=s)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    ctx.run_step(dd, tt, out, stream=s)
for rep in range(3):
    torch.cuda.synchronize()
    L.smart_debug_probes(ctx._h, None, 1)
    g.replay()
    torch.cuda.synchronize()
L.smart_debug_probes(ctx._h, buf.ctypes.data_as(C.c_void_p), 0)
st = ctx.stats()
print(name, "rows per layer", [st["layers"][l]["n_rows"] for l in range(wl["d"])], "nodes", st["nodes_local"],
      "step kernel grid", st["step_kernel_grid"])
t0 = int(buf[64])
f = lambda v: None if int(v) in (0, 2 ** 64 - 1) else round((int(v) - t0) / 1000.0, 2)
rows = [(0, "begin")]
for l in range(1, wl["d"] + 1):
    rows += [(l, f"layer{l}"), (40 + l, f"select{l}")]
rows += [(20, "mask"), (21, "verify")]
for kid, nm in rows:
    a, b = buf[64 + 2 * kid], buf[65 + 2 * kid]
    fa, fb = f(a), f(b)
    print(f"{nm:9s} start {fa} end {fb} dur {None if fa is None or fb is None else round(fb - fa, 2)}")
names = {9: "start", 10: "benefits", 11: "req-rank", 12: "sort", 13: "A5 cut", 15: "bitmaps", 16: "B6",
         17: "counts", 18: "frontier", 19: "published", 14: "adm flags", 22: "end"}
for l in range(1, wl["d"] + 1):
    c = {j: int(buf[3000 + l * 16 + (j - 9)]) for j in range(9, 23)}
    base = c[9]
    if base:
        print(f"select{l} phases (cycles):", ", ".join(f"{names[j]} {c[j]-base}" for j in (10, 11, 12, 13, 15, 16, 17, 18, 19, 14, 22) if c[j]))
