"""Phase cycles of the standalone selection at cfg5 layer 1 (b = 256; debug aid, SMART_PROBES=1 build)."""
import ctypes as C
import os
import sys

os.environ["SMART_TIMING"] = "1"
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tools")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import make_cost_fixture as mcf  # noqa: E402
from paper_2604_09731_b200 import smart as S  # noqa: E402

wl = bench.WORKLOADS["cfg5_r1distill_b256"]
fx = mcf.load(wl["fixture"])
cost = S.Cost(lam=fx["lam"], gamma=fx["gamma"], delta=fx["delta"], rho=fx["rho"], eta=fx["eta"], c_T=fx["c_T"])
if os.environ.get("CHEAP"):
    cost = S.Cost(lam=0.0005, eta=1.0, c_T=1.0)
cfg = S.Config(vocab=wl["V"], top_k=wl["k"], max_depth=wl["d"], max_frontier=wl["W"], batch_local=wl["b"],
               budget_verify=wl["B_verify"], alpha=0.8, bonus=1, logits_dtype=S.BF16, row_mode=S.ROWS_NODE)
ctx = S.Smart(cfg, cost)
T = ctx.sizes["T"]
d, tg, rt, rp = bench.make_set(0, wl, T, wl["b"], 0)
dd = bench.bf16_dev(d, torch.device("cuda"))
L = S.lib()
L.smart_debug_probes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(4096, np.uint64)
for rep in range(3):
    ctx.begin_step()
    for layer in range(1, 4):
        ctx.expand_step(layer, dd)
        torch.cuda.synchronize()
        L.smart_debug_probes(ctx._h, None, 1)
        ctx.select(layer)
        torch.cuda.synchronize()
        L.smart_debug_probes(ctx._h, buf.ctypes.data_as(C.c_void_p), 0)
        st = [int(buf[32 + j]) for j in range(32)]
        dd_ = lambda a, b: st[b] - st[a] if st[a] and st[b] else None
        if rep == 2:
            print(f"layer {layer}: theta(w1)", dd_(9, 20), "pre-B2(t0)", dd_(9, 21), "stage", dd_(9, 10), "elig+rank", dd_(10, 11), "sort", dd_(11, 12), "rule", dd_(12, 13),
                  "commit", dd_(13, 14), "tail", dd_(14, 22), "trace", ctx.stats()["layers"][layer - 1])
