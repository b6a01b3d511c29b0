"""Per-layer timeline of the cluster-team layer kernel (debug aid; SMART_TIMING=1, eager launches)."""
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

wl = bench.WORKLOADS["cfg3_llama8b_b32"]
fx = mcf.load(wl["fixture"])
cfg = S.Config(vocab=wl["V"], top_k=wl["k"], max_depth=wl["d"], max_frontier=wl["W"], batch_local=32,
               budget_verify=200, alpha=0.8, bonus=1, logits_dtype=S.BF16, row_mode=S.ROWS_NODE)
ctx = S.Smart(cfg, S.Cost(lam=fx["lam"], gamma=fx["gamma"], delta=fx["delta"], rho=fx["rho"], eta=fx["eta"],
                          c_T=fx["c_T"]))
T = ctx.sizes["T"]
d, tg, rt, rp = bench.make_set(0, wl, T, 0)
dd = bench.bf16_dev(d, torch.device("cuda"))
L = S.lib()
L.smart_debug_probes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(1024, np.uint64)
for rep in range(3):
    ctx.begin_step()
    for layer in range(1, 7):
        L.smart_debug_probes(ctx._h, None, 1)
        ctx.expand_step(layer, dd)
        ctx.select(layer)
        L.smart_debug_probes(ctx._h, buf.ctypes.data_as(C.c_void_p), 0)
        t0 = int(buf[64 + 2 * layer])

        def rel(i):
            v = int(buf[i])
            return None if v in (0, 2 ** 64 - 1) else round((v - t0) / 1000.0, 2)
        if rep == 2:
            st = [int(buf[32 + j]) for j in range(32)]
            dd_ = lambda a, b: st[b] - st[a] if st[a] and st[b] else None
            print(f"layer {layer}: R {rel(16)} staged {rel(17)} | CTA0 chunk0 data {rel(18)} softmax {rel(19)} topk {rel(20)}"
                  f" chunk1 {rel(21)} {rel(22)} {rel(23)} | slice arrive {rel(27)} | merge {rel(24)}->{rel(25)} atomic {rel(26)}"
                  f" | select {rel(28)} rows-in {rel(30)} done {rel(29)} end {rel(65 + 2 * layer)}")
            print("   list sync", rel(31), "ranked", rel(96), "sync2", rel(97), "arrived", rel(98))
            print("   chunk0 cycles: bound", dd_(24, 31), "pend", dd_(31, 25), "append", dd_(25, 26), "compact", dd_(26, 27),
                  "| chunk1: pend", dd_(28, 29), "append", dd_(29, 30))
            print("   merge cycles: Z", dd_(1, 2), "thresh+surv", dd_(2, 3), "rank+store", dd_(3, 4), "tail", dd_(4, 5), "arrive", dd_(5, 6))
            print("   select cycles: stage", dd_(9, 10), "elig+rank", dd_(10, 11), "sort", dd_(11, 12), "rule", dd_(12, 13),
                  "commit", dd_(13, 14), "tail", dd_(14, 22))
            print("   commit cycles: bitmaps", dd_(13, 15), "B6", dd_(15, 16), "counts+scan", dd_(16, 17),
                  "frontier", dd_(17, 18), "fence+flag", dd_(18, 19), "B7", dd_(19, 14))
