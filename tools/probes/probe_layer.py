"""Timing probes of the layer kernel (debug aid, not a test; SMART_TIMING=1)."""
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
dev = torch.device("cuda")
dd = bench.bf16_dev(d, dev)
L = S.lib()
L.smart_debug_probes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(64, np.uint64)
for rep in range(3):
    ctx.begin_step()
    for layer in range(1, 7):
        L.smart_debug_probes(ctx._h, None, 1)
        ctx.expand_step(layer, dd)
        ctx.select(layer)
        L.smart_debug_probes(ctx._h, buf.ctypes.data_as(C.c_void_p), 0)
        t0 = int(buf[0])

        def rel(i):
            v = int(buf[i])
            return None if v in (0, 2 ** 64 - 1) else round((v - t0) / 1000.0, 2)
        if rep == 2:
            print(f"layer {layer}: last CTA start {rel(1)} stream_end {rel(2)} first_merge {rel(8)} "
                  f"last_merge {rel(3)}->{rel(4)} select {rel(5)}->{rel(6)} end {rel(7)} us; select phases "
                  f"stage {rel(9)} rank {rel(10)} sort {rel(11)} rule {rel(12)} fscan {rel(13)} nodes {rel(14)}")
            print("   CTA0: R read", rel(16), "init", rel(17), "producer", rel(27),
                  "chunk0 (full, softmax, topk)", rel(18), rel(19), rel(20), "chunk1", rel(21), rel(22), rel(23),
                  "seg compact", rel(24), "cta merge", rel(25), "arrival", rel(26))
            st = [int(buf[32 + j]) for j in range(32)]
            print("   CTA0 warp0 chunk0 cycles: lds+unpack", st[1] - st[0], "lanemax", st[2] - st[1], "Mw", st[3] - st[2],
                  "sumexp+store", st[4] - st[3], "seed", st[5] - st[4], "scan", st[6] - st[5])
            print("   CTA0 after sync", rel(28), "cta merge pass1 end", rel(31), "pass2 end", rel(25))
            print("   row0 merge:", rel(29), "->", rel(30), "cycles: loads", st[25] - st[24], "MZ", st[26] - st[25],
                  "T", st[27] - st[26], "surv", st[28] - st[27], "rank", st[29] - st[28], "tail", st[30] - st[29])
            d = lambda a, b: st[b] - st[a] if st[a] and st[b] else None
            print("   seg_end cycles: compact", d(0, 1), "fence", d(1, 2), "sync", d(2, 3), "rankmerge", d(3, 4),
                  "seglen+fence", d(4, 5), "sync", d(5, 6), "atomic", d(6, 7), "sync", d(7, 8))
            print("   select cycles: stage", d(9, 10), "elig+rank", d(10, 11), "sort", d(11, 12), "rule", d(12, 13),
                  "commit", d(13, 22))
