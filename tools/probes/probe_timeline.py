"""Kernel timeline of one graph-captured cfg3 step (debug aid, not a test; SMART_TIMING=1)."""
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
tt = bench.bf16_dev(tg, dev)
out = ctx.alloc_outputs()
L = S.lib()
L.smart_debug_probes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(4096, np.uint64)
s = torch.cuda.Stream()


def step():
    ctx.begin_step(stream=s)
    for layer in range(1, 7):
        ctx.expand_step(layer, dd, stream=s)
        ctx.select(layer, stream=s)
    ctx.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"], stream=s)
    ctx.verify_accept(tt, out["accept_len"], out["accept_path"], out["bonus"], stream=s)


with torch.cuda.stream(s):
    step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
for rep in range(4):
    torch.cuda.synchronize()
    L.smart_debug_probes(ctx._h, None, 1)
    g.replay()
    torch.cuda.synchronize()
    L.smart_debug_probes(ctx._h, buf.ctypes.data_as(C.c_void_p), 0)
    if rep < 2:
        continue
    names = [(0, "begin")] + [(l, f"layer{l}") for l in range(1, 7)] + [(20, "mask"), (21, "verify")]
    t0 = int(buf[64])
    prev_end = None
    print(f"--- replay {rep}")
    for kid, nm in names:
        st, en = int(buf[64 + 2 * kid]), int(buf[65 + 2 * kid])
        pre = int(buf[64 + 2 * (32 + kid)]) if kid < 32 and 32 + kid < 96 else 0
        f = lambda v: None if v in (0, 2 ** 64 - 1) else round((v - t0) / 1000.0, 2)
        gap = None if prev_end is None or st in (0, 2 ** 64 - 1) else round((st - prev_end) / 1000.0, 2)
        print(f"{nm:8s} launch {f(pre)} start {f(st)} end {f(en)} dur {None if f(en) is None or f(st) is None else round(f(en) - f(st), 2)} gap_from_prev_end {gap}")
        if en not in (0, 2 ** 64 - 1):
            prev_end = en
    vs = int(buf[64 + 42])
    f2 = lambda v: None if v in (0, 2 ** 64 - 1) else round((int(v) - vs) / 1000.0, 2)
    print("verify CTA0 chunk starts", [f2(buf[100 + j]) for j in range(8)])
    for sg in range(4):
        print(f"  seg {sg}: cta-reduce+arrive {f2(buf[110 + 4 * sg])} after-sync {f2(buf[111 + 4 * sg])} "
              f"row-merged {f2(buf[112 + 4 * sg])} seg-done {f2(buf[113 + 4 * sg])}")
    ends = [(int(buf[256 + b]) - vs) / 1000.0 for b in range(296) if int(buf[256 + b]) not in (0, 2 ** 64 - 1)]
    ends.sort()
    print("verify CTA ends: n", len(ends), "min", ends[0], "p50", ends[len(ends) // 2], "p90", ends[int(len(ends) * 0.9)], "max", ends[-1])
    late = [(b, round((int(buf[256 + b]) - vs) / 1000.0, 2)) for b in range(296) if int(buf[256 + b]) not in (0, 2 ** 64 - 1) and (int(buf[256 + b]) - vs) / 1000.0 > ends[int(len(ends) * 0.9)]]
    print("late CTAs", late[:20])
