"""Per-CTA start / work-end of one cfg3 layer kernel (debug aid; needs a SMART_PROBES=1 build)."""
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
LAYER = int(os.environ.get("LAYER", "1"))
for _ in range(200):
    ctx.begin_step()
    for layer in range(1, 7):
        ctx.expand_step(layer, dd)
        ctx.select(layer)
torch.cuda.synchronize()
for rep in range(2):
    ctx.begin_step()
    for layer in range(1, LAYER):
        ctx.expand_step(layer, dd)
        ctx.select(layer)
    torch.cuda.synchronize()
    L.smart_debug_probes(ctx._h, None, 1)
    ctx.expand_step(LAYER, dd)
    torch.cuda.synchronize()
    L.smart_debug_probes(ctx._h, buf.ctypes.data_as(C.c_void_p), 0)
st = np.array([int(buf[256 + b]) for b in range(264)], dtype=np.float64)
en = np.array([int(buf[640 + b]) for b in range(264)], dtype=np.float64)
t0 = st.min()
s_ = (st - t0) / 1000
e_ = (en - t0) / 1000
print("start min/p50/max", s_.min(), np.median(s_), s_.max())
print("end   min/p50/p90/max", e_.min(), np.median(e_), np.percentile(e_, 90), e_.max())
order = np.argsort(e_)
print("latest CTAs (block, start, end):", [(int(b), round(s_[b], 2), round(e_[b], 2)) for b in order[-12:]])
print("ends by cluster (max over its CTAs):", np.round([e_[c * 8:(c + 1) * 8].max() for c in range(33)], 2))
print("starts by cluster (max):", np.round([s_[c * 8:(c + 1) * 8].max() for c in range(33)], 2))
