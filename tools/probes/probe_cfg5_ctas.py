"""Per-CTA start / end of the cfg5 layer-1 kernel (debug aid; SMART_TIMING=1)."""
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
cfg = S.Config(vocab=wl["V"], top_k=wl["k"], max_depth=wl["d"], max_frontier=wl["W"], batch_local=wl["b"],
               budget_verify=wl["B_verify"], alpha=0.8, bonus=1, logits_dtype=S.BF16, row_mode=S.ROWS_NODE)
ctx = S.Smart(cfg, S.Cost(lam=fx["lam"], gamma=fx["gamma"], delta=fx["delta"], rho=fx["rho"], eta=fx["eta"],
                          c_T=fx["c_T"]))
T = ctx.sizes["T"]
d, tg, rt, rp = bench.make_set(0, wl, T, 0)
dd = bench.bf16_dev(d, torch.device("cuda"))
L = S.lib()
L.smart_debug_probes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(1024, np.uint64)
for _ in range(int(os.environ.get("WARM", "300"))):  # clocks ramp
    ctx.begin_step()
    ctx.expand_step(1, dd)
torch.cuda.synchronize()
for rep in range(3):
    ctx.begin_step()
    torch.cuda.synchronize()
    L.smart_debug_probes(ctx._h, None, 1)
    ctx.expand_step(1, dd)
    torch.cuda.synchronize()
    L.smart_debug_probes(ctx._h, buf.ctypes.data_as(C.c_void_p), 0)
st = np.array([int(buf[256 + b]) for b in range(384)], dtype=np.float64)
en = np.array([int(buf[640 + b]) for b in range(384)], dtype=np.float64)
ok = (st > 0) & (st < 1.8e19)
t0 = st[ok].min()
s_ = (st[ok] - t0) / 1000
e_ = (en[ok] - t0) / 1000
print("CTAs", ok.sum(), "start min/p50/max", s_.min(), np.median(s_), s_.max())
print("end   min/p50/p90/max", e_.min(), np.median(e_), np.percentile(e_, 90), e_.max())
print("work dur min/p50/max", (e_ - s_).min(), np.median(e_ - s_), (e_ - s_).max())
print("kernel start/end", (int(buf[66]) - t0) / 1000, (int(buf[67]) - t0) / 1000, "launch", (int(buf[64 + 66]) - t0) / 1000)
print("sorted ends", np.round(np.sort(e_)[::16], 2))
