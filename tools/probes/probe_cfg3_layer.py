"""One cfg3 decode step with eager launches, for ncu captures of a single layer kernel (debug aid)."""
import os
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tools")
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
for rep in range(int(os.environ.get("REPS", "2"))):
    ctx.begin_step()
    for layer in range(1, 7):
        ctx.expand_step(layer, dd)
        ctx.select(layer)
torch.cuda.synchronize()
