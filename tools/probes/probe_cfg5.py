"""cfg5 layer-1 expand (256 rows x V=152064) for ncu / timing (debug aid)."""
import os
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tools")
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
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for _ in range(int(os.environ.get("WARM", "0"))):  # let the clocks ramp before timing
    ctx.begin_step()
    ctx.expand_step(1, dd)
    ctx.select(1)
torch.cuda.synchronize()
for rep in range(int(os.environ.get("REPS", "5"))):
    ctx.begin_step()
    ev[0].record(s)
    ctx.expand_step(1, dd)
    ev[1].record(s)
    ctx.select(1)
    ev[2].record(s)
    torch.cuda.synchronize()
    print(f"rep {rep}: expand {ev[0].elapsed_time(ev[1]) * 1000:.1f} us  select {ev[1].elapsed_time(ev[2]) * 1000:.1f} us"
          f"  GB/s {256 * wl['V'] * 2 / (ev[0].elapsed_time(ev[1]) / 1e3) / 1e9:.0f}")
