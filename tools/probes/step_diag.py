"""Diagnostic: is the persistent step kernel selected, and how long does a cfg3 step take on
each path (eager, CUDA events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2604_09731_b200 import smart as S
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import make_cost_fixture as mcf
from inputs import synth

fx = mcf.load("llama8b_b32")
V, b, d, k, W, Bv = 128256, 32, 6, 8, 8, 200
cfg = S.Config(vocab=V, top_k=k, max_depth=d, max_frontier=W, batch_local=b, budget_verify=Bv, alpha=0.8, bonus=1,
               logits_dtype=S.BF16, row_mode=S.ROWS_NODE)
ctx = S.Smart(cfg, S.Cost(lam=fx["lam"], beta=fx["beta"], gamma=fx["gamma"], delta=fx["delta"], rho=fx["rho"],
                          eta=fx["eta"], c_T=fx["c_T"]))
T = ctx.sizes["T"]
draft = synth.draft_pool(0, b, T, V, a_lo=12, a_hi=18)
target = synth.target_pool(draft, 7919, 2.0)
dev = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
dd, tt = dev(draft), dev(target)
out = ctx.alloc_outputs()
s = torch.cuda.Stream()
for it in range(3):
    with torch.cuda.stream(s):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ctx.run_step(dd, tt, out, stream=s)
        e1.record(s)
    s.synchronize()
    print("run_step ms", e0.elapsed_time(e1), "stats", ctx.stats()["nodes_local"], ctx.stats()["error_flags"], flush=True)
