"""One decode step per workload (toy, cfg2, cfg3 shapes) through the C-ABI, for
compute-sanitizer runs (memcheck / synccheck / racecheck):

    compute-sanitizer --tool memcheck python tools/sanitize_steps.py [--path layer|step]

Inputs are the seeded synthetic pools of inputs/synth.py; no oracle is run here.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--path", default="layer", choices=["layer", "step", "both"])
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    import torch
    from inputs import synth
    from paper_2604_09731_b200 import smart as S
    from smart_toy import toy_pool, toy_target
    toy = json.load(open(os.path.join(ROOT, "tests", "golden", "toy_cfg1.json")))
    work = {
        "toy": dict(V=32, k=2, d=3, W=0, b=1, Bv=14, dtype=S.FP32, cost=S.Cost(lam=1.0, eta=10.0, c_T=10.0)),
        "cfg2": dict(V=128256, k=10, d=6, W=10, b=1, Bv=60, dtype=S.BF16,
                     cost=S.Cost(lam=0.0117, eta=2.4631, c_T=2.4631)),
        "cfg3": dict(V=128256, k=8, d=6, W=8, b=32, Bv=200, dtype=S.BF16,
                     cost=S.Cost(lam=0.0117, gamma=0.05, delta=0.02, rho=1.3, eta=2.4631, c_T=2.4631)),
    }
    for name, w in work.items():
        if args.only and name not in args.only.split(","):
            continue
        for path in (["layer", "step"] if args.path == "both" else [args.path]):
            cfg = S.Config(vocab=w["V"], top_k=w["k"], max_depth=w["d"], max_frontier=w["W"], batch_local=w["b"],
                           budget_verify=w["Bv"], logits_dtype=w["dtype"], row_mode=S.ROWS_NODE)
            ctx = S.Smart(cfg, w["cost"])
            T = ctx.sizes["T"]
            if name == "toy":
                draft = torch.from_numpy(toy_pool(toy, T)).cuda()
                target = torch.from_numpy(toy_target(toy, T)).cuda()
            else:
                d = synth.draft_pool(1, w["b"], T, w["V"])
                t = synth.target_pool(d, 2, 1.0)
                draft = torch.from_numpy(d.view(np.int16)).view(torch.bfloat16).cuda()
                target = torch.from_numpy(t.view(np.int16)).view(torch.bfloat16).cuda()
            out = ctx.alloc_outputs()
            if path == "step":
                ctx.run_step(draft, target, out)
            else:
                ctx.begin_step()
                for l in range(1, w["d"] + 1):
                    ctx.expand_step(l, draft)
                    ctx.select(l)
                ctx.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"])
                ctx.verify_accept(target, out["accept_len"], out["accept_path"], out["bonus"])
            torch.cuda.synchronize()
            st = ctx.stats()
            print(name, path, "tree_len", out["tree_len"].tolist()[:8], "accept", out["accept_len"].tolist()[:8],
                  "flags", st["error_flags"], flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
