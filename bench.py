#!/usr/bin/env python
"""bench.py — the SMART hot path (arXiv 2604.09731) on B200: one decode step = d layers of
expand (A1+A2) + select (A3-A6), build_mask (A7) and verify_accept (A8) for a batch of
requests, on synthetic logits shaped like the paper's workloads (BASELINE.json configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3_llama8b_b32]
    python bench.py --impl reference ...      # the fp64 oracle on the host cores

Prints ONE JSON line (rank 0).  value = tree-steps/s over all ranks (requests whose tree was
built and verified per second); ms_per_step = device time of one whole-batch step.
Timing: CUDA graph per step replayed on rotating input pools larger than 4x L2, CUDA events
on the capture stream, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

METRIC = "SMART tree-steps/s & µs per decode step at batch 1-32; HBM GB/s vs peak"
UNIT = "tree-steps/s"

# BASELINE.json configs (per-rank batch for the weak-scaling multi-GPU runs)
WORKLOADS = {
    "cfg3_llama8b_b32": dict(V=128256, b=32, d=6, k=8, W=8, B_verify=200, fixture="llama8b_b32",
                             desc="Llama-3.1-8B-shaped compute-bound regime: vocab 128256, batch 32, "
                                  "depth 6, top-8, batch-global selection"),
    "cfg2_llama8b_b1": dict(V=128256, b=1, d=6, k=10, W=10, B_verify=60, fixture="llama8b_b1",
                            desc="Llama-3.1-8B-shaped: vocab 128256, batch 1, depth 6, top-10, EAGLE-style tree"),
    "cfg4_qwen2vl_b12": dict(V=152064, b=12, d=8, k=10, W=10, B_verify=200, fixture="qwen2vl7b_b12",
                             desc="Qwen2-VL-7B-shaped MSD-style: vocab 152064, batch 12, depth 8, top-10"),
    "cfg5_r1distill_b256": dict(V=152064, b=256, d=6, k=8, W=8, B_verify=2048, fixture="r1distill_b256",
                                desc="DeepSeek-R1-Distill-shaped: vocab 152064, batch 256, depth 6, top-8, "
                                     "B_verify 2048 (B = 8), HBM-bound regime"),
}
SYNTH = dict(sigma_bg=2.0, a_lo=12.0, a_hi=18.0, sigma_m=2.0)  # DESIGN.md §5 input recipe
ALPHA = 0.8


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s"


# ---------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------------------------
def make_set(seed, wl, T, r_offset):
    import numpy as np
    from inputs import synth
    draft = synth.draft_pool(seed, wl["b"], T, wl["V"], r_offset=r_offset, sigma_bg=SYNTH["sigma_bg"],
                             a_lo=SYNTH["a_lo"], a_hi=SYNTH["a_hi"])
    target = synth.target_pool(draft, seed + 7919, SYNTH["sigma_m"], r_offset=r_offset)
    rng = np.random.default_rng(seed * 1000 + r_offset)
    root_tok = rng.integers(0, wl["V"], wl["b"]).astype(np.int32)
    root_pos = rng.integers(64, 4096, wl["b"]).astype(np.int32)
    return draft, target, root_tok, root_pos


def bf16_dev(a, dev):
    import numpy as np
    import torch
    return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(dev)


# ---------------------------------------------------------------------------------------------
# reference arm: the fp64 oracle on the host cores
# ---------------------------------------------------------------------------------------------
def oracle_objects(wl, cost_fx, b_glob=None):
    from oracle import oracle as O
    cfg = O.Config(V=wl["V"], k=wl["k"], d=wl["d"], W=wl["W"], b=wl["b"], B_verify=wl["B_verify"],
                   alpha=ALPHA, omega=1, selection=O.PREFIX, accept_model=O.NODE_SUM)
    cost = O.Cost(lam=cost_fx["lam"], beta=cost_fx["beta"], gamma=cost_fx["gamma"], delta=cost_fx["delta"],
                  rho=cost_fx["rho"], eta=cost_fx["eta"], c_T=cost_fx["c_T"])
    return O, cfg, cost


def time_oracle(wl, cost_fx, sets, budget_s=12.0, min_steps=1, max_steps=None):
    """Run the oracle step over the workload's pools until ~budget_s of CPU time."""
    O, cfg, cost = oracle_objects(wl, cost_fx)
    O.build()
    n, t0 = 0, time.perf_counter()
    while True:
        d, tg, rt, rp = sets[n % len(sets)]
        O.step(cfg, cost, d, tg, root_tok=rt, root_pos=rp, dump=False)
        n += 1
        el = time.perf_counter() - t0
        if (el >= budget_s and n >= min_steps) or (max_steps and n >= max_steps):
            return n, el


def run_reference(args, wl, cost_fx):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    T = O.Config(V=wl["V"], k=wl["k"], d=wl["d"], W=wl["W"], b=wl["b"], B_verify=wl["B_verify"]).tmax()
    sets = [make_set(s, wl, T, 0) for s in range(2)]
    O_, cfg, cost = oracle_objects(wl, cost_fx)
    for i in range(args.warmup):
        d, tg, rt, rp = sets[i % 2]
        O.step(cfg, cost, d, tg, root_tok=rt, root_pos=rp, dump=False)
    t0 = time.perf_counter()
    for i in range(args.steps):
        d, tg, rt, rp = sets[i % 2]
        O.step(cfg, cost, d, tg, root_tok=rt, root_pos=rp, dump=False)
    el = time.perf_counter() - t0
    value = wl["b"] * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.workload, **{k: wl[k] for k in ("V", "b", "d", "k", "W", "B_verify")}},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} full {args.workload} decode steps ({wl['b']} requests each), "
                                   "fp64 scalar C oracle (oracle/smart_oracle.c), 1 thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3_llama8b_b32", choices=list(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cost", default="roofline", choices=["roofline", "measured"],
                    help="cost-model fixture: roofline-fitted (default) or measured on a B200 (NEXT #2)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-hbm-regime", action="store_true", help="skip the cfg5 layer-1 HBM-regime measurement")
    ap.add_argument("--steps-only", action="store_true",
                    help="profiling runs: skip the per-kernel breakdown, verify and T=1 extras after the timed steps")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    import make_cost_fixture as mcf
    cost_fx = mcf.load(wl["fixture"] if args.cost == "roofline" else "measured_" + wl["fixture"])
    if args.impl == "reference":
        return run_reference(args, wl, cost_fx)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2604_09731_b200 import smart as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    b = wl["b"]
    cfg_kwargs = dict(vocab=wl["V"], top_k=wl["k"], max_depth=wl["d"], max_frontier=wl["W"],
                      budget_verify=wl["B_verify"] * world, alpha=ALPHA, bonus=1, selection=S.PREFIX,
                      accept_model=S.NODE_SUM, marginal=S.DERIVATIVE, cost_scope=S.COST_GLOBAL,
                      logits_dtype=S.BF16, row_mode=S.ROWS_NODE)
    cost = S.Cost(lam=cost_fx["lam"], beta=cost_fx["beta"], gamma=cost_fx["gamma"], delta=cost_fx["delta"],
                  rho=cost_fx["rho"], eta=cost_fx["eta"], c_T=cost_fx["c_T"])
    sharded = None
    if world > 1:
        # weak scaling: b requests per GPU, one batch-global selection over b*world requests with
        # one NCCL all-gather per layer (paper_2604_09731_b200/dist.py)
        from paper_2604_09731_b200 import dist as SD
        sharded = SD.ShardedSmart(cfg_kwargs, cost, SD.shard(b * world, world, rank), local)
        ctx = sharded.ctx
    else:
        cfg = S.Config(batch_local=b, batch_global=b, batch_offset=0, **cfg_kwargs)
        ctx = S.Smart(cfg, cost, local)
    T = ctx.sizes["T"]
    V = wl["V"]

    # ---- inputs: 2 distinct seeded sets, replicated to enough device pools to exceed 4x L2 ----
    host_sets = [make_set(s, wl, T, rank * b) for s in range(2)]
    set_bytes = 2 * b * T * V * 2
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    n_pools = max(2, -(-4 * l2 // set_bytes) + 1)
    pools = []
    for i in range(n_pools):
        d, tg, rt, rp = host_sets[i % 2]
        pools.append(dict(draft=bf16_dev(d, dev), target=bf16_dev(tg, dev),
                          rt=torch.from_numpy(rt).to(dev), rp=torch.from_numpy(rp).to(dev),
                          out=ctx.alloc_outputs()))
    stream = torch.cuda.Stream(dev)

    def step(p, s):
        if sharded is not None:
            sharded.step(p["draft"], p["target"], p["out"], root_tok=p["rt"], root_pos=p["rp"], stream=s)
        else:
            ctx.run_step(p["draft"], p["target"], p["out"], root_tok=p["rt"], root_pos=p["rp"], stream=s)

    # per-set tree statistics (identical for every replica of a set)
    tree_stats = []
    for i in range(2):
        with torch.cuda.stream(stream):
            step(pools[i], stream)
        stream.synchronize()
        st = ctx.stats()
        tree_stats.append(st)
    # one CUDA graph per pool buffer (single GPU); eager launches when the step has collectives
    graphs = []
    if sharded is None:
        for p in pools:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(p, stream)
            graphs.append(g)
    torch.cuda.synchronize()
    # begin + d layer kernels + mask + verify stream + verify walk (+ 2 select kernels per layer when sharded)
    launches_per_step = 1 + wl["d"] + 3 + (2 * wl["d"] if world > 1 else 0)

    def replay(i):
        if graphs:
            graphs[i % n_pools].replay()
        else:
            step(pools[i % n_pools], stream)

    # ---- warm-up + timed region ----
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            replay(i)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for i in range(args.steps):
            replay(i)
        ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = b * world * args.steps / (ms / 1e3)

    # ---- per-kernel timing (outside the timed region; events on the launching stream) ----
    kt = {"expand": [], "select": [], "mask": [], "verify": [], "begin": []}
    reps = 20 if sharded is None and not args.steps_only else 0
    p = pools[0]
    for _ in range(reps):
        evs = []
        with torch.cuda.stream(stream):
            def mark():
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                evs.append(e)
            mark()
            ctx.begin_step(p["rt"], p["rp"], stream=stream)
            mark()
            for l in range(1, wl["d"] + 1):
                ctx.expand_step(l, p["draft"], stream=stream)
                mark()
                ctx.select(l, stream=stream)
                mark()
            o = p["out"]
            ctx.build_mask(o["mask"], o["pos"], o["parent"], o["tok"], o["tree_len"], stream=stream)
            mark()
            ctx.verify_accept(p["target"], o["accept_len"], o["accept_path"], o["bonus"], stream=stream)
            mark()
        stream.synchronize()
        d_ = [evs[i].elapsed_time(evs[i + 1]) for i in range(len(evs) - 1)]
        kt["begin"].append(d_[0])
        kt["expand"].append(d_[1:1 + 2 * wl["d"]:2])
        kt["select"].append(d_[2:2 + 2 * wl["d"]:2])
        kt["mask"].append(d_[-2])
        kt["verify"].append(d_[-1])
    # A8 stream + walk back to back on the same tree (each walk clears its row slots, so repeated
    # calls are valid): launch latency overlaps the previous call, so this approximates the
    # kernels' own time (used for the verify roofline)
    ver_rep = None
    if reps:
        o = p["out"]
        nrep, ngraph = 10, 5
        gv = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gv, stream=stream):
            for _ in range(nrep):
                ctx.verify_accept(p["target"], o["accept_len"], o["accept_path"], o["bonus"], stream=stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            gv.replay()
            e0.record(stream)
            for _ in range(ngraph):
                gv.replay()
            e1.record(stream)
        stream.synchronize()
        ver_rep = e0.elapsed_time(e1) / (nrep * ngraph)
    # A8 at temperature 1 (NEXT #1) on the same tree, for the breakdown (not part of the step)
    ver_t1 = []
    for rep in range(reps):
        o = p["out"]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            ctx.verify_sample(p["target"], 1.0, 1000 + rep, o["accept_len"], o["accept_path"], o["bonus"],
                              stream=stream)
            e1.record(stream)
        stream.synchronize()
        ver_t1.append(e0.elapsed_time(e1))
    if reps == 0:
        kt = {"expand": [[0.0] * wl["d"]], "select": [[0.0] * wl["d"]], "mask": [0.0], "verify": [1e-9], "begin": [0.0]}
    st0 = tree_stats[0]
    rows_layer = [st0["layers"][l]["n_rows"] if st0["layers"][l]["executed"] else 0 for l in range(wl["d"])]
    # medians over the repetitions (eager launches are exposed to host-side jitter)
    exp_ms = np.median(np.array(kt["expand"]), axis=0)        # per layer
    sel_ms = np.median(np.array(kt["select"]), axis=0)
    ver_ms = float(np.median(kt["verify"]))
    mask_ms = float(np.median(kt["mask"]))
    beg_ms = float(np.median(kt["begin"]))
    nodes = int(st0["nodes_local"])
    row_bytes = V * 2
    exp_bytes = sum(rows_layer) * row_bytes
    ver_rows = b + nodes
    ver_bytes = ver_rows * row_bytes
    peak, peak_src = read_peaks()
    exp_tot = float(exp_ms[[i for i in range(wl["d"]) if rows_layer[i] > 0]].sum()) if sum(rows_layer) else 0.0
    k_expand = dict(kernel="expand_kernel (A1+A2)", launches=int(sum(1 for r in rows_layer if r > 0)),
                    ms_total=exp_tot, bytes=exp_bytes,
                    gbs=exp_bytes / (exp_tot / 1e3) / 1e9 if exp_tot > 0 else 0.0)
    k_verify = dict(kernel="verify_kernel (A8)", launches=1, ms_total=ver_ms, bytes=ver_bytes,
                    gbs=ver_bytes / (ver_ms / 1e3) / 1e9)
    dom = k_expand if k_expand["ms_total"] >= k_verify["ms_total"] else k_verify
    # dram traffic per launch from a committed ncu --set full capture (if present)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get(args.workload, {}).get("verify" if dom is k_verify else "expand")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": dom["gbs"], "peak": peak, "unit": "GB/s",
                "frac": dom["gbs"] / peak, "traffic": traffic, "kernel": dom["kernel"],
                "per_launch_bytes": dom["bytes"] / max(dom["launches"], 1),
                "per_launch_ms": dom["ms_total"] / max(dom["launches"], 1), "peak_source": peak_src}
    step_alg_bytes = exp_bytes + ver_bytes
    roof_verify = None
    if ver_rep:
        vg = ver_bytes / (ver_rep / 1e3) / 1e9
        roof_verify = {"bound": "hbm", "kernel": "verify_kernel + verify_walk_kernel (A8), 10 back-to-back calls per CUDA graph, L2-warm (same 26 MB each call)",
                       "achieved": vg, "peak": peak, "unit": "GB/s", "frac": vg / peak,
                       "per_launch_bytes": ver_bytes, "per_launch_ms": ver_rep, "peak_source": peak_src}

    # ---- end-to-end through the public API with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        pin = []
        for i in range(2):
            d, tg, rt, rp = host_sets[i]
            pin.append(dict(draft=torch.from_numpy(d.view(np.int16)).view(torch.bfloat16).pin_memory(),
                            target=torch.from_numpy(tg.view(np.int16)).view(torch.bfloat16).pin_memory(),
                            rt=torch.from_numpy(rt).pin_memory(), rp=torch.from_numpy(rp).pin_memory()))
        dp = pools[0]
        res_host = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory()
                    for k, v in dp["out"].items() if k in ("accept_len", "bonus", "tree_len")}
        h2d = sum(int(t.numel() * t.element_size()) for t in pin[0].values())
        d2h = sum(int(t.numel() * t.element_size()) for t in res_host.values())
        def e2e_step(i):
            src = pin[i % 2]
            for k2 in ("draft", "target", "rt", "rp"):
                dp[k2].copy_(src[k2], non_blocking=True)
            step(dp, stream)
            for k2, hv in res_host.items():
                hv.copy_(dp["out"][k2], non_blocking=True)
        with torch.cuda.stream(stream):
            for i in range(3):
                e2e_step(i)
        stream.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for i in range(args.e2e_steps):
                e2e_step(i)
            e1.record(stream)
        stream.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": b * world * args.e2e_steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / args.e2e_steps,
               "path": "pinned host pools -> cudaMemcpyAsync -> smart_run_step (C-ABI) -> results to host"}

    # ---- cpu baseline: the oracle on this host (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n, el = time_oracle(wl, cost_fx, host_sets, budget_s=12.0)
        cpu = {"value": b * n / el, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{n} full {args.workload} decode steps ({b} requests each, same pools), fp64 scalar "
                         "C oracle, 1 thread, ~12 s bounded", "ms_per_step": 1e3 * el / n,
               "host_cpu": _cpu_model(), "host_nproc": os.cpu_count()}

    # ---- the HBM-bound regime of the same kernel: cfg5's first layer (256 frontier rows x
    # V = 152064 bf16 = 78 MB per launch), L2-cold rotating pools, CUDA events on the stream ----
    hbm = None
    if rank == 0 and world == 1 and not args.no_hbm_regime:
        hbm = hbm_regime(S, dev, stream, peak, peak_src)

    if rank == 0:
        beta = st0["accepted_local"] / max(st0["nodes_local"], 1)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "us_per_step": 1e3 * ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": args.workload, "desc": wl["desc"], "V": V, "batch_per_gpu": b,
                       "global_batch": b * world, "depth": wl["d"], "top_k": wl["k"], "max_frontier": wl["W"],
                       "B_verify": wl["B_verify"] * world, "alpha": ALPHA, "preset": "HOTPATH (PREFIX, NODE_SUM, omega=1)",
                       "cost_fixture": f"fixtures/cost_b200_{wl['fixture'] if args.cost == 'roofline' else 'measured_' + wl['fixture']}.txt", "synth": SYNTH,
                       "l2": f"{n_pools} rotating input pools x {set_bytes / 1e6:.1f} MB (> 4x L2 {l2 / 1e6:.0f} MB)",
                       "parallelism": f"requests sharded dp{world}" + (", NCCL all-gather per layer" if world > 1 else "")},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roofline,
            "roofline_hbm_regime": hbm,
            "roofline_verify": roof_verify,
            "cpu_baseline": cpu,
            "step_breakdown_ms": {"begin": beg_ms, "expand_per_layer": [float(x) for x in exp_ms],
                                  "select_per_layer": [float(x) for x in sel_ms], "mask": mask_ms,
                                  "verify": ver_ms,
                                  "verify_sample_T1": float(np.mean(ver_t1)) if ver_t1 else None,
                                  "note": "eager launches, event-bracketed (not the graph), medians of 20"},
            "kernels": {"expand": k_expand, "verify": k_verify},
            "step_algorithmic_bytes": step_alg_bytes,
            "step_hbm_gbs": step_alg_bytes / (ms_per_step / 1e3) / 1e9,
            "tree": {"expand_rows_per_layer": rows_layer, "verify_rows": ver_rows, "nodes": nodes,
                     "mean_nodes_per_request": nodes / b, "beta": beta,
                     "S": st0["S_final"], "layers_executed": st0["layers_executed"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    ctx.close()
    return 0


def hbm_regime(S, dev, stream, peak, peak_src, reps=30):
    """Layer kernel (A1+A2) on cfg5's first layer: 256 frontier rows of V = 152064 bf16 logits in
    FRONTIER row layout, synthetic rows shaped like inputs/synth.py (N(0, 2) background + 8 head
    tokens), generated on the device; pools rotate over > 2x L2 so every launch reads from HBM."""
    import torch
    wl = WORKLOADS["cfg5_r1distill_b256"]
    import make_cost_fixture as mcf
    fx = mcf.load(wl["fixture"])
    b, V = wl["b"], wl["V"]
    cfg = S.Config(vocab=V, top_k=wl["k"], max_depth=wl["d"], max_frontier=wl["W"], batch_local=b,
                   batch_global=b, budget_verify=wl["B_verify"], alpha=ALPHA, bonus=1, logits_dtype=S.BF16,
                   row_mode=S.ROWS_FRONTIER)
    ctx = S.Smart(cfg, S.Cost(lam=fx["lam"], beta=fx["beta"], gamma=fx["gamma"], delta=fx["delta"], rho=fx["rho"],
                              eta=fx["eta"], c_T=fx["c_T"]), dev.index or 0)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    npool = max(3, -(-2 * l2 // (b * V * 2)) + 1)
    pools = []
    for _ in range(npool):
        x = torch.randn(b, V, device=dev, generator=g) * SYNTH["sigma_bg"]
        idx = torch.randint(0, V, (b, 8), device=dev, generator=g)
        amp = (torch.rand(b, 1, device=dev, generator=g) * (SYNTH["a_hi"] - SYNTH["a_lo"]) + SYNTH["a_lo"]) * \
            torch.arange(1, 9, device=dev).float().pow(-0.7)
        x.scatter_add_(1, idx, amp)
        pools.append(x.to(torch.bfloat16))
    times = []
    with torch.cuda.stream(stream):
        for i in range(reps + 10):
            ctx.begin_step(stream=stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.expand_step(1, pools[i % npool], stream=stream)
            e1.record(stream)
            ctx.select(1, stream=stream)
            if i >= 10:
                times.append((e0, e1))
    stream.synchronize()
    ms = sorted(a.elapsed_time(c) for a, c in times)
    med = ms[len(ms) // 2]
    nbytes = b * V * 2
    ctx.close()
    gbs = nbytes / (med / 1e3) / 1e9
    return {"bound": "hbm", "workload": "cfg5_r1distill_b256 layer 1: 256 rows x 152064 bf16 (78 MB/launch)",
            "kernel": "layer_kernel (A1+A2), eager launch incl. launch latency", "achieved": gbs, "peak": peak,
            "unit": "GB/s", "frac": gbs / peak, "per_launch_ms_median": med, "per_launch_ms_min": ms[0],
            "launches": len(ms), "peak_source": peak_src,
            "l2": f"{npool} rotating pools x {nbytes / 1e6:.0f} MB"}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


if __name__ == "__main__":
    sys.exit(main())
