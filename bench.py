#!/usr/bin/env python
"""bench.py — the SMART hot path (arXiv 2604.09731) on B200: one decode step = d layers of
expand (A1+A2) + select (A3-A6), build_mask (A7) and verify_accept (A8) for a batch of
requests, on synthetic logits shaped like the paper's workloads (BASELINE.json configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3_llama8b_b32] [--scaling weak|strong]
    python bench.py --impl reference ...      # the fp64 oracle on the host cores

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py relaunches itself under
torch.distributed.run with N ranks (127.0.0.1), one process per GPU.

Prints ONE JSON line (rank 0).  value = tree-steps/s over all ranks (requests whose tree was
built and verified per second); ms_per_step = device time of one whole-batch step.
Timing: CUDA graph per step replayed on rotating input pools larger than 4x L2 (L2-cold),
CUDA events on the capture stream, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

METRIC = "SMART tree-steps/s & µs per decode step at batch 1-32; HBM GB/s vs peak"
UNIT = "tree-steps/s"

# BASELINE.json configs.  b is the global batch at N = 1; weak scaling keeps b per GPU, strong
# scaling splits b over the ranks.
WORKLOADS = {
    "cfg3_llama8b_b32": dict(V=128256, b=32, d=6, k=8, W=8, B_verify=200, fixture="llama8b_b32",
                             desc="Llama-3.1-8B-shaped compute-bound regime: vocab 128256, batch 32, "
                                  "depth 6, top-8, batch-global selection"),
    "cfg2_llama8b_b1": dict(V=128256, b=1, d=6, k=10, W=10, B_verify=60, fixture="llama8b_b1",
                            desc="Llama-3.1-8B-shaped: vocab 128256, batch 1, depth 6, top-10, EAGLE-style tree"),
    "cfg4_qwen2vl_b12": dict(V=152064, b=12, d=8, k=10, W=10, B_verify=200, fixture="qwen2vl7b_b12",
                             desc="Qwen2-VL-7B-shaped MSD-style: vocab 152064, batch 12, depth 8, top-10"),
    # the roofline fixture for a batch-256 target admits nothing (the verify forward is past its
    # compute knee: DESIGN.md §5); the bench runs cfg5 on the labelled synthetic cheap-node cost
    # so that the b = 256 path is exercised on growing trees (--cost roofline: the degenerate one)
    "cfg5_r1distill_b256": dict(V=152064, b=256, d=6, k=8, W=8, B_verify=2048, fixture="synthetic_cheap_b256",
                                fixture_roofline="r1distill_b256",
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
# workload, inputs, the config dict both arms print
# ---------------------------------------------------------------------------------------------
def fixture_name(args, wl):
    if args.cost == "measured":
        return "measured_" + wl["fixture"]
    if args.cost == "roofline" and "fixture_roofline" in wl:
        return wl["fixture_roofline"]
    return wl["fixture"]


def shape(args, wl, world):
    """(global batch, per-rank batch, global B_verify) for the scaling mode"""
    if args.scaling == "strong":
        if wl["b"] % world:
            raise SystemExit(f"strong scaling: batch {wl['b']} not divisible by {world} ranks")
        return wl["b"], wl["b"] // world, wl["B_verify"]
    return wl["b"] * world, wl["b"], wl["B_verify"] * world


def config_dict(args, wl, world):
    """the workload's config, identical in both arms (the driver compares them)"""
    b_glob, b_loc, Bv = shape(args, wl, world)
    c = {"workload": args.workload, "desc": wl["desc"], "V": wl["V"], "global_batch": b_glob, "batch_per_gpu": b_loc,
         "depth": wl["d"], "top_k": wl["k"], "max_frontier": wl["W"], "B_verify": Bv, "alpha": ALPHA,
         "preset": "HOTPATH (PREFIX, NODE_SUM, omega=1)", "cost_fixture": f"fixtures/cost_b200_{fixture_name(args, wl)}.txt",
         "synth": SYNTH, "scaling": args.scaling,
         "parallelism": f"requests sharded dp{world}" + ((", peer exchange per layer (IPC-mapped buffers)" if getattr(args, "exchange", "nccl") == "peer" else ", NCCL all-gather per layer in the step graph") if world > 1 else "")}
    return c


def make_set(seed, wl, T, b, r_offset):
    import numpy as np
    from inputs import synth
    draft = synth.draft_pool(seed, b, T, wl["V"], r_offset=r_offset, sigma_bg=SYNTH["sigma_bg"],
                             a_lo=SYNTH["a_lo"], a_hi=SYNTH["a_hi"])
    target = synth.target_pool(draft, seed + 7919, SYNTH["sigma_m"], r_offset=r_offset)
    rng = np.random.default_rng(seed * 1000 + r_offset)
    root_tok = rng.integers(0, wl["V"], b).astype(np.int32)
    root_pos = rng.integers(64, 4096, b).astype(np.int32)
    return draft, target, root_tok, root_pos


def bf16_dev(a, dev):
    import numpy as np
    import torch
    return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(dev)


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ---------------------------------------------------------------------------------------------
# the fp64 oracle (reference arm, cpu_baseline, bench parity)
# ---------------------------------------------------------------------------------------------
def oracle_objects(wl, cost_fx, b, Bv):
    from oracle import oracle as O
    cfg = O.Config(V=wl["V"], k=wl["k"], d=wl["d"], W=wl["W"], b=b, B_verify=Bv,
                   alpha=ALPHA, omega=1, selection=O.PREFIX, accept_model=O.NODE_SUM)
    cost = O.Cost(lam=cost_fx["lam"], beta=cost_fx["beta"], gamma=cost_fx["gamma"], delta=cost_fx["delta"],
                  rho=cost_fx["rho"], eta=cost_fx["eta"], c_T=cost_fx["c_T"])
    return O, cfg, cost


def time_oracle(wl, cost_fx, sets, b, Bv, threads, budget_s, min_steps=1):
    """the oracle as it stands over the workload's input sets for ~budget_s seconds"""
    O, cfg, cost = oracle_objects(wl, cost_fx, b, Bv)
    O.build()
    O.set_threads(threads)
    n, t0 = 0, time.perf_counter()
    res = None
    while True:
        d, tg, rt, rp = sets[n % len(sets)]
        r = O.step(cfg, cost, d, tg, root_tok=rt, root_pos=rp, dump=False)
        if n == 0:
            res = r
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s and n >= min_steps:
            O.set_threads(1)
            return n, el, res


def step_bytes(wl, rows_expand, verify_rows):
    return (rows_expand + verify_rows) * wl["V"] * 2


def run_reference(args, wl, cost_fx):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    b_glob, b_loc, Bv = shape(args, wl, world)
    T = O.Config(V=wl["V"], k=wl["k"], d=wl["d"], W=wl["W"], b=b_glob, B_verify=Bv).tmax()
    sets = [make_set(s, wl, T, b_glob, 0) for s in range(2)]
    O_, cfg, cost = oracle_objects(wl, cost_fx, b_glob, Bv)
    O.build()
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    for i in range(args.warmup):
        d, tg, rt, rp = sets[i % 2]
        O.step(cfg, cost, d, tg, root_tok=rt, root_pos=rp, dump=False)
    t0 = time.perf_counter()
    for i in range(args.steps):
        d, tg, rt, rp = sets[i % 2]
        O.step(cfg, cost, d, tg, root_tok=rt, root_pos=rp, dump=False)
    el = time.perf_counter() - t0
    value = b_glob * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, wl, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{args.steps} full {args.workload} decode steps ({b_glob} requests each), "
                                   f"fp64 scalar C oracle (oracle/smart_oracle.c), OpenMP over A1/A8 rows, {threads} threads",
                         "host_cpu": _cpu_model(), "host_nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(n):
    """--gpus N without a torchrun environment: run N ranks of this script on one node"""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3_llama8b_b32", choices=list(WORKLOADS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: the workload's batch per GPU; strong: the workload's batch split over the GPUs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N > 1: the per-layer exchange through the library's NCCL all-gather, or the peer "
                         "exchange (records stored straight into every rank's IPC-mapped buffer, DESIGN.md §8)")
    ap.add_argument("--cost", default="default", choices=["default", "roofline", "measured"],
                    help="cost-model fixture: the workload's default, the roofline fit, or measured on a B200 (NEXT #2)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-hbm-regime", action="store_true", help="skip the cfg5 layer-1 HBM-regime measurement")
    ap.add_argument("--steps-only", action="store_true",
                    help="profiling runs: no extras after the timed steps (percentiles, verify, e2e, oracle)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    wl = WORKLOADS[args.workload]
    import make_cost_fixture as mcf
    cost_fx = mcf.load(fixture_name(args, wl))
    if args.impl == "reference":
        return run_reference(args, wl, cost_fx)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2604_09731_b200 import smart as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    b_glob, b, Bv = shape(args, wl, world)
    cfg = S.Config(vocab=wl["V"], top_k=wl["k"], max_depth=wl["d"], max_frontier=wl["W"], batch_local=b,
                   batch_global=b_glob, batch_offset=rank * b, budget_verify=Bv, alpha=ALPHA, bonus=1,
                   selection=S.PREFIX, accept_model=S.NODE_SUM, marginal=S.DERIVATIVE, cost_scope=S.COST_GLOBAL,
                   logits_dtype=S.BF16, row_mode=S.ROWS_NODE)
    cost = S.Cost(lam=cost_fx["lam"], beta=cost_fx["beta"], gamma=cost_fx["gamma"], delta=cost_fx["delta"],
                  rho=cost_fx["rho"], eta=cost_fx["eta"], c_T=cost_fx["c_T"])
    ctx = S.Smart(cfg, cost, local)
    if world > 1 and args.exchange == "peer":
        # the peer exchange: no collective per layer (the end-of-step C2 sums stay per rank)
        from paper_2604_09731_b200 import dist as D
        _peer_keep = D.attach_peer_exchange(ctx)
    elif world > 1:
        # the library's own NCCL communicator: the per-layer all-gather and the end-of-step
        # all-reduce are enqueued on the step's stream, so the sharded step is one CUDA graph
        uid = S.nccl_unique_id() if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctx.attach_nccl(obj[0], rank, world)
    T = ctx.sizes["T"]
    V = wl["V"]

    # ---- inputs: 2 distinct seeded sets, replicated to enough device pools to exceed 4x L2 ----
    host_sets = [make_set(s, wl, T, b, rank * b) for s in range(2)]
    set_bytes = 2 * b * T * V * 2
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    n_pools = max(2, -(-4 * l2 // set_bytes) + 1)
    n_pools += n_pools % 2  # even: pool i holds set i % 2
    pools = []
    for i in range(n_pools):
        d, tg, rt, rp = host_sets[i % 2]
        pools.append(dict(draft=bf16_dev(d, dev), target=bf16_dev(tg, dev),
                          rt=torch.from_numpy(rt).to(dev), rp=torch.from_numpy(rp).to(dev),
                          out=ctx.alloc_outputs()))
    stream = torch.cuda.Stream(dev)

    def step(p, s):
        ctx.run_step(p["draft"], p["target"], p["out"], root_tok=p["rt"], root_pos=p["rp"], stream=s)

    # per-set tree statistics (identical for every replica of a set)
    tree_stats = []
    for i in range(2):
        with torch.cuda.stream(stream):
            step(pools[i], stream)
        stream.synchronize()
        tree_stats.append(ctx.stats())
    out_set0 = {k2: v.cpu().numpy() for k2, v in pools[0]["out"].items()}
    graphs = []
    for p in pools:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(p, stream)
        graphs.append(g)
    torch.cuda.synchronize()
    use_step_kernel = tree_stats[0]["step_kernel_grid"] > 0

    # ---- warm-up + timed region ----
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            graphs[i % n_pools].replay()
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
            graphs[i % n_pools].replay()
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
    value = b_glob * args.steps / (ms / 1e3)

    # ---- per-step latency percentiles: every graph replay bracketed by its own events ----
    pct = None
    if not args.steps_only:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
        with torch.cuda.stream(stream):
            for i, (a, c) in enumerate(evs):
                a.record(stream)
                graphs[i % n_pools].replay()
                c.record(stream)
        stream.synchronize()
        lat = sorted(1e3 * a.elapsed_time(c) for a, c in evs)
        pct = {"us_p10": lat[10], "us_p50": lat[50], "us_p90": lat[90], "replays": len(lat),
               "note": "one CUDA-graph replay per pair of events, rotating L2-cold pools"}

    st0 = tree_stats[0]
    rows_layer = [st0["layers"][l]["n_rows"] if st0["layers"][l]["executed"] else 0 for l in range(wl["d"])]
    nodes = int(st0["nodes_local"])
    ver_rows = b + nodes
    exp_bytes = sum(rows_layer) * V * 2
    ver_bytes = ver_rows * V * 2
    alg_bytes = exp_bytes + ver_bytes
    peak, peak_src = read_peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.workload, {}).get("step")
        except Exception:
            traffic = None
    # the dominant (and, on one GPU, only) kernel is the whole step: algorithmic bytes of one step
    # (every expanded frontier row and every verified tree row read once) over the device time of
    # one step, measured in the timed region (graph replays over L2-cold rotating pools)
    kname = ("step_kernel (persistent whole step: A1-A8)" if use_step_kernel
             else "step (per-layer kernels: layer_kernel x d, select + NCCL all-gather, mask, verify)")
    gbs = alg_bytes / (ms_per_step / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                "traffic": traffic, "kernel": kname, "per_launch_bytes": alg_bytes, "per_launch_ms": ms_per_step,
                "per_launch_source": "timed region: CUDA events over graph replays (L2-cold pools)",
                "peak_source": peak_src}

    # ---- A8 alone, L2-cold: smart_verify_accept on one tree over rotating target pools ----
    roof_verify = None
    if not args.steps_only and world == 1:
        p0 = pools[0]
        with torch.cuda.stream(stream):
            step(p0, stream)  # the tree of set 0
        stream.synchronize()
        same_set = [p for i, p in enumerate(pools) if i % 2 == 0]
        o = p0["out"]
        reps = 30
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for i in range(3):
                ctx.verify_accept(same_set[i % len(same_set)]["target"], o["accept_len"], o["accept_path"], o["bonus"],
                                  stream=stream)
            e0.record(stream)
            for i in range(reps):
                ctx.verify_accept(same_set[i % len(same_set)]["target"], o["accept_len"], o["accept_path"], o["bonus"],
                                  stream=stream)
            e1.record(stream)
        stream.synchronize()
        vms = e0.elapsed_time(e1) / reps
        vg = ver_bytes / (vms / 1e3) / 1e9
        roof_verify = {"bound": "hbm", "kernel": "verify_kernel + verify_walk_kernel (A8, standalone C-ABI call)",
                       "achieved": vg, "peak": peak, "unit": "GB/s", "frac": vg / peak, "per_launch_bytes": ver_bytes,
                       "per_launch_ms": vms, "l2": f"{len(same_set)} rotating target pools of {ver_bytes / 1e6:.0f} MB "
                       f"read rows ({b * T * V * 2 / 1e6:.0f} MB each)", "peak_source": peak_src}
        # A8 at temperature 1 (NEXT #1) on the same tree, L2-cold likewise
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for i in range(reps):
                ctx.verify_sample(same_set[i % len(same_set)]["target"], 1.0, 1000 + i, o["accept_len"],
                                  o["accept_path"], o["bonus"], stream=stream)
            e1.record(stream)
        stream.synchronize()
        roof_verify["verify_sample_T1_ms"] = e0.elapsed_time(e1) / reps

    # ---- end-to-end through the public API with host buffers ----
    e2e = None
    if args.e2e_steps > 0 and not args.steps_only:
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
        e2e = {"value": b_glob * args.e2e_steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / args.e2e_steps,
               "path": "pinned host pools -> cudaMemcpyAsync -> smart_run_step (C-ABI) -> results to host"}

    # ---- the fp64 oracle on this host (rank 0, N = 1): cpu_baseline on 1 thread and on all
    # cores, and the parity of the bench's own GPU results with the oracle on the same inputs ----
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.steps_only:
        ncores = os.cpu_count() or 1
        budget = 6.0 if wl["b"] <= 32 else 12.0
        n1, el1, orc = time_oracle(wl, cost_fx, host_sets, b, Bv, 1, budget)
        na, ela, _ = time_oracle(wl, cost_fx, host_sets, b, Bv, ncores, budget)
        cpu = {"value": b * na / ela, "unit": UNIT, "cores": ncores, "kind": "oracle",
               "sample": f"{na} full {args.workload} decode steps ({b} requests each, the bench's own input sets), "
                         f"fp64 scalar C oracle, OpenMP over A1/A8 rows, {ncores} threads, ~{budget:.0f} s bounded",
               "ms_per_step": 1e3 * ela / na, "host_gbs": alg_bytes / (ela / na) / 1e9,
               "value_1thread": b * n1 / el1, "ms_per_step_1thread": 1e3 * el1 / n1,
               "host_gbs_1thread": alg_bytes / (el1 / n1) / 1e9,
               "host_cpu": _cpu_model(), "host_nproc": ncores}
        # parity: set 0's GPU outputs (pools[0]) against the oracle's step on set 0
        checks = {}
        amb = int(orc.first_ambiguous_layer)
        if amb == 0:
            checks["tree_len"] = bool((out_set0["tree_len"] == orc.n_nodes).all())
            checks["tok"] = bool((out_set0["tok"] == orc.tok).all())
            checks["parent"] = bool((out_set0["parent"] == orc.parent).all())
            checks["pos"] = bool((out_set0["pos"] == orc.pos).all())
            checks["mask"] = bool((out_set0["mask"].view(np.uint32) == orc.mask).all())
            checks["accept_len"] = bool((out_set0["accept_len"] == orc.accept_len).all())
            checks["accept_path"] = bool((out_set0["accept_path"] == orc.accept_path).all())
            checks["bonus"] = bool((out_set0["bonus"] == orc.bonus).all())
            checks["S_rel_err"] = float(abs(st0["S_final"] - orc.S) / abs(orc.S))
        parity = {"ok": bool(amb == 0 and all(v for k2, v in checks.items() if k2 != "S_rel_err")
                             and checks.get("S_rel_err", 1.0) <= 1e-5),
                  "first_ambiguous_layer": amb, "checks": checks,
                  "what": "input set 0 of the timed pools: GPU tree / mask / walk vs the fp64 oracle (bit-exact), S within 1e-5"}

    # ---- the HBM-bound regime of the A1 kernel: cfg5's first layer (256 frontier rows x
    # V = 152064 bf16 = 78 MB per launch), L2-cold rotating pools, CUDA events on the stream ----
    hbm = None
    if rank == 0 and world == 1 and not args.no_hbm_regime and not args.steps_only:
        hbm = hbm_regime(S, dev, stream, peak, peak_src)

    if rank == 0:
        sg = tree_stats[0]  # input set 0 (C2: summed over all ranks)
        beta = sg["accepted_global"] / max(sg["nodes_global"], 1)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "us_per_step": 1e3 * ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": config_dict(args, wl, world),
            "l2_policy": f"{n_pools} rotating input pools x {set_bytes / 1e6:.1f} MB (> 4x L2 {l2 / 1e6:.0f} MB)",
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": args.steps * (1 if use_step_kernel else 1 + wl["d"] * (3 if world > 1 else 1) + 3),
            "step_kernel_grid": tree_stats[0]["step_kernel_grid"],
            "roofline": roofline,
            "roofline_hbm_regime": hbm,
            "roofline_verify": roof_verify,
            "cpu_baseline": cpu,
            "parity": parity,
            "latency": pct,
            "step_algorithmic_bytes": alg_bytes,
            "tree": {"expand_rows_per_layer": rows_layer, "verify_rows": ver_rows, "nodes": nodes,
                     "mean_nodes_per_request": nodes / b, "beta_global": beta,
                     "nodes_global": sg["nodes_global"], "accepted_global": sg["accepted_global"],
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
    tokens), generated on the device; pools rotate over > 2x L2 so every launch reads from HBM.
    Timed as back-to-back launches in one CUDA graph (no launch gaps), CUDA events around it."""
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
    # one graph: (begin + expand layer 1) per pool, back to back; at b = 256 the selection is not
    # fused into the layer kernel (its scratch exceeds the ring), so this times A1+A2 alone (plus
    # the begin kernel, which PDL overlaps with the previous layer kernel's tail)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        for i in range(npool):  # warm
            ctx.begin_step(stream=stream)
            ctx.expand_step(1, pools[i], stream=stream)
        stream.synchronize()
        with torch.cuda.graph(gr, stream=stream):
            for i in range(npool):
                ctx.begin_step(stream=stream)
                ctx.expand_step(1, pools[i], stream=stream)
    times = []
    for rep in range(reps // npool + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            gr.replay()
            e1.record(stream)
        stream.synchronize()
        if rep >= 2:
            times.append(e0.elapsed_time(e1) / npool)
    times.sort()
    med = times[len(times) // 2]
    nbytes = b * V * 2
    ctx.close()
    gbs = nbytes / (med / 1e3) / 1e9
    return {"bound": "hbm", "workload": "cfg5_r1distill_b256 layer 1: 256 rows x 152064 bf16 (78 MB/launch)",
            "kernel": "layer_kernel (A1+A2; begin_step kernels between), back-to-back launches in one CUDA graph",
            "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak, "per_launch_ms_median": med,
            "launches": len(times) * npool, "peak_source": peak_src,
            "l2": f"{npool} rotating pools x {nbytes / 1e6:.0f} MB"}


if __name__ == "__main__":
    sys.exit(main())
