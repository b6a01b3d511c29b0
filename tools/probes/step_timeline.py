"""Timeline of one persistent step (step.cu) from its globaltimer probes.
Run with SMART_PROBES=1 SMART_TIMING=1 (the probe build).  Workload: bench cfg3 (or --wl)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np, torch
os.environ.setdefault("SMART_PROBES", "1"); os.environ.setdefault("SMART_TIMING", "1")
from paper_2604_09731_b200 import _build
_build.build()
from paper_2604_09731_b200 import smart as S
import bench

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3_llama8b_b32"]
import make_cost_fixture as mcf
fx = mcf.load(wl["fixture"])
cfg = S.Config(vocab=wl["V"], top_k=wl["k"], max_depth=wl["d"], max_frontier=wl["W"], batch_local=wl["b"],
               budget_verify=wl["B_verify"], alpha=0.8, bonus=1, logits_dtype=S.BF16, row_mode=S.ROWS_NODE)
ctx = S.Smart(cfg, S.Cost(lam=fx["lam"], beta=fx["beta"], gamma=fx["gamma"], delta=fx["delta"], rho=fx["rho"],
                          eta=fx["eta"], c_T=fx["c_T"]))
T = ctx.sizes["T"]
d, tg, rt, rp = bench.make_set(0, wl, T, wl["b"], 0)
dev = torch.device("cuda")
dd, tt = bench.bf16_dev(d, dev), bench.bf16_dev(tg, dev)
out = ctx.alloc_outputs()
L = S.lib()
L.smart_debug_probes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(4096, np.uint64)
s = torch.cuda.Stream()
for it in range(6):
    L.smart_debug_probes(ctx._h, None, 2)
    with torch.cuda.stream(s):
        ctx.run_step(dd, tt, out, stream=s)
    s.synchronize()
    L.smart_debug_probes(ctx._h, buf.ctypes.data, 0)
st = ctx.stats()
rows = [st["layers"][l]["n_rows"] for l in range(wl["d"])]
g = lambda l, sl: int(buf[256 + 16 * l + sl])
mn = lambda l, sl: (~np.uint64(g(l, sl))) if g(l, sl) else 0
t0 = int(mn(0, 3))
f = lambda v: f"{(int(v) - t0) / 1e3:7.2f}" if v else "   -   "
print("rows per layer", rows, "nodes", st["nodes_local"], "err", st["error_flags"])
print("select path per layer", [st["layers"][l]["select_path"] for l in range(len(rows))], "screened", [st["layers"][l]["n_screened"] for l in range(len(rows))], "admitted", [st["layers"][l]["n_admit"] for l in range(len(rows))], "eligible", [st["layers"][l]["n_elig"] for l in range(len(rows))])
print("layer | flag seen min/max | 1st chunk min/max | 1st consumed | posted | slice end max | team lists in | team out | sync1 | merged | published | sel done")
for l in range(1, wl["d"] + 1):
    print(f"{l:5d} | {f(mn(l,3))} {f(g(l,4))} | {f(mn(l,6))} {f(g(l,7))} | {f(g(l,11))} | {f(g(l,12))} | {f(g(l,5))} | {f(g(l,13))} | {f(g(l,14))} | {f(g(l,9))} | {f(g(l,1))} | {f(g(l,2))} | {f(g(l,8))}")
v = 17
print(f"verify: published {f(g(v,2))} flag seen {f(mn(v,3))}-{f(g(v,4))} mask done {f(g(v,1))} slices end {f(g(v,5))} arrived {f(g(v,0))}")
print(f"kernel end {f(g(0,8))} us")
for l in range(1, wl["d"] + 1):
    c = [int(buf[900 + l * 8 + j]) for j in range(4)]
    print(f"layer {l}: merge cycles row0 {c[1]-c[0]}, warp0 rows {c[2]-c[0]}, barrier {c[3]-c[2]}")
names = {9: "start", 10: "benefits", 11: "req-rank", 12: "sort", 13: "A5 cut", 15: "bitmaps", 16: "B6", 20: "popc", 21: "scan",
         17: "counts", 18: "frontier", 19: "published", 14: "adm flags", 22: "end"}
for l in range(1, wl["d"] + 1):
    c = {j: int(buf[3000 + l * 16 + (j - 9)]) for j in range(9, 23)}
    base = c[9]
    if st["layers"][l - 1]["select_path"] in (1, 2):
        sn = {10: "rows", 11: "polled", 12: "A3/A4", 13: "A5 cut", 17: "counts", 18: "entries", 19: "flag", 22: "trace", 16: "end"}
        print(f"layer {l} select_small phases (cycles from start):", ", ".join(f"{sn[j]} {c[j]-base}" for j in (10, 11, 12, 13, 17, 18, 19, 22, 16) if c[j]))
    else:
        print(f"layer {l} select phases (cycles from start):", ", ".join(f"{names[j]} {c[j]-base}" for j in (10, 11, 12, 13, 15, 16, 20, 21, 17, 18, 19, 14, 22) if c[j]))
pc = []
for sidx in range(4096 // 4 - 256):
    a, b_, c_, m = (int(buf[1024 + 4 * sidx + j]) for j in range(4))
    if a:
        pc.append(((a - t0) / 1e3, (b_ - a) / 1e3, (c_ - b_) / 1e3, m & 255, (m >> 8) & 255, m >> 16, sidx))
pc.sort()
print(("A8 per-CTA (SMART_DEBUG_MODE=9): first-chunk arrival, consume time of chunk 1, rest (us), units, first row, smid, cta" if os.environ.get("SMART_DEBUG_MODE") == "9" else "layer-2 per-CTA: first-chunk arrival, consume time of chunk 1, rest of slice (us), nch, row, smid, cta"))
for x in pc[::max(1, len(pc) // 40)]:
    print("  %7.2f %5.2f %5.2f  nch %d row %d sm %d cta %d" % x)
import statistics as stt
print("consume1 median %.2f max %.2f; rest median %.2f" % (stt.median(x[1] for x in pc), max(x[1] for x in pc), stt.median(x[2] for x in pc)))
print("finalize: start %s trees staged %s vrow table %s | walk: slots loaded %s" % tuple(f(buf[j]) for j in (1000, 1001, 1002, 1003)))
