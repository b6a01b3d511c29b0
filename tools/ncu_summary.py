"""Summarise ncu outputs brought back in gpurun_out/ into committed files under profiles/.

    python tools/ncu_summary.py launches <launches.csv> <out.md>
        per-kernel share of GPU time from a `--metrics gpu__time_duration.sum
        --clock-control none` launch list (cold-cache, serialised: compare SHARES).
    python tools/ncu_summary.py full <capture.ncu-rep> <out.md> [--traffic profiles/ncu_traffic.json]
        key `--set full` metrics per launch (time, DRAM bytes, instructions, occupancy, stalls);
        --traffic also writes the mean per-launch DRAM bytes (read + write) of each kernel family,
        keyed by --workload (bench.py reads it for roofline.traffic).
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict


def short(name):
    m = re.search(r"([A-Za-z_][A-Za-z0-9_]*)(<[^()]*>)?\(", name)
    base = m.group(1) if m else name[:40]
    if "unnamed" in name or base in ("layer_kernel", "verify_kernel", "mask_kernel", "begin_step_kernel",
                                     "select_kernel", "export_frontier_kernel", "step_kernel"):
        return base
    return "torch:" + base if "at::" in name else base


def launches(path, out):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for d in csv.DictReader(io.StringIO("".join(lines))):
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        t = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] == "ns":
            t /= 1000.0
        elif d["Metric Unit"] == "ms":
            t *= 1000.0
        rows.append((short(d["Kernel Name"]), t))
    agg = OrderedDict()
    for k, t in rows:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as f:
        f.write(f"# Launch list: {path.split('/')[-1]}\n\n")
        f.write("ncu `--metrics gpu__time_duration.sum --clock-control none`, every launch of "
                "`bench.py --steps 2 --warmup 1` (cold-cache, serialised; compare shares).\n\n")
        f.write("| kernel | launches | total us | mean us | share |\n|---|---:|---:|---:|---:|\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {k} | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |\n")
        f.write(f"\nTotal {len(rows)} launches, {tot:.1f} us.\n")
    print(open(out).read())


FULL_KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %peak"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(unit, 1)


def to_us(v, unit):
    v = float(v.replace(",", ""))
    return v * {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1)


def full(path, out, traffic_json=None, workload="cfg3_llama8b_b32"):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u = r[0], r[1]
    ix = {k: h.index(k) for k, _ in FULL_KEYS if k in h}
    stall = [(i, k) for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not k.endswith("_not_issued")]
    fam = OrderedDict()
    with open(out, "w") as f:
        f.write(f"# ncu --set full: {path.split('/')[-1]}\n\n")
        f.write("| # | kernel | " + " | ".join(lbl for k, lbl in FULL_KEYS if k in ix) + " | top stalls (pc samples) |\n")
        f.write("|---|---|" + "---:|" * len(ix) + "---|\n")
        for n, row in enumerate(r[2:]):
            name = short(row[h.index("Kernel Name")])
            cells = []
            for k, lbl in FULL_KEYS:
                if k not in ix:
                    continue
                v, un = row[ix[k]], u[ix[k]]
                if k.startswith("dram__bytes"):
                    cells.append(f"{to_bytes(v, un) / 1e6:.2f} MB")
                elif k == "gpu__time_duration.sum":
                    cells.append(f"{to_us(v, un):.2f} us")
                else:
                    cells.append(v)
            st = sorted(((float(row[i].replace(",", "") or 0), k[len("smsp__pcsamp_warps_issue_stalled_"):])
                         for i, k in stall), reverse=True)[:3]
            f.write(f"| {n} | {name} | " + " | ".join(cells) + " | " + ", ".join(f"{k} {int(v)}" for v, k in st) + " |\n")
            if "dram__bytes_read.sum" in ix:
                tb = to_bytes(row[ix["dram__bytes_read.sum"]], u[ix["dram__bytes_read.sum"]]) + \
                    to_bytes(row[ix["dram__bytes_write.sum"]], u[ix["dram__bytes_write.sum"]])
                fam.setdefault(name, []).append(tb)
    if traffic_json:
        alias = {"layer_kernel": "expand", "verify_kernel": "verify", "step_kernel": "step"}
        try:
            js = json.load(open(traffic_json))
        except Exception:
            js = {}
        js[workload] = {alias.get(k, k): sum(v) / len(v) for k, v in fam.items()}
        js[workload]["capture"] = path.split("/")[-1]
        with open(traffic_json, "w") as f:
            json.dump(js, f, indent=1)
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tj = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
        wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "cfg3_llama8b_b32"
        full(sys.argv[2], sys.argv[3], tj, wl)
