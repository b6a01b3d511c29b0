"""Attribute ncu per-SASS-instruction stall samples to CUDA source lines.

    python tools/ncu_lines.py <rep.ncu-rep> <kernel-regex> <cubin> <cubin-function-regex> [--top N]

The cubin (cuobjdump -xelf all paper_2604_09731_b200/libsmart.so) must be the one profiled; its
line table (nvdisasm -g, built with -lineinfo) maps each SASS address to file:line.
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def line_table(cubin, kre):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur_fn, loc, tab = None, None, {}
    for ln in txt.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and re.search(kre, cur_fn):
            tab[int(m.group(1), 16)] = loc
    return tab


def main():
    rep, kre, cubin, fre = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kre}", "--launch-count", "1"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Address"')), len(lines))
    r = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
    h = r[0]
    ia, iss = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    stall = [(i, c) for i, c in enumerate(h) if c.startswith("stall_")]
    tab = line_table(cubin, fre)
    base = None
    agg = defaultdict(lambda: [0.0, defaultdict(float)])
    tot = 0.0
    for x in r[1:]:
        a = int(x[ia], 16) if x[ia].startswith("0x") else int(x[ia])
        base = a if base is None else base
        a -= base
        s = float(x[iss] or 0)
        tot += s
        g = agg[tab.get(a, "?")]
        g[0] += s
        for i, c in stall:
            try:
                g[1][c] += float(x[i] or 0)
            except ValueError:
                pass
    print(f"total samples {tot:.0f}")
    for loc, (s, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        reasons = ", ".join(f"{c[6:]} {v:.0f}" for c, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v > 0)
        print(f"{s:7.0f} {100 * s / tot:5.1f}%  {loc:28s} {reasons}")


if __name__ == "__main__":
    main()
