"""Aggregate ncu per-SASS-instruction stall samples into regions delimited by clock/globaltimer
reads (the probe stamps) or by fixed-size address windows.

    python tools/sass_hot.py <rep> <kernel-regex> <launch-index> [--window N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kre, li = sys.argv[1], sys.argv[2], int(sys.argv[3])
    win = int(sys.argv[sys.argv.index("--window") + 1]) if "--window" in sys.argv else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kre}", "--launch-skip", str(li), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    r = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = r[0]
    ia, isrc = h.index("Address"), h.index("Source")
    iss = h.index("Warp Stall Sampling (All Samples)")
    iex = h.index("Instructions Executed")
    stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") or "Stall" in c and i != iss]
    rows = r[1:]
    tot = sum(float(x[iss] or 0) for x in rows)
    print(f"total samples {tot:.0f}, instructions {len(rows)}")
    region, reg = 0, defaultdict(lambda: [0.0, 0.0, None, None, defaultdict(float)])
    for n, x in enumerate(rows):
        src = x[isrc]
        if win:
            region = n // win
        elif "SR_CLOCKLO" in src or "SR_GLOBALTIMERLO" in src:
            region += 1
        g = reg[region]
        g[0] += float(x[iss] or 0)
        g[1] += float(x[iex] or 0)
        g[2] = g[2] or x[ia]
        g[3] = x[ia]
    for k in sorted(reg):
        g = reg[k]
        if g[0] / tot > 0.01:
            print(f"region {k:3d} {g[2]}..{g[3]}  samples {g[0]:7.0f} ({100 * g[0] / tot:5.1f}%)  warp-inst {g[1]:9.0f}")
    # top instructions
    top = sorted(rows, key=lambda x: -float(x[iss] or 0))[:25]
    for x in top:
        print(f"  {x[ia]} {float(x[iss] or 0):6.0f}  {x[isrc].strip()[:90]}")


if __name__ == "__main__":
    main()
