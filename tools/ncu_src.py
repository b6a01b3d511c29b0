"""Per-CUDA-line stall samples and executed instructions from an ncu report (cuda,sass view).

    python tools/ncu_src.py <rep.ncu-rep> [file-substring] [--top N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else ""
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, agg, tot = None, None, [], 0.0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name" or not r[0]:
            continue
        try:
            smp = float(r[4]) if r[4] not in ("-", "") else 0.0
            ins = float(r[7]) if r[7] not in ("-", "") else 0.0
        except (ValueError, IndexError):
            continue
        tot += smp
        if filt in fname:
            agg.append((smp, ins, f"{fname}:{r[0]}", r[1].strip()[:90]))
    agg.sort(reverse=True)
    print(f"total samples {tot:.0f}; lines of '{filt}': {sum(a[0] for a in agg):.0f} samples")
    for smp, ins, loc, src in agg[:top]:
        print(f"{smp:8.0f} {ins:10.0f}  {loc:28s} {src}")


if __name__ == "__main__":
    main()
