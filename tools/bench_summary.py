"""Print the key fields of bench.py JSON lines: python tools/bench_summary.py <file.json> ..."""
import json
import sys

for f in sys.argv[1:]:
    print("==", f)
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print("  no JSON line:", e)
        continue
    print("  us/step %.1f  value %.0f %s" % (d["ms_per_step"] * 1e3, d["value"], d.get("unit")))
    for k in ("roofline", "roofline_verify", "roofline_hbm_regime", "latency", "parity", "tree", "clocks",
              "cpu_baseline", "e2e"):
        v = d.get(k)
        if isinstance(v, dict):
            v = {a: (round(b, 4) if isinstance(b, float) else b) for a, b in v.items()
                 if a not in ("sample", "note", "peak_source", "what", "desc", "path")}
        print("  ", k, v)
