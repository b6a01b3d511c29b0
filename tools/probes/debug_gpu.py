"""Ad-hoc GPU-vs-oracle diff printer (debugging aid, not a test)."""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from smart_gpu_cases import Case, make_inputs, run_gpu, run_oracle  # noqa: E402
from oracle import oracle as O  # noqa: E402

case = Case(V=40000, k=6, d=4, W=6, b=4, B_verify=48, seed=0, cost=(0.02, 0, 0.05, 0.01, 1.2, 1.0, 1.0),
            a_lo=6, a_hi=14, sigma_m=0.5)
if len(sys.argv) > 1:
    case = eval(sys.argv[1])
T = O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify).tmax()
draft, target, rt, rp = make_inputs(case, T)
orc = run_oracle(case, draft, target, rt, rp)
gpu = run_gpu(case, draft, target, rt, rp)
for l in range(1, case.d + 1):
    oc = orc.layer_cands(l)
    gc = gpu["cands"].get(l)
    print("layer", l, "orc trace", orc.trace[l - 1][:5], "gpu",
          {k: gpu["stats"]["layers"][l - 1][k] for k in ("executed", "n_rows", "n_elig", "n_admit", "N0")})
    if gc is None:
        continue
    n = min(len(oc["tok"]), len(gc["tok"]))
    bad = np.nonzero((oc["tok"][:n] != gc["tok"][:n]) | (oc["parent"][:n] != gc["parent"][:n]))[0]
    print(" ncand", len(oc["tok"]), len(gc["tok"]), "mismatch idx", bad[:20])
    for i in bad[:8]:
        print("  i", i, "orc", oc["r"][i], oc["parent"][i], oc["tok"][i], oc["p"][i], "gpu", gc["r"][i],
              gc["parent"][i], gc["tok"][i], gc["p"][i])
    if n:
        print(" p relerr max", np.max(np.abs(gc["p"][:n] - oc["p"][:n]) / oc["p"][:n]))
        print(" adm orc", oc["admitted"][:n].astype(int)[:40])
        print(" adm gpu", gc["admitted"][:n].astype(int)[:40])
print("orc tok", orc.tok[:, :8])
print("gpu tok", gpu["tree"]["tok"][:, :8])
print("orc n", orc.n_nodes, "gpu n", gpu["tree"]["n_nodes"])
