"""Select-phase timing at b = 256 (standalone 1024-thread select; debug aid, SMART_TIMING=1)."""
import ctypes as C
import os
import sys

os.environ["SMART_TIMING"] = "1"
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from smart_gpu_cases import Case, gpu_ctx, make_inputs, to_dev  # noqa: E402
from paper_2604_09731_b200 import smart as S  # noqa: E402
from oracle import oracle as O  # noqa: E402

G = int(os.environ.get("G", "1"))
case = Case(V=152064, k=8, d=6, W=8, b=256, B_verify=2048, seed=41, cost=(0.0005, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0))
T = O.Config(V=case.V, k=case.k, d=case.d, W=case.W, b=case.b, B_verify=case.B_verify).tmax()
draft, target, rt, rp = make_inputs(case, T)
ctx = gpu_ctx(case)
dd = to_dev(draft)
L = S.lib()
L.smart_debug_probes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(1024, np.uint64)
s = torch.cuda.current_stream()
for rep in range(3):
    ctx.begin_step()
    for layer in range(1, 4):
        L.smart_debug_probes(ctx._h, None, 1)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(s)
        ctx.expand_step(layer, dd)
        e[1].record(s)
        ctx.select(layer)
        e[2].record(s)
        torch.cuda.synchronize()
        L.smart_debug_probes(ctx._h, buf.ctypes.data_as(C.c_void_p), 0)
        st = [int(buf[32 + j]) for j in range(32)]
        d_ = lambda a, b: st[b] - st[a] if st[a] and st[b] else None
        if rep == 2:
            stt = ctx.stats()["layers"][layer - 1]
            print(f"layer {layer}: rows {stt['n_rows']} elig {stt['n_elig']} admit {stt['n_admit']} | expand {e[0].elapsed_time(e[1])*1e3:.1f} us"
                  f" select {e[1].elapsed_time(e[2])*1e3:.1f} us | cycles stage {d_(9, 10)} rank {d_(10, 11)} sort {d_(11, 12)}"
                  f" A5 {d_(12, 13)} commit {d_(13, 14)} tail {d_(14, 22)}")
