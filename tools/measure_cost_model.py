"""NEXT #2: measure the cost model (Eqs.(4),(5) of arXiv 2604.09731) on this B200.

The paper calibrates its draft/verify latency model per device from "five forward passes"
 but prints no constants (Q18).  This script times an 8B-shaped bf16 target forward
(Llama-3.1-8B: hidden 4096, MLP 14336, 32 layers, 32 query / 8 KV heads of 128, vocab 128256)
and an EAGLE-style draft head (one decoder layer + the full lm_head) with cuBLAS GEMMs (torch)
and flash-attention against a KV cache, at five token counts, and fits

  C_verify(b + N) - c_T = gamma * (exp(delta * N^rho) - 1)       (Eq.(5), eta = c_T)
  C_draft(N)            = lambda * N   (+ beta = 0)               (Eq.(4))

with SPEC's scheme (grid over (delta, rho), closed-form gamma, golden-section refinement;
tools/make_cost_fixture.fit_verify), c_T = the measured AR step of the batch (x = b tokens).
One decoder layer's weights are reused for all 32 layers (each layer's 436 MB still streams from
HBM: it exceeds the L2).  Timings: CUDA graphs of the whole forward, CUDA events, median of reps.

    python tools/measure_cost_model.py --b 32 --ctx 1024 --name measured_llama8b_b32
writes fixtures/cost_b200_<name>.txt (+ the raw timings in the header).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_cost_fixture as mcf  # noqa: E402

H, I, L, NH, NKV, HD, V = 4096, 14336, 32, 32, 8, 128, 128256


class Layer:
    def __init__(self, dev):
        g = torch.Generator(device=dev).manual_seed(0)
        w = lambda *s: (torch.randn(*s, device=dev, generator=g, dtype=torch.float32) * 0.02).to(torch.bfloat16)
        self.qkv = w(H, (NH + 2 * NKV) * HD)
        self.o = w(NH * HD, H)
        self.gu = w(H, 2 * I)
        self.down = w(I, H)
        self.n1 = torch.ones(H, device=dev, dtype=torch.bfloat16)
        self.n2 = torch.ones(H, device=dev, dtype=torch.bfloat16)


def rms(x, w):
    return torch.nn.functional.rms_norm(x, (x.shape[-1],), w)


def layer_fwd(lay, x, b, s, kc, vc, seqlens):
    from flash_attn import flash_attn_with_kvcache
    h = rms(x, lay.n1)
    qkv = h @ lay.qkv
    q, k, v = qkv.split([NH * HD, NKV * HD, NKV * HD], dim=-1)
    q = q.view(b, s, NH, HD)
    k = k.view(b, s, NKV, HD)
    v = v.view(b, s, NKV, HD)
    a = flash_attn_with_kvcache(q, kc, vc, k=k, v=v, cache_seqlens=seqlens, causal=True)
    x = x + a.reshape(b * s, NH * HD) @ lay.o
    h = rms(x, lay.n2)
    gu = h @ lay.gu
    gt, up = gu.split([I, I], dim=-1)
    return x + (torch.nn.functional.silu(gt) * up) @ lay.down


def make_forward(lay, lm, b, s, ctx, nlayers, dev):
    kc = torch.zeros(b, ctx + s, NKV, HD, device=dev, dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    seqlens = torch.full((b,), ctx, device=dev, dtype=torch.int32)
    x0 = torch.randn(b * s, H, device=dev, dtype=torch.bfloat16)

    def fwd():
        x = x0
        for _ in range(nlayers):
            x = layer_fwd(lay, x, b, s, kc, vc, seqlens)
        return x @ lm  # logits for every token (tree verification needs them all)
    return fwd


def time_graph(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del g
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=1024, help="KV-cache length per request")
    ap.add_argument("--budget", type=int, default=200, help="B_verify (samples span 0.1x .. 1.5x)")
    ap.add_argument("--name", default="measured_llama8b_b32")
    args = ap.parse_args()
    dev = torch.device("cuda")
    torch.backends.cuda.matmul.allow_tf32 = False
    lay = Layer(dev)
    lm = (torch.randn(H, V, device=dev, dtype=torch.float32) * 0.02).to(torch.bfloat16)
    b = args.b
    # per-request tree sizes n (tokens beyond the root); N = b * n drafted tokens in the batch
    ns = sorted({max(1, round(args.budget * f / b)) for f in (0.1, 0.4, 0.7, 1.0, 1.5)})
    while len(ns) < 5:
        ns.append(ns[-1] + 1)
    c_T = time_graph(make_forward(lay, lm, b, 1, args.ctx, L, dev))  # one AR step: x = b
    ver = {}
    for n in ns:
        ver[n] = time_graph(make_forward(lay, lm, b, 1 + n, args.ctx, L, dev))
    # draft: one decoder layer + lm_head over the N frontier tokens of a layer (EAGLE-style head)
    dr = {}
    for n in ns:
        dr[n] = time_graph(make_forward(lay, lm, b, n, args.ctx, 1, dev))
    Ns = [b * n for n in ns]
    ys = [ver[n] - c_T for n in ns]
    gamma, delta, rho, rmse = mcf.fit_verify(Ns, ys)
    xs = np.asarray(Ns, float)
    lam = float((xs * np.asarray([dr[n] for n in ns])).sum() / (xs ** 2).sum())
    fx = dict(name=args.name, lam=lam, beta=0.0, gamma=gamma, delta=delta, rho=rho, eta=c_T, c_T=c_T,
              rmse_verify_ms=rmse, samples=Ns)
    raw = dict(device=torch.cuda.get_device_name(), b=b, ctx=args.ctx, c_T_ms=c_T,
               verify_ms={str(b * n): ver[n] for n in ns}, draft_ms={str(b * n): dr[n] for n in ns})
    os.makedirs(os.path.join(mcf.ROOT, "fixtures"), exist_ok=True)
    path = os.path.join(mcf.ROOT, "fixtures", f"cost_b200_{args.name}.txt")
    with open(path, "w") as f:
        f.write("# B200 MEASURED cost model (NEXT #2): tools/measure_cost_model.py -- 8B-shaped bf16 target\n")
        f.write("# forward (cuBLAS GEMMs + flash-attention over a KV cache) and a one-layer draft head,\n")
        f.write(f"# five token counts (P:197), SPEC S:159 fit; verify-fit RMSE {rmse:.3e} ms\n")
        f.write("# raw: " + json.dumps(raw) + "\n")
        for k in ("lam", "beta", "gamma", "delta", "rho", "eta", "c_T"):
            f.write(f"{'lambda' if k == 'lam' else k}={fx[k]:.12g}\n")
    print(json.dumps({**fx, **raw}))
    print(path)


if __name__ == "__main__":
    main()
