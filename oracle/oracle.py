"""ctypes front-end of the fp64 SMART oracle (oracle/smart_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  It never
imports the product package (paper_2604_09731_b200) and the product never
imports it.

Every quantity follows PAPER.md (arXiv 2604.09731) — see the citations in
smart_oracle.c — with the readings Q1..Q26 of DESIGN.md §3.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smart_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

PREFIX, FROZEN = 0, 1
NODE_SUM, PATH_MEAN = 0, 1
DERIVATIVE, DIFFERENCE = 0, 1
BF16, FP32 = 0, 1
ROWS_NODE, ROWS_FRONTIER, ROWS_KARY, ROWS_POSITION = 0, 1, 2, 3
TRACE_F = 14
SUM_F = 9
TRACE_NAMES = ["n_rows", "n_cand", "n_elig", "n_admit", "N0", "E0", "S0", "S_after",
               "argmax_j", "dc0", "min_margin", "ambiguous", "executed", "saturated"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc -O2 (no intrinsics, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "smart_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=gnu99", "-fopenmp", "-Wall", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Cost(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("lambda_", "beta", "gamma", "delta", "rho", "eta", "c_T")]


class _Cfg(C.Structure):
    _fields_ = [("V", C.c_int32), ("k", C.c_int32), ("d", C.c_int32), ("W", C.c_int32),
                ("b", C.c_int32), ("B_verify", C.c_int32), ("alpha", C.c_double),
                ("omega", C.c_int32), ("selection", C.c_int32), ("accept_model", C.c_int32),
                ("marginal", C.c_int32), ("dtype", C.c_int32), ("row_mode", C.c_int32),
                ("T", C.c_int32), ("margin_eps", C.c_double), ("b_budget", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        d, i32, i64, vp = C.c_double, C.c_int32, C.c_int64, C.c_void_p
        pc = C.POINTER(_Cost)
        L.orc_cost_draft.argtypes = [pc, d]; L.orc_cost_draft.restype = d
        L.orc_cost_verify.argtypes = [pc, d, vp]; L.orc_cost_verify.restype = d
        L.orc_cost_spec.argtypes = [pc, d, vp]; L.orc_cost_spec.restype = d
        L.orc_dc.argtypes = [pc, C.c_int, i64, vp]; L.orc_dc.restype = d
        L.orc_speedup.argtypes = [pc, C.c_int, C.c_int, d, i64]; L.orc_speedup.restype = d
        L.orc_delta_j.argtypes = [d, d, d, d, d]; L.orc_delta_j.restype = d
        L.orc_l_tree_path_mean.argtypes = [i32, vp, vp]; L.orc_l_tree_path_mean.restype = d
        L.orc_l_tree_node_sum.argtypes = [i32, vp]; L.orc_l_tree_node_sum.restype = d
        L.orc_topk_softmax.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]
        L.orc_topk_softmax.restype = C.c_int
        L.orc_step.argtypes = ([C.POINTER(_Cfg), pc, vp, i64, i64, vp, i64, vp, vp]
                               + [vp] * 8 + [vp] * 3 + [vp, i64, vp, vp, vp])
        L.orc_step.restype = C.c_int
        L.orc_baseline_step.argtypes = [C.POINTER(_Cfg), vp, i64, vp, i64, vp, vp] + [vp] * 12
        L.orc_baseline_step.restype = C.c_int
        L.orc_verify_sample.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, i64, vp, vp, vp,
                                        d, C.c_uint64, vp, vp, vp, vp]
        L.orc_verify_sample.restype = C.c_int
        L.orc_hash.argtypes = [C.c_uint64, i64, i64, i64]
        L.orc_hash.restype = C.c_uint64
        L.orc_uniform.argtypes = [C.c_uint64, i64, i64, i64]
        L.orc_uniform.restype = d
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_set_threads.restype = None
        _lib = L
    return _lib


@dataclass
class Cost:
    """Eq.(4) lambda, beta; Eq.(5) gamma, delta, rho, eta; Eq.(1) c_T."""
    lam: float = 1.0
    beta: float = 0.0
    gamma: float = 0.0
    delta: float = 0.0
    rho: float = 1.0
    eta: float = 0.0
    c_T: float = 1.0

    def c(self) -> _Cost:
        return _Cost(self.lam, self.beta, self.gamma, self.delta, self.rho, self.eta, self.c_T)


@dataclass
class Config:
    V: int
    k: int
    d: int
    W: int = 0                 # 0 = unlimited
    b: int = 1
    B_verify: int = 200
    alpha: float = 0.8
    omega: int = 1
    selection: int = PREFIX
    accept_model: int = NODE_SUM
    marginal: int = DERIVATIVE
    dtype: int = BF16
    row_mode: int = ROWS_NODE
    T: int = 0                 # 0 -> derived: 1 + min(B, d*W)
    margin_eps: float = 1e-5   # Q24: decisions closer than 1e-5 are tie-ambiguous
    b_budget: int = 0          # requests sharing B_verify (0 = b); > b: LOCAL cost scope (Q34)

    @property
    def B(self) -> int:
        return self.B_verify // (self.b_budget or self.b)

    def tmax(self) -> int:
        if self.T:
            return self.T
        Wq = self.W if self.W > 0 else 1 << 30
        return 1 + min(self.B, self.d * Wq)

    def c(self) -> _Cfg:
        return _Cfg(self.V, self.k, self.d, self.W, self.b, self.B_verify, self.alpha, self.omega,
                    self.selection, self.accept_model, self.marginal, self.dtype, self.row_mode,
                    self.tmax(), self.margin_eps, self.b_budget)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ---- closed-form pieces -----------------------------------------------------

def cost_draft(cost: Cost, x: float) -> float:
    c = cost.c()
    return lib().orc_cost_draft(C.byref(c), float(x))


def cost_verify(cost: Cost, x: float):
    c = cost.c()
    sat = C.c_int(0)
    v = lib().orc_cost_verify(C.byref(c), float(x), C.byref(sat))
    return v, bool(sat.value)


def cost_spec(cost: Cost, x: float) -> float:
    c = cost.c()
    return lib().orc_cost_spec(C.byref(c), float(x), None)


def dc(cost: Cost, N: int, marginal: int = DERIVATIVE):
    c = cost.c()
    sat = C.c_int(0)
    v = lib().orc_dc(C.byref(c), marginal, int(N), C.byref(sat))
    return v, bool(sat.value)


def speedup(cost: Cost, omega: int, b: int, E: float, N: int) -> float:
    c = cost.c()
    return lib().orc_speedup(C.byref(c), omega, b, float(E), int(N))


def delta_j(alpha, d_target, d_spec, c_target, c_spec) -> float:
    return lib().orc_delta_j(alpha, d_target, d_spec, c_target, c_spec)


def l_tree_path_mean(parent, cum) -> float:
    parent = np.ascontiguousarray(parent, np.int32)
    cum = np.ascontiguousarray(cum, np.float64)
    return lib().orc_l_tree_path_mean(len(parent), _ptr(parent), _ptr(cum))


def l_tree_node_sum(cum) -> float:
    cum = np.ascontiguousarray(cum, np.float64)
    return lib().orc_l_tree_node_sum(len(cum), _ptr(cum))


def topk_softmax(row: np.ndarray, k: int):
    """row: uint16 (bf16 bits) or float32.  Returns (tok[k], p[k], m, Z)."""
    row = np.ascontiguousarray(row)
    dt = BF16 if row.dtype == np.uint16 else FP32
    tok = np.zeros(k, np.int32)
    p = np.zeros(k, np.float64)
    m = C.c_double()
    Z = C.c_double()
    rc = lib().orc_topk_softmax(_ptr(row), dt, row.shape[-1], k, _ptr(tok), _ptr(p),
                                C.byref(m), C.byref(Z))
    if rc:
        raise ValueError("invalid logits row (NaN/+inf or all -inf)")
    return tok, p, m.value, Z.value


@dataclass
class StepResult:
    n_nodes: np.ndarray
    tok: np.ndarray
    parent: np.ndarray
    depth: np.ndarray
    pos: np.ndarray
    p: np.ndarray
    cum: np.ndarray
    mask: np.ndarray
    accept_len: np.ndarray
    accept_path: np.ndarray
    bonus: np.ndarray
    trace: np.ndarray
    cand_i: np.ndarray
    cand_d: np.ndarray
    summary: np.ndarray
    T: int
    extra: dict = field(default_factory=dict)

    @property
    def E(self):
        return self.summary[0]

    @property
    def N(self):
        return int(self.summary[1])

    @property
    def S(self):
        return self.summary[2]

    @property
    def beta(self):
        return self.summary[4]

    @property
    def first_ambiguous_layer(self):
        return int(self.summary[5])

    def layer_cands(self, layer: int):
        """candidates of a layer: dict of arrays (r, parent, tok, c, admitted, p, cum, b)."""
        ci = self.cand_i[layer - 1]
        cd = self.cand_d[layer - 1]
        n = int(self.trace[layer - 1, 1])
        return dict(r=ci[:n, 0], parent=ci[:n, 1], tok=ci[:n, 2], c=ci[:n, 3],
                    admitted=ci[:n, 4].astype(bool), p=cd[:n, 0], cum=cd[:n, 1], b=cd[:n, 2])


def step(cfg: Config, cost: Cost, draft: np.ndarray, target: np.ndarray | None = None,
         root_tok=None, root_pos=None, layer_stride: int = 0, dump: bool = True) -> StepResult:
    """Run one SMART decode step (Algorithm 1 + mask + greedy verify) in fp64.

    draft: uint16 (bf16 bits) or float32 array whose last axis is the (possibly padded) vocab;
           ROWS_NODE: shape [b, T, ld]; ROWS_FRONTIER: [d, rows_cap, ld] (layer_stride derived);
           ROWS_KARY: [b, n_kary, ld]; ROWS_POSITION (DFLASH): [b, >= d, ld].
    target: same dtype, [b, T, ld_t] or None.
    """
    b, T, d, k = cfg.b, cfg.tmax(), cfg.d, cfg.k
    draft = np.ascontiguousarray(draft)
    want = np.uint16 if cfg.dtype == BF16 else np.float32
    assert draft.dtype == want, (draft.dtype, want)
    ld = draft.shape[-1]
    if cfg.row_mode == ROWS_FRONTIER:
        layer_stride = draft.shape[1] * ld
    elif cfg.row_mode in (ROWS_KARY, ROWS_POSITION):
        layer_stride = draft.shape[1]
    if target is not None:
        target = np.ascontiguousarray(target)
        assert target.dtype == want and target.shape[0] == b and target.shape[1] == T
    MW = (T + 31) // 32
    D = max(d, 1)
    capc = b * T * k
    out = dict(
        n_nodes=np.zeros(b, np.int32), tok=np.zeros(b * T, np.int32), parent=np.zeros(b * T, np.int32),
        depth=np.zeros(b * T, np.int32), pos=np.zeros(b * T, np.int32), p=np.zeros(b * T),
        cum=np.zeros(b * T), mask=np.zeros(b * T * MW, np.uint32), accept_len=np.zeros(b, np.int32),
        accept_path=np.full(b * D, -1, np.int32), bonus=np.zeros(b, np.int32),
        trace=np.zeros(D * TRACE_F), summary=np.zeros(SUM_F))
    cand_i = np.zeros(D * capc * 5, np.int32) if dump else None
    cand_d = np.zeros(D * capc * 3) if dump else None
    rt = np.ascontiguousarray(root_tok if root_tok is not None else np.full(b, -1), np.int32)
    rp = np.ascontiguousarray(root_pos if root_pos is not None else np.zeros(b), np.int32)
    c_cfg, c_cost = cfg.c(), cost.c()
    rc = lib().orc_step(C.byref(c_cfg), C.byref(c_cost), _ptr(draft), ld, layer_stride,
                        _ptr(target), target.shape[-1] if target is not None else 0,
                        _ptr(rt), _ptr(rp),
                        *[_ptr(out[x]) for x in ("n_nodes", "tok", "parent", "depth", "pos", "p",
                                                 "cum", "mask")],
                        _ptr(out["accept_len"]), _ptr(out["accept_path"]), _ptr(out["bonus"]),
                        _ptr(out["trace"]), capc, _ptr(cand_i), _ptr(cand_d), _ptr(out["summary"]))
    if rc == 1:
        raise ValueError("invalid config")
    if rc == 2:
        raise ValueError("invalid logits (NaN/+inf)")
    return StepResult(
        n_nodes=out["n_nodes"], tok=out["tok"].reshape(b, T), parent=out["parent"].reshape(b, T),
        depth=out["depth"].reshape(b, T), pos=out["pos"].reshape(b, T), p=out["p"].reshape(b, T),
        cum=out["cum"].reshape(b, T), mask=out["mask"].reshape(b, T, MW),
        accept_len=out["accept_len"], accept_path=out["accept_path"].reshape(b, D),
        bonus=out["bonus"], trace=out["trace"].reshape(D, TRACE_F),
        cand_i=cand_i.reshape(D, capc, 5) if dump else None,
        cand_d=cand_d.reshape(D, capc, 3) if dump else None, summary=out["summary"], T=T)


def set_threads(n: int) -> None:
    """worker threads for the row-parallel parts (A1 rows, A8 requests); 1 = serial."""
    lib().orc_set_threads(int(n))


def uniform(seed: int, r: int, u: int, v: int) -> float:
    """The counter-based uniform of the T > 0 verification (orc_uniform)."""
    return lib().orc_uniform(seed, r, u, v)


def verify_sample(target: np.ndarray, n_nodes, parent, tok, tau: float, seed: int, d: int,
                  r_off: int = 0, V: int | None = None):
    """NEXT #1 (Q31): tree verification at temperature tau > 0 over an existing tree.

    target: [b, T, ld] uint16 (bf16 bits) or float32; n_nodes [b]; parent/tok [b, T].
    Returns (accept_len [b], accept_path [b, max(d,1)], bonus [b], margin [b])."""
    target = np.ascontiguousarray(target)
    dtype = BF16 if target.dtype == np.uint16 else FP32
    b, T, ld = target.shape
    D = max(d, 1)
    V = ld if V is None else V
    out_a = np.zeros(b, np.int32)
    out_p = np.full(b * D, -1, np.int32)
    out_b = np.zeros(b, np.int32)
    mg = np.zeros(b)
    nn = np.ascontiguousarray(n_nodes, np.int32)
    pa = np.ascontiguousarray(parent, np.int32)
    tk = np.ascontiguousarray(tok, np.int32)
    rc = lib().orc_verify_sample(dtype, V, T, b, r_off, d, _ptr(target), ld, _ptr(nn), _ptr(pa), _ptr(tk),
                                 float(tau), int(seed) & ((1 << 64) - 1), _ptr(out_a), _ptr(out_p),
                                 _ptr(out_b), _ptr(mg))
    if rc == 1:
        raise ValueError("invalid arguments")
    if rc == 2:
        raise ValueError("invalid logits (NaN)")
    return out_a, out_p.reshape(b, D), out_b, mg


def baseline_T(cfg: Config) -> int:
    """tree capacity of the two-stage baseline: expanded nodes (1 + W d) and the final top-g tree."""
    g = cfg.B_verify // cfg.b
    return max(1 + g, 1 + cfg.W * max(cfg.d, 1))


def baseline_step(cfg: Config, draft: np.ndarray, target: np.ndarray | None = None, root_tok=None, root_pos=None):
    """NEXT #3 (Q32): the likelihood-maximising two-stage baseline (EAGLE-3 / MSD, Fig. 2(a)(b)).

    draft/target: [b, T, ld] (T = baseline_T(cfg); draft rows at (r, expanded node), target rows at
    (r, final node)).  cfg.W = nodes expanded per layer, cfg.k = children per node, g = B_verify // b.
    Returns a StepResult (trace/candidates empty) with extra['n_exp'] = expanded nodes per request."""
    b, d = cfg.b, cfg.d
    T = baseline_T(cfg)
    draft = np.ascontiguousarray(draft)
    if cfg.row_mode == ROWS_POSITION:  # DFLASH position rows [b, d, ld]
        assert draft.shape[0] == b and draft.shape[1] == d, (draft.shape, b, d)
    else:
        assert draft.shape[0] == b and draft.shape[1] == T, (draft.shape, b, T)
    ld = draft.shape[-1]
    if target is not None:
        target = np.ascontiguousarray(target)
        assert target.shape[:2] == (b, T)
    MW = (T + 31) // 32
    D = max(d, 1)
    out = dict(n_nodes=np.zeros(b, np.int32), tok=np.zeros(b * T, np.int32), parent=np.zeros(b * T, np.int32),
               depth=np.zeros(b * T, np.int32), pos=np.zeros(b * T, np.int32), p=np.zeros(b * T), cum=np.zeros(b * T),
               mask=np.zeros(b * T * MW, np.uint32), accept_len=np.zeros(b, np.int32),
               accept_path=np.full(b * D, -1, np.int32), bonus=np.zeros(b, np.int32), n_exp=np.zeros(b, np.int32))
    rt = np.ascontiguousarray(root_tok if root_tok is not None else np.full(b, -1), np.int32)
    rp = np.ascontiguousarray(root_pos if root_pos is not None else np.zeros(b), np.int32)
    c_cfg = Config(**{**cfg.__dict__}).c()
    c_cfg.T = T
    rc = lib().orc_baseline_step(C.byref(c_cfg), _ptr(draft), ld, _ptr(target), target.shape[-1] if target is not None else 0,
                                 _ptr(rt), _ptr(rp), *[_ptr(out[x]) for x in ("n_nodes", "tok", "parent", "depth", "pos",
                                                                            "p", "cum", "mask", "accept_len",
                                                                            "accept_path", "bonus", "n_exp")])
    if rc == 1:
        raise ValueError("invalid config")
    if rc == 2:
        raise ValueError("invalid logits")
    return StepResult(n_nodes=out["n_nodes"], tok=out["tok"].reshape(b, T), parent=out["parent"].reshape(b, T),
                      depth=out["depth"].reshape(b, T), pos=out["pos"].reshape(b, T), p=out["p"].reshape(b, T),
                      cum=out["cum"].reshape(b, T), mask=out["mask"].reshape(b, T, MW), accept_len=out["accept_len"],
                      accept_path=out["accept_path"].reshape(b, D), bonus=out["bonus"], trace=np.zeros((D, TRACE_F)),
                      cand_i=None, cand_d=None, summary=np.zeros(SUM_F), T=T, extra=dict(n_exp=out["n_exp"]))
