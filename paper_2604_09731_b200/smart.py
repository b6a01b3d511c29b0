"""Thin Python binding of libsmart.so (include/smart.h) — argument marshalling only.

Every step of the SMART hot path runs in the CUDA kernels behind the C-ABI; this module
only turns torch tensors into device pointers and streams into cudaStream_t handles.
If libsmart.so is missing or cannot be loaded, importing the binding raises: there is no
CPU fallback in the product path.

Names follow the paper (arXiv 2604.09731): k, d, alpha, B_verify, c_T, lambda, gamma,
delta, rho, eta; the calls are the C-ABI's (smart_expand_step, smart_select,
smart_build_mask, smart_verify_accept).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsmart.so")

OK, EINVAL, ECUDA, ENCCL, ECAPACITY, EDEVICE, ESTATE = range(7)
BF16, FP32 = 0, 1
PREFIX, FROZEN, BASELINE = 0, 1, 2  # BASELINE: two-stage likelihood-maximising tree (Q32)
NODE_SUM, PATH_MEAN = 0, 1
DERIVATIVE, DIFFERENCE = 0, 1
COST_GLOBAL, COST_LOCAL = 0, 1
ROWS_FRONTIER, ROWS_NODE, ROWS_POSITION = 0, 1, 2  # POSITION: DFLASH rows
MAX_DEPTH = 16

EXPORTED = ["smart_query_sizes", "smart_create", "smart_nccl_unique_id", "smart_attach_nccl",
            "smart_exchange_record_bytes", "smart_attach_exchange", "smart_select_finish",
            "smart_peer_exchange_bytes", "smart_attach_peer_exchange", "smart_ipc_get_handle",
            "smart_ipc_open_handle", "smart_ipc_close",
            "smart_destroy", "smart_begin_step", "smart_expand_step", "smart_select",
            "smart_build_mask", "smart_verify_accept", "smart_verify_sample", "smart_run_step", "smart_get_stats",
            "smart_get_tree", "smart_get_candidates", "smart_last_error", "smart_status_string"]


class SmartError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libsmart status {status}: {msg}")
        self.status = status


class _Cost(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("delta", C.c_double), ("rho", C.c_double), ("eta", C.c_double), ("c_T", C.c_double)]


class _Config(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("top_k", C.c_int32), ("max_depth", C.c_int32),
                ("max_frontier", C.c_int32), ("batch_local", C.c_int32), ("batch_global", C.c_int32),
                ("batch_offset", C.c_int32), ("budget_verify", C.c_int32), ("alpha", C.c_double),
                ("bonus", C.c_int32), ("selection", C.c_int32), ("accept_model", C.c_int32),
                ("marginal", C.c_int32), ("cost_scope", C.c_int32), ("logits_dtype", C.c_int32),
                ("row_mode", C.c_int32), ("tree_capacity", C.c_int32)]


class _Sizes(C.Structure):
    _fields_ = [("B", C.c_int32), ("T", C.c_int32), ("mask_words", C.c_int32),
                ("frontier_cap", C.c_int32), ("chunk_elems", C.c_int32)]


class _LayerTrace(C.Structure):
    _fields_ = [("executed", C.c_int32), ("n_rows", C.c_int32), ("n_cand", C.c_int32),
                ("n_elig", C.c_int32), ("n_admit", C.c_int32), ("argmax_j", C.c_int32),
                ("N0", C.c_int32), ("saturated", C.c_int32), ("select_path", C.c_int32),
                ("n_screened", C.c_int32), ("E0", C.c_double), ("S0", C.c_double),
                ("S_after", C.c_double), ("dc0", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("layers_executed", C.c_int32), ("error_flags", C.c_int32),
                ("nodes_local", C.c_int64), ("accepted_local", C.c_int64),
                ("accepted_global", C.c_int64), ("nodes_global", C.c_int64),
                ("step_kernel_grid", C.c_int32), ("reserved", C.c_int32),
                ("E_global", C.c_double), ("S_final", C.c_double),
                ("layer", _LayerTrace * MAX_DEPTH)]


_lib = None


def lib() -> C.CDLL:
    """Load libsmart.so; raise loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                              "(python -m paper_2604_09731_b200._build)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, st = C.c_void_p, C.c_int32, C.c_int64, C.c_int
        L.smart_query_sizes.argtypes = [C.POINTER(_Config), C.POINTER(_Sizes)]
        L.smart_create.argtypes = [C.POINTER(_Config), C.POINTER(_Cost), C.c_int, C.POINTER(vp)]
        L.smart_nccl_unique_id.argtypes = [C.c_char_p]
        L.smart_attach_nccl.argtypes = [vp, C.c_char_p, C.c_int, C.c_int]
        L.smart_exchange_record_bytes.argtypes = [C.POINTER(_Config), C.c_int, C.POINTER(i64)]
        L.smart_attach_exchange.argtypes = [vp, C.c_int, C.c_int, vp, vp]
        L.smart_select_finish.argtypes = [vp, i32, vp, vp, vp]
        L.smart_peer_exchange_bytes.argtypes = [C.POINTER(_Config), C.c_int, C.POINTER(i64)]
        L.smart_attach_peer_exchange.argtypes = [vp, C.c_int, C.c_int, C.POINTER(vp)]
        L.smart_ipc_get_handle.argtypes = [vp, C.c_char_p]
        L.smart_ipc_open_handle.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.smart_ipc_close.argtypes = [vp]
        L.smart_destroy.argtypes = [vp]
        L.smart_begin_step.argtypes = [vp, vp, vp, vp]
        L.smart_expand_step.argtypes = [vp, i32, vp, i64, vp]
        L.smart_select.argtypes = [vp, i32, vp, vp, vp]
        L.smart_build_mask.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.smart_verify_accept.argtypes = [vp, vp, i64, vp, vp, vp, vp]
        L.smart_verify_sample.argtypes = [vp, vp, i64, C.c_double, C.c_uint64, vp, vp, vp, vp]
        L.smart_run_step.argtypes = [vp, vp, vp, vp, i64, vp, i64] + [vp] * 8 + [vp]
        L.smart_get_stats.argtypes = [vp, C.POINTER(_Stats)]
        L.smart_get_tree.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.smart_get_candidates.argtypes = [vp, i32, i64, vp, vp, vp, vp]
        L.smart_last_error.argtypes = [vp]
        L.smart_last_error.restype = C.c_char_p
        L.smart_status_string.argtypes = [st]
        L.smart_status_string.restype = C.c_char_p
        for n in EXPORTED:
            if n not in ("smart_last_error", "smart_status_string"):
                getattr(L, n).restype = st
        _lib = L
    return _lib


def _check(status: int, ctx=None):
    if status != OK:
        msg = lib().smart_last_error(ctx).decode()
        raise SmartError(status, msg)


def _ptr(t):
    """device pointer of a torch tensor (or None)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


@dataclass
class Cost:
    """Eq.(4) lambda, beta; Eq.(5) gamma, delta, rho, eta; Eq.(1) c_T (milliseconds)."""
    lam: float
    beta: float = 0.0
    gamma: float = 0.0
    delta: float = 0.0
    rho: float = 1.0
    eta: float = 0.0
    c_T: float = 1.0

    def c(self):
        return _Cost(self.lam, self.beta, self.gamma, self.delta, self.rho, self.eta, self.c_T)


@dataclass
class Config:
    vocab: int
    top_k: int
    max_depth: int
    max_frontier: int = 0
    batch_local: int = 1
    batch_global: int = 0          # 0 -> batch_local
    batch_offset: int = 0
    budget_verify: int = 200
    alpha: float = 0.8
    bonus: int = 1
    selection: int = PREFIX
    accept_model: int = NODE_SUM
    marginal: int = DERIVATIVE
    cost_scope: int = COST_GLOBAL
    logits_dtype: int = BF16
    row_mode: int = ROWS_NODE
    tree_capacity: int = 0

    def c(self):
        return _Config(self.vocab, self.top_k, self.max_depth, self.max_frontier, self.batch_local,
                       self.batch_global or self.batch_local, self.batch_offset, self.budget_verify,
                       self.alpha, self.bonus, self.selection, self.accept_model, self.marginal,
                       self.cost_scope, self.logits_dtype, self.row_mode, self.tree_capacity)


def query_sizes(cfg: Config) -> dict:
    s = _Sizes()
    c = cfg.c()
    _check(lib().smart_query_sizes(C.byref(c), C.byref(s)))
    return dict(B=s.B, T=s.T, mask_words=s.mask_words, frontier_cap=s.frontier_cap,
                chunk_elems=s.chunk_elems)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().smart_nccl_unique_id(buf))
    return buf.raw


class Smart:
    """One SMART controller context (one CUDA device, one stream at a time)."""

    def __init__(self, cfg: Config, cost: Cost, device: int = 0):
        self.cfg, self.cost, self.device = cfg, cost, device
        self.sizes = query_sizes(cfg)
        self._h = C.c_void_p()
        c, k = cfg.c(), cost.c()
        _check(lib().smart_create(C.byref(c), C.byref(k), device, C.byref(self._h)))

    def attach_nccl(self, uid: bytes, rank: int, nranks: int):
        _check(lib().smart_attach_nccl(self._h, uid, rank, nranks), self._h)

    def exchange_record_bytes(self, nranks: int) -> int:
        n = C.c_int64()
        c = self.cfg.c()
        _check(lib().smart_exchange_record_bytes(C.byref(c), nranks, C.byref(n)))
        return n.value

    def attach_exchange(self, rank: int, nranks: int, send, recv):
        """caller-provided all-gather: send/recv are uint8 device tensors of record_bytes and
        nranks*record_bytes (see smart_attach_exchange in include/smart.h)"""
        self._xbufs = (send, recv)  # keep alive
        _check(lib().smart_attach_exchange(self._h, rank, nranks, _ptr(send), _ptr(recv)), self._h)

    def peer_exchange_bytes(self, nranks: int) -> int:
        n = C.c_int64()
        c = self.cfg.c()
        _check(lib().smart_peer_exchange_bytes(C.byref(c), nranks, C.byref(n)))
        return n.value

    def attach_peer_exchange(self, rank: int, nranks: int, recv_ptrs, keep=None):
        """peer exchange (smart_attach_peer_exchange): recv_ptrs[g] = rank g's receive buffer (an int
        device address valid in this process); `keep` holds the owning tensors alive"""
        self._xbufs = keep
        arr = (C.c_void_p * nranks)(*[C.c_void_p(int(p)) for p in recv_ptrs])
        _check(lib().smart_attach_peer_exchange(self._h, rank, nranks, arr), self._h)

    def select_finish(self, layer: int, frontier=None, frontier_count=None, stream=None):
        _check(lib().smart_select_finish(self._h, layer, _ptr(frontier), _ptr(frontier_count), _stream(stream)),
               self._h)

    def close(self):
        if self._h:
            lib().smart_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the hot path -------------------------------------------------------------------
    def begin_step(self, root_tok=None, root_pos=None, stream=None):
        _check(lib().smart_begin_step(self._h, _ptr(root_tok), _ptr(root_pos), _stream(stream)), self._h)

    def expand_step(self, layer: int, logits, stream=None):
        ld = logits.stride(-2) if logits.dim() >= 2 else logits.shape[-1]
        _check(lib().smart_expand_step(self._h, layer, _ptr(logits), ld, _stream(stream)), self._h)

    def select(self, layer: int, frontier=None, frontier_count=None, stream=None):
        _check(lib().smart_select(self._h, layer, _ptr(frontier), _ptr(frontier_count), _stream(stream)),
               self._h)

    def build_mask(self, mask=None, pos=None, parent=None, tok=None, tree_len=None, stream=None):
        _check(lib().smart_build_mask(self._h, _ptr(mask), _ptr(pos), _ptr(parent), _ptr(tok),
                                      _ptr(tree_len), _stream(stream)), self._h)

    def verify_accept(self, target, accept_len=None, accept_path=None, bonus=None, stream=None):
        ld = target.stride(-2)
        _check(lib().smart_verify_accept(self._h, _ptr(target), ld, _ptr(accept_len), _ptr(accept_path),
                                         _ptr(bonus), _stream(stream)), self._h)

    def verify_sample(self, target, temperature, seed, accept_len=None, accept_path=None, bonus=None,
                      stream=None):
        """A8 at temperature > 0 (NEXT #1): one Gumbel-max target sample per visited node."""
        ld = target.stride(-2)
        _check(lib().smart_verify_sample(self._h, _ptr(target), ld, float(temperature),
                                         int(seed) & ((1 << 64) - 1), _ptr(accept_len), _ptr(accept_path),
                                         _ptr(bonus), _stream(stream)), self._h)

    def run_step(self, draft, target, out: dict, root_tok=None, root_pos=None, stream=None):
        """begin + d x (expand, select) + mask + verify on ROWS_NODE pools (graph-capturable)."""
        _check(lib().smart_run_step(
            self._h, _ptr(root_tok), _ptr(root_pos), _ptr(draft), draft.stride(-2),
            _ptr(target), target.stride(-2) if target is not None else 0,
            _ptr(out.get("mask")), _ptr(out.get("pos")), _ptr(out.get("parent")), _ptr(out.get("tok")),
            _ptr(out.get("tree_len")), _ptr(out.get("accept_len")), _ptr(out.get("accept_path")),
            _ptr(out.get("bonus")), _stream(stream)), self._h)

    def alloc_outputs(self):
        """device output tensors sized for this context (torch, on self.device)."""
        import torch
        b, T, MW = self.cfg.batch_local, self.sizes["T"], self.sizes["mask_words"]
        D = max(self.cfg.max_depth, 1)
        dev = torch.device("cuda", self.device)
        i32 = torch.int32
        return dict(mask=torch.zeros((b, T, MW), dtype=i32, device=dev),
                    pos=torch.zeros((b, T), dtype=i32, device=dev),
                    parent=torch.zeros((b, T), dtype=i32, device=dev),
                    tok=torch.zeros((b, T), dtype=i32, device=dev),
                    tree_len=torch.zeros((b,), dtype=i32, device=dev),
                    accept_len=torch.zeros((b,), dtype=i32, device=dev),
                    accept_path=torch.zeros((b, D), dtype=i32, device=dev),
                    bonus=torch.zeros((b,), dtype=i32, device=dev))

    # ---- inspection (synchronising) ----------------------------------------------------------
    def stats(self, raise_on_device_flag: bool = False) -> dict:
        s = _Stats()
        rc = lib().smart_get_stats(self._h, C.byref(s))
        if rc != OK and (rc != EDEVICE or raise_on_device_flag):
            _check(rc, self._h)
        layers = []
        for l in range(MAX_DEPTH):
            t = s.layer[l]
            layers.append({f: getattr(t, f) for f, _ in _LayerTrace._fields_})
        return dict(layers_executed=s.layers_executed, error_flags=s.error_flags,
                    nodes_local=s.nodes_local, accepted_local=s.accepted_local,
                    accepted_global=s.accepted_global, nodes_global=s.nodes_global,
                    step_kernel_grid=s.step_kernel_grid,
                    E_global=s.E_global, S_final=s.S_final, layers=layers)

    def tree(self) -> dict:
        import numpy as np
        b, T = self.cfg.batch_local, self.sizes["T"]
        out = dict(n_nodes=np.zeros(b, np.int32), tok=np.zeros((b, T), np.int32),
                   parent=np.zeros((b, T), np.int32), depth=np.zeros((b, T), np.int32),
                   p=np.zeros((b, T), np.float32), cum=np.zeros((b, T), np.float32))
        P = lambda a: a.ctypes.data_as(C.c_void_p)
        _check(lib().smart_get_tree(self._h, P(out["n_nodes"]), P(out["tok"]), P(out["parent"]),
                                    P(out["depth"]), P(out["p"]), P(out["cum"])), self._h)
        return out

    def candidates(self, layer: int) -> dict:
        import numpy as np
        cap = self.sizes["frontier_cap"] * self.cfg.top_k
        cnt = C.c_int32()
        ints = np.zeros((cap, 4), np.int32)
        fl = np.zeros((cap, 3), np.float32)
        adm = np.zeros(cap, np.int32)
        P = lambda a: a.ctypes.data_as(C.c_void_p)
        _check(lib().smart_get_candidates(self._h, layer, cap, C.byref(cnt), P(ints), P(fl), P(adm)),
               self._h)
        n = cnt.value
        return dict(r=ints[:n, 0], parent=ints[:n, 1], tok=ints[:n, 2], c=ints[:n, 3],
                    p=fl[:n, 0], cum=fl[:n, 1], b=fl[:n, 2], admitted=adm[:n].astype(bool))


def ipc_handle(dev_ptr: int) -> bytes:
    """64-byte CUDA IPC handle of a device allocation (smart_ipc_get_handle)."""
    buf = C.create_string_buffer(64)
    _check(lib().smart_ipc_get_handle(C.c_void_p(int(dev_ptr)), buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    """Map another process's allocation into this one (smart_ipc_open_handle); returns the address."""
    p = C.c_void_p()
    _check(lib().smart_ipc_open_handle(C.c_char_p(bytes(handle)), C.byref(p)))
    return p.value


def ipc_close(dev_ptr: int) -> None:
    _check(lib().smart_ipc_close(C.c_void_p(int(dev_ptr))))
