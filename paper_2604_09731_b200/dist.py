"""Sharded SMART step across ranks (one process per GPU, torch.distributed for the plumbing).

Requests are sharded by contiguous equal ranges: rank g owns global requests
[g*b_loc, (g+1)*b_loc).  The per-request budget B = floor(B_verify / b_global) and the batch-
coupled cost model (Q13) make the selection global, so each layer has ONE exchange: every rank
packs its locally ranked eligible candidates + per-request header (n_r, E_r) into a fixed-size
record (smart_select), the records are all-gathered in rank order, and every rank runs the
same merge + rule on the gathered list and commits its own requests (smart_select_finish).

The all-gather is torch.distributed.all_gather_into_tensor on the process group (NCCL on
NVLink/NVSwitch for GPUs; gloo works for the host-side tests).  Everything else runs in the
CUDA kernels behind the C-ABI.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    b_loc: int
    b_glob: int
    offset: int


def shard(b_glob: int, world: int, rank: int) -> Shard:
    """Equal contiguous request ranges (the library requires offset = rank * b_loc)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if b_glob % world:
        raise ValueError(f"global batch {b_glob} not divisible by world size {world}")
    b_loc = b_glob // world
    return Shard(rank, world, b_loc, b_glob, rank * b_loc)


def exchange(send, recv, group=None):
    """All-gather of the per-rank exchange records, rank order (recv = cat(send_0..send_{G-1}))."""
    import torch.distributed as dist
    dist.all_gather_into_tensor(recv, send, group=group)


def broadcast_bytes(payload: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string (e.g. an NCCL unique id) from `src`."""
    import torch.distributed as dist
    obj = [payload]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def attach_peer_exchange(ctx, group=None):
    """The peer exchange (smart_attach_peer_exchange) across the processes of
    `group`, one per GPU: each rank allocates its receive buffer, the 64-byte CUDA IPC handles are
    all-gathered through torch.distributed, every rank maps the others' buffers (peer access over
    NVLink) and attaches the table.  Returns the list of mapped addresses (close with
    smart.ipc_close) and the owned buffer (keep it alive)."""
    import torch
    import torch.distributed as dist
    from . import smart as S
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    buf = torch.zeros(ctx.peer_exchange_bytes(world), dtype=torch.uint8, device="cuda")
    handles = [None] * world
    dist.all_gather_object(handles, S.ipc_handle(buf.data_ptr()), group=group)
    ptrs = [buf.data_ptr() if g == rank else S.ipc_open(handles[g]) for g in range(world)]
    ctx.attach_peer_exchange(rank, world, ptrs, keep=buf)
    dist.barrier(group)  # every buffer zeroed and mapped before the first push
    return ptrs, buf


class ShardedSmart:
    """One rank's share of a sharded decode step (caller-provided all-gather mode)."""

    def __init__(self, cfg_kwargs: dict, cost, sh: Shard, device: int, group=None):
        import torch

        from . import smart as S
        self.sh, self.group = sh, group
        cfg = S.Config(batch_local=sh.b_loc, batch_global=sh.b_glob, batch_offset=sh.offset, **cfg_kwargs)
        self.ctx = S.Smart(cfg, cost, device)
        nbytes = self.ctx.exchange_record_bytes(sh.world)
        dev = torch.device("cuda", device)
        self.send = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        self.recv = torch.zeros(sh.world * nbytes, dtype=torch.uint8, device=dev)
        self.ctx.attach_exchange(sh.rank, sh.world, self.send, self.recv)
        self.depth = cfg.max_depth

    def step(self, draft, target, out: dict, root_tok=None, root_pos=None, stream=None):
        """begin + d x (expand, select, all-gather, select_finish) + mask + verify."""
        import torch
        ctx = self.ctx
        s = stream or torch.cuda.current_stream()
        with torch.cuda.stream(s):
            ctx.begin_step(root_tok, root_pos, stream=s)
            for layer in range(1, self.depth + 1):
                ctx.expand_step(layer, draft, stream=s)
                ctx.select(layer, stream=s)
                exchange(self.send, self.recv, self.group)
                ctx.select_finish(layer, stream=s)
            ctx.build_mask(out["mask"], out["pos"], out["parent"], out["tok"], out["tree_len"], stream=s)
            if target is not None:
                ctx.verify_accept(target, out["accept_len"], out["accept_path"], out["bonus"], stream=s)
