"""Sharded apply across GPUs — one process per GPU, the middle factor as one
all-to-all (the reference is single-process).

The V^L/H side of the chain is block-diagonal per middle column node j and the
G/U^L side per middle row node i; in the reference layout every level's
leading block index carries that node in its high bits, so a node's data is a
contiguous slice. Part d of P owns nodes [d m/P, (d+1) m/P) on both sides:

    down   V*, H^{L-1}* .. H^{h}*  on input rows  [d n/P, (d+1) n/P)   (local)
    M      pack (W scaling fused) -> all-to-all (NCCL over NVLink) -> unpack
    up     G^{h} .. G^{L-1}, U     on output rows [d n/P, (d+1) n/P)   (local)

``ShardedApply`` holds the exchange orchestration; ``ShardedPlan`` binds its four
local steps to libbfly.so (``bf_apply_down``, ``bf_middle_pack``,
``bf_middle_unpack``, ``bf_apply_up``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .factors import ButterflyFactors
from .partition import DyadicPartition, level_geometry


def shard_slices(f: ButterflyFactors, part: int, nparts: int) -> dict:
    """This part's slices of every factor (leading-index ranges), full weights."""
    p = f.partition
    if p.mid_nodes % nparts:
        raise ValueError(f"{nparts} parts do not divide the {p.mid_nodes} middle nodes")

    def cut(a):
        n0 = a.shape[0]
        return a[part * n0 // nparts:(part + 1) * n0 // nparts]

    return {"u_leaf": cut(f.u_outer.blocks), "v_leaf": cut(f.v_outer.blocks), "weights": f.middle.weights,
            "g": [(t.level, cut(t.blocks)) for t in f.g_chain], "h": [(t.level, cut(t.blocks)) for t in f.h_chain]}



# Symmetric-memory barriers of the fused push exchange trap after this long instead of
# spinning forever when a peer never arrives (a hung multi-GPU job is worse than a failed one).
PUSH_BARRIER_TIMEOUT_MS = 120_000

class ShardedApply:
    """Exchange orchestration of the sharded chain; subclasses provide the local steps."""

    def __init__(self, p: DyadicPartition, r: int, part: int, nparts: int, group=None):
        if p.mid_nodes % nparts:
            raise ValueError(f"{nparts} parts do not divide the {p.mid_nodes} middle nodes")
        self.p, self.r, self.part, self.nparts, self.group = p, r, part, nparts, group
        self.mp = p.mid_nodes // nparts
        self.n_local = p.n // nparts
        self.mid_rows = self.mp * p.mid_nodes * r          # rows of this part's middle slice
        self.chunk_rows = self.mp * self.mp * r            # rows sent to each part
        self.last_exchange_ms = None

    # local steps -------------------------------------------------------------
    def down(self, x, adjoint):
        raise NotImplementedError

    def pack(self, mid, adjoint):
        raise NotImplementedError

    def unpack(self, recv, adjoint):
        raise NotImplementedError

    def up(self, mid, adjoint):
        raise NotImplementedError

    def exchange(self, send):
        """All-to-all of equal chunks (one per part)."""
        import torch
        import torch.distributed as dist
        recv = torch.empty_like(send)
        if self.nparts == 1:
            recv.copy_(send)
            return recv
        sr = torch.view_as_real(send) if send.is_complex() else send
        rr = torch.view_as_real(recv) if recv.is_complex() else recv
        dist.all_to_all_single(rr, sr, group=self.group)
        return recv

    def apply(self, g_local, adjoint: bool = False):
        """This part's rows of K g (K* g when adjoint), given its rows of g."""
        if g_local.shape[0] != self.n_local:
            raise ValueError(f"local input length {g_local.shape[0]} != {self.n_local}")
        mid = self.down(g_local, adjoint)
        recv = self.exchange(self.pack(mid, adjoint))
        return self.up(self.unpack(recv, adjoint), adjoint)


class ShardedPlan(ShardedApply):
    """A part's device plan: libbfly.so for the local steps, NCCL for the exchange."""

    def __init__(self, p: DyadicPartition, r: int, part: int, nparts: int, slices: dict, dtype: str = "c128",
                 device=None, group=None):
        super().__init__(p, r, part, nparts, group)
        torch = _lib.require_cuda()
        self.lib = _lib.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.tdt = torch.complex128 if dtype == "c128" else torch.complex64
        h = ctypes.c_void_p()
        _lib.check(self.lib.bf_plan_create_tree(ctypes.byref(h), p.n, p.levels, r, getattr(p, "branching", 2),
                                                _lib.BF_C128 if dtype == "c128" else _lib.BF_C64, self.device,
                                                part, nparts), "bf_plan_create_tree")
        self._h = h
        shapes, leaf_shape = level_geometry(p, r)
        keep = []

        def ptr(a, want_shape, real=False):
            if hasattr(a, "data_ptr"):
                t = a.detach().to(dtype=torch.float64 if real else torch.complex128).contiguous()
            else:
                t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64 if real else np.complex128))
            if want_shape is not None and tuple(t.shape) != tuple(want_shape):
                raise ValueError(f"slice shape {tuple(t.shape)} != {tuple(want_shape)}")
            keep.append(t)
            return t.data_ptr()

        local = lambda s: (s[0] // nparts,) + tuple(s[1:])  # noqa: E731
        g_ptrs = (ctypes.c_void_p * len(shapes))(*[ptr(b, local(s)) for (_, b), (_, _, s) in zip(slices["g"], shapes)])
        h_ptrs = (ctypes.c_void_p * len(shapes))(*[ptr(b, local(s)) for (_, b), (_, _, s) in zip(slices["h"], shapes)])
        _lib.check(self.lib.bf_plan_upload(h, ptr(slices["u_leaf"], local(leaf_shape)), g_ptrs,
                                           ptr(slices["weights"], (p.mid_nodes, p.mid_nodes, r), real=True), h_ptrs,
                                           ptr(slices["v_leaf"], local(leaf_shape))), "bf_plan_upload")
        del keep

    @classmethod
    def from_factors(cls, f: ButterflyFactors, part: int, nparts: int, **kw):
        return cls(f.partition, f.rank, part, nparts, shard_slices(f, part, nparts), **kw)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self.lib.bf_plan_destroy(h)
            self._h = None

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _ws(self, k):
        import torch
        wsb = int(self.lib.bf_apply_workspace_bytes(self._h, k))
        return torch.empty(wsb, dtype=torch.uint8, device=f"cuda:{self.device}"), wsb

    def down(self, x, adjoint):
        import torch
        x = x.reshape(self.n_local, -1).to(self.tdt).contiguous()
        k = x.shape[1]
        mid = torch.empty((self.mid_rows, k), dtype=self.tdt, device=x.device)
        ws, wsb = self._ws(k)
        _lib.check(self.lib.bf_apply_down(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(mid.data_ptr()), k,
                                          int(adjoint), ctypes.c_void_p(ws.data_ptr()), wsb, self._stream()))
        return mid

    def pack(self, mid, adjoint):
        import torch
        k = mid.shape[1]
        send = torch.empty((self.nparts * self.chunk_rows, k), dtype=self.tdt, device=mid.device)
        _lib.check(self.lib.bf_middle_pack(self._h, ctypes.c_void_p(mid.data_ptr()), ctypes.c_void_p(send.data_ptr()),
                                           k, int(adjoint), self._stream()))
        return send

    def unpack(self, recv, adjoint):
        import torch
        k = recv.shape[1]
        mid = torch.empty((self.mid_rows, k), dtype=self.tdt, device=recv.device)
        _lib.check(self.lib.bf_middle_unpack(self._h, ctypes.c_void_p(recv.data_ptr()),
                                             ctypes.c_void_p(mid.data_ptr()), k, int(adjoint), self._stream()))
        return mid

    def up(self, mid, adjoint):
        import torch
        k = mid.shape[1]
        out = torch.empty((self.n_local, k), dtype=self.tdt, device=mid.device)
        ws, wsb = self._ws(k)
        _lib.check(self.lib.bf_apply_up(self._h, ctypes.c_void_p(mid.data_ptr()), ctypes.c_void_p(out.data_ptr()), k,
                                        int(adjoint), ctypes.c_void_p(ws.data_ptr()), wsb, self._stream()))
        return out

    # -- fused down + exchange step (peer stores over NVLink) --

    def down_push(self, x, adjoint, peers):
        """Down half whose last level stores (weights applied) straight into every part's
        receive buffer: peers[d] = device address of part d's receive buffer."""
        import torch
        x = x.reshape(self.n_local, -1).to(self.tdt).contiguous()
        k = x.shape[1]
        ws, wsb = self._ws(k)
        arr = (ctypes.c_void_p * self.nparts)(*[int(p_) for p_ in peers])
        _lib.check(self.lib.bf_apply_down_push(self._h, ctypes.c_void_p(x.data_ptr()), arr, k, int(adjoint),
                                               ctypes.c_void_p(ws.data_ptr()), wsb, self._stream()),
                   "bf_apply_down_push")
        del torch

    def push_buffer(self, k):
        """Symmetric receive buffer (nparts * chunk_rows, k) shared over NVLink, cached per k."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        cache = self.__dict__.setdefault("_push_cache", {})
        if k not in cache:
            rows = self.nparts * self.chunk_rows
            width = 2 if self.tdt == torch.complex128 else 1  # complex128 as pairs of float64
            buf = symm.empty((rows * k * width,), dtype=torch.float64 if width == 2 else torch.complex64,
                             device=f"cuda:{self.device}")
            group = self.group if self.group is not None else dist.group.WORLD
            hdl = symm.rendezvous(buf, group)
            cache[k] = (buf, hdl, list(hdl.buffer_ptrs))
        return cache[k]

    def apply_push(self, g_local, adjoint: bool = False):
        """Sharded apply with the middle exchange fused into the last down level (peer stores)."""
        import torch
        if g_local.shape[0] != self.n_local:
            raise ValueError(f"local input length {g_local.shape[0]} != {self.n_local}")
        k = g_local.reshape(self.n_local, -1).shape[1]
        buf, hdl, ptrs = self.push_buffer(k)
        hdl.barrier(timeout_ms=PUSH_BARRIER_TIMEOUT_MS)  # every part is done reading its buffer (previous apply)
        self.down_push(g_local, adjoint, ptrs)
        hdl.barrier(timeout_ms=PUSH_BARRIER_TIMEOUT_MS)  # every part's stores into this buffer have landed
        recv = buf.view(torch.complex128) if self.tdt == torch.complex128 else buf
        recv = recv.view(self.nparts * self.chunk_rows, k)
        return self.up(self.unpack(recv, adjoint), adjoint)
