"""Multi-GPU plumbing: the all-gather callback of mpg_irka_reduce_sharded over
torch.distributed, and the sharded IRKA entry point.

One process per GPU. Every rank holds a replica of A and E and solves its share
of the (shift unit, primal/dual side) solves of each sweep (the reference's
birka.cpp:200-260 loop, split round-robin by (side * r + column) % world); the
solved columns are then all-gathered so that every rank forms the same
projection and the same next shifts. The exchange is the only collective: NCCL
over NVLink between GPUs, gloo between CPU processes (tests).

The callback receives raw buffer addresses of this rank's device. It stages
them through torch tensors with `copy(dst, src, nbytes)` (mpg_copy, a
cudaMemcpy with cudaMemcpyDefault, by default; ctypes.memmove for host
buffers) and calls all_gather_into_tensor.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from . import _lib as L
from .morprec import IrkaConfig, IrkaState, PrecondMode, ReductionReport, ShiftedOperator, _rows

CopyFn = Callable[[int, int, int], None]


def _mpg_copy(dst: int, src: int, nbytes: int) -> None:
    L.check(L.lib.mpg_copy(C.c_void_p(dst), C.c_void_p(src), C.c_int64(nbytes)))


def host_copy(dst: int, src: int, nbytes: int) -> None:
    C.memmove(dst, src, nbytes)


def shard_owner(side: int, column: int, r: int, world: int) -> int:
    """Rank that solves the unit starting at `column` on `side` (0 primal,
    1 dual) -- the assignment irka.cu uses for world > 1."""
    return (side * r + column) % world


class AllGather:
    """Callable usable as mpg_allgather_fn: concatenates `bytes_per_rank` bytes
    from every rank, in rank order, into `recv`.

    `device` is the torch device of the staging tensors ("cuda:k" with NCCL,
    "cpu" with gloo); `copy` moves bytes between the raw buffers and them."""

    def __init__(self, group=None, device: str = "cpu", copy: Optional[CopyFn] = None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.group = group
        self.device = torch.device(device)
        self.copy = copy or (_mpg_copy if self.device.type == "cuda" else host_copy)
        self.world = dist.get_world_size(group)
        self.calls = 0
        self.error: Optional[BaseException] = None
        self._fn = L.ALLGATHER_FN(self._callback)

    def __call__(self, send: int, recv: int, nbytes: int) -> None:
        torch = self.torch
        nwords = (int(nbytes) + 7) // 8
        src = torch.empty(nwords, dtype=torch.float64, device=self.device)
        dst = torch.empty(nwords * self.world, dtype=torch.float64, device=self.device)
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        self.copy(src.data_ptr(), int(send), int(nbytes))
        self.dist.all_gather_into_tensor(dst, src, group=self.group)
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        if nwords * 8 == int(nbytes):
            self.copy(int(recv), dst.data_ptr(), int(nbytes) * self.world)
        else:
            for k in range(self.world):
                self.copy(int(recv) + k * int(nbytes), dst.data_ptr() + k * nwords * 8, int(nbytes))
        self.calls += 1

    def _callback(self, ctx, send, recv, nbytes) -> int:
        try:
            self(send or 0, recv or 0, nbytes)
            return 0
        except BaseException as e:  # reported as MPG_ERR_CUDA by the library
            self.error = e
            return 1

    @property
    def c_function(self):
        return self._fn


def irka_reduce_sharded(op: ShiftedOperator, b, c, cfg: IrkaConfig, mode: int = PrecondMode.REUSE_FROZEN,
                        init_shifts=None, group=None, gather: Optional[AllGather] = None, device: int = 0):
    """Sharded IRKA (this rank's share of every sweep's solves + all-gather);
    every rank returns the same reduced model and the report rows of its own
    solves. Call from every rank of `group` with identical arguments; `device`
    is the GPU holding `op`. With gloo the exchange is staged through host
    memory (mpg_copy moves the device columns), with NCCL through the GPU."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if gather is None:
        if dist.get_backend(group) == "nccl":
            gather = AllGather(group, device=f"cuda:{device}")
        else:
            gather = AllGather(group, device="cpu", copy=_mpg_copy)
    n = op.n
    bm = np.asfortranarray(np.asarray(b, dtype=np.float64).reshape(n, -1))
    cm = np.asfortranarray(np.asarray(c, dtype=np.float64).reshape(n, -1))
    m, q, r = bm.shape[1], cm.shape[1], cfg.r
    kr = np.zeros((r, r), order="F")
    fr, cr = np.zeros((r, m), order="F"), np.zeros((r, q), order="F")
    lre, lim = np.zeros(r), np.zeros(r)
    sweeps, conv, nrows = C.c_int(), C.c_int(), C.c_int()
    maxrows = 2 * r * max(cfg.max_sweeps, 1) + 8
    rows = (L.ReportRow * maxrows)()
    ini = L.f64(init_shifts) if init_shifts is not None else None
    cc = cfg.c()
    status = L.lib.mpg_irka_reduce_sharded(
        op._h, L.ptr(bm), m, L.ptr(cm), q, C.byref(cc), mode, L.ptr(ini) if ini is not None else None, rank, world,
        gather.c_function, None, L.ptr(kr), L.ptr(fr), L.ptr(cr), L.ptr(lre), L.ptr(lim), C.byref(sweeps),
        C.byref(conv), rows, maxrows, C.byref(nrows))
    if status != L.MPG_OK and gather.error is not None:
        raise RuntimeError(f"all-gather failed: {gather.error}") from gather.error
    L.check(status)
    st = IrkaState(kr, fr, cr, None, None, lre + 1j * lim, None, None, sweeps.value)
    rep = ReductionReport(_rows(rows, min(nrows.value, maxrows)), bool(conv.value), r, sweeps.value)
    return st, rep
