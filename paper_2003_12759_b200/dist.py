"""Multi-GPU plumbing of the sharded IRKA entry point (mpg_irka_reduce_sharded).

One process per GPU. Every rank holds a replica of A and E and solves its share
of the (shift unit, primal/dual side) solves of each sweep (the reference's
birka.cpp:200-260 loop; units are placed longest-first on the least-loaded
rank by the previous sweep's iteration counts, irka.cu); the solved columns
are then all-gathered so that every rank forms the same projection and the
same next shifts. The exchange is the only collective.

Two exchanges:
* NcclComm -- the native one: libmpg.so's own NCCL communicator; the columns
  move device to device on the library stream (ncclAllGather over NVLink),
  torch.distributed only hands the NCCL unique id to the ranks.
* AllGather -- a torch.distributed callback for any backend (gloo between CPU
  processes in the tests): it stages the raw buffers through torch tensors
  with `copy(dst, src, nbytes)` (mpg_copy, a cudaMemcpy with
  cudaMemcpyDefault, by default; ctypes.memmove for host buffers).
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


def shard_cost(width: int, last_iterations: int = -1) -> float:
    """Modelled cost of a unit's solve (irka.cu shard_cost): width * K * (K + 40)."""
    return float(L.lib.mpg_shard_cost(int(width), int(last_iterations)))


def shard_plan(cost, world: int, fixed=None) -> np.ndarray:
    """Owner rank of each unit, as every rank of mpg_irka_reduce_sharded computes it."""
    c = L.f64(cost)
    f = np.ascontiguousarray(fixed if fixed is not None else -np.ones(c.size), dtype=np.int32)
    out = np.zeros(c.size, dtype=np.int32)
    L.check(L.lib.mpg_shard_plan(c.size, L.ptr(c), L.ptr(f), int(world), L.ptr(out)))
    return out


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


class NcclComm:
    """libmpg.so's native NCCL communicator for `device` (mpg_comm_*). With a
    torch.distributed group, rank 0's unique id is broadcast through it;
    without one (world = 1) the communicator is created locally."""

    def __init__(self, device: int = 0, group=None):
        if group is not None or _dist_ready():
            import torch.distributed as dist
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
        idb = (C.c_char * 128)()
        if rank == 0:
            L.check(L.lib.mpg_comm_unique_id(idb, 128))
        if world > 1:
            import torch.distributed as dist
            obj = [bytes(idb)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            idb = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        L.check(L.lib.mpg_comm_create(device, rank, world, idb, C.byref(h)))
        self._h = h
        self.rank, self.world, self.device = rank, world, device
        self.error = None
        self._fn = L.ALLGATHER_FN(C.cast(L.lib.mpg_comm_allgather, C.c_void_p).value)

    @property
    def c_function(self):
        return self._fn

    @property
    def ctx(self):
        return self._h

    def stats(self) -> dict:
        calls, nbytes = C.c_longlong(), C.c_double()
        L.check(L.lib.mpg_comm_stats(self._h, C.byref(calls), C.byref(nbytes)))
        return {"calls": calls.value, "bytes": nbytes.value}

    def close(self) -> None:
        if self._h:
            L.check(L.lib.mpg_comm_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dist_ready() -> bool:
    try:
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized()
    except Exception:
        return False


def irka_reduce_sharded(op: ShiftedOperator, b, c, cfg: IrkaConfig, mode: int = PrecondMode.REUSE_FROZEN,
                        init_shifts=None, group=None, gather=None, device: int = 0):
    """Sharded IRKA (this rank's share of every sweep's solves + all-gather);
    every rank returns the same reduced model and the report rows of its own
    solves. Call from every rank of `group` with identical arguments; `device`
    is the GPU holding `op`. `gather` is an NcclComm (default with the nccl
    backend: the native device-to-device exchange) or an AllGather (default
    otherwise: gloo, staged through host memory by mpg_copy)."""
    if gather is None:
        import torch.distributed as dist
        if dist.get_backend(group) == "nccl":
            gather = NcclComm(device, group)
        else:
            gather = AllGather(group, device="cpu", copy=_mpg_copy)
    if isinstance(gather, NcclComm):
        rank, world = gather.rank, gather.world
    else:
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
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
        gather.c_function, getattr(gather, "ctx", None), L.ptr(kr), L.ptr(fr), L.ptr(cr), L.ptr(lre), L.ptr(lim), C.byref(sweeps),
        C.byref(conv), rows, maxrows, C.byref(nrows))
    if status != L.MPG_OK and gather.error is not None:
        raise RuntimeError(f"all-gather failed: {gather.error}") from gather.error
    L.check(status)
    st = IrkaState(kr, fr, cr, None, None, lre + 1j * lim, None, None, sweeps.value)
    rep = ReductionReport(_rows(rows, min(nrows.value, maxrows)), bool(conv.value), r, sweeps.value)
    return st, rep
