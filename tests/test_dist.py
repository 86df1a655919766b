"""Multi-rank plumbing of the sharded IRKA (paper_2003_12759_b200/dist.py):
world-size-2 gloo process groups on the CPU, and (gpu) two ranks sharing one
GPU whose only meeting point is the host-side all-gather (no kernel waits on
another rank)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _gather_worker(rank, world, port, out):
    dist = _init(rank, world, port)
    from paper_2003_12759_b200 import dist as mdist
    g = mdist.AllGather(device="cpu")
    res = []
    for nbytes in (8 * 1000, 8 * 3 + 5, 8):
        send = np.frombuffer(bytes((rank * 37 + i) % 251 for i in range(nbytes)), dtype=np.uint8).copy()
        recv = np.zeros(nbytes * world, dtype=np.uint8)
        rc = g._callback(None, send.ctypes.data, recv.ctypes.data, nbytes)
        res.append((rc, recv.tobytes()))
    out.put((rank, res, g.calls))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(outs, key=lambda t: t[0])


def test_allgather_callback_concatenates_in_rank_order():
    world = 2
    outs = _spawn(_gather_worker, world)
    for rank, res, calls in outs:
        assert calls == 3
        for (rc, got), nbytes in zip(res, (8 * 1000, 8 * 3 + 5, 8)):
            assert rc == 0
            want = b"".join(bytes((r * 37 + i) % 251 for i in range(nbytes)) for r in range(world))
            assert got == want


def test_allgather_reports_failure_instead_of_raising():
    import torch.distributed as dist
    port = _free_port()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        from paper_2003_12759_b200 import dist as mdist

        def bad_copy(dst, src, n):
            raise OSError("copy failed")
        g = mdist.AllGather(device="cpu", copy=bad_copy)
        buf = np.zeros(4)
        assert g._callback(None, buf.ctypes.data, buf.ctypes.data, 32) == 1
        assert isinstance(g.error, OSError)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_owner_partitions_every_sweep(world):
    from paper_2003_12759_b200.dist import shard_owner
    r = 8
    units = [(side, c) for side in (0, 1) for c in range(r)]
    owners = [shard_owner(s, c, r, world) for s, c in units]
    assert all(0 <= o < world for o in owners)
    counts = np.bincount(owners, minlength=world)
    assert counts.max() - counts.min() <= 1  # round-robin balance over 2 r solves


def _irka_worker(rank, world, port, out):
    dist = _init(rank, world, port)
    import paper_2003_12759_b200 as mpg
    from paper_2003_12759_b200 import gen
    from paper_2003_12759_b200 import dist as mdist
    s = gen.config1(40)
    dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
    op = mpg.ShiftedOperator(dev(s.a), dev(s.e_csr()))
    cfg = mpg.IrkaConfig(r=s.r, tol=1e-8, max_sweeps=100, seed=1, gmres=mpg.GmresConfig(1e-10, 1000))
    st, rep = mdist.irka_reduce_sharded(op, s.b, s.c, cfg, mpg.PrecondMode.REUSE_FROZEN, init_shifts=s.shifts)
    ref = None
    if rank == 0:
        st1, rep1 = mpg.irka_reduce(op, s.b, s.c, cfg, mpg.PrecondMode.REUSE_FROZEN, init_shifts=s.shifts)
        ref = (np.sort_complex(st1.lam), rep1.sweeps)
    out.put((rank, np.sort_complex(st.lam), rep.sweeps, rep.converged, len(rep.rows), ref))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_irka_two_ranks_match_single_rank():
    outs = _spawn(_irka_worker, 2)
    (_, lam0, sw0, conv0, rows0, ref), (_, lam1, sw1, conv1, rows1, _) = outs
    assert conv0 and conv1 and sw0 == sw1
    assert np.array_equal(lam0, lam1)  # every rank forms the same projection
    lam_ref, sw_ref = ref
    assert abs(sw0 - sw_ref) <= max(2, sw_ref // 10)  # the summation order of the shared projection differs
    assert np.max(np.abs(lam0 - lam_ref) / np.abs(lam_ref)) <= 1e-6
    assert rows0 > 0 and rows1 > 0  # both ranks solved a share
