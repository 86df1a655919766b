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
    outs = [q.get(timeout=240) for _ in procs]
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
def test_shard_plan_balances_modelled_cost(world):
    """irka.cu's owner map: longest-first on the least-loaded rank (LPT, within 4/3 of optimal)."""
    from paper_2003_12759_b200.dist import shard_cost, shard_plan
    rng = np.random.default_rng(world)
    widths = rng.choice([1, 2], size=12)
    its = rng.integers(40, 400, size=12)
    cost = np.array([shard_cost(w, k) for w, k in zip(widths, its)])
    owner = shard_plan(cost, world)
    assert owner.min() >= 0 and owner.max() < world
    load = np.bincount(owner, weights=cost, minlength=world)
    assert load.max() <= max(cost.max(), 4.0 / 3.0 * cost.sum() / world) + 1e-9 * cost.sum()
    assert np.array_equal(owner, shard_plan(cost, world))  # deterministic: every rank computes the same map
    # first sweep: unknown iterations, a pair costs twice a real unit
    assert shard_cost(2, -1) == 2 * shard_cost(1, -1)


def test_shard_plan_keeps_pinned_units():
    from paper_2003_12759_b200.dist import shard_plan
    cost = np.array([5.0, 4.0, 3.0, 3.0, 2.0, 2.0])
    fixed = np.array([1, -1, -1, 1, -1, -1])
    owner = shard_plan(cost, 2, fixed)
    assert owner[0] == 1 and owner[3] == 1
    assert list(owner) == [1, 0, 0, 1, 0, 1]


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


@pytest.mark.gpu
def test_native_nccl_allgather_single_rank(mpg):
    """libmpg.so's own NCCL communicator (world = 1 on the one GPU here):
    mpg_comm_allgather moves device bytes on the library stream."""
    import ctypes as C
    from paper_2003_12759_b200 import _lib as L
    from paper_2003_12759_b200 import dist as mdist
    v = C.c_int()
    L.check(L.lib.mpg_nccl_version(C.byref(v)))
    assert v.value >= 22000
    comm = mdist.NcclComm(0)
    try:
        import torch
        send = torch.arange(1000, dtype=torch.float64, device="cuda:0")
        recv = torch.zeros(1000, dtype=torch.float64, device="cuda:0")
        torch.cuda.synchronize()
        assert comm.c_function(comm.ctx, send.data_ptr(), recv.data_ptr(), 8000) == 0
        L.check(L.lib.mpg_synchronize(0))
        assert torch.equal(send, recv)
        assert comm.stats() == {"calls": 1, "bytes": 8000.0}
    finally:
        comm.close()


@pytest.mark.gpu
def test_sharded_irka_through_native_nccl_matches_single(mpg, gen):
    from paper_2003_12759_b200 import dist as mdist
    s = gen.config1(40)
    dev = lambda h: mpg.SparseMatrix.from_csr(h.nrows, h.ncols, h.rowptr, h.colind, h.val)
    op = mpg.ShiftedOperator(dev(s.a), dev(s.e_csr()))
    cfg = mpg.IrkaConfig(r=s.r, tol=1e-8, max_sweeps=100, seed=1, gmres=mpg.GmresConfig(1e-10, 1000))
    comm = mdist.NcclComm(0)
    st, rep = mdist.irka_reduce_sharded(op, s.b, s.c, cfg, mpg.PrecondMode.REUSE_FROZEN, init_shifts=s.shifts,
                                        gather=comm)
    st1, rep1 = mpg.irka_reduce(op, s.b, s.c, cfg, mpg.PrecondMode.REUSE_FROZEN, init_shifts=s.shifts)
    comm.close()
    assert rep.converged and rep1.converged and rep.sweeps == rep1.sweeps
    assert np.array_equal(np.sort_complex(st.lam), np.sort_complex(st1.lam))
