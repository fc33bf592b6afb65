"""World-size-2 CPU (gloo) tests of the row-parallel path's host logic:
partition rule, the deterministic rank-ordered Gram exchange (allgather +
fixed-order sum, bitwise identical on every rank), gather_modes, and the
Gram-sum formulation of the parallel update against the reference's TSQR
formulation (dsvd.py:176-242, via the oracle).  The sm_100a kernels are
covered by the -m gpu tests; here the local Grams are formed with numpy."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2108_08845_b200.datagen import partition_bounds
        from paper_2108_08845_b200.dsvd import LocalModes, RankContext, allreduce_ordered, gather_modes

        ctx = RankContext()
        assert (ctx.rank, ctx.world_size) == (rank, world)
        from paper_2108_08845_b200.dsvd import _row_offset
        # global row offset of the randomized exchange (argmax rows are global)
        assert _row_offset(ctx, 100 + rank, "cpu") == (sum(100 + r for r in range(rank)), sum(100 + r for r in range(world)))
        a = oracle.burgers_matrix(2048, 800)
        lo, hi = partition_bounds(a.shape[0], world)[rank]
        k, ff = 10, 0.95
        U = s = None
        for c0 in range(0, 800, 200):
            blk = a[lo:hi, c0:c0 + 200]
            C = blk if U is None else np.concatenate([ff * (U * s), blk], axis=1)
            G_local = torch.from_numpy(C.T @ C)
            G = allreduce_ordered(G_local, ctx)
            parts = [torch.empty_like(G) for _ in range(world)]
            dist.all_gather(parts, G)
            assert all(torch.equal(p_, G) for p_ in parts)  # identical bits on every rank
            lam, V = np.linalg.eigh(G.numpy())
            order = np.argsort(-lam, kind="stable")[:k]
            s = np.sqrt(lam[order])
            U = C @ (V[:, order] / s)
        full = gather_modes(ctx, LocalModes(torch.from_numpy(np.ascontiguousarray(U)), torch.from_numpy(s)))
        if rank == 0:
            ref_m, ref_s = oracle.ref_parallel_stream_all(a, [(c, c + 200) for c in range(0, 800, 200)], world, k, ff)
            q.put((oracle.sigma_rel_err(s, ref_s), float(np.max(oracle.mode_angles(full.numpy(), ref_m))),
                   tuple(full.shape)))
        else:
            assert full is None
        # ranks that disagree on an exchanged shape raise the reference's ProtocolError on every rank
        from paper_2108_08845_b200.errors import ProtocolError
        bad = LocalModes(torch.zeros((4, 3 + rank), dtype=torch.float64), torch.ones(3 + rank, dtype=torch.float64))
        with pytest.raises(ProtocolError):
            gather_modes(ctx, bad)
        with pytest.raises(ProtocolError):
            _row_offset(ctx, 10, "cpu", 5 + rank)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_parallel_stream_gram_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    rel, ang, shape = q.get(timeout=10)
    assert shape == (2048, 10)
    assert rel <= 1e-10
    assert ang <= 1e-8


def test_allreduce_ordered_single_rank_is_identity():
    from paper_2108_08845_b200.dsvd import RankContext, allreduce_ordered
    t = torch.randn(5, 5, dtype=torch.float64)
    ctx = RankContext()
    if ctx.world_size == 1:
        assert allreduce_ordered(t, ctx) is t
