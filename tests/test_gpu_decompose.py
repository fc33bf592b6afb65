"""`parsvd decompose` on the device (cli.py:248-359): the four modes read a
PARSVD01 file, run the per-rank body of cli.py:_rank_work on the library, and write the reference's
five output files; the values and modes in them match the oracle on the same bytes."""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _p():
    import paper_2108_08845_b200 as p
    return p


@pytest.mark.parametrize("mode", ["serial-stream", "parallel-stream", "serial-batch", "parallel-batch"])
def test_decompose_outputs_match_oracle(tmp_path, mode):
    p = _p()
    a = oracle.burgers_matrix(4096, 800)
    path = str(tmp_path / "burgers.parsvd")
    p.write_matrix(path, a)
    out = str(tmp_path / mode)
    p.decompose(path, out, mode=mode, k=10, ff=0.95, batch=200, r1=40, r2=30)
    for f in ("singular_values.csv", "modes.csv", "modes.svg", "summary.txt"):
        assert os.path.exists(os.path.join(out, f)), f
    s = p.read_singular_values_csv(os.path.join(out, "singular_values.csv"))
    _, m = p.read_modes_csv(os.path.join(out, "modes.csv"))
    if mode in ("serial-stream", "parallel-stream"):
        rm, rs, rh = oracle.ref_stream_all([a[:, c:c + 200] for c in range(0, 800, 200)], 10, 0.95)
        hist = np.loadtxt(os.path.join(out, "singular_value_history.csv"), delimiter=",", skiprows=1)[:, 1:]
        assert hist.shape == (4, 10)
        for h, r in zip(hist, rh):
            assert oracle.sigma_rel_err(h, r) <= 1e-10
    elif mode == "serial-batch":
        ru, rsf, _ = oracle.ref_svd(a, want_vt=False)
        rm, rs = ru[:, :10], rsf[:10]
    else:
        rm, rs = oracle.ref_apmos([a], 40, 30, 10)
    assert oracle.sigma_rel_err(s, rs) <= 1e-10
    assert np.max(oracle.mode_angles(m, rm)) <= 1e-8
    assert np.all(np.sum(m * rm, axis=0) > 0)
    summary = open(os.path.join(out, "summary.txt")).read()
    assert f"mode={mode}" in summary and "rows=4096" in summary and "cols=800" in summary


def _decompose_rank_worker(rank, world, port, path, outdir, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        p.decompose(path, outdir, mode="parallel-stream", k=10, ff=0.95, batch=200)
        q.put((rank, "ok"))
    except Exception as e:
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_decompose_parallel_stream_two_ranks(tmp_path):
    """cli.py:_rank_work under two processes sharing this GPU (gloo): each rank reads its row block of
    the PARSVD01 file, the modes are gathered at the root, and rank 0 writes the outputs; they match
    the reference's serial stream on the whole matrix."""
    import socket
    import torch.multiprocessing as mp
    p = _p()
    a = oracle.burgers_matrix(4097, 800)
    path = str(tmp_path / "burgers.parsvd")
    p.write_matrix(path, a)
    out = str(tmp_path / "par2")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_decompose_rank_worker, args=(r, 2, port, path, out, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
    assert res == {0: "ok", 1: "ok"}, res
    s_ = p.read_singular_values_csv(os.path.join(out, "singular_values.csv"))
    _, m = p.read_modes_csv(os.path.join(out, "modes.csv"))
    rm, rs, _ = oracle.ref_stream_all([a[:, c:c + 200] for c in range(0, 800, 200)], 10, 0.95)
    assert m.shape == (4097, 10)
    assert oracle.sigma_rel_err(s_, rs) <= 1e-10
    assert np.max(oracle.mode_angles(m, rm)) <= 1e-8
    summary = open(os.path.join(out, "summary.txt")).read()
    assert "world_size=2" in summary and "rank0_exchange_collectives=" in summary
