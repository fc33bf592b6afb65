"""The randomized update's conditioning gate (PSVD_ST_SKETCHCOND) and its accurate route.

The reference orthonormalizes every sketch with a Householder qr (linalg.py:94-104, 143-147), which keeps
sketch directions of any size; the device's fast path orthonormalizes through the sketch Gram (CholeskyQR /
SVQB), which drops or blurs directions below ~1e-7 of the largest.  When that happens the device reports the
status bit and the update is redone as the reference's own sequence on backward-stable kernels
(linalg.accurate_randomized_update).  Cases: steep synthetic spectra through the pipelined stream_all and the
per-update calls against the oracle at the north-star bar; a mild spectrum and the Burgers stream stay on the
fast path.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SIG_TOL, ANG_TOL = 1e-10, 1e-8


def _pkg():
    import paper_2108_08845_b200 as p
    return p


def _steep(span, M=4096, n=200, r=40, seed=7):
    rng = np.random.Generator(np.random.Philox(seed))
    U, _ = np.linalg.qr(rng.standard_normal((M, r)))
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    a = (U * (span ** (1.0 / 19)) ** np.arange(r)) @ V.T   # sigma_20 / sigma_1 = span
    return [np.asfortranarray(a), np.asfortranarray(a[:, ::-1] * 0.5 + 0.1 * a)]


def _check(m, s, ref_m, ref_s):
    assert oracle.sigma_rel_err(s, ref_s) <= SIG_TOL
    assert float(np.max(oracle.mode_angles(m, ref_m))) <= ANG_TOL
    assert np.all(np.sum(m * ref_m, axis=0) > 0)   # the reference's signs


@pytest.mark.parametrize("span,q", [(1e-7, 0), (1e-8, 0), (1e-10, 1), (1e-13, 0)])
def test_steep_sketch_takes_accurate_route(span, q):
    p = _pkg()
    from paper_2108_08845_b200 import linalg
    b = _steep(span)
    sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=q, seed=0)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200, sketch=sk)
    ref_m, ref_s, _ = oracle.ref_rand_stream_all(b, 10, 0.95, 10, q, 0)
    n0 = linalg.ACCURATE_RAND_UPDATES
    st, hist = p.stream_all(b, cfg)                     # pipelined window, redone per update when gated
    assert linalg.ACCURATE_RAND_UPDATES > n0
    _check(*st.numpy(), ref_m, ref_s)
    st2 = p.stream_incorporate(p.stream_initialize(b[0], cfg), b[1], cfg)   # the per-update calls
    _check(*st2.numpy(), ref_m, ref_s)
    assert len(hist) == 2


def test_mild_sketch_and_burgers_stay_on_the_fast_path():
    p = _pkg()
    from paper_2108_08845_b200 import linalg
    sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=0, seed=0)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200, sketch=sk)
    n0 = linalg.ACCURATE_RAND_UPDATES
    b = _steep(1e-5)
    st, _ = p.stream_all(b, cfg)
    ref_m, ref_s, _ = oracle.ref_rand_stream_all(b, 10, 0.95, 10, 0, 0)
    _check(*st.numpy(), ref_m, ref_s)
    a = oracle.burgers_matrix(8192, 800)                 # the benchmark's data (config 2 at reduced rows)
    bb = [np.asfortranarray(a[:, c:c + 200]) for c in range(0, 800, 200)]
    for q in (0, 1):
        cq = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200,
                            sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=q, seed=0))
        st, _ = p.stream_all(bb, cq)
        ref_m, ref_s, _ = oracle.ref_rand_stream_all(bb, 10, 0.95, 10, q, 0)
        _check(*st.numpy(), ref_m, ref_s)
    assert linalg.ACCURATE_RAND_UPDATES == n0


def test_low_rank_svd_of_a_steep_matrix():
    """low_rank_svd (linalg.py:150-162) itself goes through the gate: u, s at the bar, vt rows following."""
    p = _pkg()
    a = _steep(1e-9)[0]
    sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=0, seed=0)
    res = p.low_rank_svd(a, sk)
    u, s, vt = oracle.ref_low_rank_svd(a, 10, 10, 0, 0)
    _check(res.u.cpu().numpy(), res.s.cpu().numpy(), u, s)


def _steep_rank_worker(rank, world, port, q, span, qit):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        from paper_2108_08845_b200 import linalg
        b = _steep(span)
        lo, hi = p.partition_bounds(b[0].shape[0], world)[rank]
        sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=qit, seed=0)
        cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200, sketch=sk)
        ctx = p.RankContext()
        n0 = linalg.ACCURATE_RAND_UPDATES
        st, hist = p.parallel_stream_all(ctx, [m[lo:hi] for m in b], cfg)      # pipelined, redone when gated
        n1 = linalg.ACCURATE_RAND_UPDATES
        st2 = p.parallel_stream_initialize(ctx, b[0][lo:hi], cfg)              # the per-update calls
        st2 = p.parallel_stream_incorporate(ctx, st2, b[1][lo:hi], cfg)
        full, full2 = p.gather_modes(ctx, st), p.gather_modes(ctx, st2)
        q.put((rank, st.singular_values.cpu().numpy(), st2.singular_values.cpu().numpy(),
               None if full is None else full.cpu().numpy(), None if full2 is None else full2.cpu().numpy(),
               (n1 - n0, linalg.ACCURATE_RAND_UPDATES - n1, len(hist))))
    except Exception as e:
        q.put((rank, "error", repr(e), None, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("span,qit", [(1e-8, 0), (1e-10, 1)])
def test_steep_sketch_row_partitioned_takes_accurate_route(span, qit):
    """The gate on the row-partitioned path (two processes sharing this GPU, gloo): the status bit comes
    from the summed Grams, so both ranks redo the update together on dsvd._parallel_accurate_rand_update
    (parallel_qr after every tall product, rank-ordered sums of the small ones, global sign rule); the
    result meets the bar against the serial R9 oracle with the reference's signs."""
    import socket
    import torch.multiprocessing as mp
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_steep_rank_worker, args=(r, 2, port, q, span, qit)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(2):
        rank, s1, s2, full, full2, counts = q.get(timeout=300)
        assert not (isinstance(s1, str) and s1 == "error"), s2
        out[rank] = (s1, s2, full, full2, counts)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert out[0][4][0] > 0 and out[0][4][1] > 0 and out[0][4][2] == 2
    ref_m, ref_s, _ = oracle.ref_rand_stream_all(_steep(span), 10, 0.95, 10, qit, 0)
    _check(out[0][2], out[0][0], ref_m, ref_s)
    _check(out[0][3], out[0][1], ref_m, ref_s)
