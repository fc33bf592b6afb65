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


@pytest.mark.parametrize("k,over", [(136, 0), (100, 20), (120, 8)])
def test_sketches_wider_than_the_fused_update(k, over):
    """Sketches of more than 112 columns (found by tools/fuzz_stream.py with FUZZ_BIG_K: the fused update's
    one-CTA solvers returned zeros without an error): psvd_rand_update refuses them and randomized_update
    composes the same sequence from the any-width kernels; stream, per-update calls and low_rank_svd (u, s
    and vt) against the oracle at the bar."""
    p = _pkg()
    rng = np.random.Generator(np.random.Philox(11))
    M, w = 3000, k + over + 40
    U, _ = np.linalg.qr(rng.standard_normal((M, 160)))
    V, _ = np.linalg.qr(rng.standard_normal((3 * w, 160)))
    a = (U * (0.93 ** np.arange(160))) @ V.T + 1e-9 * rng.standard_normal((M, 3 * w))
    b = [np.asfortranarray(a[:, i * w:(i + 1) * w]) for i in range(3)]
    sk = p.RandomSketchConfig(target_rank=k, oversampling=over, power_iterations=1, seed=2)
    cfg = p.StreamConfig(k_modes=k, forget_factor=0.95, batch_columns=w, sketch=sk)
    ref_m, ref_s, _ = oracle.ref_rand_stream_all(b, k, 0.95, over, 1, 2)
    st, hist = p.stream_all(b, cfg)
    m, s = st.numpy()
    assert len(hist) == 3 and oracle.sigma_rel_err(s, ref_s) <= SIG_TOL
    gaps = np.array([min(abs(ref_s[j] - ref_s[i]) for i in range(k) if i != j) / ref_s[j] for j in range(k)])
    sel = gaps > 1e-3
    assert float(np.max(oracle.mode_angles(m, ref_m)[sel])) <= ANG_TOL
    assert np.all(np.sum(m * ref_m, axis=0)[sel] > 0)
    res = p.low_rank_svd(b[0], sk)
    u, s1, vt = oracle.ref_low_rank_svd(b[0], k, over, 1, 2)
    assert oracle.sigma_rel_err(res.s.cpu().numpy(), s1) <= SIG_TOL
    assert float(np.max(np.abs(res.vt.cpu().numpy() - vt)[sel])) <= 1e-7
    import ctypes
    from paper_2108_08845_b200 import _native as nat
    with pytest.raises(ValueError):   # the C entry point itself fails loudly
        dev = st.modes.device
        A = nat.as_device_colmajor(b[0], dev)
        out = nat.DevMat.empty(M, k, dev)
        sig = st.singular_values.clone()
        om = p.linalg.device_omega(w, sk, dev)
        nat.call("psvd_rand_update", nat.context(dev), M, nat._vp(0), 0, nat._vp(0), 1.0, 0, nat._vp(A.data_ptr()), A.ld,
                 w, k, k + over, 1, nat.ptr(om), nat._vp(out.data_ptr()), out.ld, nat.ptr(sig), nat.stream_ptr(dev))
