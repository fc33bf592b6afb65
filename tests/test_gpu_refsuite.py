"""The reference's own test scenarios for the path, restated on the device drop-in.

test_gpu_edge.py / test_gpu_linalg.py carry most of /root/reference/pkg/tests/test_streaming.py,
test_linalg.py and test_dsvd.py; this file holds the remaining cases, one per reference test, under the
reference test's name.  Each restates the scenario with its own construction (same shapes, seeds' role and
bars as the cited lines), asserts the reference test's property on the device result, and — where the
oracle covers the call — parity with the pinned oracle on the same bytes at the north-star bar.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SIG_TOL, ANG_TOL = 1e-10, 1e-8


def _p():
    import paper_2108_08845_b200 as p
    return p


def _philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def _batches(a, w):
    return [a[:, i:i + w] for i in range(0, a.shape[1], w)]


def _constructed(rows, cols, seed):
    sv = np.concatenate([1.25 ** -np.arange(5), 1e-8 * 0.5 ** np.arange(12)])
    return _p().synthetic_spectrum_matrix(rows, cols, sv, seed=seed)


def _parity(state, ref_m, ref_s):
    m, s = state.numpy()
    assert oracle.sigma_rel_err(s, ref_s) <= SIG_TOL, (s, ref_s)
    assert np.max(oracle.mode_angles(m, ref_m)) <= ANG_TOL
    assert np.all(np.sum(m * ref_m, axis=0) > 0)
    return m, s


# ------------------------------------------------------------------ test_streaming.py

def test_initialize_diagonal_exact():
    """test_streaming.py:33-38: a 3 x 3 diagonal gives its entries and +-unit vectors exactly."""
    p = _p()
    st = p.stream_initialize(np.diag([3.0, 2.0, 1.0]), p.StreamConfig(k_modes=3, batch_columns=3))
    m, s = st.numpy()
    assert np.array_equal(s, [3.0, 2.0, 1.0])
    assert np.array_equal(np.abs(m), np.eye(3))
    assert st.iteration == 0


def test_initialize_matches_direct_svd():
    """test_streaming.py:41-48: K = all 8 columns of a 30 x 8 Gaussian equals the direct SVD."""
    p = _p()
    a0 = _philox(40).standard_normal((30, 8))
    st = p.stream_initialize(a0, p.StreamConfig(k_modes=8, batch_columns=8))
    m, s = st.numpy()
    u, sv, _ = oracle.ref_svd(a0)
    assert np.max(np.abs(s - sv) / sv) < 1e-12
    assert np.max(oracle.aligned_mode_difference(m, u)) < 1e-10
    _parity(st, *oracle.ref_stream_init(a0, 8))
    d = p.svd_full(a0)
    assert np.max(np.abs(d.s.cpu().numpy() - sv) / sv) < 1e-12


def test_initialize_needs_enough_columns():
    """test_streaming.py:51-53."""
    p = _p()
    with pytest.raises(ValueError):
        p.stream_initialize(np.ones((5, 2)), p.StreamConfig(k_modes=3))


def test_single_shot_equivalence_constructed_spectrum():
    """test_streaming.py:56-63: 60 x 36, gap after the fifth value, ff = 1, 15-column batches."""
    p = _p()
    a = _constructed(60, 36, 11)
    u, sv, _ = oracle.ref_svd(a)
    st, _ = p.stream_all(p.BatchSource.from_matrix(a, 15), p.StreamConfig(k_modes=5, forget_factor=1.0,
                                                                          batch_columns=15))
    m, s = st.numpy()
    assert np.max(np.abs(s - sv[:5]) / sv[:5]) < 1e-8
    assert np.max(oracle.aligned_mode_difference(m, u[:, :5])) < 1e-6
    _parity(st, *oracle.ref_stream_all(_batches(a, 15), 5, 1.0)[:2])


def test_forget_factor_damps_history():
    """test_streaming.py:109-116."""
    p = _p()
    a = _constructed(50, 20, 13)
    out = {}
    for ff in (1.0, 0.95):
        st, _ = p.stream_all(_batches(a, 10), p.StreamConfig(k_modes=5, forget_factor=ff, batch_columns=10))
        out[ff] = st.numpy()[1]
        _parity(st, *oracle.ref_stream_all(_batches(a, 10), 5, ff)[:2])
    assert out[0.95][0] < out[1.0][0]
    assert np.all(out[0.95] <= out[1.0] + 1e-12)


def test_variable_batch_width_accepted():
    """test_streaming.py:132-139: batches of 5, 1 and 9 columns through one stream."""
    p = _p()
    rng = _philox(43)
    cfg = p.StreamConfig(k_modes=3, forget_factor=1.0, batch_columns=5)
    b = [rng.standard_normal((20, w)) for w in (5, 1, 9)]
    st = p.stream_initialize(b[0], cfg)
    rm, rs = oracle.ref_stream_init(b[0], 3)
    for x in b[1:]:
        st = p.stream_incorporate(st, x, cfg)
        rm, rs = oracle.ref_stream_update(rm, rs, x, 3, 1.0)
    assert tuple(st.modes.shape) == (20, 3) and st.iteration == 2
    _parity(st, rm, rs)
    st2, hist = p.stream_all(b, cfg)      # the same ragged stream through the pipelined window
    assert len(hist) == 3
    _parity(st2, rm, rs)


def test_incorporate_validates_shapes():
    """test_streaming.py:142-151: wrong rows, an empty batch, a config whose K differs from the state's."""
    p = _p()
    cfg = p.StreamConfig(k_modes=2, batch_columns=4)
    st = p.stream_initialize(np.diag([2.0, 1.0, 0.5]), cfg)
    with pytest.raises(ValueError):
        p.stream_incorporate(st, np.ones((4, 2)), cfg)
    with pytest.raises(ValueError):
        p.stream_incorporate(st, np.ones((3, 0)), cfg)
    with pytest.raises(ValueError):
        p.stream_incorporate(st, np.ones((3, 2)), p.StreamConfig(k_modes=3, batch_columns=4))
    with pytest.raises(ValueError):
        p.stream_incorporate(st, np.full((3, 2), np.nan), cfg)   # linalg.py:76-77 through the update


def test_rescue_pass_restores_orthonormality():
    """test_streaming.py:154-165: a state drifted by 1e-4 comes back orthonormal to 1e-12 (the drift guard
    of streaming.py:104-110), and equals the reference's own rescued update."""
    p = _p()
    rng = _philox(44)
    q = np.linalg.qr(rng.standard_normal((30, 3)))[0]
    drifted = q + 1e-4 * rng.standard_normal((30, 3))
    sig = np.array([3.0, 2.0, 1.0])
    a = rng.standard_normal((30, 4))
    cfg = p.StreamConfig(k_modes=3, forget_factor=1.0, batch_columns=4)
    new = p.stream_incorporate(p.StreamState(drifted, sig, 0), a, cfg)
    m, s = new.numpy()
    assert np.max(np.abs(m.T @ m - np.eye(3))) < 1e-12
    assert np.all(np.diff(s) <= 0.0)
    _parity(new, *oracle.ref_stream_update(drifted, sig, a, 3, 1.0))


def test_stream_all_requires_batches():
    """test_streaming.py:168-170."""
    p = _p()
    with pytest.raises(ValueError):
        p.stream_all([], p.StreamConfig(k_modes=2))


def test_first_burgers_batch_matches_direct():
    """test_streaming.py:173-180 at the suite's Burgers fixture shape (conftest.py: 256 x 400): the first
    100 snapshots, K = 10, against the direct SVD at 1e-10 / 1e-8."""
    p = _p()
    a0 = oracle.burgers_matrix(256, 400)[:, :100]
    st = p.stream_initialize(a0, p.StreamConfig(k_modes=10, batch_columns=100))
    m, s = st.numpy()
    u, sv, _ = oracle.ref_svd(a0)
    assert np.max(np.abs(s - sv[:10]) / sv[:10]) < 1e-10
    assert np.max(oracle.aligned_mode_difference(m, u[:, :10])) < 1e-8


# ------------------------------------------------------------------ test_linalg.py (randomized part)

def test_range_finder_rejects_oversized_sketch_and_is_deterministic_per_seed():
    """test_linalg.py:141-154."""
    p = _p()
    with pytest.raises(ValueError):
        p.randomized_range(np.eye(4), p.RandomSketchConfig(target_rank=3, oversampling=2))
    a = _philox(16).standard_normal((25, 10))
    c99 = p.RandomSketchConfig(target_rank=4, oversampling=2, seed=99)
    c100 = p.RandomSketchConfig(target_rank=4, oversampling=2, seed=100)
    q1, q2, q3 = (p.randomized_range(a, c).cpu().numpy() for c in (c99, c99, c100))
    assert np.array_equal(q1, q2) and not np.array_equal(q1, q3)
    ref = oracle.ref_range(a, 6, 1, 99)
    assert np.max(np.abs(q1 - ref)) < 1e-10      # the same basis, column for column (qr with diag(r) >= 0)


def test_low_rank_svd_exact_on_low_rank_input():
    """test_linalg.py:157-167: an exactly rank-3 40 x 15 matrix, K = 3, p = 5, q = 1."""
    p = _p()
    rng = _philox(17)
    u0 = np.linalg.qr(rng.standard_normal((40, 3)))[0]
    v0 = np.linalg.qr(rng.standard_normal((15, 3)))[0]
    a = (u0 * [7.0, 4.0, 2.0]) @ v0.T
    res = p.low_rank_svd(a, p.RandomSketchConfig(target_rank=3, oversampling=5, power_iterations=1, seed=1))
    u, s, vt = (x.cpu().numpy() for x in res)
    assert np.allclose(s, [7.0, 4.0, 2.0], rtol=1e-10)
    du = oracle.ref_svd(a)[0]
    assert np.max(oracle.aligned_mode_difference(u, du[:, :3])) < 1e-9
    assert np.max(np.abs((u * s) @ vt - a)) < 1e-9
    ru, rs, rvt = oracle.ref_low_rank_svd(a, 3, 5, 1, 1)
    assert oracle.sigma_rel_err(s, rs) <= SIG_TOL
    assert np.max(oracle.mode_angles(u, ru)) <= ANG_TOL and np.all(np.sum(u * ru, axis=0) > 0)
    assert np.max(np.abs(vt - rvt)) < 1e-9


def test_low_rank_svd_on_known_diagonal():
    """test_linalg.py:170-176: 8 x 5 with diag(5..1) on top, K = 3, p = 2, q = 2."""
    p = _p()
    a = np.zeros((8, 5))
    a[:5, :5] = np.diag([5.0, 4.0, 3.0, 2.0, 1.0])
    res = p.low_rank_svd(a, p.RandomSketchConfig(target_rank=3, oversampling=2, power_iterations=2, seed=7))
    assert tuple(res.u.shape) == (8, 3) and tuple(res.vt.shape) == (3, 5)
    s = res.s.cpu().numpy()
    assert np.allclose(s, [5.0, 4.0, 3.0], atol=1e-8)
    assert oracle.sigma_rel_err(s, oracle.ref_low_rank_svd(a, 3, 2, 2, 7)[1]) <= SIG_TOL


def test_low_rank_svd_tail_quality_over_seeds():
    """test_linalg.py:179-199: sigma_j = 2^-j, 120 x 40, K = p = 10, q = 1 over 20 seeds: leading values
    within 1 %, reconstruction within 3x optimal for >= 19 seeds — and every seed at the bar against the
    reference's own result."""
    p = _p()
    sv = 2.0 ** -np.arange(1, 41)
    good_v = good_r = 0
    for seed in range(20):
        a = p.synthetic_spectrum_matrix(120, 40, sv, seed=seed)
        res = p.low_rank_svd(a, p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=1, seed=seed))
        u, s, vt = (x.cpu().numpy() for x in res)
        good_v += np.max(np.abs(s[:5] - sv[:5]) / sv[:5]) <= 0.01
        good_r += np.linalg.norm(a - (u * s) @ vt) <= 3.0 * np.linalg.norm(sv[10:])
        ru, rs, _ = oracle.ref_low_rank_svd(a, 10, 10, 1, seed)
        assert oracle.sigma_rel_err(s, rs) <= SIG_TOL, seed
        assert np.max(oracle.mode_angles(u, ru)) <= ANG_TOL, seed
    assert good_v >= 19 and good_r >= 19


# ------------------------------------------------------------------ test_dsvd.py (row-parallel part)

def test_parallel_stream_single_rank_is_serial_bitwise():
    """test_dsvd.py:214-229: with one rank the parallel entry points are the serial ones, bit for bit."""
    p = _p()
    a = _philox(68).standard_normal((24, 15))
    cfg = p.StreamConfig(k_modes=4, forget_factor=0.95, batch_columns=5)
    s = p.stream_initialize(a[:, :5], cfg)
    s = p.stream_incorporate(s, a[:, 5:10], cfg)
    s = p.stream_incorporate(s, a[:, 10:], cfg)
    ctx = p.RankContext()
    r = p.parallel_stream_initialize(ctx, a[:, :5], cfg)
    r = p.parallel_stream_incorporate(ctx, r, a[:, 5:10], cfg)
    r = p.parallel_stream_incorporate(ctx, r, a[:, 10:], cfg)
    assert np.array_equal(r.modes.cpu().numpy(), s.modes.cpu().numpy())
    assert np.array_equal(r.singular_values.cpu().numpy(), s.singular_values.cpu().numpy())
    full = p.gather_modes(ctx, r)
    assert np.array_equal(full.cpu().numpy(), s.modes.cpu().numpy())     # test_dsvd.py:288-298 at one rank


def _gapped_rank_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        sv = np.concatenate([1.3 ** -np.arange(4), 1e-9 * 0.5 ** np.arange(8)])
        a = p.synthetic_spectrum_matrix(60, 24, sv, seed=69)
        lo, hi = p.partition_bounds(60, world)[rank]
        cfg = p.StreamConfig(k_modes=4, forget_factor=1.0, batch_columns=8)
        ctx = p.RankContext()
        st = p.parallel_stream_initialize(ctx, a[lo:hi, :8], cfg)
        for c0 in (8, 16):
            st = p.parallel_stream_incorporate(ctx, st, a[lo:hi, c0:c0 + 8], cfg)
        full = p.gather_modes(ctx, st)
        q.put((rank, st.singular_values.cpu().numpy(), None if full is None else full.cpu().numpy()))
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_parallel_stream_matches_direct_on_gapped_spectrum():
    """test_dsvd.py:232-250 with four processes sharing this GPU (gloo): 60 x 24, four leading values then a
    1e-9 tail, K = 4, ff = 1, 15-row blocks of 8-column batches: the direct SVD at 1e-8 / 1e-6 (the
    reference's bars), and the reference's parallel stream at the north-star bar."""
    import socket
    import torch.multiprocessing as mp
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gapped_rank_worker, args=(r, 4, port, q)) for r in range(4)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(4):
        rank, s, full = q.get(timeout=300)
        assert not (isinstance(s, str) and s == "error"), full
        out[rank] = (s, full)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    assert all(np.array_equal(out[0][0], out[r][0]) for r in range(1, 4))
    assert all(out[r][1] is None for r in range(1, 4))                    # gathered at the root only
    p = _p()
    sv = np.concatenate([1.3 ** -np.arange(4), 1e-9 * 0.5 ** np.arange(8)])
    a = p.synthetic_spectrum_matrix(60, 24, sv, seed=69)
    u, dsv, _ = oracle.ref_svd(a)
    s, full = out[0]
    assert np.max(np.abs(s - dsv[:4]) / dsv[:4]) < 1e-8
    assert np.max(oracle.aligned_mode_difference(full, u[:, :4])) < 1e-6
    rm, rs = oracle.ref_parallel_stream_all(a, [(0, 8), (8, 16), (16, 24)], 4, 4, 1.0)
    assert oracle.sigma_rel_err(s, rs) <= SIG_TOL
    assert np.max(oracle.mode_angles(full, rm)) <= ANG_TOL
    assert np.all(np.sum(full * rm, axis=0) > 0)


def _short_block_worker(rank, world, port, q, rand):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        a = p.synthetic_spectrum_matrix(42, 120, 2.0 ** -np.arange(30), seed=5)
        lo, hi = p.partition_bounds(42, world)[rank]
        sk = p.RandomSketchConfig(target_rank=12, oversampling=8, power_iterations=1, seed=3) if rand else None
        cfg = p.StreamConfig(k_modes=20 if not rand else 12, forget_factor=0.95, batch_columns=40, sketch=sk)
        ctx = p.RankContext()
        st, hist = p.parallel_stream_all(ctx, [a[lo:hi, c:c + 40] for c in (0, 40, 80)], cfg)
        full = p.gather_modes(ctx, st)
        q.put((rank, st.singular_values.cpu().numpy(), None if full is None else full.cpu().numpy(), len(hist)))
    except Exception as e:
        q.put((rank, "error", repr(e), 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rand", [False, True])
def test_parallel_stream_all_short_blocks(rand):
    """The streaming counterpart of test_dsvd.py:196-211 (short blocks), found by tools/fuzz_parallel.py: 42
    rows over three ranks leave 14-row blocks, fewer than K = 20 (sketch width 20): the shape checks of the
    pipelined windows are the global matrix's, and the result is the serial stream's at the bar."""
    import socket
    import torch.multiprocessing as mp
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_short_block_worker, args=(r, 3, port, q, rand)) for r in range(3)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(3):
        rank, s, full, nh = q.get(timeout=300)
        assert not (isinstance(s, str) and s == "error"), full
        out[rank] = (s, full, nh)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    p = _p()
    a = p.synthetic_spectrum_matrix(42, 120, 2.0 ** -np.arange(30), seed=5)
    b = [a[:, c:c + 40] for c in (0, 40, 80)]
    rm, rs, _ = oracle.ref_rand_stream_all(b, 12, 0.95, 8, 1, 3) if rand else oracle.ref_stream_all(b, 20, 0.95)
    s, full, nh = out[0]
    assert nh == 3 and np.array_equal(s, out[1][0]) and np.array_equal(s, out[2][0])
    assert oracle.sigma_rel_err(s, rs) <= SIG_TOL
    live = rs > 1e-6 * rs[0]
    assert np.max(oracle.mode_angles(full, rm)[live]) <= ANG_TOL
    assert np.all(np.sum(full * rm, axis=0)[live] > 0)
