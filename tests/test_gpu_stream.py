"""GPU parity: the libpsvd deterministic streaming update vs the reference.

Bars (BASELINE.json north_star): singular values to relative error <= 1e-10,
modes to sign-invariant (sine-based) angles <= 1e-8 for well-separated modes.
Expected values come from the golden fixtures written by the live reference
(tests/golden) and from the pinned CPU oracle on the same input bytes.
"""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

SIG_TOL = 1e-10
ANG_TOL = 1e-8


def _pkg():
    import paper_2108_08845_b200 as p
    return p


def _batches(a, w):
    return [a[:, i:i + w] for i in range(0, a.shape[1], w)]


def _np(state):
    return state.numpy()


def _separated(sigma, rel_gap=1e-3):
    """Modes whose relative gap to both neighbours is at least rel_gap: the ones the north star's
    angle bar applies to (a mode inside a cluster is not determined by its singular value)."""
    s = np.asarray(sigma, dtype=np.float64)
    gap = np.full(s.size, np.inf)
    d = np.abs(np.diff(s))
    gap[:-1] = np.minimum(gap[:-1], d)
    gap[1:] = np.minimum(gap[1:], d)
    return gap >= rel_gap * np.maximum(s, 1e-300)


def _assert_parity(modes, sigma, ref_modes, ref_sigma, sig_tol=SIG_TOL, ang_tol=ANG_TOL, signs=True, sep=None):
    assert modes.shape == ref_modes.shape
    assert oracle.sigma_rel_err(sigma, ref_sigma) <= sig_tol, (sigma, ref_sigma)
    ang = oracle.mode_angles(modes, ref_modes)
    sel = np.ones(ang.size, dtype=bool) if sep is None else sep
    assert np.max(ang[sel]) <= ang_tol, ang
    if signs:  # the reference's sign convention is reproduced, not just the subspace
        assert np.all(np.sum(modes * ref_modes, axis=0)[sel] > 0)


def test_config1_burgers_golden(golden):
    p = _pkg()
    g = golden("det_burgers4096")
    a = p.burgers_matrix(4096, 800)
    cfg = p.StreamConfig(k_modes=10, forget_factor=1.0, batch_columns=200)
    state, hist = p.stream_all(_batches(a, 200), cfg)
    modes, sigma = _np(state)
    _assert_parity(modes, sigma, g["modes"], g["sigma"])
    for h, gh in zip(hist, g["history"]):
        assert oracle.sigma_rel_err(h.cpu().numpy(), gh) <= SIG_TOL
    assert state.iteration == 3
    gram = modes.T @ modes
    assert np.max(np.abs(gram - np.eye(10))) < 1e-12


def test_gaussian_forget_factor_golden(golden):
    p = _pkg()
    g = golden("det_gauss300")
    cfg = p.StreamConfig(k_modes=int(g["k"]), forget_factor=float(g["ff"]), batch_columns=int(g["batch"]))
    state, hist = p.stream_all(_batches(g["a"], int(g["batch"])), cfg)
    modes, sigma = _np(state)
    _assert_parity(modes, sigma, g["modes"], g["sigma"])


def test_edge_cases_golden(golden):
    p = _pkg()
    g = golden("det_edge_cases")
    st = p.stream_initialize(np.diag([3.0, 2.0, 1.0]), p.StreamConfig(k_modes=3, batch_columns=3))
    m, s = _np(st)
    assert np.allclose(s, [3.0, 2.0, 1.0], rtol=1e-15, atol=0)
    assert np.allclose(np.abs(m), np.eye(3), atol=1e-15)
    cfg = p.StreamConfig(k_modes=5, forget_factor=1.0, batch_columns=7)
    st, _ = p.stream_all(_batches(g["constructed_a"], 7), cfg)
    m, s = _np(st)
    _assert_parity(m, s, g["constructed_w7_modes"], g["constructed_w7_sigma"])
    st, _ = p.stream_all(_batches(g["rank3_a"], 6), p.StreamConfig(k_modes=3, forget_factor=1.0, batch_columns=6))
    m, s = _np(st)
    _assert_parity(m, s, g["rank3_modes"], g["rank3_sigma"])
    cfg = p.StreamConfig(k_modes=3, forget_factor=1.0, batch_columns=5)
    st = p.stream_initialize(g["varwidth_a0"], cfg)
    st = p.stream_incorporate(st, g["varwidth_a1"], cfg)
    st = p.stream_incorporate(st, g["varwidth_a2"], cfg)
    m, s = _np(st)
    _assert_parity(m, s, g["varwidth_modes"], g["varwidth_sigma"])
    assert st.iteration == 2


def test_drift_rescue_inside_pipelined_run():
    """Forced drift rescue (threshold < 0) inside the pipelined run: the gated pass,
    the sigma reorder and the T-rotation of the next batch's U^T A / U^T U must
    reproduce the unforced result (T ~ I for an orthonormal U)."""
    p = _pkg()
    from paper_2108_08845_b200 import _native as nat
    a = oracle.burgers_matrix(4096, 800)[:, :600]
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    base, _ = p.stream_all(_batches(a, 200), cfg)
    assert not (p.streaming.LAST_STATUS & nat.ST_RESCUE)
    ctx = nat.context(torch.device("cuda", 0))
    nat.call("psvd_set_drift_tol", ctx, -1.0)
    try:
        forced, _ = p.stream_all(_batches(a, 200), cfg)
        assert p.streaming.LAST_STATUS & nat.ST_RESCUE
    finally:
        nat.call("psvd_set_drift_tol", ctx, 1e-8)
    m1, s1 = forced.numpy()
    m2, s2 = base.numpy()
    _assert_parity(m1, s1, m2, s2, sig_tol=1e-13, ang_tol=1e-12)


def test_drift_rescue_golden(golden):
    p = _pkg()
    g = golden("det_edge_cases")
    state = p.StreamState(torch.as_tensor(g["rescue_modes_in"]).cuda(), torch.tensor([3.0, 2.0, 1.0]).cuda(), 0)
    new = p.stream_incorporate(state, g["rescue_batch"], p.StreamConfig(k_modes=3, forget_factor=1.0, batch_columns=4))
    m, s = _np(new)
    gram = m.T @ m
    assert np.max(np.abs(gram - np.eye(3))) < 1e-12
    assert np.all(np.diff(s) <= 0.0)
    _assert_parity(m, s, g["rescue_modes"], g["rescue_sigma"])


@pytest.mark.parametrize("rows,ff,k,b", [(65536, 0.95, 10, 200), (10007, 0.9, 8, 64), (4097, 1.0, 12, 100)])
def test_burgers_vs_oracle(rows, ff, k, b):
    p = _pkg()
    a = oracle.burgers_matrix(rows, 800)[:, : 4 * b]
    ref_m, ref_s, ref_h = oracle.ref_stream_all(_batches(a, b), k, ff)
    st, hist = p.stream_all(_batches(a, b), p.StreamConfig(k_modes=k, forget_factor=ff, batch_columns=b))
    m, s = _np(st)
    _assert_parity(m, s, ref_m, ref_s)


@pytest.mark.parametrize("rows,cols,k,b", [(1, 3, 1, 3), (7, 5, 3, 5), (31, 40, 4, 10), (33, 9, 2, 3),
                                           (300, 224, 8, 216), (129, 64, 32, 32)])
def test_shapes_vs_oracle(rows, cols, k, b):
    p = _pkg()
    rng = np.random.Generator(np.random.Philox(rows * 1000 + cols))
    a = rng.standard_normal((rows, cols))
    if k > rows:
        pytest.skip("k > rows")
    ref_m, ref_s, _ = oracle.ref_stream_all(_batches(a, b), k, 0.95)
    st, _ = p.stream_all(_batches(a, b), p.StreamConfig(k_modes=k, forget_factor=0.95, batch_columns=b))
    m, s = _np(st)
    # the north-star bar with the reference's signs, over the modes a Gaussian spectrum separates
    _assert_parity(m, s, ref_m, ref_s, sep=_separated(ref_s))


def test_deterministic_bitwise():
    p = _pkg()
    a = oracle.burgers_matrix(20000, 800)[:, :400]
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    s1, _ = p.stream_all(_batches(a, 200), cfg)
    s2, _ = p.stream_all(_batches(a, 200), cfg)
    assert torch.equal(s1.modes, s2.modes) and torch.equal(s1.singular_values, s2.singular_values)


def test_nonfinite_and_validation():
    p = _pkg()
    cfg = p.StreamConfig(k_modes=2, batch_columns=4)
    a = np.ones((10, 4))
    a[3, 2] = np.nan
    with pytest.raises(ValueError):
        p.stream_initialize(a, cfg)
    st = p.stream_initialize(np.random.default_rng(0).standard_normal((10, 4)), cfg)
    b = np.zeros((10, 3))
    b[0, 0] = np.inf
    with pytest.raises(ValueError):
        p.stream_incorporate(st, b, cfg)
    with pytest.raises(ValueError):
        p.stream_incorporate(st, np.ones((11, 2)), cfg)
    with pytest.raises(ValueError):
        p.stream_incorporate(st, np.ones((10, 2)), p.StreamConfig(k_modes=3))
    with pytest.raises(ValueError):
        p.stream_initialize(np.ones((5, 2)), p.StreamConfig(k_modes=3))
    with pytest.raises(ValueError):
        p.stream_all([], cfg)


def test_device_resident_inputs_match_host():
    p = _pkg()
    a = oracle.burgers_matrix(8192, 800)[:, :400]
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    s_host, _ = p.stream_all(_batches(a, 200), cfg)
    dev = torch.from_numpy(np.asfortranarray(a).T.copy()).cuda().T  # column-major CUDA view
    s_dev, _ = p.stream_all([dev[:, :200], dev[:, 200:]], cfg)
    assert torch.equal(s_host.modes, s_dev.modes)


def test_device_burgers_generator_matches_host():
    p = _pkg()
    host = oracle.burgers_matrix(4096, 800)
    devm = p.burgers_device(4096, 800).view.cpu().numpy()
    rel = np.abs(devm - host) / np.maximum(np.abs(host), 1e-300)
    assert np.max(rel[np.abs(host) > 1e-290]) < 1e-13
    sl = p.burgers_device(4096, 800, rows=(100, 357), cols=(13, 200)).view.cpu().numpy()
    assert np.array_equal(sl, devm[100:357, 13:200])


def test_parallel_single_rank_matches_serial():
    p = _pkg()
    a = oracle.burgers_matrix(4096, 800)[:, :600]
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    ctx = p.RankContext()
    st = p.parallel_stream_initialize(ctx, a[:, :200], cfg)
    for c in (200, 400):
        st = p.parallel_stream_incorporate(ctx, st, a[:, c:c + 200], cfg)
    # per-update serial chain: same kernels, bitwise equal (test_dsvd.py:214-229 property)
    ser = p.stream_initialize(a[:, :200], cfg)
    for c in (200, 400):
        ser = p.stream_incorporate(ser, a[:, c:c + 200], cfg)
    assert torch.equal(st.modes, ser.modes)
    assert torch.equal(st.singular_values, ser.singular_values)
    assert torch.equal(p.gather_modes(ctx, st), st.modes.contiguous())
    # the pipelined stream_all assembles the same Gram from two passes: parity, not bits
    pipe, _ = p.stream_all(_batches(a, 200), cfg)
    m1, s1 = pipe.numpy()
    m2, s2 = ser.numpy()
    _assert_parity(m1, s1, m2, s2, sig_tol=1e-13, ang_tol=1e-12)


def test_stream_all_windows_and_continuation():
    p = _pkg()
    a = oracle.burgers_matrix(6000, 800)
    ref_m, ref_s, ref_h = oracle.ref_stream_all(_batches(a, 50), 10, 0.95)
    old = (p.streaming.STREAM_WINDOW, p.streaming.STREAM_WINDOW_RESIDENT)
    try:
        p.streaming.STREAM_WINDOW = p.streaming.STREAM_WINDOW_RESIDENT = 3  # 16 batches -> windows 3,3,3,3,3,1 chained through the state
        st, hist = p.stream_all(_batches(a, 50), p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=50))
    finally:
        p.streaming.STREAM_WINDOW, p.streaming.STREAM_WINDOW_RESIDENT = old
    m, s = _np(st)
    _assert_parity(m, s, ref_m, ref_s)
    assert st.iteration == 15 and len(hist) == 16
    for h, rh in zip(hist, ref_h):
        assert oracle.sigma_rel_err(h.cpu().numpy(), rh) <= SIG_TOL


def test_stream_all_pinned_host_batches_overlap_copies():
    """Pinned host batches upload on the copy stream (per-batch ready events passed to
    psvd_stream_run): bitwise the same result as device-resident batches, in windows."""
    p = _pkg()
    a = oracle.burgers_matrix(8192, 800)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=100)
    dev_b = [torch.from_numpy(np.asfortranarray(a[:, c:c + 100])).cuda() for c in range(0, 800, 100)]
    host = torch.empty((800, 8192), dtype=torch.float64).pin_memory()
    host.copy_(torch.from_numpy(a.T.copy()))
    pin_b = [host[c:c + 100].T for c in range(0, 800, 100)]  # column-major pinned views
    old = (p.streaming.STREAM_WINDOW, p.streaming.STREAM_WINDOW_RESIDENT)
    try:
        p.streaming.STREAM_WINDOW = p.streaming.STREAM_WINDOW_RESIDENT = 3
        s1, h1 = p.stream_all(dev_b, cfg)
        s2, h2 = p.stream_all(pin_b, cfg)
    finally:
        p.streaming.STREAM_WINDOW, p.streaming.STREAM_WINDOW_RESIDENT = old
    assert torch.equal(s1.modes, s2.modes) and torch.equal(s1.singular_values, s2.singular_values)
    assert all(torch.equal(x, y) for x, y in zip(h1, h2))
    ref_m, ref_s, _ = oracle.ref_stream_all(_batches(a, 100), 10, 0.95)
    m, s = _np(s2)
    _assert_parity(m, s, ref_m, ref_s)


def test_parallel_golden_via_rank_emulation(golden):
    """4-rank golden (run_simulated of the reference) reproduced by summing the
    per-rank Grams exactly as the NCCL path does (allgather + ordered sum)."""
    p = _pkg()
    from paper_2108_08845_b200 import _native as nat
    g = golden("par_burgers2048_p4")
    a = p.burgers_matrix(2048, 800)
    bounds = p.partition_bounds(2048, 4)
    k, ff = 10, 0.95
    dev = torch.device("cuda", 0)
    c = nat.context(dev)
    st = nat.stream_ptr(dev)
    U = [None] * 4
    sig = None
    for c0 in range(0, 800, 200):
        kc = 0 if sig is None else k
        n = kc + 200
        Gs = []
        As = []
        for r, (lo, hi) in enumerate(bounds):
            A = nat.as_device_colmajor(a[lo:hi, c0:c0 + 200], dev)
            As.append(A)
            G = torch.empty((n, n), dtype=torch.float64, device=dev)
            nat.call("psvd_gram", c, hi - lo, nat._vp(U[r].data_ptr() if kc else 0), U[r].ld if kc else 0,
                     nat.ptr(sig if kc else None), ff, kc, nat._vp(A.data_ptr()), A.ld, 200, nat.ptr(G), st)
            Gs.append(G)
        parts = torch.stack(Gs)
        Gsum = torch.empty((n, n), dtype=torch.float64, device=dev)
        nat.call("psvd_sum_ordered", c, nat.ptr(parts), 4, n * n, nat.ptr(Gsum), st)
        W = torch.empty((k, n), dtype=torch.float64, device=dev)
        s_new = torch.empty(k, dtype=torch.float64, device=dev)
        nat.call("psvd_core_eig", c, nat.ptr(Gsum), n, nat.ptr(sig if kc else None), ff, kc, k, nat.ptr(W),
                 nat.ptr(s_new), st)
        newU = []
        for r, (lo, hi) in enumerate(bounds):
            out = nat.DevMat.empty(hi - lo, k, dev)
            nat.call("psvd_recompose", c, hi - lo, nat._vp(U[r].data_ptr() if kc else 0), U[r].ld if kc else 0,
                     kc, nat._vp(As[r].data_ptr()), As[r].ld, 200, nat.ptr(W), k, nat._vp(out.data_ptr()),
                     out.ld, nat._vp(0), st)
            newU.append(out)
        U, sig = newU, s_new
    modes = torch.cat([u.view for u in U], 0).cpu().numpy()
    _assert_parity(modes, sig.cpu().numpy(), g["modes"], g["sigma"])


# ---------------------------------------------------------------- randomized path (R8/R9)

@pytest.mark.parametrize("q", [0, 1])
def test_randomized_stream_golden(golden, q):
    p = _pkg()
    g = golden("rand_burgers2048")
    a = p.burgers_matrix(2048, 800)
    sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=q, seed=0)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200, sketch=sk)
    state, hist = p.stream_all(_batches(a, 200), cfg)
    modes, sigma = _np(state)
    for h, gh in zip(hist, g[f"q{q}_history"]):
        assert oracle.sigma_rel_err(h.cpu().numpy(), gh) <= SIG_TOL
    _assert_parity(modes, sigma, g[f"q{q}_modes"], g[f"q{q}_sigma"])


def test_low_rank_svd_small_golden(golden):
    p = _pkg()
    g = golden("rand_small")
    u, s, _ = p.low_rank_svd(g["lowrank_a"], p.RandomSketchConfig(target_rank=3, oversampling=5, power_iterations=1,
                                                                  seed=1))
    _assert_parity(u.cpu().numpy(), s.cpu().numpy(), g["lowrank_u"], g["lowrank_s"])
    u, s, _ = p.low_rank_svd(g["gauss_a"], p.RandomSketchConfig(target_rank=4, oversampling=2, power_iterations=0,
                                                                seed=99))
    _assert_parity(u.cpu().numpy(), s.cpu().numpy(), g["gauss_u"], g["gauss_s"], sig_tol=1e-10, ang_tol=1e-8)


@pytest.mark.parametrize("rows,k,p_,q,ff", [(65536, 10, 10, 1, 0.95), (30011, 16, 8, 0, 0.9), (5000, 30, 10, 2, 1.0)])
def test_randomized_vs_oracle(rows, k, p_, q, ff):
    p = _pkg()
    a = oracle.burgers_matrix(rows, 800)[:, :600]
    ref_m, ref_s, _ = oracle.ref_rand_stream_all(_batches(a, 200), k, ff, p_, q, 3)
    sk = p.RandomSketchConfig(target_rank=k, oversampling=p_, power_iterations=q, seed=3)
    st, _ = p.stream_all(_batches(a, 200), p.StreamConfig(k_modes=k, forget_factor=ff, batch_columns=200, sketch=sk))
    m, s = _np(st)
    _assert_parity(m, s, ref_m, ref_s)


@pytest.mark.parametrize("q", [0, 1, 2])
def test_pipelined_randomized_run_matches_per_update_and_oracle(q):
    """stream_all runs psvd_rand_stream_run (state kept as a sketch basis between updates, the
    next batch's sketch on the low-priority stream, U written once); stream_incorporate runs
    psvd_rand_update per batch.  Both against the oracle, per step: 10 batches with a ragged
    last one, so the second window starts from a materialized state (Kc = K)."""
    p = _pkg()
    a = oracle.burgers_matrix(8192, 950) + 1e-3 * np.random.default_rng(4).standard_normal((8192, 950))
    bs = _batches(a, 100)
    assert len(bs) == 10 and bs[-1].shape[1] == 50
    sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=q, seed=5)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=100, sketch=sk)
    st, hist = p.stream_all(bs, cfg)
    st2 = p.stream_initialize(bs[0], cfg)
    for b in bs[1:]:
        st2 = p.stream_incorporate(st2, b, cfg)
    ref_m, ref_s, ref_h = oracle.ref_rand_stream_all(bs, 10, 0.95, 10, q, 5)
    m, s = _np(st)
    _assert_parity(m, s, ref_m, ref_s)
    m2, s2 = _np(st2)
    _assert_parity(m2, s2, ref_m, ref_s)
    assert len(hist) == len(ref_h)
    for h, rh in zip(hist, ref_h):
        assert oracle.sigma_rel_err(h.cpu().numpy(), rh) <= SIG_TOL


@pytest.mark.parametrize("rows,b,k,p_,q", [(37, 12, 3, 2, 1), (1000, 20, 10, 0, 0), (4097, 64, 16, 16, 2),
                                          (65536, 200, 1, 1, 1), (24576, 100, 12, 20, 0),
                                          (16384, 197, 7, 6, 0), (32768, 130, 11, 9, 1)])
def test_pipelined_randomized_run_edge_shapes(rows, b, k, p_, q):
    """The pipelined randomized run at its edges: tiny and odd row counts (16-row TMA stages),
    no oversampling, the widest sketch (l = 32), K = 1, rows a multiple of 16 (32-row stages,
    register-resident W), odd batch widths and sketch widths off the 8-column grid (trimmed P-tile
    sub-blocks, SMSP-balanced tile placement): against the oracle per step."""
    p = _pkg()
    a = np.random.default_rng(rows + b).standard_normal((rows, 4 * b)) * np.linspace(2.0, 0.1, 4 * b)
    bs = _batches(a, b)
    sk = p.RandomSketchConfig(target_rank=k, oversampling=p_, power_iterations=q, seed=11)
    st, hist = p.stream_all(bs, p.StreamConfig(k_modes=k, forget_factor=0.9, batch_columns=b, sketch=sk))
    rm, rs, rh = oracle.ref_rand_stream_all(bs, k, 0.9, p_, q, 11)
    m, s_ = _np(st)
    for h, r_ in zip(hist, rh):
        assert oracle.sigma_rel_err(h.cpu().numpy(), r_) <= SIG_TOL
    gaps = np.minimum(np.abs(np.diff(np.r_[np.inf, rs])), np.abs(np.diff(np.r_[rs, 0.0]))) / rs
    sep = gaps > 1e-3  # sine angles are only defined for separated modes
    assert oracle.sigma_rel_err(s_, rs) <= SIG_TOL
    assert np.max(oracle.mode_angles(m[:, sep], rm[:, sep]), initial=0.0) <= ANG_TOL


def test_pipelined_randomized_run_bitwise_and_validation():
    p = _pkg()
    a = oracle.burgers_matrix(4096, 800)[:, :400]
    sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=1, seed=0)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200, sketch=sk)
    s1, _ = p.stream_all(_batches(a, 200), cfg)
    s2, _ = p.stream_all(_batches(a, 200), cfg)
    assert torch.equal(s1.modes, s2.modes) and torch.equal(s1.singular_values, s2.singular_values)
    bad = a.copy()
    bad[7, 250] = np.nan
    with pytest.raises(ValueError):
        p.stream_all(_batches(bad, 200), cfg)
    with pytest.raises(ValueError):  # initial batch narrower than k_modes
        p.stream_all([a[:, :5], a[:, 5:200]], cfg)


@pytest.mark.parametrize("b", [264, 300, 520])
def test_batches_wider_than_one_tma_box(b):
    """Segments wider than 256 columns take several TMA boxes; the last one may overhang the
    segment by < 8 columns only (a full-width overhang once zero-filled the next segment's
    columns).  Deterministic and randomized streams against the oracle."""
    p = _pkg()
    a = oracle.burgers_matrix(8192, 3 * b) + 1e-3 * np.random.default_rng(b).standard_normal((8192, 3 * b))
    bs = _batches(a, b)
    ref_m, ref_s, _ = oracle.ref_stream_all(bs, 10, 0.95)
    st, _ = p.stream_all(bs, p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=b))
    m, s_ = _np(st)
    _assert_parity(m, s_, ref_m, ref_s)
    sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=1, seed=2)
    ref_m, ref_s, _ = oracle.ref_rand_stream_all(bs, 10, 0.95, 10, 1, 2)
    st, _ = p.stream_all(bs, p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=b, sketch=sk))
    m, s_ = _np(st)
    _assert_parity(m, s_, ref_m, ref_s)


def test_randomized_validation():
    p = _pkg()
    with pytest.raises(ValueError):
        p.low_rank_svd(np.eye(4), p.RandomSketchConfig(target_rank=3, oversampling=2))
    with pytest.raises(ValueError):
        p.StreamConfig(k_modes=4, sketch=p.RandomSketchConfig(target_rank=3))


# ---------------------------------------------------------------- builder-defined configs 3-5
# at reduced rows against the oracle; the shapes (K, B, p) are the configs' own.

def _gap_mask(ref_s, thresh=1e-3):
    gaps = np.minimum(np.abs(np.diff(np.r_[np.inf, ref_s])), np.abs(np.diff(np.r_[ref_s, 0.0]))) / ref_s
    return gaps >= thresh


def _config_parity(a, K, B, ff, sketch=None, q=1):
    p = _pkg()
    batches = _batches(a, B)
    sk = None if sketch is None else p.RandomSketchConfig(target_rank=K, oversampling=sketch, power_iterations=q,
                                                           seed=0)
    st, hist = p.stream_all(batches, p.StreamConfig(k_modes=K, forget_factor=ff, batch_columns=B, sketch=sk))
    if sketch is None:
        rm, rs, rh = oracle.ref_stream_all(batches, K, ff)
    else:
        rm, rs, rh = oracle.ref_rand_stream_all(batches, K, ff, sketch, q, 0)
    m, s = _np(st)
    assert oracle.sigma_rel_err(s, rs) <= SIG_TOL
    ang = oracle.mode_angles(m, rm)
    mask = _gap_mask(rs)  # per-mode angles are defined for modes with relative gap >= 1e-3
    assert mask.sum() >= K // 2
    assert np.max(ang[mask]) <= ANG_TOL, ang
    assert oracle.sine_angles(m, rm).max() <= 1e-6  # whole-subspace angle
    for h, r in zip(hist, rh):
        assert oracle.sigma_rel_err(h.cpu().numpy(), r) <= SIG_TOL


def test_config5_stress_deterministic():
    from paper_2108_08845_b200 import datagen as dg
    _config_parity(dg.stress_matrix(1 << 14, 512), K=64, B=128, ff=1.0)


def test_config3_weather_randomized_wide():
    from paper_2108_08845_b200 import datagen as dg
    _config_parity(dg.weather_matrix(512, nlat=91, nlon=180), K=50, B=256, ff=0.95, sketch=10)


def test_config4_weak_randomized_wide():
    from paper_2108_08845_b200 import datagen as dg
    _config_parity(dg.weak_scaling_matrix(1 << 13, 1024), K=100, B=512, ff=0.95, sketch=10)


def test_wide_randomized_rank_deficient_core():
    """Wide route (l = 50 > 32) on a numerically rank-30 stream: the core SVD's CholeskyQR of B^T
    flags the ill-conditioned factor and the gated Jacobi on B^T itself runs; the modes above the
    noise floor match the oracle (the well-conditioned QR-then-Jacobi route is covered by the
    config 3 / 4 cases)."""
    p = _pkg()
    rng = np.random.default_rng(5)
    M, S, r = 6000, 600, 30
    U = np.linalg.qr(rng.standard_normal((M, r)))[0]
    V = np.linalg.qr(rng.standard_normal((S, r)))[0]
    a = np.asfortranarray((U * 0.8 ** np.arange(r)) @ V.T + 1e-13 * rng.standard_normal((M, S)))
    batches = _batches(a, 200)
    K = 40
    cfg = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=200,
                         sketch=p.RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=1, seed=0))
    st, hist = p.stream_all(batches, cfg)
    rm, rs, rh = oracle.ref_rand_stream_all(batches, K, 0.95, 10, 1, 0)
    m, s = _np(st)
    assert oracle.sigma_rel_err(s[:r], rs[:r]) <= SIG_TOL
    assert np.all(s[r:] < 1e-9 * s[0])
    mask = _gap_mask(rs[:r])
    ang = oracle.mode_angles(m[:, :r], rm[:, :r])
    assert mask.sum() >= r // 2
    assert np.max(ang[mask]) <= ANG_TOL, ang


def test_wide_randomized_route_matches_fused(monkeypatch):
    """The tall-skinny GEMM route (forced) and the fused passes agree to rounding."""
    p = _pkg()
    a = oracle.burgers_matrix(20000, 400)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200,
                         sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=1, seed=0))
    s1, _ = p.stream_all(_batches(a, 200), cfg)
    monkeypatch.setenv("PSVD_FORCE_WIDE", "1")
    s2, _ = p.stream_all(_batches(a, 200), cfg)
    m1, g1 = _np(s1)
    m2, g2 = _np(s2)
    _assert_parity(m2, g2, m1, g1, sig_tol=1e-13, ang_tol=1e-11)


def _wide_matrix():
    """A config-3-like field at reduced rows: the wide randomized route (K = 50, l = 60)."""
    from paper_2108_08845_b200.datagen import weather_matrix
    return weather_matrix(n_snapshots=768, nlat=91, nlon=180)


def _rand_rank_worker(rank, world, port, q, wide=False):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        a = _wide_matrix() if wide else oracle.burgers_matrix(6001, 600)
        k, b = (50, 256) if wide else (10, 200)
        lo, hi = p.partition_bounds(a.shape[0], world)[rank]
        cfg = p.StreamConfig(k_modes=k, forget_factor=0.95, batch_columns=b,
                             sketch=p.RandomSketchConfig(target_rank=k, oversampling=10, power_iterations=1, seed=0))
        ctx = p.RankContext()
        st = p.parallel_stream_initialize(ctx, a[lo:hi, :b], cfg)
        for c0 in range(b, a.shape[1], b):
            st = p.parallel_stream_incorporate(ctx, st, a[lo:hi, c0:c0 + b], cfg)
        full = p.gather_modes(ctx, st)
        if rank == 0:
            q.put((full.cpu().numpy(), st.singular_values.cpu().numpy()))
    except Exception as e:  # report instead of leaving the parent waiting
        q.put(("error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("wide", [False, True])
def test_parallel_randomized_two_ranks_match_serial_oracle(wide):
    """Row-partitioned randomized stream (§8(e)): two ranks (two processes sharing this
    GPU, gloo host-staged exchange through the library's collective hooks) reproduce
    the serial R9 composition on the whole matrix; narrow (l = 20, fused passes) and wide
    (l = 60, the tall-skinny GEMM route the config-4 weak-scaling leg runs)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rand_rank_worker, args=(r, 2, port, q, wide)) for r in range(2)]
    for pr in procs:
        pr.start()
    m, s_ = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
    assert not (isinstance(m, str) and m == "error"), s_
    assert all(pr.exitcode == 0 for pr in procs)
    if wide:
        a = _wide_matrix()
        rm, rs, _ = oracle.ref_rand_stream_all(_batches(a, 256), 50, 0.95, 10, 1, 0)
        _assert_parity(m, s_, rm, rs, sep=_separated(rs))
    else:
        a = oracle.burgers_matrix(6001, 600)
        rm, rs, _ = oracle.ref_rand_stream_all(_batches(a, 200), 10, 0.95, 10, 1, 0)
        _assert_parity(m, s_, rm, rs)


def _rand_run_rank_worker(rank, world, port, q, qit):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        p.streaming.STREAM_WINDOW = p.streaming.STREAM_WINDOW_RESIDENT = 2  # 4 batches = two windows: the second starts from a materialized state
        a = oracle.burgers_matrix(6001, 800)
        lo, hi = p.partition_bounds(a.shape[0], world)[rank]
        cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200,
                             sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=qit, seed=0))
        ctx = p.RankContext()
        n0 = p.streaming.PIPELINED_RAND_WINDOWS
        st, hist = p.parallel_stream_all(ctx, [a[lo:hi, c0:c0 + 200] for c0 in range(0, 800, 200)], cfg)
        full = p.gather_modes(ctx, st)
        q.put((rank, st.singular_values.cpu().numpy(), [h.cpu().numpy() for h in hist],
               None if full is None else full.cpu().numpy(), p.streaming.PIPELINED_RAND_WINDOWS - n0))
    except Exception as e:
        q.put((rank, "error", repr(e), None, 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("qit", [0, 1])
def test_parallel_pipelined_randomized_stream_ranks_match_serial(qit):
    """VERDICT r1 missing #5: the pipelined randomized stream row-partitioned (psvd_rand_stream_run with
    the exchange: the look-ahead sketch tiles, the projection Grams / partials and the sign rule's
    argmax pairs summed / gathered over the ranks; two processes sharing this GPU, gloo): identical
    singular values on both ranks, two windows, equal to the single-GPU pipelined run and to the
    serial R9 oracle at the bar."""
    import socket
    import torch.multiprocessing as mp
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rand_run_rank_worker, args=(r, 2, port, q, qit)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(2):
        rank, sig, hist, full, nwin = q.get(timeout=300)
        assert not (isinstance(sig, str) and sig == "error"), hist
        out[rank] = (sig, hist, full, nwin)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][3] == 2  # the pipelined run, in two windows
    p = _pkg()
    a = oracle.burgers_matrix(6001, 800)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200,
                         sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=qit, seed=0))
    old = (p.streaming.STREAM_WINDOW, p.streaming.STREAM_WINDOW_RESIDENT)
    try:
        p.streaming.STREAM_WINDOW = p.streaming.STREAM_WINDOW_RESIDENT = 2
        st, _ = p.stream_all(_batches(a, 200), cfg)
    finally:
        p.streaming.STREAM_WINDOW, p.streaming.STREAM_WINDOW_RESIDENT = old
    m1, s1 = _np(st)
    _assert_parity(out[0][2], out[0][0], m1, s1, sig_tol=1e-13, ang_tol=1e-11)
    rm, rs, rh = oracle.ref_rand_stream_all(_batches(a, 200), 10, 0.95, 10, qit, 0)
    _assert_parity(out[0][2], out[0][0], rm, rs)
    for h, r_ in zip(out[0][1], rh):
        assert oracle.sigma_rel_err(h, r_) <= SIG_TOL


def _det_run_rank_worker(rank, world, port, q, rows, cols, b):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        a = oracle.burgers_matrix(rows, cols) + 1e-4 * np.random.default_rng(9).standard_normal((rows, cols))
        lo, hi = p.partition_bounds(rows, world)[rank]
        cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=b)
        ctx = p.RankContext()
        loc = [a[lo:hi, c0:c0 + b] for c0 in range(0, cols, b)]
        st, hist = p.parallel_stream_all(ctx, loc, cfg)
        st2 = p.parallel_stream_initialize(ctx, loc[0], cfg)
        for m in loc[1:]:
            st2 = p.parallel_stream_incorporate(ctx, st2, m, cfg)
        full, full2 = p.gather_modes(ctx, st), p.gather_modes(ctx, st2)
        # the paper's class surface over the same calls (modes gathered at the root every step)
        obj = p.Parsvd_Parallel(10, 0.95, ctx=ctx).initialize(loc[0])
        for m in loc[1:]:
            obj.incorporate_data(m)
        same = (np.array_equal(obj.singular_values.cpu().numpy(), st2.singular_values.cpu().numpy()) and
                np.array_equal(obj.ulocal.cpu().numpy(), st2.modes.cpu().numpy()) and
                (obj.modes is None) == (full2 is None) and
                (full2 is None or np.array_equal(obj.modes.cpu().numpy(), full2.cpu().numpy())) and
                obj.iteration == len(loc) - 1)
        q.put((rank, st.singular_values.cpu().numpy(), [h.cpu().numpy() for h in hist],
               None if full is None else full.cpu().numpy(), None if full2 is None else full2.cpu().numpy(),
               st2.singular_values.cpu().numpy(), same))
    except Exception as e:
        q.put((rank, "error", repr(e), None, None, None, False))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols,b", [(2, 6001, 600, 200), (3, 8192, 1000, 100)])
def test_parallel_pipelined_stream_ranks_match_serial(world, rows, cols, b):
    """Row-partitioned pipelined stream (psvd_stream_run with the exchange hooks; two or three
    processes sharing this GPU, gloo through the host): identical singular values on every rank,
    the gathered modes match the serial oracle on the whole matrix and the per-update parallel
    path; 10 batches of 100 span two windows."""
    import socket
    import torch.multiprocessing as mp
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_det_run_rank_worker, args=(r, world, port, q, rows, cols, b)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(world):
        rank, sig, hist, full, full2, sig2, same = q.get(timeout=300)
        assert not (isinstance(sig, str) and sig == "error"), hist
        assert same  # Parsvd_Parallel == parallel_stream_initialize / incorporate, bitwise
        out[rank] = (sig, hist, full, full2, sig2)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    for r in range(1, world):
        assert np.array_equal(out[r][0], out[0][0])  # replicated core solve on identical bits
    a = oracle.burgers_matrix(rows, cols) + 1e-4 * np.random.default_rng(9).standard_normal((rows, cols))
    rm, rs, rh = oracle.ref_stream_all(_batches(a, b), 10, 0.95)
    _assert_parity(out[0][2], out[0][0], rm, rs)
    _assert_parity(out[0][3], out[0][4], rm, rs)
    for h, r_ in zip(out[0][1], rh):
        assert oracle.sigma_rel_err(h, r_) <= SIG_TOL


def _illcond_matrix(rows=6000, cols=320, span=1e-6, rank=40, seed=7):
    """synthetic_spectrum_matrix (datagen.py:93-115) with `rank` values log-spaced over `span`:
    a K = 40 stream whose kept spectrum is far beyond the Gram route's accuracy (eps kappa^2)."""
    import paper_2108_08845_b200 as p
    return p.synthetic_spectrum_matrix(rows, cols, np.logspace(0, np.log10(span), rank), seed=seed)


@pytest.mark.parametrize("ff,bw,span", [(1.0, 80, 1e-6), (0.95, 64, 1e-6), (0.95, 100, 1e-5)])
def test_ill_conditioned_stream_takes_accurate_route(ff, bw, span):
    """VERDICT r1 weak #2 / ADVICE: a K = 40 stream with sigma_1 / sigma_K up to 1e6.  The Gram
    route's gate (sigma_1 / sigma_K > 300) reroutes every update to the R-factor route, which
    meets the 1e-10 / 1e-8 bar against the reference with its signs, both through the pipelined
    stream_all (window redone per batch) and per update."""
    p = _pkg()
    a = _illcond_matrix(span=span)
    ref_m, ref_s, ref_h = oracle.ref_stream_all(_batches(a, bw), 40, ff)
    cfg = p.StreamConfig(k_modes=40, forget_factor=ff, batch_columns=bw)
    n0 = p.streaming.ACCURATE_UPDATES
    st, hist = p.stream_all(_batches(a, bw), cfg)
    assert p.streaming.ACCURATE_UPDATES - n0 >= len(_batches(a, bw))
    m, s = _np(st)
    _assert_parity(m, s, ref_m, ref_s)
    for h, rh in zip(hist, ref_h):
        assert oracle.sigma_rel_err(h.cpu().numpy(), rh) <= SIG_TOL
    assert np.max(np.abs(m.T @ m - np.eye(40))) < 1e-12
    # per update (stream_initialize / stream_incorporate) gives the same answer
    bs = _batches(a, bw)
    st2 = p.stream_initialize(bs[0], cfg)
    for b in bs[1:]:
        st2 = p.stream_incorporate(st2, b, cfg)
    m2, s2 = _np(st2)
    _assert_parity(m2, s2, ref_m, ref_s)


def test_gram_route_stays_on_when_well_conditioned():
    """The gate costs nothing on the benchmark's own data: Burgers K = 10 (sigma_1 / sigma_K ~ 25)
    never reroutes."""
    p = _pkg()
    a = oracle.burgers_matrix(8192, 800)
    n0 = p.streaming.ACCURATE_UPDATES
    p.stream_all(_batches(a, 200), p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200))
    assert p.streaming.ACCURATE_UPDATES == n0


def _illcond_rank_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        a = _illcond_matrix(rows=5001, cols=240)
        lo, hi = p.partition_bounds(a.shape[0], world)[rank]
        cfg = p.StreamConfig(k_modes=40, forget_factor=0.95, batch_columns=80)
        ctx = p.RankContext()
        loc = [a[lo:hi, c0:c0 + 80] for c0 in range(0, a.shape[1], 80)]
        st, hist = p.parallel_stream_all(ctx, loc, cfg)
        full = p.gather_modes(ctx, st)
        q.put((rank, st.singular_values.cpu().numpy(), None if full is None else full.cpu().numpy(),
               p.streaming.ACCURATE_UPDATES))
    except Exception as e:
        q.put((rank, "error", repr(e), 0))
        raise
    finally:
        dist.destroy_process_group()


def test_parallel_ill_conditioned_stream_accurate_route():
    """The accurate route row-partitioned (two processes sharing this GPU, gloo): every Gram and
    projection of the deflation basis is summed over the ranks through the exchange hooks, the
    small factorizations are replicated on identical bits."""
    import socket
    import torch.multiprocessing as mp
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_illcond_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(2):
        rank, sig, full, nacc = q.get(timeout=300)
        assert not (isinstance(sig, str) and sig == "error"), full
        out[rank] = (sig, full, nacc)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][2] >= 3
    a = _illcond_matrix(rows=5001, cols=240)
    rm, rs, _ = oracle.ref_stream_all(_batches(a, 80), 40, 0.95)
    _assert_parity(out[0][1], out[0][0], rm, rs)


@pytest.mark.parametrize("low_rank", [False, True])
def test_parsvd_serial_class_matches_function_api_and_oracle(low_rank):
    """PyParSVD's class surface (listing 1): Parsvd_Serial(K, ff).initialize(A0) then
    incorporate_data(A) per batch is the function API bitwise, and the reference by the oracle."""
    p = _pkg()
    a = oracle.burgers_matrix(4096, 800)
    bs = _batches(a, 200)
    obj = p.Parsvd_Serial(10, 0.95, low_rank=low_rank).initialize(bs[0])
    st = p.stream_initialize(bs[0], obj.config)
    for b in bs[1:]:
        obj.incorporate_data(b)
        st = p.stream_incorporate(st, b, obj.config)
    assert obj.iteration == 3
    assert np.array_equal(obj.singular_values.cpu().numpy(), st.singular_values.cpu().numpy())
    assert np.array_equal(obj.modes.cpu().numpy(), st.modes.cpu().numpy())
    if low_rank:
        rm, rs, _ = oracle.ref_rand_stream_all(bs, 10, 0.95, 10, 1, 0)
    else:
        rm, rs, _ = oracle.ref_stream_all(bs, 10, 0.95)
    m, s_ = _np(obj.state)
    _assert_parity(m, s_, rm, rs)


def test_parallel_randomized_single_rank_is_serial():
    p = _pkg()
    a = oracle.burgers_matrix(4096, 400)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200,
                         sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=1, seed=0))
    ctx = p.RankContext()
    st = p.parallel_stream_initialize(ctx, a[:, :200], cfg)
    st = p.parallel_stream_incorporate(ctx, st, a[:, 200:], cfg)
    ser = p.stream_incorporate(p.stream_initialize(a[:, :200], cfg), a[:, 200:], cfg)
    assert torch.equal(st.modes, ser.modes) and torch.equal(st.singular_values, ser.singular_values)


def test_core_solver_paths_both_exercised_and_exact():
    """The subspace-iteration fast path converges on the low-rank Burgers Gram; on a flat
    Gaussian spectrum its residual gate fails and the full solver runs.  Both match the oracle."""
    import ctypes
    p = _pkg()
    from paper_2108_08845_b200 import _native as nat
    dev = torch.device("cuda", 0)
    c = nat.context(dev)
    full = ctypes.c_int(-1)
    a = oracle.burgers_matrix(20000, 400)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    st = p.stream_incorporate(p.stream_initialize(a[:, :200], cfg), a[:, 200:], cfg)
    nat.call("psvd_last_core_path", c, ctypes.byref(full))
    assert full.value == 0
    rm, rs, _ = oracle.ref_stream_all(_batches(a, 200), 10, 0.95)
    m, s = _np(st)
    _assert_parity(m, s, rm, rs)
    rng = np.random.default_rng(5)
    g = rng.standard_normal((3000, 400))
    st = p.stream_incorporate(p.stream_initialize(g[:, :200], cfg), g[:, 200:], cfg)
    nat.call("psvd_last_core_path", c, ctypes.byref(full))
    assert full.value != 0
    rm, rs, _ = oracle.ref_stream_all(_batches(g, 200), 10, 0.95)
    m, s = _np(st)
    _assert_parity(m, s, rm, rs)


def test_config2_shapes_run_on_the_tma_kernels():
    """Guard against silent fallbacks: at the config-2 shapes (B = 200, K = 10, l = 20) every
    pass of the deterministic stream and of the randomized update runs on the TMA kernels."""
    p = _pkg()
    from paper_2108_08845_b200 import _native as nat
    dev = torch.device("cuda", 0)
    c = nat.context(dev)
    a = torch.from_numpy(np.asfortranarray(oracle.burgers_matrix(1 << 16, 800))).cuda()
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    before = nat.path_counters(c)
    p.stream_all([a[:, i:i + 200] for i in range(0, 800, 200)], cfg)
    d = [x - y for x, y in zip(nat.path_counters(c), before)]
    assert d[0] >= 4 and d[1] >= 4 and d[2] == 0 and d[3] == 0 and d[4] == 0, d
    rcfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200,
                          sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=1, seed=0))
    before = nat.path_counters(c)
    p.stream_all([a[:, i:i + 200] for i in range(0, 800, 200)], rcfg)
    d = [x - y for x, y in zip(nat.path_counters(c), before)]
    assert d[0] > 0 and d[2] == 0 and d[3] == 0 and d[4] == 0, d


def test_stream_all_from_parsvd_file_pinned_prefetch(tmp_path):
    """§8(f) batch ingestion: a PARSVD01 file read by a background thread into pinned
    column-major batches, uploaded on the copy stream while earlier batches update:
    bitwise the result of the device-resident stream, and the oracle's."""
    p = _pkg()
    a = oracle.burgers_matrix(12000, 800)
    path = tmp_path / "burgers.parsvd"
    p.write_matrix(path, a)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    s_dev, _ = p.stream_all([torch.from_numpy(np.asfortranarray(a[:, i:i + 200])).cuda() for i in range(0, 800, 200)],
                            cfg)
    src = p.BatchSource.from_file(path, 200, pinned=True, prefetch=2)
    batches = list(src)
    assert all(b.is_pinned() and b.stride(0) == 1 for b in batches)
    s_file, _ = p.stream_all(p.BatchSource.from_file(path, 200, pinned=True, prefetch=2), cfg)
    assert torch.equal(s_file.modes, s_dev.modes) and torch.equal(s_file.singular_values, s_dev.singular_values)
    rm, rs, _ = oracle.ref_stream_all(_batches(a, 200), 10, 0.95)
    m, s = _np(s_file)
    _assert_parity(m, s, rm, rs)
    # a rank's row block straight from the file
    lo, hi = p.partition_bounds(12000, 3)[1]
    part = np.concatenate([b.numpy() for b in p.BatchSource(200, path=path, rows=(lo, hi), pinned=True)], axis=1)
    assert np.array_equal(part, a[lo:hi])


def test_library_nccl_exchange_world_one_is_bitwise_serial():
    """The library's own NCCL data plane (psvd_nccl_*: dlopen'ed libnccl, in-stream ncclAllGather +
    rank-ordered sum at every exchange point, no Python in the loop), on a one-rank communicator:
    the pipelined deterministic stream, the randomized update and the accurate route all run
    through it and reproduce the single-GPU results bit for bit; the exchange counters
    (CommStats analogue) advance."""
    import ctypes
    from paper_2108_08845_b200 import _native as nat
    from paper_2108_08845_b200.dsvd import exchange_stats
    p = _pkg()
    dev = torch.device("cuda", 0)
    c = nat.context(dev)
    ok = ctypes.c_int(0)
    nat.lib().psvd_nccl_available(ctypes.byref(ok))
    assert ok.value == 1
    a = oracle.burgers_matrix(6000, 800)[:, :600]
    det = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    rnd = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200,
                         sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=1, seed=0))
    ill = _illcond_matrix(rows=3000, cols=160)
    icfg = p.StreamConfig(k_modes=40, forget_factor=0.95, batch_columns=80)

    def runs():
        s1, _ = p.stream_all(_batches(a, 200), det)
        s2 = p.stream_incorporate(p.stream_initialize(a[:, :200], rnd), a[:, 200:400], rnd)
        s3 = p.stream_incorporate(p.stream_initialize(ill[:, :80], icfg), ill[:, 80:], icfg)
        return s1, s2, s3

    base = runs()
    buf = ctypes.create_string_buffer(128)
    nat.call("psvd_nccl_unique_id", c, buf)
    with torch.cuda.device(dev):
        nat.call("psvd_nccl_init", c, 1, 0, buf.raw)
    calls0, _ = exchange_stats(dev)
    nat.call("psvd_nccl_enable", c, 1, 0)
    try:
        viann = runs()
    finally:
        nat.call("psvd_nccl_enable", c, 0, 0)
        nat.call("psvd_nccl_destroy", c)
    calls1, _ = exchange_stats(dev)
    assert calls1 > calls0
    for x, y in zip(base, viann):
        assert torch.equal(x.modes, y.modes) and torch.equal(x.singular_values, y.singular_values)


def test_resident_batches_run_in_longer_windows():
    """Device tensors need no upload slots, so stream_all keeps up to STREAM_WINDOW_RESIDENT of them in one
    pipelined window (a window boundary costs the pipeline its head and tail); host batches keep
    STREAM_WINDOW.  20 resident batches = one window, against the oracle's 20 updates."""
    p = _pkg()
    a = oracle.burgers_matrix(4096, 800)
    dev = torch.device("cuda", 0)
    dev_b = [torch.from_numpy(np.asfortranarray(a[:, c:c + 40])).cuda() for c in range(0, 800, 40)]
    assert p.streaming.window_length(dev_b[0], dev) == min(p.streaming.STREAM_WINDOW_RESIDENT, 32)
    assert p.streaming.window_length(a[:, :40], dev) == p.streaming.STREAM_WINDOW
    st, hist = p.stream_all(dev_b, p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=40))
    ref_m, ref_s, ref_h = oracle.ref_stream_all(_batches(a, 40), 10, 0.95)
    m, s = _np(st)
    _assert_parity(m, s, ref_m, ref_s)
    assert st.iteration == 19 and len(hist) == 20
    for h, rh in zip(hist, ref_h):
        assert oracle.sigma_rel_err(h.cpu().numpy(), rh) <= SIG_TOL
