"""GPU parity of the dense factorizations behind the reference's linalg boundary:
qr_factor / svd_full / randomized_range / low_rank_svd's vt (linalg.py:94-162) and
parallel_qr (dsvd.py:176-202), against the oracle restatement (tests follow the
reference's own test_linalg.py / test_dsvd.py cases: exact identities, sign conventions,
Gram-Schmidt agreement, exact-rank range finding, short row blocks).
"""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _p():
    import paper_2108_08845_b200 as p
    return p


def _np(t):
    return t.detach().cpu().numpy()


def _rng(seed):
    return np.random.Generator(np.random.Philox(seed))


# ---------------------------------------------------------------- qr_factor

def test_qr_identity_exact():
    res = _p().qr_factor(np.eye(4))
    assert np.array_equal(_np(res.q), np.eye(4)) and np.array_equal(_np(res.r), np.eye(4))


def test_qr_negated_identity_sign_convention():
    res = _p().qr_factor(-np.eye(3))
    q, r = _np(res.q), _np(res.r)
    assert np.all(np.diag(r) >= 0.0)
    assert np.max(np.abs(q @ r + np.eye(3))) < 1e-15


@pytest.mark.parametrize("m,n", [(8, 3), (6, 6), (3, 7), (20, 7), (5000, 40), (1 << 16, 112), (1 << 16, 210),
                                 (1 << 16, 612), (700, 700), (200, 450)])
def test_qr_matches_reference(m, n):
    a = _rng(10 + m).standard_normal((m, n))
    res = _p().qr_factor(a)
    q, r = _np(res.q), _np(res.r)
    qr_, rr = oracle.ref_qr(a)
    k = min(m, n)
    assert q.shape == (m, k) and r.shape == (k, n)
    assert np.max(np.abs(q - qr_)) < 1e-10
    assert np.max(np.abs(r - rr)) < 1e-10 * max(1.0, np.abs(rr).max())
    assert np.max(np.abs(q @ r - a)) < 1e-12 * max(1.0, np.abs(a).max()) * np.sqrt(m)
    assert np.all(np.diag(r) >= 0.0)


def test_qr_ill_conditioned_takes_shifted_route():
    # cond ~ 1e10: beyond CholeskyQR2, the shifted CholeskyQR3 keeps Q orthonormal
    rng = _rng(21)
    u = oracle.ref_qr(rng.standard_normal((400, 12)))[0]
    v = oracle.ref_qr(rng.standard_normal((12, 12)))[0]
    a = (u * np.logspace(0, -10, 12)) @ v.T
    res = _p().qr_factor(a)
    q, r = _np(res.q), _np(res.r)
    assert np.max(np.abs(q.T @ q - np.eye(12))) < 1e-12
    assert np.max(np.abs(q @ r - a)) < 1e-14
    assert np.all(np.diag(r) >= 0.0)


@pytest.mark.parametrize("n", [40, 112, 210, 612])
def test_qr_rank_deficient_burgers(n):
    """Numerically rank-deficient input (Burgers 4096 x n: ~30 significant directions), where
    CholeskyQR breaks down: the rank-robust route keeps Householder's guarantees (orthonormal q,
    q r = a to rounding, diag(r) >= 0) and the well-determined rows of r match the reference's."""
    a = oracle.burgers_matrix(4096, 800)[:, :n]
    res = _p().qr_factor(a)
    q, r = _np(res.q), _np(res.r)
    qr_, rr = oracle.ref_qr(a)
    assert np.max(np.abs(q.T @ q - np.eye(n))) < 1e-13
    assert np.max(np.abs(q @ r - a)) < 1e-13 * np.abs(a).max()
    assert np.all(np.diag(r) >= 0.0) and np.allclose(r, np.triu(r), atol=0)
    # row k of r (and column k of q) is determined to ~eps |a|_2^2 / r_kk (eps |a|_2 / r_kk) by any
    # backward-stable QR; rows at rounding level are arbitrary (Householder's too)
    s1 = np.linalg.norm(a, 2)
    lead = np.abs(np.diag(rr)) > 1e-6 * np.abs(rr[0, 0])
    k = int(np.argmin(lead)) if not lead.all() else n
    assert k >= 3
    d = np.abs(np.diag(rr))[:k]
    assert np.all(np.max(np.abs(r[:k] - rr[:k]), axis=1) < 16 * np.finfo(float).eps * s1 * s1 / d)
    assert np.all(np.max(np.abs(q[:, :k] - qr_[:, :k]), axis=0) < 16 * np.finfo(float).eps * s1 / d)


def test_qr_rejects_bad_input_and_is_deterministic():
    p = _p()
    with pytest.raises(ValueError):
        p.qr_factor(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        p.qr_factor(np.ones(4))
    with pytest.raises(ValueError):
        p.qr_factor(np.array([[1.0, np.nan], [0.0, 1.0]]))
    with pytest.raises(ValueError):
        p.qr_factor(np.array([[np.inf, 1.0], [0.0, 1.0]]))
    a = _rng(11).standard_normal((20, 7))
    r1, r2 = p.qr_factor(a), p.qr_factor(a.copy())
    assert torch.equal(r1.q, r2.q) and torch.equal(r1.r, r2.r)


# ---------------------------------------------------------------- svd_full

def test_svd_diagonal_and_identity_exact():
    p = _p()
    res = p.svd_full(np.diag([3.0, 1.0]))
    assert np.array_equal(_np(res.s), [3.0, 1.0])
    assert np.array_equal(np.abs(_np(res.u)), np.eye(2)) and np.array_equal(np.abs(_np(res.vt)), np.eye(2))
    res = p.svd_full(np.eye(5))
    assert np.array_equal(_np(res.s), np.ones(5))
    assert np.max(np.abs(_np(res.u) @ np.diag(_np(res.s)) @ _np(res.vt) - np.eye(5))) < 1e-14


@pytest.mark.parametrize("m,n", [(6, 4), (4, 6), (9, 9), (10, 6), (300, 40), (40, 300), (3000, 112), (700, 150)])
def test_svd_matches_reference(m, n):
    a = _rng(12 + m + n).standard_normal((m, n))
    res = _p().svd_full(a)
    u, s, vt = _np(res.u), _np(res.s), _np(res.vt)
    ru, rs, rvt = oracle.ref_svd(a)
    k = min(m, n)
    assert u.shape == (m, k) and s.shape == (k,) and vt.shape == (k, n)
    assert np.max(np.abs(s - rs)) < 1e-12 * rs[0]
    assert np.all(np.diff(s) <= 0.0) and np.all(s >= 0.0)
    assert np.max(np.abs(u.T @ u - np.eye(k))) < 1e-12
    assert np.max(np.abs(vt @ vt.T - np.eye(k))) < 1e-12
    assert np.max(np.abs((u * s) @ vt - a)) < 1e-12 * rs[0]
    # Gaussian spectra are well separated: the vectors match the reference, signs included
    assert np.max(np.abs(u - ru)) < 1e-9 and np.max(np.abs(vt - rvt)) < 1e-9
    peaks = u[np.argmax(np.abs(u), axis=0), np.arange(k)]
    assert np.all(peaks > 0.0)


@pytest.mark.parametrize("m,n", [(2000, 300), (300, 2000), (612, 612)])
def test_svd_wide_matches_reference(m, n):
    """Beyond the one-CTA kernels (160 columns): CholeskyQR + the multi-CTA Jacobi on R^T."""
    a = _rng(30 + m + n).standard_normal((m, n))
    res = _p().svd_full(a)
    u, s, vt = _np(res.u), _np(res.s), _np(res.vt)
    ru, rs, rvt = oracle.ref_svd(a)
    k = min(m, n)
    assert np.max(np.abs(s - rs) / rs) < 1e-10
    assert np.max(np.abs(u.T @ u - np.eye(k))) < 1e-12
    assert np.max(np.abs(vt @ vt.T - np.eye(k))) < 1e-12
    assert np.max(np.abs((u * s) @ vt - a)) < 1e-12 * rs[0]
    # well-separated modes match the reference with its signs
    gap = np.minimum(np.abs(np.diff(rs, prepend=np.inf)), np.abs(np.diff(rs, append=-np.inf))) / rs
    sep = gap > 1e-3
    assert np.max(oracle.mode_angles(u[:, sep], ru[:, sep])) < 1e-8
    assert np.all(np.sum(u * ru, axis=0)[sep] > 0)


def test_svd_burgers_4096x800_full_spectrum():
    """svd_full of the whole Burgers 4096 x 800 matrix (the reference's serial-batch mode,
    cli.py:329-340): every singular value with a relative bar that backward-stable
    algorithms can meet (sigma_k >= 1e-5 sigma_1: both sides carry O(eps sigma_1) absolute
    error, the reference's dgesdd included), the rest to 1e-13 sigma_1 absolute; the
    leading modes to 1e-8 with the reference's signs."""
    a = oracle.burgers_matrix(4096, 800)
    res = _p().svd_full(a, want_vt=False)
    ru, rs, _ = oracle.ref_svd(a, want_vt=False)
    assert res.vt is None
    s = _np(res.s)
    u = _np(res.u)
    big = rs >= 1e-5 * rs[0]
    assert big.sum() >= 20
    assert np.max(np.abs(s[big] - rs[big]) / rs[big]) < 1e-10
    assert np.max(np.abs(s - rs)) < 1e-13 * rs[0]
    assert np.max(oracle.mode_angles(u[:, :20], ru[:, :20])) < 1e-8
    assert np.all(np.sum(u[:, :20] * ru[:, :20], axis=0) > 0)


def test_svd_want_vt_false_and_zero_matrix():
    p = _p()
    a = _rng(14).standard_normal((7, 5))
    full, left = p.svd_full(a, want_vt=True), p.svd_full(a, want_vt=False)
    assert left.vt is None
    assert torch.equal(full.u, left.u) and torch.equal(full.s, left.s)
    assert np.array_equal(_np(p.svd_full(np.zeros((4, 3))).s), np.zeros(3))


# ---------------------------------------------------------------- randomized_range / low_rank_svd

def test_range_finder_exact_rank_and_reference():
    p = _p()
    rng = _rng(15)
    a = np.outer(rng.standard_normal(30), rng.standard_normal(12))
    a += np.outer(rng.standard_normal(30), rng.standard_normal(12))
    cfg = p.RandomSketchConfig(target_rank=2, oversampling=3, power_iterations=0, seed=0)
    q = _np(p.randomized_range(a, cfg))
    assert q.shape == (30, 5)
    assert np.max(np.abs(q.T @ q - np.eye(5))) < 1e-12
    assert np.max(np.abs(a - q @ (q.T @ a))) < 1e-10
    b = _rng(16).standard_normal((2000, 60))
    for it in (0, 1, 2):
        cfg = p.RandomSketchConfig(target_rank=8, oversampling=4, power_iterations=it, seed=99)
        q = _np(p.randomized_range(b, cfg))
        ref = oracle.ref_range(b, 12, it, 99)
        assert np.max(np.abs(q - ref)) < 1e-10  # same basis: qr_factor's sign convention
    with pytest.raises(ValueError):
        p.randomized_range(np.eye(4), p.RandomSketchConfig(target_rank=3, oversampling=2))


def test_low_rank_svd_vt_matches_reference():
    p = _p()
    rng = _rng(17)
    u0 = oracle.ref_qr(rng.standard_normal((40, 3)))[0]
    v0 = oracle.ref_qr(rng.standard_normal((15, 3)))[0]
    a = (u0 * [7.0, 4.0, 2.0]) @ v0.T
    res = p.low_rank_svd(a, p.RandomSketchConfig(target_rank=3, oversampling=5, power_iterations=1, seed=1))
    assert np.allclose(_np(res.s), [7.0, 4.0, 2.0], rtol=1e-10)
    assert np.max(np.abs((_np(res.u) * _np(res.s)) @ _np(res.vt) - a)) < 1e-9
    b = oracle.burgers_matrix(4096, 300)
    res = p.low_rank_svd(b, p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=1, seed=3))
    ru, rs, rvt = oracle.ref_low_rank_svd(b, 10, 10, 1, 3)
    assert oracle.sigma_rel_err(_np(res.s), rs) < 1e-10
    assert np.max(oracle.mode_angles(_np(res.vt).T, rvt.T)) < 1e-8
    assert np.all(np.sum(_np(res.vt) * rvt, axis=1) > 0)  # rows signed like the reference's


# ---------------------------------------------------------------- parallel_qr

def _qr_rank_worker(rank, world, port, q, rows, cols, seed):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_08845_b200 as p
        a = np.random.Generator(np.random.Philox(seed)).standard_normal((rows, cols))
        lo, hi = p.partition_bounds(rows, world)[rank]
        res = p.parallel_qr(p.RankContext(), a[lo:hi])
        q.put((rank, res.q.cpu().numpy(), res.r.cpu().numpy()))
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols", [(4, 32, 5), (3, 9, 5), (2, 20000, 30), (4, 40000, 210)])
def test_parallel_qr_ranks_match_serial(world, rows, cols):
    """Four ranks of 8 rows, three of 3 rows (shorter than the 5 columns: dsvd.py's short
    blocks), two of 10000: same R on every rank, stacked Q orthonormal, factors equal to
    the serial qr_factor's (test_dsvd.py:174-211)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_qr_rank_worker, args=(r, world, port, q, rows, cols, 66)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(world):
        rank, qq, rr = q.get(timeout=300)
        assert not (isinstance(qq, str) and qq == "error"), rr
        out[rank] = (qq, rr)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    r = out[0][1]
    for rank in range(1, world):
        assert np.array_equal(out[rank][1], r)
    a = np.random.Generator(np.random.Philox(66)).standard_normal((rows, cols))
    qfull = np.concatenate([out[k][0] for k in range(world)], axis=0)
    assert np.max(np.abs(qfull.T @ qfull - np.eye(cols))) < 1e-12
    assert np.max(np.abs(qfull @ r - a)) < 1e-12 * np.sqrt(rows)
    qs, rs = oracle.ref_qr(a)
    assert np.max(np.abs(r - rs)) < 1e-10 * max(1.0, np.abs(rs).max())
    assert np.max(np.abs(qfull - qs)) < 1e-10


def test_parallel_qr_world_one_is_qr_factor():
    p = _p()
    a = _rng(65).standard_normal((20, 6))
    serial = p.qr_factor(a)
    par = p.parallel_qr(p.RankContext(), a)
    assert torch.equal(par.q, serial.q) and torch.equal(par.r, serial.r)


def test_kernel_invariants_1000_matrices():
    """test_acceptance.py:226-261 on the device: 1000 seeded matrices, every dimension up to 32;
    QR and SVD post-conditions and agreement with the Gram-eigenvalue route."""
    import time
    p = _p()
    t0 = time.perf_counter()
    worst = 0.0
    for seed in range(1000):
        rng = np.random.Generator(np.random.Philox(seed))
        rows, cols = (int(x) for x in rng.integers(1, 33, size=2))
        a = rng.standard_normal((rows, cols))
        qr = p.qr_factor(a)
        q, r = _np(qr.q), _np(qr.r)
        assert np.max(np.abs(q.T @ q - np.eye(min(rows, cols)))) <= 1e-13 * max(rows, cols)
        assert np.max(np.abs(q @ r - a)) <= 1e-12 * (1 + np.max(np.abs(a)))
        assert np.all(np.diag(r) >= 0)
        res = p.svd_full(a)
        u, s, vt = _np(res.u), _np(res.s), _np(res.vt)
        assert np.all(s >= 0) and np.all(np.diff(s) <= 0)
        assert np.max(np.abs((u * s) @ vt - a)) <= 1e-12 * (1 + s[0])
        gram = a.T @ a if cols <= rows else a @ a.T
        ref = np.sqrt(np.clip(np.linalg.eigvalsh(gram)[::-1], 0.0, None))
        worst = max(worst, float(np.max(np.abs(ref - s)) / (1 + s[0])))
    assert worst <= 1e-9
    assert time.perf_counter() - t0 < 120.0


@pytest.mark.parametrize("m,n,kind", [(65, 48, "deficient"), (86, 48, "deficient"), (74, 64, "steep"),
                                      (3000, 200, "deficient"), (500, 300, "steep")])
def test_svd_weak_directions_keep_u_orthonormal(m, n, kind):
    """Rank-deficient and steep inputs (found by tools/fuzz_linalg.py): u_j = a v_j / s_j is undefined for
    s_j = 0 and orthogonal only to eps s_1 / s_j otherwise, while the reference's dgesdd returns orthonormal
    factors whatever the spectrum (linalg.py:107-123).  The factors stay orthonormal, reconstruct a, and the
    values above 1e-5 s_1 keep their relative accuracy."""
    rng = _rng(300 + m + n)
    r = n // 2 if kind == "deficient" else n
    u0 = oracle.ref_qr(rng.standard_normal((m, r)))[0]
    v0 = oracle.ref_qr(rng.standard_normal((n, r)))[0]
    span = 1e-3 if kind == "deficient" else 1e-12
    a = (u0 * span ** (np.arange(r) / (r - 1))) @ v0.T
    res = _p().svd_full(a)
    u, s, vt = _np(res.u), _np(res.s), _np(res.vt)
    _, rs, _ = oracle.ref_svd(a)
    assert np.max(np.abs(u.T @ u - np.eye(n))) < 1e-10 and np.max(np.abs(vt @ vt.T - np.eye(n))) < 1e-10
    assert np.max(np.abs((u * s) @ vt - a)) < 1e-11 * np.abs(a).max()
    assert np.all(np.diff(s) <= 0) and np.max(np.abs(s - rs)) < 1e-12 * rs[0]
    big = rs > 1e-5 * rs[0]
    assert np.max(np.abs(s[big] - rs[big]) / rs[big]) < 1e-10


@pytest.mark.parametrize("m,n,span", [(120, 100, 1e-80), (512, 200, 1e-80), (512, 200, 1e-150), (700, 300, 1e-30),
                                      (40, 60, 1e-40)])
def test_svd_graded_columns_converge(m, n, span):
    """Columns graded over tens of orders, the small ones first (found through the Burgers rows near x = 1,
    whose early snapshots are ~1e-80): the reference's dgesdd converges on any finite input
    (linalg.py:107-123); ours sorts the columns by norm and takes the QR of the unit-norm columns
    (linalg._svd_tall) instead of stalling in the Jacobi sweeps.  Values to LAPACK's absolute accuracy,
    orthonormal factors, reconstruction to eps n s_1."""
    p = _p()
    x = _rng(5).standard_normal((m, n)) * span ** (np.arange(n)[::-1] / (n - 1))
    u, s, vt = (t.cpu().numpy() for t in p.svd_full(x))
    rs = np.linalg.svd(x, compute_uv=False)
    k = min(m, n)
    assert np.max(np.abs(s - rs)) <= 1e-13 * rs[0] and np.all(np.diff(s) <= 0)
    assert np.max(np.abs(u.T @ u - np.eye(k))) <= 1e-12 and np.max(np.abs(vt @ vt.T - np.eye(k))) <= 1e-12
    assert np.max(np.abs((u * s) @ vt - x)) <= 1e-12 * rs[0]   # ~ eps n s_1


@pytest.mark.parametrize("rows", [300, 512, 2048])
def test_svd_burgers_tail_rows(rows):
    """The grid rows nearest x = 1 (the block the last rank of a row partition holds): the leading
    values at the bar against the reference, the whole spectrum to 1e-13 s_1."""
    p = _p()
    x = oracle.burgers_matrix(8192 if rows == 2048 else 2048, 800 if rows == 2048 else 200)[-rows:]
    res = p.svd_full(x, want_vt=False)
    u, s = res.u.cpu().numpy(), res.s.cpu().numpy()
    ru, rs, _ = oracle.ref_svd(x, want_vt=False)
    assert np.max(np.abs(s - rs)) <= 1e-13 * rs[0]
    lead = rs >= 1e-5 * rs[0]
    assert np.max(np.abs(s[lead] - rs[lead]) / rs[lead]) <= 1e-10
    assert np.max(np.abs(u.T @ u - np.eye(u.shape[1]))) <= 1e-12


@pytest.mark.parametrize("m,n,span,up", [(300, 40, 1e-12, True), (5000, 150, 1e-30, True), (2000, 300, 1e-80, False),
                                         (64, 64, 1e-20, True), (30, 50, 1e-20, True)])
def test_qr_graded_columns_match_reference(m, n, span, up):
    """Column norms spanning up to 1e80 (either order): the factorization of the unit-norm columns with R
    scaled back (linalg._equilibrated_tall_qr) reproduces the reference's Householder q to rounding and every
    column of r relative to that column's own norm (linalg.py:94-104), not just the rows with large pivots."""
    p = _p()
    d = span ** (np.arange(n) / (n - 1))
    x = _rng(3).standard_normal((m, n)) * (d[::-1] if up else d)
    res = p.qr_factor(x)
    q, r = res.q.cpu().numpy(), res.r.cpu().numpy()
    q0, r0 = oracle.ref_qr(x)
    cn = np.linalg.norm(x, axis=0)
    k = min(m, n)
    assert np.max(np.abs(q.T @ q - np.eye(k))) <= 1e-13
    assert np.max(np.abs(q - q0)) <= 1e-12
    assert np.max(np.abs(r - r0) / cn[None, :]) <= 1e-12
    assert np.max(np.abs(q @ r - x) / cn[None, :]) <= 1e-13
    assert np.all(np.diag(r) >= 0)
