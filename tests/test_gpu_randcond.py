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
