"""GPU parity at the benchmark's own size (VERDICT r1 "do this" #1).

BASELINE config 2 — Burgers 2^20 x 800, B = 200, K = 10, ff = 0.95 — streamed
through the public `stream_all` (the same call bench.py times) and through the
pinned CPU oracle (oracle/core.py, the reference's algorithm on numpy LAPACK) on
the SAME host bytes: the deterministic path and the randomized composition R9 at
q = 0 and q = 1 (p = 10, seed 0, the host Philox Omega of linalg.py:141-142).
Config 3 (weather field, 1,038,240 x 1024, B = 256, K = 50, p = 10, q = 1) at
its full row count on the wide randomized route.

Bars (north_star): sigma relative error <= 1e-10 at every step, per-mode
sine-based angles <= 1e-8 for well-separated modes, the reference's column
signs.  The oracle run on this box is itself pinned at full size by
fingerprints the live reference wrote (tests/golden/make_fullsize.py:
singular-value histories, signed probe rows, peak rows).

The serial oracle may use every host core (SURVEY F4 is about simulated ranks),
so these tests lift the session's one-thread BLAS pin.
"""

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

import oracle

pytestmark = pytest.mark.gpu

SIG_TOL = 1e-10
ANG_TOL = 1e-8
C2_ROWS = 1 << 20


def _pkg():
    import paper_2108_08845_b200 as p
    return p


def _fp(golden):
    try:
        return golden("fullsize_fingerprints")
    except FileNotFoundError:
        pytest.skip("tests/golden/fullsize_fingerprints.npz not generated")


@pytest.fixture(scope="module")
def config2():
    """Config-2 host bytes: burgers_matrix row slices generated on every core into one
    C-ordered matrix (as the reference generates it), plus F-ordered copies of the
    200-column batches for the device (what BatchSource / a PARSVD01 file delivers)."""
    a = np.empty((C2_ROWS, 800))
    edges = np.linspace(0, C2_ROWS, 65).astype(np.int64)

    def fill(i):
        lo, hi = int(edges[i]), int(edges[i + 1])
        a[lo:hi] = oracle.burgers_matrix(C2_ROWS, 800, rows=(lo, hi))

    with ThreadPoolExecutor(os.cpu_count()) as ex:
        list(ex.map(fill, range(64)))
    host = [a[:, c:c + 200] for c in range(0, 800, 200)]
    dev = [np.asfortranarray(b) for b in host]
    return host, dev


def _well_separated(sigma, rel_gap=1e-3):
    """Modes whose relative gap to both neighbours is >= rel_gap (north_star: angles
    are required for well-separated modes)."""
    s = np.asarray(sigma)
    k = s.size
    ok = np.ones(k, dtype=bool)
    for j in range(k):
        for i in (j - 1, j + 1):
            if 0 <= i < k and abs(s[i] - s[j]) < rel_gap * s[j]:
                ok[j] = False
    return ok


def _check(modes, sigma, hist, ref_modes, ref_sigma, ref_hist, sep=None):
    assert oracle.sigma_rel_err(sigma, ref_sigma) <= SIG_TOL
    for h, rh in zip(hist, ref_hist):
        assert oracle.sigma_rel_err(np.asarray(h), rh) <= SIG_TOL
    ang = oracle.mode_angles(modes, ref_modes)
    sel = np.ones(ang.size, dtype=bool) if sep is None else sep
    assert sel.any()
    assert np.max(ang[sel]) <= ANG_TOL, ang
    assert np.all(np.sum(modes * ref_modes, axis=0)[sel] > 0)  # the reference's signs
    gram = modes.T @ modes
    assert np.max(np.abs(gram - np.eye(gram.shape[0]))) < 1e-12
    return float(np.max(ang[sel]))


def _check_fingerprint(fp, prefix, modes, sigma, hist):
    """The live reference's own full-size run (fingerprint) vs a result."""
    assert oracle.sigma_rel_err(sigma, fp[prefix + "_sigma"]) <= SIG_TOL
    for h, rh in zip(hist, fp[prefix + "_history"]):
        assert oracle.sigma_rel_err(np.asarray(h), rh) <= SIG_TOL
    rows = fp[prefix + "_probe_rows"]
    scale = np.max(np.abs(fp[prefix + "_probe"]), axis=0)
    assert np.max(np.abs(modes[rows, :] - fp[prefix + "_probe"]) / scale) <= 1e-7
    assert np.array_equal(np.argmax(np.abs(modes), axis=0), fp[prefix + "_peak_row"])


def test_config2_deterministic_fullsize(config2, golden):
    p = _pkg()
    host, dev = config2
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)
    t0 = time.perf_counter()
    st, hist = p.stream_all(dev, cfg)
    modes, sigma = st.numpy()
    t_gpu = time.perf_counter() - t0
    hist = [h.cpu().numpy() for h in hist]
    t0 = time.perf_counter()
    with threadpool_limits(os.cpu_count()):
        ref_m, ref_s, ref_h = oracle.ref_stream_all(host, 10, 0.95)
    t_cpu = time.perf_counter() - t0
    ang = _check(modes, sigma, hist, ref_m, ref_s, ref_h)
    print(f"config2 det full size: gpu {t_gpu:.2f} s (incl. upload), oracle {t_cpu:.1f} s, "
          f"sigma {oracle.sigma_rel_err(sigma, ref_s):.2e}, angle {ang:.2e}")
    fp = _fp(golden)
    _check_fingerprint(fp, "c2_det", ref_m, ref_s, ref_h)   # the oracle at full size = the live reference
    _check_fingerprint(fp, "c2_det", modes, sigma, hist)


@pytest.mark.parametrize("q", [0, 1])
def test_config2_randomized_fullsize(config2, golden, q):
    p = _pkg()
    host, dev = config2
    sk = p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=q, seed=0)
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200, sketch=sk)
    st, hist = p.stream_all(dev, cfg)
    modes, sigma = st.numpy()
    hist = [h.cpu().numpy() for h in hist]
    with threadpool_limits(os.cpu_count()):
        ref_m, ref_s, ref_h = oracle.ref_rand_stream_all(host, 10, 0.95, 10, q, 0)
    ang = _check(modes, sigma, hist, ref_m, ref_s, ref_h)
    print(f"config2 q{q} full size: sigma {oracle.sigma_rel_err(sigma, ref_s):.2e}, angle {ang:.2e}")
    fp = _fp(golden)
    _check_fingerprint(fp, f"c2_q{q}", ref_m, ref_s, ref_h)
    _check_fingerprint(fp, f"c2_q{q}", modes, sigma, hist)


def test_config3_randomized_fullsize(golden):
    """Config 3 at its full 1,038,240 rows: K = 50, B = 256, p = 10, q = 1 (the wide
    randomized route: l = 60)."""
    p = _pkg()
    from paper_2108_08845_b200.datagen import weather_matrix
    with threadpool_limits(os.cpu_count()):
        a = weather_matrix()
    host = [a[:, c:c + 256] for c in range(0, 1024, 256)]
    sk = p.RandomSketchConfig(target_rank=50, oversampling=10, power_iterations=1, seed=0)
    cfg = p.StreamConfig(k_modes=50, forget_factor=0.95, batch_columns=256, sketch=sk)
    st, hist = p.stream_all(host, cfg)
    modes, sigma = st.numpy()
    hist = [h.cpu().numpy() for h in hist]
    with threadpool_limits(os.cpu_count()):
        ref_m, ref_s, ref_h = oracle.ref_rand_stream_all(host, 50, 0.95, 10, 1, 0)
    sep = _well_separated(ref_s)
    ang = _check(modes, sigma, hist, ref_m, ref_s, ref_h, sep=sep)
    print(f"config3 q1 full size: sigma {oracle.sigma_rel_err(sigma, ref_s):.2e}, angle {ang:.2e} "
          f"over {int(sep.sum())}/50 separated modes")
    fp = _fp(golden)
    assert oracle.sigma_rel_err(ref_s, fp["c3_q1_sigma"]) <= SIG_TOL
    assert oracle.sigma_rel_err(sigma, fp["c3_q1_sigma"]) <= SIG_TOL
