"""Pin the CPU oracle (oracle/core.py) to vectors from the live reference.

The fixtures in tests/golden/ were written by tests/golden/make_golden.py,
which ran the unmodified reference package.  These tests run on CPU only.
"""

import hashlib

import numpy as np
import pytest

import oracle


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _batches(a, w):
    return [a[:, i:i + w] for i in range(0, a.shape[1], w)]


def _close(got, want, tol=1e-13):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    assert np.max(np.abs(got - want)) <= tol * max(1.0, np.max(np.abs(want)))


def test_burgers_generator_bytes_match_reference(golden):
    g = golden("det_burgers4096")
    a = oracle.burgers_matrix(int(g["grid"]), int(g["snaps"]))
    assert _sha(a) == str(g["input_sha"])
    r = golden("rand_burgers2048")
    assert _sha(oracle.burgers_matrix(2048, 800)) == str(r["input_sha"])
    # row slices reproduce the same bytes as slicing the full matrix
    assert np.array_equal(oracle.burgers_matrix(4096, 800, rows=(100, 300)), a[100:300])


def test_config1_deterministic_stream(golden):
    g = golden("det_burgers4096")
    a = oracle.burgers_matrix(4096, 800)
    modes, sigma, hist = oracle.ref_stream_all(_batches(a, 200), 10, 1.0)
    _close(modes, g["modes"], 1e-12)
    _close(sigma, g["sigma"])
    _close(np.array(hist), g["history"])


def test_gaussian_stream_ff(golden):
    g = golden("det_gauss300")
    modes, sigma, hist = oracle.ref_stream_all(_batches(g["a"], int(g["batch"])), int(g["k"]),
                                              float(g["ff"]))
    _close(modes, g["modes"], 1e-12)
    _close(np.array(hist), g["history"])


def test_edge_cases(golden):
    g = golden("det_edge_cases")
    m, s = oracle.ref_stream_init(np.diag([3.0, 2.0, 1.0]), 3)
    assert np.array_equal(s, g["diag3_sigma"]) and np.array_equal(m, g["diag3_modes"])
    m, s, _ = oracle.ref_stream_all(_batches(g["constructed_a"], 7), 5, 1.0)
    _close(m, g["constructed_w7_modes"], 1e-12)
    _close(s, g["constructed_w7_sigma"])
    m, s, _ = oracle.ref_stream_all(_batches(g["rank3_a"], 6), 3, 1.0)
    _close(m, g["rank3_modes"], 1e-12)
    _close(s, g["rank3_sigma"])
    m, s = oracle.ref_stream_init(g["varwidth_a0"], 3)
    m, s = oracle.ref_stream_update(m, s, g["varwidth_a1"], 3, 1.0)
    m, s = oracle.ref_stream_update(m, s, g["varwidth_a2"], 3, 1.0)
    _close(m, g["varwidth_modes"], 1e-12)
    m, s = oracle.ref_stream_update(g["rescue_modes_in"], np.array([3.0, 2.0, 1.0]),
                                    g["rescue_batch"], 3, 1.0)
    _close(m, g["rescue_modes"], 1e-12)
    _close(s, g["rescue_sigma"])


@pytest.mark.parametrize("q", [0, 1])
def test_randomized_composition(golden, q):
    g = golden("rand_burgers2048")
    a = oracle.burgers_matrix(2048, 800)
    modes, sigma, hist = oracle.ref_rand_stream_all(_batches(a, 200), 10, 0.95, 10, q, 0)
    _close(modes, g[f"q{q}_modes"], 1e-11)
    _close(np.array(hist), g[f"q{q}_history"], 1e-12)


def test_low_rank_small(golden):
    g = golden("rand_small")
    u, s, _ = oracle.ref_low_rank_svd(g["lowrank_a"], 3, 5, 1, 1)
    _close(u, g["lowrank_u"], 1e-12)
    _close(s, g["lowrank_s"])
    u, s, _ = oracle.ref_low_rank_svd(g["gauss_a"], 4, 2, 0, 99)
    _close(u, g["gauss_u"], 1e-12)


def test_parallel_stream_four_ranks(golden):
    g = golden("par_burgers2048_p4")
    a = oracle.burgers_matrix(2048, 800)
    edges = [(c, c + 200) for c in range(0, 800, 200)]
    modes, sigma = oracle.ref_parallel_stream_all(a, edges, 4, 10, 0.95)
    _close(modes, g["modes"], 1e-12)
    _close(sigma, g["sigma"])


def test_partition_bounds():
    assert oracle.partition_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert oracle.partition_bounds(8, 8) == [(i, i + 1) for i in range(8)]
    with pytest.raises(ValueError):
        oracle.partition_bounds(3, 4)


def test_metrics_resolve_tiny_angles():
    rng = np.random.default_rng(0)
    u = np.linalg.qr(rng.standard_normal((100, 3)))[0]
    v = u + 1e-12 * rng.standard_normal(u.shape)
    ang = oracle.mode_angles(u, -v)
    assert np.all(ang < 1e-10) and np.all(ang > 0)


def _blocks(a, world):
    return [a[lo:hi] for lo, hi in oracle.partition_bounds(a.shape[0], world)]


def test_apmos_oracle_matches_reference(golden):
    g = golden("apmos_cases")
    a = g["gauss_a"]
    for world, (r1, r2, k) in ((1, (16, 16, 5)), (4, (16, 16, 5)), (4, (6, 8, 4)), (3, (10, 12, 6))):
        m, s = oracle.ref_apmos(_blocks(a, world), r1, r2, k)
        tag = f"gauss_p{world}_r{r1}_{r2}_{k}"
        assert oracle.sigma_rel_err(s, g[tag + "_sigma"]) <= 1e-12
        assert np.max(oracle.mode_angles(m, g[tag + "_modes"])) <= 1e-10
        assert np.max(oracle.aligned_mode_difference(m, g[tag + "_modes"])) <= 1e-10
    m, s = oracle.ref_apmos(_blocks(g["spec_a"], 3), 12, 6, 3, use_randomized=True, sketch=(6, 6, 2, 9))
    assert oracle.sigma_rel_err(s, g["spec_rand_sigma"]) <= 1e-12
    assert np.max(oracle.mode_angles(m, g["spec_rand_modes"])) <= 1e-10
    b = oracle.burgers_matrix(2048, 200)
    m, s = oracle.ref_apmos(_blocks(b, 4), 40, 30, 10)
    assert oracle.sigma_rel_err(s, g["burgers_p4_sigma"]) <= 1e-12
    assert np.max(oracle.mode_angles(m, g["burgers_p4_modes"])) <= 1e-9
