"""Generate the golden fixtures from the LIVE reference package.

Runs only in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports the unmodified reference (`parsvd` from /root/reference/pkg/src),
runs its own public functions on seeded inputs and writes inputs (or their
generator parameters + a SHA-256 of the bytes) and outputs to
tests/golden/*.npz.  BLAS is pinned to one thread so the vectors
are reproducible.  The fixtures travel to the GPU box; the reference does not.
"""

import hashlib
import os
import sys

import numpy as np
from threadpoolctl import threadpool_limits

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main():
    sys.path.insert(0, REF_SRC)
    import parsvd
    from parsvd.comm import run_simulated
    from parsvd.datagen import BurgersConfig, burgers_matrix, row_partition, synthetic_spectrum_matrix
    from parsvd.dsvd import gather_modes, parallel_stream_incorporate, parallel_stream_initialize
    from parsvd.linalg import RandomSketchConfig, low_rank_svd, qr_factor
    from parsvd.streaming import StreamConfig, StreamState, stream_all, stream_incorporate, stream_initialize

    def batches_of(a, w):
        return [a[:, i:i + w] for i in range(0, a.shape[1], w)]

    def save(name, **arrs):
        path = os.path.join(OUT, name + ".npz")
        np.savez_compressed(path, **arrs)
        print(f"wrote {path} ({os.path.getsize(path)} B)")

    # ---- G1: BASELINE config 1 exactly (Burgers 4096x800, B=200, K=10, ff=1) ----
    a = burgers_matrix(BurgersConfig(grid_points=4096, n_snapshots=800))
    cfg = StreamConfig(k_modes=10, forget_factor=1.0, batch_columns=200)
    state, hist = stream_all(batches_of(a, 200), cfg)
    save("det_burgers4096", grid=4096, snaps=800, k=10, ff=1.0, batch=200,
         input_sha=sha(a), input_probe_idx=np.array([[0, 0], [1, 1], [2047, 399], [4095, 799], [123, 456]]),
         input_probe=np.array([a[0, 0], a[1, 1], a[2047, 399], a[4095, 799], a[123, 456]]),
         modes=state.modes, sigma=state.singular_values, history=np.array(hist))

    # ---- G2: Gaussian stream, ff<1, variable last batch, init+4 updates ----
    rng = np.random.Generator(np.random.Philox(101))
    a = rng.standard_normal((300, 58))
    cfg = StreamConfig(k_modes=6, forget_factor=0.95, batch_columns=12)
    state, hist = stream_all(batches_of(a, 12), cfg)
    save("det_gauss300", a=a, k=6, ff=0.95, batch=12, modes=state.modes,
         sigma=state.singular_values, history=np.array(hist))

    # ---- G3: small / edge cases through the reference update ----
    cases = {}
    st = stream_initialize(np.diag([3.0, 2.0, 1.0]), StreamConfig(k_modes=3, batch_columns=3))
    cases["diag3_modes"], cases["diag3_sigma"] = st.modes, st.singular_values
    sv = np.concatenate([1.25 ** -np.arange(5), 1e-8 * 0.5 ** np.arange(12)])
    c = synthetic_spectrum_matrix(60, 36, sv, seed=11)
    cases["constructed_a"] = c
    st, h = stream_all(batches_of(c, 7), StreamConfig(k_modes=5, forget_factor=1.0, batch_columns=7))
    cases["constructed_w7_modes"], cases["constructed_w7_sigma"] = st.modes, st.singular_values
    r3 = synthetic_spectrum_matrix(40, 24, [4.0, 2.0, 1.0], seed=12)
    cases["rank3_a"] = r3
    st, _ = stream_all(batches_of(r3, 6), StreamConfig(k_modes=3, forget_factor=1.0, batch_columns=6))
    cases["rank3_modes"], cases["rank3_sigma"] = st.modes, st.singular_values
    rng = np.random.Generator(np.random.Philox(43))
    v0, v1, v2 = (rng.standard_normal((20, 5)), rng.standard_normal((20, 1)), rng.standard_normal((20, 9)))
    cfg = StreamConfig(k_modes=3, forget_factor=1.0, batch_columns=5)
    st = stream_incorporate(stream_incorporate(stream_initialize(v0, cfg), v1, cfg), v2, cfg)
    cases["varwidth_a0"], cases["varwidth_a1"], cases["varwidth_a2"] = v0, v1, v2
    cases["varwidth_modes"], cases["varwidth_sigma"] = st.modes, st.singular_values
    # rescue pass (streaming.py:106-115), input as in test_streaming.py:154-165
    rng = np.random.Generator(np.random.Philox(44))
    q = qr_factor(rng.standard_normal((30, 3))).q
    drifted = q + 1e-4 * rng.standard_normal((30, 3))
    batch = rng.standard_normal((30, 4))
    st = stream_incorporate(StreamState(drifted, np.array([3.0, 2.0, 1.0]), 0), batch,
                            StreamConfig(k_modes=3, forget_factor=1.0, batch_columns=4))
    cases["rescue_modes_in"], cases["rescue_batch"] = drifted, batch
    cases["rescue_modes"], cases["rescue_sigma"] = st.modes, st.singular_values
    save("det_edge_cases", **cases)

    # ---- G4: randomized composition R9 (Burgers 2048x800, B=200, K=10, p=10, ff=0.95) ----
    a = burgers_matrix(BurgersConfig(grid_points=2048, n_snapshots=800))
    out = dict(grid=2048, snaps=800, k=10, ff=0.95, batch=200, p=10, seed=0, input_sha=sha(a))
    for q_it in (0, 1):
        sk = RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=q_it, seed=0)
        u = s = None
        hist = []
        for b in batches_of(a, 200):
            m = b if u is None else np.concatenate([0.95 * (u * s), b], axis=1)
            res = low_rank_svd(m, sk)
            u, s = res.u, res.s
            hist.append(s.copy())
        out[f"q{q_it}_modes"], out[f"q{q_it}_sigma"], out[f"q{q_it}_history"] = u, s, np.array(hist)
    save("rand_burgers2048", **out)

    # ---- G5: low_rank_svd on small matrices (incl. exact low rank) ----
    rng = np.random.Generator(np.random.Philox(17))
    u0 = qr_factor(rng.standard_normal((40, 3))).q
    v0 = qr_factor(rng.standard_normal((15, 3))).q
    lr = (u0 * [7.0, 4.0, 2.0]) @ v0.T
    res = low_rank_svd(lr, RandomSketchConfig(target_rank=3, oversampling=5, power_iterations=1, seed=1))
    rng = np.random.Generator(np.random.Philox(16))
    g = rng.standard_normal((25, 10))
    res2 = low_rank_svd(g, RandomSketchConfig(target_rank=4, oversampling=2, power_iterations=0, seed=99))
    save("rand_small", lowrank_a=lr, lowrank_u=res.u, lowrank_s=res.s, gauss_a=g, gauss_u=res2.u,
         gauss_s=res2.s)

    # ---- G6: row-parallel streaming at 4 simulated ranks (Burgers 2048x800) ----
    a = burgers_matrix(BurgersConfig(grid_points=2048, n_snapshots=800))
    blocks = row_partition(a, 4)
    cfg = StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200)

    def program(ctx):
        blk = blocks[ctx.rank]
        st = parallel_stream_initialize(ctx, blk[:, :200], cfg)
        for c0 in range(200, 800, 200):
            st = parallel_stream_incorporate(ctx, st, blk[:, c0:c0 + 200], cfg)
        return gather_modes(ctx, st), st.singular_values

    modes, sig = run_simulated(4, program)[0]
    save("par_burgers2048_p4", grid=2048, snaps=800, k=10, ff=0.95, batch=200, world=4,
         input_sha=sha(a), modes=modes, sigma=sig)

    # ---- G7: apmos one-shot distributed SVD (dsvd.py:127-173, test_dsvd.py:73-133 shapes) ----
    from parsvd.dsvd import ApmosConfig, apmos
    out = {}
    rng = np.random.Generator(np.random.Philox(42))
    g = rng.standard_normal((64, 16))
    out["gauss_a"] = g
    for world, (r1, r2, k) in ((1, (16, 16, 5)), (4, (16, 16, 5)), (4, (6, 8, 4)), (3, (10, 12, 6))):
        blocks = row_partition(g, world)
        cfg_a = ApmosConfig(local_rank=r1, global_rank=r2, k_modes=k)
        modes, sig = run_simulated(world, lambda ctx: (gather_modes(ctx, apmos(ctx, blocks[ctx.rank], cfg_a)),
                                                       None))[0][0], None
        loc = run_simulated(world, lambda ctx: apmos(ctx, blocks[ctx.rank], cfg_a))[0]
        out[f"gauss_p{world}_r{r1}_{r2}_{k}_modes"] = modes
        out[f"gauss_p{world}_r{r1}_{r2}_{k}_sigma"] = loc.singular_values
    c = synthetic_spectrum_matrix(48, 12, 2.0 ** -np.arange(6), seed=64)
    out["spec_a"] = c
    blocks = row_partition(c, 3)
    sk = RandomSketchConfig(target_rank=6, oversampling=6, power_iterations=2, seed=9)
    cfg_a = ApmosConfig(local_rank=12, global_rank=6, k_modes=3, use_randomized=True, sketch=sk)
    out["spec_rand_modes"] = run_simulated(3, lambda ctx: gather_modes(ctx, apmos(ctx, blocks[ctx.rank], cfg_a)))[0]
    out["spec_rand_sigma"] = run_simulated(3, lambda ctx: apmos(ctx, blocks[ctx.rank], cfg_a))[0].singular_values
    a = burgers_matrix(BurgersConfig(grid_points=2048, n_snapshots=200))
    out["burgers_sha"] = sha(a)
    blocks = row_partition(a, 4)
    cfg_a = ApmosConfig(local_rank=40, global_rank=30, k_modes=10)
    out["burgers_p4_modes"] = run_simulated(4, lambda ctx: gather_modes(ctx, apmos(ctx, blocks[ctx.rank], cfg_a)))[0]
    out["burgers_p4_sigma"] = run_simulated(4, lambda ctx: apmos(ctx, blocks[ctx.rank], cfg_a))[0].singular_values
    save("apmos_cases", **out)

    # ---- G8: a PARSVD01 matrix file written by the reference (io.py:27-32) ----
    from parsvd.io import write_matrix
    rng = np.random.Generator(np.random.Philox(77))
    write_matrix(os.path.join(OUT, "sample_37x11.parsvd"), rng.standard_normal((37, 11)))
    print("wrote sample_37x11.parsvd")

    outputs()

    with open(os.path.join(OUT, "PROVENANCE.txt"), "w") as f:
        f.write("generated by tests/golden/make_golden.py from the live reference parsvd "
                f"{parsvd.__version__} at {REF_SRC}\n")
        f.write(f"numpy {np.__version__}; BLAS pinned to 1 thread (threadpoolctl)\n")


def outputs():
    """G9: the reference's text emitters (io.py:156-270) on seeded inputs: sigma / modes /
    history CSV (17 significant digits) and the mode SVG, byte for byte."""
    sys.path.insert(0, REF_SRC)
    from parsvd.io import write_history_csv, write_mode_svg, write_modes_csv, write_singular_values_csv
    rng = np.random.Generator(np.random.Philox(78))
    grid = np.linspace(0.0, 1.0, 33)
    modes = rng.standard_normal((33, 4))
    sigma = np.sort(np.abs(rng.standard_normal(6)))[::-1] * 1e3
    hist = np.abs(rng.standard_normal((5, 3)))
    write_singular_values_csv(os.path.join(OUT, "out_sigma.csv"), sigma)
    write_modes_csv(os.path.join(OUT, "out_modes.csv"), grid, modes)
    write_history_csv(os.path.join(OUT, "out_history.csv"), hist)
    write_mode_svg(os.path.join(OUT, "out_modes.svg"), grid, modes[:, :3])
    write_mode_svg(os.path.join(OUT, "out_flat.svg"), np.arange(5.0), np.ones((5, 2)))
    print("wrote out_sigma.csv out_modes.csv out_history.csv out_modes.svg out_flat.svg")


if __name__ == "__main__":
    with threadpool_limits(1):
        if len(sys.argv) > 1 and sys.argv[1] == "--outputs-only":
            outputs()
        else:
            main()
