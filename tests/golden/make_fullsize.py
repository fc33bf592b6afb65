"""Full-size golden fingerprints from the LIVE reference (build container only).

    python tests/golden/make_fullsize.py          # ~10 min on 8 cores

BASELINE config 2 (Burgers 2^20 x 800, B = 200, K = 10, ff = 0.95) through the
reference's own `stream_all` (deterministic) and the randomized composition R9
(`low_rank_svd` of [ff U S | A_b], p = 10, q = 0 and 1, seed 0), and config 3
(the builder-defined weather field, 1,038,240 x 1024, B = 256, K = 50, p = 10,
q = 1) through the same composition.  The modes are 84-415 MB per case, too
large to commit, so the fixture holds the singular-value history of every step
plus a fingerprint of the final modes (the signed entries at 64 fixed probe rows
and each column's peak row, which pins the sign rule).  The full-size GPU tests
(tests/test_gpu_fullsize.py) compare against the pinned oracle run live on the
box on the same bytes, and against these fingerprints.

Serial reference functions only, so BLAS may use every core (SURVEY F4 concerns
simulated ranks).
"""

import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(OUT))


def probe_rows(m):
    return np.unique(np.linspace(0, m - 1, 64).round().astype(np.int64))


def fingerprint(prefix, modes, sigma, hist, out):
    rows = probe_rows(modes.shape[0])
    out[prefix + "_sigma"] = np.asarray(sigma)
    out[prefix + "_history"] = np.array(hist)
    out[prefix + "_probe_rows"] = rows
    out[prefix + "_probe"] = modes[rows, :]
    out[prefix + "_peak_row"] = np.argmax(np.abs(modes), axis=0)
    out[prefix + "_peak_val"] = modes[out[prefix + "_peak_row"], np.arange(modes.shape[1])]


def main(which):
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, ROOT)
    from parsvd.datagen import BurgersConfig, burgers_matrix
    from parsvd.linalg import RandomSketchConfig, low_rank_svd
    from parsvd.streaming import StreamConfig, stream_all

    path = os.path.join(OUT, "fullsize_fingerprints.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}

    def rand_stream(a, bw, k, p, q, ff):
        sk = RandomSketchConfig(target_rank=k, oversampling=p, power_iterations=q, seed=0)
        u = s = None
        hist = []
        for c0 in range(0, a.shape[1], bw):
            b = a[:, c0:c0 + bw]
            m = b if u is None else np.concatenate([ff * (u * s), b], axis=1)
            res = low_rank_svd(m, sk)
            u, s = res.u, res.s
            hist.append(s.copy())
        return u, s, hist

    if "c2" in which:
        t0 = time.time()
        a = burgers_matrix(BurgersConfig(grid_points=1 << 20, n_snapshots=800), max_bytes=1 << 34)
        print(f"config 2 input {time.time() - t0:.1f} s", flush=True)
        t0 = time.time()
        st, hist = stream_all([a[:, c:c + 200] for c in range(0, 800, 200)],
                              StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=200))
        fingerprint("c2_det", st.modes, st.singular_values, hist, out)
        print(f"config 2 det {time.time() - t0:.1f} s", flush=True)
        for q in (0, 1):
            t0 = time.time()
            u, s, hist = rand_stream(a, 200, 10, 10, q, 0.95)
            fingerprint(f"c2_q{q}", u, s, hist, out)
            print(f"config 2 q{q} {time.time() - t0:.1f} s", flush=True)
        del a
        np.savez_compressed(path, **out)
    if "c3" in which:
        from paper_2108_08845_b200.datagen import weather_matrix
        t0 = time.time()
        a = weather_matrix()
        print(f"config 3 input {time.time() - t0:.1f} s", flush=True)
        t0 = time.time()
        u, s, hist = rand_stream(a, 256, 50, 10, 1, 0.95)
        fingerprint("c3_q1", u, s, hist, out)
        print(f"config 3 q1 {time.time() - t0:.1f} s", flush=True)
        np.savez_compressed(path, **out)
    print(f"wrote {path}")


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3"])
