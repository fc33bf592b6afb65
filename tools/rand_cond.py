"""Parity of the randomized stream against the oracle as the sketch's spectrum steepens (sigma_l / sigma_1 = span):
the fast path's Gram-based orthonormalization is exact to the bar down to ~1e-6; below, the device reports
PSVD_ST_SKETCHCOND and the update is redone on the accurate route (linalg.accurate_randomized_update)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import linalg
rng = np.random.Generator(np.random.Philox(7))
M, n, r, K, pov = 4096, 200, 40, 10, 10
U, _ = np.linalg.qr(rng.standard_normal((M, r)))
V, _ = np.linalg.qr(rng.standard_normal((n, r)))
for span in [1e-3, 1e-5, 1e-6, 1e-7, 1e-8, 1e-10, 1e-13]:
    c = span ** (1.0 / 19)
    a = (U * c ** np.arange(r)) @ V.T
    for q in (0, 1):
        sk = p.RandomSketchConfig(target_rank=K, oversampling=pov, power_iterations=q, seed=0)
        cfg = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=n, sketch=sk)
        b2 = [np.asfortranarray(a), np.asfortranarray(a[:, ::-1] * 0.5 + 0.1 * a)]
        ref_m, ref_s, _ = oracle.ref_rand_stream_all(b2, K, 0.95, pov, q, 0)
        n0 = linalg.ACCURATE_RAND_UPDATES
        st, _ = p.stream_all(b2, cfg)
        m, s = st.numpy()
        ang = oracle.mode_angles(m, ref_m)
        print(f"span {span:.0e} q={q}: sigma err {oracle.sigma_rel_err(s, ref_s):.2e}  max angle {ang.max():.2e}  "
              f"accurate updates {linalg.ACCURATE_RAND_UPDATES - n0}")
