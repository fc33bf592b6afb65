"""Configs 3-5 at reduced rows against the oracle (diagnostics before the parity tests)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import datagen as dg

def run(name, a, K, B, ff, sketch=None, q=1):
    batches = [a[:, i:i + B] for i in range(0, a.shape[1], B)]
    cfg = p.StreamConfig(k_modes=K, forget_factor=ff, batch_columns=B,
                         sketch=None if sketch is None else p.RandomSketchConfig(target_rank=K, oversampling=sketch, power_iterations=q, seed=0))
    t = time.time()
    try:
        st, hist = p.stream_all(batches, cfg)
        m, s = st.numpy()
    except Exception as e:
        print(name, "FAILED", type(e).__name__, e); return
    t1 = time.time() - t
    if sketch is None:
        rm, rs, _ = oracle.ref_stream_all(batches, K, ff)
    else:
        rm, rs, _ = oracle.ref_rand_stream_all(batches, K, ff, sketch, q, 0)
    ang = oracle.mode_angles(m, rm)
    gaps = np.minimum(np.abs(np.diff(np.r_[np.inf, rs])), np.abs(np.diff(np.r_[rs, 0.0]))) / rs
    print(name, f"gpu {t1:.2f}s sigma err {oracle.sigma_rel_err(s, rs):.2e} max angle {ang.max():.2e} "
          f"min gap {gaps.min():.2e} angle at gap>=1e-3 {ang[gaps >= 1e-3].max() if (gaps >= 1e-3).any() else 0:.2e}")

run("config5 det K=64 B=128", dg.stress_matrix(1 << 14, 512), 64, 128, 1.0)
run("config3 rand K=50 B=256 p=10", dg.weather_matrix(512, nlat=91, nlon=180), 50, 256, 0.95, sketch=10)
run("config4 rand K=100 B=512 p=10", dg.weak_scaling_matrix(1 << 13, 1024), 100, 512, 0.95, sketch=10)
