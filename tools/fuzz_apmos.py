"""Random shapes and spectra through the single-rank apmos (dsvd.py:39-173) against the oracle.
python tools/fuzz_apmos.py [seed] [count]"""
import random, sys
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2108_08845_b200 as p
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 30
random.seed(seed)
rng = np.random.Generator(np.random.Philox(seed))
ws = wa = 0.0
for it in range(count):
    n = random.randint(8, 220)
    m = random.choice([random.randint(n, 4000), 16 * random.randint(n // 16 + 1, 300)])
    kind = random.choice(["gauss", "decay", "steep"])
    if kind == "gauss":
        a = rng.standard_normal((m, n))
    else:
        u, _ = np.linalg.qr(rng.standard_normal((m, n)))
        v, _ = np.linalg.qr(rng.standard_normal((n, n)))
        span = 1e-4 if kind == "decay" else 1e-10
        a = (u * span ** (np.arange(n) / max(n - 1, 1))) @ v.T
    r1 = random.randint(2, min(n, 48))
    r2 = random.randint(1, r1)
    k = random.randint(1, r2)
    cfg = p.ApmosConfig(local_rank=r1, global_rank=r2, k_modes=k)
    loc = p.apmos(p.RankContext(), a, cfg)
    gm, gs = loc.modes.cpu().numpy(), loc.singular_values.cpu().numpy()
    rm, rs = oracle.ref_apmos([a], r1, r2, k)
    rm = rm[0] if isinstance(rm, (list, tuple)) else rm
    es = float(np.max(np.abs(gs - rs) / rs - 100 * np.finfo(float).eps * rs[0] / rs))
    gaps = np.array([min([abs(rs[j] - rs[i]) for i in range(k) if i != j] + [rs[j]]) / rs[j] for j in range(k)])
    sel = (gaps > 1e-3) & (rs > 1e-6 * rs[0])
    ea = float(np.max(oracle.mode_angles(gm, rm)[sel])) if sel.any() else 0.0
    ws, wa = max(ws, es), max(wa, ea)
    if es > 1e-10 or ea > 1e-8:
        print("FAIL", dict(m=m, n=n, kind=kind, r1=r1, r2=r2, k=k), es, ea); sys.exit(1)
print(f"{count} apmos cases ok: worst sigma excess {ws:.2e}, worst angle {wa:.2e}")
