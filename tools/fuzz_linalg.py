"""Random shapes and conditionings through qr_factor / svd_full / low_rank_svd against the oracle, with the
guarantees any backward-stable factorization gives (orthonormality, reconstruction, diag(R) >= 0, relative accuracy
of the values above rounding level).  python tools/fuzz_linalg.py [seed] [count]"""
import os, random, sys
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2108_08845_b200 as p
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 40
random.seed(seed)
rng = np.random.Generator(np.random.Philox(seed))
eps = np.finfo(float).eps
worst = {}
def note(k, v):
    worst[k] = max(worst.get(k, 0.0), float(v))
for it in range(count):
    n = random.choice([random.randint(1, 40), random.randint(41, 230), random.randint(231, 420)])
    m = random.choice([n, n + random.randint(0, 50), random.randint(n, 6000)])
    kind = random.choice(["gauss", "decay", "steep", "deficient", "graded"])
    if kind == "gauss":
        a = rng.standard_normal((m, n))
    elif kind == "graded":   # column norms over up to 80 orders, either direction
        d = random.choice([1e-8, 1e-30, 1e-80]) ** (np.arange(n) / max(n - 1, 1))
        a = rng.standard_normal((m, n)) * (d if random.random() < 0.5 else d[::-1])
    else:
        r = n if kind != "deficient" else max(1, n // 2)
        u, _ = np.linalg.qr(rng.standard_normal((m, r)))
        v, _ = np.linalg.qr(rng.standard_normal((n, r)))
        span = {"decay": 1e-4, "steep": 1e-12, "deficient": 1e-3}[kind]
        sv = span ** (np.arange(r) / max(r - 1, 1))
        a = (u * sv) @ v.T
    tag = (m, n, kind)
    # qr_factor
    res = p.qr_factor(a)
    q, r_ = res.q.cpu().numpy(), res.r.cpu().numpy()
    k = min(m, n)
    amax = max(np.abs(a).max(), 1e-300)
    e_orth = np.max(np.abs(q.T @ q - np.eye(k)))
    e_rec = np.max(np.abs(q @ r_ - a)) / amax
    if e_orth > 1e-11 or e_rec > 1e-11 or not np.all(np.diag(r_) >= 0.0):
        print("FAIL qr", tag, e_orth, e_rec); sys.exit(1)
    note("qr orth", e_orth); note("qr rec", e_rec)
    # svd_full
    sres = p.svd_full(a)
    u_, s_, vt_ = sres.u.cpu().numpy(), sres.s.cpu().numpy(), sres.vt.cpu().numpy()
    ru, rs, rvt = oracle.ref_svd(a)
    # relative accuracy down to where the reference's own dgesdd stops (its values carry O(eps s_1) absolute error)
    big = rs > 1e-5 * rs[0]
    e_s = np.max(np.abs(s_[big] - rs[big]) / rs[big]) if big.any() else 0.0
    e_abs = np.max(np.abs(s_ - rs)) / rs[0]
    e_rec = np.max(np.abs((u_ * s_) @ vt_ - a)) / amax
    e_orth = max(np.max(np.abs(u_.T @ u_ - np.eye(k))), np.max(np.abs(vt_ @ vt_.T - np.eye(k))))
    if e_s > 1e-9 or e_abs > 1e-12 or e_rec > 1e-11 or e_orth > 1e-10 or np.any(np.diff(s_) > 0):
        print("FAIL svd", tag, e_s, e_abs, e_rec, e_orth)
        import os
        os.makedirs("gpurun_out", exist_ok=True)
        np.save("gpurun_out/fail_svd.npy", a)
        bad = np.argsort(-np.abs(s_ - rs))[:6]
        print("  worst values", bad, s_[bad], rs[bad]); sys.exit(1)
    note("svd rel", e_s); note("svd abs", e_abs); note("svd rec", e_rec); note("svd orth", e_orth)
    # low_rank_svd
    if min(m, n) >= 6:
        kk = random.randint(1, min(16, min(m, n) // 2))
        pov = random.randint(0, min(10, min(m, n) - kk))
        qit = random.randint(0, 2)
        sk = p.RandomSketchConfig(target_rank=kk, oversampling=pov, power_iterations=qit, seed=seed)
        if os.environ.get("FUZZ_NO_LR"):   # bisecting a sequence: same random draws, no low_rank_svd call
            continue
        lr = p.low_rank_svd(a, sk)
        lu, ls, lvt = oracle.ref_low_rank_svd(a, kk, pov, qit, seed)
        gs, gu = lr.s.cpu().numpy(), lr.u.cpu().numpy()
        sel = ls > 1e-7 * ls[0]
        e_ls = np.max(np.abs(gs[sel] - ls[sel]) / ls[sel])
        gaps = np.array([min([abs(ls[j] - ls[i]) for i in range(kk) if i != j] + [ls[j]]) / ls[j] for j in range(kk)])
        ok = sel & (gaps > 1e-3)
        e_la = float(np.max(oracle.mode_angles(gu, lu)[ok])) if ok.any() else 0.0
        if e_ls > 1e-9 or e_la > 1e-7:
            print("FAIL low_rank", tag, dict(k=kk, p=pov, q=qit), e_ls, e_la); sys.exit(1)
        note("lr sigma", e_ls); note("lr angle", e_la)
print(count, "cases ok:", {k: f"{v:.1e}" for k, v in worst.items()})
