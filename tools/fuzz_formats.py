"""The same batches in every container a caller may hand over (numpy C / Fortran order, strided and offset views,
float32 / integer dtypes, CPU / pinned / CUDA torch tensors, row-major and column-major, non-contiguous slices of a
larger device matrix) through stream_all / stream_incorporate / qr_factor / svd_full: results must equal the
Fortran-order float64 baseline bit for bit (same values reach the same kernels).  python tools/fuzz_formats.py [seed] [count]"""
import random, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 20
random.seed(seed)
rng = np.random.Generator(np.random.Philox(seed))
dev = torch.device("cuda", 0)


def forms(b):
    """(name, object) containers holding exactly b's float64 values."""
    M, n = b.shape
    big = np.zeros((M + 3, 2 * n + 5))
    big[1:M + 1, 3:3 + 2 * n:2] = b
    tb = torch.from_numpy(np.ascontiguousarray(b))
    cbig = torch.zeros((M + 2, n + 7), dtype=torch.float64, device=dev)
    cbig[2:, 4:4 + n] = tb.to(dev)
    fbig = torch.zeros((n + 7, M + 3), dtype=torch.float64, device=dev).T   # column-major parent, odd offset
    fbig[1:M + 1, 5:5 + n] = tb.to(dev)
    return [
        ("np C", np.ascontiguousarray(b)), ("np F", np.asfortranarray(b)), ("np strided view", big[1:M + 1, 3:3 + 2 * n:2]),
        ("list of lists", b.tolist()) if M * n < 20000 else ("np C again", b.copy()),
        ("torch cpu", tb), ("torch cpu F", torch.from_numpy(np.asfortranarray(b).T).T), ("torch pinned", tb.pin_memory()),
        ("cuda C", tb.to(dev)), ("cuda F", tb.to(dev).T.contiguous().T), ("cuda C slice", cbig[2:, 4:4 + n]),
        ("cuda F slice, odd offset", fbig[1:M + 1, 5:5 + n]),
    ]


def same(x, y):
    return all(np.array_equal(a.cpu().numpy(), b.cpu().numpy()) for a, b in zip(x, y))


for it in range(count):
    M = random.choice([random.randint(3, 60), random.randint(61, 3000), 16 * random.randint(10, 200)])
    K = random.randint(1, min(12, M))
    w = [random.randint(K, K + 40) for _ in range(3)]
    a = rng.standard_normal((M, sum(w)))
    if random.random() < 0.5:
        a = np.round(a * 8) / 8    # exactly representable in float32 too
    batches = [a[:, sum(w[:i]):sum(w[:i + 1])] for i in range(3)]
    cfg = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=w[0])
    base, _ = p.stream_all([np.asfortranarray(b) for b in batches], cfg)
    base_q = p.qr_factor(np.asfortranarray(batches[0])) if M >= w[0] else None
    names = [n for n, _ in forms(batches[0])]
    for j, name in enumerate(names):
        bs = [forms(b)[j][1] for b in batches]
        st, _ = p.stream_all(bs, cfg)
        if not same((st.modes, st.singular_values), (base.modes, base.singular_values)):
            print("FAIL stream_all", name, dict(M=M, K=K, w=w))
            sys.exit(1)
        s2 = p.stream_initialize(bs[0], cfg)
        for b in bs[1:]:
            s2 = p.stream_incorporate(s2, b, cfg)
        if j == 0:
            base2 = s2
        elif not same((s2.modes, s2.singular_values), (base2.modes, base2.singular_values)):
            print("FAIL per-update", name, dict(M=M, K=K, w=w))
            sys.exit(1)
        if base_q is not None and not same(p.qr_factor(bs[0]), base_q):
            print("FAIL qr_factor", name, dict(M=M, K=K, w=w))
            sys.exit(1)
    if np.array_equal(a, a.astype(np.float32)):
        st, _ = p.stream_all([b.astype(np.float32) for b in batches], cfg)
        st3, _ = p.stream_all([torch.from_numpy(b.astype(np.float32)).to(dev) for b in batches], cfg)
        if not same((st.modes,), (base.modes,)) or not same((st3.modes,), (base.modes,)):
            print("FAIL float32", dict(M=M, K=K, w=w))
            sys.exit(1)
print(f"{count} cases x {len(names)} containers ok (bitwise equal to the Fortran-order float64 baseline)")
