"""Diagnostics: compare the fused pass's A_{b+1}^T Y tiles (PSVD_DUMP_FUSED dump) with numpy."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import oracle
from paper_2108_08845_b200 import streaming as S
M, B, nbt, K = 4096, 200, 3, 10
a = oracle.burgers_matrix(M, B * nbt)
cfg = S.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B)
S.stream_all([a[:, i * B:(i + 1) * B] for i in range(nbt)], cfg)
for b in range(nbt - 1):
    raw = open(f"{os.environ['PSVD_DUMP_FUSED']}_{b}.bin", "rb").read()
    NB, a0, yb, MM = np.frombuffer(raw[:16], dtype=np.int32)
    t = np.frombuffer(raw[16:16 + NB * NB * 1024 * 8], dtype=np.float64).reshape(NB, NB, 32, 32)
    off = 16 + NB * NB * 1024 * 8
    Y = np.frombuffer(raw[off:off + M * K * 8], dtype=np.float64).reshape(K, M).T
    U = np.frombuffer(raw[off + M * K * 8:off + 2 * M * K * 8], dtype=np.float64).reshape(K, M).T
    kc = 0 if b == 0 else K
    Wm = np.frombuffer(raw[off + 2 * M * K * 8:], dtype=np.float64).reshape(K, kc + B).T
    P = np.concatenate([U[:, :kc], a[:, b * B:(b + 1) * B]], axis=1)
    Yref = P @ Wm
    print("b", b, "Y err", np.abs(Y - Yref).max() / np.abs(Yref).max())
    A2 = a[:, (b + 1) * B:(b + 2) * B]
    ref = A2.T @ Y
    got = np.concatenate([t[a0 + i, yb, :, :K] for i in range((B + 31) // 32)], axis=0)[:B]
    err = np.abs(got - ref).max() / np.abs(ref).max()
    print("b", b, "NB", NB, "a0", a0, "yb", yb, "UA err", err, "YtY err",
          np.abs(t[yb, yb, :K, :K] - Y.T @ Y).max() / np.abs(Y.T @ Y).max())
    if err > 1e-12:
        d = np.abs(got - ref) / np.abs(ref).max()
        print("  bad rows", np.where(d.max(axis=1) > 1e-12)[0][:40], "bad cols", np.where(d.max(axis=0) > 1e-12)[0])
