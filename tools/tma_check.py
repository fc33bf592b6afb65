"""Check the narrow-pass kernels (TMA or fallback) against numpy: recompose Y = [U|A] W and Y^T Y."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2108_08845_b200 import _native as nat

dev = torch.device("cuda", 0)
c = nat.context(dev)
st = nat.stream_ptr(dev)
rng = np.random.default_rng(0)
for (M, kc, B, K) in [(4096, 10, 200, 10), (1000, 10, 200, 10), (4097, 0, 37, 5), (65536, 10, 200, 10), (3000, 16, 24, 16)]:
    U = rng.standard_normal((M, kc)); A = rng.standard_normal((M, B)); W = rng.standard_normal((kc + B, K))
    Ud = nat.as_device_colmajor(U, dev, "U") if kc else None
    Ad = nat.as_device_colmajor(A, dev, "A")
    Wd = torch.from_numpy(np.asfortranarray(W)).to(dev).t().contiguous().t()  # col-major n x K
    Wd = torch.from_numpy(W.T.copy()).to(dev)  # (K, n) row-major == (n, K) col-major
    out = nat.DevMat.empty(M, K, dev)
    utu = torch.empty((K, K), dtype=torch.float64, device=dev)
    nat.call("psvd_recompose", c, M, nat._vp(Ud.data_ptr() if kc else 0), Ud.ld if kc else 0, kc,
             nat._vp(Ad.data_ptr()), Ad.ld, B, nat.ptr(Wd), K, nat._vp(out.data_ptr()), out.ld, nat.ptr(utu), st)
    torch.cuda.synchronize()
    Y = out.view.cpu().numpy()
    ref = np.concatenate([U, A], axis=1) @ W
    G = utu.cpu().numpy()
    print(M, kc, B, K, "Y err", np.abs(Y - ref).max() / np.abs(ref).max(), "YtY err",
          np.abs(G - ref.T @ ref).max() / np.abs(ref.T @ ref).max())

# stream_all (fused recompose + U^T A_{b+1} passes) against the oracle
import oracle
from paper_2108_08845_b200 import streaming as S
for (M, B, nbt) in [(4096, 200, 4), (65536, 200, 3), (4096, 50, 4)]:
    a = oracle.burgers_matrix(M, B * nbt)
    cfg = S.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=B)
    st, hist = S.stream_all([a[:, i * B:(i + 1) * B] for i in range(nbt)], cfg)
    rm, rs, _ = oracle.ref_stream_all([a[:, i * B:(i + 1) * B] for i in range(nbt)], 10, 0.95)
    m, s = st.numpy()
    print("stream", M, B, nbt, "sigma err", oracle.sigma_rel_err(s, rs),
          [float(h[0]) for h in hist])
