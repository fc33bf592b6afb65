"""Narrow TMA pass on one wide segment (two TMA boxes): Y = P W and Y^T Y vs torch (diagnostics)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat
dev = torch.device("cuda", 0)
torch.manual_seed(0)
for n, K in ((248, 10), (256, 10), (264, 10), (256, 20), (264, 20), (296, 20), (264, 16)):
    M = 4096
    A = nat.DevMat.empty(M, n, dev)
    A.view.copy_(torch.randn(M, n, dtype=torch.float64, device=dev))
    W = torch.randn(K, n, dtype=torch.float64, device=dev)  # column-major n x K: W.T
    U = nat.DevMat.empty(M, K, dev)
    utu = torch.empty((K, K), dtype=torch.float64, device=dev)
    c = nat.context(dev)
    nat.call("psvd_recompose", c, M, nat._vp(0), 0, 0, nat._vp(A.data_ptr()), A.ld, n, nat.ptr(W), K,
             nat._vp(U.data_ptr()), U.ld, nat.ptr(utu), nat.stream_ptr(dev))
    ref = A.view @ W.T
    err = (U.view - ref).abs().max(dim=0).values
    print(n, "max |Y - ref| per column", [f"{e:.1e}" for e in err.tolist()])
    bad_rows = ((U.view - ref).abs().max(dim=1).values > 1e-9).nonzero().flatten()
    print("   bad rows:", bad_rows[:10].tolist(), "count", bad_rows.numel(), " UtU err",
          float((utu - ref.T @ ref).abs().max() / (ref.T @ ref).abs().max()))
