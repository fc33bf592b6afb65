"""Would splitting the deterministic fused pass pay?  Times, on config-2 shapes, the pieces a split would
use: psvd_recompose ([U | A_b] W -> U_b and U_b^T U_b: a narrow pass over 210 columns) and
psvd_tn_product (A_{b+1}^T U_b: the tall-skinny TN GEMM), against the fused pass's ncu time."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat
M, B, K = 1 << 20, 200, 10
dev = torch.device("cuda", 0)
D = p.burgers_device(M, 800, device=dev)
c = nat.context(dev)
st = nat.stream_ptr(dev)
U = nat.DevMat.empty(M, K, dev)
U.view.copy_(D.view[:, 600:610])
Uo = nat.DevMat.empty(M, K, dev)
W = torch.randn((K + B, K), dtype=torch.float64, device=dev)
UtU = torch.empty((K, K), dtype=torch.float64, device=dev)
X = torch.empty((B, K), dtype=torch.float64, device=dev)
A0, A1 = D.data_ptr(), D.data_ptr() + 8 * D.ld * B


def rec():
    nat.call("psvd_recompose", c, M, nat._vp(U.data_ptr()), U.ld, K, nat._vp(A0), D.ld, B, nat.ptr(W), K,
             nat._vp(Uo.data_ptr()), Uo.ld, nat.ptr(UtU), st)


def tn():
    nat.call("psvd_tn_product", c, M, nat._vp(A1), D.ld, B, nat._vp(Uo.data_ptr()), Uo.ld, K, nat.ptr(X), B, st)


for name, f in [("recompose", rec), ("tn_product", tn)]:
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms")
