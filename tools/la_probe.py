"""The look-ahead sketch pass's shape through psvd_fused_pass (group A = a 200-column batch under a 20-column W,
group B = a 20-column block for the B^T Y tile): timing alone, PSVD_FS_DBG=2 for the compute-only time."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat
M, B, K = 1 << 20, 200, 20
dev = torch.device("cuda", 0)
D = p.burgers_device(M, 800, device=dev)
c = nat.context(dev)
st = nat.stream_ptr(dev)
Uo = nat.DevMat.empty(M, K, dev)
W = torch.randn((K, B), dtype=torch.float64, device=dev)
UtU = torch.empty((K, K), dtype=torch.float64, device=dev)
AtU = torch.empty((K, K), dtype=torch.float64, device=dev)
A0, A1 = D.data_ptr(), D.data_ptr() + 8 * D.ld * B


def f():
    nat.call("psvd_fused_pass", c, M, None, 0, 0, nat._vp(A0), D.ld, B, nat._vp(A1), D.ld, K,
             nat.ptr(W), K, nat._vp(Uo.data_ptr()), Uo.ld, nat.ptr(UtU), nat.ptr(AtU), 1, 0, None, st)


for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
print(f"la-shaped pass: {e0.elapsed_time(e1) / 10:.3f} ms")
