"""Timing of the fused pass alone on config-2 shapes (psvd_fused_pass): mode / offloaded tiles from argv,
PSVD_FS_DBG=2 for the compute-only time."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat
M, B, K = 1 << 20, 200, 10
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
noff = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
D = p.burgers_device(M, 800, device=dev)
c = nat.context(dev)
st = nat.stream_ptr(dev)
U = nat.DevMat.empty(M, K, dev)
U.view.copy_(D.view[:, 600:610])
Uo = nat.DevMat.empty(M, K, dev)
W = torch.randn((K, K + B), dtype=torch.float64, device=dev)
UtU = torch.empty((K, K), dtype=torch.float64, device=dev)
AtU = torch.empty((K, B), dtype=torch.float64, device=dev)
off = torch.empty((49, 32, 32), dtype=torch.float64, device=dev)
A0, A1 = D.data_ptr(), D.data_ptr() + 8 * D.ld * B


def f():
    nat.call("psvd_fused_pass", c, M, nat._vp(U.data_ptr()), U.ld, K, nat._vp(A0), D.ld, B, nat._vp(A1), D.ld, B,
             nat.ptr(W), K, nat._vp(Uo.data_ptr()), Uo.ld, nat.ptr(UtU), nat.ptr(AtU), mode, noff, nat.ptr(off), st)


for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
print(f"fused pass mode {mode} noff {noff}: {e0.elapsed_time(e1) / 10:.3f} ms")
