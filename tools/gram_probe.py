"""Time psvd_gram (Gram-only pass) on a device-resident Burgers panel."""
import sys, torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat
M, n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20, int(sys.argv[2]) if len(sys.argv) > 2 else 200
dev = torch.device("cuda", 0)
D = p.burgers_device(M, 800, device=dev)
c = nat.context(dev); st = nat.stream_ptr(dev)
G = torch.empty((n, n), dtype=torch.float64, device=dev)
def run():
    nat.call("psvd_gram", c, M, nat._vp(0), 0, nat._vp(0), 1.0, 0, nat._vp(D.data_ptr()), D.ld, n, nat.ptr(G), st)
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"M={M} n={n}: {ms:.3f} ms, {M*n*(n+1)/ms/1e9:.2f} TFLOP/s useful")
