"""Randomized update timing breakdown (diagnostics): one config-2 stream, q = 0 / 1."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat
from paper_2108_08845_b200.linalg import RandomSketchConfig, device_omega
M, S, B, K = 1 << 20, 800, 200, 10
dev = torch.device("cuda", 0)
D = p.burgers_device(M, S, device=dev)
c = nat.context(dev); st = nat.stream_ptr(dev)
for q in (0, 1):
    sk = RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=q, seed=0)
    l = sk.sketch_width
    om = {n: device_omega(n, sk, dev) for n in (B, K + B)}
    Ub = [nat.DevMat.empty(M, K, dev) for _ in range(2)]
    sig = [torch.zeros(K, dtype=torch.float64, device=dev) for _ in range(2)]
    def step():
        cur = 0
        for b in range(S // B):
            kc = 0 if b == 0 else K
            nat.call("psvd_rand_update", c, M, nat._vp(Ub[cur].data_ptr()), Ub[cur].ld, nat.ptr(sig[cur]), 0.95, kc,
                     nat._vp(D.data_ptr() + 8 * D.ld * b * B), D.ld, B, K, l, q, nat.ptr(om[kc + B]),
                     nat._vp(Ub[cur ^ 1].data_ptr()), Ub[cur ^ 1].ld, nat.ptr(sig[cur ^ 1]), st)
            cur ^= 1
    for _ in range(3): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): step()
    e1.record(); torch.cuda.synchronize()
    print(f"q={q}: {e0.elapsed_time(e1)/5:.3f} ms per stream")
