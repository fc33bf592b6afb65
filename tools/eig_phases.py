"""Phase breakdown (SM cycles) of the one-CTA core eigensolver on a Burgers Gram."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2108_08845_b200 import _native as nat
import oracle

def main(n=210, K=10):
    dev = torch.device("cuda", 0)
    c = nat.context(dev); st = nat.stream_ptr(dev)
    a = oracle.burgers_matrix(65536, 800)[:, 200:200 + n]
    G = torch.as_tensor(a.T @ a).cuda()
    W = torch.empty((K, n), dtype=torch.float64, device=dev); s = torch.empty(K, dtype=torch.float64, device=dev)
    for _ in range(3):
        nat.call("psvd_core_eig", c, nat.ptr(G), n, nat._vp(0), 1.0, 0, K, nat.ptr(W), nat.ptr(s), st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        nat.call("psvd_core_eig", c, nat.ptr(G), n, nat._vp(0), 1.0, 0, K, nat.ptr(W), nat.ptr(s), st)
    e1.record(); torch.cuda.synchronize()
    t = (ctypes.c_longlong * 14)()
    nat.lib().psvd_eig_phase_cycles(c, t)
    names = ["load", "tridiag", "bisect", "twisted", "mgs", "backxf", "ldlt", "sign+W"]
    d = [t[i + 1] - t[i] for i in range(8)]
    print(f"n={n} K={K}: {e0.elapsed_time(e1)/10*1e3:.1f} us/launch; cycles", dict(zip(names, d)), "total", t[8] - t[0])
    print("tridiag sub-phases (a..e):", [t[9 + i] for i in range(5)])
    ref = np.linalg.svd(a, compute_uv=False)[:K]
    print("sigma rel err", np.max(np.abs(s.cpu().numpy() - ref) / ref))

if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
