import sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_2108_08845_b200 as p
for B in (200, 248, 256, 264, 296, 300):
    b = oracle.burgers_matrix(4096, 800)[:, :B]
    for q in (0, 1):
        res = p.low_rank_svd(b, p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=q, seed=3))
        ru, rs, rvt = oracle.ref_low_rank_svd(b, 10, 10, q, 3)
        from paper_2108_08845_b200 import _native as nat
        c = nat.context(res.s.device); import ctypes
        pc = (ctypes.c_longlong * 5)(); nat.lib().psvd_path_counters(c, pc)
        print(B, q, "sig rel", oracle.sigma_rel_err(res.s.cpu().numpy(), rs), "paths", list(pc))
