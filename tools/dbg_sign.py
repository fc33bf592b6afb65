"""Debug: signs of the accurate route vs the Gram route vs the oracle, per update (same inputs)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat

dev = torch.device('cuda', 0)
ctx = nat.context(dev)
a = oracle.burgers_matrix(4097, 800)[:, :400]
k, ff = 12, 1.0
bs = [a[:, i:i + 100] for i in range(0, 400, 100)]
U = sig = None
for step, b in enumerate(bs):
    if U is None:
        rm, rs = oracle.ref_stream_init(b, k)
    else:
        rm, rs = oracle.ref_stream_update(U, sig, b, k, ff)
    A = nat.as_device_colmajor(b, dev)
    res = {}
    for fn in ("psvd_stream_update", "psvd_stream_update_accurate"):
        out = nat.DevMat.empty(A.rows, k, dev)
        so = torch.empty(k, dtype=torch.float64, device=dev)
        if U is None:
            Ud, sd, kc = None, None, 0
        else:
            Ud = nat.as_device_colmajor(U, dev)
            sd = torch.as_tensor(sig).to(dev)
            kc = k
        nat.call(fn, ctx, A.rows, nat._vp(Ud.data_ptr() if Ud is not None else 0), Ud.ld if Ud is not None else 0,
                 nat.ptr(sd), ff, kc, nat._vp(A.data_ptr()), A.ld, A.cols, k, 1, nat._vp(out.data_ptr()), out.ld,
                 nat.ptr(so), nat.stream_ptr(dev))
        st = nat.read_status(ctx, True, dev)
        m = out.view.cpu().numpy()
        s = so.cpu().numpy()
        res[fn] = (m, s, st)
        print(step, fn, 'status', st, 'sig err', oracle.sigma_rel_err(s, rs), 'signs', np.sign(np.sum(m * rm, axis=0)).astype(int).tolist(),
              'ang', float(np.max(oracle.mode_angles(m, rm))))
    print('   kappa', rs[0] / rs[-1])
    U, sig = rm, rs
