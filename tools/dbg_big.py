import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat
for (m, n, kind) in [(4096, 800, 'burgers'), (4096, 300, 'burgers'), (4096, 112, 'burgers'), (4096, 150, 'burgers')]:
    a = oracle.burgers_matrix(m, 800)[:, :n] if kind == 'burgers' else None
    res = p.qr_factor(a)
    q, r = res.q.cpu().numpy(), res.r.cpu().numpy()
    qr_, rr = oracle.ref_qr(a)
    print(m, n, 'qr resid', np.max(np.abs(q @ r - a)) / np.abs(a).max(), 'orth', np.max(np.abs(q.T @ q - np.eye(n))),
          'zero diag', int(np.sum(np.diag(r) == 0)), 'maxR', np.abs(r).max(), 'maxRref', np.abs(rr).max())
    s_r = np.linalg.svd(r, compute_uv=False)
    rs = np.linalg.svd(a, compute_uv=False)
    print('   svd(R_gpu) vs svd(a):', np.max(np.abs(s_r - rs)) / rs[0])
    dev = torch.device('cuda', 0)
    ctx = nat.context(dev)
    R = torch.as_tensor(np.asfortranarray(r)).to(dev)
    Rm = nat.as_device_colmajor(R, dev, 'r')
    S = torch.empty(n, dtype=torch.float64, device=dev)
    UR = nat.DevMat.empty(n, n, dev); VR = nat.DevMat.empty(n, n, dev)
    nat.call('psvd_jacobi_uv', ctx, nat._vp(Rm.data_ptr()), Rm.ld, n, n, 1, nat.ptr(S), nat._vp(UR.data_ptr()), UR.ld,
             nat._vp(VR.data_ptr()), VR.ld, nat.stream_ptr(dev))
    st = nat.read_status(ctx, True, dev)
    s = S.cpu().numpy()
    print('   jacobi(R^T) S vs svd(R):', np.max(np.abs(s - s_r)) / s_r[0], 'status', st, s[:4])
    # jacobi on R (no transpose)
    nat.call('psvd_jacobi_uv', ctx, nat._vp(Rm.data_ptr()), Rm.ld, n, n, 0, nat.ptr(S), nat._vp(UR.data_ptr()), UR.ld,
             nat._vp(VR.data_ptr()), VR.ld, nat.stream_ptr(dev))
    s = S.cpu().numpy()
    print('   jacobi(R) S vs svd(R):', np.max(np.abs(s - s_r)) / s_r[0], s[:4])
