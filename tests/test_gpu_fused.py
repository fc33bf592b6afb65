"""The fused pass of the pipelined deterministic stream through the C ABI (psvd_fused_pass): the narrow TMA
pass (mode 0) and the split-ring kernel (mode 1: 32-row 3-D TMA boxes in two column-group rings, W in
registers, offloaded tiles of A_next^T A_next) against plain fp64 matrix products of the same operands:
U_out = [U | A] W (streaming.py:102-103's q @ u for the Gram route), U_out^T U_out, A_next^T U_out.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(M, Kc, B, Bn, K, mode, noff, seed=0):
    import paper_2108_08845_b200 as p
    from paper_2108_08845_b200 import _native as nat
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(seed)
    c = nat.context(dev)
    st = nat.stream_ptr(dev)

    def mat(r, k):
        m = nat.DevMat.empty(r, k, dev)
        if k:
            m.view.copy_(torch.randn((r, k), dtype=torch.float64, generator=g).to(dev))
        return m

    U, A, An, Uo = mat(M, Kc), mat(M, B), mat(M, Bn), nat.DevMat.empty(M, K, dev)
    W = torch.randn((K, Kc + B), dtype=torch.float64, generator=g).to(dev)  # (Kc + B) x K column-major
    UtU = torch.empty((K, K), dtype=torch.float64, device=dev)
    AtU = torch.empty((K, Bn), dtype=torch.float64, device=dev)  # Bn x K column-major
    nb = (Bn + 31) // 32
    off = torch.full((nb * nb, 32, 32), float("nan"), dtype=torch.float64, device=dev)
    nat.call("psvd_fused_pass", c, M, nat._vp(U.data_ptr()) if Kc else None, U.ld, Kc, nat._vp(A.data_ptr()), A.ld, B,
             nat._vp(An.data_ptr()), An.ld, Bn, nat.ptr(W), K, nat._vp(Uo.data_ptr()), Uo.ld, nat.ptr(UtU),
             nat.ptr(AtU), mode, noff, nat.ptr(off), st)
    torch.cuda.synchronize()
    P = torch.cat([U.view, A.view], dim=1) if Kc else A.view
    ref_u = P @ W.T
    scale = float(ref_u.abs().max())
    assert float((Uo.view - ref_u).abs().max()) <= 1e-12 * scale * (Kc + B) ** 0.5
    ref_uu = ref_u.T @ ref_u
    assert float((UtU.T - ref_uu).abs().max()) <= 1e-12 * float(ref_uu.abs().max())
    ref_au = An.view.T @ ref_u
    assert float((AtU.T - ref_au).abs().max()) <= 1e-12 * float(ref_au.abs().max()) + 1e-12 * scale * M ** 0.5
    if mode == 1:
        for t in range(min(noff, (Bn // 32) // 2)):
            blk = An.view[:, 64 * t:64 * t + 32].T @ An.view[:, 64 * t + 32:64 * t + 64]
            got = off[(2 * t) * nb + 2 * t + 1]
            assert float((got - blk).abs().max()) <= 1e-12 * M
    return Uo.view.clone(), UtU.clone(), AtU.clone()


@pytest.mark.parametrize("shape", [
    (4096, 10, 200, 200, 10),    # the bench's widths
    (4096, 0, 200, 200, 10),     # the first update of a stream: no state yet
    (2064, 0, 64, 96, 7),        # one Y column block, a ragged last stage (M a multiple of 16 only)
    (1 << 15, 16, 120, 136, 16),
    (4112, 12, 36, 40, 12),      # narrow batches: no full 32-column pair to offload
    (8192, 10, 208, 72, 9),
    (4096, 0, 200, 20, 20),      # the look-ahead sketch's shape: three Y column blocks, a 20-column group B
    (8192, 20, 24, 200, 20),     # the projection pass's shape: a short W range (one k part), tile warps of <= 5 sub-blocks
])
def test_split_ring_kernel_matches_products_and_narrow_pass(shape):
    M, Kc, B, Bn, K = shape
    u0, uu0, au0 = _run(M, Kc, B, Bn, K, 0, 0)
    for noff in (0, 3):
        u1, uu1, au1 = _run(M, Kc, B, Bn, K, 1, noff)
        # the two kernels sum in different orders: agreement to rounding, both checked against the products
        assert float((u1 - u0).abs().max()) <= 1e-11 * float(u0.abs().max())
        assert float((uu1 - uu0).abs().max()) <= 1e-11 * float(uu0.abs().max())
        assert float((au1 - au0).abs().max()) <= 1e-11 * float(au0.abs().max())


def test_split_ring_kernel_is_bitwise_reproducible():
    a = _run(8192, 10, 200, 200, 10, 1, 3, seed=3)
    b = _run(8192, 10, 200, 200, 10, 1, 3, seed=3)
    assert all(torch.equal(x, y) for x, y in zip(a, b))


def test_split_ring_refuses_shapes_it_cannot_take():
    with pytest.raises(ValueError):
        _run(4100, 10, 200, 200, 10, 1, 0)   # M not a multiple of 16
    with pytest.raises(ValueError):
        _run(4096, 28, 200, 200, 28, 1, 0)   # four Y column blocks (K > 24)
