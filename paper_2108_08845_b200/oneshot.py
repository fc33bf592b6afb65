"""One-shot distributed SVD (APMOS) — B200 drop-in for the reference's
ApmosConfig / generate_right_vectors / apmos (dsvd.py:39-173).

Per rank (one process per GPU), on the device:

    G_i = A_i^T A_i                        Gram pass (libpsvd; wide panels: tall-skinny TN GEMM)
    (V_i, s_i) = top-r1 eigenpairs of G_i  psvd_sym_topk, zero-padded to r1 (dsvd.py:120-123)
    W_i = V_i diag(s_i)                    n x r1, the "small Sigma V^T block" of the paper
    W = [W_0 | ... | W_{P-1}]              NCCL allgather in rank order (replaces gather + broadcast,
                                           dsvd.py:146-165): every rank factors identical bits
    X, lambda = svd_full(W)[:r2]           Gram route: eig of W^T W, X = W V_w / lambda, peak sign
                                           rule on X (linalg.py:81-91); or low_rank_svd(W, sketch)
    U_i = A_i X[:, :K] / lambda[:K]        recompose pass (libpsvd)

A zero lambda among the first K raises DegenerateModeError on every rank alike
(dsvd.py:167-171).  Singular values are those of W (= of A when untruncated)
with the Gram route's eps * (s_1 / s_k)^2 relative accuracy, far inside 1e-10
at the shapes tested against the live reference's golden vectors.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist

from . import _native as nat
from .dsvd import LocalModes, RankContext  # noqa: F401  (re-exported API surface)
from .errors import DegenerateModeError
from .linalg import RandomSketchConfig, randomized_update


@dataclass(frozen=True)
class ApmosConfig:
    """local_rank r1, global_rank r2, k_modes K <= r2; use_randomized / sketch
    factor the stacked W with the randomized kernel (dsvd.py:39-68)."""

    local_rank: int
    global_rank: int
    k_modes: int
    use_randomized: bool = False
    sketch: Optional[RandomSketchConfig] = None

    def __post_init__(self):
        if self.local_rank < 1:
            raise ValueError(f"local_rank must be >= 1, got {self.local_rank}")
        if self.global_rank < 1:
            raise ValueError(f"global_rank must be >= 1, got {self.global_rank}")
        if self.k_modes < 1:
            raise ValueError(f"k_modes must be >= 1, got {self.k_modes}")
        if self.k_modes > self.global_rank:
            raise ValueError(f"k_modes {self.k_modes} exceeds global_rank {self.global_rank}")
        if self.sketch is not None and self.sketch.target_rank < self.global_rank:
            raise ValueError(f"sketch target_rank {self.sketch.target_rank} is below "
                             f"global_rank {self.global_rank}")


def _device(x):
    if isinstance(x, torch.Tensor) and x.device.type == "cuda":
        return x.device
    nat.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _gram(A, dev):
    c = nat.context(dev)
    n = A.cols
    G = torch.empty((n, n), dtype=torch.float64, device=dev)
    nat.call("psvd_gram", c, A.rows, nat._vp(0), 0, nat._vp(0), 1.0, 0, nat._vp(A.data_ptr()), A.ld, n,
             nat.ptr(G), nat.stream_ptr(dev))
    return G


def _topk(G, n, k, dev):
    """(V n x k column-major DevMat, s (k,)) of the symmetric PSD G."""
    c = nat.context(dev)
    V = nat.DevMat.empty(n, k, dev)
    s = torch.empty(k, dtype=torch.float64, device=dev)
    nat.call("psvd_sym_topk", c, nat.ptr(G), n, k, nat._vp(V.data_ptr()), V.ld, nat.ptr(s), nat.stream_ptr(dev))
    st = nat.read_status(c, reset=True, device=dev)
    if st & nat.ST_NONFINITE:
        raise ValueError("a_local contains non-finite entries")
    return V, s


def _sign_by_peak(M, dev):
    c = nat.context(dev)
    nat.call("psvd_sign_by_peak", c, nat._vp(M.data_ptr()), M.ld, M.rows, M.cols, nat.stream_ptr(dev))


def _recompose(A, W, k, dev):
    """A (M x n) @ W (n x k) on the narrow pass."""
    c = nat.context(dev)
    out = nat.DevMat.empty(A.rows, k, dev)
    Wc = W.t().contiguous().t()  # column-major n x k with ld n
    nat.call("psvd_recompose", c, A.rows, nat._vp(0), 0, 0, nat._vp(A.data_ptr()), A.ld, A.cols,
             nat._vp(Wc.data_ptr()), k, nat._vp(out.data_ptr()), out.ld, nat._vp(0), nat.stream_ptr(dev))
    return out


def _tn(A, Y, dev):
    """A^T Y (A: M x n, Y: M x m, column-major DevMats) as an n x m column-major tensor."""
    c = nat.context(dev)
    X = torch.empty((Y.cols, A.cols), dtype=torch.float64, device=dev).t()  # column-major, ld n
    nat.call("psvd_tn_product", c, A.rows, nat._vp(A.data_ptr()), A.ld, A.cols, nat._vp(Y.data_ptr()), Y.ld, Y.cols,
             nat._vp(X.data_ptr()), A.cols, nat.stream_ptr(dev))
    return X


GRAM_EDGE = 1e-4       # s_r / s_1 below which the Gram's eigenvectors no longer give the top-r range to 1e-8
ACCURATE_FACTORS = 0   # _left_factor calls that took the svd_full route (diagnostics / tests)


def _left_factor(A, r, dev):
    """Top-r left singular vectors U (M x r, orthonormal to working precision, peak-positive
    columns) and singular values of A.  The Gram eigenvectors V0 of A^T A give the subspace;
    U is then one randomized-SVD step of A with Omega = V0 (Y = A V0, SVQB + CholeskyQR,
    B = Q^T A, one-sided Jacobi of B^T): the singular values and U are accurate to
    eps ||A|| like the reference's Householder SVD, not eps ||A||^2 / s_k like the Gram alone.
    Forming A^T A tilts V0's r-th direction by ~eps (s_1 / s_r)^2, and below sqrt(eps) s_1 the
    directions are lost altogether (mixed with A's null space when A is wide): a truncation
    (r < rank) whose edge lies below GRAM_EDGE s_1 takes the reference's own route instead, the
    backward-stable svd_full (linalg.py:107-123), truncated."""
    V0, s0 = _topk(_gram(A, dev), A.cols, r, dev)
    if r < min(A.rows, A.cols) and float(s0[r - 1]) < GRAM_EDGE * float(s0[0]):
        from .errors import ConvergenceError
        from .linalg import svd_full
        global ACCURATE_FACTORS
        try:
            res = svd_full(A.view, want_vt=False, device=dev)
            ACCURATE_FACTORS += 1
            return nat.as_device_colmajor(res.u[:, :r], dev, "u"), res.s[:r].clone()
        except ConvergenceError:
            pass  # the Jacobi sweeps ran out (columns graded over ~1e60 and more): the Gram route's result stands
    om = V0.view.t().contiguous()  # (r, n) row-major == column-major n x r, ld n
    sk = RandomSketchConfig(target_rank=r, oversampling=0, power_iterations=0, seed=0)
    return randomized_update(None, None, A, sk, 1.0, dev, omega=om)


def _right_vectors(A, local_rank, dev, signs):
    """(W or v, s): zero-padded to local_rank columns.  signs == None returns W = V S = A^T U
    (apmos: only W W^T matters); "svd" returns v = A^T U / s with u peak-positive (the
    reference's svd route); "gram" applies the peak rule to v itself."""
    n = A.cols
    keep = min(local_rank, n) if signs == "gram" else min(local_rank, n, A.rows)
    U, s = _left_factor(A, keep, dev)
    W = _tn(A, U, dev)  # = V S
    if signs is None:
        v = W
    else:
        v = W * torch.where(s > 0, 1.0 / s, torch.zeros_like(s))
        if signs == "gram":
            vm = nat.as_device_colmajor(v, dev)
            _sign_by_peak(vm, dev)
            v = vm.view
    out = torch.zeros((local_rank, n), dtype=torch.float64, device=dev).t()  # column-major n x r1
    out[:, :keep] = v
    sp = torch.zeros(local_rank, dtype=torch.float64, device=dev)
    sp[:keep] = s
    return out, sp


def generate_right_vectors(a_local, local_rank, method="svd", device=None):
    """Leading right singular vectors / values of a local slice, zero-padded to
    local_rank columns (dsvd.py:80-124).  Returns (v (n_cols x local_rank), s)."""
    dev = torch.device(device) if device is not None else _device(a_local)
    A = nat.as_device_colmajor(a_local, dev, "a_local")
    if local_rank < 1:
        raise ValueError(f"local_rank must be >= 1, got {local_rank}")
    if local_rank > A.cols:
        raise ValueError(f"local_rank {local_rank} exceeds the snapshot count {A.cols}")
    if method not in ("svd", "gram"):
        raise ValueError(f"unknown method {method!r}")
    return _right_vectors(A, local_rank, dev, method)


def _allgather_cols(ctx, w):
    """[w_0 | w_1 | ...] (rank order) of the per-rank n x r blocks, on every rank."""
    if ctx.world_size == 1:
        return w
    n, r = w.shape
    block = w.t().contiguous()  # (r, n): column-major n x r bytes
    if dist.get_backend(ctx.group) == "nccl":
        out = torch.empty((ctx.world_size * r, n), dtype=w.dtype, device=w.device)
        dist.all_gather_into_tensor(out, block, group=ctx.group)
    else:  # gloo: host staging
        parts = [torch.empty((r, n), dtype=w.dtype) for _ in range(ctx.world_size)]
        dist.all_gather(parts, block.cpu(), group=ctx.group)
        out = torch.cat(parts).to(w.device)
    return out.t()  # column-major n x (P r)


def apmos(ctx, a_local, config):
    """One-shot distributed SVD of the row-partitioned matrix (dsvd.py:127-173).
    Every rank returns LocalModes with its rows of the K leading left singular
    vectors and the (replicated) singular values."""
    dev = _device(a_local)
    A = nat.as_device_colmajor(a_local, dev, "a_local")
    r1, r2, k = config.local_rank, config.global_rank, config.k_modes
    if r2 > ctx.world_size * r1:
        raise ValueError(f"global_rank {r2} exceeds the {ctx.world_size * r1} columns the exchange can produce")
    if r1 > A.cols:
        raise ValueError(f"local_rank {r1} exceeds the snapshot count {A.cols}")
    with torch.cuda.device(dev):
        w, _ = _right_vectors(A, r1, dev, None)  # W_i = V_i S_i = A_i^T U_i (signs irrelevant)
        W = nat.as_device_colmajor(_allgather_cols(ctx, w), dev, "W")
        if config.use_randomized:
            sk = config.sketch if config.sketch is not None else RandomSketchConfig(target_rank=r2)
            u, lam = randomized_update(None, None, W, sk, 1.0, dev)
            have = lam.numel()
            x = u.view
        else:  # svd_full(W): left singular vectors, peak-positive columns (linalg.py:81-91)
            have = min(W.rows, W.cols)
            if have >= r2:
                X, lam = _left_factor(W, r2, dev)
                x = X.view
            else:
                x, lam = None, None
        if have < r2:
            raise ValueError(f"stacked exchange matrix only has {have} singular values, global_rank is {r2}")
        lam_k = lam[:k]
        zero = (lam_k == 0.0).nonzero()
        if zero.numel() > 0:
            j = int(zero[0].item())
            raise DegenerateModeError(f"mode {j} has a zero singular value and cannot be assembled")
        u_local = _recompose(A, x[:, :k] / lam_k, k, dev)
    return LocalModes(u_local.view, lam_k.clone())
