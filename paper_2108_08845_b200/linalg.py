"""Randomized range finder / low-rank SVD configuration and the randomized
streaming update (reference linalg.py:33-62, 126-162)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RandomSketchConfig:
    """Parameters of the randomized range finder (linalg.py:33-62).

    target_rank      rank of the approximation that is kept
    oversampling     extra sketch columns beyond target_rank
    power_iterations subspace iteration count (0 = plain sketch)
    seed             Philox seed for the Gaussian test matrix
    """

    target_rank: int
    oversampling: int = 10
    power_iterations: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.target_rank < 1:
            raise ValueError(f"target_rank must be >= 1, got {self.target_rank}")
        if self.oversampling < 0:
            raise ValueError(f"oversampling must be >= 0, got {self.oversampling}")
        if self.power_iterations < 0:
            raise ValueError(f"power_iterations must be >= 0, got {self.power_iterations}")
        if self.seed < 0:
            raise ValueError(f"seed must be >= 0, got {self.seed}")

    @property
    def sketch_width(self):
        return self.target_rank + self.oversampling


def gaussian_test_matrix(n_cols, config):
    """The reference's Omega, drawn on the host exactly as linalg.py:141-142
    (Philox(seed).standard_normal((n_cols, width))) and uploaded by callers, so
    both implementations see identical bytes."""
    rng = np.random.Generator(np.random.Philox(config.seed))
    return rng.standard_normal((n_cols, config.sketch_width))


_OMEGA_CACHE = {}


def device_omega(n_cols, config, device):
    """Omega on the device (cached per shape/seed/device; the same seed every
    batch reproduces the R9 composition's draw)."""
    import torch
    key = (n_cols, config.sketch_width, config.seed, str(device))
    om = _OMEGA_CACHE.get(key)
    if om is None:
        host = gaussian_test_matrix(n_cols, config)            # (n, l) C-order
        om = torch.from_numpy(np.asfortranarray(host).T.copy()).to(device)  # (l, n): col-major n x l
        if len(_OMEGA_CACHE) > 16:
            _OMEGA_CACHE.clear()
        _OMEGA_CACHE[key] = om
    return om


def randomized_update(U, sigma, A, sketch, ff, device, check=True, total_rows=None, omega=None):
    """One randomized step: low_rank_svd([ff*U*diag(sigma) | A], sketch) on the
    device (linalg.py:150-162 composed per batch).  U: DevMat or None.
    total_rows: rows of the whole (row-partitioned) panel for the width check.
    omega: optional device test matrix (n x l, column-major) replacing the Philox draw.
    Returns (DevMat M x K, sigma (K,))."""
    import torch
    from . import _native as nat
    k, l, q = sketch.target_rank, sketch.sketch_width, sketch.power_iterations
    M, B = A.rows, A.cols
    kc = 0 if U is None else U.cols
    n = kc + B
    rows = M if total_rows is None else total_rows
    if l > min(rows, n):
        raise ValueError(f"sketch width {l} exceeds min(a.shape) = {min(rows, n)}")
    om = device_omega(n, sketch, device) if omega is None else omega
    ctx = nat.context(device)
    with torch.cuda.device(device):
        out = nat.DevMat.empty(M, k, device)
        sig = torch.empty(k, dtype=torch.float64, device=device)
        nat.call("psvd_rand_update", ctx, M, nat._vp(U.data_ptr() if U is not None else 0),
                 U.ld if U is not None else 0, nat.ptr(sigma if U is not None else None), float(ff), kc,
                 nat._vp(A.data_ptr()), A.ld, B, k, l, q, nat.ptr(om), nat._vp(out.data_ptr()), out.ld,
                 nat.ptr(sig), nat.stream_ptr(device))
        if check:
            st = nat.read_status(ctx, reset=True, device=device)
            if st & nat.ST_NONFINITE:
                raise ValueError("a_new contains non-finite entries")
            if st & nat.ST_NOCONVERGE:
                from .errors import ConvergenceError
                raise ConvergenceError("randomized core SVD did not converge")
    return out, sig


def low_rank_svd(a, config, device=None):
    """Randomized truncated SVD of a device/host matrix (linalg.py:150-162):
    returns (u (m x target_rank) CUDA tensor, s (target_rank,) CUDA tensor).
    vt is not formed (the streaming update never uses it)."""
    import torch
    from . import _native as nat
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    A = nat.as_device_colmajor(a, dev, "a")
    u, s = randomized_update(None, None, A, config, 1.0, dev)
    return u.view, s
