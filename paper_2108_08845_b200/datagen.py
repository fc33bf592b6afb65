"""Snapshot generators and the row-partition rule (reference datagen.py).

burgers_solution / burgers_matrix restate datagen.py:49-90 on the host (same
operation order -> same bytes); burgers_device evaluates the same formula
with a CUDA kernel for full-size throughput runs (agrees with the host to a
few ulp: CUDA's exp/log1p vs glibc's).  partition_bounds is datagen.py:118-136.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .errors import CapacityError

# datagen.py:15-17: allocation cap of the host generator
DEFAULT_MATRIX_CAP = 1 << 30


@dataclass(frozen=True)
class BurgersConfig:
    """Domain and discretization of the analytical Burgers dataset (datagen.py:21-46)."""

    length: float = 1.0
    t_final: float = 2.0
    reynolds: float = 1000.0
    grid_points: int = 16384
    n_snapshots: int = 800

    def __post_init__(self):
        if not self.length > 0.0:
            raise ValueError(f"length must be positive, got {self.length}")
        if not self.t_final > 0.0:
            raise ValueError(f"t_final must be positive, got {self.t_final}")
        if not self.reynolds > 0.0:
            raise ValueError(f"reynolds must be positive, got {self.reynolds}")
        if self.grid_points < 2:
            raise ValueError(f"grid_points must be >= 2, got {self.grid_points}")
        if self.n_snapshots < 1:
            raise ValueError(f"n_snapshots must be >= 1, got {self.n_snapshots}")


def burgers_solution(x, t, config=None, reynolds=1000.0):
    """u(x, t) of viscous Burgers in log space (datagen.py:49-73).  `config` may be a
    BurgersConfig (the reference's signature: domain checks, its Reynolds number) or a
    float Reynolds number; scalars in give a float out."""
    if isinstance(config, BurgersConfig):
        re = config.reynolds
        xa, ta = np.asarray(x, dtype=np.float64), np.asarray(t, dtype=np.float64)
        if xa.size and (np.min(xa) < 0.0 or np.max(xa) > config.length):
            raise ValueError(f"x outside [0, {config.length}]")
        if ta.size and (np.min(ta) < 0.0 or np.max(ta) > config.t_final):
            raise ValueError(f"t outside [0, {config.t_final}]")
    else:
        re = float(config) if config is not None else reynolds
    x = np.asarray(x, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    expo = 0.5 * (np.log1p(t) - re / 8.0) + re * x * x / (4.0 * (t + 1.0))
    u = (x / (t + 1.0)) * np.exp(-np.logaddexp(0.0, expo))
    return float(u) if u.ndim == 0 else u


def burgers_matrix(grid_points=None, n_snapshots=None, length=1.0, t_final=2.0, reynolds=1000.0, rows=None,
                   cols=None, max_bytes=None):
    """u(x_i, t_j) on inclusive linspace grids.  Reference form (datagen.py:76-90):
    burgers_matrix(BurgersConfig(...), max_bytes=DEFAULT_MATRIX_CAP), CapacityError past the cap.
    Extended form: burgers_matrix(grid_points, n_snapshots, ...) with optional row / column
    slices (half-open ranges) for per-rank blocks of matrices too large to build whole."""
    if grid_points is None or isinstance(grid_points, BurgersConfig):
        cfg = grid_points if grid_points is not None else BurgersConfig()
        cap = DEFAULT_MATRIX_CAP if max_bytes is None else max_bytes
        if n_snapshots is not None and max_bytes is None:
            cap = n_snapshots  # positional max_bytes, as the reference's second parameter
        need = 8 * cfg.grid_points * cfg.n_snapshots
        if need > cap:
            raise CapacityError(f"snapshot matrix needs {need} bytes, cap is {cap}")
        grid_points, n_snapshots = cfg.grid_points, cfg.n_snapshots
        length, t_final, reynolds = cfg.length, cfg.t_final, cfg.reynolds
    x = np.linspace(0.0, length, grid_points)
    t = np.linspace(0.0, t_final, n_snapshots)
    if rows is not None:
        x = x[rows[0]:rows[1]]
    if cols is not None:
        t = t[cols[0]:cols[1]]
    return burgers_solution(x[:, None], t[None, :], reynolds)


def synthetic_spectrum_matrix(rows, cols, singular_values, seed=0):
    """Dense matrix with exactly the given leading singular values (datagen.py:93-115):
    Philox(seed) Gaussian factors orthonormalized by QR (diag(R) >= 0, as qr_factor),
    (u * sigma) @ v^T.  Host input generation, byte-identical to the reference's."""
    sv = np.asarray(singular_values, dtype=np.float64)
    if sv.ndim != 1 or sv.size < 1:
        raise ValueError("singular_values must be a non-empty 1-D sequence")
    if sv.size > min(rows, cols):
        raise ValueError(f"{sv.size} singular values do not fit a {rows}x{cols} matrix")
    if np.any(sv < 0.0):
        raise ValueError("singular values must be non-negative")
    if np.any(np.diff(sv) > 0.0):
        raise ValueError("singular values must be non-increasing")
    rng = np.random.Generator(np.random.Philox(seed))

    def orth(m):
        q, r = np.linalg.qr(m, mode="reduced")
        d = np.sign(np.diag(r))
        d[d == 0.0] = 1.0
        return q * d

    u = orth(rng.standard_normal((rows, sv.size)))
    v = orth(rng.standard_normal((cols, sv.size)))
    return (u * sv) @ v.T


def row_partition(a, world_size):
    """Per-rank row blocks (copies, in rank order) of a host matrix (datagen.py:139-142)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or min(a.shape) < 1:
        raise ValueError(f"a must be a non-empty 2-D matrix, got shape {a.shape}")
    return [a[lo:hi].copy() for lo, hi in partition_bounds(a.shape[0], world_size)]


def burgers_device(grid_points, n_snapshots, rows=None, cols=None, length=1.0, t_final=2.0,
                   reynolds=1000.0, device=None, out=None):
    """Device-side Burgers block (column-major DevMat) for rows/cols ranges."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    r0, r1 = rows if rows is not None else (0, grid_points)
    c0, c1 = cols if cols is not None else (0, n_snapshots)
    if out is None:
        out = nat.DevMat.empty(r1 - r0, c1 - c0, dev)
    ctx = nat.context(dev)
    with torch.cuda.device(dev):
        nat.call("psvd_burgers", ctx, nat._vp(out.data_ptr()), out.ld, r0, r1 - r0, grid_points, c0, c1 - c0,
                 n_snapshots, float(length), float(t_final), float(reynolds), nat.stream_ptr(dev))
    return out


def partition_bounds(rows, world_size):
    """Half-open row ranges; the first rows % P ranks get one extra row."""
    if world_size < 1:
        raise ValueError(f"world_size must be >= 1, got {world_size}")
    if world_size > rows:
        raise ValueError(f"world_size {world_size} exceeds row count {rows}")
    base, extra = divmod(rows, world_size)
    out, lo = [], 0
    for r in range(world_size):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


# ---------------------------------------------------------------------------
# Builder-defined synthetic configs (not in the reference).
# Conventions pinned here (the SURVEY lists them as open):
#   * all draws come from numpy Generator(Philox(seed)), in the order documented per function;
#   * "N(0, s)" noise means standard deviation s;
#   * Gaussian factors are NOT orthonormalized: U_f ~ N(0, 1/M), V_f ~ N(0, 1/T), so the
#     singular values of the signal are the prescribed ones up to O(sqrt(r/M)) relative;
#   * snapshots are generated column by column from the factors, so any column range
#     (a batch) can be produced alone with the same bytes as the full matrix.


def weather_matrix(n_snapshots=1024, nlat=721, nlon=1440, n_modes=60, rho=0.9, noise=1e-3, seed=1, cols=None):
    """Config 3: weather-like field on an nlat x nlon grid (rows lat-major).
    Modes sin(a*lat) * cos(b*lon + phi) with lat in [-pi/2, pi/2] (inclusive), lon in
    [0, 2*pi) (exclusive), integers a, b in 1..12, phi ~ U[0, 2pi); AR(1) coefficients
    c_i(t) = rho c_i(t-1) + sqrt(1-rho^2) e, c_i(0) ~ N(0,1), amplitudes 10 * 0.85^i.
    Draw order from Philox(seed): a, b, phi (n_modes each), c(0), innovations
    (n_modes x (T-1)); noise per column (_column_noise)."""
    g = np.random.Generator(np.random.Philox(seed))
    a = g.integers(1, 13, n_modes)
    b = g.integers(1, 13, n_modes)
    phi = g.uniform(0.0, 2.0 * np.pi, n_modes)
    c = np.empty((n_modes, n_snapshots))
    c[:, 0] = g.standard_normal(n_modes)
    innov = g.standard_normal((n_modes, n_snapshots - 1))
    for t in range(1, n_snapshots):
        c[:, t] = rho * c[:, t - 1] + np.sqrt(1.0 - rho * rho) * innov[:, t - 1]
    amp = 10.0 * 0.85 ** np.arange(n_modes)
    lat = np.linspace(-0.5 * np.pi, 0.5 * np.pi, nlat)
    lon = np.linspace(0.0, 2.0 * np.pi, nlon, endpoint=False)
    c0, c1 = cols if cols is not None else (0, n_snapshots)
    space = (np.sin(np.outer(lat, a))[:, None, :] * np.cos(lon[None, :, None] * b[None, None, :] + phi)).reshape(
        nlat * nlon, n_modes)
    out = space @ (amp[:, None] * c[:, c0:c1])
    out += noise * _column_noise(nlat * nlon, c0, c1, seed)
    return np.asfortranarray(out)


def _column_noise(rows, c0, c1, seed):
    """N(0,1) noise, column j from its own Philox stream (key = (seed + 1000) * 2^32 + j),
    so any column range reproduces the same bytes as the full matrix."""
    out = np.empty((rows, c1 - c0), order="F")
    for j in range(c0, c1):
        out[:, j - c0] = np.random.Generator(np.random.Philox(key=(seed + 1000) * 2**32 + j)).standard_normal(rows)
    return out


def factor_matrix(rows, n_snapshots, sigma, noise, seed, cols=None):
    """Configs 4 / 5: A = U_f diag(sigma) V_f^T + noise * N(0,1), Gaussian factors
    U_f ~ N(0, 1/rows) (rows x r), V_f ~ N(0, 1/n_snapshots) (n_snapshots x r), drawn in
    that order from Philox(seed); noise per column (_column_noise)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    r = sigma.size
    g = np.random.Generator(np.random.Philox(seed))
    U = g.standard_normal((rows, r)) / np.sqrt(rows)
    V = g.standard_normal((n_snapshots, r)) / np.sqrt(n_snapshots)
    c0, c1 = cols if cols is not None else (0, n_snapshots)
    out = U @ (sigma[:, None] * V[c0:c1].T)
    out += noise * _column_noise(rows, c0, c1, seed)
    return np.asfortranarray(out)


def weak_scaling_matrix(rows, n_snapshots=4096, cols=None):
    """Config 4: rank-200 signal, sigma_i = i^-1.5 (i = 1..200), noise 1e-4, seed 2."""
    return factor_matrix(rows, n_snapshots, np.arange(1, 201, dtype=np.float64) ** -1.5, 1e-4, 2, cols)


def stress_matrix(rows, n_snapshots=2048, cols=None):
    """Config 5: sigma_i = 1 / (1 + 0.01 i) for i < 512, noise 1e-6, seed 3."""
    return factor_matrix(rows, n_snapshots, 1.0 / (1.0 + 0.01 * np.arange(512, dtype=np.float64)), 1e-6, 3, cols)
