"""Snapshot generators and the row-partition rule (reference datagen.py).

burgers_solution / burgers_matrix restate datagen.py:49-90 on the host (same
operation order -> same bytes); burgers_device evaluates the same formula
with a CUDA kernel for full-size throughput runs (agrees with the host to a
few ulp: CUDA's exp/log1p vs glibc's).  partition_bounds is datagen.py:118-136.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat


def burgers_solution(x, t, reynolds=1000.0):
    x = np.asarray(x, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    expo = 0.5 * (np.log1p(t) - reynolds / 8.0) + reynolds * x * x / (4.0 * (t + 1.0))
    return (x / (t + 1.0)) * np.exp(-np.logaddexp(0.0, expo))


def burgers_matrix(grid_points, n_snapshots, length=1.0, t_final=2.0, reynolds=1000.0, rows=None, cols=None):
    """u(x_i, t_j) on inclusive linspace grids; optional row / column slices."""
    x = np.linspace(0.0, length, grid_points)
    t = np.linspace(0.0, t_final, n_snapshots)
    if rows is not None:
        x = x[rows[0]:rows[1]]
    if cols is not None:
        t = t[cols[0]:cols[1]]
    return burgers_solution(x[:, None], t[None, :], reynolds)


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
