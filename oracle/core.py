"""numpy restatement of the reference streaming-SVD path (TEST INFRASTRUCTURE).

Every function names the reference lines it restates (paths relative to
/root/reference/pkg/src/parsvd).  The arithmetic is the reference's: numpy's
LAPACK-backed `np.linalg.qr` / `np.linalg.svd` and BLAS matmul, with the same
sign conventions, the same truncation order and the same Philox draw, so the
oracle reproduces the reference's numbers on identical input bytes (pinned by
tests/test_oracle_golden.py against vectors from the live reference).

Nothing in the product package imports this module.
"""

from __future__ import annotations

import numpy as np

# streaming.py:25 — re-orthonormalize when max|U^T U - I| exceeds this
DRIFT_TOL = 1e-8


# --------------------------------------------------------------------------
# dense kernels (linalg.py)
# --------------------------------------------------------------------------

def _check(a, name="a"):
    """Input coercion of linalg.py:65-78 (2-D float64, positive dims, finite)."""
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got {m.ndim}-D")
    if min(m.shape) < 1:
        raise ValueError(f"{name} must have positive dimensions, got {m.shape}")
    if not np.isfinite(m).all():
        raise ValueError(f"{name} contains non-finite entries")
    return m


def _flip_by_peak(u, vt=None):
    """Column sign rule of linalg.py:81-91: the largest-|.| entry of each
    column of u becomes positive (first index wins ties); vt rows follow."""
    peak_rows = np.abs(u).argmax(axis=0)
    sgn = np.sign(u[peak_rows, np.arange(u.shape[1])])
    sgn = np.where(sgn == 0.0, 1.0, sgn)
    return u * sgn, (None if vt is None else vt * sgn[:, None])


def ref_qr(a):
    """Reduced QR with non-negative diag(R) — linalg.py:94-104."""
    a = _check(a)
    q, r = np.linalg.qr(a, mode="reduced")
    d = np.sign(np.diag(r))
    d = np.where(d == 0.0, 1.0, d)
    return q * d, r * d[:, None]


def ref_svd(a, want_vt=True):
    """Thin SVD, descending s, peak-positive columns — linalg.py:107-123."""
    a = _check(a)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    u, vt = _flip_by_peak(u, vt)
    return u, s, (vt if want_vt else None)


def ref_omega(n_cols, width, seed):
    """Gaussian test matrix exactly as linalg.py:141-142 draws it."""
    gen = np.random.Generator(np.random.Philox(seed))
    return gen.standard_normal((n_cols, width))


def ref_range(a, width, power_iterations, seed, omega=None):
    """Randomized range finder — linalg.py:126-147."""
    a = _check(a)
    if width > min(a.shape):
        raise ValueError(f"sketch width {width} exceeds min(a.shape) = {min(a.shape)}")
    om = ref_omega(a.shape[1], width, seed) if omega is None else omega
    q = ref_qr(a @ om)[0]
    for _ in range(power_iterations):
        q = ref_qr(a.T @ q)[0]
        q = ref_qr(a @ q)[0]
    return q


def ref_low_rank_svd(a, k, oversampling=10, power_iterations=1, seed=0, omega=None):
    """Randomized truncated SVD with the tall sign rule — linalg.py:150-162.
    Returns (u m x k, s k, vt k x n)."""
    a = _check(a)
    q = ref_range(a, k + oversampling, power_iterations, seed, omega)
    ub, sb, vtb = ref_svd(q.T @ a, want_vt=True)
    u, vt = _flip_by_peak(q @ ub[:, :k], vtb[:k])
    return u, sb[:k].copy(), vt


# --------------------------------------------------------------------------
# streaming (streaming.py)
# --------------------------------------------------------------------------

def ref_stream_init(a0, k):
    """stream_initialize — streaming.py:63-78.  Returns (modes, sigma)."""
    a0 = _check(a0, "a0")
    if a0.shape[1] < k:
        raise ValueError(f"initial batch has {a0.shape[1]} columns, need at least k_modes={k}")
    q, r = ref_qr(a0)
    u, s, _ = ref_svd(r, want_vt=False)
    return (q @ u)[:, :k], s[:k].copy()


def ref_stream_update(modes, sigma, a, k, ff, rescue=True):
    """stream_incorporate — streaming.py:81-116 (rescue pass 106-115)."""
    a = _check(a, "a_new")
    if modes.shape[1] != k:
        raise ValueError(f"state carries {modes.shape[1]} modes, config wants {k}")
    if a.shape[0] != modes.shape[0]:
        raise ValueError(f"batch rows {a.shape[0]} != mode rows {modes.shape[0]}")
    carried = ff * (modes * sigma)
    q, r = ref_qr(np.concatenate([carried, a], axis=1))
    u, s, _ = ref_svd(r, want_vt=False)
    keep = np.argsort(-s, kind="stable")[:k]
    new_modes = q @ u[:, keep]
    new_sigma = s[keep]
    if rescue:
        drift = np.abs(new_modes.T @ new_modes - np.eye(k)).max()
        if drift > DRIFT_TOL:
            qq, rr = ref_qr(new_modes)
            new_sigma = new_sigma * np.abs(np.diag(rr))
            keep = np.argsort(-new_sigma, kind="stable")
            new_modes = qq[:, keep]
            new_sigma = new_sigma[keep]
    return new_modes, new_sigma


def ref_stream_all(batches, k, ff):
    """stream_all — streaming.py:119-133.  Returns (modes, sigma, history)."""
    modes = sigma = None
    history = []
    for b in batches:
        if modes is None:
            modes, sigma = ref_stream_init(b, k)
        else:
            modes, sigma = ref_stream_update(modes, sigma, b, k, ff)
        history.append(sigma.copy())
    if modes is None:
        raise ValueError("batch stream is empty")
    return modes, sigma, history


# --------------------------------------------------------------------------
# randomized streaming composition (F2): each step is
# low_rank_svd of [ff*U*diag(s) | A_i] with the same sketch config.
# --------------------------------------------------------------------------

def ref_rand_stream_init(a0, k, oversampling, power_iterations, seed, omega=None):
    u, s, _ = ref_low_rank_svd(a0, k, oversampling, power_iterations, seed, omega)
    return u, s


def ref_rand_stream_update(modes, sigma, a, k, ff, oversampling, power_iterations,
                           seed, omega=None):
    carried = ff * (modes * sigma)
    u, s, _ = ref_low_rank_svd(np.concatenate([carried, a], axis=1), k,
                               oversampling, power_iterations, seed, omega)
    return u, s


def ref_rand_stream_all(batches, k, ff, oversampling=10, power_iterations=1, seed=0):
    modes = sigma = None
    history = []
    for b in batches:
        if modes is None:
            modes, sigma = ref_rand_stream_init(b, k, oversampling, power_iterations, seed)
        else:
            modes, sigma = ref_rand_stream_update(modes, sigma, b, k, ff, oversampling,
                                                  power_iterations, seed)
        history.append(sigma.copy())
    return modes, sigma, history


# --------------------------------------------------------------------------
# row-parallel streaming (dsvd.py), ranks simulated in-process, in rank order
# --------------------------------------------------------------------------

def partition_bounds(rows, world_size):
    """Contiguous row split, first rows % P ranks one longer — datagen.py:118-136."""
    if world_size < 1:
        raise ValueError(f"world_size must be >= 1, got {world_size}")
    if world_size > rows:
        raise ValueError(f"world_size {world_size} exceeds row count {rows}")
    base, extra = divmod(rows, world_size)
    sizes = [base + (r < extra) for r in range(world_size)]
    ends = np.cumsum(sizes)
    return [(int(e - s), int(e)) for s, e in zip(sizes, ends)]


def _tsqr_ranks(blocks):
    """parallel_qr — dsvd.py:176-202: local QR per rank, QR of the rank-ordered
    stack of R factors at the root, Q slices lifted back."""
    if len(blocks) == 1:
        q, r = ref_qr(blocks[0])
        return [q], r
    local = [ref_qr(b) for b in blocks]
    heights = [r.shape[0] for _, r in local]
    q_stack, r_final = ref_qr(np.concatenate([r for _, r in local], axis=0))
    qs, off = [], 0
    for (ql, _), h in zip(local, heights):
        qs.append(ql @ q_stack[off:off + h])
        off += h
    return qs, r_final


def ref_parallel_stream_all(a_full, batch_edges, world_size, k, ff):
    """parallel_stream_initialize/incorporate (dsvd.py:205-242) over the
    partition_bounds split, then gather_modes (dsvd.py:245-251).
    batch_edges: list of (c0, c1) column ranges.  Returns (modes, sigma)."""
    bounds = partition_bounds(a_full.shape[0], world_size)
    local_modes = None
    sigma = None
    for bi, (c0, c1) in enumerate(batch_edges):
        blocks = []
        for r, (lo, hi) in enumerate(bounds):
            blk = a_full[lo:hi, c0:c1]
            if local_modes is not None:
                blk = np.concatenate([ff * (local_modes[r] * sigma), blk], axis=1)
            blocks.append(blk)
        qs, rr = _tsqr_ranks(blocks)
        u, s, _ = ref_svd(rr, want_vt=False)
        if local_modes is None:
            local_modes = [(q @ u)[:, :k] for q in qs]
            sigma = s[:k].copy()
        else:
            order = np.argsort(-s, kind="stable")
            local_modes = [(q @ u[:, order])[:, :k] for q in qs]
            sigma = s[order][:k].copy()
    return np.concatenate(local_modes, axis=0), sigma


# --------------------------------------------------------------------------
# input generators (datagen.py)
# --------------------------------------------------------------------------

def burgers_solution(x, t, reynolds=1000.0):
    """Analytic viscous Burgers in log space — datagen.py:49-73 (same operation
    order, so the bytes match the reference's)."""
    x = np.asarray(x, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    re = reynolds
    expo = 0.5 * (np.log1p(t) - re / 8.0) + re * x * x / (4.0 * (t + 1.0))
    return (x / (t + 1.0)) * np.exp(-np.logaddexp(0.0, expo))


def burgers_matrix(grid_points, n_snapshots, length=1.0, t_final=2.0, reynolds=1000.0,
                   rows=None):
    """Snapshot matrix u(x_i, t_j) on inclusive linspace grids — datagen.py:76-90.
    `rows=(lo, hi)` returns just that row slice (same values as the slice of
    the full matrix)."""
    x = np.linspace(0.0, length, grid_points)
    t = np.linspace(0.0, t_final, n_snapshots)
    if rows is not None:
        x = x[rows[0]:rows[1]]
    return burgers_solution(x[:, None], t[None, :], reynolds)


# --------------------------------------------------------------------------
# one-shot distributed SVD (dsvd.py:39-173, APMOS)
# --------------------------------------------------------------------------

def ref_generate_right_vectors(a, local_rank, method="svd"):
    """Leading right singular vectors / values of a local slice, zero-padded to
    local_rank columns — dsvd.py:80-124."""
    a = _check(a, "a_local")
    n = a.shape[1]
    if local_rank < 1:
        raise ValueError(f"local_rank must be >= 1, got {local_rank}")
    if local_rank > n:
        raise ValueError(f"local_rank {local_rank} exceeds the snapshot count {n}")
    if method == "svd":
        _, s_all, vt = ref_svd(a, want_vt=True)
        keep = min(local_rank, s_all.size)
        v, s = vt[:keep].T.copy(), s_all[:keep].copy()
    else:  # "gram": method of snapshots (dsvd.py:108-118)
        lam, vec = np.linalg.eigh(a.T @ a)
        order = np.argsort(-lam, kind="stable")
        lam = np.clip(lam[order], 0.0, None)
        vec = vec[:, order]
        idx = np.argmax(np.abs(vec), axis=0)
        sg = np.sign(vec[idx, np.arange(vec.shape[1])])
        sg[sg == 0.0] = 1.0
        keep = min(local_rank, n)
        v, s = (vec * sg)[:, :keep], np.sqrt(lam[:keep])
    if keep < local_rank:
        v = np.hstack([v, np.zeros((n, local_rank - keep))])
        s = np.concatenate([s, np.zeros(local_rank - keep)])
    return v, s


def ref_apmos(blocks, local_rank, global_rank, k, use_randomized=False, sketch=None):
    """apmos over rank-ordered row blocks — dsvd.py:127-173.  The gather of
    W_i = V_i S_i to the root is the rank-ordered concatenation; the root's
    factorization (svd_full, or low_rank_svd with sketch = (target_rank,
    oversampling, power_iterations, seed)) is what every rank receives.
    Returns (stacked modes, singular values)."""
    if global_rank > len(blocks) * local_rank:
        raise ValueError(f"global_rank {global_rank} exceeds the {len(blocks) * local_rank} columns "
                         f"the exchange can produce")
    w = np.concatenate([v * s for v, s in (ref_generate_right_vectors(b, local_rank) for b in blocks)], axis=1)
    if use_randomized:
        tr, ov, pi, seed = sketch if sketch is not None else (global_rank, 10, 1, 0)
        u, s, _ = ref_low_rank_svd(w, tr, ov, pi, seed)
    else:
        u, s, _ = ref_svd(w, want_vt=False)
    if s.size < global_rank:
        raise ValueError(f"stacked exchange matrix only has {s.size} singular values, "
                         f"global_rank is {global_rank}")
    x, lam = u[:, :global_rank], s[:global_rank]
    for j in range(k):
        if lam[j] == 0.0:
            raise ZeroDivisionError(f"mode {j} has a zero singular value and cannot be assembled")
    modes = np.concatenate([_check(b, "a_local") @ x[:, :k] / lam[:k] for b in blocks], axis=0)
    return modes, lam[:k].copy()


# --------------------------------------------------------------------------
# comparison metrics (harness only; sine-based so angles below 1e-8 resolve,
# SURVEY F5)
# --------------------------------------------------------------------------

def sigma_rel_err(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


def mode_angles(u, v):
    """Per-column sign-invariant angle between u[:, j] and v[:, j], computed
    from the sine (norm of the orthogonal residual), accurate to ~1e-16."""
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    un = u / np.linalg.norm(u, axis=0)
    vn = v / np.linalg.norm(v, axis=0)
    c = np.sum(un * vn, axis=0)
    resid = un - vn * c
    s = np.linalg.norm(resid, axis=0)
    return np.arctan2(s, np.abs(c))


def sine_angles(a, b):
    """Principal angles between column spans via scipy's sine-based routine."""
    import scipy.linalg
    return np.sort(scipy.linalg.subspace_angles(np.asarray(a), np.asarray(b)))


def aligned_mode_difference(a, b):
    """Sign-aligned per-column max-abs difference — linalg.py:165-179."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    sgn = np.sign(np.sum(a * b, axis=0))
    sgn = np.where(sgn == 0.0, 1.0, sgn)
    return np.max(np.abs(a * sgn - b), axis=0)
