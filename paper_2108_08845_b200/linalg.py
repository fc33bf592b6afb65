"""Randomized range finder / low-rank SVD configuration and the randomized
streaming update (reference linalg.py:33-62, 126-162)."""

from __future__ import annotations

from collections import namedtuple
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


RAND_MAX_WIDTH = 112  # CHOL_NMAX: the widest sketch of the fused randomized update (psvd_rand_update)
ACCURATE_RAND_UPDATES = 0  # randomized updates redone on the accurate route (diagnostics / tests)


def accurate_randomized_update(U, sigma, A, sketch, ff, device, omega=None):
    """The randomized step on the accurate route: the reference's own sequence (linalg.py:126-162) with
    a backward-stable qr after every product -- the panel [ff U diag(sigma) | A] materialized, q =
    randomized_range(panel) (psvd_nn_product / psvd_tn_product / psvd_qr, the rank-robust Householder-quality
    route included), b^T = panel^T q, the Jacobi svd of b^T (relative accuracy on every value), u = q u_b[:, :K]
    and the tall sign rule.  Slower than psvd_rand_update (the panel is read once per product and written once);
    taken when that update reports PSVD_ST_SKETCHCOND.  Returns (DevMat M x K, sigma (K,))."""
    import torch
    from . import _native as nat
    global ACCURATE_RAND_UPDATES
    ACCURATE_RAND_UPDATES += 1
    k, l = sketch.target_rank, sketch.sketch_width
    kc = 0 if U is None else U.cols
    M, n = A.rows, kc + A.cols
    ctx, st = nat.context(device), nat.stream_ptr(device)
    with torch.cuda.device(device):
        C = nat.DevMat.empty(M, n, device)
        if kc:
            torch.mul(U.view, (ff * sigma)[None, :], out=C.view[:, :kc])
        C.view[:, kc:].copy_(A.view)
        q = nat.as_device_colmajor(_range_of(C, sketch, device, omega), device, "q")
        Z = torch.empty((l, n), dtype=torch.float64, device=device).t()  # n x l column-major: b^T = panel^T q
        nat.call("psvd_tn_product", ctx, M, nat._vp(C.data_ptr()), C.ld, n, nat._vp(q.data_ptr()), q.ld, l,
                 nat._vp(Z.data_ptr()), n, st)
        res = svd_full(Z, want_vt=True, device=device)  # b^T = u s vt, so b's left vectors are vt's rows
        W = torch.empty((k, l), dtype=torch.float64, device=device)  # (l x k) column-major = vt[:k]^T
        W.copy_(res.vt[:k, :])
        out = nat.DevMat.empty(M, k, device)
        nat.call("psvd_nn_product", ctx, M, nat._vp(q.data_ptr()), q.ld, l, nat.ptr(W), l, k,
                 nat._vp(out.data_ptr()), out.ld, st)
        nat.call("psvd_sign_by_peak", ctx, nat._vp(out.data_ptr()), out.ld, M, k, st)
        sig = res.s[:k].clone()
    return out, sig


def randomized_update(U, sigma, A, sketch, ff, device, check=True, total_rows=None, omega=None, accurate=True):
    """One randomized step: low_rank_svd([ff*U*diag(sigma) | A], sketch) on the
    device (linalg.py:150-162 composed per batch).  U: DevMat or None.
    total_rows: rows of the whole (row-partitioned) panel for the width check.
    omega: optional device test matrix (n x l, column-major) replacing the Philox draw.
    accurate: redo the step on accurate_randomized_update when the device reports
    PSVD_ST_SKETCHCOND (a sketch direction at or below 3e-7 of the largest: the Gram-based
    orthonormalization no longer reproduces the reference's Householder qr to 1e-10); the
    row-partitioned caller passes its own redo (a callable: dsvd._parallel_accurate_rand_update,
    the same sequence with the products summed over the ranks).
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
    if l > RAND_MAX_WIDTH:
        # wider than the fused update's one-CTA solvers (psvd_rand_update refuses it): the same sequence
        # composed from the any-width kernels -- the accurate route (the row-partitioned caller's own)
        if callable(accurate):
            return accurate()
        return accurate_randomized_update(U, sigma, A, sketch, ff, device, omega=omega)
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
            if accurate and (st & nat.ST_SKETCHCOND):
                if callable(accurate):
                    return accurate()
                return accurate_randomized_update(U, sigma, A, sketch, ff, device, omega=omega)
    return out, sig


def low_rank_svd(a, config, device=None):
    """Randomized truncated SVD of a device/host matrix (linalg.py:150-162):
    SvdResult(u (m x target_rank), s (target_rank,), vt (target_rank x n)) as CUDA
    tensors, the sign rule applied to u's columns and vt's rows together."""
    import torch
    from . import _native as nat
    dev = _dev(device)
    A = nat.as_device_colmajor(a, dev, "a")
    n_acc = ACCURATE_RAND_UPDATES
    u, s = randomized_update(None, None, A, config, 1.0, dev)
    k, l = config.target_rank, config.sketch_width
    ctx = nat.context(dev)
    with torch.cuda.device(dev):
        if ACCURATE_RAND_UPDATES != n_acc:
            # the any-width / accurate route ran (no fused update whose small factors psvd_rand_last_vt could
            # read): b's right vectors are vt_j = u_j^T a / s_j, rows signed with u's columns
            Z = torch.empty((k, A.cols), dtype=torch.float64, device=dev).t()  # n x k column-major: a^T u
            nat.call("psvd_tn_product", ctx, A.rows, nat._vp(A.data_ptr()), A.ld, A.cols, nat._vp(u.data_ptr()), u.ld,
                     k, nat._vp(Z.data_ptr()), A.cols, nat.stream_ptr(dev))
            return SvdResult(u.view, s, (Z / torch.where(s > 0, s, torch.ones_like(s))[None, :]).T)
        vt = torch.empty((A.cols, k), dtype=torch.float64, device=dev)  # (k x n) column-major
        nat.call("psvd_rand_last_vt", ctx, A.cols, l, k, nat.ptr(vt), k, nat.stream_ptr(dev))
    return SvdResult(u.view, s, vt.T)


# --------------------------------------------------------------------------
# dense factorizations of the reference's linalg boundary (linalg.py:94-147)
# --------------------------------------------------------------------------

QrResult = namedtuple("QrResult", ["q", "r"])
SvdResult = namedtuple("SvdResult", ["u", "s", "vt"])

QR_SMEM_COLS = 112      # CHOL_NMAX: R and R^-1 of a Gram in one CTA's shared memory (wider: psvd_big.cu)
JACOBI_SMEM_COLS = 160  # JACOBI_NMAX: the one-CTA Jacobi's rotation accumulator (wider: psvd_big.cu)


def _dev(device):
    import torch
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _check(ctx, dev, what):
    from . import _native as nat
    st = nat.read_status(ctx, reset=True, device=dev)
    if st & nat.ST_NONFINITE:
        raise ValueError(f"{what} contains non-finite entries")
    if st & nat.ST_NOCONVERGE:
        from .errors import ConvergenceError
        raise ConvergenceError(f"{what}: SVD did not converge")


def _tall_qr(A, dev):
    """(Q DevMat m x n, R (n x n) tensor) of a tall DevMat (m >= n) on the device: CholeskyQR2,
    or the rank-robust route (psvd_qr_robust) when the first Cholesky flags an
    ill-conditioned or rank-deficient input; numerically null directions get an orthonormal
    completion in q, as Householder QR gives (linalg.py:94-104)."""
    import torch
    from . import _native as nat
    m, n = A.rows, A.cols
    ctx = nat.context(dev)
    Q = nat.DevMat.empty(m, n, dev)
    R = torch.empty((n, n), dtype=torch.float64, device=dev)  # column-major (n x n): R.T is the matrix
    with torch.cuda.device(dev):
        try:
            nat.call("psvd_qr", ctx, m, n, nat._vp(A.data_ptr()), A.ld, nat._vp(Q.data_ptr()), Q.ld, nat.ptr(R),
                     nat.stream_ptr(dev))
        except ValueError:
            nat.read_status(ctx, reset=True, device=dev)  # the failed call's status bits are reported here
            raise
    return Q, R.T


def _equilibrated_tall_qr(A, dev):
    """_tall_qr of a matrix whose column norms span more than 1e3: the factorization is taken of the unit-norm
    columns and R's columns are scaled back (a = (a D^-1) D; Householder's q does not depend on the scaling,
    linalg.py:94-104).  The scaled matrix is as well conditioned as column scaling can make it, so a
    column-graded input stays on CholeskyQR2 and its small columns keep rows of R accurate relative to their
    own size, as Householder's are, instead of falling to the rank-robust route at rounding level."""
    import torch
    from . import _native as nat
    if A.cols < 2:
        return _tall_qr(A, dev)
    cn = torch.linalg.vector_norm(A.view, dim=0)
    if not float(cn.min()) < 1e-3 * float(cn.max()):  # (also the non-finite case: reported by the kernels)
        return _tall_qr(A, dev)
    scale = torch.where(cn > 0, cn, torch.ones_like(cn))
    Xs = nat.DevMat.empty(A.rows, A.cols, dev)
    torch.div(A.view, scale[None, :], out=Xs.view)
    Q, R = _tall_qr(Xs, dev)
    return Q, R * scale[None, :]


def qr_factor(a, device=None):
    """Reduced QR with diag(r) >= 0 (linalg.py:94-104): QrResult(q (m x min(m, n)),
    r (min(m, n) x n)) as CUDA tensors.  Tall inputs run CholeskyQR2 (shifted
    CholeskyQR3 when ill conditioned) on the device; wide ones factor their leading
    square block and form r's remaining columns as q^T a.  Any width (the Cholesky factors
    live in one CTA's shared memory up to 112 columns, in global memory beyond)."""
    import torch
    from . import _native as nat
    dev = _dev(device)
    A = nat.as_device_colmajor(a, dev, "a")
    m, n = A.rows, A.cols
    ctx = nat.context(dev)
    if m >= n:
        Q, R = _equilibrated_tall_qr(A, dev)
        _check(ctx, dev, "a")
        return QrResult(Q.view, R)
    lead = nat.DevMat(A.view[:, :m], A.ld)
    Q, R0 = _equilibrated_tall_qr(lead, dev)
    rest = torch.empty((n - m, m), dtype=torch.float64, device=dev)  # column-major (m x (n - m))
    with torch.cuda.device(dev):
        nat.call("psvd_tn_product", ctx, m, nat._vp(Q.data_ptr()), Q.ld, m,
                 nat._vp(A.data_ptr() + 8 * A.ld * m), A.ld, n - m, nat.ptr(rest), m, nat.stream_ptr(dev))
    _check(ctx, dev, "a")
    return QrResult(Q.view, torch.cat([R0, rest.T], dim=1))


def _svd_tall(A, dev, want_vt):
    """(U DevMat m x n, s (n,), V (n x n) column-major tensor view) of a tall DevMat."""
    import torch
    from . import _native as nat
    m, n = A.rows, A.cols
    ctx = nat.context(dev)
    st = nat.stream_ptr(dev)
    s = torch.empty(n, dtype=torch.float64, device=dev)
    Vb = torch.empty((n, n), dtype=torch.float64, device=dev)  # column-major V: Vb.T
    U = nat.DevMat.empty(m, n, dev)
    with torch.cuda.device(dev):
        # Graded columns (norms spanning more than 1e3) are factored in order of decreasing norm, the
        # pre-sorting of preconditioned Jacobi (Drmac-Veselic): without it a matrix whose small columns
        # come first (Burgers rows near x = 1: the early snapshots are ~1e-80) leaves R row-graded the
        # wrong way for the column rotations, and the sweeps stall (ConvergenceError where the
        # reference's dgesdd, linalg.py:107-123, converges).  V's rows are put back at the end.
        perm = colscale = None
        if n > 1:
            cn = torch.linalg.vector_norm(A.view, dim=0)
            if float(cn.min()) < 1e-3 * float(cn.max()):
                order = torch.argsort(cn, descending=True, stable=True)
                if not bool((order == torch.arange(n, device=dev)).all()):
                    perm = order
                    Ap = nat.DevMat.empty(m, n, dev)
                    Ap.view.copy_(A.view[:, perm])
                    A = Ap
                    cn = cn[perm]
                # ... and their QR is taken of the unit-norm columns, R's columns scaled back (exact in the
                # scaling: a = (a D^-1) D): the scaled matrix is as well conditioned as column scaling makes
                # it (van der Sluis), so CholeskyQR2 returns the triangular, properly graded R a Householder
                # QR would; the rank-robust route on the unscaled columns leaves rounding-level rows in R that
                # the sweeps cannot resolve (stall on gradings past ~1e-60)
                colscale = torch.where(cn > 0, cn, torch.ones_like(cn))

        def graded_qr(X):
            if colscale is None:
                return _tall_qr(X, dev)
            Xs = nat.DevMat.empty(m, n, dev)
            torch.div(X.view, colscale[None, :], out=Xs.view)
            Q, R = _tall_qr(Xs, dev)
            return Q, R * colscale[None, :]

        if n <= QR_SMEM_COLS:
            # QR-preconditioned one-sided Jacobi: A = Q R, R = U_R S V^T, U = Q U_R
            if m > n:
                Q, R = graded_qr(A)
                Rm = nat.as_device_colmajor(R, dev, "r")
            else:
                Q, Rm = None, A
            nat.call("psvd_jacobi", ctx, nat._vp(Rm.data_ptr()), Rm.ld, Rm.rows, n, nat.ptr(s), nat.ptr(Vb), n, st)
            UR = nat.DevMat.empty(n, n, dev)
            nat.call("psvd_small_matmul", ctx, nat._vp(Rm.data_ptr()), Rm.ld, 0, nat.ptr(Vb), n,
                     nat._vp(UR.data_ptr()), UR.ld, n, n, n, st)
            nat.call("psvd_scale_cols", ctx, nat._vp(UR.data_ptr()), UR.ld, n, n, nat.ptr(s), 1, st)
            if Q is None:
                U = UR
            else:
                nat.call("psvd_nn_product", ctx, m, nat._vp(Q.data_ptr()), Q.ld, n, nat._vp(UR.data_ptr()), UR.ld, n,
                         nat._vp(U.data_ptr()), U.ld, st)
        elif n <= JACOBI_SMEM_COLS and m <= 4 * n:
            nat.call("psvd_jacobi", ctx, nat._vp(A.data_ptr()), A.ld, m, n, nat.ptr(s), nat.ptr(Vb), n, st)
            nat.call("psvd_nn_product", ctx, m, nat._vp(A.data_ptr()), A.ld, n, nat.ptr(Vb), n, n,
                     nat._vp(U.data_ptr()), U.ld, st)
            nat.call("psvd_scale_cols", ctx, nat._vp(U.data_ptr()), U.ld, m, n, nat.ptr(s), 1, st)
        else:
            # wide cores: A = Q R (CholeskyQR2 / shifted CholeskyQR3), then the multi-CTA one-sided
            # Jacobi on R^T (psvd_big.cu): R^T J = U~ S gives R = J S U~^T, so U_R = J (the
            # accumulated rotations) and V_R = U~; U = Q U_R.  Relative accuracy on every
            # singular value, as dgesdd of the reference's R (linalg.py:107-123).
            Q, R = graded_qr(A)
            Rm = nat.as_device_colmajor(R, dev, "r")
            UR = nat.DevMat.empty(n, n, dev)
            VR = nat.DevMat.empty(n, n, dev)
            nat.call("psvd_jacobi_uv", ctx, nat._vp(Rm.data_ptr()), Rm.ld, n, n, 1, nat.ptr(s),
                     nat._vp(UR.data_ptr()), UR.ld, nat._vp(VR.data_ptr()), VR.ld, st)
            nat.call("psvd_nn_product", ctx, m, nat._vp(Q.data_ptr()), Q.ld, n, nat._vp(UR.data_ptr()), UR.ld, n,
                     nat._vp(U.data_ptr()), U.ld, st)
            Vb.T.copy_(VR.view)
        # Left vectors of weak directions: u_j = a v_j / s_j is orthogonal to the others only to
        # eps s_1 / s_j, and undefined for s_j = 0, while the reference's dgesdd returns an orthonormal u
        # whatever the spectrum (linalg.py:107-123).  So when the spectrum spans more than 1e8, the columns
        # of numerically null values are cleared and u is re-orthonormalized by our own qr (diag(r) >= 0:
        # well-determined columns keep their direction and sign; null ones get an orthonormal completion).
        sh = s.cpu()
        if n > 1 and float(sh[-1]) < 1e-8 * float(sh[0]):
            null = s <= (16.0 * n * torch.finfo(torch.float64).eps) * s[0]
            if bool(null.any()):
                U.view[:, null] = 0.0
            U, _ = _tall_qr(U, dev)
        if perm is not None:  # a[:, perm] = u s v'^T: v[perm[i], :] = v'[i, :] (Vb holds v's columns as rows)
            Vp = torch.empty_like(Vb)
            Vp[:, perm] = Vb
            Vb = Vp
        nat.call("psvd_sign_pair", ctx, nat._vp(U.data_ptr()), U.ld, m, n, nat.ptr(Vb), n, n, st)
    return U, s, Vb.T


def svd_full(a, want_vt=True, device=None):
    """Thin SVD (linalg.py:107-123): SvdResult(u, s descending, vt or None) as CUDA
    tensors with the reference's sign rule (each u column's largest-magnitude entry
    positive, first occurrence; vt's rows follow).  Any width (of the taller orientation):
    CholeskyQR then one-sided Jacobi on R (relative accuracy; the one-CTA kernels up to
    112 / 160 columns, the multi-CTA Jacobi of psvd_big.cu beyond).  Non-convergence
    raises ConvergenceError."""
    from . import _native as nat
    dev = _dev(device)
    A = nat.as_device_colmajor(a, dev, "a")
    ctx = nat.context(dev)
    if A.rows >= A.cols:
        U, s, V = _svd_tall(A, dev, want_vt)
        _check(ctx, dev, "a")
        return SvdResult(U.view, s, V.T if want_vt else None)
    # wide: svd(a^T) = V S U^T; the sign rule is on the left factor, so apply it again
    At = nat.as_device_colmajor(A.view.T, dev, "a")
    Vw, s, Uw = _svd_tall(At, dev, True)  # a^T = Vw diag(s) Uw^T
    u = nat.DevMat.empty(A.rows, A.rows, dev)
    u.view.copy_(Uw)
    vt_cols = nat.DevMat.empty(A.cols, A.rows, dev)  # v = Vw (n x k), column-major
    vt_cols.view.copy_(Vw.view)
    with __import__("torch").cuda.device(dev):
        nat.call("psvd_sign_pair", ctx, nat._vp(u.data_ptr()), u.ld, A.rows, A.rows, nat._vp(vt_cols.data_ptr()),
                 vt_cols.ld, A.cols, nat.stream_ptr(dev))
    _check(ctx, dev, "a")
    return SvdResult(u.view, s, vt_cols.view.T if want_vt else None)


def randomized_range(a, config, device=None):
    """Orthonormal basis of the sketched range (linalg.py:126-147): q = qr(a Omega).q
    with Omega = Philox(seed).standard_normal((n, width)), then `power_iterations`
    rounds of q = qr(a^T q).q, q = qr(a q).q.  Returns q (m x width), CUDA."""
    import torch
    from . import _native as nat
    dev = _dev(device)
    A = nat.as_device_colmajor(a, dev, "a")
    return _range_of(A, config, dev, None)


def _range_of(A, config, dev, omega):
    """randomized_range of a DevMat; omega: optional device test matrix (n x width, column-major)."""
    import torch
    from . import _native as nat
    m, n = A.rows, A.cols
    w = config.sketch_width
    if w > min(m, n):
        raise ValueError(f"sketch width {w} exceeds min(a.shape) = {min(m, n)}")
    ctx = nat.context(dev)
    st = nat.stream_ptr(dev)
    om = device_omega(n, config, dev) if omega is None else omega  # column-major n x w
    Y = nat.DevMat.empty(m, w, dev)
    with torch.cuda.device(dev):
        nat.call("psvd_nn_product", ctx, m, nat._vp(A.data_ptr()), A.ld, n, nat.ptr(om), n, w,
                 nat._vp(Y.data_ptr()), Y.ld, st)
        q, _ = _tall_qr(Y, dev)
        for _ in range(config.power_iterations):
            Z = nat.DevMat.empty(n, w, dev)
            nat.call("psvd_tn_product", ctx, m, nat._vp(A.data_ptr()), A.ld, n, nat._vp(q.data_ptr()), q.ld, w,
                     nat._vp(Z.data_ptr()), Z.ld, st)
            z, _ = _tall_qr(Z, dev)
            nat.call("psvd_nn_product", ctx, m, nat._vp(A.data_ptr()), A.ld, n, nat._vp(z.data_ptr()), z.ld, w,
                     nat._vp(Y.data_ptr()), Y.ld, st)
            q, _ = _tall_qr(Y, dev)
    _check(ctx, dev, "a")
    return q.view


def aligned_mode_difference(a, b):
    """Per-column max |a*sign - b| after matching each column's sign (linalg.py:165-176)."""
    import torch
    a = torch.as_tensor(a, dtype=torch.float64)
    b = torch.as_tensor(b, dtype=torch.float64, device=a.device)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    signs = torch.sign(torch.sum(a * b, dim=0))
    signs[signs == 0.0] = 1.0
    return torch.max(torch.abs(a * signs - b), dim=0).values


def subspace_angles(a, b, device=None):
    """Principal angles (ascending, radians) between the column spans (linalg.py:179-192):
    arccos of the singular values of qa^T qb, as the reference computes them."""
    import torch
    qa = qr_factor(a, device).q
    qb = qr_factor(b, device).q
    c = svd_full(_tn(qa, qb, device), want_vt=False, device=device).s
    return torch.sort(torch.arccos(torch.clamp(c, -1.0, 1.0))).values


def _tn(x, y, device):
    """x^T y for tall column-major CUDA matrices, on the library's TN product."""
    import torch
    from . import _native as nat
    dev = _dev(device)
    X = nat.as_device_colmajor(x, dev, "x")
    Y = nat.as_device_colmajor(y, dev, "y")
    out = torch.empty((Y.cols, X.cols), dtype=torch.float64, device=dev)  # column-major X.cols x Y.cols
    with torch.cuda.device(dev):
        nat.call("psvd_tn_product", nat.context(dev), X.rows, nat._vp(X.data_ptr()), X.ld, X.cols,
                 nat._vp(Y.data_ptr()), Y.ld, Y.cols, nat.ptr(out), X.cols, nat.stream_ptr(dev))
    return out.T
