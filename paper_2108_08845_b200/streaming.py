"""Streaming truncated SVD over column batches — B200 drop-in for the
reference's streaming.py (StreamConfig/StreamState/stream_initialize/
stream_incorporate/stream_all, /root/reference/pkg/src/parsvd/streaming.py:28-133).

Same update rule, same validation errors, same sign convention; the state
lives in HBM (torch CUDA tensors) and every update is a fixed sequence of
libpsvd kernels on the current stream:

    Gram of the virtual panel [ff*U*S | A]  ->  top-K eigen + sign rule (one CTA)
    ->  recompose U_new = [U | A] W  (+ U_new^T U_new)  ->  drift rescue (gated)

The optional `sketch` field (a RandomSketchConfig) selects the randomized
update: each step is low_rank_svd of [ff*U*S | A].
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as nat
from .linalg import RandomSketchConfig, randomized_update

# streaming.py:25 — re-orthonormalize when max|U^T U - I| exceeds this
ORTHO_DRIFT_TOL = 1e-8


@dataclass(frozen=True)
class StreamConfig:
    """k_modes kept per update, forget factor in (0, 1], nominal batch width
    (streaming.py:28-50).  `sketch` (B200 extension) switches to the
    randomized update; None keeps the reference's deterministic rule."""

    k_modes: int
    forget_factor: float = 0.95
    batch_columns: int = 1
    sketch: Optional[RandomSketchConfig] = None

    def __post_init__(self):
        if self.k_modes < 1:
            raise ValueError(f"k_modes must be >= 1, got {self.k_modes}")
        if not 0.0 < self.forget_factor <= 1.0:
            raise ValueError(f"forget_factor must be in (0, 1], got {self.forget_factor}")
        if self.batch_columns < 1:
            raise ValueError(f"batch_columns must be >= 1, got {self.batch_columns}")
        if self.sketch is not None and self.sketch.target_rank != self.k_modes:
            raise ValueError(
                f"sketch target_rank {self.sketch.target_rank} must equal k_modes {self.k_modes}")


@dataclass(frozen=True)
class StreamState:
    """modes (M x K, orthonormal columns; a column-major CUDA tensor view),
    singular_values (K, descending, CUDA), iteration count (streaming.py:53-60).
    numpy arrays are accepted on input and moved to the device."""

    modes: torch.Tensor
    singular_values: torch.Tensor
    iteration: int

    def to_host(self, pinned=True):
        """(modes, singular_values) as CPU tensors; modes is a column-major view filled
        by one dense device-to-host copy (into pinned memory by default)."""
        return (nat.to_host_colmajor(self.modes.detach(), pinned),
                self.singular_values.detach().cpu())

    def numpy(self):
        """(modes, singular_values) as host numpy arrays (modes Fortran-ordered)."""
        m, s = self.to_host(pinned=True)
        return np.array(m.numpy(), order="F", copy=True), s.numpy().copy()


def _device_of(*objs):
    for o in objs:
        if isinstance(o, torch.Tensor) and o.device.type == "cuda":
            return o.device
        if isinstance(o, nat.DevMat):
            return o.t.device
    nat.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


LAST_STATUS = 0  # device status word of the last checked update (diagnostics: PSVD_ST_* bits)
ACCURATE_UPDATES = 0  # updates recomputed on the accurate route (the Gram route's gate fired)
PIPELINED_RAND_WINDOWS = 0  # windows run by the pipelined randomized stream (psvd_rand_stream_run)


def _check_status(ctx, device, what):
    global LAST_STATUS
    st = nat.read_status(ctx, reset=True, device=device)
    LAST_STATUS = st
    if st & nat.ST_NONFINITE:
        raise ValueError(f"{what} contains non-finite entries")
    return st


def deterministic_update(U, sigma, A, k, ff, rescue, device, check=True, accurate_gate=True):
    """One deterministic update on the device.  U: DevMat or None (initialize),
    sigma: (Kc,) CUDA tensor, A: DevMat.  Returns (DevMat M x k, sigma (k,)).
    The Gram route runs first; when its conditioning gate fires (PSVD_ST_ILLCOND) the update
    is recomputed by psvd_stream_update_accurate (streaming.py:97-103 at any conditioning)."""
    ctx = nat.context(device)
    with torch.cuda.device(device):
        st = nat.stream_ptr(device)
        M, B = A.rows, A.cols
        kc = 0 if U is None else U.cols
        out = nat.DevMat.empty(M, k, device)
        sig = torch.empty(k, dtype=torch.float64, device=device)
        args = (ctx, M, nat._vp(U.data_ptr() if U is not None else 0), U.ld if U is not None else 0,
                nat.ptr(sigma if U is not None else None), float(ff), kc, nat._vp(A.data_ptr()), A.ld, B, k,
                int(bool(rescue)), nat._vp(out.data_ptr()), out.ld, nat.ptr(sig), st)
        nat.call("psvd_stream_update", *args)
        if check or accurate_gate:
            what = "a_new" if U is not None else "a0"
            if _check_status(ctx, device, what) & nat.ST_ILLCOND:
                # kept spectrum beyond the Gram route's accuracy (sigma_1 / sigma_K > 300): redo the
                # update on the R-factor route (Gram deflation basis + Jacobi of the small factor)
                global ACCURATE_UPDATES
                ACCURATE_UPDATES += 1
                nat.call("psvd_stream_update_accurate", *args)
                _check_status(ctx, device, what)
    return out, sig


def stream_initialize(a0, config, device=None):
    """Initial state from the first batch (streaming.py:63-78)."""
    dev = torch.device(device) if device is not None else _device_of(a0)
    A = nat.as_device_colmajor(a0, dev, "a0")
    k = config.k_modes
    if A.cols < k:
        raise ValueError(f"initial batch has {A.cols} columns, need at least k_modes={k}")
    if A.rows < k:
        raise ValueError(f"initial batch has {A.rows} rows, need at least k_modes={k}")
    if config.sketch is not None:
        u, s = randomized_update(None, None, A, config.sketch, config.forget_factor, dev)
    else:
        u, s = deterministic_update(None, None, A, k, config.forget_factor, False, dev)
    return StreamState(u.view, s, 0)


def stream_incorporate(state, a_new, config):
    """Fold one batch into the state (streaming.py:81-116)."""
    dev = _device_of(state.modes, a_new)
    k = config.k_modes
    modes = state.modes
    if modes.ndim != 2:
        raise ValueError("state.modes must be 2-D")
    if modes.shape[1] != k:
        raise ValueError(f"state carries {modes.shape[1]} modes, config wants {k}")
    A = nat.as_device_colmajor(a_new, dev, "a_new")
    if A.rows != modes.shape[0]:
        raise ValueError(f"batch rows {A.rows} != mode rows {modes.shape[0]}")
    U = nat.as_device_colmajor(modes, dev, "modes")
    sigma = nat.as_device_vector(state.singular_values, dev, k, "singular_values")
    if config.sketch is not None:
        u, s = randomized_update(U, sigma, A, config.sketch, config.forget_factor, dev)
    else:
        u, s = deterministic_update(U, sigma, A, k, config.forget_factor, True, dev)
    return StreamState(u.view, s, state.iteration + 1)


STREAM_WINDOW = 8  # most batches resident on the device per pipelined run (host batches: uploads in flight)
STREAM_WINDOW_RESIDENT = 32  # ... when the batches already are device tensors (nothing to upload)
STREAM_WINDOW_MEM_FRACTION = 0.25  # ... and at most this share of the device's memory


def window_length(batch, device):
    """Batches per pipelined window: STREAM_WINDOW (STREAM_WINDOW_RESIDENT for device tensors: every window
    boundary costs the pipeline its head, the first batch's Gram, and its tail, the last core solve, ~2 ms
    at config-2 shapes), fewer when they would take more than STREAM_WINDOW_MEM_FRACTION of HBM (at least
    2, so the look-ahead Gram still overlaps)."""
    shape = getattr(batch, "shape", None)
    if shape is None or len(shape) != 2:
        return STREAM_WINDOW
    cap = STREAM_WINDOW_RESIDENT if (torch.is_tensor(batch) and batch.is_cuda) else STREAM_WINDOW
    nbytes = 8 * int(shape[0]) * int(shape[1])
    total = torch.cuda.get_device_properties(torch.device(device)).total_memory
    return int(max(2, min(cap, (STREAM_WINDOW_MEM_FRACTION * total) // max(nbytes, 1))))


def _run_window(state, mats, config, dev, ready=None, rescue=True, ok=None, on_illcond=None, total_rows=None):
    """Deterministic updates over device batches `mats` with look-ahead
    (psvd_stream_run): the next batch's A^T A overlaps the current core solve.
    `ready`: per-batch upload events (or None) the device work waits on.  When an update
    of the window trips the Gram route's conditioning gate, the window is redone batch by
    batch from its input state: on_illcond(state, mats) (the row-parallel caller), else the
    serial per-update path with its accurate route.  total_rows: rows of the whole row-partitioned
    panel (the shape checks are the global matrix's; a rank's block may be shorter than K)."""
    k = config.k_modes
    M = mats[0].rows
    for m in mats:
        if m.rows != M:
            raise ValueError(f"batch rows {m.rows} != mode rows {M}")
    if state is None and mats[0].cols < k:
        raise ValueError(f"initial batch has {mats[0].cols} columns, need at least k_modes={k}")
    rows = M if total_rows is None else total_rows
    if state is None and rows < k:
        raise ValueError(f"initial batch has {rows} rows, need at least k_modes={k}")
    ctx = nat.context(dev)
    nb = len(mats)
    if ok is None:
        ok = ctypes.c_int(0)
        nat.call("psvd_stream_run_supported", ctx, M, k, max(m.cols for m in mats), ctypes.byref(ok))
        ok = ok.value
    if not ok:
        # batches too wide for the pipelined kernels: one psvd_stream_update per batch
        # (wide Grams on the tall-skinny TN GEMM), same update rule
        if ready is not None:
            for e in ready:
                if e is not None:
                    torch.cuda.current_stream(dev).wait_event(e)
        hist = []
        for m in mats:
            if state is None:
                state = stream_initialize(m, config, dev)
            else:
                state = stream_incorporate(state, m, config)
            hist.append(state.singular_values.clone())
        return state, hist
    with torch.cuda.device(dev):
        if state is not None:
            U = nat.as_device_colmajor(state.modes, dev, "modes")
            sig = nat.as_device_vector(state.singular_values, dev, k, "singular_values")
            kc, uptr, uld, sptr = k, nat._vp(U.data_ptr()), U.ld, nat.ptr(sig)
        else:
            U = sig = None
            kc, uptr, uld, sptr = 0, nat._vp(0), 0, nat._vp(0)
        outs = [nat.DevMat.empty(M, k, dev) for _ in range(2)]
        hist = torch.empty((nb, k), dtype=torch.float64, device=dev)
        A = (nat._vp * nb)(*[nat._vp(m.data_ptr()) for m in mats])
        lda = (ctypes.c_int64 * nb)(*[m.ld for m in mats])
        B = (ctypes.c_int * nb)(*[m.cols for m in mats])
        fin = ctypes.c_int(0)
        rd = None
        if ready is not None and any(e is not None for e in ready):
            rd = (nat._vp * nb)(*[nat._vp(e.cuda_event if e is not None else 0) for e in ready])
        nat.call("psvd_stream_run", ctx, M, uptr, uld, sptr, kc, nb, A, lda, B, k, float(config.forget_factor),
                 int(bool(rescue)),
                 nat._vp(outs[0].data_ptr()), nat._vp(outs[1].data_ptr()), outs[0].ld, nat.ptr(hist),
                 ctypes.byref(fin), rd, nat.stream_ptr(dev))
        if _check_status(ctx, dev, "a_new") & nat.ST_ILLCOND:
            # an update of the window left the Gram route's accuracy range: redo the window from its
            # input state one batch at a time (each update gated onto the accurate route as needed)
            if on_illcond is not None:
                return on_illcond(state, mats)
            return _run_window(state, mats, config, dev, None, rescue, ok=0)
    it0 = -1 if state is None else state.iteration
    new_state = StreamState(outs[fin.value].view, hist[nb - 1].clone(), it0 + nb)
    return new_state, [hist[i] for i in range(nb)]


RAND_STREAM_MAX_WIDTH = 32  # widest sketch of the pipelined randomized run (narrow TMA passes)
RAND_STREAM_MAX_K = 16      # most modes of the pipelined run (its U = Q W argmax kernel)


def _run_rand_window(state, mats, config, dev, ready=None, supported=None, on_illcond=None, total_rows=None):
    """Randomized updates over device batches `mats` through the pipelined
    psvd_rand_stream_run (SURVEY R9 per batch; the next batch's state-independent
    sketch overlaps the current small solves, U is written once at the end)."""
    from .linalg import device_omega
    sk = config.sketch
    k, l, q = sk.target_rank, sk.sketch_width, sk.power_iterations
    M = mats[0].rows
    for m in mats:
        if m.rows != M:
            raise ValueError(f"batch rows {m.rows} != mode rows {M}")
    if state is None and mats[0].cols < k:
        raise ValueError(f"initial batch has {mats[0].cols} columns, need at least k_modes={k}")
    for i, m in enumerate(mats):
        n = (k if (state is not None or i > 0) else 0) + m.cols
        rows = M if total_rows is None else total_rows  # the row-partitioned panel's check is global
        if l > min(rows, n):
            raise ValueError(f"sketch width {l} exceeds min(a.shape) = {min(rows, n)}")
    ctx = nat.context(dev)
    nb = len(mats)
    ok = ctypes.c_int(1 if supported else 0)
    if supported is None:
        nat.call("psvd_rand_stream_run_supported", ctx, M, k, l, q, max(m.cols for m in mats), ctypes.byref(ok))
    if not ok.value:  # passes beyond the pipelined kernels: psvd_rand_update per batch (wide route)
        if ready is not None:
            for e in ready:
                if e is not None:
                    torch.cuda.current_stream(dev).wait_event(e)
        hist = []
        for m in mats:
            state = stream_initialize(m, config, dev) if state is None else stream_incorporate(state, m, config)
            hist.append(state.singular_values.clone())
        return state, hist
    with torch.cuda.device(dev):
        if state is not None:
            U = nat.as_device_colmajor(state.modes, dev, "modes")
            sig = nat.as_device_vector(state.singular_values, dev, k, "singular_values")
            kc, uptr, uld, sptr = k, nat._vp(U.data_ptr()), U.ld, nat.ptr(sig)
        else:
            U = sig = None
            kc, uptr, uld, sptr = 0, nat._vp(0), 0, nat._vp(0)
        out = nat.DevMat.empty(M, k, dev)
        hist = torch.empty((nb, k), dtype=torch.float64, device=dev)
        oms = [device_omega((k if (state is not None or i > 0) else 0) + m.cols, sk, dev) for i, m in enumerate(mats)]
        A = (nat._vp * nb)(*[nat._vp(m.data_ptr()) for m in mats])
        lda = (ctypes.c_int64 * nb)(*[m.ld for m in mats])
        B = (ctypes.c_int * nb)(*[m.cols for m in mats])
        Om = (nat._vp * nb)(*[nat._vp(o.data_ptr()) for o in oms])
        rd = None
        if ready is not None and any(e is not None for e in ready):
            rd = (nat._vp * nb)(*[nat._vp(e.cuda_event if e is not None else 0) for e in ready])
        global PIPELINED_RAND_WINDOWS
        PIPELINED_RAND_WINDOWS += 1
        nat.call("psvd_rand_stream_run", ctx, M, uptr, uld, sptr, kc, nb, A, lda, B, k, l, q,
                 float(config.forget_factor), Om, nat._vp(out.data_ptr()), out.ld, nat.ptr(hist), rd,
                 nat.stream_ptr(dev))
        status = _check_status(ctx, dev, "a_new")
        if status & nat.ST_NOCONVERGE:
            from .errors import ConvergenceError
            raise ConvergenceError("randomized core SVD did not converge")
        if status & nat.ST_SKETCHCOND:
            # a sketch of the window left the Gram-based orthonormalization's accuracy range: redo the window
            # from its input state one update at a time (each one gated onto the accurate route as needed);
            # on_illcond(state, mats) is the row-parallel caller's redo
            if on_illcond is not None:
                return on_illcond(state, mats)
            hist2 = []
            for m in mats:
                state = stream_initialize(m, config, dev) if state is None else stream_incorporate(state, m, config)
                hist2.append(state.singular_values.clone())
            return state, hist2
    it0 = -1 if state is None else state.iteration
    return StreamState(out.view, hist[nb - 1].clone(), it0 + nb), [hist[i] for i in range(nb)]


def stream_all(batches, config, device=None):
    """Initialize on the first batch, incorporate the rest (streaming.py:119-133).
    Returns (final_state, history) with the singular values after every step.
    The iterable is consumed lazily, one window at a time (window_length: at most
    STREAM_WINDOW batches and a quarter of HBM), so past batches are never retained.
    Deterministic streams run in windows of resident batches
    through the pipelined psvd_stream_run (pinned host batches are uploaded on a
    side stream, overlapping the updates); randomized ones (sketch width <= 32)
    through the pipelined psvd_rand_stream_run, wider sketches per batch."""
    state = None
    history = []
    if config.sketch is not None and (config.sketch.sketch_width > RAND_STREAM_MAX_WIDTH
                                      or config.k_modes > RAND_STREAM_MAX_K):
        for batch in batches:
            if state is None:
                state = stream_initialize(batch, config, device)
            else:
                state = stream_incorporate(state, batch, config)
            history.append(state.singular_values.clone())
    else:
        dev = None if device is None else torch.device(device)
        run = _run_window if config.sketch is None else _run_rand_window
        window, ready = [], []
        wlen = None
        for batch in batches:
            if dev is None:
                dev = _device_of(batch)
            if wlen is None:
                wlen = window_length(batch, dev)
            # pinned host batches upload on a side stream: later copies overlap earlier updates
            m, ev = nat.upload_async(batch, dev, "a0" if state is None and not window else "a_new")
            window.append(m)
            ready.append(ev)
            if len(window) == wlen:
                state, h = run(state, window, config, dev, ready)
                history.extend(h)
                window, ready = [], []
        if window:
            state, h = run(state, window, config, dev, ready)
            history.extend(h)
    if state is None:
        raise ValueError("batch stream is empty")
    return state, history
