"""Row-partitioned streaming SVD across GPUs — B200 drop-in for the reference's
parallel streaming pair and gather (dsvd.py:71-77, 205-251).

Reference (dsvd.py:176-202): local QR on every rank, gather of the R factors
at rank 0, QR of the stack, point-to-point return of Q slices, broadcast of R.
Here (one process per GPU, torch.distributed over NCCL):

    local Gram G_r = C_r^T C_r of the rank's panel [ff*U_r*S | A_r]   (libpsvd)
    allgather of the n x n G_r over NVLink, summed in rank order        (bitwise
        identical on every GPU: psvd_sum_ordered, no atomics)
    replicated top-K eigen + sign rule of sum_r G_r = R^T R             (libpsvd)
    local recompose U_r <- [U_r | A_r] W, local U_r^T U_r               (libpsvd)
    allgather of the K x K U_r^T U_r, Rayleigh refinement of sigma      (libpsvd)

Two small collectives per update (n*n*8 = 353 KB at n = 210, K*K*8) replace
gather + P-1 sends + broadcast.  Like the reference there is no drift rescue
on this path (dsvd.py:220-242).

With `config.sketch` set the update is the randomized one with the
row-partitioned exchange of §8(e): the library calls back (psvd_set_exchange)
for the rank-ordered sums of Y^T Y, (Y T)^T (Y T) and D P^T Y and for the
allgather of the per-rank argmax pairs of the tall sign rule; Omega is the
replicated host draw, so every rank runs the identical small factorizations.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as nat
from .errors import ProtocolError


@dataclass(frozen=True)
class LocalModes:
    """This rank's rows of the modes plus the replicated singular values (dsvd.py:71-77)."""

    modes: torch.Tensor
    singular_values: torch.Tensor


class RankContext:
    """rank / world_size / group of the row partition.  Wraps an initialized
    torch.distributed process group (NCCL on GPUs, gloo for CPU tests); with no
    process group it is the single-rank world (dsvd.py:185-186 fast path)."""

    def __init__(self, group=None):
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world_size = dist.get_world_size(group)
        else:
            self.rank, self.world_size = 0, 1


_PY_EXCHANGE = [0, 0]  # collectives / bytes received by allreduce_ordered (the Python-level exchange)


def allreduce_ordered(t, ctx, count=True):
    """Sum of `t` over ranks, added in rank order so every rank holds the same
    bits (an allgather + fixed-order sum).  count=False for the library's
    hooks, which the library counts itself."""
    if ctx.world_size == 1:
        return t
    if count:
        _PY_EXCHANGE[0] += 1
        _PY_EXCHANGE[1] += 8 * t.numel() * (ctx.world_size - 1)
    t = t.contiguous()
    if t.device.type == "cuda" and dist.get_backend(ctx.group) != "nccl":
        return allreduce_ordered(t.cpu(), ctx, count=False).to(t.device)  # gloo: host-staged (test harness)
    if t.device.type == "cuda":
        parts = torch.empty((ctx.world_size,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(parts, t, group=ctx.group)
        out = torch.empty_like(t)
        c = nat.context(t.device)
        nat.call("psvd_sum_ordered", c, nat.ptr(parts), ctx.world_size, t.numel(), nat.ptr(out),
                 nat.stream_ptr(t.device))
        return out
    parts = [torch.empty_like(t) for _ in range(ctx.world_size)]
    dist.all_gather(parts, t, group=ctx.group)
    out = parts[0].clone()
    for p in parts[1:]:
        out += p
    return out


class _Exchange:
    """ctypes hooks (psvd_set_exchange) running the rank-ordered allreduce / the
    allgather on this RankContext, ordered on the library's stream."""

    def __init__(self, ctx, dev):
        self.ctx, self.dev = ctx, dev
        self.error = None
        self.ar = nat.ALLREDUCE_FN(self._allreduce)
        self.ag = nat.ALLGATHER_FN(self._allgather)

    def _stream(self, stream):
        if not stream:  # the legacy default stream
            return torch.cuda.default_stream(self.dev)
        return torch.cuda.ExternalStream(stream, device=self.dev)

    def _device_collectives(self):
        return dist.get_backend(self.ctx.group) == "nccl"

    def _allreduce(self, user, ptr, count, stream):
        try:
            t = nat.wrap_device(ptr, count, self.dev)
            with torch.cuda.stream(self._stream(stream)):
                if self._device_collectives():
                    t.copy_(allreduce_ordered(t, self.ctx, count=False))
                else:  # gloo: stage through the host (blocking copies keep the stream order)
                    t.copy_(allreduce_ordered(t.cpu(), self.ctx, count=False).to(self.dev))
            return 0
        except Exception as e:  # noqa: BLE001 - reported through the return code
            self.error = e
            return 1

    def _allgather(self, user, send, count, recv, stream):
        try:
            src = nat.wrap_device(send, count, self.dev)
            dst = nat.wrap_device(recv, count * self.ctx.world_size, self.dev)
            with torch.cuda.stream(self._stream(stream)):
                if self._device_collectives():
                    dist.all_gather_into_tensor(dst, src, group=self.ctx.group)
                else:
                    parts = [torch.empty(int(count), dtype=torch.float64) for _ in range(self.ctx.world_size)]
                    dist.all_gather(parts, src.cpu(), group=self.ctx.group)
                    dst.copy_(torch.cat(parts).to(self.dev))
            return 0
        except Exception as e:  # noqa: BLE001
            self.error = e
            return 1


def _row_offset(ctx, rows, dev, cols=-1):
    """Global index of this rank's first row (prefix sum of the local row counts).  With `cols`,
    the ranks' column counts travel in the same allgather and must agree (ProtocolError)."""
    if ctx.world_size == 1:
        return 0, rows
    t = torch.tensor([rows, cols], dtype=torch.int64,
                     device=dev if dist.get_backend(ctx.group) == "nccl" else "cpu")
    parts = [torch.zeros_like(t) for _ in range(ctx.world_size)]
    dist.all_gather(parts, t, group=ctx.group)
    counts = [int(x[0].item()) for x in parts]
    widths = sorted({int(x[1].item()) for x in parts})
    if len(widths) > 1:
        raise ProtocolError(f"ranks disagree on the local panel width: {widths}")
    return sum(counts[:ctx.rank]), sum(counts)


_NCCL_COMMS = {}  # device index -> the process group whose communicator the library context holds


def _nccl_exchange(ctx):
    """The library's own NCCL data plane for this group: NCCL process groups, unless
    PSVD_EXCHANGE=python asks for the torch.distributed callbacks (diagnostics)."""
    if ctx.world_size == 1 or dist.get_backend(ctx.group) != "nccl":
        return False
    if os.environ.get("PSVD_EXCHANGE", "nccl") == "python":
        return False
    ok = ctypes.c_int(0)
    nat.lib().psvd_nccl_available(ctypes.byref(ok))
    return bool(ok.value)


def _ensure_nccl_comm(ctx, dev):
    """One NCCL communicator per library context, created from a unique id rank 0 draws and
    broadcasts over the process group (psvd_nccl_unique_id / psvd_nccl_init)."""
    key = dev.index
    if _NCCL_COMMS.get(key) is ctx.group and key in _NCCL_COMMS:
        return
    c = nat.context(dev)
    idt = torch.zeros(128, dtype=torch.uint8, device=dev)
    if ctx.rank == 0:
        buf = ctypes.create_string_buffer(128)
        nat.call("psvd_nccl_unique_id", c, buf)
        idt.copy_(torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8))
    src = dist.get_global_rank(ctx.group, 0) if ctx.group is not None else 0
    dist.broadcast(idt, src=src, group=ctx.group)
    raw = bytes(idt.cpu().numpy().tobytes())
    with torch.cuda.device(dev):
        nat.call("psvd_nccl_init", c, ctx.world_size, ctx.rank, raw)
    _NCCL_COMMS[key] = ctx.group


class exchange_hooks:
    """Context manager: the library's row-partitioned exchange for the calls inside.  On NCCL
    process groups the library issues its own in-stream ncclAllGather + rank-ordered sum
    (psvd_nccl_enable: no Python in the loop); on gloo (CPU / shared-GPU test harness) it calls
    back into torch.distributed (psvd_set_exchange).  suspend() / resume() bracket calls that
    must run without it."""

    def __init__(self, ctx, dev, row_offset=None):
        self.ctx, self.dev = ctx, dev
        self.off = row_offset
        self.ex = None
        self.nccl = False

    def resume(self):
        if self.ctx.world_size == 1:
            return
        if self.nccl:
            nat.call("psvd_nccl_enable", self.c, 1, self.off)
        else:
            nat.call("psvd_set_exchange", self.c, ctypes.cast(self.ex.ar, nat._vp), ctypes.cast(self.ex.ag, nat._vp),
                     None, self.ctx.world_size, self.off)

    def suspend(self):
        if self.ctx.world_size == 1:
            return
        if self.nccl:
            nat.call("psvd_nccl_enable", self.c, 0, 0)
        else:
            nat.call("psvd_set_exchange", self.c, None, None, None, 1, 0)

    def __enter__(self):
        self.c = nat.context(self.dev)
        if self.ctx.world_size == 1:
            return self
        if self.off is None:
            raise ValueError("exchange_hooks needs the rank's global row offset")
        self.nccl = _nccl_exchange(self.ctx)
        if self.nccl:
            try:
                _ensure_nccl_comm(self.ctx, self.dev)
            except RuntimeError as e:  # no usable libnccl in this process: the torch.distributed callbacks
                import warnings
                warnings.warn(f"library NCCL exchange unavailable ({e}); using torch.distributed callbacks")
                self.nccl = False
        if not self.nccl:
            self.ex = _Exchange(self.ctx, self.dev)
        self.resume()
        return self

    def __exit__(self, et, ev, tb):
        if self.ctx.world_size > 1:
            self.suspend()
            if et is not None and issubclass(et, RuntimeError) and self.ex is not None and self.ex.error is not None:
                raise self.ex.error
        return False


def exchange_stats(device=None):
    """(collectives issued, bytes received) at the exchange points since context creation: the
    library's (NCCL data plane / hooks) plus the Python-level rank-ordered sums of the per-update
    row-parallel path — the reference's CommStats counters (comm.py:74-88)."""
    out = (ctypes.c_longlong * 2)()
    nat.call("psvd_exchange_stats", nat.context(device), out)
    return int(out[0]) + _PY_EXCHANGE[0], int(out[1]) + _PY_EXCHANGE[1]


def _parallel_rand_update(ctx, U, sigma, A, sketch, ff, dev):
    from .linalg import randomized_update
    off, total = _row_offset(ctx, A.rows, dev, A.cols)
    if ctx.world_size == 1:
        return randomized_update(U, sigma, A, sketch, ff, dev)
    redo = []
    with exchange_hooks(ctx, dev, off):
        # PSVD_ST_SKETCHCOND comes from the summed Grams (identical bits on every rank), so every
        # rank asks for the redo together; it runs after the hooks of the fast update are released
        res = randomized_update(U, sigma, A, sketch, ff, dev, total_rows=total,
                                accurate=lambda: redo.append(True))
    if redo:
        return _parallel_accurate_rand_update(ctx, U, sigma, A, sketch, ff, dev, off)
    return res


def _parallel_accurate_rand_update(ctx, U, sigma, A, sketch, ff, dev, off):
    """The row-partitioned randomized step on the accurate route (linalg.accurate_randomized_update
    with the rows spread over the ranks): the reference's sequence (linalg.py:126-162) with a
    backward-stable qr after every product.  Tall factors (the sketch y = c omega, every power
    iteration's c z) are orthonormalized by parallel_qr; the small ones (z = c^T q, b^T = c^T q)
    are rank-ordered sums of the local products, so every rank factors identical bits; the tall
    sign rule takes the global argmax (ties: the lower global row, linalg.py:81-91)."""
    from . import linalg
    linalg.ACCURATE_RAND_UPDATES += 1
    k, l = sketch.target_rank, sketch.sketch_width
    kc = 0 if U is None else U.cols
    M, n = A.rows, kc + A.cols
    c, st = nat.context(dev), nat.stream_ptr(dev)
    om = linalg.device_omega(n, sketch, dev)

    def nn(X, W, w):  # X (M x X.cols) times a column-major X.cols x w device matrix: local rows only
        wp, wld = (nat.ptr(W), W.shape[-1]) if torch.is_tensor(W) else (nat._vp(W.data_ptr()), W.ld)
        Y = nat.DevMat.empty(M, w, dev)
        nat.call("psvd_nn_product", c, M, nat._vp(X.data_ptr()), X.ld, X.cols, wp, wld, w,
                 nat._vp(Y.data_ptr()), Y.ld, st)
        return Y

    def tn(X, Q):  # X^T Q summed over the ranks: (n x l) column-major, the same bits everywhere
        Z = torch.empty((l, n), dtype=torch.float64, device=dev)
        nat.call("psvd_tn_product", c, M, nat._vp(X.data_ptr()), X.ld, n, nat._vp(Q.data_ptr()), Q.ld, l,
                 nat.ptr(Z), n, st)
        return allreduce_ordered(Z, ctx)

    with torch.cuda.device(dev):
        C = nat.DevMat.empty(M, n, dev)
        if kc:
            torch.mul(U.view, (ff * sigma)[None, :], out=C.view[:, :kc])
        C.view[:, kc:].copy_(A.view)
        q = nat.as_device_colmajor(parallel_qr(ctx, nn(C, om, l).view, dev).q, dev, "q")
        for _ in range(sketch.power_iterations):
            Z = nat.as_device_colmajor(tn(C, q).t(), dev, "z")
            z, _ = linalg._tall_qr(Z, dev)
            q = nat.as_device_colmajor(parallel_qr(ctx, nn(C, z, l).view, dev).q, dev, "q")
        res = linalg.svd_full(tn(C, q).t(), want_vt=True, device=dev)  # b^T = u s vt: b's left vectors are vt's rows
        W = torch.empty((k, l), dtype=torch.float64, device=dev)       # (l x k) column-major = vt[:k]^T
        W.copy_(res.vt[:k, :])
        out = nn(q, W, k)
        _sign_by_global_peak(ctx, out, off, dev)
        sig = res.s[:k].clone()
        status = nat.read_status(c, reset=True, device=dev)
    if status & nat.ST_NONFINITE:
        raise ValueError("a_local contains non-finite entries")
    return out, sig


def _sign_by_global_peak(ctx, X, off, dev):
    """linalg.py:81-91 on the row-stacked matrix: each column's largest-|.| entry over all ranks
    (ties keep the lower global row: the lower rank, then torch's first maximal index) made
    positive.  X: this rank's rows (DevMat), flipped in place."""
    k = X.cols
    v = X.view
    if X.rows:
        idx = torch.argmax(v.abs(), dim=0)
        mine = v[idx, torch.arange(k, device=dev)]
    else:
        mine = torch.zeros(k, dtype=torch.float64, device=dev)
    peaks = torch.zeros((ctx.world_size, k), dtype=torch.float64, device=dev)
    peaks[ctx.rank] = mine
    peaks = allreduce_ordered(peaks, ctx)          # one rank's value per row, zeros elsewhere: exact
    best = torch.argmax(peaks.abs(), dim=0)        # first maximal value: the lowest rank
    signs = torch.sign(peaks[best, torch.arange(k, device=dev)])
    signs[signs == 0.0] = 1.0
    v.mul_(signs[None, :])


def _parallel_update(ctx, U, sigma, A, k, ff, dev):
    c = nat.context(dev)
    with torch.cuda.device(dev):
        st = nat.stream_ptr(dev)
        M, B = A.rows, A.cols
        kc = 0 if U is None else U.cols
        n = kc + B
        uptr = nat._vp(U.data_ptr() if U is not None else 0)
        uld = U.ld if U is not None else 0
        sptr = nat.ptr(sigma if U is not None else None)
        G = torch.empty((n, n), dtype=torch.float64, device=dev)
        nat.call("psvd_gram", c, M, uptr, uld, sptr, float(ff), kc, nat._vp(A.data_ptr()), A.ld, B, nat.ptr(G), st)
        G = allreduce_ordered(G, ctx)
        W = torch.empty((k, n), dtype=torch.float64, device=dev)  # col-major n x k
        sig = torch.empty(k, dtype=torch.float64, device=dev)
        nat.call("psvd_core_eig", c, nat.ptr(G), n, sptr, float(ff), kc, k, nat.ptr(W), nat.ptr(sig), st)
        out = nat.DevMat.empty(M, k, dev)
        utu = torch.empty((k, k), dtype=torch.float64, device=dev)
        nat.call("psvd_recompose", c, M, uptr, uld, kc, nat._vp(A.data_ptr()), A.ld, B, nat.ptr(W), k,
                 nat._vp(out.data_ptr()), out.ld, nat.ptr(utu), st)
        utu = allreduce_ordered(utu, ctx)  # global U^T U: Rayleigh refinement of sigma, unit columns
        nat.call("psvd_refine_normalize", c, M, nat._vp(out.data_ptr()), out.ld, k, nat.ptr(utu), nat.ptr(sig), st)
        status = nat.read_status(c, reset=True, device=dev)
        if status & nat.ST_ILLCOND and not status & nat.ST_NONFINITE:
            # kept spectrum beyond the Gram route's accuracy (identical sigma bits on every rank, so
            # every rank takes this branch): the accurate route, its Grams summed over the ranks
            from . import streaming
            streaming.ACCURATE_UPDATES += 1
            off, _ = _row_offset(ctx, M, dev)
            with exchange_hooks(ctx, dev, off):
                nat.call("psvd_stream_update_accurate", c, M, uptr, uld, sptr, float(ff), kc, nat._vp(A.data_ptr()),
                         A.ld, B, k, 0, nat._vp(out.data_ptr()), out.ld, nat.ptr(sig), st)
            status |= nat.read_status(c, reset=True, device=dev)
    if status & nat.ST_NONFINITE:
        raise ValueError("a_local contains non-finite entries")
    return out, sig


def _device(x):
    if isinstance(x, torch.Tensor) and x.device.type == "cuda":
        return x.device
    nat.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def parallel_stream_initialize(ctx, a0_local, config):
    """Distributed stream_initialize (dsvd.py:205-217)."""
    dev = _device(a0_local)
    A = nat.as_device_colmajor(a0_local, dev, "a0_local")
    k = config.k_modes
    if A.cols < k:
        raise ValueError(f"initial batch has {A.cols} columns, need at least k_modes={k}")
    if config.sketch is not None:
        out, sig = _parallel_rand_update(ctx, None, None, A, config.sketch, config.forget_factor, dev)
    else:
        out, sig = _parallel_update(ctx, None, None, A, k, config.forget_factor, dev)
    return LocalModes(out.view, sig)


def parallel_stream_incorporate(ctx, state, a_new_local, config):
    """Distributed stream_incorporate (dsvd.py:220-242)."""
    dev = _device(state.modes)
    k = config.k_modes
    if state.modes.shape[1] != k:
        raise ValueError(f"state carries {state.modes.shape[1]} modes, config wants {k}")
    A = nat.as_device_colmajor(a_new_local, dev, "a_new_local")
    if A.rows != state.modes.shape[0]:
        raise ValueError(f"batch rows {A.rows} != mode rows {state.modes.shape[0]}")
    U = nat.as_device_colmajor(state.modes, dev, "modes")
    sigma = nat.as_device_vector(state.singular_values, dev, k, "singular_values")
    if config.sketch is not None:
        out, sig = _parallel_rand_update(ctx, U, sigma, A, config.sketch, config.forget_factor, dev)
    else:
        out, sig = _parallel_update(ctx, U, sigma, A, k, config.forget_factor, dev)
    return LocalModes(out.view, sig)


def parallel_stream_all(ctx, batches_local, config, device=None):
    """Row-partitioned stream over this rank's batches (B200 extension: the reference drives
    parallel_stream_initialize / parallel_stream_incorporate batch by batch, cli.py:262-276;
    same update rule, dsvd.py:205-242, no drift rescue).  The iterable is consumed lazily, one
    window at a time.  Deterministic configs run in windows
    through the pipelined psvd_stream_run with the exchange hooks: per update a rank-ordered
    sum of the streaming Gram (first rank contributes the already-global U^T U block) and of
    U^T U, so every rank factors identical bits; the next batch's A^T A still overlaps the
    replicated core solve.  Randomized configs with a sketch of at most 32 columns and K <= 16
    run the pipelined psvd_rand_stream_run with the same exchange (rank-ordered sums of the
    look-ahead sketch tiles, the projection Grams and partials, the argmax pairs of the sign
    rule); wider sketches update batch by batch.  Returns (LocalModes, history of singular
    values)."""
    from .streaming import (RAND_STREAM_MAX_K, RAND_STREAM_MAX_WIDTH, StreamState, _run_rand_window, _run_window,
                            window_length)
    k = config.k_modes
    it = iter(batches_local)
    first = next(it, None)
    if first is None:
        raise ValueError("batch stream is empty")
    dev = torch.device(device) if device is not None else _device(first)
    sk = config.sketch
    if sk is not None and (sk.sketch_width > RAND_STREAM_MAX_WIDTH or k > RAND_STREAM_MAX_K):
        # wide sketches: per batch (psvd_rand_update's GEMM route with the exchange); lazily
        st = parallel_stream_initialize(ctx, first, config)
        hist = [st.singular_values.clone()]
        for b in it:
            st = parallel_stream_incorporate(ctx, st, b, config)
            hist.append(st.singular_values.clone())
        return st, hist
    c = nat.context(dev)
    wlen = window_length(first, dev)
    if ctx.world_size > 1:
        # one window length on every rank (row blocks differ by a row, so the memory bound could round
        # differently): the windows' exchanges must line up
        wl = torch.tensor([wlen], dtype=torch.int64)
        if dist.get_backend(ctx.group) == "nccl":
            wl = wl.to(dev)
        dist.all_reduce(wl, op=dist.ReduceOp.MIN, group=ctx.group)
        wlen = int(wl.item())
    off = total = None
    ex = None  # exchange_hooks, entered at the first pipelined window
    state, hist = None, []

    def per_batch(st0, window):
        # the batches this route handles one update at a time (too wide for the pipelined kernels,
        # or an update of the window left the Gram route's accuracy range): the row-parallel update
        # (accurate route where gated), the run's exchange hooks off meanwhile
        if ex is not None:
            ex.suspend()
        try:
            st = None if st0 is None else LocalModes(st0.modes, st0.singular_values)
            out = []
            for m in window:
                st = parallel_stream_initialize(ctx, m, config) if st is None else \
                    parallel_stream_incorporate(ctx, st, m, config)
                out.append(st.singular_values.clone())
            it0 = -1 if st0 is None else st0.iteration
            return StreamState(st.modes, st.singular_values, it0 + len(window)), out
        finally:
            if ex is not None:
                ex.resume()

    def run(window):
        nonlocal state, off, total, ex
        M = window[0].rows
        ok = ctypes.c_int(0)
        if sk is None:
            nat.call("psvd_stream_run_supported", c, M, k, max(m.cols for m in window), ctypes.byref(ok))
        else:
            nat.call("psvd_rand_stream_run_supported", c, M, k, sk.sketch_width, sk.power_iterations,
                     max(m.cols for m in window), ctypes.byref(ok))
        flag = torch.tensor([float(ok.value)], dtype=torch.float64,
                            device=dev if (ctx.world_size > 1 and dist.get_backend(ctx.group) == "nccl") else "cpu")
        if ctx.world_size > 1:  # every rank takes the same route
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=ctx.group)
        if not flag.item():
            state, h = per_batch(state, window)
            hist.extend(h)
            return
        if off is None:
            off, total = _row_offset(ctx, M, dev)
            if ctx.world_size > 1:
                ex = exchange_hooks(ctx, dev, off).__enter__()
        if sk is None:
            state, h = _run_window(state, window, config, dev, rescue=False, ok=True, on_illcond=per_batch,
                                   total_rows=total)
        else:
            state, h = _run_rand_window(state, window, config, dev, supported=True,
                                        on_illcond=per_batch if ctx.world_size > 1 else None, total_rows=total)
        hist.extend(h)

    try:
        window = [nat.as_device_colmajor(first, dev, "a_local")]
        for b in it:
            if len(window) == wlen:
                run(window)
                window = []
            window.append(nat.as_device_colmajor(b, dev, "a_local"))
        run(window)
    except (RuntimeError, ValueError):
        if ex is not None and ex.ex is not None and ex.ex.error is not None:
            raise ex.ex.error
        raise
    finally:
        if ex is not None:
            ex.suspend()
    return LocalModes(state.modes, state.singular_values), hist


def gather_modes(ctx, local_modes, root=0):
    """Stack per-rank mode blocks at the root in rank order (dsvd.py:245-251).
    Returns the (total_rows, K) tensor at the root and None elsewhere: one gather to the
    root (NCCL on device buffers; staged through the host on gloo), not an allgather."""
    m = local_modes.modes
    if ctx.world_size == 1:
        return m.contiguous()
    dev = m.device
    stage = dist.get_backend(ctx.group) != "nccl"
    rows = torch.tensor([m.shape[0], m.shape[1]], dtype=torch.int64, device="cpu" if stage else dev)
    all_rows = [torch.zeros_like(rows) for _ in range(ctx.world_size)]
    dist.all_gather(all_rows, rows, group=ctx.group)
    counts = [int(r[0].item()) for r in all_rows]
    widths = sorted({int(r[1].item()) for r in all_rows})
    if len(widths) > 1:
        raise ProtocolError(f"ranks hold different numbers of modes: {widths}")
    mx = max(counts)
    pad = torch.zeros((mx, m.shape[1]), dtype=m.dtype, device="cpu" if stage else dev)
    pad[: m.shape[0]] = m
    dst = dist.get_global_rank(ctx.group, root) if ctx.group is not None else root
    if ctx.rank != root:
        dist.gather(pad, None, dst=dst, group=ctx.group)
        return None
    parts = [torch.empty_like(pad) for _ in range(ctx.world_size)]
    dist.gather(pad, parts, dst=dst, group=ctx.group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0).to(dev)


def parallel_qr(ctx, a_local, device=None):
    """Tall-skinny QR of the row-stacked global matrix (dsvd.py:176-202): QrResult(q_local,
    r) with r identical on every rank.  World size 1 is qr_factor.  Otherwise a
    distributed CholeskyQR2 (the rank-robust Gram-deflation route, psvd_qr_robust, when the
    first Cholesky flags an ill-conditioned or rank-deficient matrix): every Gram is a
    rank-ordered allreduce of the local Grams, so every rank factors identical bits, and
    q_local stays local (no q slices on the wire, unlike the reference's gather / send /
    broadcast of the TSQR tree)."""
    from .linalg import QrResult, qr_factor
    if ctx.world_size == 1:
        return qr_factor(a_local, device)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    A = nat.as_device_colmajor(a_local, dev, "a_local")
    m, n = A.rows, A.cols
    c = nat.context(dev)
    st = nat.stream_ptr(dev)
    off, m_total = _row_offset(ctx, m, dev, n)
    if m_total < n:
        raise ValueError(f"parallel_qr needs at least as many rows as columns ({m_total} < {n})")

    nccl = dist.get_backend(ctx.group) == "nccl"

    # column norms spanning more than 1e3 (rank-ordered sum of the local squares: the same bits, so the same
    # decision, on every rank): the unit-norm columns are factored and r's columns scaled back, as
    # linalg._equilibrated_tall_qr does on one GPU (Householder's q does not depend on the scaling)
    scale = None
    if n > 1:
        cn = torch.sqrt(allreduce_ordered((A.view * A.view).sum(dim=0), ctx))
        if float(cn.min()) < 1e-3 * float(cn.max()):
            scale = torch.where(cn > 0, cn, torch.ones_like(cn))
            As = nat.DevMat.empty(m, n, dev)
            torch.div(A.view, scale[None, :], out=As.view)
            A = As

    def gram(X):
        G = torch.empty((n, n), dtype=torch.float64, device=dev)
        nat.call("psvd_gram", c, X.rows, nat._vp(0), 0, nat._vp(0), 1.0, 0, nat._vp(X.data_ptr()), X.ld, n,
                 nat.ptr(G), st)
        if nccl:
            return allreduce_ordered(G, ctx).contiguous()
        return allreduce_ordered(G.cpu(), ctx).to(dev).contiguous()  # gloo: host-staged (CPU test harness)

    def chol(G):
        R = torch.empty((n, n), dtype=torch.float64, device=dev)
        T = torch.empty((n, n), dtype=torch.float64, device=dev)
        nat.call("psvd_chol", c, nat.ptr(G), n, nat.ptr(R), nat.ptr(T), st)
        return R, T

    def times(X, T):
        Y = nat.DevMat.empty(X.rows, n, dev)
        nat.call("psvd_nn_product", c, X.rows, nat._vp(X.data_ptr()), X.ld, n, nat.ptr(T), n, n,
                 nat._vp(Y.data_ptr()), Y.ld, st)
        return Y

    def rmul(Ra, Rb):
        out = torch.empty((n, n), dtype=torch.float64, device=dev)
        nat.call("psvd_small_matmul", c, nat.ptr(Ra), n, 0, nat.ptr(Rb), n, nat.ptr(out), n, n, n, n, st)
        return out

    with torch.cuda.device(dev):
        G = gram(A)
        R1, T1 = chol(G)
        flag = ctypes.c_int(0)
        nat.call("psvd_chol_illcond", c, ctypes.byref(flag), st)
        if flag.value:
            # beyond CholeskyQR2 (the flag comes from identical bits on every rank): the rank-robust
            # Gram-deflation route with every Gram / projection summed over the ranks
            Q = nat.DevMat.empty(m, n, dev)
            R = torch.empty((n, n), dtype=torch.float64, device=dev)
            with exchange_hooks(ctx, dev, off):
                nat.call("psvd_qr_robust", c, m, n, nat._vp(A.data_ptr()), A.ld, nat._vp(Q.data_ptr()), Q.ld,
                         nat.ptr(R), st)
        else:
            Q = times(A, T1)
            R2, T2 = chol(gram(Q))
            Q = times(Q, T2)
            R = rmul(R2, R1)
        st_word = nat.read_status(c, reset=True, device=dev)
    if st_word & nat.ST_NONFINITE:
        raise ValueError("a_local contains non-finite entries")
    return QrResult(Q.view, R.T if scale is None else R.T * scale[None, :])
