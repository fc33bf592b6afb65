"""ctypes binding of libpsvd.so (include/psvd.h) and device-buffer plumbing.

The product path has no CPU fallback: if the library or a CUDA device is
missing, every compute entry point raises.  torch is used only to own device
memory and streams (plumbing); all arithmetic on the hot path happens in the
library's kernels.
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

import numpy as np
import torch

from .errors import ConvergenceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libpsvd.so")
if os.environ.get("PSVD_LIB_VARIANT"):  # diagnostics: an in-tree build variant (tools/, A/B timing)
    LIB_PATH = os.path.join(_HERE, "lib", "libpsvd." + os.environ["PSVD_LIB_VARIANT"] + ".so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "psvd.h")

PSVD_OK, PSVD_EINVAL, PSVD_ENOCONV, PSVD_ECUDA = 0, 1, 2, 3
ST_NONFINITE, ST_NOCONVERGE, ST_RESCUE, ST_RANKDEF, ST_CHOLFAIL, ST_ILLCOND, ST_SKETCHCOND = 1, 2, 4, 8, 16, 32, 64

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_dbl = ctypes.c_double
_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/psvd.h
_SIGS = {
    "psvd_version": (_c_int, []),
    "psvd_create": (_c_int, [_c_int, ctypes.POINTER(_vp)]),
    "psvd_destroy": (_c_int, [_vp]),
    "psvd_last_error": (ctypes.c_char_p, [_vp]),
    "psvd_launch_count": (ctypes.c_longlong, [_vp]),
    "psvd_set_drift_tol": (_c_int, [_vp, _c_dbl]),
    "psvd_set_exchange": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _c_i64]),
    "psvd_last_core_path": (_c_int, [_vp, ctypes.POINTER(_c_int)]),
    "psvd_path_counters": (_c_int, [_vp, ctypes.POINTER(_c_i64)]),
    "psvd_sym_topk": (_c_int, [_vp, _vp, _c_int, _c_int, _vp, _c_i64, _vp, _vp]),
    "psvd_sign_by_peak": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_int, _vp]),
    "psvd_tn_product": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _vp, _c_i64, _vp]),
    "psvd_eig_phase_cycles": (_c_int, [_vp, ctypes.POINTER(ctypes.c_longlong)]),
    "psvd_read_status": (_c_int, [_vp, ctypes.POINTER(_c_int), _c_int, _vp]),
    "psvd_gram": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_dbl, _c_int, _vp, _c_i64, _c_int, _vp, _vp]),
    "psvd_core_eig": (_c_int, [_vp, _vp, _c_int, _vp, _c_dbl, _c_int, _c_int, _vp, _vp, _vp]),
    "psvd_recompose": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _vp, _c_int, _vp,
                                _c_i64, _vp, _vp]),
    "psvd_fused_pass": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _vp, _c_int,
                                 _vp, _c_i64, _vp, _vp, _c_int, _c_int, _vp, _vp]),
    "psvd_refine_normalize": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _vp, _vp, _vp]),
    "psvd_drift_rescue": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _vp, _vp, _c_dbl, _vp]),
    "psvd_stream_update": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_dbl, _c_int, _vp, _c_i64, _c_int,
                                    _c_int, _c_int, _vp, _c_i64, _vp, _vp]),
    "psvd_stream_run": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_int, _c_int, ctypes.POINTER(_vp),
                                 ctypes.POINTER(_c_i64), ctypes.POINTER(_c_int), _c_int, _c_dbl, _c_int, _vp, _vp,
                                 _c_i64, _vp, ctypes.POINTER(_c_int), ctypes.POINTER(_vp), _vp]),
    "psvd_rand_update": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_dbl, _c_int, _vp, _c_i64, _c_int, _c_int,
                                  _c_int, _c_int, _vp, _vp, _c_i64, _vp, _vp]),
    "psvd_rand_stream_run": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_int, _c_int, ctypes.POINTER(_vp),
                                      ctypes.POINTER(_c_i64), ctypes.POINTER(_c_int), _c_int, _c_int, _c_int,
                                      _c_dbl, ctypes.POINTER(_vp), _vp, _c_i64, _vp, ctypes.POINTER(_vp), _vp]),
    "psvd_chol": (_c_int, [_vp, _vp, _c_int, _vp, _vp, _vp]),
    "psvd_chol_shift": (_c_int, [_vp, _vp, _c_int, _c_i64, _vp]),
    "psvd_chol_illcond": (_c_int, [_vp, ctypes.POINTER(_c_int), _vp]),
    "psvd_nn_product": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _vp, _c_i64, _vp]),
    "psvd_small_matmul": (_c_int, [_vp, _vp, _c_int, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "psvd_qr": (_c_int, [_vp, _c_i64, _c_int, _vp, _c_i64, _vp, _c_i64, _vp, _vp]),
    "psvd_jacobi": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_int, _vp, _vp, _c_i64, _vp]),
    "psvd_sign_pair": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_int, _vp, _c_i64, _c_i64, _vp]),
    "psvd_stream_update_accurate": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_dbl, _c_int, _vp, _c_i64, _c_int,
                                             _c_int, _c_int, _vp, _c_i64, _vp, _vp]),
    "psvd_qr_robust": (_c_int, [_vp, _c_i64, _c_int, _vp, _c_i64, _vp, _c_i64, _vp, _vp]),
    "psvd_nccl_available": (_c_int, [ctypes.POINTER(_c_int)]),
    "psvd_nccl_unique_id": (_c_int, [_vp, ctypes.c_char_p]),
    "psvd_nccl_init": (_c_int, [_vp, _c_int, _c_int, ctypes.c_char_p]),
    "psvd_nccl_enable": (_c_int, [_vp, _c_int, _c_i64]),
    "psvd_nccl_destroy": (_c_int, [_vp]),
    "psvd_exchange_stats": (_c_int, [_vp, ctypes.POINTER(ctypes.c_longlong)]),
    "psvd_transpose": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp]),
    "psvd_gram_timing": (_c_int, [_vp, _c_int, ctypes.POINTER(_c_dbl)]),
    "psvd_jacobi_uv": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_int, _c_int, _vp, _vp, _c_i64, _vp, _c_i64, _vp]),
    "psvd_scale_cols": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_int, _vp, _c_int, _vp]),
    "psvd_rand_last_vt": (_c_int, [_vp, _c_int, _c_int, _c_int, _vp, _c_i64, _vp]),
    "psvd_stream_run_supported": (_c_int, [_vp, _c_i64, _c_int, _c_int, ctypes.POINTER(_c_int)]),
    "psvd_rand_stream_run_supported": (_c_int, [_vp, _c_i64, _c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_c_int)]),
    "psvd_sum_ordered": (_c_int, [_vp, _vp, _c_int, _c_i64, _vp, _vp]),
    "psvd_burgers": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_int, _c_dbl,
                              _c_dbl, _c_dbl, _vp]),
}

_lib = None
_lock = threading.RLock()
_ctxs = {}


def header_symbols():
    """Function names declared in include/psvd.h."""
    with open(HEADER) as f:
        txt = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*)\s+(psvd_\w+)\s*\(", txt, re.M)))


def lib():
    """Load libpsvd.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)")
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def _raise(rc, ctx):
    msg = lib().psvd_last_error(ctx).decode(errors="replace")
    if rc == PSVD_EINVAL:
        raise ValueError(msg)
    if rc == PSVD_ENOCONV:
        raise ConvergenceError(msg)
    raise RuntimeError(f"libpsvd CUDA error: {msg}")


def call(name, ctx, *args):
    rc = getattr(lib(), name)(ctx, *args)
    if rc != PSVD_OK:
        _raise(rc, ctx)


def path_counters(ctx):
    """(narrow TMA, TMA Gram, cp.async Gram, general cp.async, wide route) pass counts."""
    out = (_c_i64 * 5)()
    call("psvd_path_counters", ctx, out)
    return tuple(out)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2108_08845_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")


def context(device=None):
    """The library context of a CUDA device (created once per process)."""
    require_cuda()
    if device is None:
        idx = torch.cuda.current_device()
    else:
        d = torch.device(device)
        idx = d.index if d.index is not None else torch.cuda.current_device()  # 'cuda' = the current device
    if idx not in _ctxs:
        with _lock:
            if idx not in _ctxs:
                p = _vp()
                rc = lib().psvd_create(idx, ctypes.byref(p))
                if rc != PSVD_OK:
                    raise RuntimeError(f"psvd_create failed on cuda:{idx} (rc={rc})")
                _ctxs[idx] = p
    return _ctxs[idx]


def stream_ptr(device=None):
    return _vp(torch.cuda.current_stream(device).cuda_stream)


def read_status(ctx, reset=True, device=None):
    st = _c_int(0)
    call("psvd_read_status", ctx, ctypes.byref(st), int(reset), stream_ptr(device))
    return st.value


def ptr(t):
    return _vp(t.data_ptr()) if t is not None else _vp(0)


# --------------------------------------------------------------------- device matrices

class DevMat:
    """Column-major fp64 device matrix: `t` is the (rows x cols) torch view with
    strides (1, ld); ld is even and the base 16-byte aligned (the library's
    128-bit loads)."""

    __slots__ = ("t", "rows", "cols", "ld")

    def __init__(self, t, ld):
        self.t = t
        self.rows, self.cols = t.shape
        self.ld = ld

    @classmethod
    def empty(cls, rows, cols, device):
        ld = rows + (rows & 1)
        buf = torch.empty((max(cols, 1), ld), dtype=torch.float64, device=device)
        return cls(buf[:cols, :rows].T, ld)

    @property
    def view(self):
        return self.t

    def data_ptr(self):
        return self.t.data_ptr()


def _aligned_colmajor(t):
    m, n = t.shape
    if t.stride(0) != 1 and m > 1:
        return None
    ld = t.stride(1) if n > 1 else m + (m & 1)
    if ld < m or ld % 2 or t.data_ptr() % 16:
        return None
    return DevMat(t, ld)


def as_device_colmajor(a, device, name="a"):
    """Coerce an array-like / tensor to a DevMat on `device` (copying only if needed).
    Validation follows linalg.py:65-78 (2-D, positive dims); the finiteness
    check runs on the device inside the update (status bit NONFINITE)."""
    if isinstance(a, DevMat):
        return a
    if isinstance(a, torch.Tensor):
        t = a
        if t.dim() != 2:
            raise ValueError(f"{name} must be 2-D, got {t.dim()}-D")
        if min(t.shape) < 1:
            raise ValueError(f"{name} must have positive dimensions, got {tuple(t.shape)}")
        if t.device.type == "cuda" and t.dtype == torch.float64 and t.device == torch.device(device):
            dm = _aligned_colmajor(t)  # zero copy only for a tensor already on the context's device
            if dm is not None:
                return dm
        out = DevMat.empty(t.shape[0], t.shape[1], device)
        if t.dtype == torch.float64 and t.dim() == 2 and t.stride(1) == 1 and t.stride(0) >= t.shape[1]:
            # row-major fp64 (C order): bytes to the device as they are, transposed by the library
            src = t if t.device == torch.device(device) else t.to(device, non_blocking=t.is_pinned())
            _transpose_into(src, out, device)
        elif t.device.type == "cpu":
            # one H2D copy straight into the column-major buffer (async from pinned memory)
            out.view.copy_(t.to(torch.float64), non_blocking=t.is_pinned())
        else:
            out.view.copy_(t)
        return out
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got {arr.ndim}-D")
    if min(arr.shape) < 1:
        raise ValueError(f"{name} must have positive dimensions, got {arr.shape}")
    m, n = arr.shape
    out = DevMat.empty(m, n, device)
    if arr.flags.f_contiguous:
        out.view.T.copy_(torch.from_numpy(arr.T))
    else:
        # row-major host data (C order): one H2D copy of its bytes, transposed by the library's kernel
        host = torch.from_numpy(np.ascontiguousarray(arr))
        _transpose_into(host.to(device), out, device)
    return out


def _transpose_into(src, out, device):
    """out (DevMat, column-major) <- src (row-major fp64 CUDA tensor) by psvd_transpose."""
    with torch.cuda.device(device):
        call("psvd_transpose", context(device), _vp(src.data_ptr()), src.stride(0), src.shape[0], src.shape[1],
             _vp(out.data_ptr()), out.ld, stream_ptr(device))
    src.record_stream(torch.cuda.current_stream(device))


def to_host_colmajor(t, pinned=True):
    """D2H of a (column-major) CUDA matrix as ONE dense copy into (pinned) host memory;
    returns a column-major CPU view with the same shape."""
    if t.device.type != "cuda":
        return t
    m, n = t.shape
    if t.stride(0) == 1 and t.stride(1) >= m:
        src = t.T if t.stride(1) == m else t.T.contiguous()  # (n, m) row-major == column-major (m, n)
    else:
        src = t.T.contiguous()
    host = torch.empty((n, m), dtype=t.dtype, pin_memory=pinned)
    host.copy_(src)
    return host.T


# collective hooks of psvd_set_exchange (include/psvd.h)
ALLREDUCE_FN = ctypes.CFUNCTYPE(_c_int, _vp, _vp, _c_i64, _vp)
ALLGATHER_FN = ctypes.CFUNCTYPE(_c_int, _vp, _vp, _c_i64, _vp, _vp)


class _CudaBuffer:
    """Zero-copy view of a raw device pointer (for torch.as_tensor)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def wrap_device(ptr, count, device):
    """fp64 CUDA tensor aliasing `count` doubles at device pointer `ptr`."""
    return torch.as_tensor(_CudaBuffer(ptr, count), device=device)


_COPY_STREAMS = {}


def copy_stream(device):
    """Side stream for host->device batch uploads (one per device)."""
    key = torch.device(device).index
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=device)
    return _COPY_STREAMS[key]


def upload_async(a, device, name="a"):
    """(DevMat, ready event) for a pinned host fp64 matrix: the copy runs on the copy
    stream and the buffer is marked as used by the current stream.  Any other input
    goes through as_device_colmajor and returns (DevMat, None)."""
    if (isinstance(a, torch.Tensor) and a.device.type == "cpu" and a.dtype == torch.float64 and a.dim() == 2
            and min(a.shape) >= 1 and a.is_pinned()):
        cs = copy_stream(device)
        with torch.cuda.device(device), torch.cuda.stream(cs):
            out = DevMat.empty(a.shape[0], a.shape[1], device)
            out.view.copy_(a, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        out.t.record_stream(torch.cuda.current_stream(device))
        return out, ev
    return as_device_colmajor(a, device, name), None


def as_device_vector(v, device, n=None, name="v"):
    if isinstance(v, torch.Tensor):
        t = v.to(device=device, dtype=torch.float64).reshape(-1).contiguous()
    else:
        t = torch.as_tensor(np.asarray(v, dtype=np.float64).reshape(-1)).to(device)
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} has {t.numel()} entries, expected {n}")
    return t
