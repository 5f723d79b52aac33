"""ctypes binding to libirk.so (the sm_100a kernel library) and the
status-code -> exception mapping of the drop-in API.

There is no CPU fallback: importing the compute path on a machine without the
built library or without a CUDA device raises immediately with the reason.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libirk.so"

IRK_OK, IRK_EINVAL, IRK_ECUDA, IRK_ENOCONV, IRK_ENONFINITE, IRK_ESINGULAR = range(6)

_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)

# name -> argtypes (restype is int unless listed in _RESTYPES)
_SIGS = {
    "irk_ctx_create": [_int, C.POINTER(_vp)],
    "irk_ctx_destroy": [_vp],
    "irk_ctx_set_stream": [_vp, _vp],
    "irk_ctx_synchronize": [_vp],
    "irk_ctx_launch_count": [_vp],
    "irk_last_error": [],
    "irk_version": [],
    "irk_mat_from_csr": [_vp, _i64, _i64, _i64, _vp, _vp, _vp, C.POINTER(_vp)],
    "irk_mat_assemble_p1": [_vp, _int, _i64, C.POINTER(_vp), C.POINTER(_vp)],
    "irk_mat_assemble_q1": [_vp, _i64, C.POINTER(_vp), C.POINTER(_vp)],
    "irk_mat_info": [_vp, _i64p, _i64p, _i64p],
    "irk_mat_same_pattern": [_vp, _vp],
    "irk_mat_download": [_vp, _vp, _vp, _vp, _vp],
    "irk_mat_destroy": [_vp],
    "irk_mat_union": [_vp, _vp, _vp, C.POINTER(_vp), C.POINTER(_vp)],
    "irk_mat_combine": [_vp, _dbl, _vp, _dbl, _vp, C.POINTER(_vp)],
    "irk_mat_constrain": [_vp, _vp, _vp, _dbl, C.POINTER(_vp)],
    "irk_mat_on_pattern": [_vp, _vp, _vp, C.POINTER(_vp)],
    "irk_mat_semilinear_jacobian": [_vp, _vp, _vp, _dbl, _vp, _i64, _i64, C.POINTER(_vp)],
    "irk_mat_diagonal": [_vp, _vp, _vp],
    "irk_mat_rowsum": [_vp, _vp, _vp],
    "irk_mat_absrowsum": [_vp, _vp, _vp],
    "irk_mat_to_dense": [_vp, _vp, _vp],
    "irk_spmv": [_vp, _vp, _int, _vp, _vp],
    "irk_stage_apply": [_vp, _int, _vp, _vp, _dbl, _vp, _vp, _int, _vp, _vp, _vp],
    "irk_stage_apply_semilinear": [_vp, _int, _vp, _vp, _dbl, _vp, _vp, _dbl, _vp, _vp, _vp, _vp],
    "irk_stage_mix": [_vp, _i64, _int, _int, _vp, _vp, _vp],
    "irk_stage_couple": [_vp, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp, _i64],
    "irk_stage_rhs": [_vp, _i64, _int, _dbl, _vp, _vp, _vp, _vp, _vp],
    "irk_stage_update": [_vp, _i64, _int, _dbl, _vp, _vp, _int, _vp, _vp],
    "irk_stage_scale": [_vp, _i64, _int, _vp, _vp, _vp, _vp],
    "irk_stage_get": [_vp, _i64, _int, _int, _vp, _vp],
    "irk_stage_set": [_vp, _i64, _int, _int, _vp, _vp],
    "irk_to_interleaved": [_vp, _i64, _int, _vp, _vp],
    "irk_to_stage_major": [_vp, _i64, _int, _vp, _vp],
    "irk_bc_scatter": [_vp, _int, _i64, _vp, _vp, _vp],
    "irk_bc_gather": [_vp, _i64, _vp, _vp, _vp],
    "irk_bc_zero": [_vp, _int, _i64, _vp, _vp],
    "irk_bc_mask": [_vp, _i64, _i64, _vp, _vp],
    "irk_multidot": [_vp, _i64, _int, _vp, _i64, _vp, _vp],
    "irk_orth_update": [_vp, _i64, _int, _vp, _i64, _vp, _vp, _int],
    "irk_lincomb": [_vp, _i64, _int, _vp, _i64, _vp, _vp],
    "irk_axpby": [_vp, _i64, _dbl, _vp, _dbl, _vp],
    "irk_scale_dev": [_vp, _i64, _vp, _vp, _vp, _vp],
    "irk_norm2": [_vp, _i64, _vp, _vp],
    "irk_dot": [_vp, _i64, _vp, _vp, _vp],
    "irk_all_finite": [_vp, _i64, _vp, _ip],
    "irk_pcg": [_vp, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _dbl, _dbl, _int,
                _vp, _vp],
    "irk_cocg": [_vp, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _dbl, _dbl,
                 _int, _vp, _vp],
    "irk_chebyshev": [_vp, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64,
                      _int],
    "irk_semilinear_residual": [_vp, _int, _vp, _dbl, _vp, _vp, _dbl, _int, _vp, _vp, _vp, _vp,
                                _vp, _vp, _vp],
    "irk_fe_load": [_vp, _int, _i64, _vp, _vp],
    "irk_fe_mms_forcing": [_vp, _int, _i64, _dbl, _vp],
    "irk_fe_error_sq": [_vp, _int, _i64, _vp, _vp, _vp, _vp],
    "irk_ctx_log_enable": [_vp, _int],
    "irk_ctx_log_take": [_vp, _vp, _int, _vp],
    "irk_ctx_log_size": [_vp, _vp],
    "irk_mg_create": [_vp, _int, _int, _vp, _vp, _vp, _int, _int, _vp],
    "irk_mg_destroy": [_vp],
    "irk_mg_vcycle": [_vp, _vp, _vp, _vp],
    "irk_mg_set_structured": [_vp, _int],
    "irk_dense_gemv": [_vp, _i64, _vp, _vp, _i64, _vp, _i64],
    "irk_mgc_create": [_vp, _int, _int, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _dbl, _int, _int,
                       _vp],
    "irk_mgc_destroy": [_vp],
    "irk_mgc_set_structured": [_vp, _int],
    "irk_mgc_info": [_vp, _vp, _vp],
    "irk_mgc_cocg": [_vp, _vp, _vp, _i64, _vp, _i64, _dbl, _dbl, _int, _vp, _vp],
    "irk_mg_info": [_vp, _vp, _vp],
    "irk_mg_set_dst": [_vp, _int],
    "irk_mg_dst_info": [_vp, _vp, _vp],
    "irk_mgc_set_dst": [_vp, _int],
    "irk_mgc_vcycle": [_vp, _vp, _vp, _vp],
    "irk_mgc_dst_info": [_vp, _vp, _vp],
    "irk_mg_pcg_multi": [_vp, _int, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _dbl, _dbl, _int, _vp,
                         _vp],
    "irk_mgc_cocg_multi": [_vp, _int, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _dbl, _dbl, _int,
                           _vp, _vp],
    "irk_mg_pcg": [_vp, _vp, _vp, _i64, _vp, _i64, _dbl, _dbl, _int, _vp, _vp],
    "irk_bc_dae_values": [_vp, _int, _i64, _vp, _vp, _vp, _dbl, _vp, _vp],
    "irk_fgmres_work_doubles": [_int],
    "irk_fgmres_graph_create": [_vp, _vp, _i64, _int, _int, _vp, _i64, _vp, _i64, _vp, _vp, _vp,
                                _vp, _vp, C.POINTER(_vp)],
    "irk_fgmres_graph_run": [_vp, _vp, _int, _vp, _dbl, _dbl, _dbl, _vp, _vp, _vp, _vp],
    "irk_fgmres_graph_destroy": [_vp],
}
_RESTYPES = {
    "irk_last_error": C.c_char_p,
    "irk_version": C.c_char_p,
    "irk_ctx_launch_count": C.c_int64,
    "irk_fgmres_work_doubles": C.c_size_t,
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


class LibraryUnavailable(RuntimeError):
    """libirk.so is missing or cannot be loaded (there is no CPU fallback)."""


def lib_path() -> Path:
    return _LIB_PATH


def load(build_if_missing: bool = True):
    """Load libirk.so (building it in-tree first if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists() and build_if_missing:
            from . import _build

            _build.build()
        if not _LIB_PATH.exists():
            raise LibraryUnavailable(f"{_LIB_PATH} not built; run __graft_entry__.build()")
        try:
            lib = C.CDLL(str(_LIB_PATH))
        except OSError as exc:  # pragma: no cover - depends on the host
            raise LibraryUnavailable(f"cannot load {_LIB_PATH}: {exc}") from exc
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().irk_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = ""):
    """Map an irk_status onto the reference's exception classes."""
    if status == IRK_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status in (IRK_EINVAL, IRK_ENONFINITE):
        raise ValueError(msg)
    if status == IRK_ESINGULAR:
        from .sparsela import FactorizationError

        raise FactorizationError(msg)
    if status == IRK_ENOCONV:
        from .sparsela import NonConvergenceError

        raise NonConvergenceError(msg, [])
    raise RuntimeError(msg)


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)


# ---------------------------------------------------------------- context


class _Context:
    """One irk_ctx per (thread, device); follows torch's current stream."""

    def __init__(self, device: int):
        self.device = device
        self.handle = _vp()
        check(load().irk_ctx_create(device, C.byref(self.handle)), "irk_ctx_create")
        self._stream = None

    def bind(self):
        s = _raw_stream(self.device)
        if s != self._stream:
            check(load().irk_ctx_set_stream(self.handle, _vp(s)), "irk_ctx_set_stream")
            self._stream = s
        return self.handle

    def launches(self) -> int:
        return int(load().irk_ctx_launch_count(self.handle))


_tls = threading.local()


_cuda_ok = False


def _raw_stream(dev: int) -> int:
    """torch's current stream on `dev` as an integer handle (the C++ fast
    path; the Python wrapper costs microseconds per call on small problems)."""
    import torch

    fast = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if fast is not None:
        return int(fast(dev))
    return torch.cuda.current_stream(dev).cuda_stream


def device_index() -> int:
    global _cuda_ok
    import torch

    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise LibraryUnavailable(
                "paper_2403_08084_b200 needs a CUDA device (sm_100a); there is no CPU fallback"
            )
        _cuda_ok = True
    return torch.cuda.current_device()


def context() -> _Context:
    dev = device_index()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    c = ctxs.get(dev)
    if c is None:
        c = ctxs[dev] = _Context(dev)
    return c


def ctx():
    """Handle of the calling thread's context bound to torch's current stream."""
    return context().bind()


def launch_count() -> int:
    return context().launches()


class deferred_solves:
    """Context manager: inner solves that pass no status buffers run without
    a host round trip; on exit the per-solve (iterations, code) log is read
    back in one copy into ``self.entries`` (numpy, shape (n, 4))."""

    def __init__(self):
        self.entries = np.zeros((0, 4), dtype=np.int32)

    def __enter__(self):
        call("irk_ctx_log_enable", ctx(), 1)
        return self

    def __exit__(self, *exc):
        n = C.c_int(0)
        try:
            size = C.c_int64(0)
            call("irk_ctx_log_size", ctx(), C.byref(size))
            buf = np.zeros((max(int(size.value), 1), 4), dtype=np.int32)
            call("irk_ctx_log_take", ctx(), hptr(buf), len(buf), C.byref(n))
        finally:
            call("irk_ctx_log_enable", ctx(), 0)
        self.entries = buf[: n.value].copy()
        return False


# ------------------------------------------------------------- marshalling


def ptr(t) -> _vp:
    """Device/host address of a torch tensor or numpy array (None -> NULL).
    The returned pointer object keeps its array alive for the call."""
    if t is None:
        return _vp()
    if isinstance(t, np.ndarray):
        p = _vp(t.ctypes.data)
    else:
        p = _vp(t.data_ptr())
    p._keep = t
    return p


def host_f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def hptr(a) -> _vp:
    """Pointer to a contiguous float64 host copy of ``a`` (kept alive)."""
    arr = a if (isinstance(a, np.ndarray) and a.flags.c_contiguous) else np.ascontiguousarray(a)
    p = _vp(arr.ctypes.data)
    p._keep = arr
    return p
