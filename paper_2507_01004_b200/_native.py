"""ctypes binding of the C ABI in include/zeco_gla.h (libzeco_gla.so, built in-tree).

This is the only place the package touches native code.  There is no CPU
fallback: if the library is missing the import of any compute entry point
raises immediately.
"""

from __future__ import annotations

import atexit
import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libzeco_gla.so")

ZGLA_BF16, ZGLA_F32, ZGLA_F64 = 0, 1, 2
ZGLA_FWD, ZGLA_BWD = 0, 1
ZGLA_FWD_NO_SAVE = 1  # zgla_zeco_fwd_output_ex_v flag: skip the chunk-start states the backward reads
ZGLA_HOST_OVERLAP = 1

_CODES = {
    -1: errors.DimsError,
    -2: errors.DomainError,
    -3: errors.LayoutError,
    -4: errors.ConfigError,
    -5: errors.StateError,
    -6: errors.DeadlockError,
    -7: errors.UnsupportedError,
}


class Shape(ctypes.Structure):
    _fields_ = [
        ("heads", ctypes.c_int),
        ("key_dim", ctypes.c_int),
        ("value_dim", ctypes.c_int),
        ("chunk_len", ctypes.c_int),
        ("seq_len", ctypes.c_longlong),
        ("dtype", ctypes.c_int),
    ]


class Tensor(ctypes.Structure):
    """zgla_tensor: [heads][tokens][channels] view with element strides (0 = dense)."""
    _fields_ = [("data", ctypes.c_void_p), ("token_stride", ctypes.c_longlong), ("head_stride", ctypes.c_longlong)]


_P = ctypes.c_void_p
_T = ctypes.POINTER(Tensor)
_I = ctypes.c_int
_LL = ctypes.c_longlong
_SIGS = {
    "zgla_version": ([], ctypes.c_char_p),
    "zgla_last_error": ([], ctypes.c_char_p),
    "zgla_fast_path": ([ctypes.POINTER(Shape)], _I),
    "zgla_workspace_bytes": ([ctypes.POINTER(Shape)], _LL),
    "zgla_local_state_scan": ([ctypes.POINTER(Shape), _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "zgla_forward_outputs": ([ctypes.POINTER(Shape), _P, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "zgla_global_correct": ([ctypes.POINTER(Shape), _I, _P, _P, _P, _P, _P], _I),
    "zgla_reverse_boundary_scan": ([ctypes.POINTER(Shape), _P, _P, _P, _P, _P, _P, _P], _I),
    "zgla_backward": ([ctypes.POINTER(Shape)] + [_P] * 15, _I),
    "zgla_revcum": ([ctypes.POINTER(Shape), _I, _P, _P, _P], _I),
    "zgla_chunk_scalings": ([ctypes.POINTER(Shape), _P, _P, _P, _P, _P], _I),
    "zgla_check_log_decay": ([_LL, _I, _P, _P, _P], _I),
    "zgla_recurrent_forward": ([ctypes.POINTER(Shape)] + [_P] * 9, _I),
    "zgla_fd_max_state": ([], _LL),
    "zgla_fd_losses": ([ctypes.POINTER(Shape), _P, _P, _P, _P, _P, _I, _LL, _LL, ctypes.c_double, _P, _P], _I),
    "zgla_zeco_workspace_bytes": ([ctypes.POINTER(Shape), _I], _LL),
    "zgla_set_early_inputs": ([_I], _I),
    "zgla_zeco_fwd_local": ([ctypes.POINTER(Shape), _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "zgla_zeco_fwd_output": ([ctypes.POINTER(Shape), _I, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "zgla_zeco_bwd_local": ([ctypes.POINTER(Shape), _I, _P, _P, _P, _P, _P, _P], _I),
    "zgla_zeco_bwd_output": ([ctypes.POINTER(Shape), _I] + [_P] * 13, _I),
    "zgla_zeco_domain_check": ([ctypes.POINTER(Shape), _I, _P, _P], _I),
    "zgla_zeco_watch_domain": ([_P, ctypes.POINTER(ctypes.POINTER(ctypes.c_int))], _I),
    "zgla_zeco_unwatch_domain": ([_P], _I),
    "zgla_zeco_fwd_local_v": ([ctypes.POINTER(Shape), _I, _T, _T, _T, _P, _P, _P, _P], _I),
    "zgla_zeco_fwd_output_v": ([ctypes.POINTER(Shape), _I, _T, _T, _T, _T, _P, _P, _T, _P], _I),
    "zgla_zeco_fwd_output_ex_v": ([ctypes.POINTER(Shape), _I, _T, _T, _T, _T, _P, _P, _T, _I, _P], _I),
    "zgla_zeco_bwd_local_v": ([ctypes.POINTER(Shape), _I, _T, _T, _T, _P, _P, _P], _I),
    "zgla_zeco_bwd_output_v": ([ctypes.POINTER(Shape), _I, _T, _T, _T, _T, _T, _P, _P, _P, _T, _T, _T, _T, _P], _I),
    "zgla_allscan_local": ([_I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P], _I),
    "zgla_release_cached": ([], _I),
    "zgla_allscan_create": ([_I, _I, _I, _I, _I, _I, ctypes.POINTER(_P)], _I),
    "zgla_allscan_export": ([_P, _P], _I),
    "zgla_allscan_bind": ([_P, _P, _P], _I),
    "zgla_allscan_bind_local": ([_P, _P, _P], _I),
    "zgla_allscan_run": ([_P, _I, _I, _P, _P, _P, _P, _P], _I),
    "zgla_allscan_destroy": ([_P], _I),
    "zgla_allscan_status": ([_P, _I], _I),
    "zgla_allscan_bytes_sent": ([_P], _LL),
    "zgla_allscan_info": ([_P, _P, _P, _P], _I),
    "zgla_zeco_fwd_bwd_host_bytes": ([ctypes.POINTER(Shape), _I, _I], _LL),
    "zgla_zeco_fwd_bwd_host": ([ctypes.POINTER(Shape), _I, _I, _P, _I] + [_P] * 11 + [_LL, _I, _P], _I),
    "zgla_zeco_host_wait": ([_P], _I),
    "zgla_set_trace": ([_P, _I], _I),
    "zgla_selftest_tmem": ([_I, _I, _I, _P, _P, _P], _I),
    "zgla_selftest_stream": ([_P, _LL, _I, _I, _I, _I, _I, _P], _I),
    "zgla_selftest_mma": ([_P, _P, _P, _I, _I, _I, _I, _I, _I, _P], _I),
    "zgla_selftest_spin": ([_LL, _P], _I),
    "zgla_selftest_mma_rate": ([_I, _I, _I, _I, _I, _I, _P, _P], _I),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load (once) and return the native library; raises if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            # ZGLA_LIB: alternative build of the same library (compile-variant A/B experiments)
            p = path or os.environ.get("ZGLA_LIB") or LIB_PATH
            if not os.path.exists(p):
                raise errors.NativeLibraryError(
                    f"{p} is missing: build it with `make` or `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ctypes.CDLL(p)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
            atexit.register(_release_at_exit)
    return _lib


def _release_at_exit():
    """Free the library's cached device scratch while the CUDA context is still alive."""
    try:
        if _lib is not None:
            _lib.zgla_release_cached()
    except Exception:  # interpreter teardown: nothing useful to report
        pass


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    lib = load()
    detail = lib.zgla_last_error().decode(errors="replace")
    exc = _CODES.get(rc, errors.NativeLibraryError)
    raise exc(f"{what} failed (code {rc}){': ' + detail if detail else ''}")


def call(name: str, *args):
    fn = getattr(load(), name)
    rc = fn(*args)
    check(rc, name)
    return rc
