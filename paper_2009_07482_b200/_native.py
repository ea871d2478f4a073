"""ctypes binding of libhetsim.so (the C ABI in include/hetsim_c.h).

The product path has no fallback: if the shared library is missing or fails
to load, every entry point raises ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes
import json
import os
import pathlib
import threading

LIB_PATH = pathlib.Path(__file__).with_name("libhetsim.so")

_lock = threading.Lock()
_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


class HetsimError(RuntimeError):
    """Mirror of hetsim::Error: carries the Errc name and the process exit code."""

    def __init__(self, errc: str, message: str, exit_code: int | None = None):
        super().__init__(message)
        self.errc = errc
        self.exit_code = exit_code


c_int, c_int64, c_size_t, c_void_p, c_char_p = ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_char_p


class OpArgs(ctypes.Structure):
    _fields_ = [
        ("in_", c_void_p * 16),
        ("in_stride", c_int64 * 16),
        ("n_in", c_int),
        ("out", c_void_p),
        ("out_stride", c_int64),
        ("dims", c_int64 * 4),
        ("fparam", ctypes.c_float * 2),
        ("aux", c_void_p),
        ("n_out", c_int),
        ("outs", c_void_p * 4),
        ("out_strides", c_int64 * 4),
        ("out_ld", c_int64),
        ("epilogue", c_int),
        ("flags", c_int),
    ]


EPI_NONE, EPI_SOFTMAX = 0, 1
FLAG_DETERMINISTIC = 1


_PROTOS = {
    "hs_last_error": (c_char_p, []),
    "hs_last_errc": (c_int, []),
    "hs_version": (c_char_p, []),
    "hs_query": (c_void_p, [c_char_p]),
    "hs_free_string": (None, [c_void_p]),
    "hs_device_count": (c_int, [ctypes.POINTER(c_int)]),
    "hs_ctx_create": (c_int, [c_int, ctypes.POINTER(c_void_p)]),
    "hs_ctx_destroy": (c_int, [c_void_p]),
    "hs_ctx_sync": (c_int, [c_void_p]),
    "hs_stream_create": (c_int, [c_void_p, c_int, ctypes.POINTER(c_void_p)]),
    "hs_stream_destroy": (c_int, [c_void_p]),
    "hs_stream_sync": (c_int, [c_void_p]),
    "hs_event_create": (c_int, [c_void_p, c_int, ctypes.POINTER(c_void_p)]),
    "hs_event_destroy": (c_int, [c_void_p]),
    "hs_event_record": (c_int, [c_void_p, c_void_p]),
    "hs_stream_wait": (c_int, [c_void_p, c_void_p]),
    "hs_event_sync": (c_int, [c_void_p]),
    "hs_event_elapsed_ns": (c_int, [c_void_p, c_void_p, ctypes.POINTER(c_int64)]),
    "hs_malloc": (c_int, [c_void_p, c_size_t, ctypes.POINTER(c_void_p)]),
    "hs_free": (c_int, [c_void_p, c_void_p]),
    "hs_host_alloc": (c_int, [c_size_t, ctypes.POINTER(c_void_p)]),
    "hs_host_free": (c_int, [c_void_p]),
    "hs_host_pin": (c_int, [c_void_p, c_size_t]),
    "hs_host_unpin": (c_int, [c_void_p]),
    "hs_memcpy_h2d": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t]),
    "hs_memcpy_d2h": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t]),
    "hs_memcpy_d2d": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t]),
    "hs_memcpy_peer": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int, c_size_t]),
    "hs_ctx_enable_peer": (c_int, [c_void_p, c_void_p]),
    "hs_memset": (c_int, [c_void_p, c_void_p, c_int, c_size_t]),
    "hs_memcpy_2d": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t, c_size_t, c_size_t, c_int]),
    "hs_op_from_name": (c_int, [c_char_p]),
    "hs_launch": (c_int, [c_void_p, c_int, ctypes.POINTER(OpArgs), c_int, c_int]),
    "hs_host_callback": (c_int, [c_void_p, c_void_p, c_void_p]),
    "hs_capture_begin": (c_int, [c_void_p]),
    "hs_capture_end": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "hs_graph_launch": (c_int, [c_void_p, c_void_p]),
    "hs_graph_destroy": (c_int, [c_void_p]),
    "hs_launch_count": (c_int64, []),
    "hs_gemm_split_weights": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_void_p]),
    "hs_gemm_split_weights_strided": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64]),
    "hs_gemm_split_weights_ex": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_int]),
    "hs_engine_create": (c_int, [c_char_p, ctypes.POINTER(c_void_p)]),
    "hs_engine_destroy": (c_int, [c_void_p]),
    "hs_engine_bind": (c_int, [c_void_p, c_int, c_int, c_void_p, c_int64, c_int64, c_int]),
    "hs_engine_run": (c_int, [c_void_p, c_int64, c_int64, ctypes.POINTER(c_int64)]),
    "hs_engine_info": (c_int, [c_void_p, c_char_p, ctypes.POINTER(c_void_p)]),
}

EXPORTED_SYMBOLS = tuple(_PROTOS)


def lib():
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("HETSIM_LIB", str(LIB_PATH))
            if not pathlib.Path(path).exists():
                raise NativeLibraryMissing(
                    f"{path} is not built; run `make` (or __graft_entry__.build()) first. "
                    "hetsim-b200 has no pure-Python fallback.")
            try:
                handle = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
            except OSError as e:  # pragma: no cover
                raise NativeLibraryMissing(f"cannot load {path}: {e}") from e
            for name, (res, args) in _PROTOS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    l = lib()
    msg = (l.hs_last_error() or b"").decode()
    errc = msg.split(":", 1)[0] if ":" in msg else "DeviceError"
    raise HetsimError(errc, f"{what}: {msg}" if what else msg, exit_code=2 if status == 1 else 1)


def query(request: dict) -> dict:
    """hs_query: JSON request -> JSON response (raises HetsimError on failure)."""
    l = lib()
    ptr = l.hs_query(json.dumps(request).encode())
    try:
        text = ctypes.string_at(ptr).decode()
    finally:
        l.hs_free_string(ptr)
    out = json.loads(text)
    if not out.get("ok"):
        raise HetsimError(out.get("errc", "Unknown"), out.get("message", ""), out.get("exit"))
    return out
