"""ctypes binding of libstkb200.so (declarations: include/stkb200.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_2309_04671_b200.build``.  There is no fallback: if the
shared object is missing or a call fails, an exception is raised.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libstkb200.so"

STKB_OK = 0
STKB_ERR_ARG = 1
STKB_ERR_CUDA = 2
STKB_ERR_UNSUPPORTED = 3
STKB_ERR_STATE = 4
STKB_F32, STKB_F64 = 1, 2
STKB_MAP_STAR, STKB_MAP_WAVE, STKB_MAP_EXPR, STKB_MAP_BOX, STKB_MAP_XSTAR, STKB_MAP_XWAVE = 1, 2, 3, 4, 5, 6
STKB_MAP_XBOX = 7
STKB_PREC_FAST = 0
(OP_CONST, OP_READ, OP_LOCAL, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_NEG, OP_SETLOCAL, OP_STORE) = range(1, 11)
EXPR_MAX_ARGS, EXPR_MAX_LOCALS, EXPR_MAX_STACK = 8, 16, 32

# every entry point include/stkb200.h declares
EXPORTS = (
    "stkb_abi_version", "stkb_last_error", "stkb_device_count", "stkb_domain_create",
    "stkb_domain_destroy", "stkb_layout", "stkb_device_ptr", "stkb_mark_dirty", "stkb_zero", "stkb_set_stream", "stkb_upload",
    "stkb_download", "stkb_upload_async", "stkb_download_async", "stkb_upload_grid", "stkb_download_grid",
    "stkb_program_reset",
    "stkb_program_add_map", "stkb_program_add_swap", "stkb_run", "stkb_run_once", "stkb_sync",
    "stkb_elapsed_ms", "stkb_launches", "stkb_run_mode", "stkb_binding", "stkb_nonfinite", "stkb_run_target",
    "stkb_compare", "stkb_launch_map", "stkb_apply_swap", "stkb_plane_span", "stkb_launch_map_ranges",
    "stkb_stream_wait_signal", "stkb_reset_signal", "stkb_set_max_ctas", "stkb_launch_map_pull", "stkb_peer_fetch_halo", "stkb_buffer_ipc_handle",
    "stkb_flags_ipc_handle", "stkb_buffer_ptr", "stkb_flags_ptr", "stkb_ipc_open", "stkb_ipc_close", "stkb_set_peer",
    "stkb_peer_signal", "stkb_peer_wait", "stkb_set_fused_steps", "stkb_set_multi_steps", "stkb_enable_peer", "stkb_prepare",
)


class DomainDesc(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("shape", ctypes.c_int64 * 3),
        ("order", ctypes.c_int32),
        ("n_grids", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


class MapDesc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("radius", ctypes.c_int32),
        ("src", ctypes.c_int32),
        ("dst", ctypes.c_int32),
        ("prev", ctypes.c_int32),
        ("vel", ctypes.c_int32),
        ("precision", ctypes.c_int32),
        ("tag", ctypes.c_int32),
        ("coef", ctypes.c_double * 25),
        ("divisor", ctypes.c_double),
        ("wave_a", ctypes.c_double),
        ("wave_b", ctypes.c_double),
        ("lo", ctypes.c_int64 * 3),
        ("hi", ctypes.c_int64 * 3),
        ("n_args", ctypes.c_int32),
        ("args", ctypes.c_int32 * EXPR_MAX_ARGS),
        ("n_code", ctypes.c_int32),
        ("code", ctypes.POINTER(ctypes.c_int32)),
        ("n_consts", ctypes.c_int32),
        ("consts", ctypes.POINTER(ctypes.c_double)),
        ("box_coef", ctypes.c_double * 125),
        ("box_coef_ext", ctypes.POINTER(ctypes.c_double)),
    ]


class StkbError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code
        self.msg = msg


_lib = None


def load(path: os.PathLike | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("STKB_LIB", LIB_PATH))
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build the CUDA backend first (python -m paper_2309_04671_b200.build "
            "or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(str(p))
    P, V = ctypes.POINTER, ctypes.c_void_p
    i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "stkb_abi_version": [],
        "stkb_device_count": [P(i32)],
        "stkb_domain_create": [P(DomainDesc), P(V)],
        "stkb_domain_destroy": [V],
        "stkb_layout": [V, P(i64), P(i64), P(i64), P(i64)],
        "stkb_device_ptr": [V, i32, P(V)],
        "stkb_mark_dirty": [V, i32],
        "stkb_zero": [V, i32],
        "stkb_set_stream": [V, V],
        "stkb_upload": [V, i32, V],
        "stkb_download": [V, i32, V],
        "stkb_upload_async": [V, i32, V],
        "stkb_download_async": [V, i32, V],
        "stkb_upload_grid": [V, i32, V, P(i64), i32, i32],
        "stkb_download_grid": [V, i32, V, P(i64), i32, i32],
        "stkb_program_reset": [V],
        "stkb_program_add_map": [V, P(MapDesc)],
        "stkb_program_add_swap": [V, i32, i32],
        "stkb_run": [V, i64],
        "stkb_run_once": [V],
        "stkb_sync": [V],
        "stkb_elapsed_ms": [V, P(dbl)],
        "stkb_launches": [V, P(i64)],
        "stkb_run_mode": [V, P(i32)],
        "stkb_binding": [V, i32, P(i32)],
        "stkb_nonfinite": [V, i32, P(i32)],
        "stkb_run_target": [V, P(V), i64],
        "stkb_compare": [V, i32, i32, P(dbl), P(dbl), P(i64), P(dbl)],
        "stkb_launch_map": [V, i32, i64, i64],
        "stkb_apply_swap": [V, i32, i32],
        "stkb_plane_span": [V, i32, i64, i64, P(V), P(i64)],
        "stkb_launch_map_ranges": [V, i32, i32, P(i64), P(i64), i32, P(i32)],
        "stkb_stream_wait_signal": [V, V, i32, i32],
        "stkb_reset_signal": [V, i32, V],
        "stkb_set_max_ctas": [V, i32],
        "stkb_set_fused_steps": [V, i32],
        "stkb_set_multi_steps": [V, i32, i64],
        "stkb_enable_peer": [i32, i32],
        "stkb_prepare": [V],
        "stkb_launch_map_pull": [V, i32],
        "stkb_peer_fetch_halo": [V, V, i32],
        "stkb_buffer_ipc_handle": [V, i32, V],
        "stkb_flags_ipc_handle": [V, V],
        "stkb_buffer_ptr": [V, i32, P(V)],
        "stkb_flags_ptr": [V, P(V)],
        "stkb_ipc_open": [i32, V, P(V)],
        "stkb_ipc_close": [i32, V],
        "stkb_set_peer": [V, i32, i32, P(V), V, i64],
        "stkb_peer_signal": [V, V, i32],
        "stkb_peer_wait": [V, V, i32],
    }
    for name, args in sig.items():
        if os.environ.get("STKB_LIB_LENIENT") and not hasattr(lib, name):
            continue  # development A/B against an older build (tools/sweep.py)
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.stkb_last_error.argtypes = []
    lib.stkb_last_error.restype = ctypes.c_char_p
    if lib.stkb_abi_version() != 1:
        raise ImportError(f"{p}: unexpected ABI version {lib.stkb_abi_version()}")
    if path is None:
        _lib = lib
    return lib


def check(fn_name: str, rc: int) -> None:
    if rc != STKB_OK:
        msg = (_lib.stkb_last_error() or b"").decode(errors="replace") if _lib else ""
        raise StkbError(fn_name, rc, msg)


def call(name: str, *args) -> None:
    lib = load()
    check(name, getattr(lib, name)(*args))
