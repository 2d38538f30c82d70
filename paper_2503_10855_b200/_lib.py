"""ctypes binding of libjunob200.so (include/junob200.h).

The library is the product: there is no Python or CPU fallback.  If the
shared object is missing the import of this module succeeds but every call
raises ``NativeLibraryError`` so that a GPU box without the extension fails
loudly instead of silently computing something else.
"""

from __future__ import annotations

import ctypes
import os
import re

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("JB_LIB") or os.path.join(_PKG, "libjunob200.so")
HEADER_PATH = os.path.join(os.path.dirname(_PKG), "include", "junob200.h")

JB_OK, JB_EINVAL, JB_ERUNTIME, JB_ECUDA, JB_ENOTSUP = 0, 1, 2, 3, 4


class NativeLibraryError(RuntimeError):
    """libjunob200.so is missing or failed to load."""


_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_f32 = ctypes.c_float
_vp = ctypes.c_void_p

# name -> argtypes (all pointers are passed as c_void_p device addresses)
SIGNATURES = {
    "jb_matmul_f32": [_u64, _u64, _u64, _vp, _vp, _vp, _vp],
    "jb_matmul_exact_f32": [_u64, _u64, _u64, _vp, _vp, _vp, _vp],
    "jb_edge_f32": [_u64, _u64, _u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _f32, _vp, _vp],
    "jb_matmul_sched_f32": [_u64, _u64, _u64, _vp, _vp, _vp, _u32, _u32, _u32, _vp],
    "jb_edge_bits_f32": [_u64, _u64, _u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _f32, _vp, _vp],
    "jb_bits_expand_f32": [_vp, _u64, _u64, _vp, ctypes.c_int],
    "jb_edge_stages_f32": [_u64, _u64, _u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _f32, _vp,
                           _vp, _vp, _vp, _vp, _vp, _vp],
    "jb_cava_u8": [_u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "jb_srad_f32": [_u64, _u64, _u64, _f32, _vp, _vp, _vp, _vp],
    "jb_srad_exact_f32": [_u64, _u64, _u64, _f32, _vp, _vp, _vp, _vp],
    "jb_srad_extract_f32": [_u64, _vp, _vp, _vp, ctypes.c_int, _vp],
    "jb_srad_slab_step_f32": [_u64, _u64, _u64, _u64, _vp, _vp, _vp, _f32, _vp, ctypes.c_int, ctypes.c_int, _vp],
    "jb_srad_q0_f32": [_vp, _u64, _vp, _vp],
    "jb_srad_slab_p2p_step_f32": [_u64, _u64, _u64, _u64, _vp, _vp, _vp, _f32, ctypes.c_int, ctypes.c_int, _vp,
                                  _vp],
    "jb_p2p_alloc": [_u64, ctypes.POINTER(_vp)],
    "jb_p2p_free": [_vp],
    "jb_ipc_handle": [_vp, _vp],
    "jb_ipc_open": [_vp, ctypes.POINTER(_vp)],
    "jb_ipc_close": [_vp],
    "jb_euler_f32": [_u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp],
    "jb_euler_exact_f32": [_u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp],
    "jb_euler_stage_f32": [_u64, _u64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int, _vp],
    "jb_euler_stage_p2p_f32": [_u64, _u64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_uint32,
                               ctypes.c_uint32, ctypes.c_int, _vp],
    "jb_euler_push_f32": [_vp, _u64, _vp, _vp, _vp, _u64, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _vp],
    "jb_euler_step_factor_f32": [_u64, _vp, _vp, _vp, _vp],
    "jb_euler_flux_f32": [_u64, _vp, _vp, _vp, _vp, _vp, _vp],
    "jb_bfs": [_u64, _u64, _vp, _vp, _vp, _u32, _vp, _vp],
    "jb_bp_train_f32": [_u64, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "jb_host_register": [_vp, _u64],
    "jb_bind_workspace": [_vp, _u64, _vp],
    "jb_workspace_stats": [_vp, _vp, _vp],
    "jb_host_unregister": [_vp],
    "jb_selftest_fastmath": [_u64, _u64, ctypes.c_int, ctypes.c_int, _vp, _vp],
}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER_PATH) as f:
        txt = f.read()
    return sorted(set(re.findall(r"JB_API\s+[\w\s\*]*?\b(jb_\w+)\s*\(", txt)))


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is not built; run `python -m paper_2503_10855_b200.build` "
            "(there is no CPU fallback)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - environment specific
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    lib.jb_last_error.restype = ctypes.c_char_p
    lib.jb_abi_version.restype = ctypes.c_int
    lib.jb_launch_count.restype = ctypes.c_uint64
    lib.jb_release_workspace.restype = ctypes.c_int
    lib.jb_prof_enable.argtypes = [ctypes.c_int]
    lib.jb_prof_enable.restype = None
    lib.jb_prof_reset.restype = None
    lib.jb_prof_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_uint64)]
    lib.jb_prof_read.restype = ctypes.c_int
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    _lib = lib
    return lib


def last_error() -> str:
    return load().jb_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(load().jb_launch_count())


def prof_enable(on: bool = True) -> None:
    load().jb_prof_enable(1 if on else 0)


def prof_reset() -> None:
    load().jb_prof_reset()


def prof_read(name: str) -> tuple[float, int]:
    """(summed device ms, launches) of kernel `name` since the last reset."""
    ms, cnt = ctypes.c_double(0.0), ctypes.c_uint64(0)
    st = load().jb_prof_read(name.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    if st != JB_OK:
        raise RuntimeError(last_error())
    return ms.value, int(cnt.value)


class SradP2P(ctypes.Structure):
    """include/junob200.h: jb_srad_p2p"""
    _fields_ = [("peer_north", _vp), ("peer_south", _vp), ("mbox", _vp), ("flag", _vp),
                ("peer_mbox", _vp * 8), ("peer_flag", _vp * 8), ("world", ctypes.c_int),
                ("rank", ctypes.c_int), ("iter", ctypes.c_int), ("flag_base", ctypes.c_uint32),
                ("npx_global", _u64), ("grid", ctypes.c_int)]
