"""Python side of the C++ IR interpreter (oracle/ir_interp.cpp).

TEST INFRASTRUCTURE.  ``ir_execute(module, entry,
dyn_consts, args, max_steps)`` has the signature and value semantics of the
reference's ``oracle_execute`` (runtime/oracle.py:28-32): numpy arrays and
numpy scalars in, a fresh numpy array / scalar out, with the Appendix A
defects fixed and in-place writes where the written collection is dead.
Errors raise the reference's exception classes when skiff is loaded
(RuntimeError_, DynConstError, OracleLimitError), else built-ins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

from .ir_export import export_module

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libjunoir.so")
_lib = None

DTYPES = ["bool", "i8", "i16", "i32", "i64", "u8", "u16", "u32", "u64", "f32", "f64"]
_NP = [np.uint8, np.int8, np.int16, np.int32, np.int64, np.uint8, np.uint16, np.uint32, np.uint64,
       np.float32, np.float64]


class JirArg(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("ndim", ctypes.c_int), ("shape", ctypes.c_int64 * 8),
                ("data", ctypes.c_void_p)]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.jir_last_error.restype = ctypes.c_char_p
        L.jir_execute.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
                                  ctypes.POINTER(JirArg), ctypes.c_int, ctypes.c_longlong, ctypes.POINTER(JirArg),
                                  ctypes.POINTER(ctypes.c_longlong)]
        L.jir_execute.restype = ctypes.c_int
        _lib = L
    return _lib


def _dtype_code(fn_type, value) -> int:
    """The reference type of a parameter decides the code (bool arrays are
    u8 storage, types.py:147-159)."""
    kind = type(fn_type).__name__
    if kind == "ArrayType":
        fn_type = fn_type.element
        kind = type(fn_type).__name__
    if kind == "BoolType":
        return 0
    if kind == "IntType":
        return DTYPES.index(f"{'i' if fn_type.signed else 'u'}{fn_type.width}")
    if kind == "FloatType":
        return DTYPES.index(f"f{fn_type.width}")
    raise TypeError(f"unsupported parameter type {fn_type!r}")


def _raise(msg: str):
    cls, _, text = msg.partition(": ")
    targets = {"RuntimeError_": ("skiff.runtime.values", "RuntimeError_", RuntimeError),
               "DynConstError": ("skiff.dynconst", "DynConstError", ValueError),
               "OracleLimitError": ("skiff.runtime.oracle", "OracleLimitError", RuntimeError),
               "OverflowError": (None, None, OverflowError), "ValueError": (None, None, ValueError),
               "KeyError": (None, None, KeyError)}
    mod, name, default = targets.get(cls, (None, None, RuntimeError))
    exc = getattr(sys.modules.get(mod), name, None) if mod else None
    raise (exc or default)(text)


def ir_execute(module, entry: str, dyn_consts, args, max_steps: int = 50_000_000, return_steps: bool = False):
    js = export_module(module)
    fn = module.functions[entry]
    keep = []
    cargs = (JirArg * max(1, len(args)))()
    for i, (a, ty) in enumerate(zip(args, fn.param_types)):
        code = _dtype_code(ty, a)
        arr = np.asarray(a, dtype=_NP[code])
        if arr.ndim:  # (ascontiguousarray would turn a 0-d scalar into shape (1,))
            arr = np.ascontiguousarray(arr)
        keep.append(arr)
        cargs[i].dtype = code
        cargs[i].ndim = arr.ndim
        for k, s in enumerate(arr.shape):
            cargs[i].shape[k] = s
        cargs[i].data = arr.ctypes.data
    dcs = (ctypes.c_int64 * max(1, len(dyn_consts)))(*[int(x) for x in dyn_consts])
    out = JirArg()
    used = ctypes.c_longlong(0)
    rc = lib().jir_execute(js.encode(), entry.encode(), dcs, len(dyn_consts), cargs, len(args), int(max_steps),
                           ctypes.byref(out), ctypes.byref(used))
    if rc:
        _raise(lib().jir_last_error().decode())
    npdt = _NP[out.dtype]
    if out.ndim == 0:
        if out.dtype == 0:
            res = bool(ctypes.c_bool.from_address(out.data).value)
        else:
            res = np.frombuffer(ctypes.string_at(out.data, np.dtype(npdt).itemsize), dtype=npdt)[0]
    else:
        shape = tuple(out.shape[k] for k in range(out.ndim))
        n = int(np.prod(shape)) * np.dtype(npdt).itemsize
        res = np.frombuffer(ctypes.string_at(out.data, n), dtype=npdt).reshape(shape).copy()
    return (res, int(used.value)) if return_steps else res
