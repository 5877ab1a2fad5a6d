"""ctypes binding of gen/libepsgen.so (device twin of gen/synth.py)."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def load_device_gen():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libepsgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python __graft_entry__.py build`")
        lib = ctypes.CDLL(path)
        lib.epsgen_fill_bf16.restype = ctypes.c_int
        lib.epsgen_fill_bf16.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                                         ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                         ctypes.c_float, ctypes.c_void_p]
        _LIB = lib
    return _LIB


def device_fill_bf16(ptr: int, n: int, seed: int, tid: int, index_base: int, mode: int,
                     param: float, stream: int = 0) -> None:
    rc = load_device_gen().epsgen_fill_bf16(ptr, n, seed, tid, index_base, mode, param, stream)
    if rc != 0:
        raise RuntimeError(f"epsgen_fill_bf16 failed: cudaError {rc}")
