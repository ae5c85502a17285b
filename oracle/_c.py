"""ctypes loader for oracle/csrc/oracle.c (test infrastructure only; see oracle/__init__.py)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "csrc" / "oracle.c"
_LIB = _HERE / "liboracle.so"

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> Path:
    """Compile the oracle with plain gcc (-O2, OpenMP over independent outputs)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", str(tmp), str(_SRC)])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(build()))
        c_u64, c_u32, c_sz, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_void_p
        L.orc_powmod.restype = c_u64
        L.orc_powmod.argtypes = [c_u64, c_u64, c_u64]
        L.orc_negacyclic_mul.argtypes = [_u64p, _u64p, _u64p, c_u32, c_u64]
        L.orc_ntt_direct.argtypes = [_u64p, _u64p, c_u32, c_u64, c_u64]
        L.orc_ntt_direct_sampled.argtypes = [_u64p, _u32p, _u64p, c_sz, c_u32, c_u64, c_u64]
        L.orc_intt_direct.argtypes = [_u64p, _u64p, c_u32, c_u64, c_u64]
        L.orc_enc.argtypes = [_u64p, _u64p, c_sz, c_u64, c_u64, c_u64, c_u32]
        L.orc_he_conv_server.argtypes = [c_u32, c_u32, _u64p, c_u32, _u64p, c_u64, c_u32, c_u32, c_u32,
                                         _u64p, vp, _u64p, _u32p, _u64p, vp, vp, _u64p]
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def ptr_or_null(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)
