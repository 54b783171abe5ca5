"""ctypes loader for liboracle.so — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It loads the plain C
oracle (oracle.c) and marshals numpy arrays; it imports nothing from the
product package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
          "-shared", "-std=c11", "-Wall", "-Wextra"]

_DT = {"f32": np.float32, "f64": np.float64, "i32": np.int32}


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.c")
    hdr = os.path.join(HERE, "oracle.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, src])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        dp = ctypes.POINTER(ctypes.c_double)
        vpp = ctypes.POINTER(ctypes.c_void_p)
        ip = ctypes.POINTER(ctypes.c_int)
        L.oracle_arity.argtypes = [ctypes.c_char_p] + [ip] * 7
        L.oracle_default_coeffs.argtypes = [ctypes.c_char_p, dp, ctypes.c_int]
        L.oracle_step.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, i64p, dp,
                                  ctypes.c_int, vpp, vpp, ctypes.c_int]
        L.oracle_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, i64p, dp,
                                 ctypes.c_int, vpp, ctypes.c_int, ctypes.c_int, ip]
        L.oracle_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def arity(kind: str) -> dict:
    v = [ctypes.c_int() for _ in range(7)]
    if lib().oracle_arity(kind.encode(), *[ctypes.byref(x) for x in v]):
        raise ValueError(lib().oracle_error().decode())
    keys = ["n_in", "n_out", "n_bufs", "lo", "hi", "ndims", "ncoeffs"]
    return {k: x.value for k, x in zip(keys, v)}


def default_coeffs(kind: str) -> np.ndarray:
    buf = (ctypes.c_double * 32)()
    n = lib().oracle_default_coeffs(kind.encode(), buf, 32)
    if n < 0:
        raise ValueError(lib().oracle_error().decode())
    return np.array(buf[:n], dtype=np.float64)


def _dims(a: np.ndarray):
    shape = a.shape[::-1]                      # numpy (nz, ny, nx) -> (nx, ny, nz)
    return len(shape), (ctypes.c_int64 * len(shape))(*shape)


def _coeffs(coeffs):
    if coeffs is None:
        return None, 0
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    return c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(c)


def _check(arrs, dtype):
    for a in arrs:
        assert a.dtype == _DT[dtype] and a.flags["C_CONTIGUOUS"], (a.dtype, dtype)


def step(kind: str, dtype: str, ins, outs, coeffs=None, nthreads: int = 1) -> None:
    """outs[...] <- kind(ins) at interior points (ins/outs are numpy arrays)."""
    _check(list(ins) + list(outs), dtype)
    nd, dims = _dims(ins[0])
    cp, nc = _coeffs(coeffs)
    pin = (ctypes.c_void_p * len(ins))(*[a.ctypes.data for a in ins])
    pout = (ctypes.c_void_p * len(outs))(*[a.ctypes.data for a in outs])
    if lib().oracle_step(kind.encode(), dtype.encode(), nd, dims, cp, nc, pin, pout, nthreads):
        raise ValueError(lib().oracle_error().decode())


def run(kind: str, dtype: str, bufs, n_iters: int, coeffs=None, nthreads: int = 1) -> int:
    """In-place run over ``bufs``; returns the index of the result buffer."""
    _check(bufs, dtype)
    nd, dims = _dims(bufs[0])
    cp, nc = _coeffs(coeffs)
    pb = (ctypes.c_void_p * len(bufs))(*[a.ctypes.data for a in bufs])
    r = ctypes.c_int(-1)
    if lib().oracle_run(kind.encode(), dtype.encode(), nd, dims, cp, nc, pb, n_iters,
                        nthreads, ctypes.byref(r)):
        raise ValueError(lib().oracle_error().decode())
    return r.value
