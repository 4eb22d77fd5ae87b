"""Naive CPU oracle for the L_d norms of arXiv 2503.21596 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2503_21596_b200``) never imports it and shares no code with it.

Thin ctypes wrapper over ``oracle/lnorm_oracle.c`` (plain counter enumeration,
from-scratch int64 values; see the C file header for the definitions and
PAPER.md citations).  The shared object is compiled with gcc on first use (or
by ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lnorm_oracle.c")
_LIB = os.path.join(_HERE, "liblnorm_oracle.so")
_lock = threading.Lock()
_lib = None

MODE_L1, MODE_MARG, MODE_LD = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle shared object (gcc -O2 -fopenmp); returns its path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared", _SRC, "-o", _LIB + ".tmp"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.POINTER
            i32p, i8p, i64p = P(ctypes.c_int32), P(ctypes.c_int8), P(ctypes.c_int64)
            ci, u64 = ctypes.c_int, ctypes.c_uint64
            lib.oracle_value_pm.argtypes = [i32p, ci, ci, i8p, ci]
            lib.oracle_value_pm.restype = ctypes.c_int64
            lib.oracle_value_ld.argtypes = [i32p, ci, ci, ci, i8p]
            lib.oracle_value_ld.restype = ctypes.c_int64
            lib.oracle_l1.argtypes = [i32p, ci, ci, ci, ci, i64p, i8p]
            lib.oracle_marg.argtypes = [i32p, ci, ci, ci, i64p, i8p]
            lib.oracle_ld.argtypes = [i32p, ci, ci, ci, ci, ci, i64p, i8p]
            lib.oracle_prefix_max.argtypes = [i32p, ci, ci, ci, ci, ci, i8p, ci, i64p, i8p]
            lib.oracle_sample.argtypes = [i32p, ci, ci, ci, ci, u64, u64, ci, i64p]
            lib.oracle_max_threads.argtypes = []
            for f in (lib.oracle_l1, lib.oracle_marg, lib.oracle_ld, lib.oracle_prefix_max,
                      lib.oracle_sample, lib.oracle_max_threads):
                f.restype = ctypes.c_int
            _lib = lib
    return _lib


def _mat(M):
    A = np.ascontiguousarray(np.asarray(M, dtype=np.int32))
    if A.ndim != 2 or A.shape[0] < 1 or A.shape[1] < 1:
        raise ValueError("M must be a non-empty 2-D integer matrix")
    return A


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def max_threads() -> int:
    return _load().oracle_max_threads()


def value(M, strategy, d: int = 1, marg: bool = False) -> int:
    """From-scratch value of one strategy: +-1 entries for d=1 (Eq. 1/2), labels for d>=2 (Eq. 6)."""
    A = _mat(M)
    s = np.ascontiguousarray(np.asarray(strategy, dtype=np.int8))
    if s.shape != (A.shape[0],):
        raise ValueError("strategy length must equal the row count")
    lib = _load()
    if d == 1:
        return int(lib.oracle_value_pm(_ptr(A, ctypes.c_int32), A.shape[0], A.shape[1], _ptr(s, ctypes.c_int8), int(marg)))
    return int(lib.oracle_value_ld(_ptr(A, ctypes.c_int32), A.shape[0], A.shape[1], d, _ptr(s, ctypes.c_int8)))


def _call(fn, *args):
    rc = fn(*args)
    if rc != 0:
        raise ValueError("oracle rejected the arguments (size or range)")


def l1(M, fix_first: bool = True, threads: int = 0):
    """L_1(M) (Eq. 1) and its lexicographically smallest maximiser (+-1, row 0 first)."""
    A = _mat(M)
    v = ctypes.c_int64()
    arg = np.zeros(A.shape[0], dtype=np.int8)
    _call(_load().oracle_l1, _ptr(A, ctypes.c_int32), A.shape[0], A.shape[1], int(fix_first), threads,
          ctypes.byref(v), _ptr(arg, ctypes.c_int8))
    return int(v.value), arg


def marg(M, threads: int = 0):
    """L_marg(M) (Eq. 2) and its lexicographically smallest maximiser (a_0 = +1)."""
    A = _mat(M)
    v = ctypes.c_int64()
    arg = np.zeros(A.shape[0], dtype=np.int8)
    _call(_load().oracle_marg, _ptr(A, ctypes.c_int32), A.shape[0], A.shape[1], threads,
          ctypes.byref(v), _ptr(arg, ctypes.c_int8))
    return int(v.value), arg


def ld(M, d: int, fix_first: bool = True, threads: int = 0):
    """L_d(M), d >= 2 (Eq. 6) and its lexicographically smallest maximising labelling."""
    A = _mat(M)
    v = ctypes.c_int64()
    arg = np.zeros(A.shape[0], dtype=np.int8)
    _call(_load().oracle_ld, _ptr(A, ctypes.c_int32), A.shape[0], A.shape[1], d, int(fix_first), threads,
          ctypes.byref(v), _ptr(arg, ctypes.c_int8))
    return int(v.value), arg


def norm(M, d: int = 1, with_marginals: bool = False, threads: int = 0):
    """Dispatch with the library's (d, with_marginals) convention: d=1 -> L_1, d=1+marg -> L_marg."""
    if with_marginals:
        if d != 1:
            raise ValueError("with_marginals requires d == 1")
        return marg(M, threads)
    if d == 1:
        return l1(M, True, threads)
    return ld(M, d, True, threads)


def prefix_max(M, fixed_digits, d: int = 1, with_marginals: bool = False, threads: int = 0):
    """Best value over strategies whose first len(fixed_digits) rows are fixed.

    Digits: 0/1 meaning +1/-1 for d=1 (L_1/L_marg), labels for d>=2.
    Returns (value, full digit vector of the first strict maximum)."""
    A = _mat(M)
    fx = np.ascontiguousarray(np.asarray(fixed_digits, dtype=np.int8))
    mode = MODE_MARG if with_marginals else (MODE_L1 if d == 1 else MODE_LD)
    v = ctypes.c_int64()
    arg = np.zeros(A.shape[0], dtype=np.int8)
    _call(_load().oracle_prefix_max, _ptr(A, ctypes.c_int32), A.shape[0], A.shape[1], mode, max(d, 2),
          len(fx), _ptr(fx, ctypes.c_int8), threads, ctypes.byref(v), _ptr(arg, ctypes.c_int8))
    return int(v.value), arg


def sample(M, c_begin: int, c_end: int, d: int = 1, with_marginals: bool = False, threads: int = 0) -> int:
    """Max over counter values [c_begin, c_end) of the row-0-fixed space (bounded CPU timing sample)."""
    A = _mat(M)
    mode = MODE_MARG if with_marginals else (MODE_L1 if d == 1 else MODE_LD)
    v = ctypes.c_int64()
    _call(_load().oracle_sample, _ptr(A, ctypes.c_int32), A.shape[0], A.shape[1], mode, max(d, 2),
          c_begin, c_end, threads, ctypes.byref(v))
    return int(v.value)
