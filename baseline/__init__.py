"""Parallel CPU baseline for bench.py (baseline/cpu_multisplit.c): the paper's
{local, global, local} multisplit on all host cores.  Not the oracle, not the
product; built by __graft_entry__.build()."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cpu_multisplit.c")
LIB = os.path.join(_HERE, "libcpums.so")
_lib = None


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(_SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-shared", "-fPIC", "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB)
        p, u64, u32, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        _lib.cpu_multisplit.argtypes = [p, p, p, p, u64, u32, u32, u32, u32, u32, i]
        _lib.cpu_radix_sort.argtypes = [p, p, p, p, u64, u32, i]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def multisplit(keys: np.ndarray, vals, m: int, delta: int = 0, shift: int = 0, bits: int = 0,
               threads: int | None = None):
    threads = threads or len(os.sched_getaffinity(0))
    ko = np.empty_like(keys)
    vo = np.empty_like(vals) if vals is not None else None
    kind = 2 if bits else 1
    _load().cpu_multisplit(_p(keys), _p(vals), _p(ko), _p(vo), keys.size, m, kind, delta, shift, bits, threads)
    return ko, vo


def radix_sort(keys: np.ndarray, vals, r: int = 8, threads: int | None = None):
    threads = threads or len(os.sched_getaffinity(0))
    ko = np.empty_like(keys)
    vo = np.empty_like(vals) if vals is not None else None
    _load().cpu_radix_sort(_p(keys), _p(vals), _p(ko), _p(vo), keys.size, r, threads)
    return ko, vo
