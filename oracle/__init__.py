"""CPU oracle for the stable multisplit of arXiv 1701.01189.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_1701_01189_b200``):
neither imports the other.  The arithmetic lives in ``multisplit_oracle.c``
(plain single-threaded C, compiled with gcc by :func:`build`); this module is
argument marshalling only.  Every function cites the PAPER.md passage it
follows in the C source header.

Parity pins (tests/test_oracle_pins.py) tie every function here to something
other than itself: Eq.(1) brute force, exhaustive small alphabets, the SPEC /
paper worked examples, numpy's stable argsort, and invariants.  No function is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "multisplit_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")

IDENTITY, DELTA, RADIX, SPLITTERS = 0, 1, 2, 3
MAX_M = 65536
OK, ERR_INVALID, ERR_UNSUPPORTED, ERR_KEY_DOMAIN = 0, 1, 2, 5


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile the oracle C file into ``oracle/liborc.so`` (gcc, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-shared", "-fPIC",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        u32, u64, p = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p
        lib.orc_validate.argtypes = [u32, u32, u64, u32, u32]
        lib.orc_bucket.argtypes = [u32, u32, u64, u32, u32, u32, ctypes.POINTER(u32)]
        lib.orc_multisplit.argtypes = [p, p, p, p, u64, u32, u32, u64, u32, u32, p]
        lib.orc_tile_histogram.argtypes = [p, u64, u64, u32, u32, u64, u32, u32, p]
        lib.orc_global_scan.argtypes = [p, u64, u32, p]
        lib.orc_global_scan.restype = None
        lib.orc_radix_sort.argtypes = [p, p, p, p, u64, u32, u32]
        f32 = ctypes.c_float
        lib.orc_histogram_even.argtypes = [p, u64, u32, f32, f32, p]
        lib.orc_histogram_range.argtypes = [p, u64, u32, p, p]
        lib.orc_validate_ex.argtypes = [u32, u32, u64, u32, u32, p]
        lib.orc_bucket_ex.argtypes = [u32, u32, u64, u32, u32, p, u32, ctypes.POINTER(u32)]
        lib.orc_multisplit_ex.argtypes = [p, p, p, p, u64, u32, u32, u64, u32, u32, p, p]
        lib.orc_sssp.argtypes = [p, p, p, u32, u32, p]
        for f in (lib.orc_validate_ex, lib.orc_bucket_ex, lib.orc_multisplit_ex, lib.orc_sssp):
            f.restype = ctypes.c_int
        for f in (lib.orc_validate, lib.orc_bucket, lib.orc_multisplit,
                  lib.orc_tile_histogram, lib.orc_radix_sort, lib.orc_histogram_even,
                  lib.orc_histogram_range):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


class Bucket:
    """Bucket identifier f(.): kind in {IDENTITY, DELTA, RADIX, SPLITTERS}."""

    def __init__(self, kind: int, m: int, delta: int = 0, shift: int = 0, bits: int = 0,
                 splitters=None):
        self.kind, self.m, self.delta, self.shift, self.bits = kind, m, delta, shift, bits
        self.splitters = None if splitters is None else _u32(splitters)

    def extended(self) -> bool:
        """Needs the extended entry points (splitters, or m beyond the paper's 256)."""
        return self.kind == SPLITTERS or self.m > 256

    def args(self):
        return (self.kind, self.m, self.delta, self.shift, self.bits)

    def __repr__(self):
        return f"Bucket(kind={self.kind}, m={self.m}, delta={self.delta}, shift={self.shift}, bits={self.bits})"


def identity(m: int) -> Bucket:
    return Bucket(IDENTITY, m)


def delta(m: int, d: int | None = None) -> Bucket:
    """Delta buckets f(u)=min(floor(u/D), m-1); default D = ceil(2^32/m) (reading R7)."""
    if d is None:
        d = min(-(-(1 << 32) // m), (1 << 32) - 1)
    return Bucket(DELTA, m, delta=d)


def radix(shift: int, bits: int) -> Bucket:
    return Bucket(RADIX, 1 << bits, shift=shift, bits=bits)


def splitters(spl) -> Bucket:
    """Splitter buckets (reading R27): m-1 interior splitters s_1 < ... < s_{m-1};
    f(u) = the j with s_j <= u < s_{j+1} (s_0 = 0, s_m = 2^32)."""
    spl = _u32(spl)
    return Bucket(SPLITTERS, spl.size + 1, splitters=spl)


def _u32(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != np.uint32:
        a = a.astype(np.uint32)
    return a


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def bucket_of(fn: Bucket, u: int) -> int:
    b = ctypes.c_uint32(0)
    if fn.extended():
        st = _load().orc_bucket_ex(*fn.args(), _ptr(fn.splitters), int(u) & 0xFFFFFFFF, ctypes.byref(b))
    else:
        st = _load().orc_bucket(*fn.args(), int(u) & 0xFFFFFFFF, ctypes.byref(b))
    if st:
        raise OracleError(st)
    return b.value


def validate(fn: Bucket) -> int:
    if fn.extended():
        return _load().orc_validate_ex(*fn.args(), _ptr(fn.splitters))
    return _load().orc_validate(*fn.args())


def multisplit(keys, fn: Bucket, values=None):
    """Stable multisplit (Eq.1).  Returns (keys_out, values_out|None, offsets[m+1]).
    Splitter buckets and m > 256 go through orc_multisplit_ex (same definition)."""
    keys = _u32(keys)
    n = keys.size
    vals = None if values is None else _u32(values)
    ko = np.empty(n, np.uint32)
    vo = None if vals is None else np.empty(n, np.uint32)
    off = np.empty(fn.m + 1 if 1 <= fn.m <= MAX_M else 1, np.uint32)
    if fn.extended():
        st = _load().orc_multisplit_ex(_ptr(keys), _ptr(vals), _ptr(ko), _ptr(vo), n, *fn.args(),
                                       _ptr(fn.splitters), _ptr(off))
    else:
        st = _load().orc_multisplit(_ptr(keys), _ptr(vals), _ptr(ko), _ptr(vo), n, *fn.args(), _ptr(off))
    if st:
        raise OracleError(st)
    return ko, vo, off


def tile_histogram(keys, fn: Bucket, T: int) -> np.ndarray:
    """H of Eq.(2) for subproblems of T elements; returns array [L, m] (tile-major)."""
    keys = _u32(keys)
    L = -(-keys.size // T)
    H = np.empty((L, fn.m), np.uint32)
    st = _load().orc_tile_histogram(_ptr(keys), keys.size, T, *fn.args(), _ptr(H))
    if st:
        raise OracleError(st)
    return H


def global_scan(H) -> np.ndarray:
    """Exclusive scan of row-vectorized H; H given as [L, m] tile-major."""
    H = _u32(H)
    L, m = H.shape
    G = np.empty_like(H)
    _load().orc_global_scan(_ptr(H), L, m, _ptr(G))
    return G


def radix_sort(keys, values=None, begin_bit: int = 0, end_bit: int = 32):
    """Stable sort by key bits [begin_bit, end_bit) (the result of Sec.7.1's multisplit-sort)."""
    keys = _u32(keys)
    n = keys.size
    vals = None if values is None else _u32(values)
    ko = np.empty(n, np.uint32)
    vo = None if vals is None else np.empty(n, np.uint32)
    st = _load().orc_radix_sort(_ptr(keys), _ptr(vals), _ptr(ko), _ptr(vo), n, begin_bit, end_bit)
    if st:
        raise OracleError(st)
    return ko, vo


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != np.float32:
        a = a.astype(np.float32)
    return a


def histogram_even(samples, m: int, lower: float, upper: float) -> np.ndarray:
    """Even histogram (Sec.7.3): counts[m] of floor((x - s_0) / Delta)."""
    x = _f32(samples)
    c = np.empty(max(m, 1), np.uint32)
    st = _load().orc_histogram_even(_ptr(x), x.size, m, float(np.float32(lower)),
                                    float(np.float32(upper)), _ptr(c))
    if st:
        raise OracleError(st)
    return c


def histogram_range(samples, splitters) -> np.ndarray:
    """Range histogram (Sec.7.3): counts[m] by upper-bound over m+1 splitters."""
    x = _f32(samples)
    s = _f32(splitters)
    m = s.size - 1
    c = np.empty(max(m, 1), np.uint32)
    st = _load().orc_histogram_range(_ptr(x), x.size, m, _ptr(s), _ptr(c))
    if st:
        raise OracleError(st)
    return c


def sssp(row_ptr, col, w, source: int) -> np.ndarray:
    """Shortest distances from `source` (Sec.7.2, Dijkstra); 0xFFFFFFFF = unreachable."""
    row_ptr, col, w = _u32(row_ptr), _u32(col), _u32(w)
    V = row_ptr.size - 1
    dist = np.empty(max(V, 1), np.uint32)
    st = _load().orc_sssp(_ptr(row_ptr), _ptr(col), _ptr(w), V, source, _ptr(dist))
    if st:
        raise OracleError(st)
    return dist[:V]
