"""Device-side generator (gen/csrc/gen.cu -> gen/libmsgen.so): the same recipe
as gen/inputs.py, run on the GPU so that 2^28-element bench inputs are made in
HBM directly.  Holds no multisplit arithmetic."""
from __future__ import annotations

import ctypes
import os
import subprocess

from .inputs import DIST_UNIFORM, alpha32

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "gen.cu")
LIB = os.path.join(_HERE, "libmsgen.so")
_lib = None


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(_SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared",
                               "-o", tmp, _SRC])
        os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB)
        u32, u64, p = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p
        lib.msgen_keys.argtypes = [p, u64, u64, u32, u32, u32, u32, u32, u32, u64, p]
        lib.msgen_values.argtypes = [p, u64, u64, ctypes.c_int, p]
        lib.msgen_flush.argtypes = [p, u64, u32, p]
        _lib = lib
    return _lib


def _stream(stream):
    import torch
    return (stream if stream is not None else torch.cuda.current_stream()).cuda_stream


def keys_(out, seed: int, kind: int = 1, m: int = 2, delta: int = 0, shift: int = 0, bits: int = 0,
          dist: int = DIST_UNIFORM, alpha: float = 0.1, stream=None):
    """Fill the CUDA tensor `out` (int32/uint32) like gen.inputs.keys(out.numel(), ...)."""
    r = _load().msgen_keys(out.data_ptr(), out.numel(), seed, kind, m, delta, shift, bits, dist,
                           alpha32(alpha), _stream(stream))
    if r:
        raise RuntimeError(f"msgen_keys: cuda error {r}")
    return out


def values_(out, seed: int, parity: bool = True, stream=None):
    r = _load().msgen_values(out.data_ptr(), out.numel(), seed, int(parity), _stream(stream))
    if r:
        raise RuntimeError(f"msgen_values: cuda error {r}")
    return out


def flush_(scratch, value: int = 0, stream=None):
    """Overwrite a scratch CUDA tensor (bigger than L2) to evict the L2 between timed steps."""
    r = _load().msgen_flush(scratch.data_ptr(), scratch.numel() * scratch.element_size(), value,
                            _stream(stream))
    if r:
        raise RuntimeError(f"msgen_flush: cuda error {r}")
