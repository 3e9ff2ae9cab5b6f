"""paper_1701_01189_b200 -- stable multisplit and multisplit radix sort on B200.

A thin Python binding over libms.so (include/multisplit.h).  PyTorch is used
for device memory and streams only; every step of the path runs in the CUDA
kernels of ``csrc/``.  Tensors are ``torch.int32`` or ``torch.uint32`` on a
CUDA device and are read as uint32 bit patterns.

    >>> import paper_1701_01189_b200 as ms
    >>> k_out, v_out, offsets = ms.multisplit(keys, values, bucket=ms.Delta(32))
    >>> k_sorted, v_sorted = ms.radix_sort(keys, values)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import MultisplitError, check, ms_bucket_fn

__all__ = ["Bucket", "Delta", "Identity", "Radix", "Splitters", "multisplit", "radix_sort", "device_status",
           "prescan", "scan", "tile_size", "radix_pass_schedule", "workspace_size",
           "set_option", "get_option", "device_init", "sssp", "MultisplitError"]


@dataclass(frozen=True)
class Bucket:
    """A bucket identifier f(.): kind, m and its parameters."""
    kind: int
    m: int
    delta: int = 0
    shift: int = 0
    bits: int = 0
    splitters: torch.Tensor | None = None  # SPLITTERS: m-1 device words

    def c(self) -> ms_bucket_fn:
        """The C struct (built once per Bucket: the binding is on the latency path of small calls)."""
        fn = self.__dict__.get("_c")
        if fn is None:
            sp = self.splitters.data_ptr() if self.splitters is not None and self.splitters.numel() else None
            fn = ms_bucket_fn(self.kind, self.m, self.delta, self.shift, self.bits, sp)
            self.__dict__["_c"] = fn
        return fn


def Delta(m: int, delta: int | None = None) -> Bucket:
    """Delta buckets f(u) = min(floor(u/delta), m-1); default width ceil(2^32/m)."""
    if delta is None:
        fn = ms_bucket_fn()
        check(_lib.load().ms_bucket_delta_default(m, ctypes.byref(fn)), "ms_bucket_delta_default")
        delta = fn.delta
    return Bucket(_lib.MS_BUCKET_DELTA, m, delta=delta)


def Identity(m: int) -> Bucket:
    """Identity buckets f(u) = u, keys must lie in [0, m)."""
    return Bucket(_lib.MS_BUCKET_IDENTITY, m)


def Radix(shift: int, bits: int) -> Bucket:
    """Radix-digit buckets f(u) = (u >> shift) & (2^bits - 1)."""
    return Bucket(_lib.MS_BUCKET_RADIX, 1 << bits, shift=shift, bits=bits)


def Splitters(splitters: torch.Tensor) -> Bucket:
    """Splitter buckets: the m-1 interior splitters s_1 < ... < s_{m-1} as a CUDA
    int32/uint32 tensor (bit patterns read as uint32); f(u) = j with s_j <= u < s_{j+1},
    s_0 = 0 and s_m = 2^32 (reading R27).  The tensor must outlive the calls."""
    sp = _u32view(splitters, "splitters")
    return Bucket(_lib.MS_BUCKET_SPLITTERS, sp.numel() + 1, splitters=sp)


def _u32view(t: torch.Tensor, name: str, device: torch.device | None = None,
             numel: int | None = None) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype not in (torch.int32, torch.uint32):
        raise TypeError(f"{name} must be int32 or uint32, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs {numel}")
    return t


def _workspace(ws, need: int, device: torch.device) -> torch.Tensor:
    if ws is None or ws.numel() < need:
        return torch.empty(max(need, 1), dtype=torch.uint8, device=device)
    if not ws.is_cuda or ws.device != device or not ws.is_contiguous() or ws.data_ptr() % 256:
        raise ValueError("workspace must be a contiguous, 256-byte aligned tensor on the keys' device")
    return ws


_initialised: set[int] = set()


def device_init(device: torch.device | int | None = None) -> None:
    """ms_device_init: the one-time per-device probe (synchronous; outside graph capture)."""
    if device is None:
        idx = torch.cuda.current_device()
    elif isinstance(device, int):
        idx = device
    else:
        idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _initialised:
        check(_lib.load().ms_device_init(idx), "ms_device_init")
        _initialised.add(idx)


def _prepare(t: torch.Tensor) -> None:
    """Per-call device guard: the library launches on the current device."""
    if t.device.index is not None and t.device.index not in _initialised:
        device_init(t.device.index)


def _stream_ptr(stream, device: torch.device | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def set_option(option: int, value: int) -> None:
    """ms_set_option (process-wide): MS_OPT_RANK / MS_OPT_RUN_STORES / MS_OPT_PIPELINE / MS_OPT_SORT."""
    check(_lib.load().ms_set_option(option, value), "ms_set_option")


def get_option(option: int) -> int:
    return int(_lib.load().ms_get_option(option))


def workspace_size(n: int, m: int, with_values: bool) -> int:
    return int(_lib.load().ms_multisplit_workspace_size(n, m, int(with_values)))


def multisplit(keys: torch.Tensor, values: torch.Tensor | None = None, bucket: Bucket | None = None,
               *, out_keys: torch.Tensor | None = None, out_values: torch.Tensor | None = None,
               offsets: bool = True, out_offsets: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None, stream=None):
    """Stable multisplit (Eq.1).  Returns (keys_out, values_out|None, offsets|None)
    where offsets has m+1 entries (bucket starts, offsets[m] = n)."""
    if bucket is None:
        raise ValueError("bucket is required (Delta / Identity / Radix)")
    lib = _lib.load()
    keys = _u32view(keys, "keys")
    dv = keys.device
    n = keys.numel()
    pairs = values is not None
    if pairs:
        values = _u32view(values, "values", dv)
        if values.numel() != n:
            raise ValueError("keys and values differ in length")
    ko = _u32view(out_keys, "out_keys", dv, n) if out_keys is not None else torch.empty_like(keys)
    vo = None
    if pairs:
        vo = _u32view(out_values, "out_values", dv, n) if out_values is not None else torch.empty_like(values)
    off = out_offsets
    if off is None and offsets:
        off = torch.empty(bucket.m + 1, dtype=torch.int32, device=dv)
    elif off is not None:
        off = _u32view(off, "out_offsets", dv, bucket.m + 1)
    need = lib.ms_multisplit_workspace_size(n, bucket.m, int(pairs))
    ws = _workspace(workspace, need, dv)
    fn = bucket.c()
    _prepare(keys)
    if dv.index == torch.cuda.current_device():
        _call_multisplit(lib, pairs, keys, values, ko, vo, n, fn, off, ws, _stream_ptr(stream, dv))
    else:
        with torch.cuda.device(dv):
            _call_multisplit(lib, pairs, keys, values, ko, vo, n, fn, off, ws, _stream_ptr(stream, dv))
    multisplit.last_workspace = ws
    return ko, vo, off


def _call_multisplit(lib, pairs, keys, values, ko, vo, n, fn, off, ws, sp):
    if pairs:
        st = lib.ms_multisplit_pairs(keys.data_ptr(), values.data_ptr(), ko.data_ptr(), vo.data_ptr(),
                                     n, ctypes.byref(fn), off.data_ptr() if off is not None else None,
                                     ws.data_ptr(), ws.numel(), sp)
    else:
        st = lib.ms_multisplit_keys(keys.data_ptr(), ko.data_ptr(), n, ctypes.byref(fn),
                                    off.data_ptr() if off is not None else None,
                                    ws.data_ptr(), ws.numel(), sp)
    check(st, "ms_multisplit_pairs" if pairs else "ms_multisplit_keys")


def device_status(workspace: torch.Tensor | None = None, stream=None) -> int:
    """Sync and return the device-detected status of the last multisplit on `workspace`."""
    ws = workspace if workspace is not None else getattr(multisplit, "last_workspace", None)
    if ws is None:
        raise ValueError("no workspace")
    return int(_lib.load().ms_device_status(ws.data_ptr(), _stream_ptr(stream)))


def radix_sort(keys: torch.Tensor, values: torch.Tensor | None = None, *, begin_bit: int = 0,
               end_bit: int = 32, bits_per_pass: int = 0, out_keys: torch.Tensor | None = None,
               out_values: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
               stream=None):
    """LSD multisplit radix sort (Sec.7.1): stable sort by key bits [begin_bit, end_bit).
    bits_per_pass = 0: the library's choice (8-bit digits, see include/multisplit.h)."""
    lib = _lib.load()
    keys = _u32view(keys, "keys")
    dv = keys.device
    n = keys.numel()
    pairs = values is not None
    if pairs:
        values = _u32view(values, "values", dv)
        if values.numel() != n:
            raise ValueError("keys and values differ in length")
    ko = _u32view(out_keys, "out_keys", dv, n) if out_keys is not None else torch.empty_like(keys)
    vo = None
    if pairs:
        vo = _u32view(out_values, "out_values", dv, n) if out_values is not None else torch.empty_like(values)
    need = lib.ms_radix_sort_workspace_size(n, int(pairs))
    ws = _workspace(workspace, need, dv)
    _prepare(keys)
    with torch.cuda.device(dv):
        sp = _stream_ptr(stream, dv)
        if pairs:
            st = lib.ms_radix_sort_pairs(keys.data_ptr(), values.data_ptr(), ko.data_ptr(), vo.data_ptr(), n,
                                         begin_bit, end_bit, bits_per_pass, ws.data_ptr(), ws.numel(), sp)
        else:
            st = lib.ms_radix_sort_keys(keys.data_ptr(), ko.data_ptr(), n, begin_bit, end_bit, bits_per_pass,
                                        ws.data_ptr(), ws.numel(), sp)
    check(st, "ms_radix_sort_pairs" if pairs else "ms_radix_sort_keys")
    return ko, vo


def radix_sort_workspace_size(n: int, with_values: bool) -> int:
    return int(_lib.load().ms_radix_sort_workspace_size(n, int(with_values)))


def radix_pass_schedule(begin_bit: int = 0, end_bit: int = 32, bits_per_pass: int = 8):
    """Host-only: [(shift, bits), ...] of the LSD passes."""
    cap = 32
    sh = (ctypes.c_uint32 * cap)()
    bi = (ctypes.c_uint32 * cap)()
    p = _lib.load().ms_radix_pass_schedule(begin_bit, end_bit, bits_per_pass, sh, bi, cap)
    if p < 0:
        raise ValueError("invalid radix pass parameters")
    return [(sh[i], bi[i]) for i in range(p)]


def tile_size(m: int = 256, with_values: bool = False) -> int:
    return int(_lib.load().ms_multisplit_tile_size(m, int(with_values)))


def prescan(keys: torch.Tensor, bucket: Bucket, tile: int | None = None, stream=None) -> torch.Tensor:
    """Stage 1: H as an [L, m] int32 tensor (tile-major), L = ceil(n / tile)."""
    lib = _lib.load()
    keys = _u32view(keys, "keys")
    T = tile or tile_size(bucket.m)
    L = -(-keys.numel() // T)
    H = torch.empty((L, bucket.m), dtype=torch.int32, device=keys.device)
    fn = bucket.c()
    check(lib.ms_stage_prescan(keys.data_ptr(), keys.numel(), ctypes.byref(fn), H.data_ptr(), T,
                               _stream_ptr(stream)), "ms_stage_prescan")
    return H


def scan(H: torch.Tensor, stream=None):
    """Stage 2: G = exclusive scan of row-vectorized H ([L, m] tile-major), and
    the m+1 bucket offsets."""
    lib = _lib.load()
    H = _u32view(H, "H")
    L, m = H.shape
    G = torch.empty_like(H)
    off = torch.empty(m + 1, dtype=torch.int32, device=H.device)
    need = lib.ms_stage_scan_workspace_size(L, m)
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device=H.device)
    check(lib.ms_stage_scan(H.data_ptr(), G.data_ptr(), L, m, off.data_ptr(), ws.data_ptr(), ws.numel(),
                            _stream_ptr(stream)), "ms_stage_scan")
    return G, off


def _f32view(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def histogram_even(samples: torch.Tensor, m: int, lower: float, upper: float, *,
                   out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Device-wide Even histogram (Sec.7.3): counts[m] (int32 storage of uint32)."""
    samples = _f32view(samples, "samples")
    c = out if out is not None else torch.empty(m, dtype=torch.int32, device=samples.device)
    st = _lib.load().ms_histogram_even(samples.data_ptr(), samples.numel(), m, float(lower), float(upper),
                                       c.data_ptr(), _stream_ptr(stream))
    check(st, "ms_histogram_even")
    return c


def histogram_range(samples: torch.Tensor, splitters: torch.Tensor, *, out: torch.Tensor | None = None,
                    stream=None) -> torch.Tensor:
    """Device-wide Range histogram (Sec.7.3): counts[m] for m+1 splitters."""
    samples = _f32view(samples, "samples")
    splitters = _f32view(splitters, "splitters")
    m = splitters.numel() - 1
    c = out if out is not None else torch.empty(max(m, 1), dtype=torch.int32, device=samples.device)
    st = _lib.load().ms_histogram_range(samples.data_ptr(), samples.numel(), m, splitters.data_ptr(),
                                        c.data_ptr(), _stream_ptr(stream))
    check(st, "ms_histogram_range")
    return c


def sssp(row_ptr: torch.Tensor, col: torch.Tensor, weights: torch.Tensor, source: int, *,
         delta: int = 100, buckets: int = 10, out: torch.Tensor | None = None,
         workspace: torch.Tensor | None = None, stream=None, stats: bool = False):
    """ms_sssp: Multisplit-SSSP (Sec.7.2): shortest distances from `source` on a CSR graph
    (int32/uint32 CUDA tensors; weights >= 0) by delta-stepping whose bucketing is the
    stable multisplit with `buckets` splitter buckets of width `delta`.  Returns dist
    (uint32 bit patterns in an int32 tensor; 0xFFFFFFFF = unreachable), and the iteration
    statistics if stats=True.  Synchronizes once per iteration."""
    lib = _lib.load()
    rp = _u32view(row_ptr, "row_ptr")
    dv = rp.device
    V = rp.numel() - 1
    c = _u32view(col, "col", dv)
    w = _u32view(weights, "weights", dv, c.numel())
    E = c.numel()
    d = _u32view(out, "out", dv, V) if out is not None else torch.empty(max(V, 0), dtype=torch.int32, device=dv)
    ws = _workspace(workspace, lib.ms_sssp_workspace_size(V, E, buckets), dv)
    st = _lib.ms_sssp_stats()
    _prepare(rp)
    with torch.cuda.device(dv):
        check(lib.ms_sssp(rp.data_ptr(), c.data_ptr() if E else None, w.data_ptr() if E else None, V, E,
                          source, delta, buckets, d.data_ptr(), ws.data_ptr(), ws.numel(),
                          _stream_ptr(stream, dv), ctypes.byref(st)), "ms_sssp")
    if stats:
        return d, {"iterations": st.iterations, "items": st.items, "frontier": st.frontier,
                   "pushes": st.pushes}
    return d
