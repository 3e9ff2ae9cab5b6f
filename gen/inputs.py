"""Seeded, counter-based synthetic inputs (host side, numpy).

This module holds NO multisplit arithmetic: it only draws keys/values whose
bucket distribution matches the paper's workloads (uniform over buckets
P:1112-1115; alpha-uniform P:1535; binomial B(m-1, 1/2) P:1507).  It is the
one module shared by the oracle side (tests, bench cpu_baseline) and the CUDA
side (which uses the identical generator in gen/csrc/gen.cu; a GPU test
checks the two byte for byte).

Recipe:
  mix64(z)      splitmix64 finalizer
  h(s, k, i)    = mix64(seed ^ (k * 0xD1B54A32D192ED03) ^ i)          (64-bit)
  rnd32(s,k,i)  = h(s,k,i) >> 32
  below(x, w)   = (x * w) >> 32                                        in [0, w)
  uniform keys  key_i = rnd32(seed, 0, i)
  bucket draws  uniform  b_i = below(rnd32(seed,1,i), m)
                skew     hot = below(rnd32(seed,2,0), m);
                         b_i = rnd32(seed,3,i) < alpha32 ? below(rnd32(seed,1,i), m) : hot
                binomial b_i = popcount of the low (m-1) bits of h(seed,4..7,i)
  key from bucket (so that f(key) = b_i):
                IDENTITY key = b ; RADIX(s,r) key = (rnd32(seed,0,i) & ~(mask<<s)) | (b<<s)
                DELTA(D) key = lo_b + below(rnd32(seed,0,i), hi_b - lo_b),
                         lo_b = b*D, hi_b = (b == m-1) ? 2^32 : min((b+1)*D, 2^32)
  values        parity val_i = i ; throughput val_i = rnd32(seed, 8, i)
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)

IDENTITY, DELTA, RADIX = 0, 1, 2
DIST_UNIFORM, DIST_SKEW, DIST_BINOMIAL = 0, 1, 2

_CHUNK = 1 << 24


def mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * C1
        z = (z ^ (z >> np.uint64(27))) * C2
        return z ^ (z >> np.uint64(31))


def h64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(stream) * STREAM_MUL)
    return mix64(base ^ idx.astype(np.uint64))


def rnd32(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    return (h64(seed, stream, idx) >> np.uint64(32)).astype(np.uint32)


def below(x32: np.ndarray, w) -> np.ndarray:
    """Map a uniform uint32 to [0, w) by the high word of x*w (w <= 2^32)."""
    w = np.asarray(w, dtype=np.uint64)
    return ((x32.astype(np.uint64) * w) >> np.uint64(32)).astype(np.uint32)


def alpha32(alpha: float) -> int:
    return min(int(alpha * 4294967296.0), 1 << 32)


def _popcount64(x: np.ndarray) -> np.ndarray:
    return np.bitwise_count(x).astype(np.uint32)


def _bucket_draw(seed, idx, m, dist, a32):
    if dist == DIST_UNIFORM:
        return below(rnd32(seed, 1, idx), m)
    if dist == DIST_SKEW:
        hot = int(below(rnd32(seed, 2, np.zeros(1, np.uint64)), m)[0])
        u = below(rnd32(seed, 1, idx), m)
        take_uniform = rnd32(seed, 3, idx).astype(np.uint64) < np.uint64(a32)
        return np.where(take_uniform, u, np.uint32(hot)).astype(np.uint32)
    if dist == DIST_BINOMIAL:
        nbits = m - 1
        tot = np.zeros(idx.size, np.uint32)
        for w in range(4):
            take = min(max(nbits - 64 * w, 0), 64)
            if take == 0:
                break
            mask = np.uint64((1 << take) - 1) if take < 64 else M64
            tot += _popcount64(h64(seed, 4 + w, idx) & mask)
        return tot
    raise ValueError(f"unknown dist {dist}")


def _key_from_bucket(seed, idx, b, kind, m, delta, shift, bits):
    if kind == IDENTITY:
        return b.astype(np.uint32)
    r = rnd32(seed, 0, idx)
    if kind == RADIX:
        mask = np.uint32(((1 << bits) - 1) << shift)
        return ((r & ~mask) | (b.astype(np.uint32) << np.uint32(shift))).astype(np.uint32)
    if kind == DELTA:
        lo = b.astype(np.uint64) * np.uint64(delta)
        hi = np.minimum(lo + np.uint64(delta), np.uint64(1 << 32))
        hi = np.where(b == m - 1, np.uint64(1 << 32), hi)
        if np.any(lo >= np.uint64(1 << 32)):
            raise ValueError("bucket not reachable with this delta")
        return (lo + below(r, hi - lo)).astype(np.uint32)
    raise ValueError(f"unknown kind {kind}")


def keys(n: int, seed: int, kind: int = DELTA, m: int = 2, delta: int = 0, shift: int = 0,
         bits: int = 0, dist: int = DIST_UNIFORM, alpha: float = 0.1) -> np.ndarray:
    """n keys whose buckets under f = (kind, m, delta, shift, bits) follow `dist`."""
    out = np.empty(n, np.uint32)
    a32 = alpha32(alpha)
    for s in range(0, n, _CHUNK):
        idx = np.arange(s, min(n, s + _CHUNK), dtype=np.uint64)
        if dist == DIST_UNIFORM and kind != IDENTITY:
            out[s:s + idx.size] = rnd32(seed, 0, idx)
        else:
            b = _bucket_draw(seed, idx, m, dist, a32)
            out[s:s + idx.size] = _key_from_bucket(seed, idx, b, kind, m, delta, shift, bits)
    return out


def values(n: int, seed: int, parity: bool = True) -> np.ndarray:
    """Parity runs: v_i = i (stability visible).  Throughput runs: rnd32(seed, 8, i)."""
    if parity:
        return np.arange(n, dtype=np.uint32)
    out = np.empty(n, np.uint32)
    for s in range(0, n, _CHUNK):
        idx = np.arange(s, min(n, s + _CHUNK), dtype=np.uint64)
        out[s:s + idx.size] = rnd32(seed, 8, idx)
    return out


def floats(n: int, seed: int, upper: float = 1024.0) -> np.ndarray:
    """Histogram samples U[0, upper) (Sec.7.3: 2^25 floats in [0, 1024)):
    x_i = (rnd32(seed, 10, i) >> 8) * upper * 2^-24, exact in binary32 when upper
    is a power of two."""
    out = np.empty(n, np.float32)
    scale = np.float64(upper) / float(1 << 24)
    for s in range(0, n, _CHUNK):
        idx = np.arange(s, min(n, s + _CHUNK), dtype=np.uint64)
        r = (rnd32(seed, 10, idx) >> np.uint32(8)).astype(np.float64)
        out[s:s + idx.size] = (r * scale).astype(np.float32)
    return out


def splitters(m: int, seed: int, upper: float = 1024.0) -> np.ndarray:
    """Range-histogram splitters s_0 = 0 < s_1 < ... < s_m = upper: m-1 distinct
    random interior values on the same 2^-24 * upper grid."""
    got: list[float] = []
    seen = set()
    i = 0
    scale = upper / float(1 << 24)
    while len(got) < m - 1:
        r = int(rnd32(seed, 11, np.array([i], np.uint64))[0]) >> 8
        i += 1
        if r == 0 or r in seen:
            continue
        seen.add(r)
        got.append(r * scale)
    return np.array([0.0] + sorted(got) + [upper], dtype=np.float32)
