"""Seeded synthetic graphs for the SSSP application of Sec.7.2.

This module holds NO SSSP arithmetic: it draws an R-MAT edge list and lays it
out as CSR.  Recipe (SSSP):
  R-MAT (P:1831 footnote: "(a,b,c,d) = (0.5, 0.1, 0.1, 30)", read as d = 0.3, R28):
    edge e, level l = 0..scale-1: x = rnd32(seed, 16 + l, e);
      quadrant (0,0) if x < a*2^32, (0,1) if < (a+b)*2^32, (1,0) if < (a+b+c)*2^32, else (1,1);
      bit (scale-1-l) of src / dst = the quadrant's row / column bit
  weights: w_e = below(rnd32(seed, 15, e), 1001), an integer in [0, 1000]
  CSR: edges stably ordered by source (self loops and parallel edges are kept).
"""
from __future__ import annotations

import numpy as np

from gen.inputs import below, rnd32


def rmat_edges(scale: int, edge_factor: int, seed: int, a=0.5, b=0.1, c=0.1):
    V = 1 << scale
    E = V * edge_factor
    idx = np.arange(E, dtype=np.uint64)
    ta, tb, tc = (np.uint64(int(p * 4294967296.0)) for p in (a, a + b, a + b + c))
    src = np.zeros(E, np.uint32)
    dst = np.zeros(E, np.uint32)
    for lvl in range(scale):
        x = rnd32(seed, 16 + lvl, idx).astype(np.uint64)
        row = (x >= tb).astype(np.uint32)                       # quadrants (1,0), (1,1)
        col = (((x >= ta) & (x < tb)) | (x >= tc)).astype(np.uint32)  # (0,1), (1,1)
        bit = np.uint32(1 << (scale - 1 - lvl))
        src |= row * bit
        dst |= col * bit
    w = below(rnd32(seed, 15, idx), 1001)
    return V, src, dst, w


def to_csr(V: int, src, dst, w):
    order = np.argsort(src, kind="stable")
    row_ptr = np.zeros(V + 1, np.uint32)
    np.cumsum(np.bincount(src, minlength=V), out=row_ptr[1:])
    return row_ptr, dst[order].astype(np.uint32), w[order].astype(np.uint32)


def rmat_csr(scale: int, edge_factor: int, seed: int, undirected: bool = False):
    """R-MAT CSR; undirected=True adds the reverse arc of every edge (same weight), the
    paper's rmat (Table graphs: 0.8 M vertices, 4.8 M edges, average degree 12 = 2 x 4.8 / 0.8,
    and its MTEPS = 9.6 M arcs / time; reading R29)."""
    V, s, d, w = rmat_edges(scale, edge_factor, seed)
    if undirected:
        s, d, w = np.concatenate([s, d]), np.concatenate([d, s]), np.concatenate([w, w])
    return (V,) + to_csr(V, s, d, w)
