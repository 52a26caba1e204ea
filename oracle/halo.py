"""oracle/halo.py -- CPU ORACLE for update_halo! (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg may import this module; it shares no code with the product.

``update_halo`` follows the paper's halo update ("a second
function performs a halo update on it", :77 ``update_halo!(T2)``, :94) in the
order SPEC.md:211 states it: axes strictly x, then y, then z; for every field
and every side with a neighbour the send layers (full extent of the other two
axes, their halos included) are copied out, then copied into the neighbour's
receive layers; an axis completes before the next starts.  Ranges come from
``oracle.grid.halo_spec``.  Self-wrap (periodic, p=1) goes
through the same copy.

Arrays are numpy (s_z, s_y, s_x) float64 (x fastest); axis d (0=x,1=y,2=z)
is numpy axis 2-d.
"""
from __future__ import annotations

import numpy as np

from . import grid as G


def _sl(arr_ndim_axis: int, lo: int, hi: int):
    s = [slice(None)] * 3
    s[arr_ndim_axis] = slice(lo, hi)
    return tuple(s)


def update_halo(fields_by_rank: dict, dims, periodic, n, o) -> None:
    """In place.  fields_by_rank: {rank: [field arrays, same list on every rank]}."""
    ranks = sorted(fields_by_rank)
    assert ranks == list(range(dims[0] * dims[1] * dims[2]))
    nf = len(fields_by_rank[0])
    for d in range(3):                       # x -> y -> z
        ax = 2 - d
        messages = []                        # (dst rank, field, recv range, payload)
        for r in ranks:
            lower, upper = G.neighbors(r, dims, periodic)[d]
            for f in range(nf):
                A = fields_by_rank[r][f]
                hs = G.halo_spec(n[d], o[d], A.shape[ax])
                if hs["h"] == 0:
                    continue
                if upper is not None:        # my send_upper -> upper's recv_lower
                    lo, hi = hs["send_upper"]
                    messages.append((upper, f, hs["recv_lower"], A[_sl(ax, lo, hi)].copy()))
                if lower is not None:        # my send_lower -> lower's recv_upper
                    lo, hi = hs["send_lower"]
                    messages.append((lower, f, hs["recv_upper"], A[_sl(ax, lo, hi)].copy()))
        for dst, f, (lo, hi), payload in messages:   # all waits of the axis, then unpack
            fields_by_rank[dst][f][_sl(ax, lo, hi)] = payload


def pack(A: np.ndarray, d: int, lo: int, hi: int) -> np.ndarray:
    """the slab [lo,hi) of axis d as a flat buffer, x fastest,
    then y, then z."""
    return np.ascontiguousarray(A[_sl(2 - d, lo, hi)]).reshape(-1)


def unpack(buf: np.ndarray, A: np.ndarray, d: int, lo: int, hi: int) -> None:
    shape = list(A.shape)
    shape[2 - d] = hi - lo
    A[_sl(2 - d, lo, hi)] = buf.reshape(shape)
