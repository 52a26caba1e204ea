"""Pins for oracle/halo.update_halo (CPU only).

The central pin compares two independent definitions: the step-by-step
exchange algorithm and the window map:
a random global field cut into every rank's window, with the receive layers
poisoned by NaN, must be restored exactly by update_halo.  Plus SPEC's worked
examples and properties."""
import itertools
import json
import os
import random

import numpy as np
import pytest

from oracle import grid as G
from oracle import halo as HL
import synthetic_inputs as SI

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _recv_mask(shape_zyx, n, o, dims, coords, periodic):
    """True on every layer a rank receives (recv ranges of axes with a neighbour)."""
    m = np.zeros(shape_zyx, bool)
    for d in range(3):
        ax = 2 - d
        hs = G.halo_spec(n[d], o[d], shape_zyx[ax])
        if hs["h"] == 0:
            continue
        sl = [slice(None)] * 3
        if coords[d] > 0 or periodic[d]:
            sl[ax] = slice(*hs["recv_lower"]); m[tuple(sl)] = True
        if coords[d] < dims[d] - 1 or periodic[d]:
            sl[ax] = slice(*hs["recv_upper"]); m[tuple(sl)] = True
    return m


def _random_case(rng):
    dims = tuple(rng.randint(1, 3) for _ in range(3))
    o = tuple(rng.choice((2, 4)) for _ in range(3))
    n = tuple(rng.randint(o[d] + 2, o[d] + 5) for d in range(3))
    per = tuple(rng.random() < 0.4 for _ in range(3))
    nf = rng.randint(1, 3)
    sizes = [tuple(n[d] + rng.choice((-1, 0, 1)) for d in range(3)) for _ in range(nf)]
    return dims, o, n, per, sizes


def test_update_halo_restores_windows_of_global_field():
    rng = random.Random(7)
    for case in range(300):
        dims, o, n, per, sizes = _random_case(rng)
        nranks = dims[0] * dims[1] * dims[2]
        fields, expect = {}, {}
        globals_ = []
        for f, s in enumerate(sizes):
            N = [G.field_global_size(n[d], o[d], dims[d], per[d], s[d]) for d in range(3)]
            globals_.append(SI.random_field((N[2], N[1], N[0]), 100 * case + f))
        for r in range(nranks):
            c = G.coords_of_rank(r, dims)
            fields[r], expect[r] = [], []
            for f, s in enumerate(sizes):
                W = G.window(globals_[f], c, dims, n, o, per, s)
                A = W.copy()
                A[_recv_mask(A.shape, n, o, dims, c, per)] = np.nan
                fields[r].append(A); expect[r].append(W)
        HL.update_halo(fields, dims, per, n, o)
        for r in range(nranks):
            for f in range(len(sizes)):
                assert np.array_equal(fields[r][f], expect[r][f]), (case, r, f)


def test_spec_two_rank_constants():
    g = GOLD["update_halo_2rank_constants"]
    n = tuple(g["n"]); o = (g["o"],) * 3; dims = tuple(g["dims"])
    fields = {r: [np.full(n[::-1], float(r))] for r in range(2)}
    HL.update_halo(fields, dims, (0, 0, 0), n, o)
    a0, a1 = fields[0][0], fields[1][0]
    assert np.all(a0[:, :, 7] == g["rank0_layer_x8"]) and np.all(a0[:, :, :7] == 0.0)
    assert np.all(a1[:, :, 0] == g["rank1_layer_x1"]) and np.all(a1[:, :, 1:] == 1.0)


def test_spec_self_wrap():
    g = GOLD["update_halo_selfwrap"]
    n = tuple(g["n"]); o = (g["o"],) * 3
    A = np.broadcast_to(np.arange(1, 9, dtype=np.float64), n[::-1]).copy()   # data[x] = x (1-based)
    fields = {0: [A]}
    HL.update_halo(fields, (1, 1, 1), tuple(g["periodic"]), n, o)
    assert np.all(A[:, :, 0] == g["layer1_equals_old"])
    assert np.all(A[:, :, 7] == g["layer8_equals_old"])
    assert np.all(A[:, :, 1:7] == np.arange(2, 8))


def test_single_rank_nonperiodic_is_noop():
    A = SI.random_field((6, 7, 8), 3); B = A.copy()
    HL.update_halo({0: [A]}, (1, 1, 1), (0, 0, 0), (8, 7, 6), (2, 2, 2))
    assert np.array_equal(A, B)


def test_pack_layout_offset():
    g = GOLD["pack_offset"]
    nx, ny, nz = g["shape_xyz"]
    A = np.arange(nx * ny * nz, dtype=np.float64).reshape(nz, ny, nx)
    buf = HL.pack(A, 0, 6, 7)                  # any single x layer
    assert buf.size == g["buffer_len"]
    y, z = g["y_1based"] - 1, g["z_1based"] - 1
    assert buf[g["offset_0based"]] == A[z, y, 6]
    B = np.zeros_like(A)
    HL.unpack(buf, B, 0, 6, 7)
    assert np.array_equal(B[:, :, 6], A[:, :, 6]) and np.count_nonzero(B[:, :, :6]) == 0


def test_properties_noninterference_idempotence_multifield():
    rng = random.Random(11)
    for case in range(60):
        dims, o, n, per, sizes = _random_case(rng)
        nranks = dims[0] * dims[1] * dims[2]
        base = {r: [SI.random_field(s[::-1], 1000 * case + 10 * r + f) for f, s in enumerate(sizes)]
                for r in range(nranks)}
        one = {r: [a.copy() for a in base[r]] for r in base}
        HL.update_halo(one, dims, per, n, o)
        for r in range(nranks):                # non-interference
            c = G.coords_of_rank(r, dims)
            for f in range(len(sizes)):
                m = _recv_mask(base[r][f].shape, n, o, dims, c, per)
                assert np.array_equal(one[r][f][~m], base[r][f][~m])
        two = {r: [a.copy() for a in one[r]] for r in one}
        HL.update_halo(two, dims, per, n, o)
        for r in range(nranks):                # idempotence on static data
            for f in range(len(sizes)):
                assert np.array_equal(two[r][f], one[r][f])
        seq = {r: [a.copy() for a in base[r]] for r in base}
        for f in range(len(sizes)):            # multi-field == sequential single-field
            sub = {r: [seq[r][f]] for r in seq}
            HL.update_halo(sub, dims, per, n, o)
        for r in range(nranks):
            for f in range(len(sizes)):
                assert np.array_equal(seq[r][f], one[r][f])
