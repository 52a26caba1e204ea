"""Pins for oracle/grid (CPU only): SPEC worked examples (golden) and
brute-force tiling enumeration."""
import itertools
import json
import os
import random

import pytest

from oracle import grid as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["dims_create"])
def test_dims_create_examples(ex):
    assert G.dims_create(ex["nprocs"], tuple(ex["fixed"])) == tuple(ex["dims"])


def test_dims_create_properties():
    for n in range(1, 257):
        d = G.dims_create(n)
        assert d[0] * d[1] * d[2] == n
        assert d[0] >= d[1] >= d[2]          # tie-break gives earlier axes larger factors


@pytest.mark.parametrize("ex", GOLD["rank_of_coords"])
def test_rank_of_coords_examples(ex):
    assert G.rank_of_coords(ex["coords"], ex["dims"]) == ex["rank"]
    assert G.coords_of_rank(ex["rank"], ex["dims"]) == tuple(ex["coords"])


def test_rank_coords_bijection_and_neighbor_symmetry():
    for dims in itertools.product(range(1, 5), repeat=3):
        if dims[0] * dims[1] * dims[2] > 64:
            continue
        n = dims[0] * dims[1] * dims[2]
        seen = {G.coords_of_rank(r, dims) for r in range(n)}
        assert len(seen) == n
        for per in itertools.product((0, 1), repeat=3):
            for r in range(n):
                nb = G.neighbors(r, dims, per)
                for d in range(3):
                    lo, hi = nb[d]
                    if hi is not None:
                        assert G.neighbors(hi, dims, per)[d][0] == r
                    if lo is not None:
                        assert G.neighbors(lo, dims, per)[d][1] == r


@pytest.mark.parametrize("ex", GOLD["neighbors_x"])
def test_neighbors_examples(ex):
    assert list(G.neighbors(ex["rank"], ex["dims"], ex["periodic"])[0]) == ex["x"]


@pytest.mark.parametrize("ex", GOLD["global_size"])
def test_global_size_examples(ex):
    for d in range(3):
        assert G.global_size(ex["n"][d], ex["o"], ex["dims"][d], bool(ex["periodic"][d])) == ex["n_g"][d]


def _enumerate_global_layers(n, o, p, periodic):
    """Tile rank c's layers at offset c*(n-o) and count the distinct global
    layers; a periodic axis identifies the last rank's top
    o layers with the first rank's bottom o layers."""
    layers = set()
    for c in range(p):
        layers.update(range(c * (n - o), c * (n - o) + n))
    return len(layers) - (o if periodic else 0)


def test_global_size_matches_tiling_enumeration():
    for n in range(4, 11):
        for o in (2, 4):
            if n <= o:
                continue
            for p in range(1, 5):
                for per in (False, True):
                    assert G.global_size(n, o, p, per) == _enumerate_global_layers(n, o, p, per)


@pytest.mark.parametrize("ex", GOLD["local_to_global_1based"])
def test_local_to_global_examples(ex):
    assert G.local_to_global(ex["c"], ex["n"], ex["o"], ex["local"] - 1) + 1 == ex["global"]


@pytest.mark.parametrize("ex", GOLD["halo_spec_1based"])
def test_halo_spec_examples(ex):
    hs = G.halo_spec(ex["n"], ex["o"], ex["s"])
    assert hs["ol"] == ex["ol"] and hs["h"] == ex["h"]
    for k in ("send_lower", "recv_lower", "send_upper", "recv_upper"):
        if k in ex:
            lo, hi = hs[k]
            assert [i + 1 for i in range(lo, hi)] == ex[k]


def test_halo_spec_rejects_bad_stagger():
    with pytest.raises(ValueError):
        G.halo_spec(8, 2, 5)
    with pytest.raises(ValueError):
        G.halo_spec(8, 2, 11)


def test_window_map_neighbor_consistency_bruteforce():
    """my send_upper layers address the same global layers as my
    upper neighbour's recv_lower layers (and symmetrically); every global
    layer is covered; checked on random (n, o, p, s, periodic) cases."""
    rng = random.Random(1234)
    for _ in range(600):
        o = rng.choice((2, 4))
        n = rng.randint(o + 2, o + 8)
        p = rng.randint(1, 4)
        per = rng.random() < 0.5
        s = n + rng.choice((-1, 0, 1))
        hs = G.halo_spec(n, o, s)
        P = G.global_size(n, o, p, True)
        g = lambda c, l: G.local_to_global(c, n, o, l, per, P)
        for c in range(p):
            up = c + 1
            if up >= p:
                if not per:
                    continue
                up = 0
            if hs["h"] == 0:
                continue
            su = [g(c, l) for l in range(*hs["send_upper"])]
            rl = [g(up, l) for l in range(*hs["recv_lower"])]
            sl = [g(up, l) for l in range(*hs["send_lower"])]
            ru = [g(c, l) for l in range(*hs["recv_upper"])]
            assert su == rl and sl == ru
        covered = set()
        for c in range(p):
            covered.update(g(c, l) for l in range(s))
        N = G.field_global_size(n, o, p, per, s)
        assert covered == set(range(N))
