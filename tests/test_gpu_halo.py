"""GPU parity of update_halo (CUDA pack/unpack + local/NCCL/P2P transport)
against the oracle's update_halo: bit-exact, random per-rank data, staggered
multi-field lists, periodic and non-periodic, NaN-poisoned receive layers."""
import random

import numpy as np
import pytest

import paper_2211_15716_b200 as P
from oracle import grid as OG
from oracle import halo as OHL
import synthetic_inputs as SI

pytestmark = pytest.mark.gpu


def _run_case(dims, per, o, n, sizes, seed, poison=False, repeat=1):
    import torch
    nprocs = dims[0] * dims[1] * dims[2]
    host = {r: [SI.random_field(s[::-1], seed * 1000 + 10 * r + f) for f, s in enumerate(sizes)]
            for r in range(nprocs)}
    if poison:   # NaN in every receive layer: each must be overwritten
        for r in host:
            c = OG.coords_of_rank(r, dims)
            for A in host[r]:
                for d in range(3):
                    hs = OG.halo_spec(n[d], o[d], A.shape[2 - d])
                    if hs["h"] == 0:
                        continue
                    sl = [slice(None)] * 3
                    if c[d] > 0 or per[d]:
                        sl[2 - d] = slice(*hs["recv_lower"]); A[tuple(sl)] = np.nan
                    if c[d] < dims[d] - 1 or per[d]:
                        sl[2 - d] = slice(*hs["recv_upper"]); A[tuple(sl)] = np.nan
    ref = {r: [a.copy() for a in host[r]] for r in host}
    for _ in range(repeat):
        OHL.update_halo(ref, dims, per, n, o)
    g = P.init_global_grid(*n, dims=dims, periods=per, overlaps=o, local_ranks=nprocs, device=0)
    try:
        dev = [[torch.from_numpy(host[r][f]).cuda() for r in range(nprocs)] for f in range(len(sizes))]
        for _ in range(repeat):
            g.update_halo(*dev)
        a0 = g.buffer_allocs()
        g.update_halo(*dev) if repeat > 1 else None
        torch.cuda.synchronize()
        g.check()
        if repeat > 1:
            assert g.buffer_allocs() == a0
            for _ in range(1):
                OHL.update_halo(ref, dims, per, n, o)
        for f in range(len(sizes)):
            for r in range(nprocs):
                got = dev[f][r].cpu().numpy()
                assert np.array_equal(got, ref[r][f], equal_nan=False), (dims, per, o, n, sizes, r, f)
    finally:
        g.finalize()


def test_spec_two_rank_constants():
    import torch
    g = P.init_global_grid(8, 8, 8, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        A = [torch.full((8, 8, 8), float(r), dtype=torch.float64, device="cuda") for r in range(2)]
        g.update_halo(A)
        torch.cuda.synchronize()
        assert torch.all(A[0][:, :, 7] == 1.0) and torch.all(A[0][:, :, :7] == 0.0)
        assert torch.all(A[1][:, :, 0] == 0.0) and torch.all(A[1][:, :, 1:] == 1.0)
    finally:
        g.finalize()


def test_staggered_multifield_2x2x2():
    """B:10 in miniature: P (n^3), Vx (n+1,n,n), Vy, Vz on 2x2x2 virtual ranks."""
    n = (12, 10, 9)
    sizes = [n, (n[0] + 1, n[1], n[2]), (n[0], n[1] + 1, n[2]), (n[0], n[1], n[2] + 1)]
    for per in [(0, 0, 0), (1, 1, 1), (1, 0, 1)]:
        _run_case((2, 2, 2), per, (2, 2, 2), n, sizes, seed=3, poison=True)


def test_random_cases():
    rng = random.Random(4)
    for case in range(40):
        dims = tuple(rng.randint(1, 3) for _ in range(3))
        o = tuple(rng.choice((2, 4)) for _ in range(3))
        n = tuple(rng.randint(o[i] + 2, o[i] + 9) for i in range(3))
        per = tuple(rng.random() < 0.4 for _ in range(3))
        nf = rng.randint(1, 3)
        sizes = [tuple(n[i] + rng.choice((-1, 0, 1)) for i in range(3)) for _ in range(nf)]
        _run_case(dims, per, o, n, sizes, seed=case, poison=rng.random() < 0.5)


def test_idempotent_and_pool_stable():
    _run_case((2, 2, 1), (1, 0, 0), (2, 2, 2), (16, 12, 10), [(16, 12, 10), (17, 12, 10)], seed=8, repeat=3)


def test_stagger_error():
    import torch
    g = P.init_global_grid(8, 8, 8, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        A = [torch.zeros((8, 8, 11), dtype=torch.float64, device="cuda") for _ in range(2)]
        with pytest.raises(P.IggError) as e:
            g.update_halo(A)
        assert e.value.name == "IGG_E_STAGGER"
    finally:
        g.finalize()


@pytest.mark.slow
def test_full_size_staggered_update_512():
    """B:10 at n=512 on 2x2x2 virtual ranks (8 x 4 fields x ~1 GiB would not fit
    comfortably; the full-size check uses 2x1x1 with all four fields)."""
    n = (512, 512, 512)
    sizes = [n, (513, 512, 512), (512, 513, 512), (512, 512, 513)]
    _run_case((2, 1, 1), (1, 0, 0), (2, 2, 2), n, sizes, seed=12)


def test_gather_spec_example():
    """n=4, o=2, dims (2,1,1), each rank filled with its rank id -> (0,0,0,1,1,1) along x."""
    import torch
    g = P.init_global_grid(4, 4, 4, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        A = [torch.full((4, 4, 4), float(r), dtype=torch.float64, device="cuda") for r in range(2)]
        G = g.gather(A)
        assert G.shape == (4, 4, 6)
        assert np.array_equal(G[0, 0], np.array([0, 0, 0, 1, 1, 1], dtype=np.float64))
    finally:
        g.finalize()


def test_local_to_global_and_global_coord_spec_examples():
    """SPEC.md:123-126 (1-based there, 0-based here): n=8, o=2; coord 0: local 0 -> global 0; coord 1:
    local 0 -> global 6, local 7 -> global 13 == n_g - 1; global_coord = global index * spacing; a layer
    outside [0, n+o) is a bounds error."""
    g = P.init_global_grid(8, 8, 8, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        assert g.n_g[0] == 14
        assert g.local_to_global(0, 0, 0) == 0
        assert g.local_to_global(1, 0, 0) == 6
        assert g.local_to_global(1, 0, 7) == 13
        dx = 1.0 / (g.n_g[0] - 1)
        assert g.global_coord(1, 0, 7, dx) == 13 * dx
        assert g.global_coord(0, 1, 3, 0.5) == 1.5
        with pytest.raises(P.IggError):
            g.global_coord(1, 0, 10, dx)
    finally:
        g.finalize()


def test_gather_inverts_windows():
    """gather(window(G, rank)) == G for random global fields (the window map is the oracle)."""
    import torch
    rng = random.Random(21)
    for case in range(25):
        dims = tuple(rng.randint(1, 3) for _ in range(3))
        o = tuple(rng.choice((2, 4)) for _ in range(3))
        n = tuple(rng.randint(o[i] + 2, o[i] + 7) for i in range(3))
        per = tuple(rng.random() < 0.4 for _ in range(3))
        s = tuple(n[i] + rng.choice((-1, 0, 1)) for i in range(3))
        N = [OG.field_global_size(n[i], o[i], dims[i], per[i], s[i]) for i in range(3)]
        G = SI.random_field((N[2], N[1], N[0]), case)
        nprocs = dims[0] * dims[1] * dims[2]
        g = P.init_global_grid(*n, dims=dims, periods=per, overlaps=o, local_ranks=nprocs, device=0)
        try:
            loc = [torch.from_numpy(OG.window(G, OG.coords_of_rank(r, dims), dims, n, o, per, s)).cuda()
                   for r in range(nprocs)]
            out = g.gather(loc)
            assert out.shape == G.shape
            assert np.array_equal(out, G), (case, dims, o, n, per, s)
        finally:
            g.finalize()


def test_binary32_fields_random_cases():
    """update_halo of binary32 fields (igg_field.elsize = 4), mixed with binary64 ones in
    one call, bit-exact vs the oracle's update_halo."""
    import torch
    rng = random.Random(32)
    for case in range(12):
        dims = tuple(rng.randint(1, 3) for _ in range(3))
        o = (2, 2, 2)
        n = tuple(rng.randint(4, 9) for _ in range(3))
        per = tuple(rng.random() < 0.4 for _ in range(3))
        nprocs = dims[0] * dims[1] * dims[2]
        sizes = [n, (n[0] + 1, n[1], n[2])]
        host = {r: [SI.random_field(s[::-1], case * 100 + 10 * r + f).astype(np.float32 if f == 0 else np.float64)
                    for f, s in enumerate(sizes)] for r in range(nprocs)}
        ref = {r: [a.copy() for a in host[r]] for r in host}
        OHL.update_halo(ref, dims, per, n, o)
        g = P.init_global_grid(*n, dims=dims, periods=per, overlaps=o, local_ranks=nprocs, device=0)
        try:
            dev = [[torch.from_numpy(host[r][f]).cuda() for r in range(nprocs)] for f in range(2)]
            g.update_halo(*dev)
            torch.cuda.synchronize()
            g.check()
            for f in range(2):
                for r in range(nprocs):
                    got = dev[f][r].cpu().numpy()
                    assert got.dtype == ref[r][f].dtype and np.array_equal(got, ref[r][f]), (case, dims, per, r, f)
        finally:
            g.finalize()
