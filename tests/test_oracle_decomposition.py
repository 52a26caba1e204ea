"""Decomposition independence in the oracle world (CPU only).

Pins the expectation every distributed GPU parity test uses: after nt steps of
{local step!; update_halo!(T2); swap} on every rank, each
rank's local array -- halos and global-boundary layers included -- equals the
window of the single global run.
The local step is the oracle heat step on the local array with non-periodic
local semantics (cells 1..s-2), which is what the paper's kernel does per rank
(@inn writes inner points only)."""
import random

import numpy as np

from oracle import grid as G
from oracle import halo as HL
from oracle import heat3d as H
import synthetic_inputs as SI


def _distributed_run(T0g, Cig, dims, n, o, per, nt, lam, dt, d, mode):
    nranks = dims[0] * dims[1] * dims[2]
    T, T2, C = {}, {}, {}
    for r in range(nranks):
        c = G.coords_of_rank(r, dims)
        T[r] = G.window(T0g, c, dims, n, o, per, n)
        T2[r] = T[r].copy()                                  # T2 = copy(T)
        C[r] = G.window(Cig, c, dims, n, o, per, n)
    for _ in range(nt):
        for r in range(nranks):
            H.heat_step(T[r], C[r], T2[r], (0, 0, 0), lam, dt, *d, mode)
        HL.update_halo({r: [T2[r]] for r in range(nranks)}, dims, per, n, o)
        T, T2 = T2, T
    return T


def test_distributed_oracle_equals_global_windows():
    rng = random.Random(2211)
    for case in range(40):
        dims = tuple(rng.randint(1, 3) for _ in range(3))
        o = tuple(rng.choice((2, 4)) for _ in range(3))
        n = tuple(rng.randint(o[i] + 2, o[i] + 5) for i in range(3))
        per = tuple(rng.random() < 0.4 for _ in range(3))
        N = [G.global_size(n[i], o[i], dims[i], per[i]) for i in range(3)]
        if min(N) < 3:
            continue
        T0g, Cig = SI.global_heat_fields(*N, seed_T=case, seed_C=case + 99)
        d = [H.spacing(1.0, N[i], per[i]) for i in range(3)]
        dt = H.stable_dt(*d, 1.0, Cig)
        mode = H.CANONICAL if case % 2 else H.LITERAL
        ref = H.heat_run(T0g, Cig, 4, per, 1.0, dt, *d, mode)
        out = _distributed_run(T0g, Cig, dims, n, o, per, 4, 1.0, dt, d, mode)
        for r in out:
            c = G.coords_of_rank(r, dims)
            assert np.array_equal(out[r], G.window(ref, c, dims, n, o, per, n)), (case, r)


def test_b7_emulated_split_both_readings():
    """Config B:7: 32^3 local on 1x1x1 and the emulated 2x1x1 split, nt=10.
    Reading (i): 2 ranks x 32^3 -> global 62x32x32.  Reading (ii): global 32^3
    as 2 ranks of 17x32x32."""
    o = (2, 2, 2); per = (0, 0, 0)
    for n in [(32, 32, 32), (17, 32, 32)]:
        dims = (2, 1, 1)
        N = [G.global_size(n[i], o[i], dims[i], False) for i in range(3)]
        T0g, Cig = SI.global_heat_fields(*N)
        d = [H.spacing(1.0, N[i], False) for i in range(3)]
        dt = H.stable_dt(*d, 1.0, Cig)
        ref = H.heat_run(T0g, Cig, 10, per, 1.0, dt, *d, H.LITERAL)
        out = _distributed_run(T0g, Cig, dims, n, o, per, 10, 1.0, dt, d, H.LITERAL)
        for r in out:
            c = G.coords_of_rank(r, dims)
            assert np.array_equal(out[r], G.window(ref, c, dims, n, o, per, n))
