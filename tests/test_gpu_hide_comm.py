"""The generic @hide_communication API (igg_hide_communication):
any user stencil, given as a callback that enqueues the computation of a box,
is scheduled boundary-slabs-first with update_halo overlapped with the inner box
(SPEC.md:330-338).  Checked against the canonical oracle on the
global grid and against the sequential schedule, bit-exactly."""
import numpy as np
import pytest

import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import heat3d as app
from oracle import grid as OG
from oracle import heat3d as OH

from _heat_cases import oracle_global

pytestmark = pytest.mark.gpu


def _torch_heat_step(T, T2, Ci, lam, dt, d):
    """The Fig. 1 cell (canonical association) as separate torch ops on a box."""
    rx, ry, rz = 1.0 / (d[0] * d[0]), 1.0 / (d[1] * d[1]), 1.0 / (d[2] * d[2])

    def step(lr, lo, hi, stream):
        x0, y0, z0 = lo
        x1, y1, z1 = hi
        t = T[lr]
        c = t[z0:z1, y0:y1, x0:x1]
        d2x = (t[z0:z1, y0:y1, x0 + 1:x1 + 1] - c) - (c - t[z0:z1, y0:y1, x0 - 1:x1 - 1])
        d2y = (t[z0:z1, y0 + 1:y1 + 1, x0:x1] - c) - (c - t[z0:z1, y0 - 1:y1 - 1, x0:x1])
        d2z = (t[z0 + 1:z1 + 1, y0:y1, x0:x1] - c) - (c - t[z0 - 1:z1 - 1, y0:y1, x0:x1])
        lap = ((d2x * rx) + (d2y * ry)) + (d2z * rz)
        T2[lr][z0:z1, y0:y1, x0:x1] = c + dt * ((lam * Ci[lr][z0:z1, y0:y1, x0:x1]) * lap)
    return step


@pytest.mark.parametrize("case", [
    dict(n=(24, 20, 18), dims=(2, 1, 1), per=(0, 0, 0), bw=(4, 2, 2)),
    dict(n=(24, 20, 18), dims=(2, 2, 1), per=(1, 0, 0), bw=(4, 3, 2)),
    dict(n=(22, 20, 18), dims=(1, 2, 2), per=(0, 1, 1), bw=(2, 2, 2)),
    dict(n=(24, 20, 18), dims=(2, 1, 1), per=(0, 0, 0), bw=(0, 0, 0)),
])
def test_user_stencil_vs_oracle(case):
    import torch
    n, dims, per, bw = case["n"], case["dims"], case["per"], case["bw"]
    nprocs = dims[0] * dims[1] * dims[2]
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=nprocs, device=0)
    try:
        T, T2, Ci = app.alloc_fields(g)
        app.init_random(g, T, T2, Ci)
        d = app.spacing(g)
        dt = app.stable_dt(g, Ci, *d)
        for _ in range(4):
            g.hide_communication(bw, _torch_heat_step(T, T2, Ci, 1.0, dt, d), T2)
            T, T2 = T2, T
        torch.cuda.synchronize()
        N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
        can, dtr = oracle_global(N, per, 4)
        assert dt == dtr
        for r in range(nprocs):
            W = OG.window(can, OG.coords_of_rank(r, dims), dims, n, (2, 2, 2), per, n)
            assert np.array_equal(T[r].cpu().numpy(), W), r
    finally:
        g.finalize()


def test_staggered_fields_overlap_equals_sequential():
    """A user step over staggered fields (P n^3, Vx (n+1)...) with their halos exchanged
    inside hide_communication: overlap == sequential, bit-exact."""
    import torch
    n, dims, per = (20, 18, 16), (2, 2, 1), (0, 1, 0)
    sizes = [n, (n[0] + 1, n[1], n[2]), (n[0], n[1] + 1, n[2])]
    res = []
    for bw in [(0, 0, 0), (4, 4, 2)]:
        g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=4, device=0)
        try:
            gen = torch.Generator(device="cuda").manual_seed(5)
            F = [[torch.rand(s[::-1], dtype=torch.float64, device="cuda", generator=gen) for _ in range(4)]
                 for s in sizes]

            def step(lr, lo, hi, stream):
                x0, y0, z0 = lo
                x1, y1, z1 = hi
                for f in F:   # a local update of every field's cells of the box (reads P only)
                    f[lr][z0:z1, y0:y1, x0:x1] = f[lr][z0:z1, y0:y1, x0:x1] * 0.5 + F[0][lr][z0:z1, y0:y1, x0:x1] * 0.25

            for _ in range(3):
                g.hide_communication(bw, step, *F)
            torch.cuda.synchronize()
            res.append([[t.cpu().numpy() for t in f] for f in F])
        finally:
            g.finalize()
    for fa, fb in zip(res[0], res[1]):
        for a, b in zip(fa, fb):
            assert np.array_equal(a, b)


def test_width_error():
    g = P.init_global_grid(20, 18, 16, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        T, T2, Ci = app.alloc_fields(g)
        with pytest.raises(P.IggError) as e:
            g.hide_communication((1, 2, 2), lambda *a: None, T2)
        assert e.value.name == "IGG_E_WIDTH"
    finally:
        g.finalize()
