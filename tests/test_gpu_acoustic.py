"""GPU parity of the second workload: igg_acoustic_step --
compute_V under @hide_communication with update_halo!(Vx, Vy, Vz), then compute_P
-- against the acoustic oracle on the global grid (oracle/acoustic3d.py), bit for
bit, on virtual-rank topologies (config B:10's staggered field set), periodic and
not, every schedule; plus argument errors and a full-size (512^3) sampled check."""
import numpy as np
import pytest

import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import acoustic3d as app
from oracle import acoustic3d as OA
from oracle import grid as OG
import synthetic_inputs as SI

pytestmark = pytest.mark.gpu


def _run_case(n, dims, per, bw, nt, rho=1.2, K=0.8):
    import torch
    nprocs = dims[0] * dims[1] * dims[2]
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=nprocs, device=0)
    try:
        F = app.alloc_fields(g)
        app.init_random(g, F)
        d = app.spacing(g)
        dt = app.stable_dt(d, rho, K)
        app.run(g, F, nt, dt, d, rho, K, bw=bw)
        torch.cuda.synchronize()
        g.check()
        N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
        shapes = OA.field_shapes(N, per)
        ref = OA.run(*SI.global_acoustic_fields(shapes), nt, per, dt, rho, K, *d)
        sizes = [n, (n[0] + 1, n[1], n[2]), (n[0], n[1] + 1, n[2]), (n[0], n[1], n[2] + 1)]
        for f in range(4):
            for r in range(nprocs):
                W = OG.window(ref[f], OG.coords_of_rank(r, dims), dims, n, (2, 2, 2), per, sizes[f])
                got = F[f][r].cpu().numpy()
                assert np.array_equal(got, W), (n, dims, per, bw, f, r, np.argwhere(got != W)[:3])
    finally:
        g.finalize()


@pytest.mark.parametrize("case", [
    dict(n=(37, 11, 9), dims=(1, 1, 1), per=(0, 0, 0), bw=(0, 0, 0)),      # ragged, several x blocks
    dict(n=(70, 13, 40), dims=(1, 1, 1), per=(0, 0, 0), bw=(16, 4, 4)),    # > one z chunk
    dict(n=(20, 18, 16), dims=(2, 1, 1), per=(0, 0, 0), bw=(4, 4, 4)),
    dict(n=(20, 18, 16), dims=(2, 2, 1), per=(1, 0, 0), bw=(3, 3, 3)),
    dict(n=(21, 17, 16), dims=(1, 2, 2), per=(0, 1, 1), bw=(5, 4, 3)),
    dict(n=(20, 18, 16), dims=(2, 2, 2), per=(0, 0, 0), bw=(0, 0, 0)),
    dict(n=(20, 18, 16), dims=(2, 2, 2), per=(1, 1, 1), bw=(4, 4, 4)),
    dict(n=(12, 10, 9), dims=(1, 1, 1), per=(1, 1, 1), bw=(3, 3, 3)),      # self-wrap on every axis
    dict(n=(40, 36, 34), dims=(3, 1, 2), per=(1, 0, 1), bw=(16, 4, 4)),
])
def test_acoustic_vs_oracle(case):
    _run_case(case["n"], case["dims"], case["per"], case["bw"], nt=5)


def test_width_and_shape_errors():
    import torch
    g = P.init_global_grid(20, 18, 16, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        F = app.alloc_fields(g)
        for f in F:
            for t in f:
                t.zero_()
        with pytest.raises(P.IggError) as e:
            g.acoustic_step(*F, 0.01, 1.0, 1.0, 0.1, 0.1, 0.1, bw=(2, 2, 2))   # Vx overlap 3 on x
        assert e.value.name == "IGG_E_WIDTH"
        with pytest.raises(P.IggError) as e:
            g.acoustic_step(*F, 0.01, 0.0, 1.0, 0.1, 0.1, 0.1)
        assert e.value.name == "IGG_E_ARG"
        bad = [torch.zeros((16, 18, 20), dtype=torch.float64, device="cuda") for _ in range(2)]
        with pytest.raises(ValueError):
            g.acoustic_step(F[0], bad, F[2], F[3], 0.01, 1.0, 1.0, 0.1, 0.1, 0.1)
    finally:
        g.finalize()


def test_schedules_agree_bitwise():
    """hide_communication widths change only the schedule: every bw gives the same bits."""
    import torch
    res = []
    for bw in [(0, 0, 0), (3, 3, 3), (8, 6, 5)]:
        g = P.init_global_grid(24, 20, 18, dims=(2, 2, 1), periods=(0, 1, 0), local_ranks=4, device=0)
        try:
            F = app.alloc_fields(g)
            app.init_random(g, F, seed=9)
            d = app.spacing(g)
            app.run(g, F, 4, app.stable_dt(d), d, bw=bw)
            torch.cuda.synchronize()
            res.append([[t.cpu().numpy() for t in f] for f in F])
        finally:
            g.finalize()
    for other in res[1:]:
        for fa, fb in zip(res[0], other):
            for a, b in zip(fa, fb):
                assert np.array_equal(a, b)


@pytest.mark.slow
def test_full_size_512_sampled():
    """The bench configuration (512^3 local, one GPU, bw (16,4,4)), nt = 3: sub-boxes at the corners,
    faces and centre are re-run by the oracle as grids of their own; cells farther than the domain of
    dependence (2 layers per step) from a sub-box edge that is not a real boundary agree bit for bit."""
    import torch
    n, nt = (512, 512, 512), 3
    g = P.init_global_grid(*n, local_ranks=1, device=0)
    try:
        F = app.alloc_fields(g)
        app.init_random(g, F)
        F0 = [[t.clone() for t in f] for f in F]
        d = app.spacing(g)
        dt = app.stable_dt(d)
        app.run(g, F, nt, dt, d)
        torch.cuda.synchronize()
        m, L = 2 * nt + 2, 40
        stag = {1: 2, 2: 1, 3: 0}    # field -> its staggered (z, y, x) array axis
        for z0 in (0, 250, 512 - L):
            for y0 in (0, 301, 512 - L):
                for x0 in (0, 7, 512 - L):
                    start = (z0, y0, x0)
                    sub0, subg = [], []
                    for f in range(4):
                        ext = [slice(start[a], start[a] + L + (1 if stag.get(f) == a else 0)) for a in range(3)]
                        sub0.append(F0[f][0][tuple(ext)].cpu().numpy())
                        subg.append(F[f][0][tuple(ext)].cpu().numpy())
                    ref = OA.run(*sub0, nt, (0, 0, 0), dt, app.RHO, app.K, *d)
                    for f in range(4):
                        cut = tuple(slice(m if start[a] > 0 else 0,
                                          ref[f].shape[a] - (m if start[a] + L < 512 else 0)) for a in range(3))
                        assert np.array_equal(ref[f][cut], subg[f][cut]), (start, f)
    finally:
        g.finalize()


def _run_fused(n, nt, rho=1.2, K=0.8, per=(0, 0, 0), dims=(1, 1, 1)):
    """igg_acoustic_run (double-buffered; fused V+P sweep when no axis exchanges) vs the oracle."""
    import torch
    R = dims[0] * dims[1] * dims[2]
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=R, device=0)
    try:
        F = app.alloc_fields(g)
        F2 = app.alloc_fields(g)
        for f in F2:   # garbage in the second set: every element must be written
            for t in f:
                t.fill_(float("nan"))
        app.init_random(g, F)
        d = app.spacing(g)
        dt = app.stable_dt(d, rho, K)
        l0 = g.kernel_launches()
        A, B = g.acoustic_run(F, F2, nt, dt, rho, K, *d)
        torch.cuda.synchronize()
        g.check()
        N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
        ref = OA.run(*SI.global_acoustic_fields(OA.field_shapes(N, per)), nt, per, dt, rho, K, *d)
        sizes = [n, (n[0] + 1, n[1], n[2]), (n[0], n[1] + 1, n[2]), (n[0], n[1], n[2] + 1)]
        for f in range(4):
            for r in range(R):
                W = OG.window(ref[f], OG.coords_of_rank(r, dims), dims, n, (2, 2, 2), per, sizes[f])
                got = A[f][r].cpu().numpy()
                assert np.array_equal(got, W), (n, f, r, np.argwhere(got != W)[:3])
        return g.kernel_launches() - l0
    finally:
        g.finalize()


@pytest.mark.parametrize("n", [(37, 11, 9), (70, 13, 40), (33, 5, 17), (64, 8, 33), (5, 4, 3)])
@pytest.mark.parametrize("nt", [1, 4])
def test_acoustic_fused_run_vs_oracle(n, nt):
    """One fused V+P sweep per step (double-buffered, 64 B/cell): bit-exact vs the oracle on ragged sizes,
    several x-tiles / y-tiles / z-chunks, odd and even step counts (the result in either buffer set)."""
    launches = _run_fused(n, nt)
    assert launches == nt   # one kernel per step


@pytest.mark.parametrize("case", [dict(n=(20, 18, 16), dims=(2, 1, 1), per=(0, 0, 0)),
                                  dict(n=(12, 10, 9), dims=(1, 1, 1), per=(1, 1, 1))])
def test_acoustic_run_with_exchange_falls_back_to_steps(case):
    """With an exchanged axis igg_acoustic_run is igg_acoustic_step per step in place (same bits)."""
    _run_fused(case["n"], 3, per=case["per"], dims=case["dims"])


@pytest.mark.slow
def test_acoustic_fused_full_size_512_sampled():
    """The bench configuration of the fused sweep (512^3, 1 GPU): sub-boxes re-run by the oracle as grids of
    their own, cells outside the sub-box edges' domain of dependence (nt+1 layers) compared bitwise."""
    import torch
    n, nt, m, L = (512, 512, 512), 2, 3, 24
    g = P.init_global_grid(*n, device=0)
    try:
        F = app.alloc_fields(g)
        F2 = app.alloc_fields(g)
        app.init_random(g, F)
        F0 = [f[0].clone() for f in F]
        d = app.spacing(g)
        dt = app.stable_dt(d)
        A, _ = g.acoustic_run(F, F2, nt, dt, app.RHO, app.K, *d)
        torch.cuda.synchronize()
        for st in [(0, 0, 0), (200, 301, 7), (512 - L, 512 - L, 512 - L), (100, 0, 490)]:
            z0, y0, x0 = st
            sub = [F0[0][z0:z0 + L, y0:y0 + L, x0:x0 + L], F0[1][z0:z0 + L, y0:y0 + L, x0:x0 + L + 1],
                   F0[2][z0:z0 + L, y0:y0 + L + 1, x0:x0 + L], F0[3][z0:z0 + L + 1, y0:y0 + L, x0:x0 + L]]
            ref = OA.run(*[s.cpu().numpy() for s in sub], nt, (0, 0, 0), dt, app.RHO, app.K, *d)
            cut = tuple(slice(0 if st[k] == 0 else m, L - (0 if st[k] + L == 512 else m)) for k in range(3))
            got = A[0][0][z0:z0 + L, y0:y0 + L, x0:x0 + L].cpu().numpy()
            assert np.array_equal(ref[0][cut], got[cut]), st
    finally:
        g.finalize()
