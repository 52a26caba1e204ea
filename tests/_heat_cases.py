"""Shared helpers of the GPU parity tests: run the CUDA path through the
binding, run the oracle on the global grid, compare windows."""
import numpy as np

from oracle import grid as OG
from oracle import heat3d as OH
import synthetic_inputs as SI


def oracle_global(N, per, nt, init="random", mode=OH.CANONICAL, seeds=(SI.SEED_T, SI.SEED_CI)):
    """(final T, dt) of the global oracle run; N = (Nx, Ny, Nz)."""
    if init == "random":
        T0, Ci = SI.global_heat_fields(*N, seed_T=seeds[0], seed_C=seeds[1])
    else:
        T0, Ci = SI.paper_heat_fields((N[2], N[1], N[0]))
    d = [OH.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
    dt = OH.stable_dt(*d, 1.0, Ci)
    return OH.heat_run(T0, Ci, nt, per, 1.0, dt, *d, mode), dt


def gpu_run(P, app, n, dims, per, o, nt, bw, init="random", path="nccl", options=None, seeds=None, x_align=1):
    """Fig. 1 on R = prod(dims) virtual ranks of one process; returns
    (list of final local T arrays, dt, grid-allocation counts, launches)."""
    import torch
    nprocs = dims[0] * dims[1] * dims[2]
    g = P.init_global_grid(*n, dims=dims, periods=per, overlaps=o, local_ranks=nprocs, device=0, path=path)
    try:
        g.set_option(P.OPT_X_ALIGN, x_align)    # 1: the exact widths, so small grids still split
        for k, v in (options or {}).items():
            g.set_option(k, v)
        T, T2, Ci = app.alloc_fields(g)
        if init == "random":
            if seeds:
                app.init_random(g, T, T2, Ci, *seeds)
            else:
                app.init_random(g, T, T2, Ci)
        else:
            app.init_paper(g, T, T2, Ci)
        d = app.spacing(g)
        dt = app.stable_dt(g, Ci, *d)
        allocs = []
        for it in range(nt):
            g.heat_step(T2, T, Ci, 1.0, dt, *d, bw=bw)
            T, T2 = T2, T
            if it in (0, nt - 1):
                torch.cuda.synchronize()
                allocs.append(g.buffer_allocs())
        torch.cuda.synchronize()
        g.check()
        out = [t.cpu().numpy() for t in T]
        return out, dt, allocs, g.kernel_launches()
    finally:
        g.finalize()


def assert_windows(local, ref, dims, n, o, per, exact=True, rtol=1e-12):
    for r, A in enumerate(local):
        c = OG.coords_of_rank(r, dims)
        W = OG.window(ref, c, dims, n, o, per, n)
        if exact:
            if not np.array_equal(A, W):
                bad = np.argwhere(A != W)
                raise AssertionError(f"rank {r}: {len(bad)} cells differ, first {bad[:5].tolist()}")
        else:
            err = np.max(np.abs(A - W) / np.abs(W))
            assert err <= rtol, (r, err)
