"""The paper's 3-D heat diffusion xPU solver (Fig. 1) on top of
libigg.  Host-side glue only: spacing, dt, field allocation/initialisation
and the time loop; every step runs in libigg.

Constants: lam = 1, c0 = 2, lx = ly = lz = 1, nx = ny = nz =
512, nt = 100; hide_communication widths (16, 2, 2).
"""
from __future__ import annotations

import numpy as np

from .igg import Grid

LAM = 1.0
C0 = 2.0
LX = LY = LZ = 1.0
NT = 100
BW = (16, 2, 2)


def spacing(grid: Grid, lengths=(LX, LY, LZ)) -> tuple:
    """dx = lx/(nx_g()-1); lx/nx_g() on a periodic axis
    (reading 11)."""
    out = []
    for a in range(3):
        N = grid.n_global(a)
        if N == 1 and not grid.periods[a]:   # a size-1 axis (1-D/2-D grid): no spacing (reading 23)
            out.append(float("inf"))
        else:
            out.append(lengths[a] / N if grid.periods[a] else lengths[a] / (N - 1))
    return tuple(out)


def stable_dt(grid: Grid, Ci, dx: float, dy: float, dz: float, lam: float = LAM) -> float:
    """dt = min(dx^2,dy^2,dz^2)/lam/maximum(Ci)/6.1 with the
    maximum over every rank (libigg reduction kernel + NCCL max)."""
    mx = grid.field_global_max(Ci)
    return min(dx * dx, dy * dy, dz * dz) / lam / mx / 6.1


def alloc_fields(grid: Grid, device=None, dtype=None):
    """(T, T2, Ci) per local rank, canonical local shape (nz, ny, nx); float64 unless dtype is given
    (torch.float32: the binary32 variant)."""
    import torch
    nx, ny, nz = grid.n
    dt_ = dtype or torch.float64
    mk = lambda: [torch.empty((nz, ny, nx), dtype=dt_, device=device or "cuda")
                  for _ in range(grid.local_ranks)]
    return mk(), mk(), mk()


def init_paper(grid: Grid, T, T2, Ci) -> None:
    """T = 1.7, T2 = copy(T), Ci = 1/c0."""
    for r in range(grid.local_ranks):
        T[r].fill_(1.7)
        T2[r].copy_(T[r])
        Ci[r].fill_(1.0 / C0)


def init_random(grid: Grid, T, T2, Ci, seed_T=None, seed_C=None) -> None:
    """Decomposition-independent random fields (DESIGN.md input recipe):
    values are a function of the GLOBAL linear index, computed from this
    grid's own local->global map."""
    import torch
    import synthetic_inputs as SI
    seed_T = SI.SEED_T if seed_T is None else seed_T
    seed_C = SI.SEED_CI if seed_C is None else seed_C
    nx, ny, nz = grid.n
    Nx, Ny = grid.nx_g(), grid.ny_g()
    for r in range(grid.local_ranks):
        rank = grid.rank0 + r
        gx = grid.global_indices(rank, 0, nx)
        gy = grid.global_indices(rank, 1, ny)
        gz = grid.global_indices(rank, 2, nz)
        g = SI.linear_index(gx, gy, gz, Nx, Ny)
        T[r].copy_(torch.from_numpy(SI.heat_T(g, seed_T)))     # (rounded once if float32)
        Ci[r].copy_(torch.from_numpy(SI.heat_Ci(g, seed_C)))
        T2[r].copy_(T[r])


def run(grid: Grid, T, T2, Ci, nt: int, dt: float, d: tuple, lam: float = LAM, bw=BW, stream=None,
        per_step: bool = False):
    """The time loop; returns the lists (T, T2) after the swaps.  Default: one
    igg_heat_run call (consecutive steps pipelined on the fused path); per_step: nt igg_heat_step calls."""
    if not per_step:
        return grid.heat_run(T, T2, Ci, lam, dt, d[0], d[1], d[2], nt, bw=bw, stream=stream)
    for _ in range(nt):
        grid.heat_step(T2, T, Ci, lam, dt, d[0], d[1], d[2], bw=bw, stream=stream)
        T, T2 = T2, T
    return T, T2
