"""Second workload: a staggered multi-field step -- linear
acoustics, P at cell centres and Vx, Vy, Vz on the faces (config B:10's field
set) -- on top of libigg.  Host-side glue only: field allocation and
initialisation, a stable dt and the time loop; every step runs in libigg
(igg_acoustic_step: compute_V under @hide_communication with
update_halo!(Vx, Vy, Vz), then compute_P).
"""
from __future__ import annotations

import math

from .igg import Grid

RHO = 1.0
K = 1.0
BW = (16, 4, 4)   # an exchanged axis needs b >= 3, the staggered fields' overlap


def shapes(grid: Grid):
    """Local (z, y, x) shapes of P, Vx, Vy, Vz."""
    nx, ny, nz = grid.n
    return [(nz, ny, nx), (nz, ny, nx + 1), (nz, ny + 1, nx), (nz + 1, ny, nx)]


def spacing(grid: Grid, lengths=(1.0, 1.0, 1.0)) -> tuple:
    """Cell size of the global grid: l / N_g (cell-centred P, faces at both ends)."""
    return tuple(lengths[a] / grid.n_global(a) for a in range(3))


def stable_dt(d, rho: float = RHO, K: float = K) -> float:
    """Half the 3-D leapfrog CFL limit min(d)/(c*sqrt(3)), c = sqrt(K/rho)."""
    return min(d) / math.sqrt(K / rho) / math.sqrt(3.0) / 2.0


def alloc_fields(grid: Grid, device=None):
    import torch
    dev = device or "cuda"
    return [[torch.empty(s, dtype=torch.float64, device=dev) for _ in range(grid.local_ranks)]
            for s in shapes(grid)]


def init_random(grid: Grid, F, seed=None) -> None:
    """Decomposition-independent random fields (synthetic_inputs.acoustic_values of the
    GLOBAL indices this grid's own local->global map gives every local layer)."""
    import torch
    import synthetic_inputs as SI
    seed = SI.SEED_ACOUSTIC if seed is None else seed
    for f, s in enumerate(shapes(grid)):
        sz, sy, sx = s
        Sx, Sy = grid.n_global(0, sx), grid.n_global(1, sy)
        for r in range(grid.local_ranks):
            rank = grid.rank0 + r
            gx = grid.global_indices(rank, 0, sx)
            gy = grid.global_indices(rank, 1, sy)
            gz = grid.global_indices(rank, 2, sz)
            F[f][r].copy_(torch.from_numpy(SI.acoustic_values(f, gx, gy, gz, Sx, Sy, seed)))


def run(grid: Grid, F, nt: int, dt: float, d: tuple, rho: float = RHO, K: float = K, bw=BW, stream=None):
    for _ in range(nt):
        grid.acoustic_step(*F, dt, rho, K, d[0], d[1], d[2], bw=bw, stream=stream)
    return F
