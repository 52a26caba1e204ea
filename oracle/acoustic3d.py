"""oracle/acoustic3d.py -- CPU ORACLE for the second workload (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.  It never imports the product
package ``paper_2211_15716_b200`` and the product never imports it.

What it computes.  SURVEY.md 8(f) f1 asks for a staggered multi-field step (P,
Vx, Vy, Vz) using the config-B:10 halos, "the paper's real-world use is
multi-field staggered solvers".  The paper prints no
formula for such a solver, so the step is the textbook linear-acoustics
leapfrog on a staggered (MAC) grid, in the @inn/@all/@d_xi/@d_xa form of the
paper's own stencil notation:

    dV/dt = -(1/rho) grad P,   dP/dt = -K div V

  * P  at cell centres, shape (Nz, Ny, Nx);  Vx at x faces, (Nz, Ny, Nx+1);
    Vy at y faces, (Nz, Ny+1, Nx);  Vz at z faces, (Nz+1, Ny, Nx).  Vx[.,.,i]
    sits between P[.,.,i-1] and P[.,.,i].  On a periodic axis every field has
    the period's number of layers and indices wrap.
  * compute_V (@inn(Vd) = @inn(Vd) - cV_d * @d_di(P)):
        Vx[k,j,i] = Vx[k,j,i] - cVx * (P[k,j,i] - P[k,j,i-1])
    for i in [1, Nx) and j, k inner ([1, N-1)) on non-periodic axes, every layer
    on periodic ones; likewise Vy, Vz.
  * update_halo!(Vx, Vy, Vz)  (distributed runs only; the global run has none).
  * compute_P (@all(P) = @all(P) - cP * (@d_xa(Vx)*rx + @d_ya(Vy)*ry + @d_za(Vz)*rz)):
        P[k,j,i] = P[k,j,i] - cP * ((((Vx[k,j,i+1]-Vx[k,j,i])*rx) + ((Vy[k,j+1,i]-Vy[k,j,i])*ry))
                                    + ((Vz[k+1,j,i]-Vz[k,j,i])*rz))
    for every cell.
  * Coefficients, computed once from the inputs (reading A2):
        cV_d = (dt / rho) / d_d,   cP = dt * K,   r_d = 1.0 / d_d.
  * binary64, every operation rounded on its own (numpy never contracts to FMA).

Pins (tests/test_oracle_acoustic.py): the coefficients (reading A2) from the
physics alone -- a travelling periodic mode built from (rho, K, dt, d) only,
with the leapfrog dispersion relation sin^2(phi/2) = (K/rho) dt^2 sum s_d^2/d_d^2
and the wave impedance |V|/|P| = 1/sqrt(rho K), is reproduced step by step, and
the measured sound speed of a standing wave tends to sqrt(K/rho); the exact
evolution of one periodic Fourier mode (the 4x4 per-mode amplification matrix
raised to the n-th power with numpy), conservation of sum(P) with periodic
boundaries, exact mirror symmetry, the fixed point, a second pure-Python
transcription, and decomposition independence through oracle.halo.
"""
from __future__ import annotations

import numpy as np


def coefficients(dt: float, rho: float, K: float, dx: float, dy: float, dz: float) -> dict:
    """Reading A2: cV_d = (dt/rho)/d_d, cP = dt*K, r_d = 1.0/d_d."""
    a = dt / rho
    return dict(cV=(a / dx, a / dy, a / dz), cP=dt * K, r=(1.0 / dx, 1.0 / dy, 1.0 / dz))


def field_shapes(N, periodic):
    """Global shapes (z, y, x) of P, Vx, Vy, Vz for global cell counts N = (Nx, Ny, Nz)."""
    Nx, Ny, Nz = N
    sx = Nx if periodic[0] else Nx + 1
    sy = Ny if periodic[1] else Ny + 1
    sz = Nz if periodic[2] else Nz + 1
    return [(Nz, Ny, Nx), (Nz, Ny, sx), (Nz, sy, Nx), (sz, Ny, Nx)]


def _upd_range(N, periodic, diff_axis: bool):
    """Indices updated along one axis: the differenced axis of a component covers
    [1, N) (the faces between two cells), another axis the inner layers [1, N-1);
    a periodic axis every layer."""
    if periodic:
        return np.arange(N)
    return np.arange(1, N) if diff_axis else np.arange(1, N - 1)


def compute_V(P, Vx, Vy, Vz, periodic, cV) -> None:
    """compute_V! in place (module docstring).  Reads only P, so the three
    components are independent."""
    Nz, Ny, Nx = P.shape
    N = (Nx, Ny, Nz)
    for d, V in enumerate((Vx, Vy, Vz)):
        rng = [_upd_range(N[a], periodic[a], a == d) for a in range(3)]   # x, y, z
        iz, iy, ix = np.ix_(rng[2], rng[1], rng[0])                       # (z, y, x) order
        lo = [iz, iy, ix]
        # the lower cell: index - 1 along axis d (wrapping on a periodic axis)
        axis_zyx = 2 - d
        lo[axis_zyx] = (lo[axis_zyx] - 1) % N[d]
        dP = P[iz, iy, ix] - P[lo[0], lo[1], lo[2]]
        V[iz, iy, ix] = V[iz, iy, ix] - cV[d] * dP


def compute_P(P, Vx, Vy, Vz, periodic, cP, r) -> None:
    """compute_P! in place on every cell (module docstring)."""
    Nz, Ny, Nx = P.shape
    i = np.arange(Nx)
    j = np.arange(Ny)
    k = np.arange(Nz)
    ip = (i + 1) % Vx.shape[2]          # periodic: Vx has Nx layers and wraps; else Nx+1 layers
    jp = (j + 1) % Vy.shape[1]
    kp = (k + 1) % Vz.shape[0]
    dVx = Vx[:, :, ip] - Vx[:, :, i]
    dVy = Vy[:, jp, :] - Vy[:, j, :]
    dVz = Vz[kp, :, :] - Vz[k, :, :]
    div = ((dVx * r[0]) + (dVy * r[1])) + (dVz * r[2])
    P[...] = P - cP * div


def step(P, Vx, Vy, Vz, periodic, co) -> None:
    """One leapfrog step on the global grid: compute_V then compute_P."""
    compute_V(P, Vx, Vy, Vz, periodic, co["cV"])
    compute_P(P, Vx, Vy, Vz, periodic, co["cP"], co["r"])


def run(P0, Vx0, Vy0, Vz0, nt, periodic, dt, rho, K, dx, dy, dz):
    """nt steps from copies of the inputs; returns (P, Vx, Vy, Vz)."""
    co = coefficients(dt, rho, K, dx, dy, dz)
    F = [np.array(a, dtype=np.float64, order="C", copy=True) for a in (P0, Vx0, Vy0, Vz0)]
    for _ in range(nt):
        step(*F, periodic, co)
    return tuple(F)


def run_py(P0, Vx0, Vy0, Vz0, nt, periodic, dt, rho, K, dx, dy, dz):
    """The same loop as plain Python scalar loops (tiny grids only): a second,
    independent transcription used to check the vectorised indexing."""
    co = coefficients(dt, rho, K, dx, dy, dz)
    P, Vx, Vy, Vz = (np.array(a, dtype=np.float64, copy=True) for a in (P0, Vx0, Vy0, Vz0))
    Nz, Ny, Nx = P.shape
    px, py, pz = (bool(p) for p in periodic)

    def rng(N, per, diff):
        return range(N) if per else (range(1, N) if diff else range(1, N - 1))

    for _ in range(nt):
        for z in rng(Nz, pz, False):
            for y in rng(Ny, py, False):
                for x in rng(Nx, px, True):
                    Vx[z, y, x] = float(Vx[z, y, x]) - co["cV"][0] * (float(P[z, y, x]) - float(P[z, y, (x - 1) % Nx]))
        for z in rng(Nz, pz, False):
            for y in rng(Ny, py, True):
                for x in rng(Nx, px, False):
                    Vy[z, y, x] = float(Vy[z, y, x]) - co["cV"][1] * (float(P[z, y, x]) - float(P[z, (y - 1) % Ny, x]))
        for z in rng(Nz, pz, True):
            for y in rng(Ny, py, False):
                for x in rng(Nx, px, False):
                    Vz[z, y, x] = float(Vz[z, y, x]) - co["cV"][2] * (float(P[z, y, x]) - float(P[(z - 1) % Nz, y, x]))
        for z in range(Nz):
            for y in range(Ny):
                for x in range(Nx):
                    dvx = float(Vx[z, y, (x + 1) % Vx.shape[2]]) - float(Vx[z, y, x])
                    dvy = float(Vy[z, (y + 1) % Vy.shape[1], x]) - float(Vy[z, y, x])
                    dvz = float(Vz[(z + 1) % Vz.shape[0], y, x]) - float(Vz[z, y, x])
                    div = ((dvx * co["r"][0]) + (dvy * co["r"][1])) + (dvz * co["r"][2])
                    P[z, y, x] = float(P[z, y, x]) - co["cP"] * div
    return P, Vx, Vy, Vz


def local_V(P, Vx, Vy, Vz, co) -> None:
    """compute_V on ONE rank's local arrays (sizes n, staggered n+1) with local
    non-periodic semantics: the layers a rank computes itself; its halos come from
    update_halo!(Vx, Vy, Vz) afterwards (the library's kernels do the same)."""
    compute_V(P, Vx, Vy, Vz, (False, False, False), co["cV"])


def local_P(P, Vx, Vy, Vz, co) -> None:
    """compute_P on every cell of ONE rank's local P, halo cells included (@all),
    from the exchanged velocities."""
    compute_P(P, Vx, Vy, Vz, (False, False, False), co["cP"], co["r"])
