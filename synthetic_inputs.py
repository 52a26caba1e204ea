"""synthetic_inputs.py -- seeded synthetic inputs shared by the oracle side and
the CUDA side of every test and of bench.py.

It holds none of the method's arithmetic: no stencil, no halo geometry, no
index maps.  A value is a pure function of (seed, global linear index), so a
rank can generate exactly its part of a global field given global indices it
computed itself, and the oracle can generate the whole global field.

Recipe:
  * paper inputs:   T = 1.7, Ci = 1/c0 = 0.5   (a fixed point)
  * random parity inputs:            T  = 1.7 + u(seed_T, g)
                                     Ci = 0.5*(1 + 0.5*u(seed_C, g))
    with u(seed, g) = (splitmix64(seed XOR g) >> 11) * 2^-53 in [0,1), g the
    global linear index x + Nx*(y + Ny*z).  Values stay in [1.7, 2.7) and
    [0.5, 0.75), so no subnormals appear and relative errors are well defined.
"""
from __future__ import annotations

import numpy as np

SEED_T = 2211
SEED_CI = 15716

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vigna's splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + _M1
    z = (z ^ (z >> np.uint64(30))) * _M2
    z = (z ^ (z >> np.uint64(27))) * _M3
    return z ^ (z >> np.uint64(31))


def uniform01(seed: int, gidx: np.ndarray) -> np.ndarray:
    """u in [0,1) with 53 random bits, a pure function of (seed, index)."""
    g = np.asarray(gidx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        r = splitmix64(np.uint64(seed) ^ g)
    return (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def linear_index(gx: np.ndarray, gy: np.ndarray, gz: np.ndarray, Nx: int, Ny: int) -> np.ndarray:
    """Broadcast (gz[:,None,None], gy[None,:,None], gx[None,None,:]) to the
    (z,y,x) array of global linear indices x + Nx*(y + Ny*z)."""
    gx = np.asarray(gx, dtype=np.uint64)[None, None, :]
    gy = np.asarray(gy, dtype=np.uint64)[None, :, None]
    gz = np.asarray(gz, dtype=np.uint64)[:, None, None]
    return gx + np.uint64(Nx) * (gy + np.uint64(Ny) * gz)


def heat_T(gidx: np.ndarray, seed: int = SEED_T) -> np.ndarray:
    return 1.7 + uniform01(seed, gidx)


def heat_Ci(gidx: np.ndarray, seed: int = SEED_CI) -> np.ndarray:
    return 0.5 * (1.0 + 0.5 * uniform01(seed, gidx))


def global_heat_fields(Nx: int, Ny: int, Nz: int, seed_T: int = SEED_T, seed_C: int = SEED_CI):
    """(T, Ci) over a whole global grid, arrays of shape (Nz, Ny, Nx)."""
    g = linear_index(np.arange(Nx), np.arange(Ny), np.arange(Nz), Nx, Ny)
    return heat_T(g, seed_T), heat_Ci(g, seed_C)


def paper_heat_fields(shape):
    """T = ones*1.7, Ci = ones/c0 with c0 = 2.0."""
    c0 = 2.0
    return np.full(shape, 1.7), np.full(shape, 1.0 / c0)


def random_field(shape, seed: int) -> np.ndarray:
    """An arbitrary random float64 field (e.g. per-rank halo-test data)."""
    n = int(np.prod(shape))
    return uniform01(seed, np.arange(n, dtype=np.uint64)).reshape(shape) * 2.0 - 1.0


SEED_ACOUSTIC = 102


def acoustic_values(f: int, gx, gy, gz, Sx: int, Sy: int, seed: int = SEED_ACOUSTIC) -> np.ndarray:
    """Field f (0 = P, 1..3 = Vx, Vy, Vz) at global indices (gz, gy, gx) of a field whose
    global x/y sizes are Sx, Sy: P = 1 + u, V = 0.1*(2u - 1), u from the field's own seed
    and global linear index."""
    u = uniform01(seed * 8 + f, linear_index(gx, gy, gz, Sx, Sy))
    return 1.0 + u if f == 0 else 0.1 * (2.0 * u - 1.0)


def global_acoustic_fields(shapes, seed: int = SEED_ACOUSTIC):
    """Second workload: random global (P, Vx, Vy, Vz) of the given
    (z, y, x) shapes (acoustic_values over every global index)."""
    return [acoustic_values(f, np.arange(sx), np.arange(sy), np.arange(sz), sx, sy, seed)
            for f, (sz, sy, sx) in enumerate(shapes)]
