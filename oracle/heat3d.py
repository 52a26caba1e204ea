"""oracle/heat3d.py -- CPU ORACLE for the Fig. 1 heat solver (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.  It never imports the product
package ``paper_2211_15716_b200`` and the product never imports it.

Contents
  * ``build()`` / ``lib()``: compile + load ``heat3d_oracle.c`` (plain C, fp64,
    ``-O2 -ffp-contract=off``, OpenMP over z only).
  * ``spacing``  -- ``dx = lx/(nx_g()-1)``           PAPER.md:63-65 (listing 24-26)
  * ``stable_dt`` -- ``min(dx^2,dy^2,dz^2)/lam/maximum(Ci)/6.1``  PAPER.md:73 (listing 34)
  * ``heat_run`` -- the time loop of PAPER.md:68-80 on the global grid (C).
  * ``heat_run_py`` -- the same loop written in pure Python, for tiny grids
    only (a second, independent transcription used to check the C marshalling).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "heat3d_oracle.c")
_SO = os.path.join(_HERE, "libheat3d_oracle.so")
_lib = None

LITERAL = 0    # paper-literal  /(dx*dx)            (reading 7)
CANONICAL = 1  # *(1.0/(dx*dx)) computed once       (reading 9)


def build(force: bool = False) -> str:
    """Compile the C oracle (no -ffast-math, no FMA contraction: reading 8)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _SO, _SRC]
        subprocess.run(cmd, check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_heat_step.argtypes = [dp, dp, dp, ctypes.c_long, ctypes.c_long, ctypes.c_long,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_int]
        L.oracle_heat_step.restype = None
        L.oracle_heat_run.argtypes = [dp, dp, ctypes.c_long, ctypes.c_long, ctypes.c_long,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.oracle_heat_run.restype = ctypes.c_int
        fp = ctypes.POINTER(ctypes.c_float)
        L.oracle_heat_run_f32.argtypes = [fp, fp, ctypes.c_long, ctypes.c_long, ctypes.c_long,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                          ctypes.c_float, ctypes.c_float, ctypes.c_int]
        L.oracle_heat_run_f32.restype = ctypes.c_int
        L.oracle_max.argtypes = [dp, ctypes.c_long]
        L.oracle_max.restype = ctypes.c_double
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = None
        L.oracle_num_threads.argtypes = []
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def spacing(l: float, N: int, periodic: bool) -> float:
    """dx = lx/(nx_g()-1) on non-periodic axes; dx = lx/N on a
    periodic axis, where N is the period (reading 11); an axis of
    size 1 (1-D/2-D grid) has no spacing: inf, so it drops out of
    stable_dt's minimum (reading 23)."""
    if N == 1 and not periodic:
        return float("inf")
    return l / N if periodic else l / (N - 1)


def stable_dt(dx: float, dy: float, dz: float, lam: float, Ci: np.ndarray) -> float:
    """dt = min(dx^2,dy^2,dz^2)/lam/maximum(Ci)/6.1, Julia's
    left-to-right evaluation; maximum over the WHOLE global Ci (reading 12)."""
    C = np.ascontiguousarray(Ci, dtype=np.float64)
    mx = lib().oracle_max(_ptr(C), C.size)
    return min(dx * dx, dy * dy, dz * dz) / lam / mx / 6.1


def heat_step(T: np.ndarray, Ci: np.ndarray, T2: np.ndarray, periodic, lam, dt, dx, dy, dz,
              mode: int = LITERAL) -> None:
    """One step!(T2,T,Ci,...) of PAPER.md:45-51 in place into T2 (shape (Nz,Ny,Nx))."""
    Nz, Ny, Nx = T.shape
    for a in (T, Ci, T2):
        assert a.shape == (Nz, Ny, Nx)
    lib().oracle_heat_step(_ptr(T2), _ptr(T), _ptr(Ci), Nx, Ny, Nz,
                           int(periodic[0]), int(periodic[1]), int(periodic[2]),
                           lam, dt, dx, dy, dz, mode)


def heat_run(T0: np.ndarray, Ci: np.ndarray, nt: int, periodic, lam, dt, dx, dy, dz,
             mode: int = LITERAL) -> np.ndarray:
    """Fig. 1's time loop on the global grid; returns the final T.
    Arrays are (Nz, Ny, Nx) C-order float64 (x fastest)."""
    T = np.array(T0, dtype=np.float64, order="C", copy=True)
    C = np.ascontiguousarray(Ci, dtype=np.float64)
    Nz, Ny, Nx = T.shape
    assert C.shape == T.shape
    rc = lib().oracle_heat_run(_ptr(T), _ptr(C), Nx, Ny, Nz,
                               int(periodic[0]), int(periodic[1]), int(periodic[2]),
                               lam, dt, dx, dy, dz, nt, mode)
    if rc != 0:
        raise MemoryError("oracle_heat_run: allocation failed")
    return T


def heat_run_f32(T0: np.ndarray, Ci: np.ndarray, nt: int, periodic, lam, dt, dx, dy, dz) -> np.ndarray:
    """The binary32 variant of the time loop (reading 24): inputs rounded to float32 once, every
    operation in binary32, canonical association, r_d = 1/(d*d) computed in float."""
    T = np.array(T0, dtype=np.float32, order="C", copy=True)
    C = np.ascontiguousarray(Ci, dtype=np.float32)
    Nz, Ny, Nx = T.shape
    fp = ctypes.POINTER(ctypes.c_float)
    rc = lib().oracle_heat_run_f32(T.ctypes.data_as(fp), C.ctypes.data_as(fp), Nx, Ny, Nz,
                                   int(periodic[0]), int(periodic[1]), int(periodic[2]),
                                   lam, dt, dx, dy, dz, nt)
    if rc != 0:
        raise MemoryError("oracle_heat_run_f32: allocation failed")
    return T


def heat_run_py(T0, Ci, nt, periodic, lam, dt, dx, dy, dz, mode: int = LITERAL):
    """Pure-Python transcription of the same loop (tiny grids only).  Python
    floats are IEEE binary64 and Python never contracts to FMA."""
    Nz, Ny, Nx = T0.shape
    T = [[[float(T0[z, y, x]) for x in range(Nx)] for y in range(Ny)] for z in range(Nz)]
    C = [[[float(Ci[z, y, x]) for x in range(Nx)] for y in range(Ny)] for z in range(Nz)]
    T2 = [[[T[z][y][x] for x in range(Nx)] for y in range(Ny)] for z in range(Nz)]
    px, py, pz = (bool(p) for p in periodic)
    rng = lambda N, p: range(0, N) if p else range(1, N - 1)
    for _ in range(nt):
        for z in rng(Nz, pz):
            for y in rng(Ny, py):
                for x in rng(Nx, px):
                    c = T[z][y][x]
                    xm = T[z][y][(x - 1) % Nx]; xp = T[z][y][(x + 1) % Nx]
                    ym = T[z][(y - 1) % Ny][x]; yp = T[z][(y + 1) % Ny][x]
                    zm = T[(z - 1) % Nz][y][x]; zp = T[(z + 1) % Nz][y][x]
                    d2x = (xp - c) - (c - xm)
                    d2y = (yp - c) - (c - ym)
                    d2z = (zp - c) - (c - zm)
                    if mode == LITERAL:
                        lap = ((d2x / (dx * dx)) + (d2y / (dy * dy))) + (d2z / (dz * dz))
                    else:
                        lap = ((d2x * (1.0 / (dx * dx))) + (d2y * (1.0 / (dy * dy)))) + (d2z * (1.0 / (dz * dz)))
                    T2[z][y][x] = c + dt * ((lam * C[z][y][x]) * lap)
        T, T2 = T2, T
    return np.array(T, dtype=np.float64)
