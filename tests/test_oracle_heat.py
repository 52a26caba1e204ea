"""Pins for oracle/heat3d (CPU only).  Each test checks the oracle against
something the paper or the mathematics fixes, not against a retyped copy of
its own formula:

  * Fig. 1's initial condition is an exact fixed point
  * integer-linear profiles are exact steady states
  * the hand-evaluated hot cell                           (golden)
  * dt of the paper setup                                 (golden)
  * closed-form decay of discrete Fourier modes, Dirichlet and periodic,
    anisotropic spacing and non-cubic grids (an exact eigenvector of the
    7-point Laplacian: catches dropped terms, sign errors, swapped axes/spacings)
  * conservation of sum(T/Ci) on an all-periodic grid with random Ci
    (catches a Ci read at the wrong cell or a missing Ci)
  * Dirichlet boundary unchanged, maximum principle
  * literal vs canonical arithmetic within 1e-15           (reading 9)
"""
import json
import math
import os
import struct

import numpy as np
import pytest

from oracle import heat3d as H
import synthetic_inputs as SI

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("mode", [H.LITERAL, H.CANONICAL])
def test_fixed_point_paper_init(mode):
    shape = (16, 20, 24)
    T, Ci = SI.paper_heat_fields(shape)
    dx = H.spacing(1.0, 24, False); dy = H.spacing(1.0, 20, False); dz = H.spacing(1.0, 16, False)
    dt = H.stable_dt(dx, dy, dz, 1.0, Ci)
    out = H.heat_run(T, Ci, 100, (0, 0, 0), 1.0, dt, dx, dy, dz, mode)
    assert np.array_equal(out, T)


def test_integer_linear_profile_is_steady():
    Nz, Ny, Nx = 7, 8, 9
    z, y, x = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    T = (x + 2 * y + 3 * z).astype(np.float64)
    Ci = SI.random_field(T.shape, 5) * 0.25 + 0.5
    out = H.heat_run(T, Ci, 10, (0, 0, 0), 1.0, 0.01, 0.3, 0.5, 0.7, H.LITERAL)
    assert np.array_equal(out, T)


@pytest.mark.parametrize("mode", [H.LITERAL, H.CANONICAL])
def test_hot_cell_worked_example(mode):
    g = GOLD["heat_hot_cell"]
    T = np.zeros((3, 3, 3)); T[1, 1, 1] = g["center"]
    Ci = np.full((3, 3, 3), g["Ci"])
    out = H.heat_run(T, Ci, 1, (0, 0, 0), g["lam"], g["dt"], g["dx"], g["dx"], g["dx"], mode)
    v = out[1, 1, 1]
    assert struct.pack(">d", v).hex() == g["T2_center_hex"]
    assert abs(v - g["T2_center_real"]) <= 2 * np.spacing(0.4)
    mask = np.ones((3, 3, 3), bool); mask[1, 1, 1] = False
    assert np.all(out[mask] == 0.0)       # boundary layers untouched


def test_dt_paper_setup():
    g = GOLD["dt_512"]
    dx = H.spacing(g["lx"], g["n"], False)
    Ci = np.full((4, 4, 4), 1.0 / g["c0"])
    dt = H.stable_dt(dx, dx, dx, g["lam"], Ci)
    assert abs(dt - g["dt_approx"]) / g["dt_approx"] < g["rel_tol"]
    u = GOLD["dt_unit"]
    assert abs(H.stable_dt(1.0, 1.0, 1.0, 1.0, np.ones((2, 2, 2))) - u["dt"]) <= 1e-16


def test_dt_uses_global_max_and_min_spacing():
    Ci = np.full((3, 4, 5), 0.5); Ci[2, 3, 4] = 0.8
    dt = H.stable_dt(0.3, 0.1, 0.2, 2.0, Ci)
    assert dt == pytest.approx(0.01 / 2.0 / 0.8 / 6.1, rel=1e-15)


def _dirichlet_mode(N, L, k):
    """1.7 + prod_d sin(k_d*pi*g_d/(N_d-1)) on (Nz,Ny,Nx); zero on the boundary."""
    Nx, Ny, Nz = N
    sx = np.sin(k[0] * np.pi * np.arange(Nx) / (Nx - 1))
    sy = np.sin(k[1] * np.pi * np.arange(Ny) / (Ny - 1))
    sz = np.sin(k[2] * np.pi * np.arange(Nz) / (Nz - 1))
    sx[[0, -1]] = 0.0; sy[[0, -1]] = 0.0; sz[[0, -1]] = 0.0
    return sz[:, None, None] * sy[None, :, None] * sx[None, None, :]


@pytest.mark.parametrize("mode", [H.LITERAL, H.CANONICAL])
def test_fourier_mode_dirichlet(mode):
    N = (14, 12, 10); L = (1.0, 0.7, 1.3); k = (1, 2, 3); lam = 1.3; c = 0.45; nt = 100
    d = [H.spacing(L[i], N[i], False) for i in range(3)]
    M = _dirichlet_mode(N, L, k)
    A = 0.25
    T0 = 1.7 + A * M
    Ci = np.full(T0.shape, c)
    dt = H.stable_dt(d[0], d[1], d[2], lam, Ci)
    out = H.heat_run(T0, Ci, nt, (0, 0, 0), lam, dt, d[0], d[1], d[2], mode)
    Gf = 1.0 - dt * lam * c * sum(4.0 / d[i] ** 2 * math.sin(k[i] * math.pi / (2 * (N[i] - 1))) ** 2
                                  for i in range(3))
    expect = 1.7 + A * Gf ** nt * M
    assert Gf ** nt < 0.9                  # the mode has really decayed
    assert np.max(np.abs(out - expect)) <= 1e-14


def test_fourier_mode_periodic_and_mixed():
    # x periodic (cos mode, dx = lx/N), y Dirichlet (sin), z periodic
    N = (12, 9, 10); L = (1.0, 0.8, 1.1); lam = 1.0; c = 0.6; nt = 60; A = 0.3
    per = (1, 0, 1)
    d = [H.spacing(L[i], N[i], bool(per[i])) for i in range(3)]
    kx, ky, kz = 2, 1, 1
    cx = np.cos(2 * np.pi * kx * np.arange(N[0]) / N[0])
    sy = np.sin(ky * np.pi * np.arange(N[1]) / (N[1] - 1)); sy[[0, -1]] = 0.0
    cz = np.cos(2 * np.pi * kz * np.arange(N[2]) / N[2])
    M = cz[:, None, None] * sy[None, :, None] * cx[None, None, :]
    T0 = 1.7 + A * M
    Ci = np.full(T0.shape, c)
    dt = H.stable_dt(d[0], d[1], d[2], lam, Ci)
    out = H.heat_run(T0, Ci, nt, per, lam, dt, d[0], d[1], d[2], H.LITERAL)
    Gf = 1.0 - dt * lam * c * (4 / d[0] ** 2 * math.sin(math.pi * kx / N[0]) ** 2
                               + 4 / d[1] ** 2 * math.sin(ky * math.pi / (2 * (N[1] - 1))) ** 2
                               + 4 / d[2] ** 2 * math.sin(math.pi * kz / N[2]) ** 2)
    expect = 1.7 + A * Gf ** nt * M
    assert Gf ** nt < 0.9
    assert np.max(np.abs(out - expect)) <= 1e-14


def test_conservation_all_periodic_random_ci():
    N = (10, 9, 8)
    T0, Ci = SI.global_heat_fields(*N)
    d = [H.spacing(1.0, n, True) for n in N]
    dt = H.stable_dt(*d, 1.0, Ci)
    before = math.fsum((T0 / Ci).ravel())
    out = H.heat_run(T0, Ci, 50, (1, 1, 1), 1.0, dt, *d, H.LITERAL)
    after = math.fsum((out / Ci).ravel())
    assert not np.array_equal(out, T0)
    assert abs(after - before) / abs(before) <= 1e-13
    # the same data WITHOUT the 1/Ci weighting is not conserved (Ci really enters per cell)
    assert abs(math.fsum(out.ravel()) - math.fsum(T0.ravel())) / math.fsum(T0.ravel()) > 1e-9


def test_dirichlet_boundary_and_maximum_principle():
    N = (11, 10, 9)
    T0, Ci = SI.global_heat_fields(*N)
    d = [H.spacing(1.0, n, False) for n in N]
    dt = H.stable_dt(*d, 1.0, Ci)
    out = H.heat_run(T0, Ci, 40, (0, 0, 0), 1.0, dt, *d, H.LITERAL)
    inner = (slice(1, -1),) * 3
    b = np.ones(out.shape, bool); b[inner] = False
    assert np.array_equal(out[b], T0[b])
    assert out.min() >= T0.min() and out.max() <= T0.max()


def test_literal_vs_canonical_close():
    N = (18, 17, 16)
    T0, Ci = SI.global_heat_fields(*N)
    d = [H.spacing(1.0, n, False) for n in N]
    dt = H.stable_dt(*d, 1.0, Ci)
    a = H.heat_run(T0, Ci, 100, (0, 0, 0), 1.0, dt, *d, H.LITERAL)
    b = H.heat_run(T0, Ci, 100, (0, 0, 0), 1.0, dt, *d, H.CANONICAL)
    assert np.max(np.abs(a - b) / np.abs(a)) <= 1e-15


@pytest.mark.parametrize("per", [(0, 0, 0), (1, 0, 1), (1, 1, 1)])
@pytest.mark.parametrize("mode", [H.LITERAL, H.CANONICAL])
def test_c_oracle_matches_pure_python_transcription(per, mode):
    # not a pin of the formula (both transcribe it): checks the C marshalling,
    # the index order and the periodic wrap of the C implementation.
    N = (6, 5, 4)
    T0, Ci = SI.global_heat_fields(*N)
    d = [H.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
    dt = H.stable_dt(*d, 1.0, Ci)
    a = H.heat_run(T0, Ci, 3, per, 1.0, dt, *d, mode)
    b = H.heat_run_py(T0, Ci, 3, per, 1.0, dt, *d, mode)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("N,k,per", [((14, 12, 1), (1, 2, 0), (0, 0, 0)),      # 2-D (size-1 z)
                                     ((20, 1, 1), (3, 0, 0), (0, 0, 0)),       # 1-D
                                     ((12, 1, 9), (2, 0, 1), (1, 0, 0)),       # 2-D x-z, x periodic
                                     ((1, 16, 11), (0, 2, 1), (0, 0, 0))])     # 2-D y-z
@pytest.mark.parametrize("mode", [H.LITERAL, H.CANONICAL])
def test_fourier_mode_low_dimensional(N, k, per, mode):
    """1-D/2-D grids as size-1 axes (reading 23): the discrete mode decays with only the extended
    axes' factors; a size-1 axis contributes no term and its one layer is updated."""
    L = (1.0, 0.8, 1.2); lam = 1.1; c = 0.5; nt = 80; A = 0.3
    d = [H.spacing(L[i], N[i], bool(per[i])) for i in range(3)]
    prof = []
    for i in range(3):
        g = np.arange(N[i])
        if N[i] == 1:
            prof.append(np.ones(1))
        elif per[i]:
            prof.append(np.cos(2 * np.pi * k[i] * g / N[i]))
        else:
            s = np.sin(k[i] * np.pi * g / (N[i] - 1)); s[[0, -1]] = 0.0
            prof.append(s)
    M = prof[2][:, None, None] * prof[1][None, :, None] * prof[0][None, None, :]
    T0 = 1.7 + A * M
    Ci = np.full(T0.shape, c)
    dt = H.stable_dt(d[0], d[1], d[2], lam, Ci)
    assert dt == min(d[i] ** 2 for i in range(3) if N[i] > 1) / lam / c / 6.1
    out = H.heat_run(T0, Ci, nt, per, lam, dt, d[0], d[1], d[2], mode)
    lamk = 0.0
    for i in range(3):
        if N[i] == 1:
            continue
        arg = math.pi * k[i] / N[i] if per[i] else k[i] * math.pi / (2 * (N[i] - 1))
        lamk += 4.0 / d[i] ** 2 * math.sin(arg) ** 2
    Gf = 1.0 - dt * lam * c * lamk
    expect = 1.7 + A * Gf ** nt * M
    assert Gf ** nt < 0.9
    assert np.max(np.abs(out - expect)) <= 1e-14


def test_size1_axis_equals_lower_dimensional_grid():
    """A 3-D grid with a size-1 z equals the same 2-D grid embedded with nz = 3 whose z neighbours
    equal the middle layer (d2z = 0 exactly): every cell, bit for bit, in canonical mode."""
    rng = np.random.default_rng(3)
    T2d = 1.7 + rng.random((1, 9, 11)); C2d = 0.5 + 0.2 * rng.random((1, 9, 11))
    d = (0.1, 0.13, float("inf"))
    dt = H.stable_dt(*d, 1.0, C2d)
    a = H.heat_run(T2d, C2d, 5, (0, 0, 0), 1.0, dt, *d, H.CANONICAL)
    T3 = np.repeat(T2d, 3, axis=0); C3 = np.repeat(C2d, 3, axis=0)
    # z periodic with three equal layers: d2z = (c - c) - (c - c) = 0 exactly, x/y terms identical
    b = H.heat_run(T3, C3, 5, (0, 0, 1), 1.0, dt, d[0], d[1], 1.0, H.CANONICAL)
    # the 3-D sum adds (d2z*rdz2) = +0.0 last: x + y + 0.0 == x + y exactly
    assert np.array_equal(a[0], b[1])


# ---------------------------------------------------------------- binary32 variant (reading 24)
def test_f32_fixed_point_exact():
    T = np.full((6, 7, 8), 1.7, dtype=np.float32); Ci = np.full(T.shape, 0.5, dtype=np.float32)
    out = H.heat_run_f32(T, Ci, 20, (0, 1, 0), 1.0, 1e-3, 0.1, 0.1, 0.1)
    assert out.dtype == np.float32 and np.array_equal(out, T)


@pytest.mark.parametrize("per", [(0, 0, 0), (1, 0, 1)])
def test_f32_tracks_f64_within_float_precision(per):
    N = (12, 10, 9)
    T0, Ci = SI_fields(N)
    d = [H.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
    dt = H.stable_dt(*d, 1.0, Ci)
    a = H.heat_run(T0, Ci, 30, per, 1.0, dt, *d, H.CANONICAL)
    b = H.heat_run_f32(T0, Ci, 30, per, 1.0, dt, *d)
    rel = np.max(np.abs(b.astype(np.float64) - a) / np.abs(a))
    assert 1e-9 < rel < 2e-6          # really binary32, and as accurate as binary32 allows


def test_f32_fourier_mode_decay():
    N = (14, 12, 10); L = (1.0, 0.7, 1.3); k = (1, 2, 1); lam = 1.3; c = 0.45; nt = 60; A = 0.25
    d = [H.spacing(L[i], N[i], False) for i in range(3)]
    M = _dirichlet_mode(N, L, k)
    T0 = 1.7 + A * M
    Ci = np.full(T0.shape, c)
    dt = H.stable_dt(d[0], d[1], d[2], lam, Ci)
    out = H.heat_run_f32(T0, Ci, nt, (0, 0, 0), lam, dt, *d)
    Gf = 1.0 - dt * lam * c * sum(4.0 / d[i] ** 2 * math.sin(k[i] * math.pi / (2 * (N[i] - 1))) ** 2
                                  for i in range(3))
    expect = 1.7 + A * Gf ** nt * M
    assert Gf ** nt < 0.9
    assert np.max(np.abs(out - expect)) <= 2e-5


def SI_fields(N):
    import synthetic_inputs as SI
    return SI.global_heat_fields(*N)


@pytest.mark.parametrize("lx,k", [(0.7, 1), (2.3, 2)])
def test_periodic_spacing_continuum_decay(lx, k):
    """Reading 11 (dx = lx/n_g on a periodic axis: the period is the domain length lx) pinned by the
    physics, not by the oracle's own spacing: a periodic mode of physical wavelength lx/k -- k whole
    periods over the n_g cells -- decays at the continuum rate lam*c*(2 pi k/lx)^2 of dT/dt =
    lam*Ci*Laplacian(T) (Ci = c) up to the O((pi k/N)^2) + O(rate dt) discretisation
    error (~0.2 % here).  Reading dx = lx/(n_g-1) instead misses the rate by 2/N (3 %)."""
    N = (64, 4, 4); lam, c, A = 1.3, 0.45, 0.2
    L = (lx, lx, lx)
    d = [H.spacing(L[i], N[i], True) for i in range(3)]
    g = np.arange(N[0])
    M = np.broadcast_to(np.cos(2.0 * math.pi * k * g / N[0])[None, None, :], (N[2], N[1], N[0]))
    T0 = np.ascontiguousarray(1.7 + A * M)
    Ci = np.full(T0.shape, c)
    dt = H.stable_dt(d[0], d[1], d[2], lam, Ci)
    rate = lam * c * (2.0 * math.pi * k / lx) ** 2          # continuum decay rate, 1/time
    nt = int(round(1.0 / (rate * dt)))                        # about one e-folding of physical time
    out = H.heat_run(T0, Ci, nt, (1, 1, 1), lam, dt, d[0], d[1], d[2], H.LITERAL)
    amp = float(np.sum((out[0, 0, :] - 1.7) * np.cos(2.0 * math.pi * k * g / N[0]))) * 2.0 / N[0]
    measured = -math.log(amp / A) / (nt * dt)
    assert abs(measured / rate - 1.0) < 5e-3, (measured, rate)
