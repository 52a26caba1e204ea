"""Pins of the acoustic (second-workload) oracle against things other than itself
(oracle/acoustic3d.py; readings A1-A3).

* the exact evolution of one periodic Fourier mode: the staggered stencil maps
  the mode's complex amplitudes (p, vx, vy, vz) by a 4x4 matrix derived on paper
  (below); numpy.linalg.matrix_power gives n steps;
* sum(P) is conserved with periodic boundaries (the divergence telescopes);
* a mirror-symmetric state stays exactly symmetric (P even, the mirrored
  velocity odd), bit for bit -- a wrong staggering offset breaks it;
* a constant P with V = 0 is a fixed point;
* a second, scalar pure-Python transcription agrees bit for bit;
* decomposition independence: {local compute_V; update_halo!(Vx,Vy,Vz); local
  compute_P} on every rank equals the windows of the global run, staggered halos
  from oracle.halo (config B:10's field set).
"""
import math
import random

import numpy as np
import pytest

from oracle import acoustic3d as A
from oracle import grid as G
from oracle import halo as HL
import synthetic_inputs as SI


def _mode_matrix(co, theta):
    """Per-mode map of one step.  With P_i = Re(p e^{I theta.i}) and the d-velocity
    at the face i - e_d/2, Re(v_d e^{I(theta.i - theta_d/2)}):
        P_i - P_{i-e_d}          = p e^{I(theta.i - theta_d/2)} * 2I sin(theta_d/2)
        V_{i+e_d/2} - V_{i-e_d/2} = v_d e^{I theta.i}            * 2I sin(theta_d/2)
    so compute_V: v_d' = v_d - 2I cV_d s_d p, compute_P: p' = p - 2I cP sum_d r_d s_d v_d'."""
    s = [math.sin(t / 2.0) for t in theta]
    Av = np.eye(4, dtype=complex)
    for d in range(3):
        Av[1 + d, 0] = -2j * co["cV"][d] * s[d]
    Bp = np.eye(4, dtype=complex)
    for d in range(3):
        Bp[0, 1 + d] = -2j * co["cP"] * co["r"][d] * s[d]
    return Bp @ Av


@pytest.mark.parametrize("N,m", [((8, 6, 10), (1, 2, 1)), ((12, 5, 7), (3, 0, 2)), ((16, 4, 4), (1, 1, 0))])
def test_fourier_mode_exact_evolution(N, m):
    per = (1, 1, 1)
    d = [1.0 / N[i] for i in range(3)]
    rho, K = 1.3, 0.7
    dt = 0.4 * min(d) / math.sqrt(K / rho)
    co = A.coefficients(dt, rho, K, *d)
    theta = [2.0 * math.pi * m[i] / N[i] for i in range(3)]
    z, y, x = np.meshgrid(np.arange(N[2]), np.arange(N[1]), np.arange(N[0]), indexing="ij")
    phase = theta[0] * x + theta[1] * y + theta[2] * z
    P0 = np.cos(phase)
    shapes = A.field_shapes(N, per)
    V0 = [np.zeros(s) for s in shapes[1:]]
    nt = 13
    P, Vx, Vy, Vz = A.run(P0, *V0, nt, per, dt, rho, K, *d)
    amp = np.linalg.matrix_power(_mode_matrix(co, theta), nt) @ np.array([1, 0, 0, 0], dtype=complex)
    expect = [np.real(amp[0] * np.exp(1j * phase))]
    shifts = [theta[0] / 2, theta[1] / 2, theta[2] / 2]
    for dd in range(3):
        expect.append(np.real(amp[1 + dd] * np.exp(1j * (phase - shifts[dd]))))
    for got, ref in zip((P, Vx, Vy, Vz), expect):
        assert np.max(np.abs(got - ref)) < 1e-12
    # the mode is not trivial: the amplitude moved
    assert abs(amp[0] - 1) > 1e-3 or any(abs(a) > 1e-3 for a in amp[1:])


def test_sum_P_conserved_periodic():
    N, per = (9, 7, 6), (1, 1, 1)
    shapes = A.field_shapes(N, per)
    P0, Vx0, Vy0, Vz0 = SI.global_acoustic_fields(shapes, seed=3)
    d = [1.0 / N[i] for i in range(3)]
    dt = 0.3 * min(d)
    s0 = math.fsum(P0.ravel())
    P, *_ = A.run(P0, Vx0, Vy0, Vz0, 20, per, dt, 1.0, 1.0, *d)
    assert abs(math.fsum(P.ravel()) - s0) < 1e-11 * P.size
    assert np.max(np.abs(P - P0)) > 1e-3   # something happened


def test_mirror_symmetry_bitwise():
    """A state even under x -> Nx-1-x (P) with Vx odd under the face mirror i -> Nx-i
    (and even Vy, Vz) keeps that symmetry exactly; likewise in y and z."""
    N, per = (10, 9, 8), (0, 0, 0)
    shapes = A.field_shapes(N, per)
    rnd = SI.global_acoustic_fields(shapes, seed=5)
    P0 = rnd[0]
    for ax in range(3):   # a + flip(a) is exactly even; later sums keep the earlier axes exact
        P0 = P0 + np.flip(P0, axis=ax)
    V0 = [np.zeros(s) for s in shapes[1:]]
    d = (0.1, 0.12, 0.09)
    P, Vx, Vy, Vz = A.run(P0, *V0, 15, per, 0.02, 1.1, 0.9, *d)
    assert np.array_equal(P, P[:, :, ::-1]) and np.array_equal(P, P[:, ::-1, :]) and np.array_equal(P, P[::-1, :, :])
    assert np.array_equal(Vx, -Vx[:, :, ::-1]) and np.array_equal(Vx, Vx[:, ::-1, :])
    assert np.array_equal(Vy, -Vy[:, ::-1, :]) and np.array_equal(Vy, Vy[::-1, :, :])
    assert np.array_equal(Vz, -Vz[::-1, :, :]) and np.array_equal(Vz, Vz[:, :, ::-1])
    assert np.max(np.abs(Vx)) > 1e-3


def test_fixed_point():
    N, per = (7, 6, 5), (0, 1, 0)
    shapes = A.field_shapes(N, per)
    P0 = np.full(shapes[0], 2.5)
    V0 = [np.zeros(s) for s in shapes[1:]]
    out = A.run(P0, *V0, 5, per, 0.01, 1.0, 2.0, 0.1, 0.1, 0.1)
    assert np.array_equal(out[0], P0)
    for v, v0 in zip(out[1:], V0):
        assert np.array_equal(v, v0)


@pytest.mark.parametrize("per", [(0, 0, 0), (1, 0, 1), (1, 1, 1)])
def test_scalar_transcription_agrees(per):
    N = (5, 4, 6)
    shapes = A.field_shapes(N, per)
    F0 = SI.global_acoustic_fields(shapes, seed=7)
    args = (3, per, 0.013, 1.2, 0.8, 0.2, 0.25, 0.17)
    a = A.run(*F0, *args)
    b = A.run_py(*F0, *args)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def _distributed(F0, dims, n, o, per, nt, co):
    nr = dims[0] * dims[1] * dims[2]
    sizes = [n, (n[0] + 1, n[1], n[2]), (n[0], n[1] + 1, n[2]), (n[0], n[1], n[2] + 1)]
    loc = {r: [G.window(F0[f], G.coords_of_rank(r, dims), dims, n, o, per, sizes[f]) for f in range(4)]
           for r in range(nr)}
    for _ in range(nt):
        for r in range(nr):
            A.local_V(*loc[r], co)
        HL.update_halo({r: loc[r][1:] for r in range(nr)}, dims, per, n, o)
        for r in range(nr):
            A.local_P(*loc[r], co)
    return loc, sizes


def test_decomposition_independence():
    rng = random.Random(15716)
    for case in range(30):
        dims = tuple(rng.randint(1, 3) for _ in range(3))
        o = (2, 2, 2)
        n = tuple(rng.randint(4, 7) for _ in range(3))
        per = tuple(rng.random() < 0.4 for _ in range(3))
        N = [G.global_size(n[i], o[i], dims[i], per[i]) for i in range(3)]
        shapes = A.field_shapes(N, per)
        F0 = SI.global_acoustic_fields(shapes, seed=case)
        d = [1.0 / N[i] for i in range(3)]
        dt, rho, K = 0.3 * min(d), 1.0, 1.5
        co = A.coefficients(dt, rho, K, *d)
        ref = A.run(*F0, 4, per, dt, rho, K, *d)
        loc, sizes = _distributed(F0, dims, n, o, per, 4, co)
        for r in loc:
            c = G.coords_of_rank(r, dims)
            for f in range(4):
                W = G.window(ref[f], c, dims, n, o, per, sizes[f])
                assert np.array_equal(loc[r][f], W), (case, dims, n, per, r, f)


# ---------------------------------------------------------------------------------------------------
# Pins of the coefficients (reading A2) from the physics alone -- no call to A.coefficients().
#
# The continuum equations rho dV/dt = -grad P, dP/dt = -K div V (the system the leapfrog discretises)
# fix two numbers a correct discretisation must reproduce for a periodic mode with phase angles
# theta_d (s_d = sin(theta_d/2)), written only in terms of (rho, K, dt, d_d):
#   * the leapfrog dispersion relation  sin^2(phi/2) = (K/rho) dt^2 sum_d s_d^2 / d_d^2   (phi: phase
#     advance per step; a 2x2 system with determinant 1 for (P, longitudinal V)),
#   * the wave impedance of a travelling mode  |V| / |P| = 1 / sqrt(rho K), along the discrete wave
#     vector (s_d/d_d)/S, S = sqrt(sum s_d^2/d_d^2), with V lagging P by half a cell and half a step.
# A travelling mode initialised from these is reproduced step after step.  A wrong cV (e.g.
# dt/(rho d^2), or K in place of 1/rho) or a wrong cP / r_d changes phi or the impedance and fails.
def _travelling_mode(N, m, rho, K, dt, d):
    theta = [2.0 * math.pi * m[i] / N[i] for i in range(3)]
    s = [math.sin(t / 2.0) for t in theta]
    S = math.sqrt(sum(s[i] ** 2 / d[i] ** 2 for i in range(3)))
    phi = 2.0 * math.asin(math.sqrt(K / rho) * dt * S)
    Z = math.sqrt(rho * K)
    z, y, x = np.meshgrid(np.arange(N[2]), np.arange(N[1]), np.arange(N[0]), indexing="ij")
    phase = theta[0] * x + theta[1] * y + theta[2] * z

    def fields(n):
        P = np.cos(phase + n * phi)
        V = [-(1.0 / Z) * (s[dd] / d[dd]) / S * np.cos(phase - theta[dd] / 2 - phi / 2 + n * phi) for dd in range(3)]
        return [P] + V
    return fields, phi


@pytest.mark.parametrize("N,m,rho,K,d", [
    ((8, 6, 10), (1, 2, 1), 1.3, 0.7, (0.125, 0.2, 0.09)),
    ((12, 5, 7), (3, 0, 2), 2.0, 3.5, (0.1, 0.1, 0.1)),
    ((16, 4, 4), (1, 0, 0), 0.8, 1.9, (0.05, 0.3, 0.3)),
])
def test_travelling_mode_dispersion_and_impedance(N, m, rho, K, d):
    dt = 0.45 * min(d) / math.sqrt(K / rho) / math.sqrt(3.0)
    fields, phi = _travelling_mode(N, m, rho, K, dt, d)
    assert phi > 0.05                                   # the mode really moves
    F0 = fields(0)
    nt = 17
    out = A.run(*F0, nt, (1, 1, 1), dt, rho, K, *d)
    for got, ref in zip(out, fields(nt)):
        assert np.max(np.abs(got - ref)) < 1e-12


def test_sound_speed_continuum_limit():
    """A standing wave on a fine grid oscillates at omega = c k with c = sqrt(K/rho): the phase
    advance per step measured from the oracle's P (cos(phi) = (p[n+1] + p[n-1]) / (2 p[n]), the
    recurrence of a determinant-1 two-level scheme) gives c within the O((k d)^2 + (omega dt)^2)
    discretisation error."""
    N, lx, rho, K = (128, 4, 4), 1.0, 1.7, 2.9
    d = (lx / N[0], 0.5, 0.5)
    c = math.sqrt(K / rho)
    dt = 0.2 * d[0] / c
    k = 2.0 * math.pi / lx
    x = np.arange(N[0])
    F = [np.zeros(s) for s in A.field_shapes(N, (1, 1, 1))]
    F[0][...] = np.cos(k * d[0] * x)[None, None, :]
    amp = []
    for _ in range(3):
        amp.append(float(np.sum(F[0][0, 0, :] * np.cos(k * d[0] * x))) * 2.0 / N[0])
        F = list(A.run(*F, 1, (1, 1, 1), dt, rho, K, *d))
    cphi = (amp[2] + amp[0]) / (2.0 * amp[1])
    c_num = math.acos(cphi) / dt / k
    assert abs(c_num / c - 1.0) < 2e-3
    # a scheme with the wrong speed (e.g. K*rho or 1/rho in place of K/rho) is far outside that
    assert abs(math.sqrt(K * rho) / c - 1.0) > 0.1 and abs(math.sqrt(1.0 / rho) / c - 1.0) > 0.1
