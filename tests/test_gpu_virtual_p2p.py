"""The cross-rank data planes of the P2P path, emulated on ONE GPU (the driver's box), bit-exact vs the
oracle.

Ranks that share a GPU run inside one process (virtual ranks).  Two processes with spinning kernels on
one GPU are not co-scheduled (B200_PROFILING.md), so the emulation keeps every wait satisfiable:

* the fused stencil + peer-store kernel (heat_fused_kernel) covers ALL hosted ranks in ONE launch: each
  rank's face tiles store into the sibling ranks' halos / x staging buffers and publish per-(face, chunk)
  release flags; the siblings' halo tiles acquire them in the next step, the forwarders and the drain in
  the last -- the same stores, counters, flags, staging parity and forwarding as between GPUs, only the
  destination pointers are the siblings' arrays instead of CUDA-IPC mappings;
* the split path's P2P protocol (IGG_OPT_LOCAL_P2P): pack kernels store into the receiver's slot of the
  receive arena and the last CTA release-stores the epoch into its flag; flag_wait + unpack acquire it
  (packs precede the waits on the stream).
"""
import numpy as np
import pytest

import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import heat3d as app
from oracle import grid as OG
from oracle import halo as OHL
import synthetic_inputs as SI

from _heat_cases import assert_windows, oracle_global

pytestmark = pytest.mark.gpu


def _N(n, dims, per):
    return tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))


def _run(n, dims, per, nt, per_step=False, options=None, init="random"):
    import torch
    R = dims[0] * dims[1] * dims[2]
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=R, device=0, path="p2p")
    try:
        for k, v in (options or {}).items():
            g.set_option(k, v)
        T, T2, Ci = app.alloc_fields(g)
        (app.init_random if init == "random" else app.init_paper)(g, T, T2, Ci)
        d = app.spacing(g)
        dt = app.stable_dt(g, Ci, *d)
        l0 = g.kernel_launches()
        T, T2 = app.run(g, T, T2, Ci, nt, dt, d, per_step=per_step)
        torch.cuda.synchronize()
        g.check()
        return [t.cpu().numpy() for t in T], dt, g.kernel_launches() - l0
    finally:
        g.finalize()


CASES = [
    ((130, 36, 34), (2, 1, 1), (0, 0, 0)),    # x faces: staged columns
    ((130, 36, 34), (2, 1, 1), (1, 1, 1)),    # + periodic: both sides, self-wrap in y and z
    ((66, 40, 36), (1, 2, 1), (0, 1, 0)),     # y faces (p = 2 periodic: both neighbours the same rank)
    ((130, 20, 36), (1, 1, 2), (0, 0, 0)),    # z faces: the end chunks
    ((130, 36, 34), (2, 2, 1), (0, 0, 0)),    # x + y: edges forwarded x -> y
    ((130, 20, 22), (2, 2, 2), (0, 0, 0)),    # 2x2x2 (config B:9/B:10 topology): corners x -> y -> z
    ((130, 20, 22), (2, 2, 2), (1, 0, 1)),
    ((68, 18, 20), (4, 1, 1), (1, 0, 0)),     # interior ranks: both x sides
    ((130, 20, 22), (1, 2, 4), (0, 1, 1)),
    ((66, 36, 34), (2, 2, 1), (0, 1, 0)),     # two x tiles: every tile a border tile
    ((130, 6, 34), (2, 1, 2), (0, 0, 0)),     # one y tile
]


@pytest.mark.parametrize("n,dims,per", CASES)
@pytest.mark.parametrize("per_step", [False, True])
def test_fused_virtual_ranks_bit_exact(n, dims, per, per_step):
    """Fig. 1's loop on prod(dims) ranks of one GPU through the fused kernel (one launch per step over
    all ranks; igg_heat_run pipelines the steps, per_step drains each), every rank's window -- halos,
    edges and corners included -- bit-exact vs the canonical oracle on the global grid."""
    nt = 5
    out, dt, launches = _run(n, dims, per, nt, per_step=per_step)
    ref, dtr = oracle_global(_N(n, dims, per), per, nt)
    assert dt == dtr
    assert_windows(out, ref, dims, n, (2, 2, 2), per)
    # one fused launch per step for all ranks, plus one drain per complete step
    assert launches == (2 * nt if per_step else nt + 1), launches


def test_fused_virtual_ranks_paper_literal_within_1e12():
    n, dims, per, nt = (130, 36, 34), (2, 2, 1), (0, 0, 0), 6
    out, _, _ = _run(n, dims, per, nt)
    from oracle import heat3d as OH
    lit, _ = oracle_global(_N(n, dims, per), per, nt, mode=OH.LITERAL)
    assert_windows(out, lit, dims, n, (2, 2, 2), per, exact=False, rtol=1e-12)


def test_fused_virtual_ranks_full_size_512():
    """The bench configuration's cross-rank path at full size: 2 ranks of 512^3 (dims 2x1x1, the B:9 split)
    in one fused launch per step -- 64-plane middle chunks, 8-plane end chunks, x faces through the
    staging buffers -- 3 pipelined steps, every cell of both ranks bit-exact vs the oracle on the global
    1022 x 512 x 512 grid."""
    n, dims, per, nt = (512, 512, 512), (2, 1, 1), (0, 0, 0), 3
    out, dt, launches = _run(n, dims, per, nt)
    ref, dtr = oracle_global(_N(n, dims, per), per, nt)
    assert dt == dtr
    assert launches == nt + 1
    assert_windows(out, ref, dims, n, (2, 2, 2), per)


def test_fused_equals_split_path_and_sequential():
    """Decomposition/schedule independence on the GPU: fused (pipelined and per step), the split
    P2P-protocol path and the sequential schedule give identical bits."""
    n, dims, per, nt = (130, 36, 34), (2, 1, 2), (1, 0, 0), 4
    a, _, _ = _run(n, dims, per, nt)
    b, _, _ = _run(n, dims, per, nt, per_step=True)
    c, _, _ = _run(n, dims, per, nt, options={P.OPT_FUSED: 0, P.OPT_LOCAL_P2P: 1})
    for x, y, z in zip(a, b, c):
        assert np.array_equal(x, y) and np.array_equal(x, z)


@pytest.mark.parametrize("n,dims,per", [((40, 36, 34), (2, 1, 1), (0, 0, 0)), ((40, 36, 34), (2, 2, 2), (1, 0, 1)),
                                        ((24, 20, 18), (3, 1, 2), (1, 1, 1))])
def test_split_path_p2p_protocol_bit_exact(n, dims, per):
    """The split schedule (boundary slabs, then pack -> peer-slot store + release flag -> acquire wait ->
    unpack, inner box concurrent) with the P2P protocol between the virtual ranks."""
    nt = 4
    out, dt, _ = _run(n, dims, per, nt, per_step=True,
                      options={P.OPT_FUSED: 0, P.OPT_LOCAL_P2P: 1, P.OPT_X_ALIGN: 1})
    ref, dtr = oracle_global(_N(n, dims, per), per, nt)
    assert dt == dtr
    assert_windows(out, ref, dims, n, (2, 2, 2), per)


@pytest.mark.parametrize("dims,per", [((2, 2, 2), (0, 0, 0)), ((2, 2, 2), (1, 1, 1)), ((3, 2, 1), (1, 0, 1))])
def test_update_halo_p2p_protocol_staggered(dims, per):
    """config B:10's field set (P n, Vx n+1 in x, Vy, Vz) through update_halo with the P2P protocol
    between the virtual ranks, NaN-poisoned receive layers, twice (ping-pong parity), bit-exact vs the
    oracle's update_halo."""
    import torch
    n, o = (20, 18, 16), (2, 2, 2)
    sizes = [n, (n[0] + 1, n[1], n[2]), (n[0], n[1] + 1, n[2]), (n[0], n[1], n[2] + 1)]
    R = dims[0] * dims[1] * dims[2]
    host = {r: [SI.random_field(s[::-1], 9000 + 10 * r + f) for f, s in enumerate(sizes)] for r in range(R)}
    for r in host:   # NaN in every receive layer: each must be overwritten
        c = OG.coords_of_rank(r, dims)
        for A in host[r]:
            for d in range(3):
                hs = OG.halo_spec(n[d], o[d], A.shape[2 - d])
                if hs["h"] == 0:
                    continue
                sl = [slice(None)] * 3
                if c[d] > 0 or per[d]:
                    sl[2 - d] = slice(*hs["recv_lower"])
                    A[tuple(sl)] = np.nan
                if c[d] < dims[d] - 1 or per[d]:
                    sl[2 - d] = slice(*hs["recv_upper"])
                    A[tuple(sl)] = np.nan
    ref = {r: [a.copy() for a in host[r]] for r in host}
    for _ in range(2):
        OHL.update_halo(ref, dims, per, n, o)
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=R, device=0, path="p2p")
    try:
        g.set_option(P.OPT_LOCAL_P2P, 1)
        dev = [[torch.from_numpy(host[r][f]).cuda() for r in range(R)] for f in range(len(sizes))]
        for _ in range(2):
            g.update_halo(*dev)
        torch.cuda.synchronize()
        g.check()
        for f in range(len(sizes)):
            for r in range(R):
                assert np.array_equal(dev[f][r].cpu().numpy(), ref[r][f]), (dims, per, r, f)
    finally:
        g.finalize()


def _run_f32(n, dims, per, nt, per_step=False):
    import torch
    R = dims[0] * dims[1] * dims[2]
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=R, device=0, path="p2p")
    try:
        g.set_option(P.OPT_FUSED_F32, 1)
        T, T2, Ci = app.alloc_fields(g, dtype=torch.float32)
        app.init_random(g, T, T2, Ci)
        from oracle import heat3d as OH
        N = _N(n, dims, per)
        T0g, Cig = SI.global_heat_fields(*N)
        d = [OH.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
        dt = OH.stable_dt(*d, 1.0, Cig)
        l0 = g.kernel_launches()
        T, T2 = app.run(g, T, T2, Ci, nt, dt, d, per_step=per_step)
        torch.cuda.synchronize()
        g.check()
        ref = OH.heat_run_f32(T0g, Cig, nt, per, 1.0, dt, *d)
        return [t.cpu().numpy() for t in T], ref, g.kernel_launches() - l0
    finally:
        g.finalize()


F32_CASES = [   # (binary32 tiles are 128 cells wide: rows of whole float4 vectors, two x tiles at least)
    ((132, 36, 34), (2, 1, 1), (0, 0, 0)),
    ((132, 36, 34), (2, 1, 1), (1, 1, 1)),
    ((132, 36, 34), (2, 2, 1), (0, 0, 0)),
    ((132, 20, 22), (2, 2, 2), (1, 0, 1)),
    ((136, 18, 20), (4, 1, 1), (1, 0, 0)),
    ((260, 20, 22), (1, 2, 2), (0, 1, 1)),   # three x tiles
]


@pytest.mark.parametrize("n,dims,per", F32_CASES)
@pytest.mark.parametrize("per_step", [False, True])
def test_fused_binary32_virtual_ranks_bit_exact(n, dims, per, per_step):
    """The binary32 variant through the same fused kernel (float4 lanes): one launch per
    step over all ranks, pipelined (igg_heat_run_f32) and per step, bit-exact vs the binary32 oracle
    (reading 24) on the global grid."""
    nt = 5
    out, ref, launches = _run_f32(n, dims, per, nt, per_step=per_step)
    for r, got in enumerate(out):
        W = OG.window(ref, OG.coords_of_rank(r, dims), dims, n, (2, 2, 2), per, n)
        assert got.dtype == np.float32 and np.array_equal(got, W), (n, dims, per, r)
    assert launches == (2 * nt if per_step else nt + 1), launches


def test_fused_binary32_full_size_512():
    """Two binary32 ranks of 512^3 (2x1x1) in the fused kernel, 3 pipelined steps, every cell bit-exact."""
    n, dims, per, nt = (512, 512, 512), (2, 1, 1), (0, 0, 0), 3
    out, ref, launches = _run_f32(n, dims, per, nt)
    assert launches == nt + 1
    for r, got in enumerate(out):
        assert np.array_equal(got, OG.window(ref, OG.coords_of_rank(r, dims), dims, n, (2, 2, 2), per, n)), r
