"""GPU parity of the heat step (CUDA path through the C ABI) against the CPU
oracle on the global grid.  Gates (north star):
bit-exact vs the canonical oracle, max relative error <= 1e-12 vs the
paper-literal oracle, halos included; distributed == single-GPU bit-exact."""
import numpy as np
import pytest

import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import heat3d as app
from oracle import grid as OG
from oracle import heat3d as OH
import synthetic_inputs as SI

from _heat_cases import assert_windows, gpu_run, oracle_global

pytestmark = pytest.mark.gpu


def _N(n, dims, per, o):
    return tuple(OG.global_size(n[i], o[i], dims[i], bool(per[i])) for i in range(3))


@pytest.mark.parametrize("n", [(40, 33, 30), (37, 33, 30), (130, 20, 66)])
@pytest.mark.parametrize("kernel", [0, 1])
def test_single_rank_vs_oracle(n, kernel):
    dims, per, o = (1, 1, 1), (0, 0, 0), (2, 2, 2)
    out, dt, _, _ = gpu_run(P, app, n, dims, per, o, 10, (16, 2, 2), options={P.OPT_STENCIL_KERNEL: kernel})
    can, dtr = oracle_global(n, per, 10)
    assert dt == dtr
    assert_windows(out, can, dims, n, o, per)
    lit, _ = oracle_global(n, per, 10, mode=OH.LITERAL)
    assert_windows(out, lit, dims, n, o, per, exact=False)


@pytest.mark.parametrize("bw", [(0, 0, 0), (16, 2, 2), (4, 2, 2)])
@pytest.mark.parametrize("n", [(32, 32, 32), (17, 32, 32)])
def test_config_b7_emulated_2x1x1(n, bw):
    """B:7: local 32^3 nt=10 (reading i) and global 32^3 split in two 17x32x32 (reading ii)."""
    dims, per, o = (2, 1, 1), (0, 0, 0), (2, 2, 2)
    out, dt, _, _ = gpu_run(P, app, n, dims, per, o, 10, bw)
    N = _N(n, dims, per, o)
    can, dtr = oracle_global(N, per, 10)
    assert dt == dtr
    assert_windows(out, can, dims, n, o, per)
    lit, _ = oracle_global(N, per, 10, mode=OH.LITERAL)
    assert_windows(out, lit, dims, n, o, per, exact=False)


def test_config_b7_periodic_x():
    dims, per, o, n = (2, 1, 1), (1, 0, 0), (2, 2, 2), (32, 32, 32)
    out, _, _, _ = gpu_run(P, app, n, dims, per, o, 10, (4, 2, 2))
    can, _ = oracle_global(_N(n, dims, per, o), per, 10)
    assert_windows(out, can, dims, n, o, per)


@pytest.mark.parametrize("case", [
    dict(n=(24, 20, 18), dims=(2, 2, 2), per=(0, 0, 0), o=(2, 2, 2), bw=(16, 2, 2)),
    dict(n=(24, 20, 18), dims=(2, 2, 2), per=(0, 0, 0), o=(2, 2, 2), bw=(4, 3, 2)),
    dict(n=(26, 20, 18), dims=(2, 2, 1), per=(1, 0, 1), o=(2, 2, 2), bw=(4, 2, 2)),
    dict(n=(22, 21, 19), dims=(3, 1, 2), per=(0, 1, 0), o=(4, 2, 2), bw=(4, 2, 2)),
    dict(n=(20, 18, 16), dims=(1, 1, 1), per=(1, 1, 1), o=(2, 2, 2), bw=(4, 2, 2)),   # self-wrap
    dict(n=(34, 18, 16), dims=(4, 1, 1), per=(0, 0, 0), o=(2, 2, 2), bw=(2, 2, 2)),
])
@pytest.mark.parametrize("kernel", [0, 1])
def test_virtual_topologies_bit_exact(case, kernel):
    n, dims, per, o, bw = case["n"], case["dims"], case["per"], case["o"], case["bw"]
    out, dt, _, _ = gpu_run(P, app, n, dims, per, o, 6, bw, options={P.OPT_STENCIL_KERNEL: kernel})
    can, dtr = oracle_global(_N(n, dims, per, o), per, 6)
    assert dt == dtr
    assert_windows(out, can, dims, n, o, per)


@pytest.mark.parametrize("case", [
    dict(n=(260, 40, 36), dims=(2, 1, 1), per=(0, 0, 0)),
    dict(n=(200, 24, 20), dims=(2, 2, 2), per=(0, 0, 0)),
    dict(n=(136, 30, 26), dims=(2, 1, 2), per=(1, 0, 0)),
])
@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("schedule", [0, 1])
@pytest.mark.parametrize("x_align", [1, 64])
def test_schedules_bit_exact(case, kernel, schedule, x_align):
    """Both schedules, exact and 512-B-rounded x boundaries, three kernels."""
    n, dims, per, o = case["n"], case["dims"], case["per"], (2, 2, 2)
    out, _, _, _ = gpu_run(P, app, n, dims, per, o, 5, (16, 2, 2), x_align=x_align,
                           options={P.OPT_STENCIL_KERNEL: kernel, P.OPT_SCHEDULE: schedule})
    can, _ = oracle_global(_N(n, dims, per, o), per, 5)
    assert_windows(out, can, dims, n, o, per)


def test_overlap_schedule_equals_sequential():
    n, dims, per, o = (40, 24, 20), (2, 2, 1), (0, 0, 0), (2, 2, 2)
    a, _, _, _ = gpu_run(P, app, n, dims, per, o, 8, (0, 0, 0))
    b, _, _, _ = gpu_run(P, app, n, dims, per, o, 8, (16, 2, 2))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_width_precondition():
    import torch
    g = P.init_global_grid(32, 16, 16, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        T, T2, Ci = app.alloc_fields(g)
        app.init_paper(g, T, T2, Ci)
        with pytest.raises(P.IggError) as e:
            g.heat_step(T2, T, Ci, 1.0, 1e-3, 0.1, 0.1, 0.1, bw=(1, 2, 2))
        assert e.value.name == "IGG_E_WIDTH"
        g.heat_step(T2, T, Ci, 1.0, 1e-3, 0.1, 0.1, 0.1, bw=(2, 0, 0))   # y, z have no neighbours
        torch.cuda.synchronize()
    finally:
        g.finalize()


def test_fixed_point_and_buffer_reuse():
    n, dims, per, o = (34, 18, 16), (2, 1, 1), (0, 0, 0), (2, 2, 2)
    out, _, allocs, _ = gpu_run(P, app, n, dims, per, o, 100, (16, 2, 2), init="paper")
    for A in out:
        assert np.all(A == 1.7)
    assert allocs[0] == allocs[-1]


def test_state_errors():
    g = P.init_global_grid(8, 8, 8, dims=(1, 1, 1), device=0)
    g.finalize()
    with pytest.raises(P.IggError) as e:
        g.nx_g()
    assert e.value.name == "IGG_E_STATE"


def test_field_global_max_and_dt():
    import torch
    g = P.init_global_grid(20, 18, 16, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        T, T2, Ci = app.alloc_fields(g)
        app.init_random(g, T, T2, Ci)
        ref = max(float(c.max()) for c in Ci)
        assert g.field_global_max(Ci) == ref
        assert g.global_max(0.25) == 0.25
        torch.cuda.synchronize()
    finally:
        g.finalize()


def test_heat_run_host_equals_device_loop():
    import torch
    n = (40, 24, 20)
    g = P.init_global_grid(*n, dims=(2, 1, 1), local_ranks=2, device=0)
    try:
        T, T2, Ci = app.alloc_fields(g)
        app.init_random(g, T, T2, Ci)
        d = app.spacing(g)
        dt = app.stable_dt(g, Ci, *d)
        Th = torch.stack([t.cpu() for t in T]).contiguous().pin_memory()
        Ch = torch.stack([c.cpu() for c in Ci]).contiguous().pin_memory()
        g.heat_run_host(Th, Ch, 1.0, dt, *d, 7, bw=(16, 2, 2))
        T, T2 = app.run(g, T, T2, Ci, 7, dt, d)
        torch.cuda.synchronize()
        for r in range(2):
            assert torch.equal(Th[r], T[r].cpu())
    finally:
        g.finalize()


@pytest.mark.slow
@pytest.mark.parametrize("init", ["random", "paper"])
def test_full_size_512_nt100_vs_oracle(init):
    """B:8 at full size in the bench's launch configuration (1 GPU, 512^3,
    nt=100, hide_communication (16,2,2)), every cell compared."""
    n, dims, per, o = (512, 512, 512), (1, 1, 1), (0, 0, 0), (2, 2, 2)
    out, dt, _, _ = gpu_run(P, app, n, dims, per, o, 100, (16, 2, 2), init=init)
    can, dtr = oracle_global(n, per, 100, init=init)
    assert dt == dtr
    assert np.array_equal(out[0], can)
    if init == "random":
        lit, _ = oracle_global(n, per, 100, init=init, mode=OH.LITERAL)
        assert np.max(np.abs(out[0] - lit) / np.abs(lit)) <= 1e-12


@pytest.mark.ablation
@pytest.mark.parametrize("variant", list(range(2, 30)) + list(range(50, 57)))
def test_box_kernel_variants_bit_exact(variant):
    """Every tuning variant of the box kernel computes the same cells (ablations
    must be valid): 2 virtual ranks, overlap schedule, vs the canonical oracle."""
    n, dims, per, o = (130, 44, 70), (2, 1, 1), (0, 0, 0), (2, 2, 2)
    out, _, _, _ = gpu_run(P, app, n, dims, per, o, 5, (16, 2, 2), options={P.OPT_STENCIL_KERNEL: variant})
    can, _ = oracle_global(_N(n, dims, per, o), per, 5)
    assert_windows(out, can, dims, n, o, per)
    out1, _, _, _ = gpu_run(P, app, (130, 44, 70), (1, 1, 1), per, o, 5, (16, 2, 2),
                            options={P.OPT_STENCIL_KERNEL: variant})
    can1, _ = oracle_global((130, 44, 70), per, 5)
    assert np.array_equal(out1[0], can1)


@pytest.mark.parametrize("per", [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)])
def test_fused_self_wrap_one_gpu(per):
    """Periodic axes wrapping onto the one process run the fused P2P path with the rank as its own
    neighbour (faces stored into its own halos, x faces through the staging buffer); heat_run
    (pipelined) and single steps both bit-exact vs the periodic global oracle."""
    import torch
    n = (130, 36, 34)
    N = tuple(OG.global_size(n[i], 2, 1, bool(per[i])) for i in range(3))
    ref, dtr = oracle_global(N, per, 7)
    for per_step in (False, True):
        g = P.init_global_grid(*n, periods=per, local_ranks=1, device=0, path=P.PATH_P2P)
        try:
            T, T2, Ci = app.alloc_fields(g)
            app.init_random(g, T, T2, Ci)
            d = app.spacing(g)
            dt = app.stable_dt(g, Ci, *d)
            assert dt == dtr
            l0 = g.kernel_launches()
            T, T2 = app.run(g, T, T2, Ci, 7, dt, d, per_step=per_step)
            torch.cuda.synchronize()
            g.check()
            # one launch per step and one drain per complete step (run or single step)
            assert g.kernel_launches() - l0 == (7 * 2 if per_step else 8)
            assert_windows([T[0].cpu().numpy()], ref, (1, 1, 1), n, (2, 2, 2), per)
        finally:
            g.finalize()


@pytest.mark.parametrize("case", [
    dict(n=(24, 20, 1), dims=(2, 2, 1), per=(0, 1, 0)),   # 2-D (x-y), y periodic
    dict(n=(30, 1, 1), dims=(3, 1, 1), per=(1, 0, 0)),    # 1-D, periodic
    dict(n=(1, 18, 16), dims=(1, 2, 2), per=(0, 0, 0)),   # 2-D (y-z)
    dict(n=(70, 36, 1), dims=(1, 1, 1), per=(0, 0, 0)),   # 2-D, one rank
    dict(n=(20, 1, 14), dims=(2, 1, 1), per=(0, 0, 1)),   # 2-D (x-z), z periodic self-wrap
])
def test_low_dimensional_grids(case):
    """1-D/2-D grids as size-1 axes (reading 23): heat steps with update_halo on virtual
    topologies, bit-exact vs the canonical oracle on the global grid."""
    n, dims, per = case["n"], case["dims"], case["per"]
    N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
    out, dt, _, _ = gpu_run(P, app, n, dims, per, (2, 2, 2), 6, (4, 2, 2))
    ref, dtr = oracle_global(N, per, 6)
    assert dt == dtr
    assert_windows(out, ref, dims, n, (2, 2, 2), per)


def test_low_dimensional_init_rules():
    g = P.init_global_grid(24, 20, 1, local_ranks=4, device=0)   # automatic dims never split a size-1 axis
    try:
        assert g.dims[2] == 1 and g.dims[0] * g.dims[1] == 4 and g.nz_g() == 1
    finally:
        g.finalize()
    with pytest.raises(P.IggError) as e:
        P.init_global_grid(24, 20, 1, periods=(0, 0, 1), local_ranks=1, device=0)
    assert e.value.name == "IGG_E_ARG"
    with pytest.raises(P.IggError) as e:
        P.init_global_grid(24, 20, 1, dims=(1, 1, 2), local_ranks=2, device=0)
    assert e.value.name == "IGG_E_ARG"


@pytest.mark.parametrize("case", [
    dict(n=(24, 20, 18), dims=(2, 2, 1), per=(1, 0, 0)),
    dict(n=(30, 26, 1), dims=(2, 1, 1), per=(0, 0, 0)),      # 2-D
    dict(n=(40, 22, 20), dims=(1, 1, 1), per=(0, 1, 1)),     # self-wrap
    dict(n=(264, 21, 75), dims=(1, 1, 1), per=(0, 0, 0)),    # 3 x-tiles of the float4 kernel, ragged y/z
    dict(n=(132, 9, 40), dims=(2, 1, 1), per=(0, 0, 1)),     # 2 x-tiles on each of 2 ranks
    dict(n=(30, 20, 18), dims=(1, 2, 1), per=(0, 0, 0)),     # rows not 16-B aligned: the scalar kernel
    dict(n=(520, 13, 40), dims=(2, 1, 1), per=(0, 0, 0)),    # non-degenerate x split: float4 inner box
])
@pytest.mark.parametrize("bw", [(0, 0, 0), (4, 2, 2), (16, 2, 2)])
def test_binary32_heat_vs_oracle(case, bw):
    """The binary32 variant (reading 24): igg_heat_step_f32 with update_halo of a
    float field (sequential and hide_communication schedules), bit-exact vs the binary32 oracle."""
    import torch
    n, dims, per = case["n"], case["dims"], case["per"]
    nprocs = dims[0] * dims[1] * dims[2]
    N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
    T0g, Cig = SI.global_heat_fields(*N)
    d = [OH.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
    dt = OH.stable_dt(*d, 1.0, Cig)
    ref = OH.heat_run_f32(T0g, Cig, 6, per, 1.0, dt, *d)
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=nprocs, device=0)
    try:
        T, T2, Ci = app.alloc_fields(g, dtype=torch.float32)
        app.init_random(g, T, T2, Ci)
        for _ in range(6):
            g.heat_step(T2, T, Ci, 1.0, dt, *d, bw=bw)
            T, T2 = T2, T
        torch.cuda.synchronize()
        g.check()
        for r in range(nprocs):
            W = OG.window(ref, OG.coords_of_rank(r, dims), dims, n, (2, 2, 2), per, n)
            got = T[r].cpu().numpy()
            assert got.dtype == np.float32 and np.array_equal(got, W), (case, r)
    finally:
        g.finalize()


@pytest.mark.gpu
def test_binary32_full_size_512():
    """The f32 bench configuration (512^3 local, one GPU, the float4 cp.async kernel with its 64-plane
    chunks and 8-plane tail), nt = 2, every cell bit-exact vs the binary32 oracle (reading 24)."""
    import torch
    n, nt = (512, 512, 512), 2
    N = tuple(OG.global_size(n[i], 2, 1, False) for i in range(3))
    T0g, Cig = SI.global_heat_fields(*N)
    d = [OH.spacing(1.0, N[i], False) for i in range(3)]
    dt = OH.stable_dt(*d, 1.0, Cig)
    ref = OH.heat_run_f32(T0g, Cig, nt, (0, 0, 0), 1.0, dt, *d)
    del T0g, Cig
    g = P.init_global_grid(*n, local_ranks=1, device=0)
    try:
        T, T2, Ci = app.alloc_fields(g, dtype=torch.float32)
        app.init_random(g, T, T2, Ci)
        for _ in range(nt):
            g.heat_step(T2, T, Ci, 1.0, dt, *d)
            T, T2 = T2, T
        torch.cuda.synchronize()
        g.check()
        got = T[0].cpu().numpy()
        assert got.dtype == np.float32 and np.array_equal(got, ref)
    finally:
        g.finalize()


@pytest.mark.ablation
@pytest.mark.parametrize("variant", [0, 1] + list(range(100, 127)))
def test_binary32_kernel_variants_bit_exact(variant):
    """Every binary32 stencil variant (IGG_OPT_STENCIL_KERNEL; 1 = the scalar kernel, 101.. = the
    float4/float2 cp.async ablations) is valid: 2 virtual ranks, hide_communication (16,2,2) (inner
    box starting off a tile boundary, slabs through the scalar kernel), bit-exact vs the binary32 oracle."""
    import torch
    n, dims, per = (264, 21, 75), (2, 1, 1), (0, 0, 1)
    N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
    T0g, Cig = SI.global_heat_fields(*N)
    d = [OH.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
    dt = OH.stable_dt(*d, 1.0, Cig)
    ref = OH.heat_run_f32(T0g, Cig, 4, per, 1.0, dt, *d)
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=2, device=0)
    try:
        g.set_option(P.OPT_STENCIL_KERNEL, variant)
        g.set_option(P.OPT_FUSED_MODE, 2 | 16384)   # keep the x slabs (hide_communication in x)
        T, T2, Ci = app.alloc_fields(g, dtype=torch.float32)
        app.init_random(g, T, T2, Ci)
        for _ in range(4):
            g.heat_step(T2, T, Ci, 1.0, dt, *d, bw=(16, 2, 2))
            T, T2 = T2, T
        torch.cuda.synchronize()
        g.check()
        for r in range(2):
            W = OG.window(ref, OG.coords_of_rank(r, dims), dims, n, (2, 2, 2), per, n)
            assert np.array_equal(T[r].cpu().numpy(), W), (variant, r)
    finally:
        g.finalize()


@pytest.mark.ablation
def test_binary32_aligned_x_slabs():
    """fused_mode bits 16384 + 8192 (ablation): binary32 x boundary slabs kept, grown to whole 512-B segments."""
    import torch
    n, dims, per = (520, 13, 40), (2, 1, 1), (1, 0, 0)
    N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
    T0g, Cig = SI.global_heat_fields(*N)
    d = [OH.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
    dt = OH.stable_dt(*d, 1.0, Cig)
    ref = OH.heat_run_f32(T0g, Cig, 4, per, 1.0, dt, *d)
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=2, device=0)
    try:
        g.set_option(P.OPT_FUSED_MODE, 2 | 8192 | 16384)
        T, T2, Ci = app.alloc_fields(g, dtype=torch.float32)
        app.init_random(g, T, T2, Ci)
        for _ in range(4):
            g.heat_step(T2, T, Ci, 1.0, dt, *d, bw=(16, 2, 2))
            T, T2 = T2, T
        torch.cuda.synchronize()
        g.check()
        for r in range(2):
            W = OG.window(ref, OG.coords_of_rank(r, dims), dims, n, (2, 2, 2), per, n)
            assert np.array_equal(T[r].cpu().numpy(), W), r
    finally:
        g.finalize()


@pytest.mark.parametrize("per", [(1, 1, 0), (1, 0, 1)])
def test_fused_self_wrap_full_size_512(per):
    """The fused P2P kernel at the bench size (512^3, 64-plane chunks + 8-plane tail, x faces staged)
    with periodic axes wrapping onto the one GPU, through igg_heat_run (pipelined steps, drain):
    EVERY cell bit-exact vs the canonical oracle on the global grid."""
    import torch
    n, nt = (512, 512, 512), 3
    N = tuple(OG.global_size(n[i], 2, 1, bool(per[i])) for i in range(3))
    ref, dtr = oracle_global(N, per, nt)
    g = P.init_global_grid(*n, periods=per, local_ranks=1, device=0, path=P.PATH_P2P)
    try:
        T, T2, Ci = app.alloc_fields(g)
        app.init_random(g, T, T2, Ci)
        d = app.spacing(g)
        dt = app.stable_dt(g, Ci, *d)
        assert dt == dtr
        l0 = g.kernel_launches()
        T, T2 = app.run(g, T, T2, Ci, nt, dt, d)
        torch.cuda.synchronize()
        g.check()
        assert g.kernel_launches() - l0 == nt + 1          # one fused launch per step + the drain
        assert_windows([T[0].cpu().numpy()], ref, (1, 1, 1), n, (2, 2, 2), per)
    finally:
        g.finalize()


def test_reallocated_array_is_never_taken_for_the_cached_one():
    """the fused path caches peer mappings per array.  An array freed and re-allocated at the
    same address (torch caching allocator after empty_cache) must not reuse the old entry: heat_run
    re-validates the cache (allocation identity = base, size, buffer id) and stays bit-exact."""
    import torch
    n, per, nt = (130, 36, 34), (1, 1, 1), 3
    N = tuple(OG.global_size(n[i], 2, 1, bool(per[i])) for i in range(3))
    ref, dtr = oracle_global(N, per, nt)
    g = P.init_global_grid(*n, periods=per, local_ranks=1, device=0, path=P.PATH_P2P)
    try:
        for rep in range(2):
            T, T2, Ci = app.alloc_fields(g)
            app.init_random(g, T, T2, Ci)
            d = app.spacing(g)
            dt = app.stable_dt(g, Ci, *d)
            T, T2 = app.run(g, T, T2, Ci, nt, dt, d)
            torch.cuda.synchronize()
            g.check()
            assert_windows([T[0].cpu().numpy()], ref, (1, 1, 1), n, (2, 2, 2), per)
            g.release_arrays()
            del T, T2, Ci
            torch.cuda.empty_cache()
    finally:
        g.finalize()
