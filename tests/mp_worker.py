"""Multi-GPU parity worker (launched by tests/test_gpu_multi.py with torchrun,
one process per GPU).  Every check compares the CUDA path (NCCL or P2P
transport) with the CPU oracle bit-exactly; exits non-zero on any failure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch
import torch.distributed as dist

import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import acoustic3d as ac
from paper_2211_15716_b200 import heat3d as app
from oracle import acoustic3d as OA
from oracle import grid as OG
from oracle import halo as OHL
from oracle import heat3d as OH
import synthetic_inputs as SI

DIMS = {2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
# "boot" mode: one process per GPU, no NCCL communicator at all -- the library's host collectives go
# through igg_init_args.bootstrap over a gloo group, faces by CUDA-IPC peer stores / the fused kernel.
# (Never several processes on one GPU: spinning kernels of different contexts are not co-scheduled,
# B200_PROFILING.md; ranks sharing a GPU are emulated inside one process, tests/test_gpu_virtual_p2p.py.)
BOOT = False


def device():
    return int(os.environ["LOCAL_RANK"])


def init_grid(*n, **kw):
    return P.init_global_grid(*n, device=device(), bootstrap=BOOT, **kw)


def log(*a):
    print(f"[rank {dist.get_rank()}]", *a, flush=True)


def heat_case(path, n, dims, per, local, bw, nt=8, opts=None, per_step=False):
    world = dist.get_world_size()
    g = init_grid(*n, dims=dims, periods=per, local_ranks=local, path=path)
    try:
        for k, v in (opts or {}).items():
            g.set_option(k, v)
        T, T2, Ci = app.alloc_fields(g)
        app.init_random(g, T, T2, Ci)
        d = app.spacing(g)
        dt = app.stable_dt(g, Ci, *d)
        T, T2 = app.run(g, T, T2, Ci, nt, dt, d, bw=bw, per_step=per_step)
        torch.cuda.synchronize()
        g.check()
        N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
        T0g, Cig = SI.global_heat_fields(*N)
        dref = [OH.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
        dtr = OH.stable_dt(*dref, 1.0, Cig)
        assert dt == dtr, (dt, dtr)
        ref = OH.heat_run(T0g, Cig, nt, per, 1.0, dtr, *dref, OH.CANONICAL)
        for lr in range(local):
            c = OG.coords_of_rank(g.rank0 + lr, dims)
            W = OG.window(ref, c, dims, n, (2, 2, 2), per, n)
            got = T[lr].cpu().numpy()
            if not np.array_equal(got, W):
                raise AssertionError(f"heat {path} {dims} per={per} rank {g.rank0 + lr}: "
                                     f"{int((got != W).sum())} cells differ")
    finally:
        g.finalize()
    log("heat OK", path, dims, per, "local", local, "world", world, "opts", opts, "per_step", per_step)


def halo_case(path, n, dims, per, local, sizes, seed, repeat=2):
    g = init_grid(*n, dims=dims, periods=per, local_ranks=local, path=path)
    try:
        nprocs = g.nprocs
        mine = {g.rank0 + lr: [SI.random_field(s[::-1], seed * 1000 + 10 * (g.rank0 + lr) + f)
                               for f, s in enumerate(sizes)] for lr in range(local)}
        allp = [None] * dist.get_world_size()
        dist.all_gather_object(allp, mine)
        ref = {}
        for x in allp:
            ref.update(x)
        for _ in range(repeat):
            OHL.update_halo(ref, dims, per, n, (2, 2, 2))
        dev = [[torch.from_numpy(mine[g.rank0 + lr][f]).cuda() for lr in range(local)] for f in range(len(sizes))]
        for _ in range(repeat):
            g.update_halo(*dev)
        torch.cuda.synchronize()
        g.check()
        for f in range(len(sizes)):
            for lr in range(local):
                got = dev[f][lr].cpu().numpy()
                if not np.array_equal(got, ref[g.rank0 + lr][f]):
                    raise AssertionError(f"halo {path} {dims} per={per} rank {g.rank0 + lr} field {f}")
    finally:
        g.finalize()
    log("halo OK", path, dims, per, "local", local)


def gather_case(path, n, dims, per, s):
    g = init_grid(*n, dims=dims, periods=per, path=path)
    try:
        N = [OG.field_global_size(n[i], 2, dims[i], per[i], s[i]) for i in range(3)]
        G = SI.random_field((N[2], N[1], N[0]), 77)
        W = OG.window(G, OG.coords_of_rank(g.rank0, dims), dims, n, (2, 2, 2), per, s)
        out = g.gather(torch.from_numpy(W).cuda(), root=0)
        if dist.get_rank() == 0 and not np.array_equal(out, G):
            raise AssertionError(f"gather {dims} per={per} s={s}")
    finally:
        g.finalize()
    log("gather OK", dims, per, s)


def heat_f32_case(path, n, dims, per, nt=5, bw=(16, 2, 2), opts=None):
    """The binary32 variant (igg_heat_step_f32, float halos through NCCL / NVLink) vs the binary32 oracle."""
    g = init_grid(*n, dims=dims, periods=per, local_ranks=1, path=path)
    try:
        N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
        T0g, Cig = SI.global_heat_fields(*N)
        d = [OH.spacing(1.0, N[i], bool(per[i])) for i in range(3)]
        dt = OH.stable_dt(*d, 1.0, Cig)
        for key, val in (opts or {}).items():
            g.set_option(key, val)
        T, T2, Ci = app.alloc_fields(g, dtype=torch.float32)
        app.init_random(g, T, T2, Ci)
        for _ in range(nt):
            g.heat_step(T2, T, Ci, 1.0, dt, *d, bw=bw)
            T, T2 = T2, T
        torch.cuda.synchronize()
        g.check()
        ref = OH.heat_run_f32(T0g, Cig, nt, per, 1.0, dt, *d)
        W = OG.window(ref, OG.coords_of_rank(g.rank0, dims), dims, n, (2, 2, 2), per, n)
        if not np.array_equal(T[0].cpu().numpy(), W):
            raise AssertionError(f"heat f32 {path} {dims} per={per}")
    finally:
        g.finalize()
    log("heat f32 OK", path, n, dims, per, bw)


def acoustic_case(path, n, dims, per, local, bw, nt=5):
    """Second workload: staggered P, Vx, Vy, Vz with update_halo!(Vx, Vy, Vz)."""
    g = init_grid(*n, dims=dims, periods=per, local_ranks=local, path=path)
    try:
        F = ac.alloc_fields(g)
        ac.init_random(g, F)
        d = ac.spacing(g)
        dt = ac.stable_dt(d)
        ac.run(g, F, nt, dt, d, bw=bw)
        torch.cuda.synchronize()
        g.check()
        N = tuple(OG.global_size(n[i], 2, dims[i], bool(per[i])) for i in range(3))
        ref = OA.run(*SI.global_acoustic_fields(OA.field_shapes(N, per)), nt, per, dt, ac.RHO, ac.K, *d)
        sizes = [n, (n[0] + 1, n[1], n[2]), (n[0], n[1] + 1, n[2]), (n[0], n[1], n[2] + 1)]
        for lr in range(local):
            c = OG.coords_of_rank(g.rank0 + lr, dims)
            for f in range(4):
                W = OG.window(ref[f], c, dims, n, (2, 2, 2), per, sizes[f])
                if not np.array_equal(F[f][lr].cpu().numpy(), W):
                    raise AssertionError(f"acoustic {path} {dims} per={per} rank {g.rank0 + lr} field {f}")
    finally:
        g.finalize()
    log("acoustic OK", path, dims, per, "local", local)


def full_size_case(path, dtype, nt=3):
    """The bench configuration (512^3 per GPU, dims DIMS[world], bw (16,2,2); binary64 through
    igg_heat_run -- the pipelined fused path bench.py times --, binary32 through igg_heat_step) at full
    size: sub-boxes at the exchanged faces, corners and centre are re-run by the oracle as grids of their
    own from the same seeded initial values; cells farther than nt+1 layers (the domain of dependence)
    from a sub-box edge that is not a global boundary agree bit for bit."""
    n = (512, 512, 512)
    world = dist.get_world_size()
    dims = DIMS[world]
    g = init_grid(*n, dims=dims, local_ranks=1, path=path)
    try:
        f32 = dtype == "f32"
        T, T2, Ci = app.alloc_fields(g, dtype=torch.float32 if f32 else None)
        app.init_random(g, T, T2, Ci)
        T0 = T[0].clone()
        d = app.spacing(g)
        if f32:   # dt of the float fields as the binary32 bench takes it: global max(Ci) on the device
            mx = g.global_max(float(Ci[0].max().double()))
            dt = min(x * x for x in d) / 1.0 / mx / 6.1
        else:
            dt = app.stable_dt(g, Ci, *d)
        if f32:
            for _ in range(nt):
                g.heat_step(T2, T, Ci, 1.0, dt, *d, bw=(16, 2, 2))
                T, T2 = T2, T
        else:
            T, T2 = app.run(g, T, T2, Ci, nt, dt, d, app.LAM, bw=(16, 2, 2))
        torch.cuda.synchronize()
        g.check()
        Ng = [g.n_global(a) for a in range(3)]
        gi = [g.global_indices(g.rank0, a, n[a]) for a in range(3)]
        m, L = nt + 1, 36
        for z0 in (0, 251, 512 - L):
            for y0 in (0, 300, 512 - L):
                for x0 in (0, 8, 240, 512 - L):
                    st = (z0, y0, x0)
                    box = tuple(slice(st[a], st[a] + L) for a in range(3))
                    sT0 = T0[box].cpu().numpy()
                    sC = Ci[0][box].cpu().numpy()
                    got = T[0][box].cpu().numpy()
                    if f32:
                        ref = OH.heat_run_f32(sT0, sC, nt, (0, 0, 0), 1.0, dt, *d)
                    else:
                        ref = OH.heat_run(sT0, sC, nt, (0, 0, 0), app.LAM, dt, *d, mode=OH.CANONICAL)
                    # array axis k (z, y, x) is grid axis 2-k; a side is exact where it is a global boundary
                    cut = []
                    for k in range(3):
                        a = 2 - k
                        g_lo = gi[a][st[k]]
                        g_hi = gi[a][st[k] + L - 1]
                        cut.append(slice(0 if g_lo == 0 else m, L - (0 if g_hi == Ng[a] - 1 else m)))
                    cut = tuple(cut)
                    if not np.array_equal(ref[cut], got[cut]):
                        raise AssertionError(f"full-size {dtype} {path} rank {g.rank0} box {st}")
    finally:
        g.finalize()
    log("full-size OK", dtype, path, dims)


def boot_cases(world):
    """One process per GPU with the host bootstrap instead of an NCCL communicator: the fused
    stencil+NVLink-put kernel (default), the split pack/flag/unpack path, staggered update_halo, the
    acoustic step, binary32, gather and global_max through the bootstrap -- bit-exact vs the oracle."""
    dims = DIMS[world]
    n = (40, 36, 34)
    sizes = [n, (41, 36, 34), (40, 37, 34), (40, 36, 35)]
    path = "p2p"
    heat_case(path, (130, 36, 34), dims, (0, 0, 0), 1, (16, 2, 2), nt=4)                 # fused, pipelined
    heat_case(path, (130, 36, 34), dims, (1, 1, 1), 1, (16, 2, 2), nt=4)                 # + periodic, corners
    heat_case(path, (130, 36, 34), dims, (1, 1, 1), 1, (16, 2, 2), nt=3, per_step=True)  # single drained steps
    heat_case(path, n, dims, (0, 0, 0), 1, (16, 2, 2), nt=3, opts={P.OPT_FUSED: 0})     # split P2P path
    heat_case(path, (130, 36, 34), dims, (1, 0, 1), 1, (16, 2, 2), nt=3, opts={P.OPT_FUSED: 0})
    for d2 in {2: [(1, 2, 1), (1, 1, 2)], 4: [(1, 2, 2)]}.get(world, []):
        heat_case(path, (130, 36, 34), d2, (1, 1, 1), 1, (16, 2, 2), nt=3)
    halo_case(path, n, dims, (0, 0, 0), 1, sizes, seed=1)
    halo_case(path, n, dims, (1, 1, 1), 1, sizes, seed=2)
    acoustic_case(path, n, dims, (0, 0, 0), 1, (16, 4, 4), nt=3)
    heat_f32_case(path, n, dims, (1, 0, 1), nt=3)
    if 8 % world == 0 and world < 8:   # 2x2x2 as virtual ranks over the processes
        heat_case(path, (24, 20, 18), (2, 2, 2), (0, 0, 0), 8 // world, (4, 2, 2), nt=3)
    gather_case(path, (20, 18, 16), dims, (1, 0, 1), (20, 17, 16))


def main():
    global BOOT
    BOOT = len(sys.argv) > 2 and sys.argv[2] == "boot"
    torch.cuda.set_device(device())
    if BOOT:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", device()))
    world = dist.get_world_size()
    paths = sys.argv[1].split(",") if len(sys.argv) > 1 else ["nccl", "p2p"]
    if BOOT:
        boot_cases(world)
        dist.barrier()
        if dist.get_rank() == 0:
            print("BOOTSTRAP PARITY OK", world, flush=True)
        dist.destroy_process_group()
        return
    if len(sys.argv) > 2 and sys.argv[2] == "full":   # the bench configuration at full size
        for dtype in ("f64", "f32"):
            full_size_case(paths[0], dtype)
        dist.barrier()
        if dist.get_rank() == 0:
            print("MULTI-GPU FULL-SIZE OK", world, paths, flush=True)
        dist.destroy_process_group()
        return
    dims = DIMS[world]
    n = (40, 36, 34)
    sizes = [n, (41, 36, 34), (40, 37, 34), (40, 36, 35)]
    for path in paths:
        heat_case(path, n, dims, (0, 0, 0), 1, (16, 2, 2))
        heat_case(path, n, dims, (1, 0, 1), 1, (4, 2, 2))
        heat_case(path, (130, 36, 34), dims, (0, 0, 0), 1, (16, 2, 2))
        if path == "p2p":   # the fused stencil+exchange kernel is the p2p default; also check the split path
            for o in ({P.OPT_FUSED: 0}, {P.OPT_FUSED: 0, P.OPT_SCHEDULE: 1}):
                heat_case(path, n, dims, (0, 0, 0), 1, (16, 2, 2), opts=o)
                heat_case(path, (130, 36, 34), dims, (1, 1, 1), 1, (16, 2, 2), opts=o)
            heat_case(path, (130, 36, 34), dims, (1, 1, 1), 1, (16, 2, 2), nt=12)
            heat_case(path, (66, 40, 36), dims, (0, 1, 0), 1, (16, 2, 2), nt=9)
            # single igg_heat_step calls (each drained)
            heat_case(path, (130, 36, 34), dims, (1, 1, 1), 1, (16, 2, 2), nt=5, per_step=True)
            heat_case(path, (130, 36, 70), dims, (1, 0, 1), 1, (16, 2, 2), nt=5, per_step=True)
            # the fused put path on every split axis (z faces, corner forwarding x->y->z)
            extra = {2: [(1, 2, 1), (1, 1, 2)], 4: [(2, 1, 2), (1, 2, 2), (4, 1, 1), (1, 1, 4)]}.get(world, [])
            for d2 in extra:
                heat_case(path, (130, 36, 34), d2, (0, 0, 0), 1, (16, 2, 2), nt=7)
                heat_case(path, (130, 36, 34), d2, (1, 1, 1), 1, (16, 2, 2), nt=7)
        halo_case(path, n, dims, (0, 0, 0), 1, sizes, seed=1)
        acoustic_case(path, n, dims, (0, 0, 0), 1, (16, 4, 4))
        heat_f32_case(path, n, dims, (1, 0, 1))
        heat_f32_case(path, (520, 20, 34), dims, (0, 0, 0), bw=(16, 2, 2))   # hide_communication, float4 kernel
        if path == "p2p" and world == 2:
            # y / z splits: the 26-neighbour exchange beside a long inner-box kernel (the counter-reset
            # race of the exchange's last block showed up exactly here as flag timeouts)
            for d2 in ((1, 1, 2), (1, 2, 1)):
                heat_f32_case(path, (256, 256, 256), d2, (0, 0, 0), bw=(16, 2, 2), nt=12)
        heat_f32_case(path, (264, 36, 34), dims, (1, 1, 0), bw=(0, 0, 0))
        acoustic_case(path, n, dims, (1, 0, 1), 1, (4, 4, 4))
        halo_case(path, n, dims, (1, 1, 1), 1, sizes, seed=2)
        # 8 ranks as virtual ranks over the processes (2x2x2 correctness on fewer GPUs)
        if 8 % world == 0 and world < 8:
            heat_case(path, (24, 20, 18), (2, 2, 2), (0, 0, 0), 8 // world, (4, 2, 2))
            halo_case(path, (24, 20, 18), (2, 2, 2), (1, 0, 1), 8 // world,
                      [(24, 20, 18), (25, 20, 18), (24, 21, 18), (24, 20, 19)], seed=3)
    gather_case(paths[0], (20, 18, 16), dims, (0, 0, 0), (21, 18, 16))
    gather_case(paths[0], (20, 18, 16), dims, (1, 0, 1), (20, 17, 16))
    dist.barrier()
    if dist.get_rank() == 0:
        print("MULTI-GPU PARITY OK", world, paths, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
