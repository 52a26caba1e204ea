"""Small single-GPU workload for compute-sanitizer (one tool per run: memcheck, racecheck, synccheck):
every kernel family of the single-process paths on virtual ranks -- the fused stencil + peer-store
kernel over several ranks in one launch (flags, staging, forwarders, drain), the 26-neighbour
update_halo kernel, the per-axis P2P protocol (IGG_OPT_LOCAL_P2P), the split schedule's box-list / slab /
generic region kernels, the acoustic kernels (split step and fused run), the binary32 kernels, the max reduction."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import acoustic3d as ac
from paper_2211_15716_b200 import heat3d as app


def heat(n, dims, per, bw, path="nccl", opts=None, per_step=False, nt=3, dtype=None):
    R = dims[0] * dims[1] * dims[2]
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=R, device=0, path=path)
    for k, v in (opts or {}).items():
        g.set_option(k, v)
    T, T2, Ci = app.alloc_fields(g, dtype=dtype)
    app.init_random(g, T, T2, Ci)
    d = app.spacing(g)
    if dtype is None:
        dt = app.stable_dt(g, Ci, *d)
        app.run(g, T, T2, Ci, nt, dt, d, bw=bw, per_step=per_step)
    else:
        for _ in range(nt):
            g.heat_step(T2, T, Ci, 1.0, 1e-5, *d, bw=bw)
            T, T2 = T2, T
    torch.cuda.synchronize()
    g.check()
    g.finalize()


# fused kernel: several ranks in one launch, x/y/z faces, periodic, pipelined and single steps
heat((130, 20, 22), (2, 2, 2), (0, 0, 0), (16, 2, 2), path="p2p")
heat((130, 20, 22), (2, 1, 2), (1, 1, 0), (16, 2, 2), path="p2p", per_step=True)
heat((130, 20, 22), (1, 1, 1), (1, 1, 1), (16, 2, 2), path="p2p")
# split schedule with the 26-neighbour update_halo, and with the per-axis P2P protocol
heat((70, 20, 18), (2, 1, 1), (0, 0, 0), (16, 2, 2), opts={P.OPT_X_ALIGN: 1})
heat((70, 20, 18), (2, 1, 1), (1, 0, 0), (16, 2, 2), opts={P.OPT_SCHEDULE: 1})
heat((34, 20, 18), (2, 2, 2), (0, 1, 0), (4, 2, 2), opts={P.OPT_STENCIL_KERNEL: 1, P.OPT_X_ALIGN: 1})
heat((40, 20, 18), (2, 2, 1), (1, 0, 1), (4, 2, 2), path="p2p",
     opts={P.OPT_FUSED: 0, P.OPT_LOCAL_P2P: 1, P.OPT_X_ALIGN: 1})
heat((33, 20, 18), (1, 1, 1), (0, 0, 0), (0, 0, 0))
heat((132, 20, 18), (2, 1, 1), (0, 1, 0), (0, 0, 0), dtype=torch.float32)
# staggered update_halo (config B:10's field set), 26-neighbour kernel
g = P.init_global_grid(12, 10, 9, dims=(2, 2, 2), periods=(1, 0, 1), local_ranks=8, device=0)
fs = [[torch.rand(s[::-1], dtype=torch.float64, device="cuda") for _ in range(8)]
      for s in [(12, 10, 9), (13, 10, 9), (12, 11, 9), (12, 10, 10)]]
g.update_halo(*fs)
g.update_halo(*fs)
torch.cuda.synchronize()
g.check()
g.finalize()
# acoustic step on 2 ranks
g = P.init_global_grid(20, 18, 16, dims=(2, 1, 1), local_ranks=2, device=0)
F = ac.alloc_fields(g)
ac.init_random(g, F)
d = ac.spacing(g)
ac.run(g, F, 2, ac.stable_dt(d), d, bw=(4, 4, 4))
torch.cuda.synchronize()
g.check()
g.finalize()
# acoustic run on one rank: the fused V+P sweep (double-buffered)
g = P.init_global_grid(70, 20, 37, device=0)
F, F2 = ac.alloc_fields(g), ac.alloc_fields(g)
ac.init_random(g, F)
d = ac.spacing(g)
g.acoustic_run(F, F2, 3, ac.stable_dt(d), ac.RHO, ac.K, *d)
torch.cuda.synchronize()
g.check()
g.finalize()
print("SANITIZE WORKLOAD OK")
