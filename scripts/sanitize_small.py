"""Small single-GPU workload for compute-sanitizer: every kernel family of the
single-process paths (box, box-list, slab, generic region kernels, local
pack/unpack, max reduction) on 2 and 8 virtual ranks."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import heat3d as app

def heat(n, dims, per, bw, kernel, xalign, sched):
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=dims[0] * dims[1] * dims[2], device=0)
    g.set_option(P.OPT_STENCIL_KERNEL, kernel)
    g.set_option(P.OPT_X_ALIGN, xalign)
    g.set_option(P.OPT_SCHEDULE, sched)
    T, T2, Ci = app.alloc_fields(g)
    app.init_random(g, T, T2, Ci)
    d = app.spacing(g)
    dt = app.stable_dt(g, Ci, *d)
    app.run(g, T, T2, Ci, 3, dt, d, bw=bw)
    torch.cuda.synchronize()
    g.check()
    g.finalize()

heat((70, 20, 18), (2, 1, 1), (0, 0, 0), (16, 2, 2), 0, 1, 0)
heat((70, 20, 18), (2, 1, 1), (1, 0, 0), (16, 2, 2), 0, 64, 1)
heat((34, 20, 18), (2, 2, 2), (0, 1, 0), (4, 2, 2), 1, 1, 0)
heat((34, 20, 18), (2, 1, 1), (0, 0, 0), (4, 2, 2), 8, 1, 0)
heat((33, 20, 18), (1, 1, 1), (0, 0, 0), (0, 0, 0), 0, 1, 0)
g = P.init_global_grid(12, 10, 9, dims=(2, 2, 2), periods=(1, 0, 1), local_ranks=8, device=0)
fs = [[torch.rand(s[::-1], dtype=torch.float64, device="cuda") for _ in range(8)]
      for s in [(12, 10, 9), (13, 10, 9), (12, 11, 9), (12, 10, 10)]]
g.update_halo(*fs)
torch.cuda.synchronize()
g.finalize()
print("SANITIZE WORKLOAD OK")
