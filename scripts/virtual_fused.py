"""One GPU, two virtual ranks of 512^3 (dims from VF_DIMS, default 2,1,1) in the fused kernel: the
cross-rank data plane (x staging, x senders, y/z peer stores, flags) between sibling ranks in one launch.
For ncu (`-k regex:heat_fused`): DRAM bytes of a launch covering both ranks (per rank: half)."""
import os
import sys
sys.path.insert(0, ".")
import torch
import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import heat3d as app

dims = tuple(int(x) for x in os.environ.get("VF_DIMS", "2,1,1").split(","))
R = dims[0] * dims[1] * dims[2]
n = int(os.environ.get("VF_N", "512"))
g = P.init_global_grid(n, n, n, dims=dims, local_ranks=R, device=0, path="p2p")
T, T2, Ci = app.alloc_fields(g)
app.init_paper(g, T, T2, Ci)
d = app.spacing(g)
dt = app.stable_dt(g, Ci, *d)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
T, T2 = app.run(g, T, T2, Ci, 5, dt, d)
torch.cuda.synchronize()
nt = int(os.environ.get("VF_NT", "20"))
s.record()
T, T2 = app.run(g, T, T2, Ci, nt, dt, d)
e.record()
torch.cuda.synchronize()
g.check()
print(f"virtual fused dims {dims} n {n}: {s.elapsed_time(e) / nt:.4f} ms per step for {R} ranks")
g.finalize()
