"""2-process check of the split schedule on the P2P path (torchrun): SC_DIMS, SC_DTYPE (f64/f32),
SC_H26 (1: 26-neighbour update_halo, 0: per-axis), SC_FUSED (IGG_OPT_FUSED), SC_N, SC_BW; 20 steps, then
igg_check; prints the per-step time or the error."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import torch.distributed as dist
import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import heat3d as app

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
dims = tuple(int(x) for x in os.environ.get("SC_DIMS", "1,2,1").split(","))
n = int(os.environ.get("SC_N", "256"))
bw = tuple(int(x) for x in os.environ.get("SC_BW", "16,2,2").split(","))
f32 = os.environ.get("SC_DTYPE", "f32") == "f32"
g = P.init_global_grid(n, n, n, dims=dims, path="p2p", device=local)
g.set_option(P.OPT_HALO26, int(os.environ.get("SC_H26", "1")))
g.set_option(P.OPT_FUSED, int(os.environ.get("SC_FUSED", "0")))
g.set_option(P.OPT_SPIN_TIMEOUT_MS, 3000)
T, T2, Ci = app.alloc_fields(g, dtype=torch.float32 if f32 else None)
app.init_paper(g, T, T2, Ci)
d = app.spacing(g)
dist.barrier()
t0 = time.perf_counter()
try:
    for _ in range(20):
        if os.environ.get("SC_MODE") == "halo":   # update_halo alone
            g.update_halo(T2)
        else:
            g.heat_step(T2, T, Ci, 1.0, 1e-6, *d, bw=bw)
            T, T2 = T2, T
    torch.cuda.synchronize()
    g.check()
    res = f"OK {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms/step (wall)"
except Exception as e:
    res = f"FAIL {e}"
print(f"rank {dist.get_rank()} {os.environ.get('SC_MODE', 'step')} dims {dims} {'f32' if f32 else 'f64'} h26 {os.environ.get('SC_H26', '1')} "
      f"fused {os.environ.get('SC_FUSED', '0')} n {n} bw {bw}: {res}", flush=True)
g.finalize()
dist.destroy_process_group()
