"""Probe: update_halo cost of one 512^3 field with a periodic self-wrap on one GPU."""
import sys, time, json
sys.path.insert(0, ".")
import torch
import paper_2211_15716_b200 as P
axes = sys.argv[1] if len(sys.argv) > 1 else "1,0,0"
per = tuple(int(v) for v in axes.split(","))
n = 512
g = P.init_global_grid(n, n, n, dims=(1, 1, 1), periods=per, device=0)
A = torch.rand((n, n, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    g.update_halo(A)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    g.update_halo(A)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"periods": per, "ms_per_update_halo": e0.elapsed_time(e1) / 20}))
g.finalize()
