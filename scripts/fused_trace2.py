"""Diagnostics on 2 GPUs (torchrun, ablation/libigg_trace*.so): per-block %globaltimer stamps of one
steady-state fused launch at 512^3 per GPU, dims 2x1x1 (remote x faces), with and without the exchange;
each rank saves its stamps (gpurun_out/trace2_r<rank>_<skip>.npz)."""
import ctypes, os, sys
sys.path.insert(0, ".")
os.environ.setdefault("IGG_LIBRARY", "ablation/libigg_trace.so")
import numpy as np
import torch
import torch.distributed as dist
import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import heat3d as app
from paper_2211_15716_b200 import _lib

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
L = _lib.lib()
L.igg_debug_fused_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.igg_debug_trace_epoch.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
n = 512
dims = tuple(int(x) for x in os.environ.get("TRACE_DIMS", "2,1,1").split(","))
g = P.init_global_grid(n, n, n, dims=dims, path="p2p", device=local)
T, T2, Ci = app.alloc_fields(g)
app.init_paper(g, T, T2, Ci)
d = app.spacing(g)
dt = app.stable_dt(g, Ci, *d)
T, T2 = app.run(g, T, T2, Ci, 5, dt, d)
torch.cuda.synchronize()
for skip in (0, 1):
    L.igg_debug_trace_epoch(g._handle(), 6)
    if skip:
        g.set_option(P.OPT_SKIP_COMM, 1)
    dist.barrier()
    T, T2 = app.run(g, T, T2, Ci, 10, dt, d)
    torch.cuda.synchronize()
    g.set_option(P.OPT_SKIP_COMM, 0)
    nb = 16384
    buf = (ctypes.c_ulonglong * (4 * nb))()
    L.igg_debug_fused_trace(ctypes.cast(buf, ctypes.c_void_p), nb)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(nb, 4).astype(np.int64)
    a = a[a[:, 0] > 0]
    np.savez_compressed(f"gpurun_out/trace2_r{dist.get_rank()}_{skip}.npz", a=a)
    print(dist.get_rank(), skip, "span_us", (a[:, 3].max() - a[:, 0].min()) / 1e3, flush=True)
try:
    g.check()
except P.IggError:
    pass
g.finalize()
dist.destroy_process_group()
