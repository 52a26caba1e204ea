"""Diagnostics (ablation/libigg_h26trace.so, -DH26_TRACE=1): per-block %globaltimer stamps of one
26-neighbour update_halo launch on one GPU (virtual ranks): start, loop exit, after flush, end, and the
wait for the data flag.  Env: HT_DIMS, HT_PER, HT_N."""
import ctypes, os, sys
sys.path.insert(0, ".")
os.environ.setdefault("IGG_LIBRARY", "ablation/libigg_h26trace.so")
import numpy as np
import torch
import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import _lib

L = _lib.lib()
L.igg_debug_h26_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
dims = tuple(int(x) for x in os.environ.get("HT_DIMS", "1,1,1").split(","))
per = tuple(int(x) for x in os.environ.get("HT_PER", "1,1,1").split(","))
n = int(os.environ.get("HT_N", "64"))
R = dims[0] * dims[1] * dims[2]
g = P.init_global_grid(n, n, n, dims=dims, periods=per, path="p2p", local_ranks=R, device=0)
g.set_option(P.OPT_HALO_STREAM, 1)
A = [torch.rand((n, n, n), dtype=torch.float64, device="cuda") for _ in range(R)]
for _ in range(5):
    g.update_halo(A)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8 * 4096))()
L.igg_debug_h26_trace(ctypes.cast(buf, ctypes.c_void_p), 4096)
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
info = int(a[0, 7])
print(f"dims {dims} per {per} n {n}: blocks {len(a)} nchunks {info & 0xFFFFF} nstore {(info >> 20) & 0xFFFFF} "
      f"nitems {info >> 40}")
for b, r in enumerate(a):
    f = lambda k: (r[k] - t0) / 1e3 if r[k] > 0 else -1
    print(f"block {b:3d}: start {f(0):7.2f} wait {f(5):7.2f}->{f(6):7.2f} loop_exit {f(2):7.2f} "
          f"flushed {f(3):7.2f} end {f(4):7.2f}")
g.check()
g.finalize()
