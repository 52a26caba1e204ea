"""Diagnostics (ablation/libigg_trace.so, built with -DFUSED_TRACE=1): per-block %globaltimer stamps of
one steady-state fused launch at 512^3 with periodic axes wrapping onto the one GPU; prints, per setting,
the launch span, how the stencil tiles' durations split by kind (plain / x-halo / x-send / y-face /
z-face) and the timing of the last wave."""
import ctypes, json, os, sys
sys.path.insert(0, ".")
os.environ.setdefault("IGG_LIBRARY", "ablation/libigg_trace.so")
import numpy as np
import torch
import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import heat3d as app
from paper_2211_15716_b200 import _lib

L = _lib.lib()
L.igg_debug_fused_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.igg_debug_trace_epoch.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
n = int(os.environ.get("TRACE_N", "512"))
for per in [(1, 0, 0), (0, 1, 0), (0, 0, 1)]:
    g = P.init_global_grid(n, n, n, periods=per, path="p2p", device=0)
    T, T2, Ci = app.alloc_fields(g)
    app.init_paper(g, T, T2, Ci)
    d = app.spacing(g)
    dt = app.stable_dt(g, Ci, *d)
    T, T2 = app.run(g, T, T2, Ci, 5, dt, d)
    torch.cuda.synchronize()
    for skip in (0, 1):
        L.igg_debug_trace_epoch(g._handle(), 6)      # the 6th step of the next run: steady state
        if skip:
            g.set_option(P.OPT_SKIP_COMM, 1)
        T, T2 = app.run(g, T, T2, Ci, 10, dt, d)
        torch.cuda.synchronize()
        g.set_option(P.OPT_SKIP_COMM, 0)
        nb = 16384
        buf = (ctypes.c_ulonglong * (4 * nb))()
        L.igg_debug_fused_trace(ctypes.cast(buf, ctypes.c_void_p), nb)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(nb, 4).astype(np.int64)
        used = a[:, 0] > 0
        a = a[used]
        t0 = a[:, 0].min()
        st, sw, en = a[:, 0] - t0, a[:, 1] - t0, a[:, 3] - t0
        dur = en - st
        nbk = len(a)
        xt = 8
        idx = np.nonzero(used)[0]
        tx = idx % xt
        np.savez_compressed(f"gpurun_out/trace_{''.join(map(str, per))}_{skip}.npz", a=a, idx=idx)
        rec = {"periods": per, "skip_comm": skip, "blocks": int(nbk), "span_us": float(en.max() / 1e3),
               "median_block_us": float(np.median(dur) / 1e3),
               "tx0_us": float(np.median(dur[tx == 0]) / 1e3), "tx7_us": float(np.median(dur[tx == 7]) / 1e3),
               "mid_us": float(np.median(dur[(tx > 0) & (tx < 7)]) / 1e3),
               "last_start_us": float(st.max() / 1e3),
               "epilogue_us_median": float(np.median((en - sw)[sw > 0]) / 1e3)}
        print(json.dumps(rec), flush=True)
    g.finalize()
    del T, T2, Ci
    torch.cuda.empty_cache()
