"""update_halo on ONE GPU with virtual ranks (HL_DIMS, default 2,1,1; periodic): GPU time per call of the
26-neighbour kernel (halo26 = 1) and of the per-axis P2P protocol (IGG_OPT_LOCAL_P2P), n sweep.  Separates
the kernels' own cost from cross-GPU latency (scripts/halo_sweep.py is the 2/4-GPU measurement)."""
import json, os, statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2211_15716_b200 as P

dims = tuple(int(x) for x in os.environ.get("HL_DIMS", "2,1,1").split(","))
R = dims[0] * dims[1] * dims[2]
reps = int(os.environ.get("HL_REPS", "100"))
for h26, lp in ((1, 0), (0, 1)) if not os.environ.get("HL_ONLY26") else ((1, 0),):
    for n in [int(x) for x in os.environ.get("HL_SIZES", "64,128,256,512,768").split(",")]:
        g = P.init_global_grid(n, n, n, dims=dims, periods=tuple(int(x) for x in os.environ.get("HL_PER", "1,1,1").split(",")), path="p2p", local_ranks=R, device=0)
        g.set_option(P.OPT_HALO26, h26)
        g.set_option(P.OPT_LOCAL_P2P, lp)
        g.set_option(P.OPT_HALO_STREAM, 1)
        A = [torch.rand((n, n, n), dtype=torch.float64, device="cuda") for _ in range(R)]
        for _ in range(5):
            g.update_halo(A)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        xs = []
        for _ in range(10):
            torch.cuda._sleep(100_000_000)
            e0.record()
            for _ in range(reps):
                g.update_halo(A)
            e1.record()
            torch.cuda.synchronize()
            xs.append(e0.elapsed_time(e1) / reps)
        g.check()
        ms = statistics.median(xs)
        print(json.dumps({"halo26": h26, "local_p2p": lp, "n": n, "dims": dims, "ranks": R,
                          "us_per_call": ms * 1e3, "launches_per_call": None}), flush=True)
        g.finalize()
        del A
        torch.cuda.empty_cache()
