"""Config B:10: the staggered 4-field update_halo(P, Vx, Vy, Vz) on the 2x2x2 topology, n = 512 (P n^3,
Vx (n+1) n n, Vy, Vz), non-periodic and periodic: time per call (median of 20 samples of 20 calls, max
over processes) and GB/s = 24.02 MiB / t (the bytes one rank of 2x2x2 sends per call).
Eight ranks as local_ranks = 8 / world per process (labelled: ranks on one GPU exchange through that
GPU's memory, ranks on different GPUs over NVLink)."""
import json, os, statistics, sys
sys.path.insert(0, ".")
import torch
import torch.distributed as dist
import paper_2211_15716_b200 as P

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
world = int(os.environ.get("WORLD_SIZE", "1"))
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = int(os.environ.get("B10_N", "512"))
L = 8 // world
res = []
for per in ((0, 0, 0), (1, 1, 1)):
    for path, h26 in (("p2p", 1), ("p2p", 0), ("nccl", 0)):
        g = P.init_global_grid(n, n, n, dims=(2, 2, 2), periods=per, path=path, local_ranks=L, device=local)
        g.set_option(P.OPT_HALO26, h26)
        g.set_option(P.OPT_HALO_STREAM, 1)
        shapes = [(n, n, n), (n, n, n + 1), (n, n + 1, n), (n + 1, n, n)]
        F = [[torch.rand(s, dtype=torch.float64, device="cuda") for _ in range(L)] for s in shapes]
        for _ in range(5):
            g.update_halo(*F)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        xs = []
        for rep in range(20):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda._sleep(100_000_000)
            e0.record()
            for _ in range(20):
                g.update_halo(*F)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 20], device="cuda")
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            xs.append(float(t.item()))
        g.check()
        ms = statistics.median(xs)
        mib = 24.02
        res.append({"config": "B:10 staggered update_halo(P,Vx,Vy,Vz) 2x2x2", "n": n, "periods": per,
                    "path": path, "halo26": h26, "processes": world, "ranks_per_gpu": L,
                    "ms_per_call_median": ms, "ms_min": min(xs), "GBps_24.02MiB": mib * 2 ** 20 / (ms * 1e-3) / 1e9})
        g.finalize()
        del F
        torch.cuda.empty_cache()
if local == 0 and (world == 1 or dist.get_rank() == 0):
    for r in res:
        print(json.dumps(r))
if world > 1:
    dist.destroy_process_group()
