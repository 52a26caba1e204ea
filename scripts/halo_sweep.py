"""update_halo bandwidth sweep (config B:11 analogue): one periodic field of n^3 per GPU, dims by world
size (2: 2x1x1, 4: 2x2x1, 8: 2x2x2), transports: NCCL (per-axis grouped send/recv), P2P per-axis
pack/flag/unpack, and P2P 26-neighbour single kernel (default).  20 samples of 100 calls each (median),
CUDA events on the calling stream, max over ranks; GB/s per GPU = bytes this GPU sends to OTHER GPUs per
call / t; 'payload' also counts the faces a rank stores into itself (periodic self-wrap axes)."""
import json, os, statistics, sys, time
sys.path.insert(0, ".")
import torch
import torch.distributed as dist
import paper_2211_15716_b200 as P

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
world = dist.get_world_size()
dims = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}[world]
sizes = [int(x) for x in os.environ.get("HALO_SIZES", "64,96,128,192,256,384,512,640,768").split(",")]
out = []
variants = [("nccl", 0), ("p2p", 0), ("p2p", 1)]   # (path, halo26)
for path, h26 in variants:
    for n in sizes:
        g = P.init_global_grid(n, n, n, dims=dims, periods=(1, 1, 1), path=path, device=local)
        g.set_option(P.OPT_HALO26, h26)
        g.set_option(P.OPT_HALO_STREAM, 1)   # on the caller's stream (no event joins)
        A = torch.rand((n, n, n), dtype=torch.float64, device="cuda")
        for _ in range(10):
            g.update_halo(A)
        torch.cuda.synchronize(); dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        xs, host_us = [], []
        for rep in range(20):
            dist.barrier(); torch.cuda.synchronize()
            torch.cuda._sleep(200_000_000)   # the GPU stays busy while the host enqueues: GPU time only
            h0 = time.perf_counter()
            e0.record()
            for _ in range(100):
                g.update_halo(A)
            e1.record()
            host_us.append((time.perf_counter() - h0) * 1e4)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 100], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            xs.append(float(t.item()))
        g.check()
        ms = statistics.median(xs)
        remote_axes = sum(1 for d in dims if d > 1)
        sent = remote_axes * 2 * n * n * 8   # face bytes this GPU sends to other GPUs per call
        out.append({"path": path, "halo26": h26, "n": n, "dims": dims, "ms_per_call_median": ms,
                    "ms_min": min(xs), "remote_bytes": sent, "GBps_per_gpu": sent / (ms * 1e-3) / 1e9,
                    "payload_GBps": 6 * n * n * 8 / (ms * 1e-3) / 1e9,
                    "host_enqueue_us_per_call": statistics.median(host_us)})
        g.finalize()
        del A
        torch.cuda.empty_cache()
if dist.get_rank() == 0:
    for r in out:
        print(json.dumps(r))
dist.destroy_process_group()
