"""update_halo bandwidth sweep (config B:11 analogue): one periodic field of n^3
per GPU, dims 2x1x1 / 2x2x1 (/2x2x2), NCCL vs P2P; time per call (max over
ranks, CUDA events) and GB/s of halo payload each GPU sends per call."""
import json, os, sys
sys.path.insert(0, ".")
import torch
import torch.distributed as dist
import paper_2211_15716_b200 as P

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
world = dist.get_world_size()
dims = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}[world]
out = []
variants = [("nccl", 0, 1), ("p2p", 0, 1), ("p2p", 1, 1), ("p2p", 1, 0)]   # (path, caller stream, coop)
for path, on_caller, coop in variants:
    for n in (64, 96, 128, 192, 256, 384, 512, 640, 768):
        g = P.init_global_grid(n, n, n, dims=dims, periods=(1, 1, 1), path=path, device=local)
        g.set_option(P.igg.OPT_HALO_STREAM, on_caller)
        g.set_option(P.igg.OPT_COOP_HALO, coop)
        A = torch.rand((n, n, n), dtype=torch.float64, device="cuda")
        for _ in range(10):
            g.update_halo(A)
        torch.cuda.synchronize(); dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(40_000_000)   # keep the GPU busy while the host enqueues: GPU time only
        e0.record()
        for _ in range(100):
            g.update_halo(A)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 100], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        remote_axes = sum(1 for d in dims if d > 1)
        sent = remote_axes * 2 * n * n * 8   # bytes this GPU sends to other GPUs per call
        out.append({"path": path, "caller_stream": on_caller, "coop": coop, "n": n, "dims": dims, "ms_per_call": ms, "remote_bytes": sent,
                    "GBps_per_gpu": sent / (ms * 1e-3) / 1e9})
        g.finalize()
        del A
        torch.cuda.empty_cache()
if dist.get_rank() == 0:
    for r in out:
        print(json.dumps(r))
dist.destroy_process_group()
