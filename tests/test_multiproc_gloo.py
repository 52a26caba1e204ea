"""World-size-2 test of the multi-process host logic on CPU (gloo).

Two processes each ask libigg for their exchange plan (igg_plan_update_halo,
the same host code the GPU path executes) and carry it out with numpy copies
and torch.distributed gloo send/recv posted in the plan's NCCL order on ONE
tag -- the same in-order matching NCCL applies.  The resulting arrays must
equal the oracle's update_halo on all ranks' data (bit-exact)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slab(A, axis, lo, h):
    sl = [slice(None)] * 3
    sl[2 - axis] = slice(lo, lo + h)
    return tuple(sl)


def _worker(proc, nproc, port, cfg, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=proc, world_size=nproc)
    try:
        import paper_2211_15716_b200 as P
        import synthetic_inputs as SI
        n, dims, per, o, local, sizes = cfg["n"], cfg["dims"], cfg["per"], cfg["o"], cfg["local"], cfg["sizes"]
        nprocs = dims[0] * dims[1] * dims[2]
        rank0 = proc * local
        fields = {lr: [SI.random_field(tuple(s[::-1]), 97 * (rank0 + lr) + f) for f, s in enumerate(sizes)]
                  for lr in range(local)}
        before = {lr: [a.copy() for a in fields[lr]] for lr in fields}
        plan = P.plan_update_halo(n, dims, per, o, nprocs, rank0, local, "nccl", sizes)
        for axis in range(3):
            msgs = [e for e in plan if e["axis"] == axis]
            inbox = {}
            sends = sorted([e for e in msgs if e["op"] == 0 and e["transport"] == "nccl"], key=lambda e: e["order"])
            recvs = sorted([e for e in msgs if e["op"] == 1 and e["transport"] == "nccl"], key=lambda e: e["order"])
            for e in msgs:                                   # pack (all before any unpack)
                if e["op"] == 0:
                    buf = np.ascontiguousarray(fields[e["local_rank"]][e["field"]][_slab(None, axis, e["lo"], e["h"])])
                    assert buf.size == e["count"]
                    if e["transport"] == "local":
                        inbox[(e["peer"] - rank0, e["field"], e["recv_side"])] = buf
                    else:
                        e["buf"] = torch.from_numpy(buf.reshape(-1).copy())
            reqs = []
            for e in sends:
                reqs.append(dist.isend(e["buf"], dst=e["peer"] // local, tag=0))
            for e in recvs:
                e["buf"] = torch.empty(e["count"], dtype=torch.float64)
                reqs.append(dist.irecv(e["buf"], src=e["peer"] // local, tag=0))
            for r in reqs:
                r.wait()
            for e in msgs:                                   # unpack
                if e["op"] != 1:
                    continue
                A = fields[e["local_rank"]][e["field"]]
                tgt = A[_slab(None, axis, e["lo"], e["h"])]
                if e["transport"] == "local":
                    data = inbox[(e["local_rank"], e["field"], e["recv_side"])]
                else:
                    data = e["buf"].numpy().reshape(tgt.shape)
                A[_slab(None, axis, e["lo"], e["h"])] = data
        allb = [None] * nproc
        alla = [None] * nproc
        dist.all_gather_object(allb, {rank0 + lr: before[lr] for lr in before})
        dist.all_gather_object(alla, {rank0 + lr: fields[lr] for lr in fields})
        if proc == 0:
            from oracle import halo as OH
            ref = {}
            for d in allb:
                ref.update(d)
            got = {}
            for d in alla:
                got.update(d)
            OH.update_halo(ref, dims, per, n, o)
            ok = all(np.array_equal(ref[r][f], got[r][f]) for r in ref for f in range(len(sizes)))
            q.put(ok)
    except Exception as ex:  # report, never hang the parent
        q.put(repr(ex))
        raise
    finally:
        dist.destroy_process_group()


CASES = [
    dict(n=(8, 7, 6), dims=(2, 1, 1), per=(0, 0, 0), o=(2, 2, 2), local=1, sizes=[(8, 7, 6)]),
    dict(n=(8, 7, 6), dims=(2, 1, 1), per=(1, 0, 1), o=(2, 2, 2), local=1, sizes=[(8, 7, 6), (9, 7, 6)]),
    dict(n=(9, 8, 7), dims=(2, 2, 1), per=(1, 1, 0), o=(2, 4, 2), local=2,
         sizes=[(9, 8, 7), (10, 8, 7), (9, 9, 7), (9, 8, 8)]),
]


@pytest.mark.parametrize("cfg", CASES)
def test_two_process_plan_exchange_matches_oracle(cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(p, 2, port, cfg, q)) for p in range(2)]
    for p in ps:
        p.start()
    try:
        res = q.get(timeout=240)
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert res is True, res
