"""Real multi-GPU parity (one process per GPU, torchrun, NCCL and P2P
transports) -- runs only on a box with >= 2 GPUs (gpurun --gpus 2/4)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("path", ["nccl", "p2p"])
def test_torchrun_parity(path):
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "mp_worker.py"), path]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    sys.stdout.write(r.stdout[-4000:])
    sys.stderr.write(r.stderr[-4000:])
    assert r.returncode == 0
    assert "MULTI-GPU PARITY OK" in r.stdout


def test_torchrun_full_size_bench_config():
    """512^3 per GPU in the bench's launch configuration (fused pipelined binary64 run, binary32 step),
    sampled sub-boxes vs the oracle (tests/mp_worker.py full_size_case)."""
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "mp_worker.py"),
           "p2p", "full"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    sys.stdout.write(r.stdout[-4000:])
    sys.stderr.write(r.stderr[-4000:])
    assert r.returncode == 0
    assert "MULTI-GPU FULL-SIZE OK" in r.stdout


def test_torchrun_bootstrap_no_nccl():
    """One process per GPU with igg_init_args.bootstrap (host collectives over a gloo group, NO NCCL
    communicator): the P2P data planes and the collective utilities bit-exact vs the oracle
    (tests/mp_worker.py boot_cases).  Ranks that share a GPU are covered on one GPU by
    tests/test_gpu_virtual_p2p.py (emulated in one process: spinning kernels of different processes on
    one GPU are not co-scheduled)."""
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "mp_worker.py"),
           "p2p", "boot"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    sys.stdout.write(r.stdout[-4000:])
    sys.stderr.write(r.stderr[-4000:])
    assert r.returncode == 0
    assert "BOOTSTRAP PARITY OK" in r.stdout
