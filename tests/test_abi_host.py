"""The C-ABI library without a GPU: it loads, exports every symbol
include/igg.h declares, and its host logic (topology math, halo geometry,
exchange plan, argument validation) agrees with the oracle.  No compute
calls are made here."""
import ctypes
import itertools
import os
import random
import re

import pytest

import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import _lib
from oracle import grid as OG

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "igg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(igg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.SO_PATH)
    names = _declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    # and the binding declares a signature for each of them
    for name in names:
        assert name in _lib.SIGNATURES or name == "igg_last_error", name


def test_library_is_sm100a_and_links_nccl():
    data = open(_lib.SO_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_dims_create_matches_oracle():
    for n in range(1, 257):
        assert P.dims_create(n) == OG.dims_create(n)
    for n, fx in [(12, (0, 0, 1)), (8, (2, 0, 0)), (16, (0, 4, 0))]:
        assert P.dims_create(n, fx) == OG.dims_create(n, fx)
    with pytest.raises(P.IggError) as e:
        P.dims_create(7, (2, 0, 0))
    assert e.value.name == "IGG_E_ARG"


def test_rank_coords_match_oracle():
    for dims in itertools.product(range(1, 4), repeat=3):
        for r in range(dims[0] * dims[1] * dims[2]):
            c = OG.coords_of_rank(r, dims)
            assert P.coords_of_rank(dims, r) == c
            assert P.rank_of_coords(dims, c) == r


def test_global_size_and_halo_spec_match_oracle():
    for n in range(4, 12):
        for o in (2, 4):
            if n <= o:
                continue
            for p in range(1, 5):
                for per in (0, 1):
                    assert P.global_size(n, o, p, per) == OG.global_size(n, o, p, per)
            for s in range(n - o, n + o + 1):
                a, b = P.halo_spec(n, o, s), OG.halo_spec(n, o, s)
                for k in b:
                    assert tuple(a[k]) == tuple(b[k]) if isinstance(b[k], tuple) else a[k] == b[k]
    with pytest.raises(P.IggError) as e:
        P.halo_spec(8, 2, 11)
    assert e.value.name == "IGG_E_STAGGER"


def _expected_faces(rank, dims, per, n, o, sizes):
    """Faces the oracle's update_halo moves for `rank`: (axis, op, field, recv_side, peer, lo, h)."""
    out = set()
    nb = OG.neighbors(rank, dims, per)
    for d in range(3):
        for f, s in enumerate(sizes):
            hs = OG.halo_spec(n[d], o[d], s[d])
            if hs["h"] == 0:
                continue
            lo_nb, up_nb = nb[d]
            if up_nb is not None:
                out.add((d, 0, f, 0, up_nb, hs["send_upper"][0], hs["h"]))
                out.add((d, 1, f, 1, up_nb, hs["recv_upper"][0], hs["h"]))
            if lo_nb is not None:
                out.add((d, 0, f, 1, lo_nb, hs["send_lower"][0], hs["h"]))
                out.add((d, 1, f, 0, lo_nb, hs["recv_lower"][0], hs["h"]))
    return out


def test_plan_faces_match_oracle_geometry():
    rng = random.Random(5)
    for _ in range(200):
        dims = tuple(rng.randint(1, 3) for _ in range(3))
        o = tuple(rng.choice((2, 4)) for _ in range(3))
        n = tuple(rng.randint(o[i] + 2, o[i] + 6) for i in range(3))
        per = tuple(rng.random() < 0.4 for _ in range(3))
        nf = rng.randint(1, 3)
        sizes = [tuple(n[i] + rng.choice((-1, 0, 1)) for i in range(3)) for _ in range(nf)]
        nprocs = dims[0] * dims[1] * dims[2]
        local = rng.choice([l for l in (1, 2, 3, 4) if nprocs % l == 0])
        rank0 = rng.randrange(0, nprocs // local) * local
        plan = P.plan_update_halo(n, dims, per, o, nprocs, rank0, local, rng.choice(("nccl", "p2p")), sizes)
        for lr in range(local):
            got = {(e["axis"], e["op"], e["field"], e["recv_side"], e["peer"], e["lo"], e["h"])
                   for e in plan if e["local_rank"] == lr}
            assert got == _expected_faces(rank0 + lr, dims, per, n, o, sizes)
        axes = [e["axis"] for e in plan]
        assert axes == sorted(axes)                      # x -> y -> z
        for e in plan:
            assert (e["transport"] == "local") == (e["peer"] // local == rank0 // local)


def test_plan_nccl_posting_orders_match_between_processes():
    """Every NCCL send of process A to B is posted at the same position as
    B's matching receive from A (NCCL matches a pair's messages in order)."""
    rng = random.Random(9)
    for _ in range(100):
        dims = tuple(rng.randint(1, 4) for _ in range(3))
        nprocs = dims[0] * dims[1] * dims[2]
        per = tuple(rng.random() < 0.5 for _ in range(3))
        n = (7, 6, 8)
        o = (2, 2, 2)
        sizes = [(7, 6, 8), (8, 6, 8)][: rng.randint(1, 2)]
        local = rng.choice([l for l in (1, 2) if nprocs % l == 0])
        procs = nprocs // local
        plans = {p: P.plan_update_halo(n, dims, per, o, nprocs, p * local, local, "nccl", sizes) for p in range(procs)}
        for a in range(3):
            for A in range(procs):
                for B in range(procs):
                    if A == B:
                        continue
                    s = sorted([e for e in plans[A] if e["axis"] == a and e["op"] == 0 and e["peer"] // local == B],
                               key=lambda e: e["order"])
                    r = sorted([e for e in plans[B] if e["axis"] == a and e["op"] == 1 and e["peer"] // local == A],
                               key=lambda e: e["order"])
                    assert len(s) == len(r)
                    for x, y in zip(s, r):
                        assert x["count"] == y["count"]
                        assert A * local + x["local_rank"] == y["peer"] and B * local + y["local_rank"] == x["peer"]
                        assert x["field"] == y["field"] and x["recv_side"] == y["recv_side"]


@pytest.mark.parametrize("kw,status", [
    (dict(n=(2, 8, 8)), "IGG_E_ARG"),                 # n <= o
    (dict(overlaps=(3, 2, 2)), "IGG_E_ARG"),          # odd overlap
    (dict(dims=(3, 1, 1)), "IGG_E_ARG"),              # dims product != nprocs
    (dict(sizes=[(5, 8, 8)]), "IGG_E_STAGGER"),       # s < n-o
    (dict(sizes=[(11, 8, 8)]), "IGG_E_STAGGER"),      # s > n+o
])
def test_validation_errors(kw, status):
    args = dict(n=(8, 8, 8), dims=(2, 1, 1), periods=(0, 0, 0), overlaps=(2, 2, 2), nprocs=2, rank0=0,
                local_ranks=1, path="nccl", sizes=[(8, 8, 8)])
    args.update(kw)
    with pytest.raises(P.IggError) as e:
        P.plan_update_halo(**args)
    assert e.value.name == status


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.IggError) as e:
        P.init_global_grid(8, 8, 8, dims=(1, 1, 1), device=0)
    assert e.value.name == "IGG_E_CUDA"


def test_missing_library_raises_instead_of_falling_back(monkeypatch):
    """The product path has no CPU fallback: without libigg.so every call
    raises ImportError (nothing routes through oracle/)."""
    monkeypatch.setattr(_lib, "SO_PATH", os.path.join(ROOT, "no_such_dir", "libigg.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError, match="no fallback"):
        _lib.lib()
    with pytest.raises(ImportError):
        P.global_size(8, 2, 2, False)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2211_15716_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f
                assert "heat3d_oracle" not in src, f


def test_save_field_writes_spec_file_format(tmp_path):
    """header "IGRIDF1 nx ny nz\\n", then the raw little-endian binary64 values, x fastest."""
    import numpy as np
    a = np.arange(3 * 4 * 5, dtype=np.float64).reshape(5, 4, 3) * 0.25 - 1.0   # (nz, ny, nx)
    p = tmp_path / "field.igf"
    P.Grid.save_field(p, a)
    raw = p.read_bytes()
    head, _, body = raw.partition(b"\n")
    assert head == b"IGRIDF1 3 4 5"
    assert np.array_equal(np.frombuffer(body, dtype="<f8"), a.ravel())
    with pytest.raises(P.IggError):
        P.Grid.save_field(tmp_path / "missing_dir" / "x.igf", a)
