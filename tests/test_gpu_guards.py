"""Out-of-bounds and determinism checks of every kernel family (compute-sanitizer is closed on the GPU
pool, profiles/r02_sanitizer_unavailable.txt): each field the library writes is a view into a larger
allocation whose guard zones (64 KiB before and after) hold a sentinel bit pattern; after the run every
guard must be intact, and a second identical run must give identical bits (a shared-memory or flag race
would show up as run-to-run differences on random inputs).  Library-internal buffers (staging, arenas,
flags) are sized by the library; these cases exercise their edges through small, ragged shapes."""
import numpy as np
import pytest

import paper_2211_15716_b200 as P
from paper_2211_15716_b200 import acoustic3d as ac
from paper_2211_15716_b200 import heat3d as app

pytestmark = pytest.mark.gpu

GUARD = 8192
SENT = {8: -1.2345678901234567e300, 4: -1.2345678e30}   # by element size


class Guarded:
    def __init__(self):
        self.bigs = []

    def field(self, shape, dtype):
        import torch
        n = int(np.prod(shape))
        big = torch.full((n + 2 * GUARD,), SENT[torch.empty((), dtype=dtype).element_size()], dtype=dtype,
                         device="cuda")
        self.bigs.append(big)
        return big[GUARD:GUARD + n].view(shape)

    def check(self):
        import torch
        torch.cuda.synchronize()
        for big in self.bigs:
            s = torch.tensor(SENT[big.element_size()], dtype=big.dtype)
            lo, hi = big[:GUARD].cpu(), big[-GUARD:].cpu()
            assert bool((lo == s).all()) and bool((hi == s).all()), "a kernel wrote outside a field"


def _heat(n, dims, per, nt, per_step=False, options=None, dtype=None):
    import torch
    R = dims[0] * dims[1] * dims[2]
    G = Guarded()
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=R, device=0, path="p2p")
    try:
        for k, v in (options or {}).items():
            g.set_option(k, v)
        dt_ = dtype or torch.float64
        shape = (n[2], n[1], n[0])
        T, T2, Ci = ([G.field(shape, dt_) for _ in range(R)] for _ in range(3))
        app.init_random(g, T, T2, Ci)
        d = app.spacing(g)
        if dtype is None:
            dt = app.stable_dt(g, Ci, *d)
            T, T2 = app.run(g, T, T2, Ci, nt, dt, d, per_step=per_step)
        else:
            for _ in range(nt):
                g.heat_step(T2, T, Ci, 1.0, 1e-5, *d)
                T, T2 = T2, T
        torch.cuda.synchronize()
        g.check()
        G.check()
        return [t.cpu().numpy().copy() for t in T]
    finally:
        g.finalize()


@pytest.mark.parametrize("n,dims,per,per_step", [
    ((130, 20, 22), (2, 2, 2), (1, 0, 1), False),   # fused: x/y/z faces, forwarders, deferred x chunks
    ((130, 20, 22), (2, 2, 2), (0, 1, 0), True),
    ((194, 17, 37), (2, 1, 2), (1, 1, 1), False),   # ragged y/z, three x tiles
    ((66, 36, 34), (2, 2, 1), (0, 1, 0), False),    # two x tiles: every tile a border tile
])
def test_fused_guards_and_determinism(n, dims, per, per_step):
    a = _heat(n, dims, per, 6, per_step=per_step)
    b = _heat(n, dims, per, 6, per_step=per_step)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("n,dims,per,opts", [
    ((70, 20, 18), (2, 1, 1), (1, 0, 0), {P.OPT_FUSED: 0}),                         # split + halo26
    ((40, 20, 18), (2, 2, 1), (1, 0, 1), {P.OPT_FUSED: 0, P.OPT_LOCAL_P2P: 1}),     # per-axis P2P
    ((33, 21, 19), (1, 1, 1), (0, 0, 0), {}),                                       # odd rows: generic kernel
])
def test_split_schedule_guards(n, dims, per, opts):
    a = _heat(n, dims, per, 4, per_step=True, options=opts)
    b = _heat(n, dims, per, 4, per_step=True, options=opts)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("fused", [0, 1])
def test_binary32_guards(fused):
    import torch
    o = {P.OPT_FUSED_F32: fused}
    a = _heat((260, 20, 18), (2, 1, 1), (0, 1, 0), 3, dtype=torch.float32, options=o)
    b = _heat((260, 20, 18), (2, 1, 1), (0, 1, 0), 3, dtype=torch.float32, options=o)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("dims,per", [((2, 2, 2), (1, 0, 1)), ((3, 1, 2), (0, 1, 1))])
def test_staggered_update_halo_guards(dims, per):
    import torch
    n = (14, 11, 9)
    R = dims[0] * dims[1] * dims[2]
    sizes = [n, (n[0] + 1, n[1], n[2]), (n[0], n[1] + 1, n[2]), (n[0], n[1], n[2] + 1)]
    G = Guarded()
    g = P.init_global_grid(*n, dims=dims, periods=per, local_ranks=R, device=0, path="p2p")
    try:
        gen = torch.Generator(device="cuda").manual_seed(5)
        fs = []
        for s in sizes:
            lst = []
            for _ in range(R):
                v = G.field(s[::-1], torch.float64)
                v.copy_(torch.rand(s[::-1], dtype=torch.float64, device="cuda", generator=gen))
                lst.append(v)
            fs.append(lst)
        for _ in range(3):
            g.update_halo(*fs)
        g.check()
        G.check()
    finally:
        g.finalize()


def test_acoustic_guards():
    import torch
    G = Guarded()
    g = P.init_global_grid(70, 20, 37, device=0)
    try:
        F = [[G.field(tuple(s), torch.float64)] for s in ac.shapes(g)]
        F2 = [[G.field(tuple(s), torch.float64)] for s in ac.shapes(g)]
        ac.init_random(g, F)
        d = ac.spacing(g)
        A, _ = g.acoustic_run(F, F2, 3, ac.stable_dt(d), ac.RHO, ac.K, *d)
        g.check()
        G.check()
    finally:
        g.finalize()
