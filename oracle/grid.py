"""oracle/grid.py -- CPU ORACLE for the implicit global grid (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg may import this module; it shares no code with the product.

The paper states that the global grid is implied by
the local grid and the process topology, and queries it with nx_g()/ny_g()/nz_g().
It never writes the formulas; the readings below are SPEC.md's (listed in
DESIGN.md "Readings of the paper"):

  * dims_create        -- SPEC.md:37-46   (reading 4)
  * rank <-> coords    -- SPEC.md:47-55   (reading 5: last axis fastest)
  * neighbours         -- SPEC.md:56-64
  * global size        -- SPEC.md:97-98   (reading 1)
  * halo_spec          -- SPEC.md:186-207 (reading 13/14)
  * local_to_global    -- SPEC.md:119-127, periodic shift (reading 15)
  * window             -- the local array a rank must hold for a global array:
                          SURVEY.md 8(c) step 7.

All indices here are 0-based unless a name says otherwise.
"""
from __future__ import annotations

import itertools

import numpy as np

AXES = ("x", "y", "z")


# --------------------------------------------------------------------------- topology
def dims_create(nprocs: int, fixed=(0, 0, 0)) -> tuple:
    """among all ordered factorisations (px,py,pz) of nprocs that
    honour the fixed (non-zero) entries, the one minimising max-min; ties go to
    the lexicographically largest vector."""
    if nprocs < 1:
        raise ValueError("nprocs must be >= 1")
    best = None
    for px in range(1, nprocs + 1):
        for py in range(1, nprocs + 1):
            if nprocs % (px * py):
                continue
            pz = nprocs // (px * py)
            d = (px, py, pz)
            if any(f and f != v for f, v in zip(fixed, d)):
                continue
            key = (max(d) - min(d), tuple(-v for v in d))
            if best is None or key < best[0]:
                best = (key, d)
    if best is None:
        raise ValueError(f"no factorisation of {nprocs} honours fixed={fixed}")
    return best[1]


def rank_of_coords(coords, dims) -> int:
    """rank = (cx*py + cy)*pz + cz."""
    cx, cy, cz = coords
    px, py, pz = dims
    if not (0 <= cx < px and 0 <= cy < py and 0 <= cz < pz):
        raise IndexError("coords out of bounds")
    return (cx * py + cy) * pz + cz


def coords_of_rank(rank: int, dims) -> tuple:
    px, py, pz = dims
    if not 0 <= rank < px * py * pz:
        raise IndexError("rank out of bounds")
    return (rank // (py * pz), (rank // pz) % py, rank % pz)


def neighbors(rank: int, dims, periodic) -> list:
    """per axis (lower, upper); None at a non-periodic edge."""
    c = coords_of_rank(rank, dims)
    out = []
    for d in range(3):
        pair = []
        for step in (-1, +1):
            cc = list(c)
            cc[d] += step
            if 0 <= cc[d] < dims[d]:
                pair.append(rank_of_coords(cc, dims))
            elif periodic[d]:
                cc[d] %= dims[d]
                pair.append(rank_of_coords(cc, dims))
            else:
                pair.append(None)
        out.append(tuple(pair))
    return out


# --------------------------------------------------------------------------- global sizes
def global_size(n: int, o: int, p: int, periodic: bool) -> int:
    """n_g = p(n-o)+o (non-periodic), p(n-o) (periodic)."""
    return p * (n - o) if periodic else p * (n - o) + o


def field_global_size(n: int, o: int, p: int, periodic: bool, s: int) -> int:
    """Distinct global layers of a (staggered) field of local size s: the
    canonical n_g shifted by s-n on a non-periodic axis; the period on a
    periodic axis (reading 1)."""
    return p * (n - o) if periodic else p * (n - o) + o + (s - n)


def local_to_global(c: int, n: int, o: int, l: int, periodic: bool = False, P: int = 0) -> int:
    """0-based local layer l of a rank at axis coordinate c -> 0-based global layer.
    SPEC.md:122 (1-based g = l + c(n-o)); periodic: shifted by o/2 and wrapped
    mod the period P (reading 15)."""
    g = c * (n - o) + l
    if periodic:
        g = (g - o // 2) % P
    return g


# --------------------------------------------------------------------------- halo geometry
def halo_spec(n: int, o: int, s: int) -> dict:
    """ol = s-(n-o), h = floor(ol/2); 0-based half-open ranges
    send_lower [ol-h, ol), recv_lower [0, h), send_upper [s-ol, s-ol+h),
    recv_upper [s-h, s).  Raises on s < n-o or s > n+o."""
    if s < n - o or s > n + o:
        raise ValueError(f"staggered size {s} outside [{n - o}, {n + o}]")
    ol = s - (n - o)
    h = ol // 2
    return dict(ol=ol, h=h,
                send_lower=(ol - h, ol), recv_lower=(0, h),
                send_upper=(s - ol, s - ol + h), recv_upper=(s - h, s))


# --------------------------------------------------------------------------- windows
def window(G: np.ndarray, coords, dims, n, o, periodic, s) -> np.ndarray:
    """The local array (shape (s_z,s_y,s_x)) that rank `coords` holds of a global
    field G (shape (Nz,Ny,Nx), x fastest) -- every layer, halos included."""
    idx = []
    for d in range(3):  # d: 0=x,1=y,2=z
        P = global_size(n[d], o[d], dims[d], True)
        idx.append(np.array([local_to_global(coords[d], n[d], o[d], l, periodic[d], P)
                             for l in range(s[d])], dtype=np.int64))
    return G[np.ix_(idx[2], idx[1], idx[0])].copy()


def layer_sets(n, o, p, periodic, s):
    """For tests: the set of global layers each axis coordinate covers."""
    P = global_size(n, o, p, True)
    return [sorted({local_to_global(c, n, o, l, periodic, P) for l in range(s)}) for c in range(p)]


def all_coords(dims):
    return list(itertools.product(range(dims[0]), range(dims[1]), range(dims[2])))
