"""Python binding of libigg (include/igg.h): same names, argument marshalling only.

Every step of the hot path (stencil, pack/unpack, exchange, scheduling) runs
in libigg's CUDA kernels and C++ host code.  PyTorch supplies device memory
(tensors), the caller's stream and the process group used to broadcast the
NCCL unique id.

The three functions of the paper: ``init_global_grid`` (listing
23), ``Grid.update_halo`` (listing 38) and
``Grid.finalize_global_grid`` (listing 43), plus ``nx_g()``
``ny_g()`` ``nz_g()`` and the fused hide_communication heat
step.
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

from . import _lib as L

PATH_NCCL = 0
PATH_P2P = 1
_PATHS = {"nccl": PATH_NCCL, "p2p": PATH_P2P}

OPT_SKIP_COMM = 1
OPT_SPIN_TIMEOUT_MS = 2
OPT_STENCIL_KERNEL = 3
OPT_PROFILE = 4
OPT_X_ALIGN = 5
OPT_SCHEDULE = 6
OPT_FUSED = 7
OPT_FUSED_MODE = 8
OPT_FUSED_KC2 = 9
OPT_FUSED_COMM_CTAS = 10
OPT_HALO_STREAM = 12
OPT_LOCAL_P2P = 13
OPT_HALO26 = 14
OPT_FUSED_F32 = 15

STATUS = {0: "IGG_OK", 1: "IGG_E_ARG", 2: "IGG_E_STATE", 3: "IGG_E_STAGGER", 4: "IGG_E_WIDTH",
          5: "IGG_E_CUDA", 6: "IGG_E_NCCL", 7: "IGG_E_TIMEOUT", 8: "IGG_E_UNSUPPORTED", 9: "IGG_E_BOOTSTRAP"}


class IggError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


def _ok(rc: int) -> None:
    if rc != 0:
        raise IggError(rc, L.lib().igg_last_error().decode(errors="replace"))


def _i3(v) -> ctypes.Array:
    return (ctypes.c_int * 3)(*[int(x) for x in v])


# ------------------------------------------------------------------ host-only topology math
def dims_create(nprocs: int, fixed=(0, 0, 0)) -> tuple:
    out = (ctypes.c_int * 3)()
    _ok(L.lib().igg_dims_create(nprocs, _i3(fixed), out))
    return tuple(out)


def rank_of_coords(dims, coords) -> int:
    r = ctypes.c_int()
    _ok(L.lib().igg_rank_of_coords(_i3(dims), _i3(coords), ctypes.byref(r)))
    return r.value


def coords_of_rank(dims, rank: int) -> tuple:
    out = (ctypes.c_int * 3)()
    _ok(L.lib().igg_coords_of_rank(_i3(dims), rank, out))
    return tuple(out)


def global_size(n: int, o: int, p: int, periodic: bool) -> int:
    out = ctypes.c_longlong()
    _ok(L.lib().igg_global_size(n, o, p, int(bool(periodic)), ctypes.byref(out)))
    return out.value


def halo_spec(n: int, o: int, s: int) -> dict:
    hs = L.igg_halo_spec()
    _ok(L.lib().igg_halo_spec_of(n, o, s, ctypes.byref(hs)))
    return dict(ol=hs.ol, h=hs.h, send_lower=tuple(hs.send_lower), recv_lower=tuple(hs.recv_lower),
                send_upper=tuple(hs.send_upper), recv_upper=tuple(hs.recv_upper))


def _init_args(nx, ny, nz, dims, periods, overlaps, nprocs, rank0, local_ranks, device, path):
    a = L.igg_init_args()
    a.nx, a.ny, a.nz = nx, ny, nz
    for i in range(3):
        a.dims[i], a.periods[i], a.overlaps[i] = int(dims[i]), int(bool(periods[i])), int(overlaps[i])
    a.nprocs, a.rank0, a.local_ranks, a.device = nprocs, rank0, local_ranks, device
    a.path = _PATHS[path] if isinstance(path, str) else int(path)
    return a


TRANSPORTS = {0: "local", 1: "nccl", 2: "p2p"}


def plan_update_halo(n, dims, periods, overlaps, nprocs: int, rank0: int, local_ranks: int, path, sizes) -> list:
    """Host-only exchange plan of one update_halo call of a process (igg_plan_update_halo).
    sizes: list of (sx, sy, sz) per field.  Returns a list of dicts in execution order."""
    a = _init_args(*n, dims, periods, overlaps, nprocs, rank0, local_ranks, 0, path)
    sz = (ctypes.c_longlong * (3 * len(sizes)))(*[int(v) for s in sizes for v in s])
    cnt = ctypes.c_int()
    _ok(L.lib().igg_plan_update_halo(ctypes.byref(a), sz, len(sizes), None, 0, ctypes.byref(cnt)))
    out = (L.igg_plan_entry * max(cnt.value, 1))()
    _ok(L.lib().igg_plan_update_halo(ctypes.byref(a), sz, len(sizes), out, cnt.value, ctypes.byref(cnt)))
    keys = [k for k, _ in L.igg_plan_entry._fields_]
    res = [{k: getattr(out[i], k) for k in keys} for i in range(cnt.value)]
    for e in res:
        e["transport"] = TRANSPORTS[e["transport"]]
    return res


def get_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _ok(L.lib().igg_get_unique_id(buf))
    return bytes(buf)


# ------------------------------------------------------------------ tensors
def _as_list(x, n: int) -> list:
    lst = list(x) if isinstance(x, (list, tuple)) else [x]
    if len(lst) != n:
        raise ValueError(f"expected {n} per-rank tensors, got {len(lst)}")
    return lst


def _dev_ptr(t, allow_f32: bool = False) -> int:
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("fields must be torch tensors")
    ok_dtype = t.dtype == torch.float64 or (allow_f32 and t.dtype == torch.float32)
    if not t.is_cuda or not ok_dtype or not t.is_contiguous() or t.dim() != 3:
        raise ValueError("fields must be contiguous 3-D float64%s CUDA tensors of shape (sz, sy, sx)"
                         % (" or float32" if allow_f32 else ""))
    return t.data_ptr()


def _elsize(t) -> int:
    return t.element_size()


def _ptr_array(ts) -> ctypes.Array:
    return (ctypes.c_void_p * len(ts))(*[_dev_ptr(t) for t in ts])


def _stream(stream) -> int:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


# ------------------------------------------------------------------ the grid
class Grid:
    """A live implicit global grid (one process, `local_ranks` ranks on one GPU)."""

    def __init__(self, handle, me, coords, dims, n_g, n, overlaps, periods, nprocs, rank0, local_ranks, path):
        self._h = handle
        self.me, self.coords, self.dims, self.n_g = me, coords, dims, n_g
        self.n, self.overlaps, self.periods = n, overlaps, periods
        self.nprocs, self.rank0, self.local_ranks, self.path = nprocs, rank0, local_ranks, path

    # -- queries
    def _handle(self):
        if self._h is None:
            raise IggError(2, "grid already finalized")
        return self._h

    def n_global(self, axis: int, field_size: int = 0) -> int:
        out = ctypes.c_longlong()
        _ok(L.lib().igg_n_g(self._handle(), axis, field_size, ctypes.byref(out)))
        return out.value

    def nx_g(self, field_size: int = 0) -> int:
        return self.n_global(0, field_size)

    def ny_g(self, field_size: int = 0) -> int:
        return self.n_global(1, field_size)

    def nz_g(self, field_size: int = 0) -> int:
        return self.n_global(2, field_size)

    def coords_of(self, rank: int) -> tuple:
        out = (ctypes.c_int * 3)()
        _ok(L.lib().igg_coords(self._handle(), rank, out))
        return tuple(out)

    def local_to_global(self, rank: int, axis: int, l: int) -> int:
        out = ctypes.c_longlong()
        _ok(L.lib().igg_local_to_global(self._handle(), rank, axis, l, ctypes.byref(out)))
        return out.value

    def global_coord(self, rank: int, axis: int, l: int, spacing: float) -> float:
        """Physical coordinate of local layer l: igg_global_coord."""
        out = ctypes.c_double()
        _ok(L.lib().igg_global_coord(self._handle(), rank, axis, l, float(spacing), ctypes.byref(out)))
        return out.value

    def global_indices(self, rank: int, axis: int, size: int):
        import numpy as np
        return np.array([self.local_to_global(rank, axis, l) for l in range(size)], dtype=np.int64)

    def buffer_allocs(self) -> int:
        out = ctypes.c_longlong()
        _ok(L.lib().igg_buffer_allocs(self._handle(), ctypes.byref(out)))
        return out.value

    def kernel_launches(self) -> int:
        out = ctypes.c_longlong()
        _ok(L.lib().igg_kernel_launches(self._handle(), ctypes.byref(out)))
        return out.value

    # -- update_halo!
    def update_halo(self, *fields, stream=None) -> None:
        """Each field: a tensor (one local rank) or a list of local_ranks tensors."""
        per = [_as_list(f, self.local_ranks) for f in fields]
        nf = len(per)
        arr = (L.igg_field * (nf * self.local_ranks))()
        for r in range(self.local_ranks):
            for f in range(nf):
                t = per[f][r]
                e = arr[r * nf + f]
                e.ptr = _dev_ptr(t, allow_f32=True)   # binary64 or binary32
                e.elsize = _elsize(t)
                sz, sy, sx = t.shape
                e.size[0], e.size[1], e.size[2] = sx, sy, sz
        _ok(L.lib().igg_update_halo(self._handle(), arr, nf, _stream(stream)))

    # -- @hide_communication bw begin step!; update_halo!(T2) end
    def heat_step(self, T2, T, Ci, lam: float, dt: float, dx: float, dy: float, dz: float,
                  bw=(16, 2, 2), stream=None) -> None:
        n = self.local_ranks
        t2, t, c = (_as_list(x, n) for x in (T2, T, Ci))
        import torch
        if t2[0].dtype == torch.float32:   # the binary32 variant (igg_heat_step_f32)
            for x in t2 + t + c:
                if tuple(x.shape) != (self.n[2], self.n[1], self.n[0]) or x.dtype != torch.float32:
                    raise ValueError("binary32 heat_step fields must be float32 of the canonical local shape")
            arr = lambda ts: (ctypes.c_void_p * len(ts))(*[_dev_ptr(q, allow_f32=True) for q in ts])
            _ok(L.lib().igg_heat_step_f32(self._handle(), arr(t2), arr(t), arr(c), lam, dt, dx, dy, dz, _i3(bw),
                                          _stream(stream)))
            return
        for x in t2 + t + c:
            if tuple(x.shape) != (self.n[2], self.n[1], self.n[0]):
                raise ValueError("heat_step fields must have the canonical local shape (nz, ny, nx)")
        _ok(L.lib().igg_heat_step(self._handle(), _ptr_array(t2), _ptr_array(t), _ptr_array(c),
                                  lam, dt, dx, dy, dz, _i3(bw), _stream(stream)))

    def heat_run(self, T, T2, Ci, lam: float, dt: float, dx: float, dy: float, dz: float, nt: int,
                 bw=(16, 2, 2), stream=None):
        """Fig. 1's time loop on the device (igg_heat_run): nt steps with the swap; returns the lists
        (T, T2) after the swaps (T = the state after nt steps)."""
        n = self.local_ranks
        t, t2, c = (_as_list(x, n) for x in (T, T2, Ci))
        import torch
        f32 = t[0].dtype == torch.float32   # the binary32 variant (igg_heat_run_f32)
        for x in t2 + t + c:
            if tuple(x.shape) != (self.n[2], self.n[1], self.n[0]) or (f32 and x.dtype != torch.float32):
                raise ValueError("heat_run fields must have the canonical local shape (nz, ny, nx) and one dtype")
        if f32:
            arr = lambda ts: (ctypes.c_void_p * len(ts))(*[_dev_ptr(q, allow_f32=True) for q in ts])
            _ok(L.lib().igg_heat_run_f32(self._handle(), arr(t), arr(t2), arr(c), lam, dt, dx, dy, dz, int(nt),
                                         _i3(bw), _stream(stream)))
        else:
            _ok(L.lib().igg_heat_run(self._handle(), _ptr_array(t), _ptr_array(t2), _ptr_array(c), lam, dt, dx,
                                     dy, dz, int(nt), _i3(bw), _stream(stream)))
        swapped = nt % 2 == 1
        return (list(t2), list(t)) if swapped else (list(t), list(t2))

    def heat_run_host(self, T_host, Ci_host, lam, dt, dx, dy, dz, nt: int, bw=(16, 2, 2), stream=None) -> None:
        """Fig. 1 end to end from host memory (numpy arrays or CPU tensors, ideally pinned);
        T_host is overwritten with the final T."""
        def hp(a):
            if hasattr(a, "data_ptr"):
                assert not a.is_cuda and a.is_contiguous() and str(a.dtype) == "torch.float64"
                return a.data_ptr()
            assert a.dtype.name == "float64" and a.flags.c_contiguous
            return a.ctypes.data
        _ok(L.lib().igg_heat_run_host(self._handle(), hp(T_host), hp(Ci_host), lam, dt, dx, dy, dz, nt,
                                      _i3(bw), _stream(stream)))

    # -- second workload: staggered acoustic leapfrog step
    def acoustic_step(self, P, Vx, Vy, Vz, dt: float, rho: float, K: float, dx: float, dy: float, dz: float,
                      bw=(16, 4, 4), stream=None) -> None:
        """@hide_communication bw begin compute_V!; update_halo!(Vx,Vy,Vz) end; compute_P! (include/igg.h)."""
        n = self.local_ranks
        nx, ny, nz = self.n
        want = [(nz, ny, nx), (nz, ny, nx + 1), (nz, ny + 1, nx), (nz + 1, ny, nx)]
        lists = [_as_list(x, n) for x in (P, Vx, Vy, Vz)]
        for f, lst in enumerate(lists):
            for x in lst:
                if tuple(x.shape) != want[f]:
                    raise ValueError(f"acoustic_step field {f} must have shape {want[f]}, got {tuple(x.shape)}")
        _ok(L.lib().igg_acoustic_step(self._handle(), *(_ptr_array(l) for l in lists), dt, rho, K, dx, dy, dz,
                                      _i3(bw), _stream(stream)))

    def acoustic_run(self, F, F2, nt: int, dt: float, rho: float, K: float, dx: float, dy: float, dz: float,
                     bw=(16, 4, 4), stream=None):
        """nt steps with double-buffered fields (igg_acoustic_run): F, F2 = [P, Vx, Vy, Vz] lists of local_ranks
        tensors each; returns (F, F2) after the run (F = the state after nt steps)."""
        n = self.local_ranks
        nx, ny, nz = self.n
        want = [(nz, ny, nx), (nz, ny, nx + 1), (nz, ny + 1, nx), (nz + 1, ny, nx)]
        sets = [[_as_list(x, n) for x in F], [_as_list(x, n) for x in F2]]
        for S in sets:
            for f, lst in enumerate(S):
                for x in lst:
                    if tuple(x.shape) != want[f]:
                        raise ValueError(f"acoustic_run field {f} must have shape {want[f]}, got {tuple(x.shape)}")
        flat = [t for S in sets for lst in S for t in lst]
        arr = (ctypes.c_void_p * len(flat))(*[_dev_ptr(t) for t in flat])
        _ok(L.lib().igg_acoustic_run(self._handle(), arr, int(nt), dt, rho, K, dx, dy, dz, _i3(bw), _stream(stream)))
        by_ptr = {t.data_ptr(): t for t in flat}
        out = [by_ptr[arr[q]] for q in range(len(flat))]
        h = 4 * n
        first = [out[f * n:(f + 1) * n] for f in range(4)]
        second = [out[h + f * n:h + (f + 1) * n] for f in range(4)]
        return first, second

    # -- generic @hide_communication
    def hide_communication(self, bw, step, *fields, stream=None) -> None:
        """Run a user stencil `step(local_rank, lo, hi, stream)` -- which must enqueue the computation of
        the box [lo, hi) on the given torch stream -- with the boundary slabs first and update_halo(fields)
        overlapped with the inner box.  bw = (0, 0, 0): sequential."""
        import torch
        per = [_as_list(f, self.local_ranks) for f in fields]
        nf = len(per)
        arr = (L.igg_field * (nf * self.local_ranks))()
        for r in range(self.local_ranks):
            for f in range(nf):
                t = per[f][r]
                e = arr[r * nf + f]
                e.ptr = _dev_ptr(t, allow_f32=True)
                e.elsize = _elsize(t)
                sz, sy, sx = t.shape
                e.size[0], e.size[1], e.size[2] = sx, sy, sz
        streams = {}
        errors = []

        def _cb(user, lr, lo, hi, st):
            try:
                if st not in streams:
                    streams[st] = torch.cuda.ExternalStream(st)
                s_ = streams[st]
                with torch.cuda.stream(s_):
                    step(lr, (lo[0], lo[1], lo[2]), (hi[0], hi[1], hi[2]), s_)
            except Exception as ex:  # never raise through C
                errors.append(ex)

        cb = L.REGION_FN(_cb)
        _ok(L.lib().igg_hide_communication(self._handle(), _i3(bw), cb, None, arr, nf, _stream(stream)))
        if errors:
            raise errors[0]

    # -- gather
    def gather(self, field, root: int = 0, stream=None):
        """Global field (numpy, (Nz, Ny, Nx)) assembled on process `root` from the owned layers of every
        rank; None on other processes.  field: a tensor or a list of local_ranks tensors."""
        import numpy as np
        ts = _as_list(field, self.local_ranks)
        arr = (L.igg_field * self.local_ranks)()
        for r, t in enumerate(ts):
            arr[r].ptr = _dev_ptr(t)
            sz, sy, sx = t.shape
            arr[r].size[0], arr[r].size[1], arr[r].size[2] = sx, sy, sz
        sz, sy, sx = ts[0].shape
        shape = (self.n_global(2, sz), self.n_global(1, sy), self.n_global(0, sx))
        me_root = (self.rank0 // self.local_ranks) == root
        out = np.empty(shape, dtype=np.float64) if me_root else None
        _ok(L.lib().igg_gather(self._handle(), arr, root, out.ctypes.data if me_root else None, _stream(stream)))
        return out

    @staticmethod
    def save_field(path: str, array) -> None:
        """Write a gathered global field (numpy (Nz, Ny, Nx) float64) as SPEC.md:410's file: header
        "IGRIDF1 nx ny nz", then the raw little-endian binary64 values (igg_save_field)."""
        import numpy as np
        a = np.ascontiguousarray(array, dtype=np.float64)
        n = (ctypes.c_longlong * 3)(a.shape[2], a.shape[1], a.shape[0])
        _ok(L.lib().igg_save_field(str(path).encode(), a.ctypes.data, n))

    # -- reductions
    def global_max(self, local: float) -> float:
        out = ctypes.c_double()
        _ok(L.lib().igg_global_max(self._handle(), float(local), ctypes.byref(out)))
        return out.value

    def field_global_max(self, f, stream=None) -> float:
        ts = _as_list(f, self.local_ranks)
        out = ctypes.c_double()
        _ok(L.lib().igg_field_global_max(self._handle(), _ptr_array(ts), ts[0].numel(), ctypes.byref(out),
                                         _stream(stream)))
        return out.value

    # -- control
    def set_option(self, key: int, value: int) -> None:
        _ok(L.lib().igg_set_option(self._handle(), key, int(value)))

    def profile_stencil(self) -> tuple:
        """(ms_total, launches, cells) of the profiled main stencil launches; resets."""
        ms, n, c = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_longlong()
        _ok(L.lib().igg_profile_stencil(self._handle(), ctypes.byref(ms), ctypes.byref(n), ctypes.byref(c)))
        return ms.value, n.value, c.value

    def profile_timeline(self) -> dict:
        """Average overlap timeline (ms from step start) recorded with OPT_PROFILE = 2; resets."""
        out = (ctypes.c_double * 5)()
        _ok(L.lib().igg_profile_timeline(self._handle(), out))
        return dict(boundary_done=out[0], inner_start=out[1], inner_done=out[2], exchange_done=out[3],
                    steps=int(out[4]))

    def check(self) -> None:
        _ok(L.lib().igg_check(self._handle()))

    def release_arrays(self) -> None:
        """Collective: drop the peers' mappings of T / T2 arrays (igg_release_arrays); call before freeing
        arrays used in heat steps on the fused P2P path."""
        _ok(L.lib().igg_release_arrays(self._handle()))

    # -- finalize_global_grid
    def finalize_global_grid(self) -> None:
        _ok(L.lib().igg_finalize_global_grid(self._handle()))
        self._h = None

    finalize = finalize_global_grid


def _gloo_bootstrap(group):
    """The host all-gather of igg_init_args.bootstrap over a gloo process group (argument marshalling:
    bytes in, bytes out)."""
    import torch
    dist = torch.distributed
    world = dist.get_world_size(group)

    def _cb(user, mine, out, nbytes):
        try:
            t = torch.frombuffer(bytearray(ctypes.string_at(mine, nbytes)), dtype=torch.uint8)
            parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, t, group=group)
            ctypes.memmove(out, b"".join(p.numpy().tobytes() for p in parts), nbytes * world)
            return 0
        except Exception:   # never raise through C; the library reports IGG_E_BOOTSTRAP
            return 1
    return L.ALLGATHER_FN(_cb)


def init_global_grid(nx: int, ny: int, nz: int, dims=(0, 0, 0), periods=(0, 0, 0), overlaps=(2, 2, 2),
                     path: str = "nccl", local_ranks: int = 1, device: int | None = None,
                     process_group=None, bootstrap: bool = False) -> Grid:
    """init_global_grid.  With torch.distributed initialised and
    world size > 1 this is collective: process 0's NCCL unique id is broadcast
    over the process group (gloo or nccl).  bootstrap=True (path "p2p" only):
    no NCCL communicator; the library's host collectives run over a gloo
    group of the processes (igg_init_args.bootstrap) -- which also lets
    several processes share one GPU."""
    import torch
    world, prank = 1, 0
    dist = torch.distributed
    if dist.is_available() and dist.is_initialized():
        world = dist.get_world_size(process_group)
        prank = dist.get_rank(process_group)
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", torch.cuda.current_device() if torch.cuda.is_available() else 0))
    a = _init_args(nx, ny, nz, dims, periods, overlaps, world * local_ranks, prank * local_ranks, local_ranks,
                   device, path)
    boot_cb = None
    if world > 1 and bootstrap:
        group = process_group
        if dist.get_backend(group) != "gloo":
            group = dist.new_group(ranks=list(range(world)), backend="gloo")
        boot_cb = _gloo_bootstrap(group)
        a.bootstrap = ctypes.cast(boot_cb, ctypes.c_void_p)
    elif world > 1:
        obj = [get_unique_id() if prank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=process_group)
        ctypes.memmove(a.comm_id, obj[0], 128)
    h = ctypes.c_void_p()
    me = ctypes.c_int()
    c = (ctypes.c_int * 3)()
    d = (ctypes.c_int * 3)()
    ng = (ctypes.c_longlong * 3)()
    _ok(L.lib().igg_init_global_grid(ctypes.byref(a), ctypes.byref(h), ctypes.byref(me), c, d, ng))
    g = Grid(h, me.value, tuple(c), tuple(d), tuple(ng), (nx, ny, nz), tuple(int(x) for x in overlaps),
             tuple(int(bool(p)) for p in periods), a.nprocs, a.rank0, local_ranks, a.path)
    g._boot_cb = boot_cb   # the library calls it until finalize
    return g
