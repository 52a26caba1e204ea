"""ctypes declarations of libigg.so (include/igg.h).  Argument marshalling only.

The library is built in-tree (``paper_2211_15716_b200/libigg.so``, see
``build.py``).  If it is missing this module raises: the product path has no
fallback of any kind.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# IGG_LIBRARY: load another build of the same ABI (A/B timing of two builds on one box)
SO_PATH = os.environ.get("IGG_LIBRARY") or os.path.join(HERE, "libigg.so")

c_int_p = ctypes.POINTER(ctypes.c_int)
c_ll_p = ctypes.POINTER(ctypes.c_longlong)
c_dbl_p = ctypes.POINTER(ctypes.c_double)
c_dbl_pp = ctypes.POINTER(ctypes.c_void_p)


class igg_init_args(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("dims", ctypes.c_int * 3), ("periods", ctypes.c_int * 3), ("overlaps", ctypes.c_int * 3),
                ("nprocs", ctypes.c_int), ("rank0", ctypes.c_int), ("local_ranks", ctypes.c_int),
                ("device", ctypes.c_int), ("path", ctypes.c_int), ("reserved", ctypes.c_int),
                ("comm_id", ctypes.c_ubyte * 128), ("bootstrap", ctypes.c_void_p),
                ("bootstrap_user", ctypes.c_void_p)]


# int (*igg_allgather_fn)(void *user, const void *mine, void *all, unsigned long long bytes)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_ulonglong)


class igg_field(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("size", ctypes.c_longlong * 3), ("elsize", ctypes.c_int)]


class igg_halo_spec(ctypes.Structure):
    _fields_ = [("ol", ctypes.c_int), ("h", ctypes.c_int),
                ("send_lower", ctypes.c_int * 2), ("recv_lower", ctypes.c_int * 2),
                ("send_upper", ctypes.c_int * 2), ("recv_upper", ctypes.c_int * 2)]


class igg_plan_entry(ctypes.Structure):
    _fields_ = [("axis", ctypes.c_int), ("op", ctypes.c_int), ("local_rank", ctypes.c_int), ("field", ctypes.c_int),
                ("recv_side", ctypes.c_int), ("peer", ctypes.c_int), ("transport", ctypes.c_int),
                ("lo", ctypes.c_int), ("h", ctypes.c_int), ("count", ctypes.c_longlong), ("order", ctypes.c_int)]


REGION_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                             ctypes.POINTER(ctypes.c_int), ctypes.c_void_p)

# name -> (argtypes); every entry point returns igg_status (int) except igg_last_error
SIGNATURES = {
    "igg_dims_create": [ctypes.c_int, c_int_p, c_int_p],
    "igg_rank_of_coords": [c_int_p, c_int_p, c_int_p],
    "igg_coords_of_rank": [c_int_p, ctypes.c_int, c_int_p],
    "igg_global_size": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_ll_p],
    "igg_halo_spec_of": [ctypes.c_int, ctypes.c_int, ctypes.c_longlong, ctypes.POINTER(igg_halo_spec)],
    "igg_get_unique_id": [ctypes.POINTER(ctypes.c_ubyte)],
    "igg_plan_update_halo": [ctypes.POINTER(igg_init_args), c_ll_p, ctypes.c_int, ctypes.POINTER(igg_plan_entry),
                             ctypes.c_int, c_int_p],
    "igg_init_global_grid": [ctypes.POINTER(igg_init_args), ctypes.POINTER(ctypes.c_void_p), c_int_p, c_int_p,
                             c_int_p, c_ll_p],
    "igg_finalize_global_grid": [ctypes.c_void_p],
    "igg_n_g": [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, c_ll_p],
    "igg_coords": [ctypes.c_void_p, ctypes.c_int, c_int_p],
    "igg_local_to_global": [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_longlong, c_ll_p],
    "igg_global_coord": [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_longlong, ctypes.c_double,
                         ctypes.POINTER(ctypes.c_double)],
    "igg_save_field": [ctypes.c_char_p, ctypes.c_void_p, c_ll_p],
    "igg_buffer_allocs": [ctypes.c_void_p, c_ll_p],
    "igg_kernel_launches": [ctypes.c_void_p, c_ll_p],
    "igg_update_halo": [ctypes.c_void_p, ctypes.POINTER(igg_field), ctypes.c_int, ctypes.c_void_p],
    "igg_heat_step": [ctypes.c_void_p, c_dbl_pp, c_dbl_pp, c_dbl_pp, ctypes.c_double, ctypes.c_double,
                      ctypes.c_double, ctypes.c_double, ctypes.c_double, c_int_p, ctypes.c_void_p],
    "igg_heat_step_f32": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float,
                          ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float, c_int_p, ctypes.c_void_p],
    "igg_heat_run": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, c_dbl_pp, ctypes.c_double, ctypes.c_double,
                     ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, c_int_p, ctypes.c_void_p],
    "igg_heat_run_f32": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float,
                         ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_int, c_int_p,
                         ctypes.c_void_p],
    "igg_heat_run_host": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                          ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, c_int_p,
                          ctypes.c_void_p],
    "igg_global_max": [ctypes.c_void_p, ctypes.c_double, c_dbl_p],
    "igg_field_global_max": [ctypes.c_void_p, c_dbl_pp, ctypes.c_longlong, c_dbl_p, ctypes.c_void_p],
    "igg_set_option": [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong],
    "igg_check": [ctypes.c_void_p],
    "igg_release_arrays": [ctypes.c_void_p],
    "igg_hide_communication": [ctypes.c_void_p, c_int_p, REGION_FN, ctypes.c_void_p, ctypes.POINTER(igg_field),
                               ctypes.c_int, ctypes.c_void_p],
    "igg_acoustic_step": [ctypes.c_void_p, c_dbl_pp, c_dbl_pp, c_dbl_pp, c_dbl_pp, ctypes.c_double,
                          ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                          c_int_p, ctypes.c_void_p],
    "igg_gather": [ctypes.c_void_p, ctypes.POINTER(igg_field), ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p],
    "igg_acoustic_run": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                         ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, c_int_p, ctypes.c_void_p],
    "igg_profile_stencil": [ctypes.c_void_p, c_dbl_p, c_ll_p, c_ll_p],
    "igg_profile_timeline": [ctypes.c_void_p, c_dbl_p],
}

_lib = None


def lib():
    """Load libigg.so once; raises ImportError if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (there is no fallback path)")
        L = ctypes.CDLL(SO_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.igg_last_error.argtypes = []
        L.igg_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib
