"""B200-native implicit global grid (arXiv 2211.15716, ImplicitGlobalGrid):
the distributed 3-D heat-diffusion step with update_halo! and
@hide_communication, as a C-ABI library (libigg.so, include/igg.h) with a thin
Python binding.  See DESIGN.md."""
from .igg import (PATH_NCCL, PATH_P2P, OPT_SKIP_COMM, OPT_SPIN_TIMEOUT_MS, OPT_STENCIL_KERNEL, OPT_PROFILE,
                  OPT_X_ALIGN, OPT_SCHEDULE, OPT_FUSED, OPT_FUSED_MODE, OPT_FUSED_KC2, OPT_FUSED_COMM_CTAS,
                  OPT_HALO_STREAM, OPT_LOCAL_P2P, OPT_HALO26, OPT_FUSED_F32, Grid, IggError,
                  coords_of_rank, dims_create, get_unique_id, global_size, halo_spec, init_global_grid,
                  plan_update_halo, rank_of_coords)
from . import heat3d

__all__ = ["PATH_NCCL", "PATH_P2P", "OPT_SKIP_COMM", "OPT_SPIN_TIMEOUT_MS", "OPT_STENCIL_KERNEL", "OPT_PROFILE",
           "OPT_X_ALIGN", "OPT_SCHEDULE", "OPT_FUSED", "OPT_FUSED_MODE", "OPT_FUSED_KC2", "OPT_FUSED_COMM_CTAS",
           "OPT_HALO_STREAM", "OPT_LOCAL_P2P", "OPT_HALO26", "OPT_FUSED_F32", "Grid",
           "IggError", "coords_of_rank", "dims_create", "get_unique_id", "global_size", "halo_spec",
           "init_global_grid", "plan_update_halo", "rank_of_coords", "heat3d"]
