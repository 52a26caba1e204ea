/*
 * igg.h -- C ABI of the B200-native implicit global grid library (libigg.so).
 *
 * The paper (arXiv 2211.15716, PAPER.md) states the problem as "as little as
 * three functions": create the implicit global staggered grid, perform a halo
 * update on it, finalize it (Fig. 1 listing lines 23, 38, 43 =
 * PAPER.md:62, :77, :82), plus size queries nx_g()/ny_g()/nz_g()
 * (PAPER.md:63-65), and hides communication behind the stencil step with
 * @hide_communication (16,2,2).  This header is that API.
 *
 * Conventions (every entry point):
 *   - returns igg_status; IGG_OK == 0.  On error igg_last_error() returns a
 *     thread-local message naming the call and the reason.  C++ exceptions
 *     never cross this boundary.
 *   - arrays are Float64 ("@init_parallel_stencil(CUDA, Float64, 3)"),
 *     x fastest: element (x,y,z) of a field of size (sx,sy,sz) is at
 *     ptr[(z*sy + y)*sx + x], 0-based.
 *   - field memory is OWNED BY THE CALLER (e.g. torch tensors) and BORROWED
 *     for the duration of the enqueued work; the library owns its send/recv
 *     buffer pool, streams, events, NCCL communicator and peer mappings and
 *     frees them in igg_finalize_global_grid.
 *   - update_halo / heat_step are stream-ordered and host-asynchronous: they
 *     run after prior work on `stream` and later work on `stream` sees their
 *     results.  init / finalize / global_max are synchronous collectives.
 *   - collective calls: every rank calls them in the same order with the same
 *     field list.
 *   - "local ranks": one process normally hosts one rank on one GPU.  A
 *     process may host `local_ranks` consecutive ranks on its one GPU
 *     (virtual ranks, used to test topologies larger than the GPU count);
 *     then every per-rank argument is an array of local_ranks entries,
 *     rank-major.  Virtual ranks on one GPU exchange by stream-ordered copies,
 *     never by spinning kernels.
 */
#ifndef IGG_H
#define IGG_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct igg_grid igg_grid;   /* opaque, library-owned */
typedef void *igg_stream_t;          /* a cudaStream_t (0 = legacy default stream) */

typedef enum igg_status {
    IGG_OK = 0,
    IGG_E_ARG = 1,       /* bad argument: n_d <= o_d, odd/negative overlap, dims product != nprocs, bad axis, null pointer */
    IGG_E_STATE = 2,     /* use after finalize, double finalize */
    IGG_E_STAGGER = 3,   /* field size s_d outside [n_d-o_d, n_d+o_d] */
    IGG_E_WIDTH = 4,     /* 0 < b_d < ol_d on an exchanged axis */
    IGG_E_CUDA = 5,      /* a CUDA runtime call failed */
    IGG_E_NCCL = 6,      /* an NCCL call failed */
    IGG_E_TIMEOUT = 7,   /* a P2P receive flag did not arrive in time (analog of SPEC.md:273, :308) */
    IGG_E_UNSUPPORTED = 8,
    IGG_E_BOOTSTRAP = 9  /* the caller's bootstrap all-gather returned non-zero */
} igg_status;

enum {
    IGG_PATH_NCCL = 0,   /* halo faces cross GPUs with ncclSend/ncclRecv grouped per axis */
    IGG_PATH_P2P = 1     /* pack kernels store faces straight into the peer's receive buffers over NVLink */
};

/* ------------------------------------------------------------------ errors */
/* Thread-local message of the last failing call on this thread ("" if none). */
const char *igg_last_error(void);

/* ------------------------------------------------------------------ host-only topology math
 * No GPU needed.  Readings of the paper for these formulas: DESIGN.md.      */

/* SPEC.md:37-46 (paper: topology "automatically defined"): the
 * ordered factorisation of nprocs honouring non-zero entries of fixed[3] with
 * minimal max-min, ties to the lexicographically largest.  IGG_E_ARG if none. */
igg_status igg_dims_create(int nprocs, const int fixed[3], int dims_out[3]);

/* Cartesian rank order, last axis fastest: rank = (cx*py + cy)*pz + cz. */
igg_status igg_rank_of_coords(const int dims[3], const int coords[3], int *rank_out);
igg_status igg_coords_of_rank(const int dims[3], int rank, int coords_out[3]);

/* Global size of one axis, PAPER.md:63-65 nx_g(): p(n-o)+o non-periodic,
 * p(n-o) periodic.  IGG_E_ARG if n <= o or p < 1. */
igg_status igg_global_size(int n, int o, int p, int periodic, long long *out);

/* Halo geometry of a field of local size s on an axis with local size n and
 * overlap o: ol = s-(n-o), h = ol/2; 0-based half-open layer
 * ranges.  IGG_E_STAGGER if s < n-o or s > n+o. */
typedef struct igg_halo_spec {
    int ol, h;
    int send_lower[2], recv_lower[2], send_upper[2], recv_upper[2];
} igg_halo_spec;
igg_status igg_halo_spec_of(int n, int o, long long s, igg_halo_spec *out);

/* ------------------------------------------------------------------ lifecycle */
typedef struct igg_init_args igg_init_args;

/* The exchange plan of one update_halo call of THIS process (host only, no
 * GPU): every face it packs (op 0) or unpacks (op 1), axis by axis in
 * execution order.  Validates args like igg_init_global_grid
 * and sizes like igg_update_halo.  sizes: nfields*3 (sx,sy,sz).  Writes at
 * most `capacity` entries to out (out may be NULL to query) and the total to
 * *count; IGG_E_ARG if capacity is too small. */
typedef struct igg_plan_entry {
    int axis;          /* 0 = x, 1 = y, 2 = z */
    int op;            /* 0 = pack send layers toward `peer`, 1 = unpack receive layers from `peer` */
    int local_rank;    /* hosted rank index (global rank = rank0 + local_rank) */
    int field;         /* index in the call's field list */
    int recv_side;     /* halo side of the RECEIVING rank: 0 = lower, 1 = upper */
    int peer;          /* global rank at the other end */
    int transport;     /* 0 = local copy, 1 = NCCL, 2 = P2P store */
    int lo, h;         /* layers [lo, lo+h) of `axis` (0-based) */
    long long count;   /* doubles in the face: h * (other two sizes) */
    int order;         /* NCCL posting position among this axis' sends (op 0) or receives (op 1); -1 otherwise */
} igg_plan_entry;
igg_status igg_plan_update_halo(const igg_init_args *args, const long long *sizes, int nfields,
                                igg_plan_entry *out, int capacity, int *count);

/* Host bootstrap (optional, igg_init_args.bootstrap): a collective all-gather over the caller's own
 * channel (e.g. a torch gloo process group).  Every process passes `bytes` bytes in `mine` and receives
 * the contributions of all processes, in process order, in `all` (nprocs/local_ranks * bytes).  Called
 * on the thread that called into the library, only from collective entry points (init, the first use of
 * an array on the fused path, arena growth, global_max, gather, finalize).  Returns 0 on success. */
typedef int (*igg_allgather_fn)(void *user, const void *mine, void *all, unsigned long long bytes);

struct igg_init_args {
    int nx, ny, nz;          /* local size of a canonical (non-staggered) field */
    int dims[3];             /* process topology; 0 entries = automatic (igg_dims_create) */
    int periods[3];          /* 0/1 per axis; Fig. 1 passes none -> non-periodic */
    int overlaps[3];         /* even, >= 2; 0 = default 2 */
    int nprocs;              /* total number of ranks of the grid */
    int rank0;               /* first global rank hosted by this process */
    int local_ranks;         /* ranks hosted by this process (>= 1), all on `device` */
    int device;              /* CUDA device ordinal of this process */
    int path;                /* IGG_PATH_NCCL or IGG_PATH_P2P */
    int reserved;
    unsigned char comm_id[128]; /* ncclUniqueId from igg_get_unique_id on process 0, broadcast by
                                   the caller; unused when one process hosts every rank or when
                                   `bootstrap` is set */
    igg_allgather_fn bootstrap; /* NULL (default): host collectives over an NCCL communicator built
                                   from comm_id.  Set (path must be IGG_PATH_P2P): NO NCCL communicator
                                   is created; every host-side collective goes through this callback and
                                   every face moves by CUDA-IPC peer stores.  This is also what lets
                                   several processes share one GPU (NCCL refuses two ranks on one
                                   device); IGG_E_ARG with path == IGG_PATH_NCCL. */
    void *bootstrap_user;       /* passed back to bootstrap */
};


/* Fill out[128] with a fresh NCCL unique id (call on process 0 only). */
igg_status igg_get_unique_id(unsigned char out[128]);

/* init_global_grid (listing 23).  Collective over processes.
 * Validates the arguments, builds the topology, sets the device, creates the
 * priority streams, the NCCL communicator (when more than one
 * process) and the P2P mappings.  Outputs (any may be NULL): me = rank0,
 * coords of rank0, the dims used and the canonical global sizes n_g. */
igg_status igg_init_global_grid(const igg_init_args *args, igg_grid **grid_out,
                                int *me, int coords[3], int dims_out[3], long long n_g[3]);

/* finalize_global_grid (listing 43).  Collective, synchronous.
 * Frees everything the library owns.  The handle is invalid afterwards. */
igg_status igg_finalize_global_grid(igg_grid *grid);

/* ------------------------------------------------------------------ queries */
/* Distinct global layers of a field of local size field_size on axis (0=x,1=y,2=z):
 * non-periodic n_g + (s - n); periodic the period p(n-o).  field_size = 0
 * means the canonical size n (then this is nx_g()/ny_g()/nz_g()). */
igg_status igg_n_g(const igg_grid *grid, int axis, long long field_size, long long *out);

/* Coordinates of a global rank in the grid's topology. */
igg_status igg_coords(const igg_grid *grid, int rank, int coords_out[3]);

/* 0-based local layer l of `rank` on axis -> 0-based global layer:
 * g = c(n-o) + l; on a periodic axis (g - o/2) mod p(n-o) (reading 15). */
igg_status igg_local_to_global(const igg_grid *grid, int rank, int axis, long long l, long long *g_out);

/* Physical coordinate of local layer l of `rank` on axis (SPEC.md:119-122 global_coord; spacing as in
 * PAPER.md:66-68, dx = lx/(nx_g()-1)): x = g * spacing with g = igg_local_to_global(...).  Same range
 * check as igg_local_to_global (IGG_E_ARG). */
igg_status igg_global_coord(const igg_grid *grid, int rank, int axis, long long l, double spacing, double *x_out);

/* Buffer-pool allocation counter: constant once every
 * field shape has been exchanged once. */
igg_status igg_buffer_allocs(const igg_grid *grid, long long *count_out);

/* ------------------------------------------------------------------ halo update */
typedef struct igg_field {
    double *ptr;             /* device pointer, x fastest (a float array when elsize == 4) */
    long long size[3];       /* (sx, sy, sz): n_d-o_d <= s_d <= n_d+o_d; staggered fields are n+1 */
    int elsize;              /* bytes per element: 0 or 8 = binary64, 4 = binary32 (
                                igg_update_halo and igg_hide_communication; igg_gather: 8 only) */
} igg_field;

/* update_halo! (listing 38).  Collective.
 * fields: local_ranks*nfields entries, rank-major ([r*nfields + f]).
 * For axis x, then y, then z: the send layers of every field and side with a
 * neighbour (full extent of the other axes, halos included) are packed,
 * moved (locally, over NCCL, or by direct stores into the peer's receive
 * buffer), and unpacked into the neighbour's receive layers.
 * Runs on the library's high-priority comm stream, joined to `stream`.
 * Errors: IGG_E_STAGGER, IGG_E_ARG (nfields < 1, null pointer). */
igg_status igg_update_halo(igg_grid *grid, const igg_field *fields, int nfields, igg_stream_t stream);

/* ------------------------------------------------------------------ the heat step */
/* @hide_communication bw begin @parallel step!(T2,T,Ci,lam,dt,dx,dy,dz); update_halo!(T2) end
 * (PAPER.md:45-51, :75-78).  T2, T, Ci: local_ranks device pointers each, all
 * of the canonical size (nx,ny,nz).  Writes T2 at inner points 1..s-2 of
 * every axis (PAPER.md:46 @inn), then refreshes T2's halos.  T2 must be a
 * copy of T's boundary layers (PAPER.md:69 T2 = copy(T)); global-boundary
 * layers are never written (Dirichlet by initialisation).
 * Arithmetic per cell, binary64, no FMA contraction:
 *   T2 = T + dt*((lam*Ci)*(((d2x*rdx2) + (d2y*rdy2)) + (d2z*rdz2))),
 *   d2x = (T[x+1]-T[x]) - (T[x]-T[x-1]), rdx2 = 1.0/(dx*dx) (readings 6-9).
 * bw: boundary widths per axis; {0,0,0} = sequential step then update.
 * Otherwise the six boundary slabs run first on the high-priority stream,
 * the halo exchange follows them there, and the inner box [b_d, s_d-b_d)
 * runs concurrently on a low-priority stream.  An exchanged axis needs
 * b_d >= ol_d (IGG_E_WIDTH); an empty inner box degenerates to sequential. */
igg_status igg_heat_step(igg_grid *grid, double *const *T2, const double *const *T,
                         const double *const *Ci, double lam, double dt,
                         double dx, double dy, double dz, const int bw[3], igg_stream_t stream);

/* The binary32 heat step (reading 24): the same step with float fields and
 * every operation in binary32 (inputs as given, reciprocals 1.0f/(d*d) in float, no FMA, canonical
 * association), then update_halo of T2 as a binary32 field.  bw as in igg_heat_step: {0,0,0} (or NULL)
 * = sequential, else boundary slabs + exchange on the high-priority stream with the inner box
 * concurrent.  Size-1 axes allowed as in igg_heat_step.  Errors: IGG_E_ARG, IGG_E_STATE, IGG_E_WIDTH. */
igg_status igg_heat_step_f32(igg_grid *grid, float *const *T2, const float *const *T, const float *const *Ci,
                             float lam, float dt, float dx, float dy, float dz, const int bw[3],
                             igg_stream_t stream);

/* Fig. 1's time loop on the device: nt heat steps, each followed by the swap
 * T, T2 = T2, T.  T, T2: arrays of local_ranks device pointers that the library swaps in place, so on
 * return T[lr] holds the state after nt steps and T2[lr] the state before it.  Results are identical
 * to nt igg_heat_step calls; on the fused P2P path consecutive steps are pipelined (a step's tiles that
 * read halo cells wait in-kernel for the previous step's faces; only the last step waits for all of
 * them).  Stream-ordered on `stream`; complete for any later work on it.  Errors as igg_heat_step. */
igg_status igg_heat_run(igg_grid *grid, double **T, double **T2, const double *const *Ci, double lam,
                        double dt, double dx, double dy, double dz, int nt, const int bw[3],
                        igg_stream_t stream);

/* The same time loop for binary32 fields: nt igg_heat_step_f32 steps with the swap;
 * on the fused P2P path consecutive steps are pipelined exactly as in igg_heat_run (float2 lanes of the
 * same kernel).  Results identical to nt igg_heat_step_f32 calls.  Errors as igg_heat_step_f32. */
igg_status igg_heat_run_f32(igg_grid *grid, float **T, float **T2, const float *const *Ci, float lam, float dt,
                            float dx, float dy, float dz, int nt, const int bw[3], igg_stream_t stream);

/* ------------------------------------------------------------------ generic hide_communication
 * A user stencil for igg_hide_communication: compute the cells of the box [lo, hi) (0-based, of the
 * canonical local grid of hosted rank `local_rank`) by enqueuing work on `stream`; it must write only
 * cells inside the box and read only values the step does not write. */
typedef void (*igg_region_fn)(void *user, int local_rank, const int lo[3], const int hi[3], igg_stream_t stream);

/* @hide_communication bw begin <user step>; update_halo!(fields...) end (
 * SPEC.md:330-338) for any stencil: the six boundary slabs of the computed box [1, n-1)^3 are
 * requested first on the library's high-priority stream, update_halo(fields) follows them there, and
 * the inner box [max(1,b), n-b) is requested on the low-priority stream concurrently; everything is
 * joined to `stream`.  bw = {0,0,0} or an empty inner box: sequential (full box, then update_halo).
 * An exchanged axis needs b_d >= ol_d of every exchanged field (IGG_E_WIDTH).  fields: local_ranks *
 * nfields entries, rank-major, as for igg_update_halo.  fn is called on this thread before return. */
igg_status igg_hide_communication(igg_grid *grid, const int bw[3], igg_region_fn fn, void *user,
                                  const igg_field *fields, int nfields, igg_stream_t stream);

/* ------------------------------------------------------------------ second workload
 * One leapfrog step of linear acoustics on the staggered grid -- the multi-field staggered kind of
 * solver the paper scales -- in the paper's stencil notation:
 *   @hide_communication bw begin compute_V!; update_halo!(Vx, Vy, Vz) end; compute_P!
 *   compute_V: Vx[k,j,i] -= cVx*(P[k,j,i] - P[k,j,i-1]) on i in [1,nx), j in [1,ny-1), k in [1,nz-1)
 *              (Vy, Vz likewise along their own axis)
 *   compute_P: P -= cP*((((Vx[i+1]-Vx[i])*rx) + ((Vy[j+1]-Vy[j])*ry)) + ((Vz[k+1]-Vz[k])*rz)), every cell
 *   cV_d = (dt/rho)/d_d, cP = dt*K, r_d = 1.0/d_d; binary64, no FMA (readings A1-A3).
 * P, Vx, Vy, Vz: local_ranks device pointers each; P (nz,ny,nx), Vx (nz,ny,nx+1), Vy (nz,ny+1,nx),
 * Vz (nz+1,ny,nx), x fastest (config B:10's field set).  bw: boundary widths of the velocity step;
 * an exchanged axis needs b_d >= 3 (the staggered overlap, IGG_E_WIDTH); {0,0,0} = sequential.
 * Stream-ordered on `stream`.  Errors: IGG_E_ARG (null pointer, rho or a spacing zero, n_d < 3),
 * IGG_E_WIDTH, IGG_E_STATE. */
igg_status igg_acoustic_step(igg_grid *grid, double *const *P, double *const *Vx, double *const *Vy,
                             double *const *Vz, double dt, double rho, double K, double dx, double dy,
                             double dz, const int bw[3], igg_stream_t stream);

/* nt steps of the second workload with double-buffered fields: F = [P, Vx, Vy, Vz, P2, Vx2, Vy2, Vz2], each
 * local_ranks device pointers (field-major: F[f*local_ranks + r]), shapes as igg_acoustic_step.  A grid
 * without any exchanged axis runs ONE fused compute_V + compute_P sweep per step from the current set into
 * the other (every element of the other set written; 64 B/cell instead of 96) and swaps the pointer sets;
 * otherwise every step is igg_acoustic_step on the current set in place.  On return F[0..3*local_ranks+..]
 * (the first four fields) hold the state after nt steps, bit-identical to nt igg_acoustic_step calls.
 * Stream-ordered.  Errors as igg_acoustic_step. */
igg_status igg_acoustic_run(igg_grid *grid, double **F, int nt, double dt, double rho, double K, double dx,
                            double dy, double dz, const int bw[3], igg_stream_t stream);

/* Fig. 1 end to end from HOST memory: copies T (initial, local_ranks*nx*ny*nz
 * doubles, rank-major) and Ci to the device, sets T2 = copy(T), runs nt heat
 * steps with swap, and copies the final T back into T_host.
 * Device scratch comes from the library pool (allocated once per size).
 * Synchronous: returns after the result is in T_host.  Host buffers should be
 * pinned for full copy bandwidth. */
igg_status igg_heat_run_host(igg_grid *grid, double *T_host, const double *Ci_host,
                             double lam, double dt, double dx, double dy, double dz,
                             int nt, const int bw[3], igg_stream_t stream);

/* ------------------------------------------------------------------ reductions */
/* maximum over all ranks of `local` (PAPER.md:73 maximum(Ci), reading 12). */
igg_status igg_global_max(igg_grid *grid, double local, double *out);

/* maximum over all ranks and all elements of a field (local_ranks device
 * pointers of `count` doubles each), computed by the library's reduction
 * kernel and an NCCL max-allreduce.  Synchronous on `stream`. */
igg_status igg_field_global_max(igg_grid *grid, const double *const *f, long long count,
                                double *out, igg_stream_t stream);

/* gather: assemble the global field on process root_proc, in host
 * memory of the global size (igg_n_g per axis, x fastest), from every rank's OWNED layers: interior
 * ranks own local layers [h + ol%2, s - h) per axis, the first rank also the lower halo layers, the last
 * the upper ones (non-periodic), a shared middle layer (odd field overlap) the lower rank.  fields:
 * local_ranks device pointers of one field shape.  host_out is ignored on other processes.
 * Collective and synchronous (a utility, not on the hot path). */
igg_status igg_gather(igg_grid *grid, const igg_field *fields, int root_proc, double *host_out,
                      igg_stream_t stream);

/* Output of a gathered field: `path` receives the one-line header "IGRIDF1 nx ny nz\n"
 * followed by nx*ny*nz little-endian binary64 values of `host` (x fastest).  Host-only; IGG_E_ARG on a
 * null pointer, a non-positive size or a failed open/write (igg_last_error names the path). */
igg_status igg_save_field(const char *path, const double *host, const long long n[3]);

/* ------------------------------------------------------------------ control */
enum {
    IGG_OPT_SKIP_COMM = 1,       /* timing only (SURVEY.md 8(d) "comm disabled"): the exchange is skipped
                                    so exposed halo time = t(overlap) - t(overlap, comm disabled) can be
                                    measured; halo results are INVALID while it is on, and igg_check
                                    reports IGG_E_STATE for the steps taken with it */
    IGG_OPT_SPIN_TIMEOUT_MS = 2, /* P2P flag wait bound (default 20000) */
    IGG_OPT_STENCIL_KERNEL = 3,  /* 0 = auto, 1 = the generic scalar region kernel for every region (a
                                    reference kernel; same cells); other values: the tuning variants of the
                                    ablation build only (IGG_E_UNSUPPORTED in the product library) */
    IGG_OPT_PROFILE = 4,         /* 1 = bracket every main stencil launch (the full-region or
                                    inner-box kernel) with CUDA events on its own stream;
                                    2 = also record the overlap timeline (igg_profile_timeline) */
    IGG_OPT_X_ALIGN = 5,         /* x boundary-slab edges rounded to this many cells (default 64 =
                                    512-B row segments; 1 = the exact widths given) */
    IGG_OPT_SCHEDULE = 6,        /* 0 = inner box concurrent with the boundary slabs; 1 = inner box
                                    after the boundary slabs (paper order), concurrent with the exchange */
    IGG_OPT_FUSED = 7,           /* P2P path, one rank per GPU: 1 = one stencil kernel that stores its
                                    send layers straight into the neighbours' halos over NVLink, chunk
                                    by chunk; 0 = boundary/inner kernels + pack/exchange/unpack;
                                    -1 (default) = fused whenever eligible */
    IGG_OPT_FUSED_MODE = 8,      /* ablation build only (ablation/libigg_ablation.so): binary32 schedule bits
                                    8192 / 16384; the product library answers IGG_E_UNSUPPORTED */
    IGG_OPT_FUSED_KC2 = 9,       /* planes per short (end) z-chunk of the fused stencil (0 = auto: 8) */
    IGG_OPT_FUSED_COMM_CTAS = 10,/* forwarder blocks per rank in the last step of a fused run (default 1) */
    /* 11: retired (the cooperative per-axis update_halo, superseded by IGG_OPT_HALO26) */
    IGG_OPT_HALO_STREAM = 12,    /* 0 (default): update_halo runs on the library's high-priority comm
                                    stream joined to the caller's; 1: directly on the caller's stream */
    IGG_OPT_LOCAL_P2P = 13,      /* 1: update_halo runs the dimension-sequential P2P protocol (per axis: pack
                                    into the receiver's slot, release flag, acquire wait, unpack) also
                                    between the ranks hosted by this process (the cross-process protocol
                                    emulated on one GPU; results identical; tests) */
    IGG_OPT_HALO26 = 14,         /* 1 (default): update_halo without NCCL messages is ONE kernel that stores
                                    every halo region (faces, edges, corners) straight from its owner into
                                    the receiver (26-neighbour single phase, bit-identical to the
                                    dimension-sequential result); 0: the per-axis pack/flag/unpack kernels */
    IGG_OPT_FUSED_F32 = 15       /* binary32 steps on the P2P path through the fused stencil + exchange kernel
                                    (float4 lanes, 128-cell tile rows; bit-exact; needs nx % 4 == 0, nx >= 130):
                                    1 = always, 0 = never (the split schedule), -1 (default) = when the x axis is
                                    the only exchanged one (the fused binary32 sweep is 4.8 % slower than the float4
                                    box kernel, faster than the sequential x-split schedule) */
};
igg_status igg_set_option(igg_grid *grid, int key, long long value);

/* Collective, synchronous.  The fused P2P step maps every rank's T2 array into its neighbours'
 * address spaces (CUDA IPC) on the array's first use and caches the mapping.  Call this on every
 * process before freeing (or handing back to an allocator) any array used as T / T2 in a heat step,
 * so no peer keeps a mapping of freed memory.  igg_heat_run / igg_heat_run_host re-validate the cache
 * collectively on entry; a single igg_heat_step given an array that was re-allocated at a cached address
 * fails with IGG_E_STATE instead of storing into the old allocation. */
igg_status igg_release_arrays(igg_grid *grid);

/* Blocks until all work of the grid's streams is done, then reports a P2P
 * wait timeout (IGG_E_TIMEOUT) or an NCCL asynchronous error. */
igg_status igg_check(igg_grid *grid);

/* With IGG_OPT_PROFILE on: synchronizes the device, returns the summed
 * CUDA-event duration (ms) of the main stencil launches recorded since the
 * last call, their number and the cells they updated, and resets the record. */
igg_status igg_profile_stencil(igg_grid *grid, double *ms_total, long long *launches, long long *cells);

/* With IGG_OPT_PROFILE = 2: averages over the overlapped steps since the last
 * call of the times (ms, CUDA events) from the step's start on the caller's
 * stream to: [0] boundary slabs done, [1] inner box start, [2] inner box done,
 * [3] halo exchange done; [4] = number of steps.  Synchronizes; resets. */
igg_status igg_profile_timeline(igg_grid *grid, double out[5]);

/* Number of kernels the library has launched since init (launch accounting). */
igg_status igg_kernel_launches(const igg_grid *grid, long long *count_out);

#ifdef __cplusplus
}
#endif
#endif /* IGG_H */
