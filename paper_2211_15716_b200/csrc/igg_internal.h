// igg_internal.h -- internal types shared by the libigg translation units.
// Nothing here crosses the C ABI (include/igg.h is the boundary).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <list>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/igg.h"

namespace igg {

// ---------------------------------------------------------------- errors
struct Error {
    igg_status code;
    std::string msg;
};
struct IggException {
    igg_status code;
};
void set_error(const std::string &msg);
[[noreturn]] void fail(igg_status code, const std::string &msg);

#define IGG_CUDA(call)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            ::igg::fail(IGG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
    } while (0)
#define IGG_NCCL(call)                                                                      \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                              \
            ::igg::fail(IGG_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));    \
    } while (0)

#define IGG_API extern "C" __attribute__((visibility("default")))
#define IGG_TRY try {
#define IGG_CATCH                                                       \
    }                                                                   \
    catch (const ::igg::IggException &e) { return e.code; }             \
    catch (const std::exception &e) {                                   \
        ::igg::set_error(std::string("internal error: ") + e.what());   \
        return IGG_E_ARG;                                               \
    }                                                                   \
    return IGG_OK;

// ---------------------------------------------------------------- host topology math
int dims_create(int nprocs, const int fixed[3], int out[3]);          // 0 ok, -1 none
int rank_of_coords(const int dims[3], const int c[3]);
void coords_of_rank(const int dims[3], int rank, int c[3]);
long long global_size(int n, int o, int p, int periodic);
struct HaloSpec {
    int ol, h;
    int send_lo[2], recv_lo[2], send_up[2], recv_up[2];   // 0-based [a,b)
};
bool halo_spec(int n, int o, long long s, HaloSpec *out);             // false: bad stagger

// ---------------------------------------------------------------- device-side descriptors
// one face copy: the slab [lo, lo+h) of `axis` of a field <-> a contiguous buffer,
// buffer layout x fastest, then y, then z, restricted to the slab
struct CopyDesc {
    double *field;                   // element type by esz (8: double, 4: float)
    double *buf;
    long long sx, sy, sz;
    long long count;                 // h * (other two sizes), elements
    int axis, lo, h;
    int flag_slot;                   // unpack: index into WaitList flags (-1 = no wait)
    int esz;                         // bytes per element
};

constexpr int kMaxCopy = 48;
constexpr int kMaxSignal = 16;
template <int N>
struct CopyListT {
    CopyDesc d[N];
    int n;
    int blocks_per_desc;
    // pack: after every block stored its part (to peers), the last block
    // publishes `epoch` to these remote flags (st.release.sys)
    unsigned long long *signal[kMaxSignal];
    int nsignal;
    unsigned int *ticket;            // device counter for the last-block election
    unsigned int ticket_total;       // blocks over ALL chunks of this pack (the last one signals)
    // unpack: wait until *wait[flag_slot] >= epoch (ld.acquire.sys) before reading
    const unsigned long long *wait[kMaxSignal];
    unsigned long long epoch;
    long long timeout_cycles;
    int *err;                        // set to 1 on timeout
};
using CopyList = CopyListT<kMaxCopy>;
constexpr int kSmallCopy = 8;        // small calls launch with a ~1 KB parameter block

// one stencil region [x0,x0+wx) x [y0,y0+wy) x [z0,z0+wz) of one rank's field
struct HeatRegion {
    const double *T;
    const double *Ci;
    double *T2;
    int sx, sy, sz;
    int x0, y0, z0;
    int wx, wy, wz;
    int zchunks;
    int col_blocks;
    int block_begin;
    // vectorised tiling (slab / box-list kernels): lanes per row segment, z-chunk(s), tile counts
    int lx, kc, xtiles, ytiles, ax0;
    int nbig, kc2;   // box-list kernel: nbig chunks of kc planes, then chunks of kc2 planes
};
constexpr int kMaxRegions = 16;
struct HeatCoef {
    double lam, dt, rdx2, rdy2, rdz2;
};
// binary32 coefficients (rounded to float by the caller)
struct HeatCoefF {
    float lam, dt, rdx2, rdy2, rdz2;
};
struct HeatRegionList {
    HeatRegion r[kMaxRegions];
    int n;
    int total_blocks;
    HeatCoef k;
};

// ---------------------------------------------------------------- fused stencil + exchange (fused.cu)
constexpr int kMaxChunks = 128;      // z-chunks per step (flags / counters per face and chunk)
constexpr int kMaxFusedRanks = 8;    // ranks hosted on one GPU that one fused launch covers
#ifndef FUSED_DEFER   // (ablation builds sweep these three)
#define FUSED_DEFER 3
#endif
#ifndef FUSED_XSENDERS
#define FUSED_XSENDERS 16
#endif
#ifndef FUSED_XPIECE
#define FUSED_XPIECE 8
#endif
constexpr int kFusedDefer = FUSED_DEFER;         // x chunks a pipelined step leaves to the next launch's senders
constexpr int kFusedXSenders = FUSED_XSENDERS;   // x sender blocks per x face and rank
constexpr int kFusedXPiece = FUSED_XPIECE;       // planes per x sender work piece
struct FusedFace {                   // one face I send, indexed by the RECEIVER's halo side
    double *dst;                     // the receiver's T2 (a sibling's, or peer-mapped); lands in its halo layer
    unsigned long long *flag;        // receiver's data flags of (axis, side): [kMaxChunks] (z faces: [0])
    unsigned long long *xflag;       // receiver's flags of the rim/forwarded cells
    int layer;                       // my send layer along the axis
    int active;
};
struct FusedHalo {                   // one halo side I receive
    const unsigned long long *flag;  // my data flags [kMaxChunks]
    const unsigned long long *xflag; // my rim/forwarded-cell flags [kMaxChunks]
    int layer;                       // halo layer (0 or s-1)
    int active;
};
struct FusedRank {                   // one hosted rank of a fused launch
    const double *T;
    const double *Ci;
    double *T2;
    FusedFace face[3][2];
    FusedHalo halo[3][2];
    // x faces: the face tiles store their x send column z-contiguously into the local staging rows
    // xloc [side rs][y][z] and count on xcnt [rs][chunk] (GPU scope); the x sender blocks move each
    // completed chunk into the receiver's T2 halo column and publish its flag
    double *xloc;
    unsigned int *xcnt;
    // ... into the receiver's staging rows xrem [parity][side][y][z] (contiguous: whole sectors over NVLink,
    // no scattered remote stores); the receiver's halo tiles substitute them for T's halo column in their
    // sweep (no column is ever written), the forwarders read them, the drain copies the last into T2
    double *xrem;                    // mine (written by my neighbours' senders)
    double *xrem_peer[2];            // the receivers' (indexed like face[0][rs])
    unsigned int *ctr;               // [6][kMaxChunks] data-flag contribution counters (sender side)
    unsigned int *ctr_x;             // [6][kMaxChunks] rim/forwarded-cell counters
    unsigned int *rim_ticket;
    unsigned int *xpc;               // [parity][2][kMaxChunks] x-piece counters, by epoch parity: a launch
                                     // may publish a chunk for two epochs (deferred and its own)
};
struct FusedParams {
    int s[3];
    int nranks, per_rank;            // blocks per rank: [nrim | nfwd | nstencil]
    int nrim, nfwd, nstencil;
    int wait_prev;                   // tiles reading halos wait for the previous epoch's data flags
    int nchunks;
    int2 zr[kMaxChunks];             // z range of each chunk, in visit order (= chunk id)
    int zchunk[2];                   // chunk holding the z send layer of face (2, rs); -1 if none
    int xtiles, ytiles;
    int border_first;                // within a chunk: the border tiles (faces) first
    int nxs;                         // x sender (and x unpacker) blocks per x face / halo side (0: none)
    unsigned xtarget;                // x-face tile count of a chunk after this launch (cumulative)
    unsigned xtarget_prev;           // ... after the previous launch
    int defer_from;                  // x chunks [defer_from, nchunks) of this epoch are sent by the NEXT
                                     // launch's senders (nchunks: none deferred)
    int undefer_from;                // x chunks [undefer_from, nchunks) of the previous epoch, deferred by
                                     // the previous launch, are sent first by this launch's senders
    const unsigned int *tgt;         // [6][kMaxChunks] contributions completing a (face, chunk) data flag
    const unsigned int *tgt_x;       // ... an xflag (rim + forwarders)
    unsigned long long epoch;
    long long timeout_cycles;
    int *err;
    HeatCoef k;
    HeatCoefF kf;                    // (binary32 launches)
    FusedRank r[kMaxFusedRanks];
};

// ---------------------------------------------------------------- kernel launchers (kernels.cu)

// pack (op 0) or unpack (op 1) of any number of faces: chunks of kMaxCopy
// descriptors per launch; `proto` carries signals/waits/epoch; returns launches
int launch_copies(int op, const std::vector<CopyDesc> &descs, const CopyList &proto, cudaStream_t s);
// generic region kernel: any region list
void launch_heat_regions(HeatRegionList &L, cudaStream_t s);
// vectorised region-list kernel for thin boundary slabs (falls back to the generic kernel)
void launch_heat_slabs(HeatRegionList &L, cudaStream_t s);
// the production stencil: cp.async-pipelined z-sweep over a list of box regions
// (all local ranks' inner boxes, or the boundary slabs), one launch
void launch_heat_box_list(HeatRegionList &L, cudaStream_t s, int variant);
// binary32 heat step on the box [lo, hi) (size-1 axes allowed); coefficients rounded to float by the caller
HeatCoefF heat_coef_f32(float lam, float dt, float dx, float dy, float dz);
void launch_heat_f32(float *T2, const float *T, const float *Ci, const int n[3], const int lo[3], const int hi[3],
                     const HeatCoefF &k, cudaStream_t s, int variant);
// 1-D/2-D grid (size-1 axes): the stencil without the size-1 axes' terms on the updated box
void launch_heat_lowdim(double *T2, const double *T, const double *Ci, const int n[3], const HeatCoef &k,
                        cudaStream_t s);
// vectorised z-sweep kernel for one box region of an even-sx, 16-B aligned field
bool heat_box_vectorizable(const HeatRegion &r);
void launch_heat_box(const HeatRegion &r, const HeatCoef &k, cudaStream_t s, int variant);
// T2's six outer layers = T's (the cells of T2 = copy(T), that no step or exchange writes first)
void launch_copy_outer(double *T2, const double *T, const int n[3], cudaStream_t s);
// sub-box [b0, b1) of a field -> contiguous buffer (x fastest)
void launch_box_pack(const double *f, double *out, long long sx, long long sy, const int b0[3], const int b1[3],
                     cudaStream_t s);
// max over `count` doubles of each of n pointers -> partials -> *out_dev (one double)
void launch_field_max(const double *const *ptrs, int n, long long count, double *scratch,
                      int scratch_len, double *out_dev, cudaStream_t s);
int field_max_scratch_len();

// second workload (acoustic.cu): one rank's staggered fields P (n), Vx (n+1 in x), Vy, Vz
struct AcousticFields {
    double *P, *Vx, *Vy, *Vz;
    int n[3];
};
struct AcousticCoef {
    double cV[3];   // (dt/rho)/d
    double cP;      // dt*K
    double r[3];    // 1/d
};
// compute_V on the velocity box [lo, hi) (x in [1,nx), y in [1,ny), z in [1,nz))
void launch_acoustic_v(const AcousticFields &f, const AcousticCoef &c, const int lo[3], const int hi[3],
                       cudaStream_t s);
// compute_P on every cell
void launch_acoustic_p(const AcousticFields &f, const AcousticCoef &c, cudaStream_t s);
// compute_V then compute_P in one sweep from the in fields into every element of the out fields (a grid with
// no exchanged axis)
void launch_acoustic_fused(const AcousticFields &in, const AcousticFields &out, const AcousticCoef &c, cudaStream_t s);

// ---------------------------------------------------------------- geometry and exchange plan (plan.cpp)
// Validated grid geometry of one process (host only, no CUDA).
struct Geom {
    int n[3], o[3], dims[3], periods[3];
    long long ng[3];
    int nprocs, rank0, nlocal, nproc_procs, proc, device, path;
    std::vector<std::array<int, 3>> coords;              // per local rank
    std::vector<std::array<std::array<int, 2>, 3>> nbr;   // per local rank: [axis][0=lower,1=upper], -1 none
};
Geom make_geom(const igg_init_args *A);   // validates (IGG_E_ARG), fills topology

enum Transport { kLocal = 0, kNccl = 1, kP2P = 2 };
// one face of one update_halo call: op 0 packs a rank's send layers toward a
// receiver, op 1 unpacks a rank's receive layers
struct PlanMsg {
    int op, lr, field, recv_side, peer, peer_proc, peer_lr, transport;
    int lo, h;
    long long count;   // elements
    long long words;   // 8-byte words the face occupies in the arenas (NCCL message size)
    long long slot;    // word offset in the receive-arena half of the RECEIVING process
    long long sbuf;    // op 0, NCCL: word offset in the send arena
    int order;         // NCCL: posting position among this axis' sends (op 0) / recvs (op 1); else -1
};
struct Plan {
    long long block = 0;                                   // doubles per rank in the receive arena half
    std::vector<std::array<long long, 3>> sz;
    std::vector<std::array<std::array<long long, 2>, 3>> off;   // word offset of slot (field, axis, side)
    std::vector<PlanMsg> msgs[3];                          // per axis: all packs, then all unpacks
    bool any_nccl = false;
};
Plan build_plan(const Geom &G, const long long *sizes /* nf*3, (sx,sy,sz) */, int nf,
                const int *esz = nullptr /* nf bytes per element, default 8 */);

}  // namespace igg

// ---------------------------------------------------------------- the grid object
struct igg_grid : igg::Geom {
    bool finalized = false;

    // streams and events (transfers on non-blocking high-priority streams)
    cudaStream_t s_comm = nullptr, s_inner = nullptr, s_comm2 = nullptr;
    cudaEvent_t ev_start = nullptr, ev_comm = nullptr, ev_inner = nullptr, ev_bnd = nullptr, ev_comm2 = nullptr;

    // communicator: NCCL (comm), or the caller's host bootstrap (boot; then comm stays NULL)
    ncclComm_t comm = nullptr;
    igg_allgather_fn boot = nullptr;
    void *boot_user = nullptr;
    char *d_gather = nullptr;                            // small device buffer of allgather_bytes (NCCL)
    size_t d_gather_bytes = 0;

    // buffer pool: receive arena (two parity halves), send arena (NCCL path)
    char *recv_arena = nullptr;
    size_t recv_half = 0;                                // bytes per parity half
    char *send_arena = nullptr;
    size_t send_cap = 0;
    std::vector<char *> peer_recv;                       // per process: mapped recv arena (P2P)
    unsigned long long *flags = nullptr;                 // [nlocal][3][2] receive flags
    std::vector<unsigned long long *> peer_flags;        // per process: mapped flags (P2P)
    unsigned int *tickets = nullptr;                     // [3] pack last-block election
    int *d_err = nullptr;
    double *d_scratch = nullptr;                         // reductions
    double *d_pinned_out = nullptr;                      // host-pinned scalar
    unsigned long long epoch = 0;
    long long allocs = 0;
    long long launches = 0;

    // e2e scratch (igg_heat_run_host)
    double *run_T = nullptr, *run_T2 = nullptr, *run_Ci = nullptr;
    size_t run_bytes = 0;

    // profiling of the main stencil launches (IGG_OPT_PROFILE)
    int profile = 0;
    std::vector<cudaEvent_t> prof_ev;
    size_t prof_used = 0;
    long long prof_cells = 0;
    // timeline of the overlap schedule (IGG_OPT_PROFILE >= 2): per step 5 timing events
    // t0 (caller stream), boundary end, inner start, inner end, exchange end
    std::vector<cudaEvent_t> tl_ev;
    size_t tl_used = 0;

    // options
    bool skip_comm = false;
    bool skipped = false;                                // a step ran with skip_comm since the last check
    long long spin_timeout_ms = 20000;
    int stencil_kernel = 0;
    int x_align = 64;
    int schedule = 0;
    int fused = -1;                                      // IGG_OPT_FUSED (-1 auto)
    int fused_mode = 2;                                  // IGG_OPT_FUSED_MODE (ablation bits)
    int fused_kc2 = 0;                                   // IGG_OPT_FUSED_KC2: tail chunk planes (0 auto)
    int fused_ncomm = 1;                                 // IGG_OPT_FUSED_COMM_CTAS
    bool halo_on_caller = false;                         // IGG_OPT_HALO_STREAM
    bool local_p2p = false;                              // IGG_OPT_LOCAL_P2P
    int halo26 = 1;                                      // IGG_OPT_HALO26: P2P update_halo as one 26-neighbour kernel
    int fused_f32 = -1;                                  // IGG_OPT_FUSED_F32: binary32 steps through the fused kernel
                                                         // (-1: when the x axis is exchanged)
    unsigned int *h26_ctr = nullptr;                     // [claim, stores done]
    struct H26Cache {
        std::vector<long long> key;                      // field pointers, sizes, element sizes, arena
        void *dplan = nullptr;                           // device plan
        long long nchunks = 0;
    };
    std::vector<H26Cache> h26_cache;
    std::list<std::pair<std::vector<long long>, igg::Plan>> plan_cache;   // field-list shape -> plan
    unsigned int *fused_ctr = nullptr, *fused_tgt_x = nullptr, *fused_tgt_pipe = nullptr;
    int fused_geo[6] = {0, 0, 0, 0, 0, 0};               // [4] xtiles, [5] ytiles
    std::vector<int2> fused_zr;                          // z-chunks in visit order
    // peer mappings of arrays the fused path stores into (PeerMap: fused.cu)
    struct PeerMap {
        const void *ptr;                 // my array
        unsigned long long base, size;   // its allocation (cuMemGetAddressRange)
        unsigned long long buffer_id;    // CU_POINTER_ATTRIBUTE_BUFFER_ID: unique per allocation
        std::vector<double *> peers;     // per process: the same array of that process, mapped
    };
    std::vector<PeerMap> fused_peer_maps;
    std::vector<std::pair<std::string, void *>> fused_opened;                     // IPC handle -> mapping
    int fused_ntiles = 0, fused_nchunks = 0, fused_key = -1;
    int fused_zchunk[2] = {-1, -1};
    int fused_nfwd = 0;                                  // in-kernel forwarders (pipelined)
    double *fused_xloc = nullptr;                        // x-face local staging rows (fused path)
    unsigned int *fused_xcnt = nullptr;                  // x-face tile counters (cumulative)
    double *fused_xrem = nullptr;                        // x-face receive staging (IPC-mapped by the senders)
    unsigned long long fused_xsteps = 0;                 // launches with x faces since the counters' reset
    int fused_deferred = -1;                             // the last fused launch deferred x chunks from here (-1: none)
    int sm_count = 148;
    double clock_khz = 1.9e6;
};

namespace igg {
void exchange(igg_grid *g, const igg_field *fields, int nfields, cudaStream_t st, bool allow_coop = false);
// update_halo on the P2P path (halo26.cu): ONE kernel per call, every halo region -- faces, edges,
// corners -- stored straight from its owner into the receiver (26-neighbour single phase)
void exchange26(igg_grid *g, const igg_field *fields, int nfields, const Plan &plan, cudaStream_t st);
void release_h26(igg_grid *g);   // drop the cached device plans (they hold peer mappings)
const std::vector<double *> &peer_arrays_pub(igg_grid *g, double *arr);
constexpr int kH26Flags = 64;    // per hosted rank: data flags [0, 27), ready flags [32, 59) by direction
void check_live(const igg_grid *g, const char *what);
void heat_step(igg_grid *g, double *const *T2, const double *const *T, const double *const *Ci,
               double lam, double dt, double dx, double dy, double dz, const int bw[3],
               cudaStream_t s, bool wait_prev = false,
               bool drain = true);
void ensure_arena(igg_grid *g, size_t recv_half, size_t send_cap);
int local_index(const igg_grid *g, int global_rank);   // -1 if not hosted here
std::vector<char> allgather_bytes_pub(igg_grid *g, const void *mine, size_t bytes);
double host_max(igg_grid *g, double local);   // max of one double over the processes (host collective)
bool fused_eligible(const igg_grid *g);
// drop every peer mapping of caller arrays (collective: process barrier, close the IPC handles);
// the next fused step maps its arrays again
void release_peer_maps(igg_grid *g);
// collective: do all processes' cached peer mappings still describe live allocations?  If any does
// not, every process releases them (called once per igg_heat_run / igg_heat_run_host)
void validate_peer_maps(igg_grid *g);
// synchronizes the grid's device work and fails with IGG_E_TIMEOUT if a flag wait timed out
void check_device_error(igg_grid *g, const char *who);
// one fused step; pipelined schedule: wait_prev = the previous step of the same run was fused (its
// halos are awaited tile by tile), drain = wait for every incoming face at the end (step complete; a
// step that does not drain leaves its last x chunks to the next launch's senders)
void fused_step(igg_grid *g, double *const *T2, const double *const *T, const double *const *Ci, const HeatCoef &k,
                cudaStream_t s, bool wait_prev = false, bool drain = true);
// the same for binary32 fields
void fused_step_f32(igg_grid *g, float *const *T2, const float *const *T, const float *const *Ci,
                    const HeatCoefF &kf, cudaStream_t s, bool wait_prev = false, bool drain = true);
void prof_begin(igg_grid *g, cudaStream_t s);
void prof_end(igg_grid *g, cudaStream_t s, long long cells);
void tl_mark(igg_grid *g, cudaStream_t s, int k);   // k = 0..4 of the current step
int proc_of(const igg_grid *g, int global_rank);
const Plan &cached_plan(igg_grid *g, const std::vector<long long> &key, int nf);
}  // namespace igg
