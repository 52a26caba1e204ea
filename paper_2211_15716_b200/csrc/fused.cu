// fused.cu -- the fused hide_communication step: stencil + halo exchange as one-sided peer stores
// straight into the neighbours' arrays, published chunk by chunk (IGG_PATH_P2P).
//
// The paper hides update_halo! behind the inner-point computation ("pipelining is
// applied on all stages of the data transfers").  On B200 one stencil launch per step keeps
// the 1-GPU tile order (z-chunk, then y-tile, then x-tile: whole 4-KB rows stream together) and, when a
// tile holding send layers finishes its chunk, stores those cells directly into the receiving rank's
// memory -- over NVLink for a rank on another GPU (CUDA-IPC mapping), into the sibling's arrays for ranks
// hosted on the same GPU (pack, transfer and unpack fused into one store; the receiver's SMs do no copy
// work).  Faces are published per (face, z-chunk): each CTA holding part of face f in chunk c counts
// itself on counter (f, c) after a system fence; the contribution completing (f, c) release-stores the
// epoch into the receiver's flag (f, c).
//
// Pipelined schedule (igg_heat_run): step t's tiles that read halo cells wait, before their sweep, for
// step t-1's flags of exactly those cells; the z chunks holding the z send/halo layers are visited LAST
// in every step, so in the steady state no tile waits (the awaited faces were published a whole step
// earlier).  y and z faces land in the receiver's T2 halo rows/planes.  x faces (one value per row and
// plane: a T2 column) go through staging buffers laid out [parity][side][z][y] (a run of planes is one
// contiguous block): the send lanes store them into the LOCAL staging from the sweep, the tile counts
// itself after a GPU-scope release, and x sender blocks move 8-plane pieces into the receiver's staging
// under one system-scope release per piece (the last chunks of a step that does not complete its run are
// moved by the next launch's senders: no tail); the receiver's halo tiles read them into shared memory
// with their first cp.async group (never written into the T array being swept).  Face cells the stencil
// does not compute (global boundary,
// edges/corners of the dimension-sequential update_halo) are sent by rim blocks and
// forwarded by forwarder blocks of the LAST step of a run, which also drains (awaits every incoming
// face and copies the staged x columns into T2).  Hazard argument and forward progress: DESIGN.md §6.
// The final state is bit-identical to nt x {step!; update_halo!(T2)} (tests/test_gpu_virtual_p2p.py,
// tests/test_gpu_multi.py).
//
// Ranks hosted on one GPU (virtual ranks, one process) run as ONE launch over all ranks' tiles: their
// faces are the same peer stores and flags into the siblings' arrays -- the cross-rank data plane,
// emulated on one GPU (spinning kernels of separate launches are never relied on to be co-scheduled).
#include <algorithm>
#include <array>
#include <cstring>

#include "igg_internal.h"

namespace igg {

namespace {

// (after a fence.acq_rel: fence + relaxed store is the PTX release pattern; st.release would fence again)
__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void cp_async16f(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async8f(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

// element type E of the sweep: binary64 (the paper's Float64) or binary32.  A lane holds
// kV<E> x-adjacent cells, one 16-B vector (double2 / float4): a tile row is 32 kV<E> cells
template <typename E> struct VT;
template <> struct VT<double> { using t = double2; };
template <> struct VT<float> { using t = float4; };
template <typename E> using vec = typename VT<E>::t;
template <typename E> constexpr int kV = 16 / (int)sizeof(E);
template <typename E> constexpr int kTW = 32 * kV<E>;   // tile width in cells
template <typename E>
__device__ __forceinline__ vec<E> ldgv(const E *p) { return __ldg(reinterpret_cast<const vec<E> *>(p)); }
__device__ __forceinline__ double vget(const double2 &v, int k) { return k == 0 ? v.x : v.y; }
__device__ __forceinline__ float vget(const float4 &v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }
__device__ __forceinline__ void vset(double2 &v, int k, double a) { if (k == 0) v.x = a; else v.y = a; }
__device__ __forceinline__ void vset(float4 &v, int k, float a) {
    if (k == 0) v.x = a; else if (k == 1) v.y = a; else if (k == 2) v.z = a; else v.w = a;
}
template <typename E>
__device__ __forceinline__ vec<E> vzero() {
    vec<E> r;
#pragma unroll
    for (int k = 0; k < kV<E>; ++k) vset(r, k, E(0));
    return r;
}
template <typename E>
__device__ __forceinline__ void cp_elem(void *smem, const void *gmem) {   // one element
    if constexpr (sizeof(E) == 8) {
        cp_async8f(smem, gmem);
    } else {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
    }
}
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }

// the cell of PAPER.md:46-49, same explicitly rounded operations (and association) as kernels.cu's
// binary64 and binary32 kernels
template <typename E, typename K>
__device__ __forceinline__ E cell(E c, E xm, E xp, E ym, E yp, E zm, E zp, E ci, const K &k) {
    const E d2x = rsub(rsub(xp, c), rsub(c, xm));
    const E d2y = rsub(rsub(yp, c), rsub(c, ym));
    const E d2z = rsub(rsub(zp, c), rsub(c, zm));
    const E lap = radd(radd(rmul(d2x, k.rdx2), rmul(d2y, k.rdy2)), rmul(d2z, k.rdz2));
    return radd(c, rmul(k.dt, rmul(rmul(k.lam, ci), lap)));
}
__device__ __forceinline__ const HeatCoef &coef_of(const FusedParams &F, double) { return F.k; }
__device__ __forceinline__ const HeatCoefF &coef_of(const FusedParams &F, float) { return F.kf; }

// release / acquire fence at system scope: the PTX release and acquire patterns (fence.acq_rel + relaxed
// write / relaxed read + fence.acq_rel) are all the flag protocol needs; __threadfence_system is the
// heavier sequentially consistent fence.sc (measured ~6 us per face tile with NVLink stores outstanding)
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acq_gpu_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// one contribution to the data flag of (face a/rs, chunk c) of rank R; the last one publishes the epoch
__device__ __forceinline__ void contribute(const FusedParams &F, const FusedRank &R, int a, int rs, int c,
                                           unsigned long long ep) {
    const int i = (a * 2 + rs) * kMaxChunks + c;
    if (atomicAdd(R.ctr + i, 1u) == F.tgt[i] - 1) {
        fence_acq_rel_sys();   // (acquire side of the other contributors' release, then the flag's release)
        st_relaxed_sys(R.face[a][rs].flag + c, ep);
        atomicExch(R.ctr + i, 0u);
    }
}
// one x piece of (x face rs, chunk c) for epoch ep: counters by epoch parity (module comment at the
// deferral, fused_step), the chunk's count completing publishes ep
__device__ __forceinline__ void contribute_xp(const FusedParams &F, const FusedRank &R, int rs, int c,
                                              unsigned long long ep) {
    const int i = ((int)(ep & 1) * 2 + rs) * kMaxChunks + c;
    if (atomicAdd(R.xpc + i, 1u) == F.tgt[rs * kMaxChunks + c] - 1) {
        fence_acq_rel_sys();
        st_relaxed_sys(R.face[0][rs].flag + c, ep);
        atomicExch(R.xpc + i, 0u);
    }
}
// rim / forwarded cells of (face, chunk): their own counters and flags
__device__ __forceinline__ void contribute_x(const FusedParams &F, const FusedRank &R, int a, int rs, int c) {
    const int i = (a * 2 + rs) * kMaxChunks + c;
    if (atomicAdd(R.ctr_x + i, 1u) == F.tgt_x[i] - 1) {
        fence_acq_rel_sys();
        st_relaxed_sys(R.face[a][rs].xflag + c, F.epoch);
        atomicExch(R.ctr_x + i, 0u);
    }
}

// the calling thread spins (bounded) until *fl >= v; a timeout sets *err (igg_check: IGG_E_TIMEOUT)
__device__ __forceinline__ void spin_geq(const FusedParams &F, const unsigned long long *fl, unsigned long long v) {
    const long long t0 = clock64();
    while (ld_acq_sys(fl) < v) {
        if (clock64() - t0 > F.timeout_cycles) {
            atomicExch(F.err, 1);
            break;
        }
        __nanosleep(200);
    }
}

// the earlier axis whose unpack writes this cell last in the dimension-sequential exchange (-1: none)
// -- that phase forwards the cell to face a
__device__ __forceinline__ int forward_phase(const FusedParams &F, const FusedRank &R, int a, const int *c) {
    int fwd = -1;
    for (int b = 0; b < a; ++b) {
        if (c[b] == 0 && R.halo[b][0].active) fwd = b;
        if (c[b] == F.s[b] - 1 && R.halo[b][1].active) fwd = b;
    }
    return fwd;
}
// a later axis whose exchange writes this cell's receiver copy last: the cell is sent by that axis'
// phase (face or forwarding), never by this one -- so every receiver cell has ONE writer
__device__ __forceinline__ bool later_halo(const FusedParams &F, const FusedRank &R, int a, const int *c) {
    for (int b = a + 1; b < 3; ++b)
        if ((c[b] == 0 && R.halo[b][0].active) || (c[b] == F.s[b] - 1 && R.halo[b][1].active)) return true;
    return false;
}

// z range a chunk covers on the x- and y-faces (the rim planes 0 and s-1 go with the end chunks)
__device__ __forceinline__ int2 ext_range(const FusedParams &F, int c) {
    int2 r = F.zr[c];
    if (r.x == 1) r.x = 0;
    if (r.y == F.s[2] - 1) r.y = F.s[2];
    return r;
}

constexpr int kFTY = 4;    // rows per CTA (one warp each)
constexpr int kFD = 3;     // planes in flight per thread
constexpr int kFKC = 64;   // longest z-chunk

}  // namespace

// The z sweep of one tile: cp.async ring of kFD planes of T and Ci, x neighbours by shuffle, z by a
// register queue.  Faces leave from inside the sweep (no re-read of T2 afterwards):
//  * YF (CTA-uniform): the warp whose row is a y send layer stores its results also into the receiver's
//    halo row (ydst + i) -- the same 16-B stores as T2's (the z send layer, the first or last plane of an
//    end chunk, is copied after the sweep: one row per warp, just written);
//  * XS (CTA-uniform: the tile holds an x send layer): the lane holding the send cell stores its value of
//    every plane into this rank's LOCAL x staging ([z][y]), from which the x sender blocks move it into
//    the receiver's staging (one system-scope release per piece instead of one per face tile); the lane
//    holding the x halo cell substitutes the neighbour's staged value (sHx, fetched in the first cp.async
//    group) for T's, plane by plane.
// The element type E is binary64 or binary32; a lane holds one 16-B vector of kV<E> cells.
#ifndef FUSED_STCS
#define FUSED_STCS 1
#endif
// the lane's kV cells at d, cell k only where bit k of wm is set (a 16-B store when all are)
template <typename E>
__device__ __forceinline__ void store_vec(E *d, unsigned wm, const vec<E> &r) {
    if (wm == (1u << kV<E>) - 1) {
        *reinterpret_cast<vec<E> *>(d) = r;
    } else {
#pragma unroll
        for (int k = 0; k < kV<E>; ++k)
            if (wm >> k & 1) d[k] = vget(r, k);
    }
}

// UP (XS only): the tile holds the upper x send layer s-2 and the halo s-1 -- elements V-2 and V-1 of their
// lanes' vectors (s is a multiple of V) -- else the lower send layer 1 and the halo 0: elements 1 and 0
// (compile-time element choice: a run-time index measured 8 us slower per step at 2x1x1)
template <typename E, bool YF, bool XS, bool UP>
__device__ __forceinline__ void fused_sweep(const FusedParams &F, const FusedRank &R, vec<E> (*sT)[32 * kFTY],
                                            vec<E> (*sC)[32 * kFTY], int sx, long long sxy, int zs, int ze,
                                            long long i, bool row_in, unsigned wm, E *ydst, E *xdst, int xs, bool slane,
                                            bool hpatch, E h0, const E *hx_row) {
    constexpr int V = kV<E>;
    constexpr int es = UP ? V - 2 : 1, eh = UP ? V - 1 : 0;
    const E *__restrict__ T = reinterpret_cast<const E *>(R.T);
    const E *__restrict__ Ci = reinterpret_cast<const E *>(R.Ci);
    E *__restrict__ T2 = reinterpret_cast<E *>(R.T2);
    const int tid = threadIdx.x, lane = tid & 31;
#pragma unroll
    for (int q = 0; q < kFD; ++q) {
        if (row_in && zs + q < ze) {
            cp_async16f(&sT[q][tid], T + i + (q + 1) * sxy);
            cp_async16f(&sC[q][tid], Ci + i + q * sxy);
        }
        cp_commit();
    }
    const vec<E> zero = vzero<E>();
    vec<E> zm = row_in ? ldgv(T + i - sxy) : zero;
    vec<E> c = row_in ? ldgv(T + i) : zero;
    if (XS && hpatch) vset(c, eh, h0);   // (one lane) the staged x halo value instead of T's, plane zs first
    const bool lo_edge = lane == 0 && (wm & 1u), hi_edge = lane == 31 && (wm >> (V - 1) & 1u);
    const bool full = wm == (1u << V) - 1;
    int slot = 0;
#pragma unroll 2
    for (int z = zs; z < ze; ++z, i += sxy) {
        cp_wait<kFD - 1>();
        if (XS) __syncwarp();   // (the halo row in hx_row, fetched by the whole warp in group 0)
        vec<E> ym = zero, yp = zero;
        if (row_in) {
            ym = ldgv(T + i - sx);
            yp = ldgv(T + i + sx);
        }
        const vec<E> zp = sT[slot][tid];
        const vec<E> ci = sC[slot][tid];
        E xm = __shfl_up_sync(0xffffffffu, vget(c, V - 1), 1);
        E xp = __shfl_down_sync(0xffffffffu, vget(c, 0), 1);
        if (lo_edge) xm = __ldg(T + i - 1);
        if (hi_edge) xp = __ldg(T + i + V);
        vec<E> r;
#pragma unroll
        for (int k = 0; k < V; ++k)
            vset(r, k, cell(vget(c, k), k == 0 ? xm : vget(c, k - 1), k == V - 1 ? xp : vget(c, k + 1), vget(ym, k),
                            vget(yp, k), vget(zm, k), vget(zp, k), vget(ci, k), coef_of(F, E())));
        if (FUSED_STCS && full)   // T2 is not re-read in this step (evict-first keeps L2 for T)
            __stcs(reinterpret_cast<vec<E> *>(T2 + i), r);
        else
            store_vec(T2 + i, wm, r);
        if (YF && ydst) store_vec(ydst + i, wm, r);   // (warp-uniform) y face row: ydst + i
        if (XS && slane) xdst[(long long)z * xs] = vget(r, es);   // (one lane) the x send cell -> local staging
        zm = c;
        c = zp;
        if (XS && hpatch && z + 1 < ze) vset(c, eh, hx_row[z + 1 - zs]);   // plane z+1's staged x halo cell
        if (row_in && z + kFD < ze) {
            cp_async16f(&sT[slot][tid], T + i + (kFD + 1) * sxy);
            cp_async16f(&sC[slot][tid], Ci + i + kFD * sxy);
        }
        cp_commit();
        slot = slot + 1 == kFD ? 0 : slot + 1;
    }
    cp_wait<0>();
}

template <typename E>
__device__ __noinline__ void fused_extra(const FusedParams &F, const FusedRank &R, int b);

#ifndef FUSED_TRACE
#define FUSED_TRACE 0   // diagnostics build only: per-block %globaltimer stamps into g_fused_trace
#endif
#if FUSED_TRACE
__device__ unsigned long long g_fused_trace[65536 * 4];
__device__ unsigned long long g_trace_epoch;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TRACE_AT(k) \
    if (threadIdx.x == 0 && blockIdx.x < 65536 && F.epoch == g_trace_epoch) g_fused_trace[blockIdx.x * 4 + (k)] = gtimer()
#else
#define TRACE_AT(k)
#endif

// One launch over all tiles of all hosted ranks, the 1-GPU loop unchanged.  Block b of rank r:
// [0, nrim) rim, [nrim, nrim+nfwd) forwarders (last step of a run only), then the stencil tiles.
// MR: more than one hosted rank (the rank's parameters are indexed at run time).
template <bool MR, typename E>
__global__ void __launch_bounds__(32 * kFTY, 10) heat_fused_kernel(const __grid_constant__ FusedParams F) {
    TRACE_AT(0);
    __shared__ vec<E> sT[kFD][32 * kFTY];
    __shared__ vec<E> sC[kFD][32 * kFTY];
    __shared__ E sHx[kFTY][kFKC];  // the staged x halo cells of each row, plane by plane
    // (the rank index stays a run-time value even for one rank: the parameters are then read through
    // uniform registers instead of being re-materialised from the constant bank in the sweep)
    const int rank = blockIdx.x / F.per_rank;
    int b = blockIdx.x - rank * F.per_rank;
    const FusedRank &R = F.r[rank];
    if (b < F.nrim + F.nfwd + 2 * F.nxs) {   // CTA-uniform
        fused_extra<E>(F, R, b);
        TRACE_AT(3);
        return;
    }
    b -= F.nrim + F.nfwd + 2 * F.nxs;
    // tile of this block: chunks in visit order; within a chunk, when x or y faces exist, the border
    // tiles (rows ty = 0 and ytiles-1, then columns tx = 0 and xtiles-1) first -- they carry the faces and
    // take longer, so they start early instead of trailing their chunk -- then the interior, row-major.
    // (Border tiles of chunk c+1 placed before the interior of chunk c measured slower: 2x1x1 exposed
    // halo 35 us instead of 25.)
    const int nt = F.xtiles * F.ytiles, pos = b / nt;
    int tx, ty;
    {
        const int xt = F.xtiles, yt = F.ytiles, t = b - pos * nt;
        const bool ring = xt > 2 && yt > 2;   // (else every tile is a border tile, row-major)
        const int nrow = xt * 2, nborder = nrow + 2 * (yt - 2);
        if (!F.border_first || !ring) {
            tx = t % xt;
            ty = t / xt;
        } else if (t < xt) {
            tx = t;
            ty = 0;
        } else if (t < nrow) {
            tx = t - xt;
            ty = yt - 1;
        } else if (t < nborder) {
            const int u = t - nrow;
            ty = 1 + (u >> 1);
            tx = (u & 1) ? xt - 1 : 0;
        } else {
            const int v = t - nborder;
            tx = 1 + v % (xt - 2);
            ty = 1 + v / (xt - 2);
        }
    }
    const int2 zr = F.zr[pos];
    const int zs = zr.x, ze = zr.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if FUSED_TRACE
    if (tid == 0 && blockIdx.x < 65536 && F.epoch == g_trace_epoch)
        g_fused_trace[blockIdx.x * 4 + 2] = (unsigned long long)tx | ((unsigned long long)ty << 8) | ((unsigned long long)pos << 20);
#endif
    const int sx = F.s[0], sy = F.s[1];
    const int ty0 = 1 + ty * kFTY;
    const int y = ty0 + warp;
    constexpr int V = kV<E>, TW = kTW<E>;
    const int p = tx * TW + V * lane;   // my first cell
    const bool rowv = y < sy - 1;
    const bool row_in = rowv && p < sx;   // (sx is a multiple of V: a lane's cells are all in or all out)
    unsigned wm = 0u;                     // the cells of my vector that this step writes
#pragma unroll
    for (int k = 0; k < V; ++k)
        if (row_in && p + k >= 1 && p + k < sx - 1) wm |= 1u << k;
    const long long sxy = (long long)sx * sy;
    const int xlo = max(tx * TW, 1), xhi = min(tx * TW + TW, sx - 1);   // inner x of this tile
    const int yhi = min(ty0 + kFTY, sy - 1);

    // faces this tile holds (bit f = 2a + rs; rs 0: my upper send layer -> the upper neighbour's halo 0,
    // rs 1: my layer 1 -> the lower neighbour's halo s-1)
    unsigned did = 0u;
    int xrs = -1;
#pragma unroll
    for (int rs = 0; rs < 2; ++rs) {
        if (R.face[0][rs].active && R.face[0][rs].layer >= xlo && R.face[0][rs].layer < xhi) {
            did |= 1u << rs;
            xrs = rs;
        }
        if (R.face[1][rs].active && R.face[1][rs].layer >= ty0 && R.face[1][rs].layer < yhi) did |= 4u << rs;
        if (R.face[2][rs].active && F.zchunk[rs] == pos) did |= 16u << rs;
    }
    if (F.wait_prev) {   // CTA-uniform: this step's halo cells are the previous epoch's faces
        const bool xh0 = R.halo[0][0].active && tx == 0, xh1 = R.halo[0][1].active && tx == F.xtiles - 1;
        const bool yl = R.halo[1][0].active && ty == 0, yu = R.halo[1][1].active && ty == F.ytiles - 1;
        const bool zl = R.halo[2][0].active && zs == 1, zu = R.halo[2][1].active && ze == F.s[2] - 1;
        if (tid == 0) {
            const unsigned long long prev = F.epoch - 1;
            if (xh0) spin_geq(F, R.halo[0][0].flag + pos, prev);   // (the neighbour's senders staged it)
            if (xh1) spin_geq(F, R.halo[0][1].flag + pos, prev);
            if (yl) spin_geq(F, R.halo[1][0].flag + pos, prev);
            if (yu) spin_geq(F, R.halo[1][1].flag + pos, prev);
            if (zl) spin_geq(F, R.halo[2][0].flag, prev);
            if (zu) spin_geq(F, R.halo[2][1].flag, prev);
        }
        __syncthreads();
    }

    // ---- the z sweep, with the x and y faces stored from inside it
    const long long i0 = (long long)zs * sxy + (long long)y * sx + p;
    {
        E *ydst = nullptr;
        if (did & 12u) {
            const int rs = (did & 4u) ? 0 : 1;
            if (rowv && y == R.face[1][rs].layer)   // (warp-uniform) my row is the y send layer: cell i of
                                                    // my row lands at ydst + i in the receiver's halo row
                ydst = reinterpret_cast<E *>(R.face[1][rs].dst) + (long long)((rs == 0 ? 0 : sy - 1) - y) * sx;
        }
        if (xrs >= 0) {
            const int xf = R.face[0][xrs].layer - tx * TW;
            const bool slane = rowv && xf / V == lane;
            // (local staging [parity][side][z][y]: the next launch's senders may still copy this epoch's
            // deferred chunks while its own tiles stage theirs)
            E *xloc = reinterpret_cast<E *>(R.xloc) + ((long long)(F.epoch & 1) * 2 + xrs) * sy * F.s[2];
            // the x halo column beside the send layer: the neighbour's previous-epoch values, staged in my
            // receive rows by its senders (first step of a run: T holds it)
            const int hside = xrs == 0 ? 1 : 0, xh = (hside == 0 ? 0 : sx - 1) - tx * TW;
            const E *hrow = (F.wait_prev && R.halo[0][hside].active && rowv)
                                ? reinterpret_cast<const E *>(R.xrem) +
                                      ((long long)((F.epoch - 1) & 1) * 2 + hside) * sy * F.s[2] + y
                                : nullptr;   // (cell z of the row at hrow[z sy])
            const bool hpatch = hrow && xh / V == lane;
            E h0 = E(0);
            if (hrow) {   // (warp-uniform) this chunk's staged halo values of the row, into the first group
                for (int z = zs + lane; z < ze; z += 32) cp_elem<E>(&sHx[warp][z - zs], hrow + (long long)z * sy);
                if (hpatch) h0 = __ldcg(hrow + (long long)zs * sy);
            }
#define XSWEEP(YFv, UPv, YD) fused_sweep<E, YFv, true, UPv>(F, R, sT, sC, sx, sxy, zs, ze, i0, row_in, wm, YD, \
                                                             xloc + y, sy, slane, hpatch, h0, sHx[warp])
            if (xrs == 0) {   // upper: send layer s-2
                if (did & 12u) XSWEEP(true, true, ydst); else XSWEEP(false, true, nullptr);
            } else {          // lower: send layer 1
                if (did & 12u) XSWEEP(true, false, ydst); else XSWEEP(false, false, nullptr);
            }
#undef XSWEEP
        } else if (did & 12u) {
            fused_sweep<E, true, false, false>(F, R, sT, sC, sx, sxy, zs, ze, i0, row_in, wm, ydst, nullptr, 0, false,
                                               false, E(0), nullptr);
        } else {
            fused_sweep<E, false, false, false>(F, R, sT, sC, sx, sxy, zs, ze, i0, row_in, wm, nullptr, nullptr, 0,
                                                false, false, E(0), nullptr);
        }
    }
    if (did & 48u) {   // z face: my row of the layer plane (written by this thread just now) -> the receiver
        const int rs = (did & 16u) ? 0 : 1;
        const FusedFace &fz = R.face[2][rs];
        if (row_in) {
            const long long o = (long long)fz.layer * sxy + (long long)y * sx + p;
            const vec<E> v = *reinterpret_cast<const vec<E> *>(reinterpret_cast<const E *>(R.T2) + o);
            store_vec(reinterpret_cast<E *>(fz.dst) + o + (long long)((rs == 0 ? 0 : F.s[2] - 1) - fz.layer) * sxy,
                      wm, v);
        }
    }
    TRACE_AT(1);
    if (!did) {   // CTA-uniform
        TRACE_AT(3);
        return;
    }
    // one system-scope release for the CTA: the barrier orders every warp's face stores before thread
    // 0's fence.acq_rel, which is cumulative (PTX memory model), then the relaxed counters
    __syncthreads();
    if (tid == 0) {
        if (did & 60u) {   // y / z faces: their stores went to the receiver: system-scope release
#ifndef FUSED_DIAG_NOFENCE   // (diagnostics build: timing without the release, INVALID ordering)
#ifdef FUSED_DIAG_SCFENCE
            __threadfence_system();
#else
            fence_acq_rel_sys();
#endif
#endif
            for (int f = 2; f < 6; ++f)
                if (did & (1u << f)) contribute(F, R, f >> 1, f & 1, f < 4 ? pos : 0, F.epoch);
        }
        if (did & 3u) {    // x face: the local staging rows, GPU-scope release, then the senders' count
            fence_acq_rel_gpu();
            atomicAdd(R.xcnt + xrs * kMaxChunks + pos, 1u);
        }
    }
    TRACE_AT(3);
}

// forward my fresh halo line (axis b, side) x (face a, rs) over the third axis range [lo, hi)
template <typename E>
__device__ __forceinline__ bool forward_line(const FusedParams &F, const FusedRank &R, int b, int side, int a, int rs,
                                             int lo, int hi, int part, int nparts) {
    const FusedFace &fc = R.face[a][rs];
    if (!fc.active || !R.halo[b][side].active) return false;
    const int third = 3 - a - b;
    bool any = false;
    for (int t = lo + part * blockDim.x + threadIdx.x; t < hi; t += nparts * blockDim.x) {
        int c[3];
        c[b] = side == 0 ? 0 : F.s[b] - 1;
        c[a] = fc.layer;
        c[third] = t;
        if (forward_phase(F, R, a, c) != b || later_halo(F, R, a, c)) continue;
        E v;
        if (b == 0 && c[1] >= 1 && c[1] < F.s[1] - 1 && c[2] >= 1 && c[2] < F.s[2] - 1)   // staged, not in T2
            v = __ldcg(reinterpret_cast<const E *>(R.xrem) + ((long long)(F.epoch & 1) * 2 + side) * F.s[1] * F.s[2] +
                       (long long)c[2] * F.s[1] + c[1]);
        else
            v = __ldcg(reinterpret_cast<const E *>(R.T2) + ((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]);
        c[a] = rs == 0 ? 0 : F.s[a] - 1;
        reinterpret_cast<E *>(fc.dst)[((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]] = v;
        any = true;
    }
    return any;
}

// Rim and forwarders, extra blocks of the last step's launch.  Rim (blocks [0, nrim), six faces x
// nrim/6 blocks): the face cells the stencil does not compute that keep a value no earlier axis
// delivers (global-boundary values; cells a later axis overwrites are skipped); the last rim block counts
// once on every (face, chunk).  Forwarders (the next nfwd blocks): per chunk, wait for the x (then y)
// halo of the chunk -- its data and its rim/forwarded cells -- forward the edge lines later faces take
// from it, and count on those faces' xflags.  Only these few blocks wait on blocks of the same launch
// (the sibling ranks' or the peers' tiles): DESIGN.md §6 "forward progress".
// planes [za, zb) of the [z][y] x staging -- one contiguous block -- from my local staging to the
// receiver's: a flat copy, 16-B vectors when aligned, U vectors in flight per thread.  The senders take
// pieces of <= kFusedXPiece planes round-robin in chunk order, so a chunk's pieces move in parallel on
// several SMs (one SM drains NVLink stores at only ~6 GB/s: a 64-plane chunk took 45 us in one block)
// while each sender's pieces lie in different chunks.  (All senders copying a slice of every chunk
// measured slower: each pays a system fence per chunk in sequence.)
template <typename E>
__device__ __forceinline__ void x_piece_copy(const E *loc, E *dst, int za, int zb, int sy) {
    constexpr int W = 16 / sizeof(E);   // elements per 16-B word
    long long a0 = (long long)za * sy;
    const long long a1 = (long long)zb * sy;
    constexpr int U = 4;
    // (head up to a 16-B boundary; the local and the receiver's staging blocks have the same offsets from
    // 16-B aligned allocations, so both are aligned from there on)
    for (; a0 < a1 && (reinterpret_cast<uintptr_t>(loc + a0) % 16); ++a0)
        if (threadIdx.x == 0) dst[a0] = __ldcg(loc + a0);
    if (a0 < a1) {
        const uint4 *s2 = reinterpret_cast<const uint4 *>(loc + a0);
        uint4 *d2 = reinterpret_cast<uint4 *>(dst + a0);
        const long long n2 = (a1 - a0) / W;
        for (long long t0 = threadIdx.x; t0 < n2; t0 += (long long)blockDim.x * U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long t = t0 + (long long)u * blockDim.x;
                if (t < n2) v[u] = __ldcg(s2 + t);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long t = t0 + (long long)u * blockDim.x;
                if (t < n2) d2[t] = v[u];
            }
        }
        for (long long t = a0 + n2 * W + threadIdx.x; t < a1; t += blockDim.x) dst[t] = __ldcg(loc + t);   // tail
    }
}

template <typename E>
__device__ __noinline__ void fused_extra(const FusedParams &F, const FusedRank &R, int b) {
    if (b < F.nrim) {
        const int per = F.nrim / 6;
        const int f = b / per, part = b % per, a = f >> 1, rs = f & 1;
        const FusedFace &fc = R.face[a][rs];
        if (fc.active) {
            const int b1 = a == 0 ? 1 : 0, b2 = a == 2 ? 1 : 2;
            const int S1 = F.s[b1], S2 = F.s[b2];
            const long long nrim = 2LL * S2 + 2LL * (S1 - 2);
            for (long long t = (long long)part * blockDim.x + threadIdx.x; t < nrim;
                 t += (long long)per * blockDim.x) {
                int u, v;
                if (t < 2LL * S2) {
                    u = t < S2 ? 0 : S1 - 1;
                    v = (int)(t % S2);
                } else {
                    const long long r = t - 2LL * S2;
                    u = 1 + (int)(r % (S1 - 2));
                    v = r < (S1 - 2) ? 0 : S2 - 1;
                }
                int c[3];
                c[a] = fc.layer;
                c[b1] = u;
                c[b2] = v;
                if (forward_phase(F, R, a, c) >= 0 || later_halo(F, R, a, c)) continue;
                const E val = reinterpret_cast<const E *>(R.T2)[((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]];
                c[a] = rs == 0 ? 0 : F.s[a] - 1;
                reinterpret_cast<E *>(fc.dst)[((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]] = val;
            }
            fence_acq_rel_sys();
        }
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(R.rim_ticket, 1u) == (unsigned)F.nrim - 1) {
            fence_acq_rel_sys();
            for (int g = 0; g < 6; ++g) {
                const int ga = g >> 1, grs = g & 1;
                if (!R.face[ga][grs].active) continue;
                if (ga == 2)
                    contribute_x(F, R, 2, grs, 0);
                else
                    for (int ch = 0; ch < F.nchunks; ++ch) contribute_x(F, R, ga, grs, ch);
            }
            atomicExch(R.rim_ticket, 0u);
        }
        return;
    }
    if (b >= F.nrim + F.nfwd) {   // x sender: role rs, part of nxs
        const int e = b - F.nrim - F.nfwd, rs = e / F.nxs, part = e % F.nxs;
        const FusedFace &fx = R.face[0][rs];
        if (!fx.active) return;
        const int sy = F.s[1], sz = F.s[2];
        // pass 0: the previous epoch's deferred chunks (its tiles staged them in the other parity; the
        // previous launch is complete, so their count is in); pass 1: this epoch's chunks before defer_from
        for (int pass = 0; pass < 2; ++pass) {
            const unsigned long long ep = pass ? F.epoch : F.epoch - 1;
            const int c0 = pass ? 0 : F.undefer_from, c1 = pass ? F.defer_from : F.nchunks;
            const unsigned target = pass ? F.xtarget : F.xtarget_prev;
            const E *loc = reinterpret_cast<const E *>(R.xloc) + ((long long)(ep & 1) * 2 + rs) * sy * sz;
            // the receiver's staging of its halo side rs ([z][y]), the epoch's parity
            E *dst = reinterpret_cast<E *>(R.xrem_peer[rs]) + ((long long)(ep & 1) * 2 + rs) * sy * sz;
            int u = 0;   // piece index, in chunk order
            for (int pos = 0; pos < c1; ++pos) {
              const int2 zr = F.zr[pos];
              for (int za = zr.x; za < zr.y; za += kFusedXPiece, ++u) {
                if (pos < c0 || u % F.nxs != part) continue;
                if (threadIdx.x == 0) {   // every face tile of the chunk has staged its rows (GPU-scope acquire)
                    const long long t0 = clock64();
                    while (ld_acq_gpu_u32(R.xcnt + rs * kMaxChunks + pos) < target) {
                        if (clock64() - t0 > F.timeout_cycles) {
                            atomicExch(F.err, 1);
                            break;
                        }
                        __nanosleep(200);
                    }
                }
                __syncthreads();
                TRACE_AT(1);
                x_piece_copy(loc, dst, za, min(za + kFusedXPiece, zr.y), sy);
                __syncthreads();
                TRACE_AT(2);
                if (threadIdx.x == 0) {
                    fence_acq_rel_sys();
                    contribute_xp(F, R, rs, pos, ep);   // (the chunk's last piece publishes it)
                }
              }
            }
        }
        return;
    }
    const int q = b - F.nrim;   // forwarder q of nfwd: chunk by chunk, each edge line leaves as soon as
                                // its halo has arrived
    for (int ch = 0; ch < F.nchunks; ++ch) {
        const int2 zr = ext_range(F, ch);
        for (int hb = 0; hb < 2; ++hb) {
            if (!(R.halo[hb][0].active || R.halo[hb][1].active)) continue;
            if (threadIdx.x == 0)
                for (int side = 0; side < 2; ++side)
                    if (R.halo[hb][side].active) {
                        spin_geq(F, R.halo[hb][side].flag + ch, F.epoch);
                        spin_geq(F, R.halo[hb][side].xflag + ch, F.epoch);
                    }
            __syncthreads();
            bool fwd = false;
            for (int side = 0; side < 2; ++side)
                for (int rs = 0; rs < 2; ++rs) {
                    if (hb == 0) fwd |= forward_line<E>(F, R, 0, side, 1, rs, zr.x, zr.y, q, F.nfwd);
                    if (R.face[2][rs].layer >= zr.x && R.face[2][rs].layer < zr.y)
                        fwd |= forward_line<E>(F, R, hb, side, 2, rs, 0, F.s[hb == 0 ? 1 : 0], q, F.nfwd);
                }
            if (__syncthreads_or(fwd)) fence_acq_rel_sys();
            __syncthreads();
            if (threadIdx.x == 0)
                for (int a = hb + 1; a < 3; ++a)
                    for (int rs = 0; rs < 2; ++rs) {
                        if (!R.face[a][rs].active) continue;
                        if (a == 1)
                            contribute_x(F, R, 1, rs, ch);
                        else if (R.face[2][rs].layer >= zr.x && R.face[2][rs].layer < zr.y)
                            contribute_x(F, R, 2, rs, 0);
                    }
        }
    }
}

// After the last step of a run: every incoming face (data and rim/forwarded cells) of the epoch has
// arrived -- the step is complete for any later work on the stream -- and the last epoch's staged x halo
// columns (inner rows and planes) are copied into T2.  blockIdx.y = hosted rank.  (Waits only for flags
// of the launch before it on the stream.)
template <typename E>
__global__ void fused_drain_kernel(const __grid_constant__ FusedParams F) {
    const FusedRank &R = F.r[blockIdx.y];
    for (int f = threadIdx.x; f < 6 * F.nchunks; f += blockDim.x) {
        const int a = f / (2 * F.nchunks), rs = (f / F.nchunks) & 1, ch = f % F.nchunks;
        const FusedHalo &h = R.halo[a][rs];
        if (!h.active || (a == 2 && ch > 0)) continue;
        if (blockIdx.x == 0 || a == 0) spin_geq(F, h.flag + ch, F.epoch);   // (x data: every block copies)
        if (blockIdx.x == 0) spin_geq(F, h.xflag + ch, F.epoch);
    }
    __syncthreads();
    const int sx = F.s[0], sy = F.s[1], sz = F.s[2];
    const long long sxy = (long long)sx * sy, ncell = (long long)(sy - 2) * (sz - 2);
    for (int side = 0; side < 2; ++side) {
        if (!R.halo[0][side].active) continue;
        const int hx = side == 0 ? 0 : sx - 1;
        const E *stg = reinterpret_cast<const E *>(R.xrem) + ((long long)(F.epoch & 1) * 2 + side) * sy * sz;
        for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ncell;
             t += (long long)gridDim.x * blockDim.x) {
            const int y = 1 + (int)(t % (sy - 2)), z = 1 + (int)(t / (sy - 2));
            reinterpret_cast<E *>(R.T2)[(long long)z * sxy + (long long)y * sx + hx] = __ldcg(stg + (long long)z * sy + y);
        }
    }
}

// ------------------------------------------------------------------ host side
bool fused_eligible(const igg_grid *g) {
    if (g->path != IGG_PATH_P2P || g->fused == 0) return false;
    // one rank per process (peers on other GPUs), or every rank in this process (siblings on this GPU)
    if (!(g->nlocal == 1 || (g->nproc_procs == 1 && g->nlocal <= kMaxFusedRanks))) return false;
    bool any = false;
    for (int lr = 0; lr < g->nlocal; ++lr)
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < 2; ++k) any = any || g->nbr[lr][a][k] >= 0;
    if (!any) return false;                                            // nothing to exchange: plain stencil
    if (g->n[0] < 66 || g->n[0] % 2 || g->n[1] < 6 || g->n[2] < 6) return false;   // 16-B pairs, 2+ x-tiles
    return true;
}

static int g_fused_occ = -1, g_fused_nsm = 0;

// Chunks: the z range in 64-plane chunks, except about two waves' worth of tile-planes at the two ends
// in short chunks; visit order: the long middle chunks, then the short end chunks (bottom ones, then top
// ones).  The end chunks hold the z send/halo layers (planes 1, 2 .. s-3, s-2), so a step's z halo
// reads come last and wait for nothing in the steady state, and the short chunks shorten the tail.
// Depends on the geometry only: every rank numbers chunks identically (flags are per chunk position).
static void build_layout(igg_grid *g, const bool act[3][2], bool zex, int tw) {
    const int n0 = g->n[0], n1 = g->n[1], n2 = g->n[2];
    const int xtiles = (n0 - 1 + tw - 1) / tw;   // (tw: tile width in cells, 32 lanes x one 16-B vector)
    const int ytiles = (n1 - 2 + kFTY - 1) / kFTY;
    const int wz = n2 - 2;
    if (g_fused_occ < 0) {
        IGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_fused_occ, heat_fused_kernel<false, double>, 32 * kFTY, 0));
        IGG_CUDA(cudaDeviceGetAttribute(&g_fused_nsm, cudaDevAttrMultiProcessorCount, g->device));
    }
    const int kc1 = kFKC, kc2 = g->fused_kc2 > 0 ? g->fused_kc2 : 8;
    const long long ntile = (long long)xtiles * ytiles * g->nlocal;
    int small = (int)((2LL * g_fused_occ * g_fused_nsm * kc2 + ntile - 1) / ntile);
    small = std::min(((small + kc2 - 1) / kc2) * kc2, wz);
    if (zex) small = std::max(small, std::min(2 * kc2, wz));   // at least one short chunk at each end
    const int nbig = (wz - small) / kc1;
    const int rest = wz - nbig * kc1;                  // short planes, split between the two ends
    const int bot = zex ? std::min(rest, ((rest / 2 + kc2 - 1) / kc2) * kc2) : 0;
    std::vector<int2> zc;   // visit order
    for (int c = 0; c < nbig; ++c) zc.push_back(make_int2(1 + bot + c * kc1, 1 + bot + (c + 1) * kc1));
    for (int z = 1; z < 1 + bot; z += kc2) zc.push_back(make_int2(z, std::min(z + kc2, 1 + bot)));
    for (int z = 1 + bot + nbig * kc1; z < 1 + wz; z += kc2) zc.push_back(make_int2(z, std::min(z + kc2, 1 + wz)));
    const int nch = (int)zc.size();
    if (nch > kMaxChunks) fail(IGG_E_UNSUPPORTED, "fused step: too many z-chunks");
    g->fused_zr = zc;
    g->fused_zchunk[0] = g->fused_zchunk[1] = -1;
    for (int c = 0; c < nch; ++c) {
        if (n2 - 2 >= zc[c].x && n2 - 2 < zc[c].y) g->fused_zchunk[0] = c;   // upper z send layer
        if (1 >= zc[c].x && 1 < zc[c].y) g->fused_zchunk[1] = c;             // lower z send layer
    }
    // targets: contributions completing a (face, chunk) -- data flags: the stencil tiles holding it;
    // xflags: the rim (1) and the forwarders (when a later face takes an earlier axis' halo lines)
    bool xh = false, yh = false;
    for (int lr = 0; lr < g->nlocal; ++lr)
        for (int sd = 0; sd < 2; ++sd) {
            xh = xh || g->nbr[lr][0][sd] >= 0;
            yh = yh || g->nbr[lr][1][sd] >= 0;
        }
    const bool yf = act[1][0] || act[1][1], zf = act[2][0] || act[2][1];
    const bool need_fwd = (xh && (yf || zf)) || (yh && zf);
    g->fused_nfwd = need_fwd ? g->fused_ncomm : 0;
    const unsigned nf = (unsigned)g->fused_nfwd;
    std::vector<unsigned> tgt_d(6 * kMaxChunks, 0u), tgt_x(6 * kMaxChunks, 0u);
    for (int rs = 0; rs < 2; ++rs) {
        for (int c = 0; c < nch; ++c) {
            // (the x senders' pieces of the chunk publish its x face)
            tgt_d[(0 * 2 + rs) * kMaxChunks + c] = (zc[c].y - zc[c].x + kFusedXPiece - 1) / kFusedXPiece;
            tgt_x[(0 * 2 + rs) * kMaxChunks + c] = 1;
            tgt_d[(1 * 2 + rs) * kMaxChunks + c] = xtiles;
            tgt_x[(1 * 2 + rs) * kMaxChunks + c] = 1 + (xh ? nf : 0);
        }
        tgt_d[(2 * 2 + rs) * kMaxChunks] = xtiles * ytiles;
        tgt_x[(2 * 2 + rs) * kMaxChunks] = 1 + (xh ? nf : 0) + (yh ? nf : 0);
    }
    for (auto *pp : {&g->fused_tgt_pipe, &g->fused_tgt_x})
        if (!*pp) {
            IGG_CUDA(cudaMalloc(pp, 6 * kMaxChunks * sizeof(unsigned)));
            g->allocs++;
        }
    IGG_CUDA(cudaMemcpy(g->fused_tgt_pipe, tgt_d.data(), tgt_d.size() * sizeof(unsigned), cudaMemcpyHostToDevice));
    IGG_CUDA(cudaMemcpy(g->fused_tgt_x, tgt_x.data(), tgt_x.size() * sizeof(unsigned), cudaMemcpyHostToDevice));
    g->fused_ntiles = xtiles * ytiles * nch;
    g->fused_nchunks = nch;
    g->fused_geo[4] = xtiles;
    g->fused_geo[5] = ytiles;
}

// ------------------------------------------------------------------ peer arrays
// The caller's T2 lives inside some cudaMalloc allocation (e.g. a torch caching-allocator segment).
// Its base is exported with cudaIpcGetMemHandle, every process all-gathers (handle, offset) and opens
// its neighbours' handles once; the result is cached per local array (Fig. 1 alternates two arrays,
// so two collective exchanges happen, on the first two steps, on every rank).  A cached entry records
// the allocation's identity (base, size, CU_POINTER_ATTRIBUTE_BUFFER_ID -- unique per allocation for
// the life of the process), so an array freed and re-allocated at the same address is never taken
// for the old one: a stale entry fails loudly (IGG_E_STATE) on a single step, and igg_heat_run /
// igg_heat_run_host re-validate every entry collectively (validate_peer_maps) and re-map.
typedef int (*MemGetAddressRangeFn)(unsigned long long *, size_t *, unsigned long long);
typedef int (*PointerGetAttributeFn)(void *, int, unsigned long long);

struct AllocId {
    unsigned long long base = 0, size = 0, buffer_id = 0;
};

static AllocId alloc_id(const void *p) {
    static MemGetAddressRangeFn range_fn = nullptr;
    static PointerGetAttributeFn attr_fn = nullptr;
    if (!range_fn) {
        void *fn = nullptr, *fa = nullptr;
        cudaDriverEntryPointQueryResult q, qa;
        IGG_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        IGG_CUDA(cudaGetDriverEntryPoint("cuPointerGetAttribute", &fa, cudaEnableDefault, &qa));
        if (!fn || q != cudaDriverEntryPointSuccess || !fa || qa != cudaDriverEntryPointSuccess)
            fail(IGG_E_CUDA, "cuMemGetAddressRange / cuPointerGetAttribute unavailable");
        range_fn = (MemGetAddressRangeFn)fn;
        attr_fn = (PointerGetAttributeFn)fa;
    }
    AllocId id;
    size_t size = 0;
    if (range_fn(&id.base, &size, (unsigned long long)(uintptr_t)p) != 0)
        fail(IGG_E_CUDA, "cuMemGetAddressRange failed on a field array (not device memory?)");
    id.size = size;
    constexpr int kBufferIdAttr = 7;   // CU_POINTER_ATTRIBUTE_BUFFER_ID
    if (attr_fn(&id.buffer_id, kBufferIdAttr, (unsigned long long)(uintptr_t)p) != 0)
        fail(IGG_E_CUDA, "cuPointerGetAttribute(BUFFER_ID) failed on a field array");
    return id;
}

static bool same_alloc(const igg_grid::PeerMap &m, const AllocId &id) {
    return m.base == id.base && m.size == id.size && m.buffer_id == id.buffer_id;
}

void release_peer_maps(igg_grid *g) {
    if (g->nproc_procs > 1) {
        IGG_CUDA(cudaDeviceSynchronize());   // no kernel of mine still stores through a mapping
        allgather_bytes_pub(g, "", 1);       // nor any peer's (barrier)
    }
    for (auto &o : g->fused_opened) cudaIpcCloseMemHandle(o.second);
    g->fused_opened.clear();
    g->fused_peer_maps.clear();
}

void validate_peer_maps(igg_grid *g) {
    if (g->nproc_procs == 1) return;   // no mappings: siblings' arrays are used directly
    if (g->fused_peer_maps.empty() && g->fused_opened.empty()) return;   // (entries are created collectively)
    unsigned char ok = 1;
    for (auto &m : g->fused_peer_maps) ok = ok && same_alloc(m, alloc_id(m.ptr));
    std::vector<char> all = allgather_bytes_pub(g, &ok, 1);
    for (char c : all)
        if (!c) {
            release_peer_maps(g);
            return;
        }
}

// per process: the same array of that process, mapped into mine (collective on a cache miss)
static const std::vector<double *> &peer_arrays(igg_grid *g, double *T2) {
    const AllocId id = alloc_id(T2);
    for (auto &m : g->fused_peer_maps)
        if (m.ptr == (const void *)T2) {
            if (!same_alloc(m, id))
                fail(IGG_E_STATE, "fused step: an array was freed and re-allocated at the same address after its "
                                  "first fused step; call igg_release_arrays (collective) before reusing it");
            return m.peers;
        }
    igg_grid::PeerMap e;
    e.ptr = T2;
    e.base = id.base;
    e.size = id.size;
    e.buffer_id = id.buffer_id;
    struct Entry {
        cudaIpcMemHandle_t h;
        unsigned long long off;
    } mine;
    IGG_CUDA(cudaIpcGetMemHandle(&mine.h, (void *)(uintptr_t)id.base));
    mine.off = (unsigned long long)(uintptr_t)T2 - id.base;
    std::vector<char> all = allgather_bytes_pub(g, &mine, sizeof mine);
    e.peers.assign(g->nproc_procs, nullptr);
    for (int p = 0; p < g->nproc_procs; ++p) {
        if (p == g->proc) {
            e.peers[p] = T2;
            continue;
        }
        Entry pe;
        std::memcpy(&pe, all.data() + p * sizeof pe, sizeof pe);
        const std::string key(reinterpret_cast<const char *>(&pe.h), sizeof pe.h);
        void *opened = nullptr;
        for (const auto &o : g->fused_opened)
            if (o.first == key) opened = o.second;
        if (!opened) {
            IGG_CUDA(cudaIpcOpenMemHandle(&opened, pe.h, cudaIpcMemLazyEnablePeerAccess));
            g->fused_opened.push_back({key, opened});
        }
        e.peers[p] = reinterpret_cast<double *>(static_cast<char *>(opened) + pe.off);
    }
    g->fused_peer_maps.push_back(e);
    return g->fused_peer_maps.back().peers;
}

const std::vector<double *> &peer_arrays_pub(igg_grid *g, double *arr) { return peer_arrays(g, arr); }

}  // namespace igg

#if FUSED_TRACE
// diagnostics build only: the per-block stamps (start, sweep end, -, end; ns) of the last fused launch
// record the launch of epoch (current + offset)
IGG_API igg_status igg_debug_trace_epoch(igg_grid *g, long long offset) {
    IGG_TRY
    const unsigned long long e = g->epoch + offset;
    IGG_CUDA(cudaMemcpyToSymbol(igg::g_trace_epoch, &e, sizeof e));
    IGG_CATCH
}
IGG_API igg_status igg_debug_fused_trace(unsigned long long *host, int nblocks) {
    IGG_TRY
    IGG_CUDA(cudaDeviceSynchronize());
    IGG_CUDA(cudaMemcpyFromSymbol(host, igg::g_fused_trace, sizeof(unsigned long long) * 4 * std::min(nblocks, 65536)));
    IGG_CATCH
}
#endif

namespace igg {

// One step of every hosted rank: T2[lr] = step!(T[lr]) plus the faces into the receivers; element type E
// (binary64, or binary32 with kf).  wait_prev: the previous step of the same run was fused (its faces are
// awaited tile by tile); drain: the step completes the run (rim, forwarders, drain: complete on the
// stream afterwards).
template <typename E>
static void fused_step_t(igg_grid *g, E *const *T2, const E *const *T, const E *const *Ci, const HeatCoef &k,
                         const HeatCoefF &kf, cudaStream_t s, bool wait_prev, bool drain) {
    const int L = g->nlocal;
    // [data ctr | rim/forward ctr] x 6 x kMaxChunks, ticket (8), x-piece ctr [parity][2] x kMaxChunks
    const size_t ctr_words = 16 * kMaxChunks + 8;
    if (!g->fused_ctr) {
        IGG_CUDA(cudaMalloc(&g->fused_ctr, L * ctr_words * sizeof(unsigned int)));
        IGG_CUDA(cudaMemset(g->fused_ctr, 0, L * ctr_words * sizeof(unsigned int)));
        g->allocs++;
    }
    const bool comm = !g->skip_comm;
    const bool xex = comm && (g->dims[0] > 1 || g->periods[0]);   // x faces exist: local staging rows
    const size_t stg_words = 2 * (size_t)g->n[1] * g->n[2];       // [side][y][z] per rank
    if (xex && !g->fused_xloc) {
        IGG_CUDA(cudaMalloc(&g->fused_xloc, sizeof(double) * 2 * stg_words * L));   // [parity][side][z][y]
        IGG_CUDA(cudaMalloc(&g->fused_xrem, sizeof(double) * 2 * stg_words * L));   // [parity][side][y][z]
        IGG_CUDA(cudaMalloc(&g->fused_xcnt, sizeof(unsigned) * 2 * kMaxChunks * L));
        IGG_CUDA(cudaMemset(g->fused_xcnt, 0, sizeof(unsigned) * 2 * kMaxChunks * L));
        g->fused_xsteps = 0;
        g->allocs += 3;
    }
    g->epoch++;
    FusedParams F{};
    for (int a = 0; a < 3; ++a) F.s[a] = g->n[a];
    F.epoch = g->epoch;
    F.timeout_cycles = (long long)(g->spin_timeout_ms * g->clock_khz);
    F.err = g->d_err;
    F.k = k;
    F.kf = kf;
    F.nranks = L;
    bool act[3][2] = {{false, false}, {false, false}, {false, false}};
    bool zex = false;
    // flags of hosted rank lr: data (lr*6 + a*2 + rs) * kMaxChunks, rim/forwarded (L*6 + lr*6 + a*2 + rs)
    // * kMaxChunks (a remote process hosts one rank: its offsets with lr = 0, L = 1)
    for (int lr = 0; lr < L; ++lr) {
        FusedRank &R = F.r[lr];
        R.T = reinterpret_cast<const double *>(T[lr]);
        R.Ci = reinterpret_cast<const double *>(Ci[lr]);
        R.T2 = reinterpret_cast<double *>(T2[lr]);
        R.ctr = g->fused_ctr + lr * ctr_words;
        R.ctr_x = R.ctr + 6 * kMaxChunks;
        R.rim_ticket = R.ctr + 12 * kMaxChunks;
        R.xpc = R.ctr + 12 * kMaxChunks + 8;
        R.xloc = xex ? g->fused_xloc + lr * 2 * stg_words : nullptr;
        R.xrem = xex ? g->fused_xrem + lr * 2 * stg_words : nullptr;
        R.xcnt = xex ? g->fused_xcnt + lr * 2 * kMaxChunks : nullptr;
        for (int a = 0; a < 3; ++a)
            for (int rs = 0; rs < 2; ++rs) {
                // rs = receiver side: 0 <- my layer n-2 into my upper neighbour's layer 0,
                //                     1 <- my layer 1 into my lower neighbour's layer s-1
                const int nb = g->nbr[lr][a][rs == 0 ? 1 : 0];
                FusedFace &f = R.face[a][rs];
                f.layer = rs == 0 ? g->n[a] - 2 : 1;
                f.active = comm && nb >= 0;
                if (f.active) {
                    act[a][rs] = true;
                    zex = zex || a == 2;
                    const int li = local_index(g, nb);
                    if (li >= 0) {   // a rank on this GPU: its arrays directly
                        f.dst = reinterpret_cast<double *>(T2[li]);
                        f.flag = g->flags + (li * 6 + a * 2 + rs) * kMaxChunks;
                        f.xflag = g->flags + (L * 6 + li * 6 + a * 2 + rs) * kMaxChunks;
                        if (a == 0) R.xrem_peer[rs] = g->fused_xrem + li * 2 * stg_words;
                    } else {         // another process (one rank each): its arrays mapped over NVLink
                        const int pp = proc_of(g, nb);
                        f.dst = peer_arrays(g, reinterpret_cast<double *>(T2[lr]))[pp];
                        f.flag = g->peer_flags[pp] + (a * 2 + rs) * kMaxChunks;
                        f.xflag = g->peer_flags[pp] + (6 + a * 2 + rs) * kMaxChunks;
                        if (a == 0) R.xrem_peer[rs] = peer_arrays(g, g->fused_xrem)[pp];
                    }
                }
                FusedHalo &h = R.halo[a][rs];   // my halo side rs is filled by my neighbour on side rs
                h.active = comm && g->nbr[lr][a][rs] >= 0;
                h.layer = rs == 0 ? 0 : g->n[a] - 1;
                h.flag = g->flags + (lr * 6 + a * 2 + rs) * kMaxChunks;
                h.xflag = g->flags + (L * 6 + lr * 6 + a * 2 + rs) * kMaxChunks;
            }
    }
    int key = sizeof(E) == 4 ? 64 : 0;   // (the layout depends on the tile width)
    for (int a = 0; a < 3; ++a)
        for (int rs = 0; rs < 2; ++rs) key |= (act[a][rs] ? 1 : 0) << (a * 2 + rs);
    if (g->fused_key != key) {
        if (g->fused_deferred >= 0) fail(IGG_E_STATE, "fused step: topology changed inside a run");
        build_layout(g, act, zex, kTW<E>);
        g->fused_key = key;
        if (g->fused_xcnt) {   // the x senders' cumulative counters restart with the layout
            IGG_CUDA(cudaMemset(g->fused_xcnt, 0, sizeof(unsigned) * 2 * kMaxChunks * L));
            g->fused_xsteps = 0;
        }
    }
    const bool xface = act[0][0] || act[0][1];
    if (xface) ++g->fused_xsteps;   // launches whose x-face tiles count on the cumulative counters
    F.xtarget = (unsigned)((unsigned long long)g->fused_geo[5] * g->fused_xsteps);
    F.xtarget_prev = (unsigned)((unsigned long long)g->fused_geo[5] * (g->fused_xsteps - 1));
    F.nxs = xface ? kFusedXSenders : 0;
    F.nchunks = g->fused_nchunks;
    for (int c = 0; c < F.nchunks; ++c) F.zr[c] = g->fused_zr[c];
    F.xtiles = g->fused_geo[4];
    F.ytiles = g->fused_geo[5];
    F.zchunk[0] = g->fused_zchunk[0];
    F.zchunk[1] = g->fused_zchunk[1];
    F.tgt = g->fused_tgt_pipe;
    F.tgt_x = g->fused_tgt_x;
#ifndef FUSED_DIAG_NATURAL_ORDER
    F.border_first = (act[0][0] || act[0][1] || act[1][0] || act[1][1]) ? 1 : 0;
#endif
    // ONE launch on the caller's stream and, when the step must be complete on return, a drain.  The rim
    // cells and the forwarded edge lines are never read by the stencil, so only the step that completes a
    // run sends them (rim blocks + forwarders in its launch); the steps before it move only the faces the
    // next step's tiles read.  (Every schedule is one launch: kernels on other streams that would spin on
    // this launch's flags are never relied on -- nothing guarantees two launches run at the same time.)
    F.wait_prev = (wait_prev && comm) ? 1 : 0;
    F.nrim = (comm && drain) ? 48 : 0;
    F.nfwd = (comm && drain) ? g->fused_nfwd : 0;
    F.nstencil = g->fused_ntiles;
    // the x chunks visited last would trail the launch by one copy + one system fence (~8 us measured):
    // a step that does not complete its run leaves them to the next launch's senders, which send them
    // first -- the receiver reads them only at the end of its next step.  A draining step
    // publishes such a chunk for two epochs: separate counters by parity; a piece of a chunk has the
    // same sender in both passes, and every sender finishes pass 0 first, so the chunk's flag reaches
    // epoch-1 before epoch (never backwards).
    F.undefer_from = g->fused_deferred >= 0 ? g->fused_deferred : F.nchunks;
    F.defer_from = (xface && !drain && F.nchunks > kFusedDefer) ? F.nchunks - kFusedDefer : F.nchunks;
    g->fused_deferred = F.defer_from < F.nchunks ? F.defer_from : -1;
    F.per_rank = F.nrim + F.nfwd + 2 * F.nxs + F.nstencil;   // (rim, forwarders, x senders, tiles)
    const long long blocks = (long long)F.per_rank * L;
    prof_begin(g, s);
    if (L > 1)
        heat_fused_kernel<true, E><<<(unsigned)blocks, 32 * kFTY, 0, s>>>(F);
    else
        heat_fused_kernel<false, E><<<(unsigned)blocks, 32 * kFTY, 0, s>>>(F);
    IGG_CUDA(cudaGetLastError());
    g->launches++;
    prof_end(g, s, (long long)(g->n[0] - 2) * (g->n[1] - 2) * (g->n[2] - 2) * L);
    if (drain && comm) {
        fused_drain_kernel<E><<<dim3(xex ? 2 * g->sm_count / L + 1 : 1, L), 128, 0, s>>>(F);
        IGG_CUDA(cudaGetLastError());
        g->launches++;
    }
}

void fused_step(igg_grid *g, double *const *T2, const double *const *T, const double *const *Ci, const HeatCoef &k,
                cudaStream_t s, bool wait_prev, bool drain) {
    fused_step_t<double>(g, T2, T, Ci, k, HeatCoefF{}, s, wait_prev, drain);
}
void fused_step_f32(igg_grid *g, float *const *T2, const float *const *T, const float *const *Ci,
                    const HeatCoefF &kf, cudaStream_t s, bool wait_prev, bool drain) {
    fused_step_t<float>(g, T2, T, Ci, HeatCoef{}, kf, s, wait_prev, drain);
}

}  // namespace igg
