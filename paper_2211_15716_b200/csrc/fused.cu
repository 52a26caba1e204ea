// fused.cu -- the fused hide_communication step: stencil + halo exchange as
// one-sided NVLink puts straight into the neighbours' arrays, pipelined by
// z-chunks (IGG_PATH_P2P, one rank per process, every neighbour on another GPU).
//
// The paper hides update_halo! behind the inner-point computation (PAPER.md:75,
// :94 "pipelining is applied on all stages of the data transfers").
// On B200 one stencil kernel keeps the 1-GPU tile order (z-chunk, then y-tile,
// then x-tile: whole 4-KB rows stream together) and, when a tile holding send
// layers finishes its chunk, stores those cells directly into the receiving
// rank's T2 halo layers over NVLink (pack, transfer and unpack fused into one
// store; the receiver's SMs do no copy work).  Faces are published chunk by
// chunk: each CTA that holds part of face f in chunk c counts itself on
// counter (f, c) after a system fence; the contribution completing (f, c)
// release-stores the epoch into the receiver's flag (f, c).  Face cells the
// stencil does not compute come from a rim kernel (values that never change or
// are overwritten later on the receiver) or are forwarded, after the flags of
// an earlier axis arrived, by a tiny comm kernel (the fresh edge/corner values
// of the dimension-sequential update_halo).  The receiver
// waits for every flag before the step completes.  Hazard argument (DESIGN.md
// §6): a peer writes my T2(t) halo only after it received my step t-1 faces,
// i.e. after my step t-1 tiles that read those halo cells finished.  The final
// state is bit-identical to {step!; update_halo!(T2)} (tests/test_gpu_multi.py).
#include <algorithm>
#include <array>
#include <cstring>
#include <type_traits>

#include "igg_internal.h"

namespace igg {

namespace {

__device__ __forceinline__ void st_rel_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
// L2 eviction-priority hint: evict_last for the rows of the x-face tiles, whose send-layer cells the
// face epilogue re-reads after the sweep (fused_mode bit 4096, experiment)
__device__ __forceinline__ unsigned long long policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st2_hint(double *ptr, double a, double b, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(a), "d"(b), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ double2 ldg2f(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }

// the cell of PAPER.md:46-49, same explicitly rounded operations as kernels.cu
__device__ __forceinline__ double cell(double c, double xm, double xp, double ym, double yp, double zm, double zp,
                                       double ci, const HeatCoef &k) {
    const double d2x = __dsub_rn(__dsub_rn(xp, c), __dsub_rn(c, xm));
    const double d2y = __dsub_rn(__dsub_rn(yp, c), __dsub_rn(c, ym));
    const double d2z = __dsub_rn(__dsub_rn(zp, c), __dsub_rn(c, zm));
    const double lap =
        __dadd_rn(__dadd_rn(__dmul_rn(d2x, k.rdx2), __dmul_rn(d2y, k.rdy2)), __dmul_rn(d2z, k.rdz2));
    return __dadd_rn(c, __dmul_rn(k.dt, __dmul_rn(__dmul_rn(k.lam, ci), lap)));
}

__device__ __forceinline__ void contribute(const FusedParams &F, int a, int rs, int c) {
    const int i = (a * 2 + rs) * kMaxChunks + c;
    const unsigned old = atomicAdd(F.ctr + i, 1u);
    if (old == F.tgt[i] - 1) {
        __threadfence_system();
        st_rel_sys(F.face[a][rs].flag + c, F.epoch);
        atomicExch(F.ctr + i, 0u);
    }
}

__device__ __forceinline__ void st_rel_gpu(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq_gpu(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// thread 0 spins (bounded) until the local *fl >= v
__device__ __forceinline__ void spin_geq_gpu(const FusedParams &F, const unsigned long long *fl, unsigned long long v) {
    const long long t0 = clock64();
    while (ld_acq_gpu(fl) < v) {
        if (clock64() - t0 > F.timeout_cycles) {
            atomicExch(F.err, 1);
            break;
        }
        __nanosleep(100);
    }
}
// count one of `target` contributions on a local counter; the last one publishes the epoch (gpu scope)
__device__ __forceinline__ void count_local(const FusedParams &F, int i, unsigned target) {
    if (atomicAdd(F.xcnt + i, 1u) == target - 1) {
        atomicExch(F.xcnt + i, 0u);
        st_rel_gpu(F.xev + i, F.epoch);
    }
}

// rim / forwarded cells of (face, chunk) on the pipelined schedule: their own counters and flags
__device__ __forceinline__ void contribute_x(const FusedParams &F, int a, int rs, int c) {
    const int i = (a * 2 + rs) * kMaxChunks + c;
    const unsigned old = atomicAdd(F.ctr_x + i, 1u);
    if (old == F.tgt_x[i] - 1) {
        __threadfence_system();
        st_rel_sys(F.face[a][rs].xflag + c, F.epoch);
        atomicExch(F.ctr_x + i, 0u);
    }
}

// thread 0 spins (bounded) until *fl >= v; the caller synchronises the CTA
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

// the earlier axis whose unpack writes this cell last in the dimension-sequential
// exchange (-1: none) -- that unpack forwards the cell to face a
__device__ __forceinline__ int forward_phase(const FusedParams &F, int a, const int *c) {
    int fwd = -1;
    for (int b = 0; b < a; ++b) {
        if (c[b] == 0 && F.halo[b][0].active) fwd = b;
        if (c[b] == F.s[b] - 1 && F.halo[b][1].active) fwd = b;
    }
    return fwd;
}

// a later axis whose exchange writes this cell's receiver copy last: the cell is sent by that
// axis' phase (face or forwarding), never by this one -- so every receiver cell has ONE writer
__device__ __forceinline__ bool later_halo(const FusedParams &F, int a, const int *c) {
    for (int b = a + 1; b < 3; ++b)
        if ((c[b] == 0 && F.halo[b][0].active) || (c[b] == F.s[b] - 1 && F.halo[b][1].active)) return true;
    return false;
}

// staging buffer offset of (epoch parity, halo side, y, z)
__device__ __forceinline__ long long xstg_at(const FusedParams &F, unsigned long long epoch, int side, int y, int z) {
    return ((long long)((int)(epoch & 1) * 2 + side) * F.s[1] + y) * F.s[2] + z;
}

// chunk visited at order position oc: 0, cz, then the others ascending
__device__ __forceinline__ int chunk_id(const FusedParams &F, int oc) {
    if (F.cz <= 1 || oc == 0) return oc;
    if (oc == 1) return F.cz;
    return oc - 1 < F.cz ? oc - 1 : oc;
}
// z range [z0, z1) of the chunk at order position oc
__device__ __forceinline__ int2 chunk_range(const FusedParams &F, int oc) {
    const int j = chunk_id(F, oc);
    const int zmax = F.s[2] - 1;
    if (j < F.nbig) return make_int2(1 + F.kc1 * j, 1 + F.kc1 * (j + 1));
    const int z0 = 1 + F.kc1 * F.nbig + F.kc2 * (j - F.nbig);
    return make_int2(z0, min(z0 + F.kc2, zmax));
}
// z range a chunk covers on the x- and y-faces (the rim planes 0 and s-1 go with the end chunks)
__device__ __forceinline__ int2 ext_range(const FusedParams &F, int c) {
    int2 r = chunk_range(F, c);
    if (r.x == 1) r.x = 0;
    if (r.y == F.s[2] - 1) r.y = F.s[2];
    return r;
}

constexpr int kFTY = 4;    // rows per CTA (one warp each)
__device__ __forceinline__ bool pair_in_x(int p, int sx) { return p < sx; }
constexpr unsigned g_poll_ns = 1000;   // flag polling period of the waiting CTAs
constexpr int kFD = 3;     // planes in flight per thread
constexpr int kFKC = 64;   // longest z-chunk

}  // namespace

// The z sweep of one tile (cp.async ring of kFD planes of T and Ci, x neighbours by shuffle, z by a
// register queue).  CAP: the lane xl holding an x send-layer cell of its row (cell xodd of its pair)
// stores it into the receiver's staging row every plane (xdst[z]), so the face epilogue need not
// re-read the column from DRAM.
template <bool CAP>
__device__ __forceinline__ void fused_sweep(const FusedParams &F, double2 (*sT)[32 * kFTY], double2 (*sC)[32 * kFTY],
                                            double (*sH)[kFTY], double *xdst, int tid, int lane, int zs, int ze,
                                            long long i, long long sxy, int sx, bool pair_in, bool w0, bool w1,
                                            int xl, bool xodd, const double *xr, int xrl, bool xrhi,
                                            unsigned long long pol) {
    const double *__restrict__ T = F.T;
    const double *__restrict__ Ci = F.Ci;
    double *__restrict__ T2 = F.T2;
    const int warp = tid >> 5;
#pragma unroll
    for (int q = 0; q < kFD; ++q) {
        if (pair_in && zs + q < ze) {
            cp_async16f(&sT[q][tid], T + i + (q + 1) * sxy);
            cp_async16f(&sC[q][tid], Ci + i + q * sxy);
            // CAP, halo-reading lane: its x halo cell of plane zs+q+1 from the staging row (not in T)
            if (CAP && lane == xrl) cp_async8(&sH[q][warp], xr + zs + q + 1);
        }
        cp_commit();
    }
    const double2 zero2 = make_double2(0.0, 0.0);
    double2 zm = pair_in ? ldg2f(T + i - sxy) : zero2;
    double2 c = pair_in ? ldg2f(T + i) : zero2;
    if (CAP && lane == xrl) {
        const double h = __ldcg(xr + zs);
        if (xrhi) c.y = h; else c.x = h;
    }
    int slot = 0;
    {
#pragma unroll 2
        for (int z = zs; z < ze; ++z, i += sxy) {
            cp_wait<kFD - 1>();
            double2 ym = zero2, yp = zero2;
            if (pair_in) {
                ym = ldg2f(T + i - sx);
                yp = ldg2f(T + i + sx);
            }
            const double2 zp = sT[slot][tid];
            const double2 ci = sC[slot][tid];
            double xm = __shfl_up_sync(0xffffffffu, c.y, 1);
            double xp = __shfl_down_sync(0xffffffffu, c.x, 1);
            if (lane == 0 && w0) xm = __ldg(T + i - 1);
            if (lane == 31 && w1) xp = __ldg(T + i + 2);
            const double r0 = cell(c.x, xm, c.y, ym.x, yp.x, zm.x, zp.x, ci.x, F.k);
            const double r1 = cell(c.y, c.x, xp, ym.y, yp.y, zm.y, zp.y, ci.y, F.k);
            if (w0 && w1) {   // plain stores (streaming stores measured no faster; face cells stay in L2)
                if (pol)      // (CTA-uniform)
                    st2_hint(T2 + i, r0, r1, pol);
                else
                    *reinterpret_cast<double2 *>(T2 + i) = make_double2(r0, r1);
            } else {
                if (w0) T2[i] = r0;
                if (w1) T2[i + 1] = r1;
            }
            if (CAP && lane == xl) xdst[z] = xodd ? r1 : r0;   // the receiver's staging row
            zm = c;
            c = zp;
            if (CAP && lane == xrl) {
                const double h = sH[slot][warp];
                if (xrhi) c.y = h; else c.x = h;
            }
            if (pair_in && z + kFD < ze) {
                cp_async16f(&sT[slot][tid], T + i + (kFD + 1) * sxy);
                cp_async16f(&sC[slot][tid], Ci + i + kFD * sxy);
                if (CAP && lane == xrl) cp_async8(&sH[slot][warp], xr + z + kFD + 1);
            }
            cp_commit();
            slot = slot + 1 == kFD ? 0 : slot + 1;
        }
    }
    cp_wait<0>();
}

// tile of this CTA from the block index (x-tiles fastest, then y-tiles, then chunks in visit
// order); the last chunks' tiles are re-ordered, face tiles first, from the parameter table
__device__ __forceinline__ int4 fused_tile(const FusedParams &F, int b) {
    int4 td;
    if (b < F.bmain) {
        td.x = b % F.xtiles;
        const int r = b / F.xtiles;
        td.y = r % F.ytiles;
        td.z = r / F.ytiles;
    } else {
        const unsigned e = F.tail[b - F.bmain];
        td.x = e & 15u;
        td.y = (e >> 4) & 1023u;
        td.z = F.bmain / (F.xtiles * F.ytiles) + (int)(e >> 14);
    }
    td.w = 0;
    return td;
}

// Pipelined schedule, before the sweep: a tile that reads halo cells waits until the previous
// epoch's faces covering them have arrived (x: first/last x-tile of the chunk, y: first/last y-tile,
// z: the chunks holding planes 1 and s_z-2).  The same wait orders my face stores of this epoch
// after the neighbour's reads of the halo they overwrite: the neighbour's tiles that read that halo
// are the ones that published the awaited face (hazard argument).
template <bool XS>
__device__ __forceinline__ void fused_wait_halos(const FusedParams &F, int4 td, int zs, int ze) {
    const bool xlo = F.halo[0][0].active && td.x == 0, xhi = F.halo[0][1].active && td.x == F.xtiles - 1;
    if (threadIdx.x == 0) {
        const unsigned long long prev = F.epoch - 1;
        if (F.xblk) {   // my receiver blocks copied the column into this T (last step's T2)
            if (xlo) spin_geq_gpu(F, F.xev + 2 * kMaxChunks + td.z, prev);
            if (xhi) spin_geq_gpu(F, F.xev + 3 * kMaxChunks + td.z, prev);
        } else {
            if (xlo) spin_geq(F, F.halo[0][0].flag + td.z, prev);
            if (xhi) spin_geq(F, F.halo[0][1].flag + td.z, prev);
        }
        if (F.halo[1][0].active && td.y == 0) spin_geq(F, F.halo[1][0].flag + td.z, prev);
        if (F.halo[1][1].active && td.y == F.ytiles - 1) spin_geq(F, F.halo[1][1].flag + td.z, prev);
        if (F.halo[2][0].active && zs == 1) spin_geq(F, F.halo[2][0].flag, prev);
        if (F.halo[2][1].active && ze == F.s[2] - 1) spin_geq(F, F.halo[2][1].flag, prev);
    }
    __syncthreads();
    if (!XS && F.xstage && !F.xblk && (xlo || xhi)) {   // (XS: read from the staging row in the sweep)
        // my x halo column of this tile (its rows, its chunk's planes), staged by the neighbour in the
        // previous epoch -- final since the awaited flag -- into my T, just before the sweep reads it
        // (writing whole 32-B sectors instead, halo cell plus its row neighbours, measured slower)
        const int sx = F.s[0], sy = F.s[1];
        const long long sxy = (long long)sx * sy;
        const int ty0 = 1 + td.y * kFTY, nrow = min(ty0 + kFTY, sy - 1) - ty0, nz = ze - zs;
        double *Tw = const_cast<double *>(F.T);
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            if (!(side == 0 ? xlo : xhi)) continue;
            const int hx = side == 0 ? 0 : sx - 1;
            constexpr int U = kFKC / 32;   // cells per thread (4 rows x 64 planes / 128 threads)
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = threadIdx.x + u * 32 * kFTY;
                v[u] = t < nrow * nz ? __ldcg(F.xstg + xstg_at(F, F.epoch - 1, side, ty0 + t / nz, zs + t % nz)) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = threadIdx.x + u * 32 * kFTY;
                if (t < nrow * nz) Tw[(long long)(zs + t % nz) * sxy + (long long)(ty0 + t / nz) * sx + hx] = v[u];
            }
        }
        __syncthreads();
    }
}

__device__ __noinline__ void fused_extra(const FusedParams &F, int b);

// One launch over all tiles, the 1-GPU loop unchanged.  A CTA whose tile holds
// send-layer cells (x layer of its rows, a y layer row, or a z layer plane in
// its chunk) re-reads them from T2 after its sweep (its own just-written
// values) and stores them into the receivers' halos, then counts itself on the
// (face, chunk) counters.  Keeping the face work out of the z loop keeps the
// loop's instruction stream identical to the 1-GPU kernel.  (Measured: the face
// epilogue must stay inline with face_tile computed before the sweep; outlining it
// or recomputing the tile after the sweep adds spills around the loop and costs
// 2-13 % of the step.)
template <bool XS>   // XS: the x send layer goes to the neighbour from the sweep (else re-read from T2)
__global__ void __launch_bounds__(32 * kFTY, 10) heat_fused_kernel(const __grid_constant__ FusedParams F) {
    __shared__ double2 sT[kFD][32 * kFTY];
    __shared__ double2 sC[kFD][32 * kFTY];
    __shared__ double sH[XS ? kFD : 1][kFTY];   // XS: the halo-reading lanes' staged x halo cells
    int b = blockIdx.x;
    if (F.pipe) {   // pipelined schedule: rim, forwarders, x senders/receivers, then the tiles (CTA-uniform)
        if (b < F.nrim + F.nfwd + 4 * F.nxb) {
            fused_extra(F, b);
            return;
        }
        b -= F.nrim + F.nfwd + 4 * F.nxb;
    }
    const int4 td = fused_tile(F, b);
    const int2 zr = chunk_range(F, td.z);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sx = F.s[0], sy = F.s[1];
    const int y = 1 + td.y * kFTY + warp;
    const int p = td.x * 64 + 2 * lane;
    const bool pair_in = y < sy - 1 && p < sx;
    const bool w0 = pair_in && p >= 1 && p < sx - 1;
    const bool w1 = pair_in && p + 1 >= 1 && p + 1 < sx - 1;
    const int zs = zr.x, ze = zr.y;
    const long long sxy = (long long)sx * sy;
    bool face_tile = false;   // this tile holds send-layer cells
#pragma unroll
    for (int rs = 0; rs < 2; ++rs) {
        const int xl = F.face[0][rs].layer, yl = F.face[1][rs].layer;
        face_tile |= F.face[0][rs].active && xl >= max(td.x * 64, 1) && xl < min(td.x * 64 + 64, sx - 1);
        face_tile |= F.face[1][rs].active && yl >= 1 + td.y * kFTY && yl < min(1 + (td.y + 1) * kFTY, sy - 1);
        face_tile |= F.face[2][rs].active && F.zchunk[rs] == td.z;
    }
    if (F.wait_prev) fused_wait_halos<XS>(F, td, zs, ze);   // CTA-uniform
    long long i = (long long)zs * sxy + (long long)y * sx + p;
    // XS: the x send-layer cell of my row (lane xl, cell xodd of its pair) goes to the neighbour
    // plane by plane from the sweep (xdst + i = its halo cell of my row and plane)
    int xl = -1;
    bool xodd = false;
    double *xdst = nullptr;
#pragma unroll
    for (int rs = 0; rs < 2; ++rs) {
        const int L = F.face[0][rs].layer - td.x * 64;
        if (XS && !F.nostore && F.xstage && F.face[0][rs].active && y < sy - 1 && L >= 0 && L < 64 &&
            L + td.x * 64 >= 1 && L + td.x * 64 < sx - 1) {
            xl = L >> 1;
            xodd = L & 1;
            if (lane == xl) xdst = F.xstg_peer[rs] + xstg_at(F, F.epoch, rs, y, 0);
        }
    }
    // XS with staged x faces and a previous epoch: the halo-reading lane takes its x halo cell from the
    // staging row inside the sweep (no copy into T in the prologue)
    const double *xr = nullptr;
    int xrl = -1;
    bool xrhi = false;
    if (XS && F.xstage && F.wait_prev && y < sy - 1) {
        if (F.halo[0][0].active && td.x == 0) {
            xrl = 0;
            xr = F.xstg + xstg_at(F, F.epoch - 1, 0, y, 0);
        } else if (F.halo[0][1].active && td.x == F.xtiles - 1) {
            const int L = sx - 1 - td.x * 64;
            xrl = L >> 1;
            xrhi = L & 1;
            xr = F.xstg + xstg_at(F, F.epoch - 1, 1, y, 0);
        }
    }
    unsigned long long pol = 0;
    if (F.xhint) {   // x-face tile: keep its rows in L2 until the face epilogue re-reads the layer
        bool xface = false;
        for (int rs = 0; rs < 2; ++rs) {
            const int xlr = F.face[0][rs].layer;
            xface |= F.face[0][rs].active && xlr >= max(td.x * 64, 1) && xlr < min(td.x * 64 + 64, sx - 1);
        }
        if (xface) pol = policy_evict_last();
    }
    fused_sweep<XS>(F, sT, sC, sH, xdst, tid, lane, zs, ze, i, sxy, sx, pair_in, w0, w1, xl, xodd, xr, xrl, xrhi,
                    pol);
    if (!face_tile) return;   // CTA-uniform
    double *__restrict__ T2 = F.T2;
    __syncthreads();          // the CTA's T2 stores are visible to the CTA
    const int tx0 = td.x * 64, ty0 = 1 + td.y * kFTY;
    const int xlo = max(tx0, 1), xhi = min(tx0 + 64, sx - 1);   // inner x of this tile
    const int yhi = min(ty0 + kFTY, sy - 1);
    bool did[6] = {false, false, false, false, false, false};
    // Each warp copies its own row's part of every face the tile holds, with all loads of a
    // batch issued before its stores (the cells were just written by this CTA: L2 hits).
    const int yrow = ty0 + warp;               // my warp's row
    const bool rowv = yrow < yhi;
#pragma unroll
    for (int rs = 0; rs < 2 && !F.nostore; ++rs) {
        // rs = 0: the upper neighbour's lower halo layer 0; rs = 1: the lower neighbour's layer s-1
        // x face: my row's layer cell over the chunk's planes -> the peer's x halo (lanes along z)
        const FusedFace &fx = F.face[0][rs];
        if (fx.active && fx.layer >= xlo && fx.layer < xhi) {
            const int hx = rs == 0 ? 0 : sx - 1;
            if (rowv && !F.xblk) {   // (x blocks: the sender blocks move the column)
                double v[kFKC / 32];
#pragma unroll
                for (int u = 0; u < kFKC / 32; ++u) {
                    const int zz = zs + lane + 32 * u;
                    v[u] = ((!XS || !F.xstage) && zz < ze) ? T2[(long long)zz * sxy + (long long)yrow * sx + fx.layer]
                                                           : 0.0;
                }
                // staged: the receiver's staging row (lanes along z: whole sectors); else its T2 column
                double *const dst = F.xstage ? F.xstg_peer[rs] + xstg_at(F, F.epoch, rs, yrow, 0)
                                             : fx.dst + (long long)yrow * sx + hx;
                const long long zstride = F.xstage ? 1 : sxy;
#pragma unroll
                for (int u = 0; u < kFKC / 32; ++u) {
                    const int zz = zs + lane + 32 * u;
                    if ((XS && F.xstage) || zz >= ze) continue;   // XS: staged from the sweep
                    dst[(long long)zz * zstride] = v[u];
                }
            }
            did[rs] = true;
        }
        // y face: the layer row over the chunk's planes -> the peer's y halo row; the warps
        // take planes round-robin, lanes the row segment as 16-B pairs
        const FusedFace &fy = F.face[1][rs];
        if (fy.active && fy.layer >= ty0 && fy.layer < yhi) {
            const int hy = rs == 0 ? 0 : sy - 1;
            constexpr int U = 4;
            for (int zb = zs + warp; zb < ze; zb += kFTY * U) {
                double2 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int zz = zb + kFTY * u;
                    v[u] = (zz < ze && pair_in_x(p, sx))
                               ? *reinterpret_cast<const double2 *>(T2 + (long long)zz * sxy + (long long)fy.layer * sx + p)
                               : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int zz = zb + kFTY * u;
                    if (zz >= ze) continue;
                    double *d = fy.dst + (long long)zz * sxy + (long long)hy * sx + p;
                    if (p >= xlo && p + 1 < xhi) {
                        *reinterpret_cast<double2 *>(d) = v[u];
                    } else {
                        if (p >= xlo && p < xhi) d[0] = v[u].x;
                        if (p + 1 >= xlo && p + 1 < xhi) d[1] = v[u].y;
                    }
                }
            }
            did[2 + rs] = true;
        }
        // z face: my row of the layer plane -> the peer's z halo plane
        const FusedFace &fz = F.face[2][rs];
        if (fz.active && F.zchunk[rs] == td.z) {
            const int hz = rs == 0 ? 0 : F.s[2] - 1;
            if (rowv && pair_in_x(p, sx)) {
                const double2 v =
                    *reinterpret_cast<const double2 *>(T2 + (long long)fz.layer * sxy + (long long)yrow * sx + p);
                double *d = fz.dst + (long long)hz * sxy + (long long)yrow * sx + p;
                if (p >= xlo && p + 1 < xhi) {
                    *reinterpret_cast<double2 *>(d) = v;
                } else {
                    if (p >= xlo && p < xhi) d[0] = v.x;
                    if (p + 1 >= xlo && p + 1 < xhi) d[1] = v.y;
                }
            }
            did[4 + rs] = true;
        }
    }
    if (F.nostore) {   // timing experiment: count without storing (INVALID halos)
        for (int rs = 0; rs < 2; ++rs) {
            did[rs] = F.face[0][rs].active && F.face[0][rs].layer >= xlo && F.face[0][rs].layer < xhi;
            did[2 + rs] = F.face[1][rs].active && F.face[1][rs].layer >= ty0 && F.face[1][rs].layer < yhi;
            did[4 + rs] = F.face[2][rs].active && F.zchunk[rs] == td.z;
        }
    }
    // one system-scope release for the CTA: the barrier orders every warp's face stores before
    // thread 0's fence, which is cumulative (PTX memory model), then the counters
    __syncthreads();
    if (tid == 0) {
        __threadfence_system();
        for (int f = 0; f < 6; ++f) {
            if (!did[f]) continue;
            if (f < 2 && F.xblk)   // x face with sender blocks: my chunk's layer cells are computed
                count_local(F, f * kMaxChunks + td.z, F.ytiles);
            else
                contribute(F, f >> 1, f & 1, f < 4 ? td.z : 0);
        }
    }
}

// Face cells the stencil does not compute (on other axes' halo/boundary layers):
// the ones an earlier axis' unpack writes this step are forwarded by it; all
// others keep a value that never changes (global boundary) or that a later axis
// overwrites on the receiver, so the current T2 value is sent.
// One contribution to every (face, chunk) at the end (ticket).
__global__ void fused_rim_kernel(const __grid_constant__ FusedParams F, unsigned int *ticket, unsigned total) {
    const int f = blockIdx.y, a = f >> 1, rs = f & 1;
    const FusedFace &fc = F.face[a][rs];
    if (fc.active) {
        const int b1 = a == 0 ? 1 : 0, b2 = a == 2 ? 1 : 2;
        const int S1 = F.s[b1], S2 = F.s[b2];
        const long long nrim = 2LL * S2 + 2LL * (S1 - 2);
        for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nrim;
             t += (long long)gridDim.x * blockDim.x) {
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
            if (forward_phase(F, a, c) >= 0 || later_halo(F, a, c)) continue;
            const long long gi = ((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0];
            const double val = F.T2[gi];
            c[a] = rs == 0 ? 0 : F.s[a] - 1;   // the receiver's halo layer
            fc.dst[((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]] = val;
        }
        __threadfence_system();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(ticket, 1u);
        if (t == total - 1) {
            __threadfence_system();
            for (int g = 0; g < 6; ++g) {
                const int ga = g >> 1, grs = g & 1;
                if (!F.face[ga][grs].active) continue;
                if (ga == 2)
                    contribute(F, 2, grs, 0);
                else
                    for (int ch = 0; ch < F.nchunks; ++ch) contribute(F, ga, grs, ch);
            }
            atomicExch(ticket, 0u);
        }
    }
}

__device__ __forceinline__ void wait_flag(const FusedParams &F, const unsigned long long *fl) {
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        while (ld_acq_sys(fl) < F.epoch) {
            if (clock64() - t0 > F.timeout_cycles) {
                atomicExch(F.err, 1);
                break;
            }
            __nanosleep(g_poll_ns);
        }
    }
    __syncthreads();
}

// The receiver side: a few persistent CTAs (IGG_OPT_FUSED_COMM_CTAS) walk the chunks in kernel order
// and wait for every face flag (the halos themselves were stored by the peers'
// stencil CTAs).  After axis b's flags of a chunk arrived they forward the fresh
// halo cells later faces need (the edge lines where my halo layer of b meets a
// later send layer) into those receivers' halos, and count on those faces.
// The x and the y/z pipelines run as two concurrent launches.

__device__ __forceinline__ void wait_flags(const FusedParams &F, int b, int idx) {
    if (threadIdx.x < 2 && F.halo[b][threadIdx.x].active) {
        const unsigned long long *fl = F.halo[b][threadIdx.x].flag + idx;
        const long long t0 = clock64();
        while (ld_acq_sys(fl) < F.epoch) {
            if (clock64() - t0 > F.timeout_cycles) {
                atomicExch(F.err, 1);
                break;
            }
            __nanosleep(g_poll_ns);
        }
    }
    __syncthreads();
}

// forward my fresh halo line (axis b, side) x (face a, rs) over the third axis range [lo, hi)
__device__ __forceinline__ bool forward_line(const FusedParams &F, int b, int side, int a, int rs, int lo, int hi,
                                             int part, int nparts) {
    const FusedFace &fc = F.face[a][rs];
    if (!fc.active || !F.halo[b][side].active) return false;
    const int third = 3 - a - b;
    bool any = false;
    for (int t = lo + part * blockDim.x + threadIdx.x; t < hi; t += nparts * blockDim.x) {
        int c[3];
        c[b] = side == 0 ? 0 : F.s[b] - 1;
        c[a] = fc.layer;
        c[third] = t;
        if (forward_phase(F, a, c) != b || later_halo(F, a, c)) continue;
        double v;
        if (b == 0 && F.xstage && c[1] >= 1 && c[1] < F.s[1] - 1 && c[2] >= 1 && c[2] < F.s[2] - 1) {
            v = __ldcg(F.xstg + xstg_at(F, F.epoch, side, c[1], c[2]));   // staged, not yet in T2
        } else {
            v = __ldcg(F.T2 + ((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]);
        }
        c[a] = rs == 0 ? 0 : F.s[a] - 1;
        fc.dst[((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]] = v;
        any = true;
    }
    return any;
}

__global__ void __launch_bounds__(128) fused_comm_kernel(const __grid_constant__ FusedParams F, int zafter,
                                                         int axes) {
    for (int ch = 0; ch < F.nchunks; ++ch) {
        const int2 zr = ext_range(F, ch);
        for (int b = 0; b < 2; ++b) {
            if (!(axes & (1 << b)) || !(F.halo[b][0].active || F.halo[b][1].active)) continue;
            wait_flags(F, b, ch);
            bool fwd = false;
            for (int side = 0; side < 2; ++side)
                for (int rs = 0; rs < 2; ++rs) {
                    if (b == 0) fwd |= forward_line(F, 0, side, 1, rs, zr.x, zr.y, blockIdx.x, gridDim.x);   // x -> y faces
                    if (F.face[2][rs].layer >= zr.x && F.face[2][rs].layer < zr.y)   // -> z faces
                        fwd |= forward_line(F, b, side, 2, rs, 0, F.s[b == 0 ? 1 : 0], blockIdx.x, gridDim.x);
                }
            if (__syncthreads_or(fwd)) __threadfence_system();
            __syncthreads();
            if (threadIdx.x == 0)
                for (int a = b + 1; a < 3; ++a)
                    for (int rs = 0; rs < 2; ++rs) {
                        if (!F.face[a][rs].active) continue;
                        if (a == 1)
                            contribute(F, 1, rs, ch);
                        else if (F.face[2][rs].layer >= zr.x && F.face[2][rs].layer < zr.y)
                            contribute(F, 2, rs, 0);
                    }
        }
        if ((axes & 4) && ch == zafter && (F.halo[2][0].active || F.halo[2][1].active)) wait_flags(F, 2, 0);
    }
}

// The rim and forwarding roles of the pipelined schedule, as extra blocks of the stencil launch.
// Rim (blocks [0, nrim), six faces x nrim/6 blocks): the rim cells of every face (fused_rim_kernel's
// work); the last rim block counts once on every (face, chunk).  Forwarders (the next nfwd blocks):
// per chunk, wait for the x (then y) halo of the chunk -- its data and its rim/forwarded cells --
// forward the edge lines (fused_comm_kernel's work) and count on the later faces' xflags.
__device__ __noinline__ void fused_extra(const FusedParams &F, int b) {
    if (b < F.nrim) {
        const int per = F.nrim / 6;
        const int f = b / per, part = b % per, a = f >> 1, rs = f & 1;
        const FusedFace &fc = F.face[a][rs];
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
                if (forward_phase(F, a, c) >= 0 || later_halo(F, a, c)) continue;
                const double val = F.T2[((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]];
                c[a] = rs == 0 ? 0 : F.s[a] - 1;
                fc.dst[((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]] = val;
            }
            __threadfence_system();
        }
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(F.rim_ticket, 1u) == (unsigned)F.nrim - 1) {
            __threadfence_system();
            for (int g = 0; g < 6; ++g) {
                const int ga = g >> 1, grs = g & 1;
                if (!F.face[ga][grs].active) continue;
                if (ga == 2)
                    contribute_x(F, 2, grs, 0);
                else
                    for (int ch = 0; ch < F.nchunks; ++ch) contribute_x(F, ga, grs, ch);
            }
            atomicExch(F.rim_ticket, 0u);
        }
        return;
    }
    if (b >= F.nrim + F.nfwd) {   // x blocks: [senders face 0 | face 1 | receivers halo 0 | halo 1] x nxb
        const int e = b - F.nrim - F.nfwd, role = e / F.nxb, part = e % F.nxb;
        const int sx = F.s[0], sy = F.s[1];
        const long long sxy = (long long)sx * sy;
        if (role < 2) {   // sender of face rs: my layer column -> the receiver's staging, data flag
            const int rs = role;
            const FusedFace &fx = F.face[0][rs];
            if (!fx.active) return;
            double *dst = F.xstg_peer[rs];
            for (int ch = 0; ch < F.nchunks; ++ch) {
                if (threadIdx.x == 0) spin_geq_gpu(F, F.xev + rs * kMaxChunks + ch, F.epoch);
                __syncthreads();
                const int2 zr = chunk_range(F, ch);
                const int nz = zr.y - zr.x;
                const long long ncell = (long long)(sy - 2) * nz;
                constexpr int U = 4;
                for (long long t0 = (long long)part * blockDim.x * U + threadIdx.x; t0 < ncell;
                     t0 += (long long)F.nxb * blockDim.x * U) {
                    double v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {   // z fastest: whole sectors of the staging rows
                        const long long t = t0 + (long long)u * blockDim.x;
                        const int y = 1 + (int)(t / nz), z = zr.x + (int)(t % nz);
                        v[u] = t < ncell ? __ldcg(F.T2 + (long long)z * sxy + (long long)y * sx + fx.layer) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const long long t = t0 + (long long)u * blockDim.x;
                        if (t >= ncell) continue;
                        const int y = 1 + (int)(t / nz), z = zr.x + (int)(t % nz);
                        dst[xstg_at(F, F.epoch, rs, y, z)] = v[u];
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence_system();
                    contribute(F, 0, rs, ch);
                }
            }
        } else {   // receiver of halo side: the staged column -> my T2 column, xready (local)
            const int side = role - 2;
            const FusedHalo &h = F.halo[0][side];
            if (!h.active) return;
            const int hx = side == 0 ? 0 : sx - 1;
            for (int ch = 0; ch < F.nchunks; ++ch) {
                if (threadIdx.x == 0) spin_geq(F, h.flag + ch, F.epoch);
                __syncthreads();
                const int2 zr = chunk_range(F, ch);
                const int nz = zr.y - zr.x;
                const long long ncell = (long long)(sy - 2) * nz;
                for (long long t = (long long)part * blockDim.x + threadIdx.x; t < ncell;
                     t += (long long)F.nxb * blockDim.x) {
                    const int y = 1 + (int)(t / nz), z = zr.x + (int)(t % nz);
                    F.T2[(long long)z * sxy + (long long)y * sx + hx] = __ldcg(F.xstg + xstg_at(F, F.epoch, side, y, z));
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence();
                    count_local(F, (2 + side) * kMaxChunks + ch, F.nxb);
                }
            }
        }
        return;
    }
    const int q = b - F.nrim;   // forwarder q of nfwd (launched right after the rim: they wait chunk by
                                // chunk, so each edge line leaves as soon as its halo has arrived)
    for (int ch = 0; ch < F.nchunks; ++ch) {
        const int2 zr = ext_range(F, ch);
        for (int hb = 0; hb < 2; ++hb) {
            if (!(F.halo[hb][0].active || F.halo[hb][1].active)) continue;
            if (threadIdx.x == 0)
                for (int side = 0; side < 2; ++side)
                    if (F.halo[hb][side].active) {
                        spin_geq(F, F.halo[hb][side].flag + ch, F.epoch);
                        spin_geq(F, F.halo[hb][side].xflag + ch, F.epoch);
                    }
            __syncthreads();
            bool fwd = false;
            for (int side = 0; side < 2; ++side)
                for (int rs = 0; rs < 2; ++rs) {
                    if (hb == 0) fwd |= forward_line(F, 0, side, 1, rs, zr.x, zr.y, q, F.nfwd);
                    if (F.face[2][rs].layer >= zr.x && F.face[2][rs].layer < zr.y)
                        fwd |= forward_line(F, hb, side, 2, rs, 0, F.s[hb == 0 ? 1 : 0], q, F.nfwd);
                }
            if (__syncthreads_or(fwd)) __threadfence_system();
            __syncthreads();
            if (threadIdx.x == 0)
                for (int a = hb + 1; a < 3; ++a)
                    for (int rs = 0; rs < 2; ++rs) {
                        if (!F.face[a][rs].active) continue;
                        if (a == 1)
                            contribute_x(F, 1, rs, ch);
                        else if (F.face[2][rs].layer >= zr.x && F.face[2][rs].layer < zr.y)
                            contribute_x(F, 2, rs, 0);
                    }
        }
    }
}

// Pipelined schedule, after the last step of a run: every incoming face (data and rim/forwarded
// cells) of the epoch has arrived -- the step is complete for any later work on the stream.
// Staged x faces: also copies the last epoch's staged x halo columns (inner rows and planes) into T2,
// every block its share after the x data flags.
__global__ void fused_drain_kernel(const __grid_constant__ FusedParams F) {
    if (blockIdx.x == 0)
        for (int f = threadIdx.x; f < 6 * F.nchunks; f += blockDim.x) {
            const int a = f / (2 * F.nchunks), rs = (f / F.nchunks) & 1, ch = f % F.nchunks;
            const FusedHalo &h = F.halo[a][rs];
            if (!h.active || (a == 2 && ch > 0)) continue;
            spin_geq(F, h.flag + ch, F.epoch);
            spin_geq(F, h.xflag + ch, F.epoch);
        }
    if (!F.xstage || F.xblk) return;   // (x blocks: the receiver blocks already wrote the columns)
    for (int f = threadIdx.x; f < 2 * F.nchunks; f += blockDim.x)
        if (F.halo[0][f / F.nchunks].active) spin_geq(F, F.halo[0][f / F.nchunks].flag + f % F.nchunks, F.epoch);
    __syncthreads();
    const int sx = F.s[0], sy = F.s[1], sz = F.s[2];
    const long long sxy = (long long)sx * sy, ncell = (long long)(sy - 2) * (sz - 2);
    for (int side = 0; side < 2; ++side) {
        if (!F.halo[0][side].active) continue;
        const int hx = side == 0 ? 0 : sx - 1;
        for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ncell;
             t += (long long)gridDim.x * blockDim.x) {
            const int z = 1 + (int)(t % (sz - 2)), y = 1 + (int)(t / (sz - 2));
            F.T2[(long long)z * sxy + (long long)y * sx + hx] = __ldcg(F.xstg + xstg_at(F, F.epoch, side, y, z));
        }
    }
}

// ------------------------------------------------------------------ host side
bool fused_eligible(const igg_grid *g) {
    if (g->fused == 2 && g->nlocal == 1) return true;   // ablation/profiling: force the fused kernel
    if (g->path != IGG_PATH_P2P || g->nlocal != 1 || g->fused == 0) return false;
    bool any = false, self = false;
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 2; ++k) {
            const int nb = g->nbr[0][a][k];
            if (nb < 0) continue;
            any = true;
            self = self || proc_of(g, nb) == g->proc;   // a periodic axis wrapping onto this process
        }
    if (!any) return false;                               // nothing to exchange: the plain stencil
    if (self && (g->fused_mode & 128)) return false;      // legacy schedule: stream-ordered path
    if (g->n[0] < 66 || g->n[1] < 6 || g->n[2] < 6) return false;   // one x send layer per 64-cell segment
    return true;
}

static int g_fused_occ = -1, g_fused_nsm = 0;

// chunks: 64 planes, the last ~2 waves in 8-plane chunks; the chunk holding
// plane n2-2 (the upper z send layer) is visited second, right after chunk 0
// (holding plane 1).  The layout depends on the geometry only, so every rank
// numbers chunks identically (flags are per chunk position).
static void build_layout(igg_grid *g, const int layer[3][2], const bool act[3][2]) {
    const int n0 = g->n[0], n1 = g->n[1], n2 = g->n[2];
    const int xtiles = (n0 - 1 + 63) / 64;
    const int ytiles = (n1 - 2 + kFTY - 1) / kFTY;
    const int wz = n2 - 2;
    if (g_fused_occ < 0) {
        IGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_fused_occ, heat_fused_kernel<false>, 32 * kFTY, 0));
        IGG_CUDA(cudaDeviceGetAttribute(&g_fused_nsm, cudaDevAttrMultiProcessorCount, g->device));
    }
    // tail chunk planes: short chunks shorten the last wave; on the legacy schedule every chunk also
    // adds one hop to the receive side's forwarding chain when several axes exchange (measured there:
    // 8 for one axis, 16 for more); the pipelined schedule keeps forwarding off the critical path: 8
    int naxes = 0;
    for (int a = 0; a < 3; ++a) naxes += (act[a][0] || act[a][1]) ? 1 : 0;
    const bool legacy = (g->fused_mode & 128) != 0;
    const int kc1 = kFKC, kc2 = g->fused_kc2 > 0 ? g->fused_kc2 : ((naxes <= 1 || !legacy) ? 8 : 16);
    const long long ntile = (long long)xtiles * ytiles;
    int small = (int)((2LL * g_fused_occ * g_fused_nsm * kc2 + ntile - 1) / ntile);
    small = std::min(((small + kc2 - 1) / kc2) * kc2, wz);
    const int nbig = (wz - small) / kc1;
    std::vector<int2> zc;   // by chunk id
    for (int c = 0; c < nbig; ++c) zc.push_back(make_int2(1 + c * kc1, 1 + (c + 1) * kc1));
    for (int z = 1 + nbig * kc1; z < 1 + wz; z += kc2) zc.push_back(make_int2(z, std::min(z + kc2, 1 + wz)));
    const int nch = (int)zc.size();
    if (nch > kMaxChunks) fail(IGG_E_UNSUPPORTED, "fused step: too many z-chunks");
    // natural chunk order (measured best); fused_mode bit 64: visit the chunk holding the upper z send
    // layer second (ablation)
    int cz = 0;
    if ((act[2][0] || act[2][1]) && (g->fused_mode & 64))
        for (int c = 0; c < nch; ++c)
            if (n2 - 2 >= zc[c].x && n2 - 2 < zc[c].y) cz = c;
    // visit order position of each chunk id (mirror of chunk_id() on the device)
    auto id_of = [&](int oc) { return (cz <= 1 || oc == 0) ? oc : (oc == 1 ? cz : (oc - 1 < cz ? oc - 1 : oc)); };
    g->fused_zchunk[0] = g->fused_zchunk[1] = -1;
    for (int oc = 0; oc < nch; ++oc) {
        const int2 r = zc[id_of(oc)];
        for (int rs = 0; rs < 2; ++rs)
            if (act[2][rs] && layer[2][rs] >= r.x && layer[2][rs] < r.y) g->fused_zchunk[rs] = oc;
    }
    g->fused_zafter = 0;
    for (int oc = 0; oc < nch; ++oc) {
        const int2 r = zc[id_of(oc)];
        if ((1 >= r.x && 1 < r.y) || (n2 - 2 >= r.x && n2 - 2 < r.y)) g->fused_zafter = std::max(g->fused_zafter, oc);
    }
    // targets: tiles holding (face, chunk) + 1 (rim) + forwarding comm CTAs
    int xsides = 0, ysides = 0;
    for (int sd = 0; sd < 2; ++sd) {
        xsides += g->nbr[0][0][sd] >= 0 ? 1 : 0;
        ysides += g->nbr[0][1][sd] >= 0 ? 1 : 0;
    }
    const unsigned xfw = xsides ? g->fused_ncomm : 0, yfw = ysides ? g->fused_ncomm : 0;   // forwarding CTAs
    std::vector<unsigned> tgt(6 * kMaxChunks, 0u);
    for (int rs = 0; rs < 2; ++rs) {
        for (int c = 0; c < nch; ++c) {
            if (act[0][rs]) tgt[(0 * 2 + rs) * kMaxChunks + c] = ytiles + 1;
            if (act[1][rs]) tgt[(1 * 2 + rs) * kMaxChunks + c] = xtiles + 1 + xfw;
        }
        if (act[2][rs]) tgt[(2 * 2 + rs) * kMaxChunks] = xtiles * ytiles + 1 + xfw + yfw;
    }
    if (!g->fused_tgt) {
        IGG_CUDA(cudaMalloc(&g->fused_tgt, tgt.size() * sizeof(unsigned)));
        g->allocs++;
    }
    IGG_CUDA(cudaMemcpy(g->fused_tgt, tgt.data(), tgt.size() * sizeof(unsigned), cudaMemcpyHostToDevice));
    // pipelined schedule: face tiles complete the data flags; the rim (1) and the in-kernel forwarders
    // complete the xflags (forwarders exist only when a later face takes an earlier axis' halo lines)
    bool xh = false, yh = false;
    for (int sd = 0; sd < 2; ++sd) {
        xh = xh || g->nbr[0][0][sd] >= 0;
        yh = yh || g->nbr[0][1][sd] >= 0;
    }
    const bool yf = act[1][0] || act[1][1], zf = act[2][0] || act[2][1];
    // (fused_mode bit 512: timing experiment without forwarders -- edge/corner halo cells INVALID)
    const bool need_fwd = ((xh && (yf || zf)) || (yh && zf)) && !(g->fused_mode & 512);
    g->fused_nfwd = need_fwd ? g->fused_ncomm : 0;
    const unsigned nf = (unsigned)g->fused_nfwd;
    // staged x faces moved by dedicated sender blocks (their count completes the data flag)
    const bool xblk = (g->fused_mode & 2048) && !(g->fused_mode & (4 | 128 | 256));
    std::vector<unsigned> tgt_d(6 * kMaxChunks, 0u), tgt_x(6 * kMaxChunks, 0u);
    for (int rs = 0; rs < 2; ++rs) {
        for (int c = 0; c < nch; ++c) {
            if (act[0][rs]) {
                tgt_d[(0 * 2 + rs) * kMaxChunks + c] = xblk ? (unsigned)g->fused_nxb : ytiles;
                tgt_x[(0 * 2 + rs) * kMaxChunks + c] = 1;
            }
            if (act[1][rs]) {
                tgt_d[(1 * 2 + rs) * kMaxChunks + c] = xtiles;
                tgt_x[(1 * 2 + rs) * kMaxChunks + c] = 1 + (xh ? nf : 0);
            }
        }
        if (act[2][rs]) {
            tgt_d[(2 * 2 + rs) * kMaxChunks] = xtiles * ytiles;
            tgt_x[(2 * 2 + rs) * kMaxChunks] = 1 + (xh ? nf : 0) + (yh ? nf : 0);
        }
    }
    for (auto *pp : {&g->fused_tgt_pipe, &g->fused_tgt_x})
        if (!*pp) {
            IGG_CUDA(cudaMalloc(pp, 6 * kMaxChunks * sizeof(unsigned)));
            g->allocs++;
        }
    IGG_CUDA(cudaMemcpy(g->fused_tgt_pipe, tgt_d.data(), tgt_d.size() * sizeof(unsigned), cudaMemcpyHostToDevice));
    IGG_CUDA(cudaMemcpy(g->fused_tgt_x, tgt_x.data(), tgt_x.size() * sizeof(unsigned), cudaMemcpyHostToDevice));
    g->fused_ntiles = (int)(ntile * nch);
    // tail: the last chunks' tiles (about 2-3 waves), face tiles first, so the last faces
    // leave a couple of waves before the stencil ends and the forwarding chain is hidden
    g->fused_tail.clear();
    g->fused_bmain = g->fused_ntiles;
    int ntail_ch = 0;
    while (ntail_ch < std::min(4, nch - 1) && (long long)(ntail_ch + 1) * ntile <= kMaxTail) ++ntail_ch;
    bool any_face = false;
    for (int a = 0; a < 3; ++a) any_face = any_face || act[a][0] || act[a][1];
    // no faces: nothing to reorder (natural order, no table); fused_mode bit 32: no table (ablation)
    if (any_face && !(g->fused_mode & 32) && xtiles <= 16 && ytiles <= 1024 && ntail_ch > 0) {
        const int c0 = nch - ntail_ch;
        std::vector<unsigned short> face_t, rest_t;
        for (int oc = c0; oc < nch; ++oc) {
            const int2 r = zc[id_of(oc)];
            for (int yt = 0; yt < ytiles; ++yt)
                for (int xt = 0; xt < xtiles; ++xt) {
                    bool face = false;
                    const int xlo = std::max(xt * 64, 1), xhi = std::min(xt * 64 + 64, n0 - 1);
                    const int ty0 = 1 + yt * kFTY, yhi = std::min(ty0 + kFTY, n1 - 1);
                    for (int rs = 0; rs < 2; ++rs) {
                        face |= act[0][rs] && layer[0][rs] >= xlo && layer[0][rs] < xhi;
                        face |= act[1][rs] && layer[1][rs] >= ty0 && layer[1][rs] < yhi;
                        face |= act[2][rs] && layer[2][rs] >= r.x && layer[2][rs] < r.y;
                    }
                    const unsigned short e = (unsigned short)(xt | (yt << 4) | ((oc - c0) << 14));
                    (face ? face_t : rest_t).push_back(e);
                }
        }
        g->fused_tail = face_t;
        g->fused_tail.insert(g->fused_tail.end(), rest_t.begin(), rest_t.end());
        g->fused_bmain = (int)(ntile * c0);
    }
    g->fused_nchunks = nch;
    g->fused_geo[0] = nbig;
    g->fused_geo[1] = kc1;
    g->fused_geo[2] = kc2;
    g->fused_geo[3] = cz;
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
    if (g->nproc_procs == 1) {   // self-wrap on one process: entries are my own arrays; drop stale ones
        std::vector<igg_grid::PeerMap> keep;
        for (auto &m : g->fused_peer_maps)
            if (same_alloc(m, alloc_id(m.ptr))) keep.push_back(m);
        g->fused_peer_maps.swap(keep);
        return;
    }
    if (g->fused_peer_maps.empty() && g->fused_opened.empty()) {
        // nothing cached here; the other processes hold nothing either (entries are created collectively)
        return;
    }
    unsigned char ok = 1;
    for (auto &m : g->fused_peer_maps) ok = ok && same_alloc(m, alloc_id(m.ptr));
    std::vector<char> all = allgather_bytes_pub(g, &ok, 1);
    for (char c : all)
        if (!c) {
            release_peer_maps(g);
            return;
        }
}

static const std::vector<double *> &peer_arrays(igg_grid *g, double *T2) {
    const AllocId id = alloc_id(T2);
    for (auto &m : g->fused_peer_maps)
        if (m.ptr == (const void *)T2) {
            if (!same_alloc(m, id) && g->nproc_procs == 1) {   // self-wrap: the peer is this array itself
                m.base = id.base;
                m.size = id.size;
                m.buffer_id = id.buffer_id;
            } else if (!same_alloc(m, id))
                fail(IGG_E_STATE, "fused step: an array was freed and re-allocated at the same address after its "
                                  "first fused step; call igg_release_arrays (collective) before reusing it");
            return m.peers;
        }
    igg_grid::PeerMap e;
    e.ptr = T2;
    e.base = id.base;
    e.size = id.size;
    e.buffer_id = id.buffer_id;
    if (g->nproc_procs == 1) {   // self-wrap on one process: my own array
        e.peers.assign(1, T2);
        g->fused_peer_maps.push_back(e);
        return g->fused_peer_maps.back().peers;
    }
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

void fused_step(igg_grid *g, double *T2, const double *T, const double *Ci, const HeatCoef &k, cudaStream_t s,
                bool wait_prev, bool drain) {
    if (!g->fused_ctr) {   // [data ctr | rim/forward ctr] x 6 x kMaxChunks, then tickets
        IGG_CUDA(cudaMalloc(&g->fused_ctr, (12 * kMaxChunks + 8) * sizeof(unsigned int)));
        IGG_CUDA(cudaMemset(g->fused_ctr, 0, (12 * kMaxChunks + 8) * sizeof(unsigned int)));
        g->allocs++;
    }
    const bool comm = !g->skip_comm;
    static const std::vector<double *> none;
    const std::vector<double *> peer = comm ? peer_arrays(g, T2) : none;   // a copy: the map may grow
    g->epoch++;
    FusedParams F{};
    F.T = T;
    F.Ci = Ci;
    F.T2 = T2;
    for (int a = 0; a < 3; ++a) F.s[a] = g->n[a];
    F.epoch = g->epoch;
    F.timeout_cycles = (long long)(g->spin_timeout_ms * g->clock_khz);
    F.err = g->d_err;
    F.k = k;
    F.ctr = g->fused_ctr;
    F.nostore = (g->fused_mode & 8) ? 1 : 0;
    int layer[3][2];
    bool act[3][2];
    for (int a = 0; a < 3; ++a)
        for (int rs = 0; rs < 2; ++rs) {
            // rs = receiver side: 0 <- my send_upper (layer n-2) into my upper neighbour's layer 0,
            //                     1 <- my send_lower (layer 1) into my lower neighbour's layer s-1
            const int nb = g->nbr[0][a][rs == 0 ? 1 : 0];
            layer[a][rs] = rs == 0 ? g->n[a] - 2 : 1;
            act[a][rs] = comm && nb >= 0;
            FusedFace &f = F.face[a][rs];
            f.layer = layer[a][rs];
            f.active = act[a][rs];
            if (f.active) {
                const int pp = proc_of(g, nb);
                // mode bit 16 (timing experiment, INVALID halos): the face stores go to my own T2
                f.dst = (g->fused_mode & 16) ? T2 : peer[pp];
                f.flag = g->peer_flags[pp] + (a * 2 + rs) * kMaxChunks;
                f.xflag = g->peer_flags[pp] + (6 + a * 2 + rs) * kMaxChunks;   // (one rank per process)
            }
            const int hb = g->nbr[0][a][rs];   // my halo side rs is filled by my neighbour on side rs
            FusedHalo &h = F.halo[a][rs];
            h.active = comm && hb >= 0;
            h.layer = rs == 0 ? 0 : g->n[a] - 1;
            h.flag = g->flags + (a * 2 + rs) * kMaxChunks;
            h.xflag = g->flags + (6 + a * 2 + rs) * kMaxChunks;
        }
    int key = 0;
    for (int a = 0; a < 3; ++a)
        for (int rs = 0; rs < 2; ++rs) key |= (act[a][rs] ? 1 : 0) << (a * 2 + rs);
    if (g->fused_key != key) {
        build_layout(g, layer, act);
        g->fused_key = key;
    }
    F.nchunks = g->fused_nchunks;
    F.nbig = g->fused_geo[0];
    F.kc1 = g->fused_geo[1];
    F.kc2 = g->fused_geo[2];
    F.cz = g->fused_geo[3];
    F.xtiles = g->fused_geo[4];
    F.ytiles = g->fused_geo[5];
    F.bmain = g->fused_bmain;
    std::copy(g->fused_tail.begin(), g->fused_tail.end(), F.tail);
    F.zchunk[0] = g->fused_zchunk[0];
    F.zchunk[1] = g->fused_zchunk[1];
    F.tgt = g->fused_tgt;

    // a single complete step that needs edge forwarding runs the multi-stream schedule (its receive
    // kernels forward while the stencil runs; measured faster than in-kernel forwarders for one step)
    // (every schedule is ONE launch on the caller's stream: kernels on other streams that spin on this
    // launch's flags are never relied on -- nothing guarantees that two launches run at the same time)
    const bool single_fwd = false;
    if (!(g->fused_mode & 128) && !single_fwd) {
        // pipelined schedule (default): ONE launch on the caller's stream and, when the step must be
        // complete on return, a drain.  The rim cells and the forwarded edge lines are never read by
        // the stencil, so only the step that completes a run sends them (rim blocks + forwarders in
        // its launch); the steps before it move only the faces the next step's tiles read.
        const bool recv = comm && !(g->fused_mode & 4);   // mode bit 4: timing without receive side
        F.pipe = 1;
        F.wait_prev = (wait_prev && recv) ? 1 : 0;
        F.nrim = (comm && drain) ? 48 : 0;
        F.nstencil = g->fused_ntiles;
        F.nfwd = (recv && drain) ? g->fused_nfwd : 0;
        F.tgt = g->fused_tgt_pipe;
        F.ctr_x = g->fused_ctr + 6 * kMaxChunks;
        F.tgt_x = g->fused_tgt_x;
        F.rim_ticket = g->fused_ctr + 12 * kMaxChunks;
        // x faces staged in the receiver's compact buffer (default) or stored straight into its T2
        // column (fused_mode bit 256, ablation: one 8-B value per 32-B sector)
        F.xstage = (recv && !(g->fused_mode & 256) && (F.halo[0][0].active || F.halo[0][1].active)) ? 1 : 0;
        F.xhint = (g->fused_mode & 4096) ? 1 : 0;
        if (F.xstage) {
            if (!g->fused_xstg) {
                IGG_CUDA(cudaMalloc(&g->fused_xstg, sizeof(double) * 4 * (size_t)g->n[1] * g->n[2]));
                g->allocs++;
            }
            const std::vector<double *> pstg = peer_arrays(g, g->fused_xstg);
            F.xstg = g->fused_xstg;
            for (int rs = 0; rs < 2; ++rs)
                if (F.face[0][rs].active) F.xstg_peer[rs] = pstg[proc_of(g, g->nbr[0][0][rs == 0 ? 1 : 0])];
            // dedicated x sender/receiver blocks (fused_mode bit 2048, ablation: measured slower -- a few
            // blocks cannot keep up with one scattered 8-B read per row and plane; the face tiles, spread
            // over the whole grid, move the column faster)
            F.xblk = (g->fused_mode & 2048) ? 1 : 0;
            if (F.xblk) {
                if (!g->fused_xsync) {
                    const size_t bytes = 4 * kMaxChunks * (sizeof(unsigned int) + sizeof(unsigned long long));
                    IGG_CUDA(cudaMalloc(&g->fused_xsync, bytes));
                    IGG_CUDA(cudaMemset(g->fused_xsync, 0, bytes));
                    g->allocs++;
                }
                F.xev = static_cast<unsigned long long *>(g->fused_xsync);
                F.xcnt = reinterpret_cast<unsigned int *>(F.xev + 4 * kMaxChunks);
                F.nxb = g->fused_nxb;
            }
        }
        const int blocks = F.nrim + F.nfwd + 4 * F.nxb + F.nstencil;
        prof_begin(g, s);
        if (g->fused_mode & 1)
            heat_fused_kernel<true><<<blocks, 32 * kFTY, 0, s>>>(F);
        else
            heat_fused_kernel<false><<<blocks, 32 * kFTY, 0, s>>>(F);
        IGG_CUDA(cudaGetLastError());
        g->launches++;
        prof_end(g, s, (long long)(g->n[0] - 2) * (g->n[1] - 2) * (g->n[2] - 2));
        if (drain && recv) {
            fused_drain_kernel<<<(F.xstage && !F.xblk) ? 2 * g->sm_count : 1, 128, 0, s>>>(F);
            IGG_CUDA(cudaGetLastError());
            g->launches++;
        }
        return;
    }

    // legacy schedule (fused_mode bit 128, ablation): rim and receive/forward kernels on the comm
    // streams, the stencil on the inner stream, joined by events
    IGG_CUDA(cudaEventRecord(g->ev_start, s));
    IGG_CUDA(cudaStreamWaitEvent(g->s_comm, g->ev_start, 0));
    tl_mark(g, s, 0);
    if (comm) {
        // rim first (tiny), then the waiting unpack CTAs of every axis: they sit in the
        // SM slots the register-limited stencil leaves free and unpack chunk by chunk
        const int rim_blocks = 8;
        fused_rim_kernel<<<dim3(rim_blocks, 6), 256, 0, g->s_comm>>>(F, g->fused_ctr + 6 * kMaxChunks,
                                                                     rim_blocks * 6);
        IGG_CUDA(cudaGetLastError());
        g->launches++;
    }
    tl_mark(g, g->s_comm, 1);
    // the stencil on the caller's stream (fused_mode bit 1: on the low-priority inner stream)
    cudaStream_t ss = (g->fused_mode & 2) ? g->s_inner : s;
    if (ss != s) IGG_CUDA(cudaStreamWaitEvent(ss, g->ev_start, 0));
    tl_mark(g, ss, 2);
    prof_begin(g, ss);
    if (g->fused_mode & 1)
        heat_fused_kernel<true><<<g->fused_ntiles, 32 * kFTY, 0, ss>>>(F);
    else
        heat_fused_kernel<false><<<g->fused_ntiles, 32 * kFTY, 0, ss>>>(F);
    IGG_CUDA(cudaGetLastError());
    g->launches++;
    prof_end(g, ss, (long long)(g->n[0] - 2) * (g->n[1] - 2) * (g->n[2] - 2));
    tl_mark(g, ss, 3);
    if (ss != s) {
        IGG_CUDA(cudaEventRecord(g->ev_inner, ss));
        IGG_CUDA(cudaStreamWaitEvent(s, g->ev_inner, 0));
    }
    if (comm && !(g->fused_mode & 4)) {   // mode bit 4: timing experiment without receive side (INVALID)
        const bool xa = F.halo[0][0].active || F.halo[0][1].active;
        const bool yza = F.halo[1][0].active || F.halo[1][1].active || F.halo[2][0].active || F.halo[2][1].active;
        if (xa) {
            fused_comm_kernel<<<g->fused_ncomm, 128, 0, g->s_comm>>>(F, g->fused_zafter, 1);
            IGG_CUDA(cudaGetLastError());
            g->launches++;
        }
        if (yza) {
            IGG_CUDA(cudaStreamWaitEvent(g->s_comm2, g->ev_start, 0));
            fused_comm_kernel<<<g->fused_ncomm, 128, 0, g->s_comm2>>>(F, g->fused_zafter, 6);
            IGG_CUDA(cudaGetLastError());
            g->launches++;
            IGG_CUDA(cudaEventRecord(g->ev_comm2, g->s_comm2));
            IGG_CUDA(cudaStreamWaitEvent(g->s_comm, g->ev_comm2, 0));
        }
    }
    tl_mark(g, g->s_comm, 4);
    IGG_CUDA(cudaEventRecord(g->ev_comm, g->s_comm));
    IGG_CUDA(cudaStreamWaitEvent(s, g->ev_comm, 0));
}

}  // namespace igg
