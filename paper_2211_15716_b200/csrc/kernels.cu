// kernels.cu -- the sm_100a kernels of libigg: the Fig. 1 heat stencil
// (generic region-list kernel and a vectorised z-sweep box kernel), the face
// pack/unpack kernels of update_halo (with NVLink peer stores and
// release/acquire flags), and a max reduction for dt.
//
// Fp64 throughout ("@init_parallel_stencil(CUDA, Float64, 3)").
// No tensor cores: the 7-point stencil is not a contraction.
#include <algorithm>
#include <cstdio>

#include "igg_internal.h"

namespace igg {

// ============================================================== the cell
// PAPER.md:46-49 (listing 7-10) with DESIGN.md readings 6-9:
//   T2 = T + dt*((lam*Ci)*(((d2x*rdx2) + (d2y*rdy2)) + (d2z*rdz2)))
//   d2x = (T[x+1]-T[x]) - (T[x]-T[x-1])
// Every operation is an explicitly rounded binary64 op, so the compiler can
// never contract to FMA: every kernel and region computes bit-identical cells.
__device__ __forceinline__ double heat_cell(double c, double xm, double xp, double ym, double yp,
                                            double zm, double zp, double ci, const HeatCoef &k) {
    const double d2x = __dsub_rn(__dsub_rn(xp, c), __dsub_rn(c, xm));
    const double d2y = __dsub_rn(__dsub_rn(yp, c), __dsub_rn(c, ym));
    const double d2z = __dsub_rn(__dsub_rn(zp, c), __dsub_rn(c, zm));
    const double lap =
        __dadd_rn(__dadd_rn(__dmul_rn(d2x, k.rdx2), __dmul_rn(d2y, k.rdy2)), __dmul_rn(d2z, k.rdz2));
    return __dadd_rn(c, __dmul_rn(k.dt, __dmul_rn(__dmul_rn(k.lam, ci), lap)));
}

// ============================================================== generic region kernel
// One thread per (x,y) column of a region, sweeping a chunk of kRegKc planes in
// z with a register queue (T[z-1], T[z], T[z+1]); x/y neighbours come through
// L1.  Used for the six thin boundary slabs of hide_communication and for
// fields whose rows are not 16-B aligned.
constexpr int kRegThreads = 256;
constexpr int kRegKc = 32;

__global__ void __launch_bounds__(kRegThreads) heat_regions_kernel(const __grid_constant__ HeatRegionList L) {
    const int b = blockIdx.x;
    int ri = 0;
    while (ri + 1 < L.n && b >= L.r[ri + 1].block_begin) ++ri;
    const HeatRegion &R = L.r[ri];
    const int local = b - R.block_begin;
    const int cb = local % R.col_blocks, zc = local / R.col_blocks;
    const long long col = (long long)cb * kRegThreads + threadIdx.x;
    if (col >= (long long)R.wx * R.wy) return;
    const int x = R.x0 + (int)(col % R.wx);
    const int y = R.y0 + (int)(col / R.wx);
    int z = R.z0 + zc * kRegKc;
    const int zend = min(R.z0 + R.wz, z + kRegKc);
    const long long sx = R.sx, sxy = (long long)R.sx * R.sy;
    const double *__restrict__ T = R.T;
    const double *__restrict__ Ci = R.Ci;
    double *__restrict__ T2 = R.T2;
    long long i = (long long)z * sxy + (long long)y * sx + x;
    double zm = __ldg(T + i - sxy), c = __ldg(T + i);
    for (; z < zend; ++z, i += sxy) {
        const double zp = __ldg(T + i + sxy);
        const double xm = __ldg(T + i - 1), xp = __ldg(T + i + 1);
        const double ym = __ldg(T + i - sx), yp = __ldg(T + i + sx);
        const double ci = __ldg(Ci + i);
        T2[i] = heat_cell(c, xm, xp, ym, yp, zm, zp, ci, L.k);
        zm = c;
        c = zp;
    }
}

void launch_heat_regions(HeatRegionList &L, cudaStream_t s) {
    int total = 0;
    for (int r = 0; r < L.n; ++r) {
        HeatRegion &R = L.r[r];
        const long long cols = (long long)R.wx * R.wy;
        R.col_blocks = (int)((cols + kRegThreads - 1) / kRegThreads);
        R.zchunks = (R.wz + kRegKc - 1) / kRegKc;
        R.block_begin = total;
        total += R.col_blocks * R.zchunks;
    }
    L.total_blocks = total;
    if (total == 0) return;
    heat_regions_kernel<<<total, kRegThreads, 0, s>>>(L);
    IGG_CUDA(cudaGetLastError());
}

// ============================================================== vectorised box kernel
// Tile = 64 x-cells x kBoxTY rows; a warp owns one 64-cell row segment, each
// lane two consecutive cells (one 16-B double2 load/store per field).  The
// CTA sweeps kBoxKc planes in z keeping T[z-1], T[z], T[z+1] of its cells in
// registers; x neighbours come from the neighbouring lane by warp shuffle
// (lanes 0/31 fetch one scalar across the tile edge); y neighbours are the
// rows of the adjacent warps (L1 hits; tile-edge rows from L2).  DRAM sees
// T, Ci read once and T2 written once per cell plus tile-edge re-reads:
// 24 B/cell algorithmic.
constexpr int kBoxTY = 8;
constexpr int kBoxThreads = 32 * kBoxTY;
constexpr int kBoxKc = 32;

__global__ void __launch_bounds__(kBoxThreads)
    heat_box_kernel(const double *__restrict__ T, const double *__restrict__ Ci, double *__restrict__ T2,
                    int sx, int sy, int x0, int y0, int z0, int wx, int wy, int wz, int ax0, int xtiles,
                    int ytiles, const HeatCoef k) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    int b = blockIdx.x;
    const int tx = b % xtiles;
    b /= xtiles;
    const int ty = b % ytiles;
    const int tz = b / ytiles;
    const int y = y0 + ty * kBoxTY + warp;
    if (y >= y0 + wy) return;                       // whole warp leaves together
    const int p = ax0 + tx * 64 + 2 * lane;          // first of my two cells
    const int xend = x0 + wx;
    const bool pair_in = p < sx;                     // sx even: p+1 < sx too
    const bool w0 = pair_in && p >= x0 && p < xend;
    const bool w1 = pair_in && p + 1 >= x0 && p + 1 < xend;
    int z = z0 + tz * kBoxKc;
    const int zend = min(z0 + wz, z + kBoxKc);
    const long long sxy = (long long)sx * sy;
    long long i = (long long)z * sxy + (long long)y * sx + p;   // even -> 16-B aligned
    const double2 zero2 = make_double2(0.0, 0.0);
    double2 zm = pair_in ? __ldg(reinterpret_cast<const double2 *>(T + i - sxy)) : zero2;
    double2 c = pair_in ? __ldg(reinterpret_cast<const double2 *>(T + i)) : zero2;
    for (; z < zend; ++z, i += sxy) {
        double2 zp = zero2, ym = zero2, yp = zero2, ci = zero2;
        if (pair_in) {
            zp = __ldg(reinterpret_cast<const double2 *>(T + i + sxy));
            ym = __ldg(reinterpret_cast<const double2 *>(T + i - sx));
            yp = __ldg(reinterpret_cast<const double2 *>(T + i + sx));
            ci = __ldg(reinterpret_cast<const double2 *>(Ci + i));
        }
        double xm = __shfl_up_sync(0xffffffffu, c.y, 1);
        double xp = __shfl_down_sync(0xffffffffu, c.x, 1);
        if (lane == 0 && w0) xm = __ldg(T + i - 1);
        if (lane == 31 && w1) xp = __ldg(T + i + 2);
        const double r0 = heat_cell(c.x, xm, c.y, ym.x, yp.x, zm.x, zp.x, ci.x, k);
        const double r1 = heat_cell(c.y, c.x, xp, ym.y, yp.y, zm.y, zp.y, ci.y, k);
        if (w0 && w1) {
            *reinterpret_cast<double2 *>(T2 + i) = make_double2(r0, r1);
        } else {
            if (w0) T2[i] = r0;
            if (w1) T2[i + 1] = r1;
        }
        zm = c;
        c = zp;
    }
}

bool heat_box_vectorizable(const HeatRegion &r) {
    return (r.sx % 2 == 0) && ((reinterpret_cast<uintptr_t>(r.T) | reinterpret_cast<uintptr_t>(r.Ci) |
                                reinterpret_cast<uintptr_t>(r.T2)) % 16 == 0);
}

void launch_heat_box(const HeatRegion &r, const HeatCoef &k, cudaStream_t s) {
    if (r.wx <= 0 || r.wy <= 0 || r.wz <= 0) return;
    const int ax0 = r.x0 & ~1;
    const int xtiles = (r.x0 + r.wx - ax0 + 63) / 64;
    const int ytiles = (r.wy + kBoxTY - 1) / kBoxTY;
    const int ztiles = (r.wz + kBoxKc - 1) / kBoxKc;
    const long long blocks = (long long)xtiles * ytiles * ztiles;
    heat_box_kernel<<<(unsigned)blocks, kBoxThreads, 0, s>>>(r.T, r.Ci, r.T2, r.sx, r.sy, r.x0, r.y0, r.z0,
                                                             r.wx, r.wy, r.wz, ax0, xtiles, ytiles, k);
    IGG_CUDA(cudaGetLastError());
}

// ============================================================== face pack / unpack
// Buffer layout: x fastest, then y, then z, over the slab.
__device__ __forceinline__ long long face_index(const CopyDesc &d, long long i) {
    if (d.axis == 0) {
        const long long xl = i % d.h, r = i / d.h;
        const long long y = r % d.sy, z = r / d.sy;
        return (z * d.sy + y) * d.sx + d.lo + xl;
    }
    if (d.axis == 1) {
        const long long x = i % d.sx, r = i / d.sx;
        const long long yl = r % d.h, z = r / d.h;
        return (z * d.sy + d.lo + yl) * d.sx + x;
    }
    const long long x = i % d.sx, r = i / d.sx;
    const long long y = r % d.sy, zl = r / d.sy;
    return ((d.lo + zl) * d.sy + y) * d.sx + x;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

constexpr int kCopyThreads = 256;

// pack: field slab -> buffer (own send buffer, a local rank's receive slot, or a
// peer GPU's receive slot over NVLink).  If the list carries signals, the last
// CTA to finish publishes the epoch to the peers' receive flags: every thread
// fences its stores (system scope) before the CTA barrier, the elected CTA
// acquires through the ticket and release-stores each flag.
__global__ void __launch_bounds__(kCopyThreads) pack_kernel(const __grid_constant__ CopyList L) {
    const CopyDesc &d = L.d[blockIdx.y];
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < d.count; i += stride)
        d.buf[i] = d.field[face_index(d, i)];
    if (L.nsignal > 0) {
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned t = atomicAdd(L.ticket, 1u);
            if (t == L.ticket_total - 1) {
                __threadfence_system();
                for (int s = 0; s < L.nsignal; ++s) st_release_sys(L.signal[s], L.epoch);
                atomicExch(L.ticket, 0u);
            }
        }
    }
}

// unpack: buffer -> field receive slab.  A slot filled by a peer GPU is read
// only after its flag reached this call's epoch (bounded spin; a timeout sets
// *err and is reported by igg_check).
__global__ void __launch_bounds__(kCopyThreads) unpack_kernel(const __grid_constant__ CopyList L) {
    const CopyDesc &d = L.d[blockIdx.y];
    if (d.flag_slot >= 0) {
        if (threadIdx.x == 0) {
            const unsigned long long *f = L.wait[d.flag_slot];
            const long long t0 = clock64();
            while (ld_acquire_sys(f) < L.epoch) {
                if (clock64() - t0 > L.timeout_cycles) {
                    atomicExch(L.err, 1);
                    break;
                }
                __nanosleep(64);
            }
        }
        __syncthreads();
    }
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < d.count; i += stride)
        d.field[face_index(d, i)] = __ldcg(d.buf + i);
}

static int copy_blocks(const CopyDesc *d, int n) {
    long long mx = 1;
    for (int j = 0; j < n; ++j) mx = d[j].count > mx ? d[j].count : mx;
    long long b = (mx + kCopyThreads * 4 - 1) / (kCopyThreads * 4);
    if (b < 1) b = 1;
    if (b > 1024) b = 1024;
    return (int)b;
}

int launch_copies(int op, const std::vector<CopyDesc> &descs, const CopyList &proto, cudaStream_t s) {
    const int n = (int)descs.size();
    if (n == 0) return 0;
    // total blocks of all chunks: the pack block that draws the last ticket
    // (necessarily in the last chunk, stream order) publishes the flags
    unsigned total = 0;
    for (int c = 0; c < n; c += kMaxCopy) {
        const int m = std::min(kMaxCopy, n - c);
        total += (unsigned)copy_blocks(descs.data() + c, m) * m;
    }
    int launches = 0;
    for (int c = 0; c < n; c += kMaxCopy) {
        CopyList L = proto;
        L.n = std::min(kMaxCopy, n - c);
        for (int j = 0; j < L.n; ++j) L.d[j] = descs[c + j];
        L.ticket_total = total;
        dim3 grid(copy_blocks(L.d, L.n), L.n);
        if (op == 0)
            pack_kernel<<<grid, kCopyThreads, 0, s>>>(L);
        else
            unpack_kernel<<<grid, kCopyThreads, 0, s>>>(L);
        IGG_CUDA(cudaGetLastError());
        ++launches;
    }
    return launches;
}

// ============================================================== max reduction
constexpr int kMaxThreads = 256;
constexpr int kMaxPartials = 1184;   // 148 SMs x 8
constexpr int kMaxPtrs = 16;
struct PtrList {
    const double *p[kMaxPtrs];
    int n;
    long long count;
};

__device__ __forceinline__ double block_max(double v) {
    __shared__ double sm[kMaxThreads / 32];
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < kMaxThreads / 32 ? sm[threadIdx.x] : -INFINITY;
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    return v;
}

__global__ void __launch_bounds__(kMaxThreads) max_partial_kernel(const PtrList P, double *partial) {
    double v = -INFINITY;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (int j = 0; j < P.n; ++j)
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P.count; i += stride)
            v = fmax(v, __ldg(P.p[j] + i));
    v = block_max(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

__global__ void __launch_bounds__(kMaxThreads) max_final_kernel(const double *partial, int n, double *out) {
    double v = -INFINITY;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v = fmax(v, partial[i]);
    v = block_max(v);
    if (threadIdx.x == 0) *out = v;
}

int field_max_scratch_len() { return kMaxPartials; }

void launch_field_max(const double *const *ptrs, int n, long long count, double *scratch, int scratch_len,
                      double *out_dev, cudaStream_t s) {
    if (n > kMaxPtrs) fail(IGG_E_ARG, "field max: too many local ranks");
    PtrList P;
    for (int j = 0; j < n; ++j) P.p[j] = ptrs[j];
    P.n = n;
    P.count = count;
    long long b = (count + kMaxThreads - 1) / kMaxThreads;
    if (b > scratch_len) b = scratch_len;
    if (b < 1) b = 1;
    max_partial_kernel<<<(int)b, kMaxThreads, 0, s>>>(P, scratch);
    IGG_CUDA(cudaGetLastError());
    max_final_kernel<<<1, kMaxThreads, 0, s>>>(scratch, (int)b, out_dev);
    IGG_CUDA(cudaGetLastError());
}

}  // namespace igg
