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

// IGG_ABLATION (a separate build, ablation/libigg_ablation.so): the tuning variants measured in profiles/
// (IGG_OPT_STENCIL_KERNEL 2..56 binary64, 100..126 binary32); the product library has only the defaults
#ifndef IGG_ABLATION
#define IGG_ABLATION 0
#endif

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

// ============================================================== 1-D / 2-D grids
// A size-1 axis (reading 23) has no second difference: the Laplacian sums the
// extended axes' terms in x, y, z order (left to right), and its one layer is updated.  One thread per
// cell of the updated box (inner layers of the extended axes), x fastest.
__global__ void __launch_bounds__(256) heat_lowdim_kernel(double *__restrict__ T2, const double *__restrict__ T,
                                                          const double *__restrict__ Ci, int nx, int ny, int nz,
                                                          const HeatCoef k) {
    const int ax = nx > 1, ay = ny > 1, az = nz > 1;
    const int wx = ax ? nx - 2 : 1, wy = ay ? ny - 2 : 1, wz = az ? nz - 2 : 1;
    const long long cells = (long long)wx * wy * wz;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < cells;
         t += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(t % wx) + ax, y = (int)((t / wx) % wy) + ay, z = (int)(t / ((long long)wx * wy)) + az;
        const long long sx = nx, sxy = (long long)nx * ny;
        const long long i = z * sxy + y * sx + x;
        const double c = T[i];
        double lap = 0.0;
        bool first = true;
        if (ax) {
            const double d2 = __dsub_rn(__dsub_rn(T[i + 1], c), __dsub_rn(c, T[i - 1]));
            const double tt = __dmul_rn(d2, k.rdx2);
            lap = first ? tt : __dadd_rn(lap, tt);
            first = false;
        }
        if (ay) {
            const double d2 = __dsub_rn(__dsub_rn(T[i + sx], c), __dsub_rn(c, T[i - sx]));
            const double tt = __dmul_rn(d2, k.rdy2);
            lap = first ? tt : __dadd_rn(lap, tt);
            first = false;
        }
        if (az) {
            const double d2 = __dsub_rn(__dsub_rn(T[i + sxy], c), __dsub_rn(c, T[i - sxy]));
            const double tt = __dmul_rn(d2, k.rdz2);
            lap = first ? tt : __dadd_rn(lap, tt);
            first = false;
        }
        T2[i] = __dadd_rn(c, __dmul_rn(k.dt, __dmul_rn(__dmul_rn(k.lam, Ci[i]), lap)));
    }
}

void launch_heat_lowdim(double *T2, const double *T, const double *Ci, const int n[3], const HeatCoef &k,
                        cudaStream_t s) {
    const long long cells = (long long)(n[0] > 1 ? n[0] - 2 : 1) * (n[1] > 1 ? n[1] - 2 : 1) *
                            (n[2] > 1 ? n[2] - 2 : 1);
    if (cells <= 0) return;
    const int blocks = (int)std::min<long long>((cells + 255) / 256, 148LL * 16);
    heat_lowdim_kernel<<<blocks, 256, 0, s>>>(T2, T, Ci, n[0], n[1], n[2], k);
    IGG_CUDA(cudaGetLastError());
}

// ============================================================== binary32 variant
// DESIGN.md reading 24: every operation in binary32 with explicit rounding (no FMA), canonical
// association, reciprocals 1/(d*d) computed in float on the host; size-1 axes drop their term
// (reading 23).  One thread per cell of the updated box, x fastest, a z-chunk of planes per thread
// with the z neighbours in registers.
constexpr int kF32Kc = 16;
__global__ void __launch_bounds__(256) heat_f32_kernel(float *__restrict__ T2, const float *__restrict__ T,
                                                       const float *__restrict__ Ci, int nx, int ny, int nz,
                                                       int x0, int y0, int z0, int wx, int wy, int wz,
                                                       const HeatCoefF k) {
    const int ax = nx > 1, ay = ny > 1, az = nz > 1;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;   // (x, y) flattened: thin x slabs
    if (t >= (long long)wx * wy) return;                                    // keep every lane busy
    const int x = x0 + (int)(t % wx), y = y0 + (int)(t / wx);
    const int zb = z0 + blockIdx.z * kF32Kc, z1 = min(zb + kF32Kc, z0 + wz);
    const long long sx = nx, sxy = (long long)nx * ny;
    long long i = (long long)zb * sxy + (long long)y * sx + x;
    float zm = az ? __ldg(T + i - sxy) : 0.f, c = __ldg(T + i);
    for (int z = zb; z < z1; ++z, i += sxy) {
        const float zp = az ? __ldg(T + i + sxy) : 0.f;
        float lap = 0.f;
        bool first = true;
        if (ax) {
            const float t = __fmul_rn(__fsub_rn(__fsub_rn(__ldg(T + i + 1), c), __fsub_rn(c, __ldg(T + i - 1))), k.rdx2);
            lap = t;
            first = false;
        }
        if (ay) {
            const float t = __fmul_rn(__fsub_rn(__fsub_rn(__ldg(T + i + sx), c), __fsub_rn(c, __ldg(T + i - sx))), k.rdy2);
            lap = first ? t : __fadd_rn(lap, t);
            first = false;
        }
        if (az) {
            const float t = __fmul_rn(__fsub_rn(__fsub_rn(zp, c), __fsub_rn(c, zm)), k.rdz2);
            lap = first ? t : __fadd_rn(lap, t);
        }
        T2[i] = __fadd_rn(c, __fmul_rn(k.dt, __fmul_rn(__fmul_rn(k.lam, __ldg(Ci + i)), lap)));
        zm = c;
        c = zp;
    }
}

// 3-D binary32 grids with 16-B aligned rows: the binary64 cp.async pipeline (heat_box_async_kernel)
// with four floats per lane, so a warp row is again 512 B (128 cells) and every DRAM stream moves
// the same sectors per instruction as the Float64 kernel.  T[z+1] and Ci[z] are fetched D planes
// ahead into a per-thread smem ring; rows y+-1 are L2 hits from the neighbouring warps' streams.
// Box [x0, x0+wx) x [y0, y0+wy) x [z0, z0+wz); x-tiles start at the 512-B boundary below x0.
__device__ __forceinline__ float heat_cell_f(float c, float xm, float xp, float ym, float yp, float zm, float zp,
                                             float ci, const HeatCoefF &k) {
    const float tx = __fmul_rn(__fsub_rn(__fsub_rn(xp, c), __fsub_rn(c, xm)), k.rdx2);
    const float ty = __fmul_rn(__fsub_rn(__fsub_rn(yp, c), __fsub_rn(c, ym)), k.rdy2);
    const float tz = __fmul_rn(__fsub_rn(__fsub_rn(zp, c), __fsub_rn(c, zm)), k.rdz2);
    return __fadd_rn(c, __fmul_rn(k.dt, __fmul_rn(__fmul_rn(k.lam, ci), __fadd_rn(__fadd_rn(tx, ty), tz))));
}
template <int V>   // V floats global -> shared (16 B: L1-bypassing .cg; 8 B: .ca, the only 8-B form)
__device__ __forceinline__ void cp_async_f(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if (V == 4)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
template <int V> struct VecF;
template <> struct VecF<2> { using T = float2; };
template <> struct VecF<4> { using T = float4; };
template <int V>
__device__ __forceinline__ void ldv(float (&r)[V], const float *p) {
    const typename VecF<V>::T v = __ldg(reinterpret_cast<const typename VecF<V>::T *>(p));
    memcpy(r, &v, sizeof(v));
}
// TY warps per CTA (one y row each), D planes of cp.async prefetch, V floats per lane (a warp row is
// 32*V cells), ST streaming stores of T2
template <int TY, int D, int V, bool ST>
__global__ void __launch_bounds__(32 * TY)
    heat_f32_async_kernel(const float *__restrict__ T, const float *__restrict__ Ci, float *__restrict__ T2, int sx,
                          int sy, int x0, int y0, int z0, int wx, int wy, int wz, int ax0, int xtiles, int ytiles,
                          int kc1, int nbig, int kc2, const HeatCoefF k) {
    using VT = typename VecF<V>::T;
    __shared__ VT sT[D][32 * TY], sC[D][32 * TY];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntiles = xtiles * ytiles;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    int zs, ze;
    if (chunk < nbig) {
        zs = z0 + chunk * kc1;
        ze = min(zs + kc1, z0 + wz);
    } else {
        zs = z0 + nbig * kc1 + (chunk - nbig) * kc2;
        ze = min(zs + kc2, z0 + wz);
    }
    const int tx = tile % xtiles, ty = tile / xtiles;
    const int y = y0 + ty * TY + warp;
    if (y >= y0 + wy || zs >= ze) return;            // per-thread pipeline: no CTA barrier
    const int p = ax0 + tx * 32 * V + V * lane;      // cells p..p+V-1 (rows are 16-B aligned: sx % 4 == 0)
    const bool in = p < sx;
    bool w[V], wall = true;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        w[j] = in && p + j >= x0 && p + j < x0 + wx;
        wall = wall && w[j];
    }
    const long long sxy = (long long)sx * sy;
    long long i = (long long)zs * sxy + (long long)y * sx + p;
#pragma unroll
    for (int q = 0; q < D; ++q) {                    // stage q: T[zs+q+1], Ci[zs+q]
        if (in && zs + q < ze) {
            cp_async_f<V>(&sT[q][tid], T + i + (q + 1) * sxy);
            cp_async_f<V>(&sC[q][tid], Ci + i + q * sxy);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    float zm[V] = {}, c[V] = {};
    if (in) {
        ldv<V>(zm, T + i - sxy);
        ldv<V>(c, T + i);
    }
    int slot = 0;
    for (int z = zs; z < ze; ++z, i += sxy) {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        float ym[V] = {}, yp[V] = {}, zp[V], ci[V];
        if (in) {
            ldv<V>(ym, T + i - sx);
            ldv<V>(yp, T + i + sx);
        }
        {
            const VT a = sT[slot][tid], b = sC[slot][tid];
            memcpy(zp, &a, sizeof(a));
            memcpy(ci, &b, sizeof(b));
        }
        float xm = __shfl_up_sync(0xffffffffu, c[V - 1], 1);
        float xp = __shfl_down_sync(0xffffffffu, c[0], 1);
        if (lane == 0 && w[0]) xm = __ldg(T + i - 1);
        if (lane == 31 && w[V - 1]) xp = __ldg(T + i + V);
        float r[V];
#pragma unroll
        for (int j = 0; j < V; ++j)
            r[j] = heat_cell_f(c[j], j == 0 ? xm : c[j - 1], j == V - 1 ? xp : c[j + 1], ym[j], yp[j], zm[j], zp[j],
                               ci[j], k);
        if (wall) {
            VT rv;
            memcpy(&rv, r, sizeof(rv));
            if (ST)   // streaming store: T2 is not re-read this step
                __stcs(reinterpret_cast<VT *>(T2 + i), rv);
            else
                *reinterpret_cast<VT *>(T2 + i) = rv;
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (w[j]) T2[i + j] = r[j];
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            zm[j] = c[j];
            c[j] = zp[j];
        }
        if (in && z + D < ze) {                      // refill this slot with plane z+D
            cp_async_f<V>(&sT[slot][tid], T + i + (D + 1) * sxy);
            cp_async_f<V>(&sC[slot][tid], Ci + i + D * sxy);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        slot = slot + 1 == D ? 0 : slot + 1;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

HeatCoefF heat_coef_f32(float lam, float dt, float dx, float dy, float dz) {
    HeatCoefF k;
    k.lam = lam;
    k.dt = dt;
    k.rdx2 = 1.0f / (dx * dx);   // in float, as the binary32 oracle (reading 24)
    k.rdy2 = 1.0f / (dy * dy);
    k.rdz2 = 1.0f / (dz * dz);
    return k;
}

template <int TY, int D, int V, bool ST>
static void launch_f32_async(float *T2, const float *T, const float *Ci, const int n[3], const int lo[3],
                             const int hi[3], const HeatCoefF &k, cudaStream_t s, int kc1, int kc2) {
    static int occ = -1, nsm = 0;
    if (occ < 0) {
        IGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, heat_f32_async_kernel<TY, D, V, ST>, 32 * TY, 0));
        int dev = 0;
        IGG_CUDA(cudaGetDevice(&dev));
        IGG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    const int wx = hi[0] - lo[0], wy = hi[1] - lo[1], wz = hi[2] - lo[2];
    constexpr int TW = 32 * V;                       // tile width in cells
    const int ax0 = lo[0] & ~(TW - 1);
    const int xtiles = (hi[0] - ax0 + TW - 1) / TW, ytiles = (wy + TY - 1) / TY, ntiles = xtiles * ytiles;
    // z-chunks of kc1 planes; about two waves' worth of tile-planes at the end in kc2-plane chunks
    const long long conc = (long long)occ * nsm;
    int small = (int)((2 * conc * kc2 + ntiles - 1) / ntiles);
    small = std::min(((small + kc2 - 1) / kc2) * kc2, wz);
    const int nbig = (wz - small) / kc1;             // whole big chunks only; the rest goes in small ones
    const int nsmall = (wz - nbig * kc1 + kc2 - 1) / kc2;
    heat_f32_async_kernel<TY, D, V, ST><<<(unsigned)((long long)ntiles * (nbig + nsmall)), 32 * TY, 0, s>>>(
        T, Ci, T2, n[0], n[1], lo[0], lo[1], lo[2], wx, wy, wz, ax0, xtiles, ytiles, kc1, nbig, kc2, k);
    IGG_CUDA(cudaGetLastError());
}

// variant (IGG_OPT_STENCIL_KERNEL): 0 = default (TY 4, D 2, float4 lanes, streaming stores, z-chunks 48
// with an 8-plane tail: the measured best, profiles/r01_f32_variant_sweep.txt); 100.. = ablations;
// 1 = the scalar kernel
void launch_heat_f32(float *T2, const float *T, const float *Ci, const int n[3], const int lo[3], const int hi[3],
                     const HeatCoefF &k, cudaStream_t s, int variant) {
    const int wx = hi[0] - lo[0], wy = hi[1] - lo[1], wz = hi[2] - lo[2];
    if (wx <= 0 || wy <= 0 || wz <= 0) return;
    const bool aligned = n[0] % 4 == 0 && (((uintptr_t)T | (uintptr_t)T2 | (uintptr_t)Ci) & 15) == 0;
    if (n[0] > 1 && n[1] > 1 && n[2] > 1 && aligned && wx >= 64 && variant != 1) {
        switch (variant) {
#if IGG_ABLATION
            case 101: launch_f32_async<8, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 102: launch_f32_async<4, 4, 4, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 103: launch_f32_async<4, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 104: launch_f32_async<4, 3, 4, false>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 105: launch_f32_async<4, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 128, 16); break;
            case 106: launch_f32_async<4, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 32, 8); break;
            case 107: launch_f32_async<4, 3, 2, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 108: launch_f32_async<8, 3, 2, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 109: launch_f32_async<4, 4, 2, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 110: launch_f32_async<8, 4, 4, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 111: launch_f32_async<2, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;
            case 112: launch_f32_async<4, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 64, 4); break;
            case 113: launch_f32_async<4, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 32, 8); break;
            case 114: launch_f32_async<4, 4, 4, true>(T2, T, Ci, n, lo, hi, k, s, 32, 8); break;
            case 115: launch_f32_async<4, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 48, 8); break;
            case 116: launch_f32_async<4, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 24, 8); break;
            case 117: launch_f32_async<4, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 16, 8); break;
            case 118: launch_f32_async<2, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 32, 8); break;
            case 119: launch_f32_async<4, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 40, 8); break;
            case 120: launch_f32_async<4, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 56, 8); break;
            case 121: launch_f32_async<4, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 48, 4); break;
            case 122: launch_f32_async<4, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 48, 16); break;
            case 123: launch_f32_async<8, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 48, 8); break;
            case 124: launch_f32_async<4, 1, 4, true>(T2, T, Ci, n, lo, hi, k, s, 48, 8); break;
            case 125: launch_f32_async<4, 2, 4, false>(T2, T, Ci, n, lo, hi, k, s, 48, 8); break;
            case 126: launch_f32_async<4, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 48, 8); break;
            case 100: launch_f32_async<4, 3, 4, true>(T2, T, Ci, n, lo, hi, k, s, 64, 8); break;   // = f64 default
#endif
            default: launch_f32_async<4, 2, 4, true>(T2, T, Ci, n, lo, hi, k, s, 48, 8); break;   // 0 = 115
        }
        return;
    }
    const dim3 grid((unsigned)(((long long)wx * wy + 255) / 256), 1, (wz + kF32Kc - 1) / kF32Kc);
    heat_f32_kernel<<<grid, 256, 0, s>>>(T2, T, Ci, n[0], n[1], n[2], lo[0], lo[1], lo[2], wx, wy, wz, k);
    IGG_CUDA(cudaGetLastError());
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

// ============================================================== vectorised slab kernel
// Boundary slabs of hide_communication are thin (x-slabs 15 cells wide, y/z
// slabs one layer): a warp is split into 32/lx row segments of lx lanes
// (2 cells per lane, 16-B loads/stores), 4 warps per CTA, short z-chunks for
// parallelism (the slabs are latency-bound, they sit on the comm critical path).
constexpr int kSlabWarps = 4;

__global__ void __launch_bounds__(32 * kSlabWarps) heat_slabs_kernel(const __grid_constant__ HeatRegionList L) {
    const int b = blockIdx.x;
    int ri = 0;
    while (ri + 1 < L.n && b >= L.r[ri + 1].block_begin) ++ri;
    const HeatRegion &R = L.r[ri];
    const int local = b - R.block_begin;
    const int tx = local % R.xtiles;
    const int rest = local / R.xtiles;
    const int ty = rest % R.ytiles, tz = rest / R.ytiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = R.lx, rpw = 32 / lx;
    const int seg = lane / lx, l = lane % lx;
    const int yw = R.y0 + (ty * kSlabWarps + warp) * rpw;
    if (yw >= R.y0 + R.wy) return;                    // whole warp out
    const int y = yw + seg;
    const int p = R.ax0 + tx * 2 * lx + 2 * l;
    const bool pair_in = y < R.y0 + R.wy && p < R.sx;
    const bool w0 = pair_in && p >= R.x0 && p < R.x0 + R.wx;
    const bool w1 = pair_in && p + 1 >= R.x0 && p + 1 < R.x0 + R.wx;
    int z = R.z0 + tz * R.kc;
    const int zend = min(R.z0 + R.wz, z + R.kc);
    const long long sx = R.sx, sxy = (long long)R.sx * R.sy;
    const double *__restrict__ T = R.T;
    const double *__restrict__ Ci = R.Ci;
    double *__restrict__ T2 = R.T2;
    long long i = (long long)z * sxy + (long long)y * sx + p;
    const double2 zero2 = make_double2(0.0, 0.0);
    double2 zm = zero2, c = zero2;
    if (pair_in) {
        zm = __ldg(reinterpret_cast<const double2 *>(T + i - sxy));
        c = __ldg(reinterpret_cast<const double2 *>(T + i));
    }
    for (; z < zend; ++z, i += sxy) {
        double2 zp = zero2, ym = zero2, yp = zero2, ci = zero2;
        if (pair_in) {
            zp = __ldg(reinterpret_cast<const double2 *>(T + i + sxy));
            ym = __ldg(reinterpret_cast<const double2 *>(T + i - sx));
            yp = __ldg(reinterpret_cast<const double2 *>(T + i + sx));
            ci = __ldg(reinterpret_cast<const double2 *>(Ci + i));
        }
        double xm = __shfl_up_sync(0xffffffffu, c.y, 1, lx);
        double xp = __shfl_down_sync(0xffffffffu, c.x, 1, lx);
        if (l == 0 && w0) xm = __ldg(T + i - 1);
        if (l == lx - 1 && w1) xp = __ldg(T + i + 2);
        const double r0 = heat_cell(c.x, xm, c.y, ym.x, yp.x, zm.x, zp.x, ci.x, L.k);
        const double r1 = heat_cell(c.y, c.x, xp, ym.y, yp.y, zm.y, zp.y, ci.y, L.k);
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

void launch_heat_slabs(HeatRegionList &L, cudaStream_t s) {
    bool vec = true;
    for (int r = 0; r < L.n; ++r) vec = vec && heat_box_vectorizable(L.r[r]);
    if (!vec) {
        launch_heat_regions(L, s);
        return;
    }
    int total = 0;
    for (int r = 0; r < L.n; ++r) {
        HeatRegion &R = L.r[r];
        R.ax0 = R.x0 & ~1;
        const int span = R.x0 + R.wx - R.ax0;   // cells from the aligned start
        R.lx = 1;   // lanes per row segment: the smallest power of two covering the span
        while (R.lx < 32 && 2 * R.lx < span) R.lx *= 2;
        const int rows = kSlabWarps * (32 / R.lx);
        R.kc = R.wz <= 2 ? R.wz : 4;
        R.xtiles = (span + 2 * R.lx - 1) / (2 * R.lx);
        R.ytiles = (R.wy + rows - 1) / rows;
        R.zchunks = (R.wz + R.kc - 1) / R.kc;
        R.block_begin = total;
        total += R.xtiles * R.ytiles * R.zchunks;
    }
    L.total_blocks = total;
    if (total == 0) return;
    heat_slabs_kernel<<<total, 32 * kSlabWarps, 0, s>>>(L);
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
__device__ __forceinline__ double2 ldg2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }

#if IGG_ABLATION
// TY rows per CTA (one warp per row), KC planes per z-sweep.  With PF the
// loads of plane z+1 (T[z+2], T[z+1] rows y+-1, Ci[z+1]) are issued before
// plane z is computed, so every thread keeps two planes of DRAM reads in
// flight (the kernel is bound by HBM latency x bytes in flight, not by issue;
// see profiles/).
template <int TY, int KC, bool PF>
__global__ void __launch_bounds__(32 * TY, (PF ? 1024 : 1280) / (32 * TY))
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
    const int y = y0 + ty * TY + warp;
    if (y >= y0 + wy) return;                       // whole warp leaves together
    const int p = ax0 + tx * 64 + 2 * lane;          // first of my two cells
    const int xend = x0 + wx;
    const bool pair_in = p < sx;                     // sx even: p+1 < sx too
    const bool w0 = pair_in && p >= x0 && p < xend;
    const bool w1 = pair_in && p + 1 >= x0 && p + 1 < xend;
    int z = z0 + tz * KC;
    const int zend = min(z0 + wz, z + KC);
    const long long sxy = (long long)sx * sy;
    long long i = (long long)z * sxy + (long long)y * sx + p;   // even -> 16-B aligned
    const double2 zero2 = make_double2(0.0, 0.0);
    double2 zm = zero2, c = zero2, zp = zero2, ym = zero2, yp = zero2, ci = zero2;
    if (pair_in) {
        zm = ldg2(T + i - sxy);
        c = ldg2(T + i);
        if (PF) {
            zp = ldg2(T + i + sxy);
            ym = ldg2(T + i - sx);
            yp = ldg2(T + i + sx);
            ci = ldg2(Ci + i);
        }
    }
    for (; z < zend; ++z, i += sxy) {
        double2 zpn = zero2, ymn = zero2, ypn = zero2, cin = zero2;
        if (PF) {   // prefetch plane z+1 (z+2 <= sz-1 always holds inside a region)
            if (pair_in && z + 1 < zend) {
                zpn = ldg2(T + i + 2 * sxy);
                ymn = ldg2(T + i + sxy - sx);
                ypn = ldg2(T + i + sxy + sx);
                cin = ldg2(Ci + i + sxy);
            }
        } else if (pair_in) {
            zp = ldg2(T + i + sxy);
            ym = ldg2(T + i - sx);
            yp = ldg2(T + i + sx);
            ci = ldg2(Ci + i);
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
        if (PF) {
            zp = zpn;
            ym = ymn;
            yp = ypn;
            ci = cin;
        }
    }
}

template <int TY, int KC, bool PF>
static void launch_box_variant(const HeatRegion &r, const HeatCoef &k, cudaStream_t s) {
    const int ax0 = r.x0 & ~63;   // 512-B aligned row segments (the region start is masked)
    const int xtiles = (r.x0 + r.wx - ax0 + 63) / 64;
    const int ytiles = (r.wy + TY - 1) / TY;
    const int ztiles = (r.wz + KC - 1) / KC;
    const long long blocks = (long long)xtiles * ytiles * ztiles;
    heat_box_kernel<TY, KC, PF><<<(unsigned)blocks, 32 * TY, 0, s>>>(r.T, r.Ci, r.T2, r.sx, r.sy, r.x0, r.y0, r.z0,
                                                                      r.wx, r.wy, r.wz, ax0, xtiles, ytiles, k);
    IGG_CUDA(cudaGetLastError());
}

#endif  // IGG_ABLATION

bool heat_box_vectorizable(const HeatRegion &r) {
    return (r.sx % 2 == 0) && ((reinterpret_cast<uintptr_t>(r.T) | reinterpret_cast<uintptr_t>(r.Ci) |
                                reinterpret_cast<uintptr_t>(r.T2)) % 16 == 0);
}

// ------------------------------------------------------------- cp.async z-pipeline
// Same tile and arithmetic as heat_box_kernel, but the two DRAM streams of a
// plane (T[z+1] of my row, Ci[z]) are fetched D planes ahead with cp.async
// (LDGSTS, L1-bypassing) into a per-thread smem ring, so the bytes in flight
// per SM are set by D and the smem ring, not by registers.  Rows y+-1 of
// plane z were fetched by the neighbouring warps' pipelines and are L2 hits.
// Grid: x-tiles fastest, then y-tiles, then z-chunks; the last z-range is cut
// into short chunks (kc2) so the final wave's tail is short.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

#ifdef BOX_MINB   // (ablation builds: minimum resident blocks per SM, i.e. a register cap)
#define BOX_BOUNDS(t) __launch_bounds__(t, BOX_MINB)
#else
#define BOX_BOUNDS(t) __launch_bounds__(t)
#endif
template <int TY, int D, bool ST>
__global__ void BOX_BOUNDS(32 * TY)
    heat_box_async_kernel(const double *__restrict__ T, const double *__restrict__ Ci, double *__restrict__ T2,
                          int sx, int sy, int x0, int y0, int z0, int wx, int wy, int wz, int ax0, int xtiles,
                          int ytiles, int kc1, int nbig, int kc2, const HeatCoef k) {
    extern __shared__ double2 ring[];   // [D][blockDim] T rows, then [D][blockDim] Ci rows
    const int tid = threadIdx.x, bd = blockDim.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int ntiles = xtiles * ytiles;
    const int tile = blockIdx.x % ntiles;
    const int chunk = blockIdx.x / ntiles;
    int zs, ze;
    if (chunk < nbig) {
        zs = z0 + chunk * kc1;
        ze = min(zs + kc1, z0 + wz);
    } else {
        zs = z0 + nbig * kc1 + (chunk - nbig) * kc2;
        ze = min(zs + kc2, z0 + wz);
    }
    const int tx = tile % xtiles, ty = tile / xtiles;
    const int y = y0 + ty * TY + warp;
    if (y >= y0 + wy || zs >= ze) return;            // per-thread pipeline: no CTA barrier is used
    const int p = ax0 + tx * 64 + 2 * lane;
    const int xend = x0 + wx;
    const bool pair_in = p < sx;
    const bool w0 = pair_in && p >= x0 && p < xend;
    const bool w1 = pair_in && p + 1 >= x0 && p + 1 < xend;
    const long long sxy = (long long)sx * sy;
    long long i = (long long)zs * sxy + (long long)y * sx + p;
    double2 *sT = ring, *sC = ring + D * bd;
#pragma unroll
    for (int q = 0; q < D; ++q) {                    // stage q: T[zs+q+1], Ci[zs+q]
        if (pair_in && zs + q < ze) {
            cp_async16(&sT[q * bd + tid], T + i + (q + 1) * sxy);
            cp_async16(&sC[q * bd + tid], Ci + i + q * sxy);
        }
        cp_async_commit();
    }
    const double2 zero2 = make_double2(0.0, 0.0);
    double2 zm = pair_in ? ldg2(T + i - sxy) : zero2;
    double2 c = pair_in ? ldg2(T + i) : zero2;
    int slot = 0;
    for (int z = zs; z < ze; ++z, i += sxy) {
        cp_async_wait<D - 1>();
        double2 ym = zero2, yp = zero2;
        if (pair_in) {
            ym = ldg2(T + i - sx);
            yp = ldg2(T + i + sx);
        }
        const double2 zp = sT[slot * bd + tid];
        const double2 ci = sC[slot * bd + tid];
        double xm = __shfl_up_sync(0xffffffffu, c.y, 1);
        double xp = __shfl_down_sync(0xffffffffu, c.x, 1);
        if (lane == 0 && w0) xm = __ldg(T + i - 1);
        if (lane == 31 && w1) xp = __ldg(T + i + 2);
        const double r0 = heat_cell(c.x, xm, c.y, ym.x, yp.x, zm.x, zp.x, ci.x, k);
        const double r1 = heat_cell(c.y, c.x, xp, ym.y, yp.y, zm.y, zp.y, ci.y, k);
        if (w0 && w1) {
            if (ST)   // streaming store: T2 is not re-read in this step, keep L2 for T rows
                __stcs(reinterpret_cast<double2 *>(T2 + i), make_double2(r0, r1));
            else
                *reinterpret_cast<double2 *>(T2 + i) = make_double2(r0, r1);
        } else {
            if (w0) T2[i] = r0;
            if (w1) T2[i + 1] = r1;
        }
        zm = c;
        c = zp;
        // refill this slot with plane z+D (its values were consumed above)
        if (pair_in && z + D < ze) {
            cp_async16(&sT[slot * bd + tid], T + i + (D + 1) * sxy);
            cp_async16(&sC[slot * bd + tid], Ci + i + D * sxy);
        }
        cp_async_commit();
        slot = slot + 1 == D ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

template <int TY, int D, bool ST = false>
static void launch_box_async(const HeatRegion &r, const HeatCoef &k, cudaStream_t s, int kc1, int kc2) {
    const int ax0 = r.x0 & ~63;   // 512-B aligned row segments (the region start is masked)
    const int xtiles = (r.x0 + r.wx - ax0 + 63) / 64;
    const int ytiles = (r.wy + TY - 1) / TY;
    const int ntiles = xtiles * ytiles;
    const size_t smem = 2 * D * 32 * TY * sizeof(double2);
    static int occ = -1, nsm = 0;
    if (occ < 0) {
        if (smem > 48 * 1024)
            IGG_CUDA(cudaFuncSetAttribute(heat_box_async_kernel<TY, D, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        IGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, heat_box_async_kernel<TY, D, ST>, 32 * TY, smem));
        int dev = 0;
        IGG_CUDA(cudaGetDevice(&dev));
        IGG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    // tail: about two waves' worth of tile-planes at the end go in short chunks
    int small = 0;
    if (kc2 > 0 && kc2 < kc1) {
        const long long conc = (long long)occ * nsm;
        small = (int)((2 * conc * kc2 + ntiles - 1) / ntiles);
        small = ((small + kc2 - 1) / kc2) * kc2;
        if (small > r.wz) small = r.wz;
    }
    const int big = r.wz - small;
    const int nbig = (big + kc1 - 1) / kc1;
    // a partial last big chunk would overlap the small range: shrink the big range to whole chunks
    const int big_planes = nbig * kc1 > big ? (nbig - 1) * kc1 : big;
    const int nbig2 = big_planes / kc1;
    const int rest = r.wz - nbig2 * kc1;
    const int nsmall = kc2 > 0 ? (rest + kc2 - 1) / kc2 : 0;
    const long long blocks = (long long)ntiles * (nbig2 + nsmall);
    heat_box_async_kernel<TY, D, ST><<<(unsigned)blocks, 32 * TY, smem, s>>>(
        r.T, r.Ci, r.T2, r.sx, r.sy, r.x0, r.y0, r.z0, r.wx, r.wy, r.wz, ax0, xtiles, ytiles, kc1, nbig2,
        kc2 > 0 ? kc2 : kc1, k);
    IGG_CUDA(cudaGetLastError());
}

#if IGG_ABLATION
// ------------------------------------------------------------- wide tiles (ablation)
// heat_box_async_kernel with WX warps side by side along x (tile (64*WX) x TY):
// a CTA streams whole 4-KB rows when WX = 8 (DRAM page locality experiment).
template <int WX, int TY, int D>
__global__ void __launch_bounds__(32 * WX * TY)
    heat_box_wide_kernel(const double *__restrict__ T, const double *__restrict__ Ci, double *__restrict__ T2,
                         int sx, int sy, int x0, int y0, int z0, int wx, int wy, int wz, int ax0, int xtiles,
                         int ytiles, int kc1, int nbig, int kc2, const HeatCoef k) {
    constexpr int NT = 32 * WX * TY;
    __shared__ double2 sT[D][NT];
    __shared__ double2 sC[D][NT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wxi = warp % WX, wyi = warp / WX;
    const int ntiles = xtiles * ytiles;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    int zs, ze;
    if (chunk < nbig) {
        zs = z0 + chunk * kc1;
        ze = min(zs + kc1, z0 + wz);
    } else {
        zs = z0 + nbig * kc1 + (chunk - nbig) * kc2;
        ze = min(zs + kc2, z0 + wz);
    }
    const int tx = tile % xtiles, ty = tile / xtiles;
    const int y = y0 + ty * TY + wyi;
    if (y >= y0 + wy || zs >= ze) return;
    const int p = ax0 + (tx * WX + wxi) * 64 + 2 * lane;
    const int xend = x0 + wx;
    const bool pair_in = p < sx;
    const bool w0 = pair_in && p >= x0 && p < xend;
    const bool w1 = pair_in && p + 1 >= x0 && p + 1 < xend;
    const long long sxy = (long long)sx * sy;
    long long i = (long long)zs * sxy + (long long)y * sx + p;
#pragma unroll
    for (int q = 0; q < D; ++q) {
        if (pair_in && zs + q < ze) {
            cp_async16(&sT[q][tid], T + i + (q + 1) * sxy);
            cp_async16(&sC[q][tid], Ci + i + q * sxy);
        }
        cp_async_commit();
    }
    const double2 zero2 = make_double2(0.0, 0.0);
    double2 zm = pair_in ? ldg2(T + i - sxy) : zero2;
    double2 c = pair_in ? ldg2(T + i) : zero2;
    int slot = 0;
    for (int z = zs; z < ze; ++z, i += sxy) {
        cp_async_wait<D - 1>();
        double2 ym = zero2, yp = zero2;
        if (pair_in) {
            ym = ldg2(T + i - sx);
            yp = ldg2(T + i + sx);
        }
        const double2 zp = sT[slot][tid];
        const double2 ci = sC[slot][tid];
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
        if (pair_in && z + D < ze) {
            cp_async16(&sT[slot][tid], T + i + (D + 1) * sxy);
            cp_async16(&sC[slot][tid], Ci + i + D * sxy);
        }
        cp_async_commit();
        slot = slot + 1 == D ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

template <int WX, int TY, int D>
static void launch_box_wide(const HeatRegion &r, const HeatCoef &k, cudaStream_t s, int kc1, int kc2) {
    const int ax0 = r.x0 & ~63;
    const int xtiles = (r.x0 + r.wx - ax0 + 64 * WX - 1) / (64 * WX);
    const int ytiles = (r.wy + TY - 1) / TY;
    const int ntiles = xtiles * ytiles;
    static int occ = -1, nsm = 0;
    if (occ < 0) {
        IGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, heat_box_wide_kernel<WX, TY, D>, 32 * WX * TY, 0));
        int dev = 0;
        IGG_CUDA(cudaGetDevice(&dev));
        IGG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    const long long conc = (long long)occ * nsm;
    int small = (int)((2 * conc * kc2 + ntiles - 1) / ntiles);
    small = std::min(((small + kc2 - 1) / kc2) * kc2, r.wz);
    const int nbig = (r.wz - small) / kc1;
    const int rest = r.wz - nbig * kc1;
    const long long blocks = (long long)ntiles * (nbig + (rest + kc2 - 1) / kc2);
    heat_box_wide_kernel<WX, TY, D><<<(unsigned)blocks, 32 * WX * TY, 0, s>>>(
        r.T, r.Ci, r.T2, r.sx, r.sy, r.x0, r.y0, r.z0, r.wx, r.wy, r.wz, ax0, xtiles, ytiles, kc1, nbig, kc2, k);
    IGG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------- row-staged pipeline (ablation)
// Like heat_box_async_kernel, but the CTA stages whole planes of its tile --
// T rows y0-1 .. y0+TY and Ci rows y0 .. y0+TY-1 -- with cp.async into a ring
// of D+1 slots, so y neighbours and T[z+1] also come from shared memory (no
// L2 round trip inside the loop).  One CTA barrier per plane.
template <int TY, int D>
__global__ void __launch_bounds__(32 * TY)
    heat_box_rows_kernel(const double *__restrict__ T, const double *__restrict__ Ci, double *__restrict__ T2,
                         int sx, int sy, int x0, int y0, int z0, int wx, int wy, int wz, int ax0, int xtiles,
                         int ytiles, int kc1, int nbig, int kc2, const HeatCoef k) {
    constexpr int S = D + 1;
    constexpr int NT = 32 * TY;
    __shared__ double2 sT[S][TY + 2][32];
    __shared__ double2 sC[S][TY][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntiles = xtiles * ytiles;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    int zs, ze;
    if (chunk < nbig) {
        zs = z0 + chunk * kc1;
        ze = min(zs + kc1, z0 + wz);
    } else {
        zs = z0 + nbig * kc1 + (chunk - nbig) * kc2;
        ze = min(zs + kc2, z0 + wz);
    }
    const int tx = tile % xtiles, ty = tile / xtiles;
    const int ybase = y0 + ty * TY;
    const int y = ybase + warp;
    const int p0 = ax0 + tx * 64;
    const int p = p0 + 2 * lane;
    const bool row_ok = y < y0 + wy;
    const bool pair_in = row_ok && p < sx;
    const int xend = x0 + wx;
    const bool w0 = pair_in && p >= x0 && p < xend;
    const bool w1 = pair_in && p + 1 >= x0 && p + 1 < xend;
    const long long sxy = (long long)sx * sy;
    auto issue = [&](int plane, int slot) {
        const long long pb = (long long)plane * sxy;
        for (int e = tid; e < (TY + 2) * 32; e += NT) {
            const int r = e >> 5, l = e & 31;
            const int yy = ybase - 1 + r, pp = p0 + 2 * l;
            if (yy < sy && pp < sx) cp_async16(&sT[slot][r][l], T + pb + (long long)yy * sx + pp);
        }
        for (int e = tid; e < TY * 32; e += NT) {
            const int r = e >> 5, l = e & 31;
            const int yy = ybase + r, pp = p0 + 2 * l;
            if (yy < sy && pp < sx) cp_async16(&sC[slot][r][l], Ci + pb + (long long)yy * sx + pp);
        }
    };
    // prologue: stages zs .. zs+D-1 (stage q holds plane q)
#pragma unroll
    for (int q = 0; q < D; ++q) {
        if (zs + q <= ze) issue(zs + q, q);
        cp_async_commit();
    }
    const double2 zero2 = make_double2(0.0, 0.0);
    long long i = (long long)zs * sxy + (long long)y * sx + p;
    double2 zm = pair_in ? ldg2(T + i - sxy) : zero2;
    cp_async_wait<D - 1>();   // stage zs landed (its own copies; the barrier publishes them)
    __syncthreads();
    double2 c = sT[0][warp + 1][lane];
    for (int z = zs; z < ze; ++z, i += sxy) {
        const int sl = (z - zs) % S, sn = (z + 1 - zs) % S;
        cp_async_wait<D - 2>();   // stage z+1 landed
        __syncthreads();          // ... for every thread; and everyone finished plane z-1
        if (z + D <= ze) issue(z + D, (z + D - zs) % S);   // into the slot of plane z-1
        cp_async_commit();
        const double2 zp = sT[sn][warp + 1][lane];
        const double2 ym = sT[sl][warp][lane];
        const double2 yp = sT[sl][warp + 2][lane];
        const double2 ci = sC[sl][warp][lane];
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
    cp_async_wait<0>();
}

template <int TY, int D>
static void launch_box_rows(const HeatRegion &r, const HeatCoef &k, cudaStream_t s, int kc1, int kc2) {
    const int ax0 = r.x0 & ~63;
    const int xtiles = (r.x0 + r.wx - ax0 + 63) / 64;
    const int ytiles = (r.wy + TY - 1) / TY;
    const int ntiles = xtiles * ytiles;
    static int occ = -1, nsm = 0;
    if (occ < 0) {
        IGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, heat_box_rows_kernel<TY, D>, 32 * TY, 0));
        int dev = 0;
        IGG_CUDA(cudaGetDevice(&dev));
        IGG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    const long long conc = (long long)occ * nsm;
    int small = (int)((2 * conc * kc2 + ntiles - 1) / ntiles);
    small = std::min(((small + kc2 - 1) / kc2) * kc2, r.wz);
    const int nbig = (r.wz - small) / kc1;
    const int rest = r.wz - nbig * kc1;
    const long long blocks = (long long)ntiles * (nbig + (rest + kc2 - 1) / kc2);
    heat_box_rows_kernel<TY, D><<<(unsigned)blocks, 32 * TY, 0, s>>>(
        r.T, r.Ci, r.T2, r.sx, r.sy, r.x0, r.y0, r.z0, r.wx, r.wy, r.wz, ax0, xtiles, ytiles, kc1, nbig, kc2, k);
    IGG_CUDA(cudaGetLastError());
}

#endif  // IGG_ABLATION

// ------------------------------------------------------------- the production kernel
// heat_box_async_kernel's sweep over a LIST of box regions (one launch for all
// local ranks, or for all six boundary slabs).  TY=4 rows per CTA, D=3 planes
// in flight per thread, streaming stores: the configuration measured best in
// profiles/r01_box_variant_sweep.log.
constexpr int kListTY = 4;
constexpr int kListD = 3;

template <int MINB>
__global__ void __launch_bounds__(32 * kListTY, MINB) heat_box_list_kernel(const __grid_constant__ HeatRegionList L) {
    __shared__ double2 sT[kListD][32 * kListTY];
    __shared__ double2 sC[kListD][32 * kListTY];
    const int b = blockIdx.x;
    int ri = 0;
    while (ri + 1 < L.n && b >= L.r[ri + 1].block_begin) ++ri;
    const HeatRegion &R = L.r[ri];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int ntiles = R.xtiles * R.ytiles;
    const int local = b - R.block_begin;
    const int tile = local % ntiles, chunk = local / ntiles;
    int zs, ze;
    if (chunk < R.nbig) {
        zs = R.z0 + chunk * R.kc;
        ze = min(zs + R.kc, R.z0 + R.wz);
    } else {
        zs = R.z0 + R.nbig * R.kc + (chunk - R.nbig) * R.kc2;
        ze = min(zs + R.kc2, R.z0 + R.wz);
    }
    const int tx = tile % R.xtiles, ty = tile / R.xtiles;
    const int y = R.y0 + ty * kListTY + warp;
    if (y >= R.y0 + R.wy || zs >= ze) return;
    const int p = R.ax0 + tx * 64 + 2 * lane;
    const bool pair_in = p < R.sx;
    const bool w0 = pair_in && p >= R.x0 && p < R.x0 + R.wx;
    const bool w1 = pair_in && p + 1 >= R.x0 && p + 1 < R.x0 + R.wx;
    const long long sx = R.sx, sxy = (long long)R.sx * R.sy;
    const double *__restrict__ T = R.T;
    const double *__restrict__ Ci = R.Ci;
    double *__restrict__ T2 = R.T2;
    long long i = (long long)zs * sxy + (long long)y * sx + p;
#pragma unroll
    for (int q = 0; q < kListD; ++q) {
        if (pair_in && zs + q < ze) {
            cp_async16(&sT[q][tid], T + i + (q + 1) * sxy);
            cp_async16(&sC[q][tid], Ci + i + q * sxy);
        }
        cp_async_commit();
    }
    const double2 zero2 = make_double2(0.0, 0.0);
    double2 zm = pair_in ? ldg2(T + i - sxy) : zero2;
    double2 c = pair_in ? ldg2(T + i) : zero2;
    int slot = 0;
    for (int z = zs; z < ze; ++z, i += sxy) {
        cp_async_wait<kListD - 1>();
        double2 ym = zero2, yp = zero2;
        if (pair_in) {
            ym = ldg2(T + i - sx);
            yp = ldg2(T + i + sx);
        }
        const double2 zp = sT[slot][tid];
        const double2 ci = sC[slot][tid];
        double xm = __shfl_up_sync(0xffffffffu, c.y, 1);
        double xp = __shfl_down_sync(0xffffffffu, c.x, 1);
        if (lane == 0 && w0) xm = __ldg(T + i - 1);
        if (lane == 31 && w1) xp = __ldg(T + i + 2);
        const double r0 = heat_cell(c.x, xm, c.y, ym.x, yp.x, zm.x, zp.x, ci.x, L.k);
        const double r1 = heat_cell(c.y, c.x, xp, ym.y, yp.y, zm.y, zp.y, ci.y, L.k);
        if (w0 && w1) {
            __stcs(reinterpret_cast<double2 *>(T2 + i), make_double2(r0, r1));
        } else {
            if (w0) T2[i] = r0;
            if (w1) T2[i + 1] = r1;
        }
        zm = c;
        c = zp;
        if (pair_in && z + kListD < ze) {
            cp_async16(&sT[slot][tid], T + i + (kListD + 1) * sxy);
            cp_async16(&sC[slot][tid], Ci + i + kListD * sxy);
        }
        cp_async_commit();
        slot = slot + 1 == kListD ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

// variant (IGG_OPT_STENCIL_KERNEL >= 30, ablation): occupancy control by extra dynamic smem
void launch_heat_box_list(HeatRegionList &L, cudaStream_t s, int variant) {
    static int occs[64];
    static bool init = false;
    static int nsm = 0;
    if (!init) {
        for (int &o : occs) o = -1;
        init = true;
    }
#if IGG_ABLATION
    const int vi = variant >= 30 && variant < 40 ? variant - 30 : 0;
#else
    const int vi = 0;
    (void)variant;
#endif
    const size_t extra = (size_t)vi * 4096;   // 0, 4 KB, 8 KB, ...
    auto kern = heat_box_list_kernel<1>;
    int &occ = occs[vi];
    if (occ < 0) {
        IGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kListTY, extra));
        int dev = 0;
        IGG_CUDA(cudaGetDevice(&dev));
        IGG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    const int kc1 = 64, kc2 = 8;
    long long tiles_all = 0;
    for (int r = 0; r < L.n; ++r) {
        HeatRegion &R = L.r[r];
        R.ax0 = R.x0 & ~63;   // 512-B aligned row segments (cells before x0 are read, not written)
        R.xtiles = (R.x0 + R.wx - R.ax0 + 63) / 64;
        R.ytiles = (R.wy + kListTY - 1) / kListTY;
        tiles_all += (long long)R.xtiles * R.ytiles;
    }
    long long total = 0;
    for (int r = 0; r < L.n; ++r) {
        HeatRegion &R = L.r[r];
        const long long ntiles = (long long)R.xtiles * R.ytiles;
        if (R.wx <= 0 || R.wy <= 0 || R.wz <= 0) {
            R.nbig = 0;
            R.kc = kc1;
            R.kc2 = kc2;
            R.block_begin = (int)total;
            continue;
        }
        // the last ~2 waves of tile-planes run as short chunks so the tail is short
        const long long conc = (long long)occ * nsm;
        int small = (int)((2 * conc * kc2 + tiles_all - 1) / tiles_all);
        small = ((small + kc2 - 1) / kc2) * kc2;
        if (small > R.wz) small = R.wz;
        R.nbig = (R.wz - small) / kc1;
        R.kc = kc1;
        R.kc2 = kc2;
        const int rest = R.wz - R.nbig * kc1;
        R.block_begin = (int)total;
        total += ntiles * (R.nbig + (rest + kc2 - 1) / kc2);
    }
    L.total_blocks = (int)total;
    if (total == 0) return;
    kern<<<(unsigned)total, 32 * kListTY, extra, s>>>(L);
    IGG_CUDA(cudaGetLastError());
}

// variant: 0 = default (cp.async pipeline, TY=4, D=3, streaming stores, z-chunks 64 with an
// 8-plane tail); 2..24 = the ablation variants measured in profiles/ (IGG_OPT_STENCIL_KERNEL)
void launch_heat_box(const HeatRegion &r, const HeatCoef &k, cudaStream_t s, int variant) {
    if (r.wx <= 0 || r.wy <= 0 || r.wz <= 0) return;
    switch (variant) {
#if IGG_ABLATION
        case 2: launch_box_variant<8, 32, false>(r, k, s); break;
        case 4: launch_box_variant<8, 64, true>(r, k, s); break;
        case 5: launch_box_variant<16, 32, true>(r, k, s); break;
        case 6: launch_box_variant<4, 32, true>(r, k, s); break;
        case 7: launch_box_variant<8, 16, true>(r, k, s); break;
        case 8: launch_box_variant<4, 64, false>(r, k, s); break;
        case 9: launch_box_variant<16, 64, false>(r, k, s); break;
        case 10: launch_box_async<8, 4>(r, k, s, 64, 8); break;
        case 11: launch_box_async<8, 6>(r, k, s, 64, 8); break;
        case 12: launch_box_async<4, 4>(r, k, s, 64, 8); break;
        case 13: launch_box_async<8, 4>(r, k, s, 128, 16); break;
        case 14: launch_box_async<8, 4>(r, k, s, 32, 32); break;
        case 15: launch_box_async<8, 3>(r, k, s, 64, 8); break;
        case 16: launch_box_variant<4, 64, false>(r, k, s); break;
        case 17: launch_box_async<8, 3, true>(r, k, s, 64, 8); break;
        case 18: launch_box_async<4, 3>(r, k, s, 64, 8); break;
        case 19: launch_box_async<8, 2>(r, k, s, 64, 8); break;
        case 20: launch_box_async<4, 3, true>(r, k, s, 64, 8); break;
        case 21: launch_box_async<8, 3>(r, k, s, 96, 8); break;
        case 22: launch_box_async<16, 3>(r, k, s, 64, 8); break;
        case 23: launch_box_async<8, 3>(r, k, s, 64, 4); break;
        case 24: launch_box_async<8, 3>(r, k, s, 48, 8); break;
        case 25: launch_box_rows<4, 3>(r, k, s, 64, 8); break;
        case 26: launch_box_rows<4, 4>(r, k, s, 64, 8); break;
        case 27: launch_box_rows<8, 3>(r, k, s, 64, 8); break;
        case 28: launch_box_rows<8, 4>(r, k, s, 64, 8); break;
        case 29: launch_box_rows<4, 2>(r, k, s, 64, 8); break;
        case 50: launch_box_wide<8, 1, 3>(r, k, s, 64, 8); break;
        case 51: launch_box_wide<4, 1, 3>(r, k, s, 64, 8); break;
        case 52: launch_box_wide<2, 2, 3>(r, k, s, 64, 8); break;
        case 53: launch_box_wide<8, 1, 4>(r, k, s, 64, 8); break;
        case 54: launch_box_wide<4, 2, 3>(r, k, s, 64, 8); break;
        case 55: launch_box_wide<2, 1, 3>(r, k, s, 64, 8); break;
        case 56: launch_box_wide<1, 4, 3>(r, k, s, 64, 8); break;
        case 3: launch_box_variant<8, 32, true>(r, k, s); break;
#endif
        default: launch_box_async<4, 3, true>(r, k, s, 64, 8); break;   // 0 = 20: the measured best
    }
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

__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys_k() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

constexpr int kCopyThreads = 256;
constexpr int kCopyILP = 8;   // elements per thread, all loads issued before the stores

// Copies of the faces run concurrently with the bandwidth-bound inner box: each
// thread issues kCopyILP independent loads before storing, so a CTA finishes
// in about one memory round trip and holds its SM slot as briefly as possible.
template <bool PACK, typename E>
__device__ __forceinline__ void copy_face_t(const CopyDesc &d) {
    E *field = reinterpret_cast<E *>(d.field);
    E *buf = reinterpret_cast<E *>(d.buf);
    const long long chunk = (long long)kCopyThreads * kCopyILP;
    for (long long base = (long long)blockIdx.x * chunk; base < d.count; base += (long long)gridDim.x * chunk) {
        E v[kCopyILP];
#pragma unroll
        for (int u = 0; u < kCopyILP; ++u) {
            const long long i = base + u * kCopyThreads + threadIdx.x;
            if (i < d.count) v[u] = PACK ? __ldcg(field + face_index(d, i)) : __ldcg(buf + i);
        }
#pragma unroll
        for (int u = 0; u < kCopyILP; ++u) {
            const long long i = base + u * kCopyThreads + threadIdx.x;
            if (i < d.count) {
                if (PACK)
                    buf[i] = v[u];
                else
                    field[face_index(d, i)] = v[u];
            }
        }
    }
}
// binary64 or binary32 elements (a bit copy either way; CTA-uniform branch)
template <bool PACK>
__device__ __forceinline__ void copy_face(const CopyDesc &d) {
    if (d.esz == 4)
        copy_face_t<PACK, float>(d);
    else
        copy_face_t<PACK, double>(d);
}

// pack: field slab -> buffer (own send buffer, a local rank's receive slot, or a
// peer GPU's receive slot over NVLink).  If the list carries signals, the last
// CTA to finish publishes the epoch to the peers' receive flags: the CTA barrier
// orders every thread's stores before thread 0's fence.acq_rel.sys (cumulative),
// the ticket counts the CTA; the last CTA acquires with one more fence and
// stores the flags relaxed (fence + relaxed stores = one release for them all).
template <int N>
__global__ void __launch_bounds__(kCopyThreads) pack_kernel(const __grid_constant__ CopyListT<N> L) {
    const CopyDesc &d = L.d[blockIdx.y];
    copy_face<true>(d);
    if (L.nsignal > 0) {
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_acq_rel_sys_k();
            const unsigned t = atomicAdd(L.ticket, 1u);
            if (t == L.ticket_total - 1) {
                fence_acq_rel_sys_k();
                for (int s = 0; s < L.nsignal; ++s) st_relaxed_sys(L.signal[s], L.epoch);
                atomicExch(L.ticket, 0u);
            }
        }
    }
}

// unpack: buffer -> field receive slab.  A slot filled by a peer GPU is read
// only after its flag reached this call's epoch (bounded spin; a timeout sets
// *err and is reported by igg_check).
template <int N>
__global__ void __launch_bounds__(kCopyThreads) unpack_kernel(const __grid_constant__ CopyListT<N> L) {
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
    copy_face<false>(d);
}

// one CTA waits for every peer flag of this axis (bounded spin), so the
// unpack CTAs that follow never occupy SM slots while the peers are still
// packing (they would starve the concurrent inner-box kernel)
template <int N>
__global__ void flag_wait_kernel(const __grid_constant__ CopyListT<N> L) {
    const int t = threadIdx.x;
    if (t < L.nsignal) {
        const unsigned long long *f = L.wait[t];
        const long long t0 = clock64();
        while (ld_acquire_sys(f) < L.epoch) {
            if (clock64() - t0 > L.timeout_cycles) {
                atomicExch(L.err, 1);
                break;
            }
            __nanosleep(32);
        }
    }
}

static int copy_blocks(const CopyDesc *d, int n) {
    long long mx = 1;
    for (int j = 0; j < n; ++j) mx = d[j].count > mx ? d[j].count : mx;
    long long b = (mx + kCopyThreads * kCopyILP - 1) / (kCopyThreads * kCopyILP);
    if (b < 1) b = 1;
    if (b > 1024) b = 1024;
    return (int)b;
}

template <int N>
static void fill_list(CopyListT<N> &L, const CopyList &proto) {
    L.n = 0;
    L.blocks_per_desc = proto.blocks_per_desc;
    L.nsignal = proto.nsignal;
    for (int q = 0; q < kMaxSignal; ++q) {
        L.signal[q] = proto.signal[q];
        L.wait[q] = proto.wait[q];
    }
    L.ticket = proto.ticket;
    L.ticket_total = proto.ticket_total;
    L.epoch = proto.epoch;
    L.timeout_cycles = proto.timeout_cycles;
    L.err = proto.err;
}

template <int N>
static int launch_copies_n(int op, const std::vector<CopyDesc> &descs, const CopyList &proto, cudaStream_t s) {
    const int n = (int)descs.size();
    // total blocks of all chunks: the pack block that draws the last ticket
    // (necessarily in the last chunk, stream order) publishes the flags
    unsigned total = 0;
    for (int c = 0; c < n; c += N) {
        const int m = std::min(N, n - c);
        total += (unsigned)copy_blocks(descs.data() + c, m) * m;
    }
    int launches = 0;
    const bool waits = op == 1 && proto.nsignal > 0;
    if (waits) {
        CopyListT<N> W;
        fill_list(W, proto);
        flag_wait_kernel<N><<<1, 32, 0, s>>>(W);
        IGG_CUDA(cudaGetLastError());
        ++launches;
    }
    for (int c = 0; c < n; c += N) {
        CopyListT<N> L;
        fill_list(L, proto);
        L.n = std::min(N, n - c);
        for (int j = 0; j < L.n; ++j) {
            L.d[j] = descs[c + j];
            if (waits) L.d[j].flag_slot = -1;   // already waited above
        }
        L.ticket_total = total;
        dim3 grid(copy_blocks(L.d, L.n), L.n);
        if (op == 0)
            pack_kernel<N><<<grid, kCopyThreads, 0, s>>>(L);
        else
            unpack_kernel<N><<<grid, kCopyThreads, 0, s>>>(L);
        IGG_CUDA(cudaGetLastError());
        ++launches;
    }
    return launches;
}

int launch_copies(int op, const std::vector<CopyDesc> &descs, const CopyList &proto, cudaStream_t s) {
    if (descs.empty()) return 0;
    return descs.size() <= (size_t)kSmallCopy ? launch_copies_n<kSmallCopy>(op, descs, proto, s)
                                              : launch_copies_n<kMaxCopy>(op, descs, proto, s);
}


// ============================================================== box pack (gather)
// Copies the sub-box [b0, b1) of a (sx, sy, sz) field into a contiguous buffer, x fastest.
__global__ void __launch_bounds__(256) box_pack_kernel(const double *__restrict__ f, double *__restrict__ out,
                                                       long long sx, long long sy, int x0, int y0, int z0, int nx,
                                                       int ny, int nz) {
    const long long n = (long long)nx * ny * nz;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(t % nx);
        const long long r = t / nx;
        const int y = (int)(r % ny), z = (int)(r / ny);
        out[t] = f[((long long)(z0 + z) * sy + (y0 + y)) * sx + x0 + x];
    }
}

void launch_box_pack(const double *f, double *out, long long sx, long long sy, const int b0[3], const int b1[3],
                     cudaStream_t s) {
    const int nx = b1[0] - b0[0], ny = b1[1] - b0[1], nz = b1[2] - b0[2];
    if (nx <= 0 || ny <= 0 || nz <= 0) return;
    const long long n = (long long)nx * ny * nz;
    const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
    box_pack_kernel<<<blocks, 256, 0, s>>>(f, out, sx, sy, b0[0], b0[1], b0[2], nx, ny, nz);
    IGG_CUDA(cudaGetLastError());
}

// ============================================================== outer layers (T2 = copy(T) where it matters)
// PAPER.md:69 T2 = copy(T): the step writes every inner cell of T2 and update_halo! every halo cell, so only
// the six outer layers (the global-boundary values of Dirichlet-by-initialisation, reading 10, and the
// halo layers before their first exchange) need T's values -- 6 n^2 cells instead of the n^3 copy.
__global__ void __launch_bounds__(256) copy_outer_kernel(double *__restrict__ T2, const double *__restrict__ T, int nx,
                                                         int ny, int nz) {
    const long long fz = (long long)nx * ny, fy = (long long)nx * nz, fx = (long long)ny * nz;
    const long long total = 2 * (fz + fy + fx);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        long long x, y, z, r = t;
        if (r < 2 * fz) {   // planes z = 0, nz-1 (contiguous)
            z = r < fz ? 0 : nz - 1;
            r %= fz;
            x = r % nx;
            y = r / nx;
        } else if ((r -= 2 * fz) < 2 * fy) {   // rows y = 0, ny-1
            y = r < fy ? 0 : ny - 1;
            r %= fy;
            x = r % nx;
            z = r / nx;
        } else {   // columns x = 0, nx-1
            r -= 2 * fy;
            x = r < fx ? 0 : nx - 1;
            r %= fx;
            y = r % ny;
            z = r / ny;
        }
        const long long i = (z * ny + y) * nx + x;
        T2[i] = T[i];
    }
}
void launch_copy_outer(double *T2, const double *T, const int n[3], cudaStream_t s) {
    copy_outer_kernel<<<148 * 4, 256, 0, s>>>(T2, T, n[0], n[1], n[2]);
    IGG_CUDA(cudaGetLastError());
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
