// fused.cu -- the fused hide_communication step: stencil + halo exchange in
// peer memory (IGG_PATH_P2P, one rank per process, every neighbour on another GPU).
//
// The paper hides update_halo! behind the inner-point computation by computing
// boundary slabs first and exchanging while the inner box runs (PAPER.md:75,
// :94).  On B200 the same overlap is done inside ONE stencil
// kernel: its CTAs visit the tiles holding send layers first, and every cell
// of a send layer is stored straight into the receiving GPU's receive slot
// over NVLink as it is computed (the "pack" is fused into the stencil).  Each
// contributing CTA counts itself on a per-face counter after a system-scope
// fence; the CTA completing the count publishes the epoch to the receiver's
// flag (st.release.sys).  Face cells that are not computed by the stencil come
// from a small rim kernel (values that never survive or never change) or are
// forwarded by the unpack of an earlier axis (the fresh edge/corner values the
// dimension-sequential update_halo delivers).  The receiver
// waits per axis (one spinning CTA, then the unpack), x -> y -> z.  The final
// state is bit-identical to {step!; update_halo!(T2)} (tests/test_gpu_multi.py).
#include <algorithm>
#include <array>
#include <cstring>

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

// face index of a cell on a face normal to axis a.  y- and z-faces: x fastest
// (z*sx + x, y*sx + x); the x-face is stored z fastest (y*sz + z) so
// that a warp sweeping z writes its x-face cells as contiguous 256-B runs over
// NVLink (sender and receiver of the fused path both use this layout)
__device__ __forceinline__ long long fidx(int a, int x, int y, int z, const int *s) {
    return a == 0 ? (long long)y * s[2] + z : (a == 1 ? (long long)z * s[0] + x : (long long)y * s[0] + x);
}
__device__ __forceinline__ int fast_axis(int a) { return a == 0 ? 2 : 0; }
__device__ __forceinline__ int slow_axis(int a) { return a == 0 ? 1 : (a == 1 ? 2 : 1); }

// publish one contribution to face (a, rs); the completing contribution releases the flag
__device__ __forceinline__ void contribute(const FusedFace &f, unsigned long long epoch) {
    const unsigned old = atomicAdd(f.counter, 1u);
    if (old == f.target - 1) {
        __threadfence_system();
        st_rel_sys(f.flag, epoch);
        atomicExch(f.counter, 0u);
    }
}

// the stores of one cell pair into every send face it belongs to
__device__ __forceinline__ void face_store(const FusedParams &F, int p, int y, int z, bool w0, bool w1, double r0,
                                        double r1) {
    const int sx = F.s[0];
#pragma unroll
    for (int rs = 0; rs < 2; ++rs) {
        const FusedFace &fy = F.face[1][rs];
        if (fy.active && y == fy.layer) {
            if (w0) fy.dst[(long long)z * sx + p] = r0;
            if (w1) fy.dst[(long long)z * sx + p + 1] = r1;
        }
        const FusedFace &fz = F.face[2][rs];
        if (fz.active && z == fz.layer) {
            if (w0) fz.dst[(long long)y * sx + p] = r0;
            if (w1) fz.dst[(long long)y * sx + p + 1] = r1;
        }
    }
}

constexpr int kFTY = 4;   // rows per CTA (one warp each)
constexpr int kFD = 3;    // planes in flight per thread

}  // namespace

// EDGE = true: the tiles holding send layers (launched first, high priority, with the
// fused pack and the per-face counting); EDGE = false: all other tiles, the plain
// pipelined sweep (register budget of the 1-GPU kernel)
template <bool EDGE>
__global__ void __launch_bounds__(32 * kFTY, EDGE ? 8 : 10) heat_fused_kernel(const __grid_constant__ FusedParams F,
                                                                              const int4 *__restrict__ tiles) {
    __shared__ double2 sT[kFD][32 * kFTY];
    __shared__ double2 sC[kFD][32 * kFTY];
    const int4 td = tiles[blockIdx.x];   // (x-tile, y-tile, z0, z1)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sx = F.s[0], sy = F.s[1];
    const int y = 1 + td.y * kFTY + warp;
    const int p = td.x * 64 + 2 * lane;
    const bool pair_in = y < sy - 1 && p < sx;
    const bool w0 = pair_in && p >= 1 && p < sx - 1;
    const bool w1 = pair_in && p + 1 >= 1 && p + 1 < sx - 1;
    const int zs = td.z, ze = td.w;
    const long long sxy = (long long)sx * sy;
    const double *__restrict__ T = F.T;
    const double *__restrict__ Ci = F.Ci;
    double *__restrict__ T2 = F.T2;
    long long i = (long long)zs * sxy + (long long)y * sx + p;
#pragma unroll
    for (int q = 0; q < kFD; ++q) {
        if (pair_in && zs + q < ze) {
            cp_async16f(&sT[q][tid], T + i + (q + 1) * sxy);
            cp_async16f(&sC[q][tid], Ci + i + q * sxy);
        }
        cp_commit();
    }
    const double2 zero2 = make_double2(0.0, 0.0);
    double2 zm = pair_in ? ldg2f(T + i - sxy) : zero2;
    double2 c = pair_in ? ldg2f(T + i) : zero2;
    int slot = 0;
    bool fstore = false;   // this thread holds a cell of a y send layer (EDGE only)
    int zf0 = -1, zf1 = -1;
    // x send layers: the lane holding the layer cell in this warp's row segment (-1: none);
    // its per-plane values are parked one per lane and written as 32-plane runs
    // (fused_eligible requires sx >= 66, so a 64-cell segment holds at most one x send layer)
    int xrs = -1, xoff = 0;
    double xstage = 0.0;
    const int tile_x0 = td.x * 64;
    const bool row_ok = y < sy - 1;
#pragma unroll
    for (int rs = 0; rs < 2 && EDGE; ++rs) {
        const FusedFace &fx = F.face[0][rs], &fy = F.face[1][rs], &fz = F.face[2][rs];
        if (fx.active && row_ok && fx.layer >= tile_x0 && fx.layer < tile_x0 + 64) {
            xrs = rs;
            xoff = fx.layer - tile_x0;   // cell offset in the 64-cell segment
        }
        if (fy.active && pair_in && y == fy.layer) fstore = true;
        if (fz.active) (rs == 0 ? zf0 : zf1) = fz.layer;
    }
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
        if (w0 && w1) {
            __stcs(reinterpret_cast<double2 *>(T2 + i), make_double2(r0, r1));
        } else {
            if (w0) T2[i] = r0;
            if (w1) T2[i + 1] = r1;
        }
        // fused pack: send-layer cells go straight into the receivers' slots
        // (hoisted tests: only threads on an x/y send layer, or the planes of a z send layer)
        if (EDGE && (fstore || z == zf0 || z == zf1)) face_store(F, p, y, z, w0, w1, r0, r1);
        if (EDGE && xrs >= 0) {   // warp-uniform
            const double v = __shfl_sync(0xffffffffu, (xoff & 1) ? r1 : r0, xoff >> 1);
            const int k = (z - zs) & 31;
            if (lane == k) xstage = v;
            if (k == 31 || z == ze - 1) {   // flush a run of k+1 planes: dst[y*sz + zbase + lane]
                if (lane <= k) F.face[0][xrs].dst[(long long)y * F.s[2] + (z - k) + lane] = xstage;
            }
        }
        zm = c;
        c = zp;
        if (pair_in && z + kFD < ze) {
            cp_async16f(&sT[slot][tid], T + i + (kFD + 1) * sxy);
            cp_async16f(&sC[slot][tid], Ci + i + kFD * sxy);
        }
        cp_commit();
        slot = slot + 1 == kFD ? 0 : slot + 1;
    }
    cp_wait<0>();
    if (!EDGE) return;
    // count this CTA on every face whose send layer its tile holds
    unsigned mask = 0;
#pragma unroll
    for (int rs = 0; rs < 2; ++rs) {
        const int lx = F.face[0][rs].layer, ly = F.face[1][rs].layer, lz = F.face[2][rs].layer;
        if (F.face[0][rs].active && lx >= td.x * 64 && lx < td.x * 64 + 64) mask |= 1u << rs;
        if (F.face[1][rs].active && ly >= 1 + td.y * kFTY && ly < 1 + td.y * kFTY + kFTY) mask |= 1u << (2 + rs);
        if (F.face[2][rs].active && lz >= zs && lz < ze) mask |= 1u << (4 + rs);
    }
    if (mask) {
        // only the threads that stored into a peer's slot need their stores ordered
        // before the count (a system fence drains all of a thread's outstanding stores)
        if (fstore || xrs >= 0 || zf0 >= 0 || zf1 >= 0) __threadfence_system();
        __syncthreads();
        if (tid == 0)
            for (int f = 0; f < 6; ++f)
                if (mask & (1u << f)) contribute(F.face[f >> 1][f & 1], F.epoch);
    }
}

// Face cells the stencil does not compute: the send layer's cells on the other
// axes' halo/boundary layers.  Those that an earlier axis' unpack will write
// this step are forwarded by that unpack; all others keep a value that either
// never changes (global boundary) or is overwritten on the receiver by a later
// axis, so the current T2 value is sent.
__device__ __forceinline__ int forward_phase(const FusedParams &F, int a, const int *c) {
    int fwd = -1;
    for (int b = 0; b < a; ++b) {
        if (c[b] == 0 && F.halo[b][0].active) fwd = b;
        if (c[b] == F.s[b] - 1 && F.halo[b][1].active) fwd = b;
    }
    return fwd;
}

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
            if (forward_phase(F, a, c) >= 0) continue;
            const long long gi = ((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0];
            fc.dst[fidx(a, c[0], c[1], c[2], F.s)] = F.T2[gi];
        }
    }
    if (fc.active) __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(ticket, 1u);
        if (t == total - 1) {
            __threadfence_system();
            for (int g = 0; g < 6; ++g)
                if (F.face[g >> 1][g & 1].active) contribute(F.face[g >> 1][g & 1], F.epoch);
            atomicExch(ticket, 0u);
        }
    }
}

// one CTA waits until both receive flags of axis b reached this epoch
__global__ void fused_wait_kernel(const __grid_constant__ FusedParams F, int b) {
    const int side = threadIdx.x;
    if (side < 2 && F.halo[b][side].active) {
        const unsigned long long *fl = F.halo[b][side].flag;
        const long long t0 = clock64();
        while (ld_acq_sys(fl) < F.epoch) {
            if (clock64() - t0 > F.timeout_cycles) {
                atomicExch(F.err, 1);
                break;
            }
            __nanosleep(32);
        }
    }
}

// unpack axis b into T2's halo layers and forward the cells later faces need;
// kUnpackILP values per thread are loaded before any store (latency-bound
// scattered stores: the x halo is one double per row)
constexpr int kUnpackILP = 8;
__global__ void __launch_bounds__(256) fused_unpack_kernel(const __grid_constant__ FusedParams F, int b,
                                                           unsigned int *ticket, unsigned total) {
    const int side = blockIdx.y;
    const FusedHalo &h = F.halo[b][side];
    if (h.active) {
        const int b1 = fast_axis(b), b2 = slow_axis(b);   // slot index = c[b2]*S[b1] + c[b1]
        const int S1 = F.s[b1];
        const long long n = (long long)S1 * F.s[b2];
        bool fwd_any = false;
        for (int a = b + 1; a < 3; ++a) fwd_any |= F.face[a][0].active || F.face[a][1].active;
        const long long chunk = (long long)blockDim.x * kUnpackILP;
        for (long long base = (long long)blockIdx.x * chunk; base < n; base += (long long)gridDim.x * chunk) {
            double v[kUnpackILP];
#pragma unroll
            for (int u = 0; u < kUnpackILP; ++u) {
                const long long t = base + u * blockDim.x + threadIdx.x;
                v[u] = t < n ? __ldcg(h.src + t) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kUnpackILP; ++u) {
                const long long t = base + u * blockDim.x + threadIdx.x;
                if (t >= n) continue;
                int c[3];
                c[b] = h.layer;
                c[b1] = (int)(t % S1);
                c[b2] = (int)(t / S1);
                F.T2[((long long)c[2] * F.s[1] + c[1]) * F.s[0] + c[0]] = v[u];
                if (fwd_any)
                    for (int a = b + 1; a < 3; ++a)
                        for (int rs = 0; rs < 2; ++rs) {
                            const FusedFace &fc = F.face[a][rs];
                            if (fc.active && c[a] == fc.layer && forward_phase(F, a, c) == b)
                                fc.dst[fidx(a, c[0], c[1], c[2], F.s)] = v[u];
                        }
            }
        }
    }
    bool fwd = false;   // forwarded values went to peers: order them before the count
    for (int a = b + 1; a < 3; ++a) fwd |= F.face[a][0].active || F.face[a][1].active;
    if (fwd && h.active) __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(ticket, 1u);
        if (t == total - 1) {
            __threadfence_system();
            for (int a = b + 1; a < 3; ++a)
                for (int rs = 0; rs < 2; ++rs)
                    if (F.face[a][rs].active) contribute(F.face[a][rs], F.epoch);
            atomicExch(ticket, 0u);
        }
    }
}

// ------------------------------------------------------------------ host side
bool fused_eligible(const igg_grid *g) {
    if (g->fused == 2 && g->nlocal == 1) return true;   // ablation/profiling: force the fused kernel
    if (g->path != IGG_PATH_P2P || g->nlocal != 1 || g->nproc_procs < 2 || g->fused == 0) return false;
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 2; ++k) {
            const int nb = g->nbr[0][a][k];
            if (nb >= 0 && proc_of(g, nb) == g->proc) return false;   // self-wrap: stream-ordered path
        }
    for (int a = 0; a < 3; ++a)
        if (g->n[a] < 5) return false;
    if (g->n[0] < 66) return false;   // one x send layer per 64-cell segment
    return true;
}

// tile list: the tiles holding send layers first (x, then y, then z), then the rest;
// z-chunks of 64 planes with the last ~2 waves in 8-plane chunks (short tail)
static void build_tiles(igg_grid *g, const int layer[3][2], const bool act[3][2]) {
    const int n0 = g->n[0], n1 = g->n[1], n2 = g->n[2];
    const int xtiles = (n0 - 1 + 63) / 64;
    const int ytiles = (n1 - 2 + kFTY - 1) / kFTY;
    const int wz = n2 - 2;
    static int occ = -1, nsm = 0;
    if (occ < 0) {
        IGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, heat_fused_kernel<false>, 32 * kFTY, 0));
        IGG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    }
    const int kc1 = 64, kc2 = 8;
    const long long ntile = (long long)xtiles * ytiles;
    int small = (int)((2LL * occ * nsm * kc2 + ntile - 1) / ntile);
    small = std::min(((small + kc2 - 1) / kc2) * kc2, wz);
    const int nbig = (wz - small) / kc1;
    std::vector<std::array<int, 2>> chunks;
    for (int c = 0; c < nbig; ++c) chunks.push_back({1 + c * kc1, 1 + (c + 1) * kc1});
    for (int z = 1 + nbig * kc1; z < 1 + wz; z += kc2) chunks.push_back({z, std::min(z + kc2, 1 + wz)});
    std::vector<int4> edge[3], rest;
    for (const auto &ch : chunks)
        for (int yt = 0; yt < ytiles; ++yt)
            for (int xt = 0; xt < xtiles; ++xt) {
                const int4 t = make_int4(xt, yt, ch[0], ch[1]);
                int cls = -1;
                for (int rs = 0; rs < 2 && cls < 0; ++rs)
                    if (act[0][rs] && layer[0][rs] >= xt * 64 && layer[0][rs] < xt * 64 + 64) cls = 0;
                for (int rs = 0; rs < 2 && cls < 0; ++rs)
                    if (act[1][rs] && layer[1][rs] >= 1 + yt * kFTY && layer[1][rs] < 1 + yt * kFTY + kFTY) cls = 1;
                for (int rs = 0; rs < 2 && cls < 0; ++rs)
                    if (act[2][rs] && layer[2][rs] >= ch[0] && layer[2][rs] < ch[1]) cls = 2;
                (cls >= 0 ? edge[cls] : rest).push_back(t);
                if (cls < 0) {
                    const long long cx = std::min(n0 - 1, xt * 64 + 64) - std::max(1, xt * 64);
                    const long long cy = std::min(n1 - 1, 1 + yt * kFTY + kFTY) - (1 + yt * kFTY);
                    g->fused_rest_cells += cx * cy * (ch[1] - ch[0]);
                }
                for (int a = 0; a < 3; ++a)
                    for (int rs = 0; rs < 2; ++rs) {
                        if (!act[a][rs]) continue;
                        const int L = layer[a][rs];
                        const bool in = a == 0 ? (L >= xt * 64 && L < xt * 64 + 64)
                                                : (a == 1 ? (L >= 1 + yt * kFTY && L < 1 + yt * kFTY + kFTY)
                                                          : (L >= ch[0] && L < ch[1]));
                        if (in) g->fused_tiles_per_face[a][rs]++;
                    }
            }
    std::vector<int4> all;
    for (int a = 0; a < 3; ++a) all.insert(all.end(), edge[a].begin(), edge[a].end());
    g->fused_nedge = (int)all.size();
    all.insert(all.end(), rest.begin(), rest.end());
    if (g->fused_tiles) cudaFree(g->fused_tiles);
    IGG_CUDA(cudaMalloc(&g->fused_tiles, all.size() * sizeof(int4)));
    g->allocs++;
    IGG_CUDA(cudaMemcpy(g->fused_tiles, all.data(), all.size() * sizeof(int4), cudaMemcpyHostToDevice));
    g->fused_ntiles = (int)all.size();
}

void fused_step(igg_grid *g, double *T2, const double *T, const double *Ci, const HeatCoef &k, cudaStream_t s) {
    // buffer pool and slot layout of one canonical field (the same plan update_halo uses)
    const long long sizes[3] = {g->n[0], g->n[1], g->n[2]};
    const Plan plan = build_plan(*g, sizes, 1);
    const size_t half = (size_t)plan.block * sizeof(double);
    ensure_arena(g, half, 0);
    if (!g->fused_ctr) {
        IGG_CUDA(cudaMalloc(&g->fused_ctr, 16 * sizeof(unsigned int)));
        IGG_CUDA(cudaMemset(g->fused_ctr, 0, 16 * sizeof(unsigned int)));
        g->allocs++;
    }
    // receive-slot offsets of (axis, side) within one rank's block (plan order: axis-major, side)
    long long off[3][2];
    {
        long long o = 0;
        for (int a = 0; a < 3; ++a) {
            long long other = 1;
            for (int b = 0; b < 3; ++b)
                if (b != a) other *= sizes[b];
            for (int sd = 0; sd < 2; ++sd) {
                off[a][sd] = o;
                o += other;   // h = 1 for a canonical field with overlap 2
            }
        }
    }
    g->epoch++;
    const int parity = (int)(g->epoch & 1);
    FusedParams F{};
    F.T = T;
    F.Ci = Ci;
    F.T2 = T2;
    for (int a = 0; a < 3; ++a) F.s[a] = g->n[a];
    F.epoch = g->epoch;
    F.timeout_cycles = (long long)(g->spin_timeout_ms * g->clock_khz);
    F.err = g->d_err;
    F.k = k;
    const bool comm = !g->skip_comm;
    int layer[3][2];
    bool act[3][2];
    for (int a = 0; a < 3; ++a)
        for (int rs = 0; rs < 2; ++rs) {
            // rs = receiver side: 0 <- my send_upper (layer n-2) to my upper neighbour,
            //                     1 <- my send_lower (layer 1) to my lower neighbour
            const int nb = g->nbr[0][a][rs == 0 ? 1 : 0];
            layer[a][rs] = rs == 0 ? g->n[a] - 2 : 1;
            act[a][rs] = comm && nb >= 0;
            FusedFace &f = F.face[a][rs];
            f.layer = layer[a][rs];
            f.active = act[a][rs];
            f.counter = g->fused_ctr + a * 2 + rs;
            if (f.active) {
                const int pp = proc_of(g, nb);
                f.dst = reinterpret_cast<double *>(g->peer_recv[pp] + parity * g->recv_half) + off[a][rs];
                f.flag = g->peer_flags[pp] + a * 2 + rs;
            }
            const int hb = g->nbr[0][a][rs];   // my halo side rs is filled by neighbour on side rs
            FusedHalo &h = F.halo[a][rs];
            h.active = comm && hb >= 0;
            h.layer = rs == 0 ? 0 : g->n[a] - 1;
            h.src = reinterpret_cast<const double *>(g->recv_arena + parity * g->recv_half) + off[a][rs];
            h.flag = g->flags + a * 2 + rs;
        }
    // tiles (once per activity pattern)
    int key = 0;
    for (int a = 0; a < 3; ++a)
        for (int rs = 0; rs < 2; ++rs) key |= (act[a][rs] ? 1 : 0) << (a * 2 + rs);
    if (!g->fused_tiles || g->fused_key != key) {
        std::memset(g->fused_tiles_per_face, 0, sizeof g->fused_tiles_per_face);
        g->fused_rest_cells = 0;
        build_tiles(g, layer, act);
        g->fused_key = key;
    }
    bool unpack_axis[3];
    for (int b = 0; b < 3; ++b) unpack_axis[b] = F.halo[b][0].active || F.halo[b][1].active;
    for (int a = 0; a < 3; ++a)
        for (int rs = 0; rs < 2; ++rs) {
            unsigned t = (unsigned)g->fused_tiles_per_face[a][rs] + 1;   // + the rim kernel
            for (int b = 0; b < a; ++b) t += unpack_axis[b] ? 1 : 0;
            F.face[a][rs].target = t;
        }

    IGG_CUDA(cudaEventRecord(g->ev_start, s));
    IGG_CUDA(cudaStreamWaitEvent(g->s_comm, g->ev_start, 0));
    IGG_CUDA(cudaStreamWaitEvent(g->s_inner, g->ev_start, 0));
    tl_mark(g, s, 0);
    // the edge tiles with the fused pack first, high priority; the other tiles concurrently,
    // low priority (they fill the SM slots the edge CTAs leave)
    const int nedge = g->fused_nedge, nrest = g->fused_ntiles - g->fused_nedge;
    if (nedge > 0) {
        heat_fused_kernel<true><<<nedge, 32 * kFTY, 0, g->s_comm>>>(F, g->fused_tiles);
        IGG_CUDA(cudaGetLastError());
        g->launches++;
    }
    tl_mark(g, g->s_comm, 1);   // timeline: my edge tiles (and their face stores) done
    tl_mark(g, g->s_inner, 2);
    prof_begin(g, g->s_inner);
    if (nrest > 0) {
        heat_fused_kernel<false><<<nrest, 32 * kFTY, 0, g->s_inner>>>(F, g->fused_tiles + nedge);
        IGG_CUDA(cudaGetLastError());
        g->launches++;
    }
    prof_end(g, g->s_inner, g->fused_rest_cells);
    tl_mark(g, g->s_inner, 3);
    if (comm) {
        const int rim_blocks = 8;
        fused_rim_kernel<<<dim3(rim_blocks, 6), 256, 0, g->s_comm>>>(F, g->fused_ctr + 8, rim_blocks * 6);
        IGG_CUDA(cudaGetLastError());
        g->launches++;
        for (int b = 0; b < 3; ++b) {
            if (!unpack_axis[b]) continue;
            fused_wait_kernel<<<1, 32, 0, g->s_comm>>>(F, b);
            IGG_CUDA(cudaGetLastError());

            long long other = 1;
            for (int c = 0; c < 3; ++c)
                if (c != b) other *= g->n[c];
            const int blocks = (int)std::min<long long>(std::max<long long>((other + 2047) / 2048, 1), 148);
            fused_unpack_kernel<<<dim3(blocks, 2), 256, 0, g->s_comm>>>(F, b, g->fused_ctr + 9 + b, blocks * 2);
            IGG_CUDA(cudaGetLastError());
            g->launches += 2;
        }
    }
    tl_mark(g, g->s_comm, 4);
    IGG_CUDA(cudaEventRecord(g->ev_comm, g->s_comm));
    IGG_CUDA(cudaEventRecord(g->ev_inner, g->s_inner));
    IGG_CUDA(cudaStreamWaitEvent(s, g->ev_comm, 0));
    IGG_CUDA(cudaStreamWaitEvent(s, g->ev_inner, 0));
}

}  // namespace igg
