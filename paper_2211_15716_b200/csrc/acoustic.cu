// acoustic.cu -- the second workload: one leapfrog step of
// linear acoustics on the implicit global staggered grid, the multi-field
// staggered kind of solver the paper scales, written in the
// @inn/@all/@d_xi/@d_xa form of its stencil notation:
//
//   compute_V:  Vx[k,j,i] = Vx[k,j,i] - cVx*(P[k,j,i] - P[k,j,i-1])    (likewise Vy, Vz)
//               on i in [1,nx) and the inner layers [1,n-1) of the other axes
//   update_halo!(Vx, Vy, Vz)                                            (staggered: nx+1 ...)
//   compute_P:  P = P - cP*((((Vx[i+1]-Vx[i])*rx) + ((Vy[j+1]-Vy[j])*ry)) + ((Vz[k+1]-Vz[k])*rz))
//               on every cell (@all)
//
// with cV_d = (dt/rho)/d_d, cP = dt*K, r_d = 1/d_d (reading A2).  Every
// operation is an explicitly rounded binary64 op (no FMA contraction), so the
// result is bit-identical to the oracle (oracle/acoustic3d.py) and to itself
// under any decomposition.
//
// Both kernels are HBM-bound z-sweeps: one thread per x cell, a warp per row
// segment of 32 cells, 4 rows per CTA, a chunk of planes per CTA with the
// z-neighbour in a register queue and the next plane's loads issued one
// iteration ahead.  Algorithmic bytes per cell: compute_V reads P, Vx, Vy, Vz and
// writes Vx, Vy, Vz (56 B); compute_P reads P, Vx, Vy, Vz and writes P (40 B).
#include "igg_internal.h"

namespace igg {
namespace {

constexpr int kAcTY = 4;    // rows per CTA (one warp each)
constexpr int kAcKC = 8;    // planes per CTA (tiling sweep: 8 beats 12/16/32/64/128, profiles/r01_acoustic_tiling_sweep.txt)

__device__ __forceinline__ double ldg(const double *p) { return __ldg(p); }

// V -= c*(p - pm)
__device__ __forceinline__ double vupd(double v, double c, double p, double pm) {
    return __dsub_rn(v, __dmul_rn(c, __dsub_rn(p, pm)));
}

// compute_V on the box [lo, hi) of the velocity cells (x in [1,nx), y in [1,ny), z in [1,nz)):
// component d is written where its own range holds (module comment).
__global__ void __launch_bounds__(32 * kAcTY) acoustic_v_kernel(const __grid_constant__ AcousticFields F,
                                                                const __grid_constant__ AcousticCoef C,
                                                                int3 lo, int3 hi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = lo.x + blockIdx.x * 32 + lane;
    const int j = lo.y + blockIdx.y * kAcTY + warp;
    const int z0 = lo.z + blockIdx.z * kAcKC;
    const int z1 = min(z0 + kAcKC, hi.z);
    if (j >= hi.y) return;   // warp-uniform
    const bool act = i < hi.x;
    const int nx = F.n[0], ny = F.n[1], nz = F.n[2];
    const long long sxyP = (long long)nx * ny;
    const long long sxX = nx + 1, sxyX = (long long)(nx + 1) * ny;
    const long long sxyY = (long long)nx * (ny + 1);
    const bool wx = act && j < ny - 1, wy = act && i < nx - 1, wxy = act && i < nx - 1 && j < ny - 1;
    const double *__restrict__ P = F.P;
    double *__restrict__ Vx = F.Vx;
    double *__restrict__ Vy = F.Vy;
    double *__restrict__ Vz = F.Vz;
    long long ip = (long long)z0 * sxyP + (long long)j * nx + i;   // P, Vz (same x/y strides)
    long long ix = (long long)z0 * sxyX + (long long)j * sxX + i;  // Vx
    long long iy = (long long)z0 * sxyY + (long long)j * nx + i;   // Vy
    double pzm = act ? ldg(P + ip - sxyP) : 0.0;
    // current plane's loads; the next plane's are issued before this plane's math
    double p = 0.0, pym = 0.0, pxm = 0.0, vx = 0.0, vy = 0.0, vz = 0.0;
    if (act && z0 < z1) {
        p = ldg(P + ip);
        pym = ldg(P + ip - nx);
        if (lane == 0) pxm = ldg(P + ip - 1);
        vx = Vx[ix];
        vy = Vy[iy];
        vz = Vz[ip];
    }
    for (int z = z0; z < z1; ++z) {
        const bool more = act && z + 1 < z1;
        double np = 0.0, npym = 0.0, npxm = 0.0, nvx = 0.0, nvy = 0.0, nvz = 0.0;
        if (more) {
            np = ldg(P + ip + sxyP);
            npym = ldg(P + ip + sxyP - nx);
            if (lane == 0) npxm = ldg(P + ip + sxyP - 1);
            nvx = Vx[ix + sxyX];
            nvy = Vy[iy + sxyY];
            nvz = Vz[ip + sxyP];
        }
        double xm = __shfl_up_sync(0xffffffffu, p, 1);
        if (lane == 0) xm = pxm;
        const bool zin = z < nz - 1;
        if (wx && zin) Vx[ix] = vupd(vx, C.cV[0], p, xm);
        if (wy && zin) Vy[iy] = vupd(vy, C.cV[1], p, pym);
        if (wxy) Vz[ip] = vupd(vz, C.cV[2], p, pzm);
        pzm = p;
        p = np;
        pym = npym;
        pxm = npxm;
        vx = nvx;
        vy = nvy;
        vz = nvz;
        ip += sxyP;
        ix += sxyX;
        iy += sxyY;
    }
}

// compute_P on every cell [0,nx) x [0,ny) x [z-chunk)
__global__ void __launch_bounds__(32 * kAcTY) acoustic_p_kernel(const __grid_constant__ AcousticFields F,
                                                                const __grid_constant__ AcousticCoef C) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nx = F.n[0], ny = F.n[1], nz = F.n[2];
    const int i = blockIdx.x * 32 + lane;
    const int j = blockIdx.y * kAcTY + warp;
    const int z0 = blockIdx.z * kAcKC;
    const int z1 = min(z0 + kAcKC, nz);
    if (j >= ny) return;   // warp-uniform
    const bool act = i < nx;
    const bool edge = act && (lane == 31 || i + 1 == nx);   // loads its x+1 face itself
    const long long sxyP = (long long)nx * ny;
    const long long sxX = nx + 1, sxyX = (long long)(nx + 1) * ny;
    const long long sxyY = (long long)nx * (ny + 1);
    double *__restrict__ P = F.P;
    const double *__restrict__ Vx = F.Vx;
    const double *__restrict__ Vy = F.Vy;
    const double *__restrict__ Vz = F.Vz;
    long long ip = (long long)z0 * sxyP + (long long)j * nx + i;
    long long ix = (long long)z0 * sxyX + (long long)j * sxX + i;
    long long iy = (long long)z0 * sxyY + (long long)j * nx + i;
    double vzk = act ? ldg(Vz + ip) : 0.0;
    double p = 0.0, vx = 0.0, vxe = 0.0, vy = 0.0, vyp = 0.0, vzp = 0.0;
    if (act && z0 < z1) {
        p = P[ip];
        vx = ldg(Vx + ix);
        if (edge) vxe = ldg(Vx + ix + 1);
        vy = ldg(Vy + iy);
        vyp = ldg(Vy + iy + nx);
        vzp = ldg(Vz + ip + sxyP);
    }
    for (int z = z0; z < z1; ++z) {
        const bool more = act && z + 1 < z1;
        double np = 0.0, nvx = 0.0, nvxe = 0.0, nvy = 0.0, nvyp = 0.0, nvzp = 0.0;
        if (more) {
            np = P[ip + sxyP];
            nvx = ldg(Vx + ix + sxyX);
            if (edge) nvxe = ldg(Vx + ix + sxyX + 1);
            nvy = ldg(Vy + iy + sxyY);
            nvyp = ldg(Vy + iy + sxyY + nx);
            nvzp = ldg(Vz + ip + 2 * sxyP);
        }
        double vxp = __shfl_down_sync(0xffffffffu, vx, 1);
        if (edge) vxp = vxe;
        if (act) {
            const double div = __dadd_rn(__dadd_rn(__dmul_rn(__dsub_rn(vxp, vx), C.r[0]),
                                                   __dmul_rn(__dsub_rn(vyp, vy), C.r[1])),
                                         __dmul_rn(__dsub_rn(vzp, vzk), C.r[2]));
            P[ip] = __dsub_rn(p, __dmul_rn(C.cP, div));
        }
        vzk = vzp;
        p = np;
        vx = nvx;
        vxe = nvxe;
        vy = nvy;
        vyp = nvyp;
        vzp = nvzp;
        ip += sxyP;
        ix += sxyX;
        iy += sxyY;
    }
}

// ------------------------------------------------------------------ one fused V+P sweep (double-buffered)
// A grid with no exchanged axis (1 GPU, non-periodic): compute_V then compute_P in ONE z-sweep, reading
// the "in" fields and writing every element of the "out" fields -- 64 B per cell (P, Vx, Vy, Vz read once
// and written once) instead of 96 for the two in-place kernels.  Thread = one (i, j) column, lane = i:
// at plane k it computes the new velocities of its cell's lower faces (Vx(i), Vy(j), Vz(k)) from P_in, and
// the new P of plane k-1, whose upper faces are Vx(i+1) (the next lane's, shuffled; the tile's last lane
// computes it itself), Vy(j+1) (computed by this thread too, from P_in and Vy_in of row j+1) and Vz(k)
// (this iteration's).  The same explicitly rounded operations as the two-kernel step: bit-identical
// (tests/test_gpu_acoustic.py).  Boundary faces that compute_V never updates are copied.
__device__ __forceinline__ double pupd(double p, double cP, double r0, double r1, double r2, double vx, double vxp,
                                       double vy, double vyp, double vz, double vzp) {
    const double div = __dadd_rn(__dadd_rn(__dmul_rn(__dsub_rn(vxp, vx), r0), __dmul_rn(__dsub_rn(vyp, vy), r1)),
                                 __dmul_rn(__dsub_rn(vzp, vz), r2));
    return __dsub_rn(p, __dmul_rn(cP, div));
}

#ifndef AF_KC   // (ablation builds sweep these)
#define AF_KC 32
#endif
#ifndef AF_D
#define AF_D 2
#endif
#ifndef AF_TY
#define AF_TY 2
#endif
constexpr int kAfTY = AF_TY;   // rows per CTA (one warp each)
constexpr int kAfKC = AF_KC;   // P planes per CTA
constexpr int kAfD = AF_D;     // planes in flight per thread (cp.async ring)
constexpr int kAfS = 7;     // ring streams: P, Vx, Vy, Vz of my cell; P(j-1), P(j+1), Vy(j+1) of the rows beside

__device__ __forceinline__ void cp8(double *smem, const double *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpcommit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpwait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// the ring entry of plane k: issue the cp.asyncs of my cell's in-field values (nothing past the fields;
// the chunk's closing plane z1 only needs P and Vz: 1.662 vs 1.681 ms per 512^3 step)
__device__ __forceinline__ void af_issue(double (*r)[kAfS], const AcousticFields &I, bool act, int j, int k, int z1,
                                         long long ip, long long ix, long long iy) {
    const int nx = I.n[0], ny = I.n[1], nz = I.n[2];
    if (!act) return;
    cp8(&r[0][3], I.Vz + ip);   // (k <= nz: Vz has nz+1 planes)
    if (k >= nz) return;
    cp8(&r[0][0], I.P + ip);
    if (k == z1) return;
    cp8(&r[0][1], I.Vx + ix);
    cp8(&r[0][2], I.Vy + iy);
    cp8(&r[0][6], I.Vy + iy + nx);
    if (j > 0) cp8(&r[0][4], I.P + ip - nx);
    if (j + 1 < ny) cp8(&r[0][5], I.P + ip + nx);
}

// the sweep of one CTA over planes z0 .. z1 (module comment above).  (A copy specialised for CTAs whose
// columns and planes are all inner -- no range checks, ~25 % fewer instructions -- measured SLOWER,
// 1.93 vs 1.66 ms per 512^3 step: the sweep is not issue-bound.)
#ifdef AF_STCS   // (ablation: streaming stores)
#define AF_ST(p, v) __stcs((p), (v))
#else
#define AF_ST(p, v) (*(p) = (v))
#endif
__device__ __forceinline__ void af_sweep(const AcousticFields &I, const AcousticFields &O, const AcousticCoef &C,
                                         double (*ring)[32 * kAfTY][kAfS], int lane, int tid, int i, int j, int z0,
                                         int z1) {
    const int nx = I.n[0], ny = I.n[1], nz = I.n[2];
    const bool act = i < nx;
    const bool last = act && (lane == 31 || i + 1 == nx);   // computes Vx(i+1) itself
    const long long sxyP = (long long)nx * ny;
    const long long sxX = nx + 1, sxyX = (long long)(nx + 1) * ny;
    const long long sxyY = (long long)nx * (ny + 1);
    // update ranges of compute_V (oracle/acoustic3d.py, acoustic_v_kernel)
    const bool jin = j >= 1 && j < ny - 1, iin = i >= 1 && i < nx - 1;
    const bool ux = act && i >= 1 && jin;          // Vx(i): i in [1, nx), j inner (and k inner)
    const bool uxe = last && i + 1 < nx && jin;  // Vx(i+1)
    const bool uy = act && j >= 1 && iin;          // Vy(j): j in [1, ny), i inner
    const bool uye = act && j + 1 < ny && iin;       // Vy(j+1)
    const bool uz = act && iin && jin;             // Vz(k): k in [1, nz), i, j inner
    long long ip = (long long)z0 * sxyP + (long long)j * nx + i;
    long long ix = (long long)z0 * sxyX + (long long)j * sxX + i;
    long long iy = (long long)z0 * sxyY + (long long)j * nx + i;
#pragma unroll
    for (int q = 0; q < kAfD; ++q) {   // planes z0 .. z0+kAfD-1 (the loop covers z0 .. z1)
        if (z0 + q <= z1)
            af_issue(&ring[q][tid], I, act, j, z0 + q, z1, ip + q * sxyP, ix + q * sxyX, iy + q * sxyY);
        cpcommit();
    }
    double pzm = (act && z0 > 0) ? ldg(I.P + ip - sxyP) : 0.0;   // P_in of plane k-1
    double pp = 0.0, vxn = 0.0, vxpn = 0.0, vyn = 0.0, vypn = 0.0, vzn = 0.0;   // plane k-1's new values
    int slot = 0;
    for (int k = z0; k <= z1; ++k, ip += sxyP, ix += sxyX, iy += sxyY) {
        cpwait<kAfD - 1>();
        const double *e = ring[slot][tid];
        const double cp = e[0], cvz = e[3];
        // refill this slot with plane k+kAfD (after reading it: the entries are this thread's own)
        double cvx = 0.0, cvy = 0.0, cpym = 0.0, cpyp = 0.0, cvyp = 0.0;
        if (k < z1) {
            cvx = e[1];
            cvy = e[2];
            cpym = e[4];
            cpyp = e[5];
            cvyp = e[6];
        }
        double cpxm = 0.0, cvxe = 0.0, cpxp = 0.0;   // (rarely needed: plain loads)
        if (k < z1 && act && k < nz) {
            if (lane == 0 && i > 0) cpxm = ldg(I.P + ip - 1);
            if (last) {
                cvxe = ldg(I.Vx + ix + 1);
                if (i + 1 < nx) cpxp = ldg(I.P + ip + 1);
            }
        }
        if (k + kAfD <= z1)
            af_issue(&ring[slot][tid], I, act, j, k + kAfD, z1, ip + kAfD * sxyP, ix + kAfD * sxyX,
                         iy + kAfD * sxyY);
        cpcommit();
        slot = slot + 1 == kAfD ? 0 : slot + 1;
        // the new Vz(k) of my column (k == nz: the top boundary face, copied)
        const double vz = (uz && k >= 1 && k < nz) ? vupd(cvz, C.cV[2], cp, pzm) : cvz;
        if (act && (k < z1 || k == nz)) AF_ST(O.Vz + ip, vz);   // (the next chunk writes its own first face)
        if (k > z0 && act)   // P of plane k-1: its faces are all new now
            AF_ST(O.P + ip - sxyP, pupd(pp, C.cP, C.r[0], C.r[1], C.r[2], vxn, vxpn, vyn, vypn, vzn, vz));
        if (k == z1) break;
        // plane k: the new Vx(i), Vx(i+1), Vy(j), Vy(j+1) of my cell
        const bool kin = k >= 1 && k < nz - 1;
        double xm = __shfl_up_sync(0xffffffffu, cp, 1);
        if (lane == 0) xm = cpxm;
        const double vx = (ux && kin) ? vupd(cvx, C.cV[0], cp, xm) : cvx;
        const double vy = (uy && kin) ? vupd(cvy, C.cV[1], cp, cpym) : cvy;
        const double vyp = (uye && kin) ? vupd(cvyp, C.cV[1], cpyp, cp) : cvyp;
        double vxp = __shfl_down_sync(0xffffffffu, vx, 1);
        if (last) vxp = (uxe && kin) ? vupd(cvxe, C.cV[0], cpxp, cp) : cvxe;
        if (act) {
            AF_ST(O.Vx + ix, vx);
            AF_ST(O.Vy + iy, vy);
            if (j == ny - 1) O.Vy[iy + nx] = vyp;         // the top boundary row of Vy
            if (last && i + 1 == nx) O.Vx[ix + 1] = vxp;   // the right boundary face of Vx
        }
        pzm = cp;
        pp = cp;
        vxn = vx;
        vxpn = vxp;
        vyn = vy;
        vypn = vyp;
        vzn = vz;
    }
    cpwait<0>();
}

__global__ void __launch_bounds__(32 * kAfTY) acoustic_fused_kernel(const __grid_constant__ AcousticFields I,
                                                                    const __grid_constant__ AcousticFields O,
                                                                    const __grid_constant__ AcousticCoef C) {
    __shared__ double ring[kAfD][32 * kAfTY][kAfS];
#ifdef AF_PAD   // (ablation: fewer CTAs per SM)
    __shared__ char pad[AF_PAD];
    if (threadIdx.x == 1023) pad[blockIdx.x & 7] = 0;
#endif
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const int nx = I.n[0], ny = I.n[1], nz = I.n[2];
    const int i = blockIdx.x * 32 + lane;
    const int j = blockIdx.y * kAfTY + warp;
    const int z0 = blockIdx.z * kAfKC;
    const int z1 = min(z0 + kAfKC, nz);
    if (j >= ny) return;   // warp-uniform (no CTA barrier is used)
    af_sweep(I, O, C, ring, lane, tid, i, j, z0, z1);
}

}  // namespace

void launch_acoustic_fused(const AcousticFields &in, const AcousticFields &out, const AcousticCoef &c, cudaStream_t s) {
    const dim3 grid((in.n[0] + 31) / 32, (in.n[1] + kAfTY - 1) / kAfTY, (in.n[2] + kAfKC - 1) / kAfKC);
    acoustic_fused_kernel<<<grid, 32 * kAfTY, 0, s>>>(in, out, c);
    IGG_CUDA(cudaGetLastError());
}

void launch_acoustic_v(const AcousticFields &f, const AcousticCoef &c, const int lo[3], const int hi[3],
                       cudaStream_t s) {
    const int wx = hi[0] - lo[0], wy = hi[1] - lo[1], wz = hi[2] - lo[2];
    if (wx <= 0 || wy <= 0 || wz <= 0) return;
    const dim3 grid((wx + 31) / 32, (wy + kAcTY - 1) / kAcTY, (wz + kAcKC - 1) / kAcKC);
    acoustic_v_kernel<<<grid, 32 * kAcTY, 0, s>>>(f, c, make_int3(lo[0], lo[1], lo[2]),
                                                  make_int3(hi[0], hi[1], hi[2]));
    IGG_CUDA(cudaGetLastError());
}

void launch_acoustic_p(const AcousticFields &f, const AcousticCoef &c, cudaStream_t s) {
    const dim3 grid((f.n[0] + 31) / 32, (f.n[1] + kAcTY - 1) / kAcTY, (f.n[2] + kAcKC - 1) / kAcKC);
    acoustic_p_kernel<<<grid, 32 * kAcTY, 0, s>>>(f, c);
    IGG_CUDA(cudaGetLastError());
}

}  // namespace igg
