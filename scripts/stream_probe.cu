// Streaming probe (diagnostics, not the product): the best 2-read-1-write rate this B200 gives for the
// stencil's data movement (T, Ci in; T2 out: 24 B per cell), by load path:
//   v2   : 16-B LDG (ld.global.nc.v2.f64), grid-stride, 148 x k blocks
//   v4   : 32-B LDG / STG (ld.global.nc.v4.f64, st.global.v4.f64: sm_100's 256-bit accesses)
//   bulk : TMA bulk copies (cp.async.bulk global -> shared, mbarrier completion), 3-stage ring per CTA,
//          one CTA per SM, results stored from registers (16-B STG)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_probe scripts/stream_probe.cu
// Output: one line per variant, GB/s (3 x 8 B x n / median time of 20) and best.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__global__ void add_v2(const double2 *__restrict__ a, const double2 *__restrict__ b, double2 *__restrict__ c, long long n2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
        const double2 x = __ldg(a + i), y = __ldg(b + i);
        __stcs(c + i, make_double2(x.x + y.x, x.y + y.y));
    }
}

struct d4 { double x, y, z, w; };
__device__ __forceinline__ d4 ld4(const double *p) {
    d4 r;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void st4(double *p, d4 v) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}
__global__ void add_v4(const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ c, long long n4) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        const d4 x = ld4(a + 4 * i), y = ld4(b + 4 * i);
        st4(c + 4 * i, d4{x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w});
    }
}

// the acoustic step's pattern: 4 streams read, 4 written (P, Vx, Vy, Vz in; out fields), 8-B per thread
__global__ void rw44(const double *__restrict__ a, const double *__restrict__ b, const double *__restrict__ c,
                     const double *__restrict__ d, double *__restrict__ e, double *__restrict__ f,
                     double *__restrict__ g, double *__restrict__ h, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double x = __ldg(a + i), y = __ldg(b + i), z = __ldg(c + i), w = __ldg(d + i);
        e[i] = x + y; f[i] = y + z; g[i] = z + w; h[i] = w + x;
    }
}
__global__ void rw44v2(const double2 *__restrict__ a, const double2 *__restrict__ b, const double2 *__restrict__ c,
                       const double2 *__restrict__ d, double2 *__restrict__ e, double2 *__restrict__ f,
                       double2 *__restrict__ g, double2 *__restrict__ h, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 x = __ldg(a + i), y = __ldg(b + i), z = __ldg(c + i), w = __ldg(d + i);
        e[i] = make_double2(x.x + y.x, x.y + y.y); f[i] = make_double2(y.x + z.x, y.y + z.y);
        g[i] = make_double2(z.x + w.x, z.y + w.y); h[i] = make_double2(w.x + x.x, w.y + x.y);
    }
}

// TMA bulk: tiles of kT doubles of a and b per stage
constexpr int kT = 2048, kS = 3;
__global__ void __launch_bounds__(256, 1) add_bulk(const double *a, const double *b, double *c, long long ntiles) {
    extern __shared__ __align__(128) unsigned char smem[];
    double *sa = reinterpret_cast<double *>(smem);
    double *sb = sa + kS * kT;
    unsigned long long *bar = reinterpret_cast<unsigned long long *>(sb + kS * kT);
    const int tid = threadIdx.x;
    if (tid == 0)
        for (int s = 0; s < kS; ++s)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    auto issue = [&](long long t, int s) {
        const unsigned bs = (unsigned)__cvta_generic_to_shared(bar + s);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(bs), "r"(2 * kT * 8));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"((unsigned)__cvta_generic_to_shared(sa + s * kT)), "l"(a + t * kT), "r"(kT * 8), "r"(bs) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"((unsigned)__cvta_generic_to_shared(sb + s * kT)), "l"(b + t * kT), "r"(kT * 8), "r"(bs) : "memory");
    };
    const long long first = blockIdx.x, step = gridDim.x;
    if (tid == 0)
        for (int s = 0; s < kS; ++s)
            if (first + s * step < ntiles) issue(first + s * step, s);
    int s = 0;
    unsigned phase = 0;
    for (long long t = first; t < ntiles; t += step) {
        const unsigned bs = (unsigned)__cvta_generic_to_shared(bar + s);
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bs), "r"(phase));
        const double2 *a2 = reinterpret_cast<const double2 *>(sa + s * kT);
        const double2 *b2 = reinterpret_cast<const double2 *>(sb + s * kT);
        double2 *c2 = reinterpret_cast<double2 *>(c + t * kT);
        for (int i = tid; i < kT / 2; i += blockDim.x) {
            const double2 x = a2[i], y = b2[i];
            __stcs(c2 + i, make_double2(x.x + y.x, x.y + y.y));
        }
        __syncthreads();   // stage s consumed
        if (tid == 0 && t + kS * step < ntiles) issue(t + kS * step, s);
        if (++s == kS) { s = 0; phase ^= 1; }
    }
}

template <class F> static void timeit(const char *name, double bytes, F launch) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    std::vector<float> ms;
    for (int r = 0; r < 20; ++r) {
        CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float m; CK(cudaEventElapsedTime(&m, e0, e1)); ms.push_back(m);
    }
    CK(cudaGetLastError());
    std::sort(ms.begin(), ms.end());
    printf("%-28s median %8.1f GB/s  best %8.1f GB/s  (%.4f ms)\n", name, bytes / ms[10] / 1e6, bytes / ms[0] / 1e6, ms[10]);
}

int main() {
    const long long n = 1LL << 27;   // 1 GiB per array (> L2)
    double *a, *b, *c;
    CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8)); CK(cudaMalloc(&c, n * 8));
    CK(cudaMemset(a, 0, n * 8)); CK(cudaMemset(b, 0, n * 8));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const double bytes = 3.0 * 8 * n;
    for (int k : {4, 8, 16})
        for (int bs : {256, 512}) {
            char nm[64]; snprintf(nm, 64, "v2 %dx%d", k, bs);
            timeit(nm, bytes, [&] { add_v2<<<sms * k, bs>>>((const double2 *)a, (const double2 *)b, (double2 *)c, n / 2); });
            snprintf(nm, 64, "v4 %dx%d", k, bs);
            timeit(nm, bytes, [&] { add_v4<<<sms * k, bs>>>(a, b, c, n / 4); });
        }
    const int smem = 2 * kS * kT * 8 + kS * 8;
    CK(cudaFuncSetAttribute(add_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    timeit("bulk 1x256 (TMA, 3 stages)", bytes, [&] { add_bulk<<<sms, 256, smem>>>(a, b, c, n / kT); });
    {   // 4R4W over 8 arrays of 512^3 doubles (the acoustic step's 64 B per cell)
        const long long m = 1LL << 27;
        double *q[8];
        for (int t = 0; t < 8; ++t) { CK(cudaMalloc(&q[t], m * 8)); CK(cudaMemset(q[t], 0, m * 8)); }
        for (int k : {4, 8, 16}) {
            char nm[64]; snprintf(nm, 64, "4R4W 8-B %dx256", k);
            timeit(nm, 64.0 * m, [&] { rw44<<<sms * k, 256>>>(q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7], m); });
            snprintf(nm, 64, "4R4W 16-B %dx256", k);
            timeit(nm, 64.0 * m, [&] { rw44v2<<<sms * k, 256>>>((double2 *)q[0], (double2 *)q[1], (double2 *)q[2], (double2 *)q[3],
                                                             (double2 *)q[4], (double2 *)q[5], (double2 *)q[6], (double2 *)q[7], m / 2); });
        }
        for (int t = 0; t < 8; ++t) CK(cudaFree(q[t]));
    }
    cudaMemcpy(c, a, n * 8, cudaMemcpyDeviceToDevice);
    timeit("cudaMemcpy D2D (2 x 8 B)", 2.0 * 8 * n, [&] { cudaMemcpyAsync(c, a, n * 8, cudaMemcpyDeviceToDevice); });
    printf("sms %d\n", sms);
    return 0;
}
