// halo26.cu -- update_halo! on the P2P path as ONE kernel per call.
//
// The paper's update_halo is dimension-sequential (x, then y, then z; each phase over the full extent of
// the other axes, so edges and corners arrive through two or three hops).  On an
// NVSwitch every GPU reaches every other at full bandwidth, so here every halo region is stored ONCE,
// straight from the rank that owns its values, in a single phase ("26-neighbour
// single-phase exchange"): for a receiver m, a halo cell that lies in the receive range of the axes S
// (and nowhere else) takes its value from rank m + dir(S) at the matching send-range index on the axes in
// S and the same index on the others.  That is exactly the value the dimension-sequential exchange leaves
// there (its last writer is the phase of the largest axis in S, which forwards what the earlier phases
// delivered from that same owner), so the result is bit-identical (tests/test_gpu_halo.py,
// tests/test_gpu_virtual_p2p.py, against oracle.halo's dimension-sequential update).
//
// Per call, per hosted rank and field, up to 26 boxes (6 faces, 12 edges, 8 corners).  y/z faces, edges
// and corners are stored directly into the receiver's field (contiguous rows where the layout allows);
// the x faces (one 8-B value per 32-B sector of a column) go z-contiguous into the receiver's slot of the
// receive arena and the receiver's own blocks unpack them once the data flag arrived.  Protocol of epoch e:
//   * ready:  at kernel start each rank release-stores e into the "ready" flag its remote senders hold
//             for it (its halos of e-1 are no longer read: the call is stream-ordered after the work that
//             read them); a store to a remote receiver waits for that receiver's ready(e);
//   * data:   the block that completes the last store chunk (ticket, system fences) release-stores e into
//             every receiver's data flag (one per direction);
//   * unpack: x-face unpack chunks acquire the sender's data flag first;
//   * end:    the last block to leave acquires every incoming data flag, so the halos are complete for any
//             later work on the stream.
// Work is claimed in batches of chunks from a counter, store chunks first: a block only ever waits for (a)
// other GPUs, or (b) store chunks already claimed by running blocks, which never wait on this launch and
// count themselves before their block claims again -- so the launch cannot deadlock whatever the block
// residency (DESIGN.md §6 "forward progress").
#include <algorithm>
#include <cstring>

#include "igg_internal.h"

namespace igg {

namespace {

constexpr int kH26Threads = 256;
constexpr int kH26ILP = 4;
constexpr int kH26Chunk = kH26Threads * kH26ILP;   // elements per work chunk

struct H26Item {
    const char *src;
    char *dst;
    long long ssy, ssz;   // source strides (elements) of y and z
    long long dsy, dsz;   // destination strides
    int bx, by, bz;       // box extent
    int esz;              // bytes per element (8 or 4)
    int wait;             // index into waitp (-1: none): flag that must reach the epoch first
    int remote;           // 1: the destination is another GPU's memory (system-scope release)
    long long chunk0;     // first chunk of this item
    long long cells;
};

struct H26Plan {
    int nitems, nsignal, nready, nwait_end, nwaitp;
    long long nchunks, nstore_chunks;
    // offsets (in bytes from the plan base) of the arrays
    long long o_items, o_signal, o_ready, o_wait_end, o_waitp;
};

__device__ __forceinline__ void st_rel_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// (after a fence.acq_rel: the release pattern without a fence per store)
__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// the PTX release / acquire patterns (fence.acq_rel + relaxed RMW / relaxed RMW + fence.acq_rel) are all the
// protocol needs; __threadfence_system would be the heavier sequentially consistent fence.sc
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acq_gpu_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void spin(const unsigned long long *f, unsigned long long v, long long timeout, int *err) {
    const long long t0 = clock64();
    while (ld_acq_sys(f) < v) {
        if (clock64() - t0 > timeout) {
            atomicExch(err, 1);
            break;
        }
        __nanosleep(64);
    }
}

template <typename E>
__device__ __forceinline__ void copy_chunk(const H26Item &it, long long c) {
    const E *src = reinterpret_cast<const E *>(it.src);
    E *dst = reinterpret_cast<E *>(it.dst);
    const long long base = c * kH26Chunk;
    E v[kH26ILP];
    long long so[kH26ILP], dof[kH26ILP];
#pragma unroll
    for (int u = 0; u < kH26ILP; ++u) {
        const long long l = base + u * kH26Threads + threadIdx.x;
        so[u] = -1;
        if (l < it.cells) {
            const int li = (int)l;
            const int x = li % it.bx, r = li / it.bx, y = r % it.by, z = r / it.by;
            so[u] = z * it.ssz + y * it.ssy + x;
            dof[u] = z * it.dsz + y * it.dsy + x;
            v[u] = __ldcg(src + so[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < kH26ILP; ++u)
        if (so[u] >= 0) dst[dof[u]] = v[u];
}

}  // namespace

constexpr int kH26Batch = 1;   // chunks per claim (small chunks, one per claim: latency, not bandwidth, rules
                               // small halos; a trace of n = 64 showed 2.9 us per chunk in few blocks)
constexpr int kH26SmemItems = 512;   // item starts cached in shared memory (the claim's search)

#ifndef H26_TRACE
#define H26_TRACE 0   // diagnostics build only: per-block %globaltimer stamps of the last launch
#endif
#if H26_TRACE
__device__ unsigned long long g_h26_trace[4096 * 8];
__device__ __forceinline__ unsigned long long h26_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define H26_AT(k) \
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_h26_trace[blockIdx.x * 8 + (k)] = h26_gtimer()
#define H26_VAL(k, v) \
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_h26_trace[blockIdx.x * 8 + (k)] = (v)
#else
#define H26_AT(k)
#define H26_VAL(k, v)
#endif

__global__ void __launch_bounds__(kH26Threads) halo26_kernel(const char *__restrict__ base, unsigned long long epoch,
                                                             unsigned int *ctr, long long timeout, int *err) {
    H26_AT(0);
    const H26Plan &P = *reinterpret_cast<const H26Plan *>(base);
    const H26Item *items = reinterpret_cast<const H26Item *>(base + P.o_items);
    __shared__ long long s_c;
    __shared__ int s_it, s_waited;
    __shared__ long long s_chunk0[kH26SmemItems];
    const bool cached = P.nitems <= kH26SmemItems;
    if (cached)
        for (int q = threadIdx.x; q < P.nitems; q += blockDim.x) s_chunk0[q] = items[q].chunk0;
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x < P.nready) {   // my remote senders may store into me
        unsigned long long *const *ready = reinterpret_cast<unsigned long long *const *>(base + P.o_ready);
        st_rel_sys(ready[threadIdx.x], epoch);
    }
    const long long nbatch = (P.nchunks + kH26Batch - 1) / kH26Batch;
    unsigned mydone = 0;   // store chunks this block finished and has not counted yet
    bool myremote = false;   // some of them went to another GPU: system-scope release, else GPU scope
    // count my finished store chunks (after a system fence); the count completing all store chunks
    // publishes every data flag (release)
    auto flush = [&]() {
        __syncthreads();
        if (threadIdx.x == 0 && mydone) {
            // (release: the block's stores, ordered before thread 0 by the barrier; GPU scope suffices when
            // they all stayed on this GPU -- the completing block's system-scope fence and flag release
            // extend the chain to any receiver)
            if (myremote) fence_acq_rel_sys(); else fence_acq_rel_gpu();
            if (atomicAdd(ctr + 1, mydone) + mydone == (unsigned)P.nstore_chunks) {
                // acquire every other block's release, then ONE release for all the flags: fence.acq_rel +
                // relaxed stores is the PTX release pattern (a st.release per flag would fence per flag:
                // a trace showed ~1.5 us each, 40 us for the 26 flags of a periodic rank)
                fence_acq_rel_sys();
                unsigned long long *const *sig = reinterpret_cast<unsigned long long *const *>(base + P.o_signal);
                for (int q = 0; q < P.nsignal; ++q) st_relaxed_sys(sig[q], epoch);
                atomicExch(ctr + 1, 0u);   // (the last count of this launch: the counter restarts)
            }
        }
        mydone = 0;
        myremote = false;
    };
    long long bt;
    for (;;) {
        if (threadIdx.x == 0) {
            s_c = (long long)atomicAdd(ctr, 1u);
            const long long c0 = s_c * kH26Batch;
            int lo = 0, hi = P.nitems - 1;   // the item holding the batch's first chunk
            if (c0 < P.nchunks)
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if ((cached ? s_chunk0[mid] : items[mid].chunk0) <= c0) lo = mid; else hi = mid - 1;
                }
            s_it = lo;
            s_waited = -1;
        }
        __syncthreads();
        bt = s_c;
        int iti = s_it;
        if (bt >= nbatch) break;
        const long long c0 = bt * kH26Batch, c1 = min(c0 + kH26Batch, P.nchunks);
        for (long long c = c0; c < c1; ++c) {
            // before the first unpack chunk (the only ones that wait on this launch), count my store
            // chunks: claims are monotonic, so no store work follows (block-uniform)
            if (c >= P.nstore_chunks && mydone) flush();
            while (iti + 1 < P.nitems && (cached ? s_chunk0[iti + 1] : items[iti + 1].chunk0) <= c) ++iti;
            const H26Item &it = items[iti];
            if (it.wait >= 0 && s_waited != it.wait) {   // (block-uniform)
                __syncthreads();
                if (threadIdx.x == 0) {
                    const unsigned long long *const *wp =
                        reinterpret_cast<const unsigned long long *const *>(base + P.o_waitp);
                    H26_AT(5);
                    spin(wp[it.wait], epoch, timeout, err);
                    H26_AT(6);
                    s_waited = it.wait;
                }
                __syncthreads();
            }
            if (it.esz == 4)
                copy_chunk<float>(it, c - it.chunk0);
            else
                copy_chunk<double>(it, c - it.chunk0);
            if (c < P.nstore_chunks) {
                ++mydone;
                myremote = myremote || it.remote;
            }
        }
        __syncthreads();   // (s_c / s_it / s_waited are rewritten by the next claim)
        H26_AT(1);
    }
    H26_AT(2);
    flush();
    H26_AT(3);
    if (bt == nbatch + gridDim.x - 1) {   // the last block to leave: every incoming face, then reset
        const unsigned long long *const *we = reinterpret_cast<const unsigned long long *const *>(base + P.o_wait_end);
        for (int q = threadIdx.x; q < P.nwait_end; q += blockDim.x) spin(we[q], epoch, timeout, err);
        // (every block has claimed for the last time: the claim counter restarts for the next launch; the
        // store counter is reset by the block whose count completes it -- some blocks may still be counting
        // here, since the incoming faces can be complete before this launch's own stores are; resetting it
        // here let a late count land in the next launch, whose data flags were then never published)
        if (threadIdx.x == 0) ctr[0] = 0u;
    }
    H26_AT(4);
    H26_VAL(7, (unsigned long long)P.nchunks | ((unsigned long long)P.nstore_chunks << 20) |
                   ((unsigned long long)P.nitems << 40));
}

#if H26_TRACE
}  // namespace igg
IGG_API igg_status igg_debug_h26_trace(unsigned long long *host, int nblocks) {
    IGG_TRY
    IGG_CUDA(cudaDeviceSynchronize());
    IGG_CUDA(cudaMemcpyFromSymbol(host, igg::g_h26_trace, sizeof(unsigned long long) * 8 * std::min(nblocks, 4096)));
    IGG_CATCH
}
namespace igg {
#endif

// ------------------------------------------------------------------ host side
static int dir_index(int ex, int ey, int ez) { return (ex + 1) * 9 + (ey + 1) * 3 + (ez + 1); }

// flags of hosted rank lr of a process hosting L ranks: after the fused path's [2][L][6][kMaxChunks]
static unsigned long long *h26_flag(unsigned long long *flags, int L, int lr, int slot) {
    return flags + (size_t)12 * kMaxChunks * L + (size_t)lr * kH26Flags + slot;
}

void release_h26(igg_grid *g) {
    for (auto &e : g->h26_cache)
        if (e.dplan) cudaFree(e.dplan);
    g->h26_cache.clear();
}

void exchange26(igg_grid *g, const igg_field *fields, int nf, const Plan &plan, cudaStream_t st) {
    const int L = g->nlocal;
    std::vector<long long> key;
    for (int i = 0; i < L * nf; ++i) {
        key.push_back((long long)(uintptr_t)fields[i].ptr);
        for (int a = 0; a < 3; ++a) key.push_back(fields[i].size[a]);
        key.push_back(fields[i].elsize == 4 ? 4 : 8);
    }
    key.push_back((long long)(uintptr_t)g->recv_arena);
    igg_grid::H26Cache *hit = nullptr;
    for (auto &e : g->h26_cache)
        if (e.key == key) hit = &e;
    if (!hit) {
        // ---- build the plan of this process: items, flags
        std::vector<H26Item> store, unpack;
        std::vector<unsigned long long *> signal, ready;
        std::vector<const unsigned long long *> wait_end, waitp;
        auto waitp_index = [&](const unsigned long long *f) {
            for (size_t q = 0; q < waitp.size(); ++q)
                if (waitp[q] == f) return (int)q;
            waitp.push_back(f);
            return (int)waitp.size() - 1;
        };
        auto add_unique = [](auto &v, auto p) {
            if (std::find(v.begin(), v.end(), p) == v.end()) v.push_back(p);
        };
        // peer mappings of every field array (collective, same order on every process)
        std::vector<std::vector<double *>> pmap(L * nf);
        if (g->nproc_procs > 1)
            for (int lr = 0; lr < L; ++lr)
                for (int f = 0; f < nf; ++f) pmap[lr * nf + f] = peer_arrays_pub(g, fields[lr * nf + f].ptr);
        for (int lr = 0; lr < L; ++lr) {
            const int q = g->rank0 + lr;
            int cq[3];
            coords_of_rank(g->dims, q, cq);
            for (int f = 0; f < nf; ++f) {
                const igg_field &F = fields[lr * nf + f];
                const int esz = F.elsize == 4 ? 4 : 8;
                long long s[3];
                HaloSpec hs[3];
                for (int a = 0; a < 3; ++a) {
                    s[a] = F.size[a];
                    halo_spec(g->n[a], g->o[a], s[a], &hs[a]);
                }
                const long long sy = s[0], sz = s[0] * s[1];
                for (int e = 0; e < 27; ++e) {
                    const int ev[3] = {e / 9 - 1, (e / 3) % 3 - 1, e % 3 - 1};
                    if (ev[0] == 0 && ev[1] == 0 && ev[2] == 0) continue;
                    // the receiver m = q + ev (periodic wrap); every moved axis needs a neighbour and a halo
                    int cm[3];
                    bool ok = true;
                    for (int a = 0; a < 3 && ok; ++a) {
                        cm[a] = cq[a] + ev[a];
                        if (ev[a] == 0) continue;
                        if (hs[a].h == 0 || g->nbr[lr][a][ev[a] > 0 ? 1 : 0] < 0) ok = false;
                        cm[a] = (cm[a] + g->dims[a]) % g->dims[a];
                    }
                    if (!ok) continue;
                    // boxes: moved axes -> my send range, the receiver's recv range; others -> the non-halo
                    // extent (identical on both: same coordinate along that axis)
                    int b0[3], d0[3], ext[3];
                    for (int a = 0; a < 3 && ok; ++a) {
                        const int h = hs[a].h;
                        if (ev[a] == +1) {          // receiver above: my upper send layers -> its lower halo
                            b0[a] = hs[a].send_up[0];
                            d0[a] = hs[a].recv_lo[0];
                            ext[a] = h;
                        } else if (ev[a] == -1) {   // receiver below: my lower send layers -> its upper halo
                            b0[a] = hs[a].send_lo[0];
                            d0[a] = hs[a].recv_up[0];
                            ext[a] = h;
                        } else {
                            const int lo = (h > 0 && g->nbr[lr][a][0] >= 0) ? hs[a].recv_lo[1] : 0;
                            const int hi = (h > 0 && g->nbr[lr][a][1] >= 0) ? hs[a].recv_up[0] : (int)s[a];
                            b0[a] = d0[a] = lo;
                            ext[a] = hi - lo;
                        }
                        if (ext[a] <= 0) ok = false;
                    }
                    if (!ok) continue;
                    const int m = rank_of_coords(g->dims, cm);
                    const int ml = local_index(g, m);
                    const int mp = proc_of(g, m), mlr = m - mp * L;
                    H26Item it{};
                    it.esz = esz;
                    it.bx = ext[0];
                    it.by = ext[1];
                    it.bz = ext[2];
                    it.cells = (long long)ext[0] * ext[1] * ext[2];
                    it.src = reinterpret_cast<const char *>(F.ptr) + ((long long)b0[2] * sz + (long long)b0[1] * sy + b0[0]) * esz;
                    it.ssy = sy;
                    it.ssz = sz;
                    it.wait = -1;
                    unsigned long long *mflags = ml >= 0 ? g->flags : g->peer_flags[mp];
                    if (ev[1] == 0 && ev[2] == 0) {
                        // x face: z-contiguous into the receiver's arena slot (field f, axis 0, its halo side)
                        const int side = ev[0] > 0 ? 0 : 1;
                        char *arena = ml >= 0 ? g->recv_arena : g->peer_recv[mp];
                        it.dst = arena + (size_t)((long long)mlr * plan.block + plan.off[f][0][side]) * 8;
                        it.dsy = ext[0];
                        it.dsz = (long long)ext[0] * ext[1];
                    } else {
                        const long long dsy = s[0], dsz = s[0] * s[1];   // same field shape on the receiver
                        // the receiver's array: a sibling's, or process mp's array of ITS rank mlr (the
                                        // mapping of position (mlr, f) of the collective exchange)
                        char *dbase = ml >= 0 ? reinterpret_cast<char *>(fields[ml * nf + f].ptr)
                                              : reinterpret_cast<char *>(pmap[mlr * nf + f][mp]);
                        it.dst = dbase + ((long long)d0[2] * dsz + (long long)d0[1] * dsy + d0[0]) * esz;
                        it.dsy = dsy;
                        it.dsz = dsz;
                    }
                    if (ml < 0) {   // remote receiver: wait until it released its halos of the last epoch
                        it.wait = waitp_index(h26_flag(g->flags, L, lr, 32 + e));
                        it.remote = 1;
                    }
                    store.push_back(it);
                    // the receiver's data flag of the direction pointing back at me
                    add_unique(signal, h26_flag(mflags, L, mlr, dir_index(-ev[0], -ev[1], -ev[2])));
                }
                // my incoming: data flags to await; remote senders' ready flags; x-face unpacks
                for (int e = 0; e < 27; ++e) {
                    const int dv[3] = {e / 9 - 1, (e / 3) % 3 - 1, e % 3 - 1};   // from me to the sender
                    if (dv[0] == 0 && dv[1] == 0 && dv[2] == 0) continue;
                    int cs[3];
                    bool ok = true;
                    for (int a = 0; a < 3 && ok; ++a) {
                        cs[a] = cq[a] + dv[a];
                        if (dv[a] == 0) continue;
                        if (hs[a].h == 0 || g->nbr[lr][a][dv[a] > 0 ? 1 : 0] < 0) ok = false;
                        cs[a] = (cs[a] + g->dims[a]) % g->dims[a];
                    }
                    if (!ok) continue;
                    int r0[3], ext[3];
                    for (int a = 0; a < 3 && ok; ++a) {
                        const int h = hs[a].h;
                        if (dv[a] == -1) {
                            r0[a] = hs[a].recv_lo[0];
                            ext[a] = h;
                        } else if (dv[a] == +1) {
                            r0[a] = hs[a].recv_up[0];
                            ext[a] = h;
                        } else {
                            const int lo = (h > 0 && g->nbr[lr][a][0] >= 0) ? hs[a].recv_lo[1] : 0;
                            const int hi = (h > 0 && g->nbr[lr][a][1] >= 0) ? hs[a].recv_up[0] : (int)s[a];
                            r0[a] = lo;
                            ext[a] = hi - lo;
                        }
                        if (ext[a] <= 0) ok = false;
                    }
                    if (!ok) continue;
                    const int sr = rank_of_coords(g->dims, cs);
                    const int sl = local_index(g, sr);
                    const unsigned long long *mine = h26_flag(g->flags, L, lr, e);
                    add_unique(wait_end, mine);
                    if (sl < 0) {   // a remote sender: it stores into me after my ready
                        const int sp = proc_of(g, sr), slr = sr - sp * L;
                        add_unique(ready, h26_flag(g->peer_flags[sp], L, slr, 32 + dir_index(-dv[0], -dv[1], -dv[2])));
                    }
                    if (dv[1] == 0 && dv[2] == 0) {   // x face: unpack my arena slot after the data flag
                        const int side = dv[0] < 0 ? 0 : 1;
                        H26Item it{};
                        it.esz = esz;
                        it.bx = ext[0];
                        it.by = ext[1];
                        it.bz = ext[2];
                        it.cells = (long long)ext[0] * ext[1] * ext[2];
                        it.src = g->recv_arena + (size_t)((long long)lr * plan.block + plan.off[f][0][side]) * 8;
                        it.ssy = ext[0];
                        it.ssz = (long long)ext[0] * ext[1];
                        it.dst = reinterpret_cast<char *>(F.ptr) + ((long long)r0[2] * sz + (long long)r0[1] * sy + r0[0]) * esz;
                        it.dsy = sy;
                        it.dsz = sz;
                        it.wait = waitp_index(mine);
                        unpack.push_back(it);
                    }
                }
            }
        }
        // chunks: store items first, then the unpacks
        long long nch = 0, nstore = 0;
        std::vector<H26Item> items = store;
        items.insert(items.end(), unpack.begin(), unpack.end());
        for (size_t q = 0; q < items.size(); ++q) {
            items[q].chunk0 = nch;
            nch += (items[q].cells + kH26Chunk - 1) / kH26Chunk;
            if (q + 1 == store.size()) nstore = nch;
        }
        H26Plan P{};
        P.nitems = (int)items.size();
        P.nsignal = (int)signal.size();
        P.nready = (int)ready.size();
        P.nwait_end = (int)wait_end.size();
        P.nwaitp = (int)waitp.size();
        P.nchunks = nch;
        P.nstore_chunks = nstore;
        if (P.nready > kH26Threads) fail(IGG_E_UNSUPPORTED, "update_halo: too many remote senders");
        size_t off = (sizeof(H26Plan) + 15) & ~size_t(15);
        P.o_items = (long long)off;
        off += items.size() * sizeof(H26Item);
        P.o_signal = (long long)off;
        off += signal.size() * sizeof(void *);
        P.o_ready = (long long)off;
        off += ready.size() * sizeof(void *);
        P.o_wait_end = (long long)off;
        off += wait_end.size() * sizeof(void *);
        P.o_waitp = (long long)off;
        off += waitp.size() * sizeof(void *);
        std::vector<char> host(off);
        std::memcpy(host.data(), &P, sizeof P);
        if (!items.empty()) std::memcpy(host.data() + P.o_items, items.data(), items.size() * sizeof(H26Item));
        if (!signal.empty()) std::memcpy(host.data() + P.o_signal, signal.data(), signal.size() * sizeof(void *));
        if (!ready.empty()) std::memcpy(host.data() + P.o_ready, ready.data(), ready.size() * sizeof(void *));
        if (!wait_end.empty()) std::memcpy(host.data() + P.o_wait_end, wait_end.data(), wait_end.size() * sizeof(void *));
        if (!waitp.empty()) std::memcpy(host.data() + P.o_waitp, waitp.data(), waitp.size() * sizeof(void *));
        igg_grid::H26Cache e;
        e.key = key;
        e.nchunks = nch;
        IGG_CUDA(cudaMalloc(&e.dplan, off));   // (plan metadata, like the host plan cache: not a buffer-pool
                                               // allocation, so not counted by igg_buffer_allocs)
        IGG_CUDA(cudaMemcpy(e.dplan, host.data(), off, cudaMemcpyHostToDevice));
        if (g->h26_cache.size() >= 8) {   // keep the most recent shapes (Fig. 1 alternates two arrays)
            cudaFree(g->h26_cache.front().dplan);
            g->h26_cache.erase(g->h26_cache.begin());
        }
        g->h26_cache.push_back(e);
        hit = &g->h26_cache.back();
    }
    if (!g->h26_ctr) {
        IGG_CUDA(cudaMalloc(&g->h26_ctr, 2 * sizeof(unsigned int)));
        IGG_CUDA(cudaMemset(g->h26_ctr, 0, 2 * sizeof(unsigned int)));
        g->allocs++;
    }
    // every process launches (a rank with nothing to send still publishes ready and awaits its halos)
    const long long grid = std::max(1LL, std::min<long long>((hit->nchunks + kH26Batch - 1) / kH26Batch, 4LL * g->sm_count));
    halo26_kernel<<<(unsigned)grid, kH26Threads, 0, st>>>(static_cast<const char *>(hit->dplan), g->epoch, g->h26_ctr,
                                                          (long long)(g->spin_timeout_ms * g->clock_khz), g->d_err);
    IGG_CUDA(cudaGetLastError());
    g->launches++;
}

}  // namespace igg
