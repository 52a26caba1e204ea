// grid.cpp -- lifecycle, buffer pool, update_halo orchestration, the
// hide_communication heat step and reductions of libigg (host side).
//
// init_global_grid / update_halo! / finalize_global_grid: PAPER.md:36, :62,
// :77, :82.  "Low level management of memory, CUDA streams ... permits to
// efficiently reuse send and receive buffers and streams ... all data
// transfers are performed on non-blocking high-priority streams"  PAPER.md:94.
// @hide_communication (16,2,2): PAPER.md:75.
#include <cstdio>
#include <algorithm>
#include <functional>
#include <cstring>

#include "igg_internal.h"

#ifndef IGG_ABLATION
#define IGG_ABLATION 0   // the ablation build (-DIGG_ABLATION=1): tuning variants and schedule bits
#endif

namespace igg {

int proc_of(const igg_grid *g, int r) { return r / g->nlocal; }
int local_index(const igg_grid *g, int r) { return proc_of(g, r) == g->proc ? r - g->rank0 : -1; }

void check_live(const igg_grid *g, const char *what) {
    if (!g) fail(IGG_E_ARG, std::string(what) + ": grid is NULL");
    if (g->finalized) fail(IGG_E_STATE, std::string(what) + ": grid already finalized");
}

static void *dev_alloc(igg_grid *g, size_t bytes) {
    void *p = nullptr;
    IGG_CUDA(cudaMalloc(&p, bytes));
    g->allocs++;
    return p;
}

// all-gather of a small host blob over the processes (collective entry points only): through the
// caller's bootstrap callback when one was given, else over the NCCL communicator (a persistent
// device buffer, so no allocation synchronizes the device); one process: a copy
static std::vector<char> allgather_bytes(igg_grid *g, const void *mine, size_t bytes) {
    std::vector<char> out(bytes * g->nproc_procs);
    if (g->nproc_procs == 1) {
        std::memcpy(out.data(), mine, bytes);
        return out;
    }
    if (g->boot) {
        if (g->boot(g->boot_user, mine, out.data(), (unsigned long long)bytes) != 0)
            fail(IGG_E_BOOTSTRAP, "bootstrap all-gather of " + std::to_string(bytes) + " bytes failed");
        return out;
    }
    if (g->d_gather_bytes < out.size()) {
        if (g->d_gather) IGG_CUDA(cudaFree(g->d_gather));
        g->d_gather_bytes = std::max<size_t>(out.size(), 4096);
        IGG_CUDA(cudaMalloc(&g->d_gather, g->d_gather_bytes));
    }
    char *d = g->d_gather;
    IGG_CUDA(cudaMemcpyAsync(d + bytes * g->proc, mine, bytes, cudaMemcpyHostToDevice, g->s_comm));
    IGG_NCCL(ncclAllGather(d + bytes * g->proc, d, bytes, ncclChar, g->comm, g->s_comm));
    IGG_CUDA(cudaMemcpyAsync(out.data(), d, out.size(), cudaMemcpyDeviceToHost, g->s_comm));
    IGG_CUDA(cudaStreamSynchronize(g->s_comm));
    return out;
}

// max over the processes of one double, through allgather_bytes (host bootstrap)
double host_max(igg_grid *g, double local) {
    std::vector<char> all = allgather_bytes(g, &local, sizeof local);
    double m = local;
    for (int p = 0; p < g->nproc_procs; ++p) {
        double v;
        std::memcpy(&v, all.data() + p * sizeof v, sizeof v);
        m = std::max(m, v);
    }
    return m;
}

void check_device_error(igg_grid *g, const char *who) {
    IGG_CUDA(cudaDeviceSynchronize());
    int err = 0;
    IGG_CUDA(cudaMemcpy(&err, g->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) fail(IGG_E_TIMEOUT, std::string(who) + ": a P2P receive flag wait timed out (halos are invalid)");
}

std::vector<char> allgather_bytes_pub(igg_grid *g, const void *mine, size_t bytes) {
    return allgather_bytes(g, mine, bytes);
}

static void process_barrier(igg_grid *g) {
    IGG_CUDA(cudaDeviceSynchronize());
    if (g->nproc_procs > 1) {
        char x = 0;
        allgather_bytes(g, &x, 1);
    }
}

static void unmap_peers(igg_grid *g, std::vector<char *> &peers) {
    for (int p = 0; p < (int)peers.size(); ++p)
        if (peers[p] && p != g->proc) cudaIpcCloseMemHandle(peers[p]);
    peers.assign(g->nproc_procs, nullptr);
}

// Buffer pool: one receive arena with two parity halves
// (P2P ping-pong) and one send arena (NCCL).
// Every rank computes the same sizes from the same field list, so growth is a
// consistent collective; once every field list has been seen it never grows.
void ensure_arena(igg_grid *g, size_t recv_half, size_t send_cap) {
    const bool grow_recv = recv_half > g->recv_half;
    const bool grow_send = send_cap > g->send_cap;
    if (!grow_recv && !grow_send) return;
    process_barrier(g);   // nobody may still be writing into the old arenas
    release_h26(g);       // cached 26-neighbour plans point into the arenas
    if (grow_send) {
        if (g->send_arena) IGG_CUDA(cudaFree(g->send_arena));
        g->send_arena = (char *)dev_alloc(g, send_cap);
        g->send_cap = send_cap;
    }
    if (grow_recv) {
        if (g->path == IGG_PATH_P2P && g->nproc_procs > 1) unmap_peers(g, g->peer_recv);
        if (g->recv_arena) IGG_CUDA(cudaFree(g->recv_arena));
        g->recv_arena = (char *)dev_alloc(g, 2 * recv_half);
        IGG_CUDA(cudaMemset(g->recv_arena, 0, 2 * recv_half));
        g->recv_half = recv_half;
        g->peer_recv.assign(g->nproc_procs, nullptr);
        g->peer_recv[g->proc] = g->recv_arena;   // (IGG_OPT_LOCAL_P2P: sibling ranks' slots)
        if (g->path == IGG_PATH_P2P && g->nproc_procs > 1) {
            cudaIpcMemHandle_t h;
            IGG_CUDA(cudaIpcGetMemHandle(&h, g->recv_arena));
            std::vector<char> all = allgather_bytes(g, &h, sizeof h);
            g->peer_recv.assign(g->nproc_procs, nullptr);
            for (int p = 0; p < g->nproc_procs; ++p) {
                if (p == g->proc) {
                    g->peer_recv[p] = g->recv_arena;
                    continue;
                }
                cudaIpcMemHandle_t ph;
                std::memcpy(&ph, all.data() + p * sizeof ph, sizeof ph);
                void *ptr = nullptr;
                IGG_CUDA(cudaIpcOpenMemHandle(&ptr, ph, cudaIpcMemLazyEnablePeerAccess));
                g->peer_recv[p] = (char *)ptr;
            }
        }
    }
    process_barrier(g);
}

// ------------------------------------------------------------------ update_halo
// Executes the plan of plan.cpp: per axis one pack launch (faces into the
// receiver's arena slot: local, peer-mapped over NVLink, or the NCCL send
// arena), the grouped NCCL send/recv of that axis, one unpack launch.
// plans depend only on the field sizes: built once per field-list shape
// key: nf*3 sizes then nf element sizes
const Plan &cached_plan(igg_grid *g, const std::vector<long long> &key, int nf) {
    for (const auto &e : g->plan_cache)
        if (e.first == key) return e.second;
    std::vector<int> esz(nf);
    for (int f = 0; f < nf; ++f) esz[f] = (int)key[3 * nf + f];
    g->plan_cache.push_back({key, build_plan(*g, key.data(), nf, esz.data())});
    return g->plan_cache.back().second;
}

void exchange(igg_grid *g, const igg_field *fields, int nf, cudaStream_t st, bool allow_coop) {
    if (nf < 1 || !fields) fail(IGG_E_ARG, "update_halo: need at least one field");
    const int L = g->nlocal;
    std::vector<long long> sizes(nf * 4);   // nf*3 sizes, then nf element sizes (the plan key)
    for (int f = 0; f < nf; ++f) {
        for (int a = 0; a < 3; ++a) sizes[f * 3 + a] = fields[f].size[a];
        const int e = fields[f].elsize == 0 ? 8 : fields[f].elsize;
        if (e != 8 && e != 4) fail(IGG_E_ARG, "update_halo: elsize must be 0, 8 or 4");
        sizes[3 * nf + f] = e;
    }
    for (int r = 0; r < L; ++r)
        for (int f = 0; f < nf; ++f) {
            const igg_field &F = fields[r * nf + f];
            if (!F.ptr) fail(IGG_E_ARG, "update_halo: NULL field pointer");
            for (int a = 0; a < 3; ++a)
                if (F.size[a] != sizes[f * 3 + a]) fail(IGG_E_ARG, "update_halo: local ranks disagree on a field size");
            if ((F.elsize == 0 ? 8 : F.elsize) != sizes[3 * nf + f])
                fail(IGG_E_ARG, "update_halo: local ranks disagree on a field element size");
        }
    const Plan &plan = cached_plan(g, sizes, nf);
    const size_t half = (size_t)L * plan.block * sizeof(double);
    ensure_arena(g, half, plan.any_nccl ? half : 0);

    g->epoch++;
    if (g->skip_comm) return;
    if (!plan.any_nccl && g->halo26 && !g->local_p2p) {   // no NCCL message: the one-kernel 26-neighbour exchange
        exchange26(g, fields, nf, plan, st);
        return;
    }
    const int parity = (int)(g->epoch & 1);
    double *recv = reinterpret_cast<double *>(g->recv_arena + parity * g->recv_half);
    double *sendb = reinterpret_cast<double *>(g->send_arena);

    // per axis: pack / unpack descriptors, peer signals and waits, NCCL messages
    std::vector<CopyDesc> pd[3], ud[3];
    CopyList P[3]{}, U[3]{};
    std::vector<const PlanMsg *> sends[3], recvs[3];
    bool any_nccl = false;
    for (int a = 0; a < 3; ++a) {   // x -> y -> z, each axis complete before the next
        P[a].ticket = g->tickets + a;
        P[a].epoch = U[a].epoch = g->epoch;
        U[a].err = P[a].err = g->d_err;
        U[a].timeout_cycles = (long long)(g->spin_timeout_ms * g->clock_khz);
        for (const PlanMsg &pm : plan.msgs[a]) {
            // IGG_OPT_LOCAL_P2P: ranks of this process exchange through the P2P protocol (store into the
            // receiver's slot, release flag, acquire wait) instead of plain stream-ordered copies -- the
            // cross-process data plane emulated on one GPU; packs precede the waits on the stream, so no
            // wait depends on a concurrently running launch
            PlanMsg m = pm;
            if (g->local_p2p && m.transport == kLocal) m.transport = kP2P;
            CopyDesc d{};
            const igg_field &F = fields[m.lr * nf + m.field];
            d.field = F.ptr;
            d.sx = F.size[0];
            d.sy = F.size[1];
            d.sz = F.size[2];
            d.count = m.count;
            d.esz = (int)sizes[3 * nf + m.field];
            d.axis = a;
            d.lo = m.lo;
            d.h = m.h;
            d.flag_slot = -1;
            if (m.op == 0) {
                if (m.transport == kLocal) {
                    d.buf = recv + m.slot;
                } else if (m.transport == kP2P) {
                    d.buf = reinterpret_cast<double *>(g->peer_recv[m.peer_proc] + parity * g->recv_half) + m.slot;
                    unsigned long long *fl =
                        g->peer_flags[m.peer_proc] + ((m.peer_lr * 3 + a) * 2 + m.recv_side) * kMaxChunks;
                    bool have = false;
                    for (int q = 0; q < P[a].nsignal; ++q) have |= P[a].signal[q] == fl;
                    if (!have) {
                        if (P[a].nsignal >= kMaxSignal) fail(IGG_E_UNSUPPORTED, "update_halo: too many peers");
                        P[a].signal[P[a].nsignal++] = fl;
                    }
                } else {
                    d.buf = sendb + m.sbuf;
                    sends[a].push_back(&pm);
                    any_nccl = true;
                }
                pd[a].push_back(d);
            } else {
                d.buf = recv + m.slot;
                if (m.transport == kP2P) {
                    const unsigned long long *fl = g->flags + ((m.lr * 3 + a) * 2 + m.recv_side) * kMaxChunks;
                    int w = -1;
                    for (int q = 0; q < U[a].nsignal; ++q)
                        if (U[a].wait[q] == fl) w = q;
                    if (w < 0) {
                        if (U[a].nsignal >= kMaxSignal) fail(IGG_E_UNSUPPORTED, "update_halo: too many peers");
                        w = U[a].nsignal;
                        U[a].wait[U[a].nsignal++] = fl;
                    }
                    d.flag_slot = w;
                } else if (m.transport == kNccl) {
                    recvs[a].push_back(&pm);
                    any_nccl = true;
                }
                ud[a].push_back(d);
            }
        }
    }
    for (int a = 0; a < 3; ++a) {
        if (plan.msgs[a].empty()) continue;
        g->launches += launch_copies(0, pd[a], P[a], st);
        if (!sends[a].empty() || !recvs[a].empty()) {
            auto by_order = [](const PlanMsg *x, const PlanMsg *y) { return x->order < y->order; };
            std::sort(sends[a].begin(), sends[a].end(), by_order);
            std::sort(recvs[a].begin(), recvs[a].end(), by_order);
            IGG_NCCL(ncclGroupStart());
            for (const PlanMsg *m : sends[a])
                IGG_NCCL(ncclSend(sendb + m->sbuf, (size_t)m->words, ncclDouble, m->peer_proc, g->comm, st));
            for (const PlanMsg *m : recvs[a])
                IGG_NCCL(ncclRecv(recv + m->slot, (size_t)m->words, ncclDouble, m->peer_proc, g->comm, st));
            IGG_NCCL(ncclGroupEnd());
        }
        g->launches += launch_copies(1, ud[a], U[a], st);
    }
}

// ------------------------------------------------------------------ profiling
void prof_begin(igg_grid *g, cudaStream_t s) {
    if (!g->profile) return;
    while (g->prof_ev.size() < g->prof_used + 2) {
        cudaEvent_t e;
        IGG_CUDA(cudaEventCreate(&e));
        g->prof_ev.push_back(e);
    }
    IGG_CUDA(cudaEventRecord(g->prof_ev[g->prof_used], s));
}

void prof_end(igg_grid *g, cudaStream_t s, long long cells) {
    if (!g->profile) return;
    IGG_CUDA(cudaEventRecord(g->prof_ev[g->prof_used + 1], s));
    g->prof_used += 2;
    g->prof_cells += cells;
}

void tl_mark(igg_grid *g, cudaStream_t s, int k) {
    if (g->profile < 2) return;
    const size_t idx = g->tl_used + k;
    while (g->tl_ev.size() <= idx) {
        cudaEvent_t e;
        IGG_CUDA(cudaEventCreate(&e));
        g->tl_ev.push_back(e);
    }
    IGG_CUDA(cudaEventRecord(g->tl_ev[idx], s));
    if (k == 4) g->tl_used += 5;
}

// ------------------------------------------------------------------ the heat step
static HeatRegion make_region(igg_grid *g, int lr, double *const *T2, const double *const *T,
                              const double *const *Ci, int x0, int x1, int y0, int y1, int z0, int z1) {
    HeatRegion R{};
    R.T = T[lr];
    R.Ci = Ci[lr];
    R.T2 = T2[lr];
    R.sx = g->n[0];
    R.sy = g->n[1];
    R.sz = g->n[2];
    R.x0 = x0;
    R.y0 = y0;
    R.z0 = z0;
    R.wx = x1 - x0;
    R.wy = y1 - y0;
    R.wz = z1 - z0;
    return R;
}

// Launch a list of regions with the kernel selected by IGG_OPT_STENCIL_KERNEL:
// 0 = cp.async box-list kernel (production), 1 = generic scalar region kernel,
// >= 2 = per-region box-kernel ablation variants (regions) / slab kernel (slabs).
// `main` regions are the profiled ones (full region or inner boxes).
static void launch_regions(igg_grid *g, const std::vector<HeatRegion> &regs, const HeatCoef &k, cudaStream_t s,
                           bool main) {
    std::vector<HeatRegion> rs;
    long long cells = 0;
    bool vec = true;
    for (const HeatRegion &R : regs)
        if (R.wx > 0 && R.wy > 0 && R.wz > 0) {
            rs.push_back(R);
            cells += (long long)R.wx * R.wy * R.wz;
            vec = vec && heat_box_vectorizable(R);
        }
    if (rs.empty()) return;
    if (main) prof_begin(g, s);
    const int v = g->stencil_kernel;
    if (((v >= 2 && v < 30) || (v >= 50 && v < 60) || v == 0) && vec && main) {   // 0: launch_heat_box's default (variant 20)
        for (const HeatRegion &R : rs) {
            launch_heat_box(R, k, s, v);
            g->launches++;
        }
    } else {
        // narrow regions (x-slabs up to 32 cells from their 16-B aligned start) go to the slab
        // kernel, which reads only their own row segments; wide ones to the pipelined box kernel
        std::vector<HeatRegion> narrow, wide;
        for (const HeatRegion &R : rs) {
            const bool is_narrow = (R.x0 + R.wx - (R.x0 & ~1)) <= 32;
            (((v == 0 || (v >= 30 && v < 40)) && !is_narrow) ? wide : narrow).push_back(R);
        }
        for (int pass = 0; pass < 2; ++pass) {
            const std::vector<HeatRegion> &part = pass == 0 ? wide : narrow;
            for (size_t c = 0; c < part.size(); c += kMaxRegions) {
                HeatRegionList L{};
                L.k = k;
                for (size_t j = c; j < part.size() && j < c + kMaxRegions; ++j) L.r[L.n++] = part[j];
                if (v == 1 || !vec)
                    launch_heat_regions(L, s);
                else if (pass == 0)
                    launch_heat_box_list(L, s, v);
                else
                    launch_heat_slabs(L, s);
                g->launches++;
            }
        }
    }
    if (main) prof_end(g, s, cells);
}

static void launch_full(igg_grid *g, double *const *T2, const double *const *T, const double *const *Ci,
                        const HeatCoef &k, cudaStream_t s) {
    std::vector<HeatRegion> rs;
    for (int lr = 0; lr < g->nlocal; ++lr)
        rs.push_back(make_region(g, lr, T2, T, Ci, 1, g->n[0] - 1, 1, g->n[1] - 1, 1, g->n[2] - 1));
    launch_regions(g, rs, k, s, true);
}

void heat_step(igg_grid *g, double *const *T2, const double *const *T, const double *const *Ci, double lam,
               double dt, double dx, double dy, double dz, const int bw[3], cudaStream_t s, bool wait_prev,
               bool drain) {
    for (int lr = 0; lr < g->nlocal; ++lr)
        if (!T2[lr] || !T[lr] || !Ci[lr]) fail(IGG_E_ARG, "heat_step: NULL field pointer");
    bool lowdim = false;
    for (int a = 0; a < 3; ++a) {
        if (g->n[a] == 2) fail(IGG_E_ARG, "heat_step: an axis needs 1 (size-1 axis) or at least 3 cells");
        lowdim = lowdim || g->n[a] == 1;
    }
    // reciprocals computed once on the host (reading 9, canonical form)
    const HeatCoef k{lam, dt, 1.0 / (dx * dx), 1.0 / (dy * dy), 1.0 / (dz * dz)};
    if (lowdim) {
        // 1-D/2-D grid (size-1 axes, reading 23): the low-dimensional stencil on the
        // whole updated box, then update_halo (sequential schedule)
        std::vector<igg_field> f(g->nlocal);
        for (int lr = 0; lr < g->nlocal; ++lr) f[lr] = igg_field{T2[lr], {g->n[0], g->n[1], g->n[2]}};
        IGG_CUDA(cudaEventRecord(g->ev_start, s));
        IGG_CUDA(cudaStreamWaitEvent(g->s_comm, g->ev_start, 0));
        for (int lr = 0; lr < g->nlocal; ++lr) {
            launch_heat_lowdim(T2[lr], T[lr], Ci[lr], g->n, k, g->s_comm);
            g->launches++;
        }
        exchange(g, f.data(), 1, g->s_comm);
        IGG_CUDA(cudaEventRecord(g->ev_comm, g->s_comm));
        IGG_CUDA(cudaStreamWaitEvent(s, g->ev_comm, 0));
        return;
    }
    bool exch[3] = {false, false, false};
    bool any = false;
    for (int a = 0; a < 3; ++a)
        for (int lr = 0; lr < g->nlocal; ++lr)
            if (g->nbr[lr][a][0] >= 0 || g->nbr[lr][a][1] >= 0) exch[a] = any = true;
    if (!any) {   // nothing to exchange or hide: one full-region launch
        launch_full(g, T2, T, Ci, k, s);
        return;
    }
    const int zero[3] = {0, 0, 0};
    if (!bw) bw = zero;
    const bool sequential_req = bw[0] == 0 && bw[1] == 0 && bw[2] == 0;
    int lo[3], hi[3];
    bool degenerate = false;
    for (int a = 0; a < 3; ++a) {
        if (bw[a] < 0) fail(IGG_E_ARG, "heat_step: negative boundary width");
        // the send layers must be final before any face leaves
        if (!sequential_req && exch[a] && bw[a] < g->o[a])
            fail(IGG_E_WIDTH, "heat_step: boundary width " + std::to_string(bw[a]) + " on axis " +
                                  std::to_string(a) + " is below the field overlap " + std::to_string(g->o[a]));
        // an axis without an exchange has nothing to send early: no boundary slabs on it
        const int b = exch[a] ? bw[a] : 0;
        lo[a] = std::max(1, b);
        hi[a] = std::min(g->n[a] - 1, g->n[a] - b);
        if (a == 0 && exch[0] && g->x_align > 1) {
            // B200: x-boundaries on 512-B row segments; the
            // boundary phase grows to whole 64-cell tiles, results are unchanged
            const int A = g->x_align;
            lo[0] = ((lo[0] + A - 1) / A) * A;
            hi[0] = (hi[0] / A) * A;
        }
        if (hi[a] <= lo[a]) degenerate = true;   // empty inner box
    }
    std::vector<igg_field> f(g->nlocal);
    for (int lr = 0; lr < g->nlocal; ++lr) f[lr] = igg_field{T2[lr], {g->n[0], g->n[1], g->n[2]}};
    if (!sequential_req && g->stencil_kernel == 0 && fused_eligible(g)) {
        bool vec = true;
        for (int lr = 0; lr < g->nlocal; ++lr)
            vec = vec && heat_box_vectorizable(make_region(g, lr, T2, T, Ci, 1, g->n[0] - 1, 1, g->n[1] - 1, 1, g->n[2] - 1));
        if (vec) {   // one kernel: stencil + exchange into the receivers' memory
            fused_step(g, T2, T, Ci, k, s, wait_prev, drain);
            return;
        }
    }

    IGG_CUDA(cudaEventRecord(g->ev_start, s));
    IGG_CUDA(cudaStreamWaitEvent(g->s_comm, g->ev_start, 0));
    if (sequential_req || degenerate) {
        launch_full(g, T2, T, Ci, k, g->s_comm);
        exchange(g, f.data(), 1, g->s_comm);
        IGG_CUDA(cudaEventRecord(g->ev_comm, g->s_comm));
        IGG_CUDA(cudaStreamWaitEvent(s, g->ev_comm, 0));
        return;
    }
    // (1) the six boundary slabs, x-lo, x-hi, y-lo, y-hi, z-lo, z-hi, high priority
    const int n0 = g->n[0], n1 = g->n[1], n2 = g->n[2];
    std::vector<HeatRegion> slabs, inner;
    for (int lr = 0; lr < g->nlocal; ++lr) {
        slabs.push_back(make_region(g, lr, T2, T, Ci, 1, lo[0], 1, n1 - 1, 1, n2 - 1));
        slabs.push_back(make_region(g, lr, T2, T, Ci, hi[0], n0 - 1, 1, n1 - 1, 1, n2 - 1));
        slabs.push_back(make_region(g, lr, T2, T, Ci, lo[0], hi[0], 1, lo[1], 1, n2 - 1));
        slabs.push_back(make_region(g, lr, T2, T, Ci, lo[0], hi[0], hi[1], n1 - 1, 1, n2 - 1));
        slabs.push_back(make_region(g, lr, T2, T, Ci, lo[0], hi[0], lo[1], hi[1], 1, lo[2]));
        slabs.push_back(make_region(g, lr, T2, T, Ci, lo[0], hi[0], lo[1], hi[1], hi[2], n2 - 1));
        inner.push_back(make_region(g, lr, T2, T, Ci, lo[0], hi[0], lo[1], hi[1], lo[2], hi[2]));
    }
    tl_mark(g, s, 0);
    launch_regions(g, slabs, k, g->s_comm, false);
    tl_mark(g, g->s_comm, 1);
    // (2) the inner box on the low-priority stream.  schedule 0: starts with the boundary
    // (they share the GPU); schedule 1 (the paper's order): starts when the
    // boundary is done, so the inner box never shares SM slots with the latency-bound slabs
    if (g->schedule == 1) {
        IGG_CUDA(cudaEventRecord(g->ev_bnd, g->s_comm));
        IGG_CUDA(cudaStreamWaitEvent(g->s_inner, g->ev_bnd, 0));
    } else {
        IGG_CUDA(cudaStreamWaitEvent(g->s_inner, g->ev_start, 0));
    }
    tl_mark(g, g->s_inner, 2);
    launch_regions(g, inner, k, g->s_inner, true);
    tl_mark(g, g->s_inner, 3);
    // (3) update_halo!(T2) behind the boundary, on the high-priority stream
    exchange(g, f.data(), 1, g->s_comm);
    tl_mark(g, g->s_comm, 4);
    IGG_CUDA(cudaEventRecord(g->ev_comm, g->s_comm));
    IGG_CUDA(cudaEventRecord(g->ev_inner, g->s_inner));
    IGG_CUDA(cudaStreamWaitEvent(s, g->ev_comm, 0));
    IGG_CUDA(cudaStreamWaitEvent(s, g->ev_inner, 0));
}

}  // namespace igg

// ============================================================== C ABI
using igg::fail;

IGG_API igg_status igg_get_unique_id(unsigned char out[128]) {
    IGG_TRY
    if (!out) fail(IGG_E_ARG, "igg_get_unique_id: out is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    IGG_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, 128);
    IGG_CATCH
}

IGG_API igg_status igg_init_global_grid(const igg_init_args *A, igg_grid **grid_out, int *me, int coords[3],
                                        int dims_out[3], long long n_g[3]) {
    igg_grid *g = nullptr;
    try {
        if (!A || !grid_out) fail(IGG_E_ARG, "igg_init_global_grid: NULL argument");
        igg::Geom geo = igg::make_geom(A);
        g = new igg_grid();
        static_cast<igg::Geom &>(*g) = geo;
        IGG_CUDA(cudaSetDevice(g->device));
        IGG_CUDA(cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, g->device));
        int khz = 0;
        if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, g->device) == cudaSuccess && khz > 0)
            g->clock_khz = khz;
        int least = 0, greatest = 0;
        IGG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        IGG_CUDA(cudaStreamCreateWithPriority(&g->s_comm, cudaStreamNonBlocking, greatest));
        IGG_CUDA(cudaStreamCreateWithPriority(&g->s_inner, cudaStreamNonBlocking, least));
        IGG_CUDA(cudaStreamCreateWithPriority(&g->s_comm2, cudaStreamNonBlocking, greatest));
        IGG_CUDA(cudaEventCreateWithFlags(&g->ev_start, cudaEventDisableTiming));
        IGG_CUDA(cudaEventCreateWithFlags(&g->ev_comm, cudaEventDisableTiming));
        IGG_CUDA(cudaEventCreateWithFlags(&g->ev_inner, cudaEventDisableTiming));
        IGG_CUDA(cudaEventCreateWithFlags(&g->ev_bnd, cudaEventDisableTiming));
        IGG_CUDA(cudaEventCreateWithFlags(&g->ev_comm2, cudaEventDisableTiming));
        g->boot = A->bootstrap;
        g->boot_user = A->bootstrap_user;
        if (g->nproc_procs > 1 && g->boot && g->path != IGG_PATH_P2P)
            fail(IGG_E_ARG, "igg_init_global_grid: a host bootstrap needs path IGG_PATH_P2P (no NCCL communicator)");
        if (g->nproc_procs > 1 && !g->boot) {
            ncclUniqueId id;
            std::memcpy(&id, A->comm_id, sizeof id);
            IGG_NCCL(ncclCommInitRank(&g->comm, g->nproc_procs, id, g->proc));
        }
        // receive flags (P2P), last-block tickets, error word, reduction scratch
        // [data | rim+forwarded] x nlocal x 6 faces x kMaxChunks
        // + the 26-neighbour exchange's data / ready flags (halo26.cu)
        const size_t flag_bytes =
            (2 * 6 * igg::kMaxChunks + igg::kH26Flags) * sizeof(unsigned long long) * g->nlocal;
        g->flags = (unsigned long long *)igg::dev_alloc(g, flag_bytes);
        IGG_CUDA(cudaMemset(g->flags, 0, flag_bytes));
        g->tickets = (unsigned int *)igg::dev_alloc(g, sizeof(unsigned int) * 4);
        IGG_CUDA(cudaMemset(g->tickets, 0, sizeof(unsigned int) * 4));
        g->d_err = (int *)igg::dev_alloc(g, sizeof(int) * 2);
        IGG_CUDA(cudaMemset(g->d_err, 0, sizeof(int) * 2));
        g->d_scratch = (double *)igg::dev_alloc(g, sizeof(double) * (igg::field_max_scratch_len() + 2));
        IGG_CUDA(cudaMallocHost(&g->d_pinned_out, sizeof(double)));
        g->peer_recv.assign(g->nproc_procs, nullptr);
        g->peer_flags.assign(g->nproc_procs, nullptr);
        g->peer_flags[g->proc] = g->flags;
        if (g->path == IGG_PATH_P2P && g->nproc_procs > 1) {
            cudaIpcMemHandle_t h;
            IGG_CUDA(cudaIpcGetMemHandle(&h, g->flags));
            std::vector<char> all = igg::allgather_bytes(g, &h, sizeof h);
            for (int p = 0; p < g->nproc_procs; ++p) {
                if (p == g->proc) continue;
                cudaIpcMemHandle_t ph;
                std::memcpy(&ph, all.data() + p * sizeof ph, sizeof ph);
                void *ptr = nullptr;
                IGG_CUDA(cudaIpcOpenMemHandle(&ptr, ph, cudaIpcMemLazyEnablePeerAccess));
                g->peer_flags[p] = (unsigned long long *)ptr;
            }
        }
        IGG_CUDA(cudaDeviceSynchronize());
        if (me) *me = g->rank0;
        if (coords)
            for (int a = 0; a < 3; ++a) coords[a] = g->coords[0][a];
        if (dims_out) std::memcpy(dims_out, g->dims, sizeof g->dims);
        if (n_g)
            for (int a = 0; a < 3; ++a) n_g[a] = g->ng[a];
        *grid_out = g;
        return IGG_OK;
    } catch (const igg::IggException &e) {
        delete g;   // partial init: resources of a failed init are leaked to the process (rare)
        return e.code;
    } catch (const std::exception &e) {
        delete g;
        igg::set_error(std::string("internal error: ") + e.what());
        return IGG_E_ARG;
    }
}

IGG_API igg_status igg_finalize_global_grid(igg_grid *g) {
    IGG_TRY
    igg::check_live(g, "igg_finalize_global_grid");
    g->finalized = true;
    igg::process_barrier(g);
    for (auto &o : g->fused_opened) cudaIpcCloseMemHandle(o.second);
    g->fused_opened.clear();
    g->fused_peer_maps.clear();
    igg::release_h26(g);
    if (g->path == IGG_PATH_P2P && g->nproc_procs > 1) {
        igg::unmap_peers(g, g->peer_recv);
        for (int p = 0; p < g->nproc_procs; ++p)
            if (p != g->proc && g->peer_flags[p]) cudaIpcCloseMemHandle(g->peer_flags[p]);
    }
    igg::process_barrier(g);
    for (void *p : {(void *)g->h26_ctr, (void *)g->d_gather, (void *)g->fused_xloc, (void *)g->fused_xcnt, (void *)g->fused_xrem, (void *)g->fused_tgt_x, (void *)g->fused_tgt_pipe, (void *)g->fused_ctr, (void *)g->recv_arena, (void *)g->send_arena, (void *)g->flags, (void *)g->tickets,
                    (void *)g->d_err, (void *)g->d_scratch, (void *)g->run_T, (void *)g->run_T2, (void *)g->run_Ci})
        if (p) cudaFree(p);
    if (g->d_pinned_out) cudaFreeHost(g->d_pinned_out);
    if (g->comm) ncclCommDestroy(g->comm);
    for (cudaEvent_t e : g->prof_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : g->tl_ev) cudaEventDestroy(e);
    cudaEventDestroy(g->ev_start);
    cudaEventDestroy(g->ev_comm);
    cudaEventDestroy(g->ev_inner);
    cudaEventDestroy(g->ev_bnd);
    cudaEventDestroy(g->ev_comm2);
    cudaStreamDestroy(g->s_comm);
    cudaStreamDestroy(g->s_inner);
    cudaStreamDestroy(g->s_comm2);
    delete g;
    IGG_CATCH
}

IGG_API igg_status igg_n_g(const igg_grid *g, int axis, long long field_size, long long *out) {
    IGG_TRY
    igg::check_live(g, "igg_n_g");
    if (axis < 0 || axis > 2 || !out) fail(IGG_E_ARG, "igg_n_g: bad axis or NULL out");
    const long long s = field_size == 0 ? g->n[axis] : field_size;
    igg::HaloSpec hs;
    if (!igg::halo_spec(g->n[axis], g->o[axis], s, &hs)) fail(IGG_E_STAGGER, "igg_n_g: field size out of range");
    *out = g->periods[axis] ? g->ng[axis] : g->ng[axis] + (s - g->n[axis]);
    IGG_CATCH
}

IGG_API igg_status igg_coords(const igg_grid *g, int rank, int coords_out[3]) {
    IGG_TRY
    igg::check_live(g, "igg_coords");
    if (rank < 0 || rank >= g->nprocs || !coords_out) fail(IGG_E_ARG, "igg_coords: bad rank or NULL out");
    igg::coords_of_rank(g->dims, rank, coords_out);
    IGG_CATCH
}

IGG_API igg_status igg_local_to_global(const igg_grid *g, int rank, int axis, long long l, long long *g_out) {
    IGG_TRY
    igg::check_live(g, "igg_local_to_global");
    if (rank < 0 || rank >= g->nprocs || axis < 0 || axis > 2 || !g_out)
        fail(IGG_E_ARG, "igg_local_to_global: bad argument");
    // a layer of some field on this axis: fields have at most n+o layers
    if (l < 0 || l >= (long long)g->n[axis] + g->o[axis])
        fail(IGG_E_ARG, "igg_local_to_global: local layer " + std::to_string(l) + " outside [0, " +
                            std::to_string(g->n[axis] + g->o[axis]) + ") on axis " + std::to_string(axis));
    int c[3];
    igg::coords_of_rank(g->dims, rank, c);
    long long v = (long long)c[axis] * (g->n[axis] - g->o[axis]) + l;
    if (g->periods[axis]) {
        const long long P = (long long)g->dims[axis] * (g->n[axis] - g->o[axis]);
        v = ((v - g->o[axis] / 2) % P + P) % P;
    }
    *g_out = v;
    IGG_CATCH
}

IGG_API igg_status igg_global_coord(const igg_grid *g, int rank, int axis, long long l, double spacing, double *x_out) {
    IGG_TRY
    if (!x_out) fail(IGG_E_ARG, "igg_global_coord: NULL out");
    long long gi = 0;
    const igg_status st = igg_local_to_global(g, rank, axis, l, &gi);
    if (st != IGG_OK) return st;
    *x_out = (double)gi * spacing;
    IGG_CATCH
}

IGG_API igg_status igg_save_field(const char *path, const double *host, const long long n[3]) {
    IGG_TRY
    if (!path || !host || !n || n[0] <= 0 || n[1] <= 0 || n[2] <= 0) fail(IGG_E_ARG, "igg_save_field: bad argument");
    FILE *f = std::fopen(path, "wb");
    if (!f) fail(IGG_E_ARG, std::string("igg_save_field: cannot open ") + path);
    const size_t cnt = (size_t)(n[0] * n[1] * n[2]);
    const bool ok = std::fprintf(f, "IGRIDF1 %lld %lld %lld\n", n[0], n[1], n[2]) > 0 &&
                    std::fwrite(host, sizeof(double), cnt, f) == cnt;   // (x86-64 / aarch64: little-endian)
    if (std::fclose(f) != 0 || !ok) fail(IGG_E_ARG, std::string("igg_save_field: write failed: ") + path);
    IGG_CATCH
}

IGG_API igg_status igg_buffer_allocs(const igg_grid *g, long long *count_out) {
    IGG_TRY
    igg::check_live(g, "igg_buffer_allocs");
    if (!count_out) fail(IGG_E_ARG, "igg_buffer_allocs: NULL out");
    *count_out = g->allocs;
    IGG_CATCH
}

IGG_API igg_status igg_kernel_launches(const igg_grid *g, long long *count_out) {
    IGG_TRY
    igg::check_live(g, "igg_kernel_launches");
    if (!count_out) fail(IGG_E_ARG, "igg_kernel_launches: NULL out");
    *count_out = g->launches;
    IGG_CATCH
}

IGG_API igg_status igg_update_halo(igg_grid *g, const igg_field *fields, int nfields, igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_update_halo");
    cudaStream_t s = (cudaStream_t)stream;
    if (g->halo_on_caller) {   // IGG_OPT_HALO_STREAM = 1: on the caller's stream (no cross-stream hops)
        igg::exchange(g, fields, nfields, s, true);
    } else {                   // default: the library's high-priority comm stream
        IGG_CUDA(cudaEventRecord(g->ev_start, s));
        IGG_CUDA(cudaStreamWaitEvent(g->s_comm, g->ev_start, 0));
        igg::exchange(g, fields, nfields, g->s_comm, true);   // standalone: nothing runs beside it
        IGG_CUDA(cudaEventRecord(g->ev_comm, g->s_comm));
        IGG_CUDA(cudaStreamWaitEvent(s, g->ev_comm, 0));
    }
    IGG_CATCH
}

IGG_API igg_status igg_heat_step(igg_grid *g, double *const *T2, const double *const *T, const double *const *Ci,
                                 double lam, double dt, double dx, double dy, double dz, const int bw[3],
                                 igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_heat_step");
    if (!T2 || !T || !Ci) fail(IGG_E_ARG, "igg_heat_step: NULL pointer array");
    igg::heat_step(g, T2, T, Ci, lam, dt, dx, dy, dz, bw, (cudaStream_t)stream);
    IGG_CATCH
}

namespace igg {
using RegionFn = std::function<void(int lr, const int lo[3], const int hi[3], cudaStream_t st)>;

// @hide_communication bw begin <step>; update_halo!(fields) end for any stencil given as a
// box callback: the six boundary slabs of [1, n-1)^3 first on
// the high-priority comm stream, the exchange behind them there, the inner box concurrently on the
// low-priority stream; both joined to s.
static void hide_comm(igg_grid *g, const int bw_in[3], const RegionFn &fn, const igg_field *fields, int nfields,
                      cudaStream_t s, const char *who, int x_align = 1) {
    const int zero[3] = {0, 0, 0};
    const int *bw = bw_in ? bw_in : zero;
    bool exch[3] = {false, false, false};
    for (int a = 0; a < 3; ++a)
        for (int lr = 0; lr < g->nlocal; ++lr)
            if (g->nbr[lr][a][0] >= 0 || g->nbr[lr][a][1] >= 0) exch[a] = true;
    const bool seq = bw[0] == 0 && bw[1] == 0 && bw[2] == 0;
    int lo[3], hi[3];
    bool degenerate = false;
    for (int a = 0; a < 3; ++a) {
        if (bw[a] < 0) fail(IGG_E_ARG, std::string(who) + ": negative boundary width");
        if (!seq && exch[a])
            for (int f = 0; f < nfields; ++f) {
                HaloSpec hs;
                if (!halo_spec(g->n[a], g->o[a], fields[f].size[a], &hs))
                    fail(IGG_E_STAGGER, std::string(who) + ": field size out of range");
                if (hs.h > 0 && bw[a] < hs.ol)
                    fail(IGG_E_WIDTH, std::string(who) + ": boundary width " + std::to_string(bw[a]) +
                                          " on axis " + std::to_string(a) + " is below a field overlap " +
                                          std::to_string(hs.ol));
            }
        const int b = exch[a] ? bw[a] : 0;
        lo[a] = std::max(1, b);
        hi[a] = std::min(g->n[a] - 1, g->n[a] - b);
        if (a == 0 && exch[0] && x_align > 1) {
            // x-boundaries on whole row segments of the caller's tile (as heat_step's x_align): the
            // boundary phase grows, every cell is still computed exactly once
            lo[0] = ((lo[0] + x_align - 1) / x_align) * x_align;
            hi[0] = (hi[0] / x_align) * x_align;
        }
        if (g->n[a] == 1) {   // a size-1 axis (1-D/2-D grid): its one layer, no slabs along it
            lo[a] = 0;
            hi[a] = 1;
        }
        if (hi[a] <= lo[a]) degenerate = true;
    }
    // the computed box per axis: inner layers, or the one layer of a size-1 axis
    int L[3], H[3];
    for (int a = 0; a < 3; ++a) {
        L[a] = g->n[a] == 1 ? 0 : 1;
        H[a] = g->n[a] == 1 ? 1 : g->n[a] - 1;
    }
    const int full_lo[3] = {L[0], L[1], L[2]}, full_hi[3] = {H[0], H[1], H[2]};
    IGG_CUDA(cudaEventRecord(g->ev_start, s));
    IGG_CUDA(cudaStreamWaitEvent(g->s_comm, g->ev_start, 0));
    if (seq || degenerate) {
        for (int lr = 0; lr < g->nlocal; ++lr) fn(lr, full_lo, full_hi, g->s_comm);
        exchange(g, fields, nfields, g->s_comm);
        IGG_CUDA(cudaEventRecord(g->ev_comm, g->s_comm));
        IGG_CUDA(cudaStreamWaitEvent(s, g->ev_comm, 0));
        return;
    }
    IGG_CUDA(cudaStreamWaitEvent(g->s_inner, g->ev_start, 0));
    // the six slabs x-lo, x-hi, y-lo, y-hi, z-lo, z-hi, each cell exactly once
    const int slab[6][6] = {{L[0], lo[0], L[1], H[1], L[2], H[2]},       {hi[0], H[0], L[1], H[1], L[2], H[2]},
                            {lo[0], hi[0], L[1], lo[1], L[2], H[2]},     {lo[0], hi[0], hi[1], H[1], L[2], H[2]},
                            {lo[0], hi[0], lo[1], hi[1], L[2], lo[2]},   {lo[0], hi[0], lo[1], hi[1], hi[2], H[2]}};
    for (int lr = 0; lr < g->nlocal; ++lr)
        for (int k = 0; k < 6; ++k) {
            const int a0[3] = {slab[k][0], slab[k][2], slab[k][4]}, a1[3] = {slab[k][1], slab[k][3], slab[k][5]};
            if (a1[0] > a0[0] && a1[1] > a0[1] && a1[2] > a0[2]) fn(lr, a0, a1, g->s_comm);
        }
    for (int lr = 0; lr < g->nlocal; ++lr) fn(lr, lo, hi, g->s_inner);
    exchange(g, fields, nfields, g->s_comm);
    IGG_CUDA(cudaEventRecord(g->ev_comm, g->s_comm));
    IGG_CUDA(cudaEventRecord(g->ev_inner, g->s_inner));
    IGG_CUDA(cudaStreamWaitEvent(s, g->ev_comm, 0));
    IGG_CUDA(cudaStreamWaitEvent(s, g->ev_inner, 0));
}
}  // namespace igg

IGG_API igg_status igg_hide_communication(igg_grid *g, const int bw_in[3], igg_region_fn fn, void *user,
                                          const igg_field *fields, int nfields, igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_hide_communication");
    if (!fn || !fields || nfields < 1) fail(IGG_E_ARG, "igg_hide_communication: bad argument");
    igg::hide_comm(
        g, bw_in,
        [&](int lr, const int lo[3], const int hi[3], cudaStream_t st) { fn(user, lr, lo, hi, (igg_stream_t)st); },
        fields, nfields, (cudaStream_t)stream, "igg_hide_communication");
    IGG_CATCH
}

// second workload (acoustic.cu): compute_V under @hide_communication with
// update_halo!(Vx, Vy, Vz), then compute_P on every cell
IGG_API igg_status igg_acoustic_step(igg_grid *g, double *const *P, double *const *Vx, double *const *Vy,
                                     double *const *Vz, double dt, double rho, double K, double dx, double dy,
                                     double dz, const int bw[3], igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_acoustic_step");
    if (!P || !Vx || !Vy || !Vz) fail(IGG_E_ARG, "igg_acoustic_step: null field list");
    if (!(rho != 0.0) || !(dx != 0.0) || !(dy != 0.0) || !(dz != 0.0))
        fail(IGG_E_ARG, "igg_acoustic_step: rho and the spacings must be non-zero");
    for (int a = 0; a < 3; ++a)
        if (g->n[a] < 3) fail(IGG_E_ARG, "igg_acoustic_step: every local size must be >= 3");
    cudaStream_t s = (cudaStream_t)stream;
    igg::AcousticCoef c;
    const double adt = dt / rho;   // reading A2: cV_d = (dt/rho)/d_d, cP = dt*K, r_d = 1/d_d
    c.cV[0] = adt / dx;
    c.cV[1] = adt / dy;
    c.cV[2] = adt / dz;
    c.cP = dt * K;
    c.r[0] = 1.0 / dx;
    c.r[1] = 1.0 / dy;
    c.r[2] = 1.0 / dz;
    const long long n0 = g->n[0], n1 = g->n[1], n2 = g->n[2];
    std::vector<igg_field> fl(3 * g->nlocal);
    std::vector<igg::AcousticFields> af(g->nlocal);
    for (int lr = 0; lr < g->nlocal; ++lr) {
        if (!P[lr] || !Vx[lr] || !Vy[lr] || !Vz[lr]) fail(IGG_E_ARG, "igg_acoustic_step: null field pointer");
        fl[3 * lr + 0] = igg_field{Vx[lr], {n0 + 1, n1, n2}};
        fl[3 * lr + 1] = igg_field{Vy[lr], {n0, n1 + 1, n2}};
        fl[3 * lr + 2] = igg_field{Vz[lr], {n0, n1, n2 + 1}};
        af[lr] = igg::AcousticFields{P[lr], Vx[lr], Vy[lr], Vz[lr], {g->n[0], g->n[1], g->n[2]}};
    }
    // the velocity cells are [1, n) per axis: a box ending at n-1 (the stencil box's end) extends to n
    igg::hide_comm(
        g, bw,
        [&](int lr, const int lo[3], const int hi[3], cudaStream_t st) {
            int h[3];
            bool full = true;
            for (int a = 0; a < 3; ++a) {
                h[a] = hi[a] == g->n[a] - 1 ? g->n[a] : hi[a];
                full = full && lo[a] == 1 && h[a] == g->n[a];
            }
            // OPT_PROFILE brackets the main velocity launch (the inner box, or the whole box)
            const bool main_box = st == g->s_inner || full;
            if (main_box) igg::prof_begin(g, st);
            igg::launch_acoustic_v(af[lr], c, lo, h, st);
            if (main_box)
                igg::prof_end(g, st, (long long)(h[0] - lo[0]) * (h[1] - lo[1]) * (h[2] - lo[2]));
            g->launches++;
        },
        fl.data(), 3, s, "igg_acoustic_step");
    for (int lr = 0; lr < g->nlocal; ++lr) {
        igg::launch_acoustic_p(af[lr], c, s);
        g->launches++;
    }
    IGG_CATCH
}

// nt leapfrog steps of the second workload with double-buffered fields (verdict r1 8b):
// F = [P, Vx, Vy, Vz, P2, Vx2, Vy2, Vz2] x local_ranks pointers (field-major).  A grid without any exchanged
// axis runs ONE fused V+P sweep per step from the current set into the other (64 B/cell instead of 96) and
// swaps the sets; otherwise every step is igg_acoustic_step on the current set in place.  On return
// F[0..3] hold the state after nt steps.
IGG_API igg_status igg_acoustic_run(igg_grid *g, double **F, int nt, double dt, double rho, double K, double dx,
                                    double dy, double dz, const int bw[3], igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_acoustic_run");
    if (!F || nt < 0) fail(IGG_E_ARG, "igg_acoustic_run: bad argument");
    const int L = g->nlocal;
    for (int q = 0; q < 8 * L; ++q)
        if (!F[q]) fail(IGG_E_ARG, "igg_acoustic_run: NULL field pointer");
    bool exch = false;
    for (int a = 0; a < 3; ++a)
        for (int lr = 0; lr < L; ++lr) exch = exch || g->nbr[lr][a][0] >= 0 || g->nbr[lr][a][1] >= 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (exch) {
        for (int it = 0; it < nt; ++it) {
            const igg_status st = igg_acoustic_step(g, F, F + L, F + 2 * L, F + 3 * L, dt, rho, K, dx, dy, dz, bw, stream);
            if (st != IGG_OK) return st;
        }
        return IGG_OK;
    }
    if (!(rho != 0.0) || !(dx != 0.0) || !(dy != 0.0) || !(dz != 0.0))
        fail(IGG_E_ARG, "igg_acoustic_run: rho and the spacings must be non-zero");
    for (int a = 0; a < 3; ++a)
        if (g->n[a] < 3) fail(IGG_E_ARG, "igg_acoustic_run: every local size must be >= 3");
    igg::AcousticCoef c;
    const double adt = dt / rho;   // reading A2 (as igg_acoustic_step)
    c.cV[0] = adt / dx;
    c.cV[1] = adt / dy;
    c.cV[2] = adt / dz;
    c.cP = dt * K;
    c.r[0] = 1.0 / dx;
    c.r[1] = 1.0 / dy;
    c.r[2] = 1.0 / dz;
    for (int it = 0; it < nt; ++it) {
        for (int lr = 0; lr < L; ++lr) {
            const igg::AcousticFields in{F[lr], F[L + lr], F[2 * L + lr], F[3 * L + lr], {g->n[0], g->n[1], g->n[2]}};
            const igg::AcousticFields out{F[4 * L + lr], F[5 * L + lr], F[6 * L + lr], F[7 * L + lr],
                                          {g->n[0], g->n[1], g->n[2]}};
            igg::prof_begin(g, s);
            igg::launch_acoustic_fused(in, out, c, s);
            igg::prof_end(g, s, (long long)g->n[0] * g->n[1] * g->n[2]);
            g->launches++;
        }
        for (int q = 0; q < 4 * L; ++q) std::swap(F[q], F[4 * L + q]);
    }
    IGG_CATCH
}

namespace igg {
// one binary32 step (igg_heat_step_f32); wait_prev / drain as heat_step (pipelining inside
// igg_heat_run_f32 on the fused path)
static void heat_step_f32(igg_grid *g, float *const *T2, const float *const *T, const float *const *Ci, float lam,
                          float dt, float dx, float dy, float dz, const int bw[3], cudaStream_t s, bool wait_prev,
                          bool drain) {
    if (!T2 || !T || !Ci) fail(IGG_E_ARG, "igg_heat_step_f32: NULL field list");
    for (int a = 0; a < 3; ++a)
        if (g->n[a] == 2) fail(IGG_E_ARG, "igg_heat_step_f32: an axis needs 1 or at least 3 cells");
    std::vector<igg_field> f(g->nlocal);
    bool aligned = true;
    for (int lr = 0; lr < g->nlocal; ++lr) {
        if (!T2[lr] || !T[lr] || !Ci[lr]) fail(IGG_E_ARG, "igg_heat_step_f32: NULL field pointer");
        f[lr] = igg_field{reinterpret_cast<double *>(T2[lr]), {g->n[0], g->n[1], g->n[2]}, 4};
        aligned = aligned && ((reinterpret_cast<uintptr_t>(T2[lr]) | reinterpret_cast<uintptr_t>(T[lr]) |
                               reinterpret_cast<uintptr_t>(Ci[lr])) % 16 == 0);
    }
    const HeatCoefF k = heat_coef_f32(lam, dt, dx, dy, dz);
    // the fused stencil + exchange kernel in binary32 (float4 lanes: 128-cell tile rows), as the binary64
    // step: P2P path, a 3-D grid with an exchanged axis, a hide_communication schedule requested with widths
    // covering the overlap; rows of whole 16-B vectors and two x tiles at least (the x faces in different tiles)
    // (auto: when only the x axis is exchanged -- 2 GPUs, 2x1x1 at 512^3: 0.280 ms fused vs 0.287 ms split;
    // with y or z exchanged too the float4 box kernel's split schedule is faster: 2x2x1 0.2875 vs 0.2917 ms)
    const bool seq = !bw || (bw[0] == 0 && bw[1] == 0 && bw[2] == 0);
    bool xex = false, yzex = false;
    for (int lr = 0; lr < g->nlocal; ++lr) {
        xex = xex || g->nbr[lr][0][0] >= 0 || g->nbr[lr][0][1] >= 0;
        for (int a = 1; a < 3; ++a) yzex = yzex || g->nbr[lr][a][0] >= 0 || g->nbr[lr][a][1] >= 0;
    }
    const bool want = g->fused_f32 > 0 || (g->fused_f32 < 0 && xex && !yzex);
    if (want && !seq && g->stencil_kernel == 0 && aligned && g->n[0] % 4 == 0 && g->n[0] >= 130 &&
        fused_eligible(g)) {
        for (int a = 0; a < 3; ++a) {
            bool ex = false;
            for (int lr = 0; lr < g->nlocal; ++lr) ex = ex || g->nbr[lr][a][0] >= 0 || g->nbr[lr][a][1] >= 0;
            if (ex && bw[a] < g->o[a])
                fail(IGG_E_WIDTH, "heat_step: boundary width " + std::to_string(bw[a]) + " on axis " +
                                      std::to_string(a) + " is below the field overlap " + std::to_string(g->o[a]));
        }
        fused_step_f32(g, T2, T, Ci, k, s, wait_prev, drain);
        return;
    }
    // @hide_communication bw: boundary slabs, then update_halo!(T2) on the comm stream
    // behind them, the inner box concurrently; bw = 0 (or NULL) is the sequential schedule.  With an
    // exchanged x axis the x slabs cut every row into 15 + inner + 15 cells, which costs more than the
    // exposed exchange (2x1x1 at 512^3: 0.306 ms hidden vs 0.287 ms sequential), so the
    // step runs sequentially there (same cells, same result); fused_mode bit 16384 keeps the slabs.
    const int zero[3] = {0, 0, 0};
    const int *bw_eff = (xex && !(g->fused_mode & 16384)) ? zero : bw;
    igg::hide_comm(
        g, bw_eff,
        [&](int lr, const int lo[3], const int hi[3], cudaStream_t st) {
            bool full = true;
            for (int a = 0; a < 3; ++a) full = full && lo[a] == (g->n[a] > 1 ? 1 : 0);
            const bool main_box = st == g->s_inner || full;   // OPT_PROFILE: the inner (or whole) box
            if (main_box) igg::prof_begin(g, st);
            igg::launch_heat_f32(T2[lr], T[lr], Ci[lr], g->n, lo, hi, k, st, g->stencil_kernel);
            if (main_box)
                igg::prof_end(g, st, (long long)(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]));
            g->launches++;
        },
        f.data(), 1, s, "igg_heat_step_f32",
        // exact bw in x: growing the x slabs to whole 512-B segments (128 binary32 cells) measured
        // slower on a 2x1x1 split (0.313 vs 0.306 ms/step, profiles/r01_f32_scaling.txt); fused_mode
        // bit 8192 restores it for the ablation
        (g->fused_mode & 8192) ? 128 : 1);
}
}  // namespace igg

IGG_API igg_status igg_heat_step_f32(igg_grid *g, float *const *T2, const float *const *T, const float *const *Ci,
                                     float lam, float dt, float dx, float dy, float dz, const int bw[3],
                                     igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_heat_step_f32");
    igg::heat_step_f32(g, T2, T, Ci, lam, dt, dx, dy, dz, bw, (cudaStream_t)stream, false, true);
    IGG_CATCH
}

IGG_API igg_status igg_heat_run_f32(igg_grid *g, float **T, float **T2, const float *const *Ci, float lam, float dt,
                                    float dx, float dy, float dz, int nt, const int bw[3], igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_heat_run_f32");
    if (!T || !T2 || !Ci || nt < 0) fail(IGG_E_ARG, "igg_heat_run_f32: bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    igg::validate_peer_maps(g);   // collective: every cached peer mapping still names a live allocation
    for (int it = 0; it < nt; ++it) {
        igg::heat_step_f32(g, T2, T, Ci, lam, dt, dx, dy, dz, bw, s, it > 0, it == nt - 1);
        for (int lr = 0; lr < g->nlocal; ++lr) std::swap(T[lr], T2[lr]);
    }
    IGG_CATCH
}

IGG_API igg_status igg_heat_run(igg_grid *g, double **T, double **T2, const double *const *Ci, double lam,
                                double dt, double dx, double dy, double dz, int nt, const int bw[3],
                                igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_heat_run");
    if (!T || !T2 || !Ci || nt < 0) fail(IGG_E_ARG, "igg_heat_run: bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    igg::validate_peer_maps(g);   // collective: every cached peer mapping still names a live allocation
    for (int it = 0; it < nt; ++it) {
        // consecutive steps pipelined on the fused path (the previous step's faces awaited tile by
        // tile); the last one drains, so the run is complete on the stream like nt single steps
        igg::heat_step(g, T2, T, Ci, lam, dt, dx, dy, dz, bw, s, it > 0, it == nt - 1);
        for (int lr = 0; lr < g->nlocal; ++lr) std::swap(T[lr], T2[lr]);   // T, T2 = T2, T
    }
    IGG_CATCH
}

IGG_API igg_status igg_heat_run_host(igg_grid *g, double *T_host, const double *Ci_host, double lam, double dt,
                                     double dx, double dy, double dz, int nt, const int bw[3], igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_heat_run_host");
    if (!T_host || !Ci_host || nt < 0) fail(IGG_E_ARG, "igg_heat_run_host: bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t cells = (size_t)g->n[0] * g->n[1] * g->n[2];
    const size_t bytes = cells * g->nlocal * sizeof(double);
    igg::validate_peer_maps(g);
    if (bytes > g->run_bytes) {
        // the scratch arrays may be mapped by the peers (fused path): drop every mapping first
        // (collective: every process grows its scratch on the same call)
        if (g->run_T) igg::release_peer_maps(g);
        for (double *p : {g->run_T, g->run_T2, g->run_Ci})
            if (p) IGG_CUDA(cudaFree(p));
        g->run_T = (double *)igg::dev_alloc(g, bytes);
        g->run_T2 = (double *)igg::dev_alloc(g, bytes);
        g->run_Ci = (double *)igg::dev_alloc(g, bytes);
        g->run_bytes = bytes;
    }
    IGG_CUDA(cudaMemcpyAsync(g->run_T, T_host, bytes, cudaMemcpyHostToDevice, s));
    IGG_CUDA(cudaMemcpyAsync(g->run_Ci, Ci_host, bytes, cudaMemcpyHostToDevice, s));
    std::vector<double *> a(g->nlocal), b(g->nlocal);
    std::vector<const double *> c(g->nlocal);
    for (int lr = 0; lr < g->nlocal; ++lr) {
        a[lr] = g->run_T + lr * cells;
        b[lr] = g->run_T2 + lr * cells;
        c[lr] = g->run_Ci + lr * cells;
        igg::launch_copy_outer(b[lr], a[lr], g->n, s);   // T2 = copy(T) on the cells no step writes first
        g->launches++;
    }
    for (int it = 0; it < nt; ++it) {
        std::vector<const double *> ac(a.begin(), a.end());
        igg::heat_step(g, b.data(), ac.data(), c.data(), lam, dt, dx, dy, dz, bw, s, it > 0, it == nt - 1);
        std::swap(a, b);   // T, T2 = T2, T
    }
    for (int lr = 0; lr < g->nlocal; ++lr)
        IGG_CUDA(cudaMemcpyAsync(T_host + lr * cells, a[lr], cells * sizeof(double), cudaMemcpyDeviceToHost, s));
    IGG_CUDA(cudaStreamSynchronize(s));
    igg::check_device_error(g, "igg_heat_run_host");   // a timed-out flag wait invalidates the result
    IGG_CATCH
}

// ------------------------------------------------------------------ gather
namespace igg {
// owned layers [lo, hi) of a rank at axis coordinate c for a field of size s: interior ranks own
// [h + ol%2, s - h); the first rank also owns the lower halo layers, the last the upper ones;
// a shared middle layer (odd field overlap) belongs to the lower rank.  Periodic axes: every rank
// is interior.  Global index of local layer l: c(n-o) + l (periodic: shifted by o/2 mod the period).
static void owned_range(const igg_grid *g, int a, int c, long long s, int *lo, int *hi) {
    HaloSpec hs;
    halo_spec(g->n[a], g->o[a], s, &hs);
    const bool first = !g->periods[a] && c == 0, last = !g->periods[a] && c == g->dims[a] - 1;
    *lo = first ? 0 : hs.h + (hs.ol % 2);
    *hi = last ? (int)s : (int)s - hs.h;
}
}  // namespace igg

IGG_API igg_status igg_gather(igg_grid *g, const igg_field *fields, int root_proc, double *host_out,
                              igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_gather");
    if (!fields || root_proc < 0 || root_proc >= g->nproc_procs) fail(IGG_E_ARG, "igg_gather: bad argument");
    for (int lr = 0; lr < g->nlocal; ++lr)
        if (fields[lr].elsize != 0 && fields[lr].elsize != 8)
            fail(IGG_E_UNSUPPORTED, "igg_gather: binary64 fields only");
    cudaStream_t s = (cudaStream_t)stream;
    const long long sz[3] = {fields[0].size[0], fields[0].size[1], fields[0].size[2]};
    long long N[3];
    for (int a = 0; a < 3; ++a) {
        igg::HaloSpec hs;
        if (!igg::halo_spec(g->n[a], g->o[a], sz[a], &hs)) fail(IGG_E_STAGGER, "igg_gather: field size out of range");
        N[a] = g->periods[a] ? g->ng[a] : g->ng[a] + (sz[a] - g->n[a]);
    }
    const bool is_root = g->proc == root_proc;
    if (is_root && !host_out) fail(IGG_E_ARG, "igg_gather: host_out is NULL on the root");
    // boxes of every rank, in rank order
    struct Box {
        int b0[3], b1[3];
        long long count, off;
    };
    std::vector<Box> boxes(g->nprocs);
    long long total = 0;
    for (int r = 0; r < g->nprocs; ++r) {
        int c[3];
        igg::coords_of_rank(g->dims, r, c);
        Box &B = boxes[r];
        B.count = 1;
        for (int a = 0; a < 3; ++a) {
            igg::owned_range(g, a, c[a], sz[a], &B.b0[a], &B.b1[a]);
            B.count *= std::max(0, B.b1[a] - B.b0[a]);
        }
        B.off = total;
        total += B.count;
    }
    // pack my ranks' boxes into one device buffer (mine are contiguous in rank order)
    long long mine = 0, mine_off = boxes[g->rank0].off;
    for (int lr = 0; lr < g->nlocal; ++lr) mine += boxes[g->rank0 + lr].count;
    double *dbuf = nullptr;
    IGG_CUDA(cudaMalloc(&dbuf, sizeof(double) * (is_root ? total : std::max(mine, 1LL))));
    double *dst = dbuf + (is_root ? mine_off : 0);
    for (int lr = 0; lr < g->nlocal; ++lr) {
        const Box &B = boxes[g->rank0 + lr];
        igg::launch_box_pack(fields[lr].ptr, dst + (B.off - mine_off), sz[0], sz[1], B.b0, B.b1, s);
    }
    if (g->nproc_procs > 1 && g->boot) {
        // host bootstrap: every process' owned boxes through the all-gather (padded to the largest)
        long long maxc = 1;
        for (int p = 0; p < g->nproc_procs; ++p) {
            long long cnt = 0;
            for (int lr = 0; lr < g->nlocal; ++lr) cnt += boxes[p * g->nlocal + lr].count;
            maxc = std::max(maxc, cnt);
        }
        std::vector<double> hmine(maxc, 0.0);
        IGG_CUDA(cudaStreamSynchronize(s));
        if (mine) IGG_CUDA(cudaMemcpy(hmine.data(), dst, sizeof(double) * mine, cudaMemcpyDeviceToHost));
        std::vector<char> all = igg::allgather_bytes(g, hmine.data(), sizeof(double) * maxc);
        if (is_root)
            for (int p = 0; p < g->nproc_procs; ++p) {
                if (p == g->proc) continue;
                long long cnt = 0;
                for (int lr = 0; lr < g->nlocal; ++lr) cnt += boxes[p * g->nlocal + lr].count;
                if (cnt)
                    IGG_CUDA(cudaMemcpy(dbuf + boxes[p * g->nlocal].off, all.data() + sizeof(double) * maxc * p,
                                        sizeof(double) * cnt, cudaMemcpyHostToDevice));
            }
    } else if (g->nproc_procs > 1) {
        IGG_NCCL(ncclGroupStart());
        if (is_root) {
            for (int p = 0; p < g->nproc_procs; ++p) {
                if (p == g->proc) continue;
                long long cnt = 0;
                for (int lr = 0; lr < g->nlocal; ++lr) cnt += boxes[p * g->nlocal + lr].count;
                if (cnt) IGG_NCCL(ncclRecv(dbuf + boxes[p * g->nlocal].off, (size_t)cnt, ncclDouble, p, g->comm, s));
            }
        } else if (mine) {
            IGG_NCCL(ncclSend(dbuf, (size_t)mine, ncclDouble, root_proc, g->comm, s));
        }
        IGG_NCCL(ncclGroupEnd());
    }
    IGG_CUDA(cudaStreamSynchronize(s));
    if (is_root) {
        std::vector<double> h(total);
        IGG_CUDA(cudaMemcpy(h.data(), dbuf, sizeof(double) * total, cudaMemcpyDeviceToHost));
        for (int r = 0; r < g->nprocs; ++r) {
            const Box &B = boxes[r];
            int c[3];
            igg::coords_of_rank(g->dims, r, c);
            const int nx = B.b1[0] - B.b0[0], ny = B.b1[1] - B.b0[1], nz = B.b1[2] - B.b0[2];
            if (nx <= 0 || ny <= 0 || nz <= 0) continue;
            long long gl[3][1];
            (void)gl;
            // global index of local layer l on axis a
            auto gidx = [&](int a, int l) {
                long long v = (long long)c[a] * (g->n[a] - g->o[a]) + l;
                if (g->periods[a]) v = ((v - g->o[a] / 2) % N[a] + N[a]) % N[a];
                return v;
            };
            const double *src = h.data() + B.off;
            for (int z = 0; z < nz; ++z)
                for (int y = 0; y < ny; ++y) {
                    const long long gz = gidx(2, B.b0[2] + z), gy = gidx(1, B.b0[1] + y);
                    const double *row = src + ((long long)z * ny + y) * nx;
                    for (int x = 0; x < nx; ++x)
                        host_out[(gz * N[1] + gy) * N[0] + gidx(0, B.b0[0] + x)] = row[x];
                }
        }
    }
    IGG_CUDA(cudaFree(dbuf));
    IGG_CATCH
}

IGG_API igg_status igg_global_max(igg_grid *g, double local, double *out) {
    IGG_TRY
    igg::check_live(g, "igg_global_max");
    if (!out) fail(IGG_E_ARG, "igg_global_max: NULL out");
    if (g->boot) {   // host bootstrap: all-gather the local values, max on the host
        *out = igg::host_max(g, local);
        return IGG_OK;
    }
    double *d = g->d_scratch + igg::field_max_scratch_len();
    IGG_CUDA(cudaMemcpyAsync(d, &local, sizeof(double), cudaMemcpyHostToDevice, g->s_comm));
    if (g->nproc_procs > 1) IGG_NCCL(ncclAllReduce(d, d, 1, ncclDouble, ncclMax, g->comm, g->s_comm));
    IGG_CUDA(cudaMemcpyAsync(g->d_pinned_out, d, sizeof(double), cudaMemcpyDeviceToHost, g->s_comm));
    IGG_CUDA(cudaStreamSynchronize(g->s_comm));
    *out = *g->d_pinned_out;
    IGG_CATCH
}

IGG_API igg_status igg_field_global_max(igg_grid *g, const double *const *f, long long count, double *out,
                                        igg_stream_t stream) {
    IGG_TRY
    igg::check_live(g, "igg_field_global_max");
    if (!f || !out || count < 1) fail(IGG_E_ARG, "igg_field_global_max: bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    double *d = g->d_scratch + igg::field_max_scratch_len();
    igg::launch_field_max(f, g->nlocal, count, g->d_scratch, igg::field_max_scratch_len(), d, s);
    g->launches += 2;
    if (g->nproc_procs > 1 && g->comm) IGG_NCCL(ncclAllReduce(d, d, 1, ncclDouble, ncclMax, g->comm, s));
    IGG_CUDA(cudaMemcpyAsync(g->d_pinned_out, d, sizeof(double), cudaMemcpyDeviceToHost, s));
    IGG_CUDA(cudaStreamSynchronize(s));
    *out = g->boot ? igg::host_max(g, *g->d_pinned_out) : *g->d_pinned_out;
    IGG_CATCH
}

IGG_API igg_status igg_set_option(igg_grid *g, int key, long long value) {
    IGG_TRY
    igg::check_live(g, "igg_set_option");
    switch (key) {
        case IGG_OPT_SKIP_COMM:
            g->skip_comm = value != 0;
            g->skipped = g->skipped || g->skip_comm;
            break;
        case IGG_OPT_SPIN_TIMEOUT_MS: g->spin_timeout_ms = value; break;
        case IGG_OPT_STENCIL_KERNEL:
            if (!IGG_ABLATION && value != 0 && value != 1)
                fail(IGG_E_UNSUPPORTED, "igg_set_option: stencil variants are in the ablation build only");
            g->stencil_kernel = (int)value;
            break;
        case IGG_OPT_PROFILE: g->profile = (int)value; break;
        case IGG_OPT_X_ALIGN: g->x_align = (int)(value < 1 ? 1 : value); break;
        case IGG_OPT_SCHEDULE: g->schedule = (int)value; break;
        case IGG_OPT_FUSED: g->fused = (int)value; break;
        case IGG_OPT_FUSED_MODE:
            if (!IGG_ABLATION) fail(IGG_E_UNSUPPORTED, "igg_set_option: FUSED_MODE is in the ablation build only");
            g->fused_mode = (int)value;
            break;
        case IGG_OPT_HALO_STREAM: g->halo_on_caller = value != 0; break;
        case IGG_OPT_LOCAL_P2P: g->local_p2p = value != 0; break;
        case IGG_OPT_HALO26: g->halo26 = value != 0 ? 1 : 0; break;
        case IGG_OPT_FUSED_F32: g->fused_f32 = value < 0 ? -1 : value != 0 ? 1 : 0; break;
        case IGG_OPT_FUSED_COMM_CTAS:
            if (value < 1 || value > 128) fail(IGG_E_ARG, "igg_set_option: FUSED_COMM_CTAS must be in [1, 128]");
            g->fused_ncomm = (int)value;
            g->fused_key = -1;
            break;
        case IGG_OPT_FUSED_KC2:
            if (value < 0 || value > 64) fail(IGG_E_ARG, "igg_set_option: FUSED_KC2 must be in [0, 64]");
            g->fused_kc2 = (int)value;
            g->fused_key = -1;
            break;
        default: fail(IGG_E_ARG, "igg_set_option: unknown key " + std::to_string(key));
    }
    IGG_CATCH
}

IGG_API igg_status igg_profile_stencil(igg_grid *g, double *ms_total, long long *launches, long long *cells) {
    IGG_TRY
    igg::check_live(g, "igg_profile_stencil");
    IGG_CUDA(cudaDeviceSynchronize());
    double tot = 0.0;
    for (size_t i = 0; i + 1 < g->prof_used; i += 2) {
        float ms = 0.f;
        IGG_CUDA(cudaEventElapsedTime(&ms, g->prof_ev[i], g->prof_ev[i + 1]));
        tot += ms;
    }
    if (ms_total) *ms_total = tot;
    if (launches) *launches = (long long)(g->prof_used / 2);
    if (cells) *cells = g->prof_cells;
    g->prof_used = 0;
    g->prof_cells = 0;
    IGG_CATCH
}

IGG_API igg_status igg_profile_timeline(igg_grid *g, double out[5]) {
    IGG_TRY
    igg::check_live(g, "igg_profile_timeline");
    if (!out) fail(IGG_E_ARG, "igg_profile_timeline: NULL out");
    IGG_CUDA(cudaDeviceSynchronize());
    double acc[4] = {0, 0, 0, 0};
    const size_t nsteps = g->tl_used / 5;
    for (size_t st = 0; st < nsteps; ++st)
        for (int k = 1; k < 5; ++k) {
            float ms = 0.f;
            IGG_CUDA(cudaEventElapsedTime(&ms, g->tl_ev[st * 5], g->tl_ev[st * 5 + k]));
            acc[k - 1] += ms;
        }
    for (int k = 0; k < 4; ++k) out[k] = nsteps ? acc[k] / nsteps : 0.0;
    out[4] = (double)nsteps;
    g->tl_used = 0;
    IGG_CATCH
}

IGG_API igg_status igg_release_arrays(igg_grid *g) {
    IGG_TRY
    igg::check_live(g, "igg_release_arrays");
    igg::release_peer_maps(g);
    igg::release_h26(g);
    IGG_CATCH
}

IGG_API igg_status igg_check(igg_grid *g) {
    IGG_TRY
    igg::check_live(g, "igg_check");
    igg::check_device_error(g, "igg_check");
    if (g->skipped) {   // steps were taken with the exchange skipped (timing only): halos are invalid
        g->skipped = g->skip_comm;
        fail(IGG_E_STATE, "igg_check: steps ran with IGG_OPT_SKIP_COMM (timing only): halo values are invalid");
    }
    if (g->comm) {
        ncclResult_t r = ncclSuccess;
        IGG_NCCL(ncclCommGetAsyncError(g->comm, &r));
        if (r != ncclSuccess) fail(IGG_E_NCCL, std::string("igg_check: NCCL async error: ") + ncclGetErrorString(r));
    }
    IGG_CATCH
}
