// plan.cpp -- host-only geometry validation and the update_halo exchange plan.
//
// The plan is the whole host logic of update_halo! for one
// process: which layers of which field go to which rank over which transport,
// where each face lands in the receiver's buffer pool, and the posting order
// of NCCL messages.  grid.cpp executes it with kernels and NCCL; the C ABI
// exports it (igg_plan_update_halo) so that multi-process host logic can be
// tested without a GPU.
#include <algorithm>
#include <cstring>
#include <tuple>

#include "igg_internal.h"

namespace igg {

Geom make_geom(const igg_init_args *A) {
    if (!A) fail(IGG_E_ARG, "init: args is NULL");
    Geom g{};
    const int n[3] = {A->nx, A->ny, A->nz};
    for (int a = 0; a < 3; ++a) {
        g.n[a] = n[a];
        g.o[a] = A->overlaps[a] == 0 ? 2 : A->overlaps[a];
        g.periods[a] = A->periods[a] ? 1 : 0;
        if (g.o[a] < 2 || g.o[a] % 2)
            fail(IGG_E_ARG, "init: overlap must be even and >= 2 (axis " + std::to_string(a) + ")");
        if (n[a] == 1) {   // a 1-D/2-D grid: a size-1 axis, one process along it, no halo
            if (g.periods[a]) fail(IGG_E_ARG, "init: a size-1 axis cannot be periodic (axis " + std::to_string(a) + ")");
            continue;
        }
        if (n[a] <= g.o[a])
            fail(IGG_E_ARG, "init: local size " + std::to_string(n[a]) + " must exceed the overlap " +
                                std::to_string(g.o[a]) + " (axis " + std::to_string(a) + ")");
    }
    if (A->nprocs < 1 || A->local_ranks < 1 || A->nprocs % A->local_ranks || A->rank0 < 0 ||
        A->rank0 >= A->nprocs || A->rank0 % A->local_ranks)
        fail(IGG_E_ARG, "init: inconsistent nprocs/rank0/local_ranks");
    if (A->path != IGG_PATH_NCCL && A->path != IGG_PATH_P2P) fail(IGG_E_ARG, "init: unknown path");
    int d[3] = {A->dims[0], A->dims[1], A->dims[2]};
    for (int a = 0; a < 3; ++a) {
        if (n[a] == 1 && d[a] == 0) d[a] = 1;   // a size-1 axis is never split
        if (n[a] == 1 && d[a] != 1) fail(IGG_E_ARG, "init: a size-1 axis must have dims 1 (axis " + std::to_string(a) + ")");
    }
    if (d[0] == 0 || d[1] == 0 || d[2] == 0) {   // automatic topology
        if (dims_create(A->nprocs, d, d) != 0) fail(IGG_E_ARG, "init: no topology honours the given dims");
    }
    if (d[0] < 1 || d[1] < 1 || d[2] < 1 || (long long)d[0] * d[1] * d[2] != A->nprocs)
        fail(IGG_E_ARG, "init: dims product != nprocs");
    std::memcpy(g.dims, d, sizeof d);
    g.nprocs = A->nprocs;
    g.nlocal = A->local_ranks;
    g.rank0 = A->rank0;
    g.nproc_procs = A->nprocs / A->local_ranks;
    g.proc = A->rank0 / A->local_ranks;
    g.device = A->device;
    g.path = A->path;
    for (int a = 0; a < 3; ++a) g.ng[a] = global_size(g.n[a], g.o[a], g.dims[a], g.periods[a]);
    for (int lr = 0; lr < g.nlocal; ++lr) {
        int c[3];
        coords_of_rank(g.dims, g.rank0 + lr, c);
        g.coords.push_back({c[0], c[1], c[2]});
        std::array<std::array<int, 2>, 3> nb;
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < 2; ++k) {   // SPEC.md:59 neighbours, periodic wrap, p=1 self
                int cc[3] = {c[0], c[1], c[2]};
                cc[a] += k == 0 ? -1 : 1;
                if (cc[a] < 0 || cc[a] >= g.dims[a]) {
                    if (!g.periods[a]) {
                        nb[a][k] = -1;
                        continue;
                    }
                    cc[a] = (cc[a] + g.dims[a]) % g.dims[a];
                }
                nb[a][k] = rank_of_coords(g.dims, cc);
            }
        g.nbr.push_back(nb);
    }
    return g;
}

Plan build_plan(const Geom &G, const long long *sizes, int nf, const int *esz) {
    if (nf < 1) fail(IGG_E_ARG, "update_halo: need at least one field");
    if (!sizes) fail(IGG_E_ARG, "update_halo: sizes is NULL");
    Plan P;
    const int L = G.nlocal;
    std::vector<std::array<HaloSpec, 3>> hs(nf);
    P.sz.resize(nf);
    for (int f = 0; f < nf; ++f)
        for (int a = 0; a < 3; ++a) {
            P.sz[f][a] = sizes[f * 3 + a];
            if (!halo_spec(G.n[a], G.o[a], P.sz[f][a], &hs[f][a]))
                fail(IGG_E_STAGGER, "update_halo: field " + std::to_string(f) + " axis " + std::to_string(a) +
                                        " size " + std::to_string(P.sz[f][a]) + " outside [" +
                                        std::to_string(G.n[a] - G.o[a]) + ", " + std::to_string(G.n[a] + G.o[a]) +
                                        "]");
        }
    // receive-slot layout of one rank: [field][axis][side]; face = h * (other two sizes)
    std::vector<std::array<std::array<long long, 2>, 3>> off(nf);
    std::vector<std::array<long long, 3>> face(nf), words(nf);
    long long block = 0;
    for (int f = 0; f < nf; ++f)
        for (int a = 0; a < 3; ++a) {
            long long other = 1;
            for (int b = 0; b < 3; ++b)
                if (b != a) other *= P.sz[f][b];
            face[f][a] = hs[f][a].h * other;
            const long long e = esz ? esz[f] : 8;
            words[f][a] = (face[f][a] * e + 7) / 8;   // slots in 8-byte words (binary32 faces packed)
            for (int side = 0; side < 2; ++side) {
                off[f][a][side] = block;
                block += words[f][a];
            }
        }
    P.block = block;
    P.off = off;
    for (int a = 0; a < 3; ++a) {   // x -> y -> z
        std::vector<PlanMsg> packs, unpacks;
        for (int lr = 0; lr < L; ++lr)
            for (int f = 0; f < nf; ++f) {
                const HaloSpec &H = hs[f][a];
                if (H.h == 0) continue;   // ol < 2: nothing exchanged on this axis
                // k = 0: my send_upper -> upper neighbour's recv_lower (receiver side 0)
                // k = 1: my send_lower -> lower neighbour's recv_upper (receiver side 1)
                for (int k = 0; k < 2; ++k) {
                    const int nb = G.nbr[lr][a][k == 0 ? 1 : 0];
                    if (nb < 0) continue;
                    PlanMsg m{};
                    m.op = 0;
                    m.lr = lr;
                    m.field = f;
                    m.recv_side = k;
                    m.peer = nb;
                    m.peer_proc = nb / L;
                    m.peer_lr = nb - m.peer_proc * L;
                    m.transport = m.peer_proc == G.proc ? kLocal : (G.path == IGG_PATH_P2P ? kP2P : kNccl);
                    m.lo = k == 0 ? H.send_up[0] : H.send_lo[0];
                    m.h = H.h;
                    m.count = face[f][a];
                    m.words = words[f][a];
                    m.slot = (long long)m.peer_lr * block + off[f][a][k];
                    m.sbuf = (long long)lr * block + off[f][a][k];
                    m.order = -1;
                    packs.push_back(m);
                }
                for (int side = 0; side < 2; ++side) {
                    const int nb = G.nbr[lr][a][side];
                    if (nb < 0) continue;
                    PlanMsg m{};
                    m.op = 1;
                    m.lr = lr;
                    m.field = f;
                    m.recv_side = side;
                    m.peer = nb;
                    m.peer_proc = nb / L;
                    m.peer_lr = nb - m.peer_proc * L;
                    m.transport = m.peer_proc == G.proc ? kLocal : (G.path == IGG_PATH_P2P ? kP2P : kNccl);
                    m.lo = side == 0 ? H.recv_lo[0] : H.recv_up[0];
                    m.h = H.h;
                    m.count = face[f][a];
                    m.words = words[f][a];
                    m.slot = (long long)lr * block + off[f][a][side];
                    m.sbuf = -1;
                    m.order = -1;
                    unpacks.push_back(m);
                }
            }
        // NCCL has no tags: sends/recvs between a process pair match in posting
        // order, so both ends post in one canonical order, keyed by
        // (sending rank, receiving rank, field, receiver side) (reading 17)
        auto key = [&](const PlanMsg &m) {
            const int me = G.rank0 + m.lr;
            return m.op == 0 ? std::make_tuple(me, m.peer, m.field, m.recv_side)
                             : std::make_tuple(m.peer, me, m.field, m.recv_side);
        };
        for (int op = 0; op < 2; ++op) {
            std::vector<PlanMsg> &v = op == 0 ? packs : unpacks;
            std::vector<int> idx;
            for (int i = 0; i < (int)v.size(); ++i)
                if (v[i].transport == kNccl) idx.push_back(i);
            std::sort(idx.begin(), idx.end(), [&](int x, int y) { return key(v[x]) < key(v[y]); });
            for (int j = 0; j < (int)idx.size(); ++j) v[idx[j]].order = j;
            if (!idx.empty()) P.any_nccl = true;
        }
        P.msgs[a] = packs;
        P.msgs[a].insert(P.msgs[a].end(), unpacks.begin(), unpacks.end());
    }
    return P;
}

}  // namespace igg

IGG_API igg_status igg_plan_update_halo(const igg_init_args *args, const long long *sizes, int nfields,
                                        igg_plan_entry *out, int capacity, int *count) {
    IGG_TRY
    if (!count) igg::fail(IGG_E_ARG, "igg_plan_update_halo: count is NULL");
    igg::Geom G = igg::make_geom(args);
    igg::Plan P = igg::build_plan(G, sizes, nfields);
    int k = 0;
    for (int a = 0; a < 3; ++a)
        for (const igg::PlanMsg &m : P.msgs[a]) {
            if (out && k < capacity) {
                igg_plan_entry &e = out[k];
                e.axis = a;
                e.op = m.op;
                e.local_rank = m.lr;
                e.field = m.field;
                e.recv_side = m.recv_side;
                e.peer = m.peer;
                e.transport = m.transport;
                e.lo = m.lo;
                e.h = m.h;
                e.count = m.count;
                e.order = m.order;
            }
            ++k;
        }
    *count = k;
    if (out && k > capacity) igg::fail(IGG_E_ARG, "igg_plan_update_halo: capacity too small");
    IGG_CATCH
}
