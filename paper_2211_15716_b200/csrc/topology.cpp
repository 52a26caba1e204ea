// topology.cpp -- host-only grid math and the error channel of libigg.
//
// Readings of the paper ("implicit creation of the global
// computational grid based on the number of processes ... and based on the
// process topology, which can be explicitly chosen by the user or
// automatically defined"; PAPER.md:63-65 nx_g()) follow SPEC.md where the
// paper is silent; DESIGN.md lists them.
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "igg_internal.h"

namespace {
thread_local std::string g_last_error;
}  // namespace

namespace igg {

void set_error(const std::string &msg) { g_last_error = msg; }

[[noreturn]] void fail(igg_status code, const std::string &msg) {
    g_last_error = msg;
    throw IggException{code};
}

// minimal spread, ties to the lexicographically largest vector.
int dims_create(int nprocs, const int fixed[3], int out[3]) {
    if (nprocs < 1) return -1;
    bool found = false;
    int best[3] = {0, 0, 0};
    int best_spread = 0;
    for (int px = 1; px <= nprocs; ++px) {
        if (nprocs % px) continue;
        for (int py = 1; py <= nprocs / px; ++py) {
            if ((nprocs / px) % py) continue;
            int pz = nprocs / px / py;
            int d[3] = {px, py, pz};
            bool ok = true;
            for (int a = 0; a < 3; ++a)
                if (fixed && fixed[a] && fixed[a] != d[a]) ok = false;
            if (!ok) continue;
            int mx = d[0], mn = d[0];
            for (int a = 1; a < 3; ++a) {
                mx = d[a] > mx ? d[a] : mx;
                mn = d[a] < mn ? d[a] : mn;
            }
            int spread = mx - mn;
            bool better = !found || spread < best_spread ||
                          (spread == best_spread &&
                           (d[0] > best[0] || (d[0] == best[0] && (d[1] > best[1] || (d[1] == best[1] && d[2] > best[2])))));
            if (better) {
                found = true;
                best_spread = spread;
                std::memcpy(best, d, sizeof best);
            }
        }
    }
    if (!found) return -1;
    std::memcpy(out, best, sizeof best);
    return 0;
}

// rank = (cx*py + cy)*pz + cz
int rank_of_coords(const int dims[3], const int c[3]) { return (c[0] * dims[1] + c[1]) * dims[2] + c[2]; }

void coords_of_rank(const int dims[3], int rank, int c[3]) {
    c[0] = rank / (dims[1] * dims[2]);
    c[1] = (rank / dims[2]) % dims[1];
    c[2] = rank % dims[2];
}

// SPEC.md:97-98
long long global_size(int n, int o, int p, int periodic) {
    return periodic ? (long long)p * (n - o) : (long long)p * (n - o) + o;
}

// SPEC.md:186
bool halo_spec(int n, int o, long long s, HaloSpec *hs) {
    if (s < n - o || s > n + o) return false;
    int ol = (int)(s - (n - o));
    int h = ol / 2;
    hs->ol = ol;
    hs->h = h;
    hs->send_lo[0] = ol - h;        hs->send_lo[1] = ol;
    hs->recv_lo[0] = 0;             hs->recv_lo[1] = h;
    hs->send_up[0] = (int)s - ol;   hs->send_up[1] = (int)s - ol + h;
    hs->recv_up[0] = (int)s - h;    hs->recv_up[1] = (int)s;
    return true;
}

}  // namespace igg

// ============================================================== C ABI (host-only part)
IGG_API const char *igg_last_error(void) { return g_last_error.c_str(); }

IGG_API igg_status igg_dims_create(int nprocs, const int fixed[3], int dims_out[3]) {
    IGG_TRY
    if (!dims_out) igg::fail(IGG_E_ARG, "igg_dims_create: dims_out is NULL");
    if (nprocs < 1) igg::fail(IGG_E_ARG, "igg_dims_create: nprocs must be >= 1");
    if (igg::dims_create(nprocs, fixed, dims_out) != 0)
        igg::fail(IGG_E_ARG, "igg_dims_create: no factorisation of " + std::to_string(nprocs) +
                                 " honours the fixed entries");
    IGG_CATCH
}

IGG_API igg_status igg_rank_of_coords(const int dims[3], const int coords[3], int *rank_out) {
    IGG_TRY
    if (!dims || !coords || !rank_out) igg::fail(IGG_E_ARG, "igg_rank_of_coords: NULL argument");
    for (int a = 0; a < 3; ++a)
        if (dims[a] < 1 || coords[a] < 0 || coords[a] >= dims[a])
            igg::fail(IGG_E_ARG, "igg_rank_of_coords: coords out of bounds");
    *rank_out = igg::rank_of_coords(dims, coords);
    IGG_CATCH
}

IGG_API igg_status igg_coords_of_rank(const int dims[3], int rank, int coords_out[3]) {
    IGG_TRY
    if (!dims || !coords_out) igg::fail(IGG_E_ARG, "igg_coords_of_rank: NULL argument");
    for (int a = 0; a < 3; ++a)
        if (dims[a] < 1) igg::fail(IGG_E_ARG, "igg_coords_of_rank: dims must be >= 1");
    if (rank < 0 || rank >= dims[0] * dims[1] * dims[2])
        igg::fail(IGG_E_ARG, "igg_coords_of_rank: rank out of bounds");
    igg::coords_of_rank(dims, rank, coords_out);
    IGG_CATCH
}

IGG_API igg_status igg_global_size(int n, int o, int p, int periodic, long long *out) {
    IGG_TRY
    if (!out) igg::fail(IGG_E_ARG, "igg_global_size: out is NULL");
    if (n <= o || o < 0 || p < 1) igg::fail(IGG_E_ARG, "igg_global_size: need n > o >= 0 and p >= 1");
    *out = igg::global_size(n, o, p, periodic);
    IGG_CATCH
}

IGG_API igg_status igg_halo_spec_of(int n, int o, long long s, igg_halo_spec *out) {
    IGG_TRY
    if (!out) igg::fail(IGG_E_ARG, "igg_halo_spec_of: out is NULL");
    igg::HaloSpec hs;
    if (!igg::halo_spec(n, o, s, &hs))
        igg::fail(IGG_E_STAGGER, "igg_halo_spec_of: field size " + std::to_string(s) + " outside [" +
                                     std::to_string(n - o) + ", " + std::to_string(n + o) + "]");
    out->ol = hs.ol;
    out->h = hs.h;
    for (int i = 0; i < 2; ++i) {
        out->send_lower[i] = hs.send_lo[i];
        out->recv_lower[i] = hs.recv_lo[i];
        out->send_upper[i] = hs.send_up[i];
        out->recv_upper[i] = hs.recv_up[i];
    }
    IGG_CATCH
}
