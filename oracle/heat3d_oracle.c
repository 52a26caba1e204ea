/*
 * oracle/heat3d_oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this file's library.  The product path
 * (paper_2211_15716_b200/, include/, csrc/) never includes, links or calls it,
 * and this file includes nothing from the product.
 *
 * What it computes: the plain, single-process, single-array definition of the
 * paper's 3-D heat-diffusion solver on the WHOLE global grid (no halos, no
 * decomposition, no overlap):
 *
 *   PAPER.md:45-51 (Fig. 1, listing lines 6-12)
 *     @inn(T2) = @inn(T) + dt*( lam*@inn(Ci)*(@d2_xi(T)/dx^2 +
 *                                            @d2_yi(T)/dy^2 +
 *                                            @d2_zi(T)/dz^2 ) )
 *   PAPER.md:74-80 (listing 35-41): for it = 1:nt ... T, T2 = T2, T
 *   PAPER.md:68-70 (listing 29-31): T2 = copy(T)
 *
 * Readings:
 *   - @d2_xi(T)  = (T[i+1]-T[i]) - (T[i]-T[i-1])                (reading 6)
 *   - dx^2 = dx*dx; Julia evaluates a*b*c as (a*b)*c and a+b+c as (a+b)+c,
 *     so the literal form is
 *       T + dt*((lam*Ci)*(((d2x/(dx*dx)) + (d2y/(dy*dy))) + (d2z/(dz*dz))))
 *                                                                (reading 7)
 *   - "canonical" mode replaces /(d*d) by *r_d with r_d = 1.0/(d*d) computed
 *     once (reading 9); every other operation and its order is unchanged.
 *   - Non-periodic axes: only cells 1..N-2 are updated; the two outer layers
 *     keep their initial value (Dirichlet by initialisation, reading 10).
 *   - Periodic axes: every cell 0..N-1 is updated with neighbours mod N
 *     (reading 11 / SPEC.md:98).
 *   - IEEE binary64, round to nearest even, compiled with -ffp-contract=off
 *     (no FMA contraction) and without -ffast-math (reading 8).
 *   - 1-D/2-D grids are 3-D grids with size-1 axes: an axis with
 *     N == 1 has no second difference (its term is absent from the sum, the
 *     others keep their x, y, z order) and its single layer is updated
 *     (reading 23).
 *
 * Layout: x fastest: index(x,y,z) = (z*Ny + y)*Nx + x.
 * OpenMP (if compiled with -fopenmp) splits the z loop only; it never changes
 * a cell's arithmetic.
 */
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#define IDX(x, y, z, Nx, Ny) ((((size_t)(z)) * (size_t)(Ny) + (size_t)(y)) * (size_t)(Nx) + (size_t)(x))

/* neighbour index along one axis; periodic wraps mod N */
static long nb(long i, long d, long N, int periodic)
{
    long j = i + d;
    if (periodic) {
        if (j < 0) j += N;
        if (j >= N) j -= N;
    }
    return j;
}

/*
 * One explicit Euler step of Fig. 1 on the global grid.
 * Writes T2 at every updatable cell; leaves all other cells of T2 untouched.
 * mode 0 = paper-literal division by dx^2; mode 1 = canonical reciprocal.
 */
void oracle_heat_step(double *T2, const double *T, const double *Ci,
                      long Nx, long Ny, long Nz,
                      int px, int py, int pz,
                      double lam, double dt, double dx, double dy, double dz,
                      int mode)
{
    /* an axis of size 1 (a 1-D/2-D grid) is updated on its one layer, without a term */
    const int ax = Nx > 1, ay = Ny > 1, az = Nz > 1;
    const long xa = (px || !ax) ? 0 : 1, xb = (px || !ax) ? Nx : Nx - 1;
    const long ya = (py || !ay) ? 0 : 1, yb = (py || !ay) ? Ny : Ny - 1;
    const long za = (pz || !az) ? 0 : 1, zb = (pz || !az) ? Nz : Nz - 1;
    const double dx2 = dx * dx, dy2 = dy * dy, dz2 = dz * dz;
    const double rdx2 = 1.0 / dx2, rdy2 = 1.0 / dy2, rdz2 = 1.0 / dz2;
    long z;
#pragma omp parallel for schedule(static)
    for (z = za; z < zb; ++z) {
        for (long y = ya; y < yb; ++y) {
            for (long x = xa; x < xb; ++x) {
                const double c  = T[IDX(x, y, z, Nx, Ny)];
                /* @d2_xi, @d2_yi, @d2_zi, each as (a/d^2) or (a*r) by mode,
                   summed left to right over the axes that have extent */
                double lap = 0.0;
                int first = 1;
                if (ax) {
                    const double xm = T[IDX(nb(x, -1, Nx, px), y, z, Nx, Ny)];
                    const double xp = T[IDX(nb(x, +1, Nx, px), y, z, Nx, Ny)];
                    const double d2x = (xp - c) - (c - xm);
                    const double t = mode == 0 ? d2x / dx2 : d2x * rdx2;
                    lap = first ? t : lap + t;
                    first = 0;
                }
                if (ay) {
                    const double ym = T[IDX(x, nb(y, -1, Ny, py), z, Nx, Ny)];
                    const double yp = T[IDX(x, nb(y, +1, Ny, py), z, Nx, Ny)];
                    const double d2y = (yp - c) - (c - ym);
                    const double t = mode == 0 ? d2y / dy2 : d2y * rdy2;
                    lap = first ? t : lap + t;
                    first = 0;
                }
                if (az) {
                    const double zm = T[IDX(x, y, nb(z, -1, Nz, pz), Nx, Ny)];
                    const double zp = T[IDX(x, y, nb(z, +1, Nz, pz), Nx, Ny)];
                    const double d2z = (zp - c) - (c - zm);
                    const double t = mode == 0 ? d2z / dz2 : d2z * rdz2;
                    lap = first ? t : lap + t;
                    first = 0;
                }
                const double ci = Ci[IDX(x, y, z, Nx, Ny)];
                T2[IDX(x, y, z, Nx, Ny)] = c + dt * ((lam * ci) * lap);
            }
        }
    }
}

/*
 * The binary32 variant (reading 24): the same step with every
 * operation in binary32 -- inputs rounded to float once (lam, dt, dx, dy, dz, T, Ci), the
 * reciprocals r_d = 1.0f/(d*d) computed in float, canonical association only:
 *   T2 = T + dt*((lam*Ci)*(((d2x*rdx2) + (d2y*rdy2)) + (d2z*rdz2)))
 * A size-1 axis drops its term as in the binary64 step (reading 23).
 */
void oracle_heat_step_f32(float *T2, const float *T, const float *Ci,
                          long Nx, long Ny, long Nz,
                          int px, int py, int pz,
                          float lam, float dt, float dx, float dy, float dz)
{
    const int ax = Nx > 1, ay = Ny > 1, az = Nz > 1;
    const long xa = (px || !ax) ? 0 : 1, xb = (px || !ax) ? Nx : Nx - 1;
    const long ya = (py || !ay) ? 0 : 1, yb = (py || !ay) ? Ny : Ny - 1;
    const long za = (pz || !az) ? 0 : 1, zb = (pz || !az) ? Nz : Nz - 1;
    const float rdx2 = 1.0f / (dx * dx), rdy2 = 1.0f / (dy * dy), rdz2 = 1.0f / (dz * dz);
    long z;
#pragma omp parallel for schedule(static)
    for (z = za; z < zb; ++z) {
        for (long y = ya; y < yb; ++y) {
            for (long x = xa; x < xb; ++x) {
                const float c = T[IDX(x, y, z, Nx, Ny)];
                float lap = 0.0f;
                int first = 1;
                if (ax) {
                    const float d2 = (T[IDX(nb(x, +1, Nx, px), y, z, Nx, Ny)] - c) - (c - T[IDX(nb(x, -1, Nx, px), y, z, Nx, Ny)]);
                    const float t = d2 * rdx2;
                    lap = first ? t : lap + t;
                    first = 0;
                }
                if (ay) {
                    const float d2 = (T[IDX(x, nb(y, +1, Ny, py), z, Nx, Ny)] - c) - (c - T[IDX(x, nb(y, -1, Ny, py), z, Nx, Ny)]);
                    const float t = d2 * rdy2;
                    lap = first ? t : lap + t;
                    first = 0;
                }
                if (az) {
                    const float d2 = (T[IDX(x, y, nb(z, +1, Nz, pz), Nx, Ny)] - c) - (c - T[IDX(x, y, nb(z, -1, Nz, pz), Nx, Ny)]);
                    const float t = d2 * rdz2;
                    lap = first ? t : lap + t;
                    first = 0;
                }
                T2[IDX(x, y, z, Nx, Ny)] = c + dt * ((lam * Ci[IDX(x, y, z, Nx, Ny)]) * lap);
            }
        }
    }
}

/* the binary32 time loop: T2 = copy(T), nt steps with swap; T holds the result */
int oracle_heat_run_f32(float *T, const float *Ci, long Nx, long Ny, long Nz, int px, int py, int pz,
                        float lam, float dt, float dx, float dy, float dz, int nt)
{
    const size_t n = (size_t)Nx * (size_t)Ny * (size_t)Nz;
    float *T2 = (float *)malloc(n * sizeof(float));
    if (!T2) return -1;
    memcpy(T2, T, n * sizeof(float));
    float *a = T, *b = T2;
    for (int it = 0; it < nt; ++it) {
        oracle_heat_step_f32(b, a, Ci, Nx, Ny, Nz, px, py, pz, lam, dt, dx, dy, dz);
        float *t = a; a = b; b = t;
    }
    if (a != T) memcpy(T, a, n * sizeof(float));
    free(T2);
    return 0;
}

/*
 * The time loop of Fig. 1: T2 = copy(T); nt times
 * { step!(T2, T, ...); T, T2 = T2, T }.  T (in) is the initial field and on
 * return holds the final T.  Returns 0 on success, -1 on allocation failure.
 */
int oracle_heat_run(double *T, const double *Ci,
                    long Nx, long Ny, long Nz,
                    int px, int py, int pz,
                    double lam, double dt, double dx, double dy, double dz,
                    int nt, int mode)
{
    const size_t n = (size_t)Nx * (size_t)Ny * (size_t)Nz;
    double *T2 = (double *)malloc(n * sizeof(double));
    if (!T2) return -1;
    memcpy(T2, T, n * sizeof(double)); /* T2 = copy(T) */
    double *a = T, *b = T2;
    for (int it = 0; it < nt; ++it) {
        oracle_heat_step(b, a, Ci, Nx, Ny, Nz, px, py, pz, lam, dt, dx, dy, dz, mode);
        double *t = a; a = b; b = t; /* T, T2 = T2, T */
    }
    if (a != T) memcpy(T, a, n * sizeof(double));
    free(T2);
    return 0;
}

/* maximum(Ci) of PAPER.md:73 over the whole global field */
double oracle_max(const double *A, long n)
{
    double m = A[0];
    for (long i = 1; i < n; ++i)
        if (A[i] > m) m = A[i];
    return m;
}

/* set the OpenMP thread count (no-op without OpenMP) */
void oracle_set_threads(int n)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* thread count the OpenMP runtime will use (1 without OpenMP) */
int oracle_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
