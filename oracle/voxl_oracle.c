/* voxl_oracle.c -- plain-C restatement of the reference LBM hot path.
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA engines. See voxl_oracle.h
 * for who may load it. Parity of this file is pinned against the reference
 * library compiled from its own sources (oracle/_ref/libvoxl_ref.so) by
 * tests/test_oracle.py; each function cites the reference lines it restates.
 *
 * Build: gcc -O3 -ffp-contract=off (oracle/Makefile). Double arithmetic below is
 * written in the exact association order of the reference C++ expressions.
 */
#include "voxl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- lattice (proj/src/lattice.cpp:29-102) ---------------------------------- */

static void weight_for(int kind, int s2, long long* num, long long* den) {
    /* lattice.cpp:29-46 */
    *den = 1;
    switch (kind) {
        case VO_D2Q9:
            if (s2 == 0) { *num = 4; *den = 9; }
            else if (s2 == 1) { *num = 1; *den = 9; }
            else { *num = 1; *den = 36; }
            return;
        case VO_D3Q19:
            if (s2 == 0) { *num = 1; *den = 3; }
            else if (s2 == 1) { *num = 1; *den = 18; }
            else { *num = 1; *den = 36; }
            return;
        default:
            if (s2 == 0) { *num = 8; *den = 27; }
            else if (s2 == 1) { *num = 2; *den = 27; }
            else if (s2 == 2) { *num = 1; *den = 54; }
            else { *num = 1; *den = 216; }
            return;
    }
}

static int vel_less(const int* a, const int* b) {
    const int sa = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
    const int sb = b[0] * b[0] + b[1] * b[1] + b[2] * b[2];
    if (sa != sb) return sa < sb;
    if (a[0] != b[0]) return a[0] < b[0];
    if (a[1] != b[1]) return a[1] < b[1];
    return a[2] < b[2];
}

void vo_build_lattice(int kind, vo_lattice* lat) {
    /* lattice.cpp:59-102: enumerate {-1,0,1}^dim, filter by speed class, sort by
     * (|e|^2, x, y, z), exact rational weights, opposite by search. */
    memset(lat, 0, sizeof(*lat));
    lat->kind = kind;
    lat->dim = kind == VO_D2Q9 ? 2 : 3;
    const int max_s2 = kind == VO_D3Q19 ? 2 : 3;
    const int zlo = lat->dim == 3 ? -1 : 0, zhi = lat->dim == 3 ? 1 : 0;
    int n = 0;
    for (int x = -1; x <= 1; ++x)
        for (int y = -1; y <= 1; ++y)
            for (int z = zlo; z <= zhi; ++z)
                if (x * x + y * y + z * z <= max_s2) {
                    lat->e[n][0] = x;
                    lat->e[n][1] = y;
                    lat->e[n][2] = z;
                    ++n;
                }
    /* insertion sort: small and stable enough (keys are distinct) */
    for (int i = 1; i < n; ++i)
        for (int j = i; j > 0 && vel_less(lat->e[j], lat->e[j - 1]); --j) {
            int t[3];
            memcpy(t, lat->e[j], sizeof t);
            memcpy(lat->e[j], lat->e[j - 1], sizeof t);
            memcpy(lat->e[j - 1], t, sizeof t);
        }
    lat->q = n;
    for (int i = 0; i < n; ++i) {
        const int* e = lat->e[i];
        weight_for(kind, e[0] * e[0] + e[1] * e[1] + e[2] * e[2], &lat->wnum[i], &lat->wden[i]);
        lat->w[i] = (double)lat->wnum[i] / (double)lat->wden[i];
    }
    for (int i = 0; i < n; ++i) {
        lat->opp[i] = -1;
        for (int j = 0; j < n; ++j)
            if (lat->e[j][0] == -lat->e[i][0] && lat->e[j][1] == -lat->e[i][1] &&
                lat->e[j][2] == -lat->e[i][2]) {
                lat->opp[i] = j;
                break;
            }
    }
}

/* ---- moments / equilibrium / BGK (lattice.cpp:104-138) ----------------------- */

static int equilibrium(const vo_lattice* lat, double rho, const double u[3], double* f) {
    /* lattice.cpp:104-113 */
    if (!isfinite(rho) || !isfinite(u[0]) || !isfinite(u[1]) || !isfinite(u[2])) return -1;
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int i = 0; i < lat->q; ++i) {
        const int* e = lat->e[i];
        const double eu = (double)e[0] * u[0] + (double)e[1] * u[1] + (double)e[2] * u[2];
        f[i] = lat->w[i] * rho * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * uu);
    }
    return 0;
}

static int macroscopic(const vo_lattice* lat, const double* f, double* rho, double u[3]) {
    /* lattice.cpp:115-129 */
    double r = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
    for (int i = 0; i < lat->q; ++i) {
        r += f[i];
        mx += f[i] * (double)lat->e[i][0];
        my += f[i] * (double)lat->e[i][1];
        mz += f[i] * (double)lat->e[i][2];
    }
    if (!(r > 0.0)) return -1;
    *rho = r;
    u[0] = mx / r;
    u[1] = my / r;
    u[2] = mz / r;
    return 0;
}

static int bgk_relax(const vo_lattice* lat, double inv_tau, double* f) {
    /* lattice.cpp:131-138 */
    double rho, u[3], feq[27];
    if (macroscopic(lat, f, &rho, u)) return -1;
    if (equilibrium(lat, rho, u, feq)) return -1;
    const double keep = 1.0 - inv_tau;
    for (int i = 0; i < lat->q; ++i) f[i] = keep * f[i] + inv_tau * feq[i];
    return 0;
}

/* ---- rules / initial state (solver.cpp:150-187) ------------------------------ */

void vo_rules_for(int kind, int scenario, int nx, int ny, int nz, const double vel[3], vo_rules* r) {
    memset(r, 0, sizeof(*r));
    r->n[0] = nx;
    r->n[1] = ny;
    r->n[2] = nz;
    r->lid_axis = 2;
    r->lid_at_max = 1;
    const int dim = kind == VO_D2Q9 ? 2 : 3;
    if (scenario == 2) {
        r->periodic[0] = r->periodic[1] = 1;
        r->periodic[2] = dim == 3;
        memcpy(r->wrap, r->periodic, sizeof r->wrap);
    } else if (scenario == 0) {
        r->has_lid = 1;
        r->lid_axis = dim == 2 ? 1 : 2;
        r->lid_at_max = 1;
        r->lid_u[0] = vel[0];
        r->lid_u[1] = vel[1];
        r->lid_u[2] = vel[2];
    }
}

/* std::mt19937_64 */
typedef struct {
    uint64_t mt[312];
    int idx;
} vo_mt64;

static void mt_seed(vo_mt64* g, uint64_t s) {
    g->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt_next(vo_mt64* g) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
            g->mt[i] = g->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
        }
        g->idx = 0;
    }
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* libstdc++ uniform_real_distribution<double>(a,b) over generate_canonical<double,53>
 * with a 64-bit engine: one draw, x / 2^64, clamped below 1. */
static double mt_uniform(vo_mt64* g, double a, double b) {
    double c = (double)mt_next(g) / 18446744073709551616.0;
    if (c >= 1.0) c = nextafter(1.0, 0.0);
    return c * (b - a) + a;
}

void vo_initial_state(int kind, int scenario, int nx, int ny, int nz, uint64_t seed,
                      double perturbation, double* out) {
    vo_lattice lat;
    vo_build_lattice(kind, &lat);
    const int64_t vol = (int64_t)nx * ny * nz;
    double feq[27];
    if (scenario == 2 && perturbation > 0.0) {
        vo_mt64* g = (vo_mt64*)malloc(sizeof(vo_mt64));
        mt_seed(g, seed);
        for (int64_t v = 0; v < vol; ++v) {
            const double rho = 1.0 + perturbation * mt_uniform(g, -1.0, 1.0);
            double u[3];
            u[0] = 0.1 * perturbation * mt_uniform(g, -1.0, 1.0);
            u[1] = 0.1 * perturbation * mt_uniform(g, -1.0, 1.0);
            u[2] = lat.dim == 3 ? 0.1 * perturbation * mt_uniform(g, -1.0, 1.0) : 0.0;
            equilibrium(&lat, rho, u, feq);
            for (int i = 0; i < lat.q; ++i) out[v * lat.q + i] = feq[i];
        }
        free(g);
    } else {
        const double u0[3] = {0.0, 0.0, 0.0};
        equilibrium(&lat, 1.0, u0, feq);
        for (int64_t v = 0; v < vol; ++v)
            for (int i = 0; i < lat.q; ++i) out[v * lat.q + i] = feq[i];
    }
}

/* ---- dense step (lbm.hpp:40-74, lbm.cpp:104-114) ------------------------------ */

static double lid_term(const vo_lattice* lat, const vo_rules* r, int i) {
    /* lbm.hpp:66-69: val += 2.0 * w_i * kRho0 * 3.0 * eu */
    const int* e = lat->e[i];
    const double eu = (double)e[0] * r->lid_u[0] + (double)e[1] * r->lid_u[1] + (double)e[2] * r->lid_u[2];
    return 2.0 * lat->w[i] * 1.0 * 3.0 * eu;
}

int vo_dense_run(int kind, const vo_rules* r, double tau, int steps, double* state) {
    vo_lattice lat;
    vo_build_lattice(kind, &lat);
    const int q = lat.q;
    const int nx = r->n[0], ny = r->n[1], nz = r->n[2];
    const int64_t vol = (int64_t)nx * ny * nz;
    double* a = state;
    double* b = (double*)malloc(sizeof(double) * (size_t)(vol * q));
    if (!b) return -1;
    const double inv_tau = 1.0 / tau;
    int rc = 0;
    for (int s = 0; s < steps && !rc; ++s) {
        for (int z = 0; z < nz && !rc; ++z)
            for (int y = 0; y < ny && !rc; ++y)
                for (int x = 0; x < nx; ++x) {
                    const int v[3] = {x, y, z};
                    const int64_t lin = ((int64_t)z * ny + y) * nx + x;
                    double* g = b + lin * q;
                    for (int i = 0; i < q; ++i) {
                        int src[3] = {v[0] - lat.e[i][0], v[1] - lat.e[i][1], v[2] - lat.e[i][2]};
                        int oob = 0, lid = 0;
                        for (int ax = 0; ax < 3; ++ax) {
                            if (src[ax] >= 0 && src[ax] < r->n[ax]) continue;
                            if (r->wrap[ax]) {
                                src[ax] = (src[ax] + r->n[ax]) % r->n[ax];
                            } else if (r->periodic[ax]) {
                            } else {
                                oob = 1;
                                if (r->has_lid && ax == r->lid_axis &&
                                    (r->lid_at_max ? src[ax] >= r->n[ax] : src[ax] < 0))
                                    lid = 1;
                            }
                        }
                        if (!oob) {
                            const int64_t sl = ((int64_t)src[2] * ny + src[1]) * nx + src[0];
                            g[i] = a[sl * q + i];
                        } else {
                            double val = a[lin * q + lat.opp[i]];
                            if (lid) val += lid_term(&lat, r, i);
                            g[i] = val;
                        }
                    }
                    if (bgk_relax(&lat, inv_tau, g)) {
                        rc = -1;
                        break;
                    }
                }
        double* t = a;
        a = b;
        b = t;
    }
    if (a != state) {
        memcpy(state, a, sizeof(double) * (size_t)(vol * q));
        free(a);
    } else {
        free(b);
    }
    return rc;
}

/* ---- regularized reconstruction (lbm.cpp:10-59) --------------------------------- */

int vo_regularized(const vo_lattice* lat, int axis, int sign, const double u_bc[3], double* f) {
    const double u_n = u_bc[axis] * (double)sign;
    if (!(fabs(1.0 - u_n) > 1e-12)) return -1;
    double sum0 = 0.0, sum_in = 0.0;
    for (int i = 0; i < lat->q; ++i) {
        const int en = lat->e[i][axis] * sign;
        if (en == 0) sum0 += f[i];
        else if (en < 0) sum_in += f[i];
    }
    const double rho = (sum0 + 2.0 * sum_in) / (1.0 - u_n);
    double feq[27], fneq[27];
    if (equilibrium(lat, rho, u_bc, feq)) return -1;
    for (int i = 0; i < lat->q; ++i) {
        const int en = lat->e[i][axis] * sign;
        const int j = en > 0 ? lat->opp[i] : i;
        fneq[i] = f[j] - feq[j];
    }
    double pi[3][3] = {{0}};
    for (int i = 0; i < lat->q; ++i) {
        const double ev[3] = {(double)lat->e[i][0], (double)lat->e[i][1], (double)lat->e[i][2]};
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) pi[a][b] += fneq[i] * ev[a] * ev[b];
    }
    const double cs2 = 1.0 / 3.0;
    for (int i = 0; i < lat->q; ++i) {
        const double ev[3] = {(double)lat->e[i][0], (double)lat->e[i][1], (double)lat->e[i][2]};
        double qpi = 0.0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) qpi += (ev[a] * ev[b] - (a == b ? cs2 : 0.0)) * pi[a][b];
        f[i] = feq[i] + lat->w[i] * 4.5 * qpi;
    }
    return 0;
}

/* ---- diagnostics (lbm.cpp:116-138) --------------------------------------------- */

int vo_probe(int kind, const double* canonical, int64_t voxels, double* mass, double* max_speed,
             int64_t* bad_voxel, int* bad_pop) {
    vo_lattice lat;
    vo_build_lattice(kind, &lat);
    double m = 0.0, ms = 0.0;
    for (int64_t n = 0; n < voxels; ++n) {
        const double* f = canonical + n * lat.q;
        for (int i = 0; i < lat.q; ++i) {
            if (!isfinite(f[i]) || fabs(f[i]) > 1e3) {
                if (bad_voxel) *bad_voxel = n;
                if (bad_pop) *bad_pop = i;
                return -1;
            }
            m += f[i];
        }
        double rho, u[3];
        if (macroscopic(&lat, f, &rho, u)) return -1;
        const double sp = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        if (sp > ms) ms = sp;
    }
    *mass = m;
    *max_speed = ms;
    return 0;
}

/* ---- block-sparse wind tunnel (sparse.cpp:227-238, 321-394) -------------------- */

int64_t vo_obstacle_mask(int nx, int ny, int nz, double radius, uint8_t* active) {
    /* solver.cpp:272-283; radius <= 0 selects min_extent / 5 */
    int mn = nx < ny ? nx : ny;
    mn = mn < nz ? mn : nz;
    const double r = radius > 0.0 ? radius : mn / 5.0;
    const double cx = nx / 2.0 - 0.5, cy = ny / 2.0 - 0.5, cz = nz / 2.0 - 0.5;
    int64_t n = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const double dx = x - cx, dy = y - cy, dz = z - cz;
                const int a = dx * dx + dy * dy + dz * dz > r * r;
                active[((int64_t)z * ny + y) * nx + x] = (uint8_t)a;
                n += a;
            }
    return n;
}

int vo_sparse_run(int kind, int nx, int ny, int nz, const uint8_t* active, double tau,
                  const double u_bc[3], int steps, double* state) {
    vo_lattice lat;
    vo_build_lattice(kind, &lat);
    const int q = lat.q;
    const int64_t vol = (int64_t)nx * ny * nz;
    double* cur = state;
    double* nxt = (double*)malloc(sizeof(double) * (size_t)(vol * q));
    if (!nxt) return -1;
    memcpy(nxt, cur, sizeof(double) * (size_t)(vol * q));
    const double inv_tau = 1.0 / tau;
    int rc = 0;
    for (int s = 0; s < steps && !rc; ++s) {
        for (int z = 0; z < nz && !rc; ++z)
            for (int y = 0; y < ny && !rc; ++y)
                for (int x = 0; x < nx; ++x) {
                    const int64_t lin = ((int64_t)z * ny + y) * nx + x;
                    if (!active[lin]) continue;
                    double g[27];
                    for (int i = 0; i < q; ++i) {
                        const int sx = x - lat.e[i][0], sy = y - lat.e[i][1], sz = z - lat.e[i][2];
                        int solid = !(sx >= 0 && sx < nx && sy >= 0 && sy < ny && sz >= 0 && sz < nz);
                        int64_t sl = 0;
                        if (!solid) {
                            sl = ((int64_t)sz * ny + sy) * nx + sx;
                            solid = !active[sl];
                        }
                        g[i] = solid ? cur[lin * q + lat.opp[i]] : cur[sl * q + i];
                    }
                    if (x == 0 || x == nx - 1) {
                        if (vo_regularized(&lat, 0, x == 0 ? 1 : -1, u_bc, g)) { rc = -1; break; }
                    }
                    if (bgk_relax(&lat, inv_tau, g)) { rc = -1; break; }
                    memcpy(nxt + lin * q, g, sizeof(double) * q);
                }
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    if (cur != state) {
        memcpy(state, cur, sizeof(double) * (size_t)(vol * q));
        free(cur);
    } else {
        free(nxt);
    }
    return rc;
}

/* ---- multi-resolution band cavity (multires.cpp:54-192, 367-598) ---------------- */

void vo_band_level_map(int nx, int ny, int nz, int levels, int axis, int* map) {
    const int n[3] = {nx, ny, nz};
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const int v[3] = {x, y, z};
                const int k = v[axis];
                int level = levels - 1;
                for (int l = 0; l < levels - 1; ++l)
                    if (k >= (n[axis] >> (l + 1))) {
                        level = l;
                        break;
                    }
                map[((int64_t)z * ny + y) * nx + x] = level;
            }
}

typedef struct {
    int n[3];
    int64_t vol;
    uint8_t* active;       /* level cells */
    uint8_t* refined;      /* covered by the finer level */
    uint8_t* under_coarse; /* parent active at the coarser level */
    uint8_t* ghost;        /* inactive under_coarse box-neighbour of an active cell */
    uint8_t* solid;        /* obstacle extension: level-map -1 cells (finest level only) */
    double *cur, *nxt, *post, *ghostv, *coal;
    double inv_tau;
} vo_level;

#define LIN(L, x, y, z) (((int64_t)(z) * (L)->n[1] + (y)) * (L)->n[0] + (x))

static int in_level(const vo_level* L, int x, int y, int z) {
    return x >= 0 && x < L->n[0] && y >= 0 && y < L->n[1] && z >= 0 && z < L->n[2];
}

typedef struct {
    vo_lattice lat;
    int levels, dim;
    vo_level lv[4];
    vo_rules rules;
} vo_mres;

static void mres_collide(vo_mres* M, int l) {
    /* collide_level (multires.cpp:443-456): post = BGK(cur) on active cells */
    vo_level* L = &M->lv[l];
    const int q = M->lat.q;
    for (int64_t c = 0; c < L->vol; ++c) {
        if (!L->active[c]) continue;
        memcpy(L->post + c * q, L->cur + c * q, sizeof(double) * q);
        bgk_relax(&M->lat, L->inv_tau, L->post + c * q);
    }
}

static void mres_explode(vo_mres* M, int coarse) {
    /* explode (multires.cpp:458-467): ghost(l-1) <- parent post-collision */
    vo_level* F = &M->lv[coarse - 1];
    vo_level* C = &M->lv[coarse];
    const int q = M->lat.q;
    for (int z = 0; z < F->n[2]; ++z)
        for (int y = 0; y < F->n[1]; ++y)
            for (int x = 0; x < F->n[0]; ++x) {
                const int64_t c = LIN(F, x, y, z);
                if (!F->ghost[c]) continue;
                const int pz = M->dim == 3 ? z >> 1 : z;
                memcpy(F->ghostv + c * q, C->post + LIN(C, x >> 1, y >> 1, pz) * q, sizeof(double) * q);
            }
}

static void mres_coalesce(vo_mres* M, int coarse) {
    /* coalesce (multires.cpp:469-483): mean over children_of (x fastest) of the
     * fine level's current (post-stream) population i. */
    vo_level* F = &M->lv[coarse - 1];
    vo_level* C = &M->lv[coarse];
    const int q = M->lat.q;
    const double scale = 1.0 / (M->dim == 3 ? 8 : 4);
    const int zhi = M->dim == 3 ? 1 : 0;
    for (int z = 0; z < C->n[2]; ++z)
        for (int y = 0; y < C->n[1]; ++y)
            for (int x = 0; x < C->n[0]; ++x) {
                const int64_t c = LIN(C, x, y, z);
                if (!C->active[c]) continue;
                for (int i = 0; i < q; ++i) {
                    const int sx = x - M->lat.e[i][0], sy = y - M->lat.e[i][1], sz = z - M->lat.e[i][2];
                    if (!in_level(C, sx, sy, sz)) continue;
                    const int64_t s = LIN(C, sx, sy, sz);
                    if (C->active[s] || !C->refined[s]) continue;
                    double sum = 0.0;
                    for (int dz = 0; dz <= zhi; ++dz)
                        for (int dy = 0; dy <= 1; ++dy)
                            for (int dx = 0; dx <= 1; ++dx) {
                                const int cz = M->dim == 3 ? 2 * sz + dz : sz;
                                sum += F->cur[LIN(F, 2 * sx + dx, 2 * sy + dy, cz) * q + i];
                            }
                    C->coal[c * q + i] = sum * scale;
                }
            }
}

static void mres_stream(vo_mres* M, int l) {
    /* stream_voxel / stream_level (multires.cpp:485-561); fused mode produces
     * identical values (post_collision recompute, :433-441). */
    vo_level* L = &M->lv[l];
    const int q = M->lat.q;
    const vo_rules* r = &M->rules;
    for (int z = 0; z < L->n[2]; ++z)
        for (int y = 0; y < L->n[1]; ++y)
            for (int x = 0; x < L->n[0]; ++x) {
                const int64_t c = LIN(L, x, y, z);
                if (!L->active[c]) continue;
                for (int i = 0; i < q; ++i) {
                    const int src[3] = {x - M->lat.e[i][0], y - M->lat.e[i][1], z - M->lat.e[i][2]};
                    int oob = 0, lid = 0;
                    for (int a = 0; a < 3; ++a) {
                        if (src[a] >= 0 && src[a] < L->n[a]) continue;
                        oob = 1;
                        if (r->has_lid && a == r->lid_axis &&
                            (r->lid_at_max ? src[a] >= L->n[a] : src[a] < 0))
                            lid = 1;
                    }
                    double g;
                    if (oob) {
                        g = L->post[c * q + M->lat.opp[i]];
                        if (lid) g += lid_term(&M->lat, r, i);
                    } else {
                        const int64_t s = LIN(L, src[0], src[1], src[2]);
                        if (L->active[s]) g = L->post[s * q + i];
                        else if (L->solid[s]) g = L->post[c * q + M->lat.opp[i]]; /* halfway bounce-back */
                        else if (L->ghost[s]) g = L->ghostv[s * q + i];
                        else g = L->coal[c * q + i];
                    }
                    L->nxt[c * q + i] = g;
                }
            }
    double* t = L->cur;
    L->cur = L->nxt;
    L->nxt = t;
}

static void mres_advance(vo_mres* M, int l) {
    /* advance (multires.cpp:563-570) */
    mres_collide(M, l);
    if (l > 0) {
        mres_explode(M, l);
        mres_advance(M, l - 1);
        mres_advance(M, l - 1);
        mres_coalesce(M, l);
    }
    mres_stream(M, l);
}

int64_t vo_mres_run(int kind, int nx, int ny, int nz, int levels, const int* level_map, double tau,
                    const double lid_u[3], int steps, double* out, int64_t cap) {
    vo_mres* M = (vo_mres*)calloc(1, sizeof(vo_mres));
    vo_build_lattice(kind, &M->lat);
    const int q = M->lat.q;
    M->levels = levels;
    M->dim = M->lat.dim;
    const double vel[3] = {lid_u[0], lid_u[1], lid_u[2]};
    vo_rules_for(kind, 0, nx, ny, nz, vel, &M->rules);
    /* tau_l = 2 tau_{l+1} - 1/2 (multires.cpp:131-134) */
    double taus[4];
    taus[levels - 1] = tau;
    for (int l = levels - 2; l >= 0; --l) taus[l] = 2.0 * taus[l + 1] - 0.5;
    for (int l = 0; l < levels; ++l) {
        vo_level* L = &M->lv[l];
        const int s = 1 << l;
        L->n[0] = nx / s;
        L->n[1] = ny / s;
        L->n[2] = M->dim == 3 ? nz / s : nz;
        L->vol = (int64_t)L->n[0] * L->n[1] * L->n[2];
        L->active = (uint8_t*)calloc((size_t)L->vol, 1);
        L->refined = (uint8_t*)calloc((size_t)L->vol, 1);
        L->under_coarse = (uint8_t*)calloc((size_t)L->vol, 1);
        L->ghost = (uint8_t*)calloc((size_t)L->vol, 1);
        L->solid = (uint8_t*)calloc((size_t)L->vol, 1);
        if (l == 0)
            for (int64_t c = 0; c < L->vol; ++c) L->solid[c] = level_map[c] == -1;
        L->cur =(double*)calloc((size_t)(L->vol * q), sizeof(double));
        L->nxt = (double*)calloc((size_t)(L->vol * q), sizeof(double));
        L->post = (double*)calloc((size_t)(L->vol * q), sizeof(double));
        L->ghostv = (double*)calloc((size_t)(L->vol * q), sizeof(double));
        L->coal = (double*)calloc((size_t)(L->vol * q), sizeof(double));
        L->inv_tau = 1.0 / taus[l];
        /* active iff every covered finest cell carries level l (multires.cpp:290-318) */
        for (int z = 0; z < L->n[2]; ++z)
            for (int y = 0; y < L->n[1]; ++y)
                for (int x = 0; x < L->n[0]; ++x) {
                    int all = 1;
                    const int zs = M->dim == 3 ? s : 1;
                    for (int dz = 0; dz < zs && all; ++dz)
                        for (int dy = 0; dy < s && all; ++dy)
                            for (int dx = 0; dx < s && all; ++dx) {
                                const int fz = M->dim == 3 ? z * s + dz : z;
                                all = level_map[((int64_t)fz * ny + (y * s + dy)) * nx + (x * s + dx)] == l;
                            }
                    L->active[LIN(L, x, y, z)] = (uint8_t)all;
                }
    }
    for (int l = 0; l < levels; ++l) {
        vo_level* L = &M->lv[l];
        for (int z = 0; z < L->n[2]; ++z)
            for (int y = 0; y < L->n[1]; ++y)
                for (int x = 0; x < L->n[0]; ++x) {
                    const int64_t c = LIN(L, x, y, z);
                    const int pz = M->dim == 3 ? z >> 1 : z;
                    if (l + 1 < levels && M->lv[l + 1].active[LIN(&M->lv[l + 1], x >> 1, y >> 1, pz)])
                        L->under_coarse[c] = 1;
                    if (l > 0) {
                        const vo_level* F = &M->lv[l - 1];
                        const int zhi = M->dim == 3 ? 1 : 0;
                        for (int dz = 0; dz <= zhi; ++dz)
                            for (int dy = 0; dy <= 1; ++dy)
                                for (int dx = 0; dx <= 1; ++dx) {
                                    const int cz = M->dim == 3 ? 2 * z + dz : z;
                                    if (F->active[LIN(F, 2 * x + dx, 2 * y + dy, cz)]) L->refined[c] = 1;
                                }
                    }
                }
    }
    /* ghost ring (multires.cpp:350-368): inactive under_coarse box neighbours */
    for (int l = 0; l + 1 < levels; ++l) {
        vo_level* L = &M->lv[l];
        const int zlo = M->dim == 3 ? -1 : 0, zhi = M->dim == 3 ? 1 : 0;
        for (int z = 0; z < L->n[2]; ++z)
            for (int y = 0; y < L->n[1]; ++y)
                for (int x = 0; x < L->n[0]; ++x) {
                    if (!L->active[LIN(L, x, y, z)]) continue;
                    for (int dz = zlo; dz <= zhi; ++dz)
                        for (int dy = -1; dy <= 1; ++dy)
                            for (int dx = -1; dx <= 1; ++dx) {
                                if (!dx && !dy && !dz) continue;
                                if (!in_level(L, x + dx, y + dy, z + dz)) continue;
                                const int64_t n = LIN(L, x + dx, y + dy, z + dz);
                                if (!L->active[n] && L->under_coarse[n]) L->ghost[n] = 1;
                            }
                }
    }
    /* rest equilibrium everywhere (multires.cpp:574-587) */
    {
        double feq[27];
        const double u0[3] = {0.0, 0.0, 0.0};
        equilibrium(&M->lat, 1.0, u0, feq);
        for (int l = 0; l < levels; ++l)
            for (int64_t c = 0; c < M->lv[l].vol; ++c)
                memcpy(M->lv[l].cur + c * q, feq, sizeof(double) * q);
    }
    for (int s = 0; s < steps; ++s) mres_advance(M, levels - 1);

    /* canonical_state (multires.cpp:578-598): per level, pack_coord order = x
     * slowest, z fastest. */
    int64_t n = 0;
    for (int l = 0; l < levels; ++l) {
        vo_level* L = &M->lv[l];
        for (int x = 0; x < L->n[0]; ++x)
            for (int y = 0; y < L->n[1]; ++y)
                for (int z = 0; z < L->n[2]; ++z) {
                    const int64_t c = LIN(L, x, y, z);
                    if (!L->active[c]) continue;
                    if (out && n + q <= cap) memcpy(out + n, L->cur + c * q, sizeof(double) * q);
                    n += q;
                }
    }
    for (int l = 0; l < levels; ++l) {
        vo_level* L = &M->lv[l];
        free(L->active); free(L->refined); free(L->under_coarse); free(L->ghost); free(L->solid);
        free(L->cur); free(L->nxt); free(L->post); free(L->ghostv); free(L->coal);
    }
    free(M);
    return n;
}

/* ---- generic step_occ operator: five-point Jacobi (partition_test.cpp:234-247) ---- */

void vo_jacobi2_run(int nx, int ny, int nz, int steps, double* state) {
    const int64_t plane = (int64_t)nx * ny;
    const int64_t n = plane * nz * 2;
    double* nxt = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    static const int off[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
    for (int s = 0; s < steps; ++s) {
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    const int64_t v = z * plane + (int64_t)y * nx + x;
                    for (int c = 0; c < 2; ++c) {
                        double sum = 0.0;
                        int cnt = 0;
                        for (int j = 0; j < 4; ++j) {
                            const int sx = x + off[j][0], sy = y + off[j][1];
                            if (sx < 0 || sx >= nx || sy < 0 || sy >= ny) continue;
                            sum += state[(z * plane + (int64_t)sy * nx + sx) * 2 + c];
                            ++cnt;
                        }
                        nxt[v * 2 + c] = 0.5 * state[v * 2 + c] + 0.5 * (cnt ? sum / cnt : 0.0);
                    }
                }
        memcpy(state, nxt, sizeof(double) * (size_t)n);
    }
    free(nxt);
}
