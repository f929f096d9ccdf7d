/*
 * TEST INFRASTRUCTURE ONLY — see lbm_oracle.h.
 *
 * Plain-C FP64 restatement of the reference hot path for one region.  Each
 * function cites the reference file:line it restates.  Expression order is
 * kept so results are bit-identical to the compiled reference under
 * -ffp-contract=off.
 */
#include "lbm_oracle.h"

#include <math.h>
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- lattice */
/* lattice.cpp:8-46: rest first, then (cz, cy, cx)-lexicographic. */
static int C3[27][3];
static double W[27];
static int OPP[27];
static int D2T[27];          /* direction -> tensor (cx+1)+3(cy+1)+9(cz+1) */
static int ROW_Q[27][3];     /* moment row -> exponents (collision.cpp:18-42) */
static int ROW_DEG[27];
static int T2R[27];          /* tensor mu = qx+3qy+9qz -> row */
static int tables_ready = 0;

static int row_less(const int* a, const int* b) {
    int da = a[0] + a[1] + a[2], db = b[0] + b[1] + b[2];
    if (da != db) return da < db;
    if (a[2] != b[2]) return a[2] < b[2];
    if (a[1] != b[1]) return a[1] < b[1];
    return a[0] < b[0];
}

static void tables(void) {
    if (tables_ready) return;
    int n = 1;
    C3[0][0] = C3[0][1] = C3[0][2] = 0;
    for (int z = -1; z <= 1; ++z)
        for (int y = -1; y <= 1; ++y)
            for (int x = -1; x <= 1; ++x) {
                if (!x && !y && !z) continue;
                C3[n][0] = x;
                C3[n][1] = y;
                C3[n][2] = z;
                ++n;
            }
    for (int i = 0; i < 27; ++i) {
        int m2 = C3[i][0] * C3[i][0] + C3[i][1] * C3[i][1] + C3[i][2] * C3[i][2];
        W[i] = m2 == 0 ? 8.0 / 27.0 : (m2 == 1 ? 2.0 / 27.0 : (m2 == 2 ? 1.0 / 54.0 : 1.0 / 216.0));
        for (int j = 0; j < 27; ++j)
            if (C3[j][0] == -C3[i][0] && C3[j][1] == -C3[i][1] && C3[j][2] == -C3[i][2]) {
                OPP[i] = j;
                break;
            }
        D2T[i] = (C3[i][0] + 1) + 3 * (C3[i][1] + 1) + 9 * (C3[i][2] + 1);
    }
    /* insertion sort (stable) of the qz-major generated list */
    int q[27][3], k = 0;
    for (int qz = 0; qz <= 2; ++qz)
        for (int qy = 0; qy <= 2; ++qy)
            for (int qx = 0; qx <= 2; ++qx) {
                q[k][0] = qx;
                q[k][1] = qy;
                q[k][2] = qz;
                ++k;
            }
    for (int i = 1; i < 27; ++i) {
        int cur[3] = {q[i][0], q[i][1], q[i][2]};
        int j = i - 1;
        while (j >= 0 && row_less(cur, q[j])) {
            memcpy(q[j + 1], q[j], sizeof q[j]);
            --j;
        }
        memcpy(q[j + 1], cur, sizeof cur);
    }
    for (int r = 0; r < 27; ++r) {
        memcpy(ROW_Q[r], q[r], sizeof q[r]);
        ROW_DEG[r] = q[r][0] + q[r][1] + q[r][2];
        T2R[q[r][0] + 3 * q[r][1] + 9 * q[r][2]] = r;
    }
    tables_ready = 1;
}

void orc_lattice(int* c, double* w, int* opposite, int* row_exponents) {
    tables();
    for (int i = 0; i < 27; ++i) {
        for (int a = 0; a < 3; ++a) {
            if (c) c[3 * i + a] = C3[i][a];
            if (row_exponents) row_exponents[3 * i + a] = ROW_Q[i][a];
        }
        if (w) w[i] = W[i];
        if (opposite) opposite[i] = OPP[i];
    }
}

/* ------------------------------------------------------------- collision */
typedef struct {
    int kind, policy;
    double nu, eps0, rates[27];
} model_t;

/* CollisionModel::{bgk,raw_mrt,central_mrt,validate}, collision.cpp:109-146;
 * SceneConfig::make_model, scene.cpp:28-45. */
static int make_model(const lbmg_scene_config* c, model_t* m) {
    tables();
    m->kind = c->kind;
    /* scene.cpp:33-37: only central_mrt receives the policy */
    m->policy = c->kind == LBMG_CENTRAL_MRT ? c->policy : LBMG_POLICY_CONSTANT;
    m->nu = c->viscosity;
    m->eps0 = c->policy_eps0;
    if (!(c->viscosity > 0.0)) return 1;
    const double om = 1.0 / (3.0 * c->viscosity + 0.5);
    for (int r = 0; r < 27; ++r) {
        if (c->kind == LBMG_BGK) m->rates[r] = om;
        else m->rates[r] = ROW_DEG[r] < 2 ? 1.0 : (ROW_DEG[r] == 2 ? om : c->high_order_rate);
    }
    if (c->has_explicit_rates)
        for (int r = 0; r < 27; ++r) m->rates[r] = c->rates[r];
    for (int r = 0; r < 27; ++r)
        if (ROW_DEG[r] >= 2 && !(m->rates[r] > 0.0 && m->rates[r] < 2.0)) return 1;
    return 0;
}

int orc_make_rates(const lbmg_scene_config* cfg, double* rates) {
    model_t m;
    if (make_model(cfg, &m)) return 1;
    memcpy(rates, m.rates, sizeof m.rates);
    return 0;
}

/* equilibrium, collision.cpp:148-157 */
void orc_equilibrium(double rho, const double* u, double* feq) {
    tables();
    const double usq = 1.5 * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    for (int i = 0; i < 27; ++i) {
        const double cu = C3[i][0] * u[0] + C3[i][1] * u[1] + C3[i][2] * u[2];
        feq[i] = W[i] * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - usq);
    }
}

/* forward_axis / inverse_axis, collision.cpp:51-81 */
static void fwd(double* t, int stride, double s) {
    const double x0 = -1.0 - s, x1 = -s, x2 = 1.0 - s;
    const double x0s = x0 * x0, x1s = x1 * x1, x2s = x2 * x2;
    for (int hi = 0; hi < 27; hi += stride * 3)
        for (int lo = 0; lo < stride; ++lo) {
            double* p = t + hi + lo;
            const double v0 = p[0], v1 = p[stride], v2 = p[2 * stride];
            p[0] = v0 + v1 + v2;
            p[stride] = x0 * v0 + x1 * v1 + x2 * v2;
            p[2 * stride] = x0s * v0 + x1s * v1 + x2s * v2;
        }
}

static void inv(double* t, int stride, double s) {
    const double s2 = s * s;
    const double b00 = 0.5 * (s2 - s), b01 = 0.5 * (2.0 * s - 1.0), b02 = 0.5;
    const double b10 = 1.0 - s2, b11 = -2.0 * s, b12 = -1.0;
    const double b20 = 0.5 * (s2 + s), b21 = 0.5 * (2.0 * s + 1.0), b22 = 0.5;
    for (int hi = 0; hi < 27; hi += stride * 3)
        for (int lo = 0; lo < stride; ++lo) {
            double* p = t + hi + lo;
            const double m0 = p[0], m1 = p[stride], m2 = p[2 * stride];
            p[0] = b00 * m0 + b01 * m1 + b02 * m2;
            p[stride] = b10 * m0 + b11 * m1 + b12 * m2;
            p[2 * stride] = b20 * m0 + b21 * m1 + b22 * m2;
        }
}

/* collide_range + adaptive_rates, collision.cpp:159-205 (all 27 outputs;
 * the split passes produce identical values per index, collision.hpp:60-63) */
static void collide(const double* f, double rho, const double* u, const model_t* m, double* out) {
    double feq[27];
    orc_equilibrium(rho, u, feq);
    if (m->kind == LBMG_BGK) {
        const double om = 1.0 / (3.0 * m->nu + 0.5);
        for (int i = 0; i < 27; ++i) out[i] = -om * (f[i] - feq[i]);
        return;
    }
    double t[27];
    for (int i = 0; i < 27; ++i) t[D2T[i]] = f[i] - feq[i];
    const int cm = m->kind == LBMG_CENTRAL_MRT;
    const double sx = cm ? u[0] : 0.0, sy = cm ? u[1] : 0.0, sz = cm ? u[2] : 0.0;
    fwd(t, 1, sx);
    fwd(t, 3, sy);
    fwd(t, 9, sz);
    double rates[27];
    memcpy(rates, m->rates, sizeof rates);
    if (m->policy != LBMG_POLICY_CONSTANT) {
        double eps = 0.0;
        for (int i = 0; i < 27; ++i) eps += fabs(f[i] - feq[i]);
        eps /= (rho > 1e-300 ? rho : 1e-300);
        const double s = eps / (eps + m->eps0);
        for (int r = 0; r < 27; ++r) {
            if (ROW_DEG[r] < 3) continue;
            double v = rates[r] + (1.0 - rates[r]) * s;
            rates[r] = v < 0.05 ? 0.05 : (1.95 < v ? 1.95 : v);
        }
    }
    for (int mu = 0; mu < 27; ++mu) t[mu] *= rates[T2R[mu]];
    inv(t, 1, sx);
    inv(t, 3, sy);
    inv(t, 9, sz);
    for (int i = 0; i < 27; ++i) out[i] = -t[D2T[i]];
}

int orc_collide_batch(const lbmg_scene_config* cfg, size_t n, const double* f, const double* rho,
                      const double* u, double* omega) {
    model_t m;
    if (make_model(cfg, &m)) return 1;
    for (size_t k = 0; k < n; ++k) collide(f + 27 * k, rho[k], u + 3 * k, &m, omega + 27 * k);
    return 0;
}

/* ------------------------------------------------------ integer helpers */
/* morton3, ib.cpp:13-25 (bit-by-bit form; equal to the magic-mask form) */
uint64_t orc_morton3(uint32_t x, uint32_t y, uint32_t z) {
    uint64_t code = 0;
    for (int b = 0; b < 21; ++b) {
        code |= (uint64_t)((x >> b) & 1u) << (3 * b);
        code |= (uint64_t)((y >> b) & 1u) << (3 * b + 1);
        code |= (uint64_t)((z >> b) & 1u) << (3 * b + 2);
    }
    return code;
}

typedef struct {
    uint64_t a, b;
    uint32_t c, idx;
} key_t;

static int key_cmp(const void* pa, const void* pb) {
    const key_t* a = (const key_t*)pa;
    const key_t* b = (const key_t*)pb;
    if (a->a != b->a) return a->a < b->a ? -1 : 1;
    if (a->b != b->b) return a->b < b->b ? -1 : 1;
    if (a->c != b->c) return a->c < b->c ? -1 : 1;
    return 0;
}

/* reorder_samples, ib.cpp:231-292 */
int orc_reorder_permutation(size_t n, const double* pos, const uint32_t* src, int ell, uint32_t* perm) {
    if (ell < 1) return 1;
    if (n == 0) return 0;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (size_t s = 0; s < n; ++s)
        for (int a = 0; a < 3; ++a) {
            if (pos[3 * s + a] < lo[a]) lo[a] = pos[3 * s + a];
            if (pos[3 * s + a] > hi[a]) hi[a] = pos[3 * s + a];
        }
    int base[3], nb[3];
    for (int a = 0; a < 3; ++a) {
        base[a] = (int)floor(lo[a]);
        nb[a] = ((int)floor(hi[a]) - base[a]) / ell + 1;
    }
    key_t* k = (key_t*)malloc(n * sizeof *k);
    for (size_t s = 0; s < n; ++s) {
        int b[3], l[3];
        for (int a = 0; a < 3; ++a) {
            int cell = (int)floor(pos[3 * s + a]) - base[a];
            b[a] = cell / ell;
            l[a] = cell - b[a] * ell;
        }
        k[s].a = (uint64_t)b[0] + (uint64_t)nb[0] * ((uint64_t)b[1] + (uint64_t)nb[1] * (uint64_t)b[2]);
        k[s].b = orc_morton3((uint32_t)l[0], (uint32_t)l[1], (uint32_t)l[2]);
        k[s].c = src[s];
        k[s].idx = (uint32_t)s;
    }
    qsort(k, n, sizeof *k, key_cmp);
    for (size_t s = 0; s < n; ++s) perm[s] = k[s].idx;
    free(k);
    return 0;
}

/* split_domain, decomp.cpp:5-18 */
int orc_split_domain(int nz, int m, int* z0z1) {
    if (m < 1 || m > nz) return 1;
    int base = nz / m, rem = nz % m, z = 0;
    for (int r = 0; r < m; ++r) {
        int size = base + (r < rem ? 1 : 0);
        z0z1[2 * r] = z;
        z0z1[2 * r + 1] = z + size;
        z += size;
    }
    return 0;
}

/* face_owns_direction, boundary.cpp:18-40 */
static int exits(const int* ext, const int* coord, const int* c, int f) {
    int a = f / 2, src = coord[a] - c[a];
    return (f % 2 == 0) ? src < 0 : src >= ext[a];
}

static int owner(const int* ext, const int* per, int x, int y, int z, int i) {
    const int coord[3] = {x, y, z};
    for (int f = 0; f < 6; ++f) {
        if (per[f / 2]) continue;
        if (exits(ext, coord, C3[i], f)) return f;
    }
    return 255;
}

void orc_face_owner(const lbmg_scene_config* cfg, uint8_t* out) {
    tables();
    const int ext[3] = {cfg->nx, cfg->ny, cfg->nz};
    int per[3];
    for (int a = 0; a < 3; ++a) per[a] = cfg->faces[2 * a].condition == LBMG_PERIODIC;
    size_t k = 0;
    for (int z = 0; z < cfg->nz; ++z)
        for (int y = 0; y < cfg->ny; ++y)
            for (int x = 0; x < cfg->nx; ++x, ++k)
                for (int i = 0; i < 27; ++i) out[27 * k + i] = (uint8_t)owner(ext, per, x, y, z, i);
}

/* kernel_support, ib.cpp:294-308 */
int orc_kernel_support(const double* pos, int nx, int ny, int nz, int* base, double* w) {
    const int n[3] = {nx, ny, nz};
    int inside = 1;
    for (int a = 0; a < 3; ++a) {
        if (pos[a] < 0.0 || pos[a] > n[a] - 1) inside = 0;
        int b = (int)floor(pos[a]);
        if (b > n[a] - 2) b = n[a] - 2;
        if (b < 0) b = 0;
        base[a] = b;
        const double t = pos[a] - b;
        w[2 * a] = 1.0 - t;
        w[2 * a + 1] = t;
    }
    return inside;
}

/* ---------------------------------------------------------------- runner */
typedef struct {
    size_t n;
    double *pos, *ref, *ub, *force, *sampled;
    uint32_t* src;
    uint8_t* flagged;
    int moving;
    double lin[3], ang[3], center[3];
} solid_t;

struct orc_state {
    int nx, ny, nz;
    size_t n;
    int cond[6], per[3];
    double inlet[6][27];
    double body[3];
    model_t m;
    int ib_det;
    double *f, *fs, *rho, *u, *g;
    long t;
    lbmg_status status;
    int nsol;
    solid_t* sol;
    double* totals;
    size_t ntot, cap_tot;
};

static size_t nidx(const orc_state* s, int x, int y, int z) {
    return ((size_t)z * s->ny + y) * s->nx + x;
}

/* update_rigid_motion, ib.cpp:456-489 */
static void rigid_motion(orc_state* s, solid_t* so, long t) {
    const double td = (double)t;
    const double c[3] = {so->center[0] + so->lin[0] * td, so->center[1] + so->lin[1] * td,
                         so->center[2] + so->lin[2] * td};
    const double* w = so->ang;
    const double wn = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    double R[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    if (wn > 0.0) {
        const double ax = w[0] * (1.0 / wn), ay = w[1] * (1.0 / wn), az = w[2] * (1.0 / wn);
        const double th = wn * td, ct = cos(th), st = sin(th), vt = 1.0 - ct;
        R[0][0] = ct + ax * ax * vt;
        R[0][1] = ax * ay * vt - az * st;
        R[0][2] = ax * az * vt + ay * st;
        R[1][0] = ay * ax * vt + az * st;
        R[1][1] = ct + ay * ay * vt;
        R[1][2] = ay * az * vt - ax * st;
        R[2][0] = az * ax * vt - ay * st;
        R[2][1] = az * ay * vt + ax * st;
        R[2][2] = ct + az * az * vt;
    }
    for (size_t k = 0; k < so->n; ++k) {
        const double* r = so->ref + 3 * k;
        double* p = so->pos + 3 * k;
        for (int a = 0; a < 3; ++a) p[a] = c[a] + (R[a][0] * r[0] + R[a][1] * r[1] + R[a][2] * r[2]);
        const double d[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
        so->ub[3 * k + 0] = so->lin[0] + (w[1] * d[2] - w[2] * d[1]);
        so->ub[3 * k + 1] = so->lin[1] + (w[2] * d[0] - w[0] * d[2]);
        so->ub[3 * k + 2] = so->lin[2] + (w[0] * d[1] - w[1] * d[0]);
        int base[3];
        double ww[6];
        so->flagged[k] = orc_kernel_support(p, s->nx, s->ny, s->nz, base, ww) ? 0 : 1;
    }
}

/* init_fields, runner.cpp:60-107 (single region) */
static void init_fields(orc_state* s, const lbmg_scene_config* c) {
    for (int z = 0; z < s->nz; ++z)
        for (int y = 0; y < s->ny; ++y)
            for (int x = 0; x < s->nx; ++x) {
                double rho, u[3];
                if (c->init == LBMG_INIT_UNIFORM) {
                    rho = c->init_density;
                    memcpy(u, c->init_velocity, sizeof u);
                } else {
                    const double kx = 2.0 * M_PI / s->nx, ky = 2.0 * M_PI / s->ny, u0 = c->tg_u_max;
                    u[0] = -u0 * cos(kx * x) * sin(ky * y);
                    u[1] = u0 * sin(kx * x) * cos(ky * y);
                    u[2] = 0.0;
                    const double p = -0.25 * u0 * u0 * (cos(2.0 * kx * x) + cos(2.0 * ky * y));
                    rho = c->init_density + 3.0 * p;
                }
                const size_t k = nidx(s, x, y, z);
                orc_equilibrium(rho, u, s->f + 27 * k);
                memcpy(s->fs + 27 * k, s->f + 27 * k, 27 * sizeof(double));
                s->rho[k] = rho;
                memcpy(s->u + 3 * k, u, sizeof u);
            }
    for (int q = 0; q < s->nsol; ++q) rigid_motion(s, &s->sol[q], 0);
}

orc_state* orc_create(const lbmg_scene_config* c, const size_t* counts, const double* const* pos,
                      const double* const* ref, const uint32_t* const* src) {
    tables();
    orc_state* s = (orc_state*)calloc(1, sizeof *s);
    if (make_model(c, &s->m)) {
        free(s);
        return NULL;
    }
    s->nx = c->nx;
    s->ny = c->ny;
    s->nz = c->nz;
    s->n = (size_t)c->nx * c->ny * c->nz;
    for (int f = 0; f < 6; ++f) {
        s->cond[f] = c->faces[f].condition;
        orc_equilibrium(1.0, c->faces[f].velocity, s->inlet[f]);
    }
    for (int a = 0; a < 3; ++a) {
        s->per[a] = c->faces[2 * a].condition == LBMG_PERIODIC;
        s->body[a] = c->body_force[a];
    }
    s->ib_det = c->ib_mode == LBMG_IB_DETERMINISTIC;
    s->f = (double*)calloc(s->n * 27, sizeof(double));
    s->fs = (double*)calloc(s->n * 27, sizeof(double));
    s->rho = (double*)calloc(s->n, sizeof(double));
    s->u = (double*)calloc(s->n * 3, sizeof(double));
    s->g = (double*)calloc(s->n * 3, sizeof(double));
    s->status.ok = 1;
    s->status.step = -1;
    s->nsol = c->n_solids;
    s->sol = (solid_t*)calloc(s->nsol > 0 ? s->nsol : 1, sizeof(solid_t));
    for (int q = 0; q < s->nsol; ++q) {
        solid_t* so = &s->sol[q];
        const size_t n = counts[q];
        so->n = n;
        so->pos = (double*)malloc(3 * n * sizeof(double) + 8);
        so->ref = (double*)malloc(3 * n * sizeof(double) + 8);
        so->ub = (double*)calloc(3 * n + 1, sizeof(double));
        so->force = (double*)calloc(3 * n + 1, sizeof(double));
        so->sampled = (double*)calloc(3 * n + 1, sizeof(double));
        so->src = (uint32_t*)malloc(n * sizeof(uint32_t) + 4);
        so->flagged = (uint8_t*)calloc(n + 1, 1);
        memcpy(so->pos, pos[q], 3 * n * sizeof(double));
        memcpy(so->ref, ref[q], 3 * n * sizeof(double));
        memcpy(so->src, src[q], n * sizeof(uint32_t));
        const lbmg_solid_config* sc = &c->solids[q];
        so->moving = sc->has_motion;
        if (sc->has_motion) {
            memcpy(so->lin, sc->linear_velocity, sizeof so->lin);
            memcpy(so->ang, sc->angular_velocity, sizeof so->ang);
            memcpy(so->center, sc->center, sizeof so->center);
        }
    }
    init_fields(s, c);
    return s;
}

void orc_destroy(orc_state* s) {
    if (!s) return;
    for (int q = 0; q < s->nsol; ++q) {
        solid_t* so = &s->sol[q];
        free(so->pos);
        free(so->ref);
        free(so->ub);
        free(so->force);
        free(so->sampled);
        free(so->src);
        free(so->flagged);
    }
    free(s->sol);
    free(s->f);
    free(s->fs);
    free(s->rho);
    free(s->u);
    free(s->g);
    free(s->totals);
    free(s);
}

/* stream, solver.cpp:46-87 (single region: periodic z wraps locally) */
static void stream(orc_state* s) {
    for (int z = 0; z < s->nz; ++z)
        for (int y = 0; y < s->ny; ++y)
            for (int x = 0; x < s->nx; ++x) {
                const size_t k = nidx(s, x, y, z);
                for (int i = 0; i < 27; ++i) {
                    int sx = x - C3[i][0], sy = y - C3[i][1], sz = z - C3[i][2];
                    if (sx < 0 || sx >= s->nx) {
                        if (!s->per[0]) continue;
                        sx = (sx + s->nx) % s->nx;
                    }
                    if (sy < 0 || sy >= s->ny) {
                        if (!s->per[1]) continue;
                        sy = (sy + s->ny) % s->ny;
                    }
                    if (sz < 0 || sz >= s->nz) {
                        if (!s->per[2]) continue;
                        sz = (sz + s->nz) % s->nz;
                    }
                    s->fs[27 * k + i] = s->f[27 * nidx(s, sx, sy, sz) + i];
                }
            }
}

/* apply_face / apply_domain_boundaries, boundary.cpp:42-125 */
static void faces(orc_state* s) {
    const int ext[3] = {s->nx, s->ny, s->nz};
    for (int f = 0; f < 6; ++f) {
        if (s->cond[f] == LBMG_PERIODIC) continue;
        const int a = f / 2, side = f % 2 == 0 ? -1 : 1;
        const int plane = side < 0 ? 0 : ext[a] - 1;
        for (int z = 0; z < s->nz; ++z)
            for (int y = 0; y < s->ny; ++y)
                for (int x = 0; x < s->nx; ++x) {
                    const int coord[3] = {x, y, z};
                    if (coord[a] != plane) continue;
                    const size_t k = nidx(s, x, y, z);
                    for (int i = 0; i < 27; ++i) {
                        if (!((side < 0 && C3[i][a] > 0) || (side > 0 && C3[i][a] < 0))) continue;
                        if (owner(ext, s->per, x, y, z, i) != f) continue;
                        if (s->cond[f] == LBMG_NOSLIP) {
                            s->fs[27 * k + i] = s->f[27 * k + OPP[i]];
                        } else if (s->cond[f] == LBMG_INLET) {
                            s->fs[27 * k + i] = s->inlet[f][i];
                        } else {
                            int n[3] = {x, y, z};
                            n[a] -= side;
                            s->fs[27 * k + i] = s->fs[27 * nidx(s, n[0], n[1], n[2]) + i];
                        }
                    }
                }
    }
}

/* compute_moments, solver.cpp:89-137 */
static int moments(orc_state* s, int* mach) {
    int diverged = 0;
    for (size_t k = 0; k < s->n; ++k) {
        double r = 0.0, m[3] = {0.0, 0.0, 0.0};
        for (int i = 0; i < 27; ++i) {
            const double fi = s->fs[27 * k + i];
            r += fi;
            m[0] += C3[i][0] * fi;
            m[1] += C3[i][1] * fi;
            m[2] += C3[i][2] * fi;
        }
        if (!(r > 0.0) || !isfinite(r) || !isfinite(m[0]) || !isfinite(m[1]) || !isfinite(m[2])) {
            diverged = 1;
            s->rho[k] = r;
            continue;
        }
        const double inv_r = 1.0 / r;
        const double v[3] = {m[0] * inv_r, m[1] * inv_r, m[2] * inv_r};
        if (v[0] * v[0] + v[1] * v[1] + v[2] * v[2] >= 0.16) *mach = 1;
        s->rho[k] = r;
        memcpy(s->u + 3 * k, v, sizeof v);
        memcpy(s->g + 3 * k, s->body, sizeof s->body);
    }
    return diverged;
}

static int sample_active(const orc_state* s, double pz) {
    /* ib.cpp:313-317 with the single region [0, nz) */
    int bz = (int)floor(pz);
    if (bz > s->nz - 2) bz = s->nz - 2;
    if (bz < 0) bz = 0;
    return bz + 1 >= 0 && bz < s->nz;
}

/* interpolate_velocity + penalty_forces, ib.cpp:321-365 */
static void interp_penalty(orc_state* s, solid_t* so) {
    for (size_t q = 0; q < so->n; ++q) {
        int b[3];
        double w[6];
        const int inside = orc_kernel_support(so->pos + 3 * q, s->nx, s->ny, s->nz, b, w);
        so->flagged[q] = inside ? 0 : 1;
        double* us = so->sampled + 3 * q;
        double* fo = so->force + 3 * q;
        if (!inside || !sample_active(s, so->pos[3 * q + 2])) {
            us[0] = us[1] = us[2] = 0.0;
            fo[0] = fo[1] = fo[2] = 0.0;
            continue;
        }
        double v[3] = {0.0, 0.0, 0.0}, rs = 0.0;
        for (int oz = 0; oz < 2; ++oz)
            for (int oy = 0; oy < 2; ++oy)
                for (int ox = 0; ox < 2; ++ox) {
                    const double wt = w[ox] * w[2 + oy] * w[4 + oz];
                    const size_t k = nidx(s, b[0] + ox, b[1] + oy, b[2] + oz);
                    for (int a = 0; a < 3; ++a) v[a] += s->u[3 * k + a] * wt;
                }
        memcpy(us, v, sizeof v);
        for (int oz = 0; oz < 2; ++oz)
            for (int oy = 0; oy < 2; ++oy)
                for (int ox = 0; ox < 2; ++ox)
                    rs += w[ox] * w[2 + oy] * w[4 + oz] * s->rho[nidx(s, b[0] + ox, b[1] + oy, b[2] + oz)];
        for (int a = 0; a < 3; ++a) fo[a] = (so->ub[3 * q + a] - us[a]) * rs;
    }
}

/* scatter_one, ib.cpp:369-391 */
static void scatter(orc_state* s, const solid_t* so, size_t q) {
    int b[3];
    double w[6];
    orc_kernel_support(so->pos + 3 * q, s->nx, s->ny, s->nz, b, w);
    for (int oz = 0; oz < 2; ++oz)
        for (int oy = 0; oy < 2; ++oy)
            for (int ox = 0; ox < 2; ++ox) {
                const double wt = w[ox] * w[2 + oy] * w[4 + oz];
                const size_t k = nidx(s, b[0] + ox, b[1] + oy, b[2] + oz);
                for (int a = 0; a < 3; ++a) s->g[3 * k + a] += wt * so->force[3 * q + a];
            }
}

typedef struct {
    uint64_t key;
    uint32_t color, source, idx;
} rec_t;

static int rec_cmp(const void* pa, const void* pb) {
    const rec_t* a = (const rec_t*)pa;
    const rec_t* b = (const rec_t*)pb;
    if (a->color != b->color) return a->color < b->color ? -1 : 1;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->source != b->source) return a->source < b->source ? -1 : 1;
    return 0;
}

/* spread_forces, ib.cpp:393-454: atomic mode in storage order (the order a
 * single worker produces); deterministic mode in (colour, key, source) order */
static void spread(orc_state* s, const solid_t* so) {
    if (!s->ib_det) {
        for (size_t q = 0; q < so->n; ++q)
            if (!so->flagged[q] && sample_active(s, so->pos[3 * q + 2])) scatter(s, so, q);
        return;
    }
    rec_t* r = (rec_t*)malloc((so->n + 1) * sizeof *r);
    size_t nr = 0;
    for (size_t q = 0; q < so->n; ++q) {
        if (so->flagged[q] || !sample_active(s, so->pos[3 * q + 2])) continue;
        int b[3];
        double w[6];
        orc_kernel_support(so->pos + 3 * q, s->nx, s->ny, s->nz, b, w);
        uint32_t B[3], par = 0;
        for (int a = 0; a < 3; ++a) {
            B[a] = (uint32_t)(b[a] >> 1);
            par |= (B[a] & 1u) << a;
        }
        r[nr].key = orc_morton3(B[0], B[1], B[2]);
        r[nr].color = par;
        r[nr].source = so->src[q];
        r[nr].idx = (uint32_t)q;
        ++nr;
    }
    qsort(r, nr, sizeof *r, rec_cmp);
    for (size_t j = 0; j < nr; ++j) scatter(s, so, r[j].idx);
    free(r);
}

/* collide_pass, solver.cpp:149-179 */
static void collide_all(orc_state* s) {
    double om[27];
    for (size_t k = 0; k < s->n; ++k) {
        const double* fk = s->fs + 27 * k;
        collide(fk, s->rho[k], s->u + 3 * k, &s->m, om);
        const double* g = s->g + 3 * k;
        for (int i = 0; i < 27; ++i) {
            const double cg = C3[i][0] * g[0] + C3[i][1] * g[1] + C3[i][2] * g[2];
            const double Gi = W[i] * 3.0 * cg;
            s->f[27 * k + i] = fk[i] + om[i] + Gi;
        }
    }
}

/* Runner::advance, runner.cpp:121-230 (m = 1) */
int orc_advance(orc_state* s, long steps, lbmg_status* st) {
    for (long n = 0; n < steps; ++n) {
        if (!s->status.ok) break;
        stream(s);
        faces(s);
        int mach = 0;
        const int div = moments(s, &mach);
        if (mach) s->status.mach_warning = 1;
        if (div) {
            s->status.ok = 0;
            s->status.step = s->t;
            strcpy(s->status.reason, "divergence: non-positive or non-finite density");
            break;
        }
        if (s->nsol > 0) {
            for (int q = 0; q < s->nsol; ++q) {
                interp_penalty(s, &s->sol[q]);
                spread(s, &s->sol[q]);
            }
            double tot[6] = {0, 0, 0, 0, 0, 0};
            for (int q = 0; q < s->nsol; ++q) {
                /* reaction_totals, ib.cpp:491-501, centre c(t) */
                const solid_t* so = &s->sol[q];
                const double c[3] = {so->center[0] + so->lin[0] * (double)s->t,
                                     so->center[1] + so->lin[1] * (double)s->t,
                                     so->center[2] + so->lin[2] * (double)s->t};
                double part[6] = {0, 0, 0, 0, 0, 0};
                for (size_t k = 0; k < so->n; ++k) {
                    const double z = so->pos[3 * k + 2];
                    if (z < 0 || z >= s->nz) continue;
                    const double* F = so->force + 3 * k;
                    const double d[3] = {so->pos[3 * k] - c[0], so->pos[3 * k + 1] - c[1], z - c[2]};
                    part[0] -= F[0];
                    part[1] -= F[1];
                    part[2] -= F[2];
                    part[3] -= d[1] * F[2] - d[2] * F[1];
                    part[4] -= d[2] * F[0] - d[0] * F[2];
                    part[5] -= d[0] * F[1] - d[1] * F[0];
                }
                for (int a = 0; a < 6; ++a) tot[a] += part[a];
            }
            if (s->ntot == s->cap_tot) {
                s->cap_tot = s->cap_tot ? 2 * s->cap_tot : 64;
                s->totals = (double*)realloc(s->totals, s->cap_tot * 6 * sizeof(double));
            }
            memcpy(s->totals + 6 * s->ntot, tot, sizeof tot);
            ++s->ntot;
            for (int q = 0; q < s->nsol; ++q)
                if (s->sol[q].moving) rigid_motion(s, &s->sol[q], s->t + 1);
        }
        collide_all(s);
        ++s->t;
    }
    if (st) *st = s->status;
    return 0;
}

long orc_step_count(const orc_state* s) { return s->t; }

void orc_gather(const orc_state* s, int what, double* out) {
    if (what == 0) memcpy(out, s->rho, s->n * sizeof(double));
    else if (what == 1) memcpy(out, s->u, 3 * s->n * sizeof(double));
    else memcpy(out, s->f, 27 * s->n * sizeof(double));
}

size_t orc_totals_count(const orc_state* s) { return s->ntot; }
void orc_totals(const orc_state* s, double* out) { memcpy(out, s->totals, 6 * s->ntot * sizeof(double)); }

void orc_samples(const orc_state* s, int q, double* pos, double* ub, double* force, double* sampled,
                 uint8_t* flagged) {
    const solid_t* so = &s->sol[q];
    if (pos) memcpy(pos, so->pos, 3 * so->n * sizeof(double));
    if (ub) memcpy(ub, so->ub, 3 * so->n * sizeof(double));
    if (force) memcpy(force, so->force, 3 * so->n * sizeof(double));
    if (sampled) memcpy(sampled, so->sampled, 3 * so->n * sizeof(double));
    if (flagged) memcpy(flagged, so->flagged, so->n);
}

double* orc_f(orc_state* s) { return s->f; }
double* orc_f_star(orc_state* s) { return s->fs; }
