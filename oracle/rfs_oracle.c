/*
 * rfs_oracle.c -- CPU restatement of the reference RF-splatting rasterizer.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle for the B200
 * CUDA path and the "port" CPU baseline timed by bench.py.  It is never
 * linked into, loaded by, or called from the product path
 * (paper_2502_01826_b200/); only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may use it.
 *
 * Everything is float64 / complex128 like the reference package `rfsplat`
 * (numba @njit without fastmath, numpy).  Compile with -ffp-contract=off so
 * no FMA contraction changes roundings.  Each function cites the reference
 * file:line (paths under pkg/src/rfsplat/) whose algorithm it restates.
 *
 * Parity pinning: tests/golden/ holds vectors produced by the reference
 * itself (tests/golden/make_golden.py); tests/test_oracle_golden.py checks
 * this restatement against them.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TERM_EPS2 1e-12   /* _kernels.py:20 */
#define TANGENT_EPS 1e-10 /* _kernels.py:22 */
#define TILE 16           /* _kernels.py:24, splat.py:57 */

static const double PI = 3.141592653589793;
static const double TWO_PI = 6.283185307179586;
static const double RAD2DEG = 57.29577951308232; /* 180/pi, splat.py:58 */
static const double GAUSS_NORM = 0.06349363593424097; /* (2pi)^-1.5, render.py:48 */

typedef struct { double re, im; } cx;
static inline cx cx_mk(double r, double i) { cx z; z.re = r; z.im = i; return z; }
static inline cx cx_mul(cx a, cx b) { return cx_mk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static inline cx cx_add(cx a, cx b) { return cx_mk(a.re + b.re, a.im + b.im); }
static inline cx cx_rmul(double s, cx a) { return cx_mk(s * a.re, s * a.im); }
static inline cx cx_conj(cx a) { return cx_mk(a.re, -a.im); }

/* Shared context: scene arrays (read), derived arrays (written).  Python owns
 * every buffer (oracle/__init__.py mirrors this layout with ctypes). */
typedef struct {
    int64_t n, n_az, n_el, degree, n_coeffs, tiles_u, tiles_v, m;
    double rx[3], tx[3], ress_radius;
    const double *means, *quats, *log_scales, *raw, *phase, *coeffs; /* coeffs: n*K complex interleaved */
    double *covs, *inv_covs, *norm_consts, *rho, *unit_rho;          /* rho/unit_rho: complex interleaved */
    double *bearing_alpha, *bearing_beta;
    uint8_t *bearing_valid;
    double *basis, *basis_dalpha, *basis_dbeta, *psi;                /* complex interleaved */
    uint8_t *active;
    double *center_u, *center_v, *radius_px, *tile_radius, *depth, *splat_r2;
    double *ray_dirs;
    uint64_t *keys;
    int64_t *indices, *ranges;
} orc_ctx;

/* ---------------------------------------------------------------- helpers */

/* numpy float remainder (npy_divmod): result carries the divisor's sign. */
static double py_fmod(double a, double b) {
    double m = fmod(a, b);
    if (m != 0.0) {
        if ((b < 0.0) != (m < 0.0)) m += b;
    } else {
        m = copysign(0.0, b);
    }
    return m;
}
static int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}
static int64_t py_imod(int64_t a, int64_t b) { return a - floordiv(a, b) * b; }
static double clip(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

/* quats_to_rotations, scene.py:118-142 (normalizes first). */
static void quat_rot(const double *q4, double r[9]) {
    double nrm = sqrt(q4[0] * q4[0] + q4[1] * q4[1] + q4[2] * q4[2] + q4[3] * q4[3]);
    double w = q4[0] / nrm, x = q4[1] / nrm, y = q4[2] / nrm, z = q4[3] / nrm;
    r[0] = 1 - 2 * (y * y + z * z); r[1] = 2 * (x * y - w * z);     r[2] = 2 * (x * z + w * y);
    r[3] = 2 * (x * y + w * z);     r[4] = 1 - 2 * (x * x + z * z); r[5] = 2 * (y * z - w * x);
    r[6] = 2 * (x * z - w * y);     r[7] = 2 * (y * z + w * x);     r[8] = 1 - 2 * (x * x + y * y);
}

/* --------------------------------------------------- per-scene preparation */

/* covariances (scene.py:157-161), inverse + symmetrize + det normalizer and
 * complex transmittance (render.py:220-227). */
static void prepare_shapes(orc_ctx *c) {
    for (int64_t g = 0; g < c->n; ++g) {
        double r[9];
        quat_rot(c->quats + 4 * g, r);
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = exp(2.0 * c->log_scales[3 * g + a]);
        double *S = c->covs + 9 * g;
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j) acc += r[3 * i + j] * d[j] * r[3 * k + j];
                S[3 * i + k] = acc;
            }
        /* cofactor inverse of the 3x3 (numpy uses LU; agreement ~1e-16 rel) */
        double c00 = S[4] * S[8] - S[5] * S[7];
        double c01 = S[5] * S[6] - S[3] * S[8];
        double c02 = S[3] * S[7] - S[4] * S[6];
        double det = S[0] * c00 + S[1] * c01 + S[2] * c02;
        double inv[9];
        inv[0] = c00 / det;
        inv[1] = (S[2] * S[7] - S[1] * S[8]) / det;
        inv[2] = (S[1] * S[5] - S[2] * S[4]) / det;
        inv[3] = c01 / det;
        inv[4] = (S[0] * S[8] - S[2] * S[6]) / det;
        inv[5] = (S[2] * S[3] - S[0] * S[5]) / det;
        inv[6] = c02 / det;
        inv[7] = (S[1] * S[6] - S[0] * S[7]) / det;
        inv[8] = (S[0] * S[4] - S[1] * S[3]) / det;
        double *I = c->inv_covs + 9 * g;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) I[3 * i + j] = 0.5 * (inv[3 * i + j] + inv[3 * j + i]);
        c->norm_consts[g] = GAUSS_NORM / sqrt(det);
        double mag = 1.0 / (1.0 + exp(-c->raw[g]));
        double ph = c->phase[g];
        c->unit_rho[2 * g] = cos(ph);
        c->unit_rho[2 * g + 1] = sin(ph);
        c->rho[2 * g] = mag * cos(ph);
        c->rho[2 * g + 1] = mag * sin(ph);
    }
}

/* project_scene, splat.py:212-268.  Returns 1 on GeometryError. */
static int project(orc_ctx *c) {
    double cell = 360.0 / (double)c->n_az;
    double cover_all = (double)(c->n_az + c->n_el);
    for (int64_t g = 0; g < c->n; ++g) {
        double x = c->means[3 * g] - c->rx[0];
        double y = c->means[3 * g + 1] - c->rx[1];
        double z = c->means[3 * g + 2] - c->rx[2];
        double depth = sqrt((x * x + y * y) + z * z);
        if (depth < 1e-9) return 1;
        c->depth[g] = depth;
        c->active[g] = depth >= c->ress_radius;
        double alpha = py_fmod(atan2(y, x), TWO_PI);
        double beta = PI / 2.0 - acos(clip(z / depth, -1.0, 1.0));
        c->center_u[g] = alpha * RAD2DEG / cell;
        c->center_v[g] = (beta * RAD2DEG + 90.0) / cell;

        /* linearized 3-sigma radius of J Sigma J^T (splat.py:236-254) */
        double rho2 = x * x + y * y;
        double r2 = rho2 + z * z;
        double pd = 1e-12 * depth;
        int polar = rho2 <= pd * pd;
        double rho_s = sqrt(polar ? 1.0 : rho2);
        double scale = RAD2DEG / cell;
        double rc = rho2 < 1e-300 ? 1e-300 : rho2;
        double J[6] = {-y / rc, x / rc, 0.0, -z * x / (rho_s * r2), -z * y / (rho_s * r2), rho_s / r2};
        for (int i = 0; i < 6; ++i) J[i] *= scale;
        const double *S = c->covs + 9 * g;
        double cv2[4];
        for (int i = 0; i < 2; ++i)
            for (int l = 0; l < 2; ++l) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j)
                    for (int k = 0; k < 3; ++k) acc += J[3 * i + j] * S[3 * j + k] * J[3 * l + k];
                cv2[2 * i + l] = acc;
            }
        double half_tr = 0.5 * (cv2[0] + cv2[3]);
        double det2 = cv2[0] * cv2[3] - cv2[1] * cv2[2];
        double disc = half_tr * half_tr - det2;
        double lam_max = half_tr + sqrt(disc > 0.0 ? disc : 0.0);
        c->radius_px[g] = polar ? cover_all : 3.0 * sqrt(lam_max > 0.0 ? lam_max : 0.0);

        /* conservative incidence radius (splat.py:256-267).  lambda_max of
         * R diag(e^{2s}) R^T is max_a e^{2 s_a} (eigvalsh in the reference). */
        double lam3 = 0.0;
        for (int a = 0; a < 3; ++a) {
            double e = exp(2.0 * c->log_scales[3 * g + a]);
            if (e > lam3) lam3 = e;
        }
        double r3 = 3.0 * sqrt(lam3);
        int inside = depth <= r3;
        double theta = asin(clip(r3 / depth, 0.0, 1.0));
        double ca = cos(beta - theta), cb = cos(beta + theta);
        double cos_lo = ca < cb ? ca : cb;
        double st = sin(theta);
        int pole_touch = cos_lo <= st;
        double az_extent = asin(clip(st / (pole_touch ? 1.0 : cos_lo), 0.0, 1.0));
        double extent = pole_touch ? PI : (theta > az_extent ? theta : az_extent);
        double tr = extent * RAD2DEG / cell + 2.0;
        if (tr > cover_all) tr = cover_all;
        if (inside || polar) tr = cover_all;
        c->tile_radius[g] = tr;
        c->splat_r2[g] = c->active[g] ? tr * tr : -1.0; /* render.py:243 */
    }
    return 0;
}

/* ray_directions, render.py:103-117 (ray id r = u * n_el + v). */
static void ray_dirs(orc_ctx *c) {
    double cell = 360.0 / (double)c->n_az;
    for (int64_t u = 0; u < c->n_az; ++u)
        for (int64_t v = 0; v < c->n_el; ++v) {
            double al = ((double)u + 0.5) * cell * (PI / 180.0);
            double be = (((double)v + 0.5) * cell - 90.0) * (PI / 180.0);
            double *d = c->ray_dirs + 3 * (u * c->n_el + v);
            d[0] = cos(be) * cos(al);
            d[1] = cos(be) * sin(al);
            d[2] = sin(be);
        }
}

int orc_prepare(orc_ctx *c) {
    c->tiles_u = (c->n_az + TILE - 1) / TILE;
    c->tiles_v = (c->n_el + TILE - 1) / TILE;
    prepare_shapes(c);
    ray_dirs(c);
    return project(c);
}

/* -------------------------------------------------------- FLE + bearing */

static double dfact(int n) {
    double o = 1.0;
    while (n > 1) { o *= n; n -= 2; }
    return o;
}
static double fact(int n) {
    double o = 1.0;
    for (int i = 2; i <= n; ++i) o *= i;
    return o;
}

/* fle_basis_with_derivs for one direction, fle.py:153-212.  Outputs complex
 * interleaved arrays of length (L+1)^2 at index l*l + l + m. */
static void fle_one(double alpha, double beta, int L, double *basis, double *da, double *db) {
    double p[8][8], dp[8][8];
    double x = cos(beta), sg = sin(beta);
    double s = fabs(sg);
    double sgn = (sg > 0.0) - (sg < 0.0);
    double dx = -sg, ds = sgn * x;
    int n1 = L + 1;
    for (int i = 0; i < n1; ++i)
        for (int j = 0; j < n1; ++j) { p[i][j] = 0.0; dp[i][j] = 0.0; }
    for (int m = 0; m < n1; ++m) {
        double cc = ((m & 1) ? -1.0 : 1.0) * dfact(2 * m - 1);
        p[m][m] = cc * pow(s, (double)m);
        if (m > 0) dp[m][m] = cc * m * pow(s, (double)(m - 1)) * ds;
        if (m + 1 <= L) {
            p[m + 1][m] = x * (2 * m + 1) * p[m][m];
            dp[m + 1][m] = (2 * m + 1) * (dx * p[m][m] + x * dp[m][m]);
        }
        for (int l = m + 2; l < n1; ++l) {
            double a = 2 * l - 1, b = l + m - 1;
            p[l][m] = (x * a * p[l - 1][m] - b * p[l - 2][m]) / (l - m);
            dp[l][m] = (dx * a * p[l - 1][m] + x * a * dp[l - 1][m] - b * dp[l - 2][m]) / (l - m);
        }
    }
    for (int l = 0; l < n1; ++l)
        for (int m = -l; m <= l; ++m) {
            int ma = m < 0 ? -m : m;
            double pv = p[l][ma], dv = dp[l][ma];
            if (m < 0) {
                double ratio = ((ma & 1) ? -1.0 : 1.0) * (fact(l - ma) / fact(l + ma));
                pv = ratio * pv;
                dv = ratio * dv;
            }
            double ang = m * alpha;
            cx az = cx_mk(cos(ang), sin(ang));
            int idx = l * l + l + m;
            basis[2 * idx] = az.re * pv;
            basis[2 * idx + 1] = az.im * pv;
            cx im = cx_mk(0.0, (double)m);
            cx dA = cx_mul(im, az);
            da[2 * idx] = dA.re * pv;
            da[2 * idx + 1] = dA.im * pv;
            db[2 * idx] = az.re * dv;
            db[2 * idx + 1] = az.im * dv;
        }
}

/* Bearing toward tx, FLE basis and psi = sum_k c_k basis_k, render.py:229-238. */
int orc_set_tx(orc_ctx *c) {
    int64_t K = c->n_coeffs;
    for (int64_t g = 0; g < c->n; ++g) {
        double x = c->tx[0] - c->means[3 * g];
        double y = c->tx[1] - c->means[3 * g + 1];
        double z = c->tx[2] - c->means[3 * g + 2];
        double dist = sqrt((x * x + y * y) + z * z);
        int valid = dist > 1e-12;
        double safe = valid ? dist : 1.0;
        double alpha = py_fmod(atan2(y, x), TWO_PI);
        double beta = PI / 2.0 - acos(clip(z / safe, -1.0, 1.0));
        if (!valid) { alpha = 0.0; beta = 0.0; }
        c->bearing_alpha[g] = alpha;
        c->bearing_beta[g] = beta;
        c->bearing_valid[g] = (uint8_t)valid;
        double *B = c->basis + 2 * K * g, *DA = c->basis_dalpha + 2 * K * g, *DB = c->basis_dbeta + 2 * K * g;
        fle_one(alpha, beta, (int)c->degree, B, DA, DB);
        cx acc = cx_mk(0.0, 0.0);
        for (int64_t k = 0; k < K; ++k)
            acc = cx_add(acc, cx_mul(cx_mk(c->coeffs[2 * (K * g + k)], c->coeffs[2 * (K * g + k) + 1]),
                                     cx_mk(B[2 * k], B[2 * k + 1])));
        c->psi[2 * g] = acc.re;
        c->psi[2 * g + 1] = acc.im;
    }
    return 0;
}

/* -------------------------------------------------------------- binning */

typedef struct { int64_t s1_lo, s1_hi, s2_lo, s2_hi, tv_lo, tv_hi; } rect_t;

/* Tile rectangle of one splat, splat.py:308-328. */
static rect_t splat_rect(double cu, double cv, double radius, int64_t n_az, int64_t n_el, int64_t tiles_u) {
    rect_t r;
    double flo = floor(cv - radius), fhi = floor(cv + radius);
    int64_t v_lo = (int64_t)flo, v_hi = (int64_t)fhi;
    if (v_lo < 0) v_lo = 0;
    if (v_lo > n_el - 1) v_lo = n_el - 1;
    if (v_hi < -1) v_hi = -1;
    if (v_hi > n_el - 1) v_hi = n_el - 1;
    int off_grid = (fhi < 0.0) || (flo > (double)(n_el - 1));
    r.tv_lo = floordiv(v_lo, TILE);
    r.tv_hi = off_grid ? -1 : floordiv(v_hi, TILE);
    int64_t u_lo = (int64_t)floor(cu - radius), u_hi = (int64_t)floor(cu + radius);
    int span_all = (u_hi - u_lo + 1) >= n_az;
    int64_t a = py_imod(u_lo, n_az);
    int64_t b = a + (u_hi - u_lo);
    int wrap = b > n_az - 1;
    r.s1_lo = floordiv(a, TILE);
    r.s1_hi = wrap ? tiles_u - 1 : floordiv(b < n_az - 1 ? b : n_az - 1, TILE);
    r.s2_lo = 0;
    r.s2_hi = wrap ? floordiv(b - n_az, TILE) : -1;
    int full = span_all || (wrap && (r.s2_hi >= r.s1_lo));
    if (full) { r.s1_lo = 0; r.s1_hi = tiles_u - 1; r.s2_hi = -1; }
    return r;
}

/* Count pass of expand_tile_rects (_kernels.py:532-541) over active splats. */
int64_t orc_tiles_count(orc_ctx *c) {
    int64_t total = 0;
    for (int64_t g = 0; g < c->n; ++g) {
        if (!c->active[g]) continue;
        rect_t r = splat_rect(c->center_u[g], c->center_v[g], c->tile_radius[g], c->n_az, c->n_el, c->tiles_u);
        int64_t nv = r.tv_hi - r.tv_lo + 1;
        if (nv <= 0) continue;
        int64_t nu = r.s1_hi - r.s1_lo + 1;
        if (r.s2_hi >= r.s2_lo) nu += r.s2_hi - r.s2_lo + 1;
        total += nv * nu;
    }
    return total;
}

typedef struct { uint64_t key; int64_t pos; } kp_t;
static int kp_cmp(const void *a, const void *b) {
    const kp_t *x = (const kp_t *)a, *y = (const kp_t *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* Fill pass of expand_tile_rects (_kernels.py:542-559), stable argsort by key
 * and per-tile ranges (splat.py:330-343).  c->m must hold orc_tiles_count. */
int orc_tiles_fill(orc_ctx *c) {
    int64_t M = c->m, pos = 0;
    kp_t *kp = (kp_t *)malloc(sizeof(kp_t) * (M > 0 ? M : 1));
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (M > 0 ? M : 1));
    if (!kp || !idx) { free(kp); free(idx); return 5; }
    for (int64_t g = 0; g < c->n; ++g) {
        if (!c->active[g]) continue;
        rect_t r = splat_rect(c->center_u[g], c->center_v[g], c->tile_radius[g], c->n_az, c->n_el, c->tiles_u);
        if (r.tv_hi < r.tv_lo) continue;
        float df = (float)c->depth[g];
        uint32_t code;
        memcpy(&code, &df, 4);
        for (int64_t tv = r.tv_lo; tv <= r.tv_hi; ++tv) {
            int64_t row = tv * c->tiles_u;
            for (int64_t tu = r.s1_lo; tu <= r.s1_hi; ++tu) {
                kp[pos].key = ((uint64_t)(row + tu) << 32) | code; kp[pos].pos = pos; idx[pos] = g; ++pos;
            }
            for (int64_t tu = r.s2_lo; tu <= r.s2_hi; ++tu) {
                kp[pos].key = ((uint64_t)(row + tu) << 32) | code; kp[pos].pos = pos; idx[pos] = g; ++pos;
            }
        }
    }
    if (pos != M) { free(kp); free(idx); return 3; }
    qsort(kp, (size_t)M, sizeof(kp_t), kp_cmp); /* (key, position) == stable */
    int64_t n_tiles = c->tiles_u * c->tiles_v;
    for (int64_t t = 0; t < n_tiles; ++t) { c->ranges[2 * t] = 0; c->ranges[2 * t + 1] = 0; }
    for (int64_t i = 0; i < M; ++i) {
        c->keys[i] = kp[i].key;
        c->indices[i] = idx[kp[i].pos];
    }
    /* searchsorted left/right of each tile id over tile_of = keys >> 32 */
    int64_t i = 0;
    for (int64_t t = 0; t < n_tiles; ++t) {
        while (i < M && (int64_t)(c->keys[i] >> 32) < t) ++i;
        c->ranges[2 * t] = i;
        while (i < M && (int64_t)(c->keys[i] >> 32) == t) ++i;
        c->ranges[2 * t + 1] = i;
    }
    free(kp);
    free(idx);
    return 0;
}

/* ------------------------------------------------------------ hit lists */

typedef struct {
    int64_t m;
    int64_t *g;
    double *mu, *inv, *nc, *cu, *cv, *r2;
} tile_cand_t;

/* _gather_tile, _kernels.py:115-137. */
static void gather_tile(const orc_ctx *c, int64_t lo, int64_t hi, tile_cand_t *tc) {
    int64_t m = hi - lo;
    tc->m = m;
    tc->g = (int64_t *)malloc(sizeof(int64_t) * m);
    tc->mu = (double *)malloc(sizeof(double) * 3 * m);
    tc->inv = (double *)malloc(sizeof(double) * 9 * m);
    tc->nc = (double *)malloc(sizeof(double) * m);
    tc->cu = (double *)malloc(sizeof(double) * m);
    tc->cv = (double *)malloc(sizeof(double) * m);
    tc->r2 = (double *)malloc(sizeof(double) * m);
    for (int64_t i = 0; i < m; ++i) {
        int64_t g = c->indices[lo + i];
        tc->g[i] = g;
        for (int a = 0; a < 3; ++a) tc->mu[3 * i + a] = c->means[3 * g + a];
        for (int a = 0; a < 9; ++a) tc->inv[9 * i + a] = c->inv_covs[9 * g + a];
        tc->nc[i] = c->norm_consts[g];
        tc->cu[i] = c->center_u[g];
        tc->cv[i] = c->center_v[g];
        tc->r2[i] = c->splat_r2[g];
    }
}
static void free_tile(tile_cand_t *tc) {
    free(tc->g); free(tc->mu); free(tc->inv); free(tc->nc); free(tc->cu); free(tc->cv); free(tc->r2);
}

typedef struct { int64_t *g; double *tmid, *w, *d1, *d2; uint8_t *clamped; } hits_t;

static void hits_alloc(hits_t *h, int64_t m) {
    int64_t k = m > 0 ? m : 1;
    h->g = (int64_t *)malloc(sizeof(int64_t) * k);
    h->tmid = (double *)malloc(sizeof(double) * k);
    h->w = (double *)malloc(sizeof(double) * k);
    h->d1 = (double *)malloc(sizeof(double) * k);
    h->d2 = (double *)malloc(sizeof(double) * k);
    h->clamped = (uint8_t *)malloc(k);
}
static void hits_free(hits_t *h) { free(h->g); free(h->tmid); free(h->w); free(h->d1); free(h->d2); free(h->clamped); }

/* _collect_hits, _kernels.py:27-112: disc prefilter, 3-sigma quadratic,
 * midpoint density, insertion sort by (t_mid, global id). */
static int64_t collect_hits(double u, double v, const double *dir, const tile_cand_t *tc, const double *rx,
                            double min_t, double n_az, int use_disc, hits_t *h) {
    double dx = dir[0], dy = dir[1], dz = dir[2];
    int64_t count = 0;
    for (int64_t ci = 0; ci < tc->m; ++ci) {
        double r2 = tc->r2[ci];
        if (r2 < 0.0) continue;
        if (use_disc) {
            double du = fabs(u - tc->cu[ci]);
            if (n_az - du < du) du = n_az - du;
            double dv = v - tc->cv[ci];
            if (du * du + dv * dv > r2) continue;
        }
        const double *mu = tc->mu + 3 * ci, *I = tc->inv + 9 * ci;
        double mx = rx[0] - mu[0], my = rx[1] - mu[1], mz = rx[2] - mu[2];
        double i00 = I[0], i01 = I[1], i02 = I[2], i11 = I[4], i12 = I[5], i22 = I[8];
        double sx = i00 * dx + i01 * dy + i02 * dz;
        double sy = i01 * dx + i11 * dy + i12 * dz;
        double sz = i02 * dx + i12 * dy + i22 * dz;
        double a = sx * dx + sy * dy + sz * dz;
        double b = sx * mx + sy * my + sz * mz;
        double cq = (i00 * mx + i01 * my + i02 * mz) * mx + (i01 * mx + i11 * my + i12 * mz) * my +
                    (i02 * mx + i12 * my + i22 * mz) * mz;
        double disc = b * b - a * (cq - 9.0);
        if (disc < 0.0) continue;
        double sq = sqrt(disc);
        double d2 = (-b + sq) / a;
        if (d2 < min_t) continue;
        double d1 = (-b - sq) / a;
        int clamped = d1 < min_t;
        double t_in = clamped ? min_t : d1;
        double t_mid = 0.5 * (t_in + d2);
        double ex = t_mid * dx + mx, ey = t_mid * dy + my, ez = t_mid * dz + mz;
        double qf = (i00 * ex + i01 * ey + i02 * ez) * ex + (i01 * ex + i11 * ey + i12 * ez) * ey +
                    (i02 * ex + i12 * ey + i22 * ez) * ez;
        double w = tc->nc[ci] * exp(-0.5 * qf);
        int64_t g = tc->g[ci];
        int64_t j = count;
        while (j > 0 && (h->tmid[j - 1] > t_mid || (h->tmid[j - 1] == t_mid && h->g[j - 1] > g))) {
            h->tmid[j] = h->tmid[j - 1]; h->g[j] = h->g[j - 1]; h->w[j] = h->w[j - 1];
            h->d1[j] = h->d1[j - 1]; h->d2[j] = h->d2[j - 1]; h->clamped[j] = h->clamped[j - 1];
            --j;
        }
        h->tmid[j] = t_mid; h->g[j] = g; h->w[j] = w; h->d1[j] = d1; h->d2[j] = d2; h->clamped[j] = (uint8_t)clamped;
        ++count;
    }
    return count;
}

static inline cx rho_of(const orc_ctx *c, int64_t g) { return cx_mk(c->rho[2 * g], c->rho[2 * g + 1]); }
static inline cx psi_of(const orc_ctx *c, int64_t g) { return cx_mk(c->psi[2 * g], c->psi[2 * g + 1]); }

/* forward_tiled, _kernels.py:140-192.  out: n_az*n_el complex interleaved. */
int orc_forward(orc_ctx *c, double *out, int threads) {
    set_threads(threads);
    int64_t n_tiles = c->tiles_u * c->tiles_v;
    double n_az = (double)c->n_az;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < n_tiles; ++t) {
        int64_t lo = c->ranges[2 * t], hi = c->ranges[2 * t + 1];
        int64_t tu0 = (t % c->tiles_u) * TILE, tv0 = (t / c->tiles_u) * TILE;
        int64_t u_end = tu0 + TILE < c->n_az ? tu0 + TILE : c->n_az;
        int64_t v_end = tv0 + TILE < c->n_el ? tv0 + TILE : c->n_el;
        if (hi == lo) {
            for (int64_t u = tu0; u < u_end; ++u)
                for (int64_t v = tv0; v < v_end; ++v) { out[2 * (u * c->n_el + v)] = 0.0; out[2 * (u * c->n_el + v) + 1] = 0.0; }
            continue;
        }
        tile_cand_t tc;
        gather_tile(c, lo, hi, &tc);
        hits_t h;
        hits_alloc(&h, tc.m);
        for (int64_t u = tu0; u < u_end; ++u)
            for (int64_t v = tv0; v < v_end; ++v) {
                int64_t r = u * c->n_el + v;
                int64_t count = collect_hits((double)u, (double)v, c->ray_dirs + 3 * r, &tc, c->rx, c->ress_radius, n_az, 1, &h);
                cx s = cx_mk(0.0, 0.0), tr = cx_mk(1.0, 0.0);
                for (int64_t k = 0; k < count; ++k) {
                    if (tr.re * tr.re + tr.im * tr.im < TERM_EPS2) break;
                    int64_t g = h.g[k];
                    s = cx_add(s, cx_mul(cx_rmul(h.w[k], psi_of(c, g)), tr));
                    tr = cx_mul(tr, rho_of(c, g));
                }
                out[2 * r] = s.re;
                out[2 * r + 1] = s.im;
            }
        hits_free(&h);
        free_tile(&tc);
    }
    return 0;
}

/* forward_naive, _kernels.py:195-234 (every active primitive vs every ray). */
int orc_forward_naive(orc_ctx *c, double *out, int threads) {
    set_threads(threads);
    tile_cand_t tc;
    tc.m = c->n;
    tc.g = (int64_t *)malloc(sizeof(int64_t) * (c->n > 0 ? c->n : 1));
    for (int64_t g = 0; g < c->n; ++g) tc.g[g] = g;
    tc.mu = (double *)c->means;
    tc.inv = c->inv_covs;
    tc.nc = c->norm_consts;
    tc.cu = tc.cv = NULL;
    tc.r2 = c->splat_r2;
    int64_t R = c->n_az * c->n_el;
#pragma omp parallel
    {
        hits_t h;
        hits_alloc(&h, c->n);
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < R; ++r) {
            int64_t count = collect_hits(0.0, 0.0, c->ray_dirs + 3 * r, &tc, c->rx, c->ress_radius, (double)c->n_az, 0, &h);
            cx s = cx_mk(0.0, 0.0), tr = cx_mk(1.0, 0.0);
            for (int64_t k = 0; k < count; ++k) {
                if (tr.re * tr.re + tr.im * tr.im < TERM_EPS2) break;
                int64_t g = h.g[k];
                s = cx_add(s, cx_mul(cx_rmul(h.w[k], psi_of(c, g)), tr));
                tr = cx_mul(tr, rho_of(c, g));
            }
            out[2 * r] = s.re;
            out[2 * r + 1] = s.im;
        }
        hits_free(&h);
    }
    free(tc.g);
    return 0;
}

/* _live_hits, _kernels.py:237-247. */
static int64_t live_hits(const orc_ctx *c, int64_t count, const hits_t *h) {
    cx tr = cx_mk(1.0, 0.0);
    int64_t live = 0;
    for (int64_t k = 0; k < count; ++k) {
        if (tr.re * tr.re + tr.im * tr.im < TERM_EPS2) break;
        tr = cx_mul(tr, rho_of(c, h->g[k]));
        ++live;
    }
    return live;
}

/* Per-(ray,hit) slot outputs, grad.py:226-231. */
typedef struct { int64_t *g; double *pg, *dmag, *dphase, *dmu, *dcov; } slots_t;

/* _ray_backward, _kernels.py:360-522: reverse sweep with a running suffix. */
static void ray_backward(const orc_ctx *c, int64_t r, cx lam, int64_t live, const hits_t *h, const cx *trans,
                         int64_t base, slots_t *sl) {
    cx clam = cx_conj(lam);
    const double *dir = c->ray_dirs + 3 * r;
    double dx = dir[0], dy = dir[1], dz = dir[2];
    const double *rx = c->rx;
    double min_t = c->ress_radius;
    cx suffix = cx_mk(0.0, 0.0);
    for (int64_t k = live - 1; k >= 0; --k) {
        int64_t g = h->g[k];
        double w = h->w[k];
        cx tk = trans[k];
        int64_t slot = base + k;
        sl->g[slot] = g;
        cx pg = cx_mul(cx_rmul(w, clam), tk);
        sl->pg[2 * slot] = pg.re;
        sl->pg[2 * slot + 1] = pg.im;
        cx ur = cx_mk(c->unit_rho[2 * g], c->unit_rho[2 * g + 1]);
        cx zmag = cx_mul(cx_mul(cx_mul(clam, tk), ur), suffix);
        sl->dmag[slot] = zmag.re;
        cx zph = cx_mul(cx_mul(cx_mul(clam, tk), rho_of(c, g)), suffix);
        sl->dphase[slot] = -zph.im;

        cx gwc = cx_mul(cx_mul(clam, psi_of(c, g)), tk);
        double gw = gwc.re;
        const double *I = c->inv_covs + 9 * g;
        const double *mu = c->means + 3 * g;
        double i00 = I[0], i01 = I[1], i02 = I[2], i11 = I[4], i12 = I[5], i22 = I[8];
        double t_in = h->clamped[k] ? min_t : h->d1[k];
        double t_mid = 0.5 * (t_in + h->d2[k]);
        double ddx = rx[0] + t_mid * dx - mu[0];
        double ddy = rx[1] + t_mid * dy - mu[1];
        double ddz = rx[2] + t_mid * dz - mu[2];
        double q0 = i00 * ddx + i01 * ddy + i02 * ddz;
        double q1 = i01 * ddx + i11 * ddy + i12 * ddz;
        double q2 = i02 * ddx + i12 * ddy + i22 * ddz;
        double gmu[3] = {gw * w * q0, gw * w * q1, gw * w * q2};
        double f = gw * w * 0.5;
        double qv[3] = {q0, q1, q2};
        double Iv[9] = {i00, i01, i02, i01, i11, i12, i02, i12, i22};
        double cv9[9];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) cv9[3 * i + j] = f * (qv[i] * qv[j] - Iv[3 * i + j]);
        double mx = rx[0] - mu[0], my = rx[1] - mu[1], mz = rx[2] - mu[2];
        double p[3] = {i00 * dx + i01 * dy + i02 * dz, i01 * dx + i11 * dy + i12 * dz, i02 * dx + i12 * dy + i22 * dz};
        double e[3] = {i00 * mx + i01 * my + i02 * mz, i01 * mx + i11 * my + i12 * mz, i02 * mx + i12 * my + i22 * mz};
        double a = p[0] * dx + p[1] * dy + p[2] * dz;
        double b = p[0] * mx + p[1] * my + p[2] * mz;
        double cq = e[0] * mx + e[1] * my + e[2] * mz;
        double disc = b * b - a * (cq - 9.0);
        if (disc >= TANGENT_EPS) {
            double sq = sqrt(disc);
            double s_dv = q0 * dx + q1 * dy + q2 * dz;
            double dw_dt = gw * (-w) * s_dv;
            double half = 0.5 * dw_dt;
            double inv2sq = 0.5 / sq;
            int clamped = h->clamped[k];
            for (int ax = 0; ax < 3; ++ax) {
                double bmu = -p[ax], cmu = -2.0 * e[ax];
                double dd = (2.0 * b * bmu - a * cmu) * inv2sq;
                double dsum = (-bmu + dd) / a;
                if (!clamped) dsum += (-bmu - dd) / a;
                gmu[ax] += half * dsum;
            }
            double cm9 = cq - 9.0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    double da = -p[i] * p[j];
                    double db = -p[i] * e[j];
                    double dc = -e[i] * e[j];
                    double ddisc = 2.0 * b * db - cm9 * da - a * dc;
                    double dsum = (-db + ddisc * inv2sq) / a - h->d2[k] * da / a;
                    if (!clamped) dsum += (-db - ddisc * inv2sq) / a - h->d1[k] * da / a;
                    cv9[3 * i + j] += half * dsum;
                }
        }
        for (int a3 = 0; a3 < 3; ++a3) sl->dmu[3 * slot + a3] = gmu[a3];
        for (int a9 = 0; a9 < 9; ++a9) sl->dcov[9 * slot + a9] = cv9[a9];
        cx wpsi = cx_rmul(h->w[k], psi_of(c, g));
        suffix = cx_add(wpsi, cx_mul(rho_of(c, g), suffix));
    }
}

/* rotation_derivatives, grad.py:123-131. */
static void rot_derivs(const double q[4], double d[4][9]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    double t0[9] = {0, -z, y, z, 0, -x, -y, x, 0};
    double t1[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
    double t2[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
    double t3[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
    for (int i = 0; i < 9; ++i) { d[0][i] = 2.0 * t0[i]; d[1][i] = 2.0 * t1[i]; d[2][i] = 2.0 * t2[i]; d[3][i] = 2.0 * t3[i]; }
}

/* chain_cov_to_shape, grad.py:134-164 (one primitive). */
static void cov_to_shape(const double *quat, const double *log_scale, const double *dcov, double *dq, double *ds) {
    double nrm = sqrt(quat[0] * quat[0] + quat[1] * quat[1] + quat[2] * quat[2] + quat[3] * quat[3]);
    double qu[4] = {quat[0] / nrm, quat[1] / nrm, quat[2] / nrm, quat[3] / nrm};
    double R[9];
    quat_rot(qu, R);
    double dv[3];
    for (int a = 0; a < 3; ++a) dv[a] = exp(2.0 * log_scale[a]);
    for (int a = 0; a < 3; ++a) {
        double acc = 0.0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) acc += R[3 * i + a] * dcov[3 * i + j] * R[3 * j + a];
        ds[a] = 2.0 * dv[a] * acc;
    }
    double dr[4][9];
    rot_derivs(qu, dr);
    double g[4];
    for (int qi = 0; qi < 4; ++qi) {
        double acc = 0.0;
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k) {
                double s1 = 0.0, s2 = 0.0;
                for (int j = 0; j < 3; ++j) {
                    s1 += dr[qi][3 * i + j] * dv[j] * R[3 * k + j];
                    s2 += R[3 * i + j] * dv[j] * dr[qi][3 * k + j];
                }
                acc += dcov[3 * i + k] * (s1 + s2);
            }
        g[qi] = acc;
    }
    double gq = g[0] * qu[0] + g[1] * qu[1] + g[2] * qu[2] + g[3] * qu[3];
    for (int qi = 0; qi < 4; ++qi) dq[qi] = (g[qi] - gq * qu[qi]) / nrm;
}

/* backward_frame, grad.py:192-259: count -> offsets -> slots -> fixed-order
 * reduction -> d_coeffs -> direction chain -> chain_cov_to_shape. */
int orc_backward(orc_ctx *c, const double *upstream, int include_dir, double *d_mean, double *d_quat,
                 double *d_log_scale, double *d_trans_mag, double *d_trans_phase, double *d_coeffs,
                 double *d_cov, int threads) {
    set_threads(threads);
    int64_t R = c->n_az * c->n_el, n = c->n, K = c->n_coeffs;
    int64_t n_tiles = c->tiles_u * c->tiles_v;
    double n_az = (double)c->n_az;
    int64_t *counts = (int64_t *)calloc((size_t)R, sizeof(int64_t));
    int64_t *offsets = (int64_t *)calloc((size_t)R, sizeof(int64_t));
    /* count_hits_tiled, _kernels.py:250-292 */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < n_tiles; ++t) {
        int64_t lo = c->ranges[2 * t], hi = c->ranges[2 * t + 1];
        if (hi == lo) continue;
        int64_t tu0 = (t % c->tiles_u) * TILE, tv0 = (t / c->tiles_u) * TILE;
        int64_t u_end = tu0 + TILE < c->n_az ? tu0 + TILE : c->n_az;
        int64_t v_end = tv0 + TILE < c->n_el ? tv0 + TILE : c->n_el;
        tile_cand_t tc;
        gather_tile(c, lo, hi, &tc);
        hits_t h;
        hits_alloc(&h, tc.m);
        for (int64_t u = tu0; u < u_end; ++u)
            for (int64_t v = tv0; v < v_end; ++v) {
                int64_t r = u * c->n_el + v;
                int64_t cnt = collect_hits((double)u, (double)v, c->ray_dirs + 3 * r, &tc, c->rx, c->ress_radius, n_az, 1, &h);
                counts[r] = live_hits(c, cnt, &h);
            }
        hits_free(&h);
        free_tile(&tc);
    }
    int64_t total = 0;
    for (int64_t r = 0; r < R; ++r) { offsets[r] = total; total += counts[r]; }
    slots_t sl;
    int64_t tk = total > 0 ? total : 1;
    sl.g = (int64_t *)calloc((size_t)tk, sizeof(int64_t));
    sl.pg = (double *)calloc((size_t)(2 * tk), sizeof(double));
    sl.dmag = (double *)calloc((size_t)tk, sizeof(double));
    sl.dphase = (double *)calloc((size_t)tk, sizeof(double));
    sl.dmu = (double *)calloc((size_t)(3 * tk), sizeof(double));
    sl.dcov = (double *)calloc((size_t)(9 * tk), sizeof(double));
    /* backward_tiled, _kernels.py:295-357 */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < n_tiles; ++t) {
        int64_t lo = c->ranges[2 * t], hi = c->ranges[2 * t + 1];
        if (hi == lo) continue;
        int64_t tu0 = (t % c->tiles_u) * TILE, tv0 = (t / c->tiles_u) * TILE;
        int64_t u_end = tu0 + TILE < c->n_az ? tu0 + TILE : c->n_az;
        int64_t v_end = tv0 + TILE < c->n_el ? tv0 + TILE : c->n_el;
        tile_cand_t tc;
        gather_tile(c, lo, hi, &tc);
        hits_t h;
        hits_alloc(&h, tc.m);
        cx *trans = (cx *)malloc(sizeof(cx) * (tc.m > 0 ? tc.m : 1));
        for (int64_t u = tu0; u < u_end; ++u)
            for (int64_t v = tv0; v < v_end; ++v) {
                int64_t r = u * c->n_el + v;
                cx lam = cx_mk(upstream[2 * r], upstream[2 * r + 1]);
                int64_t cnt = collect_hits((double)u, (double)v, c->ray_dirs + 3 * r, &tc, c->rx, c->ress_radius, n_az, 1, &h);
                cx tr = cx_mk(1.0, 0.0);
                int64_t live = 0;
                for (int64_t k = 0; k < cnt; ++k) {
                    if (tr.re * tr.re + tr.im * tr.im < TERM_EPS2) break;
                    trans[k] = tr;
                    tr = cx_mul(tr, rho_of(c, h.g[k]));
                    ++live;
                }
                ray_backward(c, r, lam, live, &h, trans, offsets[r], &sl);
            }
        free(trans);
        hits_free(&h);
        free_tile(&tc);
    }
    /* bincount reductions in slot order, grad.py:243-255 */
    memset(d_mean, 0, sizeof(double) * 3 * n);
    memset(d_trans_mag, 0, sizeof(double) * n);
    memset(d_trans_phase, 0, sizeof(double) * n);
    memset(d_cov, 0, sizeof(double) * 9 * n);
    double *p_acc = (double *)calloc((size_t)(2 * (n > 0 ? n : 1)), sizeof(double));
    for (int64_t s = 0; s < total; ++s) {
        int64_t g = sl.g[s];
        d_trans_mag[g] += sl.dmag[s];
        d_trans_phase[g] += sl.dphase[s];
        for (int a = 0; a < 3; ++a) d_mean[3 * g + a] += sl.dmu[3 * s + a];
        for (int a = 0; a < 9; ++a) d_cov[9 * g + a] += sl.dcov[9 * s + a];
        p_acc[2 * g] += sl.pg[2 * s];
        p_acc[2 * g + 1] += sl.pg[2 * s + 1];
    }
    for (int64_t g = 0; g < n; ++g) {
        cx pc = cx_conj(cx_mk(p_acc[2 * g], p_acc[2 * g + 1]));
        for (int64_t k = 0; k < K; ++k) {
            cx bc = cx_conj(cx_mk(c->basis[2 * (K * g + k)], c->basis[2 * (K * g + k) + 1]));
            cx v = cx_mul(pc, bc);
            d_coeffs[2 * (K * g + k)] = v.re;
            d_coeffs[2 * (K * g + k) + 1] = v.im;
        }
    }
    /* _direction_chain, grad.py:167-189 */
    if (include_dir) {
        for (int64_t g = 0; g < n; ++g) {
            double r0 = c->tx[0] - c->means[3 * g], r1 = c->tx[1] - c->means[3 * g + 1], r2 = c->tx[2] - c->means[3 * g + 2];
            double zeta2 = r0 * r0 + r1 * r1 + r2 * r2;
            double rho2 = r0 * r0 + r1 * r1;
            int ok = c->bearing_valid[g] && (rho2 > 1e-18 * zeta2);
            if (!ok) continue;
            double rho = sqrt(rho2);
            cx dpa = cx_mk(0.0, 0.0), dpb = cx_mk(0.0, 0.0);
            for (int64_t k = 0; k < K; ++k) {
                cx co = cx_mk(c->coeffs[2 * (K * g + k)], c->coeffs[2 * (K * g + k) + 1]);
                dpa = cx_add(dpa, cx_mul(co, cx_mk(c->basis_dalpha[2 * (K * g + k)], c->basis_dalpha[2 * (K * g + k) + 1])));
                dpb = cx_add(dpb, cx_mul(co, cx_mk(c->basis_dbeta[2 * (K * g + k)], c->basis_dbeta[2 * (K * g + k) + 1])));
            }
            cx pa = cx_mk(p_acc[2 * g], p_acc[2 * g + 1]);
            double ga = cx_mul(pa, dpa).re, gb = cx_mul(pa, dpb).re;
            double da_dr[3] = {-r1 / rho2, r0 / rho2, 0.0};
            double db_dr[3] = {-r2 * r0 / (rho * zeta2), -r2 * r1 / (rho * zeta2), rho / zeta2};
            for (int a = 0; a < 3; ++a) d_mean[3 * g + a] += -(ga * da_dr[a] + gb * db_dr[a]);
        }
    }
    for (int64_t g = 0; g < n; ++g)
        cov_to_shape(c->quats + 4 * g, c->log_scales + 3 * g, d_cov + 9 * g, d_quat + 4 * g, d_log_scale + 3 * g);
    free(p_acc);
    free(sl.g); free(sl.pg); free(sl.dmag); free(sl.dphase); free(sl.dmu); free(sl.dcov);
    free(counts);
    free(offsets);
    return 0;
}

/* Live hit count per ray (count_hits_tiled) exposed for hit-list parity. */
int orc_live_counts(orc_ctx *c, int64_t *counts, int threads) {
    set_threads(threads);
    int64_t n_tiles = c->tiles_u * c->tiles_v;
    int64_t R = c->n_az * c->n_el;
    for (int64_t r = 0; r < R; ++r) counts[r] = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < n_tiles; ++t) {
        int64_t lo = c->ranges[2 * t], hi = c->ranges[2 * t + 1];
        if (hi == lo) continue;
        int64_t tu0 = (t % c->tiles_u) * TILE, tv0 = (t / c->tiles_u) * TILE;
        int64_t u_end = tu0 + TILE < c->n_az ? tu0 + TILE : c->n_az;
        int64_t v_end = tv0 + TILE < c->n_el ? tv0 + TILE : c->n_el;
        tile_cand_t tc;
        gather_tile(c, lo, hi, &tc);
        hits_t h;
        hits_alloc(&h, tc.m);
        for (int64_t u = tu0; u < u_end; ++u)
            for (int64_t v = tv0; v < v_end; ++v) {
                int64_t r = u * c->n_el + v;
                int64_t cnt = collect_hits((double)u, (double)v, c->ray_dirs + 3 * r, &tc, c->rx, c->ress_radius, (double)c->n_az, 1, &h);
                counts[r] = live_hits(c, cnt, &h);
            }
        hits_free(&h);
        free_tile(&tc);
    }
    return 0;
}

/* Sorted hit list of one ray (all hits, not only live), for tests and
 * diagnostics: returns the hit count, fills up to cap entries. */
int64_t orc_ray_hits(orc_ctx *c, int64_t r, int64_t cap, int64_t *g, double *tmid, double *w, double *d1,
                     double *d2, uint8_t *clamped) {
    int64_t u = r / c->n_el, v = r % c->n_el;
    int64_t t = (v / TILE) * c->tiles_u + (u / TILE);
    int64_t lo = c->ranges[2 * t], hi = c->ranges[2 * t + 1];
    if (hi == lo) return 0;
    tile_cand_t tc;
    gather_tile(c, lo, hi, &tc);
    hits_t h;
    hits_alloc(&h, tc.m);
    int64_t cnt = collect_hits((double)u, (double)v, c->ray_dirs + 3 * r, &tc, c->rx, c->ress_radius, (double)c->n_az, 1, &h);
    for (int64_t k = 0; k < cnt && k < cap; ++k) {
        g[k] = h.g[k]; tmid[k] = h.tmid[k]; w[k] = h.w[k]; d1[k] = h.d1[k]; d2[k] = h.d2[k]; clamped[k] = h.clamped[k];
    }
    hits_free(&h);
    free_tile(&tc);
    return cnt;
}

int orc_version(void) { return 1; }
