/*
 * sgwls_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, double-precision restatement of the reference SG-WLS filter path
 * (arXiv 1705.01674, /root/reference/proj).  It exists so the CUDA product
 * path can be checked against an independent CPU statement of the same
 * algorithm.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product library
 * (paper_1705_01674_b200/libsgwls_b200.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks this file against
 *   (1) the reference library itself compiled from /root/reference into
 *       oracle/_ref (bit-identical outputs expected: same operation order),
 *   (2) the golden fixtures in tests/golden/ produced by that library, and
 *   (3) the SPEC.md worked examples.
 *
 * Every function cites the reference file:line it restates.  Operation order
 * follows the reference exactly so that results are bit-identical to it.
 */
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sgwls_oracle.h"

/* proj/src/banded.cpp:10 */
#define PIVOT_FLOOR 1e-300
/* proj/src/smoother.cpp:15 */
#define MASK_FLOOR 1e-8

static void set_err(char* err, size_t errlen, const char* msg) {
    if (err && errlen) {
        strncpy(err, msg, errlen - 1);
        err[errlen - 1] = '\0';
    }
}

void oracle_config_default(oracle_config* c) {
    /* proj/include/sgwls/smoother.hpp:12-24, proj/include/sgwls/weights.hpp:14-27 */
    c->lambda = 900.0;
    c->r = 1;
    c->tau = 1;
    c->iterations = 4;
    c->first_axis = 0;
    c->threads = 1;
    c->kind = 0; /* Frac */
    c->alpha_s = 1.2;
    c->alpha_r = 1.2;
    c->sigma_s = 4.0;
    c->sigma_r = 3.0;
    c->epsilon = 1e-4;
    c->guidance_scale = 1.0;
}

/* proj/src/weights.cpp:7-12 then proj/src/smoother.cpp:103-111 (weights last) */
int oracle_validate(const oracle_config* c, char* err, size_t errlen) {
    char buf[160];
    if (!(c->lambda >= 0.0) || !isfinite(c->lambda)) {
        set_err(err, errlen, "smooth: lambda must be finite and >= 0");
        return 1;
    }
    if (c->r < 1) { set_err(err, errlen, "smooth: r must be >= 1"); return 1; }
    if (c->tau < 1 || c->tau > 2 * c->r + 1) {
        snprintf(buf, sizeof buf, "smooth: tau must be in [1, 2r+1], got %d", c->tau);
        set_err(err, errlen, buf);
        return 1;
    }
    if (c->iterations < 1) { set_err(err, errlen, "smooth: iterations must be >= 1"); return 1; }
    if (c->threads < 1) { set_err(err, errlen, "smooth: threads must be >= 1"); return 1; }
    if (!(c->epsilon > 0.0)) { set_err(err, errlen, "weights: epsilon must be > 0"); return 1; }
    if (c->kind == 1 && (!(c->sigma_s > 0.0) || !(c->sigma_r > 0.0))) {
        set_err(err, errlen, "weights: sigma_s and sigma_r must be > 0 for exponential weights");
        return 1;
    }
    if (!(c->guidance_scale > 0.0)) { set_err(err, errlen, "weights: guidance_scale must be > 0"); return 1; }
    return 0;
}

/* proj/src/snake.cpp:7-19 */
int oracle_band_centers(int extent, int r, int tau, int* out, int cap) {
    if (extent < 1 || r < 0 || tau < 1) return -1;
    if (extent < 2 * r + 1) {
        if (cap >= 1) out[0] = (extent - 1) / 2;
        return 1;
    }
    int n = 0;
    const int last = extent - 1 - r;
    int c;
    for (c = r; c <= last; c += tau) {
        if (n < cap) out[n] = c;
        n++;
    }
    if (out[n - 1] != last) {
        if (n < cap) out[n] = last;
        n++;
    }
    return n;
}

/* proj/src/snake.cpp:21-49: serpentine coordinates of one band */
typedef struct { int row, col; } coord_t;

static int band_layout(int height, int width, int center, int r, int axis, coord_t* coords) {
    const int extent = axis == 0 ? width : height;
    const int lo = center - r > 0 ? center - r : 0;
    const int hi = center + r < extent - 1 ? center + r : extent - 1;
    const int sweep = axis == 0 ? height : width;
    int n = 0;
    for (int i = 0; i < sweep; ++i) {
        const int reversed = (i % 2) != 0;
        for (int j = 0; j <= hi - lo; ++j) {
            const int k = reversed ? hi - j : lo + j;
            if (axis == 0) { coords[n].row = i; coords[n].col = k; }
            else { coords[n].row = k; coords[n].col = i; }
            n++;
        }
    }
    return n;
}

typedef struct {
    int width, height, channels;
    const double* data;
} cimg_t;

static inline double img_at(const cimg_t* im, int y, int x, int c) {
    return im->data[((size_t)y * im->width + x) * im->channels + c];
}

/* proj/src/weights.cpp:29-76 -> w[k*r + t-1] */
static void edge_weights(const cimg_t* g, const coord_t* coords, int n, int r, const oracle_config* p,
                         double* w, double* lut) {
    const int lutn = 2 * (2 * r + 1) * (2 * r + 1) + 1;
    for (int i = 0; i < lutn; ++i) lut[i] = -1.0;
    memset(w, 0, sizeof(double) * (size_t)n * r);
    for (int k = 0; k < n; ++k) {
        const int row_k = coords[k].row, col_k = coords[k].col;
        const int tmax = r < n - 1 - k ? r : n - 1 - k;
        for (int t = 1; t <= tmax; ++t) {
            const int row_j = coords[k + t].row, col_j = coords[k + t].col;
            const int dr = row_k - row_j, dc = col_k - col_j;
            const int d2 = dr * dr + dc * dc;
            double range2 = 0.0;
            for (int c = 0; c < g->channels; ++c) {
                const double dg = img_at(g, row_k, col_k, c) - img_at(g, row_j, col_j, c);
                range2 += dg * dg;
            }
            const double range_diff = sqrt(range2) * p->guidance_scale;
            double weight;
            if (p->kind == 1) {
                double* s = &lut[d2];
                if (*s < 0.0) *s = exp(-d2 / (2.0 * p->sigma_s * p->sigma_s));
                weight = *s * exp(-(range_diff * range_diff) / (2.0 * p->sigma_r * p->sigma_r));
            } else {
                double* s = &lut[d2];
                if (*s < 0.0) *s = 1.0 / (pow(sqrt((double)d2), p->alpha_s) + p->epsilon);
                weight = *s / (pow(range_diff, p->alpha_r) + p->epsilon);
            }
            w[(size_t)k * r + t - 1] = weight;
        }
    }
}

/* WeightTable::between, proj/include/sgwls/weights.hpp:42-45 */
static inline double w_between(const double* w, int n, int r, int k, int t) {
    return (k >= 0 && t >= 1 && t <= r && k + t < n) ? w[(size_t)k * r + t - 1] : 0.0;
}

/* proj/src/banded.cpp:13-42.  upper == lower for this assembly, so one array. */
static int assemble(int n, const double* w, int wr, double lambda, int r, double* diag, double* off) {
    const int rb = r < n - 1 ? r : n - 1;
    memset(off, 0, sizeof(double) * (size_t)n * (rb > 0 ? rb : 1));
    for (int k = 0; k < n; ++k) {
        double incident = 0.0;
        for (int t = 1; t <= rb && k + t < n; ++t) {
            const double wt = w_between(w, n, wr, k, t);
            incident += wt;
            off[(size_t)k * rb + t - 1] = -lambda * wt;
        }
        for (int t = 1; t <= rb && k - t >= 0; ++t) incident += w_between(w, n, wr, k - t, t);
        diag[k] = 1.0 + lambda * incident;
    }
    return rb;
}

static inline double off_at(const double* off, int n, int r, int k, int t) {
    return (t >= 1 && t <= r && k >= 0 && k + t < n) ? off[(size_t)k * r + t - 1] : 0.0;
}

/* proj/src/banded.cpp:44-87.  Returns -1 on success, else the failing row. */
static int factorize(int n, int r, const double* diag, const double* off, double* alpha, double* gamma,
                     double* beta) {
    const int rr = r > 0 ? r : 1;
    memset(gamma, 0, sizeof(double) * (size_t)n * rr);
    memset(beta, 0, sizeof(double) * (size_t)n * rr);
#define G(k, t) gamma[(size_t)(k) * r + (t) - 1]
#define B(k, t) beta[(size_t)(k) * r + (t) - 1]
    for (int k = 0; k < n; ++k) {
        double acc = 0.0;
        const int tm = k < r ? k : r;
        for (int t = 1; t <= tm; ++t) acc += G(k - t, t) * B(k - t, t);
        const double pivot = diag[k] - acc;
        if (!(pivot > PIVOT_FLOOR)) return k;
        alpha[k] = pivot;
        const int imax = (r - 1) < (n - 1 - k) ? (r - 1) : (n - 1 - k);
        for (int i = 1; i <= imax; ++i) {
            double gacc = 0.0, bacc = 0.0;
            const int tm2 = k < r - i ? k : r - i;
            for (int t = 1; t <= tm2; ++t) {
                gacc += G(k - t, i + t) * B(k - t, t);
                bacc += G(k - t, t) * B(k - t, i + t);
            }
            G(k, i) = off_at(off, n, r, k, i) - gacc;
            B(k, i) = (off_at(off, n, r, k, i) - bacc) / pivot;
        }
        if (r >= 1 && k + r < n) {
            G(k, r) = off_at(off, n, r, k, r);
            B(k, r) = off_at(off, n, r, k, r) / pivot;
        }
    }
#undef G
#undef B
    return -1;
}

/* proj/src/banded.cpp:89-102 then 104-118 */
static void substitute(int n, int r, const double* alpha, const double* gamma, const double* beta,
                       const double* rhs, double* y, double* u) {
    for (int k = 0; k < n; ++k) {
        double acc = 0.0;
        const int tm = k < r ? k : r;
        for (int t = 1; t <= tm; ++t) acc += gamma[(size_t)(k - t) * r + t - 1] * y[k - t];
        y[k] = (rhs[k] - acc) / alpha[k];
    }
    for (int k = n - 1; k >= 0; --k) {
        double acc = 0.0;
        const int tmax = r < n - 1 - k ? r : n - 1 - k;
        for (int t = 1; t <= tmax; ++t) acc += beta[(size_t)k * r + t - 1] * u[k + t];
        u[k] = y[k] - acc;
    }
}

/* ------------------------------------------------------------------ passes */

typedef struct {
    const cimg_t* src;
    const cimg_t* guid;
    const oracle_config* cfg;
    int axis;
    const int* centers;
    int ncenters;
    double** solved;    /* per band: channel-major solved[c*s + p] */
    coord_t** coords;   /* per band */
    int* sizes;
    int next;           /* work counter (guarded by mu) */
    int fail_band;      /* first failing band (smallest index) */
    int fail_row;
    pthread_mutex_t mu;
} pass_ctx;

/* Body of the run_workers lambda, proj/src/smoother.cpp:57-76 */
static int solve_band(pass_ctx* pc, int ci) {
    const cimg_t* src = pc->src;
    const int r = pc->cfg->r;
    const int extent = pc->axis == 0 ? src->width : src->height;
    const int center = pc->centers[ci];
    const int lo = center - r > 0 ? center - r : 0;
    const int hi = center + r < extent - 1 ? center + r : extent - 1;
    const int sweep = pc->axis == 0 ? src->height : src->width;
    const int s = (hi - lo + 1) * sweep;
    coord_t* coords = (coord_t*)malloc(sizeof(coord_t) * s);
    band_layout(src->height, src->width, center, r, pc->axis, coords);
    double* w = (double*)malloc(sizeof(double) * (size_t)s * r);
    double* lut = (double*)malloc(sizeof(double) * (2 * (2 * r + 1) * (2 * r + 1) + 1));
    edge_weights(pc->guid, coords, s, r, pc->cfg, w, lut);
    double* rhs = (double*)malloc(sizeof(double) * s);
    for (int p = 0; p < s; ++p) rhs[p] = img_at(src, coords[p].row, coords[p].col, 0);
    double* diag = (double*)malloc(sizeof(double) * s);
    double* off = (double*)malloc(sizeof(double) * (size_t)s * r);
    const int rb = assemble(s, w, r, pc->cfg->lambda, r, diag, off);
    const int rr = rb > 0 ? rb : 1;
    double* alpha = (double*)malloc(sizeof(double) * s);
    double* gamma = (double*)malloc(sizeof(double) * (size_t)s * rr);
    double* beta = (double*)malloc(sizeof(double) * (size_t)s * rr);
    const int bad = factorize(s, rb, diag, off, alpha, gamma, beta);
    double* solved = NULL;
    if (bad < 0) {
        const int ch = src->channels;
        solved = (double*)malloc(sizeof(double) * (size_t)ch * s);
        double* y = (double*)malloc(sizeof(double) * s);
        for (int c = 0; c < ch; ++c) {
            if (c > 0)
                for (int p = 0; p < s; ++p) rhs[p] = img_at(src, coords[p].row, coords[p].col, c);
            substitute(s, rb, alpha, gamma, beta, rhs, y, solved + (size_t)c * s);
        }
        free(y);
    }
    free(w); free(lut); free(rhs); free(diag); free(off); free(alpha); free(gamma); free(beta);
    pc->solved[ci] = solved;
    pc->coords[ci] = coords;
    pc->sizes[ci] = s;
    return bad;
}

static void* pass_worker(void* arg) {
    pass_ctx* pc = (pass_ctx*)arg;
    for (;;) {
        pthread_mutex_lock(&pc->mu);
        const int ci = pc->next++;
        pthread_mutex_unlock(&pc->mu);
        if (ci >= pc->ncenters) return NULL;
        const int bad = solve_band(pc, ci);
        if (bad >= 0) {
            pthread_mutex_lock(&pc->mu);
            if (pc->fail_band < 0 || ci < pc->fail_band) { pc->fail_band = ci; pc->fail_row = bad; }
            pthread_mutex_unlock(&pc->mu);
        }
    }
}

/* proj/src/smoother.cpp:51-99 */
static int run_pass(const cimg_t* src, const cimg_t* guid, const oracle_config* cfg, int axis, double* out,
                    char* err, size_t errlen) {
    const int extent = axis == 0 ? src->width : src->height;
    const int cap = extent + 2;
    int* centers = (int*)malloc(sizeof(int) * cap);
    const int nc = oracle_band_centers(extent, cfg->r, cfg->tau, centers, cap);
    pass_ctx pc;
    memset(&pc, 0, sizeof pc);
    pc.src = src; pc.guid = guid; pc.cfg = cfg; pc.axis = axis;
    pc.centers = centers; pc.ncenters = nc;
    pc.solved = (double**)calloc(nc, sizeof(double*));
    pc.coords = (coord_t**)calloc(nc, sizeof(coord_t*));
    pc.sizes = (int*)calloc(nc, sizeof(int));
    pc.fail_band = -1;
    pthread_mutex_init(&pc.mu, NULL);
    int nthreads = cfg->threads < nc ? cfg->threads : nc;
    if (nthreads <= 1) {
        pass_worker(&pc);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
        for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, pass_worker, &pc);
        for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
        free(th);
    }
    int rc = 0;
    if (pc.fail_band >= 0) {
        char buf[160];
        snprintf(buf, sizeof buf, "rband_lu_factorize: non-positive pivot at row %d (input not SPD)", pc.fail_row);
        set_err(err, errlen, buf);
        rc = 1;
    } else {
        /* Merge in center order, proj/src/smoother.cpp:78-88 + proj/src/snake.cpp:60-72 */
        const int ch = src->channels;
        const size_t npx = (size_t)src->width * src->height;
        double* accum = (double*)calloc(npx * ch, sizeof(double));
        double* counts = (double*)calloc(npx, sizeof(double));
        for (int ci = 0; ci < nc; ++ci) {
            const int s = pc.sizes[ci];
            for (int c = 0; c < ch; ++c) {
                const double* sol = pc.solved[ci] + (size_t)c * s;
                for (int i = 0; i < s; ++i) {
                    const size_t px = (size_t)pc.coords[ci][i].row * src->width + pc.coords[ci][i].col;
                    accum[px * ch + c] += sol[i];
                    if (c == 0) counts[px] += 1.0;
                }
            }
        }
        /* proj/src/smoother.cpp:90-97 */
        for (size_t px = 0; px < npx && rc == 0; ++px) {
            const double count = counts[px];
            if (count <= 0.0) {
                set_err(err, errlen, "smooth: pixel missed by every band (internal)");
                rc = 1;
                break;
            }
            for (int c = 0; c < ch; ++c) out[px * ch + c] = accum[px * ch + c] / count;
        }
        free(accum);
        free(counts);
    }
    for (int ci = 0; ci < nc; ++ci) { free(pc.solved[ci]); free(pc.coords[ci]); }
    free(pc.solved); free(pc.coords); free(pc.sizes); free(centers);
    pthread_mutex_destroy(&pc.mu);
    return rc;
}

/* proj/src/smoother.cpp:113-125 */
int oracle_smooth_f64(const double* target, int width, int height, int channels, const double* guidance,
                      int guidance_channels, const oracle_config* cfg, double* out, char* err, size_t errlen) {
    if (oracle_validate(cfg, err, errlen)) return 1;
    if (width <= 0 || height <= 0 || channels <= 0) { set_err(err, errlen, "smooth: empty target"); return 1; }
    (void)guidance_channels;
    const size_t n = (size_t)width * height * channels;
    double* cur = (double*)malloc(sizeof(double) * n);
    double* nxt = (double*)malloc(sizeof(double) * n);
    memcpy(cur, target, sizeof(double) * n);
    cimg_t g = {width, height, guidance_channels, guidance};
    int axis = cfg->first_axis;
    int rc = 0;
    for (int pass = 0; pass < cfg->iterations; ++pass) {
        cimg_t src = {width, height, channels, cur};
        rc = run_pass(&src, &g, cfg, axis, nxt, err, errlen);
        if (rc) break;
        double* t = cur; cur = nxt; nxt = t;
        axis = 1 - axis;
    }
    if (!rc) memcpy(out, cur, sizeof(double) * n);
    free(cur);
    free(nxt);
    return rc;
}

int oracle_smooth_f32(const float* target, int width, int height, int channels, const float* guidance,
                      int guidance_channels, const oracle_config* cfg, double* out, char* err, size_t errlen) {
    const size_t nt = (size_t)width * height * channels, ng = (size_t)width * height * guidance_channels;
    double* t = (double*)malloc(sizeof(double) * (nt ? nt : 1));
    double* g = (double*)malloc(sizeof(double) * (ng ? ng : 1));
    for (size_t i = 0; i < nt; ++i) t[i] = target[i];
    for (size_t i = 0; i < ng; ++i) g[i] = guidance[i];
    const int rc = oracle_smooth_f64(t, width, height, channels, g, guidance_channels, cfg, out, err, errlen);
    free(t);
    free(g);
    return rc;
}

/* proj/src/smoother.cpp:127-163 */
int oracle_interpolate_sparse_f32(const float* values, int width, int height, int channels, const float* mask,
                                  const float* guidance, int guidance_channels, const oracle_config* cfg,
                                  double* out, double* undefined_mask, char* err, size_t errlen) {
    const size_t npx = (size_t)width * height;
    int any = 0;
    for (size_t px = 0; px < npx; ++px) {
        const double m = mask[px];
        if (m != 0.0 && m != 1.0) { set_err(err, errlen, "interpolate_sparse: mask must be 0/1"); return 1; }
        if (m == 1.0) any = 1;
        if (m == 0.0)
            for (int c = 0; c < channels; ++c)
                if (values[px * channels + c] != 0.0) {
                    set_err(err, errlen, "interpolate_sparse: values nonzero outside mask");
                    return 1;
                }
    }
    if (!any) { set_err(err, errlen, "interpolate_sparse: empty mask"); return 1; }
    double* num = (double*)malloc(sizeof(double) * npx * channels);
    double* den = (double*)malloc(sizeof(double) * npx);
    int rc = oracle_smooth_f32(values, width, height, channels, guidance, guidance_channels, cfg, num, err, errlen);
    if (!rc) rc = oracle_smooth_f32(mask, width, height, 1, guidance, guidance_channels, cfg, den, err, errlen);
    if (!rc) {
        for (size_t px = 0; px < npx; ++px) {
            const double d = den[px];
            if (d < MASK_FLOOR) {
                for (int c = 0; c < channels; ++c) out[px * channels + c] = 0.0;
                if (undefined_mask) undefined_mask[px] = 1.0;
            } else {
                for (int c = 0; c < channels; ++c) out[px * channels + c] = num[px * channels + c] / d;
                if (undefined_mask) undefined_mask[px] = 0.0;
            }
        }
    }
    free(num);
    free(den);
    return rc;
}

/* ---------------------------------------------- 1-D kernels for unit checks */

/* Factor + solve one assembled band from raw weights: proj/src/banded.cpp:13-123 */
int oracle_solve_band(int n, int r, const double* w, double lambda, const double* rhs, double* u, double* alpha_out,
                      double* beta_out, double* gamma_out) {
    double* diag = (double*)malloc(sizeof(double) * n);
    double* off = (double*)malloc(sizeof(double) * (size_t)n * r);
    const int rb = assemble(n, w, r, lambda, r, diag, off);
    const int rr = rb > 0 ? rb : 1;
    double* alpha = (double*)malloc(sizeof(double) * n);
    double* gamma = (double*)malloc(sizeof(double) * (size_t)n * rr);
    double* beta = (double*)malloc(sizeof(double) * (size_t)n * rr);
    double* y = (double*)malloc(sizeof(double) * n);
    const int bad = factorize(n, rb, diag, off, alpha, gamma, beta);
    if (bad < 0) {
        substitute(n, rb, alpha, gamma, beta, rhs, y, u);
        if (alpha_out) memcpy(alpha_out, alpha, sizeof(double) * n);
        if (beta_out) memcpy(beta_out, beta, sizeof(double) * (size_t)n * rr);
        if (gamma_out) memcpy(gamma_out, gamma, sizeof(double) * (size_t)n * rr);
    }
    free(diag); free(off); free(alpha); free(gamma); free(beta); free(y);
    return bad;
}

/* Factor + solve an explicit symmetric banded system (diag, off[k*r+t-1]) */
int oracle_solve_system(int n, int r, const double* diag, const double* off, const double* rhs, double* u,
                        double* alpha_out, double* beta_out, double* gamma_out) {
    const int rr = r > 0 ? r : 1;
    double* alpha = (double*)malloc(sizeof(double) * n);
    double* gamma = (double*)malloc(sizeof(double) * (size_t)n * rr);
    double* beta = (double*)malloc(sizeof(double) * (size_t)n * rr);
    double* y = (double*)malloc(sizeof(double) * n);
    const int bad = factorize(n, r, diag, off, alpha, gamma, beta);
    if (bad < 0) {
        substitute(n, r, alpha, gamma, beta, rhs, y, u);
        if (alpha_out) memcpy(alpha_out, alpha, sizeof(double) * n);
        if (beta_out) memcpy(beta_out, beta, sizeof(double) * (size_t)n * rr);
        if (gamma_out) memcpy(gamma_out, gamma, sizeof(double) * (size_t)n * rr);
    }
    free(alpha); free(gamma); free(beta); free(y);
    return bad;
}

/* Serpentine coordinates of one band, proj/src/snake.cpp:21-49 */
int oracle_band_layout(int height, int width, int center, int r, int axis, int* rows, int* cols) {
    const int extent = axis == 0 ? width : height;
    const int lo = center - r > 0 ? center - r : 0;
    const int hi = center + r < extent - 1 ? center + r : extent - 1;
    const int sweep = axis == 0 ? height : width;
    coord_t* c = (coord_t*)malloc(sizeof(coord_t) * (size_t)(hi - lo + 1) * sweep);
    const int n = band_layout(height, width, center, r, axis, c);
    for (int i = 0; i < n; ++i) { rows[i] = c[i].row; cols[i] = c[i].col; }
    free(c);
    return n;
}

/* Edge weights of one band, proj/src/weights.cpp:29-76 */
int oracle_edge_weights(const double* guidance, int width, int height, int gch, int center, int r, int axis,
                        const oracle_config* cfg, double* w) {
    const int extent = axis == 0 ? width : height;
    const int lo = center - r > 0 ? center - r : 0;
    const int hi = center + r < extent - 1 ? center + r : extent - 1;
    const int sweep = axis == 0 ? height : width;
    const int s = (hi - lo + 1) * sweep;
    coord_t* c = (coord_t*)malloc(sizeof(coord_t) * s);
    band_layout(height, width, center, r, axis, c);
    double* lut = (double*)malloc(sizeof(double) * (2 * (2 * r + 1) * (2 * r + 1) + 1));
    cimg_t g = {width, height, gch, guidance};
    edge_weights(&g, c, s, r, cfg, w, lut);
    free(c);
    free(lut);
    return s;
}
