/*
 * edgealign_oracle.c -- TEST INFRASTRUCTURE: plain-C restatement of the
 * reference search path, used only as the parity checker (see
 * edgealign_oracle.h for who may call it and how it is pinned).
 *
 * Every function names the reference code it restates as path:line under
 * /root/reference/proj.  Floating-point expressions keep the reference's
 * operation order; the file is compiled with -ffp-contract=off exactly like
 * the reference (proj/CMakeLists.txt:12-14), so no mul+add is fused.
 */
#define _GNU_SOURCE
#include "edgealign_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static const double kPi = 3.14159265358979323846; /* pose.h:21 */

/* ---- errors (errors.h:14-75) ------------------------------------------- */
static __thread char g_err[512];
static __thread double g_err_value;

const char* orc_last_error(void) { return g_err; }
double orc_last_error_value(void) { return g_err_value; }

static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
#include <stdarg.h>
static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}
static int ok(void) {
    g_err[0] = 0;
    return EA_OK;
}

/* ---- pose geometry  pose.h:45-92 ---------------------------------------- */
static uint64_t axis_count(double lo, double hi, double step) { /* pose.h:45-49 */
    return (uint64_t)floor((hi - lo) / step + 1e-9) + 1;
}

int orc_grid_counts(const ea_pose_grid* g, ea_grid_counts* out) { /* pose.h:52-67 */
    if (!(isfinite(g->x0) && isfinite(g->x1) && isfinite(g->dx) && isfinite(g->y0) &&
          isfinite(g->y1) && isfinite(g->dy) && isfinite(g->t0) && isfinite(g->t1) &&
          isfinite(g->dt))) {
        return fail(EA_ERR_INVALID_ARGUMENT, "pose grid has non-finite bounds");
    }
    if (g->dx <= 0.0 || g->dy <= 0.0 || g->dt <= 0.0) {
        return fail(EA_ERR_INVALID_ARGUMENT, "pose grid steps must be positive");
    }
    if (g->x0 > g->x1 || g->y0 > g->y1 || g->t0 > g->t1) {
        return fail(EA_ERR_INVALID_ARGUMENT, "pose grid range start exceeds end");
    }
    out->nx = axis_count(g->x0, g->x1, g->dx);
    out->ny = axis_count(g->y0, g->y1, g->dy);
    out->nt = axis_count(g->t0, g->t1, g->dt);
    return ok();
}

int orc_pose_at(const ea_pose_grid* g, uint64_t index, ea_pose* out) { /* pose.h:77-92 */
    ea_grid_counts c;
    int st = orc_grid_counts(g, &c);
    if (st) return st;
    const uint64_t total = c.nx * c.ny * c.nt;
    if (index >= total) {
        return fail(EA_ERR_BOUNDS, "pose index %llu out of range (grid size %llu)",
                    (unsigned long long)index, (unsigned long long)total);
    }
    const uint64_t plane = c.nx * c.ny;
    const uint64_t it = index / plane;
    const uint64_t rem = index % plane;
    const uint64_t iy = rem / c.nx;
    const uint64_t ix = rem % c.nx;
    out->ux = g->x0 + (double)ix * g->dx;
    out->uy = g->y0 + (double)iy * g->dy;
    out->theta = g->t0 + (double)it * g->dt;
    return ok();
}

/* ---- row kernels  kernels_scalar.cpp:14-56 ------------------------------ */
static void sobel_row(const double* above, const double* mid, const double* below,
                      int width, double* gx, double* gy, double* mag) {
    for (int x = 1; x + 1 < width; ++x) {
        const double a = above[x - 1], b = above[x], c = above[x + 1];
        const double d = mid[x - 1], f = mid[x + 1];
        const double g = below[x - 1], h = below[x], i = below[x + 1];
        const double ew = f - d;
        const double ns = h - b;
        const double sx = ((c - a) + (ew + ew)) + (i - g);
        const double sy = ((g - a) + (ns + ns)) + (i - c);
        gx[x] = sx;
        gy[x] = sy;
        mag[x] = sqrt(sx * sx + sy * sy);
    }
}

static void downsample_row(const double* top, const double* bot, int out_width,
                           double* out) {
    for (int i = 0; i < out_width; ++i) {
        const double t = top[2 * i] + top[2 * i + 1];
        const double u = bot[2 * i] + bot[2 * i + 1];
        out[i] = (t + u) * 0.25;
    }
}

static double vote_span(const double* gx, const double* gy, const double* mag, int x0,
                        int x1, double dx, double dy, double eps_mag, int absolute) {
    double best = -INFINITY;
    for (int x = x0; x <= x1; ++x) {
        double cand = 0.0;
        if (mag[x] >= eps_mag) {
            cand = (dx * gx[x] + dy * gy[x]) / mag[x];
        }
        if (absolute) {
            cand = fabs(cand);
        }
        if (cand > best) {
            best = cand;
        }
    }
    return best;
}

/* ---- image  image.cpp:248-291, gradient.cpp:12-27 ------------------------ */
int orc_downsample(const double* img, int w, int h, double* out) { /* image.cpp:248-261 */
    if (w < 2 || h < 2) {
        return fail(EA_ERR_SIZE, "downsample needs at least 2x2, got %dx%d", w, h);
    }
    const int ow = w / 2, oh = h / 2;
    for (int y = 0; y < oh; ++y) {
        downsample_row(img + (size_t)(2 * y) * w, img + (size_t)(2 * y + 1) * w, ow,
                       out + (size_t)y * ow);
    }
    return ok();
}

int orc_max_pyramid_levels(int w, int h) { /* image.cpp:263-272 */
    int levels = 1;
    while (w / 2 >= 8 && h / 2 >= 8) {
        w /= 2;
        h /= 2;
        ++levels;
    }
    return levels;
}

int orc_build_pyramid(const double* img, int w, int h, int levels, double* out) {
    /* image.cpp:274-291 */
    if (levels < 1) return fail(EA_ERR_INVALID_ARGUMENT, "num_levels must be >= 1");
    const int feasible = orc_max_pyramid_levels(w, h);
    if (levels > feasible) {
        return fail(EA_ERR_SIZE,
                    "pyramid of %d levels would drop below 8x8; maximum feasible level "
                    "count is %d",
                    levels, feasible);
    }
    memcpy(out, img, sizeof(double) * (size_t)w * h);
    const double* prev = out;
    double* cur = out + (size_t)w * h;
    for (int k = 1; k < levels; ++k) {
        int st = orc_downsample(prev, w, h, cur);
        if (st) return st;
        w /= 2;
        h /= 2;
        prev = cur;
        cur += (size_t)w * h;
    }
    return ok();
}

int orc_compute_gradients(const double* img, int w, int h, double* gx, double* gy,
                          double* mag) { /* gradient.cpp:12-27 */
    if (w < 3 || h < 3) {
        return fail(EA_ERR_SIZE, "compute_gradients needs at least 3x3, got %dx%d", w, h);
    }
    const size_t n = (size_t)w * h;
    memset(gx, 0, sizeof(double) * n);
    memset(gy, 0, sizeof(double) * n);
    memset(mag, 0, sizeof(double) * n);
    for (int y = 1; y + 1 < h; ++y) {
        const size_t row = (size_t)y * w;
        sobel_row(img + row - w, img + row, img + row + w, w, gx + row, gy + row, mag + row);
    }
    return ok();
}

/* ---- edge model  edge_model.cpp:17-149 ----------------------------------- */
int orc_default_thresholds(const double* mag, int w, int h, ea_edge_thresholds* out) {
    /* edge_model.cpp:17-24 */
    double max_mag = 0.0;
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        max_mag = mag[i] > max_mag ? mag[i] : max_mag; /* std::max(max_mag, m) */
    }
    const double high = 0.3 * max_mag;
    out->low = 0.5 * high;
    out->high = high;
    return ok();
}

static int orientation_bin(double gx, double gy) { /* edge_model.cpp:34-45 */
    double a = atan2(gy, gx);
    if (a < 0.0) a += kPi;
    const double kStep = kPi / 8.0;
    if (a <= kStep) return 0;
    if (a <= 3.0 * kStep) return 1;
    if (a <= 5.0 * kStep) return 2;
    if (a <= 7.0 * kStep) return 3;
    return 0;
}

int orc_extract_edge_model(const double* gx, const double* gy, const double* mag, int w,
                           int h, const ea_edge_thresholds* th, int level,
                           ea_edge_point* pts, int cap, int* n_out, double* cx_out,
                           double* cy_out) { /* edge_model.cpp:53-149 */
    static const int kOffX[4] = {1, 1, 0, -1}; /* edge_model.cpp:48-49 */
    static const int kOffY[4] = {0, 1, 1, 1};
    (void)level;
    if (th->low < 0.0 || th->low > th->high) {
        return fail(EA_ERR_INVALID_ARGUMENT, "edge thresholds need 0 <= low <= high");
    }
    const size_t n = (size_t)w * h;
    double max_mag = 0.0;
    for (size_t i = 0; i < n; ++i) max_mag = mag[i] > max_mag ? mag[i] : max_mag;

    unsigned char* state = calloc(n ? n : 1, 1);
    unsigned char* kept = calloc(n ? n : 1, 1);
    size_t* stack = malloc(sizeof(size_t) * (n ? n : 1));
    if (!state || !kept || !stack) {
        free(state); free(kept); free(stack);
        return fail(EA_ERR_INTERNAL, "out of memory");
    }
    /* NMS, edge_model.cpp:66-85 */
    for (int y = 1; y + 1 < h; ++y) {
        for (int x = 1; x + 1 < w; ++x) {
            const size_t i = (size_t)y * w + x;
            const double m = mag[i];
            if (m <= 0.0 || m < th->low) continue;
            const int bin = orientation_bin(gx[i], gy[i]);
            const double fwd = mag[(size_t)(y + kOffY[bin]) * w + (x + kOffX[bin])];
            const double bwd = mag[(size_t)(y - kOffY[bin]) * w + (x - kOffX[bin])];
            if (m > fwd && m >= bwd) state[i] = (m >= th->high) ? 2 : 1;
        }
    }
    /* hysteresis, edge_model.cpp:87-114 */
    for (size_t i = 0; i < n; ++i) {
        if (state[i] == 2 && !kept[i]) {
            size_t sp = 0;
            kept[i] = 1;
            stack[sp++] = i;
            while (sp) {
                const size_t p = stack[--sp];
                const int px = (int)(p % (size_t)w), py = (int)(p / (size_t)w);
                for (int ddy = -1; ddy <= 1; ++ddy) {
                    for (int ddx = -1; ddx <= 1; ++ddx) {
                        if (ddx == 0 && ddy == 0) continue;
                        const int qx = px + ddx, qy = py + ddy;
                        if (qx < 0 || qx >= w || qy < 0 || qy >= h) continue;
                        const size_t q = (size_t)qy * w + qx;
                        if (!kept[q] && state[q] != 0) {
                            kept[q] = 1;
                            stack[sp++] = q;
                        }
                    }
                }
            }
        }
    }
    /* emit row-major + centroid, edge_model.cpp:116-148 */
    size_t count = 0;
    double sum_x = 0.0, sum_y = 0.0;
    for (size_t i = 0; i < n; ++i) {
        if (kept[i]) {
            ++count;
            sum_x += (double)(i % (size_t)w);
            sum_y += (double)(i / (size_t)w);
        }
    }
    if (count == 0) {
        free(state); free(kept); free(stack);
        g_err_value = max_mag;
        return fail(EA_ERR_EMPTY_MODEL,
                    "edge extraction produced an empty model (max gradient magnitude %f)",
                    max_mag);
    }
    const double cnt = (double)count;
    const double cx = sum_x / cnt, cy = sum_y / cnt;
    int j = 0;
    for (size_t i = 0; i < n; ++i) {
        if (!kept[i]) continue;
        if (j < cap) {
            const double x = (double)(i % (size_t)w), y = (double)(i / (size_t)w);
            const double m = mag[i];
            pts[j].x_rel = x - cx;
            pts[j].y_rel = y - cy;
            pts[j].dx = gx[i] / m;
            pts[j].dy = gy[i] / m;
            pts[j].mag = m;
        }
        ++j;
    }
    *n_out = (int)count;
    *cx_out = cx;
    *cy_out = cy;
    free(state); free(kept); free(stack);
    return ok();
}

/* ---- similarity  similarity.cpp:15-126 ----------------------------------- */
static int validate(const ea_score_params* p) { /* similarity.cpp:15-23 */
    if (p->neighborhood < 1 || p->neighborhood % 2 == 0) {
        return fail(EA_ERR_INVALID_ARGUMENT, "neighborhood must be odd and >= 1, got %d",
                    p->neighborhood);
    }
    if (!(p->eps_mag > 0.0)) return fail(EA_ERR_INVALID_ARGUMENT, "eps_mag must be positive");
    return EA_OK;
}

typedef struct {
    const double *gx, *gy, *mag;
    int w, h;
} field_t;

static double vote_at(double dir_x, double dir_y, const field_t* f, int cx, int cy,
                      int radius, double eps, int absolute) { /* similarity.cpp:30-52 */
    const int x0 = cx - radius < 0 ? 0 : cx - radius;
    const int x1 = cx + radius >= f->w ? f->w - 1 : cx + radius;
    const int y0 = cy - radius < 0 ? 0 : cy - radius;
    const int y1 = cy + radius >= f->h ? f->h - 1 : cy + radius;
    if (x0 > x1 || y0 > y1) return 0.0;
    double best = -INFINITY;
    for (int y = y0; y <= y1; ++y) {
        const size_t row = (size_t)y * f->w;
        const double m =
            vote_span(f->gx + row, f->gy + row, f->mag + row, x0, x1, dir_x, dir_y, eps, absolute);
        if (m > best) best = m;
    }
    return best;
}

static int round_half_up(double v) { return (int)floor(v + 0.5); } /* similarity.cpp:54-56 */

int orc_point_vote(double dir_x, double dir_y, const double* gx, const double* gy,
                   const double* mag, int w, int h, int cx, int cy,
                   const ea_score_params* p, double* out) { /* similarity.cpp:58-64 */
    int st = validate(p);
    if (st) return st;
    field_t f = {gx, gy, mag, w, h};
    *out = vote_at(dir_x, dir_y, &f, cx, cy, (p->neighborhood - 1) / 2, p->eps_mag,
                   p->polarity == EA_POLARITY_IGNORE);
    return ok();
}

int orc_rotate_model(const ea_edge_point* pts, int n, double theta, double* px,
                     double* py, double* dx, double* dy) { /* similarity.cpp:68-88 */
    const double c = cos(theta);
    const double s = sin(theta);
    for (int i = 0; i < n; ++i) {
        const ea_edge_point* p = &pts[i];
        px[i] = c * p->x_rel - s * p->y_rel;
        py[i] = s * p->x_rel + c * p->y_rel;
        const double rx = c * p->dx - s * p->dy;
        const double ry = s * p->dx + c * p->dy;
        const double norm = sqrt(rx * rx + ry * ry);
        dx[i] = rx / norm;
        dy[i] = ry / norm;
    }
    return ok();
}

typedef struct {
    double *px, *py, *dx, *dy;
    int n;
} rotated_t;

static double score_rotated(const rotated_t* r, double ux, double uy, const field_t* f,
                            const ea_score_params* p, int* n_in) { /* similarity.cpp:90-119 */
    const double kCoordGuard = 1e9; /* similarity.cpp:28 */
    const int radius = (p->neighborhood - 1) / 2;
    const int absolute = p->polarity == EA_POLARITY_IGNORE;
    double sum = 0.0;
    int inbounds = 0;
    for (int i = 0; i < r->n; ++i) {
        const double px = r->px[i] + ux;
        const double py = r->py[i] + uy;
        double vote = 0.0;
        if (px > -kCoordGuard && px < kCoordGuard && py > -kCoordGuard && py < kCoordGuard) {
            const int cx = round_half_up(px);
            const int cy = round_half_up(py);
            if (cx >= 0 && cx < f->w && cy >= 0 && cy < f->h) {
                ++inbounds;
                vote = vote_at(r->dx[i], r->dy[i], f, cx, cy, radius, p->eps_mag, absolute);
            }
        }
        sum += vote;
    }
    if (n_in) *n_in = inbounds;
    return sum / (double)r->n;
}

static int rotated_alloc(rotated_t* r, int n) {
    r->n = n;
    r->px = malloc(sizeof(double) * (size_t)(n ? n : 1) * 4);
    if (!r->px) return fail(EA_ERR_INTERNAL, "out of memory");
    r->py = r->px + n;
    r->dx = r->py + n;
    r->dy = r->dx + n;
    return EA_OK;
}

int orc_pose_score(const ea_edge_point* pts, int n, const ea_pose* pose, const double* gx,
                   const double* gy, const double* mag, int w, int h,
                   const ea_score_params* p, double* value, int* n_in) {
    /* similarity.cpp:121-126 */
    int st = validate(p);
    if (st) return st;
    if (n == 0) return fail(EA_ERR_INVALID_ARGUMENT, "pose_score needs a nonempty model");
    rotated_t r;
    if ((st = rotated_alloc(&r, n))) return st;
    orc_rotate_model(pts, n, pose->theta, r.px, r.py, r.dx, r.dy);
    field_t f = {gx, gy, mag, w, h};
    *value = score_rotated(&r, pose->ux, pose->uy, &f, p, n_in);
    free(r.px);
    return ok();
}

/* ---- search  search.cpp:26-202 ------------------------------------------ */
typedef struct {
    double score;
    uint64_t index;
} cand_t;

static int better(const cand_t* a, const cand_t* b) { /* search.cpp:36-41 */
    if (a->score != b->score) return a->score > b->score;
    return a->index < b->index;
}

typedef struct { /* TopK  search.cpp:44-67 */
    cand_t* items;
    int size, k;
} topk_t;

static void topk_offer(topk_t* t, double score, uint64_t index) {
    const cand_t c = {score, index};
    if (t->size == t->k && !better(&c, &t->items[t->size - 1])) return;
    /* upper_bound under `better`: first position whose item c is better than */
    int at = 0;
    while (at < t->size && !better(&c, &t->items[at])) ++at;
    const int last = t->size < t->k ? t->size : t->k - 1;
    memmove(&t->items[at + 1], &t->items[at], sizeof(cand_t) * (size_t)(last - at));
    t->items[at] = c;
    if (t->size < t->k) ++t->size;
}

typedef struct {
    const ea_edge_point* pts;
    int n;
    const field_t* f;
    const ea_pose_grid* g;
    ea_grid_counts counts;
    const ea_score_params* p;
    uint64_t lo, hi;
    topk_t top;
    int status;
} scan_job;

static void* scan_range(void* arg) { /* search.cpp:72-93 */
    scan_job* j = arg;
    const uint64_t plane = j->counts.nx * j->counts.ny;
    uint64_t cached_it = (uint64_t)-1;
    rotated_t r;
    if (rotated_alloc(&r, j->n)) {
        j->status = EA_ERR_INTERNAL;
        return NULL;
    }
    for (uint64_t idx = j->lo; idx < j->hi; ++idx) {
        const uint64_t it = idx / plane;
        if (it != cached_it) {
            orc_rotate_model(j->pts, j->n, j->g->t0 + (double)it * j->g->dt, r.px, r.py, r.dx,
                             r.dy);
            cached_it = it;
        }
        const uint64_t rem = idx % plane;
        const uint64_t iy = rem / j->counts.nx;
        const uint64_t ix = rem % j->counts.nx;
        const double ux = j->g->x0 + (double)ix * j->g->dx;
        const double uy = j->g->y0 + (double)iy * j->g->dy;
        topk_offer(&j->top, score_rotated(&r, ux, uy, j->f, j->p, NULL), idx);
    }
    free(r.px);
    j->status = EA_OK;
    return NULL;
}

static int cmp_better(const void* a, const void* b) {
    const cand_t *x = a, *y = b;
    if (better(x, y)) return -1;
    if (better(y, x)) return 1;
    return 0;
}

static int n_cpus(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

/* run_search (search.cpp:95-140) restricted to theta indices [it_begin, it_end). */
static int run_search(const ea_edge_point* pts, int n, const field_t* f,
                      const ea_pose_grid* g, const ea_score_params* p, int k,
                      uint64_t it_begin, uint64_t it_end, int threads, cand_t* out,
                      int* n_out) {
    int st = validate(p);
    if (st) return st;
    if (n == 0) return fail(EA_ERR_INVALID_ARGUMENT, "search needs a nonempty model");
    if (k < 1) return fail(EA_ERR_INVALID_ARGUMENT, "topk must be >= 1");
    ea_grid_counts c;
    if ((st = orc_grid_counts(g, &c))) return st;
    const uint64_t plane = c.nx * c.ny;
    if (it_end == 0 || it_end > c.nt) it_end = c.nt;
    const uint64_t lo = it_begin * plane, hi = it_end * plane;
    const uint64_t total = hi > lo ? hi - lo : 0;
    uint64_t workers = threads > 0 ? (uint64_t)threads : (uint64_t)n_cpus();
    if (workers > total) workers = total ? total : 1;

    scan_job* jobs = calloc(workers, sizeof(scan_job));
    cand_t* buf = calloc(workers * (size_t)k, sizeof(cand_t));
    pthread_t* tids = calloc(workers, sizeof(pthread_t));
    for (uint64_t w = 0; w < workers; ++w) {
        scan_job* j = &jobs[w];
        j->pts = pts; j->n = n; j->f = f; j->g = g; j->counts = c; j->p = p;
        j->lo = lo + total * w / workers;
        j->hi = lo + total * (w + 1) / workers;
        j->top.items = buf + w * (size_t)k;
        j->top.k = k;
        if (workers > 1) pthread_create(&tids[w], NULL, scan_range, j);
        else scan_range(j);
    }
    if (workers > 1)
        for (uint64_t w = 0; w < workers; ++w) pthread_join(tids[w], NULL);
    /* merge: concat, sort by `better`, truncate (search.cpp:130-139) */
    size_t m = 0;
    cand_t* merged = calloc(workers * (size_t)k + 1, sizeof(cand_t));
    for (uint64_t w = 0; w < workers; ++w) {
        memcpy(merged + m, jobs[w].top.items, sizeof(cand_t) * (size_t)jobs[w].top.size);
        m += (size_t)jobs[w].top.size;
    }
    qsort(merged, m, sizeof(cand_t), cmp_better); /* total order: indices distinct */
    if (m > (size_t)k) m = (size_t)k;
    memcpy(out, merged, sizeof(cand_t) * m);
    *n_out = (int)m;
    free(merged); free(jobs); free(buf); free(tids);
    return EA_OK;
}

int orc_search_topk(const ea_edge_point* pts, int n, const double* gx, const double* gy,
                    const double* mag, int w, int h, const ea_pose_grid* g,
                    const ea_score_params* p, int k, uint64_t it_begin, uint64_t it_end,
                    int threads, ea_scored_pose* out, int* n_out) {
    /* search_topk  search.cpp:155-167 */
    field_t f = {gx, gy, mag, w, h};
    cand_t* cands = calloc(k > 0 ? (size_t)k : 1, sizeof(cand_t));
    int m = 0;
    int st = run_search(pts, n, &f, g, p, k, it_begin, it_end, threads, cands, &m);
    if (st) {
        free(cands);
        return st;
    }
    for (int i = 0; i < m; ++i) {
        out[i].score = cands[i].score;
        out[i].grid_index = cands[i].index;
        orc_pose_at(g, cands[i].index, &out[i].pose);
    }
    *n_out = m;
    free(cands);
    return ok();
}

int orc_score_map(const ea_edge_point* pts, int n, const double* gx, const double* gy,
                  const double* mag, int w, int h, const ea_pose_grid* g,
                  const ea_score_params* p, uint64_t max_cells, double* out) {
    /* score_map  search.cpp:169-202 */
    int st = validate(p);
    if (st) return st;
    if (n == 0) return fail(EA_ERR_INVALID_ARGUMENT, "score_map needs a nonempty model");
    ea_grid_counts c;
    if ((st = orc_grid_counts(g, &c))) return st;
    const uint64_t total = c.nx * c.ny * c.nt;
    if (total > max_cells) {
        return fail(EA_ERR_BUDGET, "score_map needs %llu cells but the budget allows %llu",
                    (unsigned long long)total, (unsigned long long)max_cells);
    }
    field_t f = {gx, gy, mag, w, h};
    rotated_t r;
    if ((st = rotated_alloc(&r, n))) return st;
    const uint64_t plane = c.nx * c.ny;
    uint64_t cached_it = (uint64_t)-1;
    for (uint64_t idx = 0; idx < total; ++idx) {
        const uint64_t it = idx / plane;
        if (it != cached_it) {
            orc_rotate_model(pts, n, g->t0 + (double)it * g->dt, r.px, r.py, r.dx, r.dy);
            cached_it = it;
        }
        const uint64_t rem = idx % plane;
        const uint64_t iy = rem / c.nx;
        const uint64_t ix = rem % c.nx;
        out[idx] = score_rotated(&r, g->x0 + (double)ix * g->dx, g->y0 + (double)iy * g->dy,
                                 &f, p, NULL);
    }
    free(r.px);
    return ok();
}

/* ---- coarse to fine  search.cpp:240-357 ---------------------------------- */
typedef struct { /* BeamEntry  search.cpp:242-246 */
    ea_pose pose;
    double score;
    uint64_t top_index;
} beam_t;

static int same_pose(const ea_pose* a, const ea_pose* b) { /* search.cpp:248-250 */
    return a->ux == b->ux && a->uy == b->uy && a->theta == b->theta;
}

/* std::stable_sort by score descending (search.cpp:326-329): merge sort. */
static void stable_sort_desc(beam_t* a, beam_t* tmp, size_t n) {
    if (n < 2) return;
    const size_t mid = n / 2;
    stable_sort_desc(a, tmp, mid);
    stable_sort_desc(a + mid, tmp, n - mid);
    size_t i = 0, j = mid, k = 0;
    while (i < mid && j < n) {
        if (a[j].score > a[i].score) tmp[k++] = a[j++]; /* strictly better from right */
        else tmp[k++] = a[i++];
    }
    while (i < mid) tmp[k++] = a[i++];
    while (j < n) tmp[k++] = a[j++];
    memcpy(a, tmp, sizeof(beam_t) * n);
}

int orc_search_levels(int num_levels, const ea_edge_point* const* models,
                      const int* model_n, const double* const* gx, const double* const* gy,
                      const double* const* mag, const int* dims,
                      const ea_search_config* cfg, int threads, ea_outcome* out) {
    /* search_levels  search.cpp:254-357 */
    int st = validate(&cfg->score_params);
    if (st) return st;
    if (cfg->topk < 1 || cfg->refine_radius < 1) {
        return fail(EA_ERR_INVALID_ARGUMENT, "topk and refine_radius must be >= 1");
    }
    if (num_levels < cfg->num_levels) {
        return fail(EA_ERR_INVALID_ARGUMENT, "prepared levels do not cover num_levels");
    }
    const int top = cfg->num_levels - 1;
    const double scale = (double)(1 << top);
    ea_pose_grid tg = cfg->grid;
    tg.x0 /= scale; tg.x1 /= scale; tg.dx /= scale;
    tg.y0 /= scale; tg.y1 /= scale; tg.dy /= scale;

    memset(out, 0, sizeof(*out));
    const int k = cfg->topk;
    ea_scored_pose* seeds = calloc((size_t)k, sizeof(ea_scored_pose));
    int ns = 0;
    st = orc_search_topk(models[top], model_n[top], gx[top], gy[top], mag[top], dims[2 * top],
                         dims[2 * top + 1], &tg, &cfg->score_params, k, 0, 0, threads, seeds,
                         &ns);
    if (st) {
        free(seeds);
        return st;
    }
    const int R = cfg->refine_radius;
    const size_t side = (size_t)(2 * R + 1);
    beam_t* beam = calloc((size_t)k, sizeof(beam_t));
    size_t nb = (size_t)ns;
    for (int i = 0; i < ns; ++i) {
        beam[i].pose = seeds[i].pose;
        beam[i].score = seeds[i].score;
        beam[i].top_index = seeds[i].grid_index;
    }
    free(seeds);
    int nt = 0;
    out->trace[nt].level = top;
    out->trace[nt].pose = beam[0].pose;
    out->trace[nt].score = beam[0].score;
    ++nt;

    const double theta_floor = 0.25 * (kPi / 180.0); /* deg_to_rad(0.25), pose.h:23 */
    double step_x = tg.dx, step_y = tg.dy, step_t = tg.dt;
    beam_t* ev = calloc((size_t)k * side * side * side, sizeof(beam_t));
    beam_t* tmp = calloc((size_t)k * side * side * side, sizeof(beam_t));
    for (int level = top - 1; level >= 0; --level) {
        step_x /= 2.0;
        step_y /= 2.0;
        step_t = (step_t / 2.0 < theta_floor) ? theta_floor : step_t / 2.0; /* std::max */
        const int n = model_n[level];
        rotated_t r;
        if ((st = rotated_alloc(&r, n))) break;
        field_t f = {gx[level], gy[level], mag[level], dims[2 * level], dims[2 * level + 1]};
        size_t ne = 0;
        for (size_t pi = 0; pi < nb; ++pi) {
            const double cx = beam[pi].pose.ux * 2.0;
            const double cy = beam[pi].pose.uy * 2.0;
            const double ct = beam[pi].pose.theta;
            for (int kt = -R; kt <= R; ++kt) {
                const double theta = ct + (double)kt * step_t;
                orc_rotate_model(models[level], n, theta, r.px, r.py, r.dx, r.dy);
                for (int ky = -R; ky <= R; ++ky) {
                    for (int kx = -R; kx <= R; ++kx) {
                        beam_t e;
                        e.pose.ux = cx + (double)kx * step_x;
                        e.pose.uy = cy + (double)ky * step_y;
                        e.pose.theta = theta;
                        e.score = score_rotated(&r, e.pose.ux, e.pose.uy, &f,
                                                &cfg->score_params, NULL);
                        e.top_index = beam[pi].top_index;
                        ev[ne++] = e;
                    }
                }
            }
        }
        free(r.px);
        stable_sort_desc(ev, tmp, ne);
        size_t kept = 0;
        for (size_t i = 0; i < ne; ++i) {
            int dup = 0;
            for (size_t j = 0; j < kept; ++j) {
                if (same_pose(&beam[j].pose, &ev[i].pose)) {
                    dup = 1;
                    break;
                }
            }
            if (!dup) {
                beam[kept++] = ev[i];
                if (kept == (size_t)k) break;
            }
        }
        nb = kept;
        if (nt < EA_MAX_LEVELS) {
            out->trace[nt].level = level;
            out->trace[nt].pose = beam[0].pose;
            out->trace[nt].score = beam[0].score;
            ++nt;
        }
    }
    free(ev);
    free(tmp);
    if (st) {
        free(beam);
        return st;
    }
    out->n_trace = nt;
    out->pose = beam[0].pose;
    out->score = beam[0].score;
    out->grid_index = beam[0].top_index;
    out->found = beam[0].score >= cfg->min_score;
    free(beam);
    return ok();
}

/* ---- synthetic scenes  synth.cpp:20-300 ---------------------------------- */
static const double kGround = 200.0, kStroke = 40.0; /* synth.cpp:20-21 */

typedef struct { /* SplitMix64  synth.h:26-49 */
    uint64_t state;
    int have_spare;
    double spare;
} smx_t;

static uint64_t smx_next(smx_t* r) {
    uint64_t z = (r->state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static double smx_uniform01(smx_t* r) { return (double)(smx_next(r) >> 11) * 0x1.0p-53; }
static double smx_normal(smx_t* r) { /* synth.cpp:24-37 */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = 1.0 - smx_uniform01(r);
    const double u2 = smx_uniform01(r);
    const double rr = sqrt(-2.0 * log(u1));
    const double a = 2.0 * kPi * u2;
    r->spare = rr * sin(a);
    r->have_spare = 1;
    return rr * cos(a);
}

int orc_render_template(int id, int size, double* img) { /* synth.cpp:62-128 */
    if (size < 16) return fail(EA_ERR_SIZE, "template size must be >= 16, got %d", size);
    if (id < 0 || id > 3) return fail(EA_ERR_INVALID_ARGUMENT, "unknown template id");
    for (int i = 0; i < size * size; ++i) img[i] = kGround;
    const int margin = size / 8 > 2 ? size / 8 : 2;
    const int lo = margin, hi = size - 1 - margin;
#define STROKE(X, Y) (img[(size_t)(Y) * size + (X)] = kStroke)
    switch (id) {
        case EA_TEMPLATE_RECTANGLE:
            for (int x = lo; x <= hi; ++x)
                for (int t = 0; t < 2; ++t) {
                    STROKE(x, lo + t);
                    STROKE(x, hi - t);
                }
            for (int y = lo; y <= hi; ++y)
                for (int t = 0; t < 2; ++t) {
                    STROKE(lo + t, y);
                    STROKE(hi - t, y);
                }
            break;
        case EA_TEMPLATE_RING: {
            const double c = (size - 1) / 2.0;
            const double radius = (hi - lo) / 2.0;
            for (int y = 0; y < size; ++y)
                for (int x = 0; x < size; ++x) {
                    const double d = hypot(x - c, y - c);
                    if (fabs(d - radius) <= 1.0) STROKE(x, y);
                }
            break;
        }
        case EA_TEMPLATE_L_BRACKET:
            for (int y = lo; y <= hi; ++y) {
                STROKE(lo, y);
                STROKE(lo + 1, y);
            }
            for (int x = lo; x <= hi; ++x) {
                STROKE(x, hi);
                STROKE(x, hi - 1);
            }
            break;
        case EA_TEMPLATE_CROSS: {
            const int c = size / 2;
            for (int y = lo; y <= hi; ++y) {
                STROKE(c - 1, y);
                STROKE(c, y);
            }
            for (int x = lo; x <= hi; ++x) {
                STROKE(x, c - 1);
                STROKE(x, c);
            }
            break;
        }
    }
#undef STROKE
    return ok();
}

static void draw_clutter(double* canvas, int W, int H, int segments, uint64_t seed) {
    /* synth.cpp:140-165 */
    smx_t rng = {seed, 0, 0.0};
    for (int s = 0; s < segments; ++s) {
        const double x0 = smx_uniform01(&rng) * W;
        const double y0 = smx_uniform01(&rng) * H;
        const double x1 = smx_uniform01(&rng) * W;
        const double y1 = smx_uniform01(&rng) * H;
        const double value = smx_uniform01(&rng) * 255.0;
        const int width = 1 + (int)(smx_next(&rng) & 1ULL);
        const double len = hypot(x1 - x0, y1 - y0);
        const int steps = 1 + (int)(2.0 * len);
        for (int i = 0; i <= steps; ++i) {
            const double t = (double)i / steps;
            const int px = round_half_up(x0 + t * (x1 - x0));
            const int py = round_half_up(y0 + t * (y1 - y0));
            for (int dy = 0; dy < width; ++dy)
                for (int dx = 0; dx < width; ++dx) {
                    const int X = px + dx, Y = py + dy;
                    if (X >= 0 && X < W && Y >= 0 && Y < H) canvas[(size_t)Y * W + X] = value;
                }
        }
    }
}

/* template_edge_centroid + the occlusion model, synth.cpp:169-174,281-298 */
static int template_model(const double* tmpl, int size, ea_edge_point** pts, int* n,
                          double* cx, double* cy) {
    const size_t np = (size_t)size * size;
    double* g = malloc(sizeof(double) * np * 3);
    int st = orc_compute_gradients(tmpl, size, size, g, g + np, g + 2 * np);
    if (st) {
        free(g);
        return st;
    }
    ea_edge_thresholds th;
    orc_default_thresholds(g + 2 * np, size, size, &th);
    *pts = malloc(sizeof(ea_edge_point) * np);
    st = orc_extract_edge_model(g, g + np, g + 2 * np, size, size, &th, 0, *pts, (int)np, n,
                                cx, cy);
    free(g);
    return st;
}

int orc_compose_scene(const ea_scene_spec* s, double* canvas, double* tmpl,
                      ea_pose* truth_pose, double* occluded_fraction) {
    /* compose_scene  synth.cpp:178-300 */
    if (s->canvas_width < 16 || s->canvas_height < 16)
        return fail(EA_ERR_INVALID_ARGUMENT, "canvas must be at least 16x16");
    if (!(s->gain > 0.0) || !(s->gamma > 0.0))
        return fail(EA_ERR_INVALID_ARGUMENT, "illumination gain and gamma must be positive");
    if (s->noise_sigma < 0.0) return fail(EA_ERR_INVALID_ARGUMENT, "noise_sigma must be >= 0");
    const int W = s->canvas_width, H = s->canvas_height, T = s->template_size;
    int st = orc_render_template(s->template_id, T, tmpl);
    if (st) return st;
    ea_edge_point* pts = NULL;
    int np = 0;
    double cref_x, cref_y;
    if ((st = template_model(tmpl, T, &pts, &np, &cref_x, &cref_y))) {
        free(pts);
        return st;
    }
    const ea_pose pose = s->true_pose;
    const double c = cos(pose.theta), sn = sin(pose.theta);
    /* bbox of the transformed template, transform_point pose.h:96-102 */
    double min_x = 1e300, max_x = -1e300, min_y = 1e300, max_y = -1e300;
    const double corners[4][2] = {{0.0, 0.0}, {(double)(T - 1), 0.0}, {0.0, (double)(T - 1)},
                                  {(double)(T - 1), (double)(T - 1)}};
    for (int i = 0; i < 4; ++i) {
        const double tx = corners[i][0] - cref_x, ty = corners[i][1] - cref_y;
        const double px = (c * tx - sn * ty) + pose.ux;
        const double py = (sn * tx + c * ty) + pose.uy;
        min_x = px < min_x ? px : min_x;
        max_x = px > max_x ? px : max_x;
        min_y = py < min_y ? py : min_y;
        max_y = py > max_y ? py : max_y;
    }
    if (min_x < 0.0 || min_y < 0.0 || max_x > W - 1.0 || max_y > H - 1.0) {
        free(pts);
        return fail(EA_ERR_GEOMETRY,
                    "transformed template leaves the canvas (bbox [%f, %f] .. [%f, %f])", min_x,
                    min_y, max_x, max_y);
    }
    for (size_t i = 0; i < (size_t)W * H; ++i) canvas[i] = kGround;
    draw_clutter(canvas, W, H, s->clutter_segments, s->clutter_seed);
    /* inverse-map stamp, synth.cpp:224-244 */
    const int bx0 = (int)floor(min_x) - 1 > 0 ? (int)floor(min_x) - 1 : 0;
    const int by0 = (int)floor(min_y) - 1 > 0 ? (int)floor(min_y) - 1 : 0;
    const int bx1 = (int)ceil(max_x) + 1 < W - 1 ? (int)ceil(max_x) + 1 : W - 1;
    const int by1 = (int)ceil(max_y) + 1 < H - 1 ? (int)ceil(max_y) + 1 : H - 1;
    for (int y = by0; y <= by1; ++y) {
        for (int x = bx0; x <= bx1; ++x) {
            const double rx = x - pose.ux;
            const double ry = y - pose.uy;
            const double tx = (c * rx + sn * ry) + cref_x;
            const double ty = (-sn * rx + c * ry) + cref_y;
            const int ix = (int)ceil(tx - 0.5);
            const int iy = (int)ceil(ty - 0.5);
            if (ix >= 0 && ix < T && iy >= 0 && iy < T && tmpl[(size_t)iy * T + ix] != kGround)
                canvas[(size_t)y * W + x] = tmpl[(size_t)iy * T + ix];
        }
    }
    if (s->has_occluder) { /* synth.cpp:246-257 */
        const int ox0 = s->occ_x > 0 ? s->occ_x : 0;
        const int oy0 = s->occ_y > 0 ? s->occ_y : 0;
        const int ox1 = W - 1 < s->occ_x + s->occ_w - 1 ? W - 1 : s->occ_x + s->occ_w - 1;
        const int oy1 = H - 1 < s->occ_y + s->occ_h - 1 ? H - 1 : s->occ_y + s->occ_h - 1;
        for (int y = oy0; y <= oy1; ++y)
            for (int x = ox0; x <= ox1; ++x) canvas[(size_t)y * W + x] = s->occ_fill;
    }
    /* illumination, synth.cpp:262-269 */
    for (size_t i = 0; i < (size_t)W * H; ++i) {
        const double v = canvas[i];
        const double base = (s->gamma == 1.0) ? v : 255.0 * pow(v / 255.0, s->gamma);
        canvas[i] = s->gain * base + s->bias;
    }
    if (s->noise_sigma > 0.0) { /* synth.cpp:271-276 */
        smx_t rng = {s->noise_seed, 0, 0.0};
        for (size_t i = 0; i < (size_t)W * H; ++i) canvas[i] += s->noise_sigma * smx_normal(&rng);
    }
    *truth_pose = pose;
    *occluded_fraction = 0.0;
    if (s->has_occluder) { /* synth.cpp:281-298 */
        int covered = 0;
        for (int i = 0; i < np; ++i) {
            const double px = (c * pts[i].x_rel - sn * pts[i].y_rel) + pose.ux;
            const double py = (sn * pts[i].x_rel + c * pts[i].y_rel) + pose.uy;
            const int ix = round_half_up(px), iy = round_half_up(py);
            if (ix >= s->occ_x && ix < s->occ_x + s->occ_w && iy >= s->occ_y &&
                iy < s->occ_y + s->occ_h)
                ++covered;
        }
        *occluded_fraction = (double)covered / (double)np;
    }
    free(pts);
    return ok();
}
