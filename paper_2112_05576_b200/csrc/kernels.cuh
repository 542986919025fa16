// kernels.cuh -- launcher declarations and the exact fp64 scoring primitives
// shared by the device kernels.
#pragma once

#include <cuda_fp16.h>
#include <math.h>

#include "common.cuh"

namespace eab {

constexpr int kHistBins = 4096;           // screening-score histogram, [-1,1] in 2^-11 bins
constexpr double kCoordGuard = 1e9;       // similarity.cpp:28

// Geometry of the padded, row-skewed screening plane.
// Field pixel (x, y) lives at padded (xp, yp) = (x + 1 + PL, y + 1): a one-
// pixel zero ring plus PL / PR extra zero columns, so that the lattice
// kernel's windows never need column clamping.
struct PlaneGeom {
    int W = 0, H = 0;   // unpadded field dims
    int PL = 0, PR = 0; // extra zero columns left / right of the ring
    int PW = 0;         // row pitch in float2 (= W + 2 + PL + PR)
    int shift = 4;      // row skew: element (xp, yp) at yp*PW + (yp >> shift) + xp
    int zero = 0;       // offset of a PW + banks zero strip standing in for off-plane rows
    int elem_bytes = 8; // 8: float2 (nx, ny); 4: __half2 (nx, ny)
    size_t elems = 0;   // element count incl. the strip (whole 16 B chunks)
    size_t bytes() const { return elems * (size_t)elem_bytes; }
    int banks() const { return 128 / elem_bytes; }  // elements per 128 B wavefront
};

inline PlaneGeom plane_geom(int W, int H, int shift, int PL = 0, int PR = 0, int elem_bytes = 8) {
    PlaneGeom g;
    g.W = W;
    g.H = H;
    g.PL = PL;
    g.elem_bytes = elem_bytes;
    // pitch: 2^shift * PW must be a multiple of the wavefront's element count
    // so that lanes' slots are yg + 8*xg exactly
    const int mult = g.banks() >> shift > 1 ? g.banks() >> shift : 1;
    g.PW = W + 2 + PL + PR;
    g.PW = (g.PW + mult - 1) / mult * mult;
    g.PR = g.PW - (W + 2 + PL);
    g.shift = shift;
    const size_t B = (size_t)g.banks();
    size_t e = (size_t)(H + 2) * g.PW + (size_t)((H + 1) >> shift) + 1;
    e = (e + B - 1) / B * B;
    g.zero = (int)e;
    e += (size_t)g.PW + B;
    const size_t per16 = 16 / (size_t)elem_bytes;
    g.elems = (e + per16 - 1) / per16 * per16;
    return g;
}

// Control block shared by the top-level search kernels (one per context).
struct SearchCtrl {
    unsigned long long work_counter;  // dynamic work distribution of the screen kernel
    unsigned long long cand_count;    // poses admitted by the band threshold
    unsigned long long needed;        // histogram upper bound of cand_count
    unsigned finish_ticket;           // CTAs of the fused finish done with the rescore phase
    int flags;                        // rounding-ambiguous (theta, point) pairs
    float thr;                        // band threshold on the fp32 screen score
    int n_out;                        // entries written to the top-k output
    unsigned gfloor;                  // top-list mode: max over warps of their k-th largest
                                      // listed lane maximum (order key; 0 = none), <= M_k
};

// Monotone unsigned image of a float (0 below every float): atomicMax-able.
__device__ __forceinline__ unsigned float_order_key(float v) {
    const unsigned b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float float_from_order_key(unsigned k) {
    return k == 0u ? -INFINITY : __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// ---- exact fp64 primitives (reference op order) ------------------------------

// a1/m1 > a2/m2 for m1, m2 > 0, decided exactly from the products a1*m2 and
// a2*m1 as (rounded, fma error) pairs: rounding is monotone, so the rounded
// parts order the exact products except when they tie, where the error terms
// decide.  (A false answer on an exact tie of the quotients is harmless: equal
// quotients round to the same vote.)
__device__ __forceinline__ bool frac_greater(double a1, double m1, double a2, double m2) {
    const double h1 = __dmul_rn(a1, m2), h2 = __dmul_rn(a2, m1);
    if (h1 != h2) return h1 > h2;
    return __fma_rn(a1, m2, -h1) > __fma_rn(a2, m1, -h2);
}

// vote_at + vote_span  similarity.cpp:30-52, kernels_scalar.cpp:39-56.
// The window max of the rounded quotients (dx*gx + dy*gy) / mag equals the
// rounded quotient of the exact argmax (correct rounding is monotone), so the
// window is scanned with exact fraction comparisons (first maximum kept, as
// the reference's strict `>`) and only the winner is divided: one DDIV per
// vote instead of one per pixel.
__device__ __forceinline__ double vote_exact(const double* __restrict__ gx,
                                             const double* __restrict__ gy,
                                             const double* __restrict__ mag, int W, int H,
                                             int cx, int cy, int R, double dx, double dy,
                                             double eps, bool absolute) {
    double ba = 0.0, bm = 1.0;  // best candidate as a fraction
    bool have = false;
    if (R == 1 && cx >= 1 && cx + 1 < W && cy >= 1 && cy + 1 < H) {
        // interior 3x3 window: issue all 27 loads before any compare, so the
        // vote costs one memory latency instead of nine
        double m[9], gxv[9], gyv[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            const size_t o = (size_t)(cy - 1 + q / 3) * W + (cx - 1 + q % 3);
            m[q] = __ldg(mag + o);
            gxv[q] = __ldg(gx + o);
            gyv[q] = __ldg(gy + o);
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) {  // row-major: the reference's scan order
            double a = 0.0, d = 1.0;
            if (m[q] >= eps) {
                a = __dadd_rn(__dmul_rn(dx, gxv[q]), __dmul_rn(dy, gyv[q]));
                d = m[q];
            }
            if (absolute) a = fabs(a);
            if (!have || frac_greater(a, d, ba, bm)) {
                ba = a;
                bm = d;
                have = true;
            }
        }
        return bm == 1.0 ? ba : __ddiv_rn(ba, bm);
    }
    const int x0 = cx - R < 0 ? 0 : cx - R;
    const int x1 = cx + R >= W ? W - 1 : cx + R;
    const int y0 = cy - R < 0 ? 0 : cy - R;
    const int y1 = cy + R >= H ? H - 1 : cy + R;
    if (x0 > x1 || y0 > y1) return 0.0;
    for (int y = y0; y <= y1; ++y) {
        const size_t row = (size_t)y * W;
        for (int x = x0; x <= x1; ++x) {
            const double m = __ldg(mag + row + x);
            double a = 0.0, d = 1.0;  // below eps: candidate 0 (= 0 / 1)
            if (m >= eps) {
                a = __dadd_rn(__dmul_rn(dx, __ldg(gx + row + x)), __dmul_rn(dy, __ldg(gy + row + x)));
                d = m;
            }
            if (absolute) a = fabs(a);
            if (!have || frac_greater(a, d, ba, bm)) {
                ba = a;
                bm = d;
                have = true;
            }
        }
    }
    return bm == 1.0 ? ba : __ddiv_rn(ba, bm);
}

// One model point of score_rotated (similarity.cpp:102-116): projection,
// guard, half-up rounding, bounds test, window vote.  Returns the vote and
// sets *inb when the rounded centre is inside the field.
__device__ __forceinline__ double point_term_exact(double rpx, double rpy, double rdx,
                                                   double rdy, double ux, double uy,
                                                   const double* gx, const double* gy,
                                                   const double* mag, int W, int H, int R,
                                                   double eps, bool absolute, int* inb) {
    const double px = __dadd_rn(rpx, ux);
    const double py = __dadd_rn(rpy, uy);
    *inb = 0;
    if (px > -kCoordGuard && px < kCoordGuard && py > -kCoordGuard && py < kCoordGuard) {
        const int cx = (int)floor(__dadd_rn(px, 0.5));
        const int cy = (int)floor(__dadd_rn(py, 0.5));
        if (cx >= 0 && cx < W && cy >= 0 && cy < H) {
            *inb = 1;
            return vote_exact(gx, gy, mag, W, H, cx, cy, R, rdx, rdy, eps, absolute);
        }
    }
    return 0.0;
}

// Monotone integer image of a double under fp64 comparison (-0 == +0; the
// scores compared are never NaN): ranks and maxima run on the integer pipe,
// which on B200 is far wider than the fp64 compare path.
__device__ __forceinline__ long long order_key(double v) {
    const long long b = __double_as_longlong(v == 0.0 ? 0.0 : v);
    return b < 0 ? (b ^ 0x7FFFFFFFFFFFFFFFLL) : b;
}
__device__ __forceinline__ double from_order_key(long long k) {
    return __longlong_as_double(k < 0 ? (k ^ 0x7FFFFFFFFFFFFFFFLL) : k);
}

// pose_at arithmetic (pose.h:84-91): base + (double)i * step, no contraction.
__device__ __forceinline__ double lattice(double base, unsigned long long i, double step) {
    return __dadd_rn(base, __dmul_rn((double)i, step));
}

// ---- launchers ---------------------------------------------------------------
void launch_downsample(ea_ctx* ctx, const double* in, int w, int h, double* out);
// Pyramid levels 1..L-1 and the gradient fields of levels 0..L-1 of one
// image in one launch (pyramid_fields_kernel); false = not launched (too many
// levels for the shared-memory tiles, or EAB_NO_FUSED_PYRAMID): use
// launch_downsample + launch_sobel.
constexpr int kMaxFusedLevels = 6;
struct PyramidFieldsArgs {
    const double* img0;
    int levels, tile;
    int w[kMaxFusedLevels], h[kMaxFusedLevels];
    double* img[kMaxFusedLevels];  // level images (index 0 unused)
    double* gx[kMaxFusedLevels];
    double* gy[kMaxFusedLevels];
    double* mag[kMaxFusedLevels];
};
bool launch_pyramid_fields(ea_ctx* ctx, const PyramidFieldsArgs& a);
void launch_sobel(ea_ctx* ctx, const double* img, int w, int h, double* gx, double* gy,
                  double* mag);
// Screening plane (float2 g/|g|, zero ring/columns/strip) + clears
// clear[0 .. clear_words) and clear2[0 .. clear2_words) (the search's
// histogram and control block).
void launch_plane(ea_ctx* ctx, const ea_field* f, double eps, const PlaneGeom& g,
                  void* plane, unsigned* clear, int clear_words, unsigned* clear2,
                  int clear2_words);

// rotate_model for many thetas: rot_exact = px|py|dx|dy (each nth*n doubles),
// rot_screen = {ox, oy, dxf, dyf} per (theta, point) for the lattice kernel.
// amb (with rot_screen): [nth] rounding-ambiguous points per theta, then the
// count and the list of thetas that have any (AmbList); flags: their total.
void launch_rotate(ea_ctx* ctx, const double* pts_soa, int n, const double* cs, int nth,
                   double* rot_exact, int4* rot_screen, int* flags, int* amb = nullptr);
// Lattice point schedule per theta: points sorted by (oy, ox) and combined
// into entries -- mode 0: same-row neighbour pairs; mode 1: twins (same
// direction, offsets (1,0) / (0,1); R <= 1) -- see search_kernels.cu.
// sched: nth x sched_stride(n) int4.  twinned (mode 1, optional): += points
// in twin entries.
__host__ __device__ inline size_t sched_stride(size_t n) { return 1 + 2 * n; }
void launch_schedule(ea_ctx* ctx, const int4* rot_screen, int n, int nth, int4* sched, int mode,
                     unsigned long long* twinned);

struct ScreenArgs {
    const void* plane;        // float2 or __half2 elements (geom.elem_bytes)
    PlaneGeom geom;
    const int4* rot_screen;     // [theta - it_begin][point]
    const int4* sched;          // lattice point schedule per theta (schedule_kernel)
    const double* rot_exact;    // px | py | dx | dy, rows theta - it_begin
    size_t rot_stride;          // it_count * n (offset of py inside rot_exact)
    int n;                      // model points
    unsigned long long it_begin, it_count;
    unsigned long long nx, ny;
    // integer lattice (fast path)
    int ix0, iy0;
    // general grid
    double x0, dx, y0, dy;
    int R;
    int ignore;
    int xg;           // lattice warp tile: xg * 8 columns x (32 / xg) * 8 rows
    int sched_mode;   // schedule entry kinds: 0 singles/pairs, 1 singles/twins (launch_schedule)
    int strip;        // lattice kernels' lane-strip rows S (8, or 4 for twin schedules)
    // Integer steps sx, sy >= 1 (the paper's 3 px grid): the lattice kernels
    // tile the UNIT lattice of lnx x lny translations from (ix0, iy0) and
    // emit only the poses on the grid, (ix, iy) = (X / sx, Y / sy); unit
    // grids have sx = sy = 1, lnx = nx, lny = ny.
    int sx, sy;
    unsigned long long lnx, lny;
    int ro;           // region kernel: bound on |lattice offset| of every rotated point
    int edge;         // smem kernel: zero columns shrunk to fit, windows may need clamping
    // Thetas with a rounding-ambiguous lattice offset (amb[it] > 0) are left
    // to the general kernel (exact fp64 centres): the lattice kernels skip
    // them (item_max = +inf so compaction scans their map), the general kernel
    // runs over the list amb[nth + 1 ..] of amb[nth] entries.
    const int* amb;
    int kf;           // histogram floor rank (the search's k if <= 8, else 0 = off)
    float K;          // fixed-point fold constant 3*2^e
    unsigned B3;      // bits of K
    float scale;      // 2^(e-22) / n
    float* map;       // (it - it_begin) * nx * ny + iy * nx + ix
    float* item_max;  // best screen score per work item (lattice tile / 32 poses)
    unsigned* hist;   // kHistBins
    SearchCtrl* ctrl;
    unsigned long long* prof;  // optional phase timestamps (EAB_SCREEN_PROF)
    unsigned long long* wtrace;  // optional per-warp unit end stamps [warp][8] (EAB_SCREEN_TRACE)
    // exact-zero translation tiles (nwx * nwy flags, theta-independent; null
    // = none known): no edge pixel (|g| >= eps) within any window of any
    // pose of the tile, so every such pose scores exactly 0 (similarity.cpp:
    // 102-118, kernels_scalar.cpp:44-50) -- the screen skips their work
    const unsigned char* zero_tiles;
    // top-list mode (smem lattice kernel, 1 <= kf <= 8, no flagged theta):
    // no histogram; each CTA writes its kf largest tile maxima here
    // ([CTA][kTopK]) and the finish takes the band threshold from them
    float* cta_top;
    float map_margin;  // top-list mode: 4 delta rounded up (emit_tile's map floor)
};

// Dynamic shared memory the lattice kernel needs for a plane.
size_t fast_smem_bytes(const PlaneGeom& g);
// Returns true if the smem lattice kernel handled the launch.
bool launch_screen_fast(ea_ctx* ctx, const ScreenArgs& a);
// Region-tiled lattice kernel for planes larger than shared memory (float2
// plane in global memory, one warp tile + model-radius halo per CTA stage).
// Returns false when even one halo region does not fit.
bool launch_screen_region(ea_ctx* ctx, const ScreenArgs& a);
void launch_screen_general(ea_ctx* ctx, const ScreenArgs& a);
// Exact-zero flags of the lattice kernel's translation tiles (nwx x nwy tiles
// of tw x th poses from lattice origin (ix0, iy0)): 1 when no pixel of the
// field within `halo` of the tile has |g| >= eps.
void launch_zero_tiles(ea_ctx* ctx, const ea_field* f, double eps, int ix0, int iy0,
                       unsigned nwx, unsigned nwy, int tw, int th, int halo,
                       unsigned char* out);
// The general kernel over the flagged thetas of a lattice launch only.
void launch_screen_flagged(ea_ctx* ctx, const ScreenArgs& a);

void launch_threshold(ea_ctx* ctx, const unsigned* hist, int k, double delta, SearchCtrl* ctrl);
void launch_point_vote(ea_ctx* ctx, const ea_field* f, int cx, int cy, int R, double dx,
                       double dy, double eps, bool absolute, double* out);
// Work-item geometry of the screening map, for the compaction pass.
struct ItemGeom {
    unsigned long long n_items;
    int lattice;           // 1: items are (theta, wy, wx) tiles of cols x rows poses
    unsigned nwx, nwy, rows, cols;
    unsigned long long nx, ny, total;
    int sx, sy;            // lattice steps (tiles are on the unit lattice; see ScreenArgs)
};
ItemGeom screen_items(const ScreenArgs& a, bool fast);
// Compaction with the band threshold (see launch_threshold) computed in-kernel.
void launch_compact(ea_ctx* ctx, const float* map, const float* item_max, const ItemGeom& g,
                    SearchCtrl* ctrl, unsigned* cand, unsigned long long cap,
                    const unsigned* hist, int k, double delta, const int* flags);

struct ExactArgs {
    const double* gx;
    const double* gy;
    const double* mag;
    int W, H, R, ignore;
    double eps;
    const double* rot_exact;  // px|py|dx|dy, rows theta - it_begin, stride rot_stride
    size_t rot_stride;
    int n;
    unsigned long long nx, ny, it_begin;
    double x0, dx, y0, dy;
};
// Exact fp64 scores of candidate poses (index relative to it_begin * plane).
void launch_rescore(ea_ctx* ctx, const ExactArgs& a, const unsigned* cand,
                    const SearchCtrl* ctrl, unsigned long long cap, double* score);
// Top k of the candidates by `better` (search.cpp:36-41) -> out_score/out_index
// (global grid index).
void launch_select(ea_ctx* ctx, const unsigned* cand, const double* score,
                   SearchCtrl* ctrl, unsigned long long cap, int k,
                   unsigned long long index_base, double* out_score,
                   unsigned long long* out_index);
// Device-resident top-k rows {score, index, ux, uy, theta} (f64 x 5) of a
// search (pose_at on the device) + overflow flag; and the `better` merge of
// n such rows into k.
struct RowGrid {
    double x0, dx, y0, dy, t0, dt;
    unsigned long long nx, ny;
};
void launch_topk_rows(ea_ctx* ctx, const double* score, const unsigned long long* index,
                      const SearchCtrl* ctrl, unsigned long long cap, int k, const RowGrid& g,
                      double* rows, int* overflow);
// top_score/top_index/n_top (optional): the merged top k as a search's
// select leaves it.  n <= merge_rows_max(ctx) rows (shared-memory staging).
void launch_merge_rows(ea_ctx* ctx, const double* in, int n, int k, double* out,
                       double* top_score = nullptr, unsigned long long* top_index = nullptr,
                       int* n_top = nullptr);
int merge_rows_max(ea_ctx* ctx);
// Per-model merge of a multi-model all-gather: rank r's rows of model m at
// in[(r * n_models + m) * k ..]; model m's merged rows at out[m * k ..] and
// its seeds at top_score/top_index[m * k ..], n_top[m].
void launch_merge_rows_multi(ea_ctx* ctx, const double* in, int world, int n_models, int k,
                             double* out, double* top_score, unsigned long long* top_index,
                             int* n_top);
// compaction + rescore + select (+ rows when rows != nullptr) in one
// cooperative launch; same results as launch_compact/rescore/select/topk_rows.
struct FinishArgs {
    const float* map;
    const float* item_max;
    ItemGeom items;
    SearchCtrl* ctrl;
    unsigned* cand;
    unsigned long long cap;
    const unsigned* hist;
    unsigned* hist_rw;  // the same histogram, cleared after the threshold
    int k;
    double delta;
    const int* flags;
    ExactArgs x;
    double* cand_score;
    unsigned long long index_base;
    double* out_score;
    unsigned long long* out_index;
    RowGrid rg;
    double* rows;
    int* overflow;
    unsigned long long* prof;  // optional phase timestamps (EAB_FINISH_PROF)
    const unsigned char* zero_tiles;  // exact-zero translation tiles (ScreenArgs::zero_tiles)
    float* cta_top;            // top-list mode: [CTA][kTopK] largest tile maxima per screen CTA
    int n_lists;               // screen CTAs that wrote cta_top
};
void launch_finish(ea_ctx* ctx, const FinishArgs& f);
// Screen + finish in ONE cooperative launch (smem lattice kernel, k <= 8,
// no flagged theta): the band threshold comes from the exact k-th largest
// screen score (per-CTA top k, merged after a grid barrier) instead of the
// histogram.  false = not eligible: use the launch_screen_fast +
// launch_finish pair.
bool launch_screen_fused(ea_ctx* ctx, const ScreenArgs& a, const FinishArgs& f);
constexpr int kTopK = 8;  // largest k of the fused path (per-warp top-k lists)
// Dense exact map (score_map search.cpp:169-202).
void launch_exact_map(ea_ctx* ctx, const ExactArgs& a, unsigned long long total, double* out);

// Refinement: exact scores of an explicit pose list (ux, uy, rot slot).
void launch_refine_score(ea_ctx* ctx, const ExactArgs& a, const double* poses /*ux,uy*/,
                         const int* slot, int count, double* score, int* n_inb);
// Stable sort by score desc + exact-duplicate removal + keep topk
// (search.cpp:323-346).  entries: ux, uy, theta, parent; out beam rows.
void launch_beam_select(ea_ctx* ctx, const double* poses3, const double* score,
                        const int* parent, int count, int topk, double* beam_out,
                        int* beam_parent, int* beam_count);

}  // namespace eab
