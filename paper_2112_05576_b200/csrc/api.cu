// api.cu -- the C-ABI of include/edgealign_b200.h: host orchestration of the
// sm_100a kernels, mirroring the reference API one entry point at a time.
//
// Host fp64 arithmetic that must match the reference bit for bit (grid
// lattice, refinement lattice, glibc cos/sin of every searched theta) is
// compiled with -ffp-contract=off, like the reference (CMakeLists.txt:12-14).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "host_model.h"
#include "kernels.cuh"
#include "nccl_dl.h"
#include "model.cuh"
#include "refine.cuh"

using namespace eab;

namespace {

thread_local std::string g_err;
thread_local double g_err_value = 0.0;

template <class F>
ea_status guard(F&& f) {
    try {
        f();
        g_err.clear();
        g_err_value = 0.0;
        return EA_OK;
    } catch (const Failure& e) {
        g_err = e.what();
        g_err_value = e.value;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return EA_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return EA_ERR_INTERNAL;
    }
}

void need(const void* p, const char* what) {
    if (!p) fail(EA_ERR_INVALID_ARGUMENT, std::string(what) + " must not be null");
}

// ---- pose geometry: pose.h:45-92 ----------------------------------------------
uint64_t axis_count(double lo, double hi, double step) {  // pose.h:45-49
    return (uint64_t)std::floor((hi - lo) / step + 1e-9) + 1;
}

ea_grid_counts counts_of(const ea_pose_grid& g) {  // pose.h:52-67
    if (!(std::isfinite(g.x0) && std::isfinite(g.x1) && std::isfinite(g.dx) &&
          std::isfinite(g.y0) && std::isfinite(g.y1) && std::isfinite(g.dy) &&
          std::isfinite(g.t0) && std::isfinite(g.t1) && std::isfinite(g.dt))) {
        fail(EA_ERR_INVALID_ARGUMENT, "pose grid has non-finite bounds");
    }
    if (g.dx <= 0.0 || g.dy <= 0.0 || g.dt <= 0.0)
        fail(EA_ERR_INVALID_ARGUMENT, "pose grid steps must be positive");
    if (g.x0 > g.x1 || g.y0 > g.y1 || g.t0 > g.t1)
        fail(EA_ERR_INVALID_ARGUMENT, "pose grid range start exceeds end");
    return ea_grid_counts{axis_count(g.x0, g.x1, g.dx), axis_count(g.y0, g.y1, g.dy),
                          axis_count(g.t0, g.t1, g.dt)};
}

ea_pose pose_of(const ea_pose_grid& g, const ea_grid_counts& c, uint64_t index) {
    const uint64_t total = c.nx * c.ny * c.nt;
    if (index >= total) {
        fail(EA_ERR_BOUNDS, "pose index " + std::to_string(index) + " out of range (grid size " +
                                std::to_string(total) + ")");
    }
    const uint64_t plane = c.nx * c.ny;
    const uint64_t it = index / plane, rem = index % plane;
    const uint64_t iy = rem / c.nx, ix = rem % c.nx;
    return ea_pose{g.x0 + (double)ix * g.dx, g.y0 + (double)iy * g.dy, g.t0 + (double)it * g.dt};
}

void validate_params(const ea_score_params& p) {  // similarity.cpp:15-23
    if (p.neighborhood < 1 || p.neighborhood % 2 == 0) {
        fail(EA_ERR_INVALID_ARGUMENT,
             "neighborhood must be odd and >= 1, got " + std::to_string(p.neighborhood));
    }
    if (!(p.eps_mag > 0.0)) fail(EA_ERR_INVALID_ARGUMENT, "eps_mag must be positive");
}

// ---- device plumbing ---------------------------------------------------------
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) EAB_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

void h2d(ea_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes) EAB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
}
void d2h(ea_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes) EAB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
}
void sync(ea_ctx* ctx) { EAB_CUDA(cudaStreamSynchronize(ctx->stream)); }

// H2D of pageable host data through the context's pinned staging buffer.
void h2d_staged(ea_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, src) == cudaSuccess &&
        attr.type == cudaMemoryTypeHost) {  // already pinned
        h2d(ctx, dst, src, bytes);
        return;
    }
    cudaGetLastError();
    sync(ctx);  // staging buffer may still feed an earlier copy
    void* st = ctx->h_stage.ensure(bytes);
    std::memcpy(st, src, bytes);
    h2d(ctx, dst, st, bytes);
}

// glibc cos/sin of theta_it = t0 + (double)it * dt (scan_range search.cpp:81-84,
// rotate_model similarity.cpp:68-70), cached per grid.
const std::vector<double>& theta_cs(ea_ctx* ctx, double t0, double dt, uint64_t nt) {
    std::vector<double> key{t0, dt, (double)nt};
    auto it = ctx->cs_cache.find(key);
    if (it != ctx->cs_cache.end()) return it->second;
    if (ctx->cs_cache.size() > 64) ctx->cs_cache.clear();
    std::vector<double> cs(2 * nt);
    for (uint64_t i = 0; i < nt; ++i) {
        const double theta = t0 + (double)i * dt;
        cs[2 * i] = std::cos(theta);
        cs[2 * i + 1] = std::sin(theta);
    }
    return ctx->cs_cache.emplace(std::move(key), std::move(cs)).first->second;
}

ea_field* new_field(int w, int h) {
    auto* f = new ea_field;
    f->width = w;
    f->height = h;
    f->version = next_field_version();
    try {
        f->g.ensure(sizeof(double) * 3 * (size_t)w * h);
    } catch (...) {
        delete f;
        throw;
    }
    return f;
}

void sobel_into(ea_ctx* ctx, const double* d_img, int w, int h, ea_field* f) {
    if (w < 3 || h < 3) {
        fail(EA_ERR_SIZE, "compute_gradients needs at least 3x3, got " + std::to_string(w) + "x" +
                              std::to_string(h));
    }
    launch_sobel(ctx, d_img, w, h, f->gx(), f->gy(), f->mag());
    f->version = next_field_version();
    f->ring_max = 0.0;  // Sobel leaves the border ring at exactly 0
}

ea_model* new_model(ea_ctx* ctx, const ea_edge_point* pts, int n, double cx, double cy,
                    int level) {
    auto* m = new ea_model;
    try {
        m->n = n;
        m->centroid_x = cx;
        m->centroid_y = cy;
        m->source_level = level;
        m->host.assign(pts, pts + n);
        if (n > 0) {
            std::vector<double> soa(4 * (size_t)n);
            for (int i = 0; i < n; ++i) {
                soa[i] = pts[i].x_rel;
                soa[n + i] = pts[i].y_rel;
                soa[2 * n + i] = pts[i].dx;
                soa[3 * n + i] = pts[i].dy;
            }
            m->pts.ensure(soa.size() * sizeof(double));
            h2d_staged(ctx, m->pts.p, soa.data(), soa.size() * sizeof(double));
            sync(ctx);
        }
    } catch (...) {
        delete m;
        throw;
    }
    return m;
}

int pyramid_levels_feasible(int w, int h) {  // image.cpp:263-272
    int levels = 1;
    while (w / 2 >= 8 && h / 2 >= 8) {
        w /= 2;
        h /= 2;
        ++levels;
    }
    return levels;
}

// build_pyramid (image.cpp:274-291) on the device: level 0 at d_buf, each next
// level appended.  Returns level offsets/dims.
// build_pyramid (image.cpp:274-291) on the device.  Level 0 is read from
// `level0` (may alias d_buf); levels >= 1 are written to d_buf at *offs.
void device_pyramid_from(ea_ctx* ctx, const double* level0, double* d_buf, int w, int h,
                         int levels, std::vector<const double*>* srcs, std::vector<int>* dims) {
    if (levels < 1) fail(EA_ERR_INVALID_ARGUMENT, "num_levels must be >= 1");
    const int feasible = pyramid_levels_feasible(w, h);
    if (levels > feasible) {
        fail(EA_ERR_SIZE, "pyramid of " + std::to_string(levels) +
                              " levels would drop below 8x8; maximum feasible level count is " +
                              std::to_string(feasible));
    }
    const double* src = level0;
    double* dst = d_buf;
    for (int l = 0; l < levels; ++l) {
        srcs->push_back(src);
        dims->push_back(w);
        dims->push_back(h);
        if (l + 1 < levels) {
            launch_downsample(ctx, src, w, h, dst);
            src = dst;
            dst += (size_t)(w / 2) * (h / 2);
        }
        w /= 2;
        h /= 2;
    }
}

void device_pyramid(ea_ctx* ctx, double* d_buf, int w, int h, int levels,
                    std::vector<size_t>* offs, std::vector<int>* dims) {
    if (levels < 1) fail(EA_ERR_INVALID_ARGUMENT, "num_levels must be >= 1");
    const int feasible = pyramid_levels_feasible(w, h);
    if (levels > feasible) {
        fail(EA_ERR_SIZE, "pyramid of " + std::to_string(levels) +
                              " levels would drop below 8x8; maximum feasible level count is " +
                              std::to_string(feasible));
    }
    size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        offs->push_back(off);
        dims->push_back(w);
        dims->push_back(h);
        if (l + 1 < levels) launch_downsample(ctx, d_buf + off, w, h, d_buf + off + (size_t)w * h);
        off += (size_t)w * h;
        w /= 2;
        h /= 2;
    }
}

size_t pyramid_elems(int w, int h, int levels) {
    size_t t = 0;
    for (int l = 0; l < levels; ++l) {
        t += (size_t)w * h;
        w /= 2;
        h /= 2;
    }
    return t;
}

// ---- the top-level search --------------------------------------------------------
struct TopOut {
    std::vector<ea_scored_pose> poses;
};

bool is_int(double v) { return std::floor(v) == v && std::fabs(v) <= 1048576.0; }

ExactArgs exact_args(const ea_field* f, const ea_score_params& p, const double* rot,
                     size_t rot_stride, int n) {
    ExactArgs x{};
    x.gx = f->gx();
    x.gy = f->gy();
    x.mag = f->mag();
    x.W = f->width;
    x.H = f->height;
    x.R = (p.neighborhood - 1) / 2;
    x.ignore = p.polarity == EA_POLARITY_IGNORE;
    x.eps = p.eps_mag;
    x.rot_exact = rot;
    x.rot_stride = rot_stride;
    x.n = n;
    return x;
}

// Shared by search_topk, search_top_slab and screen_map: tables, plane and the
// screening pass.  Returns the fixed-point exponent chosen.
struct ScreenPlan {
    ea_grid_counts c{};
    uint64_t it_begin = 0, it_count = 0, slab_poses = 0;
    int fold_e = 0;
    double delta = 0.0;
    bool fast = false;
    bool fused = false;  // the screen launch also ran the finish (launch_screen_fused)
    float* cta_top = nullptr;  // top-list mode: the screen's per-CTA lists (FinishArgs::cta_top)
    const unsigned char* zero_tiles = nullptr;  // exact-zero tile flags (lattice kernel)
    ItemGeom items{};
    const double* rot = nullptr;  // exact rotation table of the slab (model cache)
    const int* flags = nullptr;   // device count of rounding-ambiguous pairs
};

// What the fused screen + finish launch needs from the search (top_enqueue).
struct FusedReq {
    unsigned long long cap;
    double* top_score;
    unsigned long long* top_index;
    double* d_rows;
    int* overflow;
};

// k: the search's top-k (enables the screen kernels' histogram floor when
// k <= kFloorK); 0 for a plain screening map.  req: a top-k search that may
// run its finish inside the screen launch (plan.fused reports whether it did).
ScreenPlan screen(ea_ctx* ctx, const ea_model* m, const ea_field* f, const ea_pose_grid& g,
                  const ea_score_params& p, uint64_t it_begin, uint64_t it_end, int k = 0,
                  const FusedReq* req = nullptr) {
    ScreenPlan plan;
    plan.c = counts_of(g);
    if (it_end == 0 || it_end > plan.c.nt) it_end = plan.c.nt;
    if (it_begin > it_end) it_begin = it_end;
    plan.it_begin = it_begin;
    plan.it_count = it_end - it_begin;
    const uint64_t plane_poses = plan.c.nx * plan.c.ny;
    plan.slab_poses = plane_poses * plan.it_count;
    if (plan.slab_poses >= (1ull << 32))
        fail(EA_ERR_INVALID_ARGUMENT, "pose grid slab exceeds 2^32 poses; shard it by theta");
    const int n = m->n;
    const int R = (p.neighborhood - 1) / 2;

    // Tables for the slab's thetas, cached on the model (see ea_model::tab_key).
    const size_t nth = plan.it_count;
    const size_t slab_pairs = nth * (size_t)n;
    ea_model* mm = const_cast<ea_model*>(m);
    // (R: twins in the schedule only for R <= 1)
    const std::vector<double> key{g.t0, g.dt, (double)plan.c.nt, (double)it_begin, (double)nth,
                                  (double)std::min(R, 2)};
    double* rot = (double*)mm->rot.ensure(sizeof(double) * 4 * (slab_pairs ? slab_pairs : 1));
    int4* scr = (int4*)mm->scr.ensure(sizeof(int4) * (slab_pairs ? slab_pairs : 1));
    // per-theta ambiguous-point counts, the flagged-theta list (ScreenArgs::amb)
    // and, in the last slot, the total of ambiguous pairs
    // (+ a 64-bit count of twinned points for the schedule mode, 8-aligned)
    const size_t amb_words = 2 * nth + 3, tw_off = (amb_words + 1) & ~(size_t)1;
    int* amb = (int*)mm->amb.ensure(sizeof(int) * tw_off + sizeof(unsigned long long));
    unsigned long long* twinned = reinterpret_cast<unsigned long long*>(amb + tw_off);
    int4* sched = (int4*)mm->sched.ensure(sizeof(int4) * (nth ? nth : 1) * sched_stride(n));
    if (key != mm->tab_key) {
        mm->tab_key.clear();
        double* d_cs = (double*)ctx->cs.ensure(sizeof(double) * 2 * (nth ? nth : 1));
        if (key != ctx->cs_dev_key) {  // device copy of the slab's cos/sin
            const std::vector<double>& cs_all = theta_cs(ctx, g.t0, g.dt, plan.c.nt);
            ctx->cs_dev_key.clear();
            h2d_staged(ctx, d_cs, cs_all.data() + 2 * it_begin, sizeof(double) * 2 * nth);
            ctx->cs_dev_key = key;
        }
        EAB_CUDA(cudaMemsetAsync(amb, 0, sizeof(int) * tw_off + sizeof(unsigned long long),
                                 ctx->stream));
        launch_rotate(ctx, m->pts.as<double>(), n, d_cs, (int)nth, rot, scr, amb + 2 * nth + 2,
                      amb);
        // Schedule mode: twins (mode 1) when R <= 1, unless fewer than a fifth
        // of the points pair up as twins (round templates) -- then pairs.
        static const bool no_twins = std::getenv("EAB_NO_TWINS") != nullptr;
        int mode = (R <= 1 && !no_twins) ? 1 : 0;
        launch_schedule(ctx, scr, n, (int)nth, sched, mode, twinned);
        // once per model and slab: does any theta need the general kernel?
        int n_flagged = 0;
        unsigned long long n_twinned = 0;
        d2h(ctx, &n_flagged, amb + nth, sizeof n_flagged);
        d2h(ctx, &n_twinned, twinned, sizeof n_twinned);
        sync(ctx);
        if (mode == 1 && n_twinned * 5 < (unsigned long long)nth * n) {
            mode = 0;
            launch_schedule(ctx, scr, n, (int)nth, sched, mode, nullptr);
        }
        mm->n_flagged = n_flagged;
        mm->sched_mode = mode;
        mm->tab_key = key;
    }
    SearchCtrl* ctrl = (SearchCtrl*)ctx->ctrl.ensure(sizeof(SearchCtrl));
    unsigned* hist = (unsigned*)ctx->hist.ensure(sizeof(unsigned) * kHistBins);
    // (both cleared by the plane kernel below)
    plan.rot = rot;
    plan.flags = amb + 2 * nth + 2;

    // Fixed-point fold exponent: sums of n votes stay below 2^31.
    int e = 0;
    while (((uint64_t)n << (22 - e)) >= (1ull << 31)) ++e;
    plan.fold_e = e;
    const float K = std::ldexp(3.0f, e);
    unsigned B3;
    std::memcpy(&B3, &K, sizeof B3);
    // |S_f - S| <= 2^(e-20) (candidate + fold rounding) + 2^-23 (final fp32 store)
    plan.delta = std::ldexp(1.0, e - 20) + std::ldexp(1.0, -23);

    // Path choice.
    // Integer origin + unit steps: every translation is an exact integer,
    // so centre = floor(px + 0.5) + u (lattice_offset); x1/y1 only bound the
    // counts and must keep |u| < 2^20.
    // Integer steps sx, sy > 1 (the paper's 3 px grid) run the same kernels
    // on the unit lattice that covers the grid and emit only the grid's poses
    // (emit_tile_strided): sx * sy times the screening work of the grid, at
    // the lattice kernels' per-pose cost instead of the general kernel's.
    const bool int_steps = is_int(g.dx) && is_int(g.dy) && g.dx >= 1.0 && g.dy >= 1.0 &&
                           g.dx <= 64.0 && g.dy <= 64.0;
    const bool lattice = is_int(g.x0) && is_int(g.y0) && std::fabs(g.x1) <= 1048576.0 &&
                         std::fabs(g.y1) <= 1048576.0 && int_steps && R <= 2 &&
                         f->ring_max < p.eps_mag;
    const int sx = lattice ? (int)g.dx : 1, sy = lattice ? (int)g.dy : 1;
    const uint64_t lnx = lattice ? (plan.c.nx - 1) * (uint64_t)sx + 1 : plan.c.nx;
    const uint64_t lny = lattice ? (plan.c.ny - 1) * (uint64_t)sy + 1 : plan.c.ny;
    // Lane strips of 8 rows (64 accumulators, 8 warps/SM) measured faster
    // than 16 rows (128 accumulators: spills) on B200.
    const int shift = 3;
    const int elem = 8;  // float2 plane (an fp16 plane measured no faster: issue-bound)
    // Zero columns beyond the ring so no lattice window needs clamping:
    // |offset| <= ceil(max |p_i|) + 1 for every rotation of the model.
    int PL = 0, PR = 0;
    int ro_int = 0;
    bool edge = false;
    int xg = 4;
    {   // warp tile 32x64 or 16x128: whichever pads the translation grid least
        auto padded = [&](uint64_t cols, uint64_t rows) {
            return ((lnx + cols - 1) / cols * cols) * ((lny + rows - 1) / rows * rows);
        };
        xg = padded(16, 128) < padded(32, 64) ? 2 : 4;
    }
    // Region mode: even the unpadded plane exceeds shared memory, so the
    // plane stays in global memory and CTAs stage halo regions of it.
    const bool region =
        lattice && (fast_smem_bytes(plane_geom(f->width, f->height, shift, 0, 0, 8)) >
                        ctx->smem_optin ||
                    std::getenv("EAB_FORCE_REGION") != nullptr);
    if (lattice) {
        double rmax = 0.0;
        for (const ea_edge_point& q : m->host)
            rmax = std::max(rmax, std::sqrt(q.x_rel * q.x_rel + q.y_rel * q.y_rel));
        const long ro = (long)std::ceil(rmax) + 2;
        ro_int = (int)std::min<long>(ro, 1 << 20);
        const long tw = 8L * xg;  // warp tile width: the lanes' last window column
        const long ix0 = (long)g.x0, span = (long)((lnx + tw - 1) / tw) * tw;
        PL = (int)std::max(0L, ro + R - 1 - ix0);
        PR = (int)std::max(0L, ix0 + span + ro + R - f->width - 1);
        const size_t budget = ctx->smem_optin;  // hist + plane must fit one CTA
        auto bytes = [&](int l, int r) {
            return fast_smem_bytes(plane_geom(f->width, f->height, shift, l, r, elem));
        };
        const int PL0 = PL, PR0 = PR;
        while ((PL > 0 || PR > 0) && bytes(PL, PR) > budget) {  // shrink: clamp path covers
            if (PL >= PR) --PL; else --PR;
        }
        edge = PL < PL0 || PR < PR0;
        if (region) PL = PR = 0;  // halo regions are zero-filled instead
    }
    PlaneGeom geom = plane_geom(f->width, f->height, shift, PL, PR, elem);
    // Twin schedules run 4-row lane strips (32 accumulators, 16 warps per SM,
    // half the unrolled body per entry kind): with 8-row strips the twin
    // kernel's bodies overflowed the instruction cache (no_instructions 23%
    // of stall samples, IPC 2.05); with 4-row strips the cache holds them
    // (IPC 2.53) and shared-memory bandwidth binds (L1 94%).  Measured on
    // B200: cfg3 screen 0.636 -> 0.617 ms, cfg2 0.430 -> 0.402, cfg1 0.275 ->
    // 0.253 against 8-row pair schedules.  EAB_S8=1 keeps 8-row strips.
    static const bool s8 = std::getenv("EAB_S8") != nullptr;
    if (!s8 && mm->sched_mode == 1 && lattice && !region && !edge && R <= 1) {
        const PlaneGeom g4 = plane_geom(f->width, f->height, 2, PL, PR, elem);
        if (fast_smem_bytes(g4) <= ctx->smem_optin) geom = g4;
    }
    void* plane = ctx->plane.ensure(geom.bytes());
    // The plane is a function of the image (field), eps and the geometry:
    // rebuilt only when one of them changed.  Its kernel also clears the
    // histogram and control block, which otherwise the previous search's
    // finish left clear (hist_clean).
    const std::vector<double> pkey{(double)reinterpret_cast<uintptr_t>(f), (double)f->version,
                                   p.eps_mag, (double)geom.W, (double)geom.H, (double)geom.PL,
                                   (double)geom.PR, (double)geom.shift, (double)geom.elem_bytes,
                                   (double)reinterpret_cast<uintptr_t>(plane)};
    const bool fused = k >= 1 && ctx->fused_finish;
    if (pkey != ctx->plane_key || !ctx->hist_clean || !fused) {
        ctx->plane_key.clear();
        launch_plane(ctx, f, p.eps_mag, geom, plane, hist, kHistBins,
                     reinterpret_cast<unsigned*>(ctrl), (int)(sizeof(SearchCtrl) / sizeof(unsigned)));
        ctx->plane_key = pkey;
    }
    // dirty until the fused finish (which restores the between-searches
    // state) has been enqueued -- see top_enqueue
    ctx->hist_clean = false;
    float* map = (float*)ctx->map.ensure(sizeof(float) * (plan.slab_poses ? plan.slab_poses : 1));
    // per-item maxima: lattice warp tiles are >= 16 columns x 32 rows (a
    // bound that holds for any grid shape, however thin); the general kernel
    // keeps one per 32 poses
    const uint64_t lattice_items = ((lnx + 15) / 16) * ((lny + 31) / 32) * plan.it_count;
    float* item_max = (float*)ctx->item_max.ensure(
        sizeof(float) * (std::max<uint64_t>(plan.slab_poses / 32 + 1, lattice_items) + 64));

    ScreenArgs a{};
    a.plane = plane;
    a.geom = geom;
    a.rot_screen = scr;
    a.rot_exact = rot;
    a.rot_stride = slab_pairs;
    a.n = n;
    a.it_begin = it_begin;
    a.it_count = plan.it_count;
    a.nx = plan.c.nx;
    a.ny = plan.c.ny;
    a.sx = sx;
    a.sy = sy;
    a.lnx = lnx;
    a.lny = lny;
    a.ix0 = lattice ? (int)g.x0 : 0;
    a.iy0 = lattice ? (int)g.y0 : 0;
    a.x0 = g.x0;
    a.dx = g.dx;
    a.y0 = g.y0;
    a.dy = g.dy;
    a.R = R;
    a.ignore = p.polarity == EA_POLARITY_IGNORE;
    a.xg = xg;
    a.sched = sched;
    a.sched_mode = mm->sched_mode;
    // lane strip of the lattice kernel that will run (screen_items' tile
    // shape): the smem kernel's from its plane skew, the region kernel's from
    // the schedule mode (launch_screen_region)
    a.strip = region ? (a.sched_mode == 1 && R <= 1 ? 4 : 8) : (geom.shift == 2 ? 4 : 8);
    a.ro = ro_int;
    a.edge = edge ? 1 : 0;
    a.amb = amb;
    a.kf = (k >= 1 && k <= 8) ? k : 0;
    // Exact-zero translation tiles of the smem lattice kernel (a function of
    // the field, eps, the lattice origin, the tile shape and the model
    // radius: cached like the plane).  Flat regions skip the screen work, and
    // a featureless frame no longer floods the band with every pose (only the
    // first k poses of each zero tile can rank; finish_tile).
    if (lattice && !region && plan.slab_poses) {
        const int tw = 8 * xg, th = (32 / xg) * (geom.shift == 2 ? 4 : 8);
        const unsigned nwx = (unsigned)((lnx + tw - 1) / tw);
        const unsigned nwy = (unsigned)((lny + th - 1) / th);
        const int halo = ro_int + R;
        unsigned char* zt = (unsigned char*)ctx->ztiles.ensure((size_t)nwx * nwy);
        const std::vector<double> zkey{(double)reinterpret_cast<uintptr_t>(f), (double)f->version,
                                       p.eps_mag, g.x0, g.y0, (double)nwx, (double)nwy,
                                       (double)xg, (double)halo,
                                       (double)reinterpret_cast<uintptr_t>(zt)};
        if (zkey != ctx->ztiles_key) {
            ctx->ztiles_key.clear();
            launch_zero_tiles(ctx, f, p.eps_mag, (int)g.x0, (int)g.y0, nwx, nwy, tw, th, halo, zt);
            ctx->ztiles_key = zkey;
        }
        a.zero_tiles = zt;
        plan.zero_tiles = zt;
    }
    a.K = K;
    a.B3 = B3;
    a.scale = (float)(std::ldexp(1.0, e - 22) / (double)n);
    a.map = map;
    a.item_max = item_max;
    a.hist = hist;
    a.ctrl = ctrl;
    plan.fast = false;
    if (ctx->timing) {
        EAB_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
        EAB_CUDA(cudaEventRecord(ctx->tev[2 * ctx->tev_next], ctx->stream));
    }
    static unsigned long long* sprof = nullptr;  // EAB_SCREEN_PROF: phase timestamps
    static int nsprof = 0;
    if (std::getenv("EAB_SCREEN_PROF") && plan.slab_poses) {
        unsigned long long h[16];
        if (!sprof) {
            EAB_CUDA(cudaMalloc(&sprof, sizeof h));
        } else if (nsprof > 0) {
            EAB_CUDA(cudaStreamSynchronize(ctx->stream));
            EAB_CUDA(cudaMemcpy(h, sprof, sizeof h, cudaMemcpyDeviceToHost));
            std::fprintf(stderr, "[screen] ns from first entry: plane landed %lld, last warp loop end "
                         "%lld, last CTA loop end %lld, last merge / barrier 1 %lld",
                         (long long)(h[0] - h[4]), (long long)(h[1] - h[4]),
                         (long long)(h[2] - h[4]), (long long)(h[3] - h[4]));
            if (h[5])  // fused finish phases
                std::fprintf(stderr, ", threshold %lld, compaction %lld, barrier 2 %lld, rescore %lld, "
                             "select+rows %lld",
                             (long long)(h[8] - h[4]), (long long)(h[9] - h[4]),
                             (long long)(h[5] - h[4]), (long long)(h[6] - h[4]),
                             (long long)(h[7] - h[4]));
            std::fprintf(stderr, "\n");
        }
        EAB_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < 16; ++i) h[i] = (i == 0 || i == 4) ? ~0ull : 0ull;
        EAB_CUDA(cudaMemcpy(sprof, h, sizeof h, cudaMemcpyHostToDevice));
        ++nsprof;
        a.prof = sprof;
    }
    static unsigned long long* wtrace = nullptr;  // EAB_SCREEN_TRACE: per-warp unit stamps
    static int nwtrace = 0;
    if (std::getenv("EAB_SCREEN_TRACE") && plan.slab_poses) {
        const size_t nw = (size_t)ctx->sm_count * 16;
        if (!wtrace) {
            EAB_CUDA(cudaMalloc(&wtrace, nw * 8 * sizeof(unsigned long long)));
        } else if (nwtrace > 0) {
            EAB_CUDA(cudaStreamSynchronize(ctx->stream));
            std::vector<unsigned long long> h(nw * 8);
            EAB_CUDA(cudaMemcpy(h.data(), wtrace, h.size() * 8, cudaMemcpyDeviceToHost));
            unsigned long long t0 = ~0ull;
            for (size_t w = 0; w < nw; ++w)
                if (h[8 * w]) t0 = std::min(t0, h[8 * w]);
            std::vector<double> first, last, start;
            std::vector<int> cnt(8, 0);
            const unsigned long long m56 = (1ull << 56) - 1;
            for (size_t w = 0; w < nw; ++w) {
                if (!h[8 * w]) continue;
                const int u = (int)(h[8 * w + 7] >> 56);
                ++cnt[std::min(u, 7)];
                start.push_back((double)(h[8 * w] - t0) * 1e-3);
                if (u >= 2) first.push_back((double)(h[8 * w + 1] - t0) * 1e-3);
                last.push_back((double)((h[8 * w + 7] & m56) - (t0 & m56)) * 1e-3);
            }
            auto pct = [](std::vector<double> v, double q) {
                if (v.empty()) return 0.0;
                std::sort(v.begin(), v.end());
                return v[(size_t)(q * (v.size() - 1))];
            };
            std::fprintf(stderr, "[trace] warps %zu; units/warp:", start.size());
            for (int u = 0; u < 8; ++u) std::fprintf(stderr, " %d:%d", u, cnt[u]);
            std::fprintf(stderr, " | start us p0/50/100 %.1f/%.1f/%.1f | first unit end %.1f/%.1f/%.1f"
                         " | loop end %.1f/%.1f/%.1f/%.1f(p90)\n",
                         pct(start, 0), pct(start, .5), pct(start, 1), pct(first, 0),
                         pct(first, .5), pct(first, 1), pct(last, 0), pct(last, .5), pct(last, 1),
                         pct(last, .9));
        }
        EAB_CUDA(cudaStreamSynchronize(ctx->stream));
        EAB_CUDA(cudaMemset(wtrace, 0, (size_t)ctx->sm_count * 16 * 8 * sizeof(unsigned long long)));
        ++nwtrace;
        a.wtrace = wtrace;
    }
    // Top-list mode for a top-k search on the smem lattice kernel: no
    // histogram, band threshold M_k - 2 delta from the k-th largest tile
    // maximum (see fused_threshold) -- fewer candidates than the histogram
    // bin's lower edge, and no per-pose histogram atomics in the screen.
    // (Flagged thetas, scored by the general kernel, publish no tile maxima:
    // M_k over the lattice tiles alone is still <= T_f, and their items carry
    // item_max = +inf, so the compaction scans them whole.)
    if (plan.slab_poses && req && ctx->toplist && ctx->fused_finish && lattice &&
        (size_t)mm->n_flagged * 2 < nth && k >= 1 && k <= kTopK && ctx->sm_count <= 512) {
        a.cta_top = (float*)ctx->cta_top.ensure(sizeof(float) * kTopK * (size_t)ctx->sm_count);
        float mm4 = (float)(4.0 * plan.delta);
        if ((double)mm4 < 4.0 * plan.delta) mm4 = std::nextafter(mm4, INFINITY);
        a.map_margin = mm4;
        plan.cta_top = a.cta_top;
    }
    if (plan.slab_poses && req && ctx->fused_screen && plan.cta_top && !region &&
        mm->n_flagged == 0) {
        // screen + finish in one cooperative launch (no histogram)
        FinishArgs fa{};
        fa.map = map;
        fa.item_max = item_max;
        fa.items = screen_items(a, true);
        fa.ctrl = ctrl;
        fa.cap = req->cap;
        fa.cand = (unsigned*)ctx->cand.ensure(sizeof(unsigned) * req->cap);
        fa.cand_score = (double*)ctx->cand_score.ensure(sizeof(double) * req->cap);
        fa.k = k;
        fa.delta = plan.delta;
        fa.flags = nullptr;
        ExactArgs x = exact_args(f, p, rot, slab_pairs, n);
        x.nx = plan.c.nx;
        x.ny = plan.c.ny;
        x.it_begin = plan.it_begin;
        x.x0 = g.x0;
        x.dx = g.dx;
        x.y0 = g.y0;
        x.dy = g.dy;
        fa.x = x;
        fa.index_base = plan.it_begin * plan.c.nx * plan.c.ny;
        fa.out_score = req->top_score;
        fa.out_index = req->top_index;
        fa.rg = RowGrid{g.x0, g.dx, g.y0, g.dy, g.t0, g.dt, plan.c.nx, plan.c.ny};
        fa.rows = req->d_rows;
        fa.overflow = req->overflow;
        fa.cta_top = plan.cta_top;
        fa.zero_tiles = plan.zero_tiles;
        plan.fused = plan.fast = launch_screen_fused(ctx, a, fa);
    }
    if (plan.slab_poses && !plan.fused) {
        if (lattice) plan.fast = region ? launch_screen_region(ctx, a) : launch_screen_fast(ctx, a);
        if (!plan.fast) launch_screen_general(ctx, a);
        else if (mm->n_flagged > 0) launch_screen_flagged(ctx, a);  // thetas the lattice kernel skipped
    }
    if (ctx->timing) {
        EAB_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
        EAB_CUDA(cudaEventRecord(ctx->tev[2 * ctx->tev_next + 1], ctx->stream));
        ctx->tev_next = (ctx->tev_next + 1) % ea_ctx::kTimeRing;
        ctx->tev_pending = std::min(ctx->tev_pending + 1, ea_ctx::kTimeRing);
    }
    ctx->stats.screen_path = plan.fast ? (region ? 3 : 1) : 2;
    plan.items = screen_items(a, plan.fast);
    return plan;
}

// run_search (search.cpp:95-140) on theta indices [it_begin, it_end), split in
// an enqueue half (everything up to the top-k select, results stay on the
// device in ctx->topk) and a collect half (one D2H + sync).
struct TopLaunch {
    ScreenPlan plan;
    unsigned long long cap = 0;
    int k = 0, n = 0;
    double* top_score = nullptr;
    unsigned long long* top_index = nullptr;
};

// d_rows: also write the k device rows {score, index, ux, uy, theta} (the
// multi-GPU data path) and raise *overflow if the band overflowed `cap`.
TopLaunch top_enqueue(ea_ctx* ctx, const ea_model* m, const ea_field* f, const ea_pose_grid& g,
                      const ea_score_params& p, int k, uint64_t it_begin, uint64_t it_end,
                      unsigned long long cap, double* d_rows = nullptr,
                      int* overflow = nullptr) {
    validate_params(p);
    if (m->n == 0) fail(EA_ERR_INVALID_ARGUMENT, "search needs a nonempty model");
    if (k < 1) fail(EA_ERR_INVALID_ARGUMENT, "topk must be >= 1");
    ctx->stats = ea_search_stats{};
    if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
    TopLaunch t;
    double* tk = (double*)ctx->topk.ensure((sizeof(double) + sizeof(unsigned long long)) * (size_t)k);
    t.top_score = tk;
    t.top_index = reinterpret_cast<unsigned long long*>(tk + k);
    const FusedReq req{cap, t.top_score, t.top_index, d_rows, overflow};
    t.plan = screen(ctx, m, f, g, p, it_begin, it_end, k, &req);
    t.k = k;
    t.n = m->n;
    t.cap = cap;
    ctx->stats.poses = t.plan.slab_poses;
    ctx->stats.pose_points = t.plan.slab_poses * (uint64_t)m->n;
    SearchCtrl* ctrl = ctx->ctrl.as<SearchCtrl>();
    if (t.plan.slab_poses == 0) return t;
    if (t.plan.fused) {  // the screen launch ran the finish; the histogram was not touched
        ctx->hist_clean = true;
        return t;
    }

    const size_t slab_pairs = t.plan.it_count * (size_t)t.n;
    ExactArgs x = exact_args(f, p, t.plan.rot, slab_pairs, t.n);
    x.nx = t.plan.c.nx;
    x.ny = t.plan.c.ny;
    x.it_begin = t.plan.it_begin;
    x.x0 = g.x0;
    x.dx = g.dx;
    x.y0 = g.y0;
    x.dy = g.dy;
    unsigned* cand = (unsigned*)ctx->cand.ensure(sizeof(unsigned) * cap);
    double* cs = (double*)ctx->cand_score.ensure(sizeof(double) * cap);
    const unsigned long long index_base = t.plan.it_begin * t.plan.c.nx * t.plan.c.ny;
    const RowGrid rg{g.x0, g.dx, g.y0, g.dy, g.t0, g.dt, t.plan.c.nx, t.plan.c.ny};
    if (ctx->fused_finish) {
        // band threshold, compaction, exact rescore, select (+ rows): one launch
        FinishArgs fa{};
        fa.map = ctx->map.as<float>();
        fa.item_max = ctx->item_max.as<float>();
        fa.items = t.plan.items;
        fa.ctrl = ctrl;
        fa.cand = cand;
        fa.cap = cap;
        fa.hist = ctx->hist.as<unsigned>();
        fa.hist_rw = ctx->hist.as<unsigned>();
        fa.k = k;
        fa.delta = t.plan.delta;
        fa.flags = t.plan.flags;
        fa.x = x;
        fa.cand_score = cs;
        fa.index_base = index_base;
        fa.out_score = t.top_score;
        fa.out_index = t.top_index;
        fa.rg = rg;
        fa.rows = d_rows;
        fa.overflow = overflow;
        fa.cta_top = t.plan.fast ? t.plan.cta_top : nullptr;
        fa.n_lists = ctx->screen_ctas;
        fa.zero_tiles = t.plan.fast && ctx->stats.screen_path == 1 ? t.plan.zero_tiles : nullptr;
        launch_finish(ctx, fa);
        ctx->hist_clean = true;
        return t;
    }
    // band threshold from the histogram, then the compaction
    launch_compact(ctx, ctx->map.as<float>(), ctx->item_max.as<float>(), t.plan.items, ctrl, cand,
                   cap, ctx->hist.as<unsigned>(), k, t.plan.delta, t.plan.flags);
    launch_rescore(ctx, x, cand, ctrl, cap, cs);
    launch_select(ctx, cand, cs, ctrl, cap, k, index_base, t.top_score, t.top_index);
    if (d_rows) launch_topk_rows(ctx, t.top_score, t.top_index, ctrl, cap, k, rg, d_rows, overflow);
    return t;
}

// Stats from the control block; false when the band overflowed the buffer.
bool top_stats(ea_ctx* ctx, const TopLaunch& t, const SearchCtrl& hc) {
    ctx->stats.candidates = hc.cand_count;
    ctx->stats.candidates_needed = hc.needed;
    ctx->stats.threshold = hc.thr;
    ctx->stats.flagged_points = hc.flags;
    ctx->stats.screen_delta = t.plan.delta;
    return hc.cand_count <= t.cap;
}

unsigned long long initial_cap(ea_ctx* ctx) {
    return std::max<size_t>(ctx->cand.cap / sizeof(unsigned), 1u << 16);
}

// Grids larger than one screening launch takes (the candidate indices are
// 32-bit and the fp32 map is 4 B/pose) are searched in theta chunks of at
// most kChunkPoses poses whose top-k lists are `better`-merged -- the merge
// is the reference's own (search.cpp:130-139), so the result is the same as
// one pass; the reference indexes poses with size_t (search.cpp:105-106).
constexpr uint64_t kChunkPoses = 1ull << 26;

// Candidate buffer of a search whose overflow cannot be retried from the host
// (device-resident and sharded searches): the whole slab when it has at most
// 2^26 poses, so the band can never overflow; larger slabs keep 2^26 and
// report an overflow (flag + an +inf row 0, see topk_rows_body).
unsigned long long async_cap(ea_ctx* ctx, uint64_t slab_poses) {
    return std::max<unsigned long long>(initial_cap(ctx),
                                        std::min<uint64_t>(slab_poses, 1ull << 26));
}

std::vector<std::pair<uint64_t, uint64_t>> theta_chunks(const ea_grid_counts& c, uint64_t b,
                                                        uint64_t e) {
    const uint64_t plane = c.nx * c.ny;
    if (plane >= (1ull << 32))
        fail(EA_ERR_INVALID_ARGUMENT, "one theta of the pose grid exceeds 2^32 translations");
    const uint64_t per = std::max<uint64_t>(1, kChunkPoses / std::max<uint64_t>(plane, 1));
    std::vector<std::pair<uint64_t, uint64_t>> out;
    for (uint64_t x = b; x < e; x += per) out.emplace_back(x, std::min(x + per, e));
    return out;
}

std::vector<ea_scored_pose> top_search_one(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                                           const ea_pose_grid& g, const ea_score_params& p, int k,
                                           uint64_t it_begin, uint64_t it_end);

std::vector<ea_scored_pose> top_search(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                                       const ea_pose_grid& g, const ea_score_params& p, int k,
                                       uint64_t it_begin, uint64_t it_end) {
    const ea_grid_counts c = counts_of(g);
    if (it_end == 0 || it_end > c.nt) it_end = c.nt;
    if (it_begin > it_end) it_begin = it_end;
    if ((it_end - it_begin) * c.nx * c.ny <= kChunkPoses)
        return top_search_one(ctx, m, f, g, p, k, it_begin, it_end);
    std::vector<ea_scored_pose> all;
    for (const auto& ch : theta_chunks(c, it_begin, it_end)) {
        const auto part = top_search_one(ctx, m, f, g, p, k, ch.first, ch.second);
        all.insert(all.end(), part.begin(), part.end());
    }
    std::stable_sort(all.begin(), all.end(), [](const ea_scored_pose& x, const ea_scored_pose& y) {
        if (x.score != y.score) return x.score > y.score;  // better: search.cpp:36-41
        return x.grid_index < y.grid_index;
    });
    if ((int)all.size() > k) all.resize(k);
    return all;
}

std::vector<ea_scored_pose> top_search_one(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                                           const ea_pose_grid& g, const ea_score_params& p, int k,
                                           uint64_t it_begin, uint64_t it_end) {
    unsigned long long cap = initial_cap(ctx);
    for (int attempt = 0; attempt < 3; ++attempt) {
        const TopLaunch t = top_enqueue(ctx, m, f, g, p, k, it_begin, it_end, cap);
        std::vector<ea_scored_pose> out;
        if (t.plan.slab_poses == 0) return out;
        const size_t res_bytes = (sizeof(double) + sizeof(unsigned long long)) * (size_t)k;
        char* h = (char*)ctx->h_out.ensure(sizeof(SearchCtrl) + res_bytes);
        d2h(ctx, h, ctx->ctrl.p, sizeof(SearchCtrl));
        d2h(ctx, h + sizeof(SearchCtrl), t.top_score, res_bytes);
        if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
        sync(ctx);
        if (ctx->timing) {
            float ms = 0.f;
            EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]));
            ctx->stats.screen_ms = ms;
            EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]));
            ctx->stats.top_ms = ms;
        }
        SearchCtrl hc;
        std::memcpy(&hc, h, sizeof hc);
        if (!top_stats(ctx, t, hc)) {  // band admitted more than the buffer: grow, redo
            cap = hc.cand_count;
            continue;
        }
        const double* hs = reinterpret_cast<const double*>(h + sizeof(SearchCtrl));
        const unsigned long long* hi = reinterpret_cast<const unsigned long long*>(hs + k);
        for (int r = 0; r < hc.n_out; ++r) {
            out.push_back(ea_scored_pose{hs[r], hi[r], pose_of(g, t.plan.c, hi[r])});
        }
        return out;
    }
    fail(EA_ERR_INTERNAL, "candidate buffer did not converge");
}

// ---- refinement (search_levels search.cpp:254-357) -----------------------------
struct Beam {
    ea_pose pose;
    double score;
    uint64_t top_index;
};

void refine_levels_host(ea_ctx* ctx, const ea_levels* lv, const ea_search_config& cfg,
                        const ea_pose_grid& top_grid, std::vector<Beam> beam, ea_outcome* out) {
    const int top = cfg.num_levels - 1;
    std::memset(out, 0, sizeof(*out));
    int nt = 0;
    auto trace = [&](int level, const Beam& b) {
        if (nt < EA_MAX_LEVELS) {
            out->trace[nt].level = level;
            out->trace[nt].pose = b.pose;
            out->trace[nt].score = b.score;
            ++nt;
        }
    };
    trace(top, beam[0]);
    const double theta_floor = 0.25 * (3.14159265358979323846 / 180.0);  // deg_to_rad(0.25)
    double step_x = top_grid.dx, step_y = top_grid.dy, step_t = top_grid.dt;
    const int R = cfg.refine_radius;
    const int side = 2 * R + 1;
    const ea_score_params& p = cfg.score_params;
    for (int level = top - 1; level >= 0; --level) {
        step_x /= 2.0;
        step_y /= 2.0;
        step_t = std::max(step_t / 2.0, theta_floor);
        const ea_model* m = lv->models[level];
        const ea_field* f = lv->fields[level];
        const int n = m->n;
        const int P = (int)beam.size();
        const int nslot = P * side;
        const int count = nslot * side * side;
        // host: thetas (glibc cos/sin) and the lattice in generation order
        const size_t cs_bytes = sizeof(double) * 2 * nslot;
        const size_t p2_bytes = sizeof(double) * 2 * count;
        const size_t p3_bytes = sizeof(double) * 3 * count;
        const size_t i_bytes = sizeof(int) * count;
        const size_t total = cs_bytes + p2_bytes + p3_bytes + 2 * i_bytes;
        sync(ctx);
        char* hb = (char*)ctx->h_stage.ensure(total);
        double* hcs = (double*)hb;
        double* hp2 = (double*)(hb + cs_bytes);
        double* hp3 = (double*)(hb + cs_bytes + p2_bytes);
        int* hslot = (int*)(hb + cs_bytes + p2_bytes + p3_bytes);
        int* hpar = hslot + count;
        int e = 0;
        for (int pi = 0; pi < P; ++pi) {
            const double cx = beam[pi].pose.ux * 2.0;
            const double cy = beam[pi].pose.uy * 2.0;
            const double ct = beam[pi].pose.theta;
            for (int kt = -R; kt <= R; ++kt) {
                const double theta = ct + (double)kt * step_t;
                const int slot = pi * side + (kt + R);
                hcs[2 * slot] = std::cos(theta);
                hcs[2 * slot + 1] = std::sin(theta);
                for (int ky = -R; ky <= R; ++ky) {
                    for (int kx = -R; kx <= R; ++kx) {
                        const double ux = cx + (double)kx * step_x;
                        const double uy = cy + (double)ky * step_y;
                        hp2[2 * e] = ux;
                        hp2[2 * e + 1] = uy;
                        hp3[3 * e] = ux;
                        hp3[3 * e + 1] = uy;
                        hp3[3 * e + 2] = theta;
                        hslot[e] = slot;
                        hpar[e] = pi;
                        ++e;
                    }
                }
            }
        }
        char* db = (char*)ctx->refine_poses.ensure(total);
        h2d(ctx, db, hb, total);
        const double* dcs = (const double*)db;
        const double* dp2 = (const double*)(db + cs_bytes);
        const double* dp3 = (const double*)(db + cs_bytes + p2_bytes);
        const int* dslot = (const int*)(db + cs_bytes + p2_bytes + p3_bytes);
        const int* dpar = dslot + count;
        const size_t pairs = (size_t)nslot * n;
        double* rot = (double*)ctx->rot_exact.ensure(sizeof(double) * 4 * (pairs ? pairs : 1));
        launch_rotate(ctx, m->pts.as<double>(), n, dcs, nslot, rot, nullptr, nullptr);
        double* sc = (double*)ctx->refine_scores.ensure(sizeof(double) * count);
        launch_refine_score(ctx, exact_args(f, p, rot, pairs, n), dp2, dslot, count, sc, nullptr);
        const int k = cfg.topk;
        char* bb = (char*)ctx->beam.ensure(sizeof(double) * 4 * k + sizeof(int) * (k + 1));
        double* bout = (double*)bb;
        int* bpar = (int*)(bb + sizeof(double) * 4 * k);
        int* bcnt = bpar + k;
        launch_beam_select(ctx, dp3, sc, dpar, count, k, bout, bpar, bcnt);
        const size_t bbytes = sizeof(double) * 4 * k + sizeof(int) * (k + 1);
        char* hbo = (char*)ctx->h_out.ensure(bbytes);
        d2h(ctx, hbo, bb, bbytes);
        sync(ctx);
        const double* hbout = (const double*)hbo;
        const int* hbpar = (const int*)(hbo + sizeof(double) * 4 * k);
        const int kept = hbpar[k];
        std::vector<Beam> next;
        for (int q = 0; q < kept; ++q) {
            next.push_back(Beam{ea_pose{hbout[4 * q], hbout[4 * q + 1], hbout[4 * q + 2]},
                                hbout[4 * q + 3], beam[hbpar[q]].top_index});
        }
        beam.swap(next);
        trace(level, beam[0]);
    }
    out->n_trace = nt;
    out->pose = beam[0].pose;
    out->score = beam[0].score;
    out->grid_index = beam[0].top_index;
    out->found = beam[0].score >= cfg.min_score ? 1 : 0;
}

// Device-resident refinement (refine_kernels.cu): host glibc cos/sin of every
// theta reachable from the seeds, then one votes + one select kernel per level
// and a single D2H of the outcome.
void refine_levels(ea_ctx* ctx, const ea_levels* lv, const ea_search_config& cfg,
                   const ea_pose_grid& top_grid, std::vector<Beam> seeds, ea_outcome* out) {
    const int top = cfg.num_levels - 1;
    const int R = cfg.refine_radius, side = 2 * R + 1, k = cfg.topk;
    const int ns = (int)seeds.size();
    const long e_max = (long)k * side * side * side;
    if (top == 0 || e_max > 4096) {
        refine_levels_host(ctx, lv, cfg, top_grid, std::move(seeds), out);
        return;
    }
    // per-level steps (search.cpp:286-295) and theta tables
    const double theta_floor = 0.25 * (3.14159265358979323846 / 180.0);
    std::vector<double> sx(top + 1), sy(top + 1), st(top + 1);
    std::vector<size_t> toff(top + 1, 0);
    double step_x = top_grid.dx, step_y = top_grid.dy, step_t = top_grid.dt;
    size_t tsize = 0, paths = (size_t)ns;
    for (int d = 1; d <= top; ++d) {
        step_x /= 2.0;
        step_y /= 2.0;
        step_t = std::max(step_t / 2.0, theta_floor);
        sx[d] = step_x;
        sy[d] = step_y;
        st[d] = step_t;
        paths *= (size_t)side;
        toff[d] = tsize;
        tsize += 3 * paths;
    }
    int n_max = 0;
    for (int l = 0; l < top; ++l) n_max = std::max(n_max, lv->models[l]->n);
    const size_t beam_bytes = sizeof(BeamDev) * (size_t)k;
    const size_t head = sizeof(ea_outcome) + 2 * beam_bytes + 2 * sizeof(int);
    const size_t host_bytes = head + sizeof(double) * tsize;
    sync(ctx);
    char* hb = (char*)ctx->h_stage.ensure(host_bytes);
    ea_outcome* hout = (ea_outcome*)hb;
    std::memset(hout, 0, sizeof(ea_outcome));
    hout->trace[0].level = top;
    hout->trace[0].pose = seeds[0].pose;
    hout->trace[0].score = seeds[0].score;
    hout->n_trace = 1;
    BeamDev* hbeam = (BeamDev*)(hb + sizeof(ea_outcome));
    for (int i = 0; i < ns; ++i) {
        hbeam[i] = BeamDev{seeds[i].pose.ux, seeds[i].pose.uy, seeds[i].pose.theta,
                           seeds[i].score, seeds[i].top_index, i, 0};
    }
    int* hcnt = (int*)(hb + sizeof(ea_outcome) + 2 * beam_bytes);
    hcnt[0] = ns;
    hcnt[1] = 0;
    double* htab = (double*)(hb + head);
    {
        std::vector<double> prev(ns);
        for (int i = 0; i < ns; ++i) prev[i] = seeds[i].pose.theta;
        for (int d = 1; d <= top; ++d) {
            std::vector<double> cur(prev.size() * side);
            double* t = htab + toff[d];
            for (size_t q = 0; q < prev.size(); ++q) {
                for (int kt = -R; kt <= R; ++kt) {
                    const size_t path = q * side + (size_t)(kt + R);
                    const double theta = prev[q] + (double)kt * st[d];  // search.cpp:305
                    cur[path] = theta;
                    t[3 * path] = theta;
                    t[3 * path + 1] = std::cos(theta);
                    t[3 * path + 2] = std::sin(theta);
                }
            }
            prev.swap(cur);
        }
    }
    const size_t ss = (size_t)side * side;
    const size_t E = (size_t)k * side * ss;
    char* db = (char*)ctx->refine_poses.ensure(host_bytes);
    h2d(ctx, db, hb, host_bytes);
    ea_outcome* dout = (ea_outcome*)db;
    BeamDev* dbeam[2] = {(BeamDev*)(db + sizeof(ea_outcome)),
                         (BeamDev*)(db + sizeof(ea_outcome) + beam_bytes)};
    int* dcnt[2] = {(int*)(db + sizeof(ea_outcome) + 2 * beam_bytes),
                    (int*)(db + sizeof(ea_outcome) + 2 * beam_bytes) + 1};
    const double* dtab = (const double*)(db + head);
    double* votes =
        (double*)ctx->refine_scores.ensure(sizeof(double) * (size_t)std::max(n_max, 1) * E);
    // entries: score|ux|uy|theta rows, order keys, dup flags
    double* entries = (double*)ctx->beam.ensure((sizeof(double) * 5 + sizeof(int)) * E);
    int* dup = (int*)(entries + 5 * E);
    const ea_score_params& sp = cfg.score_params;
    int cur = 0;
    for (int d = 1; d <= top; ++d) {
        const int level = top - d;
        const ea_model* m = lv->models[level];
        const ea_field* f = lv->fields[level];
        RefineArgs a{};
        a.pts = m->pts.as<double>();
        a.n = m->n;
        a.gx = f->gx();
        a.gy = f->gy();
        a.mag = f->mag();
        a.W = f->width;
        a.H = f->height;
        a.vote_R = (sp.neighborhood - 1) / 2;
        a.ignore = sp.polarity == EA_POLARITY_IGNORE;
        a.eps = sp.eps_mag;
        a.R = R;
        a.side = side;
        a.topk = k;
        a.max_parents = k;
        a.chunk = 16;
        a.level = level;
        a.trace_slot = d;
        a.step_x = sx[d];
        a.step_y = sy[d];
        a.min_score = cfg.min_score;
        a.table = dtab + toff[d];
        a.beam = dbeam[cur];
        a.beam_count = dcnt[cur];
        a.beam_out = dbeam[cur ^ 1];
        a.beam_count_out = dcnt[cur ^ 1];
        a.votes = votes;
        a.entries = entries;
        a.keys = reinterpret_cast<long long*>(entries + 4 * E);
        a.dup = dup;
        a.outcome = dout;
        launch_refine_level(ctx, a);
        cur ^= 1;
    }
    d2h(ctx, out, dout, sizeof(ea_outcome));
    sync(ctx);
}

// glibc (theta, cos, sin) for every refinement path of every top-level theta:
// level d holds nt * side^d entries, path = ((it*side + k1)*side + k2)...,
// theta_d = theta_{d-1} + (double)kt * step_t(d) (search.cpp:286-305).
// Cached per grid; nullptr when the tables would be too large.
const double* theta_tables(ea_ctx* ctx, const ea_pose_grid& tg, uint64_t nt, int top, int R) {
    std::vector<double> key{tg.t0, tg.dt, (double)nt, (double)top, (double)R};
    if (key == ctx->ttab_key) return ctx->ttab.as<double>();
    const int side = 2 * R + 1;
    size_t total = 0, level = nt;
    std::vector<size_t> off(top + 1, 0);
    for (int d = 1; d <= top; ++d) {
        level *= (size_t)side;
        off[d] = total;
        total += level;
        if (total > (16u << 20)) return nullptr;
    }
    std::vector<double> h(3 * (total ? total : 1));
    const double theta_floor = 0.25 * (3.14159265358979323846 / 180.0);
    std::vector<double> prev(nt), cur;
    for (uint64_t i = 0; i < nt; ++i) prev[i] = tg.t0 + (double)i * tg.dt;  // pose.h:91
    double st = tg.dt;
    for (int d = 1; d <= top; ++d) {
        st = std::max(st / 2.0, theta_floor);
        cur.assign(prev.size() * side, 0.0);
        double* t = h.data() + 3 * off[d];
        for (size_t q = 0; q < prev.size(); ++q) {
            for (int kt = -R; kt <= R; ++kt) {
                const size_t path = q * side + (size_t)(kt + R);
                const double theta = prev[q] + (double)kt * st;
                cur[path] = theta;
                t[3 * path] = theta;
                t[3 * path + 1] = std::cos(theta);
                t[3 * path + 2] = std::sin(theta);
            }
        }
        prev.swap(cur);
    }
    ctx->ttab_key.clear();
    double* d = (double*)ctx->ttab.ensure(sizeof(double) * h.size());
    h2d_staged(ctx, d, h.data(), sizeof(double) * h.size());
    sync(ctx);
    ctx->ttab_off = off;
    ctx->ttab_key = key;
    return d;
}

// Device refinement state: outcome | beam A | beam B | counts A, B.
struct RefineState {
    ea_outcome* out;
    BeamDev* beam[2];
    int* cnt[2];
};

// slot 0..2: independent states (batch mode refines image i on the refine
// stream while later images' top levels seed the other ones).
constexpr int kBatchSets = 3;
RefineState refine_state(ea_ctx* ctx, int k, int slot = 0) {
    const size_t beam_bytes = sizeof(BeamDev) * (size_t)k;
    const size_t one = (sizeof(ea_outcome) + 2 * beam_bytes + 4 * sizeof(int) + 255) & ~(size_t)255;
    char* b = (char*)ctx->rstate.ensure(kBatchSets * one) + one * slot;
    RefineState r;
    r.out = (ea_outcome*)b;
    r.beam[0] = (BeamDev*)(b + sizeof(ea_outcome));
    r.beam[1] = (BeamDev*)(b + sizeof(ea_outcome) + beam_bytes);
    r.cnt[0] = (int*)(b + sizeof(ea_outcome) + 2 * beam_bytes);
    r.cnt[1] = r.cnt[0] + 1;
    return r;
}

// Enqueue the refinement levels on a device beam (beam[0], cnt[0]).
void refine_enqueue(ea_ctx* ctx, const ea_levels* lv, const ea_search_config& cfg,
                    const ea_pose_grid& tg, const double* tables, const RefineState& st) {
    const int top = cfg.num_levels - 1;
    const int R = cfg.refine_radius, side = 2 * R + 1, k = cfg.topk;
    const size_t E = (size_t)k * side * side * side;
    int n_max = 0;
    for (int l = 0; l < top; ++l) n_max = std::max(n_max, lv->models[l]->n);
    double* votes =
        (double*)ctx->refine_scores.ensure(sizeof(double) * (size_t)std::max(n_max, 1) * E);
    // entries: score|ux|uy|theta rows, order keys, dup flags
    double* entries = (double*)ctx->beam.ensure((sizeof(double) * 5 + sizeof(int)) * E);
    int* dup = (int*)(entries + 5 * E);
    const ea_score_params& sp = cfg.score_params;
    double step_x = tg.dx, step_y = tg.dy;
    int cur = 0;
    for (int d = 1; d <= top; ++d) {
        step_x /= 2.0;  // search.cpp:293-294
        step_y /= 2.0;
        const int level = top - d;
        const ea_model* m = lv->models[level];
        const ea_field* f = lv->fields[level];
        RefineArgs a{};
        a.pts = m->pts.as<double>();
        a.n = m->n;
        a.gx = f->gx();
        a.gy = f->gy();
        a.mag = f->mag();
        a.W = f->width;
        a.H = f->height;
        a.vote_R = (sp.neighborhood - 1) / 2;
        a.ignore = sp.polarity == EA_POLARITY_IGNORE;
        a.eps = sp.eps_mag;
        a.R = R;
        a.side = side;
        a.topk = k;
        a.max_parents = k;
        a.chunk = 16;
        a.level = level;
        a.trace_slot = d;
        a.step_x = step_x;
        a.step_y = step_y;
        a.min_score = cfg.min_score;
        a.table = tables + 3 * ctx->ttab_off[d];
        a.beam = st.beam[cur];
        a.beam_count = st.cnt[cur];
        a.beam_out = st.beam[cur ^ 1];
        a.beam_count_out = st.cnt[cur ^ 1];
        a.votes = votes;
        a.entries = entries;
        a.keys = reinterpret_cast<long long*>(entries + 4 * E);
        a.dup = dup;
        a.outcome = st.out;
        launch_refine_level(ctx, a);
        cur ^= 1;
    }
}

SeedArgs seed_args(const ea_pose_grid& tg, const ea_grid_counts& c, const ea_search_config& cfg) {
    SeedArgs s{};
    s.x0 = tg.x0;
    s.dx = tg.dx;
    s.y0 = tg.y0;
    s.dy = tg.dy;
    s.t0 = tg.t0;
    s.dt = tg.dt;
    s.nx = c.nx;
    s.ny = c.ny;
    s.top_level = cfg.num_levels - 1;
    s.min_score = cfg.min_score;
    return s;
}

ea_pose_grid top_grid_of(const ea_search_config& cfg) {  // search.cpp:264-273
    const int top = cfg.num_levels - 1;
    const double scale = (double)(1 << top);
    ea_pose_grid g = cfg.grid;
    g.x0 /= scale;
    g.x1 /= scale;
    g.dx /= scale;
    g.y0 /= scale;
    g.y1 /= scale;
    g.dy /= scale;
    return g;
}

void check_search_config(const ea_levels* lv, const ea_search_config& cfg) {
    validate_params(cfg.score_params);
    if (cfg.topk < 1 || cfg.refine_radius < 1)
        fail(EA_ERR_INVALID_ARGUMENT, "topk and refine_radius must be >= 1");
    if (cfg.num_levels < 1 || (int)lv->models.size() < cfg.num_levels)
        fail(EA_ERR_INVALID_ARGUMENT, "prepared levels do not cover num_levels");
    if ((int)lv->fields.size() < cfg.num_levels)
        fail(EA_ERR_INVALID_ARGUMENT, "prepared levels have no working image");
    if (cfg.num_levels > EA_MAX_LEVELS)
        fail(EA_ERR_INVALID_ARGUMENT, "num_levels exceeds EA_MAX_LEVELS");
}

std::vector<Beam> seeds_to_beam(const std::vector<ea_scored_pose>& seeds) {
    std::vector<Beam> beam;
    for (const auto& s : seeds) beam.push_back(Beam{s.pose, s.score, s.grid_index});
    return beam;
}

void build_working(ea_ctx* ctx, ea_levels* lv, const double* d_level0, int w, int h,
                   int levels);
void build_working_into(ea_ctx* ctx, std::vector<ea_field*>& fields, DevBuf& image,
                        const double* d_level0, int w, int h, int levels);
void set_working_image(ea_ctx* ctx, ea_levels* lv, const double* image, int w, int h,
                       int levels);

// Theta tables for a config, or nullptr when refinement must be host-assisted.
const double* detect_tables(ea_ctx* ctx, const ea_search_config& cfg) {
    const int top = cfg.num_levels - 1;
    if (top == 0) return nullptr;
    const int k = cfg.topk, R = cfg.refine_radius, side = 2 * R + 1;
    if ((size_t)k * side * side * side > 4096 || k > 64) return nullptr;
    const ea_pose_grid tg = top_grid_of(cfg);
    return theta_tables(ctx, tg, counts_of(tg).nt, top, R);
}

// Enqueue search_levels (search.cpp:254-357) entirely on the device: top-level
// search -> seed beam -> refinement levels; the outcome lands in `d_out` and a
// copy of the control block (candidate count for the overflow check) in
// `d_ctrl`.  Nothing waits on the host.
TopLaunch enqueue_levels(ea_ctx* ctx, const ea_levels* lv, const ea_search_config& cfg,
                         const double* tables, unsigned long long cap, ea_outcome* d_out,
                         SearchCtrl* d_ctrl) {
    const int top = cfg.num_levels - 1;
    const int k = cfg.topk;
    const ea_pose_grid tg = top_grid_of(cfg);
    const ea_grid_counts c = counts_of(tg);
    TopLaunch t;
    if (c.nx * c.ny * c.nt > kChunkPoses) {
        // theta chunks (see kChunkPoses) merged on the device into the seeds;
        // an overflowing chunk marks its row 0 +inf, which ranks first and
        // surfaces as the outcome's top-level trace score (search_levels_device)
        const auto chunks = theta_chunks(c, 0, c.nt);
        const int n = (int)chunks.size() * k;
        if (n > merge_rows_max(ctx))
            fail(EA_ERR_INVALID_ARGUMENT, "pose grid too large for the chunk merge");
        double* tmp = (double*)ctx->chunk_rows.ensure(5 * sizeof(double) * ((size_t)n + k));
        for (size_t i = 0; i < chunks.size(); ++i) {
            const uint64_t cp = c.nx * c.ny * (chunks[i].second - chunks[i].first);
            t = top_enqueue(ctx, lv->models[top], lv->fields[top], tg, cfg.score_params, k,
                            chunks[i].first, chunks[i].second, async_cap(ctx, cp),
                            tmp + 5 * (size_t)k * i, nullptr);
        }
        launch_merge_rows(ctx, tmp, n, k, tmp + 5 * (size_t)n, t.top_score, t.top_index,
                          &ctx->ctrl.as<SearchCtrl>()->n_out);
    } else {
        t = top_enqueue(ctx, lv->models[top], lv->fields[top], tg, cfg.score_params, k, 0, 0, cap);
    }
    if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
    RefineState st = refine_state(ctx, k);
    st.out = d_out;
    EAB_CUDA(cudaMemsetAsync(st.out, 0, sizeof(ea_outcome), ctx->stream));
    launch_seed_beam(ctx, t.top_score, t.top_index, &ctx->ctrl.as<SearchCtrl>()->n_out,
                     seed_args(tg, c, cfg), st.beam[0], st.cnt[0], st.out);
    if (top > 0) refine_enqueue(ctx, lv, cfg, tg, tables, st);
    EAB_CUDA(cudaMemcpyAsync(d_ctrl, ctx->ctrl.p, sizeof(SearchCtrl), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    return t;
}

// search_levels for one image: enqueue, one D2H of (outcome, control), sync.
void search_levels_device(ea_ctx* ctx, const ea_levels* lv, const ea_search_config& cfg,
                          ea_outcome* out) {
    const int top = cfg.num_levels - 1;
    const double* tables = detect_tables(ctx, cfg);
    if (top > 0 && !tables) {  // very wide beams: host-assisted refinement
        const ea_pose_grid tg = top_grid_of(cfg);
        const auto seeds = top_search(ctx, lv->models[top], lv->fields[top], tg,
                                      cfg.score_params, cfg.topk, 0, 0);
        const ea_search_stats keep = ctx->stats;
        refine_levels(ctx, lv, cfg, tg, seeds_to_beam(seeds), out);
        const int launched = ctx->stats.kernels_launched;
        ctx->stats = keep;
        ctx->stats.kernels_launched = launched;
        return;
    }
    char* dres = (char*)ctx->rslots.ensure(sizeof(ea_outcome) + sizeof(SearchCtrl));
    ea_outcome* d_out = (ea_outcome*)dres;
    SearchCtrl* d_ctrl = (SearchCtrl*)(dres + sizeof(ea_outcome));
    unsigned long long cap = initial_cap(ctx);
    for (int attempt = 0; attempt < 3; ++attempt) {
        const TopLaunch t = enqueue_levels(ctx, lv, cfg, tables, cap, d_out, d_ctrl);
        char* h = (char*)ctx->h_out.ensure(sizeof(ea_outcome) + sizeof(SearchCtrl));
        d2h(ctx, h, dres, sizeof(ea_outcome) + sizeof(SearchCtrl));
        if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[7], ctx->stream));
        sync(ctx);
        if (ctx->timing) {
            float ms = 0.f;
            EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]));
            ctx->stats.screen_ms = ms;
            EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]));
            ctx->stats.top_ms = ms;
            EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[3], ctx->ev[7]));
            ctx->stats.refine_ms = ms;
        }
        SearchCtrl hc;
        std::memcpy(&hc, h + sizeof(ea_outcome), sizeof hc);
        if (top_stats(ctx, t, hc)) {
            std::memcpy(out, h, sizeof(ea_outcome));
            if (std::isinf(out->trace[0].score))  // a theta chunk overflowed (enqueue_levels)
                fail(EA_ERR_INTERNAL, "candidate buffer overflow in a chunked search");
            return;
        }
        cap = hc.cand_count;  // band admitted more than the buffer: grow, redo
    }
    fail(EA_ERR_INTERNAL, "candidate buffer did not converge");
}

// Batch detect (throughput mode): image i+1's H2D on a copy stream overlaps
// image i's device pipeline; outcomes come back asynchronously; one sync.
void detect_batch(ea_ctx* ctx, ea_levels* lv, const double* const* images, int count, int w,
                  int h, const ea_search_config& cfg, ea_outcome* outs) {
    const int L = cfg.num_levels;
    const double* tables = detect_tables(ctx, cfg);
    const ea_grid_counts gc0 = counts_of(top_grid_of(cfg));
    if ((L > 1 && !tables) || gc0.nx * gc0.ny * gc0.nt > kChunkPoses) {
        // host-assisted refinement, or a grid searched in theta chunks
        // (search_levels_device): no overlap, one by one
        for (int i = 0; i < count; ++i) {
            set_working_image(ctx, lv, images[i], w, h, L);
            search_levels_device(ctx, lv, cfg, outs + i);
        }
        return;
    }
    if (w < 1 || h < 1) {
        fail(EA_ERR_SIZE, "image dimensions must be at least 1x1, got " + std::to_string(w) + "x" +
                              std::to_string(h));
    }
    if (!ctx->copy_stream) EAB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream,
                                                              cudaStreamNonBlocking));
    for (auto& e : ctx->bev)
        if (!e) EAB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const size_t img_bytes = sizeof(double) * (size_t)w * h;
    double* raw[2] = {(double*)lv->raw[0].ensure(img_bytes), (double*)lv->raw[1].ensure(img_bytes)};
    const size_t slot = sizeof(ea_outcome) + sizeof(SearchCtrl);
    char* dres = (char*)ctx->rslots.ensure(slot * (size_t)count);
    char* hres = (char*)ctx->h_out.ensure(slot * (size_t)count);
    const unsigned long long cap = std::max<unsigned long long>(initial_cap(ctx), 1ull << 20);
    if (!ctx->refine_stream) {  // lowest priority: the next image's top level goes first
        int lo = 0, hi = 0;
        EAB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const int prio = std::getenv("EAB_REFINE_SAME_PRIO") ? 0 : lo;
        EAB_CUDA(cudaStreamCreateWithPriority(&ctx->refine_stream, cudaStreamNonBlocking, prio));
    }
    for (auto& e : ctx->rev)
        if (!e) EAB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // Three working sets (pyramid + fields) and refinement states: image i
    // refines on the refine stream from set/state i%3 while images i+1, i+2
    // build their pyramids and search their top levels on the compute stream.
    // (With two sets image i+1 had to wait for image i-1's refinement, which
    // the screen kernel -- holding every SM -- pushes behind itself.)
    std::vector<ea_field*>* sets[kBatchSets] = {&lv->fields, &lv->fields2, &lv->fields3};
    DevBuf* images_b[kBatchSets] = {&lv->image, &lv->image2, &lv->image3};
    const int top = L - 1;
    const ea_pose_grid tg = top_grid_of(cfg);
    const ea_grid_counts gc = counts_of(tg);
    std::vector<TopLaunch> launches;
    launches.reserve(count);
    sync(ctx);
    cudaStream_t main_stream = ctx->stream;
    for (int i = 0; i < count; ++i) {
        const int b = i % kBatchSets;  // working set + refinement state
        const int rb = i & 1;          // level-0 upload buffer
        // copy stream: wait until image i-2 released buffer rb, then H2D image i
        if (i >= 2) EAB_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->bev[2 + rb], 0));
        EAB_CUDA(cudaMemcpyAsync(raw[rb], images[i], img_bytes, cudaMemcpyHostToDevice,
                                 ctx->copy_stream));
        EAB_CUDA(cudaEventRecord(ctx->bev[rb], ctx->copy_stream));
        // compute stream: set b is free once image i-3's refinement is done
        EAB_CUDA(cudaStreamWaitEvent(main_stream, ctx->bev[rb], 0));
        if (i >= kBatchSets) EAB_CUDA(cudaStreamWaitEvent(main_stream, ctx->rev[kBatchSets + b], 0));
        build_working_into(ctx, *sets[b], *images_b[b], raw[rb], w, h, L);
        EAB_CUDA(cudaEventRecord(ctx->bev[2 + rb], main_stream));
        ea_levels view;  // template side + working set b (not owned)
        view.models = lv->models;
        view.fields = *sets[b];
        struct Release {
            ea_levels& v;
            ~Release() {
                v.models.clear();
                v.fields.clear();
            }
        } release{view};
        check_search_config(&view, cfg);
        ea_outcome* d_out = (ea_outcome*)(dres + slot * i);
        SearchCtrl* d_ctrl = (SearchCtrl*)(dres + slot * i + sizeof(ea_outcome));
        // top level + seeds on the compute stream
        const TopLaunch t = top_enqueue(ctx, view.models[top], view.fields[top], tg,
                                        cfg.score_params, cfg.topk, 0, 0, cap);
        RefineState st = refine_state(ctx, cfg.topk, b);
        st.out = d_out;
        EAB_CUDA(cudaMemsetAsync(st.out, 0, sizeof(ea_outcome), main_stream));
        launch_seed_beam(ctx, t.top_score, t.top_index, &ctx->ctrl.as<SearchCtrl>()->n_out,
                         seed_args(tg, gc, cfg), st.beam[0], st.cnt[0], st.out);
        EAB_CUDA(cudaMemcpyAsync(d_ctrl, ctx->ctrl.p, sizeof(SearchCtrl),
                                 cudaMemcpyDeviceToDevice, main_stream));
        EAB_CUDA(cudaEventRecord(ctx->rev[b], main_stream));
        launches.push_back(t);
        // refinement levels + D2H of the outcome on the refine stream
        EAB_CUDA(cudaStreamWaitEvent(ctx->refine_stream, ctx->rev[b], 0));
        ctx->stream = ctx->refine_stream;
        try {
            if (top > 0) refine_enqueue(ctx, &view, cfg, tg, tables, st);
            d2h(ctx, hres + slot * i, dres + slot * i, slot);
        } catch (...) {
            ctx->stream = main_stream;
            throw;
        }
        ctx->stream = main_stream;
        EAB_CUDA(cudaEventRecord(ctx->rev[kBatchSets + b], ctx->refine_stream));
    }
    sync(ctx);
    EAB_CUDA(cudaStreamSynchronize(ctx->refine_stream));
    EAB_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    const int last = (count - 1) % kBatchSets;  // keep "the working side is the last image's"
    if (last > 0) {
        std::swap(lv->fields, *sets[last]);
        std::swap(lv->image.p, images_b[last]->p);
        std::swap(lv->image.cap, images_b[last]->cap);
    }
    for (int i = 0; i < count; ++i) {
        SearchCtrl hc;
        std::memcpy(&hc, hres + slot * i + sizeof(ea_outcome), sizeof hc);
        if (top_stats(ctx, launches[i], hc)) {
            std::memcpy(outs + i, hres + slot * i, sizeof(ea_outcome));
        } else {  // overflowed the candidate buffer: redo this image alone
            set_working_image(ctx, lv, images[i], w, h, L);
            search_levels_device(ctx, lv, cfg, outs + i);
        }
    }
}

// Multi-model detect: the working pyramid is built once (into models[0]),
// then every model's search_levels is enqueued against it with its own
// outcome slot; one sync.  A model whose candidate band overflowed the
// buffer is redone alone (search_levels_device grows the buffer).
void detect_multi(ea_ctx* ctx, ea_levels* const* models, int n, const double* image, int w,
                  int h, const ea_search_config& cfg, ea_outcome* outs) {
    const int L = cfg.num_levels;
    for (int i = 0; i < n; ++i) {
        need(models[i], "models[i]");
        if ((int)models[i]->models.size() < L)
            fail(EA_ERR_INVALID_ARGUMENT, "prepared levels of model " + std::to_string(i) +
                                              " do not cover num_levels");
    }
    if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
    ea_levels* work = models[0];
    set_working_image(ctx, work, image, w, h, L);
    if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
    // a view = model i's template side + the shared working side (not owned)
    struct View {
        ea_levels lv;
        ~View() {
            lv.models.clear();
            lv.fields.clear();
        }
    };
    std::vector<View> views(n);
    for (int i = 0; i < n; ++i) {
        views[i].lv.models = models[i]->models;
        views[i].lv.fields = work->fields;
        check_search_config(&views[i].lv, cfg);
    }
    const double* tables = detect_tables(ctx, cfg);
    if (L > 1 && !tables) {  // host-assisted refinement: one by one
        for (int i = 0; i < n; ++i) search_levels_device(ctx, &views[i].lv, cfg, outs + i);
        return;
    }
    const size_t slot = sizeof(ea_outcome) + sizeof(SearchCtrl);
    char* dres = (char*)ctx->rslots.ensure(slot * (size_t)n);
    char* hres = (char*)ctx->h_out.ensure(slot * (size_t)n);
    const unsigned long long cap = std::max<unsigned long long>(initial_cap(ctx), 1ull << 20);
    std::vector<TopLaunch> launches;
    launches.reserve(n);
    for (int i = 0; i < n; ++i) {
        ea_outcome* d_out = (ea_outcome*)(dres + slot * i);
        SearchCtrl* d_ctrl = (SearchCtrl*)(dres + slot * i + sizeof(ea_outcome));
        launches.push_back(enqueue_levels(ctx, &views[i].lv, cfg, tables, cap, d_out, d_ctrl));
        d2h(ctx, hres + slot * i, dres + slot * i, slot);
    }
    if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[7], ctx->stream));
    sync(ctx);
    if (ctx->timing) {
        float ms = 0.f;
        EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[4], ctx->ev[5]));
        ctx->stats.image_ms = ms;
        EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[5], ctx->ev[7]));
        ctx->stats.top_ms = ms;  // all models' search_levels
        ctx->stats.refine_ms = 0.0;
    }
    std::vector<int> redo;
    for (int i = 0; i < n; ++i) {
        SearchCtrl hc;
        std::memcpy(&hc, hres + slot * i + sizeof(ea_outcome), sizeof hc);
        if (top_stats(ctx, launches[i], hc))
            std::memcpy(outs + i, hres + slot * i, sizeof(ea_outcome));
        else
            redo.push_back(i);
    }
    for (int i : redo) search_levels_device(ctx, &views[i].lv, cfg, outs + i);
}

// Template side of prepare_levels (search.cpp:222-234) for one level.
// extract_edge_model (edge_model.cpp:53-149) on a device field: peak, NMS,
// hysteresis and emission on the device (model_kernels.cu); pixels whose
// orientation bin needs glibc's atan2 are decided here with the reference's
// formula.  th == nullptr: default_thresholds (edge_model.cpp:17-24).
ea_model* extract_model_device(ea_ctx* ctx, const ea_field* f, const ea_edge_thresholds* th,
                               int level) {
    if (th && (th->low < 0.0 || th->low > th->high))
        fail(EA_ERR_INVALID_ARGUMENT, "edge thresholds need 0 <= low <= high");
    const int w = f->width, h = f->height;
    const size_t total = (size_t)w * h;
    const size_t head = 128;
    char* buf = (char*)ctx->mscratch.ensure(head + total * (sizeof(ea_edge_point) + 6));
    ModelScratch* ms = (ModelScratch*)buf;
    ea_edge_point* pts = (ea_edge_point*)(buf + head);
    int* amb = (int*)(buf + head + total * sizeof(ea_edge_point));
    unsigned char* state = (unsigned char*)(amb + total);
    unsigned char* kept = state + total;
    ModelScratch* hs = (ModelScratch*)ctx->h_out.ensure(sizeof(ModelScratch));
    std::memset(hs, 0, sizeof *hs);
    hs->use_default = th ? 0 : 1;
    if (th) {
        hs->low = th->low;
        hs->high = th->high;
    }
    h2d(ctx, ms, hs, sizeof *hs);
    launch_magmax(ctx, f->mag(), total, ms);
    launch_nms(ctx, f->gx(), f->gy(), f->mag(), w, h, ms, state, kept, amb);
    d2h(ctx, hs, ms, sizeof *hs);
    sync(ctx);
    if (hs->n_amb > 0) {  // bins on the host, with the reference's atan2 formula
        const int na = hs->n_amb;
        std::vector<double> g(3 * total);
        std::vector<int> list(na);
        std::vector<unsigned char> st(total), kp(total);
        d2h(ctx, g.data(), f->g.p, g.size() * sizeof(double));
        d2h(ctx, list.data(), amb, sizeof(int) * (size_t)na);
        d2h(ctx, st.data(), state, total);
        d2h(ctx, kp.data(), kept, total);
        sync(ctx);
        const double* gx = g.data();
        const double* gy = gx + total;
        const double* mag = gy + total;
        for (const int o : list) {
            const unsigned char v = host_nms_state(gx, gy, mag, w, o % w, o / w, hs->low, hs->high);
            st[o] = v;
            kp[o] = v == 2;
        }
        h2d_staged(ctx, state, st.data(), total);
        h2d_staged(ctx, kept, kp.data(), total);
    }
    launch_hysteresis_emit(ctx, f->gx(), f->gy(), f->mag(), state, kept, w, h, ms, pts);
    d2h(ctx, hs, ms, sizeof *hs);
    sync(ctx);
    const int n = hs->n_kept;
    if (n == 0) {
        double peak;
        std::memcpy(&peak, &hs->peak_bits, sizeof peak);
        char msg[128];
        std::snprintf(msg, sizeof msg,
                      "edge extraction produced an empty model (max gradient magnitude %f)", peak);
        fail(EA_ERR_EMPTY_MODEL, msg, peak);
    }
    std::vector<ea_edge_point> host(n);
    const double cx = hs->cx, cy = hs->cy;
    d2h(ctx, host.data(), pts, sizeof(ea_edge_point) * (size_t)n);
    sync(ctx);
    return new_model(ctx, host.data(), n, cx, cy, level);
}

// Template side of prepare_levels (search.cpp:222-234) for one level.
ea_model* template_model(ea_ctx* ctx, const double* d_img, int w, int h,
                         const ea_search_config& cfg, int level) {
    ea_field* tf = new_field(w, h);
    try {
        sobel_into(ctx, d_img, w, h, tf);
        ea_model* m = extract_model_device(ctx, tf, cfg.has_thresholds ? &cfg.thresholds : nullptr,
                                           level);
        delete tf;
        return m;
    } catch (const Failure& e) {
        delete tf;
        if (e.code == EA_ERR_EMPTY_MODEL) {
            fail(EA_ERR_EMPTY_MODEL,
                 "edge model extraction failed at pyramid level " + std::to_string(level) + ": " +
                     e.what(),
                 e.value);
        }
        throw;
    } catch (...) {
        delete tf;
        throw;
    }
}

void free_levels(ea_levels* lv) {
    if (!lv) return;
    for (auto* m : lv->models) delete m;
    for (auto* f : lv->fields) delete f;
    for (auto* f : lv->fields2) delete f;
    for (auto* f : lv->fields3) delete f;
    delete lv->shard_top;
    delete lv;
}

// Working side from a level-0 image already on the device: pyramid levels
// 1.. into lv->image, Sobel field per level (gradient.cpp:12-27).
void build_working_into(ea_ctx* ctx, std::vector<ea_field*>& fields, DevBuf& image,
                        const double* d_level0, int w, int h, int levels) {
    if (w < 1 || h < 1) {
        fail(EA_ERR_SIZE, "image dimensions must be at least 1x1, got " + std::to_string(w) + "x" +
                              std::to_string(h));
    }
    const size_t elems = pyramid_elems(w / 2, h / 2, std::max(levels - 1, 1));
    double* d = (double*)image.ensure(sizeof(double) * (elems ? elems : 1));
    // Fused when the image is small enough that its ~1/2 wave of tiles is
    // latency- rather than bandwidth-bound (cfg2 1.3 MP: 24 vs ~30 us); a 5 MP
    // image streams better through the per-level kernels (70 vs ~35 us).
    if (levels >= 1 && levels <= kMaxFusedLevels && w >= 3 && h >= 3 &&
        (size_t)w * h <= ((size_t)1 << 21) && levels <= pyramid_levels_feasible(w, h)) {
        // one launch for the whole pyramid + every level's gradient field
        PyramidFieldsArgs pa{};
        pa.img0 = d_level0;
        pa.levels = levels;
        double* dst = d;
        int lw = w, lh = h;
        for (int l = 0; l < levels; ++l) {
            if (l > 0) {
                pa.img[l] = dst;
                dst += (size_t)lw * lh;
            }
            pa.w[l] = lw;
            pa.h[l] = lh;
            if (l < (int)fields.size() && (fields[l]->width != lw || fields[l]->height != lh)) {
                delete fields[l];
                fields[l] = nullptr;
            }
            if (l >= (int)fields.size()) fields.push_back(nullptr);
            if (!fields[l]) fields[l] = new_field(lw, lh);
            pa.gx[l] = fields[l]->gx();
            pa.gy[l] = fields[l]->gy();
            pa.mag[l] = fields[l]->mag();
            lw /= 2;
            lh /= 2;
        }
        const bool small = pa.w[levels - 1] < 3 || pa.h[levels - 1] < 3;
        if (!small && launch_pyramid_fields(ctx, pa)) {
            for (int l = 0; l < levels; ++l) {
                fields[l]->version = next_field_version();
                fields[l]->ring_max = 0.0;  // Sobel leaves the border ring at exactly 0
            }
            while ((int)fields.size() > levels) {
                delete fields.back();
                fields.pop_back();
            }
            return;
        }
    }
    std::vector<const double*> srcs;
    std::vector<int> dims;
    device_pyramid_from(ctx, d_level0, d, w, h, levels, &srcs, &dims);
    for (int l = 0; l < levels; ++l) {  // reuse field objects when dims match
        const int lw = dims[2 * l], lh = dims[2 * l + 1];
        if (l < (int)fields.size() && (fields[l]->width != lw || fields[l]->height != lh)) {
            delete fields[l];
            fields[l] = nullptr;
        }
        if (l >= (int)fields.size()) fields.push_back(nullptr);
        if (!fields[l]) fields[l] = new_field(lw, lh);
        sobel_into(ctx, srcs[l], lw, lh, fields[l]);
    }
    while ((int)fields.size() > levels) {
        delete fields.back();
        fields.pop_back();
    }
}

void build_working(ea_ctx* ctx, ea_levels* lv, const double* d_level0, int w, int h,
                   int levels) {
    build_working_into(ctx, lv->fields, lv->image, d_level0, w, h, levels);
}

void set_working_image(ea_ctx* ctx, ea_levels* lv, const double* image, int w, int h,
                       int levels) {
    if (w < 1 || h < 1) {
        fail(EA_ERR_SIZE, "image dimensions must be at least 1x1, got " + std::to_string(w) + "x" +
                              std::to_string(h));
    }
    double* raw = (double*)lv->raw[0].ensure(sizeof(double) * (size_t)w * h);
    h2d_staged(ctx, raw, image, sizeof(double) * (size_t)w * h);
    build_working(ctx, lv, raw, w, h, levels);
}

// ---- theta-sharded search (search.cpp:116-139) ------------------
static_assert(sizeof(ncclUniqueId) == EA_COMM_ID_BYTES, "ea_comm_id must hold an ncclUniqueId");

ncclComm_t comm_of(const ea_ctx* ctx) {
    if (!ctx->comm)
        fail(EA_ERR_INVALID_ARGUMENT, "context has no communicator (call ea_comm_init first)");
    return static_cast<ncclComm_t>(ctx->comm);
}

void theta_slab_of(uint64_t nt, int rank, int world, uint64_t* b, uint64_t* e) {
    // search.cpp:116-120: worker w scans [total*w/W, total*(w+1)/W)
    *b = (uint64_t)((unsigned __int128)nt * (unsigned)rank / (unsigned)world);
    *e = (uint64_t)((unsigned __int128)nt * (unsigned)(rank + 1) / (unsigned)world);
}

// Sub-buffers of ctx->shard for k rows on `world` ranks.
struct ShardBufs {
    double* local;      // k rows of this rank's slab
    double* gathered;   // world * k rows
    double* merged;     // k rows
    ea_outcome* out;    // device outcome (broadcast from the root)
    int* flag;          // this rank's overflow flag
};

ShardBufs shard_bufs(ea_ctx* ctx, int k) {
    const size_t row = 5 * sizeof(double) * (size_t)k;
    const size_t out_off = (row * (2 + (size_t)ctx->comm_world) + 255) & ~(size_t)255;
    char* p = (char*)ctx->shard.ensure(out_off + sizeof(ea_outcome) + 256);
    ShardBufs b;
    b.local = (double*)p;
    b.merged = (double*)(p + row);
    b.gathered = (double*)(p + 2 * row);
    b.out = (ea_outcome*)(p + out_off);
    b.flag = (int*)(p + out_off + sizeof(ea_outcome));
    return b;
}

// All-gather of every rank's k rows + the `better` merge into d_merged; with
// seed_topk the merged top k also lands in ctx->topk / ctrl->n_out (the
// layout the seed kernel reads).  Enqueued on the context's stream.
void gather_rows(ea_ctx* ctx, const double* d_local, int k, double* d_merged, bool seed_topk) {
    ncclComm_t comm = comm_of(ctx);
    const int n = ctx->comm_world * k;
    if (n > merge_rows_max(ctx))
        fail(EA_ERR_INVALID_ARGUMENT, "world * topk exceeds " + std::to_string(merge_rows_max(ctx)) +
                                          " rows (merge staged in shared memory)");
    const ShardBufs b = shard_bufs(ctx, k);
    EAB_NCCL(nccl().AllGather(d_local, b.gathered, 5 * (size_t)k, ncclDouble, comm, ctx->stream));
    double* ts = nullptr;
    unsigned long long* ti = nullptr;
    int* nt = nullptr;
    if (seed_topk) {
        ts = (double*)ctx->topk.ensure((sizeof(double) + sizeof(unsigned long long)) * (size_t)k);
        ti = reinterpret_cast<unsigned long long*>(ts + k);
        nt = &((SearchCtrl*)ctx->ctrl.ensure(sizeof(SearchCtrl)))->n_out;
    }
    launch_merge_rows(ctx, b.gathered, n, k, d_merged, ts, ti, nt);
}

// One rank's slab of the top level -> k device rows (NaN rows past the
// count; row 0 = +inf on overflow).
void slab_rows(ea_ctx* ctx, const ea_model* m, const ea_field* f, const ea_pose_grid& tg,
               const ea_score_params& p, int k, uint64_t it_begin, uint64_t it_end,
               double* d_rows, int* flag) {
    validate_params(p);
    if (m->n == 0) fail(EA_ERR_INVALID_ARGUMENT, "search needs a nonempty model");
    if (k < 1) fail(EA_ERR_INVALID_ARGUMENT, "topk must be >= 1");
    const ea_grid_counts c = counts_of(tg);
    const uint64_t b = std::min(it_begin, c.nt), e = std::min(it_end, c.nt);
    const uint64_t poses = e > b ? c.nx * c.ny * (e - b) : 0;
    if (poses > kChunkPoses) {  // theta chunks, rows merged on the device
        const auto chunks = theta_chunks(c, b, e);
        const int n = (int)chunks.size() * k;
        if (n > merge_rows_max(ctx))
            fail(EA_ERR_INVALID_ARGUMENT, "pose grid too large for the chunk merge");
        double* tmp = (double*)ctx->chunk_rows.ensure(5 * sizeof(double) * (size_t)n);
        for (size_t i = 0; i < chunks.size(); ++i) {
            const uint64_t cp = c.nx * c.ny * (chunks[i].second - chunks[i].first);
            top_enqueue(ctx, m, f, tg, p, k, chunks[i].first, chunks[i].second, async_cap(ctx, cp),
                        tmp + 5 * (size_t)k * i, flag);
        }
        launch_merge_rows(ctx, tmp, n, k, d_rows);
        return;
    }
    const unsigned long long cap = async_cap(ctx, poses);
    if (poses > 0) {
        top_enqueue(ctx, m, f, tg, p, k, b, e, cap, d_rows, flag);
        return;
    }
    // empty slab (more ranks than thetas): k empty rows from a cleared
    // control block (never the previous search's count)
    SearchCtrl* ctrl = (SearchCtrl*)ctx->ctrl.ensure(sizeof(SearchCtrl));
    double* ts = (double*)ctx->topk.ensure((sizeof(double) + sizeof(unsigned long long)) * (size_t)k);
    EAB_CUDA(cudaMemsetAsync(ctrl, 0, sizeof(SearchCtrl), ctx->stream));
    const RowGrid g{tg.x0, tg.dx, tg.y0, tg.dy, tg.t0, tg.dt, c.nx, c.ny};
    launch_topk_rows(ctx, ts, reinterpret_cast<unsigned long long*>(ts + k), ctrl, cap, k, g,
                     d_rows, flag);
    ctx->hist_clean = false;  // the control block was cleared, not left by a finish
}

// search_levels sharded by theta (every rank calls it with its top-level
// field `ftop`): slab -> all-gather -> merge -> root refines -> outcome
// broadcast.  Root = rank 0.
void search_levels_sharded(ea_ctx* ctx, const ea_levels* lv, const ea_field* ftop,
                           const ea_search_config& cfg, ea_outcome* out) {
    ncclComm_t comm = comm_of(ctx);
    const int top = cfg.num_levels - 1, k = cfg.topk;
    const bool root = ctx->comm_rank == 0;
    const ea_pose_grid tg = top_grid_of(cfg);
    const ea_grid_counts c = counts_of(tg);
    const double* tables = root ? detect_tables(ctx, cfg) : nullptr;
    uint64_t b = 0, e = 0;
    theta_slab_of(c.nt, ctx->comm_rank, ctx->comm_world, &b, &e);
    ShardBufs sb = shard_bufs(ctx, k);
    EAB_CUDA(cudaMemsetAsync(sb.flag, 0, sizeof(int), ctx->stream));
    slab_rows(ctx, lv->models[top], ftop, tg, cfg.score_params, k, b, e, sb.local, sb.flag);
    gather_rows(ctx, sb.local, k, sb.merged, /*seed_topk=*/true);
    sb = shard_bufs(ctx, k);
    if (root) {
        SearchCtrl* ctrl = ctx->ctrl.as<SearchCtrl>();
        const double* ts = ctx->topk.as<double>();
        const unsigned long long* ti = reinterpret_cast<const unsigned long long*>(ts + k);
        if (top == 0 || tables) {  // device beam, as enqueue_levels
            RefineState st = refine_state(ctx, k);
            st.out = sb.out;
            EAB_CUDA(cudaMemsetAsync(st.out, 0, sizeof(ea_outcome), ctx->stream));
            launch_seed_beam(ctx, ts, ti, &ctrl->n_out, seed_args(tg, c, cfg), st.beam[0],
                             st.cnt[0], st.out);
            if (top > 0) refine_enqueue(ctx, lv, cfg, tg, tables, st);
        } else {  // very wide beams: host-assisted refinement from the merged rows
            std::vector<double> rows(5 * (size_t)k);
            d2h(ctx, rows.data(), sb.merged, rows.size() * sizeof(double));
            sync(ctx);
            std::vector<ea_scored_pose> seeds;
            for (int r = 0; r < k; ++r) {
                const double* q = rows.data() + 5 * (size_t)r;
                if (q[0] != q[0]) break;
                if (std::isinf(q[0])) fail(EA_ERR_INTERNAL, "candidate buffer overflow in a sharded search");
                seeds.push_back(ea_scored_pose{q[0], (uint64_t)q[1], ea_pose{q[2], q[3], q[4]}});
            }
            ea_outcome ho{};
            refine_levels(ctx, lv, cfg, tg, seeds_to_beam(seeds), &ho);
            h2d_staged(ctx, sb.out, &ho, sizeof ho);
        }
    }
    EAB_NCCL(nccl().Broadcast(sb.out, sb.out, sizeof(ea_outcome), ncclUint8, 0, comm, ctx->stream));
    char* h = (char*)ctx->h_out.ensure(sizeof(ea_outcome) + 5 * sizeof(double));
    d2h(ctx, h, sb.out, sizeof(ea_outcome));
    d2h(ctx, h + sizeof(ea_outcome), sb.merged, 5 * sizeof(double));
    sync(ctx);
    double row0;
    std::memcpy(&row0, h + sizeof(ea_outcome), sizeof row0);
    if (std::isinf(row0)) fail(EA_ERR_INTERNAL, "candidate buffer overflow in a sharded search");
    std::memcpy(out, h, sizeof(ea_outcome));
}


// ---- multi-model sharding ----------------------------------------
// (model, theta slab) work items, costed in pose-evals; see ea_plan_multi in
// the header.  Deterministic (every rank computes the same plan).
// LPT assignment of the slabs of `s[m]` per model (theta block partition,
// search.cpp:116-120): longest first, to the least loaded rank holding no
// other slab of that model; ties broken by model, slab, rank -- a total
// order, so every rank computes the same plan.  Returns the makespan.
double assign_lpt(const std::vector<double>& cost, const uint64_t* thetas,
                  const std::vector<uint64_t>& s, int world, double fixed_evals,
                  std::vector<ea_work_item>* out) {
    const int n_models = (int)cost.size();
    std::vector<ea_work_item> items;
    for (int m = 0; m < n_models; ++m) {
        for (uint64_t j = 0; j < s[m]; ++j) {
            ea_work_item it{};
            it.rank = -1;
            it.model = m;
            theta_slab_of(thetas[m], (int)j, (int)s[m], &it.it_begin, &it.it_end);
            it.cost = cost[m] * (double)(it.it_end - it.it_begin) / (double)thetas[m] + fixed_evals;
            items.push_back(it);
        }
    }
    std::stable_sort(items.begin(), items.end(), [](const ea_work_item& x, const ea_work_item& y) {
        if (x.cost != y.cost) return x.cost > y.cost;
        if (x.model != y.model) return x.model < y.model;
        return x.it_begin < y.it_begin;
    });
    std::vector<double> load(world, 0.0);
    std::vector<std::vector<char>> holds(world, std::vector<char>(n_models, 0));
    for (ea_work_item& it : items) {
        int best = -1;
        for (int r = 0; r < world; ++r) {
            if (holds[r][it.model]) continue;  // one slab of a model per rank
            if (best < 0 || load[r] < load[best]) best = r;
        }
        it.rank = best;
        load[best] += it.cost;
        holds[best][it.model] = 1;
    }
    std::stable_sort(items.begin(), items.end(), [](const ea_work_item& x, const ea_work_item& y) {
        if (x.rank != y.rank) return x.rank < y.rank;
        if (x.model != y.model) return x.model < y.model;
        return x.it_begin < y.it_begin;
    });
    *out = std::move(items);
    return *std::max_element(load.begin(), load.end());
}

// The plan with the smallest makespan among slab sizes of about 1/d of a
// rank's share (d = 1, 2, 3, 4, 6, 8) and every model cut into `world`
// slabs: coarse slabs pay fewer fixed costs, fine slabs pack better.
std::vector<ea_work_item> plan_multi(const uint64_t* plane_poses, const uint64_t* thetas,
                                     const int* n_top, int n_models, int world,
                                     double fixed_evals) {
    if (n_models < 0 || world < 1) fail(EA_ERR_INVALID_ARGUMENT, "need n_models >= 0, world >= 1");
    double total = 0.0;
    std::vector<double> cost(n_models);
    for (int m = 0; m < n_models; ++m) {
        if (n_top[m] < 0) fail(EA_ERR_INVALID_ARGUMENT, "n_top must be >= 0");
        cost[m] = (thetas[m] == 0 || plane_poses[m] == 0)
                      ? 0.0
                      : (double)plane_poses[m] * (double)thetas[m] * (double)n_top[m];
        total += cost[m];
    }
    const double share = total / world;
    std::vector<ea_work_item> best;
    double best_span = 0.0;
    for (int d : {1, 2, 3, 4, 6, 8, 0}) {  // 0: every model in `world` slabs
        std::vector<uint64_t> s(n_models, 0);
        for (int m = 0; m < n_models; ++m) {
            if (thetas[m] == 0 || plane_poses[m] == 0) continue;
            uint64_t q = d == 0 ? (uint64_t)world
                         : share > 0.0 ? (uint64_t)std::ceil(cost[m] * d / share - 1e-9) : 1;
            s[m] = std::max<uint64_t>(1, std::min<uint64_t>({q, (uint64_t)world, thetas[m]}));
        }
        std::vector<ea_work_item> items;
        const double span = assign_lpt(cost, thetas, s, world, fixed_evals, &items);
        if (best.empty() || span < best_span * (1 - 1e-12)) {
            best = std::move(items);
            best_span = span;
        }
    }
    return best;
}

// Per-search overhead of one slab search in pose-evals (the finish and the
// launch boundaries, ~30 us at ~2.2e12 pose-evals/s on B200).
constexpr double kSearchFixedEvals = 6.6e7;

void detect_multi_sharded(ea_ctx* ctx, ea_levels* const* models, int n, const double* image,
                          int w, int h, const ea_search_config& cfg, ea_outcome* outs) {
    ncclComm_t comm = comm_of(ctx);
    const bool root = ctx->comm_rank == 0;
    const int L = cfg.num_levels, top = L - 1, k = cfg.topk, world = ctx->comm_world;
    for (int i = 0; i < n; ++i) {
        need(models[i], "models[i]");
        if ((int)models[i]->models.size() < L)
            fail(EA_ERR_INVALID_ARGUMENT, "prepared levels of model " + std::to_string(i) +
                                              " do not cover num_levels");
    }
    if (L < 1 || L > EA_MAX_LEVELS) fail(EA_ERR_INVALID_ARGUMENT, "num_levels out of range");
    validate_params(cfg.score_params);
    if (k < 1 || cfg.refine_radius < 1)
        fail(EA_ERR_INVALID_ARGUMENT, "topk and refine_radius must be >= 1");
    if (w < 1 || h < 1) {
        fail(EA_ERR_SIZE, "image dimensions must be at least 1x1, got " + std::to_string(w) + "x" +
                              std::to_string(h));
    }
    if (L > pyramid_levels_feasible(w, h)) {
        fail(EA_ERR_SIZE, "pyramid of " + std::to_string(L) +
                              " levels would drop below 8x8; maximum feasible level count is " +
                              std::to_string(pyramid_levels_feasible(w, h)));
    }
    if (world * k > merge_rows_max(ctx))
        fail(EA_ERR_INVALID_ARGUMENT, "world * topk exceeds the merge's shared memory");
    ea_levels* work = models[0];
    const int wt = w >> top, ht = h >> top;
    ea_field* ftop = nullptr;
    if (root) {
        set_working_image(ctx, work, image, w, h, L);
        ftop = work->fields[top];
    } else {
        if (work->shard_top && (work->shard_top->width != wt || work->shard_top->height != ht)) {
            delete work->shard_top;
            work->shard_top = nullptr;
        }
        if (!work->shard_top) work->shard_top = new_field(wt, ht);
        ftop = work->shard_top;
    }
    EAB_NCCL(nccl().Broadcast(ftop->g.p, ftop->g.p, 3 * (size_t)wt * ht, ncclDouble, 0, comm,
                              ctx->stream));
    if (!root) {
        ftop->version = next_field_version();
        ftop->ring_max = 0.0;
    }
    // the plan (same on every rank)
    const ea_pose_grid tg = top_grid_of(cfg);
    const ea_grid_counts c = counts_of(tg);
    std::vector<uint64_t> planes(n, c.nx * c.ny), thetas(n, c.nt);
    std::vector<int> ntop(n);
    for (int i = 0; i < n; ++i) ntop[i] = models[i]->models[top]->n;
    const std::vector<ea_work_item> items =
        plan_multi(planes.data(), thetas.data(), ntop.data(), n, world, kSearchFixedEvals);
    // buffers: local rows [n][k], gathered [world][n][k], merged [n][k], seeds, outcomes
    const size_t rows_b = 5 * sizeof(double) * (size_t)n * k;
    const size_t seeds_b = (sizeof(double) + sizeof(unsigned long long)) * (size_t)n * k;
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        const size_t o = off;
        off = (off + bytes + 255) & ~(size_t)255;
        return o;
    };
    const size_t o_local = carve(rows_b), o_gath = carve(rows_b * world), o_merged = carve(rows_b),
                 o_score = carve(seeds_b), o_cnt = carve(sizeof(int) * n),
                 o_out = carve(sizeof(ea_outcome) * n), o_flag = carve(sizeof(int));
    char* base = (char*)ctx->shard.ensure(off);
    double* local = (double*)(base + o_local);
    double* gathered = (double*)(base + o_gath);
    double* merged = (double*)(base + o_merged);
    double* tscore = (double*)(base + o_score);
    unsigned long long* tindex = reinterpret_cast<unsigned long long*>(tscore + (size_t)n * k);
    int* tcount = (int*)(base + o_cnt);
    ea_outcome* d_outs = (ea_outcome*)(base + o_out);
    int* flag = (int*)(base + o_flag);
    // NaN rows for the models this rank has no slab of (0xff.. is a NaN)
    EAB_CUDA(cudaMemsetAsync(local, 0xff, rows_b, ctx->stream));
    EAB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    for (const ea_work_item& it : items) {
        if (it.rank != ctx->comm_rank) continue;
        slab_rows(ctx, models[it.model]->models[top], ftop, tg, cfg.score_params, k, it.it_begin,
                  it.it_end, local + 5 * (size_t)it.model * k, flag);
    }
    EAB_NCCL(nccl().AllGather(local, gathered, 5 * (size_t)n * k, ncclDouble, comm, ctx->stream));
    launch_merge_rows_multi(ctx, gathered, world, n, k, merged, tscore, tindex, tcount);
    if (root) {
        struct View {
            ea_levels lv;
            ~View() {
                lv.models.clear();
                lv.fields.clear();
            }
        };
        const double* tables = detect_tables(ctx, cfg);
        EAB_CUDA(cudaMemsetAsync(d_outs, 0, sizeof(ea_outcome) * n, ctx->stream));
        std::vector<double> hrows;
        if (top > 0 && !tables) {  // very wide beams: host-assisted refinement
            hrows.resize(5 * (size_t)n * k);
            d2h(ctx, hrows.data(), merged, rows_b);
            sync(ctx);
        }
        for (int i = 0; i < n; ++i) {
            View v;
            v.lv.models = models[i]->models;
            v.lv.fields = work->fields;
            if (top == 0 || tables) {
                RefineState st = refine_state(ctx, k);
                st.out = d_outs + i;
                launch_seed_beam(ctx, tscore + (size_t)i * k, tindex + (size_t)i * k, tcount + i,
                                 seed_args(tg, c, cfg), st.beam[0], st.cnt[0], st.out);
                if (top > 0) refine_enqueue(ctx, &v.lv, cfg, tg, tables, st);
            } else {
                std::vector<ea_scored_pose> seeds;
                for (int r = 0; r < k; ++r) {
                    const double* q = hrows.data() + 5 * ((size_t)i * k + r);
                    if (q[0] != q[0]) break;
                    if (std::isinf(q[0]))
                        fail(EA_ERR_INTERNAL, "candidate buffer overflow in a sharded search");
                    seeds.push_back(ea_scored_pose{q[0], (uint64_t)q[1], ea_pose{q[2], q[3], q[4]}});
                }
                ea_outcome ho{};
                refine_levels(ctx, &v.lv, cfg, tg, seeds_to_beam(seeds), &ho);
                h2d_staged(ctx, d_outs + i, &ho, sizeof ho);
            }
        }
    }
    EAB_NCCL(nccl().Broadcast(d_outs, d_outs, sizeof(ea_outcome) * n, ncclUint8, 0, comm,
                              ctx->stream));
    char* hb = (char*)ctx->h_out.ensure(sizeof(ea_outcome) * n + rows_b);
    d2h(ctx, hb, d_outs, sizeof(ea_outcome) * n);
    d2h(ctx, hb + sizeof(ea_outcome) * n, merged, rows_b);
    sync(ctx);
    for (int i = 0; i < n; ++i) {
        double row0;
        std::memcpy(&row0, hb + sizeof(ea_outcome) * n + 5 * sizeof(double) * (size_t)i * k,
                    sizeof row0);
        if (std::isinf(row0)) fail(EA_ERR_INTERNAL, "candidate buffer overflow in a sharded search");
    }
    std::memcpy(outs, hb, sizeof(ea_outcome) * n);
}

}  // namespace

// =============================================================================
// C-ABI
// =============================================================================
extern "C" {

const char* ea_last_error(void) { return g_err.c_str(); }
double ea_last_error_value(void) { return g_err_value; }

ea_status ea_ctx_create(int device, ea_ctx** out) {
    return guard([&] {
        need(out, "out");
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0) {
            cudaGetLastError();
            fail(EA_ERR_CUDA, std::string("no CUDA device available (") +
                                  (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices") +
                                  "); libedgealign_b200 has no CPU fallback");
        }
        if (device < 0 || device >= n) fail(EA_ERR_INVALID_ARGUMENT, "device index out of range");
        DeviceGuard dg(device);
        cudaDeviceProp prop{};
        EAB_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) {
            fail(EA_ERR_CUDA, std::string("device ") + prop.name +
                                  " is not sm_100 class; this build targets sm_100a only");
        }
        auto* c = new ea_ctx;
        c->device = device;
        c->sm_count = prop.multiProcessorCount;
        // dynamic shared-memory budget of the lattice kernels: the opt-in
        // limit minus their static shared memory (per-warp lists, the plane
        // barrier, merge_hist's chunk sums; checked per kernel at launch by
        // raise_smem_limit -- a 1 KB reserve let a plane near the limit fail)
        c->smem_optin = prop.sharedMemPerBlockOptin - kLatticeStaticSmem;
        cudaError_t se = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (se != cudaSuccess) {
            delete c;
            cuda_check(se, "cudaStreamCreate");
        }
        c->own_stream = true;
        *out = c;
    });
}

void ea_ctx_destroy(ea_ctx* ctx) {
    if (!ctx) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (DevBuf* b : {&ctx->cs, &ctx->rot_exact, &ctx->rot_screen, &ctx->plane, &ctx->map,
                      &ctx->item_max, &ctx->tail,
                      &ctx->hist, &ctx->ctrl, &ctx->cand, &ctx->cand_score, &ctx->topk,
                      &ctx->refine_poses, &ctx->refine_scores, &ctx->beam, &ctx->accum64,
                      &ctx->work, &ctx->ttab, &ctx->rstate, &ctx->rslots, &ctx->mscratch,
                      &ctx->cta_top, &ctx->ztiles, &ctx->chunk_rows})
        b->release();
    ctx->h_stage.release();
    ctx->h_out.release();
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->bev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->rev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->tev)
        if (e) cudaEventDestroy(e);
    if (ctx->comm) {
        try {
            nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
        } catch (...) {
        }
        ctx->comm = nullptr;
    }
    ctx->shard.release();
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->refine_stream) cudaStreamDestroy(ctx->refine_stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    if (prev >= 0) cudaSetDevice(prev);
}

ea_status ea_ctx_set_stream(ea_ctx* ctx, void* stream) {
    return guard([&] {
        need(ctx, "ctx");
        DeviceGuard dg(ctx->device);
        EAB_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->own_stream && stream) {
            cudaStreamDestroy(ctx->stream);
            ctx->own_stream = false;
        }
        if (stream) {
            ctx->stream = (cudaStream_t)stream;
        } else if (!ctx->own_stream) {
            EAB_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        }
    });
}

void* ea_ctx_stream(ea_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

ea_status ea_ctx_synchronize(ea_ctx* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        DeviceGuard dg(ctx->device);
        sync(ctx);
    });
}

ea_status ea_ctx_last_stats(const ea_ctx* ctx, ea_search_stats* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        *out = ctx->stats;
    });
}

ea_status ea_ctx_set_timing(ea_ctx* ctx, int on) {
    return guard([&] {
        need(ctx, "ctx");
        DeviceGuard dg(ctx->device);
        if (on && !ctx->ev[0]) {
            for (auto& e : ctx->ev) EAB_CUDA(cudaEventCreate(&e));
            for (auto& e : ctx->tev) EAB_CUDA(cudaEventCreate(&e));
        }
        ctx->timing = on != 0;
    });
}

uint64_t ea_ctx_kernel_launches(const ea_ctx* ctx) { return ctx ? ctx->launches : 0; }

ea_status ea_host_alloc(size_t bytes, void** out) {
    return guard([&] {
        need(out, "out");
        EAB_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
    });
}
void ea_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

// ---- geometry ----------------------------------------------------------------
ea_status ea_compute_grid_counts(const ea_pose_grid* g, ea_grid_counts* out) {
    return guard([&] {
        need(g, "grid");
        need(out, "out");
        *out = counts_of(*g);
    });
}

ea_status ea_pose_at(const ea_pose_grid* g, uint64_t index, ea_pose* out) {
    return guard([&] {
        need(g, "grid");
        need(out, "out");
        *out = pose_of(*g, counts_of(*g), index);
    });
}

// ---- image -------------------------------------------------------------------
int ea_max_pyramid_levels(int w, int h) { return pyramid_levels_feasible(w, h); }

ea_status ea_pyramid_dims(int w, int h, int levels, int* dims) {
    return guard([&] {
        need(dims, "dims");
        for (int l = 0; l < levels; ++l) {
            dims[2 * l] = w;
            dims[2 * l + 1] = h;
            w /= 2;
            h /= 2;
        }
    });
}

ea_status ea_downsample(ea_ctx* ctx, const double* image, int w, int h, double* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(image, "image");
        need(out, "out");
        if (w < 2 || h < 2) {
            fail(EA_ERR_SIZE, "downsample needs at least 2x2, got " + std::to_string(w) + "x" +
                                  std::to_string(h));
        }
        DeviceGuard dg(ctx->device);
        const size_t in = (size_t)w * h, on = (size_t)(w / 2) * (h / 2);
        double* d = (double*)ctx->work.ensure(sizeof(double) * (in + on));
        h2d_staged(ctx, d, image, sizeof(double) * in);
        launch_downsample(ctx, d, w, h, d + in);
        d2h(ctx, out, d + in, sizeof(double) * on);
        sync(ctx);
    });
}

ea_status ea_build_pyramid(ea_ctx* ctx, const double* image, int w, int h, int levels,
                           double* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(image, "image");
        need(out, "out");
        if (w < 1 || h < 1) {
            fail(EA_ERR_SIZE, "image dimensions must be at least 1x1, got " + std::to_string(w) +
                                  "x" + std::to_string(h));
        }
        DeviceGuard dg(ctx->device);
        if (levels < 1) fail(EA_ERR_INVALID_ARGUMENT, "num_levels must be >= 1");
        const size_t elems = pyramid_elems(w, h, levels);
        double* d = (double*)ctx->work.ensure(sizeof(double) * elems);
        h2d_staged(ctx, d, image, sizeof(double) * (size_t)w * h);
        std::vector<size_t> offs;
        std::vector<int> dims;
        device_pyramid(ctx, d, w, h, levels, &offs, &dims);
        d2h(ctx, out, d, sizeof(double) * elems);
        sync(ctx);
    });
}

ea_status ea_compute_gradients(ea_ctx* ctx, const double* image, int w, int h, double* gx,
                               double* gy, double* mag) {
    return guard([&] {
        need(ctx, "ctx");
        need(image, "image");
        need(gx, "gx");
        need(gy, "gy");
        need(mag, "mag");
        DeviceGuard dg(ctx->device);
        if (w < 3 || h < 3) {
            fail(EA_ERR_SIZE, "compute_gradients needs at least 3x3, got " + std::to_string(w) +
                                  "x" + std::to_string(h));
        }
        const size_t n = (size_t)w * h;
        double* d = (double*)ctx->work.ensure(sizeof(double) * 4 * n);
        h2d_staged(ctx, d, image, sizeof(double) * n);
        launch_sobel(ctx, d, w, h, d + n, d + 2 * n, d + 3 * n);
        d2h(ctx, gx, d + n, sizeof(double) * n);
        d2h(ctx, gy, d + 2 * n, sizeof(double) * n);
        d2h(ctx, mag, d + 3 * n, sizeof(double) * n);
        sync(ctx);
    });
}

ea_status ea_field_upload(ea_ctx* ctx, const double* gx, const double* gy, const double* mag,
                          int w, int h, ea_field** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        need(gx, "gx");
        need(gy, "gy");
        need(mag, "mag");
        if (w < 1 || h < 1) fail(EA_ERR_SIZE, "gradient field must be at least 1x1");
        DeviceGuard dg(ctx->device);
        ea_field* f = new_field(w, h);
        try {
            const size_t n = (size_t)w * h;
            h2d_staged(ctx, f->gx(), gx, sizeof(double) * n);
            h2d_staged(ctx, f->gy(), gy, sizeof(double) * n);
            h2d_staged(ctx, f->mag(), mag, sizeof(double) * n);
            double rm = 0.0;  // largest magnitude on the outer ring
            for (int x = 0; x < w; ++x) {
                rm = std::max(rm, std::max(mag[x], mag[(size_t)(h - 1) * w + x]));
            }
            for (int y = 0; y < h; ++y) {
                rm = std::max(rm, std::max(mag[(size_t)y * w], mag[(size_t)y * w + w - 1]));
            }
            f->ring_max = rm;
            for (size_t i = 0; i < n && std::isfinite(f->ring_max); ++i) {
                if (!std::isfinite(mag[i])) f->ring_max = INFINITY;
            }
            sync(ctx);
        } catch (...) {
            delete f;
            throw;
        }
        *out = f;
    });
}

ea_status ea_field_from_image(ea_ctx* ctx, const double* image, int w, int h, ea_field** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(image, "image");
        need(out, "out");
        DeviceGuard dg(ctx->device);
        if (w < 3 || h < 3) {
            fail(EA_ERR_SIZE, "compute_gradients needs at least 3x3, got " + std::to_string(w) +
                                  "x" + std::to_string(h));
        }
        ea_field* f = new_field(w, h);
        try {
            double* d = (double*)ctx->work.ensure(sizeof(double) * (size_t)w * h);
            h2d_staged(ctx, d, image, sizeof(double) * (size_t)w * h);
            sobel_into(ctx, d, w, h, f);
            sync(ctx);
        } catch (...) {
            delete f;
            throw;
        }
        *out = f;
    });
}

ea_status ea_field_download(ea_ctx* ctx, const ea_field* f, double* gx, double* gy,
                            double* mag) {
    return guard([&] {
        need(ctx, "ctx");
        need(f, "field");
        DeviceGuard dg(ctx->device);
        const size_t n = (size_t)f->width * f->height;
        if (gx) d2h(ctx, gx, f->gx(), sizeof(double) * n);
        if (gy) d2h(ctx, gy, f->gy(), sizeof(double) * n);
        if (mag) d2h(ctx, mag, f->mag(), sizeof(double) * n);
        sync(ctx);
    });
}

ea_status ea_field_dims(const ea_field* f, int* w, int* h) {
    return guard([&] {
        need(f, "field");
        if (w) *w = f->width;
        if (h) *h = f->height;
    });
}

void ea_field_free(ea_field* f) { delete f; }

// ---- template side -------------------------------------------------------------
ea_status ea_default_thresholds(const double* mag, int w, int h, ea_edge_thresholds* out) {
    return guard([&] {
        need(mag, "mag");
        need(out, "out");
        *out = host_default_thresholds(mag, (size_t)w * h);
    });
}

ea_status ea_extract_edge_model(const double* gx, const double* gy, const double* mag, int w,
                                int h, const ea_edge_thresholds* th, int level,
                                ea_edge_point* points, int cap, int* n_out, double* cx,
                                double* cy) {
    (void)level;
    return guard([&] {
        need(gx, "gx");
        need(gy, "gy");
        need(mag, "mag");
        need(th, "thresholds");
        need(n_out, "n_out");
        double ccx = 0, ccy = 0;
        const auto pts = host_extract_edge_model(gx, gy, mag, w, h, *th, &ccx, &ccy);
        *n_out = (int)pts.size();
        if (cx) *cx = ccx;
        if (cy) *cy = ccy;
        if (points) {
            for (int i = 0; i < (int)pts.size() && i < cap; ++i) points[i] = pts[i];
        }
    });
}

ea_status ea_field_extract_model(ea_ctx* ctx, const ea_field* field, const ea_edge_thresholds* th,
                                 int level, ea_model** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(field, "field");
        need(out, "out");
        DeviceGuard dg(ctx->device);
        *out = extract_model_device(ctx, field, th, level);
    });
}

ea_status ea_model_points(const ea_model* m, ea_edge_point* points, int cap, int* n_out,
                          double* cx, double* cy) {
    return guard([&] {
        need(m, "model");
        need(n_out, "n_out");
        *n_out = m->n;
        if (cx) *cx = m->centroid_x;
        if (cy) *cy = m->centroid_y;
        if (points)
            for (int i = 0; i < m->n && i < cap; ++i) points[i] = m->host[i];
    });
}

ea_status ea_model_create(ea_ctx* ctx, const ea_edge_point* points, int n, double cx, double cy,
                          int level, ea_model** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        if (n < 0) fail(EA_ERR_INVALID_ARGUMENT, "model point count must be >= 0");
        if (n > 0) need(points, "points");
        DeviceGuard dg(ctx->device);
        *out = new_model(ctx, points, n, cx, cy, level);
    });
}

int ea_model_size(const ea_model* m) { return m ? m->n : 0; }
void ea_model_free(ea_model* m) { delete m; }

// ---- similarity ------------------------------------------------------------------
ea_status ea_validate_params(const ea_score_params* p) {
    return guard([&] {
        need(p, "params");
        validate_params(*p);
    });
}

ea_status ea_point_vote(ea_ctx* ctx, double dir_x, double dir_y, const ea_field* f, int cx,
                        int cy, const ea_score_params* p, double* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(f, "field");
        need(p, "params");
        need(out, "out");
        validate_params(*p);
        DeviceGuard dg(ctx->device);
        double* sc = (double*)ctx->refine_scores.ensure(sizeof(double) * 2);
        launch_point_vote(ctx, f, cx, cy, (p->neighborhood - 1) / 2, dir_x, dir_y, p->eps_mag,
                          p->polarity == EA_POLARITY_IGNORE, sc);
        d2h(ctx, out, sc, sizeof(double));
        sync(ctx);
    });
}

ea_status ea_rotate_model(ea_ctx* ctx, const ea_model* m, double theta, double* px, double* py,
                          double* dx, double* dy) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "model");
        DeviceGuard dg(ctx->device);
        const int n = m->n;
        if (n == 0) return;
        const double hcs[2] = {std::cos(theta), std::sin(theta)};
        ctx->cs_dev_key.clear();
        double* dcs = (double*)ctx->cs.ensure(sizeof(double) * 2);
        h2d_staged(ctx, dcs, hcs, sizeof hcs);
        double* rot = (double*)ctx->rot_exact.ensure(sizeof(double) * 4 * n);
        launch_rotate(ctx, m->pts.as<double>(), n, dcs, 1, rot, nullptr, nullptr);
        if (px) d2h(ctx, px, rot, sizeof(double) * n);
        if (py) d2h(ctx, py, rot + n, sizeof(double) * n);
        if (dx) d2h(ctx, dx, rot + 2 * n, sizeof(double) * n);
        if (dy) d2h(ctx, dy, rot + 3 * n, sizeof(double) * n);
        sync(ctx);
    });
}

ea_status ea_pose_score(ea_ctx* ctx, const ea_model* m, const ea_pose* pose, const ea_field* f,
                        const ea_score_params* p, double* value, int* n_inbounds) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "model");
        need(pose, "pose");
        need(f, "field");
        need(p, "params");
        validate_params(*p);
        if (m->n == 0) fail(EA_ERR_INVALID_ARGUMENT, "pose_score needs a nonempty model");
        DeviceGuard dg(ctx->device);
        const int n = m->n;
        struct {
            double cs[2];
            double uxuy[2];
            int slot;
        } h{{std::cos(pose->theta), std::sin(pose->theta)}, {pose->ux, pose->uy}, 0};
        char* d = (char*)ctx->work.ensure(sizeof h);
        h2d_staged(ctx, d, &h, sizeof h);
        double* rot = (double*)ctx->rot_exact.ensure(sizeof(double) * 4 * n);
        launch_rotate(ctx, m->pts.as<double>(), n, (const double*)d, 1, rot, nullptr, nullptr);
        double* sc = (double*)ctx->refine_scores.ensure(sizeof(double) + sizeof(int));
        int* inb = (int*)(sc + 1);
        launch_refine_score(ctx, exact_args(f, *p, rot, (size_t)n, n),
                            (const double*)(d + offsetof(decltype(h), uxuy)),
                            (const int*)(d + offsetof(decltype(h), slot)), 1, sc, inb);
        double hv[2];
        d2h(ctx, hv, sc, sizeof(double) + sizeof(int));
        sync(ctx);
        if (value) *value = hv[0];
        if (n_inbounds) std::memcpy(n_inbounds, &hv[1], sizeof(int));
    });
}

// ---- search ---------------------------------------------------------------------------
ea_status ea_search_topk(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                         const ea_pose_grid* g, const ea_score_params* p, int backend_kind,
                         int k, ea_scored_pose* out, int* n_out) {
    (void)backend_kind;
    return guard([&] {
        need(ctx, "ctx");
        need(m, "model");
        need(f, "field");
        need(g, "grid");
        need(p, "params");
        need(n_out, "n_out");
        DeviceGuard dg(ctx->device);
        const auto r = top_search(ctx, m, f, *g, *p, k, 0, 0);
        if (!r.empty()) need(out, "out");
        for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
        *n_out = (int)r.size();
    });
}

ea_status ea_exhaustive_search(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                               const ea_pose_grid* g, const ea_score_params* p,
                               int backend_kind, ea_scored_pose* out) {
    int n = 0;
    return ea_search_topk(ctx, m, f, g, p, backend_kind, 1, out, &n);
}

ea_status ea_search_topk_slab(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                              const ea_pose_grid* g, const ea_score_params* p, int k,
                              uint64_t it_begin, uint64_t it_end, ea_scored_pose* out,
                              int* n_out) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "model");
        need(f, "field");
        need(g, "grid");
        need(p, "params");
        need(n_out, "n_out");
        DeviceGuard dg(ctx->device);
        *n_out = 0;
        const uint64_t nt = counts_of(*g).nt;
        if (std::min(it_end, nt) <= std::min(it_begin, nt)) return;  // empty slab
        const auto r = top_search(ctx, m, f, *g, *p, k, it_begin, it_end);
        for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
        *n_out = (int)r.size();
    });
}

ea_status ea_merge_topk(const ea_scored_pose* in, int n, int k, ea_scored_pose* out,
                        int* n_out) {
    return guard([&] {
        need(n_out, "n_out");
        if (k < 1) fail(EA_ERR_INVALID_ARGUMENT, "topk must be >= 1");
        std::vector<ea_scored_pose> v(in, in + (n > 0 ? n : 0));
        std::sort(v.begin(), v.end(), [](const ea_scored_pose& a, const ea_scored_pose& b) {
            if (a.score != b.score) return a.score > b.score;  // better(), search.cpp:36-41
            return a.grid_index < b.grid_index;
        });
        if ((int)v.size() > k) v.resize(k);
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
        *n_out = (int)v.size();
    });
}

ea_status ea_score_map(ea_ctx* ctx, const ea_model* m, const ea_field* f, const ea_pose_grid* g,
                       const ea_score_params* p, uint64_t max_cells, double* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "model");
        need(f, "field");
        need(g, "grid");
        need(p, "params");
        validate_params(*p);
        if (m->n == 0) fail(EA_ERR_INVALID_ARGUMENT, "score_map needs a nonempty model");
        const ea_grid_counts c = counts_of(*g);
        const uint64_t total = c.nx * c.ny * c.nt;
        if (total > max_cells) {
            fail(EA_ERR_BUDGET, "score_map needs " + std::to_string(total) +
                                    " cells but the budget allows " + std::to_string(max_cells));
        }
        need(out, "out");
        DeviceGuard dg(ctx->device);
        const int n = m->n;
        const std::vector<double>& cs = theta_cs(ctx, g->t0, g->dt, c.nt);
        ctx->cs_dev_key.clear();
        double* dcs = (double*)ctx->cs.ensure(sizeof(double) * 2 * c.nt);
        h2d_staged(ctx, dcs, cs.data(), sizeof(double) * 2 * c.nt);
        const size_t pairs = (size_t)c.nt * n;
        double* rot = (double*)ctx->rot_exact.ensure(sizeof(double) * 4 * pairs);
        launch_rotate(ctx, m->pts.as<double>(), n, dcs, (int)c.nt, rot, nullptr, nullptr);
        ExactArgs x = exact_args(f, *p, rot, pairs, n);
        x.nx = c.nx;
        x.ny = c.ny;
        x.it_begin = 0;
        x.x0 = g->x0;
        x.dx = g->dx;
        x.y0 = g->y0;
        x.dy = g->dy;
        double* d = (double*)ctx->work.ensure(sizeof(double) * total);
        launch_exact_map(ctx, x, total, d);
        d2h(ctx, out, d, sizeof(double) * total);
        sync(ctx);
    });
}

ea_status ea_screen_map(ea_ctx* ctx, const ea_model* m, const ea_field* f, const ea_pose_grid* g,
                        const ea_score_params* p, uint64_t max_cells, float* out, double* delta) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "model");
        need(f, "field");
        need(g, "grid");
        need(p, "params");
        validate_params(*p);
        if (m->n == 0) fail(EA_ERR_INVALID_ARGUMENT, "score_map needs a nonempty model");
        const ea_grid_counts c = counts_of(*g);
        const uint64_t total = c.nx * c.ny * c.nt;
        if (total > max_cells) {
            fail(EA_ERR_BUDGET, "score_map needs " + std::to_string(total) +
                                    " cells but the budget allows " + std::to_string(max_cells));
        }
        need(out, "out");
        DeviceGuard dg(ctx->device);
        ctx->stats = ea_search_stats{};
        const ScreenPlan plan = screen(ctx, m, f, *g, *p, 0, 0);
        int flags = 0;
        d2h(ctx, &flags, plan.flags, sizeof flags);
        d2h(ctx, out, ctx->map.p, sizeof(float) * total);
        sync(ctx);
        ctx->stats.flagged_points = flags;
        ctx->stats.screen_delta = plan.delta;
        if (delta) *delta = ctx->stats.screen_delta;
    });
}

// ---- coarse to fine ---------------------------------------------------------------------
ea_status ea_prepare_levels(ea_ctx* ctx, const double* const* tl, const int* tdims, int nt,
                            const double* const* wl, const int* wdims, int nw,
                            const ea_search_config* cfg, ea_levels** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(cfg, "config");
        need(out, "out");
        if (cfg->num_levels < 1) fail(EA_ERR_INVALID_ARGUMENT, "num_levels must be >= 1");
        const int L = cfg->num_levels;
        if (nt < L || nw < L)
            fail(EA_ERR_INVALID_ARGUMENT, "pyramids must provide " + std::to_string(L) + " levels");
        DeviceGuard dg(ctx->device);
        auto* lv = new ea_levels;
        try {
            for (int l = 0; l < L; ++l) {
                const int tw = tdims[2 * l], th = tdims[2 * l + 1];
                if (tw < 1 || th < 1) fail(EA_ERR_SIZE, "template level is empty");
                double* d = (double*)ctx->work.ensure(sizeof(double) * (size_t)tw * th);
                h2d_staged(ctx, d, tl[l], sizeof(double) * (size_t)tw * th);
                if (tw < 3 || th < 3) {
                    fail(EA_ERR_SIZE, "compute_gradients needs at least 3x3, got " +
                                          std::to_string(tw) + "x" + std::to_string(th));
                }
                lv->models.push_back(template_model(ctx, d, tw, th, *cfg, l));
                const int ww = wdims[2 * l], wh = wdims[2 * l + 1];
                if (ww < 3 || wh < 3) {
                    fail(EA_ERR_SIZE, "compute_gradients needs at least 3x3, got " +
                                          std::to_string(ww) + "x" + std::to_string(wh));
                }
                ea_field* f = new_field(ww, wh);
                lv->fields.push_back(f);
                double* dw = (double*)ctx->work.ensure(sizeof(double) * (size_t)ww * wh);
                h2d_staged(ctx, dw, wl[l], sizeof(double) * (size_t)ww * wh);
                sobel_into(ctx, dw, ww, wh, f);
                sync(ctx);
            }
        } catch (...) {
            free_levels(lv);
            throw;
        }
        *out = lv;
    });
}

ea_status ea_prepare_models(ea_ctx* ctx, const double* tmpl, int tw, int th,
                            const ea_search_config* cfg, ea_levels** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(tmpl, "template");
        need(cfg, "config");
        need(out, "out");
        DeviceGuard dg(ctx->device);
        const int L = cfg->num_levels;
        if (tw < 1 || th < 1) fail(EA_ERR_SIZE, "template image is empty");
        auto* lv = new ea_levels;
        try {
            const size_t elems = pyramid_elems(tw, th, std::max(L, 1));
            double* d = (double*)ctx->work.ensure(sizeof(double) * elems);
            h2d_staged(ctx, d, tmpl, sizeof(double) * (size_t)tw * th);
            std::vector<size_t> offs;
            std::vector<int> dims;
            device_pyramid(ctx, d, tw, th, L, &offs, &dims);
            for (int l = 0; l < L; ++l) {
                lv->models.push_back(
                    template_model(ctx, d + offs[l], dims[2 * l], dims[2 * l + 1], *cfg, l));
            }
        } catch (...) {
            free_levels(lv);
            throw;
        }
        *out = lv;
    });
}

ea_status ea_levels_set_image(ea_ctx* ctx, ea_levels* lv, const double* image, int w, int h) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(image, "image");
        DeviceGuard dg(ctx->device);
        set_working_image(ctx, lv, image, w, h, (int)lv->models.size());
        sync(ctx);
    });
}

int ea_levels_count(const ea_levels* lv) { return lv ? (int)lv->models.size() : 0; }

ea_status ea_levels_model(const ea_levels* lv, int level, ea_edge_point* points, int cap,
                          int* n_out, double* cx, double* cy) {
    return guard([&] {
        need(lv, "levels");
        need(n_out, "n_out");
        if (level < 0 || level >= (int)lv->models.size())
            fail(EA_ERR_BOUNDS, "level " + std::to_string(level) + " out of range");
        const ea_model* m = lv->models[level];
        *n_out = m->n;
        if (cx) *cx = m->centroid_x;
        if (cy) *cy = m->centroid_y;
        if (points)
            for (int i = 0; i < m->n && i < cap; ++i) points[i] = m->host[i];
    });
}

const ea_field* ea_levels_field(const ea_levels* lv, int level) {
    if (!lv || level < 0 || level >= (int)lv->fields.size()) return nullptr;
    return lv->fields[level];
}

const ea_model* ea_levels_get_model(const ea_levels* lv, int level) {
    if (!lv || level < 0 || level >= (int)lv->models.size()) return nullptr;
    return lv->models[level];
}

void ea_levels_free(ea_levels* lv) { free_levels(lv); }

ea_status ea_search_levels(ea_ctx* ctx, const ea_levels* lv, const ea_search_config* cfg,
                           ea_outcome* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(cfg, "config");
        need(out, "out");
        check_search_config(lv, *cfg);
        DeviceGuard dg(ctx->device);
        search_levels_device(ctx, lv, *cfg, out);
    });
}

ea_status ea_search_top_slab(ea_ctx* ctx, const ea_levels* lv, const ea_search_config* cfg,
                             uint64_t it_begin, uint64_t it_end, ea_scored_pose* seeds,
                             int* n_seeds) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(cfg, "config");
        need(n_seeds, "n_seeds");
        check_search_config(lv, *cfg);
        DeviceGuard dg(ctx->device);
        const int top = cfg->num_levels - 1;
        const uint64_t nt = counts_of(top_grid_of(*cfg)).nt;
        *n_seeds = 0;
        if (std::min(it_end, nt) <= std::min(it_begin, nt)) return;  // empty slab
        const auto r = top_search(ctx, lv->models[top], lv->fields[top], top_grid_of(*cfg),
                                  cfg->score_params, cfg->topk, it_begin, it_end);
        for (size_t i = 0; i < r.size(); ++i) seeds[i] = r[i];
        *n_seeds = (int)r.size();
    });
}

ea_status ea_search_top_slab_async(ea_ctx* ctx, const ea_levels* lv,
                                   const ea_search_config* cfg, uint64_t it_begin,
                                   uint64_t it_end, double* d_rows) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(cfg, "config");
        need(d_rows, "d_rows");
        check_search_config(lv, *cfg);
        DeviceGuard dg(ctx->device);
        const int top = cfg->num_levels - 1;
        if (!ctx->async_flag.p) {
            ctx->async_flag.ensure(sizeof(int));
            EAB_CUDA(cudaMemsetAsync(ctx->async_flag.p, 0, sizeof(int), ctx->stream));
        }
        // the candidate buffer covers the whole slab (async_cap), so the band
        // cannot overflow for slabs up to 2^26 poses; beyond, an overflow is
        // flagged for ea_ctx_async_status and marked in row 0
        slab_rows(ctx, lv->models[top], lv->fields[top], top_grid_of(*cfg), cfg->score_params,
                  cfg->topk, it_begin, it_end, d_rows, ctx->async_flag.as<int>());
    });
}

ea_status ea_merge_rows_async(ea_ctx* ctx, const double* d_rows, int n_rows, int k,
                              double* d_out) {
    return guard([&] {
        need(ctx, "ctx");
        need(d_rows, "d_rows");
        need(d_out, "d_out");
        if (k < 1) fail(EA_ERR_INVALID_ARGUMENT, "topk must be >= 1");
        if (n_rows < 0 || n_rows > merge_rows_max(ctx))
            fail(EA_ERR_INVALID_ARGUMENT,
                 "0 <= n_rows <= " + std::to_string(merge_rows_max(ctx)) + " required");
        DeviceGuard dg(ctx->device);
        launch_merge_rows(ctx, d_rows, n_rows, k, d_out);
    });
}

ea_status ea_ctx_async_status(ea_ctx* ctx, int* overflowed, float* screen_ms, int cap,
                              int* n_times) {
    return guard([&] {
        need(ctx, "ctx");
        DeviceGuard dg(ctx->device);
        sync(ctx);
        int of = 0;
        if (ctx->async_flag.p) {
            EAB_CUDA(cudaMemcpy(&of, ctx->async_flag.p, sizeof of, cudaMemcpyDeviceToHost));
            EAB_CUDA(cudaMemset(ctx->async_flag.p, 0, sizeof(int)));
        }
        if (overflowed) *overflowed = of;
        if (ctx->trace_on && !ctx->trace.empty()) {  // per-launch end-to-end deltas
            std::map<std::string, std::pair<double, int>> agg;
            for (size_t i = 1; i < ctx->trace.size(); ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, ctx->trace[i - 1].second, ctx->trace[i].second);
                auto& a = agg[ctx->trace[i].first];
                a.first += ms;
                a.second += 1;
            }
            for (auto& kv : agg)
                std::fprintf(stderr, "[trace] %-28s n=%5d avg_us=%8.2f\n", kv.first.c_str(),
                             kv.second.second, 1e3 * kv.second.first / kv.second.second);
            for (auto& t : ctx->trace) cudaEventDestroy(t.second);
            ctx->trace.clear();
        }
        int n = 0;
        if (ctx->timing) {
            const int pend = ctx->tev_pending;
            for (int q = 0; q < pend && n < cap; ++q) {
                const int slot = (ctx->tev_next - pend + q + ea_ctx::kTimeRing) % ea_ctx::kTimeRing;
                float ms = 0.f;
                EAB_CUDA(cudaEventElapsedTime(&ms, ctx->tev[2 * slot], ctx->tev[2 * slot + 1]));
                if (screen_ms) screen_ms[n] = ms;
                ++n;
            }
            ctx->tev_pending = 0;
        }
        if (n_times) *n_times = n;
    });
}

ea_status ea_refine(ea_ctx* ctx, const ea_levels* lv, const ea_search_config* cfg,
                    const ea_scored_pose* seeds, int n_seeds, ea_outcome* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(cfg, "config");
        need(out, "out");
        check_search_config(lv, *cfg);
        if (n_seeds < 1) fail(EA_ERR_INVALID_ARGUMENT, "refinement needs at least one seed");
        need(seeds, "seeds");
        DeviceGuard dg(ctx->device);
        const int k = cfg->topk, top = cfg->num_levels - 1, R = cfg->refine_radius;
        const int side = 2 * R + 1;
        std::vector<ea_scored_pose> v(seeds, seeds + std::min(n_seeds, k));
        const ea_pose_grid tg = top_grid_of(*cfg);
        const ea_grid_counts c = counts_of(tg);
        const double* tables = nullptr;
        if (top > 0 && (size_t)k * side * side * side <= 4096 && k <= 64)
            tables = theta_tables(ctx, tg, c.nt, top, R);
        if (top > 0 && !tables) {
            refine_levels(ctx, lv, *cfg, tg, seeds_to_beam(v), out);
            return;
        }
        // seeds -> device beam (theta path = the seed's theta index)
        const RefineState st = refine_state(ctx, k);
        const size_t bytes = sizeof(ea_outcome) + sizeof(BeamDev) * v.size() + sizeof(int);
        sync(ctx);
        char* hb = (char*)ctx->h_stage.ensure(bytes);
        ea_outcome* ho = (ea_outcome*)hb;
        std::memset(ho, 0, sizeof(ea_outcome));
        ho->trace[0].level = top;
        ho->trace[0].pose = v[0].pose;
        ho->trace[0].score = v[0].score;
        ho->n_trace = 1;
        if (top == 0) {
            ho->pose = v[0].pose;
            ho->score = v[0].score;
            ho->grid_index = v[0].grid_index;
            ho->found = v[0].score >= cfg->min_score ? 1 : 0;
            *out = *ho;
            return;
        }
        BeamDev* hbeam = (BeamDev*)(hb + sizeof(ea_outcome));
        const uint64_t plane = c.nx * c.ny;
        for (size_t i = 0; i < v.size(); ++i) {
            hbeam[i] = BeamDev{v[i].pose.ux, v[i].pose.uy, v[i].pose.theta, v[i].score,
                               v[i].grid_index, (int)(v[i].grid_index / plane), 0};
        }
        *(int*)(hb + sizeof(ea_outcome) + sizeof(BeamDev) * v.size()) = (int)v.size();
        h2d(ctx, st.out, ho, sizeof(ea_outcome));
        h2d(ctx, st.beam[0], hbeam, sizeof(BeamDev) * v.size());
        h2d(ctx, st.cnt[0], hb + sizeof(ea_outcome) + sizeof(BeamDev) * v.size(), sizeof(int));
        refine_enqueue(ctx, lv, *cfg, tg, tables, st);
        d2h(ctx, out, st.out, sizeof(ea_outcome));
        sync(ctx);
    });
}

// ---- multi-GPU -------------------------------------------------------------------------------
void ea_theta_slab(uint64_t nt, int rank, int world, uint64_t* it_begin, uint64_t* it_end) {
    uint64_t b = 0, e = 0;
    if (world >= 1 && rank >= 0 && rank < world) theta_slab_of(nt, rank, world, &b, &e);
    if (it_begin) *it_begin = b;
    if (it_end) *it_end = e;
}

ea_status ea_comm_unique_id(ea_comm_id* out) {
    return guard([&] {
        need(out, "out");
        ncclUniqueId id;
        EAB_NCCL(nccl().GetUniqueId(&id));
        std::memcpy(out->internal, &id, sizeof id);
    });
}

ea_status ea_comm_init(ea_ctx* ctx, int rank, int world, const ea_comm_id* id) {
    return guard([&] {
        need(ctx, "ctx");
        need(id, "id");
        if (world < 1 || rank < 0 || rank >= world)
            fail(EA_ERR_INVALID_ARGUMENT, "need 0 <= rank < world");
        DeviceGuard dg(ctx->device);
        const NcclApi& api = nccl();
        if (ctx->comm) {
            sync(ctx);
            api.CommDestroy(static_cast<ncclComm_t>(ctx->comm));
            ctx->comm = nullptr;
        }
        ncclUniqueId uid;
        std::memcpy(&uid, id->internal, sizeof uid);
        ncclComm_t c = nullptr;
        EAB_NCCL(api.CommInitRank(&c, world, uid, rank));
        ctx->comm = c;
        ctx->comm_rank = rank;
        ctx->comm_world = world;
    });
}

ea_status ea_comm_info(const ea_ctx* ctx, int* rank, int* world) {
    return guard([&] {
        need(ctx, "ctx");
        comm_of(ctx);
        if (rank) *rank = ctx->comm_rank;
        if (world) *world = ctx->comm_world;
    });
}

ea_status ea_comm_destroy(ea_ctx* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        if (!ctx->comm) return;
        DeviceGuard dg(ctx->device);
        sync(ctx);
        EAB_NCCL(nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm)));
        ctx->comm = nullptr;
        ctx->comm_rank = 0;
        ctx->comm_world = 1;
    });
}

ea_status ea_gather_rows_async(ea_ctx* ctx, const double* d_local, int k, double* d_merged) {
    return guard([&] {
        need(ctx, "ctx");
        need(d_local, "d_local");
        need(d_merged, "d_merged");
        if (k < 1) fail(EA_ERR_INVALID_ARGUMENT, "topk must be >= 1");
        DeviceGuard dg(ctx->device);
        gather_rows(ctx, d_local, k, d_merged, /*seed_topk=*/false);
    });
}

ea_status ea_search_levels_sharded(ea_ctx* ctx, const ea_levels* lv, const ea_search_config* cfg,
                                   ea_outcome* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(cfg, "config");
        need(out, "out");
        check_search_config(lv, *cfg);
        comm_of(ctx);
        DeviceGuard dg(ctx->device);
        const uint64_t launched0 = ctx->launches;
        search_levels_sharded(ctx, lv, lv->fields[cfg->num_levels - 1], *cfg, out);
        ctx->stats.kernels_launched = (int)(ctx->launches - launched0);
    });
}

ea_status ea_detect_sharded(ea_ctx* ctx, ea_levels* lv, const double* image, int w, int h,
                            const ea_search_config* cfg, ea_outcome* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(cfg, "config");
        need(out, "out");
        comm_of(ctx);
        const bool root = ctx->comm_rank == 0;
        if (root) need(image, "image");
        DeviceGuard dg(ctx->device);
        const int L = cfg->num_levels;
        if (L < 1 || (int)lv->models.size() < L)
            fail(EA_ERR_INVALID_ARGUMENT, "prepared levels do not cover num_levels");
        if (L > EA_MAX_LEVELS) fail(EA_ERR_INVALID_ARGUMENT, "num_levels exceeds EA_MAX_LEVELS");
        validate_params(cfg->score_params);
        if (cfg->topk < 1 || cfg->refine_radius < 1)
            fail(EA_ERR_INVALID_ARGUMENT, "topk and refine_radius must be >= 1");
        if (w < 1 || h < 1) {
            fail(EA_ERR_SIZE, "image dimensions must be at least 1x1, got " + std::to_string(w) +
                                  "x" + std::to_string(h));
        }
        const int feasible = pyramid_levels_feasible(w, h);
        if (L > feasible) {
            fail(EA_ERR_SIZE, "pyramid of " + std::to_string(L) +
                                  " levels would drop below 8x8; maximum feasible level count is " +
                                  std::to_string(feasible));
        }
        const uint64_t launched0 = ctx->launches;
        if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
        const int top = L - 1, wt = w >> top, ht = h >> top;
        ea_field* ftop = nullptr;
        if (root) {  // the whole working pyramid and every level's field
            set_working_image(ctx, lv, image, w, h, L);
            ftop = lv->fields[top];
        } else {  // only the top level's field, from the root
            if (lv->shard_top && (lv->shard_top->width != wt || lv->shard_top->height != ht)) {
                delete lv->shard_top;
                lv->shard_top = nullptr;
            }
            if (!lv->shard_top) lv->shard_top = new_field(wt, ht);
            ftop = lv->shard_top;
        }
        // SURVEY §8(e) e1 input distribution: one broadcast of gx|gy|mag of
        // the top level (cfg3: 162 x 121 x 24 B = 470 KB) instead of the
        // 40 MB level-0 image on every rank
        EAB_NCCL(nccl().Broadcast(ftop->g.p, ftop->g.p, 3 * (size_t)wt * ht, ncclDouble, 0,
                                  comm_of(ctx), ctx->stream));
        if (!root) {
            ftop->version = next_field_version();
            ftop->ring_max = 0.0;  // a Sobel field: the border ring is exactly 0
        }
        if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
        search_levels_sharded(ctx, lv, ftop, *cfg, out);
        if (ctx->timing) {
            float ms = 0.f;
            EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[4], ctx->ev[5]));
            ctx->stats.image_ms = ms;
        }
        ctx->stats.kernels_launched = (int)(ctx->launches - launched0);
    });
}

ea_status ea_plan_multi(const uint64_t* plane_poses, const uint64_t* thetas, const int* n_top,
                        int n_models, int world, double fixed_evals, ea_work_item* items,
                        int cap, int* n_items) {
    return guard([&] {
        need(n_items, "n_items");
        if (n_models > 0) {
            need(plane_poses, "plane_poses");
            need(thetas, "thetas");
            need(n_top, "n_top");
        }
        const std::vector<ea_work_item> v =
            plan_multi(plane_poses, thetas, n_top, n_models, world, fixed_evals);
        *n_items = (int)v.size();
        if ((int)v.size() > cap) fail(EA_ERR_INVALID_ARGUMENT, "items buffer too small");
        for (size_t i = 0; i < v.size(); ++i) items[i] = v[i];
    });
}

ea_status ea_gather_rows_multi_async(ea_ctx* ctx, const double* d_local, int n_models, int k,
                                     double* d_merged) {
    return guard([&] {
        need(ctx, "ctx");
        need(d_local, "d_local");
        need(d_merged, "d_merged");
        if (k < 1 || n_models < 1) fail(EA_ERR_INVALID_ARGUMENT, "need topk >= 1, n_models >= 1");
        ncclComm_t comm = comm_of(ctx);
        const int world = ctx->comm_world;
        if (world * k > merge_rows_max(ctx))
            fail(EA_ERR_INVALID_ARGUMENT, "world * topk exceeds the merge's shared memory");
        DeviceGuard dg(ctx->device);
        const size_t rows = 5 * (size_t)n_models * k;
        const size_t o_seed = (sizeof(double) * rows * world + 255) & ~(size_t)255;
        const size_t seeds = (sizeof(double) + sizeof(unsigned long long)) * (size_t)n_models * k;
        char* base = (char*)ctx->mscratch.ensure(o_seed + seeds + sizeof(int) * n_models);
        double* gathered = (double*)base;
        double* ts = (double*)(base + o_seed);
        EAB_NCCL(nccl().AllGather(d_local, gathered, rows, ncclDouble, comm, ctx->stream));
        launch_merge_rows_multi(ctx, gathered, world, n_models, k, d_merged, ts,
                                reinterpret_cast<unsigned long long*>(ts + (size_t)n_models * k),
                                (int*)(base + o_seed + seeds));
    });
}

ea_status ea_detect_multi_sharded(ea_ctx* ctx, ea_levels* const* models, int n,
                                  const double* image, int w, int h,
                                  const ea_search_config* cfg, ea_outcome* outs) {
    return guard([&] {
        need(ctx, "ctx");
        need(cfg, "config");
        if (n <= 0) return;
        need(models, "models");
        need(outs, "outs");
        comm_of(ctx);
        if (ctx->comm_rank == 0) need(image, "image");
        DeviceGuard dg(ctx->device);
        const uint64_t launched0 = ctx->launches;
        detect_multi_sharded(ctx, models, n, image, w, h, *cfg, outs);
        ctx->stats.kernels_launched = (int)(ctx->launches - launched0);
    });
}

ea_status ea_coarse_to_fine(ea_ctx* ctx, const double* const* tl, const int* tdims, int nt,
                            const double* const* wl, const int* wdims, int nw,
                            const ea_search_config* cfg, ea_outcome* out) {
    ea_levels* lv = nullptr;
    ea_status st = ea_prepare_levels(ctx, tl, tdims, nt, wl, wdims, nw, cfg, &lv);
    if (st != EA_OK) return st;
    st = ea_search_levels(ctx, lv, cfg, out);
    free_levels(lv);
    return st;
}

ea_status ea_detect(ea_ctx* ctx, ea_levels* lv, const double* image, int w, int h,
                    const ea_search_config* cfg, ea_outcome* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(image, "image");
        need(cfg, "config");
        need(out, "out");
        DeviceGuard dg(ctx->device);
        if ((int)lv->models.size() < cfg->num_levels)
            fail(EA_ERR_INVALID_ARGUMENT, "prepared levels do not cover num_levels");
        if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
        set_working_image(ctx, lv, image, w, h, cfg->num_levels);
        if (ctx->timing) EAB_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
        check_search_config(lv, *cfg);
        const int launched0 = ctx->launches;
        search_levels_device(ctx, lv, *cfg, out);
        if (ctx->timing) {
            float ms = 0.f;
            EAB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[4], ctx->ev[5]));
            ctx->stats.image_ms = ms;
        }
        ctx->stats.kernels_launched = (int)(ctx->launches - launched0);
    });
}

ea_status ea_detect_batch(ea_ctx* ctx, ea_levels* lv, const double* const* images, int count,
                          int w, int h, const ea_search_config* cfg, ea_outcome* outs) {
    return guard([&] {
        need(ctx, "ctx");
        need(lv, "levels");
        need(cfg, "config");
        if (count <= 0) return;
        need(images, "images");
        need(outs, "outs");
        DeviceGuard dg(ctx->device);
        if ((int)lv->models.size() < cfg->num_levels)
            fail(EA_ERR_INVALID_ARGUMENT, "prepared levels do not cover num_levels");
        const uint64_t launched0 = ctx->launches;
        detect_batch(ctx, lv, images, count, w, h, *cfg, outs);
        ctx->stats.kernels_launched = (int)(ctx->launches - launched0);
    });
}

ea_status ea_detect_multi(ea_ctx* ctx, ea_levels* const* models, int n, const double* image,
                          int w, int h, const ea_search_config* cfg, ea_outcome* outs) {
    return guard([&] {
        need(ctx, "ctx");
        need(cfg, "config");
        if (n <= 0) return;
        need(models, "models");
        need(image, "image");
        need(outs, "outs");
        DeviceGuard dg(ctx->device);
        const uint64_t launched0 = ctx->launches;
        detect_multi(ctx, models, n, image, w, h, *cfg, outs);
        ctx->stats.kernels_launched = (int)(ctx->launches - launched0);
    });
}

// ---- Netpbm codecs ---------------------------------------------------------------------------
uint8_t ea_luminance_to_byte(double v) { return host_luminance_to_byte(v); }

ea_status ea_load_pgm(const uint8_t* bytes, size_t size, double* out, size_t cap, int* w,
                      int* h) {
    return guard([&] {
        need(bytes, "bytes");
        need(w, "width");
        need(h, "height");
        std::vector<double> img;
        host_load_pgm(bytes, size, out ? &img : nullptr, w, h);
        if (out) {
            if (cap < img.size())
                fail(EA_ERR_INVALID_ARGUMENT, "output capacity " + std::to_string(cap) +
                                                  " < " + std::to_string(img.size()) + " pixels");
            std::memcpy(out, img.data(), sizeof(double) * img.size());
        }
    });
}

ea_status ea_save_pgm(const double* image, int w, int h, uint8_t* out, size_t cap,
                      size_t* n_out) {
    return guard([&] {
        need(image, "image");
        need(n_out, "n_out");
        const auto b = host_save_pgm(image, w, h);
        *n_out = b.size();
        if (out) {
            if (cap < b.size()) fail(EA_ERR_INVALID_ARGUMENT, "output capacity too small");
            std::memcpy(out, b.data(), b.size());
        }
    });
}

ea_status ea_save_ppm(const double* image, int w, int h, const int* xy, int n_xy, uint8_t r,
                      uint8_t g, uint8_t b, uint8_t* out, size_t cap, size_t* n_out) {
    return guard([&] {
        need(image, "image");
        need(n_out, "n_out");
        if (n_xy > 0) need(xy, "overlay");
        const auto bytes = host_save_ppm(image, w, h, xy, std::max(n_xy, 0), r, g, b);
        *n_out = bytes.size();
        if (out) {
            if (cap < bytes.size()) fail(EA_ERR_INVALID_ARGUMENT, "output capacity too small");
            std::memcpy(out, bytes.data(), bytes.size());
        }
    });
}

ea_status ea_overlay_points(const ea_edge_point* points, int n, const ea_pose* pose,
                            int* out_xy) {
    return guard([&] {
        need(pose, "pose");
        if (n < 0) fail(EA_ERR_INVALID_ARGUMENT, "point count must be >= 0");
        if (n > 0) {
            need(points, "points");
            need(out_xy, "out");
        }
        host_overlay_points(points, n, *pose, out_xy);
    });
}

// ---- synthetic scenes ----------------------------------------------------------------------
ea_status ea_render_template(int template_id, int size, double* out) {
    return guard([&] {
        need(out, "out");
        host_render_template(template_id, size, out);
    });
}

ea_status ea_compose_scene(const ea_scene_spec* spec, double* canvas, double* tmpl,
                           ea_pose* truth_pose, double* occluded_fraction) {
    return guard([&] {
        need(spec, "spec");
        need(canvas, "canvas");
        need(tmpl, "template");
        ea_pose tp{};
        double occ = 0.0;
        host_compose_scene(*spec, canvas, tmpl, &tp, &occ);
        if (truth_pose) *truth_pose = tp;
        if (occluded_fraction) *occluded_fraction = occ;
    });
}

ea_status ea_compose_multi(const ea_scene_spec* spec, const ea_stamp* stamps, int n_stamps,
                           double* canvas) {
    return guard([&] {
        need(spec, "spec");
        need(canvas, "canvas");
        host_compose_multi(*spec, stamps, n_stamps, canvas);
    });
}

}  // extern "C"
