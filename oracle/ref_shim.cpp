// ref_shim.cpp -- TEST INFRASTRUCTURE, not product code.
//
// A C-ABI over the UNMODIFIED reference library compiled from its own sources
// under /root/reference/proj/src (recipe: oracle/Makefile, outputs only into
// oracle/_ref/).  It lets Python tests, the golden-vector generator and
// bench.py's CPU-baseline leg run the reference itself.  Every entry point
// forwards to the reference function named in its comment; nothing here
// re-implements reference arithmetic.
//
// Plain-data structs come from include/edgealign_b200.h (shared vocabulary
// only; none of the product library is linked).
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "edgealign/edge_model.h"
#include "edgealign/errors.h"
#include "edgealign/gradient.h"
#include "edgealign/image.h"
#include "edgealign/pose.h"
#include "edgealign/search.h"
#include "edgealign/similarity.h"
#include "edgealign/simd/kernels.h"
#include "edgealign/synth.h"

#include "../include/edgealign_b200.h"

using namespace edgealign;

namespace {

thread_local std::string g_err;
thread_local double g_err_value = 0.0;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        return EA_OK;
    } catch (const EmptyModelError& e) {
        g_err = e.what();
        g_err_value = e.max_magnitude();
        return EA_ERR_EMPTY_MODEL;
    } catch (const ParseError& e) {
        g_err = e.what();
        g_err_value = static_cast<double>(e.offset());
        return EA_ERR_PARSE;
    } catch (const SizeError& e) {
        g_err = e.what();
        return EA_ERR_SIZE;
    } catch (const BoundsError& e) {
        g_err = e.what();
        return EA_ERR_BOUNDS;
    } catch (const BudgetError& e) {
        g_err = e.what();
        return EA_ERR_BUDGET;
    } catch (const GeometryError& e) {
        g_err = e.what();
        return EA_ERR_GEOMETRY;
    } catch (const InvalidArgument& e) {
        g_err = e.what();
        return EA_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return EA_ERR_INTERNAL;
    }
}

Image make_image(const double* data, int w, int h) {
    Image img(w, h);
    std::memcpy(img.data.data(), data, sizeof(double) * static_cast<std::size_t>(w) * h);
    return img;
}

GradientField make_field(const double* gx, const double* gy, const double* mag, int w,
                         int h) {
    GradientField f(w, h);
    const std::size_t n = static_cast<std::size_t>(w) * h;
    std::memcpy(f.gx.data(), gx, sizeof(double) * n);
    std::memcpy(f.gy.data(), gy, sizeof(double) * n);
    std::memcpy(f.mag.data(), mag, sizeof(double) * n);
    return f;
}

EdgeModel make_model(const ea_edge_point* pts, int n, double cx, double cy) {
    EdgeModel m;
    m.centroid_x = cx;
    m.centroid_y = cy;
    m.points.resize(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
        m.points[i] = EdgePoint{pts[i].x_rel, pts[i].y_rel, pts[i].dx, pts[i].dy,
                                pts[i].mag};
    }
    return m;
}

PoseGrid make_grid(const ea_pose_grid* g) {
    PoseGrid p;
    p.x0 = g->x0; p.x1 = g->x1; p.dx = g->dx;
    p.y0 = g->y0; p.y1 = g->y1; p.dy = g->dy;
    p.t0 = g->t0; p.t1 = g->t1; p.dt = g->dt;
    return p;
}

ScoreParams make_params(const ea_score_params* p) {
    ScoreParams s;
    s.neighborhood = p->neighborhood;
    s.polarity = p->polarity == EA_POLARITY_IGNORE ? Polarity::Ignore : Polarity::Signed;
    s.eps_mag = p->eps_mag;
    return s;
}

Backend make_backend(int kind, int workers) {
    Backend b;
    b.kind = kind == EA_BACKEND_PARALLEL ? BackendKind::Parallel : BackendKind::Serial;
    b.worker_count = workers;
    return b;
}

SearchConfig make_config(const ea_search_config* c) {
    SearchConfig s;
    s.grid = make_grid(&c->grid);
    s.num_levels = c->num_levels;
    s.score_params = make_params(&c->score_params);
    if (c->has_thresholds) {
        s.thresholds = EdgeThresholds{c->thresholds.low, c->thresholds.high};
    }
    s.min_score = c->min_score;
    s.topk = c->topk;
    s.refine_radius = c->refine_radius;
    s.backend = make_backend(c->backend_kind, c->worker_count);
    return s;
}

void fill_outcome(const SearchOutcome& o, ea_outcome* out) {
    std::memset(out, 0, sizeof(*out));
    out->found = o.found ? 1 : 0;
    out->pose = ea_pose{o.best.pose.ux, o.best.pose.uy, o.best.pose.theta};
    out->score = o.best.score;
    out->grid_index = o.best.grid_index;
    out->n_trace = static_cast<int32_t>(o.best.level_trace.size());
    for (std::size_t i = 0; i < o.best.level_trace.size() && i < EA_MAX_LEVELS; ++i) {
        const LevelTrace& t = o.best.level_trace[i];
        out->trace[i].level = t.level;
        out->trace[i].pose = ea_pose{t.pose.ux, t.pose.uy, t.pose.theta};
        out->trace[i].score = t.score;
    }
}

Pyramid make_pyramid(const double* const* levels, const int* dims, int n) {
    Pyramid p;
    for (int l = 0; l < n; ++l) {
        p.levels.push_back(make_image(levels[l], dims[2 * l], dims[2 * l + 1]));
    }
    return p;
}

}  // namespace

struct eref_levels {
    PyramidLevels lv;
};

extern "C" {

const char* eref_last_error(void) { return g_err.c_str(); }
double eref_last_error_value(void) { return g_err_value; }

// simd::set_active  dispatch.cpp:38-54 (0 = scalar, 1 = avx2)
int eref_set_isa(int isa) {
    return guard([&] { simd::set_active(isa == 1 ? simd::Isa::Avx2 : simd::Isa::Scalar); });
}
int eref_isa_supported(int isa) {
    return simd::supported(isa == 1 ? simd::Isa::Avx2 : simd::Isa::Scalar) ? 1 : 0;
}
// Kernels::sobel_row / downsample_row / vote_span  kernels.h:18-44
int eref_sobel_row(int isa, const double* a, const double* m, const double* b, int width,
                   double* gx, double* gy, double* mag) {
    return guard([&] {
        simd::kernels(isa == 1 ? simd::Isa::Avx2 : simd::Isa::Scalar)
            .sobel_row(a, m, b, width, gx, gy, mag);
    });
}
int eref_downsample_row(int isa, const double* top, const double* bot, int out_width,
                        double* out) {
    return guard([&] {
        simd::kernels(isa == 1 ? simd::Isa::Avx2 : simd::Isa::Scalar)
            .downsample_row(top, bot, out_width, out);
    });
}
int eref_vote_span(int isa, const double* gx, const double* gy, const double* mag, int x0,
                   int x1, double dx, double dy, double eps, int absolute, double* out) {
    return guard([&] {
        *out = simd::kernels(isa == 1 ? simd::Isa::Avx2 : simd::Isa::Scalar)
                   .vote_span(gx, gy, mag, x0, x1, dx, dy, eps, absolute != 0);
    });
}

// grid_counts / pose_at  pose.h:52-92
int eref_grid_counts(const ea_pose_grid* g, ea_grid_counts* out) {
    return guard([&] {
        const GridCounts c = grid_counts(make_grid(g));
        *out = ea_grid_counts{c.nx, c.ny, c.nt};
    });
}
int eref_pose_at(const ea_pose_grid* g, uint64_t index, ea_pose* out) {
    return guard([&] {
        const Pose p = pose_at(make_grid(g), static_cast<std::size_t>(index));
        *out = ea_pose{p.ux, p.uy, p.theta};
    });
}

// downsample / max_pyramid_levels / build_pyramid  image.cpp:248-291
int eref_downsample(const double* img, int w, int h, double* out) {
    return guard([&] {
        const Image o = downsample(make_image(img, w, h));
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
    });
}
int eref_max_pyramid_levels(int w, int h) { return max_pyramid_levels(Image(w, h)); }
int eref_build_pyramid(const double* img, int w, int h, int levels, double* out) {
    return guard([&] {
        const Pyramid p = build_pyramid(make_image(img, w, h), levels);
        std::size_t off = 0;
        for (const Image& l : p.levels) {
            std::memcpy(out + off, l.data.data(), sizeof(double) * l.data.size());
            off += l.data.size();
        }
    });
}

// compute_gradients  gradient.cpp:12-27
int eref_compute_gradients(const double* img, int w, int h, double* gx, double* gy,
                           double* mag) {
    return guard([&] {
        if (w < 1 || h < 1) {
            throw SizeError("image dimensions must be at least 1x1");
        }
        const GradientField f = compute_gradients(make_image(img, w, h));
        std::memcpy(gx, f.gx.data(), sizeof(double) * f.gx.size());
        std::memcpy(gy, f.gy.data(), sizeof(double) * f.gy.size());
        std::memcpy(mag, f.mag.data(), sizeof(double) * f.mag.size());
    });
}

// default_thresholds / extract_edge_model  edge_model.cpp:17-149
int eref_default_thresholds(const double* gx, const double* gy, const double* mag, int w,
                            int h, ea_edge_thresholds* out) {
    return guard([&] {
        const EdgeThresholds t = default_thresholds(make_field(gx, gy, mag, w, h));
        *out = ea_edge_thresholds{t.low, t.high};
    });
}
int eref_extract_edge_model(const double* gx, const double* gy, const double* mag, int w,
                            int h, const ea_edge_thresholds* th, int level,
                            ea_edge_point* pts, int cap, int* n_out, double* cx,
                            double* cy) {
    return guard([&] {
        const EdgeModel m = extract_edge_model(make_field(gx, gy, mag, w, h),
                                               EdgeThresholds{th->low, th->high}, level);
        const int n = static_cast<int>(m.points.size());
        *n_out = n;
        *cx = m.centroid_x;
        *cy = m.centroid_y;
        for (int i = 0; i < n && i < cap; ++i) {
            const EdgePoint& p = m.points[i];
            pts[i] = ea_edge_point{p.x_rel, p.y_rel, p.dx, p.dy, p.mag};
        }
    });
}

// point_vote / rotate_model / pose_score  similarity.cpp:58-126
int eref_point_vote(double dir_x, double dir_y, const double* gx, const double* gy,
                    const double* mag, int w, int h, int cx, int cy,
                    const ea_score_params* p, double* out) {
    return guard([&] {
        *out = point_vote(dir_x, dir_y, make_field(gx, gy, mag, w, h), cx, cy,
                          make_params(p));
    });
}
int eref_rotate_model(const ea_edge_point* pts, int n, double theta, double* px, double* py,
                      double* dx, double* dy) {
    return guard([&] {
        const RotatedModel r = rotate_model(make_model(pts, n, 0, 0), theta);
        for (int i = 0; i < n; ++i) {
            px[i] = r.px[i];
            py[i] = r.py[i];
            dx[i] = r.dx[i];
            dy[i] = r.dy[i];
        }
    });
}
int eref_pose_score(const ea_edge_point* pts, int n, const ea_pose* pose, const double* gx,
                    const double* gy, const double* mag, int w, int h,
                    const ea_score_params* p, double* value, int* n_in) {
    return guard([&] {
        const PoseScore s = pose_score(make_model(pts, n, 0, 0),
                                       Pose{pose->ux, pose->uy, pose->theta},
                                       make_field(gx, gy, mag, w, h), make_params(p));
        *value = s.value;
        *n_in = s.n_inbounds;
    });
}

// search_topk / exhaustive_search / score_map  search.cpp:144-202
int eref_search_topk(const ea_edge_point* pts, int n, const double* gx, const double* gy,
                     const double* mag, int w, int h, const ea_pose_grid* g,
                     const ea_score_params* p, int backend_kind, int workers, int k,
                     ea_scored_pose* out, int* n_out) {
    return guard([&] {
        const auto r = search_topk(make_model(pts, n, 0, 0), make_field(gx, gy, mag, w, h),
                                   make_grid(g), make_params(p),
                                   make_backend(backend_kind, workers), k);
        *n_out = static_cast<int>(r.size());
        for (std::size_t i = 0; i < r.size(); ++i) {
            out[i] = ea_scored_pose{r[i].score, r[i].grid_index,
                                    ea_pose{r[i].pose.ux, r[i].pose.uy, r[i].pose.theta}};
        }
    });
}
int eref_exhaustive_search(const ea_edge_point* pts, int n, const double* gx,
                           const double* gy, const double* mag, int w, int h,
                           const ea_pose_grid* g, const ea_score_params* p,
                           int backend_kind, int workers, ea_scored_pose* out) {
    return guard([&] {
        const Detection d = exhaustive_search(make_model(pts, n, 0, 0),
                                              make_field(gx, gy, mag, w, h), make_grid(g),
                                              make_params(p),
                                              make_backend(backend_kind, workers));
        *out = ea_scored_pose{d.score, d.grid_index, ea_pose{d.pose.ux, d.pose.uy, d.pose.theta}};
    });
}
int eref_score_map(const ea_edge_point* pts, int n, const double* gx, const double* gy,
                   const double* mag, int w, int h, const ea_pose_grid* g,
                   const ea_score_params* p, uint64_t max_cells, double* out) {
    return guard([&] {
        const auto m = score_map(make_model(pts, n, 0, 0), make_field(gx, gy, mag, w, h),
                                 make_grid(g), make_params(p),
                                 static_cast<std::size_t>(max_cells));
        std::memcpy(out, m.data(), sizeof(double) * m.size());
    });
}

// prepare_levels / search_levels / coarse_to_fine  search.cpp:208-364
int eref_prepare_levels(const double* const* tl, const int* tdims, int nt,
                        const double* const* wl, const int* wdims, int nw,
                        const ea_search_config* cfg, eref_levels** out) {
    return guard([&] {
        auto* h = new eref_levels;
        try {
            h->lv = prepare_levels(make_pyramid(tl, tdims, nt), make_pyramid(wl, wdims, nw),
                                   make_config(cfg));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
int eref_levels_model(const eref_levels* h, int level, ea_edge_point* pts, int cap,
                      int* n_out, double* cx, double* cy) {
    return guard([&] {
        const EdgeModel& m = h->lv.models.at(static_cast<std::size_t>(level));
        *n_out = static_cast<int>(m.points.size());
        *cx = m.centroid_x;
        *cy = m.centroid_y;
        for (int i = 0; i < *n_out && i < cap; ++i) {
            const EdgePoint& p = m.points[i];
            pts[i] = ea_edge_point{p.x_rel, p.y_rel, p.dx, p.dy, p.mag};
        }
    });
}
int eref_levels_field(const eref_levels* h, int level, double* gx, double* gy,
                      double* mag) {
    return guard([&] {
        const GradientField& f = h->lv.fields.at(static_cast<std::size_t>(level));
        std::memcpy(gx, f.gx.data(), sizeof(double) * f.gx.size());
        std::memcpy(gy, f.gy.data(), sizeof(double) * f.gy.size());
        std::memcpy(mag, f.mag.data(), sizeof(double) * f.mag.size());
    });
}
int eref_search_levels(const eref_levels* h, const ea_search_config* cfg, ea_outcome* out) {
    return guard([&] { fill_outcome(search_levels(h->lv, make_config(cfg)), out); });
}
void eref_levels_free(eref_levels* h) { delete h; }

int eref_coarse_to_fine(const double* const* tl, const int* tdims, int nt,
                        const double* const* wl, const int* wdims, int nw,
                        const ea_search_config* cfg, ea_outcome* out) {
    return guard([&] {
        fill_outcome(coarse_to_fine(make_pyramid(tl, tdims, nt), make_pyramid(wl, wdims, nw),
                                    make_config(cfg)),
                     out);
    });
}

// render_template / compose_scene  synth.cpp:62-300
int eref_render_template(int id, int size, double* out) {
    return guard([&] {
        if (id < 0 || id > 3) {
            throw InvalidArgument("unknown template id");
        }
        const Image img = render_template(static_cast<TemplateId>(id), size);
        std::memcpy(out, img.data.data(), sizeof(double) * img.data.size());
    });
}
int eref_compose_scene(const ea_scene_spec* s, double* canvas, double* tmpl,
                       ea_pose* truth_pose, double* occluded_fraction) {
    return guard([&] {
        SceneSpec spec;
        spec.canvas_width = s->canvas_width;
        spec.canvas_height = s->canvas_height;
        if (s->template_id < 0 || s->template_id > 3) {
            throw InvalidArgument("unknown template id");
        }
        spec.template_id = static_cast<TemplateId>(s->template_id);
        spec.template_size = s->template_size;
        spec.true_pose = Pose{s->true_pose.ux, s->true_pose.uy, s->true_pose.theta};
        spec.clutter_segments = s->clutter_segments;
        spec.clutter_seed = s->clutter_seed;
        if (s->has_occluder) {
            spec.occluder = OccluderSpec{s->occ_x, s->occ_y, s->occ_w, s->occ_h, s->occ_fill};
        }
        spec.illumination = IlluminationSpec{s->gain, s->bias, s->gamma};
        spec.noise_sigma = s->noise_sigma;
        spec.noise_seed = s->noise_seed;
        const auto [scene, truth] = compose_scene(spec);
        std::memcpy(canvas, scene.data.data(), sizeof(double) * scene.data.size());
        std::memcpy(tmpl, truth.template_image.data.data(),
                    sizeof(double) * truth.template_image.data.size());
        *truth_pose = ea_pose{truth.pose.ux, truth.pose.uy, truth.pose.theta};
        *occluded_fraction = truth.occluded_fraction;
    });
}

// Netpbm codecs  image.cpp:26-219 (bytes in, bytes out)
int eref_luminance_to_byte(double v) { return luminance_to_byte(v); }
int eref_load_pgm(const unsigned char* bytes, size_t size, double* out, size_t cap, int* w,
                  int* h) {
    return guard([&] {
        const Image img = load_pgm(bytes, size);
        *w = img.width;
        *h = img.height;
        if (out && cap >= img.data.size())
            std::memcpy(out, img.data.data(), sizeof(double) * img.data.size());
    });
}
int eref_save_pgm(const double* img, int w, int h, unsigned char* out, size_t cap, size_t* n) {
    return guard([&] {
        Image im(w, h);
        std::memcpy(im.data.data(), img, sizeof(double) * im.data.size());
        const auto b = save_pgm(im);
        *n = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    });
}
int eref_save_ppm(const double* img, int w, int h, const int* xy, int n_xy, int r, int g, int b,
                  unsigned char* out, size_t cap, size_t* n) {
    return guard([&] {
        Image im(w, h);
        std::memcpy(im.data.data(), img, sizeof(double) * im.data.size());
        std::vector<std::pair<int, int>> ov;
        for (int i = 0; i < n_xy; ++i) ov.emplace_back(xy[2 * i], xy[2 * i + 1]);
        const auto bytes = save_ppm(im, ov, Rgb{(std::uint8_t)r, (std::uint8_t)g, (std::uint8_t)b});
        *n = bytes.size();
        if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
    });
}

// resolved_workers  search.cpp:15-24
int eref_resolved_workers(int kind, int workers) {
    return resolved_workers(make_backend(kind, workers));
}

}  // extern "C"
