// edgealign_b200.hpp -- header-only C++ mirror of the reference `edgealign`
// API (proj/include/edgealign/*.h) over the C-ABI in edgealign_b200.h.
//
// Same function names and argument meaning as the reference; failures throw
// the reference's exception classes (errors.h:14-75) with the same messages.
// Images are row-major std::vector<double> (edgealign::Image, image.h:19-44).
// The one addition is a Context: the device, its stream and scratch arena.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "edgealign_b200.h"

namespace edgealign_b200 {

// ---- errors.h:14-75 -----------------------------------------------------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : Error {
    ParseError(const std::string& m, std::size_t off) : Error(m), offset_(off) {}
    std::size_t offset() const noexcept { return offset_; }
    std::size_t offset_;
};
struct SizeError : Error { using Error::Error; };
struct EmptyModelError : Error {
    EmptyModelError(const std::string& m, double mm) : Error(m), max_magnitude_(mm) {}
    double max_magnitude() const noexcept { return max_magnitude_; }
    double max_magnitude_;
};
struct BoundsError : Error { using Error::Error; };
struct BudgetError : Error { using Error::Error; };
struct GeometryError : Error { using Error::Error; };
struct InvalidArgument : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

inline void check(ea_status st) {
    if (st == EA_OK) return;
    const std::string m = ea_last_error();
    const double v = ea_last_error_value();
    switch (st) {
        case EA_ERR_INVALID_ARGUMENT: throw InvalidArgument(m);
        case EA_ERR_SIZE: throw SizeError(m);
        case EA_ERR_EMPTY_MODEL: throw EmptyModelError(m, v);
        case EA_ERR_BOUNDS: throw BoundsError(m);
        case EA_ERR_BUDGET: throw BudgetError(m);
        case EA_ERR_GEOMETRY: throw GeometryError(m);
        case EA_ERR_PARSE: throw ParseError(m, static_cast<std::size_t>(v));
        case EA_ERR_CUDA: throw CudaError(m);
        default: throw Error(m);
    }
}

// ---- plain data (reference struct names) ---------------------------------------
using Pose = ea_pose;
using PoseGrid = ea_pose_grid;
using GridCounts = ea_grid_counts;
using ScoreParams = ea_score_params;
using EdgeThresholds = ea_edge_thresholds;
using EdgePoint = ea_edge_point;
using ScoredPose = ea_scored_pose;
using SearchConfig = ea_search_config;
using SearchOutcome = ea_outcome;
using SceneSpec = ea_scene_spec;

struct Image {  // image.h:19-44
    int width = 0, height = 0;
    std::vector<double> data;
};
struct GradientField {  // gradient.h:17-36
    int width = 0, height = 0;
    std::vector<double> gx, gy, mag;
};
struct EdgeModel {  // edge_model.h:40-45
    std::vector<EdgePoint> points;
    double centroid_x = 0, centroid_y = 0;
    int source_level = 0;
};
using Pyramid = std::vector<Image>;

inline GridCounts grid_counts(const PoseGrid& g) {  // pose.h:52-67
    GridCounts c{};
    check(ea_compute_grid_counts(&g, &c));
    return c;
}
inline Pose pose_at(const PoseGrid& g, std::uint64_t i) {  // pose.h:77-92
    Pose p{};
    check(ea_pose_at(&g, i, &p));
    return p;
}

class Context {
public:
    explicit Context(int device = 0) {
        ea_ctx* c = nullptr;
        check(ea_ctx_create(device, &c));
        ctx_.reset(c);
    }
    ea_ctx* get() const { return ctx_.get(); }

private:
    struct Del {
        void operator()(ea_ctx* c) const { ea_ctx_destroy(c); }
    };
    std::unique_ptr<ea_ctx, Del> ctx_;
};

inline GradientField compute_gradients(Context& ctx, const Image& img) {  // gradient.cpp:12-27
    GradientField f{img.width, img.height, {}, {}, {}};
    const std::size_t n = static_cast<std::size_t>(img.width) * img.height;
    f.gx.resize(n);
    f.gy.resize(n);
    f.mag.resize(n);
    check(ea_compute_gradients(ctx.get(), img.data.data(), img.width, img.height, f.gx.data(),
                               f.gy.data(), f.mag.data()));
    return f;
}

inline Pyramid build_pyramid(Context& ctx, const Image& img, int levels) {  // image.cpp:274-291
    std::vector<int> dims(2 * static_cast<std::size_t>(levels > 0 ? levels : 1));
    check(ea_pyramid_dims(img.width, img.height, levels, dims.data()));
    std::size_t total = 0;
    for (int l = 0; l < levels; ++l) total += static_cast<std::size_t>(dims[2 * l]) * dims[2 * l + 1];
    std::vector<double> buf(total ? total : 1);
    check(ea_build_pyramid(ctx.get(), img.data.data(), img.width, img.height, levels, buf.data()));
    Pyramid p;
    std::size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        const std::size_t n = static_cast<std::size_t>(dims[2 * l]) * dims[2 * l + 1];
        p.push_back(Image{dims[2 * l], dims[2 * l + 1],
                          std::vector<double>(buf.begin() + off, buf.begin() + off + n)});
        off += n;
    }
    return p;
}

inline EdgeThresholds default_thresholds(const GradientField& f) {  // edge_model.cpp:17-24
    EdgeThresholds t{};
    check(ea_default_thresholds(f.mag.data(), f.width, f.height, &t));
    return t;
}

inline EdgeModel extract_edge_model(const GradientField& f, const EdgeThresholds& th,
                                    int level) {  // edge_model.cpp:53-149
    EdgeModel m;
    m.points.resize(static_cast<std::size_t>(f.width) * f.height);
    int n = 0;
    check(ea_extract_edge_model(f.gx.data(), f.gy.data(), f.mag.data(), f.width, f.height, &th,
                                level, m.points.data(), static_cast<int>(m.points.size()), &n,
                                &m.centroid_x, &m.centroid_y));
    m.points.resize(static_cast<std::size_t>(n));
    m.source_level = level;
    return m;
}

namespace detail {
struct Handles {
    ea_model* m = nullptr;
    ea_field* f = nullptr;
    ~Handles() {
        ea_model_free(m);
        ea_field_free(f);
    }
};
inline void upload(Context& ctx, const EdgeModel& model, const GradientField& field, Handles& h) {
    check(ea_model_create(ctx.get(), model.points.data(), static_cast<int>(model.points.size()),
                          model.centroid_x, model.centroid_y, model.source_level, &h.m));
    check(ea_field_upload(ctx.get(), field.gx.data(), field.gy.data(), field.mag.data(),
                          field.width, field.height, &h.f));
}
}  // namespace detail

// search_topk  search.cpp:155-167
inline std::vector<ScoredPose> search_topk(Context& ctx, const EdgeModel& model,
                                           const GradientField& field, const PoseGrid& grid,
                                           const ScoreParams& params, int k) {
    detail::Handles h;
    detail::upload(ctx, model, field, h);
    std::vector<ScoredPose> out(static_cast<std::size_t>(k > 0 ? k : 1));
    int n = 0;
    check(ea_search_topk(ctx.get(), h.m, h.f, &grid, &params, EA_BACKEND_CUDA, k, out.data(), &n));
    out.resize(static_cast<std::size_t>(n));
    return out;
}

// exhaustive_search  search.cpp:144-153
inline ScoredPose exhaustive_search(Context& ctx, const EdgeModel& model,
                                    const GradientField& field, const PoseGrid& grid,
                                    const ScoreParams& params) {
    return search_topk(ctx, model, field, grid, params, 1).at(0);
}

// score_map  search.cpp:169-202
inline std::vector<double> score_map(Context& ctx, const EdgeModel& model,
                                     const GradientField& field, const PoseGrid& grid,
                                     const ScoreParams& params, std::uint64_t max_cells) {
    detail::Handles h;
    detail::upload(ctx, model, field, h);
    const GridCounts c = grid_counts(grid);
    std::vector<double> out(c.nx * c.ny * c.nt <= max_cells ? c.nx * c.ny * c.nt : 1);
    check(ea_score_map(ctx.get(), h.m, h.f, &grid, &params, max_cells, out.data()));
    return out;
}

// coarse_to_fine  search.cpp:359-364
inline SearchOutcome coarse_to_fine(Context& ctx, const Pyramid& tmpl, const Pyramid& work,
                                    const SearchConfig& cfg) {
    std::vector<const double*> tp, wp;
    std::vector<int> td, wd;
    for (const Image& i : tmpl) {
        tp.push_back(i.data.data());
        td.push_back(i.width);
        td.push_back(i.height);
    }
    for (const Image& i : work) {
        wp.push_back(i.data.data());
        wd.push_back(i.width);
        wd.push_back(i.height);
    }
    SearchOutcome out{};
    check(ea_coarse_to_fine(ctx.get(), tp.data(), td.data(), static_cast<int>(tp.size()),
                            wp.data(), wd.data(), static_cast<int>(wp.size()), &cfg, &out));
    return out;
}

// Production detect: template models prepared once, host image per call.
class Detector {
public:
    Detector(Context& ctx, const Image& tmpl, const SearchConfig& cfg) : ctx_(ctx), cfg_(cfg) {
        ea_levels* lv = nullptr;
        check(ea_prepare_models(ctx.get(), tmpl.data.data(), tmpl.width, tmpl.height, &cfg, &lv));
        lv_.reset(lv);
    }
    SearchOutcome detect(const Image& img) {
        SearchOutcome out{};
        check(ea_detect(ctx_.get(), lv_.get(), img.data.data(), img.width, img.height, &cfg_,
                        &out));
        return out;
    }

private:
    struct Del {
        void operator()(ea_levels* l) const { ea_levels_free(l); }
    };
    Context& ctx_;
    SearchConfig cfg_;
    std::unique_ptr<ea_levels, Del> lv_;
};

// compose_scene  synth.cpp:178-300 (host)
inline std::pair<Image, Image> compose_scene(const SceneSpec& s, Pose* truth = nullptr,
                                             double* occluded = nullptr) {
    Image canvas{s.canvas_width, s.canvas_height,
                 std::vector<double>(static_cast<std::size_t>(s.canvas_width > 0 ? s.canvas_width : 1) *
                                     (s.canvas_height > 0 ? s.canvas_height : 1))};
    Image tmpl{s.template_size, s.template_size,
               std::vector<double>(static_cast<std::size_t>(s.template_size > 0 ? s.template_size : 1) *
                                   (s.template_size > 0 ? s.template_size : 1))};
    check(ea_compose_scene(&s, canvas.data.data(), tmpl.data.data(), truth, occluded));
    return {std::move(canvas), std::move(tmpl)};
}

}  // namespace edgealign_b200
