// host_synth.cpp -- deterministic synthetic scenes for tests and the bench
// (the reference's testkit, synth.cpp:24-300, SceneSpec synth.h:56-79).
//
// This is an input generator, not part of the detector: it stays on the host
// because it is libm-bound (pow/log/sin/cos/hypot) and must reproduce the
// reference's bytes exactly so that identical scenes reach the reference CPU
// path and the device path.  The template's edge centroid (which defines the
// stamped pose) is derived with a private host Sobel + the shared host edge
// extraction, as the reference's template_edge_centroid does (synth.cpp:169-174).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "host_model.h"

namespace eab {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kBackground = 200.0;  // synth.cpp:20
constexpr double kInk = 40.0;          // synth.cpp:21

// SplitMix64 with the constants and shifts of synth.h:26-49.
struct Rng {
    uint64_t s;
    bool spare_ok = false;
    double spare = 0.0;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
    double gauss() {  // Box-Muller pair, cosine branch first (synth.cpp:24-37)
        if (spare_ok) {
            spare_ok = false;
            return spare;
        }
        const double u1 = 1.0 - unit();
        const double u2 = unit();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * kPi * u2;
        spare = r * std::sin(a);
        spare_ok = true;
        return r * std::cos(a);
    }
};

inline int nearest_up(double v) { return (int)std::floor(v + 0.5); }

// Host Sobel (same operation order as the device kernel) for the template
// centroid only.
void sobel_host(const double* img, int w, int h, std::vector<double>& gx,
                std::vector<double>& gy, std::vector<double>& mag) {
    const size_t n = (size_t)w * h;
    gx.assign(n, 0.0);
    gy.assign(n, 0.0);
    mag.assign(n, 0.0);
    for (int y = 1; y + 1 < h; ++y) {
        for (int x = 1; x + 1 < w; ++x) {
            const double* up = img + (size_t)(y - 1) * w + x;
            const double* md = img + (size_t)y * w + x;
            const double* dn = img + (size_t)(y + 1) * w + x;
            const double ew = md[1] - md[-1];
            const double ns = dn[0] - up[0];
            const double sx = ((up[1] - up[-1]) + (ew + ew)) + (dn[1] - dn[-1]);
            const double sy = ((dn[-1] - up[-1]) + (ns + ns)) + (dn[1] - up[1]);
            const size_t o = (size_t)y * w + x;
            gx[o] = sx;
            gy[o] = sy;
            mag[o] = std::sqrt(sx * sx + sy * sy);
        }
    }
}

}  // namespace

void host_render_template(int id, int size, double* img) {
    if (size < 16) fail(EA_ERR_SIZE, "template size must be >= 16, got " + std::to_string(size));
    if (id < EA_TEMPLATE_RECTANGLE || id > EA_TEMPLATE_CROSS) {
        fail(EA_ERR_INVALID_ARGUMENT, "unknown template id " + std::to_string(id) +
                                          " (expected rectangle|ring|l_bracket|cross)");
    }
    std::fill(img, img + (size_t)size * size, kBackground);
    auto ink = [&](int x, int y) { img[(size_t)y * size + x] = kInk; };
    const int inset = std::max(2, size / 8);
    const int a = inset, b = size - 1 - inset;
    if (id == EA_TEMPLATE_RECTANGLE) {  // 2-px outline
        for (int t = a; t <= b; ++t) {
            for (int d = 0; d < 2; ++d) {
                ink(t, a + d);
                ink(t, b - d);
            }
        }
        for (int t = a; t <= b; ++t) {
            for (int d = 0; d < 2; ++d) {
                ink(a + d, t);
                ink(b - d, t);
            }
        }
    } else if (id == EA_TEMPLATE_RING) {  // |dist - radius| <= 1
        const double c = (size - 1) / 2.0;
        const double radius = (b - a) / 2.0;
        for (int y = 0; y < size; ++y)
            for (int x = 0; x < size; ++x)
                if (std::fabs(std::hypot(x - c, y - c) - radius) <= 1.0) ink(x, y);
    } else if (id == EA_TEMPLATE_L_BRACKET) {  // left bar + bottom bar
        for (int t = a; t <= b; ++t) {
            ink(a, t);
            ink(a + 1, t);
        }
        for (int t = a; t <= b; ++t) {
            ink(t, b);
            ink(t, b - 1);
        }
    } else {  // cross through the centre
        const int c = size / 2;
        for (int t = a; t <= b; ++t) {
            ink(c - 1, t);
            ink(c, t);
        }
        for (int t = a; t <= b; ++t) {
            ink(t, c - 1);
            ink(t, c);
        }
    }
}

namespace {

// One template placed at a pose: the rendered template, its edge centroid
// (template_edge_centroid, synth.cpp:169-174) and the forward-mapped bbox,
// which must stay on the canvas (synth.cpp:196-217).
struct Stamp {
    int T = 0;
    std::vector<double> tmpl;
    std::vector<ea_edge_point> pts;
    double ccx = 0.0, ccy = 0.0;
    ea_pose pose{};
    double c = 1.0, sn = 0.0;
    double lo_x = 0, hi_x = 0, lo_y = 0, hi_y = 0;
};

Stamp make_stamp(int template_id, int T, ea_pose pose, int W, int H) {
    Stamp st;
    st.T = T;
    st.pose = pose;
    st.tmpl.assign((size_t)std::max(T, 1) * std::max(T, 1), 0.0);
    host_render_template(template_id, T, st.tmpl.data());
    std::vector<double> tgx, tgy, tmag;
    sobel_host(st.tmpl.data(), T, T, tgx, tgy, tmag);
    st.pts = host_extract_edge_model(tgx.data(), tgy.data(), tmag.data(), T, T,
                                     host_default_thresholds(tmag.data(), tmag.size()), &st.ccx,
                                     &st.ccy);
    st.c = std::cos(pose.theta);
    st.sn = std::sin(pose.theta);
    st.lo_x = st.lo_y = 1e300;
    st.hi_x = st.hi_y = -1e300;
    for (int corner = 0; corner < 4; ++corner) {
        const double tx = (corner & 1 ? (double)(T - 1) : 0.0) - st.ccx;
        const double ty = (corner & 2 ? (double)(T - 1) : 0.0) - st.ccy;
        const double px = (st.c * tx - st.sn * ty) + pose.ux;
        const double py = (st.sn * tx + st.c * ty) + pose.uy;
        st.lo_x = std::min(st.lo_x, px);
        st.hi_x = std::max(st.hi_x, px);
        st.lo_y = std::min(st.lo_y, py);
        st.hi_y = std::max(st.hi_y, py);
    }
    if (st.lo_x < 0.0 || st.lo_y < 0.0 || st.hi_x > W - 1.0 || st.hi_y > H - 1.0) {
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "transformed template leaves the canvas (bbox [%f, %f] .. [%f, %f])",
                      st.lo_x, st.lo_y, st.hi_x, st.hi_y);
        fail(EA_ERR_GEOMETRY, buf);
    }
    return st;
}

void check_spec(const ea_scene_spec& s) {
    if (s.canvas_width < 16 || s.canvas_height < 16)
        fail(EA_ERR_INVALID_ARGUMENT, "canvas must be at least 16x16");
    if (!(s.gain > 0.0) || !(s.gamma > 0.0))
        fail(EA_ERR_INVALID_ARGUMENT, "illumination gain and gamma must be positive");
    if (s.noise_sigma < 0.0) fail(EA_ERR_INVALID_ARGUMENT, "noise_sigma must be >= 0");
}

// Background + clutter line segments (draw_clutter, synth.cpp:134-165).
void draw_background(const ea_scene_spec& s, double* canvas) {
    const int W = s.canvas_width, H = s.canvas_height;
    std::fill(canvas, canvas + (size_t)W * H, kBackground);
    Rng rng(s.clutter_seed);
    for (int seg = 0; seg < s.clutter_segments; ++seg) {
        const double ax = rng.unit() * W, ay = rng.unit() * H;
        const double bx = rng.unit() * W, by = rng.unit() * H;
        const double value = rng.unit() * 255.0;
        const int pen = 1 + (int)(rng.next() & 1ULL);
        const int steps = 1 + (int)(2.0 * std::hypot(bx - ax, by - ay));
        for (int i = 0; i <= steps; ++i) {
            const double t = (double)i / steps;
            const int px = nearest_up(ax + t * (bx - ax));
            const int py = nearest_up(ay + t * (by - ay));
            for (int dy = 0; dy < pen; ++dy)
                for (int dx = 0; dx < pen; ++dx) {
                    const int X = px + dx, Y = py + dy;
                    if (X >= 0 && X < W && Y >= 0 && Y < H) canvas[(size_t)Y * W + X] = value;
                }
        }
    }
}

// Inverse-mapped stamp, template lookup rounds half down (synth.cpp:224-244).
void paste(const Stamp& st, int W, int H, double* canvas) {
    const int x_lo = std::max(0, (int)std::floor(st.lo_x) - 1);
    const int y_lo = std::max(0, (int)std::floor(st.lo_y) - 1);
    const int x_hi = std::min(W - 1, (int)std::ceil(st.hi_x) + 1);
    const int y_hi = std::min(H - 1, (int)std::ceil(st.hi_y) + 1);
    const int T = st.T;
    for (int y = y_lo; y <= y_hi; ++y) {
        for (int x = x_lo; x <= x_hi; ++x) {
            const double rx = x - st.pose.ux, ry = y - st.pose.uy;
            const int ix = (int)std::ceil(((st.c * rx + st.sn * ry) + st.ccx) - 0.5);
            const int iy = (int)std::ceil(((-st.sn * rx + st.c * ry) + st.ccy) - 0.5);
            if (ix < 0 || ix >= T || iy < 0 || iy >= T) continue;
            const double v = st.tmpl[(size_t)iy * T + ix];
            if (v != kBackground) canvas[(size_t)y * W + x] = v;
        }
    }
}

// Occluder, gamma then gain/bias, noise (synth.cpp:246-285).
void finish(const ea_scene_spec& s, double* canvas) {
    const int W = s.canvas_width, H = s.canvas_height;
    if (s.has_occluder) {
        const int x_lo = std::max(0, s.occ_x), y_lo = std::max(0, s.occ_y);
        const int x_hi = std::min(W - 1, s.occ_x + s.occ_w - 1);
        const int y_hi = std::min(H - 1, s.occ_y + s.occ_h - 1);
        for (int y = y_lo; y <= y_hi; ++y)
            for (int x = x_lo; x <= x_hi; ++x) canvas[(size_t)y * W + x] = s.occ_fill;
    }
    for (size_t i = 0; i < (size_t)W * H; ++i) {
        const double v = canvas[i];
        const double g = (s.gamma == 1.0) ? v : 255.0 * std::pow(v / 255.0, s.gamma);
        canvas[i] = s.gain * g + s.bias;
    }
    if (s.noise_sigma > 0.0) {
        Rng rng(s.noise_seed);
        for (size_t i = 0; i < (size_t)W * H; ++i) canvas[i] += s.noise_sigma * rng.gauss();
    }
}

double occluded_fraction(const ea_scene_spec& s, const Stamp& st) {
    if (!s.has_occluder) return 0.0;
    int hit = 0;
    for (const ea_edge_point& p : st.pts) {
        const int ix = nearest_up((st.c * p.x_rel - st.sn * p.y_rel) + st.pose.ux);
        const int iy = nearest_up((st.sn * p.x_rel + st.c * p.y_rel) + st.pose.uy);
        if (ix >= s.occ_x && ix < s.occ_x + s.occ_w && iy >= s.occ_y && iy < s.occ_y + s.occ_h)
            ++hit;
    }
    return (double)hit / (double)st.pts.size();
}

}  // namespace

void host_compose_scene(const ea_scene_spec& s, double* canvas, double* tmpl,
                        ea_pose* truth_pose, double* occluded) {
    check_spec(s);
    const Stamp st = make_stamp(s.template_id, s.template_size, s.true_pose, s.canvas_width,
                                s.canvas_height);
    std::copy(st.tmpl.begin(), st.tmpl.end(), tmpl);
    draw_background(s, canvas);
    paste(st, s.canvas_width, s.canvas_height, canvas);
    finish(s, canvas);
    *truth_pose = st.pose;
    *occluded = occluded_fraction(s, st);
}

void host_compose_multi(const ea_scene_spec& s, const ea_stamp* stamps, int n, double* canvas) {
    check_spec(s);
    if (n < 0 || (n > 0 && !stamps)) fail(EA_ERR_INVALID_ARGUMENT, "bad stamp list");
    std::vector<Stamp> sts;
    sts.reserve(n);
    for (int i = 0; i < n; ++i)
        sts.push_back(make_stamp(stamps[i].template_id, stamps[i].template_size, stamps[i].pose,
                                 s.canvas_width, s.canvas_height));
    draw_background(s, canvas);
    for (const Stamp& st : sts) paste(st, s.canvas_width, s.canvas_height, canvas);
    finish(s, canvas);
}

}  // namespace eab
