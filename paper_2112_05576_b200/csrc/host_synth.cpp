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

void host_compose_scene(const ea_scene_spec& s, double* canvas, double* tmpl,
                        ea_pose* truth_pose, double* occluded_fraction) {
    if (s.canvas_width < 16 || s.canvas_height < 16)
        fail(EA_ERR_INVALID_ARGUMENT, "canvas must be at least 16x16");
    if (!(s.gain > 0.0) || !(s.gamma > 0.0))
        fail(EA_ERR_INVALID_ARGUMENT, "illumination gain and gamma must be positive");
    if (s.noise_sigma < 0.0) fail(EA_ERR_INVALID_ARGUMENT, "noise_sigma must be >= 0");
    const int W = s.canvas_width, H = s.canvas_height, T = s.template_size;

    host_render_template(s.template_id, T, tmpl);
    std::vector<double> tgx, tgy, tmag;
    sobel_host(tmpl, T, T, tgx, tgy, tmag);
    double ccx = 0.0, ccy = 0.0;
    const std::vector<ea_edge_point> pts = host_extract_edge_model(
        tgx.data(), tgy.data(), tmag.data(), T, T,
        host_default_thresholds(tmag.data(), tmag.size()), &ccx, &ccy);

    const ea_pose pose = s.true_pose;
    const double c = std::cos(pose.theta), sn = std::sin(pose.theta);
    // Forward-mapped template corners must stay on the canvas.
    double lo_x = 1e300, hi_x = -1e300, lo_y = 1e300, hi_y = -1e300;
    for (int corner = 0; corner < 4; ++corner) {
        const double tx = (corner & 1 ? (double)(T - 1) : 0.0) - ccx;
        const double ty = (corner & 2 ? (double)(T - 1) : 0.0) - ccy;
        const double px = (c * tx - sn * ty) + pose.ux;
        const double py = (sn * tx + c * ty) + pose.uy;
        lo_x = std::min(lo_x, px);
        hi_x = std::max(hi_x, px);
        lo_y = std::min(lo_y, py);
        hi_y = std::max(hi_y, py);
    }
    if (lo_x < 0.0 || lo_y < 0.0 || hi_x > W - 1.0 || hi_y > H - 1.0) {
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "transformed template leaves the canvas (bbox [%f, %f] .. [%f, %f])", lo_x,
                      lo_y, hi_x, hi_y);
        fail(EA_ERR_GEOMETRY, buf);
    }

    std::fill(canvas, canvas + (size_t)W * H, kBackground);
    {  // clutter line segments
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
    {  // inverse-mapped stamp, template lookup rounds half down
        const int x_lo = std::max(0, (int)std::floor(lo_x) - 1);
        const int y_lo = std::max(0, (int)std::floor(lo_y) - 1);
        const int x_hi = std::min(W - 1, (int)std::ceil(hi_x) + 1);
        const int y_hi = std::min(H - 1, (int)std::ceil(hi_y) + 1);
        for (int y = y_lo; y <= y_hi; ++y) {
            for (int x = x_lo; x <= x_hi; ++x) {
                const double rx = x - pose.ux, ry = y - pose.uy;
                const int ix = (int)std::ceil(((c * rx + sn * ry) + ccx) - 0.5);
                const int iy = (int)std::ceil(((-sn * rx + c * ry) + ccy) - 0.5);
                if (ix < 0 || ix >= T || iy < 0 || iy >= T) continue;
                const double v = tmpl[(size_t)iy * T + ix];
                if (v != kBackground) canvas[(size_t)y * W + x] = v;
            }
        }
    }
    if (s.has_occluder) {
        const int x_lo = std::max(0, s.occ_x), y_lo = std::max(0, s.occ_y);
        const int x_hi = std::min(W - 1, s.occ_x + s.occ_w - 1);
        const int y_hi = std::min(H - 1, s.occ_y + s.occ_h - 1);
        for (int y = y_lo; y <= y_hi; ++y)
            for (int x = x_lo; x <= x_hi; ++x) canvas[(size_t)y * W + x] = s.occ_fill;
    }
    for (size_t i = 0; i < (size_t)W * H; ++i) {  // gamma, then gain/bias
        const double v = canvas[i];
        const double g = (s.gamma == 1.0) ? v : 255.0 * std::pow(v / 255.0, s.gamma);
        canvas[i] = s.gain * g + s.bias;
    }
    if (s.noise_sigma > 0.0) {
        Rng rng(s.noise_seed);
        for (size_t i = 0; i < (size_t)W * H; ++i) canvas[i] += s.noise_sigma * rng.gauss();
    }
    *truth_pose = pose;
    *occluded_fraction = 0.0;
    if (s.has_occluder) {
        int hit = 0;
        for (const ea_edge_point& p : pts) {
            const int ix = nearest_up((c * p.x_rel - sn * p.y_rel) + pose.ux);
            const int iy = nearest_up((sn * p.x_rel + c * p.y_rel) + pose.uy);
            if (ix >= s.occ_x && ix < s.occ_x + s.occ_w && iy >= s.occ_y && iy < s.occ_y + s.occ_h)
                ++hit;
        }
        *occluded_fraction = (double)hit / (double)pts.size();
    }
}

}  // namespace eab
