// host_model.cpp -- template-side helpers on the host.
//
// The template side (prepare_levels, search.cpp:208-238) runs on the device:
// Sobel, peak, NMS, hysteresis and emission (model_kernels.cu, SURVEY.md
// §8(f)-1).  This file keeps (a) the reference's orientation bin with the
// host libm's atan2 -- the same library the reference links -- for the few
// pixels whose bin the device cannot decide exactly (host_nms_state), and (b)
// a whole host extraction behind ea_extract_edge_model, the host-array entry
// point of the C-ABI (edge_model.cpp:17-149).
//
// Compiled with -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <deque>
#include <string>
#include <vector>

#include "host_model.h"

namespace eab {

namespace {
constexpr double kPi = 3.14159265358979323846;  // pose.h:21

// Gradient direction folded into [0, pi) and binned at 0/45/90/135 degrees,
// boundaries to the lower bin (edge_model.cpp:34-45).
int direction_bin(double gx, double gy) {
    double a = std::atan2(gy, gx);
    if (a < 0.0) a += kPi;
    const double step = kPi / 8.0;
    if (a <= step) return 0;
    if (a <= 3.0 * step) return 1;
    if (a <= 5.0 * step) return 2;
    if (a <= 7.0 * step) return 3;
    return 0;
}
}  // namespace

unsigned char host_nms_state(const double* gx, const double* gy, const double* mag, int w, int x,
                             int y, double low, double high) {
    static const int step_x[4] = {1, 1, 0, -1};
    static const int step_y[4] = {0, 1, 1, 1};
    const size_t o = (size_t)y * w + x;
    const double m = mag[o];
    if (m <= 0.0 || m < low) return 0;
    const int b = direction_bin(gx[o], gy[o]);
    const double ahead = mag[(size_t)(y + step_y[b]) * w + (x + step_x[b])];
    const double behind = mag[(size_t)(y - step_y[b]) * w + (x - step_x[b])];
    if (m > ahead && m >= behind) return m >= high ? 2 : 1;
    return 0;
}

ea_edge_thresholds host_default_thresholds(const double* mag, size_t count) {
    double peak = 0.0;
    for (size_t i = 0; i < count; ++i) peak = mag[i] > peak ? mag[i] : peak;
    const double high = 0.3 * peak;
    return ea_edge_thresholds{0.5 * high, high};
}

std::vector<ea_edge_point> host_extract_edge_model(const double* gx, const double* gy,
                                                   const double* mag, int w, int h,
                                                   const ea_edge_thresholds& th,
                                                   double* centroid_x, double* centroid_y) {
    if (th.low < 0.0 || th.low > th.high) {
        fail(EA_ERR_INVALID_ARGUMENT, "edge thresholds need 0 <= low <= high");
    }
    const size_t total = (size_t)w * h;
    double peak = 0.0;
    for (size_t i = 0; i < total; ++i) peak = mag[i] > peak ? mag[i] : peak;

    // 0 = suppressed, 1 = weak, 2 = strong.  A pixel survives when it beats
    // its +direction neighbour strictly and its -direction one non-strictly.
    static const int step_x[4] = {1, 1, 0, -1};
    static const int step_y[4] = {0, 1, 1, 1};
    std::vector<uint8_t> cls(total, 0);
    for (int y = 1; y + 1 < h; ++y) {
        for (int x = 1; x + 1 < w; ++x) {
            const size_t o = (size_t)y * w + x;
            const double m = mag[o];
            if (m <= 0.0 || m < th.low) continue;
            const int b = direction_bin(gx[o], gy[o]);
            const double ahead = mag[(size_t)(y + step_y[b]) * w + (x + step_x[b])];
            const double behind = mag[(size_t)(y - step_y[b]) * w + (x - step_x[b])];
            if (m > ahead && m >= behind) cls[o] = m >= th.high ? 2 : 1;
        }
    }
    // Hysteresis: every weak pixel 8-connected to a strong one is kept.
    std::vector<uint8_t> keep(total, 0);
    std::deque<size_t> frontier;
    for (size_t s = 0; s < total; ++s) {
        if (cls[s] != 2 || keep[s]) continue;
        keep[s] = 1;
        frontier.push_back(s);
        while (!frontier.empty()) {
            const size_t p = frontier.front();
            frontier.pop_front();
            const int px = (int)(p % (size_t)w), py = (int)(p / (size_t)w);
            for (int dy = -1; dy <= 1; ++dy) {
                const int qy = py + dy;
                if (qy < 0 || qy >= h) continue;
                for (int dx = -1; dx <= 1; ++dx) {
                    const int qx = px + dx;
                    if ((dx | dy) == 0 || qx < 0 || qx >= w) continue;
                    const size_t q = (size_t)qy * w + qx;
                    if (!keep[q] && cls[q]) {
                        keep[q] = 1;
                        frontier.push_back(q);
                    }
                }
            }
        }
    }
    // Row-major emission (the order scores are summed in) and the centroid.
    size_t count = 0;
    double sx = 0.0, sy = 0.0;
    for (size_t i = 0; i < total; ++i) {
        if (!keep[i]) continue;
        ++count;
        sx += (double)(i % (size_t)w);
        sy += (double)(i / (size_t)w);
    }
    if (count == 0) {
        char buf[128];
        std::snprintf(buf, sizeof buf,
                      "edge extraction produced an empty model (max gradient magnitude %f)", peak);
        fail(EA_ERR_EMPTY_MODEL, buf, peak);
    }
    const double cx = sx / (double)count, cy = sy / (double)count;
    std::vector<ea_edge_point> pts;
    pts.reserve(count);
    for (size_t i = 0; i < total; ++i) {
        if (!keep[i]) continue;
        const double m = mag[i];
        pts.push_back(ea_edge_point{(double)(i % (size_t)w) - cx, (double)(i / (size_t)w) - cy,
                                    gx[i] / m, gy[i] / m, m});
    }
    *centroid_x = cx;
    *centroid_y = cy;
    return pts;
}

}  // namespace eab
