// host_io.cpp -- Netpbm codecs on either side of the path:
// PGM P2/P5 in, PGM P5 / PPM P6 out, the export rounding, and the overlay
// of a model at a pose (image.cpp:26-219, image.h:52-80; the overlay the
// reference's CLI spec draws, SPEC.md cli-bench cmd_detect).  Bytes in,
// bytes out -- file I/O stays with the caller.  Host code: parsing is
// branchy byte work with nothing to parallelise.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "host_model.h"

namespace eab {

namespace {

bool pgm_space(uint8_t c) {
    return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\f' || c == '\v';
}

[[noreturn]] void parse_fail(const std::string& msg, size_t offset) {
    fail(EA_ERR_PARSE, msg + " (byte offset " + std::to_string(offset) + ")", (double)offset);
}

// Header / plain-payload tokenizer; errors carry the byte offset.
struct Cursor {
    const uint8_t* b;
    size_t n, pos = 0;
    bool eof() const { return pos >= n; }
    void skip() {
        while (!eof()) {
            if (pgm_space(b[pos])) {
                ++pos;
            } else if (b[pos] == '#') {
                while (!eof() && b[pos] != '\n') ++pos;
            } else {
                break;
            }
        }
    }
    long number(const char* what, long limit) {
        skip();
        if (eof()) parse_fail(std::string("truncated header: missing ") + what, pos);
        if (b[pos] < '0' || b[pos] > '9')
            parse_fail(std::string("expected unsigned integer for ") + what, pos);
        const size_t start = pos;
        long v = 0;
        while (!eof() && b[pos] >= '0' && b[pos] <= '9') {
            v = v * 10 + (b[pos] - '0');
            if (v > limit)
                parse_fail(std::string(what) + " exceeds limit " + std::to_string(limit), start);
            ++pos;
        }
        return v;
    }
};

void header(std::vector<uint8_t>& out, const char* magic, int w, int h) {
    char buf[64];
    const int k = std::snprintf(buf, sizeof buf, "%s\n%d %d\n255\n", magic, w, h);
    out.insert(out.end(), buf, buf + k);
}

}  // namespace

uint8_t host_luminance_to_byte(double v) {
    if (!(v > 0.0)) return 0;
    if (v >= 255.0) return 255;
    return (uint8_t)std::floor(v + 0.5);
}

void host_load_pgm(const uint8_t* bytes, size_t size, std::vector<double>* out, int* w, int* h) {
    if (size < 2 || bytes[0] != 'P') parse_fail("not a PGM stream: missing P2/P5 magic", 0);
    const char kind = (char)bytes[1];
    if (kind != '2' && kind != '5')
        parse_fail(std::string("unsupported magic \"P") + kind + "\"; only P2 and P5 are accepted",
                   0);
    Cursor c{bytes, size, 2};
    const long width = c.number("width", 1 << 20);
    const long height = c.number("height", 1 << 20);
    if (width < 1 || height < 1) parse_fail("image dimensions must be at least 1x1", c.pos);
    c.skip();
    const size_t maxval_at = c.pos;
    const long maxval = c.number("maxval", 65535);
    if (maxval < 1 || maxval > 255)
        parse_fail("unsupported maxval " + std::to_string(maxval) + " (only <= 255)", maxval_at);
    const size_t count = (size_t)width * (size_t)height;
    *w = (int)width;
    *h = (int)height;
    if (out) out->assign(count, 0.0);
    if (kind == '5') {
        if (c.eof() || !pgm_space(bytes[c.pos]))
            parse_fail("expected single whitespace before binary payload", c.pos);
        ++c.pos;
        if (size - c.pos < count)
            parse_fail("truncated pixel payload: need " + std::to_string(count) + " bytes, have " +
                           std::to_string(size - c.pos),
                       c.pos);
        for (size_t i = 0; i < count; ++i) {
            const uint8_t v = bytes[c.pos + i];
            if (v > maxval)
                parse_fail("pixel value " + std::to_string(v) + " exceeds maxval " +
                               std::to_string(maxval),
                           c.pos + i);
            if (out) (*out)[i] = (double)v;
        }
    } else {
        for (size_t i = 0; i < count; ++i) {
            const long v = c.number("pixel value", 255);
            if (v > maxval)
                parse_fail("pixel value " + std::to_string(v) + " exceeds maxval " +
                               std::to_string(maxval),
                           c.pos);
            if (out) (*out)[i] = (double)v;
        }
    }
}

std::vector<uint8_t> host_save_pgm(const double* img, int w, int h) {
    if (w < 1 || h < 1)
        fail(EA_ERR_SIZE, "image dimensions must be at least 1x1, got " + std::to_string(w) + "x" +
                              std::to_string(h));
    std::vector<uint8_t> out;
    out.reserve((size_t)w * h + 32);
    header(out, "P5", w, h);
    for (size_t i = 0; i < (size_t)w * h; ++i) out.push_back(host_luminance_to_byte(img[i]));
    return out;
}

std::vector<uint8_t> host_save_ppm(const double* img, int w, int h, const int* xy, int n_xy,
                                   uint8_t r, uint8_t g, uint8_t b) {
    if (w < 1 || h < 1)
        fail(EA_ERR_SIZE, "image dimensions must be at least 1x1, got " + std::to_string(w) + "x" +
                              std::to_string(h));
    std::vector<uint8_t> out;
    out.reserve((size_t)w * h * 3 + 32);
    header(out, "P6", w, h);
    const size_t base = out.size();
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        const uint8_t v = host_luminance_to_byte(img[i]);
        out.push_back(v);
        out.push_back(v);
        out.push_back(v);
    }
    for (int i = 0; i < n_xy; ++i) {
        const int x = xy[2 * i], y = xy[2 * i + 1];
        if (x < 0 || x >= w || y < 0 || y >= h) continue;
        const size_t at = base + 3 * ((size_t)y * w + x);
        out[at] = r;
        out[at + 1] = g;
        out[at + 2] = b;
    }
    return out;
}

// Overlay pixels of a model at a pose: each point's projection exactly as the
// scorer computes it (rotate_model similarity.cpp:79-80, then + u and
// floor(v + 0.5), similarity.cpp:104-108).
void host_overlay_points(const ea_edge_point* pts, int n, const ea_pose& pose, int* xy) {
    const double cos_t = std::cos(pose.theta), sin_t = std::sin(pose.theta);
    for (int i = 0; i < n; ++i) {
        const double px = cos_t * pts[i].x_rel - sin_t * pts[i].y_rel;
        const double py = sin_t * pts[i].x_rel + cos_t * pts[i].y_rel;
        xy[2 * i] = (int)std::floor((px + pose.ux) + 0.5);
        xy[2 * i + 1] = (int)std::floor((py + pose.uy) + 0.5);
    }
}

}  // namespace eab
