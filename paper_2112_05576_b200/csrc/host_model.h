// host_model.h -- host-side helpers of libedgealign_b200 (template side and
// the synthetic scene generator).
#pragma once

#include <cstdint>
#include <vector>

#include "failure.h"

namespace eab {


ea_edge_thresholds host_default_thresholds(const double* mag, size_t count);
std::vector<ea_edge_point> host_extract_edge_model(const double* gx, const double* gy,
                                                   const double* mag, int w, int h,
                                                   const ea_edge_thresholds& th,
                                                   double* centroid_x, double* centroid_y);

// NMS state (0 out, 1 weak, 2 strong) of interior pixel (x, y) with the
// reference's atan2 bins (edge_model.cpp:34-45, 77-90); the device extraction
// asks for the pixels whose bin it cannot decide without glibc.
unsigned char host_nms_state(const double* gx, const double* gy, const double* mag, int w, int x,
                             int y, double low, double high);

// Synthetic scenes (synth.cpp:24-300), host only: libm-dependent generator.
void host_render_template(int id, int size, double* out);
void host_compose_multi(const ea_scene_spec& s, const ea_stamp* stamps, int n, double* canvas);
void host_compose_scene(const ea_scene_spec& s, double* canvas, double* tmpl,
                        ea_pose* truth_pose, double* occluded_fraction);

// Netpbm codecs and the model overlay (host_io.cpp, image.cpp:26-219).
uint8_t host_luminance_to_byte(double v);
void host_load_pgm(const uint8_t* bytes, size_t size, std::vector<double>* out, int* w, int* h);
std::vector<uint8_t> host_save_pgm(const double* img, int w, int h);
std::vector<uint8_t> host_save_ppm(const double* img, int w, int h, const int* xy, int n_xy,
                                   uint8_t r, uint8_t g, uint8_t b);
void host_overlay_points(const ea_edge_point* pts, int n, const ea_pose& pose, int* xy);

}  // namespace eab
