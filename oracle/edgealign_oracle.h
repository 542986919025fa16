/*
 * edgealign_oracle.h -- TEST INFRASTRUCTURE: the CPU parity oracle.
 *
 * A plain-C restatement of the reference search path (arxiv 2112.05576
 * reference, `edgealign`, proj/src/ (*.cpp)).  Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's cpu_baseline leg may load it, and only as
 * the checker: the product library never links or calls it.
 *
 * Parity is PINNED two ways (see tests/test_oracle_ref.py):
 *   - bit-exact agreement with the reference itself, compiled from its own
 *     sources by oracle/Makefile into oracle/_ref/libedgealign_ref.so;
 *   - the committed golden fixtures in tests/golden/ (generated from that
 *     build by tests/golden/make_golden.py) and the reference's own
 *     known-answer tests (proj/tests/ (*.cpp)) restated as pytest cases.
 *
 * Plain-data structs are the C-ABI vocabulary of include/edgealign_b200.h.
 * Status codes are ea_status values; orc_last_error() holds the message.
 */
#ifndef EDGEALIGN_ORACLE_H
#define EDGEALIGN_ORACLE_H

#include "../include/edgealign_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
double orc_last_error_value(void);

int orc_grid_counts(const ea_pose_grid* g, ea_grid_counts* out);
int orc_pose_at(const ea_pose_grid* g, uint64_t index, ea_pose* out);

int orc_downsample(const double* img, int w, int h, double* out);
int orc_max_pyramid_levels(int w, int h);
int orc_build_pyramid(const double* img, int w, int h, int levels, double* out);
int orc_compute_gradients(const double* img, int w, int h, double* gx, double* gy,
                          double* mag);

int orc_default_thresholds(const double* mag, int w, int h, ea_edge_thresholds* out);
int orc_extract_edge_model(const double* gx, const double* gy, const double* mag, int w,
                           int h, const ea_edge_thresholds* th, int level,
                           ea_edge_point* pts, int cap, int* n_out, double* cx,
                           double* cy);

int orc_point_vote(double dir_x, double dir_y, const double* gx, const double* gy,
                   const double* mag, int w, int h, int cx, int cy,
                   const ea_score_params* p, double* out);
int orc_rotate_model(const ea_edge_point* pts, int n, double theta, double* px,
                     double* py, double* dx, double* dy);
int orc_pose_score(const ea_edge_point* pts, int n, const ea_pose* pose, const double* gx,
                   const double* gy, const double* mag, int w, int h,
                   const ea_score_params* p, double* value, int* n_in);

/* run_search over theta indices [it_begin, it_end) with `threads` workers
 * (0 = all online CPUs); it_end = 0 means the whole grid. */
int orc_search_topk(const ea_edge_point* pts, int n, const double* gx, const double* gy,
                    const double* mag, int w, int h, const ea_pose_grid* g,
                    const ea_score_params* p, int k, uint64_t it_begin, uint64_t it_end,
                    int threads, ea_scored_pose* out, int* n_out);
int orc_score_map(const ea_edge_point* pts, int n, const double* gx, const double* gy,
                  const double* mag, int w, int h, const ea_pose_grid* g,
                  const ea_score_params* p, uint64_t max_cells, double* out);

/* search_levels from explicit per-level models and fields. */
int orc_search_levels(int num_levels, const ea_edge_point* const* models,
                      const int* model_n, const double* const* gx, const double* const* gy,
                      const double* const* mag, const int* dims,
                      const ea_search_config* cfg, int threads, ea_outcome* out);

int orc_render_template(int id, int size, double* out);
int orc_compose_scene(const ea_scene_spec* s, double* canvas, double* tmpl,
                      ea_pose* truth_pose, double* occluded_fraction);

#ifdef __cplusplus
}
#endif
#endif
