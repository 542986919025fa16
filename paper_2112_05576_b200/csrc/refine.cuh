// refine.cuh -- device-resident beam refinement (search.cpp:254-357).
#pragma once

#include "common.cuh"

namespace eab {

// One beam entry: pose in the current level's coordinates (BeamEntry,
// search.cpp:242-246) + the kt path that indexes its theta table.
struct BeamDev {
    double ux, uy, theta, score;
    unsigned long long top_index;
    int path;
    int _pad;
};

struct RefineArgs {
    const double* pts;  // model SoA x|y|dx|dy at this level
    int n;
    const double* gx;
    const double* gy;
    const double* mag;
    int W, H;
    int vote_R, ignore;
    double eps;
    int R, side, topk, max_parents, chunk, level, trace_slot;
    double step_x, step_y, min_score;
    const double* table;  // (theta, cos, sin) per path of this level
    const BeamDev* beam;  // parents
    const int* beam_count;
    BeamDev* beam_out;
    int* beam_count_out;
    double* votes;        // [entry][point] vote rows when they do not fit shared memory
    int votes_in_smem;    // set by launch_refine_level
    double* entries;      // [entry] score, ux, uy, theta
    long long* keys;      // order_key(score), LLONG_MIN for duplicates
    int* dup;             // [entry] an earlier entry has the same pose
    ea_outcome* outcome;  // device copy of the result
};

// threads per pose (refine_entry_kernel): 625 CTAs of a k = 5, radius 2
// level fit one wave at 60 registers x 192 threads (5 CTAs per SM); 256
// threads (4 per SM) left 33 CTAs for a second wave -- 21.1 -> 17.7 us per
// level on cfg3 (128: 18.0, 96: 18.6, 64: 20.9)
constexpr int kRefineThreads = 192;
constexpr size_t kRefineSmemMax = 96 * 1024;      // vote rows in smem up to this size
void launch_refine_level(ea_ctx* ctx, const RefineArgs& a);

// Top-level grid + search params the seed kernel needs.
struct SeedArgs {
    double x0, dx, y0, dy, t0, dt;
    unsigned long long nx, ny;
    int top_level;
    double min_score;
};
void launch_seed_beam(ea_ctx* ctx, const double* top_score, const unsigned long long* top_index,
                      const int* n_top, const SeedArgs& s, BeamDev* beam, int* beam_count,
                      ea_outcome* out);

}  // namespace eab
