// model.cuh -- device edge-model extraction (model_kernels.cu).
#pragma once

#include "common.cuh"

namespace eab {

// Device scratch of one extraction.
struct ModelScratch {
    unsigned long long peak_bits;  // max magnitude as a bit pattern
    int use_default;               // thresholds from the peak (default_thresholds)
    int n_amb;                     // pixels whose orientation bin the host decides
    int n_kept;                    // model points
    int _pad;
    double low, high;              // thresholds in use
    double cx, cy;                 // centroid
};

void launch_magmax(ea_ctx* ctx, const double* mag, size_t total, ModelScratch* ms);
void launch_nms(ea_ctx* ctx, const double* gx, const double* gy, const double* mag, int w, int h,
                ModelScratch* ms, unsigned char* state, unsigned char* kept, int* amb_list);
void launch_hysteresis_emit(ea_ctx* ctx, const double* gx, const double* gy, const double* mag,
                            const unsigned char* state, unsigned char* kept, int w, int h,
                            ModelScratch* ms, ea_edge_point* out);

}  // namespace eab
