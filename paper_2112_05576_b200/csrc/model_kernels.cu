// model_kernels.cu -- template-side edge model extraction on the device
// (extract_edge_model edge_model.cpp:53-149, default_thresholds 17-24;
// SURVEY.md §8(f)-1).
//
//   magmax_kernel      peak magnitude (bit-pattern max of non-negative doubles)
//   nms_kernel         direction-binned non-maximum suppression -> state
//                      0 out / 1 weak / 2 strong; pixels whose orientation bin
//                      cannot be decided without glibc's atan2 go to a list
//   hysteresis_kernel  8-connected flood from strong through weak pixels,
//                      iterated to the fixpoint in one CTA
//   emit_kernel        row-major compaction + centroid + model points
//
// Orientation bins without atan2: the reference folds atan2(gy, gx) into
// [0, pi) and compares it with k*pi/8 (edge_model.cpp:34-45).  For a direction
// (X, Y) with Y > 0 (gy < 0 folded to (-gx, -gy)), phi > k*pi/8 is the sign of
// a cross product with the boundary direction, i.e. of Y - t*X, t*Y - X,
// -t*Y - X and -(Y + t*X) with t = tan(pi/8).  When |value| is within
// 1e-12 * (|X| + |Y|) of zero (far wider than atan2's error, the rounding of
// pi/8 and of the fold) the pixel is listed and the host decides it with the
// reference's own formula and libm.  gy == 0 is bin 0 for every gx (atan2
// gives +-0 or +-pi, folded to 0 or pi).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.cuh"
#include "model.cuh"

namespace eab {

__global__ void __launch_bounds__(256) magmax_kernel(const double* __restrict__ mag,
                                                     size_t total, ModelScratch* ms) {
    using Reduce = cub::BlockReduce<unsigned long long, 256>;
    __shared__ typename Reduce::TempStorage tmp;
    unsigned long long best = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (size_t)gridDim.x * blockDim.x) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(__ldg(mag + i));
        best = b > best ? b : best;  // mag >= +0: bit order == value order
    }
    best = Reduce(tmp).Reduce(best, cub::Max());
    if (threadIdx.x == 0) atomicMax(&ms->peak_bits, best);
}

__device__ __forceinline__ int orientation_bin_dev(double gx, double gy, bool* amb) {
    if (gy == 0.0) return 0;
    const double X = gy > 0.0 ? gx : -gx, Y = gy > 0.0 ? gy : -gy;
    const double t = 0.41421356237309503;  // tan(pi/8)
    const double tol = 1e-12 * (fabs(X) + Y);
    const double v1 = Y - t * X;       // phi > pi/8
    if (fabs(v1) <= tol) *amb = true;
    if (!(v1 > 0.0)) return 0;
    const double v3 = t * Y - X;       // phi > 3pi/8
    if (fabs(v3) <= tol) *amb = true;
    if (!(v3 > 0.0)) return 1;
    const double v5 = -t * Y - X;      // phi > 5pi/8
    if (fabs(v5) <= tol) *amb = true;
    if (!(v5 > 0.0)) return 2;
    const double v7 = -(Y + t * X);    // phi > 7pi/8
    if (fabs(v7) <= tol) *amb = true;
    if (!(v7 > 0.0)) return 3;
    return 0;
}

__global__ void __launch_bounds__(256) nms_kernel(const double* __restrict__ gx,
                                                  const double* __restrict__ gy,
                                                  const double* __restrict__ mag, int w, int h,
                                                  ModelScratch* ms, unsigned char* state,
                                                  unsigned char* kept, int* amb_list) {
    const size_t total = (size_t)w * h;
    const size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= total) return;
    const int x = (int)(o % (size_t)w), y = (int)(o / (size_t)w);
    double low = ms->low, high = ms->high;
    if (ms->use_default) {  // default_thresholds, edge_model.cpp:17-24
        const double peak = __longlong_as_double((long long)ms->peak_bits);
        high = __dmul_rn(0.3, peak);
        low = __dmul_rn(0.5, high);
        if (o == 0) {
            ms->low = low;
            ms->high = high;
        }
    }
    unsigned char st = 0;
    if (x >= 1 && x + 1 < w && y >= 1 && y + 1 < h) {
        const double m = mag[o];
        if (!(m <= 0.0 || m < low)) {
            bool amb = false;
            const int b = orientation_bin_dev(gx[o], gy[o], &amb);
            if (amb) {
                st = 3;  // the host decides (glibc atan2)
                amb_list[atomicAdd(&ms->n_amb, 1)] = (int)o;
            } else {
                const int sx = b == 0 ? 1 : (b == 3 ? -1 : (b == 2 ? 0 : 1));
                const int sy = b == 0 ? 0 : 1;
                const double fwd = mag[(size_t)(y + sy) * w + (x + sx)];
                const double bwd = mag[(size_t)(y - sy) * w + (x - sx)];
                if (m > fwd && m >= bwd) st = m >= high ? 2 : 1;
            }
        }
    }
    state[o] = st;
    kept[o] = st == 2;
}

// Reachability from strong pixels through weak ones (8-connected): kept is
// the least fixpoint, reached whatever the update order.
__global__ void __launch_bounds__(1024) hysteresis_kernel(const unsigned char* __restrict__ state,
                                                          unsigned char* kept, int w, int h) {
    __shared__ int changed;
    const size_t total = (size_t)w * h;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) changed = 0;
        __syncthreads();
        int mine = 0;
        for (size_t i = threadIdx.x; i < total; i += blockDim.x) {
            if (kept[i] || state[i] == 0) continue;
            const int x = (int)(i % (size_t)w), y = (int)(i / (size_t)w);
            bool hit = false;
            for (int dy = -1; dy <= 1 && !hit; ++dy) {
                const int qy = y + dy;
                if (qy < 0 || qy >= h) continue;
                for (int dx = -1; dx <= 1; ++dx) {
                    const int qx = x + dx;
                    if ((dx | dy) == 0 || qx < 0 || qx >= w) continue;
                    if (kept[(size_t)qy * w + qx]) {
                        hit = true;
                        break;
                    }
                }
            }
            if (hit) {
                kept[i] = 1;
                mine = 1;
            }
        }
        if (mine) changed = 1;
        __syncthreads();
        if (!changed) break;
    }
}

// Row-major emission (the order scores are summed in, edge_model.cpp:116-148):
// thread t owns a contiguous pixel chunk; a block scan gives its output
// offset.  Coordinate sums are integers < 2^53, so the reference's sequential
// double sums are exact and equal these integer sums.
__global__ void __launch_bounds__(1024) emit_kernel(const double* __restrict__ gx,
                                                    const double* __restrict__ gy,
                                                    const double* __restrict__ mag,
                                                    const unsigned char* __restrict__ kept, int w,
                                                    int h, ModelScratch* ms,
                                                    ea_edge_point* out) {
    using Scan = cub::BlockScan<int, 1024>;
    using Reduce = cub::BlockReduce<unsigned long long, 1024>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ typename Reduce::TempStorage red_tmp;
    __shared__ double cxy[2];
    const size_t total = (size_t)w * h;
    const size_t chunk = (total + blockDim.x - 1) / blockDim.x;
    const size_t b0 = min(total, chunk * threadIdx.x), b1 = min(total, b0 + chunk);
    int cnt = 0;
    unsigned long long sx = 0, sy = 0;
    for (size_t i = b0; i < b1; ++i) {
        if (!kept[i]) continue;
        ++cnt;
        sx += i % (size_t)w;
        sy += i / (size_t)w;
    }
    int off = 0, n = 0;
    Scan(scan_tmp).ExclusiveSum(cnt, off, n);
    __syncthreads();
    const unsigned long long tx = Reduce(red_tmp).Sum(sx);
    __syncthreads();
    const unsigned long long ty = Reduce(red_tmp).Sum(sy);
    if (threadIdx.x == 0) {
        ms->n_kept = n;
        if (n > 0) {
            cxy[0] = __ddiv_rn((double)tx, (double)n);
            cxy[1] = __ddiv_rn((double)ty, (double)n);
            ms->cx = cxy[0];
            ms->cy = cxy[1];
        }
    }
    __syncthreads();
    if (n == 0) return;
    const double cx = cxy[0], cy = cxy[1];
    for (size_t i = b0; i < b1; ++i) {
        if (!kept[i]) continue;
        const double m = mag[i];
        ea_edge_point p;
        p.x_rel = __dsub_rn((double)(i % (size_t)w), cx);
        p.y_rel = __dsub_rn((double)(i / (size_t)w), cy);
        p.dx = __ddiv_rn(gx[i], m);
        p.dy = __ddiv_rn(gy[i], m);
        p.mag = m;
        out[off++] = p;
    }
}

void launch_magmax(ea_ctx* ctx, const double* mag, size_t total, ModelScratch* ms) {
    unsigned blocks = (unsigned)std::min<size_t>((total + 255) / 256, (size_t)ctx->sm_count * 4);
    magmax_kernel<<<blocks ? blocks : 1, 256, 0, ctx->stream>>>(mag, total, ms);
    check_launch("magmax_kernel");
    count_launch(ctx);
}

void launch_nms(ea_ctx* ctx, const double* gx, const double* gy, const double* mag, int w, int h,
                ModelScratch* ms, unsigned char* state, unsigned char* kept, int* amb_list) {
    const size_t total = (size_t)w * h;
    nms_kernel<<<(unsigned)((total + 255) / 256), 256, 0, ctx->stream>>>(gx, gy, mag, w, h, ms,
                                                                         state, kept, amb_list);
    check_launch("nms_kernel");
    count_launch(ctx);
}

void launch_hysteresis_emit(ea_ctx* ctx, const double* gx, const double* gy, const double* mag,
                            const unsigned char* state, unsigned char* kept, int w, int h,
                            ModelScratch* ms, ea_edge_point* out) {
    hysteresis_kernel<<<1, 1024, 0, ctx->stream>>>(state, kept, w, h);
    check_launch("hysteresis_kernel");
    emit_kernel<<<1, 1024, 0, ctx->stream>>>(gx, gy, mag, kept, w, h, ms, out);
    check_launch("emit_kernel");
    count_launch(ctx, 2);
}

}  // namespace eab
