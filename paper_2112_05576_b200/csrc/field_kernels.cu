// field_kernels.cu -- search-image side: 2x2 box pyramid, 3x3 Sobel gradient
// field, and the normalised float2 screening plane.
//
// All fp64 arithmetic uses explicit round-to-nearest intrinsics so that no
// multiply-add is contracted (the reference builds with -ffp-contract=off,
// proj/CMakeLists.txt:12-14) and every value is bit-identical to the
// reference's scalar kernels (proj/src/simd/kernels_scalar.cpp:14-37).
#include "kernels.cuh"

namespace eab {

// downsample_row  kernels_scalar.cpp:30-37 / image.cpp:248-261:
//   out[i] = ((top[2i] + top[2i+1]) + (bot[2i] + bot[2i+1])) * 0.25
__global__ void downsample_kernel(const double* __restrict__ in, int w, int h,
                                  double* __restrict__ out, int ow, int oh) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= ow || y >= oh) return;
    const double* top = in + (size_t)(2 * y) * w;
    const double* bot = top + w;
    const double t = __dadd_rn(__ldg(top + 2 * x), __ldg(top + 2 * x + 1));
    const double u = __dadd_rn(__ldg(bot + 2 * x), __ldg(bot + 2 * x + 1));
    out[(size_t)y * ow + x] = __dmul_rn(__dadd_rn(t, u), 0.25);
}

// sobel_row  kernels_scalar.cpp:14-28 / compute_gradients gradient.cpp:12-27.
// Writes every pixel; the one-pixel border ring is 0 as in GradientField's
// zero initialisation (gradient.h:22-27).
__global__ void sobel_kernel(const double* __restrict__ img, int w, int h,
                             double* __restrict__ gx, double* __restrict__ gy,
                             double* __restrict__ mag) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= w || y >= h) return;
    const size_t o = (size_t)y * w + x;
    if (x == 0 || y == 0 || x == w - 1 || y == h - 1) {
        gx[o] = 0.0;
        gy[o] = 0.0;
        mag[o] = 0.0;
        return;
    }
    const double* above = img + o - w;
    const double* mid = img + o;
    const double* below = img + o + w;
    const double a = __ldg(above - 1), b = __ldg(above), c = __ldg(above + 1);
    const double d = __ldg(mid - 1), f = __ldg(mid + 1);
    const double g = __ldg(below - 1), hh = __ldg(below), i = __ldg(below + 1);
    const double ew = __dsub_rn(f, d);
    const double ns = __dsub_rn(hh, b);
    const double sx = __dadd_rn(__dadd_rn(__dsub_rn(c, a), __dadd_rn(ew, ew)), __dsub_rn(i, g));
    const double sy = __dadd_rn(__dadd_rn(__dsub_rn(g, a), __dadd_rn(ns, ns)), __dsub_rn(i, c));
    gx[o] = sx;
    gy[o] = sy;
    mag[o] = __dsqrt_rn(__dadd_rn(__dmul_rn(sx, sx), __dmul_rn(sy, sy)));
}

// Screening plane: padded (W+2) x (H+2) float2 (one zero ring), rows skewed by
// (yp >> shift) for conflict-free lane strides (see search_kernels.cu).
// n = (gx/mag, gy/mag) rounded to fp32 when mag >= eps, else (0, 0) -- the
// latter gives exactly the reference's neutral 0 vote (kernels_scalar.cpp:44-47).
// One launch writes every element a screening kernel reads: field pixels,
// the zero ring and zero columns, and the zero strip that stands in for
// off-plane rows (so the buffer needs no memset); block (0, 0) also clears
// the search's histogram and control block (`clear`, `clear2`).
__global__ void plane_kernel(const double* __restrict__ gx, const double* __restrict__ gy,
                             const double* __restrict__ mag, int W, int H, double eps, int PW,
                             int PL, int shift, int zero, int zero_len,
                             float2* __restrict__ plane, unsigned* __restrict__ clear,
                             int clear_words, unsigned* __restrict__ clear2, int clear2_words) {
    const int xp = blockIdx.x * blockDim.x + threadIdx.x;
    const int yp = blockIdx.y;
    if (blockIdx.x == 0 && blockIdx.y == 0) {
        for (int i = threadIdx.x; i < clear_words; i += blockDim.x) clear[i] = 0u;
        for (int i = threadIdx.x; i < clear2_words; i += blockDim.x) clear2[i] = 0u;
    }
    if (yp == H + 2) {  // the zero strip
        for (int i = xp; i < zero_len; i += gridDim.x * blockDim.x)
            plane[zero + i] = make_float2(0.f, 0.f);
        return;
    }
    if (xp >= PW) return;
    double nx = 0.0, ny = 0.0;
    const int x = xp - 1 - PL, y = yp - 1;
    if (x >= 0 && x < W && y >= 0 && y < H) {
        const size_t o = (size_t)y * W + x;
        const double m = mag[o];
        if (m >= eps) {
            nx = __ddiv_rn(gx[o], m);
            ny = __ddiv_rn(gy[o], m);
        }
    }
    plane[(size_t)yp * PW + (yp >> shift) + xp] = make_float2((float)nx, (float)ny);
}

void launch_downsample(ea_ctx* ctx, const double* in, int w, int h, double* out) {
    const int ow = w / 2, oh = h / 2;
    if (ow < 1 || oh < 1) return;
    dim3 grid((ow + 127) / 128, oh);
    downsample_kernel<<<grid, 128, 0, ctx->stream>>>(in, w, h, out, ow, oh);
    check_launch("downsample_kernel");
    count_launch(ctx);
}

void launch_sobel(ea_ctx* ctx, const double* img, int w, int h, double* gx, double* gy,
                  double* mag) {
    dim3 grid((w + 127) / 128, h);
    sobel_kernel<<<grid, 128, 0, ctx->stream>>>(img, w, h, gx, gy, mag);
    check_launch("sobel_kernel");
    count_launch(ctx);
}

void launch_plane(ea_ctx* ctx, const ea_field* f, double eps, const PlaneGeom& g,
                  void* plane, unsigned* clear, int clear_words, unsigned* clear2,
                  int clear2_words) {
    dim3 grid((g.PW + 127) / 128, g.H + 3);  // + one row of blocks for the zero strip
    plane_kernel<<<grid, 128, 0, ctx->stream>>>(f->gx(), f->gy(), f->mag(), g.W, g.H, eps,
                                                 g.PW, g.PL, g.shift, g.zero,
                                                 (int)(g.elems - (size_t)g.zero),
                                                 static_cast<float2*>(plane), clear,
                                                 clear_words, clear2, clear2_words);
    check_launch("plane_kernel");
    count_launch(ctx);
}

}  // namespace eab
