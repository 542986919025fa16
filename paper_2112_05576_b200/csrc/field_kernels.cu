// field_kernels.cu -- search-image side: 2x2 box pyramid, 3x3 Sobel gradient
// field, and the normalised float2 screening plane.
//
// All fp64 arithmetic uses explicit round-to-nearest intrinsics so that no
// multiply-add is contracted (the reference builds with -ffp-contract=off,
// proj/CMakeLists.txt:12-14) and every value is bit-identical to the
// reference's scalar kernels (proj/src/simd/kernels_scalar.cpp:14-37).
#include <cstdlib>

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

// The whole working pyramid of one image in ONE launch: a CTA owns a TT x TT
// tile of the top level, i.e. a (TT << (L-1-l))-square tile of level l, and
// keeps in shared memory each level's tile plus the halo its Sobel and the
// levels above need (h_l = 2^(L-1-l) pixels: 1 at the top, doubling down).
// It loads the level-0 region once, builds levels 1..L-1 by the 2x2 box
// (downsample_kernel's arithmetic), and writes every level's image (l >= 1)
// and gradient field (sobel_kernel's arithmetic, zero ring) for its tile.
// Pixels of a region outside the level are never a source of an in-range
// pixel (floor halving) and only feed border pixels, whose output is 0.
// Replaces 2L - 1 dependent launches (and L reads of the level images).
__global__ void __launch_bounds__(256) pyramid_fields_kernel(const PyramidFieldsArgs a) {
    extern __shared__ double ps[];
    const int L = a.levels, TT = a.tile;
    // level l's region starts after the regions of levels 0..l-1
    auto reg = [&](int l) {
        int off = 0;
        for (int j = 0; j < l; ++j) {
            const int R = (TT + 2) << (L - 1 - j);
            off += R * R;
        }
        return ps + off;
    };
    // level 0 region: [X0 - h0, X0 + T0 + h0) x same in y
    {
        const int h0 = 1 << (L - 1), T0 = TT << (L - 1), R = T0 + 2 * h0;
        const int x0 = blockIdx.x * T0 - h0, y0 = blockIdx.y * T0 - h0;
        const int W = a.w[0], H = a.h[0];
        double* r0 = reg(0);
        // 32 x 8 threads: coalesced rows, four row-loads in flight per thread
        const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
        for (int ry0 = 0; ry0 < R; ry0 += 32) {
            for (int rx = tx; rx < R; rx += 32) {
                const int x = x0 + rx;
                double v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int ry = ry0 + ty + 8 * q, y = y0 + ry;
                    v[q] = (ry < R && x >= 0 && x < W && y >= 0 && y < H)
                               ? __ldg(a.img0 + (size_t)y * W + x) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int ry = ry0 + ty + 8 * q;
                    if (ry < R) r0[ry * R + rx] = v[q];
                }
            }
        }
    }
    __syncthreads();
    for (int l = 1; l < L; ++l) {  // level l region from level l-1 region (2x2 box)
        const int hl = 1 << (L - 1 - l), Tl = TT << (L - 1 - l), R = Tl + 2 * hl;
        const int Rp = 2 * R;  // level l-1 region side
        const int x0 = blockIdx.x * Tl - hl, y0 = blockIdx.y * Tl - hl;
        const int W = a.w[l], H = a.h[l];
        double* out = a.img[l];
        const double* prev = reg(l - 1);
        double* cur = reg(l);
        const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
        for (int ry = ty; ry < R; ry += 8)
        for (int rx = tx; rx < R; rx += 32) {
            const int i = ry * R + rx;
            const double* top = prev + (size_t)(2 * ry) * Rp + 2 * rx;
            const double t = __dadd_rn(top[0], top[1]);
            const double u = __dadd_rn(top[Rp], top[Rp + 1]);
            const double v = __dmul_rn(__dadd_rn(t, u), 0.25);
            cur[i] = v;
            const int x = x0 + rx, y = y0 + ry;
            if (rx >= hl && rx < hl + Tl && ry >= hl && ry < hl + Tl && x < W && y < H)
                out[(size_t)y * W + x] = v;  // the tile's own pixels of the level image
        }
        __syncthreads();
    }
    for (int l = 0; l < L; ++l) {  // Sobel of each level's tile
        const int hl = 1 << (L - 1 - l), Tl = TT << (L - 1 - l), R = Tl + 2 * hl;
        const int W = a.w[l], H = a.h[l];
        const int x0 = blockIdx.x * Tl, y0 = blockIdx.y * Tl;
        double* gx = a.gx[l];
        double* gy = a.gy[l];
        double* mg = a.mag[l];
        const double* rl = reg(l);
        const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
        for (int ty = ly; ty < Tl; ty += 8)
        for (int tx = lx; tx < Tl; tx += 32) {
            const int x = x0 + tx, y = y0 + ty;
            if (x >= W || y >= H) continue;
            const size_t o = (size_t)y * W + x;
            if (x == 0 || y == 0 || x == W - 1 || y == H - 1) {
                gx[o] = 0.0;
                gy[o] = 0.0;
                mg[o] = 0.0;
                continue;
            }
            const double* mid = rl + (size_t)(ty + hl) * R + (tx + hl);
            const double* above = mid - R;
            const double* below = mid + R;
            const double aa = above[-1], b = above[0], c = above[1];
            const double d = mid[-1], f = mid[1];
            const double g = below[-1], hh = below[0], ii = below[1];
            const double ew = __dsub_rn(f, d);
            const double ns = __dsub_rn(hh, b);
            const double sx =
                __dadd_rn(__dadd_rn(__dsub_rn(c, aa), __dadd_rn(ew, ew)), __dsub_rn(ii, g));
            const double sy =
                __dadd_rn(__dadd_rn(__dsub_rn(g, aa), __dadd_rn(ns, ns)), __dsub_rn(ii, c));
            gx[o] = sx;
            gy[o] = sy;
            mg[o] = __dsqrt_rn(__dadd_rn(__dmul_rn(sx, sx), __dmul_rn(sy, sy)));
        }
    }
}

size_t pyramid_fields_smem(int levels, int tile) {
    size_t n = 0;
    for (int l = 0; l < levels; ++l) {
        const size_t R = (size_t)(tile + 2) << (levels - 1 - l);
        n += R * R;
    }
    return n * sizeof(double);
}

bool launch_pyramid_fields(ea_ctx* ctx, const PyramidFieldsArgs& a_in) {
    if (a_in.levels < 1 || a_in.levels > kMaxFusedLevels) return false;
    if (std::getenv("EAB_NO_FUSED_PYRAMID")) return false;
    PyramidFieldsArgs a = a_in;
    // largest power-of-two top tile (<= 16) whose regions fit in 100 KB
    // (a tile below 8 reads the level-0 halo >= 2.25x over: slower than the
    // per-level kernels -- measured on cfg3, 5 levels)
    int tile = 16;
    while (tile > 8 && pyramid_fields_smem(a.levels, tile) > 100 * 1024) tile /= 2;
    const size_t smem = pyramid_fields_smem(a.levels, tile);
    if (smem > 100 * 1024) return false;
    a.tile = tile;
    raise_smem_limit(ctx, (const void*)pyramid_fields_kernel, 100 * 1024);
    const int T0 = tile << (a.levels - 1);
    dim3 grid((a.w[0] + T0 - 1) / T0, (a.h[0] + T0 - 1) / T0);
    pyramid_fields_kernel<<<grid, 256, smem, ctx->stream>>>(a);
    check_launch("pyramid_fields_kernel");
    count_launch(ctx);
    return true;
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
