// search_kernels.cu -- top-level exhaustive (x, y, theta) pose search and the
// per-level refinement, as sm_100a kernels.
//
// Pipeline of one top-level search (reference: run_search search.cpp:95-140,
// scan_range 72-93, score_rotated similarity.cpp:90-119):
//
//  1. rotate_kernel      rotate_model (similarity.cpp:68-88) for every theta of
//                        the grid, exact fp64, plus an fp32 screening table.
//  2. screen_*_kernel    fp32 screening score S_f of EVERY pose, written as a
//                        map + a 4096-bin histogram.  Votes are max-reduced in
//                        a fixed-point form (v + 3*2^e, summed as IEEE bit
//                        patterns), so the sum is exact and order-free and
//                        |S_f - S| <= delta for the reference fp64 score S.
//  3. threshold_kernel   k-th largest S_f bin  ->  band threshold T - 2*delta.
//  4. compact_kernel     candidates {S_f >= threshold}.
//  5. rescore_kernel     exact fp64 score of each candidate, reference order.
//  6. select_kernel      top k by `better` (score desc, index asc).
//
// Why this is exact: if |S_f - S| <= delta for every pose and T is at most
// the k-th largest S_f, every pose of the true top k has S_f >= T - 2*delta,
// so the exact pass sees all of them (and every pose tied with the k-th);
// selecting by `better` over exact scores reproduces search_topk bit for bit.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace eab {

// ---- 1. rotation tables ------------------------------------------------------

// floor(p + 0.5) for the lattice kernel: exact for every integer shift u with
// |p + u| < 2^21 unless frac(p) lies within 2^-28 of 0.5 (then the two
// roundings of (p + u) + 0.5 could cross an integer) -- such pairs are
// counted and widen the screening bound instead.
__device__ __forceinline__ int lattice_offset(double p, bool* amb) {
    if (!(p > -1048576.0 && p < 1048576.0)) {
        *amb = true;
        return 0;
    }
    const double fl = floor(p);
    const double fr = __dsub_rn(p, fl);  // exact
    const double d = fabs(__dsub_rn(fr, 0.5));
    if (d != 0.0 && d < 3.725290298461914e-09) *amb = true;  // 2^-28
    return (int)floor(__dadd_rn(p, 0.5));
}

__global__ void rotate_kernel(const double* __restrict__ pts, int n,
                              const double* __restrict__ cs, int nth,
                              double* __restrict__ rot, int4* __restrict__ scr,
                              int* __restrict__ flags, int* __restrict__ amb_list) {
    const size_t total = (size_t)nth * n;
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int th = (int)(t / n), i = (int)(t % n);
    const double c = cs[2 * th], s = cs[2 * th + 1];
    const double x = pts[i], y = pts[n + i], dx = pts[2 * n + i], dy = pts[3 * n + i];
    // similarity.cpp:79-86
    const double px = __dsub_rn(__dmul_rn(c, x), __dmul_rn(s, y));
    const double py = __dadd_rn(__dmul_rn(s, x), __dmul_rn(c, y));
    const double rx = __dsub_rn(__dmul_rn(c, dx), __dmul_rn(s, dy));
    const double ry = __dadd_rn(__dmul_rn(s, dx), __dmul_rn(c, dy));
    const double norm = __dsqrt_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)));
    const double ndx = __ddiv_rn(rx, norm), ndy = __ddiv_rn(ry, norm);
    rot[t] = px;
    rot[total + t] = py;
    rot[2 * total + t] = ndx;
    rot[3 * total + t] = ndy;
    if (scr) {
        bool amb = false;
        const int ox = lattice_offset(px, &amb);
        const int oy = lattice_offset(py, &amb);
        scr[t] = make_int4(ox, oy, __float_as_int((float)ndx), __float_as_int((float)ndy));
        if (amb) {
            atomicAdd(flags, 1);
            if (amb_list && atomicAdd(amb_list + th, 1) == 0) {  // first ambiguous point of th
                const int pos = atomicAdd(amb_list + nth, 1);
                amb_list[nth + 1 + pos] = th;
            }
        }
    }
}

void launch_rotate(ea_ctx* ctx, const double* pts_soa, int n, const double* cs, int nth,
                   double* rot_exact, int4* rot_screen, int* flags, int* amb) {
    const size_t total = (size_t)nth * n;
    if (total == 0) return;
    rotate_kernel<<<(unsigned)((total + 255) / 256), 256, 0, ctx->stream>>>(
        pts_soa, n, cs, nth, rot_exact, rot_screen, flags, amb);
    check_launch("rotate_kernel");
    count_launch(ctx);
}

// ---- 2. screening ------------------------------------------------------------

// 1D bulk copy global -> shared through the TMA engine, completing on an
// mbarrier (cp.async.bulk + mbarrier expect_tx; sizes multiple of 16 B).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_copy_to_smem(void* dst, const void* src, unsigned bytes,
                                                  unsigned long long* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    constexpr unsigned kChunk = 32768;
    for (unsigned off = 0; off < bytes; off += kChunk) {
        const unsigned len = bytes - off < kChunk ? bytes - off : kChunk;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(static_cast<char*>(dst) + off)),
            "l"(static_cast<const char*>(src) + off), "r"(len), "r"(smem_u32(bar))
            : "memory");
    }
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

template <int K>
__device__ __forceinline__ float max_run(const float* v) {
    if constexpr (K == 1) {
        return v[0];
    } else if constexpr (K == 3) {
        return fmax3(v[0], v[1], v[2]);
    } else if constexpr (K == 5) {
        return fmax3(fmax3(v[0], v[1], v[2]), v[3], v[4]);
    } else {
        float m = v[0];
#pragma unroll
        for (int i = 1; i < K; ++i) m = fmaxf(m, v[i]);
        return m;
    }
}

__device__ __forceinline__ int hist_bin(float s) {
    int b = __float2int_rd((s + 1.0f) * 2048.0f);
    return b < 0 ? 0 : (b >= kHistBins ? kHistBins - 1 : b);
}

// Adds a CTA's shared histogram into the global one (after a __syncthreads).
// With kf > 0 only the bins at or above the CTA's own kf-th largest score
// are added: that score is at most the global kf-th largest T_f, so every bin
// from bin(T_f) up keeps its exact global count and the threshold bin found
// by block_threshold is unchanged -- while a CTA adds a handful of bins
// instead of hundreds (global atomics were ~12% of a theta-slab launch).
__device__ __forceinline__ void merge_hist(const unsigned* __restrict__ hist,
                                           unsigned* __restrict__ ghist, int kf) {
    constexpr int kChunks = 256, kPer = kHistBins / kChunks;  // chunk c: bins from the top
    __shared__ unsigned csum[kChunks];
    __shared__ int kbin;
    int lo = 0;
    if (kf > 0) {
        for (int c = threadIdx.x; c < kChunks; c += blockDim.x) {
            unsigned v = 0;
#pragma unroll
            for (int j = 0; j < kPer; ++j) v += hist[kHistBins - 1 - (c * kPer + j)];
            csum[c] = v;
        }
        if (threadIdx.x == 0) kbin = 0;
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            constexpr int kLane = kChunks / 32;
            unsigned mine = 0;
#pragma unroll
            for (int j = 0; j < kLane; ++j) mine += csum[lane * kLane + j];
            unsigned incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            unsigned run = incl - mine;  // poses in higher lanes' chunks
            if (run < (unsigned)kf && incl >= (unsigned)kf) {
                for (int c = lane * kLane; c < (lane + 1) * kLane; ++c) {
                    if (run + csum[c] >= (unsigned)kf) {
                        for (int j = 0; j < kPer; ++j) {
                            const int b = kHistBins - 1 - (c * kPer + j);
                            run += hist[b];
                            if (run >= (unsigned)kf) {
                                kbin = b;
                                break;
                            }
                        }
                        break;
                    }
                    run += csum[c];
                }
            }
        }
        __syncthreads();
        lo = kbin;
    }
    for (int b = lo + (int)threadIdx.x; b < kHistBins; b += blockDim.x) {
        const unsigned v = hist[b];
        if (v) atomicAdd(&ghist[b], v);
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// CTA size of the lattice kernel (one CTA per SM).
#ifndef EAB_SCREEN_THREADS
#define EAB_SCREEN_THREADS 384  // fully padded planes: 12 warps x 166 regs, no spills (-3.6% vs 8 warps)
#endif
constexpr int kFastThreads = EAB_SCREEN_THREADS;  // fully padded planes
constexpr int kTW = 8;  // poses per lane along x

// One model point (NP = 1) or a pair of points on the same lattice row whose
// windows start DXP columns apart (NP = 2) over a lane's 8 x S pose block:
// walk the S + 2R plane rows the windows touch.  A pair loads the union of
// its two windows once (8 + 2R + DXP pixels per row instead of 2 x (8 + 2R)).
// (Packed FFMA2 scoring of a pixel against both points was tried: at this
// register pressure the pair-alignment MOVs cost more than it saved.)  CLAMP=false is the
// warp-uniform interior case (every column of the warp's windows lies inside
// the padded plane): loads address [row + immediate]; CLAMP=true clamps each
// column into the zero ring.  STRIP=false (region kernel): every row is
// inside the staged region.  Votes are accumulated as raw bit patterns
// bits(K + vote); the caller subtracts (points processed) x bits(K) once.
template <int R, int S, int SHIFT, bool IGNORE, bool CLAMP, bool STRIP, int NP, int DXP>
__device__ __forceinline__ void point_rows(const float2* __restrict__ P, const int PW,
                                           const int XL, const int cx_lo, const int cx_hi,
                                           const int H1, const int Z, const int cb,
                                           const int rb, const int ry_lo, const int ry_hi,
                                           const float dx1, const float dy1, const float dx2,
                                           const float dy2, const float K,
                                           unsigned (&acc)[S][kTW]) {
    constexpr int NC = kTW + 2 * R;                     // columns per point window
    constexpr int NCU = NC + (NP == 2 ? DXP : 0);       // columns of the union
    constexpr int NR = S + 2 * R;                       // rows per point
    constexpr int HP = 2 * R > 0 ? 2 * R : 1;
    int col[CLAMP ? NCU : 1];
    if constexpr (CLAMP) {
#pragma unroll
        for (int m = 0; m < NCU; ++m) col[m] = min(max(cb + m, 0), XL);
    }
    // For R <= 1 the zero ring makes an off-field centre vote exactly 0; a
    // 5-wide window can reach real pixels, so R >= 2 masks those centres.
    unsigned cmask1 = 0xffu, cmask2 = 0xffu;
    if constexpr (R >= 2) {
        cmask1 = cmask2 = 0u;
#pragma unroll
        for (int j = 0; j < kTW; ++j) {
            const int c1 = cb + R + j, c2 = c1 + DXP;  // padded columns of the centres
            cmask1 |= (c1 >= cx_lo && c1 <= cx_hi) ? (1u << j) : 0u;
            cmask2 |= (c2 >= cx_lo && c2 <= cx_hi) ? (1u << j) : 0u;
        }
    }
    float hprev1[HP][kTW], hprev2[NP == 2 ? HP : 1][kTW];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        // Rows off the plane read the zero strip at an offset congruent (mod
        // one wavefront of elements) to where the row would be, so the lanes'
        // bank spacing survives at the top/bottom edges.
        constexpr int kBankMask = 128 / (int)sizeof(float2) - 1;
        const int yv = rb + r;
        const int va = yv * PW + (yv >> SHIFT);
        const float2* row = P + (!STRIP || (unsigned)yv <= (unsigned)H1 ? va : Z + (va & kBankMask));
        if constexpr (!CLAMP) row += cb;
        float c1[NCU], c2[NP == 2 ? NCU : 1];
#pragma unroll
        for (int m = 0; m < NCU; ++m) {
            const float2 v = CLAMP ? row[col[m]] : row[m];
            if constexpr (NP == 2) {
                if constexpr (IGNORE) {
                    c1[m] = fabsf(fmaf(dy1, v.y, dx1 * v.x));
                    c2[m] = fabsf(fmaf(dy2, v.y, dx2 * v.x));
                } else {
                    c1[m] = fmaf(dy1, v.y, fmaf(dx1, v.x, K));
                    c2[m] = fmaf(dy2, v.y, fmaf(dx2, v.x, K));
                }
            } else if constexpr (IGNORE) {
                c1[m] = fabsf(fmaf(dy1, v.y, dx1 * v.x));
            } else {
                c1[m] = fmaf(dy1, v.y, fmaf(dx1, v.x, K));
            }
        }
        float h1[kTW], h2[NP == 2 ? kTW : 1];
#pragma unroll
        for (int j = 0; j < kTW; ++j) h1[j] = max_run<2 * R + 1>(c1 + j);
        if constexpr (NP == 2) {
#pragma unroll
            for (int j = 0; j < kTW; ++j) h2[j] = max_run<2 * R + 1>(c2 + DXP + j);
        }
        if (r >= 2 * R) {
            const int s = r - 2 * R;
            const int cys = rb + R + s;  // padded row of the window centres
            const bool row_in = R < 2 || (cys >= ry_lo && cys <= ry_hi);
#pragma unroll
            for (int j = 0; j < kTW; ++j) {
                float cv[2 * R + 1];
#pragma unroll
                for (int q = 0; q < 2 * R; ++q) cv[q] = hprev1[q][j];
                cv[2 * R] = h1[j];
                float v1 = max_run<2 * R + 1>(cv);
                if constexpr (IGNORE) v1 = v1 + K;
                if constexpr (R >= 2) v1 = (row_in && ((cmask1 >> j) & 1u)) ? v1 : K;
                if constexpr (NP == 2) {
#pragma unroll
                    for (int q = 0; q < 2 * R; ++q) cv[q] = hprev2[q][j];
                    cv[2 * R] = h2[j];
                    float v2 = max_run<2 * R + 1>(cv);
                    if constexpr (IGNORE) v2 = v2 + K;
                    if constexpr (R >= 2) v2 = (row_in && ((cmask2 >> j) & 1u)) ? v2 : K;
                    acc[s][j] += __float_as_uint(v1) + __float_as_uint(v2);
                } else {
                    acc[s][j] += __float_as_uint(v1);
                }
            }
        }
        if constexpr (R > 0) {
#pragma unroll
            for (int q = 0; q + 1 < 2 * R; ++q)
#pragma unroll
                for (int j = 0; j < kTW; ++j) {
                    hprev1[q][j] = hprev1[q + 1][j];
                    if constexpr (NP == 2) hprev2[q][j] = hprev2[q + 1][j];
                }
#pragma unroll
            for (int j = 0; j < kTW; ++j) {
                hprev1[2 * R - 1][j] = h1[j];
                if constexpr (NP == 2) hprev2[2 * R - 1][j] = h2[j];
            }
        }
    }
}

// A twin entry (two points with the same screening direction whose lattice
// offsets differ by (0,0): TW = 1, (1,0): TW = 2, (0,1): TW = 3) over a
// lane's 8 x S pose block: one candidate per pixel of the union window, one
// horizontal max per union column and one vertical max per union row serve
// both points; the second point's votes are the first's shifted by the
// offset, so acc += bits(V[s][j]) + bits(V[s + DY][j + DX]) (IADD3).  R <= 1
// (the zero ring stands in for the window-centre masks).
template <int R, int S, int SHIFT, bool IGNORE, bool CLAMP, bool STRIP, int TW>
__device__ __forceinline__ void twin_rows(const float2* __restrict__ P, const int PW,
                                          const int XL, const int H1, const int Z, const int cb,
                                          const int rb, const float dx, const float dy,
                                          const float K, unsigned (&acc)[S][kTW]) {
    static_assert(R <= 1, "twins need the zero ring (R <= 1)");
    constexpr int DX = TW == 2 ? 1 : 0, DY = TW == 3 ? 1 : 0;
    constexpr int NC = kTW + 2 * R + DX;  // union columns
    constexpr int NH = kTW + DX;          // horizontal maxima (window starts)
    constexpr int NR = S + 2 * R + DY;    // union rows
    constexpr int HP = 2 * R > 0 ? 2 * R : 1;
    int col[CLAMP ? NC : 1];
    if constexpr (CLAMP) {
#pragma unroll
        for (int m = 0; m < NC; ++m) col[m] = min(max(cb + m, 0), XL);
    }
    float hprev[HP][NH];
    float vprev[DY ? kTW : 1];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        constexpr int kBankMask = 128 / (int)sizeof(float2) - 1;
        const int yv = rb + r;
        const int va = yv * PW + (yv >> SHIFT);
        const float2* row = P + (!STRIP || (unsigned)yv <= (unsigned)H1 ? va : Z + (va & kBankMask));
        if constexpr (!CLAMP) row += cb;
        float c[NC];
#pragma unroll
        for (int m = 0; m < NC; ++m) {
            const float2 v = CLAMP ? row[col[m]] : row[m];
            if constexpr (IGNORE) c[m] = fabsf(fmaf(dy, v.y, dx * v.x));
            else c[m] = fmaf(dy, v.y, fmaf(dx, v.x, K));
        }
        float h[NH];
#pragma unroll
        for (int j = 0; j < NH; ++j) h[j] = max_run<2 * R + 1>(c + j);
        if (r >= 2 * R) {
            const int q = r - 2 * R;  // union output row
            float V[NH];
#pragma unroll
            for (int j = 0; j < NH; ++j) {
                float cv[2 * R + 1];
#pragma unroll
                for (int t = 0; t < 2 * R; ++t) cv[t] = hprev[t][j];
                cv[2 * R] = h[j];
                V[j] = max_run<2 * R + 1>(cv);
                if constexpr (IGNORE) V[j] = V[j] + K;
            }
            if constexpr (TW == 1) {
#pragma unroll
                for (int j = 0; j < kTW; ++j)
                    acc[q][j] += __float_as_uint(V[j]) + __float_as_uint(V[j]);
            } else if constexpr (TW == 2) {
#pragma unroll
                for (int j = 0; j < kTW; ++j)
                    acc[q][j] += __float_as_uint(V[j]) + __float_as_uint(V[j + 1]);
            } else {
                if (q >= 1) {
#pragma unroll
                    for (int j = 0; j < kTW; ++j)
                        acc[q - 1][j] += __float_as_uint(vprev[j]) + __float_as_uint(V[j]);
                }
#pragma unroll
                for (int j = 0; j < kTW; ++j) vprev[j] = V[j];
            }
        }
        if constexpr (R > 0) {
#pragma unroll
            for (int t = 0; t + 1 < 2 * R; ++t)
#pragma unroll
                for (int j = 0; j < NH; ++j) hprev[t][j] = hprev[t + 1][j];
#pragma unroll
            for (int j = 0; j < NH; ++j) hprev[2 * R - 1][j] = h[j];
        }
    }
}

// ---- point schedule ------------------------------------------------------------
// Per theta, the lattice kernels walk a schedule instead of the raw point
// list.  Points are sorted by (oy, ox) and combined into entries of one of
// three kinds; which three is the schedule's mode (each mode is its own
// kernel instantiation: a kernel that unrolls more bodies than three
// overflows the instruction cache -- six bodies measured IPC 2.51 -> 1.87,
// no_instructions stalls 4% -> 28%):
//  * mode 0 (pairs): singles; same-row neighbours whose windows start 0 or 1
//    column apart, sharing their window loads;
//  * mode 1 (twins): singles; two points with the SAME screening direction
//    (fp32 dx, dy bit patterns) whose lattice offsets differ by (1,0) or
//    (0,1) -- points along a straight template edge rotate to identical
//    directions -- sharing their candidates (one dot product per pixel for
//    both) and their horizontal and vertical window maxima (the second
//    point's windows are the first's shifted): ~4.3 instructions per
//    pose-eval instead of ~7.9.  R <= 1 only (the R >= 2 centre masks are
//    per point).
// The host builds mode 1 when R <= 1 and switches to mode 0 when fewer than
// a fifth of the points are twinned (round templates).  Layout per theta
// (stride sched_stride(n) = 1 + 2n int4): header {kind-0, kind-1, kind-2
// counts, 0}, then 2 int4 per entry {ox, oy, dxf, dyf} x {second point of a
// pair, or unused}, in kind order.  The sum over points is integer and
// order-free, so the schedule does not change a score.
constexpr int kMaxPairDx = 1;  // dx = 2 pairs: a fourth unrolled body, net loss (icache)
constexpr int kPairMaxN = 1024;  // larger models: singles only

__global__ void __launch_bounds__(256) schedule_kernel(const int4* __restrict__ scr, int n,
                                                       int4* __restrict__ sched, int dmin,
                                                       int dmax, int mode,
                                                       unsigned long long* __restrict__ twinned) {
    const int th = blockIdx.x;
    const int4* pts = scr + (size_t)th * n;
    int4* out = sched + (size_t)th * sched_stride(n);
    __shared__ int4 sp[kPairMaxN];       // the theta's points
    __shared__ short order[kPairMaxN];   // sorted position -> point
    __shared__ short part[kPairMaxN];    // sorted position -> partner position (-1: none)
    __shared__ unsigned char kind[kPairMaxN];  // entry kind at the first position; 255: second
    __shared__ short slot[kPairMaxN];    // sorted position -> output entry
    if (n > kPairMaxN) {
        if (threadIdx.x == 0) out[0] = make_int4(n, 0, 0, 0);
        for (int i = threadIdx.x; i < n; i += blockDim.x) out[1 + 2 * i] = __ldg(pts + i);
        return;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sp[i] = __ldg(pts + i);
    __syncthreads();
    // rank by (oy, ox, index): n^2 / 256 smem comparisons per thread
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int4 p = sp[i];
        int rank = 0;
        for (int k = 0; k < n; ++k) {
            const int4 q = sp[k];
            rank += (q.y < p.y) || (q.y == p.y && (q.x < p.x || (q.x == p.x && k < i)));
        }
        order[rank] = (short)i;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        part[i] = -1;
        kind[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode == 1) {
            // twins, greedily along the sorted list: (1,0) first (just after
            // i on its row), then (0,1) (binary search of the next row)
            for (int i = 0; i < n; ++i) {
                if (part[i] >= 0 || kind[i] == 255) continue;
                const int4 a = sp[order[i]];
                int mate = -1, k = 0;
                for (int j = i + 1; j < n; ++j) {
                    const int4 b = sp[order[j]];
                    if (b.y != a.y || b.x > a.x + 1) break;
                    if (b.x != a.x + 1 || part[j] >= 0 || kind[j] == 255 || b.z != a.z ||
                        b.w != a.w)
                        continue;
                    mate = j;
                    k = 1;
                    break;
                }
                if (mate < 0) {  // (0, 1): lower bound of (a.y + 1, a.x)
                    int lo = i + 1, hi = n;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        const int4 b = sp[order[mid]];
                        if (b.y < a.y + 1 || (b.y == a.y + 1 && b.x < a.x)) lo = mid + 1;
                        else hi = mid;
                    }
                    for (int j = lo; j < n; ++j) {
                        const int4 b = sp[order[j]];
                        if (b.y != a.y + 1 || b.x != a.x) break;
                        if (part[j] >= 0 || kind[j] == 255 || b.z != a.z || b.w != a.w) continue;
                        mate = j;
                        k = 2;
                        break;
                    }
                }
                if (mate >= 0) {
                    part[i] = (short)mate;
                    kind[i] = (unsigned char)k;
                    kind[mate] = 255;
                }
            }
        } else {
            // pairs: consecutive points of one row, windows dmin..dmax apart
            for (int i = 0; i + 1 < n;) {
                const int4 a = sp[order[i]], b = sp[order[i + 1]];
                const int d = b.x - a.x;
                if (b.y == a.y && d >= dmin && d <= dmax) {
                    part[i] = (short)(i + 1);
                    kind[i] = (unsigned char)(1 + d);
                    kind[i + 1] = 255;
                    i += 2;
                } else {
                    ++i;
                }
            }
        }
        int c[3] = {0, 0, 0};
        for (int i = 0; i < n; ++i)
            if (kind[i] != 255) ++c[kind[i]];
        int cur[3] = {0, c[0], c[0] + c[1]};
        for (int i = 0; i < n; ++i) slot[i] = kind[i] == 255 ? (short)-1 : (short)cur[kind[i]]++;
        out[0] = make_int4(c[0], c[1], c[2], 0);
        if (twinned && mode == 1) atomicAdd(twinned, 2ull * (unsigned long long)(c[1] + c[2]));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {  // scatter the entries
        const int e = slot[i];
        if (e < 0) continue;
        out[1 + 2 * e] = sp[order[i]];
        if (part[i] >= 0) out[2 + 2 * e] = sp[order[part[i]]];
    }
}

void launch_schedule(ea_ctx* ctx, const int4* scr, int n, int nth, int4* sched, int mode,
                     unsigned long long* twinned) {
    if (nth == 0 || n == 0) return;
    // EAB_NO_PAIRS=1: singles only (A/B measurements)
    static const int dmax = std::getenv("EAB_NO_PAIRS") ? -1 : kMaxPairDx;
    schedule_kernel<<<nth, 256, 0, ctx->stream>>>(scr, n, sched, 0, dmax, mode, twinned);
    check_launch("schedule_kernel");
    count_launch(ctx);
}

// Geometry a lane needs to walk schedule entries (see run_entries).
struct LaneGeom {
    const float2* P;
    int PW, XL, cx_lo, cx_hi, H1, Z;
    int cbase, rbase;  // window start = (ox + cbase, oy + rbase) in padded/region coordinates
    int ry_lo, ry_hi;  // field rows (window-centre mask for R >= 2)
    int cwbase, wspan; // EDGE: warp's first column = ox + cwbase; lanes span wspan more columns
};

template <int R, int S, int SHIFT, bool IGNORE, bool EDGE, bool STRIP, int NP, int DXP>
__device__ __forceinline__ void one_entry(const LaneGeom& g, const int4 p, const float dx2,
                                          const float dy2, const float K,
                                          unsigned (&acc)[S][kTW]) {
    const float dx1 = __int_as_float(p.z), dy1 = __int_as_float(p.w);
    const int cb = p.x + g.cbase, rb = p.y + g.rbase;
    constexpr int NCU = kTW + 2 * R + (NP == 2 ? DXP : 0);
    if constexpr (EDGE) {
        const int cw = p.x + g.cwbase;  // warp-uniform
        if (!(cw >= 0 && cw + g.wspan + NCU - 1 <= g.XL)) {
            point_rows<R, S, SHIFT, IGNORE, true, STRIP, NP, DXP>(
                g.P, g.PW, g.XL, g.cx_lo, g.cx_hi, g.H1, g.Z, cb, rb, g.ry_lo, g.ry_hi, dx1, dy1,
                dx2, dy2, K, acc);
            return;
        }
    }
    point_rows<R, S, SHIFT, IGNORE, false, STRIP, NP, DXP>(g.P, g.PW, g.XL, g.cx_lo, g.cx_hi,
                                                           g.H1, g.Z, cb, rb, g.ry_lo, g.ry_hi,
                                                           dx1, dy1, dx2, dy2, K, acc);
}

template <int R, int S, int SHIFT, bool IGNORE, bool EDGE, bool STRIP, int TW>
__device__ __forceinline__ void twin_entry(const LaneGeom& g, const int4 p, const float K,
                                           unsigned (&acc)[S][kTW]) {
    const float dx = __int_as_float(p.z), dy = __int_as_float(p.w);
    const int cb = p.x + g.cbase, rb = p.y + g.rbase;
    constexpr int NC = kTW + 2 * R + (TW == 2 ? 1 : 0);
    if constexpr (EDGE) {
        const int cw = p.x + g.cwbase;  // warp-uniform
        if (!(cw >= 0 && cw + g.wspan + NC - 1 <= g.XL)) {
            twin_rows<R, S, SHIFT, IGNORE, true, STRIP, TW>(g.P, g.PW, g.XL, g.H1, g.Z, cb, rb,
                                                           dx, dy, K, acc);
            return;
        }
    }
    twin_rows<R, S, SHIFT, IGNORE, false, STRIP, TW>(g.P, g.PW, g.XL, g.H1, g.Z, cb, rb, dx, dy,
                                                    K, acc);
}

// One lane block over schedule entries [e0, e1): singles, pairs by dx, then
// twins by offset (entry kinds in schedule order).
// Returns the number of model points processed (for the bits(K) correction).
template <int R, int S, int SHIFT, bool IGNORE, bool EDGE, bool STRIP, int MODE>
__device__ __forceinline__ int run_entries(const int4* __restrict__ ent, const int4 hdr, int e0,
                                           int e1, const LaneGeom& g, const float K,
                                           unsigned (&acc)[S][kTW]) {
    static_assert(MODE == 0 || R <= 1, "twin schedules need R <= 1");
    int done = 0;
    int lo = 0;
    const int bounds[3] = {hdr.x, hdr.y, hdr.z};
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const int hi = lo + bounds[t];
        const int b = max(lo, e0), e = min(hi, e1);
        // Entries arrive 32 at a time, one per lane, and are broadcast by
        // shuffles: no global load sits inside the row loop (a per-entry
        // prefetch shared a scoreboard with the shared-memory loads and
        // stalled the FMAs on L2 latency).
        for (int base = b; base < e; base += 32) {
            const int mine = base + lane;
            int4 pl = make_int4(0, 0, 0, 0), ql = make_int4(0, 0, 0, 0);
            if (mine < e) {
                pl = __ldg(ent + 2 * mine);
                if (MODE == 0 && t != 0) ql = __ldg(ent + 2 * mine + 1);
            }
            const int cnt = min(32, e - base);
            for (int j = 0; j < cnt; ++j) {
                int4 p;
                p.x = __shfl_sync(0xffffffffu, pl.x, j);
                p.y = __shfl_sync(0xffffffffu, pl.y, j);
                p.z = __shfl_sync(0xffffffffu, pl.z, j);
                p.w = __shfl_sync(0xffffffffu, pl.w, j);
                if (t == 0) {
                    one_entry<R, S, SHIFT, IGNORE, EDGE, STRIP, 1, 0>(g, p, 0.f, 0.f, K, acc);
                } else if constexpr (MODE == 0) {
                    const float dx2 = __int_as_float(__shfl_sync(0xffffffffu, ql.z, j));
                    const float dy2 = __int_as_float(__shfl_sync(0xffffffffu, ql.w, j));
                    if (t == 1)
                        one_entry<R, S, SHIFT, IGNORE, EDGE, STRIP, 2, 0>(g, p, dx2, dy2, K, acc);
                    else
                        one_entry<R, S, SHIFT, IGNORE, EDGE, STRIP, 2, 1>(g, p, dx2, dy2, K, acc);
                } else if constexpr (R <= 1) {
                    if (t == 1)
                        twin_entry<R, S, SHIFT, IGNORE, EDGE, STRIP, 2>(g, p, K, acc);
                    else
                        twin_entry<R, S, SHIFT, IGNORE, EDGE, STRIP, 3>(g, p, K, acc);
                }
            }
        }
        if (e > b) done += (e - b) * (t == 0 ? 1 : 2);
        lo = hi;
    }
    return done;
}

// The smem lattice kernel (integer top-level lattice with unit steps).
//
// A CTA is persistent (one per SM) and holds the whole padded screening
// plane of the top level in shared memory.  Work items are (theta, warp
// tile) pairs handed out by an atomic counter.  A warp tile is 32 x 8*S
// poses; lane (yg = lane&7, xg = lane>>3) owns an 8 x S block and keeps its
// 8*S fixed-point score accumulators in registers.  Per model point the lane
// walks the S + 2R plane rows its windows touch: 8 + 2R float2 loads, two FMAs
// per candidate, a horizontal (2R+1)-max (FMNMX3) and, once 2R+1 rows are in
// flight, the vertical max -- each plane pixel loaded serves up to (2R+1)^2
// window slots.  Bank mapping: a lane's float2 slot (mod 16) is
// yg*(2^SHIFT*PW + 1) + 8*xg = yg + 8*xg thanks to the row skew (yp >> SHIFT),
// so each half-warp (yg 0..7 x two xg) covers all 16 bank pairs once: LDS.64
// at the 2-wavefront minimum.
// Tail split: N items on P warps leave a last partial round of N mod P items;
// those are cut into f point-chunks (micro-items) so every warp ends with a
// short piece.  Chunk partial sums are exact int32, merged with coalesced
// reductions in L2; the chunk that arrives last finalises the tile.
struct TailPlan {
    unsigned long long n_main;  // items processed whole
    unsigned long long n_tail;  // items split into f point-chunks
    int f;
    int* part;                  // [n_tail][S*8][32] partial sums
    unsigned* done;             // [n_tail] arrival counters
};

// Lane epilogue shared by the lattice kernels: scores of the lane's 8 x S
// block into the map and the CTA histogram, warp max into item_max[item].
//
// Histogram floor: a pose whose score is below `floor` (the kf-th largest
// maximum among the warp's finished items, kf = k) is not counted -- there
// are kf distinct poses at or above the floor, so floor <= T_f (the k-th
// largest score), every bin above bin(T_f) keeps its exact count and bin
// (T_f) still reaches k: the threshold bin is unchanged.
constexpr int kFloorK = 8;  // k <= 8 uses the floor
__device__ __forceinline__ float warp_floor(const float* wtop, int kf) {
    return kf > 0 ? wtop[kf - 1] : -INFINITY;
}
__device__ __forceinline__ void floor_insert(float* wtop, float best, int lane) {
    if (lane == 0 && best > wtop[kFloorK - 1]) {
        int i = kFloorK - 1;
        while (i > 0 && wtop[i - 1] < best) {
            wtop[i] = wtop[i - 1];
            --i;
        }
        wtop[i] = best;
    }
    __syncwarp();
}

// Inserts a finished tile's largest lane maxima (up to kf of them; each lane
// maximum is the score of a distinct pose, so after ONE tile the warp's
// kf-th entry is a lower bound of T_f, the kf-th largest score -- with tile
// maxima alone it took kf tiles, and most of a launch's map was written
// before the floor rose).  Warp-uniform: one redux per round, rounds stop
// at the first value that does not enter the list.
__device__ __forceinline__ void floor_insert_lanes(float* wtop, float v, int kf, int lane) {
    const int rounds = kf > 0 ? kf : 1;
    for (int r = 0; r < rounds; ++r) {
        const unsigned key = float_order_key(v);
        const unsigned top = __reduce_max_sync(0xffffffffu, key);
        const float m = float_from_order_key(top);
        if (!(m > wtop[kFloorK - 1])) break;
        floor_insert(wtop, m, lane);
        const unsigned who = __ballot_sync(0xffffffffu, key == top);
        if (lane == __ffs(who) - 1) v = -INFINITY;
    }
}

// Top-list mode: after a warp's tile maxima list grows, publish its k-th
// largest (<= M_k) to the launch-wide floor; tiles below (global floor -
// 4 delta) are not written to the map (emit_tile).
__device__ __forceinline__ void publish_floor(const ScreenArgs& a, const float* wtop, int lane) {
    if (lane == 0 && a.kf > 0) {
        const float f = wtop[a.kf - 1];
        if (f > -INFINITY) atomicMax(&a.ctrl->gfloor, float_order_key(f));
    }
}
__device__ __forceinline__ float map_floor_of(const ScreenArgs& a, float own) {
    const float g = float_from_order_key(__ldcg(&a.ctrl->gfloor));
    return __fsub_rd(fmaxf(own, g), a.map_margin);
}

// emit_tile for integer steps sx, sy > 1: the lane's 8 x S block is on the
// unit lattice; only translations X % sx == 0, Y % sy == 0 are grid poses
// (ix, iy) = (X / sx, Y / sy).  Kept out of line of the unit-step path.
template <int S, bool HIST>
__device__ __noinline__ float emit_tile_strided(const ScreenArgs& a, const int (&acc)[S][kTW],
                                                const int X, const int Y, unsigned long long itr,
                                                unsigned long long item, unsigned* hist,
                                                const int lane, const float floor,
                                                const float map_floor, float& lbest) {
    float best = -INFINITY;
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int j = 0; j < kTW; ++j) {
            const int ux = X + j, uy = Y + s;
            if (ux % a.sx == 0 && uy % a.sy == 0 &&
                (unsigned long long)(ux / a.sx) < a.nx && (unsigned long long)(uy / a.sy) < a.ny)
                best = fmaxf(best, (float)acc[s][j] * a.scale);
        }
    lbest = best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) a.item_max[item] = best;
    if (best < map_floor) return best;  // warp-uniform
    float* out = a.map + (size_t)itr * (a.nx * a.ny);
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int j = 0; j < kTW; ++j) {
            const int ux = X + j, uy = Y + s;
            if (ux % a.sx != 0 || uy % a.sy != 0) continue;
            const unsigned long long ix = (unsigned long long)(ux / a.sx);
            const unsigned long long iy = (unsigned long long)(uy / a.sy);
            if (ix < a.nx && iy < a.ny) {
                const float sc = (float)acc[s][j] * a.scale;
                out[iy * a.nx + ix] = sc;
                if constexpr (HIST)
                    if (hist && sc >= floor) atomicAdd(&hist[hist_bin(sc)], 1u);
            }
        }
    return best;
}

template <int S, bool HIST = true>
__device__ __forceinline__ float emit_tile(const ScreenArgs& a, const int (&acc)[S][kTW],
                                           const int X, const int Y, unsigned long long itr,
                                           unsigned long long item, unsigned* hist,
                                           const int lane, const float floor,
                                           const float map_floor, float& lbest) {
    // Top-list mode passes map_floor = (the warp's k-th largest tile maximum
    // so far) - 4 delta, rounded down: a tile whose maximum is below it can
    // never reach the band (its max < M_k - 2 delta, the finish's threshold),
    // so its scores are not written -- most tiles of a search, and most of
    // the map's DRAM write traffic.
    if (a.sx != 1 || a.sy != 1)  // integer steps > 1: only the grid's poses
        return emit_tile_strided<S, HIST>(a, acc, X, Y, itr, item, hist, lane, floor, map_floor,
                                          lbest);
    float best = -INFINITY;
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int j = 0; j < kTW; ++j)
            if ((unsigned long long)(X + j) < a.nx && (unsigned long long)(Y + s) < a.ny)
                best = fmaxf(best, (float)acc[s][j] * a.scale);
    lbest = best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) a.item_max[item] = best;
    if (best < map_floor) return best;  // warp-uniform
    float* out = a.map + (size_t)itr * (a.nx * a.ny);
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const unsigned long long iy = (unsigned long long)(Y + s);
#pragma unroll
        for (int j = 0; j < kTW; ++j) {
            const unsigned long long ix = (unsigned long long)(X + j);
            if (ix < a.nx && iy < a.ny) {
                const float sc = (float)acc[s][j] * a.scale;
                out[iy * a.nx + ix] = sc;
                if constexpr (HIST)
                    if (hist && sc >= floor) atomicAdd(&hist[hist_bin(sc)], 1u);
            }
        }
    }
    return best;
}

// k largest values (with multiplicity) of up to 32*Q descending lists of
// kTopK floats (list i at src + i * kTopK, 16-byte aligned), by one warp:
// each lane folds its lists into a register top-kTopK (insertion network),
// then k rounds of a warp max over the lanes' heads, the winning lane
// popping one instance per round.  Returns the k-th largest (-inf if fewer
// than k finite values); lane 0 writes the k values to out (if given).
template <int Q, bool GLOBAL>
__device__ __forceinline__ float warp_kth_of_lists(const float* src, int nlists, int k, float* out,
                                                   int lane) {
    float L[kTopK];
#pragma unroll
    for (int i = 0; i < kTopK; ++i) L[i] = -INFINITY;
    float4 buf[Q][2];
#pragma unroll
    for (int q = 0; q < Q; ++q) {  // all loads first: one round trip
        const int li = lane + 32 * q;
        const float4* p = reinterpret_cast<const float4*>(src + (size_t)li * kTopK);
        const float4 ninf = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        buf[q][0] = li < nlists ? (GLOBAL ? __ldcg(p) : p[0]) : ninf;
        buf[q][1] = li < nlists ? (GLOBAL ? __ldcg(p + 1) : p[1]) : ninf;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const float v[kTopK] = {buf[q][0].x, buf[q][0].y, buf[q][0].z, buf[q][0].w,
                                buf[q][1].x, buf[q][1].y, buf[q][1].z, buf[q][1].w};
#pragma unroll
        for (int j = 0; j < kTopK; ++j) {
            float x = v[j];
#pragma unroll
            for (int i = 0; i < kTopK; ++i) {
                const float hi = fmaxf(L[i], x);
                x = fminf(L[i], x);
                L[i] = hi;
            }
        }
    }
    float t = -INFINITY;
    for (int r = 0; r < k; ++r) {
        float m = L[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const int win = __ffs(__ballot_sync(0xffffffffu, L[0] == m)) - 1;
        if (lane == win) {
#pragma unroll
            for (int i = 0; i + 1 < kTopK; ++i) L[i] = L[i + 1];
            L[kTopK - 1] = -INFINITY;
        }
        if (out && lane == 0) out[r] = m;
        t = m;
    }
    return t;
}

// Fused path: band threshold thr = M_k - 2 delta, M_k the kf-th largest
// TILE maximum, from the CTAs' lists (cta_top[G][kTopK], each descending, of
// their warps' largest tile maxima).  The k tiles whose maxima are >= M_k
// hold k distinct poses with S_f >= M_k, so M_k <= T_f (the k-th largest S_f)
// and every pose of the true top k has S_f >= T_f - 2 delta >= M_k - 2 delta
// (DESIGN.md §4).  M_k is a map value, so the comparison is exact.
//
// Compact, rolled code on purpose: everything after the screen loop runs
// once, from a cold instruction cache (the loop's ~50 KB of SASS evicted it
// and the step's L2 flush evicted L2), so its cost tracks its code size --
// a fully unrolled warp merge measured 8.7 us here against 3.2 us rolled.
__device__ __forceinline__ float fused_threshold(const FinishArgs& f, float* ttop) {
    __shared__ float thr_s;
    const int n = f.n_lists * kTopK;  // the screen launch's CTAs (not this grid's)
    for (int i = threadIdx.x; i < n; i += blockDim.x) ttop[i] = __ldcg(f.cta_top + i);
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        // lane owns lists lane, lane + 32, ... (head index per list in a bit
        // field: 4 bits each, kTopK <= 8; up to 16 lists per lane)
        const int G = f.n_lists;
        unsigned long long heads = 0ull;
        float t = -INFINITY;
        for (int r = 0; r < f.k; ++r) {
            float mine = -INFINITY;
            int src = -1;
#pragma unroll 1
            for (int q = 0; q < 16 && lane + 32 * q < G; ++q) {
                const int h = (int)((heads >> (4 * q)) & 15ull);
                const float x = h < kTopK ? ttop[(lane + 32 * q) * kTopK + h] : -INFINITY;
                if (x > mine) {
                    mine = x;
                    src = q;
                }
            }
            float m = mine;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            const int win = __ffs(__ballot_sync(0xffffffffu, mine == m && src >= 0)) - 1;
            if (lane == win) heads += 1ull << (4 * src);
            t = m;
        }
        if (lane == 0) {
            float thr = -INFINITY;
            if (t > -INFINITY) {  // else fewer than k poses: every pose is a candidate
                const double th = (double)t - 2.0 * f.delta;
                thr = (float)th;
                if ((double)thr > th) thr = nextafterf(thr, -INFINITY);
            }
            thr_s = thr;
        }
    }
    __syncthreads();
    return thr_s;
}

// Region-tiled lattice kernel: the plane lives in global memory (zero ring,
// row skew as in PlaneGeom) and each CTA stages, in shared memory, the
// window that one warp tile of translations can touch: the tile plus a halo
// h = ro + R, where ro bounds |lattice offset| of every rotated model point.
// Inside the region no window needs clamping and no row leaves it, so the
// inner loop is the smem kernel's unclamped path.  Cells of the region off
// the padded plane are zero (a zero plane pixel contributes the fixed-point
// zero vote, exactly like the ring).
//
// Work: CTA items (warp tile m, theta group g) of kGroup thetas, one per
// warp, ordered tile-major and split into contiguous equal runs per CTA, so a
// CTA reloads its region only when its run crosses into the next tile.
struct RegionPlan {
    int RW, RH;              // region pitch (elements; even, a multiple of 4 for 4-row strips) and rows
    int elems16;             // region size in 16 B chunks
    unsigned long long n_items;  // warp tiles x theta groups
    unsigned groups;         // theta groups per warp tile
};
// thetas per CTA item (= warps per CTA): 12 warps x 8-row strips (168 regs; 8
// warps measured 1.2% slower for 3x3 windows and 19% slower for 5x5, where
// 12 warps spill ~650 B), 16 x 4-row
template <int R, int S>
constexpr int region_group() { return S == 4 ? 16 : 12; }

// SHIFT: the region's row skew in shared memory (lane strips of S = 2^SHIFT
// rows); the global plane keeps its own (a.geom.shift).
template <int R, int S, int SHIFT, bool IGNORE, int XG, int MODE>
__global__ void __launch_bounds__(region_group<R, S>() * 32, 1)
    screen_region_kernel(const ScreenArgs a, const unsigned nwx, const unsigned nwy,
                         const RegionPlan rp) {
    constexpr int kGroup = region_group<R, S>();
    extern __shared__ __align__(16) unsigned char smem[];
    const bool toplist = a.cta_top != nullptr;  // no histogram (see ScreenArgs::cta_top)
    unsigned* hist = reinterpret_cast<unsigned*>(smem);
    float2* P = reinterpret_cast<float2*>(smem + (toplist ? 0 : kHistBins * sizeof(unsigned)));
    if (!toplist)
        for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) hist[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl->cand_count = 0ull;  // for the finish
    __shared__ __align__(16) float wtop_all[kGroup][kFloorK];
    float* wtop = wtop_all[threadIdx.x >> 5];
    if ((threadIdx.x & 31) < kFloorK) wtop[threadIdx.x & 31] = -INFINITY;

    constexpr int YG = 32 / XG;
    constexpr int TWX = 8 * XG, TWY = YG * S;  // warp tile
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int yg = lane % YG, xg = lane / YG;
    const int h = a.ro + R;
    const int PW = a.geom.PW, GH = a.geom.H + 2, GSH = a.geom.shift;
    const float2* G = static_cast<const float2*>(a.plane);
    const float K = a.K;

    const unsigned long long b0 = rp.n_items * blockIdx.x / gridDim.x;
    const unsigned long long b1 = rp.n_items * (blockIdx.x + 1) / gridDim.x;
    long long loaded = -1;
    for (unsigned long long ci = b0; ci < b1; ++ci) {
        const unsigned long long tile = ci / rp.groups;
        const unsigned g = (unsigned)(ci % rp.groups);
        const unsigned wx = (unsigned)(tile % nwx), wy = (unsigned)(tile / nwx);
        const int TX0 = (int)wx * TWX, TY0 = (int)wy * TWY;
        // region (0, 0) = padded plane (C0, R0)
        const int C0 = TX0 + a.ix0 + 1 + a.geom.PL - h;
        const int R0 = TY0 + a.iy0 + 1 - h;
        if ((long long)tile != loaded) {
            __syncthreads();  // previous item's readers are done
            for (int r = warp; r < rp.RH; r += nwarp) {
                const int gr = R0 + r;
                float2* srow = P + r * rp.RW + (r >> SHIFT);
                if (gr >= 0 && gr < GH) {
                    const float2* grow = G + (size_t)gr * PW + (gr >> GSH);
                    for (int c = lane; c < rp.RW; c += 32) {
                        const int gc = C0 + c;
                        srow[c] = (gc >= 0 && gc < PW) ? __ldg(grow + gc) : make_float2(0.f, 0.f);
                    }
                } else {
                    for (int c = lane; c < rp.RW; c += 32) srow[c] = make_float2(0.f, 0.f);
                }
            }
            __syncthreads();
            loaded = (long long)tile;
        }
        const unsigned long long itr = (unsigned long long)g * kGroup + warp;
        if (itr >= a.it_count) continue;  // warp-uniform; barriers above are CTA-uniform
        const unsigned long long item = (itr * nwy + wy) * nwx + wx;
        if (__ldg(a.amb + itr) != 0) {  // flagged theta: the general kernel scores it
            if (lane == 0) a.item_max[item] = INFINITY;
            continue;
        }
        const int Xr = xg * kTW, Yr = yg * S;  // lane block inside the tile
        LaneGeom lg;
        lg.P = P;
        lg.PW = rp.RW;
        lg.XL = rp.RW - 1;
        lg.cx_lo = 1 + a.geom.PL - C0;  // field bounds in region coordinates
        lg.cx_hi = a.geom.W + a.geom.PL - C0;
        lg.H1 = rp.RH - 1;
        lg.Z = 0;
        lg.cbase = Xr + h - R;  // region column of the window start - ox
        lg.rbase = Yr + h - R;  // region row of the window start - oy
        lg.ry_lo = 1 - R0;
        lg.ry_hi = a.geom.H - R0;
        lg.cwbase = lg.wspan = 0;
        const int4* sch = a.sched + itr * sched_stride(a.n);
        const int4 hdr = __ldg(sch);

        unsigned uacc[S][kTW];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int j = 0; j < kTW; ++j) uacc[s][j] = 0u;
        const int done = run_entries<R, S, SHIFT, IGNORE, false, false, MODE>(
            sch + 1, hdr, 0, hdr.x + hdr.y + hdr.z, lg, K, uacc);
        int acc[S][kTW];
        const unsigned corr = (unsigned)done * a.B3;
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int j = 0; j < kTW; ++j) acc[s][j] = (int)(uacc[s][j] - corr);
        const float wf = warp_floor(wtop, a.kf);
        float lbest;
        emit_tile<S>(a, acc, TX0 + Xr, TY0 + Yr, itr, item, toplist ? nullptr : hist, lane, wf,
                     toplist ? map_floor_of(a, wf) : -INFINITY, lbest);
        floor_insert_lanes(wtop, lbest, a.kf, lane);
        if (toplist) publish_floor(a, wtop, lane);
    }
    __syncthreads();
    if (toplist) {  // the CTA's kf largest tile maxima (merge of its warps' lists)
        if (threadIdx.x < 32) {
            float* out = a.cta_top + blockIdx.x * kTopK;
            warp_kth_of_lists<1, false>(&wtop_all[0][0], kGroup, a.kf, out, threadIdx.x);
            if (threadIdx.x >= a.kf && threadIdx.x < kTopK) out[threadIdx.x] = -INFINITY;
        }
    } else {
        merge_hist(hist, a.hist, a.kf);
    }
}

static RegionPlan region_plan(const ScreenArgs& a, int R, int S) {
    const int YG = 32 / a.xg;
    const int h = a.ro + R;
    const int shift = S == 4 ? 2 : 3;
    RegionPlan rp{};
    rp.RW = 8 * a.xg + 2 * h;
    // lane slots stay yg + 8*xg (mod 16): S * RW must be a multiple of 16
    const int mult = S == 4 ? 4 : 2;
    rp.RW = (rp.RW + mult - 1) / mult * mult;
    rp.RH = YG * S + 2 * h;
    const size_t elems = (size_t)rp.RH * rp.RW + (size_t)((rp.RH - 1) >> shift) + 1;
    rp.elems16 = (int)((elems * sizeof(float2) + 15) / 16);
    return rp;
}

static size_t region_smem(const RegionPlan& rp, bool toplist) {
    return (toplist ? 0 : kHistBins * sizeof(unsigned)) + (size_t)rp.elems16 * 16;
}

template <int R, int S, bool IGNORE, int XG, int MODE>
static void run_region(ea_ctx* ctx, const ScreenArgs& a, RegionPlan rp) {
    constexpr int YG = 32 / XG, kGroup = region_group<R, S>();
    const unsigned nwx = (unsigned)((a.lnx + 8 * XG - 1) / (8 * XG));
    const unsigned nwy = (unsigned)((a.lny + YG * S - 1) / (YG * S));
    rp.groups = (unsigned)((a.it_count + kGroup - 1) / kGroup);
    rp.n_items = (unsigned long long)nwx * nwy * rp.groups;
    const size_t smem = region_smem(rp, a.cta_top != nullptr);
    auto kern = screen_region_kernel<R, S, S == 4 ? 2 : 3, IGNORE, XG, MODE>;
    raise_smem_limit(ctx, (const void*)kern, smem);
    unsigned long long ctas = std::min<unsigned long long>(rp.n_items, (unsigned)ctx->sm_count);
    if (ctas == 0) ctas = 1;
    ctx->screen_ctas = (int)ctas;  // the finish merges this many per-CTA top lists
    kern<<<(unsigned)ctas, kGroup * 32, smem, ctx->stream>>>(a, nwx, nwy, rp);
    check_launch("screen_region_kernel");
    count_launch(ctx);
}

bool launch_screen_region(ea_ctx* ctx, const ScreenArgs& a) {
    if (a.geom.shift != 3 || a.geom.elem_bytes != 8 || a.R > 2) return false;
    if (a.sched_mode == 1 && a.R > 1) return false;
    // twin schedules: 4-row strips x 16 warps (the fast kernel's reasoning)
    const int S = a.sched_mode == 1 ? 4 : 8;
    const RegionPlan rp = region_plan(a, a.R, S);
    if (region_smem(rp, a.cta_top != nullptr) > ctx->smem_optin) return false;
    const bool ig = a.ignore != 0;
#define EAB_REGION_M(RR, SS, MM)                                                \
    if (a.xg == 2) {                                                            \
        if (ig) run_region<RR, SS, true, 2, MM>(ctx, a, rp);                    \
        else run_region<RR, SS, false, 2, MM>(ctx, a, rp);                      \
    } else {                                                                    \
        if (ig) run_region<RR, SS, true, 4, MM>(ctx, a, rp);                    \
        else run_region<RR, SS, false, 4, MM>(ctx, a, rp);                      \
    }
#define EAB_REGION(RR)                                                          \
    if (a.R == RR) {                                                            \
        if (a.sched_mode == 1) {                                                \
            EAB_REGION_M(RR, 4, 1)                                              \
        } else {                                                                \
            EAB_REGION_M(RR, 8, 0)                                              \
        }                                                                       \
        return true;                                                            \
    }
    EAB_REGION(1)
    EAB_REGION(0)
    if (a.R == 2) {
        EAB_REGION_M(2, 8, 0)
        return true;
    }
#undef EAB_REGION
#undef EAB_REGION_M
    return false;
}

// General screening kernel: any grid (non-integer or non-unit steps), any
// neighbourhood, any field border.  One thread per pose; projections are the
// reference's exact fp64 ones, windows are clipped exactly; the candidate and
// fixed-point arithmetic is the same as the lattice kernel's.
template <bool IGNORE>
__global__ void __launch_bounds__(256)
    screen_general_kernel(const ScreenArgs a, unsigned long long total, const int* tlist) {
    __shared__ unsigned hist[kHistBins];
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) hist[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl->cand_count = 0ull;  // for the finish
    __syncthreads();
    const unsigned long long plane_poses = a.nx * a.ny;
    // list mode: logical theta j -> slab theta tlist[j + 1], tlist[0] entries
    if (tlist) total = (unsigned long long)__ldg(tlist) * plane_poses;
    const int W = a.geom.W, H = a.geom.H, PW = a.geom.PW, SH = a.geom.shift;
    const int R = a.R;
    const float K = a.K;
    const int B3 = (int)a.B3;
    const int lane = threadIdx.x & 31;
    for (unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
         t0 < total; t0 += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long t = t0 + lane;
        float sc = -INFINITY;
        if (t < total) {
        const unsigned long long itr = tlist ? (unsigned long long)__ldg(tlist + 1 + t / plane_poses)
                                             : t / plane_poses;
        const unsigned long long rem = t % plane_poses;
        const unsigned long long iy = rem / a.nx, ix = rem % a.nx;
        const double ux = lattice(a.x0, ix, a.dx);
        const double uy = lattice(a.y0, iy, a.dy);
        const size_t base = (size_t)itr * a.n;
        int acc = 0;
        for (int i = 0; i < a.n; ++i) {
            const double px = __dadd_rn(__ldg(a.rot_exact + base + i), ux);
            const double py = __dadd_rn(__ldg(a.rot_exact + a.rot_stride + base + i), uy);
            if (!(px > -kCoordGuard && px < kCoordGuard && py > -kCoordGuard &&
                  py < kCoordGuard))
                continue;
            const int cx = (int)floor(__dadd_rn(px, 0.5));
            const int cy = (int)floor(__dadd_rn(py, 0.5));
            if (cx < 0 || cx >= W || cy < 0 || cy >= H) continue;
            const int4 q = __ldg(a.rot_screen + base + i);
            const float dxf = __int_as_float(q.z), dyf = __int_as_float(q.w);
            const int x0 = max(cx - R, 0), x1 = min(cx + R, W - 1);
            const int y0 = max(cy - R, 0), y1 = min(cy + R, H - 1);
            float best = -INFINITY;
            for (int y = y0; y <= y1; ++y) {
                const int yp = y + 1;
                const float2* row = static_cast<const float2*>(a.plane) + (size_t)yp * PW +
                                    (yp >> SH) + 1 + a.geom.PL;
                for (int x = x0; x <= x1; ++x) {
                    const float2 v = __ldg(row + x);
                    const float c = IGNORE ? fabsf(fmaf(dyf, v.y, dxf * v.x))
                                           : fmaf(dyf, v.y, fmaf(dxf, v.x, K));
                    best = fmaxf(best, c);
                }
            }
            if constexpr (IGNORE) best = best + K;
            acc += __float_as_int(best) - B3;
        }
        sc = (float)acc * a.scale;
        a.map[itr * plane_poses + rem] = sc;
        if (!a.cta_top) atomicAdd(&hist[hist_bin(sc)], 1u);  // top-list mode: no histogram
        }
        if (tlist) continue;  // item_max belongs to the lattice items (set to +inf)
        float best = sc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) a.item_max[t0 >> 5] = best;
    }
    __syncthreads();
    if (!a.cta_top) merge_hist(hist, a.hist, a.kf);
}

// One CTA per translation tile: any |g| >= eps within the tile's halo?
__global__ void __launch_bounds__(256) zero_tiles_kernel(const double* __restrict__ mag, int W,
                                                         int H, double eps, int ix0, int iy0,
                                                         unsigned nwx, int tw, int th, int halo,
                                                         unsigned char* __restrict__ out) {
    const unsigned t = blockIdx.x;
    const int wx = (int)(t % nwx), wy = (int)(t / nwx);
    const int x0 = max(ix0 + wx * tw - halo, 0), x1 = min(ix0 + wx * tw + tw - 1 + halo, W - 1);
    const int y0 = max(iy0 + wy * th - halo, 0), y1 = min(iy0 + wy * th + th - 1 + halo, H - 1);
    int any = 0;
    if (x0 <= x1 && y0 <= y1) {
        const int cols = x1 - x0 + 1;
        const long long n = (long long)cols * (y1 - y0 + 1);
        for (long long i = threadIdx.x; i < n && !any; i += blockDim.x) {
            const int y = y0 + (int)(i / cols), x = x0 + (int)(i % cols);
            any = __ldg(mag + (size_t)y * W + x) >= eps;
        }
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) out[t] = any ? 0 : 1;
}

void launch_zero_tiles(ea_ctx* ctx, const ea_field* f, double eps, int ix0, int iy0,
                       unsigned nwx, unsigned nwy, int tw, int th, int halo,
                       unsigned char* out) {
    const unsigned long long n = (unsigned long long)nwx * nwy;
    if (n == 0) return;
    zero_tiles_kernel<<<(unsigned)n, 256, 0, ctx->stream>>>(f->mag(), f->width, f->height, eps,
                                                            ix0, iy0, nwx, tw, th, halo, out);
    check_launch("zero_tiles_kernel");
    count_launch(ctx);
}

void launch_screen_general(ea_ctx* ctx, const ScreenArgs& a) {
    const unsigned long long total = a.nx * a.ny * a.it_count;
    unsigned long long blocks = (total + 255) / 256;
    const unsigned long long cap = (unsigned long long)ctx->sm_count * 8;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    if (a.ignore)
        screen_general_kernel<true><<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, total, nullptr);
    else
        screen_general_kernel<false><<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, total, nullptr);
    check_launch("screen_general_kernel");
    count_launch(ctx);
}

// Flagged thetas (a few per full rotation, e.g. 90/180/270 deg for a model
// with half-integer coordinates): their count lives on the device, so the
// grid is sized for the worst case and idle blocks exit at once.
void launch_screen_flagged(ea_ctx* ctx, const ScreenArgs& a) {
    const unsigned long long worst = a.nx * a.ny * a.it_count;
    unsigned long long blocks = std::min<unsigned long long>((worst + 255) / 256,
                                                             (unsigned long long)ctx->sm_count * 2);
    if (blocks == 0) blocks = 1;
    const int* tlist = a.amb + a.it_count;
    if (a.ignore)
        screen_general_kernel<true><<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, 0, tlist);
    else
        screen_general_kernel<false><<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, 0, tlist);
    check_launch("screen_general_kernel(flagged)");
    count_launch(ctx);
}

// ---- 3. threshold --------------------------------------------------------------
// Finds bin b holding the k-th largest screening score (b = bin(T_f) because
// fewer than k scores lie strictly above T_f), sets thr = lo(b) - 2*delta -
// 2^-20 (the slack covers fp32 rounding inside hist_bin) and an upper bound
// of the candidate count.
template <int BLOCK>
__device__ __forceinline__ float block_threshold(const unsigned* __restrict__ hist, int k,
                                                 double delta, SearchCtrl* ctrl,
                                                 bool write) {
    using Scan = cub::BlockScan<unsigned long long, BLOCK>;
    constexpr int PER = kHistBins / BLOCK;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int kbin;
    __shared__ float thr_s;
    const int t = threadIdx.x;
    unsigned long long local[PER], sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        local[j] = __ldcg(hist + kHistBins - 1 - (PER * t + j));
        sum += local[j];
    }
    unsigned long long excl;
    Scan(tmp).ExclusiveSum(sum, excl);
    if (t == 0) kbin = -1;
    __syncthreads();
    unsigned long long run = excl;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const unsigned long long before = run;
        run += local[j];
        if (before < (unsigned long long)k && run >= (unsigned long long)k)
            kbin = kHistBins - 1 - (PER * t + j);
    }
    __syncthreads();
    if (t == 0) {
        float thr = -INFINITY;
        if (kbin >= 0) {  // else fewer than k poses: every pose is a candidate
            const double lo = (double)kbin / 2048.0 - 1.0;
            const double th = lo - 2.0 * delta - 9.5367431640625e-07;  // 2^-20
            thr = (float)th;
            if ((double)thr > th) thr = nextafterf(thr, -INFINITY);
        }
        thr_s = thr;
        if (write) ctrl->thr = thr;
    }
    __syncthreads();
    return thr_s;
}

// Finds bin b holding the k-th largest screening score (b = bin(T_f) because
// fewer than k scores lie strictly above T_f) and sets thr = lo(b) - 2*delta -
// 2^-20 (the slack covers fp32 rounding inside hist_bin).
__global__ void __launch_bounds__(256) threshold_kernel(const unsigned* __restrict__ hist, int k,
                                                        double delta, SearchCtrl* ctrl) {
    block_threshold<256>(hist, k, delta, ctrl, true);
}

void launch_threshold(ea_ctx* ctx, const unsigned* hist, int k, double delta, SearchCtrl* ctrl) {
    threshold_kernel<<<1, 256, 0, ctx->stream>>>(hist, k, delta, ctrl);
    check_launch("threshold_kernel");
    count_launch(ctx);
}

// ---- 4. compaction -----------------------------------------------------------
// One warp per screening work item; items whose best score is below the band
// threshold are skipped without touching the map (typically all but the few
// tiles around the peaks).  Every block derives the band threshold from the
// histogram itself (block 0 publishes it), so no separate threshold launch.
__device__ __forceinline__ void compact_body(const float* __restrict__ map,
                                             const float* __restrict__ item_max,
                                             const ItemGeom& g, SearchCtrl* ctrl,
                                             unsigned* __restrict__ cand, unsigned long long cap,
                                             const float thr) {
    const int lane = threadIdx.x & 31;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const unsigned long long plane = g.nx * g.ny;
    for (unsigned long long it0 = warp; it0 < g.n_items; it0 += 8 * nwarps) {
        float best[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const unsigned long long it = it0 + q * nwarps;
            best[q] = it < g.n_items ? __ldg(item_max + it) : -INFINITY;
        }
#pragma unroll 1
        for (int q = 0; q < 8; ++q) {
        const unsigned long long it = it0 + q * nwarps;
        if (it >= g.n_items || !(best[q] >= thr)) continue;
        // a lane covers column (lane % cols) of rows (lane / cols) + k * rstep
        const unsigned rstep = g.lattice ? 32u / g.cols : 1u;
        const unsigned steps = g.lattice ? g.rows / rstep : 1u;
        unsigned long long base = 0, x = 0, y0 = 0;
        if (g.lattice) {
            const unsigned long long wx = it % g.nwx, rest = it / g.nwx;
            const unsigned long long wy = rest % g.nwy, itr = rest / g.nwy;
            base = itr * plane;
            x = wx * g.cols + lane % g.cols;
            y0 = wy * g.rows + lane / g.cols;
        }
        for (unsigned r0 = 0; r0 < steps; r0 += 16) {
            // 16 rows of loads in flight before any ballot/atomic
            float v[16];
            unsigned long long idx[16];
            bool okk[16];
#pragma unroll
            for (int qq = 0; qq < 16; ++qq) {
                const unsigned r = r0 + qq;
                if (g.lattice) {
                    const unsigned long long y = y0 + (unsigned long long)r * rstep;
                    okk[qq] = r < steps && x < g.nx && y < g.ny;
                    idx[qq] = base + y * g.nx + x;
                } else {
                    idx[qq] = it * 32 + lane;
                    okk[qq] = qq == 0 && idx[qq] < g.total;
                }
                v[qq] = okk[qq] ? __ldg(map + idx[qq]) : -INFINITY;
            }
#pragma unroll
            for (int qq = 0; qq < 16; ++qq) {
                const unsigned long long i = idx[qq];
                const bool pred = okk[qq] && v[qq] >= thr;
                const unsigned mask = __ballot_sync(0xffffffffu, pred);
                if (mask) {
                    const int leader = __ffs(mask) - 1;
                    unsigned long long slot0 = 0;
                    if (lane == leader)
                        slot0 = atomicAdd(&ctrl->cand_count, (unsigned long long)__popc(mask));
                    slot0 = __shfl_sync(0xffffffffu, slot0, leader);
                    if (pred) {
                        const unsigned long long slot = slot0 + __popc(mask & ((1u << lane) - 1u));
                        if (slot < cap) cand[slot] = (unsigned)i;
                    }
                }
            }
        }
        }
    }
}

__global__ void __launch_bounds__(256) compact_kernel(const float* __restrict__ map,
                                                      const float* __restrict__ item_max,
                                                      const ItemGeom g, SearchCtrl* ctrl,
                                                      unsigned* __restrict__ cand,
                                                      unsigned long long cap,
                                                      const unsigned* __restrict__ hist, int k,
                                                      double delta, const int* flags) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && flags) ctrl->flags = *flags;  // for the stats
    const float thr = block_threshold<256>(hist, k, delta, ctrl, blockIdx.x == 0);
    compact_body(map, item_max, g, ctrl, cand, cap, thr);
}

ItemGeom screen_items(const ScreenArgs& a, bool fast) {
    ItemGeom g{};
    g.nx = a.nx;
    g.ny = a.ny;
    g.total = a.nx * a.ny * a.it_count;
    if (fast) {
        const unsigned S = (unsigned)a.strip;  // lane-strip rows of the kernel that ran
        const unsigned XG = a.xg == 2 ? 2u : 4u;
        g.lattice = 1;
        g.cols = 8 * XG;
        g.rows = (32 / XG) * S;
        g.nwx = (unsigned)((a.lnx + g.cols - 1) / g.cols);
        g.nwy = (unsigned)((a.lny + g.rows - 1) / g.rows);
        g.sx = a.sx;
        g.sy = a.sy;
        g.n_items = (unsigned long long)g.nwx * g.nwy * a.it_count;
    } else {
        g.lattice = 0;
        g.n_items = (g.total + 31) / 32;
    }
    return g;
}

void launch_compact(ea_ctx* ctx, const float* map, const float* item_max, const ItemGeom& g,
                    SearchCtrl* ctrl, unsigned* cand, unsigned long long cap,
                    const unsigned* hist, int k, double delta, const int* flags) {
    unsigned long long blocks = (g.n_items * 32 + 255) / 256;
    const unsigned long long maxb = (unsigned long long)ctx->sm_count;
    if (blocks > maxb) blocks = maxb;
    if (blocks == 0) blocks = 1;
    compact_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(map, item_max, g, ctrl, cand, cap,
                                                              hist, k, delta, flags);
    check_launch("compact_kernel");
    count_launch(ctx);
}

// ---- 5. exact rescoring ------------------------------------------------------
// One warp per pose: lanes evaluate points lane, lane+32, ...; the votes are
// then added in model-point order (similarity.cpp:109-118) by a shuffle walk,
// so the fp64 sum is the reference's to the last bit.
__device__ __forceinline__ double warp_pose_score(const ExactArgs& a, size_t base, double ux,
                                                  double uy, int lane, int* n_inb) {
    const size_t S = a.rot_stride;
    double sum = 0.0;
    int inb_total = 0;
    for (int q = 0; q < a.n; q += 32) {
        const int i = q + lane;
        double v = 0.0;
        int inb = 0;
        if (i < a.n) {
            v = point_term_exact(__ldg(a.rot_exact + base + i), __ldg(a.rot_exact + S + base + i),
                                 __ldg(a.rot_exact + 2 * S + base + i),
                                 __ldg(a.rot_exact + 3 * S + base + i), ux, uy, a.gx, a.gy,
                                 a.mag, a.W, a.H, a.R, a.eps, a.ignore != 0, &inb);
        }
        inb_total += __popc(__ballot_sync(0xffffffffu, inb));
        const int lim = a.n - q < 32 ? a.n - q : 32;
        for (int l = 0; l < lim; ++l) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, v, l));
    }
    if (n_inb) *n_inb = inb_total;
    return __ddiv_rn(sum, (double)a.n);
}

// One CTA per candidate pose: every (model point, window pixel) candidate of
// the pose is evaluated in parallel in exact fp64 (kernels_scalar.cpp:43-54),
// the per-point window maximum is taken with integer-key shared atomics (max
// is order-free), and thread 0 adds the votes in model-point order
// (similarity.cpp:109-118) -- the reference's fp64 score to the last bit.
constexpr int kRescoreChunk = 256;

__device__ __forceinline__ void rescore_body(const ExactArgs& a,
                                             const unsigned* __restrict__ cand,
                                             const SearchCtrl* ctrl, unsigned long long cap,
                                             double* __restrict__ score) {
    __shared__ long long vmax[kRescoreChunk];
    __shared__ int2 centre[kRescoreChunk];
    unsigned long long nc = ctrl->cand_count;
    if (nc > cap) nc = cap;
    const unsigned long long plane = a.nx * a.ny;
    const int side = 2 * a.R + 1, W2 = side * side;
    const size_t S = a.rot_stride;
    const bool absolute = a.ignore != 0;
    for (unsigned long long c = blockIdx.x; c < nc; c += gridDim.x) {
        const unsigned long long rel = cand[c];
        const unsigned long long itl = rel / plane, rem = rel % plane;
        const double ux = lattice(a.x0, rem % a.nx, a.dx);
        const double uy = lattice(a.y0, rem / a.nx, a.dy);
        const size_t base = (size_t)itl * a.n;
        double sum = 0.0;
        for (int p0 = 0; p0 < a.n; p0 += kRescoreChunk) {
            const int cn = min(kRescoreChunk, a.n - p0);
            for (int t = threadIdx.x; t < cn; t += blockDim.x) {
                const size_t q = base + p0 + t;
                const double px = __dadd_rn(__ldg(a.rot_exact + q), ux);
                const double py = __dadd_rn(__ldg(a.rot_exact + S + q), uy);
                int2 cc = make_int2(-1, -1);  // (-1,-1): centre off the field, vote 0
                if (px > -kCoordGuard && px < kCoordGuard && py > -kCoordGuard &&
                    py < kCoordGuard) {
                    const int cx = (int)floor(__dadd_rn(px, 0.5));
                    const int cy = (int)floor(__dadd_rn(py, 0.5));
                    if (cx >= 0 && cx < a.W && cy >= 0 && cy < a.H) cc = make_int2(cx, cy);
                }
                centre[t] = cc;
                vmax[t] = LLONG_MIN;
            }
            __syncthreads();
            for (int t = threadIdx.x; t < cn * W2; t += blockDim.x) {
                const int i = t / W2, w = t % W2;
                const int2 cc = centre[i];
                if (cc.x < 0) continue;
                const int x = cc.x + w % side - a.R, y = cc.y + w / side - a.R;
                if (x < 0 || x >= a.W || y < 0 || y >= a.H) continue;  // clipped window
                const size_t o = (size_t)y * a.W + x;
                const size_t q = base + p0 + i;
                const double m = __ldg(a.mag + o);
                double cnd = 0.0;
                if (m >= a.eps) {
                    cnd = __ddiv_rn(__dadd_rn(__dmul_rn(__ldg(a.rot_exact + 2 * S + q), __ldg(a.gx + o)),
                                              __dmul_rn(__ldg(a.rot_exact + 3 * S + q), __ldg(a.gy + o))),
                                    m);
                }
                if (absolute) cnd = fabs(cnd);
                atomicMax(&vmax[i], order_key(cnd));
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int i = 0; i < cn; ++i)
                    sum = __dadd_rn(sum, centre[i].x < 0 ? 0.0 : from_order_key(vmax[i]));
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) score[c] = __ddiv_rn(sum, (double)a.n);
    }
}

__global__ void __launch_bounds__(256) rescore_kernel(const ExactArgs a,
                                                      const unsigned* __restrict__ cand,
                                                      const SearchCtrl* ctrl,
                                                      unsigned long long cap,
                                                      double* __restrict__ score) {
    rescore_body(a, cand, ctrl, cap, score);
}

void launch_rescore(ea_ctx* ctx, const ExactArgs& a, const unsigned* cand,
                    const SearchCtrl* ctrl, unsigned long long cap, double* score) {
    unsigned long long blocks = cap;
    const unsigned long long maxb = (unsigned long long)ctx->sm_count * 8;
    if (blocks > maxb) blocks = maxb;
    if (blocks == 0) blocks = 1;
    rescore_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, cand, ctrl, cap, score);
    check_launch("rescore_kernel");
    count_launch(ctx);
}

// ---- 6. top-k by `better` --------------------------------------------------------
struct Best {
    long long k;
    unsigned long long i;
    int ok;
};

// better (search.cpp:36-41) on order keys: score desc, then index asc.
__device__ __forceinline__ bool better_k(long long ka, unsigned long long ia, long long kb,
                                         unsigned long long ib) {
    if (ka != kb) return ka > kb;
    return ia < ib;
}

__device__ __forceinline__ Best pick(Best x, Best y) {
    if (!x.ok) return y;
    if (!y.ok) return x;
    return better_k(x.k, x.i, y.k, y.i) ? x : y;
}

constexpr int kStage = 2048;  // candidates staged in shared memory by select_body
// Shared-memory scratch of select_body (static in select_kernel /
// finish_kernel; carved from the plane's dynamic shared memory in the fused
// screen kernel, whose plane is dead by then).
struct SelectSmem {
    long long skey[kStage];
    unsigned long long sidx[kStage];
    Best warp_best[32];
    Best prev;
};

__device__ __forceinline__ void select_body(const unsigned* __restrict__ cand,
                                            const double* __restrict__ score, SearchCtrl* ctrl,
                                            unsigned long long cap, int k,
                                            unsigned long long index_base, double* out_score,
                                            unsigned long long* out_index, SelectSmem& sm) {
    long long* skey = sm.skey;
    unsigned long long* sidx = sm.sidx;
    Best* warp_best = sm.warp_best;
    Best& prev = sm.prev;
    unsigned long long nc = ctrl->cand_count;
    if (nc > cap) nc = cap;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (nc <= kStage) {
        // the block stages (score key, global index); one warp selects
        for (unsigned long long c = t; c < nc; c += blockDim.x) {
            skey[c] = order_key(score[c]);
            sidx[c] = index_base + cand[c];
        }
        __syncthreads();
        if (w != 0) return;
        Best p{0, 0ull, 0};
        int r = 0;
        for (; r < k; ++r) {
            Best b{0, 0ull, 0};
            for (int c = lane; c < (int)nc; c += 32) {
                const Best x{skey[c], sidx[c], 1};
                if (p.ok && !better_k(p.k, p.i, x.k, x.i)) continue;
                b = pick(b, x);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                Best o;
                o.k = __shfl_xor_sync(0xffffffffu, b.k, off);
                o.i = __shfl_xor_sync(0xffffffffu, b.i, off);
                o.ok = __shfl_xor_sync(0xffffffffu, b.ok, off);
                b = pick(b, o);
            }
            if (!b.ok) break;
            if (lane == 0) {
                out_score[r] = from_order_key(b.k);
                out_index[r] = b.i;
            }
            p = b;
        }
        if (lane == 0) ctrl->n_out = r;
        return;
    }
    // many candidates (degenerate, e.g. flat images): block-wide rounds
    int r = 0;
    for (; r < k; ++r) {
        Best b{0, 0ull, 0};
        for (unsigned long long c = t; c < nc; c += blockDim.x) {
            const long long kk = order_key(score[c]);
            const unsigned long long idx = index_base + cand[c];
            if (r > 0 && !better_k(prev.k, prev.i, kk, idx)) continue;
            b = pick(b, Best{kk, idx, 1});
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            Best o;
            o.k = __shfl_down_sync(0xffffffffu, b.k, off);
            o.i = __shfl_down_sync(0xffffffffu, b.i, off);
            o.ok = __shfl_down_sync(0xffffffffu, b.ok, off);
            b = pick(b, o);
        }
        if (lane == 0) warp_best[w] = b;
        __syncthreads();
        if (t == 0) {
            Best f{0, 0ull, 0};
            for (int q = 0; q < (int)(blockDim.x >> 5); ++q) f = pick(f, warp_best[q]);
            prev = f;
            if (f.ok) {
                out_score[r] = from_order_key(f.k);
                out_index[r] = f.i;
            }
        }
        __syncthreads();
        if (!prev.ok) break;
    }
    if (t == 0) ctrl->n_out = r;
}

__global__ void __launch_bounds__(256) select_kernel(const unsigned* __restrict__ cand,
                                                     const double* __restrict__ score,
                                                     SearchCtrl* ctrl, unsigned long long cap,
                                                     int k, unsigned long long index_base,
                                                     double* out_score,
                                                     unsigned long long* out_index) {
    __shared__ SelectSmem sm;
    select_body(cand, score, ctrl, cap, k, index_base, out_score, out_index, sm);
}

void launch_select(ea_ctx* ctx, const unsigned* cand, const double* score, SearchCtrl* ctrl,
                   unsigned long long cap, int k, unsigned long long index_base,
                   double* out_score, unsigned long long* out_index) {
    select_kernel<<<1, 256, 0, ctx->stream>>>(cand, score, ctrl, cap, k, index_base, out_score,
                                               out_index);
    check_launch("select_kernel");
    count_launch(ctx);
}

// ---- device-resident top-k rows (multi-GPU data path) ------------------------
// Row = {score, grid_index, ux, uy, theta} as five doubles (grid indices are
// < 2^53, so exact); rows past the count carry a NaN score.  The same layout
// is all-gathered over NCCL and merged on the device.
__device__ __forceinline__ void topk_rows_body(const double* __restrict__ score,
                                               const unsigned long long* __restrict__ index,
                                               const SearchCtrl* __restrict__ ctrl,
                                               unsigned long long cap, int k, const RowGrid& g,
                                               double* __restrict__ rows, int* overflow) {
    const int n = ctrl->n_out;
    // Band overflow (more candidates than the buffer): the rows are not the
    // slab's top k.  Flag it, and mark row 0 with score +inf so that the
    // mark survives an all-gather + `better` merge (it ranks first) and
    // every rank of a sharded search sees it.
    const bool over = ctrl->cand_count > cap;
    if (threadIdx.x == 0 && over && overflow) atomicOr(overflow, 1);
    const unsigned long long plane = g.nx * g.ny;
    for (int r = threadIdx.x; r < k; r += blockDim.x) {
        double* o = rows + 5 * (size_t)r;
        if (over && r == 0) {
            o[0] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
            o[1] = o[2] = o[3] = o[4] = 0.0;
        } else if (r < n) {
            const unsigned long long idx = index[r];
            const unsigned long long it = idx / plane, rem = idx % plane;
            o[0] = score[r];
            o[1] = (double)idx;
            o[2] = lattice(g.x0, rem % g.nx, g.dx);  // pose_at, pose.h:84-91
            o[3] = lattice(g.y0, rem / g.nx, g.dy);
            o[4] = lattice(g.t0, it, g.dt);
        } else {
            o[0] = __longlong_as_double(0x7ff8000000000000LL);  // NaN: empty row
            o[1] = o[2] = o[3] = o[4] = 0.0;
        }
    }
}

__global__ void topk_rows_kernel(const double* __restrict__ score,
                                 const unsigned long long* __restrict__ index,
                                 const SearchCtrl* __restrict__ ctrl, unsigned long long cap,
                                 int k, RowGrid g, double* __restrict__ rows, int* overflow) {
    topk_rows_body(score, index, ctrl, cap, k, g, rows, overflow);
}

// ---- fused finish: band threshold -> compaction -> exact rescore -> top k
// (-> rows) in ONE cooperative launch.  The separate kernels are latency
// chains (a few dependent memory round trips and barriers each, ~50 us for
// the four); here every phase is written for the shortest dependent chain:
//  A  threshold   every CTA scans the 4096-bin histogram (16 bins/thread,
//                 one load round trip, shuffle scans);
//  B  compaction  a warp tests 32 item maxima per load and gathers a
//                 qualifying tile with all 64 loads per lane in flight, one
//                 atomic slot reservation per tile;
//     grid barrier (the candidate count is final);
//  C  rescore     one CTA per candidate, one thread per model point: the
//                 window argmax by exact fraction compare and one division
//                 (vote_exact), votes added in point order by one thread;
//  D  select      the last CTA to finish C ranks the candidates by `better`
//                 (rank = how many candidates beat it: one pass, no rounds)
//                 and writes the top k (and the device rows).
// A: band threshold (block_threshold's result) with one load round trip.
__device__ __forceinline__ float finish_threshold(const unsigned* __restrict__ hist, int k,
                                                  double delta) {
    constexpr int PER = kHistBins / 256;  // blockDim.x == 256
    __shared__ unsigned wsum[8];
    __shared__ int kbin;
    __shared__ float thr_s;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    unsigned v[PER], sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {  // chunk t: bins counted from the top
        v[j] = __ldcg(hist + kHistBins - 1 - (PER * t + j));
        sum += v[j];
    }
    unsigned incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[w] = incl;
    if (t == 0) kbin = -1;
    __syncthreads();
    unsigned run = incl - sum;
    for (int q = 0; q < w; ++q) run += wsum[q];
    if (run < (unsigned)k && run + sum >= (unsigned)k) {
#pragma unroll 1
        for (int j = 0; j < PER; ++j) {
            run += v[j];
            if (run >= (unsigned)k) {
                kbin = kHistBins - 1 - (PER * t + j);
                break;
            }
        }
    }
    __syncthreads();
    if (t == 0) {
        float thr = -INFINITY;
        if (kbin >= 0) {  // else fewer than k poses: every pose is a candidate
            const double lo = (double)kbin / 2048.0 - 1.0;
            const double th = lo - 2.0 * delta - 9.5367431640625e-07;  // 2^-20
            thr = (float)th;
            if ((double)thr > th) thr = nextafterf(thr, -INFINITY);
        }
        thr_s = thr;
    }
    __syncthreads();
    return thr_s;
}

// B: one warp, one qualifying work item: every pose with S_f >= thr.  Lane
// addresses are one pointer + a 32-bit row stride, so the 64 loads issue back
// to back (64-bit index math per load made this a 4 us instruction chain).
// finish_tile for integer steps > 1: the unit-lattice tile's grid poses are
// the rectangle [ceil(x0/sx), ceil(x1/sx)) x [ceil(y0/sy), ceil(y1/sy)) of
// the grid; lanes walk it row-major (an exact-zero tile: its first k).
__device__ __noinline__ void finish_tile_strided(const FinishArgs& f, unsigned long long it,
                                                  float thr, int lane) {
    const ItemGeom& g = f.items;
    const unsigned long long wx = it % g.nwx, rest = it / g.nwx;
    const unsigned long long wy = rest % g.nwy, itr = rest / g.nwy;
    const unsigned long long sx = (unsigned)g.sx, sy = (unsigned)g.sy;
    const unsigned long long ix0 = (wx * g.cols + sx - 1) / sx;
    const unsigned long long ix1 = min(((wx + 1) * g.cols + sx - 1) / sx, g.nx);
    const unsigned long long iy0 = (wy * g.rows + sy - 1) / sy;
    const unsigned long long iy1 = min(((wy + 1) * g.rows + sy - 1) / sy, g.ny);
    if (ix0 >= ix1 || iy0 >= iy1) return;
    const unsigned long long w = ix1 - ix0, n = w * (iy1 - iy0);
    const unsigned long long base = itr * (g.nx * g.ny);
    const bool zero = f.zero_tiles && __ldg(f.zero_tiles + it % ((unsigned long long)g.nwx * g.nwy));
    const unsigned long long lim = zero ? min(n, (unsigned long long)f.k) : n;
    for (unsigned long long i0 = 0; i0 < lim; i0 += 32) {
        const unsigned long long i = i0 + lane;
        bool take = false;
        unsigned long long idx = 0;
        if (i < lim) {
            idx = base + (iy0 + i / w) * g.nx + ix0 + i % w;
            take = zero ? 0.0f >= thr : __ldcg(f.map + idx) >= thr;
        }
        const unsigned mask = __ballot_sync(0xffffffffu, take);
        if (!mask) continue;
        const int leader = __ffs(mask) - 1;
        unsigned long long slot0 = 0;
        if (lane == leader) slot0 = atomicAdd(&f.ctrl->cand_count, (unsigned long long)__popc(mask));
        slot0 = __shfl_sync(0xffffffffu, slot0, leader);
        if (take) {
            const unsigned long long slot = slot0 + __popc(mask & ((1u << lane) - 1u));
            if (slot < f.cap) f.cand[slot] = (unsigned)idx;
        }
    }
}

__device__ __forceinline__ void finish_tile(const FinishArgs& f, unsigned long long it,
                                            float thr, int lane) {
    const ItemGeom& g = f.items;
    if (g.lattice && (g.sx != 1 || g.sy != 1)) {  // integer steps > 1: the tile's grid poses
        finish_tile_strided(f, it, thr, lane);
        return;
    }
    if (f.zero_tiles && g.lattice && __ldg(f.zero_tiles + it % ((unsigned long long)g.nwx * g.nwy))) {
        // exact-zero tile: every pose scores 0 (and 0 >= thr, or none is a
        // candidate); only its first k poses in index order can rank -- any
        // other has k poses of equal score and smaller index in this tile
        if (lane == 0 && 0.0f >= thr) {
            const unsigned long long wx = it % g.nwx, rest = it / g.nwx;
            const unsigned long long wy = rest % g.nwy, itr = rest / g.nwy;
            const unsigned long long x0 = wx * g.cols, y0 = wy * g.rows;
            int got = 0;
            for (unsigned long long y = y0; y < y0 + g.rows && y < g.ny && got < f.k; ++y)
                for (unsigned long long x = x0; x < x0 + g.cols && x < g.nx && got < f.k; ++x, ++got) {
                    const unsigned long long slot = atomicAdd(&f.ctrl->cand_count, 1ull);
                    if (slot < f.cap) f.cand[slot] = (unsigned)(itr * (g.nx * g.ny) + y * g.nx + x);
                }
        }
        return;
    }
    constexpr int kMaxSteps = 64;  // 32 lanes x 64 = one 2048-pose lattice tile
    const float kNaN = __int_as_float(0x7fffffff);  // never >= thr, even thr = -inf
    const float* p;
    unsigned stride = 0;
    int nrows;  // rows of this lane inside the grid
    unsigned long long first;  // slab-relative pose index of the lane's row 0
    if (g.lattice) {
        const unsigned rstep = 32u / g.cols;
        const unsigned long long wx = it % g.nwx, rest = it / g.nwx;
        const unsigned long long wy = rest % g.nwy, itr = rest / g.nwy;
        const unsigned long long x = wx * g.cols + lane % g.cols;
        const unsigned long long y0 = wy * g.rows + lane / g.cols;
        const unsigned steps = g.rows / rstep;
        nrows = 0;
        if (x < g.nx && y0 < g.ny) {
            const unsigned long long left = (g.ny - y0 + rstep - 1) / rstep;
            nrows = (int)(left < steps ? left : steps);
        }
        stride = rstep * (unsigned)g.nx;
        first = itr * (g.nx * g.ny) + y0 * g.nx + x;
    } else {
        first = it * 32 + lane;
        nrows = first < g.total ? 1 : 0;
    }
    p = f.map + first;
    float v[kMaxSteps];
#pragma unroll
    for (int r = 0; r < kMaxSteps; ++r) v[r] = r < nrows ? __ldcg(p + r * stride) : kNaN;
    unsigned cnt = 0;
#pragma unroll
    for (int r = 0; r < kMaxSteps; ++r) cnt += v[r] >= thr ? 1u : 0u;
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    unsigned long long slot0 = 0;
    if (lane == 31) slot0 = atomicAdd(&f.ctrl->cand_count, (unsigned long long)total);
    unsigned long long slot = __shfl_sync(0xffffffffu, slot0, 31) + (incl - cnt);
    if (cnt == 0) return;
#pragma unroll
    for (int r = 0; r < kMaxSteps; ++r) {  // unrolled: v stays in registers
        if (v[r] >= thr) {
            if (slot < f.cap) f.cand[slot] = (unsigned)(first + (unsigned long long)r * stride);
            ++slot;
        }
    }
}

// C: exact fp64 score of candidate c with the whole CTA (reference order).
constexpr int kMaxFinishThreads = 384;  // finish phases run with 256 (finish_kernel) or 384 threads

__device__ __forceinline__ void finish_rescore(const ExactArgs& a, unsigned rel_idx,
                                               double* out, double* votes /* smem, blockDim */) {
    const unsigned long long plane = a.nx * a.ny;
    const unsigned long long itl = rel_idx / plane, rem = rel_idx % plane;
    const double ux = lattice(a.x0, rem % a.nx, a.dx);
    const double uy = lattice(a.y0, rem / a.nx, a.dy);
    const size_t S = a.rot_stride, base = (size_t)itl * a.n;
    const int t = threadIdx.x;
    double sum = 0.0;
    const int nt = blockDim.x;
    for (int p0 = 0; p0 < a.n; p0 += nt) {
        const int i = p0 + t;
        double v = 0.0;  // off-field centre / guarded coordinate: vote 0 (x + 0.0 == x)
        if (i < a.n) {
            const double px = __dadd_rn(__ldg(a.rot_exact + base + i), ux);
            const double py = __dadd_rn(__ldg(a.rot_exact + S + base + i), uy);
            if (px > -kCoordGuard && px < kCoordGuard && py > -kCoordGuard && py < kCoordGuard) {
                const int cx = (int)floor(__dadd_rn(px, 0.5));
                const int cy = (int)floor(__dadd_rn(py, 0.5));
                if (cx >= 0 && cx < a.W && cy >= 0 && cy < a.H)
                    v = vote_exact(a.gx, a.gy, a.mag, a.W, a.H, cx, cy, a.R,
                                   __ldg(a.rot_exact + 2 * S + base + i),
                                   __ldg(a.rot_exact + 3 * S + base + i), a.eps, a.ignore != 0);
            }
        }
        votes[t] = v;
        __syncthreads();
        if (t == 0) {
            const int cn = min(nt, a.n - p0);
            int j = 0;
            for (; j + 8 <= cn; j += 8) {  // 8 loads in flight, then the ordered adds
                double b[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) b[q] = votes[j + q];
#pragma unroll
                for (int q = 0; q < 8; ++q) sum = __dadd_rn(sum, b[q]);
            }
            for (; j < cn; ++j) sum = __dadd_rn(sum, votes[j]);
        }
        __syncthreads();
    }
    if (t == 0) *out = __ddiv_rn(sum, (double)a.n);
}

// D: top k by `better` (score desc, index asc) as ranks; n_out = min(k, nc).
constexpr int kRankMax = 512;  // candidates ranked in one pass; more: select_body rounds
__device__ __forceinline__ void finish_select(const FinishArgs& f, unsigned long long nc,
                                              long long* skey, unsigned long long* sidx) {
    const int t = threadIdx.x;
    for (unsigned long long c = t; c < nc; c += blockDim.x) {
        skey[c] = order_key(__ldcg(f.cand_score + c));
        sidx[c] = f.index_base + __ldcg(f.cand + c);
    }
    __syncthreads();
    for (unsigned long long c = t; c < nc; c += blockDim.x) {
        const long long kc = skey[c];
        const unsigned long long ic = sidx[c];
        int r = 0;
        for (unsigned long long j = 0; j < nc && r < f.k; ++j)
            r += better_k(skey[j], sidx[j], kc, ic) ? 1 : 0;
        if (r < f.k) {
            f.out_score[r] = from_order_key(kc);
            f.out_index[r] = ic;
        }
    }
    if (t == 0) f.ctrl->n_out = (int)(nc < (unsigned long long)f.k ? nc : (unsigned long long)f.k);
}

#define EAB_PROF(slot)                                                                    \
    if (f.prof) {                                                                         \
        __syncthreads();                                                                  \
        if (threadIdx.x == 0) atomicMax(f.prof + (slot), gtimer() - f.prof[15]);          \
    }

// B: warps take 32 consecutive items per item_max load.  Lane l of warp w
// tests item w + l*nwarps (+ 32*nwarps per round): the qualifying tiles
// cluster around the peaks (same translation tile, adjacent thetas) and this
// spreads them over warps.
__device__ __forceinline__ void finish_compact_phase(const FinishArgs& f, float thr) {
    const int lane = threadIdx.x & 31;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long tb0 = f.prof ? gtimer() : 0;
    unsigned ntiles = 0;
    for (unsigned long long b0 = warp; b0 < f.items.n_items; b0 += nwarps * 32) {
        const unsigned long long it = b0 + (unsigned long long)lane * nwarps;
        const float m = it < f.items.n_items ? __ldcg(f.item_max + it)
                                             : __int_as_float(0x7fffffff);  // NaN: skip
        unsigned mask = __ballot_sync(0xffffffffu, m >= thr);
        while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            finish_tile(f, b0 + (unsigned long long)j * nwarps, thr, lane);
            ++ntiles;
        }
    }
    if (f.prof && lane == 0) {
        atomicMax(f.prof + 8, (unsigned long long)ntiles);
        atomicMax(f.prof + 10, gtimer() - tb0);
    }
}

// C: one CTA per candidate (after a grid barrier: the count is final).
// Shared-memory scratch of the finish phases C and D.
constexpr int kMaxScreenCtas = 512;  // per-CTA top lists merged by fused_threshold
union FinishSmem {
    double votes[kMaxFinishThreads];
    SelectSmem sel;
    float ttop[kMaxScreenCtas * kTopK];
};

__device__ __forceinline__ unsigned long long finish_rescore_phase(const FinishArgs& f,
                                                                   FinishSmem& sm) {
    unsigned long long nc = __ldcg(&f.ctrl->cand_count);
    if (nc > f.cap) nc = f.cap;  // overflow: reported, the caller retries with a larger cap
    for (unsigned long long c = blockIdx.x; c < nc; c += gridDim.x)
        finish_rescore(f.x, __ldcg(f.cand + c), f.cand_score + c, sm.votes);
    return nc;
}

// D on the CTA that finishes C last: select + rows; resets the ticket.
__device__ __forceinline__ void finish_select_phase(const FinishArgs& f, unsigned long long nc,
                                                    FinishSmem& sm) {
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&f.ctrl->finish_ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    __syncthreads();  // the rescore's vote scratch is reused below
    if (nc <= (unsigned long long)kRankMax)
        finish_select(f, nc, sm.sel.skey, sm.sel.sidx);
    else
        select_body(f.cand, f.cand_score, f.ctrl, f.cap, f.k, f.index_base, f.out_score,
                    f.out_index, sm.sel);
    if (threadIdx.x == 0) f.ctrl->finish_ticket = 0u;
    __syncthreads();
    if (f.rows) topk_rows_body(f.out_score, f.out_index, f.ctrl, f.cap, f.k, f.rg, f.rows,
                               f.overflow);
}

__global__ void __launch_bounds__(256) finish_kernel(const FinishArgs f) {
    cg::grid_group grid = cg::this_grid();
    if (f.prof && blockIdx.x == 0 && threadIdx.x == 0) {
        f.prof[15] = gtimer();
        __threadfence();
    }
    if (f.prof) grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0 && f.flags) f.ctrl->flags = *f.flags;
    __shared__ FinishSmem sm;
    // band threshold: from the screen's per-CTA lists of largest tile maxima
    // (top-list mode) or from the histogram
    const float thr = f.cta_top ? fused_threshold(f, sm.ttop) : finish_threshold(f.hist, f.k, f.delta);
    if (blockIdx.x == 0 && threadIdx.x == 0) f.ctrl->thr = thr;
    EAB_PROF(0)
    finish_compact_phase(f, thr);
    EAB_PROF(1)
    grid.sync();
    EAB_PROF(2)
    // Every CTA has read the histogram: leave it zero, and the screen's work
    // counter at 0, for the next search (which may skip the plane kernel that
    // would otherwise clear them).  (Top-list mode never touched it.)
    if (!f.cta_top)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kHistBins;
             i += gridDim.x * blockDim.x)
            f.hist_rw[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        f.ctrl->work_counter = 0ull;
        f.ctrl->gfloor = 0u;  // the screen's top-list floor, for the next search
    }
    const unsigned long long nc = finish_rescore_phase(f, sm);
    EAB_PROF(3)
    finish_select_phase(f, nc, sm);
    EAB_PROF(4)
    EAB_PROF(5)
}
#undef EAB_PROF

// ---- the smem lattice kernel (after the finish phases: its fused variant runs them)
// FUSED: the finish (band threshold from the exact k-th largest score,
// compaction, exact rescore, select, rows) runs in the same cooperative
// launch after grid barriers; no histogram (its 16 KB go to the plane).
template <int R, int S, int SHIFT, bool IGNORE, int XG, bool EDGE, int THREADS, bool FUSED,
          int MODE>
__global__ void __launch_bounds__(THREADS, 1)
    screen_fast_kernel(const ScreenArgs a, const unsigned nwx, const unsigned nwy,
                       const TailPlan tp, const int vec16, const FinishArgs fa) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned* hist = reinterpret_cast<unsigned*>(smem);
    float2* P = reinterpret_cast<float2*>(smem + (FUSED ? 0 : kHistBins * sizeof(unsigned)));
    static_assert(kFloorK == kTopK, "one per-warp list serves both paths");
    __shared__ __align__(16) float wtop_all[16][kFloorK];
    __shared__ __align__(8) unsigned long long plane_bar;
    float* wtop = wtop_all[threadIdx.x >> 5];
    if ((threadIdx.x & 31) < kFloorK) wtop[threadIdx.x & 31] = -INFINITY;
    if (a.prof && threadIdx.x == 0) atomicMin(a.prof + 4, gtimer());  // first CTA entry
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl->cand_count = 0ull;  // for the finish
    // The plane arrives by bulk copy (TMA engine, one thread issues it) while
    // the threads clear the histogram.
    if (threadIdx.x == 0) {
        mbar_init(&plane_bar, 1);
        bulk_copy_to_smem(P, a.plane, (unsigned)vec16 * 16u, &plane_bar);
    }
    // top-list mode (fused, or a.cta_top set): no histogram -- the band
    // threshold comes from the CTAs' lists of their largest tile maxima
    const bool toplist = FUSED || a.cta_top != nullptr;
    if (!toplist)
        for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    mbar_wait_parity(&plane_bar, 0);
    if (a.prof && threadIdx.x == 0) atomicMin(a.prof + 0, gtimer());  // first plane landed

    constexpr int NACC = S * kTW;
    const int lane = threadIdx.x & 31;
    constexpr int YG = 32 / XG;  // lane strips along y; XG groups of 8 columns along x
    const int yg = lane % YG, xg = lane / YG;
    const float K = a.K;
    const unsigned long long total = tp.n_main + tp.n_tail * (unsigned long long)tp.f;
    const size_t sstride = sched_stride(a.n);

    LaneGeom g;
    g.P = P;
    g.PW = a.geom.PW;
    g.XL = a.geom.PW - 1;
    g.cx_lo = 1 + a.geom.PL;
    g.cx_hi = a.geom.W + a.geom.PL;
    g.H1 = a.geom.H + 1;
    g.Z = a.geom.zero;
    g.ry_lo = 1;
    g.ry_hi = a.geom.H;
    g.wspan = 8 * (XG - 1);

    unsigned long long* wt = a.wtrace ? a.wtrace + 8 * (size_t)(blockIdx.x * (blockDim.x >> 5) +
                                                                 (threadIdx.x >> 5))
                                      : nullptr;
    int units = 0;
    if (wt && lane == 0) wt[0] = gtimer();
    for (;;) {
        if (wt && lane == 0 && units > 0 && units < 7) wt[units] = gtimer();
        unsigned long long work = 0;
        if (lane == 0) work = atomicAdd(&a.ctrl->work_counter, 1ull);
        work = __shfl_sync(0xffffffffu, work, 0);
        if (work >= total) break;
        ++units;
        unsigned long long item = work;
        long long tslot = -1;
        int ch = 0;
        if (work >= tp.n_main) {
            const unsigned long long m = work - tp.n_main;
            tslot = (long long)(m / (unsigned)tp.f);
            ch = (int)(m % (unsigned)tp.f);
            item = tp.n_main + (unsigned long long)tslot;
        }
        const unsigned wx = (unsigned)(item % nwx);
        const unsigned long long rest = item / nwx;
        const unsigned wy = (unsigned)(rest % nwy);
        const unsigned long long itr = rest / nwy;
        const int X0 = (int)wx * (8 * XG);
        const int X = X0 + xg * kTW;
        const int Y = (int)wy * (YG * S) + yg * S;
        if (__ldg(a.amb + itr) != 0) {  // flagged theta: the general kernel scores it
            if (lane == 0) a.item_max[item] = INFINITY;
            continue;
        }
        const int4* sch = a.sched + itr * sstride;
        const int4 hdr = __ldg(sch);
        const int n_ent = hdr.x + hdr.y + hdr.z;
        int e0 = 0, e1 = n_ent;
        if (tslot >= 0) {
            e0 = (int)((long long)ch * n_ent / tp.f);
            e1 = (int)((long long)(ch + 1) * n_ent / tp.f);
        }
        // exact-zero tile: no entries, every score the fixed-point 0
        if (a.zero_tiles && __ldg(a.zero_tiles + (size_t)wy * nwx + wx)) e0 = e1 = 0;
        g.cbase = a.ix0 + X - R + g.cx_lo;   // padded column of the window start - ox
        g.rbase = a.iy0 + Y - R + 1;         // padded row of the window start - oy
        g.cwbase = a.ix0 + X0 - R + g.cx_lo; // warp's first column - ox

        unsigned acc[S][kTW];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int j = 0; j < kTW; ++j) acc[s][j] = 0u;
        const int done = run_entries<R, S, SHIFT, IGNORE, EDGE, true, MODE>(sch + 1, hdr, e0, e1,
                                                                           g, K, acc);
        int sc[S][kTW];
        const unsigned corr = (unsigned)done * a.B3;
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int j = 0; j < kTW; ++j) sc[s][j] = (int)(acc[s][j] - corr);
        if (tslot >= 0) {  // micro-item: merge, last arrival finalises
            int* part = tp.part + (size_t)tslot * NACC * 32;
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int j = 0; j < kTW; ++j) atomicAdd(part + (s * kTW + j) * 32 + lane, sc[s][j]);
            __threadfence();
            unsigned old = 0;
            if (lane == 0) old = atomicAdd(tp.done + tslot, 1u);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old != (unsigned)tp.f - 1u) continue;
            __threadfence();
            // read the merged sums and leave the slot zeroed for the next
            // launch (no per-launch memset of the partial buffer)
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int j = 0; j < kTW; ++j) {
                    sc[s][j] = __ldcg(part + (s * kTW + j) * 32 + lane);
                    __stcg(part + (s * kTW + j) * 32 + lane, 0);
                }
            if (lane == 0) tp.done[tslot] = 0u;
        }
        // fused: no histogram; wtop keeps the warp's 8 largest tile maxima
        const float wf = warp_floor(wtop, a.kf);
        float lbest;
        emit_tile<S, !FUSED>(a, sc, X, Y, itr, item, toplist ? nullptr : hist, lane, wf,
                             toplist ? map_floor_of(a, wf) : -INFINITY, lbest);
        floor_insert_lanes(wtop, lbest, a.kf, lane);
        if (toplist) publish_floor(a, wtop, lane);
    }
    if (wt && lane == 0) wt[7] = ((unsigned long long)units << 56) | (gtimer() & ((1ull << 56) - 1));
    if (a.prof && (threadIdx.x & 31) == 0) atomicMax(a.prof + 1, gtimer());  // last warp's loop end
    __syncthreads();
    if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 2, gtimer());  // last CTA's loop end
    if (toplist) {
        // the CTA's kf largest tile maxima (merge of its warps' lists, warp 0)
        if (threadIdx.x < 32) {
            float* out = a.cta_top + blockIdx.x * kTopK;
            warp_kth_of_lists<1, false>(&wtop_all[0][0], blockDim.x >> 5, a.kf, out, threadIdx.x);
            if (threadIdx.x >= a.kf && threadIdx.x < kTopK) out[threadIdx.x] = -INFINITY;
        }
    } else {
        merge_hist(hist, a.hist, a.kf);
    }
    if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 3, gtimer());  // last merge end
    if constexpr (FUSED) {
        cg::grid_group grid = cg::this_grid();
        grid.sync();  // every CTA's list is written; the work counter is free
        if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 11, gtimer());  // barrier 1 passed
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.ctrl->work_counter = 0ull;
            a.ctrl->gfloor = 0u;
            a.ctrl->flags = 0;
        }
        // the plane is dead: its shared memory becomes the finish's scratch
        const float thr = fused_threshold(fa, reinterpret_cast<float*>(smem));
        if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl->thr = thr;
        if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 8, gtimer());  // threshold known
        finish_compact_phase(fa, thr);
        if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 9, gtimer());  // compaction done
        grid.sync();
        if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 5, gtimer());  // barrier 2 passed
        FinishSmem& fsm = *reinterpret_cast<FinishSmem*>(smem);
        const unsigned long long nc = finish_rescore_phase(fa, fsm);
        if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 6, gtimer());  // rescore done
        finish_select_phase(fa, nc, fsm);
        if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 7, gtimer());  // select + rows done
    }
}

template <int R, int S, int SHIFT, bool IGNORE, int XG, bool EDGE, int THREADS, bool FUSED,
          int MODE>
static void run_fast(ea_ctx* ctx, const ScreenArgs& a, const FinishArgs* fin) {
    constexpr int YG = 32 / XG;
    const unsigned nwx = (unsigned)((a.lnx + 8 * XG - 1) / (8 * XG));
    const unsigned nwy = (unsigned)((a.lny + YG * S - 1) / (YG * S));
    const unsigned long long items = (unsigned long long)nwx * nwy * a.it_count;
    const size_t plane_bytes = (a.geom.bytes() + 15) & ~(size_t)15;
    // fused: no histogram; the plane's bytes are reused by the finish phases
    const size_t smem =
        FUSED ? std::max({plane_bytes, sizeof(FinishSmem),
                          (size_t)ctx->sm_count * kTopK * sizeof(float)})
              : kHistBins * sizeof(unsigned) + plane_bytes;
    auto kern = screen_fast_kernel<R, S, SHIFT, IGNORE, XG, EDGE, THREADS, FUSED, MODE>;
    raise_smem_limit(ctx, (const void*)kern, smem);
    constexpr int threads = THREADS;
    const unsigned long long warps_per_cta = threads / 32;
    const bool split = std::getenv("EAB_NO_TAIL_SPLIT") == nullptr;
    // Full grid (one CTA per SM) whenever the items can be split into enough
    // point-chunks to occupy it: a theta slab of a sharded search (or any
    // small grid) has fewer warp tiles than the P resident warps.
    const int fmax = split && a.n >= 8 ? std::min(a.n / 4, 64) : 1;
    unsigned long long ctas = (items * (unsigned long long)fmax + warps_per_cta - 1) / warps_per_cta;
    if (ctas > (unsigned long long)ctx->sm_count) ctas = ctx->sm_count;
    if (ctas == 0) ctas = 1;
    // tail split (see TailPlan): the last partial round of `rem` items is cut
    // into f chunks, f minimising the tail's makespan in item units
    //   max(rem * (1 + c*f) / P, 1/f + c)
    // -- warps pull micro-items dynamically, so the tail ends when either its
    // total work (spread over P warps) or one chunk's latency is done; c ~ 6%
    // of an item is a chunk's fixed cost (prologue, partial-sum merge,
    // finalise).  Fitted on the B200 (profiles/r01.md, EAB_TAIL_F sweep): a
    // 1/8 theta slab of cfg2 (900 items on 1776 warps) is fastest at f = 2
    // (0.095 ms screen vs 0.118 at the f = 7 the older ceil-rounds model
    // chose), cfg3's slab at f = 6-9; a tail of nearly a full round (full
    // cfg3: 1632 items on 1776 warps) stays unsplit -- f = 2 measured +4%.
    TailPlan tp{items, 0, 1, nullptr, nullptr};
    const unsigned long long P = ctas * warps_per_cta;
    const unsigned long long rem = items % P;
    if (rem > 0 && fmax >= 2) {
        constexpr double c = 0.06;
        auto makespan = [&](int ff) {  // an unsplit item pays no chunk cost
            const double cf = ff > 1 ? c : 0.0;
            return std::max((double)rem * (1.0 + cf * ff) / (double)P, 1.0 / ff + cf);
        };
        int f = 1;
        double best = makespan(1);
        for (int ff = 2; ff <= fmax; ++ff) {
            const double cost = makespan(ff);
            if (cost < best - 1e-9) {
                best = cost;
                f = ff;
            }
        }
        // A chunk count just above P puts a second wave of chunks at the
        // end: with near-uniform item costs (cfg3: 49 points, per-theta cost
        // spread 0.9%) its 1/8 theta slab (204 tail items on 1776 warps) ended
        // its loop at 94-98 us with f = 9 (1836 chunks); cut to the largest f
        // that still fits one wave when that keeps a split.
        if (f >= 2 && rem * (unsigned long long)f > P && rem * (unsigned long long)f * 5 < P * 6 &&
            P / rem >= 2)
            f = (int)(P / rem);
        if (const char* ef = std::getenv("EAB_TAIL_F")) {  // diagnostic A/B of the split factor
            const int v = std::atoi(ef);
            if (v >= 1 && v <= fmax) f = v;
        }
        if (f >= 2) {
            tp.n_main = items - rem;
            tp.n_tail = rem;
            tp.f = f;
            // Partial sums and arrival counters are zero between launches:
            // cleared once at allocation, then by each slot's finaliser.
            const size_t part_bytes = rem * (size_t)S * kTW * 32 * sizeof(int);
            const size_t bytes = part_bytes + rem * sizeof(unsigned);
            const void* before = ctx->tail.p;
            const size_t cap_before = ctx->tail.cap;
            char* buf = (char*)ctx->tail.ensure(bytes);
            if (buf != before || ctx->tail.cap != cap_before)
                EAB_CUDA(cudaMemsetAsync(buf, 0, ctx->tail.cap, ctx->stream));
            // layout: partials of slot i at [i], counters after the largest
            // partial block the buffer can hold, so a slot's counter never
            // aliases another launch's partials
            tp.part = (int*)buf;
            tp.done = (unsigned*)(buf + ctx->tail.cap - rem * sizeof(unsigned));
        }
    }
    ctx->screen_ctas = (int)ctas;  // the finish merges this many per-CTA top lists
    const int vec16 = (int)(plane_bytes / 16);
    if constexpr (FUSED) {
        // every CTA must be resident for the grid barriers (one per SM)
        FinishArgs fa = *fin;
        fa.n_lists = (int)ctas;
        ScreenArgs sa = a;
        unsigned gx = nwx, gy = nwy;
        TailPlan t = tp;
        int v16 = vec16;
        void* args[] = {&sa, &gx, &gy, &t, &v16, &fa};
        EAB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)ctas), dim3(threads),
                                             args, smem, ctx->stream));
        check_launch("screen_fast_kernel(fused)");
    } else {
        kern<<<(unsigned)ctas, threads, smem, ctx->stream>>>(a, nwx, nwy, tp, vec16, FinishArgs{});
        check_launch("screen_fast_kernel");
    }
    count_launch(ctx);
}

// CTA size of the fully padded 8-row kernel: kFastThreads (12 warps x 168
// registers) for 3x3 windows; 8 warps for 5x5 (R = 2 spilled ~600 B at 168
// registers; cfg2 at nb 5: 1.167 -> 1.101 ms).
constexpr int fast_threads(int R) { return R >= 2 ? 256 : kFastThreads; }

size_t fast_smem_bytes(const PlaneGeom& g) {
    return kHistBins * sizeof(unsigned) + ((g.bytes() + 15) & ~(size_t)15);
}

bool launch_screen_fast(ea_ctx* ctx, const ScreenArgs& a) {
    if (fast_smem_bytes(a.geom) > ctx->smem_optin) return false;
    if (a.geom.elem_bytes != 8) return false;
    if (a.sched_mode == 1 && a.R > 1) return false;
    const bool ig = a.ignore != 0;
    if (a.geom.shift == 2) {  // 4-row lane strips: 32 accumulators, 16 warps (EAB_S4)
        if (a.edge != 0 || a.R > 1) return false;
#define EAB_FAST4(RR, MM)                                                                    \
    if (a.xg == 2) {                                                                         \
        if (ig) run_fast<RR, 4, 2, true, 2, false, 512, false, MM>(ctx, a, nullptr);        \
        else run_fast<RR, 4, 2, false, 2, false, 512, false, MM>(ctx, a, nullptr);          \
    } else {                                                                                 \
        if (ig) run_fast<RR, 4, 2, true, 4, false, 512, false, MM>(ctx, a, nullptr);        \
        else run_fast<RR, 4, 2, false, 4, false, 512, false, MM>(ctx, a, nullptr);          \
    }
        if (a.R == 1) {
            if (a.sched_mode == 1) { EAB_FAST4(1, 1) } else { EAB_FAST4(1, 0) }
        } else {
            if (a.sched_mode == 1) { EAB_FAST4(0, 1) } else { EAB_FAST4(0, 0) }
        }
#undef EAB_FAST4
        return true;
    }
    if (a.geom.shift != 3) return false;  // 8-row lane strips
    // Windows that may leave the padded plane (padding shrunk to fit shared
    // memory) need the clamping variant; fully padded planes run the lighter
    // kernel, whose register budget allows kFastThreads threads.
    const bool edge = a.edge != 0;
#define EAB_FAST_XG(RR, XGV, MM)                                                                \
    if (edge) {                                                                                 \
        if (ig) run_fast<RR, 8, 3, true, XGV, true, 256, false, MM>(ctx, a, nullptr);          \
        else run_fast<RR, 8, 3, false, XGV, true, 256, false, MM>(ctx, a, nullptr);            \
    } else {                                                                                    \
        if (ig) run_fast<RR, 8, 3, true, XGV, false, fast_threads(RR), false, MM>(ctx, a, nullptr);\
        else run_fast<RR, 8, 3, false, XGV, false, fast_threads(RR), false, MM>(ctx, a, nullptr);  \
    }
#define EAB_FAST_M(RR, MM)                                                  \
    if (a.xg == 2) {                                                        \
        EAB_FAST_XG(RR, 2, MM)                                              \
    } else {                                                                \
        EAB_FAST_XG(RR, 4, MM)                                              \
    }
#define EAB_FAST(RR)                                                        \
    if (a.R == RR) {                                                        \
        if (a.sched_mode == 1) {                                            \
            EAB_FAST_M(RR, 1)                                               \
        } else {                                                            \
            EAB_FAST_M(RR, 0)                                               \
        }                                                                   \
        return true;                                                        \
    }
    EAB_FAST(1)
    EAB_FAST(0)
    if (a.R == 2) {
        EAB_FAST_M(2, 0)
        return true;
    }
#undef EAB_FAST
#undef EAB_FAST_M
#undef EAB_FAST_XG
    return false;
}

bool launch_screen_fused(ea_ctx* ctx, const ScreenArgs& a, const FinishArgs& f) {
    if (fast_smem_bytes(a.geom) > ctx->smem_optin) return false;
    if (a.geom.shift != 3 || a.geom.elem_bytes != 8) return false;
    if (a.edge != 0 || a.kf < 1 || a.kf > kTopK || f.k != a.kf || !f.cta_top) return false;
    if (a.sched_mode == 1 && a.R > 1) return false;
    const bool ig = a.ignore != 0;
#define EAB_FUSED_M(RR, MM)                                                                       \
    if (a.xg == 2) {                                                                              \
        if (ig) run_fast<RR, 8, 3, true, 2, false, kFastThreads, true, MM>(ctx, a, &f);           \
        else run_fast<RR, 8, 3, false, 2, false, kFastThreads, true, MM>(ctx, a, &f);             \
    } else {                                                                                      \
        if (ig) run_fast<RR, 8, 3, true, 4, false, kFastThreads, true, MM>(ctx, a, &f);           \
        else run_fast<RR, 8, 3, false, 4, false, kFastThreads, true, MM>(ctx, a, &f);             \
    }
#define EAB_FUSED(RR)                                                                             \
    if (a.R == RR) {                                                                              \
        if (a.sched_mode == 1) {                                                                  \
            EAB_FUSED_M(RR, 1)                                                                    \
        } else {                                                                                  \
            EAB_FUSED_M(RR, 0)                                                                    \
        }                                                                                         \
        return true;                                                                              \
    }
    EAB_FUSED(1)
    EAB_FUSED(0)
    if (a.R == 2) {
        EAB_FUSED_M(2, 0)
        return true;
    }
#undef EAB_FUSED
#undef EAB_FUSED_M
    return false;
}


void launch_finish(ea_ctx* ctx, const FinishArgs& f) {
    static int per_sm = -1;  // co-resident CTAs per SM (same binary for every device)
    if (per_sm < 0) {
        EAB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, finish_kernel, 256, 0));
        if (per_sm < 1) fail(EA_ERR_CUDA, "finish_kernel cannot be resident");
    }
    // One CTA per SM: rescoring is one CTA per candidate; more CTAs only make
    // the grid barrier dearer for the common case of a handful of candidates.
    static const int per_sm_use = std::getenv("EAB_FINISH_PER_SM")
                                      ? std::atoi(std::getenv("EAB_FINISH_PER_SM")) : 1;
    const unsigned blocks = (unsigned)ctx->sm_count * (unsigned)std::max(1, std::min(per_sm, per_sm_use));
    FinishArgs fa = f;
    static unsigned long long* prof = nullptr;  // EAB_FINISH_PROF: phase timestamps
    static int nprof = 0;
    if (std::getenv("EAB_FINISH_PROF")) {
        unsigned long long h[16];
        if (!prof) {
            EAB_CUDA(cudaMalloc(&prof, 16 * sizeof(unsigned long long)));
        } else if (nprof > 0) {
            EAB_CUDA(cudaStreamSynchronize(ctx->stream));
            EAB_CUDA(cudaMemcpy(h, prof, sizeof h, cudaMemcpyDeviceToHost));
            std::fprintf(stderr, "[finish] ns thr/compact/barrier/rescore/select/rows:");
            for (int i = 0; i < 6; ++i) std::fprintf(stderr, " %llu", h[i]);
            std::fprintf(stderr, " | tile_load %llu atomic %llu max_tiles/warp %llu tiles %llu warp_B %llu",
                         h[6], h[7], h[8], h[9], h[10]);
            std::fprintf(stderr, "\n");
        }
        std::memset(h, 0, sizeof h);
        h[8] = ~0ull;
        EAB_CUDA(cudaMemcpy(prof, h, sizeof h, cudaMemcpyHostToDevice));
        ++nprof;
        fa.prof = prof;
    }
    void* args[] = {&fa};
    EAB_CUDA(cudaLaunchCooperativeKernel((const void*)finish_kernel, dim3(blocks), dim3(256), args,
                                         0, ctx->stream));
    check_launch("finish_kernel");
    count_launch(ctx);
}

// The `better` merge of several slabs' rows (search.cpp:130-139): rank of
// each valid row among all valid rows by (score desc, index asc); rows with
// rank < k land at their rank, the rest of the output is NaN rows.  With
// top_score/top_index/n_top set it also writes the merged top k in the
// layout a search's select leaves (the seed kernel's input), so a sharded
// search refines from the merge without a host round trip.
__global__ void __launch_bounds__(256) merge_rows_kernel(const double* __restrict__ in, int n,
                                                         int k, double* __restrict__ out,
                                                         double* __restrict__ top_score,
                                                         unsigned long long* __restrict__ top_index,
                                                         int* __restrict__ n_top) {
    extern __shared__ long long mk[];  // order key | index per input row
    long long* key = mk;
    unsigned long long* idx = reinterpret_cast<unsigned long long*>(mk + n);
    __shared__ int valid;
    if (threadIdx.x == 0) valid = 0;
    __syncthreads();
    int mine = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double sc = in[5 * (size_t)i];
        key[i] = sc != sc ? LLONG_MIN : order_key(sc);
        idx[i] = (unsigned long long)in[5 * (size_t)i + 1];
        mine += sc == sc;
    }
    if (mine) atomicAdd(&valid, mine);
    for (int r = threadIdx.x; r < k; r += blockDim.x) {
        double* o = out + 5 * (size_t)r;
        o[0] = __longlong_as_double(0x7ff8000000000000LL);
        o[1] = o[2] = o[3] = o[4] = 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (key[i] == LLONG_MIN) continue;
        int rank = 0;
        for (int j = 0; j < n; ++j)
            rank += key[j] > key[i] || (key[j] == key[i] && key[j] != LLONG_MIN &&
                                        (idx[j] < idx[i] || (idx[j] == idx[i] && j < i)));
        if (rank < k) {
            for (int c = 0; c < 5; ++c) out[5 * (size_t)rank + c] = in[5 * (size_t)i + c];
            if (top_score) {
                top_score[rank] = in[5 * (size_t)i];
                top_index[rank] = idx[i];
            }
        }
    }
    if (n_top && threadIdx.x == 0) *n_top = valid < k ? valid : k;
}

void launch_topk_rows(ea_ctx* ctx, const double* score, const unsigned long long* index,
                      const SearchCtrl* ctrl, unsigned long long cap, int k, const RowGrid& g,
                      double* rows, int* overflow) {
    topk_rows_kernel<<<1, 64, 0, ctx->stream>>>(score, index, ctrl, cap, k, g, rows, overflow);
    check_launch("topk_rows_kernel");
    count_launch(ctx);
}

// Per-model `better` merge of a multi-model all-gather (one CTA per model):
// rank r's rows of model m are in[(r * n_models + m) * k + j], j < k.
// Writes model m's k merged rows to out[m * k ..] and its seeds to
// top_score/top_index[m * k ..], n_top[m].
__global__ void __launch_bounds__(256) merge_rows_multi_kernel(
    const double* __restrict__ in, int world, int n_models, int k, double* __restrict__ out,
    double* __restrict__ top_score, unsigned long long* __restrict__ top_index,
    int* __restrict__ n_top) {
    extern __shared__ long long mk[];
    const int m = blockIdx.x, n = world * k;
    long long* key = mk;
    unsigned long long* idx = reinterpret_cast<unsigned long long*>(mk + n);
    __shared__ int valid;
    if (threadIdx.x == 0) valid = 0;
    __syncthreads();
    auto row = [&](int i) { return in + 5 * ((size_t)((i / k) * n_models + m) * k + i % k); };
    int mine = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double sc = row(i)[0];
        key[i] = sc != sc ? LLONG_MIN : order_key(sc);
        idx[i] = (unsigned long long)row(i)[1];
        mine += sc == sc;
    }
    if (mine) atomicAdd(&valid, mine);
    double* o = out + 5 * (size_t)m * k;
    for (int r = threadIdx.x; r < k; r += blockDim.x) {
        o[5 * r] = __longlong_as_double(0x7ff8000000000000LL);
        o[5 * r + 1] = o[5 * r + 2] = o[5 * r + 3] = o[5 * r + 4] = 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (key[i] == LLONG_MIN) continue;
        int rank = 0;
        for (int j = 0; j < n; ++j)
            rank += key[j] > key[i] || (key[j] == key[i] && key[j] != LLONG_MIN &&
                                        (idx[j] < idx[i] || (idx[j] == idx[i] && j < i)));
        if (rank < k) {
            for (int c = 0; c < 5; ++c) o[5 * rank + c] = row(i)[c];
            top_score[(size_t)m * k + rank] = row(i)[0];
            top_index[(size_t)m * k + rank] = idx[i];
        }
    }
    if (threadIdx.x == 0) n_top[m] = valid < k ? valid : k;
}

void launch_merge_rows_multi(ea_ctx* ctx, const double* in, int world, int n_models, int k,
                             double* out, double* top_score, unsigned long long* top_index,
                             int* n_top) {
    const size_t smem = (size_t)world * k * 16;
    if (smem + 1024 > 48 * 1024)
        raise_smem_limit(ctx, (const void*)merge_rows_multi_kernel, ctx->smem_optin);
    merge_rows_multi_kernel<<<n_models, 256, smem, ctx->stream>>>(in, world, n_models, k, out,
                                                                 top_score, top_index, n_top);
    check_launch("merge_rows_multi_kernel");
    count_launch(ctx);
}

int merge_rows_max(ea_ctx* ctx) { return (int)(ctx->smem_optin / 16); }

void launch_merge_rows(ea_ctx* ctx, const double* in, int n, int k, double* out,
                       double* top_score, unsigned long long* top_index, int* n_top) {
    const size_t smem = (size_t)n * 16;
    // dynamic shared memory beyond 48 KB (minus the kernel's static bytes) is
    // opt-in: raise the limit once, to the context's budget
    if (smem + 1024 > 48 * 1024)
        raise_smem_limit(ctx, (const void*)merge_rows_kernel, ctx->smem_optin);
    merge_rows_kernel<<<1, 256, smem, ctx->stream>>>(in, n, k, out, top_score, top_index, n_top);
    check_launch("merge_rows_kernel");
    count_launch(ctx);
}

// ---- dense exact map (score_map) -------------------------------------------------
__global__ void __launch_bounds__(256) exact_map_kernel(const ExactArgs a,
                                                        unsigned long long total,
                                                        double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const unsigned long long plane = a.nx * a.ny;
    for (unsigned long long t = warp; t < total; t += nwarps) {
        const unsigned long long it = t / plane;
        const unsigned long long rem = t % plane;
        const double ux = lattice(a.x0, rem % a.nx, a.dx);
        const double uy = lattice(a.y0, rem / a.nx, a.dy);
        const double s = warp_pose_score(a, (size_t)it * a.n, ux, uy, lane, nullptr);
        if (lane == 0) out[t] = s;
    }
}

void launch_exact_map(ea_ctx* ctx, const ExactArgs& a, unsigned long long total, double* out) {
    unsigned long long blocks = (total * 32 + 255) / 256;
    const unsigned long long maxb = (unsigned long long)ctx->sm_count * 16;
    if (blocks > maxb) blocks = maxb;
    if (blocks == 0) blocks = 1;
    exact_map_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, total, out);
    check_launch("exact_map_kernel");
    count_launch(ctx);
}

// ---- point_vote (similarity.cpp:58-64) ---------------------------------------------
__global__ void point_vote_kernel(const double* gx, const double* gy, const double* mag, int W,
                                  int H, int cx, int cy, int R, double dx, double dy, double eps,
                                  int absolute, double* out) {
    *out = vote_exact(gx, gy, mag, W, H, cx, cy, R, dx, dy, eps, absolute != 0);
}

void launch_point_vote(ea_ctx* ctx, const ea_field* f, int cx, int cy, int R, double dx,
                       double dy, double eps, bool absolute, double* out) {
    point_vote_kernel<<<1, 1, 0, ctx->stream>>>(f->gx(), f->gy(), f->mag(), f->width, f->height,
                                                cx, cy, R, dx, dy, eps, absolute ? 1 : 0, out);
    check_launch("point_vote_kernel");
    count_launch(ctx);
}

// ---- refinement --------------------------------------------------------------------
__global__ void __launch_bounds__(256) refine_score_kernel(const ExactArgs a,
                                                           const double* __restrict__ poses,
                                                           const int* __restrict__ slot,
                                                           int count,
                                                           double* __restrict__ score,
                                                           int* __restrict__ n_inb) {
    const int lane = threadIdx.x & 31;
    const int warp = (int)(((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)(((unsigned long long)gridDim.x * blockDim.x) >> 5);
    for (int e = warp; e < count; e += nwarps) {
        int inb = 0;
        const double s = warp_pose_score(a, (size_t)slot[e] * a.n, poses[2 * e], poses[2 * e + 1],
                                         lane, &inb);
        if (lane == 0) {
            score[e] = s;
            if (n_inb) n_inb[e] = inb;
        }
    }
}

void launch_refine_score(ea_ctx* ctx, const ExactArgs& a, const double* poses, const int* slot,
                         int count, double* score, int* n_inb) {
    if (count <= 0) return;
    unsigned long long blocks = ((unsigned long long)count * 32 + 255) / 256;
    const unsigned long long maxb = (unsigned long long)ctx->sm_count * 16;
    if (blocks > maxb) blocks = maxb;
    refine_score_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, poses, slot, count, score,
                                                                  n_inb);
    check_launch("refine_score_kernel");
    count_launch(ctx);
}

// std::stable_sort(score desc) + exact-duplicate removal + keep topk
// (search.cpp:323-346).  Stable rank = #{j : s_j > s_e or (s_j == s_e and j < e)}.
__global__ void __launch_bounds__(1024) beam_select_kernel(const double* __restrict__ poses3,
                                                           const double* __restrict__ score,
                                                           const int* __restrict__ parent,
                                                           int count, int topk,
                                                           int* __restrict__ order,
                                                           double* __restrict__ beam_out,
                                                           int* __restrict__ beam_parent,
                                                           int* __restrict__ beam_count) {
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        const double s = score[e];
        int r = 0;
        for (int j = 0; j < count; ++j) {
            const double sj = score[j];
            r += (sj > s) || (sj == s && j < e);
        }
        order[r] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int kept = 0;
        for (int r = 0; r < count && kept < topk; ++r) {
            const int e = order[r];
            const double ux = poses3[3 * e], uy = poses3[3 * e + 1], th = poses3[3 * e + 2];
            bool dup = false;
            for (int q = 0; q < kept; ++q) {
                if (beam_out[4 * q] == ux && beam_out[4 * q + 1] == uy && beam_out[4 * q + 2] == th) {
                    dup = true;
                    break;
                }
            }
            if (!dup) {
                beam_out[4 * kept] = ux;
                beam_out[4 * kept + 1] = uy;
                beam_out[4 * kept + 2] = th;
                beam_out[4 * kept + 3] = score[e];
                beam_parent[kept] = parent[e];
                ++kept;
            }
        }
        *beam_count = kept;
    }
}

void launch_beam_select(ea_ctx* ctx, const double* poses3, const double* score,
                        const int* parent, int count, int topk, double* beam_out,
                        int* beam_parent, int* beam_count) {
    int* order = reinterpret_cast<int*>(ctx->work.ensure(sizeof(int) * (size_t)(count + 1)));
    beam_select_kernel<<<1, 1024, 0, ctx->stream>>>(poses3, score, parent, count, topk, order,
                                                    beam_out, beam_parent, beam_count);
    check_launch("beam_select_kernel");
    count_launch(ctx);
}

}  // namespace eab
