// refine_kernels.cu -- per-level beam refinement of search_levels
// (search.cpp:254-357) with the whole beam on the device.
//
// Every theta the refinement can reach is  theta_seed + kt1*st1 + kt2*st2 ...
// (search.cpp:295,305), a function of the seed and the kt path only, so the
// host evaluates glibc cos/sin for all paths of the k seeds once (k * sum
// side^d values) and the levels run without host round trips:
//
//   refine_entry_kernel   one CTA per pose: the pose and the model's exact
//                         rotation (similarity.cpp:79-86), exact votes of all
//                         points into a shared-memory row, ordered fp64 sum
//                         (model-point order, then /n) + "an earlier entry
//                         has this pose".
//   refine_rank_kernel    one warp per pose: rank among first occurrences in
//                         the stable-sort order -> new beam slot, trace,
//                         final outcome.
#include <algorithm>
#include <climits>

#include "kernels.cuh"
#include "refine.cuh"

namespace eab {

// Lattice pose e of a level (search.cpp:295-312): parent = e / side^3, kt
// path step (e / side^2) % side, (ky, kx) from e % side^2 -- the same
// arithmetic the host loop uses (2 * parent + k * step, no contraction).
__device__ __forceinline__ void refine_pose(const RefineArgs& a, int e, double& ux, double& uy,
                                            double& th, double& c, double& s) {
    const int side = a.side, ss = side * side;
    const int pk = e / ss, j = e % ss;
    const BeamDev& parent = a.beam[pk / side];
    const int path = parent.path * side + (pk % side);
    th = a.table[3 * path];
    c = a.table[3 * path + 1];
    s = a.table[3 * path + 2];
    const int ky = j / side - a.R, kx = j % side - a.R;
    ux = __dadd_rn(__dmul_rn(parent.ux, 2.0), __dmul_rn((double)kx, a.step_x));
    uy = __dadd_rn(__dmul_rn(parent.uy, 2.0), __dmul_rn((double)ky, a.step_y));
}

// Score of each lattice pose (score_rotated, similarity.cpp:102-118): one
// CTA per pose.  Threads rotate the model points for the pose's theta
// (rotate_model, similarity.cpp:79-86: glibc cos/sin from the path table)
// and compute their exact votes into a vote row (shared memory, or global
// for very large models); then thread 0 adds them in model-point order --
// the reference's sequential fp64 sum, bit for bit -- and divides by n,
// while warp 1 checks whether an earlier entry in generation order has the
// identical pose: identical poses score identically, so after the stable
// sort the first occurrence is the one kept (search.cpp:330-345).  (The
// rotation is recomputed by each of a (parent, kt) pair's side^2 poses: a
// separate rotation launch cost more than the arithmetic.)
__global__ void __launch_bounds__(kRefineThreads) refine_entry_kernel(const RefineArgs a) {
    extern __shared__ double sv[];
    __shared__ int dup_s;
    const int side = a.side, ss = side * side;
    const int E = *a.beam_count * side * ss;
    const int e = blockIdx.x;
    if (e >= E) return;  // whole CTA
    double px, py, pt, c, s;
    refine_pose(a, e, px, py, pt, c, s);
    const int n = a.n;
    double* vb = a.votes_in_smem ? sv : a.votes + (size_t)e * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double x = a.pts[i], y = a.pts[n + i];
        const double dx = a.pts[2 * n + i], dy = a.pts[3 * n + i];
        const double rx = __dsub_rn(__dmul_rn(c, dx), __dmul_rn(s, dy));
        const double ry = __dadd_rn(__dmul_rn(s, dx), __dmul_rn(c, dy));
        const double norm = __dsqrt_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)));
        int inb;
        vb[i] = point_term_exact(__dsub_rn(__dmul_rn(c, x), __dmul_rn(s, y)),
                                 __dadd_rn(__dmul_rn(s, x), __dmul_rn(c, y)),
                                 __ddiv_rn(rx, norm), __ddiv_rn(ry, norm), px, py, a.gx, a.gy,
                                 a.mag, a.W, a.H, a.vote_R, a.eps, a.ignore != 0, &inb);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 1) {
        int dup = 0;
        for (int q = lane; q < e; q += 32) {
            double qx, qy, qt, qc, qs;
            refine_pose(a, q, qx, qy, qt, qc, qs);
            dup |= (qx == px && qy == py && qt == pt) ? 1 : 0;
        }
        dup = __any_sync(0xffffffffu, dup);
        if (lane == 0) dup_s = dup;
    }
    double score = 0.0;
    if (threadIdx.x == 0) {
        double sum = 0.0;
        int i = 0;
        for (; i + 4 <= n; i += 4) {  // independent loads, one dependent add chain
            const double v0 = vb[i], v1 = vb[i + 1], v2 = vb[i + 2], v3 = vb[i + 3];
            sum = __dadd_rn(sum, v0);
            sum = __dadd_rn(sum, v1);
            sum = __dadd_rn(sum, v2);
            sum = __dadd_rn(sum, v3);
        }
        for (; i < n; ++i) sum = __dadd_rn(sum, vb[i]);
        score = __ddiv_rn(sum, (double)n);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int dup = dup_s;
        double* out = a.entries + 4 * (size_t)e;
        out[0] = score;
        out[1] = px;
        out[2] = py;
        out[3] = pt;
        a.dup[e] = dup;
        a.keys[e] = dup ? LLONG_MIN : order_key(score);
    }
}

__device__ __forceinline__ unsigned long long eq_key(double v) {
    return (unsigned long long)__double_as_longlong(v == 0.0 ? 0.0 : v);
}

// std::stable_sort by score (search.cpp:326-329) + exact-duplicate removal +
// keep topk (search.cpp:330-345), as a one-warp selection: each round takes
// the next entry in (score desc, generation order asc) -- the stable order --
// and keeps it unless a kept entry has the same pose.
// New beam (search.cpp:323-346): among first occurrences, the rank of entry e
// in (score desc, generation index asc) -- the stable-sort order -- decides
// its slot; one warp per entry, no serial walk.
__global__ void __launch_bounds__(256) refine_rank_kernel(const RefineArgs a) {
    const int side = a.side, ss = side * side;
    const int E = *a.beam_count * side * ss;
    const int lane = threadIdx.x & 31;
    const int e = (int)(((unsigned)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (e >= E) return;
    const long long ke = a.keys[e];
    const bool mine = ke != LLONG_MIN;  // first occurrence of its pose
    int rank = 0, distinct = 0;
#pragma unroll 4
    for (int q = lane; q < E; q += 32) {
        const long long kq = a.keys[q];
        distinct += kq != LLONG_MIN;
        rank += (kq > ke) || (kq == ke && q < e);  // duplicates never outrank
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        rank += __shfl_xor_sync(0xffffffffu, rank, o);
        distinct += __shfl_xor_sync(0xffffffffu, distinct, o);
    }
    if (!mine || rank >= a.topk || lane != 0) return;
    const double* in = a.entries + 4 * (size_t)e;
    const int pk = e / ss;
    const BeamDev& parent = a.beam[pk / side];
    BeamDev b;
    b.score = in[0];
    b.ux = in[1];
    b.uy = in[2];
    b.theta = in[3];
    b.top_index = parent.top_index;
    b.path = parent.path * side + (pk % side);
    b._pad = 0;
    a.beam_out[rank] = b;
    if (rank == 0) {
        *a.beam_count_out = distinct < a.topk ? distinct : a.topk;
        ea_outcome* o = a.outcome;
        if (a.trace_slot < EA_MAX_LEVELS) {
            o->trace[a.trace_slot].level = a.level;
            o->trace[a.trace_slot].pose = ea_pose{b.ux, b.uy, b.theta};
            o->trace[a.trace_slot].score = b.score;
            o->n_trace = a.trace_slot + 1;
        }
        if (a.level == 0) {
            o->pose = ea_pose{b.ux, b.uy, b.theta};
            o->score = b.score;
            o->grid_index = b.top_index;
            o->found = b.score >= a.min_score ? 1 : 0;
        }
    }
}

// Beam seeds straight from the top-level top-k on the device (search.cpp:
// 276-284): pose_at of each index (pose.h:84-91), theta path = theta index.
__global__ void seed_beam_kernel(const double* __restrict__ top_score,
                                 const unsigned long long* __restrict__ top_index,
                                 const int* __restrict__ n_top, SeedArgs s, BeamDev* beam,
                                 int* beam_count, ea_outcome* out) {
    const int n = *n_top;
    const unsigned long long plane = s.nx * s.ny;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long idx = top_index[i];
        const unsigned long long it = idx / plane, rem = idx % plane;
        BeamDev b;
        b.ux = __dadd_rn(s.x0, __dmul_rn((double)(rem % s.nx), s.dx));
        b.uy = __dadd_rn(s.y0, __dmul_rn((double)(rem / s.nx), s.dy));
        b.theta = __dadd_rn(s.t0, __dmul_rn((double)it, s.dt));
        b.score = top_score[i];
        b.top_index = idx;
        b.path = (int)it;
        b._pad = 0;
        beam[i] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *beam_count = n;
        const BeamDev b0 = beam[0];
        out->trace[0].level = s.top_level;
        out->trace[0].pose = ea_pose{b0.ux, b0.uy, b0.theta};
        out->trace[0].score = b0.score;
        out->n_trace = 1;
        if (s.top_level == 0) {  // no refinement: the seed is the answer
            out->pose = ea_pose{b0.ux, b0.uy, b0.theta};
            out->score = b0.score;
            out->grid_index = b0.top_index;
            out->found = b0.score >= s.min_score ? 1 : 0;
        }
    }
}

void launch_seed_beam(ea_ctx* ctx, const double* top_score, const unsigned long long* top_index,
                      const int* n_top, const SeedArgs& s, BeamDev* beam, int* beam_count,
                      ea_outcome* out) {
    seed_beam_kernel<<<1, 64, 0, ctx->stream>>>(top_score, top_index, n_top, s, beam,
                                                beam_count, out);
    check_launch("seed_beam_kernel");
    count_launch(ctx);
}

void launch_refine_level(ea_ctx* ctx, const RefineArgs& a_in) {
    RefineArgs a = a_in;
    const int e_max = a.max_parents * a.side * a.side * a.side;
    const size_t smem = sizeof(double) * (size_t)a.n;
    a.votes_in_smem = smem <= kRefineSmemMax ? 1 : 0;
    raise_smem_limit(ctx, (const void*)refine_entry_kernel, kRefineSmemMax);
    refine_entry_kernel<<<e_max, kRefineThreads, a.votes_in_smem ? smem : 0, ctx->stream>>>(a);
    check_launch("refine_entry_kernel");
    count_launch(ctx);
    refine_rank_kernel<<<(e_max * 32 + 255) / 256, 256, 0, ctx->stream>>>(a);
    check_launch("refine_rank_kernel");
    count_launch(ctx);
}

}  // namespace eab
