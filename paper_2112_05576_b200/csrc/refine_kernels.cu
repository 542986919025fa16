// refine_kernels.cu -- per-level beam refinement of search_levels
// (search.cpp:254-357) with the whole beam on the device.
//
// Every theta the refinement can reach is  theta_seed + kt1*st1 + kt2*st2 ...
// (search.cpp:295,305), a function of the seed and the kt path only, so the
// host evaluates glibc cos/sin for all paths of the k seeds once (k * sum
// side^d values) and the levels run without host round trips:
//
//   refine_votes_kernel   one CTA per (parent, kt, point chunk): rotates the
//                         chunk exactly (similarity.cpp:79-86), then every
//                         thread computes exact fp64 votes of (pose, point)
//                         pairs for the side^2 lattice poses.  votes[i][e].
//   refine_sum_kernel     one warp per pose: ordered fp64 sum (model-point
//                         order, then /n) + "an earlier entry has this pose".
//   refine_rank_kernel    one warp per pose: rank among first occurrences in
//                         the stable-sort order -> new beam slot, trace,
//                         final outcome.
#include <climits>

#include "kernels.cuh"
#include "refine.cuh"

namespace eab {

__global__ void __launch_bounds__(256) refine_votes_kernel(const RefineArgs a) {
    extern __shared__ double rot[];  // px | py | dx | dy of this chunk
    const int side = a.side, R = a.R;
    const int pk = blockIdx.x;         // parent * side + (kt + R)
    const int p = pk / side;
    if (p >= *a.beam_count) return;
    const int i0 = blockIdx.y * a.chunk;
    const int cn = min(a.chunk, a.n - i0);
    if (cn <= 0) return;
    const BeamDev parent = a.beam[p];
    const int path = parent.path * side + (pk % side);
    const double c = a.table[3 * path + 1], s = a.table[3 * path + 2];
    for (int t = threadIdx.x; t < cn; t += blockDim.x) {
        const int i = i0 + t;
        const double x = a.pts[i], y = a.pts[a.n + i];
        const double dx = a.pts[2 * a.n + i], dy = a.pts[3 * a.n + i];
        const double rx = __dsub_rn(__dmul_rn(c, dx), __dmul_rn(s, dy));
        const double ry = __dadd_rn(__dmul_rn(s, dx), __dmul_rn(c, dy));
        const double norm = __dsqrt_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)));
        rot[t] = __dsub_rn(__dmul_rn(c, x), __dmul_rn(s, y));
        rot[a.chunk + t] = __dadd_rn(__dmul_rn(s, x), __dmul_rn(c, y));
        rot[2 * a.chunk + t] = __ddiv_rn(rx, norm);
        rot[3 * a.chunk + t] = __ddiv_rn(ry, norm);
    }
    __syncthreads();
    const double cx = __dmul_rn(parent.ux, 2.0), cy = __dmul_rn(parent.uy, 2.0);
    const int ss = side * side;
    for (int t = threadIdx.x; t < ss * cn; t += blockDim.x) {
        const int j = t / cn, ii = t % cn;
        const int ky = j / side - R, kx = j % side - R;
        const double ux = __dadd_rn(cx, __dmul_rn((double)kx, a.step_x));
        const double uy = __dadd_rn(cy, __dmul_rn((double)ky, a.step_y));
        int inb;
        const double v = point_term_exact(rot[ii], rot[a.chunk + ii], rot[2 * a.chunk + ii],
                                          rot[3 * a.chunk + ii], ux, uy, a.gx, a.gy, a.mag, a.W,
                                          a.H, a.vote_R, a.eps, a.ignore != 0, &inb);
        a.votes[((size_t)pk * ss + j) * a.n + i0 + ii] = v;  // pose-major
    }
}

__device__ __forceinline__ void entry_pose(const RefineArgs& a, int e, double* ux, double* uy,
                                           double* th) {
    const int side = a.side, ss = side * side;
    const int pk = e / ss, j = e % ss;
    const BeamDev& parent = a.beam[pk / side];
    const int ky = j / side - a.R, kx = j % side - a.R;
    *ux = __dadd_rn(__dmul_rn(parent.ux, 2.0), __dmul_rn((double)kx, a.step_x));
    *uy = __dadd_rn(__dmul_rn(parent.uy, 2.0), __dmul_rn((double)ky, a.step_y));
    *th = a.table[3 * (parent.path * side + (pk % side))];
}

// Ordered fp64 sum of each lattice pose's votes (model-point order, then /n,
// similarity.cpp:109-118): one warp per pose; lanes load 32 consecutive votes,
// every lane walks them in order through shuffles (the chain is the
// reference's sequential sum).  Also emits the pose (search.cpp:308-312).
__global__ void __launch_bounds__(256) refine_sum_kernel(const RefineArgs a) {
    const int side = a.side, R = a.R, ss = side * side;
    const int E = *a.beam_count * side * ss;
    const int lane = threadIdx.x & 31;
    const int e = (int)(((unsigned)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (e >= E) return;
    const double* row = a.votes + (size_t)e * a.n;
    double sum = 0.0;
    for (int q = 0; q < a.n; q += 32) {
        const double v = q + lane < a.n ? __ldg(row + q + lane) : 0.0;
        const int lim = a.n - q < 32 ? a.n - q : 32;
        double t[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) t[l] = __shfl_sync(0xffffffffu, v, l);
#pragma unroll
        for (int l = 0; l < 32; ++l)
            if (l < lim) sum = __dadd_rn(sum, t[l]);
    }
    // The pose of entry e (search.cpp:305-312) and whether an earlier entry in
    // generation order has the identical pose: identical poses score
    // identically, so after the stable sort the first occurrence is the one
    // kept (search.cpp:330-345).
    double px, py, pt;
    entry_pose(a, e, &px, &py, &pt);
    int dup = 0;
    for (int q0 = 0; q0 < e; q0 += 32) {  // warp-uniform trip count
        const int q = q0 + lane;
        if (q < e) {
            double qx, qy, qt;
            entry_pose(a, q, &qx, &qy, &qt);
            dup |= (qx == px && qy == py && qt == pt) ? 1 : 0;
        }
        if (__any_sync(0xffffffffu, dup)) break;
    }
    dup = __any_sync(0xffffffffu, dup);
    if (lane == 0) {
        double* out = a.entries + 4 * (size_t)e;
        out[0] = __ddiv_rn(sum, (double)a.n);
        out[1] = px;
        out[2] = py;
        out[3] = pt;
        a.dup[e] = dup;
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
    const long long ke = order_key(a.entries[4 * (size_t)e]);
    const bool mine = a.dup[e] == 0;
    int rank = 0, distinct = 0;
    for (int q = lane; q < E; q += 32) {
        if (a.dup[q]) continue;
        ++distinct;
        const long long kq = order_key(a.entries[4 * (size_t)q]);
        rank += (kq > ke) || (kq == ke && q < e);
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

void launch_refine_level(ea_ctx* ctx, const RefineArgs& a) {
    const int grid_x = a.max_parents * a.side;
    const int grid_y = (a.n + a.chunk - 1) / a.chunk;
    refine_votes_kernel<<<dim3(grid_x, grid_y), 256, 4 * sizeof(double) * a.chunk,
                          ctx->stream>>>(a);
    check_launch("refine_votes_kernel");
    const int e_max = a.max_parents * a.side * a.side * a.side;
    refine_sum_kernel<<<(e_max * 32 + 255) / 256, 256, 0, ctx->stream>>>(a);
    check_launch("refine_sum_kernel");
    refine_rank_kernel<<<(e_max * 32 + 255) / 256, 256, 0, ctx->stream>>>(a);
    check_launch("refine_rank_kernel");
    count_launch(ctx, 3);
}

}  // namespace eab
