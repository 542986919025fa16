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
//   refine_select_kernel  one CTA: ordered sums (model-point order, then /n),
//                         std::stable_sort rank by score, exact-duplicate
//                         removal, keep topk, level trace / final outcome.
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
    if (lane == 0) {
        const int pk = e / ss, j = e % ss;
        const BeamDev parent = a.beam[pk / side];
        const int path = parent.path * side + (pk % side);
        const int ky = j / side - R, kx = j % side - R;
        double* out = a.entries + 4 * (size_t)e;
        out[0] = __ddiv_rn(sum, (double)a.n);
        out[1] = __dadd_rn(__dmul_rn(parent.ux, 2.0), __dmul_rn((double)kx, a.step_x));
        out[2] = __dadd_rn(__dmul_rn(parent.uy, 2.0), __dmul_rn((double)ky, a.step_y));
        out[3] = a.table[3 * path];
    }
}

__device__ __forceinline__ unsigned long long eq_key(double v) {
    return (unsigned long long)__double_as_longlong(v == 0.0 ? 0.0 : v);
}

__global__ void __launch_bounds__(1024) refine_select_kernel(const RefineArgs a) {
    extern __shared__ long long smk[];
    const int side = a.side, ss = side * side;
    const int P = *a.beam_count;
    const int E = P * side * ss;
    const int Emax = a.max_parents * side * ss;
    long long* key = smk;
    int* order = reinterpret_cast<int*>(key + Emax);
    for (int e = threadIdx.x; e < E; e += blockDim.x) key[e] = order_key(a.entries[4 * (size_t)e]);
    __syncthreads();
    // stable rank by score descending (std::stable_sort, search.cpp:326-329)
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const long long k = key[e];
        int r = 0;
        for (int j = 0; j < E; ++j) {
            const long long kj = key[j];
            r += (kj > k) | ((kj == k) & (j < e));
        }
        order[r] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // walk in rank order, drop exact duplicates of kept poses, keep topk
        // (search.cpp:330-345)
        unsigned long long kx[64], ky[64], kt[64];
        const int cap = a.topk < 64 ? a.topk : 64;
        int kept = 0;
        for (int r = 0; r < E && kept < cap; ++r) {
            const int e = order[r];
            const double* in = a.entries + 4 * (size_t)e;
            const unsigned long long x = eq_key(in[1]), y = eq_key(in[2]), t = eq_key(in[3]);
            bool dup = false;
            for (int q = 0; q < kept && !dup; ++q) dup = kx[q] == x && ky[q] == y && kt[q] == t;
            if (dup) continue;
            kx[kept] = x;
            ky[kept] = y;
            kt[kept] = t;
            const int pk = e / ss;
            const BeamDev parent = a.beam[pk / side];
            BeamDev b;
            b.score = in[0];
            b.ux = in[1];
            b.uy = in[2];
            b.theta = in[3];
            b.top_index = parent.top_index;
            b.path = parent.path * side + (pk % side);
            b._pad = 0;
            a.beam_out[kept++] = b;
        }
        *a.beam_count_out = kept;
        ea_outcome* o = a.outcome;
        const BeamDev b0 = a.beam_out[0];
        if (a.trace_slot < EA_MAX_LEVELS) {
            o->trace[a.trace_slot].level = a.level;
            o->trace[a.trace_slot].pose = ea_pose{b0.ux, b0.uy, b0.theta};
            o->trace[a.trace_slot].score = b0.score;
            o->n_trace = a.trace_slot + 1;
        }
        if (a.level == 0) {
            o->pose = ea_pose{b0.ux, b0.uy, b0.theta};
            o->score = b0.score;
            o->grid_index = b0.top_index;
            o->found = b0.score >= a.min_score ? 1 : 0;
        }
    }
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
    const size_t Emax = (size_t)a.max_parents * a.side * a.side * a.side;
    const size_t smem = Emax * (sizeof(long long) + sizeof(int));
    EAB_CUDA(cudaFuncSetAttribute(refine_select_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    refine_select_kernel<<<1, 1024, smem, ctx->stream>>>(a);
    check_launch("refine_select_kernel");
    count_launch(ctx, 3);
}

}  // namespace eab
