// common.cuh -- shared host/device infrastructure of libedgealign_b200.
#pragma once

#include <atomic>
#include <cstdlib>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "failure.h"

namespace eab {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fail(EA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define EAB_CUDA(x) ::eab::cuda_check((x), #x)

// ---- growable device buffer ------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void* ensure(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            size_t want = bytes < 256 ? 256 : bytes;
            EAB_CUDA(cudaMalloc(&p, want));
            cap = want;
        }
        return p;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// ---- pinned host staging ---------------------------------------------------
struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() { release(); }
    void* ensure(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            size_t want = bytes < 4096 ? 4096 : bytes;
            EAB_CUDA(cudaHostAlloc(&p, want, cudaHostAllocDefault));
            cap = want;
        }
        return p;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace eab

// ---- opaque handles of the C-ABI ------------------------------------------
// Content version of gradient fields: every write (Sobel, upload) takes a
// new number, so a cache keyed on (field, version) can never go stale.
inline uint64_t next_field_version() {
    static std::atomic<uint64_t> v{0};
    return ++v;
}

struct ea_field {
    int width = 0, height = 0;
    uint64_t version = 0;
    double ring_max = INFINITY;  // largest |g| on the outer pixel ring
    eab::DevBuf g;  // gx | gy | mag, each width*height doubles
    double* gx() const { return g.as<double>(); }
    double* gy() const { return g.as<double>() + (size_t)width * height; }
    double* mag() const { return g.as<double>() + 2 * (size_t)width * height; }
};

struct ea_model {
    int n = 0;
    double centroid_x = 0, centroid_y = 0;
    int source_level = 0;
    std::vector<ea_edge_point> host;  // AoS copy (template side stays on host too)
    eab::DevBuf pts;                  // device SoA: x_rel | y_rel | dx | dy
    // Rotation tables, ambiguity list and lattice schedule of the theta slab
    // searched last: the model is immutable, so they depend only on the grid's
    // theta axis and are reused by every later search of that slab (one
    // detect per image).  Written on the owning context's stream.
    std::vector<double> tab_key;
    eab::DevBuf rot, scr, amb, sched;
    int n_flagged = 0;  // flagged thetas of the cached slab
    int sched_mode = 0;  // entry kinds of the cached schedule (launch_schedule)
};

struct ea_levels {
    std::vector<ea_model*> models;  // owned
    std::vector<ea_field*> fields;  // owned; may be empty until set_image
    eab::DevBuf image;              // working pyramid levels >= 1
    eab::DevBuf raw[2];             // level-0 images (double-buffered in batch mode)
    std::vector<ea_field*> fields2; // batch mode: second and third working sets (owned)
    eab::DevBuf image2;
    std::vector<ea_field*> fields3;
    eab::DevBuf image3;
    // theta-sharded detect on a rank other than the root: the top level's
    // field as broadcast by the root (the only level such a rank searches)
    ea_field* shard_top = nullptr;
};

struct ea_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 0;
    size_t smem_optin = 0;
    uint64_t launches = 0;
    ea_search_stats stats{};
    bool timing = false;
    bool trace_on = std::getenv("EAB_TRACE") != nullptr;
    // Screening plane cache: the float2 plane in `plane` was built from this
    // (field, version, eps, geometry); a search on the same image skips the
    // plane kernel.  hist_clean: the histogram / control block are in their
    // between-searches state (zero hist and work counter), which the fused
    // finish restores; a screen without a finish (screen_map) clears it.
    std::vector<double> plane_key;
    bool hist_clean = false;
    std::vector<std::pair<const char*, cudaEvent_t>> trace;
    // one cooperative finish launch after the screen (EAB_NO_FUSED_FINISH=1:
    // the separate compact/rescore/select/rows launches, for A/B measurements)
    bool fused_finish = std::getenv("EAB_NO_FUSED_FINISH") == nullptr;
    // screen + finish in one cooperative launch where eligible (top-list
    // mode); off by default: measured on B200 it saves the finish launch on a
    // full search (-13 us of 650) but costs a theta slab +6 us (the
    // cooperative launch waits for the whole GPU) and batch detect +3 %
    // (a cooperative grid cannot overlap the refinement stream);
    // EAB_FUSED_SCREEN=1 enables it (tested)
    bool fused_screen = std::getenv("EAB_FUSED_SCREEN") != nullptr &&
                        std::getenv("EAB_NO_FUSED_FINISH") == nullptr;
    // top-list mode of the smem lattice kernel (see screen(), api.cu);
    // EAB_NO_TOPLIST=1: the histogram threshold (A/B, tested both ways)
    bool toplist = std::getenv("EAB_NO_TOPLIST") == nullptr;
    cudaEvent_t ev[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    // scratch
    eab::DevBuf cs, rot_exact, rot_screen, plane, map, item_max, tail, hist, ctrl, cand, cand_score, topk,
        refine_poses, refine_scores, beam, accum64, work, mscratch, cta_top, ztiles, chunk_rows;
    std::vector<double> ztiles_key;  // what ztiles holds (see screen(), api.cu)
    eab::HostBuf h_stage, h_out;
    // glibc cos/sin tables of theta grids, cached per (t0, dt, nt)
    std::map<std::vector<double>, std::vector<double>> cs_cache;
    std::vector<double> cs_dev_key;  // what ctx->cs currently holds on the device
    // glibc (theta, cos, sin) of every refinement path of every top-level theta
    std::vector<double> ttab_key;
    std::vector<size_t> ttab_off;
    eab::DevBuf ttab, rstate, rslots;
    cudaStream_t copy_stream = nullptr;    // batch-mode H2D
    cudaStream_t refine_stream = nullptr;  // batch-mode refinement
    cudaEvent_t bev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t rev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // seeds ready / refine done, per working set
    // async (device-resident) searches: overflow flag and a ring of screen
    // kernel event pairs read back by ea_ctx_async_status
    eab::DevBuf async_flag;
    // multi-GPU: NCCL communicator (ea_comm_init) and the sharded path's
    // buffers (local rows, all-gathered rows, merged rows, outcome)
    void* comm = nullptr;  // ncclComm_t
    int comm_rank = 0, comm_world = 1;
    int screen_ctas = 0;  // grid of the last smem lattice screen launch
    eab::DevBuf shard;
    static constexpr int kTimeRing = 64;
    cudaEvent_t tev[2 * kTimeRing] = {};
    int tev_next = 0, tev_pending = 0;
};

namespace eab {

// Launch bookkeeping (the bench's gpu_launches claim comes from here).
inline const char*& last_launch_name() {
    static thread_local const char* name = "";
    return name;
}

inline void count_launch(ea_ctx* ctx, int n = 1) {
    ctx->launches += (uint64_t)n;
    ctx->stats.kernels_launched += n;
    if (ctx->trace_on) {  // EAB_TRACE: an event after every launch (diagnostics)
        cudaEvent_t e;
        if (cudaEventCreate(&e) == cudaSuccess) {
            cudaEventRecord(e, ctx->stream);
            ctx->trace.emplace_back(last_launch_name(), e);
        }
    }
}

// Raises kernel `fn`'s dynamic shared-memory limit to at least `bytes` on
// the context's device.  Function attributes are per device, so the record
// of what was raised is keyed by (function, device) -- not a process-wide
// flag -- and guarded for contexts driven from several host threads.
// Static shared memory the lattice kernels may declare on top of their
// dynamic budget (ea_ctx::smem_optin = opt-in limit - this).
constexpr size_t kLatticeStaticSmem = 2688;

inline void raise_smem_limit(const ea_ctx* ctx, const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> raised;
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = raised[{fn, ctx->device}];
    if (cur >= bytes) return;
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess &&
        bytes + fa.sharedSizeBytes > ctx->smem_optin + kLatticeStaticSmem)
        fail(EA_ERR_INTERNAL, "kernel needs " + std::to_string(bytes) + " B dynamic + " +
                                  std::to_string(fa.sharedSizeBytes) +
                                  " B static shared memory, over the opt-in limit "
                                  "(raise kLatticeStaticSmem)");
    const cudaError_t e =
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess)
        fail(EA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    cur = bytes;
}

inline void check_launch(const char* what) {
    last_launch_name() = what;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fail(EA_ERR_CUDA, std::string("kernel launch ") + what + ": " + cudaGetErrorString(e));
    }
}

}  // namespace eab
