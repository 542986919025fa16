/*
 * edgealign_b200.h -- C-ABI of the B200-native edge-alignment detector.
 *
 * This is the drop-in boundary for the reference's search path
 * (arxiv 2112.05576 reference, library `edgealign`, namespace edgealign).
 * Every entry point names the reference interface it replaces as
 * `path:line` under the reference tree (proj/...).  Signatures use plain
 * pointers, sizes and POD structs only: no C++ or torch types cross it.
 *
 * Ownership: the caller owns every host buffer; a context (ea_ctx) owns the
 * device memory and the CUDA stream its work is queued on; handles
 * (ea_field, ea_model, ea_levels) are freed with their *_free function.
 * Threading: one host thread per context at a time (the reference API is
 * pure and reentrant, proj/include/edgealign/search.h:14-20; contexts are the
 * unit of reentrancy here).
 * Errors: every call returns ea_status.  ea_last_error() returns the message
 * the reference would have put in the matching exception
 * (proj/include/edgealign/errors.h:14-75); the C++ wrapper
 * (include/edgealign_b200.hpp) rethrows the same exception classes.
 *
 * There is no CPU fallback: entry points that compute on the search image
 * fail with EA_ERR_CUDA when no device is present.
 */
#ifndef EDGEALIGN_B200_H
#define EDGEALIGN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per exception class of errors.h:14-75 ---------- */
typedef enum {
    EA_OK = 0,
    EA_ERR_INVALID_ARGUMENT = 1, /* edgealign::InvalidArgument  errors.h:72-75 */
    EA_ERR_SIZE = 2,             /* edgealign::SizeError        errors.h:32-35 */
    EA_ERR_EMPTY_MODEL = 3,      /* edgealign::EmptyModelError  errors.h:39-51 */
    EA_ERR_BOUNDS = 4,           /* edgealign::BoundsError      errors.h:54-57 */
    EA_ERR_BUDGET = 5,           /* edgealign::BudgetError      errors.h:60-63 */
    EA_ERR_GEOMETRY = 6,         /* edgealign::GeometryError    errors.h:66-69 */
    EA_ERR_PARSE = 7,            /* edgealign::ParseError       errors.h:20-29 */
    EA_ERR_CUDA = 8,             /* device missing / CUDA runtime failure       */
    EA_ERR_INTERNAL = 9,
    EA_ERR_NCCL = 10             /* NCCL missing / collective failure (multi-GPU) */
} ea_status;

/* Message of the last failing call on this host thread ("" if none). */
const char* ea_last_error(void);
/* EmptyModelError::max_magnitude() / ParseError::offset() of that failure. */
double ea_last_error_value(void);

/* ---- plain data, layout-compatible with the reference structs ----------- */

/* edgealign::Pose  pose.h:27-31 */
typedef struct {
    double ux, uy, theta;
} ea_pose;

/* edgealign::PoseGrid  pose.h:34-38 */
typedef struct {
    double x0, x1, dx;
    double y0, y1, dy;
    double t0, t1, dt;
} ea_pose_grid;

/* edgealign::GridCounts  pose.h:40-42 */
typedef struct {
    uint64_t nx, ny, nt;
} ea_grid_counts;

enum { EA_POLARITY_SIGNED = 0, EA_POLARITY_IGNORE = 1 }; /* similarity.h:29 */

/* edgealign::ScoreParams  similarity.h:31-35 */
typedef struct {
    int32_t neighborhood;
    int32_t polarity;
    double eps_mag;
} ea_score_params;

/* edgealign::EdgeThresholds  edge_model.h:19-22 */
typedef struct {
    double low, high;
} ea_edge_thresholds;

/* edgealign::EdgePoint  edge_model.h:29-35 */
typedef struct {
    double x_rel, y_rel, dx, dy, mag;
} ea_edge_point;

/* edgealign::BackendKind  search.h:26-31.  The reference's Serial/Parallel
 * kinds are accepted for source compatibility; every kind executes on the
 * context's device (results are bit-equal across kinds by contract,
 * search.h:14-20). */
enum { EA_BACKEND_SERIAL = 0, EA_BACKEND_PARALLEL = 1, EA_BACKEND_CUDA = 2 };

/* edgealign::ScoredPose  search.h:67-71 */
typedef struct {
    double score;
    uint64_t grid_index;
    ea_pose pose;
} ea_scored_pose;

/* edgealign::LevelTrace  search.h:36-40 */
typedef struct {
    int32_t level;
    int32_t _pad;
    ea_pose pose;
    double score;
} ea_level_trace;

#define EA_MAX_LEVELS 16

/* edgealign::SearchOutcome + Detection  search.h:42-47,62-65 */
typedef struct {
    int32_t found;
    int32_t n_trace;
    ea_pose pose;           /* level-0 coordinates */
    double score;
    uint64_t grid_index;    /* winning top-level pose index */
    ea_level_trace trace[EA_MAX_LEVELS]; /* coarse to fine */
} ea_outcome;

/* edgealign::SearchConfig  search.h:49-58 */
typedef struct {
    ea_pose_grid grid;       /* level-0 scale */
    int32_t num_levels;
    int32_t has_thresholds;  /* std::optional<EdgeThresholds> engaged? */
    ea_score_params score_params;
    ea_edge_thresholds thresholds;
    double min_score;
    int32_t topk;
    int32_t refine_radius;
    int32_t backend_kind;
    int32_t worker_count;
} ea_search_config;

/* edgealign::SceneSpec (+ OccluderSpec, IlluminationSpec)  synth.h:56-79 */
enum { EA_TEMPLATE_RECTANGLE = 0, EA_TEMPLATE_RING = 1, EA_TEMPLATE_L_BRACKET = 2,
       EA_TEMPLATE_CROSS = 3 };
typedef struct {
    int32_t canvas_width, canvas_height;
    int32_t template_id, template_size;
    ea_pose true_pose;
    int32_t clutter_segments;
    int32_t has_occluder;
    uint64_t clutter_seed;
    int32_t occ_x, occ_y, occ_w, occ_h;
    double occ_fill;
    double gain, bias, gamma;
    double noise_sigma;
    uint64_t noise_seed;
} ea_scene_spec;

/* One template of a multi-stamp scene. */
typedef struct {
    int32_t template_id, template_size;
    ea_pose pose;
} ea_stamp;

/* Device-side accounting of the last top-level search on a context. */
typedef struct {
    uint64_t poses;            /* grid poses screened                          */
    uint64_t pose_points;      /* poses x model points (the bench metric unit) */
    uint64_t candidates;       /* poses re-scored exactly in fp64               */
    uint64_t candidates_needed;/* candidates the threshold admitted             */
    double screen_delta;       /* rigorous |fp32 screen - fp64 score| bound     */
    double threshold;          /* band threshold used for the exact pass        */
    int32_t screen_path;       /* 1 = smem lattice, 2 = general, 3 = region lattice */
    int32_t flagged_points;    /* rounding-ambiguous (theta, point) pairs        */
    int32_t kernels_launched;  /* kernels of this library in the last search    */
    int32_t _pad;
    double screen_ms;          /* CUDA-event time of the screening kernel        */
    double top_ms;             /* CUDA-event time of the whole top-level search  */
    double image_ms;           /* ea_detect: H2D + pyramid + gradients           */
    double refine_ms;          /* refinement down the pyramid (incl. host prep)  */
} ea_search_stats;

/* ---- context ------------------------------------------------------------ */
typedef struct ea_ctx ea_ctx;
typedef struct ea_field ea_field;
typedef struct ea_model ea_model;
typedef struct ea_levels ea_levels;

/* Create a context on CUDA device `device` with its own stream. */
ea_status ea_ctx_create(int device, ea_ctx** out);
void ea_ctx_destroy(ea_ctx* ctx);
/* Queue subsequent work on a caller-owned cudaStream_t (NULL = own stream). */
ea_status ea_ctx_set_stream(ea_ctx* ctx, void* cuda_stream);
void* ea_ctx_stream(ea_ctx* ctx);
ea_status ea_ctx_synchronize(ea_ctx* ctx);
ea_status ea_ctx_last_stats(const ea_ctx* ctx, ea_search_stats* out);
/* Record CUDA events around the screening kernel and the top-level search
 * (on the context's stream) and report them in ea_search_stats. */
ea_status ea_ctx_set_timing(ea_ctx* ctx, int on);
/* Number of kernels this library has launched on the context so far. */
uint64_t ea_ctx_kernel_launches(const ea_ctx* ctx);
/* Pinned host buffers for fast H2D/D2H (cudaHostAlloc). */
ea_status ea_host_alloc(size_t bytes, void** out);
void ea_host_free(void* p);

/* ---- pose geometry (header-only in the reference, pose.h:45-113) -------- */
ea_status ea_compute_grid_counts(const ea_pose_grid* grid, ea_grid_counts* out); /* pose.h:52-67 */
ea_status ea_pose_at(const ea_pose_grid* grid, uint64_t index, ea_pose* out); /* pose.h:77-92 */

/* ---- image + gradients (image.cpp:248-291, gradient.cpp:12-27) ---------- */
int ea_max_pyramid_levels(int width, int height);                  /* image.cpp:263-272 */
/* Level dims of a pyramid (floor halving), dims[2*l], dims[2*l+1]. */
ea_status ea_pyramid_dims(int width, int height, int num_levels, int* dims);
/* downsample  image.cpp:248-261, device 2x2 box mean. */
ea_status ea_downsample(ea_ctx* ctx, const double* image, int width, int height,
                        double* out);
/* build_pyramid  image.cpp:274-291; levels concatenated level-major. */
ea_status ea_build_pyramid(ea_ctx* ctx, const double* image, int width, int height,
                           int num_levels, double* out_levels);
/* compute_gradients  gradient.cpp:12-27 on the device (host in/out). */
ea_status ea_compute_gradients(ea_ctx* ctx, const double* image, int width, int height,
                               double* gx, double* gy, double* mag);

/* Device gradient fields (edgealign::GradientField, gradient.h:17-36). */
ea_status ea_field_upload(ea_ctx* ctx, const double* gx, const double* gy,
                          const double* mag, int width, int height, ea_field** out);
ea_status ea_field_from_image(ea_ctx* ctx, const double* image, int width, int height,
                              ea_field** out);
ea_status ea_field_download(ea_ctx* ctx, const ea_field* f, double* gx, double* gy,
                            double* mag);
ea_status ea_field_dims(const ea_field* f, int* width, int* height);
void ea_field_free(ea_field* f);

/* ---- template side (edge_model.cpp:17-149), host C++ -------------------- */
ea_status ea_default_thresholds(const double* mag, int width, int height,
                                ea_edge_thresholds* out);       /* edge_model.cpp:17-24 */
/* extract_edge_model  edge_model.cpp:53-149.  `cap` >= width*height always
 * suffices; *n_out receives the point count. */
ea_status ea_extract_edge_model(const double* gx, const double* gy, const double* mag,
                                int width, int height, const ea_edge_thresholds* th,
                                int level, ea_edge_point* points, int cap, int* n_out,
                                double* centroid_x, double* centroid_y);

/* Device edge models (edgealign::EdgeModel, edge_model.h:40-45). */
/* extract_edge_model on a device field (edge_model.cpp:53-149): peak, NMS,
 * hysteresis and emission on the device; th == NULL uses default_thresholds
 * (edge_model.cpp:17-24).  Same points, order and centroid as the host
 * ea_extract_edge_model. */
ea_status ea_field_extract_model(ea_ctx* ctx, const ea_field* field, const ea_edge_thresholds* th,
                                 int level, ea_model** out);
/* Points (AoS, model order) and centroid of a model. */
ea_status ea_model_points(const ea_model* m, ea_edge_point* points, int cap, int* n_out,
                          double* centroid_x, double* centroid_y);
ea_status ea_model_create(ea_ctx* ctx, const ea_edge_point* points, int n,
                          double centroid_x, double centroid_y, int source_level,
                          ea_model** out);
int ea_model_size(const ea_model* m);
void ea_model_free(ea_model* m);

/* ---- similarity (similarity.cpp:15-126) --------------------------------- */
ea_status ea_validate_params(const ea_score_params* p);           /* similarity.cpp:15-23 */
/* point_vote  similarity.cpp:58-64 */
ea_status ea_point_vote(ea_ctx* ctx, double dir_x, double dir_y, const ea_field* f,
                        int cx, int cy, const ea_score_params* p, double* out);
/* rotate_model  similarity.cpp:68-88; outputs n doubles each. */
ea_status ea_rotate_model(ea_ctx* ctx, const ea_model* m, double theta, double* px,
                          double* py, double* dx, double* dy);
/* pose_score  similarity.cpp:121-126 */
ea_status ea_pose_score(ea_ctx* ctx, const ea_model* m, const ea_pose* pose,
                        const ea_field* f, const ea_score_params* p, double* value,
                        int* n_inbounds);

/* ---- search (search.cpp:144-202) ---------------------------------------- */
/* exhaustive_search  search.cpp:144-153 (k = 1). */
ea_status ea_exhaustive_search(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                               const ea_pose_grid* grid, const ea_score_params* p,
                               int backend_kind, ea_scored_pose* out);
/* search_topk  search.cpp:155-167. `out` holds k entries; *n_out <= k. */
ea_status ea_search_topk(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                         const ea_pose_grid* grid, const ea_score_params* p,
                         int backend_kind, int k, ea_scored_pose* out, int* n_out);
/* Top-k restricted to theta indices [it_begin, it_end): one shard of the
 * reference's contiguous index partition (search.cpp:116-120) snapped to
 * theta.  Merging shard results with ea_merge_topk equals search_topk. */
ea_status ea_search_topk_slab(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                              const ea_pose_grid* grid, const ea_score_params* p,
                              int k, uint64_t it_begin, uint64_t it_end,
                              ea_scored_pose* out, int* n_out);
/* The run_search merge (search.cpp:130-139): sort by `better`, keep k. */
ea_status ea_merge_topk(const ea_scored_pose* in, int n, int k, ea_scored_pose* out,
                        int* n_out);
/* score_map  search.cpp:169-202 (exact fp64). */
ea_status ea_score_map(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                       const ea_pose_grid* grid, const ea_score_params* p,
                       uint64_t max_cells, double* out);
/* The fp32 screening map the top-level kernel produces (|map-exact| <=
 * stats.screen_delta per pose).  Not in the reference; exposed for tests. */
ea_status ea_screen_map(ea_ctx* ctx, const ea_model* m, const ea_field* f,
                        const ea_pose_grid* grid, const ea_score_params* p,
                        uint64_t max_cells, float* out, double* delta);

/* ---- coarse to fine (search.cpp:204-364) -------------------------------- */
/* prepare_levels  search.cpp:208-238 from host pyramids (level-major
 * pointer arrays). */
ea_status ea_prepare_levels(ea_ctx* ctx, const double* const* tmpl_levels,
                            const int* tmpl_dims, int n_tmpl,
                            const double* const* work_levels, const int* work_dims,
                            int n_work, const ea_search_config* cfg, ea_levels** out);
/* Template side only (models for every level); the working side is attached
 * per image by ea_levels_set_image.  Template pyramid is built on device. */
ea_status ea_prepare_models(ea_ctx* ctx, const double* tmpl, int tw, int th,
                            const ea_search_config* cfg, ea_levels** out);
/* Working side from a level-0 host image: H2D, device pyramid + gradients. */
ea_status ea_levels_set_image(ea_ctx* ctx, ea_levels* lv, const double* image, int w,
                              int h);
int ea_levels_count(const ea_levels* lv);
ea_status ea_levels_model(const ea_levels* lv, int level, ea_edge_point* points,
                          int cap, int* n_out, double* centroid_x, double* centroid_y);
const ea_field* ea_levels_field(const ea_levels* lv, int level);
const ea_model* ea_levels_get_model(const ea_levels* lv, int level);
void ea_levels_free(ea_levels* lv);

/* search_levels  search.cpp:254-357 */
ea_status ea_search_levels(ea_ctx* ctx, const ea_levels* lv, const ea_search_config* cfg,
                           ea_outcome* out);
/* The two halves of search_levels, for theta-sharded multi-GPU runs:
 * top-level seeds on a theta slab, then refinement from merged seeds. */
ea_status ea_search_top_slab(ea_ctx* ctx, const ea_levels* lv,
                             const ea_search_config* cfg, uint64_t it_begin,
                             uint64_t it_end, ea_scored_pose* seeds, int* n_seeds);
/* Device-resident form of ea_search_top_slab (the multi-GPU data path):
 * enqueued on the context's stream, no host sync.  Writes k rows of five
 * doubles {score, grid_index, ux, uy, theta} to device memory d_rows (rows
 * past the count have a NaN score) -- the layout all-gathered over NCCL. */
ea_status ea_search_top_slab_async(ea_ctx* ctx, const ea_levels* lv,
                                   const ea_search_config* cfg, uint64_t it_begin,
                                   uint64_t it_end, double* d_rows);
/* The `better` merge (search.cpp:130-139) of n_rows device rows into k
 * device rows, enqueued on the context's stream. */
ea_status ea_merge_rows_async(ea_ctx* ctx, const double* d_rows, int n_rows, int k,
                              double* d_out);
/* Synchronises the context; *overflowed = 1 if an async search since the
 * last call admitted more candidates than its buffer (its rows are then
 * unreliable: rerun with ea_search_top_slab); screen_ms[0..*n_times) = the
 * screening-kernel times of the timed searches since the last call. */
ea_status ea_ctx_async_status(ea_ctx* ctx, int* overflowed, float* screen_ms, int cap,
                              int* n_times);
ea_status ea_refine(ea_ctx* ctx, const ea_levels* lv, const ea_search_config* cfg,
                    const ea_scored_pose* seeds, int n_seeds, ea_outcome* out);
/* coarse_to_fine  search.cpp:359-364 */
ea_status ea_coarse_to_fine(ea_ctx* ctx, const double* const* tmpl_levels,
                            const int* tmpl_dims, int n_tmpl,
                            const double* const* work_levels, const int* work_dims,
                            int n_work, const ea_search_config* cfg, ea_outcome* out);
/* Production detect: models prepared once, one host image per call
 * (H2D + pyramid + gradients + search_levels + D2H). */
ea_status ea_detect(ea_ctx* ctx, ea_levels* lv, const double* image, int w, int h,
                    const ea_search_config* cfg, ea_outcome* out);

/* Multi-model detect (BASELINE configs[4]): one host image, n prepared
 * template sides (one ea_levels per model, all prepared for cfg).  The
 * working pyramid is built once -- into models[0]'s working side -- and
 * every model's search_levels runs against it, back to back on the stream
 * with one sync; outs[n].  Equals ea_detect per model. */
ea_status ea_detect_multi(ea_ctx* ctx, ea_levels* const* models, int n, const double* image,
                          int w, int h, const ea_search_config* cfg, ea_outcome* outs);

/* Throughput mode (BASELINE configs[3]): `count` host images of one size,
 * image i+1's H2D overlapping image i's device pipeline; outs[count]. */
ea_status ea_detect_batch(ea_ctx* ctx, ea_levels* lv, const double* const* images, int count,
                          int w, int h, const ea_search_config* cfg, ea_outcome* outs);

/* ---- multi-GPU: theta-slab sharding ------------
 * One process (or host thread) per GPU, one context per GPU.  The
 * reference partitions the theta-major pose index into contiguous blocks,
 * one per worker (search.cpp:116-120), and merges the per-worker top-k
 * lists by `better` (search.cpp:130-139); snapped to theta the blocks are
 * theta slabs, and because the merge is an associative, commutative total
 * order, one all-gather of every rank's k rows reproduces search_topk bit
 * for bit.  The collectives are NCCL (loaded at run time, the copy torch
 * already mapped when there is one), enqueued on the context's stream. */
#define EA_COMM_ID_BYTES 128
typedef struct {
    char internal[EA_COMM_ID_BYTES]; /* ncclUniqueId */
} ea_comm_id;

/* [it_begin, it_end) of `rank` among `world`: the reference's block
 * partition (search.cpp:116-120) on the theta axis.  Host only. */
void ea_theta_slab(uint64_t nt, int rank, int world, uint64_t* it_begin, uint64_t* it_end);
/* Rank 0 creates the id and hands it to every rank out of band (MPI, a TCP
 * store, torch.distributed, ...). */
ea_status ea_comm_unique_id(ea_comm_id* out);
/* Join the context's device to the communicator (ncclCommInitRank;
 * collective: every rank calls it). */
ea_status ea_comm_init(ea_ctx* ctx, int rank, int world, const ea_comm_id* id);
ea_status ea_comm_info(const ea_ctx* ctx, int* rank, int* world);
ea_status ea_comm_destroy(ea_ctx* ctx);
/* The exchange step of a sharded search (search.cpp:130-139), no host sync:
 * all-gather every rank's k device rows {score, index, ux, uy, theta} (as
 * ea_search_top_slab_async writes them) and `better`-merge them into k rows
 * at d_merged on every rank.  Collective. */
ea_status ea_gather_rows_async(ea_ctx* ctx, const double* d_local, int k, double* d_merged);
/* search_levels (search.cpp:254-357) sharded by theta: every rank screens
 * and verifies its slab of the top level (lv's working image must be set on
 * every rank), one NCCL all-gather of the k rows, the `better` merge, then
 * rank 0 refines down the pyramid and broadcasts the outcome.  `out` equals
 * ea_search_levels' on every rank.  Collective. */
ea_status ea_search_levels_sharded(ea_ctx* ctx, const ea_levels* lv,
                                   const ea_search_config* cfg, ea_outcome* out);
/* Production detect sharded by theta (BASELINE configs[2]): rank 0 uploads
 * the level-0 host image and builds the pyramid and fields; the top level's
 * field is broadcast over NCCL (the other ranks pass image = NULL and only
 * the dimensions); then as ea_search_levels_sharded.  Collective. */
ea_status ea_detect_sharded(ea_ctx* ctx, ea_levels* lv, const double* image, int w, int h,
                            const ea_search_config* cfg, ea_outcome* out);

/* Multi-model sharding (BASELINE configs[4]): the
 * reference searches each model with its own search_topk (search.cpp:
 * 155-167); here every (model, theta slab) is a work item costed in
 * pose-evals (poses x top-level model points, + fixed_evals per search for
 * the launch / finish overhead), big models split into slabs of about one
 * rank's share, small ones kept whole, assigned longest-first to the least
 * loaded rank that holds no other slab of the model.  Deterministic: every
 * rank computes the same plan. */
typedef struct {
    int32_t rank;
    int32_t model;
    uint64_t it_begin, it_end; /* theta slab [it_begin, it_end) of the model */
    double cost;               /* pose-evals + fixed_evals */
} ea_work_item;

/* plane_poses[m] = nx * ny, thetas[m] = nt, n_top[m] = top-level model
 * points.  items: cap entries; *n_items receives the count (<= n_models *
 * world).  Host only. */
ea_status ea_plan_multi(const uint64_t* plane_poses, const uint64_t* thetas, const int* n_top,
                        int n_models, int world, double fixed_evals, ea_work_item* items,
                        int cap, int* n_items);
/* The exchange step of a multi-model sharded search: all-gather every
 * rank's n_models x k device rows (model m's k rows at d_local + 5*k*m;
 * NaN rows for models the rank has no slab of) and `better`-merge them per
 * model into d_merged (same layout).  Collective, no host sync. */
ea_status ea_gather_rows_multi_async(ea_ctx* ctx, const double* d_local, int n_models, int k,
                                     double* d_merged);
/* Multi-model detect sharded over the communicator (collective): rank 0
 * uploads the host image and builds the shared pyramid (into models[0]'s
 * working side), the top level's field is broadcast, every rank searches
 * its ea_plan_multi items, one NCCL all-gather of all models' k rows, a
 * `better` merge per model, rank 0 refines every model and broadcasts the
 * outcomes.  outs[n] equals ea_detect_multi's on every rank. */
ea_status ea_detect_multi_sharded(ea_ctx* ctx, ea_levels* const* models, int n,
                                  const double* image, int w, int h,
                                  const ea_search_config* cfg, ea_outcome* outs);

/* ---- Netpbm codecs (image.cpp:26-219), host C++, bytes in / bytes out ---- */
/* luminance_to_byte  image.cpp:26-34: clamp to [0, 255], round half up. */
uint8_t ea_luminance_to_byte(double v);
/* load_pgm  image.cpp:90-147 (P2 / P5, maxval <= 255).  out == NULL: only the
 * dimensions.  Parse errors: EA_ERR_PARSE, ea_last_error_value() = offset. */
ea_status ea_load_pgm(const uint8_t* bytes, size_t size, double* out, size_t cap, int* width,
                      int* height);
/* save_pgm  image.cpp:189-197 (P5).  out == NULL: *n_out = bytes needed. */
ea_status ea_save_pgm(const double* image, int width, int height, uint8_t* out, size_t cap,
                      size_t* n_out);
/* save_ppm  image.cpp:203-227 (P6, gray + overlay points in one colour;
 * out-of-bounds points skipped).  overlay_xy: n_overlay (x, y) pairs. */
ea_status ea_save_ppm(const double* image, int width, int height, const int* overlay_xy,
                      int n_overlay, uint8_t r, uint8_t g, uint8_t b, uint8_t* out, size_t cap,
                      size_t* n_out);
/* Pixels of model points projected at a pose, as the scorer projects them
 * (similarity.cpp:79-80, 104-108): the overlay of a detection. */
ea_status ea_overlay_points(const ea_edge_point* points, int n, const ea_pose* pose,
                            int* out_xy);

/* ---- synthetic scenes (synth.cpp:24-300), host C++ ---------------------- */
ea_status ea_render_template(int template_id, int size, double* out);  /* synth.cpp:62-128 */
/* compose_scene  synth.cpp:178-300.  canvas: W*H, tmpl: size*size. */
ea_status ea_compose_scene(const ea_scene_spec* spec, double* canvas, double* tmpl,
                           ea_pose* truth_pose, double* occluded_fraction);
/* Multi-stamp scene (BASELINE configs[4]; not in the reference, which stamps
 * one template per scene -- SURVEY.md H8): background + clutter as
 * compose_scene, then each stamp in order with compose_scene's inverse-mapped
 * paste (synth.cpp:224-244), then occluder / illumination / noise.  The
 * spec's template_id, template_size and true_pose are ignored.  With one stamp
 * the canvas equals ea_compose_scene's. */
ea_status ea_compose_multi(const ea_scene_spec* spec, const ea_stamp* stamps, int n_stamps,
                           double* canvas);

#ifdef __cplusplus
}
#endif
#endif /* EDGEALIGN_B200_H */
