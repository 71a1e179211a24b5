/*
 * svlf_b200.h -- C ABI of the B200-native SVLF render/train path.
 *
 * This is the drop-in boundary. The reference (/root/reference/proj) is a C++
 * static library (svlf_core, src/CMakeLists.txt:1-18) with no FFI; every entry
 * point below replaces one reference interface, cited per function. The C++
 * API in include/svlf/ headers (same names and signatures as the reference
 * headers) is a thin shim over these calls, and the Python package
 * paper_2205_07058_b200 binds them with ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes; no exceptions cross the ABI. Every call returns
 *    an svlf_status; on failure svlf_last_error() (thread-local) holds the
 *    reference's exception message, e.g. "empty occupancy", "tangent ray",
 *    "point not in voxel", "surface point outside voxel". The C++ shim
 *    rethrows the same exception type with the same message
 *    (SVLF_ERR_INVALID_ARGUMENT -> std::invalid_argument, SVLF_ERR_RUNTIME ->
 *    std::runtime_error, SVLF_ERR_OUT_OF_RANGE -> std::out_of_range).
 *  - Geometry is fp64, features/decoders fp32 (reference geometry.hpp:8).
 *  - Host-pointer calls are synchronous: results are in the caller's buffers
 *    on return. *_device calls take device pointers and are asynchronous on
 *    the context stream (svlf_ctx_synchronize to wait).
 *  - Flat decoder layout: per layer l, W_l row-major [out][in] then b_l
 *    (reference include/svlf/mlp.hpp:50-53). f_T 134->128->2 (17,538 floats),
 *    f_C 38->128->128->128->3 (38,403 floats).
 *  - There is no CPU fallback: a missing or failing CUDA device is an error.
 */
#ifndef SVLF_B200_H
#define SVLF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVLF_ABI_VERSION 1
#define SVLF_FEAT_T_DIM 64   /* model.hpp:13 kThicknessFeatDim */
#define SVLF_FEAT_C_DIM 32   /* model.hpp:14 kColorFeatDim */
#define SVLF_DEC_T_SIZE 17538
#define SVLF_DEC_C_SIZE 38403

typedef enum svlf_status {
    SVLF_OK = 0,
    SVLF_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    SVLF_ERR_RUNTIME = 2,          /* std::runtime_error */
    SVLF_ERR_OUT_OF_RANGE = 3,     /* std::out_of_range */
    SVLF_ERR_CUDA = 4,             /* device failure (no reference analogue) */
    SVLF_ERR_CAPACITY = 5          /* caller buffer too small; required size reported */
} svlf_status;

/* Decoder arithmetic for render: FP32 = CUDA-core fp32 in the reference's
 * accumulation order (parity: max-abs <= 1e-3); BF16 / FP16 = the fused
 * tcgen05 tensor-core decoder with bf16 or fp16 operands and fp32
 * accumulation in TMEM (parity: PSNR delta <= 0.05 dB; same tensor rate,
 * fp16 carries 3 more mantissa bits). */
typedef enum svlf_precision {
    SVLF_PRECISION_FP32 = 0,
    SVLF_PRECISION_BF16 = 1,
    SVLF_PRECISION_FP16 = 2,
    SVLF_PRECISION_TF32 = 3,  /* train step only: weight-gradient GEMMs on tensor cores with TF32 operands */
    SVLF_PRECISION_TF32X3 = 4 /* train step only: every dense-layer GEMM on tensor cores as three TF32
                                 products of split (hi, lo) operands: fp32-level accuracy */
} svlf_precision;

/* reference LossMode (src/train.cpp:37): stage 1 = SURFACE, stages 2-3 = VOLUMETRIC */
typedef enum svlf_loss_mode { SVLF_LOSS_SURFACE = 0, SVLF_LOSS_VOLUMETRIC = 1 } svlf_loss_mode;

typedef struct svlf_ctx svlf_ctx;
typedef struct svlf_octree svlf_octree;
typedef struct svlf_model svlf_model;

/* GridConfig, include/svlf/octree.hpp:13-19 */
typedef struct svlf_grid {
    uint32_t resolution;
    uint32_t dilation;
    double lo[3];
    double hi[3];
} svlf_grid;

/* Camera, include/svlf/camera.hpp:12-33 (row-major camera_to_world) */
typedef struct svlf_camera {
    double fx, fy, cx, cy;
    double camera_to_world[16];
    uint32_t width, height;
} svlf_camera;

/* RenderStats, include/svlf/render.hpp:94-100 (additive counters) */
typedef struct svlf_render_stats {
    long long rays, rays_with_hits, traversal_hits, thickness_queries, color_queries;
} svlf_render_stats;

/* LossWeights, include/svlf/train.hpp:43-48 */
typedef struct svlf_loss_weights {
    double eta, tau, empty, alpha;
} svlf_loss_weights;

/* LossStats, include/svlf/train.hpp:50-54 (additive counters) */
typedef struct svlf_loss_stats {
    long long rays, skipped_rays, eta_skipped;
} svlf_loss_stats;

typedef struct svlf_octree_info {
    int leaf_level;
    uint32_t vertex_count;
    size_t leaf_count;
    size_t dropped_points;
    double cell_size;
    size_t level_size[22];
} svlf_octree_info;

/* Per-launch device timings of the last render/train call (CUDA events on the
 * context stream), milliseconds. */
typedef struct svlf_timings {
    float traverse_ms, emit_ms, decode_ms, composite_ms, backward_ms, adam_ms, total_ms;
    long long hits;
    long long overflow_rays; /* rays re-traversed by the per-ray fallback walker */
    long long dense_rays;    /* rays whose block queue overflowed, re-run by the second (16-ray) cooperative pass */
} svlf_timings;

/* ---- context -------------------------------------------------------- */
const char* svlf_last_error(void);
int svlf_abi_version(void);
svlf_status svlf_ctx_create(int device, svlf_ctx** out);
svlf_status svlf_ctx_destroy(svlf_ctx* ctx);
svlf_status svlf_ctx_synchronize(svlf_ctx* ctx);
/* Run the context's work on an external cudaStream_t (e.g. a framework's
 * current stream, so its CUDA events time this library); NULL restores the
 * context's own stream. */
svlf_status svlf_ctx_set_stream(svlf_ctx* ctx, void* cuda_stream);
svlf_status svlf_ctx_last_timings(const svlf_ctx* ctx, svlf_timings* out);
/* Diagnostics: with counting enabled, traversals run a variant of the
 * cooperative passes that counts ray-box tests (root + each occupied child of
 * every expanded node: the reference's ray_aabb calls in
 * SparseOctree::traverse, src/octree.cpp:185-235; tiles handed to the next
 * pass are counted by the pass that completes them; the per-ray fallback
 * walker is not counted). svlf_ctx_last_node_tests reads the count of the
 * last traversal (last band of a banded frame; 32-bit; synchronizes). */
svlf_status svlf_ctx_set_node_test_counting(svlf_ctx* ctx, int enable);
svlf_status svlf_ctx_last_node_tests(svlf_ctx* ctx, long long* out);
/* Arithmetic of the train step's dense layers (no cuBLAS: this library's
 * tcgen05 kernels, gemm_x3.cu): SVLF_PRECISION_FP32 (default) and
 * SVLF_PRECISION_TF32X3 both run every GEMM on the tensor cores as
 * hi*lo + lo*hi + hi*hi of TF32 splits x = hi + lo with fp32 accumulation
 * (fp32-level accuracy: gradients within 1e-4 rel-L2 of the reference);
 * weight gradients are reduced in a fixed CTA order, so steps are bitwise
 * reproducible run to run. SVLF_PRECISION_TF32 runs the weight-gradient
 * reductions with plain TF32 operands (gradients within 2e-2, the 16-bit
 * tolerance of SURVEY.md §8(c)). */
svlf_status svlf_ctx_set_train_precision(svlf_ctx* ctx, svlf_precision precision);
/* Diagnostics: one train-step dense-layer GEMM (gemm_x3.cu) on device
 * buffers of the current device, synchronous. kind 0: out[j][:n] = relu(W
 * in[K rows] + bias) (W O x K, O <= 128); 1: out[j][:n] = sum_o W[o][k0+j]
 * in[o][:n], zeroed where mask[j][:] <= 0 (mask may be NULL); 2: out (O x K)
 * = in (O rows) in2^T (K rows), out2 (O) = row sums of in; matrices have row
 * stride ld floats. products: 3 (3xTF32) or 1 (TF32, kind 2 only). */
svlf_status svlf_debug_gemm_x3(int kind, const float* W, uint32_t O, uint32_t K, uint32_t k0, const float* bias,
                               const float* in, const float* in2, const float* mask, float* out, float* out2,
                               uint32_t n, uint32_t ld, int products);
/* Count of this library's kernel launches on the context since creation. */
long long svlf_ctx_kernel_launches(const svlf_ctx* ctx);

/* Page-locked host memory. Frame outputs passed to svlf_render_frame in
 * page-locked memory (from here, cudaMallocHost or cudaHostRegister) receive
 * the device-to-host copies directly, band by band, with no staging copy. */
svlf_status svlf_host_alloc(size_t bytes, void** out);
svlf_status svlf_host_free(void* p);

/* ---- data parallelism (one process per GPU, NCCL over NVLink) ----------
 * svlf_nccl_unique_id fills 128 bytes on one rank; every rank passes the same
 * bytes to svlf_ctx_attach_nccl. With a communicator attached, train steps
 * all-reduce (sum) the loss, the loss statistics, the decoder gradients and
 * the feature gradients before the (replicated, identical) Adam update, so
 * each rank trains on its own shard of the batch. Feature
 * gradients are exchanged sparsely: only rows touched by any rank's hits
 * (union of per-rank touched-row masks) are reduced. */
svlf_status svlf_nccl_unique_id(void* out128);
svlf_status svlf_ctx_attach_nccl(svlf_ctx* ctx, const void* unique_id128, int rank, int world);
svlf_status svlf_ctx_detach_nccl(svlf_ctx* ctx);
/* The same exchange through a host callback (gloo, MPI, a test harness)
 * instead of NCCL: the library copies each buffer to page-locked host memory,
 * calls fn to all-reduce it in place across the `world` ranks (every rank
 * calls fn the same number of times with the same counts, in the same order),
 * and copies it back. fn returns 0 on success. */
typedef enum svlf_dtype { SVLF_DTYPE_F32 = 0, SVLF_DTYPE_F64 = 1, SVLF_DTYPE_U8 = 2 } svlf_dtype;
typedef enum svlf_reduce_op { SVLF_REDUCE_SUM = 0, SVLF_REDUCE_MAX = 1 } svlf_reduce_op;
typedef int (*svlf_allreduce_fn)(void* user, void* host_buf, size_t count, svlf_dtype dtype, svlf_reduce_op op);
svlf_status svlf_ctx_attach_collective(svlf_ctx* ctx, svlf_allreduce_fn fn, void* user, int rank, int world);

/* ---- per-point / per-ray operations of the reference's public API, batched
 * on the GPU (host buffers in and out; tests and debugging, not the frame or
 * train paths, which fuse the same arithmetic). Single-point results are
 * bit-identical to the reference built without FMA contraction. Errors carry
 * the reference's messages: "point not in voxel" (runtime), "unknown voxel
 * id" (out_of_range), "tangent ray" (runtime), "negative optical thickness"
 * (invalid_argument), "surface point outside voxel" (runtime). */
/* local_coords (features.hpp:69, src/features.cpp:22-31): u n x 3 */
svlf_status svlf_local_coords(svlf_ctx* ctx, const svlf_octree* tree, const uint64_t* voxel_ids,
                              const double* points, size_t n, double* u_out);
/* interpolate (features.hpp:72-74, src/features.cpp:33-47) for a volume of
 * `rows` x `dim` values (f32 or f64): out n x dim */
svlf_status svlf_interpolate(svlf_ctx* ctx, const svlf_octree* tree, svlf_dtype dtype, const void* volume,
                             uint32_t rows, uint32_t dim, const uint64_t* voxel_ids, const double* points, size_t n,
                             void* out);
/* interpolate_backward (features.hpp:76-80, src/features.cpp:49-84):
 * grad_buf (rows x dim) += w_b * upstream (n x dim) per point (points that
 * share a row are summed in an unspecified order); pos_jac (n x dim x 3,
 * optional) = d z / d point */
svlf_status svlf_interpolate_backward(svlf_ctx* ctx, const svlf_octree* tree, svlf_dtype dtype, const void* volume,
                                      uint32_t rows, uint32_t dim, const uint64_t* voxel_ids, const double* points,
                                      size_t n, const void* upstream, void* grad_buf, double* pos_jac);
/* parameterize_ray (render.hpp:28, src/render.cpp:16-28): rays n x 6, boxes
 * n x (lo xyz, hi xyz) -> n x (p1 xyz, p2 xyz) */
svlf_status svlf_parameterize_rays(svlf_ctx* ctx, const double* rays, const double* boxes, size_t n, double* out6);
/* composite (render.hpp:60-62, src/render.cpp:65-87) of n_lists sample lists
 * (list l = samples offsets[l] .. offsets[l+1]-1): colour (3 per list) and
 * alpha; weights (per sample) optional; with t_s (per sample) the expected
 * depth of render_ray (src/render.cpp:106-114) into out_depth */
svlf_status svlf_composite(svlf_ctx* ctx, const uint64_t* offsets, size_t n_lists, const double* taus,
                           const double* colors, const double* t_s, double* out_color, double* out_alpha,
                           double* out_depth, double* weights);
/* evaluate_voxel (render.hpp:49-51, src/render.cpp:30-63) for n (ray, hit)
 * pairs with the fp32 decoders: tau, eta, x_s (3), t_s = eta t_in + (1 - eta)
 * t_out, colour (3); any output may be NULL */
svlf_status svlf_evaluate_voxels(svlf_ctx* ctx, svlf_model* model, const double* rays, const uint64_t* voxel_ids,
                                 const double* t_in, const double* t_out, size_t n, double* tau, double* eta,
                                 double* x_s, double* t_s, double* color);
/* eta_gt (train.hpp:41, src/train.cpp:30-35) */
svlf_status svlf_eta_gt(svlf_ctx* ctx, const double* t_in, const double* t_out, const double* depth, size_t n,
                        double* out);

/* ---- octree: SparseOctree::build / from_leaves (octree.hpp:47,82; src/octree.cpp:30-142)
 * ctx may be NULL: the octree is then host-only and is uploaded to the device
 * of the first context that renders/traverses with it. */
svlf_status svlf_octree_build(svlf_ctx* ctx, const svlf_grid* grid, const double* points_xyz,
                              size_t n_points, svlf_octree** out);
/* With a context, svlf_octree_build runs on its GPU (radix sort / unique,
 * octree_build.cu; byte-identical to the host build); _device takes points
 * already in device memory (e.g. back-projected on the GPU). */
svlf_status svlf_octree_build_device(svlf_ctx* ctx, const svlf_grid* grid, const double* d_points_xyz,
                                     size_t n_points, svlf_octree** out);
svlf_status svlf_octree_from_leaves(svlf_ctx* ctx, const svlf_grid* grid, const uint64_t* leaf_codes,
                                    size_t n_leaves, svlf_octree** out);
svlf_status svlf_octree_destroy(svlf_octree* tree);
svlf_status svlf_octree_get_info(const svlf_octree* tree, svlf_octree_info* out);
svlf_status svlf_octree_level_codes(const svlf_octree* tree, int level, uint64_t* out);
/* corner_vertices for every leaf, leaf-code order, 8 ids per leaf (octree.hpp:69-71) */
svlf_status svlf_octree_corner_ids(const svlf_octree* tree, uint32_t* out);

/* ---- traversal: SparseOctree::traverse (octree.hpp:75-78; src/octree.cpp:185-235)
 * Batched: rays are n x (origin xyz, unit dir xyz). offsets[n+1] is the CSR
 * row pointer. Hits (voxel_id = leaf Morton code, t_in, t_out, and x1/x2 as
 * 6 doubles when x12 is non-null) are written only if the total fits
 * `capacity`; *total always receives the required count (SVLF_ERR_CAPACITY
 * otherwise). Bit-exact with the reference built without FMA contraction. */
svlf_status svlf_traverse(svlf_ctx* ctx, const svlf_octree* tree, const double* rays, size_t n,
                          uint64_t* offsets, size_t capacity, uint64_t* voxel_ids, double* t_in,
                          double* t_out, double* x12, size_t* total);

/* ---- model: SvlfModel + ModelAdam (model.hpp:16-34,80-90) ----------- */
/* The model runs on `ctx`; destroy models before their context. */
svlf_status svlf_model_create(svlf_ctx* ctx, const svlf_octree* tree, svlf_model** out);
svlf_status svlf_model_destroy(svlf_model* model);
/* init_model(octree, seed), src/model.cpp:15-28 (bit-identical parameters) */
svlf_status svlf_model_init(svlf_model* model, uint64_t seed);
svlf_status svlf_model_set_params(svlf_model* model, const float* feat_t, const float* feat_c,
                                  const float* dec_t, const float* dec_c);
svlf_status svlf_model_get_params(svlf_model* model, float* feat_t, float* feat_c, float* dec_t,
                                  float* dec_c);
/* Gradients of the last svlf_loss_grads / svlf_train_step call (sums over rays). */
svlf_status svlf_model_get_grads(svlf_model* model, float* feat_t, float* feat_c, float* dec_t,
                                 float* dec_c);
/* Adam state, tensor order: feat_t, feat_c, then per layer W,b of f_T, then
 * per layer W,b of f_C (ModelAdam, model.hpp:83-90). steps[] has 14 entries. */
svlf_status svlf_model_get_adam(svlf_model* model, float* m_all, float* v_all, uint64_t* steps);
svlf_status svlf_model_set_adam(svlf_model* model, const float* m_all, const float* v_all,
                                const uint64_t* steps);
/* AdamState::beta1 / beta2 / eps of the 14 tensors (mlp.hpp:117-128; same
 * order); the defaults are 0.9f / 0.999f / 1e-8f, svlf_model_init resets them. */
svlf_status svlf_model_set_adam_hyper(svlf_model* model, const float* beta1, const float* beta2, const float* eps);
svlf_status svlf_model_get_adam_hyper(svlf_model* model, float* beta1, float* beta2, float* eps);
size_t svlf_model_param_count(const svlf_model* model);

/* ---- render: render_frame(model, camera, out, stats, background) (render.hpp:104-105;
 * src/render.cpp:209-247). Host buffers: rgb W*H*3 interleaved, alpha W*H,
 * depth W*H (0 where alpha <= 1e-4). background may be NULL (black). stats may
 * be NULL; counters are added to it. */
svlf_status svlf_render_frame(svlf_ctx* ctx, svlf_model* model, const svlf_camera* cam,
                              const float* background, svlf_precision precision, float* rgb,
                              float* alpha, float* depth, svlf_render_stats* stats);
/* Pipelined variant: submit enqueues the whole frame and its device-to-host
 * copies and returns a ticket; wait completes it (host buffers valid, stats
 * added). Up to two frames may be in flight per context, so one frame's copies
 * overlap the next frame's rendering. The host buffers must stay valid until
 * the wait; page-locked buffers receive the copies directly. */
svlf_status svlf_render_frame_submit(svlf_ctx* ctx, svlf_model* model, const svlf_camera* cam,
                                     const float* background, svlf_precision precision, float* rgb,
                                     float* alpha, float* depth, uint64_t* ticket);
svlf_status svlf_render_frame_wait(svlf_ctx* ctx, uint64_t ticket, svlf_render_stats* stats);
/* Same with DEVICE output buffers, asynchronous (inputs resident in HBM). */
svlf_status svlf_render_frame_device(svlf_ctx* ctx, svlf_model* model, const svlf_camera* cam,
                                     const float* background, svlf_precision precision,
                                     float* d_rgb, float* d_alpha, float* d_depth,
                                     svlf_render_stats* stats);
/* svlf_render_frame_device in two phases: the submit enqueues the frame on
 * the context's stream and returns (no host round trip in the 16-bit modes);
 * the finish waits for it, checks the hit counters and the device error flag,
 * adds the frame's statistics and, if the hit buffers overflowed, renders the
 * frame again synchronously. One pending frame per context: any other call
 * that renders, traverses or trains on the context fails until the finish. */
svlf_status svlf_render_frame_device_submit(svlf_ctx* ctx, svlf_model* model, const svlf_camera* cam,
                                            const float* background, svlf_precision precision,
                                            float* d_rgb, float* d_alpha, float* d_depth);
svlf_status svlf_render_frame_device_finish(svlf_ctx* ctx, svlf_render_stats* stats);
/* Sub-rectangle of rows [row0, row0+rows) of the camera's image (tile
 * sharding across ranks); output buffers hold W*rows pixels. Device buffers. */
/* Tile-interleaved share of one frame (multi-GPU render of a frame, SURVEY.md
 * §8(e)): the image is cut into tile_w x tile_h tiles (both must divide the
 * image size) numbered in raster order; rank r renders tiles r, r + world,
 * r + 2 world, ... (svlf_tiles_owned of them). Output buffers hold those tiles
 * in that order, each tile_w x tile_h row-major. Device buffers; bit-identical
 * to the same pixels of a full frame. */
svlf_status svlf_render_tiles_device(svlf_ctx* ctx, svlf_model* model, const svlf_camera* cam, uint32_t tile_w,
                                     uint32_t tile_h, uint32_t rank, uint32_t world, const float* background,
                                     svlf_precision precision, float* d_rgb, float* d_alpha, float* d_depth,
                                     svlf_render_stats* stats);
size_t svlf_tiles_owned(const svlf_camera* cam, uint32_t tile_w, uint32_t tile_h, uint32_t rank, uint32_t world);
svlf_status svlf_render_rows_device(svlf_ctx* ctx, svlf_model* model, const svlf_camera* cam,
                                    uint32_t row0, uint32_t rows, const float* background,
                                    svlf_precision precision, float* d_rgb, float* d_alpha,
                                    float* d_depth, svlf_render_stats* stats);
/* Arbitrary rays (render_ray per ray, render.hpp:75), host buffers. */
svlf_status svlf_render_rays(svlf_ctx* ctx, svlf_model* model, const double* rays, size_t n,
                             const float* background, svlf_precision precision, float* rgb,
                             float* alpha, float* depth, svlf_render_stats* stats);

/* ---- train: one optimizer step over a ray batch (src/train.cpp:443-479 body:
 * loss_chunk over the batch, gradient sum, adam_model_step). Rays n x 6,
 * c_gt n x 3, depth_gt n (Euclidean, 0 = background), alpha_gt n (0/1).
 * Surface mode drops rays with no resolved surface voxel (counted as skipped).
 * loss_sum = sum of per-ray losses (the reference logs loss_sum / n). */
svlf_status svlf_train_step(svlf_ctx* ctx, svlf_model* model, const double* rays,
                            const float* c_gt, const double* depth_gt, const uint8_t* alpha_gt,
                            size_t n, svlf_loss_mode mode, int color_frozen, float lr,
                            const svlf_loss_weights* lw, svlf_loss_stats* stats,
                            double* loss_sum);
/* Same with the batch already resident in DEVICE memory (rays, c_gt,
 * depth_gt, alpha_gt are device pointers). */
svlf_status svlf_train_step_device(svlf_ctx* ctx, svlf_model* model, const double* rays,
                                   const float* c_gt, const double* depth_gt,
                                   const uint8_t* alpha_gt, size_t n, svlf_loss_mode mode,
                                   int color_frozen, float lr, const svlf_loss_weights* lw,
                                   svlf_loss_stats* stats, double* loss_sum);
/* Pipelined steps over HOST batches (the reference's per-frame loop,
 * src/train.cpp:452-479, with the next frame's upload overlapping the current
 * step). svlf_train_batch_stage queues a batch into one of the context's two
 * device input slots and returns at once: page-locked inputs are copied by
 * DMA on the context's copy stream, pageable ones through page-locked staging
 * filled by a background host thread; *slot receives the slot. The caller
 * keeps the arrays unchanged until the slot has been stepped or discarded.
 * INVALID_ARGUMENT when both slots already hold batches.
 * svlf_train_step_staged runs svlf_train_step on a staged slot (waiting for
 * its copy) and frees the slot; svlf_train_batch_discard frees it unstepped.
 * Loop: stage(0); for k: stage(k + 1); step_staged(k). */
svlf_status svlf_train_batch_stage(svlf_ctx* ctx, const double* rays, const float* c_gt,
                                   const double* depth_gt, const uint8_t* alpha_gt, size_t n,
                                   int* slot);
svlf_status svlf_train_step_staged(svlf_ctx* ctx, svlf_model* model, int slot, svlf_loss_mode mode,
                                   int color_frozen, float lr, const svlf_loss_weights* lw,
                                   svlf_loss_stats* stats, double* loss_sum);
svlf_status svlf_train_batch_discard(svlf_ctx* ctx, int slot);
/* Loss and summed gradients only (no Adam), the gradient oracle entry for
 * surface_loss / volumetric_loss summed over rays (train.hpp:60-71). */
svlf_status svlf_loss_grads(svlf_ctx* ctx, svlf_model* model, const double* rays,
                            const float* c_gt, const double* depth_gt, const uint8_t* alpha_gt,
                            size_t n, svlf_loss_mode mode, int color_frozen,
                            const svlf_loss_weights* lw, svlf_loss_stats* stats, double* loss_sum);

/* ---- ground truth, occupancy and metrics on the GPU ----
 * Analytic scene (reference include/svlf/scene.hpp:12-33): spheres n x 7
 * (center xyz, radius, albedo rgb), boxes n x 9 (lo xyz, hi xyz, albedo rgb),
 * host arrays. */
typedef struct svlf_scene_desc {
    const double* spheres;
    size_t n_spheres;
    const double* boxes;
    size_t n_boxes;
    double light_dir[3], light_rgb[3], ambient[3], background[3];
} svlf_scene_desc;

/* generate_dataset's pixel loop (src/dataset.cpp:61-83): raycast + shade per
 * pixel -> rgb W*H*3, Euclidean depth W*H (0 = background), mask W*H; device
 * buffers. Bit-exact with the reference built without FMA contraction. */
svlf_status svlf_render_gt_device(svlf_ctx* ctx, const svlf_scene_desc* scene, const svlf_camera* cam,
                                  float* d_rgb, float* d_depth, float* d_mask);
/* train()'s occupancy points (src/train.cpp:376-386): foreground pixels of a
 * depth map -> ray.at(double(depth)), appended in unspecified order; *n_out =
 * points produced (SVLF_ERR_CAPACITY when above capacity). */
svlf_status svlf_backproject_device(svlf_ctx* ctx, const svlf_camera* cam, const float* d_depth, double* d_points,
                                    size_t capacity, size_t* n_out);
/* psnr (src/metrics.cpp:57-68) over n values (any channel count). */
svlf_status svlf_psnr_device(svlf_ctx* ctx, const float* d_pred, const float* d_gt, size_t n_values,
                             double* psnr);
/* ssim (src/metrics.cpp:70-113): per-channel 11x11 Gaussian (sigma 1.5)
 * windowed SSIM over the valid region, K1 = 0.01, K2 = 0.03, dynamic range 1,
 * averaged over pixels and channels; images interleaved W*H*channels floats.
 * SVLF_ERR_INVALID_ARGUMENT ("image smaller than the SSIM window") when W or
 * H < 11. */
svlf_status svlf_ssim_device(svlf_ctx* ctx, const float* d_pred, const float* d_gt, uint32_t width, uint32_t height,
                             uint32_t channels, double* ssim);
/* depth_errors (src/metrics.cpp:115-136): RMSE / MAE over pixels with gt
 * mask >= 0.5; empty mask -> (0, 0) and *empty_mask = 1. */
svlf_status svlf_depth_errors_device(svlf_ctx* ctx, const float* d_pred_depth, const float* d_gt_depth,
                                     const float* d_gt_mask, size_t n_px, double* rmse, double* mae,
                                     int* empty_mask);

#ifdef __cplusplus
}
#endif
#endif /* SVLF_B200_H */
