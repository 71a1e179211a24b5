// C ABI implementation (include/svlf_b200.h): contexts, device mirrors of
// octrees and models, and the render / traversal / train pipelines.
#include <algorithm>
#include <functional>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <future>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "device.cuh"
#include "host_octree.hpp"
#include "host_pool.hpp"
#include "host_rng.hpp"
#include "nccl_dyn.hpp"

#include "train.cuh"

namespace svlfb {

std::atomic<long long> g_kernel_launches{0};
size_t pack_f32_floats();

namespace {

thread_local std::string g_last_error;

template <typename F>
svlf_status guard(F&& f) {
    try {
        f();
        return SVLF_OK;
    } catch (const SvlfError& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return SVLF_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SVLF_ERR_RUNTIME;
    }
}

void require(bool cond, const char* msg) {
    if (!cond) fail(SVLF_ERR_INVALID_ARGUMENT, msg);
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        SVLF_CUDA(cudaGetDevice(&prev));
        if (prev != dev) SVLF_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

// Data-parallel exchange over an NCCL communicator (NVLink / NVSwitch).
struct NcclCollective final : Collective {
    ncclComm_t comm = nullptr;
    ~NcclCollective() override {
        if (comm) nccl_api().CommDestroy(comm);
    }
    void allreduce(void* dev, size_t count, CollType t, CollOp op, cudaStream_t s) override {
        const ncclDataType_t dt = t == CollType::F32 ? ncclFloat32 : t == CollType::F64 ? ncclFloat64 : ncclUint8;
        nccl_check(nccl_api().AllReduce(dev, dev, count, dt, op == CollOp::Sum ? ncclSum : ncclMax, comm, s));
    }
};

// Host-staged exchange: the buffer is copied to page-locked memory, reduced in
// place by a host callback (gloo, MPI, a test harness), and copied back. Used
// where the ranks are not on NVLink peers; synchronizes the stream per call.
struct HostCollective final : Collective {
    svlf_allreduce_fn fn = nullptr;
    void* user = nullptr;
    void* stage = nullptr;
    size_t stage_bytes = 0;
    ~HostCollective() override {
        if (stage) cudaFreeHost(stage);
    }
    void allreduce(void* dev, size_t count, CollType t, CollOp op, cudaStream_t s) override {
        const size_t esz = t == CollType::F32 ? 4 : t == CollType::F64 ? 8 : 1;
        const size_t bytes = count * esz;
        if (!bytes) return;
        SVLF_CUDA(cudaStreamSynchronize(s));  // the previous call's copy-back has landed
        if (bytes > stage_bytes) {
            if (stage) SVLF_CUDA(cudaFreeHost(stage));
            stage = nullptr;
            stage_bytes = 0;
            SVLF_CUDA(cudaMallocHost(&stage, bytes));
            stage_bytes = bytes;
        }
        SVLF_CUDA(cudaMemcpyAsync(stage, dev, bytes, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        const svlf_dtype dt = t == CollType::F32 ? SVLF_DTYPE_F32 : t == CollType::F64 ? SVLF_DTYPE_F64 : SVLF_DTYPE_U8;
        const int rc = fn(user, stage, count, dt, op == CollOp::Sum ? SVLF_REDUCE_SUM : SVLF_REDUCE_MAX);
        if (rc != 0) fail(SVLF_ERR_RUNTIME, "all-reduce callback failed");
        SVLF_CUDA(cudaMemcpyAsync(dev, stage, bytes, cudaMemcpyHostToDevice, s));
    }
};

const char* dev_error_message(int code) {
    switch (code) {
        case kErrTangentRay: return "tangent ray";
        case kErrPointNotInVoxel: return "point not in voxel";
        case kErrSurfaceOutside: return "surface point outside voxel";
        case kErrNegativeTau: return "negative optical thickness";
        case kErrUnknownVoxel: return "unknown voxel id";
        case -1: return "device error on another rank";
        default: return "device error";
    }
}

}  // namespace
}  // namespace svlfb

using namespace svlfb;

enum EvIdx { EV_START, EV_COUNT, EV_EMIT, EV_DECODE, EV_COMPOSITE, EV_BACKWARD, EV_ADAM, EV_N };

struct svlf_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;      // active stream
    cudaStream_t own_stream = nullptr;  // created with the context
    DevBuf rays, counts, offsets, scan_tmp, hit_leaf, hit_tin, hit_tout, hit_ray;
    DevBuf h_tau, h_eta, h_rgb, out_rgb, out_alpha, out_depth, misc, tmp64, tmpx12, tc_scratch, overflow;
    DevBuf csr_off, csr_leaf, csr_tin, csr_tout, csr_ray, overflow2;
    size_t hit_cap = 0;
    long long last_overflow_rays = 0;  // rays that reached the per-ray fallback walker
    long long last_dense_rays = 0;     // rays re-run by the second (16-ray) cooperative pass
    std::unique_ptr<Collective> coll;   // data-parallel exchange (optional): NCCL or host-staged
    bool train_tf32 = false;            // train-step weight-gradient GEMMs with plain TF32 operands
    bool count_node_tests = false;      // traversal variant that counts ray-box tests (diagnostics)
    int rank = 0, world = 1;
    TrainScratch train;
    int* h_pinned = nullptr;  // small pinned mailbox for counters/flags
    cudaEvent_t ev[EV_N] = {};
    // host-buffer frames: banded render, D2H on a copy stream into the caller's
    // page-locked buffers or pinned staging (then parallel host copies); two
    // frame slots so a submitted frame's copies overlap the next frame's work
    static constexpr int kMaxBands = 8;
    struct FrameSlot {
        DevBuf rgb, alpha, depth, ctr;  // device outputs; per-band counters + misc snapshot
        DevBuf pk_vals, pk_tab;         // sparse transfer: foreground pixels, per-block masks/bases
        float* h_stage = nullptr;       // dense: the frame; sparse: the foreground pixels (5 floats each)
        size_t h_stage_floats = 0;
        uint32_t* h_tab = nullptr;  // sparse: the block table, page-locked
        size_t h_tab_words = 0;
        bool sparse = false;
        uint32_t pk_copied[kMaxBands] = {};  // foreground pixels per band copied by the submit
        uint32_t* h_ctr = nullptr;  // pinned mailbox: band counters, error flag, fg count
        cudaEvent_t band_done[kMaxBands] = {}, band_copied[kMaxBands] = {};
        bool busy = false;
        uint64_t id = 0;
        // the submission
        svlf_model* m = nullptr;
        svlf_camera cam{};
        float bg[3] = {0, 0, 0};
        bool has_bg = false;
        svlf_precision prec = SVLF_PRECISION_FP32;
        float *u_rgb = nullptr, *u_alpha = nullptr, *u_depth = nullptr;
        bool direct = false;
        uint32_t n = 0, nb = 0, band_rows = 0;
    };
    FrameSlot slot[2];
    uint64_t next_frame = 1;
    uint32_t pk_hint[kMaxBands] = {};  // sparse transfer: foreground pixels per band of the last frame
    // device-buffer frame enqueued by svlf_render_frame_device_submit, not yet finished
    struct DeviceFrame {
        bool active = false;
        svlf_model* m = nullptr;
        svlf_camera cam{};
        float bg[3] = {0, 0, 0};
        bool has_bg = false;
        svlf_precision prec = SVLF_PRECISION_FP32;
        float *rgb = nullptr, *alpha = nullptr, *depth = nullptr;
        uint32_t n = 0;
    } dev_frame;
    cudaStream_t copy_stream = nullptr;
    std::unique_ptr<HostPool> pool;
    svlf_timings last{};
    std::mutex mu;  // one pipeline at a time per context
    // staged train batches (svlf_train_batch_stage / svlf_train_step_staged):
    // two device input slots, filled on the copy stream while a step runs
    struct TrainSlot {
        DevBuf rays, c_gt, depth, alpha;
        char* h_stage = nullptr;  // page-locked staging for pageable batches
        size_t h_stage_bytes = 0;
        cudaEvent_t copied = nullptr;
        std::future<void> job;  // pageable batch: host copy into h_stage, then the DMA
        size_t n = 0;
        bool staged = false;
    };
    TrainSlot tslot[2];
    int next_tslot = 0;
    std::unique_ptr<HostPool> stage_pool;  // host copies of staged batches (own pool: runs beside `pool`)
    std::mutex stage_mu;                   // one staging job on stage_pool at a time
};

// Host octree; its device mirror is uploaded lazily to the device of the
// first context that uses it (an octree built with ctx == NULL is host-only
// until then, which keeps build/load usable without a GPU).
struct svlf_octree {
    HostOctree host;
    mutable int device = -1;
    mutable DevBuf nodes, corners, leaf_codes;
    mutable DevOctree view{};
};

struct svlf_model {
    svlf_ctx* ctx = nullptr;  // must outlive the model (destroy models first)
    int device = 0;
    const svlf_octree* tree = nullptr;
    uint32_t V = 0;
    size_t n_ft = 0, n_fc = 0, n_total = 0;
    DevBuf params, grads, adam_m, adam_v, pack_f32, pack_bf16;
    uint64_t steps[14] = {};
    AdamHyper hyper[14];
    uint64_t version = 1, pack_f32_version = 0, pack_bf16_version = 0;

    float* p() const { return params.as<float>(); }
    DevModel view() const {
        return DevModel{p(), p() + n_ft, p() + n_ft + n_fc, p() + n_ft + n_fc + SVLF_DEC_T_SIZE, V};
    }
};

namespace svlfb {
namespace {

// Device mirror of `t` on the current device (uploaded on first use).
const DevOctree& dev_view(const svlf_octree* t) {
    int dev = -1;
    SVLF_CUDA(cudaGetDevice(&dev));
    if (t->device == dev) return t->view;
    for (DevBuf* b : {&t->nodes, &t->corners, &t->leaf_codes}) {
        if (b->p) SVLF_CUDA(cudaFree(b->p));
        b->p = nullptr;
        b->cap = 0;
    }
    const HostOctree& h = t->host;
    const size_t internal = h.node_first_child.size();
    uint2* nd = t->nodes.ensure<uint2>(internal);
    std::vector<uint2> packed(internal);
    for (size_t i = 0; i < internal; ++i) packed[i] = make_uint2(h.node_first_child[i], h.node_mask[i]);
    uint32_t* cr = t->corners.ensure<uint32_t>(h.corner_ids.size());
    uint64_t* lc = t->leaf_codes.ensure<uint64_t>(h.leaves().size());
    SVLF_CUDA(cudaMemcpy(nd, packed.data(), internal * sizeof(uint2), cudaMemcpyHostToDevice));
    SVLF_CUDA(cudaMemcpy(cr, h.corner_ids.data(), h.corner_ids.size() * 4, cudaMemcpyHostToDevice));
    SVLF_CUDA(cudaMemcpy(lc, h.leaves().data(), h.leaves().size() * 8, cudaMemcpyHostToDevice));
    DevOctree& v = t->view;
    v = DevOctree{};
    v.nodes = nd;
    v.corners = cr;
    v.leaf_codes = lc;
    for (int l = 0; l <= h.leaf_level + 1 && l < kMaxLevelsDev + 2; ++l) v.level_off[l] = h.level_off[l];
    const double extent = h.grid.hi[0] - h.grid.lo[0];
    for (int l = 0; l <= h.leaf_level; ++l) v.cell[l] = extent / (1u << l);  // src/octree.cpp:205
    for (int a = 0; a < 3; ++a) {
        v.lo[a] = h.grid.lo[a];
        v.hi[a] = h.grid.hi[a];
    }
    v.cell_size = h.cell_size;
    {
        int e = 0;
        v.inv_cell_pow2 = std::frexp(h.cell_size, &e) == 0.5 ? 1.0 / h.cell_size : 0.0;
    }
    v.L = h.leaf_level;
    v.res = h.grid.resolution;
    v.n_leaves = uint32_t(h.leaves().size());
    t->device = dev;
    return v;
}

DevCamera to_dev_camera(const svlf_camera& c) {
    DevCamera d;
    d.fx = c.fx;
    d.fy = c.fy;
    d.cx = c.cx;
    d.cy = c.cy;
    std::memcpy(d.m, c.camera_to_world, sizeof d.m);
    d.width = c.width;
    d.height = c.height;
    return d;
}

void ensure_pack_f32(svlf_model* m, cudaStream_t s) {
    if (m->pack_f32_version == m->version) return;
    float* pk = m->pack_f32.ensure<float>(pack_f32_floats());
    launch_pack_f32(m->view(), pk, s);
    m->pack_f32_version = m->version;
}

// Synchronizes and raises the device error flag, unless `discard` (the
// pass is being redone, e.g. after a hit-buffer overflow, so errors raised on
// its partial data are meaningless): then the flag is just cleared.
void check_device_error(svlf_ctx* ctx, bool discard = false) {
    int* flag = ctx->misc.as<int>();
    int code = 0;
    SVLF_CUDA(cudaMemcpyAsync(ctx->h_pinned, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    code = ctx->h_pinned[0];
    if (code != 0) {
        SVLF_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
        if (!discard) fail(SVLF_ERR_RUNTIME, dev_error_message(code));
    }
}

// misc buffer layout: [0] int error flag, [8] u64 fg counter, [16] u64 aux
void reset_misc(svlf_ctx* ctx) {
    if (ctx->dev_frame.active)
        fail(SVLF_ERR_INVALID_ARGUMENT, "a frame from svlf_render_frame_device_submit is pending on this context: "
                                        "call svlf_render_frame_device_finish first");
    ctx->misc.ensure<unsigned long long>(8);
    SVLF_CUDA(cudaMemsetAsync(ctx->misc.p, 0, 64, ctx->stream));
}
unsigned long long* misc_fg(svlf_ctx* ctx) { return reinterpret_cast<unsigned long long*>(ctx->misc.as<char>() + 8); }

// Traversal for `n` rays: rays are either generated from `cam` (rows
// row0 .. row0+rows) or already resident in ctx->rays. Enqueues the three
// traversal kernels (cooperative pass, dense pass over overflowed tiles,
// per-ray fallback) with no host round trip; leaves per-ray segments
// (ctx->offsets = start, ctx->counts = count) and sorted hits in ctx->hit_*,
// counters at traversal_counters(ctx): [0] hits, [1] overflow, [2] capacity
// exceeded, [3] dense overflow, [7] ray-box tests of the cooperative passes.
uint32_t* traversal_counters(svlf_ctx* ctx) { return reinterpret_cast<uint32_t*>(ctx->misc.as<char>() + 16); }

// Buffers of a traversal of n rays (grown here, never inside a graph capture).
TraverseOut prepare_traversal(svlf_ctx* ctx, uint32_t n) {
    double* rays = ctx->rays.ensure<double>(size_t(n) * 6 + 6);
    uint32_t* ray_off = ctx->offsets.ensure<uint32_t>(size_t(n) + 1);
    uint32_t* ray_cnt = ctx->counts.ensure<uint32_t>(size_t(n) + 1);
    uint32_t* ovl = ctx->overflow.ensure<uint32_t>(size_t(n) + 64);
    uint32_t* ovl2 = ctx->overflow2.ensure<uint32_t>(size_t(n) + 64);
    uint32_t* counters = traversal_counters(ctx);
    size_t cap = std::max<size_t>(ctx->hit_cap, std::max<size_t>(size_t(n) * 4, size_t(1) << 20));
    cap = std::min<size_t>(cap, 0xfffff000u);
    ctx->hit_leaf.ensure<uint32_t>(cap);
    ctx->hit_tin.ensure<double>(cap);
    ctx->hit_tout.ensure<double>(cap);
    ctx->hit_ray.ensure<uint32_t>(cap);
    ctx->hit_cap = cap;
    return TraverseOut{ray_off, ray_cnt, ctx->hit_leaf.as<uint32_t>(), ctx->hit_tin.as<double>(),
                       ctx->hit_tout.as<double>(), ctx->hit_ray.as<uint32_t>(), counters, ovl, ovl2, rays,
                       uint32_t(cap)};
}

// The traversal's launches into prepared buffers; `capturing`: inside a CUDA
// graph capture (the timing events become event-record nodes).
void launch_traversal(svlf_ctx* ctx, const svlf_octree* tree, const DevCamera* cam, uint32_t row0, uint32_t rows,
                      uint32_t n, const TraverseOut& o, bool capturing = false) {
    cudaStream_t s = ctx->stream;
    auto ev = [&](int k) {
        if (capturing) SVLF_CUDA(cudaEventRecordWithFlags(ctx->ev[k], s, cudaEventRecordExternal));
        else SVLF_CUDA(cudaEventRecord(ctx->ev[k], s));
    };
    SVLF_CUDA(cudaMemsetAsync(o.counters, 0, 32, s));  // hit/overflow counters, tile cursors, node tests
    ev(EV_START);
    launch_traverse(dev_view(tree), cam, row0, rows, n, o, s, ctx->count_node_tests);
    ev(EV_COUNT);
    launch_traverse_dense(dev_view(tree), cam, row0, o, s, ctx->count_node_tests);
    launch_traverse_fallback(dev_view(tree), cam, row0, o, s);
    ev(EV_EMIT);
}

void enqueue_traversal(svlf_ctx* ctx, const svlf_octree* tree, const DevCamera* cam, uint32_t row0, uint32_t rows,
                       uint32_t n) {
    const TraverseOut o = prepare_traversal(ctx, n);
    launch_traversal(ctx, tree, cam, row0, rows, n, o);
}

// Reads the traversal counters (synchronizes). Returns false when the hit
// buffers were too small (ctx->hit_cap has been grown; re-run the traversal).
bool read_traversal(svlf_ctx* ctx, uint32_t* total) {
    SVLF_CUDA(cudaMemcpyAsync(ctx->h_pinned + 4, traversal_counters(ctx), 16, cudaMemcpyDeviceToHost, ctx->stream));
    SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    *total = uint32_t(ctx->h_pinned[4]);
    ctx->last_overflow_rays = ctx->h_pinned[7];
    ctx->last_dense_rays = ctx->h_pinned[5];
    if (ctx->h_pinned[6] == 0) return true;
    ctx->hit_cap = size_t(*total) + *total / 4 + 1024;
    return false;
}

// Traversal with a synchronous hit count (fp32 render, API traversal, train).
uint32_t run_traversal(svlf_ctx* ctx, const svlf_octree* tree, const DevCamera* cam, uint32_t row0,
                       uint32_t rows, uint32_t n) {
    for (int attempt = 0; attempt < 3; ++attempt) {
        enqueue_traversal(ctx, tree, cam, row0, rows, n);
        uint32_t total = 0;
        if (read_traversal(ctx, &total)) return total;
    }
    fail(SVLF_ERR_RUNTIME, "traversal output capacity could not be satisfied");
}

// decode + composite into device output buffers. total_host = hit count if
// known on the host (fp32 path needs it); the tensor-core path reads the
// device-side counter.
void run_decode_composite(svlf_ctx* ctx, svlf_model* m, uint32_t n, uint32_t total_host, const float* bg,
                          svlf_precision prec, float* d_rgb, float* d_alpha, float* d_depth) {
    cudaStream_t s = ctx->stream;
    const uint32_t cap = uint32_t(ctx->hit_cap);
    HitOut ho{ctx->h_tau.ensure<float>(cap), ctx->h_eta.ensure<float>(cap), ctx->h_rgb.ensure<float>(size_t(cap) * 3)};
    const DevOctree& T = dev_view(m->tree);
    int* err = ctx->misc.as<int>();
    if (prec == SVLF_PRECISION_BF16 || prec == SVLF_PRECISION_FP16) {
        const bool bf16 = prec == SVLF_PRECISION_BF16;
        ensure_pack_tc(m->view(), T, m->pack_bf16, m->pack_bf16_version, m->version, bf16, s);
        void* scratch = ctx->tc_scratch.ensure<uint8_t>(decode_tc_scratch_bytes(cap));
        launch_decode_tc(T, m->view(), m->pack_bf16.as<char>(), bf16, ctx->rays.as<double>(),
                         ctx->hit_ray.as<uint32_t>(), ctx->hit_leaf.as<uint32_t>(), ctx->hit_tin.as<double>(),
                         ctx->hit_tout.as<double>(), traversal_counters(ctx), cap, ho, err, scratch, s);
    } else {
        if (prec != SVLF_PRECISION_FP32) fail(SVLF_ERR_INVALID_ARGUMENT, "unknown precision");
        ensure_pack_f32(m, s);
        launch_decode_f32(T, m->view(), pack_f32_view(m->pack_f32.as<float>()), ctx->rays.as<double>(),
                          ctx->hit_ray.as<uint32_t>(), ctx->hit_leaf.as<uint32_t>(),
                          ctx->hit_tin.as<double>(), ctx->hit_tout.as<double>(), total_host, ho, err, s);
    }
    SVLF_CUDA(cudaEventRecord(ctx->ev[EV_DECODE], s));
    launch_composite(ctx->offsets.as<uint32_t>(), ctx->counts.as<uint32_t>(), ctx->hit_tin.as<double>(),
                     ctx->hit_tout.as<double>(), ho, n, bg, d_rgb, d_alpha, d_depth, misc_fg(ctx), prec == SVLF_PRECISION_FP32, s);
    SVLF_CUDA(cudaEventRecord(ctx->ev[EV_COMPOSITE], s));
}

// One synchronization per frame: counters, fg count and error flag.
// Returns false if the traversal overflowed the hit buffers (re-render).
bool finish_render(svlf_ctx* ctx, uint32_t n, svlf_render_stats* stats) {
    cudaStream_t s = ctx->stream;
    SVLF_CUDA(cudaMemcpyAsync(ctx->h_pinned + 8, misc_fg(ctx), 8, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaMemcpyAsync(ctx->h_pinned + 4, traversal_counters(ctx), 16, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaStreamSynchronize(s));
    const uint32_t total = uint32_t(ctx->h_pinned[4]);
    ctx->last_overflow_rays = ctx->h_pinned[7];
    ctx->last_dense_rays = ctx->h_pinned[5];
    if (ctx->h_pinned[6] != 0) {  // hit buffers overflowed: decode saw partial lists, redo
        check_device_error(ctx, true);
        ctx->hit_cap = size_t(total) + total / 4 + 1024;
        return false;
    }
    check_device_error(ctx);
    unsigned long long fg = 0;
    std::memcpy(&fg, ctx->h_pinned + 8, 8);
    float ms[4] = {};
    cudaEventElapsedTime(&ms[0], ctx->ev[EV_START], ctx->ev[EV_COUNT]);
    cudaEventElapsedTime(&ms[1], ctx->ev[EV_COUNT], ctx->ev[EV_EMIT]);
    cudaEventElapsedTime(&ms[2], ctx->ev[EV_EMIT], ctx->ev[EV_DECODE]);
    cudaEventElapsedTime(&ms[3], ctx->ev[EV_DECODE], ctx->ev[EV_COMPOSITE]);
    ctx->last = svlf_timings{ms[0], ms[1], ms[2], ms[3], 0.f, 0.f, ms[0] + ms[1] + ms[2] + ms[3],
                             (long long)total, ctx->last_overflow_rays, ctx->last_dense_rays};
    if (stats) {
        stats->rays += n;
        stats->rays_with_hits += (long long)fg;
        stats->traversal_hits += total;
        stats->thickness_queries += total;
        stats->color_queries += total;
    }
    return true;
}

// Full frame (or row band) into device buffers: traversal, decode, composite.
void render_pipeline(svlf_ctx* ctx, svlf_model* m, const DevCamera* cam, uint32_t row0, uint32_t rows, uint32_t n,
                     const float* bg, svlf_precision prec, float* d_rgb, float* d_alpha, float* d_depth,
                     svlf_render_stats* stats) {
    for (int attempt = 0; attempt < 3; ++attempt) {
        reset_misc(ctx);
        uint32_t total = 0;
        if (prec == SVLF_PRECISION_FP32) {
            total = run_traversal(ctx, m->tree, cam, row0, rows, n);
        } else {
            enqueue_traversal(ctx, m->tree, cam, row0, rows, n);
        }
        run_decode_composite(ctx, m, n, total, bg, prec, d_rgb, d_alpha, d_depth);
        if (finish_render(ctx, n, stats)) return;
    }
    fail(SVLF_ERR_RUNTIME, "traversal output capacity could not be satisfied");
}

// Tiles of rank `rank` in a tile-interleaved split of the image across `world` ranks.
uint32_t owned_tiles(const svlf_camera& c, uint32_t tw, uint32_t th, uint32_t rank, uint32_t world) {
    const uint32_t total = (c.width / tw) * (c.height / th);
    return rank < total ? (total - 1 - rank) / world + 1 : 0;
}

void render_tiles_device(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, uint32_t tw, uint32_t th,
                         uint32_t rank, uint32_t world, const float* bg, svlf_precision prec, float* d_rgb,
                         float* d_alpha, float* d_depth, svlf_render_stats* stats) {
    require(cam != nullptr, "camera is null");
    require(tw > 0 && th > 0 && cam->width % tw == 0 && cam->height % th == 0,
            "tile size must divide the image size");
    require(world >= 1 && rank < world, "bad rank/world");
    const uint32_t k = owned_tiles(*cam, tw, th, rank, world);
    const uint64_t n64 = uint64_t(k) * tw * th;
    require(n64 < (1ull << 31), "too many pixels in one call");
    if (n64 == 0) return;
    DevCamera dc = to_dev_camera(*cam);
    dc.width = tw;  // ray index space: this rank's tiles stacked vertically
    dc.height = k * th;
    dc.tile_w = tw;
    dc.tile_h = th;
    dc.tiles_x = cam->width / tw;
    dc.tiles_rank = rank;
    dc.tiles_world = world;
    render_pipeline(ctx, m, &dc, 0, k * th, uint32_t(n64), bg, prec, d_rgb, d_alpha, d_depth, stats);
}

void render_device(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, uint32_t row0, uint32_t rows,
                   const float* bg, svlf_precision prec, float* d_rgb, float* d_alpha, float* d_depth,
                   svlf_render_stats* stats) {
    require(cam != nullptr, "camera is null");
    if (cam->width == 0 || cam->height == 0) fail(SVLF_ERR_INVALID_ARGUMENT, "zero-size image");
    require(row0 + rows <= cam->height, "row range outside the image");
    const uint64_t n64 = uint64_t(cam->width) * rows;
    require(n64 < (1ull << 31), "too many pixels in one call");
    const uint32_t n = uint32_t(n64);
    const DevCamera dc = to_dev_camera(*cam);
    render_pipeline(ctx, m, &dc, row0, rows, n, bg, prec, d_rgb, d_alpha, d_depth, stats);
}

// Frame into HOST buffers, in two phases so frames can be pipelined.
// submit: the image is rendered in `bands` row bands, all enqueued without a
// host round trip; each finished band is copied device-to-host on
// ctx->copy_stream (into the caller's buffers when they are page-locked, else
// into the slot's pinned staging) while later bands / the next frame render.
// complete: waits for the bands in order (host copies from staging overlap
// the GPU), then checks the frame's counters: a hit-buffer overflow in any
// band re-renders the frame synchronously with grown buffers (errors raised
// on the partial hit lists are discarded).
using FrameSlot = svlf_ctx::FrameSlot;

// Frame counters (FrameSlot::ctr / h_ctr): 4 traversal counters per band, the
// misc snapshot (error flag, foreground count), foreground pixels per band.
constexpr uint32_t kCtrMisc = 4 * svlf_ctx::kMaxBands, kCtrPack = kCtrMisc + 4,
                   kCtrWords = kCtrPack + svlf_ctx::kMaxBands;

// Host frames move only the foreground pixels over the host link (rays with
// hits: ~10 % of a C2 frame) plus a 36-byte table row per 256 pixels, and the
// host fills the background pixels ((bg, 0, 0) exactly, as the composite
// writes them). A dense 51 MB device-to-host copy per C2 frame otherwise runs
// beside the next frame's kernels and slows them (measured: +0.12 ms per
// frame). $SVLF_SPARSE_FRAMES=0: dense copies.
bool sparse_frames() {
    static const bool on = [] {
        const char* e = std::getenv("SVLF_SPARSE_FRAMES");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool is_pinned(const void* ptr) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

void frame_submit(svlf_ctx* ctx, FrameSlot& F, uint32_t bands) {
    const uint32_t W = F.cam.width, H = F.cam.height, n = F.n;
    const DevCamera dc = to_dev_camera(F.cam);
    cudaStream_t s = ctx->stream, c = ctx->copy_stream;
    float* d_rgb = F.rgb.ensure<float>(size_t(n) * 3);
    float* d_alpha = F.alpha.ensure<float>(n);
    float* d_depth = F.depth.ensure<float>(n);
    F.sparse = sparse_frames();
    if ((!F.direct || F.sparse) && F.h_stage_floats < size_t(n) * 5) {
        if (F.h_stage) SVLF_CUDA(cudaFreeHost(F.h_stage));
        F.h_stage = nullptr;
        SVLF_CUDA(cudaMallocHost(&F.h_stage, size_t(n) * 5 * sizeof(float)));
        F.h_stage_floats = size_t(n) * 5;
    }
    float* st_rgb = F.direct ? F.u_rgb : F.h_stage;
    float* st_alpha = F.direct ? F.u_alpha : st_rgb + size_t(n) * 3;
    float* st_depth = F.direct ? F.u_depth : st_alpha + n;
    bands = std::max<uint32_t>(1, std::min<uint32_t>({bands, uint32_t(svlf_ctx::kMaxBands), H}));
    F.band_rows = (H + bands - 1) / bands;
    uint32_t* ctr = F.ctr.ensure<uint32_t>(kCtrWords);
    const float* bg = F.has_bg ? F.bg : nullptr;
    float* pk_vals = nullptr;
    uint32_t* pk_tab = nullptr;
    if (F.sparse) {
        const size_t tab_words = 9 * (size_t(n) / kPackBlock + svlf_ctx::kMaxBands + 1);
        pk_vals = F.pk_vals.ensure<float>(size_t(n) * 5);
        pk_tab = F.pk_tab.ensure<uint32_t>(tab_words);
        if (F.h_tab_words < tab_words) {
            if (F.h_tab) SVLF_CUDA(cudaFreeHost(F.h_tab));
            F.h_tab = nullptr;
            F.h_tab_words = 0;
            SVLF_CUDA(cudaMallocHost(&F.h_tab, tab_words * 4));
            F.h_tab_words = tab_words;
        }
    }
    reset_misc(ctx);
    if (F.sparse) SVLF_CUDA(cudaMemsetAsync(ctr + kCtrPack, 0, 4 * svlf_ctx::kMaxBands, s));
    uint32_t nb = 0;
    size_t tb = 0;  // sparse: table rows of the earlier bands
    for (uint32_t r0 = 0; r0 < H; r0 += F.band_rows, ++nb) {
        const uint32_t rows = std::min(F.band_rows, H - r0);
        const size_t off = size_t(r0) * W, cnt = size_t(rows) * W;
        uint32_t total = 0;
        if (F.prec == SVLF_PRECISION_FP32) total = run_traversal(ctx, F.m->tree, &dc, r0, rows, uint32_t(cnt));
        else enqueue_traversal(ctx, F.m->tree, &dc, r0, rows, uint32_t(cnt));
        run_decode_composite(ctx, F.m, uint32_t(cnt), total, bg, F.prec, d_rgb + off * 3, d_alpha + off,
                             d_depth + off);
        SVLF_CUDA(cudaMemcpyAsync(ctr + 4 * nb, traversal_counters(ctx), 16, cudaMemcpyDeviceToDevice, s));
        if (r0 + F.band_rows >= H)  // last band: snapshot of the error flag and the foreground count
            SVLF_CUDA(cudaMemcpyAsync(ctr + 4 * svlf_ctx::kMaxBands, ctx->misc.p, 16, cudaMemcpyDeviceToDevice, s));
        const size_t rows_tab = (cnt + kPackBlock - 1) / kPackBlock;
        if (F.sparse)
            launch_pack_fg(ctx->counts.as<uint32_t>(), uint32_t(cnt), d_rgb + off * 3, d_alpha + off, d_depth + off,
                           pk_vals + 5 * off, pk_tab + 9 * tb, ctr + kCtrPack + nb, s);
        SVLF_CUDA(cudaEventRecord(F.band_done[nb], s));
        SVLF_CUDA(cudaStreamWaitEvent(c, F.band_done[nb], 0));
        if (F.sparse) {
            // the table, and as many foreground pixels as the last frame's band had (+1/8);
            // the completion copies any excess
            const uint32_t hint = ctx->pk_hint[nb];
            const uint32_t est = uint32_t(std::min<size_t>(cnt, hint ? hint : cnt / 8 + 1024));
            F.pk_copied[nb] = est;
            SVLF_CUDA(cudaMemcpyAsync(F.h_ctr + kCtrPack + nb, ctr + kCtrPack + nb, 4, cudaMemcpyDeviceToHost, c));
            SVLF_CUDA(cudaMemcpyAsync(F.h_tab + 9 * tb, pk_tab + 9 * tb, rows_tab * 36, cudaMemcpyDeviceToHost, c));
            if (est)
                SVLF_CUDA(cudaMemcpyAsync(F.h_stage + 5 * off, pk_vals + 5 * off, size_t(est) * 20,
                                          cudaMemcpyDeviceToHost, c));
        } else {
            SVLF_CUDA(cudaMemcpyAsync(st_rgb + off * 3, d_rgb + off * 3, cnt * 12, cudaMemcpyDeviceToHost, c));
            SVLF_CUDA(cudaMemcpyAsync(st_alpha + off, d_alpha + off, cnt * 4, cudaMemcpyDeviceToHost, c));
            SVLF_CUDA(cudaMemcpyAsync(st_depth + off, d_depth + off, cnt * 4, cudaMemcpyDeviceToHost, c));
        }
        tb += rows_tab;
        if (r0 + F.band_rows >= H)
            SVLF_CUDA(cudaMemcpyAsync(F.h_ctr, ctr, 4 * kCtrWords, cudaMemcpyDeviceToHost, c));
        SVLF_CUDA(cudaEventRecord(F.band_copied[nb], c));
    }
    F.nb = nb;
}

// The context's host worker pool (sparse frame expansion, pageable-batch
// staging): $SVLF_HOST_THREADS threads, else this process's share of the host
// threads (hardware threads / $LOCAL_WORLD_SIZE, at most 16): the sparse
// expansion writes the whole frame (51 MB on C2) while the GPU renders the
// next one (8 threads: 0.70 ms per C2 frame, 16: 0.43 ms).
std::unique_ptr<HostPool>& host_pool(std::unique_ptr<HostPool>& p) {
    if (!p) {
        const char* e = std::getenv("SVLF_HOST_THREADS");
        const char* lw = std::getenv("LOCAL_WORLD_SIZE");
        const int hw = int(std::thread::hardware_concurrency());
        const int share = hw / std::max(1, lw ? std::atoi(lw) : 1);
        p = std::make_unique<HostPool>(e ? std::max(0, std::atoi(e) - 1) : std::clamp(share - 1, 0, 15));
    }
    return p;
}

// Sparse transfer, host side, one band (as soon as its copies landed, while
// later bands render): copies the foreground pixels the submit did not (more
// than the estimate), then writes the band into the caller's buffers from the
// block table: foreground pixels from the packed values, background pixels
// (bg, 0, 0); the thread pool takes 64 table rows (16 K pixels) per task.
void frame_expand_band(svlf_ctx* ctx, FrameSlot& F, uint32_t b) {
    const uint32_t W = F.cam.width, H = F.cam.height;
    const size_t off = size_t(b) * F.band_rows * W, cnt = size_t(std::min(F.band_rows, H - b * F.band_rows)) * W;
    const size_t tab0 = size_t(b) * ((size_t(F.band_rows) * W + kPackBlock - 1) / kPackBlock);  // earlier bands' rows
    const size_t rows = (cnt + kPackBlock - 1) / kPackBlock;
    const uint32_t fg = F.h_ctr[kCtrPack + b];
    if (fg > F.pk_copied[b]) {
        // (blocking copy: the band's values are complete; the copy stream may already hold
        // later bands' copies waiting for their kernels)
        SVLF_CUDA(cudaMemcpy(F.h_stage + 5 * (off + F.pk_copied[b]), F.pk_vals.as<float>() + 5 * (off + F.pk_copied[b]),
                             size_t(fg - F.pk_copied[b]) * 20, cudaMemcpyDeviceToHost));
    }
    ctx->pk_hint[b] = uint32_t(std::min<size_t>(cnt, size_t(fg) + fg / 8 + 1024));
    float bg_row[3 * kPackBlock];  // a table row's worth of background rgb
    for (uint32_t i = 0; i < kPackBlock; ++i)
        for (int c = 0; c < 3; ++c) bg_row[3 * i + c] = F.bg[c];
    constexpr size_t kRows = 64;  // table rows per task
    ctx->pool->parallel_for(int((rows + kRows - 1) / kRows), [&](int t) {
        for (size_t r = size_t(t) * kRows; r < std::min(rows, size_t(t + 1) * kRows); ++r) {
            const uint32_t* row = F.h_tab + 9 * (tab0 + r);
            const size_t p0 = off + r * kPackBlock, pe = std::min(off + cnt, p0 + kPackBlock);
            const float* v = F.h_stage + 5 * (off + row[8]);
            // background everywhere (streaming fills), then the foreground pixels over it
            std::memcpy(F.u_rgb + 3 * p0, bg_row, (pe - p0) * 12);
            std::memset(F.u_alpha + p0, 0, (pe - p0) * 4);
            std::memset(F.u_depth + p0, 0, (pe - p0) * 4);
            for (uint32_t w = 0; w < kPackBlock / 32; ++w)
                for (uint32_t m = row[w]; m; m &= m - 1) {
                    const size_t p = p0 + 32 * w + uint32_t(__builtin_ctz(m));
                    F.u_rgb[3 * p] = v[0];
                    F.u_rgb[3 * p + 1] = v[1];
                    F.u_rgb[3 * p + 2] = v[2];
                    F.u_alpha[p] = v[3];
                    F.u_depth[p] = v[4];
                    v += 5;
                }
        }
    });
}

// Returns false when the frame has to be redone (hit buffers overflowed).
bool frame_complete(svlf_ctx* ctx, FrameSlot& F, svlf_render_stats* stats) {
    const uint32_t W = F.cam.width, H = F.cam.height, n = F.n;
    if (!F.direct || F.sparse) host_pool(ctx->pool);
    const float* st_rgb = F.h_stage;
    const float* st_alpha = st_rgb + size_t(n) * 3;
    const float* st_depth = st_alpha + n;
    for (uint32_t b = 0; b < F.nb; ++b) {
        SVLF_CUDA(cudaEventSynchronize(F.band_copied[b]));
        if (F.sparse) frame_expand_band(ctx, F, b);
        if (F.direct || F.sparse) continue;
        const size_t off = size_t(b) * F.band_rows * W;
        const size_t cnt = size_t(std::min(F.band_rows, H - b * F.band_rows)) * W;
        constexpr size_t kPart = 64 * 1024;  // pixels per host copy task
        const int parts = int((cnt + kPart - 1) / kPart);
        ctx->pool->parallel_for(parts, [&](int i) {
            const size_t p0 = off + size_t(i) * kPart, pc = std::min(kPart, off + cnt - p0);
            std::memcpy(F.u_rgb + p0 * 3, st_rgb + p0 * 3, pc * 12);
            std::memcpy(F.u_alpha + p0, st_alpha + p0, pc * 4);
            std::memcpy(F.u_depth + p0, st_depth + p0, pc * 4);
        });
    }
    uint64_t total = 0, dense = 0, fallback = 0, worst = 0;
    bool overflow = false;
    for (uint32_t b = 0; b < F.nb; ++b) {
        const uint32_t* c = F.h_ctr + 4 * b;
        total += c[0];
        dense += c[1];
        overflow |= c[2] != 0;
        fallback += c[3];
        worst = std::max<uint64_t>(worst, c[0]);
    }
    const uint32_t* snap = F.h_ctr + kCtrMisc;
    const int err = int(snap[0]);
    unsigned long long fg = 0;
    std::memcpy(&fg, snap + 2, 8);
    ctx->last_overflow_rays = (long long)fallback;
    ctx->last_dense_rays = (long long)dense;
    if (overflow) {
        ctx->hit_cap = std::max(ctx->hit_cap, size_t(worst) + worst / 4 + 1024);
        return false;
    }
    if (err) fail(SVLF_ERR_RUNTIME, dev_error_message(err));
    float ms[4] = {};  // last band's stage times
    cudaEventElapsedTime(&ms[0], ctx->ev[EV_START], ctx->ev[EV_COUNT]);
    cudaEventElapsedTime(&ms[1], ctx->ev[EV_COUNT], ctx->ev[EV_EMIT]);
    cudaEventElapsedTime(&ms[2], ctx->ev[EV_EMIT], ctx->ev[EV_DECODE]);
    cudaEventElapsedTime(&ms[3], ctx->ev[EV_DECODE], ctx->ev[EV_COMPOSITE]);
    cudaGetLastError();
    ctx->last = svlf_timings{ms[0], ms[1], ms[2], ms[3], 0.f, 0.f, ms[0] + ms[1] + ms[2] + ms[3],
                             (long long)total, ctx->last_overflow_rays, ctx->last_dense_rays};
    if (stats) {
        stats->rays += n;
        stats->rays_with_hits += (long long)fg;
        stats->traversal_hits += (long long)total;
        stats->thickness_queries += (long long)total;
        stats->color_queries += (long long)total;
    }
    return true;
}

uint32_t default_bands(uint32_t n) {
    // ~700K rays per band for a synchronous frame (fewer bands: less per-band
    // launch/tail cost; more: shorter exposed copy of the last band)
    static const uint32_t band_rays = [] {
        const char* e = std::getenv("SVLF_BAND_RAYS");
        return e ? uint32_t(std::max(1, std::atoi(e))) : 700000u;  // measured best for C2 (3 bands)
    }();
    return std::max<uint32_t>(1, n / band_rays);
}

FrameSlot& frame_setup(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, const float* bg, svlf_precision prec,
                       float* rgb, float* alpha, float* depth) {
    require(cam != nullptr, "camera is null");
    if (cam->width == 0 || cam->height == 0) fail(SVLF_ERR_INVALID_ARGUMENT, "zero-size image");
    const uint64_t n64 = uint64_t(cam->width) * cam->height;
    require(n64 < (1ull << 31), "too many pixels in one call");
    if (prec != SVLF_PRECISION_FP32 && prec != SVLF_PRECISION_FP16 && prec != SVLF_PRECISION_BF16)
        fail(SVLF_ERR_INVALID_ARGUMENT, "unknown precision");
    FrameSlot* F = !ctx->slot[0].busy ? &ctx->slot[0] : (!ctx->slot[1].busy ? &ctx->slot[1] : nullptr);
    if (!F) fail(SVLF_ERR_INVALID_ARGUMENT, "two frames already in flight on this context");
    F->m = m;
    F->cam = *cam;
    F->has_bg = bg != nullptr;
    for (int i = 0; i < 3; ++i) F->bg[i] = bg ? bg[i] : 0.f;
    F->prec = prec;
    F->u_rgb = rgb;
    F->u_alpha = alpha;
    F->u_depth = depth;
    F->direct = is_pinned(rgb) && is_pinned(alpha) && is_pinned(depth);
    F->n = uint32_t(n64);
    F->id = ctx->next_frame++;
    return *F;
}

// Completes F, redoing it synchronously after a hit-buffer overflow.
void frame_finish(svlf_ctx* ctx, FrameSlot& F, svlf_render_stats* stats) {
    struct Release {
        FrameSlot& f;
        ~Release() { f.busy = false; }
    } release{F};
    for (int attempt = 0; attempt < 3; ++attempt) {
        if (frame_complete(ctx, F, stats)) return;
        frame_submit(ctx, F, default_bands(F.n));
    }
    fail(SVLF_ERR_RUNTIME, "traversal output capacity could not be satisfied");
}

void render_frame_host(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, const float* bg, svlf_precision prec,
                       float* rgb, float* alpha, float* depth, svlf_render_stats* stats) {
    FrameSlot& F = frame_setup(ctx, m, cam, bg, prec, rgb, alpha, depth);
    F.busy = true;
    try {
        frame_submit(ctx, F, default_bands(F.n));
    } catch (...) {
        F.busy = false;
        throw;
    }
    frame_finish(ctx, F, stats);
}

size_t model_param_count(uint32_t V) { return size_t(V) * 96 + SVLF_DEC_T_SIZE + SVLF_DEC_C_SIZE; }

}  // namespace
}  // namespace svlfb

// ============================================================================
extern "C" {

const char* svlf_last_error(void) { return g_last_error.c_str(); }
int svlf_abi_version(void) { return SVLF_ABI_VERSION; }
long long svlf_ctx_kernel_launches(const svlf_ctx*) { return g_kernel_launches.load(); }

svlf_status svlf_ctx_create(int device, svlf_ctx** out) {
    return guard([&] {
        require(out != nullptr, "out is null");
        int count = 0;
        const cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            fail(SVLF_ERR_CUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
        require(device >= 0 && device < count, "device ordinal out of range");
        auto ctx = std::make_unique<svlf_ctx>();
        ctx->device = device;
        DeviceGuard g(device);
        SVLF_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        ctx->stream = ctx->own_stream;
        SVLF_CUDA(cudaMallocHost(&ctx->h_pinned, 256));
        for (auto& e2 : ctx->ev) SVLF_CUDA(cudaEventCreate(&e2));
        SVLF_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (auto& fs : ctx->slot) {
            for (int b = 0; b < svlf_ctx::kMaxBands; ++b) {
                SVLF_CUDA(cudaEventCreateWithFlags(&fs.band_done[b], cudaEventDisableTiming));
                SVLF_CUDA(cudaEventCreateWithFlags(&fs.band_copied[b], cudaEventDisableTiming));
            }
            SVLF_CUDA(cudaMallocHost(&fs.h_ctr, 4 * kCtrWords));
        }
        for (auto& ts : ctx->tslot) SVLF_CUDA(cudaEventCreateWithFlags(&ts.copied, cudaEventDisableTiming));
        ctx->misc.ensure<unsigned long long>(8);
        SVLF_CUDA(cudaMemset(ctx->misc.p, 0, 64));
        *out = ctx.release();
    });
}

svlf_status svlf_ctx_destroy(svlf_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        {
            DeviceGuard g(ctx->device);
            cudaStreamSynchronize(ctx->stream);
            ctx->coll.reset();
            cudaStreamSynchronize(ctx->copy_stream);
            for (auto& e : ctx->ev) cudaEventDestroy(e);
            for (auto& fs : ctx->slot) {
                for (int b = 0; b < svlf_ctx::kMaxBands; ++b) {
                    cudaEventDestroy(fs.band_done[b]);
                    cudaEventDestroy(fs.band_copied[b]);
                }
                if (fs.h_stage) cudaFreeHost(fs.h_stage);
                if (fs.h_tab) cudaFreeHost(fs.h_tab);
                if (fs.h_ctr) cudaFreeHost(fs.h_ctr);
            }
            for (auto& ts : ctx->tslot) {
                if (ts.job.valid()) ts.job.wait();
                cudaEventDestroy(ts.copied);
                if (ts.h_stage) cudaFreeHost(ts.h_stage);
            }
            cudaStreamSynchronize(ctx->copy_stream);
            if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
            cudaStreamDestroy(ctx->copy_stream);
            cudaStreamDestroy(ctx->own_stream);
        }
        delete ctx;
    });
}

// ---- ground truth / occupancy / metrics (scene.cu) ---------------------------
svlf_status svlf_render_gt_device(svlf_ctx* ctx, const svlf_scene_desc* scene, const svlf_camera* cam, float* d_rgb,
                                  float* d_depth, float* d_mask) {
    return guard([&] {
        require(ctx && scene && cam && d_rgb && d_depth && d_mask, "null argument");
        require(scene->n_spheres == 0 || scene->spheres, "spheres is null");
        require(scene->n_boxes == 0 || scene->boxes, "boxes is null");
        if (cam->width == 0 || cam->height == 0) fail(SVLF_ERR_INVALID_ARGUMENT, "zero-size image");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        cudaStream_t s = ctx->stream;
        double* prims = ctx->tmp64.ensure<double>(scene->n_spheres * 7 + scene->n_boxes * 9 + 1);
        if (scene->n_spheres)
            SVLF_CUDA(cudaMemcpyAsync(prims, scene->spheres, scene->n_spheres * 56, cudaMemcpyHostToDevice, s));
        if (scene->n_boxes)
            SVLF_CUDA(cudaMemcpyAsync(prims + scene->n_spheres * 7, scene->boxes, scene->n_boxes * 72,
                                      cudaMemcpyHostToDevice, s));
        launch_render_gt(*scene, prims, prims + scene->n_spheres * 7, to_dev_camera(*cam), d_rgb, d_depth, d_mask, s);
        SVLF_CUDA(cudaStreamSynchronize(s));  // the primitive upload buffer is reused by the next call
    });
}

svlf_status svlf_backproject_device(svlf_ctx* ctx, const svlf_camera* cam, const float* d_depth, double* d_points,
                                    size_t capacity, size_t* n_out) {
    return guard([&] {
        require(ctx && cam && d_depth && n_out, "null argument");
        require(d_points != nullptr || capacity == 0, "points is null");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        cudaStream_t s = ctx->stream;
        unsigned long long* cnt = ctx->tmpx12.ensure<unsigned long long>(1);
        SVLF_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
        launch_backproject(to_dev_camera(*cam), d_depth, d_points, capacity, cnt, s);
        SVLF_CUDA(cudaMemcpyAsync(ctx->h_pinned, cnt, 8, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        unsigned long long k = 0;
        std::memcpy(&k, ctx->h_pinned, 8);
        *n_out = size_t(k);
        if (k > capacity) fail(SVLF_ERR_CAPACITY, "back-projected points exceed the capacity");
    });
}

svlf_status svlf_psnr_device(svlf_ctx* ctx, const float* d_pred, const float* d_gt, size_t n, double* psnr) {
    return guard([&] {
        require(ctx && d_pred && d_gt && psnr, "null argument");
        if (n == 0) fail(SVLF_ERR_INVALID_ARGUMENT, "empty image");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        std::vector<double> h(reduction_partials());
        const double se = device_sq_err(d_pred, d_gt, n, ctx->tmp64.ensure<double>(reduction_partials()), h.data(),
                                        ctx->stream);
        const double mse = se / double(n);
        *psnr = mse == 0.0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / mse));
    });
}

svlf_status svlf_ssim_device(svlf_ctx* ctx, const float* d_pred, const float* d_gt, uint32_t w, uint32_t h,
                             uint32_t channels, double* ssim) {
    return guard([&] {
        require(ctx && d_pred && d_gt && ssim, "null argument");
        if (w < 11 || h < 11) fail(SVLF_ERR_INVALID_ARGUMENT, "image smaller than the SSIM window");
        if (channels == 0) fail(SVLF_ERR_INVALID_ARGUMENT, "channels must be > 0");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        std::vector<double> hp(reduction_partials());
        DevBuf tmp;
        double* t = tmp.ensure<double>(ssim_scratch_doubles(w, h));
        *ssim = device_ssim(d_pred, d_gt, w, h, channels, t, ctx->tmp64.ensure<double>(reduction_partials()),
                            hp.data(), ctx->stream);
    });
}

svlf_status svlf_depth_errors_device(svlf_ctx* ctx, const float* pd, const float* gd, const float* gm, size_t n,
                                     double* rmse, double* mae, int* empty) {
    return guard([&] {
        require(ctx && pd && gd && gm && rmse && mae, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        std::vector<double> h(reduction_partials());
        double s2 = 0, s1 = 0, c = 0;
        device_depth_err(pd, gd, gm, n, ctx->tmp64.ensure<double>(reduction_partials()), h.data(), &s2, &s1, &c,
                         ctx->stream);
        if (empty) *empty = c == 0.0;
        *rmse = c > 0 ? std::sqrt(s2 / c) : 0.0;
        *mae = c > 0 ? s1 / c : 0.0;
    });
}

svlf_status svlf_host_alloc(size_t bytes, void** out) {
    return guard([&] {
        require(out != nullptr, "out is null");
        *out = nullptr;
        if (bytes) SVLF_CUDA(cudaMallocHost(out, bytes));
    });
}

svlf_status svlf_host_free(void* p) {
    return guard([&] {
        if (p) SVLF_CUDA(cudaFreeHost(p));
    });
}

svlf_status svlf_nccl_unique_id(void* out128) {
    return guard([&] {
        require(out128 != nullptr, "out is null");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId id;
        nccl_check(nccl_api().GetUniqueId(&id));
        std::memcpy(out128, &id, sizeof id);
    });
}

svlf_status svlf_ctx_attach_nccl(svlf_ctx* ctx, const void* id128, int rank, int world) {
    return guard([&] {
        require(ctx && id128, "null argument");
        require(world >= 1 && rank >= 0 && rank < world, "bad rank/world");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->coll.reset();
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof id);
        auto c = std::make_unique<NcclCollective>();
        nccl_check(nccl_api().CommInitRank(&c->comm, world, id, rank));
        c->rank = rank;
        c->world = world;
        ctx->coll = std::move(c);
        ctx->rank = rank;
        ctx->world = world;
    });
}

svlf_status svlf_ctx_attach_collective(svlf_ctx* ctx, svlf_allreduce_fn fn, void* user, int rank, int world) {
    return guard([&] {
        require(ctx && fn, "null argument");
        require(world >= 1 && rank >= 0 && rank < world, "bad rank/world");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->coll.reset();
        auto c = std::make_unique<HostCollective>();
        c->fn = fn;
        c->user = user;
        c->rank = rank;
        c->world = world;
        ctx->coll = std::move(c);
        ctx->rank = rank;
        ctx->world = world;
    });
}

svlf_status svlf_ctx_detach_nccl(svlf_ctx* ctx) {
    return guard([&] {
        require(ctx != nullptr, "ctx is null");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->coll.reset();
        ctx->rank = 0;
        ctx->world = 1;
    });
}

svlf_status svlf_ctx_set_stream(svlf_ctx* ctx, void* stream) {
    return guard([&] {
        require(ctx != nullptr, "ctx is null");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    });
}

svlf_status svlf_ctx_set_train_precision(svlf_ctx* ctx, svlf_precision precision) {
    return guard([&] {
        require(ctx != nullptr, "null argument");
        if (precision != SVLF_PRECISION_FP32 && precision != SVLF_PRECISION_TF32 &&
            precision != SVLF_PRECISION_TF32X3)
            fail(SVLF_ERR_INVALID_ARGUMENT, "train precision must be fp32, tf32x3 or tf32");
        std::lock_guard<std::mutex> lk(ctx->mu);
        ctx->train_tf32 = precision == SVLF_PRECISION_TF32;
    });
}

svlf_status svlf_ctx_set_node_test_counting(svlf_ctx* ctx, int enable) {
    return guard([&] {
        require(ctx != nullptr, "null argument");
        std::lock_guard<std::mutex> lk(ctx->mu);
        ctx->count_node_tests = enable != 0;
    });
}

svlf_status svlf_ctx_last_node_tests(svlf_ctx* ctx, long long* out) {
    return guard([&] {
        require(ctx && out, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        uint32_t v = 0;
        if (ctx->misc.p) {
            SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
            SVLF_CUDA(cudaMemcpy(&v, traversal_counters(ctx) + 7, 4, cudaMemcpyDeviceToHost));
        }
        *out = (long long)v;
    });
}

svlf_status svlf_ctx_synchronize(svlf_ctx* ctx) {
    return guard([&] {
        require(ctx != nullptr, "ctx is null");
        DeviceGuard g(ctx->device);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

svlf_status svlf_ctx_last_timings(const svlf_ctx* ctx, svlf_timings* out) {
    return guard([&] {
        require(ctx && out, "null argument");
        *out = ctx->last;
    });
}

// ---- octree -----------------------------------------------------------------
static svlf_status make_octree(svlf_ctx* ctx, HostOctree&& h, svlf_octree** out) {
    return guard([&] {
        auto t = std::make_unique<svlf_octree>();
        t->host = std::move(h);
        if (ctx) {
            DeviceGuard g(ctx->device);
            dev_view(t.get());
        }
        *out = t.release();
    });
}

svlf_status svlf_octree_build(svlf_ctx* ctx, const svlf_grid* grid, const double* pts, size_t n,
                              svlf_octree** out) {
    HostOctree h;
    const svlf_status st = guard([&] {
        require(grid && out, "null argument");
        require(pts != nullptr || n == 0, "points is null");
        if (!ctx) {  // host-only build (no device needed)
            h = HostOctree::build(std::span<const double>(pts, pts ? 3 * n : 0), *grid);
            return;
        }
        validate_grid(*grid);
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        DevBuf d;
        double* dp = d.ensure<double>(std::max<size_t>(3 * n, 1));
        if (n) SVLF_CUDA(cudaMemcpyAsync(dp, pts, 3 * n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        h = build_octree_gpu(*grid, dp, n, ctx->stream);
    });
    if (st != SVLF_OK) return st;
    return make_octree(ctx, std::move(h), out);
}

svlf_status svlf_octree_build_device(svlf_ctx* ctx, const svlf_grid* grid, const double* d_points, size_t n,
                                     svlf_octree** out) {
    HostOctree h;
    const svlf_status st = guard([&] {
        require(ctx && grid && out, "null argument");
        require(d_points != nullptr || n == 0, "points is null");
        validate_grid(*grid);
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        h = build_octree_gpu(*grid, d_points, n, ctx->stream);
    });
    if (st != SVLF_OK) return st;
    return make_octree(ctx, std::move(h), out);
}

svlf_status svlf_octree_from_leaves(svlf_ctx* ctx, const svlf_grid* grid, const uint64_t* codes, size_t n,
                                    svlf_octree** out) {
    HostOctree h;
    const svlf_status st = guard([&] {
        require(grid && out, "null argument");
        require(codes != nullptr || n == 0, "codes is null");
        h = HostOctree::from_leaves(std::vector<uint64_t>(codes, codes + n), *grid);
    });
    if (st != SVLF_OK) return st;
    return make_octree(ctx, std::move(h), out);
}

svlf_status svlf_octree_destroy(svlf_octree* t) {
    return guard([&] {
        if (!t) return;
        if (t->device >= 0) {
            DeviceGuard g(t->device);
            delete t;
        } else {
            delete t;
        }
    });
}

svlf_status svlf_octree_get_info(const svlf_octree* t, svlf_octree_info* out) {
    return guard([&] {
        require(t && out, "null argument");
        *out = svlf_octree_info{};
        out->leaf_level = t->host.leaf_level;
        out->vertex_count = t->host.vertex_count;
        out->leaf_count = t->host.leaves().size();
        out->dropped_points = t->host.dropped_points;
        out->cell_size = t->host.cell_size;
        for (int l = 0; l <= t->host.leaf_level; ++l) out->level_size[l] = t->host.levels[l].size();
    });
}

svlf_status svlf_octree_level_codes(const svlf_octree* t, int level, uint64_t* out) {
    return guard([&] {
        require(t && out, "null argument");
        require(level >= 0 && level <= t->host.leaf_level, "level out of range");
        const auto& v = t->host.levels[level];
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

svlf_status svlf_octree_corner_ids(const svlf_octree* t, uint32_t* out) {
    return guard([&] {
        require(t && out, "null argument");
        std::memcpy(out, t->host.corner_ids.data(), t->host.corner_ids.size() * 4);
    });
}

// ---- traversal --------------------------------------------------------------
svlf_status svlf_traverse(svlf_ctx* ctx, const svlf_octree* tree, const double* rays, size_t n,
                          uint64_t* offsets, size_t capacity, uint64_t* voxel_ids, double* t_in,
                          double* t_out, double* x12, size_t* total) {
    return guard([&] {
        require(ctx && tree && offsets && total, "null argument");
        require(rays != nullptr || n == 0, "rays is null");
        require(n < (1ull << 31), "too many rays");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        cudaStream_t s = ctx->stream;
        const uint32_t nn = uint32_t(n);
        reset_misc(ctx);
        double* d_rays = ctx->rays.ensure<double>(size_t(nn) * 6 + 6);
        if (nn) SVLF_CUDA(cudaMemcpyAsync(d_rays, rays, size_t(nn) * 48, cudaMemcpyHostToDevice, s));
        const uint32_t tot = nn ? run_traversal(ctx, tree, nullptr, 0, 0, nn) : 0;
        *total = tot;
        // CSR (ray order) view: row pointer = exclusive scan of per-ray counts
        std::vector<uint32_t> off32(size_t(nn) + 1, 0);
        if (nn) {
            uint32_t* cnt = ctx->counts.as<uint32_t>();
            uint32_t* csr = ctx->csr_off.ensure<uint32_t>(size_t(nn) + 1);
            SVLF_CUDA(cudaMemsetAsync(cnt + nn, 0, 4, s));
            const size_t tb = scan_temp_bytes(nn + 1);
            launch_exclusive_scan(ctx->scan_tmp.ensure<char>(tb), tb, cnt, csr, nn + 1, s);
            SVLF_CUDA(cudaMemcpyAsync(off32.data(), csr, (size_t(nn) + 1) * 4, cudaMemcpyDeviceToHost, s));
            if (tot <= capacity && tot > 0) {
                require(voxel_ids && t_in && t_out, "hit output is null");
                uint32_t* lf = ctx->csr_leaf.ensure<uint32_t>(tot);
                double* ti = ctx->csr_tin.ensure<double>(tot);
                double* to = ctx->csr_tout.ensure<double>(tot);
                uint32_t* ry = ctx->csr_ray.ensure<uint32_t>(tot);
                launch_to_csr(ctx->offsets.as<uint32_t>(), cnt, csr, nn, ctx->hit_leaf.as<uint32_t>(),
                              ctx->hit_tin.as<double>(), ctx->hit_tout.as<double>(), lf, ti, to, ry, s);
                uint64_t* codes = ctx->tmp64.ensure<uint64_t>(tot);
                launch_gather_leaf_codes(dev_view(tree).leaf_codes, lf, codes, tot, s);
                SVLF_CUDA(cudaMemcpyAsync(voxel_ids, codes, size_t(tot) * 8, cudaMemcpyDeviceToHost, s));
                SVLF_CUDA(cudaMemcpyAsync(t_in, ti, size_t(tot) * 8, cudaMemcpyDeviceToHost, s));
                SVLF_CUDA(cudaMemcpyAsync(t_out, to, size_t(tot) * 8, cudaMemcpyDeviceToHost, s));
                if (x12) {
                    double* dx = ctx->tmpx12.ensure<double>(size_t(tot) * 6);
                    launch_hit_points(d_rays, ry, ti, to, dx, tot, s);
                    SVLF_CUDA(cudaMemcpyAsync(x12, dx, size_t(tot) * 48, cudaMemcpyDeviceToHost, s));
                }
            }
        }
        SVLF_CUDA(cudaStreamSynchronize(s));
        for (size_t i = 0; i <= n; ++i) offsets[i] = off32[i];
        ctx->last = svlf_timings{};  // the traversal's pass counts (diagnostics)
        ctx->last.hits = tot;
        ctx->last.overflow_rays = ctx->last_overflow_rays;
        ctx->last.dense_rays = ctx->last_dense_rays;
        if (tot > capacity) fail(SVLF_ERR_CAPACITY, "hit capacity too small");
    });
}

// ---- model --------------------------------------------------------------------
svlf_status svlf_model_create(svlf_ctx* ctx, const svlf_octree* tree, svlf_model** out) {
    return guard([&] {
        require(ctx && tree && out, "null argument");
        DeviceGuard g(ctx->device);
        auto m = std::make_unique<svlf_model>();
        m->ctx = ctx;
        m->device = ctx->device;
        m->tree = tree;
        m->V = tree->host.vertex_count;
        m->n_ft = size_t(m->V) * SVLF_FEAT_T_DIM;
        m->n_fc = size_t(m->V) * SVLF_FEAT_C_DIM;
        m->n_total = model_param_count(m->V);
        std::lock_guard<std::mutex> lk(ctx->mu);
        for (DevBuf* b : {&m->params, &m->grads, &m->adam_m, &m->adam_v}) {
            b->ensure<float>(m->n_total);
            SVLF_CUDA(cudaMemsetAsync(b->p, 0, m->n_total * 4, ctx->stream));
        }
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = m.release();
    });
}

svlf_status svlf_model_destroy(svlf_model* m) {
    return guard([&] {
        if (!m) return;
        DeviceGuard g(m->device);
        delete m;
    });
}

size_t svlf_model_param_count(const svlf_model* m) { return m ? m->n_total : 0; }

svlf_status svlf_model_init(svlf_model* m, uint64_t seed) {
    return guard([&] {
        require(m != nullptr, "model is null");
        // init_model, src/model.cpp:15-28; init_features features.cpp:10-19;
        // MlpParams::init mlp.cpp:40-56
        std::vector<float> host(m->n_total);
        const HostRng root(seed);
        auto features = [&](float* dst, size_t count, uint32_t dim, uint64_t s) {
            const double bound = 1.0 / std::sqrt(double(dim));
            HostRng r(s);
            for (size_t i = 0; i < count; ++i) dst[i] = float(r.uniform(-bound, bound));
        };
        auto mlp = [&](float* dst, const uint32_t* dims, int layers, uint64_t s) {
            HostRng r(s);
            size_t o = 0;
            for (int l = 0; l < layers; ++l) {
                const uint32_t in = dims[l], outd = dims[l + 1];
                const double bound = std::sqrt(6.0 / (in + outd));
                for (size_t i = 0; i < size_t(in) * outd; ++i) dst[o++] = float(r.uniform(-bound, bound));
                for (uint32_t i = 0; i < outd; ++i) dst[o++] = 0.f;
            }
        };
        static const uint32_t dt[3] = {134, 128, 2}, dc[5] = {38, 128, 128, 128, 3};
        features(host.data(), m->n_ft, SVLF_FEAT_T_DIM, root.sub(kStreamFeatT).next_u64());
        features(host.data() + m->n_ft, m->n_fc, SVLF_FEAT_C_DIM, root.sub(kStreamFeatC).next_u64());
        mlp(host.data() + m->n_ft + m->n_fc, dt, 2, root.sub(kStreamDecT).next_u64());
        mlp(host.data() + m->n_ft + m->n_fc + SVLF_DEC_T_SIZE, dc, 4, root.sub(kStreamDecC).next_u64());
        DeviceGuard g(m->ctx->device);
        std::lock_guard<std::mutex> lk(m->ctx->mu);
        cudaStream_t s = m->ctx->stream;
        SVLF_CUDA(cudaMemcpyAsync(m->params.p, host.data(), m->n_total * 4, cudaMemcpyHostToDevice, s));
        for (DevBuf* b : {&m->grads, &m->adam_m, &m->adam_v}) SVLF_CUDA(cudaMemsetAsync(b->p, 0, m->n_total * 4, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        std::fill(std::begin(m->steps), std::end(m->steps), 0);
        std::fill(std::begin(m->hyper), std::end(m->hyper), AdamHyper{});
        ++m->version;
    });
}

// Host <-> device copies of a model's tensors, ordered on the context stream
// after any enqueued work that uses them (frames in flight, train steps) and
// complete on return. The caller holds ctx->mu.
static void copy_params(svlf_model* m, DevBuf& buf, float* ft, float* fc, float* dt, float* dc, bool to_dev,
                        const float* sft = nullptr, const float* sfc = nullptr, const float* sdt = nullptr,
                        const float* sdc = nullptr) {
    DeviceGuard g(m->ctx->device);
    cudaStream_t s = m->ctx->stream;
    float* base = buf.as<float>();
    const size_t sizes[4] = {m->n_ft, m->n_fc, SVLF_DEC_T_SIZE, SVLF_DEC_C_SIZE};
    size_t off = 0;
    for (int i = 0; i < 4; ++i) {
        if (to_dev) {
            const float* src = i == 0 ? sft : i == 1 ? sfc : i == 2 ? sdt : sdc;
            if (src) SVLF_CUDA(cudaMemcpyAsync(base + off, src, sizes[i] * 4, cudaMemcpyHostToDevice, s));
        } else {
            float* dst = i == 0 ? ft : i == 1 ? fc : i == 2 ? dt : dc;
            if (dst) SVLF_CUDA(cudaMemcpyAsync(dst, base + off, sizes[i] * 4, cudaMemcpyDeviceToHost, s));
        }
        off += sizes[i];
    }
    SVLF_CUDA(cudaStreamSynchronize(s));
}

svlf_status svlf_model_set_params(svlf_model* m, const float* ft, const float* fc, const float* dt,
                                  const float* dc) {
    return guard([&] {
        require(m != nullptr, "model is null");
        std::lock_guard<std::mutex> lk(m->ctx->mu);
        copy_params(m, m->params, nullptr, nullptr, nullptr, nullptr, true, ft, fc, dt, dc);
        ++m->version;
    });
}

svlf_status svlf_model_get_params(svlf_model* m, float* ft, float* fc, float* dt, float* dc) {
    return guard([&] {
        require(m != nullptr, "model is null");
        std::lock_guard<std::mutex> lk(m->ctx->mu);
        copy_params(m, m->params, ft, fc, dt, dc, false);
    });
}

svlf_status svlf_model_get_grads(svlf_model* m, float* ft, float* fc, float* dt, float* dc) {
    return guard([&] {
        require(m != nullptr, "model is null");
        std::lock_guard<std::mutex> lk(m->ctx->mu);
        copy_params(m, m->grads, ft, fc, dt, dc, false);
    });
}

svlf_status svlf_model_get_adam(svlf_model* m, float* m_all, float* v_all, uint64_t* steps) {
    return guard([&] {
        require(m != nullptr, "model is null");
        DeviceGuard g(m->ctx->device);
        std::lock_guard<std::mutex> lk(m->ctx->mu);
        cudaStream_t s = m->ctx->stream;
        if (m_all) SVLF_CUDA(cudaMemcpyAsync(m_all, m->adam_m.p, m->n_total * 4, cudaMemcpyDeviceToHost, s));
        if (v_all) SVLF_CUDA(cudaMemcpyAsync(v_all, m->adam_v.p, m->n_total * 4, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        if (steps) std::memcpy(steps, m->steps, sizeof m->steps);
    });
}

svlf_status svlf_model_set_adam(svlf_model* m, const float* m_all, const float* v_all, const uint64_t* steps) {
    return guard([&] {
        require(m != nullptr, "model is null");
        DeviceGuard g(m->ctx->device);
        std::lock_guard<std::mutex> lk(m->ctx->mu);
        cudaStream_t s = m->ctx->stream;
        if (m_all) SVLF_CUDA(cudaMemcpyAsync(m->adam_m.p, m_all, m->n_total * 4, cudaMemcpyHostToDevice, s));
        if (v_all) SVLF_CUDA(cudaMemcpyAsync(m->adam_v.p, v_all, m->n_total * 4, cudaMemcpyHostToDevice, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        if (steps) std::memcpy(m->steps, steps, sizeof m->steps);
    });
}

svlf_status svlf_model_set_adam_hyper(svlf_model* m, const float* beta1, const float* beta2, const float* eps) {
    return guard([&] {
        require(m && beta1 && beta2 && eps, "null argument");
        std::lock_guard<std::mutex> lk(m->ctx->mu);
        for (int i = 0; i < 14; ++i) m->hyper[i] = AdamHyper{beta1[i], beta2[i], eps[i]};
    });
}

svlf_status svlf_model_get_adam_hyper(svlf_model* m, float* beta1, float* beta2, float* eps) {
    return guard([&] {
        require(m && beta1 && beta2 && eps, "null argument");
        std::lock_guard<std::mutex> lk(m->ctx->mu);
        for (int i = 0; i < 14; ++i) {
            beta1[i] = m->hyper[i].beta1;
            beta2[i] = m->hyper[i].beta2;
            eps[i] = m->hyper[i].eps;
        }
    });
}

// ---- render -------------------------------------------------------------------
svlf_status svlf_render_frame_device(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, const float* bg,
                                     svlf_precision prec, float* d_rgb, float* d_alpha, float* d_depth,
                                     svlf_render_stats* stats) {
    return guard([&] {
        require(ctx && m && cam && d_rgb && d_alpha && d_depth, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        render_device(ctx, m, cam, 0, cam->height, bg, prec, d_rgb, d_alpha, d_depth, stats);
    });
}

// Two-phase svlf_render_frame_device: the submit enqueues the frame (16-bit
// modes: no host round trip; fp32 reads the hit count) and returns; the
// finish synchronizes, checks the counters and the error flag, fills the
// statistics and re-renders the frame synchronously if the hit buffers
// overflowed. Used to time the frame on the device without the host's
// synchronisation in the timed region.
svlf_status svlf_render_frame_device_submit(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, const float* bg,
                                            svlf_precision prec, float* d_rgb, float* d_alpha, float* d_depth) {
    return guard([&] {
        require(ctx && m && cam && d_rgb && d_alpha && d_depth, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (cam->width == 0 || cam->height == 0) fail(SVLF_ERR_INVALID_ARGUMENT, "zero-size image");
        const uint64_t n64 = uint64_t(cam->width) * cam->height;
        require(n64 < (1ull << 31), "too many pixels in one call");
        const uint32_t n = uint32_t(n64);
        const DevCamera dc = to_dev_camera(*cam);
        reset_misc(ctx);  // fails while a submitted frame is pending
        uint32_t total = 0;
        if (prec == SVLF_PRECISION_FP32) total = run_traversal(ctx, m->tree, &dc, 0, cam->height, n);
        else enqueue_traversal(ctx, m->tree, &dc, 0, cam->height, n);
        run_decode_composite(ctx, m, n, total, bg, prec, d_rgb, d_alpha, d_depth);
        auto& D = ctx->dev_frame;
        D.m = m;
        D.cam = *cam;
        D.has_bg = bg != nullptr;
        if (bg) std::copy(bg, bg + 3, D.bg);
        D.prec = prec;
        D.rgb = d_rgb;
        D.alpha = d_alpha;
        D.depth = d_depth;
        D.n = n;
        D.active = true;
    });
}

svlf_status svlf_render_frame_device_finish(svlf_ctx* ctx, svlf_render_stats* stats) {
    return guard([&] {
        require(ctx != nullptr, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        auto& D = ctx->dev_frame;
        require(D.active, "no frame from svlf_render_frame_device_submit is pending");
        D.active = false;
        if (finish_render(ctx, D.n, stats)) return;
        render_device(ctx, D.m, &D.cam, 0, D.cam.height, D.has_bg ? D.bg : nullptr, D.prec, D.rgb, D.alpha,
                      D.depth, stats);
    });
}

svlf_status svlf_render_rows_device(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, uint32_t row0,
                                    uint32_t rows, const float* bg, svlf_precision prec, float* d_rgb,
                                    float* d_alpha, float* d_depth, svlf_render_stats* stats) {
    return guard([&] {
        require(ctx && m && cam && d_rgb && d_alpha && d_depth, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        render_device(ctx, m, cam, row0, rows, bg, prec, d_rgb, d_alpha, d_depth, stats);
    });
}

svlf_status svlf_render_tiles_device(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, uint32_t tile_w,
                                     uint32_t tile_h, uint32_t rank, uint32_t world, const float* bg,
                                     svlf_precision prec, float* d_rgb, float* d_alpha, float* d_depth,
                                     svlf_render_stats* stats) {
    return guard([&] {
        require(ctx && m && cam && d_rgb && d_alpha && d_depth, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        render_tiles_device(ctx, m, cam, tile_w, tile_h, rank, world, bg, prec, d_rgb, d_alpha, d_depth, stats);
    });
}

size_t svlf_tiles_owned(const svlf_camera* cam, uint32_t tile_w, uint32_t tile_h, uint32_t rank, uint32_t world) {
    if (!cam || !tile_w || !tile_h || !world || cam->width % tile_w || cam->height % tile_h) return 0;
    return owned_tiles(*cam, tile_w, tile_h, rank, world);
}

svlf_status svlf_render_frame(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, const float* bg,
                              svlf_precision prec, float* rgb, float* alpha, float* depth,
                              svlf_render_stats* stats) {
    return guard([&] {
        require(ctx && m && cam && rgb && alpha && depth, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        render_frame_host(ctx, m, cam, bg, prec, rgb, alpha, depth, stats);
    });
}

svlf_status svlf_render_frame_submit(svlf_ctx* ctx, svlf_model* m, const svlf_camera* cam, const float* bg,
                                     svlf_precision prec, float* rgb, float* alpha, float* depth, uint64_t* ticket) {
    return guard([&] {
        require(ctx && m && cam && rgb && alpha && depth && ticket, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        FrameSlot& F = frame_setup(ctx, m, cam, bg, prec, rgb, alpha, depth);
        F.busy = true;
        try {
            frame_submit(ctx, F, 1);  // whole frame: its copies overlap the next submitted frame
        } catch (...) {
            F.busy = false;
            throw;
        }
        *ticket = F.id;
    });
}

svlf_status svlf_render_frame_wait(svlf_ctx* ctx, uint64_t ticket, svlf_render_stats* stats) {
    return guard([&] {
        require(ctx != nullptr, "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        FrameSlot* F = nullptr;
        for (auto& fs : ctx->slot)
            if (fs.busy && fs.id == ticket) F = &fs;
        require(F != nullptr, "unknown or already completed frame ticket");
        frame_finish(ctx, *F, stats);
    });
}

svlf_status svlf_render_rays(svlf_ctx* ctx, svlf_model* m, const double* rays, size_t n, const float* bg,
                             svlf_precision prec, float* rgb, float* alpha, float* depth,
                             svlf_render_stats* stats) {
    return guard([&] {
        require(ctx && m, "null argument");
        require(n == 0 || (rays && rgb && alpha && depth), "null argument");
        require(n < (1ull << 31), "too many rays");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        const uint32_t nn = uint32_t(n);
        reset_misc(ctx);
        double* d_rays = ctx->rays.ensure<double>(size_t(nn) * 6 + 6);
        SVLF_CUDA(cudaMemcpyAsync(d_rays, rays, size_t(nn) * 48, cudaMemcpyHostToDevice, s));
        float* d_rgb = ctx->out_rgb.ensure<float>(n * 3);
        float* d_alpha = ctx->out_alpha.ensure<float>(n);
        float* d_depth = ctx->out_depth.ensure<float>(n);
        render_pipeline(ctx, m, nullptr, 0, 0, nn, bg, prec, d_rgb, d_alpha, d_depth, stats);
        SVLF_CUDA(cudaMemcpyAsync(rgb, d_rgb, n * 12, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaMemcpyAsync(alpha, d_alpha, n * 4, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaMemcpyAsync(depth, d_depth, n * 4, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

// ---- per-point / per-ray reference operations (perray.cu) ----------------------
// Host buffers in and out, one synchronisation per call: these back the
// reference's single-ray API (tests, debugging), not the frame / train paths.
namespace {

// device copies of a call's host arrays, freed on scope exit
struct CallBufs {
    std::vector<void*> ptrs;
    cudaStream_t s;
    explicit CallBufs(cudaStream_t st) : s(st) {}
    ~CallBufs() {
        cudaStreamSynchronize(s);
        for (void* p : ptrs) cudaFree(p);
    }
    template <typename T>
    T* alloc(size_t n) {
        void* p = nullptr;
        SVLF_CUDA(cudaMalloc(&p, std::max<size_t>(n * sizeof(T), 16)));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <typename T>
    T* up(const T* h, size_t n) {
        T* d = alloc<T>(n);
        if (n) SVLF_CUDA(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
        return d;
    }
    template <typename T>
    void down(T* h, const T* d, size_t n) {
        if (h && n) SVLF_CUDA(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
};

// synchronizes; a raised device error becomes the reference's exception type
void finish_call(svlf_ctx* ctx) {
    int* flag = ctx->misc.as<int>();
    SVLF_CUDA(cudaMemcpyAsync(ctx->h_pinned, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    const int code = ctx->h_pinned[0];
    if (!code) return;
    SVLF_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    const svlf_status st = code == kErrNegativeTau   ? SVLF_ERR_INVALID_ARGUMENT
                           : code == kErrUnknownVoxel ? SVLF_ERR_OUT_OF_RANGE
                                                      : SVLF_ERR_RUNTIME;
    fail(st, dev_error_message(code));
}

}  // namespace

extern "C" {

svlf_status svlf_local_coords(svlf_ctx* ctx, const svlf_octree* tree, const uint64_t* voxel_ids,
                              const double* points, size_t n, double* u_out) {
    return guard([&] {
        require(ctx && tree && (n == 0 || (voxel_ids && points && u_out)), "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        reset_misc(ctx);
        CallBufs B(ctx->stream);
        double* u = B.alloc<double>(3 * n);
        launch_local_coords(dev_view(tree), B.up(voxel_ids, n), B.up(points, 3 * n), n, u, ctx->misc.as<int>(),
                            ctx->stream);
        finish_call(ctx);
        B.down(u_out, u, 3 * n);
        finish_call(ctx);
    });
}

svlf_status svlf_interpolate(svlf_ctx* ctx, const svlf_octree* tree, svlf_dtype dtype, const void* volume,
                             uint32_t rows, uint32_t dim, const uint64_t* voxel_ids, const double* points, size_t n,
                             void* out) {
    return guard([&] {
        require(ctx && tree && volume && (n == 0 || (voxel_ids && points && out)), "null argument");
        require(dtype == SVLF_DTYPE_F32 || dtype == SVLF_DTYPE_F64, "volume dtype must be f32 or f64");
        require(dim >= 1, "dim must be >= 1");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        reset_misc(ctx);
        CallBufs B(ctx->stream);
        const DevOctree& T = dev_view(tree);
        const uint64_t* ids = B.up(voxel_ids, n);
        const double* pts = B.up(points, 3 * n);
        if (dtype == SVLF_DTYPE_F32) {
            float* o = B.alloc<float>(n * dim);
            launch_interpolate<float>(T, B.up(static_cast<const float*>(volume), size_t(rows) * dim), rows, dim, ids,
                                      pts, n, o, ctx->misc.as<int>(), ctx->stream);
            finish_call(ctx);
            B.down(static_cast<float*>(out), o, n * dim);
        } else {
            double* o = B.alloc<double>(n * dim);
            launch_interpolate<double>(T, B.up(static_cast<const double*>(volume), size_t(rows) * dim), rows, dim,
                                       ids, pts, n, o, ctx->misc.as<int>(), ctx->stream);
            finish_call(ctx);
            B.down(static_cast<double*>(out), o, n * dim);
        }
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

svlf_status svlf_interpolate_backward(svlf_ctx* ctx, const svlf_octree* tree, svlf_dtype dtype, const void* volume,
                                      uint32_t rows, uint32_t dim, const uint64_t* voxel_ids, const double* points,
                                      size_t n, const void* upstream, void* grad_buf, double* pos_jac) {
    return guard([&] {
        require(ctx && tree && volume && grad_buf && (n == 0 || (voxel_ids && points && upstream)), "null argument");
        require(dtype == SVLF_DTYPE_F32 || dtype == SVLF_DTYPE_F64, "volume dtype must be f32 or f64");
        require(dim >= 1, "dim must be >= 1");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        reset_misc(ctx);
        CallBufs B(ctx->stream);
        const DevOctree& T = dev_view(tree);
        const uint64_t* ids = B.up(voxel_ids, n);
        const double* pts = B.up(points, 3 * n);
        double* jac = pos_jac ? B.alloc<double>(n * dim * 3) : nullptr;
        const size_t gsz = size_t(rows) * dim;
        if (dtype == SVLF_DTYPE_F32) {
            float* gb = B.up(static_cast<const float*>(grad_buf), gsz);
            launch_interpolate_backward<float>(T, B.up(static_cast<const float*>(volume), gsz), rows, dim, ids, pts, n,
                                               B.up(static_cast<const float*>(upstream), n * dim), gb, jac,
                                               ctx->misc.as<int>(), ctx->stream);
            finish_call(ctx);
            B.down(static_cast<float*>(grad_buf), gb, gsz);
        } else {
            double* gb = B.up(static_cast<const double*>(grad_buf), gsz);
            launch_interpolate_backward<double>(T, B.up(static_cast<const double*>(volume), gsz), rows, dim, ids, pts,
                                                n, B.up(static_cast<const double*>(upstream), n * dim), gb, jac,
                                                ctx->misc.as<int>(), ctx->stream);
            finish_call(ctx);
            B.down(static_cast<double*>(grad_buf), gb, gsz);
        }
        if (jac) B.down(pos_jac, jac, n * dim * 3);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

svlf_status svlf_parameterize_rays(svlf_ctx* ctx, const double* rays, const double* boxes, size_t n, double* out6) {
    return guard([&] {
        require(ctx && (n == 0 || (rays && boxes && out6)), "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        reset_misc(ctx);
        CallBufs B(ctx->stream);
        double* o = B.alloc<double>(6 * n);
        launch_parameterize(B.up(rays, 6 * n), B.up(boxes, 6 * n), n, o, ctx->misc.as<int>(), ctx->stream);
        finish_call(ctx);
        B.down(out6, o, 6 * n);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

svlf_status svlf_composite(svlf_ctx* ctx, const uint64_t* offsets, size_t n_lists, const double* taus,
                           const double* colors, const double* t_s, double* out_color, double* out_alpha,
                           double* out_depth, double* weights) {
    return guard([&] {
        require(ctx && offsets && (n_lists == 0 || (out_color && out_alpha)), "null argument");
        require(!out_depth || t_s, "expected depth needs t_s");
        const size_t ns = offsets[n_lists];
        require(ns == 0 || (taus && colors), "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        reset_misc(ctx);
        CallBufs B(ctx->stream);
        double* c = B.alloc<double>(3 * n_lists);
        double* a = B.alloc<double>(n_lists);
        double* d = out_depth ? B.alloc<double>(n_lists) : nullptr;
        double* w = weights ? B.alloc<double>(ns) : nullptr;
        launch_composite_lists(B.up(offsets, n_lists + 1), n_lists, B.up(taus, ns), B.up(colors, 3 * ns),
                               t_s ? B.up(t_s, ns) : nullptr, c, a, d, w, ctx->misc.as<int>(), ctx->stream);
        finish_call(ctx);
        B.down(out_color, c, 3 * n_lists);
        B.down(out_alpha, a, n_lists);
        if (d) B.down(out_depth, d, n_lists);
        if (w) B.down(weights, w, ns);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

svlf_status svlf_evaluate_voxels(svlf_ctx* ctx, svlf_model* m, const double* rays, const uint64_t* voxel_ids,
                                 const double* t_in, const double* t_out, size_t n, double* tau, double* eta,
                                 double* x_s, double* t_s, double* color) {
    return guard([&] {
        require(ctx && m && (n == 0 || (rays && voxel_ids && t_in && t_out)), "null argument");
        require(n < (1ull << 31), "too many voxels");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        reset_misc(ctx);
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        CallBufs B(s);
        const DevOctree& T = dev_view(m->tree);
        const double* dr = B.up(rays, 6 * n);
        const double* ti = B.up(t_in, n);
        const double* to = B.up(t_out, n);
        uint32_t* leaf = B.alloc<uint32_t>(n);
        uint32_t* ray = B.alloc<uint32_t>(n);
        launch_leaf_lookup(T, B.up(voxel_ids, n), n, leaf, ray, ctx->misc.as<int>(), s);
        finish_call(ctx);
        // the fp32 decoders of render_frame_ref (reference arithmetic order), one hit per voxel
        HitOut ho{B.alloc<float>(n), B.alloc<float>(n), B.alloc<float>(3 * n)};
        ensure_pack_f32(m, s);
        launch_decode_f32(T, m->view(), pack_f32_view(m->pack_f32.as<float>()), dr, ray, leaf, ti, to, uint32_t(n), ho,
                          ctx->misc.as<int>(), s);
        double* xs = B.alloc<double>(3 * n);
        double* ts = B.alloc<double>(n);
        launch_voxel_finish(dr, ti, to, ho.eta, n, xs, ts, s);
        finish_call(ctx);
        std::vector<float> ht(n), he(n), hc(3 * n);
        B.down(ht.data(), ho.tau, n);
        B.down(he.data(), ho.eta, n);
        B.down(hc.data(), ho.rgb, 3 * n);
        B.down(x_s, xs, 3 * n);
        B.down(t_s, ts, n);
        SVLF_CUDA(cudaStreamSynchronize(s));
        for (size_t i = 0; i < n; ++i) {  // static_cast<double>(T) of the decoder outputs (render.cpp:46-47,58)
            if (tau) tau[i] = double(ht[i]);
            if (eta) eta[i] = double(he[i]);
            if (color)
                for (int k = 0; k < 3; ++k) color[3 * i + k] = double(hc[3 * i + k]);
        }
    });
}

svlf_status svlf_eta_gt(svlf_ctx* ctx, const double* t_in, const double* t_out, const double* depth, size_t n,
                        double* out) {
    return guard([&] {
        require(ctx && (n == 0 || (t_in && t_out && depth && out)), "null argument");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        reset_misc(ctx);
        CallBufs B(ctx->stream);
        double* o = B.alloc<double>(n);
        launch_eta_gt(B.up(t_in, n), B.up(t_out, n), B.up(depth, n), n, o, ctx->misc.as<int>(), ctx->stream);
        finish_call(ctx);
        B.down(out, o, n);
        SVLF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"

extern "C" {

// ---- train --------------------------------------------------------------------
namespace {


// A host train batch (rays, c_gt, depth_gt, alpha_gt) and its device destinations.
struct HostBatch {
    struct Part {
        const void* src;
        void* dst;
        size_t elem;
    };
    static constexpr size_t kPerRay = 48 + 12 + 8 + 1;
    Part parts[4];

    bool pinned() const {
        for (const Part& p : parts)
            if (!is_pinned(p.src)) return false;
        return true;
    }
    void dma(cudaStream_t s, uint32_t nn) const {
        for (const Part& p : parts) SVLF_CUDA(cudaMemcpyAsync(p.dst, p.src, p.elem * nn, cudaMemcpyHostToDevice, s));
    }
    // pageable: copied into page-locked `stage` by the pool in chunks, each
    // chunk's DMA overlapping the next chunk's host copy
    void staged_dma(std::unique_ptr<HostPool>& pool, char* stage, cudaStream_t s, uint32_t nn) const {
        const uint32_t chunks = nn >= (1u << 16) ? 4u : 1u;
        for (uint32_t c = 0; c < chunks; ++c) {
            const size_t r0 = size_t(nn) * c / chunks, r1 = size_t(nn) * (c + 1) / chunks;
            const int tasks = pool->size() * 2;
            pool->parallel_for(tasks, [&](int i) {
                const size_t a = r0 + (r1 - r0) * size_t(i) / size_t(tasks);
                const size_t b = r0 + (r1 - r0) * size_t(i + 1) / size_t(tasks);
                size_t base = 0;
                for (const Part& p : parts) {
                    std::memcpy(stage + base + a * p.elem, static_cast<const char*>(p.src) + a * p.elem,
                                (b - a) * p.elem);
                    base += p.elem * nn;
                }
            });
            size_t base = 0;
            for (const Part& p : parts) {
                SVLF_CUDA(cudaMemcpyAsync(static_cast<char*>(p.dst) + r0 * p.elem, stage + base + r0 * p.elem,
                                          (r1 - r0) * p.elem, cudaMemcpyHostToDevice, s));
                base += p.elem * nn;
            }
        }
    }
};

}  // namespace

static void train_common(svlf_ctx* ctx, svlf_model* m, const double* rays, const float* c_gt,
                         const double* depth_gt, const uint8_t* alpha_gt, size_t n, svlf_loss_mode mode,
                         int color_frozen, const svlf_loss_weights* lw, bool adam, float lr,
                         svlf_loss_stats* stats, double* loss_sum, bool device_inputs = false,
                         cudaEvent_t inputs_ready = nullptr) {
    require(ctx && m && lw, "null argument");
    require(n == 0 || (rays && c_gt && depth_gt && alpha_gt), "null argument");
    require(n < (1ull << 31), "too many rays");
    require(mode == SVLF_LOSS_SURFACE || mode == SVLF_LOSS_VOLUMETRIC, "bad loss mode");
    DeviceGuard g(ctx->device);
    std::lock_guard<std::mutex> lk(ctx->mu);
    cudaStream_t s = ctx->stream;
    const uint32_t nn = uint32_t(n);
    reset_misc(ctx);
    TrainScratch& S = ctx->train;
    double* d_rays = ctx->rays.ensure<double>(size_t(nn) * 6 + 6);
    float* d_cgt = S.c_gt.ensure<float>(size_t(nn) * 3 + 3);
    double* d_depth = S.depth.ensure<double>(size_t(nn) + 1);
    uint8_t* d_alpha = S.alpha.ensure<uint8_t>(size_t(nn) + 1);
    if (inputs_ready) SVLF_CUDA(cudaStreamWaitEvent(s, inputs_ready, 0));
    if (nn && inputs_ready) {  // a staged slot (alternating buffers): all copied, so the step's pointers repeat
        SVLF_CUDA(cudaMemcpyAsync(d_rays, rays, size_t(nn) * 48, cudaMemcpyDeviceToDevice, s));
        SVLF_CUDA(cudaMemcpyAsync(d_cgt, c_gt, size_t(nn) * 12, cudaMemcpyDeviceToDevice, s));
        SVLF_CUDA(cudaMemcpyAsync(d_depth, depth_gt, size_t(nn) * 8, cudaMemcpyDeviceToDevice, s));
        SVLF_CUDA(cudaMemcpyAsync(d_alpha, alpha_gt, size_t(nn), cudaMemcpyDeviceToDevice, s));
    } else if (nn && device_inputs) {  // rays copied (the traversal writes into ctx->rays), supervision read in place
        SVLF_CUDA(cudaMemcpyAsync(d_rays, rays, size_t(nn) * 48, cudaMemcpyDeviceToDevice, s));
        d_cgt = const_cast<float*>(c_gt);
        d_depth = const_cast<double*>(depth_gt);
        d_alpha = const_cast<uint8_t*>(alpha_gt);
    } else if (nn) {
        const HostBatch hb{{{rays, d_rays, 48}, {c_gt, d_cgt, 12}, {depth_gt, d_depth, 8}, {alpha_gt, d_alpha, 1}}};
        if (hb.pinned()) {
            hb.dma(s, nn);
        } else {
            if (S.h_stage_bytes < HostBatch::kPerRay * nn) {
                if (S.h_stage) SVLF_CUDA(cudaFreeHost(S.h_stage));
                S.h_stage = nullptr;
                S.h_stage_bytes = 0;
                SVLF_CUDA(cudaMallocHost(&S.h_stage, HostBatch::kPerRay * nn));
                S.h_stage_bytes = HostBatch::kPerRay * nn;
            }
            hb.staged_dma(host_pool(ctx->pool), static_cast<char*>(S.h_stage), s, nn);
        }
    }
    // Traversal and step are enqueued with no host round trip; the step's one
    // readback reports a hit-buffer or exchange-buffer overflow (any rank), in
    // which case nothing was updated and the whole step is re-run with larger
    // buffers.
    TrainOptions opt{mode == SVLF_LOSS_SURFACE, color_frozen != 0, adam, *lw, lr, ctx->coll.get(), ctx->train_tf32};
    TrainModelRefs mr{m->view(), m->params.as<float>(), m->grads.as<float>(), m->adam_m.as<float>(),
                      m->adam_v.as<float>(), m->n_ft, m->n_fc, m->steps, m->hyper};
    TrainResult r;
    float trav_ms = 0.f;
    for (int attempt = 0;; ++attempt) {
        // the traversal runs inside the step's graph (captured with it)
        TraverseOut to{};
        std::function<void(bool)> pre;
        std::vector<uint64_t> pre_key;
        if (nn) {
            to = prepare_traversal(ctx, nn);
            const svlf_octree* tree = m->tree;
            pre = [ctx, tree, nn, to](bool capturing) { launch_traversal(ctx, tree, nullptr, 0, 0, nn, to, capturing); };
            for (const void* p : {(const void*)to.ray_off, (const void*)to.ray_cnt, (const void*)to.hit_leaf,
                                  (const void*)to.hit_tin, (const void*)to.hit_tout, (const void*)to.hit_ray,
                                  (const void*)to.counters, (const void*)to.overflow_rays, (const void*)to.overflow_dense,
                                  (const void*)to.rays, (const void*)tree})
                pre_key.push_back(reinterpret_cast<uint64_t>(p));
            pre_key.push_back(to.capacity);
            pre_key.push_back(ctx->count_node_tests ? 1 : 0);
        } else {
            ctx->hit_cap = std::max<size_t>(ctx->hit_cap, 32);
            ctx->hit_leaf.ensure<uint32_t>(ctx->hit_cap);
            ctx->hit_tin.ensure<double>(ctx->hit_cap);
            ctx->hit_tout.ensure<double>(ctx->hit_cap);
            SVLF_CUDA(cudaMemsetAsync(traversal_counters(ctx), 0, 32, s));
        }
        TrainBatchDev b{d_rays, d_cgt, d_depth, d_alpha, nn, ctx->offsets.ensure<uint32_t>(size_t(nn) + 1),
                        ctx->counts.ensure<uint32_t>(size_t(nn) + 1), ctx->hit_leaf.as<uint32_t>(),
                        ctx->hit_tin.as<double>(), ctx->hit_tout.as<double>(), traversal_counters(ctx),
                        uint32_t(ctx->hit_cap)};
        if (nn) {
            b.pre = &pre;
            b.pre_key = &pre_key;
        }
        r = run_train_step(S, dev_view(m->tree), mr, b, opt, s, ctx->misc.as<int>());
        if (nn) cudaEventElapsedTime(&trav_ms, ctx->ev[EV_START], ctx->ev[EV_EMIT]);
        if (r.error || !r.flags) break;
        if (attempt >= 3) fail(SVLF_ERR_RUNTIME, "train step buffers could not be sized");
        if ((r.flags & kStepHitOverflow) && r.hits > ctx->hit_cap)  // else the step grew its own matrices
            ctx->hit_cap = std::min<size_t>(size_t(r.hits) + r.hits / 4 + 1024, 0xfffff000u);
    }
    r.timings.traverse_ms = trav_ms;
    if (r.error) fail(SVLF_ERR_RUNTIME, dev_error_message(r.error));
    if (r.updated) {  // the Adam steps that ran (colour tensors frozen: not advanced)
        for (int i = 0; i < 14; ++i)
            if (!color_frozen || !(i == 1 || i >= 6)) ++m->steps[i];
        ++m->version;
    }
    ctx->last = r.timings;
    if (stats) {
        stats->rays += r.rays;
        stats->skipped_rays += r.skipped;
        stats->eta_skipped += r.eta_skipped;
    }
    if (loss_sum) *loss_sum = r.loss;
}

svlf_status svlf_train_step(svlf_ctx* ctx, svlf_model* m, const double* rays, const float* c_gt,
                            const double* depth_gt, const uint8_t* alpha_gt, size_t n, svlf_loss_mode mode,
                            int color_frozen, float lr, const svlf_loss_weights* lw, svlf_loss_stats* stats,
                            double* loss_sum) {
    return guard([&] {
        train_common(ctx, m, rays, c_gt, depth_gt, alpha_gt, n, mode, color_frozen, lw, true, lr, stats,
                     loss_sum);
    });
}

svlf_status svlf_train_step_device(svlf_ctx* ctx, svlf_model* m, const double* rays, const float* c_gt,
                                   const double* depth_gt, const uint8_t* alpha_gt, size_t n, svlf_loss_mode mode,
                                   int color_frozen, float lr, const svlf_loss_weights* lw, svlf_loss_stats* stats,
                                   double* loss_sum) {
    return guard([&] {
        train_common(ctx, m, rays, c_gt, depth_gt, alpha_gt, n, mode, color_frozen, lw, true, lr, stats, loss_sum,
                     true);
    });
}

svlf_status svlf_train_batch_stage(svlf_ctx* ctx, const double* rays, const float* c_gt, const double* depth_gt,
                                   const uint8_t* alpha_gt, size_t n, int* slot) {
    return guard([&] {
        require(ctx && slot, "null argument");
        require(n == 0 || (rays && c_gt && depth_gt && alpha_gt), "null argument");
        require(n < (1ull << 31), "too many rays");
        DeviceGuard g(ctx->device);
        std::lock_guard<std::mutex> lk(ctx->mu);
        const int k = ctx->next_tslot;
        svlf_ctx::TrainSlot& T = ctx->tslot[k];
        require(!T.staged, "both train staging slots hold batches that have not been stepped");
        const uint32_t nn = uint32_t(n);
        const HostBatch hb{{{rays, T.rays.ensure<double>(size_t(nn) * 6 + 6), 48},
                            {c_gt, T.c_gt.ensure<float>(size_t(nn) * 3 + 3), 12},
                            {depth_gt, T.depth.ensure<double>(size_t(nn) + 1), 8},
                            {alpha_gt, T.alpha.ensure<uint8_t>(size_t(nn) + 1), 1}}};
        cudaStream_t c = ctx->copy_stream;
        if (nn == 0 || hb.pinned()) {
            if (nn) hb.dma(c, nn);
            SVLF_CUDA(cudaEventRecord(T.copied, c));
        } else {
            if (T.h_stage_bytes < HostBatch::kPerRay * nn) {
                if (T.h_stage) SVLF_CUDA(cudaFreeHost(T.h_stage));
                T.h_stage = nullptr;
                T.h_stage_bytes = 0;
                SVLF_CUDA(cudaMallocHost(&T.h_stage, HostBatch::kPerRay * nn));
                T.h_stage_bytes = HostBatch::kPerRay * nn;
            }
            host_pool(ctx->stage_pool);
            const int dev = ctx->device;
            T.job = std::async(std::launch::async, [ctx, &T, hb, c, nn, dev] {
                DeviceGuard g2(dev);
                std::lock_guard<std::mutex> lk2(ctx->stage_mu);
                hb.staged_dma(ctx->stage_pool, T.h_stage, c, nn);
                SVLF_CUDA(cudaEventRecord(T.copied, c));
            });
        }
        T.n = nn;
        T.staged = true;
        ctx->next_tslot ^= 1;
        *slot = k;
    });
}

static svlf_ctx::TrainSlot& staged_slot(svlf_ctx* ctx, int slot) {
    require(ctx, "null argument");
    require(slot == 0 || slot == 1, "bad staging slot");
    svlf_ctx::TrainSlot& T = ctx->tslot[slot];
    require(T.staged, "no batch staged in this slot");
    if (T.job.valid()) T.job.get();  // rethrows a failed host copy
    return T;
}

svlf_status svlf_train_step_staged(svlf_ctx* ctx, svlf_model* m, int slot, svlf_loss_mode mode, int color_frozen,
                                   float lr, const svlf_loss_weights* lw, svlf_loss_stats* stats,
                                   double* loss_sum) {
    return guard([&] {
        svlf_ctx::TrainSlot& T = staged_slot(ctx, slot);
        struct Release {
            svlf_ctx::TrainSlot& t;
            ~Release() { t.staged = false; }
        } release{T};
        train_common(ctx, m, T.rays.as<double>(), T.c_gt.as<float>(), T.depth.as<double>(), T.alpha.as<uint8_t>(),
                     T.n, mode, color_frozen, lw, true, lr, stats, loss_sum, true, T.copied);
    });
}

svlf_status svlf_train_batch_discard(svlf_ctx* ctx, int slot) {
    return guard([&] {
        require(ctx, "null argument");
        require(slot == 0 || slot == 1, "bad staging slot");
        svlf_ctx::TrainSlot& T = ctx->tslot[slot];
        require(T.staged, "no batch staged in this slot");
        struct Release {
            svlf_ctx::TrainSlot& t;
            ~Release() { t.staged = false; }
        } release{T};
        if (T.job.valid()) T.job.wait();  // a failed host copy is dropped with the batch
        T.job = {};
        DeviceGuard g(ctx->device);
        SVLF_CUDA(cudaEventSynchronize(T.copied));
    });
}

svlf_status svlf_loss_grads(svlf_ctx* ctx, svlf_model* m, const double* rays, const float* c_gt,
                            const double* depth_gt, const uint8_t* alpha_gt, size_t n, svlf_loss_mode mode,
                            int color_frozen, const svlf_loss_weights* lw, svlf_loss_stats* stats,
                            double* loss_sum) {
    return guard([&] {
        train_common(ctx, m, rays, c_gt, depth_gt, alpha_gt, n, mode, color_frozen, lw, false, 0.f, stats,
                     loss_sum);
    });
}

}  // extern "C"
