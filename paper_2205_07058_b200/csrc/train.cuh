// Train-step pipeline interface (train.cu).
#pragma once

#include <functional>
#include <vector>

#include "device.cuh"

namespace svlfb {

// A supervised ray batch resident on the device plus its traversal output
// (per-ray segments of sorted hits, see TraverseOut). The hit count is never
// read on the host: trav_counters[0] is the number of hits, trav_counters[2]
// is set when the traversal overflowed hit_cap (the step then skips its
// optimizer update and reports the overflow so the caller re-runs it).
struct TrainBatchDev {
    const double* rays;      // n x 6
    const float* c_gt;       // n x 3
    const double* depth_gt;  // n (Euclidean, 0 = background)
    const uint8_t* alpha_gt; // n (0/1)
    uint32_t n;
    const uint32_t* ray_off;
    const uint32_t* ray_cnt;
    const uint32_t* hit_leaf;
    const double* hit_tin;
    const double* hit_tout;
    const uint32_t* trav_counters;
    uint32_t hit_cap;
    // Work enqueued ahead of the step on the same stream and captured with it into
    // the step's graph (the traversal); its key lists what it bakes in. The
    // argument is true while a graph is being captured.
    const std::function<void(bool)>* pre = nullptr;
    const std::vector<uint64_t>* pre_key = nullptr;
};

// In-place all-reduce used by the data-parallel step (enqueued on stream s).
// NCCL (ncclAllReduce over NVLink) in production; a host-staged variant lets a
// CPU-side framework (gloo, MPI) or a test drive the same exchange.
enum class CollType { F32, F64, U8 };
enum class CollOp { Sum, Max };
struct Collective {
    int rank = 0, world = 1;
    virtual ~Collective() = default;
    virtual void allreduce(void* dev, size_t count, CollType t, CollOp op, cudaStream_t s) = 0;
};

struct TrainOptions {
    bool surface;       // LossMode::Surface (stage 1) vs Volumetric (stages 2-3)
    bool color_frozen;  // stage 2
    bool adam;          // false: loss + gradients only
    svlf_loss_weights lw;
    float lr;
    Collective* coll = nullptr;  // data-parallel gradient exchange when set
    bool tf32 = false;           // weight-gradient GEMMs with plain TF32 operands (16-bit tolerance)
};

// Adam hyperparameters of one ModelAdam tensor (AdamState, mlp.hpp:117-128)
struct AdamHyper {
    float beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f;
};

struct TrainModelRefs {
    DevModel view;
    float* params;
    float* grads;
    float* adam_m;
    float* adam_v;
    size_t n_ft, n_fc;
    const uint64_t* steps;    // 14 Adam step counters (host), ModelAdam order; advanced by the caller
    const AdamHyper* hyper;   // 14 entries, ModelAdam order
};

// Status bits of a step (TrainResult::flags)
// kStepHitOverflow: the traversal's hit buffers or the per-active-hit matrices were too small;
// kStepRowOverflow: the exchanged-row buffer was (data parallel). Both grow before the re-run.
enum : uint32_t { kStepHitOverflow = 1u, kStepRowOverflow = 2u };

struct TrainResult {
    double loss = 0;
    long long rays = 0, skipped = 0, eta_skipped = 0;
    int error = 0;            // device error code (tangent ray, ...); the update was skipped
    uint32_t flags = 0;       // kStep* overflow bits (any rank); the update was skipped, re-run the step
    uint32_t hits = 0;        // traversal hits (this rank)
    uint32_t active = 0;      // active hits (this rank)
    uint32_t touched_rows = 0;  // feature rows exchanged (data-parallel; union over ranks)
    bool updated = false;     // Adam ran (advance the step counters)
    svlf_timings timings{};
};

struct TrainScratch {
    DevBuf c_gt, depth, alpha;                                    // uploaded supervision
    DevBuf act_first, act_cnt, dpos, surf_rel, eta_gt, ray_loss;  // per ray
    DevBuf dhit, dray, hitf, hitd;                                // per active hit
    DevBuf acts, deltas, dxs;                                     // feature-major matrices (row stride ld)
    DevBuf scan_tmp, counters, loss_out, status;
    DevBuf touched, rows, n_rows, packed, red;  // sparse feature-gradient exchange
    DevBuf wimg, dw_part;                       // weight images, weight-gradient partials (gemm_x3.cu)
    uint32_t rows_cap = 0;                      // capacity of the exchanged-row buffer (grows on overflow)
    uint32_t act_cap = 0;                       // capacity of the per-active-hit matrices (grows on overflow)
    uint64_t* h_mail = nullptr;                 // pinned readback mailbox (one sync per step)
    void* h_plan = nullptr;                     // pinned staging of the step's Adam plan
    void* h_stage = nullptr;                    // pinned staging of a pageable host batch
    size_t h_stage_bytes = 0;
    DevBuf plan;                                // the Adam plan on the device
    void* graph = nullptr;                      // cudaGraphExec_t of the captured step (replayed while the key holds)
    std::vector<uint64_t> graph_key, last_key;
    long long graph_captures = 0, graph_replays = 0, graph_launches = 0;
    cudaEvent_t ev[8] = {};
    ~TrainScratch();
};

// Enqueues the whole step (no host round trip) and synchronizes once at the
// end to read the loss, the statistics and the status.
TrainResult run_train_step(TrainScratch& S, const DevOctree& T, const TrainModelRefs& M, const TrainBatchDev& b,
                           const TrainOptions& o, cudaStream_t s, int* err_flag);

// Dense Adam over the model with the gradients currently in M.grads
// (adam_model_step, src/train.cpp:345-360), enqueued on s; skipped on the
// device when *skip_if is non-zero (skip_if may be null).
void launch_adam(const TrainModelRefs& M, bool color_frozen, float lr, const uint32_t* skip_if, const int* err,
                 cudaStream_t s);

}  // namespace svlfb
