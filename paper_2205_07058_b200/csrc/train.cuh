// Train-step pipeline interface (train.cu).
#pragma once

#include "device.cuh"

namespace svlfb {

// A supervised ray batch resident on the device plus its traversal output
// (per-ray segments of sorted hits, see TraverseOut).
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
    uint32_t total_hits;
};

struct TrainOptions {
    bool surface;       // LossMode::Surface (stage 1) vs Volumetric (stages 2-3)
    bool color_frozen;  // stage 2
    bool adam;          // false: loss + gradients only
    svlf_loss_weights lw;
    float lr;
    void* nccl_comm = nullptr;  // ncclComm_t: data-parallel gradient exchange when set
    int world = 1;
    bool tf32 = false;          // weight-gradient GEMMs on tensor cores (TF32 operands)
    bool tf32x3 = false;        // every GEMM as hi*hi + hi*lo + lo*hi of TF32 splits (tensor cores)
};

struct TrainModelRefs {
    DevModel view;
    float* params;
    float* grads;
    float* adam_m;
    float* adam_v;
    size_t n_ft, n_fc;
    uint64_t* steps;  // 14 Adam step counters (host), ModelAdam order
    DecPackF32 pack;  // transposed fp32 decoders (current version)
};

struct TrainResult {
    double loss = 0;
    long long rays = 0, skipped = 0, eta_skipped = 0;
    int error = 0;
    svlf_timings timings{};
    long long exchanged_rows = 0;  // feature rows all-reduced (data-parallel)
};

struct TrainScratch {
    DevBuf c_gt, depth, alpha;                                    // uploaded supervision
    DevBuf act_first, act_cnt, dpos, surf_rel, eta_gt, ray_loss;  // per ray
    DevBuf dhit, dray, hitf, hitd;                                // per active hit
    DevBuf acts, deltas;                                          // feature-major scratch
    DevBuf scan_tmp, counters, loss_out;
    DevBuf touched, rows, n_rows, packed, red;  // sparse feature-gradient exchange
    DevBuf dxs, ones;                           // layer-0 input gradients, ones vector (bias sums)
    DevBuf wimg;                                // 3xTF32 weight image (gemm_x3.cu)
    void* blas = nullptr;                       // cublasHandle_t (fp32 dense-layer GEMMs)
    int* h_pinned = nullptr;
    cudaEvent_t ev[8] = {};
    ~TrainScratch();
};

TrainResult run_train_step(TrainScratch& S, const DevOctree& T, TrainModelRefs& M, const TrainBatchDev& b,
                           const TrainOptions& o, cudaStream_t s, int* err_flag);

}  // namespace svlfb
