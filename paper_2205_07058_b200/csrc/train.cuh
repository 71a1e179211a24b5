// Train-step pipeline interface (train.cu).
#pragma once

#include "device.cuh"

namespace svlfb {

struct TrainArgs {
    const double* rays;      // host, n x 6
    const float* c_gt;       // host, n x 3
    const double* depth_gt;  // host, n
    const uint8_t* alpha_gt; // host, n
    uint32_t n;
    bool surface;       // LossMode::Surface (stage 1) vs Volumetric
    bool color_frozen;  // stage 2
    svlf_loss_weights lw;
    bool adam;  // false: loss + grads only
    float lr;
};

struct TrainModelRefs {
    DevModel view;
    float* params;
    float* grads;
    float* adam_m;
    float* adam_v;
    size_t n_ft, n_fc;
    uint64_t* steps;  // 14 Adam step counters (host)
};

struct TrainResult {
    double loss = 0;
    long long rays = 0, skipped = 0, eta_skipped = 0;
    int error = 0;
    svlf_timings timings{};
};

struct TrainScratch {
    DevBuf in_rays, in_cgt, in_depth, in_alpha;         // uploaded batch
    DevBuf counts, offsets, scan_tmp, hit_leaf, hit_tin, hit_tout, hit_ray;
    DevBuf ray_info, hit_state, hit_col, stats, pack;   // per-ray / per-hit state
    DevBuf loss_parts;
    int* h_pinned = nullptr;
    cudaEvent_t ev[8] = {};
    ~TrainScratch();
};

TrainResult run_train_step(TrainScratch& S, const DevOctree& T, TrainModelRefs& M, const TrainArgs& a,
                           cudaStream_t s, int* err_flag);

}  // namespace svlfb
