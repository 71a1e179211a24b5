// svlf/train.hpp — the training step (reference include/svlf/train.hpp:31-71
// and the per-frame body of train(), src/train.cpp:443-479).
//
// The reference has no public step API; train_step below is the one SURVEY.md
// §8(b) defines: loss + summed gradients over the batch + adam_model_step,
// executed on the GPU. Gradients are sums over rays (no 1/N); lr is rounded
// to float; the colour tensors are frozen (no gradient, no Adam step) when
// color_frozen is set.
#pragma once

#include <array>
#include <span>
#include <string>
#include <vector>

#include "svlf/dataset.hpp"
#include "svlf/model.hpp"
#include "svlf/render.hpp"

namespace svlf {

struct RaySupervision {
    Ray ray;
    float c_gt[3] = {0, 0, 0};
    double depth_gt = 0;  // Euclidean depth along the ray, 0 = background
    bool alpha_gt = false;
};

// Within-voxel depth target (train.hpp:38-41): (t_out - depth) / (t_out - t_in)
// clamped to [0,1]; throws runtime_error("surface point outside voxel") beyond
// 1e-6 (svlf_eta_gt).
double eta_gt(const RayVoxelHit& hit, double depth_gt);

struct LossWeights {
    double eta = 1.0;
    double tau = 0.01;
    double empty = 0.01;  // stage-1 pre-surface penalty; 0 = surface voxel only
    double alpha = 0.1;
};

struct LossStats {
    long long rays = 0;
    long long skipped_rays = 0;
    long long eta_skipped = 0;
};

// The reference's per-ray losses (train.hpp:56-71): loss of one ray with its
// gradients ADDED into `grads` (null: loss only), through the GPU train
// kernels (svlf_loss_grads on a one-ray batch). Float models only.
template <typename T>
double surface_loss(const SvlfModelT<T>& model, const RaySupervision& sup, const LossWeights& lw,
                    ModelGradsT<T>* grads, LossStats* stats = nullptr);
template <typename T>
double volumetric_loss(const SvlfModelT<T>& model, const RaySupervision& sup, const LossWeights& lw,
                       bool color_frozen, ModelGradsT<T>* grads, LossStats* stats = nullptr);

enum class LossMode { Surface = 0, Volumetric = 1 };

// One optimizer step; returns the loss summed over the batch. Updates
// `model` and `adam` in place (the device copy is synchronised back).
double train_step(SvlfModel& model, ModelAdam& adam, std::span<const RaySupervision> batch, LossMode mode,
                  bool color_frozen, float lr, const LossWeights& lw = {}, LossStats* stats = nullptr);

// ---- the stage driver (reference include/svlf/train.hpp:12-29,73-94;
// src/train.cpp:364-527) on top of train_step: occupancy from the training
// views' back-projected depth, octree, init_model, three stages of epochs
// over the training views in the reference's seeded shuffle order (one Adam
// step per view), mean loss, divergence guard, validation PSNR (fp32
// renders), train.log and stage checkpoints. The model stays on the GPU for
// the whole run (svlf::b200::DeviceModel) and is copied back for checkpoints
// and the result.
struct TrainConfig {
    std::array<int, 3> epochs{100, 150, 50};
    double lr_main = 1e-3;      // stages 1-2
    double lr_finetune = 2e-4;  // stage 3
    double lambda_eta = 1.0;
    double lambda_tau = 0.01;
    double lambda_empty = 0.01;
    double lambda_alpha = 0.1;
    uint64_t seed = 0;
    uint32_t grid_resolution = 128;
    uint32_t dilation = 1;
    uint32_t train_res = 0;  // 0 = native dataset resolution
    std::string out_dir;     // checkpoints + train.log; empty = no files

    void validate() const;
};

struct EpochLog {
    int stage = 0;  // 1-based
    int epoch = 0;  // 1-based within the stage
    double mean_loss = 0;
    double val_psnr = 0;
    double seconds = 0;
};

struct TrainResult {
    SvlfModel model;
    ModelAdam adam;
    std::vector<EpochLog> log;
    std::array<double, 3> stage_lrs{};
    long long skipped_rays = 0;
    long long dropped_points = 0;
    bool diverged = false;
    std::array<std::string, 4> checkpoints;  // stage1..3 boundaries + final
};

TrainResult train(const TrainConfig& config, const SceneDataset& dataset);

// Loss and gradients only: sum over the batch of surface_loss /
// volumetric_loss (reference train.hpp:60-71) with grads accumulated.
double loss_grads(const SvlfModel& model, std::span<const RaySupervision> batch, LossMode mode,
                  bool color_frozen, const LossWeights& lw, ModelGrads* grads, LossStats* stats = nullptr);

}  // namespace svlf
