// svlf/train.hpp — the training step (reference include/svlf/train.hpp:31-71
// and the per-frame body of train(), src/train.cpp:443-479).
//
// The reference has no public step API; train_step below is the one SURVEY.md
// §8(b) defines: loss + summed gradients over the batch + adam_model_step,
// executed on the GPU. Gradients are sums over rays (no 1/N); lr is rounded
// to float; the colour tensors are frozen (no gradient, no Adam step) when
// color_frozen is set.
#pragma once

#include <span>

#include "svlf/model.hpp"

namespace svlf {

struct RaySupervision {
    Ray ray;
    float c_gt[3] = {0, 0, 0};
    double depth_gt = 0;  // Euclidean depth along the ray, 0 = background
    bool alpha_gt = false;
};

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

enum class LossMode { Surface = 0, Volumetric = 1 };

// One optimizer step; returns the loss summed over the batch. Updates
// `model` and `adam` in place (the device copy is synchronised back).
double train_step(SvlfModel& model, ModelAdam& adam, std::span<const RaySupervision> batch, LossMode mode,
                  bool color_frozen, float lr, const LossWeights& lw = {}, LossStats* stats = nullptr);

// Loss and gradients only: sum over the batch of surface_loss /
// volumetric_loss (reference train.hpp:60-71) with grads accumulated.
double loss_grads(const SvlfModel& model, std::span<const RaySupervision> batch, LossMode mode,
                  bool color_frozen, const LossWeights& lw, ModelGrads* grads, LossStats* stats = nullptr);

}  // namespace svlf
