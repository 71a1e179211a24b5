// svlf/b200.hpp — B200-specific controls of the C++ API (no reference
// counterpart).
//
// * Process-wide session: one svlf_ctx (CUDA device + stream + arenas) used by
//   the drop-in functions in render.hpp / train.hpp / octree.hpp. Calls are
//   serialised by a mutex, so concurrent read-only renders are safe.
// * DeviceModel: the explicit fast path. The device copy is authoritative;
//   train steps do not round-trip the tensors to the host; sync_to() copies
//   them back on demand (validation renders on the host side, checkpoints).
#pragma once

#include <deque>
#include <memory>
#include <span>

#include "svlf/render.hpp"
#include "svlf/train.hpp"

struct svlf_ctx;
struct svlf_model;

namespace svlf::b200 {

enum class Precision { FP32 = 0, BF16 = 1, FP16 = 2 };

void set_device(int device);  // before first use; default $SVLF_DEVICE or 0
void set_render_precision(Precision p);
Precision render_precision();
// Dense-layer GEMMs of the train step (tcgen05 kernels in every mode): FP32
// (default) and TF32X3 run three TF32 products of split operands (fp32 parity
// gates); TF32 runs the weight gradients in plain TF32 (16-bit gates).
enum class TrainPrecision { FP32 = 0, TF32X3 = 4, TF32 = 3 };
void set_train_precision(TrainPrecision p);
svlf_ctx* session_context();  // creates the session on first call

class DeviceModel {
  public:
    explicit DeviceModel(const SvlfModel& model);
    DeviceModel(const SvlfModel& model, const ModelAdam& adam);
    ~DeviceModel();
    DeviceModel(const DeviceModel&) = delete;
    DeviceModel& operator=(const DeviceModel&) = delete;

    void upload(const SvlfModel& model);
    void upload(const ModelAdam& adam);
    void sync_to(SvlfModel& model) const;
    void sync_to(ModelAdam& adam) const;

    void render(const Camera& camera, FrameBuffers& out, RenderStats* stats = nullptr,
                const float* background = nullptr) const;
    // fp32 CUDA-core decoders in the reference's arithmetic order
    void render_ref(const Camera& camera, FrameBuffers& out, RenderStats* stats = nullptr,
                    const float* background = nullptr) const;
    double train_step(std::span<const RaySupervision> batch, LossMode mode, bool color_frozen, float lr,
                      const LossWeights& lw = {}, LossStats* stats = nullptr);
    // Pipelined steps (svlf_train_batch_stage / svlf_train_step_staged):
    // stage_batch uploads a batch asynchronously (at most two staged);
    // train_staged runs train_step on the oldest staged batch. Staging batch
    // k + 1 before stepping batch k overlaps its upload with the step.
    void stage_batch(std::span<const RaySupervision> batch);
    double train_staged(LossMode mode, bool color_frozen, float lr, const LossWeights& lw = {},
                        LossStats* stats = nullptr);
    size_t staged_batches() const { return staged_.size(); }

    svlf_model* handle() const { return m_; }

  private:
    struct StagedBatch;
    SparseOctree octree_;  // keeps the library octree alive
    svlf_model* m_ = nullptr;
    std::deque<std::unique_ptr<StagedBatch>> staged_;
};

}  // namespace svlf::b200
