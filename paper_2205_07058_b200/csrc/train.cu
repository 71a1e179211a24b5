// Train step: placeholder until the fused backward lands.
#include "train.cuh"

namespace svlfb {

TrainScratch::~TrainScratch() {
    if (h_pinned) cudaFreeHost(h_pinned);
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
}

TrainResult run_train_step(TrainScratch&, const DevOctree&, TrainModelRefs&, const TrainArgs&, cudaStream_t,
                           int*) {
    fail(SVLF_ERR_RUNTIME, "train step not implemented yet");
}

}  // namespace svlfb
