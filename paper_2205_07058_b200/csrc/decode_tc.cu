// tcgen05 bf16 decoder: placeholder.
#include "device.cuh"

namespace svlfb {

void ensure_pack_bf16(const DevModel&, DevBuf&, uint64_t&, uint64_t, cudaStream_t) {
    fail(SVLF_ERR_RUNTIME, "bf16 decoder not implemented yet");
}

void launch_decode_bf16(const DevOctree&, const DevModel&, const char*, const double*, const uint32_t*,
                        const uint32_t*, const double*, const double*, uint32_t, HitOut, int*, cudaStream_t) {
    fail(SVLF_ERR_RUNTIME, "bf16 decoder not implemented yet");
}

}  // namespace svlfb
