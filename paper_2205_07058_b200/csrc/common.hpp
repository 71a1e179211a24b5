// Shared host-side plumbing: status codes, thread-local error text, CUDA
// checks. Errors raised anywhere below the C ABI are SvlfError carrying the
// svlf_status and the reference's exception message; capi.cu converts them
// to return codes (no exception crosses the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "svlf_b200.h"

namespace svlfb {

struct SvlfError : std::runtime_error {
    svlf_status status;
    SvlfError(svlf_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(svlf_status s, const std::string& m) { throw SvlfError(s, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        fail(SVLF_ERR_CUDA, std::string("CUDA error in ") + what + " (" + file + ":" +
                                std::to_string(line) + "): " + cudaGetErrorString(e));
}

}  // namespace svlfb

#define SVLF_CUDA(x) ::svlfb::cuda_check((x), #x, __FILE__, __LINE__)
