// Internal: the process-wide session of the C++ API (one svlf_ctx) and the
// status -> exception mapping of the C ABI.
#pragma once

#include <mutex>
#include <stdexcept>
#include <string>

#include "svlf/b200.hpp"
#include "svlf/model.hpp"
#include "svlf_b200.h"

namespace svlf::detail {

// Re-throws a C ABI status as the reference's exception type and message.
inline void check(svlf_status s) {
    if (s == SVLF_OK) return;
    std::string msg = svlf_last_error();
    switch (s) {
        case SVLF_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SVLF_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

std::recursive_mutex& session_mutex();
// The device copy of a host model (cached per model object, refreshed when the host tensors change).
svlf_model* device_model(const SvlfModel& m);
svlf_precision to_c(b200::Precision p);

}  // namespace svlf::detail
