// svlf/metrics.hpp — image metrics used by training validation (reference
// include/svlf/metrics.hpp:21-24).
#pragma once

#include "svlf/image.hpp"

namespace svlf {

constexpr double kPsnrCap = 99.0;  // returned when the MSE is exactly zero

// 10 log10(1/MSE) over all channels (double accumulation in pixel order).
double psnr(const Image& pred, const Image& gt);

}  // namespace svlf
