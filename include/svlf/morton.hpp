// svlf/morton.hpp — 63-bit Morton codes, 21 bits per axis; bit k of x goes
// to bit 3k, y to 3k+1, z to 3k+2 (reference include/svlf/morton.hpp:9-37).
#pragma once

#include <cstdint>

namespace svlf {

namespace detail {
// magic-number bit spreading: each step doubles the gap between bit groups
inline constexpr uint64_t kSpreadMask[6] = {0x00000000001fffffULL, 0x001f00000000ffffULL, 0x001f0000ff0000ffULL,
                                            0x100f00f00f00f00fULL, 0x10c30c30c30c30c3ULL, 0x1249249249249249ULL};
inline constexpr int kSpreadShift[5] = {32, 16, 8, 4, 2};
}  // namespace detail

inline uint64_t morton_spread(uint64_t v) {
    v &= detail::kSpreadMask[0];
    for (int i = 0; i < 5; ++i) v = (v | (v << detail::kSpreadShift[i])) & detail::kSpreadMask[i + 1];
    return v;
}

inline uint64_t morton_compact(uint64_t v) {
    v &= detail::kSpreadMask[5];
    for (int i = 4; i >= 0; --i) v = (v ^ (v >> detail::kSpreadShift[i])) & detail::kSpreadMask[i];
    return v;
}

inline uint64_t morton_encode(uint32_t x, uint32_t y, uint32_t z) {
    return morton_spread(x) | morton_spread(y) << 1 | morton_spread(z) << 2;
}

inline void morton_decode(uint64_t code, uint32_t& x, uint32_t& y, uint32_t& z) {
    x = uint32_t(morton_compact(code));
    y = uint32_t(morton_compact(code >> 1));
    z = uint32_t(morton_compact(code >> 2));
}

}  // namespace svlf
