// Host-side sparse voxel octree: the build/load half of the boundary
// (reference SparseOctree::build / from_leaves, src/octree.cpp:30-142) plus
// the flattened node table the traversal kernel walks.
//
// Device layout (uploaded once per octree, read-only afterwards):
//   nodes[g]   = {first_child_global_index, child_mask}  for every internal
//                node g; levels 0..L-1 are concatenated in level order and,
//                within a level, in ascending Morton order, so the children of
//                a node are contiguous and ranked by popcount of the mask.
//   level_off  = global index of the first node of each level (leaves last),
//                so leaf index = global - level_off[L] = position in the
//                reference's leaf_codes() vector.
//   corners    = 8 dense vertex ids per leaf, corner order b=(bz<<2)|(by<<1)|bx.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include <cuda_runtime.h>

#include "svlf_b200.h"

namespace svlfb {

constexpr int kMaxLevels = 21;  // 21 bits per Morton axis

struct HostOctree {
    svlf_grid grid{};
    int leaf_level = 0;
    double cell_size = 0.0;  // extent / resolution
    std::vector<std::vector<uint64_t>> levels;  // sorted Morton codes, [0..leaf_level]
    std::vector<uint32_t> corner_ids;           // 8 per leaf
    uint32_t vertex_count = 0;
    size_t dropped_points = 0;

    // flattened node table for the device
    std::vector<uint32_t> node_first_child;  // per internal node
    std::vector<uint8_t> node_mask;
    std::vector<uint32_t> level_off;  // size leaf_level + 2

    static HostOctree build(std::span<const double> points_xyz, const svlf_grid& grid);
    static HostOctree from_leaves(std::vector<uint64_t> leaves, const svlf_grid& grid);

    const std::vector<uint64_t>& leaves() const { return levels[leaf_level]; }

  private:
    void finalize();
};

void validate_grid(const svlf_grid& g);

// The same build on the GPU from device-resident points (octree_build.cu);
// byte-identical result.
HostOctree build_octree_gpu(const svlf_grid& grid, const double* d_points, size_t n, cudaStream_t s);

// Morton helpers (reference include/svlf/morton.hpp:9-37 convention: x -> bit
// 3k, y -> 3k+1, z -> 3k+2).
inline uint64_t morton_spread3(uint64_t v) {
    v &= 0x1fffffULL;
    v = (v | v << 32) & 0x1f00000000ffffULL;
    v = (v | v << 16) & 0x1f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}
inline uint64_t morton_code(uint32_t x, uint32_t y, uint32_t z) {
    return morton_spread3(x) | morton_spread3(y) << 1 | morton_spread3(z) << 2;
}
inline uint32_t morton_gather3(uint64_t v) {
    v &= 0x1249249249249249ULL;
    v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ULL;
    v = (v ^ (v >> 4)) & 0x100f00f00f00f00fULL;
    v = (v ^ (v >> 8)) & 0x1f0000ff0000ffULL;
    v = (v ^ (v >> 16)) & 0x1f00000000ffffULL;
    v = (v ^ (v >> 32)) & 0x1fffffULL;
    return static_cast<uint32_t>(v);
}

}  // namespace svlfb
