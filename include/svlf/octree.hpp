// svlf/octree.hpp — sparse voxel octree of the B200 SVLF C++ API.
//
// Same public surface as the reference SparseOctree (reference
// include/svlf/octree.hpp:13-99): build/from_leaves/level queries/corner ids/
// locate/traverse. The structure is built on the host by the library
// (bit-identical codes and vertex ids, csrc/host_octree.cpp) and mirrored to
// HBM on first device use; traverse() runs the GPU traversal kernel through
// the C ABI (svlf_traverse) and returns the reference's hit order, bit-exact
// against the reference built without FMA contraction.
//
// SparseOctree is a cheap-to-copy value: copies share one immutable
// library octree (svlf_octree*), which also keys the device mirror.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "svlf/geometry.hpp"

struct svlf_octree;

namespace svlf {

struct GridConfig {
    uint32_t resolution = 128;              // voxels per axis, power of two >= 2
    Aabb scene_aabb{{0, 0, 0}, {1, 1, 1}};  // a cube
    uint32_t dilation = 1;                  // Chebyshev dilation radius of the occupancy
    void validate() const;                  // std::invalid_argument on violation
};

struct RayVoxelHit {
    uint64_t voxel_id = 0;  // leaf Morton code
    double t_in = 0.0, t_out = 0.0;
    Vec3 x1, x2;  // ray.at(t_in), ray.at(t_out)
};

// Kept for signature compatibility (the GPU traversal needs no host stack).
struct TraversalScratch {
    std::vector<std::pair<int, uint64_t>> stack;
};

class SparseOctree {
  public:
    SparseOctree() = default;

    // "empty occupancy" (std::runtime_error) when no point lands in the box.
    static SparseOctree build(std::span<const Vec3> points, const GridConfig& config);
    static SparseOctree from_leaves(std::vector<uint64_t> leaf_codes, const GridConfig& config);

    const GridConfig& config() const;
    int leaf_level() const;
    const std::vector<uint64_t>& level_codes(int level) const;
    const std::vector<uint64_t>& leaf_codes() const { return level_codes(leaf_level()); }
    size_t leaf_count() const { return leaf_codes().size(); }
    uint32_t vertex_count() const;
    size_t dropped_points() const;
    double cell_size() const;

    Aabb voxel_aabb(uint64_t voxel_id) const;
    Vec3 voxel_center(uint64_t voxel_id) const { return voxel_aabb(voxel_id).center(); }
    std::optional<uint32_t> leaf_index(uint64_t voxel_id) const;
    std::array<uint32_t, 8> corner_vertices(uint64_t voxel_id) const;  // std::out_of_range if unknown
    std::optional<uint64_t> locate(const Vec3& point) const;

    // Hits sorted by (t_in, code); kept iff t_out - t_in > 1e-12. GPU.
    std::vector<RayVoxelHit> traverse(const Ray& ray) const;
    void traverse(const Ray& ray, std::vector<RayVoxelHit>& out, TraversalScratch& scratch) const;
    // Batched form (the natural GPU entry): CSR offsets[n+1] into `hits`.
    void traverse_batch(std::span<const Ray> rays, std::vector<uint64_t>& offsets,
                        std::vector<RayVoxelHit>& hits) const;

    // library handle (nullptr for a default-constructed octree)
    svlf_octree* handle() const;

    struct State;

  private:
    std::shared_ptr<const State> s_;
};

inline SparseOctree build_octree(std::span<const Vec3> points, const GridConfig& config) {
    return SparseOctree::build(points, config);
}

}  // namespace svlf
