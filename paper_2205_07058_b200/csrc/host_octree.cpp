// Host octree build (reference semantics: src/octree.cpp:20-142).
//
// Occupancy: half-open quantization with the max face clamped into the last
// cell, Chebyshev dilation clipped to the grid, ancestors by code >> 3, and
// dense vertex ids ranked by the packed corner-lattice key (cz*lat+cy)*lat+cx.
// All outputs (codes per level, vertex ids, counts) are byte-identical to the
// reference's; tests/test_octree_parity.py checks that against the oracle.
#include "host_octree.hpp"

#include <algorithm>
#include <bit>
#include <cmath>

#include "common.hpp"

namespace svlfb {

void validate_grid(const svlf_grid& g) {  // GridConfig::validate, src/octree.cpp:20-28
    const uint32_t r = g.resolution;
    if (r < 2 || (r & (r - 1)) != 0)
        fail(SVLF_ERR_INVALID_ARGUMENT, "resolution must be a power of two >= 2");
    if (r > (1u << kMaxLevels)) fail(SVLF_ERR_INVALID_ARGUMENT, "resolution exceeds 2^21");
    const double ex = g.hi[0] - g.lo[0], ey = g.hi[1] - g.lo[1], ez = g.hi[2] - g.lo[2];
    if (ex <= 0 || ey <= 0 || ez <= 0)
        fail(SVLF_ERR_INVALID_ARGUMENT, "scene_aabb must have positive extent");
    const double tol = 1e-12 * std::max({ex, ey, ez});
    if (std::abs(ex - ey) > tol || std::abs(ex - ez) > tol)
        fail(SVLF_ERR_INVALID_ARGUMENT, "scene_aabb must be a cube");
}

namespace {

void sort_unique(std::vector<uint64_t>& v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
}

HostOctree empty_tree(const svlf_grid& grid) {
    HostOctree t;
    t.grid = grid;
    t.leaf_level = std::countr_zero(grid.resolution);
    t.cell_size = (grid.hi[0] - grid.lo[0]) / grid.resolution;
    t.levels.assign(t.leaf_level + 1, {});
    return t;
}

}  // namespace

HostOctree HostOctree::build(std::span<const double> pts, const svlf_grid& grid) {
    validate_grid(grid);
    HostOctree t = empty_tree(grid);
    const uint32_t res = grid.resolution;
    const double h = (grid.hi[0] - grid.lo[0]) / res;
    const size_t n = pts.size() / 3;

    std::vector<uint64_t> cells;
    cells.reserve(n);
    size_t dropped = 0;
    for (size_t i = 0; i < n; ++i) {
        const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
        bool inside = true;
        for (int a = 0; a < 3; ++a) inside = inside && p[a] >= grid.lo[a] && p[a] <= grid.hi[a];
        if (!inside) {
            ++dropped;
            continue;
        }
        uint32_t c[3];
        for (int a = 0; a < 3; ++a)
            c[a] = std::min(static_cast<uint32_t>((p[a] - grid.lo[a]) / h), res - 1);
        cells.push_back(morton_code(c[0], c[1], c[2]));
    }
    if (cells.empty()) fail(SVLF_ERR_RUNTIME, "empty occupancy");
    sort_unique(cells);

    if (grid.dilation > 0) {
        const int r = static_cast<int>(grid.dilation);
        const int ires = static_cast<int>(res);
        std::vector<uint64_t> grown;
        grown.reserve(cells.size() * static_cast<size_t>((2 * r + 1) * (2 * r + 1) * (2 * r + 1)));
        for (uint64_t code : cells) {
            const int x = morton_gather3(code), y = morton_gather3(code >> 1),
                      z = morton_gather3(code >> 2);
            for (int nz = std::max(0, z - r); nz <= std::min(ires - 1, z + r); ++nz)
                for (int ny = std::max(0, y - r); ny <= std::min(ires - 1, y + r); ++ny)
                    for (int nx = std::max(0, x - r); nx <= std::min(ires - 1, x + r); ++nx)
                        grown.push_back(morton_code(nx, ny, nz));
        }
        sort_unique(grown);
        cells.swap(grown);
    }
    t.dropped_points = dropped;
    t.levels[t.leaf_level] = std::move(cells);
    t.finalize();
    return t;
}

HostOctree HostOctree::from_leaves(std::vector<uint64_t> leaves, const svlf_grid& grid) {
    validate_grid(grid);
    if (leaves.empty()) fail(SVLF_ERR_RUNTIME, "empty occupancy");
    HostOctree t = empty_tree(grid);
    sort_unique(leaves);
    const uint64_t limit = uint64_t(1) << (3 * t.leaf_level);
    if (leaves.back() >= limit) fail(SVLF_ERR_INVALID_ARGUMENT, "leaf code outside the grid");
    t.levels[t.leaf_level] = std::move(leaves);
    t.finalize();
    return t;
}

void HostOctree::finalize() {
    // ancestors: parents of a sorted code list are sorted, so uniquing
    // consecutive duplicates suffices
    for (int l = leaf_level; l > 0; --l) {
        const auto& kids = levels[l];
        std::vector<uint64_t> parents;
        parents.reserve(kids.size() / 2 + 1);
        for (uint64_t c : kids)
            if (parents.empty() || parents.back() != (c >> 3)) parents.push_back(c >> 3);
        levels[l - 1] = std::move(parents);
    }

    // dense vertex ids over the leaf-corner lattice
    const auto& lv = leaves();
    const uint64_t lat = uint64_t(grid.resolution) + 1;
    std::vector<uint64_t> keys(lv.size() * 8);
    for (size_t i = 0; i < lv.size(); ++i) {
        const uint64_t x = morton_gather3(lv[i]), y = morton_gather3(lv[i] >> 1),
                       z = morton_gather3(lv[i] >> 2);
        for (uint32_t b = 0; b < 8; ++b)
            keys[8 * i + b] = ((z + ((b >> 2) & 1)) * lat + (y + ((b >> 1) & 1))) * lat + (x + (b & 1));
    }
    std::vector<uint64_t> lattice = keys;
    sort_unique(lattice);
    vertex_count = static_cast<uint32_t>(lattice.size());
    corner_ids.resize(keys.size());
    for (size_t i = 0; i < keys.size(); ++i)
        corner_ids[i] = static_cast<uint32_t>(
            std::lower_bound(lattice.begin(), lattice.end(), keys[i]) - lattice.begin());

    // flattened node table: each internal node's children are the run of
    // next-level codes with (code >> 3) == node code
    level_off.assign(leaf_level + 2, 0);
    for (int l = 0; l <= leaf_level; ++l) level_off[l + 1] = level_off[l] + uint32_t(levels[l].size());
    const size_t internal = level_off[leaf_level];
    node_first_child.assign(internal, 0);
    node_mask.assign(internal, 0);
    for (int l = 0; l < leaf_level; ++l) {
        const auto& parents = levels[l];
        const auto& kids = levels[l + 1];
        size_t k = 0;
        for (size_t p = 0; p < parents.size(); ++p) {
            const size_t g = level_off[l] + p;
            node_first_child[g] = level_off[l + 1] + uint32_t(k);
            uint8_t mask = 0;
            while (k < kids.size() && (kids[k] >> 3) == parents[p]) {
                mask |= uint8_t(1u << (kids[k] & 7));
                ++k;
            }
            node_mask[g] = mask;
        }
    }
}

}  // namespace svlfb
