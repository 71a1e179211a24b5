// C++ API over the C ABI: geometry helpers, camera, GridConfig and the
// SparseOctree value type (include/svlf/{geometry,camera,octree}.hpp).
//
// Reference interfaces mirrored: include/svlf/geometry.hpp:80 (ray_aabb),
// src/camera.cpp:8-40 (validate, make_lookat_camera), src/octree.cpp:20-28
// (GridConfig::validate), include/svlf/octree.hpp:39-94 (SparseOctree).
// The octree structure comes from the library (svlf_octree_build /
// from_leaves, host-side, bit-identical); traverse() is the GPU kernel.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>

#include "session.hpp"
#include "svlf/camera.hpp"
#include "svlf/morton.hpp"
#include "svlf/octree.hpp"

namespace svlf {

std::optional<Interval> ray_aabb(const Ray& ray, const Aabb& box) {
    Interval iv{0.0, std::numeric_limits<double>::infinity()};
    for (int a = 0; a < 3; ++a) {
        const double o = ray.origin[a], d = ray.dir[a];
        if (d == 0.0) {  // parallel to the slab: inside or missed
            if (o < box.lo[a] || o > box.hi[a]) return std::nullopt;
            continue;
        }
        const double inv = 1.0 / d;
        const double tl = (box.lo[a] - o) * inv, th = (box.hi[a] - o) * inv;
        iv.t0 = std::max(iv.t0, std::min(tl, th));
        iv.t1 = std::min(iv.t1, std::max(tl, th));
        if (iv.t1 < iv.t0) return std::nullopt;
    }
    return iv;
}

void Camera::validate() const {
    if (fx <= 0 || fy <= 0) throw std::invalid_argument("camera focal lengths must be positive");
    if (width == 0 || height == 0) throw std::invalid_argument("camera resolution must be positive");
    const double* m = camera_to_world.data();
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double g = m[i] * m[j] + m[4 + i] * m[4 + j] + m[8 + i] * m[8 + j];
            if (std::abs(g - (i == j ? 1.0 : 0.0)) > 1e-9)
                throw std::invalid_argument("camera rotation is not orthonormal");
        }
}

Camera make_lookat_camera(const Vec3& eye, const Vec3& target, uint32_t width, uint32_t height, double focal_px) {
    const Vec3 fwd = normalized(target - eye);
    const Vec3 up = std::abs(dot(fwd, Vec3(0, 0, 1))) > 0.999 ? Vec3(0, 1, 0) : Vec3(0, 0, 1);
    const Vec3 right = normalized(cross(fwd, up));
    const Vec3 down = cross(fwd, right);
    Camera c;
    c.width = width;
    c.height = height;
    c.fx = c.fy = focal_px;
    c.cx = width * 0.5;
    c.cy = height * 0.5;
    const Vec3 cols[4] = {right, down, fwd, eye};
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 4; ++k) c.camera_to_world[4 * r + k] = cols[k][r];
    c.camera_to_world[15] = 1.0;
    return c;
}

void GridConfig::validate() const {
    if (resolution < 2 || (resolution & (resolution - 1)))
        throw std::invalid_argument("resolution must be a power of two >= 2");
    const Vec3 e = scene_aabb.extent();
    if (!(e.x > 0) || !(e.y > 0) || !(e.z > 0)) throw std::invalid_argument("scene_aabb must have positive extent");
    const double tol = 1e-12 * std::max({e.x, e.y, e.z});
    if (std::abs(e.x - e.y) > tol || std::abs(e.x - e.z) > tol)
        throw std::invalid_argument("scene_aabb must be a cube");
}

// ---- SparseOctree ---------------------------------------------------------
struct SparseOctree::State {
    svlf_octree* h = nullptr;
    GridConfig config;
    int leaf_level = 0;
    uint32_t vertex_count = 0;
    size_t dropped = 0;
    double cell = 0;
    std::vector<std::vector<uint64_t>> levels;
    std::vector<uint32_t> corners;  // 8 per leaf

    ~State() {
        if (h) svlf_octree_destroy(h);
    }
};

namespace {

svlf_grid to_c(const GridConfig& g) {
    svlf_grid c{};
    c.resolution = g.resolution;
    c.dilation = g.dilation;
    for (int a = 0; a < 3; ++a) {
        c.lo[a] = g.scene_aabb.lo[a];
        c.hi[a] = g.scene_aabb.hi[a];
    }
    return c;
}

std::shared_ptr<const SparseOctree::State> adopt(svlf_octree* h, const GridConfig& cfg) {
    auto s = std::make_shared<SparseOctree::State>();
    s->h = h;
    s->config = cfg;
    svlf_octree_info info{};
    detail::check(svlf_octree_get_info(h, &info));
    s->leaf_level = info.leaf_level;
    s->vertex_count = info.vertex_count;
    s->dropped = info.dropped_points;
    s->cell = info.cell_size;
    s->levels.resize(size_t(info.leaf_level) + 1);
    for (int l = 0; l <= info.leaf_level; ++l) {
        s->levels[l].resize(info.level_size[l]);
        detail::check(svlf_octree_level_codes(h, l, s->levels[l].data()));
    }
    s->corners.resize(info.leaf_count * 8);
    detail::check(svlf_octree_corner_ids(h, s->corners.data()));
    return s;
}

const SparseOctree::State& need(const std::shared_ptr<const SparseOctree::State>& s) {
    if (!s) throw std::logic_error("empty SparseOctree");
    return *s;
}

}  // namespace

SparseOctree SparseOctree::build(std::span<const Vec3> points, const GridConfig& config) {
    config.validate();
    std::vector<double> xyz(points.size() * 3);
    for (size_t i = 0; i < points.size(); ++i) {
        xyz[3 * i] = points[i].x;
        xyz[3 * i + 1] = points[i].y;
        xyz[3 * i + 2] = points[i].z;
    }
    const svlf_grid g = to_c(config);
    svlf_octree* h = nullptr;
    detail::check(svlf_octree_build(nullptr, &g, xyz.data(), points.size(), &h));
    SparseOctree t;
    t.s_ = adopt(h, config);
    return t;
}

SparseOctree SparseOctree::from_leaves(std::vector<uint64_t> leaf_codes, const GridConfig& config) {
    config.validate();
    const svlf_grid g = to_c(config);
    svlf_octree* h = nullptr;
    detail::check(svlf_octree_from_leaves(nullptr, &g, leaf_codes.data(), leaf_codes.size(), &h));
    SparseOctree t;
    t.s_ = adopt(h, config);
    return t;
}

const GridConfig& SparseOctree::config() const {
    static const GridConfig empty{};
    return s_ ? s_->config : empty;
}
int SparseOctree::leaf_level() const { return s_ ? s_->leaf_level : 0; }
const std::vector<uint64_t>& SparseOctree::level_codes(int level) const {
    static const std::vector<uint64_t> none;
    if (!s_) return none;
    return s_->levels.at(size_t(level));
}
uint32_t SparseOctree::vertex_count() const { return s_ ? s_->vertex_count : 0; }
size_t SparseOctree::dropped_points() const { return s_ ? s_->dropped : 0; }
double SparseOctree::cell_size() const { return s_ ? s_->cell : 0.0; }
svlf_octree* SparseOctree::handle() const { return s_ ? s_->h : nullptr; }

Aabb SparseOctree::voxel_aabb(uint64_t voxel_id) const {
    const State& s = need(s_);
    uint32_t ix, iy, iz;
    morton_decode(voxel_id, ix, iy, iz);
    const Vec3 lo = s.config.scene_aabb.lo;
    const double h = s.cell;
    return Aabb{Vec3(lo.x + ix * h, lo.y + iy * h, lo.z + iz * h),
                Vec3(lo.x + (ix + 1) * h, lo.y + (iy + 1) * h, lo.z + (iz + 1) * h)};
}

std::optional<uint32_t> SparseOctree::leaf_index(uint64_t voxel_id) const {
    const auto& v = leaf_codes();
    auto it = std::lower_bound(v.begin(), v.end(), voxel_id);
    if (it == v.end() || *it != voxel_id) return std::nullopt;
    return uint32_t(it - v.begin());
}

std::array<uint32_t, 8> SparseOctree::corner_vertices(uint64_t voxel_id) const {
    const auto i = leaf_index(voxel_id);
    if (!i) throw std::out_of_range("unknown voxel id");
    std::array<uint32_t, 8> c;
    std::copy_n(s_->corners.begin() + size_t(*i) * 8, 8, c.begin());
    return c;
}

std::optional<uint64_t> SparseOctree::locate(const Vec3& p) const {
    const State& s = need(s_);
    if (!s.config.scene_aabb.contains(p)) return std::nullopt;
    const Vec3 lo = s.config.scene_aabb.lo;
    const uint32_t last = s.config.resolution - 1;
    auto cell = [&](double x, double l) { return std::min(uint32_t((x - l) / s.cell), last); };
    const uint64_t code = morton_encode(cell(p.x, lo.x), cell(p.y, lo.y), cell(p.z, lo.z));
    if (!leaf_index(code)) return std::nullopt;
    return code;
}

void SparseOctree::traverse_batch(std::span<const Ray> rays, std::vector<uint64_t>& offsets,
                                  std::vector<RayVoxelHit>& hits) const {
    const State& s = need(s_);
    const size_t n = rays.size();
    std::vector<double> r6(n * 6);
    for (size_t i = 0; i < n; ++i) {
        const Ray& r = rays[i];
        const double v[6] = {r.origin.x, r.origin.y, r.origin.z, r.dir.x, r.dir.y, r.dir.z};
        std::copy(v, v + 6, r6.begin() + 6 * i);
    }
    offsets.assign(n + 1, 0);
    std::vector<uint64_t> ids;
    std::vector<double> tin, tout, x12;
    size_t cap = std::max<size_t>(64, n * 4), total = 0;
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    svlf_ctx* ctx = b200::session_context();
    for (;;) {
        ids.resize(cap);
        tin.resize(cap);
        tout.resize(cap);
        x12.resize(cap * 6);
        const svlf_status st = svlf_traverse(ctx, s.h, r6.data(), n, offsets.data(), cap, ids.data(), tin.data(),
                                             tout.data(), x12.data(), &total);
        if (st == SVLF_ERR_CAPACITY && total > cap) {
            cap = total;
            continue;
        }
        detail::check(st);
        break;
    }
    hits.resize(total);
    for (size_t j = 0; j < total; ++j) {
        const double* x = &x12[6 * j];
        hits[j] = RayVoxelHit{ids[j], tin[j], tout[j], Vec3(x[0], x[1], x[2]), Vec3(x[3], x[4], x[5])};
    }
}

void SparseOctree::traverse(const Ray& ray, std::vector<RayVoxelHit>& out, TraversalScratch&) const {
    std::vector<uint64_t> off;
    std::vector<RayVoxelHit> h;
    traverse_batch(std::span<const Ray>(&ray, 1), off, h);
    out.insert(out.end(), h.begin(), h.end());
}

std::vector<RayVoxelHit> SparseOctree::traverse(const Ray& ray) const {
    std::vector<RayVoxelHit> out;
    TraversalScratch scratch;
    traverse(ray, out, scratch);
    return out;
}

}  // namespace svlf
