// The reference's per-point / per-ray public operations over the C ABI's
// batched GPU entries (include/svlf/{features,render,train}.hpp):
// init_features, local_coords, interpolate(_backward), parameterize_ray,
// evaluate_voxel, composite, render_ray, eta_gt, surface_loss,
// volumetric_loss. Every evaluation runs on the GPU; this file converts
// between the reference's value types and the ABI's flat arrays.
#include <cmath>
#include <stdexcept>
#include <type_traits>

#include "session.hpp"
#include "svlf/features.hpp"
#include "svlf/render.hpp"
#include "svlf/rng.hpp"
#include "svlf/train.hpp"

namespace svlf {

namespace {

svlf_octree* tree_handle(const SparseOctree& t) {
    svlf_octree* h = t.handle();
    if (!h) throw std::invalid_argument("octree is empty");
    return h;
}

template <typename T>
constexpr svlf_dtype dtype_of() {
    return sizeof(T) == 4 ? SVLF_DTYPE_F32 : SVLF_DTYPE_F64;
}

}  // namespace

// src/features.cpp:10-20 (host generator, like init_model's streams)
FeatureVolume init_features(uint32_t vertex_count, uint32_t dim, uint64_t seed) {
    if (vertex_count < 1 || dim < 1) throw std::invalid_argument("vertex_count and dim must be >= 1");
    FeatureVolume v;
    v.dim = dim;
    v.data.resize(size_t(vertex_count) * dim);
    v.grad.assign(v.data.size(), 0.0f);
    const double bound = 1.0 / std::sqrt(static_cast<double>(dim));
    Rng rng(seed);
    for (float& x : v.data) x = static_cast<float>(rng.uniform(-bound, bound));
    return v;
}

Vec3 local_coords(const SparseOctree& octree, uint64_t voxel_id, const Vec3& point) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    const double p[3] = {point.x, point.y, point.z};
    double u[3];
    detail::check(svlf_local_coords(b200::session_context(), tree_handle(octree), &voxel_id, p, 1, u));
    return Vec3{u[0], u[1], u[2]};
}

template <typename T>
void interpolate(const FeatureVolumeT<T>& volume, const SparseOctree& octree, uint64_t voxel_id, const Vec3& point,
                 T* out) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    const double p[3] = {point.x, point.y, point.z};
    detail::check(svlf_interpolate(b200::session_context(), tree_handle(octree), dtype_of<T>(), volume.data.data(),
                                   uint32_t(volume.rows()), volume.dim, &voxel_id, p, 1, out));
}

template <typename T>
void interpolate_backward(const FeatureVolumeT<T>& volume, const SparseOctree& octree, uint64_t voxel_id,
                          const Vec3& point, const T* upstream, T* grad_buf, double* pos_jac) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    const double p[3] = {point.x, point.y, point.z};
    detail::check(svlf_interpolate_backward(b200::session_context(), tree_handle(octree), dtype_of<T>(),
                                            volume.data.data(), uint32_t(volume.rows()), volume.dim, &voxel_id, p, 1,
                                            upstream, grad_buf, pos_jac));
}

template void interpolate<float>(const FeatureVolumeT<float>&, const SparseOctree&, uint64_t, const Vec3&, float*);
template void interpolate<double>(const FeatureVolumeT<double>&, const SparseOctree&, uint64_t, const Vec3&,
                                  double*);
template void interpolate_backward<float>(const FeatureVolumeT<float>&, const SparseOctree&, uint64_t, const Vec3&,
                                          const float*, float*, double*);
template void interpolate_backward<double>(const FeatureVolumeT<double>&, const SparseOctree&, uint64_t,
                                           const Vec3&, const double*, double*, double*);

RayParam6 parameterize_ray(const Ray& ray, const Aabb& box) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    const double r[6] = {ray.origin.x, ray.origin.y, ray.origin.z, ray.dir.x, ray.dir.y, ray.dir.z};
    const double b[6] = {box.lo.x, box.lo.y, box.lo.z, box.hi.x, box.hi.y, box.hi.z};
    double q[6];
    detail::check(svlf_parameterize_rays(b200::session_context(), r, b, 1, q));
    return RayParam6{{q[0], q[1], q[2]}, {q[3], q[4], q[5]}};
}

namespace {

// the voxel samples of `hits` along `ray` (one batched GPU evaluation)
std::vector<VoxelSample> evaluate_hits(const SvlfModel& model, std::span<const RayVoxelHit> hits, const Ray& ray,
                                       std::vector<double>* t_s = nullptr) {
    const size_t n = hits.size();
    std::vector<VoxelSample> out(n);
    if (!n) return out;
    std::vector<double> rays(6 * n), tin(n), tout(n), tau(n), eta(n), xs(3 * n), ts(n), col(3 * n);
    std::vector<uint64_t> ids(n);
    for (size_t i = 0; i < n; ++i) {
        const double r[6] = {ray.origin.x, ray.origin.y, ray.origin.z, ray.dir.x, ray.dir.y, ray.dir.z};
        std::copy(r, r + 6, rays.begin() + 6 * i);
        ids[i] = hits[i].voxel_id;
        tin[i] = hits[i].t_in;
        tout[i] = hits[i].t_out;
    }
    detail::check(svlf_evaluate_voxels(b200::session_context(), detail::device_model(model), rays.data(), ids.data(),
                                       tin.data(), tout.data(), n, tau.data(), eta.data(), xs.data(), ts.data(),
                                       col.data()));
    for (size_t i = 0; i < n; ++i) {
        VoxelSample& s = out[i];
        s.voxel_id = ids[i];
        s.t_in = tin[i];
        s.t_out = tout[i];
        s.tau = tau[i];
        s.eta = eta[i];
        s.x_s = Vec3{xs[3 * i], xs[3 * i + 1], xs[3 * i + 2]};
        for (int k = 0; k < 3; ++k) s.color[k] = col[3 * i + k];
    }
    if (t_s) *t_s = std::move(ts);
    return out;
}

}  // namespace

template <typename T>
VoxelSample evaluate_voxel(const SvlfModelT<T>& model, const RayVoxelHit& hit, const Ray& ray,
                           QueryCounters* counters) {
    static_assert(std::is_same_v<T, float>, "the device path is fp32");
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    VoxelSample s = evaluate_hits(model, {&hit, 1}, ray)[0];
    if (counters) {
        counters->thickness_queries++;
        counters->color_queries++;
    }
    return s;
}
template VoxelSample evaluate_voxel<float>(const SvlfModel&, const RayVoxelHit&, const Ray&, QueryCounters*);

CompositeResult composite(std::span<const double> taus, std::span<const std::array<double, 3>> colors,
                          std::vector<double>* weights) {
    if (taus.size() != colors.size()) throw std::invalid_argument("composite size mismatch");
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    const uint64_t off[2] = {0, taus.size()};
    CompositeResult r;
    std::vector<double> w(taus.size());
    detail::check(svlf_composite(b200::session_context(), off, 1, taus.data(), colors.empty() ? nullptr : colors[0].data(),
                                 nullptr, r.color, &r.alpha, nullptr, weights ? w.data() : nullptr));
    if (weights) *weights = std::move(w);
    return r;
}

template <typename T>
RenderOutput render_ray(const SvlfModelT<T>& model, const Ray& ray, QueryCounters* counters) {
    static_assert(std::is_same_v<T, float>, "the device path is fp32");
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    const std::vector<RayVoxelHit> hits = model.octree.traverse(ray);
    const size_t n = hits.size();
    if (counters) counters->traversal_hits += static_cast<long long>(n);
    RenderOutput out;
    std::vector<double> ts;
    out.samples = evaluate_hits(model, hits, ray, &ts);
    if (counters) {
        counters->thickness_queries += static_cast<long long>(n);
        counters->color_queries += static_cast<long long>(n);
    }
    std::vector<double> taus(n), cols(3 * n);
    for (size_t i = 0; i < n; ++i) {
        taus[i] = out.samples[i].tau;
        for (int k = 0; k < 3; ++k) cols[3 * i + k] = out.samples[i].color[k];
    }
    // expected depth: sum_i w_i t_s,i / alpha above kAlphaDepthThreshold (src/render.cpp:106-114)
    const uint64_t off[2] = {0, n};
    detail::check(svlf_composite(b200::session_context(), off, 1, taus.data(), cols.data(), ts.data(), out.color,
                                 &out.alpha, &out.expected_depth, nullptr));
    return out;
}
template RenderOutput render_ray<float>(const SvlfModel&, const Ray&, QueryCounters*);

double eta_gt(const RayVoxelHit& hit, double depth_gt) {
    std::lock_guard<std::recursive_mutex> lk(detail::session_mutex());
    double e = 0;
    detail::check(svlf_eta_gt(b200::session_context(), &hit.t_in, &hit.t_out, &depth_gt, 1, &e));
    return e;
}

template <typename T>
double surface_loss(const SvlfModelT<T>& model, const RaySupervision& sup, const LossWeights& lw, ModelGradsT<T>* grads,
                    LossStats* stats) {
    static_assert(std::is_same_v<T, float>, "the device path is fp32");
    return loss_grads(model, {&sup, 1}, LossMode::Surface, false, lw, grads, stats);
}
template double surface_loss<float>(const SvlfModel&, const RaySupervision&, const LossWeights&, ModelGrads*,
                                    LossStats*);

template <typename T>
double volumetric_loss(const SvlfModelT<T>& model, const RaySupervision& sup, const LossWeights& lw,
                       bool color_frozen, ModelGradsT<T>* grads, LossStats* stats) {
    static_assert(std::is_same_v<T, float>, "the device path is fp32");
    return loss_grads(model, {&sup, 1}, LossMode::Volumetric, color_frozen, lw, grads, stats);
}
template double volumetric_loss<float>(const SvlfModel&, const RaySupervision&, const LossWeights&, bool, ModelGrads*,
                                       LossStats*);

}  // namespace svlf
