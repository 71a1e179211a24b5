// The reference's per-point / per-ray public operations, batched on the GPU
// (include/svlf/features.hpp:63-80, render.hpp:28-76, train.hpp:41):
// local_coords, interpolate / interpolate_backward (float and double
// volumes, any feature width), parameterize_ray, composite, the voxel
// bookkeeping of evaluate_voxel and eta_gt. The frame and train pipelines do
// not use these (they fuse the same arithmetic into their kernels); they
// back the drop-in single-ray API (render_ray, evaluate_voxel, surface_loss,
// ...) and its tests. Arithmetic follows the reference operand by operand
// with no contraction (nvcc -fmad=false and explicit _rn intrinsics), so
// single-point results are bit-identical to the reference built without FMA.
#include "device.cuh"

namespace svlfb {

namespace {

__device__ __forceinline__ void voxel_box(const DevOctree& T, uint64_t code, double* lo, double* hi) {
    cell_box(T, T.cell_size, morton_gather3_dev(code), morton_gather3_dev(code >> 1), morton_gather3_dev(code >> 2),
             lo, hi);
}

// leaf index of a voxel code (SparseOctree::leaf_index, src/octree.cpp:158-163)
__device__ __forceinline__ bool find_leaf(const DevOctree& T, uint64_t code, uint32_t& leaf) {
    uint32_t a = 0, b = T.n_leaves;
    while (a < b) {
        const uint32_t m = (a + b) >> 1;
        if (T.leaf_codes[m] < code) a = m + 1;
        else b = m;
    }
    if (a == T.n_leaves || T.leaf_codes[a] != code) return false;
    leaf = a;
    return true;
}

// local_coords (src/features.cpp:22-31): box check with 1e-7 slack, u = (p - lo) / h clamped
__device__ __forceinline__ bool local_u(const DevOctree& T, uint64_t code, const double* p, double* u) {
    double lo[3], hi[3];
    voxel_box(T, code, lo, hi);
#pragma unroll
    for (int a = 0; a < 3; ++a)
        if (!(p[a] >= dsub(lo[a], 1e-7) && p[a] <= dadd(hi[a], 1e-7))) return false;
#pragma unroll
    for (int a = 0; a < 3; ++a) u[a] = fmin(fmax(ddiv(dsub(p[a], lo[a]), T.cell_size), 0.0), 1.0);
    return true;
}

__device__ __forceinline__ void weights_d(const double* u, double* w) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const double wx = (b & 1) ? u[0] : dsub(1.0, u[0]);
        const double wy = (b & 2) ? u[1] : dsub(1.0, u[1]);
        const double wz = (b & 4) ? u[2] : dsub(1.0, u[2]);
        w[b] = dmul(dmul(wx, wy), wz);
    }
}

__device__ __forceinline__ float tadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double tadd(double a, double b) { return dadd(a, b); }
__device__ __forceinline__ float tmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double tmul(double a, double b) { return dmul(a, b); }

__global__ void k_local_coords(DevOctree T, const uint64_t* ids, const double* pts, size_t n, double* u_out,
                               int* err) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double u[3];
    if (!local_u(T, ids[i], pts + 3 * i, u)) {
        raise_error(err, kErrPointNotInVoxel);
        return;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) u_out[3 * i + a] = u[a];
}

// interpolate (src/features.cpp:33-47): out[d] = sum_b T(w_b) * row_b[d] in corner order
template <typename Tv>
__global__ void k_interpolate(DevOctree T, const Tv* vol, uint32_t rows, uint32_t dim, const uint64_t* ids,
                              const double* pts, size_t n, Tv* out, int* err) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double u[3];
    if (!local_u(T, ids[i], pts + 3 * i, u)) {
        raise_error(err, kErrPointNotInVoxel);
        return;
    }
    uint32_t leaf;
    if (!find_leaf(T, ids[i], leaf)) {
        raise_error(err, kErrUnknownVoxel);
        return;
    }
    double w[8];
    weights_d(u, w);
    Tv* o = out + i * dim;
    for (uint32_t d = 0; d < dim; ++d) o[d] = Tv(0);
    for (int b = 0; b < 8; ++b) {
        const uint32_t c = T.corners[8 * size_t(leaf) + b];
        if (c >= rows) {
            raise_error(err, kErrUnknownVoxel);
            return;
        }
        const Tv wb = Tv(w[b]);
        const Tv* row = vol + size_t(c) * dim;
        for (uint32_t d = 0; d < dim; ++d) o[d] = tadd(o[d], tmul(wb, row[d]));
    }
}

// interpolate_backward (src/features.cpp:49-84): grad rows += T(w_b) * upstream;
// pos_jac[d][a] = sum_b dw_b/du_a * z_b[d] * (1/h) in double
template <typename Tv>
__global__ void k_interpolate_backward(DevOctree T, const Tv* vol, uint32_t rows, uint32_t dim, const uint64_t* ids,
                                       const double* pts, size_t n, const Tv* up, Tv* grad, double* jac, int* err) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double u[3];
    if (!local_u(T, ids[i], pts + 3 * i, u)) {
        raise_error(err, kErrPointNotInVoxel);
        return;
    }
    uint32_t leaf;
    if (!find_leaf(T, ids[i], leaf)) {
        raise_error(err, kErrUnknownVoxel);
        return;
    }
    double w[8];
    weights_d(u, w);
    uint32_t cs[8];
    for (int b = 0; b < 8; ++b) {
        cs[b] = T.corners[8 * size_t(leaf) + b];
        if (cs[b] >= rows) {
            raise_error(err, kErrUnknownVoxel);
            return;
        }
    }
    const Tv* g = up + i * dim;
    for (int b = 0; b < 8; ++b) {
        const Tv wb = Tv(w[b]);
        Tv* grow = grad + size_t(cs[b]) * dim;
        for (uint32_t d = 0; d < dim; ++d) atomicAdd(grow + d, tmul(wb, g[d]));
    }
    if (!jac) return;
    const double inv_h = ddiv(1.0, T.cell_size);
    const double wx[2] = {dsub(1.0, u[0]), u[0]}, wy[2] = {dsub(1.0, u[1]), u[1]}, wz[2] = {dsub(1.0, u[2]), u[2]};
    const double dx[2] = {-1.0, 1.0};
    double* J = jac + i * size_t(dim) * 3;
    for (uint32_t k = 0; k < 3 * dim; ++k) J[k] = 0.0;
    for (int b = 0; b < 8; ++b) {
        const int bx = b & 1, by = (b >> 1) & 1, bz = (b >> 2) & 1;
        const double gw[3] = {dmul(dmul(dx[bx], wy[by]), wz[bz]), dmul(dmul(wx[bx], dx[by]), wz[bz]),
                              dmul(dmul(wx[bx], wy[by]), dx[bz])};
        const Tv* row = vol + size_t(cs[b]) * dim;
        for (uint32_t d = 0; d < dim; ++d) {
            const double z = double(row[d]);
#pragma unroll
            for (int a = 0; a < 3; ++a) J[d * 3 + a] = dadd(J[d * 3 + a], dmul(dmul(gw[a], z), inv_h));
        }
    }
}

// parameterize_ray (src/render.cpp:16-28) against an arbitrary box (lo xyz, hi xyz)
__global__ void k_parameterize(const double* rays, const double* boxes, size_t n, double* out, int* err) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    Ray r;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.o[a] = rays[6 * i + a];
        r.d[a] = rays[6 * i + 3 + a];
    }
    if (!parameterize_d(r, boxes + 6 * i, boxes + 6 * i + 3, out + 6 * i)) raise_error(err, kErrTangentRay);
}

// composite (src/render.cpp:65-87) per sample list, fp64 front to back; with
// t_s the expected depth of render_ray (:106-114): sum w_i t_s,i / alpha when
// alpha > kAlphaDepthThreshold, else 0
__global__ void k_composite_lists(const uint64_t* off, size_t lists, const double* taus, const double* colors,
                                  const double* t_s, double* color, double* alpha, double* depth, double* weights,
                                  int* err) {
    const size_t l = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (l >= lists) return;
    double c[3] = {0.0, 0.0, 0.0}, a = 0.0, tr = 1.0;
    for (uint64_t i = off[l]; i < off[l + 1]; ++i) {
        if (taus[i] < 0.0) {
            raise_error(err, kErrNegativeTau);
            return;
        }
        const double e = exp(-taus[i]);
        const double w = dmul(tr, dsub(1.0, e));
#pragma unroll
        for (int k = 0; k < 3; ++k) c[k] = dadd(c[k], dmul(w, colors[3 * i + k]));
        a = dadd(a, w);
        tr = dmul(tr, e);
        if (weights) weights[i] = w;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) color[3 * l + k] = c[k];
    alpha[l] = a;
    if (depth) {
        double acc = 0.0;
        if (a > 1e-4) {
            double tr2 = 1.0;
            for (uint64_t i = off[l]; i < off[l + 1]; ++i) {
                const double e = exp(-taus[i]);
                acc = dadd(acc, dmul(dmul(tr2, dsub(1.0, e)), t_s[i]));
                tr2 = dmul(tr2, e);
            }
            acc = ddiv(acc, a);
        }
        depth[l] = acc;
    }
}

__global__ void k_leaf_lookup(DevOctree T, const uint64_t* ids, size_t n, uint32_t* leaf, uint32_t* ray, int* err) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    uint32_t l = 0;
    if (!find_leaf(T, ids[i], l)) raise_error(err, kErrUnknownVoxel);
    leaf[i] = l;
    ray[i] = uint32_t(i);
}

// evaluate_voxel bookkeeping (src/render.cpp:44-49, :106-114): x_s = x1 eta + x2 (1 - eta) with eta
// the decoder's float promoted to double, and t_s = eta t_in + (1 - eta) t_out
__global__ void k_voxel_finish(const double* rays, const double* tin, const double* tout, const float* eta, size_t n,
                               double* xs, double* ts) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double e = double(eta[i]), ome = dsub(1.0, e);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double o = rays[6 * i + a], d = rays[6 * i + 3 + a];
        const double x1 = dadd(o, dmul(d, tin[i])), x2 = dadd(o, dmul(d, tout[i]));
        xs[3 * i + a] = dadd(dmul(x1, e), dmul(x2, ome));
    }
    ts[i] = dadd(dmul(e, tin[i]), dmul(ome, tout[i]));
}

// eta_gt (src/train.cpp:30-35)
__global__ void k_eta_gt(const double* tin, const double* tout, const double* depth, size_t n, double* out, int* err) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double d = depth[i];
    if (d < dsub(tin[i], 1e-6) || d > dadd(tout[i], 1e-6)) {
        raise_error(err, kErrSurfaceOutside);
        return;
    }
    out[i] = fmin(fmax(ddiv(dsub(tout[i], d), dsub(tout[i], tin[i])), 0.0), 1.0);
}

unsigned blocks(size_t n) { return unsigned((n + 127) / 128); }

}  // namespace

void launch_local_coords(const DevOctree& T, const uint64_t* ids, const double* pts, size_t n, double* u, int* err,
                         cudaStream_t s) {
    if (!n) return;
    k_local_coords<<<blocks(n), 128, 0, s>>>(T, ids, pts, n, u, err);
    note_launch();
}

template <typename Tv>
void launch_interpolate(const DevOctree& T, const Tv* vol, uint32_t rows, uint32_t dim, const uint64_t* ids,
                        const double* pts, size_t n, Tv* out, int* err, cudaStream_t s) {
    if (!n) return;
    k_interpolate<Tv><<<blocks(n), 128, 0, s>>>(T, vol, rows, dim, ids, pts, n, out, err);
    note_launch();
}

template <typename Tv>
void launch_interpolate_backward(const DevOctree& T, const Tv* vol, uint32_t rows, uint32_t dim, const uint64_t* ids,
                                 const double* pts, size_t n, const Tv* up, Tv* grad, double* jac, int* err,
                                 cudaStream_t s) {
    if (!n) return;
    k_interpolate_backward<Tv><<<blocks(n), 128, 0, s>>>(T, vol, rows, dim, ids, pts, n, up, grad, jac, err);
    note_launch();
}

template void launch_interpolate<float>(const DevOctree&, const float*, uint32_t, uint32_t, const uint64_t*,
                                        const double*, size_t, float*, int*, cudaStream_t);
template void launch_interpolate<double>(const DevOctree&, const double*, uint32_t, uint32_t, const uint64_t*,
                                         const double*, size_t, double*, int*, cudaStream_t);
template void launch_interpolate_backward<float>(const DevOctree&, const float*, uint32_t, uint32_t, const uint64_t*,
                                                 const double*, size_t, const float*, float*, double*, int*,
                                                 cudaStream_t);
template void launch_interpolate_backward<double>(const DevOctree&, const double*, uint32_t, uint32_t,
                                                  const uint64_t*, const double*, size_t, const double*, double*,
                                                  double*, int*, cudaStream_t);

void launch_parameterize(const double* rays, const double* boxes, size_t n, double* out, int* err, cudaStream_t s) {
    if (!n) return;
    k_parameterize<<<blocks(n), 128, 0, s>>>(rays, boxes, n, out, err);
    note_launch();
}

void launch_composite_lists(const uint64_t* off, size_t lists, const double* taus, const double* colors,
                            const double* t_s, double* color, double* alpha, double* depth, double* weights, int* err,
                            cudaStream_t s) {
    if (!lists) return;
    k_composite_lists<<<blocks(lists), 128, 0, s>>>(off, lists, taus, colors, t_s, color, alpha, depth, weights, err);
    note_launch();
}

void launch_leaf_lookup(const DevOctree& T, const uint64_t* ids, size_t n, uint32_t* leaf, uint32_t* ray, int* err,
                        cudaStream_t s) {
    if (!n) return;
    k_leaf_lookup<<<blocks(n), 128, 0, s>>>(T, ids, n, leaf, ray, err);
    note_launch();
}

void launch_voxel_finish(const double* rays, const double* tin, const double* tout, const float* eta, size_t n,
                         double* xs, double* ts, cudaStream_t s) {
    if (!n) return;
    k_voxel_finish<<<blocks(n), 128, 0, s>>>(rays, tin, tout, eta, n, xs, ts);
    note_launch();
}

void launch_eta_gt(const double* tin, const double* tout, const double* depth, size_t n, double* out, int* err,
                   cudaStream_t s) {
    if (!n) return;
    k_eta_gt<<<blocks(n), 128, 0, s>>>(tin, tout, depth, n, out, err);
    note_launch();
}

}  // namespace svlfb
