// Sparse-voxel-octree ray traversal (reference SparseOctree::traverse,
// src/octree.cpp:192-235), one ray per thread, two passes:
//   count: walk the tree, count kept leaves per ray (and materialise camera rays)
//   scan:  CSR row pointer (cub::DeviceScan)
//   emit:  walk again, write (leaf index, t_in, t_out, ray) into the ray's
//          segment, then an in-place insertion sort by (t_in, leaf index).
//
// The walk visits children in front-to-back octant order (octant i ^ sign
// mask of the direction), which leaves a segment almost sorted, so the
// insertion sort is ~linear. Leaf index order equals Morton order (leaves
// are stored sorted), so the (t_in, index) sort equals the reference's
// (t_in, code) total order. The set of kept leaves is order-independent: a
// node is tested iff its parent was hit, with the reference's exact box
// formula and slab test (geom.cuh), so ids, order and t values match the
// reference bit for bit.
#include <cub/device/device_scan.cuh>

#include "device.cuh"

namespace svlfb {

namespace {

constexpr double kMinHitSpan = 1e-12;  // tie rule, src/octree.cpp:16

// Depth-first walk calling on_leaf(leaf_index, t0, t1) for every kept leaf.
template <typename OnLeaf>
__device__ __forceinline__ void walk(const DevOctree& T, const RayPre& p, OnLeaf&& on_leaf) {
    double lo[3], hi[3], t0, t1;
    cell_box(T, T.cell[0], 0, 0, 0, lo, hi);
    if (!slab_test(p, lo, hi, t0, t1)) return;

    const uint32_t s = (p.r.d[0] < 0.0 ? 1u : 0u) | (p.r.d[1] < 0.0 ? 2u : 0u) | (p.r.d[2] < 0.0 ? 4u : 0u);
    uint32_t st_node[kMaxLevelsDev], st_x[kMaxLevelsDev], st_y[kMaxLevelsDev], st_z[kMaxLevelsDev];
    uint32_t st_it[kMaxLevelsDev];
    int lvl = 0;
    st_node[0] = 0;
    st_x[0] = st_y[0] = st_z[0] = 0;
    st_it[0] = 0;
    const int L = T.L;
    while (lvl >= 0) {
        const uint32_t it = st_it[lvl];
        if (it == 8) {
            --lvl;
            continue;
        }
        st_it[lvl] = it + 1;
        const uint32_t oct = it ^ s;
        const uint32_t g = st_node[lvl];
        const uint32_t m = T.mask[g];
        if (!((m >> oct) & 1u)) continue;
        const uint32_t child = T.first_child[g] + __popc(m & ((1u << oct) - 1u));
        const uint32_t cx = 2u * st_x[lvl] + (oct & 1u);
        const uint32_t cy = 2u * st_y[lvl] + ((oct >> 1) & 1u);
        const uint32_t cz = 2u * st_z[lvl] + ((oct >> 2) & 1u);
        const int cl = lvl + 1;
        cell_box(T, T.cell[cl], cx, cy, cz, lo, hi);
        if (!slab_test(p, lo, hi, t0, t1)) continue;
        if (cl == L) {
            if (dsub(t1, t0) > kMinHitSpan) on_leaf(child - T.level_off[L], t0, t1);
            continue;
        }
        lvl = cl;
        st_node[lvl] = child;
        st_x[lvl] = cx;
        st_y[lvl] = cy;
        st_z[lvl] = cz;
        st_it[lvl] = 0;
    }
}

__device__ __forceinline__ Ray load_ray(const double* rays, size_t i) {
    Ray r;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.o[a] = rays[6 * i + a];
        r.d[a] = rays[6 * i + 3 + a];
    }
    return r;
}

template <bool kCamera>
__global__ void __launch_bounds__(128) k_traverse_count(DevOctree T, DevCamera cam, uint32_t row0,
                                                        double* rays, uint32_t n, uint32_t* counts) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Ray r;
    if constexpr (kCamera) {
        const uint64_t px = uint64_t(row0) * cam.width + i;
        r = pixel_ray(cam, uint32_t(px % cam.width), uint32_t(px / cam.width));
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            rays[6 * size_t(i) + a] = r.o[a];
            rays[6 * size_t(i) + 3 + a] = r.d[a];
        }
    } else {
        r = load_ray(rays, i);
    }
    const RayPre p = precompute(r);
    uint32_t c = 0;
    walk(T, p, [&](uint32_t, double, double) { ++c; });
    counts[i] = c;
}

__global__ void __launch_bounds__(128) k_traverse_emit(DevOctree T, const double* rays, uint32_t n,
                                                       const uint32_t* offsets, uint32_t* hit_leaf,
                                                       double* hit_tin, double* hit_tout,
                                                       uint32_t* hit_ray) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t base = offsets[i], end = offsets[i + 1];
    if (base == end) return;
    const RayPre p = precompute(load_ray(rays, i));
    uint32_t k = base;
    walk(T, p, [&](uint32_t leaf, double t0, double t1) {
        hit_leaf[k] = leaf;
        hit_tin[k] = t0;
        hit_tout[k] = t1;
        hit_ray[k] = i;
        ++k;
    });
    // insertion sort of the (nearly sorted) segment by (t_in, leaf index)
    for (uint32_t a = base + 1; a < end; ++a) {
        const double ti = hit_tin[a], to = hit_tout[a];
        const uint32_t lf = hit_leaf[a];
        uint32_t b = a;
        while (b > base) {
            const double tp = hit_tin[b - 1];
            const uint32_t lp = hit_leaf[b - 1];
            if (tp < ti || (tp == ti && lp < lf)) break;
            hit_tin[b] = tp;
            hit_tout[b] = hit_tout[b - 1];
            hit_leaf[b] = lp;
            --b;
        }
        hit_tin[b] = ti;
        hit_tout[b] = to;
        hit_leaf[b] = lf;
    }
}

__global__ void k_gather_codes(const uint64_t* codes, const uint32_t* leaf, uint64_t* out, size_t n) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = codes[leaf[i]];
}

// x1 = ray.at(t_in), x2 = ray.at(t_out) (src/octree.cpp:216-217)
__global__ void k_hit_points(const double* rays, const uint32_t* hit_ray, const double* tin,
                             const double* tout, double* x12, size_t n) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const Ray r = load_ray(rays, hit_ray[i]);
    double p[3];
    ray_at(r, tin[i], p);
    for (int a = 0; a < 3; ++a) x12[6 * i + a] = p[a];
    ray_at(r, tout[i], p);
    for (int a = 0; a < 3; ++a) x12[6 * i + 3 + a] = p[a];
}

}  // namespace

void launch_gather_leaf_codes(const uint64_t* leaf_codes, const uint32_t* hit_leaf, uint64_t* out, size_t n,
                              cudaStream_t s) {
    if (!n) return;
    k_gather_codes<<<unsigned((n + 255) / 256), 256, 0, s>>>(leaf_codes, hit_leaf, out, n);
    note_launch();
}

void launch_hit_points(const double* rays, const uint32_t* hit_ray, const double* tin, const double* tout,
                       double* x12, size_t n, cudaStream_t s) {
    if (!n) return;
    k_hit_points<<<unsigned((n + 255) / 256), 256, 0, s>>>(rays, hit_ray, tin, tout, x12, n);
    note_launch();
}

void launch_traverse_count(const DevOctree& T, const DevCamera* cam, uint32_t row0, double* rays,
                           uint32_t n, uint32_t* counts, cudaStream_t s) {
    if (n == 0) return;
    const uint32_t blocks = (n + 127) / 128;
    if (cam)
        k_traverse_count<true><<<blocks, 128, 0, s>>>(T, *cam, row0, rays, n, counts);
    else
        k_traverse_count<false><<<blocks, 128, 0, s>>>(T, DevCamera{}, 0, rays, n, counts);
    note_launch();
}

void launch_traverse_emit(const DevOctree& T, const double* rays, uint32_t n, const uint32_t* offsets,
                          uint32_t* hit_leaf, double* hit_tin, double* hit_tout, uint32_t* hit_ray,
                          cudaStream_t s) {
    if (n == 0) return;
    k_traverse_emit<<<(n + 127) / 128, 128, 0, s>>>(T, rays, n, offsets, hit_leaf, hit_tin, hit_tout,
                                                     hit_ray);
    note_launch();
}

size_t scan_temp_bytes(uint32_t n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), int(n));
    return bytes;
}

void launch_exclusive_scan(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out,
                           uint32_t n, cudaStream_t s) {
    SVLF_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, int(n), s));
    note_launch();
}

}  // namespace svlfb
