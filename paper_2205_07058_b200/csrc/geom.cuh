// Device-side geometry shared by the traversal, decode and train kernels.
//
// Bit-exactness rule: every fp64 expression is written with
// explicit round-to-nearest intrinsics in the reference's operand order, so
// no multiply-add is ever contracted (the library is also compiled with
// -fmad=false). With that, ray generation, box bounds, slab tests and hit
// points are bit-identical to the reference built with -ffp-contract=off.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

namespace svlfb {

constexpr int kMaxLevelsDev = 21;

// Read-only device mirror of a HostOctree (see host_octree.hpp for layout).
struct DevOctree {
    const uint2* nodes;           // per internal node: {first child (global index), child mask}
    const uint32_t* corners;      // 8 per leaf
    const uint64_t* leaf_codes;   // sorted
    uint32_t level_off[kMaxLevelsDev + 2];
    double cell[kMaxLevelsDev + 1];  // extent / (1u << level), src/octree.cpp:205
    double lo[3];
    double cell_size;                // extent / resolution (voxel_aabb, local_coords)
    double inv_cell_pow2;            // 1 / cell_size when cell_size is a power of two, else 0
    double hi[3];
    int L;
    uint32_t res;
    uint32_t n_leaves;
};

struct Ray {
    double o[3];
    double d[3];
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// dot(a, b) = a.x*b.x + a.y*b.y + a.z*b.z, left to right (geometry.hpp:34)
__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return dadd(dadd(dmul(a[0], b[0]), dmul(a[1], b[1])), dmul(a[2], b[2]));
}

// origin + dir * t (geometry.hpp:56)
__device__ __forceinline__ void ray_at(const Ray& r, double t, double* p) {
#pragma unroll
    for (int a = 0; a < 3; ++a) p[a] = dadd(r.o[a], dmul(r.d[a], t));
}

// Camera::pixel_ray (camera.hpp:26-29): pixel centre, row-major c2w rotation,
// normalized() = three true divisions by sqrt(dot(v, v)).
// width = the row length of the ray index space (the image width, or the tile
// width in tile-interleaved mode); tiles_world != 0 selects the interleaved
// mapping of cam_pixel.
struct DevCamera {
    double fx, fy, cx, cy;
    double m[16];
    uint32_t width, height;
    uint32_t tile_w = 0, tile_h = 0, tiles_x = 0, tiles_rank = 0, tiles_world = 0;
};

// Pixel of ray index gi of a pass over rows [row0, ...) of the ray index space.
// Plain: pixel (gi % width, row0 + gi / width). Tile-interleaved (multi-GPU
// render of one frame): the image is cut into tile_w x tile_h tiles numbered in
// raster order and rank r owns tiles r, r + world, r + 2 world, ...; its index
// space stacks them vertically (tile j at rows j*tile_h ..), so every 8 x 4
// traversal block stays inside one tile.
__device__ __forceinline__ void cam_pixel(const DevCamera& c, uint32_t gi, uint32_t row0, uint32_t& ix,
                                          uint32_t& iy) {
    const uint32_t vx = gi % c.width, vy = row0 + gi / c.width;
    if (c.tiles_world == 0) {
        ix = vx;
        iy = vy;
        return;
    }
    const uint32_t j = vy / c.tile_h, t = c.tiles_rank + c.tiles_world * j;
    ix = (t % c.tiles_x) * c.tile_w + vx;
    iy = (t / c.tiles_x) * c.tile_h + vy % c.tile_h;
}

__device__ __forceinline__ Ray pixel_ray(const DevCamera& c, uint32_t ix, uint32_t iy) {
    const double v[3] = {ddiv(dsub(dadd(double(ix), 0.5), c.cx), c.fx),
                         ddiv(dsub(dadd(double(iy), 0.5), c.cy), c.fy), 1.0};
    double r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        r[i] = dadd(dadd(dmul(c.m[4 * i], v[0]), dmul(c.m[4 * i + 1], v[1])), dmul(c.m[4 * i + 2], v[2]));
    const double n = __dsqrt_rn(dot3(r, r));
    Ray out;
    out.o[0] = c.m[3];
    out.o[1] = c.m[7];
    out.o[2] = c.m[11];
#pragma unroll
    for (int i = 0; i < 3; ++i) out.d[i] = ddiv(r[i], n);
    return out;
}

// Ray with the per-axis reciprocal hoisted: 1.0/d is the same IEEE result in
// every ray_aabb call of a ray, so computing it once is bit-neutral.
struct RayPre {
    Ray r;
    double inv[3];
};

__device__ __forceinline__ RayPre precompute(const Ray& r) {
    RayPre p;
    p.r = r;
#pragma unroll
    for (int a = 0; a < 3; ++a) p.inv[a] = r.d[a] == 0.0 ? 0.0 : ddiv(1.0, r.d[a]);
    return p;
}

// ray_aabb, src/geometry.cpp:5-26: slab test clipped to t >= 0; a zero
// direction component is an inside-the-slab test; reject iff t1 < t0.
__device__ __forceinline__ bool slab_test(const RayPre& p, const double* lo, const double* hi,
                                          double& t0, double& t1) {
    t0 = 0.0;
    t1 = CUDART_INF;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double o = p.r.o[a];
        if (p.r.d[a] == 0.0) {
            if (o < lo[a] || o > hi[a]) return false;
            continue;
        }
        double ta = dmul(dsub(lo[a], o), p.inv[a]);
        double tb = dmul(dsub(hi[a], o), p.inv[a]);
        if (ta > tb) {
            const double s = ta;
            ta = tb;
            tb = s;
        }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t1 < t0) return false;
    }
    return true;
}

// Cell box at a level from integer coordinates: lo + x*cell, lo + (x+1)*cell
// (src/octree.cpp:205-210; voxel_aabb, :144-152 at the leaf level).
__device__ __forceinline__ void cell_box(const DevOctree& T, double cell, uint32_t x, uint32_t y,
                                         uint32_t z, double* lo, double* hi) {
    const uint32_t c[3] = {x, y, z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = dadd(T.lo[a], dmul(double(c[a]), cell));
        hi[a] = dadd(T.lo[a], dmul(double(c[a] + 1u), cell));
    }
}

__device__ __forceinline__ uint32_t morton_gather3_dev(uint64_t v) {
    v &= 0x1249249249249249ULL;
    v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ULL;
    v = (v ^ (v >> 4)) & 0x100f00f00f00f00fULL;
    v = (v ^ (v >> 8)) & 0x1f0000ff0000ffULL;
    v = (v ^ (v >> 16)) & 0x1f00000000ffffULL;
    v = (v ^ (v >> 32)) & 0x1fffffULL;
    return uint32_t(v);
}

__device__ __forceinline__ void leaf_box(const DevOctree& T, uint32_t leaf, double* lo, double* hi) {
    const uint64_t code = T.leaf_codes[leaf];
    cell_box(T, T.cell_size, morton_gather3_dev(code), morton_gather3_dev(code >> 1),
             morton_gather3_dev(code >> 2), lo, hi);
}

// ---- per-hit geometry (fp64, reference operand order) --------------------

// parameterize_ray, src/render.cpp:16-28: the RayParam6 in double (p1, p2).
// Returns false on "tangent ray".
__device__ __forceinline__ bool parameterize_d(const Ray& r, const double* lo, const double* hi, double* q) {
    double c[3], oc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        c[a] = dmul(dadd(lo[a], hi[a]), 0.5);
        oc[a] = dsub(r.o[a], c[a]);
    }
    // 0.5 * sqrt(3.0): the correctly rounded sqrt(3) is 0x3FFBB67AE8584CAA
    constexpr double kHalfSqrt3 = 0.5 * 1.7320508075688772;
    const double radius = dmul(kHalfSqrt3, dsub(hi[0], lo[0]));
    const double b = dot3(oc, r.d);
    const double cc = dsub(dot3(oc, oc), dmul(radius, radius));
    const double disc = dsub(dmul(b, b), cc);
    if (disc < 1e-14) return false;
    const double s = __dsqrt_rn(disc);
    double p1[3], p2[3];
    ray_at(r, dsub(-b, s), p1);
    ray_at(r, dadd(-b, s), p2);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        p1[a] = dsub(p1[a], c[a]);
        p2[a] = dsub(p2[a], c[a]);
    }
    const double n1 = __dsqrt_rn(dot3(p1, p1)), n2 = __dsqrt_rn(dot3(p2, p2));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        q[a] = ddiv(p1[a], n1);
        q[3 + a] = ddiv(p2[a], n2);
    }
    return true;
}

// ... cast to the MLP's float input rows (RayParam6::write, render.hpp:16-24)
__device__ __forceinline__ bool parameterize(const Ray& r, const double* lo, const double* hi, float* r6) {
    double q[6];
    if (!parameterize_d(r, lo, hi, q)) return false;
#pragma unroll
    for (int a = 0; a < 6; ++a) r6[a] = float(q[a]);
    return true;
}

// x / cell_size. When the cell size is a power of two (the unit scene box
// with a power-of-two resolution, and many others) the division is an exact
// scaling, identical bit for bit to the multiplication by the exact
// reciprocal, which is much cheaper in fp64.
__device__ __forceinline__ double div_cell(const DevOctree& T, double x) {
    return T.inv_cell_pow2 != 0.0 ? dmul(x, T.inv_cell_pow2) : ddiv(x, T.cell_size);
}

// local_coords + trilinear_weights (features.cpp:22-31, features.hpp:13-21).
// Returns false on "point not in voxel". The clamped local coordinates are
// also returned when `u_out` is given.
__device__ __forceinline__ bool trilinear_at(const double* p, const double* lo, const double* hi,
                                             const DevOctree& T, float* w, double* u_out = nullptr) {
    double u[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!(p[a] >= dsub(lo[a], 1e-7) && p[a] <= dadd(hi[a], 1e-7))) return false;
        u[a] = fmin(fmax(div_cell(T, dsub(p[a], lo[a])), 0.0), 1.0);
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const double wx = (b & 1) ? u[0] : dsub(1.0, u[0]);
        const double wy = (b & 2) ? u[1] : dsub(1.0, u[1]);
        const double wz = (b & 4) ? u[2] : dsub(1.0, u[2]);
        w[b] = float(dmul(dmul(wx, wy), wz));
    }
    if (u_out)
#pragma unroll
        for (int a = 0; a < 3; ++a) u_out[a] = u[a];
    return true;
}

// Device error codes raised by kernels, mapped to the reference's messages.
enum DevError : int {
    kErrNone = 0,
    kErrTangentRay = 1,       // "tangent ray" (render.cpp:23)
    kErrPointNotInVoxel = 2,  // "point not in voxel" (features.cpp:25)
    kErrSurfaceOutside = 3,   // "surface point outside voxel" (train.cpp:32)
    kErrNegativeTau = 4,      // "negative optical thickness" (render.cpp:76)
    kErrUnknownVoxel = 5,     // "unknown voxel id" (octree.cpp:167)
};

__device__ __forceinline__ void raise_error(int* flag, int code) {
    if (*flag == 0) atomicCAS(flag, 0, code);
}

}  // namespace svlfb
