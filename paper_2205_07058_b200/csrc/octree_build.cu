// Octree build on the GPU (reference SparseOctree::build + finalize_from_leaves,
// src/octree.cpp:30-142), byte-identical to the host build (host_octree.cpp):
//   quantize   per point: inside test against the scene box, half-open cells
//              with the max face clamped into the last cell (fp64, correctly
//              rounded division as in the reference), Morton code; dropped
//              points counted and mapped to a sentinel that sorts last
//   cells      radix sort + unique
//   dilation   (2r+1)^3 Chebyshev neighbours per cell, clipped to the grid,
//              radix sort + unique
//   levels     ancestors by code >> 3 (a sorted list stays sorted) + unique
//   vertices   8 corner-lattice keys per leaf, (cz*lat + cy)*lat + cx; sort +
//              unique = dense vertex ids; each corner's id by binary search
//   nodes      per child: parent by binary search, child-mask bit, first
//              child of each parent at the start of its run
// Results are downloaded into a HostOctree (the host API and the traversal's
// device mirror are unchanged).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "device.cuh"
#include "host_octree.hpp"

namespace svlfb {

namespace {

__device__ __forceinline__ uint64_t spread3(uint64_t v) {
    v &= 0x1fffffULL;
    v = (v | v << 32) & 0x1f00000000ffffULL;
    v = (v | v << 16) & 0x1f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}
__device__ __forceinline__ uint32_t gather3(uint64_t v) {
    v &= 0x1249249249249249ULL;
    v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ULL;
    v = (v ^ (v >> 4)) & 0x100f00f00f00f00fULL;
    v = (v ^ (v >> 8)) & 0x1f0000ff0000ffULL;
    v = (v ^ (v >> 16)) & 0x1f00000000ffffULL;
    v = (v ^ (v >> 32)) & 0x1fffffULL;
    return uint32_t(v);
}
__device__ __forceinline__ uint64_t mcode(uint32_t x, uint32_t y, uint32_t z) {
    return spread3(x) | spread3(y) << 1 | spread3(z) << 2;
}

struct BoxArgs {
    double lo[3], hi[3], h;
    uint32_t res;
    uint64_t sentinel;
};

__global__ void k_quantize(const double* __restrict__ pts, size_t n, BoxArgs B, uint64_t* codes,
                           unsigned long long* dropped) {
    unsigned long long local = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        double p[3];
        bool inside = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            p[a] = pts[3 * i + a];
            inside = inside && p[a] >= B.lo[a] && p[a] <= B.hi[a];
        }
        if (!inside) {
            codes[i] = B.sentinel;
            ++local;
            continue;
        }
        uint32_t c[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const uint32_t q = uint32_t(__ddiv_rn(__dsub_rn(p[a], B.lo[a]), B.h));
            c[a] = q < B.res - 1 ? q : B.res - 1;
        }
        codes[i] = mcode(c[0], c[1], c[2]);
    }
    if (local) atomicAdd(dropped, local);
}

__global__ void k_dilate(const uint64_t* __restrict__ cells, size_t m, int r, uint32_t res, uint64_t sentinel,
                         uint64_t* out) {
    const int w = 2 * r + 1;
    const size_t per = size_t(w) * w * w;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < m * per; i += size_t(gridDim.x) * blockDim.x) {
        const size_t cell = i / per;
        const int k = int(i % per);
        const uint64_t code = cells[cell];
        const int x = int(gather3(code)) + k % w - r, y = int(gather3(code >> 1)) + (k / w) % w - r,
                  z = int(gather3(code >> 2)) + k / (w * w) - r;
        const int ires = int(res);
        out[i] = (x < 0 || y < 0 || z < 0 || x >= ires || y >= ires || z >= ires)
                     ? sentinel
                     : mcode(uint32_t(x), uint32_t(y), uint32_t(z));
    }
}

__global__ void k_shift3(const uint64_t* __restrict__ in, size_t n, uint64_t* out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        out[i] = in[i] >> 3;
}

__global__ void k_lattice_keys(const uint64_t* __restrict__ leaves, size_t n, uint64_t lat, uint64_t* keys) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n * 8; i += size_t(gridDim.x) * blockDim.x) {
        const uint64_t code = leaves[i >> 3];
        const uint32_t b = uint32_t(i & 7);
        const uint64_t x = gather3(code) + (b & 1), y = gather3(code >> 1) + ((b >> 1) & 1),
                       z = gather3(code >> 2) + ((b >> 2) & 1);
        keys[i] = (z * lat + y) * lat + x;
    }
}

__device__ __forceinline__ size_t lower_bound_u64(const uint64_t* a, size_t n, uint64_t v) {
    size_t lo = 0, hi = n;
    while (lo < hi) {
        const size_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_rank(const uint64_t* __restrict__ keys, size_t n, const uint64_t* __restrict__ lattice, size_t v,
                       uint32_t* ids) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        ids[i] = uint32_t(lower_bound_u64(lattice, v, keys[i]));
}

// children kids[0..nk) of parents[0..np) (both sorted): mask bits, first child
__global__ void k_node_table(const uint64_t* __restrict__ parents, size_t np, const uint64_t* __restrict__ kids,
                             size_t nk, uint32_t kid_off, uint32_t* first, uint32_t* mask) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nk; i += size_t(gridDim.x) * blockDim.x) {
        const uint64_t pc = kids[i] >> 3;
        const size_t p = lower_bound_u64(parents, np, pc);
        atomicOr(mask + p, 1u << uint32_t(kids[i] & 7));
        if (i == 0 || (kids[i - 1] >> 3) != pc) first[p] = kid_off + uint32_t(i);
    }
}

unsigned grid_for(size_t n) { return unsigned(std::min<size_t>((n + 255) / 256, 148 * 32)); }

template <typename T>
std::vector<T> download(const T* d, size_t n, cudaStream_t s) {
    std::vector<T> h(n);
    if (n) SVLF_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaStreamSynchronize(s));
    return h;
}

// sort + unique `n` keys of `bits` bits in `buf` (ping-pong with `tmp`); returns the count
size_t sort_unique_dev(DevBuf& buf, DevBuf& tmp, DevBuf& scratch, DevBuf& count, size_t n, int bits,
                       cudaStream_t s) {
    if (n == 0) return 0;
    uint64_t* a = buf.as<uint64_t>();
    uint64_t* b = tmp.ensure<uint64_t>(n);
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t1, a, b, n, 0, bits, s);
    uint64_t* dummy = nullptr;
    cub::DeviceSelect::Unique(nullptr, t2, b, dummy, count.ensure<unsigned long long>(1), n, s);
    char* tb = scratch.ensure<char>(std::max(t1, t2));
    SVLF_CUDA(cub::DeviceRadixSort::SortKeys(tb, t1, a, b, n, 0, bits, s));
    SVLF_CUDA(cub::DeviceSelect::Unique(tb, t2, b, a, count.as<unsigned long long>(), n, s));
    unsigned long long m = 0;
    SVLF_CUDA(cudaMemcpyAsync(&m, count.p, 8, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaStreamSynchronize(s));
    return size_t(m);
}

}  // namespace

HostOctree build_octree_gpu(const svlf_grid& grid, const double* d_pts, size_t n, cudaStream_t s) {
    validate_grid(grid);
    HostOctree t;
    t.grid = grid;
    const uint32_t res = grid.resolution;
    int L = 0;
    while ((1u << L) < res) ++L;
    t.leaf_level = L;
    t.cell_size = (grid.hi[0] - grid.lo[0]) / res;
    t.levels.assign(size_t(L) + 1, {});
    const uint64_t sentinel = uint64_t(1) << (3 * L);  // sorts after every code
    const int bits = 3 * L + 1;

    DevBuf codes, tmp, scratch, count, dropped;
    unsigned long long* d_dropped = dropped.ensure<unsigned long long>(1);
    SVLF_CUDA(cudaMemsetAsync(d_dropped, 0, 8, s));
    BoxArgs B{};
    for (int a = 0; a < 3; ++a) {
        B.lo[a] = grid.lo[a];
        B.hi[a] = grid.hi[a];
    }
    B.h = (grid.hi[0] - grid.lo[0]) / res;
    B.res = res;
    B.sentinel = sentinel;
    uint64_t* c = codes.ensure<uint64_t>(std::max<size_t>(n, 1));
    if (n) k_quantize<<<grid_for(n), 256, 0, s>>>(d_pts, n, B, c, d_dropped);
    size_t m = sort_unique_dev(codes, tmp, scratch, count, n, bits, s);
    unsigned long long dr = 0;
    SVLF_CUDA(cudaMemcpy(&dr, d_dropped, 8, cudaMemcpyDeviceToHost));
    t.dropped_points = size_t(dr);
    auto strip_sentinel = [&](size_t cnt) {
        if (cnt == 0) return cnt;
        uint64_t last = 0;
        SVLF_CUDA(cudaMemcpy(&last, codes.as<uint64_t>() + cnt - 1, 8, cudaMemcpyDeviceToHost));
        return last == sentinel ? cnt - 1 : cnt;
    };
    m = strip_sentinel(m);
    if (m == 0) fail(SVLF_ERR_RUNTIME, "empty occupancy");
    if (grid.dilation > 0) {
        const int r = int(std::min<uint32_t>(grid.dilation, res));
        const size_t per = size_t(2 * r + 1) * (2 * r + 1) * (2 * r + 1);
        DevBuf grown;
        uint64_t* g = grown.ensure<uint64_t>(m * per);
        k_dilate<<<grid_for(m * per), 256, 0, s>>>(codes.as<uint64_t>(), m, r, res, sentinel, g);
        std::swap(codes.p, grown.p);
        std::swap(codes.cap, grown.cap);
        m = strip_sentinel(sort_unique_dev(codes, tmp, scratch, count, m * per, bits, s));
    }
    t.levels[size_t(L)] = download(codes.as<uint64_t>(), m, s);

    // ancestors, level by level (device lists kept for the node table)
    std::vector<DevBuf> lv(size_t(L) + 1);
    lv[size_t(L)].ensure<uint64_t>(m);
    SVLF_CUDA(cudaMemcpyAsync(lv[size_t(L)].p, codes.p, m * 8, cudaMemcpyDeviceToDevice, s));
    std::vector<size_t> sizes(size_t(L) + 1, 0);
    sizes[size_t(L)] = m;
    for (int l = L; l > 0; --l) {
        const size_t nk = sizes[size_t(l)];
        uint64_t* par = lv[size_t(l - 1)].ensure<uint64_t>(nk);
        uint64_t* sh = tmp.ensure<uint64_t>(nk);
        k_shift3<<<grid_for(nk), 256, 0, s>>>(lv[size_t(l)].as<uint64_t>(), nk, sh);
        size_t t2 = 0;
        cub::DeviceSelect::Unique(nullptr, t2, sh, par, count.ensure<unsigned long long>(1), nk, s);
        SVLF_CUDA(cub::DeviceSelect::Unique(scratch.ensure<char>(t2), t2, sh, par, count.as<unsigned long long>(), nk, s));
        unsigned long long np = 0;
        SVLF_CUDA(cudaMemcpyAsync(&np, count.p, 8, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        sizes[size_t(l - 1)] = size_t(np);
        t.levels[size_t(l - 1)] = download(par, size_t(np), s);
    }

    // dense vertex ids over the leaf-corner lattice
    const uint64_t lat = uint64_t(res) + 1;
    DevBuf keys, lattice;
    uint64_t* k = keys.ensure<uint64_t>(m * 8);
    k_lattice_keys<<<grid_for(m * 8), 256, 0, s>>>(lv[size_t(L)].as<uint64_t>(), m, lat, k);
    lattice.ensure<uint64_t>(m * 8);
    SVLF_CUDA(cudaMemcpyAsync(lattice.p, k, m * 64, cudaMemcpyDeviceToDevice, s));
    int kbits = 1;
    while (kbits < 64 && (uint64_t(1) << kbits) <= lat * lat * lat) ++kbits;
    const size_t V = sort_unique_dev(lattice, tmp, scratch, count, m * 8, kbits, s);
    t.vertex_count = uint32_t(V);
    DevBuf ids;
    uint32_t* d_ids = ids.ensure<uint32_t>(m * 8);
    k_rank<<<grid_for(m * 8), 256, 0, s>>>(k, m * 8, lattice.as<uint64_t>(), V, d_ids);
    t.corner_ids = download(d_ids, m * 8, s);

    // node table
    t.level_off.assign(size_t(L) + 2, 0);
    for (int l = 0; l <= L; ++l) t.level_off[size_t(l) + 1] = t.level_off[size_t(l)] + uint32_t(sizes[size_t(l)]);
    const size_t internal = t.level_off[size_t(L)];
    DevBuf first, mask;
    uint32_t* d_first = first.ensure<uint32_t>(std::max<size_t>(internal, 1));
    uint32_t* d_mask = mask.ensure<uint32_t>(std::max<size_t>(internal, 1));
    SVLF_CUDA(cudaMemsetAsync(d_mask, 0, internal * 4, s));
    for (int l = 0; l < L; ++l)
        k_node_table<<<grid_for(sizes[size_t(l) + 1]), 256, 0, s>>>(
            lv[size_t(l)].as<uint64_t>(), sizes[size_t(l)], lv[size_t(l) + 1].as<uint64_t>(), sizes[size_t(l) + 1],
            t.level_off[size_t(l) + 1], d_first + t.level_off[size_t(l)], d_mask + t.level_off[size_t(l)]);
    t.node_first_child = download(d_first, internal, s);
    const auto m32 = download(d_mask, internal, s);
    t.node_mask.assign(m32.begin(), m32.end());
    note_launch(5 + L + L);
    return t;
}

}  // namespace svlfb
