// Sparse-voxel-octree ray traversal (reference SparseOctree::traverse,
// src/octree.cpp:192-235).
//
// Main kernel: level-synchronous, block-cooperative traversal. A block owns
// 64 rays (an 8x8 pixel tile in camera mode). Starting from the (ray, root)
// pairs whose root box is hit, it expands the active (ray, node) pairs one
// level at a time: thread e takes pair e, tests the node's existing children
// front to back, and an order-preserving block scan appends the hit children
// to the next level's queue in shared memory. Pairs stay grouped by ray and,
// within a ray, in front-to-back depth-first order, so at the leaf level each
// ray's hits are contiguous and nearly sorted; an insertion sort per ray
// finishes the (t_in, code) order, one atomic per block allocates the block's
// output range and the hits are written coalesced. Every warp instruction
// works on 32 independent pairs, so SIMT efficiency does not depend on how
// unequal the rays' paths are, and the octree is walked once (no count pass).
// Tiles whose queues overflow shared memory are handed to the per-ray
// fallback walker (k_traverse_fallback).
//
// Exactness. The reference tests each child box with ray_aabb on
// [lo + x*cell_l, lo + (x+1)*cell_l]. Child planes coincide bit-for-bit with
// parent planes (2x * cell_l/2 and x * cell_l round the same real number;
// cell_l/2 is exact), so a node computes its three planes per axis (lo, mid,
// hi) and their parametric values (plane - o) * (1/d) once, exactly as
// ray_aabb would, and each child's slab interval is a selection of those.
// t0 = max(0, ta_x, ta_y, ta_z), t1 = min(...) with "reject iff t1 < t0" is
// the reference's axis-by-axis early exit (t0 only grows, t1 only shrinks);
// zero direction components are the reference's inside-the-slab test; leaves
// are kept iff t1 - t0 > 1e-12; leaf index order is Morton order. So hit ids,
// order and t values are bit-identical to the reference built without FMA.
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include "device.cuh"

namespace svlfb {

namespace {

constexpr double kMinHitSpan = 1e-12;  // tie rule, src/octree.cpp:16
#ifndef SVLF_BFS_W0
#define SVLF_BFS_W0 1  // ray-indexed scans (root queue, segment offsets) as first-warp shuffle scans
#endif
#ifndef SVLF_BFS_PARTIAL
#define SVLF_BFS_PARTIAL 1  // queue overflow hands only the rays reaching the overflowing chunk to the next pass
#endif
#ifndef SVLF_BFS_EMPTY_EXIT
#define SVLF_BFS_EMPTY_EXIT 1  // tiles whose pairs all die before the leaf level skip the segment scan and sort
#endif

// Slab intervals of the two halves of a node along each axis.
struct NodeSplit {
    double lo_a[3], lo_b[3];  // low half:  [lo_a, lo_b]
    double hi_a[3], hi_b[3];  // high half: [hi_a, hi_b]
};

// zmask bit a: the ray's direction component a is zero
// kLoZero: the box origin is (+-0, +-0, +-0): lo + m * cell == m * cell bit for bit (m * cell >= +0)
template <bool kLoZero = false>
__device__ __forceinline__ void split_node_z(const DevOctree& T, const double* o, uint32_t zmask,
                                             const double* inv, int level, uint32_t x, uint32_t y, uint32_t z,
                                             NodeSplit& s) {
    const uint32_t c[3] = {x, y, z};
    const double cl = T.cell[level], ch = T.cell[level + 1];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double mlo = dmul(double(c[a]), cl), mhi = dmul(double(c[a] + 1u), cl);
        const double mmid = dmul(double(2u * c[a] + 1u), ch);
        const double plo = kLoZero ? mlo : dadd(T.lo[a], mlo);
        const double phi = kLoZero ? mhi : dadd(T.lo[a], mhi);
        const double pmid = kLoZero ? mmid : dadd(T.lo[a], mmid);
        if (!((zmask >> a) & 1u)) {
            const double tl = dmul(dsub(plo, o[a]), inv[a]);
            const double tm = dmul(dsub(pmid, o[a]), inv[a]);
            const double th = dmul(dsub(phi, o[a]), inv[a]);
            // "if (ta > tb) swap" exactly (keeps the reference's choice of signed zeros)
            const bool swl = tl > tm, swh = tm > th;
            s.lo_a[a] = swl ? tm : tl;
            s.lo_b[a] = swl ? tl : tm;
            s.hi_a[a] = swh ? th : tm;
            s.hi_b[a] = swh ? tm : th;
        } else {  // inside-the-slab test per half (geometry.cpp:13-16)
            const bool in_lo = !(o[a] < plo || o[a] > pmid);
            const bool in_hi = !(o[a] < pmid || o[a] > phi);
            s.lo_a[a] = in_lo ? -CUDART_INF : CUDART_INF;
            s.lo_b[a] = in_lo ? CUDART_INF : -CUDART_INF;
            s.hi_a[a] = in_hi ? -CUDART_INF : CUDART_INF;
            s.hi_b[a] = in_hi ? CUDART_INF : -CUDART_INF;
        }
    }
}

__device__ __forceinline__ uint32_t zero_mask(const double* d) {
    return (d[0] == 0.0 ? 1u : 0u) | (d[1] == 0.0 ? 2u : 0u) | (d[2] == 0.0 ? 4u : 0u);
}

__device__ __forceinline__ void split_node(const DevOctree& T, const double* o, const double* d,
                                           const double* inv, int level, uint32_t x, uint32_t y, uint32_t z,
                                           NodeSplit& s) {
    split_node_z(T, o, zero_mask(d), inv, level, x, y, z, s);
}

__device__ __forceinline__ bool child_hit(const NodeSplit& s, uint32_t oct, double& t0, double& t1) {
    t0 = 0.0;
    t1 = CUDART_INF;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool hi = (oct >> a) & 1u;
        const double ta = hi ? s.hi_a[a] : s.lo_a[a];
        const double tb = hi ? s.hi_b[a] : s.lo_b[a];
        if (ta > t0) t0 = ta;  // src/geometry.cpp:21-22
        if (tb < t1) t1 = tb;
    }
    return !(t1 < t0);
}

// child_hit for all eight octants at once (bit oct of the result; kLeaf: also
// t1 - t0 > kMinHitSpan). Each octant's t0 / t1 is the same left-to-right
// max / min chain over the axes as child_hit's, so the results are
// bit-identical; the x and xy prefixes of the chains are shared between
// octants (14 compare-selects per chain instead of 24).
template <bool kLeaf>
__device__ __forceinline__ uint32_t child_hits(const NodeSplit& s) {
    double t0x[2], t1x[2], t0xy[4], t1xy[4];
#pragma unroll
    for (int hx = 0; hx < 2; ++hx) {
        const double ta = hx ? s.hi_a[0] : s.lo_a[0], tb = hx ? s.hi_b[0] : s.lo_b[0];
        t0x[hx] = ta > 0.0 ? ta : 0.0;
        t1x[hx] = tb < CUDART_INF ? tb : CUDART_INF;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int hx = i & 1, hy = i >> 1;
        const double ta = hy ? s.hi_a[1] : s.lo_a[1], tb = hy ? s.hi_b[1] : s.lo_b[1];
        t0xy[i] = ta > t0x[hx] ? ta : t0x[hx];
        t1xy[i] = tb < t1x[hx] ? tb : t1x[hx];
    }
    uint32_t m = 0;
#pragma unroll
    for (int oct = 0; oct < 8; ++oct) {
        const int i = oct & 3, hz = oct >> 2;
        const double ta = hz ? s.hi_a[2] : s.lo_a[2], tb = hz ? s.hi_b[2] : s.lo_b[2];
        const double t0 = ta > t0xy[i] ? ta : t0xy[i];
        const double t1 = tb < t1xy[i] ? tb : t1xy[i];
        const bool hit = kLeaf ? (!(t1 < t0) && dsub(t1, t0) > kMinHitSpan) : !(t1 < t0);
        m |= hit ? 1u << oct : 0u;
    }
    return m;
}

// Octant mask reindexed in front-to-back order: bit it of the result is bit
// (it ^ s) of m, so walking its set bits from the lowest visits the children
// in the order `for it: oct = it ^ s` does, one iteration per set bit.
__device__ __forceinline__ uint32_t front_to_back(uint32_t m, uint32_t s) {
    if (s & 1u) m = ((m & 0x55u) << 1) | ((m >> 1) & 0x55u);
    if (s & 2u) m = ((m & 0x33u) << 2) | ((m >> 2) & 0x33u);
    if (s & 4u) m = ((m & 0x0fu) << 4) | ((m >> 4) & 0x0fu);
    return m;
}

__device__ __forceinline__ uint32_t sign_mask(const double* d) {
    return (d[0] < 0.0 ? 1u : 0u) | (d[1] < 0.0 ? 2u : 0u) | (d[2] < 0.0 ? 4u : 0u);
}

__device__ __forceinline__ uint64_t pack_xyz(uint32_t x, uint32_t y, uint32_t z) {
    return uint64_t(x) | (uint64_t(y) << 21) | (uint64_t(z) << 42);
}

// ---- per-ray depth-first walker (fallback for overflowing tiles) -----------
template <typename OnLeaf>
__device__ __forceinline__ void walk(const DevOctree& T, const RayPre& p, OnLeaf&& on_leaf) {
    {
        double lo[3], hi[3], t0, t1;
        cell_box(T, T.cell[0], 0, 0, 0, lo, hi);
        if (!slab_test(p, lo, hi, t0, t1)) return;
    }
    const uint32_t s = sign_mask(p.r.d);
    const int L = T.L;
    uint2 st_node[kMaxLevelsDev];
    uint64_t st_xyz[kMaxLevelsDev];
    int lvl = 0;
    uint32_t x = 0, y = 0, z = 0, it = 0;
    uint2 node = T.nodes[0];
    NodeSplit sp;
    split_node(T, p.r.o, p.r.d, p.inv, 0, x, y, z, sp);
    while (true) {
        if (it == 8) {
            if (lvl == 0) break;
            --lvl;
            node = st_node[lvl];
            it = node.y >> 8;
            node.y &= 0xffu;
            const uint64_t c = st_xyz[lvl];
            x = uint32_t(c & 0x1fffffu);
            y = uint32_t((c >> 21) & 0x1fffffu);
            z = uint32_t(c >> 42);
            split_node(T, p.r.o, p.r.d, p.inv, lvl, x, y, z, sp);
            continue;
        }
        const uint32_t oct = it ^ s;
        ++it;
        if (!((node.y >> oct) & 1u)) continue;
        double t0, t1;
        if (!child_hit(sp, oct, t0, t1)) continue;
        const uint32_t child = node.x + __popc(node.y & ((1u << oct) - 1u));
        if (lvl + 1 == L) {
            if (dsub(t1, t0) > kMinHitSpan) on_leaf(child - T.level_off[L], t0, t1);
            continue;
        }
        st_node[lvl] = make_uint2(node.x, node.y | (it << 8));
        st_xyz[lvl] = pack_xyz(x, y, z);
        x = 2u * x + (oct & 1u);
        y = 2u * y + ((oct >> 1) & 1u);
        z = 2u * z + ((oct >> 2) & 1u);
        ++lvl;
        it = 0;
        node = T.nodes[child];
        split_node(T, p.r.o, p.r.d, p.inv, lvl, x, y, z, sp);
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

__device__ __forceinline__ void store_ray(double* rays, size_t i, const Ray& r) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        rays[6 * i + a] = r.o[a];
        rays[6 * i + 3 + a] = r.d[a];
    }
}

// Insertion sort of hits [b, e) by (t_in, leaf index).
template <typename TinArr, typename LeafArr>
__device__ __forceinline__ void sort_segment(TinArr tin, LeafArr leaf, uint32_t b, uint32_t e) {
    for (uint32_t a = b + 1; a < e; ++a) {
        const double ti = tin[a];
        const uint32_t lf = leaf[a];
        uint32_t k = a;
        while (k > b) {
            const double tp = tin[k - 1];
            const uint32_t lp = leaf[k - 1];
            if (tp < ti || (tp == ti && lp < lf)) break;
            tin[k] = tp;
            leaf[k] = lp;
            --k;
        }
        tin[k] = ti;
        leaf[k] = lf;
    }
}

// ---- block-cooperative level-synchronous traversal -------------------------
// First pass: kRays-ray tiles processed by kThreads threads (one warp when
// kThreads == 32, kBlockThreads / kThreads independent tiles per block) with
// a kQCap-pair level queue. Tiles whose queue overflows are redone by a second
// pass with more threads per ray and a much larger queue; anything still
// overflowing goes to a per-ray walker.
#ifndef SVLF_BFS_RAYS
#define SVLF_BFS_RAYS 32
#endif
#ifndef SVLF_BFS_THREADS
#define SVLF_BFS_THREADS 128
#endif
#ifndef SVLF_BFS_BLOCK
#define SVLF_BFS_BLOCK SVLF_BFS_THREADS
#endif
#ifndef SVLF_BFS_QCAP
#define SVLF_BFS_QCAP 768
#endif
#ifndef SVLF_RAYS_DENSE
#define SVLF_RAYS_DENSE 16
#endif
#ifndef SVLF_DENSE_QCAP
#define SVLF_DENSE_QCAP 1536
#endif
constexpr int kRays = SVLF_BFS_RAYS;         // rays per tile, first pass
constexpr int kThreads = SVLF_BFS_THREADS;   // threads per tile, first pass
constexpr int kBlockThreads = SVLF_BFS_BLOCK;  // threads per block, first pass
constexpr int kQCap = SVLF_BFS_QCAP;         // (ray, node) pairs per level, first pass
constexpr int kRaysDense = SVLF_RAYS_DENSE;  // rays per block, second pass
#ifndef SVLF_DENSE_THREADS
#define SVLF_DENSE_THREADS 256
#endif
constexpr int kThreadsDense = SVLF_DENSE_THREADS;
constexpr int kQCapDense = SVLF_DENSE_QCAP;

template <int kR, int kQ, int kT>
struct BfsSmem {
    double o[3][kR], d[3][kR], inv[3][kR];
    uint64_t qxyz[2][kQ];
    uint32_t qnode[2][kQ];
    uint32_t pos[kQ];  // leaf level: output position of each pair's first hit
    uint8_t kmask[kQ];  // leaf level: each pair's kept children (pass A -> pass B)
    uint8_t qray[2][kQ];
    uint8_t dflags[kR];  // per ray: direction sign bits (0-2) and zero-component bits (3-5)
    uint32_t rcount[kR], roff[kR];
    uint32_t gray[kR];
    uint32_t n_q, base, overflow, next_tile;
    uint32_t evict, cut;  // partial hand-over: rays leaving the tile, kept length of the next queue
    uint32_t nlev[2];     // next-level pair counts of the first-warp levels (alternating by level)
    uint32_t wtot[2];             // per-warp totals of the two-warp (kT == 64) scan
    unsigned long long unsorted;  // rays whose segment needs the insertion sort
    struct NoScan {};
    // cub's block scan only for whole-block tiles; 32/64-thread tiles scan with shuffles
    typename std::conditional<(kT > 64), typename cub::BlockScan<uint32_t, kT>::TempStorage, NoScan>::type scan;
};

struct BfsArgs {
    uint32_t* ray_off;
    uint32_t* ray_cnt;
    uint32_t* hit_leaf;
    double* hit_tin;
    double* hit_tout;
    uint32_t* hit_ray;
    uint32_t* counters;  // [0] hits allocated, [1] overflow rays, [2] capacity exceeded, [3] dense overflow,
                         // [5] / [6] next tile of the first / second cooperative pass,
                         // [7] ray-box tests (root + every occupied child of an expanded node, 32-bit)
    uint32_t* overflow_rays;
    uint32_t* overflow_dense;
    double* rays;
    uint32_t capacity;
};

// kR rays per block. kList = false: tiles of the image / ray buffer (first
// pass, overflow -> overflow_rays); kList = true: consecutive entries of
// overflow_rays (second pass, overflow -> overflow_dense).
// A tile is processed by kT threads: a whole block (kT > 32, block barriers
// and cub::BlockScan) or a single warp (kT == 32, warp barriers and shuffle
// scans: the warps of a block then run independent tiles).
template <int kT>
__device__ __forceinline__ void tile_sync() {
    if constexpr (kT == 32) {
        __syncwarp();
    } else if constexpr (kT == 64) {  // two-warp group: its own named barrier (id 1 + group)
        asm volatile("bar.sync %0, 64;" ::"r"(1u + threadIdx.x / 64u) : "memory");
    } else {
        __syncthreads();
    }
}

// Exclusive sum over the 32 lanes of one warp (values of the tile's first warp
// when only its lanes hold non-zero values: rays, or a level of <= 32 pairs)
__device__ __forceinline__ void warp_excl_sum(uint32_t v, uint32_t& off, uint32_t& tot) {
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= uint32_t(d)) x += y;
    }
    tot = __shfl_sync(0xffffffffu, x, 31);
    off = x - v;
}

// Exclusive sum over the tile. Every call site is followed by a tile_sync()
// before the next scan, so the kT == 64 variant's single barrier is enough to
// protect its two-word exchange.
template <int kT, typename Smem>
__device__ __forceinline__ void tile_excl_sum(Smem& S, uint32_t v, uint32_t& off, uint32_t& tot) {
    if constexpr (kT == 32 || kT == 64) {
        const uint32_t lane = threadIdx.x & 31u;
        uint32_t x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= uint32_t(d)) x += y;
        }
        const uint32_t wt = __shfl_sync(0xffffffffu, x, 31);
        if constexpr (kT == 32) {
            tot = wt;
            off = x - v;
        } else {
            const uint32_t w = (threadIdx.x >> 5) & 1u;
            if (lane == 31) S.wtot[w] = wt;
            tile_sync<kT>();
            const uint32_t w0 = S.wtot[0];
            tot = w0 + S.wtot[1];
            off = x - v + (w ? w0 : 0u);
        }
    } else {
        cub::BlockScan<uint32_t, kT>(S.scan).ExclusiveSum(v, off, tot);
    }
}

// camera tile shape for kR rays: 8 x kR/8 pixels, or 4 x 2 for 8-ray tiles
template <int kR>
struct TileShape {
    static constexpr int W = kR >= 32 ? 8 : 4;
    static constexpr int H = kR / W;
};

template <bool kCamera, int kR, int kQ, int kT, bool kList, bool kCount, bool kLoZero>
__device__ __forceinline__ void bfs_tile(const DevOctree& T, const DevCamera& cam, uint32_t row0, uint32_t rows,
                                         uint32_t n, const BfsArgs& A, BfsSmem<kR, kQ, kT>& S, uint32_t tile,
                                         uint32_t& tests_done) {
    const uint32_t tid = threadIdx.x & uint32_t(kT - 1);
    uint32_t tests = 0;  // this tile's ray-box tests; counted only if the tile completes here

    // ---- rays of this tile; root test
    uint32_t my_ray = 0xffffffffu;
    if (tid < kR) {
        uint32_t gi;
        bool ok;
        if constexpr (kList) {
            const uint32_t k = tile * kR + tid;
            gi = k < A.counters[1] ? A.overflow_rays[k] : 0xffffffffu;
            ok = gi != 0xffffffffu;
        } else if constexpr (kCamera) {
            using TS = TileShape<kR>;
            const uint32_t tiles_x = (cam.width + TS::W - 1) / TS::W;
            const uint32_t tx = tile % tiles_x, ty = tile / tiles_x;
            const uint32_t px = tx * TS::W + tid % TS::W, py = ty * TS::H + tid / TS::W;
            ok = px < cam.width && py < rows;
            gi = py * cam.width + px;
        } else {
            gi = tile * kR + tid;
            ok = gi < n;
        }
        S.gray[tid] = ok ? gi : 0xffffffffu;
        S.rcount[tid] = 0;
        if (ok) {
            my_ray = gi;
            Ray r;
            if constexpr (kCamera) {
                uint32_t ix, iy;
                cam_pixel(cam, gi, row0, ix, iy);
                r = pixel_ray(cam, ix, iy);
            } else {
                r = load_ray(A.rays, gi);
            }
            const RayPre p = precompute(r);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                S.o[a][tid] = r.o[a];
                S.d[a][tid] = r.d[a];
                S.inv[a][tid] = p.inv[a];
            }
            S.dflags[tid] = uint8_t(sign_mask(r.d) | (zero_mask(r.d) << 3));
        }
    }
    static_assert(kR <= 64, "per-tile ray mask");
    static_assert(kR <= 32 || !SVLF_BFS_W0, "first-warp scans: at most 32 rays per tile");
    static_assert(kR <= 32 || !SVLF_BFS_PARTIAL, "partial hand-over: 32-bit ray mask");
    if (tid == 0) {
        S.n_q = 0;
        S.overflow = 0;
        S.unsorted = 0;
    }
    if (!SVLF_BFS_W0) tile_sync<kT>();  // (W0: every value read before the next barrier is the reader's own)
    {
        uint32_t hit = 0;
        if (my_ray != 0xffffffffu) {
            double lo[3], hi[3], t0, t1, o[3], d[3];
            RayPre p;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                o[a] = S.o[a][tid];
                d[a] = S.d[a][tid];
                p.r.o[a] = o[a];
                p.r.d[a] = d[a];
                p.inv[a] = S.inv[a][tid];
            }
            cell_box(T, T.cell[0], 0, 0, 0, lo, hi);
            hit = slab_test(p, lo, hi, t0, t1) ? 1u : 0u;
            if constexpr (kCount) ++tests;
        }
        if (SVLF_BFS_W0 && kT > 32) {  // only the first warp holds rays: warp scan, one barrier
            if (tid < 32) {
                uint32_t off, tot;
                warp_excl_sum(hit, off, tot);
                if (hit) {
                    S.qnode[0][off] = 0;
                    S.qxyz[0][off] = 0;
                    S.qray[0][off] = uint8_t(tid);
                }
                if (tid == 0) S.n_q = tot;
            }
        } else {
            uint32_t off, tot;
            tile_excl_sum<kT>(S, hit, off, tot);
            if (hit) {
                S.qnode[0][off] = 0;
                S.qxyz[0][off] = 0;
                S.qray[0][off] = uint8_t(tid);
            }
            if (tid == 0) S.n_q = tot;
        }
        tile_sync<kT>();
    }

    // ---- internal levels: expand (ray, node) pairs into the next level's queue
    int cur = 0;
    uint32_t n_cur = S.n_q;
    int level = 0;
    for (; level + 1 < T.L && n_cur > 0; ++level) {
        uint32_t n_out = 0;
        if (SVLF_BFS_W0 && kT > 32 && n_cur <= 32) {
            // the whole level in the first warp (at most 256 children: no overflow): warp scan,
            // one barrier instead of three
            static_assert(kQ >= 256, "a 32-pair level always fits the next queue");
            if (tid < 32) {
                uint32_t hitmask = 0, cnt = 0, ri = 0, x = 0, y = 0, z = 0, s = 0;
                uint2 node = make_uint2(0, 0);
                if (tid < n_cur) {
                    ri = S.qray[cur][tid];
                    node = T.nodes[S.qnode[cur][tid]];
                    const uint64_t xyz = S.qxyz[cur][tid];
                    x = uint32_t(xyz & 0x1fffffu);
                    y = uint32_t((xyz >> 21) & 0x1fffffu);
                    z = uint32_t(xyz >> 42);
                    double o[3], inv[3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        o[a] = S.o[a][ri];
                        inv[a] = S.inv[a][ri];
                    }
                    const uint32_t fl = S.dflags[ri];
                    NodeSplit sp;
                    split_node_z<kLoZero>(T, o, fl >> 3, inv, level, x, y, z, sp);
                    s = fl & 7u;
                    if constexpr (kCount) tests += __popc(node.y);
                    hitmask = child_hits<false>(sp) & node.y & 0xffu;
                    cnt = __popc(hitmask);
                }
                uint32_t off, tot;
                warp_excl_sum(cnt, off, tot);
                uint32_t w = off;
                for (uint32_t todo = front_to_back(hitmask, s); todo; todo &= todo - 1) {
                    const uint32_t oct = uint32_t(__ffs(todo) - 1) ^ s;
                    S.qnode[cur ^ 1][w] = node.x + __popc(node.y & ((1u << oct) - 1u));
                    S.qxyz[cur ^ 1][w] =
                        pack_xyz(2u * x + (oct & 1u), 2u * y + ((oct >> 1) & 1u), 2u * z + ((oct >> 2) & 1u));
                    S.qray[cur ^ 1][w] = uint8_t(ri);
                    ++w;
                }
                if (tid == 0) S.nlev[level & 1] = tot;
            }
            tile_sync<kT>();
            n_cur = S.nlev[level & 1];  // (the next level writes the other slot)
            cur ^= 1;
            continue;
        }
        for (uint32_t base = 0; base < n_cur; base += kT) {
            const uint32_t e = base + tid;
            uint32_t hitmask = 0, cnt = 0, ri = 0, x = 0, y = 0, z = 0, s = 0;
            uint2 node = make_uint2(0, 0);
            if (e < n_cur) {
                ri = S.qray[cur][e];
                node = T.nodes[S.qnode[cur][e]];
                const uint64_t xyz = S.qxyz[cur][e];
                x = uint32_t(xyz & 0x1fffffu);
                y = uint32_t((xyz >> 21) & 0x1fffffu);
                z = uint32_t(xyz >> 42);
                double o[3], inv[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    o[a] = S.o[a][ri];
                    inv[a] = S.inv[a][ri];
                }
                const uint32_t fl = S.dflags[ri];
                NodeSplit sp;
                split_node_z<kLoZero>(T, o, fl >> 3, inv, level, x, y, z, sp);
                s = fl & 7u;
                if constexpr (kCount) tests += __popc(node.y);
                hitmask = child_hits<false>(sp) & node.y & 0xffu;
                cnt = __popc(hitmask);
            }
            uint32_t off, tot;
            tile_excl_sum<kT>(S, cnt, off, tot);
            if (n_out + tot > kQ) {
                if (kCount || !SVLF_BFS_PARTIAL) {  // whole tile to the next pass (exact test counts)
                    if (tid == 0) S.overflow = 1;
                    tile_sync<kT>();
                    break;
                }
                // Partial hand-over: the rays with pairs in this chunk or later leave the tile for
                // the next pass (redone there from the root); the earlier rays, whose children are
                // all in the next queue, continue here. The queues are grouped by ray in order, so
                // the next queue is cut before the first child of the first leaving ray.
                const uint32_t R = S.qray[cur][base];
                if (tid == 0) {
                    S.evict = 0;
                    S.cut = n_out;
                }
                tile_sync<kT>();
                for (uint32_t i = base + tid; i < n_cur; i += kT) atomicOr(&S.evict, 1u << S.qray[cur][i]);
                for (uint32_t i = tid; i < n_out; i += kT)
                    if (S.qray[cur ^ 1][i] == R && (i == 0 || S.qray[cur ^ 1][i - 1] != R)) S.cut = i;
                tile_sync<kT>();
                const uint32_t ev = S.evict;
                if (tid == 0) S.base = atomicAdd(&A.counters[kList ? 3 : 1], uint32_t(__popc(ev)));
                tile_sync<kT>();
                if (tid < kR && ((ev >> tid) & 1u)) {
                    (kList ? A.overflow_dense : A.overflow_rays)[S.base + __popc(ev & ((1u << tid) - 1u))] = S.gray[tid];
                    S.gray[tid] = 0xffffffffu;  // not finalised by this pass
                }
                n_out = S.cut;
                tile_sync<kT>();
                break;
            }
            uint32_t w = n_out + off;  // children in front-to-back octant order
            for (uint32_t todo = front_to_back(hitmask, s); todo; todo &= todo - 1) {
                const uint32_t oct = uint32_t(__ffs(todo) - 1) ^ s;
                S.qnode[cur ^ 1][w] = node.x + __popc(node.y & ((1u << oct) - 1u));
                S.qxyz[cur ^ 1][w] =
                    pack_xyz(2u * x + (oct & 1u), 2u * y + ((oct >> 1) & 1u), 2u * z + ((oct >> 2) & 1u));
                S.qray[cur ^ 1][w] = uint8_t(ri);
                ++w;
            }
            n_out += tot;
            tile_sync<kT>();
        }
        if (S.overflow) break;
        n_cur = n_out;
        cur ^= 1;  // the chunk barrier above already orders this level's appends before the next level
    }

    if (S.overflow) {  // (this tile's tests are not counted: the pass that completes its rays counts them)  // hand the whole tile (kept contiguous) to the next pass
        if (tid == 0) S.base = atomicAdd(&A.counters[kList ? 3 : 1], uint32_t(kR));
        tile_sync<kT>();
        if (tid < kR) (kList ? A.overflow_dense : A.overflow_rays)[S.base + tid] = S.gray[tid];
        return;
    }

    // ---- leaf level, two passes: (A) count kept leaves per pair, scan, allocate;
    // (B) recompute and write each pair's leaves straight to their final slots.
    // Pairs are grouped by ray in order, so the pair scan is also the per-ray
    // segment layout; each ray's segment is then sorted in place.
    const bool leaf_pass = level + 1 == T.L && n_cur > 0;
#if SVLF_BFS_EMPTY_EXIT
    if (!leaf_pass) {  // no (ray, node) pair reached the leaf level: every ray of the tile has no hits
        if (tid < kR && S.gray[tid] != 0xffffffffu) {
            A.ray_off[S.gray[tid]] = 0;  // (what the segment scan gives a tile without hits)
            A.ray_cnt[S.gray[tid]] = 0;
        }
        if constexpr (kCount) tests_done += tests;
        return;
    }
#endif
    uint32_t total = 0;
    if (leaf_pass) {
        for (uint32_t base = 0; base < n_cur; base += kT) {
            const uint32_t e = base + tid;
            uint32_t cnt = 0, ri = 0;
            if (e < n_cur) {
                ri = S.qray[cur][e];
                const uint2 node = T.nodes[S.qnode[cur][e]];
                const uint64_t xyz = S.qxyz[cur][e];
                double o[3], inv[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    o[a] = S.o[a][ri];
                    inv[a] = S.inv[a][ri];
                }
                NodeSplit sp;
                split_node_z<kLoZero>(T, o, uint32_t(S.dflags[ri]) >> 3, inv, level, uint32_t(xyz & 0x1fffffu),
                             uint32_t((xyz >> 21) & 0x1fffffu), uint32_t(xyz >> 42), sp);
                if constexpr (kCount) tests += __popc(node.y);
                const uint32_t keep = child_hits<true>(sp) & node.y & 0xffu;
                S.kmask[e] = uint8_t(keep);
                cnt = __popc(keep);
                if (cnt) atomicAdd(&S.rcount[ri], cnt);
            }
            uint32_t off, tot;
            tile_excl_sum<kT>(S, cnt, off, tot);
            if (e < n_cur) S.pos[e] = total + off;
            total += tot;
            tile_sync<kT>();
        }
    }
    if (SVLF_BFS_W0 && kT > 32) {  // per-ray segment offsets: the rays are the first warp's lanes
        if (tid < 32) {
            const uint32_t c = tid < kR ? S.rcount[tid] : 0u;
            uint32_t off, tot;
            warp_excl_sum(c, off, tot);
            if (tid < kR) S.roff[tid] = off;
            if (tid == 0) {
                const uint32_t b = tot ? atomicAdd(&A.counters[0], tot) : 0u;
                S.base = b;
                if (b + tot > A.capacity) atomicExch(&A.counters[2], 1u);
            }
        }
        tile_sync<kT>();
    } else {
        const uint32_t c = tid < kR ? S.rcount[tid] : 0u;
        uint32_t off, tot;
        tile_excl_sum<kT>(S, c, off, tot);
        if (tid < kR) S.roff[tid] = off;
        if (tid == 0) {
            const uint32_t b = tot ? atomicAdd(&A.counters[0], tot) : 0u;
            S.base = b;
            if (b + tot > A.capacity) atomicExch(&A.counters[2], 1u);
        }
        tile_sync<kT>();
    }
    const uint32_t gbase = S.base;
    const bool fits = gbase + total <= A.capacity;
    if (leaf_pass && fits) {
        for (uint32_t e = tid; e < n_cur; e += kT) {
            const uint32_t keep = S.kmask[e];  // pass A's kept children
            if (!keep) continue;
            const uint32_t ri = S.qray[cur][e];
            const uint2 node = T.nodes[S.qnode[cur][e]];
            const uint64_t xyz = S.qxyz[cur][e];
            double o[3], inv[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                o[a] = S.o[a][ri];
                inv[a] = S.inv[a][ri];
            }
            const uint32_t fl = S.dflags[ri];
            NodeSplit sp;
            split_node_z<kLoZero>(T, o, fl >> 3, inv, level, uint32_t(xyz & 0x1fffffu), uint32_t((xyz >> 21) & 0x1fffffu),
                         uint32_t(xyz >> 42), sp);
            const uint32_t s = fl & 7u;
            uint32_t w = gbase + S.pos[e];
            const uint32_t gr = S.gray[ri];
            for (uint32_t todo = front_to_back(keep, s); todo; todo &= todo - 1) {
                const uint32_t oct = uint32_t(__ffs(todo) - 1) ^ s;
                double t0, t1;
                child_hit(sp, oct, t0, t1);
                A.hit_leaf[w] = node.x + __popc(node.y & ((1u << oct) - 1u)) - T.level_off[T.L];
                A.hit_tin[w] = t0;
                A.hit_tout[w] = t1;
                A.hit_ray[w] = gr;
                ++w;
            }
        }
    }
    tile_sync<kT>();
    // The front-to-back expansion already emits each ray's leaves in t_in order
    // except at ties; a parallel, coalesced pass over the tile's hits finds the
    // segments with an inversion, and only those get the serial insertion sort.
    if (leaf_pass && fits) {
        for (uint32_t e = tid; e + 1 < total; e += kT) {
            const uint32_t w = gbase + e;
            if (A.hit_ray[w] != A.hit_ray[w + 1]) continue;
            const double t0 = A.hit_tin[w], t1 = A.hit_tin[w + 1];
            if (t0 < t1 || (t0 == t1 && A.hit_leaf[w] < A.hit_leaf[w + 1])) continue;
            for (uint32_t r = 0; r < uint32_t(kR); ++r)
                if (S.rcount[r] && S.roff[r] <= e && e < S.roff[r] + S.rcount[r]) {
                    atomicOr(&S.unsorted, 1ull << r);
                    break;
                }
        }
    }
    tile_sync<kT>();
    if (tid < kR && S.gray[tid] != 0xffffffffu && fits) {
        const uint32_t c = S.rcount[tid], b = gbase + S.roff[tid];
        A.ray_off[S.gray[tid]] = b;
        A.ray_cnt[S.gray[tid]] = c;
        // insertion sort of the (nearly sorted) segment by (t_in, leaf index), carrying t_out
        if ((S.unsorted >> tid) & 1ull)
        for (uint32_t a = b + 1; a < b + c; ++a) {
            const double ti = A.hit_tin[a], to = A.hit_tout[a];
            const uint32_t lf = A.hit_leaf[a];
            uint32_t k = a;
            while (k > b) {
                const double tp = A.hit_tin[k - 1];
                const uint32_t lp = A.hit_leaf[k - 1];
                if (tp < ti || (tp == ti && lp < lf)) break;
                A.hit_tin[k] = tp;
                A.hit_tout[k] = A.hit_tout[k - 1];
                A.hit_leaf[k] = lp;
                --k;
            }
            A.hit_tin[k] = ti;
            A.hit_tout[k] = to;
            A.hit_leaf[k] = lf;
        }
        if (kCamera && c > 0) {  // later stages read foreground rays only
            Ray r;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                r.o[a] = S.o[a][tid];
                r.d[a] = S.d[a][tid];
            }
            store_ray(A.rays, S.gray[tid], r);
        }
    }
    if constexpr (kCount) tests_done += tests;
}

// Persistent: each tile group (a block, or each warp of a block when kT ==
// 32) takes tiles from a device-side cursor until they run out. kList passes
// read their tile count from the device (no host round trip).
#ifndef SVLF_BFS_MINB
#define SVLF_BFS_MINB 8  // resident 128-thread blocks per SM (256-thread second pass: 4): at most 64 registers
#endif
template <bool kCamera, int kR, int kQ, int kT, int kBlock, bool kList, bool kCount, bool kLoZero>
__global__ void __launch_bounds__(kBlock, kBlock == 128 ? SVLF_BFS_MINB : (kBlock == 256 ? 4 : 1)) k_traverse_bfs(DevOctree T, DevCamera cam, uint32_t row0, uint32_t rows,
                                                         uint32_t n, uint32_t n_tiles, BfsArgs A) {
    extern __shared__ __align__(16) uint8_t bfs_smem[];
    static_assert(kBlock % kT == 0, "tile groups per block");
    const uint32_t g = threadIdx.x / kT;
    auto& S = reinterpret_cast<BfsSmem<kR, kQ, kT>*>(bfs_smem)[g];
    const uint32_t tiles = kList ? (A.counters[1] + kR - 1) / kR : n_tiles;
    // dynamic tile assignment (one atomic per tile): tiles differ widely in
    // cost (background vs dense foreground), so a static round-robin leaves a
    // long tail
    uint32_t* next = A.counters + (kList ? 6 : 5);
    uint32_t tests = 0;
    for (;;) {
        if ((threadIdx.x & uint32_t(kT - 1)) == 0) S.next_tile = atomicAdd(next, 1u);
        tile_sync<kT>();
        const uint32_t tile = S.next_tile;
        if (tile >= tiles) break;
        bfs_tile<kCamera, kR, kQ, kT, kList, kCount, kLoZero>(T, cam, row0, rows, n, A, S, tile, tests);
        tile_sync<kT>();
    }
    if constexpr (kCount) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) tests += __shfl_xor_sync(0xffffffffu, tests, d);
        if ((threadIdx.x & 31u) == 0 && tests) atomicAdd(&A.counters[7], tests);
    }
}

template <bool kCamera>
__device__ __forceinline__ void fallback_ray(const DevOctree& T, const DevCamera& cam, uint32_t row0,
                                                  const BfsArgs& A, uint32_t i) {
    if (i == 0xffffffffu) return;
    Ray r;
    if constexpr (kCamera) {
        uint32_t ix, iy;
        cam_pixel(cam, i, row0, ix, iy);
        r = pixel_ray(cam, ix, iy);
    } else {
        r = load_ray(A.rays, i);
    }
    const RayPre p = precompute(r);
    uint32_t c = 0;
    walk(T, p, [&](uint32_t, double, double) { ++c; });
    const uint32_t base = c ? atomicAdd(&A.counters[0], c) : 0u;
    A.ray_off[i] = base;
    A.ray_cnt[i] = c;
    if (kCamera && c > 0) store_ray(A.rays, i, r);
    if (base + c > A.capacity) {
        atomicExch(&A.counters[2], 1u);
        return;
    }
    uint32_t w = base;
    walk(T, p, [&](uint32_t leaf, double t0, double t1) {
        A.hit_leaf[w] = leaf;
        A.hit_tin[w] = t0;
        A.hit_tout[w] = t1;
        A.hit_ray[w] = i;
        ++w;
    });
    // sort (t_in, leaf) carrying t_out
    for (uint32_t a = base + 1; a < base + c; ++a) {
        const double ti = A.hit_tin[a], to = A.hit_tout[a];
        const uint32_t lf = A.hit_leaf[a];
        uint32_t b = a;
        while (b > base) {
            const double tp = A.hit_tin[b - 1];
            const uint32_t lp = A.hit_leaf[b - 1];
            if (tp < ti || (tp == ti && lp < lf)) break;
            A.hit_tin[b] = tp;
            A.hit_tout[b] = A.hit_tout[b - 1];
            A.hit_leaf[b] = lp;
            --b;
        }
        A.hit_tin[b] = ti;
        A.hit_tout[b] = to;
        A.hit_leaf[b] = lf;
    }
}

// Per-ray depth-first traversal of the rays that overflowed both cooperative
// passes (persistent grid-stride over the device-side list).
template <bool kCamera>
__global__ void __launch_bounds__(128) k_traverse_fallback(DevOctree T, DevCamera cam, uint32_t row0,
                                                           const uint32_t* n_list, BfsArgs A) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < *n_list; k += gridDim.x * blockDim.x)
        fallback_ray<kCamera>(T, cam, row0, A, A.overflow_dense[k]);
}

// CSR view (ray order) of the traversal output: out[csr[i] + k] = in[off[i] + k]
__global__ void k_to_csr(const uint32_t* ray_off, const uint32_t* ray_cnt, const uint32_t* csr, uint32_t n,
                         const uint32_t* leaf, const double* tin, const double* tout, uint32_t* leaf_o,
                         double* tin_o, double* tout_o, uint32_t* ray_o) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = ray_off[i], c = ray_cnt[i], d = csr[i];
    for (uint32_t k = 0; k < c; ++k) {
        leaf_o[d + k] = leaf[s + k];
        tin_o[d + k] = tin[s + k];
        tout_o[d + k] = tout[s + k];
        ray_o[d + k] = i;
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

static BfsArgs bfs_args(const TraverseOut& o) {
    return BfsArgs{o.ray_off, o.ray_cnt, o.hit_leaf, o.hit_tin, o.hit_tout, o.hit_ray,
                   o.counters, o.overflow_rays, o.overflow_dense, o.rays, o.capacity};
}
static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        SVLF_CUDA(cudaGetDevice(&dev));
        SVLF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return sms;
}
#ifndef SVLF_BFS_BLOCKS_PER_SM
#define SVLF_BFS_BLOCKS_PER_SM 8
#endif
constexpr int kBfsBlocksPerSm = SVLF_BFS_BLOCKS_PER_SM;

// the octree box starts at the origin (the unit scene box): split planes without the origin add
static bool box_origin_zero(const DevOctree& T) { return T.lo[0] == 0.0 && T.lo[1] == 0.0 && T.lo[2] == 0.0; }

template <bool kCamera, int kR, int kQ, int kT, int kBlock, bool kList, bool kCount, bool kLoZero>
static void set_bfs_attr() {
    static bool done = false;
    if (done) return;
    SVLF_CUDA(cudaFuncSetAttribute(k_traverse_bfs<kCamera, kR, kQ, kT, kBlock, kList, kCount, kLoZero>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(sizeof(BfsSmem<kR, kQ, kT>) * (kBlock / kT))));
    done = true;
}

template <bool kCount, bool kLoZero>
static void launch_traverse_t(const DevOctree& T, const DevCamera* cam, uint32_t row0, uint32_t rows, uint32_t n,
                              const TraverseOut& o, cudaStream_t s) {
    const BfsArgs A = bfs_args(o);
    constexpr uint32_t kGroups = kBlockThreads / kThreads;
    const size_t smem = sizeof(BfsSmem<kRays, kQCap, kThreads>) * kGroups;
    const uint32_t cap_grid = uint32_t(num_sms() * kBfsBlocksPerSm);
    if (cam) {
        set_bfs_attr<true, kRays, kQCap, kThreads, kBlockThreads, false, kCount, kLoZero>();
        using TS = TileShape<kRays>;
        const uint32_t tiles = ((cam->width + TS::W - 1) / TS::W) * ((rows + TS::H - 1) / TS::H);
        const uint32_t blocks = std::min((tiles + kGroups - 1) / kGroups, cap_grid);
        k_traverse_bfs<true, kRays, kQCap, kThreads, kBlockThreads, false, kCount, kLoZero><<<blocks, kBlockThreads, smem, s>>>(
            T, *cam, row0, rows, n, tiles, A);
    } else {
        set_bfs_attr<false, kRays, kQCap, kThreads, kBlockThreads, false, kCount, kLoZero>();
        const uint32_t tiles = (n + kRays - 1) / kRays;
        const uint32_t blocks = std::min((tiles + kGroups - 1) / kGroups, cap_grid);
        k_traverse_bfs<false, kRays, kQCap, kThreads, kBlockThreads, false, kCount, kLoZero><<<blocks, kBlockThreads, smem, s>>>(
            T, DevCamera{}, 0, 0, n, tiles, A);
    }
}

void launch_traverse(const DevOctree& T, const DevCamera* cam, uint32_t row0, uint32_t rows, uint32_t n,
                     const TraverseOut& o, cudaStream_t s, bool count) {
    if (n == 0) return;
    const bool lz = box_origin_zero(T);
    if (count)
        lz ? launch_traverse_t<true, true>(T, cam, row0, rows, n, o, s)
           : launch_traverse_t<true, false>(T, cam, row0, rows, n, o, s);
    else
        lz ? launch_traverse_t<false, true>(T, cam, row0, rows, n, o, s)
           : launch_traverse_t<false, false>(T, cam, row0, rows, n, o, s);
    note_launch();
}

template <bool kCount, bool kLoZero>
static void launch_traverse_dense_t(const DevOctree& T, const DevCamera* cam, uint32_t row0, const TraverseOut& o,
                                    cudaStream_t s) {
    const BfsArgs A = bfs_args(o);
    using Sm = BfsSmem<kRaysDense, kQCapDense, kThreadsDense>;
    const uint32_t per_sm = std::max<uint32_t>(1, uint32_t(200 * 1024 / sizeof(Sm)));
    const uint32_t grid = uint32_t(num_sms()) * per_sm;
    if (cam) {
        set_bfs_attr<true, kRaysDense, kQCapDense, kThreadsDense, kThreadsDense, true, kCount, kLoZero>();
        k_traverse_bfs<true, kRaysDense, kQCapDense, kThreadsDense, kThreadsDense, true, kCount, kLoZero>
            <<<grid, kThreadsDense, sizeof(Sm), s>>>(T, *cam, row0, 0, 0, 0, A);
    } else {
        set_bfs_attr<false, kRaysDense, kQCapDense, kThreadsDense, kThreadsDense, true, kCount, kLoZero>();
        k_traverse_bfs<false, kRaysDense, kQCapDense, kThreadsDense, kThreadsDense, true, kCount, kLoZero>
            <<<grid, kThreadsDense, sizeof(Sm), s>>>(T, DevCamera{}, 0, 0, 0, 0, A);
    }
}

void launch_traverse_dense(const DevOctree& T, const DevCamera* cam, uint32_t row0, const TraverseOut& o,
                           cudaStream_t s, bool count) {
    const bool lz = box_origin_zero(T);
    if (count)
        lz ? launch_traverse_dense_t<true, true>(T, cam, row0, o, s) : launch_traverse_dense_t<true, false>(T, cam, row0, o, s);
    else
        lz ? launch_traverse_dense_t<false, true>(T, cam, row0, o, s)
           : launch_traverse_dense_t<false, false>(T, cam, row0, o, s);
    note_launch();
}

void launch_traverse_fallback(const DevOctree& T, const DevCamera* cam, uint32_t row0, const TraverseOut& o,
                              cudaStream_t s) {
    const BfsArgs A = bfs_args(o);
    const uint32_t grid = uint32_t(num_sms() * 4);
    if (cam)
        k_traverse_fallback<true><<<grid, 128, 0, s>>>(T, *cam, row0, o.counters + 3, A);
    else
        k_traverse_fallback<false><<<grid, 128, 0, s>>>(T, DevCamera{}, 0, o.counters + 3, A);
    note_launch();
}

void launch_to_csr(const uint32_t* ray_off, const uint32_t* ray_cnt, const uint32_t* csr, uint32_t n,
                   const uint32_t* leaf, const double* tin, const double* tout, uint32_t* leaf_o, double* tin_o,
                   double* tout_o, uint32_t* ray_o, cudaStream_t s) {
    if (n == 0) return;
    k_to_csr<<<(n + 127) / 128, 128, 0, s>>>(ray_off, ray_cnt, csr, n, leaf, tin, tout, leaf_o, tin_o, tout_o,
                                             ray_o);
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
