// Train-step dense layers on the tensor cores with fp32-level accuracy:
// 3xTF32 (every operand x = hi + lo with hi = x rounded to TF32 and lo the
// remainder rounded to TF32; C = A_hi B_lo + A_lo B_hi + A_hi B_hi, fp32
// accumulation in TMEM), tcgen05.mma.cta_group::1.kind::tf32.
//
// The three GEMM shapes of mlp_forward / mlp_backward (src/mlp.cpp:98-230) on
// the feature-major matrices of train.cu (row r = one feature over all hits,
// row stride ld):
//   Fwd  Y[j][n]  = relu(sum_k W[j][k] X[k][n] + b[j])       M = 128 output features, N = hits, K = inputs
//   Bwd  dX[j][n] = sum_o W[o][k0 + j] D[o][n]  (x relu'(h))  M = 128 input features, N = hits, K = outputs
//   Dw   dW[o][k] = sum_n D[o][n] X[k][n], db[o] = sum_n D[o][n]
//                                              M = O (<= 128), N = K + 1 (bias column), K = hits
// Every hit operand is read straight from its feature-major matrix by TMA
// (cp.async.bulk.tensor, 128-byte swizzle): for Fwd / Bwd the hits are the
// MMA's N dimension and the matrix rows are K, i.e. an MN-major B operand
// (32 hits x 32 K-rows per box); for Dw the hits are K and both operands are
// K-major (32 hits per 128-byte row). No register staging of global loads.
// The only register pass is the split: converter warps rewrite each landed
// tile in place as hi and write lo beside it (elementwise, same swizzled
// addresses). The weight operand of Fwd / Bwd is pre-split into a global
// image (one launch builds every layer's image per step) and fetched with a
// 1-D bulk copy.
//
// Warp roles (persistent CTA, one per SM): a TMA producer thread, an MMA
// thread, four converter warps and (Fwd / Bwd) four epilogue warps; stages
// and TMEM accumulators handed over with mbarriers. Dw: each CTA reduces a
// contiguous hit range into its own partial; the partials are summed in a
// fixed order (bitwise reproducible, no atomics). Hit counts are read on the
// device, so nothing here needs the host.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <string>

#include "device.cuh"
#include "gemm_x3.cuh"
#include "tc_common.cuh"

namespace svlfb {

namespace {

using namespace tc;

constexpr uint32_t kChunk = 32;  // K elements per pipeline stage

// ---- PTX helpers ------------------------------------------------------------------
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// TMA store of a shared-memory box (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int kN>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kN) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// L2 prefetch of a future tile (no shared memory): the loads of the stages
// then hit L2 instead of waiting out the DRAM latency
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
#ifndef SVLF_GEMM_PREFETCH
#define SVLF_GEMM_PREFETCH 0  // chunks ahead of the one being loaded (0: off; measured: 4 and 8 slower)
#endif
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 128-byte-swizzled operand descriptors (layout type at bits 61-63): 2 =
// SWIZZLE_128B (16-byte granules; the K-major Dw operands), 1 =
// SWIZZLE_128B_BASE32B (32-byte granules, 4-row atoms: the only MN-major
// layout for 32-bit operands)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return make_desc(saddr, lbo, sbo) | (uint64_t(2) << 61);
}
__device__ __forceinline__ uint64_t desc_sw128_b32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return make_desc(saddr, lbo, sbo) | (uint64_t(1) << 61);
}

__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ float ld_shared_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    return h;
}

// x -> (hi, lo): hi = x rounded to TF32 (half away from zero: add half an ulp
// of the 10-bit mantissa to the magnitude bits, clear the low 13 bits; finite
// inputs), lo = x - hi (exact in fp32, |lo| <= 2^-12 |x|; the tensor core
// reads its top 19 bits, an error <= 2^-23 |x|). Three integer / fp32 ops per
// element (cvt.rna.tf32 is an emulated sequence on sm_100a).
__device__ __forceinline__ void split(uint32_t x, uint32_t& hi, uint32_t& lo) {
    hi = (x + 0x1000u) & 0xffffe000u;
    lo = __float_as_uint(__fsub_rn(__uint_as_float(x), __uint_as_float(hi)));
}

// ---- weight images ------------------------------------------------------------
// Image of one job: chunk c (32 K) of the 128-row A operand as [hi | lo], each
// 16 KB, K-major without swizzle (core matrix = 8 rows x 16 B: LBO = 128 B
// between K-adjacent core matrices, SBO = 1024 B between 8-row groups), zero
// padded.
constexpr uint32_t kFA = 128 * kChunk * 4;  // 16 KB: one 128 x 32 hi (or lo) tile

__host__ __device__ constexpr uint32_t off32(uint32_t r, uint32_t k) {
    return (r >> 3) * 1024u + (k >> 2) * 128u + (r & 7u) * 16u + (k & 3u) * 4u;
}

__global__ void k_wimages(X3ImageJobs J, uint8_t* buf) {
    const X3ImageJob jb = J.job[blockIdx.y];
    uint8_t* img = buf + J.offset[blockIdx.y];
    const uint32_t kred = jb.bwd ? jb.O : jb.K;
    const uint32_t nch = (kred + kChunk - 1) / kChunk;
    const uint32_t total = nch * 128 * kChunk;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t c = i / (128 * kChunk), rem = i % (128 * kChunk), j = rem / kChunk, kk = rem % kChunk;
        const uint32_t k = c * kChunk + kk;
        float v = 0.f;
        if (k < kred) {
            if (!jb.bwd) v = j < jb.O ? jb.W[size_t(j) * jb.K + k] : 0.f;
            else v = (jb.k0 + j < jb.K) ? jb.W[size_t(k) * jb.K + jb.k0 + j] : 0.f;
        }
        uint32_t h, l;
        split(__float_as_uint(v), h, l);
        uint8_t* base = img + size_t(c) * 2 * kFA;
        *reinterpret_cast<uint32_t*>(base + off32(j, kk)) = h;
        *reinterpret_cast<uint32_t*>(base + kFA + off32(j, kk)) = l;
    }
}

// ---- Fwd / Bwd -------------------------------------------------------------------
// Stage: A image chunk [hi 16 KB | lo 16 KB], B hi (raw tile split in place)
// 32 KB, B lo 32 KB. B tile = up to 8 TMA boxes of 32 hits x 32 K-rows (4 KB,
// MN-major, 128-byte swizzle with 32-byte atoms: a K-row is one 128-byte line
// of 32 hits, swizzled in 4-row atoms); box b at +4 KB * b, so the MMA's MN
// blocks are LBO = 4 KB apart and its 4-row K groups SBO = 512 B apart (one
// MMA, K = 8, spans two).
#ifndef SVLF_GEMM_NT
#define SVLF_GEMM_NT 128
#endif
#ifndef SVLF_GEMM_FSTAGES
#define SVLF_GEMM_FSTAGES 3
#endif
constexpr uint32_t kNT = SVLF_GEMM_NT;                // max hits per tile (MMA N)
constexpr uint32_t kFB = kNT * kChunk * 4;             // B hi (or lo) tile
constexpr uint32_t kFStage = 2 * kFA + 2 * kFB;
constexpr uint32_t kFStages = SVLF_GEMM_FSTAGES;
#ifndef SVLF_FEAT_SPLIT_WARPS
#define SVLF_FEAT_SPLIT_WARPS 8
#endif
constexpr uint32_t kFSplitWarps = SVLF_FEAT_SPLIT_WARPS;
constexpr uint32_t kFThreads = 64 + 32 * kFSplitWarps + 128;  // warp 0 TMA, 1 MMA, split warps, 4 epilogue warps
// epilogue staging: per epilogue warp two 32 x 32 fp32 boxes (128-byte swizzle), stored by TMA
constexpr uint32_t kFEpi = 4 * 2 * 4096;
constexpr uint32_t kFHeadW = kFStages * kFStage + kFEpi + 256;  // head weights: float2 {W0, W1} + float W2 per row
constexpr uint32_t kFSmem = kFStages * kFStage + kFEpi + 1024 + 256 + 128 * 12;
static_assert(kFSmem <= 232448, "shared memory budget");
constexpr uint32_t kTmemAcc = kNT;  // TMEM columns per accumulator (two: tile t's epilogue overlaps t+1's MMAs)
constexpr uint32_t kTmemCols = 2 * kTmemAcc <= 256 ? 256 : 512;  // allocation: a power of two

// hits per tile: <= kNT, a multiple of 32, sized so the tiles fill whole waves of the grid
__device__ __forceinline__ uint32_t tile_hits(uint32_t n, uint32_t ctas) {
    const uint32_t waves = max(1u, (n + ctas * kNT - 1) / (ctas * kNT));
    const uint32_t per = (n + ctas * waves - 1) / (ctas * waves);
    return min(kNT, max(32u, (per + 31) / 32 * 32));
}

template <bool kBwd>
__global__ void __launch_bounds__(kFThreads, 1)
    k_gemm_feat(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
                const __grid_constant__ CUtensorMap mask_map, const uint8_t* __restrict__ wimg, float* __restrict__ out,
                const float* __restrict__ bias, const float* __restrict__ mask, const uint32_t* __restrict__ n_dev,
                uint32_t cap, uint32_t ld, uint32_t kred, uint32_t n_out, const float* __restrict__ head_w,
                uint32_t head_c, float* __restrict__ head_out) {
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kFStages * kFStage + kFEpi);
    uint64_t* full = bars;                       // [stages] TMA landed
    uint64_t* split_done = bars + kFStages;      // [stages] converters done (one arrival per split warp)
    uint64_t* empty = bars + 2 * kFStages;       // [stages] MMAs of the stage done (commit)
    uint64_t* accf = bars + 3 * kFStages;        // [2] accumulator ready (commit)
    uint64_t* acce = bars + 3 * kFStages + 2;    // [2] accumulator drained (4 arrivals)
    uint64_t* mbox = bars + 3 * kFStages + 4;    // [4 warps][2 buffers] mask box landed (Bwd)
    uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 3 * kFStages + 12);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (uint32_t i = 0; i < kFStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&split_done[i], kFSplitWarps);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&accf[i], 1);
            mbar_init(&acce[i], 4);
        }
        for (int i = 0; i < 8; ++i) mbar_init(&mbox[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&in_map);
        prefetch_tmap(&out_map);
        if (kBwd && mask) prefetch_tmap(&mask_map);
    }
    if (warp == 1) tmem_alloc(holder, kTmemCols);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *holder;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t n = min(*n_dev, cap);
    const uint32_t nt = tile_hits(n, gridDim.x);
    const uint32_t nb = nt / 32;  // TMA boxes per B tile
    const uint32_t nch = (kred + kChunk - 1) / kChunk;
    const uint32_t ntiles = (n + nt - 1) / nt;
    const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t total = my_tiles * nch;
    auto stage_a = [&](uint32_t s) { return sbase + s * kFStage; };
    auto stage_b = [&](uint32_t s) { return sbase + s * kFStage + 2 * kFA; };

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            for (uint32_t g = 0; g < total; ++g) {
                const uint32_t s = g % kFStages, u = g / kFStages, c = g % nch;
                const uint32_t tile = blockIdx.x + (g / nch) * gridDim.x;
                if (SVLF_GEMM_PREFETCH && g == 0)  // the first chunks' tiles
                    for (uint32_t gp = 0; gp < min(total, uint32_t(SVLF_GEMM_PREFETCH)); ++gp)
                        for (uint32_t b = 0; b < nb; ++b)
                            tma_prefetch_2d(&in_map, int((blockIdx.x + (gp / nch) * gridDim.x) * nt + 32 * b),
                                            int((gp % nch) * kChunk));
                if (SVLF_GEMM_PREFETCH && g + SVLF_GEMM_PREFETCH < total) {
                    const uint32_t gp = g + SVLF_GEMM_PREFETCH;
                    const uint32_t tp = blockIdx.x + (gp / nch) * gridDim.x;
                    for (uint32_t b = 0; b < nb; ++b)
                        tma_prefetch_2d(&in_map, int(tp * nt + 32 * b), int((gp % nch) * kChunk));
                }
                if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
                mbar_expect_tx(&full[s], 2 * kFA + nb * 4096);
                bulk_g2s(stage_a(s), wimg + size_t(c) * 2 * kFA, 2 * kFA, &full[s]);
                for (uint32_t b = 0; b < nb; ++b)
                    tma_2d(stage_b(s) + b * 4096, &in_map, int(tile * nt + 32 * b), int(c * kChunk), &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            const uint32_t idesc = idesc_tf32(128, nt, 0, 1);
            for (uint32_t t = 0; t < my_tiles; ++t) {
                const uint32_t b = t & 1, v = t >> 1;
                if (v > 0) mbar_wait(&acce[b], (v - 1) & 1);
                fence_after_sync();
                const uint32_t d = tmem + kTmemAcc * b;
                for (uint32_t c = 0; c < nch; ++c) {
                    const uint32_t g = t * nch + c, s = g % kFStages, u = g / kFStages;
                    mbar_wait(&full[s], u & 1);  // the A image landed (bulk copy)
                    mbar_wait(&split_done[s], u & 1);
                    fence_after_sync();
                    const uint32_t sa = stage_a(s), sb = stage_b(s);
#pragma unroll
                    for (uint32_t ks = 0; ks < kChunk / 8; ++ks) {
                        const uint64_t ahi = make_desc(sa + ks * 256, 128, 1024);
                        const uint64_t alo = make_desc(sa + kFA + ks * 256, 128, 1024);
                        const uint64_t bhi = desc_sw128_b32(sb + ks * 1024, 4096, 512);
                        const uint64_t blo = desc_sw128_b32(sb + kFB + ks * 1024, 4096, 512);
                        static_assert(kFB % 4096 == 0, "B tiles are whole 4 KB boxes");
                        mma_tf32(d, ahi, blo, idesc, (c | ks) ? 1u : 0u);
                        mma_tf32(d, alo, bhi, idesc, 1u);
                        mma_tf32(d, ahi, bhi, idesc, 1u);
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&accf[b]);
            }
        }
    } else if (warp < 2 + kFSplitWarps) {  // split: B tile -> hi in place, lo beside it
        const uint32_t ct = tid - 64;
        for (uint32_t g = 0; g < total; ++g) {
            const uint32_t s = g % kFStages, u = g / kFStages;
            mbar_wait(&full[s], u & 1);
            const uint32_t hi = stage_b(s), lo = hi + kFB;
#pragma unroll 4
            for (uint32_t i = ct; i < nb * 256; i += 32 * kFSplitWarps) {
                const uint4 x = ld_shared_v4(hi + 16 * i);
                uint4 h, l;
                split(x.x, h.x, l.x);
                split(x.y, h.y, l.y);
                split(x.z, h.z, l.z);
                split(x.w, h.w, l.w);
                st_shared_v4(hi + 16 * i, h.x, h.y, h.z, h.w);
                st_shared_v4(lo + 16 * i, l.x, l.y, l.z, l.w);
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive1(&split_done[s]);
        }
    } else {  // epilogue: TMEM -> bias + relu (Fwd) / relu' mask (Bwd) -> shared box -> TMA store
        const uint32_t q = warp & 3u, j = 32 * q + lane, ew = warp - 2 - kFSplitWarps;
        const float bj = (!kBwd && j < n_out) ? __ldg(bias + j) : 0.f;
        // this warp's two staging boxes: row r (= lane) holds 32 hits, 16-byte chunk c at c ^ (r & 7).
        // Bwd with a mask: the box first receives the mask (TMA load, same swizzle), each thread
        // masks its row in place, and the box is stored back to the output.
        const uint32_t stage0 = sbase + kFStages * kFStage + ew * 8192;
        // head weights of this warp's rows: {W[0][k], W[1][k]} pairs and W[2][k]
        const uint32_t hw01 = sbase + kFHeadW + 8 * (32 * q), hw2 = sbase + kFHeadW + 1024 + 4 * (32 * q);
        if (!kBwd && head_c) {
            const uint32_t k = 32 * q + lane;
            const float w0 = __ldg(head_w + k), w1 = head_c > 1 ? __ldg(head_w + n_out + k) : 0.f;
            const float w2 = head_c > 2 ? __ldg(head_w + 2 * n_out + k) : 0.f;
            asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(hw01 + 8 * lane), "f"(w0), "f"(w1) : "memory");
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(hw2 + 4 * lane), "f"(w2) : "memory");
            __syncwarp();
        }
        const bool use_mask = kBwd && mask != nullptr && 32 * q < n_out;
        const uint32_t nboxes = my_tiles * nb;
        uint32_t mphase = 0;  // parity bit per buffer
        auto box_h0 = [&](uint32_t k) { return (blockIdx.x + (k / nb) * gridDim.x) * nt + 32 * (k % nb); };
        auto load_mask = [&](uint32_t k) {  // lane 0
            if (box_h0(k) >= n) return;
            uint64_t* bar = &mbox[2 * ew + (k & 1)];
            mbar_expect_tx(bar, 4096);
            tma_2d(stage0 + (k & 1) * 4096, &mask_map, int(box_h0(k)), int(32 * q), bar);
        };
        if (use_mask && lane == 0 && nboxes) load_mask(0);
        for (uint32_t k = 0; k < nboxes; ++k) {
            const uint32_t t = k / nb, bt = k % nb, b = t & 1, v = t >> 1;
            if (bt == 0) {
                mbar_wait(&accf[b], v & 1);
                fence_after_sync();
            }
            float r[32];
            tmem_ld32(tmem + kTmemAcc * b + ((32u * q) << 16) + 32 * bt, r);
            tmem_wait_ld();
            const uint32_t h0 = box_h0(k);
            const uint32_t buf = stage0 + (k & 1) * 4096;
            if (32 * q < n_out && h0 < n) {  // warp-uniform: else nothing of this box is stored
                if (use_mask) {
                    // the next box's mask into the other buffer (its previous store must have read it)
                    if (lane == 0) {
                        bulk_wait_read<0>();
                        if (k + 1 < nboxes) load_mask(k + 1);
                    }
                    mbar_wait(&mbox[2 * ew + (k & 1)], (mphase >> (k & 1)) & 1);
                    mphase ^= 1u << (k & 1);
#pragma unroll
                    for (uint32_t c = 0; c < 8; ++c) {
                        const uint4 m = ld_shared_v4(buf + lane * 128 + ((c ^ (lane & 7)) << 4));
                        if (!(__uint_as_float(m.x) > 0.f)) r[4 * c] = 0.f;
                        if (!(__uint_as_float(m.y) > 0.f)) r[4 * c + 1] = 0.f;
                        if (!(__uint_as_float(m.z) > 0.f)) r[4 * c + 2] = 0.f;
                        if (!(__uint_as_float(m.w) > 0.f)) r[4 * c + 3] = 0.f;
                    }
                } else {
                    if (lane == 0) bulk_wait_read<1>();  // the previous store from this buffer has read it
                    if constexpr (!kBwd) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) r[i] = fmaxf(r[i] + bj, 0.f);
                    }
                }
                __syncwarp();
                // rows past n_out and hits past the matrix width are clipped by the tensor map;
                // columns past n carry values of stale inputs and are never read
#pragma unroll
                for (uint32_t c = 0; c < 8; ++c)
                    st_shared_v4(buf + lane * 128 + ((c ^ (lane & 7)) << 4), __float_as_uint(r[4 * c]),
                                 __float_as_uint(r[4 * c + 1]), __float_as_uint(r[4 * c + 2]),
                                 __float_as_uint(r[4 * c + 3]));
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&out_map, buf, int(h0), int(32 * q));
                    bulk_commit();
                }
                if (!kBwd && head_c) {
                    // head layer partial over this warp's 32 rows, lane = hit of the box (read back
                    // transposed from the swizzled box): head_out[q * head_c + c] = sum_r W[c][32q + r] h
                    float hp[3] = {0.f, 0.f, 0.f};
#pragma unroll 8
                    for (uint32_t r = 0; r < 32; ++r) {
                        const float v = ld_shared_f32(buf + r * 128 + (((lane >> 2) ^ (r & 7)) << 4) + (lane & 3) * 4);
                        float w0, w1, w2;  // broadcast loads
                        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(w0), "=f"(w1) : "r"(hw01 + 8 * r));
                        w2 = ld_shared_f32(hw2 + 4 * r);
                        hp[0] = __fmaf_rn(w0, v, hp[0]);
                        hp[1] = __fmaf_rn(w1, v, hp[1]);
                        hp[2] = __fmaf_rn(w2, v, hp[2]);
                    }
                    if (h0 + lane < n)
#pragma unroll
                        for (uint32_t c = 0; c < 3; ++c)
                            if (c < head_c) head_out[size_t(q * head_c + c) * ld + h0 + lane] = hp[c];
                }
            } else if (use_mask && lane == 0 && k + 1 < nboxes) {
                bulk_wait_read<0>();
                load_mask(k + 1);
            }
            if (bt + 1 == nb) {
                fence_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive1(&acce[b]);
            }
        }
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 1) {
        fence_after_sync();
        tmem_dealloc(tmem, kTmemCols);
    }
}

// ---- Dw: part[cta][o][k] = sum over this CTA's hits of D[o][n] X[k][n] ----------
// Stage: A = D tile (128 rows x 32 hits, K-major, 128-byte swizzle: a row is
// one 128-byte line; 8-row groups SBO = 1 KB apart) hi 16 KB + lo 16 KB;
// B = X tile (Nr <= 144 rows x 32 hits, same layout) hi + lo. Row K of B is
// the bias column (ones); rows past the operand's extent arrive as zeros (TMA
// out-of-bounds fill), and hits past n are zeroed by the split.
constexpr uint32_t kDA = 128 * 128;     // 16 KB
constexpr uint32_t kDBMax = 144 * 128;  // 18 KB
constexpr uint32_t kDStage = 2 * kDA + 2 * kDBMax;
constexpr uint32_t kDStages = 3;
#ifndef SVLF_DW_SPLIT_WARPS
#define SVLF_DW_SPLIT_WARPS 12  // measured: 8 -> 12 split warps, dW -1 %
#endif
constexpr uint32_t kDSplitWarps = SVLF_DW_SPLIT_WARPS;
constexpr uint32_t kDThreads = 64 + 32 * kDSplitWarps;  // warp 0 TMA, 1 MMA, the rest split (2-5 also the epilogue)
constexpr uint32_t kDSmem = kDStages * kDStage + 1024 + 256;

template <bool kX3>
__global__ void __launch_bounds__(kDThreads, 1)
    k_gemm_dw(const __grid_constant__ CUtensorMap d_map, const __grid_constant__ CUtensorMap x_map,
              float* __restrict__ part, const uint32_t* __restrict__ n_dev, uint32_t cap, uint32_t O, uint32_t K,
              uint32_t Nr) {
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kDStages * kDStage);
    uint64_t* full = bars;                   // [3]
    uint64_t* split_done = bars + kDStages;  // [3]
    uint64_t* empty = bars + 2 * kDStages;   // [3]
    uint64_t* accf = bars + 3 * kDStages;
    uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 3 * kDStages + 1);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (uint32_t i = 0; i < kDStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&split_done[i], kDSplitWarps);
            mbar_init(&empty[i], 1);
        }
        mbar_init(accf, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&d_map);
        prefetch_tmap(&x_map);
    }
    if (warp == 1) tmem_alloc(holder, 256);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *holder;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t n = min(*n_dev, cap);
    const uint32_t per = ((n + gridDim.x - 1) / gridDim.x + kChunk - 1) / kChunk * kChunk;
    const uint32_t h0 = min(n, blockIdx.x * per), h1 = min(n, h0 + per);
    const uint32_t nch = (h1 - h0 + kChunk - 1) / kChunk;
    const uint32_t bB = Nr * 128;  // bytes of one B hi (or lo) tile
    auto sa = [&](uint32_t s) { return sbase + s * kDStage; };
    auto sb = [&](uint32_t s) { return sbase + s * kDStage + 2 * kDA; };

    if (warp == 0) {
        if (lane == 0) {
            for (uint32_t c = 0; c < nch; ++c) {
                const uint32_t s = c % kDStages, u = c / kDStages;
                if (SVLF_GEMM_PREFETCH && c == 0)
                    for (uint32_t cp = 0; cp < min(nch, uint32_t(SVLF_GEMM_PREFETCH)); ++cp) {
                        tma_prefetch_2d(&d_map, int(h0 + cp * kChunk), 0);
                        tma_prefetch_2d(&x_map, int(h0 + cp * kChunk), 0);
                    }
                if (SVLF_GEMM_PREFETCH && c + SVLF_GEMM_PREFETCH < nch) {
                    tma_prefetch_2d(&d_map, int(h0 + (c + SVLF_GEMM_PREFETCH) * kChunk), 0);
                    tma_prefetch_2d(&x_map, int(h0 + (c + SVLF_GEMM_PREFETCH) * kChunk), 0);
                }
                if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
                mbar_expect_tx(&full[s], 128 * (O + K));
                tma_2d(sa(s), &d_map, int(h0 + c * kChunk), 0, &full[s]);
                tma_2d(sb(s), &x_map, int(h0 + c * kChunk), 0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32(128, Nr, 0, 0);
            for (uint32_t c = 0; c < nch; ++c) {
                const uint32_t s = c % kDStages, u = c / kDStages;
                mbar_wait(&full[s], u & 1);
                mbar_wait(&split_done[s], u & 1);
                fence_after_sync();
#pragma unroll
                for (uint32_t ks = 0; ks < kChunk / 8; ++ks) {
                    const uint64_t ahi = desc_sw128(sa(s) + 32 * ks, 16, 1024);
                    const uint64_t bhi = desc_sw128(sb(s) + 32 * ks, 16, 1024);
                    if constexpr (kX3) {
                        const uint64_t alo = desc_sw128(sa(s) + kDA + 32 * ks, 16, 1024);
                        const uint64_t blo = desc_sw128(sb(s) + bB + 32 * ks, 16, 1024);
                        mma_tf32(tmem, ahi, blo, idesc, (c | ks) ? 1u : 0u);
                        mma_tf32(tmem, alo, bhi, idesc, 1u);
                        mma_tf32(tmem, ahi, bhi, idesc, 1u);
                    } else {
                        mma_tf32(tmem, ahi, bhi, idesc, (c | ks) ? 1u : 0u);
                    }
                }
                mma_commit(&empty[s]);
            }
            if (nch) mma_commit(accf);
        }
    } else {
        const uint32_t ct = tid - 64;
        // The boxes carry only the O rows of D and the K rows of X; the rest of every stage is
        // constant and written once: A rows O..127 and B rows K+1.. zero (hi and lo), B row K the
        // bias column (hi 1.0, lo 0; hits past the range zeroed in the tail chunk below).
        for (uint32_t s = 0; s < kDStages; ++s) {
            const uint32_t a = sa(s), bsm = sb(s);
            for (uint32_t i = ct; i < (128 - O) * 8; i += 32 * kDSplitWarps) {
                st_shared_v4(a + O * 128 + 16 * i, 0u, 0u, 0u, 0u);
                st_shared_v4(a + kDA + O * 128 + 16 * i, 0u, 0u, 0u, 0u);
            }
            const uint32_t one = __float_as_uint(1.f);
            for (uint32_t i = ct; i < (Nr - K) * 8; i += 32 * kDSplitWarps) {
                const uint32_t v = i < 8 ? one : 0u;
                st_shared_v4(bsm + K * 128 + 16 * i, v, v, v, v);
                st_shared_v4(bsm + bB + K * 128 + 16 * i, 0u, 0u, 0u, 0u);
            }
        }
        for (uint32_t c = 0; c < nch; ++c) {
            const uint32_t s = c % kDStages, u = c / kDStages;
            const uint32_t hb = h0 + c * kChunk;
            const bool tail = hb + kChunk > h1;
            mbar_wait(&full[s], u & 1);
            // 16-byte chunk i of a tile: row r = i / 8, physical chunk p = i % 8 holding hits
            // 4 * (p ^ (r & 7)) .. + 3 of the chunk (128-byte swizzle)
            auto do_rows = [&](uint32_t hi, uint32_t lo_off, uint32_t rows) {
#pragma unroll 4
                for (uint32_t i = ct; i < rows * 8; i += 32 * kDSplitWarps) {
                    uint4 x = ld_shared_v4(hi + 16 * i);
                    if (tail) {  // hits past the range: zero (stale matrix columns)
                        const uint32_t hit = hb + 4 * ((i & 7) ^ ((i >> 3) & 7));
                        if (hit >= h1) x.x = 0u;
                        if (hit + 1 >= h1) x.y = 0u;
                        if (hit + 2 >= h1) x.z = 0u;
                        if (hit + 3 >= h1) x.w = 0u;
                    }
                    if constexpr (kX3) {
                        uint4 h, l;
                        split(x.x, h.x, l.x);
                        split(x.y, h.y, l.y);
                        split(x.z, h.z, l.z);
                        split(x.w, h.w, l.w);
                        st_shared_v4(hi + 16 * i, h.x, h.y, h.z, h.w);
                        st_shared_v4(hi + lo_off + 16 * i, l.x, l.y, l.z, l.w);
                    } else if (tail) {
                        st_shared_v4(hi + 16 * i, x.x, x.y, x.z, x.w);
                    }
                }
            };
            do_rows(sa(s), kDA, O);
            do_rows(sb(s), bB, K);
            if (tail)  // the bias column: ones for the hits in range only
                for (uint32_t i = ct; i < 8; i += 32 * kDSplitWarps) {
                    const uint32_t hit = hb + 4 * (i ^ (K & 7));
                    const uint32_t one = __float_as_uint(1.f);
                    st_shared_v4(sb(s) + K * 128 + 16 * i, hit < h1 ? one : 0u, hit + 1 < h1 ? one : 0u,
                                 hit + 2 < h1 ? one : 0u, hit + 3 < h1 ? one : 0u);
                }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive1(&split_done[s]);
        }
        // epilogue (warps 2-5): this CTA's partial, rows o < O, columns j <= K (zeros for a CTA
        // without hits)
        if (warp >= 6) goto done;
        if (nch) {
            mbar_wait(accf, 0);
            fence_after_sync();
        }
        const uint32_t q = warp & 3u, o = 32 * q + lane;
        float* dst = part + (size_t(blockIdx.x) * O + o) * (K + 1);
        for (uint32_t c0 = 0; c0 <= K; c0 += 32) {
            float v[32];
            if (nch) {
                tmem_ld32(tmem + ((32u * q) << 16) + c0, v);
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0.f;
            }
            if (o < O) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (c0 + i <= K) dst[c0 + i] = v[i];
            }
        }
    }
done:
    fence_before_sync();
    __syncthreads();
    if (warp == 1) {
        fence_after_sync();
        tmem_dealloc(tmem, 256);
    }
}

// dW / db = sum over CTAs of the partials, in a fixed order (bitwise
// reproducible): thread (g, e) of a block sums the partials of CTAs
// c = g, g + 8, g + 16, ... in order for output element e, then group sums
// are added g = 0..7 in order. 8-way independent load streams per element.
constexpr uint32_t kRedGroups = 8, kRedElems = 32;
__global__ void __launch_bounds__(kRedGroups * kRedElems)
    k_dw_reduce(const float* __restrict__ part, uint32_t ctas, uint32_t O, uint32_t K, float* __restrict__ dW,
                float* __restrict__ db) {
    __shared__ float sh[kRedGroups][kRedElems];
    const uint32_t cols = K + 1, per = O * cols;
    const uint32_t el = threadIdx.x % kRedElems, g = threadIdx.x / kRedElems;
    const uint32_t e = blockIdx.x * kRedElems + el;
    float acc = 0.f;
    if (e < per) {
        uint32_t c = g;
        for (; c + 3 * kRedGroups < ctas; c += 4 * kRedGroups) {  // four loads in flight, adds in order
            const float a0 = __ldg(part + size_t(c) * per + e), a1 = __ldg(part + size_t(c + kRedGroups) * per + e);
            const float a2 = __ldg(part + size_t(c + 2 * kRedGroups) * per + e);
            const float a3 = __ldg(part + size_t(c + 3 * kRedGroups) * per + e);
            acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, a0), a1), a2), a3);
        }
        for (; c < ctas; c += kRedGroups) acc = __fadd_rn(acc, __ldg(part + size_t(c) * per + e));
    }
    sh[g][el] = acc;
    __syncthreads();
    if (g == 0 && e < per) {
        float t = sh[0][el];
#pragma unroll
        for (uint32_t k = 1; k < kRedGroups; ++k) t = __fadd_rn(t, sh[k][el]);
        const uint32_t o = e / cols, j = e % cols;
        if (j < K) dW[size_t(o) * K + j] = t;
        else db[o] = t;
    }
}

struct DwRedJob {
    const float* part;
    float* dW;
    float* db;
    uint32_t O, K, blocks;  // blocks: (O * (K + 1) + elems - 1) / elems
    uint32_t ctas;          // partials to sum
    uint32_t groups;        // partial-sum groups per element (8, or 32 for many partials); elems = 256 / groups
};
struct DwRedJobs {
    DwRedJob job[kX3MaxDwJobs];
    uint32_t first_block[kX3MaxDwJobs + 1];
    int count;
};

__host__ __device__ inline uint32_t red_groups(uint32_t ctas) { return ctas > 256 ? 32u : kRedGroups; }

// k_dw_reduce over several jobs in one launch (blockIdx.x -> job by block
// ranges): thread (g, e) sums the partials g, g + G, ... of element e in
// order, then the G group sums are added in order (G fixed per job: bitwise
// reproducible)
__global__ void __launch_bounds__(kRedGroups * kRedElems) k_dw_reduce_jobs(DwRedJobs J) {
    __shared__ float sh[kRedGroups * kRedElems];
    int t = 0;
    while (t + 1 < J.count && blockIdx.x >= J.first_block[t + 1]) ++t;
    const DwRedJob jb = J.job[t];
    const uint32_t ctas = jb.ctas, G = jb.groups, E = (kRedGroups * kRedElems) / G;
    const uint32_t cols = jb.K + 1, per = jb.O * cols;
    const uint32_t el = threadIdx.x % E, g = threadIdx.x / E;
    const uint32_t e = (blockIdx.x - J.first_block[t]) * E + el;
    float acc = 0.f;
    if (e < per) {
        uint32_t c = g;
        for (; c + 3 * G < ctas; c += 4 * G) {
            const float a0 = __ldg(jb.part + size_t(c) * per + e);
            const float a1 = __ldg(jb.part + size_t(c + G) * per + e);
            const float a2 = __ldg(jb.part + size_t(c + 2 * G) * per + e);
            const float a3 = __ldg(jb.part + size_t(c + 3 * G) * per + e);
            acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, a0), a1), a2), a3);
        }
        for (; c < ctas; c += G) acc = __fadd_rn(acc, __ldg(jb.part + size_t(c) * per + e));
    }
    sh[g * E + el] = acc;
    __syncthreads();
    if (g == 0 && e < per) {
        float v = sh[el];
        for (uint32_t k = 1; k < G; ++k) v = __fadd_rn(v, sh[k * E + el]);
        const uint32_t o = e / cols, j = e % cols;
        if (j < jb.K) jb.dW[size_t(o) * jb.K + j] = v;
        else jb.db[o] = v;
    }
}

int g_sms = 0;
bool g_attr = false;

void setup() {
    if (!g_sms) {
        int dev = 0;
        SVLF_CUDA(cudaGetDevice(&dev));
        SVLF_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (!g_attr) {
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_dw<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDSmem)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_dw<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDSmem)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_feat<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFSmem)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_feat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFSmem)));
        g_attr = true;
    }
}

// Tensor map of `rows` rows of a feature-major matrix (row stride ld floats,
// `cols` columns = hits): boxes of 32 hits x box_rows rows, 128-byte swizzle
// (16- or 32-byte atoms); rows past `rows` and columns past `cols` read as zeros.
// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time
// libcuda dependency: the library loads on machines without a driver).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        SVLF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) fail(SVLF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

CUtensorMap feature_map(const float* base, uint32_t rows, uint32_t cols, uint32_t ld, uint32_t box_rows,
                        CUtensorMapSwizzle swz) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
    const cuuint32_t box[2] = {32, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                                              strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SVLF_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

uint32_t round16(uint32_t v) { return (v + 15u) & ~15u; }

// persistent grid: one CTA per SM, fewer when the capacity has fewer tiles of 32 hits
uint32_t feat_grid(uint32_t cap) { return std::max<uint32_t>(1, std::min<uint32_t>(uint32_t(g_sms), (cap + 31) / 32)); }
uint32_t dw_grid(uint32_t cap) { return std::max<uint32_t>(1, std::min<uint32_t>(uint32_t(g_sms), (cap + 31) / 32)); }

}  // namespace

size_t gemm_x3_image_bytes(uint32_t kred) { return size_t((kred + kChunk - 1) / kChunk) * 2 * kFA; }

void gemm_x3_build_images(X3ImageJobs& jobs, uint8_t* buf, cudaStream_t s) {
    uint32_t off = 0;
    for (int i = 0; i < jobs.count; ++i) {
        jobs.offset[i] = off;
        off += uint32_t(gemm_x3_image_bytes(jobs.job[i].bwd ? jobs.job[i].O : jobs.job[i].K));
    }
    if (!jobs.count) return;
    k_wimages<<<dim3(32, unsigned(jobs.count)), 256, 0, s>>>(jobs, buf);
    note_launch();
}

void gemm_x3_fwd(const float* x, const uint8_t* img, const float* bias, float* y, uint32_t O, uint32_t K,
                 const uint32_t* n_dev, uint32_t cap, uint32_t ld, cudaStream_t s, const X3Head* head) {
    if (cap == 0) return;
    setup();
    if (head && (head->c < 1 || head->c > 3 || O != 128))
        fail(SVLF_ERR_INVALID_ARGUMENT, "head epilogue: 1..3 outputs over 128 rows");
    const CUtensorMap map = feature_map(x, K, ld, ld, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const CUtensorMap omap = feature_map(y, O, ld, ld, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    k_gemm_feat<false><<<feat_grid(cap), kFThreads, kFSmem, s>>>(
        map, omap, omap, img, y, bias, nullptr, n_dev, cap, ld, K, O, head ? head->w : nullptr, head ? head->c : 0u,
        head ? head->out : nullptr);
    note_launch();
}

void gemm_x3_bwd(const float* d, const uint8_t* img, uint32_t O, uint32_t K, uint32_t k0, float* dx,
                 const float* mask, const uint32_t* n_dev, uint32_t cap, uint32_t ld, cudaStream_t s) {
    if (cap == 0) return;
    setup();
    const CUtensorMap map = feature_map(d, O, ld, ld, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const CUtensorMap omap = feature_map(dx, K - k0, ld, ld, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap mmap = mask ? feature_map(mask, K - k0, ld, ld, 32, CU_TENSOR_MAP_SWIZZLE_128B) : omap;
    k_gemm_feat<true><<<feat_grid(cap), kFThreads, kFSmem, s>>>(map, omap, mmap, img, dx, nullptr, mask, n_dev, cap,
                                                                ld, O, K - k0, nullptr, 0u, nullptr);
    note_launch();
}

size_t gemm_x3_dw_partial_floats(uint32_t O, uint32_t K) {
    int sms = g_sms;
    if (!sms) {
        int dev = 0;
        SVLF_CUDA(cudaGetDevice(&dev));
        SVLF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return size_t(sms) * O * (K + 1);
}

void gemm_x3_dw_batch(const X3DwJob* jobs, int count, const uint32_t* n_dev, uint32_t cap, uint32_t ld, float* part,
                      int products, cudaStream_t s) {
    if (count <= 0) return;
    if (count > kX3MaxDwJobs) fail(SVLF_ERR_INVALID_ARGUMENT, "too many weight-gradient jobs");
    setup();
    const uint32_t ctas = dw_grid(cap);
    DwRedJobs R{};
    size_t off = 0;
    uint32_t blocks = 0;
    for (int i = 0; i < count; ++i) {
        const X3DwJob& jb = jobs[i];
        const uint32_t per = jb.O * (jb.K + 1);
        if (jb.ext_part) {  // partials from another kernel: reduction only
            const uint32_t G = red_groups(jb.ext_ctas), E = kRedGroups * kRedElems / G;
            R.job[i] = DwRedJob{jb.ext_part, jb.dW, jb.db, jb.O, jb.K, (per + E - 1) / E, jb.ext_ctas, G};
            R.first_block[i] = blocks;
            blocks += R.job[i].blocks;
            continue;
        }
        const uint32_t Nr = round16(jb.K + 1);
        if (Nr > 144) fail(SVLF_ERR_INVALID_ARGUMENT, "weight-gradient GEMM: K too large");
        const CUtensorMap dmap = feature_map(jb.d, jb.O, ld, ld, jb.O, CU_TENSOR_MAP_SWIZZLE_128B);
        const CUtensorMap xmap = feature_map(jb.x, jb.K, ld, ld, jb.K, CU_TENSOR_MAP_SWIZZLE_128B);
        float* p = part + off;
        if (products == 1)
            k_gemm_dw<false><<<ctas, kDThreads, kDSmem, s>>>(dmap, xmap, p, n_dev, cap, jb.O, jb.K, Nr);
        else
            k_gemm_dw<true><<<ctas, kDThreads, kDSmem, s>>>(dmap, xmap, p, n_dev, cap, jb.O, jb.K, Nr);
        const uint32_t G = red_groups(ctas), E = kRedGroups * kRedElems / G;
        R.job[i] = DwRedJob{p, jb.dW, jb.db, jb.O, jb.K, (per + E - 1) / E, ctas, G};
        R.first_block[i] = blocks;
        blocks += R.job[i].blocks;
        off += size_t(ctas) * per;
    }
    R.first_block[count] = blocks;
    R.count = count;
    k_dw_reduce_jobs<<<blocks, kRedGroups * kRedElems, 0, s>>>(R);
    int gemms = 0;
    for (int i = 0; i < count; ++i) gemms += jobs[i].ext_part ? 0 : 1;
    note_launch(gemms + 1);
}

void gemm_x3_dw(const float* d, const float* x, uint32_t O, uint32_t K, float* dW, float* db, const uint32_t* n_dev,
                uint32_t cap, uint32_t ld, float* part, int products, cudaStream_t s) {
    setup();
    const uint32_t Nr = round16(K + 1), ctas = dw_grid(cap);
    if (Nr > 144) fail(SVLF_ERR_INVALID_ARGUMENT, "weight-gradient GEMM: K too large");
    const CUtensorMap dmap = feature_map(d, O, ld, ld, O, CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap xmap = feature_map(x, K, ld, ld, K, CU_TENSOR_MAP_SWIZZLE_128B);
    if (products == 1)
        k_gemm_dw<false><<<ctas, kDThreads, kDSmem, s>>>(dmap, xmap, part, n_dev, cap, O, K, Nr);
    else
        k_gemm_dw<true><<<ctas, kDThreads, kDSmem, s>>>(dmap, xmap, part, n_dev, cap, O, K, Nr);
    const uint32_t per = O * (K + 1);
    k_dw_reduce<<<(per + kRedElems - 1) / kRedElems, kRedGroups * kRedElems, 0, s>>>(part, ctas, O, K, dW, db);
    note_launch(2);
}

}  // namespace svlfb

// ---- unit-test entry (C ABI svlf_debug_gemm_x3; tests/test_gemm_gpu.py) ----------
extern "C" svlf_status svlf_debug_gemm_x3(int kind, const float* W, uint32_t O, uint32_t K, uint32_t k0,
                                          const float* bias, const float* in, const float* in2, const float* mask,
                                          float* out, float* out2, uint32_t n, uint32_t ld, int products) {
    using namespace svlfb;
    try {
        uint32_t* nd = nullptr;
        SVLF_CUDA(cudaMalloc(&nd, 4));
        SVLF_CUDA(cudaMemcpy(nd, &n, 4, cudaMemcpyHostToDevice));
        uint8_t* img = nullptr;
        float* part = nullptr;
        if (kind == 0 || kind == 1) {
            X3ImageJobs jobs{};
            jobs.job[0] = {W, O, K, k0, uint32_t(kind)};
            jobs.count = 1;
            SVLF_CUDA(cudaMalloc(&img, gemm_x3_image_bytes(kind ? O : K)));
            gemm_x3_build_images(jobs, img, 0);
            if (kind == 0) gemm_x3_fwd(in, img, bias, out, O, K, nd, n, ld, 0);
            else gemm_x3_bwd(in, img, O, K, k0, out, mask, nd, n, ld, 0);
        } else {
            SVLF_CUDA(cudaMalloc(&part, gemm_x3_dw_partial_floats(O, K) * 4));
            gemm_x3_dw(in, in2, O, K, out, out2, nd, n, ld, part, products, 0);
        }
        SVLF_CUDA(cudaDeviceSynchronize());
        cudaFree(nd);
        if (img) cudaFree(img);
        if (part) cudaFree(part);
        return SVLF_OK;
    } catch (const std::exception&) {
        return SVLF_ERR_CUDA;
    }
}
