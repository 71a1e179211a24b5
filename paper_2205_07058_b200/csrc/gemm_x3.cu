// Train-step dense layers on the tensor cores with fp32-level accuracy:
// 3xTF32 (every operand x = hi + lo with hi = x rounded to TF32 and lo the
// exact fp32 remainder; C = A_hi B_lo + A_lo B_hi + A_hi B_hi, accumulated in
// fp32 in TMEM), tcgen05.mma.cta_group::1.kind::tf32, operands staged by the
// threads (the split needs a register pass) into K-major shared-memory tiles.
//
// The three GEMM shapes of mlp_forward / mlp_backward (src/mlp.cpp:98-230) on
// the feature-major matrices of train.cu (row r of a block = one feature over
// all hits, row stride ld):
//   Fwd  Y[j][n]  = relu(sum_k W[j][k] X[k][n] + b[j])       M = 128 hits, N = O
//   Bwd  dX[j][n] = sum_o W[o][k0 + j] D[o][n]  (x relu'(h))  M = 128 hits, N = K - k0
//   Dw   dW[o][k] = sum_n D[o][n] X[k][n], db[o] = sum_n D[o][n]
//                                              M = O (<= 128), N = K + 1 (bias column), K = hits
// Fwd / Bwd: one CTA per 128-hit tile (persistent), weights pre-split into a
// global image in the shared-memory layout. Dw: each CTA reduces a contiguous
// hit range and adds its partial dW / db with fp32 atomics.
#include "device.cuh"
#include "gemm_x3.cuh"
#include "tc_common.cuh"

namespace svlfb {

namespace {

using namespace tc;

#ifndef SVLF_GEMM_SWAP
#define SVLF_GEMM_SWAP 1  // Fwd / Bwd with M = output features, N = up to 256 hits (k_gemm_feat)
#endif
constexpr uint32_t kChunk = 32;                        // K elements per pipeline stage
constexpr uint32_t kThreads = 512;
constexpr uint32_t kRowsA = 128;                       // M
constexpr uint32_t kMaxN = 144;                        // N <= 144 (Dw: K + 1 <= 135)
constexpr uint32_t kABytes = kRowsA * kChunk * 4;      // 16 KB per hi / lo
constexpr uint32_t kBBytes = kMaxN * kChunk * 4;       // 18 KB per hi / lo
constexpr uint32_t kStageBytes = 2 * kABytes + 2 * kBBytes;
constexpr uint32_t kStages = 3;
constexpr uint32_t kSmemBytes = kStages * kStageBytes + 128;

// K-major, no swizzle, 32-bit elements: core matrix = 8 rows x 16 B (4 elements);
// LBO = 128 B (K-adjacent core matrices), SBO = 1024 B (8-row groups).
__host__ __device__ constexpr uint32_t off32(uint32_t r, uint32_t k) {
    return (r >> 3) * 1024u + (k >> 2) * 128u + (r & 7u) * 16u + (k & 3u) * 4u;
}

__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void split4(const float4 v, uint4& hi, uint4& lo) {
    const float x[4] = {v.x, v.y, v.z, v.w};
    uint32_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h[i]) : "f"(x[i]));
        l[i] = __float_as_uint(__fsub_rn(x[i], __uint_as_float(h[i])));
    }
    hi = make_uint4(h[0], h[1], h[2], h[3]);
    lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Weight image for Fwd / Bwd: chunk c of B (N rows x 32 K) as [hi | lo] in
// the shared-memory layout, zero padded. Fwd: B[j][k] = W[j][k];
// Bwd: B[j][k] = W[k][k0 + j].
__global__ void k_wimage(const float* __restrict__ W, uint32_t O, uint32_t K, uint32_t k0, bool bwd, uint32_t N,
                         uint32_t kred, uint32_t nchunks, uint8_t* img) {
    const uint32_t total = nchunks * N * kChunk;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t c = i / (N * kChunk), rem = i % (N * kChunk), j = rem / kChunk, kk = rem % kChunk;
        const uint32_t k = c * kChunk + kk;
        float v = 0.f;
        if (k < kred) {
            if (!bwd) v = j < O ? W[size_t(j) * K + k] : 0.f;
            else v = (k0 + j < K) ? W[size_t(k) * K + k0 + j] : 0.f;
        }
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
        const float l = __fsub_rn(v, __uint_as_float(h));
        uint8_t* base = img + size_t(c) * 2 * kBBytes;
        *reinterpret_cast<uint32_t*>(base + off32(j, kk)) = h;
        *reinterpret_cast<float*>(base + kBBytes + off32(j, kk)) = l;
    }
}

// MMAs of one staged chunk: 4 K-steps of 8, three split products each.
__device__ __forceinline__ void issue_chunk(uint32_t tmem, uint32_t sa, uint32_t sb, uint32_t idesc, bool first) {
#pragma unroll
    for (uint32_t ks = 0; ks < kChunk / 8; ++ks) {
        const uint64_t ahi = make_desc(sa + ks * 256, 128, 1024), alo = make_desc(sa + kABytes + ks * 256, 128, 1024);
        const uint64_t bhi = make_desc(sb + ks * 256, 128, 1024), blo = make_desc(sb + kBBytes + ks * 256, 128, 1024);
        mma_tf32(tmem, ahi, blo, idesc, (first && ks == 0) ? 0u : 1u);
        mma_tf32(tmem, alo, bhi, idesc, 1u);
        mma_tf32(tmem, ahi, bhi, idesc, 1u);
    }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int kN>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(kN) : "memory");
}

// barriers: [0, kStages) stage reuse, kStages / kStages + 1 accumulator 0 / 1 done
__device__ __forceinline__ uint32_t kernel_init(uint8_t* sm, uint64_t*& bars) {
    bars = reinterpret_cast<uint64_t*>(sm + kStages * kStageBytes);
    uint32_t* holder = reinterpret_cast<uint32_t*>(bars + kStages + 2);
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < kStages + 2; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if ((threadIdx.x >> 5) == 0) tmem_alloc(holder, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    return *holder;
}

__device__ __forceinline__ void kernel_fini(uint32_t tmem) {
    fence_before_sync();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        fence_after_sync();
        tmem_dealloc(tmem, 512);
    }
}

// Chunk pipeline shared by both kernels: chunk g's operands are fetched
// (registers / cp.async) while chunk g-1's MMAs run; stage g % kStages is
// reused once the MMAs of chunk g - kStages have completed.
struct StageSync {
    uint64_t* bars;
    uint32_t phase = 0, used = 0;
    __device__ __forceinline__ void acquire(uint32_t s) {
        if ((used >> s) & 1u) {
            mbar_wait(&bars[s], (phase >> s) & 1u);
            phase ^= 1u << s;
        }
        used |= 1u << s;
    }
    __device__ __forceinline__ void wait_final(uint32_t b = 0) {  // accumulator b's MMAs done
        mbar_wait(&bars[kStages + b], (phase >> (kStages + b)) & 1u);
        phase ^= 1u << (kStages + b);
        fence_after_sync();
    }
};

// ---- Fwd / Bwd: out[j][n0 + m] for 128-hit tiles ------------------------------
template <bool kBwd>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_hits(const float* __restrict__ in, const uint8_t* __restrict__ wimg, float* __restrict__ out,
                const float* __restrict__ bias, const float* __restrict__ mask, uint32_t n, uint32_t ld,
                uint32_t kred, uint32_t N, uint32_t n_out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars;
    const uint32_t tmem = kernel_init(sm, bars);
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t idesc = idesc_tf32(128, N);
    const uint32_t nch = (kred + kChunk - 1) / kChunk;
    const uint32_t ntiles = (n + 127) / 128;
    const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t total = my_tiles * nch;
    StageSync ss{bars};
    constexpr uint32_t kQ = kChunk / 4 / (kThreads / 128);  // K quads per thread per chunk
    const uint32_t m = tid & 127, qb = tid >> 7;              // hit row m, quads qb, qb + kThreads/128, ...
    const uint32_t bwords = (N * kChunk * 4) / 16;            // 16 B words of one hi (or lo) B image chunk
    float4 areg[2][kQ];  // A operands of chunks g and g + 1 (prefetch distance 2)
    auto fetch_a = [&](uint32_t g, float4* dst) {
        const uint32_t tile = blockIdx.x + (g / nch) * gridDim.x, c = g % nch, hit = tile * 128 + m;
#pragma unroll
        for (uint32_t i = 0; i < kQ; ++i) {
            const uint32_t k = c * kChunk + 4 * (qb + i * (kThreads / 128));
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (hit < n) {
                const float* p = in + size_t(k) * ld + hit;
                if (k < kred) v.x = p[0];
                if (k + 1 < kred) v.y = p[ld];
                if (k + 2 < kred) v.z = p[2 * size_t(ld)];
                if (k + 3 < kred) v.w = p[3 * size_t(ld)];
            }
            dst[i] = v;
        }
    };
    auto fetch_b = [&](uint32_t g, uint32_t s) {  // weight image chunk -> stage s (async)
        const uint32_t c = g % nch;
        const uint8_t* src = wimg + size_t(c) * 2 * kBBytes;
        const uint32_t sb = sbase + s * kStageBytes + 2 * kABytes;
        for (uint32_t i = tid; i < 2 * bwords; i += kThreads) {
            const uint32_t off = i < bwords ? 16 * i : kBBytes + 16 * (i - bwords);
            cp_async16(sb + off, src + off);
        }
        cp_async_commit();
    };
    // tile t accumulates in TMEM columns 256 (t & 1); its epilogue runs after
    // the next tile's first chunk has been issued, so the tensor pipe keeps
    // working while the previous tile is written out
    auto epilogue = [&](uint32_t t_local) {
        const uint32_t b = t_local & 1u;
        ss.wait_final(b);
        const uint32_t tile = blockIdx.x + t_local * gridDim.x;
        const uint32_t acc = tmem + 256 * b;
        const uint32_t lane_off = (32u * (warp & 3u)) << 16, r = 32 * (warp & 3u) + (tid & 31);
        const uint32_t groups = kThreads / 128, h = warp >> 2;
        const uint32_t per = ((N + groups - 1) / groups + 31) & ~31u;
        const uint32_t hit_r = tile * 128 + r;
        for (uint32_t c0 = h * per; c0 < min(N, (h + 1) * per); c0 += 32) {
            float v[32];
            tmem_ld32(acc + lane_off + c0, v);
            tmem_wait_ld();
            if (hit_r < n) {
                if constexpr (kBwd) {
                    if (mask) {  // all 32 mask loads in flight before the stores
                        float mk[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            mk[i] = c0 + i < n_out ? __ldg(mask + size_t(c0 + i) * ld + hit_r) : 0.f;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!(mk[i] > 0.f)) v[i] = 0.f;
                    }
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const uint32_t j = c0 + i;
                    if (j < n_out) {
                        float y = v[i];
                        if constexpr (!kBwd) y = fmaxf(y + __ldg(bias + j), 0.f);
                        out[size_t(j) * ld + hit_r] = y;
                    }
                }
            }
        }
        fence_before_sync();  // ordered before the next chunk barrier (accumulator reuse two tiles later)
    };
    auto body = [&](uint32_t g, float4* cur) {
        const uint32_t s = g % kStages, c = g % nch, sn = (g + 1) % kStages, t_local = g / nch;
        const uint32_t sa = sbase + s * kStageBytes, sb = sa + 2 * kABytes;
#pragma unroll
        for (uint32_t i = 0; i < kQ; ++i) {
            uint4 hi, lo;
            split4(cur[i], hi, lo);
            const uint32_t q = qb + i * (kThreads / 128);
            st_shared_v4(sa + off32(m, 4 * q), hi.x, hi.y, hi.z, hi.w);
            st_shared_v4(sa + kABytes + off32(m, 4 * q), lo.x, lo.y, lo.z, lo.w);
        }
        if (g + 2 < total) fetch_a(g + 2, cur);  // this register set is free again
        if (g + 1 < total) {  // next chunk's weights: its stage is free once chunk g+1-kStages completed
            ss.acquire(sn);
            fetch_b(g + 1, sn);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        fence_async_smem();
        fence_before_sync();
        __syncthreads();
        if (tid == 0) {
            fence_after_sync();
            issue_chunk(tmem + 256 * (t_local & 1u), sa, sb, idesc, c == 0);
            mma_commit(&bars[s]);
            if (c + 1 == nch) mma_commit(&bars[kStages + (t_local & 1u)]);
        }
        if (c == 0 && t_local > 0) epilogue(t_local - 1);
    };
    if (total) {
        ss.acquire(0);
        fetch_b(0, 0);
        fetch_a(0, areg[0]);
        if (total > 1) fetch_a(1, areg[1]);
    }
    for (uint32_t g = 0; g < total; g += 2) {
        body(g, areg[0]);
        if (g + 1 < total) body(g + 1, areg[1]);
    }
    if (my_tiles) epilogue(my_tiles - 1);
    kernel_fini(tmem);
}

// ---- Fwd / Bwd with the roles swapped: M = 128 output features (weights as
// the A operand), N = nt hits (<= 256) per tile. Per K-step an MMA reads the
// weight tile once for nt hits instead of once per 128 hits.
constexpr uint32_t kFA = 128 * kChunk * 4;       // 16 KB: A (weights) hi or lo
constexpr uint32_t kFB = 256 * kChunk * 4;       // 32 KB: B (hits) hi or lo
constexpr uint32_t kFStage = 2 * kFA + 2 * kFB;  // 96 KB
constexpr uint32_t kFStages = 2;
constexpr uint32_t kFSmem = kFStages * kFStage + 128;

template <bool kBwd>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_feat(const float* __restrict__ in, const uint8_t* __restrict__ wimg, float* __restrict__ out,
                const float* __restrict__ bias, const float* __restrict__ mask, uint32_t n, uint32_t ld,
                uint32_t kred, uint32_t nt, uint32_t n_out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kFStages * kFStage);  // [0,1] stages, [2,3] accumulators
    uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 4);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (uint32_t i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(holder, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *holder;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t idesc = idesc_tf32(128, nt);
    const uint32_t nch = (kred + kChunk - 1) / kChunk;
    const uint32_t ntiles = (n + nt - 1) / nt;
    const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t total = my_tiles * nch;
    uint32_t phase = 0, used = 0;
    auto acquire = [&](uint32_t st) {
        if ((used >> st) & 1u) {
            mbar_wait(&bars[st], (phase >> st) & 1u);
            phase ^= 1u << st;
        }
        used |= 1u << st;
    };
    // B staging: hit row hn of the tile, K quads qb, qb + 2, qb + 4, qb + 6
    const uint32_t hn = tid & 255, qb = tid >> 8;
    constexpr uint32_t kQ = kChunk / 4 / 2;
    float4 breg[2][kQ];
    auto fetch_b = [&](uint32_t g, float4* dst) {
        const uint32_t tile = blockIdx.x + (g / nch) * gridDim.x, c = g % nch, hit = tile * nt + hn;
        const bool ok = hn < nt && hit < n;
#pragma unroll
        for (uint32_t i = 0; i < kQ; ++i) {
            const uint32_t k = c * kChunk + 4 * (qb + 2 * i);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok) {
                const float* p = in + size_t(k) * ld + hit;
                if (k < kred) v.x = __ldg(p);
                if (k + 1 < kred) v.y = __ldg(p + ld);
                if (k + 2 < kred) v.z = __ldg(p + 2 * size_t(ld));
                if (k + 3 < kred) v.w = __ldg(p + 3 * size_t(ld));
            }
            dst[i] = v;
        }
    };
    auto fetch_a = [&](uint32_t g, uint32_t st) {  // weight image chunk (first 128 rows) -> stage st
        const uint32_t c = g % nch;
        const uint8_t* src = wimg + size_t(c) * 2 * kBBytes;
        const uint32_t sa = sbase + st * kFStage;
        for (uint32_t i = tid; i < 2 * (kFA / 16); i += kThreads) {
            const uint32_t half = i >= kFA / 16, w = i - half * (kFA / 16);
            cp_async16(sa + half * kFA + 16 * w, src + half * kBBytes + 16 * w);
        }
        cp_async_commit();
    };
    auto epilogue = [&](uint32_t t_local) {
        const uint32_t b = t_local & 1u;
        mbar_wait(&bars[2 + b], (phase >> (2 + b)) & 1u);
        phase ^= 1u << (2 + b);
        fence_after_sync();
        const uint32_t tile = blockIdx.x + t_local * gridDim.x;
        const uint32_t lane_off = (32u * (warp & 3u)) << 16, j = 32 * (warp & 3u) + lane, cg = warp >> 2;
        const uint32_t batches = (nt + 31) / 32;
        const float bj = (!kBwd && j < n_out) ? __ldg(bias + j) : 0.f;
        for (uint32_t bt = cg; bt < batches; bt += 4) {
            float v[32];
            tmem_ld32(tmem + 256 * b + lane_off + 32 * bt, v);
            tmem_wait_ld();
            if (j >= n_out) continue;
            const uint32_t h0 = tile * nt + 32 * bt;
            const uint32_t cnt = min(min(32u, nt - 32 * bt), n > h0 ? n - h0 : 0u);
            float* o = out + size_t(j) * ld + h0;
            if constexpr (kBwd) {
                if (mask) {
                    const float* mk = mask + size_t(j) * ld + h0;
                    float mv[32];
                    if (cnt == 32) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float4 q = __ldg(reinterpret_cast<const float4*>(mk) + i);
                            mv[4 * i] = q.x; mv[4 * i + 1] = q.y; mv[4 * i + 2] = q.z; mv[4 * i + 3] = q.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) mv[i] = uint32_t(i) < cnt ? __ldg(mk + i) : 0.f;
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (!(mv[i] > 0.f)) v[i] = 0.f;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i] + bj, 0.f);
            }
            if (cnt == 32) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    reinterpret_cast<float4*>(o)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (uint32_t(i) < cnt) o[i] = v[i];
            }
        }
        fence_before_sync();
    };
    auto body = [&](uint32_t g, float4* cur) {
        const uint32_t st = g % kFStages, c = g % nch, t_local = g / nch;
        const uint32_t sa = sbase + st * kFStage, sb = sa + 2 * kFA;
        if (hn < nt) {
#pragma unroll
            for (uint32_t i = 0; i < kQ; ++i) {
                uint4 hi, lo;
                split4(cur[i], hi, lo);
                const uint32_t q = qb + 2 * i;
                st_shared_v4(sb + off32(hn, 4 * q), hi.x, hi.y, hi.z, hi.w);
                st_shared_v4(sb + kFB + off32(hn, 4 * q), lo.x, lo.y, lo.z, lo.w);
            }
        }
        if (g + 2 < total) fetch_b(g + 2, cur);
        if (g + 1 < total) {
            acquire((g + 1) % kFStages);
            fetch_a(g + 1, (g + 1) % kFStages);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        fence_async_smem();
        fence_before_sync();
        __syncthreads();
        if (tid == 0) {
            fence_after_sync();
            const uint32_t d = tmem + 256 * (t_local & 1u);
#pragma unroll
            for (uint32_t ks = 0; ks < kChunk / 8; ++ks) {
                const uint64_t ahi = make_desc(sa + ks * 256, 128, 1024), alo = make_desc(sa + kFA + ks * 256, 128, 1024);
                const uint64_t bhi = make_desc(sb + ks * 256, 128, 1024), blo = make_desc(sb + kFB + ks * 256, 128, 1024);
                mma_tf32(d, ahi, blo, idesc, (c == 0 && ks == 0) ? 0u : 1u);
                mma_tf32(d, alo, bhi, idesc, 1u);
                mma_tf32(d, ahi, bhi, idesc, 1u);
            }
            mma_commit(&bars[st]);
            if (c + 1 == nch) mma_commit(&bars[2 + (t_local & 1u)]);
        }
        if (c == 0 && t_local > 0) epilogue(t_local - 1);
    };
    if (total) {
        acquire(0);
        fetch_a(0, 0);
        fetch_b(0, breg[0]);
        if (total > 1) fetch_b(1, breg[1]);
    }
    for (uint32_t g = 0; g < total; g += 2) {
        body(g, breg[0]);
        if (g + 1 < total) body(g + 1, breg[1]);
    }
    if (my_tiles) epilogue(my_tiles - 1);
    fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        fence_after_sync();
        tmem_dealloc(tmem, 512);
    }
}

// ---- Dw: dW[o][k] += sum over this CTA's hits of D[o][n] X[k][n] -------------
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_dw(const float* __restrict__ dmat, const float* __restrict__ xmat, float* __restrict__ dW,
              float* __restrict__ db, uint32_t n, uint32_t ld, uint32_t O, uint32_t K, uint32_t N,
              uint32_t hits_per_cta) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars;
    const uint32_t tmem = kernel_init(sm, bars);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t idesc = idesc_tf32(128, N);
    const uint32_t h0 = blockIdx.x * hits_per_cta, h1 = min(n, h0 + hits_per_cta);
    const uint32_t nch = h0 < h1 ? (h1 - h0 + kChunk - 1) / kChunk : 0;
    StageSync ss{bars};
    // work units of a chunk: 8 rows x 4 quads (one warp instruction, conflict-free
    // v4 stores); A units first (128 rows), then B units (N rows)
    const uint32_t r_lo = lane & 7, q_lo = lane >> 3;
    const uint32_t units = (kRowsA / 8) * 2 + (N / 8) * 2;
    constexpr uint32_t kU = ((kRowsA / 8) * 2 + (kMaxN / 8) * 2 + kThreads / 32 - 1) / (kThreads / 32);
    float4 reg[2][kU];  // chunks c and c + 1 (prefetch distance 2)
    auto unit_of = [&](uint32_t u, uint32_t& r, uint32_t& q, bool& isA) {
        isA = u < (kRowsA / 8) * 2;
        const uint32_t t = isA ? u : u - (kRowsA / 8) * 2;
        r = 8 * (t >> 1) + r_lo;
        q = 4 * (t & 1) + q_lo;
    };
    auto fetch = [&](uint32_t c, float4* dst) {
        const uint32_t hb = h0 + c * kChunk;
#pragma unroll
        for (uint32_t i = 0; i < kU; ++i) {
            const uint32_t u = warp + i * (kThreads / 32);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (u < units) {
                uint32_t r, q;
                bool isA;
                unit_of(u, r, q, isA);
                const uint32_t hit = hb + 4 * q;
                const float* p = nullptr;
                if (isA && r < O) p = dmat + size_t(r) * ld + hit;
                else if (!isA && r < K) p = xmat + size_t(r) * ld + hit;
                if (p) {
                    if (hit + 3 < h1) {
                        v = *reinterpret_cast<const float4*>(p);
                    } else {
                        if (hit < h1) v.x = p[0];
                        if (hit + 1 < h1) v.y = p[1];
                        if (hit + 2 < h1) v.z = p[2];
                    }
                } else if (!isA && r == K) {  // bias column: ones over the valid hits
                    v.x = hit < h1 ? 1.f : 0.f;
                    v.y = hit + 1 < h1 ? 1.f : 0.f;
                    v.z = hit + 2 < h1 ? 1.f : 0.f;
                    v.w = hit + 3 < h1 ? 1.f : 0.f;
                }
            }
            dst[i] = v;
        }
    };
    auto body = [&](uint32_t c, float4* cur) {
        const uint32_t s = c % kStages;
        ss.acquire(s);
        const uint32_t sa = sbase + s * kStageBytes, sb = sa + 2 * kABytes;
#pragma unroll
        for (uint32_t i = 0; i < kU; ++i) {
            const uint32_t u = warp + i * (kThreads / 32);
            if (u < units) {
                uint32_t r, q;
                bool isA;
                unit_of(u, r, q, isA);
                uint4 hi, lo;
                split4(cur[i], hi, lo);
                const uint32_t base = isA ? sa : sb, lo_off = isA ? kABytes : kBBytes;
                st_shared_v4(base + off32(r, 4 * q), hi.x, hi.y, hi.z, hi.w);
                st_shared_v4(base + lo_off + off32(r, 4 * q), lo.x, lo.y, lo.z, lo.w);
            }
        }
        if (c + 2 < nch) fetch(c + 2, cur);  // in flight during the next chunks' MMAs
        fence_async_smem();
        fence_before_sync();
        __syncthreads();
        if (tid == 0) {
            fence_after_sync();
            issue_chunk(tmem, sa, sb, idesc, c == 0);
            mma_commit(&bars[s]);
            if (c + 1 == nch) mma_commit(&bars[kStages]);
        }
    };
    if (nch) fetch(0, reg[0]);
    if (nch > 1) fetch(1, reg[1]);
    for (uint32_t c = 0; c < nch; c += 2) {
        body(c, reg[0]);
        if (c + 1 < nch) body(c + 1, reg[1]);
    }
    if (nch) {
        ss.wait_final();
        const uint32_t lane_off = (32u * (warp & 3u)) << 16, o = 32 * (warp & 3u) + lane;
        const uint32_t groups = kThreads / 128, h = warp >> 2;
        const uint32_t per = ((N + groups - 1) / groups + 31) & ~31u;
        for (uint32_t c0 = h * per; c0 < min(N, (h + 1) * per); c0 += 32) {
            float v[32];
            tmem_ld32(tmem + lane_off + c0, v);
            tmem_wait_ld();
            if (o < O) {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const uint32_t j = c0 + i;
                    if (j < K) atomicAdd(dW + size_t(o) * K + j, v[i]);
                    else if (j == K) atomicAdd(db + o, v[i]);
                }
            }
        }
    }
    kernel_fini(tmem);
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
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_hits<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_hits<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_dw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_feat<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFSmem)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_feat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFSmem)));
        g_attr = true;
    }
}

uint32_t round16(uint32_t v) { return (v + 15u) & ~15u; }

}  // namespace

size_t gemm_x3_image_bytes(uint32_t kred) { return size_t((kred + kChunk - 1) / kChunk) * 2 * kBBytes; }

// hits per tile for the swapped kernels: <= 256, a multiple of 16, sized so
// the tiles fill whole waves of one CTA per SM
static uint32_t tile_hits(uint32_t n) {
    const uint32_t sms = uint32_t(g_sms), waves = std::max<uint32_t>(1, (n + sms * 256 - 1) / (sms * 256));
    const uint32_t per = (n + sms * waves - 1) / (sms * waves);
    return std::min<uint32_t>(256, std::max<uint32_t>(16, (per + 15) / 16 * 16));
}

void gemm_x3_fwd(const float* x, const float* W, const float* bias, float* y, uint32_t O, uint32_t K, uint32_t n,
                 uint32_t ld, uint8_t* img, cudaStream_t s) {
    if (n == 0) return;
    setup();
    const uint32_t nch = (K + kChunk - 1) / kChunk;
#if SVLF_GEMM_SWAP
    k_wimage<<<64, 256, 0, s>>>(W, O, K, 0, false, 128, K, nch, img);
    const uint32_t nt = tile_hits(n), tiles = (n + nt - 1) / nt;
    k_gemm_feat<false><<<std::min<uint32_t>(tiles, uint32_t(g_sms)), kThreads, kFSmem, s>>>(x, img, y, bias, nullptr,
                                                                                              n, ld, K, nt, O);
#else
    const uint32_t N = round16(O);
    k_wimage<<<64, 256, 0, s>>>(W, O, K, 0, false, N, K, nch, img);
    const uint32_t tiles = (n + 127) / 128;
    k_gemm_hits<false><<<std::min<uint32_t>(tiles, uint32_t(g_sms)), kThreads, kSmemBytes, s>>>(
        x, img, y, bias, nullptr, n, ld, K, N, O);
#endif
    note_launch(2);
}

void gemm_x3_bwd(const float* d, const float* W, uint32_t O, uint32_t K, uint32_t k0, float* dx, const float* mask,
                 uint32_t n, uint32_t ld, uint8_t* img, cudaStream_t s) {
    if (n == 0) return;
    setup();
    const uint32_t nout = K - k0, nch = (O + kChunk - 1) / kChunk;
#if SVLF_GEMM_SWAP
    k_wimage<<<64, 256, 0, s>>>(W, O, K, k0, true, 128, O, nch, img);
    const uint32_t nt = tile_hits(n), tiles = (n + nt - 1) / nt;
    k_gemm_feat<true><<<std::min<uint32_t>(tiles, uint32_t(g_sms)), kThreads, kFSmem, s>>>(d, img, dx, nullptr, mask,
                                                                                             n, ld, O, nt, nout);
#else
    const uint32_t N = round16(nout);
    k_wimage<<<64, 256, 0, s>>>(W, O, K, k0, true, N, O, nch, img);
    const uint32_t tiles = (n + 127) / 128;
    k_gemm_hits<true><<<std::min<uint32_t>(tiles, uint32_t(g_sms)), kThreads, kSmemBytes, s>>>(
        d, img, dx, nullptr, mask, n, ld, O, N, nout);
#endif
    note_launch(2);
}

void gemm_x3_dw(const float* d, const float* x, uint32_t O, uint32_t K, float* dW, float* db, uint32_t n,
                uint32_t ld, cudaStream_t s) {
    SVLF_CUDA(cudaMemsetAsync(dW, 0, size_t(O) * K * 4, s));
    SVLF_CUDA(cudaMemsetAsync(db, 0, size_t(O) * 4, s));
    if (n == 0) return;
    setup();
    const uint32_t N = round16(K + 1);
    const uint32_t ctas = uint32_t(g_sms);
    const uint32_t per = ((n + ctas - 1) / ctas + kChunk - 1) / kChunk * kChunk;
    k_gemm_dw<<<(n + per - 1) / per, kThreads, kSmemBytes, s>>>(d, x, dW, db, n, ld, O, K, N, per);
    note_launch();
}

}  // namespace svlfb
