// Train-step dense layers on the tensor cores with fp32-level accuracy:
// 3xTF32 (every operand x = hi + lo with hi = x rounded to TF32 and lo the
// exact fp32 remainder; C = A_hi B_lo + A_lo B_hi + A_hi B_hi, accumulated in
// fp32 in TMEM), tcgen05.mma.cta_group::1.kind::tf32, operands staged by the
// threads (the split needs a register pass) into K-major shared-memory tiles.
//
// The three GEMM shapes of mlp_forward / mlp_backward (src/mlp.cpp:98-230) on
// the feature-major matrices of train.cu (row r of a block = one feature over
// all hits, row stride ld):
//   Fwd  Y[j][n]  = relu(sum_k W[j][k] X[k][n] + b[j])       M = 128 output features, N = hits
//   Bwd  dX[j][n] = sum_o W[o][k0 + j] D[o][n]  (x relu'(h))  M = 128 input features, N = hits
//   Dw   dW[o][k] = sum_n D[o][n] X[k][n], db[o] = sum_n D[o][n]
//                                              M = O (<= 128), N = K + 1 (bias column), K = hits
// Fwd / Bwd: persistent CTAs over tiles of up to 256 hits, the weight operand
// from a pre-split global image (one launch builds every layer's image per
// step). Dw: each CTA reduces a contiguous hit range into its own partial;
// the partials are summed in CTA order (deterministic, no atomics).
// The hit count is read on the device, so nothing here needs the host.
#include "device.cuh"
#include "gemm_x3.cuh"
#include "tc_common.cuh"

namespace svlfb {

namespace {

using namespace tc;

constexpr uint32_t kChunk = 32;  // K elements per pipeline stage
constexpr uint32_t kThreads = 512;

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

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int kN>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(kN) : "memory");
}

// ---- weight images ------------------------------------------------------------
// Image of one job: chunk c (32 K) of the 128-row B operand as [hi | lo], each
// 16 KB in the shared-memory layout, zero padded.
constexpr uint32_t kFA = 128 * kChunk * 4;  // 16 KB: one 128 x 32 hi (or lo) tile

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
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
        const float l = __fsub_rn(v, __uint_as_float(h));
        uint8_t* base = img + size_t(c) * 2 * kFA;
        *reinterpret_cast<uint32_t*>(base + off32(j, kk)) = h;
        *reinterpret_cast<float*>(base + kFA + off32(j, kk)) = l;
    }
}

// ---- Fwd / Bwd: M = 128 output features (weights as the A operand), N = nt
// hits (<= 256) per tile. Per K-step an MMA reads the weight tile once for nt
// hits. The hit operand is split in registers and staged K-major.
constexpr uint32_t kFB = 256 * kChunk * 4;       // 32 KB: B (hits) hi or lo
constexpr uint32_t kFStage = 2 * kFA + 2 * kFB;  // 96 KB
constexpr uint32_t kFStages = 2;
constexpr uint32_t kFSmem = kFStages * kFStage + 128;

// hits per tile: <= 256, a multiple of 16, sized so the tiles fill whole waves of the grid
__device__ __forceinline__ uint32_t tile_hits(uint32_t n, uint32_t ctas) {
    const uint32_t waves = max(1u, (n + ctas * 256 - 1) / (ctas * 256));
    const uint32_t per = (n + ctas * waves - 1) / (ctas * waves);
    return min(256u, max(16u, (per + 15) / 16 * 16));
}

template <bool kBwd>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_feat(const float* __restrict__ in, const uint8_t* __restrict__ wimg, float* __restrict__ out,
                const float* __restrict__ bias, const float* __restrict__ mask, const uint32_t* __restrict__ n_dev,
                uint32_t cap, uint32_t ld, uint32_t kred, uint32_t n_out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kFStages * kFStage);  // [0,1] stages, [2,3] accumulators
    uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 4);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t n = min(*n_dev, cap);
    const uint32_t nt = tile_hits(n, gridDim.x);
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
    auto fetch_a = [&](uint32_t g, uint32_t st) {  // weight image chunk -> stage st
        const uint32_t c = g % nch;
        const uint8_t* src = wimg + size_t(c) * 2 * kFA;
        const uint32_t sa = sbase + st * kFStage;
        for (uint32_t i = tid; i < 2 * (kFA / 16); i += kThreads) cp_async16(sa + 16 * i, src + 16 * i);
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

// ---- Dw: part[cta][o][k] = sum over this CTA's hits of D[o][n] X[k][n] ---------
constexpr uint32_t kRowsA = 128;                   // M
constexpr uint32_t kMaxN = 144;                    // N = K + 1 <= 144
constexpr uint32_t kABytes = kRowsA * kChunk * 4;  // 16 KB per hi / lo
constexpr uint32_t kBBytes = kMaxN * kChunk * 4;   // 18 KB per hi / lo
constexpr uint32_t kStageBytes = 2 * kABytes + 2 * kBBytes;
constexpr uint32_t kStages = 3;
constexpr uint32_t kSmemBytes = kStages * kStageBytes + 128;

template <bool kX3>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_dw(const float* __restrict__ dmat, const float* __restrict__ xmat, float* __restrict__ part,
              const uint32_t* __restrict__ n_dev, uint32_t cap, uint32_t ld, uint32_t O, uint32_t K, uint32_t N) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kStages * kStageBytes);  // stages, then the accumulator
    uint32_t* holder = reinterpret_cast<uint32_t*>(bars + kStages + 1);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (uint32_t i = 0; i < kStages + 1; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(holder, 256);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *holder;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t idesc = idesc_tf32(128, N);
    const uint32_t n = min(*n_dev, cap);
    const uint32_t per = ((n + gridDim.x - 1) / gridDim.x + kChunk - 1) / kChunk * kChunk;
    const uint32_t h0 = min(n, blockIdx.x * per), h1 = min(n, h0 + per);
    const uint32_t nch = (h1 - h0 + kChunk - 1) / kChunk;
    uint32_t phase = 0, used = 0;
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
        if ((used >> s) & 1u) {
            mbar_wait(&bars[s], (phase >> s) & 1u);
            phase ^= 1u << s;
        }
        used |= 1u << s;
        const uint32_t sa = sbase + s * kStageBytes, sb = sa + 2 * kABytes;
#pragma unroll
        for (uint32_t i = 0; i < kU; ++i) {
            const uint32_t u = warp + i * (kThreads / 32);
            if (u < units) {
                uint32_t r, q;
                bool isA;
                unit_of(u, r, q, isA);
                const uint32_t base = isA ? sa : sb, lo_off = isA ? kABytes : kBBytes;
                if constexpr (kX3) {
                    uint4 hi, lo;
                    split4(cur[i], hi, lo);
                    st_shared_v4(base + off32(r, 4 * q), hi.x, hi.y, hi.z, hi.w);
                    st_shared_v4(base + lo_off + off32(r, 4 * q), lo.x, lo.y, lo.z, lo.w);
                } else {  // plain TF32: the tensor core truncates the fp32 operand bits
                    st_shared_v4(base + off32(r, 4 * q), __float_as_uint(cur[i].x), __float_as_uint(cur[i].y),
                                 __float_as_uint(cur[i].z), __float_as_uint(cur[i].w));
                }
            }
        }
        if (c + 2 < nch) fetch(c + 2, cur);  // in flight during the next chunks' MMAs
        fence_async_smem();
        fence_before_sync();
        __syncthreads();
        if (tid == 0) {
            fence_after_sync();
#pragma unroll
            for (uint32_t ks = 0; ks < kChunk / 8; ++ks) {
                const uint64_t ahi = make_desc(sa + ks * 256, 128, 1024), bhi = make_desc(sb + ks * 256, 128, 1024);
                if constexpr (kX3) {
                    const uint64_t alo = make_desc(sa + kABytes + ks * 256, 128, 1024);
                    const uint64_t blo = make_desc(sb + kBBytes + ks * 256, 128, 1024);
                    mma_tf32(tmem, ahi, blo, idesc, (c == 0 && ks == 0) ? 0u : 1u);
                    mma_tf32(tmem, alo, bhi, idesc, 1u);
                    mma_tf32(tmem, ahi, bhi, idesc, 1u);
                } else {
                    mma_tf32(tmem, ahi, bhi, idesc, (c == 0 && ks == 0) ? 0u : 1u);
                }
            }
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
    // epilogue: this CTA's partial, rows o < O, columns j <= K (zeros for a CTA without hits)
    if (nch) {
        mbar_wait(&bars[kStages], 0);
        fence_after_sync();
    }
    const uint32_t lane_off = (32u * (warp & 3u)) << 16, o = 32 * (warp & 3u) + lane;
    const uint32_t groups = kThreads / 128, h = warp >> 2;
    const uint32_t per_g = ((N + groups - 1) / groups + 31) & ~31u;
    float* dst = part + (size_t(blockIdx.x) * O + o) * (K + 1);
    for (uint32_t c0 = h * per_g; c0 < min(N, (h + 1) * per_g); c0 += 32) {
        float v[32];
        if (nch) {
            tmem_ld32(tmem + lane_off + c0, v);
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
    fence_before_sync();
    __syncthreads();
    if (warp == 0) {
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

int g_sms = 0;
bool g_attr = false;

void setup() {
    if (!g_sms) {
        int dev = 0;
        SVLF_CUDA(cudaGetDevice(&dev));
        SVLF_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (!g_attr) {
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_dw<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_dw<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_feat<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFSmem)));
        SVLF_CUDA(cudaFuncSetAttribute(k_gemm_feat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFSmem)));
        g_attr = true;
    }
}

uint32_t round16(uint32_t v) { return (v + 15u) & ~15u; }

// persistent grid: one CTA per SM, fewer when the capacity has fewer tiles of 16 hits
uint32_t feat_grid(uint32_t cap) { return std::max<uint32_t>(1, std::min<uint32_t>(uint32_t(g_sms), (cap + 15) / 16)); }
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
                 const uint32_t* n_dev, uint32_t cap, uint32_t ld, cudaStream_t s) {
    if (cap == 0) return;
    setup();
    k_gemm_feat<false><<<feat_grid(cap), kThreads, kFSmem, s>>>(x, img, y, bias, nullptr, n_dev, cap, ld, K, O);
    note_launch();
}

void gemm_x3_bwd(const float* d, const uint8_t* img, uint32_t O, uint32_t K, uint32_t k0, float* dx,
                 const float* mask, const uint32_t* n_dev, uint32_t cap, uint32_t ld, cudaStream_t s) {
    if (cap == 0) return;
    setup();
    k_gemm_feat<true><<<feat_grid(cap), kThreads, kFSmem, s>>>(d, img, dx, nullptr, mask, n_dev, cap, ld, O, K - k0);
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

void gemm_x3_dw(const float* d, const float* x, uint32_t O, uint32_t K, float* dW, float* db, const uint32_t* n_dev,
                uint32_t cap, uint32_t ld, float* part, int products, cudaStream_t s) {
    setup();
    const uint32_t N = round16(K + 1), ctas = dw_grid(cap);
    if (products == 1)
        k_gemm_dw<false><<<ctas, kThreads, kSmemBytes, s>>>(d, x, part, n_dev, cap, ld, O, K, N);
    else
        k_gemm_dw<true><<<ctas, kThreads, kSmemBytes, s>>>(d, x, part, n_dev, cap, ld, O, K, N);
    const uint32_t per = O * (K + 1);
    k_dw_reduce<<<(per + kRedElems - 1) / kRedElems, kRedGroups * kRedElems, 0, s>>>(part, ctas, O, K, dW, db);
    note_launch(2);
}

}  // namespace svlfb
