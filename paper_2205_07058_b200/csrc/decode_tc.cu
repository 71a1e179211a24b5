// Fused tcgen05 decoder (bf16 operands, fp32 accumulation in TMEM).
//
// One persistent CTA per SM, 256 threads = two independent 128-row "slots".
// A slot owns one M=128 tile of hits at a time (thread r = row r = one hit)
// and runs the whole per-hit chain of the reference's batch_forward
// (src/voxel_batch.hpp:69-151) for its tile:
//   geometry (fp64): x1, x2, parameterize_ray, trilinear weights
//   gather psi_T(x1), psi_T(x2) (bf16 feature rows, fp32 accumulate) -> A tile
//   MMA  f_T layer 0:  [128 x 144] x [144 x 128] -> TMEM        (9 x K16)
//   epilogue: +b, relu, f_T head (tau relu, eta sigmoid) on CUDA cores
//   x_s = eta x1 + (1-eta) x2, gather psi_C(x_s) -> A tile
//   MMA  f_C layer 0:  [128 x 48] x [48 x 128]                 (3 x K16)
//   epilogue +b, relu -> bf16 A tile; MMA f_C layer 1 (8 x K16); same for
//   layer 2; epilogue: +b, relu, f_C head (3 x sigmoid).
// The two slots interleave, so one slot's MMAs overlap the other slot's
// gathers/epilogues; all four weight matrices stay resident in shared memory
// for the whole kernel (112 KB bf16), each slot has one 36 KB A buffer and a
// 128-column fp32 TMEM accumulator.
//
// Input K ordering is permuted so the 16-byte core-matrix chunks are aligned:
//   f_T A columns: [psi_T(x1) 0..63 | psi_T(x2) 64..127 | r6 128..133 | 0]
//   f_C A columns: [psi_C(x_s) 0..31 | r6 32..37 | 0]
// and the packed weights use the same permutation, so the products equal
// the reference's W . [r6 | psi | psi] (only the fp32 summation order differs).
#include "device.cuh"
#include "tc_common.cuh"

namespace svlfb {

namespace {

using namespace tc;

constexpr uint32_t KT = 144;  // f_T input, padded
constexpr uint32_t KC = 48;   // f_C input, padded
constexpr uint32_t KH = 128;  // hidden

// pack layout (bytes)
constexpr uint32_t OFF_WT0 = 0;
constexpr uint32_t OFF_WC0 = OFF_WT0 + 128 * KT * 2;  // 36864
constexpr uint32_t OFF_WC1 = OFF_WC0 + 128 * KC * 2;  // 49152
constexpr uint32_t OFF_WC2 = OFF_WC1 + 128 * KH * 2;  // 81920
constexpr uint32_t OFF_VEC = OFF_WC2 + 128 * KH * 2;  // 114688
// fp32 vectors (float offsets within VEC)
constexpr uint32_t V_BT0 = 0, V_WT1 = 128, V_BT1 = 384, V_BC0 = 388, V_BC1 = 516, V_BC2 = 644, V_WC3 = 772,
                   V_BC3 = 1156, V_N = 1160;
constexpr uint32_t SMEM_WEIGHTS = OFF_VEC + V_N * 4;  // 119328
constexpr uint32_t OFF_FEAT = (SMEM_WEIGHTS + 255) & ~255u;
// kernel smem
constexpr uint32_t SM_A0 = (SMEM_WEIGHTS + 1023) & ~1023u;  // 120832
constexpr uint32_t A_BYTES = 128 * KT * 2;                  // 36864
constexpr uint32_t SM_BAR = SM_A0 + 2 * A_BYTES;
constexpr uint32_t SM_TOTAL = SM_BAR + 64;

constexpr uint32_t kIdesc = make_idesc(128, 128, true);

__device__ __forceinline__ float sigmoidf_fast(float x) { return 1.0f / (1.0f + __expf(-x)); }

// ---- pack: fp32 flat params -> bf16 UMMA tiles + fp32 vectors + bf16 features
__global__ void k_pack_tc(const float* __restrict__ mt, const float* __restrict__ mc, uint8_t* pack) {
    using D = DecOffsets;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    __nv_bfloat16* wt0 = reinterpret_cast<__nv_bfloat16*>(pack + OFF_WT0);
    __nv_bfloat16* wc0 = reinterpret_cast<__nv_bfloat16*>(pack + OFF_WC0);
    __nv_bfloat16* wc1 = reinterpret_cast<__nv_bfloat16*>(pack + OFF_WC1);
    __nv_bfloat16* wc2 = reinterpret_cast<__nv_bfloat16*>(pack + OFF_WC2);
    float* vec = reinterpret_cast<float*>(pack + OFF_VEC);
    if (tid < 128 * KT) {  // f_T layer 0, K permuted
        const uint32_t n = tid / KT, k = tid % KT;
        const int src = k < 128 ? int(6 + k) : (k < 134 ? int(k - 128) : -1);
        const float w = src >= 0 ? mt[D::T_W0 + n * kInT + src] : 0.f;
        wt0[core_offset(n, k, KT) / 2] = __float2bfloat16_rn(w);
    }
    if (tid < 128 * KC) {  // f_C layer 0
        const uint32_t n = tid / KC, k = tid % KC;
        const int src = k < 32 ? int(6 + k) : (k < 38 ? int(k - 32) : -1);
        const float w = src >= 0 ? mc[D::C_W0 + n * kInC + src] : 0.f;
        wc0[core_offset(n, k, KC) / 2] = __float2bfloat16_rn(w);
    }
    if (tid < 128 * KH) {
        const uint32_t n = tid / KH, k = tid % KH;
        wc1[core_offset(n, k, KH) / 2] = __float2bfloat16_rn(mc[D::C_W1 + n * kHid + k]);
        wc2[core_offset(n, k, KH) / 2] = __float2bfloat16_rn(mc[D::C_W2 + n * kHid + k]);
    }
    if (tid < 128) {
        vec[V_BT0 + tid] = mt[D::T_B0 + tid];
        vec[V_BC0 + tid] = mc[D::C_B0 + tid];
        vec[V_BC1 + tid] = mc[D::C_B1 + tid];
        vec[V_BC2 + tid] = mc[D::C_B2 + tid];
    }
    if (tid < 256) vec[V_WT1 + tid] = mt[D::T_W1 + tid];
    if (tid < 384) vec[V_WC3 + tid] = mc[D::C_W3 + tid];
    if (tid < 4) vec[V_BT1 + tid] = tid < 2 ? mt[D::T_B1 + tid] : 0.f;
    if (tid < 4) vec[V_BC3 + tid] = tid < 3 ? mc[D::C_B3 + tid] : 0.f;
}

__global__ void k_feat_bf16(const float* __restrict__ src, __nv_bfloat16* dst, size_t n) {
    const size_t i = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) * 4;
    if (i + 3 < n) {
        const float4 v = *reinterpret_cast<const float4*>(src + i);
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
        *reinterpret_cast<__nv_bfloat162*>(dst + i) = a;
        *reinterpret_cast<__nv_bfloat162*>(dst + i + 2) = b;
    } else {
        for (size_t k = i; k < n; ++k) dst[k] = __float2bfloat16_rn(src[k]);
    }
}

__device__ __forceinline__ void unpack8(const uint4& q, float* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

// Issue the K-loop of one layer: D[tmem] = A[128 x K] . B[128 x K]^T
__device__ __forceinline__ void issue_layer(uint32_t tmem_d, uint32_t a_base, uint32_t b_base, uint32_t K) {
    const uint32_t sbo = (K / 8) * 128;
#pragma unroll 1
    for (uint32_t k = 0; k < K / 16; ++k) {
        const uint64_t ad = make_desc(a_base + 256 * k, 128, sbo);
        const uint64_t bd = make_desc(b_base + 256 * k, 128, sbo);
        mma_f16(tmem_d, ad, bd, kIdesc, k > 0);
    }
}

__global__ void __launch_bounds__(256, 1)
    k_decode_tc(DevOctree T, const uint8_t* __restrict__ pack, const __nv_bfloat16* __restrict__ ft16,
                const __nv_bfloat16* __restrict__ fc16, const double* __restrict__ rays,
                const uint32_t* __restrict__ hit_ray, const uint32_t* __restrict__ hit_leaf,
                const double* __restrict__ hit_tin, const double* __restrict__ hit_tout, uint32_t n, HitOut out,
                int* err) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t tid = threadIdx.x;
    const uint32_t slot = tid >> 7;
    const uint32_t r = tid & 127;
    const uint32_t warp = tid >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + SM_BAR);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sm + SM_BAR + 32);
    const float* vec = reinterpret_cast<const float*>(sm + OFF_VEC);

    // weights + vectors -> smem (once per CTA)
    {
        const uint4* src = reinterpret_cast<const uint4*>(pack);
        uint4* dst = reinterpret_cast<uint4*>(sm);
        for (uint32_t i = tid; i < SMEM_WEIGHTS / 16; i += blockDim.x) dst[i] = src[i];
    }
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(tmem_holder, 256);
    fence_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tmem_holder;
    const uint32_t tmem_acc = tmem + slot * 128;                   // column offset
    const uint32_t tmem_row = tmem_acc + ((32u * (warp & 3u)) << 16);  // this warp's lanes
    const uint32_t sbase = smem_u32(sm);
    const uint32_t a_base = sbase + SM_A0 + slot * A_BYTES;
    uint8_t* A = sm + SM_A0 + slot * A_BYTES;
    uint64_t* bar = &bars[slot];
    uint32_t phase = 0;
    const uint32_t ntiles = (n + 127) / 128;
    const uint32_t bar_id = 1 + slot;

    for (uint32_t tile = blockIdx.x * 2 + slot; tile < ntiles; tile += gridDim.x * 2) {
        const uint32_t j = tile * 128 + r;
        bool valid = j < n;
        float r6[6] = {0, 0, 0, 0, 0, 0};
        uint32_t corners[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        float w1[8], w2[8];
        double x1[3] = {0, 0, 0}, x2[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
        if (valid) {
            Ray ray;
            const uint32_t ri = hit_ray[j];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                ray.o[a] = rays[6 * size_t(ri) + a];
                ray.d[a] = rays[6 * size_t(ri) + 3 + a];
            }
            const uint32_t leaf = hit_leaf[j];
            leaf_box(T, leaf, lo, hi);
            ray_at(ray, hit_tin[j], x1);
            ray_at(ray, hit_tout[j], x2);
            if (!parameterize(ray, lo, hi, r6)) {
                raise_error(err, kErrTangentRay);
                valid = false;
            }
            if (!trilinear_at(x1, lo, hi, T.cell_size, w1) || !trilinear_at(x2, lo, hi, T.cell_size, w2)) {
                raise_error(err, kErrPointNotInVoxel);
                valid = false;
            }
            const uint4* cp = reinterpret_cast<const uint4*>(T.corners + 8 * size_t(leaf));
            const uint4 c0 = __ldg(cp), c1 = __ldg(cp + 1);
            corners[0] = c0.x; corners[1] = c0.y; corners[2] = c0.z; corners[3] = c0.w;
            corners[4] = c1.x; corners[5] = c1.y; corners[6] = c1.z; corners[7] = c1.w;
        }
        if (!valid) {
#pragma unroll
            for (int b = 0; b < 8; ++b) w1[b] = w2[b] = 0.f;
        }

        // ---- gather psi_T(x1), psi_T(x2) -> A (K = 144)
#pragma unroll 1
        for (uint32_t c = 0; c < 8; ++c) {  // 8-dim chunks of the 64 thickness features
            float a1[8], a2[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a1[i] = a2[i] = 0.f;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(ft16 + size_t(corners[b]) * 64) + c);
                float f[8];
                unpack8(q, f);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    a1[i] = __fmaf_rn(w1[b], f[i], a1[i]);
                    a2[i] = __fmaf_rn(w2[b], f[i], a2[i]);
                }
            }
            st_shared_v4(a_base + core_offset(r, 8 * c, KT), pack_bf16x2(a1[0], a1[1]), pack_bf16x2(a1[2], a1[3]),
                         pack_bf16x2(a1[4], a1[5]), pack_bf16x2(a1[6], a1[7]));
            st_shared_v4(a_base + core_offset(r, 64 + 8 * c, KT), pack_bf16x2(a2[0], a2[1]),
                         pack_bf16x2(a2[2], a2[3]), pack_bf16x2(a2[4], a2[5]), pack_bf16x2(a2[6], a2[7]));
        }
        st_shared_v4(a_base + core_offset(r, 128, KT), pack_bf16x2(r6[0], r6[1]), pack_bf16x2(r6[2], r6[3]),
                     pack_bf16x2(r6[4], r6[5]), 0u);
        st_shared_v4(a_base + core_offset(r, 136, KT), 0u, 0u, 0u, 0u);

        fence_async_smem();
        fence_before_sync();
        named_sync(bar_id, 128);
        if (r == 0) {
            fence_after_sync();
            issue_layer(tmem_acc, a_base, sbase + OFF_WT0, KT);
            mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        fence_after_sync();

        // ---- epilogue f_T: +b, relu, head (tau, eta)
        float y0 = vec[V_BT1], y1 = vec[V_BT1 + 1];
#pragma unroll 1
        for (uint32_t c = 0; c < 4; ++c) {
            float v[32];
            tmem_ld32(tmem_row + 32 * c, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const uint32_t col = 32 * c + i;
                const float h = fmaxf(v[i] + vec[V_BT0 + col], 0.f);
                y0 = __fmaf_rn(vec[V_WT1 + col], h, y0);
                y1 = __fmaf_rn(vec[V_WT1 + 128 + col], h, y1);
            }
        }
        const float tau = fmaxf(y0, 0.f);
        const float eta = sigmoidf_fast(y1);

        // ---- x_s, psi_C(x_s) -> A (K = 48)
        float ws[8];
        if (valid) {
            const double e = double(eta), ome = 1.0 - e;
            double xs[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) xs[a] = dadd(dmul(x1[a], e), dmul(x2[a], ome));
            if (!trilinear_at(xs, lo, hi, T.cell_size, ws)) {
                raise_error(err, kErrPointNotInVoxel);
                valid = false;
            }
        }
        if (!valid) {
#pragma unroll
            for (int b = 0; b < 8; ++b) ws[b] = 0.f;
        }
#pragma unroll 1
        for (uint32_t c = 0; c < 4; ++c) {
            float a1[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a1[i] = 0.f;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(fc16 + size_t(corners[b]) * 32) + c);
                float f[8];
                unpack8(q, f);
#pragma unroll
                for (int i = 0; i < 8; ++i) a1[i] = __fmaf_rn(ws[b], f[i], a1[i]);
            }
            st_shared_v4(a_base + core_offset(r, 8 * c, KC), pack_bf16x2(a1[0], a1[1]), pack_bf16x2(a1[2], a1[3]),
                         pack_bf16x2(a1[4], a1[5]), pack_bf16x2(a1[6], a1[7]));
        }
        st_shared_v4(a_base + core_offset(r, 32, KC), pack_bf16x2(r6[0], r6[1]), pack_bf16x2(r6[2], r6[3]),
                     pack_bf16x2(r6[4], r6[5]), 0u);
        st_shared_v4(a_base + core_offset(r, 40, KC), 0u, 0u, 0u, 0u);

        fence_async_smem();
        fence_before_sync();
        named_sync(bar_id, 128);
        if (r == 0) {
            fence_after_sync();
            issue_layer(tmem_acc, a_base, sbase + OFF_WC0, KC);
            mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        fence_after_sync();

        // ---- hidden layers of f_C: epilogue -> bf16 A (K = 128) -> next MMA
#pragma unroll 1
        for (uint32_t layer = 0; layer < 2; ++layer) {
            const float* bias = vec + (layer == 0 ? V_BC0 : V_BC1);
#pragma unroll 1
            for (uint32_t c = 0; c < 4; ++c) {
                float v[32];
                tmem_ld32(tmem_row + 32 * c, v);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float h[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) h[i] = fmaxf(v[8 * q + i] + bias[32 * c + 8 * q + i], 0.f);
                    st_shared_v4(a_base + core_offset(r, 32 * c + 8 * q, KH), pack_bf16x2(h[0], h[1]),
                                 pack_bf16x2(h[2], h[3]), pack_bf16x2(h[4], h[5]), pack_bf16x2(h[6], h[7]));
                }
            }
            fence_async_smem();
            fence_before_sync();
            named_sync(bar_id, 128);
            if (r == 0) {
                fence_after_sync();
                issue_layer(tmem_acc, a_base, sbase + (layer == 0 ? OFF_WC1 : OFF_WC2), KH);
                mma_commit(bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            fence_after_sync();
        }

        // ---- final epilogue: +b, relu, f_C head (3 x sigmoid)
        float o0 = vec[V_BC3], o1 = vec[V_BC3 + 1], o2 = vec[V_BC3 + 2];
#pragma unroll 1
        for (uint32_t c = 0; c < 4; ++c) {
            float v[32];
            tmem_ld32(tmem_row + 32 * c, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const uint32_t col = 32 * c + i;
                const float h = fmaxf(v[i] + vec[V_BC2 + col], 0.f);
                o0 = __fmaf_rn(vec[V_WC3 + col], h, o0);
                o1 = __fmaf_rn(vec[V_WC3 + 128 + col], h, o1);
                o2 = __fmaf_rn(vec[V_WC3 + 256 + col], h, o2);
            }
        }
        if (j < n) {
            out.tau[j] = tau;
            out.eta[j] = eta;
            out.rgb[3 * size_t(j)] = sigmoidf_fast(o0);
            out.rgb[3 * size_t(j) + 1] = sigmoidf_fast(o1);
            out.rgb[3 * size_t(j) + 2] = sigmoidf_fast(o2);
        }
        fence_before_sync();  // TMEM reads complete before the next tile's MMA overwrites
    }

    fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        fence_after_sync();
        tmem_dealloc(tmem, 256);
    }
}

int g_num_sms = 0;

}  // namespace

size_t pack_tc_bytes(uint32_t V) { return OFF_FEAT + size_t(V) * 96 * 2; }

void ensure_pack_bf16(const DevModel& M, DevBuf& pack, uint64_t& pack_version, uint64_t version, cudaStream_t s) {
    if (pack_version == version && pack.p) return;
    uint8_t* p = pack.ensure<uint8_t>(pack_tc_bytes(M.V));
    k_pack_tc<<<(128 * KT + 255) / 256, 256, 0, s>>>(M.mt, M.mc, p);
    note_launch();
    __nv_bfloat16* ft16 = reinterpret_cast<__nv_bfloat16*>(p + OFF_FEAT);
    __nv_bfloat16* fc16 = ft16 + size_t(M.V) * 64;
    const size_t nt = size_t(M.V) * 64, nc = size_t(M.V) * 32;
    k_feat_bf16<<<unsigned((nt / 4 + 255) / 256 + 1), 256, 0, s>>>(M.ft, ft16, nt);
    k_feat_bf16<<<unsigned((nc / 4 + 255) / 256 + 1), 256, 0, s>>>(M.fc, fc16, nc);
    note_launch(2);
    pack_version = version;
}

void launch_decode_bf16(const DevOctree& T, const DevModel& M, const char* pack, const double* rays,
                        const uint32_t* hit_ray, const uint32_t* hit_leaf, const double* hit_tin,
                        const double* hit_tout, uint32_t n_hits, HitOut out, int* err, cudaStream_t s) {
    if (n_hits == 0) return;
    if (g_num_sms == 0) {
        int dev = 0;
        SVLF_CUDA(cudaGetDevice(&dev));
        SVLF_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
        SVLF_CUDA(cudaFuncSetAttribute(k_decode_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SM_TOTAL)));
    }
    const uint8_t* p = reinterpret_cast<const uint8_t*>(pack);
    const __nv_bfloat16* ft16 = reinterpret_cast<const __nv_bfloat16*>(p + OFF_FEAT);
    const __nv_bfloat16* fc16 = ft16 + size_t(M.V) * 64;
    const uint32_t tiles = (n_hits + 127) / 128;
    const uint32_t grid = std::min<uint32_t>(uint32_t(g_num_sms), (tiles + 1) / 2);
    k_decode_tc<<<grid, 256, SM_TOTAL, s>>>(T, p, ft16, fc16, rays, hit_ray, hit_leaf, hit_tin, hit_tout, n_hits,
                                            out, err);
    note_launch();
}

}  // namespace svlfb
