// Tensor-core decoder (tcgen05, 16-bit operands, fp32 accumulation in TMEM).
//
// Two kernels per frame, both over the flat hit list:
//   k_decode_t  per hit (thread = hit, fp64 in the reference's operand order):
//               x1, x2, parameterize_ray (r6), trilinear weights w1, w2, local
//               coordinates u1, u2 ("tangent ray" / "point not in voxel" raised
//               like the reference); then f_T (src/voxel_batch.hpp:69-114):
//               gather psi_T(x1), psi_T(x2) with packed 16-bit FMA, MMA
//               128x144x128, relu epilogue, head MMA 128x144x16 -> tau = relu,
//               eta = sigmoid; finally the f_C record of the hit: r6 and the
//               trilinear weights at u_s = eta u1 + (1-eta) u2 (32 bytes).
//   k_decode_c  f_C (src/voxel_batch.hpp:119-142): gather psi_C(x_s), MMA
//               128x48x128, two hidden MMAs 128x128x128, head MMA 128x128x16
//               -> rgb sigmoid.
// Each decode kernel is persistent (one CTA per SM, 512 threads = four
// independent 128-row slots; thread r of a slot owns hit r of the slot's
// tile). A slot's chain is gather -> MMA -> epilogue -> MMA ...; four slots
// per SM keep the tensor pipe fed while other slots gather. All weight tiles
// live in shared memory for the kernel's lifetime; each slot has one A buffer
// and a 128-column fp32 accumulator (4 x 128 = all 512 TMEM columns); head
// MMAs reuse the first 16 accumulator columns once the epilogue has read them.
//
// Biases of the input layers are folded into the MMA (A carries a constant
// 1.0 in the first padding column, the weight tile carries the bias there);
// hidden-layer biases are one extra K = 16 MMA of a shared constant-1 tile
// against a (hi, lo) 16-bit split of the bias, so the epilogue reads no bias
// from shared memory (those broadcast loads were a quarter of the f_C
// kernel's LSU wavefronts). Input K is permuted so
// 16-byte core-matrix chunks stay aligned (the weights use the same order):
//   f_T input  [psi_T(x1) 0..63 | psi_T(x2) 64..127 | r6 128..133 | 1 | 0...]
//   f_C input  [psi_C(x_s) 0..31 | r6 32..37 | 1 | 0...]
#include "device.cuh"
#include "tc_common.cuh"

namespace svlfb {

namespace {

using namespace tc;

constexpr uint32_t KT = 144;  // f_T input (+1 bias column, padded); f_T hidden->head (+bias)
constexpr uint32_t KC = 48;   // f_C input (+1 bias column, padded)
constexpr uint32_t KH = 128;  // f_C hidden layers (bias in epilogue)

// ---- weight pack (bytes), UMMA core-matrix layout
constexpr uint32_t OFF_WT0 = 0;                       // 128 x 144
constexpr uint32_t OFF_WT1 = OFF_WT0 + 128 * KT * 2;  // 16 x 144 (rows 0,1 = tau, eta; bias col 128)
constexpr uint32_t T_WEIGHTS = OFF_WT1 + 16 * KT * 2;  // 41472
constexpr uint32_t OFF_WC0 = (T_WEIGHTS + 1023) & ~1023u;  // 128 x 48
constexpr uint32_t OFF_WC1 = OFF_WC0 + 128 * KC * 2;       // 128 x 128
constexpr uint32_t OFF_WC2 = OFF_WC1 + 128 * KH * 2;       // 128 x 128
constexpr uint32_t OFF_WC3 = OFF_WC2 + 128 * KH * 2;       // 16 x 128 (rows 0..2 = rgb)
constexpr uint32_t OFF_WB1 = OFF_WC3 + 16 * KH * 2;        // 128 x 16: b_C1 as (hi, lo) 16-bit pair in k = 0, 1
constexpr uint32_t OFF_WB2 = OFF_WB1 + 128 * 16 * 2;       // 128 x 16: b_C2 likewise
constexpr uint32_t OFF_ONES = OFF_WB2 + 128 * 16 * 2;      // 128 x 16 A tile: 1.0 in k = 0, 1
constexpr uint32_t OFF_CVEC = OFF_ONES + 128 * 16 * 2;     // fp32: b_C1[128], b_C2[128], b_C3[4]
constexpr uint32_t C_WEIGHTS = OFF_CVEC + (128 + 128 + 4) * 4 - OFF_WC0;  // bytes from OFF_WC0
constexpr uint32_t OFF_FEAT = (OFF_WC0 + C_WEIGHTS + 255) & ~255u;

// ---- A-operand (activation) tiles: K-chunk stride LBO = 128*16 + 16 bytes,
// 8-row-group stride SBO = 128 bytes. The 16-byte skew per K chunk makes both
// store patterns conflict-free: 8 lanes writing the 8 chunks of one row, and
// 8 lanes writing one chunk of 8 consecutive rows, each hit 8 distinct
// 16-byte bank groups.
constexpr uint32_t kALbo = 128 * 16 + 16;  // 2064
__host__ __device__ constexpr uint32_t a_off(uint32_t r, uint32_t k) {
    return (k >> 3) * kALbo + (r >> 3) * 128u + (r & 7u) * 16u + (k & 7u) * 2u;
}

// ---- kernel shared memory
#ifndef SVLF_DEC_EXP
#define SVLF_DEC_EXP 0  // timing experiments only: f_C (1, 2) / f_T (3, 4) producers skip the gather / consumers skip the MMAs
#endif
#ifndef SVLF_DEC_C_TMEM
#define SVLF_DEC_C_TMEM 1
#endif
#ifndef SVLF_DEC_T_WS
#define SVLF_DEC_T_WS 1
#endif
#ifndef SVLF_DEC_EPI64
#define SVLF_DEC_EPI64 0
#endif
#ifndef SVLF_DEC_SLOTS
#define SVLF_DEC_SLOTS 4
#endif
constexpr uint32_t kSlots = SVLF_DEC_SLOTS;  // 128-row chains per CTA (one CTA per SM)
constexpr uint32_t T_A_BYTES = (KT / 8) * kALbo;  // 37152
constexpr uint32_t T_SM_A0 = (T_WEIGHTS + 1023) & ~1023u;
constexpr uint32_t T_SM_BAR = T_SM_A0 + kSlots * T_A_BYTES;
constexpr uint32_t T_SM_TOTAL = T_SM_BAR + 64;
constexpr uint32_t C_A_BYTES = (KH / 8) * kALbo;  // 33024 (>= the K=48 input tile)
constexpr uint32_t C_SM_A0 = (C_WEIGHTS + 1023) & ~1023u;
constexpr uint32_t C_SM_BAR = C_SM_A0 + kSlots * C_A_BYTES;
constexpr uint32_t C_SM_TOTAL = C_SM_BAR + 64;
static_assert(T_SM_TOTAL <= 232448 && C_SM_TOTAL <= 232448, "shared memory budget");
// f_C with the hidden activations in TMEM (k_decode_c_tm), warp-specialised:
// kProducers warps gather input tiles (K = 48) into a kRing-entry shared
// ring; two 4-warp consumer chains run the MMAs, each with a 128-column
// accumulator and a 64-column 16-bit A operand in TMEM.
#ifndef SVLF_DEC_C_PRODUCERS
#define SVLF_DEC_C_PRODUCERS 8
#endif
constexpr uint32_t kProducers = SVLF_DEC_C_PRODUCERS;
#ifndef SVLF_RING_SLEEP_NS
#define SVLF_RING_SLEEP_NS 128  // f_C producers polling for a free ring entry
#endif
#ifndef SVLF_DEC_EPI_PIPE
#define SVLF_DEC_EPI_PIPE 1  // f_C TMEM chains: 16-column epilogue chunks with the next load in flight
#endif
#ifndef SVLF_DEC_C_PUNROLL
#define SVLF_DEC_C_PUNROLL 2  // f_C producer: gather passes unrolled (loads in flight per warp)
#endif
#ifndef SVLF_DEC_TRACE
#define SVLF_DEC_TRACE 0
#endif
#if SVLF_DEC_TRACE
// timing probe (diagnostics build only): clock64 stamps of chains 0 and 2 of CTA 0, 10 per tile
__device__ unsigned long long g_dec_trace[3][64][10];
#define DEC_STAMP(i)                                                                     \
    do {                                                                                 \
        if (blockIdx.x == 0 && r == 0 && k / kChains < 64) g_dec_trace[chain][k / kChains][i] = clock64(); \
    } while (0)
#else
#define DEC_STAMP(i) \
    do {             \
    } while (0)
#endif
#ifndef SVLF_DEC_C_SMCHAINS
#define SVLF_DEC_C_SMCHAINS 1
#endif
#ifndef SVLF_DEC_C_TMCHAINS
#define SVLF_DEC_C_TMCHAINS 2
#endif
constexpr uint32_t kChainsTm = SVLF_DEC_C_TMCHAINS;    // chains with A in TMEM (192 columns each)
constexpr uint32_t kChainsSm = SVLF_DEC_C_SMCHAINS;    // chains with A in shared memory (128 columns)
constexpr uint32_t kChains = kChainsTm + kChainsSm;
#ifndef SVLF_DEC_C_RING
#define SVLF_DEC_C_RING 0
#endif
constexpr uint32_t kRing = SVLF_DEC_C_RING ? SVLF_DEC_C_RING : (kChainsSm ? 7 : 10);
constexpr uint32_t kCtThreads = (kProducers + 4 * kChains) * 32;
constexpr uint32_t CT_A_BYTES = (KC / 8) * kALbo;  // 12384
constexpr uint32_t CT_SMA0 = C_SM_A0 + kRing * CT_A_BYTES;
constexpr uint32_t CT_SM_BAR = CT_SMA0 + kChainsSm * C_A_BYTES;
constexpr uint32_t CT_SM_TOTAL = CT_SM_BAR + 4 * 8 + (2 * kRing + 1) * 4;
static_assert(kChainsTm * 192 + kChainsSm * 128 <= 512, "TMEM columns");
// f_T warp-specialised (k_decode_t_ws): 4-warp producer groups (geometry +
// gather) feed 4-warp MMA chains through a 4-entry ring (input tile + per-row
// side data: u1, u2, r6 pairs); entry e is filled by group e % TW_GROUPS and
// consumed by chain e % TW_CHAINS.
constexpr uint32_t TW_RING0 = (T_WEIGHTS + 1023) & ~1023u;
constexpr uint32_t TW_SIDE = 11 * 128 * 4;                // u[6] fp32, r6 pairs[3], t_in, t_out (fp32), SoA
constexpr uint32_t TW_ENTRY = T_A_BYTES + TW_SIDE;        // 42784
constexpr uint32_t TW_ENTRIES = 4;
#ifndef SVLF_DEC_T_GROUPS
#define SVLF_DEC_T_GROUPS 4
#endif
#ifndef SVLF_DEC_T_CHAINS
#define SVLF_DEC_T_CHAINS 1
#endif
constexpr uint32_t TW_GROUPS = SVLF_DEC_T_GROUPS;  // 4-warp producer groups
constexpr uint32_t TW_CHAINS = SVLF_DEC_T_CHAINS;  // 4-warp MMA chains
constexpr uint32_t TW_THREADS = 128 * (TW_GROUPS + TW_CHAINS);
static_assert(TW_ENTRIES % TW_GROUPS == 0 && TW_ENTRIES % TW_CHAINS == 0 && TW_CHAINS <= 2,
              "each ring entry has one producer group and one chain (mbarrier parity)");
constexpr uint32_t TW_SM_BAR = TW_RING0 + TW_ENTRIES * TW_ENTRY;
constexpr uint32_t TW_SM_TOTAL = TW_SM_BAR + (2 + 2 * TW_ENTRIES) * 8 + 16;
static_assert(TW_SM_TOTAL <= 232448, "shared memory budget");
static_assert(CT_SM_TOTAL <= 232448, "shared memory budget");

// Operand format traits: fp16 (11-bit mantissa) or bf16 (north-star format);
// both run at the same tensor-core rate.
template <bool kBF16>
struct Fmt;
template <>
struct Fmt<false> {
    using H = __half;
    using H2 = __half2;
    static __device__ __forceinline__ H2 splat(float x) { return __float2half2_rn(x); }
    static __host__ __device__ __forceinline__ H cvt(float x) { return __float2half_rn(x); }
    static __device__ __forceinline__ float tof(H x) { return __half2float(x); }
    static __device__ __forceinline__ uint32_t relu_pack(float lo, float hi) {
        uint32_t r;
        asm("cvt.rn.satfinite.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
        return r;
    }
    static __device__ __forceinline__ uint32_t pack(float lo, float hi) {
        uint32_t r;
        asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
        return r;
    }
    static constexpr uint32_t kOne = 0x00003C00u;  // (1.0, 0.0)
    static __device__ __forceinline__ H2 lo2(H2 p) { return __low2half2(p); }
    static __device__ __forceinline__ H2 hi2(H2 p) { return __high2half2(p); }
};
template <>
struct Fmt<true> {
    using H = __nv_bfloat16;
    using H2 = __nv_bfloat162;
    static __device__ __forceinline__ H2 splat(float x) { return __float2bfloat162_rn(x); }
    static __host__ __device__ __forceinline__ H cvt(float x) { return __float2bfloat16_rn(x); }
    static __device__ __forceinline__ float tof(H x) { return __bfloat162float(x); }
    static __device__ __forceinline__ uint32_t relu_pack(float lo, float hi) {
        uint32_t r;
        asm("cvt.rn.satfinite.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
        return r;
    }
    static __device__ __forceinline__ uint32_t pack(float lo, float hi) {
        uint32_t r;
        asm("cvt.rn.satfinite.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
        return r;
    }
    static constexpr uint32_t kOne = 0x00003F80u;
    static __device__ __forceinline__ H2 lo2(H2 p) { return __low2bfloat162(p); }
    static __device__ __forceinline__ H2 hi2(H2 p) { return __high2bfloat162(p); }
};

template <typename T2>
__device__ __forceinline__ uint32_t h2u(T2 h) {
    return *reinterpret_cast<uint32_t*>(&h);
}
template <typename T2>
__device__ __forceinline__ T2 u2h(uint32_t u) {
    return *reinterpret_cast<T2*>(&u);
}

// ---- pack: fp32 flat params -> 16-bit UMMA tiles (+ folded biases), fp32 bias vectors
template <bool kBF16>
__global__ void k_pack_tc(const float* __restrict__ mt, const float* __restrict__ mc, uint8_t* pack) {
    using D = DecOffsets;
    using F = Fmt<kBF16>;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    auto put = [&](uint32_t off, uint32_t n, uint32_t k, uint32_t K, float w) {
        reinterpret_cast<typename F::H*>(pack + off)[core_offset(n, k, K) / 2] = F::cvt(w);
    };
    if (tid < 128 * KT) {  // f_T layer 0: permuted input + bias column 134
        const uint32_t n = tid / KT, k = tid % KT;
        float w = 0.f;
        if (k < 128) w = mt[D::T_W0 + n * kInT + 6 + k];
        else if (k < 134) w = mt[D::T_W0 + n * kInT + (k - 128)];
        else if (k == 134) w = mt[D::T_B0 + n];
        put(OFF_WT0, n, k, KT, w);
    }
    if (tid < 16 * KT) {  // f_T head, N = 16, bias column 128
        const uint32_t n = tid / KT, k = tid % KT;
        float w = 0.f;
        if (n < 2) w = k < 128 ? mt[D::T_W1 + n * kHid + k] : (k == 128 ? mt[D::T_B1 + n] : 0.f);
        put(OFF_WT1, n, k, KT, w);
    }
    if (tid < 128 * KC) {  // f_C layer 0: permuted input + bias column 38
        const uint32_t n = tid / KC, k = tid % KC;
        float w = 0.f;
        if (k < 32) w = mc[D::C_W0 + n * kInC + 6 + k];
        else if (k < 38) w = mc[D::C_W0 + n * kInC + (k - 32)];
        else if (k == 38) w = mc[D::C_B0 + n];
        put(OFF_WC0, n, k, KC, w);
    }
    if (tid < 128 * KH) {
        const uint32_t n = tid / KH, k = tid % KH;
        put(OFF_WC1, n, k, KH, mc[D::C_W1 + n * kHid + k]);
        put(OFF_WC2, n, k, KH, mc[D::C_W2 + n * kHid + k]);
    }
    if (tid < 16 * KH) {
        const uint32_t n = tid / KH, k = tid % KH;
        put(OFF_WC3, n, k, KH, n < 3 ? mc[D::C_W3 + n * kHid + k] : 0.f);
    }
    if (tid < 128 * 16) {  // hidden-layer biases as an extra K = 16 MMA against a constant-1 tile
        const uint32_t n = tid / 16, k = tid % 16;
        auto hilo = [&](float b) { return k == 0 ? b : (k == 1 ? b - F::tof(F::cvt(b)) : 0.f); };
        put(OFF_WB1, n, k, 16, hilo(mc[D::C_B1 + n]));
        put(OFF_WB2, n, k, 16, hilo(mc[D::C_B2 + n]));
        put(OFF_ONES, n, k, 16, k < 2 ? 1.f : 0.f);
    }
    float* cvec = reinterpret_cast<float*>(pack + OFF_CVEC);
    if (tid < 128) {
        cvec[tid] = mc[D::C_B1 + tid];
        cvec[128 + tid] = mc[D::C_B2 + tid];
    }
    if (tid < 4) cvec[256 + tid] = tid < 3 ? mc[D::C_B3 + tid] : 0.f;
}

template <bool kBF16>
__global__ void k_feat_cvt(const float* __restrict__ src, typename Fmt<kBF16>::H* dst, size_t n) {
    using F = Fmt<kBF16>;
    const size_t i = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) * 4;
    for (size_t k = i; k < i + 4 && k < n; ++k) dst[k] = F::cvt(src[k]);
}

// ---- per-hit geometry, fp64 in the reference's operand order, one thread per
// hit: x1, x2, parameterize_ray (r6), trilinear weights w1, w2 (16-bit pairs)
// and local coordinates u1, u2 (fp32, for x_s after the f_T pass). Raises
// "tangent ray" / "point not in voxel" like the reference.
// Hit geometry for the 16-bit decoders. The tests that raise the reference's
// errors ("tangent ray": the discriminant; "point not in voxel": the slab
// bounds) and the chord end points run in fp64 in the reference's operand
// order; the results are rounded to 16 bits for the MMA, so the unit
// direction normalisations (two fp64 square roots, six divisions) and the
// trilinear weight products run in fp32 (their rounding is far below the
// 16-bit quantisation).
__device__ __forceinline__ bool parameterize_tc(const Ray& r, const double* lo, const double* hi, float* r6) {
    double c[3], oc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        c[a] = dmul(dadd(lo[a], hi[a]), 0.5);
        oc[a] = dsub(r.o[a], c[a]);
    }
    constexpr double kHalfSqrt3 = 0.5 * 1.7320508075688772;
    const double radius = dmul(kHalfSqrt3, dsub(hi[0], lo[0]));
    const double b = dot3(oc, r.d);
    const double cc = dsub(dot3(oc, oc), dmul(radius, radius));
    const double disc = dsub(dmul(b, b), cc);
    if (disc < 1e-14) return false;
    const double s = __dsqrt_rn(disc);
    const double t1 = dsub(-b, s), t2 = dadd(-b, s);
    float p1[3], p2[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        p1[a] = float(dsub(dadd(r.o[a], dmul(r.d[a], t1)), c[a]));
        p2[a] = float(dsub(dadd(r.o[a], dmul(r.d[a], t2)), c[a]));
    }
    const float i1 = rsqrtf(p1[0] * p1[0] + p1[1] * p1[1] + p1[2] * p1[2]);
    const float i2 = rsqrtf(p2[0] * p2[0] + p2[1] * p2[1] + p2[2] * p2[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r6[a] = p1[a] * i1;
        r6[3 + a] = p2[a] * i2;
    }
    return true;
}

__device__ __forceinline__ bool trilinear_tc(const double* p, const double* lo, const DevOctree& T, const double* hi,
                                             float* w, double* u) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!(p[a] >= dsub(lo[a], 1e-7) && p[a] <= dadd(hi[a], 1e-7))) return false;
        u[a] = fmin(fmax(div_cell(T, dsub(p[a], lo[a])), 0.0), 1.0);
    }
    const float fx[2] = {1.f - float(u[0]), float(u[0])}, fy[2] = {1.f - float(u[1]), float(u[1])},
                fz[2] = {1.f - float(u[2]), float(u[2])};
#pragma unroll
    for (int b = 0; b < 8; ++b) w[b] = fx[b & 1] * fy[(b >> 1) & 1] * fz[b >> 2];
    return true;
}

template <bool kBF16>
__device__ __forceinline__ void hit_geom_regs(const DevOctree& T, const double* __restrict__ rays, uint32_t ri,
                                              uint32_t leaf, double tin, double tout, uint32_t* r6p, uint32_t* wp,
                                              float* u, int* err) {
    using F = Fmt<kBF16>;
    Ray ray;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        ray.o[a] = rays[6 * size_t(ri) + a];
        ray.d[a] = rays[6 * size_t(ri) + 3 + a];
    }
    double lo[3], hi[3], x1[3], x2[3];
    leaf_box(T, leaf, lo, hi);
    ray_at(ray, tin, x1);
    ray_at(ray, tout, x2);
    float r6[6] = {0, 0, 0, 0, 0, 0}, w1[8], w2[8];
    double u1[3] = {0, 0, 0}, u2[3] = {0, 0, 0};  // local coordinates (features.cpp:22-31)
    if (!parameterize_tc(ray, lo, hi, r6)) raise_error(err, kErrTangentRay);
    if (!trilinear_tc(x1, lo, T, hi, w1, u1) || !trilinear_tc(x2, lo, T, hi, w2, u2)) {
        raise_error(err, kErrPointNotInVoxel);
#pragma unroll
        for (int b = 0; b < 8; ++b) w1[b] = w2[b] = 0.f;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        u[a] = float(u1[a]);
        u[3 + a] = float(u2[a]);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) r6p[i] = F::pack(r6[2 * i], r6[2 * i + 1]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        wp[i] = F::pack(w1[2 * i], w1[2 * i + 1]);
        wp[4 + i] = F::pack(w2[2 * i], w2[2 * i + 1]);
    }
}

// D[tmem] (+)= A . B^T over K: A in the skewed activation layout (a_off),
// B (weights, N rows) in the dense layout core_offset(n, k, K).
__device__ __forceinline__ void issue_layer(uint32_t tmem_d, uint32_t a_base, uint32_t b_base, uint32_t K,
                                            uint32_t idesc) {
    const uint32_t b_sbo = (K / 8) * 128;
#pragma unroll 1
    for (uint32_t k = 0; k < K / 16; ++k)
        mma_f16(tmem_d, make_desc(a_base + 2 * k * kALbo, kALbo, 128), make_desc(b_base + 256 * k, 128, b_sbo),
                idesc, k > 0);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 TMEM columns into registers, and the wait for them: the wait names the
// destination registers as in-out operands so no use of them can be scheduled
// before it (loads of the next chunk are then in flight while the current one
// is converted)
// 4 TMEM columns (the heads' outputs)
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* v) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16u(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld16(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// Epilogue: TMEM acc (128 fp32, + optional fp32 bias) -> relu -> 16-bit -> A tile (K layout)
template <bool kBF16, bool kBias>
__device__ __forceinline__ void hidden_epilogue(uint32_t tmem_row, uint32_t a_base, uint32_t r, uint32_t K,
                                                const float* bias) {
    using F = Fmt<kBF16>;
    if constexpr (!kBias && SVLF_DEC_EPI_PIPE) {
        // 16-column chunks, the next chunk's load in flight while this one is packed and stored
        uint32_t ra[16], rb[16];
        tmem_ld16u(tmem_row, ra);
        tmem_wait_ld16(ra);
#pragma unroll
        for (uint32_t c = 0; c < 8; ++c) {
            uint32_t(&cur)[16] = (c & 1) ? rb : ra;
            uint32_t(&nxt)[16] = (c & 1) ? ra : rb;
            if (c + 1 < 8) tmem_ld16u(tmem_row + 16 * (c + 1), nxt);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t* w = cur + 8 * q;
                st_shared_v4(a_base + a_off(r, 16 * c + 8 * q),
                             F::relu_pack(__uint_as_float(w[0]), __uint_as_float(w[1])),
                             F::relu_pack(__uint_as_float(w[2]), __uint_as_float(w[3])),
                             F::relu_pack(__uint_as_float(w[4]), __uint_as_float(w[5])),
                             F::relu_pack(__uint_as_float(w[6]), __uint_as_float(w[7])));
            }
            if (c + 1 < 8) tmem_wait_ld16(nxt);
        }
        return;
    }
#pragma unroll 1
    for (uint32_t c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(tmem_row + 32 * c, v);
        tmem_wait_ld();
        if constexpr (kBias) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                const float4 b = *reinterpret_cast<const float4*>(bias + 32 * c + i);
                v[i] += b.x;
                v[i + 1] += b.y;
                v[i + 2] += b.z;
                v[i + 3] += b.w;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            st_shared_v4(a_base + a_off(r, 32 * c + 8 * q), F::relu_pack(v[8 * q], v[8 * q + 1]),
                         F::relu_pack(v[8 * q + 2], v[8 * q + 3]), F::relu_pack(v[8 * q + 4], v[8 * q + 5]),
                         F::relu_pack(v[8 * q + 6], v[8 * q + 7]));
    }
}

struct Slot {
    uint64_t* bar;
    uint32_t phase;
    uint32_t bar_id;
    uint32_t r;
    // all writes to the slot's A buffer done -> one thread issues, everyone waits for completion
    template <typename Issue>
    __device__ __forceinline__ void mma(Issue&& issue) {
        fence_async_smem();
        fence_before_sync();
        named_sync(bar_id, 128);
        if (r == 0) {
            fence_after_sync();
            issue();
            mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        fence_after_sync();
    }
};

// Common prologue of the decode kernels: weights -> smem, barriers, TMEM.
__device__ __forceinline__ uint32_t kernel_setup(uint8_t* sm, const uint8_t* weights, uint32_t wbytes,
                                                 uint32_t bar_off) {
    const uint32_t tid = threadIdx.x;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + bar_off);
    uint32_t* holder = reinterpret_cast<uint32_t*>(sm + bar_off + 48);
    {
        const uint4* src = reinterpret_cast<const uint4*>(weights);
        uint4* dst = reinterpret_cast<uint4*>(sm);
        for (uint32_t i = tid; i < wbytes / 16; i += blockDim.x) dst[i] = src[i];
    }
    if (tid == 0) {
        for (uint32_t s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if ((tid >> 5) == 0) tmem_alloc(holder, 512);
    fence_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    return *holder;
}

__device__ __forceinline__ void kernel_teardown(uint32_t tmem) {
    fence_before_sync();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        fence_after_sync();
        tmem_dealloc(tmem, 512);
    }
}

__device__ __forceinline__ void load_corners(const DevOctree& T, uint32_t leaf, uint32_t* c) {
    const uint4* cp = reinterpret_cast<const uint4*>(T.corners + 8 * size_t(leaf));
    const uint4 a = __ldg(cp), b = __ldg(cp + 1);
    c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w;
    c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
}

// ---- f_T pass ---------------------------------------------------------------
template <bool kBF16>
__global__ void __launch_bounds__(kSlots * 128, 1)
    k_decode_t(DevOctree T, const uint8_t* __restrict__ pack, const typename Fmt<kBF16>::H* __restrict__ ft16,
               const double* __restrict__ rays, const uint32_t* __restrict__ hit_ray,
               const uint32_t* __restrict__ hit_leaf, const double* __restrict__ hit_tin,
               const double* __restrict__ hit_tout, const uint32_t* n_dev, uint32_t cap, HitOut out,
               uint4* __restrict__ crec, int* err) {
    using F = Fmt<kBF16>;
    using H2 = typename F::H2;
    constexpr uint32_t kIdesc = make_idesc(128, 128, kBF16);
    constexpr uint32_t kIdescHead = make_idesc(128, 16, kBF16);
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t tmem = kernel_setup(sm, pack + OFF_WT0, T_WEIGHTS, T_SM_BAR);
    const uint32_t tid = threadIdx.x, slot = tid >> 7, r = tid & 127, warp = tid >> 5;
    const uint32_t lane_off = (32u * (warp & 3u)) << 16;
    const uint32_t acc = tmem + slot * 128;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t a_base = sbase + T_SM_A0 + slot * T_A_BYTES;
    Slot S{reinterpret_cast<uint64_t*>(sm + T_SM_BAR) + slot, 0u, 1u + slot, r};
    const uint32_t n = min(*n_dev, cap);
    const uint32_t ntiles = (n + 127) / 128;

    // The per-hit scalars of a slot's NEXT tile are loaded one tile ahead, so
    // the dependent chain leaf -> corners -> feature rows starts from registers.
    const uint32_t tstride = gridDim.x * kSlots;
    uint32_t nleaf = 0, nray = 0;
    double ntin = 0.0, ntout = 0.0;
    auto prefetch = [&](uint32_t t) {
        const uint32_t jn = t * 128 + r;
        if (t < ntiles && jn < n) {
            nleaf = hit_leaf[jn];
            nray = hit_ray[jn];
            ntin = hit_tin[jn];
            ntout = hit_tout[jn];
        }
    };
    prefetch(blockIdx.x * kSlots + slot);
    for (uint32_t tile = blockIdx.x * kSlots + slot; tile < ntiles; tile += tstride) {
        const uint32_t j = tile * 128 + r;
        const bool valid = j < n;
        uint32_t corners[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t r6p[3] = {0, 0, 0}, wp[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // r6, (w1, w2) as 16-bit pairs
        float u[6] = {0, 0, 0, 0, 0, 0};
        const uint32_t leaf = nleaf, ray_i = nray;
        const double tin = ntin, tout = ntout;
        prefetch(tile + tstride);
        if (valid) {
            load_corners(T, leaf, corners);
            hit_geom_regs<kBF16>(T, rays, ray_i, leaf, tin, tout, r6p, wp, u, err);
        }
        // Warp-cooperative gather: the warp owns rows 32w..32w+31 of the tile; in
        // pass p lanes 8q..8q+7 gather row 4p+q, lane chunk c = 8 features, so
        // one LDG.128 instruction covers 4 whole 128-byte feature rows.
        const uint32_t lane = r & 31, q = lane >> 3, ch = lane & 7, row0 = r & ~31u;
#pragma unroll 2
        for (uint32_t p = 0; p < 8; ++p) {
            const uint32_t src = 4 * p + q;
            uint32_t cb[8], w[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) cb[b] = __shfl_sync(0xffffffffu, corners[b], src);
#pragma unroll
            for (int b = 0; b < 8; ++b) w[b] = __shfl_sync(0xffffffffu, wp[b], src);
            uint4 fq[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) fq[b] = __ldg(reinterpret_cast<const uint4*>(ft16 + size_t(cb[b]) * 64) + ch);
            H2 a1[4], a2[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a1[i] = a2[i] = F::splat(0.f);
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const H2 p1 = u2h<H2>(w[b / 2]), p2 = u2h<H2>(w[4 + b / 2]);
                const H2 h1 = (b & 1) ? F::hi2(p1) : F::lo2(p1);
                const H2 h2 = (b & 1) ? F::hi2(p2) : F::lo2(p2);
                const H2* f = reinterpret_cast<const H2*>(&fq[b]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a1[i] = __hfma2(h1, f[i], a1[i]);
                    a2[i] = __hfma2(h2, f[i], a2[i]);
                }
            }
            const uint32_t row = row0 + src;
            st_shared_v4(a_base + a_off(row, 8 * ch), h2u(a1[0]), h2u(a1[1]), h2u(a1[2]), h2u(a1[3]));
            st_shared_v4(a_base + a_off(row, 64 + 8 * ch), h2u(a2[0]), h2u(a2[1]), h2u(a2[2]),
                         h2u(a2[3]));
        }
        st_shared_v4(a_base + a_off(r, 128), r6p[0], r6p[1], r6p[2], F::kOne);
        st_shared_v4(a_base + a_off(r, 136), 0u, 0u, 0u, 0u);

        S.mma([&] { issue_layer(acc, a_base, sbase + OFF_WT0, KT, kIdesc); });
        hidden_epilogue<kBF16, false>(acc + lane_off, a_base, r, KT, nullptr);
        st_shared_v4(a_base + a_off(r, 128), F::kOne, 0u, 0u, 0u);
        st_shared_v4(a_base + a_off(r, 136), 0u, 0u, 0u, 0u);
        S.mma([&] { issue_layer(acc, a_base, sbase + OFF_WT1, KT, kIdescHead); });
        float hv[16];
        tmem_ld16(acc + lane_off, hv);
        tmem_wait_ld();
        if (valid) {
            const float e = __fdividef(1.0f, 1.0f + __expf(-hv[1])), ome = 1.0f - e;
            out.tau[j] = fmaxf(hv[0], 0.f);
            out.eta[j] = float(tin) * e + float(tout) * (1.f - e);  // 16-bit path: t_s for the composite
            // f_C record: r6 and the trilinear weights at x_s = eta x1 + (1-eta) x2,
            // u_s = eta u1 + (1-eta) u2 (voxel_batch.hpp:111)
            const float us[3] = {u[0] * e + u[3] * ome, u[1] * e + u[4] * ome, u[2] * e + u[5] * ome};
            float ws[8];
#pragma unroll
            for (int b = 0; b < 8; ++b)
                ws[b] = ((b & 1) ? us[0] : 1.f - us[0]) * ((b & 2) ? us[1] : 1.f - us[1]) *
                        ((b & 4) ? us[2] : 1.f - us[2]);
            crec[2 * size_t(j)] = make_uint4(r6p[0], r6p[1], r6p[2], 0u);
            crec[2 * size_t(j) + 1] = make_uint4(F::pack(ws[0], ws[1]), F::pack(ws[2], ws[3]), F::pack(ws[4], ws[5]),
                                                 F::pack(ws[6], ws[7]));
        }
        fence_before_sync();
    }
    kernel_teardown(tmem);
}

// ---- f_C pass ---------------------------------------------------------------
template <bool kBF16>
__global__ void __launch_bounds__(kSlots * 128, 1)
    k_decode_c(DevOctree T, const uint8_t* __restrict__ pack, const typename Fmt<kBF16>::H* __restrict__ fc16,
               const uint32_t* __restrict__ hit_leaf, const uint4* __restrict__ crec, const uint32_t* n_dev,
               uint32_t cap, HitOut out) {
    using F = Fmt<kBF16>;
    using H2 = typename F::H2;
    constexpr uint32_t kIdesc = make_idesc(128, 128, kBF16);
    constexpr uint32_t kIdescHead = make_idesc(128, 16, kBF16);
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t tmem = kernel_setup(sm, pack + OFF_WC0, C_WEIGHTS, C_SM_BAR);
    const uint32_t tid = threadIdx.x, slot = tid >> 7, r = tid & 127, warp = tid >> 5;
    const uint32_t lane_off = (32u * (warp & 3u)) << 16;
    const uint32_t acc = tmem + slot * 128;
    const uint32_t sbase = smem_u32(sm);
    constexpr uint32_t W0 = 0, W1 = OFF_WC1 - OFF_WC0, W2 = OFF_WC2 - OFF_WC0, W3 = OFF_WC3 - OFF_WC0;
    constexpr uint32_t WB1 = OFF_WB1 - OFF_WC0, WB2 = OFF_WB2 - OFF_WC0;
    const uint64_t ones = make_desc(sbase + (OFF_ONES - OFF_WC0), 128, 256);
    const float* cvec = reinterpret_cast<const float*>(sm + (OFF_CVEC - OFF_WC0));
    const uint32_t a_base = sbase + C_SM_A0 + slot * C_A_BYTES;
    Slot S{reinterpret_cast<uint64_t*>(sm + C_SM_BAR) + slot, 0u, 1u + slot, r};
    const uint32_t n = min(*n_dev, cap);
    const uint32_t ntiles = (n + 127) / 128;

    // Next tile's inputs are loaded one tile ahead in two steps (its leaf index
    // at the start of this tile, its corners and f_C record after this tile's
    // gather), so no load waits on another inside the critical path.
    const uint32_t tstride = gridDim.x * kSlots;
    uint32_t ncorners[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint4 ng0 = make_uint4(0, 0, 0, 0), ng1 = ng0;
    uint32_t nleaf = 0;
    auto fetch_leaf = [&](uint32_t t) {
        const uint32_t jn = t * 128 + r;
        if (t < ntiles && jn < n) nleaf = hit_leaf[jn];
    };
    auto fetch_rest = [&](uint32_t t) {
        const uint32_t jn = t * 128 + r;
        if (t < ntiles && jn < n) {
            load_corners(T, nleaf, ncorners);
            ng0 = crec[2 * size_t(jn)];      // r6 pairs
            ng1 = crec[2 * size_t(jn) + 1];  // trilinear weights at x_s, 16-bit pairs
        }
    };
    fetch_leaf(blockIdx.x * kSlots + slot);
    fetch_rest(blockIdx.x * kSlots + slot);
    for (uint32_t tile = blockIdx.x * kSlots + slot; tile < ntiles; tile += tstride) {
        const uint32_t j = tile * 128 + r;
        const bool valid = j < n;
        uint32_t corners[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) corners[b] = valid ? ncorners[b] : 0u;
        const uint4 g0 = valid ? ng0 : make_uint4(0, 0, 0, 0), g1 = valid ? ng1 : make_uint4(0, 0, 0, 0);
        fetch_leaf(tile + tstride);
        // Warp-cooperative gather: pass p, lanes 4q..4q+3 gather row 8p+q of the
        // warp's 32 rows, lane chunk = 8 of the 32 colour features.
        const uint32_t lane = r & 31, q = lane >> 2, ch = lane & 3, row0 = r & ~31u;
        const uint32_t wsp[4] = {g1.x, g1.y, g1.z, g1.w};
#pragma unroll 2
        for (uint32_t p = 0; p < 4; ++p) {
            const uint32_t src = 8 * p + q;
            uint32_t cb[8], w[4];
#pragma unroll
            for (int b = 0; b < 8; ++b) cb[b] = __shfl_sync(0xffffffffu, corners[b], src);
#pragma unroll
            for (int b = 0; b < 4; ++b) w[b] = __shfl_sync(0xffffffffu, wsp[b], src);
            uint4 fq[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) fq[b] = __ldg(reinterpret_cast<const uint4*>(fc16 + size_t(cb[b]) * 32) + ch);
            H2 a1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a1[i] = F::splat(0.f);
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const H2 pw = u2h<H2>(w[b / 2]);
                const H2 hw = (b & 1) ? F::hi2(pw) : F::lo2(pw);
                const H2* f = reinterpret_cast<const H2*>(&fq[b]);
#pragma unroll
                for (int i = 0; i < 4; ++i) a1[i] = __hfma2(hw, f[i], a1[i]);
            }
            st_shared_v4(a_base + a_off(row0 + src, 8 * ch), h2u(a1[0]), h2u(a1[1]), h2u(a1[2]),
                         h2u(a1[3]));
        }
        st_shared_v4(a_base + a_off(r, 32), g0.x, g0.y, g0.z, F::kOne);
        st_shared_v4(a_base + a_off(r, 40), 0u, 0u, 0u, 0u);
        fetch_rest(tile + tstride);
        S.mma([&] { issue_layer(acc, a_base, sbase + W0, KC, kIdesc); });
        hidden_epilogue<kBF16, false>(acc + lane_off, a_base, r, KH, nullptr);
        S.mma([&] {
            issue_layer(acc, a_base, sbase + W1, KH, kIdesc);
            mma_f16(acc, ones, make_desc(sbase + WB1, 128, 256), kIdesc, true);
        });
        hidden_epilogue<kBF16, false>(acc + lane_off, a_base, r, KH, nullptr);
        S.mma([&] {
            issue_layer(acc, a_base, sbase + W2, KH, kIdesc);
            mma_f16(acc, ones, make_desc(sbase + WB2, 128, 256), kIdesc, true);
        });
        hidden_epilogue<kBF16, false>(acc + lane_off, a_base, r, KH, nullptr);
        S.mma([&] { issue_layer(acc, a_base, sbase + W3, KH, kIdescHead); });
        float hv[16];
        tmem_ld16(acc + lane_off, hv);
        tmem_wait_ld();
        if (valid) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
                out.rgb[3 * size_t(j) + c] = __fdividef(1.0f, 1.0f + __expf(-(hv[c] + cvec[256 + c])));
        }
        fence_before_sync();
    }
    kernel_teardown(tmem);
}

// ---- f_C pass, hidden activations in TMEM -----------------------------------
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// D[tmem] (+)= A[tmem] . B^T: A is 128 lanes x K/2 columns (16-bit K pairs per
// 32-bit column, 8 columns per K = 16 step), B in the dense smem layout.
__device__ __forceinline__ void issue_layer_ta(uint32_t tmem_d, uint32_t a_tmem, uint32_t b_base, uint32_t K,
                                               uint32_t idesc) {
    const uint32_t b_sbo = (K / 8) * 128;
#pragma unroll 1
    for (uint32_t k = 0; k < K / 16; ++k)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "r"(a_tmem + 8 * k), "l"(make_desc(b_base + 256 * k, 128, b_sbo)), "r"(idesc), "r"(k > 0 ? 1u : 0u));
}

template <bool kBF16>
__global__ void __launch_bounds__(kCtThreads, 1)
    k_decode_c_tm(DevOctree T, const uint8_t* __restrict__ pack, const typename Fmt<kBF16>::H* __restrict__ fc16,
                  const uint32_t* __restrict__ hit_leaf, const uint4* __restrict__ crec, const uint32_t* n_dev,
                  uint32_t cap, HitOut out) {
    using F = Fmt<kBF16>;
    using H2 = typename F::H2;
    constexpr uint32_t kIdesc = make_idesc(128, 128, kBF16);
    constexpr uint32_t kIdescHead = make_idesc(128, 16, kBF16);
    extern __shared__ __align__(1024) uint8_t sm[];
    // Ring hand-off by tile-number flags (not mbarrier parity: several
    // producers and chains share each ring entry, so a waiter can be more than
    // one phase behind): full[s] = k + 1 once tile k is in entry s, empty[s] =
    // k + 1 once the layer-0 MMA that read it completed.
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + CT_SM_BAR);  // [0..3] chain MMA barriers
    uint32_t* full = reinterpret_cast<uint32_t*>(bars + 4);
    uint32_t* empty = full + kRing;
    uint32_t* holder = empty + kRing;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        const uint4* src = reinterpret_cast<const uint4*>(pack + OFF_WC0);
        uint4* dst = reinterpret_cast<uint4*>(sm);
        for (uint32_t i = tid; i < C_WEIGHTS / 16; i += blockDim.x) dst[i] = src[i];
    }
    if (tid == 0) {
        for (uint32_t i = 0; i < kChains; ++i) mbar_init(&bars[i], 1);
        for (uint32_t i = 0; i < kRing; ++i) {
            full[i] = 0;
            empty[i] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(holder, 512);
    fence_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *holder;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t ring0 = sbase + C_SM_A0;
    const uint32_t n = min(*n_dev, cap);
    const uint32_t ntiles = (n + 127) / 128;
    auto tile_of = [&](uint32_t k) { return blockIdx.x + k * gridDim.x; };

    if (warp < kProducers) {
        // ---- producer warp: whole input tiles, k = warp, warp + kProducers, ...
        // Per 32-row group, lane l holds row 32g + l (leaf, f_C record). The
        // features come from the per-leaf table (8 corner rows of 64 B per
        // leaf): in pass p, lanes 8h..8h+7 gather row 4p+h of the group, lane
        // (cp, ch) = corners 2k + cp of chunk ch, so one load instruction reads
        // 4 whole 128-byte lines (corners 2k, 2k+1 of 4 rows); the two corner
        // halves are summed with one shuffle.
        const uint32_t hsub = lane >> 3, cp = (lane >> 2) & 1u, ch = lane & 3;
        uint32_t leaves[4], lf_cur = 0, lf_next = 0;
        uint4 g0, g1, ng0, ng1;
        auto fetch_leaves = [&](uint32_t t) {
#pragma unroll
            for (uint32_t g = 0; g < 4; ++g) {
                const uint32_t j = t * 128 + 32 * g + lane;
                leaves[g] = (t < ntiles && j < n) ? hit_leaf[j] : 0xffffffffu;
            }
        };
        auto fetch = [&](uint32_t t, uint32_t leaf, uint32_t g) {
            const uint32_t j = t * 128 + 32 * g + lane;
            lf_next = leaf;
            if (leaf != 0xffffffffu) {
                ng0 = crec[2 * size_t(j)];
                ng1 = crec[2 * size_t(j) + 1];
            } else {
                lf_next = 0;
                ng0 = ng1 = make_uint4(0, 0, 0, 0);
            }
        };
        fetch_leaves(tile_of(warp));
        for (uint32_t k = warp; tile_of(k) < ntiles; k += kProducers) {
            const uint32_t slot = k % kRing, use = k / kRing;
            const uint32_t t = tile_of(k);
            fetch(t, leaves[0], 0);
            if (use > 0)
                while (ld_acquire(&empty[slot]) != k - kRing + 1) __nanosleep(SVLF_RING_SLEEP_NS);
            const uint32_t a_base = ring0 + slot * CT_A_BYTES;
#pragma unroll 1
            for (uint32_t g = 0; g < (SVLF_DEC_EXP == 1 ? 0 : 4); ++g) {
                lf_cur = lf_next;
                g0 = ng0;
                g1 = ng1;
                if (g < 3) {
                    const uint32_t lf = g == 0 ? leaves[1] : (g == 1 ? leaves[2] : leaves[3]);
                    fetch(t, lf, g + 1);
                } else {
                    fetch_leaves(tile_of(k + kProducers));
                }
                const uint32_t wsp[4] = {g1.x, g1.y, g1.z, g1.w};
#if SVLF_DEC_C_PUNROLL == 4
#pragma unroll 4
#elif SVLF_DEC_C_PUNROLL == 8
#pragma unroll 8
#elif SVLF_DEC_C_PUNROLL == 1
#pragma unroll 1
#else
#pragma unroll 2
#endif
                for (uint32_t p = 0; p < 8; ++p) {
                    const uint32_t src = 4 * p + hsub;
                    const uint32_t lf = __shfl_sync(0xffffffffu, lf_cur, src);
                    uint32_t wt[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) wt[i] = __shfl_sync(0xffffffffu, wsp[i], src);
                    const uint4* row = reinterpret_cast<const uint4*>(fc16 + size_t(lf) * 256) + cp * 4 + ch;
                    uint4 fq[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) fq[i] = __ldg(row + 8 * i);  // corner 2i + cp
                    H2 a1[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) a1[i] = F::splat(0.f);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const H2 pw = u2h<H2>(wt[i]);
                        const H2 hw = cp ? F::hi2(pw) : F::lo2(pw);
                        const H2* f = reinterpret_cast<const H2*>(&fq[i]);
#pragma unroll
                        for (int e = 0; e < 4; ++e) a1[e] = __hfma2(hw, f[e], a1[e]);
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        a1[e] = __hadd2(a1[e], u2h<H2>(__shfl_xor_sync(0xffffffffu, h2u(a1[e]), 4)));
                    if (cp == 0)
                        st_shared_v4(a_base + a_off(32 * g + src, 8 * ch), h2u(a1[0]), h2u(a1[1]), h2u(a1[2]),
                                     h2u(a1[3]));
                }
                st_shared_v4(a_base + a_off(32 * g + lane, 32), g0.x, g0.y, g0.z, F::kOne);
                st_shared_v4(a_base + a_off(32 * g + lane, 40), 0u, 0u, 0u, 0u);
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) st_release(&full[slot], k + 1);
        }
    } else {
        // ---- consumer chain: 4 warps, thread r owns row (TMEM lane) r; k = chain, chain + kChains, ...
        // TMEM: accumulators of chains 0, 1, 2 at columns 0, 128, 256; the
        // 16-bit A operands of chains 0, 1 at 384, 448. Chain 2 (if present)
        // keeps its A operand in shared memory.
        const uint32_t chain = (warp - kProducers) >> 2, r = tid & 127;
        const bool tm = chain < kChainsTm;
        const uint32_t lane_off = (32u * (warp & 3u)) << 16;
        const uint32_t acc = tmem + chain * 128, a_t = tmem + 384 + 64 * chain;
        const uint32_t a_sm = sbase + CT_SMA0 + (chain - kChainsTm) * C_A_BYTES;
        constexpr uint32_t W0 = 0, W1 = OFF_WC1 - OFF_WC0, W2 = OFF_WC2 - OFF_WC0, W3 = OFF_WC3 - OFF_WC0;
        constexpr uint32_t WB1 = OFF_WB1 - OFF_WC0, WB2 = OFF_WB2 - OFF_WC0;
        const uint64_t ones = make_desc(sbase + (OFF_ONES - OFF_WC0), 128, 256);
        const float* cvec = reinterpret_cast<const float*>(sm + (OFF_CVEC - OFF_WC0));
        uint64_t* cbar = &bars[chain];
        uint32_t phase = 0;
        const uint32_t bar_id = 1 + chain;
        auto sync_issue = [&](auto&& f) {
            fence_async_smem();
            fence_before_sync();
            named_sync(bar_id, 128);
            if (r == 0) {
                fence_after_sync();
                f();
                mma_commit(cbar);
            }
        };
        auto wait = [&]() {
            mbar_wait(cbar, phase);
            phase ^= 1;
            fence_after_sync();
        };
        auto epilogue = [&]() {  // acc -> relu -> 16-bit pairs -> A (TMEM or shared memory)
            if (!tm) {
                hidden_epilogue<kBF16, false>(acc + lane_off, a_sm, r, KH, nullptr);
                return;
            }
#if SVLF_DEC_EPI64
#pragma unroll 1
            for (uint32_t hh = 0; hh < 2; ++hh) {
                float v[64];
                tmem_ld32(acc + lane_off + 64 * hh, v);
                tmem_ld32(acc + lane_off + 64 * hh + 32, v + 32);
                tmem_wait_ld();
                uint32_t pk[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) pk[i] = F::relu_pack(v[2 * i], v[2 * i + 1]);
                tmem_st16(a_t + lane_off + 32 * hh, pk);
                tmem_st16(a_t + lane_off + 32 * hh + 16, pk + 16);
            }
#elif SVLF_DEC_EPI_PIPE
            // 16-column chunks, the next chunk's load in flight while this one is packed
            uint32_t ra[16], rb[16];
            tmem_ld16u(acc + lane_off, ra);
            tmem_wait_ld16(ra);
#pragma unroll
            for (uint32_t c = 0; c < 8; ++c) {
                uint32_t(&cur)[16] = (c & 1) ? rb : ra;
                uint32_t(&nxt)[16] = (c & 1) ? ra : rb;
                if (c + 1 < 8) tmem_ld16u(acc + lane_off + 16 * (c + 1), nxt);
                uint32_t pk[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    pk[i] = F::relu_pack(__uint_as_float(cur[2 * i]), __uint_as_float(cur[2 * i + 1]));
                tmem_st8(a_t + lane_off + 8 * c, pk);
                if (c + 1 < 8) tmem_wait_ld16(nxt);
            }
#else
#pragma unroll 1
            for (uint32_t hh = 0; hh < 4; ++hh) {
                float v[32];
                tmem_ld32(acc + lane_off + 32 * hh, v);
                tmem_wait_ld();
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) pk[i] = F::relu_pack(v[2 * i], v[2 * i + 1]);
                tmem_st16(a_t + lane_off + 16 * hh, pk);
            }
#endif
            tmem_wait_st();
        };
        auto hidden = [&](uint32_t w, uint32_t K, uint32_t idesc) {
            if (tm)
                issue_layer_ta(acc, a_t, sbase + w, K, idesc);
            else
                issue_layer(acc, a_sm, sbase + w, K, idesc);
        };
        for (uint32_t k = chain; tile_of(k) < ntiles; k += kChains) {
            const uint32_t slot = k % kRing, use = k / kRing;
            DEC_STAMP(0);
            if (r == 0)
                while (ld_acquire(&full[slot]) != k + 1) {
                }
            DEC_STAMP(1);
            if (SVLF_DEC_EXP == 2) {
                named_sync(bar_id, 128);
                if (r == 0) st_release(&empty[slot], k + 1);
                continue;
            }
            sync_issue([&] {
                issue_layer(acc, ring0 + slot * CT_A_BYTES, sbase + W0, KC, kIdesc);
            });
            wait();
            DEC_STAMP(2);
            if (r == 0) st_release(&empty[slot], k + 1);  // the input tile is free once layer 0 completed
            epilogue();
            DEC_STAMP(3);
            sync_issue([&] {
                hidden(W1, KH, kIdesc);
                mma_f16(acc, ones, make_desc(sbase + WB1, 128, 256), kIdesc, true);
            });
            wait();
            DEC_STAMP(4);
            epilogue();
            DEC_STAMP(5);
            sync_issue([&] {
                hidden(W2, KH, kIdesc);
                mma_f16(acc, ones, make_desc(sbase + WB2, 128, 256), kIdesc, true);
            });
            wait();
            DEC_STAMP(6);
            epilogue();
            DEC_STAMP(7);
            float hv[4];  // rgb (columns 0..2)
            if (SVLF_DEC_EXP != 5) {
            sync_issue([&] { hidden(W3, KH, kIdescHead); });
            wait();
            DEC_STAMP(8);
            tmem_ld4(acc + lane_off, hv);
            tmem_wait_ld();
            } else { named_sync(bar_id, 128); hv[0]=hv[1]=hv[2]=0.f; }
            const uint32_t j = tile_of(k) * 128 + r;
            if (j < n) {
#pragma unroll
                for (int cc = 0; cc < 3; ++cc)
                    out.rgb[3 * size_t(j) + cc] = __fdividef(1.0f, 1.0f + __expf(-(hv[cc] + cvec[256 + cc])));
            }
            DEC_STAMP(9);
        }
    }
    kernel_teardown(tmem);
}

// ---- f_T pass, warp-specialised ----------------------------------------------
template <bool kBF16>
__global__ void __launch_bounds__(TW_THREADS, 1)
    k_decode_t_ws(DevOctree T, const uint8_t* __restrict__ pack, const typename Fmt<kBF16>::H* __restrict__ ft16,
                  const double* __restrict__ rays, const uint32_t* __restrict__ hit_ray,
                  const uint32_t* __restrict__ hit_leaf, const double* __restrict__ hit_tin,
                  const double* __restrict__ hit_tout, const uint32_t* n_dev, uint32_t cap, HitOut out,
                  uint4* __restrict__ crec, int* err) {
    using F = Fmt<kBF16>;
    using H2 = typename F::H2;
    constexpr uint32_t kIdesc = make_idesc(128, 128, kBF16);
    constexpr uint32_t kIdescHead = make_idesc(128, 16, kBF16);
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + TW_SM_BAR);  // [0,1] chains, full[4], empty[4]
    uint64_t* full = bars + 2;
    uint64_t* empty = full + TW_ENTRIES;
    uint32_t* holder = reinterpret_cast<uint32_t*>(empty + TW_ENTRIES);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        const uint4* src = reinterpret_cast<const uint4*>(pack + OFF_WT0);
        uint4* dst = reinterpret_cast<uint4*>(sm);
        for (uint32_t i = tid; i < T_WEIGHTS / 16; i += blockDim.x) dst[i] = src[i];
    }
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        for (uint32_t i = 0; i < TW_ENTRIES; ++i) {
            mbar_init(&full[i], 4);
            mbar_init(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(holder, 512);
    fence_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *holder;
    const uint32_t sbase = smem_u32(sm);
    const uint32_t n = min(*n_dev, cap);
    const uint32_t ntiles = (n + 127) / 128;
    auto tile_of = [&](uint32_t k) { return blockIdx.x + k * gridDim.x; };

    if (warp < 4 * TW_GROUPS) {
        // ---- producer warp: group g = warp / 4, rows 32 (warp % 4) .. + 31 of tiles k = g, g + TW_GROUPS, ...
        const uint32_t g = warp >> 2, row = 32 * (warp & 3u) + lane;
        const uint32_t q = lane >> 3, ch = lane & 7;
        // the per-hit scalars of a group's next tile are loaded a tile ahead
        uint32_t nleaf = 0, nray = 0;
        double ntin = 0.0, ntout = 0.0;
        auto prefetch = [&](uint32_t t) {
            const uint32_t jn = t * 128 + row;
            if (t < ntiles && jn < n) {
                nleaf = hit_leaf[jn];
                nray = hit_ray[jn];
                ntin = hit_tin[jn];
                ntout = hit_tout[jn];
            }
        };
        prefetch(tile_of(g));
        for (uint32_t k = g; tile_of(k) < ntiles; k += TW_GROUPS) {
            const uint32_t e = k % TW_ENTRIES, use = k / TW_ENTRIES;
            const uint32_t j = tile_of(k) * 128 + row;
            uint32_t r6p[3] = {0, 0, 0}, wp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            float u[6] = {0, 0, 0, 0, 0, 0};
            const uint32_t leaf = nleaf, ray_i = nray;
            const double tin = ntin, tout = ntout;
            prefetch(tile_of(k + TW_GROUPS));
            if (j < n && SVLF_DEC_EXP != 3)
                hit_geom_regs<kBF16>(T, rays, ray_i, leaf, tin, tout, r6p, wp, u, err);
            const uint32_t my_leaf = j < n ? leaf : 0u;
            if (use > 0) mbar_wait_sleep(&empty[e], (use - 1) & 1);
            const uint32_t a_base = sbase + TW_RING0 + e * TW_ENTRY;
            uint32_t* side = reinterpret_cast<uint32_t*>(sm + TW_RING0 + e * TW_ENTRY + T_A_BYTES);
#pragma unroll 2
            for (uint32_t p = 0; p < (SVLF_DEC_EXP == 3 ? 0 : 8); ++p) {
                const uint32_t src = 4 * p + q;
                const uint32_t lf = __shfl_sync(0xffffffffu, my_leaf, src);
                uint32_t w[8];
#pragma unroll
                for (int b = 0; b < 8; ++b) w[b] = __shfl_sync(0xffffffffu, wp[b], src);
                // the leaf's 8 corner rows are contiguous in the per-leaf table (1 KB per leaf)
                const uint4* lrow = reinterpret_cast<const uint4*>(ft16 + size_t(lf) * 512) + ch;
                uint4 fq[8];
#pragma unroll
                for (int b = 0; b < 8; ++b) fq[b] = __ldg(lrow + 8 * b);
                H2 a1[4], a2[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a1[i] = a2[i] = F::splat(0.f);
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const H2 p1 = u2h<H2>(w[b / 2]), p2 = u2h<H2>(w[4 + b / 2]);
                    const H2 h1 = (b & 1) ? F::hi2(p1) : F::lo2(p1);
                    const H2 h2 = (b & 1) ? F::hi2(p2) : F::lo2(p2);
                    const H2* f = reinterpret_cast<const H2*>(&fq[b]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        a1[i] = __hfma2(h1, f[i], a1[i]);
                        a2[i] = __hfma2(h2, f[i], a2[i]);
                    }
                }
                const uint32_t rr = (row & ~31u) + src;
                st_shared_v4(a_base + a_off(rr, 8 * ch), h2u(a1[0]), h2u(a1[1]), h2u(a1[2]), h2u(a1[3]));
                st_shared_v4(a_base + a_off(rr, 64 + 8 * ch), h2u(a2[0]), h2u(a2[1]), h2u(a2[2]), h2u(a2[3]));
            }
            st_shared_v4(a_base + a_off(row, 128), r6p[0], r6p[1], r6p[2], F::kOne);
            st_shared_v4(a_base + a_off(row, 136), 0u, 0u, 0u, 0u);
#pragma unroll
            for (int i = 0; i < 6; ++i) side[i * 128 + row] = __float_as_uint(u[i]);
#pragma unroll
            for (int i = 0; i < 3; ++i) side[(6 + i) * 128 + row] = r6p[i];
            side[9 * 128 + row] = __float_as_uint(float(tin));
            side[10 * 128 + row] = __float_as_uint(float(tout));
            fence_async_smem();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[e])) : "memory");
        }
    } else {
        // ---- MMA chain c: 4 warps, thread r owns row (TMEM lane) r
        // TMEM (256 columns per chain): accumulator, head output, and the 16-bit
        // A operand (hidden activations + the head's bias column).
        const uint32_t c = (warp - 4 * TW_GROUPS) >> 2, r = tid & 127;
        const uint32_t lane_off = (32u * (warp & 3u)) << 16;
        const uint32_t acc = tmem + 256 * c, a_t = acc + 160;  // [acc 128 | head 16 | .. | A 72]
        uint64_t* cbar = &bars[c];
        uint32_t phase = 0;
        const uint32_t bar_id = 1 + c;
        {  // constant head-input columns: K 128 = 1 (bias), K 129..143 = 0
            const uint32_t k1[8] = {F::kOne, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                             a_t + lane_off + 64),
                         "r"(k1[0]), "r"(k1[1]), "r"(k1[2]), "r"(k1[3]), "r"(k1[4]), "r"(k1[5]), "r"(k1[6]),
                         "r"(k1[7])
                         : "memory");
            tmem_wait_st();
        }
        auto sync_issue = [&](auto&& f) {
            fence_before_sync();
            named_sync(bar_id, 128);
            if (r == 0) {
                fence_after_sync();
                f();
                mma_commit(cbar);
            }
        };
        auto wait = [&]() {
            mbar_wait(cbar, phase);
            phase ^= 1;
            fence_after_sync();
        };
        // Software-pipelined chain: the head MMA of tile k (into columns
        // 128..143) and layer 0 of tile k + TW_CHAINS are issued together, so
        // each tile costs one MMA round trip; tile k's outputs are written
        // while tile k + TW_CHAINS's epilogue is next.
        const uint32_t d_head = acc + 128;
        float u[6], ft[2];
        uint32_t r6p[3];
        auto read_side = [&](uint32_t e) {
            const uint32_t* side = reinterpret_cast<const uint32_t*>(sm + TW_RING0 + e * TW_ENTRY + T_A_BYTES);
#pragma unroll
            for (int i = 0; i < 6; ++i) u[i] = __uint_as_float(side[i * 128 + r]);
#pragma unroll
            for (int i = 0; i < 3; ++i) r6p[i] = side[(6 + i) * 128 + r];
            ft[0] = __uint_as_float(side[9 * 128 + r]);
            ft[1] = __uint_as_float(side[10 * 128 + r]);
        };
        auto layer0 = [&](uint32_t k) {
            const uint32_t e = k % TW_ENTRIES;
            issue_layer(acc, sbase + TW_RING0 + e * TW_ENTRY, sbase + OFF_WT0, KT, kIdesc);
            mma_commit(&empty[e]);  // the ring entry is free once layer 0 completed
        };
        uint32_t k = c;
        if (tile_of(k) < ntiles) {
            mbar_wait(&full[k % TW_ENTRIES], (k / TW_ENTRIES) & 1);
            read_side(k % TW_ENTRIES);
            sync_issue([&] { layer0(k); });
            wait();
        }
        for (; tile_of(k) < ntiles; k += TW_CHAINS) {
#if SVLF_DEC_EPI_PIPE
            {  // acc -> relu -> 16-bit pairs -> A (TMEM), 16-column chunks, the next load in flight
                uint32_t ra[16], rb[16];
                tmem_ld16u(acc + lane_off, ra);
                tmem_wait_ld16(ra);
#pragma unroll
                for (uint32_t c = 0; c < 8; ++c) {
                    uint32_t(&cur)[16] = (c & 1) ? rb : ra;
                    uint32_t(&nxt)[16] = (c & 1) ? ra : rb;
                    if (c + 1 < 8) tmem_ld16u(acc + lane_off + 16 * (c + 1), nxt);
                    uint32_t pk[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        pk[i] = F::relu_pack(__uint_as_float(cur[2 * i]), __uint_as_float(cur[2 * i + 1]));
                    tmem_st8(a_t + lane_off + 8 * c, pk);
                    if (c + 1 < 8) tmem_wait_ld16(nxt);
                }
            }
#else
#pragma unroll 1
            for (uint32_t hh = 0; hh < 4; ++hh) {  // acc -> relu -> 16-bit pairs -> A (TMEM)
                float v[32];
                tmem_ld32(acc + lane_off + 32 * hh, v);
                tmem_wait_ld();
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) pk[i] = F::relu_pack(v[2 * i], v[2 * i + 1]);
                tmem_st16(a_t + lane_off + 16 * hh, pk);
            }
#endif
            tmem_wait_st();
            const uint32_t kn = k + TW_CHAINS;
            const bool next = tile_of(kn) < ntiles;
            float cu[6];
            const float cft0 = ft[0], cft1 = ft[1];
            uint32_t cr6[3];
#pragma unroll
            for (int i = 0; i < 6; ++i) cu[i] = u[i];
#pragma unroll
            for (int i = 0; i < 3; ++i) cr6[i] = r6p[i];
            if (next) {
                mbar_wait(&full[kn % TW_ENTRIES], (kn / TW_ENTRIES) & 1);
                read_side(kn % TW_ENTRIES);
            }
            sync_issue([&] {
                if (SVLF_DEC_EXP != 6) issue_layer_ta(d_head, a_t, sbase + OFF_WT1, KT, kIdescHead);
                if (next) layer0(kn);
            });
            wait();
            float hv[4];  // tau, eta (columns 0, 1)
            tmem_ld4(d_head + lane_off, hv);
            tmem_wait_ld();
            const uint32_t j = tile_of(k) * 128 + r;
            if (j < n) {
                const float ee = __fdividef(1.0f, 1.0f + __expf(-hv[1])), ome = 1.0f - ee;
                out.tau[j] = fmaxf(hv[0], 0.f);
                out.eta[j] = cft0 * ee + cft1 * (1.f - ee);  // t_s for the composite (as it computed it)
                const float us[3] = {cu[0] * ee + cu[3] * ome, cu[1] * ee + cu[4] * ome, cu[2] * ee + cu[5] * ome};
                float ws[8];
#pragma unroll
                for (int b = 0; b < 8; ++b)
                    ws[b] = ((b & 1) ? us[0] : 1.f - us[0]) * ((b & 2) ? us[1] : 1.f - us[1]) *
                            ((b & 4) ? us[2] : 1.f - us[2]);
                crec[2 * size_t(j)] = make_uint4(cr6[0], cr6[1], cr6[2], 0u);
                crec[2 * size_t(j) + 1] = make_uint4(F::pack(ws[0], ws[1]), F::pack(ws[2], ws[3]),
                                                     F::pack(ws[4], ws[5]), F::pack(ws[6], ws[7]));
            }
        }
    }
    kernel_teardown(tmem);
}

int g_num_sms = 0;

}  // namespace

// [weights | f_T 16-bit V x 64 | f_C 16-bit V x 32 | f_C per leaf: 8 corner rows, L x 8 x 32]
// The per-leaf tables start on 1 KB boundaries, so every 128-byte row (f_T) or
// corner pair (f_C) of a leaf is one whole L1 line (V * 192 B alone is only
// 64-byte aligned for odd V).
size_t align1k(size_t x) { return (x + 1023) & ~size_t(1023); }
size_t pack_leafc_offset(uint32_t V) { return align1k(OFF_FEAT + size_t(V) * 96 * 2); }
size_t pack_leaft_offset(uint32_t V, uint32_t L) { return align1k(pack_leafc_offset(V) + size_t(L) * 8 * 32 * 2); }
size_t pack_tc_bytes(uint32_t V, uint32_t L) { return pack_leaft_offset(V, L) + size_t(L) * 8 * 64 * 2; }

// Per-leaf copy of the 8 corner rows of the 16-bit f_C features (512 contiguous
// bytes per leaf), so the f_C gather reads whole 128-byte lines.
template <uint32_t kChunks>  // 16-byte chunks per row: 4 (f_C, 64 B) or 8 (f_T, 128 B)
__global__ void k_leaf_rows(const uint32_t* __restrict__ corners, const uint4* __restrict__ rows, uint4* leaf_rows,
                            size_t words) {  // words = L * 8 corners * kChunks
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < words; i += size_t(gridDim.x) * blockDim.x)
        leaf_rows[i] = __ldg(rows + size_t(corners[i / kChunks]) * kChunks + (i % kChunks));
}

void ensure_pack_tc(const DevModel& M, const DevOctree& T, DevBuf& pack, uint64_t& pack_version, uint64_t version,
                    bool bf16, cudaStream_t s) {
    const uint64_t tag = version | (bf16 ? (uint64_t(1) << 63) : 0);  // format in the top bit
    if (pack_version == tag && pack.p) return;
    uint8_t* p = pack.ensure<uint8_t>(pack_tc_bytes(M.V, T.n_leaves));
    const size_t nt = size_t(M.V) * 64, nc = size_t(M.V) * 32;
    const unsigned gt = unsigned((nt / 4 + 255) / 256 + 1), gc = unsigned((nc / 4 + 255) / 256 + 1);
    if (bf16) {
        using H = Fmt<true>::H;
        k_pack_tc<true><<<(128 * KT + 255) / 256, 256, 0, s>>>(M.mt, M.mc, p);
        H* ft = reinterpret_cast<H*>(p + OFF_FEAT);
        k_feat_cvt<true><<<gt, 256, 0, s>>>(M.ft, ft, nt);
        k_feat_cvt<true><<<gc, 256, 0, s>>>(M.fc, ft + nt, nc);
    } else {
        using H = Fmt<false>::H;
        k_pack_tc<false><<<(128 * KT + 255) / 256, 256, 0, s>>>(M.mt, M.mc, p);
        H* ft = reinterpret_cast<H*>(p + OFF_FEAT);
        k_feat_cvt<false><<<gt, 256, 0, s>>>(M.ft, ft, nt);
        k_feat_cvt<false><<<gc, 256, 0, s>>>(M.fc, ft + nt, nc);
    }
    const size_t words = size_t(T.n_leaves) * 8 * 4;
    if (words) {
        const unsigned grid = unsigned(std::min<size_t>((words + 255) / 256, 148 * 32));
        k_leaf_rows<4><<<grid, 256, 0, s>>>(T.corners, reinterpret_cast<const uint4*>(p + OFF_FEAT + size_t(M.V) * 64 * 2),
                                           reinterpret_cast<uint4*>(p + pack_leafc_offset(M.V)), words);
        k_leaf_rows<8><<<grid, 256, 0, s>>>(T.corners, reinterpret_cast<const uint4*>(p + OFF_FEAT),
                                           reinterpret_cast<uint4*>(p + pack_leaft_offset(M.V, T.n_leaves)),
                                           2 * words);
    }
    note_launch(5);
    pack_version = tag;
}

template <bool kBF16>
static void decode_tc_impl(const DevOctree& T, const DevModel& M, const uint8_t* p, const double* rays,
                           const uint32_t* hit_ray, const uint32_t* hit_leaf, const double* hit_tin,
                           const double* hit_tout, const uint32_t* n_dev, uint32_t cap, HitOut out, int* err,
                           uint4* crec, cudaStream_t s) {
    using H = typename Fmt<kBF16>::H;
    static bool attr = false;
    if (!attr) {
        SVLF_CUDA(cudaFuncSetAttribute(k_decode_t<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(T_SM_TOTAL)));
        SVLF_CUDA(cudaFuncSetAttribute(k_decode_c<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C_SM_TOTAL)));
        SVLF_CUDA(cudaFuncSetAttribute(k_decode_t_ws<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(TW_SM_TOTAL)));
        SVLF_CUDA(cudaFuncSetAttribute(k_decode_c_tm<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(CT_SM_TOTAL)));
        attr = true;
    }
    const H* ft = reinterpret_cast<const H*>(p + OFF_FEAT);
    const H* fc = ft + size_t(M.V) * 64;
#if SVLF_DEC_T_WS
    const H* leaft = reinterpret_cast<const H*>(p + pack_leaft_offset(M.V, T.n_leaves));
    k_decode_t_ws<kBF16><<<g_num_sms, TW_THREADS, TW_SM_TOTAL, s>>>(T, p, leaft, rays, hit_ray, hit_leaf, hit_tin,
                                                                   hit_tout, n_dev, cap, out, crec, err);
#else
    k_decode_t<kBF16><<<g_num_sms, kSlots * 128, T_SM_TOTAL, s>>>(T, p, ft, rays, hit_ray, hit_leaf, hit_tin, hit_tout, n_dev,
                                                         cap, out, crec, err);
#endif
#if SVLF_DEC_C_TMEM
    const H* leafc = reinterpret_cast<const H*>(p + pack_leafc_offset(M.V));
    k_decode_c_tm<kBF16><<<g_num_sms, kCtThreads, CT_SM_TOTAL, s>>>(T, p, leafc, hit_leaf, crec, n_dev, cap, out);
#else
    k_decode_c<kBF16><<<g_num_sms, kSlots * 128, C_SM_TOTAL, s>>>(T, p, fc, hit_leaf, crec, n_dev, cap, out);
#endif
    note_launch(2);
}

#if SVLF_DEC_TRACE
extern "C" int svlf_debug_dec_trace(unsigned long long* out) {  // 3 x 64 x 10 stamps
    return int(cudaMemcpyFromSymbol(out, g_dec_trace, sizeof(g_dec_trace)));
}
#endif

void launch_decode_tc(const DevOctree& T, const DevModel& M, const char* pack, bool bf16, const double* rays,
                      const uint32_t* hit_ray, const uint32_t* hit_leaf, const double* hit_tin,
                      const double* hit_tout, const uint32_t* n_dev, uint32_t cap, HitOut out, int* err,
                      void* scratch, cudaStream_t s) {
    if (cap == 0) return;
    if (g_num_sms == 0) {
        int dev = 0;
        SVLF_CUDA(cudaGetDevice(&dev));
        SVLF_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    uint4* crec = static_cast<uint4*>(scratch);
    const uint8_t* p = reinterpret_cast<const uint8_t*>(pack);
    if (bf16)
        decode_tc_impl<true>(T, M, p, rays, hit_ray, hit_leaf, hit_tin, hit_tout, n_dev, cap, out, err, crec, s);
    else
        decode_tc_impl<false>(T, M, p, rays, hit_ray, hit_leaf, hit_tin, hit_tout, n_dev, cap, out, err, crec, s);
}

size_t decode_tc_scratch_bytes(uint32_t n_hits) { return size_t(n_hits) * 32; }

}  // namespace svlfb
