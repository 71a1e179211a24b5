// CUDA-core fp32 building blocks shared by the fp32 render decoder and the
// train step: the transposed fp32 decoder pack, trilinear feature gathers and
// dense layers over one hit per thread, with activations stored feature-major
// (element k of a column at col[k * stride]). Every sum runs in the
// reference's order with no FMA contraction (dense_forward, src/mlp.cpp:98-116;
// interp_into_column, src/voxel_batch.hpp:22-37).
#pragma once

#include "device.cuh"

namespace svlfb {

__host__ __device__ constexpr size_t r4(size_t x) { return (x + 3) & ~size_t(3); }

struct PackOff {
    size_t t_w0t, t_b0, t_w1, t_b1, c_w0t, c_b0, c_w1t, c_b1, c_w2t, c_b2, c_w3, c_b3, total;
};

__host__ __device__ constexpr PackOff pack_offsets() {
    PackOff p{};
    size_t o = 0;
    p.t_w0t = o; o = r4(o + size_t(kInT) * kHid);
    p.t_b0 = o;  o = r4(o + kHid);
    p.t_w1 = o;  o = r4(o + 2 * kHid);
    p.t_b1 = o;  o = r4(o + 2);
    p.c_w0t = o; o = r4(o + size_t(kInC) * kHid);
    p.c_b0 = o;  o = r4(o + kHid);
    p.c_w1t = o; o = r4(o + size_t(kHid) * kHid);
    p.c_b1 = o;  o = r4(o + kHid);
    p.c_w2t = o; o = r4(o + size_t(kHid) * kHid);
    p.c_b2 = o;  o = r4(o + kHid);
    p.c_w3 = o;  o = r4(o + 3 * kHid);
    p.c_b3 = o;  o = r4(o + 3);
    p.total = o;
    return p;
}
inline constexpr PackOff kPack = pack_offsets();
static_assert(kPack.total >= kPackF32Floats, "pack size");

// z = sum_b w_b * row_b (b in order, fp32, no FMA) into a feature-major column.
template <int DIM>
__device__ __forceinline__ void gather_col(const float* __restrict__ vol, const uint32_t* corners,
                                           const float* w, float* col, size_t stride) {
#pragma unroll 1
    for (int d4 = 0; d4 < DIM / 4; ++d4) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(vol + size_t(corners[b]) * DIM) + d4);
            acc.x = __fadd_rn(acc.x, __fmul_rn(w[b], v.x));
            acc.y = __fadd_rn(acc.y, __fmul_rn(w[b], v.y));
            acc.z = __fadd_rn(acc.z, __fmul_rn(w[b], v.z));
            acc.w = __fadd_rn(acc.w, __fmul_rn(w[b], v.w));
        }
        col[(4 * d4 + 0) * stride] = acc.x;
        col[(4 * d4 + 1) * stride] = acc.y;
        col[(4 * d4 + 2) * stride] = acc.z;
        col[(4 * d4 + 3) * stride] = acc.w;
    }
}

// Hidden layer over one column: y[o] = relu(b[o] + sum_k W[o][k] x[k]), k in order.
__device__ __forceinline__ void dense_relu_col(const float* __restrict__ wt, const float* __restrict__ bias,
                                               const float* x, int in, float* y, size_t stride) {
#pragma unroll 1
    for (int o0 = 0; o0 < kHid; o0 += 16) {
        float acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = __ldg(bias + o0 + i);
#pragma unroll 2
        for (int k = 0; k < in; ++k) {
            const float xv = x[k * stride];
            const float4* wr = reinterpret_cast<const float4*>(wt + size_t(k) * kHid + o0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 w = __ldg(wr + q);
                acc[4 * q + 0] = __fadd_rn(acc[4 * q + 0], __fmul_rn(w.x, xv));
                acc[4 * q + 1] = __fadd_rn(acc[4 * q + 1], __fmul_rn(w.y, xv));
                acc[4 * q + 2] = __fadd_rn(acc[4 * q + 2], __fmul_rn(w.z, xv));
                acc[4 * q + 3] = __fadd_rn(acc[4 * q + 3], __fmul_rn(w.w, xv));
            }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) y[(o0 + i) * stride] = acc[i] > 0.f ? acc[i] : 0.f;
    }
}

// Output unit o over a 128-wide hidden column (pre-activation).
__device__ __forceinline__ float head_dot(const float* __restrict__ w, float b, const float* x, size_t stride) {
    float acc = b;
#pragma unroll 4
    for (int k = 0; k < kHid; ++k) acc = __fadd_rn(acc, __fmul_rn(__ldg(w + k), x[k * stride]));
    return acc;
}

// sigmoid as T(1)/(T(1)+exp(-x)) (mlp.cpp:81-84). exp is evaluated in fp64
// and rounded, which reproduces a correctly rounded expf.
__device__ __forceinline__ float sigmoid_ref(float x) {
    const float e = float(exp(-double(x)));
    return __fdiv_rn(1.0f, __fadd_rn(1.0f, e));
}


}  // namespace svlfb
