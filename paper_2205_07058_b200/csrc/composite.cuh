// Front-to-back compositing of one ray for the 16-bit tensor-core modes
// (render_tile, src/render.cpp:165-193), warp-cooperative, fp32. Built with
// -fmad=false: no contraction.
#pragma once

#include <cstdint>

namespace svlfb {

// Pixel outputs of a band: ray i -> rgb[3i..3i+2], alpha[i], depth[i].
struct PixelOut {
    const uint32_t* ray_off;
    const uint32_t* ray_cnt;
    float bg0, bg1, bg2;
    float* rgb;
    float* alpha;
    float* depth;
};

// Sum over the warp of five per-lane values, as a reduce-scatter: three
// halving steps (4 + 2 + 1 shuffles) leave each lane with the partial sum of
// value (lane >> 2) & 7 over its half-warp group, two butterfly steps finish
// it (9 shuffles instead of 25 for five full butterflies). Lane L returns the
// warp total of value (L >> 2) & 7 (zero for indices 5..7).
__device__ __forceinline__ float warp_sum5_scatter(const float (&s)[5]) {
    const uint32_t lane = threadIdx.x & 31u;
    const float v8[8] = {s[0], s[1], s[2], s[3], s[4], 0.f, 0.f, 0.f};
    float t[4], u[2];
    const bool h16 = lane & 16u, h8 = lane & 8u, h4 = lane & 4u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float mine = h16 ? v8[4 + i] : v8[i], other = h16 ? v8[i] : v8[4 + i];
        t[i] = mine + __shfl_xor_sync(0xffffffffu, other, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float mine = h8 ? t[2 + i] : t[i], other = h8 ? t[i] : t[2 + i];
        u[i] = mine + __shfl_xor_sync(0xffffffffu, other, 8);
    }
    float v = (h4 ? u[1] : u[0]) + __shfl_xor_sync(0xffffffffu, h4 ? u[0] : u[1], 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v;
}

// A warp composites one ray of `cnt` hits (cnt warp-uniform), 32 hits at a
// time, one hit per lane: transmittance is a warp prefix product of
// exp(-tau), the colour / alpha / depth sums warp reductions. load(k, e, r,
// g, b, ts) supplies hit k's exp(-tau), colour and t_s. Lane L returns the
// ray's sum of value (L >> 2) & 7 of {r, g, b, alpha, depth numerator}.
template <typename Load>
__device__ __forceinline__ float warp_composite_ray(uint32_t cnt, Load&& load) {
    const uint32_t lane = threadIdx.x & 31u;
    float Tr = 1.f, acc = 0.f;
    for (uint32_t k0 = 0; k0 < cnt; k0 += 32) {
        const uint32_t k = k0 + lane;
        float e = 1.f, r = 0.f, g = 0.f, bl = 0.f, ts = 0.f;
        if (k < cnt) load(k, e, r, g, bl, ts);
        // exclusive prefix product of e over the lanes
        float incl = e;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const float v = __shfl_up_sync(0xffffffffu, incl, d);
            if (int(lane) >= d) incl *= v;
        }
        float excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = 1.f;
        const float w = Tr * excl * (1.f - e);
        const float s[5] = {w * r, w * g, w * bl, w, w * ts};
        acc += warp_sum5_scatter(s);
        Tr *= __shfl_sync(0xffffffffu, incl, 31);
    }
    return acc;
}

struct RayComposite {
    float c0, c1, c2, a, d;
};

// rgb = c + (1 - alpha) bg; depth = sum w t_s / alpha above the threshold (src/render.cpp:106-114)
__device__ __forceinline__ void write_pixel(const PixelOut& P, uint32_t ray, const RayComposite& c) {
    const float oma = 1.f - c.a;
    P.rgb[3 * size_t(ray)] = c.c0 + oma * P.bg0;
    P.rgb[3 * size_t(ray) + 1] = c.c1 + oma * P.bg1;
    P.rgb[3 * size_t(ray) + 2] = c.c2 + oma * P.bg2;
    P.alpha[ray] = c.a;
    P.depth[ray] = c.a > 1e-4f ? c.d / c.a : 0.f;
}

}  // namespace svlfb
