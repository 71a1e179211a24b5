// Render-path kernels besides traversal:
//   pack_f32     decoder weights -> transposed fp32 pack (per parameter version)
//   decode_f32   per hit: ray parameterisation, trilinear gather at x1/x2,
//                f_T, x_s, gather at x_s, f_C  (CUDA cores, fp32, the
//                reference's accumulation order, no FMA contraction)
//   composite    per ray: front-to-back alpha compositing in fp64
//
// References: parameterize_ray src/render.cpp:16-28; local_coords
// src/features.cpp:22-31; trilinear_weights include/svlf/features.hpp:13-21;
// interp_into_column src/voxel_batch.hpp:22-37; batch_forward_thickness /
// _color src/voxel_batch.hpp:69-142; dense_forward src/mlp.cpp:98-116;
// render_tile composite src/render.cpp:160-193.
#include "composite.cuh"
#include "device.cuh"
#include "mlp_simt.cuh"

namespace svlfb {

namespace {

__global__ void k_pack_f32(const float* __restrict__ mt, const float* __restrict__ mc, float* pack) {
    using D = DecOffsets;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    // transposes: dst[k*128 + o] = W[o*in + k]
    auto tr = [&](const float* W, int in, float* dst, int idx) {
        if (idx < in * kHid) {
            const int k = idx / kHid, o = idx % kHid;
            dst[idx] = W[o * in + k];
        }
    };
    tr(mt + D::T_W0, kInT, pack + kPack.t_w0t, tid);
    tr(mc + D::C_W0, kInC, pack + kPack.c_w0t, tid);
    tr(mc + D::C_W1, kHid, pack + kPack.c_w1t, tid);
    tr(mc + D::C_W2, kHid, pack + kPack.c_w2t, tid);
    if (tid < kHid) {
        pack[kPack.t_b0 + tid] = mt[D::T_B0 + tid];
        pack[kPack.c_b0 + tid] = mc[D::C_B0 + tid];
        pack[kPack.c_b1 + tid] = mc[D::C_B1 + tid];
        pack[kPack.c_b2 + tid] = mc[D::C_B2 + tid];
    }
    if (tid < 2 * kHid) pack[kPack.t_w1 + tid] = mt[D::T_W1 + tid];
    if (tid < 3 * kHid) pack[kPack.c_w3 + tid] = mc[D::C_W3 + tid];
    if (tid < 2) pack[kPack.t_b1 + tid] = mt[D::T_B1 + tid];
    if (tid < 3) pack[kPack.c_b3 + tid] = mc[D::C_B3 + tid];
}

constexpr int kDecBlock = 64;
constexpr int kXRows = 136;  // >= 134 input rows, reused for hidden columns

__global__ void __launch_bounds__(kDecBlock) k_decode_f32(DevOctree T, DevModel M, DecPackF32 P,
                                                          const double* __restrict__ rays,
                                                          const uint32_t* __restrict__ hit_ray,
                                                          const uint32_t* __restrict__ hit_leaf,
                                                          const double* __restrict__ hit_tin,
                                                          const double* __restrict__ hit_tout,
                                                          uint32_t n, HitOut out, int* err) {
    extern __shared__ float smem[];
    const uint32_t j = blockIdx.x * kDecBlock + threadIdx.x;
    if (j >= n) return;
    float* X = smem + threadIdx.x;                      // [136][64] column
    float* H = smem + kXRows * kDecBlock + threadIdx.x; // [128][64] column
    constexpr int S = kDecBlock;

    Ray r;
    const uint32_t ri = hit_ray[j];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.o[a] = rays[6 * size_t(ri) + a];
        r.d[a] = rays[6 * size_t(ri) + 3 + a];
    }
    const uint32_t leaf = hit_leaf[j];
    const double tin = hit_tin[j], tout = hit_tout[j];
    double lo[3], hi[3], x1[3], x2[3];
    leaf_box(T, leaf, lo, hi);
    ray_at(r, tin, x1);
    ray_at(r, tout, x2);

    float r6[6];
    if (!parameterize(r, lo, hi, r6)) {
        raise_error(err, kErrTangentRay);
        return;
    }
    uint32_t corners[8];
    {
        const uint4* cp = reinterpret_cast<const uint4*>(T.corners + 8 * size_t(leaf));
        const uint4 a = __ldg(cp), b = __ldg(cp + 1);
        corners[0] = a.x; corners[1] = a.y; corners[2] = a.z; corners[3] = a.w;
        corners[4] = b.x; corners[5] = b.y; corners[6] = b.z; corners[7] = b.w;
    }
    float w1[8], w2[8];
    if (!trilinear_at(x1, lo, hi, T, w1) || !trilinear_at(x2, lo, hi, T, w2)) {
        raise_error(err, kErrPointNotInVoxel);
        return;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) X[k * S] = r6[k];
    gather_col<kFt>(M.ft, corners, w1, X + 6 * S, S);
    gather_col<kFt>(M.ft, corners, w2, X + (6 + kFt) * S, S);

    // f_T: 134 -> 128 (relu) -> (tau relu, eta sigmoid)
    dense_relu_col(P.t_w0t, P.t_b0, X, kInT, H, S);
    const float y0 = head_dot(P.t_w1, __ldg(P.t_b1), H, S);
    const float y1 = head_dot(P.t_w1 + kHid, __ldg(P.t_b1 + 1), H, S);
    const float tau = y0 > 0.f ? y0 : 0.f;
    const float eta = sigmoid_ref(y1);
    out.tau[j] = tau;
    out.eta[j] = eta;

    // x_s = x1*eta + x2*(1-eta) (voxel_batch.hpp:111)
    const double e = double(eta), ome = dsub(1.0, e);
    double xs[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) xs[a] = dadd(dmul(x1[a], e), dmul(x2[a], ome));
    float ws[8];
    if (!trilinear_at(xs, lo, hi, T, ws)) {
        raise_error(err, kErrPointNotInVoxel);
        return;
    }
    // f_C input: [r6 | psi_C(x_s)] in X rows 0..37
    gather_col<kFc>(M.fc, corners, ws, X + 6 * S, S);
    dense_relu_col(P.c_w0t, P.c_b0, X, kInC, H, S);
    dense_relu_col(P.c_w1t, P.c_b1, H, kHid, X, S);
    dense_relu_col(P.c_w2t, P.c_b2, X, kHid, H, S);
#pragma unroll
    for (int c = 0; c < 3; ++c)
        out.rgb[3 * size_t(j) + c] = sigmoid_ref(head_dot(P.c_w3 + c * kHid, __ldg(P.c_b3 + c), H, S));
}

// render_tile composite, src/render.cpp:165-193 (fp64 accumulation).
__global__ void __launch_bounds__(128) k_composite(const uint32_t* __restrict__ ray_off,
                                                   const uint32_t* __restrict__ ray_cnt,
                                                   const double* __restrict__ tin,
                                                   const double* __restrict__ tout, HitOut h,
                                                   uint32_t n, float bg0, float bg1, float bg2,
                                                   float* rgb, float* alpha, float* depth,
                                                   unsigned long long* fg_count) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    bool fg = false;
    if (i < n) {
        const uint32_t h0 = ray_off[i], h1 = h0 + ray_cnt[i];
        double c0 = 0, c1 = 0, c2 = 0, a = 0, dacc = 0, T = 1.0;
        for (uint32_t j = h0; j < h1; ++j) {
            const double e = exp(-double(h.tau[j]));
            const double w = dmul(T, dsub(1.0, e));
            c0 = dadd(c0, dmul(w, double(h.rgb[3 * size_t(j)])));
            c1 = dadd(c1, dmul(w, double(h.rgb[3 * size_t(j) + 1])));
            c2 = dadd(c2, dmul(w, double(h.rgb[3 * size_t(j) + 2])));
            const double eta = double(h.eta[j]);
            const double ts = dadd(dmul(tin[j], eta), dmul(tout[j], dsub(1.0, eta)));
            dacc = dadd(dacc, dmul(w, ts));
            a = dadd(a, w);
            T = dmul(T, e);
        }
        fg = h1 > h0;
        const double oma = dsub(1.0, a);
        rgb[3 * size_t(i)] = float(dadd(c0, dmul(oma, double(bg0))));
        rgb[3 * size_t(i) + 1] = float(dadd(c1, dmul(oma, double(bg1))));
        rgb[3 * size_t(i) + 2] = float(dadd(c2, dmul(oma, double(bg2))));
        alpha[i] = float(a);
        depth[i] = a > 1e-4 ? float(ddiv(dacc, a)) : 0.f;
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, fg);
    if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(fg_count, (unsigned long long)__popc(ballot));
}

// Composite for the 16-bit tensor-core modes (fp32; the decoder outputs it
// composites are 16-bit-operand results; the fp32 mode keeps the reference's
// sequential fp64 composite above). A warp owns 32 consecutive rays and walks
// each foreground ray's (sorted) segment with warp_composite_ray (coalesced
// hit loads); the five sums of each ray land in a per-warp shared table (one
// store by the five lanes holding them) and every lane writes its own ray's
// pixel at the end. One foreground-count atomic per block.
#ifndef SVLF_COMP_BLOCK
#define SVLF_COMP_BLOCK 128  // (64 / 128 / 256 / 512 measured: 128 best by ~1-2 %)
#endif
constexpr int kCompBlock = SVLF_COMP_BLOCK;
__global__ void __launch_bounds__(kCompBlock) k_composite_warp(HitOut h, uint32_t n, PixelOut P,
                                                               unsigned long long* fg_count) {
    __shared__ float sums[kCompBlock / 32][32][5];
    __shared__ uint32_t s_fg, s_done;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_fg = 0;
        s_done = 0;
    }
    __syncthreads();
    const uint32_t my = blockIdx.x * kCompBlock + threadIdx.x;
    const uint32_t cnt_l = my < n ? P.ray_cnt[my] : 0u, off_l = my < n ? P.ray_off[my] : 0u;
    const unsigned fg = __ballot_sync(0xffffffffu, cnt_l > 0);
    if (lane == 0 && fg) atomicAdd(&s_fg, uint32_t(__popc(fg)));
    const uint32_t vi = (lane >> 2) & 7u;  // which of the ray's five sums this lane ends up holding
    unsigned todo = fg;
    while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t b = __shfl_sync(0xffffffffu, off_l, src), cnt = __shfl_sync(0xffffffffu, cnt_l, src);
        const float v = warp_composite_ray(cnt, [&](uint32_t k, float& e, float& r, float& g, float& bl, float& ts) {
            const uint32_t j = b + k;
            e = __expf(-h.tau[j]);
            r = h.rgb[3 * size_t(j)];
            g = h.rgb[3 * size_t(j) + 1];
            bl = h.rgb[3 * size_t(j) + 2];
            ts = h.eta[j];  // the tensor-core decoder stores t_s = eta t_in + (1 - eta) t_out (fp32)
        });
        if ((lane & 3u) == 0 && vi < 5) sums[warp][src][vi] = v;
    }
    __syncwarp();
    if (my < n) {
        RayComposite c{0.f, 0.f, 0.f, 0.f, 0.f};
        if (cnt_l > 0) c = RayComposite{sums[warp][lane][0], sums[warp][lane][1], sums[warp][lane][2],
                                        sums[warp][lane][3], sums[warp][lane][4]};
        write_pixel(P, my, c);
    }
    // the block's last warp to finish adds the block's foreground count (no block barrier at the end)
    if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&s_done, 1u) == kCompBlock / 32 - 1) {
            const uint32_t t = atomicAdd(&s_fg, 0u);
            if (t) atomicAdd(fg_count, (unsigned long long)t);
        }
    }
}

}  // namespace

DecPackF32 pack_f32_view(float* b) {
    return DecPackF32{b + kPack.t_w0t, b + kPack.t_b0, b + kPack.t_w1, b + kPack.t_b1,
                      b + kPack.c_w0t, b + kPack.c_b0, b + kPack.c_w1t, b + kPack.c_b1,
                      b + kPack.c_w2t, b + kPack.c_b2, b + kPack.c_w3,  b + kPack.c_b3};
}

size_t pack_f32_floats() { return kPack.total; }

void launch_pack_f32(const DevModel& M, float* pack, cudaStream_t s) {
    const int n = kInT * kHid;  // largest segment
    k_pack_f32<<<(n + 255) / 256, 256, 0, s>>>(M.mt, M.mc, pack);
    note_launch();
}

void launch_decode_f32(const DevOctree& T, const DevModel& M, const DecPackF32& P, const double* rays,
                       const uint32_t* hit_ray, const uint32_t* hit_leaf, const double* hit_tin,
                       const double* hit_tout, uint32_t n_hits, HitOut out, int* err, cudaStream_t s) {
    if (n_hits == 0) return;
    const size_t smem = size_t(kXRows + kHid) * kDecBlock * sizeof(float);
    static bool attr = false;
    if (!attr) {
        SVLF_CUDA(cudaFuncSetAttribute(k_decode_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = true;
    }
    k_decode_f32<<<(n_hits + kDecBlock - 1) / kDecBlock, kDecBlock, smem, s>>>(
        T, M, P, rays, hit_ray, hit_leaf, hit_tin, hit_tout, n_hits, out, err);
    note_launch();
}

namespace {
__global__ void __launch_bounds__(kPackBlock) k_pack_fg(const uint32_t* __restrict__ ray_cnt, uint32_t n,
                                                        const float* __restrict__ rgb,
                                                        const float* __restrict__ alpha,
                                                        const float* __restrict__ depth, float* __restrict__ vals,
                                                        uint32_t* __restrict__ tab, uint32_t* count) {
    __shared__ uint32_t wmask[kPackBlock / 32], wbase[kPackBlock / 32 + 1];
    const uint32_t p = blockIdx.x * kPackBlock + threadIdx.x, lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const bool fg = p < n && ray_cnt[p] > 0;
    const uint32_t m = __ballot_sync(0xffffffffu, fg);
    if (lane == 0) wmask[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t w = 0; w < kPackBlock / 32; ++w) {
            wbase[w] = t;
            t += __popc(wmask[w]);
        }
        wbase[kPackBlock / 32] = t ? atomicAdd(count, t) : 0u;
    }
    __syncthreads();
    if (threadIdx.x <= kPackBlock / 32)
        tab[9 * size_t(blockIdx.x) + threadIdx.x] =
            threadIdx.x < kPackBlock / 32 ? wmask[threadIdx.x] : wbase[kPackBlock / 32];
    if (fg) {
        const uint32_t k = wbase[kPackBlock / 32] + wbase[warp] + __popc(m & ((1u << lane) - 1u));
        float* v = vals + 5 * size_t(k);
        v[0] = rgb[3 * size_t(p)];
        v[1] = rgb[3 * size_t(p) + 1];
        v[2] = rgb[3 * size_t(p) + 2];
        v[3] = alpha[p];
        v[4] = depth[p];
    }
}
}  // namespace

void launch_pack_fg(const uint32_t* ray_cnt, uint32_t n, const float* rgb, const float* alpha, const float* depth,
                    float* vals, uint32_t* tab, uint32_t* count, cudaStream_t s) {
    static_assert(kPackBlock == 256, "8 mask words + base per table row");
    if (n == 0) return;
    k_pack_fg<<<(n + kPackBlock - 1) / kPackBlock, kPackBlock, 0, s>>>(ray_cnt, n, rgb, alpha, depth, vals, tab,
                                                                       count);
    note_launch();
}

void launch_composite(const uint32_t* ray_off, const uint32_t* ray_cnt, const double* hit_tin,
                      const double* hit_tout, HitOut hits, uint32_t n_rays, const float* bg3, float* rgb,
                      float* alpha, float* depth, unsigned long long* fg_count, bool exact, cudaStream_t s) {
    if (n_rays == 0) return;
    const float b0 = bg3 ? bg3[0] : 0.f, b1 = bg3 ? bg3[1] : 0.f, b2 = bg3 ? bg3[2] : 0.f;
    if (exact)
        k_composite<<<(n_rays + 127) / 128, 128, 0, s>>>(ray_off, ray_cnt, hit_tin, hit_tout, hits, n_rays, b0, b1,
                                                          b2, rgb, alpha, depth, fg_count);
    else
        k_composite_warp<<<(n_rays + kCompBlock - 1) / kCompBlock, kCompBlock, 0, s>>>(
            hits, n_rays, PixelOut{ray_off, ray_cnt, b0, b1, b2, rgb, alpha, depth}, fg_count);
    note_launch();
}

}  // namespace svlfb
