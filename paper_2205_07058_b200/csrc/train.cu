// Train step on the GPU: the per-frame body of the reference's train()
// (src/train.cpp:443-479): loss_chunk over the batch (:65-287), gradient sum,
// adam_model_step (:345-360).
//
// Pipeline (rays already traversed, per-ray hit segments sorted):
//   k_prep     per ray: surface voxel (locate() of ray.at(depth_gt) matched
//              against the ray's hits), eta_gt with the reference's
//              "surface point outside voxel" check, active hit range per mode
//              (stage 1 keeps pre-surface + surface hits, or the surface hit
//              only when lambda_empty == 0), skipped / eta_skipped counters.
//   scan/expand  dense list of active hits.
//   forward    per hit: f_T input column (geometry, trilinear gathers);
//              dense layers as GEMMs on feature-major activation matrices
//              (cuBLAS SGEMM in pedantic fp32, or the 3xTF32 tensor-core
//              kernels of gemm_x3.cu) + bias/relu epilogue;
//              per hit: f_T heads, x_s, f_C input column; f_C layers as
//              GEMMs; per hit: rgb head. Activations kept for backward.
//   k_loss     per ray: Eq. 4 surface loss or composite + volumetric loss in
//              fp64 and the composite backward dtau_j = dw_j T_j e_j -
//              sum_{i>j} dw_i w_i (reverse scan), per-ray loss.
//   backward   per hit: f_C head; GEMMs dX = W^T D with relu masks; per hit:
//              colour-feature scatter (unless frozen), positional Jacobian
//              d eta += <dx_s, x1 - x2>, f_T heads; GEMM dX_T; per hit:
//              thickness-feature scatter (atomics); weight gradients
//              dW = D X^T and db = D 1 as GEMM/GEMV over all hits.
//   k_adam     dense bias-corrected Adam in fp64 over every parameter
//              (src/mlp.cpp:277-296), colour tensors skipped when frozen.
// Gradients are sums over rays (no 1/N), as in the reference.
#include <cmath>
#include <cstring>

#include "cublas_dyn.hpp"
#include "nccl_dyn.hpp"

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "gemm_x3.cuh"
#include "mlp_simt.cuh"
#include "train.cuh"

namespace svlfb {

namespace {

// feature-major activation rows (x N hits)
constexpr int A_XT = 0, A_HT = 134, A_XC = 262, A_H1 = 300, A_H2 = 428, A_H3 = 556, A_ROWS = 684;
// feature-major delta rows (dL/d pre-activation of each layer)
constexpr int D_T0 = 0, D_T1 = 128, D_C0 = 130, D_C1 = 258, D_C2 = 386, D_C3 = 514, D_ROWS = 517;

struct PrepArgs {
    const double* rays;
    const double* depth;
    const uint8_t* alpha;
    uint32_t n;
    const uint32_t* ray_off;
    const uint32_t* ray_cnt;
    const uint32_t* hit_leaf;
    const double* hit_tin;
    const double* hit_tout;
    bool surface;
    bool empty_zero;
    uint32_t* act_first;
    uint32_t* act_cnt;
    int* surf_rel;
    double* eta_gt;
    unsigned long long* counters;  // [0] skipped, [1] eta_skipped
};

__device__ __forceinline__ Ray ray_of(const double* rays, uint32_t i) {
    Ray r;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.o[a] = rays[6 * size_t(i) + a];
        r.d[a] = rays[6 * size_t(i) + 3 + a];
    }
    return r;
}

// loss_chunk gather step (src/train.cpp:75-124) for one ray.
__global__ void k_prep(DevOctree T, PrepArgs A, int* err) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= A.n) return;
    const uint32_t off = A.ray_off[r], cnt = A.ray_cnt[r];
    int surf = -1;
    double eg = 0.0;
    if (A.alpha[r]) {
        const Ray ray = ray_of(A.rays, r);
        double p[3];
        ray_at(ray, A.depth[r], p);
        bool inside = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) inside = inside && p[a] >= T.lo[a] && p[a] <= T.hi[a];
        if (inside) {  // locate(), src/octree.cpp:173-183
            uint32_t c[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const uint32_t q = uint32_t(div_cell(T, dsub(p[a], T.lo[a])));
                c[a] = q < T.res - 1 ? q : T.res - 1;
            }
            uint64_t code = 0;
            for (int bit = 0; bit < 21; ++bit)
                code |= (uint64_t((c[0] >> bit) & 1u) << (3 * bit)) | (uint64_t((c[1] >> bit) & 1u) << (3 * bit + 1)) |
                        (uint64_t((c[2] >> bit) & 1u) << (3 * bit + 2));
            for (uint32_t k = 0; k < cnt; ++k) {
                if (T.leaf_codes[A.hit_leaf[off + k]] == code) {
                    surf = int(k);
                    const double tin = A.hit_tin[off + k], tout = A.hit_tout[off + k], d = A.depth[r];
                    if (d < dsub(tin, 1e-6) || d > dadd(tout, 1e-6)) raise_error(err, kErrSurfaceOutside);
                    // eta_gt, src/train.cpp:30-35
                    eg = fmin(fmax(ddiv(dsub(tout, d), dsub(tout, tin)), 0.0), 1.0);
                    break;
                }
            }
        }
    }
    uint32_t first = off, n_act = cnt;
    int srel = surf;
    if (A.surface) {
        if (!A.alpha[r] || surf < 0) {
            atomicAdd(&A.counters[0], 1ull);
            n_act = 0;
            srel = -1;
        } else if (A.empty_zero) {  // surface voxel only (src/train.cpp:105-109)
            first = off + uint32_t(surf);
            n_act = 1;
            srel = 0;
        } else {
            n_act = uint32_t(surf) + 1;
        }
    } else if (A.alpha[r] && surf < 0) {
        atomicAdd(&A.counters[1], 1ull);
    }
    A.act_first[r] = first;
    A.act_cnt[r] = n_act;
    A.surf_rel[r] = srel;
    A.eta_gt[r] = eg;
}

__global__ void k_expand(uint32_t n, const uint32_t* act_first, const uint32_t* act_cnt, const uint32_t* dpos,
                         uint32_t* dhit, uint32_t* dray) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t b = dpos[r], f = act_first[r];
    for (uint32_t k = 0; k < act_cnt[r]; ++k) {
        dhit[b + k] = f + k;
        dray[b + k] = r;
    }
}

struct HitArgs {
    const double* rays;
    const uint32_t* hit_leaf;
    const double* hit_tin;
    const double* hit_tout;
    const uint32_t* dhit;
    const uint32_t* dray;
    const uint32_t* dpos;
    const int* surf_rel;
    uint32_t N;
    uint32_t ld;    // row stride of acts / deltas / dX: N rounded up to 32 (aligned GEMM operands)
    bool surface;
    float* acts;    // A_ROWS x ld
    float* deltas;  // D_ROWS x ld
    float* tau;
    float* eta;
    float* rgb;     // 3 x N (channel-major)
    float* drgb;    // 3 x N
    double* dtau;
    double* deta;
};

__device__ __forceinline__ bool has_color(const HitArgs& H, uint32_t j) {
    if (!H.surface) return true;
    const uint32_t r = H.dray[j];
    return H.surf_rel[r] >= 0 && j == H.dpos[r] + uint32_t(H.surf_rel[r]);
}

// Per-hit geometry shared by forward and backward.
struct HitGeom {
    Ray ray;
    double lo[3], hi[3], x1[3], x2[3];
    uint32_t corners[8];
    float r6[6], w1[8], w2[8];
};

__device__ __forceinline__ bool hit_geom(const DevOctree& T, const HitArgs& H, uint32_t j, HitGeom& g, int* err) {
    const uint32_t h = H.dhit[j];
    g.ray = ray_of(H.rays, H.dray[j]);
    const uint32_t leaf = H.hit_leaf[h];
    leaf_box(T, leaf, g.lo, g.hi);
    ray_at(g.ray, H.hit_tin[h], g.x1);
    ray_at(g.ray, H.hit_tout[h], g.x2);
    if (!parameterize(g.ray, g.lo, g.hi, g.r6)) {
        raise_error(err, kErrTangentRay);
        return false;
    }
    if (!trilinear_at(g.x1, g.lo, g.hi, T, g.w1) || !trilinear_at(g.x2, g.lo, g.hi, T, g.w2)) {
        raise_error(err, kErrPointNotInVoxel);
        return false;
    }
    const uint4* cp = reinterpret_cast<const uint4*>(T.corners + 8 * size_t(leaf));
    const uint4 a = __ldg(cp), b = __ldg(cp + 1);
    g.corners[0] = a.x; g.corners[1] = a.y; g.corners[2] = a.z; g.corners[3] = a.w;
    g.corners[4] = b.x; g.corners[5] = b.y; g.corners[6] = b.z; g.corners[7] = b.w;
    return true;
}

// x_s = x1*eta + x2*(1-eta) and its local coordinates (voxel_batch.hpp:111,129)
__device__ __forceinline__ bool xs_coords(const DevOctree& T, const HitGeom& g, float eta, double* xs, double* u) {
    const double e = double(eta), ome = dsub(1.0, e);
#pragma unroll
    for (int a = 0; a < 3; ++a) xs[a] = dadd(dmul(g.x1[a], e), dmul(g.x2[a], ome));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!(xs[a] >= dsub(g.lo[a], 1e-7) && xs[a] <= dadd(g.hi[a], 1e-7))) return false;
        u[a] = fmin(fmax(div_cell(T, dsub(xs[a], g.lo[a])), 0.0), 1.0);
    }
    return true;
}

__device__ __forceinline__ void weights_from_u(const double* u, float* w) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const double wx = (b & 1) ? u[0] : dsub(1.0, u[0]);
        const double wy = (b & 2) ? u[1] : dsub(1.0, u[1]);
        const double wz = (b & 4) ? u[2] : dsub(1.0, u[2]);
        w[b] = float(dmul(dmul(wx, wy), wz));
    }
}

// ---- forward ------------------------------------------------------------------
// The dense layers are GEMMs over the feature-major activation matrices
// (cuBLAS SGEMM, fp32; see run_train_step); these kernels are the per-hit
// parts around them.

// f_T input column: [r6 | psi_T(x1) | psi_T(x2)] (voxel_batch.hpp:69-96).
// Warp-cooperative: a warp owns 32 consecutive hits (geometry lane = hit); each
// hit's 8 corner rows are read coalesced (lane = 2 features), accumulated in
// the reference's corner order without FMA, staged transposed in shared
// memory and written row by row (coalesced feature-major stores).
constexpr int kInWarps = 2;
__global__ void __launch_bounds__(32 * kInWarps) k_fwd_in_t(DevOctree T, DevModel M, HitArgs H, int* err) {
    __shared__ float st[kInWarps][2 * kFt][33];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t N = H.N;
    const size_t L = H.ld;  // row stride of the feature-major matrices
    const uint32_t j0 = (blockIdx.x * kInWarps + warp) * 32;
    if (j0 >= N) return;
    const uint32_t j = j0 + lane;
    HitGeom g;
    const bool ok = j < N && hit_geom(T, H, j, g, err);
    float* X = H.acts + j;
    if (j < N)
#pragma unroll
        for (int k = 0; k < 6; ++k) X[(A_XT + k) * L] = ok ? g.r6[k] : 0.f;
    uint32_t cs[8];
    float w1[8], w2[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        cs[b] = ok ? g.corners[b] : 0u;
        w1[b] = ok ? g.w1[b] : 0.f;
        w2[b] = ok ? g.w2[b] : 0.f;
    }
    const unsigned live = __ballot_sync(0xffffffffu, ok);
    const uint32_t d = 2 * lane;
    for (int h = 0; h < 32; ++h) {
        float2 a1 = make_float2(0.f, 0.f), a2 = a1;
        if ((live >> h) & 1u) {
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint32_t c = __shfl_sync(0xffffffffu, cs[b], h);
                const float wa = __shfl_sync(0xffffffffu, w1[b], h), wb = __shfl_sync(0xffffffffu, w2[b], h);
                const float2 v = __ldg(reinterpret_cast<const float2*>(M.ft + size_t(c) * kFt) + lane);
                a1.x = __fadd_rn(a1.x, __fmul_rn(wa, v.x));
                a1.y = __fadd_rn(a1.y, __fmul_rn(wa, v.y));
                a2.x = __fadd_rn(a2.x, __fmul_rn(wb, v.x));
                a2.y = __fadd_rn(a2.y, __fmul_rn(wb, v.y));
            }
        }
        st[warp][d][h] = a1.x;
        st[warp][d + 1][h] = a1.y;
        st[warp][kFt + d][h] = a2.x;
        st[warp][kFt + d + 1][h] = a2.y;
    }
    __syncwarp();
    if (j < N)
#pragma unroll 8
        for (int r = 0; r < 2 * kFt; ++r) X[(A_XT + 6 + r) * L] = st[warp][r][lane];
}

// y = relu(y + b[row]) over a rows x N feature-major block (GEMM epilogue)
__global__ void k_bias_relu(float* __restrict__ Y, const float* __restrict__ bias, size_t N, size_t ld) {
    const uint32_t row = blockIdx.y;
    const float b = __ldg(bias + row);
    float* y = Y + size_t(row) * ld;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < N; i += size_t(gridDim.x) * blockDim.x)
        y[i] = fmaxf(y[i] + b, 0.f);
}

// f_T head (tau relu, eta sigmoid), x_s and the f_C input column
// [r6 | psi_C(x_s)] for hits whose colour enters the loss (zeros otherwise).
// The colour gather is warp-cooperative (lane = feature, one coalesced
// 128-byte row per corner) with the result staged transposed in shared memory.
__global__ void __launch_bounds__(32 * kInWarps) k_fwd_mid(DevOctree T, DevModel M, HitArgs H, int* err) {
    using D = DecOffsets;
    __shared__ float st[kInWarps][kFc][33];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t N = H.N;
    const size_t L = H.ld;  // row stride of the feature-major matrices
    const uint32_t j0 = (blockIdx.x * kInWarps + warp) * 32;
    if (j0 >= N) return;
    const uint32_t j = j0 + lane;
    const bool valid = j < N;
    float* X = H.acts + j;
    float eta = 0.5f;
    if (valid) {
        const float* h = X + A_HT * L;
        float y0 = __ldg(M.mt + D::T_B1), y1 = __ldg(M.mt + D::T_B1 + 1);
#pragma unroll 16
        for (int k = 0; k < kHid; ++k) {
            const float v = __ldg(h + size_t(k) * L);
            y0 = fmaf(__ldg(M.mt + D::T_W1 + k), v, y0);
            y1 = fmaf(__ldg(M.mt + D::T_W1 + kHid + k), v, y1);
        }
        eta = sigmoid_ref(y1);
        H.tau[j] = y0 > 0.f ? y0 : 0.f;
        H.eta[j] = eta;
    }
    bool ok = false;
    HitGeom g;
    float ws[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (valid && has_color(H, j) && hit_geom(T, H, j, g, err)) {
        double xs[3], u[3];
        if (!xs_coords(T, g, eta, xs, u)) {
            raise_error(err, kErrPointNotInVoxel);
        } else {
            weights_from_u(u, ws);
            ok = true;
        }
    }
    if (valid)
#pragma unroll
        for (int k = 0; k < 6; ++k) X[(A_XC + k) * L] = ok ? g.r6[k] : 0.f;
    uint32_t cs[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) cs[b] = ok ? g.corners[b] : 0u;
    const unsigned live = __ballot_sync(0xffffffffu, ok);
    for (int h = 0; h < 32; ++h) {
        float acc = 0.f;
        if ((live >> h) & 1u) {
#pragma unroll
            for (int b = 0; b < 8; ++b) {  // corner order, no FMA: interp_into_column (voxel_batch.hpp:22-37)
                const uint32_t c = __shfl_sync(0xffffffffu, cs[b], h);
                const float w = __shfl_sync(0xffffffffu, ws[b], h);
                acc = __fadd_rn(acc, __fmul_rn(w, __ldg(M.fc + size_t(c) * kFc + lane)));
            }
        }
        st[warp][lane][h] = acc;
    }
    __syncwarp();
    if (valid)
#pragma unroll 8
        for (int r = 0; r < kFc; ++r) X[(A_XC + 6 + r) * L] = st[warp][r][lane];
}

// f_C head: rgb = sigmoid(W3 h3 + b3)
__global__ void __launch_bounds__(128) k_fwd_rgb(DevModel M, HitArgs H) {
    using D = DecOffsets;
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= H.N) return;
    const size_t N = H.N;
    const size_t L = H.ld;  // row stride of the feature-major matrices
    if (!has_color(H, j)) {
        for (int c = 0; c < 3; ++c) H.rgb[c * N + j] = 0.f;
        return;
    }
    const float* h = H.acts + A_H3 * L + j;
    float y[3] = {__ldg(M.mc + D::C_B3), __ldg(M.mc + D::C_B3 + 1), __ldg(M.mc + D::C_B3 + 2)};
#pragma unroll 16
    for (int k = 0; k < kHid; ++k) {
        const float v = __ldg(h + size_t(k) * L);
#pragma unroll
        for (int c = 0; c < 3; ++c) y[c] = fmaf(__ldg(M.mc + D::C_W3 + c * kHid + k), v, y[c]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) H.rgb[c * N + j] = sigmoid_ref(y[c]);
}

// ---- loss + composite backward (per ray) ---------------------------------------
struct LossArgs {
    const float* c_gt;
    const uint8_t* alpha;
    const uint32_t* dpos;
    const uint32_t* act_cnt;
    const int* surf_rel;
    const double* eta_gt;
    const double* hit_tin;  // unused: t_s is not part of the loss
    uint32_t n;
    bool surface;
    svlf_loss_weights lw;
    double* ray_loss;
    double* ehit;
    double* trans;
    double* wgt;
};

__global__ void k_loss(LossArgs L, HitArgs H) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= L.n) return;
    const size_t N = H.N;
    const uint32_t b = L.dpos[r], cnt = L.act_cnt[r];
    const int srel = L.surf_rel[r];
    const double eg = L.eta_gt[r];
    double loss = 0.0;
    const double cg[3] = {double(L.c_gt[3 * size_t(r)]), double(L.c_gt[3 * size_t(r) + 1]),
                          double(L.c_gt[3 * size_t(r) + 2])};
    if (L.surface) {  // src/train.cpp:158-181
        if (cnt == 0) {
            L.ray_loss[r] = 0.0;
            return;
        }
        const uint32_t js = b + uint32_t(srel);
        double dc[3];
        for (int ch = 0; ch < 3; ++ch) {
            const double diff = dsub(double(H.rgb[ch * N + js]), cg[ch]);
            loss = dadd(loss, dmul(diff, diff));
            dc[ch] = dmul(2.0, diff);
        }
        const double ediff = dsub(double(H.eta[js]), eg);
        loss = dadd(loss, dmul(dmul(L.lw.eta, ediff), ediff));
        H.deta[js] = dadd(H.deta[js], dmul(dmul(2.0, L.lw.eta), ediff));
        const double e2 = exp(dmul(-2.0, double(H.tau[js])));
        loss = dadd(loss, dmul(L.lw.tau, e2));
        H.dtau[js] = dadd(H.dtau[js], dmul(dmul(-2.0, L.lw.tau), e2));
        for (uint32_t k = 0; k < uint32_t(srel); ++k) {
            const uint32_t j = b + k;
            const double e = exp(-double(H.tau[j]));
            const double olap = dsub(1.0, e);
            loss = dadd(loss, dmul(dmul(L.lw.empty, olap), olap));
            H.dtau[j] = dadd(H.dtau[j], dmul(dmul(dmul(2.0, L.lw.empty), olap), e));
        }
        for (int ch = 0; ch < 3; ++ch) H.drgb[ch * N + js] = float(dc[ch]);
        L.ray_loss[r] = loss;
        return;
    }
    // volumetric: composite, src/train.cpp:184-232
    double color[3] = {0.0, 0.0, 0.0}, alpha = 0.0, Tr = 1.0;
    for (uint32_t k = 0; k < cnt; ++k) {
        const uint32_t j = b + k;
        const double e = exp(-double(H.tau[j]));
        const double w = dmul(Tr, dsub(1.0, e));
        L.ehit[j] = e;
        L.trans[j] = Tr;
        L.wgt[j] = w;
        for (int ch = 0; ch < 3; ++ch) color[ch] = dadd(color[ch], dmul(w, double(H.rgb[ch * N + j])));
        alpha = dadd(alpha, w);
        Tr = dmul(Tr, e);
    }
    double d_color[3];
    for (int ch = 0; ch < 3; ++ch) {
        const double diff = dsub(color[ch], cg[ch]);
        loss = dadd(loss, dmul(diff, diff));
        d_color[ch] = dmul(2.0, diff);
    }
    const double agt = L.alpha[r] ? 1.0 : 0.0;
    loss = dadd(loss, dmul(dmul(L.lw.alpha, dsub(alpha, agt)), dsub(alpha, agt)));
    const double d_alpha = dmul(dmul(2.0, L.lw.alpha), dsub(alpha, agt));
    if (L.alpha[r] && srel >= 0) {
        const uint32_t js = b + uint32_t(srel);
        const double ediff = dsub(double(H.eta[js]), eg);
        loss = dadd(loss, dmul(dmul(L.lw.eta, ediff), ediff));
        H.deta[js] = dadd(H.deta[js], dmul(dmul(2.0, L.lw.eta), ediff));
    }
    double suffix = 0.0;
    for (int64_t k = int64_t(cnt) - 1; k >= 0; --k) {
        const uint32_t j = b + uint32_t(k);
        double dw = d_alpha;
        for (int ch = 0; ch < 3; ++ch) dw = dadd(dw, dmul(d_color[ch], double(H.rgb[ch * N + j])));
        H.dtau[j] = dadd(H.dtau[j], dsub(dmul(dmul(dw, L.trans[j]), L.ehit[j]), suffix));
        suffix = dadd(suffix, dmul(dw, L.wgt[j]));
        for (int ch = 0; ch < 3; ++ch) H.drgb[ch * N + j] = float(dmul(L.wgt[j], d_color[ch]));
    }
    L.ray_loss[r] = loss;
}

// ---- backward -----------------------------------------------------------------
// Layer deltas D (dL/d pre-activation, feature-major) flow through cuBLAS
// GEMMs dX = W^T D; these kernels are the per-hit heads, relu masks and the
// feature-gradient scatters (src/mlp.cpp:151-230, src/train.cpp:243-285).

// f_C head (sigmoid') and its 3 -> 128 back-projection masked by relu'(h3)
__global__ void __launch_bounds__(128) k_bwd_head_c(DevModel M, HitArgs H) {
    using D = DecOffsets;
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= H.N) return;
    const size_t N = H.N;
    const size_t L = H.ld;  // row stride of the feature-major matrices
    float* Dl = H.deltas + j;
    float d3[3] = {0.f, 0.f, 0.f};
    if (has_color(H, j))
        for (int o = 0; o < 3; ++o) {
            const float a = H.rgb[o * N + j];
            d3[o] = H.drgb[o * N + j] * a * (1.0f - a);
        }
#pragma unroll
    for (int o = 0; o < 3; ++o) Dl[(D_C3 + o) * L] = d3[o];
    const float* h3 = H.acts + A_H3 * L + j;
    for (int k0 = 0; k0 < kHid; k0 += 16) {  // 16 activation loads in flight before the stores
        float hv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) hv[i] = __ldg(h3 + size_t(k0 + i) * L);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int k = k0 + i;
            float v = 0.f;
            if (hv[i] > 0.f) {
                v = __ldg(M.mc + D::C_W3 + k) * d3[0];
                v = fmaf(__ldg(M.mc + D::C_W3 + kHid + k), d3[1], v);
                v = fmaf(__ldg(M.mc + D::C_W3 + 2 * kHid + k), d3[2], v);
            }
            Dl[(D_C2 + k) * L] = v;
        }
    }
}

// D *= relu'(H) over a rows x N block
__global__ void k_relu_mask(float* __restrict__ Dm, const float* __restrict__ Hm, size_t count) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x)
        if (!(Hm[i] > 0.f)) Dm[i] = 0.f;
}

// The two feature-gradient kernels below are warp-cooperative: a warp owns 32
// consecutive hits. Per-hit geometry runs lane = hit; the hits' input
// gradients are staged transposed in shared memory (coalesced row loads), and
// each hit's scatter is issued by the whole warp as 16-byte vector atomics
// over contiguous feature rows (8 lanes per 32-float row segment).
constexpr int kScWarps = 4;

// Colour-feature gradient scatter (unless frozen) and the positional
// Jacobian into eta (src/train.cpp:244-265), then the f_T heads' deltas and
// their 2 -> 128 back-projection masked by relu'(h_T).
__global__ void __launch_bounds__(32 * kScWarps) k_bwd_feat_c(DevOctree T, DevModel M, HitArgs H,
                                                               const float* __restrict__ dX, bool color_frozen,
                                                               float* g_fc, int* err) {
    using D = DecOffsets;
    __shared__ float zs[kScWarps][kFc][33];
    __shared__ uint32_t cs[kScWarps][32][8];
    __shared__ float ws_s[kScWarps][32][8];
    __shared__ double dots[kScWarps][32][8];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t N = H.N;
    const size_t L = H.ld;  // row stride of the feature-major matrices
    const uint32_t j0 = (blockIdx.x * kScWarps + warp) * 32;
    if (j0 >= N) return;
    const uint32_t j = j0 + lane;
    const bool valid = j < N;
    HitGeom g;
    double u[3] = {0.0, 0.0, 0.0};
    bool act = valid && has_color(H, j) && hit_geom(T, H, j, g, err);
    if (act) {
        double xs[3];
        if (!xs_coords(T, g, H.eta[j], xs, u)) {
            raise_error(err, kErrPointNotInVoxel);
            act = false;
        }
    }
    {
        float ws[8];
        if (act) weights_from_u(u, ws);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            cs[warp][lane][b] = act ? g.corners[b] : 0u;
            ws_s[warp][lane][b] = act ? ws[b] : 0.f;
        }
    }
#pragma unroll 4
    for (int d = 0; d < kFc; ++d) zs[warp][d][lane] = act ? dX[(6 + d) * L + j] : 0.f;
    __syncwarp();
    unsigned live = __ballot_sync(0xffffffffu, act);
    // scatter + <z_b, dz> per corner, hit by hit
    const uint32_t grp = lane >> 3, f4 = (lane & 7) * 4;   // scatter: corner grp (+4), features f4..f4+3
    const uint32_t cb = lane >> 2, ck = (lane & 3) * 8;    // dots: corner cb, features ck..ck+7
    while (live) {
        const int h = __ffs(live) - 1;
        live &= live - 1;
        if (!color_frozen) {
#pragma unroll
            for (int bp = 0; bp < 2; ++bp) {
                const uint32_t b = grp + 4 * bp;
                const float w = ws_s[warp][h][b];
                const float4 v = make_float4(w * zs[warp][f4][h], w * zs[warp][f4 + 1][h], w * zs[warp][f4 + 2][h],
                                             w * zs[warp][f4 + 3][h]);
                atomicAdd(reinterpret_cast<float4*>(g_fc + size_t(cs[warp][h][b]) * kFc + f4), v);
            }
        }
        const float4* zb = reinterpret_cast<const float4*>(M.fc + size_t(cs[warp][h][cb]) * kFc + ck);
        const float4 za = __ldg(zb), zc = __ldg(zb + 1);
        const float zv[8] = {za.x, za.y, za.z, za.w, zc.x, zc.y, zc.z, zc.w};
        double part = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) part = dadd(part, dmul(double(zv[i]), double(zs[warp][ck + i][h])));
        part = dadd(part, __shfl_xor_sync(0xffffffffu, part, 1));
        part = dadd(part, __shfl_xor_sync(0xffffffffu, part, 2));
        if ((lane & 3) == 0) dots[warp][h][cb] = part;
    }
    __syncwarp();
    double deta = valid ? H.deta[j] : 0.0;
    if (act) {
        // dx_s = sum_b dw_b/du <z_b, dz> / h; d eta += <dx_s, x1 - x2>
        const double inv_h = ddiv(1.0, T.cell_size);
        const double wxv[2] = {dsub(1.0, u[0]), u[0]}, wyv[2] = {dsub(1.0, u[1]), u[1]},
                     wzv[2] = {dsub(1.0, u[2]), u[2]}, dxv[2] = {-1.0, 1.0};
        double dxs[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int bx = b & 1, by = (b >> 1) & 1, bz = (b >> 2) & 1;
            const double gw[3] = {dmul(dmul(dxv[bx], wyv[by]), wzv[bz]), dmul(dmul(wxv[bx], dxv[by]), wzv[bz]),
                                  dmul(dmul(wxv[bx], wyv[by]), dxv[bz])};
            const double sc = dmul(dots[warp][lane][b], inv_h);
#pragma unroll
            for (int a = 0; a < 3; ++a) dxs[a] = dadd(dxs[a], dmul(gw[a], sc));
        }
        const double dx12[3] = {dsub(g.x1[0], g.x2[0]), dsub(g.x1[1], g.x2[1]), dsub(g.x1[2], g.x2[2])};
        deta = dadd(deta, dot3(dxs, dx12));
    }
    if (!valid) return;
    // f_T heads: relu (tau), sigmoid (eta)
    float* Dl = H.deltas + j;
    const float tau = H.tau[j], eta = H.eta[j];
    const float d0 = tau > 0.f ? float(H.dtau[j]) : 0.f;
    const float d1 = float(deta) * eta * (1.0f - eta);
    Dl[D_T1 * L] = d0;
    Dl[(D_T1 + 1) * L] = d1;
    const float* ht = H.acts + A_HT * L + j;
    for (int k0 = 0; k0 < kHid; k0 += 16) {  // 16 activation loads in flight before the stores
        float hv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) hv[i] = __ldg(ht + size_t(k0 + i) * L);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int k = k0 + i;
            float v = 0.f;
            if (hv[i] > 0.f) v = fmaf(__ldg(M.mt + D::T_W1 + kHid + k), d1, __ldg(M.mt + D::T_W1 + k) * d0);
            Dl[(D_T0 + k) * L] = v;
        }
    }
}

// Thickness-feature gradient scatter: g[corner_b] += w1_b dz1 + w2_b dz2
// (dz1, dz2 = rows 6..69 and 70..133 of dX_T), in two 32-feature halves.
__global__ void __launch_bounds__(32 * kScWarps) k_bwd_feat_t(DevOctree T, HitArgs H, const float* __restrict__ dX,
                                                               float* g_ft, int* err) {
    __shared__ float zs[kScWarps][64][33];
    __shared__ uint32_t cs[kScWarps][32][8];
    __shared__ float w1s[kScWarps][32][8], w2s[kScWarps][32][8];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t N = H.N;
    const size_t L = H.ld;  // row stride of the feature-major matrices
    const uint32_t j0 = (blockIdx.x * kScWarps + warp) * 32;
    if (j0 >= N) return;
    const uint32_t j = j0 + lane;
    HitGeom g;
    const bool act = j < N && hit_geom(T, H, j, g, err);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        cs[warp][lane][b] = act ? g.corners[b] : 0u;
        w1s[warp][lane][b] = act ? g.w1[b] : 0.f;
        w2s[warp][lane][b] = act ? g.w2[b] : 0.f;
    }
    const unsigned live0 = __ballot_sync(0xffffffffu, act);
    const uint32_t grp = lane >> 3, f4 = (lane & 7) * 4;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
        __syncwarp();
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
            zs[warp][r][lane] = act ? dX[(6 + 32 * half + r) * L + j] : 0.f;
            zs[warp][32 + r][lane] = act ? dX[(6 + kFt + 32 * half + r) * L + j] : 0.f;
        }
        __syncwarp();
        unsigned live = live0;
        while (live) {
            const int h = __ffs(live) - 1;
            live &= live - 1;
#pragma unroll
            for (int bp = 0; bp < 2; ++bp) {
                const uint32_t b = grp + 4 * bp;
                const float a1 = w1s[warp][h][b], a2 = w2s[warp][h][b];
                float4 v;
                v.x = fmaf(a1, zs[warp][f4][h], a2 * zs[warp][32 + f4][h]);
                v.y = fmaf(a1, zs[warp][f4 + 1][h], a2 * zs[warp][32 + f4 + 1][h]);
                v.z = fmaf(a1, zs[warp][f4 + 2][h], a2 * zs[warp][32 + f4 + 2][h]);
                v.w = fmaf(a1, zs[warp][f4 + 3][h], a2 * zs[warp][32 + f4 + 3][h]);
                atomicAdd(reinterpret_cast<float4*>(g_ft + size_t(cs[warp][h][b]) * kFt + 32 * half + f4), v);
            }
        }
    }
}

__global__ void k_fill(float* p, float v, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = v;
}

// rows (vertices) whose features any active hit touches
__global__ void k_touched(DevOctree T, const uint32_t* hit_leaf, const uint32_t* dhit, uint32_t N, uint8_t* touched) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const uint32_t* c = T.corners + 8 * size_t(hit_leaf[dhit[j]]);
#pragma unroll
    for (int b = 0; b < 8; ++b) touched[c[b]] = 1;
}

// pack / unpack the touched rows of both feature gradients: row r -> [ft 64 | fc 32]
__global__ void k_pack_rows(const uint32_t* rows, const uint32_t* n_rows, const float* g_ft, const float* g_fc,
                            float* packed, bool unpack, float* g_ft_w, float* g_fc_w) {
    const uint32_t k = blockIdx.x;
    if (k >= *n_rows) return;
    const size_t r = rows[k];
    for (uint32_t d = threadIdx.x; d < 96; d += blockDim.x) {
        float* dst = packed + size_t(k) * 96 + d;
        if (!unpack) {
            *dst = d < 64 ? g_ft[r * 64 + d] : g_fc[r * 32 + (d - 64)];
        } else if (d < 64) {
            g_ft_w[r * 64 + d] = *dst;
        } else {
            g_fc_w[r * 32 + (d - 64)] = *dst;
        }
    }
}

struct AdamSeg {
    float* p;
    const float* g;
    float* m;
    float* v;
    size_t n;
    double corr1, corr2;
};
struct AdamSegs {
    AdamSeg seg[14];
    int count;
};

// adam_step, src/mlp.cpp:277-296 (fp64 math, fp32 storage; beta/eps are
// float fields promoted to double; lr is rounded to float first, :427).
__global__ void k_adam(AdamSegs S, float lr) {
    const AdamSeg sg = S.seg[blockIdx.y];
    const double b1 = double(0.9f), b2 = double(0.999f), eps = double(1e-8f);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < sg.n; i += size_t(gridDim.x) * blockDim.x) {
        const double g = sg.g[i];
        const double m = dadd(dmul(b1, double(sg.m[i])), dmul(dsub(1.0, b1), g));
        const double v = dadd(dmul(b2, double(sg.v[i])), dmul(dmul(dsub(1.0, b2), g), g));
        sg.m[i] = float(m);
        sg.v[i] = float(v);
        const double mh = ddiv(m, sg.corr1), vh = ddiv(v, sg.corr2);
        sg.p[i] = float(dsub(double(sg.p[i]), ddiv(dmul(double(lr), mh), dadd(__dsqrt_rn(vh), eps))));
    }
}

}  // namespace

TrainScratch::~TrainScratch() {
    if (blas) cublas_api().Destroy(static_cast<cublasHandle_t>(blas));
    if (h_pinned) cudaFreeHost(h_pinned);
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
}

TrainResult run_train_step(TrainScratch& S, const DevOctree& T, TrainModelRefs& M, const TrainBatchDev& b,
                           const TrainOptions& o, cudaStream_t s, int* err_flag) {
    using D = DecOffsets;
    TrainResult res;
    res.rays = b.n;
    if (!S.h_pinned) {
        SVLF_CUDA(cudaMallocHost(&S.h_pinned, 256));
        for (auto& e : S.ev) SVLF_CUDA(cudaEventCreate(&e));
    }
    const size_t P = M.n_ft + M.n_fc + SVLF_DEC_T_SIZE + SVLF_DEC_C_SIZE;
    SVLF_CUDA(cudaMemsetAsync(M.grads, 0, P * 4, s));
    const uint32_t n = b.n;
    SVLF_CUDA(cudaEventRecord(S.ev[0], s));

    // ---- per-ray preparation and dense active-hit list
    uint32_t* act_first = S.act_first.ensure<uint32_t>(n + 1);
    uint32_t* act_cnt = S.act_cnt.ensure<uint32_t>(n + 1);
    uint32_t* dpos = S.dpos.ensure<uint32_t>(n + 1);
    int* surf_rel = S.surf_rel.ensure<int>(n + 1);
    double* eta_gt = S.eta_gt.ensure<double>(n + 1);
    double* ray_loss = S.ray_loss.ensure<double>(n + 1);
    unsigned long long* counters = S.counters.ensure<unsigned long long>(4);
    double* loss_out = S.loss_out.ensure<double>(1);
    SVLF_CUDA(cudaMemsetAsync(counters, 0, 32, s));
    SVLF_CUDA(cudaMemsetAsync(act_cnt + n, 0, 4, s));
    PrepArgs pa{b.rays, b.depth_gt, b.alpha_gt, n, b.ray_off, b.ray_cnt, b.hit_leaf, b.hit_tin, b.hit_tout,
                o.surface, o.lw.empty == 0.0, act_first, act_cnt, surf_rel, eta_gt, counters};
    if (n) k_prep<<<(n + 127) / 128, 128, 0, s>>>(T, pa, err_flag);
    {
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, act_cnt, dpos, int(n + 1));
        SVLF_CUDA(cub::DeviceScan::ExclusiveSum(S.scan_tmp.ensure<char>(tb), tb, act_cnt, dpos, int(n + 1), s));
    }
    SVLF_CUDA(cudaMemcpyAsync(S.h_pinned, dpos + n, 4, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaMemcpyAsync(S.h_pinned + 4, counters, 16, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaStreamSynchronize(s));
    const uint32_t N = uint32_t(S.h_pinned[0]);
    unsigned long long cnts[2];
    std::memcpy(cnts, S.h_pinned + 4, 16);
    res.skipped = (long long)cnts[0];
    res.eta_skipped = (long long)cnts[1];

    uint32_t* dhit = S.dhit.ensure<uint32_t>(N + 1);
    uint32_t* dray = S.dray.ensure<uint32_t>(N + 1);
    float* hitf = S.hitf.ensure<float>(size_t(N) * 8 + 8);
    double* hitd = S.hitd.ensure<double>(size_t(N) * 5 + 5);
    // feature-major matrices with rows padded to 32 floats: aligned leading
    // dimensions let cuBLAS use its vectorised (align4) SGEMM kernels
    const uint32_t Np = (N + 31u) & ~31u;
    float* acts = S.acts.ensure<float>(size_t(A_ROWS) * Np + 1);
    float* deltas = S.deltas.ensure<float>(size_t(D_ROWS) * Np + 1);
    SVLF_CUDA(cudaMemsetAsync(hitd, 0, size_t(N) * 2 * 8, s));                 // dtau, deta
    SVLF_CUDA(cudaMemsetAsync(hitf + size_t(N) * 5, 0, size_t(N) * 3 * 4, s));  // drgb
    float* dxs = S.dxs.ensure<float>(size_t(kInT) * Np + 1);                     // dL/d layer-0 inputs
    if (n) k_expand<<<(n + 127) / 128, 128, 0, s>>>(n, act_first, act_cnt, dpos, dhit, dray);

    // Dense layers as fp32 GEMMs on the feature-major matrices. A feature-major
    // R x N block is the column-major N x R matrix (ld N); a row-major [O][K]
    // weight is the column-major K x O matrix (ld K).
    if (!S.blas) {
        const CublasApi& B = cublas_api();
        cublasHandle_t hb = nullptr;
        cublas_check(B.Create(&hb), "cublasCreate");
        S.blas = hb;
    }
    const CublasApi& B = cublas_api();
    cublasHandle_t hb = static_cast<cublasHandle_t>(S.blas);
    cublas_check(B.SetStream(hb, s), "cublasSetStream");
    // fp32 mode: true fp32 (no TF32) cuBLAS GEMMs on the CUDA cores. tf32 mode:
    // the weight-gradient GEMMs (reductions over all hits) on tensor cores with
    // TF32 operands. tf32x3 mode: every GEMM on the tensor cores as three
    // products of split TF32 operands (gemm_x3.cu), fp32-level accuracy.
    const bool x3 = o.tf32x3;
    cublas_check(B.SetMathMode(hb, CUBLAS_PEDANTIC_MATH), "cublasSetMathMode");
    const float one = 1.f, zero = 0.f;
    const int Ni = int(N), Li = int(Np);
    uint8_t* wimg = x3 ? S.wimg.ensure<uint8_t>(gemm_x3_image_bytes(kInT)) : nullptr;
    // Y(O x N) = W X: rows [xrow, xrow+K) -> [yrow, yrow+O) of acts
    auto layer_fwd = [&](const float* W, int O, int K, int xrow, int yrow, const float* bias) {
        if (x3) {
            gemm_x3_fwd(acts + size_t(xrow) * Np, W, bias, acts + size_t(yrow) * Np, O, K, N, Np, wimg, s);
            return;
        }
        cublas_check(B.Sgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, Ni, O, K, &one, acts + size_t(xrow) * Np, Li, W, K, &zero,
                             acts + size_t(yrow) * Np, Li),
                     "sgemm fwd");
        k_bias_relu<<<dim3(unsigned(std::min<size_t>((N + 255) / 256, 1184)), unsigned(O)), 256, 0, s>>>(
            acts + size_t(yrow) * Np, bias, N, Np);
    };
    // dX rows [k0, K) (x N) = W^T D, D = delta rows [drow, drow+O); with mask_row >= 0 the
    // result is the next delta block: zeroed where the layer's activation (acts row mask_row..) <= 0
    const unsigned mask_blocks = unsigned(std::min<size_t>((size_t(kHid) * Np + 255) / 256, 4736));
    auto layer_bwd = [&](const float* W, int O, int K, int k0, int drow, float* dst, int mask_row) {
        const float* mask = mask_row >= 0 ? acts + size_t(mask_row) * Np : nullptr;
        if (x3) {
            gemm_x3_bwd(deltas + size_t(drow) * Np, W, O, K, k0, dst, mask, N, Np, wimg, s);
            return;
        }
        cublas_check(B.Sgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, Ni, K - k0, O, &one, deltas + size_t(drow) * Np, Li, W + k0,
                             K, &zero, dst, Li),
                     "sgemm bwd");
        if (mask) k_relu_mask<<<mask_blocks, 256, 0, s>>>(dst, mask, size_t(K - k0) * Np);
    };
    // dW(O x K) = D X^T, db = D 1
    float* ones = S.ones.ensure<float>(size_t(N) + 1);
    auto layer_dw = [&](int drow, int O, int xrow, int K, float* dW, float* db) {
        if (x3) {
            gemm_x3_dw(deltas + size_t(drow) * Np, acts + size_t(xrow) * Np, O, K, dW, db, N, Np, s);
            return;
        }
        cublas_check(B.Sgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, K, O, Ni, &one, acts + size_t(xrow) * Np, Li,
                             deltas + size_t(drow) * Np, Li, &zero, dW, K),
                     "sgemm dW");
        cublas_check(B.Sgemv(hb, CUBLAS_OP_T, Ni, O, &one, deltas + size_t(drow) * Np, Li, ones, 1, &zero, db, 1),
                     "sgemv db");
    };
    const unsigned hit_blocks = (N + 127) / 128;

    HitArgs H{b.rays, b.hit_leaf, b.hit_tin, b.hit_tout, dhit, dray, dpos, surf_rel, N, Np, o.surface, acts, deltas,
              hitf, hitf + N, hitf + 2 * size_t(N), hitf + 5 * size_t(N), hitd, hitd + N};
    SVLF_CUDA(cudaEventRecord(S.ev[1], s));
    if (N) {
        k_fill<<<std::min<unsigned>(hit_blocks, 1184), 128, 0, s>>>(ones, 1.f, N);
        k_fwd_in_t<<<unsigned((size_t(N) + 32 * kInWarps - 1) / (32 * kInWarps)), 32 * kInWarps, 0, s>>>(
            T, M.view, H, err_flag);
        layer_fwd(M.view.mt + D::T_W0, kHid, kInT, A_XT, A_HT, M.view.mt + D::T_B0);
        k_fwd_mid<<<unsigned((size_t(N) + 32 * kInWarps - 1) / (32 * kInWarps)), 32 * kInWarps, 0, s>>>(
            T, M.view, H, err_flag);
        layer_fwd(M.view.mc + D::C_W0, kHid, kInC, A_XC, A_H1, M.view.mc + D::C_B0);
        layer_fwd(M.view.mc + D::C_W1, kHid, kHid, A_H1, A_H2, M.view.mc + D::C_B1);
        layer_fwd(M.view.mc + D::C_W2, kHid, kHid, A_H2, A_H3, M.view.mc + D::C_B2);
        k_fwd_rgb<<<hit_blocks, 128, 0, s>>>(M.view, H);
        note_launch(9);
    }
    SVLF_CUDA(cudaEventRecord(S.ev[2], s));
    LossArgs L{b.c_gt, b.alpha_gt, dpos, act_cnt, surf_rel, eta_gt, b.hit_tin, n, o.surface, o.lw, ray_loss,
               hitd + 2 * size_t(N), hitd + 3 * size_t(N), hitd + 4 * size_t(N)};
    if (n) k_loss<<<(n + 127) / 128, 128, 0, s>>>(L, H);
    {
        size_t tb = 0;
        cub::DeviceReduce::Sum(nullptr, tb, ray_loss, loss_out, int(n));
        if (n) SVLF_CUDA(cub::DeviceReduce::Sum(S.scan_tmp.ensure<char>(std::max(tb, size_t(16))), tb, ray_loss,
                                                loss_out, int(n), s));
        else SVLF_CUDA(cudaMemsetAsync(loss_out, 0, 8, s));
    }
    SVLF_CUDA(cudaEventRecord(S.ev[3], s));

    // ---- backward
    float* g_ft = M.grads;
    float* g_fc = M.grads + M.n_ft;
    float* g_mt = g_fc + M.n_fc;
    float* g_mc = g_mt + SVLF_DEC_T_SIZE;
    if (N) {
        // f_C: head -> D_C2; D_C1 = relu'(h2) W2^T D_C2; D_C0 = relu'(h1) W1^T D_C1; dX_C = W0^T D_C0
        k_bwd_head_c<<<hit_blocks, 128, 0, s>>>(M.view, H);
        layer_bwd(M.view.mc + D::C_W2, kHid, kHid, 0, D_C2, deltas + size_t(D_C1) * Np, A_H2);
        layer_bwd(M.view.mc + D::C_W1, kHid, kHid, 0, D_C1, deltas + size_t(D_C0) * Np, A_H1);
        layer_bwd(M.view.mc + D::C_W0, kHid, kInC, 6, D_C0, dxs + 6 * size_t(Np), -1);
        // colour-feature scatter, positional Jacobian, f_T heads -> D_T0
        const unsigned sc_blocks = unsigned((size_t(N) + 32 * kScWarps - 1) / (32 * kScWarps));
        k_bwd_feat_c<<<sc_blocks, 32 * kScWarps, 0, s>>>(T, M.view, H, dxs, o.color_frozen, g_fc, err_flag);
        layer_bwd(M.view.mt + D::T_W0, kHid, kInT, 6, D_T0, dxs + 6 * size_t(Np), -1);
        k_bwd_feat_t<<<sc_blocks, 32 * kScWarps, 0, s>>>(T, H, dxs, g_ft, err_flag);
        // weight gradients (sums over hits)
        if (o.tf32 && !x3) cublas_check(B.SetMathMode(hb, CUBLAS_TF32_TENSOR_OP_MATH), "cublasSetMathMode");
        layer_dw(D_T0, kHid, A_XT, kInT, g_mt + D::T_W0, g_mt + D::T_B0);
        layer_dw(D_T1, 2, A_HT, kHid, g_mt + D::T_W1, g_mt + D::T_B1);
        if (!o.color_frozen) {
            layer_dw(D_C0, kHid, A_XC, kInC, g_mc + D::C_W0, g_mc + D::C_B0);
            layer_dw(D_C1, kHid, A_H1, kHid, g_mc + D::C_W1, g_mc + D::C_B1);
            layer_dw(D_C2, kHid, A_H2, kHid, g_mc + D::C_W2, g_mc + D::C_B2);
            layer_dw(D_C3, 3, A_H3, kHid, g_mc + D::C_W3, g_mc + D::C_B3);
        }
        note_launch(6);
    }
    // ---- data parallel: all-reduce loss, statistics and gradients (NCCL)
    if (o.nccl_comm) {
        ncclComm_t comm = static_cast<ncclComm_t>(o.nccl_comm);
        const NcclApi& api = nccl_api();
        auto nccl = nccl_check;
        // loss and counters (as doubles) in one reduction
        double* red = S.red.ensure<double>(4);
        SVLF_CUDA(cudaMemcpyAsync(red, loss_out, 8, cudaMemcpyDeviceToDevice, s));
        const double local_cnt[3] = {double(res.skipped), double(res.eta_skipped), double(res.rays)};
        SVLF_CUDA(cudaMemcpyAsync(red + 1, local_cnt, 24, cudaMemcpyHostToDevice, s));
        nccl(api.AllReduce(red, red, 4, ncclFloat64, ncclSum, comm, s));
        SVLF_CUDA(cudaMemcpyAsync(loss_out, red, 8, cudaMemcpyDeviceToDevice, s));
        // decoders: dense
        nccl(api.AllReduce(g_mt, g_mt, SVLF_DEC_T_SIZE + SVLF_DEC_C_SIZE, ncclFloat32, ncclSum, comm, s));
        // features: union of touched rows (max of 0/1 flags), compacted, summed, scattered back
        const uint32_t V = M.view.V;
        uint8_t* touched = S.touched.ensure<uint8_t>(V);
        SVLF_CUDA(cudaMemsetAsync(touched, 0, V, s));
        if (N) k_touched<<<(N + 127) / 128, 128, 0, s>>>(T, b.hit_leaf, dhit, N, touched);
        nccl(api.AllReduce(touched, touched, V, ncclUint8, ncclMax, comm, s));
        uint32_t* rows = S.rows.ensure<uint32_t>(V);
        uint32_t* n_rows = S.n_rows.ensure<uint32_t>(1);
        size_t tb = 0;
        cub::CountingInputIterator<uint32_t> idx(0);
        cub::DeviceSelect::Flagged(nullptr, tb, idx, touched, rows, n_rows, int(V));
        SVLF_CUDA(cub::DeviceSelect::Flagged(S.scan_tmp.ensure<char>(tb), tb, idx, touched, rows, n_rows, int(V), s));
        SVLF_CUDA(cudaMemcpyAsync(S.h_pinned + 12, n_rows, 4, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        const uint32_t K = uint32_t(S.h_pinned[12]);
        res.exchanged_rows = K;
        if (K) {
            float* packed = S.packed.ensure<float>(size_t(K) * 96);
            k_pack_rows<<<K, 96, 0, s>>>(rows, n_rows, g_ft, g_fc, packed, false, g_ft, g_fc);
            nccl(api.AllReduce(packed, packed, size_t(K) * 96, ncclFloat32, ncclSum, comm, s));
            k_pack_rows<<<K, 96, 0, s>>>(rows, n_rows, g_ft, g_fc, packed, true, g_ft, g_fc);
            note_launch(2);
        }
        SVLF_CUDA(cudaMemcpyAsync(S.h_pinned + 16, red + 1, 24, cudaMemcpyDeviceToHost, s));
        SVLF_CUDA(cudaStreamSynchronize(s));
        double cnt[3];
        std::memcpy(cnt, S.h_pinned + 16, 24);
        res.skipped = (long long)cnt[0];
        res.eta_skipped = (long long)cnt[1];
        res.rays = (long long)cnt[2];  // statistics of the whole (all-rank) batch
        note_launch(2);
    }
    SVLF_CUDA(cudaEventRecord(S.ev[4], s));

    // ---- Adam (adam_model_step, src/train.cpp:345-360)
    if (o.adam) {
        AdamSegs segs{};
        float* p_ft = M.params;
        float* p_fc = p_ft + M.n_ft;
        float* p_mt = p_fc + M.n_fc;
        float* p_mc = p_mt + SVLF_DEC_T_SIZE;
        const size_t off_fc = M.n_ft, off_mt = M.n_ft + M.n_fc, off_mc = off_mt + SVLF_DEC_T_SIZE;
        auto add = [&](int sid, size_t off, size_t cnt) {
            const uint64_t step = ++M.steps[sid];
            const double c1 = 1.0 - std::pow(double(0.9f), double(step));
            const double c2 = 1.0 - std::pow(double(0.999f), double(step));
            segs.seg[segs.count++] = AdamSeg{M.params + off, M.grads + off, M.adam_m + off, M.adam_v + off, cnt, c1, c2};
        };
        (void)p_ft; (void)p_fc; (void)p_mt; (void)p_mc;
        // ModelAdam tensor order: feat_t, feat_c, f_T (W0,b0,W1,b1), f_C (W0,b0,...,W3,b3)
        add(0, 0, M.n_ft);
        const size_t t_seg[4][2] = {{D::T_W0, kHid * kInT}, {D::T_B0, kHid}, {D::T_W1, 2 * kHid}, {D::T_B1, 2}};
        for (int i = 0; i < 4; ++i) add(2 + i, off_mt + t_seg[i][0], t_seg[i][1]);
        if (!o.color_frozen) {
            add(1, off_fc, M.n_fc);
            const size_t c_seg[8][2] = {{D::C_W0, kHid * kInC}, {D::C_B0, kHid},  {D::C_W1, kHid * kHid},
                                        {D::C_B1, kHid},        {D::C_W2, kHid * kHid}, {D::C_B2, kHid},
                                        {D::C_W3, 3 * kHid},    {D::C_B3, 3}};
            for (int i = 0; i < 8; ++i) add(6 + i, off_mc + c_seg[i][0], c_seg[i][1]);
        }
        dim3 grid(1024, segs.count);
        k_adam<<<grid, 256, 0, s>>>(segs, o.lr);
        note_launch();
    }
    SVLF_CUDA(cudaEventRecord(S.ev[5], s));
    note_launch(6);

    SVLF_CUDA(cudaMemcpyAsync(S.h_pinned + 8, loss_out, 8, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaMemcpyAsync(S.h_pinned + 10, err_flag, 4, cudaMemcpyDeviceToHost, s));
    SVLF_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&res.loss, S.h_pinned + 8, 8);
    res.error = S.h_pinned[10];
    if (res.error) SVLF_CUDA(cudaMemsetAsync(err_flag, 0, 4, s));
    float t[5] = {};
    cudaEventElapsedTime(&t[0], S.ev[0], S.ev[1]);
    cudaEventElapsedTime(&t[1], S.ev[1], S.ev[2]);
    cudaEventElapsedTime(&t[2], S.ev[2], S.ev[3]);
    cudaEventElapsedTime(&t[3], S.ev[3], S.ev[4]);
    cudaEventElapsedTime(&t[4], S.ev[4], S.ev[5]);
    res.timings = svlf_timings{t[0], 0.f, t[1], t[2], t[3], t[4], t[0] + t[1] + t[2] + t[3] + t[4], (long long)N, 0};
    return res;
}

}  // namespace svlfb
