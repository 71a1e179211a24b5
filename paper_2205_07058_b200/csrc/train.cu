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
//   scan/expand  dense list of active hits (its length stays on the device).
//   forward    per hit: f_T input column (geometry, trilinear gathers);
//              dense layers as 3xTF32 tensor-core GEMMs (gemm_x3.cu) with the
//              bias + relu epilogue fused; per hit: f_T heads, x_s, f_C input
//              column; f_C layers; per hit: rgb head. Activations kept for
//              backward.
//   k_loss     per ray: Eq. 4 surface loss or composite + volumetric loss in
//              fp64 and the composite backward dtau_j = dw_j T_j e_j -
//              sum_{i>j} dw_i w_i (reverse scan), per-ray loss.
//   backward   per hit: f_C head; GEMMs dX = W^T D with fused relu masks; per
//              hit: colour-feature scatter (unless frozen), positional
//              Jacobian d eta += <dx_s, x1 - x2>, f_T heads; GEMM dX_T; per
//              hit: thickness-feature scatter; weight gradients dW = D X^T and
//              db = D 1 as deterministic (CTA-ordered) tensor-core reductions.
//   exchange   (data parallel) loss/statistics, decoder gradients and the
//              union of touched feature rows all-reduced (Collective).
//   k_adam     dense bias-corrected Adam in fp64 over every parameter
//              (src/mlp.cpp:277-296), colour tensors skipped when frozen;
//              skipped on the device when the step raised an error or
//              overflowed a buffer on any rank.
// Gradients are sums over rays (no 1/N), as in the reference.
//
// Nothing in the step reads a count on the host: every per-hit kernel reads
// the active-hit count from the device and loops over it (grids sized by the
// hit capacity), and the single host synchronisation is the final readback
// of one small status record.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "gemm_x3.cuh"
#include "mlp_simt.cuh"
#include "train.cuh"

namespace svlfb {

namespace {

// feature-major activation rows (x ld hits)
constexpr int A_XT = 0, A_HT = 134, A_XC = 262, A_H1 = 300, A_H2 = 428, A_H3 = 556;
// head-layer partials from the forward GEMM epilogues (X3Head): 4 row quarters x outputs
constexpr int A_YT = 684, A_YC = 692, A_ROWS = 704;
// feature-major delta rows (dL/d pre-activation of each layer)
constexpr int D_T0 = 0, D_T1 = 128, D_C0 = 130, D_C1 = 258, D_C2 = 386, D_C3 = 514, D_ROWS = 517;

enum : uint32_t { kStepDeviceError = 4u };

// Status record read back once per step.
struct StepMail {
    double loss, skipped, eta_skipped, rays;
    uint32_t err, flags, hits, active, rows, pad;
};

// red[]: the all-reduced (data parallel) per-step scalars
enum { R_LOSS, R_SKIPPED, R_ETA_SKIPPED, R_RAYS, R_OVERFLOW, R_ERROR, R_COUNT };

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
    const uint32_t* trav_counters;  // [2] != 0: the traversal overflowed its capacity
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
    if (A.trav_counters[2]) {  // hit lists incomplete: the step is a no-op and is re-run
        A.act_first[r] = 0;
        A.act_cnt[r] = 0;
        A.surf_rel[r] = -1;
        A.eta_gt[r] = 0.0;
        return;
    }
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

struct HitArgs {
    const double* rays;
    const uint32_t* hit_leaf;
    const double* hit_tin;
    const double* hit_tout;
    const uint32_t* dhit;
    const uint32_t* dray;
    const uint32_t* dpos;
    const int* surf_rel;
    const uint32_t* n_dev;  // active hits (dpos[n]), read on the device
    uint32_t cap;           // capacity of every per-hit buffer (>= the active hits)
    uint32_t ld;            // row / channel stride of the per-hit matrices: cap rounded up to 32
    bool surface;
    float* acts;    // A_ROWS x ld
    float* deltas;  // D_ROWS x ld
    float* tau;
    float* eta;
    float* rgb;     // 3 x ld (channel-major)
    float* drgb;    // 3 x ld
    double* dtau;
    double* deta;
};

__device__ __forceinline__ uint32_t active_hits(const HitArgs& H) { return min(*H.n_dev, H.cap); }

__device__ __forceinline__ bool has_color(const HitArgs& H, uint32_t j) {
    if (!H.surface) return true;
    const uint32_t r = H.dray[j];
    return H.surf_rel[r] >= 0 && j == H.dpos[r] + uint32_t(H.surf_rel[r]);
}

// dense active-hit list; zeroes the per-hit loss gradients of each active hit
__global__ void k_expand(uint32_t n, const uint32_t* act_first, const uint32_t* act_cnt, const uint32_t* dpos,
                         HitArgs H, uint32_t* dhit, uint32_t* dray) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t b = dpos[r], f = act_first[r], cnt = act_cnt[r];
    for (uint32_t k = 0; k < cnt && b + k < H.cap; ++k) {
        const uint32_t j = b + k;
        dhit[j] = f + k;
        dray[j] = r;
        H.dtau[j] = 0.0;
        H.deta[j] = 0.0;
        H.drgb[j] = 0.f;
        H.drgb[H.ld + j] = 0.f;
        H.drgb[2 * size_t(H.ld) + j] = 0.f;
    }
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
// (gemm_x3.cu); these kernels are the per-hit parts around them. The
// warp-cooperative kernels loop over 32-hit warp tiles up to the device-side
// active count.

// f_T input column: [r6 | psi_T(x1) | psi_T(x2)] (voxel_batch.hpp:69-96).
// A warp owns 32 consecutive hits (geometry lane = hit); each hit's 8 corner
// rows are read coalesced (lane = 2 features), accumulated in the reference's
// corner order without FMA, staged transposed in shared memory 16 hits at a
// time (8.7 KB per warp) and written two rows per store instruction
// (coalesced feature-major half-rows).
constexpr int kInWarps = 2;
__global__ void __launch_bounds__(32 * kInWarps) k_fwd_in_t(DevOctree T, DevModel M, HitArgs H, int* err) {
    __shared__ float st[kInWarps][2 * kFt][17];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t N = active_hits(H);
    const size_t L = H.ld;
    for (uint32_t tile = blockIdx.x * kInWarps + warp; tile * 32 < N; tile += gridDim.x * kInWarps) {
        const uint32_t j = tile * 32 + lane;
        HitGeom g;
        const bool ok = j < N && hit_geom(T, H, j, g, err);
        if (j < N) {
            float* X = H.acts + j;
#pragma unroll
            for (int k = 0; k < 6; ++k) X[(A_XT + k) * L] = ok ? g.r6[k] : 0.f;
        }
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
        const uint32_t sub = lane & 15, rsel = lane >> 4;  // store: hit 16 hh + sub of row r + rsel
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
            __syncwarp();
            for (int h = 16 * hh; h < 16 * hh + 16; ++h) {
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
                const int hl = h - 16 * hh;
                st[warp][d][hl] = a1.x;
                st[warp][d + 1][hl] = a1.y;
                st[warp][kFt + d][hl] = a2.x;
                st[warp][kFt + d + 1][hl] = a2.y;
            }
            __syncwarp();
            const uint32_t jh = tile * 32 + 16 * hh + sub;
            if (jh < N) {
                float* X = H.acts + jh;
#pragma unroll 8
                for (int r = 0; r < 2 * kFt; r += 2) X[(A_XT + 6 + r + rsel) * L] = st[warp][r + rsel][sub];
            }
        }
    }
}

// f_T head (tau relu, eta sigmoid), x_s and the f_C input column
// [r6 | psi_C(x_s)] for hits whose colour enters the loss (zeros otherwise).
// The colour gather is warp-cooperative (lane = feature, one coalesced
// 128-byte row per corner) with the result staged transposed in shared memory.
__global__ void __launch_bounds__(32 * kInWarps) k_fwd_mid(DevOctree T, DevModel M, HitArgs H, int* err) {
    using D = DecOffsets;
    __shared__ float st[kInWarps][kFc][33];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t N = active_hits(H);
    const size_t L = H.ld;
    for (uint32_t tile = blockIdx.x * kInWarps + warp; tile * 32 < N; tile += gridDim.x * kInWarps) {
        const uint32_t j = tile * 32 + lane;
        const bool valid = j < N;
        float* X = H.acts + j;
        float eta = 0.5f;
        if (valid) {
            // bias + the four 32-row partials of the f_T layer-0 GEMM's head epilogue, in order
            const float* y = X + A_YT * L;
            float y0 = __ldg(M.mt + D::T_B1), y1 = __ldg(M.mt + D::T_B1 + 1);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                y0 = __fadd_rn(y0, y[size_t(2 * q) * L]);
                y1 = __fadd_rn(y1, y[size_t(2 * q + 1) * L]);
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
        __syncwarp();
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
}

// f_C head: rgb = sigmoid(W3 h3 + b3)
__global__ void __launch_bounds__(128) k_fwd_rgb(DevModel M, HitArgs H) {
    using D = DecOffsets;
    const uint32_t N = active_hits(H);
    const size_t L = H.ld;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
        if (!has_color(H, j)) {
            for (int c = 0; c < 3; ++c) H.rgb[c * L + j] = 0.f;
            continue;
        }
        // bias + the four 32-row partials of the last f_C GEMM's head epilogue, in order
        const float* yq = H.acts + A_YC * L + j;
        float y[3] = {__ldg(M.mc + D::C_B3), __ldg(M.mc + D::C_B3 + 1), __ldg(M.mc + D::C_B3 + 2)};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int c = 0; c < 3; ++c) y[c] = __fadd_rn(y[c], yq[size_t(3 * q + c) * L]);
#pragma unroll
        for (int c = 0; c < 3; ++c) H.rgb[c * L + j] = sigmoid_ref(y[c]);
    }
}

// ---- loss + composite backward (per ray) ---------------------------------------
struct LossArgs {
    const float* c_gt;
    const uint8_t* alpha;
    const uint32_t* dpos;
    const uint32_t* act_cnt;
    const int* surf_rel;
    const double* eta_gt;
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
    const size_t S = H.ld;
    const uint32_t b = L.dpos[r];
    const uint32_t cnt = b < H.cap ? min(L.act_cnt[r], H.cap - b) : 0u;
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
            const double diff = dsub(double(H.rgb[ch * S + js]), cg[ch]);
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
        for (int ch = 0; ch < 3; ++ch) H.drgb[ch * S + js] = float(dc[ch]);
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
        for (int ch = 0; ch < 3; ++ch) color[ch] = dadd(color[ch], dmul(w, double(H.rgb[ch * S + j])));
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
    if (L.alpha[r] && srel >= 0 && uint32_t(srel) < cnt) {
        const uint32_t js = b + uint32_t(srel);
        const double ediff = dsub(double(H.eta[js]), eg);
        loss = dadd(loss, dmul(dmul(L.lw.eta, ediff), ediff));
        H.deta[js] = dadd(H.deta[js], dmul(dmul(2.0, L.lw.eta), ediff));
    }
    double suffix = 0.0;
    for (int64_t k = int64_t(cnt) - 1; k >= 0; --k) {
        const uint32_t j = b + uint32_t(k);
        double dw = d_alpha;
        for (int ch = 0; ch < 3; ++ch) dw = dadd(dw, dmul(d_color[ch], double(H.rgb[ch * S + j])));
        H.dtau[j] = dadd(H.dtau[j], dsub(dmul(dmul(dw, L.trans[j]), L.ehit[j]), suffix));
        suffix = dadd(suffix, dmul(dw, L.wgt[j]));
        for (int ch = 0; ch < 3; ++ch) H.drgb[ch * S + j] = float(dmul(L.wgt[j], d_color[ch]));
    }
    L.ray_loss[r] = loss;
}

// Per-step scalars: red[R_LOSS] is summed by cub (deterministic), the rest here.
// Overflow: the traversal exceeded the hit buffers, or the active hits
// exceeded the per-hit matrices (act_cap); either way nothing is updated.
__global__ void k_step_scalars(uint32_t n, const unsigned long long* counters, const uint32_t* trav_counters,
                               const uint32_t* n_act, uint32_t act_cap, const int* err, double* red) {
    red[R_SKIPPED] = double(counters[0]);
    red[R_ETA_SKIPPED] = double(counters[1]);
    red[R_RAYS] = double(n);
    red[R_OVERFLOW] = (trav_counters[2] || *n_act > act_cap) ? 1.0 : 0.0;
    red[R_ERROR] = *err ? 1.0 : 0.0;
}

// ---- backward -----------------------------------------------------------------
// Layer deltas D (dL/d pre-activation, feature-major) flow through the GEMMs
// dX = W^T D; these kernels are the per-hit heads and the feature-gradient
// scatters (src/mlp.cpp:151-230, src/train.cpp:243-285).

// f_C head (sigmoid') and its 3 -> 128 back-projection masked by relu'(h3),
// plus the head's weight gradient dW3 = D3 H3^T, db3 = sum D3 (src/mlp.cpp:
// 151-230) from the h3 rows this kernel reads anyway: each warp stages its 32
// hits' h3 rows 32 at a time transposed in shared memory and lane k
// accumulates sum_h d3[c][h] h3[k][h] (fixed order, FMA); the block's warps
// are summed in order into one partial per block (3 x 129 floats), and the
// weight-gradient reduction launch sums the partials in block order
// (bitwise reproducible, like the GEMM partials).
constexpr int kHcThreads = 256;
constexpr uint32_t kHcPartial = 3 * (kHid + 1);
#ifndef SVLF_HC_MINB
#define SVLF_HC_MINB 3  // resident 256-thread blocks per SM (caps the registers at 85)
#endif
__global__ void __launch_bounds__(kHcThreads, SVLF_HC_MINB) k_bwd_head_c(DevModel M, HitArgs H, float* __restrict__ wpart) {
    using D = DecOffsets;
    constexpr int kW = kHcThreads / 32;
    __shared__ float tt[kW][32][33];
    __shared__ float4 dd[kW][32];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t N = active_hits(H);
    const size_t L = H.ld;
    float acc[3][kHid / 32];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < kHid / 32; ++q) acc[c][q] = 0.f;
    float accb = 0.f;  // lanes 0..2: bias gradient of output lane
    for (uint32_t j0 = blockIdx.x * kHcThreads; j0 < N; j0 += gridDim.x * kHcThreads) {
        const uint32_t j = j0 + threadIdx.x;
        const bool valid = j < N;
        float* Dl = H.deltas + j;
        float d3[3] = {0.f, 0.f, 0.f};
        if (valid && has_color(H, j))
            for (int o = 0; o < 3; ++o) {
                const float a = H.rgb[o * L + j];
                d3[o] = H.drgb[o * L + j] * a * (1.0f - a);
            }
        if (valid)
#pragma unroll
            for (int o = 0; o < 3; ++o) Dl[(D_C3 + o) * L] = d3[o];
        dd[warp][lane] = make_float4(d3[0], d3[1], d3[2], 0.f);
        const float* h3 = H.acts + A_H3 * L + j;
#pragma unroll
        for (int q = 0; q < kHid / 32; ++q) {
            const int k0 = 32 * q;
            float hv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) hv[i] = valid ? __ldg(h3 + size_t(k0 + i) * L) : 0.f;
            if (valid)
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int k = k0 + i;
                    float v = 0.f;
                    if (hv[i] > 0.f) {
                        v = __ldg(M.mc + D::C_W3 + k) * d3[0];
                        v = fmaf(__ldg(M.mc + D::C_W3 + kHid + k), d3[1], v);
                        v = fmaf(__ldg(M.mc + D::C_W3 + 2 * kHid + k), d3[2], v);
                    }
                    Dl[(D_C2 + k) * L] = v;
                }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 32; ++i) tt[warp][i][lane] = hv[i];
            __syncwarp();
#pragma unroll 8
            for (int h = 0; h < 32; ++h) {  // lane = k0 + lane, hits in order
                const float t = tt[warp][lane][h];
                const float4 dh = dd[warp][h];
                acc[0][q] = __fmaf_rn(dh.x, t, acc[0][q]);
                acc[1][q] = __fmaf_rn(dh.y, t, acc[1][q]);
                acc[2][q] = __fmaf_rn(dh.z, t, acc[2][q]);
            }
        }
        if (lane < 3)
            for (int h = 0; h < 32; ++h) {
                const float4 dh = dd[warp][h];
                accb = __fadd_rn(accb, lane == 0 ? dh.x : (lane == 1 ? dh.y : dh.z));
            }
        __syncwarp();
    }
    // block partial: warps summed in order; element c * 129 + k (k = 128: bias)
    __syncthreads();
    float* red = &tt[0][0][0];  // kW x kHcPartial floats
    static_assert(kW * kHcPartial <= kW * 32 * 33, "partial staging fits");
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < kHid / 32; ++q) red[warp * kHcPartial + c * (kHid + 1) + 32 * q + lane] = acc[c][q];
    if (lane < 3) red[warp * kHcPartial + lane * (kHid + 1) + kHid] = accb;
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < kHcPartial; e += kHcThreads) {
        float t = red[e];
        for (int w = 1; w < kW; ++w) t = __fadd_rn(t, red[w * kHcPartial + e]);
        wpart[size_t(blockIdx.x) * kHcPartial + e] = t;
    }
}

// The two feature-gradient kernels below are warp-cooperative: a warp owns 32
// consecutive hits. Per-hit geometry runs lane = hit; the hits' input
// gradients are staged transposed in shared memory (coalesced row loads), and
// each hit's scatter is issued by the whole warp as 16-byte vector atomics
// over contiguous feature rows (8 lanes per 32-float row segment).
constexpr int kScWarps = 4;

// Colour-feature gradient scatter (unless frozen) and the positional
// Jacobian into eta (src/train.cpp:244-265), then the f_T heads' deltas,
// their 2 -> 128 back-projection masked by relu'(h_T), and the f_T head's
// weight gradient from the same h_T rows (as in k_bwd_head_c: per-warp
// transposed staging, one partial of 2 x 129 floats per block).
constexpr uint32_t kHtPartial = 2 * (kHid + 1);
#ifndef SVLF_FEATC_MINB
#define SVLF_FEATC_MINB 5  // resident blocks per SM: caps the registers at 96 (no spills; 128 uncapped)
#endif
__global__ void __launch_bounds__(32 * kScWarps, SVLF_FEATC_MINB) k_bwd_feat_c(DevOctree T, DevModel M, HitArgs H,
                                                               const float* __restrict__ dX, bool color_frozen,
                                                               float* g_fc, int* err, float* __restrict__ wpart) {
    using D = DecOffsets;
    __shared__ float zs[kScWarps][kFc][33];
    __shared__ uint32_t cs[kScWarps][32][8];
    __shared__ float ws_s[kScWarps][32][8];
    __shared__ double dots[kScWarps][32][8];
    __shared__ float2 ddt[kScWarps][32];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t N = active_hits(H);
    const size_t L = H.ld;
    float hacc[2][kHid / 32];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < kHid / 32; ++q) hacc[c][q] = 0.f;
    float haccb = 0.f;  // lanes 0, 1: bias gradient of head output lane
    for (uint32_t tile = blockIdx.x * kScWarps + warp; tile * 32 < N; tile += gridDim.x * kScWarps) {
        const uint32_t j = tile * 32 + lane;
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
        __syncwarp();
        {
            float ws[8];
            if (act) weights_from_u(u, ws);
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                cs[warp][lane][b] = act ? g.corners[b] : 0u;
                ws_s[warp][lane][b] = act ? ws[b] : 0.f;
            }
        }
#pragma unroll
        for (int d = 0; d < kFc; ++d) zs[warp][d][lane] = act ? dX[(6 + d) * L + j] : 0.f;
        __syncwarp();
        unsigned live = __ballot_sync(0xffffffffu, act);
        // scatter + <z_b, dz> per corner, hit by hit
        const uint32_t grp = lane >> 3, f4 = (lane & 7) * 4;  // scatter: corner grp (+4), features f4..f4+3
        const uint32_t cb = lane >> 2, ck = (lane & 3) * 8;   // dots: corner cb, features ck..ck+7
        while (live) {
            const int h = __ffs(live) - 1;
            live &= live - 1;
            if (!color_frozen) {
#pragma unroll
                for (int bp = 0; bp < 2; ++bp) {
                    const uint32_t b = grp + 4 * bp;
                    const float w = ws_s[warp][h][b];
                    const float4 v = make_float4(w * zs[warp][f4][h], w * zs[warp][f4 + 1][h],
                                                 w * zs[warp][f4 + 2][h], w * zs[warp][f4 + 3][h]);
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
        // f_T heads: relu (tau), sigmoid (eta)
        float* Dl = H.deltas + j;
        float d0 = 0.f, d1 = 0.f;
        if (valid) {
            const float tau = H.tau[j], eta = H.eta[j];
            d0 = tau > 0.f ? float(H.dtau[j]) : 0.f;
            d1 = float(deta) * eta * (1.0f - eta);
            Dl[D_T1 * L] = d0;
            Dl[(D_T1 + 1) * L] = d1;
        }
        ddt[warp][lane] = make_float2(d0, d1);
        const float* ht = H.acts + A_HT * L + j;
        float* tt = &zs[warp][0][0];  // [32][33]: free once the scatter above is done
#pragma unroll
        for (int q = 0; q < kHid / 32; ++q) {
            const int k0 = 32 * q;
            float hv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) hv[i] = valid ? __ldg(ht + size_t(k0 + i) * L) : 0.f;
            if (valid)
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int k = k0 + i;
                    float v = 0.f;
                    if (hv[i] > 0.f) v = fmaf(__ldg(M.mt + D::T_W1 + kHid + k), d1, __ldg(M.mt + D::T_W1 + k) * d0);
                    Dl[(D_T0 + k) * L] = v;
                }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 32; ++i) tt[i * 33 + lane] = hv[i];
            __syncwarp();
#pragma unroll 8
            for (int h = 0; h < 32; ++h) {  // lane = k0 + lane, hits in order
                const float t = tt[lane * 33 + h];
                const float2 dh = ddt[warp][h];
                hacc[0][q] = __fmaf_rn(dh.x, t, hacc[0][q]);
                hacc[1][q] = __fmaf_rn(dh.y, t, hacc[1][q]);
            }
        }
        if (lane < 2)
            for (int h = 0; h < 32; ++h) {
                const float2 dh = ddt[warp][h];
                haccb = __fadd_rn(haccb, lane == 0 ? dh.x : dh.y);
            }
        __syncwarp();
    }
    // block partial of the f_T head's weight gradient: warps summed in order
    __syncthreads();
    float* red = &zs[0][0][0];
    static_assert(kScWarps * kHtPartial <= kScWarps * kFc * 33, "partial staging fits");
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < kHid / 32; ++q) red[warp * kHtPartial + c * (kHid + 1) + 32 * q + lane] = hacc[c][q];
    if (lane < 2) red[warp * kHtPartial + lane * (kHid + 1) + kHid] = haccb;
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < kHtPartial; e += 32 * kScWarps) {
        float t = red[e];
        for (uint32_t w = 1; w < kScWarps; ++w) t = __fadd_rn(t, red[w * kHtPartial + e]);
        wpart[size_t(blockIdx.x) * kHtPartial + e] = t;
    }
}

// Thickness-feature gradient scatter: g[corner_b] += w1_b dz1 + w2_b dz2
// (dz1, dz2 = rows 6..69 and 70..133 of dX_T), in two 32-feature halves.
__global__ void __launch_bounds__(32 * kScWarps, 4) k_bwd_feat_t(DevOctree T, HitArgs H, const float* __restrict__ dX,
                                                               float* g_ft, int* err) {
    __shared__ float zs[kScWarps][64][33];
    __shared__ uint32_t cs[kScWarps][32][8];
    __shared__ float w1s[kScWarps][32][8], w2s[kScWarps][32][8];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t N = active_hits(H);
    const size_t L = H.ld;
    for (uint32_t tile = blockIdx.x * kScWarps + warp; tile * 32 < N; tile += gridDim.x * kScWarps) {
        const uint32_t j = tile * 32 + lane;
        HitGeom g;
        const bool act = j < N && hit_geom(T, H, j, g, err);
        __syncwarp();
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
#pragma unroll
            for (int r = 0; r < 32; ++r) {  // all 64 row loads in flight
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
}

// rows (vertices) whose features any active hit touches
__global__ void k_touched(DevOctree T, const uint32_t* hit_leaf, const uint32_t* dhit, const uint32_t* n_dev,
                          uint32_t cap, uint8_t* touched) {
    const uint32_t N = min(*n_dev, cap);
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
        const uint32_t* c = T.corners + 8 * size_t(hit_leaf[dhit[j]]);
#pragma unroll
        for (int b = 0; b < 8; ++b) touched[c[b]] = 1;
    }
}

// pack / unpack the touched rows of both feature gradients: row r -> [ft 64 | fc 32].
// Pack writes rows_cap rows (zeros past the touched count) and flags a count
// above rows_cap (the step is then skipped and re-run with a larger buffer).
__global__ void k_pack_rows(const uint32_t* rows, const uint32_t* n_rows, uint32_t rows_cap, float* g_ft, float* g_fc,
                            float* packed, bool unpack, uint32_t* status) {
    const uint32_t nr = *n_rows;
    if (!unpack && nr > rows_cap && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, uint32_t(kStepRowOverflow));
    const uint32_t lim = unpack ? min(nr, rows_cap) : rows_cap;
    const uint32_t kt = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
    for (uint32_t k = blockIdx.x * warps + kt; k < lim; k += gridDim.x * warps) {
        float* dst = packed + size_t(k) * 96;
        if (k >= nr) {
            for (uint32_t d = lane; d < 96; d += 32) dst[d] = 0.f;
            continue;
        }
        const size_t r = rows[k];
        if (!unpack) {
            dst[lane] = g_ft[r * 64 + lane];
            dst[32 + lane] = g_ft[r * 64 + 32 + lane];
            dst[64 + lane] = g_fc[r * 32 + lane];
        } else {
            g_ft[r * 64 + lane] = dst[lane];
            g_ft[r * 64 + 32 + lane] = dst[32 + lane];
            g_fc[r * 32 + lane] = dst[64 + lane];
        }
    }
}

// skip bits of the step from the (all-reduced) flags
__global__ void k_step_status(const double* red, uint32_t* status) {
    uint32_t s = *status;
    if (red[R_OVERFLOW] > 0.0) s |= kStepHitOverflow;
    if (red[R_ERROR] > 0.0) s |= kStepDeviceError;
    *status = s;
}

__global__ void k_step_mail(const double* red, const uint32_t* status, const int* err, const uint32_t* trav_counters,
                            const uint32_t* n_act, uint32_t cap, const uint32_t* n_rows, StepMail* mail) {
    StepMail m;
    m.loss = red[R_LOSS];
    m.skipped = red[R_SKIPPED];
    m.eta_skipped = red[R_ETA_SKIPPED];
    m.rays = red[R_RAYS];
    m.err = uint32_t(*err);
    m.flags = *status;
    m.hits = trav_counters[0];
    m.active = *n_act;  // unclamped: sizes the next step's matrices
    m.rows = n_rows ? *n_rows : 0u;
    m.pad = 0;
    *mail = m;
}

// Dense Adam over the flat parameter buffer [feat_t | feat_c | f_T W0 b0 W1 b1 |
// f_C W0 b0 .. W3 b3], whose tensor order is ModelAdam's: tensor t covers
// [end[t-1], end[t]) with its own step-count correction and hyperparameters.
struct AdamPlan {
    size_t end[14];
    double corr1[14], corr2[14];
    float beta1[14], beta2[14], eps[14];
    uint32_t active;  // bit t: tensor t is updated (colour tensors frozen: not)
    float lr;
};

// adam_step, src/mlp.cpp:277-296 (fp64 math, fp32 storage; beta/eps are the
// AdamState float fields promoted to double; lr is rounded to float first,
// src/train.cpp:427), one element.
__device__ __forceinline__ void adam_elem(const AdamPlan& A, int t, double lr, float& p, float g, float& m, float& v) {
    // g = m = v = +0: the update is exactly the identity (m, v stay +0, the step is
    // 0 / (0 + eps) = 0 and p - 0 = p), and every fp64 operation below would take
    // its special-case slow path; rows untouched since initialisation are all such
    if ((__float_as_uint(g) | __float_as_uint(m) | __float_as_uint(v)) == 0u) return;
    const double b1 = double(A.beta1[t]), b2 = double(A.beta2[t]), eps = double(A.eps[t]);
    const double gd = g;
    const double mm = dadd(dmul(b1, double(m)), dmul(dsub(1.0, b1), gd));
    const double vv = dadd(dmul(b2, double(v)), dmul(dmul(dsub(1.0, b2), gd), gd));
    m = float(mm);
    v = float(vv);
    const double mh = ddiv(mm, A.corr1[t]), vh = ddiv(vv, A.corr2[t]);
    p = float(dsub(double(p), ddiv(dmul(lr, mh), dadd(__dsqrt_rn(vh), eps))));
}

__device__ __forceinline__ int adam_tensor(const AdamPlan& A, size_t i) {
    int t = 0;
#pragma unroll 1
    while (t < 13 && i >= A.end[t]) ++t;
    return t;
}

// Grid-stride over groups of kAdamVec consecutive parameters of all four
// arrays (vector loads; 28 B per parameter); a group that straddles a tensor
// boundary goes element by element. The fp64 divisions / square root make it
// issue-bound rather than HBM-bound, so the group width and the occupancy are
// build parameters (measured on the B200). Skipped when the step is flagged.
#ifndef SVLF_ADAM_VEC
#define SVLF_ADAM_VEC 4
#endif
#ifndef SVLF_ADAM_MINB
#define SVLF_ADAM_MINB 4
#endif
constexpr int kAdamVec = SVLF_ADAM_VEC;
template <int V>
struct VecF;
template <>
struct VecF<1> {
    using T = float;
};
template <>
struct VecF<2> {
    using T = float2;
};
template <>
struct VecF<4> {
    using T = float4;
};

__global__ void __launch_bounds__(256, SVLF_ADAM_MINB)
    k_adam(float* __restrict__ P, const float* __restrict__ G, float* __restrict__ M, float* __restrict__ Vv,
           size_t total, const AdamPlan* __restrict__ plan, const uint32_t* skip_if, const int* err) {
    using VT = typename VecF<kAdamVec>::T;
    if ((skip_if && *skip_if) || (err && *err)) return;
    __shared__ AdamPlan A;  // the step's corrections / hyperparameters (device memory: graph replays stay valid)
    if (threadIdx.x == 0) A = *plan;
    __syncthreads();
    const double lrd = double(A.lr);
    const size_t groups = (total + kAdamVec - 1) / kAdamVec;
    for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < groups; q += size_t(gridDim.x) * blockDim.x) {
        const size_t i0 = kAdamVec * q;
        const int t = adam_tensor(A, i0);
        if (i0 + kAdamVec - 1 < total && i0 + kAdamVec - 1 < A.end[t]) {
            if (!((A.active >> t) & 1u)) continue;
            VT p = reinterpret_cast<VT*>(P)[q];
            const VT g = __ldg(reinterpret_cast<const VT*>(G) + q);
            VT m = reinterpret_cast<VT*>(M)[q];
            VT v = reinterpret_cast<VT*>(Vv)[q];
            float* pp = reinterpret_cast<float*>(&p);
            const float* gg = reinterpret_cast<const float*>(&g);
            float* mm = reinterpret_cast<float*>(&m);
            float* vv = reinterpret_cast<float*>(&v);
#pragma unroll
            for (int k = 0; k < kAdamVec; ++k) adam_elem(A, t, lrd, pp[k], gg[k], mm[k], vv[k]);
            reinterpret_cast<VT*>(P)[q] = p;
            reinterpret_cast<VT*>(M)[q] = m;
            reinterpret_cast<VT*>(Vv)[q] = v;
        } else {
            for (size_t i = i0; i < i0 + kAdamVec && i < total; ++i) {
                const int te = adam_tensor(A, i);
                if (!((A.active >> te) & 1u)) continue;
                adam_elem(A, te, lrd, P[i], G[i], M[i], Vv[i]);
            }
        }
    }
}

int g_sms = 0;
uint32_t sms() {
    if (!g_sms) {
        int dev = 0;
        SVLF_CUDA(cudaGetDevice(&dev));
        SVLF_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return uint32_t(g_sms);
}

// grid of a loop over `items` work items of `per_block` each: no more blocks
// than the items need, at most `per_sm` blocks per SM
unsigned loop_grid(size_t items, size_t per_block, uint32_t per_sm) {
    const size_t need = std::max<size_t>(1, (items + per_block - 1) / per_block);
    return unsigned(std::min<size_t>(need, size_t(sms()) * per_sm));
}

}  // namespace

TrainScratch::~TrainScratch() {
    if (graph) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph));
    if (h_mail) cudaFreeHost(h_mail);
    if (h_plan) cudaFreeHost(h_plan);
    if (h_stage) cudaFreeHost(h_stage);
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
}

namespace {

// The Adam plan of a step (per-tensor bias corrections from the step counters,
// hyperparameters, lr), ModelAdam order = flat buffer order.
AdamPlan adam_plan(const TrainModelRefs& M, bool color_frozen, float lr) {
    using D = DecOffsets;
    AdamPlan A{};
    const size_t sizes[14] = {M.n_ft,      M.n_fc,      size_t(kHid) * kInT, kHid, 2 * kHid, 2,
                              size_t(kHid) * kInC, kHid, size_t(kHid) * kHid, kHid, size_t(kHid) * kHid, kHid,
                              3 * kHid,    3};
    static_assert(D::T_SIZE == kHid * kInT + kHid + 2 * kHid + 2, "f_T layout");
    size_t end = 0;
    for (int t = 0; t < 14; ++t) {
        end += sizes[t];
        A.end[t] = end;
        const AdamHyper& h = M.hyper[t];
        const uint64_t step = M.steps[t] + 1;  // the caller advances the counters when the update ran
        A.corr1[t] = 1.0 - std::pow(double(h.beta1), double(step));
        A.corr2[t] = 1.0 - std::pow(double(h.beta2), double(step));
        A.beta1[t] = h.beta1;
        A.beta2[t] = h.beta2;
        A.eps[t] = h.eps;
        if (!color_frozen || !(t == 1 || t >= 6)) A.active |= 1u << t;
    }
    A.lr = lr;
    return A;
}

void enqueue_adam(const TrainModelRefs& M, const AdamPlan* d_plan, size_t total, const uint32_t* skip_if,
                  const int* err, cudaStream_t s) {
    const size_t groups = (total + kAdamVec - 1) / kAdamVec;
    const unsigned grid = unsigned(std::min<size_t>((groups + 255) / 256, size_t(sms()) * SVLF_ADAM_MINB));
    k_adam<<<grid, 256, 0, s>>>(M.params, M.grads, M.adam_m, M.adam_v, total, d_plan, skip_if, err);
    note_launch();
}

}  // namespace

void launch_adam(const TrainModelRefs& M, bool color_frozen, float lr, const uint32_t* skip_if, const int* err,
                 cudaStream_t s) {
    const AdamPlan A = adam_plan(M, color_frozen, lr);
    AdamPlan* d = nullptr;
    SVLF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(AdamPlan), s));
    SVLF_CUDA(cudaMemcpyAsync(d, &A, sizeof A, cudaMemcpyHostToDevice, s));
    enqueue_adam(M, d, A.end[13], skip_if, err, s);
    SVLF_CUDA(cudaFreeAsync(d, s));
    SVLF_CUDA(cudaStreamSynchronize(s));  // the host plan is a stack object
}

namespace {

// Graph key of a step: every pointer, size and flag its launches bake in.
struct KeyBuilder {
    std::vector<uint64_t> v;
    template <typename X>
    void add(const X& x) {
        uint64_t w[(sizeof(X) + 7) / 8] = {};
        std::memcpy(w, &x, sizeof(X));
        v.insert(v.end(), w, w + (sizeof(X) + 7) / 8);
    }
};

}  // namespace

TrainResult run_train_step(TrainScratch& S, const DevOctree& T, const TrainModelRefs& M, const TrainBatchDev& b,
                           const TrainOptions& o, cudaStream_t s, int* err_flag) {
    using D = DecOffsets;
    TrainResult res;
    if (!S.h_mail) {
        SVLF_CUDA(cudaMallocHost(&S.h_mail, sizeof(StepMail)));
        SVLF_CUDA(cudaMallocHost(&S.h_plan, sizeof(AdamPlan)));
        for (auto& e : S.ev) SVLF_CUDA(cudaEventCreate(&e));
    }
    const size_t P = M.n_ft + M.n_fc + SVLF_DEC_T_SIZE + SVLF_DEC_C_SIZE;
    const uint32_t n = b.n;
    // Per-active-hit buffers (the feature-major matrices: ~5.3 KB per hit) are
    // sized from the previous step's active count with headroom, not from the
    // traversal's hit capacity: tighter rows (row stride ld) and bounded
    // memory. A step whose active hits exceed it is flagged and re-run.
    if (S.act_cap == 0) S.act_cap = std::max<uint32_t>(65536, n);
    const uint32_t cap = std::min<uint32_t>(std::max<uint32_t>(b.hit_cap, 32), S.act_cap);
    const uint32_t ld = (cap + 31u) & ~31u;
    const bool dp = o.coll && o.coll->world > 1;
    const uint32_t V = M.view.V;

    // ---- every buffer of the step, allocated before anything is enqueued (the
    // enqueue below must not reallocate: it may be captured into a graph)
    uint32_t* act_first = S.act_first.ensure<uint32_t>(n + 1);
    uint32_t* act_cnt = S.act_cnt.ensure<uint32_t>(n + 1);
    uint32_t* dpos = S.dpos.ensure<uint32_t>(n + 1);
    int* surf_rel = S.surf_rel.ensure<int>(n + 1);
    double* eta_gt = S.eta_gt.ensure<double>(n + 1);
    double* ray_loss = S.ray_loss.ensure<double>(n + 1);
    unsigned long long* counters = S.counters.ensure<unsigned long long>(4);
    double* red = S.red.ensure<double>(R_COUNT);
    uint32_t* status = S.status.ensure<uint32_t>(4);
    StepMail* mail = reinterpret_cast<StepMail*>(S.loss_out.ensure<char>(sizeof(StepMail)));
    AdamPlan* d_plan = S.plan.ensure<AdamPlan>(1);
    uint32_t* dhit = S.dhit.ensure<uint32_t>(cap);
    uint32_t* dray = S.dray.ensure<uint32_t>(cap);
    float* hitf = S.hitf.ensure<float>(size_t(ld) * 8);    // tau, eta, rgb[3], drgb[3]
    double* hitd = S.hitd.ensure<double>(size_t(ld) * 5);  // dtau, deta, e, T, w
    float* acts = S.acts.ensure<float>(size_t(A_ROWS) * ld);
    float* deltas = S.deltas.ensure<float>(size_t(D_ROWS) * ld);
    float* dxs = S.dxs.ensure<float>(size_t(kInT) * ld);  // dL/d layer-0 inputs
    X3ImageJobs jobs{};
    enum { J_FT0, J_FC0, J_FC1, J_FC2, J_BC2, J_BC1, J_BC0, J_BT0 };
    jobs.job[J_FT0] = {M.view.mt + D::T_W0, kHid, kInT, 0, 0};
    jobs.job[J_FC0] = {M.view.mc + D::C_W0, kHid, kInC, 0, 0};
    jobs.job[J_FC1] = {M.view.mc + D::C_W1, kHid, kHid, 0, 0};
    jobs.job[J_FC2] = {M.view.mc + D::C_W2, kHid, kHid, 0, 0};
    jobs.job[J_BC2] = {M.view.mc + D::C_W2, kHid, kHid, 0, 1};
    jobs.job[J_BC1] = {M.view.mc + D::C_W1, kHid, kHid, 0, 1};
    jobs.job[J_BC0] = {M.view.mc + D::C_W0, kHid, kInC, 6, 1};
    jobs.job[J_BT0] = {M.view.mt + D::T_W0, kHid, kInT, 6, 1};
    jobs.count = 8;
    size_t img_bytes = 0;
    for (int i = 0; i < jobs.count; ++i)
        img_bytes += gemm_x3_image_bytes(jobs.job[i].bwd ? jobs.job[i].O : jobs.job[i].K);
    uint8_t* wimg = S.wimg.ensure<uint8_t>(img_bytes);
    const size_t gemm_part = gemm_x3_dw_partial_floats(kHid, kInT) + gemm_x3_dw_partial_floats(kHid, kInC) +
                             2 * gemm_x3_dw_partial_floats(kHid, kHid);
    float* part = S.dw_part.ensure<float>(gemm_part + size_t(sms()) * (4 * kHcPartial + 8 * kHtPartial));
    float* head_part = part + gemm_part;                    // k_bwd_head_c's block partials (<= 4 blocks per SM)
    float* ht_part = head_part + size_t(sms()) * 4 * kHcPartial;  // k_bwd_feat_c's (<= 8 blocks per SM)
    size_t tb_scan = 0, tb_red = 0, tb_sel = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb_scan, act_cnt, dpos, int(n + 1));
    cub::DeviceReduce::Sum(nullptr, tb_red, ray_loss, red + R_LOSS, int(std::max<uint32_t>(n, 1)));
    uint8_t* touched = nullptr;
    uint32_t *rows = nullptr, *n_rows = nullptr;
    float* packed = nullptr;
    uint32_t rc = 0;
    if (dp) {
        touched = S.touched.ensure<uint8_t>(V);
        rows = S.rows.ensure<uint32_t>(V);
        n_rows = S.n_rows.ensure<uint32_t>(1);
        cub::CountingInputIterator<uint32_t> idx(0);
        cub::DeviceSelect::Flagged(nullptr, tb_sel, idx, touched, rows, n_rows, int(V));
        if (S.rows_cap == 0) S.rows_cap = std::min<uint32_t>(V, 1u << 16);
        rc = std::min<uint32_t>(S.rows_cap, V);
        packed = S.packed.ensure<float>(size_t(rc) * 96);
    }
    char* scan_tmp = S.scan_tmp.ensure<char>(std::max({tb_scan, tb_red, tb_sel, size_t(16)}));
    const uint32_t* n_act = dpos + n;  // active hits, on the device
    HitArgs H{b.rays,   b.hit_leaf, b.hit_tin, b.hit_tout, dhit,   dray,  dpos, surf_rel, n_act, cap, ld, o.surface,
              acts,     deltas,     hitf,      hitf + ld,  hitf + 2 * size_t(ld), hitf + 5 * size_t(ld), hitd,
              hitd + ld};
    PrepArgs pa{b.rays,   b.depth_gt, b.alpha_gt, n,         b.ray_off, b.ray_cnt, b.hit_leaf, b.hit_tin,
                b.hit_tout, b.trav_counters, o.surface, o.lw.empty == 0.0, act_first, act_cnt, surf_rel, eta_gt,
                counters};
    LossArgs L{b.c_gt, b.alpha_gt, dpos, act_cnt, surf_rel, eta_gt, n, o.surface, o.lw, ray_loss,
               hitd + 2 * size_t(ld), hitd + 3 * size_t(ld), hitd + 4 * size_t(ld)};
    float* g_ft = M.grads;
    float* g_fc = M.grads + M.n_ft;
    float* g_mt = g_fc + M.n_fc;
    float* g_mc = g_mt + SVLF_DEC_T_SIZE;
    const unsigned in_grid = loop_grid(cap, 32 * kInWarps, 16);
    const unsigned hit_grid = loop_grid(cap, 128, 16);
    const unsigned hc_grid = loop_grid(cap, kHcThreads, 4);
    const unsigned sc_grid = loop_grid(cap, 32 * kScWarps, 8);
    auto A = [&](int row) { return acts + size_t(row) * ld; };
    auto Dm = [&](int row) { return deltas + size_t(row) * ld; };
    const int prod = o.tf32 ? 1 : 3;
    const uint32_t* n_rows_dev = dp ? n_rows : nullptr;
    bool capturing = false;  // inside a graph capture the timing events become event-record nodes
    auto ev = [&](int k) {
        if (capturing) SVLF_CUDA(cudaEventRecordWithFlags(S.ev[k], s, cudaEventRecordExternal));
        else SVLF_CUDA(cudaEventRecord(S.ev[k], s));
    };

    // ---- the step, enqueued without a host round trip
    auto enqueue = [&]() {
        long long launches = 0;
        if (b.pre) (*b.pre)(capturing);
        ev(0);
        SVLF_CUDA(cudaMemsetAsync(M.grads, 0, P * 4, s));
        SVLF_CUDA(cudaMemsetAsync(counters, 0, 32, s));
        SVLF_CUDA(cudaMemsetAsync(status, 0, 16, s));
        SVLF_CUDA(cudaMemsetAsync(act_cnt + n, 0, 4, s));
        // per-ray preparation and the dense active-hit list
        if (n) {
            k_prep<<<(n + 127) / 128, 128, 0, s>>>(T, pa, err_flag);
            ++launches;
        }
        SVLF_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, tb_scan, act_cnt, dpos, int(n + 1), s));
        ++launches;
        if (n) {
            k_expand<<<(n + 127) / 128, 128, 0, s>>>(n, act_first, act_cnt, dpos, H, dhit, dray);
            ++launches;
        }
        // weight operand images of every forward / input-gradient GEMM (one launch)
        gemm_x3_build_images(jobs, wimg, s);
        auto img = [&](int i) { return wimg + jobs.offset[i]; };
        ev(1);
        // forward
        k_fwd_in_t<<<in_grid, 32 * kInWarps, 0, s>>>(T, M.view, H, err_flag);
        const X3Head head_t{M.view.mt + D::T_W1, 2, A(A_YT)}, head_c{M.view.mc + D::C_W3, 3, A(A_YC)};
        gemm_x3_fwd(A(A_XT), img(J_FT0), M.view.mt + D::T_B0, A(A_HT), kHid, kInT, n_act, cap, ld, s, &head_t);
        k_fwd_mid<<<in_grid, 32 * kInWarps, 0, s>>>(T, M.view, H, err_flag);
        gemm_x3_fwd(A(A_XC), img(J_FC0), M.view.mc + D::C_B0, A(A_H1), kHid, kInC, n_act, cap, ld, s);
        gemm_x3_fwd(A(A_H1), img(J_FC1), M.view.mc + D::C_B1, A(A_H2), kHid, kHid, n_act, cap, ld, s);
        gemm_x3_fwd(A(A_H2), img(J_FC2), M.view.mc + D::C_B2, A(A_H3), kHid, kHid, n_act, cap, ld, s, &head_c);
        k_fwd_rgb<<<hit_grid, 128, 0, s>>>(M.view, H);
        launches += 3;
        ev(2);
        if (n) {
            k_loss<<<(n + 127) / 128, 128, 0, s>>>(L, H);
            ++launches;
        }
        ev(3);
        // backward. f_C: head -> D_C2; D_C1 = relu'(h2) W2^T D_C2; D_C0 = relu'(h1) W1^T D_C1; dX_C = W0^T D_C0
        k_bwd_head_c<<<hc_grid, kHcThreads, 0, s>>>(M.view, H, head_part);
        gemm_x3_bwd(Dm(D_C2), img(J_BC2), kHid, kHid, 0, Dm(D_C1), A(A_H2), n_act, cap, ld, s);
        gemm_x3_bwd(Dm(D_C1), img(J_BC1), kHid, kHid, 0, Dm(D_C0), A(A_H1), n_act, cap, ld, s);
        gemm_x3_bwd(Dm(D_C0), img(J_BC0), kHid, kInC, 6, dxs + 6 * size_t(ld), nullptr, n_act, cap, ld, s);
        // colour-feature scatter, positional Jacobian, f_T heads -> D_T0
        k_bwd_feat_c<<<sc_grid, 32 * kScWarps, 0, s>>>(T, M.view, H, dxs, o.color_frozen, g_fc, err_flag, ht_part);
        gemm_x3_bwd(Dm(D_T0), img(J_BT0), kHid, kInT, 6, dxs + 6 * size_t(ld), nullptr, n_act, cap, ld, s);
        k_bwd_feat_t<<<sc_grid, 32 * kScWarps, 0, s>>>(T, H, dxs, g_ft, err_flag);
        launches += 3;
        // weight gradients (sums over hits, CTA-ordered partials, one reduction launch)
        {
            X3DwJob dw[kX3MaxDwJobs];
            int nj = 0;
            dw[nj++] = {Dm(D_T0), A(A_XT), kHid, kInT, g_mt + D::T_W0, g_mt + D::T_B0};
            dw[nj++] = {nullptr, nullptr, 2, kHid, g_mt + D::T_W1, g_mt + D::T_B1, ht_part, sc_grid};
            if (!o.color_frozen) {
                dw[nj++] = {Dm(D_C0), A(A_XC), kHid, kInC, g_mc + D::C_W0, g_mc + D::C_B0};
                dw[nj++] = {Dm(D_C1), A(A_H1), kHid, kHid, g_mc + D::C_W1, g_mc + D::C_B1};
                dw[nj++] = {Dm(D_C2), A(A_H2), kHid, kHid, g_mc + D::C_W2, g_mc + D::C_B2};
                dw[nj++] = {nullptr, nullptr, 3, kHid, g_mc + D::C_W3, g_mc + D::C_B3, head_part, hc_grid};
            }
            gemm_x3_dw_batch(dw, nj, n_act, cap, ld, part, prod, s);
        }
        if (n) {
            SVLF_CUDA(cub::DeviceReduce::Sum(scan_tmp, tb_red, ray_loss, red + R_LOSS, int(n), s));
        } else {
            SVLF_CUDA(cudaMemsetAsync(red + R_LOSS, 0, 8, s));
        }
        k_step_scalars<<<1, 1, 0, s>>>(n, counters, b.trav_counters, n_act, cap, err_flag, red);
        launches += 2;
        // data parallel: all-reduce the scalars, the decoder gradients and the union of touched feature rows
        if (dp) {
            Collective& C = *o.coll;
            C.allreduce(red, R_COUNT, CollType::F64, CollOp::Sum, s);
            C.allreduce(g_mt, SVLF_DEC_T_SIZE + SVLF_DEC_C_SIZE, CollType::F32, CollOp::Sum, s);
            SVLF_CUDA(cudaMemsetAsync(touched, 0, V, s));
            k_touched<<<loop_grid(cap, 256, 8), 256, 0, s>>>(T, b.hit_leaf, dhit, n_act, cap, touched);
            C.allreduce(touched, V, CollType::U8, CollOp::Max, s);
            cub::CountingInputIterator<uint32_t> idx(0);
            SVLF_CUDA(cub::DeviceSelect::Flagged(scan_tmp, tb_sel, idx, touched, rows, n_rows, int(V), s));
            k_pack_rows<<<loop_grid(rc, 8, 8), 256, 0, s>>>(rows, n_rows, rc, g_ft, g_fc, packed, false, status);
            C.allreduce(packed, size_t(rc) * 96, CollType::F32, CollOp::Sum, s);
            k_pack_rows<<<loop_grid(rc, 8, 8), 256, 0, s>>>(rows, n_rows, rc, g_ft, g_fc, packed, true, status);
            launches += 4;
        }
        k_step_status<<<1, 1, 0, s>>>(red, status);
        ++launches;
        ev(4);
        // Adam (adam_model_step, src/train.cpp:345-360), skipped on the device when the step is flagged
        if (o.adam) {
            enqueue_adam(M, d_plan, P, status, nullptr, s);
            ++launches;
        }
        ev(5);
        k_step_mail<<<1, 1, 0, s>>>(red, status, err_flag, b.trav_counters, n_act, cap, n_rows_dev, mail);
        ++launches;
        SVLF_CUDA(cudaMemcpyAsync(S.h_mail, mail, sizeof(StepMail), cudaMemcpyDeviceToHost, s));
        return launches;
    };

    // The step's Adam plan (bias corrections change every step) goes to the
    // device ahead of the step, outside any graph.
    if (o.adam) {
        *static_cast<AdamPlan*>(S.h_plan) = adam_plan(M, o.color_frozen, o.lr);
        SVLF_CUDA(cudaMemcpyAsync(d_plan, S.h_plan, sizeof(AdamPlan), cudaMemcpyHostToDevice, s));
    }
    // CUDA graph: the step is captured once and replayed while nothing it bakes
    // in changes (pointers, sizes, modes, loss weights); not with a host-staged
    // exchange (it synchronizes inside the step) or $SVLF_TRAIN_GRAPHS=0.
    static const bool graphs_env = [] {
        const char* e = std::getenv("SVLF_TRAIN_GRAPHS");
        return !(e && e[0] == '0');
    }();
    const bool use_graph = graphs_env && !dp;
    long long launches = 0;
    if (use_graph) {
        KeyBuilder k;
        k.add(T);
        k.add(M.view);
        k.add(M.params);
        k.add(M.grads);
        k.add(M.adam_m);
        k.add(M.adam_v);
        k.add(M.n_ft);
        k.add(M.n_fc);
        {
            TrainBatchDev kb = b;  // the pre-work is keyed by its own key, not by the functor's address
            kb.pre = nullptr;
            kb.pre_key = nullptr;
            k.add(kb);
        }
        k.add(o.surface);
        k.add(o.color_frozen);
        k.add(o.adam);
        k.add(o.tf32);
        k.add(o.lw);
        k.add(s);
        k.add(err_flag);
        k.add(cap);
        k.add(ld);
        const DevBuf* bufs[] = {&S.act_first, &S.act_cnt, &S.dpos,    &S.surf_rel, &S.eta_gt, &S.ray_loss,
                                &S.counters,  &S.red,     &S.status,  &S.loss_out, &S.plan,   &S.dhit,
                                &S.dray,      &S.hitf,    &S.hitd,    &S.acts,     &S.deltas, &S.dxs,
                                &S.wimg,      &S.dw_part, &S.scan_tmp};
        for (const DevBuf* d : bufs) k.add(d->p);
        k.add(S.h_mail);
        if (b.pre_key) k.v.insert(k.v.end(), b.pre_key->begin(), b.pre_key->end());
        // Replay when the key matches the captured graph; capture when the same key
        // came twice in a row (a steady workload); otherwise run eagerly (a batch
        // whose size changes every step, e.g. stage 1's foreground rays, would
        // pay a capture per step).
        const bool replay = S.graph && k.v == S.graph_key;
        const bool capture = !replay && k.v == S.last_key;
        if (capture) {
            if (S.graph) SVLF_CUDA(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(S.graph)));
            S.graph = nullptr;
            S.graph_key.clear();
            cudaGraph_t g = nullptr;
            SVLF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            capturing = true;
            try {
                launches = enqueue();
            } catch (...) {
                capturing = false;
                cudaStreamEndCapture(s, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            capturing = false;
            SVLF_CUDA(cudaStreamEndCapture(s, &g));
            cudaGraphExec_t ge = nullptr;
            SVLF_CUDA(cudaGraphInstantiate(&ge, g, 0));
            SVLF_CUDA(cudaGraphDestroy(g));
            S.graph = ge;
            S.graph_key = k.v;
            S.graph_launches = launches;
            ++S.graph_captures;
        }
        S.last_key = std::move(k.v);
        if (replay || capture) {
            SVLF_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(S.graph), s));
            ++S.graph_replays;
            note_launch(S.graph_launches);
        } else {
            note_launch(enqueue());
        }
    } else {
        note_launch(enqueue());
    }
    SVLF_CUDA(cudaStreamSynchronize(s));
    StepMail hm;
    std::memcpy(&hm, S.h_mail, sizeof hm);
    res.loss = hm.loss;
    res.skipped = (long long)hm.skipped;
    res.eta_skipped = (long long)hm.eta_skipped;
    res.rays = (long long)hm.rays;
    res.error = int(hm.err);
    if (!res.error && (hm.flags & kStepDeviceError)) res.error = -1;  // raised on another rank
    res.flags = hm.flags & (kStepHitOverflow | kStepRowOverflow);
    res.hits = hm.hits;
    res.active = hm.active;
    // activation capacity for the next step: grow with 25 % headroom on overflow, shrink when a
    // quarter of it is used
    if (hm.active > cap || hm.active < S.act_cap / 4) S.act_cap = std::max<uint32_t>(4096, hm.active + hm.active / 4);
    res.touched_rows = hm.rows;
    res.updated = o.adam && hm.flags == 0 && hm.err == 0;
    if (hm.err) SVLF_CUDA(cudaMemsetAsync(err_flag, 0, 4, s));
    if (dp) {  // next step's exchange buffer: 25 % headroom over this step's touched rows
        const uint32_t want = std::max<uint32_t>(4096, hm.rows + hm.rows / 4);
        if ((hm.flags & kStepRowOverflow) || want < S.rows_cap / 2 || want > S.rows_cap) S.rows_cap = want;
    }
    float t[5] = {};
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], S.ev[i], S.ev[i + 1]);
    res.timings = svlf_timings{t[0], 0.f, t[1], t[2], t[3], t[4], t[0] + t[1] + t[2] + t[3] + t[4],
                               (long long)hm.active, 0, 0};
    return res;
}

}  // namespace svlfb
