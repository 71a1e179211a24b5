// Kernel launch interface between the C ABI (capi.cu) and the kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "common.hpp"
#include "composite.cuh"
#include "geom.cuh"

namespace svlfb {

// Process-wide count of this library's kernel launches (svlf_ctx_kernel_launches).
extern std::atomic<long long> g_kernel_launches;
inline void note_launch(long long n = 1) { g_kernel_launches.fetch_add(n, std::memory_order_relaxed); }

constexpr int kFt = 64;       // thickness feature dim
constexpr int kFc = 32;       // color feature dim
constexpr int kHid = 128;     // hidden width
constexpr int kInT = 6 + 2 * kFt;  // 134
constexpr int kInC = 6 + kFc;      // 38

// Flat decoder offsets (W_l row-major [out][in], then b_l), mlp.hpp:50-53.
struct DecOffsets {
    // f_T
    static constexpr int T_W0 = 0, T_B0 = T_W0 + kHid * kInT, T_W1 = T_B0 + kHid, T_B1 = T_W1 + 2 * kHid,
                         T_SIZE = T_B1 + 2;
    // f_C
    static constexpr int C_W0 = 0, C_B0 = C_W0 + kHid * kInC, C_W1 = C_B0 + kHid,
                         C_B1 = C_W1 + kHid * kHid, C_W2 = C_B1 + kHid, C_B2 = C_W2 + kHid * kHid,
                         C_W3 = C_B2 + kHid, C_B3 = C_W3 + 3 * kHid, C_SIZE = C_B3 + 3;
};
static_assert(DecOffsets::T_SIZE == SVLF_DEC_T_SIZE, "f_T size");
static_assert(DecOffsets::C_SIZE == SVLF_DEC_C_SIZE, "f_C size");

// Device view of a model's learnable tensors.
struct DevModel {
    const float* ft;  // [V][64]
    const float* fc;  // [V][32]
    const float* mt;  // f_T flat
    const float* mc;  // f_C flat
    uint32_t V;
};

// fp32 decoder pack for the CUDA-core path: hidden layers transposed to
// [in][128] so a thread streams 16 consecutive outputs per float4 x4 load.
struct DecPackF32 {
    const float* t_w0t;  // [134][128]
    const float* t_b0;   // [128]
    const float* t_w1;   // [2][128]
    const float* t_b1;   // [2]
    const float* c_w0t;  // [38][128]
    const float* c_b0;
    const float* c_w1t;  // [128][128]
    const float* c_b1;
    const float* c_w2t;
    const float* c_b2;
    const float* c_w3;   // [3][128]
    const float* c_b3;
};
constexpr size_t kPackF32Floats = size_t(kInT) * kHid + kHid + 2 * kHid + 2 + size_t(kInC) * kHid + kHid +
                                  2 * (size_t(kHid) * kHid + kHid) + 3 * kHid + 3;

// Grow-only device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* ensure(size_t n) {
        const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
        if (bytes > cap) {
            if (p) SVLF_CUDA(cudaFree(p));
            p = nullptr;
            cap = 0;
            const size_t want = bytes + bytes / 4;
            SVLF_CUDA(cudaMalloc(&p, want));
            cap = want;
        }
        return static_cast<T*>(p);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Per-hit decoder outputs consumed by composite.
struct HitOut {
    float* tau;
    float* eta;  // fp32 decoder: eta; tensor-core decoders: t_s = eta t_in + (1 - eta) t_out (fp32), which is
                 // all the 16-bit composite needs from eta (so it does not re-read t_in / t_out)
    float* rgb;  // 3 per hit
};

// ---- traversal (traverse.cu)
// Output of one traversal: each ray i owns hits [ray_off[i], ray_off[i] + ray_cnt[i])
// sorted by (t_in, leaf index); segments of different rays are placed in
// arbitrary order. counters: [0] hits allocated, [1] overflow rays (first
// pass), [2] capacity exceeded (host grows the buffers and re-runs),
// [3] overflow rays of the dense second pass.
struct TraverseOut {
    uint32_t* ray_off;
    uint32_t* ray_cnt;
    uint32_t* hit_leaf;
    double* hit_tin;
    double* hit_tout;
    uint32_t* hit_ray;
    uint32_t* counters;
    uint32_t* overflow_rays;
    uint32_t* overflow_dense;
    double* rays;  // n x 6: input rays (buffer mode) or camera rays written for foreground rays
    uint32_t capacity;
};
// count = true: the variant that also counts ray-box tests into counters[7]
void launch_traverse(const DevOctree& T, const DevCamera* cam, uint32_t row0, uint32_t rows, uint32_t n,
                     const TraverseOut& o, cudaStream_t s, bool count = false);
// second cooperative pass (16 rays per block) over the rays of overflowed tiles
void launch_traverse_dense(const DevOctree& T, const DevCamera* cam, uint32_t row0, const TraverseOut& o,
                           cudaStream_t s, bool count = false);
// per-ray depth-first walker for whatever still overflowed
void launch_traverse_fallback(const DevOctree& T, const DevCamera* cam, uint32_t row0, const TraverseOut& o,
                              cudaStream_t s);
void launch_to_csr(const uint32_t* ray_off, const uint32_t* ray_cnt, const uint32_t* csr, uint32_t n,
                   const uint32_t* leaf, const double* tin, const double* tout, uint32_t* leaf_o, double* tin_o,
                   double* tout_o, uint32_t* ray_o, cudaStream_t s);
size_t scan_temp_bytes(uint32_t n);
void launch_exclusive_scan(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out,
                           uint32_t n, cudaStream_t s);

// ---- render (render.cu)
DecPackF32 pack_f32_view(float* base);
void launch_pack_f32(const DevModel& M, float* pack, cudaStream_t s);
void launch_decode_f32(const DevOctree& T, const DevModel& M, const DecPackF32& P, const double* rays,
                       const uint32_t* hit_ray, const uint32_t* hit_leaf, const double* hit_tin,
                       const double* hit_tout, uint32_t n_hits, HitOut out, int* err, cudaStream_t s);
void launch_composite(const uint32_t* ray_off, const uint32_t* ray_cnt, const double* hit_tin,
                      const double* hit_tout, HitOut hits, uint32_t n_rays, const float* bg3, float* rgb,
                      float* alpha, float* depth, unsigned long long* fg_count, bool exact, cudaStream_t s);

// Sparse host-frame transfer: pixel blocks of 256 (kPackBlock); block j of the
// band writes its foreground mask (rays with hits, 8 words) and the base of its
// foreground pixels in tab[9j .. 9j+8], and the foreground pixels' (r, g, b,
// alpha, depth) to vals[5 (base + rank)] (base from an atomic on *count, so the
// block order in vals varies; the table makes the expansion deterministic).
// Background pixels are (bg, 0, 0) exactly and are filled on the host.
constexpr uint32_t kPackBlock = 256;
void launch_pack_fg(const uint32_t* ray_cnt, uint32_t n, const float* rgb, const float* alpha, const float* depth,
                    float* vals, uint32_t* tab, uint32_t* count, cudaStream_t s);

// ---- tcgen05 decoder (decode_tc.cu)
void ensure_pack_tc(const DevModel& M, const DevOctree& T, DevBuf& pack, uint64_t& pack_version, uint64_t version,
                    bool bf16, cudaStream_t s);
// n_dev: device-side hit count (traversal counter), clamped to cap (buffer capacity)
void launch_decode_tc(const DevOctree& T, const DevModel& M, const char* pack, bool bf16, const double* rays,
                      const uint32_t* hit_ray, const uint32_t* hit_leaf, const double* hit_tin,
                      const double* hit_tout, const uint32_t* n_dev, uint32_t cap, HitOut out, int* err,
                      void* scratch, cudaStream_t s);
size_t decode_tc_scratch_bytes(uint32_t n_hits);

// ---- misc device utilities (traverse.cu)
void launch_gather_leaf_codes(const uint64_t* leaf_codes, const uint32_t* hit_leaf, uint64_t* out,
                              size_t n, cudaStream_t s);
void launch_hit_points(const double* rays, const uint32_t* hit_ray, const double* tin,
                       const double* tout, double* x12, size_t n, cudaStream_t s);

// ---- per-point / per-ray reference operations (perray.cu)
void launch_local_coords(const DevOctree& T, const uint64_t* ids, const double* pts, size_t n, double* u, int* err,
                         cudaStream_t s);
template <typename Tv>
void launch_interpolate(const DevOctree& T, const Tv* vol, uint32_t rows, uint32_t dim, const uint64_t* ids,
                        const double* pts, size_t n, Tv* out, int* err, cudaStream_t s);
template <typename Tv>
void launch_interpolate_backward(const DevOctree& T, const Tv* vol, uint32_t rows, uint32_t dim, const uint64_t* ids,
                                 const double* pts, size_t n, const Tv* up, Tv* grad, double* jac, int* err,
                                 cudaStream_t s);
void launch_parameterize(const double* rays, const double* boxes, size_t n, double* out, int* err, cudaStream_t s);
void launch_composite_lists(const uint64_t* off, size_t lists, const double* taus, const double* colors,
                            const double* t_s, double* color, double* alpha, double* depth, double* weights, int* err,
                            cudaStream_t s);
void launch_leaf_lookup(const DevOctree& T, const uint64_t* ids, size_t n, uint32_t* leaf, uint32_t* ray, int* err,
                        cudaStream_t s);
void launch_voxel_finish(const double* rays, const double* tin, const double* tout, const float* eta, size_t n,
                         double* xs, double* ts, cudaStream_t s);
void launch_eta_gt(const double* tin, const double* tout, const double* depth, size_t n, double* out, int* err,
                   cudaStream_t s);

// scene.cu: ground truth, occupancy back-projection, metrics
void launch_render_gt(const svlf_scene_desc& d, const double* d_spheres, const double* d_boxes, const DevCamera& cam,
                      float* rgb, float* depth, float* mask, cudaStream_t s);
void launch_backproject(const DevCamera& cam, const float* depth, double* pts, size_t cap, unsigned long long* count,
                        cudaStream_t s);
double device_sq_err(const float* pred, const float* gt, size_t n, double* part, double* h_part, cudaStream_t s);
// ssim (src/metrics.cpp:70-113); tmp holds ssim_scratch_doubles(w, h) doubles
size_t ssim_scratch_doubles(uint32_t w, uint32_t h);
double device_ssim(const float* pred, const float* gt, uint32_t w, uint32_t h, uint32_t channels, double* tmp,
                   double* part, double* h_part, cudaStream_t s);
void device_depth_err(const float* pd, const float* gd, const float* gm, size_t n, double* part, double* h_part,
                      double* sum2, double* sum1, double* count, cudaStream_t s);
size_t reduction_partials();

}  // namespace svlfb
