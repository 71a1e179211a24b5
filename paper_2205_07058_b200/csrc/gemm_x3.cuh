// 3xTF32 tensor-core GEMMs of the train step's dense layers (gemm_x3.cu).
// Matrices are feature-major (row = one feature over all hits, row stride ld,
// 16-byte aligned rows); weights are the reference's row-major [O][K].
// Hit counts are read on the device (n_dev, clamped to cap), so a train step
// enqueues every GEMM without a host round trip.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace svlfb {

// One weight operand image: B[j][k] = W[j][k] (forward, j < O, k < K) or
// B[j][k] = W[k][k0 + j] (input gradient, j < K - k0, k < O), split into TF32
// hi / lo parts in the kernels' shared-memory layout, 128 rows x 32-K chunks.
struct X3ImageJob {
    const float* W;
    uint32_t O, K, k0;
    uint32_t bwd;
};
constexpr int kX3MaxJobs = 8;
struct X3ImageJobs {
    X3ImageJob job[kX3MaxJobs];
    uint32_t offset[kX3MaxJobs];  // byte offset of each image in the buffer
    int count;
};
// bytes of one image with reduction length kred
size_t gemm_x3_image_bytes(uint32_t kred);
// builds every image of `jobs` (offsets filled in here) into buf with one launch
void gemm_x3_build_images(X3ImageJobs& jobs, uint8_t* buf, cudaStream_t s);

// y[j][:] = relu(sum_k W[j][k] x[k][:] + bias[j]), j < O, k < K; img from a forward job
// Optional head epilogue of a forward GEMM with O = 128: the partial products of
// a following 128 -> c layer (c <= 3, weights w row-major c x 128) over each
// 32-row quarter q of y, written to out rows q * c + (0..c-1) (stride ld); the
// consumer adds the bias and the four quarters in order.
struct X3Head {
    const float* w;
    uint32_t c;
    float* out;
};
void gemm_x3_fwd(const float* x, const uint8_t* img, const float* bias, float* y, uint32_t O, uint32_t K,
                 const uint32_t* n_dev, uint32_t cap, uint32_t ld, cudaStream_t s, const X3Head* head = nullptr);
// dx[j][:] = sum_o W[o][k0 + j] d[o][:], j < K - k0; zeroed where mask[j][:] <= 0 (mask may be
// null); img from a backward job
void gemm_x3_bwd(const float* d, const uint8_t* img, uint32_t O, uint32_t K, uint32_t k0, float* dx,
                 const float* mask, const uint32_t* n_dev, uint32_t cap, uint32_t ld, cudaStream_t s);
// dW[o][k] = sum_n d[o][n] x[k][n], db[o] = sum_n d[o][n] (overwritten). Each CTA reduces a
// contiguous hit range into its own partial (part: gemm_x3_dw_partial_floats floats) and the
// partials are summed in CTA order, so the result is bitwise reproducible. products = 3
// (hi*lo + lo*hi + hi*hi: fp32-level accuracy) or 1 (plain TF32).
size_t gemm_x3_dw_partial_floats(uint32_t O, uint32_t K);
// Several weight gradients at once: one GEMM launch per job, then one launch
// reducing every job's partials (part holds the jobs' partials back to back:
// sum of gemm_x3_dw_partial_floats over the jobs).
struct X3DwJob {
    const float* d;
    const float* x;
    uint32_t O, K;
    float* dW;
    float* db;
    // partials already produced by another kernel (ext_ctas of O x (K + 1)
    // floats, CTA-major): no GEMM, only the fixed-order reduction
    const float* ext_part = nullptr;
    uint32_t ext_ctas = 0;
};
constexpr int kX3MaxDwJobs = 6;
void gemm_x3_dw_batch(const X3DwJob* jobs, int count, const uint32_t* n_dev, uint32_t cap, uint32_t ld, float* part,
                      int products, cudaStream_t s);
void gemm_x3_dw(const float* d, const float* x, uint32_t O, uint32_t K, float* dW, float* db, const uint32_t* n_dev,
                uint32_t cap, uint32_t ld, float* part, int products, cudaStream_t s);

}  // namespace svlfb
