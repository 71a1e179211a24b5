// 3xTF32 tensor-core GEMMs of the train step's dense layers (gemm_x3.cu).
// Matrices are feature-major (row = one feature over all hits, row stride ld,
// 16-byte aligned rows); weights are the reference's row-major [O][K].
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace svlfb {

// bytes of the per-call weight image for a reduction length kred
size_t gemm_x3_image_bytes(uint32_t kred);
// y[j][:] = relu(sum_k W[j][k] x[k][:] + bias[j]), j < O, k < K
void gemm_x3_fwd(const float* x, const float* W, const float* bias, float* y, uint32_t O, uint32_t K, uint32_t n,
                 uint32_t ld, uint8_t* img, cudaStream_t s);
// dx[j][:] = sum_o W[o][k0 + j] d[o][:], j < K - k0; zeroed where mask[j][:] <= 0 (mask may be null)
void gemm_x3_bwd(const float* d, const float* W, uint32_t O, uint32_t K, uint32_t k0, float* dx, const float* mask,
                 uint32_t n, uint32_t ld, uint8_t* img, cudaStream_t s);
// dW[o][k] = sum_n d[o][n] x[k][n], db[o] = sum_n d[o][n] (overwritten)
void gemm_x3_dw(const float* d, const float* x, uint32_t O, uint32_t K, float* dW, float* db, uint32_t n,
                uint32_t ld, cudaStream_t s);

}  // namespace svlfb
