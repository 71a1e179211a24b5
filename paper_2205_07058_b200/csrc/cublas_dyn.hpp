// cuBLAS (fp32 SGEMM/SGEMV, pedantic fp32 math: no TF32) resolved at run time
// like NCCL (nccl_dyn.hpp): if the host framework already loaded its
// libcublas.so.12, the same library is shared. Used only for the train step's
// plain dense-layer GEMMs; every gather, scatter, activation, loss and
// optimizer step around them is this library's own kernels.
#pragma once

#include <cublas_v2.h>
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "common.hpp"

namespace svlfb {

struct CublasApi {
    cublasStatus_t (*Create)(cublasHandle_t*) = nullptr;
    cublasStatus_t (*Destroy)(cublasHandle_t) = nullptr;
    cublasStatus_t (*SetStream)(cublasHandle_t, cudaStream_t) = nullptr;
    cublasStatus_t (*SetMathMode)(cublasHandle_t, cublasMath_t) = nullptr;
    cublasStatus_t (*Sgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const float*,
                            const float*, int, const float*, int, const float*, float*, int) = nullptr;
    cublasStatus_t (*Sgemv)(cublasHandle_t, cublasOperation_t, int, int, const float*, const float*, int,
                            const float*, int, const float*, float*, int) = nullptr;
};

inline const CublasApi& cublas_api() {
    static CublasApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        const char* name = std::getenv("SVLF_CUBLAS_LIB");
        void* h = dlopen(name ? name : "libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load cuBLAS: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* s) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, s));
            if (!fn) err = std::string("cuBLAS symbol missing: ") + s;
        };
        sym(api.Create, "cublasCreate_v2");
        sym(api.Destroy, "cublasDestroy_v2");
        sym(api.SetStream, "cublasSetStream_v2");
        sym(api.SetMathMode, "cublasSetMathMode");
        sym(api.Sgemm, "cublasSgemm_v2");
        sym(api.Sgemv, "cublasSgemv_v2");
    });
    if (!err.empty()) fail(SVLF_ERR_CUDA, err);
    return api;
}

inline void cublas_check(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS) fail(SVLF_ERR_CUDA, std::string("cuBLAS error ") + std::to_string(int(s)) + " in " + what);
}

}  // namespace svlfb
