// NCCL entry points resolved at run time (dlopen), so loading this library
// never pins an NCCL build into the process: when PyTorch (or another host
// framework) has already loaded its libnccl.so.2, dlopen returns that same
// library and both share it. $SVLF_NCCL_LIB overrides the soname.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "common.hpp"

namespace svlfb {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        const char* name = std::getenv("SVLF_NCCL_LIB");
        void* h = dlopen(name ? name : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load NCCL: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* s) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, s));
            if (!fn) err = std::string("NCCL symbol missing: ") + s;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.AllReduce, "ncclAllReduce");
        sym(api.GetErrorString, "ncclGetErrorString");
    });
    if (!err.empty()) fail(SVLF_ERR_CUDA, err);
    return api;
}

inline void nccl_check(ncclResult_t r) {
    if (r != ncclSuccess) fail(SVLF_ERR_CUDA, std::string("NCCL: ") + nccl_api().GetErrorString(r));
}

}  // namespace svlfb
