// Shared helpers for the extern "C" layer: exception -> status code mapping
// (reference semantics: std::invalid_argument -> PP_EINVAL, std::runtime_error ->
// PP_ERUNTIME; proj/src/cli.cpp:145-154) and small RAII device buffers.
#pragma once
#include "pp_b200.h"
#include "gemm.hpp"
#include "util.hpp"

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace pp {

extern thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_last_error.clear();
        return PP_OK;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return PP_EINVAL;
    } catch (const NcclError& e) {
        g_last_error = e.what();
        return PP_ENCCL;
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return PP_ECUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return PP_ERUNTIME;
    }
}

inline Elem elem_of(int dtype) {
    if (dtype == PP_DTYPE_BF16) return Elem::BF16;
    if (dtype == PP_DTYPE_FP32) return Elem::F32;
    throw std::invalid_argument("unknown dtype " + std::to_string(dtype));
}

// Fails loudly when no sm_100 device is present: there is no CPU fallback.
inline void require_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw CudaError("no CUDA device available: the B200 kernels cannot run (no CPU fallback)");
    }
    int dev = 0, major = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) throw CudaError("device is not sm_100 (Blackwell B200)");
}

struct DeviceScratch {
    void* ptr = nullptr;
    explicit DeviceScratch(size_t bytes) {
        if (bytes) CUDA_CHECK(cudaMalloc(&ptr, bytes));
    }
    ~DeviceScratch() {
        if (ptr) cudaFree(ptr);
    }
    DeviceScratch(const DeviceScratch&) = delete;
    DeviceScratch& operator=(const DeviceScratch&) = delete;
};

}  // namespace pp
