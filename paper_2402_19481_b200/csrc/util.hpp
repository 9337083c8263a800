// Error types shared by the runtime and the C ABI.
//   std::invalid_argument -> PP_EINVAL   (reference: std::invalid_argument, CLI exit 2)
//   std::runtime_error    -> PP_ERUNTIME (reference: std::runtime_error,   CLI exit 1)
//   pp::CudaError         -> PP_ECUDA
//   pp::NcclError         -> PP_ENCCL
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace pp {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

[[noreturn]] inline void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    throw CudaError(std::string("CUDA error '") + cudaGetErrorString(e) + "' at " + file + ":" +
                    std::to_string(line) + " (" + what + ")");
}

}  // namespace pp

#define CUDA_CHECK(x)                                                 \
    do {                                                              \
        cudaError_t e_ = (x);                                         \
        if (e_ != cudaSuccess) ::pp::cuda_fail(e_, #x, __FILE__, __LINE__); \
    } while (0)
