// C ABI: error plumbing, device queries and the device-pointer GEMM / conv entries.
#include "capi_common.hpp"
#include "gemm.hpp"

#include <cuda_runtime.h>

namespace pp {
thread_local std::string g_last_error;
}

extern "C" {

PP_API const char* pp_last_error(void) { return pp::g_last_error.c_str(); }

PP_API int pp_version(void) { return 1; }

PP_API int pp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int good = 0;
    for (int d = 0; d < n; ++d) {
        int major = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
        if (major == 10) ++good;
    }
    return good;
}

PP_API int pp_dev_gemm(int dtype, const void* A, int M, int K, long long lda, const void* B, int N,
                       long long ldb, const float* bias, void* D, long long ldd, int out_f32,
                       int force_splits, int force_block_n, void* stream) {
    return pp::guard([&] {
        pp::require_device();
        const pp::Elem e = pp::elem_of(dtype);
        pp::EpilogueSpec ep;
        ep.out = D;
        ep.out_ld = ldd;
        ep.n_valid = N;
        ep.out_f32 = out_f32 != 0;
        ep.bias = bias;
        pp::GemmPlan plan;
        const size_t ws_bytes = size_t(16) * M * ((N + 15) / 16 * 16) * sizeof(float);
        pp::DeviceScratch ws(ws_bytes), tk(size_t(1) << 20);
        CUDA_CHECK(cudaMemset(tk.ptr, 0, size_t(1) << 20));
        pp::GemmScratch sc;
        sc.ws = static_cast<float*>(ws.ptr);
        sc.ws_bytes = ws_bytes;
        sc.tickets = static_cast<unsigned int*>(tk.ptr);
        sc.n_tickets = (size_t(1) << 20) / 4;
        pp::plan_gemm(plan, e, A, M, K, lda, B, N, ldb, ep, sc, pp::device_sm_count(), force_splits,
                      force_block_n);
        pp::launch_gemm(plan, static_cast<cudaStream_t>(stream));
        CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    });
}

PP_API int pp_dev_conv(int dtype, const void* in, int rows, int W, int C_in_pad, int stride,
                       const void* weights, int n_pad, int c_out, const float* bias, void* D,
                       long long ldd, int out_f32, const void* residual, long long res_ld,
                       int force_splits, int force_block_n, void* stream) {
    return pp::guard([&] {
        pp::require_device();
        const pp::Elem e = pp::elem_of(dtype);
        pp::EpilogueSpec ep;
        ep.out = D;
        ep.out_ld = ldd;
        ep.n_valid = c_out;
        ep.out_f32 = out_f32 != 0;
        ep.bias = bias;
        ep.residual = residual;
        ep.res_ld = res_ld;
        pp::GemmPlan plan;
        const long long m_pix = (long long)(stride == 1 ? rows : rows / 2) * (stride == 1 ? W : W / 2);
        const size_t ws_bytes = size_t(16) * m_pix * n_pad * sizeof(float);
        pp::DeviceScratch ws(ws_bytes), tk(size_t(1) << 20);
        CUDA_CHECK(cudaMemset(tk.ptr, 0, size_t(1) << 20));
        pp::GemmScratch sc;
        sc.ws = static_cast<float*>(ws.ptr);
        sc.ws_bytes = ws_bytes;
        sc.tickets = static_cast<unsigned int*>(tk.ptr);
        sc.n_tickets = (size_t(1) << 20) / 4;
        pp::plan_conv(plan, e, in, rows, W, C_in_pad, stride, weights, n_pad, ep, sc,
                      pp::device_sm_count(), force_splits, force_block_n);
        pp::launch_gemm(plan, static_cast<cudaStream_t>(stream));
        CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    });
}

}  // extern "C"
