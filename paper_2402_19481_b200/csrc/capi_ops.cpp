// C ABI: error plumbing, device queries and the device-pointer GEMM / conv entries.
#include "capi_common.hpp"
#include "gemm.hpp"
#include "pdl.cuh"

#include <cuda_runtime.h>

namespace pp {
thread_local std::string g_last_error;
}

extern "C" {

PP_API const char* pp_last_error(void) { return pp::g_last_error.c_str(); }

PP_API int pp_version(void) { return 1; }

PP_API void pp_set_pdl(int on) { pp::pdl_flag().store(on ? 1 : 0); }

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

// Micro-benchmark: plan once, launch `reps` times back to back, return mean ms per launch
// (CUDA events).  kind 0 = plain GEMM (A [M][K]), kind 1/2 = implicit conv stride 1/2 over a
// padded band [rows+2][W][K] (M = output pixels).  Buffers are allocated here (random data
// is irrelevant for timing).
PP_API int pp_dev_gemm_bench(int dtype, int kind, int M_or_rows, int W, int K, int N,
                             int force_splits, int force_block_n, int reps, double* ms_out) {
    // flags in the high bits of reps: bit 20 = fused GroupNorm statistics (32 groups),
    // bit 21 = flush L2 (256 MiB memset) before every timed launch; bits 22..29 = kernel debug
    // flags (1 no MMA, 2 no TMA, 4 no epilogue work; effective only in a -DPP_GEMM_DEBUG build)
    const bool gn = reps > 0 && (reps & (1 << 20));
    const bool flush = reps > 0 && (reps & (1 << 21));
    const int debug = reps > 0 ? (reps >> 22) & 255 : 0;
    reps &= 0xFFFFF;
    return pp::guard([&] {
        pp::require_device();
        const pp::Elem e = pp::elem_of(dtype);
        const size_t eb = pp::elem_bytes(e);
        const int n_pad = (N + 15) / 16 * 16;
        const long long m_pix = kind == 0 ? M_or_rows
                                          : (long long)(kind == 1 ? M_or_rows : M_or_rows / 2) *
                                                (kind == 1 ? W : W / 2);
        const size_t a_elems = kind == 0 ? size_t(M_or_rows) * K : size_t(M_or_rows + 2) * W * K;
        const size_t b_elems = size_t(n_pad) * K * (kind == 0 ? 1 : 9);
        pp::DeviceScratch A(a_elems * eb), B(b_elems * eb), D(size_t(m_pix) * n_pad * 2);
        CUDA_CHECK(cudaMemset(A.ptr, 0, a_elems * eb));
        CUDA_CHECK(cudaMemset(B.ptr, 0, b_elems * eb));
        const size_t ws_bytes = size_t(8) * m_pix * n_pad * sizeof(float);
        pp::DeviceScratch ws(ws_bytes), tk(size_t(1) << 20);
        CUDA_CHECK(cudaMemset(tk.ptr, 0, size_t(1) << 20));
        pp::GemmScratch sc;
        sc.ws = static_cast<float*>(ws.ptr);
        sc.ws_bytes = ws_bytes;
        sc.tickets = static_cast<unsigned int*>(tk.ptr);
        sc.n_tickets = (size_t(1) << 20) / 4;
        pp::EpilogueSpec ep;
        ep.out = D.ptr;
        ep.out_ld = n_pad;
        ep.n_valid = N;
        pp::DeviceScratch gp(size_t(1) << 22), gt(1024), go(32 * 16);
        if (gn) {
            CUDA_CHECK(cudaMemset(gt.ptr, 0, 1024));
            sc.gn_part = static_cast<double*>(gp.ptr);
            sc.gn_part_len = (size_t(1) << 22) / 8;
            sc.gn_ticket = static_cast<unsigned int*>(gt.ptr);
            ep.gn_groups = 32;
            ep.gn_out = static_cast<double*>(go.ptr);
        }
        pp::DeviceScratch fl(flush ? size_t(256) << 20 : 16);
        pp::GemmPlan plan;
        if (kind == 0)
            pp::plan_gemm(plan, e, A.ptr, M_or_rows, K, K, B.ptr, N, K, ep, sc, pp::device_sm_count(),
                          force_splits, force_block_n);
        else
            pp::plan_conv(plan, e, A.ptr, M_or_rows, W, K, kind, B.ptr, n_pad, ep, sc,
                          pp::device_sm_count(), force_splits, force_block_n);
        plan.a.debug = debug;
        cudaStream_t s;
        CUDA_CHECK(cudaStreamCreate(&s));
        for (int i = 0; i < 3; ++i) pp::launch_gemm(plan, s);
        cudaEvent_t a, b;
        CUDA_CHECK(cudaEventCreate(&a));
        CUDA_CHECK(cudaEventCreate(&b));
        float ms = 0;
        if (!flush) {
            CUDA_CHECK(cudaEventRecord(a, s));
            for (int i = 0; i < reps; ++i) pp::launch_gemm(plan, s);
            CUDA_CHECK(cudaEventRecord(b, s));
            CUDA_CHECK(cudaEventSynchronize(b));
            CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
        } else {
            for (int i = 0; i < reps; ++i) {
                CUDA_CHECK(cudaMemsetAsync(fl.ptr, i & 0xff, size_t(256) << 20, s));
                CUDA_CHECK(cudaEventRecord(a, s));
                pp::launch_gemm(plan, s);
                CUDA_CHECK(cudaEventRecord(b, s));
                CUDA_CHECK(cudaEventSynchronize(b));
                float one = 0;
                CUDA_CHECK(cudaEventElapsedTime(&one, a, b));
                ms += one;
            }
        }
        ms_out[0] = ms / reps;
        ms_out[1] = plan.a.block_n;
        ms_out[2] = plan.a.splits;
        ms_out[3] = plan.a.stages;
        ms_out[4] = plan.grid;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaStreamDestroy(s);
    });
}

}  // extern "C"

#include "kernels.hpp"

#include <functional>

extern "C" {

// Micro-benchmark of the fused GroupNorm apply (and the standalone statistics kernel) on a
// [pix][C] bf16/fp32 band: mean us per launch over `reps` back-to-back launches.
// out[0] = gn_apply, out[1] = gn_stats.  flags: 1 SiLU, 2 temb, 4 skip.
PP_API int pp_dev_gn_bench(int dtype, long long pix, int C, int G, int flags, int reps,
                           double* out) {
    return pp::guard([&] {
        pp::require_device();
        const pp::Elem e = pp::elem_of(dtype);
        const size_t eb = pp::elem_bytes(e);
        pp::DeviceScratch x(pix * C * eb), y(pix * C * eb), sk(pix * C * eb), st(G * 16),
            gam(C * 4), bet(C * 4), te(C * 4), part(size_t(4) << 20), tick(1024);
        CUDA_CHECK(cudaMemset(x.ptr, 0x3c, pix * C * eb));
        CUDA_CHECK(cudaMemset(sk.ptr, 0x3c, pix * C * eb));
        CUDA_CHECK(cudaMemset(gam.ptr, 0, C * 4));
        CUDA_CHECK(cudaMemset(bet.ptr, 0, C * 4));
        CUDA_CHECK(cudaMemset(te.ptr, 0, C * 4));
        CUDA_CHECK(cudaMemset(st.ptr, 0, G * 16));
        CUDA_CHECK(cudaMemset(tick.ptr, 0, 1024));
        pp::GnCombine cb{};
        cb.mode = 0;
        cb.fresh = static_cast<const double*>(st.ptr);
        cb.eps = 1e-5f;
        cudaStream_t s;
        CUDA_CHECK(cudaStreamCreate(&s));
        cudaEvent_t a, b;
        CUDA_CHECK(cudaEventCreate(&a));
        CUDA_CHECK(cudaEventCreate(&b));
        pp::DeviceScratch st2(G * 16), tick2(1024);
        CUDA_CHECK(cudaMemset(tick2.ptr, 0, 1024));
        pp::GnStatsOut so;   // flags & 8: fused statistics of the output
        if (flags & 8) {
            so.G = G;
            so.count = double(C / G) * double(pix);
            so.partial = static_cast<double*>(part.ptr);
            so.ticket = static_cast<unsigned int*>(tick2.ptr);
            so.out = static_cast<double*>(st2.ptr);
        }
        auto apply = [&] {
            pp::gn_apply(e, x.ptr, y.ptr, pix, C, C, G, cb, static_cast<const float*>(gam.ptr),
                         static_cast<const float*>(bet.ptr), flags & 1,
                         (flags & 2) ? static_cast<const float*>(te.ptr) : nullptr,
                         (flags & 4) ? sk.ptr : nullptr, false, s, &so);
        };
        auto stats = [&] {
            pp::gn_stats(e, x.ptr, pix, C, C, G, double(C / G) * double(pix),
                         static_cast<double*>(part.ptr), static_cast<unsigned int*>(tick.ptr),
                         static_cast<double*>(st.ptr), s);
        };
        for (int k = 0; k < 2; ++k) {
            auto fn = k == 0 ? std::function<void()>(apply) : std::function<void()>(stats);
            for (int i = 0; i < 3; ++i) fn();
            CUDA_CHECK(cudaEventRecord(a, s));
            for (int i = 0; i < reps; ++i) fn();
            CUDA_CHECK(cudaEventRecord(b, s));
            CUDA_CHECK(cudaEventSynchronize(b));
            float ms = 0;
            CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
            out[k] = ms * 1e3 / reps;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaStreamDestroy(s);
    });
}

}  // extern "C"
