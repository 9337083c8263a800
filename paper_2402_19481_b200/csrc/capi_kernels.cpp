// C ABI: kernel-level operators with the reference's tensor semantics
// (proj/include/patchsim/tensor.hpp:77-118).  Host NCHW fp32 in / out; every entry
// point runs the sm_100a kernels of the hot path (layout conversion to NHWC bands on
// the host, compute on the device).  Used for per-operator parity tests.
#include "capi_common.hpp"
#include "gemm.hpp"
#include "kernels.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

namespace {

using pp::Elem;

uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}
float tf32(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & ~0x1fffu;
    std::memcpy(&f, &u, 4);
    return f;
}

int round_up(int a, int b) { return (a + b - 1) / b * b; }

// Device buffer holding `v` as element type e (bf16, or fp32 rounded to tf32 when `gemm`).
struct DevElems {
    pp::DeviceScratch mem;
    DevElems(const std::vector<float>& v, Elem e, bool gemm)
        : mem(v.size() * pp::elem_bytes(e) + 16) {
        if (e == Elem::BF16) {
            std::vector<uint16_t> h(v.size());
            for (size_t i = 0; i < v.size(); ++i) h[i] = f2bf(v[i]);
            CUDA_CHECK(cudaMemcpy(mem.ptr, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
        } else {
            std::vector<float> h(v);
            if (gemm)
                for (float& x : h) x = tf32(x);
            CUDA_CHECK(cudaMemcpy(mem.ptr, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
        }
    }
};

struct DevF32 {
    pp::DeviceScratch mem;
    explicit DevF32(size_t n) : mem(n * 4 + 16) { CUDA_CHECK(cudaMemset(mem.ptr, 0, n * 4 + 16)); }
    DevF32(const float* src, size_t n) : mem(n * 4 + 16) {
        CUDA_CHECK(cudaMemcpy(mem.ptr, src, n * 4, cudaMemcpyHostToDevice));
    }
    float* p() const { return static_cast<float*>(mem.ptr); }
    std::vector<float> get(size_t n) const {
        std::vector<float> h(n);
        CUDA_CHECK(cudaMemcpy(h.data(), mem.ptr, n * 4, cudaMemcpyDeviceToHost));
        return h;
    }
};

struct Scratch {
    pp::DeviceScratch ws, tk, gp, gt;
    pp::GemmScratch sc;
    explicit Scratch(size_t ws_bytes)
        : ws(ws_bytes), tk(size_t(1) << 20), gp(size_t(1) << 20), gt(1024) {
        CUDA_CHECK(cudaMemset(tk.ptr, 0, size_t(1) << 20));
        CUDA_CHECK(cudaMemset(gt.ptr, 0, 1024));
        sc.ws = static_cast<float*>(ws.ptr);
        sc.ws_bytes = ws_bytes;
        sc.tickets = static_cast<unsigned int*>(tk.ptr);
        sc.n_tickets = (size_t(1) << 20) / 4;
        sc.gn_part = static_cast<double*>(gp.ptr);
        sc.gn_part_len = (size_t(1) << 20) / 8;
        sc.gn_ticket = static_cast<unsigned int*>(gt.ptr);
    }
};

// out[M][N] fp32 = A[M][K] * B[N][K]^T + bias  (A, B host fp32, K padded to 128 bytes)
std::vector<float> gemm_host(Elem e, const std::vector<float>& A, int M, int K,
                             const std::vector<float>& B, int N, const float* bias) {
    const int kel = int(128 / pp::elem_bytes(e));
    const int Kp = round_up(K, kel);
    std::vector<float> Ap(size_t(M) * Kp, 0.0f), Bp(size_t(N) * Kp, 0.0f);
    for (int i = 0; i < M; ++i) std::memcpy(&Ap[size_t(i) * Kp], &A[size_t(i) * K], K * 4);
    for (int i = 0; i < N; ++i) std::memcpy(&Bp[size_t(i) * Kp], &B[size_t(i) * K], K * 4);
    DevElems dA(Ap, e, true), dB(Bp, e, true);
    DevF32 dbias(bias ? bias : Ap.data(), bias ? N : 1);
    DevF32 out(size_t(M) * N);
    pp::EpilogueSpec ep;
    ep.out = out.p();
    ep.out_ld = N;
    ep.n_valid = N;
    ep.out_f32 = true;
    ep.bias = bias ? dbias.p() : nullptr;
    Scratch s(size_t(8) * M * round_up(N, 16) * 4 + 1024);
    pp::GemmPlan plan;
    pp::plan_gemm(plan, e, dA.mem.ptr, M, Kp, Kp, dB.mem.ptr, N, Kp, ep, s.sc, pp::device_sm_count());
    pp::launch_gemm(plan, 0);
    CUDA_CHECK(cudaDeviceSynchronize());
    return out.get(size_t(M) * N);
}

std::vector<float> to_host(const float* p, size_t n) { return std::vector<float>(p, p + n); }

}  // namespace

extern "C" {

PP_API int pp_conv2d_region(int dtype, const float* x, int n, int c, int h, int w, int r0, int r1,
                            const float* weight, int c_out, int k, const float* bias, int stride,
                            int pad, float* out) {
    // conv2d_region (proj/src/tensor.cpp:79-130)
    return pp::guard([&] {
        if (!(0 <= r0 && r0 < r1 && r1 <= h) || w <= 0)
            throw std::invalid_argument("conv2d_region: invalid region [" + std::to_string(r0) + "," +
                                        std::to_string(r1) + ") of " + std::to_string(h) + "x" +
                                        std::to_string(w));
        if (k % 2 != 1) throw std::invalid_argument("conv2d: kernel must be square and odd");
        if (stride != 1 && stride != 2) throw std::invalid_argument("conv2d: stride must be 1 or 2");
        if (k != 3 || pad != 1)
            throw std::invalid_argument("conv2d: the B200 path implements the model's 3x3 / pad-1 conv");
        pp::require_device();
        const Elem e = pp::elem_of(dtype);
        const int kel = int(128 / pp::elem_bytes(e));
        const int out_h = (h + 2 * pad - k) / stride + 1;
        const int out_w = (w + 2 * pad - k) / stride + 1;
        const int oy0 = std::min((r0 + stride - 1) / stride, out_h);
        const int oy1 = std::min((r1 + stride - 1) / stride, out_h);
        if (oy0 >= oy1) throw std::invalid_argument("conv2d_region: region maps to no output rows");
        const int rows_out = oy1 - oy0;
        const int cp = round_up(c, kel);
        const int wb = stride == 2 ? round_up(w, 2) : w;               // even width for stride 2
        const int rows_in = stride == 1 ? rows_out : 2 * rows_out;     // band rows (no halos)
        const int first = oy0 * stride;                                 // first band row (input)
        const int n_pad = round_up(c_out, 16);
        // weights [n_pad][3][3][cp]
        std::vector<float> wp(size_t(n_pad) * 9 * cp, 0.0f);
        for (int co = 0; co < c_out; ++co)
            for (int ci = 0; ci < c; ++ci)
                for (int t = 0; t < 9; ++t)
                    wp[(size_t(co) * 9 + t) * cp + ci] = weight[(size_t(co) * c + ci) * 9 + t];
        DevElems dW(wp, e, true);
        DevF32 db(bias, c_out);
        Scratch s(size_t(8) * rows_out * out_w * n_pad * 4 + 1024);
        for (int b = 0; b < n; ++b) {
            // padded NHWC band: row 0 = halo above, rows 1..rows_in = band, last = halo below
            std::vector<float> band(size_t(rows_in + 2) * wb * cp, 0.0f);
            for (int yy = -1; yy <= rows_in; ++yy) {
                const int gy = first + yy;
                if (gy < 0 || gy >= h) continue;
                for (int xx = 0; xx < w; ++xx)
                    for (int ci = 0; ci < c; ++ci)
                        band[(size_t(yy + 1) * wb + xx) * cp + ci] =
                            x[((size_t(b) * c + ci) * h + gy) * w + xx];
            }
            DevElems dIn(band, e, true);
            DevF32 dOut(size_t(rows_out) * out_w * c_out);
            pp::EpilogueSpec ep;
            ep.out = dOut.p();
            ep.out_ld = c_out;
            ep.n_valid = c_out;
            ep.out_f32 = true;
            ep.bias = db.p();
            pp::GemmPlan plan;
            pp::plan_conv(plan, e, dIn.mem.ptr, rows_in, wb, cp, stride, dW.mem.ptr, n_pad, ep, s.sc,
                          pp::device_sm_count());
            pp::launch_gemm(plan, 0);
            CUDA_CHECK(cudaDeviceSynchronize());
            const std::vector<float> o = dOut.get(size_t(rows_out) * out_w * c_out);
            for (int co = 0; co < c_out; ++co)
                for (int yy = 0; yy < rows_out; ++yy)
                    for (int xx = 0; xx < out_w; ++xx)
                        out[((size_t(b) * c_out + co) * rows_out + yy) * out_w + xx] =
                            o[(size_t(yy) * out_w + xx) * c_out + co];
        }
    });
}

PP_API int pp_linear(int dtype, const float* tokens, int n, int t, int in_f, const float* weight,
                     int out_f, const float* bias, float* out) {
    // linear (proj/src/tensor.cpp:139-161)
    return pp::guard([&] {
        pp::require_device();
        const Elem e = pp::elem_of(dtype);
        const auto A = to_host(tokens, size_t(n) * t * in_f);
        const auto B = to_host(weight, size_t(out_f) * in_f);
        const auto o = gemm_host(e, A, n * t, in_f, B, out_f, bias);
        std::memcpy(out, o.data(), o.size() * 4);
    });
}

PP_API int pp_attention(int dtype, const float* q, const float* k, const float* v, int n, int m,
                        int s, int d, int dv, float scale, float* out) {
    // attention (proj/src/tensor.cpp:163-199) through the product path: S = Q K^T tcgen05
    // GEMM with the softmax in its epilogue (per key tile row max) -> attn_rescale (row max,
    // row sum) -> O = P V tcgen05 GEMM (bf16: V MN-major; 1/l in the epilogue)
    return pp::guard([&] {
        if (m <= 0 || s <= 0 || d <= 0 || dv <= 0)
            throw std::invalid_argument("attention: empty operand");
        pp::require_device();
        const Elem e = pp::elem_of(dtype);
        const int kel = int(128 / pp::elem_bytes(e));
        const int dp = round_up(d, kel), dvp = round_up(dv, kel);
        const int sp = round_up(s, 64);
        const size_t eb = pp::elem_bytes(e);
        for (int b = 0; b < n; ++b) {
            // padded row-major copies (zero channels beyond d / dv)
            std::vector<float> Q(size_t(m) * dp, 0.0f), K(size_t(s) * dp, 0.0f), V(size_t(s) * dvp, 0.0f);
            for (int i = 0; i < m; ++i)
                std::memcpy(&Q[size_t(i) * dp], q + (size_t(b) * m + i) * d, size_t(d) * 4);
            for (int j = 0; j < s; ++j) {
                std::memcpy(&K[size_t(j) * dp], k + (size_t(b) * s + j) * d, size_t(d) * 4);
                std::memcpy(&V[size_t(j) * dvp], v + (size_t(b) * s + j) * dv, size_t(dv) * 4);
            }
            DevElems dQ(Q, e, true), dK(K, e, true), dV(V, e, true);
            pp::DeviceScratch dP(size_t(m) * sp * eb + 16);
            CUDA_CHECK(cudaMemset(dP.ptr, 0, size_t(m) * sp * eb + 16));
            DevF32 rscale{size_t(m)};
            DevF32 dO(size_t(m) * dvp);
            Scratch sc(size_t(8) * m * std::max(sp, dvp) * 4 + 1024);
            const int sms = pp::device_sm_count();
            pp::EpilogueSpec es;
            es.out = dP.ptr;
            es.out_ld = sp;
            es.out_f32 = e == Elem::F32;
            es.round_tf32 = e == Elem::F32;
            es.n_valid = s;
            es.sm_rowmax = rscale.p();   // placeholder: marks the softmax epilogue
            es.sm_scale = scale;
            es.sm_ld = m;
            pp::GemmPlan splan, pvplan;
            pp::plan_gemm(splan, e, dQ.mem.ptr, m, dp, dp, dK.mem.ptr, s, dp, es, sc.sc, sms);
            DevF32 rowmax{size_t(splan.a.n_tiles) * m};
            splan.a.sm_rowmax = rowmax.p();
            pp::EpilogueSpec ep;
            ep.out = dO.p();
            ep.out_ld = dvp;
            ep.n_valid = dvp;
            ep.out_f32 = true;
            ep.row_scale = rscale.p();
            std::unique_ptr<pp::DeviceScratch> dVt;
            if (e == Elem::BF16) {
                pp::plan_gemm_bmn(pvplan, e, dP.ptr, m, sp, sp, dV.mem.ptr, s, dvp, dvp, ep, sc.sc, sms);
            } else {   // TF32: B K-major only, V^T by the transpose kernel
                dVt.reset(new pp::DeviceScratch(size_t(dvp) * sp * eb + 16));
                CUDA_CHECK(cudaMemset(dVt->ptr, 0, size_t(dvp) * sp * eb + 16));
                pp::transpose(e, dV.mem.ptr, s, dvp, dvp, dVt->ptr, sp, 0);
                pp::plan_gemm(pvplan, e, dP.ptr, m, sp, sp, dVt->ptr, dvp, sp, ep, sc.sc, sms);
            }
            pp::launch_gemm(splan, 0);
            pp::attn_rescale(e, dP.ptr, sp, m, s, rowmax.p(), splan.a.n_tiles, splan.a.block_n, m,
                             rscale.p(), e == Elem::F32, 0);
            pp::launch_gemm(pvplan, 0);
            CUDA_CHECK(cudaDeviceSynchronize());
            const auto o = dO.get(size_t(m) * dvp);
            for (int i = 0; i < m; ++i)
                std::memcpy(out + (size_t(b) * m + i) * dv, &o[size_t(i) * dvp], size_t(dv) * 4);
        }
    });
}

PP_API int pp_group_stats(int dtype, const float* x, int n, int c, int h, int w, int groups,
                          int row_start, int row_end, double* mean, double* mean_sq) {
    // group_stats (proj/src/tensor.cpp:203-235)
    return pp::guard([&] {
        if (groups <= 0 || c % groups != 0)
            throw std::invalid_argument("group_stats: channels " + std::to_string(c) +
                                        " not divisible by groups " + std::to_string(groups));
        int y0 = 0, y1 = h;
        if (row_start >= 0) {
            if (!(0 <= row_start && row_start < row_end && row_end <= h))
                throw std::invalid_argument("group_stats: invalid region");
            y0 = row_start;
            y1 = row_end;
        }
        pp::require_device();
        const Elem e = pp::elem_of(dtype);
        const int ld = round_up(c, 8);
        for (int b = 0; b < n; ++b) {
            std::vector<float> band(size_t(y1 - y0) * w * ld, 0.0f);
            for (int ci = 0; ci < c; ++ci)
                for (int yy = y0; yy < y1; ++yy)
                    for (int xx = 0; xx < w; ++xx)
                        band[(size_t(yy - y0) * w + xx) * ld + ci] = x[((size_t(b) * c + ci) * h + yy) * w + xx];
            DevElems dx(band, e, false);
            const long long pix = (long long)(y1 - y0) * w;
            pp::DeviceScratch part(size_t(pp::gn_stats_blocks(pix)) * groups * 16 + 16), tk(1024), st(size_t(groups) * 16);
            CUDA_CHECK(cudaMemset(tk.ptr, 0, 1024));
            pp::gn_stats(e, dx.mem.ptr, pix, c, ld, groups, double(c / groups) * double(pix),
                         static_cast<double*>(part.ptr), static_cast<unsigned int*>(tk.ptr),
                         static_cast<double*>(st.ptr), 0);
            std::vector<double> h2(size_t(groups) * 2);
            CUDA_CHECK(cudaMemcpy(h2.data(), st.ptr, h2.size() * 8, cudaMemcpyDeviceToHost));
            for (int g = 0; g < groups; ++g) {
                mean[size_t(b) * groups + g] = h2[g * 2];
                mean_sq[size_t(b) * groups + g] = h2[g * 2 + 1];
            }
        }
    });
}

PP_API int pp_group_norm_apply(int dtype, const float* x, int n, int c, int h, int w,
                               int row_start, int row_end, int groups, const double* mean,
                               const double* mean_sq, const float* gamma, const float* beta,
                               float eps, float* out) {
    // group_norm_apply (proj/src/tensor.cpp:237-277): rows outside the region pass through
    return pp::guard([&] {
        if (groups <= 0 || c % groups != 0)
            throw std::invalid_argument("group_norm_apply: stats shape does not match input");
        for (int i = 0; i < n * groups; ++i)
            if (mean_sq[i] - mean[i] * mean[i] < 0.0)
                throw std::runtime_error(
                    "group_norm_apply: negative variance (caller must substitute fallback stats)");
        int y0 = 0, y1 = h;
        if (row_start >= 0) {
            y0 = row_start;
            y1 = row_end;
        }
        pp::require_device();
        const Elem e = pp::elem_of(dtype);
        const int ld = round_up(c, 8);
        std::memcpy(out, x, size_t(n) * c * h * w * 4);
        std::vector<float> gp(ld, 0.0f), bp(ld, 0.0f);
        std::memcpy(gp.data(), gamma, c * 4);
        std::memcpy(bp.data(), beta, c * 4);
        DevF32 dg(gp.data(), ld), dbeta(bp.data(), ld);
        for (int b = 0; b < n; ++b) {
            std::vector<float> band(size_t(y1 - y0) * w * ld, 0.0f);
            for (int ci = 0; ci < c; ++ci)
                for (int yy = y0; yy < y1; ++yy)
                    for (int xx = 0; xx < w; ++xx)
                        band[(size_t(yy - y0) * w + xx) * ld + ci] = x[((size_t(b) * c + ci) * h + yy) * w + xx];
            DevElems dx(band, e, false);
            pp::DeviceScratch dy(band.size() * pp::elem_bytes(e) + 16), st(size_t(groups) * 16), err(16);
            CUDA_CHECK(cudaMemset(err.ptr, 0, 16));
            std::vector<double> s2(size_t(groups) * 2);
            for (int g = 0; g < groups; ++g) {
                s2[g * 2] = mean[size_t(b) * groups + g];
                s2[g * 2 + 1] = mean_sq[size_t(b) * groups + g];
            }
            CUDA_CHECK(cudaMemcpy(st.ptr, s2.data(), s2.size() * 8, cudaMemcpyHostToDevice));
            pp::GnCombine cb{};
            cb.mode = pp::GN_USE_LOCAL;
            cb.fresh = static_cast<const double*>(st.ptr);
            cb.all_cur = cb.all_prev = cb.fresh;
            cb.n = 1;
            cb.eps = eps;
            cb.err = static_cast<int*>(err.ptr);
            const long long pix = (long long)(y1 - y0) * w;
            pp::gn_apply(e, dx.mem.ptr, dy.ptr, pix, c, ld, groups, cb, dg.p(), dbeta.p(), false,
                         nullptr, nullptr, false, 0);
            DevF32 f(band.size());
            pp::elem_to_f32(e, dy.ptr, f.p(), (long long)band.size(), 0);
            CUDA_CHECK(cudaDeviceSynchronize());
            const auto o = f.get(band.size());
            for (int ci = 0; ci < c; ++ci)
                for (int yy = y0; yy < y1; ++yy)
                    for (int xx = 0; xx < w; ++xx)
                        out[((size_t(b) * c + ci) * h + yy) * w + xx] = o[(size_t(yy - y0) * w + xx) * ld + ci];
        }
    });
}

PP_API int pp_silu(int dtype, const float* x, long count, float* out) {
    // silu (proj/src/tensor.cpp:297-306)
    return pp::guard([&] {
        pp::require_device();
        const Elem e = pp::elem_of(dtype);
        const long padded = (count + 7) / 8 * 8;
        std::vector<float> v(padded, 0.0f);
        std::memcpy(v.data(), x, count * 4);
        DevElems dx(v, e, false);
        pp::DeviceScratch dy(padded * pp::elem_bytes(e) + 16);
        pp::silu(e, dx.mem.ptr, dy.ptr, padded, false, 0);
        DevF32 f(padded);
        pp::elem_to_f32(e, dy.ptr, f.p(), padded, 0);
        CUDA_CHECK(cudaDeviceSynchronize());
        const auto o = f.get(padded);
        std::memcpy(out, o.data(), count * 4);
    });
}

PP_API int pp_upsample_nearest2x(int dtype, const float* x, int n, int c, int h, int w, float* out) {
    // upsample_nearest2x (proj/src/tensor.cpp:317-334)
    return pp::guard([&] {
        pp::require_device();
        const Elem e = pp::elem_of(dtype);
        const int ld = round_up(c, 8);
        for (int b = 0; b < n; ++b) {
            std::vector<float> band(size_t(h) * w * ld, 0.0f);
            for (int ci = 0; ci < c; ++ci)
                for (int yy = 0; yy < h; ++yy)
                    for (int xx = 0; xx < w; ++xx)
                        band[(size_t(yy) * w + xx) * ld + ci] = x[((size_t(b) * c + ci) * h + yy) * w + xx];
            DevElems dx(band, e, false);
            const size_t on = size_t(4) * h * w * ld;
            pp::DeviceScratch dy(on * pp::elem_bytes(e) + 16);
            pp::upsample2x(e, dx.mem.ptr, dy.ptr, h, w, ld, 0);
            DevF32 f(on);
            pp::elem_to_f32(e, dy.ptr, f.p(), (long long)on, 0);
            CUDA_CHECK(cudaDeviceSynchronize());
            const auto o = f.get(on);
            for (int ci = 0; ci < c; ++ci)
                for (int yy = 0; yy < 2 * h; ++yy)
                    for (int xx = 0; xx < 2 * w; ++xx)
                        out[((size_t(b) * c + ci) * 2 * h + yy) * 2 * w + xx] = o[(size_t(yy) * 2 * w + xx) * ld + ci];
        }
    });
}

PP_API int pp_ddim_update(const float* x, const float* eps, long count, double abar_t,
                          double abar_next, float* out) {
    // ddim_update (proj/src/sampler.cpp:46-61), fp64 math on the device
    return pp::guard([&] {
        pp::require_device();
        DevF32 dx(x, count), de(eps, count), dy(count);
        pp::ddim_update(dx.p(), de.p(), dy.p(), count, 1, abar_t, abar_next, Elem::F32, nullptr, 0, 0);
        CUDA_CHECK(cudaDeviceSynchronize());
        const auto o = dy.get(count);
        std::memcpy(out, o.data(), count * 4);
    });
}

}  // extern "C"
