// HBM-bound kernels (see kernels.hpp).  128-bit vectorised NHWC access; all
// reductions are fixed-order (no float atomics) so every run is bit-deterministic.
#include "kernels.hpp"
#include "util.hpp"

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

namespace pp {

namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float rtf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

template <class T>
struct Vec {
    static constexpr int N = 16 / sizeof(T);
};

template <class T>
__device__ __forceinline__ void load_vec(const T* p, float* f);
template <>
__device__ __forceinline__ void load_vec<float>(const float* p, float* f) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
}
template <>
__device__ __forceinline__ void load_vec<bf16>(const bf16* p, float* f) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}
template <class T>
__device__ __forceinline__ void store_vec(T* p, const float* f, bool round_tf32);
template <>
__device__ __forceinline__ void store_vec<float>(float* p, const float* f, bool r) {
    float4 v = make_float4(f[0], f[1], f[2], f[3]);
    if (r) {
        v.x = rtf32(v.x); v.y = rtf32(v.y); v.z = rtf32(v.z); v.w = rtf32(v.w);
    }
    *reinterpret_cast<float4*>(p) = v;
}
template <>
__device__ __forceinline__ void store_vec<bf16>(bf16* p, const float* f, bool) {
    uint4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = v;
}
template <class T>
__device__ __forceinline__ T from_float(float x, bool r);
template <>
__device__ __forceinline__ float from_float<float>(float x, bool r) { return r ? rtf32(x) : x; }
template <>
__device__ __forceinline__ bf16 from_float<bf16>(float x, bool) { return __float2bfloat16(x); }
__device__ __forceinline__ float to_float(float x) { return x; }
__device__ __forceinline__ float to_float(bf16 x) { return __bfloat162float(x); }

int grid_for(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    return int(std::max<long long>(1, std::min<long long>(b, 148LL * 16)));
}

// ---------------------------------------------------------------- GroupNorm stats
constexpr int kGnThreads = 256;
constexpr int kGnPixels = 32;

// One launch: every block reduces kGnPixels pixels to per-group fp64 partials; the last
// block to finish (ticket) folds all partials in a fixed order into out[G][2] =
// (mean, mean_sq) -- group_stats (tensor.cpp:203-235) with fp32 per-thread sums over
// <= 64 values and fp64 everywhere above that.  Deterministic for a given grid.
template <class T>
__global__ void gn_stats_kernel(const T* __restrict__ x, long long pix, int C, int ld, int G,
                                double count, double* __restrict__ partial,
                                unsigned int* __restrict__ ticket, double* __restrict__ out) {
    constexpr int VEC = Vec<T>::N;
    extern __shared__ unsigned char sm_raw[];
    __shared__ bool is_last;
    const int nvec = C / VEC;
    const int L = max(1, kGnThreads / nvec);
    float* s_sum = reinterpret_cast<float*>(sm_raw);
    float* s_sq = s_sum + L * C;
    double* c_sum = reinterpret_cast<double*>(s_sq + L * C);
    double* c_sq = c_sum + C;
    const long long p0 = (long long)blockIdx.x * kGnPixels;
    const long long p1 = min(p0 + kGnPixels, pix);
    for (int idx = threadIdx.x; idx < L * nvec; idx += blockDim.x) {
        const int pl = idx / nvec, v = idx - pl * nvec;
        float a[VEC], b[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) a[i] = b[i] = 0.0f;
        for (long long p = p0 + pl; p < p1; p += 4 * L) {
            float f[4][VEC];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (p + u * L < p1) {
                    load_vec<T>(x + (p + u * L) * ld + v * VEC, f[u]);
                } else {
#pragma unroll
                    for (int i = 0; i < VEC; ++i) f[u][i] = 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < VEC; ++i) {
                    a[i] += f[u][i];
                    b[i] = fmaf(f[u][i], f[u][i], b[i]);
                }
        }
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            s_sum[pl * C + v * VEC + i] = a[i];
            s_sq[pl * C + v * VEC + i] = b[i];
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        double a = 0.0, b = 0.0;
        for (int pl = 0; pl < L; ++pl) {
            a += double(s_sum[pl * C + c]);
            b += double(s_sq[pl * C + c]);
        }
        c_sum[c] = a;
        c_sq[c] = b;
    }
    __syncthreads();
    const int cpg = C / G;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        double a = 0.0, b = 0.0;
        for (int c = g * cpg; c < (g + 1) * cpg; ++c) {
            a += c_sum[c];
            b += c_sq[c];
        }
        partial[((long long)blockIdx.x * G + g) * 2] = a;
        partial[((long long)blockIdx.x * G + g) * 2 + 1] = b;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
    const int blocks = gridDim.x;
    for (int g = warp; g < G; g += nw) {
        double a = 0.0, b = 0.0;
        for (int k = lane; k < blocks; k += 32) {
            a += __ldcg(partial + ((long long)k * G + g) * 2);
            b += __ldcg(partial + ((long long)k * G + g) * 2 + 1);
        }
        for (int o = 16; o; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if (lane == 0) {
            out[g * 2] = a / count;
            out[g * 2 + 1] = b / count;
        }
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

// Device-order weighted mean (collectives.cpp:150-172), no FMA contraction.
__device__ void weighted_mean(const double* all, int n, const double* w, int G, int g, double& m,
                              double& q) {
    if (n == 1) {
        m = all[g * 2];
        q = all[g * 2 + 1];
        return;
    }
    double tw = 0.0;
    for (int d = 0; d < n; ++d) tw = __dadd_rn(tw, w[d]);
    double a = 0.0, b = 0.0;
    for (int d = 0; d < n; ++d) {
        a = __dadd_rn(a, __dmul_rn(w[d], all[((long long)d * G + g) * 2]));
        b = __dadd_rn(b, __dmul_rn(w[d], all[((long long)d * G + g) * 2 + 1]));
    }
    m = __ddiv_rn(a, tw);
    q = __ddiv_rn(b, tw);
}

// The statistics a band normalises with (runtime.cpp:242-300 + corrected_gn_stats,
// runtime.cpp:85-106); returns (mean, 1/sqrt(var + eps)).
__device__ void gn_use_of(const GnCombine& cb, int G, int g, float& mu, float& inv, bool& neg) {
    double m = cb.fresh[g * 2], q = cb.fresh[g * 2 + 1];
    if (cb.mode == GN_USE_GLOBAL) {
        weighted_mean(cb.all_cur, cb.n, cb.weights, G, g, m, q);
    } else if (cb.mode == GN_USE_STALE) {
        weighted_mean(cb.all_prev, cb.n, cb.weights, G, g, m, q);
    } else if (cb.mode == GN_USE_CORRECTED) {
        const double lm = cb.all_prev[((long long)cb.rank * G + g) * 2];
        const double lq = cb.all_prev[((long long)cb.rank * G + g) * 2 + 1];
        double gm, gq;
        weighted_mean(cb.all_prev, cb.n, cb.weights, G, g, gm, gq);
        if (!(gm == lm && gq == lq)) {
            const double cm = __dadd_rn(gm, __dsub_rn(m, lm));
            const double cq = __dadd_rn(gq, __dsub_rn(q, lq));
            if (!(__dsub_rn(cq, __dmul_rn(cm, cm)) < 0.0)) {
                m = cm;
                q = cq;
            }
        }
    }
    const double var = __dsub_rn(q, __dmul_rn(m, m));
    neg = var < 0.0;
    mu = float(m);
    inv = float(1.0 / sqrt(__dadd_rn(fmax(var, 0.0), double(cb.eps))));
}

template <class T>
__global__ void gn_apply_kernel(const T* __restrict__ x, T* __restrict__ y, int pix, int C, int ld,
                                int G, const GnCombine cb, const float* __restrict__ gamma,
                                const float* __restrict__ beta, int do_silu,
                                const float* __restrict__ temb, const T* __restrict__ skip,
                                int round_tf32) {
    constexpr int VEC = Vec<T>::N;
    extern __shared__ float s_tab[];   // [4][ld]: mean, inv_std*gamma, beta, temb
    __shared__ float s_use[2 * 1024];
    float* s_mu = s_tab;
    float* s_sc = s_tab + ld;
    float* s_be = s_tab + 2 * ld;
    float* s_te = s_tab + 3 * ld;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        float mu, inv;
        bool neg;
        gn_use_of(cb, G, g, mu, inv, neg);
        s_use[2 * g] = mu;
        s_use[2 * g + 1] = inv;
        // group_norm_apply contract (tensor.cpp:256-259), reported once per launch
        if (neg && blockIdx.x == 0 && cb.err) atomicExch(cb.err, 1);
    }
    __syncthreads();
    const int cpg = C / G;
    for (int c = threadIdx.x; c < ld; c += blockDim.x) {
        if (c < C) {
            const int g = c / cpg;
            s_mu[c] = s_use[2 * g];
            s_sc[c] = s_use[2 * g + 1] * gamma[c];
            s_be[c] = beta[c];
            s_te[c] = temb ? temb[c] : 0.0f;
        } else {
            s_mu[c] = s_sc[c] = s_be[c] = s_te[c] = 0.0f;
        }
    }
    __syncthreads();
    const unsigned nvec = unsigned(ld / VEC);
    const unsigned total = unsigned(pix) * nvec;
    const unsigned stride = gridDim.x * blockDim.x;
    constexpr int U = 4;   // vectors in flight per thread
    for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += U * stride) {
        float f[U][VEC], sk[U][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned j = idx + u * stride;
            if (j < total) {
                load_vec<T>(x + size_t(j) * VEC, f[u]);
                if (skip) load_vec<T>(skip + size_t(j) * VEC, sk[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned j = idx + u * stride;
            if (j >= total) continue;
            const int c0 = int(j % nvec) * VEC;
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
                const int c = c0 + i;
                float v = (f[u][i] - s_mu[c]) * s_sc[c] + s_be[c];
                if (do_silu) {
                    if constexpr (sizeof(T) == 2)
                        v = __fdividef(v, 1.0f + __expf(-v));
                    else
                        v = v / (1.0f + expf(-v));
                }
                v = v + s_te[c];
                if (skip) v = v + sk[u][i];
                f[u][i] = v;
            }
            if (c0 + VEC > C) {
#pragma unroll
                for (int i = 0; i < VEC; ++i)
                    if (c0 + i >= C) f[u][i] = 0.0f;
            }
            store_vec<T>(y + size_t(j) * VEC, f[u], round_tf32 != 0);
        }
    }
}

// 2-D mapping: threadIdx.x / blockIdx.x select a fixed 16-byte channel vector (its GN
// coefficients live in registers), threadIdx.y / blockIdx.y stride over pixels with four
// vectors in flight per thread.  A warp touches 32 consecutive vectors of one pixel.
template <class T>
__global__ void __launch_bounds__(256, 4)
    gn_apply_2d_kernel(const T* __restrict__ x, T* __restrict__ y, int pix, int C,
                                   int ld, int G, const GnCombine cb,
                                   const float* __restrict__ gamma, const float* __restrict__ beta,
                                   int do_silu, const float* __restrict__ temb,
                                   const T* __restrict__ skip, int round_tf32) {
    constexpr int VEC = Vec<T>::N;
    __shared__ float s_use[2 * 1024];
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (int g = tid; g < G; g += blockDim.x * blockDim.y) {
        float mu, inv;
        bool neg;
        gn_use_of(cb, G, g, mu, inv, neg);
        s_use[2 * g] = mu;
        s_use[2 * g + 1] = inv;
        // group_norm_apply contract (tensor.cpp:256-259), reported once per launch
        if (neg && blockIdx.x == 0 && blockIdx.y == 0 && cb.err) atomicExch(cb.err, 1);
    }
    __syncthreads();
    // per-channel coefficients of this block's channel slice: (mean, inv_std*gamma, beta, temb)
    __shared__ float4 s_coef[1024];
    const int nvec = ld / VEC;
    const int cbase = blockIdx.x * blockDim.x * VEC;
    const int cpg = C / G;
    // layout [i][tx] (element i of thread tx's vector): a warp's LDS.128 of one i is
    // 512 contiguous bytes -> conflict-free
    for (int k = tid; k < int(blockDim.x) * VEC; k += blockDim.x * blockDim.y) {
        const int txk = k / VEC, i = k - txk * VEC;
        const int c = cbase + k;
        float4 k4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < C) {
            const int g = c / cpg;
            k4 = make_float4(s_use[2 * g], s_use[2 * g + 1] * gamma[c], beta[c], temb ? temb[c] : 0.0f);
        }
        s_coef[i * blockDim.x + txk] = k4;
    }
    __syncthreads();
    const int cv = blockIdx.x * blockDim.x + threadIdx.x;
    if (cv >= nvec) return;
    const int c0 = cv * VEC;
    const float4* coef = s_coef + threadIdx.x;
    const int cstride = blockDim.x;
    const int pstride = blockDim.y * gridDim.y;
    constexpr int U = 4;   // raw 16-byte vectors in flight per thread (4 registers each)
    const uint4* xv = reinterpret_cast<const uint4*>(x) + cv;
    const uint4* sv = reinterpret_cast<const uint4*>(skip) + cv;
    for (int p = blockIdx.y * blockDim.y + threadIdx.y; p < pix; p += U * pstride) {
        uint4 rx[U], rs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int pp = p + u * pstride;
            if (pp < pix) {
                rx[u] = __ldcs(xv + size_t(pp) * nvec);
                if (skip) rs[u] = __ldcs(sv + size_t(pp) * nvec);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int pp = p + u * pstride;
            if (pp >= pix) continue;
            float f[VEC], sk[VEC];
            load_vec<T>(reinterpret_cast<const T*>(&rx[u]), f);
            if (skip) load_vec<T>(reinterpret_cast<const T*>(&rs[u]), sk);
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
                const float4 k4 = coef[i * cstride];
                float v = (f[i] - k4.x) * k4.y + k4.z;
                if (do_silu) {
                    if constexpr (sizeof(T) == 2)
                        v = __fdividef(v, 1.0f + __expf(-v));
                    else
                        v = v / (1.0f + expf(-v));
                }
                v = v + k4.w;
                if (skip) v = v + sk[i];
                f[i] = (c0 + i < C) ? v : 0.0f;
            }
            store_vec<T>(y + (size_t(pp) * nvec + cv) * VEC, f, round_tf32 != 0);
        }
    }
}

// ---------------------------------------------------------------- pointwise
template <class T>
__global__ void silu_kernel(const T* __restrict__ x, T* __restrict__ y, long long nv, int r) {
    constexpr int VEC = Vec<T>::N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv;
         i += (long long)gridDim.x * blockDim.x) {
        float f[VEC];
        load_vec<T>(x + i * VEC, f);
#pragma unroll
        for (int k = 0; k < VEC; ++k) f[k] = f[k] / (1.0f + expf(-f[k]));
        store_vec<T>(y + i * VEC, f, r != 0);
    }
}

template <class T>
__global__ void add_kernel(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ o,
                           long long nv, int r) {
    constexpr int VEC = Vec<T>::N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv;
         i += (long long)gridDim.x * blockDim.x) {
        float a[VEC], b[VEC];
        load_vec<T>(x + i * VEC, a);
        load_vec<T>(y + i * VEC, b);
#pragma unroll
        for (int k = 0; k < VEC; ++k) a[k] = a[k] + b[k];
        store_vec<T>(o + i * VEC, a, r != 0);
    }
}

template <class T>
__global__ void add_channel_kernel(const T* __restrict__ x, const float* __restrict__ vec,
                                   const T* __restrict__ skip, T* __restrict__ o, long long pix,
                                   int ld, int r) {
    constexpr int VEC = Vec<T>::N;
    const int nvec = ld / VEC;
    const long long total = pix * nvec;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c0 = int(i % nvec) * VEC;
        float a[VEC];
        if (x) {
            load_vec<T>(x + i * VEC, a);
        } else {
#pragma unroll
            for (int k = 0; k < VEC; ++k) a[k] = 0.0f;
        }
#pragma unroll
        for (int k = 0; k < VEC; ++k) a[k] = x ? a[k] + vec[c0 + k] : vec[c0 + k];
        if (skip) {
            float b[VEC];
            load_vec<T>(skip + i * VEC, b);
#pragma unroll
            for (int k = 0; k < VEC; ++k) a[k] = a[k] + b[k];
        }
        store_vec<T>(o + i * VEC, a, r != 0);
    }
}

template <class T>
__global__ void upsample_kernel(const T* __restrict__ x, T* __restrict__ y, int rows, int W,
                                int ld) {
    constexpr int VEC = Vec<T>::N;
    const int nvec = ld / VEC;
    const long long total = (long long)rows * W * nvec;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int v = int(i % nvec);
        const long long p = i / nvec;
        const int xx = int(p % W), yy = int(p / W);
        const uint4 val = *reinterpret_cast<const uint4*>(x + p * ld + v * VEC);
        const long long W2 = 2LL * W;
        const long long o00 = ((2LL * yy) * W2 + 2 * xx) * ld + v * VEC;
        *reinterpret_cast<uint4*>(y + o00) = val;
        *reinterpret_cast<uint4*>(y + o00 + ld) = val;
        *reinterpret_cast<uint4*>(y + o00 + W2 * ld) = val;
        *reinterpret_cast<uint4*>(y + o00 + W2 * ld + ld) = val;
    }
}

// ---------------------------------------------------------------- attention helpers
template <class T>
__global__ void softmax_kernel(const float* __restrict__ S, int ns, long long lds, float scale,
                               T* __restrict__ P, long long ldp) {
    const int row = blockIdx.x;
    const float* s = S + (long long)row * lds;
    __shared__ float red[32];
    float mx = -INFINITY;
    for (int j = threadIdx.x; j < ns; j += blockDim.x) mx = fmaxf(mx, s[j] * scale);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    float sum = 0.0f;
    for (int j = threadIdx.x; j < ns; j += blockDim.x) sum += expf(s[j] * scale - mx);
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = 1.0f / red[0];
    T* pr = P + (long long)row * ldp;
    for (int j = threadIdx.x; j < ns; j += blockDim.x)
        pr[j] = from_float<T>(expf(s[j] * scale - mx) * inv, true);
}

template <class T>
__global__ void transpose_kernel(const T* __restrict__ V, int ns, int C, long long ldv,
                                 T* __restrict__ Vt, long long ldt) {
    __shared__ T tile[32][33];
    const int j0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int j = j0 + k, c = c0 + threadIdx.x;
        if (j < ns && c < C) tile[k][threadIdx.x] = V[(long long)j * ldv + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int c = c0 + k, j = j0 + threadIdx.x;
        if (j < ns && c < C) Vt[(long long)c * ldt + j] = tile[threadIdx.x][k];
    }
}

// ---------------------------------------------------------------- embeddings / projections
__global__ void time_projection_kernel(const TembLayer* __restrict__ layers,
                                       const __grid_constant__ EmbArg emb_arg) {
    extern __shared__ float emb[];
    const int dim = emb_arg.dim;
    for (int i = threadIdx.x; i < dim; i += blockDim.x) emb[i] = emb_arg.v[i];
    __syncthreads();
    const TembLayer L = layers[blockIdx.y];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nw = blockDim.x / 32;
    for (int c = blockIdx.x * nw + warp; c < L.C; c += gridDim.x * nw) {
        double acc = 0.0;
        for (int i = lane; i < dim; i += 32) acc += double(emb[i]) * double(L.W[(long long)c * dim + i]);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) L.out[c] = float(acc + double(L.b[c]));
    }
}

__global__ void time_projection_plan_kernel(const TembLayer* __restrict__ layers,
                                            const float* __restrict__ embs, int dim,
                                            float* __restrict__ table, int n_layers, int ldt) {
    extern __shared__ float emb[];
    const int step = blockIdx.z;
    for (int i = threadIdx.x; i < dim; i += blockDim.x) emb[i] = embs[(size_t)step * dim + i];
    __syncthreads();
    const TembLayer L = layers[blockIdx.y];
    float* out = table + ((size_t)step * n_layers + blockIdx.y) * ldt;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nw = blockDim.x / 32;
    for (int c = blockIdx.x * nw + warp; c < L.C; c += gridDim.x * nw) {
        double acc = 0.0;
        for (int i = lane; i < dim; i += 32) acc += double(emb[i]) * double(L.W[(long long)c * dim + i]);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[c] = float(acc + double(L.b[c]));
    }
}

__global__ void gemv_f64_kernel(const float* __restrict__ W, const float* __restrict__ b,
                                const float* __restrict__ x, int rows, int cols,
                                float* __restrict__ out) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nw = blockDim.x / 32;
    for (int r = blockIdx.x * nw + warp; r < rows; r += gridDim.x * nw) {
        double acc = 0.0;
        for (int i = lane; i < cols; i += 32) acc += double(x[i]) * double(W[(long long)r * cols + i]);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[r] = float(acc + double(b[r]));
    }
}

// ---------------------------------------------------------------- sampler / layout
template <class T>
__global__ void ddim_kernel(const float* __restrict__ x, const float* __restrict__ eps,
                            float* __restrict__ xo, long long n, int C, double sa, double s1,
                            double sn, double s1n, T* __restrict__ stem, int stem_ld) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double e = double(eps[i]);
        const double x0 = __ddiv_rn(__dsub_rn(double(x[i]), __dmul_rn(s1, e)), sa);
        const float v = float(__dadd_rn(__dmul_rn(sn, x0), __dmul_rn(s1n, e)));
        xo[i] = v;
        if (stem) {
            const long long p = i / C;
            stem[p * stem_ld + (i - p * C)] = from_float<T>(v, true);
        }
    }
}

template <class T>
__global__ void nchw_to_nhwc_kernel(const float* __restrict__ src, int C, int H, int W, int r0,
                                    int rows, T* __restrict__ dst, int ld, int r) {
    const long long total = (long long)rows * W * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = int(i % C);
        const long long p = i / C;
        const int xx = int(p % W), yy = int(p / W);
        dst[p * ld + c] = from_float<T>(src[((long long)c * H + r0 + yy) * W + xx], r != 0);
    }
}

template <class T>
__global__ void nhwc_to_nchw_kernel(const T* __restrict__ src, int ld, int C, int rows, int W,
                                    float* __restrict__ dst, int* nonfinite) {
    const long long total = (long long)rows * W * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int xx = int(i % W);
        const long long rest = i / W;
        const int yy = int(rest % rows), c = int(rest / rows);
        const float v = to_float(src[((long long)yy * W + xx) * ld + c]);
        dst[i] = v;
        if (nonfinite && !isfinite(v)) atomicExch(nonfinite, 1);
    }
}

template <class T>
__global__ void crop_kernel(const float* __restrict__ src, int C, int H, int W, int y0, int x0,
                            int rows, int cols, T* __restrict__ dst, int ld, int r) {
    const long long total = (long long)rows * cols * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = int(i % C);
        const long long p = i / C;
        const int xx = int(p % cols), yy = int(p / cols);
        dst[p * ld + c] = from_float<T>(src[((long long)c * H + y0 + yy) * W + x0 + xx], r != 0);
    }
}

__global__ void scatter_patch_kernel(const float* __restrict__ patch, int C, int rows, int cols,
                                     float* __restrict__ dst, int H, int W, int y0, int x0,
                                     int* nonfinite) {
    const long long total = (long long)rows * cols * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = int(i % C);
        const long long p = i / C;
        const int xx = int(p % cols), yy = int(p / cols);
        const float v = patch[i];
        dst[((long long)c * H + y0 + yy) * W + x0 + xx] = v;
        if (nonfinite && !isfinite(v)) atomicExch(nonfinite, 1);
    }
}

template <class T>
__global__ void f32_to_elem_kernel(const float* __restrict__ s, T* __restrict__ d, long long n, int r) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        d[i] = from_float<T>(s[i], r != 0);
}
template <class T>
__global__ void elem_to_f32_kernel(const T* __restrict__ s, float* __restrict__ d, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        d[i] = to_float(s[i]);
}

#define DISPATCH(e, ...)                          \
    do {                                          \
        if ((e) == Elem::BF16) {                  \
            using T = bf16;                       \
            __VA_ARGS__;                          \
        } else {                                  \
            using T = float;                      \
            __VA_ARGS__;                          \
        }                                         \
    } while (0)

}  // namespace

int gn_stats_blocks(long long pix) { return int((pix + kGnPixels - 1) / kGnPixels); }

void gn_stats(Elem e, const void* x, long long pix, int C, int ld, int groups, double count,
              double* partial, unsigned int* ticket, double* out, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    if (C % VEC || ld % VEC || C % groups)
        throw std::invalid_argument("group_stats: channels must be a multiple of the vector width");
    const int nvec = C / VEC;
    const int L = std::max(1, kGnThreads / nvec);
    const size_t smem = size_t(2) * L * C * 4 + size_t(2) * C * 8;
    DISPATCH(e, gn_stats_kernel<T><<<gn_stats_blocks(pix), kGnThreads, smem, s>>>(
                    static_cast<const T*>(x), pix, C, ld, groups, count, partial, ticket, out));
    CUDA_CHECK(cudaGetLastError());
}

void gn_apply(Elem e, const void* x, void* y, long long pix, int C, int ld, int groups,
              const GnCombine& cb, const float* gamma, const float* beta, bool do_silu,
              const float* temb, const void* skip, bool round_tf32, cudaStream_t s) {
    if (groups > 1024) throw std::invalid_argument("group_norm_apply: too many groups");
    const int VEC = e == Elem::BF16 ? 8 : 4;
    if (pix * (ld / VEC) >= (1LL << 31)) throw std::invalid_argument("group_norm_apply: band too large");
    // block = vx channel vectors x vy pixel lanes (~256 threads); grid fills ~4 waves of SMs
    const int nvec = ld / VEC;
    int vx = nvec;
    while (vx > 128 && vx % 2 == 0) vx /= 2;
    if (vx > 128) vx = 128;
    const int gx = (nvec + vx - 1) / vx;
    const int vy = std::max(1, 256 / vx);
    // one wave of ~4 blocks per SM; each thread keeps 4 vectors in flight per iteration
    const long long rows_needed = (pix + vy - 1) / vy;
    const int gy = int(std::max<long long>(1, std::min<long long>(rows_needed, (148LL * 4) / gx)));
    DISPATCH(e, gn_apply_2d_kernel<T><<<dim3(gx, gy), dim3(vx, vy), 0, s>>>(
                    static_cast<const T*>(x), static_cast<T*>(y), int(pix), C, ld, groups, cb, gamma,
                    beta, do_silu ? 1 : 0, temb, static_cast<const T*>(skip), round_tf32 ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void silu(Elem e, const void* x, void* y, long long n, bool r, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    DISPATCH(e, silu_kernel<T><<<grid_for(n / VEC, 256), 256, 0, s>>>(
                    static_cast<const T*>(x), static_cast<T*>(y), n / VEC, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void add(Elem e, const void* x, const void* y, void* o, long long n, bool r, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    DISPATCH(e, add_kernel<T><<<grid_for(n / VEC, 256), 256, 0, s>>>(
                    static_cast<const T*>(x), static_cast<const T*>(y), static_cast<T*>(o),
                    n / VEC, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void add_channel(Elem e, const void* x, const float* vec, const void* skip, void* o,
                 long long pix, int ld, bool, bool r, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    DISPATCH(e, add_channel_kernel<T><<<grid_for(pix * ld / VEC, 256), 256, 0, s>>>(
                    static_cast<const T*>(x), vec, static_cast<const T*>(skip), static_cast<T*>(o),
                    pix, ld, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void upsample2x(Elem e, const void* x, void* y, int rows, int W, int ld, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    DISPATCH(e, upsample_kernel<T><<<grid_for((long long)rows * W * ld / VEC, 256), 256, 0, s>>>(
                    static_cast<const T*>(x), static_cast<T*>(y), rows, W, ld));
    CUDA_CHECK(cudaGetLastError());
}

void softmax_rows(Elem e, const float* S, int m, int ns, long long lds, float scale, void* P,
                  long long ldp, cudaStream_t s) {
    DISPATCH(e, softmax_kernel<T><<<m, 256, 0, s>>>(S, ns, lds, scale, static_cast<T*>(P), ldp));
    CUDA_CHECK(cudaGetLastError());
}

void transpose(Elem e, const void* V, int ns, int C, long long ldv, void* Vt, long long ldt,
               cudaStream_t s) {
    dim3 grid((ns + 31) / 32, (C + 31) / 32), block(32, 8);
    DISPATCH(e, transpose_kernel<T><<<grid, block, 0, s>>>(static_cast<const T*>(V), ns, C, ldv,
                                                          static_cast<T*>(Vt), ldt));
    CUDA_CHECK(cudaGetLastError());
}

void time_projection(const TembLayer* layers_dev, int n_layers, int max_c, const float* emb,
                     int dim, cudaStream_t s) {
    if (n_layers == 0) return;
    if (dim > kMaxEmb) throw std::invalid_argument("timestep_embedding: dim too large for the B200 path");
    EmbArg arg;
    arg.dim = dim;
    for (int i = 0; i < dim; ++i) arg.v[i] = emb[i];
    dim3 grid(std::max(1, (max_c + 7) / 8), n_layers);
    time_projection_kernel<<<grid, 256, dim * sizeof(float), s>>>(layers_dev, arg);
    CUDA_CHECK(cudaGetLastError());
}

void time_projection_plan(const TembLayer* layers_dev, int n_layers, int max_c,
                          const float* embs_dev, int n_steps, int dim, float* table, int ldt,
                          cudaStream_t s) {
    if (n_layers == 0 || n_steps == 0) return;
    dim3 grid(std::max(1, (max_c + 7) / 8), n_layers, n_steps);
    time_projection_plan_kernel<<<grid, 256, dim * sizeof(float), s>>>(layers_dev, embs_dev, dim,
                                                                        table, n_layers, ldt);
    CUDA_CHECK(cudaGetLastError());
}

void gemv_f64(const float* W, const float* b, const float* x, int rows, int cols, float* out,
              cudaStream_t s) {
    gemv_f64_kernel<<<std::max(1, std::min(148, (rows + 7) / 8)), 256, 0, s>>>(W, b, x, rows, cols,
                                                                              out);
    CUDA_CHECK(cudaGetLastError());
}

void ddim_update(const float* x, const float* eps, float* xo, long long n, int C, double abar_t,
                 double abar_n, Elem e, void* stem, int stem_ld, cudaStream_t s) {
    const double sa = std::sqrt(abar_t), s1 = std::sqrt(1.0 - abar_t);
    const double sn = std::sqrt(abar_n), s1n = std::sqrt(1.0 - abar_n);
    DISPATCH(e, ddim_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(x, eps, xo, n, C, sa, s1, sn, s1n,
                                                                static_cast<T*>(stem), stem_ld));
    CUDA_CHECK(cudaGetLastError());
}

void nchw_to_nhwc(const float* src, int C, int H, int W, int r0, int rows, Elem e, void* dst,
                  int ld, bool r, cudaStream_t s) {
    DISPATCH(e, nchw_to_nhwc_kernel<T><<<grid_for((long long)rows * W * C, 256), 256, 0, s>>>(
                    src, C, H, W, r0, rows, static_cast<T*>(dst), ld, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void nhwc_to_nchw(Elem e, const void* src, int ld, int C, int rows, int W, float* dst,
                  int* nonfinite, cudaStream_t s) {
    DISPATCH(e, nhwc_to_nchw_kernel<T><<<grid_for((long long)rows * W * C, 256), 256, 0, s>>>(
                    static_cast<const T*>(src), ld, C, rows, W, dst, nonfinite));
    CUDA_CHECK(cudaGetLastError());
}

void nhwc_f32_to_nchw(const float* src, int C, int rows, int W, float* dst, int* nonfinite,
                      cudaStream_t s) {
    nhwc_to_nchw_kernel<float><<<grid_for((long long)rows * W * C, 256), 256, 0, s>>>(
        src, C, C, rows, W, dst, nonfinite);
    CUDA_CHECK(cudaGetLastError());
}

void crop_nchw_to_nhwc(const float* src, int C, int H, int W, int y0, int x0, int rows, int cols,
                       Elem e, void* dst, int ld, bool r, cudaStream_t s) {
    DISPATCH(e, crop_kernel<T><<<grid_for((long long)rows * cols * C, 256), 256, 0, s>>>(
                    src, C, H, W, y0, x0, rows, cols, static_cast<T*>(dst), ld, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void scatter_nhwc_to_nchw(const float* patch, int C, int rows, int cols, float* dst, int H, int W,
                          int y0, int x0, int* nonfinite, cudaStream_t s) {
    scatter_patch_kernel<<<grid_for((long long)rows * cols * C, 256), 256, 0, s>>>(
        patch, C, rows, cols, dst, H, W, y0, x0, nonfinite);
    CUDA_CHECK(cudaGetLastError());
}

void f32_to_elem(const float* src, Elem e, void* dst, long long n, bool r, cudaStream_t s) {
    DISPATCH(e, f32_to_elem_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(src, static_cast<T*>(dst), n,
                                                                       r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void elem_to_f32(Elem e, const void* src, float* dst, long long n, cudaStream_t s) {
    DISPATCH(e, elem_to_f32_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(static_cast<const T*>(src),
                                                                       dst, n));
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace pp
