// HBM-bound kernels (see kernels.hpp).  128-bit vectorised NHWC access; all
// reductions are fixed-order (no float atomics) so every run is bit-deterministic.
#include "kernels.hpp"
#include "pdl.cuh"
#include "util.hpp"

#include <cuda_bf16.h>
#include <cuda_fp16.h>

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
__device__ __forceinline__ void gn_use_of_multi(const GnCombine& cb, int G, int g, float& mu,
                                                float& inv, bool& neg);
// Fast path: one band's own fresh statistics.
__device__ __forceinline__ void gn_use_of(const GnCombine& cb, int G, int g, float& mu, float& inv,
                                          bool& neg) {
    if (cb.mode == GN_USE_LOCAL || (cb.mode == GN_USE_GLOBAL && cb.n == 1)) {
        const double m = cb.fresh[g * 2], q = cb.fresh[g * 2 + 1];
        const double var = __dsub_rn(q, __dmul_rn(m, m));
        neg = var < 0.0;
        mu = float(m);
        inv = float(1.0 / sqrt(__dadd_rn(fmax(var, 0.0), double(cb.eps))));
        return;
    }
    gn_use_of_multi(cb, G, g, mu, inv, neg);
}

__device__ __forceinline__ void gn_use_of_multi(const GnCombine& cb, int G, int g, float& mu,
                                                float& inv, bool& neg) {
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

// One pass over a band for GroupNorm: APPLY computes y = GN(x) [-> SiLU] [+ temb] [+ skip]
// (group_norm_apply, tensor.cpp:240-277, with the fused SiLU / AddTimeEmb / AddSkip of the
// following layers); STATS folds the group statistics of the stored values (y, or x when
// !APPLY) into out[G][2] = (mean, mean_sq) (group_stats, tensor.cpp:203-235).
// Thread (tx, ty) owns one 16-byte channel vector and kGnU pixels (all loads in flight at
// once); its GN coefficients live in registers (two groups at most per vector).  Statistics:
// fp32 per-thread sums over kGnU pixels, fp64 above, fixed-order block reduction and a
// fixed-order fold by the last block -> deterministic.  gamma / beta are weights and are
// loaded before griddepcontrol.wait; everything else after it.
constexpr int kGnU = 4;         // pixels per thread (apply)
constexpr int kGnUStats = 8;   // pixels per thread with statistics (fewer blocks to fold)

constexpr int kGnRange = 32;   // blocks per first-level statistics fold

// gpu-scope acq_rel ticket (release: cumulative over the block's partials stored before the
// preceding __syncthreads; acquire: the folding block sees the other blocks' partials)
__device__ __forceinline__ unsigned int atom_add_acq_rel(unsigned int* p, unsigned int v) {
    unsigned int old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// dst[g] = sum_{k < n} src[k * G + g] / div (double2 = (sum, sum_sq)), fixed order: thread
// (part, g) sums k = part, part + parts, ...; the parts are added in order through smem
// (scratch >= 2 * parts * G doubles).  Reads with ld.global.cg (partials of other blocks).
__device__ void fold_fixed(const double2* src, int n, int G, double2* dst, double div, int tid,
                           int nthr, double* scratch) {
    const int parts = max(1, min(8, nthr / G));
    if (tid < parts * G) {
        const int g = tid % G, pt = tid / G;
        double a = 0.0, b = 0.0;
        for (int k0 = pt; k0 < n; k0 += 8 * parts) {
            double2 v[8];   // one round of loads covers a 32-block range (parts >= 4)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = k0 + u * parts;
                v[u] = k < n ? __ldcg(src + size_t(k) * G + g) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                a += v[u].x;
                b += v[u].y;
            }
        }
        scratch[(pt * G + g) * 2] = a;
        scratch[(pt * G + g) * 2 + 1] = b;
    }
    __syncthreads();
    for (int g = tid; g < G; g += nthr) {
        double a = 0.0, b = 0.0;
        for (int pt = 0; pt < parts; ++pt) {
            a += scratch[(pt * G + g) * 2];
            b += scratch[(pt * G + g) * 2 + 1];
        }
        dst[g] = make_double2(a / div, b / div);
    }
    __syncthreads();
}

template <class T, bool APPLY, bool STATS, int U>
__global__ void __launch_bounds__(256, (STATS ? 2 : 3))
    gn_pass_kernel(const T* __restrict__ x, T* __restrict__ y, int pix, int C, int ld, int G,
                   const GnCombine cb, const float* __restrict__ gamma,
                   const float* __restrict__ beta, int do_silu, const float* __restrict__ temb,
                   const T* __restrict__ skip, int round_tf32, const GnStatsOut so, int up_w) {
    constexpr int VEC = Vec<T>::N;
    const int vx = blockDim.x, vy = blockDim.y;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * vx + tx;
    const int nthr = vx * vy;
    const int nvec = ld / VEC;
    const int cv = blockIdx.x * vx + tx;
    const bool active = cv < nvec;
    const int c0 = cv * VEC;
    const int cb0 = blockIdx.x * vx * VEC;    // first channel of this block
    const int bch = vx * VEC;                 // channels of this block
    const bool full = active && c0 + VEC <= C;
    float sc[VEC], sh[VEC], tb[VEC];
    if (APPLY) {   // weights: safe to read before the previous kernel completes
        if (full) {
            load_vec<float>(gamma + c0, sc);
            load_vec<float>(beta + c0, sh);
            if constexpr (VEC == 8) {
                load_vec<float>(gamma + c0 + 4, sc + 4);
                load_vec<float>(beta + c0 + 4, sh + 4);
            }
        } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
                const bool ok = active && c0 + i < C;
                sc[i] = ok ? gamma[c0 + i] : 0.0f;
                sh[i] = ok ? beta[c0 + i] : 0.0f;
            }
        }
    }
    pdl_wait();
    pdl_trigger();
    const int pstride = vy * gridDim.y;
    const int p_first = blockIdx.y * vy + ty;
    if (APPLY) {
        // (mean, 1/std) of the groups this block touches, one thread per group
        __shared__ float s_mi[2 * 1024];
        const int cpg = C / G;
        const int g_first = min(cb0, C - 1) / cpg;
        const int n_g = (min(cb0 + bch, C) - 1) / cpg - g_first + 1;
        for (int j = tid; j < n_g; j += nthr) {
            float m_, i_;
            bool neg;
            gn_use_of(cb, G, g_first + j, m_, i_, neg);
            // group_norm_apply contract (tensor.cpp:256-259)
            if (neg && cb.err) atomicExch(cb.err, 1);
            s_mi[2 * j] = m_;
            s_mi[2 * j + 1] = i_;
        }
        if (temb) {
            if (full) {
                load_vec<float>(temb + c0, tb);
                if constexpr (VEC == 8) load_vec<float>(temb + c0 + 4, tb + 4);
            } else {
#pragma unroll
                for (int i = 0; i < VEC; ++i) tb[i] = (active && c0 + i < C) ? temb[c0 + i] : 0.0f;
            }
        } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) tb[i] = 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < VEC; ++i) {   // y = x * sc + sh  (sc = gamma / std, sh = beta - mean * sc)
            const int j = min(c0 + i, C - 1) / cpg - g_first;
            sc[i] *= s_mi[2 * j + 1];
            sh[i] = fmaf(-s_mi[2 * j], sc[i], sh[i]);
        }
    }
    // first round of loads
    const uint4* xv = reinterpret_cast<const uint4*>(x) + cv;
    const uint4* sv = reinterpret_cast<const uint4*>(skip) + cv;
    uint4 rx[U], rs[U];
    if (active) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int pp = p_first + u * pstride;
            if (pp < pix) {
                rx[u] = __ldcs(xv + size_t(pp) * nvec);
                if (APPLY && skip) rs[u] = __ldcs(sv + size_t(pp) * nvec);
            }
        }
    }
    float ss[VEC], sq[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) ss[i] = sq[i] = 0.0f;
    if (active) {
        for (int p = p_first; p < pix; p += U * pstride) {
            if (p != p_first) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int pp = p + u * pstride;
                    if (pp < pix) {
                        rx[u] = __ldcs(xv + size_t(pp) * nvec);
                        if (APPLY && skip) rs[u] = __ldcs(sv + size_t(pp) * nvec);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int pp = p + u * pstride;
                if (pp >= pix) continue;
                float f[VEC];
                load_vec<T>(reinterpret_cast<const T*>(&rx[u]), f);
                if (APPLY) {
                    float sk[VEC];
                    if (skip) load_vec<T>(reinterpret_cast<const T*>(&rs[u]), sk);
#pragma unroll
                    for (int i = 0; i < VEC; ++i) f[i] = fmaf(f[i], sc[i], sh[i]);
                    if (do_silu) {
                        if constexpr (sizeof(T) == 2) {
                            // bf16 output: silu(v) = h + h tanh(h), h = v / 2, with one
                            // tanh.approx.f32 (MUFU.TANH) per element (the SFU-bound ex2 + rcp
                            // form was 2 MUFU ops); |err| ~ 2^-11, below the bf16 rounding
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                const float h = 0.5f * f[i];
                                float t;
                                asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
                                f[i] = fmaf(h, t, h);
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < VEC; ++i) f[i] = f[i] / (1.0f + expf(-f[i]));
                        }
                    }
#pragma unroll
                    for (int i = 0; i < VEC; ++i) {
                        float v = f[i] + tb[i];
                        if (skip) v = v + sk[i];
                        f[i] = (c0 + i < C) ? v : 0.0f;
                    }
                    uint4 o;
                    store_vec<T>(reinterpret_cast<T*>(&o), f, round_tf32 != 0);
                    if (up_w) {
                        // fused nearest 2x upsample (upsample_nearest2x, tensor.cpp:323-334):
                        // low-res pixel (py, px) -> the 2x2 block at (2py, 2px) of a 2W-wide map
                        const int py = pp / up_w, px = pp - py * up_w;
                        const size_t q = (size_t(2 * py) * (2 * up_w) + 2 * px) * nvec + cv;
                        const size_t row = size_t(2 * up_w) * nvec;
                        uint4* yv = reinterpret_cast<uint4*>(y);
                        yv[q] = o;
                        yv[q + nvec] = o;
                        yv[q + row] = o;
                        yv[q + row + nvec] = o;
                    } else {
                        *reinterpret_cast<uint4*>(y + (size_t(pp) * nvec + cv) * VEC) = o;
                    }
                    if (STATS) load_vec<T>(reinterpret_cast<const T*>(&o), f);   // stored values
                }
                if (STATS) {
#pragma unroll
                    for (int i = 0; i < VEC; ++i) {
                        ss[i] += f[i];
                        sq[i] = fmaf(f[i], f[i], sq[i]);
                    }
                }
            }
        }
    }
    if (!STATS) return;
    // ---- block reduction: per channel over ty (fp64, fixed order), then per group
    __shared__ float r_s[256 * VEC], r_q[256 * VEC];
    __shared__ double c_sq2[2048];
    double* c_s = c_sq2;
    double* c_q = c_sq2 + 1024;
    __shared__ bool is_last;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
        r_s[(ty * vx + tx) * VEC + i] = ss[i];
        r_q[(ty * vx + tx) * VEC + i] = sq[i];
    }
    __syncthreads();
    for (int c = tid; c < bch; c += nthr) {
        double a = 0.0, b = 0.0;
        for (int r = 0; r < vy; ++r) {
            a += double(r_s[r * bch + c]);
            b += double(r_q[r * bch + c]);
        }
        c_s[c] = a;
        c_q[c] = b;
    }
    __syncthreads();
    const int Gs = so.G;
    const int cpg2 = C / Gs;
    const size_t blk = size_t(blockIdx.y) * gridDim.x + blockIdx.x;
    for (int g = tid; g < Gs; g += nthr) {
        double a = 0.0, b = 0.0;
        const int lo = max(g * cpg2, cb0), hi = min((g + 1) * cpg2, min(cb0 + bch, C));
        for (int c = lo; c < hi; ++c) {
            a += c_s[c - cb0];
            b += c_q[c - cb0];
        }
        reinterpret_cast<double2*>(so.partial)[blk * Gs + g] = make_double2(a, b);
    }
    // ---- two-level fixed-order fold: the last block of each range of kGnRange blocks (by
    // block index) folds that range; the last range folder folds the range sums.  Counters:
    // ticket[0] = ranges done, ticket[1 + r] = blocks of range r done (each reset by its folder).
    const int nblk = gridDim.x * gridDim.y;
    const int nrange = (nblk + kGnRange - 1) / kGnRange;
    const int r = int(blk / kGnRange);
    const int rsize = min(kGnRange, nblk - r * kGnRange);
    double2* part1 = reinterpret_cast<double2*>(so.partial);
    double2* part2 = part1 + size_t(nblk) * Gs;
    __syncthreads();
    if (tid == 0) {
        is_last = atom_add_acq_rel(so.ticket + 1 + r, 1u) == unsigned(rsize - 1);
    }
    __syncthreads();
    if (!is_last) return;
    fold_fixed(part1 + size_t(r) * kGnRange * Gs, rsize, Gs, part2 + size_t(r) * Gs, 1.0, tid, nthr,
               c_s);
    if (tid == 0) so.ticket[1 + r] = 0u;
    __syncthreads();
    if (tid == 0) {
        is_last = atom_add_acq_rel(so.ticket, 1u) == unsigned(nrange - 1);
    }
    __syncthreads();
    if (!is_last) return;
    fold_fixed(part2, nrange, Gs, reinterpret_cast<double2*>(so.out), so.count, tid, nthr, c_s);
    if (tid == 0) *so.ticket = 0u;
}

// ---------------------------------------------------------------- context exchange
__global__ void __launch_bounds__(256) copy_chunks_kernel(const CopyChunk* __restrict__ chunks) {
    const CopyChunk c = chunks[blockIdx.x];
    const uint4* src = static_cast<const uint4*>(c.src);
    uint4* dst = static_cast<uint4*>(c.dst);
    const int n = int(c.bytes / 16);
    for (int i = threadIdx.x; i < n; i += 256) dst[i] = __ldcg(src + i);
}

__global__ void __launch_bounds__(256) copy_rows_kernel(const RowCopies c, long long nv) {
    pdl_wait();
    pdl_trigger();
    const int k = blockIdx.y;
    if (!c.src[k]) return;
    const uint4* src = static_cast<const uint4*>(c.src[k]);
    uint4* dst = static_cast<uint4*>(c.dst[k]);
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < nv; i += 256LL * gridDim.x)
        dst[i] = __ldcg(src + i);
}

// ---------------------------------------------------------------- pointwise
template <class T>
__global__ void silu_kernel(const T* __restrict__ x, T* __restrict__ y, long long nv, int r) {
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
__global__ void transpose_kernel(const T* __restrict__ V, int ns, int C, long long ldv,
                                 T* __restrict__ Vt, long long ldt) {
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        d[i] = from_float<T>(s[i], r != 0);
}
template <class T>
__global__ void elem_to_f32_kernel(const T* __restrict__ s, float* __restrict__ d, long long n) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        d[i] = to_float(s[i]);
}


// ---------------------------------------------------------------- attention (tcgen05 path)
// attention (proj/src/tensor.cpp:163-199) runs as S GEMM -> P with the softmax in the GEMM
// epilogue (P = exp(S scale - tile max) from the TMEM accumulator, tile max per row and key
// tile) -> attn_rescale -> PV GEMM with 1/l in its epilogue (V read MN-major in bf16).
// attn_rescale, one warp per query row: m = max over the key tiles' maxima, P of tile t *=
// 2^(max_t - m) (the tile holding the row max is left as is), l = sum of the row's stored P
// (what the PV GEMM multiplies; lanes sum fixed column residues, then a fixed xor tree ->
// deterministic) -> row_scale = 1 / l.
template <class T>
__global__ void __launch_bounds__(256) attn_rescale_kernel(T* __restrict__ P, long long ldp, int m,
                                                           int s, const float* __restrict__ rowmax,
                                                           int n_tiles, int block_n, int ld_rm,
                                                           float* __restrict__ row_scale,
                                                           int round_tf32) {
    constexpr int VEC = Vec<T>::N;
    extern __shared__ float s_alpha[];   // [8 warps][n_tiles]
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int r = blockIdx.x * 8 + wib;
    if (r >= m) return;
    float* alpha = s_alpha + wib * n_tiles;
    float mx = -INFINITY;
    for (int t = lane; t < n_tiles; t += 32) mx = fmaxf(mx, rowmax[(long long)t * ld_rm + r]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int t = lane; t < n_tiles; t += 32) {
        const float d = rowmax[(long long)t * ld_rm + r] - mx;
        float a;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(d));
        alpha[t] = d == 0.0f ? 1.0f : a;
    }
    __syncwarp();
    T* row = P + (long long)r * ldp;
    const int nv = (s + VEC - 1) / VEC;   // vectors holding keys (the padding stays zero)
    float sum = 0.0f;
    for (int v0 = lane; v0 < nv; v0 += 32 * 4) {
        uint4 raw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int v = v0 + u * 32;
            if (v < nv) raw[u] = *reinterpret_cast<const uint4*>(row + (long long)v * VEC);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int v = v0 + u * 32;
            if (v >= nv) continue;
            const float a = alpha[(v * VEC) / block_n];
            float f[VEC];
            load_vec<T>(reinterpret_cast<const T*>(&raw[u]), f);
            if (a != 1.0f) {
#pragma unroll
                for (int i = 0; i < VEC; ++i) f[i] *= a;
                uint4 o;
                store_vec<T>(reinterpret_cast<T*>(&o), f, round_tf32 != 0);
                *reinterpret_cast<uint4*>(row + (long long)v * VEC) = o;
                load_vec<T>(reinterpret_cast<const T*>(&o), f);   // the stored values
            }
#pragma unroll
            for (int i = 0; i < VEC; ++i) sum += f[i];
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) row_scale[r] = 1.0f / sum;
}

// ---------------------------------------------------------------- stem im2col
// The stem conv (conv2d_region, proj/src/tensor.cpp:79-130, 4 -> 320 channels) as a plain
// tcgen05 GEMM with K = 9 taps x 4 channels in ONE 128-byte K block: this kernel gathers the
// 36 values of every output pixel (tap-major, channel-minor; zero outside the image, the halo
// rows come from the padded band) into out[pixel][kpad] (the padding columns stay zero).
template <class T>
__global__ void __launch_bounds__(256) stem_im2col_kernel(const T* __restrict__ in, int rows, int W,
                                                          int ld_in, int C_in, T* __restrict__ out,
                                                          int kpad) {
    pdl_wait();
    pdl_trigger();
    const long long n = (long long)rows * W * 9;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long p = i / 9;
        const int tap = int(i - p * 9), ky = tap / 3, kx = tap - 3 * ky;
        const int y = int(p / W), x = int(p - (long long)y * W);
        const int xx = x + kx - 1;
        T v[4];
        if (xx >= 0 && xx < W) {
            const T* src = in + ((long long)(y + ky) * W + xx) * ld_in;   // padded row y + ky
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] = c < C_in ? src[c] : from_float<T>(0.0f, false);
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] = from_float<T>(0.0f, false);
        }
        T* dst = out + p * kpad + tap * 4;
        if constexpr (sizeof(T) == 2) {
            *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(v);
        } else {
            *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(v);
        }
    }
}

__global__ void cfg_combine_kernel(float* out, const float* ec, const float* eu, long long n,
                                   double scale) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double u = double(eu[i]);
        out[i] = float(__dadd_rn(u, __dmul_rn(scale, __dsub_rn(double(ec[i]), u))));
    }
}

// --stress-sched: a single thread sleeping `us` microseconds on the stream (scheduling noise)
__global__ void sleep_kernel(unsigned int us) {
    for (unsigned int i = 0; i < us; ++i) __nanosleep(1000);
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

// Launch shape of gn_pass_kernel: block = vx channel vectors x vy pixel lanes (~256
// threads), grid.y sized so every thread owns kGnU pixels (one round of loads in flight),
// capped at ~8 resident blocks per SM.
struct GnShape {
    dim3 grid, block;
};
GnShape gn_shape(Elem e, long long pix, int ld, int U, int max_blocks = 1184) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    const int nvec = ld / VEC;
    int vx = nvec;
    while (vx > 128 && vx % 2 == 0) vx /= 2;
    if (vx > 128) vx = 128;
    const int gx = (nvec + vx - 1) / vx;
    const int vy = std::max(1, 256 / vx);
    const long long want = (pix + (long long)vy * U - 1) / ((long long)vy * U);
    const int gy = int(std::max<long long>(1, std::min<long long>(want, std::max(1, max_blocks / gx))));
    return {dim3(gx, gy), dim3(vx, vy)};
}

// One wave of gn_pass blocks: `per_sm` resident blocks (the __launch_bounds__ minimum) on
// every SM of the current device.  A grid larger than one wave leaves a partial second wave
// whose blocks each pay a full load round trip; capping grid.y to one wave makes the threads
// loop instead (measured: 34.10 vs 34.65 ms per 1024^2 generation).
int gn_wave_blocks(int per_sm) {
    static int sms_of[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& sms = sms_of[dev & 63];
    if (!sms && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
    return std::max(1, std::min(1184, per_sm * sms));
}

// >= gx * gy of every gn_shape, plus the second-level range sums
int gn_stats_blocks(long long) { return 1184 + 1184 + 80; }

void gn_stats(Elem e, const void* x, long long pix, int C, int ld, int groups, double count,
              double* partial, unsigned int* ticket, double* out, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    if (C % VEC || ld % VEC || C % groups)
        throw std::invalid_argument("group_stats: channels must be a multiple of the vector width");
    if (pix * (ld / VEC) >= (1LL << 31)) throw std::invalid_argument("group_stats: band too large");
    const GnShape sh = gn_shape(e, pix, ld, kGnUStats, gn_wave_blocks(2));
    GnStatsOut so;
    so.G = groups;
    so.count = count;
    so.partial = partial;
    so.ticket = ticket;
    so.out = out;
    GnCombine cb{};
    DISPATCH(e, launch_pdl(gn_pass_kernel<T, false, true, kGnUStats>, sh.grid, sh.block, 0, s, 1,
                           static_cast<const T*>(x), static_cast<T*>(nullptr), int(pix), C, ld,
                           groups, cb, static_cast<const float*>(nullptr),
                           static_cast<const float*>(nullptr), 0, static_cast<const float*>(nullptr),
                           static_cast<const T*>(nullptr), 0, so, 0));
    CUDA_CHECK(cudaGetLastError());
}

void gn_apply(Elem e, const void* x, void* y, long long pix, int C, int ld, int groups,
              const GnCombine& cb, const float* gamma, const float* beta, bool do_silu,
              const float* temb, const void* skip, bool round_tf32, cudaStream_t s,
              const GnStatsOut* out_stats, int up_w) {
    if (groups > 1024) throw std::invalid_argument("group_norm_apply: too many groups");
    const int VEC = e == Elem::BF16 ? 8 : 4;
    if (pix * (ld / VEC) >= (1LL << 31)) throw std::invalid_argument("group_norm_apply: band too large");
    const bool st = out_stats && out_stats->G > 0;
    const GnShape sh = gn_shape(e, pix, ld, st ? kGnUStats : kGnU,
                                gn_wave_blocks(st ? 2 : 3));
    if (st) {
        if (C % out_stats->G) throw std::invalid_argument("group_stats: channels not divisible by groups");
        DISPATCH(e, launch_pdl(gn_pass_kernel<T, true, true, kGnUStats>, sh.grid, sh.block, 0, s, 1,
                               static_cast<const T*>(x), static_cast<T*>(y), int(pix), C, ld, groups,
                               cb, gamma, beta, do_silu ? 1 : 0, temb, static_cast<const T*>(skip),
                               round_tf32 ? 1 : 0, *out_stats, up_w));
    } else {
        DISPATCH(e, launch_pdl(gn_pass_kernel<T, true, false, kGnU>, sh.grid, sh.block, 0, s, 1,
                               static_cast<const T*>(x), static_cast<T*>(y), int(pix), C, ld, groups,
                               cb, gamma, beta, do_silu ? 1 : 0, temb, static_cast<const T*>(skip),
                               round_tf32 ? 1 : 0, GnStatsOut{}, up_w));
    }
    CUDA_CHECK(cudaGetLastError());
}

void silu(Elem e, const void* x, void* y, long long n, bool r, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    DISPATCH(e, launch_pdl(silu_kernel<T>, dim3(grid_for(n / VEC, 256)), dim3(256), 0, s, 1, 
                    static_cast<const T*>(x), static_cast<T*>(y), n / VEC, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void add(Elem e, const void* x, const void* y, void* o, long long n, bool r, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    DISPATCH(e, launch_pdl(add_kernel<T>, dim3(grid_for(n / VEC, 256)), dim3(256), 0, s, 1, 
                    static_cast<const T*>(x), static_cast<const T*>(y), static_cast<T*>(o),
                    n / VEC, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void add_channel(Elem e, const void* x, const float* vec, const void* skip, void* o,
                 long long pix, int ld, bool, bool r, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    DISPATCH(e, launch_pdl(add_channel_kernel<T>, dim3(grid_for(pix * ld / VEC, 256)), dim3(256), 0, s, 1, 
                    static_cast<const T*>(x), vec, static_cast<const T*>(skip), static_cast<T*>(o),
                    pix, ld, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void copy_chunks(const CopyChunk* chunks, int n, cudaStream_t s) {
    if (n <= 0) return;
    copy_chunks_kernel<<<n, 256, 0, s>>>(chunks);
    CUDA_CHECK(cudaGetLastError());
}

void copy_rows(const RowCopies& c, unsigned long long bytes, cudaStream_t s) {
    int k = 0;
    for (int i = 0; i < 4; ++i) k += c.src[i] != nullptr;
    if (!k || !bytes) return;
    const long long v = (long long)(bytes / 16);
    const int per = int(std::min<long long>(std::max<long long>((v + 255) / 256, 1), 64));
    launch_pdl(copy_rows_kernel, dim3(per, 4), dim3(256), 0, s, 1, c, v);
    CUDA_CHECK(cudaGetLastError());
}

void upsample2x(Elem e, const void* x, void* y, int rows, int W, int ld, cudaStream_t s) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    DISPATCH(e, launch_pdl(upsample_kernel<T>, dim3(grid_for((long long)rows * W * ld / VEC, 256)), dim3(256), 0, s, 1, 
                    static_cast<const T*>(x), static_cast<T*>(y), rows, W, ld));
    CUDA_CHECK(cudaGetLastError());
}


void transpose(Elem e, const void* V, int ns, int C, long long ldv, void* Vt, long long ldt,
               cudaStream_t s) {
    dim3 grid((ns + 31) / 32, (C + 31) / 32), block(32, 8);
    DISPATCH(e, launch_pdl(transpose_kernel<T>, dim3(grid), dim3(block), 0, s, 1, static_cast<const T*>(V), ns, C, ldv,
                                                          static_cast<T*>(Vt), ldt));
    CUDA_CHECK(cudaGetLastError());
}

void attn_rescale(Elem e, void* P, long long ldp, int m, int s, const float* rowmax, int n_tiles,
                  int block_n, int ld_rm, float* row_scale, bool round_tf32, cudaStream_t st) {
    const int VEC = e == Elem::BF16 ? 8 : 4;
    if (block_n % VEC || ldp % VEC)
        throw std::invalid_argument("attention: P tiles must hold whole 16-byte vectors");
    const size_t smem = size_t(8) * n_tiles * sizeof(float);
    DISPATCH(e, launch_pdl(attn_rescale_kernel<T>, dim3((m + 7) / 8), dim3(256), smem, st, 1,
                           static_cast<T*>(P), ldp, m, s, rowmax, n_tiles, block_n, ld_rm,
                           row_scale, round_tf32 ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void stem_im2col(Elem e, const void* in, int rows, int W, int ld_in, int C_in, void* out, int kpad,
                 cudaStream_t s) {
    if (C_in > 4 || kpad < 36) throw std::invalid_argument("stem_im2col: <= 4 channels, kpad >= 36");
    DISPATCH(e, launch_pdl(stem_im2col_kernel<T>, dim3(grid_for((long long)rows * W * 9, 256)),
                           dim3(256), 0, s, 1, static_cast<const T*>(in), rows, W, ld_in, C_in,
                           static_cast<T*>(out), kpad));
    CUDA_CHECK(cudaGetLastError());
}

void cfg_combine_eps(float* out, const float* eps_c, const float* eps_u, long long n, double scale,
                     cudaStream_t s) {
    launch_pdl(cfg_combine_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, 1, out, eps_c, eps_u, n, scale);
    CUDA_CHECK(cudaGetLastError());
}

void stream_sleep(unsigned int us, cudaStream_t s) {
    sleep_kernel<<<1, 1, 0, s>>>(us);
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
    launch_pdl(time_projection_kernel, dim3(grid), dim3(256), dim * sizeof(float), s, 1, layers_dev, arg);
    CUDA_CHECK(cudaGetLastError());
}

void time_projection_plan(const TembLayer* layers_dev, int n_layers, int max_c,
                          const float* embs_dev, int n_steps, int dim, float* table, int ldt,
                          cudaStream_t s) {
    if (n_layers == 0 || n_steps == 0) return;
    dim3 grid(std::max(1, (max_c + 7) / 8), n_layers, n_steps);
    launch_pdl(time_projection_plan_kernel, dim3(grid), dim3(256), dim * sizeof(float), s, 1, layers_dev, embs_dev, dim,
                                                                        table, n_layers, ldt);
    CUDA_CHECK(cudaGetLastError());
}

void gemv_f64(const float* W, const float* b, const float* x, int rows, int cols, float* out,
              cudaStream_t s) {
    launch_pdl(gemv_f64_kernel, dim3(std::max(1, std::min(148, (rows + 7) / 8))), dim3(256), 0, s, 1, W, b, x, rows, cols,
                                                                              out);
    CUDA_CHECK(cudaGetLastError());
}

void ddim_update(const float* x, const float* eps, float* xo, long long n, int C, double abar_t,
                 double abar_n, Elem e, void* stem, int stem_ld, cudaStream_t s) {
    const double sa = std::sqrt(abar_t), s1 = std::sqrt(1.0 - abar_t);
    const double sn = std::sqrt(abar_n), s1n = std::sqrt(1.0 - abar_n);
    DISPATCH(e, launch_pdl(ddim_kernel<T>, dim3(grid_for(n, 256)), dim3(256), 0, s, 1, x, eps, xo, n, C, sa, s1, sn, s1n,
                                                                static_cast<T*>(stem), stem_ld));
    CUDA_CHECK(cudaGetLastError());
}

void nchw_to_nhwc(const float* src, int C, int H, int W, int r0, int rows, Elem e, void* dst,
                  int ld, bool r, cudaStream_t s) {
    DISPATCH(e, launch_pdl(nchw_to_nhwc_kernel<T>, dim3(grid_for((long long)rows * W * C, 256)), dim3(256), 0, s, 1, 
                    src, C, H, W, r0, rows, static_cast<T*>(dst), ld, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void nhwc_to_nchw(Elem e, const void* src, int ld, int C, int rows, int W, float* dst,
                  int* nonfinite, cudaStream_t s) {
    DISPATCH(e, launch_pdl(nhwc_to_nchw_kernel<T>, dim3(grid_for((long long)rows * W * C, 256)), dim3(256), 0, s, 1, 
                    static_cast<const T*>(src), ld, C, rows, W, dst, nonfinite));
    CUDA_CHECK(cudaGetLastError());
}

void nhwc_f32_to_nchw(const float* src, int C, int rows, int W, float* dst, int* nonfinite,
                      cudaStream_t s) {
    launch_pdl(nhwc_to_nchw_kernel<float>, dim3(grid_for((long long)rows * W * C, 256)), dim3(256), 0, s, 1, 
        src, C, C, rows, W, dst, nonfinite);
    CUDA_CHECK(cudaGetLastError());
}

void crop_nchw_to_nhwc(const float* src, int C, int H, int W, int y0, int x0, int rows, int cols,
                       Elem e, void* dst, int ld, bool r, cudaStream_t s) {
    DISPATCH(e, launch_pdl(crop_kernel<T>, dim3(grid_for((long long)rows * cols * C, 256)), dim3(256), 0, s, 1, 
                    src, C, H, W, y0, x0, rows, cols, static_cast<T*>(dst), ld, r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void scatter_nhwc_to_nchw(const float* patch, int C, int rows, int cols, float* dst, int H, int W,
                          int y0, int x0, int* nonfinite, cudaStream_t s) {
    launch_pdl(scatter_patch_kernel, dim3(grid_for((long long)rows * cols * C, 256)), dim3(256), 0, s, 1, 
        patch, C, rows, cols, dst, H, W, y0, x0, nonfinite);
    CUDA_CHECK(cudaGetLastError());
}

void f32_to_elem(const float* src, Elem e, void* dst, long long n, bool r, cudaStream_t s) {
    DISPATCH(e, launch_pdl(f32_to_elem_kernel<T>, dim3(grid_for(n, 256)), dim3(256), 0, s, 1, src, static_cast<T*>(dst), n,
                                                                       r ? 1 : 0));
    CUDA_CHECK(cudaGetLastError());
}

void elem_to_f32(Elem e, const void* src, float* dst, long long n, cudaStream_t s) {
    DISPATCH(e, launch_pdl(elem_to_f32_kernel<T>, dim3(grid_for(n, 256)), dim3(256), 0, s, 1, static_cast<const T*>(src),
                                                                       dst, n));
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace pp
