// sm_100a tcgen05 GEMM / implicit-GEMM 3x3 conv (see gemm.hpp for the contract).
//
// Warp roles (480 threads, 1 CTA per SM, persistent over output tiles):
//   warps 0, 6  TMA producers (one lane each, alternate stages): A boxes + B box per stage
//   warp 1      TMEM owner + MMA issuer (one lane): 4 x tcgen05.mma per 128-byte K block
//   warps 2-5, 7-14  epilogue (three warps per TMEM lane quarter): tcgen05.ld ->
//               bias/residual -> NHWC stores (+ GN statistics)
// Pipelines: smem ring (full/empty mbarriers, TMA <-> MMA) and a 2-deep TMEM
// accumulator ring (tmem_full/tmem_empty, MMA <-> epilogue), so the epilogue of
// tile i overlaps the main loop of tile i+1.
#include "gemm.hpp"
#include "pdl.cuh"
#include "ptx.cuh"
#include "util.hpp"

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

namespace pp {

namespace {

// warp 0: TMA, 1: MMA, 6: TMA, the rest epilogue: kEpiPerQuarter warps per TMEM lane quarter
constexpr int kEpiPerQuarter = 3;
constexpr int kEpiThreads = 128 * kEpiPerQuarter;
constexpr int kThreads = 96 + kEpiThreads;
constexpr int kTileM = 128;
constexpr int kBlockBytes = 128;   // K block = 128 bytes of each operand row
constexpr int kTmemCols = 512;     // 2 accumulators x 256 columns
constexpr int kSmemMax = 232448;
// Kernel debug flags (GemmArgs::debug: 1 no MMA, 2 no TMA, 4 no epilogue, 1024 one K block; the
// GroupNorm-statistics epilogue: 8 no column sums, 16 no per-tile section, 32 no fold, 64 relaxed
// ticket) exist for the micro-benchmarks only and are compiled out of the shipped library.
#ifdef PP_GEMM_DEBUG
constexpr bool kGemmDebug = true;
#else
constexpr bool kGemmDebug = false;
#endif

__device__ __forceinline__ float round_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void epi_bar() {
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

struct TileCoord {
    int m, ty, tx, nt, split;
};

// Work unit t -> (split, N tile, M unit); the CTA's M tile is unit * P + rank (P = CTAs
// per cluster).  m >= tiles_y * tiles_x only for the peer of an odd last unit.
template <int P>
__device__ __forceinline__ TileCoord decode_tile(const GemmArgs& a, int t, int rank) {
    TileCoord c;
    c.split = t % a.splits;
    int rest = t / a.splits;
    c.nt = rest % a.n_tiles;
    c.m = (rest / a.n_tiles) * P + rank;
    c.tx = c.m % a.tiles_x;
    c.ty = c.m / a.tiles_x;
    return c;
}

// Smem layout after the operand stages (all offsets from the 1024-aligned base).
struct SmemTail {
    uint64_t* full_bar;
    uint64_t* empty_bar;
    uint64_t* tfull_bar;
    uint64_t* tempty_bar;
    uint64_t* slab_full;    // [kMaxSlabSlots] A-slab ring (slab mode)
    uint64_t* slab_empty;   // [kMaxSlabSlots]
    uint32_t* tmem_slot;
    int* flags;        // [4]
    float* bias;       // [2][block_n]
    float* gn;         // [4 warps][block_n cols][2]  (also the GN fold scratch)
};

constexpr int kMaxSlabSlots = 4;

// Sized by block_n so that the fused-GN variant keeps the same pipeline depth.
__host__ __device__ inline size_t tail_bytes(int stages, bool gn, int block_n) {
    // gn: the GroupNorm column-sum scratch [4][block_n][2], also the attention epilogues' row
    // scratch (>= 3 x 128 floats)
    return size_t(2 * stages + 4 + 2 * kMaxSlabSlots) * 8 + 16 + 16 + size_t(2) * block_n * 4 +
           (gn ? (block_n >= 48 ? size_t(4) * block_n * 2 * 4 : size_t(384) * 4) : 0);
}

// B box of one stage: a CTA stages block_n / P weight rows (in a CTA pair each CTA loads its
// share `rank` of the rows).  bcoord = first weight row of this CTA's share.  kPair:
// complete_tx on the leader's barrier (shared::cluster address bar_cl), else on the local
// barrier bar.
template <bool kPair, bool kBmn = false>
__device__ __forceinline__ void load_b(uint8_t* sb, const CUtensorMap* tm, uint64_t* bar,
                                       uint32_t bar_cl, int bcoord, int kb, const GemmArgs& a,
                                       int kel = 0) {
    if (kBmn) {   // V [K][N] (MN-major): box {kel N, kps * kel K rows, block_n / P / kel chunks}
        if (kPair)
            ptx::tma_load_3d_pair(sb, tm, bar_cl, 0, kb * kel, bcoord / kel);
        else
            ptx::tma_load_3d(sb, tm, bar, 0, kb * kel, bcoord / kel);
        return;
    }
    if (a.slab) {   // K block kb = chunk * 9 + tap; one stage = kps taps
        const int chunk = kb / 9, tap = kb - chunk * 9;
        if (kPair)
            ptx::tma_load_4d_pair(sb, tm, bar_cl, 0, bcoord, chunk, tap);
        else
            ptx::tma_load_4d(sb, tm, bar, 0, bcoord, chunk, tap);
        return;
    }
    if (kPair)
        ptx::tma_load_3d_pair(sb, tm, bar_cl, 0, bcoord, kb);
    else
        ptx::tma_load_3d(sb, tm, bar, 0, bcoord, kb);
}

// Final values of one 16-column chunk of one row: bias, residual, store, GN sums.
// srow != nullptr: the row goes to the smem staging tile (dense [row][block_n], stored later
// by one TMA box) instead of straight to global memory.
template <bool kTF32>
__device__ __forceinline__ void finish_chunk(const GemmArgs& a, float* v, const float* sbias,
                                             int c0, int n0, long long p, bool valid,
                                             float* sgn_warp, int lane, uint8_t* srow) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = v[j] * a.scale + sbias[c0 + j];
    const bool full = n0 + 16 <= a.n_valid;
    // fused nearest 2x upsample of the output (up_w = input width): row p -> the 2x2 block
    long long prow = p;
    if (a.up_w) {
        const long long py = p / a.up_w, px = p - py * a.up_w;
        prow = (2 * py) * (2LL * a.up_w) + 2 * px;
    }
    const long long up_dy = 2LL * a.up_w * a.out_ld;   // elements to the row below
    if (valid) {
        if (kTF32 || a.out_f32) {
            float* dst = reinterpret_cast<float*>(a.out) + prow * a.out_ld + n0;
            const float* res =
                a.residual ? reinterpret_cast<const float*>(a.residual) + p * a.res_ld + n0 : nullptr;
            if (full && (a.out_ld % 4) == 0 && (!res || (a.res_ld % 4) == 0)) {
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    if (res) {
                        const float4 q = *reinterpret_cast<const float4*>(res + j);
                        v[j] += q.x; v[j + 1] += q.y; v[j + 2] += q.z; v[j + 3] += q.w;
                    }
                    if (a.round_tf32) {
                        v[j] = round_tf32(v[j]); v[j + 1] = round_tf32(v[j + 1]);
                        v[j + 2] = round_tf32(v[j + 2]); v[j + 3] = round_tf32(v[j + 3]);
                    }
                }
                if (!srow && (a.out_ld % 8) == 0) {
                    // two 256-bit stores: whole 32-byte sectors
#pragma unroll
                    for (int j = 0; j < 16; j += 8) {
                        const uint4 lo = make_uint4(__float_as_uint(v[j]), __float_as_uint(v[j + 1]),
                                                    __float_as_uint(v[j + 2]), __float_as_uint(v[j + 3]));
                        const uint4 hi = make_uint4(__float_as_uint(v[j + 4]), __float_as_uint(v[j + 5]),
                                                    __float_as_uint(v[j + 6]), __float_as_uint(v[j + 7]));
                        ptx::st_global_v8(dst + j, lo, hi);
                        if (a.up_w) {
                            ptx::st_global_v8(dst + a.out_ld + j, lo, hi);
                            ptx::st_global_v8(dst + up_dy + j, lo, hi);
                            ptx::st_global_v8(dst + up_dy + a.out_ld + j, lo, hi);
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        const float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                        if (srow) {
                            *reinterpret_cast<float4*>(srow + (c0 + j) * 4) = o;
                        } else {
                            *reinterpret_cast<float4*>(dst + j) = o;
                            if (a.up_w) {
                                *reinterpret_cast<float4*>(dst + a.out_ld + j) = o;
                                *reinterpret_cast<float4*>(dst + up_dy + j) = o;
                                *reinterpret_cast<float4*>(dst + up_dy + a.out_ld + j) = o;
                            }
                        }
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (n0 + j < a.n_valid) {
                        float o = v[j] + (res ? res[j] : 0.0f);
                        o = a.round_tf32 ? round_tf32(o) : o;
                        if (!srow) dst[j] = o;
                        v[j] = o;
                    } else {
                        v[j] = 0.0f;
                    }
                }
                if (srow) {
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<float4*>(srow + (c0 + j) * 4) =
                            make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                }
            }
        } else {
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(a.out) + prow * a.out_ld + n0;
            const __nv_bfloat16* res =
                a.residual ? reinterpret_cast<const __nv_bfloat16*>(a.residual) + p * a.res_ld + n0
                           : nullptr;
            if (full && (a.out_ld % 8) == 0 && (!res || (a.res_ld % 8) == 0)) {
                uint4 o[2];
#pragma unroll
                for (int j = 0; j < 16; j += 8) {
                    if (res) {
                        const uint4 q = *reinterpret_cast<const uint4*>(res + j);
                        const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float2 f = __bfloat1622float2(q2[i]);
                            v[j + 2 * i] += f.x;
                            v[j + 2 * i + 1] += f.y;
                        }
                    }
                    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o[j / 8]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        o2[i] = __floats2bfloat162_rn(v[j + 2 * i], v[j + 2 * i + 1]);
                        const float2 back = __bfloat1622float2(o2[i]);   // stats see stored values
                        v[j + 2 * i] = back.x;
                        v[j + 2 * i + 1] = back.y;
                    }
                }
                if (srow) {
                    *reinterpret_cast<uint4*>(srow + c0 * 2) = o[0];
                    *reinterpret_cast<uint4*>(srow + (c0 + 8) * 2) = o[1];
                } else if (a.out_ld % 16 == 0) {
                    // one 256-bit store: the whole 32-byte sector of this row chunk
                    ptx::st_global_v8(dst, o[0], o[1]);
                    if (a.up_w) {
                        ptx::st_global_v8(dst + a.out_ld, o[0], o[1]);
                        ptx::st_global_v8(dst + up_dy, o[0], o[1]);
                        ptx::st_global_v8(dst + up_dy + a.out_ld, o[0], o[1]);
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        *reinterpret_cast<uint4*>(dst + 8 * h) = o[h];
                        if (a.up_w) {
                            *reinterpret_cast<uint4*>(dst + a.out_ld + 8 * h) = o[h];
                            *reinterpret_cast<uint4*>(dst + up_dy + 8 * h) = o[h];
                            *reinterpret_cast<uint4*>(dst + up_dy + a.out_ld + 8 * h) = o[h];
                        }
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (n0 + j < a.n_valid) {
                        float o = v[j] + (res ? __bfloat162float(res[j]) : 0.0f);
                        const __nv_bfloat16 b = __float2bfloat16(o);
                        if (!srow) dst[j] = b;
                        v[j] = __bfloat162float(b);
                    } else {
                        v[j] = 0.0f;
                    }
                }
                if (srow) {
#pragma unroll
                    for (int j = 0; j < 16; j += 8) {
                        uint4 o;
                        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            o2[i] = __floats2bfloat162_rn(v[j + 2 * i], v[j + 2 * i + 1]);
                        *reinterpret_cast<uint4*>(srow + (c0 + j) * 2) = o;
                    }
                }
            }
        }
    }
    if (a.gn_groups && !(kGemmDebug && (a.debug & 8))) {
        // Column sums over the warp's 32 rows (invalid rows contribute 0) by a butterfly
        // transpose-reduce: each xor step halves the columns a lane keeps, so 16 columns
        // cost 16+8+4+2+1 shuffles per quantity instead of 16*5.  Lane l ends up with the
        // sum of column 8*b4 + 4*b3 + 2*b2 + b1 (b = bits of l), duplicated on l ^ 1.
        float s[16], q[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            s[j] = valid ? v[j] : 0.0f;
            q[j] = s[j] * s[j];
        }
#pragma unroll
        for (int o = 16, w = 8; o >= 2; o >>= 1, w >>= 1) {
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int j = 0; j < w; ++j) {
                const float gs = upper ? s[j] : s[j + w];
                const float gq = upper ? q[j] : q[j + w];
                const float ks = upper ? s[j + w] : s[j];
                const float kq = upper ? q[j + w] : q[j];
                s[j] = ks + __shfl_xor_sync(0xffffffffu, gs, o);
                q[j] = kq + __shfl_xor_sync(0xffffffffu, gq, o);
            }
        }
        s[0] += __shfl_xor_sync(0xffffffffu, s[0], 1);
        q[0] += __shfl_xor_sync(0xffffffffu, q[0], 1);
        if ((lane & 1) == 0) {
            const int col = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                            ((lane >> 1) & 1);
            sgn_warp[(c0 + col) * 2] = s[0];
            sgn_warp[(c0 + col) * 2 + 1] = q[0];
        }
    }
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Attention S-GEMM epilogue (softmax in the epilogue, proj/src/tensor.cpp:163-199): one
// 16-column chunk of row p of S = Q K^T -> P = 2^(S * sl2 - shift) with shift = the row's
// max over the tile (so P <= 1), stored in the P element type (keys >= n_valid: not stored,
// the P buffer's padding columns stay zero).
template <bool kTF32>
__device__ __forceinline__ void softmax_chunk(const GemmArgs& a, float* v, int n0, long long p,
                                              bool valid, float sl2, float shift) {
    if (!valid) return;
    const bool full = n0 + 16 <= a.n_valid;
    if (kTF32 || a.out_f32) {
        float* dst = reinterpret_cast<float*>(a.out) + p * a.out_ld + n0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            v[j] = ex2_approx(fmaf(v[j], sl2, -shift));
            if (a.round_tf32) v[j] = round_tf32(v[j]);
        }
        if (full && (a.out_ld % 8) == 0) {
#pragma unroll
            for (int j = 0; j < 16; j += 8) {
                uint4 lo, hi;
                lo = make_uint4(__float_as_uint(v[j]), __float_as_uint(v[j + 1]),
                                __float_as_uint(v[j + 2]), __float_as_uint(v[j + 3]));
                hi = make_uint4(__float_as_uint(v[j + 4]), __float_as_uint(v[j + 5]),
                                __float_as_uint(v[j + 6]), __float_as_uint(v[j + 7]));
                ptx::st_global_v8(dst + j, lo, hi);
            }
        } else {
            for (int j = 0; j < 16; ++j)
                if (n0 + j < a.n_valid) dst[j] = v[j];
        }
    } else {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(a.out) + p * a.out_ld + n0;
        uint4 o[2];
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(o);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            o2[i] = __floats2bfloat162_rn(ex2_approx(fmaf(v[2 * i], sl2, -shift)),
                                          ex2_approx(fmaf(v[2 * i + 1], sl2, -shift)));
        if (full && (a.out_ld % 16) == 0) {
            ptx::st_global_v8(dst, o[0], o[1]);
        } else {
            const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(o);
            for (int j = 0; j < 16; ++j)
                if (n0 + j < a.n_valid) dst[j] = ob[j];
        }
    }
}

// kAttn: 0 = conv / linear (no attention code compiled in), 1 = attention S GEMM (softmax
// epilogue), 2 = attention PV GEMM (1/l row scale) with the B operand MN-major (bf16: V
// [keys][d] as staged by TMA, no transpose), 3 = PV GEMM with B = V^T K-major (TF32, or
// channel counts that do not fill 128-byte chunks).
template <bool kTF32, bool kPair, int kAttn>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, const GemmArgs a) {
    constexpr bool kBmn = kAttn == 2;
    static_assert(!(kBmn && kTF32), "MN-major B is bf16 only");
    constexpr int P = kPair ? 2 : 1;   // CTAs per cluster
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte aligned base derived from smem_raw by pointer arithmetic (not an integer
    // cast), so the compiler keeps the shared address space: LDS/STS for the tail arrays
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int stages = a.stages;
    const int kps = a.kps;                                      // K blocks per stage (1 or 2)
    const uint32_t a_slot = kTileM * kBlockBytes;               // one A box slot
    const uint32_t b_slot = uint32_t(a.block_n / P) * kBlockBytes;
    // slab mode (stride-1 conv, one output row per tile): A comes from a 2-4 slot ring of im2col
    // slabs (3 input rows x (w_box + 2) pixels x 128 B per channel chunk) that serve all nine
    // taps; the stage ring then holds B only
    const uint32_t a_stage_bytes = a.slab ? 0u : kps * a_slot;
    uint8_t* const ring = smem + (a.slab ? uint32_t(a.slab_slots) * a.slab_bytes : 0u);
    const uint32_t b_stage_bytes = kps * b_slot;
    const uint32_t stage_bytes = a_stage_bytes + b_stage_bytes;
    SmemTail st;
    {
        uint8_t* p = ring + size_t(stages) * stage_bytes;
        st.full_bar = reinterpret_cast<uint64_t*>(p);
        st.empty_bar = st.full_bar + stages;
        st.tfull_bar = st.empty_bar + stages;
        st.tempty_bar = st.tfull_bar + 2;
        st.slab_full = st.tempty_bar + 2;
        st.slab_empty = st.slab_full + kMaxSlabSlots;
        st.tmem_slot = reinterpret_cast<uint32_t*>(st.slab_empty + kMaxSlabSlots);
        st.flags = reinterpret_cast<int*>(st.tmem_slot + 4);
        st.bias = reinterpret_cast<float*>(st.flags + 4);
        st.gn = st.bias + 2 * a.block_n;
    }

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int dbg = kGemmDebug ? a.debug : 0;
    const int crank = kPair ? int(ptx::cluster_ctarank()) : 0;   // rank in the cluster
    const int rank = crank & 1;            // rank in the CTA pair
    const uint32_t ldr = uint32_t(crank & ~1);                // the pair's leader CTA
    const uint16_t pair_mask = uint16_t(3u << ldr);

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        if (a.tma_store) ptx::prefetch_tmap(&tmD);
        for (int s = 0; s < stages; ++s) {
            ptx::mbar_init(&st.full_bar[s], 1);
            ptx::mbar_init(&st.empty_bar[s], 1);
        }
        for (int s = 0; s < kMaxSlabSlots; ++s) {
            ptx::mbar_init(&st.slab_full[s], 1);
            ptx::mbar_init(&st.slab_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&st.tfull_bar[s], 1);
            ptx::mbar_init(&st.tempty_bar[s], 4 * kEpiPerQuarter * P);
        }
        ptx::fence_barrier_init();
        ptx::fence_proxy_async();
    }
    if (warp == 1) {
        if (kPair)
            ptx::tmem_alloc_pair(st.tmem_slot, kTmemCols);
        else
            ptx::tmem_alloc(st.tmem_slot, kTmemCols);
    }
    ptx::tc_fence_before();
    if (kPair)
        ptx::cluster_sync();   // peer barriers initialised before any multicast commit
    else
        __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *st.tmem_slot;
    pdl_trigger();   // the next kernel on the stream may start its own prologue now

    const int m_tiles = a.tiles_y * a.tiles_x;
    const int total_tiles = (m_tiles + P - 1) / P * a.n_tiles * a.splits;
    const int tile0 = blockIdx.x / P, tile_step = gridDim.x / P;
    const int conv = a.mode != 0;
    const int a_box_bytes = a.slab ? 0 : conv ? a.rows_box * a.w_box * kBlockBytes : int(a_slot);

    if (warp == 0 || warp == 6) {
        // ===== TMA producers: two warps, stage-interleaved (warp-uniform loops, one elected
        // lane issues).  One stage = kps consecutive 128-byte K blocks: kps A boxes and one
        // 3-D B box, completing on one full barrier.  Both warps walk the same (tile, K)
        // sequence; warp pw only waits/issues on the stages with iteration index % 2 == pw,
        // which halves the serial control work (mbarrier wait, expect_tx, TMA issue) each
        // warp does per stage.
        const int pw = warp == 0 ? 0 : 1;
        int stage = 0;
        uint32_t phase = 0;
        const int kel = kTF32 ? 32 : 64;  // elements per 128-byte K block
        // pair: every box completes on the leader's full barrier
        const uint32_t full_leader = kPair ? ptx::mapa(ptx::smem_u32(st.full_bar), ldr) : 0u;
        // PDL: the weights (B) do not depend on the previous kernel, so the first tile's
        // first `pre` stages get their B boxes (and are armed for A + B) before waiting for
        // it; only the A boxes (activations) wait.
        int pre = 0;
        if (a.b_static && tile0 < total_tiles && !(dbg & 2)) {
            const TileCoord tc = decode_tile<P>(a, tile0, crank);
            const int kb0 = tc.split * a.kb_per_split;
            const int kb1 = (dbg & 1024) ? kb0 + 1 : min(kb0 + a.kb_per_split, a.k_blocks);
            pre = min(stages, (kb1 - kb0 + kps - 1) / kps);
            const int bcoord = tc.nt * a.block_n + rank * (a.block_n / P);
            for (int i = pw; i < pre; i += 2) {
                if (ptx::elect_one()) {
                    uint8_t* sb = ring + size_t(i) * stage_bytes + a_stage_bytes;
                    const int nk = min(kps, kb1 - (kb0 + i * kps));
                    if (rank == 0)
                        ptx::mbar_arrive_expect_tx(&st.full_bar[i],
                                                   P * (nk * a_box_bytes + b_stage_bytes));
                    load_b<kPair, kBmn>(sb, &tmB, &st.full_bar[i], full_leader + uint32_t(i) * 8u,
                                        bcoord, kb0 + i * kps, a, kel);
                }
                __syncwarp();
            }
        }
        if (a.b_static && pw == 0 && a.b_bytes > 0 && !(dbg & 2)) {
            // The weights are streamed from HBM once per layer (155 MB per UNet step do not
            // stay in L2): pull this CTA's 1/grid slice of the whole B tensor into L2 now,
            // so the B boxes of later K blocks hit L2 instead of paying HBM latency in the
            // K loop.  Issued before pdl_wait: overlaps the previous kernel's tail.
            const long long per = ((a.b_bytes + gridDim.x - 1) / gridDim.x + 15) / 16 * 16;
            const long long lo = per * blockIdx.x;
            const long long hi = min(a.b_bytes, lo + per);
            if (ptx::elect_one()) {
                const char* base = static_cast<const char*>(a.b_base);
                for (long long off = lo; off < hi; off += 32768)
                    ptx::prefetch_l2_bulk(base + off, uint32_t(min(32768LL, hi - off)));
            }
            __syncwarp();
        }
        pdl_wait();
        // loop-invariant launch parameters, read once
        const bool no_tma = dbg & 2;
        const bool slab = a.slab != 0;
        const bool stride2 = a.mode == 2;
        const int cin_chunks = a.cin_chunks;
        int it = 0;
        int sl_slot = 0;          // slab mode: A-slab ring slot / phase (both producer warps)
        uint32_t sl_phase = 0;
        const uint32_t slab_leader = kPair ? ptx::mapa(ptx::smem_u32(st.slab_full), ldr) : 0u;
        for (int t = tile0; t < total_tiles; t += tile_step) {
            const TileCoord tc = decode_tile<P>(a, t, crank);
            const int kb0 = tc.split * a.kb_per_split;
            const int kb1 = (dbg & 1024) ? kb0 + 1 : min(kb0 + a.kb_per_split, a.k_blocks);
            const int oy0 = tc.ty * a.rows_box, ox0 = tc.tx * a.w_box;
            const int bcoord = tc.nt * a.block_n + rank * (a.block_n / P);
            const int arow = tc.ty * kTileM;
            // conv K position of block kb0: tap (ky, kx), channel chunk cj
            int cj = kb0 % a.cin_chunks;
            const int tap0 = kb0 / a.cin_chunks;
            int ky = tap0 / 3, kx = tap0 - 3 * (tap0 / 3);
            for (int kb = kb0; kb < kb1; kb += kps) {
                const int nk = min(kps, kb1 - kb);
                if ((it & 1) == pw) {
                    ptx::mbar_wait(&st.empty_bar[stage], phase ^ 1);
                    uint8_t* sa = ring + size_t(stage) * stage_bytes;
                    uint8_t* sb = sa + a_stage_bytes;
                    if (ptx::elect_one()) {
                        if (no_tma) {   // micro-benchmark: barriers only, no data movement
                            ptx::mbar_arrive(&st.full_bar[stage]);
                        } else {
                            const bool b_done = it < pre;   // armed + B issued before pdl_wait
                            if (rank == 0 && !b_done)
                                ptx::mbar_arrive_expect_tx(&st.full_bar[stage],
                                                           P * (nk * a_box_bytes + b_stage_bytes));
                            const uint32_t fb = kPair ? full_leader + uint32_t(stage) * 8u : 0u;
                            if (slab && kb % 9 == 0) {
                                // first stage of a channel chunk: its im2col slab (3 input rows
                                // x (w_box + 2) pixels, TMA zero-fill = the left/right padding)
                                ptx::mbar_wait(&st.slab_empty[sl_slot], sl_phase ^ 1);
                                if (rank == 0)
                                    ptx::mbar_arrive_expect_tx(&st.slab_full[sl_slot],
                                                               P * a.slab_box_bytes);
                                uint8_t* dst = smem + size_t(sl_slot) * a.slab_bytes;
                                const int ch = kb / 9;
                                if (kPair)
                                    ptx::tma_load_5d_pair(dst, &tmA, slab_leader + uint32_t(sl_slot) * 8u,
                                                          ch * kel, 0, ox0 - 1, 0, oy0);
                                else
                                    ptx::tma_load_5d(dst, &tmA, &st.slab_full[sl_slot], ch * kel, 0,
                                                     ox0 - 1, 0, oy0);
                            }
                            int c_j = cj, c_x = kx, c_y = ky;
                            for (int j = 0; j < nk && !slab; ++j) {
                                uint8_t* dst = sa + j * a_slot;
                                if (!conv) {
                                    if (kPair)
                                        ptx::tma_load_2d_pair(dst, &tmA, fb, (kb + j) * kel, arow);
                                    else
                                        ptx::tma_load_2d(dst, &tmA, &st.full_bar[stage],
                                                         (kb + j) * kel, arow);
                                } else {
                                    int c1 = 0, c2 = ox0 + c_x - 1, c3 = 0, c4 = oy0 + c_y;
                                    if (stride2) {
                                        c1 = c_x == 1 ? 0 : 1; c2 = ox0 + (c_x == 0 ? -1 : 0);
                                        c3 = c_y == 1 ? 1 : 0; c4 = oy0 + (c_y == 2 ? 1 : 0);
                                    }
                                    if (kPair)
                                        ptx::tma_load_5d_pair(dst, &tmA, fb, c_j * kel, c1, c2, c3, c4);
                                    else
                                        ptx::tma_load_5d(dst, &tmA, &st.full_bar[stage], c_j * kel,
                                                         c1, c2, c3, c4);
                                    if (++c_j == cin_chunks) {
                                        c_j = 0;
                                        if (++c_x == 3) {
                                            c_x = 0;
                                            ++c_y;
                                        }
                                    }
                                }
                            }
                            if (!b_done) {
                                load_b<kPair, kBmn>(sb, &tmB, &st.full_bar[stage], fb, bcoord, kb, a, kel);
                            }
                        }
                    }
                    __syncwarp();
                }
                ++it;
                if (slab && kb % 9 + kps >= 9 && ++sl_slot == a.slab_slots) {
                    sl_slot = 0;
                    sl_phase ^= 1;
                }
                for (int j = 0; j < nk; ++j) {
                    if (++cj == cin_chunks) {
                        cj = 0;
                        if (++kx == 3) {
                            kx = 0;
                            ++ky;
                        }
                    }
                }
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ===== MMA issuer (warp-uniform loop, one elected lane issues) =====
        // Descriptors: stage s, block j, K step k = base + s * (stage_bytes >> 4) +
        // j * (slot >> 4) + 2 * k (the start address field is addr >> 4; +32 bytes per
        // 16-element bf16 / 8-element tf32 step).
        const uint32_t smem0 = ptx::smem_u32(ring);
        const uint64_t desc_a0 = ptx::smem_desc_sw128(smem0);
        // kBmn: each 128-byte N chunk of a stage's B box holds kps * kel K rows (LBO apart)
        constexpr int kelB = kTF32 ? 32 : 64;
        const uint64_t desc_b0 =
            kBmn ? ptx::smem_desc_sw128_mn(smem0 + a_stage_bytes, uint32_t(kps * kelB * kBlockBytes))
                 : ptx::smem_desc_sw128(smem0 + a_stage_bytes);
        const uint32_t slab0 = ptx::smem_u32(smem);   // slab mode: slot s at slab0 + s * slab_bytes
        const uint64_t desc_stride = stage_bytes >> 4;
        const uint64_t a_next = a_slot >> 4;
        const uint64_t b_next = kBmn ? uint64_t(kelB * kBlockBytes) >> 4 : b_slot >> 4;
        // loop-invariant launch parameters, read once (the issue loop is on the critical path)
        const bool do_mma = !(dbg & 1);
        const bool slab = a.slab != 0;
        const uint32_t idesc = a.idesc;
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        int ms_slot = 0;          // slab mode: A-slab ring slot / phase
        uint32_t ms_phase = 0;
        for (int t = tile0; t < total_tiles; t += tile_step) {
            const TileCoord tc = decode_tile<P>(a, t, crank);
            const int kb0 = tc.split * a.kb_per_split;
            const int kb1 = (dbg & 1024) ? kb0 + 1 : min(kb0 + a.kb_per_split, a.k_blocks);
            ptx::mbar_wait(&st.tempty_bar[acc], acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem_base + uint32_t(acc * 256);
            for (int kb = kb0; kb < kb1; kb += kps) {
                if (slab) {
                    // one stage = taps sg .. sg + 2 (one kernel row) of channel chunk kb / 9:
                    // A rows of tap (ky, kx) start (ky * slab_px + kx) 128-byte rows into the
                    // slab (a start address that is not swizzle-atom aligned)
                    const int sg = kb % 9;
                    if (sg == 0) {
                        ptx::mbar_wait(&st.slab_full[ms_slot], ms_phase);
                        ptx::tc_fence_after();
                    }
                    ptx::mbar_wait(&st.full_bar[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t db = desc_b0 + uint64_t(stage) * desc_stride;
                    const uint32_t sbase = slab0 + uint32_t(ms_slot) * a.slab_bytes;
                    if (ptx::elect_one()) {
                        if (do_mma) {
                            for (int j = 0; j < kps; ++j) {
                                const int tap = sg + j;
                                if (tap < 9) {
                                    const int ky = tap / 3, kx = tap - 3 * ky;
                                    const uint32_t off = uint32_t(ky * a.slab_px + kx);
                                    // the SW128 XOR pattern is applied to absolute smem address
                                    // bits (as TMA wrote it), so an unaligned start needs no base
                                    // offset (measured: setting bits 49-51 breaks it)
                                    const uint64_t da = ptx::smem_desc_sw128(sbase + off * kBlockBytes);
                                    const uint32_t acc0 = (kb > kb0 || j > 0) ? 1u : 0u;
                                    const uint64_t dbj = db + uint64_t(j) * b_next;
                                    if (kPair) {
                                        if (kTF32)
                                            ptx::mma4_tf32_pair(d_tmem, da, dbj, idesc, acc0);
                                        else
                                            ptx::mma4_bf16_pair(d_tmem, da, dbj, idesc, acc0);
                                    } else {
                                        if (kTF32)
                                            ptx::mma4_tf32(d_tmem, da, dbj, idesc, acc0);
                                        else
                                            ptx::mma4_bf16(d_tmem, da, dbj, idesc, acc0);
                                    }
                                }
                            }
                        }
                        if (kPair) {
                            ptx::mma_commit_pair(&st.empty_bar[stage], pair_mask);
                            if (sg + kps >= 9) ptx::mma_commit_pair(&st.slab_empty[ms_slot], pair_mask);
                        } else {
                            ptx::mma_commit(&st.empty_bar[stage]);
                            if (sg + kps >= 9) ptx::mma_commit(&st.slab_empty[ms_slot]);
                        }
                    }
                    __syncwarp();
                    if (sg + kps >= 9 && ++ms_slot == a.slab_slots) {
                        ms_slot = 0;
                        ms_phase ^= 1;
                    }
                    if (++stage == stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                    continue;
                }
                const bool two = kb + 1 < kb1 && kps == 2;
                ptx::mbar_wait(&st.full_bar[stage], phase);
                ptx::tc_fence_after();
                const uint64_t da = desc_a0 + uint64_t(stage) * desc_stride;
                const uint64_t db = desc_b0 + uint64_t(stage) * desc_stride;
                if (ptx::elect_one()) {
                    if (do_mma) {
                        const uint32_t acc0 = kb > kb0 ? 1u : 0u;
                        if (kPair && kBmn) {
                            ptx::mma4_bf16_pair_bmn(d_tmem, da, db, idesc, acc0);
                            if (two) ptx::mma4_bf16_pair_bmn(d_tmem, da + a_next, db + b_next, idesc, 1u);
                        } else if (kPair) {
                            if (kTF32) {
                                ptx::mma4_tf32_pair(d_tmem, da, db, idesc, acc0);
                                if (two) ptx::mma4_tf32_pair(d_tmem, da + a_next, db + b_next, idesc, 1u);
                            } else {
                                ptx::mma4_bf16_pair(d_tmem, da, db, idesc, acc0);
                                if (two) ptx::mma4_bf16_pair(d_tmem, da + a_next, db + b_next, idesc, 1u);
                            }
                        } else if (kBmn) {
                            ptx::mma4_bf16_bmn(d_tmem, da, db, idesc, acc0);
                            if (two) ptx::mma4_bf16_bmn(d_tmem, da + a_next, db + b_next, idesc, 1u);
                        } else {
                            if (kTF32) {
                                ptx::mma4_tf32(d_tmem, da, db, idesc, acc0);
                                if (two) ptx::mma4_tf32(d_tmem, da + a_next, db + b_next, idesc, 1u);
                            } else {
                                ptx::mma4_bf16(d_tmem, da, db, idesc, acc0);
                                if (two) ptx::mma4_bf16(d_tmem, da + a_next, db + b_next, idesc, 1u);
                            }
                        }
                    }
                    if (kPair)
                        ptx::mma_commit_pair(&st.empty_bar[stage], pair_mask);
                    else
                        ptx::mma_commit(&st.empty_bar[stage]);
                }
                __syncwarp();
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (ptx::elect_one()) {
                if (kPair)
                    ptx::mma_commit_pair(&st.tfull_bar[acc], pair_mask);
                else
                    ptx::mma_commit(&st.tfull_bar[acc]);
            }
            __syncwarp();
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 2 && warp != 6) {
        // ===== epilogue (warps 2-5 and 7..; TMEM lane quarter = warp % 4, kEpiPerQuarter warps
        // per quarter: warp `half` of its quarter takes the 16-column chunks half, half + K, ...
        const int quarter = warp & 3;
        const int half = warp <= 5 ? 0 : (warp - 3) / 4;   // 7-10 -> 1, 11-14 -> 2
        const int r = quarter * 32 + lane;  // tile row owned by this thread
        const int et = warp <= 5 ? int(threadIdx.x) - 64 : int(threadIdx.x) - 96;   // 0..kEpiThreads-1
        constexpr int kCS = 16 * kEpiPerQuarter;   // chunk stride of one warp
        float* sgn_warp = st.gn + quarter * 2 * a.block_n;   // [block_n / cpg][2] used
        // accumulator release: the MMA issuer (the leader's, for a pair) waits for 4*P warps
        const uint32_t tempty_leader = kPair ? ptx::mapa(ptx::smem_u32(st.tempty_bar), ldr) : 0u;
        auto release = [&](int which) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (kPair)
                    ptx::mbar_arrive_cluster(tempty_leader + uint32_t(which) * 8u);
                else
                    ptx::mbar_arrive(&st.tempty_bar[which]);
            }
        };
        int acc = 0;
        uint32_t acc_phase = 0;
        // attention epilogues read what the previous kernel wrote (row norms, partial row
        // sums) ahead of the accumulator: wait for it here (the loads then overlap the MMAs)
        constexpr bool softmax = kAttn == 1;
        constexpr bool pv = kAttn >= 2;
        if (pv) pdl_wait();   // row_scale comes from the previous kernel
        const float sl2 = a.sm_scale * 1.4426950408889634f;   // scale * log2(e)
        float* const s_row = st.gn;   // softmax: [3][128] partial row maxima
        for (int t = tile0; t < total_tiles; t += tile_step) {
            const int cur = acc;
            const uint32_t cur_phase = acc_phase;
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
            const TileCoord tc = decode_tile<P>(a, t, crank);
            const int m_tile = tc.m;
            const int tile_id = m_tile * a.n_tiles + tc.nt;
            long long p;
            bool valid;
            if (conv) {
                const int ry = r / a.w_box, rx = r - ry * a.w_box;
                const int oy = tc.ty * a.rows_box + ry, ox = tc.tx * a.w_box + rx;
                valid = r < a.rows_box * a.w_box && oy < a.out_rows && ox < a.out_w;
                p = (long long)oy * a.out_w + ox;
            } else {
                p = (long long)tc.ty * kTileM + r;
                valid = p < a.out_rows;
            }
            const int nbase = tc.nt * a.block_n;
            float* sbias = st.bias + cur * a.block_n;
            // the CTA's last tile: the smem ring is idle once its accumulator is full, so the
            // output tile is staged there and written by one TMA box (coalesced) instead of
            // 128 per-thread row stores
            const bool stage_out = a.tma_store && t + tile_step >= total_tiles;
            const int eb_out = (kTF32 || a.out_f32) ? 4 : 2;
            uint8_t* srow = stage_out ? smem + size_t(r) * a.block_n * eb_out : nullptr;
            for (int c = et; c < a.block_n; c += kEpiThreads)
                sbias[c] = (a.bias && nbase + c < a.n_valid) ? a.bias[nbase + c] : 0.0f;
            const float rinv = (pv && valid) ? __ldg(a.row_scale + p) : 1.0f;
            ptx::mbar_wait(&st.tfull_bar[cur], cur_phase);
            ptx::tc_fence_after();
            if ((dbg & 4) || (kPair && m_tile >= m_tiles)) {
                // micro-benchmark (no epilogue work) / the empty half of an odd last pair unit
                release(cur);
                continue;
            }
            epi_bar();
            const uint32_t t_row = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(cur * 256);

            if (a.splits > 1) {
                // 2-way split-K.  The split that finishes its main loop first publishes its
                // fp32 partial tile; the second adds it to its own TMEM accumulator.  fp32
                // addition is commutative, so own + other is bitwise the same whichever split
                // is second: deterministic.  The first never waits after taking its ticket,
                // so the second's spin always terminates.
                unsigned int* ticket = a.tile_ticket + 2 * size_t(tile_id);
                unsigned int* ready = ticket + 1;
                if (et == 0) st.flags[cur] = int(atomicAdd(ticket, 1u));
                epi_bar();
                const bool first = st.flags[cur] == 0;
                // partial tile layout [block_n / 4][128 rows] of float4: for a fixed column
                // quad the 32 lanes of a warp touch 512 contiguous bytes (coalesced)
                float4* part = reinterpret_cast<float4*>(a.partial) +
                               size_t(tile_id) * (kTileM / 4) * a.block_n + r;
                if (first) {
                    for (int c0 = half * 16; c0 < a.block_n; c0 += kCS) {
                        float v[16];
                        ptx::tmem_ld16(t_row + c0, v);
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            __stcg(part + size_t((c0 + j) / 4) * kTileM,
                                   make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                    }
                    release(cur);
                    // publish: CTA barrier, then one gpu-scope fence + flag (the fence is
                    // cumulative over the other threads' stores ordered before the barrier)
                    epi_bar();
                    if (et == 0) ptx::st_release_gpu(ready, 1u);
                    continue;
                }
                if (et == 0) {
                    while (ptx::ld_acquire_gpu(ready) == 0u) __nanosleep(64);
                }
                epi_bar();
                for (int c0 = half * 16; c0 < a.block_n; c0 += kCS) {
                    float o[16], v[16];
                    if (valid) {
#pragma unroll
                        for (int j = 0; j < 16; j += 4) {
                            const float4 q = __ldcg(part + size_t((c0 + j) / 4) * kTileM);
                            o[j] = q.x; o[j + 1] = q.y; o[j + 2] = q.z; o[j + 3] = q.w;
                        }
                    }
                    ptx::tmem_ld16(t_row + c0, v);
                    if (valid) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = v[j] + o[j];
                    }
                    if (pv) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] *= rinv;
                    }
                    finish_chunk<kTF32>(a, v, sbias, c0, nbase + c0, p, valid, sgn_warp, lane, srow);
                }
                release(cur);
                if (et == 0) {
                    *ticket = 0u;
                    *ready = 0u;
                }
            } else if (softmax) {
                // pass 1: the row's max over this tile's keys (three chunk-interleaved warps
                // per row, combined through smem); pass 2: P = 2^(S sl2 - max) <= 1.  Two
                // TMEM loads in flight per wait.
                const bool full_tile = nbase + a.block_n <= a.n_valid;
                float mx = -INFINITY;
                for (int c0 = half * 16; c0 < a.block_n; c0 += 2 * kCS) {
                    float v0[16], v1[16];
                    const bool two = c0 + kCS < a.block_n;
                    ptx::tmem_ld16_nowait(t_row + c0, v0);
                    if (two) ptx::tmem_ld16_nowait(t_row + c0 + kCS, v1);
                    ptx::tmem_wait_ld();
                    ptx::tmem_pin16(v0);
                    if (two) ptx::tmem_pin16(v1);
                    if (full_tile) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) mx = fmaxf(mx, v0[j]);
                        if (two) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) mx = fmaxf(mx, v1[j]);
                        }
                    } else {
                        const int n0 = nbase + c0;
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (n0 + j < a.n_valid) mx = fmaxf(mx, v0[j]);
                        if (two) {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (n0 + kCS + j < a.n_valid) mx = fmaxf(mx, v1[j]);
                        }
                    }
                }
                s_row[half * kTileM + r] = mx;
                epi_bar();
                mx = fmaxf(fmaxf(s_row[r], s_row[kTileM + r]), s_row[2 * kTileM + r]);
                const float shift = mx * sl2;
                for (int c0 = half * 16; c0 < a.block_n; c0 += 2 * kCS) {
                    float v0[16], v1[16];
                    const bool two = c0 + kCS < a.block_n;
                    ptx::tmem_ld16_nowait(t_row + c0, v0);
                    if (two) ptx::tmem_ld16_nowait(t_row + c0 + kCS, v1);
                    ptx::tmem_wait_ld();
                    ptx::tmem_pin16(v0);
                    if (two) ptx::tmem_pin16(v1);
                    softmax_chunk<kTF32>(a, v0, nbase + c0, p, valid, sl2, shift);
                    if (two) softmax_chunk<kTF32>(a, v1, nbase + c0 + kCS, p, valid, sl2, shift);
                }
                release(cur);
                if (half == 0 && valid) a.sm_rowmax[size_t(tc.nt) * a.sm_ld + p] = shift;
                epi_bar();   // s_row is rewritten by the next tile
            } else {
                for (int c0 = half * 16; c0 < a.block_n; c0 += kCS) {
                    float v[16];
                    ptx::tmem_ld16(t_row + c0, v);
                    if (pv) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] *= rinv;
                    }
                    finish_chunk<kTF32>(a, v, sbias, c0, nbase + c0, p, valid, sgn_warp, lane, srow);
                }
                release(cur);
            }

            if (stage_out) {
                ptx::fence_proxy_async();   // staged rows -> visible to the TMA engine
                epi_bar();
                if (et == 0) {
                    if (conv)
                        ptx::tma_store_3d(&tmD, smem, nbase, tc.tx * a.w_box, tc.ty * a.rows_box);
                    else
                        ptx::tma_store_2d(&tmD, smem, nbase, tc.ty * kTileM);
                    ptx::bulk_commit();   // read completion awaited before the CTA exits
                }
            }
            if (a.gn_groups && !(dbg & 16)) {
                epi_bar();
                const int cpg = a.gn_cpg;
                const int g0 = nbase / cpg;
                const int gn_here = a.block_n / cpg;
                // 8 threads per group: lane sub of the 8 sums the (warp, column) entries
                // e = sub, sub + 8, ... of the group's 4 * cpg column sums, then a fixed
                // xor-tree over the 8 lanes -> deterministic, short dependency chains.
                const int sub = et & 7;
                const unsigned gmask = 0xFFu << (lane & 24);
                const int n_e = 4 * cpg;
                for (int gl = et >> 3; gl < gn_here; gl += kEpiThreads / 8) {
                    double s = 0.0, q = 0.0;
                    for (int e = sub; e < n_e; e += 8) {
                        const int w = e / cpg;
                        const int c = gl * cpg + (e - w * cpg);
                        const float2 v = *reinterpret_cast<const float2*>(st.gn + (w * a.block_n + c) * 2);
                        s += double(v.x);
                        q += double(v.y);
                    }
#pragma unroll
                    for (int o = 4; o; o >>= 1) {
                        s += __shfl_xor_sync(gmask, s, o);
                        q += __shfl_xor_sync(gmask, q, o);
                    }
                    if (sub == 0) {
                        double2* dst = reinterpret_cast<double2*>(a.gn_part) + (size_t)m_tile * a.gn_groups + g0 + gl;
                        *dst = make_double2(s, q);
                    }
                }
                epi_bar();
                // the last M tile of this N tile folds the N tile's groups (the N tiles fold
                // disjoint groups in parallel); counter gn_ticket[1 + nt]
                // (a thread other than the one that issued the last tile's TMA store: its
                // release fence would also wait for that store)
                if (et == kEpiThreads - 1) {
                    // release: cumulative over the partials stored before the barrier;
                    // acquire: the folding CTA sees every other tile's partials
                    st.flags[2] = ((dbg & 64) ? atomicAdd(a.gn_ticket + 1 + tc.nt, 1u)
                                              : ptx::atom_add_acq_rel_gpu(a.gn_ticket + 1 + tc.nt, 1u)) ==
                                  unsigned(m_tiles - 1);
                }
                epi_bar();
                if (st.flags[2] && !(dbg & 32)) {
                    // P threads per group each sum a fixed residue class of M tiles (16 loads
                    // in flight), the P partials are added in order -> deterministic
                    const int G = a.gn_groups;
                    int P = 1;
                    while (P * 2 * gn_here <= kEpiThreads && P * 2 * gn_here <= 2 * a.block_n) P *= 2;
                    double* sfold = reinterpret_cast<double*>(st.gn);   // [P][gn_here][2]
                    if (et < P * gn_here) {
                        const int gl = et % gn_here, part = et / gn_here;
                        const double2* src = reinterpret_cast<const double2*>(a.gn_part) + g0 + gl;
                        double s = 0.0, q = 0.0;
                        for (int m0 = part; m0 < m_tiles; m0 += 16 * P) {
                            double2 v[16];
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const int m = m0 + u * P;
                                v[u] = m < m_tiles ? __ldcg(src + (size_t)m * G) : make_double2(0.0, 0.0);
                            }
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                s += v[u].x;
                                q += v[u].y;
                            }
                        }
                        sfold[(part * gn_here + gl) * 2] = s;
                        sfold[(part * gn_here + gl) * 2 + 1] = q;
                    }
                    epi_bar();
                    for (int gl = et; gl < gn_here; gl += kEpiThreads) {
                        double s = 0.0, q = 0.0;
                        for (int part = 0; part < P; ++part) {
                            s += sfold[(part * gn_here + gl) * 2];
                            q += sfold[(part * gn_here + gl) * 2 + 1];
                        }
                        a.gn_out[(g0 + gl) * 2] = s / a.gn_count;
                        a.gn_out[(g0 + gl) * 2 + 1] = q / a.gn_count;
                    }
                    if (et == 0) a.gn_ticket[1 + tc.nt] = 0u;
                    epi_bar();
                }
            }
        }
        // the last tile's TMA store must have read its staging smem before the CTA exits (not
        // earlier: the GroupNorm section of that tile does not wait for it)
        if (et == 0 && a.tma_store) ptx::bulk_wait_read();
    }

    ptx::tc_fence_before();
    if (kPair)
        ptx::cluster_sync();   // the leader's last MMAs wrote the peer's TMEM
    else
        __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        if (kPair)
            ptx::tmem_dealloc_pair(tmem_base, kTmemCols);
        else
            ptx::tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---- host side ------------------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess)
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

void encode(CUtensorMap* m, Elem e, int rank, const void* base, const uint64_t* dims,
            const uint64_t* strides_bytes, const uint32_t* box) {
    uint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUresult r = get_encode()(
        m, e == Elem::BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
        rank, const_cast<void*>(base), dims, strides_bytes, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

// B operand [rows][K] (K-major, leading dim ld elements) as a 3-D map {kel, rows, K/kel}
// (dim 2 = 128-byte K block, stride 128 B): a {kel, box_rows, kps} box lands as kps
// consecutive [box_rows][128 B] swizzled slots.
void encode_b(CUtensorMap* m, Elem e, const void* base, int rows, int K, long long ld, int box_rows,
              int kps) {
    const uint64_t eb = elem_bytes(e);
    const int kel = int(kBlockBytes / eb);
    uint64_t d[3] = {uint64_t(kel), uint64_t(rows), uint64_t(K / kel)};
    uint64_t st[2] = {uint64_t(ld) * eb, uint64_t(kBlockBytes)};
    uint32_t b[3] = {uint32_t(kel), uint32_t(box_rows), uint32_t(kps)};
    encode(m, e, 3, base, d, st, b);
}

// Output map for the TMA-store epilogue (no swizzle): rank 2/3, dims/strides as given.
void encode_plain(CUtensorMap* m, bool f32, int rank, const void* base, const uint64_t* dims,
                  const uint64_t* strides_bytes, const uint32_t* box) {
    uint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUresult r = get_encode()(
        m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
        const_cast<void*>(base), dims, strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw std::runtime_error("cuTensorMapEncodeTiled (output) failed (" + std::to_string(int(r)) + ")");
}

// Enable the TMA-store epilogue when the output rows are 16-byte aligned.
void plan_output_map(GemmPlan& p, bool conv) {
    GemmArgs& a = p.a;
    const bool f32 = p.elem == Elem::F32 || a.out_f32;
    const uint64_t eb = f32 ? 4 : 2;
    a.tma_store = 0;
    if ((uint64_t(a.out_ld) * eb) % 16 || (reinterpret_cast<uintptr_t>(a.out) % 16)) return;
    if (a.up_w) return;            // fused upsample: four row stores per output row
    if (a.sm_rowmax) return;       // softmax epilogue: P rows stored directly
    if (conv) {
        uint64_t d[3] = {uint64_t(a.n_valid), uint64_t(a.out_w), uint64_t(a.out_rows)};
        uint64_t st[2] = {uint64_t(a.out_ld) * eb, uint64_t(a.out_w) * a.out_ld * eb};
        uint32_t b[3] = {uint32_t(a.block_n), uint32_t(a.w_box), uint32_t(a.rows_box)};
        encode_plain(&p.tmD, f32, 3, a.out, d, st, b);
    } else {
        uint64_t d[2] = {uint64_t(a.n_valid), uint64_t(a.out_rows)};
        uint64_t st[1] = {uint64_t(a.out_ld) * eb};
        uint32_t b[2] = {uint32_t(a.block_n), uint32_t(kTileM)};
        encode_plain(&p.tmD, f32, 2, a.out, d, st, b);
    }
    a.tma_store = 1;
}

uint32_t make_idesc(Elem e, int n, int m, bool b_mn = false) {
    uint32_t d = 0;
    if (b_mn) d |= 1u << 16;                         // B MN-major
    d |= 1u << 4;                                    // D format f32
    const uint32_t fmt = e == Elem::BF16 ? 1u : 2u;  // BF16 / TF32
    d |= fmt << 7;                                   // A format
    d |= fmt << 10;                                  // B format
    d |= uint32_t(n >> 3) << 17;                     // N
    d |= uint32_t(m >> 4) << 24;                     // M = 128 (single CTA) / 256 (pair)
    return d;
}

size_t smem_for(int block_n, int stages, bool gn, int pair, int kps, uint32_t slab_bytes = 0,
                int slab_slots = 2) {
    const size_t a_stage = slab_bytes ? 0 : kTileM * kBlockBytes;
    return size_t(slab_slots) * slab_bytes +
           size_t(stages) * kps * (a_stage + block_n / (pair ? 2 : 1) * kBlockBytes) + 1024 +
           tail_bytes(stages, gn, block_n);
}

int stages_for(int block_n, bool gn, int pair, int kps, uint32_t slab_bytes = 0, int slab_slots = 2) {
    int s = 8;
    while (s > 2 && smem_for(block_n, s, gn, pair, kps, slab_bytes, slab_slots) > size_t(kSmemMax)) --s;
    return s;
}

// K blocks per stage: 2 halves the per-block barrier / issue work of the single-thread TMA
// and MMA loops (measured ~450 cycles per iteration, more than the MMAs of a block_n <= 224
// block take), as long as at least 3 stages (6 blocks) still fit (3 blocks per stage:
// measured slower, 35.72 vs 33.61 ms per generation).
int choose_kps(int block_n, bool gn, int pair) {
    return stages_for(block_n, gn, pair, 2) >= 3 ? 2 : 1;
}

// Per-tile tensor-pipe efficiency by (pair, block_n): measured on B200 with
// scripts/gemm_micro.py on the SDXL-shape conv layers.  The single-CTA kernel is bound by
// shared-memory bandwidth (TMA writes + MMA operand reads of a 128 x block_n tile); the
// CTA pair halves the B bytes per SM.
double tile_eff(int pair, int bn) {
    if (pair) return bn >= 256 ? 0.90 : bn >= 160 ? 0.64 : bn >= 128 ? 0.35 : 0.27;
    return bn >= 256 ? 0.75 : bn >= 160 ? 0.62 : bn >= 128 ? 0.36 : 0.28;
}

// Pick (pair, block_n, split-K).  Cost model (cycles per SM): a 128-byte K block costs
// 2 * block_n MMA cycles / tile_eff; tiles are quantised into waves over the SMs (pairs
// over SM pairs); split-K pays a partial write + read.
//   force_splits: bits 0-3 = splits (0 auto), bit 4 = force pair, bit 5 = force single CTA
void choose_tiling(int m_tiles, int n_pad, int k_blocks, int num_sms, int gn_cpg, int force_splits,
                   int force_block_n, int& block_n, int& splits, int& pair, bool gemm = false,
                   int bn_mult = 16) {
    double best = 1e300;
    block_n = 16;
    splits = 1;
    pair = 0;
    const int fs = force_splits & 15;
    const bool force_pair = force_splits & 16, force_single = force_splits & 32;
    for (int pr = 0; pr <= 1; ++pr) {
        if ((force_pair && !pr) || (force_single && pr)) continue;
        if (pr && m_tiles < 2 && !force_pair) continue;
        const int P = pr ? 2 : 1;
        const int slots = num_sms / P;
        const int units = (m_tiles + P - 1) / P;
        for (int bn = 256; bn >= 16; bn -= 16) {
            if (force_block_n && bn != force_block_n) continue;
            if (n_pad % bn || bn % (bn_mult * (bn_mult > 16 ? P : 1))) continue;
            if (gn_cpg && bn % gn_cpg) continue;
            const int nt = n_pad / bn;
            for (int s : {1, 2}) {
                if (fs && s != std::min(fs, 2)) continue;
                if (s > k_blocks) continue;
                // split only when one wave leaves more than half of the SMs idle
                if (!fs && s == 2 && ((long long)units * nt * 2 > slots || k_blocks < 16)) continue;
                const long long tiles = (long long)units * nt * s;
                const double waves = std::ceil(double(tiles) / slots);
                const double per_kb = 2.0 * bn / tile_eff(pr, bn);
                const double kbs = std::ceil(double(k_blocks) / s);
                double cost = waves * (kbs * per_kb + 2500.0);
                if (s > 1) cost += 2.0 * 128.0 * bn * 4.0 / 20.0;
                if (cost < best * 0.98) {
                    best = cost;
                    block_n = bn;
                    splits = s;
                    pair = pr;
                }
            }
        }
    }
    if (force_block_n) block_n = force_block_n;
    // Plain GEMMs that fit one wave of single-CTA tiles (the 1024-token attention S / PV and
    // linear layers): each CTA runs a short K loop once, so the time is latency, not
    // shared-memory throughput -- the smallest per-CTA tile that still fits one wave wins
    // (measured, scripts/attn_gemm_sweep.py: PV 8.3 us at block_n 80 vs 10.8 us at pair 160).
    if (gemm && !force_block_n && !fs && !force_pair && !gn_cpg) {
        double lbest = 1e300;
        int lbn = 0;
        for (int bn = 256; bn >= 64; bn -= 16) {   // >= 64: the measured range
            if (n_pad % bn || bn % bn_mult) continue;
            const long long tiles = (long long)m_tiles * (n_pad / bn);
            if (tiles > num_sms) continue;
            const double cost = double(k_blocks) * 2.0 * bn + 2500.0;
            if (cost < lbest) {
                lbest = cost;
                lbn = bn;
            }
        }
        if (lbn) {
            block_n = lbn;
            splits = 1;
            pair = 0;
        }
    }
}

void finish_plan(GemmPlan& p, int m_tiles, int n_pad, int k_blocks, const EpilogueSpec& ep,
                 const GemmScratch& sc, int num_sms, int force_splits, int force_block_n,
                 bool b_mn = false) {
    GemmArgs& a = p.a;
    // the attention epilogues use the GroupNorm scratch region for their row values
    const bool gn = ep.gn_groups > 0 || ep.sm_rowmax;
    int cpg = 0;
    if (ep.gn_groups > 0) {
        if (ep.n_valid % ep.gn_groups)
            throw std::invalid_argument("GroupNorm statistics: channels not divisible by groups");
        cpg = ep.n_valid / ep.gn_groups;
        if (n_pad != ep.n_valid)
            throw std::invalid_argument("GroupNorm statistics need unpadded output channels");
    }
    int bn, splits, pair;
    if (force_block_n > 256) throw std::invalid_argument("GEMM: block_n must be <= 256");
    // MN-major B: whole 128-byte N chunks per tile, single CTA; softmax epilogue: whole K per
    // tile (no split-K)
    // (a CTA pair stages block_n / 2 columns per CTA: block_n a multiple of two chunks)
    const int bn_mult = b_mn ? int(kBlockBytes / elem_bytes(p.elem)) : 16;
    if (b_mn && p.elem != Elem::BF16) throw std::invalid_argument("GEMM: MN-major B is bf16 only");
    choose_tiling(m_tiles, n_pad, k_blocks, num_sms, cpg, force_splits, force_block_n, bn, splits,
                  pair, a.mode == 0, bn_mult);
    if (ep.sm_rowmax) splits = 1;
    if (bn % bn_mult) throw std::invalid_argument("GEMM: block_n must be a multiple of the B chunk");
    if (cpg && bn % cpg) throw std::invalid_argument("GroupNorm statistics: block_n not group aligned");
    if (pair && bn % 16) throw std::invalid_argument("CTA-pair GEMM: block_n % 16 != 0");
    p.pair = pair;
    a.block_n = bn;
    a.n_tiles = n_pad / bn;
    a.k_blocks = k_blocks;
    a.n_pad = n_pad;
    splits = std::min(splits, 2);
    if (splits > 1 && ((size_t)m_tiles * kTileM * n_pad * sizeof(float) > sc.ws_bytes ||
                       2 * size_t(m_tiles) * a.n_tiles > sc.n_tickets))
        splits = 1;
    a.kps = choose_kps(bn, gn, pair);
    if (a.slab) {
        // one stage = three taps (one kernel row) of a chunk; a whole channel chunk (nine
        // taps) per stage where the MMAs are tiny (block_n <= 32: the head conv): a third of
        // the handshakes, the issue loop being the bound there (L62 16.4 -> 13.7 us)
        a.kps = bn <= 32 ? 9 : 3;
    }
    a.splits = splits;
    a.kb_per_split = (k_blocks + splits - 1) / splits;
    a.kb_per_split = (a.kb_per_split + a.kps - 1) / a.kps * a.kps;   // whole stages per split
    if (a.slab) a.kb_per_split = (a.kb_per_split + 8) / 9 * 9;         // whole channel chunks
    a.splits = (k_blocks + a.kb_per_split - 1) / a.kb_per_split;
    a.stages = stages_for(bn, gn, pair, a.kps, a.slab ? a.slab_bytes : 0u);
    a.slab_slots = 2;
    if (a.slab) {
        // deeper slab ring where smem is left over (small block_n: the head conv), never at the
        // cost of B stages; a slab per channel chunk, so no more slots than chunks
        for (int s = kMaxSlabSlots; s > 2; --s) {
            if (s > a.cin_chunks) continue;
            if (smem_for(bn, a.stages, gn, pair, a.kps, a.slab_bytes, s) > size_t(kSmemMax)) continue;
            a.slab_slots = s;
            break;
        }
    }
    a.idesc = make_idesc(p.elem, bn, pair ? 2 * kTileM : kTileM, b_mn);
    a.b_mn = b_mn ? 1 : 0;
    a.sm_rowmax = ep.sm_rowmax;
    a.sm_scale = ep.sm_scale;
    a.sm_ld = ep.sm_ld;
    a.row_scale = ep.row_scale;
    a.out = ep.out;
    a.out_ld = ep.out_ld;
    a.n_valid = ep.n_valid;
    a.out_f32 = ep.out_f32 ? 1 : 0;
    a.round_tf32 = ep.round_tf32 ? 1 : 0;
    a.bias = ep.bias;
    a.residual = ep.residual;
    a.res_ld = ep.res_ld;
    a.scale = ep.scale;
    a.partial = a.splits > 1 ? sc.ws : nullptr;
    a.tile_ticket = sc.tickets;
    if (ep.gn_groups > 0) {
        if (size_t(m_tiles) * ep.gn_groups * 2 > sc.gn_part_len || !sc.gn_ticket)
            throw std::invalid_argument("GroupNorm statistics scratch too small");
        a.gn_groups = ep.gn_groups;
        a.gn_cpg = cpg;
        a.gn_count = double(cpg) * double(a.m_pix);
        a.gn_part = sc.gn_part;
        a.gn_ticket = sc.gn_ticket;
        a.gn_out = ep.gn_out;
    }
    const int P = pair ? 2 : 1;
    const int units = (m_tiles + P - 1) / P * a.n_tiles * a.splits;
    p.grid = P * std::min(units, num_sms / P);
    p.smem = smem_for(bn, a.stages, gn, pair, a.kps, a.slab ? a.slab_bytes : 0u, a.slab_slots);
}

}  // namespace

int device_sm_count() {
    int dev = 0, n = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

void plan_conv(GemmPlan& p, Elem e, const void* in, int rows_in, int W, int C_in_pad, int stride,
               const void* weights, int n_pad, const EpilogueSpec& ep, const GemmScratch& sc,
               int num_sms, int force_splits, int force_block_n) {
    std::memset(&p, 0, sizeof(p));
    p.elem = e;
    const size_t eb = elem_bytes(e);
    const int kel = int(kBlockBytes / eb);
    if (C_in_pad % kel) throw std::invalid_argument("plan_conv: C_in_pad must fill 128-byte blocks");
    if (n_pad % 16) throw std::invalid_argument("plan_conv: n_pad % 16 != 0");
    if (stride != 1 && stride != 2) throw std::invalid_argument("plan_conv: stride must be 1 or 2");
    GemmArgs& a = p.a;
    a.mode = stride == 1 ? 1 : 2;
    const int out_w = stride == 1 ? W : W / 2;
    const int out_rows = stride == 1 ? rows_in : rows_in / 2;
    if (stride == 2 && ((W % 2) || (rows_in % 2)))
        throw std::invalid_argument("plan_conv: stride-2 band must have even rows and width");
    int wb = 1;
    for (int d = std::min(out_w, kTileM); d >= 1; --d)
        if (out_w % d == 0) {
            wb = d;
            break;
        }
    a.w_box = wb;
    a.rows_box = std::min(kTileM / wb, out_rows);
    a.tiles_x = out_w / wb;
    a.tiles_y = (out_rows + a.rows_box - 1) / a.rows_box;
    a.out_rows = out_rows;
    a.out_w = out_w;
    a.cin_chunks = C_in_pad / kel;
    a.m_pix = out_rows * out_w;
    // slab mode: stride 1, one output row per tile (w_box > 64)
    a.slab = (stride == 1 && a.rows_box == 1 && wb + 2 <= 256) ? 1 : 0;
    if (a.slab) {
        a.slab_px = wb + 2;
        a.slab_box_bytes = uint32_t(3 * a.slab_px * kBlockBytes);
        a.slab_bytes = (a.slab_box_bytes + 1023u) / 1024u * 1024u;
    }
    const int k_blocks = 9 * a.cin_chunks;

    // A: 5-D view of the padded band [rows_in+2][W][C_in_pad]
    const int rows_pad = rows_in + 2;
    uint64_t dims[5], strides[4];
    uint32_t box[5];
    const uint64_t pix = uint64_t(C_in_pad) * eb;
    if (stride == 1) {
        dims[0] = C_in_pad; dims[1] = 1; dims[2] = W; dims[3] = 1; dims[4] = rows_pad;
        strides[0] = pix; strides[1] = pix; strides[2] = pix * W; strides[3] = pix * W;
    } else {
        dims[0] = C_in_pad; dims[1] = 2; dims[2] = W / 2; dims[3] = 2; dims[4] = rows_pad / 2;
        strides[0] = pix; strides[1] = 2 * pix; strides[2] = pix * W; strides[3] = 2 * pix * W;
    }
    box[0] = kel; box[1] = 1; box[2] = wb; box[3] = 1; box[4] = a.rows_box;
    if (a.slab) {
        box[2] = a.slab_px;
        box[4] = 3;
    }
    encode(&p.tmA, e, 5, in, dims, strides, box);
    finish_plan(p, a.tiles_y * a.tiles_x, n_pad, k_blocks, ep, sc, num_sms, force_splits,
                force_block_n);
    // B: weights [n_pad][9*C_in_pad] viewed as [K blocks][n_pad][kel]: one box = kps blocks
    if (a.slab) {
        // B as [tap][chunk][n][kel]: box {kel, rows, 1 chunk, 3 taps}
        uint64_t d[4] = {uint64_t(kel), uint64_t(n_pad), uint64_t(a.cin_chunks), 9};
        uint64_t st[3] = {uint64_t(9) * C_in_pad * eb, uint64_t(kBlockBytes), uint64_t(C_in_pad) * eb};
        uint32_t b[4] = {uint32_t(kel), uint32_t(a.block_n / (p.pair ? 2 : 1)), 1, uint32_t(a.kps)};
        encode(&p.tmB, e, 4, weights, d, st, b);
    } else {
        encode_b(&p.tmB, e, weights, n_pad, 9 * C_in_pad, 9LL * C_in_pad, a.block_n / (p.pair ? 2 : 1),
                 a.kps);
    }
    p.flops = 2.0 * a.m_pix * double(ep.n_valid) * 9.0 * C_in_pad;
    a.b_static = 1;   // conv weights
    plan_output_map(p, true);
    a.b_base = weights;
    a.b_bytes = (long long)n_pad * 9 * C_in_pad * (long long)eb;
}

void plan_gemm(GemmPlan& p, Elem e, const void* A, int M, int K, long long lda, const void* B,
               int N, long long ldb, const EpilogueSpec& ep, const GemmScratch& sc, int num_sms,
               int force_splits, int force_block_n, bool b_static) {
    std::memset(&p, 0, sizeof(p));
    p.elem = e;
    const size_t eb = elem_bytes(e);
    const int kel = int(kBlockBytes / eb);
    if (K % kel) throw std::invalid_argument("plan_gemm: K must fill 128-byte blocks");
    GemmArgs& a = p.a;
    a.mode = 0;
    a.tiles_y = (M + kTileM - 1) / kTileM;
    a.tiles_x = 1;
    a.out_rows = M;
    a.out_w = 1;
    a.rows_box = kTileM;
    a.w_box = 1;
    a.cin_chunks = K / kel;
    a.m_pix = M;
    const int n_pad = (N + 15) / 16 * 16;
    uint64_t ad[2] = {uint64_t(K), uint64_t(M)};
    uint64_t as[1] = {uint64_t(lda) * eb};
    uint32_t ab[2] = {uint32_t(kel), uint32_t(kTileM)};
    encode(&p.tmA, e, 2, A, ad, as, ab);
    finish_plan(p, a.tiles_y, n_pad, K / kel, ep, sc, num_sms, force_splits, force_block_n);
    encode_b(&p.tmB, e, B, N, K, ldb, a.block_n / (p.pair ? 2 : 1), a.kps);
    p.flops = 2.0 * double(M) * N * K;
    a.b_static = b_static ? 1 : 0;
    a.up_w = ep.up_w;
    if (ep.up_w && (ep.n_valid % 16 || ep.out_ld % 8 || ep.gn_groups))
        throw std::invalid_argument("plan_gemm: fused upsample needs full 16-column tiles");
    plan_output_map(p, false);
    a.b_base = B;
    a.b_bytes = b_static ? ((long long)(N - 1) * ldb + K) * (long long)eb / 16 * 16 : 0;
}

void plan_gemm_bmn(GemmPlan& p, Elem e, const void* A, int M, int K, long long lda, const void* V,
                   int v_rows, int N, long long ldv, const EpilogueSpec& ep, const GemmScratch& sc,
                   int num_sms) {
    std::memset(&p, 0, sizeof(p));
    p.elem = e;
    const size_t eb = elem_bytes(e);
    const int kel = int(kBlockBytes / eb);
    if (K % kel) throw std::invalid_argument("plan_gemm_bmn: K must fill 128-byte blocks");
    if (N % kel) throw std::invalid_argument("plan_gemm_bmn: N must fill 128-byte chunks");
    if (v_rows > K) throw std::invalid_argument("plan_gemm_bmn: more V rows than K");
    GemmArgs& a = p.a;
    a.mode = 0;
    a.tiles_y = (M + kTileM - 1) / kTileM;
    a.tiles_x = 1;
    a.out_rows = M;
    a.out_w = 1;
    a.rows_box = kTileM;
    a.w_box = 1;
    a.cin_chunks = K / kel;
    a.m_pix = M;
    uint64_t ad[2] = {uint64_t(K), uint64_t(M)};
    uint64_t as[1] = {uint64_t(lda) * eb};
    uint32_t ab[2] = {uint32_t(kel), uint32_t(kTileM)};
    encode(&p.tmA, e, 2, A, ad, as, ab);
    finish_plan(p, a.tiles_y, N, K / kel, ep, sc, num_sms, 0, 0, /*b_mn=*/true);
    // V [v_rows <= K][N] (row stride ldv) as {kel, K, N / kel}: a box {kel, kps * kel, block_n / kel}
    // lands as block_n / kel consecutive [kps * kel rows][128 B] swizzled N chunks; rows >= K
    // (the keys' padding) are zero-filled
    uint64_t d[3] = {uint64_t(kel), uint64_t(v_rows), uint64_t(N / kel)};
    uint64_t st[2] = {uint64_t(ldv) * eb, uint64_t(kBlockBytes)};
    uint32_t b[3] = {uint32_t(kel), uint32_t(a.kps * kel), uint32_t(a.block_n / (p.pair ? 2 : 1) / kel)};
    encode(&p.tmB, e, 3, V, d, st, b);
    p.flops = 2.0 * double(M) * N * K;
    a.b_static = 0;
    plan_output_map(p, false);
}

template <bool kTF32, bool kPair, int kAttn = 0>
void launch_variant(const GemmPlan& p, cudaStream_t s) {
    // the dynamic-smem attribute is per device: remember which devices have it
    static std::mutex mu;
    static unsigned long long done = 0;
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!(done >> dev & 1ull)) {
            CUDA_CHECK(cudaFuncSetAttribute(gemm_kernel<kTF32, kPair, kAttn>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
            done |= 1ull << dev;
        }
    }
    launch_pdl(gemm_kernel<kTF32, kPair, kAttn>, dim3(p.grid), dim3(kThreads), p.smem, s, kPair ? 2 : 1,
               p.tmA, p.tmB, p.tmD, p.a);
}

void launch_gemm(const GemmPlan& p, cudaStream_t s) {
    const int attn = p.a.sm_rowmax ? 1 : p.a.row_scale ? 2 : 0;
    if (p.a.b_mn && (attn != 2 || p.elem != Elem::BF16))
        throw std::logic_error("GEMM: MN-major B is the bf16 attention PV GEMM only");
    if (attn == 1) {
        if (p.elem == Elem::F32) {
            if (p.pair) launch_variant<true, true, 1>(p, s);
            else launch_variant<true, false, 1>(p, s);
        } else {
            if (p.pair) launch_variant<false, true, 1>(p, s);
            else launch_variant<false, false, 1>(p, s);
        }
        return;
    }
    if (attn == 2) {
        if (p.a.b_mn) {
            if (p.pair) launch_variant<false, true, 2>(p, s);
            else launch_variant<false, false, 2>(p, s);
        } else if (p.elem == Elem::F32) {
            if (p.pair) launch_variant<true, true, 3>(p, s);
            else launch_variant<true, false, 3>(p, s);
        } else {
            if (p.pair) launch_variant<false, true, 3>(p, s);
            else launch_variant<false, false, 3>(p, s);
        }
        return;
    }
    if (p.elem == Elem::F32) {
        if (p.pair) launch_variant<true, true>(p, s);
        else launch_variant<true, false>(p, s);
    } else {
        if (p.pair) launch_variant<false, true>(p, s);
        else launch_variant<false, false>(p, s);
    }
}

}  // namespace pp
