// Host interface of the sm_100a tcgen05 GEMM / implicit-GEMM conv kernel.
//
// One persistent, warp-specialised kernel serves every tensor-core op on the
// hot path:
//   * conv2d_region  (proj/src/tensor.cpp:79-130)  -> implicit GEMM, A operand
//     gathered by 5-D TMA boxes straight out of the halo-padded NHWC band,
//     M = output pixels, N = C_out, K = 9 * C_in (tap-major, channel-minor);
//   * linear         (proj/src/tensor.cpp:139-161) -> plain GEMM;
//   * attention      (proj/src/tensor.cpp:163-199) -> S = Q K^T and O = P V^T.
// Operands are staged by TMA into 128B-swizzled shared memory, multiplied by
// tcgen05.mma (kind::f16 for bf16, kind::tf32 for the fp32 mode) into a
// double-buffered TMEM accumulator, and drained by twelve epilogue warps that
// add bias / residual, store NHWC rows and (optionally) fold the stored values
// into GroupNorm statistics of the next layer (group_stats, tensor.cpp:203-235).
// Split-K (2-way) is reduced inside the kernel: the split that finishes first
// publishes its fp32 partial tile, the second adds it to its own TMEM accumulator
// (fp32 addition is commutative -> deterministic), no second launch.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pp {

enum class Elem : int { BF16 = 0, F32 = 1 };  // F32: fp32 storage, TF32 tensor-core multiply

inline size_t elem_bytes(Elem e) { return e == Elem::BF16 ? 2 : 4; }

struct GemmArgs {
    int mode;                 // 0 = plain row-major A (2-D map), 1 = conv stride 1, 2 = conv stride 2
    int rows_box, w_box;      // conv: output rows / cols covered by one 128-row M tile
    int tiles_y, tiles_x;     // M-tile grid (plain: tiles_y = ceil(M/128), tiles_x = 1)
    int out_rows, out_w;      // valid output extent in pixels (plain: M, 1)
    int n_tiles, block_n;     // N tiling (block_n % 16 == 0, <= 256)
    int cin_chunks;           // conv: channel chunks of 128 B per tap; plain: k_blocks
    int k_blocks;             // total 128-byte K blocks
    int splits, kb_per_split; // split-K
    int stages;               // smem pipeline depth
    int kps;                  // 128-byte K blocks per pipeline stage (1 or 2; slab mode 3 or 9)
    // slab mode (stride-1 conv, rows_box == 1): A from a 2-slot ring of im2col slabs
    // [3 rows][slab_px = w_box + 2][128 B] shared by the nine taps of a channel chunk; the
    // K index is chunk * 9 + tap (three taps per stage), B comes from a 4-D map
    int slab;
    int slab_slots;           // slab ring depth (2..4: deeper when small block_n leaves smem free)
    int slab_px;
    uint32_t slab_bytes;      // smem per slot (1024-aligned)
    uint32_t slab_box_bytes;  // TMA bytes per slab
    uint32_t idesc;           // tcgen05 instruction descriptor
    // epilogue
    void* out;                // output base (already offset to pixel 0 of the band)
    long long out_ld;         // elements between consecutive output pixels / rows
    int n_valid;              // columns actually stored
    int out_f32;              // 1: fp32 output, 0: bf16 (bf16 mode) ; fp32 mode always fp32
    int round_tf32;           // fp32 mode: round stored values to tf32 (they feed another GEMM)
    const float* bias;        // [n] or null
    const void* residual;     // same element type/layout as out (ld = res_ld) or null
    long long res_ld;
    float scale;              // multiplier applied to the accumulator before bias (1 = none)
    // split-K workspace
    float* partial;           // [m_pix][n_pad] fp32: the first split's partial tiles
    unsigned int* tile_ticket;// [m_tiles * n_tiles][2] (ticket, ready), zero, reset by the second split
    int m_pix, n_pad;
    // fused GroupNorm statistics of the stored output (gn_groups == 0: off)
    int gn_groups, gn_cpg;
    double gn_count;          // elements per group (cpg * pixels)
    double* gn_part;          // [m_tiles][groups][2]
    unsigned int* gn_ticket;  // [1 + n_tiles] zeroed counters, each reset by its folder
    double* gn_out;           // [groups][2] = (mean, mean_sq)
    const void* b_base;       // B tensor (weights) and its size: with b_static, every CTA
    long long b_bytes;        // prefetches its 1/grid slice into L2 at kernel start
    int tma_store;            // 1: the CTA's last tile is stored through tmD (smem staging)
    int up_w;                 // > 0: store the nearest-2x upsample (output row p of an up_w-wide
                              //      map -> 2x2 block of the 2 up_w-wide output)
    int b_static;             // 1: B is weights (not written by an earlier kernel on the stream):
                              //    its first boxes are prefetched before griddepcontrol.wait
    int debug;                // micro-benchmarks only (compiled out unless -DPP_GEMM_DEBUG)
    // attention (tensor.cpp:163-199) as two GEMMs around a TMEM-side softmax:
    //  S GEMM (sm_rowmax != null): the epilogue finds each row's max over the tile's keys in
    //    TMEM, stores P = exp(S * sm_scale - tile max) (<= 1) and the tile max (log2 units) at
    //    sm_rowmax[nt * sm_ld + r]; attn_rescale then brings every tile to the row max and
    //    sums the row;
    //  PV GEMM (row_scale != null): row r of the accumulator is multiplied by row_scale[r]
    //    (1 / row sum).
    float* sm_rowmax;
    float sm_scale;
    int sm_ld;
    const float* row_scale;
    int b_mn;                 // B operand MN-major: B = [K][N] with N contiguous (V rows)
};

struct GemmPlan {
    CUtensorMap tmA;
    CUtensorMap tmB;
    CUtensorMap tmD;          // output (TMA-store epilogue)
    GemmArgs a;
    int grid = 0;
    size_t smem = 0;
    Elem elem = Elem::BF16;
    int pair = 0;             // 1: CTA-pair (cta_group::2, M = 256) kernel, clusters of 2
    double flops = 0;         // algorithmic 2*M*N*K of the layer (for rooflines)
};

struct EpilogueSpec {
    void* out = nullptr;
    long long out_ld = 0;
    int n_valid = 0;
    bool out_f32 = false;
    bool round_tf32 = false;
    const float* bias = nullptr;
    const void* residual = nullptr;
    long long res_ld = 0;
    float scale = 1.0f;
    // GroupNorm statistics of the output (groups == 0: off)
    int gn_groups = 0;
    double* gn_out = nullptr;
    int up_w = 0;             // plain GEMM: > 0 = fused nearest-2x upsample of the output
    // attention epilogues (GemmArgs::sm_* / row_scale)
    float* sm_rowmax = nullptr;
    float sm_scale = 0.0f;
    int sm_ld = 0;
    const float* row_scale = nullptr;
};

// Scratch shared by all GEMMs issued on one stream (they run one after another).
struct GemmScratch {
    float* ws = nullptr;
    size_t ws_bytes = 0;
    unsigned int* tickets = nullptr;   // >= max tiles, zeroed
    size_t n_tickets = 0;
    double* gn_part = nullptr;         // >= max m_tiles * groups * 2
    size_t gn_part_len = 0;
    unsigned int* gn_ticket = nullptr; // zeroed counters: [1 + N tiles] (>= 256)
};

// Conv over a halo-padded NHWC band: in = [rows_in + 2][W][C_in_pad] (row 0 = the halo
// row above the band, row rows_in + 1 = the halo row below). weights = [n_pad][9][C_in_pad]
// (K-major). Output pixel (oy, ox) of the band is stored at out + (oy*out_w + ox)*out_ld.
void plan_conv(GemmPlan& p, Elem e, const void* in, int rows_in, int W, int C_in_pad, int stride,
               const void* weights, int n_pad, const EpilogueSpec& ep, const GemmScratch& sc,
               int num_sms, int force_splits = 0, int force_block_n = 0);

// Plain GEMM: D[M][N] = A[M][K] * B[N][K]^T (both K-major, leading dims in elements).
// b_static: B holds weights that no kernel on the stream writes (prefetched under PDL).
void plan_gemm(GemmPlan& p, Elem e, const void* A, int M, int K, long long lda, const void* B,
               int N, long long ldb, const EpilogueSpec& ep, const GemmScratch& sc, int num_sms,
               int force_splits = 0, int force_block_n = 0, bool b_static = false);

// Attention PV GEMM: D[M][N] = P[M][K] * V[K][N] with V row-major (N contiguous, leading
// dim ldv): the B operand is staged MN-major by TMA straight from V (no transpose).
// V has v_rows <= K rows; rows v_rows..K-1 read as zero.
void plan_gemm_bmn(GemmPlan& p, Elem e, const void* A, int M, int K, long long lda, const void* V,
                   int v_rows, int N, long long ldv, const EpilogueSpec& ep, const GemmScratch& sc,
                   int num_sms);

void launch_gemm(const GemmPlan& p, cudaStream_t s);



int device_sm_count();

}  // namespace pp
