// HBM-bound kernels on the hot path (everything that is not a tensor-core GEMM).
// All activations are NHWC bands: `pix` pixels x `ld` channels (ld >= C, padded
// channels hold zeros), element type bf16 (bf16 mode) or fp32 (fp32 mode).
#pragma once
#include "gemm.hpp"

#include <cuda_runtime.h>

#include <cstdint>

namespace pp {

// ---- GroupNorm (proj/src/tensor.cpp:203-277, proj/src/runtime.cpp:85-106) ----------------
// One launch: per-block fp32/fp64 partial sums, folded by the last block (fixed order)
// into stats_out[groups][2] = (mean, mean_sq); `ticket` is a zeroed device counter.
int gn_stats_blocks(long long pix);
void gn_stats(Elem e, const void* x, long long pix, int C, int ld, int groups, double count,
              double* partial, unsigned int* ticket, double* stats_out, cudaStream_t s);

// Which statistics a band normalises with (evaluated in the apply kernel's prologue):
//   GN_USE_LOCAL      fresh local                      (N == 1 sync, or scheme Separate)
//   GN_USE_GLOBAL     weighted device-order mean of all ranks' locals (sync, N > 1)
//   GN_USE_CORRECTED  corrected_gn_stats(fresh, prev_local, prev_global)
//   GN_USE_STALE      prev_global
// all_cur / all_prev are [n][groups][2] tables (rank order); weights = band pixel counts
// (collectives.cpp:150-172 weighting).
enum GnUse : int { GN_USE_LOCAL = 0, GN_USE_GLOBAL = 1, GN_USE_CORRECTED = 2, GN_USE_STALE = 3 };
struct GnCombine {
    int mode;
    const double* fresh;
    const double* all_cur;
    const double* all_prev;
    int n, rank;
    const double* weights;
    float eps;
    int* err;   // set to 1 when a group's variance is negative
};

// Group statistics of a band written by a GroupNorm pass (the next layer's GroupNorm):
// out[G][2] = (mean, mean_sq) of the stored values; partial >= gn_stats_blocks() * G * 2.
struct GnStatsOut {
    int G = 0;                      // 0: off
    double count = 0;               // elements per group (channels/group * pixels)
    double* partial = nullptr;
    unsigned int* ticket = nullptr; // zero; reset by the last block
    double* out = nullptr;
};

// y = GN(x) [-> SiLU] [+ temb[c]] [+ skip]  (fused GroupNorm / SiLU / AddTimeEmb / AddSkip),
// optionally with the statistics of y for a following GroupNorm
void gn_apply(Elem e, const void* x, void* y, long long pix, int C, int ld, int groups,
              const GnCombine& cb, const float* gamma, const float* beta, bool silu,
              const float* temb, const void* skip, bool round_tf32, cudaStream_t s,
              const GnStatsOut* out_stats = nullptr, int up_w = 0);
// up_w > 0: y is the nearest-2x upsample of the result (y is [2 rows][2 up_w] per input row;
// up_w = the input width in pixels)

// ---- pointwise (proj/src/tensor.cpp:297-334, model.cpp:278-298) ---------------------------
void silu(Elem e, const void* x, void* y, long long n, bool round_tf32, cudaStream_t s);
void add(Elem e, const void* x, const void* y, void* out, long long n, bool round_tf32,
         cudaStream_t s);
// out[p][c] = x[p][c] + vec[c]   (AddTimeEmb / CrossAttn broadcast, with optional skip)
void add_channel(Elem e, const void* x, const float* vec, const void* skip, void* out,
                 long long pix, int ld, bool vec_first, bool round_tf32, cudaStream_t s);
void upsample2x(Elem e, const void* x, void* y, int rows, int W, int ld, cudaStream_t s);

// ---- attention helpers (proj/src/tensor.cpp:163-199) -------------------------------------
// Attention between the two tcgen05 GEMMs (gemm.hpp sm_* / row_scale epilogues): P [m][ldp]
// holds each key tile (block_n keys) scaled by its own row max (rowmax[t * ld_rm + r], log2
// units); brings every tile to the row max and writes row_scale[r] = 1 / (sum of row r).
void attn_rescale(Elem e, void* P, long long ldp, int m, int s, const float* rowmax, int n_tiles,
                  int block_n, int ld_rm, float* row_scale, bool round_tf32, cudaStream_t st);
// Vt[c][j] = V[j][c] for j < ns (ld of V = ldv, ld of Vt = ldt): the TF32 PV GEMM's B operand
void transpose(Elem e, const void* V, int ns, int C, long long ldv, void* Vt, long long ldt,
               cudaStream_t s);

// ---- stem im2col (conv2d_region, tensor.cpp:79-130, C_in <= 4) ------------------------------
// in = halo-padded band [rows + 2][W][ld_in]; out[p][tap * 4 + c] for the 9 taps (zero outside
// the image); columns 36..kpad-1 are left untouched (zero).
void stem_im2col(Elem e, const void* in, int rows, int W, int ld_in, int C_in, void* out, int kpad,
                 cudaStream_t s);

// classifier-free guidance: out[i] <- eps_u + scale (eps_c - eps_u), in fp64 (no contraction);
// out may alias eps_c or eps_u
void cfg_combine_eps(float* out, const float* eps_c, const float* eps_u, long long n, double scale,
                     cudaStream_t s);

// --stress-sched: one thread sleeping `us` microseconds on stream s
void stream_sleep(unsigned int us, cudaStream_t s);

// ---- context exchange (displaced patch parallelism) ----------------------------------------
// A batch of exchange copies in ONE launch (in-process transport: every band's halo rows,
// K/V band and GroupNorm statistics of a batch of layers): chunk i = {src, dst, bytes},
// 16-byte aligned, bytes <= 64 KiB (one block per chunk).
struct CopyChunk {
    const void* src;
    void* dst;
    unsigned long long bytes;
};
void copy_chunks(const CopyChunk* chunks_dev, int n, cudaStream_t s);
// Up to four equal-size row copies (null src = skipped) in one small launch: halo pack /
// unpack and the K/V own-band copies on the compute stream.
struct RowCopies {
    const void* src[4];
    void* dst[4];
};
void copy_rows(const RowCopies& c, unsigned long long bytes, cudaStream_t s);

// ---- time embedding / condition projection ----------------------------------------------
// proj[l][c] for every AddTimeEmb layer in one launch: proj = W_l emb + b_l (fp64
// accumulate, fp32 result; layer_time_emb, model.cpp:278-289).  `emb` is the host
// timestep_embedding(t, dim) (model.cpp:220-231), passed by value as a kernel argument.
struct TembLayer {
    const float* W;   // [C][dim] fp32 (reference layout)
    const float* b;   // [C]
    float* out;       // [ld] fp32 (padding stays 0)
    int C;
};
constexpr int kMaxEmb = 960;
struct EmbArg {
    int dim;
    float v[kMaxEmb];
};
void time_projection(const TembLayer* layers_dev, int n_layers, int max_c, const float* emb,
                     int dim, cudaStream_t s);
// The same projections for every timestep of a sampling plan at once:
// table[step][layer][ldt] (fp32) from embs_dev[step][dim].
void time_projection_plan(const TembLayer* layers_dev, int n_layers, int max_c,
                          const float* embs_dev, int n_steps, int dim, float* table, int ldt,
                          cudaStream_t s);
// v[c] = W[c][:] . cond + b[c] in fp64 (project_condition value half, model.cpp:252-263)
void gemv_f64(const float* W, const float* b, const float* x, int rows, int cols, float* out,
              cudaStream_t s);

// ---- sampler / layout conversion -----------------------------------------------------------
// x_nhwc (fp32 band) <- DDIM-eta0 update with eps (sampler.cpp:46-61, fp64 math) and the
// next step's stem input (T, NHWC, ld channels) refreshed in the same pass.
void ddim_update(const float* x, const float* eps, float* x_out, long long n, int C,
                 double abar_t, double abar_n, Elem e, void* stem, int stem_ld, cudaStream_t s);
// NCHW fp32 rows [r0, r0+rows) of a (C, H, W) image -> NHWC band (T or fp32) with ld.
void nchw_to_nhwc(const float* src, int C, int H, int W, int r0, int rows, Elem e, void* dst,
                  int ld, bool round_tf32, cudaStream_t s);
// NHWC band (T or fp32) -> NCHW fp32 band (C, rows, W); sets *nonfinite if any value is
// not finite (require_finite, tensor.cpp:36-42).
void nhwc_to_nchw(Elem e, const void* src, int ld, int C, int rows, int W, float* dst,
                  int* nonfinite, cudaStream_t s);
void nhwc_f32_to_nchw(const float* src, int C, int rows, int W, float* dst, int* nonfinite,
                      cudaStream_t s);
void f32_to_elem(const float* src, Elem e, void* dst, long long n, bool round_tf32,
                 cudaStream_t s);
// Naive-patch helpers (step_naive, proj/src/runtime.cpp:398-452): crop rows [y0, y0+rows) x
// cols [x0, x0+cols) of an NCHW fp32 image into an NHWC patch (T, ld), and scatter an NHWC
// fp32 patch (C channels) back into an NCHW fp32 image at (y0, x0).
void crop_nchw_to_nhwc(const float* src, int C, int H, int W, int y0, int x0, int rows, int cols,
                       Elem e, void* dst, int ld, bool round_tf32, cudaStream_t s);
void scatter_nhwc_to_nchw(const float* patch, int C, int rows, int cols, float* dst, int H, int W,
                          int y0, int x0, int* nonfinite, cudaStream_t s);
void elem_to_f32(Elem e, const void* src, float* dst, long long n, cudaStream_t s);

}  // namespace pp
