/*
 * pp_b200.h — C ABI of the B200-native displaced-patch-parallel runtime.
 *
 * This is the drop-in boundary for the reference's hot path (patchsim,
 * /root/reference/proj).  Every entry point cites the reference interface it
 * replaces.  Conventions:
 *   - plain pointers and sizes only; tensors are NCHW fp32 like patchsim::Tensor
 *     (proj/include/patchsim/tensor.hpp:16-29) unless a function says "device";
 *   - caller-allocated outputs; opaque handles own all device memory;
 *   - status codes: PP_EINVAL  <-> std::invalid_argument (CLI exit 2),
 *                   PP_ERUNTIME <-> std::runtime_error    (CLI exit 1),
 *     with the reference's message text available from pp_last_error()
 *     (thread-local), e.g. "not divisible", "no cached activation for layer".
 *   - no CPU fallback: every compute entry point runs sm_100a kernels and
 *     returns PP_ECUDA when no usable B200 is present.
 */
#ifndef PP_B200_H
#define PP_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(PP_BUILDING_LIB)
#define PP_API __attribute__((visibility("default")))
#else
#define PP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PP_OK 0
#define PP_EINVAL 1
#define PP_ERUNTIME 2
#define PP_ECUDA 3
#define PP_ENCCL 4

/* compute precision: bf16 storage + bf16 tensor cores (fp32 accumulate), or fp32
 * storage + TF32 tensor cores (fp32 accumulate) */
#define PP_DTYPE_BF16 0
#define PP_DTYPE_FP32 1

/* RunMode, proj/include/patchsim/runtime.hpp:20 */
#define PP_MODE_REFERENCE 0
#define PP_MODE_NAIVE 1
#define PP_MODE_SYNC 2
#define PP_MODE_DISPLACED 3
/* GnScheme, proj/include/patchsim/runtime.hpp:21 */
#define PP_GN_CORRECTED 0
#define PP_GN_STALE 1
#define PP_GN_SEPARATE 2
/* exchange transport of the multi-process layout (world > 1) */
#define PP_TRANSPORT_NCCL 0
#define PP_TRANSPORT_IPC 1
/* step entries, PatchRunner::run_step / step_* (proj/include/patchsim/runtime.hpp:64-71) */
#define PP_STEP_RUN 0
#define PP_STEP_REFERENCE 1
#define PP_STEP_NAIVE 2
#define PP_STEP_SYNC 3
#define PP_STEP_DISPLACED 4

PP_API const char* pp_last_error(void);
PP_API int pp_version(void);
/* programmatic dependent launch on (1, default) / off (0) for later launches and graph
 * captures; off is a measurement control (strictly serialised kernels, exact per-kernel
 * device times), results are identical either way */
PP_API void pp_set_pdl(int on);
/* number of visible CUDA devices with compute capability 10.x (0 on a CPU-only host) */
PP_API int pp_device_count(void);

/* ---- model: ModelConfig / LayerDescriptor / build_model -------------------------------
 * proj/include/patchsim/model.hpp:30-59, proj/src/model.cpp:158-218 */
typedef struct {
    int in_channels, base_channels, levels, groups, cond_dim, attn_at_level;
    /* deeper graphs (beyond the reference API; 0 = the reference graph): residual blocks per
     * level (0 -> 1), attention-level bit mask (0 -> attn_at_level only), attention blocks
     * after each residual block there (0 -> 1), attention on the up path too (0 / 1) */
    int res_blocks, attn_levels, attn_depth, attn_up;
} pp_model_config;

typedef struct {
    int id, kind; /* LayerKind order of model.hpp:15-26 */
    int in_ch, out_ch, kernel, stride, pad, groups;
    float eps;
    int cond_dim, skip_source, scale_in, scale_out;
    int weight, bias, weight2, bias2; /* weight-pool handles, -1 when absent */
} pp_layer_desc;

typedef struct pp_model pp_model;

/* build_model(cfg, seed): host splitmix64 init, bit-identical to the reference pool */
PP_API int pp_model_build(const pp_model_config* cfg, uint64_t seed, pp_model** out);
/* layer graph of cfg with weights taken from a caller pool laid out like
 * dump_weights (proj/src/io.cpp:133-143): every pool tensor in handle order */
PP_API int pp_model_from_pool(const pp_model_config* cfg, const float* pool, size_t pool_len,
                              pp_model** out);
PP_API void pp_model_destroy(pp_model* m);
PP_API int pp_model_num_layers(const pp_model* m);
PP_API int pp_model_layer(const pp_model* m, int id, pp_layer_desc* out);
PP_API int pp_model_num_weights(const pp_model* m);
PP_API int pp_model_weight_shape(const pp_model* m, int handle, int* nchw4);
PP_API size_t pp_model_pool_size(const pp_model* m);
PP_API int pp_model_pool(const pp_model* m, float* dst);
/* zero_weights (proj/src/model.cpp:375-388) */
PP_API int pp_model_zero_weights(pp_model* m, int keep_biases);
/* model_total_macs (proj/src/costmodel.cpp:64-71) */
PP_API uint64_t pp_model_total_macs(const pp_model* m, int h, int w);

/* ---- host-side partition logic (proj/src/runtime.cpp:46-83, 480-492) ------------------- */
PP_API int pp_partition_rows(int h, int n_devices, int full_w, int* out4n);
/* writes L (row_start,row_end,full_h,full_w) regions to layer_in4 and layer_out4 */
PP_API int pp_derive_patch_spec(const pp_model* m, const int* region4, int* layer_in4,
                                int* layer_out4);
/* corrected_gn_stats (proj/src/runtime.cpp:85-106); each stats arg = mean[g] then mean_sq[g] */
PP_API int pp_corrected_gn_stats(int groups, const double* fresh_local, const double* prev_local,
                                 const double* prev_global, double* out);
/* RunConfig::validate (proj/src/runtime.cpp:480-492) */
typedef struct {
    int mode, n_devices, h, w, num_steps, warmup, gn_scheme, dtype;
    uint64_t model_seed, noise_seed, cond_seed;
    pp_model_config model;
    int schedule_steps;
    double beta_start, beta_end;
} pp_run_config;
PP_API void pp_run_config_default(pp_run_config* cfg);
PP_API int pp_run_config_validate(const pp_run_config* cfg);
/* make_schedule / make_plan (proj/src/sampler.cpp:17-44) */
PP_API int pp_make_schedule(int total_steps, double beta_start, double beta_end, double* abar);
PP_API int pp_make_plan(int total_steps, int num_steps, int* timesteps);
PP_API int pp_random_normal(int n, int c, int h, int w, uint64_t seed, float* out);
PP_API int pp_random_condition(int dim, uint64_t seed, float* out);
PP_API uint64_t pp_macs_of_layer(const pp_model* m, int layer, const int* region4);

/* ---- PatchRunner (proj/include/patchsim/runtime.hpp:57-80) ------------------------------ */
typedef struct {
    int mode;         /* PP_MODE_* */
    int n_devices;    /* patches (row bands) */
    int warmup_steps; /* displaced: sync steps after the first (default 4) */
    int gn_scheme;    /* PP_GN_* */
    int dtype;        /* PP_DTYPE_* */
    /* process layout: world == 1 runs all n_devices bands in this process, on CUDA device
     * `device` (a single-GPU simulation of the N-device run); world == n_devices runs
     * band `rank` only on its own GPU, exchanging with the other ranks over NCCL
     * (nccl_id = the 128-byte ncclUniqueId shared by all ranks) or CUDA IPC */
    int world, rank;
    const void* nccl_id;
    int device;       /* CUDA device of band 0 (world == 1) or of this rank */
    int profile;      /* record per-kernel CUDA events (pp_runner_profile) */
    int transport;    /* world > 1: PP_TRANSPORT_NCCL (nccl_id) or PP_TRANSPORT_IPC (CUDA IPC
                       * peer mappings + copy engines; pp_runner_ipc_export / _connect before
                       * the first step; graph-captured like NCCL) */
    int no_comm;      /* ablation only, the paper's "No Comm." row: every
                       * exchange (halo rows, K/V, GroupNorm statistics) is skipped and each
                       * band normalises with its own statistics; compute is identical, the
                       * results are NOT the reference's.  Default 0. */
    int stress;       /* --stress-sched (proj/src/collectives.cpp:45-56): perturb the device
                       * schedule around every exchange with seeded sleep kernels on the
                       * compute and exchange streams; results must not change.  Default 0. */
    unsigned long long stress_seed;   /* default 0xC0FFEE */
    /* classifier-free guidance (beyond the reference API): cfg_scale != 0 runs a second,
     * unconditional U-Net pass per step (condition `uncond`, cond_dim floats; NULL = zeros)
     * concurrently with the conditional one and denoises with
     * eps = eps_u + cfg_scale (eps_c - eps_u).  world > 1 with NCCL: cfg_nccl_id = a second
     * ncclUniqueId for the unconditional pass.  Default 0 (off). */
    double cfg_scale;
    const float* uncond;
    const void* cfg_nccl_id;
    /* condition tokens (beyond the reference API, which projects one): cond (and uncond) hold
     * cond_tokens x model cond_dim floats and every CrossAttn layer attends over the
     * cond_tokens projected rows; default 1 (the reference's layer_cross_attn exactly) */
    int cond_tokens;
    /* CFG batch split across two GPU groups (beyond the reference API):
     * cfg_pair_role 0 / 1 = this rank runs only the conditional / unconditional pass of its
     * band (conditioned on cond / uncond -- both ranks of a pair pass the same two) and swaps
     * eps bands with its partner after every pass; both then hold the same guided latent.
     * cfg_pair_transport: PP_TRANSPORT_NCCL (a two-rank communicator per pair, cfg_nccl_id =
     * its ncclUniqueId) or PP_TRANSPORT_IPC (pp_runner_pair_export / _connect); both
     * graph-captured.  One band per process.  Default -1: both passes in this runner (cfg_scale). */
    int cfg_pair_role;
    int cfg_pair_transport;
} pp_runner_opts;
PP_API void pp_runner_opts_default(pp_runner_opts* o);

typedef struct pp_runner pp_runner;

/* PatchRunner(model, cond, h, w, opts); the model is copied to the device */
PP_API int pp_runner_create(const pp_model* m, const float* cond, int cond_dim, int h, int w,
                            const pp_runner_opts* opts, pp_runner** out);
PP_API void pp_runner_destroy(pp_runner* r);
/* run_step / step_reference / step_naive / step_sync / step_displaced
 * (runtime.cpp:382-476): x and eps are full NCHW (1, C, h, w) fp32 host buffers */
PP_API int pp_runner_step(pp_runner* r, int entry, const float* x, int t, int step_index,
                          float* eps);
/* PatchSpec of one band: L layer_in regions then L layer_out regions (4 ints each) */
PP_API int pp_runner_patch_spec(const pp_runner* r, int device, int* layer_in4, int* layer_out4);
/* cached_input(device, layer): the full-shape context the band's gather layer last used
 * (stale full map, halo rows or K/V) as NCHW fp32; returns element count, 0 if absent */
PP_API long pp_runner_cached_input(pp_runner* r, int device, int layer, float* dst, int* nchw4);
PP_API uint64_t pp_runner_total_macs(const pp_runner* r);
PP_API int pp_runner_step_device_macs(const pp_runner* r, int step, uint64_t* per_device);
/* bytes this runtime actually moved: {allgather_recv, allgather_sent, halo_recv, halo_sent,
 * statreduce_recv, statreduce_sent} (CommVolumes, proj/include/patchsim/trace.hpp:37-52) */
PP_API int pp_runner_volumes(const pp_runner* r, uint64_t* v6);
/* RawTrace of one device (PatchRunner::trace(), proj/include/patchsim/runtime.hpp:71): rows
 * of 9 uint64 {device, step, layer, kind (0 Compute/1 Post/2 Wait), prim (0 AllGather/
 * 1 Halo/2 StatReduce), macs, bytes_recv, bytes_sent, tag}; Post bytes follow the
 * reference hub's accounting.  Returns the event count (-1 on error); out9 may be NULL. */
PP_API long pp_runner_trace(const pp_runner* r, int device, uint64_t* out9, long cap);
/* sample() (proj/src/sampler.cpp:76-95) with the DDIM-eta0 update on the GPU:
 * x_T (NCHW host), plan timesteps, alpha_bar table; x0 out; trajectory optional
 * (num_steps model inputs x_t, NCHW). */
PP_API int pp_runner_sample(pp_runner* r, const float* x_T, const int* timesteps, int num_steps,
                            const double* alpha_bar, int schedule_steps, float* x0,
                            float* trajectory);
/* per-kernel-class device time of the last sample()/step with profile=1:
 * out[0] = conv GEMM ms, out[1] = conv flops, out[2] = all GEMM ms, out[3] = all GEMM flops,
 * out[4] = GN ms, out[5] = other ms, out[6] = launches */
PP_API int pp_runner_profile(pp_runner* r, double* out7);
/* kernels launched by the last step / sample call */
PP_API long pp_runner_launches(const pp_runner* r);
/* device time (CUDA events on the band compute streams, max over local bands) of the
 * last pp_runner_sample denoising loop, excluding the x_T upload and x0 download */
PP_API double pp_runner_last_device_ms(const pp_runner* r);
/* switch per-kernel CUDA-event timing on/off (resets the pp_runner_profile totals) */
PP_API int pp_runner_set_profile(pp_runner* r, int on);
/* ncclGetUniqueId for the multi-process (one rank per GPU) layout */
/* CFG pair link over CUDA IPC (cfg_pair_transport == PP_TRANSPORT_IPC): this rank's handle
 * blob (call with out = NULL for the size), then connect with the partner's blob before the
 * first step.  Replaces nothing in the reference (beyond its API). */
PP_API int pp_runner_pair_export(pp_runner* r, void* out, long cap, long* size);
PP_API int pp_runner_pair_connect(pp_runner* r, const void* blob, long size);
PP_API int pp_nccl_unique_id(void* out128);
/* PP_TRANSPORT_IPC: this rank's CUDA IPC handle blob (receive buffers + flags); *size = its
 * byte count, copied to out when cap suffices.  Replaces the hub registration of
 * CollectiveHub (proj/src/collectives.cpp:62-115) for one-process-per-GPU runs. */
PP_API int pp_runner_ipc_export(pp_runner* r, void* out, long cap, long* size);
/* every rank's blob concatenated in rank order (per_rank bytes each); opens the peers'
 * mappings.  Must precede the first step. */
PP_API int pp_runner_ipc_connect(pp_runner* r, const void* blobs, long per_rank);
/* host stitching of a rank-ordered band all-gather [n][c][rows][w] into NCHW (c, n*rows, w),
 * as run_workers stitches eps rows (proj/src/runtime.cpp:368-377) */
PP_API int pp_assemble_bands(const float* gathered, int n_bands, int c, int rows, int w,
                             float* out);

/* ---- run_sampling (proj/src/runtime.cpp:494-526) ------------------------------------------ */
PP_API int pp_run_sampling(const pp_run_config* cfg, float* x0, float* trajectory,
                           uint64_t* total_macs);

/* ---- kernel-level operators (proj/src/tensor.cpp), host NCHW fp32 in / out ---------------- */
PP_API int pp_conv2d_region(int dtype, const float* x, int n, int c, int h, int w, int row_start,
                            int row_end, const float* weight, int c_out, int k, const float* bias,
                            int stride, int pad, float* out);
PP_API int pp_linear(int dtype, const float* tokens, int n, int t, int in_f, const float* weight,
                     int out_f, const float* bias, float* out);
PP_API int pp_attention(int dtype, const float* q, const float* k, const float* v, int n, int m,
                        int s, int d, int dv, float scale, float* out);
PP_API int pp_group_stats(int dtype, const float* x, int n, int c, int h, int w, int groups,
                          int row_start, int row_end, double* mean, double* mean_sq);
PP_API int pp_group_norm_apply(int dtype, const float* x, int n, int c, int h, int w,
                               int row_start, int row_end, int groups, const double* mean,
                               const double* mean_sq, const float* gamma, const float* beta,
                               float eps, float* out);
PP_API int pp_silu(int dtype, const float* x, long count, float* out);
PP_API int pp_upsample_nearest2x(int dtype, const float* x, int n, int c, int h, int w,
                                 float* out);
PP_API int pp_ddim_update(const float* x, const float* eps, long count, double abar_t,
                          double abar_next, float* out);

/* ---- device-pointer GEMM entry (unit tests / benchmarks of the tcgen05 kernel) -------------- */
/* D[M][N] (fp32 or dtype, ld = ldd) = A[M][K] * B[N][K]^T (+ bias), all device pointers */
PP_API int pp_dev_gemm(int dtype, const void* A, int M, int K, long long lda, const void* B, int N,
                       long long ldb, const float* bias, void* D, long long ldd, int out_f32,
                       int force_splits, int force_block_n, void* stream);
/* implicit-GEMM 3x3 conv over a halo-padded NHWC band (device pointers):
 * in [rows+2][W][C_in_pad], weights [n_pad][3][3][C_in_pad], out pixel p at D + p*ldd */
PP_API int pp_dev_conv(int dtype, const void* in, int rows, int W, int C_in_pad, int stride,
                       const void* weights, int n_pad, int c_out, const float* bias, void* D,
                       long long ldd, int out_f32, const void* residual, long long res_ld,
                       int force_splits, int force_block_n, void* stream);

/* micro-benchmark of the tcgen05 kernel: kind 0 = GEMM [M][K]x[N][K]^T, 1/2 = implicit
 * 3x3 conv stride 1/2 over a padded band (rows, W, K = C_in); ms_out[5] = {ms per launch,
 * block_n, splits, stages, grid} */
PP_API int pp_dev_gemm_bench(int dtype, int kind, int M_or_rows, int W, int K, int N,
                             int force_splits, int force_block_n, int reps, double* ms_out);

/* micro-benchmark of the fused GroupNorm apply / statistics kernels on a [pix][C] band:
 * out[2] = {us per gn_apply, us per gn_stats}; flags: 1 SiLU, 2 temb, 4 skip */
PP_API int pp_dev_gn_bench(int dtype, long long pix, int C, int G, int flags, int reps,
                           double* out);

#ifdef __cplusplus
}
#endif
#endif /* PP_B200_H */
