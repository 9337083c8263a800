// B200 host runtime for displaced patch parallelism.
//
// Replaces PatchRunner (proj/include/patchsim/runtime.hpp:57-108,
// proj/src/runtime.cpp:110-476).  Each row band ("device" in the reference) is a
// Program: the layer graph compiled for that band's geometry into fused
// sm_100a launches on the band's CUDA device, with its own compute stream and
// comm stream.  Context exchange follows the reference's step semantics
// exactly (posted at layer l of step s, consumed at layer l of step s+1 in
// displaced steps; posted and consumed in the same step in synchronous ones),
// but moves only what the operators read:
//   Conv / DownConv  -> one halo row from each neighbour (DownConv: the row above);
//   SelfAttn         -> the full K/V map (all-gather of the bands);
//   GroupNorm        -> per-group (mean, mean_sq) of every band (all-gather).
// Stale context lives in parity double buffers indexed by step % 2.
#pragma once
#include "gemm.hpp"
#include "kernels.hpp"
#include "model.hpp"

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace pp {

enum RunMode : int { MODE_REFERENCE = 0, MODE_NAIVE = 1, MODE_SYNC = 2, MODE_DISPLACED = 3 };
enum GnScheme : int { GN_CORRECTED = 0, GN_STALE = 1, GN_SEPARATE = 2 };
enum StepEntry : int { STEP_RUN = 0, STEP_REFERENCE = 1, STEP_NAIVE = 2, STEP_SYNC = 3, STEP_DISPLACED = 4 };

struct RunnerOptions {
    int mode = MODE_REFERENCE;
    int n_devices = 1;
    int warmup = 4;
    int gn_scheme = GN_CORRECTED;
    Elem elem = Elem::BF16;
    int world = 1, rank = 0;          // world > 1: one band per process, NCCL exchange
    std::vector<uint8_t> nccl_id;     // 128-byte ncclUniqueId (world > 1, NCCL transport)
    int transport = 0;                // world > 1: 0 NCCL, 1 CUDA IPC + copy engines
    int device = 0;                   // CUDA device of every local band / of this rank
    bool profile = false;
    bool no_comm = false;             // ablation ("No Comm."): exchanges skipped, local GN stats
    bool stress = false;              // scheduling noise around the exchanges (determinism check)
    uint64_t stress_seed = 0xC0FFEE;
    // classifier-free guidance (beyond the reference API): cfg_scale != 0
    // runs the U-Net a second time per step under the `uncond` condition (zeros if empty) on
    // its own band streams, concurrently with the conditional pass, and denoises with
    // eps = eps_u + cfg_scale (eps_c - eps_u).  world > 1 + NCCL: cfg_nccl_id = the id of the
    // unconditional pass's communicator.
    double cfg_scale = 0.0;
    std::vector<float> uncond;
    // condition tokens (beyond the reference API, which has one): cond holds cond_tokens x
    // cond_dim floats and every CrossAttn layer attends over the cond_tokens projected rows
    int cond_tokens = 1;
    std::vector<uint8_t> cfg_nccl_id;
    // CFG batch split across two GPU groups (beyond the reference API): cfg_pair_role 0 / 1 =
    // this rank runs only the conditional / unconditional pass of its band (conditioned on
    // `cond` / `uncond`) and swaps eps bands with its partner rank after every pass over
    // cfg_pair_transport (0: a two-rank NCCL communicator, id cfg_nccl_id; 1: CUDA IPC,
    // pair_export / pair_connect).  -1 (default): both passes in this runner.
    int cfg_pair_role = -1;
    int cfg_pair_transport = 0;
};

struct CommVolumes {
    uint64_t allgather_recv = 0, allgather_sent = 0;
    uint64_t halo_recv = 0, halo_sent = 0;
    uint64_t statreduce_recv = 0, statreduce_sent = 0;
};

// One entry of the reference's RawTrace (proj/include/patchsim/trace.hpp:18-35): per-device
// program order, no wall clock.  kind 0 Compute / 1 Post / 2 Wait; prim 0 AllGather / 1 Halo /
// 2 StatReduce.  Post bytes use the reference hub's accounting (the full fp32 layer input
// gathered to every device, collectives.cpp:70-72) so simulate_timeline sees the same
// trace; the bytes the B200 runtime actually moves (halo rows, K/V bands, stats) are
// reported separately by volumes().
struct TraceEvent {
    int device = 0, step = 0, layer = -1, kind = 0, prim = 0;
    uint64_t macs = 0, bytes_recv = 0, bytes_sent = 0, tag = 0;
};

struct ProfileTotals {
    double conv_ms = 0, conv_flops = 0, gemm_ms = 0, gemm_flops = 0, gn_ms = 0, other_ms = 0;
    long launches = 0;
};

struct DeviceWeights;  // packed weights on one CUDA device
struct Program;        // one band compiled for one CUDA device
class Transport;
class PairLink;
struct XItem;

class Runner {
public:
    Runner(const Model& m, const std::vector<float>& cond, int h, int w, const RunnerOptions& o);
    ~Runner();
    Runner(const Runner&) = delete;
    Runner& operator=(const Runner&) = delete;

    // run_step / step_* (runtime.cpp:382-476): full NCHW host x and eps.
    void step(int entry, const float* x, int t, int step_index, float* eps);
    // sample() (sampler.cpp:76-95) with the DDIM update on the GPU.
    void sample(const float* x_T, const int* timesteps, int num_steps, const double* abar,
                int schedule_steps, float* x0, float* trajectory);

    const PatchSpec& patch_spec(int device) const;
    long cached_input(int device, int layer, float* dst, int* nchw4);
    uint64_t total_macs() const { return total_macs_ + (cfg_ ? cfg_->total_macs() : 0); }
    const std::vector<TraceEvent>& trace(int device) const;
    std::vector<uint64_t> step_device_macs(int step) const;
    CommVolumes volumes() const;
    ProfileTotals profile() const { return prof_; }
    long launches() const { return launches_; }
    // device time (CUDA events on the band compute streams, max over local bands) of the
    // last sample()'s denoising loop, excluding the x_T upload and x0 download
    double last_device_ms() const { return last_device_ms_; }
    int n_devices() const { return n_dev_; }
    void set_profile(bool on);
    // IPC transport (world > 1, transport 1): this rank's handle blob, then every rank's blob
    std::vector<uint8_t> ipc_export();
    void ipc_connect(const uint8_t* blobs, size_t per_rank);
    // CFG pair link over CUDA IPC: this rank's handle blob, then the partner's
    std::vector<uint8_t> pair_export();
    void pair_connect(const uint8_t* blob, size_t size);

private:
    friend struct Program;
    friend class Transport;
    void check_displaced_ready(int step_index) const;
    // eps left on the devices; `progs` is bands_ (exchanging bands) or a naive patch program
    void run_bands(std::vector<std::unique_ptr<Program>>& progs, int t, int step_index,
                   bool displaced);
    void run_bands(int t, int step_index, bool displaced) { run_bands(bands_, t, step_index, displaced); }
    // naive patch parallelism (step_naive, runtime.cpp:398-452): validates the step's patch
    // geometry, returns the patch program (stream ordered after the previous naive step)
    std::vector<std::unique_ptr<Program>>& naive_begin(int step_index);
    // every patch: crop nx_ -> forward -> scatter into neps_ (full NCHW, fp32) on progs[0]
    void run_naive_patches(std::vector<std::unique_ptr<Program>>& progs, int t, int step_index);
    void sample_naive(const float* x_T, const int* ts, int n, const std::vector<double>& abar_of,
                      float* x0, float* traj);
    const DeviceWeights* weights_for(int dev);
    void load_x(const float* x_host_nchw);                    // x -> every band's stem input
    void store_eps(float* eps_host_nchw);                     // band eps -> host NCHW
    void check_flags(const char* who);
    void count_macs(int step_index, bool naive);
    void begin_profile();
    void end_profile();

    const Model& m_;
    std::vector<float> cond_;
    RunnerOptions o_;
    int h_, w_, n_dev_;
    std::vector<PatchSpec> specs_;
    std::vector<std::unique_ptr<DeviceWeights>> weights_;   // one per CUDA device used
    std::vector<std::unique_ptr<Program>> bands_;            // local bands
    std::vector<std::unique_ptr<Program>> naive_rows_, naive_cols_;   // one patch program each
    float* nx_ = nullptr;       // naive: full NCHW x_t (fp32, device o_.device)
    float* neps_ = nullptr;     // naive: full NCHW eps
    cudaEvent_t nev_ = nullptr; // naive: end of the previous naive step's work
    std::unique_ptr<Transport> transport_;
    std::vector<int> posted_;      // per layer: last step whose gather exchange was posted
    std::vector<uint64_t> stress_state_;   // --stress-sched: per band splitmix64 state
    std::unique_ptr<Runner> cfg_;          // classifier-free guidance: the unconditional pass
    uint64_t cfg_graph_macs_ = 0;
    std::vector<cudaEvent_t> cfg_ev_;      // per band: [2d] uncond eps ready, [2d+1] x_t refreshed
    void cfg_combine();                    // eps of every band <- the guided eps
    void cfg_refresh_stem();               // the unconditional pass's stem input <- x_t
    std::unique_ptr<PairLink> pair_;       // CFG batch split: eps swap with the partner rank
    void pair_combine();                   // own eps <- guided eps from own + partner's band
    void end_epoch();                      // transports' per-call flag reset (epoch_end)
    void stress_jitter(Program& b, int band);
    std::vector<int> gn_posted_;   // per layer: last step whose GN stats were posted
    uint64_t total_macs_ = 0;
    // RawTrace mirror (record_trace): per device events + the reference's cache-step state
    std::vector<std::vector<TraceEvent>> trace_;
    std::vector<std::vector<int>> tr_act_step_, tr_gn_step_;
    void record_trace(int s, int kind);   // kind: 0 reference, 1 sync, 2 displaced, 3 naive
    // the two exchange batches of a displaced step (layers of the first / second half)
    std::vector<std::vector<XItem>> xbatch_;
    void plan_exchanges();
    std::vector<std::vector<uint64_t>> step_device_macs_;
    CommVolumes volumes_;
    ProfileTotals prof_;
    long launches_ = 0;
    double last_device_ms_ = 0;
    // CUDA graph of the whole denoising loop (sample()), keyed by plan and mode
    bool graphs_enabled_ = true;
    cudaGraphExec_t graph_exec_ = nullptr;
    std::vector<double> graph_key_;
    std::vector<cudaEvent_t> graph_events_;
    uint64_t graph_macs_ = 0;
    std::vector<std::vector<uint64_t>> graph_step_macs_;
    CommVolumes graph_vol_;
    long graph_launches_ = 0;
    // host staging (pinned)
    float* h_x_ = nullptr;      // full NCHW image
    float* h_eps_ = nullptr;    // full NCHW image
    int* h_flags_ = nullptr;
};

}  // namespace pp
