// One row band compiled for one CUDA device (internal to the runtime).
//
// Buffers (all NHWC, element type bf16 or fp32, channels padded to a 128-byte
// multiple `ld`):
//   act[l]       output of layer l: [rows+2][W][ld]; row 0 / row rows+1 are the halo
//                rows a following conv reads (zero at the image border);
//   stem         the band of the latent x_t, same padded layout (input of layer 0);
//   eps          fp32 [rows][W][C] output of the head conv (the band of eps);
//   x_state      fp32 [rows][W][C] band of the sampler state x_t.
// Exchange buffers (parity double-buffered, index = step % 2), per gather / GN layer:
//   send_rows    [2][W][ld]  own first / last row (halo source)
//   halo_recv    [2][W][ld]  row above (from band-1) / row below (from band+1)
//   kv           [H_l*W][ld] full map for self-attention (own rows + gathered rows)
//   stats        [N][G][2]   every band's local (mean, mean_sq), fp64
#pragma once
#include "runtime.hpp"

#include <array>
#include <functional>
#include <vector>

namespace pp {

struct LayerWeights {
    void* w = nullptr;       // conv: [n_pad][9][cin_ld]; linear: [n_pad][cin_ld] (T)
    int n_pad = 0;
    float* bias = nullptr;   // [n_pad] fp32
    float* gamma = nullptr;  // [ld] fp32 (GroupNorm)
    float* beta = nullptr;
    float* temb_w = nullptr;  // AddTimeEmb: [C][time_dim] fp32 (reference layout)
    float* temb_b = nullptr;
    float* cross_v = nullptr; // CrossAttn: projected value vector [ld] fp32 (one token)
    // CrossAttn over T > 1 condition tokens (beyond the reference API): the projected keys and
    // values in the element type, [T][ld] each (K: the S GEMM's B; V: the PV GEMM's B, read
    // MN-major), and V^T [ld][T_pad] for the TF32 PV GEMM
    void* cross_k_tok = nullptr;
    void* cross_v_tok = nullptr;
    void* cross_vt_tok = nullptr;
    int tokens = 1, tokens_pad = 0;
    // stem conv with in_ch <= 4 as one-K-block GEMM: [n_pad][kStemK] (tap-major, 4 channels)
    void* w_stem = nullptr;
};

struct DeviceWeights {
    int dev = 0;
    Elem e = Elem::BF16;
    std::vector<LayerWeights> L;
    std::vector<void*> allocs;
    // cond = tokens x cond_dim floats (tokens > 1: multi-token cross-attention)
    DeviceWeights(const Model& m, const std::vector<float>& cond, int dev, Elem e, int tokens = 1);
    ~DeviceWeights();
    void* alloc(size_t bytes);
};

// A fused launch group: layers [first, last] executed as one op.
struct Group {
    Kind kind{};
    int first = 0, last = 0;
    bool silu = false;   // GroupNorm + SiLU
    int temb = -1;       // + AddTimeEmb (layer id)
    int skip = -1;       // + AddSkip (skip source layer id)
};
std::vector<Group> fuse_layers(const Model& m);

struct Program {
    Runner* r = nullptr;
    const Model* m = nullptr;
    const DeviceWeights* wts = nullptr;
    int dev = 0;
    int band = 0, nb = 1;    // band index / number of bands in the exchange
    int H = 0, W = 0;        // latent size of the image this program covers
    Elem e = Elem::BF16;
    size_t eb = 2;
    int kel = 64;            // elements per 128-byte block
    bool rnd = false;        // fp32 mode: round stored activations to tf32
    PatchSpec spec;
    cudaStream_t cs = nullptr, xs = nullptr;

    struct Act {
        void* base = nullptr;   // padded buffer
        int rows = 0, w = 0, ld = 0, C = 0;
        void* interior(size_t eb) const {
            return static_cast<char*>(base) + size_t(w) * ld * eb;
        }
        long long pix() const { return (long long)rows * w; }
    };
    std::vector<Act> act;   // [L] (base == nullptr when fused away; last layer -> eps)
    Act stem;
    float* eps = nullptr;       // fp32 NHWC band
    float* x_state = nullptr;   // fp32 NHWC band (sampler)
    float* x_full = nullptr;    // fp32 NCHW full image (step API upload)
    float* band_nchw = nullptr; // fp32 NCHW band (eps / x download)
    int* flags = nullptr;       // [0] non-finite, [1] negative GN variance

    struct LayerX {
        std::array<void*, 2> send_rows{{nullptr, nullptr}};
        std::array<void*, 2> halo_recv{{nullptr, nullptr}};
        std::array<void*, 2> kv{{nullptr, nullptr}};
        std::array<double*, 2> stats{{nullptr, nullptr}};
        double* weights = nullptr;   // [nb] band pixel counts
        int G = 0;
        size_t row_bytes = 0;        // one halo row
        size_t band_bytes = 0;       // own K/V rows
    };
    std::vector<LayerX> lx;
    std::vector<Group> groups;
    std::vector<std::array<GemmPlan, 2>> plans;    // per group, per step parity: conv / linear;
                                                   // attention PV per K/V parity
    std::vector<std::array<GemmPlan, 2>> s_plans;  // attention S = Q K^T per K/V parity
    std::vector<char> fused_stats;                 // per GN layer: stats come from the conv epilogue
    std::vector<char> merged_into_prev;            // per group: computed by the previous group
    std::vector<char> stem_gemm;                   // per group: stem conv as im2col + GEMM
    void* stem_cols = nullptr;                     // [pix][kStemK] im2col of the stem input
    GemmScratch sc;
    // scratch
    double* gn_partial = nullptr;
    unsigned int* gn_ticket = nullptr;
    // attention scratch per attention group (self-attention, or cross-attention over T > 1
    // tokens): P = softmax numerators [m][s_pad] (padding columns stay zero), per key tile row
    // maxima [n_tiles][m], 1 / row sums [m]; V^T [C][s_pad] when the PV GEMM cannot read V
    // MN-major (TF32, or channels not filling 128-byte chunks)
    struct AttnScratch {
        void* P = nullptr;
        int s_pad = 0;
        float* rowmax = nullptr;
        float* rscale = nullptr;
        void* Vt = nullptr;
        bool v_mn = false;
    };
    std::vector<AttnScratch> attn_sc;   // per group
    // time embedding
    std::vector<float*> temb_out;   // per layer (nullptr unless AddTimeEmb)
    TembLayer* temb_dev = nullptr;
    int n_temb = 0, temb_max_c = 0;
    // per-plan table of every step's projections (sample()): [step][slot][temb_ldt]
    std::vector<int> temb_slot;     // layer -> slot among the AddTimeEmb layers
    int temb_ldt = 0;
    float* temb_plan = nullptr;
    size_t temb_plan_cap = 0;
    float* temb_embs = nullptr;
    size_t temb_embs_cap = 0;
    const float* temb_step_base = nullptr;   // non-null: this step reads the plan table
    const float* temb_ptr(int l) const {
        return temb_step_base ? temb_step_base + size_t(temb_slot[l]) * temb_ldt : temb_out[l];
    }
    std::vector<int> temb_plan_key;   // timesteps the table holds
    void prepare_temb_plan(const int* ts, int n);
    void use_temb_step(int i) {
        temb_step_base = i < 0 ? nullptr : temb_plan + size_t(i) * n_temb * temb_ldt;
    }
    // events
    std::vector<cudaEvent_t> ready;               // per layer
    std::vector<std::array<cudaEvent_t, 2>> sent; // per layer, per parity
    cudaEvent_t gather_ev = nullptr;              // compute <-> comm stream join (gathers)
    std::vector<void*> allocs;
    // profiling
    struct Timed {
        int cat;
        cudaEvent_t a, b;
        double flops;
    };
    std::vector<Timed> timed;
    std::vector<cudaEvent_t> event_pool;
    size_t event_next = 0;
    bool profile = false;

    Program(Runner* r, const Model& m, const DeviceWeights* w, int dev, int band, int nb, int H,
            int W, const PatchSpec& spec, Elem e, bool profile);
    ~Program();
    Program(const Program&) = delete;
    Program& operator=(const Program&) = delete;

    void* alloc(size_t bytes);
    void set_profile(bool on);
    const Act& input_of(int l) const { return l == 0 ? stem : act[l - 1]; }
    void count(long n);
    void run_timed(int cat, double flops, const std::function<void()>& fn);

    // per-step pieces (issued by Runner in layer order)
    void time_projection(int t);
    void halo_rows(const Group& g, int par_pack, int par_unpack);
    void conv(const Group& g, int par);
    void own_kv(const Group& g, int par_post, int par_use);
    void attention(const Group& g, int par, int par_out);
    // CrossAttn over T > 1 condition tokens: S GEMM (softmax epilogue) -> rescale -> PV GEMM
    void cross_attention(const Group& g);
    void gn_stats(const Group& g, int par);
    void gn_apply(const Group& g, int combine_mode, int par_cur, int par_prev);
    void simple(const Group& g, int par);
    void record_ready(int l);
};

// One exchange of a batch: layer and what moves (halo rows, K/V band, GroupNorm statistics).
struct XItem {
    enum Kind { HALO = 0, KV = 1, STATS = 2 };
    int layer = 0;
    int kind = HALO;
    bool top_only = false;   // halo of a stride-2 DownConv: only the row above is needed
};

class Transport {
public:
    virtual ~Transport() = default;
    // Exchange the layer-l context of the current step into parity `par` buffers.
    // Precondition: every local band recorded ready[l] after packing.
    virtual void halo(int l, int par, bool top_only) = 0;
    virtual void kv(int l, int par) = 0;
    virtual void stats(int l, int par) = 0;
    // Displaced steps: the layers' posts of one step, exchanged together into parity `par`
    // (their consumers read them one step later).  Precondition: every local band recorded
    // ready[l] for every listed layer; afterwards sent[l][par] of every listed layer marks the
    // exchange, so wait() is unchanged.  Default: one exchange per item.
    // Every exchange this runner will issue (the displaced batches and the single-layer
    // exchanges of synchronous steps), announced once before any capture: a transport may
    // build its device-side tables here (no allocation or synchronous copy during a capture).
    virtual void prepare(const std::vector<std::vector<XItem>>& exchanges) { (void)exchanges; }
    virtual void batch(const std::vector<XItem>& items, int par) {
        for (const XItem& it : items) {
            if (it.kind == XItem::HALO) halo(it.layer, par, it.top_only);
            else if (it.kind == XItem::KV) kv(it.layer, par);
            else stats(it.layer, par);
        }
    }
    // Make band b's compute stream wait until the (l, par) exchange has landed.
    virtual void wait(Program& b, int l, int par) = 0;
    // All-gather equal float chunks (rank order) on band b's compute stream (NCCL only).
    virtual void gather_floats(Program& b, const float* send, float* recv, size_t count) = 0;
    // End of a runner call (sample / step), eager, on band b's compute stream: a transport
    // whose flags carry per-call sequence numbers returns them to zero here, so every call --
    // and every replay of a graph captured in one -- starts from the same flag state.
    virtual void epoch_end(Program& b) { (void)b; }
};

std::unique_ptr<Transport> make_inproc_transport(std::vector<Program*> bands);
std::unique_ptr<Transport> make_nccl_transport(Program* band, int world, int rank,
                                               const std::vector<uint8_t>& id);
// Copy-engine transport over CUDA IPC peer mappings (world > 1, no NCCL on the data path):
// export this rank's handle blob, then connect with every rank's blob (rank order).
std::unique_ptr<Transport> make_ipc_transport(Program* band, int world, int rank);
std::vector<uint8_t> ipc_export(Transport& t);
void ipc_connect(Transport& t, const uint8_t* blobs, size_t per_rank);

// Classifier-free guidance batch split (beyond the reference API): the conditional and the
// unconditional pass of one band run on two ranks (two GPU groups); after every U-Net pass
// the pair swaps its eps bands.  role 0 = conditional rank, 1 = unconditional rank.
class PairLink {
public:
    virtual ~PairLink() = default;
    // Enqueue on s: send `mine` (the n floats of this rank's eps band) to the partner and
    // receive the partner's.  Returns the device buffer that holds the partner's eps in stream
    // order on s, valid until the next exchange call.
    virtual const float* exchange(cudaStream_t s, const float* mine) = 0;
    virtual bool capturable() const = 0;
    virtual void epoch_end(cudaStream_t s) { (void)s; }   // as Transport::epoch_end
    virtual std::vector<uint8_t> export_blob() const;
    virtual void connect(const uint8_t* blob, size_t size);
};
// two-rank NCCL communicator (rank = role): ncclSend / ncclRecv on the stream, graph-capturable
std::unique_ptr<PairLink> make_nccl_pair(int dev, int role, const std::vector<uint8_t>& id, size_t n);
// CUDA IPC: the partner pushes into one of two parity receive buffers with the copy engine and
// bumps a flag with a stream memory operation (per-call sequence numbers, reset by epoch_end)
std::unique_ptr<PairLink> make_ipc_pair(int dev, int role, size_t n);

}  // namespace pp
