// Host-side model description: the reference's layer graph and weight pool.
//
// Mirrors ModelConfig / LayerDescriptor / build_model (proj/include/patchsim/model.hpp,
// proj/src/model.cpp:39-218) and its seeded splitmix64 weight init, so a model built
// here is bit-identical to the reference's (checked in tests/test_model_host.py).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pp {

enum class Kind : int {
    Conv = 0,
    GroupNorm,
    SiLU,
    DownConv,
    Upsample,
    SelfAttn,
    CrossAttn,
    Linear,
    AddSkip,
    AddTimeEmb,
};
const char* kind_name(Kind k);

struct ModelConfig {
    int in_channels = 4;
    int base_channels = 16;
    int levels = 3;
    int groups = 4;
    int cond_dim = 8;
    int attn_at_level = -1;
    // Deeper graphs (beyond the reference API; the defaults build the
    // reference graph exactly): res_blocks residual blocks per level on both paths, attention
    // at the levels of the attn_levels bit mask (0: attn_level() only), attn_depth attention
    // blocks after every residual block there, and attn_up: also on the up path.
    int res_blocks = 1;
    int attn_levels = 0;
    int attn_depth = 1;
    int attn_up = 0;
    int attn_level() const { return attn_at_level < 0 ? levels - 1 : attn_at_level; }
    bool has_attn(int lv) const {
        return attn_levels ? ((attn_levels >> lv) & 1) != 0 : lv == attn_level();
    }
    int depth_divisor() const { return 1 << (levels - 1); }
    void validate() const;  // throws std::invalid_argument (model.cpp:25-33)
};

struct Layer {
    int id = -1;
    Kind kind{};
    int in_ch = 0, out_ch = 0;
    int kernel = 0, stride = 1, pad = 0;
    int groups = 0;
    float eps = 1e-5f;
    int cond_dim = 0;
    int skip_source = -1;
    int scale_in = 1, scale_out = 1;
    int weight = -1, bias = -1, weight2 = -1, bias2 = -1;
    bool needs_gather() const {
        return kind == Kind::Conv || kind == Kind::DownConv || kind == Kind::SelfAttn;
    }
};

struct WeightTensor {
    int n = 0, c = 0, h = 0, w = 0;
    std::vector<float> data;
    size_t size() const { return data.size(); }
};

struct Model {
    ModelConfig cfg;
    uint64_t seed = 0;
    std::vector<Layer> layers;
    std::vector<WeightTensor> weights;
    int time_dim() const { return 2 * cfg.base_channels; }
};

// Graph only (weights zero); build_model = graph + seeded init.
Model build_graph(const ModelConfig& cfg);
Model build_model(const ModelConfig& cfg, uint64_t seed);

// ---- host RNG (proj/include/patchsim/rng.hpp) ----------------------------------------
struct SplitMix64 {
    uint64_t state = 0;
    explicit SplitMix64(uint64_t s = 0) : state(s) {}
    uint64_t next() {
        state += 0x9E3779B97F4A7C15ULL;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double unit() { return double(next() >> 11) * 0x1.0p-53; }
};
uint64_t substream_seed(uint64_t seed, uint64_t a, uint64_t b = 0);
// Box-Muller standard normals (tensor.cpp:374-394): cos first, sin as the spare.
std::vector<float> gaussian(uint64_t seed, size_t count);

// ---- region logic (proj/src/runtime.cpp:46-83) -----------------------------------------
struct Region {
    int row_start = 0, row_end = 0, full_h = 0, full_w = 0;
    int rows() const { return row_end - row_start; }
    void validate(const std::string& who) const;
};
std::vector<Region> partition_rows(int h, int n_devices, int full_w);
struct PatchSpec {
    Region input;
    std::vector<Region> layer_in, layer_out;
};
PatchSpec derive_patch_spec(const Model& m, const Region& input);

uint64_t macs_of_layer(const Layer& d, const Region& r);    // costmodel.cpp:33-62
uint64_t model_total_macs(const Model& m, int h, int w);     // costmodel.cpp:64-71

std::vector<float> timestep_embedding(int t, int dim);      // model.cpp:220-231

// Rank-ordered all-gather result [N][C][rows][W] (each band NCHW) -> full NCHW image
// (C, N*rows, W); the assembly run_workers does when stitching eps (runtime.cpp:368-377).
void assemble_bands(const float* gathered, int n_bands, int C, int rows, int W, float* out);

// ---- sampler schedule (proj/src/sampler.cpp:17-44) ---------------------------------------
std::vector<double> make_schedule(int total, double beta_start, double beta_end);
std::vector<int> make_plan(int total, int num_steps);

}  // namespace pp
