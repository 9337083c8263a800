// Host-side model graph, seeded weight init and band/region logic (see model.hpp).
#include "model.hpp"

#include <cmath>
#include <cstring>
#include <stdexcept>

namespace pp {

const char* kind_name(Kind k) {
    switch (k) {
        case Kind::Conv: return "Conv";
        case Kind::GroupNorm: return "GroupNorm";
        case Kind::SiLU: return "SiLU";
        case Kind::DownConv: return "DownConv";
        case Kind::Upsample: return "Upsample";
        case Kind::SelfAttn: return "SelfAttn";
        case Kind::CrossAttn: return "CrossAttn";
        case Kind::Linear: return "Linear";
        case Kind::AddSkip: return "AddSkip";
        case Kind::AddTimeEmb: return "AddTimeEmb";
    }
    return "?";
}

void ModelConfig::validate() const {
    if (in_channels <= 0 || base_channels <= 0 || cond_dim <= 0)
        throw std::invalid_argument("ModelConfig: channel/cond counts must be positive");
    if (levels < 1) throw std::invalid_argument("ModelConfig: levels must be >= 1");
    if (groups <= 0 || base_channels % groups != 0)
        throw std::invalid_argument("ModelConfig: base_channels must be divisible by groups");
    if (attn_level() < 0 || attn_level() >= levels)
        throw std::invalid_argument("ModelConfig: attn_at_level out of range");
    if (res_blocks < 1 || attn_depth < 1)
        throw std::invalid_argument("ModelConfig: res_blocks and attn_depth must be >= 1");
    if (attn_levels < 0 || attn_levels >= (1 << levels))
        throw std::invalid_argument("ModelConfig: attn_levels names a level that does not exist");
}

uint64_t substream_seed(uint64_t seed, uint64_t a, uint64_t b) {
    SplitMix64 m(seed);
    uint64_t s = m.next();
    m.state = s ^ (a * 0x9E3779B97F4A7C15ULL);
    s = m.next();
    m.state = s ^ (b * 0xD1B54A32D192ED03ULL);
    return m.next();
}

std::vector<float> gaussian(uint64_t seed, size_t count) {
    std::vector<float> out(count);
    SplitMix64 rng(seed);
    for (size_t i = 0; i < count; i += 2) {
        const double u1 = (double(rng.next() >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = rng.unit();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * 3.14159265358979323846 * u2;
        out[i] = float(r * std::cos(th));
        if (i + 1 < count) out[i + 1] = float(r * std::sin(th));
    }
    return out;
}

namespace {

struct GraphBuilder {
    Model m;
    int level_ch(int lv) const { return m.cfg.base_channels << lv; }
    Layer& push(Kind k, int scale) {
        Layer d;
        d.id = int(m.layers.size());
        d.kind = k;
        d.scale_in = d.scale_out = scale;
        m.layers.push_back(d);
        return m.layers.back();
    }
    int alloc(int n, int c, int h, int w) {
        WeightTensor t;
        t.n = n; t.c = c; t.h = h; t.w = w;
        t.data.assign(size_t(n) * c * h * w, 0.0f);
        m.weights.push_back(std::move(t));
        return int(m.weights.size()) - 1;
    }
    void conv(Kind k, int cin, int cout, int scale) {
        Layer& d = push(k, scale);
        d.in_ch = cin;
        d.out_ch = cout;
        d.kernel = 3;
        d.pad = 1;
        d.stride = k == Kind::DownConv ? 2 : 1;
        if (k == Kind::DownConv) d.scale_out = scale * 2;
        d.weight = alloc(cout, cin, 3, 3);
        d.bias = alloc(cout, 1, 1, 1);
    }
    void gn(int ch, int scale) {
        Layer& d = push(Kind::GroupNorm, scale);
        d.in_ch = d.out_ch = ch;
        d.groups = m.cfg.groups;
        d.weight = alloc(ch, 1, 1, 1);
        d.bias = alloc(ch, 1, 1, 1);
    }
    void silu(int ch, int scale) {
        Layer& d = push(Kind::SiLU, scale);
        d.in_ch = d.out_ch = ch;
    }
    void temb(int ch, int scale) {
        Layer& d = push(Kind::AddTimeEmb, scale);
        d.in_ch = d.out_ch = ch;
        d.weight = alloc(ch, m.time_dim(), 1, 1);
        d.bias = alloc(ch, 1, 1, 1);
    }
    void add_skip(int src, int ch, int scale) {
        Layer& d = push(Kind::AddSkip, scale);
        d.in_ch = d.out_ch = ch;
        d.skip_source = src;
    }
    int res_block(int ch, int scale, int entry) {
        for (int r = 0; r < 2; ++r) {
            conv(Kind::Conv, ch, ch, scale);
            gn(ch, scale);
            silu(ch, scale);
            temb(ch, scale);
        }
        add_skip(entry, ch, scale);
        return int(m.layers.size()) - 1;
    }
    void attn_block(int ch, int scale) {
        int pre = int(m.layers.size()) - 1;
        Layer& sa = push(Kind::SelfAttn, scale);
        sa.in_ch = sa.out_ch = ch;
        add_skip(pre, ch, scale);
        pre = int(m.layers.size()) - 1;
        Layer& ca = push(Kind::CrossAttn, scale);  // alloc() never touches m.layers
        ca.in_ch = ca.out_ch = ch;
        ca.cond_dim = m.cfg.cond_dim;
        ca.weight = alloc(ch, m.cfg.cond_dim, 1, 1);   // key projection
        ca.bias = alloc(ch, 1, 1, 1);
        ca.weight2 = alloc(ch, m.cfg.cond_dim, 1, 1);  // value projection
        ca.bias2 = alloc(ch, 1, 1, 1);
        add_skip(pre, ch, scale);
        pre = int(m.layers.size()) - 1;
        Layer& ff = push(Kind::Linear, scale);
        ff.in_ch = ff.out_ch = ch;
        ff.weight = alloc(ch, ch, 1, 1);
        ff.bias = alloc(ch, 1, 1, 1);
        add_skip(pre, ch, scale);
    }
    void upsample(int ch, int scale) {
        Layer& d = push(Kind::Upsample, scale);
        d.in_ch = d.out_ch = ch;
        d.scale_out = scale / 2;
    }
};

double fan_in(const Layer& d, int time_dim) {
    switch (d.kind) {
        case Kind::Conv:
        case Kind::DownConv: return double(d.in_ch) * d.kernel * d.kernel;
        case Kind::GroupNorm:
        case Kind::Linear: return double(d.in_ch);
        case Kind::AddTimeEmb: return double(time_dim);
        case Kind::CrossAttn: return double(d.cond_dim);
        default: return 1.0;
    }
}

}  // namespace

Model build_graph(const ModelConfig& cfg) {
    cfg.validate();
    GraphBuilder b;
    b.m.cfg = cfg;
    b.conv(Kind::Conv, cfg.in_channels, b.level_ch(0), 1);
    std::vector<int> exits(cfg.levels, -1);
    for (int lv = 0; lv < cfg.levels; ++lv) {
        const int scale = 1 << lv;
        for (int rb = 0; rb < cfg.res_blocks; ++rb) {
            const int entry = int(b.m.layers.size()) - 1;
            exits[lv] = b.res_block(b.level_ch(lv), scale, entry);
            if (cfg.has_attn(lv)) {
                for (int k = 0; k < cfg.attn_depth; ++k) b.attn_block(b.level_ch(lv), scale);
                exits[lv] = int(b.m.layers.size()) - 1;
            }
        }
        if (lv + 1 < cfg.levels) b.conv(Kind::DownConv, b.level_ch(lv), b.level_ch(lv + 1), scale);
    }
    for (int lv = cfg.levels - 2; lv >= 0; --lv) {
        const int scale = 1 << lv;
        b.upsample(b.level_ch(lv + 1), scale * 2);
        b.conv(Kind::Conv, b.level_ch(lv + 1), b.level_ch(lv), scale);
        b.add_skip(exits[lv], b.level_ch(lv), scale);
        for (int rb = 0; rb < cfg.res_blocks; ++rb) {
            const int entry = int(b.m.layers.size()) - 1;
            b.res_block(b.level_ch(lv), scale, entry);
            if (cfg.attn_up && cfg.has_attn(lv))
                for (int k = 0; k < cfg.attn_depth; ++k) b.attn_block(b.level_ch(lv), scale);
        }
    }
    b.gn(b.level_ch(0), 1);
    b.silu(b.level_ch(0), 1);
    b.conv(Kind::Conv, b.level_ch(0), cfg.in_channels, 1);
    return std::move(b.m);
}

Model build_model(const ModelConfig& cfg, uint64_t seed) {
    Model m = build_graph(cfg);
    m.seed = seed;
    for (const Layer& d : m.layers) {
        const int handles[4] = {d.weight, d.bias, d.weight2, d.bias2};
        for (int slot = 0; slot < 4; ++slot) {
            if (handles[slot] < 0) continue;
            const double s = 1.0 / std::sqrt(fan_in(d, m.time_dim()));
            SplitMix64 rng(substream_seed(seed, uint64_t(d.id), uint64_t(slot)));
            const bool gamma = d.kind == Kind::GroupNorm && slot == 0;
            for (float& v : m.weights[handles[slot]].data) {
                const double u = -s + (s - -s) * rng.unit();
                v = float(gamma ? 1.0 + u : u);
            }
        }
    }
    return m;
}

void Region::validate(const std::string& who) const {
    if (!(0 <= row_start && row_start < row_end && row_end <= full_h) || full_w <= 0)
        throw std::invalid_argument(who + ": invalid region [" + std::to_string(row_start) + "," +
                                    std::to_string(row_end) + ") of " + std::to_string(full_h) +
                                    "x" + std::to_string(full_w));
}

std::vector<Region> partition_rows(int h, int n, int w) {
    if (n < 1) throw std::invalid_argument("partition_rows: need at least one device");
    if (h <= 0 || h % n != 0)
        throw std::invalid_argument("partition_rows: " + std::to_string(h) +
                                    " rows not divisible by " + std::to_string(n) + " devices");
    std::vector<Region> out;
    const int band = h / n;
    for (int d = 0; d < n; ++d) out.push_back(Region{d * band, (d + 1) * band, h, w});
    return out;
}

PatchSpec derive_patch_spec(const Model& m, const Region& input) {
    input.validate("derive_patch_spec");
    PatchSpec s;
    s.input = input;
    Region cur = input;
    for (const Layer& d : m.layers) {
        s.layer_in.push_back(cur);
        Region out = cur;
        if (d.kind == Kind::DownConv) {
            if (cur.row_start % 2 || cur.row_end % 2 || cur.full_h % 2 || cur.full_w % 2)
                throw std::invalid_argument(
                    "patch rows [" + std::to_string(cur.row_start) + "," +
                    std::to_string(cur.row_end) + ") of " + std::to_string(cur.full_h) +
                    " are not divisible at layer " + std::to_string(d.id) +
                    " (DownConv); choose h divisible by devices*2^(levels-1)");
            out = Region{cur.row_start / 2, cur.row_end / 2, cur.full_h / 2, cur.full_w / 2};
        } else if (d.kind == Kind::Upsample) {
            out = Region{cur.row_start * 2, cur.row_end * 2, cur.full_h * 2, cur.full_w * 2};
        }
        s.layer_out.push_back(out);
        cur = out;
    }
    return s;
}

uint64_t macs_of_layer(const Layer& d, const Region& r) {
    if (r.rows() == 0) return 0;
    r.validate("macs_of_layer");
    const uint64_t rows = uint64_t(r.rows()), w = uint64_t(r.full_w);
    switch (d.kind) {
        case Kind::Conv:
        case Kind::DownConv:
            return (rows / d.stride) * (w / d.stride) * uint64_t(d.out_ch) * uint64_t(d.in_ch) *
                   uint64_t(d.kernel) * uint64_t(d.kernel);
        case Kind::Linear: return rows * w * uint64_t(d.in_ch) * uint64_t(d.out_ch);
        case Kind::SelfAttn: return 2 * rows * w * uint64_t(r.full_h) * w * uint64_t(d.in_ch);
        case Kind::CrossAttn: return 2 * rows * w * uint64_t(d.in_ch);
        default: return 0;
    }
}

uint64_t model_total_macs(const Model& m, int h, int w) {
    uint64_t t = 0;
    for (const Layer& d : m.layers) {
        const int lh = h / d.scale_in, lw = w / d.scale_in;
        t += macs_of_layer(d, Region{0, lh, lh, lw});
    }
    return t;
}

std::vector<float> timestep_embedding(int t, int dim) {
    if (dim < 2 || dim % 2) throw std::invalid_argument("timestep_embedding: dim must be even and >= 2");
    std::vector<float> e(dim);
    const int half = dim / 2;
    for (int i = 0; i < half; ++i) {
        const double f = std::pow(10000.0, -2.0 * i / double(dim));
        e[i] = float(std::sin(t * f));
        e[half + i] = float(std::cos(t * f));
    }
    return e;
}

void assemble_bands(const float* g, int n, int C, int rows, int W, float* out) {
    const size_t band = size_t(C) * rows * W;
    const size_t H = size_t(n) * rows;
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < C; ++c)
            std::memcpy(out + (size_t(c) * H + size_t(r) * rows) * W, g + r * band + size_t(c) * rows * W,
                        size_t(rows) * W * sizeof(float));
}

std::vector<double> make_schedule(int total, double b0, double b1) {
    if (total < 1) throw std::invalid_argument("make_schedule: total_steps must be >= 1");
    if (b0 < 0.0 || b1 < 0.0 || b0 >= 1.0 || b1 >= 1.0)
        throw std::invalid_argument("make_schedule: betas must lie in [0, 1)");
    std::vector<double> a(total);
    double prod = 1.0;
    for (int t = 0; t < total; ++t) {
        const double frac = total == 1 ? 0.0 : double(t) / double(total - 1);
        prod *= 1.0 - (b0 + (b1 - b0) * frac);
        a[t] = prod;
    }
    return a;
}

std::vector<int> make_plan(int total, int num_steps) {
    if (num_steps < 1 || num_steps > total)
        throw std::invalid_argument("make_plan: num_steps out of range");
    std::vector<int> ts;
    const int stride = total / num_steps;
    for (int i = num_steps - 1; i >= 0; --i) ts.push_back(i * stride);
    return ts;
}

}  // namespace pp
