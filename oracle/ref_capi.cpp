// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A C shim over the UNMODIFIED reference sources (compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests and bench.py's cpu_baseline / --impl reference leg call the
// reference's own fp32/fp64 CPU path through ctypes:
//   * model build / weight pool      proj/src/model.cpp:158-218
//   * forward_collect                 proj/src/model.cpp:302-361
//   * PatchRunner step entries        proj/src/runtime.cpp:382-476
//   * run_sampling                    proj/src/runtime.cpp:494-526
//   * per-kernel operators            proj/src/tensor.cpp:79-394
// Exceptions are mapped to status codes: 1 = std::invalid_argument,
// 2 = std::runtime_error (proj/src/cli.cpp:145-154 maps them to exit 2 / 1).
#include "patchsim/costmodel.hpp"
#include "patchsim/model.hpp"
#include "patchsim/io.hpp"
#include "patchsim/runtime.hpp"
#include "patchsim/sampler.hpp"
#include "patchsim/tensor.hpp"

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

using namespace patchsim;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Tensor make(int n, int c, int h, int w, const float* src) {
    Tensor t(n, c, h, w);
    if (src) std::memcpy(t.data.data(), src, t.size() * sizeof(float));
    return t;
}
void put(const Tensor& t, float* dst) { std::memcpy(dst, t.data.data(), t.size() * sizeof(float)); }

ModelConfig cfg_of(const int* c) {
    ModelConfig m;
    m.in_channels = c[0];
    m.base_channels = c[1];
    m.levels = c[2];
    m.groups = c[3];
    m.cond_dim = c[4];
    m.attn_at_level = c[5];
    return m;
}

struct RunnerBox {
    std::unique_ptr<Model> model;
    std::unique_ptr<PatchRunner> runner;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// cfg6 = {in_channels, base_channels, levels, groups, cond_dim, attn_at_level}
void* ref_model_build(const int* cfg6, uint64_t seed) {
    Model* m = nullptr;
    if (guard([&] { m = new Model(build_model(cfg_of(cfg6), seed)); })) return nullptr;
    return m;
}
void ref_model_free(void* m) { delete static_cast<Model*>(m); }
int ref_model_num_layers(void* m) { return int(static_cast<Model*>(m)->layers.size()); }
// out15 = kind,in,out,kernel,stride,pad,groups,cond_dim,skip,scale_in,scale_out,w,b,w2,b2
void ref_model_layer(void* mp, int id, int* o, float* eps) {
    const LayerDescriptor& d = static_cast<Model*>(mp)->layers.at(id);
    const int v[15] = {int(d.kind), d.in_ch,   d.out_ch,   d.kernel,   d.stride,
                       d.pad,       d.groups,  d.cond_dim, d.skip_source, d.scale_in,
                       d.scale_out, d.weight,  d.bias,     d.weight2,  d.bias2};
    std::memcpy(o, v, sizeof(v));
    *eps = d.eps;
}
int ref_model_num_weights(void* m) { return int(static_cast<Model*>(m)->weights.size()); }
void ref_model_weight_shape(void* m, int h, int* nchw) {
    const Tensor& t = static_cast<Model*>(m)->weights.at(h);
    nchw[0] = t.n; nchw[1] = t.c; nchw[2] = t.h; nchw[3] = t.w;
}
void ref_model_weight_get(void* m, int h, float* dst) { put(static_cast<Model*>(m)->weights.at(h), dst); }
void ref_model_weight_set(void* m, int h, const float* src) {
    Tensor& t = static_cast<Model*>(m)->weights.at(h);
    std::memcpy(t.data.data(), src, t.size() * sizeof(float));
}
void ref_model_zero_weights(void* m, int keep_biases) { zero_weights(*static_cast<Model*>(m), keep_biases != 0); }
uint64_t ref_model_total_macs(void* m, int h, int w) { return model_total_macs(*static_cast<Model*>(m), h, w); }

// forward_collect: writes every layer output back to back (layer l output is
// (1, out_ch, H/scale_out, W/scale_out)).
int ref_forward_collect(void* mp, const float* x, int c, int h, int w, int t, const float* cond,
                        int cond_n, float* outs) {
    return guard([&] {
        Condition cd;
        cd.values.assign(cond, cond + cond_n);
        auto all = forward_collect(*static_cast<Model*>(mp), make(1, c, h, w, x), t, cd);
        std::size_t off = 0;
        for (const Tensor& o : all) {
            put(o, outs + off);
            off += o.size();
        }
    });
}
int ref_forward_full(void* mp, const float* x, int c, int h, int w, int t, const float* cond,
                     int cond_n, float* out) {
    return guard([&] {
        Condition cd;
        cd.values.assign(cond, cond + cond_n);
        put(forward_full(*static_cast<Model*>(mp), make(1, c, h, w, x), t, cd), out);
    });
}

// ---- PatchRunner ---------------------------------------------------------------
void* ref_runner_create(void* mp, const float* cond, int cond_n, int h, int w, int mode,
                        int n_dev, int warmup, int gn_scheme, int stress) {
    RunnerBox* b = new RunnerBox;
    const int rc = guard([&] {
        Condition cd;
        cd.values.assign(cond, cond + cond_n);
        RunnerOptions o;
        o.mode = RunMode(mode);
        o.n_devices = n_dev;
        o.warmup_steps = warmup;
        o.gn_scheme = GnScheme(gn_scheme);
        o.stress = stress != 0;
        b->runner = std::make_unique<PatchRunner>(*static_cast<Model*>(mp), cd, h, w, o);
    });
    if (rc) {
        delete b;
        return nullptr;
    }
    return b;
}
void ref_runner_free(void* r) { delete static_cast<RunnerBox*>(r); }
// which: 0 run_step, 1 step_reference, 2 step_naive, 3 step_sync, 4 step_displaced
int ref_runner_step(void* rp, int which, const float* x, int c, int h, int w, int t, int step,
                    float* eps) {
    PatchRunner& r = *static_cast<RunnerBox*>(rp)->runner;
    return guard([&] {
        const Tensor xt = make(1, c, h, w, x);
        Tensor e;
        switch (which) {
            case 0: e = r.run_step(xt, t, step); break;
            case 1: e = r.step_reference(xt, t, step); break;
            case 2: e = r.step_naive(xt, t, step); break;
            case 3: e = r.step_sync(xt, t, step); break;
            case 4: e = r.step_displaced(xt, t, step); break;
            default: throw std::invalid_argument("bad step entry");
        }
        put(e, eps);
    });
}
// Returns element count (0 if absent); copies when dst != nullptr.
long ref_runner_cached_input(void* rp, int dev, int layer, float* dst, int* nchw) {
    auto p = static_cast<RunnerBox*>(rp)->runner->cached_input(dev, layer);
    if (!p) return 0;
    nchw[0] = p->n; nchw[1] = p->c; nchw[2] = p->h; nchw[3] = p->w;
    if (dst) put(*p, dst);
    return long(p->size());
}
uint64_t ref_runner_total_macs(void* rp) { return static_cast<RunnerBox*>(rp)->runner->total_macs(); }
void ref_runner_volumes(void* rp, uint64_t* v6) {
    const CommVolumes v = static_cast<RunnerBox*>(rp)->runner->volumes();
    v6[0] = v.allgather_recv; v6[1] = v.allgather_sent; v6[2] = v.halo_recv;
    v6[3] = v.halo_sent; v6[4] = v.statreduce_recv; v6[5] = v.statreduce_sent;
}

// trace rows of 9 uint64 {device, step, layer, kind, prim, macs, recv, sent, tag}
long ref_runner_trace(void* rp, int dev, uint64_t* out9, long cap) {
    const RawTrace& t = static_cast<RunnerBox*>(rp)->runner->trace();
    if (dev < 0 || dev >= int(t.per_device.size())) return 0;
    const auto& v = t.per_device[size_t(dev)];
    const long n = long(v.size());
    for (long i = 0; out9 && i < n && i < cap; ++i) {
        const RawEvent& e = v[size_t(i)];
        uint64_t* o = out9 + 9 * i;
        o[0] = uint64_t(e.device); o[1] = uint64_t(e.step); o[2] = uint64_t(int64_t(e.layer));
        o[3] = uint64_t(e.kind); o[4] = uint64_t(e.prim); o[5] = e.macs;
        o[6] = e.bytes_recv; o[7] = e.bytes_sent; o[8] = e.tag;
    }
    return n;
}

// ---- artifacts (proj/src/io.cpp) --------------------------------------------------
int ref_write_tnsr(const float* x, int n, int c, int h, int w, const char* path) {
    return guard([&] { write_tnsr(make(n, c, h, w, x), path); });
}
int ref_read_tnsr_dims(const char* path, int* dims4) {
    return guard([&] {
        const Tensor t = read_tnsr(path);
        dims4[0] = t.n; dims4[1] = t.c; dims4[2] = t.h; dims4[3] = t.w;
    });
}
int ref_read_tnsr(const char* path, float* dst) {
    return guard([&] { put(read_tnsr(path), dst); });
}
int ref_write_pgm(const float* x, int n, int c, int h, int w, double lo, double hi, const char* path) {
    return guard([&] { write_pgm(make(n, c, h, w, x), path, lo, hi); });
}
double ref_psnr(const float* a, const float* b, int n, int c, int h, int w, double peak) {
    double r = 0;
    guard([&] { r = psnr(make(n, c, h, w, a), make(n, c, h, w, b), peak); });
    return r;
}

// ---- run_sampling ----------------------------------------------------------------
// icfg = {mode, n_devices, h, w, num_steps, warmup, gn_scheme, stress, schedule_steps}
// seeds = {model, noise, cond}; traj may be null (num_steps * 4*h*w floats).
int ref_run_sampling(const int* cfg6, const int* icfg, const uint64_t* seeds, double beta_start,
                     double beta_end, float* x0, float* traj, uint64_t* total_macs,
                     uint64_t* vol6) {
    return guard([&] {
        RunConfig rc;
        rc.model = cfg_of(cfg6);
        rc.mode = RunMode(icfg[0]);
        rc.n_devices = icfg[1];
        rc.h = icfg[2];
        rc.w = icfg[3];
        rc.num_steps = icfg[4];
        rc.warmup = icfg[5];
        rc.gn_scheme = GnScheme(icfg[6]);
        rc.stress = icfg[7] != 0;
        rc.schedule_steps = icfg[8];
        rc.model_seed = seeds[0];
        rc.noise_seed = seeds[1];
        rc.cond_seed = seeds[2];
        rc.beta_start = beta_start;
        rc.beta_end = beta_end;
        const RunResult r = run_sampling(rc);
        put(r.x0, x0);
        if (traj)
            for (std::size_t i = 0; i < r.trajectory.size(); ++i)
                put(r.trajectory[i].x, traj + i * r.x0.size());
        if (total_macs) *total_macs = r.total_macs;
        if (vol6) {
            vol6[0] = r.volumes.allgather_recv; vol6[1] = r.volumes.allgather_sent;
            vol6[2] = r.volumes.halo_recv; vol6[3] = r.volumes.halo_sent;
            vol6[4] = r.volumes.statreduce_recv; vol6[5] = r.volumes.statreduce_sent;
        }
    });
}

// ---- partitioning ---------------------------------------------------------------------
int ref_partition_rows(int h, int n, int w, int* out4n) {
    return guard([&] {
        auto rs = partition_rows(h, n, w);
        for (int i = 0; i < n; ++i) {
            out4n[4 * i] = rs[i].row_start; out4n[4 * i + 1] = rs[i].row_end;
            out4n[4 * i + 2] = rs[i].full_h; out4n[4 * i + 3] = rs[i].full_w;
        }
    });
}
// out = layer_in regions then layer_out regions (4 ints each, L layers)
int ref_derive_patch_spec(void* mp, const int* region4, int* out) {
    return guard([&] {
        const Region r{region4[0], region4[1], region4[2], region4[3]};
        const PatchSpec s = derive_patch_spec(*static_cast<Model*>(mp), r);
        const std::size_t L = s.layer_in.size();
        for (std::size_t l = 0; l < L; ++l) {
            const Region& a = s.layer_in[l];
            const Region& b = s.layer_out[l];
            int* p = out + 4 * l;
            p[0] = a.row_start; p[1] = a.row_end; p[2] = a.full_h; p[3] = a.full_w;
            int* q = out + 4 * (L + l);
            q[0] = b.row_start; q[1] = b.row_end; q[2] = b.full_h; q[3] = b.full_w;
        }
    });
}
int ref_run_config_validate(const int* cfg6, const int* icfg) {
    return guard([&] {
        RunConfig rc;
        rc.model = cfg_of(cfg6);
        rc.mode = RunMode(icfg[0]);
        rc.n_devices = icfg[1];
        rc.h = icfg[2];
        rc.w = icfg[3];
        rc.num_steps = icfg[4];
        rc.warmup = icfg[5];
        rc.validate();
    });
}

// ---- kernels ------------------------------------------------------------------------
// x (n,c,h,w), weight (co,c,k,k); region rows [r0,r1). out rows computed by caller.
int ref_conv2d_region(const float* x, int n, int c, int h, int w, int r0, int r1, const float* wt,
                      int co, int k, const float* bias, int stride, int pad, float* out) {
    return guard([&] {
        const Tensor xt = make(n, c, h, w, x), wtt = make(co, c, k, k, wt);
        const Tensor y = conv2d_region(xt, Region{r0, r1, h, w}, wtt,
                                       std::span<const float>(bias, co), stride, pad);
        put(y, out);
    });
}
int ref_attention(const float* q, const float* k, const float* v, int n, int m, int s, int d,
                  int dv, float scale, float* out) {
    return guard([&] {
        put(attention(make(n, 1, m, d, q), make(n, 1, s, d, k), make(n, 1, s, dv, v), scale), out);
    });
}
int ref_linear(const float* tok, int n, int t, int in_f, const float* wt, int out_f,
               const float* bias, float* out) {
    return guard([&] {
        put(linear(make(n, 1, t, in_f, tok), make(out_f, in_f, 1, 1, wt),
                   std::span<const float>(bias, out_f)),
            out);
    });
}
// r0 < 0 selects the full extent.
int ref_group_stats(const float* x, int n, int c, int h, int w, int groups, int r0, int r1,
                    double* mean, double* mean_sq) {
    return guard([&] {
        std::optional<Region> reg;
        if (r0 >= 0) reg = Region{r0, r1, h, w};
        const GnStats s = group_stats(make(n, c, h, w, x), groups, reg);
        std::memcpy(mean, s.mean.data(), s.mean.size() * sizeof(double));
        std::memcpy(mean_sq, s.mean_sq.data(), s.mean_sq.size() * sizeof(double));
    });
}
int ref_group_norm_apply(const float* x, int n, int c, int h, int w, int r0, int r1, int groups,
                         const double* mean, const double* mean_sq, const float* gamma,
                         const float* beta, float eps, float* out) {
    return guard([&] {
        std::optional<Region> reg;
        if (r0 >= 0) reg = Region{r0, r1, h, w};
        GnStats s(n, groups);
        std::memcpy(s.mean.data(), mean, s.mean.size() * sizeof(double));
        std::memcpy(s.mean_sq.data(), mean_sq, s.mean_sq.size() * sizeof(double));
        put(group_norm_apply(make(n, c, h, w, x), reg, s, std::span<const float>(gamma, c),
                             std::span<const float>(beta, c), eps),
            out);
    });
}
int ref_corrected_gn_stats(int groups, const double* f, const double* pl, const double* pg,
                           double* out) {
    // each input: mean[groups] followed by mean_sq[groups]
    return guard([&] {
        auto mk = [&](const double* p) {
            GnStats s(1, groups);
            std::memcpy(s.mean.data(), p, groups * sizeof(double));
            std::memcpy(s.mean_sq.data(), p + groups, groups * sizeof(double));
            return s;
        };
        const GnStats o = corrected_gn_stats(mk(f), mk(pl), mk(pg));
        std::memcpy(out, o.mean.data(), groups * sizeof(double));
        std::memcpy(out + groups, o.mean_sq.data(), groups * sizeof(double));
    });
}
int ref_silu(const float* x, long count, float* out) {
    return guard([&] { put(silu(make(1, 1, 1, int(count), x)), out); });
}
int ref_upsample(const float* x, int n, int c, int h, int w, float* out) {
    return guard([&] { put(upsample_nearest2x(make(n, c, h, w, x)), out); });
}
int ref_random_normal(int n, int c, int h, int w, uint64_t seed, float* out) {
    return guard([&] { put(random_normal(n, c, h, w, seed), out); });
}
int ref_random_condition(int dim, uint64_t seed, float* out) {
    return guard([&] {
        const Condition c = random_condition(dim, seed);
        std::memcpy(out, c.values.data(), dim * sizeof(float));
    });
}
int ref_timestep_embedding(int t, int dim, float* out) {
    return guard([&] {
        auto e = timestep_embedding(t, dim);
        std::memcpy(out, e.data(), dim * sizeof(float));
    });
}
int ref_make_schedule(int total, double b0, double b1, double* abar) {
    return guard([&] {
        const NoiseSchedule s = make_schedule(total, b0, b1);
        std::memcpy(abar, s.alpha_bar.data(), total * sizeof(double));
    });
}
int ref_make_plan(int total, int steps, int* ts) {
    return guard([&] {
        const SamplerPlan p = make_plan(make_schedule(total), steps);
        std::memcpy(ts, p.timesteps.data(), steps * sizeof(int));
    });
}
int ref_ddim_update(const float* x, const float* eps, long count, double abar_t, double abar_n,
                    float* out) {
    return guard([&] {
        put(ddim_update(make(1, 1, 1, int(count), x), make(1, 1, 1, int(count), eps), abar_t,
                        abar_n),
            out);
    });
}
uint64_t ref_macs_of_layer(void* mp, int layer, int r0, int r1, int fh, int fw) {
    return macs_of_layer(static_cast<Model*>(mp)->layers.at(layer), Region{r0, r1, fh, fw});
}

}  // extern "C"
