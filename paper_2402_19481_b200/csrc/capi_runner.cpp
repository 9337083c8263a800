// C ABI: model, partition logic, PatchRunner and run_sampling entry points.
#include "capi_common.hpp"
#include "model.hpp"
#include "runtime.hpp"

#include <nccl.h>

#include <cmath>
#include <cstring>
#include <memory>

struct pp_model {
    pp::Model m;
};

struct pp_runner {
    pp::Model graph;  // layer graph (host weights released after upload)
    std::unique_ptr<pp::Runner> r;
};

namespace {

pp::ModelConfig cfg_of(const pp_model_config* c) {
    pp::ModelConfig m;
    m.in_channels = c->in_channels;
    m.base_channels = c->base_channels;
    m.levels = c->levels;
    m.groups = c->groups;
    m.cond_dim = c->cond_dim;
    m.attn_at_level = c->attn_at_level;
    m.res_blocks = c->res_blocks ? c->res_blocks : 1;
    m.attn_levels = c->attn_levels;
    m.attn_depth = c->attn_depth ? c->attn_depth : 1;
    m.attn_up = c->attn_up;
    return m;
}

void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string(what) + ": null pointer");
}

pp::RunnerOptions opts_of(const pp_runner_opts* o) {
    pp::RunnerOptions r;
    r.mode = o->mode;
    if (r.mode < 0 || r.mode > 3) throw std::invalid_argument("run_step: bad mode");
    r.n_devices = o->n_devices;
    r.warmup = o->warmup_steps;
    r.gn_scheme = o->gn_scheme;
    if (r.gn_scheme < 0 || r.gn_scheme > 2) throw std::invalid_argument("bad gn scheme");
    r.elem = pp::elem_of(o->dtype);
    r.world = o->world < 1 ? 1 : o->world;
    r.rank = o->rank;
    r.transport = o->transport;
    if (r.transport != PP_TRANSPORT_NCCL && r.transport != PP_TRANSPORT_IPC)
        throw std::invalid_argument("pp_runner_create: bad transport");
    if (r.world > 1 && r.transport == PP_TRANSPORT_NCCL) {
        need(o->nccl_id, "pp_runner_create(nccl_id)");
        const uint8_t* p = static_cast<const uint8_t*>(o->nccl_id);
        r.nccl_id.assign(p, p + 128);
    }
    r.device = o->device;
    r.profile = o->profile != 0;
    r.no_comm = o->no_comm != 0;
    r.stress = o->stress != 0;
    r.stress_seed = o->stress_seed;
    r.cfg_scale = o->cfg_scale;
    r.cond_tokens = o->cond_tokens;
    if (r.cond_tokens < 1) throw std::invalid_argument("pp_runner_create: cond_tokens must be >= 1");
    if (!std::isfinite(r.cfg_scale)) throw std::invalid_argument("pp_runner_create: cfg_scale not finite");
    r.cfg_pair_role = o->cfg_pair_role;
    r.cfg_pair_transport = o->cfg_pair_transport;
    if (r.cfg_pair_role < -1 || r.cfg_pair_role > 1)
        throw std::invalid_argument("pp_runner_create: cfg_pair_role must be -1, 0 or 1");
    const bool need_cfg_id = r.cfg_pair_role >= 0 ? r.cfg_pair_transport == PP_TRANSPORT_NCCL
                                                  : r.world > 1 && r.transport == PP_TRANSPORT_NCCL;
    if (r.cfg_scale != 0.0 && need_cfg_id) {
        need(o->cfg_nccl_id, "pp_runner_create(cfg_nccl_id)");
        const uint8_t* p = static_cast<const uint8_t*>(o->cfg_nccl_id);
        r.cfg_nccl_id.assign(p, p + 128);
    }
    return r;
}

}  // namespace

extern "C" {

PP_API int pp_model_build(const pp_model_config* cfg, uint64_t seed, pp_model** out) {
    return pp::guard([&] {
        need(cfg, "pp_model_build");
        need(out, "pp_model_build");
        auto m = std::make_unique<pp_model>();
        m->m = pp::build_model(cfg_of(cfg), seed);
        *out = m.release();
    });
}

PP_API int pp_model_from_pool(const pp_model_config* cfg, const float* pool, size_t pool_len,
                              pp_model** out) {
    return pp::guard([&] {
        need(cfg, "pp_model_from_pool");
        need(pool, "pp_model_from_pool");
        auto m = std::make_unique<pp_model>();
        m->m = pp::build_graph(cfg_of(cfg));
        size_t total = 0;
        for (auto& w : m->m.weights) total += w.size();
        if (total != pool_len)
            throw std::invalid_argument("weight pool has " + std::to_string(pool_len) +
                                        " floats, model expects " + std::to_string(total));
        size_t off = 0;
        for (auto& w : m->m.weights) {
            std::memcpy(w.data.data(), pool + off, w.size() * 4);
            off += w.size();
        }
        *out = m.release();
    });
}

PP_API void pp_model_destroy(pp_model* m) { delete m; }

PP_API int pp_model_num_layers(const pp_model* m) { return m ? int(m->m.layers.size()) : 0; }

PP_API int pp_model_layer(const pp_model* m, int id, pp_layer_desc* o) {
    return pp::guard([&] {
        need(m, "pp_model_layer");
        need(o, "pp_model_layer");
        if (id < 0 || id >= int(m->m.layers.size())) throw std::invalid_argument("layer id out of range");
        const pp::Layer& d = m->m.layers[id];
        o->id = d.id; o->kind = int(d.kind); o->in_ch = d.in_ch; o->out_ch = d.out_ch;
        o->kernel = d.kernel; o->stride = d.stride; o->pad = d.pad; o->groups = d.groups;
        o->eps = d.eps; o->cond_dim = d.cond_dim; o->skip_source = d.skip_source;
        o->scale_in = d.scale_in; o->scale_out = d.scale_out; o->weight = d.weight;
        o->bias = d.bias; o->weight2 = d.weight2; o->bias2 = d.bias2;
    });
}

PP_API int pp_model_num_weights(const pp_model* m) { return m ? int(m->m.weights.size()) : 0; }

PP_API int pp_model_weight_shape(const pp_model* m, int h, int* s) {
    return pp::guard([&] {
        need(m, "pp_model_weight_shape");
        const pp::WeightTensor& t = m->m.weights.at(size_t(h));
        s[0] = t.n; s[1] = t.c; s[2] = t.h; s[3] = t.w;
    });
}

PP_API size_t pp_model_pool_size(const pp_model* m) {
    size_t t = 0;
    if (m)
        for (auto& w : m->m.weights) t += w.size();
    return t;
}

PP_API int pp_model_pool(const pp_model* m, float* dst) {
    return pp::guard([&] {
        need(m, "pp_model_pool");
        need(dst, "pp_model_pool");
        size_t off = 0;
        for (auto& w : m->m.weights) {
            std::memcpy(dst + off, w.data.data(), w.size() * 4);
            off += w.size();
        }
    });
}

PP_API int pp_model_zero_weights(pp_model* m, int keep_biases) {
    return pp::guard([&] {
        need(m, "pp_model_zero_weights");
        for (const pp::Layer& d : m->m.layers) {
            for (int h : {d.weight, d.weight2})
                if (h >= 0) std::fill(m->m.weights[h].data.begin(), m->m.weights[h].data.end(), 0.0f);
            if (!keep_biases)
                for (int h : {d.bias, d.bias2})
                    if (h >= 0) std::fill(m->m.weights[h].data.begin(), m->m.weights[h].data.end(), 0.0f);
        }
    });
}

PP_API uint64_t pp_model_total_macs(const pp_model* m, int h, int w) {
    uint64_t r = 0;
    pp::guard([&] {
        need(m, "pp_model_total_macs");
        r = pp::model_total_macs(m->m, h, w);
    });
    return r;
}

PP_API int pp_partition_rows(int h, int n, int w, int* out) {
    return pp::guard([&] {
        auto rs = pp::partition_rows(h, n, w);
        for (int i = 0; i < n; ++i) {
            out[4 * i] = rs[i].row_start; out[4 * i + 1] = rs[i].row_end;
            out[4 * i + 2] = rs[i].full_h; out[4 * i + 3] = rs[i].full_w;
        }
    });
}

PP_API int pp_derive_patch_spec(const pp_model* m, const int* r4, int* lin, int* lout) {
    return pp::guard([&] {
        need(m, "pp_derive_patch_spec");
        const pp::PatchSpec s = pp::derive_patch_spec(m->m, pp::Region{r4[0], r4[1], r4[2], r4[3]});
        for (size_t l = 0; l < s.layer_in.size(); ++l) {
            const pp::Region& a = s.layer_in[l];
            const pp::Region& b = s.layer_out[l];
            lin[4 * l] = a.row_start; lin[4 * l + 1] = a.row_end; lin[4 * l + 2] = a.full_h; lin[4 * l + 3] = a.full_w;
            lout[4 * l] = b.row_start; lout[4 * l + 1] = b.row_end; lout[4 * l + 2] = b.full_h; lout[4 * l + 3] = b.full_w;
        }
    });
}

PP_API int pp_corrected_gn_stats(int g, const double* f, const double* pl, const double* pg,
                                 double* out) {
    // corrected_gn_stats (proj/src/runtime.cpp:85-106), host restatement for the C ABI
    return pp::guard([&] {
        if (g <= 0) throw std::invalid_argument("corrected_gn_stats: group-count mismatch");
        for (int e = 0; e < g; ++e) {
            double m = f[e], q = f[g + e];
            if (!(pg[e] == pl[e] && pg[g + e] == pl[g + e])) {
                const double cm = pg[e] + (f[e] - pl[e]);
                const double cq = pg[g + e] + (f[g + e] - pl[g + e]);
                if (!(cq - cm * cm < 0.0)) {
                    m = cm;
                    q = cq;
                }
            }
            out[e] = m;
            out[g + e] = q;
        }
    });
}

PP_API void pp_run_config_default(pp_run_config* c) {
    if (!c) return;
    c->mode = PP_MODE_REFERENCE;
    c->n_devices = 1;
    c->h = c->w = 48;
    c->num_steps = 50;
    c->warmup = 4;
    c->gn_scheme = PP_GN_CORRECTED;
    c->dtype = PP_DTYPE_BF16;
    c->model_seed = 42;
    c->noise_seed = 1234;
    c->cond_seed = 7;
    c->model = pp_model_config{4, 16, 3, 4, 8, -1, 0, 0, 0, 0};
    c->schedule_steps = 1000;
    c->beta_start = 1e-4;
    c->beta_end = 2e-2;
}

static void validate_cfg(const pp_run_config* c) {
    // RunConfig::validate (proj/src/runtime.cpp:480-492)
    const pp::ModelConfig mc = cfg_of(&c->model);
    mc.validate();
    if (c->n_devices < 1) throw std::invalid_argument("config: devices must be >= 1");
    if (c->num_steps < 1 || c->num_steps > c->schedule_steps)
        throw std::invalid_argument("config: steps out of range");
    if (c->warmup < 0) throw std::invalid_argument("config: warmup must be >= 0");
    if (c->h <= 0 || c->w <= 0) throw std::invalid_argument("config: bad image size");
    const int div = mc.depth_divisor() * c->n_devices;
    if (c->h % div != 0 || c->w % div != 0)
        throw std::invalid_argument("config: size " + std::to_string(c->h) + "x" + std::to_string(c->w) +
                                    " must be divisible by devices*2^(levels-1) = " + std::to_string(div));
}

PP_API int pp_run_config_validate(const pp_run_config* c) {
    return pp::guard([&] {
        need(c, "pp_run_config_validate");
        validate_cfg(c);
    });
}

PP_API int pp_make_schedule(int total, double b0, double b1, double* abar) {
    return pp::guard([&] {
        auto a = pp::make_schedule(total, b0, b1);
        std::memcpy(abar, a.data(), a.size() * 8);
    });
}

PP_API int pp_make_plan(int total, int steps, int* ts) {
    return pp::guard([&] {
        auto p = pp::make_plan(total, steps);
        std::memcpy(ts, p.data(), p.size() * 4);
    });
}

PP_API int pp_random_normal(int n, int c, int h, int w, uint64_t seed, float* out) {
    return pp::guard([&] {
        auto v = pp::gaussian(seed, size_t(n) * c * h * w);
        std::memcpy(out, v.data(), v.size() * 4);
    });
}

PP_API int pp_random_condition(int dim, uint64_t seed, float* out) {
    return pp::guard([&] {
        auto v = pp::gaussian(seed, size_t(dim));
        std::memcpy(out, v.data(), v.size() * 4);
    });
}

PP_API uint64_t pp_macs_of_layer(const pp_model* m, int layer, const int* r4) {
    uint64_t v = 0;
    pp::guard([&] {
        need(m, "pp_macs_of_layer");
        v = pp::macs_of_layer(m->m.layers.at(size_t(layer)), pp::Region{r4[0], r4[1], r4[2], r4[3]});
    });
    return v;
}

PP_API void pp_runner_opts_default(pp_runner_opts* o) {
    if (!o) return;
    o->mode = PP_MODE_REFERENCE;
    o->n_devices = 1;
    o->warmup_steps = 4;
    o->gn_scheme = PP_GN_CORRECTED;
    o->dtype = PP_DTYPE_BF16;
    o->world = 1;
    o->rank = 0;
    o->nccl_id = nullptr;
    o->device = 0;
    o->profile = 0;
    o->transport = PP_TRANSPORT_NCCL;
    o->no_comm = 0;
    o->stress = 0;
    o->stress_seed = 0xC0FFEEull;
    o->cfg_scale = 0.0;
    o->uncond = nullptr;
    o->cfg_nccl_id = nullptr;
    o->cond_tokens = 1;
    o->cfg_pair_role = -1;
    o->cfg_pair_transport = PP_TRANSPORT_NCCL;
}

PP_API int pp_runner_create(const pp_model* m, const float* cond, int cond_dim, int h, int w,
                            const pp_runner_opts* opts, pp_runner** out) {
    return pp::guard([&] {
        need(m, "pp_runner_create(model)");
        need(opts, "pp_runner_create(opts)");
        need(out, "pp_runner_create(out)");
        auto r = std::make_unique<pp_runner>();
        r->graph = m->m;
        std::vector<float> c(cond, cond + (cond ? cond_dim : 0));
        pp::RunnerOptions ro = opts_of(opts);
        if (ro.cfg_scale != 0.0 && opts->uncond) ro.uncond.assign(opts->uncond, opts->uncond + cond_dim);
        r->r = std::make_unique<pp::Runner>(r->graph, c, h, w, ro);
        for (auto& t : r->graph.weights) std::vector<float>().swap(t.data);
        *out = r.release();
    });
}

PP_API void pp_runner_destroy(pp_runner* r) { delete r; }

PP_API int pp_runner_step(pp_runner* r, int entry, const float* x, int t, int step, float* eps) {
    return pp::guard([&] {
        need(r, "pp_runner_step");
        need(x, "pp_runner_step(x)");
        need(eps, "pp_runner_step(eps)");
        if (entry < 0 || entry > 4) throw std::invalid_argument("run_step: bad mode");
        r->r->step(entry, x, t, step, eps);
    });
}

PP_API int pp_runner_patch_spec(const pp_runner* r, int device, int* lin, int* lout) {
    return pp::guard([&] {
        need(r, "pp_runner_patch_spec");
        const pp::PatchSpec& s = r->r->patch_spec(device);
        for (size_t l = 0; l < s.layer_in.size(); ++l) {
            const pp::Region& a = s.layer_in[l];
            const pp::Region& b = s.layer_out[l];
            lin[4 * l] = a.row_start; lin[4 * l + 1] = a.row_end; lin[4 * l + 2] = a.full_h; lin[4 * l + 3] = a.full_w;
            lout[4 * l] = b.row_start; lout[4 * l + 1] = b.row_end; lout[4 * l + 2] = b.full_h; lout[4 * l + 3] = b.full_w;
        }
    });
}

PP_API long pp_runner_cached_input(pp_runner* r, int device, int layer, float* dst, int* nchw4) {
    long n = -1;
    pp::guard([&] {
        need(r, "pp_runner_cached_input");
        n = r->r->cached_input(device, layer, dst, nchw4);
    });
    return n;
}

PP_API uint64_t pp_runner_total_macs(const pp_runner* r) { return r ? r->r->total_macs() : 0; }

PP_API int pp_runner_step_device_macs(const pp_runner* r, int step, uint64_t* per_device) {
    return pp::guard([&] {
        need(r, "pp_runner_step_device_macs");
        auto v = r->r->step_device_macs(step);
        if (v.empty()) throw std::invalid_argument("step index out of range");
        std::memcpy(per_device, v.data(), v.size() * 8);
    });
}

PP_API int pp_runner_volumes(const pp_runner* r, uint64_t* v6) {
    return pp::guard([&] {
        need(r, "pp_runner_volumes");
        const pp::CommVolumes v = r->r->volumes();
        v6[0] = v.allgather_recv; v6[1] = v.allgather_sent; v6[2] = v.halo_recv;
        v6[3] = v.halo_sent; v6[4] = v.statreduce_recv; v6[5] = v.statreduce_sent;
    });
}

// RawTrace of `device` (proj/include/patchsim/trace.hpp:18-35) as rows of 9 uint64:
// {device, step, layer (int64), kind, prim, macs, bytes_recv, bytes_sent, tag}.  Returns the
// event count (rows written: min(count, cap)); out may be null to query the count.
PP_API long pp_runner_trace(const pp_runner* r, int device, uint64_t* out9, long cap) {
    long n = -1;
    const int rc = pp::guard([&] {
        need(r, "pp_runner_trace");
        const auto& t = r->r->trace(device);
        n = long(t.size());
        if (!out9) return;
        for (long i = 0; i < n && i < cap; ++i) {
            const pp::TraceEvent& e = t[size_t(i)];
            uint64_t* o = out9 + 9 * i;
            o[0] = uint64_t(e.device); o[1] = uint64_t(e.step); o[2] = uint64_t(int64_t(e.layer));
            o[3] = uint64_t(e.kind); o[4] = uint64_t(e.prim); o[5] = e.macs;
            o[6] = e.bytes_recv; o[7] = e.bytes_sent; o[8] = e.tag;
        }
    });
    return rc == PP_OK ? n : -1;
}

PP_API int pp_runner_sample(pp_runner* r, const float* x_T, const int* ts, int n, const double* abar,
                            int total, float* x0, float* traj) {
    return pp::guard([&] {
        need(r, "pp_runner_sample");
        need(x_T, "pp_runner_sample(x_T)");
        need(ts, "pp_runner_sample(timesteps)");
        need(abar, "pp_runner_sample(alpha_bar)");
        need(x0, "pp_runner_sample(x0)");
        r->r->sample(x_T, ts, n, abar, total, x0, traj);
    });
}

PP_API int pp_runner_profile(pp_runner* r, double* o) {
    return pp::guard([&] {
        need(r, "pp_runner_profile");
        const pp::ProfileTotals p = r->r->profile();
        o[0] = p.conv_ms; o[1] = p.conv_flops; o[2] = p.gemm_ms; o[3] = p.gemm_flops;
        o[4] = p.gn_ms; o[5] = p.other_ms; o[6] = double(r->r->launches());
    });
}

PP_API long pp_runner_launches(const pp_runner* r) { return r ? r->r->launches() : 0; }

PP_API double pp_runner_last_device_ms(const pp_runner* r) { return r ? r->r->last_device_ms() : 0.0; }

PP_API int pp_runner_set_profile(pp_runner* r, int on) {
    return pp::guard([&] {
        need(r, "pp_runner_set_profile");
        r->r->set_profile(on != 0);
    });
}

PP_API int pp_assemble_bands(const float* gathered, int n_bands, int c, int rows, int w,
                             float* out) {
    return pp::guard([&] {
        need(gathered, "pp_assemble_bands");
        need(out, "pp_assemble_bands");
        if (n_bands < 1 || c < 1 || rows < 1 || w < 1) throw std::invalid_argument("pp_assemble_bands: bad shape");
        pp::assemble_bands(gathered, n_bands, c, rows, w, out);
    });
}

PP_API int pp_runner_ipc_export(pp_runner* r, void* out, long cap, long* size) {
    return pp::guard([&] {
        need(r, "pp_runner_ipc_export");
        need(size, "pp_runner_ipc_export(size)");
        const auto blob = r->r->ipc_export();
        *size = long(blob.size());
        if (out && cap >= *size) std::memcpy(out, blob.data(), blob.size());
    });
}

PP_API int pp_runner_ipc_connect(pp_runner* r, const void* blobs, long per_rank) {
    return pp::guard([&] {
        need(r, "pp_runner_ipc_connect");
        need(blobs, "pp_runner_ipc_connect");
        if (per_rank <= 0) throw std::invalid_argument("pp_runner_ipc_connect: bad blob size");
        r->r->ipc_connect(static_cast<const uint8_t*>(blobs), size_t(per_rank));
    });
}

PP_API int pp_runner_pair_export(pp_runner* r, void* out, long cap, long* size) {
    return pp::guard([&] {
        need(r, "pp_runner_pair_export");
        need(size, "pp_runner_pair_export(size)");
        const auto blob = r->r->pair_export();
        *size = long(blob.size());
        if (out && cap >= *size) std::memcpy(out, blob.data(), blob.size());
    });
}

PP_API int pp_runner_pair_connect(pp_runner* r, const void* blob, long size) {
    return pp::guard([&] {
        need(r, "pp_runner_pair_connect");
        need(blob, "pp_runner_pair_connect");
        if (size <= 0) throw std::invalid_argument("pp_runner_pair_connect: bad blob size");
        r->r->pair_connect(static_cast<const uint8_t*>(blob), size_t(size));
    });
}

PP_API int pp_nccl_unique_id(void* out128) {
    return pp::guard([&] {
        need(out128, "pp_nccl_unique_id");
        ncclUniqueId id;
        const ncclResult_t rc = ncclGetUniqueId(&id);
        if (rc != ncclSuccess) throw pp::NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(rc));
        std::memcpy(out128, &id, sizeof(id));
    });
}

PP_API int pp_run_sampling(const pp_run_config* c, float* x0, float* traj, uint64_t* total_macs) {
    // run_sampling (proj/src/runtime.cpp:494-526)
    return pp::guard([&] {
        need(c, "pp_run_sampling");
        need(x0, "pp_run_sampling(x0)");
        validate_cfg(c);
        const pp::ModelConfig mc = cfg_of(&c->model);
        const pp::Model model = pp::build_model(mc, c->model_seed);
        const std::vector<float> cond = pp::gaussian(c->cond_seed, size_t(mc.cond_dim));
        const std::vector<double> abar = pp::make_schedule(c->schedule_steps, c->beta_start, c->beta_end);
        const std::vector<int> plan = pp::make_plan(c->schedule_steps, c->num_steps);
        pp::RunnerOptions o;
        o.mode = c->mode;
        o.n_devices = c->mode == PP_MODE_REFERENCE ? 1 : c->n_devices;
        o.warmup = c->warmup;
        o.gn_scheme = c->gn_scheme;
        o.elem = pp::elem_of(c->dtype);
        pp::Runner runner(model, cond, c->h, c->w, o);
        const std::vector<float> xT = pp::gaussian(c->noise_seed, size_t(mc.in_channels) * c->h * c->w);
        runner.sample(xT.data(), plan.data(), int(plan.size()), abar.data(), c->schedule_steps, x0, traj);
        if (total_macs) *total_macs = runner.total_macs();
    });
}

}  // extern "C"
