// C-ABI wrappers of the host tiers (net init, profile, stream, planner,
// simulator). These are the bit-exact, host-side parts of the contract: the
// implementations are the drop-in headers under include/ferret/, and
// tests/test_host_parity.py byte-diffs their output against the reference.
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "common.hpp"
#include "ferret/net.hpp"
#include "ferret/planner.hpp"
#include "ferret/profile.hpp"
#include "ferret/sim.hpp"
#include "ferret/stream.hpp"
#include "schedule.hpp"

namespace fb200 {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

} // namespace fb200

using fb200::fail;
using fb200::guarded;


namespace {

ferret::ModelProfile to_profile(const ferret_layer_profile* layers, int32_t n) {
    if (!layers || n <= 0) fail(FERRET_E_INVALID_ARG, "profile: no layers");
    ferret::ModelProfile p;
    for (int32_t i = 0; i < n; ++i) p.layers.push_back({layers[i].t_f, layers[i].t_b, layers[i].w, layers[i].a});
    return p;
}

ferret::StreamSpec to_spec(const ferret_stream_spec* s) {
    ferret::StreamSpec spec;
    if (s) spec = {s->t_d, s->decay_c, s->value, s->horizon};
    return spec;
}

std::vector<std::size_t> to_widths(const uint64_t* widths, int32_t n) {
    if (!widths || n < 0) fail(FERRET_E_INVALID_ARG, "widths: null");
    return std::vector<std::size_t>(widths, widths + n);
}

size_t copy_text(const std::string& s, char* buf, size_t cap) {
    if (buf && cap > 0) {
        const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return s.size() + 1;
}

} // namespace

extern "C" {

const char* ferret_last_error(void) { return fb200::g_last_error.c_str(); }

const char* ferret_version(void) { return "ferret-b200 0.1 (sm_100a)"; }

size_t ferret_net_param_count(const uint64_t* widths, int32_t n_widths) {
    size_t total = 0;
    for (int32_t i = 0; i + 1 < n_widths; ++i) total += widths[i] * widths[i + 1] + widths[i + 1];
    return total;
}

ferret_status ferret_make_dense_net(const uint64_t* widths, int32_t n_widths, uint64_t seed, int32_t hidden_act,
                                    double* params_out, size_t n_params) {
    return guarded([&] {
        const ferret::DenseNet net = ferret::make_dense_net(to_widths(widths, n_widths), seed,
                                                            static_cast<ferret::Activation>(hidden_act));
        if (n_params != net.n_params()) fail(FERRET_E_INVALID_ARG, "make_dense_net: params_out size mismatch");
        size_t at = 0;
        for (const auto& l : net.layers) {
            std::memcpy(params_out + at, l.W.data(), l.W.size() * sizeof(double));
            at += l.W.size();
            std::memcpy(params_out + at, l.b.data(), l.b.size() * sizeof(double));
            at += l.b.size();
        }
    });
}

ferret_status ferret_profile_from_widths(const uint64_t* widths, int32_t n_widths, double seconds_per_param,
                                         ferret_layer_profile* layers_out) {
    return guarded([&] {
        if (n_widths < 2) fail(FERRET_E_CONFIG, "net needs at least input and output widths");
        ferret::DenseNet net;
        for (int32_t i = 0; i + 1 < n_widths; ++i) {
            ferret::DenseLayer l;
            l.in = widths[i];
            l.out = widths[i + 1];
            l.W.resize(l.in * l.out);
            l.b.resize(l.out);
            net.layers.push_back(std::move(l));
        }
        const ferret::ModelProfile p = ferret::profile_from_net(net, seconds_per_param);
        for (size_t i = 0; i < p.layers.size(); ++i)
            layers_out[i] = {p.layers[i].t_f, p.layers[i].t_b, p.layers[i].w, p.layers[i].a};
    });
}

ferret_status ferret_synth_drift_stream(size_t n, size_t n_features, size_t n_classes, int32_t drift, uint64_t seed,
                                        double rotate_rate, double noise, double* features_out,
                                        uint64_t* labels_out) {
    return guarded([&] {
        const ferret::DataStream ds = ferret::synth_drift_stream(n, n_features, n_classes,
                                                                 static_cast<ferret::DriftKind>(drift), seed,
                                                                 rotate_rate, noise);
        for (size_t i = 0; i < n; ++i) {
            std::memcpy(features_out + i * n_features, ds.items[i].features.data(), n_features * sizeof(double));
            labels_out[i] = ds.items[i].label;
        }
    });
}

ferret_status ferret_schedule_plan(const ferret_layer_profile* layers, int32_t n_layers, double t_d,
                                   const ferret_stream_spec* spec, uint64_t budget, int32_t max_stages,
                                   size_t n_items, ferret_schedule** out) {
    return guarded([&] {
        auto s = std::make_unique<ferret_schedule>();
        s->spec = to_spec(spec);
        ferret::PlanFilter filt;
        filt.max_stages = max_stages > 0 ? static_cast<std::size_t>(max_stages) : 0;
        const ferret::ModelProfile prof = to_profile(layers, n_layers);
        s->plan = ferret::plan_within(prof, t_d, s->spec, budget, filt);
        const ferret::StageStats st = ferret::stage_stats(prof, s->plan.partition);
        s->trace = ferret::simulate(st, s->plan.config, s->spec, n_items);
        *out = s.release();
    });
}

ferret_status ferret_schedule_forced(const ferret_layer_profile* layers, int32_t n_layers, double t_d,
                                     const ferret_stream_spec* spec, const uint64_t* bounds, int32_t n_bounds,
                                     int32_t recompute, size_t n_items, ferret_schedule** out) {
    return guarded([&] {
        auto s = std::make_unique<ferret_schedule>();
        s->spec = to_spec(spec);
        const ferret::ModelProfile prof = to_profile(layers, n_layers);
        s->plan.partition.bounds.assign(bounds, bounds + n_bounds);
        const ferret::StageStats st = ferret::stage_stats(prof, s->plan.partition);
        s->plan.config = ferret::default_config(st, t_d, recompute);
        s->plan.rate = ferret::adaptation_rate(st, s->plan.config, s->spec);
        s->plan.memory = ferret::memory_footprint(st, s->plan.config);
        s->trace = ferret::simulate(st, s->plan.config, s->spec, n_items);
        *out = s.release();
    });
}

ferret_status ferret_schedule_load(const char* plan_text, size_t plan_len, const char* trace_text, size_t trace_len,
                                   ferret_schedule** out) {
    return guarded([&] {
        if (!plan_text || !trace_text || !out) fail(FERRET_E_INVALID_ARG, "schedule_load: null argument");
        auto s = std::make_unique<ferret_schedule>();
        std::istringstream pin(std::string(plan_text, plan_len));
        s->plan = ferret::parse_plan(pin, "plan");
        std::istringstream tin(std::string(trace_text, trace_len));
        ferret::LoadedTrace lt = ferret::parse_trace(tin, "trace");
        s->trace = std::move(lt.trace);
        s->spec.t_d = s->trace.t_d;
        s->spec.horizon = static_cast<double>(s->trace.n_items) * s->trace.t_d;
        const std::size_t P = s->plan.partition.stages();
        for (const ferret::SimEvent& e : s->trace.events)
            if (e.stage >= static_cast<int>(P)) fail(FERRET_E_SCHEMA, "trace: event stage beyond the plan's partition");
        *out = s.release();
    });
}

int32_t ferret_schedule_bounds(const ferret_schedule* s, uint64_t* out, int32_t cap) {
    const auto& b = s->plan.partition.bounds;
    for (int32_t i = 0; i < cap && i < static_cast<int32_t>(b.size()); ++i) out[i] = b[static_cast<size_t>(i)];
    return static_cast<int32_t>(b.size());
}

size_t ferret_schedule_event_count(const ferret_schedule* s) { return s->trace.events.size(); }

ferret_status ferret_schedule_events(const ferret_schedule* s, ferret_event* out, size_t cap) {
    return guarded([&] {
        if (cap < s->trace.events.size()) fail(FERRET_E_INVALID_ARG, "schedule_events: buffer too small");
        size_t i = 0;
        for (const ferret::SimEvent& e : s->trace.events)
            out[i++] = ferret_event{e.time, static_cast<int32_t>(e.kind), e.worker, e.stage, e.staleness, e.item,
                                    e.version};
    });
}

size_t ferret_schedule_plan_text(const ferret_schedule* s, char* buf, size_t cap) {
    std::ostringstream os;
    ferret::write_plan(os, s->plan);
    return copy_text(os.str(), buf, cap);
}

size_t ferret_schedule_trace_text(const ferret_schedule* s, char* buf, size_t cap) {
    std::ostringstream os;
    ferret::write_trace(os, s->trace, s->spec);
    return copy_text(os.str(), buf, cap);
}

void ferret_schedule_destroy(ferret_schedule* s) { delete s; }

struct ferret_csv {
    ferret::DataStream ds;
};

ferret_status ferret_csv_load(const char* path, const char* label_column, ferret_csv** out) {
    return guarded([&] {
        if (!path || !label_column || !out) fail(FERRET_E_INVALID_ARG, "csv_load: null argument");
        auto c = std::make_unique<ferret_csv>();
        c->ds = ferret::load_csv_stream(path, label_column);
        *out = c.release();
    });
}

ferret_status ferret_csv_shape(const ferret_csv* c, size_t* n_items, size_t* n_features, size_t* n_classes) {
    return guarded([&] {
        if (!c || !n_items || !n_features || !n_classes) fail(FERRET_E_INVALID_ARG, "csv_shape: null argument");
        *n_items = c->ds.items.size();
        *n_features = c->ds.n_features;
        *n_classes = c->ds.n_classes;
    });
}

ferret_status ferret_csv_read(const ferret_csv* c, double* features, uint64_t* labels) {
    return guarded([&] {
        if (!c || !features || !labels) fail(FERRET_E_INVALID_ARG, "csv_read: null argument");
        const size_t f = c->ds.n_features;
        for (size_t i = 0; i < c->ds.items.size(); ++i) {
            std::memcpy(features + i * f, c->ds.items[i].features.data(), f * sizeof(double));
            labels[i] = c->ds.items[i].label;
        }
    });
}

void ferret_csv_destroy(ferret_csv* c) { delete c; }

ferret_status ferret_apply_skip_policy(size_t n_items, double t_d, int32_t kind, uint64_t window, uint64_t keep,
                                      uint64_t seed, double processing_time, int64_t* kept_out, double* start_out,
                                      size_t* n_kept) {
    return guarded([&] {
        if (!n_kept || (n_items && !kept_out)) fail(FERRET_E_INVALID_ARG, "apply_skip_policy: null buffer");
        if (kind < 0 || kind > 3) fail(FERRET_E_CONFIG, "unknown skip policy");
        ferret::SkipPolicy p;
        p.kind = static_cast<ferret::SkipKind>(kind);
        p.window = static_cast<std::size_t>(window);
        p.keep = static_cast<std::size_t>(keep);
        p.seed = seed;
        const ferret::FilteredStream fs = ferret::apply_skip_policy(n_items, t_d, p, processing_time);
        for (size_t i = 0; i < fs.kept.size(); ++i) {
            kept_out[i] = fs.kept[i].index;
            if (start_out) start_out[i] = fs.kept[i].start;
        }
        *n_kept = fs.kept.size();
    });
}

void ferret_train_opts_default(ferret_train_opts* o) {
    o->policy = FERRET_POLICY_NONE;
    o->lr = 1e-3;
    o->eta_lambda = 1e-3;
    o->lambda0 = 0.2;
    o->alpha = 0.99;
    o->nu = 2e-6;
    o->replay = 0;
    o->replay_seed = 0;
    o->replay_capacity = 5000;
    o->precision = FERRET_PREC_FP32;
    o->micro_batch = 1;
    o->device = 0;
    o->as_shipped = 0;
}

} // extern "C"
