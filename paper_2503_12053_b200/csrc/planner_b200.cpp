// The reference planner re-costed for B200 (north-star item 4; C ABI in ferret_b200.h,
// drop-in C++ in include/ferret/b200_cost.hpp).
//
// The reference prices plans with synthetic times (profile_from_net, net.hpp:263-274:
// t_f = 1e-6 s per parameter, t_b = 2 t_f) and memory in parameter/activation COUNT
// units (analytics.hpp:58-104: per worker and stage, multiplicity x (w + a)). Here the
// search itself (planner.hpp:108-215) is unchanged; what changes is what it is fed:
//   * t_f / t_b measured on the device (ferret_measure_profile): the mean device time of
//     one forward / backward + update event of each layer, replaying the real kernels
//     with one layer per stage;
//   * w / a in HBM bytes of this trainer's layout (ferret_b200_byte_profile);
//   * the plan-independent bytes (compensator state, normalizer, staging, replay pool)
//     taken off the budget up front;
//   * candidate partitions limited to max_stages = #GPUs.
// The chosen plan is then priced EXACTLY: a plan-only trainer (no device) runs the dry
// pass over the plan's event log that sizes the version rings and the stash
// (ferret_trainer_footprint). If that exceeds the budget, the search is re-run under a
// proportionally tightened budget (the reference model and the exact retention differ:
// the reference counts a version per worker, the trainer keeps a version as long as
// any in-flight unit reads it).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "common.hpp"
#include "ferret/net.hpp"
#include "ferret/stream.hpp"
#include "schedule.hpp"

using fb200::fail;
using fb200::guarded;

namespace {

struct TrainerGuard {
    ferret_trainer* t = nullptr;
    ~TrainerGuard() {
        if (t) ferret_trainer_destroy(t);
    }
};

void check(ferret_status s) {
    if (s != FERRET_OK) fail(s, ferret_last_error());
}

std::vector<ferret_event> to_events(const ferret::SimTrace& tr) {
    std::vector<ferret_event> ev;
    ev.reserve(tr.events.size());
    for (const ferret::SimEvent& e : tr.events)
        ev.push_back(ferret_event{e.time, static_cast<int32_t>(e.kind), e.worker, e.stage, e.staleness, e.item,
                                  e.version});
    return ev;
}

struct DenseDesc {
    std::vector<uint64_t> in, out;
    std::vector<int32_t> act;
    ferret_net_desc desc{};
    DenseDesc(const uint64_t* widths, int32_t n_widths, const double* params) {
        for (int32_t i = 0; i + 1 < n_widths; ++i) {
            in.push_back(widths[i]);
            out.push_back(widths[i + 1]);
            act.push_back(i + 2 < n_widths ? FERRET_ACT_RELU : FERRET_ACT_IDENTITY);
        }
        desc.n_layers = n_widths - 1;
        desc.in = in.data();
        desc.out = out.data();
        desc.act = act.data();
        desc.params = params;
        desc.geom = nullptr;
    }
};

ferret_train_opts train_opts(const ferret_b200_cost& c, int32_t device) {
    ferret_train_opts o{};
    ferret_train_opts_default(&o);
    o.policy = c.policy;
    o.eta_lambda = c.eta_lambda;
    o.replay = c.replay;
    o.replay_capacity = c.replay_capacity;
    o.precision = c.precision;
    o.micro_batch = c.micro_batch;
    o.device = device;
    return o;
}

// exact HBM bytes of a trainer running `events` with partition `bounds` (plan-only: no device)
ferret_footprint trainer_footprint(const uint64_t* widths, int32_t n_widths, const std::vector<uint64_t>& bounds,
                                   const ferret_b200_cost& c, const std::vector<ferret_event>& events,
                                   size_t chunk_units) {
    DenseDesc net(widths, n_widths, nullptr);
    const ferret_train_opts o = train_opts(c, -1);
    TrainerGuard g;
    check(ferret_trainer_create(&net.desc, bounds.data(), static_cast<int32_t>(bounds.size()), &o, &g.t));
    check(ferret_trainer_set_schedule(g.t, events.data(), events.size(),
                                      chunk_units * static_cast<size_t>(std::max(c.micro_batch, 1))));
    ferret_footprint f{};
    check(ferret_trainer_footprint(g.t, &f));
    return f;
}

ferret::ModelProfile byte_profile(const ferret::ModelProfile& p, const ferret_b200_cost& c) {
    ferret::ModelProfile out = p;
    const uint64_t per_version = sizeof(float) + (c.precision == FERRET_PREC_BF16 ? sizeof(uint16_t) : 0);
    const uint64_t per_act = 2 * sizeof(float) * static_cast<uint64_t>(std::max(c.micro_batch, 1));
    for (ferret::LayerProfile& l : out.layers) {
        l.w *= per_version;
        l.a *= per_act;
    }
    return out;
}

ferret::ModelProfile to_profile(const ferret_layer_profile* layers, int32_t n) {
    if (!layers || n <= 0) fail(FERRET_E_INVALID_ARG, "profile: no layers");
    ferret::ModelProfile p;
    for (int32_t i = 0; i < n; ++i) p.layers.push_back({layers[i].t_f, layers[i].t_b, layers[i].w, layers[i].a});
    return p;
}

void validate_cost(const ferret_b200_cost* c) {
    if (!c) fail(FERRET_E_INVALID_ARG, "b200 cost: null");
    if (c->micro_batch < 1 || c->micro_batch > 16) fail(FERRET_E_CONFIG, "b200 cost: micro_batch must be in [1, 16]");
}

} // namespace

extern "C" {

void ferret_b200_cost_default(ferret_b200_cost* c) {
    if (!c) return;
    *c = ferret_b200_cost{};
    c->micro_batch = 1;
    c->precision = FERRET_PREC_FP32;
    c->policy = FERRET_POLICY_ITER_FISHER;
    c->eta_lambda = 1e-3;
    c->replay = 0;
    c->replay_capacity = 5000;
    c->chunk_units = 0;
}

ferret_status ferret_b200_byte_profile(const ferret_layer_profile* layers, int32_t n_layers,
                                       const ferret_b200_cost* cost, ferret_layer_profile* out) {
    return guarded([&] {
        validate_cost(cost);
        if (!out) fail(FERRET_E_INVALID_ARG, "byte_profile: null output");
        const ferret::ModelProfile p = byte_profile(to_profile(layers, n_layers), *cost);
        for (int32_t i = 0; i < n_layers; ++i) {
            const ferret::LayerProfile& l = p.layers[static_cast<size_t>(i)];
            out[i] = {l.t_f, l.t_b, l.w, l.a};
        }
    });
}

ferret_status ferret_measure_profile(const uint64_t* widths, int32_t n_widths, const ferret_b200_cost* cost,
                                     int32_t units, int32_t device, ferret_layer_profile* layers_out) {
    return guarded([&] {
        validate_cost(cost);
        if (!widths || n_widths < 2 || !layers_out) fail(FERRET_E_INVALID_ARG, "measure_profile: bad arguments");
        if (units < 4) fail(FERRET_E_INVALID_ARG, "measure_profile: at least 4 units");
        const int32_t L = n_widths - 1;
        if (L > 16) fail(FERRET_E_CONFIG, "measure_profile: at most 16 layers (one stage per layer)");
        const std::vector<size_t> w(widths, widths + n_widths);
        // the reference's counts and synthetic times, then one stage per layer
        std::vector<ferret_layer_profile> syn(static_cast<size_t>(L));
        check(ferret_profile_from_widths(widths, n_widths, 1e-6, syn.data()));
        double t_d = 0.0;
        for (const auto& l : syn) t_d = std::max(t_d, l.t_f);
        std::vector<uint64_t> bounds(static_cast<size_t>(L) + 1);
        for (int32_t i = 0; i <= L; ++i) bounds[static_cast<size_t>(i)] = static_cast<uint64_t>(i);
        const ferret_stream_spec spec{t_d, 0.0, 1.0, units * t_d};
        ferret_schedule* sp = nullptr;
        check(ferret_schedule_forced(syn.data(), L, t_d, &spec, bounds.data(), L + 1, 0, static_cast<size_t>(units), &sp));
        std::unique_ptr<ferret_schedule, void (*)(ferret_schedule*)> sched(sp, ferret_schedule_destroy);
        const std::vector<ferret_event> events = to_events(sched->trace);
        const size_t B = static_cast<size_t>(cost->micro_batch);
        const size_t chunk = static_cast<size_t>(units) * B;
        const ferret::DataStream ds =
            ferret::synth_drift_stream(2 * chunk, w.front(), w.back(), ferret::DriftKind::split_tasks, 7, 1.5e-4, 0.55);
        std::vector<double> feats(2 * chunk * w.front());
        std::vector<uint64_t> labels(2 * chunk);
        for (size_t i = 0; i < 2 * chunk; ++i) {
            std::memcpy(feats.data() + i * w.front(), ds.items[i].features.data(), w.front() * sizeof(double));
            labels[i] = ds.items[i].label;
        }
        const ferret::DenseNet dn = ferret::make_dense_net(w, 1, ferret::Activation::relu);
        std::vector<double> params;
        params.reserve(dn.n_params());
        for (const auto& l : dn.layers) {
            params.insert(params.end(), l.W.begin(), l.W.end());
            params.insert(params.end(), l.b.begin(), l.b.end());
        }
        DenseDesc net(widths, n_widths, params.data());
        const ferret_train_opts o = train_opts(*cost, device);
        TrainerGuard g;
        check(ferret_trainer_create(&net.desc, bounds.data(), L + 1, &o, &g.t));
        check(ferret_trainer_load_stream(g.t, feats.data(), labels.data(), 2 * chunk, w.front()));
        check(ferret_trainer_set_schedule(g.t, events.data(), events.size(), chunk));
        check(ferret_trainer_execute(g.t, 0));  // warm-up (graph build)
        check(ferret_trainer_set_profiling(g.t, 1));
        check(ferret_trainer_execute(g.t, 1));
        std::vector<double> f(static_cast<size_t>(L)), b(f), u(f);
        check(ferret_trainer_profile_stages(g.t, f.data(), b.data(), u.data(), L));
        for (int32_t i = 0; i < L; ++i) {
            const size_t k = static_cast<size_t>(i);
            layers_out[i] = {std::max(f[k], 1e-3) * 1e-6, std::max(b[k] + u[k], 1e-3) * 1e-6, syn[k].w, syn[k].a};
        }
    });
}

ferret_status ferret_plan_b200(const uint64_t* widths, int32_t n_widths, const ferret_layer_profile* layers, double t_d,
                               const ferret_stream_spec* spec, uint64_t budget_bytes, int32_t max_stages,
                               const ferret_b200_cost* cost, size_t n_items, ferret_schedule** out,
                               ferret_b200_plan_report* report) {
    return guarded([&] {
        validate_cost(cost);
        if (!widths || n_widths < 2 || !spec || !out) fail(FERRET_E_INVALID_ARG, "plan_b200: bad arguments");
        const int32_t L = n_widths - 1;
        for (int32_t i = 0; i < L; ++i)
            if (layers[i].w != widths[i] * widths[i + 1] + widths[i + 1] || layers[i].a != widths[i + 1])
                fail(FERRET_E_INVALID_ARG, "plan_b200: profile counts differ from the widths (pass count units)");
        const ferret::ModelProfile costed = byte_profile(to_profile(layers, L), *cost);
        const size_t chunk_units = cost->chunk_units ? cost->chunk_units : n_items;
        auto s = std::make_unique<ferret_schedule>();
        s->spec = {spec->t_d, spec->decay_c, spec->value, spec->horizon};

        // plan-independent bytes: a one-stage probe of the same net and options
        uint64_t fixed = 0;
        {
            const std::vector<uint64_t> one{0, static_cast<uint64_t>(L)};
            const ferret::StageStats st = ferret::stage_stats(costed, ferret::PartitionScheme{one});
            const ferret::PipelineConfig cfg = ferret::default_config(st, t_d, 0);
            const ferret::SimTrace tr = ferret::simulate(st, cfg, s->spec, std::min<size_t>(n_items, 4));
            const ferret_footprint f = trainer_footprint(widths, n_widths, one, *cost, to_events(tr), chunk_units);
            fixed = f.comp_state + f.other;
        }
        ferret::PlanFilter filt;
        filt.max_stages = max_stages > 0 ? static_cast<std::size_t>(max_stages) : 0;
        const bool unconstrained = budget_bytes == 0;
        if (!unconstrained && budget_bytes <= fixed)
            fail(FERRET_E_BOUND, "plan_b200: the budget does not cover the plan-independent bytes (" +
                                     std::to_string(fixed) + ")");
        uint64_t planner_budget = unconstrained ? (UINT64_MAX >> 2) : budget_bytes - fixed;
        ferret_b200_plan_report rep{};
        rep.budget_bytes = budget_bytes;
        rep.fixed_bytes = fixed;
        for (int pass = 1;; ++pass) {
            ferret::PlanResult pr = ferret::plan_within(costed, t_d, s->spec, planner_budget, filt);
            const ferret::StageStats st = ferret::stage_stats(costed, pr.partition);
            ferret::SimTrace tr = ferret::simulate(st, pr.config, s->spec, n_items);
            const ferret_footprint f =
                trainer_footprint(widths, n_widths, pr.partition.bounds, *cost, to_events(tr), chunk_units);
            rep.planner_budget = planner_budget;
            rep.planner_bytes = pr.memory;
            rep.predicted_bytes = fixed + pr.memory;
            rep.trainer_bytes = f.total;
            rep.passes = pass;
            rep.stages = static_cast<int32_t>(pr.partition.stages());
            rep.fits = !pr.infeasible && (unconstrained || f.total <= budget_bytes);
            const bool last = rep.fits || pass >= 12 || pr.infeasible;
            if (last) {
                s->plan = std::move(pr);
                s->trace = std::move(tr);
                break;
            }
            // tighten in proportion to the overshoot of the plan-dependent bytes
            const double scale = static_cast<double>(budget_bytes - fixed) / static_cast<double>(f.total - fixed);
            const uint64_t next = static_cast<uint64_t>(
                std::floor(static_cast<double>(std::min<uint64_t>(planner_budget, pr.memory)) * scale * 0.99));
            if (next == 0 || next >= planner_budget) {
                s->plan = std::move(pr);
                s->trace = std::move(tr);
                break;
            }
            planner_budget = next;
        }
        if (!rep.fits) s->plan.infeasible = true;
        if (report) *report = rep;
        *out = s.release();
    });
}

} // extern "C"
