// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into, loaded by, or called
// from the product path (paper_2503_12053_b200/). Only tests/, the smoke()
// check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
// legs load it, and only as the checker or the timed CPU reference.
//
// Built by oracle/Makefile from the REFERENCE'S OWN HEADERS where they lie
// (/root/reference/proj/include/ferret/*.hpp, -I on the command line; nothing
// is copied into this repo) into oracle/_ref/libferret_oracle.so. Everything
// below calls the reference implementation directly (make_dense_net,
// synth_drift_stream, profile_from_net, plan, default_config, stage_stats,
// simulate, write_plan, write_trace, compensate_*, forward_backward,
// apply_sgd, ReplayBuffer, StageVersions, RunningNormalizer, predict_class)
// except one class:
//
//   RestatedTrainer — a restatement of PipelineTrainer (learner.hpp:330-520)
//   that keys in-flight state by item instead of (worker, item). As shipped,
//   arrivals are logged with worker -1 (sim.hpp:234) and looked up with the
//   real worker (learner.hpp:408 vs 413/436/483), so the reference trainer
//   never trains. The restatement keeps every other step of
//   the reference in the same order: log order, hold at forward, release at
//   update, per-stage Compensator per pending gradient, mean then SGD, replay
//   after each stage-0 update pushing every stage. It also generalises the
//   pipeline unit to a micro-batch of B stream samples (mean reduction as in
//   net.hpp:162); at B = 1 every operation is the reference's exactly.
//   ferret_oracle_train(..., as_shipped=1) runs the reference's own
//   ferret::train_pipeline unchanged instead.
//
// Parity status: the host tiers are the reference itself; the trainer
// restatement is pinned by (a) bit-for-bit equality (log and parameters, every
// policy, with and without replay, micro-batch 1) with the reference's own
// train_pipeline built from learner.hpp with only the in-flight key patched
// (keyed_ref.cpp; tests/test_abi_and_oracle.py::
// test_restatement_equals_key_patched_reference), (b) equality with the
// as-shipped reference where it trains at all (predictions before the first
// update; tests/test_abi_and_oracle.py), (c) the SPEC worked examples
// (tests/cpp/host_kats.cpp -> tests/golden/host_kats.txt, tests/test_host_parity.py),
// and (d) the replay-index cross-check below (restated index reservoir vs the
// reference ReplayBuffer's returned sample, asserted on every draw).
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "ferret/analytics.hpp"
#include "ferret/compensate.hpp"
#include "ferret/learner.hpp"
#include "ferret/metrics.hpp"
#include "ferret/net.hpp"
#include "ferret/planner.hpp"
#include "ferret/profile.hpp"
#include "ferret/sim.hpp"
#include "ferret/stream.hpp"
#include "ferret/types.hpp"

#define ORACLE_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// layout mirrors of the product's C structs (ferret_b200.h); kept in sync by
// tests/test_abi_and_oracle.py, which checks their sizes against ctypes.
struct OEvent {
    double time;
    int32_t kind, worker, stage, staleness;
    int64_t item, version;
};
struct ORecord {
    int64_t item;
    int32_t outcome, pad;
    uint64_t predicted, label;
};
struct OProfile {
    double t_f, t_b;
    uint64_t w, a;
};
struct OOpts {
    int32_t policy;
    double lr, eta_lambda, lambda0, alpha, nu;
    int32_t replay;
    uint64_t replay_seed, replay_capacity;
    int32_t precision, micro_batch, device, as_shipped;
};
struct ONet {
    int32_t n_layers;
    const uint64_t* in;
    const uint64_t* out;
    const int32_t* act;
    const double* params;
};

ferret::DenseNet to_net(const ONet& d) {
    ferret::DenseNet net;
    size_t at = 0;
    for (int32_t l = 0; l < d.n_layers; ++l) {
        ferret::DenseLayer L;
        L.in = d.in[l];
        L.out = d.out[l];
        L.act = static_cast<ferret::Activation>(d.act[l]);
        L.W.assign(d.params + at, d.params + at + L.in * L.out);
        at += L.in * L.out;
        L.b.assign(d.params + at, d.params + at + L.out);
        at += L.out;
        net.layers.push_back(std::move(L));
    }
    return net;
}

// Restated ferret::Compensator (learner.hpp:83-127) with its state visible.
struct OracleCompensator {
    ferret::CompensationPolicy policy;
    ferret::CompensatorState state;
    ferret::ParamVec fixed_lambda;
    ferret::ParamVec mean_gap;

    OracleCompensator(ferret::CompensationPolicy p, size_t n, double lambda0, double eta, double alpha, double nu)
        : policy(p) {
        if (p == ferret::CompensationPolicy::iter_fisher)
            state = ferret::CompensatorState::make(n, lambda0, eta, alpha, nu);
        else if (p == ferret::CompensationPolicy::fisher)
            fixed_lambda.assign(n, lambda0);
        else if (p == ferret::CompensationPolicy::gap)
            mean_gap.assign(n, 0.0);
    }

    ferret::ParamVec apply(const ferret::ParamVec& g, const std::vector<ferret::ParamVec>& chain) {
        const int tau = static_cast<int>(chain.size()) - 1;
        switch (policy) {
            case ferret::CompensationPolicy::none: return g;
            case ferret::CompensationPolicy::step: return ferret::compensate_step_aware(g, tau);
            case ferret::CompensationPolicy::gap: {
                const auto& now = chain.back();
                const auto& read = chain.front();
                ferret::ParamVec out = ferret::compensate_gap_aware(g, now, read, mean_gap);
                for (size_t i = 0; i < mean_gap.size(); ++i)
                    mean_gap[i] = 0.99 * mean_gap[i] + 0.01 * std::abs(now[i] - read[i]);
                return out;
            }
            case ferret::CompensationPolicy::fisher:
                return ferret::compensate_fisher(g, chain.back(), chain.front(), fixed_lambda);
            default: {
                auto [out, st] = ferret::compensate_iterative(g, chain, std::move(state));
                state = std::move(st);
                return out;
            }
        }
    }
};

// Index reservoir restated from ReplayBuffer (learner.hpp:56-80); runs beside
// the reference buffer so every sampled index is cross-checked.
struct IndexReservoir {
    size_t cap;
    ferret::Rng rng;
    uint64_t seen = 0;
    std::vector<int64_t> items;
    IndexReservoir(size_t c, uint64_t seed) : cap(c), rng(seed ^ 0xbf58476d1ce4e5b9ULL) {}
    void add(int64_t id) {
        ++seen;
        if (items.size() < cap) {
            items.push_back(id);
        } else {
            const uint64_t at = rng.below(seen);
            if (at < cap) items[static_cast<size_t>(at)] = id;
        }
    }
    int64_t sample() { return items[static_cast<size_t>(rng.below(items.size()))]; }
};

class RestatedTrainer {
  public:
    RestatedTrainer(ferret::DenseNet net, const ferret::PartitionScheme& scheme, const OOpts& o)
        : net_(std::move(net)),
          spans_(ferret::detail::stage_spans(scheme)),
          opt_(o),
          B_(o.micro_batch),
          norm_(net_.n_inputs()),
          buffer_(o.replay_capacity, o.replay_seed),
          index_(o.replay_capacity, o.replay_seed) {
        net_.validate();
        scheme.validate(net_.layers.size());
        if (B_ < 1) throw std::invalid_argument("micro_batch must be >= 1");
        versions_.resize(spans_.size());
        for (size_t j = 0; j < spans_.size(); ++j) {
            versions_[j].init(ferret::detail::stage_params(net_, spans_[j]));
            comps_.emplace_back(static_cast<ferret::CompensationPolicy>(o.policy),
                                ferret::detail::stage_params(net_, spans_[j]).size(), o.lambda0, o.eta_lambda,
                                o.alpha, o.nu);
        }
    }

    std::vector<ferret::StepRecord> run(const std::vector<ferret::SimEvent>& events, const ferret::DataStream& stream) {
        std::vector<ferret::StepRecord> log(stream.items.size());
        std::unordered_set<int64_t> dropped;
        for (const auto& e : events)
            if (e.kind == ferret::EventKind::drop) dropped.insert(e.item);
        for (const auto& e : events) {
            switch (e.kind) {
                case ferret::EventKind::arrival: on_arrival(e, stream, dropped, log); break;
                case ferret::EventKind::forward: on_forward(e); break;
                case ferret::EventKind::backward: on_backward(e); break;
                case ferret::EventKind::update: on_update(e); break;
                default: break;
            }
        }
        return log;
    }

    ferret::DenseNet net_;
    std::vector<ferret::detail::StageSpan> spans_;
    OOpts opt_;
    int B_;
    ferret::RunningNormalizer norm_;
    ferret::ReplayBuffer buffer_;
    IndexReservoir index_;
    std::vector<int64_t> replay_ids;
    std::vector<ferret::detail::StageVersions> versions_;
    std::vector<OracleCompensator> comps_;
    std::vector<std::vector<double>> xs_;  // normalised features per stream sample (for the replay cross-check)

  private:
    struct InFlight {
        std::vector<std::vector<double>> input;                 // per sample
        std::vector<size_t> label;                              // per sample
        std::vector<int64_t> read_version;                      // per stage
        std::vector<std::vector<std::vector<std::vector<double>>>> acts;  // stage -> sample -> layer -> out
        std::vector<std::vector<double>> delta;                 // per sample
    };
    struct PendingGrad {
        ferret::ParamVec grad;
        int64_t read_version;
    };
    std::map<int64_t, InFlight> inflight_;                      // keyed by item (the fix)
    std::map<std::pair<int, int>, std::vector<PendingGrad>> acc_;

    void on_arrival(const ferret::SimEvent& e, const ferret::DataStream& stream,
                    const std::unordered_set<int64_t>& dropped, std::vector<ferret::StepRecord>& log) {
        const bool drop = dropped.count(e.item) != 0;
        InFlight fl;
        for (int b = 0; b < B_; ++b) {
            const size_t s = static_cast<size_t>(e.item) * static_cast<size_t>(B_) + static_cast<size_t>(b);
            const auto& item = stream.items[s];
            norm_.observe(item.features);
            if (drop) {
                log[s] = {static_cast<int64_t>(s), ferret::StepOutcome::dropped, 0, item.label};
                continue;
            }
            fl.input.push_back(norm_.apply(item.features));
            fl.label.push_back(item.label);
        }
        if (drop) return;
        for (int b = 0; b < B_; ++b) {
            const size_t s = static_cast<size_t>(e.item) * static_cast<size_t>(B_) + static_cast<size_t>(b);
            const size_t pred = ferret::predict_class(net_, fl.input[static_cast<size_t>(b)]);
            const size_t label = fl.label[static_cast<size_t>(b)];
            log[s] = {static_cast<int64_t>(s), pred == label ? ferret::StepOutcome::correct : ferret::StepOutcome::wrong,
                      pred, label};
        }
        fl.read_version.assign(spans_.size(), -1);
        fl.acts.resize(spans_.size());
        fl.delta.resize(static_cast<size_t>(B_));
        if (opt_.replay) {
            for (int b = 0; b < B_; ++b) {
                const int64_t s = e.item * B_ + b;
                buffer_.add({fl.input[static_cast<size_t>(b)], fl.label[static_cast<size_t>(b)]});
                index_.add(s);
                if (xs_.size() <= static_cast<size_t>(s)) xs_.resize(static_cast<size_t>(s) + 1);
                xs_[static_cast<size_t>(s)] = fl.input[static_cast<size_t>(b)];
            }
        }
        inflight_[e.item] = std::move(fl);
    }

    void on_forward(const ferret::SimEvent& e) {
        auto it = inflight_.find(e.item);
        if (it == inflight_.end()) return;
        InFlight& fl = it->second;
        const size_t j = static_cast<size_t>(e.stage);
        const int64_t v = versions_[j].current();
        fl.read_version[j] = v;
        versions_[j].hold(v);
        ferret::DenseNet stage_net = net_;
        ferret::detail::set_stage_params(stage_net, spans_[j], versions_[j].at(v));
        fl.acts[j].assign(static_cast<size_t>(B_), {});
        for (int b = 0; b < B_; ++b) {
            const std::vector<double>* cur =
                j == 0 ? &fl.input[static_cast<size_t>(b)] : &fl.acts[j - 1][static_cast<size_t>(b)].back();
            auto& acts = fl.acts[j][static_cast<size_t>(b)];
            for (size_t l = spans_[j].lo; l < spans_[j].hi; ++l) {
                std::vector<double> z;
                ferret::detail::affine_forward(stage_net.layers[l], *cur, z);
                ferret::detail::apply_activation(stage_net.layers[l].act, z);
                acts.push_back(std::move(z));
                cur = &acts.back();
            }
        }
    }

    void on_backward(const ferret::SimEvent& e) {
        auto it = inflight_.find(e.item);
        if (it == inflight_.end()) return;
        InFlight& fl = it->second;
        const size_t j = static_cast<size_t>(e.stage);
        ferret::DenseNet stage_net = net_;
        ferret::detail::set_stage_params(stage_net, spans_[j], versions_[j].at(fl.read_version[j]));
        const double inv_b = 1.0 / static_cast<double>(B_);
        // per-layer gradients of this stage, summed over the micro-batch
        std::vector<ferret::ParamVec> layer_grads(spans_[j].hi - spans_[j].lo);
        for (size_t l = spans_[j].lo; l < spans_[j].hi; ++l) {
            const auto& layer = stage_net.layers[l];
            layer_grads[l - spans_[j].lo].assign(layer.W.size() + layer.b.size(), 0.0);
        }
        for (int b = 0; b < B_; ++b) {
            const size_t bb = static_cast<size_t>(b);
            std::vector<double> delta;
            if (j + 1 == spans_.size()) {
                delta = ferret::detail::softmax(fl.acts[j][bb].back());
                delta[fl.label[bb]] -= 1.0;
                for (auto& v : delta) v *= inv_b;
            } else {
                delta = fl.delta[bb];
            }
            for (size_t l = spans_[j].hi; l-- > spans_[j].lo;) {
                const auto& layer = stage_net.layers[l];
                const size_t local = l - spans_[j].lo;
                const std::vector<double>& input =
                    local == 0 ? (j == 0 ? fl.input[bb] : fl.acts[j - 1][bb].back()) : fl.acts[j][bb][local - 1];
                if (layer.act == ferret::Activation::relu)
                    for (size_t r = 0; r < layer.out; ++r)
                        if (fl.acts[j][bb][local][r] <= 0.0) delta[r] = 0.0;
                auto& lg = layer_grads[local];
                for (size_t r = 0; r < layer.out; ++r) {
                    const double d = delta[r];
                    for (size_t c = 0; c < layer.in; ++c) lg[r * layer.in + c] += d * input[c];
                    lg[layer.W.size() + r] += d;
                }
                std::vector<double> prev(layer.in, 0.0);
                for (size_t r = 0; r < layer.out; ++r) {
                    const double d = delta[r];
                    const double* row = layer.W.data() + r * layer.in;
                    for (size_t c = 0; c < layer.in; ++c) prev[c] += d * row[c];
                }
                delta = std::move(prev);
            }
            fl.delta[bb] = std::move(delta);
        }
        ferret::ParamVec grad;
        for (const auto& lg : layer_grads) grad.insert(grad.end(), lg.begin(), lg.end());
        acc_[{e.worker, e.stage}].push_back({std::move(grad), fl.read_version[j]});
    }

    void on_update(const ferret::SimEvent& e) {
        const size_t j = static_cast<size_t>(e.stage);
        auto it = acc_.find({e.worker, e.stage});
        if (it == acc_.end() || it->second.empty()) return;
        ferret::ParamVec mean;
        for (const auto& pg : it->second) {
            const auto chain = versions_[j].chain_from(pg.read_version);
            ferret::ParamVec g = comps_[j].apply(pg.grad, chain);
            if (mean.empty()) mean.assign(g.size(), 0.0);
            for (size_t i = 0; i < g.size(); ++i) mean[i] += g[i];
        }
        const double inv = 1.0 / static_cast<double>(it->second.size());
        ferret::ParamVec params = versions_[j].at(versions_[j].current());
        for (size_t i = 0; i < params.size(); ++i) params[i] -= opt_.lr * inv * mean[i];
        ferret::detail::set_stage_params(net_, spans_[j], params);
        versions_[j].push(std::move(params));
        for (const auto& pg : it->second) versions_[j].release(pg.read_version);
        it->second.clear();
        if (j == 0 && opt_.replay && !buffer_.empty()) replay_step();
    }

    void replay_step() {
        ferret::Batch batch;
        for (int b = 0; b < B_; ++b) {
            const ferret::Sample& s = buffer_.sample();
            const int64_t id = index_.sample();
            if (xs_[static_cast<size_t>(id)] != s.x)
                throw std::logic_error("oracle: restated replay index disagrees with the reference ReplayBuffer");
            replay_ids.push_back(id);
            batch.push_back(s);
        }
        auto [loss, grads] = ferret::forward_backward(net_, batch);
        (void)loss;
        ferret::apply_sgd(net_, grads, opt_.lr);
        for (size_t j = 0; j < spans_.size(); ++j) versions_[j].push(ferret::detail::stage_params(net_, spans_[j]));
    }
};

ferret::DataStream to_stream(const double* features, const uint64_t* labels, size_t n, size_t f) {
    ferret::DataStream ds;
    ds.n_features = f;
    for (size_t i = 0; i < n; ++i) {
        ferret::StreamItem it;
        it.index = static_cast<int64_t>(i);
        it.features.assign(features + i * f, features + (i + 1) * f);
        it.label = static_cast<size_t>(labels[i]);
        ds.n_classes = std::max(ds.n_classes, it.label + 1);
        ds.items.push_back(std::move(it));
    }
    return ds;
}

std::vector<ferret::SimEvent> to_events(const OEvent* ev, size_t n) {
    std::vector<ferret::SimEvent> out(n);
    for (size_t i = 0; i < n; ++i)
        out[i] = {ev[i].time, static_cast<ferret::EventKind>(ev[i].kind), ev[i].worker, ev[i].stage, ev[i].item,
                  ev[i].version, ev[i].staleness};
    return out;
}

void copy_records(const std::vector<ferret::StepRecord>& log, ORecord* out) {
    for (size_t i = 0; i < log.size(); ++i)
        out[i] = {log[i].item, static_cast<int32_t>(log[i].outcome), 0, static_cast<uint64_t>(log[i].predicted),
                  static_cast<uint64_t>(log[i].label)};
}

size_t put_text(const std::string& s, char* buf, size_t cap) {
    if (buf && cap) {
        const size_t n = std::min(s.size(), cap - 1);
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return s.size() + 1;
}

struct OSchedule {
    ferret::PlanResult plan;
    ferret::StreamSpec spec;
    ferret::SimTrace trace;
};

} // namespace

ORACLE_API const char* ferret_oracle_last_error() { return g_err.c_str(); }

ORACLE_API int ferret_oracle_make_dense_net(const uint64_t* widths, int32_t n, uint64_t seed, int32_t act, double* out) {
    return guard([&] {
        const auto net = ferret::make_dense_net(std::vector<size_t>(widths, widths + n), seed,
                                                static_cast<ferret::Activation>(act));
        const auto flat = ferret::flatten(net);
        std::memcpy(out, flat.data(), flat.size() * sizeof(double));
    });
}

ORACLE_API int ferret_oracle_profile_from_widths(const uint64_t* widths, int32_t n, double spp, OProfile* out) {
    return guard([&] {
        const auto net = ferret::make_dense_net(std::vector<size_t>(widths, widths + n), 0);
        const auto p = ferret::profile_from_net(net, spp);
        for (size_t i = 0; i < p.layers.size(); ++i) out[i] = {p.layers[i].t_f, p.layers[i].t_b, p.layers[i].w, p.layers[i].a};
    });
}

ORACLE_API int ferret_oracle_synth_drift_stream(size_t n, size_t f, size_t c, int32_t drift, uint64_t seed, double rot,
                                                double noise, double* features, uint64_t* labels) {
    return guard([&] {
        const auto ds = ferret::synth_drift_stream(n, f, c, static_cast<ferret::DriftKind>(drift), seed, rot, noise);
        for (size_t i = 0; i < n; ++i) {
            std::memcpy(features + i * f, ds.items[i].features.data(), f * sizeof(double));
            labels[i] = ds.items[i].label;
        }
    });
}

// plan (planner.hpp:192) or forced bounds + default_config, then simulate.
ORACLE_API int ferret_oracle_schedule(const OProfile* layers, int32_t n_layers, double t_d, const double* spec4,
                                      uint64_t budget, const uint64_t* forced, int32_t n_forced, int32_t recompute,
                                      size_t n_items, void** handle) {
    return guard([&] {
        auto* s = new OSchedule;
        s->spec = {spec4[0], spec4[1], spec4[2], spec4[3]};
        ferret::ModelProfile prof;
        for (int32_t i = 0; i < n_layers; ++i) prof.layers.push_back({layers[i].t_f, layers[i].t_b, layers[i].w, layers[i].a});
        if (forced) {
            s->plan.partition.bounds.assign(forced, forced + n_forced);
            const auto st = ferret::stage_stats(prof, s->plan.partition);
            s->plan.config = ferret::default_config(st, t_d, recompute);
            s->plan.rate = ferret::adaptation_rate(st, s->plan.config, s->spec);
            s->plan.memory = ferret::memory_footprint(st, s->plan.config);
        } else {
            s->plan = ferret::plan(prof, t_d, s->spec, budget);
        }
        const auto st = ferret::stage_stats(prof, s->plan.partition);
        s->trace = ferret::simulate(st, s->plan.config, s->spec, n_items);
        *handle = s;
    });
}

ORACLE_API size_t ferret_oracle_schedule_plan_text(void* h, char* buf, size_t cap) {
    std::ostringstream os;
    ferret::write_plan(os, static_cast<OSchedule*>(h)->plan);
    return put_text(os.str(), buf, cap);
}

ORACLE_API size_t ferret_oracle_schedule_trace_text(void* h, char* buf, size_t cap) {
    auto* s = static_cast<OSchedule*>(h);
    std::ostringstream os;
    ferret::write_trace(os, s->trace, s->spec);
    return put_text(os.str(), buf, cap);
}

ORACLE_API size_t ferret_oracle_schedule_events(void* h, OEvent* out, size_t cap) {
    auto* s = static_cast<OSchedule*>(h);
    const auto& ev = s->trace.events;
    for (size_t i = 0; i < ev.size() && i < cap; ++i)
        out[i] = {ev[i].time, static_cast<int32_t>(ev[i].kind), ev[i].worker, ev[i].stage, ev[i].staleness, ev[i].item,
                  ev[i].version};
    return ev.size();
}

ORACLE_API int32_t ferret_oracle_schedule_bounds(void* h, uint64_t* out, int32_t cap) {
    const auto& b = static_cast<OSchedule*>(h)->plan.partition.bounds;
    for (int32_t i = 0; i < cap && i < static_cast<int32_t>(b.size()); ++i) out[i] = b[static_cast<size_t>(i)];
    return static_cast<int32_t>(b.size());
}

ORACLE_API void ferret_oracle_schedule_destroy(void* h) { delete static_cast<OSchedule*>(h); }

// The pipelined trainer on the CPU. Outputs (any may be NULL):
//   log_out[n_items], params_out[n_params] (flatten order),
//   lambda/v_r/v_a/gap_out[n_params] (stage states concatenated in flatten order),
//   norm_count/mean/m2, replay_ids (cap entries) + n_replay.
ORACLE_API int ferret_oracle_train(const ONet* net, const uint64_t* bounds, int32_t n_bounds, const OOpts* opts,
                                   const OEvent* events, size_t n_events, const double* features,
                                   const uint64_t* labels, size_t n_items, size_t n_features, ORecord* log_out,
                                   double* params_out, double* lambda_out, double* v_r_out, double* v_a_out,
                                   double* gap_out, uint64_t* norm_count, double* norm_mean, double* norm_m2,
                                   int64_t* replay_ids, size_t replay_cap, size_t* n_replay) {
    return guard([&] {
        ferret::DenseNet dn = to_net(*net);
        ferret::PartitionScheme scheme;
        scheme.bounds.assign(bounds, bounds + n_bounds);
        const ferret::DataStream ds = to_stream(features, labels, n_items, n_features);
        const auto ev = to_events(events, n_events);
        if (opts->as_shipped) {
            if (opts->micro_batch != 1) throw std::invalid_argument("as_shipped requires micro_batch 1");
            ferret::SimTrace tr;
            tr.events = ev;
            ferret::PipelineTrainOptions po;
            po.policy = static_cast<ferret::CompensationPolicy>(opts->policy);
            po.lr = opts->lr;
            po.eta_lambda = opts->eta_lambda;
            po.replay = opts->replay != 0;
            po.replay_seed = opts->replay_seed;
            const ferret::TrainOutcome out = ferret::train_pipeline(std::move(dn), scheme, tr, ds, po);
            if (log_out) copy_records(out.log, log_out);
            if (params_out) {
                const auto flat = ferret::flatten(out.net);
                std::memcpy(params_out, flat.data(), flat.size() * sizeof(double));
            }
            if (n_replay) *n_replay = 0;
            return;
        }
        RestatedTrainer tr(std::move(dn), scheme, *opts);
        const auto log = tr.run(ev, ds);
        if (log_out) copy_records(log, log_out);
        if (params_out) {
            const auto flat = ferret::flatten(tr.net_);
            std::memcpy(params_out, flat.data(), flat.size() * sizeof(double));
        }
        size_t at = 0;
        for (size_t j = 0; j < tr.spans_.size(); ++j) {
            const auto& c = tr.comps_[j];
            const size_t n = ferret::detail::stage_params(tr.net_, tr.spans_[j]).size();
            auto put = [&](double* dst, const ferret::ParamVec& src, double fill) {
                if (!dst) return;
                for (size_t i = 0; i < n; ++i) dst[at + i] = src.empty() ? fill : src[i];
            };
            if (c.policy == ferret::CompensationPolicy::iter_fisher) put(lambda_out, c.state.lambda, 0.0);
            else put(lambda_out, c.fixed_lambda, 0.0);
            put(v_r_out, c.state.v_r, 0.0);
            put(v_a_out, c.state.v_a, 0.0);
            put(gap_out, c.mean_gap, 0.0);
            at += n;
        }
        if (norm_count || norm_mean || norm_m2) {
            // RunningNormalizer has no accessors: recover mean / m2 by probing apply()
            // is lossy, so re-run observe() over the arrivals the trainer saw.
            ferret::RunningNormalizer probe(n_features);
            uint64_t cnt = 0;
            std::vector<double> mean(n_features, 0.0), m2(n_features, 0.0);
            for (const auto& e : ev) {
                if (e.kind != ferret::EventKind::arrival) continue;
                for (int b = 0; b < opts->micro_batch; ++b) {
                    const auto& x = ds.items[static_cast<size_t>(e.item * opts->micro_batch + b)].features;
                    ++cnt;
                    for (size_t f = 0; f < n_features; ++f) {  // stream.hpp:312-319
                        const double d = x[f] - mean[f];
                        mean[f] += d / static_cast<double>(cnt);
                        m2[f] += d * (x[f] - mean[f]);
                    }
                }
            }
            if (norm_count) *norm_count = cnt;
            if (norm_mean) std::memcpy(norm_mean, mean.data(), n_features * sizeof(double));
            if (norm_m2) std::memcpy(norm_m2, m2.data(), n_features * sizeof(double));
        }
        if (n_replay) *n_replay = tr.replay_ids.size();
        if (replay_ids)
            for (size_t i = 0; i < tr.replay_ids.size() && i < replay_cap; ++i) replay_ids[i] = tr.replay_ids[i];
    });
}

// Reference compensators in fp64 (compensate.hpp), for the device unit tests.
// policy: 0 none 1 step 2 gap(apply semantics, mean_gap updated) 3 fisher(lambda array) 4 iterative
ORACLE_API int ferret_oracle_compensate(int32_t policy, const double* g, const double* const* chain, int32_t chain_len,
                                        double* lambda, double* v_r, double* v_a, double* mean_gap, size_t n,
                                        double alpha, double eta, double nu, double* out) {
    return guard([&] {
        const ferret::ParamVec gv(g, g + n);
        std::vector<ferret::ParamVec> ch;
        for (int32_t i = 0; i < chain_len; ++i) ch.emplace_back(chain[i], chain[i] + n);
        ferret::ParamVec res;
        if (policy == 0) {
            res = gv;
        } else if (policy == 1) {
            res = ferret::compensate_step_aware(gv, chain_len - 1);
        } else if (policy == 2) {
            ferret::ParamVec mg(mean_gap, mean_gap + n);
            res = ferret::compensate_gap_aware(gv, ch.back(), ch.front(), mg);
            for (size_t i = 0; i < n; ++i) mean_gap[i] = 0.99 * mg[i] + 0.01 * std::abs(ch.back()[i] - ch.front()[i]);
        } else if (policy == 3) {
            res = ferret::compensate_fisher(gv, ch.back(), ch.front(), ferret::ParamVec(lambda, lambda + n));
        } else {
            ferret::CompensatorState st;
            st.lambda.assign(lambda, lambda + n);
            if (eta > 0.0) {
                st.v_r.assign(v_r, v_r + n);
                st.v_a.assign(v_a, v_a + n);
            }
            st.alpha = alpha;
            st.eta_lambda = eta;
            st.nu = nu;
            auto [o, s2] = ferret::compensate_iterative(gv, ch, std::move(st));
            res = std::move(o);
            std::memcpy(lambda, s2.lambda.data(), n * sizeof(double));
            if (eta > 0.0) {
                std::memcpy(v_r, s2.v_r.data(), n * sizeof(double));
                std::memcpy(v_a, s2.v_a.data(), n * sizeof(double));
            }
        }
        std::memcpy(out, res.data(), n * sizeof(double));
    });
}

// RunningNormalizer::observe+apply over a stream (stream.hpp:307-334), for the
// device normalizer bit-exactness test.
ORACLE_API int ferret_oracle_normalize(const double* features, size_t n, size_t f, double* out) {
    return guard([&] {
        ferret::RunningNormalizer norm(f);
        for (size_t i = 0; i < n; ++i) {
            const std::vector<double> x(features + i * f, features + (i + 1) * f);
            norm.observe(x);
            const auto z = norm.apply(x);
            std::memcpy(out + i * f, z.data(), f * sizeof(double));
        }
    });
}

// ---------------------------------------------------------------------------
// Sequential learners, the reference's own code unchanged (learner.hpp:132-225):
// StaleHarness::ocl_step per item, and train_sequential with apply_skip_policy.
// ---------------------------------------------------------------------------
ORACLE_API int ferret_oracle_harness(const ONet* net, int32_t policy, uint64_t ring_depth, double lr, double eta_lambda,
                                     const double* features, const uint64_t* labels, const int32_t* taus, size_t n,
                                     size_t f, uint64_t* preds, double* params_out) {
    return guard([&] {
        ferret::StaleHarness h(to_net(*net), static_cast<ferret::CompensationPolicy>(policy), ring_depth, lr, eta_lambda);
        const ferret::DataStream ds = to_stream(features, labels, n, f);
        for (size_t i = 0; i < n; ++i) preds[i] = h.ocl_step(ds.items[i], taus[i]);
        const ferret::ParamVec p = ferret::flatten(h.net());
        std::copy(p.begin(), p.end(), params_out);
    });
}

ORACLE_API int ferret_oracle_train_sequential(const ONet* net, const double* features, const uint64_t* labels, size_t n,
                                              size_t f, double t_d, int32_t skip_kind, uint64_t window, uint64_t keep,
                                              uint64_t skip_seed, double processing_time, double lr, int32_t replay,
                                              uint64_t replay_seed, ORecord* log_out, double* params_out,
                                              int64_t* kept_out, size_t* n_kept) {
    return guard([&] {
        ferret::SkipPolicy sp;
        sp.kind = static_cast<ferret::SkipKind>(skip_kind);
        sp.window = window;
        sp.keep = keep;
        sp.seed = skip_seed;
        const ferret::DataStream ds = to_stream(features, labels, n, f);
        const ferret::TrainOutcome out =
            ferret::train_sequential(to_net(*net), ds, t_d, sp, processing_time, lr, replay != 0, replay_seed);
        copy_records(out.log, log_out);
        const ferret::ParamVec p = ferret::flatten(out.net);
        std::copy(p.begin(), p.end(), params_out);
        const ferret::FilteredStream fs = ferret::apply_skip_policy(n, t_d, sp, processing_time);
        for (size_t i = 0; i < fs.kept.size(); ++i) kept_out[i] = fs.kept[i].index;
        *n_kept = fs.kept.size();
    });
}

// load_csv_stream of the reference (stream.hpp:144-186), gzip included.
ORACLE_API int ferret_oracle_csv(const char* path, const char* label_column, double* features, uint64_t* labels,
                                 size_t cap_rows, size_t* n, size_t* f, size_t* n_classes) {
    return guard([&] {
        const ferret::DataStream ds = ferret::load_csv_stream(path, label_column);
        *n = ds.items.size();
        *f = ds.n_features;
        *n_classes = ds.n_classes;
        if (cap_rows < ds.items.size()) return;
        for (size_t i = 0; i < ds.items.size(); ++i) {
            std::memcpy(features + i * ds.n_features, ds.items[i].features.data(), ds.n_features * sizeof(double));
            labels[i] = ds.items[i].label;
        }
    });
}

#include "conv_oracle.hpp"
