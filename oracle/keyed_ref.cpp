// ORACLE — TEST INFRASTRUCTURE ONLY (see ferret_oracle.cpp's header).
//
// The reference's own PipelineTrainer with ONLY its in-flight key patched, to pin the
// restatement (RestatedTrainer in ferret_oracle.cpp) bit for bit.
//
// oracle/Makefile generates _ref/keyed/ferret/learner.hpp from the reference's
// /root/reference/proj/include/ferret/learner.hpp with one sed expression that replaces
// the (worker, item) in-flight key by (0, item) at its four sites — learner.hpp:408
// (on_arrival insert), :413 (on_forward lookup), :436 (on_backward lookup) and :483
// (inflight_erase_when_done lookup). Nothing else of the header changes and the file
// exists only under _ref/ (git-ignored). This translation unit is compiled with
// -I_ref/keyed ahead of -I/root/reference/proj/include, so "ferret/learner.hpp" is the
// patched copy and every other header is the reference's, in place. It is a separate
// shared object so the patched PipelineTrainer never shares a program with the unpatched
// one (ferret_oracle.cpp includes the shipped header).
//
// ferret_keyed_train runs ferret::train_pipeline (learner.hpp:522-526) — the reference's
// trainer, arithmetic, Compensator, ReplayBuffer and RunningNormalizer unchanged — on a
// caller-supplied net, partition, event log and stream, and returns the StepRecord log and
// the final flattened parameters. tests/test_abi_and_oracle.py asserts that the
// restatement's log and parameters equal these bit for bit at micro-batch 1 (every
// policy, with and without replay).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ferret/learner.hpp"

#define KEYED_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

struct KEvent {  // == ferret_event / OEvent
    double time;
    int32_t kind, worker, stage, staleness;
    int64_t item, version;
};
struct KRecord {  // == ferret_step_record / ORecord
    int64_t item;
    int32_t outcome, pad;
    uint64_t predicted, label;
};

}  // namespace

KEYED_API const char* ferret_keyed_last_error() { return g_err.c_str(); }

// widths: n_layers + 1 entries; hidden layers relu, the last identity (make_dense_net's layout)
KEYED_API int ferret_keyed_train(const uint64_t* widths, int32_t n_widths, const double* params,
                                 const uint64_t* bounds, int32_t n_bounds, int32_t policy, double lr,
                                 double eta_lambda, int32_t replay, uint64_t replay_seed, const KEvent* events,
                                 size_t n_events, const double* features, const uint64_t* labels, size_t n_items,
                                 size_t n_features, KRecord* log_out, double* params_out) {
    try {
        ferret::DenseNet net;
        size_t at = 0;
        for (int32_t l = 0; l + 1 < n_widths; ++l) {
            ferret::DenseLayer L;
            L.in = widths[l];
            L.out = widths[l + 1];
            L.act = l + 2 == n_widths ? ferret::Activation::identity : ferret::Activation::relu;
            L.W.assign(params + at, params + at + L.in * L.out);
            at += L.in * L.out;
            L.b.assign(params + at, params + at + L.out);
            at += L.out;
            net.layers.push_back(std::move(L));
        }
        ferret::PartitionScheme scheme;
        scheme.bounds.assign(bounds, bounds + n_bounds);
        ferret::DataStream ds;
        ds.n_features = n_features;
        for (size_t i = 0; i < n_items; ++i) {
            ferret::StreamItem it;
            it.index = static_cast<int64_t>(i);
            it.features.assign(features + i * n_features, features + (i + 1) * n_features);
            it.label = static_cast<size_t>(labels[i]);
            ds.n_classes = std::max(ds.n_classes, it.label + 1);
            ds.items.push_back(std::move(it));
        }
        ferret::SimTrace tr;
        for (size_t i = 0; i < n_events; ++i)
            tr.events.push_back({events[i].time, static_cast<ferret::EventKind>(events[i].kind), events[i].worker,
                                 events[i].stage, events[i].item, events[i].version, events[i].staleness});
        ferret::PipelineTrainOptions po;
        po.policy = static_cast<ferret::CompensationPolicy>(policy);
        po.lr = lr;
        po.eta_lambda = eta_lambda;
        po.replay = replay != 0;
        po.replay_seed = replay_seed;
        const ferret::TrainOutcome out = ferret::train_pipeline(std::move(net), scheme, tr, ds, po);
        for (size_t i = 0; i < out.log.size() && log_out; ++i)
            log_out[i] = {out.log[i].item, static_cast<int32_t>(out.log[i].outcome), 0,
                          static_cast<uint64_t>(out.log[i].predicted), static_cast<uint64_t>(out.log[i].label)};
        if (params_out) {
            const auto flat = ferret::flatten(out.net);
            std::memcpy(params_out, flat.data(), flat.size() * sizeof(double));
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
