// ferret-b200 drop-in: the planner re-costed for B200 (north-star item 4).
//
// The reference plans with plan() (planner.hpp:180-215) on profile_from_net's synthetic
// times (net.hpp:263-274) and memory in count units (analytics.hpp:58-104). plan_b200()
// runs the same search (planner.hpp, byte-identical to the reference) on
//   * measure_b200_profile(): per-layer t_f / t_b measured on the device with the real
//     kernels (one layer per stage, a profiled chunk after a warm-up chunk);
//   * w / a in HBM bytes of the B200 trainer's layout (b200_byte_profile);
//   * partitions of at most max_stages stages (#GPUs: one stage per GPU at most),
// then prices the chosen plan exactly with the trainer's own dry-run footprint of the
// plan's event log (ferret_trainer_footprint, no device needed) and re-plans under a
// tightened budget until it fits. The result is the reference's PlanResult (memory in
// bytes) and SimTrace, ready for train_pipeline().
//
// C ABI: ferret_measure_profile / ferret_b200_byte_profile / ferret_plan_b200
// (include/ferret_b200.h, csrc/planner_b200.cpp).
#pragma once

#include <cstdint>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "ferret/b200_status.hpp"
#include "ferret/compensate.hpp"
#include "ferret/net.hpp"
#include "ferret/planner.hpp"
#include "ferret/sim.hpp"
#include "ferret/types.hpp"
#include "ferret_b200.h"

namespace ferret {

// What the B200 planner prices (ferret_b200_cost).
struct B200CostModel {
    int micro_batch = 1;                                  // stream samples per pipeline unit
    int precision = FERRET_PREC_FP32;                     // bf16: + a bf16 copy of every weight version
    CompensationPolicy policy = CompensationPolicy::iter_fisher;
    double eta_lambda = 1e-3;                             // iter_fisher: > 0 keeps v_r / v_a state
    bool replay = false;
    std::size_t replay_capacity = kReplayCapacityDefault;
    std::size_t chunk_units = 0;                          // units per compiled chunk (0: the trace's items)

    static constexpr std::size_t kReplayCapacityDefault = 5000;

    ferret_b200_cost c() const {
        ferret_b200_cost o{};
        ferret_b200_cost_default(&o);
        o.micro_batch = micro_batch;
        o.precision = precision;
        o.policy = static_cast<int32_t>(policy);
        o.eta_lambda = eta_lambda;
        o.replay = replay ? 1 : 0;
        o.replay_capacity = replay_capacity;
        o.chunk_units = chunk_units;
        return o;
    }
};

struct B200PlanReport {
    std::uint64_t budget_bytes = 0;     // the caller's HBM budget (0: unconstrained)
    std::uint64_t fixed_bytes = 0;      // plan-independent: compensator state, normalizer, staging
    std::uint64_t planner_budget = 0;   // what the reference search was given on the last pass
    std::uint64_t planner_bytes = 0;    // the reference memory model of the plan, in bytes
    std::uint64_t predicted_bytes = 0;  // fixed + planner
    std::uint64_t trainer_bytes = 0;    // exact: the trainer's footprint of the plan's event log
    int passes = 0;
    std::size_t stages = 0;
    bool fits = false;
};

struct B200Plan {
    PlanResult plan;  // the reference's plan record; plan.memory is in bytes
    SimTrace trace;   // simulate() of the plan over the requested items
    B200PlanReport report;
};

namespace detail {

inline std::vector<std::uint64_t> widths_of(const DenseNet& net) {
    std::vector<std::uint64_t> w;
    if (net.layers.empty()) throw ConfigError("net needs at least one layer");
    w.push_back(net.layers.front().in);
    for (const DenseLayer& l : net.layers) w.push_back(l.out);
    return w;
}

inline std::vector<ferret_layer_profile> c_profile(const ModelProfile& p) {
    std::vector<ferret_layer_profile> out;
    for (const LayerProfile& l : p.layers) out.push_back({l.t_f, l.t_b, l.w, l.a});
    return out;
}

inline ModelProfile from_c(const std::vector<ferret_layer_profile>& v) {
    ModelProfile p;
    for (const ferret_layer_profile& l : v) p.layers.push_back({l.t_f, l.t_b, l.w, l.a});
    return p;
}

inline std::string schedule_text(const ferret_schedule* s, std::size_t (*fn)(const ferret_schedule*, char*, std::size_t)) {
    const std::size_t n = fn(s, nullptr, 0);
    std::string buf(n, '\0');
    fn(s, buf.data(), n);
    buf.resize(n > 0 ? n - 1 : 0);
    return buf;
}

} // namespace detail

// profile_from_net (net.hpp:263-274) with measured device times.
inline ModelProfile measure_b200_profile(const DenseNet& net, const B200CostModel& cost, int device = 0,
                                         int units = 48) {
    const std::vector<std::uint64_t> w = detail::widths_of(net);
    std::vector<ferret_layer_profile> out(net.layers.size());
    const ferret_b200_cost c = cost.c();
    b200_check(ferret_measure_profile(w.data(), static_cast<int32_t>(w.size()), &c, units, device, out.data()));
    return detail::from_c(out);
}

// w -> bytes of one weight version of the layer, a -> stash bytes per in-flight unit.
inline ModelProfile b200_byte_profile(const ModelProfile& prof, const B200CostModel& cost) {
    std::vector<ferret_layer_profile> in = detail::c_profile(prof), out(in.size());
    const ferret_b200_cost c = cost.c();
    b200_check(ferret_b200_byte_profile(in.data(), static_cast<int32_t>(in.size()), &c, out.data()));
    return detail::from_c(out);
}

// plan() + simulate() re-costed for B200: `prof` in seconds and count units (as
// profile_from_net / measure_b200_profile give), budget in HBM bytes (0: unconstrained),
// max_stages = #GPUs (0: unlimited), n_items = units of the simulated trace.
inline B200Plan plan_b200(const DenseNet& net, const ModelProfile& prof, double t_d, const StreamSpec& s,
                          std::uint64_t budget_bytes, std::size_t max_stages, const B200CostModel& cost,
                          std::size_t n_items) {
    const std::vector<std::uint64_t> w = detail::widths_of(net);
    const std::vector<ferret_layer_profile> layers = detail::c_profile(prof);
    const ferret_stream_spec spec{s.t_d, s.decay_c, s.value, s.horizon};
    const ferret_b200_cost c = cost.c();
    ferret_schedule* raw = nullptr;
    ferret_b200_plan_report rep{};
    b200_check(ferret_plan_b200(w.data(), static_cast<int32_t>(w.size()), layers.data(), t_d, &spec, budget_bytes,
                                static_cast<int32_t>(max_stages), &c, n_items, &raw, &rep));
    std::unique_ptr<ferret_schedule, void (*)(ferret_schedule*)> sched(raw, ferret_schedule_destroy);
    B200Plan out;
    std::istringstream pin(detail::schedule_text(sched.get(), ferret_schedule_plan_text));
    out.plan = parse_plan(pin, "plan_b200");
    std::istringstream tin(detail::schedule_text(sched.get(), ferret_schedule_trace_text));
    out.trace = parse_trace(tin, "plan_b200").trace;
    out.report = {rep.budget_bytes, rep.fixed_bytes,   rep.planner_budget,
                  rep.planner_bytes, rep.predicted_bytes, rep.trainer_bytes,
                  rep.passes,        static_cast<std::size_t>(rep.stages), rep.fits != 0};
    return out;
}

} // namespace ferret
