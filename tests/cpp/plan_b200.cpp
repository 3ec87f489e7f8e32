// plan_b200 through the C++ drop-in (include/ferret/b200_cost.hpp): the reference's
// plan() + simulate() flow with the B200 cost model. Runs without a GPU (the plan is
// priced by a plan-only trainer's dry-run footprint). argv[1] = budget fraction of the
// unconstrained plan's exact bytes, argv[2] = max stages; prints key/value lines.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ferret/b200_cost.hpp"
#include "ferret/net.hpp"
#include "ferret/planner.hpp"

int main(int argc, char** argv) {
    const double frac = argc > 1 ? std::atof(argv[1]) : 1.0;
    const std::size_t max_stages = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 8;
    std::vector<std::size_t> widths{784};
    for (int i = 0; i < 7; ++i) widths.push_back(256);
    widths.push_back(10);
    const ferret::DenseNet net = ferret::make_dense_net(widths, 1);
    const ferret::ModelProfile prof = ferret::profile_from_net(net);
    double t_d = 0.0, total = 0.0;
    for (const auto& l : prof.layers) {
        t_d = std::max(t_d, l.t_f);
        total += l.t_f + l.t_b;
    }
    const std::size_t units = 64;
    ferret::StreamSpec s;
    s.t_d = t_d;
    s.decay_c = std::log(2.0) / total;
    s.horizon = static_cast<double>(units) * t_d;
    ferret::B200CostModel cost;
    cost.micro_batch = 16;
    cost.chunk_units = units;
    const ferret::B200Plan free_plan = ferret::plan_b200(net, prof, t_d, s, 0, max_stages, cost, units);
    const auto budget = static_cast<std::uint64_t>(frac * static_cast<double>(free_plan.report.trainer_bytes));
    const ferret::B200Plan p = ferret::plan_b200(net, prof, t_d, s, budget, max_stages, cost, units);
    std::printf("free_trainer_bytes %llu\n", static_cast<unsigned long long>(free_plan.report.trainer_bytes));
    std::printf("budget %llu\n", static_cast<unsigned long long>(budget));
    std::printf("trainer_bytes %llu\n", static_cast<unsigned long long>(p.report.trainer_bytes));
    std::printf("fixed_bytes %llu\n", static_cast<unsigned long long>(p.report.fixed_bytes));
    std::printf("planner_bytes %llu\n", static_cast<unsigned long long>(p.report.planner_bytes));
    std::printf("plan_memory %llu\n", static_cast<unsigned long long>(p.plan.memory));
    std::printf("fits %d\n", p.report.fits ? 1 : 0);
    std::printf("passes %d\n", p.report.passes);
    std::printf("stages %zu\n", p.plan.partition.stages());
    std::printf("events %zu\n", p.trace.events.size());
    std::printf("rate %.17g\n", p.plan.rate);
    return 0;
}
