// Drop-in check: a program written against the reference's C++ API (the
// names and signatures of proj/include/ferret/*.hpp) compiled against this
// repo's include/ferret/ and linked with libferret_b200.so, running every
// trainer on the device: train_pipeline (learner.hpp:522-526), StaleHarness
// (:132-170), train_sequential (:197-225), test_accuracy (:185-192).
// Prints one line per result for tests/test_dropin_cpp.py to compare with the
// Python mirror of the same calls.
#include <cstdio>
#include <vector>

#include "ferret/learner.hpp"
#include "ferret/planner.hpp"
#include "ferret/sim.hpp"

int main() {
    using namespace ferret;
    const std::vector<std::size_t> widths{96, 128, 64, 10};
    const DenseNet net = make_dense_net(widths, 1);
    const DataStream stream = synth_drift_stream(240, 96, 10, DriftKind::split_tasks, 7);
    // pipeline: 2 stages, iter_fisher
    const ModelProfile prof = profile_from_net(net);
    double t_d = 0.0;
    for (const auto& l : prof.layers) t_d = std::max(t_d, l.t_f);
    StreamSpec spec;
    spec.t_d = t_d;
    spec.horizon = 240 * t_d;
    const PartitionScheme scheme{{0, 1, 3}};
    const StageStats st = stage_stats(prof, scheme);
    const PipelineConfig cfg = default_config(st, t_d, 0);
    const SimTrace trace = simulate(st, cfg, spec, 240);
    PipelineTrainOptions po;
    po.policy = CompensationPolicy::iter_fisher;
    const TrainOutcome pipe = train_pipeline(net, scheme, trace, stream, po);
    std::printf("pipeline_oacc %.6f\n", pipe.oacc());
    // StaleHarness, tau = i % 5, ring depth 4
    StaleHarness h(net, CompensationPolicy::iter_fisher, 4);
    std::size_t correct = 0;
    for (std::size_t i = 0; i < stream.items.size(); ++i)
        correct += h.ocl_step(stream.items[i], static_cast<int>(i % 5)) == stream.items[i].label ? 1 : 0;
    std::printf("harness_correct %zu\n", correct);
    double s = 0.0;
    for (double v : flatten(h.net())) s += v;
    std::printf("harness_param_sum %.9e\n", s);
    // train_sequential, one_skip, replay
    SkipPolicy sp;
    sp.kind = SkipKind::one_skip;
    const TrainOutcome seq = train_sequential(net, stream, 1.0, sp, 1.5, kLearningRate, true, 3);
    std::printf("sequential_oacc %.6f\n", seq.oacc());
    std::vector<Sample> held;
    for (std::size_t i = 200; i < 240; ++i) held.push_back({stream.items[i].features, stream.items[i].label});
    std::printf("test_accuracy %.6f\n", test_accuracy(seq.net, seq.normalizer, held));
    return 0;
}
