// The conv extension through the C++ API (include/ferret/conv.hpp): a ResNet-style
// net built with resnet_cifar_layout, trained by ConvPipelineTrainer on a schedule,
// stream and initial parameters read from <dir> (written by tests/test_dropin_cpp.py);
// writes the final parameters and the predictions for the test to compare with the
// Python mirror's run of the same inputs.
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "ferret/conv.hpp"

template <class T>
static std::vector<T> read_all(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    const std::string buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::vector<T> v(buf.size() / sizeof(T));
    std::copy(buf.data(), buf.data() + v.size() * sizeof(T), reinterpret_cast<char*>(v.data()));
    return v;
}

template <class T>
static void write_all(const std::string& path, const std::vector<T>& v) {
    std::ofstream(path, std::ios::binary).write(reinterpret_cast<const char*>(v.data()),
                                                static_cast<std::streamsize>(v.size() * sizeof(T)));
}

int main(int argc, char** argv) {
    using namespace ferret;
    if (argc < 3) return 2;
    const std::string dir = argv[1];
    const std::size_t width = std::stoul(argv[2]);
    ConvNet net = resnet_cifar_layout(width);
    net.params = read_all<double>(dir + "/params.bin");
    std::printf("n_params %zu\n", net.n_params());
    const std::vector<uint64_t> bounds = read_all<uint64_t>(dir + "/bounds.bin");
    PartitionScheme scheme;
    scheme.bounds.assign(bounds.begin(), bounds.end());
    // ferret_event records (the Python EVENT_DTYPE)
    const std::vector<ferret_event> ev = read_all<ferret_event>(dir + "/events.bin");
    SimTrace trace;
    for (const ferret_event& e : ev) {
        SimEvent s;
        s.time = e.time;
        s.kind = static_cast<EventKind>(e.kind);
        s.worker = e.worker;
        s.stage = e.stage;
        s.item = e.item;
        s.version = e.version;
        s.staleness = e.staleness;
        trace.events.push_back(s);
    }
    const std::vector<double> feats = read_all<double>(dir + "/features.bin");
    const std::vector<uint64_t> labels = read_all<uint64_t>(dir + "/labels.bin");
    DataStream stream;
    stream.n_features = net.n_inputs();
    stream.n_classes = net.n_outputs();
    for (std::size_t i = 0; i < labels.size(); ++i)
        stream.items.push_back({static_cast<std::int64_t>(i),
                                std::vector<double>(feats.begin() + i * stream.n_features,
                                                    feats.begin() + (i + 1) * stream.n_features),
                                static_cast<std::size_t>(labels[i])});
    PipelineTrainOptions po;
    po.policy = CompensationPolicy::iter_fisher;
    po.replay = true;
    po.replay_seed = 3;
    ConvPipelineTrainer tr(net, scheme, po);
    const std::vector<StepRecord> log = tr.run(trace, stream);
    std::vector<uint64_t> pred;
    for (const StepRecord& r : log) pred.push_back(r.predicted);
    write_all(dir + "/out_params.bin", tr.params());
    write_all(dir + "/out_pred.bin", pred);
    std::printf("items %zu\n", log.size());
    return 0;
}
