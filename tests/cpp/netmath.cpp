// The reference's dense-net math API (proj/include/ferret/net.hpp:99-208) exercised by a
// program written against the reference's names and signatures. It compiles unchanged
// against both header trees:
//   * the reference's own headers (CPU, fp64)      -> tests/golden/netmath_ref.txt
//   * this repo's drop-in headers + libferret_b200  -> the same calls on the device (fp64)
// tests/test_netmath.py compares the two outputs value by value.
// Output: one "key index value" line per number, values as %.17g.
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "ferret/net.hpp"
#include "ferret/stream.hpp"

using namespace ferret;

static void put(const char* key, const std::vector<double>& v) {
    for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s %zu %.17g\n", key, i, v[i]);
}

int main() {
    const std::vector<std::size_t> widths{64, 48, 32, 10};
    DenseNet net = make_dense_net(widths, 1);
    const DataStream stream = synth_drift_stream(12, 64, 10, DriftKind::split_tasks, 7);
    // detail::affine_forward + apply_activation on layer 0 (net.hpp:99-113)
    std::vector<double> z;
    detail::affine_forward(net.layers[0], stream.items[0].features, z);
    put("affine", z);
    detail::apply_activation(net.layers[0].act, z);
    put("relu", z);
    // forward_all / predict_logits / predict_class (net.hpp:130-154)
    for (std::size_t s = 0; s < 4; ++s) {
        const auto acts = forward_all(net, stream.items[s].features);
        for (std::size_t l = 0; l < acts.size(); ++l) put(("act" + std::to_string(s) + "_" + std::to_string(l)).c_str(), acts[l]);
        put(("logits" + std::to_string(s)).c_str(), predict_logits(net, stream.items[s].features));
        std::printf("class %zu %zu\n", s, predict_class(net, stream.items[s].features));
    }
    // detail::softmax (net.hpp:115-125)
    put("softmax", detail::softmax(predict_logits(net, stream.items[1].features)));
    // forward_backward over a batch of 8 (net.hpp:157-200) and apply_sgd (net.hpp:202-208)
    Batch batch;
    for (std::size_t s = 0; s < 8; ++s) batch.push_back({stream.items[s].features, stream.items[s].label});
    auto [loss, grads] = forward_backward(net, batch);
    std::printf("loss 0 %.17g\n", loss);
    for (std::size_t l = 0; l < grads.W.size(); ++l) {
        put(("gW" + std::to_string(l)).c_str(), grads.W[l]);
        put(("gb" + std::to_string(l)).c_str(), grads.b[l]);
    }
    apply_sgd(net, grads, 1e-3);
    for (std::size_t l = 0; l < net.layers.size(); ++l) {
        put(("W" + std::to_string(l)).c_str(), net.layers[l].W);
        put(("b" + std::to_string(l)).c_str(), net.layers[l].b);
    }
    // the reference's exceptions
    int caught = 0;
    try {
        forward_backward(net, Batch{});
    } catch (const std::invalid_argument&) {
        ++caught;
    }
    try {
        forward_backward(net, Batch{{stream.items[0].features, 10}});
    } catch (const std::invalid_argument&) {
        ++caught;
    }
    try {
        forward_backward(net, Batch{{std::vector<double>(3, 0.0), 0}});
    } catch (const std::invalid_argument&) {
        ++caught;
    }
    std::printf("exceptions 0 %d\n", caught);
    return 0;
}
