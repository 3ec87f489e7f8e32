// Convolutional extension of the drop-in API (BASELINE config 3: "ResNet-18-style CNN").
// The reference has no convolution, so nothing here replaces a reference header; the
// types follow the reference's conventions (by-value nets, PartitionScheme, SimTrace,
// DataStream, PipelineTrainOptions, TrainOutcome-style results, exceptions from status
// codes) and the trainer is the same device trainer as PipelineTrainer
// (ferret_trainer_create with ferret_net_desc::geom, FERRET_LAYER_* in ferret_b200.h).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "ferret/learner.hpp"

namespace ferret {

enum class LayerKind : int32_t { dense = FERRET_LAYER_DENSE, conv = FERRET_LAYER_CONV, gap_dense = FERRET_LAYER_GAP_DENSE };

/// One layer: dense (c_in = in, h = w = 1), conv (k x k, stride, zero padding; residual adds
/// the shortcut of the input of the layer below: identity, or stride subsample + zero
/// channels) or gap_dense (global average pool fused into a dense head).
struct ConvLayer {
    LayerKind kind = LayerKind::conv;
    std::size_t c_in = 0, h_in = 1, w_in = 1, c_out = 0;
    std::size_t k = 1, stride = 1, pad = 0;
    bool residual = false;
    Activation act = Activation::relu;

    std::size_t h_out() const { return kind == LayerKind::conv ? (h_in + 2 * pad - k) / stride + 1 : 1; }
    std::size_t w_out() const { return kind == LayerKind::conv ? (w_in + 2 * pad - k) / stride + 1 : 1; }
    std::size_t in_width() const { return c_in * h_in * w_in; }
    std::size_t out_width() const { return c_out * h_out() * w_out(); }
    std::size_t n_params() const { return c_out * (kind == LayerKind::conv ? c_in * k * k : c_in) + c_out; }
};

/// A conv net: layers plus flat parameters (per layer W = c_out x (c_in k k | c_in), then b).
struct ConvNet {
    std::vector<ConvLayer> layers;
    ParamVec params;

    std::size_t n_params() const {
        std::size_t n = 0;
        for (const ConvLayer& l : layers) n += l.n_params();
        return n;
    }
    std::size_t n_inputs() const { return layers.front().in_width(); }
    std::size_t n_outputs() const { return layers.back().out_width(); }
    void validate() const {
        if (layers.empty()) throw ConfigError("conv net: no layers");
        for (std::size_t l = 1; l < layers.size(); ++l)
            if (layers[l].in_width() != layers[l - 1].out_width())
                throw ConfigError("conv net: layer " + std::to_string(l) + ": input width mismatch");
        if (params.size() != n_params()) throw ConfigError("conv net: parameter count mismatch");
    }
};

/// The ResNet-18 layout for CIFAR-shaped inputs (3x3 stem, 2+2+2+2 basic blocks at widths
/// width x 1/2/4/8, option-A shortcuts, GAP + dense head); parameters left empty.
inline ConvNet resnet_cifar_layout(std::size_t width = 64, std::size_t n_classes = 10, std::size_t c = 3,
                                   std::size_t h = 32, std::size_t w = 32) {
    ConvNet net;
    net.layers.push_back({LayerKind::conv, c, h, w, width, 3, 1, 1, false, Activation::relu});
    c = width;
    for (std::size_t g = 0; g < 4; ++g) {
        const std::size_t cg = width << g;
        for (std::size_t b = 0; b < 2; ++b) {
            const std::size_t s = (g > 0 && b == 0) ? 2 : 1;
            net.layers.push_back({LayerKind::conv, c, h, w, cg, 3, s, 1, false, Activation::relu});
            h = (h + 2 - 3) / s + 1;
            w = (w + 2 - 3) / s + 1;
            net.layers.push_back({LayerKind::conv, cg, h, w, cg, 3, 1, 1, true, Activation::relu});
            c = cg;
        }
    }
    net.layers.push_back({LayerKind::gap_dense, c, h, w, n_classes, 1, 1, 0, false, Activation::identity});
    return net;
}

/// The pipelined trainer (PipelineTrainer's contract) over a conv net.
class ConvPipelineTrainer {
  public:
    ConvPipelineTrainer(ConvNet net, const PartitionScheme& scheme, const PipelineTrainOptions& opt,
                        const B200Options& b200 = B200Options{})
        : net_(std::move(net)) {
        net_.validate();
        std::vector<uint64_t> in, out, bounds(scheme.bounds.begin(), scheme.bounds.end());
        std::vector<int32_t> act, geom;
        for (const ConvLayer& l : net_.layers) {
            in.push_back(l.in_width());
            out.push_back(l.out_width());
            act.push_back(static_cast<int32_t>(l.act));
            for (std::size_t v : {static_cast<std::size_t>(l.kind), l.c_in, l.h_in, l.w_in, l.c_out, l.k, l.stride,
                                  l.pad, static_cast<std::size_t>(l.residual ? 1 : 0)})
                geom.push_back(static_cast<int32_t>(v));
        }
        const ferret_net_desc desc{static_cast<int32_t>(net_.layers.size()), in.data(), out.data(), act.data(),
                                   net_.params.data(), geom.data()};
        ferret_train_opts o;
        ferret_train_opts_default(&o);
        o.policy = static_cast<int32_t>(opt.policy);
        o.lr = opt.lr;
        o.eta_lambda = opt.eta_lambda;
        o.replay = opt.replay ? 1 : 0;
        o.replay_seed = opt.replay_seed;
        o.replay_capacity = kReplayBuffer;
        o.precision = b200.precision;
        o.micro_batch = b200.micro_batch;
        o.device = b200.device;
        ferret_trainer* raw = nullptr;
        b200_check(ferret_trainer_create(&desc, bounds.data(), static_cast<int32_t>(bounds.size()), &o, &raw));
        handle_.reset(raw);
    }

    /// PipelineTrainer::run (learner.hpp:348-363): the StepRecord log of the stream.
    std::vector<StepRecord> run(const SimTrace& trace, const DataStream& stream) {
        std::vector<ferret_event> events;
        events.reserve(trace.events.size());
        for (const SimEvent& e : trace.events)
            events.push_back(ferret_event{e.time, static_cast<int32_t>(e.kind), e.worker, e.stage, e.staleness, e.item,
                                          e.version});
        const std::size_t n = stream.items.size(), f = stream.n_features;
        std::vector<double> features(n * f);
        std::vector<uint64_t> labels(n);
        for (std::size_t i = 0; i < n; ++i) {
            std::copy(stream.items[i].features.begin(), stream.items[i].features.end(), features.begin() + i * f);
            labels[i] = stream.items[i].label;
        }
        std::vector<ferret_step_record> raw_log(n);
        b200_check(ferret_trainer_run(handle_.get(), events.data(), events.size(), features.data(), labels.data(), n, f,
                                      raw_log.data()));
        std::vector<StepRecord> log(n);
        for (std::size_t i = 0; i < n; ++i)
            log[i] = StepRecord{raw_log[i].item, static_cast<StepOutcome>(raw_log[i].outcome),
                                static_cast<std::size_t>(raw_log[i].predicted),
                                static_cast<std::size_t>(raw_log[i].label)};
        return log;
    }

    /// The live parameters (flat, fp64).
    ParamVec params() {
        ParamVec p(net_.n_params());
        b200_check(ferret_trainer_params(handle_.get(), p.data(), p.size()));
        return p;
    }

  private:
    struct Release {
        void operator()(ferret_trainer* t) const { ferret_trainer_destroy(t); }
    };
    ConvNet net_;
    std::unique_ptr<ferret_trainer, Release> handle_;
};

}  // namespace ferret
