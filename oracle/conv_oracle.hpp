// ORACLE — TEST INFRASTRUCTURE ONLY (see ferret_oracle.cpp's header). Included
// at the end of ferret_oracle.cpp (same translation unit: it reuses OOpts,
// OEvent, ORecord, OracleCompensator, IndexReservoir, guard, to_stream,
// to_events and copy_records).
//
// CPU oracle for the convolutional nets of BASELINE config 3 ("ResNet-18-style
// CNN on CIFAR-shaped synthetic stream with ER replay, 4 stages"). The
// reference has no convolution ("CNN: parity unpinned"),
// so this file RESTATES the reference's dense algorithm with the layer
// generalised; everything that is not a layer operation is the reference's own
// code or the RestatedTrainer's order of operations:
//
//   * layer kinds (the geometry ferret_b200.h documents as FERRET_LAYER_*):
//       dense      z = W x + b                         net.hpp:99-108
//       conv       z[co][oh][ow] = b[co] + sum_{ci,kh,kw} W[co][ci][kh][kw] x[ci][oh*s-p+kh][ow*s-p+kw]
//                  (zero padding), optional residual: z += S(x_block) with
//                  x_block = the input of layer l-1 (a two-conv basic block),
//                  S = identity when shapes match, else "option A" (He et al.
//                  2016, CIFAR ResNets): spatial subsample by the stride,
//                  channels [0, c_block) copied, the rest zero
//       gap_dense  z = W mean_hw(x) + b  (global average pool fused into the head)
//     then the reference's activation (net.hpp:110-113).
//   * backward per layer as in on_backward / forward_backward (learner.hpp:456-474,
//     net.hpp:175-196): mask the incoming delta by the layer's own ReLU output,
//     accumulate gW/gb, prev = W^T delta (the transposed convolution for conv);
//     a residual layer m also sends S^T(delta_m) to the input of layer m-1,
//     added to layer m-1's prev.
//   * RestatedConvTrainer: on_arrival / on_forward / on_backward / on_update /
//     replay_step in exactly RestatedTrainer's order (and thus learner.hpp:389-519's),
//     with the reference's StageVersions, Compensator arithmetic, ReplayBuffer and
//     RunningNormalizer.
//
// Parity status: layer arithmetic UNPINNED against the reference (there is none);
// cross-checked instead (tests/test_conv_oracle.py) by (a) a conv net whose every
// layer is 1x1 on a 1x1 map equals the dense RestatedTrainer bit for bit, and
// (b) finite differences of the loss against forward_backward's gradients.

namespace {
namespace convo {

struct CGeom {
    int32_t kind, c_in, h_in, w_in, c_out, k, stride, pad, res;
    int h_out() const { return kind == 1 ? (h_in + 2 * pad - k) / stride + 1 : 1; }
    int w_out() const { return kind == 1 ? (w_in + 2 * pad - k) / stride + 1 : 1; }
    size_t in_w() const { return static_cast<size_t>(c_in) * h_in * w_in; }
    size_t out_w() const { return static_cast<size_t>(c_out) * h_out() * w_out(); }
    size_t cols() const { return kind == 1 ? static_cast<size_t>(c_in) * k * k : static_cast<size_t>(c_in); }
    size_t n_w() const { return static_cast<size_t>(c_out) * cols(); }
    size_t n_params() const { return n_w() + static_cast<size_t>(c_out); }
};

struct ConvNet {
    std::vector<CGeom> g;
    std::vector<int32_t> act;      // 0 relu, 1 identity
    std::vector<size_t> off;       // per layer: offset of W in the flat params; off[L] = total
    std::vector<double> params;

    size_t L() const { return g.size(); }
    const double* W(size_t l) const { return params.data() + off[l]; }
    const double* b(size_t l) const { return params.data() + off[l] + g[l].n_w(); }

    void validate() const {
        for (size_t l = 0; l < L(); ++l) {
            const CGeom& q = g[l];
            if (q.kind < 0 || q.kind > 2) throw std::invalid_argument("conv net: unknown layer kind");
            if (q.kind == 1 && (q.k < 1 || q.stride < 1 || q.pad < 0 || q.h_out() < 1 || q.w_out() < 1))
                throw std::invalid_argument("conv net: bad convolution geometry");
            if (l > 0 && q.in_w() != g[l - 1].out_w())
                throw std::invalid_argument("conv net: layer " + std::to_string(l) + ": input width mismatch");
            if (q.res) {
                if (q.kind != 1 || l < 1) throw std::invalid_argument("conv net: residual needs a conv after a layer");
                const CGeom& a = g[l - 1];
                if (a.c_in > q.c_out || a.h_in % q.h_out() != 0 || a.w_in % q.w_out() != 0 ||
                    a.h_in / q.h_out() != a.w_in / q.w_out())
                    throw std::invalid_argument("conv net: residual shortcut shape");
            }
        }
    }
};

// block input (shape of layer l-1's input) -> shortcut added to layer l's output
inline void shortcut_add(const CGeom& blk, const CGeom& q, const std::vector<double>& xs, std::vector<double>& z) {
    const int ho = q.h_out(), wo = q.w_out(), st = blk.h_in / ho;
    for (int c = 0; c < blk.c_in; ++c)
        for (int h = 0; h < ho; ++h)
            for (int w = 0; w < wo; ++w)
                z[(static_cast<size_t>(c) * ho + h) * wo + w] +=
                    xs[(static_cast<size_t>(c) * blk.h_in + h * st) * blk.w_in + w * st];
}

// S^T: delta at layer l's output (masked) -> gradient at the block input
inline std::vector<double> shortcut_grad(const CGeom& blk, const CGeom& q, const std::vector<double>& dz) {
    std::vector<double> gx(blk.in_w(), 0.0);
    const int ho = q.h_out(), wo = q.w_out(), st = blk.h_in / ho;
    for (int c = 0; c < blk.c_in; ++c)
        for (int h = 0; h < ho; ++h)
            for (int w = 0; w < wo; ++w)
                gx[(static_cast<size_t>(c) * blk.h_in + h * st) * blk.w_in + w * st] =
                    dz[(static_cast<size_t>(c) * ho + h) * wo + w];
    return gx;
}

// post-activation output of layer l; `xs` = the input of layer l-1 when layer l is residual
inline void layer_forward(const ConvNet& n, size_t l, const double* W, const double* b, const std::vector<double>& x,
                          const std::vector<double>* xs, std::vector<double>& z) {
    const CGeom& q = n.g[l];
    z.assign(q.out_w(), 0.0);
    if (q.kind == 1) {
        const int ho = q.h_out(), wo = q.w_out();
        for (int co = 0; co < q.c_out; ++co)
            for (int oh = 0; oh < ho; ++oh)
                for (int ow = 0; ow < wo; ++ow) {
                    double acc = b[co];
                    for (int ci = 0; ci < q.c_in; ++ci)
                        for (int kh = 0; kh < q.k; ++kh) {
                            const int ih = oh * q.stride - q.pad + kh;
                            if (ih < 0 || ih >= q.h_in) continue;
                            for (int kw = 0; kw < q.k; ++kw) {
                                const int iw = ow * q.stride - q.pad + kw;
                                if (iw < 0 || iw >= q.w_in) continue;
                                acc += W[((static_cast<size_t>(co) * q.c_in + ci) * q.k + kh) * q.k + kw] *
                                       x[(static_cast<size_t>(ci) * q.h_in + ih) * q.w_in + iw];
                            }
                        }
                    z[(static_cast<size_t>(co) * ho + oh) * wo + ow] = acc;
                }
        if (q.res) shortcut_add(n.g[l - 1], q, *xs, z);
    } else {
        std::vector<double> pooled;
        const std::vector<double>* in = &x;
        if (q.kind == 2) {
            const size_t hw = static_cast<size_t>(q.h_in) * q.w_in;
            pooled.assign(static_cast<size_t>(q.c_in), 0.0);
            for (int c = 0; c < q.c_in; ++c) {
                double s = 0.0;
                for (size_t p = 0; p < hw; ++p) s += x[c * hw + p];
                pooled[static_cast<size_t>(c)] = s / static_cast<double>(hw);
            }
            in = &pooled;
        }
        for (int r = 0; r < q.c_out; ++r) {  // net.hpp:99-108
            double acc = b[r];
            const double* row = W + static_cast<size_t>(r) * q.c_in;
            for (int c = 0; c < q.c_in; ++c) acc += row[c] * (*in)[static_cast<size_t>(c)];
            z[static_cast<size_t>(r)] = acc;
        }
    }
    if (n.act[l] == 0)  // net.hpp:110-113
        for (auto& v : z) v = v > 0.0 ? v : 0.0;
}

// dz = delta at layer l's pre-activation (already masked). Accumulates gW, gb
// (layer-local, W then b) and returns prev = d loss / d input (unmasked) when wanted.
inline void layer_backward(const ConvNet& n, size_t l, const double* W, const std::vector<double>& x,
                           const std::vector<double>& dz, double* grad, std::vector<double>* prev) {
    const CGeom& q = n.g[l];
    double* gW = grad;
    double* gb = grad + q.n_w();
    if (prev) prev->assign(q.in_w(), 0.0);
    if (q.kind == 1) {
        const int ho = q.h_out(), wo = q.w_out();
        for (int co = 0; co < q.c_out; ++co)
            for (int oh = 0; oh < ho; ++oh)
                for (int ow = 0; ow < wo; ++ow) {
                    const double d = dz[(static_cast<size_t>(co) * ho + oh) * wo + ow];
                    gb[co] += d;
                    for (int ci = 0; ci < q.c_in; ++ci)
                        for (int kh = 0; kh < q.k; ++kh) {
                            const int ih = oh * q.stride - q.pad + kh;
                            if (ih < 0 || ih >= q.h_in) continue;
                            for (int kw = 0; kw < q.k; ++kw) {
                                const int iw = ow * q.stride - q.pad + kw;
                                if (iw < 0 || iw >= q.w_in) continue;
                                const size_t wi = ((static_cast<size_t>(co) * q.c_in + ci) * q.k + kh) * q.k + kw;
                                const size_t xi = (static_cast<size_t>(ci) * q.h_in + ih) * q.w_in + iw;
                                gW[wi] += d * x[xi];
                                if (prev) (*prev)[xi] += d * W[wi];
                            }
                        }
                }
        return;
    }
    std::vector<double> pooled;
    const std::vector<double>* in = &x;
    const size_t hw = static_cast<size_t>(q.h_in) * q.w_in;
    if (q.kind == 2) {
        pooled.assign(static_cast<size_t>(q.c_in), 0.0);
        for (int c = 0; c < q.c_in; ++c) {
            double s = 0.0;
            for (size_t p = 0; p < hw; ++p) s += x[c * hw + p];
            pooled[static_cast<size_t>(c)] = s / static_cast<double>(hw);
        }
        in = &pooled;
    }
    std::vector<double> pp(static_cast<size_t>(q.c_in), 0.0);
    for (int r = 0; r < q.c_out; ++r) {  // learner.hpp:462-474
        const double d = dz[static_cast<size_t>(r)];
        gb[r] += d;
        for (int c = 0; c < q.c_in; ++c) {
            gW[static_cast<size_t>(r) * q.c_in + c] += d * (*in)[static_cast<size_t>(c)];
            pp[static_cast<size_t>(c)] += d * W[static_cast<size_t>(r) * q.c_in + c];
        }
    }
    if (!prev) return;
    if (q.kind == 0) {
        *prev = std::move(pp);
    } else {
        for (int c = 0; c < q.c_in; ++c)
            for (size_t p = 0; p < hw; ++p) (*prev)[c * hw + p] = pp[static_cast<size_t>(c)] / static_cast<double>(hw);
    }
}

inline void mask_relu(const ConvNet& n, size_t l, const std::vector<double>& y, std::vector<double>& d) {
    if (n.act[l] == 0)
        for (size_t r = 0; r < d.size(); ++r)
            if (y[r] <= 0.0) d[r] = 0.0;
}

// forward over layers [lo, hi) from `x` (the input of layer lo); `xprev` = the
// input of layer lo-1 (needed when lo is residual — never, bounds respect blocks)
inline void forward_span(const ConvNet& n, const std::vector<double>& params, size_t base, size_t lo, size_t hi,
                         const std::vector<double>& x, std::vector<std::vector<double>>& acts) {
    acts.clear();
    for (size_t l = lo; l < hi; ++l) {
        const std::vector<double>& in = l == lo ? x : acts[l - lo - 1];
        const std::vector<double>* xs = nullptr;
        if (n.g[l].res) xs = l - 1 == lo ? &x : &acts[l - lo - 2];
        std::vector<double> z;
        const double* W = params.data() + (n.off[l] - base);
        layer_forward(n, l, W, W + n.g[l].n_w(), in, xs, z);
        acts.push_back(std::move(z));
    }
}

// backward over layers [lo, hi) given delta at the output of layer hi-1
// (unmasked); grads (stage-local flat, W then b per layer) accumulate; returns
// the delta at the input of layer lo (prev of layer lo), computed when want_prev.
inline std::vector<double> backward_span(const ConvNet& n, const std::vector<double>& params, size_t base, size_t lo,
                                         size_t hi, const std::vector<double>& x,
                                         const std::vector<std::vector<double>>& acts, std::vector<double> delta,
                                         double* grads, bool want_prev_lo) {
    std::vector<double> skip;  // S^T(dz_{l+1}) pending for layer l's prev
    for (size_t l = hi; l-- > lo;) {
        const std::vector<double>& in = l == lo ? x : acts[l - lo - 1];
        mask_relu(n, l, acts[l - lo], delta);
        std::vector<double> next_skip;
        if (n.g[l].res) next_skip = shortcut_grad(n.g[l - 1], n.g[l], delta);
        const double* W = params.data() + (n.off[l] - base);
        std::vector<double> prev;
        const bool want = l > lo || want_prev_lo;
        layer_backward(n, l, W, in, delta, grads + (n.off[l] - n.off[lo]), want ? &prev : nullptr);
        if (!skip.empty() && want)
            for (size_t i = 0; i < prev.size(); ++i) prev[i] += skip[i];
        skip = std::move(next_skip);
        delta = std::move(prev);
    }
    return delta;
}

inline size_t predict(const ConvNet& n, const std::vector<double>& x) {
    std::vector<std::vector<double>> acts;
    forward_span(n, n.params, 0, 0, n.L(), x, acts);
    const auto& lg = acts.back();
    return static_cast<size_t>(std::max_element(lg.begin(), lg.end()) - lg.begin());  // net.hpp:150-154
}

// forward_backward (net.hpp:157-200) generalised: mean CE over the batch, no
// dX for layer 0; returns the flat gradient
inline std::vector<double> forward_backward(const ConvNet& n, const std::vector<const ferret::Sample*>& batch) {
    std::vector<double> grads(n.params.size(), 0.0);
    const double inv_n = 1.0 / static_cast<double>(batch.size());
    for (const ferret::Sample* s : batch) {
        std::vector<std::vector<double>> acts;
        forward_span(n, n.params, 0, 0, n.L(), s->x, acts);
        std::vector<double> delta = ferret::detail::softmax(acts.back());
        delta[s->label] -= 1.0;
        for (auto& v : delta) v *= inv_n;
        backward_span(n, n.params, 0, 0, n.L(), s->x, acts, std::move(delta), grads.data(), false);
    }
    return grads;
}

class RestatedConvTrainer {
  public:
    RestatedConvTrainer(ConvNet net, const std::vector<size_t>& bounds, const OOpts& o)
        : net_(std::move(net)), bounds_(bounds), opt_(o), B_(o.micro_batch), norm_(net_.g.front().in_w()),
          buffer_(o.replay_capacity, o.replay_seed), index_(o.replay_capacity, o.replay_seed) {
        net_.validate();
        if (bounds_.size() < 2 || bounds_.front() != 0 || bounds_.back() != net_.L())
            throw ferret::ConfigError("partition bounds must run from 0 to the layer count");
        for (size_t i = 1; i < bounds_.size(); ++i) {
            if (bounds_[i] <= bounds_[i - 1]) throw ferret::ConfigError("partition bounds must be strictly increasing");
            if (bounds_[i] < net_.L() && net_.g[bounds_[i]].res)
                throw ferret::ConfigError("partition bound splits a residual block");
        }
        if (B_ < 1) throw std::invalid_argument("micro_batch must be >= 1");
        const size_t P = bounds_.size() - 1;
        versions_.resize(P);
        for (size_t j = 0; j < P; ++j) {
            versions_[j].init(stage_params(j));
            comps_.emplace_back(static_cast<ferret::CompensationPolicy>(o.policy), stage_params(j).size(), o.lambda0,
                                o.eta_lambda, o.alpha, o.nu);
        }
    }

    std::vector<double> stage_params(size_t j) const {
        return {net_.params.begin() + static_cast<long>(net_.off[bounds_[j]]),
                net_.params.begin() + static_cast<long>(net_.off[bounds_[j + 1]])};
    }
    void set_stage_params(size_t j, const std::vector<double>& p) {
        std::copy(p.begin(), p.end(), net_.params.begin() + static_cast<long>(net_.off[bounds_[j]]));
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

    ConvNet net_;
    std::vector<size_t> bounds_;
    OOpts opt_;
    int B_;
    ferret::RunningNormalizer norm_;
    ferret::ReplayBuffer buffer_;
    IndexReservoir index_;
    std::vector<int64_t> replay_ids;
    std::vector<ferret::detail::StageVersions> versions_;
    std::vector<OracleCompensator> comps_;
    std::vector<std::vector<double>> xs_;

  private:
    struct InFlight {
        std::vector<std::vector<double>> input;
        std::vector<size_t> label;
        std::vector<int64_t> read_version;
        std::vector<std::vector<std::vector<std::vector<double>>>> acts;  // stage -> sample -> layer -> out
        std::vector<std::vector<double>> delta;
    };
    struct PendingGrad {
        ferret::ParamVec grad;
        int64_t read_version;
    };
    std::map<int64_t, InFlight> inflight_;
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
            const size_t pred = predict(net_, fl.input[static_cast<size_t>(b)]);
            const size_t label = fl.label[static_cast<size_t>(b)];
            log[s] = {static_cast<int64_t>(s), pred == label ? ferret::StepOutcome::correct : ferret::StepOutcome::wrong,
                      pred, label};
        }
        const size_t P = bounds_.size() - 1;
        fl.read_version.assign(P, -1);
        fl.acts.resize(P);
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

    const std::vector<double>& stage_input(const InFlight& fl, size_t j, size_t b) const {
        return j == 0 ? fl.input[b] : fl.acts[j - 1][b].back();
    }

    void on_forward(const ferret::SimEvent& e) {
        auto it = inflight_.find(e.item);
        if (it == inflight_.end()) return;
        InFlight& fl = it->second;
        const size_t j = static_cast<size_t>(e.stage);
        const int64_t v = versions_[j].current();
        fl.read_version[j] = v;
        versions_[j].hold(v);
        const std::vector<double> p = versions_[j].at(v);
        fl.acts[j].assign(static_cast<size_t>(B_), {});
        for (size_t b = 0; b < static_cast<size_t>(B_); ++b)
            forward_span(net_, p, net_.off[bounds_[j]], bounds_[j], bounds_[j + 1], stage_input(fl, j, b), fl.acts[j][b]);
    }

    void on_backward(const ferret::SimEvent& e) {
        auto it = inflight_.find(e.item);
        if (it == inflight_.end()) return;
        InFlight& fl = it->second;
        const size_t j = static_cast<size_t>(e.stage);
        const std::vector<double> p = versions_[j].at(fl.read_version[j]);
        const double inv_b = 1.0 / static_cast<double>(B_);
        ferret::ParamVec grad(p.size(), 0.0);
        for (size_t b = 0; b < static_cast<size_t>(B_); ++b) {
            std::vector<double> delta;
            if (j + 2 == bounds_.size()) {
                delta = ferret::detail::softmax(fl.acts[j][b].back());
                delta[fl.label[b]] -= 1.0;
                for (auto& v : delta) v *= inv_b;
            } else {
                delta = fl.delta[b];
            }
            fl.delta[b] = backward_span(net_, p, net_.off[bounds_[j]], bounds_[j], bounds_[j + 1], stage_input(fl, j, b),
                                        fl.acts[j][b], std::move(delta), grad.data(), true);
        }
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
        set_stage_params(j, params);
        versions_[j].push(std::move(params));
        for (const auto& pg : it->second) versions_[j].release(pg.read_version);
        it->second.clear();
        if (j == 0 && opt_.replay && !buffer_.empty()) replay_step();
    }

    void replay_step() {
        std::vector<const ferret::Sample*> batch;
        for (int b = 0; b < B_; ++b) {
            const ferret::Sample& s = buffer_.sample();
            const int64_t id = index_.sample();
            if (xs_[static_cast<size_t>(id)] != s.x)
                throw std::logic_error("oracle: restated replay index disagrees with the reference ReplayBuffer");
            replay_ids.push_back(id);
            batch.push_back(&s);
        }
        const std::vector<double> grads = forward_backward(net_, batch);
        for (size_t i = 0; i < grads.size(); ++i) net_.params[i] -= opt_.lr * grads[i];  // net.hpp:202-208
        for (size_t j = 0; j + 1 < bounds_.size(); ++j) versions_[j].push(stage_params(j));
    }
};

inline ConvNet to_conv_net(int32_t n_layers, const int32_t* geom, const int32_t* act, const double* params) {
    ConvNet n;
    size_t at = 0;
    for (int32_t l = 0; l < n_layers; ++l) {
        const int32_t* q = geom + 9 * l;
        n.g.push_back({q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7], q[8]});
        n.act.push_back(act[l]);
        n.off.push_back(at);
        at += n.g.back().n_params();
    }
    n.off.push_back(at);
    n.params.assign(params, params + at);
    return n;
}

}  // namespace convo
}  // namespace

// Conv-net pipelined trainer oracle. geom: n_layers x 9 int32
// {kind, c_in, h_in, w_in, c_out, k, stride, pad, res}; params flat (per layer W then b).
ORACLE_API int ferret_oracle_train_conv(int32_t n_layers, const int32_t* geom, const int32_t* act, const double* params,
                                        const uint64_t* bounds, int32_t n_bounds, const OOpts* opts,
                                        const OEvent* events, size_t n_events, const double* features,
                                        const uint64_t* labels, size_t n_items, size_t n_features, ORecord* log_out,
                                        double* params_out, double* lambda_out, double* v_r_out, double* v_a_out,
                                        int64_t* replay_ids, size_t replay_cap, size_t* n_replay) {
    return guard([&] {
        convo::ConvNet net = convo::to_conv_net(n_layers, geom, act, params);
        if (net.g.front().in_w() != n_features) throw std::invalid_argument("conv oracle: feature width mismatch");
        std::vector<size_t> b(bounds, bounds + n_bounds);
        const ferret::DataStream ds = to_stream(features, labels, n_items, n_features);
        const auto ev = to_events(events, n_events);
        convo::RestatedConvTrainer tr(std::move(net), b, *opts);
        const auto log = tr.run(ev, ds);
        if (log_out) copy_records(log, log_out);
        if (params_out) std::memcpy(params_out, tr.net_.params.data(), tr.net_.params.size() * sizeof(double));
        size_t at = 0;
        for (size_t j = 0; j < tr.comps_.size(); ++j) {
            const auto& c = tr.comps_[j];
            const size_t n = tr.stage_params(j).size();
            auto put = [&](double* dst, const ferret::ParamVec& src) {
                if (!dst) return;
                for (size_t i = 0; i < n; ++i) dst[at + i] = src.empty() ? 0.0 : src[i];
            };
            if (c.policy == ferret::CompensationPolicy::iter_fisher) put(lambda_out, c.state.lambda);
            put(v_r_out, c.state.v_r);
            put(v_a_out, c.state.v_a);
            at += n;
        }
        if (n_replay) *n_replay = tr.replay_ids.size();
        if (replay_ids)
            for (size_t i = 0; i < tr.replay_ids.size() && i < replay_cap; ++i) replay_ids[i] = tr.replay_ids[i];
    });
}

// One generalised forward_backward (mean CE) on the conv net: gradient + loss-free check entry
// for the finite-difference test; also the per-sample forward (logits) for spot checks.
ORACLE_API int ferret_oracle_conv_grad(int32_t n_layers, const int32_t* geom, const int32_t* act, const double* params,
                                       const double* x, const uint64_t* labels, size_t batch, double* grad_out,
                                       double* logits_out) {
    return guard([&] {
        convo::ConvNet net = convo::to_conv_net(n_layers, geom, act, params);
        net.validate();
        const size_t F = net.g.front().in_w(), C = net.g.back().out_w();
        std::vector<ferret::Sample> samples(batch);
        std::vector<const ferret::Sample*> ptr;
        for (size_t i = 0; i < batch; ++i) {
            samples[i].x.assign(x + i * F, x + (i + 1) * F);
            samples[i].label = labels[i];
            ptr.push_back(&samples[i]);
        }
        if (grad_out) {
            const auto g = convo::forward_backward(net, ptr);
            std::memcpy(grad_out, g.data(), g.size() * sizeof(double));
        }
        if (logits_out)
            for (size_t i = 0; i < batch; ++i) {
                std::vector<std::vector<double>> acts;
                convo::forward_span(net, net.params, 0, 0, net.L(), samples[i].x, acts);
                std::memcpy(logits_out + i * C, acts.back().data(), C * sizeof(double));
            }
    });
}
