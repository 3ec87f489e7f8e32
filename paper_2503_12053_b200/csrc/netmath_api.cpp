// C-ABI entries of the reference's dense-net math (net.hpp:99-208) on the device, fp64
// (netmath.cu). The drop-in include/ferret/net.hpp calls these from detail::affine_forward,
// detail::apply_activation, detail::softmax, forward_all (-> predict_logits,
// predict_class), forward_backward and apply_sgd, keeping the reference's signatures and
// exceptions (std::invalid_argument for an empty batch, a feature-width mismatch or a
// label out of range, net.hpp:159-167; ConfigError from DenseNet::validate).
//
// Each call runs on the calling thread's current CUDA device (sm_100 required: there is
// no CPU fallback) on a private stream, synchronously: host buffers in, host buffers out.
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "common.hpp"
#include "netmath.cuh"

using fb200::fail;
using fb200::guarded;

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(FERRET_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int current_device() {
    int n = 0, dev = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        fail(FERRET_E_NO_DEVICE, "no sm_100 device visible (libferret_b200 has no CPU fallback)");
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    cudaDeviceProp p{};
    ck(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
    if (p.major != 10)
        fail(FERRET_E_NO_DEVICE, "current device is not sm_100 (libferret_b200 has no CPU fallback)");
    return dev;
}

// device buffers of one call, freed on scope exit
struct Scratch {
    std::vector<void*> ptrs;
    cudaStream_t st = nullptr;
    Scratch() {
        current_device();
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    ~Scratch() {
        if (st) cudaStreamSynchronize(st);
        for (void* p : ptrs) cudaFree(p);
        if (st) cudaStreamDestroy(st);
    }
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    T* upload(const T* h, size_t n) {
        T* d = alloc<T>(n);
        if (n) ck(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
        return d;
    }
    template <class T>
    void download(T* h, const T* d, size_t n) {
        if (n) ck(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, st), "D2H");
    }
    void sync() { ck(cudaStreamSynchronize(st), "cudaStreamSynchronize"); }
};

struct NetView {
    std::vector<int> in, out, relu;
    std::vector<size_t> w_off, b_off;  // offsets inside the flattened params (flatten() order)
    size_t n_params = 0;
    size_t act_total = 0;              // sum of layer output widths
};

NetView view(const ferret_net_desc* net) {
    if (!net || net->n_layers <= 0 || !net->in || !net->out || !net->act)
        fail(FERRET_E_CONFIG, "net needs at least one layer");
    if (net->geom) fail(FERRET_E_CONFIG, "net math entries take dense nets only");
    NetView v;
    size_t at = 0;
    for (int32_t l = 0; l < net->n_layers; ++l) {
        if (l > 0 && net->out[l - 1] != net->in[l])
            fail(FERRET_E_CONFIG, "layer " + std::to_string(l) + ": input width mismatch");
        v.in.push_back(static_cast<int>(net->in[l]));
        v.out.push_back(static_cast<int>(net->out[l]));
        v.relu.push_back(net->act[l] == FERRET_ACT_RELU ? 1 : 0);
        v.w_off.push_back(at);
        at += net->in[l] * net->out[l];
        v.b_off.push_back(at);
        at += net->out[l];
        v.act_total += net->out[l];
    }
    v.n_params = at;
    return v;
}

// every layer's post-activation output for n samples: acts row s = [layer 0 | layer 1 | ...]
void forward_dev(Scratch& S, const NetView& v, const double* dP, const double* dX, size_t n, double* dA) {
    const long long lda = static_cast<long long>(v.act_total);
    size_t col = 0;
    const double* x = dX;
    long long ldx = v.in[0];
    for (size_t l = 0; l < v.in.size(); ++l) {
        ck(fb200::nm_affine(dP + v.w_off[l], dP + v.b_off[l], x, ldx, dA + col, lda, v.in[l], v.out[l],
                            static_cast<int>(n), v.relu[l], S.st),
           "affine_forward");
        x = dA + col;
        ldx = lda;
        col += static_cast<size_t>(v.out[l]);
    }
}

}  // namespace

extern "C" {

ferret_status ferret_affine_forward(const double* W, const double* b, uint64_t in, uint64_t out, const double* x,
                                    double* z) {
    return guarded([&] {
        if (!W || !b || !x || !z) fail(FERRET_E_INVALID_ARG, "affine_forward: null buffer");
        Scratch S;
        const double* dW = S.upload(W, in * out);
        const double* db = S.upload(b, out);
        const double* dx = S.upload(x, in);
        double* dz = S.alloc<double>(out);
        ck(fb200::nm_affine(dW, db, dx, static_cast<long long>(in), dz, static_cast<long long>(out),
                            static_cast<int>(in), static_cast<int>(out), 1, 0, S.st),
           "affine_forward");
        S.download(z, dz, out);
        S.sync();
    });
}

ferret_status ferret_apply_activation(int32_t act, double* z, size_t n) {
    return guarded([&] {
        if (act != FERRET_ACT_RELU && act != FERRET_ACT_IDENTITY) fail(FERRET_E_INVALID_ARG, "unknown activation");
        if (!n) return;
        if (!z) fail(FERRET_E_INVALID_ARG, "apply_activation: null buffer");
        Scratch S;
        double* dz = S.upload(z, n);
        if (act == FERRET_ACT_RELU) ck(fb200::nm_relu(dz, n, S.st), "apply_activation");
        S.download(z, dz, n);
        S.sync();
    });
}

ferret_status ferret_softmax(const double* z, size_t n, double* p) {
    return guarded([&] {
        if (!n) fail(FERRET_E_INVALID_ARG, "softmax: empty input");
        if (!z || !p) fail(FERRET_E_INVALID_ARG, "softmax: null buffer");
        Scratch S;
        const double* dz = S.upload(z, n);
        double* dp = S.alloc<double>(n);
        ck(fb200::nm_softmax(dz, static_cast<long long>(n), static_cast<int>(n), 1, dp, nullptr, 0.0, nullptr, nullptr,
                             S.st),
           "softmax");
        S.download(p, dp, n);
        S.sync();
    });
}

ferret_status ferret_net_forward_all(const ferret_net_desc* net, const double* x, size_t n, double* acts) {
    return guarded([&] {
        const NetView v = view(net);
        if (!net->params || !x || !acts) fail(FERRET_E_INVALID_ARG, "forward_all: null buffer");
        if (!n) return;
        Scratch S;
        const double* dP = S.upload(net->params, v.n_params);
        const double* dX = S.upload(x, n * static_cast<size_t>(v.in[0]));
        double* dA = S.alloc<double>(n * v.act_total);
        forward_dev(S, v, dP, dX, n, dA);
        S.download(acts, dA, n * v.act_total);
        S.sync();
    });
}

ferret_status ferret_net_forward_backward(const ferret_net_desc* net, const double* x, const uint64_t* labels,
                                          size_t n, double* loss, double* grads) {
    return guarded([&] {
        const NetView v = view(net);
        if (n == 0) fail(FERRET_E_INVALID_ARG, "forward_backward: empty batch");
        if (!net->params || !x || !labels || !loss || !grads) fail(FERRET_E_INVALID_ARG, "forward_backward: null buffer");
        const int k = v.out.back();
        for (size_t s = 0; s < n; ++s)
            if (labels[s] >= static_cast<uint64_t>(k)) fail(FERRET_E_INVALID_ARG, "forward_backward: label out of range");
        Scratch S;
        const int L = static_cast<int>(v.in.size());
        const long long lda = static_cast<long long>(v.act_total);
        const double* dP = S.upload(net->params, v.n_params);
        const double* dX = S.upload(x, n * static_cast<size_t>(v.in[0]));
        const unsigned long long* dY =
            S.upload(reinterpret_cast<const unsigned long long*>(labels), n);
        double* dA = S.alloc<double>(n * v.act_total);
        double* dG = S.alloc<double>(v.n_params);
        double* dprob = S.alloc<double>(n * static_cast<size_t>(k));
        double* dlogp = S.alloc<double>(n);
        double* dloss = S.alloc<double>(1);
        int maxw = 0;
        for (int l = 0; l < L; ++l) maxw = std::max(maxw, std::max(v.in[l], v.out[l]));
        double* dd[2] = {S.alloc<double>(n * maxw), S.alloc<double>(n * maxw)};
        forward_dev(S, v, dP, dX, n, dA);
        const double inv_n = 1.0 / static_cast<double>(n);
        const size_t last_col = v.act_total - static_cast<size_t>(k);
        ck(fb200::nm_softmax(dA + last_col, lda, k, static_cast<int>(n), dprob, dY, inv_n, dlogp, dd[0], S.st), "softmax");
        ck(fb200::nm_loss(dlogp, static_cast<int>(n), inv_n, dloss, S.st), "loss");
        size_t col = last_col;
        int cur = 0;
        for (int l = L - 1; l >= 0; --l) {
            if (v.relu[l]) ck(fb200::nm_mask(dd[cur], dA + col, lda, v.out[l], static_cast<int>(n), S.st), "mask");
            const double* input = l == 0 ? dX : dA + (col - static_cast<size_t>(v.in[l]));
            const long long ldin = l == 0 ? v.in[0] : lda;
            ck(fb200::nm_wgrad(dd[cur], input, ldin, dG + v.w_off[l], dG + v.b_off[l], v.in[l], v.out[l],
                               static_cast<int>(n), S.st),
               "weight gradient");
            if (l == 0) break;  // net.hpp:191: no input gradient for the first layer
            ck(fb200::nm_dgrad(dd[cur], dP + v.w_off[l], dd[cur ^ 1], v.in[l], v.out[l], static_cast<int>(n), S.st),
               "input gradient");
            cur ^= 1;
            col -= static_cast<size_t>(v.in[l]);
        }
        S.download(grads, dG, v.n_params);
        S.download(loss, dloss, 1);
        S.sync();
    });
}

ferret_status ferret_net_apply_sgd(double* params, const double* grads, size_t n, double lr) {
    return guarded([&] {
        if (!n) return;
        if (!params || !grads) fail(FERRET_E_INVALID_ARG, "apply_sgd: null buffer");
        Scratch S;
        double* dp = S.upload(params, n);
        const double* dg = S.upload(grads, n);
        ck(fb200::nm_sgd(dp, dg, n, lr, S.st), "apply_sgd");
        S.download(params, dp, n);
        S.sync();
    });
}

}  // extern "C"
