// The reference's per-sample dense-net math (proj/include/ferret/net.hpp:99-208) on the
// device, in fp64 with the reference's accumulation order: the drop-in's
// detail::affine_forward / apply_activation / softmax, forward_all / predict_logits /
// predict_class, forward_backward and apply_sgd (include/ferret/net.hpp) are thin C++
// wrappers over the C-ABI entries of netmath_api.cpp, which launch these kernels.
//
// Exactness: every sum is one thread's sequential loop in the reference's index order with
// separately rounded products and sums (__dmul_rn / __dadd_rn: no FMA contraction), so
// affine_forward, the weight / bias gradients, the input gradient and apply_sgd are
// bit-identical to the reference's scalar loops. exp / log are CUDA's fp64 functions
// (<= 1-2 ulp from glibc's), so softmax, the loss and — through the softmax delta — the
// gradients agree with the reference to ~1e-15 relative, not bit for bit.
//
// These are the API's standalone entry points; the pipelined trainer's hot path runs the
// fp32 / tensor-core kernels of kernels.cu / mma.cu instead.
#include <cuda_runtime.h>

#include "netmath.cuh"

namespace fb200 {
namespace {

constexpr int kT = 256;

inline unsigned blocks(size_t n) { return static_cast<unsigned>((n + kT - 1) / kT); }

// z[s][r] = act(b[r] + sum_c W[r][c] x[s][c])   net.hpp:99-113 (acc starts at b[r])
__global__ void affine_f64_kernel(const double* __restrict__ W, const double* __restrict__ b,
                                  const double* __restrict__ X, long long ldx, double* __restrict__ Z, long long ldz,
                                  int in, int out, int n, int relu) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= (long long)n * out) return;
    const int s = (int)(i / out), r = (int)(i % out);
    const double* row = W + (size_t)r * in;
    const double* x = X + (size_t)s * ldx;
    double acc = b[r];
    for (int c = 0; c < in; ++c) acc = __dadd_rn(acc, __dmul_rn(row[c], x[c]));
    if (relu) acc = acc > 0.0 ? acc : 0.0;
    Z[(size_t)s * ldz + r] = acc;
}

// v = v > 0 ? v : 0   net.hpp:110-113
__global__ void relu_f64_kernel(double* z, size_t n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) z[i] = z[i] > 0.0 ? z[i] : 0.0;
}

// softmax of one row per thread (max-shifted exp, sequential sum, divide)   net.hpp:115-125;
// with labels: loss term log(max(p[label], 1e-300)) and delta = (p - onehot) * inv_n
// (net.hpp:171-177)
__global__ void softmax_f64_kernel(const double* __restrict__ Z, long long ldz, int k, int n, double* __restrict__ P,
                                   const unsigned long long* __restrict__ labels, double inv_n,
                                   double* __restrict__ logp, double* __restrict__ delta) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const double* z = Z + (size_t)s * ldz;
    double m = z[0];
    for (int i = 1; i < k; ++i)
        if (z[i] > m) m = z[i];
    double* p = P + (size_t)s * k;
    double sum = 0.0;
    for (int i = 0; i < k; ++i) {
        p[i] = exp(__dadd_rn(z[i], -m));
        sum = __dadd_rn(sum, p[i]);
    }
    for (int i = 0; i < k; ++i) p[i] = __ddiv_rn(p[i], sum);
    if (labels) {
        const int y = (int)labels[s];
        logp[s] = log(fmax(p[y], 1e-300));
        double* d = delta + (size_t)s * k;
        for (int i = 0; i < k; ++i) {
            const double v = i == y ? __dadd_rn(p[i], -1.0) : p[i];
            d[i] = __dmul_rn(v, inv_n);
        }
    }
}

// loss = 0; for each sample in order: loss -= inv_n * logp[s]   net.hpp:163,173
__global__ void loss_f64_kernel(const double* logp, int n, double inv_n, double* loss) {
    if (blockIdx.x || threadIdx.x) return;
    double l = 0.0;
    for (int s = 0; s < n; ++s) l = __dadd_rn(l, -__dmul_rn(inv_n, logp[s]));
    *loss = l;
}

// ReLU mask of the layer's output: delta[s][r] = 0 where act[s][r] <= 0   net.hpp:181-183
__global__ void mask_f64_kernel(double* delta, const double* act, long long lda, int out, int n) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= (long long)n * out) return;
    const int s = (int)(i / out), r = (int)(i % out);
    if (act[(size_t)s * lda + r] <= 0.0) delta[(size_t)s * out + r] = 0.0;
}

// gW[r][c] = sum over samples in order of delta[s][r] * input[s][c] (from 0); gb[r] likewise
// net.hpp:184-190 (Gradients::zeros_like, then += per sample)
__global__ void wgrad_f64_kernel(const double* __restrict__ delta, const double* __restrict__ X, long long ldx,
                                 double* __restrict__ gW, double* __restrict__ gb, int in, int out, int n) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nw = (long long)in * out;
    if (i < nw) {
        const int r = (int)(i / in), c = (int)(i % in);
        double g = 0.0;
        for (int s = 0; s < n; ++s) g = __dadd_rn(g, __dmul_rn(delta[(size_t)s * out + r], X[(size_t)s * ldx + c]));
        gW[i] = g;
    } else if (i < nw + out) {
        const int r = (int)(i - nw);
        double g = 0.0;
        for (int s = 0; s < n; ++s) g = __dadd_rn(g, delta[(size_t)s * out + r]);
        gb[r] = g;
    }
}

// prev[s][c] = sum over r in order of delta[s][r] * W[r][c] (from 0)   net.hpp:192-197
__global__ void dgrad_f64_kernel(const double* __restrict__ delta, const double* __restrict__ W,
                                 double* __restrict__ prev, int in, int out, int n) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= (long long)n * in) return;
    const int s = (int)(i / in), c = (int)(i % in);
    const double* d = delta + (size_t)s * out;
    double acc = 0.0;
    for (int r = 0; r < out; ++r) acc = __dadd_rn(acc, __dmul_rn(d[r], W[(size_t)r * in + c]));
    prev[i] = acc;
}

// theta -= lr * g   net.hpp:202-208
__global__ void sgd_f64_kernel(double* p, const double* g, size_t n, double lr) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = __dadd_rn(p[i], -__dmul_rn(lr, g[i]));
}

}  // namespace

cudaError_t nm_affine(const double* W, const double* b, const double* X, long long ldx, double* Z, long long ldz,
                      int in, int out, int n, int relu, cudaStream_t st) {
    affine_f64_kernel<<<blocks((size_t)n * out), kT, 0, st>>>(W, b, X, ldx, Z, ldz, in, out, n, relu);
    return cudaGetLastError();
}

cudaError_t nm_relu(double* z, size_t n, cudaStream_t st) {
    if (n) relu_f64_kernel<<<blocks(n), kT, 0, st>>>(z, n);
    return cudaGetLastError();
}

cudaError_t nm_softmax(const double* Z, long long ldz, int k, int n, double* P, const unsigned long long* labels,
                       double inv_n, double* logp, double* delta, cudaStream_t st) {
    softmax_f64_kernel<<<blocks(n), kT, 0, st>>>(Z, ldz, k, n, P, labels, inv_n, logp, delta);
    return cudaGetLastError();
}

cudaError_t nm_loss(const double* logp, int n, double inv_n, double* loss, cudaStream_t st) {
    loss_f64_kernel<<<1, 32, 0, st>>>(logp, n, inv_n, loss);
    return cudaGetLastError();
}

cudaError_t nm_mask(double* delta, const double* act, long long lda, int out, int n, cudaStream_t st) {
    mask_f64_kernel<<<blocks((size_t)n * out), kT, 0, st>>>(delta, act, lda, out, n);
    return cudaGetLastError();
}

cudaError_t nm_wgrad(const double* delta, const double* X, long long ldx, double* gW, double* gb, int in, int out,
                     int n, cudaStream_t st) {
    wgrad_f64_kernel<<<blocks((size_t)in * out + out), kT, 0, st>>>(delta, X, ldx, gW, gb, in, out, n);
    return cudaGetLastError();
}

cudaError_t nm_dgrad(const double* delta, const double* W, double* prev, int in, int out, int n, cudaStream_t st) {
    dgrad_f64_kernel<<<blocks((size_t)n * in), kT, 0, st>>>(delta, W, prev, in, out, n);
    return cudaGetLastError();
}

cudaError_t nm_sgd(double* p, const double* g, size_t n, double lr, cudaStream_t st) {
    if (n) sgd_f64_kernel<<<blocks(n), kT, 0, st>>>(p, g, n, lr);
    return cudaGetLastError();
}


namespace {
// Compensator::apply per element, the reference's fp64 expressions evaluated left to right
// with separately rounded operations (bit-identical to the host build, which has no FMA):
//   step   g * (1 / (1 + tau))                                    compensate.hpp:107-113
//   gap    g / (1 + |now - read| / max(m, 1e-12)); m = 0.99 m + 0.01 |now - read|
//                                                                 compensate.hpp:117-130, learner.hpp:104-111
//   fisher g + lambda0 g g (now - read)                           compensate.hpp:42-51
//   iter_fisher: the lambda / v_r / v_a step (eta > 0, >= 2 versions), then
//          out += lambda out out (theta_{s+1} - theta_s) over the chain   compensate.hpp:82-104
__global__ void compensate_f64_kernel(int policy, const double* __restrict__ g, const double* const* __restrict__ chain,
                                      int chain_len, double* lambda, double* v_r, double* v_a, double* mean_gap,
                                      size_t n, double lambda0, double alpha, double eta, double nu, double* out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double gi = g[i];
    const double now = chain[chain_len - 1][i], read = chain[0][i];
    const int tau = chain_len - 1;
    double o = gi;
    if (policy == 1) {
        o = __dmul_rn(gi, __ddiv_rn(1.0, __dadd_rn(1.0, static_cast<double>(tau))));
    } else if (policy == 2) {
        const double m = mean_gap[i];
        const double gap = fabs(__dsub_rn(now, read));
        o = __ddiv_rn(gi, __dadd_rn(1.0, __ddiv_rn(gap, fmax(m, 1e-12))));
        mean_gap[i] = __dadd_rn(__dmul_rn(0.99, m), __dmul_rn(0.01, gap));
    } else if (policy == 3) {
        o = __dadd_rn(gi, __dmul_rn(__dmul_rn(__dmul_rn(lambda0, gi), gi), __dsub_rn(now, read)));
    } else if (policy == 4) {
        double lam = lambda[i];
        if (eta > 0.0 && chain_len >= 2 && v_r && v_a) {
            const double one_m_a = __dsub_rn(1.0, alpha);
            double vr = v_r[i], va = v_a[i];
            const double dv_r = __dmul_rn(one_m_a, __dsub_rn(gi, vr));
            const double resid = __dsub_rn(dv_r, __dmul_rn(lam, va));
            const double grad_l = __dadd_rn(__dmul_rn(__dmul_rn(-2.0, resid), va), __dmul_rn(__dmul_rn(2.0, nu), lam));
            lam = __dsub_rn(lam, __dmul_rn(eta, grad_l));
            const double dtheta = __dsub_rn(chain[1][i], chain[0][i]);
            vr = __dadd_rn(__dmul_rn(alpha, vr), __dmul_rn(one_m_a, gi));
            va = __dadd_rn(__dmul_rn(alpha, va), __dmul_rn(__dmul_rn(__dmul_rn(one_m_a, gi), gi), dtheta));
            lambda[i] = lam;
            v_r[i] = vr;
            v_a[i] = va;
        }
        for (int s = 0; s + 1 < chain_len; ++s)
            o = __dadd_rn(o, __dmul_rn(__dmul_rn(__dmul_rn(lam, o), o), __dsub_rn(chain[s + 1][i], chain[s][i])));
    }
    out[i] = o;
}
}  // namespace

cudaError_t nm_compensate(int policy, const double* g, const double* const* chain, int chain_len, double* lambda,
                          double* v_r, double* v_a, double* mean_gap, size_t n, double lambda0, double alpha,
                          double eta, double nu, double* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    compensate_f64_kernel<<<blocks(n), kT, 0, st>>>(policy, g, chain, chain_len, lambda, v_r, v_a, mean_gap, n,
                                                     lambda0, alpha, eta, nu, out);
    return cudaGetLastError();
}

}  // namespace fb200
