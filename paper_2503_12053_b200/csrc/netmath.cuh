// Launchers of the fp64 dense-net math kernels (netmath.cu). Device pointers,
// row-major; see netmath.cu for the reference lines each one restates.
#pragma once

#include <cstddef>

#include <cuda_runtime.h>

namespace fb200 {

cudaError_t nm_affine(const double* W, const double* b, const double* X, long long ldx, double* Z, long long ldz,
                      int in, int out, int n, int relu, cudaStream_t st);
cudaError_t nm_relu(double* z, size_t n, cudaStream_t st);
cudaError_t nm_softmax(const double* Z, long long ldz, int k, int n, double* P, const unsigned long long* labels,
                       double inv_n, double* logp, double* delta, cudaStream_t st);
cudaError_t nm_loss(const double* logp, int n, double inv_n, double* loss, cudaStream_t st);
cudaError_t nm_mask(double* delta, const double* act, long long lda, int out, int n, cudaStream_t st);
cudaError_t nm_wgrad(const double* delta, const double* X, long long ldx, double* gW, double* gb, int in, int out,
                     int n, cudaStream_t st);
cudaError_t nm_dgrad(const double* delta, const double* W, double* prev, int in, int out, int n, cudaStream_t st);
cudaError_t nm_sgd(double* p, const double* g, size_t n, double lr, cudaStream_t st);
// Compensator::apply (learner.hpp:97-120) in fp64: chain = chain_len device pointers (any
// length), oldest first; state arrays updated in place (NULL where the policy has none)
cudaError_t nm_compensate(int policy, const double* g, const double* const* chain, int chain_len, double* lambda,
                          double* v_r, double* v_a, double* mean_gap, size_t n, double lambda0, double alpha,
                          double eta, double nu, double* out, cudaStream_t st);

}  // namespace fb200
