// Device kernels of the ferret-b200 trainer and their launch records.
//
// Each struct below is the full argument set of one kernel launch; the trainer
// (trainer.cpp) compiles the event log into a vector of these records with
// every device pointer resolved, then replays them on one CUDA stream (or as
// one CUDA graph). Kernels are SIMT fp32: at micro-batch B <= 16 every
// stage op is a skinny GEMM with arithmetic intensity ~B/4 flop/byte, far
// below the tensor-core ridge (~200 flop/byte), so the roofline is HBM (or L2
// for nets that fit in it) and the design goal is coalesced, vectorised
// streaming of the weights and version slots.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace fb200 {

constexpr int kMaxBatch = 16;      // micro-batch ceiling (one register lane per sample)
constexpr int kMaxStageLayers = 16;
constexpr int kMaxPending = 16;    // pending gradients folded by one update launch
constexpr int kMaxVersions = 64;   // chain length of the unit compensation entry

// z[b][r] = act(bias[r] + sum_c W[r][c] * x_b[c])    (reference net.hpp:99-113)
struct FwdArgs {
    const float* W;      // out x in, row-major
    const float* bias;   // out
    const float* X;      // base of the input rows
    long long xoff[kMaxBatch]; // row b of the input is X + xoff[b] (gather for replay)
    float* Y;            // B x out, row-major
    int in, out, B;
    int relu;
};

// Softmax head over the last layer (reference net.hpp:115-125, learner.hpp:443-447):
// mode 0: predicted class = first argmax (net.hpp:150-154) -> pred[b]
// mode 1: delta[b][k] = scale * (softmax(z_b)[k] - [k == label_b])
struct HeadArgs {
    const float* logits; // B x n_out
    int n_out, B, mode;
    int labels[kMaxBatch];
    int* pred;
    float* delta;        // B x n_out
    float scale;
};

// d_in[b][c] = mask_b[c] * sum_r W[r][c] * d_out[b][r]   (reference learner.hpp:468-474)
// mask (nullable) = post-activation output of the layer below (relu: keep where > 0)
struct BwdArgs {
    const float* W;
    const float* d_out;  // B x out
    const float* mask;   // B x in or nullptr
    float* d_in;         // B x in
    int in, out, B;
    int row_splits;      // grid.y; >1 uses `partial` + `counters` (last CTA reduces)
    float* partial;      // row_splits x B x in
    unsigned* counters;  // one per column tile, self-resetting
};

struct UpdLayer {
    int in, out;
    long long woff, boff;  // float offsets inside a stage slot
    int row0;              // first flat row of this layer in the stage
    long long xin_off;     // stash offset of this layer's input (activation of layer l-1); -1 = net input
    long long dlt_off;     // stash offset of this layer's delta
};

struct UpdPending {
    const float* stash;    // the unit's stash slot (activations + deltas)
    const float* x0;       // net-input rows of the unit (used when the stage holds layer 0)
    long long read_version;
};

// One stage update (reference learner.hpp:491-510 + compensate.hpp:42-130):
// for every parameter, for each pending gradient k (in order):
//   g_k = sum_b delta_k[b][r] * x_k[b][c]   (bias: sum_b delta_k[b][r])
//   out_k = Compensator::apply(g_k, versions read_k .. cur)
// then theta_new = theta_cur - step * sum_k out_k, written to version cur+1.
// Version v of the stage lives in ring slot (v mod depth).
struct UpdArgs {
    int n_layers, total_rows, B, K, policy;
    const UpdLayer* L;       // device array, n_layers entries
    UpdPending pend[kMaxPending];
    int x0_gather;           // 1: net-input row b of pending 0 is x0 + x0off[b] (replay)
    int x0_ld;               // else row b is x0 + b * x0_ld
    long long x0off[kMaxBatch];
    const float* ring;
    long long slot_floats;
    int depth;
    long long cur_version;
    float* lam_d;   // iter_fisher: lambda - lambda0 (fp32 offset keeps the 1e-10 drift exact)
    float* v_r;
    float* v_a;
    float* gap;     // gap policy running mean
    float lambda0, alpha, eta, nu;
    float step;     // lr / K
};

// RunningNormalizer over a run of arrivals (reference stream.hpp:307-334):
// fp64, one thread per feature, sequential over items; bit-exact with the host.
struct NormArgs {
    const double* raw;   // n x F
    long long n;
    int F;
    unsigned long long count0;
    double* mean;
    double* m2;
    float* out;          // n x F
};

void launch_fwd(const FwdArgs& a, cudaStream_t s);
void launch_head(const HeadArgs& a, cudaStream_t s);
void launch_bwd(const BwdArgs& a, cudaStream_t s);
void launch_update(const UpdArgs& a, cudaStream_t s);
void launch_normalize(const NormArgs& a, cudaStream_t s);
// column tiles / rows per split the bwd launcher uses (for scratch sizing)
int bwd_col_tiles(int in);
int bwd_row_splits(int in, int out);

// Unit entry for ferret_compensate (fp32 arrays, absolute lambda).
struct CompArgs {
    int policy;
    const float* g;
    const float* chain[kMaxVersions];
    int chain_len;
    float* lambda;
    float* v_r;
    float* v_a;
    float* gap;
    long long n;
    float lambda0, alpha, eta, nu;
    float* out;
};
void launch_compensate(const CompArgs& a, cudaStream_t s);

} // namespace fb200
