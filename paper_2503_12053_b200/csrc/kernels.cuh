// Device kernels of the ferret-b200 trainer and their launch arguments.
//
// The trainer (trainer.cpp) compiles the event log into kernel launches with
// every device pointer resolved on the host. Kernels are SIMT fp32: at
// micro-batch B <= 16 every stage op is a skinny GEMM (arithmetic intensity
// ~B/4 flop/byte, far below the ~200 flop/byte tensor-core ridge), so the
// bound is memory — HBM for large stages, L2 + latency for the small nets of
// configs 1-4 — and the design goal is grid-wide parallelism with coalesced
// float4 streaming of weights and version slots.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda.h>
#include <cuda_runtime.h>

namespace fb200 {

constexpr int kMaxBatch = 16;      // micro-batch ceiling (register accumulators per sample)
constexpr int kMaxStageLayers = 16;
constexpr int kMaxPending = 16;    // pending gradients folded by one update launch
constexpr int kMaxChain = 48;      // parameter versions one update launch may read
constexpr int kMaxVersions = 64;   // chain length of the unit compensation entry

// z[b][r] = act(bias[r] + sum_c W[r][c] * x_b[c])    (reference net.hpp:99-113)
// Split-K CTA tiles: each CTA owns a few output rows, its 8 warps split K.
struct HeadArgs;
struct FwdArgs {
    const float* W;      // out x in, row-major
    const float* bias;   // out
    const float* X;      // base of the input rows
    const int* xidx;     // nullable: input row b is X + xidx[b] * in (replay gather), else X + b * in
    float* Y;            // B x out, row-major
    int in, out, B;
    int relu;
    // fused softmax head on the logits this launch produced (last layer, when one CTA
    // computes every output row — fwd_single_cta): -1 none, else HeadArgs::mode
    int head_mode;
    const int* labels;   // head: label of sample b = labels[b]
    int* pred;           // head mode 0
    float* delta;        // head mode 1 (B x out)
    float scale;         // head mode 1
};

// Softmax head over the last layer (reference net.hpp:115-125, learner.hpp:443-447):
// mode 0: predicted class = first argmax (net.hpp:150-154) -> pred[b]
// mode 1: delta[b][k] = scale * (softmax(z_b)[k] - [k == label_b])
struct HeadArgs {
    const float* logits; // B x n_out
    int n_out, B, mode;
    const int* labels;   // label of sample b: labels[lidx ? lidx[b] : b]
    const int* lidx;     // nullable (replay: pool positions)
    int* pred;
    float* delta;        // B x n_out
    float scale;
};

// d_in[b][c] = mask_b[c] * sum_r W[r][c] * d_out[b][r]   (reference learner.hpp:468-474)
// mask (nullable) = post-activation output of the layer below (ReLU: keep where > 0).
// Column tiles x row splits; warps of a CTA split its rows and reduce in smem;
// with row_splits > 1 the last CTA of a column tile sums the split partials.
struct BwdArgs {
    const float* W;
    const float* d_out;  // B x out
    const float* mask;   // B x in or nullptr
    float* d_in;         // B x in
    int in, out, B;
    int row_splits;
    float* partial;      // row_splits x B x in
    unsigned* counters;  // one per column tile, self-resetting
};

// A contiguous run of update work items inside one stage: the weight matrix
// of a layer (items = out x in/V, V = 4 when rows are float4-aligned) or its
// bias vector (items = out, V = 1).
struct UpdSeg {
    int layer;            // index into the stage's layers (0-based)
    int bias;             // 1 = bias segment
    int vec;              // elements per item (1 or 4)
    int per_row;          // items per row (in / vec) for weight segments
    long long item0;      // first item of this segment
    long long elem0;      // float offset of element 0 inside a stage slot
    int in, out;
    long long xin_off;    // stash offset of the layer input (activation of layer l-1); -1 = net input
    long long dlt_off;    // stash offset of the layer's delta
    long long g_off;      // >= 0: the segment's gradient is materialised in the stash at this offset
                          // (convolutions: conv_wgrad writes it), element (r, c) at g_off + r * in + c
};

// One CTA of the update kernel: `nrows` rows x 256 columns of a layer's
// weights starting at (r0, c0), or 256 consecutive bias elements from r0.
constexpr int kUpdTileCols = 256;
constexpr int kUpdMaxTileRows = 16;
struct UpdTile {
    int seg;    // index into the stage's segment table
    int r0;     // first row (weights) or first bias element
    int nrows;  // rows in this tile (weights) / elements (bias)
    int c0;     // first column (weights)
};

// The tile and its segment's fields in one record: the update kernels need one
// dependent load (not two) before every other address is known.
struct UpdWork {
    long long elem0;      // float offset of the segment's element 0 inside a stage slot
    long long xin_off;    // stash offset of the layer input; -1 = net input
    long long dlt_off;    // stash offset of the layer's delta
    int in, out, bias;
    int r0, nrows, c0;
    long long g_off = -1; // >= 0: materialised gradient in the stash (UpdSeg::g_off of this tile's segment)
};

struct UpdPending {
    const float* stash;   // the unit's stash slot (activations + deltas)
    const float* x0;      // net-input rows of the unit (when the stage holds layer 0)
    int first;            // index of its read version in vers[]
};

// One stage update (reference learner.hpp:491-510 + compensate.hpp:42-130):
// for every parameter, for each pending gradient k (in order):
//   g_k = sum_b delta_k[b][r] * x_k[b][c]   (bias: sum_b delta_k[b][r])
//   out_k = Compensator::apply(g_k, vers[first_k .. nv-1])
// then theta_new = theta_cur - step * sum_k out_k, written to `dst`.
struct UpdArgs {
    int n_segs, B, K, policy;
    int gmat;                // some segment reads a materialised gradient (UpdSeg::g_off)
    int pipe;                // update_iter1_kernel: double-buffered row batches (set by spec_update)
    long long n_items;
    long long n_elems;       // parameters of the stage (chooses the HBM- or latency-shaped kernel)
    const UpdSeg* segs;      // device array
    const UpdTile* tiles;    // device array, one per CTA
    const UpdWork* works;    // the same tiles with their segment fields (one per CTA)
    int n_tiles;
    const UpdWork* works4;   // float4 tiles (4 columns per thread) when every weight row is 16-byte aligned
    int n_tiles4, threads4;  // their CTA count and CTA size
    UpdPending pend[kMaxPending];
    const int* x0idx;        // nullable: net-input row b is x0 + x0idx[b] * x0_ld (replay), else x0 + b * x0_ld
    int x0_ld;
    const float* vers[kMaxChain]; // oldest needed version .. current (vers[nv-1])
    int nv;
    float* dst;              // new version slot
    unsigned short* dst16;   // bf16 fast mode: the slot's bf16 copy read by the tensor-core layers (nullable)
    float* lam_d;   // iter_fisher: lambda - lambda0 (fp32 offset keeps the ~1e-10 drift)
    float* v_r;
    float* v_a;
    float* gap;     // gap policy running mean
    float lambda0, alpha, eta, nu;
    float step;     // lr / K
};

// A GROUP of consecutive iter_fisher updates of one stage (one pending gradient each),
// fused into one launch: update k of the group is learner.hpp:491-510 with the chain
// [vers[first_k] .. version cur0 + k]; the versions after cur0 are the group's own outputs,
// kept in registers, so the chain is read from HBM once for the whole group and the
// compensator state is read and written once. Per element the arithmetic is exactly
// update_iter1_kernel's, update after update (bit-identical results). The trainer forms
// groups while compiling the log (trainer.cpp: pending update groups): a group is emitted
// as late as the first later node that touches one of its resources, so deferring its
// members past the nodes in between never changes what any node reads.
constexpr int kGroupMax = 4;         // updates per group (their unit inputs are staged in smem)
constexpr int kGroupChainMax = 24;   // versions a group spans: HBM chain + its own outputs
constexpr int kGroupRows = 4;        // weight rows per tile (a tile: 4 rows x 128 columns, a thread: one column)
constexpr int kGroupCols = 128;      // weight columns per tile
// A weight segment of a group stage: its tiles are tile0 .. tile0 + ceil(in / kGroupCols) * nrt - 1,
// column block after column block, nrt = ceil(out / kGroupRows) row tiles each (the producer decodes a
// tile's position arithmetically instead of loading its UpdWork)
constexpr int kGroupMaxSegs = 8;
struct GroupSeg {
    long long elem0, xin_off, dlt_off;
    int in, out, tile0, nrt;
};
struct GroupArgs {
    int n_gsegs;
    GroupSeg gseg[kGroupMaxSegs];
    const UpdWork* works;            // the stage's group tiles: weights (<= 4 rows x 128 columns, column
                                     // block major) first, then bias runs of 256
    int n_tiles, n_wtiles;           // all tiles / weight tiles
    int B, G, n0;                    // micro-batch, updates, chain versions read from HBM
    int learn;                       // eta_lambda > 0 (v_r / v_a tracked)
    const float* vers[kGroupChainMax];  // vers[0] = oldest read version ... vers[n0 - 1] = cur0
    UpdPending pend[kGroupMax];      // update k: its unit's stash, net-input rows, first chain index
    float* dst[kGroupMax];           // slot of version cur0 + 1 + k
    unsigned short* dst16[kGroupMax];  // its bf16 copy (bf16 fast mode) or null
    const int* x0idx;
    int x0_ld;
    float* lam_d;
    float* v_r;
    float* v_a;
    float lambda0, alpha, eta, nu, step;
};

// RunningNormalizer over a run of arrivals (reference stream.hpp:307-334):
// fp64, one thread per feature, sequential over items; bit-exact with the host.
struct NormArgs {
    const double* raw;   // n x F
    long long n;
    int F;
    const unsigned long long* count_base;  // device: observations before this chunk
    unsigned long long count_off;          // observations of this chunk before this group
    double* mean;
    double* m2;
    float* out;          // n x F
    int apply_only;      // 1: standardise with the current state, observe nothing (held-out evaluation)
    // two-phase form (spec_welford + spec_standardize): the Welford chain writes
    // the post-observation mean / M2 of every (sample, feature) here, and the
    // standardisation of all samples then runs in parallel
    double* mu_i;        // n x F (nullable: single-kernel form)
    double* m2_i;        // n x F
};

// Replay-pool insertion at an arrival (ReplayBuffer::add, learner.hpp:61-69):
// sample b of the unit goes to pool position dst[b] (>= 0) or is skipped.
struct PoolArgs {
    const float* x;      // B x F normalised rows of the unit
    const int* labels;   // B labels of the unit
    const int* dst;      // B pool positions (or -1), filled per chunk by the host reservoir
    float* pool_x;       // capacity x F
    int* pool_labels;    // capacity
    int B, F;
};

// Stage-to-stage hand-off between ranks (one process per GPU): the sender
// stores the message straight into the receiver's inbox (CUDA-IPC mapped peer
// memory, NVLink on a multi-GPU box) and then publishes flag = epoch with a
// system-scope release; the receiver spins on its flag with acquire loads and
// copies the message into its stash (applying the ReLU mask of its own layer,
// which the sender does not hold).
// Programmatic dependent launch (graph edges of type Programmatic, trainer.cpp GraphBuilder):
// every graph kernel first waits for its upstream kernels' completion and memory flush
// (a no-op without a programmatic upstream), then lets its own dependents launch, so a
// dependent's CTAs are resident and waiting when this kernel drains instead of paying the
// launch latency after it.
#define FB_PDL_ENTRY()                                                  \
    do {                                                                \
        asm volatile("griddepcontrol.wait;" ::: "memory");              \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    } while (0)

struct SendArgs {
    const float* src;
    float* dst;                // peer inbox
    unsigned* flag;            // peer flag
    const unsigned* epoch;     // control block (this chunk's epoch)
    int n;
    const unsigned* ack;       // own memory: the receiver's last consumed epoch of this inbox slot
    unsigned* error;           // own hand-off error word
};
struct RecvArgs {
    const float* src;          // own inbox
    float* dst;
    const float* mask;         // nullable
    unsigned* flag;            // own flag
    const unsigned* epoch;
    int n;
    unsigned* error;           // set to 1 when the flag did not arrive within 10 s (the chunk's results are invalid)
    unsigned* ack;             // the sender's ack slot of this message (peer memory)
};

// A fully resolved kernel launch: the trainer either launches it on a stream
// or adds it to its CUDA graph as a node with explicit dependencies.
struct KernelSpec {
    const void* func = nullptr;
    dim3 grid, block;
    size_t smem = 0;
    alignas(64) unsigned char arg0[2048];  // the kernel's struct argument
    int arg1 = 0;                         // optional trailing int argument
    int nargs = 1;
    // the kernel splits its prologue around griddepcontrol.wait (update_iter1_kernel): it may
    // be the programmatic dependent of the previous update of its stage (trainer.cpp)
    bool chain_pdl = false;
    void* params[2];
    KernelSpec() = default;
    KernelSpec(const KernelSpec&) = delete;
    KernelSpec& operator=(const KernelSpec&) = delete;
    void** kernel_params() {
        params[0] = arg0;
        params[1] = &arg1;
        return params;
    }
};

// Fast precision modes: one dense layer (forward or input-gradient) on the
// tensor cores, tcgen05.mma kind::tf32 on the fp32 weights or kind::f16 on a
// bf16 copy, A streamed by TMA, fp32 accumulator in TMEM (mma.cu).
struct MmaArgs {
    CUtensorMap tmap;      // W (out x in, row-major) as a TMA tensor
    const float* bias;     // forward
    const float* X;        // B operand rows (K-major): row n at X + (xidx ? xidx[n] : n) * ldx
    const int* xidx;
    const float* mask;     // backward: ReLU mask of the layer below (nullable)
    float* Y;              // output: element (m, n) at Y[n * ldy + m]
    int M, K, N, ldx, ldy;
    int katoms, atoms_per_cta, stages;
    int relu, vec;
    int splits;            // CTAs splitting K per M tile
    float* partial;        // split-K scratch: mtiles x splits x 16 x 128 floats
    unsigned* counters;    // one per M tile, zero between launches (self-resetting)
    unsigned long long* stamps;  // nullable: 8 phase timestamps per CTA (measurement)
};
struct MmaLayer {
    const void* W;         // fp32 (tf32 mode) or bf16 weights, out x in row-major
    bool bwd = false;      // false: Y = act(W X + b); true: Y = mask * (W^T X)
    bool bf16 = false;
    bool split = false;    // fp32 weights: 3xTF32 (about fp32 accuracy) instead of plain tf32
    const float* bias = nullptr;
    const float* X = nullptr;
    const int* xidx = nullptr;
    const float* mask = nullptr;
    float* Y = nullptr;
    int in = 0, out = 0, B = 0, relu = 0;
    float* partial = nullptr;     // split-K scratch (MmaGeom::partial_floats), nullable when S == 1
    unsigned* counters = nullptr; // MmaGeom::mtiles zeroed counters
    unsigned long long* stamps = nullptr;
};
struct MmaGeom {
    int mtiles, katoms, S, apc, stages;
    size_t smem;
    size_t partial_floats;
};
bool mma_supported(bool bf16, int in, int out);
MmaGeom mma_geom(bool bf16, bool bwd, int in, int out, bool split = false);
void spec_mma(const MmaLayer& L, KernelSpec& k);

void spec_fwd(const FwdArgs& a, KernelSpec& k);
// true when spec_fwd computes every output row in one CTA (the head can be fused)
bool fwd_single_cta(int in, int out, int B, bool vec);
void spec_head(const HeadArgs& a, KernelSpec& k);
void spec_bwd(const BwdArgs& a, KernelSpec& k);
void spec_update(const UpdArgs& a, KernelSpec& k);
void spec_update_group(const GroupArgs& a, KernelSpec& k);
void spec_normalize(const NormArgs& a, KernelSpec& k);
void spec_welford(const NormArgs& a, KernelSpec& k);
void spec_standardize(const NormArgs& a, KernelSpec& k);
void spec_pool(const PoolArgs& a, KernelSpec& k);
void spec_send(const SendArgs& a, KernelSpec& k);
void spec_recv(const RecvArgs& a, KernelSpec& k);
cudaError_t launch_spec(KernelSpec& k, cudaStream_t s);

// ---------------------------------------------------------------------------
// Convolutional layers (conv.cu; BASELINE config 3 — the reference has no
// convolution; the CPU checker lives with the tests). Activations are
// NCHW per sample, rows of B samples as everywhere else. Each op is an implicit
// GEMM C[M x N] = A[M x K] B[K x N] on 64x64 CTA tiles (fp32 SIMT, 4x4 outputs
// per thread), optionally split over K into `partial` with an ordered
// reduction + epilogue kernel (deterministic):
//   fwd    M = c_out, N = B*h_out*w_out, K = c_in*k*k   Y = act(A B + b + shortcut)
//   dgrad  M = c_in,  N = B*h_in*w_in,   K = c_out*k*k  Y = mask * (A B + skip)
//   wgrad  M = c_out, N = c_in*k*k,      K = B*h_out*w_out   Y = gW (then gb, conv_bgrad)
struct ConvArgs {
    const float* W;      // c_out x c_in x k x k
    const float* bias;   // fwd
    const float* X;      // fwd / wgrad: the layer input rows (B x c_in*h_in*w_in)
    const int* xidx;     // nullable: input row b at X + xidx[b] * in_w (replay gather)
    const float* D;      // dgrad / wgrad: delta at the layer output (masked), B x c_out*h_out*w_out
    float* Y;
    const float* res;    // fwd: block input rows (shortcut); dgrad: delta of the residual layer above (skip)
    int rc, rh, rw;      // fwd: block input c/h/w; dgrad: the residual layer's output c/h/w
    const float* mask;   // dgrad: output of the layer below (ReLU mask), nullable
    int relu;
    int B, ci, hi, wi, co, ho, wo, k, s, p;
    int M, N, K, splits, kchunk;
    float* partial;      // splits x M x N (splits > 1)
    // tensor cores (conv_mma_kernel): 0 = SIMT FFMA; 1 = tcgen05 kind::tf32; 2 = kind::f16
    // on bf16 operands; 3 = 3xTF32 (fp32-accurate: the fp32 parity mode)
    int tc;
    int apc;             // tensor-core path: 128-byte K atoms per split
    const float* Wt;     // kt: the weights as the A operand rows in (tap, channel) order, M x K
                         // (spec_conv_wprep writes it before the GEMM): 16-byte copies instead of a
                         // stride-k*k gather
    unsigned long long* stamps;  // nullable: 8 globaltimer phase stamps per CTA (measurement)
    int dbg;             // measurement only (FERRET_CONV_DBG): 1 = skip the A copies, 2 = skip the B copies
    int bcol;            // tensor-core wgrad: GEMM column N-1 is the bias gradient (a ones column of B),
                         // written at Y + M * (N - 1) + m (after the M x (N-1) weight gradient)
    int kt;              // tensor-core fwd / dgrad: K ordered (tap, channel) instead of (channel, tap),
                         // when the channel count is a multiple of the atom: a thread's run of k is
                         // one tap's consecutive channels (one bounds check, constant address step)
};
enum { kConvFwd = 0, kConvDgrad = 1, kConvWgrad = 2 };
// fills M, N, K, splits, kchunk for the op; returns the partial floats needed
size_t conv_plan(ConvArgs& a, int mode, size_t max_partial);
// one or two kernels (GEMM, then the ordered split reduction + epilogue)
int spec_conv(const ConvArgs& a, int mode, KernelSpec& gemm, KernelSpec& reduce);
// kt paths: Wt (M x K, tap-major) from W, one small transpose per GEMM launch
void spec_conv_wprep(const ConvArgs& a, int mode, KernelSpec& k);  // writes a.Wt
// gb[co] = sum over samples and pixels of D (wgrad's bias part), written at Y
void spec_conv_bgrad(const ConvArgs& a, float* gb, KernelSpec& k);
// global average pool (GAP_DENSE input): pooled[b][c] = mean_p x[b][c][p]
struct PoolMeanArgs {
    const float* X;
    const int* xidx;
    float* Y;            // B x C
    float* dX;           // unpool: d_in[b][c][p] = mask * dY[b][c] / HW
    const float* dY;
    const float* mask;
    int B, C, HW;
};
void spec_gap(const PoolMeanArgs& a, KernelSpec& k);
void spec_ungap(const PoolMeanArgs& a, KernelSpec& k);
// grid geometry of the bwd launcher (for scratch sizing)
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
