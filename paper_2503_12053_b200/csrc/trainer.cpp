// ferret_trainer: PipelineTrainer (reference learner.hpp:330-526) on one B200.
//
// The reference interprets the simulator's event log one event at a time on
// the host, copying whole nets per event. Here the log is compiled ONCE per
// schedule into a CUDA graph of sm_100a kernels and replayed per stream chunk:
//
//   set_schedule   analyse the log: drops, per-unit last use, which (unit,
//                  stage) backwards exist, which updates fire.
//   build_graph    (first execute) a dry pass sizes the HBM structures — the
//                  per-stage version ring (depth = the longest live chain + 1;
//                  the reference's hold set leaks, learner.hpp:419/507) and the
//                  stash slots (one per in-flight unit, freed at its last use)
//                  — then a second pass launches every kernel in log order
//                  under stream capture. All launch parameters are chunk
//                  invariant: chunk data sit in fixed staging buffers, version
//                  slots are relative to the chunk start (the live version is
//                  moved back to slot 0 at the end of the graph), and the
//                  per-chunk replay decisions are read from device arrays.
//   execute(c)     host: run the replay reservoir over chunk c (the only
//                  stateful host arithmetic, identical RNG draws to
//                  learner.hpp:56-80) and copy its decisions + the chunk's
//                  stream data into the staging buffers; device: one
//                  cudaGraphLaunch.
//
// Everything the north star requires to be bit-exact (routing, schedule,
// replay indices) is decided on the host with the reference's own arithmetic;
// the device does fp32 math plus the fp64 normalizer.
//
// HBM layout: per stage a ring of `depth` version slots (fp32,
// per-layer W/b at 128-byte aligned offsets) and the compensator state of the
// same shape (lambda offset, v_r, v_a or mean_gap); the resident stream
// (fp64 raw, int32 labels, int32 predictions); per chunk the raw/normalised
// staging rows; the stash (per in-flight unit: every layer's activation and
// delta, B x width); the replay pool (capacity x F normalised rows + labels).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cxxabi.h>
#include <functional>
#include <map>
#include <set>
#include <tuple>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "common.hpp"
#include "ferret/rng.hpp"
#include "kernels.cuh"
#include "netmath.cuh"

using fb200::fail;
using fb200::guarded;

namespace {

// Plan-only trainers (device -1) run the host passes without any device: every
// allocation is null and CUDA calls are skipped. Used to check the multi-rank
// hand-off plan on machines without a GPU (tests/test_shard_plan.py).
thread_local bool t_plan_only = false;

struct PlanOnlyScope {
    bool prev;
    explicit PlanOnlyScope(bool on) : prev(t_plan_only) { t_plan_only = on; }
    ~PlanOnlyScope() { t_plan_only = prev; }
};

void cuda_check(cudaError_t e, const char* what) {
    if (t_plan_only) return;
    if (e != cudaSuccess) fail(FERRET_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

long long align_up(long long v, long long a) { return (v + a - 1) / a * a; }

// fp32 -> bf16 bits, round to nearest even (the device's __float2bfloat16_rn)
uint16_t bf16_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);  // NaN stays NaN
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// Plan-only trainers count what they would allocate (ferret_trainer_footprint) and get null.
template <class T>
T* dalloc(size_t n, size_t& counter) {
    void* p = nullptr;
    if (n == 0) n = 1;
    counter += n * sizeof(T);
    if (t_plan_only) return nullptr;
    cuda_check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    return static_cast<T*>(p);
}

void dfree(void* p) {
    if (p) cudaFree(p);
}

// Reservoir over pool positions (reference ReplayBuffer, learner.hpp:56-80):
// the same RNG draws, tracking where each added sample lands instead of the
// sample itself — the normalised rows live in the device pool.
struct Reservoir {
    uint64_t cap = 0;
    ferret::Rng rng{0};
    uint64_t seen = 0;
    uint64_t size = 0;

    Reservoir() = default;
    Reservoir(uint64_t capacity, uint64_t seed) : cap(capacity), rng(seed ^ 0xbf58476d1ce4e5b9ULL) {}

    std::vector<int> label_at;      // label of the sample held at each pool position
    std::vector<int64_t> id_at;     // stream sample index held at each pool position
    std::vector<int64_t> draws;     // stream sample index of every replay draw, in draw order

    int add(int label, int64_t id) {  // pool position the new sample is written to, or -1
        ++seen;
        int pos = -1;
        if (size < cap) {
            pos = static_cast<int>(size++);
        } else {
            const uint64_t at = rng.below(seen);
            if (at < cap) pos = static_cast<int>(at);
        }
        if (pos >= 0) {
            if (label_at.size() <= static_cast<size_t>(pos)) label_at.resize(static_cast<size_t>(pos) + 1);
            label_at[static_cast<size_t>(pos)] = label;
            if (id_at.size() <= static_cast<size_t>(pos)) id_at.resize(static_cast<size_t>(pos) + 1, -1);
            id_at[static_cast<size_t>(pos)] = id;
        }
        return pos;
    }
    int sample() {
        const int pos = static_cast<int>(rng.below(size));
        draws.push_back(static_cast<size_t>(pos) < id_at.size() ? id_at[static_cast<size_t>(pos)] : -1);
        return pos;
    }
};

struct HostState {
    std::vector<long long> current;  // per stage: absolute version of the live parameters
    Reservoir replay;
    uint64_t norm_count = 0;
};

// softmax head fused into the last layer's forward (one CTA computes every logit)
struct Head {
    int mode = -1;  // -1 none, 0 argmax -> pred, 1 scale * (softmax - onehot) -> delta
    const int* labels = nullptr;
    int* pred = nullptr;
    float* delta = nullptr;
    float scale = 1.f;
};

struct LayerDev {
    int in = 0, out = 0, act = 0, stage = 0;  // in / out: activation widths (c*h*w for convolutions)
    long long woff = 0, boff = 0;        // inside the stage slot
    long long host_off = 0;              // in flatten() order of the whole net
    long long act_off = 0, dlt_off = 0;  // inside a stash slot
    // convolutional extension (ferret_b200.h FERRET_LAYER_*); dense layers: kind 0,
    // rows = out, cols = in
    int kind = FERRET_LAYER_DENSE;
    int ci = 0, hi = 1, wi = 1, co = 0, ho = 1, wo = 1, k = 1, st = 1, pad = 0, res = 0;
    int rows = 0, cols = 0;              // parameter matrix: rows x cols, then rows biases
    long long g_off = -1;                // conv: materialised gradient (rows x cols, then rows) in a stash slot
    long long pool_off = -1, pdl_off = -1;  // gap_dense: pooled input and its delta (B x ci) in a stash slot
    long long nw() const { return static_cast<long long>(rows) * cols; }
    bool conv() const { return kind == FERRET_LAYER_CONV; }
    bool gap() const { return kind == FERRET_LAYER_GAP_DENSE; }
};

struct StageDev {
    int lo = 0, hi = 0;
    long long n_params = 0, slot_floats = 0, host_off = 0;
    int depth = 0;
    float* ring = nullptr;
    uint16_t* ring16 = nullptr;  // bf16 fast mode: bf16 copy of every ring slot (tensor-core operand)
    float* lam_d = nullptr;
    float* v_r = nullptr;
    float* v_a = nullptr;
    float* gap = nullptr;
    fb200::UpdSeg* segs_dev = nullptr;
    int n_segs = 0;
    bool gmat = false;  // holds a convolution: its update reads materialised gradients
    fb200::UpdTile* tiles_dev = nullptr;
    fb200::UpdWork* works_dev = nullptr;
    fb200::UpdWork* works4_dev = nullptr;  // float4 tiles (nullptr when a weight row is not 16-byte aligned)
    int n_tiles4 = 0, threads4 = 0;
    int n_tiles = 0;
    fb200::UpdWork* works_g_dev = nullptr;  // update-group tiles (kernels.cuh GroupArgs::works)
    int n_tiles_g = 0, n_wtiles_g = 0;
    std::vector<fb200::GroupSeg> gsegs;  // the weight segments' tile ranges (GroupArgs::gseg)
    bool group_ok = false;  // update groups apply: a large dense stage with 16-byte aligned weight rows
    long long n_items = 0;
    // slot of a version counted from the chunk start (the live version is in slot 0 between chunks)
    float* slot(long long rel) const { return ring + (rel % depth) * slot_floats; }
    // the bf16 copy of the slot a float pointer into the ring lies in
    const uint16_t* shadow(const float* p) const { return ring16 + (p - ring); }
};

// Schedule facts independent of the mutable state (computed once per log).
struct Schedule {
    std::vector<ferret_event> events;
    size_t n_units = 0;
    size_t chunk_items = 0;                    // stream samples per execute()
    std::vector<char> dropped;                 // per unit
    std::vector<char> has_bwd;                 // per unit x stage
    std::vector<char> update_fires;            // per event: an update with pending gradients
    std::vector<std::vector<size_t>> free_at;  // per event index: units whose stash frees after it
};

// What the device graph needs from the host for one chunk.
struct ChunkPlan {
    std::vector<int> pool_dst;  // per chunk sample: replay-pool position or -1
    std::vector<int> rep_ids;   // per replay step x B: pool positions sampled
    std::vector<int> rep_labels;  // their labels
    size_t n_replays = 0;
};

// Builds the chunk graph as a DAG. Every node declares the HBM resources it
// reads and writes; it depends on the last writer of each (RAW/WAW) and, for
// writes, on the readers since that writer (WAR). Events that touch disjoint
// resources — different stages, different in-flight units — therefore run
// concurrently, which is the pipeline parallelism of the 1F1B schedule
// realised on one GPU. `serial` chains every node instead (timing mode).
struct GraphBuilder {
    // kAct / kDlt: one unit stash slot's activations / deltas of one stage's layers
    // (key(kind, slot, stage)): a stage's update reads its own deltas and activations while
    // the backward of the stage below writes only that stage's deltas
    enum : uint64_t { kVSlot = 1, kState, kStash, kPred, kNorm, kNormState, kPool, kReplay, kNormScratch, kWt, kAct, kDlt };
    static uint64_t key(uint64_t kind, uint64_t a, uint64_t b = 0) { return (kind << 56) | (a << 32) | b; }

    cudaGraph_t g = nullptr;
    bool serial = false;
    // FERRET_PDL=1: kernel -> kernel edges programmatic (A/B knob). Off: measured C2 1.12M ->
    // 0.85M samples/s (graph launch dearer, early-resident CTAs crowd the concurrent DAG),
    // C5 and C3 neutral (profiles/r2/pdl_ab.txt)
    bool pdl = std::getenv("FERRET_PDL") && std::atoi(std::getenv("FERRET_PDL")) != 0;
    // the next kernel node's programmatic upstream when the kernel supports it (KernelSpec::chain_pdl):
    // the previous update of the same stage (set by the trainer, consumed by kernel())
    int pdl_pred = -1;
    cudaGraphNode_t last = nullptr;
    uint64_t kernels = 0;
    // Logical DAG (node index = creation order), kept in both modes: the
    // profile mode (serial graph, events around every node) uses it to
    // compute the critical path the concurrent graph is bound by.
    std::vector<std::vector<int>> ldeps;
    std::vector<int> category;
    int cur_category = 0;
    int cur_stage = -1;           // pipeline stage the next node works for (-1: none)
    double cur_bytes = 0.0;       // algorithmic HBM bytes of the next node (set by the emitter)
    std::vector<double> bytes;
    std::vector<int> stage_of;
    const void* cur_func = nullptr;  // kernel of the next node (null: copy / memset / event)
    std::vector<const void*> funcs;
    struct Res {
        int writer = -1;
        std::vector<int> readers;
    };
    std::map<uint64_t, Res> res;
    std::vector<cudaGraphNode_t> nodes;
    // profiling: an event before and after every node
    std::vector<cudaEvent_t>* prof_events = nullptr;

    explicit GraphBuilder(bool serial_) : serial(serial_) { cuda_check(cudaGraphCreate(&g, 0), "cudaGraphCreate"); }
    // Long logs: the graph is cut into segments launched in stream order, so every
    // dependency across a cut is honoured by the stream; only the concurrency across
    // the cut is lost. done_segments holds the finished graphs, g the open one.
    std::vector<cudaGraph_t> done_segments;
    size_t seg_first_node = 0;
    size_t nodes_in_segment() const { return nodes.size() - seg_first_node; }
    void new_segment() {
        done_segments.push_back(g);
        cuda_check(cudaGraphCreate(&g, 0), "cudaGraphCreate");
        res.clear();
        last = nullptr;
        seg_first_node = nodes.size();
    }
    explicit GraphBuilder(cudaStream_t s) : eager(s) {}
    ~GraphBuilder() {
        if (g) cudaGraphDestroy(g);
        for (cudaGraph_t x : done_segments) cudaGraphDestroy(x);
    }

    std::vector<int> logical(const std::vector<uint64_t>& reads, const std::vector<uint64_t>& writes) {
        std::vector<int> d;
        for (uint64_t r : reads) {
            auto it = res.find(r);
            if (it != res.end() && it->second.writer >= 0) d.push_back(it->second.writer);
        }
        for (uint64_t w : writes) {
            auto it = res.find(w);
            if (it == res.end()) continue;
            if (it->second.writer >= 0) d.push_back(it->second.writer);
            d.insert(d.end(), it->second.readers.begin(), it->second.readers.end());
        }
        std::sort(d.begin(), d.end());
        d.erase(std::unique(d.begin(), d.end()), d.end());
        return d;
    }

    std::vector<cudaGraphNode_t> deps(const std::vector<int>& ld) {
        std::vector<cudaGraphNode_t> d;
        if (serial) {
            if (last) d.push_back(last);
            if (prof_events) {  // event before the node
                const size_t i = nodes.size();
                while (prof_events->size() < 2 * i + 2) {
                    cudaEvent_t e;
                    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
                    prof_events->push_back(e);
                }
                cudaGraphNode_t n;
                cuda_check(cudaGraphAddEventRecordNode(&n, g, d.data(), d.size(), (*prof_events)[2 * i]),
                           "cudaGraphAddEventRecordNode");
                d.assign(1, n);
            }
            return d;
        }
        for (int x : ld) d.push_back(nodes[static_cast<size_t>(x)]);
        return d;
    }

    void commit(cudaGraphNode_t n, const std::vector<int>& ld, const std::vector<uint64_t>& reads,
                const std::vector<uint64_t>& writes) {
        const int idx = static_cast<int>(nodes.size());
        nodes.push_back(n);
        ldeps.push_back(ld);
        category.push_back(cur_category);
        bytes.push_back(cur_bytes);
        stage_of.push_back(cur_stage);
        funcs.push_back(cur_func);
        cur_bytes = 0.0;
        cur_func = nullptr;
        last = n;
        if (serial && prof_events) {  // event after the node
            cudaGraphNode_t e;
            cuda_check(cudaGraphAddEventRecordNode(&e, g, &n, 1, (*prof_events)[2 * static_cast<size_t>(idx) + 1]),
                       "cudaGraphAddEventRecordNode");
            last = e;
        }
        for (uint64_t r : reads) res[r].readers.push_back(idx);
        for (uint64_t w : writes) {
            Res& x = res[w];
            x.writer = idx;
            x.readers.clear();
        }
    }

    // eager mode (sequential learners): launch on this stream instead of adding
    // graph nodes (the caller may be capturing the stream into a graph)
    cudaStream_t eager = nullptr;

    // Called before a node is added with the resources it will read and write (the
    // trainer's pending update groups flush themselves here on a conflict). The
    // emitter's next-node fields are preserved across the call.
    std::function<void(const std::vector<uint64_t>&, const std::vector<uint64_t>&)> before;
    bool in_before = false;
    void check_before(const std::vector<uint64_t>& reads, const std::vector<uint64_t>& writes) {
        if (!before || in_before) return;
        in_before = true;
        const int cc = cur_category, cs = cur_stage;
        const double cb = cur_bytes;
        before(reads, writes);
        cur_category = cc;
        cur_stage = cs;
        cur_bytes = cb;
        in_before = false;
    }

    cudaGraphNode_t kernel(fb200::KernelSpec& k, const std::vector<uint64_t>& reads, const std::vector<uint64_t>& writes) {
        if (eager) {
            cuda_check(fb200::launch_spec(k, eager), "kernel launch");
            ++kernels;
            cur_bytes = 0.0;
            return nullptr;
        }
        check_before(reads, writes);
        const std::vector<int> ld = logical(reads, writes);
        // kernel -> kernel edges are programmatic (every kernel starts with FB_PDL_ENTRY:
        // griddepcontrol.wait, then launch_dependents), so this node's CTAs launch while its
        // upstream kernels drain; edges from copies / events stay full dependencies
        std::vector<int> normal, prog;
        const int chain_pred = k.chain_pdl && !serial ? pdl_pred : -1;
        pdl_pred = -1;
        for (int x : ld)
            ((pdl && !serial && funcs[static_cast<size_t>(x)]) || x == chain_pred ? prog : normal).push_back(x);
        const std::vector<cudaGraphNode_t> d = deps(normal);
        cudaKernelNodeParams p{};
        p.func = const_cast<void*>(k.func);
        p.gridDim = k.grid;
        p.blockDim = k.block;
        p.sharedMemBytes = static_cast<unsigned>(k.smem);
        p.kernelParams = k.kernel_params();
        cudaGraphNode_t n;
        cuda_check(cudaGraphAddKernelNode(&n, g, d.data(), d.size(), &p), "cudaGraphAddKernelNode");
        for (int x : prog) {
            cudaGraphEdgeData e{};
            e.from_port = cudaGraphKernelNodePortProgrammatic;
            e.type = cudaGraphDependencyTypeProgrammatic;
            cuda_check(cudaGraphAddDependencies_v2(g, &nodes[static_cast<size_t>(x)], &n, &e, 1), "programmatic edge");
        }
        cur_func = k.func;
        // FERRET_NODE_PRIORITY=<class digits>: those node classes (1 predict, 2 forward,
        // 3 backward, 4 update) run at the device's highest kernel priority, so the
        // per-stage version chain (the DAG's critical path) is not queued behind others
        static const char* prio = std::getenv("FERRET_NODE_PRIORITY");
        if (prio && std::strchr(prio, '0' + cur_category)) {
            int lo = 0, hi = 0;
            cudaDeviceGetStreamPriorityRange(&lo, &hi);
            cudaKernelNodeAttrValue v{};
            v.priority = hi;
            cuda_check(cudaGraphKernelNodeSetAttribute(n, cudaKernelNodeAttributePriority, &v), "node priority");
        }
        commit(n, ld, reads, writes);
        ++kernels;
        return n;
    }

    cudaGraphNode_t copy(void* dst, const void* src, size_t bytes, const std::vector<uint64_t>& reads,
                         const std::vector<uint64_t>& writes) {
        if (eager) {
            cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, eager), "cudaMemcpyAsync");
            return nullptr;
        }
        check_before(reads, writes);
        const std::vector<int> ld = logical(reads, writes);
        const std::vector<cudaGraphNode_t> d = deps(ld);
        cudaGraphNode_t n;
        cuda_check(cudaGraphAddMemcpyNode1D(&n, g, d.data(), d.size(), dst, src, bytes, cudaMemcpyDeviceToDevice),
                   "cudaGraphAddMemcpyNode1D");
        commit(n, ld, reads, writes);
        return n;
    }

    // event record node after `last` (serial mode only: brackets a kernel)
    void event(cudaEvent_t e) {
        cudaGraphNode_t n;
        cuda_check(cudaGraphAddEventRecordNode(&n, g, last ? &last : nullptr, last ? 1 : 0, e), "cudaGraphAddEventRecordNode");
        last = n;
    }
};

// node classes reported by the profile mode
enum { kCatNorm = 0, kCatPredict, kCatForward, kCatBackward, kCatUpdate, kCatReplay, kCatOther, kNumCat };

struct PassResult {
    std::vector<size_t> inbox_bytes, inbox_flags;  // per rank: incoming message bytes / flags per chunk
    std::vector<int> need_depth;
    std::vector<long long> pushes;
    int need_slots = 0;
    size_t n_replays = 0;
    size_t n_updates_timed = 0;
};

} // namespace

struct ferret_trainer {
    ferret_train_opts opt{};
    int B = 1, P = 0, L = 0, F = 0, n_out = 0;
    std::vector<LayerDev> layers;
    std::vector<StageDev> stages;
    std::vector<double> init_params;
    std::vector<int32_t> geom;  // conv nets: the descriptor's geometry (empty: all dense)

    // FERRET_LAYER_* geometry of layer l (ferret_b200.h), checked against the widths
    void set_geometry(LayerDev& ld, int l, const int32_t* q) {
        const std::string at = "layer " + std::to_string(l) + ": ";
        ld.kind = q[0];
        const long long in_w = static_cast<long long>(q[1]) * q[2] * q[3];
        if (q[1] < 1 || q[2] < 1 || q[3] < 1 || q[4] < 1) fail(FERRET_E_CONFIG, at + "geometry sizes must be positive");
        if (in_w != ld.in) fail(FERRET_E_CONFIG, at + "c_in*h_in*w_in differs from the input width");
        ld.ci = q[1];
        ld.hi = q[2];
        ld.wi = q[3];
        ld.co = q[4];
        ld.res = q[8];
        if (ld.kind == FERRET_LAYER_CONV) {
            ld.k = q[5];
            ld.st = q[6];
            ld.pad = q[7];
            if (ld.k < 1 || ld.st < 1 || ld.pad < 0) fail(FERRET_E_CONFIG, at + "bad convolution geometry");
            ld.ho = (ld.hi + 2 * ld.pad - ld.k) / ld.st + 1;
            ld.wo = (ld.wi + 2 * ld.pad - ld.k) / ld.st + 1;
            if (ld.ho < 1 || ld.wo < 1) fail(FERRET_E_CONFIG, at + "empty convolution output");
            if (static_cast<long long>(ld.co) * ld.ho * ld.wo != ld.out)
                fail(FERRET_E_CONFIG, at + "c_out*h_out*w_out differs from the output width");
            ld.rows = ld.co;
            ld.cols = ld.ci * ld.k * ld.k;
        } else if (ld.kind == FERRET_LAYER_DENSE || ld.kind == FERRET_LAYER_GAP_DENSE) {
            if (ld.co != ld.out) fail(FERRET_E_CONFIG, at + "c_out differs from the output width");
            if (ld.kind == FERRET_LAYER_DENSE && (ld.hi != 1 || ld.wi != 1))
                fail(FERRET_E_CONFIG, at + "a dense layer has h_in = w_in = 1");
            ld.rows = ld.co;
            ld.cols = ld.ci;
        } else {
            fail(FERRET_E_CONFIG, at + "unknown layer kind");
        }
        if (ld.res) {
            if (!ld.conv() || l < 2 || !layers[static_cast<size_t>(l - 1)].conv())
                fail(FERRET_E_CONFIG, at + "a residual layer is the second convolution of a block after layer 1");
            const LayerDev& a = layers[static_cast<size_t>(l - 1)];
            if (a.ci > ld.co || a.hi % ld.ho != 0 || a.wi % ld.wo != 0 || a.hi / ld.ho != a.wi / ld.wo)
                fail(FERRET_E_CONFIG, at + "residual shortcut shape");
        }
    }
    cudaStream_t stream = nullptr;
    cudaStream_t nstream = nullptr;  // side stream: the normalizer runs ahead of training
    static constexpr size_t kNormGroup = 16;
    std::vector<cudaEvent_t> norm_events;
    cudaEvent_t fork_event = nullptr;
    size_t device_bytes = 0;

    // resident stream
    double* d_raw = nullptr;
    int* d_lab = nullptr;
    int* d_pred = nullptr;
    size_t n_loaded = 0;
    std::vector<int> labels;
    double* d_norm_mean = nullptr;
    double* d_norm_m2 = nullptr;

    // per-chunk staging (fixed addresses baked into the graph)
    size_t chunk_cap = 0;
    size_t stream_cap = 0;  // samples the resident-stream buffers hold
    double* d_rawc = nullptr;
    double* d_norm_mu = nullptr;   // per chunk sample x feature: mean / M2 after observing it (two-phase normalizer)
    double* d_norm_m2i = nullptr;
    float* d_xc = nullptr;
    int* d_labc = nullptr;
    int* d_predc = nullptr;
    // control block: [count_base u64][pool_dst chunk_cap x i32][rep_ids max_rep x B x i32]
    unsigned char* d_ctl = nullptr;
    std::vector<unsigned char*> h_ctl;  // pinned, double-buffered
    std::vector<cudaEvent_t> ctl_done;
    size_t ctl_bytes = 0, max_rep = 0;
    int ctl_flip = 0;

    // replay pool
    float* d_pool_x = nullptr;
    int* d_pool_lab = nullptr;

    // scratch
    float* d_stash = nullptr;
    long long stash_stride = 0;
    int stash_slots = 0;
    long long pred_off = 0;       // predict ping-pong scratch (2 x B x max_width) inside a stash slot
    long long pred_stride = 0;
    float* d_replay = nullptr;    // one stash-shaped slot
    // bwd split-reduction scratch, one region per stash slot (+1 for replay) so
    // that concurrent backwards of different units never share it
    float* d_partial = nullptr;
    unsigned* d_counters = nullptr;
    size_t max_partial = 1, max_tiles = 1;
    int scratch_slots = 0;
    GraphBuilder* gb = nullptr;   // set while the graph is being built
    bool plan_only = false;       // created with device -1: host passes only
    void require_device_mode() const {
        if (plan_only) fail(FERRET_E_NO_DEVICE, "plan-only trainer (device -1) cannot run device work");
    }

    // stage sharding across ranks (one process per GPU); world 1 = everything local
    int rank = 0, world = 1;
    std::vector<int> owner;                 // per stage: owning rank
    bool mine(int j) const { return owner[static_cast<size_t>(j)] == rank; }
    unsigned char* d_inbox = nullptr;       // this rank's incoming hand-offs: data, then flags
    size_t inbox_alloc = 0;
    std::vector<size_t> inbox_data_bytes;   // per rank: data bytes (flags follow, 256-aligned)
    std::vector<float*> peer_data;          // per rank: inbox data base (own included)
    std::vector<unsigned*> peer_flags;
    std::vector<void*> peer_opened;         // IPC mappings to close
    std::vector<unsigned*> peer_acks;       // per rank: its ack region (own rank: this rank's)
    std::vector<size_t> inbox_flag_counts;  // per rank: incoming messages per chunk
    std::vector<size_t> ack_off;            // per destination: first ack slot of messages to it
    unsigned epoch_counter = 0;

    void set_shard(int r, int w, const int32_t* own) {
        if (w < 1 || r < 0 || r >= w) fail(FERRET_E_CONFIG, "shard: rank must lie in [0, world)");
        for (int j = 0; j < P; ++j)
            if (own[j] < 0 || own[j] >= w) fail(FERRET_E_CONFIG, "shard: stage owner out of range");
        for (int j = 1; j < P; ++j)
            if (own[j] < own[j - 1]) fail(FERRET_E_CONFIG, "shard: stages must be assigned to ranks in order");
        if (own[0] != 0) fail(FERRET_E_CONFIG, "shard: stage 0 (the stream input) must live on rank 0");
        rank = r;
        world = w;
        owner.assign(own, own + P);
        peer_data.assign(static_cast<size_t>(w), nullptr);
        peer_flags.assign(static_cast<size_t>(w), nullptr);
        peer_acks.assign(static_cast<size_t>(w), nullptr);
        have_schedule = false;
        invalidate_graph();
    }

    // Size and allocate this rank's inbox from the message plan of the log.
    // last word of the inbox allocation: a receive that timed out sets it
    unsigned* handoff_error() const {
        return d_inbox ? reinterpret_cast<unsigned*>(d_inbox + inbox_alloc - sizeof(unsigned)) : nullptr;
    }
    void check_handoffs() {
        if (world == 1 || !d_inbox || plan_only) return;
        unsigned e = 0;
        cuda_check(cudaMemcpy(&e, handoff_error(), sizeof(e), cudaMemcpyDeviceToHost), "D2H hand-off status");
        if (e) fail(FERRET_E_CUDA, "stage hand-off timed out: a peer rank did not deliver within 10 s");
    }

    void setup_inbox() {
        if (world == 1) return;
        HostState probe = hs;
        const PassResult plan = run_pass<true>(probe, false);
        inbox_data_bytes = plan.inbox_bytes;
        inbox_flag_counts = plan.inbox_flags;
        // layout: [incoming message data][incoming flags][acks of this rank's outgoing
        // messages, per destination d: inbox_flags[d] slots][pad; last word: error]
        ack_off.assign(static_cast<size_t>(world), 0);
        size_t n_acks = 0;
        for (int d = 0; d < world; ++d) {
            ack_off[static_cast<size_t>(d)] = n_acks;
            n_acks += inbox_flag_counts[static_cast<size_t>(d)];
        }
        const size_t data = (inbox_data_bytes[static_cast<size_t>(rank)] + 255) / 256 * 256;
        const size_t need = data + (plan.inbox_flags[static_cast<size_t>(rank)] + n_acks) * sizeof(unsigned) + 256;
        cuda_check(cudaStreamSynchronize(stream), "sync");
        if (need > inbox_alloc) {
            dfree(d_inbox);
            d_inbox = dalloc<unsigned char>(need, device_bytes);
            inbox_alloc = need;
        }
        // every schedule change re-opens the peers: a peer may have reallocated its inbox, and
        // the flag offsets inside it follow the new plan's data size (stale mappings would
        // publish flags at the old plan's positions)
        for (size_t p = 0; p < peer_opened.size(); ++p)
            if (peer_opened[p]) cudaIpcCloseMemHandle(peer_opened[p]);
        peer_opened.assign(static_cast<size_t>(world), nullptr);
        std::fill(peer_data.begin(), peer_data.end(), nullptr);
        std::fill(peer_flags.begin(), peer_flags.end(), nullptr);
        peer_acks.assign(static_cast<size_t>(world), nullptr);
        invalidate_graph();
        cuda_check(cudaMemset(d_inbox, 0, inbox_alloc), "memset inbox");  // flags and acks start at epoch 0
        epoch_counter = 0;  // every rank re-sets its schedule together: epochs restart in step
        peer_data[static_cast<size_t>(rank)] = reinterpret_cast<float*>(d_inbox);
        peer_flags[static_cast<size_t>(rank)] = reinterpret_cast<unsigned*>(d_inbox + data);
        peer_acks[static_cast<size_t>(rank)] = peer_flags[static_cast<size_t>(rank)] + plan.inbox_flags[static_cast<size_t>(rank)];
    }

    void open_peer(int p, const void* handle) {
        if (p < 0 || p >= world || p == rank) fail(FERRET_E_INVALID_ARG, "open_peer: bad peer rank");
        if (inbox_data_bytes.empty()) fail(FERRET_E_LOGIC, "open_peer: set_schedule first");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        void* ptr = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        if (peer_opened.size() < static_cast<size_t>(world)) peer_opened.resize(static_cast<size_t>(world), nullptr);
        if (peer_opened[static_cast<size_t>(p)]) cudaIpcCloseMemHandle(peer_opened[static_cast<size_t>(p)]);
        peer_opened[static_cast<size_t>(p)] = ptr;
        const size_t data = (inbox_data_bytes[static_cast<size_t>(p)] + 255) / 256 * 256;
        peer_data[static_cast<size_t>(p)] = static_cast<float*>(ptr);
        peer_flags[static_cast<size_t>(p)] = reinterpret_cast<unsigned*>(static_cast<unsigned char*>(ptr) + data);
        peer_acks[static_cast<size_t>(p)] = peer_flags[static_cast<size_t>(p)] + inbox_flag_counts[static_cast<size_t>(p)];
        invalidate_graph();
    }

    HostState hs;
    Schedule sched;
    bool have_schedule = false;

    // the compiled graph of the current schedule
    cudaGraphExec_t graph_exec = nullptr;
    std::vector<cudaGraphExec_t> more_execs;  // further segments of a long log, launched after graph_exec
    // nodes per graph segment (FERRET_GRAPH_SEGMENT_NODES overrides; tests use small values)
    size_t seg_nodes = std::getenv("FERRET_GRAPH_SEGMENT_NODES")
                           ? static_cast<size_t>(std::atoll(std::getenv("FERRET_GRAPH_SEGMENT_NODES")))
                           : static_cast<size_t>(65536);
    bool graph_timing = false;
    bool graph_seen_any = false;  // reservoir non-empty at chunk start when captured
    PassResult graph_shape;

    ferret_trainer_stats stats{};
    uint64_t launches = 0;

    // profile mode: serial graph with events around every node + the logical DAG
    bool profiling = false, graph_profiling = false;
    std::vector<cudaEvent_t> prof_events;
    std::vector<std::vector<int>> prof_ldeps;
    std::vector<int> prof_cat;
    std::vector<double> prof_bytes;
    std::vector<double> crit_class_ms;     // critical path composition of the last profile()
    std::vector<uint64_t> crit_class_nodes;
    std::vector<int> prof_stage;
    std::vector<const void*> prof_func;

    // optional per-launch timing of the update kernel (event record nodes)
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    double upd_alg_bytes = 0.0;
    uint64_t upd_timed = 0;

    ~ferret_trainer() {
        cudaSetDevice(opt.device);
        if (stream) cudaStreamSynchronize(stream);
        if (nstream) cudaStreamSynchronize(nstream);
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        for (cudaGraphExec_t x : more_execs) cudaGraphExecDestroy(x);
        for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
        for (cudaEvent_t e : prof_events) cudaEventDestroy(e);
        for (void* p : peer_opened)
            if (p) cudaIpcCloseMemHandle(p);
        dfree(d_inbox);
        for (cudaEvent_t e : norm_events) cudaEventDestroy(e);
        for (cudaEvent_t e : ctl_done) cudaEventDestroy(e);
        if (fork_event) cudaEventDestroy(fork_event);
        for (unsigned char* p : h_ctl) cudaFreeHost(p);
        for (StageDev& s : stages) {
            dfree(s.ring);
            dfree(s.lam_d);
            dfree(s.v_r);
            dfree(s.v_a);
            dfree(s.gap);
            dfree(s.segs_dev);
            dfree(s.tiles_dev);
            dfree(s.works_dev);
            dfree(s.works4_dev);
            dfree(s.works_g_dev);
            dfree(s.ring16);
        }
        for (auto& kv : mma_scratch) {
            dfree(kv.second.first);
            dfree(kv.second.second);
        }
        wt_reset();
        for (auto& kv : conv_scratch) dfree(kv.second);
        for (void* p : {static_cast<void*>(d_raw), static_cast<void*>(d_lab), static_cast<void*>(d_pred),
                        static_cast<void*>(d_norm_mean), static_cast<void*>(d_norm_m2), static_cast<void*>(d_rawc),
                        static_cast<void*>(d_norm_mu), static_cast<void*>(d_norm_m2i),
                        static_cast<void*>(d_xc), static_cast<void*>(d_labc), static_cast<void*>(d_predc),
                        static_cast<void*>(d_ctl), static_cast<void*>(d_pool_x), static_cast<void*>(d_pool_lab),
                        static_cast<void*>(d_stash), static_cast<void*>(d_replay),
                        static_cast<void*>(d_partial), static_cast<void*>(d_counters)})
            dfree(p);
        release_ingest();
        if (ing.copy) cudaStreamDestroy(ing.copy);
        if (ing.back) cudaStreamDestroy(ing.back);
        if (stream) cudaStreamDestroy(stream);
        if (nstream) cudaStreamDestroy(nstream);
    }

    void invalidate_graph() {
        if (graph_exec) {
            cudaStreamSynchronize(stream);
            cudaGraphExecDestroy(graph_exec);
            graph_exec = nullptr;
            for (cudaGraphExec_t x : more_execs) cudaGraphExecDestroy(x);
            more_execs.clear();
        }
    }

    // ------------------------------------------------------------------ setup
    void build(const ferret_net_desc& net, const uint64_t* bounds, int32_t n_bounds) {
        L = net.n_layers;
        if (L <= 0) fail(FERRET_E_CONFIG, "net needs at least one layer");
        if (n_bounds < 2 || bounds[0] != 0 || bounds[n_bounds - 1] != static_cast<uint64_t>(L))
            fail(FERRET_E_CONFIG, "partition bounds must run from 0 to the layer count");
        for (int32_t i = 1; i < n_bounds; ++i)
            if (bounds[i] <= bounds[i - 1]) fail(FERRET_E_CONFIG, "partition bounds must be strictly increasing");
        P = n_bounds - 1;
        if (P > 16) fail(FERRET_E_CONFIG, "at most 16 stages per trainer");
        B = opt.micro_batch;
        if (B < 1 || B > fb200::kMaxBatch) fail(FERRET_E_CONFIG, "micro_batch must lie in [1, 16]");
        if (opt.policy < 0 || opt.policy > 4) fail(FERRET_E_CONFIG, "unknown compensation policy");
        if (opt.precision != FERRET_PREC_FP32 && opt.precision != FERRET_PREC_BF16 && opt.precision != FERRET_PREC_TF32)
            fail(FERRET_E_CONFIG, "precision must be FERRET_PREC_FP32, FERRET_PREC_BF16 or FERRET_PREC_TF32");
        if (opt.replay && (opt.replay_capacity == 0 || opt.replay_capacity > (1ull << 30)))
            fail(FERRET_E_CONFIG, "replay capacity must lie in [1, 2^30]");
        layers.resize(static_cast<size_t>(L));
        long long host_off = 0;
        for (int l = 0; l < L; ++l) {
            LayerDev& ld = layers[static_cast<size_t>(l)];
            ld.in = static_cast<int>(net.in[l]);
            ld.out = static_cast<int>(net.out[l]);
            ld.act = net.act[l];
            if (l > 0 && net.in[l] != net.out[l - 1])
                fail(FERRET_E_CONFIG, "layer " + std::to_string(l) + ": input width mismatch");
            ld.rows = ld.out;
            ld.cols = ld.in;
            ld.co = ld.out;
            ld.ci = ld.in;
            if (net.geom) set_geometry(ld, l, net.geom + static_cast<size_t>(l) * FERRET_GEOM_INTS);
            ld.host_off = host_off;
            host_off += ld.nw() + ld.rows;
        }
        if (net.geom) {
            geom.assign(net.geom, net.geom + static_cast<size_t>(L) * FERRET_GEOM_INTS);
            for (int32_t i = 1; i + 1 < n_bounds; ++i)
                if (layers[static_cast<size_t>(bounds[i])].res)
                    fail(FERRET_E_CONFIG, "partition bound " + std::to_string(bounds[i]) + " splits a residual block");
        }
        F = layers.front().in;
        n_out = layers.back().out;
        if (net.params) init_params.assign(net.params, net.params + host_off);
        else if (!t_plan_only) fail(FERRET_E_INVALID_ARG, "net params: null (allowed for plan-only trainers only)");
        long long cursor = 0;
        int max_width = F;
        for (LayerDev& ld : layers) {
            ld.act_off = align_up(cursor, 32);
            cursor = ld.act_off + static_cast<long long>(B) * ld.out;
            ld.dlt_off = align_up(cursor, 32);
            cursor = ld.dlt_off + static_cast<long long>(B) * ld.out;
            max_width = std::max(max_width, ld.out);
            if (ld.conv()) {
                ld.g_off = align_up(cursor, 32);
                cursor = ld.g_off + ld.nw() + ld.rows;
            }
            if (ld.gap()) {
                ld.pool_off = align_up(cursor, 32);
                cursor = ld.pool_off + static_cast<long long>(B) * ld.ci;
                ld.pdl_off = align_up(cursor, 32);
                cursor = ld.pdl_off + static_cast<long long>(B) * ld.ci;
            }
        }
        // predict scratch: three rotating buffers (a residual layer reads the input of
        // the layer below while writing its own output)
        pred_stride = align_up(static_cast<long long>(B) * max_width, 64);
        pred_off = align_up(cursor, 64);
        stash_stride = align_up(pred_off + 3 * pred_stride, 64);
        stages.resize(static_cast<size_t>(P));
        hs.current.assign(static_cast<size_t>(P), 0);
        owner.assign(static_cast<size_t>(P), 0);
        peer_data.assign(1, nullptr);
        peer_flags.assign(1, nullptr);
        peer_acks.assign(1, nullptr);
        for (int j = 0; j < P; ++j) {
            StageDev& s = stages[static_cast<size_t>(j)];
            s.lo = static_cast<int>(bounds[j]);
            s.hi = static_cast<int>(bounds[j + 1]);
            if (s.hi - s.lo > fb200::kMaxStageLayers) fail(FERRET_E_CONFIG, "at most 16 layers per stage");
            s.host_off = layers[static_cast<size_t>(s.lo)].host_off;
            long long c = 0;
            std::vector<fb200::UpdSeg> tab;
            for (int l = s.lo; l < s.hi; ++l) {
                LayerDev& ld = layers[static_cast<size_t>(l)];
                ld.stage = j;
                ld.woff = align_up(c, 32);
                c = ld.woff + ld.nw();
                ld.boff = align_up(c, 32);
                c = ld.boff + ld.rows;
                s.n_params += ld.nw() + ld.rows;
                // float4 items need 16-byte aligned weight rows and input rows
                // (stash rows are B x in; x rows are F wide with F == in at layer 0)
                const int vec = (ld.cols % 4 == 0) ? 4 : 1;
                fb200::UpdSeg w{};
                w.layer = l - s.lo;
                w.bias = 0;
                w.vec = vec;
                w.per_row = ld.cols / vec;
                w.item0 = s.n_items;
                w.elem0 = ld.woff;
                w.in = ld.cols;
                w.out = ld.rows;
                // gW = delta (x) input, recomputed by the update from the stash; a
                // convolution's gradient is materialised there by conv_wgrad instead
                w.xin_off = ld.gap() ? ld.pool_off : l == 0 ? -1 : layers[static_cast<size_t>(l - 1)].act_off;
                w.dlt_off = ld.dlt_off;
                w.g_off = ld.conv() ? ld.g_off : -1;
                s.gmat = s.gmat || ld.conv();
                tab.push_back(w);
                s.n_items += static_cast<long long>(ld.rows) * w.per_row;
                fb200::UpdSeg bs = w;
                bs.bias = 1;
                bs.vec = 1;
                bs.per_row = 1;
                bs.item0 = s.n_items;
                bs.elem0 = ld.boff;
                bs.g_off = ld.conv() ? ld.g_off + ld.nw() : -1;
                tab.push_back(bs);
                s.n_items += ld.rows;
                if (l > 0 && !ld.conv()) {
                    max_partial = std::max(max_partial, static_cast<size_t>(fb200::bwd_row_splits(ld.cols, ld.rows)) *
                                                            static_cast<size_t>(B) * static_cast<size_t>(ld.cols));
                    max_tiles = std::max(max_tiles, static_cast<size_t>(fb200::bwd_col_tiles(ld.cols)));
                }
            }
            s.slot_floats = align_up(c, 64);
            s.n_segs = static_cast<int>(tab.size());
            s.segs_dev = dalloc<fb200::UpdSeg>(tab.size(), device_bytes);
            cuda_check(cudaMemcpy(s.segs_dev, tab.data(), tab.size() * sizeof(fb200::UpdSeg), cudaMemcpyHostToDevice),
                       "upload segment table");
            // update tiles: R rows x 256 columns per CTA. In the concurrent chunk graph
            // fewer, fuller CTAs per kernel leave the SMs to the other nodes
            long long row_tiles = 0;
            for (const fb200::UpdSeg& sg : tab)
                if (!sg.bias) row_tiles += static_cast<long long>(sg.out) * ((sg.in + fb200::kUpdTileCols - 1) / fb200::kUpdTileCols);
            const int r400 = static_cast<int>(std::min<long long>(fb200::kUpdMaxTileRows, std::max<long long>(1, (row_tiles + 399) / 400)));
            // measured per update kernel (profiles/README.md): the iter_fisher kernel with
            // 8-row tiles at micro-batch >= 8 (3.25 vs 3.8 ms per config-2 chunk), 2-row
            // tiles at micro-batch 1; the generic kernel with ~400 CTAs per update
            int R = opt.policy == FERRET_POLICY_ITER_FISHER ? (B >= 8 ? fb200::kUpdMaxTileRows : 2) : r400;
            if (const char* rows = std::getenv("FERRET_UPD_ROWS"))  // tile-shape experiment knob (0: ~400 CTAs)
                R = std::atoi(rows) <= 0 ? r400 : std::max(1, std::min(fb200::kUpdMaxTileRows, std::atoi(rows)));
            std::vector<fb200::UpdTile> tiles;
            for (size_t q = 0; q < tab.size(); ++q) {
                const fb200::UpdSeg& sg = tab[q];
                if (sg.bias) {
                    for (int r0 = 0; r0 < sg.out; r0 += fb200::kUpdTileCols)
                        tiles.push_back({static_cast<int>(q), r0, std::min(fb200::kUpdTileCols, sg.out - r0), 0});
                } else {
                    for (int r0 = 0; r0 < sg.out; r0 += R)
                        for (int c0 = 0; c0 < sg.in; c0 += fb200::kUpdTileCols)
                            tiles.push_back({static_cast<int>(q), r0, std::min(R, sg.out - r0), c0});
                }
            }
            s.n_tiles = static_cast<int>(tiles.size());
            std::vector<fb200::UpdWork> works;
            for (const fb200::UpdTile& t : tiles) {
                const fb200::UpdSeg& sg = tab[static_cast<size_t>(t.seg)];
                works.push_back({sg.elem0, sg.xin_off, sg.dlt_off, sg.in, sg.out, sg.bias, t.r0, t.nrows, t.c0, sg.g_off});
            }
            // float4 tiles: a thread owns 4 consecutive columns of R4 rows; CTA =
            // threads4 threads (enough for the widest row, <= 256) covering
            // 4 x threads4 columns; bias segments keep one element per thread
            bool aligned = true;
            int widest = 0;
            for (const fb200::UpdSeg& sg : tab)
                if (!sg.bias) {
                    aligned = aligned && sg.in % 4 == 0;
                    widest = std::max(widest, sg.in);
                }
            // measured: ~2.5 % faster than the scalar kernel on HBM-bound 33 M-param
            // stages (config 5), ~10 % slower on L2-resident small stages (config 2,
            // lower occupancy) -> only for large stages
            const char* v4min = std::getenv("FERRET_UPDATE_V4_MIN_PARAMS");  // test / experiment knob
            if (aligned && s.n_params >= (v4min ? std::atoll(v4min) : (1LL << 22))) {
                s.threads4 = std::min(256, std::max(32, ((widest / 4 + 31) / 32) * 32));
                const int cols4 = 4 * s.threads4;
                long long rt4 = 0;
                for (const fb200::UpdSeg& sg : tab)
                    if (!sg.bias) rt4 += static_cast<long long>(sg.out) * ((sg.in + cols4 - 1) / cols4);
                const int R4 = static_cast<int>(std::min<long long>(fb200::kUpdMaxTileRows, std::max<long long>(1, (rt4 + 295) / 296)));
                std::vector<fb200::UpdWork> w4;
                for (const fb200::UpdSeg& sg : tab) {
                    if (sg.bias) {
                        for (int r0 = 0; r0 < sg.out; r0 += s.threads4)
                            w4.push_back({sg.elem0, sg.xin_off, sg.dlt_off, sg.in, sg.out, 1, r0, std::min(s.threads4, sg.out - r0), 0});
                    } else {
                        for (int r0 = 0; r0 < sg.out; r0 += R4)
                            for (int c0 = 0; c0 < sg.in; c0 += cols4)
                                w4.push_back({sg.elem0, sg.xin_off, sg.dlt_off, sg.in, sg.out, 0, r0, std::min(R4, sg.out - r0), c0});
                    }
                }
                s.n_tiles4 = static_cast<int>(w4.size());
                s.works4_dev = dalloc<fb200::UpdWork>(w4.size(), device_bytes);
                cuda_check(cudaMemcpy(s.works4_dev, w4.data(), w4.size() * sizeof(fb200::UpdWork), cudaMemcpyHostToDevice),
                           "upload work table");
            }
            s.works_dev = dalloc<fb200::UpdWork>(works.size(), device_bytes);
            cuda_check(cudaMemcpy(s.works_dev, works.data(), works.size() * sizeof(fb200::UpdWork), cudaMemcpyHostToDevice),
                       "upload work table");
            // update groups (kernels.cuh GroupArgs) pay off only where a stage's chain is far larger
            // than its unit inputs: dense stages of at least FERRET_UPDATE_GROUPS_MIN parameters
            // (default 8M), weight rows 16-byte aligned for the kernel's bulk copies
            s.group_ok = group_updates && !s.gmat && opt.policy == FERRET_POLICY_ITER_FISHER &&
                         s.slot_floats >= group_min_params;
            int n_wsegs = 0;
            for (const fb200::UpdSeg& sg : tab) {
                if (!sg.bias && sg.in % 4 != 0) s.group_ok = false;
                n_wsegs += sg.bias ? 0 : 1;
            }
            if (n_wsegs > fb200::kGroupMaxSegs) s.group_ok = false;
            s.gsegs.clear();
            if (s.group_ok) {  // tiles: kGroupRows rows x kGroupCols columns, column-block major (a CTA's
                               // range shares its column block's unit inputs), then bias runs of 256
                std::vector<fb200::UpdWork> wg;
                for (const fb200::UpdSeg& sg : tab)
                    if (!sg.bias) {
                        s.gsegs.push_back({sg.elem0, sg.xin_off, sg.dlt_off, sg.in, sg.out, static_cast<int>(wg.size()),
                                           (sg.out + fb200::kGroupRows - 1) / fb200::kGroupRows});
                        for (int c0 = 0; c0 < sg.in; c0 += fb200::kGroupCols)
                            for (int r0 = 0; r0 < sg.out; r0 += fb200::kGroupRows)
                                wg.push_back({sg.elem0, sg.xin_off, sg.dlt_off, sg.in, sg.out, 0, r0,
                                              std::min(fb200::kGroupRows, sg.out - r0), c0, sg.g_off});
                    }
                s.n_wtiles_g = static_cast<int>(wg.size());
                for (const fb200::UpdSeg& sg : tab)
                    if (sg.bias)
                        for (int r0 = 0; r0 < sg.out; r0 += fb200::kUpdTileCols)
                            wg.push_back({sg.elem0, sg.xin_off, sg.dlt_off, sg.in, sg.out, 1, r0,
                                          std::min(fb200::kUpdTileCols, sg.out - r0), 0, sg.g_off});
                s.n_tiles_g = static_cast<int>(wg.size());
                s.works_g_dev = dalloc<fb200::UpdWork>(wg.size(), device_bytes);
                cuda_check(cudaMemcpy(s.works_g_dev, wg.data(), wg.size() * sizeof(fb200::UpdWork), cudaMemcpyHostToDevice),
                           "upload group work table");
            }
            s.tiles_dev = dalloc<fb200::UpdTile>(tiles.size(), device_bytes);
            cuda_check(cudaMemcpy(s.tiles_dev, tiles.data(), tiles.size() * sizeof(fb200::UpdTile), cudaMemcpyHostToDevice),
                       "upload tile table");
            const size_t n = static_cast<size_t>(s.slot_floats);
            if (opt.policy == FERRET_POLICY_ITER_FISHER) {
                s.lam_d = dalloc<float>(n, device_bytes);
                cuda_check(cudaMemset(s.lam_d, 0, n * sizeof(float)), "memset");
                if (opt.eta_lambda > 0.0) {
                    s.v_r = dalloc<float>(n, device_bytes);
                    s.v_a = dalloc<float>(n, device_bytes);
                    cuda_check(cudaMemset(s.v_r, 0, n * sizeof(float)), "memset");
                    cuda_check(cudaMemset(s.v_a, 0, n * sizeof(float)), "memset");
                }
            } else if (opt.policy == FERRET_POLICY_GAP) {
                s.gap = dalloc<float>(n, device_bytes);
                cuda_check(cudaMemset(s.gap, 0, n * sizeof(float)), "memset");
            }
            grow_ring(s, 2);
        }
        if (!t_plan_only) upload_initial_params();
        d_replay = dalloc<float>(static_cast<size_t>(stash_stride), device_bytes);
        d_norm_mean = dalloc<double>(static_cast<size_t>(F), device_bytes);
        d_norm_m2 = dalloc<double>(static_cast<size_t>(F), device_bytes);
        cuda_check(cudaMemset(d_norm_mean, 0, static_cast<size_t>(F) * sizeof(double)), "memset");
        cuda_check(cudaMemset(d_norm_m2, 0, static_cast<size_t>(F) * sizeof(double)), "memset");
        if (opt.replay) {
            d_pool_x = dalloc<float>(static_cast<size_t>(opt.replay_capacity) * static_cast<size_t>(F), device_bytes);
            d_pool_lab = dalloc<int>(static_cast<size_t>(opt.replay_capacity), device_bytes);
        }
        hs.replay = Reservoir(opt.replay_capacity, opt.replay_seed);
        cuda_check(cudaEventCreateWithFlags(&fork_event, cudaEventDisableTiming), "cudaEventCreate");
    }

    void upload_initial_params() {
        for (StageDev& s : stages) {
            std::vector<float> slot(static_cast<size_t>(s.slot_floats), 0.f);
            for (int l = s.lo; l < s.hi; ++l) {
                const LayerDev& ld = layers[static_cast<size_t>(l)];
                const double* src = init_params.data() + ld.host_off;
                const long long nw = ld.nw();
                for (long long i = 0; i < nw; ++i) slot[static_cast<size_t>(ld.woff + i)] = static_cast<float>(src[i]);
                for (int r = 0; r < ld.rows; ++r)
                    slot[static_cast<size_t>(ld.boff + r)] = static_cast<float>(src[nw + r]);
            }
            cuda_check(cudaMemcpy(s.slot(0), slot.data(), slot.size() * sizeof(float), cudaMemcpyHostToDevice),
                       "upload params");
            if (s.ring16) {
                std::vector<uint16_t> h(slot.size());
                for (size_t i = 0; i < slot.size(); ++i) h[i] = bf16_bits(slot[i]);
                cuda_check(cudaMemcpy(s.ring16, h.data(), h.size() * sizeof(uint16_t), cudaMemcpyHostToDevice),
                           "upload bf16 params");
            }
        }
    }

    // Grow a stage ring to `depth` slots; the live version is in slot 0 between chunks.
    void grow_ring(StageDev& s, int depth) {
        if (depth <= s.depth) return;
        float* fresh = dalloc<float>(static_cast<size_t>(depth) * static_cast<size_t>(s.slot_floats), device_bytes);
        if (s.depth > 0) {  // (plan-only trainers count the old ring without holding it)
            if (s.ring) {
                cuda_check(cudaStreamSynchronize(stream), "sync");
                cuda_check(cudaMemcpy(fresh, s.ring, static_cast<size_t>(s.slot_floats) * sizeof(float),
                                      cudaMemcpyDeviceToDevice),
                           "ring copy");
                cudaFree(s.ring);
            }
            device_bytes -= static_cast<size_t>(s.depth) * static_cast<size_t>(s.slot_floats) * sizeof(float);
        }
        s.ring = fresh;
        if (opt.precision == FERRET_PREC_BF16) {
            uint16_t* fresh16 =
                dalloc<uint16_t>(static_cast<size_t>(depth) * static_cast<size_t>(s.slot_floats), device_bytes);
            if (s.depth > 0) {
                if (s.ring16) {
                    cuda_check(cudaMemcpy(fresh16, s.ring16, static_cast<size_t>(s.slot_floats) * sizeof(uint16_t),
                                          cudaMemcpyDeviceToDevice),
                               "ring copy");
                    cudaFree(s.ring16);
                }
                device_bytes -= static_cast<size_t>(s.depth) * static_cast<size_t>(s.slot_floats) * sizeof(uint16_t);
            }
            s.ring16 = fresh16;
        }
        s.depth = depth;
    }

    // per-slot bwd reduction scratch: slots 0..stash_slots-1 for units, the last for replay
    void ensure_scratch(int slots) {
        if (slots <= scratch_slots) return;
        cuda_check(cudaStreamSynchronize(stream), "sync");
        dfree(d_partial);
        dfree(d_counters);
        device_bytes -= static_cast<size_t>(scratch_slots) * (max_partial * sizeof(float) + max_tiles * sizeof(unsigned));
        d_partial = dalloc<float>(static_cast<size_t>(slots) * max_partial, device_bytes);
        d_counters = dalloc<unsigned>(static_cast<size_t>(slots) * max_tiles, device_bytes);
        cuda_check(cudaMemset(d_counters, 0, static_cast<size_t>(slots) * max_tiles * sizeof(unsigned)), "memset");
        scratch_slots = slots;
    }

    void ensure_stash(int slots) {
        if (slots <= stash_slots) return;
        cuda_check(cudaStreamSynchronize(stream), "sync");
        if (d_stash) cudaFree(d_stash);
        device_bytes -= static_cast<size_t>(stash_slots) * static_cast<size_t>(stash_stride) * sizeof(float);
        d_stash = dalloc<float>(static_cast<size_t>(slots) * static_cast<size_t>(stash_stride), device_bytes);
        stash_slots = slots;
    }

    // ---------------------------------------------------------------- stream
    void load_stream(const double* features, const uint64_t* lab, size_t n, size_t f) {
        if (static_cast<int>(f) != F) fail(FERRET_E_INVALID_ARG, "stream feature width does not match the net input");
        std::vector<int> l32(n);
        for (size_t i = 0; i < n; ++i) {
            if (lab[i] >= static_cast<uint64_t>(n_out)) fail(FERRET_E_INVALID_ARG, "forward_backward: label out of range");
            l32[i] = static_cast<int>(lab[i]);
        }
        cuda_check(cudaStreamSynchronize(stream), "sync");
        if (n > n_loaded || !d_raw) {
            dfree(d_raw);
            dfree(d_lab);
            dfree(d_pred);
            if (d_raw) device_bytes -= stream_cap * (f * sizeof(double) + 2 * sizeof(int));
            stream_cap = n;
            d_raw = dalloc<double>(n * f, device_bytes);
            d_lab = dalloc<int>(n, device_bytes);
            d_pred = dalloc<int>(n, device_bytes);
        }
        n_loaded = n;
        labels = std::move(l32);
        cuda_check(cudaMemcpyAsync(d_raw, features, n * f * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D stream");
        cuda_check(cudaMemcpyAsync(d_lab, labels.data(), n * sizeof(int), cudaMemcpyHostToDevice, stream), "H2D labels");
        cuda_check(cudaStreamSynchronize(stream), "sync");  // `labels` may be reassigned by the next load
    }

    void set_schedule(const ferret_event* ev, size_t n_ev, size_t chunk_items) {
        // same log and chunking: keep the compiled graph
        if (have_schedule && sched.events.size() == n_ev && (chunk_items ? chunk_items : sched.chunk_items) == sched.chunk_items &&
            (n_ev == 0 || std::memcmp(sched.events.data(), ev, n_ev * sizeof(ferret_event)) == 0))
            return;
        Schedule s;
        s.events.assign(ev, ev + n_ev);
        long long expect = 0;
        for (const ferret_event& e : s.events) {
            if (e.kind == FERRET_EV_ARRIVAL) {
                if (e.item != expect) fail(FERRET_E_INVALID_ARG, "event log: arrivals must cover items 0..n-1 in order");
                ++expect;
            }
        }
        s.n_units = static_cast<size_t>(expect);
        s.chunk_items = chunk_items ? chunk_items : s.n_units * static_cast<size_t>(B);
        if (s.n_units * static_cast<size_t>(B) > s.chunk_items)
            fail(FERRET_E_INVALID_ARG, "event log covers more samples than one chunk");
        s.dropped.assign(s.n_units, 0);
        s.has_bwd.assign(s.n_units * static_cast<size_t>(P), 0);
        s.update_fires.assign(s.events.size(), 0);
        std::vector<long long> last_use(s.n_units, -1);
        std::map<std::pair<int, int>, std::vector<long long>> open;  // (worker, stage) -> units awaiting update
        for (size_t i = 0; i < s.events.size(); ++i) {
            const ferret_event& e = s.events[i];
            const bool staged = e.kind == FERRET_EV_FORWARD || e.kind == FERRET_EV_BACKWARD || e.kind == FERRET_EV_UPDATE;
            if (e.kind < FERRET_EV_ARRIVAL || e.kind > FERRET_EV_UPDATE) fail(FERRET_E_INVALID_ARG, "event log: unknown event kind");
            if (staged && (e.stage < 0 || e.stage >= P))
                fail(FERRET_E_INVALID_ARG, "event log: stage out of range for this partition");
            if (e.kind != FERRET_EV_UPDATE && (e.item < 0 || static_cast<size_t>(e.item) >= s.n_units))
                fail(FERRET_E_INVALID_ARG, "event log: item out of range");
            const size_t u = static_cast<size_t>(e.item);
            switch (e.kind) {
                case FERRET_EV_DROP: s.dropped[u] = 1; break;
                case FERRET_EV_ARRIVAL:
                case FERRET_EV_FORWARD: last_use[u] = static_cast<long long>(i); break;
                case FERRET_EV_BACKWARD:
                    last_use[u] = static_cast<long long>(i);
                    s.has_bwd[u * static_cast<size_t>(P) + static_cast<size_t>(e.stage)] = 1;
                    open[{e.worker, e.stage}].push_back(static_cast<long long>(u));
                    break;
                case FERRET_EV_UPDATE: {
                    auto it = open.find({e.worker, e.stage});
                    if (it == open.end() || it->second.empty()) break;
                    s.update_fires[i] = 1;
                    for (long long uu : it->second) last_use[static_cast<size_t>(uu)] = static_cast<long long>(i);
                    it->second.clear();
                    break;
                }
                default: break;
            }
        }
        s.free_at.assign(s.events.size(), {});
        for (size_t u = 0; u < s.n_units; ++u)
            if (!s.dropped[u] && last_use[u] >= 0) s.free_at[static_cast<size_t>(last_use[u])].push_back(u);
        sched = std::move(s);
        have_schedule = true;
        invalidate_graph();
        alloc_chunk_buffers();
        setup_inbox();
    }

    void alloc_chunk_buffers() {
        const size_t cap = sched.chunk_items;
        // replay steps per chunk <= stage-0 updates that fire
        size_t upd0 = 0;
        for (size_t i = 0; i < sched.events.size(); ++i)
            if (sched.update_fires[i] && sched.events[i].stage == 0) ++upd0;
        const size_t need_rep = opt.replay ? upd0 : 0;
        const size_t need_ctl =
            kCtlHeader + (cap + 2 * std::max<size_t>(need_rep, 1) * static_cast<size_t>(B)) * sizeof(int);
        if (cap > chunk_cap) {
            cuda_check(cudaStreamSynchronize(stream), "sync");
            for (void* p : {static_cast<void*>(d_rawc), static_cast<void*>(d_xc), static_cast<void*>(d_labc),
                            static_cast<void*>(d_predc), static_cast<void*>(d_norm_mu), static_cast<void*>(d_norm_m2i)})
                dfree(p);
            device_bytes -= chunk_cap * (static_cast<size_t>(F) * (3 * sizeof(double) + sizeof(float)) + 3 * sizeof(int));
            d_rawc = dalloc<double>(cap * static_cast<size_t>(F), device_bytes);
            d_norm_mu = dalloc<double>(cap * static_cast<size_t>(F), device_bytes);
            d_norm_m2i = dalloc<double>(cap * static_cast<size_t>(F), device_bytes);
            d_xc = dalloc<float>(cap * static_cast<size_t>(F), device_bytes);
            d_labc = dalloc<int>(cap, device_bytes);
            d_predc = dalloc<int>(cap, device_bytes);
            chunk_cap = cap;
        }
        if (need_ctl > ctl_bytes) {
            cuda_check(cudaStreamSynchronize(stream), "sync");
            dfree(d_ctl);
            device_bytes -= ctl_bytes;
            for (unsigned char* p : h_ctl) cudaFreeHost(p);
            h_ctl.clear();
            d_ctl = dalloc<unsigned char>(need_ctl, device_bytes);
            for (int k = 0; k < 2; ++k) {
                void* p = nullptr;
                cuda_check(cudaMallocHost(&p, need_ctl), "cudaMallocHost");
                h_ctl.push_back(static_cast<unsigned char*>(p));
                if (ctl_done.size() < 2) {
                    cudaEvent_t e;
                    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
                    ctl_done.push_back(e);
                    cuda_check(cudaEventRecord(e, stream), "cudaEventRecord");
                }
            }
            ctl_bytes = need_ctl;
        }
        max_rep = std::max<size_t>(need_rep, 1);
    }

    // control block: [count u64][epoch u32][pad u32][pool_dst x chunk_cap][rep_ids x max_rep*B][rep_labels x max_rep*B]
    static constexpr size_t kCtlHeader = 16;
    unsigned long long* ctl_count() const { return reinterpret_cast<unsigned long long*>(d_ctl); }
    const unsigned* ctl_epoch() const { return reinterpret_cast<const unsigned*>(d_ctl + 8); }
    int* ctl_pool_dst() const { return reinterpret_cast<int*>(d_ctl + kCtlHeader); }
    int* ctl_rep_ids() const { return reinterpret_cast<int*>(d_ctl + kCtlHeader + chunk_cap * sizeof(int)); }
    int* ctl_rep_labels() const {
        return reinterpret_cast<int*>(d_ctl + kCtlHeader + (chunk_cap + max_rep * static_cast<size_t>(B)) * sizeof(int));
    }

    // -------------------------------------------------- host reservoir per chunk
    // Walks the log exactly like the reference trainer's buffer_ calls
    // (learner.hpp:409 add at every non-dropped arrival, :509/:514 sample at
    // every firing stage-0 update while non-empty).
    ChunkPlan plan_chunk(Reservoir& res, const int* chunk_labels, int64_t sample_base) const {
        ChunkPlan cp;
        cp.pool_dst.assign(sched.chunk_items, -1);
        if (!opt.replay || opt.as_shipped) return cp;
        for (size_t i = 0; i < sched.events.size(); ++i) {
            const ferret_event& e = sched.events[i];
            if (e.kind == FERRET_EV_ARRIVAL && !sched.dropped[static_cast<size_t>(e.item)]) {
                for (int b = 0; b < B; ++b) {
                    const size_t s = static_cast<size_t>(e.item) * static_cast<size_t>(B) + static_cast<size_t>(b);
                    cp.pool_dst[s] = res.add(chunk_labels[s], sample_base + static_cast<int64_t>(s));
                }
            } else if (e.kind == FERRET_EV_UPDATE && e.stage == 0 && sched.update_fires[i] && res.size > 0) {
                for (int b = 0; b < B; ++b) {
                    const int pos = res.sample();
                    cp.rep_ids.push_back(pos);
                    cp.rep_labels.push_back(res.label_at[static_cast<size_t>(pos)]);
                }
                ++cp.n_replays;
            }
        }
        return cp;
    }

    // -------------------------------------------------------------- execute
    void execute(size_t chunk) {
        if (!have_schedule) fail(FERRET_E_LOGIC, "execute: no schedule set");
        const size_t base = chunk * sched.chunk_items;
        const size_t n_samples = sched.n_units * static_cast<size_t>(B);
        if (base + n_samples > n_loaded) fail(FERRET_E_OUT_OF_RANGE, "execute: chunk lies beyond the loaded stream");
        execute_from(labels.data() + base, d_raw + base * static_cast<size_t>(F), d_lab + base, d_pred + base);
    }

    // One chunk of the compiled schedule over device-resident rows: raw features
    // and labels are copied into the graph's fixed staging, predictions out to
    // `dst_pred`. `chunk_labels` (host) drive the replay reservoir.
    void execute_from(const int* chunk_labels, const double* src_raw, const int* src_lab, int* dst_pred) {
        const size_t n_samples = sched.n_units * static_cast<size_t>(B);
        const bool seen_any = hs.replay.seen > 0;
        if (graph_exec && (graph_timing != timing || graph_profiling != profiling || graph_seen_any != seen_any))
            invalidate_graph();
        if (!graph_exec) build_graph(seen_any);
        // host decisions for this chunk
        const ChunkPlan cp = plan_chunk(hs.replay, chunk_labels, static_cast<int64_t>(hs.norm_count));
        if (cp.n_replays != graph_shape.n_replays)
            fail(FERRET_E_LOGIC, "replay pattern of this chunk differs from the compiled graph");
        // control block -> device (double-buffered pinned staging)
        unsigned char* h = h_ctl[static_cast<size_t>(ctl_flip)];
        cuda_check(cudaEventSynchronize(ctl_done[static_cast<size_t>(ctl_flip)]), "cudaEventSynchronize");
        const unsigned long long count = hs.norm_count;
        const unsigned epoch = ++epoch_counter;  // hand-off flags of this chunk (identical on every rank)
        std::memcpy(h, &count, 8);
        std::memcpy(h + 8, &epoch, 4);
        std::memcpy(h + kCtlHeader, cp.pool_dst.data(), cp.pool_dst.size() * sizeof(int));
        const size_t rep_off = kCtlHeader + chunk_cap * sizeof(int);
        const size_t lab_off = rep_off + max_rep * static_cast<size_t>(B) * sizeof(int);
        if (!cp.rep_ids.empty()) {
            std::memcpy(h + rep_off, cp.rep_ids.data(), cp.rep_ids.size() * sizeof(int));
            std::memcpy(h + lab_off, cp.rep_labels.data(), cp.rep_labels.size() * sizeof(int));
        }
        const size_t used = cp.rep_ids.empty() ? rep_off : lab_off + cp.rep_labels.size() * sizeof(int);
        cuda_check(cudaMemcpyAsync(d_ctl, h, used, cudaMemcpyHostToDevice, stream), "H2D control");
        cuda_check(cudaEventRecord(ctl_done[static_cast<size_t>(ctl_flip)], stream), "cudaEventRecord");
        ctl_flip ^= 1;
        // chunk data -> staging
        cuda_check(cudaMemcpyAsync(d_rawc, src_raw, n_samples * static_cast<size_t>(F) * sizeof(double),
                                   cudaMemcpyDeviceToDevice, stream),
                   "D2D chunk");
        cuda_check(cudaMemcpyAsync(d_labc, src_lab, n_samples * sizeof(int), cudaMemcpyDeviceToDevice, stream),
                   "D2D labels");
        cuda_check(cudaGraphLaunch(graph_exec, stream), "cudaGraphLaunch");
        for (cudaGraphExec_t x : more_execs) cuda_check(cudaGraphLaunch(x, stream), "cudaGraphLaunch");
        cuda_check(cudaMemcpyAsync(dst_pred, d_predc, n_samples * sizeof(int), cudaMemcpyDeviceToDevice, stream),
                   "D2D predictions");
        hs.norm_count += n_samples;
        for (int j = 0; j < P; ++j) hs.current[static_cast<size_t>(j)] += graph_shape.pushes[static_cast<size_t>(j)];
        stats.kernel_launches = launches;
        stats.stash_slots = stash_slots;
        for (int j = 0; j < P && j < 16; ++j) stats.ring_depth[j] = stages[static_cast<size_t>(j)].depth;
    }

    // HBM the trainer holds once the current schedule's chunk graph is built (north-star item 4:
    // the planner's memory in bytes): the dry pass that build_graph() runs sizes the version
    // rings and the stash; everything else is already allocated (or, for a plan-only trainer,
    // counted). Graph-build scratch of the tensor-core layers (split-K partials, conv weight
    // copies) is not included.
    ferret_footprint footprint() {
        if (!have_schedule) fail(FERRET_E_LOGIC, "footprint: set_schedule first");
        HostState probe = hs;
        const PassResult need = [&] {
            PlanOnlyScope scope(true);
            return run_pass<true>(probe, hs.replay.seen > 0);
        }();
        ferret_footprint f{};
        const size_t per_float = sizeof(float) + (opt.precision == FERRET_PREC_BF16 ? sizeof(uint16_t) : 0);
        size_t total = device_bytes;
        for (int j = 0; j < P; ++j) {
            const StageDev& sd = stages[static_cast<size_t>(j)];
            const int d = std::max(sd.depth, need.need_depth[static_cast<size_t>(j)]);
            total += static_cast<size_t>(d - sd.depth) * static_cast<size_t>(sd.slot_floats) * per_float;
            f.rings += static_cast<size_t>(d) * static_cast<size_t>(sd.slot_floats) * per_float;
            const size_t nstate = (sd.lam_d ? 1 : 0) + (sd.v_r ? 2 : 0) + (sd.gap ? 1 : 0);
            const size_t plan_state = plan_only ? (opt.policy == FERRET_POLICY_ITER_FISHER ? (opt.eta_lambda > 0.0 ? 3 : 1)
                                                   : opt.policy == FERRET_POLICY_GAP ? 1 : 0)
                                                : nstate;
            f.comp_state += plan_state * static_cast<size_t>(sd.slot_floats) * sizeof(float);
            if (j < 16) f.ring_depth[j] = d;
        }
        const int slots = std::max({need.need_slots, 1, stash_slots});
        total += static_cast<size_t>(slots - stash_slots) * static_cast<size_t>(stash_stride) * sizeof(float);
        f.stash = static_cast<size_t>(slots + 1) * static_cast<size_t>(stash_stride) * sizeof(float);  // + replay slot
        const int ss = std::max(slots + 1, scratch_slots);
        const size_t per_scratch = max_partial * sizeof(float) + max_tiles * sizeof(unsigned);
        total += static_cast<size_t>(ss - scratch_slots) * per_scratch;
        f.scratch = static_cast<size_t>(ss) * per_scratch;
        f.stash_slots = slots;
        f.total = total;
        f.other = total - f.rings - f.comp_state - f.stash - f.scratch;
        return f;
    }

    void build_graph(bool seen_any) {
        HostState probe = hs;
        const PassResult need = run_pass<true>(probe, seen_any);
        for (int j = 0; j < P; ++j) grow_ring(stages[static_cast<size_t>(j)], need.need_depth[static_cast<size_t>(j)]);
        ensure_stash(std::max(need.need_slots, 1));
        ensure_scratch(stash_slots + 1);
        if (timing)
            while (ev_pool.size() < 2 * need.n_updates_timed) {
                cudaEvent_t e;
                cuda_check(cudaEventCreate(&e), "cudaEventCreate");
                ev_pool.push_back(e);
            }
        cuda_check(cudaStreamSynchronize(stream), "sync");
        // timing / profile modes serialise the graph so events bracket one node each
        GraphBuilder builder(timing || profiling);
        wt_reset();  // tap-major weight copies are (re)allocated and (re)prepared inside each graph
        if (profiling) builder.prof_events = &prof_events;
        gb = &builder;
        PassResult got;
        try {
            HostState cap = hs;
            got = run_pass<false>(cap, seen_any);
        } catch (...) {
            gb = nullptr;
            throw;
        }
        gb = nullptr;
        if (builder.done_segments.empty()) {
            cuda_check(cudaGraphInstantiate(&graph_exec, builder.g, 0), "cudaGraphInstantiate");
        } else {
            builder.done_segments.push_back(builder.g);
            builder.g = nullptr;
            for (size_t i = 0; i < builder.done_segments.size(); ++i) {
                cudaGraphExec_t x = nullptr;
                cuda_check(cudaGraphInstantiate(&x, builder.done_segments[i], 0), "cudaGraphInstantiate");
                if (i == 0) graph_exec = x;
                else more_execs.push_back(x);
            }
        }
        launches = builder.kernels;
        prof_ldeps = std::move(builder.ldeps);
        prof_cat = std::move(builder.category);
        prof_bytes = std::move(builder.bytes);
        prof_stage = std::move(builder.stage_of);
        prof_func = std::move(builder.funcs);
        graph_profiling = profiling;
        graph_shape = got;
        graph_timing = timing;
        graph_seen_any = seen_any;
    }

    // One pass over the log. DRY only sizes; otherwise every kernel is
    // launched on `stream`/`nstream` (under capture). `seen_any`: the replay
    // buffer already holds samples at the chunk start.
    template <bool DRY>
    PassResult run_pass(HostState& st, bool seen_any) {
        PassResult res;
        res.need_depth.assign(static_cast<size_t>(P), 2);
        res.pushes.assign(static_cast<size_t>(P), 0);
        const bool as_shipped = opt.as_shipped != 0;
        const size_t n_units = sched.n_units;
        std::vector<long long> rel(static_cast<size_t>(P), 0);  // versions pushed since the chunk start
        std::vector<int> slot_of(n_units, -1);
        std::vector<int> free_slots;
        int slots_used = 0;
        std::vector<char> inflight(n_units, 0);
        std::vector<long long> read_ver(n_units * static_cast<size_t>(P), -1);
        std::vector<std::map<long long, int>> live(static_cast<size_t>(P));  // live read versions per stage
        struct Pend {
            size_t u;
            long long read;
        };
        std::map<std::pair<int, int>, std::vector<Pend>> pending;
        bool buffer_nonempty = seen_any;
        uint64_t n_upd = 0, n_pred = 0;
        std::vector<double> tau_sum(static_cast<size_t>(P), 0.0);
        std::vector<uint64_t> tau_cnt(static_cast<size_t>(P), 0);
        if (!DRY) {
            launches = 0;
            ev_used = 0;
            upd_alg_bytes = 0.0;
            upd_timed = 0;
        }

        auto floor_of = [&](int j) {
            const long long cur = rel[static_cast<size_t>(j)];
            const auto& m = live[static_cast<size_t>(j)];
            return m.empty() ? cur : std::min(m.begin()->first, cur);
        };
        auto note_push = [&](int j) {  // a new version of stage j is about to be written
            const long long span = rel[static_cast<size_t>(j)] - floor_of(j) + 2;
            int& d = res.need_depth[static_cast<size_t>(j)];
            d = std::max(d, static_cast<int>(span));
            if (!DRY && span > stages[static_cast<size_t>(j)].depth)
                fail(FERRET_E_LOGIC, "version ring undersized (dry run disagrees with the real pass)");
        };
        auto stash = [&](size_t u) { return d_stash + static_cast<long long>(slot_of[u]) * stash_stride; };
        auto xrows = [&](size_t u) { return d_xc + u * static_cast<size_t>(B) * static_cast<size_t>(F); };

        using GB = GraphBuilder;
        auto vslot = [&](int j, long long v) {  // resource key of the ring slot holding version v of stage j
            return GB::key(GB::kVSlot, static_cast<uint64_t>(j), static_cast<uint64_t>(v % stages[static_cast<size_t>(j)].depth));
        };
        // a unit's stash regions: activations / deltas of stage r's layers
        auto uact = [&](size_t u, int r) {
            return GB::key(GB::kAct, static_cast<uint64_t>(slot_of[u]), static_cast<uint64_t>(r));
        };
        auto udlt = [&](size_t u, int r) {
            return GB::key(GB::kDlt, static_cast<uint64_t>(slot_of[u]), static_cast<uint64_t>(r));
        };
        auto ngroup = [&](size_t u) { return GB::key(GB::kNorm, u / kNormGroup); };
        // what stage j's work on unit u reads of the stage below: its output activation, or
        // the unit's normalised rows for stage 0
        auto uin = [&](size_t u, int j) { return j > 0 ? uact(u, j - 1) : ngroup(u); };

        // Cross-rank hand-off: every rank numbers every message identically (same
        // log, same pass), so the sender knows where the receiver's inbox slot and
        // flag are. Only the sender emits the send node and only the receiver the
        // recv node; message bytes land in `dst_key` on the receiver.
        std::vector<size_t> in_off(static_cast<size_t>(world), 0), in_flags(static_cast<size_t>(world), 0);
        auto xfer = [&](int src, int dst, auto src_ptr, auto dst_ptr, size_t n, const float* mask, uint64_t key) {
            if (src == dst) return;
            const size_t off = in_off[static_cast<size_t>(dst)], fl = in_flags[static_cast<size_t>(dst)];
            in_off[static_cast<size_t>(dst)] += (n * sizeof(float) + 255) / 256 * 256;
            in_flags[static_cast<size_t>(dst)] += 1;
            if (DRY) return;
            if (rank == src && !peer_data[static_cast<size_t>(dst)])
                fail(FERRET_E_LOGIC, "hand-off to rank " + std::to_string(dst) + ": peer inbox not opened");
            if (rank == src) {
                fb200::SendArgs a{src_ptr(), peer_data[static_cast<size_t>(dst)] + off / sizeof(float),
                                  peer_flags[static_cast<size_t>(dst)] + fl, ctl_epoch(), static_cast<int>(n),
                                  peer_acks[static_cast<size_t>(rank)] + ack_off[static_cast<size_t>(dst)] + fl,
                                  handoff_error()};
                fb200::KernelSpec k;
                fb200::spec_send(a, k);
                gb->cur_category = kCatOther;
                gb->cur_bytes = 4.0 * static_cast<double>(n);
                gb->kernel(k, {key}, {});
            }
            if (rank == dst) {
                if (!peer_acks[static_cast<size_t>(src)])
                    fail(FERRET_E_LOGIC, "hand-off from rank " + std::to_string(src) + ": peer inbox not opened");
                fb200::RecvArgs a{peer_data[static_cast<size_t>(rank)] + off / sizeof(float), dst_ptr(), mask,
                                  peer_flags[static_cast<size_t>(rank)] + fl, ctl_epoch(), static_cast<int>(n),
                                  handoff_error(),
                                  peer_acks[static_cast<size_t>(src)] + ack_off[static_cast<size_t>(rank)] + fl};
                fb200::KernelSpec k;
                fb200::spec_recv(a, k);
                gb->cur_category = kCatOther;
                gb->cur_bytes = 4.0 * static_cast<double>(n);
                gb->kernel(k, {}, {key});
            }
        };

        if (!DRY && mine(0)) {
            // normalizer groups: a chain of their own (mean/m2 state), each unit's
            // ops wait only for the group holding its rows
            const size_t groups = (n_units + kNormGroup - 1) / kNormGroup;
            for (size_t g = 0; g < groups; ++g) {
                const size_t u0 = g * kNormGroup, u1 = std::min(n_units, u0 + kNormGroup);
                const size_t s0 = u0 * static_cast<size_t>(B);
                const size_t ns = (u1 - u0) * static_cast<size_t>(B);
                const size_t o = s0 * static_cast<size_t>(F);
                fb200::NormArgs na{d_rawc + o, static_cast<long long>(ns), F, ctl_count(),
                                   static_cast<unsigned long long>(s0), d_norm_mean, d_norm_m2, d_xc + o, 0,
                                   d_norm_mu + o, d_norm_m2i + o};
                gb->cur_category = kCatNorm; gb->cur_stage = -1;
                // the recurrence (a chain across groups), then the group's rows in parallel
                fb200::KernelSpec kw;
                fb200::spec_welford(na, kw);
                gb->cur_bytes = 24.0 * static_cast<double>(ns) * F;  // raw fp64 in, mean_i / M2_i out
                gb->kernel(kw, {}, {GB::key(GB::kNormScratch, g), GB::key(GB::kNormState, 0)});
                fb200::KernelSpec ks;
                fb200::spec_standardize(na, ks);
                gb->cur_bytes = 28.0 * static_cast<double>(ns) * F;  // raw, mean_i, M2_i in, fp32 out
                gb->kernel(ks, {GB::key(GB::kNormScratch, g)}, {GB::key(GB::kNorm, g)});
            }
        }

        // ---- pending update groups (kernels.cuh GroupArgs): consecutive iter_fisher updates of
        // a stage (one pending gradient each) are collected instead of emitted; the group is
        // emitted as ONE node as soon as a later node would read what it writes (a version it
        // produces, the compensator state) or write what it reads (a member's stash slot, a
        // chain version), when it is full, and at the end of the log. Every node emitted in
        // between touches none of the group's resources, so deferring the members past them
        // is exactly equivalent; the DAG the builder derives is the same one with the
        // members' nodes merged.
        struct PGroup {
            long long cur0 = 0, oldest = 0;
            std::vector<Pend> members;
            std::vector<const float*> stash_of, x0_of;  // captured at join (a unit's slot is freed after its update)
            std::vector<uint64_t> reads, writes;  // sorted, unique
        };
        std::vector<PGroup> groups(static_cast<size_t>(P));
        std::vector<int> last_update_node(static_cast<size_t>(P), -1);  // graph node of stage j's last update
        const bool grouping = !DRY && group_updates && !timing && !as_shipped && opt.policy == FERRET_POLICY_ITER_FISHER;
        auto add_keys = [](std::vector<uint64_t>& v, std::initializer_list<uint64_t> ks) {
            v.insert(v.end(), ks.begin(), ks.end());
        };
        auto tidy = [](std::vector<uint64_t>& v) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
        };
        auto flush_group = [&](int j) {
            PGroup g = std::move(groups[static_cast<size_t>(j)]);
            groups[static_cast<size_t>(j)] = PGroup{};
            if (g.members.empty()) return;
            const StageDev& sd = stages[static_cast<size_t>(j)];
            if (g.members.size() == 1) {  // a lone member: the single-update kernels stream it faster
                fb200::UpdArgs a = update_args(j, g.cur0, g.oldest);
                a.policy = opt.policy;
                a.K = 1;
                a.pend[0] = {g.stash_of[0], g.x0_of[0], static_cast<int>(g.members[0].read - g.oldest)};
                a.step = static_cast<float>(opt.lr);
                fb200::KernelSpec k;
                fb200::spec_update(a, k);
                gb->cur_bytes = update_bytes(j, opt.policy, {g.members[0].read}, g.cur0);
                gb->cur_category = kCatUpdate;
                gb->cur_stage = j;
                if (update_pdl) gb->pdl_pred = last_update_node[static_cast<size_t>(j)];
                gb->kernel(k, g.reads, g.writes);
                last_update_node[static_cast<size_t>(j)] = static_cast<int>(gb->nodes.size()) - 1;
                wt_invalidate(sd, a.dst);
                ++n_single_groups;
                return;
            }
            fb200::GroupArgs a{};
            a.works = sd.works_g_dev;
            a.n_gsegs = static_cast<int>(sd.gsegs.size());
            for (size_t q = 0; q < sd.gsegs.size(); ++q) a.gseg[q] = sd.gsegs[q];
            a.n_tiles = sd.n_tiles_g;
            a.n_wtiles = sd.n_wtiles_g;
            a.B = B;
            a.G = static_cast<int>(g.members.size());
            a.n0 = static_cast<int>(g.cur0 - g.oldest + 1);
            a.learn = (opt.eta_lambda > 0.0 && sd.v_r) ? 1 : 0;
            for (long long v = g.oldest; v <= g.cur0; ++v) a.vers[v - g.oldest] = sd.slot(v);
            for (size_t k = 0; k < g.members.size(); ++k) {
                const Pend& m = g.members[k];
                a.pend[k] = {g.stash_of[k], g.x0_of[k], static_cast<int>(m.read - g.oldest)};
                a.dst[k] = sd.slot(g.cur0 + 1 + static_cast<long long>(k));
                a.dst16[k] = sd.ring16 ? const_cast<uint16_t*>(sd.shadow(a.dst[k])) : nullptr;
            }
            a.x0idx = nullptr;
            a.x0_ld = F;
            a.lam_d = sd.lam_d;
            a.v_r = sd.v_r;
            a.v_a = sd.v_a;
            a.lambda0 = static_cast<float>(opt.lambda0);
            a.alpha = static_cast<float>(opt.alpha);
            a.eta = static_cast<float>(opt.eta_lambda);
            a.nu = static_cast<float>(opt.nu);
            a.step = static_cast<float>(opt.lr * (1.0 / 1.0));
            fb200::KernelSpec k;
            fb200::spec_update_group(a, k);
            gb->cur_bytes = group_bytes(j, a.n0, a.G);
            gb->cur_category = kCatUpdate;
            gb->cur_stage = j;
            gb->kernel(k, g.reads, g.writes);
            // no programmatic edge out of a group: a chained single update loads its older versions
            // before griddepcontrol.wait, and a group writes several of them
            last_update_node[static_cast<size_t>(j)] = -1;
            for (int q = 0; q < a.G; ++q) wt_invalidate(sd, a.dst[q]);
            ++n_group_nodes;
        };
        auto hits = [](const std::vector<uint64_t>& sorted, const std::vector<uint64_t>& keys) {
            for (uint64_t x : keys)
                if (std::binary_search(sorted.begin(), sorted.end(), x)) return true;
            return false;
        };
        struct HookReset {
            GraphBuilder* b;
            ~HookReset() {
                if (b) b->before = nullptr;
            }
        } hook_reset{grouping ? gb : nullptr};
        if (grouping)
            gb->before = [&](const std::vector<uint64_t>& r, const std::vector<uint64_t>& w) {
                for (int q = 0; q < P; ++q) {
                    const PGroup& g = groups[static_cast<size_t>(q)];
                    if (g.members.empty()) continue;
                    if (hits(g.writes, r) || hits(g.writes, w) || hits(g.reads, w)) flush_group(q);
                }
            };
        if (!DRY) n_group_nodes = n_single_groups = 0;

        for (size_t idx = 0; idx < sched.events.size(); ++idx) {
            if (!DRY && !gb->prof_events && gb->nodes_in_segment() >= seg_nodes) gb->new_segment();
            const ferret_event& e = sched.events[idx];
            const size_t u = static_cast<size_t>(e.item);
            const int j = e.stage;
            switch (e.kind) {
                case FERRET_EV_ARRIVAL: {  // learner.hpp:389-410
                    if (sched.dropped[u]) break;
                    inflight[u] = 1;
                    if (!as_shipped) {
                        if (free_slots.empty()) free_slots.push_back(slots_used++);
                        slot_of[u] = free_slots.back();
                        free_slots.pop_back();
                    }
                    ++n_pred;
                    emit_predict<DRY>(u, rel, as_shipped ? -1 : slot_of[u], xfer, vslot, ngroup);
                    if (opt.replay && !as_shipped) {
                        buffer_nonempty = true;
                        if (!DRY && mine(0)) {
                            fb200::PoolArgs pa{xrows(u), d_labc + u * static_cast<size_t>(B),
                                               ctl_pool_dst() + u * static_cast<size_t>(B), d_pool_x, d_pool_lab, B, F};
                            fb200::KernelSpec k;
                            fb200::spec_pool(pa, k);
                            gb->cur_bytes = 8.0 * B * F;
                            gb->cur_category = kCatOther; gb->cur_stage = -1;
                            gb->kernel(k, {ngroup(u)}, {GB::key(GB::kPool, 0)});
                        }
                    }
                    break;
                }
                case FERRET_EV_FORWARD: {  // learner.hpp:412-433
                    if (as_shipped || !inflight[u]) break;
                    const long long v = rel[static_cast<size_t>(j)];
                    read_ver[u * static_cast<size_t>(P) + static_cast<size_t>(j)] = v;
                    if (sched.has_bwd[u * static_cast<size_t>(P) + static_cast<size_t>(j)]) live[static_cast<size_t>(j)][v] += 1;
                    if (!DRY && mine(j))
                        launch_stage_forward(j, stages[static_cast<size_t>(j)].slot(v), stash(u), xrows(u),
                                             {vslot(j, v), ngroup(u), uin(u, j)},
                                             j == P - 1 ? std::vector<uint64_t>{uact(u, j), udlt(u, j)}
                                                        : std::vector<uint64_t>{uact(u, j)},
                                             d_labc + u * static_cast<size_t>(B));
                    if (j + 1 < P) {  // hand the stage output to the next stage's rank
                        const LayerDev& top = layers[static_cast<size_t>(stages[static_cast<size_t>(j)].hi - 1)];
                        const long long off = top.act_off;
                        xfer(owner[static_cast<size_t>(j)], owner[static_cast<size_t>(j + 1)], [&] { return stash(u) + off; },
                             [&] { return stash(u) + off; }, static_cast<size_t>(B) * top.out, nullptr, uact(u, j));
                    }
                    break;
                }
                case FERRET_EV_BACKWARD: {  // learner.hpp:435-479
                    if (as_shipped || !inflight[u]) break;
                    const long long r = read_ver[u * static_cast<size_t>(P) + static_cast<size_t>(j)];
                    if (r < 0) fail(FERRET_E_OUT_OF_RANGE, "stage version evicted");
                    // the input gradient of the stage's first layer goes to stage j-1;
                    // across ranks it is sent unmasked (the ReLU mask lives there)
                    const bool cross = j > 0 && owner[static_cast<size_t>(j - 1)] != owner[static_cast<size_t>(j)];
                    if (!DRY && mine(j))
                        launch_stage_backward(j, stages[static_cast<size_t>(j)].slot(r), stash(u),
                                              d_labc + u * static_cast<size_t>(B), slot_of[u],
                                              {vslot(j, r), ngroup(u), uin(u, j), uact(u, j)},
                                              j > 0 ? std::vector<uint64_t>{udlt(u, j), udlt(u, j - 1)}
                                                    : std::vector<uint64_t>{udlt(u, j)},
                                              cross, xrows(u));
                    if (cross && sched.has_bwd[u * static_cast<size_t>(P) + static_cast<size_t>(j - 1)]) {
                        const LayerDev& below = layers[static_cast<size_t>(stages[static_cast<size_t>(j)].lo - 1)];
                        const long long doff = below.dlt_off, aoff = below.act_off;
                        const bool relu = below.act == FERRET_ACT_RELU;
                        xfer(owner[static_cast<size_t>(j)], owner[static_cast<size_t>(j - 1)], [&] { return stash(u) + doff; },
                             [&] { return stash(u) + doff; }, static_cast<size_t>(B) * below.out,
                             relu ? stash(u) + aoff : nullptr, udlt(u, j - 1));
                    }
                    pending[{e.worker, j}].push_back({u, r});
                    break;
                }
                case FERRET_EV_UPDATE: {  // learner.hpp:491-510
                    if (as_shipped) break;
                    auto it = pending.find({e.worker, j});
                    if (it == pending.end() || it->second.empty()) break;
                    const std::vector<Pend>& pl = it->second;
                    if (pl.size() > static_cast<size_t>(fb200::kMaxPending))
                        fail(FERRET_E_CONFIG, "accumulation count above 16 is not supported by the update kernel");
                    note_push(j);
                    const long long cur = rel[static_cast<size_t>(j)];
                    long long oldest = cur;
                    for (const Pend& p : pl) {
                        tau_sum[static_cast<size_t>(j)] += static_cast<double>(cur - p.read);
                        tau_cnt[static_cast<size_t>(j)] += 1;
                        oldest = std::min(oldest, p.read);
                    }
                    ++n_upd;
                    if (timing && mine(j)) ++res.n_updates_timed;
                    const bool join = grouping && mine(j) && pl.size() == 1 && stages[static_cast<size_t>(j)].group_ok &&
                                      stages[static_cast<size_t>(j)].lam_d &&
                                      (cur - pl[0].read + 2) <= fb200::kGroupChainMax;
                    if (join) {
                        PGroup& g = groups[static_cast<size_t>(j)];
                        const long long rd = pl[0].read;
                        if (!g.members.empty()) {
                            const long long span = (g.cur0 - std::min(g.oldest, rd) + 1) +
                                                   static_cast<long long>(g.members.size()) + 1;
                            if (static_cast<int>(g.members.size()) >= fb200::kGroupMax || span > fb200::kGroupChainMax)
                                flush_group(j);
                        }
                        if (g.members.empty()) {
                            g.cur0 = cur;
                            g.oldest = rd;
                        } else if (cur != g.cur0 + static_cast<long long>(g.members.size()) || rd > g.cur0) {
                            fail(FERRET_E_LOGIC, "update group: a stage version advanced outside its pending group");
                        }
                        g.oldest = std::min(g.oldest, rd);
                        g.members.push_back(pl[0]);
                        g.stash_of.push_back(stash(pl[0].u));
                        g.x0_of.push_back(xrows(pl[0].u));
                        add_keys(g.reads, {uin(pl[0].u, j), uact(pl[0].u, j), udlt(pl[0].u, j), ngroup(pl[0].u)});
                        for (long long v = rd; v <= g.cur0; ++v) g.reads.push_back(vslot(j, v));
                        add_keys(g.writes, {vslot(j, cur + 1), GB::key(GB::kState, static_cast<uint64_t>(j))});
                        tidy(g.reads);
                        tidy(g.writes);
                    }
                    if (!DRY && mine(j) && !join) {
                        fb200::UpdArgs a = update_args(j, cur, oldest);
                        a.policy = opt.policy;
                        a.K = static_cast<int>(pl.size());
                        std::vector<long long> reads;
                        std::vector<uint64_t> rk;
                        for (size_t k = 0; k < pl.size(); ++k) {
                            a.pend[k] = {stash(pl[k].u), xrows(pl[k].u), static_cast<int>(pl[k].read - oldest)};
                            reads.push_back(pl[k].read);
                            rk.push_back(uin(pl[k].u, j));
                            rk.push_back(uact(pl[k].u, j));
                            rk.push_back(udlt(pl[k].u, j));
                            rk.push_back(ngroup(pl[k].u));
                        }
                        for (long long v = oldest; v <= cur; ++v) rk.push_back(vslot(j, v));
                        a.step = static_cast<float>(opt.lr * (1.0 / static_cast<double>(pl.size())));
                        fb200::KernelSpec k;
                        fb200::spec_update(a, k);
                        gb->cur_bytes = update_bytes(j, opt.policy, reads, cur);
                        time_begin();
                        gb->cur_category = kCatUpdate; gb->cur_stage = j;
                        if (update_pdl && !timing) gb->pdl_pred = last_update_node[static_cast<size_t>(j)];
                        gb->kernel(k, rk, {vslot(j, cur + 1), GB::key(GB::kState, static_cast<uint64_t>(j))});
                        last_update_node[static_cast<size_t>(j)] = static_cast<int>(gb->nodes.size()) - 1;
                        wt_invalidate(stages[static_cast<size_t>(j)], a.dst);
                        time_end(update_bytes(j, opt.policy, reads, cur));
                    }
                    rel[static_cast<size_t>(j)] += 1;
                    res.pushes[static_cast<size_t>(j)] += 1;
                    for (const Pend& p : pl) {
                        auto& m = live[static_cast<size_t>(j)];
                        auto lv = m.find(p.read);
                        if (lv != m.end() && --lv->second == 0) m.erase(lv);
                    }
                    it->second.clear();
                    if (j == 0 && opt.replay && buffer_nonempty) {  // learner.hpp:509, 513-519
                        replay_step<DRY>(res.n_replays, rel, note_push, vslot, xfer);
                        for (int s = 0; s < P; ++s) res.pushes[static_cast<size_t>(s)] += 1;
                        ++res.n_replays;
                    }
                    break;
                }
                default: break;  // drop, recompute: no trainer work (learner.hpp:359)
            }
            if (!as_shipped)
                for (size_t fu : sched.free_at[idx])
                    if (slot_of[fu] >= 0) {
                        free_slots.push_back(slot_of[fu]);
                        slot_of[fu] = -1;
                    }
        }
        for (int q = 0; q < P; ++q) flush_group(q);
        if (!DRY) {
            // leave every stage's live version in slot 0 for the next chunk
            for (int j = 0; j < P; ++j) {
                const StageDev& s = stages[static_cast<size_t>(j)];
                const long long fin = rel[static_cast<size_t>(j)] % s.depth;
                if (fin != 0 && mine(j)) {
                    gb->cur_category = kCatOther;
                    gb->cur_stage = -1;
                    gb->cur_bytes = 8.0 * static_cast<double>(s.slot_floats);
                    gb->copy(s.ring, s.slot(fin), static_cast<size_t>(s.slot_floats) * sizeof(float), {vslot(j, fin)},
                             {vslot(j, 0)});
                    wt_invalidate(s, s.ring);
                    if (s.ring16)
                        gb->copy(s.ring16, s.shadow(s.slot(fin)), static_cast<size_t>(s.slot_floats) * sizeof(uint16_t),
                                 {vslot(j, fin)}, {vslot(j, 0)});
                }
            }
            stats.events = sched.events.size();
            stats.updates = n_upd;
            stats.replays = res.n_replays;
            stats.predicts = n_pred;
            for (int j = 0; j < P && j < 16; ++j) {
                const double cnt = static_cast<double>(tau_cnt[static_cast<size_t>(j)]);
                stats.mean_tau[j] = cnt > 0 ? tau_sum[static_cast<size_t>(j)] / cnt : 0.0;
                stats.update_elems[j] = static_cast<uint64_t>(stages[static_cast<size_t>(j)].n_params) *
                                        tau_cnt[static_cast<size_t>(j)];
            }
        }
        res.need_slots = slots_used;
        res.inbox_bytes = in_off;
        res.inbox_flags = in_flags;
        (void)st;
        return res;
    }

    // Launch arguments of one update of stage j: the chain table holds the
    // versions oldest_read .. cur (ring slots resolved here), dst = slot(cur+1).
    fb200::UpdArgs update_args(int j, long long cur, long long oldest) {
        const StageDev& s = stages[static_cast<size_t>(j)];
        fb200::UpdArgs a{};
        a.n_segs = s.n_segs;
        a.gmat = s.gmat ? 1 : 0;
        a.n_items = s.n_items;
        a.n_elems = s.slot_floats;
        a.B = B;
        a.segs = s.segs_dev;
        a.tiles = s.tiles_dev;
        a.works = s.works_dev;
        a.works4 = s.works4_dev;
        a.n_tiles4 = s.n_tiles4;
        a.threads4 = s.threads4;
        a.n_tiles = s.n_tiles;
        a.x0idx = nullptr;
        a.x0_ld = F;
        if (cur - oldest + 1 > fb200::kMaxChain)
            fail(FERRET_E_CONFIG, "staleness chain longer than 48 versions is not supported by the update kernel");
        a.nv = static_cast<int>(cur - oldest + 1);
        for (long long v = oldest; v <= cur; ++v) a.vers[v - oldest] = s.slot(v);
        a.dst = s.slot(cur + 1);
        a.dst16 = s.ring16 ? const_cast<uint16_t*>(s.shadow(a.dst)) : nullptr;
        a.lam_d = s.lam_d;
        a.v_r = s.v_r;
        a.v_a = s.v_a;
        a.gap = s.gap;
        a.lambda0 = static_cast<float>(opt.lambda0);
        a.alpha = static_cast<float>(opt.alpha);
        a.eta = static_cast<float>(opt.eta_lambda);
        a.nu = static_cast<float>(opt.nu);
        return a;
    }

    // ----------------------------------------------------- node helpers
    // One dense layer on B samples (input row b = X + (xidx ? xidx[b] : b) * in).
    // split-K scratch of the tensor-core layers, one region per written resource
    // (nodes writing the same resource are serialised by the DAG, so they can
    // share it); allocated while the graph is built, counters zeroed
    std::map<uint64_t, std::pair<float*, unsigned*>> mma_scratch;
    size_t mma_partial_floats = 0, mma_counter_n = 0;
    std::pair<float*, unsigned*> mma_scratch_for(uint64_t key) {
        auto it = mma_scratch.find(key);
        if (it != mma_scratch.end()) return it->second;
        if (!mma_partial_floats) {
            const bool bf16 = opt.precision == FERRET_PREC_BF16;
            for (const LayerDev& ld : layers)
                for (bool bwd : {false, true}) {
                    if (ld.kind != FERRET_LAYER_DENSE) continue;
                    const fb200::MmaGeom g =
                        fb200::mma_geom(bf16, bwd, ld.in, ld.out, opt.precision == FERRET_PREC_FP32);
                    mma_partial_floats = std::max(mma_partial_floats, g.partial_floats);
                    mma_counter_n = std::max(mma_counter_n, static_cast<size_t>(g.mtiles));
                }
        }
        float* p = dalloc<float>(std::max<size_t>(mma_partial_floats, 1), device_bytes);
        unsigned* c = dalloc<unsigned>(mma_counter_n, device_bytes);
        if (c) cuda_check(cudaMemset(c, 0, mma_counter_n * sizeof(unsigned)), "memset");
        return mma_scratch[key] = {p, c};
    }

    // fast modes: this layer's forward / input gradient runs on the tensor cores
    // Layers under 256K weights stay on the SIMT kernels in the fast modes too: on
    // config 2 (layers of 200K and 65K weights, many kernels in flight) the tensor-core
    // path is neutral at 200K and slower at 65K (profiles/README.md).
    // FERRET_MMA_MIN_PARAMS overrides the threshold (tests force 0).
    long long mma_min_params =
        std::getenv("FERRET_MMA_MIN_PARAMS") ? std::atoll(std::getenv("FERRET_MMA_MIN_PARAMS")) : (1LL << 18);
    // fp32 parity mode: layers of >= 1M weights run the fp32-accurate 3xTF32 split on the
    // tensor cores (FERRET_SPLIT_MIN_PARAMS overrides; 0 = every layer, -1 = none)
    long long split_min_params =
        std::getenv("FERRET_SPLIT_MIN_PARAMS") ? std::atoll(std::getenv("FERRET_SPLIT_MIN_PARAMS")) : (1LL << 20);
    bool use_split(const LayerDev& ld) const {
        return ld.kind == FERRET_LAYER_DENSE && opt.precision == FERRET_PREC_FP32 && split_min_params >= 0 &&
               static_cast<long long>(ld.in) * ld.out >= split_min_params && fb200::mma_supported(false, ld.in, ld.out);
    }
    bool use_mma(const LayerDev& ld) const {
        if (opt.precision == FERRET_PREC_FP32) return use_split(ld);
        return ld.kind == FERRET_LAYER_DENSE && static_cast<long long>(ld.in) * ld.out >= mma_min_params &&
               fb200::mma_supported(opt.precision == FERRET_PREC_BF16, ld.in, ld.out);
    }
    void emit_mma(const LayerDev& ld, const float* stage_slot, bool bwd, const float* X, const int* xidx,
                  const float* mask, float* Y, const std::vector<uint64_t>& reads, const std::vector<uint64_t>& writes) {
        const bool bf16 = opt.precision == FERRET_PREC_BF16;
        const StageDev& s = stages[static_cast<size_t>(ld.stage)];
        fb200::MmaLayer m;
        m.W = bf16 ? static_cast<const void*>(s.shadow(stage_slot + ld.woff)) : static_cast<const void*>(stage_slot + ld.woff);
        m.bwd = bwd;
        m.bf16 = bf16;
        m.split = opt.precision == FERRET_PREC_FP32;
        m.bias = bwd ? nullptr : stage_slot + ld.boff;
        m.X = X;
        m.xidx = xidx;
        m.mask = mask;
        m.Y = Y;
        m.in = ld.in;
        m.out = ld.out;
        m.B = B;
        m.relu = !bwd && ld.act == FERRET_ACT_RELU;
        if (!plan_only) std::tie(m.partial, m.counters) = mma_scratch_for(writes.at(0));
        fb200::KernelSpec k;
        if (!plan_only) fb200::spec_mma(m, k);
        const double wbytes = (bf16 ? 2.0 : 4.0) * ld.in * ld.out;
        gb->cur_bytes = bwd ? wbytes + 4.0 * B * (ld.out + 2.0 * ld.in)
                            : wbytes + 4.0 * ld.out + 4.0 * B * (ld.in + ld.out);
        gb->kernel(k, reads, writes);
    }

    bool can_fuse_head() const {
        const LayerDev& last = layers.back();
        return !use_mma(last) && !last.conv() && fb200::fwd_single_cta(last.cols, last.rows, B, last.cols % 4 == 0);
    }

    // `blk`: the block input (input of layer l-1) of a residual convolution;
    // `pooled`: B x c_in scratch of a gap_dense layer
    void emit_layer(const LayerDev& ld, const float* stage_slot, const float* X, const int* xidx, float* Y,
                    const std::vector<uint64_t>& reads, const std::vector<uint64_t>& writes,
                    const Head& head = Head{}, const float* blk = nullptr, float* pooled = nullptr) {
        if (ld.conv()) {
            fb200::ConvArgs c = conv_args(ld);
            c.W = stage_slot + ld.woff;
            c.bias = stage_slot + ld.boff;
            c.X = X;
            c.xidx = xidx;
            c.Y = Y;
            c.relu = ld.act == FERRET_ACT_RELU;
            if (ld.res) {
                const LayerDev& a = layers[static_cast<size_t>(&ld - layers.data() - 1)];
                c.res = blk;
                c.rc = a.ci;
                c.rh = a.hi;
                c.rw = a.wi;
            }
            return emit_conv(c, fb200::kConvFwd, reads, writes,
                             4.0 * (ld.nw() + ld.rows) + 4.0 * B * (ld.in + ld.out) + (ld.res ? 4.0 * B * ld.out : 0.0));
        }
        if (ld.gap()) {
            fb200::PoolMeanArgs g{X, xidx, pooled, nullptr, nullptr, nullptr, B, ld.ci, ld.hi * ld.wi};
            fb200::KernelSpec kg;
            fb200::spec_gap(g, kg);
            gb->cur_bytes = 4.0 * B * (ld.in + ld.ci);
            gb->kernel(kg, reads, writes);
            X = pooled;
            xidx = nullptr;
        }
        if (use_mma(ld)) return emit_mma(ld, stage_slot, false, X, xidx, nullptr, Y, reads, writes);
        fb200::FwdArgs a{};
        a.head_mode = head.mode;
        a.labels = head.labels;
        a.pred = head.pred;
        a.delta = head.delta;
        a.scale = head.scale;
        a.W = stage_slot + ld.woff;
        a.bias = stage_slot + ld.boff;
        a.X = X;
        a.xidx = xidx;
        a.Y = Y;
        a.in = ld.cols;
        a.out = ld.rows;
        a.B = B;
        a.relu = ld.act == FERRET_ACT_RELU;
        fb200::KernelSpec k;
        fb200::spec_fwd(a, k);
        gb->cur_bytes = 4.0 * ld.cols * ld.rows + 4.0 * ld.rows + 4.0 * B * (ld.cols + ld.rows);  // W, b, X, Y
        gb->kernel(k, reads, writes);
    }

    // ------------------------------------------------ convolutions (conv.cu)
    static constexpr size_t kConvPartialCap = size_t{1} << 22;  // split-K partial floats per scratch region
    std::map<uint64_t, float*> conv_scratch;
    // convolutions on the tensor cores: fp32 parity mode 3xTF32, fast modes tf32 / bf16;
    // FERRET_CONV_TC overrides (0 = the SIMT kernels)
    int conv_tc = std::getenv("FERRET_CONV_TC") ? std::atoi(std::getenv("FERRET_CONV_TC")) : -1;
    fb200::ConvArgs conv_args(const LayerDev& ld) const {
        fb200::ConvArgs c{};
        c.tc = conv_tc >= 0 ? conv_tc
               : opt.precision == FERRET_PREC_BF16 ? 2 : opt.precision == FERRET_PREC_TF32 ? 1 : 3;
        c.B = B;
        c.ci = ld.ci;
        c.hi = ld.hi;
        c.wi = ld.wi;
        c.co = ld.co;
        c.ho = ld.ho;
        c.wo = ld.wo;
        c.k = ld.k;
        c.s = ld.st;
        c.p = ld.pad;
        return c;
    }
    // split-K scratch, one region per written resource (nodes writing the same
    // resource are serialised by the DAG)
    float* conv_scratch_for(uint64_t key) {
        auto it = conv_scratch.find(key);
        if (it != conv_scratch.end()) return it->second;
        return conv_scratch[key] = dalloc<float>(kConvPartialCap, device_bytes);
    }
    // tap-major weight copies for the tensor-core A operand: one buffer per (weight version
    // slot + layer, direction), valid from its prep node until the slot is rewritten
    std::map<std::pair<const float*, int>, std::pair<float*, uint32_t>> wt_buf;
    std::set<std::pair<const float*, int>> wt_valid;
    size_t wt_bytes = 0;
    // Called before every graph build (the previous graph is already destroyed): ring
    // reallocation (grow_ring) may hand a freed slot's address to another stage or layer,
    // so a pointer-keyed buffer must never outlive the graph it was sized for.
    void wt_reset() {
        for (auto& kv : wt_buf) dfree(kv.second.first);
        device_bytes -= wt_bytes;
        wt_bytes = 0;
        wt_buf.clear();
        wt_valid.clear();
    }
    void wt_invalidate(const StageDev& s, const float* slot) {
        for (auto it = wt_valid.begin(); it != wt_valid.end();)
            it = (it->first >= slot && it->first < slot + s.slot_floats) ? wt_valid.erase(it) : std::next(it);
    }
    void emit_conv(fb200::ConvArgs& c, int mode, const std::vector<uint64_t>& reads, const std::vector<uint64_t>& writes,
                   double bytes) {
        fb200::conv_plan(c, mode, kConvPartialCap);
        if (c.splits > 1) c.partial = conv_scratch_for(writes.at(0));
        std::vector<uint64_t> rd = reads;
        if (c.kt && mode != fb200::kConvWgrad) {
            // the tap-major copy of this weight version, prepared once per version inside the
            // graph and reused by every launch that reads the version (predict, forward, input
            // gradient, replay); the update writing the slot invalidates it (wt_invalidate)
            const std::pair<const float*, int> k{c.W, mode};
            auto it = wt_buf.find(k);
            if (it == wt_buf.end()) {
                float* buf = dalloc<float>(static_cast<size_t>(c.M) * c.K, device_bytes);
                wt_bytes += static_cast<size_t>(c.M) * c.K * sizeof(float);
                it = wt_buf.emplace(k, std::make_pair(buf, static_cast<uint32_t>(wt_buf.size()))).first;
            }
            c.Wt = it->second.first;
            const uint64_t wk = GraphBuilder::key(GraphBuilder::kWt, it->second.second);
            if (!wt_valid.count(k)) {
                fb200::KernelSpec kw;
                fb200::spec_conv_wprep(c, mode, kw);
                gb->cur_bytes = 8.0 * static_cast<double>(c.M) * c.K;
                gb->kernel(kw, reads, {wk});
                wt_valid.insert(k);
            }
            rd.push_back(wk);
        }
        fb200::KernelSpec g, r;
        const int n = fb200::spec_conv(c, mode, g, r);
        gb->cur_bytes = bytes;
        gb->kernel(g, rd, writes);
        if (n == 2) {
            gb->cur_bytes = 8.0 * c.splits * static_cast<double>(c.M) * c.N;
            gb->kernel(r, rd, writes);
        }
    }
    // the weight and bias gradient of convolution `ld` into its stash region
    void emit_conv_wgrad(const LayerDev& ld, float* stash_u, const float* X, const int* xidx,
                         const std::vector<uint64_t>& reads, const std::vector<uint64_t>& writes) {
        fb200::ConvArgs c = conv_args(ld);
        c.X = X;
        c.xidx = xidx;
        c.D = stash_u + ld.dlt_off;
        c.Y = stash_u + ld.g_off;
        // tensor cores: the bias gradient is the GEMM's extra ones column (one launch less per weight
        // gradient; FERRET_CONV_BIAS_COL=0: the separate conv_bgrad_kernel)
        c.bcol = c.tc && !(std::getenv("FERRET_CONV_BIAS_COL") && std::atoi(std::getenv("FERRET_CONV_BIAS_COL")) == 0);
        emit_conv(c, fb200::kConvWgrad, reads, writes, 4.0 * ld.nw() + 4.0 * B * (ld.in + ld.out));
        if (c.bcol) return;
        fb200::KernelSpec kb;
        fb200::spec_conv_bgrad(c, stash_u + ld.g_off + ld.nw(), kb);
        gb->cur_bytes = 4.0 * B * ld.out + 4.0 * ld.rows;
        gb->kernel(kb, reads, writes);
    }

    // predict_class(net_, x) at the arrival (learner.hpp:398-399): full net at
    // the live versions, ping-pong scratch inside the unit's stash slot (as
    // shipped there is no slot: the replay stash's scratch is used, serialised).
    // Where the next stage lives on another rank the running activation is
    // handed over.
    template <bool DRY, class Xfer, class VSlot, class NGroup>
    void emit_predict(size_t u, const std::vector<long long>& rel, int slot, Xfer& xfer, VSlot& vslot, NGroup& ngroup) {
        using GB = GraphBuilder;
        float* scratch = (slot >= 0 ? d_stash + static_cast<long long>(slot) * stash_stride : d_replay) + pred_off;
        const uint64_t sk = slot >= 0 ? GB::key(GB::kPred, static_cast<uint64_t>(slot)) : GB::key(GB::kReplay, 0);
        const float* x0 = d_xc + u * static_cast<size_t>(B) * static_cast<size_t>(F);
        for (int j = 0; j < P; ++j) {
            const StageDev& s = stages[static_cast<size_t>(j)];
            if (j > 0) {
                const int l = s.lo - 1;
                float* buf = scratch + (l % 3) * pred_stride;
                xfer(owner[static_cast<size_t>(j - 1)], owner[static_cast<size_t>(j)], [&] { return buf; },
                     [&] { return buf; }, static_cast<size_t>(B) * layers[static_cast<size_t>(l)].out, nullptr, sk);
            }
            if (DRY || !mine(j)) continue;
            gb->cur_category = kCatPredict;
            gb->cur_stage = -1;
            const std::vector<uint64_t> reads{vslot(j, rel[static_cast<size_t>(j)]), ngroup(u)};
            for (int l = s.lo; l < s.hi; ++l) {
                const float* X = l == 0 ? x0 : scratch + ((l - 1) % 3) * pred_stride;
                Head h;
                if (l == L - 1 && can_fuse_head()) {
                    h.mode = 0;
                    h.pred = d_predc + u * static_cast<size_t>(B);
                }
                const LayerDev& ld = layers[static_cast<size_t>(l)];
                // the block input of a residual layer is the input of layer l-1: buffer (l-2) % 3,
                // which a gap_dense layer (never residual) uses as its pooled scratch
                float* third = scratch + ((l + 1) % 3) * pred_stride;
                emit_layer(ld, s.slot(rel[static_cast<size_t>(j)]), X, nullptr, scratch + (l % 3) * pred_stride, reads,
                           {sk}, h, ld.res ? third : nullptr, ld.gap() ? third : nullptr);
            }
        }
        if (DRY || !mine(P - 1) || can_fuse_head()) return;
        fb200::HeadArgs h{};
        h.logits = scratch + ((L - 1) % 3) * pred_stride;
        h.n_out = n_out;
        h.B = B;
        h.mode = 0;
        h.pred = d_predc + u * static_cast<size_t>(B);
        fb200::KernelSpec k;
        fb200::spec_head(h, k);
        gb->cur_bytes = 4.0 * B * n_out + 4.0 * B;
        gb->kernel(k, {}, {sk});
    }

    void launch_stage_forward(int j, const float* slot, float* stash_u, const float* x0, const std::vector<uint64_t>& reads,
                              const std::vector<uint64_t>& writes, const int* lab) {
        gb->cur_category = kCatForward;
        gb->cur_stage = j;
        const StageDev& s = stages[static_cast<size_t>(j)];
        for (int l = s.lo; l < s.hi; ++l) {
            const LayerDev& ld = layers[static_cast<size_t>(l)];
            const float* X = l == 0 ? x0 : stash_u + layers[static_cast<size_t>(l - 1)].act_off;
            // the logits' delta (learner.hpp:443-447) is a function of the stashed logits and
            // the labels alone: computed here, consumed by the stage's backward
            Head h;
            if (l == L - 1 && can_fuse_head()) {
                h.mode = 1;
                h.labels = lab;
                h.delta = stash_u + ld.dlt_off;
                h.scale = 1.0f / static_cast<float>(B);
            }
            emit_layer(ld, slot, X, nullptr, stash_u + ld.act_off, reads, writes, h,
                       ld.res ? stash_u + layers[static_cast<size_t>(l - 2)].act_off : nullptr,
                       ld.gap() ? stash_u + ld.pool_off : nullptr);
        }
    }

    // delta at the logits (last stage) then per layer prev = W^T delta with the
    // ReLU mask of the layer below applied on write (learner.hpp:443-476);
    // `cross`: the stage below is on another rank, which applies the mask.
    void launch_stage_backward(int j, const float* slot, float* stash_u, const int* lab, int scratch,
                               const std::vector<uint64_t>& reads, const std::vector<uint64_t>& writes, bool cross,
                               const float* x0 = nullptr, const int* x0idx = nullptr) {
        gb->cur_category = kCatBackward;
        gb->cur_stage = j;
        const StageDev& s = stages[static_cast<size_t>(j)];
        if (j == P - 1 && !can_fuse_head()) emit_delta_head(stash_u, lab, nullptr, 1.0f / static_cast<float>(B), reads, writes);
        for (int l = s.hi - 1; l >= s.lo; --l) {
            const LayerDev& ld = layers[static_cast<size_t>(l)];
            if (ld.conv())  // a convolution's weight gradient is materialised for the update
                emit_conv_wgrad(ld, stash_u, l == 0 ? x0 : stash_u + layers[static_cast<size_t>(l - 1)].act_off,
                                l == 0 ? x0idx : nullptr, reads, writes);
            if (l == 0) break;  // no input gradient for the first layer
            emit_layer_backward(l, slot, stash_u, scratch, reads, writes, !(cross && l == s.lo));
        }
    }

    void emit_delta_head(float* stash_u, const int* lab, const int* lidx, float scale, const std::vector<uint64_t>& reads,
                         const std::vector<uint64_t>& writes) {
        const LayerDev& last = layers.back();
        fb200::HeadArgs h{};
        h.logits = stash_u + last.act_off;
        h.n_out = n_out;
        h.B = B;
        h.mode = 1;
        h.labels = lab;
        h.lidx = lidx;
        h.delta = stash_u + last.dlt_off;
        h.scale = scale;
        fb200::KernelSpec k;
        fb200::spec_head(h, k);
        gb->cur_bytes = 8.0 * B * n_out;
        gb->kernel(k, reads, writes);
    }

    void emit_layer_backward(int l, const float* slot, float* stash_u, int scratch, const std::vector<uint64_t>& reads,
                             const std::vector<uint64_t>& writes, bool mask_on_write = true) {
        const LayerDev& ld = layers[static_cast<size_t>(l)];
        const LayerDev& below = layers[static_cast<size_t>(l - 1)];
        const float* mask = mask_on_write && below.act == FERRET_ACT_RELU ? stash_u + below.act_off : nullptr;
        if (ld.conv()) {  // transposed convolution, plus the shortcut's gradient when a residual layer sits above
            fb200::ConvArgs c = conv_args(ld);
            c.W = slot + ld.woff;
            c.D = stash_u + ld.dlt_off;
            c.Y = stash_u + below.dlt_off;
            c.mask = mask;
            if (l + 1 < L && layers[static_cast<size_t>(l + 1)].res) {
                const LayerDev& r = layers[static_cast<size_t>(l + 1)];
                c.res = stash_u + r.dlt_off;
                c.rc = r.co;
                c.rh = r.ho;
                c.rw = r.wo;
            }
            return emit_conv(c, fb200::kConvDgrad, reads, writes,
                             4.0 * ld.nw() + 4.0 * B * (ld.out + 2.0 * ld.in));
        }
        if (ld.gap()) {  // W^T delta into the pooled delta, then spread over the pixels (/HW, ReLU mask)
            fb200::BwdArgs a{};
            a.W = slot + ld.woff;
            a.d_out = stash_u + ld.dlt_off;
            a.d_in = stash_u + ld.pdl_off;
            a.in = ld.cols;
            a.out = ld.rows;
            a.B = B;
            a.row_splits = fb200::bwd_row_splits(ld.cols, ld.rows);
            a.partial = d_partial + static_cast<size_t>(scratch) * max_partial;
            a.counters = d_counters + static_cast<size_t>(scratch) * max_tiles;
            fb200::KernelSpec k;
            fb200::spec_bwd(a, k);
            gb->cur_bytes = 4.0 * ld.nw() + 4.0 * B * (ld.rows + ld.cols);
            gb->kernel(k, reads, writes);
            fb200::PoolMeanArgs g{nullptr, nullptr, nullptr, stash_u + below.dlt_off, stash_u + ld.pdl_off, mask,
                                  B, ld.ci, ld.hi * ld.wi};
            fb200::KernelSpec ku;
            fb200::spec_ungap(g, ku);
            gb->cur_bytes = 4.0 * B * (ld.ci + 2.0 * ld.in);
            gb->kernel(ku, reads, writes);
            return;
        }
        if (use_mma(ld))
            return emit_mma(ld, slot, true, stash_u + ld.dlt_off,  nullptr,
                            mask_on_write && below.act == FERRET_ACT_RELU ? stash_u + below.act_off : nullptr,
                            stash_u + below.dlt_off, reads, writes);
        fb200::BwdArgs a{};
        a.W = slot + ld.woff;
        a.d_out = stash_u + ld.dlt_off;
        a.mask = mask_on_write && below.act == FERRET_ACT_RELU ? stash_u + below.act_off : nullptr;
        a.d_in = stash_u + below.dlt_off;
        a.in = ld.in;
        a.out = ld.out;
        a.B = B;
        a.row_splits = fb200::bwd_row_splits(ld.in, ld.out);
        a.partial = d_partial + static_cast<size_t>(scratch) * max_partial;
        a.counters = d_counters + static_cast<size_t>(scratch) * max_tiles;
        fb200::KernelSpec k;
        fb200::spec_bwd(a, k);
        gb->cur_bytes = 4.0 * ld.in * ld.out + 4.0 * B * (ld.out + 2.0 * ld.in);  // W, delta_out, mask, delta_in
        gb->kernel(k, reads, writes);
    }

    // ------------------------------------------------ exact resume
    // "ferret-state v2": everything a pipeline trainer carries from one chunk to
    // the next — the live parameters of every stage (ring slot 0 between chunks),
    // the compensator state, the RunningNormalizer, the version counters and the
    // replay reservoir (host RNG state, positions' labels, pool rows). A text
    // header (shape and options, checked on load) followed by raw little-endian
    // arrays in the device slot layout. Loading it into a trainer built with the
    // same net, bounds and options continues training bit for bit.
    // the options a saved state depends on; the compensator constants and lr are written as
    // exact hex floats (lambda is stored as an offset from lambda0, so a state is only valid
    // for the lambda0 it was saved with)
    std::string options_line() const {
        std::ostringstream o;
        o << "options policy " << opt.policy << " replay " << opt.replay << " capacity " << opt.replay_capacity
          << " precision " << opt.precision << " micro_batch " << B << std::hexfloat << " lr " << opt.lr
          << " lambda0 " << opt.lambda0 << " eta_lambda " << opt.eta_lambda << " alpha " << opt.alpha << " nu "
          << opt.nu;
        return o.str();
    }

    std::string save_state() {
        if (sq.on) fail(FERRET_E_CONFIG, "save_state: sequential learners carry no pipeline state");
        cuda_check(cudaStreamSynchronize(stream), "sync");
        std::string bin;
        auto put_dev = [&](const void* dev, size_t bytes) {
            const size_t at = bin.size();
            bin.resize(at + bytes);
            if (bytes) cuda_check(cudaMemcpy(&bin[at], dev, bytes, cudaMemcpyDeviceToHost), "D2H state");
        };
        for (const StageDev& st : stages) {
            const size_t sb = static_cast<size_t>(st.slot_floats) * sizeof(float);
            put_dev(st.slot(0), sb);
            for (const float* a : {st.lam_d, st.v_r, st.v_a, st.gap})
                if (a) put_dev(a, sb);
        }
        put_dev(d_norm_mean, static_cast<size_t>(F) * sizeof(double));
        put_dev(d_norm_m2, static_cast<size_t>(F) * sizeof(double));
        if (opt.replay && hs.replay.size) {
            put_dev(d_pool_x, static_cast<size_t>(hs.replay.size) * static_cast<size_t>(F) * sizeof(float));
            put_dev(d_pool_lab, static_cast<size_t>(hs.replay.size) * sizeof(int));
        }
        std::ostringstream h;
        h << "ferret-state v2\n" << "layers";
        for (const LayerDev& ld : layers) h << ' ' << ld.in << 'x' << ld.out << ':' << ld.act;
        for (size_t i = 0; i < geom.size(); ++i) h << (i ? "," : "\ngeometry ") << geom[i];
        h << "\nbounds";
        for (const StageDev& st : stages) h << ' ' << st.lo;
        h << ' ' << L << "\n" << options_line() << "\n"
          << "norm_count " << hs.norm_count << "\nversions";
        for (long long v : hs.current) h << ' ' << v;
        h << "\nreservoir " << hs.replay.seen << ' ' << hs.replay.size << "\nrng " << hs.replay.rng.state()
          << "\nlabels";
        for (uint64_t i = 0; i < hs.replay.size; ++i) h << ' ' << hs.replay.label_at[static_cast<size_t>(i)];
        h << "\nids";
        for (uint64_t i = 0; i < hs.replay.size; ++i)
            h << ' ' << (i < hs.replay.id_at.size() ? hs.replay.id_at[static_cast<size_t>(i)] : -1);
        h << "\nbinary " << bin.size() << "\n";
        return h.str() + bin;
    }

    void load_state(const char* data, size_t len) {
        if (sq.on) fail(FERRET_E_CONFIG, "load_state: sequential learners carry no pipeline state");
        const std::string all(data, len);
        std::istringstream in(all);
        std::string line;
        auto expect = [&](const std::string& want) {
            if (!std::getline(in, line) || line != want) fail(FERRET_E_SCHEMA, "state: expected '" + want + "'");
        };
        expect("ferret-state v2");
        {
            std::ostringstream l, b, o;
            l << "layers";
            for (const LayerDev& ld : layers) l << ' ' << ld.in << 'x' << ld.out << ':' << ld.act;
            for (size_t i = 0; i < geom.size(); ++i) l << (i ? "," : "\ngeometry ") << geom[i];
            b << "bounds";
            for (const StageDev& st : stages) b << ' ' << st.lo;
            b << ' ' << L;
            o << options_line();
            std::istringstream ls(l.str());  // "layers" and, for conv nets, "geometry"
            for (std::string want; std::getline(ls, want);) expect(want);
            expect(b.str());
            expect(o.str());
        }
        auto record = [&](const char* key) {
            if (!std::getline(in, line)) fail(FERRET_E_SCHEMA, std::string("state: truncated before '") + key + "'");
            std::istringstream f(line);
            std::string got;
            f >> got;
            if (got != key) fail(FERRET_E_SCHEMA, std::string("state: expected '") + key + "'");
            return f;
        };
        uint64_t norm_count = 0, seen = 0, size = 0;
        if (!(record("norm_count") >> norm_count)) fail(FERRET_E_SCHEMA, "state: bad norm_count");
        std::vector<long long> versions(static_cast<size_t>(P));
        {
            auto f = record("versions");
            for (long long& v : versions)
                if (!(f >> v)) fail(FERRET_E_SCHEMA, "state: bad versions");
        }
        {
            auto f = record("reservoir");
            if (!(f >> seen >> size) || size > opt.replay_capacity || size > seen)
                fail(FERRET_E_SCHEMA, "state: bad reservoir");
        }
        std::string rng_state;
        {
            if (!std::getline(in, line) || line.compare(0, 4, "rng ") != 0) fail(FERRET_E_SCHEMA, "state: bad rng");
            rng_state = line.substr(4);
        }
        std::vector<int> labels(static_cast<size_t>(size));
        {
            auto f = record("labels");
            for (int& x : labels)
                if (!(f >> x)) fail(FERRET_E_SCHEMA, "state: bad labels");
        }
        std::vector<int64_t> ids(static_cast<size_t>(size));
        {
            auto f = record("ids");
            for (int64_t& x : ids)
                if (!(f >> x)) fail(FERRET_E_SCHEMA, "state: bad ids");
        }
        size_t nbin = 0;
        if (!(record("binary") >> nbin)) fail(FERRET_E_SCHEMA, "state: bad binary size");
        const size_t off = static_cast<size_t>(in.tellg());
        if (off + nbin != len) fail(FERRET_E_SCHEMA, "state: binary section size mismatch");
        {  // the expected binary layout, checked before any device slot is overwritten
            size_t want = 0;
            for (const StageDev& st : stages) {
                size_t arrays = 1;
                for (const float* a : {st.lam_d, st.v_r, st.v_a, st.gap})
                    if (a) ++arrays;
                want += arrays * static_cast<size_t>(st.slot_floats) * sizeof(float);
            }
            want += 2 * static_cast<size_t>(F) * sizeof(double);
            if (opt.replay && size) want += static_cast<size_t>(size) * (static_cast<size_t>(F) * sizeof(float) + sizeof(int));
            if (nbin != want) fail(FERRET_E_SCHEMA, "state: binary section does not match this trainer's layout");
        }
        const char* p = data + off;
        size_t left = nbin;
        auto take_dev = [&](void* dev, size_t bytes) {
            if (bytes > left) fail(FERRET_E_SCHEMA, "state: binary section too short");
            if (bytes) cuda_check(cudaMemcpy(dev, p, bytes, cudaMemcpyHostToDevice), "H2D state");
            p += bytes;
            left -= bytes;
        };
        invalidate_graph();
        cuda_check(cudaStreamSynchronize(stream), "sync");
        for (StageDev& st : stages) {
            const size_t sb = static_cast<size_t>(st.slot_floats) * sizeof(float);
            if (sb > left) fail(FERRET_E_SCHEMA, "state: binary section too short");
            if (st.ring16) {  // the bf16 copy of the live slot
                std::vector<float> h(static_cast<size_t>(st.slot_floats));
                std::memcpy(h.data(), p, sb);
                std::vector<uint16_t> h16(h.size());
                for (size_t i = 0; i < h.size(); ++i) h16[i] = bf16_bits(h[i]);
                cuda_check(cudaMemcpy(st.ring16, h16.data(), h16.size() * sizeof(uint16_t), cudaMemcpyHostToDevice),
                           "H2D state");
            }
            take_dev(st.slot(0), sb);
            for (float* a : {st.lam_d, st.v_r, st.v_a, st.gap})
                if (a) take_dev(a, sb);
        }
        take_dev(d_norm_mean, static_cast<size_t>(F) * sizeof(double));
        take_dev(d_norm_m2, static_cast<size_t>(F) * sizeof(double));
        if (opt.replay && size) {
            take_dev(d_pool_x, static_cast<size_t>(size) * static_cast<size_t>(F) * sizeof(float));
            take_dev(d_pool_lab, static_cast<size_t>(size) * sizeof(int));
        }
        if (left) fail(FERRET_E_SCHEMA, "state: trailing bytes in the binary section");
        hs.norm_count = norm_count;
        hs.current = versions;
        hs.replay.seen = seen;
        hs.replay.size = size;
        hs.replay.rng.restore(rng_state);
        hs.replay.label_at = labels;
        hs.replay.id_at = ids;
        hs.replay.draws.clear();
    }

    // ------------------------------------------------ sequential learners
    // StaleHarness (learner.hpp:132-170) and train_sequential (learner.hpp:197-225)
    // on the device. The trainer holds every layer in one stage; each item's
    // kernels are issued in item order on the trainer's stream through the
    // graph builder's eager mode, and one call's items are captured into a
    // single CUDA graph (every item depends on the previous update).
    struct Seq {
        bool on = false;
        long long version = 0;     // absolute version of the live parameters (ring slot version % depth)
        long long ring_size = 1;   // versions the reference's VersionRing holds (compensate.hpp:140-170)
        long long ring_cap = 1;
        uint64_t norm_count = 0;
        unsigned long long* d_zero = nullptr;
        float* d_ux = nullptr;     // the unit's input rows: the item (row 0), the replay sample (row 1)
        double* d_raw = nullptr;   // raw features of the call
        int* d_lab = nullptr;      // per item: label, replay-sample label
        int* d_pred = nullptr;
        float* d_px = nullptr;     // held-out rows (16 x F), standardised
        float* d_pp = nullptr;     // their layer ping-pong (2 x 16 x max width)
        size_t cap = 0;
        std::unique_ptr<GraphBuilder> gb;  // eager builder on the trainer's stream
    } sq;

    void seq_init(long long ring_depth) {
        if (ring_depth + 1 > fb200::kMaxChain)
            fail(FERRET_E_CONFIG, "ring depth above 47 versions is not supported by the update kernel");
        sq.on = true;
        sq.ring_cap = std::max<long long>(ring_depth, 1);
        grow_ring(stages[0], static_cast<int>(sq.ring_cap + 1));  // + the slot written while the chain is read
        ensure_stash(1);
        ensure_scratch(2);
        sq.d_zero = dalloc<unsigned long long>(1, device_bytes);
        cuda_check(cudaMemset(sq.d_zero, 0, sizeof(unsigned long long)), "memset");
        sq.d_ux = dalloc<float>(2 * static_cast<size_t>(F), device_bytes);
        cuda_check(cudaMemset(sq.d_ux, 0, 2 * static_cast<size_t>(F) * sizeof(float)), "memset");
        sq.gb = std::make_unique<GraphBuilder>(stream);
        if (opt.precision != FERRET_PREC_FP32)  // split-K scratch exists before any capture
            for (uint64_t k : {GraphBuilder::key(GraphBuilder::kPred, 0), GraphBuilder::key(GraphBuilder::kStash, 0)})
                mma_scratch_for(k);
    }

    void seq_upload(const double* features, const uint64_t* labels, size_t n) {
        if (n > sq.cap) {
            cuda_check(cudaStreamSynchronize(stream), "sync");
            dfree(sq.d_raw);
            dfree(sq.d_lab);
            dfree(sq.d_pred);
            sq.cap = std::max(n, 2 * sq.cap);
            sq.d_raw = dalloc<double>(sq.cap * static_cast<size_t>(F), device_bytes);
            sq.d_lab = dalloc<int>(2 * sq.cap, device_bytes);
            sq.d_pred = dalloc<int>(sq.cap, device_bytes);
        }
        cuda_check(cudaMemcpyAsync(sq.d_raw, features, n * static_cast<size_t>(F) * sizeof(double),
                                   cudaMemcpyHostToDevice, stream),
                   "H2D features");
        std::vector<int> lab(2 * n, 0);
        for (size_t i = 0; i < n; ++i) {
            if (labels[i] >= static_cast<uint64_t>(n_out)) fail(FERRET_E_INVALID_ARG, "label out of range");
            lab[2 * i] = static_cast<int>(labels[i]);
        }
        seq_labels = std::move(lab);
    }
    std::vector<int> seq_labels;  // host copy, replay labels filled in while the items are emitted

    // One item: RunningNormalizer observe + apply, predict_class at the live
    // version, forward_backward of the `rows`-row batch at version `read`, then
    // Compensator::apply over the chain [read .. live] and the SGD step into a
    // new version (learner.hpp:145-160; with policy none and read = live this is
    // forward_backward + apply_sgd of train_sequential, learner.hpp:207-220).
    void seq_item(size_t i, long long read, int rows, int policy) {
        using GB = GraphBuilder;
        fb200::NormArgs na{sq.d_raw + i * static_cast<size_t>(F), 1, F, sq.d_zero,
                           static_cast<unsigned long long>(sq.norm_count), d_norm_mean, d_norm_m2, sq.d_ux, 0,
                           nullptr, nullptr};
        fb200::KernelSpec kn;
        fb200::spec_normalize(na, kn);
        gb->kernel(kn, {}, {});
        ++sq.norm_count;
        const StageDev& s = stages[0];
        float* su = d_stash;
        const int keep_b = B;
        B = 1;
        for (int l = 0; l < L; ++l) {  // predict_class (net.hpp:150-154)
            const float* X = l == 0 ? sq.d_ux : su + pred_off + ((l - 1) & 1) * pred_stride;
            emit_layer(layers[static_cast<size_t>(l)], s.slot(sq.version), X, nullptr, su + pred_off + (l & 1) * pred_stride,
                       {}, {GB::key(GB::kPred, 0)});
        }
        fb200::HeadArgs h{};
        h.logits = su + pred_off + ((L - 1) & 1) * pred_stride;
        h.n_out = n_out;
        h.B = 1;
        h.mode = 0;
        h.pred = sq.d_pred + i;
        fb200::KernelSpec kh;
        fb200::spec_head(h, kh);
        gb->kernel(kh, {}, {});
        B = rows;
        for (int l = 0; l < L; ++l) {  // forward_backward (net.hpp:157-200) at the read version
            const LayerDev& ld = layers[static_cast<size_t>(l)];
            const float* X = l == 0 ? sq.d_ux : su + layers[static_cast<size_t>(l - 1)].act_off;
            emit_layer(ld, s.slot(read), X, nullptr, su + ld.act_off, {}, {GB::key(GB::kStash, 0)});
        }
        emit_delta_head(su, sq.d_lab + 2 * i, nullptr, 1.0f / static_cast<float>(rows), {}, {GB::key(GB::kStash, 0)});
        for (int l = L - 1; l >= 1; --l) emit_layer_backward(l, s.slot(read), su, 0, {}, {GB::key(GB::kStash, 0)}, true);
        fb200::UpdArgs a = update_args(0, sq.version, read);
        a.policy = policy;
        a.K = 1;
        a.pend[0] = {su, sq.d_ux, 0};
        a.step = static_cast<float>(opt.lr);
        fb200::KernelSpec ku;
        fb200::spec_update(a, ku);
        gb->kernel(ku, {}, {});
        B = keep_b;
        ++sq.version;
        sq.ring_size = std::min(sq.ring_size + 1, sq.ring_cap);
    }

    // Runs `emit(i)` for every item in captured graphs on the trainer's stream, at most
    // kSeqBlock items per graph (each item is ~8-12 nodes; long streams stay bounded).
    static constexpr size_t kSeqBlock = 1024;
    template <class Emit>
    void seq_run(size_t n, Emit&& emit) {
        for (size_t i0 = 0; i0 < n; i0 += kSeqBlock)
            seq_run_block(i0, std::min(n, i0 + kSeqBlock), emit);
    }
    template <class Emit>
    void seq_run_block(size_t i0, size_t i1, Emit& emit) {
        gb = sq.gb.get();
        cudaGraph_t g = nullptr;
        cuda_check(cudaStreamBeginCapture(stream, cudaStreamCaptureModeRelaxed), "cudaStreamBeginCapture");
        try {
            for (size_t i = i0; i < i1; ++i) emit(i);
        } catch (...) {
            cudaStreamEndCapture(stream, &g);
            if (g) cudaGraphDestroy(g);
            gb = nullptr;
            throw;
        }
        cuda_check(cudaStreamEndCapture(stream, &g), "cudaStreamEndCapture");
        gb = nullptr;
        cudaGraphExec_t ge = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        cuda_check(e, "cudaGraphInstantiate");
        const cudaError_t l = cudaGraphLaunch(ge, stream);
        const cudaError_t y = cudaStreamSynchronize(stream);
        cudaGraphExecDestroy(ge);
        cuda_check(l, "cudaGraphLaunch");
        cuda_check(y, "sequential run");
    }

    // predict_class at the live version for held-out items, standardised with the
    // current normalizer state and observing nothing (test_accuracy, learner.hpp:185-192):
    // groups of up to 16 rows through the layer kernels.
    void seq_predict(const double* features, size_t n, uint64_t* preds) {
        if (n == 0) return;
        using GB = GraphBuilder;
        constexpr int G = fb200::kMaxBatch;
        int max_width = F;
        for (const LayerDev& ld : layers) max_width = std::max(max_width, ld.out);
        if (!sq.d_px) {
            sq.d_px = dalloc<float>(static_cast<size_t>(G) * static_cast<size_t>(F), device_bytes);
            sq.d_pp = dalloc<float>(2 * static_cast<size_t>(G) * static_cast<size_t>(max_width), device_bytes);
            if (opt.precision != FERRET_PREC_FP32) mma_scratch_for(GB::key(GB::kReplay, 1));
        }
        std::vector<uint64_t> none(n, 0);
        seq_upload(features, none.data(), n);
        const size_t pstride = static_cast<size_t>(G) * static_cast<size_t>(max_width);
        const StageDev& s = stages[0];
        const int keep_b = B;
        seq_run((n + G - 1) / G, [&](size_t g) {
            const size_t i0 = g * G;
            const int rows = static_cast<int>(std::min<size_t>(G, n - i0));
            fb200::NormArgs na{sq.d_raw + i0 * static_cast<size_t>(F), rows, F, sq.d_zero,
                               static_cast<unsigned long long>(sq.norm_count), d_norm_mean, d_norm_m2, sq.d_px, 1,
                               nullptr, nullptr};
            fb200::KernelSpec kn;
            fb200::spec_normalize(na, kn);
            gb->kernel(kn, {}, {});
            B = rows;
            for (int l = 0; l < L; ++l) {
                const float* X = l == 0 ? sq.d_px : sq.d_pp + static_cast<size_t>((l - 1) & 1) * pstride;
                emit_layer(layers[static_cast<size_t>(l)], s.slot(sq.version), X, nullptr,
                           sq.d_pp + static_cast<size_t>(l & 1) * pstride, {}, {GB::key(GB::kReplay, 1)});
            }
            fb200::HeadArgs h{};
            h.logits = sq.d_pp + static_cast<size_t>((L - 1) & 1) * pstride;
            h.n_out = n_out;
            h.B = rows;
            h.mode = 0;
            h.pred = sq.d_pred + i0;
            fb200::KernelSpec kh;
            fb200::spec_head(h, kh);
            gb->kernel(kh, {}, {});
            B = keep_b;
        });
        std::vector<int> p(n);
        cuda_check(cudaMemcpy(p.data(), sq.d_pred, n * sizeof(int), cudaMemcpyDeviceToHost), "D2H predictions");
        for (size_t i = 0; i < n; ++i) preds[i] = static_cast<uint64_t>(p[i]);
    }

    void set_normalizer(uint64_t count, const double* mean, const double* m2) {
        cuda_check(cudaStreamSynchronize(stream), "sync");
        cuda_check(cudaMemcpy(d_norm_mean, mean, static_cast<size_t>(F) * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(d_norm_m2, m2, static_cast<size_t>(F) * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        sq.norm_count = count;
    }

    // StaleHarness::ocl_step over n items (learner.hpp:145-163)
    void harness_steps(const double* features, const uint64_t* labels, const int32_t* taus, size_t n,
                       uint64_t* preds) {
        if (n == 0) return;
        seq_upload(features, labels, n);
        cuda_check(cudaMemcpyAsync(sq.d_lab, seq_labels.data(), 2 * n * sizeof(int), cudaMemcpyHostToDevice, stream),
                   "H2D labels");
        seq_run(n, [&](size_t i) {
            const long long eff = std::min<long long>(std::max(taus[i], 0), sq.ring_size - 1);
            seq_item(i, sq.version - eff, 1, opt.policy);
        });
        std::vector<int> p(n);
        cuda_check(cudaMemcpy(p.data(), sq.d_pred, n * sizeof(int), cudaMemcpyDeviceToHost), "D2H predictions");
        for (size_t i = 0; i < n; ++i) preds[i] = static_cast<uint64_t>(p[i]);
    }

    // train_sequential over the kept items (learner.hpp:207-222): predict,
    // forward_backward on {item} (+ one replay sample drawn before the item is
    // added, mean over the batch), apply_sgd, then ReplayBuffer::add.
    void sequential_train(const double* features, const uint64_t* labels, size_t n, const int64_t* kept,
                          size_t n_kept, ferret_step_record* log) {
        for (size_t i = 0; i < n; ++i) log[i] = {static_cast<int64_t>(i), FERRET_STEP_DROPPED, 0, 0, labels[i]};
        if (n_kept == 0) return;
        std::vector<double> kf(n_kept * static_cast<size_t>(F));
        std::vector<uint64_t> kl(n_kept);
        for (size_t k = 0; k < n_kept; ++k) {
            if (kept[k] < 0 || static_cast<size_t>(kept[k]) >= n) fail(FERRET_E_INVALID_ARG, "kept index out of range");
            std::memcpy(kf.data() + k * static_cast<size_t>(F), features + static_cast<size_t>(kept[k]) * static_cast<size_t>(F),
                        static_cast<size_t>(F) * sizeof(double));
            kl[k] = labels[kept[k]];
        }
        seq_upload(kf.data(), kl.data(), n_kept);
        std::vector<int> rows(n_kept, 1);
        std::vector<int> src(n_kept, -1), dst(n_kept, -1);  // replay sample drawn / pool position written
        for (size_t k = 0; k < n_kept; ++k) {  // the reservoir's host arithmetic, in item order
            if (opt.replay && hs.replay.size > 0) {
                src[k] = hs.replay.sample();
                seq_labels[2 * k + 1] = hs.replay.label_at[static_cast<size_t>(src[k])];
                rows[k] = 2;
            }
            if (opt.replay) dst[k] = hs.replay.add(seq_labels[2 * k], kept[k]);
        }
        cuda_check(cudaMemcpyAsync(sq.d_lab, seq_labels.data(), 2 * n_kept * sizeof(int), cudaMemcpyHostToDevice, stream),
                   "H2D labels");
        const size_t row_bytes = static_cast<size_t>(F) * sizeof(float);
        seq_run(n_kept, [&](size_t k) {
            if (src[k] >= 0)
                cuda_check(cudaMemcpyAsync(sq.d_ux + F, d_pool_x + static_cast<size_t>(src[k]) * static_cast<size_t>(F),
                                           row_bytes, cudaMemcpyDeviceToDevice, stream),
                           "replay row");
            seq_item(k, sq.version, rows[k], FERRET_POLICY_NONE);
            if (dst[k] >= 0)
                cuda_check(cudaMemcpyAsync(d_pool_x + static_cast<size_t>(dst[k]) * static_cast<size_t>(F), sq.d_ux,
                                           row_bytes, cudaMemcpyDeviceToDevice, stream),
                           "replay add");
        });
        std::vector<int> p(n_kept);
        cuda_check(cudaMemcpy(p.data(), sq.d_pred, n_kept * sizeof(int), cudaMemcpyDeviceToHost), "D2H predictions");
        for (size_t k = 0; k < n_kept; ++k) {
            ferret_step_record& r = log[kept[k]];
            r.predicted = static_cast<uint64_t>(p[k]);
            r.outcome = r.predicted == r.label ? FERRET_STEP_CORRECT : FERRET_STEP_WRONG;
        }
    }

    // replay_step (learner.hpp:513-519): forward_backward(net_, {buffer.sample()})
    // with mean reduction (net.hpp:157-200), apply_sgd on every stage, push a
    // version per stage. B pool samples per replay step at micro-batch B; the
    // pool positions and their labels come from the control block (row r).
    // Across ranks: activations hand forward, deltas (unmasked) hand back.
    template <bool DRY, class NotePush, class VSlot, class Xfer>
    void replay_step(size_t r, std::vector<long long>& rel, NotePush& note_push, VSlot& vslot, Xfer& xfer) {
        using GB = GraphBuilder;
        for (int j = 0; j < P; ++j) note_push(j);
        // replay stash resources per layer: its activation (act), the delta at its output (dlt)
        // and its materialised conv weight gradient (grd), so a layer's weight gradient runs
        // beside its input gradient and a stage's SGD step starts once its own layers are done
        // (one key for the whole replay stash chained every replay node after the previous)
        auto ract = [](int l) { return GB::key(GB::kReplay, 1, static_cast<uint64_t>(l)); };
        auto rdlt = [](int l) { return GB::key(GB::kReplay, 2, static_cast<uint64_t>(l)); };
        auto rgrd = [](int l) { return GB::key(GB::kReplay, 3, static_cast<uint64_t>(l)); };
        const uint64_t pk = GB::key(GB::kPool, 0);
        const int* ids = ctl_rep_ids() + r * static_cast<size_t>(B);
        auto owner_of = [&](int j) { return owner[static_cast<size_t>(j)]; };
        for (int j = 0; j < P; ++j) {  // forward sweep
            const StageDev& s = stages[static_cast<size_t>(j)];
            if (j > 0) {
                const LayerDev& in_l = layers[static_cast<size_t>(s.lo - 1)];
                float* buf = d_replay + in_l.act_off;
                xfer(owner_of(j - 1), owner_of(j), [&] { return buf; }, [&] { return buf; },
                     static_cast<size_t>(B) * in_l.out, nullptr, ract(s.lo - 1));
            }
            if (DRY || !mine(j)) continue;
            gb->cur_category = kCatReplay;
            gb->cur_stage = -1;
            for (int l = s.lo; l < s.hi; ++l) {
                const LayerDev& ld = layers[static_cast<size_t>(l)];
                const float* X = l == 0 ? d_pool_x : d_replay + layers[static_cast<size_t>(l - 1)].act_off;
                std::vector<uint64_t> rd{vslot(j, rel[static_cast<size_t>(j)]), l == 0 ? pk : ract(l - 1)};
                if (ld.res) rd.push_back(ract(l - 2));
                emit_layer(ld, s.slot(rel[static_cast<size_t>(j)]), X, l == 0 ? ids : nullptr, d_replay + ld.act_off, rd,
                           {ract(l)}, Head{}, ld.res ? d_replay + layers[static_cast<size_t>(l - 2)].act_off : nullptr,
                           ld.gap() ? d_replay + ld.pool_off : nullptr);
            }
        }
        if (!DRY && mine(P - 1)) {
            gb->cur_category = kCatReplay;
            emit_delta_head(d_replay, ctl_rep_labels() + r * static_cast<size_t>(B), nullptr,
                            1.0f / static_cast<float>(B), {ract(L - 1)}, {rdlt(L - 1)});
        }
        for (int j = P - 1; j >= 0; --j) {  // backward sweep
            const StageDev& s = stages[static_cast<size_t>(j)];
            const bool cross = j > 0 && owner_of(j - 1) != owner_of(j);
            if (!DRY && mine(j)) {
                gb->cur_category = kCatReplay;
                for (int l = s.hi - 1; l >= s.lo; --l) {
                    const LayerDev& ld = layers[static_cast<size_t>(l)];
                    if (ld.conv())
                        emit_conv_wgrad(ld, d_replay, l == 0 ? d_pool_x : d_replay + layers[static_cast<size_t>(l - 1)].act_off,
                                        l == 0 ? ids : nullptr,
                                        {vslot(j, rel[static_cast<size_t>(j)]), l == 0 ? pk : ract(l - 1), rdlt(l)},
                                        {rgrd(l)});
                    if (l == 0) break;
                    std::vector<uint64_t> rd{vslot(j, rel[static_cast<size_t>(j)]), rdlt(l), ract(l - 1)};
                    if (l + 1 < L && layers[static_cast<size_t>(l + 1)].res) rd.push_back(rdlt(l + 1));
                    emit_layer_backward(l, s.slot(rel[static_cast<size_t>(j)]), d_replay, stash_slots, rd, {rdlt(l - 1)},
                                        !(cross && l == s.lo));
                }
            }
            if (cross) {
                const LayerDev& below = layers[static_cast<size_t>(s.lo - 1)];
                float* buf = d_replay + below.dlt_off;
                xfer(owner_of(j), owner_of(j - 1), [&] { return buf; }, [&] { return buf; },
                     static_cast<size_t>(B) * below.out, below.act == FERRET_ACT_RELU ? d_replay + below.act_off : nullptr,
                     rdlt(s.lo - 1));
            }
        }
        if (!DRY) {
            for (int j = 0; j < P; ++j) {
                if (!mine(j)) continue;
                gb->cur_category = kCatReplay;
                const StageDev& s = stages[static_cast<size_t>(j)];
                const long long cur = rel[static_cast<size_t>(j)];
                fb200::UpdArgs a = update_args(j, cur, cur);
                a.policy = FERRET_POLICY_NONE;
                a.K = 1;
                a.pend[0] = {d_replay, d_pool_x, 0};
                a.x0idx = ids;
                a.step = static_cast<float>(opt.lr);
                fb200::KernelSpec k;
                fb200::spec_update(a, k);
                std::vector<uint64_t> rd{pk, vslot(j, cur)};
                for (int l = s.lo; l < s.hi; ++l) {
                    rd.push_back(rdlt(l));
                    if (l > 0) rd.push_back(ract(l - 1));
                    if (layers[static_cast<size_t>(l)].conv()) rd.push_back(rgrd(l));
                    if (layers[static_cast<size_t>(l)].gap()) rd.push_back(ract(l));  // the pooled input
                }
                gb->cur_bytes = update_bytes(j, FERRET_POLICY_NONE, {cur}, cur);
                gb->kernel(k, rd, {vslot(j, cur + 1)});
                wt_invalidate(stages[static_cast<size_t>(j)], a.dst);
            }
        }
        for (int j = 0; j < P; ++j) rel[static_cast<size_t>(j)] += 1;
    }

    // --------------------------------------------------------------- timing
    // timing mode builds a serial graph, so an event node before and after an
    // update node brackets that kernel alone
    void time_begin() {
        if (!timing) return;
        gb->event(ev_pool[ev_used]);
    }
    void time_end(double alg_bytes) {
        if (!timing) return;
        gb->event(ev_pool[ev_used + 1]);
        ev_used += 2;
        upd_alg_bytes += alg_bytes;
        upd_timed += 1;
    }
    // Algorithmic bytes of one update launch: every parameter element reads the
    // versions it needs + its compensator state and writes the new version +
    // state; plus the deltas and layer inputs of each pending gradient.
    // Update groups (same results): consecutive iter_fisher updates of a large dense stage fused
    // into one update_group_kernel launch that reads the version chain and the compensator state
    // once; one-member groups go to the single-update kernels. C5 fp32: 3.87k -> 4.85k samples/s
    // (profiles/r2/ab_update_groups_final.txt). FERRET_UPDATE_GROUPS=0: every update its own node
    bool group_updates = !std::getenv("FERRET_UPDATE_GROUPS") || std::atoi(std::getenv("FERRET_UPDATE_GROUPS")) != 0;
    long long group_min_params = std::getenv("FERRET_UPDATE_GROUPS_MIN") ? std::atoll(std::getenv("FERRET_UPDATE_GROUPS_MIN"))
                                                                          : 8ll << 20;
    // Consecutive updates of a stage joined by programmatic edges (KernelSpec::chain_pdl kernels:
    // the next update launches and loads its unit's inputs and older versions while the previous
    // one drains): C2 1.10M -> 1.23M samples/s, its critical path being the stage-0 update chain
    // (profiles/r2/update_pdl_ab.txt). FERRET_UPDATE_PDL=0: full dependencies (A/B knob)
    bool update_pdl = !std::getenv("FERRET_UPDATE_PDL") || std::atoi(std::getenv("FERRET_UPDATE_PDL")) != 0;
    size_t n_group_nodes = 0, n_single_groups = 0;  // group launches / one-member groups sent to the single-update kernels
    // algorithmic HBM bytes of one update group of stage j: the n0 chain versions read once,
    // lambda / v_r / v_a read and written once, G new versions written (+ their bf16 copies),
    // plus every member's unit activations and deltas
    double group_bytes(int j, int n0, int G) const {
        const StageDev& s = stages[static_cast<size_t>(j)];
        const double state = s.v_r ? 24.0 : 8.0;
        const double per = 4.0 * n0 + state + (4.0 + (s.ring16 ? 2.0 : 0.0)) * G;
        double side = 0.0;
        for (int l = s.lo; l < s.hi; ++l) {
            const LayerDev& ld = layers[static_cast<size_t>(l)];
            side += ld.conv() ? 4.0 * static_cast<double>(ld.nw() + ld.rows) : 4.0 * B * (ld.cols + ld.rows);
        }
        return per * static_cast<double>(s.n_params) + side * G;
    }

    double update_bytes(int j, int policy, const std::vector<long long>& reads, long long cur) const {
        const StageDev& s = stages[static_cast<size_t>(j)];
        long long lo = cur;
        for (long long r : reads) lo = std::min(lo, r);
        double per = 0.0;
        switch (policy) {
            case FERRET_POLICY_ITER_FISHER:
                per = 4.0 * static_cast<double>(cur - lo + 1) + 4.0 + 4.0 * (s.v_r ? 6.0 : 2.0);
                break;
            case FERRET_POLICY_GAP: per = 4.0 * static_cast<double>(std::min<long long>(cur - lo, 1) + 1) + 4.0 + 8.0; break;
            case FERRET_POLICY_FISHER: {
                std::vector<long long> d(reads.begin(), reads.end());
                d.push_back(cur);
                std::sort(d.begin(), d.end());
                d.erase(std::unique(d.begin(), d.end()), d.end());
                per = 4.0 * static_cast<double>(d.size()) + 4.0;
                break;
            }
            default: per = 8.0;
        }
        double side = 0.0;
        for (int l = s.lo; l < s.hi; ++l) {
            const LayerDev& ld = layers[static_cast<size_t>(l)];
            side += ld.conv() ? 4.0 * static_cast<double>(ld.nw() + ld.rows) : 4.0 * B * (ld.cols + ld.rows);
        }
        return per * static_cast<double>(s.n_params) + side * static_cast<double>(reads.size());
    }

    // ------------------------------------------------------------------ output
    // StepRecords of one chunk from its predictions and labels (items numbered from item0)
    void fill_log(const int* pred, const int* lab, size_t item0, ferret_step_record* out) const {
        for (size_t u = 0; u < sched.n_units; ++u)
            for (int b = 0; b < B; ++b) {
                const size_t i = u * static_cast<size_t>(B) + static_cast<size_t>(b);
                ferret_step_record& r = out[i];
                r = ferret_step_record{static_cast<int64_t>(item0 + i), FERRET_STEP_DROPPED, 0, 0,
                                       static_cast<uint64_t>(lab[i])};
                if (!sched.dropped[u]) {
                    r.predicted = static_cast<uint64_t>(pred[i]);
                    r.outcome = pred[i] == lab[i] ? FERRET_STEP_CORRECT : FERRET_STEP_WRONG;
                }
            }
    }

    // ---------------------------------------------------------------- ingest
    // Stream ingest at rate: n host samples (a whole number of chunks) run chunk
    // after chunk through the compiled schedule. Host->device copies of chunk c+1
    // (on a copy stream, into one of two device staging slots) overlap the graph
    // of chunk c; predictions come back on the copy stream into pinned buffers
    // while later chunks compute. With pinned `features` the copies are true DMA.
    struct Ingest {
        size_t cap = 0;
        double* d_raw[2] = {nullptr, nullptr};
        int* d_lab[2] = {nullptr, nullptr};
        int* d_pred[2] = {nullptr, nullptr};
        int* h_lab[2] = {nullptr, nullptr};   // pinned
        int* h_pred[2] = {nullptr, nullptr};  // pinned
        cudaEvent_t in[2] = {}, freed[2] = {}, out[2] = {};
        cudaStream_t copy = nullptr;  // inbound (H2D)
        cudaStream_t back = nullptr;  // outbound (D2H): a separate queue, so chunk c+1's copy-in never waits
                                      // behind chunk c's copy-out (which waits for chunk c's graph)
    } ing;

    void ensure_ingest(size_t chunk) {
        if (ing.cap >= chunk) return;
        cuda_check(cudaDeviceSynchronize(), "sync");
        release_ingest();
        for (int s = 0; s < 2; ++s) {
            ing.d_raw[s] = dalloc<double>(chunk * static_cast<size_t>(F), device_bytes);
            ing.d_lab[s] = dalloc<int>(chunk, device_bytes);
            ing.d_pred[s] = dalloc<int>(chunk, device_bytes);
            cuda_check(cudaMallocHost(&ing.h_lab[s], chunk * sizeof(int)), "cudaMallocHost");
            cuda_check(cudaMallocHost(&ing.h_pred[s], chunk * sizeof(int)), "cudaMallocHost");
            for (cudaEvent_t* e : {&ing.in[s], &ing.freed[s], &ing.out[s]})
                cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
        }
        if (!ing.copy) cuda_check(cudaStreamCreateWithFlags(&ing.copy, cudaStreamNonBlocking), "stream");
        if (!ing.back) cuda_check(cudaStreamCreateWithFlags(&ing.back, cudaStreamNonBlocking), "stream");
        ing.cap = chunk;
    }

    void release_ingest() {
        for (int s = 0; s < 2; ++s) {
            dfree(ing.d_raw[s]);
            dfree(ing.d_lab[s]);
            dfree(ing.d_pred[s]);
            if (ing.h_lab[s]) cudaFreeHost(ing.h_lab[s]);
            if (ing.h_pred[s]) cudaFreeHost(ing.h_pred[s]);
            for (cudaEvent_t e : {ing.in[s], ing.freed[s], ing.out[s]})
                if (e) cudaEventDestroy(e);
            ing.d_raw[s] = nullptr;
            ing.d_lab[s] = ing.d_pred[s] = ing.h_lab[s] = ing.h_pred[s] = nullptr;
            ing.in[s] = ing.freed[s] = ing.out[s] = nullptr;
        }
        device_bytes -= 2 * ing.cap * (static_cast<size_t>(F) * sizeof(double) + 2 * sizeof(int));
        ing.cap = 0;
    }

    void ingest(const double* features, const uint64_t* lab, size_t n, size_t f, ferret_step_record* log) {
        if (!have_schedule) fail(FERRET_E_LOGIC, "ingest: no schedule set");
        // (stage-sharded trainers reuse their inboxes every chunk: the per-message acks of
        // send_kernel / recv_kernel keep a chunk's sends behind the previous chunk's reads)
        if (static_cast<int>(f) != F) fail(FERRET_E_INVALID_ARG, "stream feature width does not match the net input");
        const size_t chunk = sched.chunk_items;
        if (n % chunk) fail(FERRET_E_INVALID_ARG, "ingest: sample count must be a whole number of chunks");
        std::vector<int> l32(n);
        for (size_t i = 0; i < n; ++i) {
            if (lab[i] >= static_cast<uint64_t>(n_out)) fail(FERRET_E_INVALID_ARG, "forward_backward: label out of range");
            l32[i] = static_cast<int>(lab[i]);
        }
        ensure_ingest(chunk);
        const size_t nch = n / chunk;
        auto drain = [&](size_t c) {
            const int s = static_cast<int>(c & 1);
            cuda_check(cudaEventSynchronize(ing.out[s]), "cudaEventSynchronize");
            fill_log(ing.h_pred[s], l32.data() + c * chunk, c * chunk, log + c * chunk);
        };
        for (size_t c = 0; c < nch; ++c) {
            const int s = static_cast<int>(c & 1);
            if (c >= 2) drain(c - 2);  // slot s: its predictions are home, its pinned labels free
            std::memcpy(ing.h_lab[s], l32.data() + c * chunk, chunk * sizeof(int));
            if (c >= 2) cuda_check(cudaStreamWaitEvent(ing.copy, ing.freed[s], 0), "cudaStreamWaitEvent");
            cuda_check(cudaMemcpyAsync(ing.d_raw[s], features + c * chunk * f, chunk * f * sizeof(double),
                                       cudaMemcpyHostToDevice, ing.copy),
                       "H2D chunk");
            cuda_check(cudaMemcpyAsync(ing.d_lab[s], ing.h_lab[s], chunk * sizeof(int), cudaMemcpyHostToDevice, ing.copy),
                       "H2D labels");
            cuda_check(cudaEventRecord(ing.in[s], ing.copy), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(stream, ing.in[s], 0), "cudaStreamWaitEvent");
            execute_from(l32.data() + c * chunk, ing.d_raw[s], ing.d_lab[s], ing.d_pred[s]);
            cuda_check(cudaEventRecord(ing.freed[s], stream), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(ing.back, ing.freed[s], 0), "cudaStreamWaitEvent");
            cuda_check(cudaMemcpyAsync(ing.h_pred[s], ing.d_pred[s], chunk * sizeof(int), cudaMemcpyDeviceToHost, ing.back),
                       "D2H predictions");
            cuda_check(cudaEventRecord(ing.out[s], ing.back), "cudaEventRecord");
        }
        for (size_t c = nch >= 2 ? nch - 2 : 0; c < nch; ++c) drain(c);
    }

    void fetch_log(size_t chunk, ferret_step_record* out) {
        if (!have_schedule) fail(FERRET_E_LOGIC, "fetch_log: no schedule set");
        const size_t base = chunk * sched.chunk_items;
        const size_t n_samples = sched.n_units * static_cast<size_t>(B);
        if (base + n_samples > n_loaded) fail(FERRET_E_OUT_OF_RANGE, "fetch_log: chunk lies beyond the loaded stream");
        std::vector<int> pred(n_samples);
        cuda_check(cudaMemcpyAsync(pred.data(), d_pred + base, n_samples * sizeof(int), cudaMemcpyDeviceToHost, stream),
                   "D2H predictions");
        cuda_check(cudaStreamSynchronize(stream), "sync");
        for (size_t i = 0; i < sched.chunk_items; ++i) out[i] = ferret_step_record{0, FERRET_STEP_DROPPED, 0, 0, 0};
        for (size_t u = 0; u < sched.n_units; ++u) {
            for (int b = 0; b < B; ++b) {
                const size_t i = u * static_cast<size_t>(B) + static_cast<size_t>(b);
                const int label = labels[base + i];
                ferret_step_record& r = out[i];
                r.item = static_cast<int64_t>(i);
                r.label = static_cast<uint64_t>(label);
                if (sched.dropped[u]) {
                    r.outcome = FERRET_STEP_DROPPED;
                    r.predicted = 0;
                } else {
                    r.predicted = static_cast<uint64_t>(pred[i]);
                    r.outcome = pred[i] == label ? FERRET_STEP_CORRECT : FERRET_STEP_WRONG;
                }
            }
        }
    }

    void read_params(double* out, size_t n) {
        if (n != init_params.size()) fail(FERRET_E_INVALID_ARG, "params: size mismatch");
        cuda_check(cudaStreamSynchronize(stream), "sync");
        for (int j = 0; j < P; ++j) {
            const StageDev& s = stages[static_cast<size_t>(j)];
            std::vector<float> slot(static_cast<size_t>(s.slot_floats));
            cuda_check(cudaMemcpy(slot.data(), s.slot(sq.on ? sq.version : 0), slot.size() * sizeof(float),
                                  cudaMemcpyDeviceToHost),
                       "D2H params");
            unpack_stage(s, slot, out, 0.0);
        }
    }

    // stage slot layout -> flatten() order, adding `offset` to every element
    void unpack_stage(const StageDev& s, const std::vector<float>& slot, double* out, double offset) const {
        for (int l = s.lo; l < s.hi; ++l) {
            const LayerDev& ld = layers[static_cast<size_t>(l)];
            double* dst = out + ld.host_off;
            const long long nw = ld.nw();
            for (long long i = 0; i < nw; ++i) dst[i] = offset + static_cast<double>(slot[static_cast<size_t>(ld.woff + i)]);
            for (int r = 0; r < ld.rows; ++r) dst[nw + r] = offset + static_cast<double>(slot[static_cast<size_t>(ld.boff + r)]);
        }
    }

    void read_state(int j, const float* dev, double* out, size_t n, double offset) {
        const StageDev& s = stages[static_cast<size_t>(j)];
        if (n != static_cast<size_t>(s.n_params)) fail(FERRET_E_INVALID_ARG, "comp_state: size mismatch");
        if (!dev) {
            for (long long i = 0; i < s.n_params; ++i) out[i] = offset;
            return;
        }
        std::vector<double> full(init_params.size());
        std::vector<float> slot(static_cast<size_t>(s.slot_floats));
        cuda_check(cudaMemcpy(slot.data(), dev, slot.size() * sizeof(float), cudaMemcpyDeviceToHost), "D2H state");
        unpack_stage(s, slot, full.data(), offset);
        std::copy(full.begin() + s.host_off, full.begin() + s.host_off + s.n_params, out);
    }
};

namespace {

bool device_ok(int dev) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= dev || dev < 0) return false;
    cudaDeviceProp p{};
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return false;
    return p.major == 10;
}

void require_device(int dev) {
    if (!device_ok(dev))
        fail(FERRET_E_NO_DEVICE, "no sm_100 device at ordinal " + std::to_string(dev) +
                                     " (libferret_b200 has no CPU fallback)");
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
}

} // namespace

extern "C" {

int32_t ferret_device_available(void) { return device_ok(0) ? 1 : 0; }

ferret_status ferret_trainer_create(const ferret_net_desc* net, const uint64_t* bounds, int32_t n_bounds,
                                    const ferret_train_opts* opts, ferret_trainer** out) {
    return guarded([&] {
        if (!net || !bounds || !opts || !out) fail(FERRET_E_INVALID_ARG, "trainer_create: null argument");
        const bool plan_only = opts->device < 0;
        if (!plan_only) require_device(opts->device);
        PlanOnlyScope scope(plan_only);
        auto t = std::make_unique<ferret_trainer>();
        t->opt = *opts;
        t->plan_only = plan_only;
        cuda_check(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&t->nstream, cudaStreamNonBlocking), "stream");
        t->build(*net, bounds, n_bounds);
        cuda_check(cudaDeviceSynchronize(), "create");
        *out = t.release();
    });
}

ferret_status ferret_trainer_save_state(ferret_trainer* t, void* buf, size_t cap, size_t* size) {
    return guarded([&] {
        if (!size) fail(FERRET_E_INVALID_ARG, "save_state: null size");
        t->require_device_mode();
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        const std::string s = t->save_state();
        *size = s.size();
        if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
    });
}

ferret_status ferret_trainer_load_state(ferret_trainer* t, const void* buf, size_t len) {
    return guarded([&] {
        if (!buf) fail(FERRET_E_INVALID_ARG, "load_state: null buffer");
        t->require_device_mode();
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->load_state(static_cast<const char*>(buf), len);
    });
}

ferret_status ferret_seq_create(const ferret_net_desc* net, const ferret_seq_opts* o, ferret_trainer** out) {
    return guarded([&] {
        if (!net || !o || !out) fail(FERRET_E_INVALID_ARG, "seq_create: null argument");
        if (net->n_layers <= 0) fail(FERRET_E_CONFIG, "net needs at least one layer");
        if (net->n_layers > fb200::kMaxStageLayers) fail(FERRET_E_CONFIG, "at most 16 layers per sequential learner");
        if (net->geom) fail(FERRET_E_CONFIG, "sequential learners take dense nets (convolutions: the pipeline trainer)");
        require_device(o->device);
        ferret_train_opts t_o{};
        ferret_train_opts_default(&t_o);
        t_o.policy = o->policy;
        t_o.lr = o->lr;
        t_o.eta_lambda = o->eta_lambda;
        t_o.replay = o->replay;
        t_o.replay_seed = o->replay_seed;
        t_o.replay_capacity = o->replay_capacity;
        t_o.precision = o->precision;
        t_o.micro_batch = o->replay ? 2 : 1;  // train_sequential's batch: the item + one replay sample
        t_o.device = o->device;
        auto t = std::make_unique<ferret_trainer>();
        t->opt = t_o;
        cuda_check(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&t->nstream, cudaStreamNonBlocking), "stream");
        const uint64_t bounds[2] = {0, static_cast<uint64_t>(net->n_layers)};
        t->build(*net, bounds, 2);
        t->seq_init(static_cast<long long>(std::max<uint64_t>(o->ring_depth, 1)));
        cuda_check(cudaDeviceSynchronize(), "create");
        *out = t.release();
    });
}

ferret_status ferret_seq_ocl_steps(ferret_trainer* t, const double* features, const uint64_t* labels,
                                   const int32_t* taus, size_t n_items, size_t n_features, uint64_t* preds_out) {
    return guarded([&] {
        if (!t->sq.on) fail(FERRET_E_CONFIG, "seq_ocl_steps: not a sequential learner (ferret_seq_create)");
        if (n_features != static_cast<size_t>(t->F)) fail(FERRET_E_INVALID_ARG, "feature width mismatch");
        if (n_items && (!features || !labels || !taus || !preds_out)) fail(FERRET_E_INVALID_ARG, "null buffer");
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->harness_steps(features, labels, taus, n_items, preds_out);
    });
}

ferret_status ferret_seq_predict(ferret_trainer* t, const double* features, size_t n_items, size_t n_features,
                                 uint64_t* preds_out) {
    return guarded([&] {
        if (!t->sq.on) fail(FERRET_E_CONFIG, "seq_predict: not a sequential learner (ferret_seq_create)");
        if (n_features != static_cast<size_t>(t->F)) fail(FERRET_E_INVALID_ARG, "feature width mismatch");
        if (n_items && (!features || !preds_out)) fail(FERRET_E_INVALID_ARG, "null buffer");
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->seq_predict(features, n_items, preds_out);
    });
}

ferret_status ferret_seq_set_normalizer(ferret_trainer* t, uint64_t count, const double* mean, const double* m2,
                                        size_t n_features) {
    return guarded([&] {
        if (!t->sq.on) fail(FERRET_E_CONFIG, "seq_set_normalizer: not a sequential learner (ferret_seq_create)");
        if (n_features != static_cast<size_t>(t->F)) fail(FERRET_E_INVALID_ARG, "normalizer: width mismatch");
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->set_normalizer(count, mean, m2);
    });
}

ferret_status ferret_seq_train(ferret_trainer* t, const double* features, const uint64_t* labels, size_t n_items,
                               size_t n_features, const int64_t* kept, size_t n_kept, ferret_step_record* log_out) {
    return guarded([&] {
        if (!t->sq.on) fail(FERRET_E_CONFIG, "seq_train: not a sequential learner (ferret_seq_create)");
        if (n_features != static_cast<size_t>(t->F)) fail(FERRET_E_INVALID_ARG, "feature width mismatch");
        if (n_items && (!features || !labels || !log_out)) fail(FERRET_E_INVALID_ARG, "null buffer");
        if (n_kept && !kept) fail(FERRET_E_INVALID_ARG, "null kept index list");
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->sequential_train(features, labels, n_items, kept, n_kept, log_out);
    });
}

ferret_status ferret_trainer_load_stream(ferret_trainer* t, const double* features, const uint64_t* labels,
                                         size_t n_items, size_t n_features) {
    return guarded([&] {
        t->require_device_mode();
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->load_stream(features, labels, n_items, n_features);
    });
}

ferret_status ferret_trainer_set_schedule(ferret_trainer* t, const ferret_event* events, size_t n_events,
                                          size_t n_chunk_items) {
    return guarded([&] {
        PlanOnlyScope scope(t->plan_only);
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->set_schedule(events, n_events, n_chunk_items);
    });
}

ferret_status ferret_trainer_handoff_plan(ferret_trainer* t, uint64_t* bytes_to_rank, uint64_t* msgs_to_rank,
                                          int32_t world) {
    return guarded([&] {
        if (world != t->world) fail(FERRET_E_INVALID_ARG, "handoff_plan: world mismatch");
        if (!t->have_schedule) fail(FERRET_E_LOGIC, "handoff_plan: set_schedule first");
        PlanOnlyScope scope(true);  // sizing pass only: no device work
        HostState probe = t->hs;
        const PassResult plan = t->run_pass<true>(probe, false);
        for (int32_t r = 0; r < world; ++r) {
            bytes_to_rank[r] = plan.inbox_bytes[static_cast<size_t>(r)];
            msgs_to_rank[r] = plan.inbox_flags[static_cast<size_t>(r)];
        }
    });
}

ferret_status ferret_trainer_execute(ferret_trainer* t, size_t chunk) {
    return guarded([&] {
        t->require_device_mode();
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->execute(chunk);
    });
}

ferret_status ferret_trainer_fetch_log(ferret_trainer* t, size_t chunk, ferret_step_record* log_out) {
    return guarded([&] {
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->fetch_log(chunk, log_out);
    });
}

ferret_status ferret_trainer_sync(ferret_trainer* t) {
    return guarded([&] {
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        t->check_handoffs();
    });
}

void* ferret_trainer_stream(ferret_trainer* t) { return static_cast<void*>(t->stream); }

ferret_status ferret_trainer_run(ferret_trainer* t, const ferret_event* events, size_t n_events, const double* features,
                                 const uint64_t* labels, size_t n_items, size_t n_features,
                                 ferret_step_record* log_out) {
    return guarded([&] {
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->load_stream(features, labels, n_items, n_features);
        t->set_schedule(events, n_events, n_items);
        t->execute(0);
        t->fetch_log(0, log_out);
    });
}

ferret_status ferret_trainer_ingest(ferret_trainer* t, const double* features, const uint64_t* labels, size_t n_items,
                                    size_t n_features, ferret_step_record* log_out) {
    return guarded([&] {
        t->require_device_mode();
        if (n_items && (!features || !labels || !log_out)) fail(FERRET_E_INVALID_ARG, "ingest: null buffer");
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->ingest(features, labels, n_items, n_features, log_out);
    });
}

ferret_status ferret_trainer_params(ferret_trainer* t, double* out, size_t n) {
    return guarded([&] {
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->read_params(out, n);
    });
}

ferret_status ferret_trainer_comp_state(ferret_trainer* t, int32_t stage, double* lambda, double* v_r, double* v_a,
                                        double* mean_gap, size_t n) {
    return guarded([&] {
        if (stage < 0 || stage >= t->P) fail(FERRET_E_OUT_OF_RANGE, "comp_state: stage out of range");
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        const StageDev& s = t->stages[static_cast<size_t>(stage)];
        const double lam0 = t->opt.policy == FERRET_POLICY_ITER_FISHER || t->opt.policy == FERRET_POLICY_FISHER
                                ? t->opt.lambda0
                                : 0.0;
        if (lambda) t->read_state(stage, s.lam_d, lambda, n, lam0);
        if (v_r) t->read_state(stage, s.v_r, v_r, n, 0.0);
        if (v_a) t->read_state(stage, s.v_a, v_a, n, 0.0);
        if (mean_gap) t->read_state(stage, s.gap, mean_gap, n, 0.0);
    });
}

ferret_status ferret_trainer_replay_draws(ferret_trainer* t, int64_t* out, size_t cap, size_t* n) {
    return guarded([&] {
        if (!t) fail(FERRET_E_INVALID_ARG, "replay_draws: null trainer");
        const std::vector<int64_t>& d = t->hs.replay.draws;
        if (out)
            for (size_t i = 0; i < d.size() && i < cap; ++i) out[i] = d[i];
        if (n) *n = d.size();
    });
}

ferret_status ferret_trainer_normalizer(ferret_trainer* t, uint64_t* count, double* mean, double* m2, size_t n_features) {
    return guarded([&] {
        if (n_features != static_cast<size_t>(t->F)) fail(FERRET_E_INVALID_ARG, "normalizer: width mismatch");
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        *count = t->sq.on ? t->sq.norm_count : t->hs.norm_count;
        cuda_check(cudaMemcpy(mean, t->d_norm_mean, n_features * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(m2, t->d_norm_m2, n_features * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    });
}

ferret_status ferret_trainer_get_stats(ferret_trainer* t, ferret_trainer_stats* out) {
    return guarded([&] {
        *out = t->stats;
        out->device_bytes = t->device_bytes;
    });
}

ferret_status ferret_trainer_footprint(ferret_trainer* t, ferret_footprint* out) {
    return guarded([&] {
        if (!out) fail(FERRET_E_INVALID_ARG, "footprint: null output");
        *out = t->footprint();
    });
}

void ferret_trainer_destroy(ferret_trainer* t) { delete t; }

ferret_status ferret_trainer_set_timing(ferret_trainer* t, int32_t enable) {
    return guarded([&] {
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        t->timing = enable != 0;
    });
}

ferret_status ferret_trainer_set_shard(ferret_trainer* t, int32_t rank, int32_t world, const int32_t* stage_owner) {
    return guarded([&] {
        PlanOnlyScope scope(t->plan_only);
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->set_shard(rank, world, stage_owner);
    });
}

ferret_status ferret_trainer_inbox_handle(ferret_trainer* t, void* out, size_t cap) {
    return guarded([&] {
        if (cap < sizeof(cudaIpcMemHandle_t)) fail(FERRET_E_INVALID_ARG, "inbox_handle: buffer smaller than 64 bytes");
        if (!t->d_inbox) fail(FERRET_E_LOGIC, "inbox_handle: no inbox (world 1, or set_schedule not called)");
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        cudaIpcMemHandle_t h;
        cuda_check(cudaIpcGetMemHandle(&h, t->d_inbox), "cudaIpcGetMemHandle");
        std::memcpy(out, &h, sizeof h);
    });
}

ferret_status ferret_trainer_open_peer(ferret_trainer* t, int32_t peer, const void* handle) {
    return guarded([&] {
        cuda_check(cudaSetDevice(t->opt.device), "cudaSetDevice");
        t->open_peer(peer, handle);
    });
}

ferret_status ferret_trainer_set_profiling(ferret_trainer* t, int32_t enable) {
    return guarded([&] {
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        t->profiling = enable != 0;
        if (t->profiling) t->timing = false;
    });
}

ferret_status ferret_trainer_profile(ferret_trainer* t, double* class_ms, uint64_t* class_nodes, double* class_bytes,
                                     int32_t n_classes, double* critical_ms, double* serial_ms) {
    return guarded([&] {
        if (!t->graph_profiling) fail(FERRET_E_LOGIC, "profile: the last execute() did not run a profiling graph");
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        const size_t n = t->prof_cat.size();
        std::vector<double> dur(n, 0.0), finish(n, 0.0);
        for (int c = 0; c < n_classes; ++c) {
            class_ms[c] = 0.0;
            class_nodes[c] = 0;
            class_bytes[c] = 0.0;
        }
        double total = 0.0, crit = 0.0;
        std::vector<int> pred_node(n, -1);
        size_t last = 0;
        for (size_t i = 0; i < n; ++i) {
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, t->prof_events[2 * i], t->prof_events[2 * i + 1]), "cudaEventElapsedTime");
            dur[i] = ms;
            total += ms;
            const int c = t->prof_cat[i];
            if (c < n_classes) {
                class_ms[c] += ms;
                class_nodes[c] += 1;
                class_bytes[c] += t->prof_bytes[i];
            }
            double start = 0.0;
            for (int d : t->prof_ldeps[i])
                if (finish[static_cast<size_t>(d)] > start) {
                    start = finish[static_cast<size_t>(d)];
                    pred_node[i] = d;
                }
            finish[i] = start + ms;
            if (finish[i] > crit) {
                crit = finish[i];
                last = i;
            }
        }
        *critical_ms = crit;
        *serial_ms = total;
        // critical path composition (per class), reported after the n_classes slots
        t->crit_class_ms.assign(static_cast<size_t>(kNumCat), 0.0);
        t->crit_class_nodes.assign(static_cast<size_t>(kNumCat), 0);
        for (long long i = n ? static_cast<long long>(last) : -1; i >= 0; i = pred_node[static_cast<size_t>(i)]) {
            const int c = t->prof_cat[static_cast<size_t>(i)];
            t->crit_class_ms[static_cast<size_t>(c)] += dur[static_cast<size_t>(i)];
            t->crit_class_nodes[static_cast<size_t>(c)] += 1;
        }
    });
}

ferret_status ferret_trainer_profile_kernels(ferret_trainer* t, char* names, size_t names_cap, double* ms,
                                             uint64_t* launches, double* alg_bytes, int32_t cap, int32_t* n_kernels) {
    return guarded([&] {
        if (!t->graph_profiling) fail(FERRET_E_LOGIC, "profile: the last execute() did not run a profiling graph");
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        std::vector<const void*> order;
        std::map<const void*, std::tuple<double, uint64_t, double>> agg;
        for (size_t i = 0; i < t->prof_func.size(); ++i) {
            const void* f = t->prof_func[i];
            if (!f) continue;
            float m = 0.f;
            cuda_check(cudaEventElapsedTime(&m, t->prof_events[2 * i], t->prof_events[2 * i + 1]), "cudaEventElapsedTime");
            auto it = agg.find(f);
            if (it == agg.end()) {
                order.push_back(f);
                it = agg.emplace(f, std::make_tuple(0.0, uint64_t{0}, 0.0)).first;
            }
            std::get<0>(it->second) += m;
            std::get<1>(it->second) += 1;
            std::get<2>(it->second) += t->prof_bytes[i];
        }
        std::string text;
        int32_t k = 0;
        for (const void* f : order) {
            const char* raw = nullptr;
            std::string name = "?";
            if (cudaFuncGetName(&raw, f) == cudaSuccess && raw) {
                int st = 0;
                char* dem = abi::__cxa_demangle(raw, nullptr, nullptr, &st);
                name = (st == 0 && dem) ? dem : raw;
                std::free(dem);
            }
            if (k < cap) {
                ms[k] = std::get<0>(agg[f]);
                launches[k] = std::get<1>(agg[f]);
                alg_bytes[k] = std::get<2>(agg[f]);
            }
            text += name + "\n";
            ++k;
        }
        *n_kernels = k;
        if (names && names_cap) {
            const size_t m = std::min(text.size(), names_cap - 1);
            std::memcpy(names, text.data(), m);
            names[m] = '\0';
        }
    });
}

ferret_status ferret_trainer_profile_stages(ferret_trainer* t, double* fwd_us, double* bwd_us, double* upd_us,
                                            int32_t n_stages) {
    return guarded([&] {
        if (!t->graph_profiling) fail(FERRET_E_LOGIC, "profile: the last execute() did not run a profiling graph");
        if (n_stages != t->P) fail(FERRET_E_INVALID_ARG, "profile_stages: stage count mismatch");
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        // mean time of one forward / backward / update EVENT of each stage (an
        // event may be several nodes: one per layer, plus the head)
        std::vector<double> f(static_cast<size_t>(n_stages), 0.0), b(f), u(f);
        for (size_t i = 0; i < t->prof_cat.size(); ++i) {
            const int s = t->prof_stage[i];
            if (s < 0 || s >= n_stages) continue;
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, t->prof_events[2 * i], t->prof_events[2 * i + 1]), "cudaEventElapsedTime");
            const int c = t->prof_cat[i];
            (c == kCatForward ? f : c == kCatBackward ? b : u)[static_cast<size_t>(s)] += 1e3 * ms;
        }
        const auto& st = t->stats;
        for (int32_t s = 0; s < n_stages; ++s) {
            // events per stage in the profiled chunk: updates counted, forwards /
            // backwards ~ one per non-dropped unit
            const double units = static_cast<double>(st.predicts > 0 ? st.predicts : 1);
            fwd_us[s] = f[static_cast<size_t>(s)] / units;
            bwd_us[s] = b[static_cast<size_t>(s)] / units;
            upd_us[s] = u[static_cast<size_t>(s)] / units;
        }
    });
}

ferret_status ferret_trainer_profile_critical(ferret_trainer* t, double* class_ms, uint64_t* class_nodes,
                                              int32_t n_classes) {
    return guarded([&] {
        if (t->crit_class_ms.empty()) fail(FERRET_E_LOGIC, "profile_critical: call ferret_trainer_profile first");
        for (int32_t c = 0; c < n_classes && c < kNumCat; ++c) {
            class_ms[c] = t->crit_class_ms[static_cast<size_t>(c)];
            class_nodes[c] = t->crit_class_nodes[static_cast<size_t>(c)];
        }
    });
}

ferret_status ferret_trainer_update_timing(ferret_trainer* t, double* total_ms, uint64_t* launches, double* alg_bytes) {
    return guarded([&] {
        cuda_check(cudaStreamSynchronize(t->stream), "sync");
        double ms = 0.0;
        if (t->graph_timing)
            for (size_t i = 0; i + 1 < t->ev_used; i += 2) {
                float part = 0.f;
                cuda_check(cudaEventElapsedTime(&part, t->ev_pool[i], t->ev_pool[i + 1]), "cudaEventElapsedTime");
                ms += part;
            }
        *total_ms = ms;
        *launches = t->graph_timing ? t->upd_timed : 0;
        *alg_bytes = t->graph_timing ? t->upd_alg_bytes : 0.0;
    });
}

ferret_status ferret_dense_layer(int32_t precision, int32_t direction, const float* W, const float* bias,
                                 const float* X, const float* mask, int32_t B, int32_t in, int32_t out, int32_t relu,
                                 float* Y) {
    return guarded([&] {
        if (precision != FERRET_PREC_TF32 && precision != FERRET_PREC_BF16 && precision != FERRET_PREC_FP32)
            fail(FERRET_E_CONFIG, "dense_layer: unknown precision");
        if (direction != 0 && direction != 1) fail(FERRET_E_INVALID_ARG, "dense_layer: direction must be 0 or 1");
        if (B < 1 || B > fb200::kMaxBatch) fail(FERRET_E_INVALID_ARG, "dense_layer: batch must lie in [1, 16]");
        if (in < 1 || out < 1) fail(FERRET_E_INVALID_ARG, "dense_layer: empty layer");
        if (!W || !X || !Y || (direction == 0 && !bias)) fail(FERRET_E_INVALID_ARG, "dense_layer: null buffer");
        const bool bf16 = precision == FERRET_PREC_BF16;
        if (!fb200::mma_supported(bf16, in, out))
            fail(FERRET_E_CONFIG, "dense_layer: row stride of W must be a multiple of 16 bytes");
        require_device(0);
        const size_t nw = static_cast<size_t>(in) * out;
        const size_t nx = static_cast<size_t>(B) * (direction == 0 ? in : out);
        const size_t ny = static_cast<size_t>(B) * (direction == 0 ? out : in);
        size_t bytes = 0;
        std::vector<void*> bufs;
        struct Cleanup {
            std::vector<void*>& b;
            ~Cleanup() {
                for (void* p : b) cudaFree(p);
            }
        } cleanup{bufs};
        auto up = [&](const void* src, size_t nbytes) {
            unsigned char* d = dalloc<unsigned char>(nbytes, bytes);
            bufs.push_back(d);
            if (src) cuda_check(cudaMemcpy(d, src, nbytes, cudaMemcpyHostToDevice), "H2D");
            return d;
        };
        void* dW;
        if (bf16) {
            std::vector<uint16_t> h(nw);
            for (size_t i = 0; i < nw; ++i) h[i] = bf16_bits(W[i]);
            dW = up(h.data(), nw * 2);
        } else {
            dW = up(W, nw * 4);
        }
        fb200::MmaLayer L;
        L.W = dW;
        L.bwd = direction == 1;
        L.bf16 = bf16;
        L.bias = direction == 0 ? reinterpret_cast<const float*>(up(bias, static_cast<size_t>(out) * 4)) : nullptr;
        L.X = reinterpret_cast<const float*>(up(X, nx * 4));
        L.mask = direction == 1 && mask ? reinterpret_cast<const float*>(up(mask, ny * 4)) : nullptr;
        L.Y = reinterpret_cast<float*>(up(nullptr, ny * 4));
        L.in = in;
        L.out = out;
        L.B = B;
        L.relu = relu;
        L.split = precision == FERRET_PREC_FP32;
        const fb200::MmaGeom g = fb200::mma_geom(bf16, L.bwd, in, out, L.split);
        if (g.partial_floats) {
            L.partial = reinterpret_cast<float*>(up(nullptr, g.partial_floats * 4));
            L.counters = reinterpret_cast<unsigned*>(up(nullptr, static_cast<size_t>(g.mtiles) * 4));
            cuda_check(cudaMemset(L.counters, 0, static_cast<size_t>(g.mtiles) * 4), "memset");
        }
        // FERRET_MMA_STAMPS=<file>: append the per-CTA phase timestamps (measurement)
        const char* stamp_file = std::getenv("FERRET_MMA_STAMPS");
        const size_t n_stamps = static_cast<size_t>(g.S) * g.mtiles * 8;
        if (stamp_file) {
            L.stamps = reinterpret_cast<unsigned long long*>(up(nullptr, n_stamps * 8));
            cuda_check(cudaMemset(L.stamps, 0, n_stamps * 8), "memset");
        }
        fb200::KernelSpec k;
        fb200::spec_mma(L, k);
        if (stamp_file) {  // measurement: W cold in HBM like inside a chunk (the upload left it in L2)
            void* flush = up(nullptr, 256u << 20);
            cuda_check(cudaMemset(flush, 1, 256u << 20), "L2 flush");
        }
        cuda_check(fb200::launch_spec(k, nullptr), "dense_layer launch");
        cuda_check(cudaDeviceSynchronize(), "dense_layer");
        if (stamp_file) {
            std::vector<unsigned long long> h(n_stamps);
            cuda_check(cudaMemcpy(h.data(), L.stamps, n_stamps * 8, cudaMemcpyDeviceToHost), "D2H");
            if (FILE* f = std::fopen(stamp_file, "a")) {
                std::fprintf(f, "layer %d %d %d %d %d\n", precision, direction, in, out, g.S * g.mtiles);
                for (size_t i = 0; i < n_stamps; i += 8)
                    std::fprintf(f, "%llu %llu %llu %llu %llu %llu %llu %llu\n", h[i], h[i + 1], h[i + 2], h[i + 3],
                                 h[i + 4], h[i + 5], h[i + 6], h[i + 7]);
                std::fclose(f);
            }
        }
        cuda_check(cudaMemcpy(Y, L.Y, ny * 4, cudaMemcpyDeviceToHost), "D2H");
    });
}

ferret_status ferret_conv_layer(int32_t tc, int32_t mode, const int32_t* geom, int32_t B, const float* W,
                                const float* bias, const float* X, const float* D, const float* res, int32_t rc,
                                int32_t rh, int32_t rw, const float* mask, int32_t relu, float* Y) {
    return guarded([&] {
        if (tc < 0 || tc > 3) fail(FERRET_E_CONFIG, "conv_layer: tc must lie in [0, 3]");
        if (mode < 0 || mode > 2) fail(FERRET_E_INVALID_ARG, "conv_layer: mode must be 0 (fwd), 1 (dgrad) or 2 (wgrad)");
        if (!geom || !W || !Y || B < 1) fail(FERRET_E_INVALID_ARG, "conv_layer: null buffer or empty batch");
        if (geom[0] != FERRET_LAYER_CONV) fail(FERRET_E_CONFIG, "conv_layer: geometry kind must be FERRET_LAYER_CONV");
        require_device(0);
        fb200::ConvArgs c{};
        c.B = B;
        c.ci = geom[1];
        c.hi = geom[2];
        c.wi = geom[3];
        c.co = geom[4];
        c.k = geom[5];
        c.s = geom[6];
        c.p = geom[7];
        c.ho = (c.hi + 2 * c.p - c.k) / c.s + 1;
        c.wo = (c.wi + 2 * c.p - c.k) / c.s + 1;
        if (c.ci < 1 || c.co < 1 || c.k < 1 || c.s < 1 || c.p < 0 || c.ho < 1 || c.wo < 1)
            fail(FERRET_E_CONFIG, "conv_layer: bad geometry");
        c.tc = tc;
        c.relu = relu;
        c.rc = rc;
        c.rh = rh;
        c.rw = rw;
        const size_t nw = static_cast<size_t>(c.co) * c.ci * c.k * c.k;
        const size_t nin = static_cast<size_t>(B) * c.ci * c.hi * c.wi, nout = static_cast<size_t>(B) * c.co * c.ho * c.wo;
        const size_t nres = static_cast<size_t>(B) * rc * rh * rw;
        const size_t ny = mode == fb200::kConvFwd ? nout : mode == fb200::kConvDgrad ? nin : nw;
        size_t bytes = 0;
        std::vector<void*> bufs;
        struct Cleanup {
            std::vector<void*>& b;
            ~Cleanup() {
                for (void* p : b) cudaFree(p);
            }
        } cleanup{bufs};
        auto up = [&](const void* src, size_t n) -> float* {
            float* d = dalloc<float>(std::max<size_t>(n, 1), bytes);
            bufs.push_back(d);
            if (src) cuda_check(cudaMemcpy(d, src, n * 4, cudaMemcpyHostToDevice), "H2D");
            return d;
        };
        c.W = up(W, nw);
        if (mode == fb200::kConvFwd) c.bias = up(bias, static_cast<size_t>(c.co));
        if (mode != fb200::kConvDgrad) c.X = up(X, nin);
        if (mode != fb200::kConvFwd) c.D = up(D, nout);
        if (res && mode != fb200::kConvWgrad) c.res = up(res, nres);
        if (mask && mode == fb200::kConvDgrad) c.mask = up(mask, nin);
        c.Y = up(nullptr, ny);
        const size_t part = fb200::conv_plan(c, mode, 0);
        if (part) c.partial = up(nullptr, part);
        if (c.kt && mode != fb200::kConvWgrad) {
            c.Wt = up(nullptr, nw);
            fb200::KernelSpec kw;
            fb200::spec_conv_wprep(c, mode, kw);
            cuda_check(fb200::launch_spec(kw, nullptr), "conv_layer weight prep");
        }
        // FERRET_CONV_STAMPS=<file>: append per-CTA phase timestamps of the tensor-core kernel
        const char* stamp_file = std::getenv("FERRET_CONV_STAMPS");
        const size_t n_ctas = static_cast<size_t>((c.N + 127) / 128) * ((c.M + 127) / 128) * c.splits;
        if (stamp_file && tc) {
            c.stamps = reinterpret_cast<unsigned long long*>(up(nullptr, n_ctas * 16));
            cuda_check(cudaMemset(c.stamps, 0, n_ctas * 64), "memset");
        }
        fb200::KernelSpec g, r;
        const int n = fb200::spec_conv(c, mode, g, r);
        cuda_check(fb200::launch_spec(g, nullptr), "conv_layer launch");
        if (n == 2) cuda_check(fb200::launch_spec(r, nullptr), "conv_layer reduce");
        cuda_check(cudaDeviceSynchronize(), "conv_layer");
        if (c.stamps) {
            std::vector<unsigned long long> h(n_ctas * 8);
            cuda_check(cudaMemcpy(h.data(), c.stamps, n_ctas * 64, cudaMemcpyDeviceToHost), "D2H");
            if (FILE* f = std::fopen(stamp_file, "a")) {
                std::fprintf(f, "conv tc %d mode %d geom %d %d %d %d B %d grid %d %d %d atoms/cta %d\n", tc, mode, c.ci,
                             c.hi, c.co, c.k, B, (c.N + 127) / 128, (c.M + 127) / 128, c.splits, c.apc);
                for (size_t i = 0; i < n_ctas; ++i)
                    std::fprintf(f, "%llu %llu %llu %llu %llu %llu %llu\n", h[8 * i], h[8 * i + 1], h[8 * i + 2],
                                 h[8 * i + 3], h[8 * i + 4], h[8 * i + 5], h[8 * i + 6]);
                std::fclose(f);
            }
        }
        cuda_check(cudaMemcpy(Y, c.Y, ny * 4, cudaMemcpyDeviceToHost), "D2H");
    });
}

ferret_status ferret_compensate(int32_t policy, const double* g, const double* const* chain, int32_t chain_len,
                                double* lambda, double* v_r, double* v_a, double* mean_gap, size_t n, double lambda0,
                                double alpha, double eta_lambda, double nu, double* out) {
    return guarded([&] {
        if (chain_len < 1) fail(FERRET_E_INVALID_ARG, "compensate_iterative: empty version chain");
        if (policy < 0 || policy > 4) fail(FERRET_E_CONFIG, "unknown compensation policy");
        if (policy == FERRET_POLICY_ITER_FISHER && !lambda) fail(FERRET_E_INVALID_ARG, "compensate: lambda required");
        if (policy == FERRET_POLICY_GAP && !mean_gap) fail(FERRET_E_INVALID_ARG, "compensate: mean_gap required");
        require_device(0);
        // fp64 end to end (the reference's arithmetic): the state round-trips without
        // rounding, and the chain is a device pointer table of any length
        size_t bytes = 0;
        const size_t nn = n ? n : 1;
        std::vector<void*> bufs;
        struct Cleanup {
            std::vector<void*>& b;
            ~Cleanup() {
                for (void* p : b) cudaFree(p);
            }
        } cleanup{bufs};
        auto up = [&](const double* src) {
            double* d = dalloc<double>(nn, bytes);
            bufs.push_back(d);
            if (src && n) cuda_check(cudaMemcpy(d, src, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
            return d;
        };
        auto down = [&](const double* d, double* dst) {
            if (n) cuda_check(cudaMemcpy(dst, d, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        };
        const double* dg = up(g);
        std::vector<const double*> links(static_cast<size_t>(chain_len));
        for (int32_t i = 0; i < chain_len; ++i) links[static_cast<size_t>(i)] = up(chain[i]);
        const double** dchain = dalloc<const double*>(links.size(), bytes);
        bufs.push_back(const_cast<double**>(dchain));
        cuda_check(cudaMemcpy(dchain, links.data(), links.size() * sizeof(double*), cudaMemcpyHostToDevice), "H2D chain");
        const bool learn = policy == FERRET_POLICY_ITER_FISHER && v_r && v_a && eta_lambda > 0.0;
        double* dl = policy == FERRET_POLICY_ITER_FISHER ? up(lambda) : nullptr;
        double* dvr = learn ? up(v_r) : nullptr;
        double* dva = learn ? up(v_a) : nullptr;
        double* dgap = policy == FERRET_POLICY_GAP ? up(mean_gap) : nullptr;
        double* dout = up(nullptr);
        cuda_check(fb200::nm_compensate(policy, dg, dchain, chain_len, dl, dvr, dva, dgap, n, lambda0, alpha,
                                        learn ? eta_lambda : 0.0, nu, dout, nullptr),
                   "compensate launch");
        cuda_check(cudaDeviceSynchronize(), "compensate");
        down(dout, out);
        if (dl) down(dl, lambda);
        if (dvr) down(dvr, v_r);
        if (dva) down(dva, v_a);
        if (dgap) down(dgap, mean_gap);
    });
}

} // extern "C"
