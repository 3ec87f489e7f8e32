/* ferret-b200 C ABI — the boundary between the reference-shaped C++ API
 * (the headers in include/ferret/, namespace ferret) and the sm_100a implementation in
 * libferret_b200.so. Plain C types only: no torch, no STL, no CUDA types.
 *
 * Every entry point below replaces one reference interface; the citation is
 * the reference file:line of the call it stands in for
 * (reference root: proj/include/ferret/).
 *
 * Conventions
 *   - Caller owns every input buffer (read-only; copied as needed) and every
 *     output buffer (caller-allocated, sizes stated per function).
 *   - Every function returns ferret_status; FERRET_OK == 0. On failure
 *     ferret_last_error() returns the message (thread-local), and the status
 *     maps 1:1 onto the exception type the reference throws
 *     (types.hpp:13-25, compensate.hpp:17, learner.hpp:276, sim.hpp:396).
 *   - A trainer is single-threaded like the reference's PipelineTrainer
 *     (learner.hpp:330); one trainer per host thread.
 *   - There is no CPU fallback: without a usable sm_100 device every
 *     trainer/compute call returns FERRET_E_NO_DEVICE.
 */
#ifndef FERRET_B200_H
#define FERRET_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FERRET_API __attribute__((visibility("default")))
#else
#define FERRET_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FERRET_OK = 0,
    FERRET_E_SCHEMA = 1,       /* ferret::SchemaError            types.hpp:13 */
    FERRET_E_BOUND = 2,        /* ferret::BoundError             types.hpp:18 */
    FERRET_E_CONFIG = 3,       /* ferret::ConfigError            types.hpp:23 */
    FERRET_E_INVALID_ARG = 4,  /* std::invalid_argument          compensate.hpp:17, net.hpp:159 */
    FERRET_E_OUT_OF_RANGE = 5, /* std::out_of_range              learner.hpp:276, compensate.hpp:155 */
    FERRET_E_LOGIC = 6,        /* std::logic_error               sim.hpp:396 */
    FERRET_E_CUDA = 7,         /* CUDA runtime failure (no reference counterpart) */
    FERRET_E_NO_DEVICE = 8     /* no sm_100 device visible (no reference counterpart) */
} ferret_status;

/* EventKind, sim.hpp:23 */
enum { FERRET_EV_ARRIVAL = 0, FERRET_EV_DROP = 1, FERRET_EV_FORWARD = 2,
       FERRET_EV_RECOMPUTE = 3, FERRET_EV_BACKWARD = 4, FERRET_EV_UPDATE = 5 };
/* CompensationPolicy, compensate.hpp:20 */
enum { FERRET_POLICY_NONE = 0, FERRET_POLICY_STEP = 1, FERRET_POLICY_GAP = 2,
       FERRET_POLICY_FISHER = 3, FERRET_POLICY_ITER_FISHER = 4 };
/* Activation, net.hpp:17 */
enum { FERRET_ACT_RELU = 0, FERRET_ACT_IDENTITY = 1 };
/* StepOutcome, metrics.hpp:15 */
enum { FERRET_STEP_CORRECT = 0, FERRET_STEP_WRONG = 1, FERRET_STEP_DROPPED = 2 };
/* arithmetic of the device path (no reference counterpart: the reference is fp64) */
/* FP32: parity mode (SIMT fp32, 1e-4 parameter parity with the fp64 oracle).
 * BF16 / TF32: fast modes — dense-layer forward and input-gradient on the
 * tcgen05 tensor cores (bf16 copies of the weight versions, or tf32 reads of
 * the fp32 versions), fp32 accumulation; the compensation + SGD update stays
 * fp32 on the fp32 master versions. Parity bar: online accuracy within 0.5 pp. */
enum { FERRET_PREC_FP32 = 0, FERRET_PREC_BF16 = 1, FERRET_PREC_TF32 = 2 };

/* Convolutional extension (BASELINE config 3, "ResNet-18-style CNN"; the
 * reference has no convolution): an optional geometry per layer,
 * FERRET_GEOM_INTS int32 each = {kind, c_in, h_in, w_in, c_out, k, stride, pad, res}.
 *   DENSE      z = W x + b (the reference's layer; c_in = in, h_in = w_in = 1)
 *   CONV       z[co][oh][ow] = b[co] + sum W[co][ci][kh][kw] x[ci][oh*s-p+kh][ow*s-p+kw]
 *              (zero padding, NCHW per sample); res = 1 adds the shortcut of the
 *              input of layer l-1 (a two-conv basic block): identity, or when the
 *              block downsamples, stride subsample + zero channels ("option A")
 *   GAP_DENSE  z = W mean_hw(x) + b (global average pool fused into the head)
 * then the layer's activation. Activation widths (in[l], out[l]) are c*h*w;
 * parameters per layer: W (c_out x c_in*k*k, or c_out x c_in) then b (c_out).
 * Partition bounds may not split a residual block (FERRET_E_CONFIG). */
enum { FERRET_LAYER_DENSE = 0, FERRET_LAYER_CONV = 1, FERRET_LAYER_GAP_DENSE = 2 };
#define FERRET_GEOM_INTS 9

/* DenseNet, net.hpp:20-51. params in flatten() order (learner.hpp:26-34):
 * per layer W (row-major out x in) then b. */
typedef struct {
    int32_t n_layers;
    const uint64_t* in;
    const uint64_t* out;
    const int32_t* act;
    const double* params;
    const int32_t* geom;  /* nullable (all dense, the reference's DenseNet): n_layers x FERRET_GEOM_INTS */
} ferret_net_desc;

/* PipelineTrainOptions, learner.hpp:319-325, plus the Compensator constants
 * (learner.hpp:85-86, compensate.hpp:59-64), the replay capacity
 * (learner.hpp:24) and the B200-side knobs. Fill with
 * ferret_train_opts_default() before editing. */
typedef struct {
    int32_t policy;            /* FERRET_POLICY_*; reference default none */
    double lr;                 /* 1e-3 */
    double eta_lambda;         /* 1e-3 */
    double lambda0;            /* 0.2 */
    double alpha;              /* 0.99 */
    double nu;                 /* 2e-6 */
    int32_t replay;            /* 0/1 */
    uint64_t replay_seed;      /* 0 */
    uint64_t replay_capacity;  /* 5000 */
    int32_t precision;         /* FERRET_PREC_FP32 */
    int32_t micro_batch;       /* stream samples per pipeline unit; 1 = reference semantics */
    int32_t device;            /* CUDA ordinal of this stage group */
    int32_t as_shipped;        /* 1: reproduce the reference's worker-keyed no-op trainer */
} ferret_train_opts;

/* SimEvent, sim.hpp:38-46 */
typedef struct {
    double time;
    int32_t kind;
    int32_t worker;
    int32_t stage;
    int32_t staleness;
    int64_t item;
    int64_t version;
} ferret_event;

/* StepRecord, metrics.hpp:18-23 */
typedef struct {
    int64_t item;
    int32_t outcome;
    int32_t _pad;
    uint64_t predicted;
    uint64_t label;
} ferret_step_record;

/* LayerProfile, types.hpp:35-40 */
typedef struct {
    double t_f;
    double t_b;
    uint64_t w;
    uint64_t a;
} ferret_layer_profile;

/* StreamSpec, types.hpp:139-151 */
typedef struct {
    double t_d;
    double decay_c;
    double value;
    double horizon;
} ferret_stream_spec;

FERRET_API const char* ferret_last_error(void);
FERRET_API const char* ferret_version(void);
/* 1 if an sm_100 device is visible and the kernels in this library load on it */
FERRET_API int32_t ferret_device_available(void);

FERRET_API void ferret_train_opts_default(ferret_train_opts* opts);

/* ---------------- host tiers (bit-exact with the reference) ---------------- */

/* make_dense_net, net.hpp:54-71; params_out sized ferret_net_param_count */
FERRET_API size_t ferret_net_param_count(const uint64_t* widths, int32_t n_widths);
FERRET_API ferret_status ferret_make_dense_net(const uint64_t* widths, int32_t n_widths, uint64_t seed,
                                    int32_t hidden_act, double* params_out, size_t n_params);

/* profile_from_net, net.hpp:263-274; layers_out has n_widths-1 entries */
FERRET_API ferret_status ferret_profile_from_widths(const uint64_t* widths, int32_t n_widths,
                                         double seconds_per_param, ferret_layer_profile* layers_out);

/* synth_drift_stream, stream.hpp:43-87; features_out n*n_features (row-major), labels_out n */
FERRET_API ferret_status ferret_synth_drift_stream(size_t n, size_t n_features, size_t n_classes, int32_t drift,
                                        uint64_t seed, double rotate_rate, double noise,
                                        double* features_out, uint64_t* labels_out);

/* A schedule = plan (planner.hpp:192) or forced partition + default_config
 * (planner.hpp:54), stage_stats (profile.hpp:167) and simulate (sim.hpp:401). */
typedef struct ferret_schedule ferret_schedule;

FERRET_API ferret_status ferret_schedule_plan(const ferret_layer_profile* layers, int32_t n_layers, double t_d,
                                   const ferret_stream_spec* spec, uint64_t budget, int32_t max_stages,
                                   size_t n_items, ferret_schedule** out);
FERRET_API ferret_status ferret_schedule_forced(const ferret_layer_profile* layers, int32_t n_layers, double t_d,
                                     const ferret_stream_spec* spec, const uint64_t* bounds,
                                     int32_t n_bounds, int32_t recompute, size_t n_items,
                                     ferret_schedule** out);
/* number of bounds; copies min(n, cap) into out */
/* A schedule from persisted text (no reference counterpart: the reference
 * writes plans and traces, planner.hpp:217-246, sim.hpp:406-436, and reads
 * only plans, planner.hpp:248-309): ferret-plan v1 gives the partition, the
 * ferret-trace v1 event log the replay. Malformed text -> FERRET_E_SCHEMA. */
FERRET_API ferret_status ferret_schedule_load(const char* plan_text, size_t plan_len, const char* trace_text,
                                              size_t trace_len, ferret_schedule** out);
FERRET_API int32_t ferret_schedule_bounds(const ferret_schedule* s, uint64_t* out, int32_t cap);
FERRET_API size_t ferret_schedule_event_count(const ferret_schedule* s);
FERRET_API ferret_status ferret_schedule_events(const ferret_schedule* s, ferret_event* out, size_t cap);
/* write_plan (planner.hpp:219) / write_trace (sim.hpp:408) text; returns bytes
 * needed incl. NUL, copies up to cap */
FERRET_API size_t ferret_schedule_plan_text(const ferret_schedule* s, char* buf, size_t cap);
FERRET_API size_t ferret_schedule_trace_text(const ferret_schedule* s, char* buf, size_t cap);
FERRET_API void ferret_schedule_destroy(ferret_schedule* s);

/* ---------------- planner re-costed for B200 (north-star item 4) ----------------
 * The reference planner (planner.hpp:180-215, analytics.hpp:72-104) prices a plan with
 * synthetic per-layer times (net.hpp:263-274: 1e-6 s per parameter) and memory in
 * parameter/activation COUNT units. The B200 planner keeps its search unchanged and
 * feeds it (1) per-layer t_f / t_b measured on the device and (2) w / a in HBM BYTES
 * of this trainer's layout; the chosen plan is then priced exactly by the trainer's own
 * dry-run footprint (ferret_trainer_footprint) and re-planned under a tightened budget
 * until it fits. Candidate partitions are limited to max_stages (= #GPUs, one stage per
 * GPU at most). */
typedef struct {
    int32_t micro_batch;       /* stream samples per pipeline unit */
    int32_t precision;         /* FERRET_PREC_*: bf16 keeps a bf16 copy of every weight version (+2 B) */
    int32_t policy;            /* FERRET_POLICY_*: compensator state bytes */
    double eta_lambda;         /* iter_fisher: > 0 learns lambda (v_r, v_a state) */
    int32_t replay;            /* ER replay pool */
    uint64_t replay_capacity;
    uint64_t chunk_units;      /* pipeline units per compiled chunk (staging); 0 = n_items */
} ferret_b200_cost;
FERRET_API void ferret_b200_cost_default(ferret_b200_cost* c);

/* profile_from_net (net.hpp:263-274) re-costed on the device: per layer, t_f = measured
 * mean device seconds of the layer's forward event and t_b = its backward + compensated
 * update, from a profiled replay of the real kernels with one layer per stage (`units`
 * pipeline units of a synthetic stream, after one warm-up chunk); w / a are the
 * reference's counts. layers_out has n_widths - 1 entries. */
FERRET_API ferret_status ferret_measure_profile(const uint64_t* widths, int32_t n_widths, const ferret_b200_cost* cost,
                                                int32_t units, int32_t device, ferret_layer_profile* layers_out);

/* A (measured) profile with w = HBM bytes of one weight version of the layer and
 * a = stash bytes one in-flight unit holds for it (activation + delta, micro_batch rows):
 * the reference planner's count units become bytes. */
FERRET_API ferret_status ferret_b200_byte_profile(const ferret_layer_profile* layers, int32_t n_layers,
                                                  const ferret_b200_cost* cost, ferret_layer_profile* out);

typedef struct {
    uint64_t budget_bytes;     /* the caller's HBM budget for the whole pipeline */
    uint64_t fixed_bytes;      /* plan-independent: compensator state, normalizer, staging, replay pool */
    uint64_t planner_budget;   /* budget handed to the reference search (bytes) on the last pass */
    uint64_t planner_bytes;    /* the reference memory model of the chosen plan, in bytes */
    uint64_t predicted_bytes;  /* fixed + planner */
    uint64_t trainer_bytes;    /* exact: the trainer's footprint for the plan's event log */
    int32_t passes;            /* planner passes (1 = the first plan fit) */
    int32_t stages;
    int32_t fits;              /* trainer_bytes <= budget_bytes */
} ferret_b200_plan_report;

/* plan_b200: widths give the net (dense, ReLU hidden), layers the measured profile
 * (ferret_measure_profile, or any ModelProfile with times in seconds and count units),
 * budget in bytes (0 = unconstrained), max_stages = #GPUs (0 = unlimited). The
 * schedule's plan is a reference PlanResult whose `memory` is in bytes. */
FERRET_API ferret_status ferret_plan_b200(const uint64_t* widths, int32_t n_widths, const ferret_layer_profile* layers,
                                          double t_d, const ferret_stream_spec* spec, uint64_t budget_bytes,
                                          int32_t max_stages, const ferret_b200_cost* cost, size_t n_items,
                                          ferret_schedule** out, ferret_b200_plan_report* report);

/* ---------------- hot path: PipelineTrainer on sm_100a ---------------- */

typedef struct ferret_trainer ferret_trainer;

/* PipelineTrainer(DenseNet, PartitionScheme, PipelineTrainOptions), learner.hpp:332-346 */
FERRET_API ferret_status ferret_trainer_create(const ferret_net_desc* net, const uint64_t* bounds, int32_t n_bounds,
                                    const ferret_train_opts* opts, ferret_trainer** out);

/* PipelineTrainer::run(trace, stream), learner.hpp:348-363 — end to end:
 * copies the host stream in, replays the event log on the device, copies the
 * StepRecord log out (n_items entries). Synchronous. n_items counts stream
 * samples (= trace items x micro_batch). */
FERRET_API ferret_status ferret_trainer_run(ferret_trainer* t, const ferret_event* events, size_t n_events,
                                 const double* features, const uint64_t* labels, size_t n_items,
                                 size_t n_features, ferret_step_record* log_out);

/* Split form of ferret_trainer_run for device-resident timing:
 * load_stream (H2D) -> execute(chunk) (async on ferret_trainer_stream) ->
 * fetch_log (D2H). execute() replays the event log over samples
 * [chunk*n_chunk_items, (chunk+1)*n_chunk_items) of the loaded stream and
 * continues training from the current state (normalizer included). */
FERRET_API ferret_status ferret_trainer_load_stream(ferret_trainer* t, const double* features, const uint64_t* labels,
                                         size_t n_items, size_t n_features);
FERRET_API ferret_status ferret_trainer_set_schedule(ferret_trainer* t, const ferret_event* events, size_t n_events,
                                          size_t n_chunk_items);
FERRET_API ferret_status ferret_trainer_execute(ferret_trainer* t, size_t chunk);
FERRET_API ferret_status ferret_trainer_fetch_log(ferret_trainer* t, size_t chunk, ferret_step_record* log_out);
FERRET_API ferret_status ferret_trainer_sync(ferret_trainer* t);
/* Stream ingest at rate (PipelineTrainer::run over a long stream, chunk by
 * chunk): n_items host samples, a whole number of set_schedule chunks, replay
 * the schedule chunk after chunk, continuing from the current state; log_out
 * gets n_items StepRecords (items numbered within the call). Host->device
 * copies of chunk c+1 overlap chunk c's graph through two device staging slots
 * on a copy stream; pass pinned host memory (cudaMallocHost) for true DMA.
 * Synchronous from the caller's view. */
FERRET_API ferret_status ferret_trainer_ingest(ferret_trainer* t, const double* features, const uint64_t* labels,
                                               size_t n_items, size_t n_features, ferret_step_record* log_out);

/* cudaStream_t the trainer launches on, as an opaque pointer (for CUDA-event timing) */
FERRET_API void* ferret_trainer_stream(ferret_trainer* t);

/* Stage sharding, one process per GPU (no reference counterpart: the reference
 * is single-process, learner.hpp:384-385 keeps every stage in one object).
 * Call set_shard before set_schedule on every rank with the same stage->rank
 * map (non-decreasing, stage 0 on rank 0). set_schedule then sizes this rank's
 * inbox from the log's hand-off plan; exchange inbox_handle() (a 64-byte CUDA
 * IPC handle) between ranks and open_peer() every rank this one sends to.
 * Each rank replays the whole log but launches only its stages' kernels; stage
 * outputs, input gradients (sent unmasked, masked by the receiver) and the
 * predict / replay sweeps cross ranks as direct stores into the peer's inbox
 * followed by a release flag (NVLink P2P on an 8xB200 box). Flow control is
 * on the device: the receiver acknowledges every consumed message by storing
 * the chunk's epoch into the sender's ack slot, and the sender of the next
 * chunk's message in that slot waits for it, so ranks run chunk after chunk
 * (and ingest() many chunks per call) with no host barrier. Only the
 * rank owning the last stage produces predictions (fetch_log); only rank 0
 * holds the normalizer; params/comp_state are valid for the stages a rank owns. */
FERRET_API ferret_status ferret_trainer_set_shard(ferret_trainer* t, int32_t rank, int32_t world,
                                                  const int32_t* stage_owner);
FERRET_API ferret_status ferret_trainer_inbox_handle(ferret_trainer* t, void* out, size_t cap);
FERRET_API ferret_status ferret_trainer_open_peer(ferret_trainer* t, int32_t peer, const void* handle);
/* The hand-off plan of the current schedule: per destination rank, incoming
 * message bytes and message count per chunk. Works on plan-only trainers
 * (created with opts.device = -1: host passes only, no device touched), so the
 * multi-rank logic can be checked without a GPU. */
FERRET_API ferret_status ferret_trainer_handoff_plan(ferret_trainer* t, uint64_t* bytes_to_rank, uint64_t* msgs_to_rank,
                                                     int32_t world);

/* TrainOutcome::net (learner.hpp:177-181): current params, fp64, flatten() order */
FERRET_API ferret_status ferret_trainer_params(ferret_trainer* t, double* out, size_t n);
/* per-stage compensator state (compensate.hpp:55-58); any pointer may be NULL.
 * mean_gap is the gap policy's running mean (learner.hpp:126). n = stage params */
FERRET_API ferret_status ferret_trainer_comp_state(ferret_trainer* t, int32_t stage, double* lambda, double* v_r,
                                        double* v_a, double* mean_gap, size_t n);
/* TrainOutcome::normalizer (learner.hpp:180): count, mean[f], m2[f] */
FERRET_API ferret_status ferret_trainer_normalizer(ferret_trainer* t, uint64_t* count, double* mean, double* m2,
                                        size_t n_features);
/* ---- The reference's dense-net math (net.hpp:99-208) on the device, fp64 ----
 * Host buffers in and out, synchronous, on the calling thread's current CUDA device.
 * Every sum runs in the reference's index order with separately rounded products and
 * sums, so affine_forward / forward_all / the gradients / apply_sgd are bit-identical to
 * the reference's loops; exp and log are CUDA's (<= 2 ulp from glibc), so softmax and the
 * loss (and the gradients through the softmax delta) agree to ~1e-15 relative.
 * detail::affine_forward (net.hpp:99-108): z = W x + b, W row-major out x in */
FERRET_API ferret_status ferret_affine_forward(const double* W, const double* b, uint64_t in, uint64_t out,
                                               const double* x, double* z);
/* detail::apply_activation (net.hpp:110-113), in place */
FERRET_API ferret_status ferret_apply_activation(int32_t act, double* z, size_t n);
/* detail::softmax (net.hpp:115-125) */
FERRET_API ferret_status ferret_softmax(const double* z, size_t n, double* p);
/* forward_all (net.hpp:130-142) for n samples (x: n x in, row-major): acts row s holds every
 * layer's post-activation output, layer after layer (n x sum(out)) */
FERRET_API ferret_status ferret_net_forward_all(const ferret_net_desc* net, const double* x, size_t n, double* acts);
/* forward_backward (net.hpp:157-200): mean softmax cross-entropy over the batch and its
 * gradients in flatten() order (per layer W then b); FERRET_E_INVALID_ARG for an empty
 * batch or a label out of range */
FERRET_API ferret_status ferret_net_forward_backward(const ferret_net_desc* net, const double* x,
                                                     const uint64_t* labels, size_t n, double* loss, double* grads);
/* apply_sgd (net.hpp:202-208): params -= lr * grads, in place, flatten() order */
FERRET_API ferret_status ferret_net_apply_sgd(double* params, const double* grads, size_t n, double lr);

/* The replay draws made so far (ReplayBuffer::sample, learner.hpp:75-78, called by
 * replay_step :513-519): the stream sample index of every drawn sample, in draw order,
 * across every run/execute/ingest call of this trainer (B draws per replay step at
 * micro-batch B). Writes min(cap, total) indices to `out` (may be NULL) and the total
 * to *n. The reservoir arithmetic is the reference's (same mt19937_64 draws), so these
 * equal the reference trainer's replay indices element for element. */
FERRET_API ferret_status ferret_trainer_replay_draws(ferret_trainer* t, int64_t* out, size_t cap, size_t* n);
/* counters of the last execute/run: kernel launches, ring depth per stage, ... */
typedef struct {
    uint64_t kernel_launches;
    uint64_t events;
    uint64_t updates;
    uint64_t replays;
    uint64_t predicts;
    int32_t ring_depth[16];
    int32_t stash_slots;
    double mean_tau[16];         /* mean trainer staleness per update, per stage */
    uint64_t update_elems[16];   /* params touched by updates per stage */
    uint64_t device_bytes;       /* HBM the trainer allocated */
} ferret_trainer_stats;
FERRET_API ferret_status ferret_trainer_get_stats(ferret_trainer* t, ferret_trainer_stats* out);
/* HBM footprint of the current schedule (no reference counterpart; north-star item 4, the
 * planner re-costed in bytes): what the trainer holds once execute() has compiled the
 * schedule's chunk graph, from the same dry pass over the event log that sizes the version
 * rings (exact retention) and the stash. Works on plan-only trainers (device -1), so a
 * planner can price a candidate plan without a GPU. Excludes the tensor-core layers'
 * graph-build scratch (split-K partials, conv weight copies). */
typedef struct {
    uint64_t total;        /* bytes */
    uint64_t rings;        /* weight-version rings, fp32 (+ bf16 copies in bf16 mode) */
    uint64_t comp_state;   /* compensator state (iter_fisher: lambda, v_r, v_a; gap: mean gap) */
    uint64_t stash;        /* in-flight unit activations and deltas (+ the replay slot) */
    uint64_t scratch;      /* backward split-reduction scratch */
    uint64_t other;        /* staging, control block, normalizer, replay pool, resident stream, tables */
    int32_t ring_depth[16];
    int32_t stash_slots;
} ferret_footprint;
FERRET_API ferret_status ferret_trainer_footprint(ferret_trainer* t, ferret_footprint* out);
FERRET_API void ferret_trainer_destroy(ferret_trainer* t);

/* Measurement hook (no reference counterpart): when enabled, every update
 * launch (the fused compensation + SGD kernel, learner.hpp:491-504) is
 * bracketed by CUDA events on the trainer's stream. update_timing() returns the
 * summed kernel time, the number of timed launches and their algorithmic HBM
 * bytes, then resets the counters. */
FERRET_API ferret_status ferret_trainer_set_timing(ferret_trainer* t, int32_t enable);
/* Profile mode (no reference counterpart): the next execute() runs the chunk
 * graph serialised with an event pair around every node. profile() returns per
 * node class {normalize, predict, forward, backward, update, replay, other}
 * the summed device time, node count and algorithmic HBM bytes,
 * the serial total, and the critical
 * path of the concurrent DAG computed from the measured node times. */
FERRET_API ferret_status ferret_trainer_set_profiling(ferret_trainer* t, int32_t enable);
/* After a profiled execute(): per KERNEL SYMBOL (demangled, '\n'-separated in `names`, in
 * first-launch order) the summed device ms, launch count and algorithmic HBM bytes of its
 * launches in the chunk. Writes min(cap, n) entries; *n_kernels = distinct kernels. */
FERRET_API ferret_status ferret_trainer_profile_kernels(ferret_trainer* t, char* names, size_t names_cap,
                                                        double* ms, uint64_t* launches, double* alg_bytes,
                                                        int32_t cap, int32_t* n_kernels);
/* After ferret_trainer_profile: per node class, device ms and node count along the critical path. */
FERRET_API ferret_status ferret_trainer_profile_critical(ferret_trainer* t, double* class_ms, uint64_t* class_nodes,
                                                         int32_t n_classes);
/* After a profiled execute(): mean device microseconds per processed unit of
 * each stage's forward, backward and update work (the measured costs the
 * planner's LayerProfile t_f / t_b stand for, profile.hpp / net.hpp:263). */
FERRET_API ferret_status ferret_trainer_profile_stages(ferret_trainer* t, double* fwd_us, double* bwd_us,
                                                       double* upd_us, int32_t n_stages);
FERRET_API ferret_status ferret_trainer_profile(ferret_trainer* t, double* class_ms, uint64_t* class_nodes,
                                                double* class_bytes, int32_t n_classes, double* critical_ms,
                                                double* serial_ms);
FERRET_API ferret_status ferret_trainer_update_timing(ferret_trainer* t, double* total_ms, uint64_t* launches,
                                                      double* alg_bytes);

/* Exact resume (ferret-ckpt v1, net.hpp:210-259, extended with the
 * trainer state): "ferret-state v2" = text header (net shape, bounds, options,
 * normalizer count, version counters, replay reservoir RNG state and labels)
 * + raw arrays (live parameters per stage in the device slot layout,
 * compensator state, normalizer mean/M2, replay pool rows). Valid between
 * execute()/run() calls. save_state: *size = bytes needed; the state is
 * written when buf has room. load_state into a trainer built with the same
 * net, bounds and options continues bit for bit; mismatch -> FERRET_E_SCHEMA. */
FERRET_API ferret_status ferret_trainer_save_state(ferret_trainer* t, void* buf, size_t cap, size_t* size);
FERRET_API ferret_status ferret_trainer_load_state(ferret_trainer* t, const void* buf, size_t len);

/* ---------------- sequential learners on the device ---------------- */

/* Options of a sequential learner: StaleHarness(net, policy, ring_depth, lr,
 * eta_lambda) (learner.hpp:134-143) and train_sequential's lr / replay /
 * replay_seed (learner.hpp:197-199). Compensator constants as in
 * ferret_train_opts_default (lambda0 0.2, alpha 0.99, nu 2e-6). */
typedef struct {
    int32_t policy;            /* FERRET_POLICY_*: the harness's compensation (train_sequential: none) */
    uint64_t ring_depth;       /* VersionRing capacity (harness); 1 for train_sequential */
    double lr;                 /* 1e-3 */
    double eta_lambda;         /* 1e-3 */
    int32_t replay;            /* train_sequential: one ER sample per step */
    uint64_t replay_seed;
    uint64_t replay_capacity;  /* 5000 (kReplayBuffer) */
    int32_t precision;         /* FERRET_PREC_* */
    int32_t device;
} ferret_seq_opts;

/* A sequential learner: a trainer holding every layer in one stage, whose items
 * run in order (each item's kernels captured into one CUDA graph per call).
 * ferret_trainer_params / _normalizer / _comp_state / _destroy apply to it. */
FERRET_API ferret_status ferret_seq_create(const ferret_net_desc* net, const ferret_seq_opts* opts,
                                           ferret_trainer** out);
/* StaleHarness::ocl_step (learner.hpp:145-163) for n_items items in order:
 * observe + standardise, predict with the live net (preds_out[i]), gradient at
 * the version taus[i] steps behind (clamped to the ring), Compensator::apply
 * over the chain, SGD, push. One call with n items == n ocl_step calls. */
FERRET_API ferret_status ferret_seq_ocl_steps(ferret_trainer* t, const double* features, const uint64_t* labels,
                                              const int32_t* taus, size_t n_items, size_t n_features,
                                              uint64_t* preds_out);
/* train_sequential (learner.hpp:197-225) over the kept items of the stream
 * (indices from ferret_apply_skip_policy, ascending): log_out gets n_items
 * StepRecords, skipped items logged as dropped. */
FERRET_API ferret_status ferret_seq_train(ferret_trainer* t, const double* features, const uint64_t* labels,
                                          size_t n_items, size_t n_features, const int64_t* kept, size_t n_kept,
                                          ferret_step_record* log_out);
/* predict_class (net.hpp:150-154) at the live version for n_items held-out rows,
 * standardised with the learner's normalizer state, observing nothing
 * (test_accuracy, learner.hpp:185-192). */
FERRET_API ferret_status ferret_seq_predict(ferret_trainer* t, const double* features, size_t n_items,
                                            size_t n_features, uint64_t* preds_out);
/* Restore a RunningNormalizer state (count, mean[f], m2[f]) into the learner. */
FERRET_API ferret_status ferret_seq_set_normalizer(ferret_trainer* t, uint64_t count, const double* mean,
                                                   const double* m2, size_t n_features);
/* load_csv_stream (stream.hpp:144-186): header row, numeric cells, one label
 * column, optional gzip (.gz, zlib), host-side like the reference; errors as
 * SchemaError. Read the rows with ferret_csv_read into n_items x n_features
 * features (row-major) and n_items labels. */
typedef struct ferret_csv ferret_csv;
FERRET_API ferret_status ferret_csv_load(const char* path, const char* label_column, ferret_csv** out);
FERRET_API ferret_status ferret_csv_shape(const ferret_csv* c, size_t* n_items, size_t* n_features, size_t* n_classes);
FERRET_API ferret_status ferret_csv_read(const ferret_csv* c, double* features, uint64_t* labels);
FERRET_API void ferret_csv_destroy(ferret_csv* c);
/* apply_skip_policy (stream.hpp:225-304) on the host: kind 0 oracle, 1 one_skip,
 * 2 random_n, 3 last_n (SkipPolicy{kind, window, keep, seed}); kept_out and
 * start_out (nullable) hold up to n_items entries, *n_kept is set. */
FERRET_API ferret_status ferret_apply_skip_policy(size_t n_items, double t_d, int32_t kind, uint64_t window,
                                                  uint64_t keep, uint64_t seed, double processing_time,
                                                  int64_t* kept_out, double* start_out, size_t* n_kept);

/* ---------------- unit entry: the fused compensation kernel ---------------- */

/* One Compensator::apply (learner.hpp:97-120) on the device in fp64 with the reference's
 * operation order (bit-identical to the reference's host arithmetic; the trainer's own fused
 * update kernels compute in fp32): chain = chain_len parameter versions oldest first
 * (chain_len = tau + 1, any length),
 * state arrays updated in place (lambda/v_r/v_a for iter_fisher, mean_gap for gap;
 * NULL where the policy has none). lambda0 is the fisher policy's fixed lambda. */
FERRET_API ferret_status ferret_compensate(int32_t policy, const double* g, const double* const* chain,
                                int32_t chain_len, double* lambda, double* v_r, double* v_a,
                                double* mean_gap, size_t n, double lambda0, double alpha,
                                double eta_lambda, double nu, double* out);

/* ---------------- unit entry: one dense layer on the tensor cores ---------------- */

/* One dense layer on the tensor cores (tcgen05.mma, TMA-fed, TMEM accumulator),
 * host fp32 buffers in and out. precision FERRET_PREC_BF16 (W and X rounded to
 * bf16), FERRET_PREC_TF32 (tf32 operands) or FERRET_PREC_FP32 (3xTF32 split:
 * x = hi + lo per operand, hi*hi + hi*lo + lo*hi — about fp32 accuracy, the
 * parity mode's path for large layers); fp32 accumulation in every case.
 *   direction 0 — affine_forward + apply_activation (net.hpp:99-113):
 *       Y[b][r] = act(sum_c W[r][c] X[b][c] + bias[r]); X: B x in, Y: B x out; act = ReLU if relu
 *   direction 1 — the input gradient of learner.hpp:468-474:
 *       Y[b][c] = [mask[b][c] > 0] * sum_r W[r][c] X[b][r]; X: B x out, Y (and mask, nullable): B x in
 * W is out x in row-major; 1 <= B <= 16. */
FERRET_API ferret_status ferret_dense_layer(int32_t precision, int32_t direction, const float* W, const float* bias,
                                            const float* X, const float* mask, int32_t B, int32_t in, int32_t out,
                                            int32_t relu, float* Y);

/* One convolution (FERRET_LAYER_CONV geometry, 9 ints) on B samples, host
 * buffers in and out (unit checks of the conv kernels). tc: 0 SIMT fp32,
 * 1 tcgen05 tf32, 2 tcgen05 bf16, 3 tcgen05 3xTF32. mode 0 forward
 * Y = act(W * X + b + shortcut(res: B x rc x rh x rw)); mode 1 input gradient
 * Y = mask * (W^T * D + skip(res: the residual layer's delta, B x rc x rh x rw));
 * mode 2 weight gradient Y = D (x) im2col(X) (c_out x c_in*k*k). */
FERRET_API ferret_status ferret_conv_layer(int32_t tc, int32_t mode, const int32_t* geom, int32_t B, const float* W,
                                           const float* bias, const float* X, const float* D, const float* res,
                                           int32_t rc, int32_t rh, int32_t rw, const float* mask, int32_t relu,
                                           float* Y);

#ifdef __cplusplus
}
#endif

#endif /* FERRET_B200_H */
