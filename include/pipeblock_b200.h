/*
 * pipeblock_b200.h — C-ABI boundary of the B200-native V-shape pipeline executor.
 *
 * The reference ("pipeblock", /root/reference/proj/include/pipeblock) is a C++
 * schedule synthesizer.  Its front end (build_entry -> assemble -> GridSchedule,
 * or parse(json) -> ScheduleDocument) stays the producer of the per-device op
 * order.  This header is what that front end (or any FFI: ctypes, cgo, JNI)
 * binds to hand a schedule to CUDA and get a measured TimedSchedule back — the
 * real-hardware counterpart of simulate() (simulate.hpp:22).
 *
 * Conventions: plain C types only; devices and stages are 1-based exactly as in
 * the reference; every function returns PB_OK (0) or a negative PB_E* code and
 * sets a thread-local message readable with pb_last_error().  The caller owns
 * every input array (the library copies what it keeps) and allocates every
 * output array.
 */
#ifndef PIPEBLOCK_B200_H
#define PIPEBLOCK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PB_ABI_VERSION 1

enum {
    PB_OK = 0,
    PB_EINVAL = -1,   /* std::invalid_argument in the reference (model.hpp:223, assemble.hpp:86-89,206,408-414) */
    PB_EDOC = -2,     /* DocumentError (document.hpp:13-16) */
    PB_ECUDA = -3,    /* CUDA / driver failure, or no sm_100 device */
    PB_ESPACE = -4,   /* caller-provided output buffer too small */
    PB_ESTATE = -5    /* handle used out of order (e.g. step before connect) */
};

/* PassKind (model.hpp:15): F=0, B=1, W=2, BW=3 (fused backward, two cells). */
enum { PB_F = 0, PB_B = 1, PB_W = 2, PB_BW = 3 };

/* GridPass (model.hpp:162-176, ScheduledPassT<long long>). */
typedef struct pb_pass {
    int32_t device;
    int32_t stage;
    int32_t kind;
    int32_t microbatch;
    int64_t start;
    int64_t duration;
} pb_pass;

/* TimedPass (model.hpp:176, ScheduledPassT<double>); times in milliseconds when
 * produced by the executor, in profile units when produced by pb_simulate. */
typedef struct pb_timed_pass {
    int32_t device;
    int32_t stage;
    int32_t kind;
    int32_t microbatch;
    double start;
    double duration;
} pb_timed_pass;

/* Topology (model.hpp:50-56), single default route 1..num_stages. */
typedef struct pb_topology {
    int32_t devices;
    int32_t num_stages;
    const int32_t* placement; /* num_stages entries, placement[s-1] = device of stage s */
    const double* stage_mem;  /* num_stages entries; NULL = all 1.0 */
} pb_topology;

/* RunTimeProfile (model.hpp:189-206). */
typedef struct pb_profile {
    double f, b, w, comm;
} pb_profile;

/* SimResult scalars (simulate.hpp:9-17); per-device vectors go to caller arrays. */
typedef struct pb_sim_stats {
    double makespan;
    double bubble_rate;
} pb_sim_stats;

const char* pb_last_error(void);
int pb_abi_version(void);

/* ------------------------------------------------------------------ schedules
 * An immutable, validated GridSchedule.  Shareable across threads. */
typedef struct pb_schedule pb_schedule;

/* assemble(build_entry(entry, devices), microbatches, {squeeze, reorder})
 *   replaces gallery.hpp:499 build_entry + assemble.hpp:405 assemble. */
int pb_schedule_build(const char* entry, int32_t devices, int32_t microbatches, int32_t do_squeeze,
                      int32_t do_reorder, pb_schedule** out);
/* build_entry(entry, d) alone (gallery.hpp:499-557): validates the entry / device count and reports the
 * block's microbatches per block (assemble needs a multiple of it) and whether it needs replicated
 * weights (gems, chimera: generated and analysed, not executable). */
int pb_build_info(const char* entry, int32_t devices, int32_t* microbatches_per_block, int32_t* replicated_weights);
/* A caller-made GridSchedule (e.g. converted from pipeblock::GridSchedule);
 * validated like validate_schedule (assemble.hpp:138-183). */
int pb_schedule_create(const pb_topology* topo, const pb_pass* passes, size_t n, int32_t microbatches,
                       pb_schedule** out);
/* parse(text, strict) (document.hpp:192); units must be "cells". */
int pb_schedule_parse(const char* json_text, int32_t strict, pb_schedule** out);
/* emit(document) (document.hpp:188): writes up to cap bytes incl. NUL; *len = bytes needed excl. NUL. */
int pb_schedule_emit(const pb_schedule* s, char* buf, size_t cap, size_t* len);
int pb_schedule_info(const pb_schedule* s, int32_t* devices, int32_t* num_stages, int32_t* microbatches,
                     size_t* num_passes);
int pb_schedule_topology(const pb_schedule* s, int32_t* placement, double* stage_mem);
/* Passes in canonical (device, start, stage, microbatch) order (assemble.hpp:50-57). */
int pb_schedule_passes(const pb_schedule* s, pb_pass* out, size_t n);
/* exact_peak (memory.hpp:63-91): one value per device. */
int pb_schedule_exact_peak(const pb_schedule* s, double* per_device);
/* simulate (simulate.hpp:22-86). out: n passes (canonical order) or NULL; per-device arrays may be NULL. */
int pb_simulate(const pb_schedule* s, const pb_profile* prof, pb_timed_pass* out, size_t n, pb_sim_stats* stats,
                double* busy, double* idle_total, double* idle_span, double* peak);
/* simulate() with one duration per pass (canonical order, n = pass count) and a
 * per-crossing latency `comm`: replays measured pass times in grid order. */
int pb_replay(const pb_schedule* s, const double* durations, size_t n, double comm, pb_timed_pass* out,
              pb_sim_stats* stats, double* busy, double* idle_total, double* idle_span, double* peak);
/* The same accounting over measured passes (bubble = 1 - sum busy / (d * makespan), simulate.hpp:81-82). */
int pb_account(const pb_topology* topo, const pb_timed_pass* passes, size_t n, pb_sim_stats* stats, double* busy,
               double* peak);
void pb_schedule_destroy(pb_schedule* s);

/* ------------------------------------------------------------------ analysis
 * Stable-phase growth of the schedule's building block (growth.hpp), the
 * adaptive V-family search (search.hpp) and Gantt rendering (render.hpp).
 * Growth needs a schedule that carries its block (built by pb_schedule_build
 * or pb_search, or parsed from a document with a "block"). */
typedef struct pb_growth_report { /* GrowthReport (growth.hpp:13-22) */
    int32_t cycle_length;
    double growth;           /* time gained per period */
    double max_work;
    double repeating_bubble; /* max(0, growth - max_work) */
    int32_t linear_bubble;   /* O(n) bubble */
    int32_t tie;
} pb_growth_report;
/* growth_rate (growth.hpp:141-187).  work: `devices` entries or NULL; witness:
 * the maximal chain, one "F(stage s, slot k)@periodP" per line (len = bytes needed). */
int pb_growth_rate(const pb_schedule* s, const pb_profile* prof, pb_growth_report* out, double* work, char* witness,
                   size_t cap, size_t* len);
int pb_growth_rate_unrolled(const pb_schedule* s, const pb_profile* prof, int32_t periods, double* out); /* :132 */
int pb_vhalf_condition(const pb_profile* prof, int32_t* out);                                           /* :190 */
int pb_lower_bound(int64_t n, int64_t d, int64_t k, int64_t* out);                                      /* :195 */
int pb_min_memory_for_od_bubble(int32_t d, double* out);                                                /* :202 */

typedef struct pb_search_spec { /* SearchSpec (search.hpp:15-25) */
    int32_t devices;
    int32_t microbatches; /* 0 = 3 * devices */
    pb_profile profile;
    double memory_limit; /* units of m */
    int64_t delta_max, tau_max;
} pb_search_spec;
typedef struct pb_search_params { /* SearchParams (search.hpp:27-42) */
    int32_t K;
    int64_t d0_lo, d1_lo, d0_hi, d1_hi, tau1, tau2, tau3;
} pb_search_params;
typedef struct pb_search_result { /* SearchResult scalars (search.hpp:44-56) */
    int32_t feasible;
    pb_search_params best;
    double bubble_rate, exact_peak;
    int64_t enumerated, evaluated;
    double family_min_peak;
    int32_t turn_devices_exercised;
} pb_search_result;
typedef struct pb_frontier_point { /* FrontierPoint (search.hpp:58-64) */
    double limit;
    int32_t feasible;
    double bubble_rate, exact_peak;
    pb_search_params best;
} pb_frontier_point;
/* search (search.hpp:235).  message: the infeasibility text ("" when feasible).
 * schedule (optional): the winner assembled at spec->microbatches, executable by
 * pb_exec_create unchanged; NULL when infeasible. */
int pb_search(const pb_search_spec* spec, pb_search_result* out, char* message, size_t cap, size_t* len,
              pb_schedule** schedule);
/* The family block of one parameter tuple (e.g. a pb_search winner, search.hpp:208-216 rebuild)
 * assembled at `microbatches` (squeeze + reorder), validated like validate_block + residue check:
 * runs on the executor at the step's own microbatch count. */
int pb_search_assemble(int32_t devices, const pb_search_params* params, int32_t microbatches, pb_schedule** out);
int pb_frontier(const pb_search_spec* spec, const double* limits, size_t n, pb_frontier_point* out); /* :240 */

enum { PB_RENDER_SVG = 0, PB_RENDER_ASCII = 1 };
/* render_svg / render_ascii (render.hpp:83,177) of the schedule's document. */
int pb_render(const pb_schedule* s, int32_t format, const char* title, int32_t ascii_max_width, int32_t ascii_color,
              char* buf, size_t cap, size_t* len);
/* A measured timeline as a "time" ScheduleDocument (document_from_timed, document.hpp:413), emitted as JSON or rendered. */
int pb_timed_emit(const pb_topology* topo, const pb_timed_pass* passes, size_t n, int32_t microbatches, char* buf,
                  size_t cap, size_t* len);
int pb_timed_render(const pb_topology* topo, const pb_timed_pass* passes, size_t n, int32_t microbatches,
                    int32_t format, const char* title, int32_t ascii_max_width, char* buf, size_t cap, size_t* len);

/* ------------------------------------------------------------------ executor
 * GPT-style decoder stack (pre-norm RMSNorm, causal MHA with head_dim 128,
 * GELU MLP 4h, residual, untied embedding / LM head, mean cross-entropy),
 * split into num_stages equal chunks of layers.  Stage 1 also holds the token
 * embedding; the last stage holds the final norm, LM head and loss.  bf16
 * weights/activations, fp32 accumulation, fp32 gradients, AdamW in fp32. */
typedef struct pb_model_cfg {
    int32_t layers;
    int32_t hidden;
    int32_t heads;
    int32_t seq;
    int32_t vocab;
    int32_t micro_batch; /* sequences per microbatch */
    uint64_t seed;
    float lr, beta1, beta2, eps, weight_decay;
    int32_t optimizer; /* 1 = AdamW step after the flush, 0 = gradients only */
    int32_t flags;     /* PB_FLAG_* */
    /* NULL: layers / num_stages per stage.  Else num_stages entries >= 1 summing to `layers`
     * (e.g. fewer layers on the stages that also carry the embedding / LM head; the
     * schedule is unchanged, only the work per pass).  Copied at pb_exec_create. */
    const int32_t* stage_layers;
} pb_model_cfg;

#define PB_FLAG_SERIAL 1     /* device-synchronise after every pass (race check mode) */
#define PB_FLAG_TIMELINE 2   /* record per-pass CUDA events (TimedSchedule output) */
#define PB_FLAG_GEMM_TIMING 4 /* CUDA events around every GEMM launch (roofline of the dominant kernel) */
#define PB_FLAG_KERNEL_TIMING 8 /* CUDA events around every launch, per-kernel report (pb_exec_kernel_report) */
#define PB_FLAG_SOLO 32      /* run this device's op list alone (no peers connected): cross-device inputs
                                are not pulled (the receive slot keeps its contents) and outputs are not
                                signalled.  Real kernels, real op order, real memory footprint — for
                                memory / per-pass timing probes of one device of a p-device pipeline */
#define PB_FLAG_ISOLATE 16   /* in-process group: one pass at a time over all devices (a group-wide GPU
                                token taken after the pass's cross-device waits), each synchronised —
                                clean stand-alone per-pass times for pb_replay */

typedef struct pb_exec_stats {
    double loss;            /* mean CE over all tokens of the step (last-stage device; NaN elsewhere) */
    double step_ms;         /* this device: CUDA events from the start of the step's enqueue (before the
                               token / label copies) to its end (after the gamma fold, AdamW and the loss
                               D2H), i.e. the whole step on this device's compute stream */
    double busy_ms;         /* this device: sum of pass durations */
    int64_t pool_slots;     /* activation slots allocated = predicted exact_peak on this device */
    int64_t pool_peak;      /* slots live at once over the op order as enqueued (a host-side count, not a
                               device measurement; device bytes come from pb_exec_memory) */
    int64_t slot_bytes;     /* bytes per activation slot */
    int64_t pool_bytes;     /* slot_bytes * pool_slots + the LM-head pool (head slot bytes * head slots,
                               last-stage device only: final-norm output and logits) */
    int64_t peer_bytes;     /* bytes pulled from peers during the step */
    int64_t kernel_launches;/* kernels this device launched during the step */
    double gemm_ms;         /* PB_FLAG_GEMM_TIMING: summed GEMM launch durations (CUDA events, compute stream) */
    double gemm_flops;      /* algorithmic FLOPs of those GEMMs (2*M*N*K each) */
    int64_t gemm_launches;
    double copy_ms;         /* summed durations of this device's stage-boundary pulls (CUDA events on the
                               copy stream); peer_bytes / copy_ms = achieved transfer bandwidth */
} pb_exec_stats;

typedef struct pb_exec pb_exec;

/* One pipeline device (1-based `device` of the schedule's topology) bound to
 * CUDA ordinal `cuda_device`.  Allocates weights (seeded init), gradients,
 * optimizer state and the lifespan-bounded activation pool. */
int pb_exec_create(const pb_model_cfg* cfg, const pb_schedule* plan, int32_t device, int32_t cuda_device,
                   pb_exec** out);
/* Peer wiring.  Same process: pass the peer handles directly.  Separate
 * processes: export an IPC blob, exchange blobs (e.g. torch.distributed
 * all_gather_object), then connect with all devices' blobs in device order. */
int pb_exec_connect_local(pb_exec* const* all_devices, int32_t n);
int pb_exec_export(pb_exec* e, void* blob, size_t cap, size_t* len);
int pb_exec_connect_ipc(pb_exec* e, const void* const* blobs, const size_t* lens, int32_t n);
/* One training step: every pass of this device in grid order, then the
 * optimizer.  tokens/labels: micro_batch*seq*microbatches int32 each,
 * microbatch-major; host pointers when inputs_on_host != 0 (copied in on the
 * compute stream inside the step), else device pointers.  Only stage-1's
 * device reads tokens and only the last stage's device reads labels.
 * Ids must lie in [0, vocab).  Host inputs are checked before anything is
 * enqueued by every device that is given the arrays (pass the same arrays to
 * every device of a group so they fail together): PB_EINVAL.  Device inputs
 * are checked by the kernels that index with them (the row is skipped, never
 * read or written out of bounds) and the step's sync returns PB_EINVAL.
 * timeline: NULL or an array of this device's pass count (canonical order). */
int pb_exec_step(pb_exec* e, const int32_t* tokens, const int32_t* labels, int32_t inputs_on_host,
                 pb_timed_pass* timeline, size_t timeline_n, pb_exec_stats* stats);
/* JSON {"label": [ms, launches], ...} of the last PB_FLAG_KERNEL_TIMING step. */
int pb_exec_kernel_report(pb_exec* e, char* buf, size_t cap, size_t* len);
/* Enqueue-only variant for CUDA-event timing by the caller: no host sync. */
int pb_exec_step_async(pb_exec* e, const int32_t* tokens, const int32_t* labels, int32_t inputs_on_host);
int pb_exec_sync(pb_exec* e, pb_timed_pass* timeline, size_t timeline_n, pb_exec_stats* stats);
int pb_exec_num_passes(const pb_exec* e, size_t* n);
/* Change PB_FLAG_* between steps (e.g. one GEMM-timed step for the roofline). */
int pb_exec_set_flags(pb_exec* e, int32_t flags);
void* pb_exec_stream(pb_exec* e); /* cudaStream_t of the compute stream */
/* Parameter access for parity tests: tensors are enumerated per stage owned
 * by this device; names like "s3.l1.wqkv", "s1.emb", "s8.head", "s8.norm". */
int pb_exec_param_count(const pb_exec* e, int32_t* n);
int pb_exec_param_info(const pb_exec* e, int32_t i, char* name, size_t cap, int64_t* numel);
int pb_exec_param_get(pb_exec* e, int32_t i, int32_t which /*0 weight bf16->f32, 1 grad f32*/, float* host);
int pb_exec_param_set(pb_exec* e, int32_t i, const float* host); /* rounds to bf16, sets fp32 master */
int pb_exec_zero_grads(pb_exec* e);

/* Device memory of one executor.  The executor allocates everything at pb_exec_create (no
 * allocation inside a step apart from the W-pass GEMM tables of the first step), so
 * device_used_high (cudaMemGetInfo total - free, sampled after creation, after every
 * synchronised step and at this call; whole device, all contexts) is the high-water mark. */
typedef struct pb_exec_memory_t {
    int64_t weights;          /* fp32 masters + bf16 compute copies */
    int64_t grads;            /* fp32 gradients (+ the gamma-folded projection gradient buffer) */
    int64_t optimizer;        /* AdamW first / second moments */
    int64_t activation_pool;  /* lifespan pool: slot_bytes * exact_peak slots */
    int64_t head_pool;        /* LM-head pool (final-norm output, logits), last-stage device */
    int64_t transfer;         /* outbox slots + flag words of the stage-boundary protocol */
    int64_t scratch;          /* attention / GEMM scratch, step inputs, loss */
    int64_t executor_total;   /* every cudaMalloc of this executor (sum of the above) */
    int64_t device_total;     /* cudaMemGetInfo total */
    int64_t device_used_at_create; /* total - free just before this executor allocated */
    int64_t device_used_high; /* max sampled total - free */
} pb_exec_memory_t;
int pb_exec_memory(pb_exec* e, pb_exec_memory_t* out);

/* The host-side execution plan of one pipeline device — a pure function of the
 * schedule, so every rank derives its peers' outbox layout without talking
 * (csrc/exec/plan.hpp).  Needs no GPU. */
typedef struct pb_plan_op {
    int32_t stage, kind, microbatch;
    int32_t slot;        /* activation-pool slot of (stage, microbatch) on this device */
    int64_t start;       /* grid cell */
    int32_t recv_from;   /* 0, or the device whose outbox this op pulls its input from */
    int32_t recv_outbox; /* outbox slot on recv_from */
    uint32_t recv_gen;   /* generation of that outbox slot within the step */
    int32_t send_to;     /* 0, or the device that consumes this op's output */
    int32_t send_outbox; /* outbox slot on this device */
    uint32_t send_gen;
} pb_plan_op;
/* Passes of `device` in grid order; *slots = activation slots (= exact_peak), *outboxes = outbox slots. */
int pb_plan_device(const pb_schedule* s, int32_t device, pb_plan_op* out, size_t cap, size_t* n, int32_t* slots,
                   int32_t* outboxes);
void pb_exec_destroy(pb_exec* e);

#ifdef __cplusplus
}
#endif
#endif /* PIPEBLOCK_B200_H */
