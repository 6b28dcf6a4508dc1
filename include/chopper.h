/*
 * chopper.h -- C ABI of the B200-native Chopper analysis hot path.
 *
 * Chopper (arXiv 2512.08242) turns per-GPU kernel traces, serialized
 * hardware-counter passes and 1 ms frequency / power samples of an FSDP LLM
 * training run into multi-granularity attributions (kernel -> operation ->
 * layer -> phase -> iteration -> GPU) and the paper's
 * theoretical-vs-observed gap breakdown (Eqs. 4-8).
 * This library implements that analysis as hand-written sm_100a CUDA; the
 * readings of every silent / ambiguous point are DESIGN.md D1..D22.
 *
 * Conventions
 *  - All timestamps are int64 nanoseconds.  t_l = host dispatch, t_ks =
 *    device start, t_ke = device end.
 *  - Every pointer documented "device" must be device memory of `device`
 *    (e.g. a torch CUDA tensor); "host" pointers are host memory.
 *  - Input buffers are BORROWED: they must stay alive and unmodified until
 *    chopper_destroy (or the next chopper_load_columns).
 *  - The library never allocates device memory: all intermediates live in
 *    the caller's scratch buffer of chopper_scratch_bytes() bytes.
 *  - Every call enqueues work on the ctx stream: the library's own stream of
 *    the device's greatest priority, ordered after the caller's stream
 *    (chopper_create's cuda_stream) at the call's start, and the caller's
 *    stream ordered after the call's work at its end, so to the caller the
 *    work behaves as if it were enqueued on its stream.  Host-detectable errors
 *    (bad arguments, call order) are returned immediately; device-detected
 *    errors latch into a status mask read by chopper_status_sync().  Some
 *    calls synchronize the stream internally (documented per call).
 *  - Nothing throws across the ABI.  chopper_last_error() holds a message.
 *  - Calls must come in order: load_columns -> align -> attribute ->
 *    overlap -> breakdown -> reduce_ranks (align may be skipped when there
 *    are no counters and only one rank; otherwise CHOPPER_E_STATE).
 */
#ifndef CHOPPER_H
#define CHOPPER_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHOPPER_ABI_VERSION 8

typedef struct chopper_ctx chopper_ctx;
typedef int32_t chopper_status;

/* status codes; codes 1 and 3 mirror SPEC.md:544 exit codes */
enum {
    CHOPPER_OK = 0,
    CHOPPER_E_VALIDATION = 1,        /* input invariant violated */
    CHOPPER_E_INVALID_ARG = 2,
    CHOPPER_E_ALIGNMENT = 3,         /* counter pass name sequence mismatch / conflict */
    CHOPPER_E_AMBIGUOUS_SPANS = 4,   /* a dispatch falls where same-level spans cross */
    CHOPPER_E_RANGE = 5,             /* a size exceeds a configured bound */
    CHOPPER_E_INSUFFICIENT_DATA = 6,
    CHOPPER_E_CUDA = 7,
    CHOPPER_E_NCCL = 8,
    CHOPPER_E_STATE = 9              /* call out of order */
};

/* event kinds (low 8 bits of meta) */
enum { CK_COMPUTE = 0, CK_AG = 1, CK_RS = 2, CK_COMM_OTHER = 3, CK_COPY = 4, CK_MEMOP = 5, CK_OTHER = 6 };

/* validation rules, index into chopper_report.val_count / val_first */
enum {
    CV_START_AFTER_END = 0,     /* t_ks > t_ke                                          (fatal) */
    CV_GPU_NOT_GROUPED = 1,     /* events not grouped by gpu ascending                  (fatal) */
    CV_DISPATCH_DECREASING = 2, /* t_l decreases within a gpu                           (fatal) */
    CV_BAD_META = 3,            /* kind > 6, gpu >= n_traced_gpus, compute stream > 253 (fatal) */
    CV_TS_RANGE = 4,            /* max - min over all event timestamps >= 2^52          (fatal) */
    CV_STREAM_OVERLAP = 5,      /* same (gpu, compute stream) intervals overlap         (data)  */
    CV_SPAN_BAD = 6,            /* span end < start, level > 3, gpu >= n_traced_gpus     (fatal) */
    CV_SAMPLES_UNSORTED = 7,    /* samples not sorted by (gpu, ts) / bad gpu            (fatal) */
    CV_COUNTER_NONFINITE = 8,   /* a counter pass holds a non-finite value (pass skipped)       */
    CV_NRULES = 9
};

/* Kernel events, SoA, device.  Grouped by gpu ascending; within a gpu in
 * dispatch order (t_l non-decreasing; ties keep input order = correlation
 * order).  meta = (gpu << 24) | (stream << 8) | kind, stream dense
 * per gpu.  A rank passes only the traced GPUs it owns. */
typedef struct {
    int64_t n;
    const int64_t *dispatch_ns, *start_ns, *end_ns;
    const uint32_t *meta;
    const int32_t *name_id;
} chopper_events;

/* Annotation spans, SoA, device, any order.  gpu_level = (gpu << 8) | level,
 * level 0 iteration, 1 phase, 2 layer, 3 operation.  Half-open [start, end)
 * on the host (dispatch) timeline (D3).  label: iteration -> step number
 * (joins iterations across GPUs, D5); operation -> op label id
 * (0..n_labels-1); phase / layer -> free. */
typedef struct {
    int64_t n;
    const uint32_t *gpu_level;
    const int64_t *start_ns, *end_ns;
    const int32_t *label;
} chopper_spans;

/* 1 ms frequency / power samples, SoA, device, sorted by (gpu, ts).
 * Zero-order hold with extended ends (D10). */
typedef struct {
    int64_t n;
    const int32_t *gpu;
    const int64_t *ts_ns;
    const int32_t *freq_mhz, *power_mw;
} chopper_samples;

/* One serialized counter pass of one gpu: the name ids of
 * that gpu's non-MEMOP kernels in dispatch order (D2) and k counters per
 * kernel.  name_id, values: device; slot: host. */
typedef struct {
    int32_t gpu;
    int64_t n;
    const int32_t *name_id;     /* [n] */
    int32_t k;
    const int32_t *slot;        /* host [k]: counter slot in 0..n_counters-1 */
    const double *values;       /* [k][n] */
} chopper_counter_pass;

typedef struct {
    int32_t n_traced_gpus;      /* traced GPUs in the whole run (all ranks) */
    int32_t n_labels;           /* op label vocabulary size (identical on every rank) */
    int32_t max_iters;          /* bound on iteration rank (fixed exchange shapes) */
    int32_t max_coll_per_class; /* bound on AG (and RS) events per traced GPU */
} chopper_config;

/* Breakdown parameters.  Arrays are host memory. */
typedef struct {
    double tpt_peak;            /* TPT_peak, FLOP/s */
    double freq_peak_hz;        /* Freq_peak, Hz */
    int64_t batch, seq, ranks;  /* b, s, R: tokens per iteration = b*s*R */
    int32_t warmup;             /* iterations with rank < warmup are not sampled */
    int32_t slot_gpu_cycles, slot_perf_flops, slot_util_num, slot_util_den;  /* -1 = absent */
    const double *f_gemm;       /* [n_labels] theoretical FLOPs per point (Eq. 4) */
    const int32_t *op_type;     /* [n_labels] 1 gemm, 2 fa, 0 other */
    int32_t n_ratios;           /* derived ratio-of-sums rates */
    const int32_t *ratio_num;   /* [n_ratios] counter slot */
    const int32_t *ratio_den;   /* [n_ratios] counter slot, or -1 = busy seconds */
    const double *ratio_scale;  /* [n_ratios] */
} chopper_bd_params;

/* Row table (device SoA; pointers into ctx scratch; valid until the next
 * chopper_load_columns / chopper_destroy).  Columns are [n] unless noted. */
typedef struct {
    int64_t n;
    int64_t stride;                           /* column stride of counters / rates (>= n: the table capacity) */
    const int32_t *gpu, *it, *ph, *ly, *op;   /* caller span indices, -1 = none (unlabeled) */
    const int32_t *label;                     /* op label (points, instances), -1 otherwise */
    const int32_t *rank;                      /* iteration rank (iteration rows, points) else -1 */
    const int64_t *n_events, *n_compute, *busy, *first_ks, *first_idx, *first_pred, *last_ke;
    const int64_t *prep, *call, *ovl, *phi, *psi, *copy_ns, *ag_ns, *rs_ns;
    const double *counters;                   /* [n_counters][stride] */
    const double *rates;                      /* [n_ratios][stride] (points, iterations) or NULL */
    /* iteration rows only (else NULL) */
    const int64_t *wall, *comm_union, *aligned_first, *aligned_last;
    const int32_t *step;
    const double *metrics;                    /* [n_metrics][stride] registry values (points, iterations) or NULL */
} chopper_rows;

typedef struct {
    chopper_rows inst, layer, phase, iter, gpu, point;
    int64_t n_bd;                             /* local breakdown rows */
    int32_t n_metrics;                        /* derived-metric registry size (chopper_set_metrics) */
    const double *bd;                         /* device [n_bd][16], layout as chopper_global.bd */
} chopper_tables;

/* Host-visible global results (chopper_reduce_ranks). bd rows: 16 doubles:
 * 0 n_points, 1 method (0 bucket, 1 fit), 2 D_act s, 3 D0 s, 4 D50 s,
 * 5 D_thr, 6 Ovr_inst, 7 Ovr_util, 8 Ovr_overlap, 9 D_peak, 10 Ovr_freq,
 * 11 Ovr_launch, 12 residual, 13 Ovr_freq_samples, 14 flags, 15 label. */
typedef struct {
    int64_t n_iters;                          /* iterations of the reference gpu */
    int32_t step[4096], complete[4096], sampled[4096];
    int64_t T[4096], aligned_first[4096], aligned_last[4096];
    double throughput[4096];
    double throughput_median;
    int64_t n_bd;
    double bd[256 * 16];
    int64_t delta[256];                       /* clock offsets per traced gpu (D13) */
    int32_t delta_flag[256];
    int64_t max_skew_ag, max_skew_rs;
    /* report statistics per op label (O14): 16 doubles per label:
     * 0 n_points, 1-5 duration q0, q25, q50, q75, q100 (ns), 6-10 overlap ratio q0..q100,
     * 11 Pearson(overlap ratio, duration) (NaN if either is constant), 12 label, 13 mean duration (ns).
     * Quantiles interpolate linearly at h = q (n - 1) (R9). */
    int64_t n_report;
    double report[256 * 16];
    /* end-to-end phase x op-type breakdown (O16, Fig. 4; R12): e2e[0] = number
     * of (gpu, iteration) points; e2e[1 + 4 P + k], P = phase-span label 0..7, k = 0 vector / other,
     * 1 gemm, 2 fa (summed instance durations, ns), 3 launch overhead (prep + call, ns): medians over the
     * points (cells without instances count 0). */
    double e2e[1 + 8 * 4];
} chopper_global;

/* Device-side report read back by chopper_load_columns (host struct). */
typedef struct {
    int64_t val_count[CV_NRULES];
    int64_t val_first[CV_NRULES];             /* smallest offending index, -1 none */
    int64_t n_local_gpus;
    int32_t local_gpu[256];
    int64_t t_min, t_max;
    int32_t full_sort_used;                   /* 1: timestamp radix sort ran (groups not start-monotone) */
    int32_t non_laminar_lists;                /* (gpu, level) span lists needing the exact sweep path */
} chopper_report;

/* Scratch plan (SURVEY §7 hard part 5: 1B events on one B200).  The library never allocates device memory:
 * every intermediate lives in the caller's scratch arena, so the arena's size is planned from the trace's
 * shape.  Each item is an upper bound on the bytes the ctx keeps for it; total = persistent items + the
 * largest transient sort buffer + fixed slack.  The bounds that keep it near the real use are structural:
 * inside a gpu the events are dispatch-ordered and an event's instance key is a step function of its dispatch
 * time with steps only at that gpu's span endpoints, so instance runs (and instance rows) number at most
 * min(N, 2 S + N / 2048 + G + 1), and rows of a level above the operation at most 2 * (spans of the levels
 * above it) + G.  chopper_scratch_used reports the measured high-water mark to compare with.
 *   n_spans[4]: spans per level (iteration, phase, layer, operation) on this rank;
 *   n_comm: communication events (AG / RS / COMM_OTHER), -1 = unknown (n_events);
 *   n_local_gpus: traced GPUs with events on this rank, <= 0 = n_traced_gpus;
 *   max_compute_streams: per gpu, <= 0 = unknown (254): above 1 the general sort path and the explicit
 *     compute union are planned;
 *   laminar: 1 = no two same-level spans of a gpu cross (FSDP annotations), else the exact sweep's per-event
 *     table is planned.
 * items may be NULL.  Returns items->total. */
typedef struct {
    int64_t n_events;
    int64_t n_spans[4];
    int64_t n_samples;
    int64_t n_comm;
    int32_t n_counters;
    int32_t n_local_gpus;
    int32_t max_compute_streams;
    int32_t laminar;
} chopper_shape;
typedef struct {
    size_t events;       /* per-event columns the ctx keeps: permutation, chain ends, counter positions, ... */
    size_t spans;        /* push-ordered span table, Euler boundary tables, merged key table */
    size_t unions;       /* communication / compute unions, frequency-power timeline, sample prefixes */
    size_t subruns;      /* event-pass rows (one per instance run) and their counter sums */
    size_t instances;    /* instance table */
    size_t rollups;      /* layer, phase, iteration, gpu tables */
    size_t points;       /* (gpu, iteration, label) points */
    size_t exchange;     /* clock-offset and dense-row exchange blocks, breakdown / report work arrays */
    size_t transient;    /* the largest sort buffer (released after its stage) */
    size_t total;
} chopper_scratch_items;
size_t chopper_scratch_plan(const chopper_config *cfg, const chopper_shape *shape, chopper_scratch_items *items);

/* Worst-case scratch bytes knowing only the sizes: chopper_scratch_plan with every span counted at the
 * iteration level, n_comm = n_events, unknown stream count and laminarity. */
size_t chopper_scratch_bytes(const chopper_config *cfg, int64_t n_events, int64_t n_spans, int64_t n_samples,
                             int32_t n_counters);

/* nccl_comm: ncclComm_t of the process group (borrowed), NULL when nranks == 1 (or when a transport is
 * installed with chopper_set_allgather before chopper_align).
 * cuda_stream: cudaStream_t (borrowed), NULL = legacy default stream: every call is ordered after the work
 * already on it and before the work enqueued on it afterwards (the calls run on an internal stream of the
 * greatest priority, whose kernels the block scheduler places ahead of the library's side-stream work). */
chopper_status chopper_create(chopper_ctx **out, const chopper_config *cfg, int device, void *cuda_stream,
                              void *nccl_comm, int rank, int nranks, void *scratch, size_t scratch_bytes);

/* a1 pack + validate, a2 timestamp sort (stable by (gpu, group, t_ks), D1),
 * same-stream disjointness and the launch chain predecessor.
 * samples may be NULL.  Synchronizes the stream (reads the report). */
chopper_status chopper_load_columns(chopper_ctx *ctx, const chopper_events *ev, const chopper_spans *sp,
                                    const chopper_samples *smp);

/* a3 counter alignment and a4 clock offsets (D13; NCCL
 * all-gather #1 when nranks > 1).  counters_out: device [n_counters][n_events]
 * in input order, or NULL (tables-only).  offsets_ns: host [n_traced_gpus] or
 * NULL.  Synchronizes the stream. */
chopper_status chopper_align(chopper_ctx *ctx, const chopper_counter_pass *passes, int32_t n_passes,
                             int32_t n_counters, double *counters_out, int64_t *offsets_ns);

/* a5 interval-containment attribution.
 * span_idx: device [4][n_events] caller span index per level, -1 none,
 * -2 ambiguous (D4), or NULL.  Synchronizes the stream. */
chopper_status chopper_attribute(chopper_ctx *ctx, int32_t *span_idx);

/* a6 overlap (D9), a7 launch overhead Eqs. 1-3 (D6-D8), a8 DVFS integrals
 * (D10), fused with the time reductions of a9.  Each output is device [n]
 * or NULL: ovl (COMPUTE: |[t_ks,t_ke) ∩ comm union|; comm: |∩ compute
 * union|), prep, call, phi (MHz*ns), psi (mW*ns). */
chopper_status chopper_overlap(chopper_ctx *ctx, int64_t *ovl_ns, int64_t *prep_ns, int64_t *call_ns,
                               int64_t *phi, int64_t *psi);

/* a9 segmented reductions + roll-ups (instance -> layer -> phase -> iteration -> GPU, points summed across
 * layers) and a10 gap decomposition (Eqs. 4-8 plus the launch term,
 * PAPER.md:727-791; D14-D20) over this rank's points.  p: host parameters (read during the call).
 * Fills *out with device table pointers into the ctx scratch (valid until the next chopper_load_columns).
 * Errors: slot / ratio indices out of range -> CHOPPER_E_INVALID_ARG; iteration rank >= max_iters or op label
 * >= n_labels -> CHOPPER_E_RANGE (latched, reported by chopper_reduce_ranks).  Synchronizes. */
chopper_status chopper_breakdown(chopper_ctx *ctx, const chopper_bd_params *p, chopper_tables *out);

/* a11: all-gather #2 of the dense per-gpu rows (NCCL or the chopper_set_allgather transport), then the global
 * composition every rank computes in the same fixed order: per-iteration T = max over GPUs of busy + launch,
 * throughput b*s*R / T and its median over sampled iterations, the
 * breakdown over all GPUs' points, clock offsets and collective skew (D13), report
 * statistics.  out: host struct, overwritten.  Errors: more than 4096 iterations / 256 breakdown rows or
 * labels -> CHOPPER_E_RANGE; a peer rank failed earlier in the step -> CHOPPER_E_STATE.  Synchronizes. */
chopper_status chopper_reduce_ranks(chopper_ctx *ctx, chopper_global *out);

/* Per-GPU overlap CDFs of every op label (report statistics; Fig. 7;
 * SPEC.md:494-497; R11), from the results of chopper_reduce_ranks (call it after that call).
 * For each op label and traced gpu (ascending), the gpu's sampled points of the label (as in the breakdown)
 * sorted by duration (ties: iteration rank); rows of 5 doubles: label, gpu, duration / the gpu's minimum
 * duration, overlap ratio, empirical CDF (k + 1) / n.  out: host buffer of cap rows (may be NULL when cap is
 * 0); *n_rows = number of rows (the first min(cap, *n_rows) are written).  Synchronizes the ctx stream. */
chopper_status chopper_report_cdf(chopper_ctx *ctx, double *out, int64_t cap, int64_t *n_rows);

/* Chrome-trace ingest on the device (R15): the
 * step before chopper_load_columns.  json: DEVICE bytes of a Chrome-trace document ({"traceEvents": [...]});
 * device events = ph "X" with cat "kernel" or "gpu_*" (pid = gpu 0..255, tid = stream, args.correlation),
 * host launches = flow-start events (ph "s", id = correlation, ts = dispatch), spans = ph "X" with cat
 * "user_annotation" (pid = gpu, args.level 0..3, args.label); other events are ignored.  Times: decimal
 * microseconds -> integer ns rounded half to even; end = start + duration.  Kinds by the first matching
 * rule: cat gpu_memset -> MEMOP, gpu_memcpy -> COPY, other gpu_* -> OTHER; for cat kernel the lower-cased name
 * containing allgather / all_gather -> AG, reducescatter / reduce_scatter -> RS, nccl / rccl -> COMM_OTHER,
 * fsdp_copy -> COPY (D7), else COMPUTE.  name_id = order of first appearance of the (decoded) name among the
 * device events.  A kernel whose correlation has no launch gets dispatch = start (counted in n_missing).
 * Outputs (DEVICE, caller capacity ev_cap / span_cap): the chopper_events columns grouped by gpu and
 * dispatch-ordered (ties: file order), spans in file order.  scratch: caller device buffer of
 * chopper_ingest_scratch_bytes(n_bytes) (the ctx arena is not used; sized for event objects of >= 16 bytes,
 * a denser document returns CHOPPER_E_RANGE).  Errors: unbalanced JSON, no traceEvents
 * array or a malformed event object -> CHOPPER_E_VALIDATION (report.bad_offset = the object's byte offset);
 * output capacity or time range -> CHOPPER_E_RANGE.  Synchronizes the ctx stream. */
typedef struct {
    int64_t *t_l, *t_ks, *t_ke;
    uint32_t *meta;
    int32_t *name_id;
    int64_t ev_cap;
    uint32_t *span_gl;
    int64_t *span_start, *span_end;
    int32_t *span_label;
    int64_t span_cap;
} chopper_ingest_out;
typedef struct {
    int64_t n_objects, n_kernels, n_flows, n_spans, n_missing, n_names;
    int64_t bad_offset;            /* -1, or the byte offset of the first malformed event object */
} chopper_ingest_report;
size_t chopper_ingest_scratch_bytes(int64_t n_bytes);
chopper_status chopper_ingest_chrome(chopper_ctx *ctx, const char *json, int64_t n_bytes, void *scratch,
                                     size_t scratch_bytes, const chopper_ingest_out *out, chopper_ingest_report *rep);

/* Derived-metric registry ("calculating bandwidth from
 * transferred bytes and kernel duration"; R14).  exprs: n infix expressions (host strings) over
 * names[slot] (host strings: the counter slot names) and dur_s (the row's busy time, seconds): numbers,
 * identifiers, + - * /, parentheses, unary minus; * and / bind tighter than + and -, binary operators are
 * left-associative.  Compiled once on the host to postfix programs; every later chopper_breakdown evaluates
 * them on the device for each point and iteration row over the row's summed counters (chopper_rows.metrics,
 * [n][stride]).  A zero divisor, or a quotient that is not finite, gives NaN for that row (DivisionByZero).  Errors: an unknown name (MissingCounter) or a syntax
 * error (ParseError) -> CHOPPER_E_INVALID_ARG, *bad_expr = the failing index (-1 on success), the registry is
 * cleared; a name whose slot the trace lacks -> CHOPPER_E_INVALID_ARG at chopper_breakdown.  n = 0 clears. */
chopper_status chopper_set_metrics(chopper_ctx *ctx, int32_t n, const char *const *exprs, int32_t n_names,
                                   const char *const *names, int32_t *bad_expr);

/* CPU utilization (Sec. "CPU Utilization": C_active = sum_i [Util_i > 0],
 * C_min = sum_i Util_i / 100, logical -> physical cores; R13).
 * samples: n host-core utilisation samples, DEVICE pointers, sorted by (ts_ns, logical_core) with
 *   0 <= util_pct <= 100 and 0 <= logical_core < n_logical.  topology: DEVICE [n_logical] logical -> physical
 *   core id (>= 0).  Per distinct timestamp: C_active = #samples with util > 0, C_min = sum of util / 100 in
 *   logical-core order.  c_active / c_min: DEVICE outputs of cap entries (nullable; the first min(cap, n_ts)
 *   are written).  *out (host): timestamps, D21 medians and maxima of C_active and C_min, physical occupancy
 *   (#physical cores with an active logical core at any timestamp / #physical cores) and SMT co-activity
 *   (fraction of (timestamp, physical core) pairs with an active logical core that have two or more).
 * Borrowed inputs, scratch from the ctx arena (released before returning).  Unsorted or out-of-range samples
 * or a negative topology entry -> CHOPPER_E_VALIDATION (*out not written, per-timestamp outputs undefined).  Independent of the trace calls
 * (valid at any stage after chopper_create).  Synchronizes the ctx stream. */
typedef struct {
    int64_t n;
    const int64_t *ts_ns;
    const int32_t *logical_core;
    const double *util_pct;
} chopper_cpu_samples;
typedef struct {
    int64_t n_ts;
    int32_t n_logical, n_physical;
    double c_active_median, c_min_median, c_active_max, c_min_max;
    double physical_occupancy, smt_coactive;
} chopper_cpu_summary;
chopper_status chopper_cpu_util(chopper_ctx *ctx, const chopper_cpu_samples *samples, const int32_t *topology,
                                int32_t n_logical, int64_t *c_active, double *c_min, int64_t cap,
                                chopper_cpu_summary *out);

/* Cross-rank exchange transport.  By default the two exchange steps -- all-gather #1 of the
 * collective-end vectors inside chopper_align (clock offsets, D13) and all-gather #2 of the dense per-GPU row
 * blocks inside chopper_reduce_ranks (throughput takes the max over GPUs, the breakdown
 * medians pool all GPUs) -- are one ncclAllGather each on the ctx stream over the borrowed nccl_comm.
 * chopper_set_allgather replaces that call for this ctx: fn(user, send, recv, bytes_per_rank, rank, nranks,
 * cuda_stream) must leave in DEVICE recv[r * bytes_per_rank ...] the send block of rank r for every r, ordered
 * after the work already enqueued on cuda_stream, and return 0 (non-zero -> CHOPPER_E_NCCL).  fn = NULL restores
 * NCCL.  With a transport set, chopper_create's nccl_comm may be NULL for nranks > 1.
 *
 * Failure protocol (nranks > 1): every rank makes all six trace calls of a step in order, even after one of
 * them failed.  A call made after this rank's failure does no work and returns CHOPPER_E_STATE, but
 * chopper_align and chopper_reduce_ranks still take part in their all-gather with a block marked failed, so
 * no rank waits forever; a rank that receives such a block returns CHOPPER_E_STATE from that call ("a peer
 * rank failed"), and so do its later calls of the step.  chopper_load_columns starts a new step. */
typedef int32_t (*chopper_allgather_fn)(void *user, const void *send, void *recv, size_t bytes_per_rank,
                                        int32_t rank, int32_t nranks, void *cuda_stream);
chopper_status chopper_set_allgather(chopper_ctx *ctx, chopper_allgather_fn fn, void *user);

/* In-process loopback transport: nranks contexts on one device, each driven by its own host thread (tests
 * run P = 1/2/4/8 ranks on one GPU this way and require identical chopper_global results).  Pass
 * chopper_loopback_allgather and the group as chopper_set_allgather's fn / user.  The all-gather synchronizes
 * the caller's stream, waits until all nranks threads arrived (60 s limit -> returns non-zero), copies every
 * rank's send block device-to-device into recv, synchronizes again and waits for all ranks to finish copying.
 * create returns NULL for nranks outside 1..256; destroy frees the group (no thread may be inside it). */
void *chopper_loopback_create(int32_t nranks);
void chopper_loopback_destroy(void *group);
int32_t chopper_loopback_allgather(void *group, const void *send, void *recv, size_t bytes_per_rank, int32_t rank,
                                   int32_t nranks, void *cuda_stream);

/* report of the last chopper_load_columns (host copy) */
chopper_status chopper_get_report(const chopper_ctx *ctx, chopper_report *out);
/* synchronizes the ctx stream; returns the first latched error and fills the
 * latched mask (bit c set for each latched status code c) if mask != NULL */
chopper_status chopper_status_sync(chopper_ctx *ctx, uint32_t *mask);
const char *chopper_last_error(const chopper_ctx *ctx);
void chopper_destroy(chopper_ctx *ctx);

/* number of device kernels this ctx launched since creation (bench evidence) */
int64_t chopper_kernel_launches(const chopper_ctx *ctx);
/* number of host synchronizations with the ctx stream since creation (each waits for the queued work) */
int64_t chopper_host_syncs(const chopper_ctx *ctx);
int32_t chopper_abi_version(void);

/* introspection after chopper_align: first name-sequence divergence / first
 * conflicting value index of pass p (-1 none), and slot presence per gpu */
int64_t chopper_pass_mismatch(const chopper_ctx *ctx, int32_t p);
int64_t chopper_pass_conflict(const chopper_ctx *ctx, int32_t p);
int32_t chopper_counter_present(const chopper_ctx *ctx, int32_t gpu, int32_t slot);
/* high-water mark of the ctx's scratch arena since chopper_create (bytes) */
int64_t chopper_scratch_used(const chopper_ctx *ctx);

/* Device timing of pipeline phases with CUDA events recorded on the ctx
 * stream (off by default).  phase: 0 load, 1 align, 2 attribute,
 * 3 overlap prep, 4 event pass (its seed / window / head passes and the main kernel), 5 tables,
 * 6 breakdown, 7 reduce_ranks, 8 the main event-pass kernel alone (k_events_w / k_events), 9 the counter-pass kernel
 * alone (k_counters_tiled, on its side stream; counters only).  chopper_phase_time returns 0 and *ms for the most recent
 * run of that phase, CHOPPER_E_STATE if it was not timed. */
void chopper_set_timing(chopper_ctx *ctx, int32_t on);
chopper_status chopper_phase_time(chopper_ctx *ctx, int32_t phase, float *ms);

#ifdef __cplusplus
}
#endif
#endif
