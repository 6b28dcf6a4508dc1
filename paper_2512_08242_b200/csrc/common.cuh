// common.cuh -- internals of the B200 Chopper library (sm_100a only).
// Context, scratch arena, error latching, warp / block primitives shared by
// the kernels in this directory.  Nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <string>
#include <vector>

#include "../../include/chopper.h"

#define CH_MAX_GPUS 256
#define CH_NONE_TS INT64_MIN
#define CH_INVALID_KEY 0xFFFFFFFFFFFFFFFFull
#define CH_FULL 0xFFFFFFFFu

// ---------------------------------------------------------------------------
// device report (a1 validation + ranges), mirrored on the host
// ---------------------------------------------------------------------------
struct DevReport {
    unsigned long long val_count[CV_NRULES];
    unsigned long long val_first[CV_NRULES];    // ULLONG_MAX = none
    unsigned long long t_min_enc, t_max_enc;    // order-preserving encodings of int64
    unsigned long long s_min_enc, s_max_enc;    // spans start min / end max
    unsigned long long gbeg[CH_MAX_GPUS], gend[CH_MAX_GPUS];  // event ranges per traced gpu
    unsigned long long sbeg[CH_MAX_GPUS], send[CH_MAX_GPUS];  // sample ranges per traced gpu
    unsigned int max_stream[CH_MAX_GPUS];       // max compute stream id + 1 (0 = no compute)
    unsigned int n_comm[CH_MAX_GPUS];
    unsigned int flags;                         // bit0: non-monotone group in partition order
    unsigned int latched;                       // latched status mask (bit = status code)
    unsigned long long n_nonlaminar;
};

__host__ __device__ inline unsigned long long enc_i64(int64_t v) { return (unsigned long long)v ^ 0x8000000000000000ull; }
__host__ __device__ inline int64_t dec_i64(unsigned long long u) { return (int64_t)(u ^ 0x8000000000000000ull); }

// ---------------------------------------------------------------------------
// row tables (SoA, int64 field-major) -- see tables.cu
// ---------------------------------------------------------------------------
enum RowField {
    RF_NEV = 0, RF_N, RF_BUSY, RF_FIRST_IDX, RF_LAST_KE, RF_PREP, RF_CALL, RF_OVL, RF_PHI, RF_PSI, RF_COPY, RF_AG,
    RF_RS, RF_FIRST_KS, RF_NFIELDS
};

struct RowTable {
    int64_t cap = 0;
    int64_t n = 0;                  // host copy after count read-back
    int64_t *n_dev = nullptr;       // device count (kernels read it: no host round trip between stages)
    unsigned long long *key = nullptr;
    int64_t *first_event = nullptr;  // for sub-runs; row: first child
    int64_t *f = nullptr;            // [RF_NFIELDS][cap]
    double *cnt = nullptr;           // [C][cap]
    int32_t *gpu = nullptr, *it = nullptr, *ph = nullptr, *ly = nullptr, *op = nullptr, *label = nullptr,
            *rank = nullptr;         // decoded identity columns (outputs)
    int64_t *first_ks = nullptr, *first_pred = nullptr;
    double *rates = nullptr;
    double *metrics = nullptr;       // [n_metrics][cap] derived-metric registry values (points, iterations)
};

struct PassDesc {          // device copy of one counter pass
    const int32_t *name_id;
    const double *values;
    int64_t n;
    int32_t k;
    int32_t lg;
};

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct chopper_ctx {
    chopper_config cfg{};
    int device = 0;
    cudaStream_t st = nullptr;             // the library's own stream (greatest priority), joined to user_st per call
    cudaStream_t user_st = nullptr;        // the caller's stream (chopper_create)
    bool prep_deferred = false;            // chopper_attribute: the overlap preparation is still to be enqueued
    cudaEvent_t call_in = nullptr, call_out = nullptr;
    cudaStream_t side[3] = {nullptr, nullptr, nullptr};   // fork / join of independent small kernels
    cudaEvent_t fork_ev = nullptr, join_ev[3] = {nullptr, nullptr, nullptr};
    // span push-order sort enqueued on side[2] at the end of chopper_load_columns (spans.cu), so that it runs
    // beside chopper_align; chopper_attribute joins it.  Its buffers stay allocated for the step.
    cudaEvent_t span_fork = nullptr, span_join = nullptr;
    bool span_pending = false;       // the sort's kernels were enqueued on side[2] and are not joined yet
    bool span_launched = false;      // ch_span_sort_launch ran for this step (its buffers are allocated)
    // the union / sample / timeline preparation of chopper_overlap, enqueued on side[1] by chopper_attribute
    cudaEvent_t prep_join = nullptr;
    bool prep_done = false, prep_pending = false;
    struct SpanSort {
        unsigned long long *k1, *k2, *lb, *lb2;
        uint32_t *v1, *v2, *order;
        unsigned long long *okeys;
        unsigned int *big;
        int32_t *Plist;
        int rbits, lbits;
        int64_t smin, emax;
    } ss{};
    void *nccl = nullptr;
    int rank = 0, nranks = 1;
    chopper_allgather_fn ag_fn = nullptr;    // exchange transport (chopper_set_allgather), else NCCL
    void *ag_user = nullptr;
    // failure protocol (nranks > 1, chopper.h): first failure of this rank in the current step, 0 = none;
    // whether this step's all-gather #1 / #2 already happened (a failing call makes the missing one)
    chopper_status poison = CHOPPER_OK;
    bool x_exchanged = false, d_exchanged = false;
    int v_blocks = 0;                // k_validate_events grid: one wave of resident blocks on ctx->device
    size_t mark_base = 0;            // scratch offset after the report (poison exchanges allocate from here)
    char *scratch = nullptr;
    size_t scratch_bytes = 0, used = 0, high = 0;   // bump arena: bytes in use, high-water mark
    bool hold_scratch = false;       // inside a side-stream branch: temporaries are not released (see tables.cu)
    int64_t launches = 0;
    int64_t syncs = 0;               // host synchronizations with the ctx stream
    // pinned read-back ring: device->host copies of a stage land here asynchronously and are copied to
    // their destinations at the stage's ch_sync (a pageable destination would block the host per copy)
    unsigned char *h_pin = nullptr;
    size_t pin_cap = 0, pin_used = 0;
    struct PinCopy { void *dst; const void *src; size_t n; };
    std::vector<PinCopy> pin_pending;
    std::string err;
    int stage = 0;                 // 1 loaded, 2 aligned, 3 attributed, 4 overlapped, 5 breakdown
    bool loaded_ok = false;

    // borrowed inputs
    chopper_events ev{};
    chopper_spans sp{};
    chopper_samples smp{};
    bool has_smp = false;
    int64_t N = 0, S = 0, M = 0;

    // report
    chopper_report rep{};
    DevReport *d_rep = nullptr;
    DevReport h_rep{};

    // local gpus
    int n_lg = 0;
    int lg_gpu[CH_MAX_GPUS];
    int gpu_lg_h[CH_MAX_GPUS];
    int32_t *d_gpu_lg = nullptr;     // [256] gpu -> lg or -1
    int64_t g_beg[CH_MAX_GPUS + 1];  // input ranges per lg
    int max_stream = 0;              // max compute stream id + 1 over local gpus
    int NG = 0, n_buckets = 0;
    int64_t t0 = 0, t_max = 0;
    bool multi_stream = false;

    // a2 sort
    uint32_t *d_perm = nullptr;      // sorted position -> input index
    int64_t *d_bucket_beg = nullptr; // [n_buckets + 1]
    std::vector<int64_t> bucket_beg;
    int64_t *d_pred_end = nullptr;   // [N] end of chain predecessor or NONE
    bool full_sort = false;
    bool lean = false;               // one compute stream per gpu, start-monotone in dispatch order (lean a2)
    // lean a2's communication sort, checked late (load.cu ch_comm_sort_settle)
    bool ss_pending = false;
    unsigned int *d_ss_fail = nullptr, h_ss_fail = 0;
    uint32_t *d_ss_save = nullptr;
    std::vector<int64_t> ss_seg_lo, ss_seg_pre;
    int64_t ss_M = 0;
    int64_t *d_meta_tc = nullptr;    // [3][N / 2048] non-MEMOP / AG / RS tile counts from the lean a2 (align reuses)
    bool counters_early = false;     // the counter pass was launched beside the event pass (ch_event_pass)
    bool t_run_rank = false;         // d_t_run holds in-tile head ranks (k_tile_heads), not global run ids
    bool tables_radix = false;       // sticky: a trace of this ctx needed the radix instance sort (tables.cu)
    unsigned int *d_prefix_bad = nullptr;   // deferred instance-order check, read with the tables' row counts

    // spans (push order)
    int64_t S_loc = 0;               // spans of local gpus with positive length
    int64_t *P_start = nullptr, *P_end = nullptr;
    int32_t *P_orig = nullptr, *P_label = nullptr, *P_parent = nullptr;
    int64_t *d_list_beg = nullptr;   // [n_lg*4 + 2] push-order begin of each (lg, level) list
    std::vector<int64_t> list_beg;
    int32_t *d_list_flags = nullptr; // [n_lg*4] 1 = non-laminar
    std::vector<int32_t> list_flags;
    int32_t *d_attr_pre = nullptr;   // [4][N] precomputed (non-laminar lists)
    // Euler boundary tables (all lists laminar): per list, the time-ordered span endpoints with the innermost
    // owner after each one (rank + 1, 0 = none); list l occupies [2*list_beg[l] + l, 2*list_beg[l+1] + l + 1)
    int64_t *ET_t = nullptr;
    int32_t *ET_c = nullptr;
    int64_t *d_et_beg = nullptr;     // [n_lg*4 + 1]
    bool et_ok = false;
    // combined key table (et_ok): per lg, the four levels' Euler entries merged by time, each with the full
    // instance key after it; lg occupies [kt_beg[lg], kt_beg[lg+1]), entry 0 = (-inf, invalid)
    int64_t *KT_t = nullptr;
    unsigned long long *KT_k = nullptr;
    int64_t *d_kt_beg = nullptr;     // [n_lg + 1]
    // timeline (et_ok): per lg, comm-union boundaries and samples merged by time with the coverage and the
    // frequency / power prefix integrals as affine functions of (t - t0) after each entry
    int64_t *TL_t = nullptr;
    int64_t *TL_v = nullptr;         // [3][cap]: coverage, frequency and power intercepts
    int32_t *TL_s = nullptr;         // [3][cap]: in-union flag, f, p slopes
    int64_t *d_tl_beg = nullptr;     // [n_lg + 1] capacity layout
    int64_t *d_tl_len = nullptr;     // [n_lg] entries in use
    int64_t tl_cap = 0;
    int kb[4] = {0, 0, 0, 0};        // key bits per level
    int kg = 0;                      // key bits for lg
    int64_t max_it_list = 0;         // longest iteration-span list of a local gpu (iteration ranks < this)
    int64_t n_layer_spans = 0;       // layer spans of the local gpus (fan-out hint for the roll-ups)

    // samples
    int64_t *d_smp_phi = nullptr, *d_smp_psi = nullptr;  // prefix integrals at sample k
    int64_t *d_smp_lo = nullptr, *d_smp_hi = nullptr;    // [n_lg] sample ranges per lg
    std::vector<int64_t> smp_lo, smp_hi;

    // comm union per lg (merged intervals) and compute-union strategy
    int64_t *U_s = nullptr, *U_e = nullptr, *U_P = nullptr;
    int64_t *d_U_beg = nullptr, *d_U_cnt = nullptr;      // [n_lg]
    int64_t *V_s = nullptr, *V_e = nullptr, *V_P = nullptr;
    int64_t *d_V_beg = nullptr, *d_V_cnt = nullptr;      // [n_lg]
    uint32_t *d_vperm = nullptr;     // compute events sorted by (lg, t_ks) (multi-stream only)
    int v_general = 0;               // 1 = compute union built explicitly

    // sub-runs (a9 time part), produced by the fused event pass
    int64_t R = 0;
    RowTable sub;
    int64_t *d_tile_sub = nullptr;   // [ntile + 1] first sub-run id of each 2048-event tile (event pass)
    int32_t *d_t_run = nullptr;      // [ntile * 256] run id before each event-pass thread's first event
    uint8_t *d_t_hm = nullptr;       // [ntile * 256] that thread's head mask (the counter pass derives run ids)
    int32_t *d_t_nm = nullptr;       // [ntile * 256] non-MEMOP rank before each thread's first event (a3 positions)
    int64_t *d_nm_base = nullptr;    // [n_lg + 1] non-MEMOP rank of each local gpu's first event
    unsigned long long *d_tile_state = nullptr;
    unsigned int *d_tile_ticket = nullptr;

    // alignment
    int C = 0;
    std::vector<PassDesc> passes;
    PassDesc *d_passes = nullptr;
    int32_t *d_slot_pass = nullptr;  // [n_lg][C] pass index providing the slot, -1 absent
    int32_t *d_nm_rank = nullptr;    // [N] rank among non-MEMOP events of its gpu (full-mode counter output only)
    int64_t *d_mg = nullptr;         // [n_lg] non-MEMOP events per local gpu (counter column length)
    std::vector<int64_t> h_mg;
    std::vector<int32_t> h_pass_off, h_pass_idx;   // a3: passes grouped by local gpu (upload staging)
    std::vector<int32_t> h_lg_gpu;    // host staging of lg -> gpu (async copies read it)
    int64_t *d_delta = nullptr;      // [n_traced]
    int32_t *d_delta_flag = nullptr;
    std::vector<int64_t> delta;
    std::vector<int32_t> delta_flag;
    int64_t max_skew[2] = {0, 0};
    unsigned long long off_hs[2] = {0, 0};      // a4 read-back staging (ch_offsets_launch / _finish)
    unsigned int off_ovf = 0;
    std::vector<int64_t> off_hdr;
    bool off_pending = false;
    std::vector<int32_t> present;    // [n_lg][C]
    int32_t *d_present = nullptr;    // [n_lg][C]
    const double **d_col = nullptr;  // [n_lg][C] value column of the pass providing the slot
    std::vector<int64_t> pass_mismatch, pass_conflict;
    // counter-pass bookkeeping kept across calls (the caller's slot arrays are only valid in chopper_align)
    std::vector<std::vector<int32_t>> pass_slots;   // [n_passes][k]
    std::vector<int> pass_bad;                      // 1 = pass holds a non-finite value (known)
    std::vector<int> pass_covered;                  // 1 = every column feeds a slot: finiteness checked by
                                                    //     the counter pass in ch_tables, else k_pass_finite
    std::vector<int32_t> sel_pass;                  // [n_lg][C] pass providing the slot, -1 absent
    unsigned int *d_colbad = nullptr;               // [n_lg][C] non-finite value seen by the counter pass
    unsigned int *d_pass_bad = nullptr;             // [n_passes] k_pass_finite result (uncovered passes)
    unsigned long long *d_conf = nullptr;           // [n_passes] first conflicting position
    double *counters_out = nullptr;                 // full-mode [C][N] output (rewritten if slots change)
    const double **h_col_dev = nullptr;             // device array behind d_col (mutable)
    std::vector<int> gpu_present;    // [n_traced] gpu has events on some rank
    int64_t *d_xsend = nullptr;      // clock-offset exchange block of this rank [xslots][xW]
    unsigned int *d_xovf = nullptr;
    int64_t xW = 0;
    int xslots = 0;

    // tables
    RowTable inst, layer, phase, iter, gpurow, point;
    int64_t *iter_wall = nullptr, *iter_cu = nullptr, *iter_af = nullptr, *iter_al = nullptr;
    int32_t *iter_step = nullptr;
    double *d_bd = nullptr;
    int64_t n_bd = 0;
    chopper_bd_params bd{};
    std::vector<double> f_gemm;
    std::vector<int32_t> op_type;
    double *d_f_gemm = nullptr;
    int32_t *d_op_type = nullptr;
    int32_t *d_ratio = nullptr;      // [2][n_ratios]
    double *d_ratio_scale = nullptr;
    int n_ratios = 0;
    // derived-metric registry (metrics.cu): postfix programs, host copies
    int n_metrics = 0;
    std::vector<int32_t> met_ops, met_arg, met_beg;
    std::vector<double> met_const;
    int32_t *d_has_smp = nullptr;    // [n_lg]
    // phase timing (chopper_set_timing)
    bool timing = false;
    cudaEvent_t tev[10][2] = {};
    bool timed[10] = {};
    int64_t *d_dense = nullptr;      // local dense exchange blocks [dense_slots][W]
    unsigned int *d_dense_ovf = nullptr;
    int64_t *d_all = nullptr;        // all-gathered dense blocks (chopper_reduce_ranks), read by the report CDF
    int32_t *d_all_order = nullptr;
    int all_slots = 0;
    int dense_slots = 0;
    bool offsets_done = false;

    size_t mark_after_load = 0;
    uint32_t latched_host = 0;      // host-detected latched status bits
};

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
#define CH_CUDA(ctx, call)                                                                 \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            (ctx)->err = std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #call;     \
            (ctx)->pin_pending.clear();                                                    \
            return CHOPPER_E_CUDA;                                                         \
        }                                                                                  \
    } while (0)

#define CH_TRY(expr)                          \
    do {                                      \
        chopper_status s_ = (expr);           \
        if (s_ != CHOPPER_OK) return s_;      \
    } while (0)

// development aid (CHOPPER_DBG_HOST=1): host time from each stream synchronization's return to the next
// kernel launch -- the stretch in which the GPU idles waiting for the host -- attributed to that launch's line
struct HostProf {
    bool on = getenv("CHOPPER_DBG_HOST") != nullptr;
    bool armed = false;
    double t_sync = 0.0, t_wait = 0.0;
    std::vector<std::pair<std::string, double>> gaps;     // (launch site, gap us)
    std::vector<double> waits;                            // sync wait us
    static double now_us() {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    void launch(const char *f, int line) {
        if (!on || !armed) return;
        armed = false;
        const char *b = strrchr(f, '/');
        gaps.push_back({std::string(b ? b + 1 : f) + ":" + std::to_string(line), now_us() - t_sync});
    }
    void dump() {
        if (!on || gaps.empty()) return;
        double s = 0, w = 0;
        for (auto &g : gaps) s += g.second;
        for (double x : waits) w += x;
        fprintf(stderr, "[host] syncs %zu wait %.1f us, sync->launch gaps %.1f us:", waits.size(), w, s);
        for (auto &g : gaps) fprintf(stderr, " %s=%.1f", g.first.c_str(), g.second);
        fprintf(stderr, "\n");
        gaps.clear();
        waits.clear();
    }
};
extern HostProf g_hprof;
// development aid (CHOPPER_DBG_MARKS=1): device timestamps at marked points of the ctx stream, printed (deltas)
// at the next chopper_load_columns
struct DevMarks {
    bool on = getenv("CHOPPER_DBG_MARKS") != nullptr;
    cudaEvent_t ev[64] = {};
    const char *lab[64] = {};
    int n = 0;
    void mark(cudaStream_t st, const char *l) {
        if (!on || n >= 64) return;
        if (!ev[n]) cudaEventCreate(&ev[n]);
        cudaEventRecord(ev[n], st);
        lab[n++] = l;
    }
    void dump() {
        if (!on || n < 2) { n = 0; return; }
        cudaEventSynchronize(ev[n - 1]);
        fprintf(stderr, "[marks]");
        for (int i = 1; i < n; i++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, " %s %.3f", lab[i], ms);
        }
        fprintf(stderr, "\n");
        n = 0;
    }
};
extern DevMarks g_marks;

#define CH_LAUNCHED(ctx)                                                                   \
    do {                                                                                   \
        g_hprof.launch(__FILE__, __LINE__);                                                \
        (ctx)->launches++;                                                                 \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess) {                                                           \
            (ctx)->pin_pending.clear();                                                    \
            (ctx)->err = std::string("CUDA launch: ") + cudaGetErrorString(e_) + " @" +      \
                         std::to_string(__LINE__) + " " + __FILE__;                        \
            return CHOPPER_E_CUDA;                                                         \
        }                                                                                  \
    } while (0)

chopper_status ch_fail(chopper_ctx *ctx, chopper_status s, const std::string &msg);
chopper_status ch_prep_side(chopper_ctx *ctx);   // api.cu: chopper_overlap's preparation on side[1]
// host synchronization with the ctx stream (counted: chopper_host_syncs)
inline cudaError_t ch_sync(chopper_ctx *ctx) {
    ctx->syncs++;
    const double t_a = g_hprof.on ? HostProf::now_us() : 0.0;
    const cudaError_t e = cudaStreamSynchronize(ctx->st);
    if (g_hprof.on) {
        g_hprof.t_sync = HostProf::now_us();
        g_hprof.waits.push_back(g_hprof.t_sync - t_a);
        g_hprof.armed = true;
    }
    if (e == cudaSuccess)
        for (const auto &p : ctx->pin_pending) memcpy(p.dst, p.src, p.n);
    ctx->pin_pending.clear();
    ctx->pin_used = 0;
    return e;
}
// a pinned ring slot of n bytes (16 B aligned), or nullptr when the ring is full / absent
inline unsigned char *ch_pin_slot(chopper_ctx *ctx, size_t n) {
    const size_t a = (ctx->pin_used + 15) & ~(size_t)15;
    if (!ctx->h_pin || a + n > ctx->pin_cap) return nullptr;
    ctx->pin_used = a + n;
    return ctx->h_pin + a;
}
// device -> host copy on the ctx stream whose destination is valid after the next ch_sync (the caller
// reads it only after synchronizing, in the same scope for stack destinations)
inline cudaError_t ch_d2h(chopper_ctx *ctx, void *dst, const void *src, size_t n) {
    if (n == 0) return cudaSuccess;
    unsigned char *slot = ch_pin_slot(ctx, n);
    if (!slot) return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, ctx->st);   // pageable: blocking
    const cudaError_t e = cudaMemcpyAsync(slot, src, n, cudaMemcpyDeviceToHost, ctx->st);
    if (e == cudaSuccess) ctx->pin_pending.push_back({dst, slot, n});
    return e;
}
inline cudaError_t ch_d2h_2d(chopper_ctx *ctx, void *dst, size_t dpitch, const void *src, size_t spitch,
                             size_t width, size_t height) {
    if (width == 0 || height == 0) return cudaSuccess;
    unsigned char *slot = dpitch == width ? ch_pin_slot(ctx, width * height) : nullptr;
    if (!slot) return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, ctx->st);
    const cudaError_t e = cudaMemcpy2DAsync(slot, width, src, spitch, width, height, cudaMemcpyDeviceToHost, ctx->st);
    if (e == cudaSuccess) ctx->pin_pending.push_back({dst, slot, width * height});
    return e;
}
inline void ch_tick_on(chopper_ctx *ctx, int phase, int end, cudaStream_t st) {
    if (!ctx->timing) return;
    if (!ctx->tev[phase][end]) cudaEventCreate(&ctx->tev[phase][end]);
    cudaEventRecord(ctx->tev[phase][end], st);
    if (end) ctx->timed[phase] = true;
}
inline void ch_tick(chopper_ctx *ctx, int phase, int end) { ch_tick_on(ctx, phase, end, ctx->st); }
chopper_status ch_fill_u64(chopper_ctx *ctx, unsigned long long *p, int64_t n, unsigned long long v);

// ---------------------------------------------------------------------------
// scratch arena (256 B aligned bump allocator)
// ---------------------------------------------------------------------------
template <class T>
inline T *ch_alloc(chopper_ctx *ctx, int64_t n, chopper_status *st) {
    size_t bytes = (size_t)(n > 0 ? n : 1) * sizeof(T);
    size_t off = (ctx->used + 255) & ~(size_t)255;
    if (off + bytes > ctx->scratch_bytes) {
        if (*st == CHOPPER_OK) {
            *st = CHOPPER_E_RANGE;
            ctx->err = "scratch exhausted (need " + std::to_string(off + bytes) + " of " +
                       std::to_string(ctx->scratch_bytes) + " bytes)";
        }
        return nullptr;
    }
    ctx->used = off + bytes;
    if (ctx->used > ctx->high) ctx->high = ctx->used;
    return reinterpret_cast<T *>(ctx->scratch + off);
}
#define CH_ALLOC(ctx, T, n) ch_alloc<T>((ctx), (n), &st_)
#define CH_ALLOC_BEGIN chopper_status st_ = CHOPPER_OK
#define CH_ALLOC_END(ctx)            \
    do {                             \
        if (st_ != CHOPPER_OK) return st_; \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int bits_for(uint64_t v) {  // bits needed to represent values 0..v
    int b = 0;
    while (b < 64 && (v >> b) != 0) b++;
    return b;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int kind_of(uint32_t m) { return (int)(m & 0xFFu); }
__device__ __forceinline__ int stream_of(uint32_t m) { return (int)((m >> 8) & 0xFFFFu); }
__device__ __forceinline__ int gpu_of(uint32_t m) { return (int)(m >> 24); }
__device__ __forceinline__ bool is_comm(int k) { return k == CK_AG || k == CK_RS || k == CK_COMM_OTHER; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
// asynchronous global -> shared copies (cp.async, L2 -> SMEM without registers)
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// chain predecessor end (a7, D7/D8) of COMPUTE event i: the materialized column when the general a2 path built
// one, else -- the lean a2 path, one start-monotone compute stream per gpu -- the end of the previous COMPUTE event
// of the same gpu in dispatch order, found by walking back over the non-COMPUTE events in between
struct PredView {
    const int64_t *pred_end;     // [N] or NULL (lean)
    const uint32_t *meta;
    const int64_t *ke;
};
__device__ __forceinline__ int64_t pred_of(const PredView &v, int64_t i) {
    if (v.pred_end) return v.pred_end[i];
    const int g = (int)(__ldg(v.meta + i) >> 24);
    for (int64_t q = i - 1; q >= 0; q--) {
        const uint32_t m = __ldg(v.meta + q);
        if ((int)(m >> 24) != g) break;
        if ((m & 0xFFu) == CK_COMPUTE) return __ldg(v.ke + q);
    }
    return CH_NONE_TS;
}

// record a validation violation (count + smallest index)
__device__ __forceinline__ void viol(DevReport *r, int rule, int64_t idx) {
    atomicAdd(&r->val_count[rule], 1ull);
    atomicMin(&r->val_first[rule], (unsigned long long)idx);
}
__device__ __forceinline__ void latch(DevReport *r, int code) { atomicOr(&r->latched, 1u << code); }

// last index in [lo, hi) with a[idx] <= t, or lo - 1
__device__ __forceinline__ int64_t last_le(const int64_t *__restrict__ a, int64_t lo, int64_t hi, int64_t t) {
    int64_t l = lo, h = hi;
    while (l < h) {
        int64_t m = (l + h) >> 1;
        if (__ldg(a + m) <= t) l = m + 1; else h = m;
    }
    return l - 1;
}

// last_le by a whole warp (every lane calls it, every lane gets the answer): 32 probes per round, so a
// search over n entries takes about log32(n) dependent loads instead of log2(n)
__device__ __forceinline__ int64_t warp_last_le(const int64_t *__restrict__ a, int64_t lo, int64_t hi, int64_t t) {
    const int lane = threadIdx.x & 31;
    int64_t l = lo, h = hi;              // entries before l are <= t, entries from h on are > t
    while (h - l > 32) {
        const int64_t step = (h - l + 31) >> 5;
        const int64_t p = l + (int64_t)(lane + 1) * step - 1;
        const int c = __popc(__ballot_sync(0xFFFFFFFFu, p < h && __ldg(a + p) <= t));
        const int64_t nh = l + (int64_t)(c + 1) * step - 1;
        l += (int64_t)c * step;
        if (nh < h) h = nh;
    }
    const int64_t p = l + lane;
    return l + __popc(__ballot_sync(0xFFFFFFFFu, p < h && __ldg(a + p) <= t)) - 1;
}

// warp inclusive scan (sum) of int64
__device__ __forceinline__ int64_t warp_incl_sum(int64_t v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(CH_FULL, v, o);
        if (lane_id() >= o) v += y;
    }
    return v;
}
// block exclusive scan (sum) of int64 for blockDim.x <= 1024; returns total via *total
template <int NT>
__device__ __forceinline__ int64_t block_excl_sum(int64_t v, int64_t *total, int64_t *smem /*[32]*/) {
    int w = threadIdx.x >> 5, l = lane_id();
    int64_t inc = warp_incl_sum(v);
    if (l == 31) smem[w] = inc;
    __syncthreads();
    if (w == 0) {
        int64_t x = (l < NT / 32) ? smem[l] : 0;
        int64_t xi = warp_incl_sum(x);
        if (l < NT / 32) smem[l] = xi - x;
        if (l == NT / 32 - 1) smem[32] = xi;
    }
    __syncthreads();
    int64_t r = smem[w] + inc - v;
    if (total) *total = smem[32];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// cross-file host entry points
// ---------------------------------------------------------------------------
// prims.cu
// exclusive scan of NON-NEGATIVE int64 values (< 2^62: the single-pass tile states keep two flag bits on top)
chopper_status ch_scan_excl_i64(chopper_ctx *ctx, const int64_t *in, int64_t *out, int64_t n, int64_t *total_dev);
chopper_status ch_seg_scan_i64(chopper_ctx *ctx, const int64_t *in, const uint8_t *head, int64_t *out, int64_t n,
                               int op /*0 sum excl, 1 max incl, 2 sum incl*/);
chopper_status ch_radix_sort(chopper_ctx *ctx, unsigned long long *keys, uint32_t *vals, unsigned long long *keys_alt,
                             uint32_t *vals_alt, int64_t n, int bit_lo, int bit_hi, bool *result_in_alt);
chopper_status ch_radix_partition_meta(chopper_ctx *ctx, const uint32_t *meta, const int32_t *gpu_lg, int NG,
                                       int other_group, uint32_t *vals_out, int64_t n);
// load.cu
chopper_status ch_load(chopper_ctx *ctx);
// spans.cu
chopper_status ch_build_spans(chopper_ctx *ctx);
chopper_status ch_span_sort_launch(chopper_ctx *ctx);
chopper_status ch_comm_sort_settle(chopper_ctx *ctx);
chopper_status ch_counters_launch(chopper_ctx *ctx, double *cnt, unsigned int *colbad, int t_rank);
chopper_status ch_attr_pass(chopper_ctx *ctx, int32_t *span_idx);
// events.cu
chopper_status ch_overlap_prep(chopper_ctx *ctx);
chopper_status ch_event_pass(chopper_ctx *ctx, int64_t *ovl, int64_t *prep, int64_t *call, int64_t *phi, int64_t *psi);
// align.cu
chopper_status ch_align(chopper_ctx *ctx, const chopper_counter_pass *passes, int32_t n_passes, int32_t n_counters,
                        double *counters_out);
chopper_status ch_assign_slots(chopper_ctx *ctx);          // slot -> column from the passes' known state
chopper_status ch_counters_full(chopper_ctx *ctx);         // full-mode [C][N] counter matrix
chopper_status ch_offsets(chopper_ctx *ctx);
chopper_status ch_offsets_launch(chopper_ctx *ctx);
// tables.cu
chopper_status ch_tables(chopper_ctx *ctx);
// compose.cu
chopper_status ch_breakdown_local(chopper_ctx *ctx);
chopper_status ch_reduce_ranks(chopper_ctx *ctx, chopper_global *out);
chopper_status ch_report_cdf(chopper_ctx *ctx, double *out, int64_t cap, int64_t *n_rows);
size_t ch_ingest_scratch_bytes(int64_t n_bytes);
chopper_status ch_ingest_chrome(chopper_ctx *ctx, const char *js, int64_t L, void *scratch, size_t scratch_bytes,
                                const chopper_ingest_out *out, chopper_ingest_report *rep);
chopper_status ch_compile_metrics(chopper_ctx *ctx, int32_t n, const char *const *exprs, int32_t n_names,
                                  const char *const *names, int32_t *bad_expr);
chopper_status ch_eval_metrics(chopper_ctx *ctx, RowTable &t);
chopper_status ch_cpu_util(chopper_ctx *ctx, const chopper_cpu_samples *s, const int32_t *topology, int32_t n_logical,
                           int64_t *c_active, double *c_min, int64_t cap, chopper_cpu_summary *out);
chopper_status ch_nccl_allgather(chopper_ctx *ctx, const void *send, void *recv, size_t bytes_per_rank);
// failure protocol: this rank's side of exchange #which (1 offsets, 2 dense rows) as a block marked failed
chopper_status ch_exchange_poison(chopper_ctx *ctx, int which);
int64_t ch_dense_width(chopper_ctx *ctx);        // int64 words per dense slot (compose.cu)

// lookup of an event's innermost span per level (spans.cu; used by events.cu)
struct SpanView {
    const int64_t *P_start, *P_end;
    const int32_t *P_parent;
    const int64_t *list_beg;     // [n_lg*4 + 1]
    const int32_t *list_flags;   // non-laminar lists
    const int32_t *attr_pre;     // [4][N] for non-laminar lists
    int64_t N;
};

// innermost span (push-order global index) containing t in list (lg, lv), -1 none, -2 ambiguous
__device__ __forceinline__ int64_t span_lookup(const SpanView &v, int lg, int lv, int64_t t, int64_t i, int64_t *cursor) {
    int list = lg * 4 + lv;
    if (v.list_flags[list]) {
        int32_t a = v.attr_pre[(int64_t)lv * v.N + i];
        return a;   // already a push-order global index, -1 or -2
    }
    int64_t lb = v.list_beg[list], le = v.list_beg[list + 1];
    if (le <= lb) return -1;
    int64_t c = *cursor;
    // seeded search: walk forward a few steps from the previous answer, else binary search
    if (c >= lb - 1 && c < le && (c < lb || __ldg(v.P_start + c) <= t)) {
        int steps = 0;
        while (c + 1 < le && __ldg(v.P_start + c + 1) <= t && steps < 8) { c++; steps++; }
        if (c + 1 < le && __ldg(v.P_start + c + 1) <= t) c = last_le(v.P_start, c + 1, le, t);
    } else {
        c = last_le(v.P_start, lb, le, t);
    }
    *cursor = c;
    while (c >= lb && __ldg(v.P_end + c) <= t) c = __ldg(v.P_parent + c);
    return c >= lb ? c : -1;
}
