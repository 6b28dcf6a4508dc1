// api.cu -- the C ABI (include/chopper.h): argument checks, call order,
// status latching.  Every compute step runs in the kernels of this directory.
#include "common.cuh"

#include <chrono>
#include <condition_variable>
#include <mutex>

chopper_status ch_fail(chopper_ctx *ctx, chopper_status s, const std::string &msg) {
    ctx->pin_pending.clear();            // read-backs of the failed stage are dropped (stack destinations)
    ctx->err = msg;
    ctx->latched_host |= 1u << s;
    return s;
}

// failure protocol (chopper.h): remember this rank's first failure of the step (several ranks only)
static chopper_status step(chopper_ctx *ctx, chopper_status s) {
    g_marks.mark(ctx->st, "call_end");
    if (s != CHOPPER_OK) ctx->pin_pending.clear();
    if (s != CHOPPER_OK && ctx->nranks > 1 && ctx->poison == CHOPPER_OK) ctx->poison = s;
    return s;
}
// a call made after this rank's failure: no work, E_STATE (keeps the first error's message)
static chopper_status dead_call(chopper_ctx *ctx) {
    ctx->latched_host |= 1u << CHOPPER_E_STATE;
    if (ctx->err.empty()) ctx->err = "call after a failed call of this step";
    return CHOPPER_E_STATE;
}

// in-process loopback transport (chopper_loopback_*): a generation barrier over the group's threads
namespace {
struct LoopGroup {
    int n = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    int64_t gen = 0;
    std::vector<const void *> send;
};
bool loop_barrier(LoopGroup *g) {
    std::unique_lock<std::mutex> lk(g->m);
    const int64_t my = g->gen;
    if (++g->arrived == g->n) {
        g->arrived = 0;
        g->gen++;
        g->cv.notify_all();
        return true;
    }
    return g->cv.wait_for(lk, std::chrono::seconds(60), [&] { return g->gen != my; });
}
}  // namespace

extern "C" {

int32_t chopper_abi_version(void) { return CHOPPER_ABI_VERSION; }

size_t chopper_scratch_plan(const chopper_config *cfg, const chopper_shape *sh, chopper_scratch_items *items) {
    chopper_scratch_items it{};
    if (!cfg || !sh) {
        if (items) *items = it;
        return 0;
    }
    auto pos = [](int64_t v) { return (size_t)(v > 0 ? v : 0); };
    const size_t N = pos(sh->n_events), M = pos(sh->n_samples);
    const size_t S0 = pos(sh->n_spans[0]), S1 = pos(sh->n_spans[1]), S2 = pos(sh->n_spans[2]), S3 = pos(sh->n_spans[3]);
    const size_t S = S0 + S1 + S2 + S3;
    const size_t C = pos(sh->n_counters);
    const size_t Gt = pos(cfg->n_traced_gpus) > 0 ? pos(cfg->n_traced_gpus) : 1;
    const size_t G = sh->n_local_gpus > 0 ? pos(sh->n_local_gpus) : Gt;
    const size_t NC = sh->n_comm >= 0 ? std::min(pos(sh->n_comm), N) : N;
    const bool multi = sh->max_compute_streams != 1;
    const bool laminar = sh->laminar == 1;
    const size_t MI = pos(cfg->max_iters) > 0 ? pos(cfg->max_iters) : 1, L = pos(cfg->n_labels) > 0 ? pos(cfg->n_labels) : 1;
    const size_t K = pos(cfg->max_coll_per_class) > 0 ? pos(cfg->max_coll_per_class) : 1;
    const size_t tiles = (N + 2047) / 2048 + 1;
    const size_t Rb = std::min(N, 2 * S + tiles + G + 1) + 1;          // instance runs / instance rows
    const size_t row = 8 + 8 * RF_NFIELDS + 8 * std::max<size_t>(C, 1) + 7 * 4 + 8;   // RowTable with identity
    // events: permutation + chain predecessor end; counter-pass position + run id (counters); the exact
    // sweep's [4][N] span table (non-laminar); the explicit compute union + its permutation (several streams);
    // the head pre-count's key-table index per event (4 B, whole tiles) and, without counters, its per-thread
    // head masks / ranks
    it.events = N * 12 + (C ? N * 8 : 0) + (laminar ? 0 : N * 16) + (multi ? N * 28 : 0) + tiles * 2048 * 4 +
                (C ? 0 : tiles * 256 * 5);
    // push-order span arrays (32 B), Euler tables (12 B per endpoint), merged key table (16 B per endpoint),
    // chunk stacks and sparse tables (~8 B)
    it.spans = S * 32 + (2 * S + 4 * G + 2) * 28 + S * 8 + 4096 * (G + 1);
    // the push-order sort's key / value buffers, held from chopper_load_columns to chopper_attribute (the sort
    // runs beside chopper_align)
    it.spans += S * 24 + 16 * (4 * G + 2);
    it.unions = NC * 24 + (NC + M + 2 * G) * 44 + M * 40;
    // the preparation runs beside chopper_attribute and keeps its transients for the step: the compute-union sort
    // keys (several streams) and the sample terms
    it.unions += (multi ? N * 20 : 0) + M * 17;
    it.subruns = Rb * 144 + Rb * 8 * C + tiles * (8 * 3 + 16 + 64);
    it.instances = Rb * (row + 16);                                       // + group starts
    size_t roll = 0;
    const size_t above[4] = {G, 2 * S0 + G, 2 * (S0 + S1) + G, 2 * (S0 + S1 + S2) + G};
    for (int d = 0; d < 4; d++) roll += (std::min(Rb, above[d]) + 2) * (row + 16);
    it.rollups = roll + (std::min(Rb, above[1]) + 2) * 44;              // iteration extras
    const size_t its = std::min(MI, S0 + 1);
    const size_t cells = L * G * its;
    it.points = cells * (row + 8 * RF_NFIELDS + 8 * std::max<size_t>(C, 1) + 16) + Rb * 16;
    const size_t W1 = 4 + 4 * K;
    const size_t W2 = 4 + C + 8 * MI + 9 * MI * L + 32 * MI;
    it.exchange = (Gt + 8) * (W1 + W2) * 8 * 2 + L * 16 * 8 * MI * Gt * 2 + L * 4 * 8 * MI * Gt + 32 * 8 * MI * Gt;
    // sort buffers: events (general path: keys, values, alternates), spans, instance runs
    it.transient = std::max({(multi ? N : NC) * 24, S * 24, Rb * 24, N * (multi ? 20 : 0)});
    it.total = it.events + it.spans + it.unions + it.subruns + it.instances + it.rollups + it.points + it.exchange +
               it.transient;
    it.total += it.total / 16 + ((size_t)64 << 20);                     // alignment + small buffers
    if (items) *items = it;
    return it.total;
}

size_t chopper_scratch_bytes(const chopper_config *cfg, int64_t n_events, int64_t n_spans, int64_t n_samples,
                             int32_t n_counters) {
    if (!cfg) return 0;
    chopper_shape sh{};
    sh.n_events = n_events;
    sh.n_spans[0] = n_spans;
    sh.n_samples = n_samples;
    sh.n_comm = -1;
    sh.n_counters = n_counters;
    sh.n_local_gpus = 0;
    sh.max_compute_streams = 0;
    sh.laminar = 0;
    return chopper_scratch_plan(cfg, &sh, nullptr);
}

// orders a call's work after the caller's stream and the caller's stream after the call's work
struct CallJoin {
    chopper_ctx *c;
    explicit CallJoin(chopper_ctx *ctx) : c(ctx) {
        if (c && c->st) {
            cudaEventRecord(c->call_in, c->user_st);
            cudaStreamWaitEvent(c->st, c->call_in, 0);
        }
    }
    ~CallJoin() {
        if (c && c->st) {
            cudaEventRecord(c->call_out, c->st);
            cudaStreamWaitEvent(c->user_st, c->call_out, 0);
        }
    }
};

HostProf g_hprof;
DevMarks g_marks;

chopper_status chopper_create(chopper_ctx **out, const chopper_config *cfg, int device, void *cuda_stream,
                              void *nccl_comm, int rank, int nranks, void *scratch, size_t scratch_bytes) {
    if (!out || !cfg || !scratch) return CHOPPER_E_INVALID_ARG;
    if (cfg->n_traced_gpus <= 0 || cfg->n_traced_gpus > CH_MAX_GPUS || cfg->n_labels < 0 || cfg->max_iters <= 0 ||
        cfg->max_coll_per_class < 0 || nranks <= 0 || rank < 0 || rank >= nranks)
        return CHOPPER_E_INVALID_ARG;
    chopper_ctx *c = new chopper_ctx();
    c->cfg = *cfg;
    c->device = device;
    c->user_st = (cudaStream_t)cuda_stream;
    c->nccl = nccl_comm;
    c->rank = rank;
    c->nranks = nranks;
    c->scratch = (char *)scratch;
    c->scratch_bytes = scratch_bytes;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete c;
        return CHOPPER_E_CUDA;
    }
    // the library's work runs on a stream of the device's greatest priority: the block scheduler then dispatches
    // the main path's kernels ahead of pending blocks of the side streams (the counter pass, the span sort), which
    // fill the SMs the main path leaves idle.  Every call is ordered after the caller's stream and the caller's
    // stream after the call (CallJoin).
    {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        if (cudaStreamCreateWithPriority(&c->st, cudaStreamNonBlocking, greatest) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->call_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->call_out, cudaEventDisableTiming) != cudaSuccess) {
            delete c;
            return CHOPPER_E_CUDA;
        }
    }
    for (int q = 0; q < 3; q++) {
        if (cudaStreamCreateWithFlags(&c->side[q], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->join_ev[q], cudaEventDisableTiming) != cudaSuccess) {
            delete c;
            return CHOPPER_E_CUDA;
        }
    }
    if (cudaEventCreateWithFlags(&c->prep_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->span_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->span_join, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return CHOPPER_E_CUDA;
    }
    if (cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return CHOPPER_E_CUDA;
    }
    // pinned host ring for the stage read-backs (host memory; device memory is never allocated)
    c->pin_cap = 4u << 20;
    if (cudaHostAlloc(&c->h_pin, c->pin_cap, cudaHostAllocDefault) != cudaSuccess) {
        c->h_pin = nullptr;              // pageable read-backs (correct, slower)
        c->pin_cap = 0;
        cudaGetLastError();
    }
    *out = c;
    return CHOPPER_OK;
}

static chopper_status load_columns(chopper_ctx *ctx, const chopper_events *ev, const chopper_spans *sp,
                                   const chopper_samples *smp);
chopper_status chopper_load_columns(chopper_ctx *ctx, const chopper_events *ev, const chopper_spans *sp,
                                    const chopper_samples *smp) {
    g_hprof.dump();
    g_marks.dump();
    if (!ctx) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    g_marks.mark(ctx->st, "begin");
    ctx->poison = CHOPPER_OK;             // a new step
    ctx->x_exchanged = ctx->d_exchanged = false;
    ctx->stage = 0;
    return step(ctx, load_columns(ctx, ev, sp, smp));
}

static chopper_status load_columns(chopper_ctx *ctx, const chopper_events *ev, const chopper_spans *sp,
                                   const chopper_samples *smp) {
    if (!ev || !sp) return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "NULL events / spans");
    if (ev->n < 0 || ev->n > 0x7fffffffll || sp->n < 0 || sp->n > 0x7fffffffll)
        return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "event / span count out of range");
    if (ev->n > 0 && (!ev->dispatch_ns || !ev->start_ns || !ev->end_ns || !ev->meta || !ev->name_id))
        return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "NULL event column");
    if (sp->n > 0 && (!sp->gpu_level || !sp->start_ns || !sp->end_ns || !sp->label))
        return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "NULL span column");
    ctx->ev = *ev;
    ctx->sp = *sp;
    ctx->has_smp = smp && smp->n > 0;
    if (ctx->has_smp && (!smp->gpu || !smp->ts_ns || !smp->freq_mhz || !smp->power_mw))
        return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "NULL sample column");
    ctx->smp = ctx->has_smp ? *smp : chopper_samples{};
    ctx->N = ev->n;
    ctx->S = sp->n;
    ctx->M = ctx->has_smp ? smp->n : 0;
    ctx->stage = 0;
    ctx->latched_host = 0;
    ctx->offsets_done = false;
    ctx->C = 0;
    ctx->d_col = nullptr;
    ctx->d_nm_rank = nullptr;
    ctx->d_bd = nullptr;            // (reduce_ranks reuses this step's local breakdown with one rank)
    ctx->n_bd = 0;
    ctx->present.clear();
    ctx->err.clear();
    memset(&ctx->rep, 0, sizeof(ctx->rep));
    if (cudaSetDevice(ctx->device) != cudaSuccess) return ch_fail(ctx, CHOPPER_E_CUDA, "cudaSetDevice");
    ch_tick(ctx, 0, 0);
    chopper_status s = ch_load(ctx);
    if (s != CHOPPER_OK) return s;
    ch_tick(ctx, 0, 1);
    ctx->stage = 1;
    return CHOPPER_OK;
}

static chopper_status align(chopper_ctx *ctx, const chopper_counter_pass *passes, int32_t n_passes,
                            int32_t n_counters, double *counters_out, int64_t *offsets_ns) {
    if (ctx->stage != 1 || !ctx->loaded_ok) return ch_fail(ctx, CHOPPER_E_STATE, "chopper_align before load");
    if (n_passes < 0 || n_counters < 0 || (n_passes > 0 && !passes))
        return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "bad counter passes");
    ch_tick(ctx, 1, 0);
    CH_TRY(ch_align(ctx, passes, n_passes, n_counters, counters_out));
    CH_TRY(ch_offsets(ctx));
    ch_tick(ctx, 1, 1);
    ctx->offsets_done = true;
    if (offsets_ns)
        for (int g = 0; g < ctx->cfg.n_traced_gpus; g++) offsets_ns[g] = ctx->delta[g];
    ctx->stage = 2;
    return CHOPPER_OK;
}

chopper_status chopper_align(chopper_ctx *ctx, const chopper_counter_pass *passes, int32_t n_passes,
                             int32_t n_counters, double *counters_out, int64_t *offsets_ns) {
    if (!ctx) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    ctx->C = n_counters > 0 ? n_counters : 0;     // fixes the shape of exchange #2 even if this call fails
    if (ctx->poison != CHOPPER_OK) {
        chopper_status s = ch_exchange_poison(ctx, 1);
        return s != CHOPPER_OK ? s : dead_call(ctx);
    }
    chopper_status s = step(ctx, align(ctx, passes, n_passes, n_counters, counters_out, offsets_ns));
    if (s != CHOPPER_OK) ch_exchange_poison(ctx, 1);     // no-op if this rank's all-gather #1 already ran
    return s;
}

}  // extern "C"
// chopper_overlap's preparation on side[1] (see attribute)
chopper_status ch_prep_side(chopper_ctx *ctx) {
    ctx->prep_deferred = false;
    // ordered after the main stream's work at chopper_attribute's start (span_fork, recorded there; the load's
    // span sort consumed its previous record), not after the span kernels enqueued since
    CH_CUDA(ctx, cudaStreamWaitEvent(ctx->side[1], ctx->span_fork, 0));
    cudaStream_t main_st = ctx->st;
    ctx->st = ctx->side[1];
    ctx->hold_scratch = true;
    const chopper_status ps = ch_overlap_prep(ctx);
    ctx->hold_scratch = false;
    CH_CUDA(ctx, cudaEventRecord(ctx->prep_join, ctx->st));
    ctx->st = main_st;
    CH_TRY(ps);
    ctx->prep_done = ctx->prep_pending = true;
    return CHOPPER_OK;
}
extern "C" {

static chopper_status attribute(chopper_ctx *ctx, int32_t *span_idx) {
    if (ctx->stage == 1 && ctx->nranks == 1) {
        // align may be skipped on one rank without counters
        CH_TRY(ch_align(ctx, nullptr, 0, 0, nullptr));
        CH_TRY(ch_offsets(ctx));
        ctx->offsets_done = true;
        ctx->stage = 2;
    }
    if (ctx->stage != 2) return ch_fail(ctx, CHOPPER_E_STATE, "chopper_attribute out of order");
    ch_tick(ctx, 2, 0);
    // chopper_overlap's preparation (comm union, sample integrals, timeline) needs nothing from the span tables:
    // it runs on side[1] beside the span build, whose kernels are small and whose host synchronizations would
    // leave the gpu idle; chopper_overlap joins it.  Its host part is done inside the span build, once the
    // Euler-table kernels are enqueued (ch_prep_side), so that the gpu runs them meanwhile
    CH_CUDA(ctx, cudaEventRecord(ctx->span_fork, ctx->st));
    ctx->prep_deferred = true;
    CH_TRY(ch_build_spans(ctx));
    if (ctx->prep_deferred) CH_TRY(ch_prep_side(ctx));
    CH_TRY(ch_attr_pass(ctx, span_idx));
    ch_tick(ctx, 2, 1);
    ctx->stage = 3;
    return CHOPPER_OK;
}

chopper_status chopper_attribute(chopper_ctx *ctx, int32_t *span_idx) {
    if (!ctx) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    if (ctx->poison != CHOPPER_OK) return dead_call(ctx);
    return step(ctx, attribute(ctx, span_idx));
}

static chopper_status overlap(chopper_ctx *ctx, int64_t *ovl_ns, int64_t *prep_ns, int64_t *call_ns, int64_t *phi,
                              int64_t *psi) {
    if (ctx->stage != 3) return ch_fail(ctx, CHOPPER_E_STATE, "chopper_overlap out of order");
    ch_tick(ctx, 3, 0);
    if (ctx->prep_pending) {                    // enqueued beside chopper_attribute
        CH_CUDA(ctx, cudaStreamWaitEvent(ctx->st, ctx->prep_join, 0));
        ctx->prep_pending = false;
    }
    g_marks.mark(ctx->st, "ov_prep_join");
    if (!ctx->prep_done) CH_TRY(ch_overlap_prep(ctx));
    ctx->prep_done = false;
    ch_tick(ctx, 3, 1);
    CH_TRY(ch_event_pass(ctx, ovl_ns, prep_ns, call_ns, phi, psi));
    ctx->stage = 4;
    return CHOPPER_OK;
}

chopper_status chopper_overlap(chopper_ctx *ctx, int64_t *ovl_ns, int64_t *prep_ns, int64_t *call_ns, int64_t *phi,
                               int64_t *psi) {
    if (!ctx) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    if (ctx->poison != CHOPPER_OK) return dead_call(ctx);
    return step(ctx, overlap(ctx, ovl_ns, prep_ns, call_ns, phi, psi));
}

static void fill_rows(chopper_rows &r, const RowTable &t, bool iter, chopper_ctx *ctx) {
    memset(&r, 0, sizeof(r));
    r.n = t.n;
    r.stride = t.cap;
    r.gpu = t.gpu; r.it = t.it; r.ph = t.ph; r.ly = t.ly; r.op = t.op; r.label = t.label; r.rank = t.rank;
    r.n_events = t.f + (int64_t)RF_NEV * t.cap;
    r.n_compute = t.f + (int64_t)RF_N * t.cap;
    r.busy = t.f + (int64_t)RF_BUSY * t.cap;
    r.first_ks = t.f + (int64_t)RF_FIRST_KS * t.cap;
    r.first_idx = t.f + (int64_t)RF_FIRST_IDX * t.cap;
    r.first_pred = t.first_pred;
    r.last_ke = t.f + (int64_t)RF_LAST_KE * t.cap;
    r.prep = t.f + (int64_t)RF_PREP * t.cap;
    r.call = t.f + (int64_t)RF_CALL * t.cap;
    r.ovl = t.f + (int64_t)RF_OVL * t.cap;
    r.phi = t.f + (int64_t)RF_PHI * t.cap;
    r.psi = t.f + (int64_t)RF_PSI * t.cap;
    r.copy_ns = t.f + (int64_t)RF_COPY * t.cap;
    r.ag_ns = t.f + (int64_t)RF_AG * t.cap;
    r.rs_ns = t.f + (int64_t)RF_RS * t.cap;
    r.counters = t.cnt;
    r.rates = t.rates;
    r.metrics = t.metrics;
    if (iter) {
        r.wall = ctx->iter_wall;
        r.comm_union = ctx->iter_cu;
        r.aligned_first = ctx->iter_af;
        r.aligned_last = ctx->iter_al;
        r.step = ctx->iter_step;
    }
}

static chopper_status breakdown(chopper_ctx *ctx, const chopper_bd_params *p, chopper_tables *out) {
    if (ctx->stage != 4) return ch_fail(ctx, CHOPPER_E_STATE, "chopper_breakdown out of order");
    if (!p || !out || (ctx->cfg.n_labels > 0 && (!p->f_gemm || !p->op_type)) || p->n_ratios < 0 ||
        (p->n_ratios > 0 && (!p->ratio_num || !p->ratio_den || !p->ratio_scale)))
        return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "bad breakdown parameters");
    const int C = ctx->C;
    auto bad_slot = [&](int s) { return s >= C || s < -1; };
    if (bad_slot(p->slot_gpu_cycles) || bad_slot(p->slot_perf_flops) || bad_slot(p->slot_util_num) ||
        bad_slot(p->slot_util_den))
        return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "breakdown counter slot out of range");
    for (int q = 0; q < p->n_ratios; q++)
        if (p->ratio_num[q] < 0 || p->ratio_num[q] >= C || p->ratio_den[q] < -1 || p->ratio_den[q] >= C)
            return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "ratio slot out of range");
    ctx->bd = *p;
    const int L = ctx->cfg.n_labels;
    ctx->f_gemm.assign(p->f_gemm, p->f_gemm + L);
    ctx->op_type.assign(p->op_type, p->op_type + L);
    ctx->n_ratios = p->n_ratios;
    CH_ALLOC_BEGIN;
    ctx->d_f_gemm = CH_ALLOC(ctx, double, std::max(L, 1));
    ctx->d_op_type = CH_ALLOC(ctx, int32_t, std::max(L, 1));
    ctx->d_ratio = CH_ALLOC(ctx, int32_t, 2 * std::max(p->n_ratios, 1));
    ctx->d_ratio_scale = CH_ALLOC(ctx, double, std::max(p->n_ratios, 1));
    CH_ALLOC_END(ctx);
    if (L > 0) {
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_f_gemm, ctx->f_gemm.data(), 8 * L, cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_op_type, ctx->op_type.data(), 4 * L, cudaMemcpyHostToDevice, ctx->st));
    }
    if (p->n_ratios > 0) {
        std::vector<int32_t> r(2 * p->n_ratios);
        for (int q = 0; q < p->n_ratios; q++) { r[q] = p->ratio_num[q]; r[p->n_ratios + q] = p->ratio_den[q]; }
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_ratio, r.data(), 4 * r.size(), cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_ratio_scale, p->ratio_scale, 8 * p->n_ratios, cudaMemcpyHostToDevice,
                                     ctx->st));
    }
    ch_tick(ctx, 5, 0);
    CH_TRY(ch_tables(ctx));
    ch_tick(ctx, 5, 1);
    ch_tick(ctx, 6, 0);
    CH_TRY(ch_breakdown_local(ctx));
    ch_tick(ctx, 6, 1);
    memset(out, 0, sizeof(*out));
    fill_rows(out->inst, ctx->inst, false, ctx);
    fill_rows(out->layer, ctx->layer, false, ctx);
    fill_rows(out->phase, ctx->phase, false, ctx);
    fill_rows(out->iter, ctx->iter, true, ctx);
    fill_rows(out->gpu, ctx->gpurow, false, ctx);
    fill_rows(out->point, ctx->point, false, ctx);
    out->n_bd = ctx->n_bd;
    out->bd = ctx->d_bd;
    out->n_metrics = ctx->n_metrics;
    ctx->stage = 5;
    return CHOPPER_OK;
}

chopper_status chopper_breakdown(chopper_ctx *ctx, const chopper_bd_params *p, chopper_tables *out) {
    if (!ctx) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    if (ctx->poison != CHOPPER_OK) return dead_call(ctx);
    return step(ctx, breakdown(ctx, p, out));
}

static chopper_status reduce_ranks(chopper_ctx *ctx, chopper_global *out) {
    if (!out) return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "NULL chopper_global");
    if (ctx->stage != 5) return ch_fail(ctx, CHOPPER_E_STATE, "chopper_reduce_ranks out of order");
    memset(out, 0, sizeof(*out));
    ch_tick(ctx, 7, 0);
    CH_TRY(ch_reduce_ranks(ctx, out));
    ch_tick(ctx, 7, 1);
    ctx->stage = 6;
    return CHOPPER_OK;
}

chopper_status chopper_reduce_ranks(chopper_ctx *ctx, chopper_global *out) {
    if (!ctx) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    if (ctx->poison != CHOPPER_OK) {
        chopper_status s = ch_exchange_poison(ctx, 2);
        return s != CHOPPER_OK ? s : dead_call(ctx);
    }
    chopper_status s = step(ctx, reduce_ranks(ctx, out));
    if (s != CHOPPER_OK) ch_exchange_poison(ctx, 2);     // no-op if this rank's all-gather #2 already ran
    return s;
}

chopper_status chopper_report_cdf(chopper_ctx *ctx, double *out, int64_t cap, int64_t *n_rows) {
    if (!ctx || !n_rows || cap < 0 || (cap > 0 && !out)) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    if (ctx->stage != 6) return ch_fail(ctx, CHOPPER_E_STATE, "chopper_report_cdf before chopper_reduce_ranks");
    return ch_report_cdf(ctx, out, cap, n_rows);
}

size_t chopper_ingest_scratch_bytes(int64_t n_bytes) { return n_bytes < 0 ? 0 : ch_ingest_scratch_bytes(n_bytes); }

chopper_status chopper_ingest_chrome(chopper_ctx *ctx, const char *json, int64_t n_bytes, void *scratch,
                                     size_t scratch_bytes, const chopper_ingest_out *out, chopper_ingest_report *rep) {
    CallJoin join_(ctx);
    if (!ctx || n_bytes < 0 || (n_bytes > 0 && !json) || !scratch || !out || !rep || out->ev_cap < 0 ||
        out->span_cap < 0 || (out->ev_cap > 0 && (!out->t_l || !out->t_ks || !out->t_ke || !out->meta || !out->name_id)) ||
        (out->span_cap > 0 && (!out->span_gl || !out->span_start || !out->span_end || !out->span_label)))
        return CHOPPER_E_INVALID_ARG;
    return ch_ingest_chrome(ctx, json, n_bytes, scratch, scratch_bytes, out, rep);
}

chopper_status chopper_set_metrics(chopper_ctx *ctx, int32_t n, const char *const *exprs, int32_t n_names,
                                   const char *const *names, int32_t *bad_expr) {
    if (!ctx || n < 0 || n_names < 0 || (n > 0 && !exprs) || (n_names > 0 && !names)) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    return ch_compile_metrics(ctx, n, exprs, n_names, names, bad_expr);
}

chopper_status chopper_cpu_util(chopper_ctx *ctx, const chopper_cpu_samples *samples, const int32_t *topology,
                                int32_t n_logical, int64_t *c_active, double *c_min, int64_t cap,
                                chopper_cpu_summary *out) {
    CallJoin join_(ctx);
    if (!ctx || !samples || !out || samples->n < 0 || n_logical <= 0 || !topology || cap < 0 ||
        (samples->n > 0 && (!samples->ts_ns || !samples->logical_core || !samples->util_pct)))
        return CHOPPER_E_INVALID_ARG;
    return ch_cpu_util(ctx, samples, topology, n_logical, c_active, c_min, cap, out);
}

chopper_status chopper_set_allgather(chopper_ctx *ctx, chopper_allgather_fn fn, void *user) {
    if (!ctx) return CHOPPER_E_INVALID_ARG;
    ctx->ag_fn = fn;
    ctx->ag_user = fn ? user : nullptr;
    return CHOPPER_OK;
}

void *chopper_loopback_create(int32_t nranks) {
    if (nranks < 1 || nranks > CH_MAX_GPUS) return nullptr;
    LoopGroup *g = new LoopGroup();
    g->n = nranks;
    g->send.assign(nranks, nullptr);
    return g;
}

void chopper_loopback_destroy(void *group) { delete static_cast<LoopGroup *>(group); }

int32_t chopper_loopback_allgather(void *group, const void *send, void *recv, size_t bytes_per_rank, int32_t rank,
                                   int32_t nranks, void *cuda_stream) {
    LoopGroup *g = static_cast<LoopGroup *>(group);
    if (!g || nranks != g->n || rank < 0 || rank >= nranks) return 1;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if (cudaStreamSynchronize(st) != cudaSuccess) return 2;       // this rank's send block is complete
    {
        std::lock_guard<std::mutex> lk(g->m);
        g->send[rank] = send;
    }
    if (!loop_barrier(g)) return 3;                                 // every send block is complete
    for (int r = 0; r < nranks; r++)
        if (cudaMemcpyAsync((char *)recv + (size_t)r * bytes_per_rank, g->send[r], bytes_per_rank,
                            cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return 4;
    if (cudaStreamSynchronize(st) != cudaSuccess) return 5;
    if (!loop_barrier(g)) return 6;                                 // nobody reuses a send block early
    return 0;
}

chopper_status chopper_get_report(const chopper_ctx *ctx, chopper_report *out) {
    if (!ctx || !out) return CHOPPER_E_INVALID_ARG;
    *out = ctx->rep;
    return CHOPPER_OK;
}

chopper_status chopper_status_sync(chopper_ctx *ctx, uint32_t *mask) {
    if (!ctx) return CHOPPER_E_INVALID_ARG;
    CallJoin join_(ctx);
    uint32_t m = ctx->latched_host;
    unsigned int dl = 0;
    if (ctx->d_rep && ch_d2h(ctx, &dl, &ctx->d_rep->latched, 4) != cudaSuccess) m |= 1u << CHOPPER_E_CUDA;
    if (ch_sync(ctx) != cudaSuccess) m |= 1u << CHOPPER_E_CUDA;     // (one synchronization, the flag with it)
    m |= dl;
    if (mask) *mask = m;
    const chopper_status order[] = {CHOPPER_E_CUDA, CHOPPER_E_NCCL, CHOPPER_E_VALIDATION, CHOPPER_E_ALIGNMENT,
                                    CHOPPER_E_AMBIGUOUS_SPANS, CHOPPER_E_RANGE, CHOPPER_E_INSUFFICIENT_DATA,
                                    CHOPPER_E_INVALID_ARG, CHOPPER_E_STATE};
    for (chopper_status s : order)
        if (m & (1u << s)) return s;
    return CHOPPER_OK;
}

const char *chopper_last_error(const chopper_ctx *ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

void chopper_destroy(chopper_ctx *ctx) {
    if (!ctx) return;
    for (auto &p : ctx->tev)
        for (auto &e : p)
            if (e) cudaEventDestroy(e);
    for (int q = 0; q < 3; q++) {
        if (ctx->side[q]) cudaStreamDestroy(ctx->side[q]);
        if (ctx->join_ev[q]) cudaEventDestroy(ctx->join_ev[q]);
    }
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->span_fork) cudaEventDestroy(ctx->span_fork);
    if (ctx->prep_join) cudaEventDestroy(ctx->prep_join);
    if (ctx->span_join) cudaEventDestroy(ctx->span_join);
    if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
    if (ctx->st) cudaStreamDestroy(ctx->st);
    if (ctx->call_in) cudaEventDestroy(ctx->call_in);
    if (ctx->call_out) cudaEventDestroy(ctx->call_out);
    delete ctx;
}

int64_t chopper_kernel_launches(const chopper_ctx *ctx) { return ctx ? ctx->launches : 0; }
int64_t chopper_host_syncs(const chopper_ctx *ctx) { return ctx ? ctx->syncs : 0; }

/* extra introspection used by the Python binding / tests */
int64_t chopper_pass_mismatch(const chopper_ctx *ctx, int32_t p) {
    return (ctx && p >= 0 && p < (int)ctx->pass_mismatch.size()) ? ctx->pass_mismatch[p] : -1;
}
int64_t chopper_pass_conflict(const chopper_ctx *ctx, int32_t p) {
    return (ctx && p >= 0 && p < (int)ctx->pass_conflict.size()) ? ctx->pass_conflict[p] : -1;
}
int32_t chopper_counter_present(const chopper_ctx *ctx, int32_t gpu, int32_t slot) {
    if (!ctx || gpu < 0 || gpu >= CH_MAX_GPUS || slot < 0 || slot >= ctx->C) return 0;
    int lg = ctx->gpu_lg_h[gpu];
    return lg >= 0 && (size_t)lg * ctx->C + slot < ctx->present.size() ? ctx->present[(size_t)lg * ctx->C + slot] : 0;
}
int64_t chopper_scratch_used(const chopper_ctx *ctx) { return ctx ? (int64_t)ctx->high : 0; }

void chopper_set_timing(chopper_ctx *ctx, int32_t on) {
    if (ctx) ctx->timing = on != 0;
}

chopper_status chopper_phase_time(chopper_ctx *ctx, int32_t phase, float *ms) {
    if (!ctx || !ms || phase < 0 || phase >= 10) return CHOPPER_E_INVALID_ARG;
    if (!ctx->timed[phase]) return CHOPPER_E_STATE;
    if (cudaEventSynchronize(ctx->tev[phase][1]) != cudaSuccess) return CHOPPER_E_CUDA;
    if (cudaEventElapsedTime(ms, ctx->tev[phase][0], ctx->tev[phase][1]) != cudaSuccess) return CHOPPER_E_CUDA;
    return CHOPPER_OK;
}

}  // extern "C"
