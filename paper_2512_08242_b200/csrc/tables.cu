// tables.cu -- a9 segmented reductions and roll-ups (chopper_breakdown part 1).
//
// Sub-runs from the event pass are stably radix-sorted by their packed
// instance key (gpu, iteration, phase, layer, op ranks in push order, 0 =
// none); each maximal group of equal keys is one instance row (SPEC.md:186-194,
// PAPER.md:411).  Because the key packs the hierarchy most-significant first,
// parents are contiguous groups of the children sorted by key >> shift:
// instance -> layer -> phase -> iteration -> GPU, each parent the sum of its
// children in ascending key order (D12).  Points (gpu, iteration, op label)
// sum instances across layers.  Counter sums (fp64)
// are per sub-run warp reductions in a fixed order, then summed in key order.
#include "common.cuh"

namespace {
constexpr int NT = 256;

// counter sums of each sub-run over its COMPUTE events, tiled like the event pass (2048 events per
// block, 8 consecutive per thread; sub-runs never cross tiles).  Slots are processed SG at a time.
// Pieces spanning threads are completed through shared memory in forward (input) order.
constexpr int CT_NT = 256, CT_IPT = 8, CT_TILE = CT_NT * CT_IPT, CT_SG = 8;
__global__ void __launch_bounds__(CT_NT) k_counters_tiled(const uint32_t *__restrict__ meta,
                                                          const int32_t *__restrict__ run_id,
                                                          const int32_t *__restrict__ nm_rank,
                                                          const int32_t *__restrict__ gpu_lg,
                                                          const double *const *__restrict__ col, int C, int s0,
                                                          int64_t N, double *__restrict__ out, int64_t cap) {
    __shared__ double fp[CT_SG][CT_NT], lp[CT_SG][CT_NT];
    __shared__ unsigned char hh[CT_NT];
    const int tid = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * CT_TILE, i0 = base + (int64_t)tid * CT_IPT;
    double acc[CT_SG];
#pragma unroll
    for (int q = 0; q < CT_SG; q++) acc[q] = 0.0;
    bool has = false;
    int32_t cur = -1, first_head = -1;
    int32_t prev = (i0 > base && i0 < N) ? run_id[i0 - 1] : -1;
    for (int k = 0; k < CT_IPT; k++) {
        int64_t i = i0 + k;
        if (i >= N) break;
        int32_t rid = run_id[i];
        if (i == base || rid != prev) {
            if (!has) {
#pragma unroll
                for (int q = 0; q < CT_SG; q++) fp[q][tid] = acc[q];
                has = true;
                first_head = rid;
            } else {
#pragma unroll
                for (int q = 0; q < CT_SG; q++)
                    if (s0 + q < C) out[(int64_t)(s0 + q) * cap + cur] = acc[q];
            }
#pragma unroll
            for (int q = 0; q < CT_SG; q++) acc[q] = 0.0;
            cur = rid;
        }
        prev = rid;
        uint32_t m = meta[i];
        if (kind_of(m) == CK_COMPUTE) {
            int lg = gpu_lg[gpu_of(m)];
            int64_t j = nm_rank[i];
#pragma unroll
            for (int q = 0; q < CT_SG; q++) {
                int s = s0 + q;
                if (s < C) {
                    const double *c = col[lg * C + s];
                    if (c) acc[q] += c[j];
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < CT_SG; q++) {
        if (has) lp[q][tid] = acc[q];
        else fp[q][tid] = acc[q];
    }
    hh[tid] = has;
    __syncthreads();
    // a sub-run ending inside this thread's first piece started at the nearest earlier thread with a head
    auto complete = [&](int upto, bool own_last, int32_t id) {
        int u = upto - 1;
        while (!hh[u]) u--;
        for (int q = 0; q < CT_SG; q++) {
            if (s0 + q >= C) break;
            double s = lp[q][u];
            for (int v = u + 1; v < upto; v++) s += fp[q][v];
            s += own_last ? lp[q][upto] : fp[q][upto];
            out[(int64_t)(s0 + q) * cap + id] = s;
        }
    };
    if (has && tid > 0 && base < N) complete(tid, false, first_head - 1);
    if (tid == CT_NT - 1 && base < N) {
        int64_t last = base + CT_TILE - 1 < N ? base + CT_TILE - 1 : N - 1;
        int32_t id = run_id[last];
        if (has) {
            for (int q = 0; q < CT_SG; q++)
                if (s0 + q < C) out[(int64_t)(s0 + q) * cap + id] = lp[q][tid];
        } else {
            complete(tid, false, id);
        }
    }
}

__global__ void k_copy_keys(const unsigned long long *__restrict__ k, int64_t n, unsigned long long *__restrict__ out,
                            uint32_t *__restrict__ v) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { out[i] = k[i]; v[i] = (uint32_t)i; }
}

// heads of groups of equal (key >> shift) among valid keys; also the valid count
__global__ void k_group_heads(const unsigned long long *__restrict__ key, int64_t n, int shift,
                              int64_t *__restrict__ head, unsigned long long *__restrict__ nvalid) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    unsigned long long k = key[j];
    bool valid = k != CH_INVALID_KEY;
    if (!valid) { head[j] = 0; atomicMin(nvalid, (unsigned long long)j); return; }
    unsigned long long g = shift >= 64 ? 0 : (k >> shift);
    head[j] = (j == 0 || (key[j - 1] >> shift) != g) ? 1 : 0;
}

__global__ void k_group_starts(const int64_t *__restrict__ head, const int64_t *__restrict__ ex, int64_t n,
                               int64_t *__restrict__ starts) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n && head[j]) starts[ex[j]] = j;
}

struct TabView {
    unsigned long long *key;
    int64_t *f;
    double *cnt;
    int64_t cap;     // field stride (field-major tables: capacity; AoS sub-runs: 1)
    int64_t ccap;    // counter-column capacity
    int64_t rs;      // row stride (field-major: 1; AoS sub-runs: 16)
};

// parent row p = sum of children [starts[p], starts[p+1]) visited in order (through perm if given)
__global__ void k_sum_rows(TabView ch, const uint32_t *__restrict__ perm, const int64_t *__restrict__ starts,
                           int64_t ng, int shift, int C, TabView pa) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= ng) return;
    int64_t lo = starts[p], hi = starts[p + 1];
    int64_t v[RF_NFIELDS];
#pragma unroll
    for (int f = 0; f < RF_NFIELDS; f++) v[f] = 0;
    v[RF_FIRST_IDX] = INT64_MAX;
    v[RF_FIRST_KS] = INT64_MAX;
    v[RF_LAST_KE] = INT64_MIN;
    unsigned long long k0 = 0;
    for (int64_t j = lo; j < hi; j++) {
        int64_t c = perm ? (int64_t)perm[j] : j;
        if (j == lo) k0 = ch.key[c];
#pragma unroll
        for (int f = 0; f < RF_NFIELDS; f++) {
            int64_t x = ch.f[(int64_t)f * ch.cap + c * ch.rs];
            if (f == RF_FIRST_IDX || f == RF_FIRST_KS) continue;
            if (f == RF_LAST_KE) { if (x > v[f]) v[f] = x; continue; }
            v[f] += x;
        }
        int64_t cks = ch.f[(int64_t)RF_FIRST_KS * ch.cap + c * ch.rs], cidx = ch.f[(int64_t)RF_FIRST_IDX * ch.cap + c * ch.rs];
        if (cks < v[RF_FIRST_KS] || (cks == v[RF_FIRST_KS] && cidx < v[RF_FIRST_IDX])) {
            v[RF_FIRST_KS] = cks;
            v[RF_FIRST_IDX] = cidx;
        }
    }
#pragma unroll
    for (int f = 0; f < RF_NFIELDS; f++) pa.f[(int64_t)f * pa.cap + p] = v[f];
    pa.key[p] = shift >= 64 ? 0ull : ((k0 >> shift) << shift);
    for (int s = 0; s < C; s++) {
        double acc = 0.0;
        for (int64_t j = lo; j < hi; j++) {
            int64_t c = perm ? (int64_t)perm[j] : j;
            acc += ch.cnt[(int64_t)s * ch.ccap + c];
        }
        pa.cnt[(int64_t)s * pa.ccap + p] = acc;
    }
}

struct KeyLayout {
    int sh_op, sh_ly, sh_ph, sh_it, sh_lg;
    int kb[4];
};

__device__ __forceinline__ int64_t comp(unsigned long long key, int sh, int bits) {
    return bits == 0 ? 0 : (int64_t)((key >> sh) & ((1ull << bits) - 1));
}

// identity columns of a row table: caller span indices, gpu, op label, iteration rank
__global__ void k_decode(const unsigned long long *__restrict__ key, int64_t n, KeyLayout L, int depth,
                         const int32_t *__restrict__ lg_gpu, const int64_t *__restrict__ list_beg,
                         const int32_t *__restrict__ P_orig, const int32_t *__restrict__ P_label,
                         const int64_t *__restrict__ f, int64_t cap, const int64_t *__restrict__ pred_end,
                         int32_t *gpu, int32_t *it, int32_t *ph, int32_t *ly, int32_t *op, int32_t *label,
                         int32_t *rank, int64_t *first_pred) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    unsigned long long k = key[j];
    int lg = (int)(k >> L.sh_lg);
    int64_t r[4] = {comp(k, L.sh_it, L.kb[0]), comp(k, L.sh_ph, L.kb[1]), comp(k, L.sh_ly, L.kb[2]),
                    comp(k, L.sh_op, L.kb[3])};
    int32_t idx[4];
    for (int lv = 0; lv < 4; lv++) {
        idx[lv] = (lv < depth && r[lv] > 0) ? P_orig[list_beg[lg * 4 + lv] + r[lv] - 1] : -1;
    }
    gpu[j] = lg_gpu[lg];
    it[j] = idx[0];
    ph[j] = idx[1];
    ly[j] = idx[2];
    op[j] = idx[3];
    label[j] = (depth >= 4 && r[3] > 0) ? P_label[list_beg[lg * 4 + 3] + r[3] - 1] : -1;
    rank[j] = depth >= 1 && r[0] > 0 ? (int32_t)(r[0] - 1) : -1;
    int64_t fi = f[(int64_t)RF_FIRST_IDX * cap + j];
    first_pred[j] = (fi != INT64_MAX) ? pred_end[fi] : CH_NONE_TS;
}

// point key: (op label, gpu, iteration rank); instances without an op span are dropped
__global__ void k_point_keys(const unsigned long long *__restrict__ key, int64_t n, KeyLayout L,
                             const int64_t *__restrict__ list_beg, const int32_t *__restrict__ P_label, int kg,
                             unsigned long long *__restrict__ out, uint32_t *__restrict__ v) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    unsigned long long k = key[j];
    int lg = (int)(k >> L.sh_lg);
    int64_t rop = comp(k, L.sh_op, L.kb[3]);
    int64_t rit = comp(k, L.sh_it, L.kb[0]);
    unsigned long long o = CH_INVALID_KEY;
    if (rop > 0) {
        unsigned long long lab = (unsigned long long)P_label[list_beg[lg * 4 + 3] + rop - 1];
        o = (lab << (kg + L.kb[0])) | ((unsigned long long)lg << L.kb[0]) | (unsigned long long)rit;
    }
    out[j] = o;
    v[j] = (uint32_t)j;
}

__global__ void k_decode_points(const unsigned long long *__restrict__ key, int64_t n, int kg, int kb0,
                                const int32_t *__restrict__ lg_gpu, const int64_t *__restrict__ list_beg,
                                const int32_t *__restrict__ P_orig, const int64_t *__restrict__ f, int64_t cap,
                                const int64_t *__restrict__ pred_end, int32_t *gpu, int32_t *it, int32_t *ph,
                                int32_t *ly, int32_t *op, int32_t *label, int32_t *rank, int64_t *first_pred) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    unsigned long long k = key[j];
    int64_t rit = (int64_t)(k & ((1ull << kb0) - 1));
    int lg = (int)((k >> kb0) & ((1ull << kg) - 1));
    int lab = (int)(k >> (kg + kb0));
    gpu[j] = lg_gpu[lg];
    it[j] = rit > 0 ? P_orig[list_beg[lg * 4] + rit - 1] : -1;
    ph[j] = ly[j] = op[j] = -1;
    label[j] = lab;
    rank[j] = (int32_t)(rit - 1);
    int64_t fi = f[(int64_t)RF_FIRST_IDX * cap + j];
    first_pred[j] = (fi != INT64_MAX) ? pred_end[fi] : CH_NONE_TS;
}

// iteration extras: wall (telescoping chain span), comm union inside the iteration, aligned bounds, step
__global__ void k_iter_extras(int64_t n, const int64_t *__restrict__ f, int64_t cap, const int32_t *__restrict__ gpu,
                              const int32_t *__restrict__ it, const int64_t *__restrict__ first_pred,
                              const int32_t *__restrict__ gpu_lg, const int32_t *__restrict__ span_label,
                              const int64_t *__restrict__ Us, const int64_t *__restrict__ Ue,
                              const int64_t *__restrict__ UP, const int64_t *__restrict__ Ubeg,
                              const int64_t *__restrict__ Ucnt, const int64_t *__restrict__ delta,
                              int64_t *__restrict__ wall, int64_t *__restrict__ cu, int64_t *__restrict__ af,
                              int64_t *__restrict__ al, int32_t *__restrict__ step) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int g = gpu[j];
    step[j] = span_label[it[j]];
    int64_t nn = f[(int64_t)RF_N * cap + j];
    int64_t fk = f[(int64_t)RF_FIRST_KS * cap + j], lk = f[(int64_t)RF_LAST_KE * cap + j];
    if (nn > 0) {
        int64_t fp = first_pred[j];
        wall[j] = lk - (fp != CH_NONE_TS ? fp : fk);
        int lg = gpu_lg[g];
        int64_t lo = Ubeg[lg], hi = lo + Ucnt[lg];
        auto cov = [&](int64_t t) -> int64_t {
            int64_t u = last_le(Us, lo, hi, t);
            if (u < lo) return 0;
            int64_t x = t - Us[u], len = Ue[u] - Us[u];
            return UP[u] + (x < len ? x : len);
        };
        cu[j] = cov(lk) - cov(fk);
        af[j] = fk - delta[g];
        al[j] = lk - delta[g];
    } else {
        wall[j] = 0; cu[j] = 0; af[j] = 0; al[j] = 0;
    }
}

__global__ void k_rates(int64_t n, const int64_t *__restrict__ f, const double *__restrict__ cnt, int64_t cap,
                        int nr, const int32_t *__restrict__ rnum, const int32_t *__restrict__ rden,
                        const double *__restrict__ rsc, double *__restrict__ out) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    for (int q = 0; q < nr; q++) {
        double num = cnt[(int64_t)rnum[q] * cap + j];
        double den = rden[q] < 0 ? (double)f[(int64_t)RF_BUSY * cap + j] * 1e-9 : cnt[(int64_t)rden[q] * cap + j];
        out[(int64_t)q * n + j] = num / den * rsc[q];
    }
}
__global__ void k_gather_keys(const unsigned long long *k, const int64_t *starts, int64_t n, unsigned long long *out) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) out[j] = k[starts[j]];
}
}  // namespace

static chopper_status alloc_table(chopper_ctx *ctx, RowTable &t, int64_t cap, int C, bool identity) {
    CH_ALLOC_BEGIN;
    t.cap = cap;
    t.key = CH_ALLOC(ctx, unsigned long long, cap + 1);
    t.f = CH_ALLOC(ctx, int64_t, (int64_t)RF_NFIELDS * cap);
    t.cnt = CH_ALLOC(ctx, double, (int64_t)(C > 0 ? C : 1) * cap);
    if (identity) {
        t.gpu = CH_ALLOC(ctx, int32_t, cap);
        t.it = CH_ALLOC(ctx, int32_t, cap);
        t.ph = CH_ALLOC(ctx, int32_t, cap);
        t.ly = CH_ALLOC(ctx, int32_t, cap);
        t.op = CH_ALLOC(ctx, int32_t, cap);
        t.label = CH_ALLOC(ctx, int32_t, cap);
        t.rank = CH_ALLOC(ctx, int32_t, cap);
        t.first_pred = CH_ALLOC(ctx, int64_t, cap);
    }
    CH_ALLOC_END(ctx);
    return CHOPPER_OK;
}

// group the n sorted children (keys via perm) by key >> shift; returns group starts (device) and count
static chopper_status group(chopper_ctx *ctx, const unsigned long long *keys_sorted, int64_t n, int shift,
                            int64_t **starts_out, int64_t *ng_out) {
    CH_ALLOC_BEGIN;
    int64_t *head = CH_ALLOC(ctx, int64_t, n + 1);
    int64_t *ex = CH_ALLOC(ctx, int64_t, n + 1);
    int64_t *starts = CH_ALLOC(ctx, int64_t, n + 2);
    unsigned long long *nv = CH_ALLOC(ctx, unsigned long long, 1);
    int64_t *tot = CH_ALLOC(ctx, int64_t, 1);
    CH_ALLOC_END(ctx);
    unsigned long long init = (unsigned long long)n;
    CH_CUDA(ctx, cudaMemcpyAsync(nv, &init, 8, cudaMemcpyHostToDevice, ctx->st));
    if (n > 0) {
        k_group_heads<<<(unsigned)ceil_div(n, NT), NT, 0, ctx->st>>>(keys_sorted, n, shift, head, nv);
        CH_LAUNCHED(ctx);
        CH_TRY(ch_scan_excl_i64(ctx, head, ex, n, tot));
        k_group_starts<<<(unsigned)ceil_div(n, NT), NT, 0, ctx->st>>>(head, ex, n, starts);
        CH_LAUNCHED(ctx);
    }
    int64_t ng = 0;
    unsigned long long hv = init;
    if (n > 0) CH_CUDA(ctx, cudaMemcpyAsync(&ng, tot, 8, cudaMemcpyDeviceToHost, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(&hv, nv, 8, cudaMemcpyDeviceToHost, ctx->st));
    CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    int64_t nvalid = (int64_t)hv;
    CH_CUDA(ctx, cudaMemcpyAsync(starts + ng, &nvalid, 8, cudaMemcpyHostToDevice, ctx->st));
    CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    *starts_out = starts;
    *ng_out = ng;
    return CHOPPER_OK;
}

static TabView view(RowTable &t) { return TabView{t.key, t.f, t.cnt, t.cap, t.cap, 1}; }

static chopper_status rollup(chopper_ctx *ctx, RowTable &child, RowTable &parent, int shift, int depth,
                             const KeyLayout &L, int32_t *lg_gpu_d) {
    int64_t *starts;
    int64_t ng;
    CH_TRY(group(ctx, child.key, child.n, shift, &starts, &ng));
    CH_TRY(alloc_table(ctx, parent, std::max<int64_t>(ng, 1), ctx->C, true));
    parent.n = ng;
    if (ng > 0) {
        k_sum_rows<<<(unsigned)ceil_div(ng, NT), NT, 0, ctx->st>>>(view(child), nullptr, starts, ng, shift, ctx->C,
                                                                   view(parent));
        CH_LAUNCHED(ctx);
        k_decode<<<(unsigned)ceil_div(ng, NT), NT, 0, ctx->st>>>(parent.key, ng, L, depth, lg_gpu_d, ctx->d_list_beg,
                                                                 ctx->P_orig, ctx->P_label, parent.f, parent.cap,
                                                                 ctx->d_pred_end, parent.gpu, parent.it, parent.ph,
                                                                 parent.ly, parent.op, parent.label, parent.rank,
                                                                 parent.first_pred);
        CH_LAUNCHED(ctx);
    }
    return CHOPPER_OK;
}

chopper_status ch_tables(chopper_ctx *ctx) {
    const int C = ctx->C;
    const int64_t R = ctx->R;
    KeyLayout L;
    L.kb[0] = ctx->kb[0]; L.kb[1] = ctx->kb[1]; L.kb[2] = ctx->kb[2]; L.kb[3] = ctx->kb[3];
    L.sh_op = 0;
    L.sh_ly = L.kb[3];
    L.sh_ph = L.sh_ly + L.kb[2];
    L.sh_it = L.sh_ph + L.kb[1];
    L.sh_lg = L.sh_it + L.kb[0];
    const int key_bits = L.sh_lg + ctx->kg;
    CH_ALLOC_BEGIN;
    int32_t *lg_gpu_d = CH_ALLOC(ctx, int32_t, ctx->n_lg + 1);
    ctx->sub.cnt = CH_ALLOC(ctx, double, (int64_t)(C > 0 ? C : 1) * std::max<int64_t>(R, 1));
    CH_ALLOC_END(ctx);
    {
        std::vector<int32_t> h(ctx->lg_gpu, ctx->lg_gpu + ctx->n_lg);
        if (ctx->n_lg) CH_CUDA(ctx, cudaMemcpyAsync(lg_gpu_d, h.data(), 4 * ctx->n_lg, cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    }
    ctx->sub.cap = std::max<int64_t>(R, 1);
    // sub-run fields were written with capacity N; re-point the table view at that layout
    TabView subv{ctx->sub.key, ctx->sub.f, ctx->sub.cnt, 1, std::max<int64_t>(R, 1), 16};   // AoS sub-run rows
    if (C > 0 && R > 0) {
        for (int s0 = 0; s0 < C; s0 += CT_SG) {
            k_counters_tiled<<<(unsigned)ceil_div(ctx->N, CT_TILE), CT_NT, 0, ctx->st>>>(
                ctx->ev.meta, ctx->d_run_id, ctx->d_nm_rank, ctx->d_gpu_lg, ctx->d_col, C, s0, ctx->N, subv.cnt,
                subv.ccap);
            CH_LAUNCHED(ctx);
        }
    }
    // instances: stable sort of sub-runs by key, then group equal keys
    unsigned long long *k1 = CH_ALLOC(ctx, unsigned long long, R + 1), *k2 = CH_ALLOC(ctx, unsigned long long, R + 1);
    uint32_t *v1 = CH_ALLOC(ctx, uint32_t, R + 1), *v2 = CH_ALLOC(ctx, uint32_t, R + 1);
    CH_ALLOC_END(ctx);
    if (R > 0) {
        k_copy_keys<<<(unsigned)ceil_div(R, NT), NT, 0, ctx->st>>>(ctx->sub.key, R, k1, v1);
        CH_LAUNCHED(ctx);
    }
    bool alt = false;
    CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, R, 0, key_bits, &alt));
    unsigned long long *ks = alt ? k2 : k1;
    uint32_t *so = alt ? v2 : v1;
    {
        int64_t *starts;
        int64_t ng;
        CH_TRY(group(ctx, ks, R, 0, &starts, &ng));
        CH_TRY(alloc_table(ctx, ctx->inst, std::max<int64_t>(ng, 1), C, true));
        ctx->inst.n = ng;
        if (ng > 0) {
            k_sum_rows<<<(unsigned)ceil_div(ng, NT), NT, 0, ctx->st>>>(subv, so, starts, ng, 0, C, view(ctx->inst));
            CH_LAUNCHED(ctx);
            k_decode<<<(unsigned)ceil_div(ng, NT), NT, 0, ctx->st>>>(
                ctx->inst.key, ng, L, 4, lg_gpu_d, ctx->d_list_beg, ctx->P_orig, ctx->P_label, ctx->inst.f,
                ctx->inst.cap, ctx->d_pred_end, ctx->inst.gpu, ctx->inst.it, ctx->inst.ph, ctx->inst.ly, ctx->inst.op,
                ctx->inst.label, ctx->inst.rank, ctx->inst.first_pred);
            CH_LAUNCHED(ctx);
        }
    }
    // roll-ups (D12)
    CH_TRY(rollup(ctx, ctx->inst, ctx->layer, L.sh_ly, 3, L, lg_gpu_d));
    CH_TRY(rollup(ctx, ctx->layer, ctx->phase, L.sh_ph, 2, L, lg_gpu_d));
    CH_TRY(rollup(ctx, ctx->phase, ctx->iter, L.sh_it, 1, L, lg_gpu_d));
    CH_TRY(rollup(ctx, ctx->iter, ctx->gpurow, L.sh_lg, 0, L, lg_gpu_d));
    // iteration extras
    {
        int64_t n = ctx->iter.n;
        int64_t cap = std::max<int64_t>(n, 1);
        ctx->iter_wall = CH_ALLOC(ctx, int64_t, cap);
        ctx->iter_cu = CH_ALLOC(ctx, int64_t, cap);
        ctx->iter_af = CH_ALLOC(ctx, int64_t, cap);
        ctx->iter_al = CH_ALLOC(ctx, int64_t, cap);
        ctx->iter_step = CH_ALLOC(ctx, int32_t, cap);
        CH_ALLOC_END(ctx);
        if (n > 0) {
            k_iter_extras<<<(unsigned)ceil_div(n, NT), NT, 0, ctx->st>>>(
                n, ctx->iter.f, ctx->iter.cap, ctx->iter.gpu, ctx->iter.it, ctx->iter.first_pred, ctx->d_gpu_lg,
                ctx->sp.label, ctx->U_s, ctx->U_e, ctx->U_P, ctx->d_U_beg, ctx->d_U_cnt, ctx->d_delta, ctx->iter_wall,
                ctx->iter_cu, ctx->iter_af, ctx->iter_al, ctx->iter_step);
            CH_LAUNCHED(ctx);
        }
    }
    // points (label, gpu, iteration)
    {
        int64_t n = ctx->inst.n;
        int lbits = bits_for((uint64_t)std::max(ctx->cfg.n_labels, 1));
        int pbits = lbits + ctx->kg + L.kb[0];
        if (pbits > 63) return ch_fail(ctx, CHOPPER_E_RANGE, "point key exceeds 63 bits");
        unsigned long long *p1 = CH_ALLOC(ctx, unsigned long long, n + 1), *p2 = CH_ALLOC(ctx, unsigned long long, n + 1);
        uint32_t *q1 = CH_ALLOC(ctx, uint32_t, n + 1), *q2 = CH_ALLOC(ctx, uint32_t, n + 1);
        CH_ALLOC_END(ctx);
        if (n > 0) {
            k_point_keys<<<(unsigned)ceil_div(n, NT), NT, 0, ctx->st>>>(ctx->inst.key, n, L, ctx->d_list_beg,
                                                                        ctx->P_label, ctx->kg, p1, q1);
            CH_LAUNCHED(ctx);
        }
        bool a2 = false;
        CH_TRY(ch_radix_sort(ctx, p1, q1, p2, q2, n, 0, pbits, &a2));
        unsigned long long *pk = a2 ? p2 : p1;
        uint32_t *po = a2 ? q2 : q1;
        int64_t *starts;
        int64_t ng;
        CH_TRY(group(ctx, pk, n, 0, &starts, &ng));
        CH_TRY(alloc_table(ctx, ctx->point, std::max<int64_t>(ng, 1), C, true));
        ctx->point.n = ng;
        if (ng > 0) {
            // sum instance rows into points, key = point key of the first instance
            TabView iv = view(ctx->inst);
            TabView pv = view(ctx->point);
            k_sum_rows<<<(unsigned)ceil_div(ng, NT), NT, 0, ctx->st>>>(iv, po, starts, ng, 64, C, pv);
            CH_LAUNCHED(ctx);
            // point keys: the sorted point keys at the group starts
            k_gather_keys<<<(unsigned)ceil_div(ng, NT), NT, 0, ctx->st>>>(pk, starts, ng, ctx->point.key);
            CH_LAUNCHED(ctx);
            k_decode_points<<<(unsigned)ceil_div(ng, NT), NT, 0, ctx->st>>>(
                ctx->point.key, ng, ctx->kg, L.kb[0], lg_gpu_d, ctx->d_list_beg, ctx->P_orig, ctx->point.f,
                ctx->point.cap, ctx->d_pred_end, ctx->point.gpu, ctx->point.it, ctx->point.ph, ctx->point.ly,
                ctx->point.op, ctx->point.label, ctx->point.rank, ctx->point.first_pred);
            CH_LAUNCHED(ctx);
        }
    }
    // derived ratio-of-sums rates
    if (ctx->n_ratios > 0) {
        RowTable *ts[2] = {&ctx->point, &ctx->iter};
        for (RowTable *t : ts) {
            t->rates = CH_ALLOC(ctx, double, (int64_t)ctx->n_ratios * std::max<int64_t>(t->n, 1));
            CH_ALLOC_END(ctx);
            if (t->n > 0) {
                k_rates<<<(unsigned)ceil_div(t->n, NT), NT, 0, ctx->st>>>(t->n, t->f, t->cnt, t->cap, ctx->n_ratios,
                                                                          ctx->d_ratio, ctx->d_ratio + ctx->n_ratios,
                                                                          ctx->d_ratio_scale, t->rates);
                CH_LAUNCHED(ctx);
            }
        }
    }
    CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return CHOPPER_OK;
}
