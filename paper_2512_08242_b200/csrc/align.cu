// align.cu -- a3 counter alignment and a4 cross-GPU clock offsets (chopper_align).
//
// a3 (D2): every counter pass of
//   gpu g enumerates g's non-MEMOP kernels in dispatch order.  The name-id
//   sequence must match exactly (first divergence -> CHOPPER_E_ALIGNMENT);
//   counters then merge positionally: event i of gpu g takes value j = its
//   rank among g's non-MEMOP events.  A slot present in two passes must agree
//   within 1e-9 relative; the first pass wins.
// a4 (D13): E_{g,k}[j] = t_ke of the j-th class-k (AG, RS) event of gpu g in
//   dispatch order; the vectors of all traced GPUs are all-gathered (NCCL #1)
//   and delta_g = lower median over (k, j < m_k) of E_{g,k}[j] - E_{ref,k}[j],
//   ref = lowest traced gpu, via an in-block radix select.
#include <dlfcn.h>

#include "common.cuh"

namespace {
constexpr int NT = 256;


// name-sequence check of every pass of the event's gpu
__global__ void k_pass_check(const uint32_t *__restrict__ meta, const int32_t *__restrict__ name_id, int64_t n,
                             const int32_t *__restrict__ gpu_lg, const int32_t *__restrict__ nm_rank,
                             const PassDesc *__restrict__ passes, const int32_t *__restrict__ pass_off,
                             const int32_t *__restrict__ pass_idx, unsigned long long *__restrict__ mis) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t m = meta[i];
    if (kind_of(m) == CK_MEMOP) return;
    int lg = gpu_lg[gpu_of(m)];
    int64_t j = nm_rank[i];
    int32_t nm = name_id[i];
    for (int q = pass_off[lg]; q < pass_off[lg + 1]; q++) {
        int p = pass_idx[q];
        if (j < passes[p].n && passes[p].name_id[j] != nm) atomicMin(&mis[p], (unsigned long long)j);
    }
}

// non-finite values in any pass (blockIdx.y = pass): streaming read, 4 doubles per thread step
__global__ void k_pass_finite(const PassDesc *__restrict__ passes, unsigned int *__restrict__ bad) {
    const int p = blockIdx.y;
    const PassDesc d = passes[p];
    const int64_t tot = d.n * d.k;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool ok = true;
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; x + 3 * stride < tot; x += 4 * stride) {
        double a = d.values[x], b = d.values[x + stride], c = d.values[x + 2 * stride], e = d.values[x + 3 * stride];
        ok &= isfinite(a) && isfinite(b) && isfinite(c) && isfinite(e);
    }
    for (; x < tot; x += stride) ok &= (bool)isfinite(d.values[x]);
    if (__any_sync(CH_FULL, !ok) && lane_id() == 0) atomicOr(&bad[p], 1u);
}

// values of the same slot from two passes must agree within 1e-9 relative
__global__ void k_pass_conflict(const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                                unsigned long long *__restrict__ conf) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        double x = a[j], y = b[j];
        if (fabs(x - y) > 1e-9 * fmax(fabs(x), fabs(y))) atomicMin(conf, (unsigned long long)j);
    }
}

__global__ void k_counters_out(const uint32_t *__restrict__ meta, int64_t n, const int32_t *__restrict__ gpu_lg,
                               const int32_t *__restrict__ nm_rank, const double *const *__restrict__ col, int C,
                               double *__restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t m = meta[i];
    int lg = gpu_lg[gpu_of(m)];
    bool mem = kind_of(m) == CK_MEMOP;
    int64_t j = nm_rank[i];
    for (int s = 0; s < C; s++) {
        const double *c = col[lg * C + s];
        out[(int64_t)s * n + i] = (c && !mem) ? c[j] : 0.0;
    }
}

// ---- per-gpu ranks from meta: non-MEMOP (counter-pass position), AG and RS (collective index) -------
// tile = 2048 events; counts of the three predicates packed 21 bits apart
constexpr int MR_NT = 256, MR_IPT = 8, MR_TILE = MR_NT * MR_IPT;
__device__ __forceinline__ unsigned long long pred3(uint32_t m) {
    int k = kind_of(m);
    return (k != CK_MEMOP ? 1ull : 0ull) | (k == CK_AG ? 1ull << 21 : 0ull) | (k == CK_RS ? 1ull << 42 : 0ull);
}
__global__ void __launch_bounds__(MR_NT) k_meta_tiles(const uint32_t *__restrict__ meta, int64_t n,
                                                      int64_t *__restrict__ tc, int64_t ntile) {
    __shared__ int64_t sm[33];
    int64_t i0 = (int64_t)blockIdx.x * MR_TILE + (int64_t)threadIdx.x * MR_IPT;
    unsigned long long c = 0;
    for (int k = 0; k < MR_IPT; k++)
        if (i0 + k < n) c += pred3(meta[i0 + k]);
    int64_t tot;
    block_excl_sum<MR_NT>((int64_t)c, &tot, sm);
    if (threadIdx.x == 0) {
        unsigned long long t = (unsigned long long)tot;
        tc[blockIdx.x] = (int64_t)(t & 0x1FFFFF);
        tc[ntile + blockIdx.x] = (int64_t)((t >> 21) & 0x1FFFFF);
        tc[2 * ntile + blockIdx.x] = (int64_t)(t >> 42);
    }
}
// base[c][lg] = global exclusive count of predicate c at the gpu's first event (lg = n_lg -> N);
// also writes the exchange header (gpu, present, #AG, #RS) of every local gpu
__global__ void k_gpu_bases(const uint32_t *__restrict__ meta, int64_t n, const int64_t *__restrict__ tex,
                            int64_t ntile, const int64_t *__restrict__ gbeg, int n_lg, int64_t *__restrict__ base,
                            const int32_t *__restrict__ lg_gpu, int64_t *__restrict__ xsend, int64_t W) {
    int t = threadIdx.x;
    if (t < 3 * (n_lg + 1)) {
        int c = t / (n_lg + 1), lg = t % (n_lg + 1);
        int64_t pos = gbeg[lg];
        int64_t tile = pos / MR_TILE;
        int64_t b = 0;
        if (tile < ntile) {
            b = tex[c * ntile + tile];
            for (int64_t i = tile * MR_TILE; i < pos; i++) b += (int64_t)((pred3(meta[i]) >> (21 * c)) & 0x1FFFFF);
        } else {
            b = tex[c * ntile + ntile - 1];
            for (int64_t i = (ntile - 1) * MR_TILE; i < n; i++) b += (int64_t)((pred3(meta[i]) >> (21 * c)) & 0x1FFFFF);
        }
        base[c * (n_lg + 1) + lg] = b;
    }
    __syncthreads();
    if (t < n_lg && xsend) {
        int64_t *h = xsend + (int64_t)t * W;
        h[0] = lg_gpu[t];
        h[1] = 1;
        h[2] = base[1 * (n_lg + 1) + t + 1] - base[1 * (n_lg + 1) + t];
        h[3] = base[2 * (n_lg + 1) + t + 1] - base[2 * (n_lg + 1) + t];
    }
}
__global__ void __launch_bounds__(MR_NT) k_meta_apply(const uint32_t *__restrict__ meta, const int64_t *__restrict__ ks,
                                                      const int64_t *__restrict__ ke, int64_t n,
                                                      const int32_t *__restrict__ gpu_lg, const int64_t *__restrict__ tex,
                                                      int64_t ntile, const int64_t *__restrict__ base, int n_lg,
                                                      int32_t *__restrict__ nm_rank, int64_t *__restrict__ xsend,
                                                      int64_t K, int64_t W, unsigned int *__restrict__ ovf) {
    __shared__ int64_t sm[33];
    int64_t i0 = (int64_t)blockIdx.x * MR_TILE + (int64_t)threadIdx.x * MR_IPT;
    uint32_t mm[MR_IPT];
    unsigned long long c = 0;
#pragma unroll
    for (int k = 0; k < MR_IPT; k++) {
        mm[k] = i0 + k < n ? meta[i0 + k] : (uint32_t)CK_MEMOP;
        if (i0 + k < n) c += pred3(mm[k]);
    }
    int64_t tot;
    unsigned long long ex = (unsigned long long)block_excl_sum<MR_NT>((int64_t)c, &tot, sm);
    int64_t r0 = tex[blockIdx.x] + (int64_t)(ex & 0x1FFFFF);
    int64_t r1 = tex[ntile + blockIdx.x] + (int64_t)((ex >> 21) & 0x1FFFFF);
    int64_t r2 = tex[2 * ntile + blockIdx.x] + (int64_t)(ex >> 42);
#pragma unroll
    for (int k = 0; k < MR_IPT; k++) {
        int64_t i = i0 + k;
        if (i >= n) break;
        uint32_t m = mm[k];
        int lg = gpu_lg[gpu_of(m)];
        int kd = kind_of(m);
        nm_rank[i] = (int32_t)(r0 - base[lg]);
        if (kd == CK_AG || kd == CK_RS) {
            int64_t j = kd == CK_AG ? r1 - base[(n_lg + 1) + lg] : r2 - base[2 * (n_lg + 1) + lg];
            if (j >= K) atomicOr(ovf, 1u);
            else if (xsend) {
                int64_t *b = xsend + (int64_t)lg * W + 4 + (kd == CK_AG ? 0 : 2 * K);
                b[j] = ks[i];
                b[K + j] = ke[i];
            }
        }
        if (kd != CK_MEMOP) r0++;
        if (kd == CK_AG) r1++;
        if (kd == CK_RS) r2++;
    }
}



// one block per gathered gpu slot: lower median of collective-end differences (radix select)
__global__ void __launch_bounds__(256) k_delta(const int64_t *__restrict__ all, int nslots, int64_t W, int64_t K,
                                               int64_t *__restrict__ delta, int32_t *__restrict__ dflag) {
    __shared__ unsigned int hist[256];
    __shared__ int s_ref;
    __shared__ int64_t s_m[2];
    __shared__ unsigned long long s_prefix;
    __shared__ int64_t s_k;
    const int64_t *me = all + (int64_t)blockIdx.x * W;
    if (me[1] == 0) return;
    int g = (int)me[0];
    if (threadIdx.x == 0) {
        int ref = -1, refg = 1 << 30;
        int64_t m0 = -1, m1 = -1;
        for (int b = 0; b < nslots; b++) {
            const int64_t *x = all + (int64_t)b * W;
            if (x[1] == 0) continue;
            if ((int)x[0] < refg) { refg = (int)x[0]; ref = b; }
            if (m0 < 0 || x[2] < m0) m0 = x[2];
            if (m1 < 0 || x[3] < m1) m1 = x[3];
        }
        s_ref = ref;
        s_m[0] = m0 < 0 ? 0 : m0;
        s_m[1] = m1 < 0 ? 0 : m1;
    }
    __syncthreads();
    const int64_t *rf = all + (int64_t)s_ref * W;
    int64_t m0 = s_m[0], m1 = s_m[1], nd = m0 + m1;
    if (nd == 0) {
        if (threadIdx.x == 0) { delta[g] = 0; dflag[g] = 1; }
        return;
    }
    auto dval = [&](int64_t q) -> unsigned long long {
        int64_t d;
        if (q < m0) d = me[4 + K + q] - rf[4 + K + q];
        else d = me[4 + 3 * K + (q - m0)] - rf[4 + 3 * K + (q - m0)];
        return enc_i64(d);
    };
    if (threadIdx.x == 0) { s_prefix = 0; s_k = (nd - 1) / 2; }
    __syncthreads();
    for (int byte = 7; byte >= 0; byte--) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        unsigned long long pre = s_prefix;
        unsigned long long hmask = byte == 7 ? 0ull : (~0ull << (8 * (byte + 1)));
        for (int64_t q = threadIdx.x; q < nd; q += blockDim.x) {
            unsigned long long v = dval(q);
            if ((v & hmask) == (pre & hmask)) atomicAdd(&hist[(v >> (8 * byte)) & 0xFF], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t k = s_k;
            int d = 0;
            for (; d < 256; d++) {
                if (k < (int64_t)hist[d]) break;
                k -= hist[d];
            }
            s_k = k;
            s_prefix = pre | ((unsigned long long)d << (8 * byte));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { delta[g] = dec_i64(s_prefix); dflag[g] = 0; }
}

__global__ void k_skew(const int64_t *__restrict__ all, int nslots, int64_t W, int64_t K,
                       const int64_t *__restrict__ delta, unsigned long long *__restrict__ maxskew) {
    __shared__ int64_t s_m[2];
    if (threadIdx.x == 0) {
        int64_t m0 = -1, m1 = -1;
        for (int b = 0; b < nslots; b++) {
            const int64_t *x = all + (int64_t)b * W;
            if (x[1] == 0) continue;
            if (m0 < 0 || x[2] < m0) m0 = x[2];
            if (m1 < 0 || x[3] < m1) m1 = x[3];
        }
        s_m[0] = m0 < 0 ? 0 : m0;
        s_m[1] = m1 < 0 ? 0 : m1;
    }
    __syncthreads();
    for (int cls = 0; cls < 2; cls++) {
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < s_m[cls]; j += (int64_t)gridDim.x * blockDim.x) {
            int64_t lo = INT64_MAX, hi = INT64_MIN;
            for (int b = 0; b < nslots; b++) {
                const int64_t *x = all + (int64_t)b * W;
                if (x[1] == 0) continue;
                int64_t a = x[4 + 2 * K * cls + j] - delta[x[0]];
                lo = a < lo ? a : lo;
                hi = a > hi ? a : hi;
            }
            atomicMax(&maxskew[cls], (unsigned long long)(hi - lo));
        }
    }
}
}  // namespace

chopper_status ch_nccl_allgather(chopper_ctx *ctx, const void *send, void *recv, size_t bytes_per_rank) {
    typedef int (*fn_t)(const void *, void *, size_t, int, void *, cudaStream_t);
    static fn_t fn = nullptr;
    if (!fn) {
        fn = (fn_t)dlsym(RTLD_DEFAULT, "ncclAllGather");
        if (!fn) {
            void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (h) fn = (fn_t)dlsym(h, "ncclAllGather");
        }
        if (!fn) return ch_fail(ctx, CHOPPER_E_NCCL, "ncclAllGather not found (load torch's NCCL first)");
    }
    int r = fn(send, recv, bytes_per_rank, /*ncclInt8*/ 0, ctx->nccl, ctx->st);
    if (r != 0) return ch_fail(ctx, CHOPPER_E_NCCL, "ncclAllGather failed: " + std::to_string(r));
    return CHOPPER_OK;
}

chopper_status ch_align(chopper_ctx *ctx, const chopper_counter_pass *passes, int32_t n_passes, int32_t n_counters,
                        double *counters_out) {
    const int64_t N = ctx->N;
    const int n_lg = ctx->n_lg, C = n_counters;
    ctx->C = C;
    ctx->passes.clear();
    std::vector<std::vector<int>> by_lg(n_lg);
    for (int p = 0; p < n_passes; p++) {
        const chopper_counter_pass &q = passes[p];
        int lg = (q.gpu >= 0 && q.gpu < CH_MAX_GPUS) ? ctx->gpu_lg_h[q.gpu] : -1;
        if (lg < 0) return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "counter pass for a gpu without events on this rank");
        for (int kk = 0; kk < q.k; kk++)
            if (q.slot[kk] < 0 || q.slot[kk] >= C) return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "counter slot out of range");
        ctx->passes.push_back(PassDesc{q.name_id, q.values, q.n, q.k, lg});
        by_lg[lg].push_back(p);
    }
    CH_ALLOC_BEGIN;
    ctx->d_nm_rank = CH_ALLOC(ctx, int32_t, N);
    ctx->d_passes = CH_ALLOC(ctx, PassDesc, n_passes + 1);
    ctx->d_present = CH_ALLOC(ctx, int32_t, (int64_t)n_lg * (C > 0 ? C : 1));
    const double **col = CH_ALLOC(ctx, const double *, (int64_t)n_lg * (C > 0 ? C : 1));
    int64_t *dgbeg = CH_ALLOC(ctx, int64_t, n_lg + 1);
    CH_ALLOC_END(ctx);
    ctx->present.assign((size_t)n_lg * (C > 0 ? C : 1), 0);
    std::vector<const double *> hcol((size_t)n_lg * (C > 0 ? C : 1), nullptr);
    CH_CUDA(ctx, cudaMemcpyAsync(dgbeg, ctx->g_beg, 8 * (n_lg + 1), cudaMemcpyHostToDevice, ctx->st));
    // clock-offset exchange block of this rank (filled by the rank pass, consumed by ch_offsets)
    {
        const int64_t K = std::max(1, ctx->cfg.max_coll_per_class);
        ctx->xW = 4 + 4 * K;
        ctx->xslots = (int)ceil_div(ctx->cfg.n_traced_gpus, ctx->nranks);
        if (n_lg > ctx->xslots) return ch_fail(ctx, CHOPPER_E_RANGE, "more local gpus than ceil(n_traced_gpus / nranks)");
        ctx->d_xsend = CH_ALLOC(ctx, int64_t, (int64_t)ctx->xslots * ctx->xW);
        ctx->d_xovf = CH_ALLOC(ctx, unsigned int, 1);
        CH_ALLOC_END(ctx);
        CH_CUDA(ctx, cudaMemsetAsync(ctx->d_xsend, 0, 8 * (size_t)ctx->xslots * ctx->xW, ctx->st));
        CH_CUDA(ctx, cudaMemsetAsync(ctx->d_xovf, 0, 4, ctx->st));
    }
    if (N > 0 && n_lg > 0) {
        // one tile-count pass and one apply pass over meta: non-MEMOP rank (counter-pass position, D2),
        // AG / RS collective index (D13) written straight into the exchange block
        const int64_t K = ctx->xW / 4 - 1;
        int64_t ntile = ceil_div(N, MR_TILE);
        size_t mark = ctx->used;
        int64_t *tc = CH_ALLOC(ctx, int64_t, 3 * ntile), *tex = CH_ALLOC(ctx, int64_t, 3 * ntile);
        int64_t *base = CH_ALLOC(ctx, int64_t, 3 * (n_lg + 1));
        int32_t *dlg = CH_ALLOC(ctx, int32_t, n_lg + 1);
        CH_ALLOC_END(ctx);
        std::vector<int32_t> hlg(ctx->lg_gpu, ctx->lg_gpu + n_lg);
        CH_CUDA(ctx, cudaMemcpyAsync(dlg, hlg.data(), 4 * n_lg, cudaMemcpyHostToDevice, ctx->st));
        k_meta_tiles<<<(unsigned)ntile, MR_NT, 0, ctx->st>>>(ctx->ev.meta, N, tc, ntile);
        CH_LAUNCHED(ctx);
        for (int c = 0; c < 3; c++) CH_TRY(ch_scan_excl_i64(ctx, tc + c * ntile, tex + c * ntile, ntile, nullptr));
        k_gpu_bases<<<1, 3 * (n_lg + 1) > 32 ? 3 * (n_lg + 1) : 32, 0, ctx->st>>>(
            ctx->ev.meta, N, tex, ntile, dgbeg, n_lg, base, dlg, ctx->d_xsend, ctx->xW);
        CH_LAUNCHED(ctx);
        k_meta_apply<<<(unsigned)ntile, MR_NT, 0, ctx->st>>>(ctx->ev.meta, ctx->ev.start_ns, ctx->ev.end_ns, N,
                                                             ctx->d_gpu_lg, tex, ntile, base, n_lg, ctx->d_nm_rank,
                                                             ctx->d_xsend, K, ctx->xW, ctx->d_xovf);
        CH_LAUNCHED(ctx);
        std::vector<int64_t> hb(3 * (n_lg + 1));
        CH_CUDA(ctx, cudaMemcpyAsync(hb.data(), base, 8 * hb.size(), cudaMemcpyDeviceToHost, ctx->st));
        CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
        ctx->used = mark;
        std::vector<int64_t> m_g(n_lg);
        for (int l = 0; l < n_lg; l++) m_g[l] = hb[l + 1] - hb[l];

        if (n_passes > 0) {
            std::vector<int32_t> off(n_lg + 1, 0), idx;
            for (int l = 0; l < n_lg; l++) {
                off[l] = (int32_t)idx.size();
                for (int p : by_lg[l]) idx.push_back(p);
            }
            off[n_lg] = (int32_t)idx.size();
            int32_t *doff = CH_ALLOC(ctx, int32_t, n_lg + 1), *didx = CH_ALLOC(ctx, int32_t, n_passes);
            unsigned long long *mis = CH_ALLOC(ctx, unsigned long long, n_passes);
            unsigned int *bad = CH_ALLOC(ctx, unsigned int, n_passes);
            unsigned long long *conf = CH_ALLOC(ctx, unsigned long long, n_passes);
            CH_ALLOC_END(ctx);
            CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_passes, ctx->passes.data(), sizeof(PassDesc) * n_passes,
                                         cudaMemcpyHostToDevice, ctx->st));
            CH_CUDA(ctx, cudaMemcpyAsync(doff, off.data(), 4 * (n_lg + 1), cudaMemcpyHostToDevice, ctx->st));
            CH_CUDA(ctx, cudaMemcpyAsync(didx, idx.data(), 4 * n_passes, cudaMemcpyHostToDevice, ctx->st));
            CH_TRY(ch_fill_u64(ctx, mis, n_passes, ~0ull));
            CH_TRY(ch_fill_u64(ctx, conf, n_passes, ~0ull));
            CH_CUDA(ctx, cudaMemsetAsync(bad, 0, 4 * n_passes, ctx->st));
            k_pass_check<<<(unsigned)ceil_div(N, NT), NT, 0, ctx->st>>>(ctx->ev.meta, ctx->ev.name_id, N, ctx->d_gpu_lg,
                                                                        ctx->d_nm_rank, ctx->d_passes, doff, didx, mis);
            CH_LAUNCHED(ctx);
            k_pass_finite<<<dim3(148 * 2, n_passes), NT, 0, ctx->st>>>(ctx->d_passes, bad);
            CH_LAUNCHED(ctx);
            std::vector<unsigned long long> hmis(n_passes);
            std::vector<unsigned int> hbad(n_passes);
            CH_CUDA(ctx, cudaMemcpyAsync(hmis.data(), mis, 8 * n_passes, cudaMemcpyDeviceToHost, ctx->st));
            CH_CUDA(ctx, cudaMemcpyAsync(hbad.data(), bad, 4 * n_passes, cudaMemcpyDeviceToHost, ctx->st));
            CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
            ctx->pass_mismatch.assign(n_passes, -1);
            ctx->pass_conflict.assign(n_passes, -1);
            // slot assignment: first valid pass wins; later passes checked for conflicts
            std::vector<std::pair<int, int>> first((size_t)n_lg * (C > 0 ? C : 1), {-1, -1});
            for (int p = 0; p < n_passes; p++) {
                const PassDesc &d = ctx->passes[p];
                int64_t mg = m_g[d.lg];
                int64_t lim = d.n < mg ? d.n : mg;
                int64_t mj = hmis[p] == ~0ull ? -1 : (int64_t)hmis[p];
                if (mj < 0 && d.n != mg) mj = lim;
                if (mj >= 0) {
                    ctx->pass_mismatch[p] = mj;
                    ctx->latched_host |= 1u << CHOPPER_E_ALIGNMENT;
                    continue;
                }
                if (hbad[p]) {
                    ctx->rep.val_count[CV_COUNTER_NONFINITE]++;
                    if (ctx->rep.val_first[CV_COUNTER_NONFINITE] < 0 || p < ctx->rep.val_first[CV_COUNTER_NONFINITE])
                        ctx->rep.val_first[CV_COUNTER_NONFINITE] = p;
                    ctx->latched_host |= 1u << CHOPPER_E_VALIDATION;
                    continue;
                }
                for (int kk = 0; kk < d.k; kk++) {
                    int s = passes[p].slot[kk];
                    auto &f0 = first[(size_t)d.lg * C + s];
                    if (f0.first < 0) {
                        f0 = {p, kk};
                        hcol[(size_t)d.lg * C + s] = d.values + (int64_t)kk * d.n;
                        ctx->present[(size_t)d.lg * C + s] = 1;
                    } else {
                        const PassDesc &a = ctx->passes[f0.first];
                        k_pass_conflict<<<64, NT, 0, ctx->st>>>(a.values + (int64_t)f0.second * a.n,
                                                                d.values + (int64_t)kk * d.n, d.n, conf + p);
                        CH_LAUNCHED(ctx);
                    }
                }
            }
            std::vector<unsigned long long> hconf(n_passes);
            CH_CUDA(ctx, cudaMemcpyAsync(hconf.data(), conf, 8 * n_passes, cudaMemcpyDeviceToHost, ctx->st));
            CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
            for (int p = 0; p < n_passes; p++)
                if (hconf[p] != ~0ull) {
                    ctx->pass_conflict[p] = (int64_t)hconf[p];
                    ctx->latched_host |= 1u << CHOPPER_E_ALIGNMENT;
                }
        }
    }
    if (C > 0) {
        CH_CUDA(ctx, cudaMemcpyAsync(col, hcol.data(), sizeof(double *) * hcol.size(), cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_present, ctx->present.data(), 4 * ctx->present.size(),
                                     cudaMemcpyHostToDevice, ctx->st));
    }
    ctx->d_col = col;
    if (counters_out && C > 0 && N > 0) {
        k_counters_out<<<(unsigned)ceil_div(N, NT), NT, 0, ctx->st>>>(ctx->ev.meta, N, ctx->d_gpu_lg, ctx->d_nm_rank, col,
                                                                      C, counters_out);
        CH_LAUNCHED(ctx);
    }
    CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return CHOPPER_OK;
}

chopper_status ch_offsets(chopper_ctx *ctx) {
    const int n_lg = ctx->n_lg, G = ctx->cfg.n_traced_gpus;
    const int64_t W = ctx->xW, K = W / 4 - 1;
    const int slots = ctx->xslots;
    (void)n_lg;
    CH_ALLOC_BEGIN;
    int64_t *all = CH_ALLOC(ctx, int64_t, (int64_t)slots * W * ctx->nranks);
    ctx->d_delta = CH_ALLOC(ctx, int64_t, G);
    ctx->d_delta_flag = CH_ALLOC(ctx, int32_t, G);
    unsigned long long *mskew = CH_ALLOC(ctx, unsigned long long, 2);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemsetAsync(ctx->d_delta, 0, 8 * G, ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(ctx->d_delta_flag, 0, 4 * G, ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(mskew, 0, 16, ctx->st));
    // NCCL all-gather #1: every rank's collective-end vectors (D13)
    if (ctx->nranks > 1) {
        CH_TRY(ch_nccl_allgather(ctx, ctx->d_xsend, all, sizeof(int64_t) * slots * W));
    } else {
        CH_CUDA(ctx, cudaMemcpyAsync(all, ctx->d_xsend, 8 * slots * W, cudaMemcpyDeviceToDevice, ctx->st));
    }
    int nslots = slots * ctx->nranks;
    k_delta<<<nslots, 256, 0, ctx->st>>>(all, nslots, W, K, ctx->d_delta, ctx->d_delta_flag);
    CH_LAUNCHED(ctx);
    k_skew<<<64, 256, 0, ctx->st>>>(all, nslots, W, K, ctx->d_delta, mskew);
    CH_LAUNCHED(ctx);
    ctx->delta.assign(G, 0);
    ctx->delta_flag.assign(G, 1);
    unsigned long long hs[2] = {0, 0};
    unsigned int hovf = 0;
    std::vector<int64_t> hdr(2 * (size_t)nslots);
    CH_CUDA(ctx, cudaMemcpyAsync(ctx->delta.data(), ctx->d_delta, 8 * G, cudaMemcpyDeviceToHost, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(ctx->delta_flag.data(), ctx->d_delta_flag, 4 * G, cudaMemcpyDeviceToHost, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(hs, mskew, 16, cudaMemcpyDeviceToHost, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(&hovf, ctx->d_xovf, 4, cudaMemcpyDeviceToHost, ctx->st));
    CH_CUDA(ctx, cudaMemcpy2DAsync(hdr.data(), 16, all, 8 * (size_t)W, 16, nslots, cudaMemcpyDeviceToHost, ctx->st));
    CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    // gpus absent from every rank keep flag 1 (no events)
    ctx->gpu_present.assign(G, 0);
    for (int b = 0; b < nslots; b++)
        if (hdr[2 * (size_t)b + 1]) ctx->gpu_present[hdr[2 * (size_t)b]] = 1;
    for (int g = 0; g < G; g++) if (!ctx->gpu_present[g]) { ctx->delta_flag[g] = 1; ctx->delta[g] = 0; }
    ctx->max_skew[0] = (int64_t)hs[0];
    ctx->max_skew[1] = (int64_t)hs[1];
    if (hovf) return ch_fail(ctx, CHOPPER_E_RANGE, "more collectives per class than max_coll_per_class");
    return CHOPPER_OK;
}
