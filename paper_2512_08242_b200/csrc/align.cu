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


constexpr int PC_MAXP = 256;           // counter passes per rank (staged in shared memory by the rank pass)

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
// a thread's 8 consecutive metas (two 16 B loads when whole and aligned; MEMOP past the end)
__device__ __forceinline__ void load_meta8(const uint32_t *__restrict__ meta, int64_t i0, int64_t n, uint32_t (&mm)[8]) {
    if (i0 + 8 <= n && (((uintptr_t)(meta + i0)) & 15u) == 0) {
        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(meta + i0)), b = __ldg(reinterpret_cast<const uint4 *>(meta + i0) + 1);
        mm[0] = a.x; mm[1] = a.y; mm[2] = a.z; mm[3] = a.w; mm[4] = b.x; mm[5] = b.y; mm[6] = b.z; mm[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < 8; k++) mm[k] = i0 + k < n ? meta[i0 + k] : (uint32_t)CK_MEMOP;
    }
}
__device__ __forceinline__ unsigned long long pred3(uint32_t m) {
    int k = kind_of(m);
    return (k != CK_MEMOP ? 1ull : 0ull) | (k == CK_AG ? 1ull << 21 : 0ull) | (k == CK_RS ? 1ull << 42 : 0ull);
}
__global__ void __launch_bounds__(MR_NT) k_meta_tiles(const uint32_t *__restrict__ meta, int64_t n,
                                                      int64_t *__restrict__ tc, int64_t ntile) {
    __shared__ int64_t sm[33];
    int64_t i0 = (int64_t)blockIdx.x * MR_TILE + (int64_t)threadIdx.x * MR_IPT;
    unsigned long long c = 0;
    uint32_t mm[MR_IPT];
    load_meta8(meta, i0, n, mm);
#pragma unroll
    for (int k = 0; k < MR_IPT; k++)
        if (i0 + k < n) c += pred3(mm[k]);
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
// non-MEMOP events per local gpu (the length of its counter columns)
__global__ void k_mg(const int64_t *__restrict__ base, int n_lg, int64_t *__restrict__ mg) {
    for (int l = threadIdx.x; l < n_lg; l += blockDim.x) mg[l] = base[l + 1] - base[l];
}

// one warp per (predicate, gpu boundary): tile prefix + the packed counts of the partial tile before it
__global__ void k_gpu_bases(const uint32_t *__restrict__ meta, int64_t n, const int64_t *__restrict__ tex,
                            int64_t ntile, const int64_t *__restrict__ gbeg, int n_lg, int64_t *__restrict__ base,
                            const int32_t *__restrict__ lg_gpu, int64_t *__restrict__ xsend, int64_t W) {
    const int w = threadIdx.x >> 5, l = lane_id();
    for (int job = w; job < 3 * (n_lg + 1); job += blockDim.x >> 5) {
        int c = job / (n_lg + 1), lg = job % (n_lg + 1);
        int64_t pos = gbeg[lg];
        int64_t tile = pos / MR_TILE;
        int64_t lo, hi, b;
        if (tile < ntile) { b = tex[c * ntile + tile]; lo = tile * MR_TILE; hi = pos; }
        else { b = tex[c * ntile + ntile - 1]; lo = (ntile - 1) * MR_TILE; hi = n; }
        int64_t part = 0;
        for (int64_t i = lo + l; i < hi; i += 32) part += (int64_t)((pred3(meta[i]) >> (21 * c)) & 0x1FFFFF);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(CH_FULL, part, o);
        if (l == 0) base[c * (n_lg + 1) + lg] = b + part;
    }
    __syncthreads();
    const int t = threadIdx.x;
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
                                                      int64_t K, int64_t W, unsigned int *__restrict__ ovf,
                                                      const int32_t *__restrict__ name_id,
                                                      const PassDesc *__restrict__ passes,
                                                      const int32_t *__restrict__ pass_off,
                                                      const int32_t *__restrict__ pass_idx, int n_passes,
                                                      unsigned long long *__restrict__ mis,
                                                      int32_t *__restrict__ t_nm) {
    __shared__ int64_t sm[33];
    __shared__ PassDesc sp[PC_MAXP];
    __shared__ int32_t soff[PC_MAXP + 1];
    int64_t i0 = (int64_t)blockIdx.x * MR_TILE + (int64_t)threadIdx.x * MR_IPT;
    uint32_t mm[MR_IPT];
    unsigned long long c = 0;
    if (n_passes > 0) {                  // (visible after block_excl_sum's barriers)
        for (int q = threadIdx.x; q < n_passes; q += MR_NT) sp[q] = passes[pass_idx[q]];
        for (int q = threadIdx.x; q <= n_lg; q += MR_NT) soff[q] = pass_off[q];
    }
    load_meta8(meta, i0, n, mm);
#pragma unroll
    for (int k = 0; k < MR_IPT; k++)
        if (i0 + k < n) c += pred3(mm[k]);
    int64_t tot;
    unsigned long long ex = (unsigned long long)block_excl_sum<MR_NT>((int64_t)c, &tot, sm);
    int64_t r0 = tex[blockIdx.x] + (int64_t)(ex & 0x1FFFFF);
    if (t_nm) t_nm[(int64_t)blockIdx.x * MR_NT + threadIdx.x] = (int32_t)r0;   // the counter pass's positions
    int64_t r1 = tex[ntile + blockIdx.x] + (int64_t)((ex >> 21) & 0x1FFFFF);
    int64_t r2 = tex[2 * ntile + blockIdx.x] + (int64_t)(ex >> 42);
    int32_t nr[MR_IPT];
    int gcur = -1, lg = 0;                // the gpu's local index and rank base, reloaded when the gpu changes
    int64_t b0 = 0;
#pragma unroll
    for (int k = 0; k < MR_IPT; k++) {
        int64_t i = i0 + k;
        if (i >= n) break;
        uint32_t m = mm[k];
        if (gpu_of(m) != gcur) {
            gcur = gpu_of(m);
            lg = gpu_lg[gcur];
            b0 = base[lg];
        }
        int kd = kind_of(m);
        nr[k] = (int32_t)(r0 - b0);
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
    if (n_passes > 0) {
        // a3 name-sequence check (D2): the pass entry at this event's rank must carry its name id
        int32_t nn[MR_IPT];
        if (i0 + MR_IPT <= n && (((uintptr_t)(name_id + i0)) & 15u) == 0) {
            const int4 a = reinterpret_cast<const int4 *>(name_id + i0)[0], b = reinterpret_cast<const int4 *>(name_id + i0)[1];
            nn[0] = a.x; nn[1] = a.y; nn[2] = a.z; nn[3] = a.w; nn[4] = b.x; nn[5] = b.y; nn[6] = b.z; nn[7] = b.w;
        } else {
#pragma unroll
            for (int k = 0; k < MR_IPT; k++) nn[k] = i0 + k < n ? name_id[i0 + k] : 0;
        }
        bool one_gpu = i0 + MR_IPT <= n;
#pragma unroll
        for (int k = 1; k < MR_IPT; k++) one_gpu &= gpu_of(mm[k]) == gpu_of(mm[0]);
        if (one_gpu) {                   // usual case: pass-outer, the thread's 8 name loads in flight together
            const int lg = gpu_lg[gpu_of(mm[0])];
            for (int q = soff[lg]; q < soff[lg + 1]; q++) {
                const PassDesc d = sp[q];
                int32_t got[MR_IPT];
#pragma unroll
                for (int k = 0; k < MR_IPT; k++)
                    got[k] = kind_of(mm[k]) != CK_MEMOP && nr[k] < d.n ? __ldg(d.name_id + nr[k]) : nn[k];
                int64_t bad = INT64_MAX;
#pragma unroll
                for (int k = MR_IPT - 1; k >= 0; k--)
                    if (got[k] != nn[k]) bad = nr[k];
                if (bad != INT64_MAX) atomicMin(&mis[pass_idx[q]], (unsigned long long)bad);
            }
        } else {
#pragma unroll
            for (int k = 0; k < MR_IPT; k++) {
                if (i0 + k >= n || kind_of(mm[k]) == CK_MEMOP) continue;
                const int lg = gpu_lg[gpu_of(mm[k])];
                const int64_t j = nr[k];
                for (int q = soff[lg]; q < soff[lg + 1]; q++) {
                    const PassDesc &d = sp[q];
                    if (j < d.n && __ldg(d.name_id + j) != nn[k]) atomicMin(&mis[pass_idx[q]], (unsigned long long)j);
                }
            }
        }
    }
    if (!nm_rank) return;                // no counters: the counter-pass positions are not needed
    if (i0 + MR_IPT <= n && (((uintptr_t)(nm_rank + i0)) & 15u) == 0) {
        reinterpret_cast<int4 *>(nm_rank + i0)[0] = make_int4(nr[0], nr[1], nr[2], nr[3]);
        reinterpret_cast<int4 *>(nm_rank + i0)[1] = make_int4(nr[4], nr[5], nr[6], nr[7]);
    } else {
#pragma unroll
        for (int k = 0; k < MR_IPT; k++)
            if (i0 + k < n) nm_rank[i0 + k] = nr[k];
    }
}



// one block per gathered gpu slot: lower median of collective-end differences (radix select)
// one 1024-thread block per gathered gpu slot: lower median of the collective-end differences by radix
// select on (d - min d): a min/max pass first, so only the bytes in which the differences vary are
// selected on (differences are microseconds: 2-3 passes instead of 8), with per-warp histograms.
constexpr int DL_NT = 1024, DL_W = DL_NT / 32;
__global__ void __launch_bounds__(DL_NT) k_delta(const int64_t *__restrict__ all, int nslots, int64_t W, int64_t K,
                                                 int64_t *__restrict__ delta, int32_t *__restrict__ dflag) {
    __shared__ unsigned int hist[DL_W][256];
    __shared__ int s_ref;
    __shared__ int64_t s_m[2];
    __shared__ unsigned long long s_prefix, s_lo[DL_W], s_hi[DL_W];
    __shared__ int64_t s_k;
    const int64_t *me = all + (int64_t)blockIdx.x * W;
    if (me[1] == 0) return;
    const int g = (int)me[0];
    const int w = threadIdx.x >> 5, l = lane_id();
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
    const int64_t m0 = s_m[0], m1 = s_m[1], nd = m0 + m1;
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
    // range of the (order-preserving encoded) differences
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t q = threadIdx.x; q < nd; q += DL_NT) {
        unsigned long long v = dval(q);
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a2 = __shfl_xor_sync(CH_FULL, lo, o), b2 = __shfl_xor_sync(CH_FULL, hi, o);
        lo = a2 < lo ? a2 : lo;
        hi = b2 > hi ? b2 : hi;
    }
    if (l == 0) { s_lo[w] = lo; s_hi[w] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a2 = ~0ull, b2 = 0ull;
        for (int x = 0; x < DL_W; x++) { a2 = s_lo[x] < a2 ? s_lo[x] : a2; b2 = s_hi[x] > b2 ? s_hi[x] : b2; }
        s_lo[0] = a2;
        s_hi[0] = b2;
        s_prefix = 0;
        s_k = (nd - 1) / 2;
    }
    __syncthreads();
    const unsigned long long vmin = s_lo[0], span = s_hi[0] - vmin;
    int top = 0;
    while (top < 8 && (span >> (8 * top)) != 0) top++;      // bytes of (v - vmin) that vary
    for (int byte = top - 1; byte >= 0; byte--) {
        for (int d = threadIdx.x; d < DL_W * 256; d += DL_NT) (&hist[0][0])[d] = 0;
        __syncthreads();
        const unsigned long long pre = s_prefix;
        const unsigned long long hmask = ~0ull << (8 * (byte + 1));
        for (int64_t q = threadIdx.x; q < nd; q += DL_NT) {
            unsigned long long v = dval(q) - vmin;
            if ((v & hmask) == (pre & hmask)) atomicAdd(&hist[w][(v >> (8 * byte)) & 0xFF], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 256) {        // fold the per-warp histograms
            unsigned int c = 0;
            for (int x = 0; x < DL_W; x++) c += hist[x][threadIdx.x];
            hist[0][threadIdx.x] = c;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t k = s_k;
            int d = 0;
            for (; d < 256; d++) {
                if (k < (int64_t)hist[0][d]) break;
                k -= hist[0][d];
            }
            s_k = k;
            s_prefix = pre | ((unsigned long long)d << (8 * byte));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { delta[g] = dec_i64(s_prefix + vmin); dflag[g] = 0; }
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
    if (ctx->ag_fn) {
        int32_t r = ctx->ag_fn(ctx->ag_user, send, recv, bytes_per_rank, ctx->rank, ctx->nranks, (void *)ctx->st);
        if (r != 0) return ch_fail(ctx, CHOPPER_E_NCCL, "all-gather transport failed: " + std::to_string(r));
        return CHOPPER_OK;
    }
    if (!ctx->nccl) return ch_fail(ctx, CHOPPER_E_NCCL, "nranks > 1 without an NCCL communicator or a transport");
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
    ctx->off_pending = false;
    ctx->passes.clear();
    ctx->pass_slots.clear();
    std::vector<std::vector<int>> by_lg(n_lg);
    for (int p = 0; p < n_passes; p++) {
        const chopper_counter_pass &q = passes[p];
        int lg = (q.gpu >= 0 && q.gpu < CH_MAX_GPUS) ? ctx->gpu_lg_h[q.gpu] : -1;
        if (lg < 0) return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "counter pass for a gpu without events on this rank");
        for (int kk = 0; kk < q.k; kk++)
            if (q.slot[kk] < 0 || q.slot[kk] >= C) return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "counter slot out of range");
        ctx->passes.push_back(PassDesc{q.name_id, q.values, q.n, q.k, lg});
        ctx->pass_slots.push_back(std::vector<int32_t>(q.slot, q.slot + q.k));
        by_lg[lg].push_back(p);
    }
    CH_ALLOC_BEGIN;
    // counter-pass positions (D2): per event only for the full-mode [C][N] output; the counter pass derives them
    // from the rank before each thread's first event (t_nm) and each gpu's first rank (nm_base)
    ctx->d_nm_rank = (C > 0 && counters_out) ? CH_ALLOC(ctx, int32_t, N) : nullptr;
    ctx->d_t_nm = C > 0 ? CH_ALLOC(ctx, int32_t, ceil_div(std::max<int64_t>(N, 1), MR_TILE) * MR_NT) : nullptr;
    ctx->d_nm_base = nullptr;
    ctx->d_passes = CH_ALLOC(ctx, PassDesc, n_passes + 1);
    int64_t *dgbeg = CH_ALLOC(ctx, int64_t, n_lg + 1);
    CH_ALLOC_END(ctx);
    ctx->d_conf = nullptr;
    ctx->h_col_dev = nullptr;
    ctx->d_present = nullptr;
    ctx->pass_mismatch.assign(n_passes, -1);
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
        ctx->d_mg = CH_ALLOC(ctx, int64_t, n_lg + 1);
        CH_ALLOC_END(ctx);
        static_assert(MR_TILE == 2048, "the lean a2's tile counts use 2048-event tiles");
        int64_t *tc = ctx->d_meta_tc ? ctx->d_meta_tc : CH_ALLOC(ctx, int64_t, 3 * ntile);
        int64_t *tex = CH_ALLOC(ctx, int64_t, 3 * ntile);
        int64_t *base = CH_ALLOC(ctx, int64_t, 3 * (n_lg + 1));
        ctx->d_nm_base = base;           // component 0: non-MEMOP rank of each local gpu's first event
        int32_t *dlg = CH_ALLOC(ctx, int32_t, n_lg + 1);
        CH_ALLOC_END(ctx);
        std::vector<int32_t> hlg(ctx->lg_gpu, ctx->lg_gpu + n_lg);
        CH_CUDA(ctx, cudaMemcpyAsync(dlg, hlg.data(), 4 * n_lg, cudaMemcpyHostToDevice, ctx->st));
        if (!ctx->d_meta_tc) {            // (the general a2 path: a count pass of its own)
            k_meta_tiles<<<(unsigned)ntile, MR_NT, 0, ctx->st>>>(ctx->ev.meta, N, tc, ntile);
            CH_LAUNCHED(ctx);
        }
        for (int c = 0; c < 3; c++) CH_TRY(ch_scan_excl_i64(ctx, tc + c * ntile, tex + c * ntile, ntile, nullptr));
        k_gpu_bases<<<1, 1024, 0, ctx->st>>>(
            ctx->ev.meta, N, tex, ntile, dgbeg, n_lg, base, dlg, ctx->d_xsend, ctx->xW);
        CH_LAUNCHED(ctx);
        // pass descriptors grouped by local gpu: the a3 name-sequence check runs inside the rank pass
        int32_t *doff = nullptr, *didx = nullptr;
        unsigned long long *mis = nullptr;
        if (n_passes > 0) {
            if (n_passes > PC_MAXP || n_lg > PC_MAXP) return ch_fail(ctx, CHOPPER_E_RANGE, "more than 256 counter passes");
            std::vector<int32_t> &off = ctx->h_pass_off, &idx = ctx->h_pass_idx;
            off.assign(n_lg + 1, 0);
            idx.clear();
            for (int l = 0; l < n_lg; l++) {
                off[l] = (int32_t)idx.size();
                for (int p : by_lg[l]) idx.push_back(p);
            }
            off[n_lg] = (int32_t)idx.size();
            doff = CH_ALLOC(ctx, int32_t, n_lg + 1);
            didx = CH_ALLOC(ctx, int32_t, n_passes);
            mis = CH_ALLOC(ctx, unsigned long long, n_passes);
            CH_ALLOC_END(ctx);
            CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_passes, ctx->passes.data(), sizeof(PassDesc) * n_passes,
                                         cudaMemcpyHostToDevice, ctx->st));
            CH_CUDA(ctx, cudaMemcpyAsync(doff, off.data(), 4 * (n_lg + 1), cudaMemcpyHostToDevice, ctx->st));
            CH_CUDA(ctx, cudaMemcpyAsync(didx, idx.data(), 4 * n_passes, cudaMemcpyHostToDevice, ctx->st));
            CH_TRY(ch_fill_u64(ctx, mis, n_passes, ~0ull));
        }
        g_marks.mark(ctx->st, "al_pre_rank");
        k_meta_apply<<<(unsigned)ntile, MR_NT, 0, ctx->st>>>(ctx->ev.meta, ctx->ev.start_ns, ctx->ev.end_ns, N,
                                                             ctx->d_gpu_lg, tex, ntile, base, n_lg, ctx->d_nm_rank,
                                                             ctx->d_xsend, K, ctx->xW, ctx->d_xovf, ctx->ev.name_id,
                                                             ctx->d_passes, doff, didx, n_passes, mis, ctx->d_t_nm);
        CH_LAUNCHED(ctx);
        k_mg<<<1, 256, 0, ctx->st>>>(base, n_lg, ctx->d_mg);
        CH_LAUNCHED(ctx);
        g_marks.mark(ctx->st, "al_rank");
        CH_TRY(ch_offsets_launch(ctx));                 // the exchange block is complete: a4 shares the read-back
        g_marks.mark(ctx->st, "al_offsets");

        if (n_passes > 0) {
            // one read-back: the name-sequence divergences and the per-gpu non-MEMOP counts
            std::vector<unsigned long long> hmis(n_passes);
            std::vector<int64_t> &m_g = ctx->h_mg;
            m_g.assign(n_lg, 0);
            CH_CUDA(ctx, ch_d2h(ctx, hmis.data(), mis, 8 * n_passes));
            CH_CUDA(ctx, ch_d2h(ctx, m_g.data(), ctx->d_mg, 8 * n_lg));
            CH_CUDA(ctx, ch_sync(ctx));
            ctx->pass_mismatch.assign(n_passes, -1);
            for (int p = 0; p < n_passes; p++) {
                const PassDesc &d = ctx->passes[p];
                int64_t mg = m_g[d.lg];
                int64_t lim = d.n < mg ? d.n : mg;
                int64_t mj = hmis[p] == ~0ull ? -1 : (int64_t)hmis[p];
                if (mj < 0 && d.n != mg) mj = lim;
                ctx->pass_mismatch[p] = mj;
            }
        }
    }
    // slot assignment, speculatively treating every name-matching pass as finite: the columns that feed
    // a slot are checked for finiteness by the counter pass itself (ch_tables), which then redoes the
    // assignment if one was not; name-matching passes with a column feeding no slot are checked here.
    ctx->pass_bad.assign(n_passes, 0);
    CH_TRY(ch_assign_slots(ctx));
    if (n_passes > 0) {
        ctx->d_pass_bad = CH_ALLOC(ctx, unsigned int, n_passes);
        CH_ALLOC_END(ctx);
        CH_CUDA(ctx, cudaMemsetAsync(ctx->d_pass_bad, 0, 4 * n_passes, ctx->st));
        bool any = false;
        for (int p = 0; p < n_passes; p++) any |= ctx->pass_mismatch[p] < 0 && !ctx->pass_covered[p];
        if (any) {
            // every pass gets a grid row; covered / mismatched ones exit at once
            std::vector<PassDesc> pd(ctx->passes);
            for (int p = 0; p < n_passes; p++)
                if (ctx->pass_mismatch[p] >= 0 || ctx->pass_covered[p]) pd[p].n = 0;
            PassDesc *dpd = CH_ALLOC(ctx, PassDesc, n_passes);
            CH_ALLOC_END(ctx);
            CH_CUDA(ctx, cudaMemcpyAsync(dpd, pd.data(), sizeof(PassDesc) * n_passes, cudaMemcpyHostToDevice, ctx->st));
            k_pass_finite<<<dim3(148 * 2, n_passes), NT, 0, ctx->st>>>(dpd, ctx->d_pass_bad);
            CH_LAUNCHED(ctx);
        }
    }
    ctx->counters_out = (counters_out && C > 0 && N > 0) ? counters_out : nullptr;
    CH_TRY(ch_counters_full(ctx));
    return CHOPPER_OK;
}

chopper_status ch_counters_full(chopper_ctx *ctx) {
    if (!ctx->counters_out) return CHOPPER_OK;
    k_counters_out<<<(unsigned)ceil_div(ctx->N, NT), NT, 0, ctx->st>>>(ctx->ev.meta, ctx->N, ctx->d_gpu_lg, ctx->d_nm_rank,
                                                                       ctx->d_col, ctx->C, ctx->counters_out);
    CH_LAUNCHED(ctx);
    return CHOPPER_OK;
}

// slot -> value column: in pass order, the first pass that matches the name sequence and is not known
// to be non-finite provides each slot (O3); later passes with the same slot are checked for conflicts.
chopper_status ch_assign_slots(chopper_ctx *ctx) {
    const int n_lg = ctx->n_lg, C = ctx->C;
    const int n_passes = (int)ctx->passes.size();
    const size_t nc = (size_t)std::max(n_lg, 1) * (C > 0 ? C : 1);
    ctx->present.assign(nc, 0);
    ctx->sel_pass.assign(nc, -1);
    ctx->pass_conflict.assign(n_passes, -1);
    ctx->pass_covered.assign(n_passes, 0);
    std::vector<int> sel_k(nc, -1);
    std::vector<const double *> hcol(nc, nullptr);
    if (!ctx->d_conf && n_passes > 0) {
        CH_ALLOC_BEGIN;
        ctx->d_conf = CH_ALLOC(ctx, unsigned long long, n_passes);
        CH_ALLOC_END(ctx);
    }
    if (n_passes > 0) CH_TRY(ch_fill_u64(ctx, ctx->d_conf, n_passes, ~0ull));
    bool conflicts = false;
    for (int p = 0; p < n_passes; p++) {
        const PassDesc &d = ctx->passes[p];
        if (ctx->pass_mismatch[p] >= 0 || ctx->pass_bad[p]) continue;
        int cov = 1;
        for (int kk = 0; kk < d.k; kk++) {
            int s = ctx->pass_slots[p][kk];
            size_t q = (size_t)d.lg * C + s;
            if (ctx->sel_pass[q] < 0) {
                ctx->sel_pass[q] = p;
                sel_k[q] = kk;
                hcol[q] = d.values + (int64_t)kk * d.n;
                ctx->present[q] = 1;
            } else {
                cov = 0;
                const PassDesc &a = ctx->passes[ctx->sel_pass[q]];
                k_pass_conflict<<<64, NT, 0, ctx->st>>>(a.values + (int64_t)sel_k[q] * a.n, d.values + (int64_t)kk * d.n,
                                                        d.n, ctx->d_conf + p);
                CH_LAUNCHED(ctx);
                conflicts = true;
            }
        }
        ctx->pass_covered[p] = cov;
    }
    if (conflicts) {
        std::vector<unsigned long long> hconf(n_passes);
        CH_CUDA(ctx, ch_d2h(ctx, hconf.data(), ctx->d_conf, 8 * n_passes));
        CH_CUDA(ctx, ch_sync(ctx));
        for (int p = 0; p < n_passes; p++)
            if (hconf[p] != ~0ull) ctx->pass_conflict[p] = (int64_t)hconf[p];
    }
    // E_ALIGNMENT from name mismatches and conflicts of this assignment
    ctx->latched_host &= ~(1u << CHOPPER_E_ALIGNMENT);
    for (int p = 0; p < n_passes; p++)
        if (ctx->pass_mismatch[p] >= 0 || ctx->pass_conflict[p] >= 0) ctx->latched_host |= 1u << CHOPPER_E_ALIGNMENT;
    if (C > 0) {
        if (!ctx->h_col_dev) {
            CH_ALLOC_BEGIN;
            ctx->h_col_dev = CH_ALLOC(ctx, const double *, (int64_t)nc);
            ctx->d_present = CH_ALLOC(ctx, int32_t, (int64_t)nc);
            CH_ALLOC_END(ctx);
        }
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->h_col_dev, hcol.data(), sizeof(double *) * nc, cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_present, ctx->present.data(), 4 * nc, cudaMemcpyHostToDevice, ctx->st));
    }
    ctx->d_col = ctx->h_col_dev;
    return CHOPPER_OK;
}

// a4 in two halves: the launch half (exchange, lower medians, skew, asynchronous read-backs) is issued by
// ch_align before its own read-back, so both share one host synchronization; the finish half reads them
chopper_status ch_offsets_launch(chopper_ctx *ctx) {
    const int G = ctx->cfg.n_traced_gpus;
    const int64_t W = ctx->xW, K = W / 4 - 1;
    const int slots = ctx->xslots;
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
        ctx->x_exchanged = true;       // this rank took part (even if the transport reports an error)
        CH_TRY(ch_nccl_allgather(ctx, ctx->d_xsend, all, sizeof(int64_t) * slots * W));
    } else {
        CH_CUDA(ctx, cudaMemcpyAsync(all, ctx->d_xsend, 8 * slots * W, cudaMemcpyDeviceToDevice, ctx->st));
    }
    const int nslots = slots * ctx->nranks;
    k_delta<<<nslots, DL_NT, 0, ctx->st>>>(all, nslots, W, K, ctx->d_delta, ctx->d_delta_flag);
    CH_LAUNCHED(ctx);
    k_skew<<<64, 256, 0, ctx->st>>>(all, nslots, W, K, ctx->d_delta, mskew);
    CH_LAUNCHED(ctx);
    ctx->delta.assign(G, 0);
    ctx->delta_flag.assign(G, 1);
    ctx->off_hs[0] = ctx->off_hs[1] = 0;
    ctx->off_ovf = 0;
    ctx->off_hdr.assign(2 * (size_t)nslots, 0);
    CH_CUDA(ctx, ch_d2h(ctx, ctx->delta.data(), ctx->d_delta, 8 * G));
    CH_CUDA(ctx, ch_d2h(ctx, ctx->delta_flag.data(), ctx->d_delta_flag, 4 * G));
    CH_CUDA(ctx, ch_d2h(ctx, ctx->off_hs, mskew, 16));
    CH_CUDA(ctx, ch_d2h(ctx, &ctx->off_ovf, ctx->d_xovf, 4));
    CH_CUDA(ctx, ch_d2h_2d(ctx, ctx->off_hdr.data(), 16, all, 8 * (size_t)W, 16, nslots));
    if (ctx->ss_pending) CH_CUDA(ctx, ch_d2h(ctx, &ctx->h_ss_fail, ctx->d_ss_fail, 4));   // (load's deferred check)
    ctx->off_pending = true;
    return CHOPPER_OK;
}

chopper_status ch_offsets_finish(chopper_ctx *ctx) {
    const int G = ctx->cfg.n_traced_gpus;
    if (!ctx->off_pending) CH_TRY(ch_offsets_launch(ctx));
    CH_CUDA(ctx, ch_sync(ctx));          // (already reached when ch_align synchronized)
    ctx->off_pending = false;
    CH_TRY(ch_comm_sort_settle(ctx));
    const int nslots = (int)(ctx->off_hdr.size() / 2);
    // gpus absent from every rank keep flag 1 (no events)
    ctx->gpu_present.assign(G, 0);
    for (int b = 0; b < nslots; b++)
        if (ctx->off_hdr[2 * (size_t)b + 1]) ctx->gpu_present[ctx->off_hdr[2 * (size_t)b]] = 1;
    for (int g = 0; g < G; g++) if (!ctx->gpu_present[g]) { ctx->delta_flag[g] = 1; ctx->delta[g] = 0; }
    // a slot whose gpu field is -1 is a failed rank's block (ch_exchange_poison): the step is dead everywhere
    for (int b = 0; b < nslots; b++)
        if (ctx->off_hdr[2 * (size_t)b] == -1)
            return ch_fail(ctx, CHOPPER_E_STATE, "a peer rank failed earlier in this step (all-gather #1)");
    ctx->max_skew[0] = (int64_t)ctx->off_hs[0];
    ctx->max_skew[1] = (int64_t)ctx->off_hs[1];
    if (ctx->off_ovf) return ch_fail(ctx, CHOPPER_E_RANGE, "more collectives per class than max_coll_per_class");
    return CHOPPER_OK;
}

chopper_status ch_offsets(chopper_ctx *ctx) { return ch_offsets_finish(ctx); }

// failure protocol (chopper.h): a rank that failed still makes this step's missing all-gather, with a block of
// the shape every healthy rank sends (derived from chopper_config, nranks and n_counters only) whose first slot
// header carries gpu = -1.  The step's scratch content is dead, so the blocks reuse the arena from mark_base.
chopper_status ch_exchange_poison(chopper_ctx *ctx, int which) {
    if (ctx->nranks <= 1) return CHOPPER_OK;
    if (which == 1 ? ctx->x_exchanged : ctx->d_exchanged) return CHOPPER_OK;
    const int slots = (int)ceil_div(ctx->cfg.n_traced_gpus, ctx->nranks);
    const int64_t W = which == 1 ? 4 + 4 * (int64_t)std::max(1, ctx->cfg.max_coll_per_class) : ch_dense_width(ctx);
    ctx->used = ctx->mark_base;
    CH_ALLOC_BEGIN;
    int64_t *send = CH_ALLOC(ctx, int64_t, (int64_t)slots * W);
    int64_t *recv = CH_ALLOC(ctx, int64_t, (int64_t)slots * W * ctx->nranks);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemsetAsync(send, 0, 8 * (size_t)slots * W, ctx->st));
    static const int64_t failed = -1;
    CH_CUDA(ctx, cudaMemcpyAsync(send, &failed, 8, cudaMemcpyHostToDevice, ctx->st));
    if (which == 1) ctx->x_exchanged = true; else ctx->d_exchanged = true;
    CH_TRY(ch_nccl_allgather(ctx, send, recv, sizeof(int64_t) * (size_t)slots * W));
    CH_CUDA(ctx, ch_sync(ctx));
    return CHOPPER_OK;
}
