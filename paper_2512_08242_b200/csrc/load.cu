// load.cu -- a1 pack + validate and a2 timestamp sort (chopper_load_columns).
//
// a1: one streaming pass over the event columns
//   checks t_ks <= t_ke, gpu grouping, non-decreasing dispatch per gpu, meta
//   ranges, and collects per-gpu ranges, the max compute stream and the
//   global timestamp range (< 2^52).
// a2 (D1): stable sort of events by (gpu, group, t_ks) with group = 0 for
//   communication, 1 + stream for COMPUTE, "other" last.  B200 path: one
//   stable counting pass keyed by (gpu, group) straight from meta; if any
//   communication or compute group is then not start-monotone, a full LSD
//   radix sort on (bucket, t_ks - t0) replaces it.  The same pass derives the
//   launch chain predecessor (previous COMPUTE kernel on the
//   same stream) and the same-stream disjointness check.
#include "common.cuh"

namespace {
constexpr int NT = 256;

__global__ void k_validate_events(const int64_t *__restrict__ tl, const int64_t *__restrict__ ks,
                                  const int64_t *__restrict__ ke, const uint32_t *__restrict__ meta, int64_t n,
                                  int G, DevReport *rep) {
    __shared__ unsigned int smax[CH_MAX_GPUS];
    for (int g = threadIdx.x; g < CH_MAX_GPUS; g += blockDim.x) smax[g] = 0;
    __syncthreads();
    unsigned long long lo = ~0ull, hi = 0ull;
    int sg = -1;
    unsigned smx = 0;                      // max compute stream + 1 of gpu sg (flushed on change: few atomics)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;                   // events per iteration: all loads issued before the checks
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
        uint32_t mm[U], mpv[U], mnv[U];
        int64_t av[U], bv[U], cv[U], apv[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = i0 + u * stride;
            const bool ok = i < n;
            mm[u] = ok ? meta[i] : 0u;
            av[u] = ok ? tl[i] : 0;
            bv[u] = ok ? ks[i] : 0;
            cv[u] = ok ? ke[i] : 0;
            mpv[u] = (ok && i > 0) ? meta[i - 1] : 0u;
            apv[u] = (ok && i > 0) ? tl[i - 1] : 0;
            mnv[u] = (ok && i + 1 < n) ? meta[i + 1] : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
        const int64_t i = i0 + u * stride;
        if (i >= n) break;
        const uint32_t m = mm[u];
        int g = gpu_of(m), k = kind_of(m), s = stream_of(m);
        int64_t a = av[u], b = bv[u], c = cv[u];
        if (b > c) viol(rep, CV_START_AFTER_END, i);
        if (i > 0) {
            uint32_t mp = mpv[u];
            int gp = gpu_of(mp);
            if (g < gp) viol(rep, CV_GPU_NOT_GROUPED, i);
            if (g == gp && a < apv[u]) viol(rep, CV_DISPATCH_DECREASING, i);
        }
        bool bad = k > CK_OTHER || g >= G || (k == CK_COMPUTE && s > 253);
        if (bad) {
            viol(rep, CV_BAD_META, i);
        } else {
            if (i == 0 || gpu_of(mpv[u]) != g) atomicMin(&rep->gbeg[g], (unsigned long long)i);
            if (i == n - 1 || gpu_of(mnv[u]) != g) atomicMax(&rep->gend[g], (unsigned long long)(i + 1));
            if (k == CK_COMPUTE) {
                if (g != sg) {
                    if (sg >= 0 && smx) atomicMax(&smax[sg], smx);
                    sg = g;
                    smx = 0;
                }
                smx = smx > (unsigned)(s + 1) ? smx : (unsigned)(s + 1);
            }
        }
        unsigned long long ea = enc_i64(a), eb = enc_i64(b), ec = enc_i64(c);
        unsigned long long mn = ea < eb ? ea : eb, mx = ea > eb ? ea : eb;
        mn = mn < ec ? mn : ec;
        mx = mx > ec ? mx : ec;
        lo = lo < mn ? lo : mn;
        hi = hi > mx ? hi : mx;
        }
    }
    if (sg >= 0 && smx) atomicMax(&smax[sg], smx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a = __shfl_xor_sync(CH_FULL, lo, o), b = __shfl_xor_sync(CH_FULL, hi, o);
        lo = lo < a ? lo : a;
        hi = hi > b ? hi : b;
    }
    if (lane_id() == 0) {
        atomicMin(&rep->t_min_enc, lo);
        atomicMax(&rep->t_max_enc, hi);
    }
    __syncthreads();
    for (int g = threadIdx.x; g < G; g += blockDim.x)
        if (smax[g]) atomicMax(&rep->max_stream[g], smax[g]);
}

__global__ void k_validate_spans(const uint32_t *__restrict__ gl, const int64_t *__restrict__ s,
                                 const int64_t *__restrict__ e, int64_t n, int G, DevReport *rep) {
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = gl[j];
        if (e[j] < s[j] || (x & 0xFFu) > 3 || (int)(x >> 8) >= G) {
            viol(rep, CV_SPAN_BAD, j);
            continue;
        }
        unsigned long long a = enc_i64(s[j]), b = enc_i64(e[j]);
        lo = lo < a ? lo : a;
        hi = hi > b ? hi : b;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a = __shfl_xor_sync(CH_FULL, lo, o), b = __shfl_xor_sync(CH_FULL, hi, o);
        lo = lo < a ? lo : a;
        hi = hi > b ? hi : b;
    }
    if (lane_id() == 0) {
        atomicMin(&rep->s_min_enc, lo);
        atomicMax(&rep->s_max_enc, hi);
    }
}

__global__ void k_validate_samples(const int32_t *__restrict__ g, const int64_t *__restrict__ ts, int64_t n, int G,
                                   DevReport *rep) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        int x = g[k];
        if (x < 0 || x >= G) { viol(rep, CV_SAMPLES_UNSORTED, k); continue; }
        if (k > 0 && (x < g[k - 1] || (x == g[k - 1] && ts[k] < ts[k - 1]))) viol(rep, CV_SAMPLES_UNSORTED, k);
        if (k == 0 || g[k - 1] != x) atomicMin(&rep->sbeg[x], (unsigned long long)k);
        if (k == n - 1 || g[k + 1] != x) atomicMax(&rep->send[x], (unsigned long long)(k + 1));
    }
}

__device__ __forceinline__ int bucket_of(uint32_t m, const int32_t *gpu_lg, int NG, int other) {
    int k = kind_of(m), g;
    if (is_comm(k)) g = 0;
    else if (k == CK_COMPUTE) g = 1 + stream_of(m);
    else g = other;
    return gpu_lg[gpu_of(m)] * NG + g;
}

__global__ void k_make_keys(const uint32_t *__restrict__ meta, const int64_t *__restrict__ ks, int64_t n,
                            const int32_t *__restrict__ gpu_lg, int NG, int other, int64_t t0, int tsbits,
                            unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long b = (unsigned long long)bucket_of(meta[i], gpu_lg, NG, other);
    keys[i] = tsbits ? (b << tsbits) | (unsigned long long)(ks[i] - t0) : b;
    vals[i] = (uint32_t)i;
}

// chain predecessor + monotonicity + same-stream disjointness, in sorted order
// 4 consecutive sorted positions per thread: the gathers of a position double as the predecessor's for
// the next one, and all of them are issued before the checks
constexpr int CHN = 4;
__global__ void k_chain(const uint32_t *__restrict__ perm, const uint32_t *__restrict__ meta,
                        const int64_t *__restrict__ ks, const int64_t *__restrict__ ke, int64_t n,
                        const int32_t *__restrict__ gpu_lg, int NG, int other, int64_t *__restrict__ pred_end,
                        DevReport *rep, unsigned int *__restrict__ bflag, unsigned long long *__restrict__ beg) {
    const int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * CHN;
    if (j0 >= n) return;
    uint32_t ii[CHN + 1], mm[CHN + 1];
    int64_t sv[CHN + 1], ev[CHN + 1];
#pragma unroll
    for (int u = 0; u <= CHN; u++) {                  // u = 0: the predecessor of j0
        const int64_t j = j0 + u - 1;
        ii[u] = (j >= 0 && j < n) ? perm[j] : 0u;
    }
#pragma unroll
    for (int u = 0; u <= CHN; u++) {
        const int64_t j = j0 + u - 1;
        const bool ok = j >= 0 && j < n;
        mm[u] = ok ? meta[ii[u]] : 0u;
        sv[u] = ok ? ks[ii[u]] : 0;
        ev[u] = ok ? ke[ii[u]] : 0;
    }
#pragma unroll
    for (int u = 1; u <= CHN; u++) {
        const int64_t j = j0 + u - 1;
        if (j >= n) break;
        const uint32_t i = ii[u], ip = ii[u - 1];
        const uint32_t m = mm[u];
        const int b = bucket_of(m, gpu_lg, NG, other);
        const int grp = b % NG;
        const bool same = j > 0 && bucket_of(mm[u - 1], gpu_lg, NG, other) == b;
        if (!same) beg[b] = (unsigned long long)j;     // first sorted position of the bucket
        int64_t pe = CH_NONE_TS;
        if (same && grp != other) {
            const int64_t a = sv[u];
            if (a < sv[u - 1]) bflag[b] = 1u;              // bucket not start-monotone: sort it
            if (grp >= 1) {
                pe = ev[u - 1];
                if (a < pe) viol(rep, CV_STREAM_OVERLAP, i);
            }
        }
        (void)ip;
        if (kind_of(m) == CK_COMPUTE) pred_end[i] = pe;
    }
}

// ---- lean a2 (every gpu has at most one compute stream): no full partition.  The compute group of a gpu in
// dispatch order IS its (g, stream, t_ks) order when it is start-monotone (checked here; otherwise the full
// path runs), so the chain predecessor is the previous COMPUTE event of the gpu in input order.  Only the
// communication and compute buckets of the permutation are written (the union and the full-mode compute
// overlap read them); the other bucket is never read.
constexpr int LN_NT = 256, LN_IPT = 8, LN_TILE = LN_NT * LN_IPT;
// per tile: communication / compute counts, the last compute index; per bucket counts (global atomics)
__global__ void __launch_bounds__(LN_NT) k_lean_tiles(const uint32_t *__restrict__ meta, int64_t n,
                                                      const int32_t *__restrict__ gpu_lg, int NG, int other,
                                                      int64_t *__restrict__ t_comm, int64_t *__restrict__ t_comp,
                                                      int64_t *__restrict__ t_last, unsigned long long *__restrict__ bcnt,
                                                      int nb, int64_t *__restrict__ mtc, int64_t ntile) {
    extern __shared__ unsigned int ln_h[];               // [nb]
    __shared__ int64_t sm[33];
    for (int b = threadIdx.x; b < nb; b += LN_NT) ln_h[b] = 0;
    __syncthreads();
    const int64_t i0 = (int64_t)blockIdx.x * LN_TILE + (int64_t)threadIdx.x * LN_IPT;
    int64_t cc = 0, cp = 0, last = -1;
    unsigned long long c3 = 0;           // non-MEMOP / AG / RS counts packed 21 bits apart (chopper_align's ranks)
    int hb = -1;                         // bucket histogram: one shared atomic per run of equal bucket
    unsigned hc = 0;
    uint32_t mv[LN_IPT];
    if (i0 + LN_IPT <= n && ((uintptr_t)(meta + i0) & 15u) == 0) {
        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(meta + i0)), b = __ldg(reinterpret_cast<const uint4 *>(meta + i0) + 1);
        mv[0] = a.x; mv[1] = a.y; mv[2] = a.z; mv[3] = a.w; mv[4] = b.x; mv[5] = b.y; mv[6] = b.z; mv[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < LN_IPT; k++) mv[k] = i0 + k < n ? meta[i0 + k] : 0u;
    }
#pragma unroll
    for (int k = 0; k < LN_IPT; k++) {
        const int64_t i = i0 + k;
        if (i >= n) break;
        const uint32_t m = mv[k];
        const int kd = kind_of(m);
        if (is_comm(kd)) cc++;
        else if (kd == CK_COMPUTE) { cp++; last = i; }
        c3 += (kd != CK_MEMOP ? 1ull : 0ull) | (kd == CK_AG ? 1ull << 21 : 0ull) | (kd == CK_RS ? 1ull << 42 : 0ull);
        const int b = bucket_of(m, gpu_lg, NG, other);
        if (b != hb) {
            if (hc) atomicAdd(&ln_h[hb], hc);
            hb = b;
            hc = 0;
        }
        hc++;
    }
    if (hc) atomicAdd(&ln_h[hb], hc);
    int64_t tc, tp;
    {                                    // (tile counts < 2^32: both totals from one packed scan)
        int64_t t2;
        block_excl_sum<LN_NT>(cc | (cp << 32), &t2, sm);
        tc = t2 & 0xFFFFFFFFll;
        tp = t2 >> 32;
    }
    if (mtc) {                           // the tile counts of chopper_align's rank pass (its tiles are these)
        int64_t t3;
        block_excl_sum<LN_NT>((int64_t)c3, &t3, sm);
        if (threadIdx.x == 0) {
            const unsigned long long t = (unsigned long long)t3;
            mtc[blockIdx.x] = (int64_t)(t & 0x1FFFFF);
            mtc[ntile + blockIdx.x] = (int64_t)((t >> 21) & 0x1FFFFF);
            mtc[2 * ntile + blockIdx.x] = (int64_t)(t >> 42);
        }
    }
    // block max of last
    int64_t x = last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { const int64_t y = __shfl_xor_sync(CH_FULL, x, o); x = y > x ? y : x; }
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t mx = -1;
        for (int w = 0; w < LN_NT / 32; w++) mx = sm[w] > mx ? sm[w] : mx;
        t_comm[blockIdx.x] = tc;
        t_comp[blockIdx.x] = tp;
        t_last[blockIdx.x] = mx;
    }
    for (int b = threadIdx.x; b < nb; b += LN_NT)
        if (ln_h[b]) atomicAdd(&bcnt[b], (unsigned long long)ln_h[b]);
}
// one block: exclusive max-scan of the tiles' last compute index (carry into every tile), bucket begins
// (exclusive scan of the bucket counts), and per-lg communication / compute ranks at the gpu's start
__global__ void k_lean_small(const int64_t *__restrict__ t_last, int64_t ntile, int64_t *__restrict__ carry,
                             const unsigned long long *__restrict__ bcnt, int nb, int NG,
                             int64_t *__restrict__ bbeg, int64_t *__restrict__ lg_comm0, int64_t *__restrict__ lg_comp0,
                             int n_lg) {
    __shared__ int64_t s_run;
    if (threadIdx.x == 0) {
        s_run = -1;
        int64_t acc = 0, c0 = 0, p0 = 0;
        for (int b = 0; b < nb; b++) {
            bbeg[b] = acc;
            acc += (int64_t)bcnt[b];
        }
        bbeg[nb] = acc;
        for (int l = 0; l < n_lg; l++) {
            lg_comm0[l] = c0;
            lg_comp0[l] = p0;
            c0 += (int64_t)bcnt[l * NG + 0];
            p0 += (int64_t)bcnt[l * NG + 1];
        }
    }
    __syncthreads();
    for (int64_t b0 = 0; b0 < ntile; b0 += blockDim.x) {
        const int64_t t = b0 + threadIdx.x;
        int64_t v = t < ntile ? t_last[t] : -1;
        // inclusive max-scan in the block (warp shuffles + a warp of partials)
        __shared__ int64_t wm[32];
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int64_t y = __shfl_up_sync(CH_FULL, x, o); if ((threadIdx.x & 31) >= o && y > x) x = y; }
        if ((threadIdx.x & 31) == 31) wm[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            int64_t z = threadIdx.x < blockDim.x / 32 ? wm[threadIdx.x] : -1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const int64_t y = __shfl_up_sync(CH_FULL, z, o); if ((int)threadIdx.x >= o && y > z) z = y; }
            wm[threadIdx.x] = z;
        }
        __syncthreads();
        int64_t inc = x;
        if ((threadIdx.x >> 5) > 0 && wm[(threadIdx.x >> 5) - 1] > inc) inc = wm[(threadIdx.x >> 5) - 1];
        if (s_run > inc) inc = s_run;
        // exclusive: the inclusive value of the previous tile
        int64_t ex = __shfl_up_sync(CH_FULL, inc, 1);
        if ((threadIdx.x & 31) == 0) ex = (threadIdx.x >> 5) > 0 ? (wm[(threadIdx.x >> 5) - 1] > s_run ? wm[(threadIdx.x >> 5) - 1] : s_run) : s_run;
        if (t < ntile) carry[t] = ex;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_run = inc;
        __syncthreads();
    }
}
// the chain and the two buckets, per tile of 2048 events (8 consecutive per thread)
__global__ void __launch_bounds__(LN_NT) k_lean_chain(const uint32_t *__restrict__ meta,
                                                      const int64_t *__restrict__ ks, const int64_t *__restrict__ ke,
                                                      int64_t n, const int32_t *__restrict__ gpu_lg, int NG,
                                                      const int64_t *__restrict__ g_beg,
                                                      const int64_t *__restrict__ t_comm_ex,
                                                      const int64_t *__restrict__ t_comp_ex,
                                                      const int64_t *__restrict__ carry,
                                                      const int64_t *__restrict__ bbeg,
                                                      const int64_t *__restrict__ lg_comm0,
                                                      const int64_t *__restrict__ lg_comp0,
                                                      uint32_t *__restrict__ perm, int64_t *__restrict__ pred_end,
                                                      DevReport *rep, unsigned int *__restrict__ nonmono) {
    __shared__ int64_t sm[33];
    __shared__ int64_t wl[LN_NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * LN_TILE + (int64_t)tid * LN_IPT;
    const int nv = i0 >= n ? 0 : (int)min((int64_t)LN_IPT, n - i0);
    uint32_t mt[LN_IPT];
    int64_t vs[LN_IPT], ve[LN_IPT];
    if (nv == LN_IPT && ((((uintptr_t)(meta + i0)) | ((uintptr_t)(ks + i0)) | ((uintptr_t)(ke + i0))) & 15u) == 0) {
#pragma unroll
        for (int h = 0; h < LN_IPT / 4; h++) {
            const uint4 x = __ldg(reinterpret_cast<const uint4 *>(meta + i0) + h);
            mt[4 * h] = x.x; mt[4 * h + 1] = x.y; mt[4 * h + 2] = x.z; mt[4 * h + 3] = x.w;
        }
#pragma unroll
        for (int h = 0; h < LN_IPT / 2; h++) {
            const longlong2 x = __ldg(reinterpret_cast<const longlong2 *>(ks + i0) + h);
            const longlong2 y = __ldg(reinterpret_cast<const longlong2 *>(ke + i0) + h);
            vs[2 * h] = x.x; vs[2 * h + 1] = x.y;
            ve[2 * h] = y.x; ve[2 * h + 1] = y.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < LN_IPT; k++) {
            const bool ok = k < nv;
            mt[k] = ok ? meta[i0 + k] : (uint32_t)CK_MEMOP;
            vs[k] = ok ? ks[i0 + k] : 0;
            ve[k] = ok ? ke[i0 + k] : 0;
        }
    }
    int64_t cc = 0, cp = 0, last = -1;
#pragma unroll
    for (int k = 0; k < LN_IPT; k++) {
        const int kd = kind_of(mt[k]);
        if (k < nv && is_comm(kd)) cc++;
        else if (k < nv && kd == CK_COMPUTE) { cp++; last = i0 + k; }
    }
    const int64_t ex2 = block_excl_sum<LN_NT>(cc | (cp << 32), nullptr, sm);   // (tile counts < 2^32: one packed scan)
    int64_t ex_c = (ex2 & 0xFFFFFFFFll) + t_comm_ex[blockIdx.x];
    int64_t ex_p = (ex2 >> 32) + t_comp_ex[blockIdx.x];
    // the last compute index before this thread
    int64_t x = last;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int64_t y = __shfl_up_sync(CH_FULL, x, o); if (lane >= o && y > x) x = y; }
    if (lane == 31) wl[w] = x;
    __syncthreads();
    int64_t before = carry[blockIdx.x];
    for (int q = 0; q < w; q++) before = wl[q] > before ? wl[q] : before;
    const int64_t xp = __shfl_up_sync(CH_FULL, x, 1);
    if (lane > 0 && xp > before) before = xp;
    // the predecessor's start / end: from global memory for the thread's first compute event, then registers
    int64_t p_ks = 0, p_ke = 0;
    if (before >= 0 && cp > 0) { p_ks = ks[before]; p_ke = ke[before]; }
    int64_t pes[LN_IPT];                  // chain ends (CH_NONE_TS at non-compute events: never read there)
    // per-gpu bases, reloaded only when the gpu changes (a thread's 8 events are nearly always one gpu's)
    int gcur = -1;
    int64_t cbase = 0, pbase = 0, gb0 = 0;
#pragma unroll
    for (int k = 0; k < LN_IPT; k++) {
        pes[k] = CH_NONE_TS;
        if (k >= nv) break;
        const int64_t i = i0 + k;
        const uint32_t m = mt[k];
        const int kd = kind_of(m);
        if (gpu_of(m) != gcur && (is_comm(kd) || kd == CK_COMPUTE)) {
            gcur = gpu_of(m);
            const int lg = gpu_lg[gcur];
            cbase = bbeg[lg * NG + 0] - lg_comm0[lg];
            pbase = bbeg[lg * NG + 1] - lg_comp0[lg];
            gb0 = g_beg[lg];
        }
        if (is_comm(kd)) {
            perm[cbase + ex_c] = (uint32_t)i;
            ex_c++;
        } else if (kd == CK_COMPUTE) {
            perm[pbase + ex_p] = (uint32_t)i;
            ex_p++;
            int64_t pe = CH_NONE_TS;
            if (before >= gb0) {
                pe = p_ke;
                if (vs[k] < p_ks) atomicOr(nonmono, 1u);          // not start-monotone: the full path sorts it
                if (vs[k] < pe) viol(rep, CV_STREAM_OVERLAP, i);
            }
            pes[k] = pe;
            before = i;
            p_ks = vs[k];
            p_ke = ve[k];
        }
    }
    if (!pred_end) return;                // lean a2: the event pass and the tables derive the chain themselves
    if (nv == LN_IPT && (((uintptr_t)(pred_end + i0)) & 15u) == 0) {
#pragma unroll
        for (int h = 0; h < LN_IPT / 2; h++)
            reinterpret_cast<longlong2 *>(pred_end + i0)[h] = make_longlong2(pes[2 * h], pes[2 * h + 1]);
    } else {
#pragma unroll
        for (int k = 0; k < LN_IPT; k++)
            if (k < nv && kind_of(mt[k]) == CK_COMPUTE) pred_end[i0 + k] = pes[k];
    }
}

// keys of the events in the flagged bucket segments: (segment, t_ks - t0), value = input index
__global__ void k_seg_keys(const uint32_t *__restrict__ perm, const int64_t *__restrict__ ks,
                           const int64_t *__restrict__ lo, const int64_t *__restrict__ pre, int nseg, int64_t M,
                           int64_t t0, int tsbits, unsigned long long *__restrict__ key, uint32_t *__restrict__ val) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= M) return;
    int a = 0, b = nseg;                       // segment: last pre[s] <= t
    while (b - a > 1) { int m = (a + b) >> 1; if (pre[m] <= t) a = m; else b = m; }
    uint32_t i = perm[lo[a] + (t - pre[a])];
    key[t] = ((unsigned long long)a << tsbits) | (unsigned long long)(ks[i] - t0);
    val[t] = i;
}
__global__ void k_seg_scatter(const uint32_t *__restrict__ sorted, const int64_t *__restrict__ lo,
                              const int64_t *__restrict__ pre, int nseg, int64_t M, uint32_t *__restrict__ perm) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= M) return;
    int a = 0, b = nseg;
    while (b - a > 1) { int m = (a + b) >> 1; if (pre[m] <= t) a = m; else b = m; }
    perm[lo[a] + (t - pre[a])] = sorted[t];
}

// ---- stream-merge fast path for the non-monotone buckets (D1) ------------------------------------
// A bucket mixing several streams (all-gathers and reduce-scatters) is not start-monotone in dispatch
// order, but each stream serializes its kernels, so each stream's events usually are.  Then the stable
// timestamp sort of the bucket is a merge of its per-stream lists: an element's position is its index in
// its stream's list plus, for every other stream of the bucket, the number of that stream's events with
// a smaller (t_ks, input index) -- a binary search.  Lists come from a one-byte stable partition.
constexpr int SS_STREAMS = 256;
__device__ __forceinline__ int seg_of(const int64_t *__restrict__ pre, int nseg, int64_t t) {
    int a = 0, b = nseg;
    while (b - a > 1) { int m = (a + b) >> 1; if (pre[m] <= t) a = m; else b = m; }
    return a;
}
__global__ void k_ss_keys(const uint32_t *__restrict__ perm, const uint32_t *__restrict__ meta,
                          const int64_t *__restrict__ lo, const int64_t *__restrict__ pre, int nseg, int64_t M,
                          unsigned long long *__restrict__ key, uint32_t *__restrict__ val, unsigned int *__restrict__ cnt,
                          unsigned int *__restrict__ fail, uint32_t *__restrict__ save) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= M) return;
    const int a = seg_of(pre, nseg, t);
    const uint32_t i = perm[lo[a] + (t - pre[a])];
    if (save) save[t] = i;                    // the unsorted segments, for a redo by the radix path
    const int st = stream_of(meta[i]);
    if (st >= SS_STREAMS) atomicOr(fail, 1u);
    const int cell = a * SS_STREAMS + (st & (SS_STREAMS - 1));
    key[t] = (unsigned long long)cell;
    val[t] = i;
    atomicAdd(&cnt[cell], 1u);
}
// each stream list start-monotone?
__global__ void k_ss_check(const unsigned long long *__restrict__ key, const uint32_t *__restrict__ val, int64_t M,
                           const int64_t *__restrict__ ks, unsigned int *__restrict__ fail) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0 || t >= M) return;
    if (key[t] == key[t - 1] && ks[val[t]] < ks[val[t - 1]]) atomicOr(fail, 2u);
}
// the non-empty stream cells of each segment (block a, thread = cell): cl[a * SS_STREAMS + k], k < cl_n[a], so an
// element's rank searches only the streams present, not all SS_STREAMS cells
__global__ void __launch_bounds__(SS_STREAMS) k_ss_cells(const unsigned int *__restrict__ cnt, int32_t *__restrict__ cl,
                                                         int32_t *__restrict__ cl_n) {
    __shared__ int64_t sm[33];
    const int a = blockIdx.x, c = threadIdx.x;
    const int cell = a * SS_STREAMS + c;
    const bool on = cnt[cell] != 0;
    int64_t tot;
    const int64_t pos = block_excl_sum<SS_STREAMS>(on ? 1 : 0, &tot, sm);
    if (on) cl[a * SS_STREAMS + pos] = cell;
    if (c == 0) cl_n[a] = (int32_t)tot;
}
__global__ void k_ss_rank(const unsigned long long *__restrict__ key, const uint32_t *__restrict__ val, int64_t M,
                          const int64_t *__restrict__ ks, const unsigned int *__restrict__ cnt,
                          const int64_t *__restrict__ cstart, const int64_t *__restrict__ lo,
                          const int32_t *__restrict__ cl, const int32_t *__restrict__ cl_n,
                          uint32_t *__restrict__ perm) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= M) return;
    const int cell = (int)key[t];
    const int a = cell / SS_STREAMS;
    const uint32_t x = val[t];
    const int64_t kx = ks[x];
    int64_t r = t - cstart[cell];
    for (int q = 0; q < cl_n[a]; q++) {
        const int c2 = cl[a * SS_STREAMS + q];
        const unsigned int n2 = cnt[c2];
        if (c2 == cell) continue;
        int64_t l = cstart[c2], h = l + n2;           // count of (ks, idx) < (kx, x) in list c2
        const int64_t l0 = l;
        while (l < h) {
            const int64_t m = (l + h) >> 1;
            const uint32_t y = val[m];
            const int64_t ky = ks[y];
            if (ky < kx || (ky == kx && y < x)) l = m + 1; else h = m;
        }
        r += l - l0;
    }
    perm[lo[a] + r] = x;
}
__global__ void k_u32_i64(const unsigned int *__restrict__ a, int64_t *__restrict__ b, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}

__global__ void k_init_report(DevReport *r) {
    int t = threadIdx.x;
    if (t < CV_NRULES) { r->val_count[t] = 0; r->val_first[t] = ~0ull; }
    for (int g = t; g < CH_MAX_GPUS; g += blockDim.x) {
        r->gbeg[g] = ~0ull; r->gend[g] = 0; r->sbeg[g] = ~0ull; r->send[g] = 0; r->max_stream[g] = 0; r->n_comm[g] = 0;
    }
    if (t == 0) {
        r->t_min_enc = ~0ull; r->t_max_enc = 0; r->s_min_enc = ~0ull; r->s_max_enc = 0; r->flags = 0; r->latched = 0;
        r->n_nonlaminar = 0;
    }
}

__global__ void k_fill_u64(unsigned long long *p, int64_t n, unsigned long long v) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
}  // namespace

chopper_status ch_fill_u64(chopper_ctx *ctx, unsigned long long *p, int64_t n, unsigned long long v) {
    if (n <= 0) return CHOPPER_OK;
    k_fill_u64<<<(unsigned)ceil_div(n, NT), NT, 0, ctx->st>>>(p, n, v);
    CH_LAUNCHED(ctx);
    return CHOPPER_OK;
}

static chopper_status read_report(chopper_ctx *ctx) {
    CH_CUDA(ctx, ch_d2h(ctx, &ctx->h_rep, ctx->d_rep, sizeof(DevReport)));
    CH_CUDA(ctx, ch_sync(ctx));
    return CHOPPER_OK;
}

static void fill_public_report(chopper_ctx *ctx) {
    DevReport &h = ctx->h_rep;
    chopper_report &r = ctx->rep;
    for (int q = 0; q < CV_NRULES; q++) {
        r.val_count[q] = (int64_t)h.val_count[q];
        r.val_first[q] = h.val_first[q] == ~0ull ? -1 : (int64_t)h.val_first[q];
    }
    r.n_local_gpus = ctx->n_lg;
    for (int l = 0; l < ctx->n_lg; l++) r.local_gpu[l] = ctx->lg_gpu[l];
    r.t_min = ctx->t0;
    r.t_max = ctx->t_max;
    r.full_sort_used = ctx->full_sort ? 1 : 0;
}

static chopper_status finish_load(chopper_ctx *ctx) {
    // same-stream overlaps are data: reported, processing continues
    fill_public_report(ctx);
    if (ctx->h_rep.val_count[CV_STREAM_OVERLAP]) ctx->latched_host |= 1u << CHOPPER_E_VALIDATION;
    ctx->loaded_ok = true;
    ctx->mark_after_load = ctx->used;
    return CHOPPER_OK;
}

// the lean a2 (see k_lean_chain); *fell_back = true when a compute group is not start-monotone (the caller then
// runs the full partition + chain, which resets the overlap report it recomputes)
// stable timestamp sort of the permutation segments [seg_lo[s], seg_lo[s] + size) (D1): a stream-merge fast
// path (partition by stream + binary-search ranks), else a radix sort on (segment, t_ks - t0)
// the radix path: a stable sort of the segments by (segment, t_ks - t0)
static chopper_status sort_segments_radix(chopper_ctx *ctx, const std::vector<int64_t> &seg_lo,
                                          const std::vector<int64_t> &seg_pre, int64_t Mseg) {
    const int nseg = (int)seg_lo.size() - 1;         // (both arrays carry their end entry)
    const int tsbits = bits_for((uint64_t)(ctx->t_max - ctx->t0)), sb = bits_for((uint64_t)nseg);
    if (tsbits + sb > 64) return ch_fail(ctx, CHOPPER_E_RANGE, "sort key exceeds 64 bits");
    const size_t mk = ctx->used;
    CH_ALLOC_BEGIN;
    unsigned long long *k1 = CH_ALLOC(ctx, unsigned long long, Mseg), *k2 = CH_ALLOC(ctx, unsigned long long, Mseg);
    uint32_t *v1 = CH_ALLOC(ctx, uint32_t, Mseg), *v2 = CH_ALLOC(ctx, uint32_t, Mseg);
    int64_t *dlo = CH_ALLOC(ctx, int64_t, nseg + 1), *dpre = CH_ALLOC(ctx, int64_t, nseg + 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemcpyAsync(dlo, seg_lo.data(), 8 * (nseg + 1), cudaMemcpyHostToDevice, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(dpre, seg_pre.data(), 8 * (nseg + 1), cudaMemcpyHostToDevice, ctx->st));
    k_seg_keys<<<(unsigned)ceil_div(Mseg, NT), NT, 0, ctx->st>>>(ctx->d_perm, ctx->ev.start_ns, dlo, dpre, nseg, Mseg,
                                                                 ctx->t0, tsbits, k1, v1);
    CH_LAUNCHED(ctx);
    bool alt;
    CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, Mseg, 0, tsbits + sb, &alt));
    k_seg_scatter<<<(unsigned)ceil_div(Mseg, NT), NT, 0, ctx->st>>>(alt ? v2 : v1, dlo, dpre, nseg, Mseg, ctx->d_perm);
    CH_LAUNCHED(ctx);
    ctx->used = mk;
    return CHOPPER_OK;
}

// Stable timestamp sort of the permutation segments [seg_lo[s], seg_lo[s] + size) (D1): the stream-merge fast
// path (partition by stream + binary-search ranks), else the radix path.  defer: the fast path's validity flag is
// not waited for here -- it is read with chopper_align's read-back (ch_comm_sort_settle), and a failed check then
// restores the saved unsorted segments and takes the radix path before anything reads them (the communication
// buckets are first read by chopper_overlap's preparation)
static chopper_status sort_segments(chopper_ctx *ctx, std::vector<int64_t> seg_lo, std::vector<int64_t> seg_pre,
                                    int64_t Mseg, bool defer = false) {
    const int64_t n = ctx->N;
    CH_ALLOC_BEGIN;
    const int nseg = (int)seg_lo.size();
    seg_pre.push_back(Mseg);
    seg_lo.push_back(n);
    const int sb = bits_for((uint64_t)nseg);
    if (bits_for((uint64_t)(ctx->t_max - ctx->t0)) + sb > 64) return ch_fail(ctx, CHOPPER_E_RANGE, "sort key exceeds 64 bits");
    unsigned int *fail = nullptr;
    if (defer) {
        // kept until chopper_align: the flag and the unsorted segments (for a redo)
        fail = CH_ALLOC(ctx, unsigned int, 1);
        ctx->d_ss_save = CH_ALLOC(ctx, uint32_t, Mseg);
        CH_ALLOC_END(ctx);                   // (filled by k_ss_keys)
    }
    size_t mk = ctx->used;
    unsigned long long *k1 = CH_ALLOC(ctx, unsigned long long, Mseg), *k2 = CH_ALLOC(ctx, unsigned long long, Mseg);
    uint32_t *v1 = CH_ALLOC(ctx, uint32_t, Mseg), *v2 = CH_ALLOC(ctx, uint32_t, Mseg);
    int64_t *dlo = CH_ALLOC(ctx, int64_t, nseg + 1), *dpre = CH_ALLOC(ctx, int64_t, nseg + 1);
    const int64_t cells = (int64_t)nseg * SS_STREAMS;
    unsigned int *cnt = CH_ALLOC(ctx, unsigned int, cells);
    if (!fail) fail = CH_ALLOC(ctx, unsigned int, 1);
    int64_t *c64 = CH_ALLOC(ctx, int64_t, cells), *cst = CH_ALLOC(ctx, int64_t, cells);
    int32_t *dcl = CH_ALLOC(ctx, int32_t, cells), *dcn = CH_ALLOC(ctx, int32_t, nseg + 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemcpyAsync(dlo, seg_lo.data(), 8 * (nseg + 1), cudaMemcpyHostToDevice, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(dpre, seg_pre.data(), 8 * (nseg + 1), cudaMemcpyHostToDevice, ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(cnt, 0, 4 * (size_t)cells, ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(fail, 0, 4, ctx->st));
    k_ss_keys<<<(unsigned)ceil_div(Mseg, NT), NT, 0, ctx->st>>>(ctx->d_perm, ctx->ev.meta, dlo, dpre, nseg, Mseg,
                                                                k1, v1, cnt, fail, defer ? ctx->d_ss_save : nullptr);
    CH_LAUNCHED(ctx);
    bool alt2;
    CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, Mseg, 0, sb + 8, &alt2));
    unsigned long long *ksd = alt2 ? k2 : k1;
    uint32_t *vsd = alt2 ? v2 : v1;
    k_ss_check<<<(unsigned)ceil_div(Mseg, NT), NT, 0, ctx->st>>>(ksd, vsd, Mseg, ctx->ev.start_ns, fail);
    CH_LAUNCHED(ctx);
    k_u32_i64<<<(unsigned)ceil_div(cells, NT), NT, 0, ctx->st>>>(cnt, c64, cells);
    CH_LAUNCHED(ctx);
    CH_TRY(ch_scan_excl_i64(ctx, c64, cst, cells, nullptr));
    k_ss_cells<<<nseg, SS_STREAMS, 0, ctx->st>>>(cnt, dcl, dcn);
    CH_LAUNCHED(ctx);
    if (defer) {
        // speculative: valid unless the flag is set (then ch_comm_sort_settle redoes the segments)
        k_ss_rank<<<(unsigned)ceil_div(Mseg, NT), NT, 0, ctx->st>>>(ksd, vsd, Mseg, ctx->ev.start_ns, cnt, cst, dlo,
                                                                    dcl, dcn, ctx->d_perm);
        CH_LAUNCHED(ctx);
        ctx->d_ss_fail = fail;
        ctx->ss_seg_lo = seg_lo;
        ctx->ss_seg_pre = seg_pre;
        ctx->ss_M = Mseg;
        ctx->ss_pending = true;
        ctx->used = mk;
        return CHOPPER_OK;
    }
    unsigned int hfail = 0;
    CH_CUDA(ctx, ch_d2h(ctx, &hfail, fail, 4));
    CH_CUDA(ctx, ch_sync(ctx));
    if (!hfail) {
        k_ss_rank<<<(unsigned)ceil_div(Mseg, NT), NT, 0, ctx->st>>>(ksd, vsd, Mseg, ctx->ev.start_ns, cnt, cst, dlo,
                                                                    dcl, dcn, ctx->d_perm);
        CH_LAUNCHED(ctx);
        ctx->used = mk;
        return CHOPPER_OK;
    }
    ctx->used = mk;
    return sort_segments_radix(ctx, seg_lo, seg_pre, Mseg);
}

// the deferred check of the lean path's communication sort (called right after chopper_align's synchronization,
// which also brought h_ss_fail): a failed stream-merge check restores the unsorted segments and sorts by radix
chopper_status ch_comm_sort_settle(chopper_ctx *ctx) {
    if (!ctx->ss_pending) return CHOPPER_OK;
    ctx->ss_pending = false;
    if (!ctx->h_ss_fail) return CHOPPER_OK;
    const int nseg = (int)ctx->ss_seg_lo.size() - 1;
    for (int a = 0; a < nseg; a++)
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_perm + ctx->ss_seg_lo[a], ctx->d_ss_save + ctx->ss_seg_pre[a],
                                     4 * (size_t)(ctx->ss_seg_pre[a + 1] - ctx->ss_seg_pre[a]), cudaMemcpyDeviceToDevice,
                                     ctx->st));
    return sort_segments_radix(ctx, ctx->ss_seg_lo, ctx->ss_seg_pre, ctx->ss_M);
}

static chopper_status lean_a2(chopper_ctx *ctx, bool *fell_back);

chopper_status ch_load(chopper_ctx *ctx) {
    const int G = ctx->cfg.n_traced_gpus;
    const int64_t n = ctx->N;
    // a span sort of an earlier step that was never joined (the step failed) must finish before its scratch is
    // reused
    if (ctx->span_pending) {
        CH_CUDA(ctx, cudaStreamWaitEvent(ctx->st, ctx->span_join, 0));
        ctx->span_pending = false;
    }
    ctx->span_launched = false;
    ctx->d_meta_tc = nullptr;
    ctx->ss_pending = false;
    if (ctx->prep_pending) {                    // likewise chopper_overlap's preparation
        CH_CUDA(ctx, cudaStreamWaitEvent(ctx->st, ctx->prep_join, 0));
        ctx->prep_pending = false;
    }
    ctx->prep_done = false;
    ctx->used = 0;
    CH_ALLOC_BEGIN;
    ctx->d_rep = CH_ALLOC(ctx, DevReport, 1);
    ctx->d_gpu_lg = CH_ALLOC(ctx, int32_t, CH_MAX_GPUS);
    CH_ALLOC_END(ctx);
    ctx->mark_base = ctx->used;
    k_init_report<<<1, 256, 0, ctx->st>>>(ctx->d_rep);
    CH_LAUNCHED(ctx);
    // one full wave of resident blocks (grid-stride): no partial last wave; sized once per ctx for its device
    if (!ctx->v_blocks) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_validate_events, NT, 0);
        ctx->v_blocks = std::max(per, 1) * sms;
    }
    unsigned grid = (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(n, NT), 1), ctx->v_blocks);
    if (n > 0) {
        k_validate_events<<<grid, NT, 0, ctx->st>>>(ctx->ev.dispatch_ns, ctx->ev.start_ns, ctx->ev.end_ns, ctx->ev.meta,
                                                    n, G, ctx->d_rep);
        CH_LAUNCHED(ctx);
    }
    if (ctx->S > 0) {
        unsigned gs = (unsigned)std::min<int64_t>(ceil_div(ctx->S, NT), 148 * 8);
        k_validate_spans<<<gs, NT, 0, ctx->st>>>(ctx->sp.gpu_level, ctx->sp.start_ns, ctx->sp.end_ns, ctx->S, G,
                                                 ctx->d_rep);
        CH_LAUNCHED(ctx);
    }
    if (ctx->has_smp && ctx->M > 0) {
        unsigned gs = (unsigned)std::min<int64_t>(ceil_div(ctx->M, NT), 148 * 8);
        k_validate_samples<<<gs, NT, 0, ctx->st>>>(ctx->smp.gpu, ctx->smp.ts_ns, ctx->M, G, ctx->d_rep);
        CH_LAUNCHED(ctx);
    }
    g_marks.mark(ctx->st, "ld_validate");
    CH_TRY(read_report(ctx));
    DevReport &h = ctx->h_rep;
    ctx->t0 = n > 0 ? dec_i64(h.t_min_enc) : 0;
    ctx->t_max = n > 0 ? dec_i64(h.t_max_enc) : 0;
    if (n > 0 && (uint64_t)ctx->t_max - (uint64_t)ctx->t0 >= (1ull << 52)) {
        h.val_count[CV_TS_RANGE] = 1;
        h.val_first[CV_TS_RANGE] = 0;
    }
    // local gpus (events grouped ascending)
    ctx->n_lg = 0;
    for (int g = 0; g < CH_MAX_GPUS; g++) ctx->gpu_lg_h[g] = -1;
    int ms = 0;
    for (int g = 0; g < G; g++) {
        if (h.gend[g] > 0 && h.gbeg[g] != ~0ull) {
            ctx->gpu_lg_h[g] = ctx->n_lg;
            ctx->lg_gpu[ctx->n_lg] = g;
            ctx->g_beg[ctx->n_lg] = (int64_t)h.gbeg[g];
            ctx->n_lg++;
            ms = std::max(ms, (int)h.max_stream[g]);
        }
    }
    ctx->g_beg[ctx->n_lg] = n;
    ctx->max_stream = ms;
    ctx->multi_stream = ms > 1;
    ctx->NG = ms + 2;
    ctx->n_buckets = ctx->n_lg * ctx->NG;
    fill_public_report(ctx);
    const int fatal[] = {CV_START_AFTER_END, CV_GPU_NOT_GROUPED, CV_DISPATCH_DECREASING, CV_BAD_META, CV_TS_RANGE,
                         CV_SPAN_BAD, CV_SAMPLES_UNSORTED};
    for (int q : fatal)
        if (h.val_count[q]) {
            ctx->loaded_ok = false;
            return ch_fail(ctx, CHOPPER_E_VALIDATION, "input validation failed (rule " + std::to_string(q) + ")");
        }
    if (ctx->n_lg == 0) {
        ctx->loaded_ok = true;
        return CHOPPER_OK;
    }
    CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_gpu_lg, ctx->gpu_lg_h, sizeof(int32_t) * CH_MAX_GPUS, cudaMemcpyHostToDevice,
                                 ctx->st));
    // the spans are validated: their push-order sort starts now on a side stream, beside the rest of the load
    // and chopper_align and their host synchronizations (spans.cu; chopper_attribute joins it)
    CH_TRY(ch_span_sort_launch(ctx));
    // a2: partition by (lg, dense group); full radix sort only if a group is not start-monotone
    ctx->d_perm = CH_ALLOC(ctx, uint32_t, n);
    ctx->d_pred_end = nullptr;       // materialized by the general path only (k_chain); lean: derived (PredView)
    ctx->d_bucket_beg = CH_ALLOC(ctx, int64_t, ctx->n_buckets + 1);
    CH_ALLOC_END(ctx);
    const int NG = ctx->NG, other = NG - 1;
    ctx->lean = false;
    if (!ctx->multi_stream && ctx->n_buckets <= 1024) {
        bool fell_back = false;
        CH_TRY(lean_a2(ctx, &fell_back));
        if (!fell_back) {
            ctx->lean = true;          // compute kernels of every gpu are start-monotone in dispatch order
            return finish_load(ctx);
        }
    }
    ctx->d_pred_end = CH_ALLOC(ctx, int64_t, n);
    CH_ALLOC_END(ctx);
    size_t mark = ctx->used;
    if (ctx->n_buckets <= 256) {
        CH_TRY(ch_radix_partition_meta(ctx, ctx->ev.meta, ctx->d_gpu_lg, NG, other, ctx->d_perm, n));
    } else {
        unsigned long long *k1 = CH_ALLOC(ctx, unsigned long long, n), *k2 = CH_ALLOC(ctx, unsigned long long, n);
        uint32_t *v2 = CH_ALLOC(ctx, uint32_t, n);
        CH_ALLOC_END(ctx);
        k_make_keys<<<(unsigned)ceil_div(n, NT), NT, 0, ctx->st>>>(ctx->ev.meta, ctx->ev.start_ns, n, ctx->d_gpu_lg,
                                                                   NG, other, 0, 0, k1, ctx->d_perm);
        CH_LAUNCHED(ctx);
        bool alt;
        CH_TRY(ch_radix_sort(ctx, k1, ctx->d_perm, k2, v2, n, 0, bits_for((uint64_t)ctx->n_buckets), &alt));
        if (alt) CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_perm, v2, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, ctx->st));
    }
    ctx->used = mark;
    ctx->full_sort = false;
    const int nb = ctx->n_buckets;
    unsigned int *bflag = CH_ALLOC(ctx, unsigned int, nb + 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemsetAsync(bflag, 0, 4 * (nb + 1), ctx->st));
    // bucket begins (unchanged by the per-bucket timestamp sort below)
    unsigned long long *beg = reinterpret_cast<unsigned long long *>(ctx->d_bucket_beg);
    CH_TRY(ch_fill_u64(ctx, beg, nb + 1, ~0ull));
    k_chain<<<(unsigned)ceil_div(n, NT * CHN), NT, 0, ctx->st>>>(ctx->d_perm, ctx->ev.meta, ctx->ev.start_ns,
                                                           ctx->ev.end_ns, n, ctx->d_gpu_lg, NG, other,
                                                           ctx->d_pred_end, ctx->d_rep, bflag, beg);
    CH_LAUNCHED(ctx);
    ctx->bucket_beg.assign(nb + 1, 0);
    std::vector<unsigned int> hflag(nb + 1, 0);
    CH_CUDA(ctx, ch_d2h(ctx, ctx->bucket_beg.data(), beg, 8 * (nb + 1)));
    CH_CUDA(ctx, ch_d2h(ctx, hflag.data(), bflag, 4 * (nb + 1)));
    CH_TRY(read_report(ctx));
    ctx->bucket_beg[nb] = n;
    for (int b = nb - 1; b >= 0; b--)
        if ((unsigned long long)ctx->bucket_beg[b] == ~0ull) ctx->bucket_beg[b] = ctx->bucket_beg[b + 1];
    CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_bucket_beg, ctx->bucket_beg.data(), 8 * (nb + 1), cudaMemcpyHostToDevice,
                                 ctx->st));
    // buckets that are not start-monotone in dispatch order: stable timestamp sort of just those segments (D1)
    std::vector<int64_t> seg_lo, seg_pre;
    bool compute_resorted = false;
    int64_t Mseg = 0;
    for (int b = 0; b < nb; b++)
        if (hflag[b]) {
            seg_lo.push_back(ctx->bucket_beg[b]);
            seg_pre.push_back(Mseg);
            Mseg += ctx->bucket_beg[b + 1] - ctx->bucket_beg[b];
            if (b % NG >= 1 && b % NG != other) compute_resorted = true;
        }
    if (Mseg > 0) {
        CH_TRY(sort_segments(ctx, seg_lo, seg_pre, Mseg));
        ctx->full_sort = true;
        if (compute_resorted) {
            // chain predecessors and the disjointness check depend on the corrected order
            unsigned long long zero = 0, none = ~0ull;
            CH_CUDA(ctx, cudaMemcpyAsync(&ctx->d_rep->val_count[CV_STREAM_OVERLAP], &zero, 8, cudaMemcpyHostToDevice,
                                         ctx->st));
            CH_CUDA(ctx, cudaMemcpyAsync(&ctx->d_rep->val_first[CV_STREAM_OVERLAP], &none, 8, cudaMemcpyHostToDevice,
                                         ctx->st));
            k_chain<<<(unsigned)ceil_div(n, NT * CHN), NT, 0, ctx->st>>>(ctx->d_perm, ctx->ev.meta, ctx->ev.start_ns,
                                                                   ctx->ev.end_ns, n, ctx->d_gpu_lg, NG, other,
                                                                   ctx->d_pred_end, ctx->d_rep, bflag, beg);
            CH_LAUNCHED(ctx);
            CH_TRY(read_report(ctx));
        }
    }
    return finish_load(ctx);
}

static chopper_status lean_a2(chopper_ctx *ctx, bool *fell_back) {
    const int64_t n = ctx->N;
    const int NG = ctx->NG, other = NG - 1, nb = ctx->n_buckets, n_lg = ctx->n_lg;
    *fell_back = false;
    const int64_t ntile = ceil_div(n, LN_TILE);
    CH_ALLOC_BEGIN;
    ctx->d_meta_tc = CH_ALLOC(ctx, int64_t, 3 * ntile);       // kept for chopper_align (no separate count pass)
    CH_ALLOC_END(ctx);
    const size_t keep = ctx->used;
    int64_t *tcm = CH_ALLOC(ctx, int64_t, ntile + 1), *tcp = CH_ALLOC(ctx, int64_t, ntile + 1);
    int64_t *tla = CH_ALLOC(ctx, int64_t, ntile + 1), *tcme = CH_ALLOC(ctx, int64_t, ntile + 1);
    int64_t *tcpe = CH_ALLOC(ctx, int64_t, ntile + 1), *carry = CH_ALLOC(ctx, int64_t, ntile + 1);
    unsigned long long *bcnt = CH_ALLOC(ctx, unsigned long long, nb + 1);
    int64_t *lc0 = CH_ALLOC(ctx, int64_t, n_lg + 1), *lp0 = CH_ALLOC(ctx, int64_t, n_lg + 1);
    int64_t *gb = CH_ALLOC(ctx, int64_t, n_lg + 1);
    unsigned int *nonmono = CH_ALLOC(ctx, unsigned int, 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemsetAsync(bcnt, 0, 8 * (size_t)(nb + 1), ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(nonmono, 0, 4, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(gb, ctx->g_beg, 8 * (n_lg + 1), cudaMemcpyHostToDevice, ctx->st));
    k_lean_tiles<<<(unsigned)ntile, LN_NT, 4 * nb, ctx->st>>>(ctx->ev.meta, n, ctx->d_gpu_lg, NG, other, tcm, tcp, tla,
                                                              bcnt, nb, ctx->d_meta_tc, ntile);
    CH_LAUNCHED(ctx);
    CH_TRY(ch_scan_excl_i64(ctx, tcm, tcme, ntile, nullptr));
    CH_TRY(ch_scan_excl_i64(ctx, tcp, tcpe, ntile, nullptr));
    k_lean_small<<<1, 1024, 0, ctx->st>>>(tla, ntile, carry, bcnt, nb, NG, ctx->d_bucket_beg, lc0, lp0, n_lg);
    CH_LAUNCHED(ctx);
    k_lean_chain<<<(unsigned)ntile, LN_NT, 0, ctx->st>>>(ctx->ev.meta, ctx->ev.start_ns, ctx->ev.end_ns, n, ctx->d_gpu_lg,
                                                         NG, gb, tcme, tcpe, carry, ctx->d_bucket_beg, lc0, lp0,
                                                         ctx->d_perm, nullptr, ctx->d_rep, nonmono);
    CH_LAUNCHED(ctx);
    ctx->bucket_beg.assign(nb + 1, 0);
    unsigned int hnm = 0;
    CH_CUDA(ctx, ch_d2h(ctx, ctx->bucket_beg.data(), ctx->d_bucket_beg, 8 * (nb + 1)));
    CH_CUDA(ctx, ch_d2h(ctx, &hnm, nonmono, 4));
    CH_TRY(read_report(ctx));
    ctx->used = keep;
    if (hnm) {
        // a compute group out of start order: the full path (it resets and recomputes the overlap report)
        unsigned long long zero = 0, none = ~0ull;
        CH_CUDA(ctx, cudaMemcpyAsync(&ctx->d_rep->val_count[CV_STREAM_OVERLAP], &zero, 8, cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(&ctx->d_rep->val_first[CV_STREAM_OVERLAP], &none, 8, cudaMemcpyHostToDevice, ctx->st));
        *fell_back = true;
        return CHOPPER_OK;
    }
    ctx->full_sort = false;
    // communication buckets: a stable timestamp sort of each (streams interleave); one segment per gpu
    std::vector<int64_t> seg_lo, seg_pre;
    int64_t Mseg = 0;
    for (int l = 0; l < n_lg; l++) {
        const int b = l * NG;
        const int64_t c = ctx->bucket_beg[b + 1] - ctx->bucket_beg[b];
        if (c >= 2) {
            seg_lo.push_back(ctx->bucket_beg[b]);
            seg_pre.push_back(Mseg);
            Mseg += c;
        }
    }
    if (Mseg > 0) {
        CH_TRY(sort_segments(ctx, seg_lo, seg_pre, Mseg, true));
        ctx->full_sort = true;
    }
    return CHOPPER_OK;
}
