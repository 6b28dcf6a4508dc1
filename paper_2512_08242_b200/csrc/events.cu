// events.cu -- the per-event hot pass (chopper_overlap).
//
// One fused, tiled pass over the event columns in dispatch (input) order:
//   a5  attribution key per event: innermost span per level (spans.cu),
//   a6  overlap: COMPUTE -> |[t_ks,t_ke) ∩ U_g| with U_g the union of the
//       gpu's communication intervals (D9), as
//       cov(t_ke) - cov(t_ks) over prefix lengths of the merged union;
//       communication -> |[t_ks,t_ke) ∩ V_g| (compute union),
//   a7  launch overhead Eqs. 1-3 with the chain
//       predecessor from a2 and dispatch clamped to start (D6),
//   a8  frequency / power integrals over a zero-order hold (D10) as
//       differences of prefix integrals,
//   a9  (time part) reduction of each maximal run of equal instance key into
//       a sub-run row: thread-sequential folding, in-tile completion through
//       shared memory, sub-run ids from a decoupled look-back chained scan.
// Each 2048-event tile is cut at its boundary so sub-runs never cross tiles;
// sub-runs with equal keys are merged into instances in tables.cu.
#include "common.cuh"

#include <cuda.h>

SpanView ch_span_view(chopper_ctx *ctx);

namespace {
constexpr int NT = 256;
constexpr int EV_NT = 256, EV_IPT = 8, EV_TILE = EV_NT * EV_IPT;
constexpr unsigned long long FLAG_A = 1ull << 62, FLAG_P = 2ull << 62, VAL_MASK = (1ull << 62) - 1;

// ---- comm / compute unions: one block per local gpu ----------------------------------------------
// positions pos[lo..hi) index events sorted by t_ks; output merged intervals at out[lo + m].
// 4 consecutive sorted intervals per thread (all gathers in flight at once), 4096 per block iteration:
// inclusive prefix max of the ends -> a head wherever a start exceeds the running max end -> merged
// intervals, then prefix lengths.
constexpr int UN_IPT = 4, UN_NT = 1024, UN_CH = UN_NT * UN_IPT;
__global__ void __launch_bounds__(UN_NT) k_union_block(const uint32_t *__restrict__ pos, const int64_t *__restrict__ seg_lo,
                                                       const int64_t *__restrict__ seg_hi, const int64_t *__restrict__ ks,
                                                       const int64_t *__restrict__ ke, int64_t *__restrict__ Us,
                                                       int64_t *__restrict__ Ue, int64_t *__restrict__ UP,
                                                       int64_t *__restrict__ Ubeg, int64_t *__restrict__ Ucnt,
                                                       const int64_t *__restrict__ obase) {
    __shared__ int64_t sm[33];
    __shared__ int64_t smax[32];
    __shared__ int64_t s_carry_max, s_m, s_next_s;
    const int lg = blockIdx.x;
    const int64_t lo = seg_lo[lg], hi = seg_hi[lg];
    const int64_t ob = obase ? obase[lg] : lo;     // output offset of this gpu's merged intervals
    const int tid = threadIdx.x, w = tid >> 5, l = lane_id();
    if (tid == 0) { s_carry_max = INT64_MIN; s_m = 0; }
    __syncthreads();
    for (int64_t base = lo; base < hi; base += UN_CH) {
        const int64_t j0 = base + (int64_t)tid * UN_IPT;
        int64_t sv[UN_IPT], ev[UN_IPT];
        uint32_t pi[UN_IPT];
#pragma unroll
        for (int u = 0; u < UN_IPT; u++) pi[u] = j0 + u < hi ? pos[j0 + u] : 0u;
#pragma unroll
        for (int u = 0; u < UN_IPT; u++) {
            const bool ok = j0 + u < hi;
            sv[u] = ok ? ks[pi[u]] : INT64_MAX;
            ev[u] = ok ? ke[pi[u]] : INT64_MIN;
        }
        // thread max, then block inclusive prefix max of the thread maxima
        int64_t tmax = INT64_MIN;
#pragma unroll
        for (int u = 0; u < UN_IPT; u++) tmax = ev[u] > tmax ? ev[u] : tmax;
        int64_t v = tmax;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(CH_FULL, v, o);
            if (l >= o && y > v) v = y;
        }
        if (l == 31) smax[w] = v;
        __syncthreads();
        if (w == 0) {
            int64_t x = smax[l];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(CH_FULL, x, o);
                if (l >= o && y > x) x = y;
            }
            smax[l] = x;
        }
        __syncthreads();
        // running max before this thread's first interval
        int64_t run = s_carry_max;
        const int64_t wpre = w > 0 ? smax[w - 1] : INT64_MIN;
        if (wpre > run) run = wpre;
        const int64_t lpre = __shfl_up_sync(CH_FULL, v, 1);
        if (l > 0 && lpre > run) run = lpre;
        bool hd[UN_IPT];
        int64_t mi[UN_IPT];
        int nh = 0;
#pragma unroll
        for (int u = 0; u < UN_IPT; u++) {
            hd[u] = j0 + u < hi && sv[u] > run;     // run = INT64_MIN for the very first interval
            nh += hd[u];
            if (ev[u] > run) run = ev[u];
            mi[u] = run;                            // inclusive max through this interval
        }
        int64_t tot;
        const int64_t ex = block_excl_sum<UN_NT>(nh, &tot, sm);
        const int64_t m0 = s_m;
        // the first start of the next thread decides whether this thread's last interval closes a run
        int64_t k = m0 + ex;
#pragma unroll
        for (int u = 0; u < UN_IPT; u++) {
            if (hd[u]) { Us[ob + k] = sv[u]; k++; }
            bool close = false;
            if (j0 + u < hi) {
                if (u + 1 < UN_IPT) close = !(j0 + u + 1 < hi) || hd[u + 1];
                else close = true;   // resolved below against the next thread's first start
            }
            if (close && u + 1 < UN_IPT) Ue[ob + k - 1] = mi[u];
        }
        // last interval of the thread: closes a run if the next interval (next thread / next chunk) is a head
        const int64_t jl = j0 + UN_IPT - 1;
        if (jl < hi) {
            bool nexthead = true;
            if (jl + 1 < hi) nexthead = ks[pos[jl + 1]] > mi[UN_IPT - 1];
            if (nexthead) Ue[ob + k - 1] = mi[UN_IPT - 1];
        }
        __syncthreads();
        if (tid == UN_NT - 1) s_carry_max = run;
        if (tid == 0) s_m = m0 + tot;
        __syncthreads();
    }
    const int64_t mcount = s_m;
    // prefix lengths (UN_IPT consecutive merged intervals per thread)
    int64_t acc = 0;
    for (int64_t b2 = 0; b2 < mcount; b2 += UN_CH) {
        const int64_t m0 = b2 + (int64_t)tid * UN_IPT;
        int64_t len[UN_IPT], s = 0;
#pragma unroll
        for (int u = 0; u < UN_IPT; u++) {
            len[u] = m0 + u < mcount ? Ue[ob + m0 + u] - Us[ob + m0 + u] : 0;
            s += len[u];
        }
        int64_t tot;
        int64_t ex = block_excl_sum<UN_NT>(s, &tot, sm);
#pragma unroll
        for (int u = 0; u < UN_IPT; u++) {
            if (m0 + u < mcount) UP[ob + m0 + u] = acc + ex;
            ex += len[u];
        }
        acc += tot;
    }
    if (tid == 0) { Ubeg[lg] = ob; Ucnt[lg] = mcount; }
    (void)s_next_s;
}

// sample prefix inputs: f_k * (tau_{k+1} - tau_k) within a gpu, 0 at a gpu's last sample
__global__ void k_smp_terms(const int32_t *__restrict__ g, const int64_t *__restrict__ ts,
                            const int32_t *__restrict__ f, const int32_t *__restrict__ p, int64_t n,
                            int64_t *__restrict__ tf, int64_t *__restrict__ tp, uint8_t *__restrict__ head) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    bool last = (k == n - 1) || g[k + 1] != g[k];
    int64_t dt = last ? 0 : ts[k + 1] - ts[k];
    tf[k] = (int64_t)f[k] * dt;
    tp[k] = (int64_t)p[k] * dt;
    head[k] = (k == 0) || g[k - 1] != g[k];
}


// ---- timeline: comm-union boundaries and samples of a gpu merged by time (window-staged event pass) ----
// Entry j of gpu lg holds, for every t from its time up to the next entry's: coverage cov(t) = V0 + S0*(t - t0),
// frequency integral F(t) = V1 + S1*(t - t0) and power integral Pw(t) = V2 + S2*(t - t0) (MHz*ns, mW*ns; the
// prefix integrals of the zero-order hold, D10).  Intercepts wrap modulo 2^64 like the prefix sums they come
// from, so differences F(t_ke) - F(t_ks) are the exact int64 integrals.  Ties: union entries before samples.
__global__ void k_timeline(const int64_t *__restrict__ tl_beg, const int64_t *__restrict__ ncomm, int n_lg,
                           int64_t cap_total, const int64_t *__restrict__ Us, const int64_t *__restrict__ Ue,
                           const int64_t *__restrict__ UP, const int64_t *__restrict__ Ubeg,
                           const int64_t *__restrict__ Ucnt, const int64_t *__restrict__ ts,
                           const int64_t *__restrict__ phi, const int64_t *__restrict__ psi,
                           const int32_t *__restrict__ sf, const int32_t *__restrict__ sp,
                           const int64_t *__restrict__ slo_a, const int64_t *__restrict__ shi_a, int64_t T0,
                           int64_t cap, int64_t *__restrict__ Tt, int64_t *__restrict__ Tv, int32_t *__restrict__ Ts,
                           int64_t *__restrict__ tl_len) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cap_total) return;
    int l = 0, h = n_lg;
    while (h - l > 1) {
        const int m = (l + h) >> 1;
        if (tl_beg[m] <= j) l = m; else h = m;
    }
    const int lg = l;
    const int64_t beg = tl_beg[lg], a = j - beg, nc = ncomm[lg];
    const int64_t ub = Ubeg[lg], U = Ucnt[lg], slo = slo_a[lg], shi = shi_a[lg];
    int64_t t, pos;
    if (a == 0) {
        t = INT64_MIN;
        pos = beg;
        tl_len[lg] = 1 + 2 * U + (shi - slo);
    } else if (a - 1 < 2 * nc) {
        const int64_t u = (a - 1) >> 1, e = (a - 1) & 1;
        if (u >= U) return;
        t = e ? Ue[ub + u] : Us[ub + u];
        int64_t l2 = slo, h2 = shi;                  // samples strictly before t
        while (l2 < h2) {
            const int64_t m = (l2 + h2) >> 1;
            if (ts[m] < t) l2 = m + 1; else h2 = m;
        }
        pos = beg + 1 + 2 * u + e + (l2 - slo);
    } else {
        const int64_t b = a - 1 - 2 * nc;
        if (b >= shi - slo) return;
        t = ts[slo + b];
        const int64_t uu = last_le(Us, ub, ub + U, t);
        const int64_t cu = uu < ub ? 0 : 2 * (uu - ub + 1) - (Ue[uu] > t ? 1 : 0);   // union entries at or before t
        pos = beg + 1 + b + cu;
    }
    // state after the entry
    unsigned long long c0 = 0, c1 = 0, c2 = 0;
    int32_t inu = 0, f = 0, pw = 0;
    const int64_t uu = last_le(Us, ub, ub + U, t);
    if (uu >= ub) {
        const int64_t s0 = Us[uu], e0 = Ue[uu];
        if (t < e0) {
            inu = 1;
            c0 = (unsigned long long)UP[uu] - (unsigned long long)(s0 - T0);
        } else {
            c0 = (unsigned long long)UP[uu] + (unsigned long long)(e0 - s0);
        }
    }
    if (shi > slo) {
        int64_t q = last_le(ts, slo, shi, t);
        if (q < slo) q = slo;                        // before the first sample: f_0 extended backwards (D10)
        f = sf[q];
        pw = sp[q];
        const unsigned long long dq = (unsigned long long)(ts[q] - T0);
        c1 = (unsigned long long)phi[q] - (unsigned long long)(int64_t)f * dq;
        c2 = (unsigned long long)psi[q] - (unsigned long long)(int64_t)pw * dq;
    }
    Tt[pos] = t;
    Tv[pos] = (int64_t)c0;
    Tv[cap + pos] = (int64_t)c1;
    Tv[2 * cap + pos] = (int64_t)c2;
    Ts[pos] = inu;
    Ts[cap + pos] = f;
    Ts[2 * cap + pos] = pw;
}

// ---- compute-union keys for multi-stream gpus -----------------------------------------------------
__global__ void k_vkeys(const uint32_t *__restrict__ meta, const int64_t *__restrict__ ks, int64_t n,
                        const int32_t *__restrict__ gpu_lg, int64_t t0, int tsbits, int lgbits,
                        unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t m = meta[i];
    unsigned long long k;
    if (kind_of(m) == CK_COMPUTE)
        k = ((unsigned long long)gpu_lg[gpu_of(m)] << tsbits) | (unsigned long long)(ks[i] - t0);
    else
        k = ((1ull << lgbits) - 1) << tsbits;    // sorts after every gpu
    keys[i] = k;
    vals[i] = (uint32_t)i;
}

// ---- fused event pass ---------------------------------------------------------------------------
struct TileWin;
struct EvParams {
    const int64_t *tl, *ks, *ke;
    const uint32_t *meta;
    int64_t N;
    const int32_t *gpu_lg;
    SpanView sv;
    int sh_op, sh_ly, sh_ph, sh_it, sh_lg;
    const int64_t *pred_end;
    const int64_t *Us, *Ue, *UP, *Ubeg, *Ucnt;
    int v_general;
    const int64_t *Vs, *Ve, *VP, *Vbeg, *Vcnt;
    const uint32_t *perm;
    const int64_t *bucket_beg;
    int NG;
    const int64_t *smp_ts;
    const int32_t *smp_f, *smp_p;
    const int64_t *phi_pre, *psi_pre, *smp_lo, *smp_hi;
    int64_t *o_ovl, *o_prep, *o_call, *o_phi, *o_psi;
    int32_t *o_run;               // (unused: the counter pass reads the per-thread values below)
    int32_t *t_run;               // [ntile][256] run id before each thread's first event (counters only)
    uint8_t *t_hm;                // [ntile][256] head mask of each thread's 8 events
    unsigned long long *sr_key;
    int64_t *sr_first;
    int64_t *sr_f;
    int64_t cap;
    unsigned long long *tile_state;
    unsigned int *ticket;
    // window-staged pass: combined key table, timeline and per-tile seeds
    const int64_t *KTt;
    const unsigned long long *KTk;
    const int64_t *kt_beg;
    const int64_t *TLt, *TLv;
    const int32_t *TLs;
    const int64_t *tl_beg, *tl_len;
    int64_t tl_cap, t0;
    const int32_t *seeds;
    int64_t ntile;
    const int64_t *tile_base;     // [ntile + 1] first sub-run id of each tile
    const struct TileWin *twin;   // [ntile] placed windows
    const struct TileWinL *twinl; // [ntile] placed windows of the lean pass
    // lean pass: the head pre-count's results, so the event pass does no key lookups of its own
    uint32_t *kidx;               // [ntile * 2048] key-table index of each event (written by k_tile_heads)
    const int32_t *h_run;         // [ntile][256] in-tile head rank before each thread's first event
    const uint8_t *h_hm;          // [ntile][256] head mask of each thread's 8 events
};


// last index in [lo, hi) with a[idx] <= t, seeded by the previous answer (t mostly non-decreasing)
__device__ __forceinline__ int64_t seek(const int64_t *__restrict__ a, int64_t lo, int64_t hi, int64_t t, int64_t *cur) {
    int64_t c = *cur;
    if (c >= lo - 1 && c < hi && (c < lo || __ldg(a + c) <= t)) {
        int steps = 0;
        while (c + 1 < hi && __ldg(a + c + 1) <= t && steps < 4) { c++; steps++; }
        if (c + 1 < hi && __ldg(a + c + 1) <= t) c = last_le(a, c + 1, hi, t);
    } else {
        c = last_le(a, lo, hi, t);
    }
    *cur = c;
    return c;
}

// coverage of (-inf, t) by a merged union with prefix lengths
__device__ __forceinline__ int64_t cov(const int64_t *Us, const int64_t *Ue, const int64_t *UP, int64_t lo, int64_t hi,
                                       int64_t t, int64_t *cur) {
    if (hi <= lo) return 0;
    int64_t u = seek(Us, lo, hi, t, cur);
    if (u < lo) return 0;
    int64_t s = __ldg(Us + u), e = __ldg(Ue + u);
    int64_t x = t - s;
    if (x > e - s) x = e - s;
    return __ldg(UP + u) + x;
}

// |[a, b) ∩ compute intervals| for the single-stream fast path: intervals sorted and disjoint
__device__ int64_t covl_fast(const EvParams &P, int lg, int64_t a, int64_t b) {
    int64_t lo = P.bucket_beg[lg * P.NG + 1], hi = P.bucket_beg[lg * P.NG + 2];
    // first compute interval with end > a (ends are sorted for disjoint sorted intervals)
    int64_t l = lo, h = hi;
    while (l < h) {
        int64_t m = (l + h) >> 1;
        if (__ldg(P.ke + P.perm[m]) > a) h = m; else l = m + 1;
    }
    int64_t tot = 0;
    for (int64_t j = l; j < hi; j++) {
        uint32_t i = P.perm[j];
        int64_t s = __ldg(P.ks + i);
        if (s >= b) break;
        int64_t e = __ldg(P.ke + i);
        int64_t x = s > a ? s : a, y = e < b ? e : b;
        if (y > x) tot += y - x;
    }
    return tot;
}

// per-event overlap of communication kernels with the compute union (R6), one thread per comm event;
// comm events are the first bucket of each gpu in sorted order
__global__ void k_covl(EvParams P, int n_lg) {
    int lg = blockIdx.y;
    int64_t lo = P.bucket_beg[lg * P.NG], hi = P.bucket_beg[lg * P.NG + 1];
    for (int64_t j = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < hi; j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t i = P.perm[j];
        int64_t ks = P.ks[i], ke = P.ke[i], ovl;
        if (P.v_general) {
            int64_t vlo = P.Vbeg[lg], vhi = vlo + P.Vcnt[lg];
            int64_t c1 = -2, c2 = -2;
            ovl = cov(P.Vs, P.Ve, P.VP, vlo, vhi, ke, &c1) - cov(P.Vs, P.Ve, P.VP, vlo, vhi, ks, &c2);
        } else {
            ovl = covl_fast(P, lg, ks, ke);
        }
        P.o_ovl[i] = ovl;
    }
}

// ---- sub-run aggregate ----------------------------------------------------------------------------
// Counts and the first-event offset are tile-local 32-bit (a tile holds 2048 events); the rest are the
// int64 row fields.  merge() is commutative and associative: sums, max(last_ke) and the lexicographic
// min of (first_ks, first offset) -- so the segmented scan below may combine in any grouping.
struct Acc {
    int32_t nev, n, foff;
    int64_t busy, prep, call, ovl, phi, psi, copy, ag, rs, fks, lke;
    __device__ __forceinline__ void zero() {
        nev = 0; n = 0; foff = INT32_MAX;
        busy = prep = call = ovl = phi = psi = copy = ag = rs = 0;
        fks = INT64_MAX; lke = INT64_MIN;
    }
    __device__ __forceinline__ void merge(const Acc &b) {
        nev += b.nev; n += b.n;
        busy += b.busy; prep += b.prep; call += b.call; ovl += b.ovl; phi += b.phi; psi += b.psi;
        copy += b.copy; ag += b.ag; rs += b.rs;
        if (b.lke > lke) lke = b.lke;
        if (b.fks < fks || (b.fks == fks && b.foff < foff)) { fks = b.fks; foff = b.foff; }
    }
    __device__ __forceinline__ Acc shfl_up(int o) const {
        Acc r;
        r.nev = __shfl_up_sync(CH_FULL, nev, o); r.n = __shfl_up_sync(CH_FULL, n, o);
        r.foff = __shfl_up_sync(CH_FULL, foff, o);
        r.busy = __shfl_up_sync(CH_FULL, busy, o); r.prep = __shfl_up_sync(CH_FULL, prep, o);
        r.call = __shfl_up_sync(CH_FULL, call, o); r.ovl = __shfl_up_sync(CH_FULL, ovl, o);
        r.phi = __shfl_up_sync(CH_FULL, phi, o); r.psi = __shfl_up_sync(CH_FULL, psi, o);
        r.copy = __shfl_up_sync(CH_FULL, copy, o); r.ag = __shfl_up_sync(CH_FULL, ag, o);
        r.rs = __shfl_up_sync(CH_FULL, rs, o); r.fks = __shfl_up_sync(CH_FULL, fks, o);
        r.lke = __shfl_up_sync(CH_FULL, lke, o);
        return r;
    }
};

// sub-run rows are AoS: 16 int64 (14 fields in RowField order + pad) = one 128 B line per row
constexpr int SR_W = 16;
__device__ __forceinline__ void write_subrun(const EvParams &P, int64_t id, const Acc &a, int64_t base) {
    if (id >= P.cap) return;      // beyond the structural bound (host reports CHOPPER_E_RANGE)
    longlong2 *dst = reinterpret_cast<longlong2 *>(P.sr_f + id * SR_W);
    const int64_t fidx = a.foff == INT32_MAX ? INT64_MAX : base + a.foff;
    // RowField: NEV N BUSY FIRST_IDX LAST_KE PREP CALL OVL PHI PSI COPY AG RS FIRST_KS
    dst[0] = make_longlong2(a.nev, a.n);
    dst[1] = make_longlong2(a.busy, fidx);
    dst[2] = make_longlong2(a.lke, a.prep);
    dst[3] = make_longlong2(a.call, a.ovl);
    dst[4] = make_longlong2(a.phi, a.psi);
    dst[5] = make_longlong2(a.copy, a.ag);
    dst[6] = make_longlong2(a.rs, a.fks);
    dst[7] = make_longlong2(0, 0);
}

// ---- register caches for the per-event lookups (events of a gpu come in dispatch order) ----
// innermost span of one (gpu, level) list: unchanged while t < start of the next span in push order
// and t < end of the current answer (descendants on the chain already ended before the previous t)
struct LvCache {
    int32_t lb, le, c0, res;
    int64_t next_start, res_end;
    bool pre;
};
// seed = last push-order index with start <= the thread's first dispatch (warp_seeds), or -2 (none): the
// first lookup then walks forward / up from the seed instead of binary-searching the whole list
__device__ __forceinline__ void lv_reset(LvCache &c, const SpanView &v, int list, int32_t seed = -2) {
    c.lb = (int32_t)v.list_beg[list];
    c.le = (int32_t)v.list_beg[list + 1];
    c.pre = v.list_flags[list] != 0;
    c.c0 = seed >= c.lb - 1 && seed < c.le ? seed : -2;
    c.res = -1;
    c.next_start = INT64_MIN;      // forces the first lookup through the walk
}
__device__ __forceinline__ int32_t lv_lookup(LvCache &c, const SpanView &v, int lv, int64_t t, int64_t i) {
    if (c.pre) return v.attr_pre[(int64_t)lv * v.N + i];
    if (c.le <= c.lb) return -1;
    if (c.c0 != -2 && t < c.next_start && (c.res < 0 || t < c.res_end)) return c.res;
    int64_t c0 = c.c0;
    if (c0 == -2) {
        c0 = last_le(v.P_start, c.lb, c.le, t);
    } else {
        int steps = 0;
        while (c0 + 1 < c.le && __ldg(v.P_start + c0 + 1) <= t && steps < 4) { c0++; steps++; }
        if (c0 + 1 < c.le && __ldg(v.P_start + c0 + 1) <= t) c0 = last_le(v.P_start, c0 + 1, c.le, t);
    }
    int64_t r = c0;
    while (r >= c.lb && __ldg(v.P_end + r) <= t) r = __ldg(v.P_parent + r);
    if (r < c.lb) r = -1;
    c.c0 = (int32_t)c0;
    c.res = (int32_t)r;
    c.next_start = c0 + 1 < c.le ? __ldg(v.P_start + c0 + 1) : INT64_MAX;
    c.res_end = r >= 0 ? __ldg(v.P_end + r) : 0;
    return (int32_t)r;
}

// coverage of (-inf, t) by the gpu's merged comm union, caching the current merged interval
struct CovCache {
    int32_t lo, hi, u;
    int64_t us, len, up, next_s;
};
__device__ __forceinline__ void cov_reset(CovCache &c, int64_t lo, int64_t cnt) {
    c.lo = (int32_t)lo;
    c.hi = (int32_t)(lo + cnt);
    c.u = -2;
}
// position the cache at merged interval u (last start <= the thread's first query), loading its fields
__device__ __forceinline__ void cov_seed(CovCache &c, const int64_t *Us, const int64_t *Ue, const int64_t *UP,
                                         int32_t u) {
    if (c.hi <= c.lo || u < c.lo - 1 || u >= c.hi) return;
    c.u = u;
    c.next_s = u + 1 < c.hi ? __ldg(Us + u + 1) : INT64_MAX;
    if (u >= c.lo) {
        c.us = __ldg(Us + u);
        c.len = __ldg(Ue + u) - c.us;
        c.up = __ldg(UP + u);
    }
}
__device__ __forceinline__ int64_t cov_c(CovCache &c, const int64_t *Us, const int64_t *Ue, const int64_t *UP, int64_t t) {
    if (c.hi <= c.lo) return 0;
    if (!(c.u != -2 && t < c.next_s && (c.u < c.lo || t >= c.us))) {
        int64_t u;
        if (c.u != -2 && c.u >= c.lo && t >= c.us) {     // forward from the cached interval
            u = c.u;
            int steps = 0;
            while (u + 1 < c.hi && __ldg(Us + u + 1) <= t && steps < 4) { u++; steps++; }
            if (u + 1 < c.hi && __ldg(Us + u + 1) <= t) u = last_le(Us, u + 1, c.hi, t);
        } else {
            u = last_le(Us, c.lo, c.hi, t);
        }
        c.u = (int32_t)u;
        c.next_s = u + 1 < c.hi ? __ldg(Us + u + 1) : INT64_MAX;
        if (u >= c.lo) {
            c.us = __ldg(Us + u);
            c.len = __ldg(Ue + u) - c.us;
            c.up = __ldg(UP + u);
        }
    }
    if (c.u < c.lo) return 0;
    int64_t x = t - c.us;
    return c.up + (x < c.len ? x : c.len);
}

// prefix integral F(t) of a zero-order-hold sample stream, caching the current sample window
struct SmpCache {
    int32_t lo, hi, q;
    int64_t ts, next, phi, psi;
    int32_t f, p;
};
__device__ __forceinline__ void smp_reset(SmpCache &c, int64_t lo, int64_t hi) {
    c.lo = (int32_t)lo;
    c.hi = (int32_t)hi;
    c.q = -2;
}
__device__ __forceinline__ void smp_seed(SmpCache &c, const EvParams &P, int32_t q) {
    if (c.hi <= c.lo || q < c.lo - 1 || q >= c.hi) return;
    if (q < c.lo) q = c.lo;            // before the first sample: f_0 extended backwards (D10)
    c.q = q;
    c.ts = __ldg(P.smp_ts + q);
    c.next = q + 1 < c.hi ? __ldg(P.smp_ts + q + 1) : INT64_MAX;
    c.phi = __ldg(P.phi_pre + q);
    c.psi = __ldg(P.psi_pre + q);
    c.f = __ldg(P.smp_f + q);
    c.p = __ldg(P.smp_p + q);
}

// ---- warp-cooperative seeding of the per-thread caches -------------------------------------------
// For NQ sorted tables a[lo, hi) (warp-uniform) and one query t per lane, every lane gets the last
// index with a[idx] <= t (lo - 1 if none; -2 for lanes that do not take part).  A 32-ary descent on the
// warp's smallest query (one probe per lane per round, all tables in lockstep) replaces each lane's
// ~18-step dependent binary search; lanes then resolve their own query in 32-element register chunks
// (shuffle binary search), walking forward chunk by chunk.
struct SeedQ {
    const int64_t *a;
    int64_t lo, hi;
    int64_t t;
    bool on;
};
template <int NQ>
__device__ __forceinline__ void warp_seeds(const SeedQ (&q)[NQ], int32_t (&ans)[NQ]) {
    const int lane = lane_id();
    int64_t l[NQ], h[NQ], qmin[NQ];
    bool act[NQ];
#pragma unroll
    for (int j = 0; j < NQ; j++) {
        act[j] = __any_sync(CH_FULL, q[j].on) && q[j].hi > q[j].lo;
        int64_t x = q[j].on ? q[j].t : INT64_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            int64_t y = __shfl_xor_sync(CH_FULL, x, o);
            x = y < x ? y : x;
        }
        qmin[j] = x;
        l[j] = q[j].lo;
        h[j] = q[j].hi;
        ans[j] = -2;
    }
    while (true) {
        bool any = false;
        int64_t v[NQ], step[NQ];
#pragma unroll
        for (int j = 0; j < NQ; j++) {
            v[j] = INT64_MAX;
            step[j] = 0;
            if (act[j] && h[j] - l[j] > 32) {
                step[j] = (h[j] - l[j] + 31) >> 5;
                int64_t p = l[j] + lane * step[j];
                if (p < h[j]) v[j] = __ldg(q[j].a + p);
                any = true;
            }
        }
        if (!any) break;
#pragma unroll
        for (int j = 0; j < NQ; j++) {
            if (step[j] == 0) continue;
            int c = __popc(__ballot_sync(CH_FULL, v[j] <= qmin[j]));
            if (c == 0) {
                h[j] = l[j];                  // answer l - 1
            } else {
                int64_t nl = l[j] + (int64_t)(c - 1) * step[j];
                h[j] = nl + step[j] < h[j] ? nl + step[j] : h[j];
                l[j] = nl + 1;                // answer in [nl, h - 1]
            }
        }
    }
    // chunks from l: every element before l is <= the smallest query
#pragma unroll
    for (int j = 0; j < NQ; j++) {
        if (!act[j]) continue;
        const int64_t t = q[j].on ? q[j].t : INT64_MIN;
        bool done = !q[j].on;
        int64_t c0 = l[j];
        while (__any_sync(CH_FULL, !done)) {
            int64_t val = c0 + lane < q[j].hi ? __ldg(q[j].a + c0 + lane) : INT64_MAX;
            int pos = 0;
#pragma unroll
            for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                int64_t x = __shfl_sync(CH_FULL, val, pos + s2 - 1);
                if (x <= t) pos += s2;
            }
            if (__shfl_sync(CH_FULL, val, 31) <= t) pos = 32;
            if (!done && pos < 32) { ans[j] = (int32_t)(c0 - 1 + pos); done = true; }
            if (!done && c0 + 32 >= q[j].hi) { ans[j] = (int32_t)(q[j].hi - 1); done = true; }
            c0 += 32;
        }
    }
}
__device__ __forceinline__ void smp_F(SmpCache &c, const EvParams &P, int64_t t, int64_t *F, int64_t *Pw) {
    if (!(c.q != -2 && t < c.next && (c.q == c.lo || t >= c.ts))) {
        int64_t q;
        if (c.q != -2 && t >= c.next) {    // forward from the cached window (t mostly increases)
            q = c.q + 1;
            int steps = 0;
            while (q + 1 < c.hi && __ldg(P.smp_ts + q + 1) <= t && steps < 4) { q++; steps++; }
            if (q + 1 < c.hi && __ldg(P.smp_ts + q + 1) <= t) q = last_le(P.smp_ts, q + 1, c.hi, t);
        } else {
            q = last_le(P.smp_ts, c.lo, c.hi, t);
        }
        if (q < c.lo) q = c.lo;            // before the first sample: f_0 extended backwards (D10)
        c.q = (int32_t)q;
        c.ts = __ldg(P.smp_ts + q);
        c.next = q + 1 < c.hi ? __ldg(P.smp_ts + q + 1) : INT64_MAX;
        c.phi = __ldg(P.phi_pre + q);
        c.psi = __ldg(P.psi_pre + q);
        c.f = __ldg(P.smp_f + q);
        c.p = __ldg(P.smp_p + q);
    }
    int64_t dt = t - c.ts;
    *F = c.phi + (int64_t)c.f * dt;
    *Pw = c.psi + (int64_t)c.p * dt;
}


// ---- tile staging: cp.async 16 B units into an XOR-swizzled thread-blocked layout ------------------
// Thread t owns events [8t, 8t+8) of the tile.  An int64 column keeps thread t's 64 B as four 16 B
// units, unit j stored at slot t*4 + (j ^ ((t >> 1) & 3)); a u32 column keeps 32 B as two units at
// t*2 + (j ^ ((t >> 2) & 1)).  Both the coalesced cp.async writes (consecutive units) and the per-thread
// 128-bit reads (unit j of 8 consecutive threads) then touch all 32 banks once.
__device__ __forceinline__ int sw64(int t, int j) { return t * 4 + (j ^ ((t >> 1) & 3)); }
__device__ __forceinline__ int sw32(int t, int j) { return t * 2 + (j ^ ((t >> 2) & 1)); }


constexpr int EV_WARPS = EV_NT / 32;
struct EvSmem {
    static constexpr int NT = EV_NT, TILE = EV_TILE, WARPS = EV_WARPS;
    longlong2 col[4][EV_TILE / 2];        // t_l, t_ks, t_ke, pred_end (64 KB)
    uint4 meta[EV_TILE / 4];              // 8 KB
    unsigned long long key[EV_IPT][EV_NT];  // instance key per event, [k][thread] (16 KB)
    Acc wagg[EV_WARPS], wcarry[EV_WARPS];
    int wflag[EV_WARPS], wcflag[EV_WARPS];
    int wheads[EV_WARPS];
    int64_t tile, excl;
    int tot;
};
// element k of thread t in the swizzled layouts
template <class SM>
__device__ __forceinline__ int64_t ev_col(const SM &S, int c, int t, int k) {
    return reinterpret_cast<const int64_t *>(&S.col[c][sw64(t, k >> 1)])[k & 1];
}
template <class SM>
__device__ __forceinline__ uint32_t ev_meta(const SM &S, int t, int k) {
    return reinterpret_cast<const uint32_t *>(&S.meta[sw32(t, k >> 2)])[k & 3];
}

template <class SM>
__device__ __forceinline__ void stage_tile(SM &S, const EvParams &P, int64_t base, bool vec) {
    const int tid = threadIdx.x;
    const int64_t *src[4] = {P.tl, P.ks, P.ke, P.pred_end};
    if (vec) {
#pragma unroll
        for (int c = 0; c < 4; c++) {
#pragma unroll
            for (int r = 0; r < 4; r++) {
                int u = tid + r * SM::NT;    // 16 B unit of the column: events 2u, 2u+1
                cp_async16(&S.col[c][sw64(u >> 2, u & 3)], src[c] + base + 2 * u);
            }
        }
#pragma unroll
        for (int r = 0; r < 2; r++) {
            int u = tid + r * SM::NT;        // events 4u .. 4u+3
            cp_async16(&S.meta[sw32(u >> 1, u & 1)], P.meta + base + 4 * u);
        }
        cp_async_wait_all();
        __syncthreads();
    } else {
        // partial or unaligned tile: element-wise, same layout
        for (int e = tid; e < SM::TILE; e += SM::NT) {
            int64_t i = base + e;
            int t = e >> 3, k = e & 7;
            int64_t *dst;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                dst = reinterpret_cast<int64_t *>(&S.col[c][sw64(t, k >> 1)]) + (k & 1);
                *dst = i < P.N ? src[c][i] : 0;
            }
            reinterpret_cast<uint32_t *>(&S.meta[sw32(t, k >> 2)])[k & 3] = i < P.N ? P.meta[i] : 0u;
        }
    }
    __syncthreads();
}


// ---- sub-run heads: the tile start is always a head (sub-runs never cross tiles); block exclusive scan of
// the per-thread head counts.  Keys of the tile are in S.key (written before the call).
__device__ __forceinline__ int tile_head_scan(EvSmem &S, unsigned &hmask, int nv, int *tot_out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __syncthreads();
    if (nv > 0 && (tid == 0 || S.key[0][tid] != S.key[EV_IPT - 1][tid - 1])) hmask |= 1u;
    const int nh = __popc(hmask);
    int wex = nh;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(CH_FULL, wex, o);
        if (lane >= o) wex += y;
    }
    if (lane == 31) S.wheads[warp] = wex;
    wex -= nh;
    __syncthreads();
    int wbase = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < EV_WARPS; w++) {
        int c = S.wheads[w];
        if (w < warp) wbase += c;
        tot += c;
    }
    *tot_out = tot;
    return wbase + wex;
}

// the same scan when the caller has already decided whether the thread's first event is a head
template <class SM>
__device__ __forceinline__ int tile_head_scan_h(SM &S, unsigned &hmask, bool head0, int *tot_out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (head0) hmask |= 1u;
    const int nh = __popc(hmask);
    int wex = nh;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(CH_FULL, wex, o);
        if (lane >= o) wex += y;
    }
    if (lane == 31) S.wheads[warp] = wex;
    wex -= nh;
    __syncthreads();
    int wbase = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < SM::WARPS; w++) {
        int c = S.wheads[w];
        if (w < warp) wbase += c;
        tot += c;
    }
    *tot_out = tot;
    return wbase + wex;
}

// ---- decoupled look-back (warp 0, 32 predecessors per probe): global id of the tile's first head ----
__device__ __forceinline__ void tile_lookback(EvSmem &S, const EvParams &P, int64_t tile, int tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {
        int64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&P.tile_state[0], FLAG_P | (unsigned long long)tot);
        } else {
            if (lane == 0) atomicExch(&P.tile_state[tile], FLAG_A | (unsigned long long)tot);
            int64_t p = tile - 1 - lane;
            while (true) {
                unsigned long long s = (unsigned long long)FLAG_P;
                if (p >= 0) s = *((volatile unsigned long long *)&P.tile_state[p]);
                unsigned fl = (unsigned)(s >> 62);
                unsigned pm = __ballot_sync(CH_FULL, fl == 2u), zm = __ballot_sync(CH_FULL, fl == 0u);
                int fp = pm ? __ffs(pm) - 1 : 32;
                unsigned need = fp >= 31 ? CH_FULL : ((2u << fp) - 1u);
                if (zm & need) continue;                       // a predecessor has not published yet
                int64_t v = lane <= fp ? (int64_t)(s & VAL_MASK) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CH_FULL, v, o);
                excl += v;
                if (fp < 32) break;
                p -= 32;
            }
            if (lane == 0) atomicExch(&P.tile_state[tile], FLAG_P | (unsigned long long)(excl + tot));
        }
        if (lane == 0) { S.excl = excl; S.tot = tot; }
    }
    __syncthreads();
}

// ---- runs that span threads: segmented inclusive scan of (has, tail-or-whole) over the tile ----
template <class SM>
__device__ __forceinline__ void tile_finish(SM &S, const EvParams &P, bool has, const Acc &cur, const Acc &p0,
                                            int64_t run0, int64_t base) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t N = P.N;
    bool f = has;
    Acc v = cur;
    if (!__all_sync(CH_FULL, has)) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            Acc pv = v.shfl_up(o);
            bool pf = __shfl_up_sync(CH_FULL, f, o);
            if (lane >= o) {
                if (!f) { pv.merge(v); v = pv; }
                f = f || pf;
            }
        }
    }
    if (lane == 31) { S.wagg[warp] = v; S.wflag[warp] = f; }
    __syncthreads();
    if (tid < SM::WARPS) {                 // carry into warp tid: segmented combine of earlier warps
        Acc c;
        c.zero();
        int cf = 0;
#pragma unroll
        for (int w = 0; w < SM::WARPS - 1; w++) {   // unrolled, predicated: the shared loads issue together
            if (w < tid) {
                if (S.wflag[w]) { c = S.wagg[w]; cf = 1; }
                else c.merge(S.wagg[w]);
            }
        }
        S.wcarry[tid] = c;
        S.wcflag[tid] = cf;
    }
    __syncthreads();
    // exclusive value at this thread: warp-exclusive, completed with the warp carry if no head precedes
    Acc e = v.shfl_up(1);
    bool ef = __shfl_up_sync(CH_FULL, f, 1);
    if (lane == 0) { e.zero(); ef = false; }
    if (!ef) {
        Acc c = S.wcarry[warp];
        c.merge(e);
        e = c;
    }
    // the run that ends in this thread's first piece (or at the end of the previous thread)
    if (has && tid > 0) {
        e.merge(p0);
        write_subrun(P, run0 - 1, e, base);
    }
    // the run open at the end of the tile
    if (tid == SM::NT - 1 && base < N) {
        Acc last = v;
        if (!f) {
            Acc c = S.wcarry[warp];
            c.merge(v);
            last = c;
        }
        write_subrun(P, S.excl + S.tot - 1, last, base);
    }
}

// first sub-run id of every tile from the look-back states (inclusive prefixes) of k_events
__global__ void k_tile_sub_state(const unsigned long long *__restrict__ state, int64_t ntile,
                                 int64_t *__restrict__ tile_sub) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) tile_sub[0] = 0;
    if (t < ntile) tile_sub[t + 1] = (int64_t)(state[t] & VAL_MASK);
}

// the chain predecessor column of a lean-loaded trace (general event passes read it)
__global__ void k_pred_lean(PredView pv, int64_t n, int64_t *__restrict__ pred_end) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) pred_end[i] = kind_of(pv.meta[i]) == CK_COMPUTE ? pred_of(pv, i) : CH_NONE_TS;
}

// the fused pass: one 2048-event tile per block, 8 consecutive events per thread
__global__ void __launch_bounds__(EV_NT, 2) k_events(EvParams P, int vec_ok) {
    extern __shared__ __align__(16) unsigned char ev_dsm[];
    EvSmem &S = *reinterpret_cast<EvSmem *>(ev_dsm);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) S.tile = (int64_t)atomicAdd(P.ticket, 1u);
    __syncthreads();
    const int64_t tile = S.tile;
    const int64_t base = tile * EV_TILE;
    const int64_t i0 = base + (int64_t)tid * EV_IPT;
    const int64_t N = P.N;
    stage_tile(S, P, base, vec_ok && base + EV_TILE <= N);
    const int nv = i0 >= N ? 0 : (int)min((int64_t)EV_IPT, N - i0);    // valid events of this thread

    // ---- phase 0: seeds for the span, comm-union and sample caches (lanes of one gpu) ----
    int32_t seed[6];
    int seed_lg;
    {
        int64_t t0 = 0, ksc = 0;
        bool hc = false;
        int lg0 = -1;
        if (nv > 0) {
            t0 = reinterpret_cast<const int64_t *>(&S.col[0][sw64(tid, 0)])[0];
            lg0 = P.gpu_lg[gpu_of(reinterpret_cast<const uint32_t *>(&S.meta[sw32(tid, 0)])[0])];
            for (int k = 0; k < nv && !hc; k++) {
                uint32_t m = reinterpret_cast<const uint32_t *>(&S.meta[sw32(tid, k >> 2)])[k & 3];
                if (kind_of(m) == CK_COMPUTE && P.gpu_lg[gpu_of(m)] == lg0) {
                    ksc = reinterpret_cast<const int64_t *>(&S.col[1][sw64(tid, k >> 1)])[k & 1];
                    hc = true;
                }
            }
        }
        const int lgw = __shfl_sync(CH_FULL, lg0, 0);
        const bool mine = nv > 0 && lg0 == lgw && lgw >= 0;
        SeedQ qs[6];
        const int64_t *lb = P.sv.list_beg;
#pragma unroll
        for (int lv = 0; lv < 4; lv++) {
            qs[lv].a = P.sv.P_start;
            qs[lv].lo = lgw >= 0 ? lb[lgw * 4 + lv] : 0;
            qs[lv].hi = lgw >= 0 ? lb[lgw * 4 + lv + 1] : 0;
            qs[lv].t = t0;
            qs[lv].on = mine && lgw >= 0 && !P.sv.list_flags[lgw * 4 + lv];
        }
        qs[4].a = P.Us;
        qs[4].lo = lgw >= 0 ? P.Ubeg[lgw] : 0;
        qs[4].hi = lgw >= 0 ? P.Ubeg[lgw] + P.Ucnt[lgw] : 0;
        qs[4].t = ksc;
        qs[4].on = mine && hc;
        qs[5].a = P.smp_ts;
        qs[5].lo = lgw >= 0 ? P.smp_lo[lgw] : 0;
        qs[5].hi = lgw >= 0 ? P.smp_hi[lgw] : 0;
        qs[5].t = ksc;
        qs[5].on = mine && hc;
        warp_seeds<6>(qs, seed);
        seed_lg = mine ? lgw : -1;
    }

    // ---- phase A: instance key of every event (attribution, a5) ----
    unsigned hmask = 0;
    {
        LvCache lc[4];
        int lgp = -1;
        unsigned long long prevk = CH_INVALID_KEY;
#pragma unroll 1
        for (int k = 0; k < EV_IPT; k++) {           // one event per iteration: one inlined copy of the lookups
            unsigned long long kk = CH_INVALID_KEY;
            if (k < nv) {
                const int64_t i = i0 + k;
                const int64_t t = ev_col(S, 0, tid, k);
                const int lg = P.gpu_lg[gpu_of(ev_meta(S, tid, k))];
                if (lg != lgp) {
#pragma unroll
                    for (int lv = 0; lv < 4; lv++)
                        lv_reset(lc[lv], P.sv, lg * 4 + lv, lgp < 0 && lg == seed_lg ? seed[lv] : -2);
                    lgp = lg;
                }
                int32_t r[4];
                bool ok = true;
#pragma unroll
                for (int lv = 0; lv < 4; lv++) {
                    int32_t c = lv_lookup(lc[lv], P.sv, lv, t, i);
                    ok &= c != -2;
                    r[lv] = c >= 0 ? c - lc[lv].lb + 1 : 0;
                }
                if (ok && r[0] != 0)
                    kk = ((unsigned long long)lg << P.sh_lg) | ((unsigned long long)r[0] << P.sh_it) |
                         ((unsigned long long)r[1] << P.sh_ph) | ((unsigned long long)r[2] << P.sh_ly) |
                         (unsigned long long)r[3];
                if (k > 0 && kk != prevk) hmask |= 1u << k;
            }
            S.key[k][tid] = kk;
            prevk = kk;
        }
    }
    int tot;
    const int ex = tile_head_scan(S, hmask, nv, &tot);   // heads before this thread in the tile
    tile_lookback(S, P, tile, tot);
    const int64_t run0 = S.excl + ex;     // global id of this thread's first head
    if (P.t_run) {                        // the counter pass's view of the runs: 5 B per thread
        P.t_run[tile * (int64_t)blockDim.x + threadIdx.x] = (int32_t)(run0 - 1);    // (k_events: ticketed tiles)
        P.t_hm[tile * (int64_t)blockDim.x + threadIdx.x] = (uint8_t)hmask;
    }

    // ---- phase B: per-event values (a6-a8), outputs, thread-sequential folding (a9) ----
    Acc cur, p0;
    cur.zero();
    p0.zero();
    bool has = false;
    int64_t curid = run0 - 1;
    CovCache cc;
    SmpCache sc;
    bool smp = false;
    int lgp = -1;
#pragma unroll 1
    for (int k = 0; k < EV_IPT; k++) {              // one event per iteration (one inlined copy of the caches)
        {
            if (k >= nv) break;
            const int64_t i = i0 + k;
            const uint32_t m = ev_meta(S, tid, k);
            const int lg = P.gpu_lg[gpu_of(m)];
            if (lg != lgp) {
                cov_reset(cc, P.Ubeg[lg], P.Ucnt[lg]);
                int64_t slo = P.smp_lo[lg], shi = P.smp_hi[lg];
                smp = shi > slo;
                smp_reset(sc, slo, shi);
                if (lgp < 0 && lg == seed_lg) {
                    if (seed[4] != -2) cov_seed(cc, P.Us, P.Ue, P.UP, seed[4]);
                    if (seed[5] != -2 && smp) smp_seed(sc, P, seed[5]);
                }
                lgp = lg;
            }
            if ((hmask >> k) & 1u) {
                if (!has) { p0 = cur; has = true; }
                else write_subrun(P, curid, cur, base);
                curid++;
                cur.zero();
                if (curid < P.cap) {
                    P.sr_key[curid] = S.key[k][tid];
                    P.sr_first[curid] = i;
                }
            }
            const int kd = kind_of(m);
            const int64_t ks = ev_col(S, 1, tid, k), ke = ev_col(S, 2, tid, k);
            const int64_t dur = ke - ks;
            int64_t ovl = 0, prep = 0, call = 0, phi = 0, psi = 0;
            cur.nev += 1;
            if (kd == CK_COMPUTE) {
                const int64_t pe = ev_col(S, 3, tid, k);
                if (pe != CH_NONE_TS) {
                    const int64_t tl = ev_col(S, 0, tid, k);
                    const int64_t t2 = tl < ks ? tl : ks;                  // D6: dispatch clamped to start
                    const int64_t a = t2 - pe;
                    prep = a > 0 ? a : 0;                                   // Eq. 1
                    const int64_t c1 = ks - t2, c2 = ks - pe;
                    const int64_t c = c1 < c2 ? c1 : c2;                    // Eq. 2
                    call = c > 0 ? c : 0;
                }
                const int64_t c_ks = cov_c(cc, P.Us, P.Ue, P.UP, ks);
                const int64_t c_ke = cov_c(cc, P.Us, P.Ue, P.UP, ke);
                ovl = c_ke - c_ks;                                          // |[t_ks, t_ke) ∩ U_g| (D9)
                if (smp) {
                    int64_t Fa, Pa, Fb, Pb;
                    smp_F(sc, P, ks, &Fa, &Pa);
                    smp_F(sc, P, ke, &Fb, &Pb);
                    phi = Fb - Fa;                                          // MHz*ns
                    psi = Pb - Pa;                                          // mW*ns
                }
                cur.n += 1;
                cur.busy += dur;
                cur.prep += prep;
                cur.call += call;
                cur.ovl += ovl;
                cur.phi += phi;
                cur.psi += psi;
                if (ks < cur.fks || (ks == cur.fks && tid * EV_IPT + k < cur.foff)) {
                    cur.fks = ks;
                    cur.foff = tid * EV_IPT + k;
                }
                if (ke > cur.lke) cur.lke = ke;
            } else {
                if (kd == CK_COPY || kd == CK_OTHER) cur.copy += dur;
                else if (kd == CK_AG) cur.ag += dur;
                else if (kd == CK_RS) cur.rs += dur;
                // communication overlap with the compute union feeds no table: k_covl writes it (full mode)
            }
            if (P.o_ovl && !is_comm(kd)) P.o_ovl[i] = ovl;
            if (P.o_prep) P.o_prep[i] = prep;
            if (P.o_call) P.o_call[i] = call;
            if (P.o_phi) P.o_phi[i] = phi;
            if (P.o_psi) P.o_psi[i] = psi;
        }
    }

    tile_finish(S, P, has, cur, p0, run0, base);
}

// =================================================================================================
// Window-staged event pass (every span list laminar).  The per-event lookups become forward walks over
// shared-memory windows of six sorted tables: the Euler boundary tables of the four span levels (spans.cu:
// the innermost owner is a direct read, no parent walk), the merged comm union and the sample stream.
// k_tile_seeds finds, per tile, the entry each table's window starts at (last entry <= the tile's first
// query); the window ends at the next tile's seed, which bounds every query of the tile when the gpu's
// queries are monotone (dispatch times always; compute start/end times on one compute stream).  Queries
// outside a window (several compute streams, a tile straddling two gpus, a window larger than the pool)
// take a binary search over the whole table in global memory: same answer, slower.
// =================================================================================================
constexpr int NTAB = 2;                // 0 combined key table (by dispatch time), 1 timeline (by start / end time)
constexpr int W_NT = 256, W_TILE = W_NT * EV_IPT, W_WARPS = W_NT / 32;   // 2048-event tiles, 2 blocks per SM
constexpr int POOL = 28672;            // bytes of staged windows per tile
constexpr int SEED_W = 4;              // per tile: 2 seeds, the tile's gpu (lg), pad
constexpr int KT_B = 16, TL_B = 44;    // staged bytes per entry: time + key; time + 3 intercepts + 3 slopes

struct TabWin {
    int64_t lo;           // global index of window entry 0 (the gpu's table starts with a -inf sentinel)
    int64_t gb, ge;       // the gpu's table in global memory
    int64_t next;         // time of the entry after the window (INT64_MAX at the table end)
    int n, off;           // staged entries, byte offset in the pool
};
struct TileWin {          // per tile: both windows, placed (k_tile_windows), and the tile's gpu
    TabWin tw[2];
    int64_t lg;
};
struct EvSmemW {
    static constexpr int NT = W_NT, TILE = W_TILE, WARPS = W_WARPS;
    longlong2 col[4][W_TILE / 2];         // t_l, t_ks, t_ke, pred_end (32 KB)
    uint4 meta[W_TILE / 4];               // 4 KB
    uint32_t kidx[EV_IPT][W_NT];          // key of each event as a key-table index (4 KB), see key_at
    unsigned long long lastk[W_NT];       // key of each thread's last event slot
    Acc wagg[W_WARPS], wcarry[W_WARPS];
    int wflag[W_WARPS], wcflag[W_WARPS];
    int wheads[W_WARPS];
    int64_t tile, excl;
    int tot;
    TabWin tw[NTAB];
    int lgP;
    __align__(16) unsigned char pool[POOL];
};
static_assert(sizeof(EvSmemW) <= 113 * 1024, "two event-pass blocks per SM");

__device__ __forceinline__ void tab_bounds(const EvParams &P, int x, int lg, int64_t *gb, int64_t *ge) {
    if (x == 0) { *gb = P.kt_beg[lg]; *ge = P.kt_beg[lg + 1]; }
    else { *gb = P.tl_beg[lg]; *ge = *gb + P.tl_len[lg]; }
}

// per tile: the entry each window starts at -- last entry <= the tile's first dispatch (key table) and <= the
// start of its first COMPUTE event among the first 32 (timeline)
__global__ void k_tile_seeds(EvParams P, int32_t *__restrict__ seeds) {
    const int lane = threadIdx.x & 31;
    const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (tile >= P.ntile) return;
    const int64_t base = tile * W_TILE, i = base + lane;
    const int lg = P.gpu_lg[gpu_of(P.meta[base])];
    const uint32_t m = i < P.N ? P.meta[i] : 0u;
    const bool cmp = i < P.N && kind_of(m) == CK_COMPUTE && P.gpu_lg[gpu_of(m)] == lg;
    const unsigned cm = __ballot_sync(CH_FULL, cmp);
    int64_t s = 0;
    if (lane < NTAB) {
        const int64_t t = lane == 0 ? P.tl[base] : (cm ? P.ks[base + __ffs(cm) - 1] : P.tl[base]);
        int64_t gb, ge;
        tab_bounds(P, lane, lg, &gb, &ge);
        s = last_le(lane == 0 ? P.KTt : P.TLt, gb, ge, t);     // >= gb: entry 0 is -inf
    } else if (lane == NTAB) {
        s = lg;
    }
    if (lane < SEED_W) seeds[tile * SEED_W + lane] = (int32_t)s;
}

// Windows of the tile: bounds from this tile's and the next tile's seeds (threads 0, 1), pool placement (thread 0;
// a window that does not fit is cut short), then cp.async copies by all threads (the caller waits).
// Windows of every tile, one thread per tile: from this tile's seed to the next tile's (same gpu), placed in the
// shared-memory pool (timeline first, then the key table; a window that does not fit is cut short and later
// queries read global memory), with the time of the first entry after each window.
__global__ void k_tile_windows(EvParams P, TileWin *__restrict__ out) {
    const int64_t tile = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= P.ntile) return;
    const int32_t *sd = P.seeds + tile * SEED_W;
    const int lg = sd[NTAB];
    TileWin r;
    r.lg = lg;
    int off = 0;
#pragma unroll
    for (int x = NTAB - 1; x >= 0; x--) {
        TabWin &w = r.tw[x];
        tab_bounds(P, x, lg, &w.gb, &w.ge);
        int64_t lo = sd[x], hi = w.ge;
        if (tile + 1 < P.ntile && sd[SEED_W + NTAB] == lg) {
            hi = (int64_t)sd[SEED_W + x] + 1 + (x == 1 ? 4 : 0);    // timeline: a little slack
            if (hi < lo + 1) hi = lo + 1;
            if (hi > w.ge) hi = w.ge;
        }
        const int eb = x == 0 ? KT_B : TL_B;
        int64_t n = hi - lo, fit = (POOL - off) / eb;
        if (n > fit) n = fit & ~3;
        w.lo = lo;
        w.n = (int)n;
        w.off = off;
        off += (int)((n * eb + 15) & ~15);
        const int64_t *T = x == 0 ? P.KTt : P.TLt;
        w.next = lo + n < w.ge ? T[lo + n] : INT64_MAX;
    }
    out[tile] = r;
}

__device__ __forceinline__ void stage_windows(EvSmemW &W, const EvParams &P, int64_t tile) {
    const int tid = threadIdx.x;
    if (tid < NTAB) W.tw[tid] = P.twin[tile].tw[tid];
    if (tid == 0) W.lgP = (int)P.twin[tile].lg;
    __syncthreads();
    {
        const TabWin w = W.tw[0];
        unsigned char *b = W.pool + w.off;
        for (int j = tid; j < w.n; j += W_NT) {
            cp_async8(b + 8 * j, P.KTt + w.lo + j);
            cp_async8(b + 8 * (w.n + j), P.KTk + w.lo + j);
        }
    }
    {
        const TabWin w = W.tw[1];
        unsigned char *b = W.pool + w.off;
        const int64_t cap = P.tl_cap;
        for (int j = tid; j < w.n; j += W_NT) {
            const int64_t g = w.lo + j;
            cp_async8(b + 8 * j, P.TLt + g);
            cp_async8(b + 8 * (w.n + j), P.TLv + g);
            cp_async8(b + 8 * (2 * w.n + j), P.TLv + cap + g);
            cp_async8(b + 8 * (3 * w.n + j), P.TLv + 2 * cap + g);
            cp_async4(b + 32 * w.n + 4 * j, P.TLs + g);
            cp_async4(b + 36 * w.n + 4 * j, P.TLs + cap + g);
            cp_async4(b + 40 * w.n + 4 * j, P.TLs + 2 * cap + g);
        }
    }
}

// A lookup table of one gpu, [gb, ge) in global memory (entry gb = -inf sentinel), with entries [lo, lo + n)
// staged in shared memory.  Lookups walk the staged copy; a query beyond it (a window cut short, a second
// gpu's events in the tile, an earlier time on another compute stream) reads the same table in global memory:
// latency, never a different answer.
struct WinR {
    const int64_t *T;     // staged times (payload follows)
    const int64_t *G;     // global time column
    int64_t lo, gb, ge, next;
    int n;
};
__device__ __forceinline__ WinR win_reg(const EvSmemW &W, int x, const EvParams &P) {
    const TabWin &w = W.tw[x];
    WinR r;
    r.T = reinterpret_cast<const int64_t *>(W.pool + w.off);
    r.G = x == 0 ? P.KTt : P.TLt;
    r.lo = w.lo;
    r.n = w.n;
    r.gb = w.gb;
    r.ge = w.ge;
    r.next = w.next;
    return r;
}
// a global-only view of table x of gpu lg (events of a second gpu in the tile); out of line, it is rare
__device__ __noinline__ longlong2 tab_bounds_ool(const int64_t *beg, const int64_t *len, int lg) {
    const int64_t b = beg[lg];
    return make_longlong2(b, len ? b + len[lg] : beg[lg + 1]);
}
__device__ __forceinline__ WinR win_global(const EvParams &P, int x, int lg) {
    WinR r;
    r.T = nullptr;
    r.G = x == 0 ? P.KTt : P.TLt;
    r.lo = 0;
    r.n = 0;
    const longlong2 b = x == 0 ? tab_bounds_ool(P.kt_beg, nullptr, lg) : tab_bounds_ool(P.tl_beg, P.tl_len, lg);
    r.gb = b.x;
    r.ge = b.y;
    r.next = INT64_MAX;
    return r;
}
__device__ __forceinline__ bool win_in(const WinR &w, int64_t j) { return (uint64_t)(j - w.lo) < (uint64_t)w.n; }
__device__ __forceinline__ int64_t win_t(const WinR &w, int64_t j) {
    return win_in(w, j) ? w.T[j - w.lo] : __ldg(w.G + j);
}
// slow path: last entry <= t over [gb, ge) in global memory, starting from the cursor when it is behind t
__device__ __noinline__ longlong2 seek_global(const int64_t *G, const int64_t *T, int64_t lo, int n, int64_t gb,
                                              int64_t ge, int64_t j, int64_t t) {
    int64_t l = gb;
    if (j >= gb && j < ge && __ldg(G + j) <= t) {
        // forward walk first (queries mostly increase; consecutive entries share L1 lines), then bisect
        for (int s = 0; s < 16; s++) {
            if (j + 1 >= ge || __ldg(G + j + 1) > t) {
                const int64_t b = j + 1 >= ge ? INT64_MAX
                                              : ((uint64_t)(j + 1 - lo) < (uint64_t)n ? T[j + 1 - lo] : __ldg(G + j + 1));
                return make_longlong2(j, b);
            }
            j++;
        }
        // gallop: G[j] <= t; double the step until an entry past t (or the end) bounds the search
        int64_t step = 32, hi = ge;
        while (j + step < ge) {
            if (__ldg(G + j + step) > t) { hi = j + step; break; }
            j += step;
            step <<= 1;
        }
        const int64_t r0 = last_le(G, j, hi, t);
        const int64_t b0 = r0 + 1 >= ge ? INT64_MAX
                                        : ((uint64_t)(r0 + 1 - lo) < (uint64_t)n ? T[r0 + 1 - lo] : __ldg(G + r0 + 1));
        return make_longlong2(r0, b0);
    }
    const int64_t r = last_le(G, l, ge, t);
    const int64_t b = r + 1 >= ge ? INT64_MAX : ((uint64_t)(r + 1 - lo) < (uint64_t)n ? T[r + 1 - lo] : __ldg(G + r + 1));
    return make_longlong2(r, b);
}
constexpr uint32_t KIDX_NONE = 0xFFFFFFFFu;   // event slot past the end of the events
// cursor: entry j answers every t in [a, b)
struct WCur {
    int64_t j, a, b;
};
__device__ __forceinline__ void wcur_init(WCur &k) { k.j = -1; k.a = INT64_MAX; k.b = INT64_MIN; }
// returns true when the cursor moved
__device__ __forceinline__ bool wcur_seek(const WinR &w, WCur &k, int64_t t) {
    if (t >= k.a && t < k.b) return false;
    int c = (int)(k.j - w.lo);
    if (!(win_in(w, k.j) && t >= k.a)) {
        // fresh position: binary search of the staged window when t is inside it
        c = -1;
        if (w.n > 0 && w.T[0] <= t) {
            int l = 1, h = w.n;
            while (l < h) {
                const int m = (l + h) >> 1;
                if (w.T[m] <= t) l = m + 1; else h = m;
            }
            c = l - 1;
        }
    }
    if (c >= 0) {
        while (c + 1 < w.n && w.T[c + 1] <= t) c++;            // forward walk in shared memory
        if (c + 1 < w.n) { k.j = w.lo + c; k.a = w.T[c]; k.b = w.T[c + 1]; return true; }
        if (t < w.next) { k.j = w.lo + c; k.a = w.T[c]; k.b = w.next; return true; }
    }
    const longlong2 r = seek_global(w.G, w.T, w.lo, w.n, w.gb, w.ge, k.j, t);
    k.j = r.x;
    k.a = win_t(w, r.x);
    k.b = r.y;
    return true;
}
__device__ __forceinline__ unsigned long long key_at(const WinR &w, const EvParams &P, int64_t j) {
    return win_in(w, j) ? reinterpret_cast<const unsigned long long *>(w.T + w.n)[j - w.lo] : __ldg(P.KTk + j);
}
// timeline entry j: intercepts (cov, F, Pw) and slopes (in-union, f, p)
struct TlEnt {
    unsigned long long v0, v1, v2;
    int32_t s0, s1, s2;
};
__device__ __forceinline__ TlEnt tl_ent(const WinR &w, const EvParams &P, int64_t j) {
    TlEnt e;
    if (win_in(w, j)) {
        const int c = (int)(j - w.lo);
        const int32_t *s32 = reinterpret_cast<const int32_t *>(w.T + 4 * w.n);
        e.v0 = w.T[w.n + c]; e.v1 = w.T[2 * w.n + c]; e.v2 = w.T[3 * w.n + c];
        e.s0 = s32[c]; e.s1 = s32[w.n + c]; e.s2 = s32[2 * w.n + c];
    } else {
        const int64_t cap = P.tl_cap;
        e.v0 = __ldg(P.TLv + j); e.v1 = __ldg(P.TLv + cap + j); e.v2 = __ldg(P.TLv + 2 * cap + j);
        e.s0 = __ldg(P.TLs + j); e.s1 = __ldg(P.TLs + cap + j); e.s2 = __ldg(P.TLs + 2 * cap + j);
    }
    return e;
}

// ---- sub-run heads per tile (first pass): the same keys and head rule as k_events_w, counted, so that the main
// pass knows every tile's first sub-run id up front (an exclusive scan of the counts) instead of waiting on a
// look-back chain that any slow tile would stall for all later ones.  Columns are read straight from global
// memory (8 consecutive events per thread, 16 B loads); only the key-table window is staged.
constexpr int HD_POOL = 28672;
__global__ void __launch_bounds__(W_NT, 4) k_tile_heads(EvParams P, int64_t *__restrict__ tile_cnt) {
    __shared__ __align__(16) unsigned char pool[HD_POOL];
    __shared__ int64_t s_lo, s_next;
    __shared__ int s_n, s_lg;
    __shared__ unsigned long long s_last[W_WARPS];
    __shared__ int s_cnt[W_WARPS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = blockIdx.x, base = tile * W_TILE, i0 = base + (int64_t)tid * EV_IPT, N = P.N;
    if (tid == 0) {
        const TabWin w = P.twin[tile].tw[0];
        int n = w.n;
        if (n > HD_POOL / KT_B) n = (HD_POOL / KT_B) & ~3;
        s_lo = w.lo; s_n = n; s_lg = (int)P.twin[tile].lg;
        s_next = n == w.n ? w.next : __ldg(P.KTt + w.lo + n);
    }
    __syncthreads();
    {
        const int64_t lo = s_lo;
        const int n = s_n;
        for (int j = tid; j < n; j += W_NT) {
            cp_async8(pool + 8 * j, P.KTt + lo + j);
            cp_async8(pool + 8 * (n + j), P.KTk + lo + j);
        }
    }
    int64_t tl[EV_IPT];
    uint32_t mt[EV_IPT];
    const int nv = i0 >= N ? 0 : (int)min((int64_t)EV_IPT, N - i0);
    if (nv == EV_IPT && ((((uintptr_t)(P.tl + i0)) | ((uintptr_t)(P.meta + i0))) & 15u) == 0) {
#pragma unroll
        for (int u = 0; u < EV_IPT / 2; u++) {
            const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(P.tl + i0) + u);
            tl[2 * u] = v.x; tl[2 * u + 1] = v.y;
        }
#pragma unroll
        for (int u = 0; u < EV_IPT / 4; u++) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(P.meta + i0) + u);
            mt[4 * u] = v.x; mt[4 * u + 1] = v.y; mt[4 * u + 2] = v.z; mt[4 * u + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < EV_IPT; k++) {
            tl[k] = k < nv ? P.tl[i0 + k] : 0;
            mt[k] = k < nv ? P.meta[i0 + k] : 0u;
        }
    }
    cp_async_wait_all();
    __syncthreads();
    const int lgP = s_lg;
    WinR wk;
    wk.T = reinterpret_cast<const int64_t *>(pool);
    wk.G = P.KTt;
    wk.lo = s_lo;
    wk.n = s_n;
    wk.gb = P.kt_beg[lgP];
    wk.ge = P.kt_beg[lgP + 1];
    wk.next = s_next;
    WCur ck;
    wcur_init(ck);
    int lgc = lgP;
    unsigned long long prevk = CH_INVALID_KEY, first = CH_INVALID_KEY;
    int64_t prevj = -1;
    int nh = 0;
    unsigned hm = 0;                      // head mask of the thread's 8 events (the event pass's rule)
    uint32_t kx[EV_IPT];                  // key-table index of each event (the lean event pass reads it)
#pragma unroll
    for (int k = 0; k < EV_IPT; k++) {
        kx[k] = KIDX_NONE;
        if (k < nv) {
            const int lg = P.gpu_lg[gpu_of(mt[k])];
            if (lg != lgc) { wk = win_global(P, 0, lg); wcur_init(ck); lgc = lg; }
            wcur_seek(wk, ck, tl[k]);
            kx[k] = (uint32_t)ck.j;
            if (ck.j != prevj) {
                const unsigned long long kk = key_at(wk, P, ck.j);
                if (k > 0 && kk != prevk) { nh++; hm |= 1u << k; }
                prevk = kk;
                prevj = ck.j;
            }
        } else {
            prevk = CH_INVALID_KEY;
            prevj = -1;
        }
        if (k == 0) first = prevk;
    }
    // head at the thread's first event: tile start, or a key change from the previous thread's last event
    unsigned long long pl = __shfl_up_sync(CH_FULL, prevk, 1);
    if (lane == 31) s_last[warp] = prevk;
    __syncthreads();
    if (lane == 0) pl = warp > 0 ? s_last[warp - 1] : CH_INVALID_KEY;
    if (nv > 0 && (tid == 0 || first != pl)) { nh++; hm |= 1u; }
    // in-tile exclusive head count before this thread (warp scan + warp totals)
    int inc = nh;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(CH_FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_cnt[warp] = inc;
    __syncthreads();
    int wb = 0, t = 0;
#pragma unroll
    for (int w = 0; w < W_WARPS; w++) {
        const int c = s_cnt[w];
        if (w < warp) wb += c;
        t += c;
    }
    if (tid == 0) tile_cnt[tile] = t;
    if (P.t_run) {                        // the counter pass's view: head mask + in-tile rank (plus the tile base there)
        P.t_run[tile * (int64_t)W_NT + tid] = wb + inc - nh;
        P.t_hm[tile * (int64_t)W_NT + tid] = (uint8_t)hm;
    }
    if (P.kidx) {                         // (the column has whole tiles: no bounds check)
        uint4 *o = reinterpret_cast<uint4 *>(P.kidx + i0);
        o[0] = make_uint4(kx[0], kx[1], kx[2], kx[3]);
        o[1] = make_uint4(kx[4], kx[5], kx[6], kx[7]);
    }
}

__global__ void __launch_bounds__(W_NT, 2) k_events_w(EvParams P, int vec_ok) {
    extern __shared__ __align__(16) unsigned char ev_dsm[];
    EvSmemW &S = *reinterpret_cast<EvSmemW *>(ev_dsm);
    const int tid = threadIdx.x;
    const int64_t tile = blockIdx.x;
    if (tid == 0) { S.excl = P.tile_base[tile]; S.tot = (int)(P.tile_base[tile + 1] - P.tile_base[tile]); }
    const int64_t base = tile * W_TILE;
    const int64_t i0 = base + (int64_t)tid * EV_IPT;
    const int64_t N = P.N;
    stage_windows(S, P, tile);
    stage_tile(S, P, base, vec_ok && base + W_TILE <= N);
    cp_async_wait_all();
    __syncthreads();
    const int nv = i0 >= N ? 0 : (int)min((int64_t)EV_IPT, N - i0);
    const int lgP = S.lgP;
    const WinR wkP = win_reg(S, 0, P);

    // ---- phase A: instance key of every event (a5): the combined key table at the dispatch time ----
    unsigned hmask = 0;
    unsigned long long firstk = CH_INVALID_KEY;
    {
        WinR wk = wkP;
        int lgc = lgP;
        WCur ck;
        wcur_init(ck);
        unsigned long long prevk = CH_INVALID_KEY;
        int64_t prevj = -1;
#pragma unroll 1
        for (int k = 0; k < EV_IPT; k++) {
            uint32_t v = KIDX_NONE;
            if (k < nv) {
                const int64_t t = ev_col(S, 0, tid, k);
                const int lg = P.gpu_lg[gpu_of(ev_meta(S, tid, k))];
                if (lg != lgc) { wk = win_global(P, 0, lg); wcur_init(ck); lgc = lg; }
                wcur_seek(wk, ck, t);
                v = (uint32_t)ck.j;
                if (ck.j != prevj) {                  // same entry => same key; else compare the keys
                    const unsigned long long kk = key_at(wk, P, ck.j);
                    if (k > 0 && kk != prevk) hmask |= 1u << k;
                    prevk = kk;
                    prevj = ck.j;
                }
            } else {
                prevk = CH_INVALID_KEY;
                prevj = -1;
            }
            if (k == 0) firstk = prevk;
            S.kidx[k][tid] = v;
        }
        S.lastk[tid] = prevk;
    }
    __syncthreads();
    int tot;
    const int ex = tile_head_scan_h(S, hmask, nv > 0 && (tid == 0 || firstk != S.lastk[tid - 1]), &tot);
    const int64_t run0 = S.excl + ex;
    if (P.t_run) {                        // the counter pass's view of the runs: 5 B per thread
        P.t_run[tile * (int64_t)blockDim.x + threadIdx.x] = (int32_t)(run0 - 1);    // (k_events: ticketed tiles)
        P.t_hm[tile * (int64_t)blockDim.x + threadIdx.x] = (uint8_t)hmask;
    }

    // ---- phase B: per-event values (a6-a8), outputs, thread-sequential folding (a9) ----
    Acc cur, p0;
    cur.zero();
    p0.zero();
    bool has = false;
    int64_t curid = run0 - 1;
    const WinR wtP = win_reg(S, 1, P);
    WinR wt = wtP;
    int lgc = lgP;
    WCur ct;
    wcur_init(ct);
    TlEnt te{};
#pragma unroll 1
    for (int k = 0; k < EV_IPT; k++) {
        if (k >= nv) break;
        const int64_t i = i0 + k;
        const uint32_t m = ev_meta(S, tid, k);
        const int lg = P.gpu_lg[gpu_of(m)];
        const bool prim = lg == lgP;
        if ((hmask >> k) & 1u) {
            if (!has) { p0 = cur; has = true; }
            else write_subrun(P, curid, cur, base);
            curid++;
            cur.zero();
            const uint32_t v = S.kidx[k][tid];
            if (curid < P.cap) {
                P.sr_key[curid] = key_at(prim ? wkP : win_global(P, 0, lg), P, (int64_t)v);
                P.sr_first[curid] = i;
            }
        }
        const int kd = kind_of(m);
        const int64_t ks = ev_col(S, 1, tid, k), ke = ev_col(S, 2, tid, k);
        const int64_t dur = ke - ks;
        int64_t ovl = 0, prep = 0, call = 0, phi = 0, psi = 0;
        cur.nev += 1;
        if (kd == CK_COMPUTE) {
            const int64_t pe = ev_col(S, 3, tid, k);
            if (pe != CH_NONE_TS) {
                const int64_t tl = ev_col(S, 0, tid, k);
                const int64_t t2 = tl < ks ? tl : ks;                  // D6: dispatch clamped to start
                const int64_t a = t2 - pe;
                prep = a > 0 ? a : 0;                                   // Eq. 1
                const int64_t c1 = ks - t2, c2 = ks - pe;
                const int64_t c = c1 < c2 ? c1 : c2;                    // Eq. 2
                call = c > 0 ? c : 0;
            }
            if (lg != lgc) { wt = win_global(P, 1, lg); wcur_init(ct); lgc = lg; }
            if (wcur_seek(wt, ct, ks)) te = tl_ent(wt, P, ct.j);
            if (ke < ct.b) {
                // one timeline entry covers [t_ks, t_ke): the integrals are its slopes times the duration
                ovl = te.s0 ? dur : 0;                                  // |[t_ks, t_ke) ∩ U_g| (D9)
                phi = (int64_t)te.s1 * dur;                             // MHz*ns (D10)
                psi = (int64_t)te.s2 * dur;                             // mW*ns
            } else {
                const unsigned long long ua = (unsigned long long)(ks - P.t0);
                const unsigned long long ca = te.v0 + (te.s0 ? ua : 0ull);
                const unsigned long long fa = te.v1 + (unsigned long long)(int64_t)te.s1 * ua;
                const unsigned long long pa = te.v2 + (unsigned long long)(int64_t)te.s2 * ua;
                wcur_seek(wt, ct, ke);
                te = tl_ent(wt, P, ct.j);
                const unsigned long long ub = (unsigned long long)(ke - P.t0);
                ovl = (int64_t)(te.v0 + (te.s0 ? ub : 0ull) - ca);
                phi = (int64_t)(te.v1 + (unsigned long long)(int64_t)te.s1 * ub - fa);
                psi = (int64_t)(te.v2 + (unsigned long long)(int64_t)te.s2 * ub - pa);
            }
            cur.n += 1;
            cur.busy += dur;
            cur.prep += prep;
            cur.call += call;
            cur.ovl += ovl;
            cur.phi += phi;
            cur.psi += psi;
            if (ks < cur.fks || (ks == cur.fks && tid * EV_IPT + k < cur.foff)) {
                cur.fks = ks;
                cur.foff = tid * EV_IPT + k;
            }
            if (ke > cur.lke) cur.lke = ke;
        } else {
            if (kd == CK_COPY || kd == CK_OTHER) cur.copy += dur;
            else if (kd == CK_AG) cur.ag += dur;
            else if (kd == CK_RS) cur.rs += dur;
        }
        if (P.o_ovl && !is_comm(kd)) P.o_ovl[i] = ovl;
        if (P.o_prep) P.o_prep[i] = prep;
        if (P.o_call) P.o_call[i] = call;
        if (P.o_phi) P.o_phi[i] = phi;
        if (P.o_psi) P.o_psi[i] = psi;
    }
    tile_finish(S, P, has, cur, p0, run0, base);
}

// =================================================================================================
// Lean event pass (the FSDP case: every span list laminar, one compute stream per gpu whose kernels are
// start-monotone in dispatch order -- the lean a2 of load.cu).  Same tiles, head rule, sub-run rows and
// results as k_events_w, built for the B200 memory system:
//   * the tile's event columns arrive by TMA: one elected thread issues 2-D tensor loads (t_l, t_ks, t_ke as
//     [rows of 8 int64], meta as [rows of 8 uint32]) whose hardware 64 B / 32 B swizzle is the thread-blocked
//     layout ev_col / ev_meta read (thread t owns row t: conflict-free 16 B shared loads), and 1-D bulk copies
//     (cp.async.bulk) of the key-table and timeline windows; one mbarrier with the transaction byte count;
//   * the launch chain (a7) needs no predecessor column: on one start-monotone compute stream the predecessor
//     of a COMPUTE kernel is the previous COMPUTE kernel of its gpu in dispatch order, so each thread carries
//     the last one's end through its 8 events, takes the value before its first event from a block scan of
//     (position, end), and the tile's carry-in comes from k_tile_seeds_l (a backward search before the tile);
//   * per-event outputs are compiled in only for full mode (OUT).
// =================================================================================================
constexpr int L_POOL = 28672;          // bytes of staged windows per tile (larger windows: global fallback)

struct TabWinL {
    int64_t lo, gb, ge, next;  // logical window [lo, lo + n) of the gpu's table [gb, ge); time after it
    int n, shift, a_n, off;    // copied: a_n entries from lo - shift (16 B-aligned), at byte off of the pool
};
struct TileWinL {
    TabWinL tw[2];
    int64_t lg;                // local gpu of the tile's first event
    int64_t pe;                // chain carry: end of the last COMPUTE event of that gpu before the tile, or NONE
};
struct EvSmemL {
    static constexpr int NT = W_NT, TILE = W_TILE, WARPS = W_WARPS;
    longlong2 col[3][W_TILE / 2];         // t_l, t_ks, t_ke (48 KB), 64 B-swizzled rows (TMA)
    uint4 meta[W_TILE / 4];               // 8 KB, 32 B-swizzled rows (TMA)
    uint32_t kidx[W_TILE];                // key of each event as a key-table index (8 KB, k_tile_heads; bulk copy)
    Acc wagg[W_WARPS], wcarry[W_WARPS];
    int wflag[W_WARPS], wcflag[W_WARPS];
    int wheads[W_WARPS];
    int32_t wpos[W_WARPS];                // chain scan: last COMPUTE position / end per warp
    int64_t wend[W_WARPS];
    int64_t tile, excl;
    int tot;
    unsigned long long bar[2];
    __align__(16) unsigned char pool[L_POOL];
};
static_assert(sizeof(EvSmemL) <= 113 * 1024, "two lean event-pass blocks per SM");

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *map, int c0, int c1, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// per tile (a warp each): the windows' seeds as k_tile_seeds, and the chain carry -- the end of the last COMPUTE
// event of the tile's first gpu before the tile (NONE when the gpu starts in this tile or has none before)
__global__ void k_tile_seeds_l(EvParams P, int32_t *__restrict__ seeds, int64_t *__restrict__ tile_pe) {
    const int lane = threadIdx.x & 31;
    const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (tile >= P.ntile) return;
    const int64_t base = tile * W_TILE, i = base + lane;
    const uint32_t m0 = P.meta[base];
    const int lg = P.gpu_lg[gpu_of(m0)];
    const uint32_t m = i < P.N ? P.meta[i] : 0u;
    const bool cmp = i < P.N && kind_of(m) == CK_COMPUTE && P.gpu_lg[gpu_of(m)] == lg;
    const unsigned cm = __ballot_sync(CH_FULL, cmp);
    int64_t s = lane == NTAB ? lg : 0;
#pragma unroll
    for (int x = 0; x < NTAB; x++) {          // (the whole warp searches each table: log32 dependent loads)
        const int64_t t = x == 0 ? P.tl[base] : (cm ? P.ks[base + __ffs(cm) - 1] : P.tl[base]);
        int64_t gb, ge;
        tab_bounds(P, x, lg, &gb, &ge);
        const int64_t r = warp_last_le(x == 0 ? P.KTt : P.TLt, gb, ge, t);
        if (lane == x) s = r;
    }
    if (lane < SEED_W) seeds[tile * SEED_W + lane] = (int32_t)s;
    // backward search for the chain carry, 32 events per probe
    int64_t pe = CH_NONE_TS;
    for (int64_t p = base - 1; p >= 0; p -= 32) {
        const int64_t q = p - lane;
        const uint32_t mq = q >= 0 ? P.meta[q] : 0u;
        const bool other = q < 0 || gpu_of(mq) != gpu_of(m0);
        const bool hit = !other && kind_of(mq) == CK_COMPUTE;
        const unsigned hm = __ballot_sync(CH_FULL, hit), om = __ballot_sync(CH_FULL, other);
        if (hm | om) {
            const int f = __ffs(hm | om) - 1;
            if ((hm >> f) & 1u) pe = P.ke[p - f];
            break;
        }
    }
    if (lane == 0) tile_pe[tile] = pe;
}

// window placement with 16 B-aligned copies: the key table (times, keys: 2 entries per 16 B) and the timeline
// (times, 3 intercepts, 3 int32 slopes: 4 entries per 16 B) are copied from an aligned start, the logical
// window begins `shift` entries in
__global__ void k_tile_windows_l(EvParams P, const int64_t *__restrict__ tile_pe, TileWinL *__restrict__ out) {
    const int64_t tile = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= P.ntile) return;
    const int32_t *sd = P.seeds + tile * SEED_W;
    const int lg = sd[NTAB];
    TileWinL r;
    r.lg = lg;
    r.pe = tile_pe[tile];
    int off = 0;
#pragma unroll
    for (int x = NTAB - 1; x >= 0; x--) {
        TabWinL &w = r.tw[x];
        tab_bounds(P, x, lg, &w.gb, &w.ge);
        int64_t lo = sd[x], hi = w.ge;
        if (tile + 1 < P.ntile && sd[SEED_W + NTAB] == lg) {
            hi = (int64_t)sd[SEED_W + x] + 1 + (x == 1 ? 4 : 0);
            if (hi < lo + 1) hi = lo + 1;
            if (hi > w.ge) hi = w.ge;
        }
        const int A = x == 0 ? 2 : 4, eb = x == 0 ? KT_B : TL_B;
        const int shift = (int)(lo & (A - 1));
        int64_t n = hi - lo;
        const int64_t fit = ((L_POOL - off) / eb) & ~(int64_t)(A - 1);
        if (shift + n > fit) n = fit - shift > 0 ? fit - shift : 0;
        const int a_n = n > 0 ? (int)((shift + n + A - 1) & ~(int64_t)(A - 1)) : 0;
        w.lo = lo;
        w.n = (int)n;
        w.shift = shift;
        w.a_n = a_n;
        w.off = off;
        off += a_n * eb;
        const int64_t *T = x == 0 ? P.KTt : P.TLt;
        w.next = lo + n < w.ge ? T[lo + n] : INT64_MAX;
    }
    out[tile] = r;
}

struct WinL {              // a staged window (logical entries [lo, lo + n)) of one table, or global only (n = 0)
    const int64_t *T;      // logical times
    const int64_t *G;      // global times
    int64_t lo, gb, ge, next;
    int n, stride, shift;  // payload column stride (entries) in the pool; logical start - aligned copy start
};
__device__ __forceinline__ WinL winl_reg(const TabWinL &w, const EvSmemL &S, int x, const EvParams &P) {
    WinL r;
    r.T = reinterpret_cast<const int64_t *>(S.pool + w.off) + w.shift;
    r.G = x == 0 ? P.KTt : P.TLt;
    r.lo = w.lo;
    r.n = w.n;
    r.stride = w.a_n;
    r.shift = w.shift;
    r.gb = w.gb;
    r.ge = w.ge;
    r.next = w.next;
    return r;
}
__device__ __forceinline__ WinL winl_global(const EvParams &P, int x, int lg) {
    WinL r;
    r.T = nullptr;
    r.G = x == 0 ? P.KTt : P.TLt;
    r.lo = 0;
    r.n = 0;
    r.stride = 0;
    r.shift = 0;
    const longlong2 b = x == 0 ? tab_bounds_ool(P.kt_beg, nullptr, lg) : tab_bounds_ool(P.tl_beg, P.tl_len, lg);
    r.gb = b.x;
    r.ge = b.y;
    r.next = INT64_MAX;
    return r;
}
__device__ __forceinline__ bool winl_in(const WinL &w, int64_t j) { return (uint64_t)(j - w.lo) < (uint64_t)w.n; }
__device__ __forceinline__ bool winl_seek(const WinL &w, WCur &k, int64_t t) {
    if (t >= k.a && t < k.b) return false;
    int c = (int)(k.j - w.lo);
    if (!(winl_in(w, k.j) && t >= k.a)) {
        c = -1;
        if (w.n > 0 && w.T[0] <= t) {
            int l = 1, h = w.n;
            while (l < h) {
                const int mm = (l + h) >> 1;
                if (w.T[mm] <= t) l = mm + 1; else h = mm;
            }
            c = l - 1;
        }
    }
    if (c >= 0) {
        while (c + 1 < w.n && w.T[c + 1] <= t) c++;
        if (c + 1 < w.n) { k.j = w.lo + c; k.a = w.T[c]; k.b = w.T[c + 1]; return true; }
        if (t < w.next) { k.j = w.lo + c; k.a = w.T[c]; k.b = w.next; return true; }
    }
    const longlong2 r = seek_global(w.G, w.T, w.lo, w.n, w.gb, w.ge, k.j, t);
    k.j = r.x;
    k.a = winl_in(w, r.x) ? w.T[r.x - w.lo] : __ldg(w.G + r.x);
    k.b = r.y;
    return true;
}
__device__ __forceinline__ unsigned long long keyl_at(const WinL &w, const EvParams &P, int64_t j) {
    return winl_in(w, j) ? reinterpret_cast<const unsigned long long *>(w.T + w.stride)[j - w.lo] : __ldg(P.KTk + j);
}
__device__ __forceinline__ TlEnt tll_ent(const WinL &w, const EvParams &P, int64_t j) {
    TlEnt e;
    if (winl_in(w, j)) {
        // copy layout (from the aligned start): times, 3 intercept columns (int64), 3 slope columns (int32), each
        // column `stride` entries; T is the logical start, so every column is offset by the same shift
        const int c = (int)(j - w.lo), st = w.stride;
        const int64_t *v = w.T + st;
        e.v0 = v[c]; e.v1 = v[st + c]; e.v2 = v[2 * st + c];
        const int32_t *s0 = reinterpret_cast<const int32_t *>(w.T - w.shift + 4 * st) + w.shift;
        e.s0 = s0[c]; e.s1 = s0[st + c]; e.s2 = s0[2 * st + c];
    } else {
        const int64_t cap = P.tl_cap;
        e.v0 = __ldg(P.TLv + j); e.v1 = __ldg(P.TLv + cap + j); e.v2 = __ldg(P.TLv + 2 * cap + j);
        e.s0 = __ldg(P.TLs + j); e.s1 = __ldg(P.TLs + cap + j); e.s2 = __ldg(P.TLs + 2 * cap + j);
    }
    return e;
}

// element k of thread t in the TMA-swizzled rows (k is a constant after unrolling: one LOP for the swizzle)
__device__ __forceinline__ int64_t rcol(const EvSmemL &S, int c, int t, int x64, int k) {
    return reinterpret_cast<const int64_t *>(&S.col[c][t * 4 + ((k >> 1) ^ x64)])[k & 1];
}
__device__ __forceinline__ uint32_t rmeta(const EvSmemL &S, int t, int x32, int k) {
    return reinterpret_cast<const uint32_t *>(&S.meta[t * 2 + ((k >> 2) ^ x32)])[k & 3];
}
// the window of table x for gpu g: the staged one for the tile's gpu, else the gpu's table in global memory
// (inline: a non-inlined callee taking EvParams by reference would force a stack copy of the whole struct)
__device__ __forceinline__ WinL winl_for(const EvParams &P, int x, int g, int lgP, const WinL &staged) {
    const int lg = P.gpu_lg[g];
    return lg == lgP ? staged : winl_global(P, x, lg);
}

template <bool OUT>
__global__ void __launch_bounds__(W_NT, 2) k_events_l(EvParams P, const __grid_constant__ CUtensorMap tm_tl,
                                                      const __grid_constant__ CUtensorMap tm_ks,
                                                      const __grid_constant__ CUtensorMap tm_ke,
                                                      const __grid_constant__ CUtensorMap tm_meta) {
    extern __shared__ __align__(1024) unsigned char evl_dsm[];
    EvSmemL &S = *reinterpret_cast<EvSmemL *>(evl_dsm);       // the TMA swizzle needs a 1024 B-aligned base
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = blockIdx.x;
    const int64_t base = tile * W_TILE;
    const int64_t i0 = base + (int64_t)tid * EV_IPT;
    const int64_t N = P.N;
    // ---- staging: the columns by TMA (warp 0) and the key-table / timeline windows by bulk copies (warps 1, 2)
    // on two mbarriers; every thread reads the tile's scalars and window descriptors itself (broadcast loads),
    // so nobody waits at a barrier for another thread's global loads ----
    if (tid == 0) {
        if (smem_u32(evl_dsm) & 1023u) __trap();
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 2);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const TileWinL *twp = P.twinl + tile;
    if (tid == 0) {
        mbar_arrive_tx(&S.bar[0], 3u * 16384u + 8192u + 8192u);
        const int row = (int)(base >> 3);
        tma_2d(&S.col[0][0], &tm_tl, 0, row, &S.bar[0]);
        tma_2d(&S.col[1][0], &tm_ks, 0, row, &S.bar[0]);
        tma_2d(&S.col[2][0], &tm_ke, 0, row, &S.bar[0]);
        tma_2d(&S.meta[0], &tm_meta, 0, row, &S.bar[0]);
        bulk_g2s(&S.kidx[0], P.kidx + base, 8192u, &S.bar[0]);     // (the column has whole tiles)
        S.excl = P.tile_base[tile];
        S.tot = (int)(P.tile_base[tile + 1] - P.tile_base[tile]);
    } else if (tid == 32) {
        const TabWinL k = twp->tw[0];
        mbar_arrive_tx(&S.bar[1], (unsigned)k.a_n * KT_B);
        if (k.a_n > 0) {
            unsigned char *b = S.pool + k.off;
            const int64_t a0 = k.lo - k.shift;
            bulk_g2s(b, P.KTt + a0, 8u * k.a_n, &S.bar[1]);
            bulk_g2s(b + 8 * k.a_n, P.KTk + a0, 8u * k.a_n, &S.bar[1]);
        }
    } else if (tid == 64) {
        const TabWinL t = twp->tw[1];
        mbar_arrive_tx(&S.bar[1], (unsigned)t.a_n * TL_B);
        if (t.a_n > 0) {
            unsigned char *b = S.pool + t.off;
            const int64_t a0 = t.lo - t.shift, cap = P.tl_cap;
            const unsigned n8 = 8u * t.a_n, n4 = 4u * t.a_n;
            bulk_g2s(b, P.TLt + a0, n8, &S.bar[1]);
            bulk_g2s(b + n8, P.TLv + a0, n8, &S.bar[1]);
            bulk_g2s(b + 2 * n8, P.TLv + cap + a0, n8, &S.bar[1]);
            bulk_g2s(b + 3 * n8, P.TLv + 2 * cap + a0, n8, &S.bar[1]);
            bulk_g2s(b + 4 * n8, P.TLs + a0, n4, &S.bar[1]);
            bulk_g2s(b + 4 * n8 + n4, P.TLs + cap + a0, n4, &S.bar[1]);
            bulk_g2s(b + 4 * n8 + 2 * n4, P.TLs + 2 * cap + a0, n4, &S.bar[1]);
        }
    }
    const int lgP = (int)twp->lg;
    const int gP = gpu_of(__ldg(P.meta + base));
    mbar_wait(&S.bar[0], 0);
    mbar_wait(&S.bar[1], 0);
    const int nv = i0 >= N ? 0 : (int)min((int64_t)EV_IPT, N - i0);
    const int x64 = (tid >> 1) & 3, x32 = (tid >> 2) & 1;
    if (nv > 0 && nv < EV_IPT) {
        // the last partial row (N % 8 events) lies outside the tensor maps: this thread fills it in
        for (int k = 0; k < nv; k++) {
            const int64_t i = i0 + k;
            reinterpret_cast<int64_t *>(&S.col[0][tid * 4 + ((k >> 1) ^ x64)])[k & 1] = P.tl[i];
            reinterpret_cast<int64_t *>(&S.col[1][tid * 4 + ((k >> 1) ^ x64)])[k & 1] = P.ks[i];
            reinterpret_cast<int64_t *>(&S.col[2][tid * 4 + ((k >> 1) ^ x64)])[k & 1] = P.ke[i];
            reinterpret_cast<uint32_t *>(&S.meta[tid * 2 + ((k >> 2) ^ x32)])[k & 3] = P.meta[i];
        }
    }
    const WinL wkP = winl_reg(twp->tw[0], S, 0, P);

    // ---- phase A: the thread's last COMPUTE kernel (a7 chain).  The instance keys (a5) -- each event's
    // key-table index, the head masks and the in-tile head ranks -- come from the head pre-count ----
    const int64_t th = tile * (int64_t)W_NT + tid;
    unsigned hmask = P.h_hm[th];
    const int32_t hrank = P.h_run[th];
    int32_t lpos = -1;                         // tile offset of the thread's last COMPUTE event
    int64_t lend = 0;
#pragma unroll
    for (int k = 0; k < EV_IPT; k++)
        if (k < nv && kind_of(rmeta(S, tid, x32, k)) == CK_COMPUTE) { lpos = tid * EV_IPT + k; lend = rcol(S, 2, tid, x64, k); }
    // chain scan: the last COMPUTE event before this thread (position, end); the later position wins
    int32_t xpos = lpos;
    int64_t xend = lend;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t yp = __shfl_up_sync(CH_FULL, xpos, o);
        const int64_t ye = __shfl_up_sync(CH_FULL, xend, o);
        if (lane >= o && yp > xpos) { xpos = yp; xend = ye; }
    }
    if (lane == 31) { S.wpos[warp] = xpos; S.wend[warp] = xend; }
    __syncthreads();
    const int64_t run0 = S.excl + hrank;
    int32_t ppos = __shfl_up_sync(CH_FULL, xpos, 1);
    int64_t pend = __shfl_up_sync(CH_FULL, xend, 1);
    if (lane == 0) { ppos = -1; pend = 0; }
    for (int w = warp - 1; w >= 0 && ppos < 0; w--)
        if (S.wpos[w] >= 0) { ppos = S.wpos[w]; pend = S.wend[w]; }
    // the predecessor of the thread's first COMPUTE event: an earlier one in the tile (its gpu), else the tile
    // carry, which belongs to the tile's first gpu
    int pgpu;
    if (ppos >= 0) {
        const int pt = ppos >> 3, pk = ppos & 7;
        pgpu = gpu_of(reinterpret_cast<const uint32_t *>(&S.meta[pt * 2 + ((pk >> 2) ^ ((pt >> 2) & 1))])[pk & 3]);
    } else {
        pend = twp->pe;
        pgpu = pend == CH_NONE_TS ? -1 : gP;
    }

    // ---- phase B: per-event values (a6-a8), thread-sequential folding (a9) ----
    Acc cur, p0;
    cur.zero();
    p0.zero();
    bool has = false;
    int64_t curid = run0 - 1;
    const WinL wtP = winl_reg(twp->tw[1], S, 1, P);
    WinL wt = wtP;
    int gc = gP;
    WCur ct;
    wcur_init(ct);
    TlEnt te{};
    const int64_t t0 = P.t0, cap = P.cap;
#pragma unroll 1
    for (int k = 0; k < EV_IPT; k++) {
        if (k < nv) {
            const int64_t i = i0 + k;
            const uint32_t m = rmeta(S, tid, x32, k);
            const int g = gpu_of(m);
            if ((hmask >> k) & 1u) {
                if (!has) { p0 = cur; has = true; }
                else write_subrun(P, curid, cur, base);
                curid++;
                cur.zero();
                const uint32_t v = S.kidx[tid * EV_IPT + k];
                if (curid < cap) {
                    P.sr_key[curid] = keyl_at(g == gP ? wkP : winl_for(P, 0, g, lgP, wkP), P, (int64_t)v);
                    P.sr_first[curid] = i;
                }
            }
            const int kd = kind_of(m);
            const int64_t ks = rcol(S, 1, tid, x64, k), ke = rcol(S, 2, tid, x64, k);
            const int64_t dur = ke - ks;
            int64_t ovl = 0, prep = 0, call = 0, phi = 0, psi = 0;
            cur.nev += 1;
            if (kd == CK_COMPUTE) {
                if (pgpu == g) {
                    const int64_t tl = rcol(S, 0, tid, x64, k);
                    const int64_t t2 = tl < ks ? tl : ks;              // D6: dispatch clamped to start
                    const int64_t a = t2 - pend;
                    prep = a > 0 ? a : 0;                               // Eq. 1
                    const int64_t c1 = ks - t2, c2 = ks - pend;
                    const int64_t c = c1 < c2 ? c1 : c2;                // Eq. 2
                    call = c > 0 ? c : 0;
                }
                pgpu = g;
                pend = ke;
                if (g != gc) { wt = winl_for(P, 1, g, lgP, wtP); wcur_init(ct); gc = g; }
                if (!(ks < ct.b && ks >= ct.a) && winl_seek(wt, ct, ks)) te = tll_ent(wt, P, ct.j);
                if (ke < ct.b) {
                    ovl = te.s0 ? dur : 0;                              // |[t_ks, t_ke) ∩ U_g| (D9)
                    phi = (int64_t)te.s1 * dur;                         // MHz*ns (D10)
                    psi = (int64_t)te.s2 * dur;                         // mW*ns
                } else {
                    const unsigned long long ua = (unsigned long long)(ks - t0);
                    const unsigned long long ca = te.v0 + (te.s0 ? ua : 0ull);
                    const unsigned long long fa = te.v1 + (unsigned long long)(int64_t)te.s1 * ua;
                    const unsigned long long pa = te.v2 + (unsigned long long)(int64_t)te.s2 * ua;
                    winl_seek(wt, ct, ke);
                    te = tll_ent(wt, P, ct.j);
                    const unsigned long long ub = (unsigned long long)(ke - t0);
                    ovl = (int64_t)(te.v0 + (te.s0 ? ub : 0ull) - ca);
                    phi = (int64_t)(te.v1 + (unsigned long long)(int64_t)te.s1 * ub - fa);
                    psi = (int64_t)(te.v2 + (unsigned long long)(int64_t)te.s2 * ub - pa);
                }
                cur.n += 1;
                cur.busy += dur;
                cur.prep += prep;
                cur.call += call;
                cur.ovl += ovl;
                cur.phi += phi;
                cur.psi += psi;
                if (ks < cur.fks) {                  // one start-monotone stream: the first COMPUTE event wins
                    cur.fks = ks;
                    cur.foff = tid * EV_IPT + k;
                }
                if (ke > cur.lke) cur.lke = ke;
            } else {
                if (kd == CK_COPY || kd == CK_OTHER) cur.copy += dur;
                else if (kd == CK_AG) cur.ag += dur;
                else if (kd == CK_RS) cur.rs += dur;
            }
            if (OUT) {
                if (P.o_ovl && !is_comm(kd)) P.o_ovl[i] = ovl;
                if (P.o_prep) P.o_prep[i] = prep;
                if (P.o_call) P.o_call[i] = call;
                if (P.o_phi) P.o_phi[i] = phi;
                if (P.o_psi) P.o_psi[i] = psi;
            }
        }
    }
    tile_finish(S, P, has, cur, p0, run0, base);
}
}  // namespace

chopper_status ch_overlap_prep(chopper_ctx *ctx) {
    const int n_lg = ctx->n_lg, NG = ctx->NG;
    const int64_t N = ctx->N;
    CH_ALLOC_BEGIN;
    ctx->d_U_beg = CH_ALLOC(ctx, int64_t, n_lg + 1);
    ctx->d_U_cnt = CH_ALLOC(ctx, int64_t, n_lg + 1);
    ctx->d_V_beg = CH_ALLOC(ctx, int64_t, n_lg + 1);
    ctx->d_V_cnt = CH_ALLOC(ctx, int64_t, n_lg + 1);
    // comm union U_g over the communication bucket of each gpu (all comm streams, D9): at most one merged
    // interval per communication event, stored compactly (gpu after gpu)
    std::vector<int64_t> lo(n_lg + 1), hi(n_lg + 1), ob(n_lg + 1, 0);
    for (int l = 0; l < n_lg; l++) {
        lo[l] = ctx->bucket_beg[l * NG];
        hi[l] = ctx->bucket_beg[l * NG + 1];
        ob[l + 1] = ob[l] + (hi[l] - lo[l]);
    }
    const int64_t n_comm = ob[n_lg];
    ctx->U_s = CH_ALLOC(ctx, int64_t, n_comm);
    ctx->U_e = CH_ALLOC(ctx, int64_t, n_comm);
    ctx->U_P = CH_ALLOC(ctx, int64_t, n_comm);
    ctx->d_smp_lo = CH_ALLOC(ctx, int64_t, n_lg + 1);
    ctx->d_smp_hi = CH_ALLOC(ctx, int64_t, n_lg + 1);
    int64_t *seg_lo = CH_ALLOC(ctx, int64_t, n_lg + 1);
    int64_t *seg_hi = CH_ALLOC(ctx, int64_t, n_lg + 1);
    int64_t *seg_ob = CH_ALLOC(ctx, int64_t, n_lg + 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemcpyAsync(seg_lo, lo.data(), 8 * n_lg, cudaMemcpyHostToDevice, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(seg_hi, hi.data(), 8 * n_lg, cudaMemcpyHostToDevice, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(seg_ob, ob.data(), 8 * n_lg, cudaMemcpyHostToDevice, ctx->st));
    if (n_lg > 0) {
        k_union_block<<<n_lg, UN_NT, 0, ctx->st>>>(ctx->d_perm, seg_lo, seg_hi, ctx->ev.start_ns, ctx->ev.end_ns, ctx->U_s,
                                                  ctx->U_e, ctx->U_P, ctx->d_U_beg, ctx->d_U_cnt, seg_ob);
        CH_LAUNCHED(ctx);
    }
    // compute union V_g: explicit only with several compute streams or same-stream overlaps
    ctx->v_general = (ctx->multi_stream || ctx->h_rep.val_count[CV_STREAM_OVERLAP] > 0) ? 1 : 0;
    if (ctx->v_general && n_lg > 0) {
        ctx->V_s = CH_ALLOC(ctx, int64_t, N);
        ctx->V_e = CH_ALLOC(ctx, int64_t, N);
        ctx->V_P = CH_ALLOC(ctx, int64_t, N);
        ctx->d_vperm = CH_ALLOC(ctx, uint32_t, N);
        int64_t *vlo = CH_ALLOC(ctx, int64_t, n_lg + 1), *vhi = CH_ALLOC(ctx, int64_t, n_lg + 1);
        CH_ALLOC_END(ctx);
        size_t mark = ctx->used;
        unsigned long long *k1 = CH_ALLOC(ctx, unsigned long long, N), *k2 = CH_ALLOC(ctx, unsigned long long, N);
        uint32_t *v2 = CH_ALLOC(ctx, uint32_t, N);
        CH_ALLOC_END(ctx);
        int tsbits = bits_for((uint64_t)(ctx->t_max - ctx->t0));
        int lgbits = bits_for((uint64_t)n_lg);
        if (tsbits + lgbits > 64) return ch_fail(ctx, CHOPPER_E_RANGE, "compute-union key exceeds 64 bits");
        k_vkeys<<<(unsigned)ceil_div(N, NT), NT, 0, ctx->st>>>(ctx->ev.meta, ctx->ev.start_ns, N, ctx->d_gpu_lg, ctx->t0,
                                                               tsbits, lgbits, k1, ctx->d_vperm);
        CH_LAUNCHED(ctx);
        bool alt;
        CH_TRY(ch_radix_sort(ctx, k1, ctx->d_vperm, k2, v2, N, 0, tsbits + lgbits, &alt));
        if (alt) CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_vperm, v2, 4 * N, cudaMemcpyDeviceToDevice, ctx->st));
        if (!ctx->hold_scratch) ctx->used = mark;
        // compute events of lg are contiguous in vperm: counts per gpu from the buckets
        std::vector<int64_t> a(n_lg), b(n_lg);
        int64_t off = 0;
        for (int l = 0; l < n_lg; l++) {
            int64_t c = ctx->bucket_beg[l * NG + NG - 1] - ctx->bucket_beg[l * NG + 1];
            a[l] = off; b[l] = off + c; off += c;
        }
        CH_CUDA(ctx, cudaMemcpyAsync(vlo, a.data(), 8 * n_lg, cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(vhi, b.data(), 8 * n_lg, cudaMemcpyHostToDevice, ctx->st));
        k_union_block<<<n_lg, UN_NT, 0, ctx->st>>>(ctx->d_vperm, vlo, vhi, ctx->ev.start_ns, ctx->ev.end_ns, ctx->V_s,
                                                  ctx->V_e, ctx->V_P, ctx->d_V_beg, ctx->d_V_cnt, nullptr);
        CH_LAUNCHED(ctx);
    }
    // sample prefix integrals (D10)
    ctx->smp_lo.assign(n_lg, 0);
    ctx->smp_hi.assign(n_lg, 0);
    for (int l = 0; l < n_lg; l++) {
        int g = ctx->lg_gpu[l];
        if (ctx->has_smp && ctx->h_rep.send[g] > 0 && ctx->h_rep.sbeg[g] != ~0ull) {
            ctx->smp_lo[l] = (int64_t)ctx->h_rep.sbeg[g];
            ctx->smp_hi[l] = (int64_t)ctx->h_rep.send[g];
        }
    }
    CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_smp_lo, ctx->smp_lo.data(), 8 * n_lg, cudaMemcpyHostToDevice, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_smp_hi, ctx->smp_hi.data(), 8 * n_lg, cudaMemcpyHostToDevice, ctx->st));
    if (ctx->has_smp && ctx->M > 0) {
        const int64_t M = ctx->M;
        ctx->d_smp_phi = CH_ALLOC(ctx, int64_t, M);
        ctx->d_smp_psi = CH_ALLOC(ctx, int64_t, M);
        CH_ALLOC_END(ctx);
        size_t mark = ctx->used;
        int64_t *tf = CH_ALLOC(ctx, int64_t, M), *tp = CH_ALLOC(ctx, int64_t, M);
        uint8_t *hd = CH_ALLOC(ctx, uint8_t, M);
        CH_ALLOC_END(ctx);
        k_smp_terms<<<(unsigned)ceil_div(M, NT), NT, 0, ctx->st>>>(ctx->smp.gpu, ctx->smp.ts_ns, ctx->smp.freq_mhz,
                                                                   ctx->smp.power_mw, M, tf, tp, hd);
        CH_LAUNCHED(ctx);
        CH_TRY(ch_seg_scan_i64(ctx, tf, hd, ctx->d_smp_phi, M, 0));
        CH_TRY(ch_seg_scan_i64(ctx, tp, hd, ctx->d_smp_psi, M, 0));
        if (!ctx->hold_scratch) ctx->used = mark;
    }
    // timeline for the window-staged event passes (built before the span lists' laminarity is known when this
    // runs beside chopper_attribute; unused for a non-laminar trace)
    if (n_lg > 0) {
        std::vector<int64_t> tb(n_lg + 1), nc(n_lg);
        int64_t off = 0;
        for (int l = 0; l < n_lg; l++) {
            nc[l] = ctx->bucket_beg[l * NG + 1] - ctx->bucket_beg[l * NG];
            tb[l] = off;
            off += 1 + 2 * nc[l] + (ctx->smp_hi[l] - ctx->smp_lo[l]);
        }
        tb[n_lg] = off;
        // column stride a multiple of 4 entries: every column starts 16 B-aligned (bulk window copies); + 8
        // entries of padding so an aligned copy may read past a gpu's last entry
        const int64_t cap = (off + 3) & ~(int64_t)3;
        ctx->tl_cap = cap;
        ctx->TL_t = CH_ALLOC(ctx, int64_t, cap + 8);
        ctx->TL_v = CH_ALLOC(ctx, int64_t, 3 * cap + 8);
        ctx->TL_s = CH_ALLOC(ctx, int32_t, 3 * cap + 8);
        ctx->d_tl_beg = CH_ALLOC(ctx, int64_t, n_lg + 1);
        ctx->d_tl_len = CH_ALLOC(ctx, int64_t, n_lg + 1);
        int64_t *dnc = CH_ALLOC(ctx, int64_t, n_lg + 1);
        CH_ALLOC_END(ctx);
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_tl_beg, tb.data(), 8 * (n_lg + 1), cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(dnc, nc.data(), 8 * n_lg, cudaMemcpyHostToDevice, ctx->st));
        k_timeline<<<(unsigned)ceil_div(off, NT), NT, 0, ctx->st>>>(
            ctx->d_tl_beg, dnc, n_lg, off, ctx->U_s, ctx->U_e, ctx->U_P, ctx->d_U_beg, ctx->d_U_cnt, ctx->smp.ts_ns,
            ctx->d_smp_phi, ctx->d_smp_psi, ctx->smp.freq_mhz, ctx->smp.power_mw, ctx->d_smp_lo, ctx->d_smp_hi, ctx->t0,
            cap, ctx->TL_t, ctx->TL_v, ctx->TL_s, ctx->d_tl_len);
        CH_LAUNCHED(ctx);
    }
    // lg -> has samples (breakdown flag)
    ctx->d_has_smp = CH_ALLOC(ctx, int32_t, n_lg + 1);
    CH_ALLOC_END(ctx);
    {
        std::vector<int32_t> hs(n_lg + 1, 0);
        for (int l = 0; l < n_lg; l++) hs[l] = ctx->smp_hi[l] > ctx->smp_lo[l] ? 1 : 0;
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_has_smp, hs.data(), 4 * (n_lg + 1), cudaMemcpyHostToDevice, ctx->st));
    }
    return CHOPPER_OK;
}

// 2-D tensor map of an event column as [N / 8 rows][8 elements] (one row per thread of the lean pass), box of
// 256 rows, with the 64 B (int64) / 32 B (uint32) swizzle that matches ev_col / ev_meta
typedef CUresult (*encode_tiled_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static encode_tiled_fn tensor_map_encoder() {
    static encode_tiled_fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (encode_tiled_fn)p;
    }
    return fn;
}
static bool column_map(CUtensorMap *m, const void *col, int64_t n, int elem) {
    encode_tiled_fn enc = tensor_map_encoder();
    if (!enc || ((uintptr_t)col & 15u) || n < 8) return false;
    const cuuint64_t dims[2] = {8, (cuuint64_t)(n / 8)};
    const cuuint64_t strides[1] = {(cuuint64_t)8 * elem};
    const cuuint32_t box[2] = {8, W_NT};
    const cuuint32_t es[2] = {1, 1};
    return enc(m, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(col),
               dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               elem == 8 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

chopper_status ch_event_pass(chopper_ctx *ctx, int64_t *ovl, int64_t *prep, int64_t *call, int64_t *phi, int64_t *psi) {
    const int64_t N = ctx->N;
    ctx->R = 0;
    if (N == 0) return CHOPPER_OK;
    int64_t ntile = ceil_div(N, EV_TILE);
    CH_ALLOC_BEGIN;
    // sub-run capacity: inside one gpu the events are dispatch-ordered and an event's instance key is a step
    // function of its dispatch time with steps only at the gpu's span endpoints, so the key changes at most
    // 2 * (spans of the gpu) times; runs also break at tile and gpu boundaries
    const int64_t cap = std::min<int64_t>(N, 2 * ctx->S_loc + ceil_div(N, std::min(EV_TILE, W_TILE)) + ctx->n_lg + 1);
    ctx->sub.cap = cap;
    ctx->sub.key = CH_ALLOC(ctx, unsigned long long, cap + 1);
    ctx->sub.first_event = CH_ALLOC(ctx, int64_t, cap + 1);
    ctx->sub.f = CH_ALLOC(ctx, int64_t, (int64_t)SR_W * cap);
    ctx->d_tile_sub = CH_ALLOC(ctx, int64_t, ceil_div(N, W_TILE) + 1);      // kept: the counter pass's run ids
    // per-thread run ids and head masks (2048-event tiles of 256 threads) for the counter pass (counters only)
    const int64_t nthr = ceil_div(N, W_TILE) * W_NT;
    ctx->d_t_run = ctx->C > 0 ? CH_ALLOC(ctx, int32_t, nthr) : nullptr;
    ctx->d_t_hm = ctx->C > 0 ? CH_ALLOC(ctx, uint8_t, nthr) : nullptr;
    // the counter pass's sums ([cap][C]) and non-finite flags: it can start once the head pre-count is scanned
    double *sub_cnt = ctx->C > 0 ? CH_ALLOC(ctx, double, (int64_t)ctx->C * cap) : nullptr;
    unsigned int *colbad = ctx->C > 0 ? CH_ALLOC(ctx, unsigned int, (int64_t)ctx->n_lg * ctx->C) : nullptr;
    ctx->counters_early = false;
    ctx->t_run_rank = false;
    ctx->d_tile_state = CH_ALLOC(ctx, unsigned long long, ceil_div(N, W_TILE));   // >= tiles of either pass
    ctx->d_tile_ticket = CH_ALLOC(ctx, unsigned int, 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemsetAsync(ctx->d_tile_state, 0, 8 * ntile, ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(ctx->d_tile_ticket, 0, 4, ctx->st));
    EvParams P;
    P.tl = ctx->ev.dispatch_ns;
    P.ks = ctx->ev.start_ns;
    P.ke = ctx->ev.end_ns;
    P.meta = ctx->ev.meta;
    P.N = N;
    P.gpu_lg = ctx->d_gpu_lg;
    P.sv = ch_span_view(ctx);
    P.sh_op = 0;
    P.sh_ly = ctx->kb[3];
    P.sh_ph = P.sh_ly + ctx->kb[2];
    P.sh_it = P.sh_ph + ctx->kb[1];
    P.sh_lg = P.sh_it + ctx->kb[0];
    P.pred_end = ctx->d_pred_end;
    P.Us = ctx->U_s; P.Ue = ctx->U_e; P.UP = ctx->U_P; P.Ubeg = ctx->d_U_beg; P.Ucnt = ctx->d_U_cnt;
    P.v_general = ctx->v_general;
    P.Vs = ctx->V_s; P.Ve = ctx->V_e; P.VP = ctx->V_P; P.Vbeg = ctx->d_V_beg; P.Vcnt = ctx->d_V_cnt;
    P.perm = ctx->d_perm;
    P.bucket_beg = ctx->d_bucket_beg;
    P.NG = ctx->NG;
    P.smp_ts = ctx->smp.ts_ns; P.smp_f = ctx->smp.freq_mhz; P.smp_p = ctx->smp.power_mw;
    P.phi_pre = ctx->d_smp_phi; P.psi_pre = ctx->d_smp_psi; P.smp_lo = ctx->d_smp_lo; P.smp_hi = ctx->d_smp_hi;
    P.o_ovl = ovl; P.o_prep = prep; P.o_call = call; P.o_phi = phi; P.o_psi = psi;
    P.o_run = nullptr;
    P.t_run = ctx->d_t_run;
    P.t_hm = ctx->d_t_hm;
    P.kidx = nullptr;
    P.h_run = nullptr;
    P.h_hm = nullptr;
    P.sr_key = ctx->sub.key; P.sr_first = ctx->sub.first_event; P.sr_f = ctx->sub.f; P.cap = cap;
    P.tile_state = ctx->d_tile_state; P.ticket = ctx->d_tile_ticket;
    P.KTt = ctx->KT_t; P.KTk = ctx->KT_k; P.kt_beg = ctx->d_kt_beg;
    P.TLt = ctx->TL_t; P.TLv = ctx->TL_v; P.TLs = ctx->TL_s; P.tl_beg = ctx->d_tl_beg; P.tl_len = ctx->d_tl_len;
    P.tl_cap = ctx->tl_cap; P.t0 = ctx->t0; P.ntile = ntile;
    // 16 B cp.async staging needs 16 B aligned event columns (tile bases are multiples of 2048 events)
    auto al16 = [](const void *p) { return ((uintptr_t)p & 15u) == 0; };
    int vec_ok = al16(P.tl) && al16(P.ks) && al16(P.ke) && al16(P.pred_end) && al16(P.meta);
    CUtensorMap tm[4];
    // CHOPPER_EVENT_PASS=general forces the window-staged general pass (k_events_w) on lean traces (A/B runs)
    static const bool force_general = getenv("CHOPPER_EVENT_PASS") && !strcmp(getenv("CHOPPER_EVENT_PASS"), "general");
    const bool lean_pass = ctx->et_ok && ctx->lean && !force_general &&
                           column_map(&tm[0], P.tl, N, 8) && column_map(&tm[1], P.ks, N, 8) &&
                           column_map(&tm[2], P.ke, N, 8) && column_map(&tm[3], P.meta, N, 4);
    if (!lean_pass && !ctx->d_pred_end) {
        // a lean-loaded trace on a general event pass: materialize the chain predecessor column it reads
        CH_ALLOC_BEGIN;
        ctx->d_pred_end = CH_ALLOC(ctx, int64_t, N);
        CH_ALLOC_END(ctx);
        k_pred_lean<<<(unsigned)ceil_div(N, NT), NT, 0, ctx->st>>>(PredView{nullptr, ctx->ev.meta, ctx->ev.end_ns}, N,
                                                                  ctx->d_pred_end);
        CH_LAUNCHED(ctx);
        P.pred_end = ctx->d_pred_end;
    }
    if (lean_pass) {
        // the lean pass: TMA staging, launch chain from the tile (no predecessor column)
        ntile = ceil_div(N, W_TILE);
        P.ntile = ntile;
        size_t mark = ctx->used;
        int32_t *seeds = CH_ALLOC(ctx, int32_t, ntile * SEED_W);
        int64_t *tpe = CH_ALLOC(ctx, int64_t, ntile + 1);
        int64_t *tcnt = CH_ALLOC(ctx, int64_t, ntile + 1), *tbase = ctx->d_tile_sub;
        TileWin *twin = CH_ALLOC(ctx, TileWin, ntile);
        TileWinL *twinl = CH_ALLOC(ctx, TileWinL, ntile);
        // the head pre-count's per-event key indices and per-thread head masks / ranks, read by the event pass
        P.kidx = CH_ALLOC(ctx, uint32_t, ntile * W_TILE);
        if (!P.t_run) {                       // (without counters the counter pass's copies do not exist)
            P.t_run = CH_ALLOC(ctx, int32_t, ntile * W_NT);
            P.t_hm = CH_ALLOC(ctx, uint8_t, ntile * W_NT);
        }
        CH_ALLOC_END(ctx);
        P.h_run = P.t_run;
        P.h_hm = P.t_hm;
        P.seeds = seeds;
        const size_t dsm = sizeof(EvSmemL);
        static bool attr_l = false;
        if (!attr_l) {
            CH_CUDA(ctx, cudaFuncSetAttribute(k_events_l<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
            CH_CUDA(ctx, cudaFuncSetAttribute(k_events_l<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
            attr_l = true;
        }
        g_marks.mark(ctx->st, "ev_prologue");
        ch_tick(ctx, 4, 0);
        k_tile_seeds_l<<<(unsigned)ceil_div(ntile * 32, NT), NT, 0, ctx->st>>>(P, seeds, tpe);
        CH_LAUNCHED(ctx);
        k_tile_windows<<<(unsigned)ceil_div(ntile, NT), NT, 0, ctx->st>>>(P, twin);
        CH_LAUNCHED(ctx);
        k_tile_windows_l<<<(unsigned)ceil_div(ntile, NT), NT, 0, ctx->st>>>(P, tpe, twinl);
        CH_LAUNCHED(ctx);
        P.twin = twin;
        P.twinl = twinl;
        g_marks.mark(ctx->st, "seeds_windows");
        k_tile_heads<<<(unsigned)ntile, W_NT, 0, ctx->st>>>(P, tcnt);      // (+ head masks / ranks for counters)
        CH_LAUNCHED(ctx);
        g_marks.mark(ctx->st, "heads");
        CH_TRY(ch_scan_excl_i64(ctx, tcnt, tbase, ntile, tbase + ntile));
        P.tile_base = tbase;
        if (sub_cnt) {                        // the counter pass beside the event pass (side[0])
            ctx->sub.cnt = sub_cnt;
            CH_TRY(ch_counters_launch(ctx, sub_cnt, colbad, 1));
            ctx->counters_early = true;
        }
        P.t_run = nullptr;                    // (already written by the pre-count)
        P.t_hm = nullptr;
        ctx->t_run_rank = true;
        const bool out = ovl || prep || call || phi || psi;
        ch_tick(ctx, 8, 0);
        g_marks.mark(ctx->st, "scan_counters_fork");
        if (out) k_events_l<true><<<(unsigned)ntile, W_NT, dsm, ctx->st>>>(P, tm[0], tm[1], tm[2], tm[3]);
        else k_events_l<false><<<(unsigned)ntile, W_NT, dsm, ctx->st>>>(P, tm[0], tm[1], tm[2], tm[3]);
        CH_LAUNCHED(ctx);
        g_marks.mark(ctx->st, "events_l");
        ch_tick(ctx, 8, 1);
        ch_tick(ctx, 4, 1);
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_tile_state + ntile - 1, tbase + ntile, 8, cudaMemcpyDeviceToDevice, ctx->st));
        ctx->used = mark;
    } else if (ctx->et_ok) {
        // every span list laminar: Euler boundary tables, window-staged lookups
        ntile = ceil_div(N, W_TILE);
        P.ntile = ntile;
        size_t mark = ctx->used;
        int32_t *seeds = CH_ALLOC(ctx, int32_t, ntile * SEED_W);
        int64_t *tcnt = CH_ALLOC(ctx, int64_t, ntile + 1), *tbase = ctx->d_tile_sub;
        TileWin *twin = CH_ALLOC(ctx, TileWin, ntile);
        CH_ALLOC_END(ctx);
        P.seeds = seeds;
        size_t dsm = sizeof(EvSmemW);
        static bool attr_w = false;
        if (!attr_w) {
            CH_CUDA(ctx, cudaFuncSetAttribute(k_events_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
            attr_w = true;
        }
        ch_tick(ctx, 4, 0);
        k_tile_seeds<<<(unsigned)ceil_div(ntile * 32, NT), NT, 0, ctx->st>>>(P, seeds);
        CH_LAUNCHED(ctx);
        k_tile_windows<<<(unsigned)ceil_div(ntile, NT), NT, 0, ctx->st>>>(P, twin);
        CH_LAUNCHED(ctx);
        P.twin = twin;
        k_tile_heads<<<(unsigned)ntile, W_NT, 0, ctx->st>>>(P, tcnt);
        CH_LAUNCHED(ctx);
        CH_TRY(ch_scan_excl_i64(ctx, tcnt, tbase, ntile, tbase + ntile));
        P.tile_base = tbase;
        if (sub_cnt) {
            ctx->sub.cnt = sub_cnt;
            CH_TRY(ch_counters_launch(ctx, sub_cnt, colbad, 1));
            ctx->counters_early = true;
        }
        P.t_run = nullptr;
        P.t_hm = nullptr;
        ctx->t_run_rank = true;
        ch_tick(ctx, 8, 0);
        k_events_w<<<(unsigned)ntile, W_NT, dsm, ctx->st>>>(P, vec_ok);
        CH_LAUNCHED(ctx);
        ch_tick(ctx, 8, 1);
        ch_tick(ctx, 4, 1);
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_tile_state + ntile - 1, tbase + ntile, 8, cudaMemcpyDeviceToDevice, ctx->st));
        ctx->used = mark;
    } else {
        P.seeds = nullptr;
        size_t dsm = sizeof(EvSmem);
        static bool attr_set = false;
        if (!attr_set) {
            CH_CUDA(ctx, cudaFuncSetAttribute(k_events, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
            attr_set = true;
        }
        ch_tick(ctx, 4, 0);
        ch_tick(ctx, 8, 0);
        k_events<<<(unsigned)ntile, EV_NT, dsm, ctx->st>>>(P, vec_ok);
        CH_LAUNCHED(ctx);
        ch_tick(ctx, 8, 1);
        ch_tick(ctx, 4, 1);
        k_tile_sub_state<<<(unsigned)ceil_div(ntile + 1, NT), NT, 0, ctx->st>>>(ctx->d_tile_state, ntile, ctx->d_tile_sub);
        CH_LAUNCHED(ctx);
    }
    if (ovl && ctx->n_lg > 0) {
        k_covl<<<dim3(64, ctx->n_lg), 128, 0, ctx->st>>>(P, ctx->n_lg);
        CH_LAUNCHED(ctx);
    }
    unsigned long long last = 0;
    CH_CUDA(ctx, ch_d2h(ctx, &last, ctx->d_tile_state + ntile - 1, 8));
    CH_CUDA(ctx, ch_sync(ctx));
    ctx->R = (int64_t)(last & VAL_MASK);
    if (ctx->R > cap) return ch_fail(ctx, CHOPPER_E_RANGE, "sub-runs exceed their structural bound");
    // sentinel: sub-run R begins at N
    int64_t nv = N;
    CH_CUDA(ctx, cudaMemcpyAsync(ctx->sub.first_event + ctx->R, &nv, 8, cudaMemcpyHostToDevice, ctx->st));
    return CHOPPER_OK;
}

// event-pass launch geometry (for the bench's algorithmic-bytes accounting)
int64_t ch_event_tile() { return EV_TILE; }
