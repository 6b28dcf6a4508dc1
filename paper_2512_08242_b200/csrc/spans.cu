// spans.cu -- a5 interval-containment attribution structures (chopper_attribute).
//
// PAPER.md:100-102, 211-214; readings D3 (half-open spans,
// containment on dispatch time t_l) and D4 (innermost wins; ambiguity only
// where crossing spans both contain a dispatch).
//
// Spans of each (gpu, level) list are radix-sorted into "push order"
// (start asc, end desc, index desc): the innermost span containing t is then
// the last span with start <= t, walked up its parent chain while end <= t.
// parent(q) = nearest earlier span of the list with end >= end(q) (previous
// greater-or-equal element), computed per 256-span chunk with a stack and
// resolved across chunks with a sparse table of chunk maxima.  A list is
// laminar iff no span between parent(q) and q ends after start(q); lists
// that are not laminar use an exact sequential sweep on the device
// (k_attr_sweep) instead of the parent walk.
#include "common.cuh"

namespace {
constexpr int NT = 256;
constexpr int CHUNK = 64;
constexpr int UNRES = -3;
constexpr int SWEEP_MAX_ACTIVE = 64;

__device__ __forceinline__ bool span_valid(uint32_t gl, int64_t s, int64_t e, const int32_t *gpu_lg) {
    int g = (int)(gl >> 8), lv = (int)(gl & 0xFFu);
    return lv <= 3 && g < CH_MAX_GPUS && gpu_lg[g] >= 0 && e > s;
}

// sort 1: end descending, ties index descending (initial order = reversed index)
__global__ void k_span_key1(const uint32_t *__restrict__ gl, const int64_t *__restrict__ s,
                            const int64_t *__restrict__ e, int64_t S, int64_t emax,
                            unsigned long long *__restrict__ key, uint32_t *__restrict__ val) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= S) return;
    int64_t j = S - 1 - q;
    int64_t ee = e[j];
    key[q] = (ee <= emax) ? (unsigned long long)(emax - ee) : 0ull;
    val[q] = (uint32_t)j;
}

// sort 2: (list, start) with list = lg*4 + level, excluded spans -> list n_lg*4
__global__ void k_span_key2(const uint32_t *__restrict__ gl, const int64_t *__restrict__ s,
                            const int64_t *__restrict__ e, const uint32_t *__restrict__ val, int64_t S,
                            const int32_t *__restrict__ gpu_lg, int n_lg, int64_t smin, int sbits,
                            unsigned long long *__restrict__ key) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= S) return;
    uint32_t j = val[q];
    uint32_t x = gl[j];
    int64_t a = s[j], b = e[j];
    unsigned long long list;
    unsigned long long off = 0;
    if (span_valid(x, a, b, gpu_lg)) {
        list = (unsigned long long)(gpu_lg[x >> 8] * 4 + (int)(x & 0xFFu));
        off = (unsigned long long)(a - smin);
    } else {
        list = (unsigned long long)(n_lg * 4);
    }
    key[q] = (list << sbits) | off;
}

// (list, start) keys straight from the caller's arrays, identity values
__global__ void k_span_key_fast(const uint32_t *__restrict__ gl, const int64_t *__restrict__ s,
                                const int64_t *__restrict__ e, int64_t S, const int32_t *__restrict__ gpu_lg, int n_lg,
                                int64_t smin, int sbits, unsigned long long *__restrict__ key,
                                uint32_t *__restrict__ val) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= S) return;
    uint32_t x = gl[q];
    int64_t a = s[q], b = e[q];
    unsigned long long list, off = 0;
    if (span_valid(x, a, b, gpu_lg)) {
        list = (unsigned long long)(gpu_lg[x >> 8] * 4 + (int)(x & 0xFFu));
        off = (unsigned long long)(a - smin);
    } else {
        list = (unsigned long long)(n_lg * 4);
    }
    key[q] = (list << sbits) | off;
    val[q] = (uint32_t)q;
}

// runs of equal (list, start) are in index-ascending order after the stable sort: reorder each run by
// (end desc, index desc) with an insertion sort; runs longer than 256 set *big (two-sort fallback)
__global__ void k_fix_ties(const unsigned long long *__restrict__ key, uint32_t *__restrict__ order,
                           const int64_t *__restrict__ e, int64_t S, unsigned long long excl_key, unsigned int *big) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= S - 1) return;
    unsigned long long k = key[q];
    if (k >= excl_key) return;                       // excluded spans: order irrelevant
    if (key[q + 1] != k || (q > 0 && key[q - 1] == k)) return;
    int64_t hi = q + 1;
    while (hi < S && key[hi] == k && hi - q <= 256) hi++;
    if (hi - q > 256) { atomicOr(big, 1u); return; }
    for (int64_t a = q + 1; a < hi; a++) {
        uint32_t v = order[a];
        int64_t ev = e[v];
        int64_t b = a - 1;
        // element v goes before order[b] if (end desc, index desc) ranks it first
        while (b >= q) {
            uint32_t w = order[b];
            int64_t ew = e[w];
            if (ew > ev || (ew == ev && w > v)) break;
            order[b + 1] = w;
            b--;
        }
        order[b + 1] = v;
    }
}

__global__ void k_span_gather(const uint32_t *__restrict__ order, const uint32_t *__restrict__ gl,
                              const int64_t *__restrict__ s, const int64_t *__restrict__ e,
                              const int32_t *__restrict__ lab, int64_t S, const int32_t *__restrict__ gpu_lg, int n_lg,
                              int64_t *__restrict__ Ps, int64_t *__restrict__ Pe, int32_t *__restrict__ Po,
                              int32_t *__restrict__ Pl, int32_t *__restrict__ Plist,
                              unsigned long long *__restrict__ lbeg) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= S) return;
    uint32_t j = order[q];
    uint32_t x = gl[j];
    int64_t a = s[j], b = e[j];
    int list = span_valid(x, a, b, gpu_lg) ? gpu_lg[x >> 8] * 4 + (int)(x & 0xFFu) : n_lg * 4;
    Ps[q] = a;
    Pe[q] = b;
    Po[q] = (int32_t)j;
    Pl[q] = lab[j];
    Plist[q] = list;
    int prev = -1;
    if (q > 0) {
        uint32_t jp = order[q - 1];
        uint32_t xp = gl[jp];
        prev = span_valid(xp, s[jp], e[jp], gpu_lg) ? gpu_lg[xp >> 8] * 4 + (int)(xp & 0xFFu) : n_lg * 4;
    }
    if (list != prev) lbeg[list] = (unsigned long long)q;   // sorted: first q of each list is unique
}

// per-chunk sequential stack: previous greater-or-equal end inside the chunk
// 64 chunks per block: the block's 64 x CHUNK span ends are staged by coalesced loads (chunk-major, pitch
// CHUNK + 1: conflict-free when 64 threads walk their chunks in step); list changes come from list_beg
// (one read of the chunk's first list), not from a per-span list column
constexpr int CS_NT = 64, CS_PITCH = CHUNK + 1;
__global__ void __launch_bounds__(CS_NT) k_chunk_stack(const int64_t *__restrict__ Pe, const int32_t *__restrict__ Plist,
                                                       int64_t S, int32_t *__restrict__ parent,
                                                       int32_t *__restrict__ cstack, int32_t *__restrict__ csp,
                                                       int64_t *__restrict__ cmax, const int64_t *__restrict__ list_beg) {
    __shared__ int64_t s_e[CS_NT * CS_PITCH];
    const int tid = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * CS_NT * CHUNK;
    const int nb = (int)min((int64_t)CS_NT * CHUNK, S - base);
    for (int i = tid; i < nb; i += CS_NT) s_e[(i / CHUNK) * CS_PITCH + (i % CHUNK)] = Pe[base + i];
    __syncthreads();
    const int64_t c = (int64_t)blockIdx.x * CS_NT + tid;
    const int64_t lo = c * CHUNK;
    if (lo >= S) return;
    const int64_t hi = lo + CHUNK < S ? lo + CHUNK : S;
    const int64_t *e_s = s_e + tid * CS_PITCH;
    int32_t si[CHUNK];                 // the stack (indices and ends) stays thread-local
    int64_t se[CHUNK];
    int sp = 0;
    int list = Plist[lo];
    int64_t lbeg = list_beg[list], lnext = list_beg[list + 1];
    for (int64_t q = lo; q < hi; q++) {
        while (q >= lnext) { list++; lbeg = lnext; lnext = list_beg[list + 1]; sp = 0; }
        const int64_t e = e_s[q - lo];
        while (sp > 0 && se[sp - 1] < e) sp--;
        if (sp > 0) parent[q] = si[sp - 1];
        else parent[q] = (lbeg >= lo) ? -1 : UNRES;
        si[sp] = (int32_t)q;
        se[sp] = e;
        sp++;
    }
    int32_t *stk = cstack + lo;
    for (int k = 0; k < sp; k++) stk[k] = si[k];
    csp[c] = sp;
    cmax[c] = sp > 0 ? se[0] : INT64_MIN;   // bottom of the final stack = max end of the last list
}

// up to 3 sparse-table levels per launch: level k-1+g (g = 1..ng) at c is the max of level k-1 at
// c - m w, m < 2^g (w = 2^(k-1)), so one launch reads 2^ng entries of level k-1 and writes ng levels
__global__ void k_sparse_levels(const int64_t *__restrict__ prev, int64_t *__restrict__ next, int64_t nch, int64_t w,
                                int ng) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    int64_t v[8];
#pragma unroll
    for (int m = 0; m < 8; m++) v[m] = (m < (1 << ng) && c - m * w >= 0) ? prev[c - m * w] : INT64_MIN;
    int64_t mx = v[0];
#pragma unroll
    for (int g = 1; g <= 3; g++) {
        if (g > ng) break;
        for (int m = 1 << (g - 1); m < (1 << g); m++) mx = v[m] > mx ? v[m] : mx;
        next[(int64_t)(g - 1) * nch + c] = mx;
    }
}

__global__ void k_resolve(const int64_t *__restrict__ Pe, const int32_t *__restrict__ Plist, int64_t S,
                          int32_t *__restrict__ parent, const int32_t *__restrict__ cstack,
                          const int32_t *__restrict__ csp, const int64_t *__restrict__ sparse, int levels,
                          int64_t nch, const int64_t *__restrict__ list_beg) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= S || parent[q] != UNRES) return;
    int64_t x = Pe[q];
    int64_t lbc = list_beg[Plist[q]] / CHUNK;
    int64_t c = q / CHUNK - 1;
    // largest chunk index c >= lbc whose max >= x: skip blocks of chunks entirely below x
    for (int k = levels - 1; k >= 0; k--) {
        int64_t w = 1ll << k;
        if (c - w + 1 >= lbc && sparse[(int64_t)k * nch + c] < x) c -= w;
    }
    int32_t res = -1;
    if (c >= lbc && sparse[c] >= x) {
        const int32_t *stk = cstack + c * CHUNK;
        int n = csp[c];
        // topmost stack entry with end >= x (ends non-increasing bottom -> top)
        int l = 0, h = n;
        while (l < h) {
            int m = (l + h) >> 1;
            if (Pe[stk[m]] >= x) l = m + 1; else h = m;
        }
        if (l > 0) res = stk[l - 1];
    }
    parent[q] = res;
}

// laminarity: no span strictly between parent(q) and q (push order) ends after start(q)
__global__ void k_laminar(const int64_t *__restrict__ Ps, const int64_t *__restrict__ Pe,
                          const int32_t *__restrict__ Plist, const int32_t *__restrict__ parent, int64_t S,
                          const int64_t *__restrict__ list_beg, int n_lists, int32_t *__restrict__ flags) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= S) return;
    int list = Plist[q];
    if (list >= n_lists) return;
    int64_t lb = list_beg[list];
    int64_t p = parent[q] >= 0 ? parent[q] : lb - 1;
    int64_t sq = Ps[q];
    int64_t j = q - 1;
    int steps = 0;
    while (j > p) {
        if (Pe[j] > sq || ++steps > 64) { flags[list] = 1; return; }
        int32_t pj = parent[j];
        j = pj >= 0 ? pj : lb - 1;
    }
}

// exact sequential sweep for a non-laminar (gpu, level) list: active set in push order
__global__ void k_attr_sweep(const int *__restrict__ lists, int n_sweep, const int64_t *__restrict__ list_beg,
                             const int64_t *__restrict__ Ps, const int64_t *__restrict__ Pe,
                             const int64_t *__restrict__ gbeg, const int64_t *__restrict__ tl, int64_t N,
                             int32_t *__restrict__ attr_pre, DevReport *rep) {
    int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= n_sweep) return;
    int list = lists[w];
    int lg = list / 4, lv = list % 4;
    int64_t lb = list_beg[list], le = list_beg[list + 1];
    int64_t act[SWEEP_MAX_ACTIVE];
    int na = 0;
    int64_t nxt = lb;
    for (int64_t i = gbeg[lg]; i < gbeg[lg + 1]; i++) {
        int64_t t = tl[i];
        while (nxt < le && Ps[nxt] <= t) {
            if (na == SWEEP_MAX_ACTIVE) { latch(rep, CHOPPER_E_RANGE); break; }
            act[na++] = nxt++;
        }
        int k = 0;
        for (int a = 0; a < na; a++) if (Pe[act[a]] > t) act[k++] = act[a];
        na = k;
        int32_t r = -1;
        if (na > 0) {
            bool chain = true;
            for (int a = 1; a < na; a++) if (Pe[act[a]] > Pe[act[a - 1]]) chain = false;
            if (chain) r = (int32_t)act[na - 1];
            else { r = -2; latch(rep, CHOPPER_E_AMBIGUOUS_SPANS); }
        }
        attr_pre[(int64_t)lv * N + i] = r;
    }
}

// ---- Euler boundary tables (every list laminar) ----------------------------------------------------
// In a laminar list the push order is a pre-order of the nesting forest, so the time-ordered sequence of
// span endpoints is its Euler tour: before start(q) come the r starts of the earlier spans (r = rank of q in
// the list) and the ends of those of them that are not ancestors of q (r - depth(q)); end(q) follows the
// 2*size(q) - 1 endpoints of q's subtree.  Each entry records the innermost span after it: q after start(q),
// parent(q) after end(q).  Equal times keep the tour order, so "last entry with time <= t" is the innermost
// span containing t (half-open, D3; ties innermost = push-order last, D4) -- the owner the parent walk finds.
__global__ void k_euler(const int64_t *__restrict__ Ps, const int64_t *__restrict__ Pe,
                        const int32_t *__restrict__ parent, const int32_t *__restrict__ Plist, int64_t SL,
                        const int64_t *__restrict__ list_beg, int64_t *__restrict__ Et, int32_t *__restrict__ Ec) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= SL) return;
    const int list = Plist[q];
    const int64_t lb = list_beg[list], le = list_beg[list + 1];
    const int64_t r = q - lb;
    int64_t d = 0;
    for (int32_t p = parent[q]; p >= 0; p = parent[p]) d++;
    const int64_t e = Pe[q];
    // subtree = [q, first later span of the list starting at or after end(q))
    int64_t l = q + 1, h = le;
    while (l < h) {
        int64_t m = (l + h) >> 1;
        if (__ldg(Ps + m) < e) l = m + 1; else h = m;
    }
    const int64_t base = 2 * lb + list + 1;       // entry 0 of the list is the (-inf, none) sentinel
    const int64_t ps = base + 2 * r - d, pe = ps + 2 * (l - q) - 1;
    Et[ps] = Ps[q];
    Ec[ps] = (int32_t)(r + 1);
    Et[pe] = e;
    const int32_t p = parent[q];
    Ec[pe] = p >= 0 ? (int32_t)(p - lb + 1) : 0;
}
__global__ void k_euler_sentinels(const int64_t *__restrict__ list_beg, int n_lists, int64_t *__restrict__ Et,
                                  int32_t *__restrict__ Ec, int64_t *__restrict__ et_beg) {
    int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l > n_lists) return;
    const int64_t b = 2 * list_beg[l] + l;
    et_beg[l] = b;
    if (l == n_lists) return;
    Et[b] = INT64_MIN;
    Ec[b] = 0;
}
// the tour must come out time-sorted; anything else sends the event pass down the parent-walk path
__global__ void k_euler_check(const int64_t *__restrict__ Et, const int64_t *__restrict__ et_beg, int n_lists,
                              int64_t n, unsigned int *bad) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j + 1 >= n) return;
    if (Et[j + 1] < Et[j]) {
        // a list boundary is allowed to decrease (next list's sentinel is INT64_MIN)
        if (Et[j + 1] != INT64_MIN) atomicOr(bad, 1u);
    }
}

// combined key table: every non-sentinel Euler entry of (lg, level) goes to its position in the time-merge of the
// gpu's four lists (ties: lower level first, then list order) and records the instance key after it -- its own
// level's code and, for the other levels, the code of their last entry at or before its time.  The last entry
// at any time therefore carries the full key there; entry 0 of each gpu is (-inf, invalid).
// Done in blocks of KT_CH consecutive entries of one list: the other three lists' entries between the
// block's first and last time are staged in shared memory once per block (they are few: a block of op entries
// spans a handful of layer / phase / iteration boundaries), so each entry's three rank searches run there.
constexpr int KT_NT = 256, KT_CH = 2048, KT_WIN = 1024;
__global__ void __launch_bounds__(KT_NT) k_keytab_blk(const int64_t *__restrict__ Et, const int32_t *__restrict__ Ec,
                                                      const int64_t *__restrict__ et_beg,
                                                      const int64_t *__restrict__ list_beg,
                                                      const int64_t *__restrict__ chunk_beg, int n_lists, int sh_it,
                                                      int sh_ph, int sh_ly, int sh_lg, int64_t *__restrict__ Kt,
                                                      unsigned long long *__restrict__ Kk) {
    __shared__ int64_t s_t[3][KT_WIN];
    __shared__ int32_t s_c[3][KT_WIN];
    __shared__ int64_t s_lo[3], s_n[3];
    __shared__ int s_list;
    __shared__ int64_t s_j0, s_j1;
    const int tid = threadIdx.x;
    const int64_t cb = blockIdx.x;
    if (tid == 0) {
        int l = 0, h = n_lists;                          // list of chunk cb: last l with chunk_beg[l] <= cb
        while (h - l > 1) {
            const int m = (l + h) >> 1;
            if (chunk_beg[m] <= cb) l = m; else h = m;
        }
        s_list = l;
        const int64_t b = et_beg[l], e = et_beg[l + 1];
        s_j0 = b + (cb - chunk_beg[l]) * KT_CH;
        s_j1 = s_j0 + KT_CH < e ? s_j0 + KT_CH : e;
    }
    __syncthreads();
    const int l = s_list, lg = l >> 2, lv = l & 3;
    const int64_t j0 = s_j0, j1 = s_j1;
    if (tid < 3 * 32) {                                     // warp q: the window of the q-th other list
        const int q = tid >> 5, o = q + (q >= lv ? 1 : 0);
        const int64_t b = et_beg[lg * 4 + o], e = et_beg[lg * 4 + o + 1];
        const int64_t lo = warp_last_le(Et, b, e, Et[j0]);  // >= b (sentinel)
        const int64_t hi = warp_last_le(Et, lo, e, Et[j1 - 1]) + 1;
        if ((tid & 31) == 0) {
            s_lo[q] = lo;
            s_n[q] = hi - lo <= KT_WIN ? hi - lo : -1;      // -1: search global memory
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; q++) {
        const int64_t n = s_n[q];
        for (int i = tid; i < n; i += KT_NT) {
            s_t[q][i] = Et[s_lo[q] + i];
            s_c[q][i] = Ec[s_lo[q] + i];
        }
    }
    __syncthreads();
#pragma unroll 1
    for (int64_t j = j0 + tid; j < j1; j += KT_NT) {
    const int64_t a = j - et_beg[l];
    const int64_t kb = 2 * list_beg[lg * 4] + lg;
    if (a == 0) {
        if (lv == 0) { Kt[kb] = INT64_MIN; Kk[kb] = CH_INVALID_KEY; }
        continue;
    }
    const int64_t t = Et[j];
    int64_t pos = kb + a;
    uint32_t code[4];
    code[lv] = (uint32_t)Ec[j];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        const int o = q + (q >= lv ? 1 : 0);
        const int64_t b = et_beg[lg * 4 + o];
        int64_t le, c;
        const int64_t n = s_n[q];
        if (n > 0) {
            int lo2 = 0, hi2 = (int)n;                      // last staged entry <= t (t >= the first)
            while (lo2 < hi2) {
                const int m = (lo2 + hi2) >> 1;
                if (s_t[q][m] <= t) lo2 = m + 1; else hi2 = m;
            }
            int x = lo2 - 1;
            code[o] = (uint32_t)s_c[q][x];
            le = s_lo[q] + x;
            if (o > lv) while (x > 0 && s_t[q][x] == t) x--;
            c = s_lo[q] + x;
            if (o > lv && x == 0 && s_t[q][0] == t) {         // ties reach the window start: finish in global memory
                c = le;
                while (c > b && Et[c] == t) c--;
            }
        } else {
            const int64_t e = et_beg[lg * 4 + o + 1];
            le = last_le(Et, b, e, t);
            code[o] = (uint32_t)Ec[le];
            c = le;
            if (o > lv) while (c > b && Et[c] == t) c--;
        }
        pos += c - b;
    }
    Kt[pos] = t;
    Kk[pos] = code[0] == 0 ? CH_INVALID_KEY
                           : ((unsigned long long)lg << sh_lg) | ((unsigned long long)code[0] << sh_it) |
                                 ((unsigned long long)code[1] << sh_ph) | ((unsigned long long)code[2] << sh_ly) |
                                 (unsigned long long)code[3];
    }
}

__global__ void k_attr_out(SpanView v, const int64_t *__restrict__ tl, const uint32_t *__restrict__ meta, int64_t N,
                           const int32_t *__restrict__ gpu_lg, const int32_t *__restrict__ Po,
                           int32_t *__restrict__ out) {
    // blocked: each thread handles 8 consecutive events so the seeded search walks forward
    int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    int64_t cur[4] = {-2, -2, -2, -2};
    int lgp = -1;
    for (int k = 0; k < 8; k++) {
        int64_t i = base + k;
        if (i >= N) break;
        int lg = gpu_lg[gpu_of(meta[i])];
        if (lg != lgp) { cur[0] = cur[1] = cur[2] = cur[3] = -2; lgp = lg; }
        int64_t t = tl[i];
#pragma unroll
        for (int lv = 0; lv < 4; lv++) {
            int64_t c = span_lookup(v, lg, lv, t, i, &cur[lv]);
            out[(int64_t)lv * N + i] = c >= 0 ? Po[c] : (int32_t)c;
        }
    }
}
}  // namespace

// The push-order sort (a5, first half): one stable (list, start) radix sort with input order as tie-break, equal-
// start runs reordered by (end desc, index desc) in place, then the gather into push order with the list
// begins.  Enqueued by chopper_load_columns on side[2] once the spans are validated, so that it runs beside
// chopper_align (whose host synchronizations would otherwise leave the gpu idle); every buffer it touches is
// allocated here and kept for the step.
chopper_status ch_span_sort_launch(chopper_ctx *ctx) {
    ctx->span_pending = false;
    ctx->span_launched = true;
    const int64_t S = ctx->S;
    const int n_lg = ctx->n_lg;
    const int n_lists = n_lg * 4;
    CH_ALLOC_BEGIN;
    ctx->d_list_beg = CH_ALLOC(ctx, int64_t, n_lists + 2);
    ctx->d_list_flags = CH_ALLOC(ctx, int32_t, n_lists + 1);
    ctx->P_start = CH_ALLOC(ctx, int64_t, S);
    ctx->P_end = CH_ALLOC(ctx, int64_t, S);
    ctx->P_orig = CH_ALLOC(ctx, int32_t, S);
    ctx->P_label = CH_ALLOC(ctx, int32_t, S);
    ctx->P_parent = CH_ALLOC(ctx, int32_t, S);
    ctx->ss.Plist = CH_ALLOC(ctx, int32_t, S);
    CH_ALLOC_END(ctx);
    if (n_lg == 0 || S == 0) return CHOPPER_OK;
    int64_t smin = dec_i64(ctx->h_rep.s_min_enc), emax = dec_i64(ctx->h_rep.s_max_enc);
    if (ctx->h_rep.s_min_enc == ~0ull) { smin = 0; emax = 0; }
    const int rbits = bits_for((uint64_t)(emax - smin));
    const int lbits = bits_for((uint64_t)n_lists);
    if (rbits + lbits > 64) return ch_fail(ctx, CHOPPER_E_RANGE, "span sort key exceeds 64 bits");
    auto &q = ctx->ss;
    q.smin = smin; q.emax = emax; q.rbits = rbits; q.lbits = lbits;
    q.k1 = CH_ALLOC(ctx, unsigned long long, S); q.k2 = CH_ALLOC(ctx, unsigned long long, S);
    q.v1 = CH_ALLOC(ctx, uint32_t, S); q.v2 = CH_ALLOC(ctx, uint32_t, S);
    q.lb = CH_ALLOC(ctx, unsigned long long, n_lists + 1);
    q.lb2 = CH_ALLOC(ctx, unsigned long long, n_lists + 1);
    CH_ALLOC_END(ctx);
    q.big = reinterpret_cast<unsigned int *>(q.lb + n_lists);
    // side stream: ordered after everything chopper_load_columns enqueued
    CH_CUDA(ctx, cudaEventRecord(ctx->span_fork, ctx->st));
    CH_CUDA(ctx, cudaStreamWaitEvent(ctx->side[2], ctx->span_fork, 0));
    cudaStream_t main_st = ctx->st;
    ctx->st = ctx->side[2];
    ctx->hold_scratch = true;                   // the sort's own scratch must outlive the launches
    chopper_status st = [&]() -> chopper_status {
        CH_CUDA(ctx, cudaMemsetAsync(ctx->d_list_flags, 0, sizeof(int32_t) * (n_lists + 1), ctx->st));
        const unsigned g = (unsigned)ceil_div(S, NT);
        bool alt;
        k_span_key_fast<<<g, NT, 0, ctx->st>>>(ctx->sp.gpu_level, ctx->sp.start_ns, ctx->sp.end_ns, S, ctx->d_gpu_lg,
                                               n_lg, smin, rbits, q.k1, q.v1);
        CH_LAUNCHED(ctx);
        CH_TRY(ch_radix_sort(ctx, q.k1, q.v1, q.k2, q.v2, S, 0, rbits + lbits, &alt));
        q.order = alt ? q.v2 : q.v1;
        q.okeys = alt ? q.k2 : q.k1;
        CH_CUDA(ctx, cudaMemsetAsync(q.big, 0, 4, ctx->st));
        k_fix_ties<<<g, NT, 0, ctx->st>>>(q.okeys, q.order, ctx->sp.end_ns, S, (unsigned long long)n_lists << rbits, q.big);
        CH_LAUNCHED(ctx);
        // gather speculatively (long equal-start runs are rare); one read-back for the flag and the list begins
        CH_TRY(ch_fill_u64(ctx, q.lb2, n_lists + 1, ~0ull));
        k_span_gather<<<g, NT, 0, ctx->st>>>(q.order, ctx->sp.gpu_level, ctx->sp.start_ns, ctx->sp.end_ns,
                                             ctx->sp.label, S, ctx->d_gpu_lg, n_lg, ctx->P_start, ctx->P_end,
                                             ctx->P_orig, ctx->P_label, q.Plist, q.lb2);
        CH_LAUNCHED(ctx);
        return CHOPPER_OK;
    }();
    ctx->hold_scratch = false;
    CH_CUDA(ctx, cudaEventRecord(ctx->span_join, ctx->st));
    ctx->st = main_st;
    CH_TRY(st);
    ctx->span_pending = true;
    return CHOPPER_OK;
}

chopper_status ch_build_spans(chopper_ctx *ctx) {
    CH_ALLOC_BEGIN;
    const int64_t S = ctx->S;
    const int n_lg = ctx->n_lg;
    const int n_lists = n_lg * 4;
    if (!ctx->span_launched) CH_TRY(ch_span_sort_launch(ctx));     // (not launched by the load)
    g_marks.mark(ctx->st, "at_begin");
    if (ctx->span_pending) {
        CH_CUDA(ctx, cudaStreamWaitEvent(ctx->st, ctx->span_join, 0));
        ctx->span_pending = false;
    }
    g_marks.mark(ctx->st, "at_span_join");
    int32_t *Plist = ctx->ss.Plist;
    ctx->list_beg.assign(n_lists + 2, 0);
    ctx->S_loc = 0;
    if (n_lg == 0) {                 // a rank without events (its traced GPUs are empty): no span lists
        CH_CUDA(ctx, cudaMemsetAsync(ctx->d_list_beg, 0, sizeof(int64_t) * (n_lists + 2), ctx->st));
        CH_CUDA(ctx, cudaMemsetAsync(ctx->d_list_flags, 0, sizeof(int32_t) * (n_lists + 1), ctx->st));
        ctx->et_ok = false;
        return CHOPPER_OK;
    }
    if (S == 0) CH_CUDA(ctx, cudaMemsetAsync(ctx->d_list_flags, 0, sizeof(int32_t) * (n_lists + 1), ctx->st));
    if (S > 0) {
        auto &q = ctx->ss;
        const int64_t emax = q.emax, smin = q.smin;
        const int rbits = q.rbits, lbits = q.lbits;
        const unsigned g = (unsigned)ceil_div(S, NT);
        unsigned long long *k1 = q.k1, *k2 = q.k2, *lb2 = q.lb2;
        uint32_t *v1 = q.v1, *v2 = q.v2, *order = q.order;
        bool alt;
        auto gather = [&](const uint32_t *ord) -> chopper_status {
            CH_TRY(ch_fill_u64(ctx, lb2, n_lists + 1, ~0ull));
            k_span_gather<<<g, NT, 0, ctx->st>>>(ord, ctx->sp.gpu_level, ctx->sp.start_ns, ctx->sp.end_ns,
                                                 ctx->sp.label, S, ctx->d_gpu_lg, n_lg, ctx->P_start, ctx->P_end,
                                                 ctx->P_orig, ctx->P_label, Plist, lb2);
            CH_LAUNCHED(ctx);
            return CHOPPER_OK;
        };
        std::vector<unsigned long long> hb(n_lists + 1);
        unsigned int hbig = 0;
        CH_CUDA(ctx, ch_d2h(ctx, &hbig, q.big, 4));
        CH_CUDA(ctx, ch_d2h(ctx, hb.data(), lb2, 8 * (n_lists + 1)));
        CH_CUDA(ctx, ch_sync(ctx));
        if (hbig) {
            // very long runs of equal starts: exact two-sort path (end desc, then (list, start) stable)
            k_span_key1<<<g, NT, 0, ctx->st>>>(ctx->sp.gpu_level, ctx->sp.start_ns, ctx->sp.end_ns, S, emax, k1, v1);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, S, 0, rbits, &alt));
            uint32_t *vs = alt ? v2 : v1;
            unsigned long long *ks = alt ? k2 : k1, *ko = alt ? k1 : k2;
            uint32_t *vo = alt ? v1 : v2;
            k_span_key2<<<g, NT, 0, ctx->st>>>(ctx->sp.gpu_level, ctx->sp.start_ns, ctx->sp.end_ns, vs, S,
                                               ctx->d_gpu_lg, n_lg, smin, rbits, ks);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_radix_sort(ctx, ks, vs, ko, vo, S, 0, rbits + lbits, &alt));
            order = alt ? vo : vs;
            CH_TRY(gather(order));
            CH_CUDA(ctx, ch_d2h(ctx, hb.data(), lb2, 8 * (n_lists + 1)));
            CH_CUDA(ctx, ch_sync(ctx));
        }
        ctx->list_beg[n_lists + 1] = S;
        for (int l = n_lists; l >= 0; l--) ctx->list_beg[l] = hb[l] == ~0ull ? ctx->list_beg[l + 1] : (int64_t)hb[l];
        ctx->S_loc = ctx->list_beg[n_lists];
    }
    CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_list_beg, ctx->list_beg.data(), 8 * (n_lists + 2), cudaMemcpyHostToDevice,
                                 ctx->st));
    // key bit widths: component = rank + 1 in [0, list size]; never all-ones
    int64_t mx[4] = {0, 0, 0, 0};
    for (int l = 0; l < n_lists; l++) mx[l % 4] = std::max(mx[l % 4], ctx->list_beg[l + 1] - ctx->list_beg[l]);
    ctx->kg = bits_for((uint64_t)n_lg);
    ctx->max_it_list = mx[0];
    ctx->n_layer_spans = 0;
    for (int l = 0; l < n_lists; l++)
        if (l % 4 == 2) ctx->n_layer_spans += ctx->list_beg[l + 1] - ctx->list_beg[l];
    int tot = ctx->kg;
    for (int lv = 0; lv < 4; lv++) { ctx->kb[lv] = bits_for((uint64_t)mx[lv] + 1); tot += ctx->kb[lv]; }
    if (tot > 64) return ch_fail(ctx, CHOPPER_E_RANGE, "instance key exceeds 64 bits");

    const int64_t SL = ctx->S_loc;
    ctx->list_flags.assign(n_lists, 0);
    const int64_t net = 2 * SL + n_lists;
    ctx->ET_t = CH_ALLOC(ctx, int64_t, net);
    ctx->ET_c = CH_ALLOC(ctx, int32_t, net);
    ctx->d_et_beg = CH_ALLOC(ctx, int64_t, n_lists + 1);
    unsigned int *et_bad = CH_ALLOC(ctx, unsigned int, 1);
    CH_ALLOC_END(ctx);
    unsigned int h_et_bad = 0;
    CH_CUDA(ctx, cudaMemsetAsync(et_bad, 0, 4, ctx->st));
    k_euler_sentinels<<<(unsigned)ceil_div(n_lists + 1, NT), NT, 0, ctx->st>>>(ctx->d_list_beg, n_lists, ctx->ET_t,
                                                                              ctx->ET_c, ctx->d_et_beg);
    CH_LAUNCHED(ctx);
    if (SL > 0) {
        int64_t nch = ceil_div(SL, CHUNK);
        int levels = 1;
        while ((1ll << levels) < nch) levels++;
        size_t mark = ctx->used;
        int32_t *cstack = CH_ALLOC(ctx, int32_t, nch * CHUNK);
        int32_t *csp = CH_ALLOC(ctx, int32_t, nch);
        int64_t *sparse = CH_ALLOC(ctx, int64_t, (int64_t)levels * nch);
        CH_ALLOC_END(ctx);
        k_chunk_stack<<<(unsigned)ceil_div(nch, CS_NT), CS_NT, 0, ctx->st>>>(ctx->P_end, Plist, SL, ctx->P_parent, cstack, csp,
                                                                      sparse, ctx->d_list_beg);
        CH_LAUNCHED(ctx);
        for (int k = 1; k < levels; k += 3) {
            const int ng = std::min(3, levels - k);
            k_sparse_levels<<<(unsigned)ceil_div(nch, NT), NT, 0, ctx->st>>>(sparse + (int64_t)(k - 1) * nch,
                                                                             sparse + (int64_t)k * nch, nch,
                                                                             1ll << (k - 1), ng);
            CH_LAUNCHED(ctx);
        }
        unsigned g = (unsigned)ceil_div(SL, NT);
        k_resolve<<<g, NT, 0, ctx->st>>>(ctx->P_end, Plist, SL, ctx->P_parent, cstack, csp, sparse, levels, nch,
                                         ctx->d_list_beg);
        CH_LAUNCHED(ctx);
        k_laminar<<<g, NT, 0, ctx->st>>>(ctx->P_start, ctx->P_end, Plist, ctx->P_parent, SL, ctx->d_list_beg, n_lists,
                                         ctx->d_list_flags);
        CH_LAUNCHED(ctx);
        // Euler boundary tables, built before the laminarity is known (used only if every list is laminar; in a
        // non-laminar list the positions stay inside the list's range and are simply never read)
        k_euler<<<(unsigned)ceil_div(SL, NT), NT, 0, ctx->st>>>(ctx->P_start, ctx->P_end, ctx->P_parent, Plist, SL,
                                                               ctx->d_list_beg, ctx->ET_t, ctx->ET_c);
        CH_LAUNCHED(ctx);
        k_euler_check<<<(unsigned)ceil_div(net, NT), NT, 0, ctx->st>>>(ctx->ET_t, ctx->d_et_beg, n_lists, net, et_bad);
        CH_LAUNCHED(ctx);
        // one read-back: laminarity flags and the tour check
        CH_CUDA(ctx, ch_d2h(ctx, ctx->list_flags.data(), ctx->d_list_flags, 4 * n_lists));
        CH_CUDA(ctx, ch_d2h(ctx, &h_et_bad, et_bad, 4));
        // chopper_overlap's preparation: its host work while the gpu runs the kernels above.  Its buffers are
        // allocated above this block's transients, which therefore stay allocated for the step (the scratch plan
        // counts the chunk stacks and sparse tables per span)
        const bool prep_here = ctx->prep_deferred;
        if (prep_here) CH_TRY(ch_prep_side(ctx));
        CH_CUDA(ctx, ch_sync(ctx));
        if (!prep_here) ctx->used = mark;
    }
    // exact sweep for non-laminar lists
    std::vector<int> sweep;
    for (int l = 0; l < n_lists; l++) if (ctx->list_flags[l]) sweep.push_back(l);
    ctx->rep.non_laminar_lists = (int32_t)sweep.size();
    ctx->d_attr_pre = nullptr;
    ctx->et_ok = sweep.empty() && h_et_bad == 0;
    if (ctx->et_ok) {
        const int64_t nkt = 2 * SL + n_lg;
        ctx->KT_t = CH_ALLOC(ctx, int64_t, nkt + 8);              // + 8: 16 B-aligned bulk copies of windows
        ctx->KT_k = CH_ALLOC(ctx, unsigned long long, nkt + 8);
        ctx->d_kt_beg = CH_ALLOC(ctx, int64_t, n_lg + 1);
        CH_ALLOC_END(ctx);
        std::vector<int64_t> kb(n_lg + 1);
        for (int l = 0; l <= n_lg; l++) kb[l] = 2 * ctx->list_beg[l * 4] + l;
        CH_CUDA(ctx, cudaMemcpyAsync(ctx->d_kt_beg, kb.data(), 8 * (n_lg + 1), cudaMemcpyHostToDevice, ctx->st));
        const int sh_ly = ctx->kb[3], sh_ph = sh_ly + ctx->kb[2], sh_it = sh_ph + ctx->kb[1], sh_lg = sh_it + ctx->kb[0];
        // chunks of KT_CH entries per Euler list (host-known list sizes)
        std::vector<int64_t> cbeg(n_lists + 1);
        int64_t nch = 0;
        for (int l = 0; l < n_lists; l++) {
            cbeg[l] = nch;
            const int64_t len = 2 * (ctx->list_beg[l + 1] - ctx->list_beg[l]) + 1;
            nch += ceil_div(len, KT_CH);
        }
        cbeg[n_lists] = nch;
        size_t mk = ctx->used;
        int64_t *dcb = CH_ALLOC(ctx, int64_t, n_lists + 1);
        CH_ALLOC_END(ctx);
        CH_CUDA(ctx, cudaMemcpyAsync(dcb, cbeg.data(), 8 * (n_lists + 1), cudaMemcpyHostToDevice, ctx->st));
        k_keytab_blk<<<(unsigned)nch, KT_NT, 0, ctx->st>>>(ctx->ET_t, ctx->ET_c, ctx->d_et_beg, ctx->d_list_beg, dcb,
                                                           n_lists, sh_it, sh_ph, sh_ly, sh_lg, ctx->KT_t, ctx->KT_k);
        CH_LAUNCHED(ctx);
        ctx->used = mk;
        (void)net;
    }
    if (!sweep.empty()) {
        ctx->d_attr_pre = CH_ALLOC(ctx, int32_t, 4 * ctx->N);
        int *dl = CH_ALLOC(ctx, int, (int64_t)sweep.size());
        int64_t *dg = CH_ALLOC(ctx, int64_t, n_lg + 1);
        CH_ALLOC_END(ctx);
        CH_CUDA(ctx, cudaMemcpyAsync(dl, sweep.data(), 4 * sweep.size(), cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(dg, ctx->g_beg, 8 * (n_lg + 1), cudaMemcpyHostToDevice, ctx->st));
        k_attr_sweep<<<(unsigned)ceil_div((int64_t)sweep.size(), 32), 32, 0, ctx->st>>>(
            dl, (int)sweep.size(), ctx->d_list_beg, ctx->P_start, ctx->P_end, dg, ctx->ev.dispatch_ns, ctx->N,
            ctx->d_attr_pre, ctx->d_rep);
        CH_LAUNCHED(ctx);
    }
    return CHOPPER_OK;
}

SpanView ch_span_view(chopper_ctx *ctx) {
    SpanView v;
    v.P_start = ctx->P_start;
    v.P_end = ctx->P_end;
    v.P_parent = ctx->P_parent;
    v.list_beg = ctx->d_list_beg;
    v.list_flags = ctx->d_list_flags;
    v.attr_pre = ctx->d_attr_pre;
    v.N = ctx->N;
    return v;
}

chopper_status ch_attr_pass(chopper_ctx *ctx, int32_t *span_idx) {
    if (!span_idx || ctx->N == 0) return CHOPPER_OK;
    int64_t threads = ceil_div(ctx->N, 8);
    k_attr_out<<<(unsigned)ceil_div(threads, NT), NT, 0, ctx->st>>>(ch_span_view(ctx), ctx->ev.dispatch_ns, ctx->ev.meta,
                                                                    ctx->N, ctx->d_gpu_lg, ctx->P_orig, span_idx);
    CH_LAUNCHED(ctx);
    return CHOPPER_OK;
}
