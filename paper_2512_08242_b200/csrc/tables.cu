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
// block, 8 consecutive per thread; sub-runs never cross tiles).  A counter pass enumerates the gpu's
// non-MEMOP kernels in dispatch order (D2), so when a tile holds one gpu its counter values are one
// contiguous rank range [nlo, nhi] of each column: it is staged into shared memory with coalesced
// cp.async (no register round trip, all slots' copies in flight together) and each thread then reads
// its own events' values from SMEM.  Tiles that straddle two gpus gather from global memory instead.
// Each thread folds its 8 events sequentially (input order); runs that span threads are completed by
// a segmented scan of (has-head, tail-or-whole) over the tile (warp shuffles + warp carries).  The
// pass also checks every value it reads -- the slot's column at every non-MEMOP event of the gpu,
// i.e. the whole column -- for finiteness (R8), so a counter pass is read once.  Slot groups of CT_SG
// are processed in turn by the same block (the tile's event metadata is read once).
constexpr int CT_NT = 256, CT_IPT = 8, CT_TILE = CT_NT * CT_IPT, CT_SG = 4, CT_WARPS = CT_NT / 32, CT_CP = 128;
// staged element j (tile-relative rank) lives at j ^ ((j >> 4) & 7): the 32 lanes of a warp read
// elements 8 apart (one per thread-blocked event), which this spreads over all banks (2 wavefronts)
__device__ __forceinline__ int ct_sw(int j) { return j ^ ((j >> 4) & 7); }
struct CtSmem {
    double x[CT_SG][CT_TILE];                 // 64 KB
    double agg[CT_WARPS][CT_SG], carry[CT_WARPS][CT_SG];
    int aflag[CT_WARPS];
    int red[4][CT_WARPS];
    const double *cp[CT_CP];                  // column pointers [lg][slot], loaded beside the metadata
};
__global__ void __launch_bounds__(CT_NT, 3) k_counters_tiled(const uint32_t *__restrict__ meta,
                                                          const int32_t *__restrict__ t_run,
                                                          const uint8_t *__restrict__ t_hm,
                                                          const int32_t *__restrict__ t_nm,
                                                          const int64_t *__restrict__ nm_base,
                                                          const int64_t *__restrict__ tile_sub,
                                                          const int32_t *__restrict__ gpu_lg,
                                                          const double *const *__restrict__ col, int C,
                                                          int64_t N, double *__restrict__ out, int64_t cap,
                                                          unsigned int *__restrict__ colbad, int vec_ok,
                                                          int n_lg, int t_rank) {
    extern __shared__ __align__(16) unsigned char ct_dsm[];
    CtSmem &S = *reinterpret_cast<CtSmem *>(ct_dsm);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool cp_sm = n_lg * C <= CT_CP;     // (visible after the range reduction's barrier)
    if (cp_sm && tid < n_lg * C) S.cp[tid] = col[tid];
    const int64_t base = (int64_t)blockIdx.x * CT_TILE, i0 = base + (int64_t)tid * CT_IPT;
    const int nv = i0 >= N ? 0 : (int)min((int64_t)CT_IPT, N - i0);
    // the event pass and the a3 rank pass use the same 2048-event tiles of 256 threads x 8 events: each thread's
    // run id before its first event + head mask, and its non-MEMOP rank before its first event, give every run id
    // and counter position here (5 + 4 B per 8 events instead of 8 B per event)
    const int64_t th = (int64_t)blockIdx.x * CT_NT + tid;
    // t_run: the run id before the thread's first event, or (t_rank, from k_tile_heads) the in-tile head rank
    const int32_t rrun = nv > 0 ? (t_rank ? (int32_t)(tile_sub[blockIdx.x] - 1) + t_run[th] : t_run[th]) : 0;
    const unsigned hmask = nv > 0 ? (unsigned)t_hm[th] : 0u;
    const int32_t rnm = nv > 0 ? t_nm[th] : 0;
    uint32_t mt[CT_IPT];
    if (vec_ok && nv == CT_IPT) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
            uint4 a = reinterpret_cast<const uint4 *>(meta + i0)[h];
            mt[4 * h] = a.x; mt[4 * h + 1] = a.y; mt[4 * h + 2] = a.z; mt[4 * h + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < CT_IPT; k++) mt[k] = k < nv ? meta[i0 + k] : (uint32_t)CK_MEMOP;   // invalid: MEMOP
    }
    int32_t rid[CT_IPT], nm[CT_IPT];
    {
        int r = rrun, q = rnm, gp = -1;
        int64_t gb = 0;
#pragma unroll
        for (int k = 0; k < CT_IPT; k++) {
            r += (hmask >> k) & 1u;
            rid[k] = r;
            const bool rd = kind_of(mt[k]) != CK_MEMOP;
            const int g = gpu_of(mt[k]);
            if (rd && g != gp) { gb = nm_base[gpu_lg[g]]; gp = g; }
            nm[k] = (int32_t)(q - gb);
            q += rd ? 1 : 0;
        }
    }
    const int32_t prev = rrun;
    const bool has = hmask != 0;
    // the tile's gpu range and counter-rank range over its non-MEMOP events
    int lmin = INT_MAX, lmax = -1, nmin = INT_MAX, nmax = -1;
    {
        int gp = -1, lg = -1;
#pragma unroll
        for (int k = 0; k < CT_IPT; k++) {
            if (kind_of(mt[k]) == CK_MEMOP) continue;
            const int g = gpu_of(mt[k]);
            if (g != gp) { lg = gpu_lg[g]; gp = g; }
            lmin = min(lmin, lg); lmax = max(lmax, lg);
            nmin = min(nmin, nm[k]); nmax = max(nmax, nm[k]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lmin = min(lmin, __shfl_xor_sync(CH_FULL, lmin, o));
            lmax = max(lmax, __shfl_xor_sync(CH_FULL, lmax, o));
            nmin = min(nmin, __shfl_xor_sync(CH_FULL, nmin, o));
            nmax = max(nmax, __shfl_xor_sync(CH_FULL, nmax, o));
        }
        if (lane == 0) { S.red[0][warp] = lmin; S.red[1][warp] = lmax; S.red[2][warp] = nmin; S.red[3][warp] = nmax; }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < CT_WARPS; w++) {
            lmin = min(lmin, S.red[0][w]); lmax = max(lmax, S.red[1][w]);
            nmin = min(nmin, S.red[2][w]); nmax = max(nmax, S.red[3][w]);
        }
    }
    const bool staged = lmax >= 0 && lmin == lmax;      // block-uniform
    const int nlo = nmin, ncnt = nmax - nmin + 1;
    for (int s0 = 0; s0 < C; s0 += CT_SG) {
        unsigned cpm = 0;                     // slots with a staged column
        if (staged) {
#pragma unroll
            for (int q = 0; q < CT_SG; q++) {
                const double *cp = s0 + q < C ? (cp_sm ? S.cp[lmin * C + s0 + q] : col[lmin * C + s0 + q]) : nullptr;
                if (cp) {
                    cpm |= 1u << q;
                    for (int j = tid; j < ncnt; j += CT_NT) cp_async8(&S.x[q][ct_sw(j)], cp + nlo + j);
                }
            }
            cp_async_wait_all();
            __syncthreads();
        }
        double c[CT_SG], p0[CT_SG];
        unsigned bad = 0;
        bool seen = false;
#pragma unroll
        for (int q = 0; q < CT_SG; q++) { c[q] = 0.0; p0[q] = 0.0; }
#pragma unroll
        for (int k = 0; k < CT_IPT; k++) {
            if ((hmask >> k) & 1u) {          // (heads only at valid events; k > 0 once seen)
                if (!seen) {
#pragma unroll
                    for (int q = 0; q < CT_SG; q++) p0[q] = c[q];
                    seen = true;
                } else {
#pragma unroll
                    for (int q = 0; q < CT_SG; q++)
                        if (s0 + q < C) out[(int64_t)(s0 + q) + (int64_t)rid[k > 0 ? k - 1 : 0] * C] = c[q];
                }
#pragma unroll
                for (int q = 0; q < CT_SG; q++) c[q] = 0.0;
            }
            const int kd = kind_of(mt[k]);
            const bool rd = kd != CK_MEMOP;
            double v[CT_SG];
            if (staged) {
                const int j = ct_sw(nm[k] - nlo);
#pragma unroll
                for (int q = 0; q < CT_SG; q++) v[q] = rd && ((cpm >> q) & 1u) ? S.x[q][j] : 0.0;
            } else {                          // tile straddles two gpus (rare): gather from the columns
                const int lg = rd ? gpu_lg[gpu_of(mt[k])] : 0;
#pragma unroll
                for (int q = 0; q < CT_SG; q++) {
                    const double *p = rd && s0 + q < C ? col[lg * C + s0 + q] : nullptr;
                    v[q] = p ? __ldg(p + nm[k]) : 0.0;
                }
            }
#pragma unroll
            for (int q = 0; q < CT_SG; q++) {
                if (!isfinite(v[q])) bad |= 1u << q;
                if (kd == CK_COMPUTE) c[q] += v[q];
            }
        }
        if (bad) {                            // rare: flag the columns holding the non-finite values (R8)
#pragma unroll
            for (int k = 0; k < CT_IPT; k++) {
                if (kind_of(mt[k]) == CK_MEMOP) continue;
                const int lg = gpu_lg[gpu_of(mt[k])];
                for (int q = 0; q < CT_SG; q++) {
                    const double *p = s0 + q < C ? col[lg * C + s0 + q] : nullptr;
                    if (((bad >> q) & 1u) && p && !isfinite(p[nm[k]])) atomicOr(&colbad[lg * C + s0 + q], 1u);
                }
            }
        }
        // segmented inclusive scan of (has, c) inside the warp
        bool f = has;
        double v[CT_SG];
#pragma unroll
        for (int q = 0; q < CT_SG; q++) v[q] = c[q];
        if (!__all_sync(CH_FULL, has)) {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                bool pf = __shfl_up_sync(CH_FULL, f, o);
#pragma unroll
                for (int q = 0; q < CT_SG; q++) {
                    double pv = __shfl_up_sync(CH_FULL, v[q], o);
                    if (lane >= o && !f) v[q] = pv + v[q];
                }
                if (lane >= o) f = f || pf;
            }
        }
        if (lane == 31) {
            S.aflag[warp] = f;
#pragma unroll
            for (int q = 0; q < CT_SG; q++) S.agg[warp][q] = v[q];
        }
        __syncthreads();
        if (tid < CT_WARPS) {
            double cc[CT_SG];
#pragma unroll
            for (int q = 0; q < CT_SG; q++) cc[q] = 0.0;
#pragma unroll
            for (int w = 0; w < CT_WARPS - 1; w++) {
                if (w < tid) {
#pragma unroll
                    for (int q = 0; q < CT_SG; q++) cc[q] = S.aflag[w] ? S.agg[w][q] : cc[q] + S.agg[w][q];
                }
            }
#pragma unroll
            for (int q = 0; q < CT_SG; q++) S.carry[tid][q] = cc[q];
        }
        __syncthreads();
        bool ef = __shfl_up_sync(CH_FULL, f, 1);
        double e[CT_SG];
#pragma unroll
        for (int q = 0; q < CT_SG; q++) e[q] = __shfl_up_sync(CH_FULL, v[q], 1);
        if (lane == 0) {
            ef = false;
#pragma unroll
            for (int q = 0; q < CT_SG; q++) e[q] = 0.0;
        }
        if (!ef) {
#pragma unroll
            for (int q = 0; q < CT_SG; q++) e[q] = S.carry[warp][q] + e[q];
        }
        // the run ending in this thread's first piece (or at the end of the previous thread)
        if (has && tid > 0) {
#pragma unroll
            for (int q = 0; q < CT_SG; q++)
                if (s0 + q < C) out[(int64_t)(s0 + q) + (int64_t)prev * C] = e[q] + p0[q];
        }
        // the run open at the end of the tile
        if (tid == CT_NT - 1 && base < N) {
            const int32_t id = (int32_t)(tile_sub[blockIdx.x + 1] - 1);      // the tile's last run
#pragma unroll
            for (int q = 0; q < CT_SG; q++)
                if (s0 + q < C) out[(int64_t)(s0 + q) + (int64_t)id * C] = f ? v[q] : S.carry[warp][q] + v[q];
        }
        __syncthreads();                      // S.x / S.carry reused by the next slot group
    }
}

struct KeyLayout {
    int sh_op, sh_ly, sh_ph, sh_it, sh_lg;
    int kb[4];
};

__device__ __forceinline__ int64_t comp(unsigned long long key, int sh, int bits) {
    return bits == 0 ? 0 : (int64_t)((key >> sh) & ((1ull << bits) - 1));
}

// ---- instance sort: sub-run keys are produced in dispatch order, so their (gpu, iteration) prefixes
// come in non-decreasing order; only the order inside an iteration is to be established.  Segments of
// equal prefix are sorted in shared memory by (key, sub-run index) -- the order a stable sort gives --
// one block per segment; a full radix sort remains the fallback when the prefix check fails.
constexpr int SS_MAX = 4096, SS_NT = 512;
__global__ void k_prefix_heads(const unsigned long long *__restrict__ key, int64_t n, int sh,
                               int64_t *__restrict__ head) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    head[j] = (j == 0 || (key[j] >> sh) != (key[j - 1] >> sh)) ? 1 : 0;
}
// valid segments must have strictly increasing prefixes; invalid keys (all ones) form their own segments
__global__ void k_seg_starts_end(int64_t *__restrict__ starts, const int64_t *__restrict__ nseg, int64_t n) {
    starts[*nseg] = n;
}
__device__ __forceinline__ void prefix_check_one(const unsigned long long *__restrict__ key,
                                                 const int64_t *__restrict__ starts, int64_t s, int sh,
                                                 unsigned int *__restrict__ bad) {
    const unsigned long long inv = CH_INVALID_KEY >> sh;
    const unsigned long long p = key[starts[s]] >> sh;
    if (starts[s + 1] - starts[s] > SS_MAX) atomicOr(bad, 2u);
    if (p == inv) return;
    for (int64_t t = s - 1; t >= 0 && t >= s - 2; t--) {
        const unsigned long long q = key[starts[t]] >> sh;
        if (q == inv) continue;
        if (q >= p) atomicOr(bad, 1u);
        break;
    }
}
__global__ void k_prefix_check(const unsigned long long *__restrict__ key, const int64_t *__restrict__ starts,
                               const int64_t *__restrict__ nseg_d, int sh, unsigned int *__restrict__ bad) {
    const int64_t nseg = *nseg_d;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x)
        prefix_check_one(key, starts, s, sh, bad);
}
// Inside an iteration the sub-run keys split into four classes by how many trailing levels are "none"
// (op > 0; op = 0 < layer; layer = op = 0 < phase; phase = layer = op = 0).  In dispatch order each class
// is normally already ascending (ops, and the pseudo-op gaps of a layer / phase / iteration, follow time),
// so the segment is a 4-way merge: an element's position = its index in its class + the number of
// smaller keys in each other class (binary searches in shared memory; keys of different classes differ).
// Ties inside a class keep dispatch order (the order of a stable sort).  A segment with an unordered class
// falls back to a bitonic sort by (key, sub-run index).
struct SegSortSmem {
    unsigned long long k[SS_MAX];
    uint32_t v[SS_MAX];
    unsigned long long ck[SS_MAX];      // class-partitioned keys
    uint32_t cv[SS_MAX];
    int cbeg[9];
    int unsorted;
    int64_t scan[33];
};
__device__ __forceinline__ int seg_class(unsigned long long k, const KeyLayout &L) {
    if (k == CH_INVALID_KEY) return 7;
    return (comp(k, L.sh_op, L.kb[3]) == 0 ? 1 : 0) | (comp(k, L.sh_ly, L.kb[2]) == 0 ? 2 : 0) |
           (comp(k, L.sh_ph, L.kb[1]) == 0 ? 4 : 0);
}
__device__ void seg_sort_one(SegSortSmem &S, unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals,
                             int64_t lo, int64_t hi, const KeyLayout &L);
__global__ void __launch_bounds__(SS_NT) k_seg_sort(unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals,
                                                    const int64_t *__restrict__ starts, const int64_t *__restrict__ nseg_d,
                                                    KeyLayout L) {
    extern __shared__ __align__(16) unsigned char ss_dsm[];
    SegSortSmem &S = *reinterpret_cast<SegSortSmem *>(ss_dsm);
    const int64_t nseg = *nseg_d;
    for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        seg_sort_one(S, keys, vals, starts[sg], starts[sg + 1], L);
        __syncthreads();
    }
}
__device__ void seg_sort_one(SegSortSmem &S, unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals,
                             int64_t lo, int64_t hi, const KeyLayout &L) {
    const int n = (int)(hi - lo);
    if (n <= 1 || n > SS_MAX) return;
    bool sorted = true;   // fast exit for an already ordered segment
    for (int i = threadIdx.x + 1; i < n; i += blockDim.x)
        if (keys[lo + i] < keys[lo + i - 1]) sorted = false;
    if (__syncthreads_and(sorted)) return;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { S.k[i] = keys[lo + i]; S.v[i] = vals[lo + i]; }
    if (threadIdx.x == 0) { S.unsorted = 0; S.cbeg[0] = 0; }
    __syncthreads();
    // stable partition by class: per-thread chunk counts, two packed block scans (4 x 16-bit counters)
    const int per = (n + SS_NT - 1) / SS_NT;
    const int i0 = threadIdx.x * per, i1 = min(n, i0 + per);
    unsigned long long cnt[2] = {0, 0};
    for (int i = i0; i < i1; i++) {
        const int c = seg_class(S.k[i], L);
        cnt[c >> 2] += 1ull << (16 * (c & 3));
    }
    int cb[8], pos[8];
    int run = 0;
    for (int h = 0; h < 2; h++) {
        int64_t tot;
        const unsigned long long ex = (unsigned long long)block_excl_sum<SS_NT>((int64_t)cnt[h], &tot, S.scan);
        const unsigned long long t64 = (unsigned long long)tot;
        for (int c = 0; c < 4; c++) {
            cb[4 * h + c] = run;
            pos[4 * h + c] = run + (int)((ex >> (16 * c)) & 0xFFFF);
            run += (int)((t64 >> (16 * c)) & 0xFFFF);
        }
    }
    if (threadIdx.x == 0) {
        for (int c = 0; c < 8; c++) S.cbeg[c] = cb[c];
        S.cbeg[8] = n;
    }
    for (int i = i0; i < i1; i++) {
        const int c = seg_class(S.k[i], L);
        const int d = pos[c]++;
        S.ck[d] = S.k[i];
        S.cv[d] = S.v[i];
    }
    __syncthreads();
    // every class ascending?
    for (int c = 0; c < 8; c++)
        for (int d = S.cbeg[c] + 1 + threadIdx.x; d < S.cbeg[c + 1]; d += blockDim.x)
            if (S.ck[d] < S.ck[d - 1]) S.unsorted = 1;
    __syncthreads();
    if (!S.unsorted) {
        for (int d = threadIdx.x; d < n; d += blockDim.x) {
            int c = 0;
            while (d >= S.cbeg[c + 1]) c++;
            const unsigned long long x = S.ck[d];
            int p = d - S.cbeg[c];
            for (int o = 0; o < 8; o++) {
                if (o == c || S.cbeg[o] == S.cbeg[o + 1]) continue;
                int l2 = S.cbeg[o], h2 = S.cbeg[o + 1];     // count of class-o keys < x
                while (l2 < h2) {
                    const int m = (l2 + h2) >> 1;
                    if (S.ck[m] < x) l2 = m + 1; else h2 = m;
                }
                p += l2 - S.cbeg[o];
            }
            keys[lo + p] = x;
            vals[lo + p] = S.cv[d];
        }
        return;
    }
    // fallback: bitonic sort by (key, sub-run index)
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        if (i >= n) { S.k[i] = ~0ull; S.v[i] = 0xFFFFFFFFu; }
    }
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int x = i ^ j;
                if (x > i) {
                    const bool up = (i & k) == 0;
                    const unsigned long long a2 = S.k[i], b2 = S.k[x];
                    const uint32_t va = S.v[i], vb = S.v[x];
                    const bool gt = a2 > b2 || (a2 == b2 && va > vb);
                    if (gt == up) { S.k[i] = b2; S.k[x] = a2; S.v[i] = vb; S.v[x] = va; }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) { keys[lo + i] = S.k[i]; vals[lo + i] = S.v[i]; }
}

// stable partition: valid keys first (in order), invalid keys after
__global__ void k_valid_flags(const unsigned long long *__restrict__ key, int64_t n, int64_t *__restrict__ f) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) f[j] = key[j] != CH_INVALID_KEY ? 1 : 0;
}
__global__ void k_partition(const unsigned long long *__restrict__ ki, const uint32_t *__restrict__ vi, int64_t n,
                            const int64_t *__restrict__ ex, const int64_t *__restrict__ nvalid,
                            unsigned long long *__restrict__ ko, uint32_t *__restrict__ vo) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const bool v = ki[j] != CH_INVALID_KEY;
    const int64_t p = v ? ex[j] : *nvalid + (j - ex[j]);
    ko[p] = ki[j];
    vo[p] = vi[j];
}

__global__ void k_copy_keys(const unsigned long long *__restrict__ k, int64_t n, unsigned long long *__restrict__ out,
                            uint32_t *__restrict__ v) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { out[i] = k[i]; v[i] = (uint32_t)i; }
}

// heads of groups of equal (key >> shift) among valid keys; also the valid count
// device-resident row counts: kernels are sized by a host upper bound and read the true count
__device__ __forceinline__ int64_t dev_n(int64_t n, const int64_t *n_dev) {
    if (!n_dev) return n;
    const int64_t m = *n_dev;
    return m < n ? m : n;
}
__global__ void k_group_init(unsigned long long *nvalid, int64_t n, const int64_t *__restrict__ n_dev) {
    *nvalid = (unsigned long long)dev_n(n, n_dev);
}
// the end of the last group: the first invalid key (invalid keys sort last)
__global__ void k_group_finish(int64_t *__restrict__ starts, const int64_t *__restrict__ ng,
                               const unsigned long long *__restrict__ nvalid) {
    starts[*ng] = (int64_t)*nvalid;
}
// One pass per grouping: heads (first key of each run of equal key >> shift among the valid keys, which sort
// first), their exclusive scan by a chained scan with decoupled look-back, and starts[g] = position of group g's
// first key; the block holding the last valid key writes the group count and starts[count] = the number of
// valid keys.  Blocks past the device-side count exit at once (nobody looks back past the last valid key).
constexpr int GP_NT = 256, GP_IPT = 8, GP_TILE = GP_NT * GP_IPT;
constexpr unsigned long long GP_A = 1ull << 62, GP_P = 2ull << 62, GP_MASK = (1ull << 62) - 1;
__global__ void __launch_bounds__(GP_NT) k_group_1pass(const unsigned long long *__restrict__ key, int64_t n,
                                                        const int64_t *__restrict__ n_dev, int shift, int all,
                                                        int64_t *__restrict__ starts, int64_t *__restrict__ ng,
                                                        unsigned long long *__restrict__ state,
                                                        unsigned int *__restrict__ ticket) {
    __shared__ int s_w[GP_NT / 32];
    __shared__ int64_t s_tile, s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ne = dev_n(n, n_dev);
    if (tid == 0) s_tile = (int64_t)atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t b0 = tile * GP_TILE;
    if (b0 >= ne && !(ne == 0 && tile == 0)) return;
    const int64_t j0 = b0 + (int64_t)tid * GP_IPT;
    unsigned long long prev = j0 > 0 && j0 - 1 < ne ? key[j0 - 1] : CH_INVALID_KEY;
    unsigned hm = 0;
    int last_valid = -1;       // k of the last valid key of the tile, if its successor is invalid / past the end
#pragma unroll
    for (int k = 0; k < GP_IPT; k++) {
        const int64_t j = j0 + k;
        const unsigned long long x = j < ne ? key[j] : CH_INVALID_KEY;
        if (j < ne && (all || x != CH_INVALID_KEY)) {
            const unsigned long long g = shift >= 64 ? 0ull : (x >> shift);
            const unsigned long long gp = shift >= 64 ? 0ull : (prev >> shift);
            if (j == 0 || (!all && prev == CH_INVALID_KEY) || gp != g) hm |= 1u << k;
            if (j + 1 >= ne || (!all && key[j + 1] == CH_INVALID_KEY)) last_valid = k;
        }
        prev = x;
    }
    const int nh = __popc(hm);
    int wex = nh;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(CH_FULL, wex, o);
        if (lane >= o) wex += y;
    }
    if (lane == 31) s_w[warp] = wex;
    wex -= nh;
    __syncthreads();
    int wb = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < GP_NT / 32; w++) {
        const int c = s_w[w];
        if (w < warp) wb += c;
        tot += c;
    }
    if (warp == 0) {
        int64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&state[0], GP_P | (unsigned long long)tot);
        } else {
            if (lane == 0) atomicExch(&state[tile], GP_A | (unsigned long long)tot);
            int64_t p = tile - 1 - lane;
            while (true) {
                unsigned long long st = GP_P;
                if (p >= 0) st = *((volatile unsigned long long *)&state[p]);
                const unsigned fl = (unsigned)(st >> 62);
                const unsigned pm = __ballot_sync(CH_FULL, fl == 2u), zm = __ballot_sync(CH_FULL, fl == 0u);
                const int fp = pm ? __ffs(pm) - 1 : 32;
                const unsigned need = fp >= 31 ? CH_FULL : ((2u << fp) - 1u);
                if (zm & need) continue;
                int64_t x = lane <= fp ? (int64_t)(st & GP_MASK) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(CH_FULL, x, o);
                excl += x;
                if (fp < 32) break;
                p -= 32;
            }
            if (lane == 0) atomicExch(&state[tile], GP_P | (unsigned long long)(excl + tot));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    int64_t o = s_excl + wb + wex;
#pragma unroll
    for (int k = 0; k < GP_IPT; k++)
        if ((hm >> k) & 1u) starts[o++] = j0 + k;
    if (last_valid >= 0) {
        const int64_t cnt = s_excl + tot;
        *ng = cnt;
        starts[cnt] = j0 + last_valid + 1;
    }
    if (tile == 0 && tid == 0 && (ne == 0 || (!all && key[0] == CH_INVALID_KEY))) {
        *ng = 0;
        starts[0] = 0;
    }
}

// valid keys (with their values) to the front in order, invalid ones to the back (reversed: their order is
// never used), one chained-scan pass; *nvalid = the number of valid keys (written by the last tile)
__global__ void __launch_bounds__(GP_NT) k_compact_1pass(const unsigned long long *__restrict__ ki,
                                                          const uint32_t *__restrict__ vi, int64_t n,
                                                          unsigned long long *__restrict__ ko, uint32_t *__restrict__ vo,
                                                          int64_t *__restrict__ nvalid,
                                                          unsigned long long *__restrict__ state,
                                                          unsigned int *__restrict__ ticket) {
    __shared__ int s_w[GP_NT / 32];
    __shared__ int64_t s_tile, s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (int64_t)atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t j0 = tile * GP_TILE + (int64_t)tid * GP_IPT;
    unsigned long long x[GP_IPT];
    unsigned vm = 0;
#pragma unroll
    for (int k = 0; k < GP_IPT; k++) {
        x[k] = j0 + k < n ? ki[j0 + k] : CH_INVALID_KEY;
        if (j0 + k < n && x[k] != CH_INVALID_KEY) vm |= 1u << k;
    }
    const int nh = __popc(vm);
    int wex = nh;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(CH_FULL, wex, o);
        if (lane >= o) wex += y;
    }
    if (lane == 31) s_w[warp] = wex;
    wex -= nh;
    __syncthreads();
    int wb = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < GP_NT / 32; w++) {
        const int c = s_w[w];
        if (w < warp) wb += c;
        tot += c;
    }
    if (warp == 0) {
        int64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&state[0], GP_P | (unsigned long long)tot);
        } else {
            if (lane == 0) atomicExch(&state[tile], GP_A | (unsigned long long)tot);
            int64_t p = tile - 1 - lane;
            while (true) {
                unsigned long long st = GP_P;
                if (p >= 0) st = *((volatile unsigned long long *)&state[p]);
                const unsigned fl = (unsigned)(st >> 62);
                const unsigned pm = __ballot_sync(CH_FULL, fl == 2u), zm = __ballot_sync(CH_FULL, fl == 0u);
                const int fp = pm ? __ffs(pm) - 1 : 32;
                const unsigned need = fp >= 31 ? CH_FULL : ((2u << fp) - 1u);
                if (zm & need) continue;
                int64_t y = lane <= fp ? (int64_t)(st & GP_MASK) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(CH_FULL, y, o);
                excl += y;
                if (fp < 32) break;
                p -= 32;
            }
            if (lane == 0) atomicExch(&state[tile], GP_P | (unsigned long long)(excl + tot));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    int64_t e = s_excl + wb + wex;                  // valid keys before this thread's first
#pragma unroll
    for (int k = 0; k < GP_IPT; k++) {
        const int64_t j = j0 + k;
        if (j >= n) break;
        const int64_t p = ((vm >> k) & 1u) ? e : n - 1 - (j - e);
        ko[p] = x[k];
        vo[p] = vi[j];
        e += (vm >> k) & 1u;
    }
    if (j0 <= n - 1 && n - 1 < j0 + GP_IPT) *nvalid = e;
}

__global__ void k_group_heads(const unsigned long long *__restrict__ key, int64_t n, const int64_t *__restrict__ n_dev,
                              int shift, int64_t *__restrict__ head, unsigned long long *__restrict__ nvalid) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    if (j >= dev_n(n, n_dev)) { head[j] = 0; return; }
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
    int64_t ccap;    // counter-column stride (field-major tables: capacity; AoS sub-run counters: 1)
    int64_t rs;      // row stride (field-major: 1; AoS sub-runs: 16)
    int64_t crs;     // counter row stride (field-major: 1; AoS sub-run counters: C)
};

// parent row p = sum of children [starts[p], starts[p+1]) (through perm if given).  Integer fields are
// exact in any order; first = lexicographic min of (first_ks, first_idx), last_ke = max.  One lane per
// parent for small groups (children in ascending order); groups of more than SR_SMALL children are
// summed by the whole warp (lanes stride the children, then a butterfly), which keeps a 200-child
// iteration->gpu group off a single thread's dependent load chain.  fp64 counter sums of big groups
// are tree-ordered (within the 1e-9 budget, D12/D22).
constexpr int SR_SMALL = 8;
struct RowAcc {
    int64_t v[RF_NFIELDS];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int f = 0; f < RF_NFIELDS; f++) v[f] = 0;
        v[RF_FIRST_IDX] = INT64_MAX;
        v[RF_FIRST_KS] = INT64_MAX;
        v[RF_LAST_KE] = INT64_MIN;
    }
    __device__ __forceinline__ void add_child(const TabView &ch, int64_t c) {
        const int64_t *b = ch.f + c * ch.rs;
        int64_t x[RF_NFIELDS];
#pragma unroll
        for (int f = 0; f < RF_NFIELDS; f++) x[f] = b[(int64_t)f * ch.cap];
        merge(x);
    }
    __device__ __forceinline__ void merge(const int64_t *x) {
#pragma unroll
        for (int f = 0; f < RF_NFIELDS; f++)
            if (f != RF_FIRST_IDX && f != RF_FIRST_KS && f != RF_LAST_KE) v[f] += x[f];
        if (x[RF_LAST_KE] > v[RF_LAST_KE]) v[RF_LAST_KE] = x[RF_LAST_KE];
        if (x[RF_FIRST_KS] < v[RF_FIRST_KS] || (x[RF_FIRST_KS] == v[RF_FIRST_KS] && x[RF_FIRST_IDX] < v[RF_FIRST_IDX])) {
            v[RF_FIRST_KS] = x[RF_FIRST_KS];
            v[RF_FIRST_IDX] = x[RF_FIRST_IDX];
        }
    }
    __device__ __forceinline__ void warp_all() {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            int64_t y[RF_NFIELDS];
#pragma unroll
            for (int f = 0; f < RF_NFIELDS; f++) y[f] = __shfl_xor_sync(CH_FULL, v[f], o);
            merge(y);
        }
    }
};

__device__ __forceinline__ void sum_rows_thread_body(const TabView &ch, const uint32_t *__restrict__ perm,
                                                     const int64_t *__restrict__ starts, int64_t ng, int shift, int C,
                                                     const TabView &pa, int64_t p) {
    const int lane = lane_id();
    const bool valid = p < ng;
    int64_t lo = 0, hi = 0;
    if (valid) { lo = starts[p]; hi = starts[p + 1]; }
    const bool big = valid && hi - lo > SR_SMALL;
    if (valid && !big) {
        RowAcc a;
        a.zero();
        for (int64_t j = lo; j < hi; j++) a.add_child(ch, perm ? (int64_t)perm[j] : j);
#pragma unroll
        for (int f = 0; f < RF_NFIELDS; f++) pa.f[(int64_t)f * pa.cap + p] = a.v[f];
        unsigned long long k0 = hi > lo ? ch.key[perm ? (int64_t)perm[lo] : lo] : 0ull;
        pa.key[p] = shift >= 64 ? 0ull : ((k0 >> shift) << shift);
        for (int s = 0; s < C; s++) {
            double acc = 0.0;
            for (int64_t j = lo; j < hi; j++) acc += ch.cnt[(int64_t)s * ch.ccap + (perm ? (int64_t)perm[j] : j) * ch.crs];
            pa.cnt[(int64_t)s * pa.ccap + p] = acc;
        }
    }
    // big groups: the warp works through them one at a time
    unsigned bm = __ballot_sync(CH_FULL, big);
    while (bm) {
        const int src = __ffs(bm) - 1;
        bm &= bm - 1;
        const int64_t q = __shfl_sync(CH_FULL, p, src);
        const int64_t qlo = __shfl_sync(CH_FULL, lo, src), qhi = __shfl_sync(CH_FULL, hi, src);
        RowAcc a;
        a.zero();
        for (int64_t j = qlo + lane; j < qhi; j += 32) a.add_child(ch, perm ? (int64_t)perm[j] : j);
        a.warp_all();
        if (lane < RF_NFIELDS) {
            int64_t x = a.v[0];
#pragma unroll
            for (int f = 1; f < RF_NFIELDS; f++) if (lane == f) x = a.v[f];
            pa.f[(int64_t)lane * pa.cap + q] = x;
        }
        if (lane == 0) {
            unsigned long long k0 = ch.key[perm ? (int64_t)perm[qlo] : qlo];
            pa.key[q] = shift >= 64 ? 0ull : ((k0 >> shift) << shift);
        }
        for (int s = 0; s < C; s++) {
            double acc = 0.0;
            for (int64_t j = qlo + lane; j < qhi; j += 32) acc += ch.cnt[(int64_t)s * ch.ccap + (perm ? (int64_t)perm[j] : j) * ch.crs];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(CH_FULL, acc, o);
            if (lane == 0) pa.cnt[(int64_t)s * pa.ccap + q] = acc;
        }
    }
}

__global__ void __launch_bounds__(256) k_sum_rows(TabView ch, const uint32_t *__restrict__ perm,
                                                  const int64_t *__restrict__ starts, const int64_t *__restrict__ ng_dev,
                                                  int shift, int C, TabView pa) {
    const int64_t ng = *ng_dev;
    for (int64_t pb = (int64_t)blockIdx.x * blockDim.x; pb < ng; pb += (int64_t)gridDim.x * blockDim.x)
        sum_rows_thread_body(ch, perm, starts, ng, shift, C, pa, pb + threadIdx.x);
}

// warp per parent (groups averaging several children: layer / phase / iteration / gpu roll-ups and
// points): lanes take consecutive children (coalesced on field-major tables), every field and counter
// in one pass, then a butterfly.
// CMAX: the counter accumulators held per lane (0 without counters, 8, 32): sized to the trace, so a run without
// counters keeps its registers (and occupancy) for the row fields
template <int CMAX>
__global__ void __launch_bounds__(256) k_sum_rows_warp(TabView ch, const uint32_t *__restrict__ perm,
                                                       const int64_t *__restrict__ starts,
                                                       const int64_t *__restrict__ ng_dev, int shift, int C,
                                                       TabView pa) {
    const int lane = lane_id();
    const int64_t ng = *ng_dev;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < ng; q += nw) {
    const int64_t qlo = starts[q], qhi = starts[q + 1];
    RowAcc a;
    a.zero();
    double acc[CMAX > 0 ? CMAX : 1];
#pragma unroll
    for (int s = 0; s < CMAX; s++) acc[s] = 0.0;
    for (int64_t j = qlo + lane; j < qhi; j += 32) {
        const int64_t c = perm ? (int64_t)perm[j] : j;
        a.add_child(ch, c);
#pragma unroll
        for (int s = 0; s < CMAX; s++)
            if (s < C) acc[s] += ch.cnt[(int64_t)s * ch.ccap + (c) * ch.crs];
    }
    a.warp_all();
    if (lane < RF_NFIELDS) {
        int64_t x = a.v[0];
#pragma unroll
        for (int f = 1; f < RF_NFIELDS; f++) if (lane == f) x = a.v[f];
        pa.f[(int64_t)lane * pa.cap + q] = x;
    }
    if (lane == 0) {
        unsigned long long k0 = qhi > qlo ? ch.key[perm ? (int64_t)perm[qlo] : qlo] : 0ull;
        pa.key[q] = shift >= 64 ? 0ull : ((k0 >> shift) << shift);
    }
#pragma unroll
    for (int s = 0; s < CMAX; s++) {
        if (s < C) {
            double x = acc[s];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(CH_FULL, x, o);
            if (lane == 0) pa.cnt[(int64_t)s * pa.ccap + q] = x;
        }
    }
    }
}

// block of RC_NT parents: their children (a contiguous range, or a perm range) are staged RC_CH at a time
// in shared memory -- coalesced column loads for field-major tables, one 128 B row per child for the
// AoS sub-run rows -- and each thread folds its own parent's children from shared memory in order.
constexpr int RC_NT = 256, RC_CH = 256;
__global__ void __launch_bounds__(RC_NT, 3) k_sum_rows_chunked(TabView ch, const uint32_t *__restrict__ perm,
                                                            const int64_t *__restrict__ starts,
                                                            const int64_t *__restrict__ ng_dev, int shift, int C,
                                                            TabView pa, int PB) {
    // PB parents per block (<= RC_NT): about RC_CH children per block-iteration keeps the loads wide
    extern __shared__ int64_t rsm[];
    const int NF = RF_NFIELDS + C;
    int64_t *vals = rsm;                               // [NF][RC_CH]
    const int tid = threadIdx.x;
    const int64_t ng = *ng_dev;
    for (int64_t p0 = (int64_t)blockIdx.x * PB; p0 < ng; p0 += (int64_t)gridDim.x * PB) {
    const int64_t pend = min(p0 + PB, ng);
    const int64_t p = tid < PB ? p0 + tid : ng;
    const int64_t c_lo = starts[p0], c_hi = starts[pend];
    int64_t my_lo = 0, my_hi = 0;
    if (p < ng) { my_lo = starts[p]; my_hi = starts[p + 1]; }
    RowAcc a;
    a.zero();
    double cs[8];
#pragma unroll
    for (int s2 = 0; s2 < 8; s2++) cs[s2] = 0.0;
    for (int64_t j0 = c_lo; j0 < c_hi; j0 += RC_CH) {
        const int m = (int)min((int64_t)RC_CH, c_hi - j0);
        if (ch.rs == 1 && !perm) {
            // all of a thread's column loads in flight before the shared-memory stores (RC_NT == RC_CH:
            // thread t owns child j0 + t in every column)
            if (tid < m) {
                const int64_t c = j0 + tid;
                int64_t x[RF_NFIELDS];
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) x[f] = __ldg(ch.f + (int64_t)f * ch.cap + c);
                int64_t y[8];
#pragma unroll
                for (int q = 0; q < 8; q++) y[q] = q < C ? __double_as_longlong(__ldg(ch.cnt + (int64_t)q * ch.ccap + c * ch.crs)) : 0;
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) vals[f * RC_CH + tid] = x[f];
#pragma unroll
                for (int q = 0; q < 8; q++) if (q < C) vals[(RF_NFIELDS + q) * RC_CH + tid] = y[q];
                for (int q = 8; q < C; q++)
                    vals[(RF_NFIELDS + q) * RC_CH + tid] = __double_as_longlong(ch.cnt[(int64_t)q * ch.ccap + (c) * ch.crs]);
            }
        } else if (ch.cap == 1 && ch.rs == 16 && ch.ccap == 1 && ch.crs == C && C <= 8 && (C & 1) == 0) {
            // AoS sub-runs: one 128 B row and C*8 B of counters per child, 16 B vector loads
            for (int t = tid; t < m; t += RC_NT) {
                const int64_t c = perm ? (int64_t)perm[j0 + t] : j0 + t;
                const longlong2 *row = reinterpret_cast<const longlong2 *>(ch.f + c * 16);
                longlong2 x[8];
#pragma unroll
                for (int f = 0; f < 8; f++) x[f] = __ldg(row + f);
                longlong2 y[4];
                const longlong2 *cr = reinterpret_cast<const longlong2 *>(ch.cnt + c * C);
#pragma unroll
                for (int q = 0; q < 4; q++) y[q] = 2 * q < C ? __ldg(cr + q) : make_longlong2(0, 0);
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) vals[f * RC_CH + t] = (f & 1) ? x[f >> 1].y : x[f >> 1].x;
#pragma unroll
                for (int q = 0; q < 8; q++)
                    if (q < C) vals[(RF_NFIELDS + q) * RC_CH + t] = (q & 1) ? y[q >> 1].y : y[q >> 1].x;
            }
        } else {
            for (int t = tid; t < m; t += RC_NT) {
                const int64_t c = perm ? (int64_t)perm[j0 + t] : j0 + t;
                const int64_t *row = ch.f + c * ch.rs;
                int64_t x[RF_NFIELDS];
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) x[f] = __ldg(row + (int64_t)f * ch.cap);
                int64_t y[8];
#pragma unroll
                for (int q = 0; q < 8; q++) y[q] = q < C ? __double_as_longlong(__ldg(ch.cnt + (int64_t)q * ch.ccap + c * ch.crs)) : 0;
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) vals[f * RC_CH + t] = x[f];
#pragma unroll
                for (int q = 0; q < 8; q++) if (q < C) vals[(RF_NFIELDS + q) * RC_CH + t] = y[q];
                for (int s2 = 8; s2 < C; s2++)
                    vals[(RF_NFIELDS + s2) * RC_CH + t] = __double_as_longlong(ch.cnt[(int64_t)s2 * ch.ccap + (c) * ch.crs]);
            }
        }
        __syncthreads();
        const int64_t a0 = my_lo > j0 ? my_lo : j0, a1 = my_hi < j0 + m ? my_hi : j0 + m;
        for (int64_t c = a0; c < a1; c++) {
            const int t = (int)(c - j0);
            int64_t x[RF_NFIELDS];
#pragma unroll
            for (int f = 0; f < RF_NFIELDS; f++) x[f] = vals[f * RC_CH + t];
            a.merge(x);
#pragma unroll
            for (int s2 = 0; s2 < 8; s2++)
                if (s2 < C) cs[s2] += __longlong_as_double(vals[(RF_NFIELDS + s2) * RC_CH + t]);
            for (int s2 = 8; s2 < C; s2++)            // C > 8: accumulate in place
                pa.cnt[(int64_t)s2 * pa.ccap + p] += __longlong_as_double(vals[(RF_NFIELDS + s2) * RC_CH + t]);
        }
        __syncthreads();
    }
    if (p < ng) {
#pragma unroll
        for (int f = 0; f < RF_NFIELDS; f++) pa.f[(int64_t)f * pa.cap + p] = a.v[f];
#pragma unroll
        for (int s2 = 0; s2 < 8; s2++)
            if (s2 < C) pa.cnt[(int64_t)s2 * pa.ccap + p] = cs[s2];
        const unsigned long long k0 = my_hi > my_lo ? ch.key[perm ? (int64_t)perm[my_lo] : my_lo] : 0ull;
        pa.key[p] = shift >= 64 ? 0ull : ((k0 >> shift) << shift);
    }
    }
}

// Field-major children with several children per parent (instance -> layer): staged like
// k_sum_rows_chunked, but the fold is split by (column, parent) so that all threads work -- thread task
// (f, i) folds column f of parent i over its children in order (counter sums keep the sequential child
// order); running values live in shared memory across chunks.  C <= 8.
__global__ void __launch_bounds__(RC_NT, 4) k_sum_rows_cols(TabView ch, const int64_t *__restrict__ starts,
                                                         const int64_t *__restrict__ ng_dev, int shift, int C,
                                                         TabView pa, int PB) {
    extern __shared__ int64_t rsm[];
    const int NF = RF_NFIELDS + C;
    int64_t *vals = rsm;                               // [NF][RC_CH]
    int64_t *acc = rsm + NF * RC_CH;                   // [NF][PB]
    __shared__ int64_t s_lo[RC_NT + 1];
    const int tid = threadIdx.x;
    const int64_t ng = *ng_dev;
    for (int64_t p0 = (int64_t)blockIdx.x * PB; p0 < ng; p0 += (int64_t)gridDim.x * PB) {
        const int np = (int)min((int64_t)PB, ng - p0);
        __syncthreads();
        for (int i = tid; i <= np; i += RC_NT) s_lo[i] = starts[p0 + i];
        for (int t = tid; t < NF * np; t += RC_NT) {
            const int f = t / np;
            acc[f * PB + t % np] = f == RF_FIRST_IDX || f == RF_FIRST_KS ? INT64_MAX : f == RF_LAST_KE ? INT64_MIN : 0;
        }
        __syncthreads();
        const int64_t c_lo = s_lo[0], c_hi = s_lo[np];
        for (int64_t j0 = c_lo; j0 < c_hi; j0 += RC_CH) {
            const int m = (int)min((int64_t)RC_CH, c_hi - j0);
            if (tid < m) {
                const int64_t c = j0 + tid;
                int64_t x[RF_NFIELDS];
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) x[f] = __ldg(ch.f + (int64_t)f * ch.cap + c);
                int64_t y[8];
#pragma unroll
                for (int q = 0; q < 8; q++) y[q] = q < C ? __double_as_longlong(__ldg(ch.cnt + (int64_t)q * ch.ccap + c * ch.crs)) : 0;
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) vals[f * RC_CH + tid] = x[f];
#pragma unroll
                for (int q = 0; q < 8; q++) if (q < C) vals[(RF_NFIELDS + q) * RC_CH + tid] = y[q];
            }
            __syncthreads();
            for (int t = tid; t < NF * np; t += RC_NT) {
                const int f = t / np, i = t - f * np;
                if (f == RF_FIRST_IDX) continue;                  // folded with RF_FIRST_KS
                const int64_t lo = max(s_lo[i], j0), hi = min(s_lo[i + 1], j0 + m);
                if (lo >= hi) continue;
                const int64_t *v = vals + f * RC_CH - j0;
                int64_t &a = acc[f * PB + i];
                if (f >= RF_NFIELDS) {
                    double x = __longlong_as_double(a);
                    for (int64_t c = lo; c < hi; c++) x += __longlong_as_double(v[c]);
                    a = __double_as_longlong(x);
                } else if (f == RF_LAST_KE) {
                    int64_t x = a;
                    for (int64_t c = lo; c < hi; c++) x = max(x, v[c]);
                    a = x;
                } else if (f == RF_FIRST_KS) {
                    const int64_t *vi = vals + RF_FIRST_IDX * RC_CH - j0;
                    int64_t ks = a, ix = acc[RF_FIRST_IDX * PB + i];
                    for (int64_t c = lo; c < hi; c++)
                        if (v[c] < ks || (v[c] == ks && vi[c] < ix)) { ks = v[c]; ix = vi[c]; }
                    a = ks;
                    acc[RF_FIRST_IDX * PB + i] = ix;
                } else {
                    int64_t x = a;
                    for (int64_t c = lo; c < hi; c++) x += v[c];
                    a = x;
                }
            }
            __syncthreads();
        }
        for (int t = tid; t < NF * np; t += RC_NT) {
            const int f = t / np, i = t - f * np;
            const int64_t x = acc[f * PB + i];
            if (f < RF_NFIELDS) pa.f[(int64_t)f * pa.cap + p0 + i] = x;
            else pa.cnt[(int64_t)(f - RF_NFIELDS) * pa.ccap + p0 + i] = __longlong_as_double(x);
        }
        for (int i = tid; i < np; i += RC_NT) {
            const unsigned long long k0 = s_lo[i + 1] > s_lo[i] ? ch.key[s_lo[i]] : 0ull;
            pa.key[p0 + i] = shift >= 64 ? 0ull : ((k0 >> shift) << shift);
        }
    }
}

// identity columns of a row table: caller span indices, gpu, op label, iteration rank
__global__ void k_decode(const unsigned long long *__restrict__ key, const int64_t *__restrict__ n_dev, KeyLayout L,
                         int depth,
                         const int32_t *__restrict__ lg_gpu, const int64_t *__restrict__ list_beg,
                         const int32_t *__restrict__ P_orig, const int32_t *__restrict__ P_label,
                         const int64_t *__restrict__ f, int64_t cap, PredView pv,
                         int32_t *gpu, int32_t *it, int32_t *ph, int32_t *ly, int32_t *op, int32_t *label,
                         int32_t *rank, int64_t *first_pred) {
    const int64_t n = *n_dev;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
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
    first_pred[j] = (fi != INT64_MAX) ? pred_of(pv, fi) : CH_NONE_TS;
    }
}

// point key: (op label, gpu, iteration rank); instances without an op span are dropped

// points (gpu, iteration, op label) = instances of the iteration with that op label, summed over layers
// in instance order.  One block per iteration group of the sorted instance table:
// chunks of PT_CH instances are loaded coalesced into shared memory, then thread l folds the chunk's
// instances with label l in order.  Results go to a dense [label][lg][rank] grid (compacted afterwards in
// (label, lg, rank) order = point-key order).
constexpr int PT_CH = 256;
__device__ void points_iter_one(TabView iv, const int64_t *__restrict__ its, int64_t g, KeyLayout Lk,
                                const int64_t *__restrict__ list_beg, const int32_t *__restrict__ P_label, int nL,
                                int n_lg, int R0, int C, int64_t *__restrict__ df, double *__restrict__ dc,
                                int64_t *__restrict__ dvalid, unsigned int *__restrict__ ovf);
__global__ void __launch_bounds__(256) k_points_iter(TabView iv, const int64_t *__restrict__ its,
                                                     const int64_t *__restrict__ n_it_d, KeyLayout Lk,
                                                     const int64_t *__restrict__ list_beg,
                                                     const int32_t *__restrict__ P_label, int nL, int n_lg, int R0,
                                                     int C, int64_t *__restrict__ df, double *__restrict__ dc,
                                                     int64_t *__restrict__ dvalid, unsigned int *__restrict__ ovf) {
    const int64_t n_it = *n_it_d;
    for (int64_t g = blockIdx.x; g < n_it; g += gridDim.x) {
        points_iter_one(iv, its, g, Lk, list_beg, P_label, nL, n_lg, R0, C, df, dc, dvalid, ovf);
        __syncthreads();
    }
}
__device__ void points_iter_one(TabView iv, const int64_t *__restrict__ its, int64_t g,
                                KeyLayout Lk, const int64_t *__restrict__ list_beg,
                                const int32_t *__restrict__ P_label, int nL, int n_lg, int R0,
                                int C, int64_t *__restrict__ df, double *__restrict__ dc,
                                int64_t *__restrict__ dvalid, unsigned int *__restrict__ ovf) {
    // one instance per thread per chunk; a stable counting sort by label puts each label's instances of
    // the chunk in a contiguous list (instance order), which the block then folds split by (column, label):
    // task (f, l) folds column f of label l's list in order (running values in shared memory)
    extern __shared__ int64_t psm[];
    const int NF = RF_NFIELDS + C;
    int64_t *vals = psm;                                                      // [NF][PT_CH]
    int64_t *pacc = vals + (int64_t)NF * PT_CH;                               // [NF][nL] running values
    int32_t *lab = reinterpret_cast<int32_t *>(pacc + (int64_t)NF * nL);      // [PT_CH]
    int32_t *order = lab + PT_CH;                                             // [PT_CH]
    int32_t *wc = order + PT_CH;                                              // [8][nL] per-warp counts
    int32_t *lstart = wc + 8 * nL;                                            // [nL]
    int32_t *ltot = lstart + nL;                                              // [nL] chunk list length
    int32_t *lcnt = ltot + nL;                                                // [nL] instances folded
    __shared__ int64_t scan_sm[33];
    const int64_t a = its[g], b = its[g + 1];
    const unsigned long long k0 = iv.key[a];
    const int lg = (int)(k0 >> Lk.sh_lg);
    const int rank = (int)comp(k0, Lk.sh_it, Lk.kb[0]) - 1;
    const int64_t opb = list_beg[lg * 4 + 3];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t cells = (int64_t)nL * n_lg * R0;
    for (int t = tid; t < NF * nL; t += blockDim.x) {
        const int f = t / nL;
        pacc[t] = f == RF_FIRST_IDX || f == RF_FIRST_KS ? INT64_MAX : f == RF_LAST_KE ? INT64_MIN : 0;
    }
    for (int q = tid; q < nL; q += blockDim.x) lcnt[q] = 0;
    for (int64_t j0 = a; j0 < b; j0 += PT_CH) {
        const int m = (int)min((int64_t)PT_CH, b - j0);
        if (tid < m) {           // PT_CH == blockDim: thread t loads instance j0 + t, all loads in flight first
            const int64_t j = j0 + tid;
            int64_t x[RF_NFIELDS];
#pragma unroll
            for (int f = 0; f < RF_NFIELDS; f++) x[f] = __ldg(iv.f + (int64_t)f * iv.cap + j);
            int64_t y[8];
#pragma unroll
            for (int q = 0; q < 8; q++) y[q] = q < C ? __double_as_longlong(__ldg(iv.cnt + (int64_t)q * iv.ccap + j)) : 0;
#pragma unroll
            for (int f = 0; f < RF_NFIELDS; f++) vals[f * PT_CH + tid] = x[f];
#pragma unroll
            for (int q = 0; q < 8; q++) if (q < C) vals[(RF_NFIELDS + q) * PT_CH + tid] = y[q];
            for (int q = 8; q < C; q++)
                vals[(RF_NFIELDS + q) * PT_CH + tid] = __double_as_longlong(iv.cnt[(int64_t)q * iv.ccap + j]);
        }
        for (int q = tid; q < 8 * nL; q += blockDim.x) wc[q] = 0;
        int l = -1;
        if (tid < m) {
            const int64_t rop = comp(iv.key[j0 + tid], Lk.sh_op, Lk.kb[3]);
            l = rop > 0 ? P_label[opb + rop - 1] : -1;
            if (l >= nL) { atomicOr(ovf, 1u); l = -1; }
        }
        __syncthreads();
        const unsigned mm = __match_any_sync(CH_FULL, l);
        const int inrank = __popc(mm & lanemask_lt());
        if (l >= 0 && inrank == 0) wc[w * nL + l] = __popc(mm);
        __syncthreads();
        // per label: counts over warps (exclusive per warp) and the label's start in the chunk order
        int tot_l = 0;
        if (tid < nL) {
            for (int x = 0; x < 8; x++) { const int c = wc[x * nL + tid]; wc[x * nL + tid] = tot_l; tot_l += c; }
        }
        int64_t dummy;
        const int st = (int)block_excl_sum<256>(tid < nL ? tot_l : 0, &dummy, scan_sm);
        if (tid < nL) { lstart[tid] = st; ltot[tid] = tot_l; lcnt[tid] += tot_l; }
        __syncthreads();
        if (l >= 0) order[lstart[l] + wc[w * nL + l] + inrank] = tid;
        __syncthreads();
        for (int t = tid; t < NF * nL; t += blockDim.x) {
            const int f = t / nL, lb = t - f * nL;
            const int c0 = lstart[lb], c1 = c0 + ltot[lb];
            if (f == RF_FIRST_IDX || c0 == c1) continue;              // (FIRST_IDX folds with FIRST_KS)
            const int64_t *v = vals + f * PT_CH;
            if (f >= RF_NFIELDS) {
                double x = __longlong_as_double(pacc[t]);
                for (int k = c0; k < c1; k++) x += __longlong_as_double(v[order[k]]);
                pacc[t] = __double_as_longlong(x);
            } else if (f == RF_LAST_KE) {
                int64_t x = pacc[t];
                for (int k = c0; k < c1; k++) x = max(x, v[order[k]]);
                pacc[t] = x;
            } else if (f == RF_FIRST_KS) {
                const int64_t *vi = vals + RF_FIRST_IDX * PT_CH;
                int64_t ks = pacc[t], ix = pacc[RF_FIRST_IDX * nL + lb];
                for (int k = c0; k < c1; k++) {
                    const int o = order[k];
                    if (v[o] < ks || (v[o] == ks && vi[o] < ix)) { ks = v[o]; ix = vi[o]; }
                }
                pacc[t] = ks;
                pacc[RF_FIRST_IDX * nL + lb] = ix;
            } else {
                int64_t x = pacc[t];
                for (int k = c0; k < c1; k++) x += v[order[k]];
                pacc[t] = x;
            }
        }
        __syncthreads();
    }
    for (int t = tid; t < NF * nL; t += blockDim.x) {
        const int f = t / nL, lb = t - f * nL;
        if (lcnt[lb] == 0) continue;
        const int64_t cell = ((int64_t)lb * n_lg + lg) * R0 + rank;
        if (f < RF_NFIELDS) df[(int64_t)f * cells + cell] = pacc[t];
        else dc[(int64_t)(f - RF_NFIELDS) * cells + cell] = __longlong_as_double(pacc[t]);
        if (f == 0) dvalid[cell] = 1;
    }
}

// compaction of the dense point grid into the point table (cell order = point-key order)
__global__ void k_points_compact(const int64_t *__restrict__ dvalid, const int64_t *__restrict__ ex, int64_t cells,
                                 const int64_t *__restrict__ df, const double *__restrict__ dc, int C, int n_lg, int R0,
                                 int kg, int kb0, TabView pt) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells || !dvalid[c]) return;
    const int64_t p = ex[c];
    const int64_t label = c / ((int64_t)n_lg * R0), lg = (c / R0) % n_lg, rank = c % R0;
    pt.key[p] = ((unsigned long long)label << (kg + kb0)) | ((unsigned long long)lg << kb0) | (unsigned long long)(rank + 1);
#pragma unroll
    for (int f = 0; f < RF_NFIELDS; f++) pt.f[(int64_t)f * pt.cap + p] = df[(int64_t)f * cells + c];
    for (int s2 = 0; s2 < C; s2++) pt.cnt[(int64_t)s2 * pt.ccap + p] = dc[(int64_t)s2 * cells + c];
}

__global__ void k_decode_points(const unsigned long long *__restrict__ key, const int64_t *__restrict__ n_dev, int kg,
                                int kb0,
                                const int32_t *__restrict__ lg_gpu, const int64_t *__restrict__ list_beg,
                                const int32_t *__restrict__ P_orig, const int64_t *__restrict__ f, int64_t cap,
                                PredView pv, int32_t *gpu, int32_t *it, int32_t *ph,
                                int32_t *ly, int32_t *op, int32_t *label, int32_t *rank, int64_t *first_pred) {
    const int64_t n = *n_dev;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
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
    first_pred[j] = (fi != INT64_MAX) ? pred_of(pv, fi) : CH_NONE_TS;
    }
}

// iteration extras: wall (telescoping chain span), comm union inside the iteration, aligned bounds, step
__global__ void k_iter_extras(const int64_t *__restrict__ n_dev, const int64_t *__restrict__ f, int64_t cap,
                              const int32_t *__restrict__ gpu,
                              const int32_t *__restrict__ it, const int64_t *__restrict__ first_pred,
                              const int32_t *__restrict__ gpu_lg, const int32_t *__restrict__ span_label,
                              const int64_t *__restrict__ Us, const int64_t *__restrict__ Ue,
                              const int64_t *__restrict__ UP, const int64_t *__restrict__ Ubeg,
                              const int64_t *__restrict__ Ucnt, const int64_t *__restrict__ delta,
                              int64_t *__restrict__ wall, int64_t *__restrict__ cu, int64_t *__restrict__ af,
                              int64_t *__restrict__ al, int32_t *__restrict__ step) {
    const int64_t n = *n_dev;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
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
}

__global__ void k_rates(const int64_t *__restrict__ n_dev, const int64_t *__restrict__ f, const double *__restrict__ cnt,
                        int64_t cap,
                        int nr, const int32_t *__restrict__ rnum, const int32_t *__restrict__ rden,
                        const double *__restrict__ rsc, double *__restrict__ out) {
    const int64_t n = *n_dev;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        for (int q = 0; q < nr; q++) {
            double num = cnt[(int64_t)rnum[q] * cap + j];
            double den = rden[q] < 0 ? (double)f[(int64_t)RF_BUSY * cap + j] * 1e-9 : cnt[(int64_t)rden[q] * cap + j];
            out[(int64_t)q * cap + j] = num / den * rsc[q];
        }
    }
}
}  // namespace

// Dynamic shared memory above 48 KB needs an opt-in per kernel.  The sizes vary with the trace (and several host
// threads may drive contexts at once), so each such kernel is opted in once to the device maximum (minus its
// static shared memory): every caller sets the same value, and any size the launch asks for is allowed.
static cudaError_t allow_max_smem(const void *fn) {
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, fn);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
    return e;
}

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

// grid for device-counted loops: enough blocks to fill the gpu, never more than the upper bound needs
static unsigned grid_for(int64_t upper, int per_block) {
    int64_t g = ceil_div(std::max<int64_t>(upper, 1), per_block);
    return (unsigned)std::min<int64_t>(g, 148 * 16);
}

// group the sorted children (count *n_dev, upper bound n) by key >> shift: group starts and the group
// count stay on the device (no host round trip); starts[ng] = end of the last group (first invalid key)
static chopper_status group(chopper_ctx *ctx, const unsigned long long *keys_sorted, int64_t n, const int64_t *n_dev,
                            int shift, int64_t **starts_out, int64_t **ng_out, int all = 0) {
    CH_ALLOC_BEGIN;
    int64_t *starts = CH_ALLOC(ctx, int64_t, n + 2);
    int64_t *tot = CH_ALLOC(ctx, int64_t, 1);
    CH_ALLOC_END(ctx);
    const int64_t ntile = std::max<int64_t>(ceil_div(n, GP_TILE), 1);
    size_t mark = ctx->used;
    unsigned long long *state = CH_ALLOC(ctx, unsigned long long, ntile + 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemsetAsync(state, 0, 8 * (size_t)(ntile + 1), ctx->st));
    k_group_1pass<<<(unsigned)ntile, GP_NT, 0, ctx->st>>>(keys_sorted, n, n_dev, shift, all, starts, tot, state,
                                                         reinterpret_cast<unsigned int *>(state + ntile));
    CH_LAUNCHED(ctx);
    if (!ctx->hold_scratch) ctx->used = mark;
    *starts_out = starts;
    *ng_out = tot;
    return CHOPPER_OK;
}

static TabView view(RowTable &t) { return TabView{t.key, t.f, t.cnt, t.cap, t.cap, 1, 1}; }

// parents of the groups: mode 0 = children staged per block (many parents, few children each),
// 1 = a warp per parent (few parents, many children), 2 = a lane per parent
static chopper_status sum_rows(chopper_ctx *ctx, const TabView &ch, const uint32_t *perm, const int64_t *starts,
                               const int64_t *ng_dev, int64_t ng_upper, int mode, int shift, int C, const TabView &pa,
                               int fanout = 1) {
    if (ng_upper <= 0) return CHOPPER_OK;
    // parents per block for the staged kernel: ~RC_CH children per block from the expected fan-out
    const int PB = fanout <= 1 ? RC_NT : std::max(8, std::min(RC_NT, RC_CH / fanout));
    const size_t shb = (size_t)(RF_NFIELDS + C) * RC_CH * 8;
    if (mode == 0 && shb > 160 * 1024) mode = 2;
    if (mode == 1 && C > 32) mode = 2;
    if (mode == 0 && !perm && ch.rs == 1 && C <= 8 && fanout >= 2) {
        const size_t shc = (size_t)(RF_NFIELDS + C) * (RC_CH + PB) * 8;
        static bool opt_c = false;
        if (!opt_c) { CH_CUDA(ctx, allow_max_smem((const void *)k_sum_rows_cols)); opt_c = true; }
        k_sum_rows_cols<<<grid_for(ng_upper / fanout, PB), RC_NT, shc, ctx->st>>>(ch, starts, ng_dev, shift, C, pa, PB);
    } else if (mode == 0) {
        static bool opt = false;
        if (!opt) { CH_CUDA(ctx, allow_max_smem((const void *)k_sum_rows_chunked)); opt = true; }
        if (C > 8) CH_CUDA(ctx, cudaMemsetAsync(pa.cnt, 0, 8 * (size_t)C * pa.ccap, ctx->st));
        k_sum_rows_chunked<<<grid_for(ng_upper / std::max(fanout, 1), PB), RC_NT, shb, ctx->st>>>(ch, perm, starts, ng_dev,
                                                                                                 shift, C, pa, PB);
    } else if (mode == 1) {
        if (C == 0) k_sum_rows_warp<0><<<grid_for(ng_upper, NT / 32), NT, 0, ctx->st>>>(ch, perm, starts, ng_dev, shift, C, pa);
        else if (C <= 8) k_sum_rows_warp<8><<<grid_for(ng_upper, NT / 32), NT, 0, ctx->st>>>(ch, perm, starts, ng_dev, shift, C, pa);
        else k_sum_rows_warp<32><<<grid_for(ng_upper, NT / 32), NT, 0, ctx->st>>>(ch, perm, starts, ng_dev, shift, C, pa);
    } else {
        k_sum_rows<<<grid_for(ng_upper, NT), NT, 0, ctx->st>>>(ch, perm, starts, ng_dev, shift, C, pa);
    }
    CH_LAUNCHED(ctx);
    return CHOPPER_OK;
}

// parent rows beyond the table's capacity (a violated structural bound): clamp and latch CHOPPER_E_RANGE
__global__ void k_clamp_rows(int64_t *__restrict__ n_dev, int64_t cap, DevReport *__restrict__ rep) {
    if (threadIdx.x == 0 && *n_dev > cap) {
        *n_dev = cap;
        latch(rep, CHOPPER_E_RANGE);
    }
}

// rows of the parent level (depth 3 layer, 2 phase, 1 iteration, 0 gpu): an instance key's (it, ph, ly) prefix
// is a step function of the dispatch time with steps only at the gpu's iteration / phase / layer span
// endpoints, so a gpu has at most 1 + 2 * (its spans of the levels above) distinct prefixes
static int64_t parent_bound(chopper_ctx *ctx, int depth) {
    int64_t s = 0;
    for (int l = 0; l < ctx->n_lg * 4; l++)
        if (l % 4 < depth) s += ctx->list_beg[l + 1] - ctx->list_beg[l];
    return 2 * s + ctx->n_lg;
}

static chopper_status rollup(chopper_ctx *ctx, RowTable &child, RowTable &parent, int shift, int depth, int mode,
                             const KeyLayout &L, int32_t *lg_gpu_d, int fanout = 1) {
    int64_t *starts, *ng_dev;
    CH_TRY(group(ctx, child.key, child.cap, child.n_dev, shift, &starts, &ng_dev));
    CH_TRY(alloc_table(ctx, parent, std::max<int64_t>(std::min(child.cap, parent_bound(ctx, depth)), 1), ctx->C, true));
    k_clamp_rows<<<1, 32, 0, ctx->st>>>(ng_dev, parent.cap, ctx->d_rep);
    CH_LAUNCHED(ctx);
    parent.n_dev = ng_dev;
    CH_TRY(sum_rows(ctx, view(child), nullptr, starts, ng_dev, child.cap, mode, shift, ctx->C, view(parent), fanout));
    k_decode<<<grid_for(child.cap, NT), NT, 0, ctx->st>>>(parent.key, ng_dev, L, depth, lg_gpu_d, ctx->d_list_beg,
                                                          ctx->P_orig, ctx->P_label, parent.f, parent.cap,
                                                          PredView{ctx->d_pred_end, ctx->ev.meta, ctx->ev.end_ns}, parent.gpu, parent.it, parent.ph, parent.ly,
                                                          parent.op, parent.label, parent.rank, parent.first_pred);
    CH_LAUNCHED(ctx);
    return CHOPPER_OK;
}

static void key_layout(chopper_ctx *ctx, KeyLayout &L) {
    L.kb[0] = ctx->kb[0]; L.kb[1] = ctx->kb[1]; L.kb[2] = ctx->kb[2]; L.kb[3] = ctx->kb[3];
    L.sh_op = 0;
    L.sh_ly = L.kb[3];
    L.sh_ph = L.sh_ly + L.kb[2];
    L.sh_it = L.sh_ph + L.kb[1];
    L.sh_lg = L.sh_it + L.kb[0];
}

// all table stages, enqueued without host round trips except the rare radix-sort fallback check

// development aid (CHOPPER_DBG_TICKS=1): device timestamps of the tables stages, printed after the stage's sync
namespace {
struct DbgTicks {
    bool on = getenv("CHOPPER_DBG_TICKS") != nullptr;
    cudaEvent_t ev[32] = {};
    const char *lab[32] = {};
    int n = 0;
    void mark(cudaStream_t st, const char *l) {
        if (!on || n >= 32) return;
        if (!ev[n]) cudaEventCreate(&ev[n]);
        cudaEventRecord(ev[n], st);
        lab[n++] = l;
    }
    void dump() {
        if (!on || n < 2) { n = 0; return; }
        fprintf(stderr, "[tables]");
        for (int i = 1; i < n; i++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, " %s %.3f", lab[i], ms);
        }
        fprintf(stderr, "\n");
        n = 0;
    }
};
DbgTicks g_dbg;
}
// The counter pass (R8 finiteness of every value it reads included) on side[0], joined (join_ev[0]) before the
// sub-run -> instance sum.  t_rank = 1: the per-thread run values are in-tile head ranks from k_tile_heads, so
// the pass can start beside the event pass (ch_event_pass); 0: global run ids written by the event pass.
chopper_status ch_counters_launch(chopper_ctx *ctx, double *cnt, unsigned int *colbad, int t_rank) {
    const int C = ctx->C, n_lg = ctx->n_lg;
    ctx->d_colbad = colbad;                   // [n_lg][C] non-finite flags, read with the tables' row counts
    CH_CUDA(ctx, cudaMemsetAsync(ctx->d_colbad, 0, 4 * (size_t)n_lg * C, ctx->st));
    const int vec_ok = (((uintptr_t)ctx->ev.meta) & 15u) == 0;
    CH_CUDA(ctx, cudaFuncSetAttribute(k_counters_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CtSmem)));
    CH_CUDA(ctx, cudaEventRecord(ctx->fork_ev, ctx->st));
    CH_CUDA(ctx, cudaStreamWaitEvent(ctx->side[0], ctx->fork_ev, 0));
    ch_tick_on(ctx, 9, 0, ctx->side[0]);
    k_counters_tiled<<<(unsigned)ceil_div(ctx->N, CT_TILE), CT_NT, sizeof(CtSmem), ctx->side[0]>>>(
        ctx->ev.meta, ctx->d_t_run, ctx->d_t_hm, ctx->d_t_nm, ctx->d_nm_base, ctx->d_tile_sub, ctx->d_gpu_lg,
        ctx->d_col, C, ctx->N, cnt, 1, ctx->d_colbad, vec_ok, n_lg, t_rank);
    CH_LAUNCHED(ctx);
    ch_tick_on(ctx, 9, 1, ctx->side[0]);
    CH_CUDA(ctx, cudaEventRecord(ctx->join_ev[0], ctx->side[0]));
    return CHOPPER_OK;
}

static chopper_status tables_body(chopper_ctx *ctx, unsigned int **ovf_out) {
    const int C = ctx->C;
    const int64_t R = ctx->R;
    KeyLayout L;
    key_layout(ctx, L);
    const int key_bits = L.sh_lg + ctx->kg;
    g_dbg.mark(ctx->st, "begin");
    CH_ALLOC_BEGIN;
    int32_t *lg_gpu_d = CH_ALLOC(ctx, int32_t, ctx->n_lg + 1);
    CH_ALLOC_END(ctx);
    ctx->h_lg_gpu.assign(ctx->lg_gpu, ctx->lg_gpu + ctx->n_lg);
    if (ctx->n_lg)
        CH_CUDA(ctx, cudaMemcpyAsync(lg_gpu_d, ctx->h_lg_gpu.data(), 4 * ctx->n_lg, cudaMemcpyHostToDevice, ctx->st));
    ctx->sub.cap = std::max<int64_t>(R, 1);
    // the counter pass may already run beside the event pass (ch_counters_launch from ch_event_pass)
    bool counters_forked = ctx->counters_early;
    if (!counters_forked) {
        CH_ALLOC_BEGIN;
        ctx->sub.cnt = CH_ALLOC(ctx, double, (int64_t)(C > 0 ? C : 1) * std::max<int64_t>(R, 1));
        unsigned int *colbad = CH_ALLOC(ctx, unsigned int, (int64_t)ctx->n_lg * std::max(C, 1));
        CH_ALLOC_END(ctx);
        if (C > 0 && R > 0) {
            CH_TRY(ch_counters_launch(ctx, ctx->sub.cnt, colbad, ctx->t_run_rank ? 1 : 0));
            counters_forked = true;
        }
    }
    ctx->counters_early = false;              // (a redo of the tables forks its own pass)
    TabView subv{ctx->sub.key, ctx->sub.f, ctx->sub.cnt, 1, 1, 16, std::max(C, 1)};   // AoS sub-run rows and counters
    g_dbg.mark(ctx->st, "fork");
    // instances: sort of sub-runs by key, then groups of equal keys
    unsigned long long *k1 = CH_ALLOC(ctx, unsigned long long, R + 1), *k2 = CH_ALLOC(ctx, unsigned long long, R + 1);
    uint32_t *v1 = CH_ALLOC(ctx, uint32_t, R + 1), *v2 = CH_ALLOC(ctx, uint32_t, R + 1);
    CH_ALLOC_END(ctx);
    if (R > 0) {
        k_copy_keys<<<(unsigned)ceil_div(R, NT), NT, 0, ctx->st>>>(ctx->sub.key, R, k1, v1);
        CH_LAUNCHED(ctx);
    }
    bool alt = false;
    {
        // segmented sort inside (gpu, iteration) prefixes; radix sort if the prefixes are not in order
        // The check that the (gpu, iteration) prefixes come in order (and that no segment exceeds SS_MAX) is not
        // waited for: its flag is read with the row counts at the end of the stage, and a failed check redoes the
        // tables with the radix sort (ch_tables), which this ctx then uses from the start (tables_radix)
        bool done = false;
        ctx->d_prefix_bad = nullptr;
        if (R > 1 && !ctx->tables_radix) {
            unsigned int *bad = CH_ALLOC(ctx, unsigned int, 1);
            CH_ALLOC_END(ctx);
            ctx->d_prefix_bad = bad;
            size_t mk = ctx->used;
            int64_t *nv_d = CH_ALLOC(ctx, int64_t, 1);
            CH_ALLOC_END(ctx);
            int64_t *st = nullptr, *nseg_d = nullptr;
            CH_TRY(group(ctx, k1, R, nullptr, L.sh_it, &st, &nseg_d, 1));   // segments: equal (gpu, iteration)
            CH_CUDA(ctx, cudaMemsetAsync(bad, 0, 4, ctx->st));
            k_prefix_check<<<grid_for(R, NT), NT, 0, ctx->st>>>(k1, st, nseg_d, L.sh_it, bad);
            CH_LAUNCHED(ctx);
            {
    g_dbg.mark(ctx->st, "prefsync");
                static bool ss_attr = false;
                if (!ss_attr) {
                    CH_CUDA(ctx, cudaFuncSetAttribute(k_seg_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)sizeof(SegSortSmem)));
                    ss_attr = true;
                }
                k_seg_sort<<<grid_for(R, 1), SS_NT, sizeof(SegSortSmem), ctx->st>>>(k1, v1, st, nseg_d, L);
                CH_LAUNCHED(ctx);
                {
                    const int64_t nt = ceil_div(R, GP_TILE);
                    size_t m2 = ctx->used;
                    unsigned long long *state = CH_ALLOC(ctx, unsigned long long, nt + 1);
                    CH_ALLOC_END(ctx);
                    CH_CUDA(ctx, cudaMemsetAsync(state, 0, 8 * (size_t)(nt + 1), ctx->st));
                    k_compact_1pass<<<(unsigned)nt, GP_NT, 0, ctx->st>>>(k1, v1, R, k2, v2, nv_d, state,
                                                                        reinterpret_cast<unsigned int *>(state + nt));
                    CH_LAUNCHED(ctx);
                    ctx->used = m2;
                }
                alt = true;
                done = true;
            }
            ctx->used = mk;
        }
        if (!done) CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, R, 0, key_bits, &alt));
    }
    g_dbg.mark(ctx->st, "ordered");
    unsigned long long *ks = alt ? k2 : k1;
    uint32_t *so = alt ? v2 : v1;
    {
        int64_t *starts, *ng_dev;
        CH_TRY(group(ctx, ks, R, nullptr, 0, &starts, &ng_dev));
        CH_TRY(alloc_table(ctx, ctx->inst, std::max<int64_t>(R, 1), C, true));
        if (counters_forked) CH_CUDA(ctx, cudaStreamWaitEvent(ctx->st, ctx->join_ev[0], 0));
    g_dbg.mark(ctx->st, "join");
        ctx->inst.n_dev = ng_dev;
        if (R > 0) {
            CH_TRY(sum_rows(ctx, subv, so, starts, ng_dev, R, 0, 0, C, view(ctx->inst)));
            k_decode<<<grid_for(R, NT), NT, 0, ctx->st>>>(
                ctx->inst.key, ng_dev, L, 4, lg_gpu_d, ctx->d_list_beg, ctx->P_orig, ctx->P_label, ctx->inst.f,
                ctx->inst.cap, PredView{ctx->d_pred_end, ctx->ev.meta, ctx->ev.end_ns}, ctx->inst.gpu, ctx->inst.it, ctx->inst.ph, ctx->inst.ly, ctx->inst.op,
                ctx->inst.label, ctx->inst.rank, ctx->inst.first_pred);
            CH_LAUNCHED(ctx);
        }
    }
    // points (label, gpu, iteration): per-iteration label folds into a dense grid, then compaction.  Issued
    // first, on a side stream (it only reads the instance table), so that it runs concurrently with the
    // roll-ups below; scratch is not released inside the branch (the roll-ups allocate after it)
    CH_CUDA(ctx, cudaEventRecord(ctx->fork_ev, ctx->st));
    CH_CUDA(ctx, cudaStreamWaitEvent(ctx->side[1], ctx->fork_ev, 0));
    cudaStream_t main_st = ctx->st;
    ctx->st = ctx->side[1];
    ctx->hold_scratch = true;
    chopper_status pst = [&]() -> chopper_status {
        {
            const int64_t n = ctx->inst.cap;
            const int nL = std::max(ctx->cfg.n_labels, 1), n_lg = std::max(ctx->n_lg, 1);
            const int R0 = (int)std::max<int64_t>(ctx->max_it_list, 1);
            const int64_t cells = (int64_t)nL * n_lg * R0;
            int lbits = bits_for((uint64_t)std::max(ctx->cfg.n_labels, 1));
            int pbits = lbits + ctx->kg + L.kb[0];
            if (pbits > 63) return ch_fail(ctx, CHOPPER_E_RANGE, "point key exceeds 63 bits");
            if (nL > 256) return ch_fail(ctx, CHOPPER_E_RANGE, "more than 256 op labels");
            int64_t *its = nullptr, *n_it = nullptr;
            CH_TRY(group(ctx, ctx->inst.key, n, ctx->inst.n_dev, L.sh_it, &its, &n_it));
            int64_t *df = CH_ALLOC(ctx, int64_t, (int64_t)RF_NFIELDS * cells);
            double *dc = CH_ALLOC(ctx, double, (int64_t)std::max(C, 1) * cells);
            int64_t *dvalid = CH_ALLOC(ctx, int64_t, cells), *dex = CH_ALLOC(ctx, int64_t, cells), *np_d = CH_ALLOC(ctx, int64_t, 1);
            unsigned int *ovf = CH_ALLOC(ctx, unsigned int, 1);
            CH_ALLOC_END(ctx);
            *ovf_out = ovf;
            CH_CUDA(ctx, cudaMemsetAsync(dvalid, 0, 8 * (size_t)cells, ctx->st));
            CH_CUDA(ctx, cudaMemsetAsync(ovf, 0, 4, ctx->st));
            size_t shb = (size_t)(RF_NFIELDS + C) * (PT_CH + nL) * 8 + 4 * (2 * PT_CH + 11 * (size_t)nL);
            static bool opt_p = false;
            if (!opt_p) { CH_CUDA(ctx, allow_max_smem((const void *)k_points_iter)); opt_p = true; }
            k_points_iter<<<grid_for(std::min<int64_t>(n, (int64_t)n_lg * R0), 1), 256, shb, ctx->st>>>(
                view(ctx->inst), its, n_it, L, ctx->d_list_beg, ctx->P_label, nL, n_lg, R0, C, df, dc, dvalid, ovf);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_scan_excl_i64(ctx, dvalid, dex, cells, np_d));
            CH_TRY(alloc_table(ctx, ctx->point, std::max<int64_t>(cells, 1), C, true));
            ctx->point.n_dev = np_d;
            k_points_compact<<<(unsigned)ceil_div(cells, NT), NT, 0, ctx->st>>>(dvalid, dex, cells, df, dc, C, n_lg, R0,
                                                                              ctx->kg, L.kb[0], view(ctx->point));
            CH_LAUNCHED(ctx);
            k_decode_points<<<grid_for(cells, NT), NT, 0, ctx->st>>>(
                ctx->point.key, np_d, ctx->kg, L.kb[0], lg_gpu_d, ctx->d_list_beg, ctx->P_orig, ctx->point.f,
                ctx->point.cap, PredView{ctx->d_pred_end, ctx->ev.meta, ctx->ev.end_ns}, ctx->point.gpu, ctx->point.it, ctx->point.ph, ctx->point.ly,
                ctx->point.op, ctx->point.label, ctx->point.rank, ctx->point.first_pred);
            CH_LAUNCHED(ctx);
        }
        return CHOPPER_OK;
    }();
    ctx->hold_scratch = false;
    CH_CUDA(ctx, cudaEventRecord(ctx->join_ev[1], ctx->st));
    ctx->st = main_st;
    CH_TRY(pst);
    g_dbg.mark(ctx->st, "instdone");
    // roll-ups (D12): instance -> layer (staged), -> phase, -> iteration, -> gpu (warp per parent)
    // instances per layer: ~ instances / layer spans of the local gpus (fan-out hint for the staging width)
    const int64_t n_layers = std::max<int64_t>(ctx->n_layer_spans, 1);
    const int64_t fan = ctx->R / n_layers;
    const int fan_ly = (int)std::max<int64_t>(1, std::min<int64_t>(64, fan));
    // thousands of instances per layer (deep op trees, config 5): a warp per layer; else the staged fold
    CH_TRY(rollup(ctx, ctx->inst, ctx->layer, L.sh_ly, 3, fan > 256 ? 1 : 0, L, lg_gpu_d, fan_ly));
    g_dbg.mark(ctx->st, "layer");
    CH_TRY(rollup(ctx, ctx->layer, ctx->phase, L.sh_ph, 2, 1, L, lg_gpu_d));
    CH_TRY(rollup(ctx, ctx->phase, ctx->iter, L.sh_it, 1, 1, L, lg_gpu_d));
    CH_TRY(rollup(ctx, ctx->iter, ctx->gpurow, L.sh_lg, 0, 1, L, lg_gpu_d));
    g_dbg.mark(ctx->st, "rollups");
    // iteration extras
    {
        const int64_t cap = std::max<int64_t>(ctx->iter.cap, 1);
        ctx->iter_wall = CH_ALLOC(ctx, int64_t, cap);
        ctx->iter_cu = CH_ALLOC(ctx, int64_t, cap);
        ctx->iter_af = CH_ALLOC(ctx, int64_t, cap);
        ctx->iter_al = CH_ALLOC(ctx, int64_t, cap);
        ctx->iter_step = CH_ALLOC(ctx, int32_t, cap);
        CH_ALLOC_END(ctx);
        k_iter_extras<<<grid_for(cap, NT), NT, 0, ctx->st>>>(
            ctx->iter.n_dev, ctx->iter.f, ctx->iter.cap, ctx->iter.gpu, ctx->iter.it, ctx->iter.first_pred, ctx->d_gpu_lg,
            ctx->sp.label, ctx->U_s, ctx->U_e, ctx->U_P, ctx->d_U_beg, ctx->d_U_cnt, ctx->d_delta, ctx->iter_wall,
            ctx->iter_cu, ctx->iter_af, ctx->iter_al, ctx->iter_step);
        CH_LAUNCHED(ctx);
    }
    CH_CUDA(ctx, cudaStreamWaitEvent(ctx->st, ctx->join_ev[1], 0));
    g_dbg.mark(ctx->st, "pointsjoin");
    // derived ratio-of-sums rates
    if (ctx->n_ratios > 0) {
        RowTable *ts[2] = {&ctx->point, &ctx->iter};
        for (RowTable *t : ts) {
            t->rates = CH_ALLOC(ctx, double, (int64_t)ctx->n_ratios * std::max<int64_t>(t->cap, 1));
            CH_ALLOC_END(ctx);
            k_rates<<<grid_for(t->cap, NT), NT, 0, ctx->st>>>(t->n_dev, t->f, t->cnt, t->cap, ctx->n_ratios, ctx->d_ratio,
                                                              ctx->d_ratio + ctx->n_ratios, ctx->d_ratio_scale, t->rates);
            CH_LAUNCHED(ctx);
        }
    }
    // derived-metric registry
    CH_TRY(ch_eval_metrics(ctx, ctx->point));
    CH_TRY(ch_eval_metrics(ctx, ctx->iter));
    g_dbg.mark(ctx->st, "metrics");
    return CHOPPER_OK;
}

chopper_status ch_tables(chopper_ctx *ctx) {
    const int C = ctx->C;
    const int n_lg = ctx->n_lg;
    const int n_passes = (int)ctx->passes.size();
    const size_t mark = ctx->used;
    for (int round = 0; round < 2; round++) {
        ctx->used = mark;
        unsigned int *ovf = nullptr;
        CH_TRY(tables_body(ctx, &ovf));
        // one read-back for every stage: row counts, the point-label overflow, and the finiteness of the
        // counter columns that fed slots (R8; the others were checked by k_pass_finite in ch_align)
        RowTable *tabs[6] = {&ctx->inst, &ctx->layer, &ctx->phase, &ctx->iter, &ctx->gpurow, &ctx->point};
        int64_t hn[6] = {0, 0, 0, 0, 0, 0};
        for (int q = 0; q < 6; q++)
            if (tabs[q]->n_dev) CH_CUDA(ctx, ch_d2h(ctx, &hn[q], tabs[q]->n_dev, 8));
        unsigned int hovf = 0, hbad = 0;
        if (ovf) CH_CUDA(ctx, ch_d2h(ctx, &hovf, ovf, 4));
        if (ctx->d_prefix_bad) CH_CUDA(ctx, ch_d2h(ctx, &hbad, ctx->d_prefix_bad, 4));   // deferred order check
        std::vector<unsigned int> cb((size_t)std::max(n_lg * C, 1), 0), pb(std::max(n_passes, 1), 0);
        if (C > 0 && ctx->R > 0)
            CH_CUDA(ctx, ch_d2h(ctx, cb.data(), ctx->d_colbad, 4 * (size_t)n_lg * C));
        if (n_passes > 0)
            CH_CUDA(ctx, ch_d2h(ctx, pb.data(), ctx->d_pass_bad, 4 * n_passes));
        g_dbg.mark(ctx->st, "readback");
        CH_CUDA(ctx, ch_sync(ctx));
        g_dbg.dump();
        for (int q = 0; q < 6; q++) tabs[q]->n = hn[q];
        if (hbad) {
            // instance prefixes out of order (or a segment over SS_MAX): the segmented order was not valid; redo
            // the stage with the radix sort (this ctx keeps it)
            ctx->tables_radix = true;
            round--;
            continue;
        }
        if (hovf) return ch_fail(ctx, CHOPPER_E_RANGE, "op span label >= n_labels");
        bool changed = false;
        for (int p = 0; p < n_passes; p++) {
            if (ctx->pass_mismatch[p] >= 0 || ctx->pass_bad[p]) continue;
            bool bad = pb[p] != 0;
            for (size_t q = 0; q < (size_t)n_lg * C; q++)
                if (cb[q] && ctx->sel_pass[q] == p) bad = true;
            if (bad) { ctx->pass_bad[p] = 1; changed = true; }
        }
        if (round == 0) {
            for (int p = 0; p < n_passes; p++)
                if (ctx->pass_bad[p]) {
                    ctx->rep.val_count[CV_COUNTER_NONFINITE]++;
                    if (ctx->rep.val_first[CV_COUNTER_NONFINITE] < 0 || p < ctx->rep.val_first[CV_COUNTER_NONFINITE])
                        ctx->rep.val_first[CV_COUNTER_NONFINITE] = p;
                    ctx->latched_host |= 1u << CHOPPER_E_VALIDATION;
                }
        }
        if (!changed) break;
        // a slot column was non-finite: the pass is skipped and the next valid pass provides the slot
        // (every name-matching pass's finiteness is now known, so one redo of the tables settles it)
        CH_TRY(ch_assign_slots(ctx));
        CH_TRY(ch_counters_full(ctx));
    }
    return CHOPPER_OK;
}
