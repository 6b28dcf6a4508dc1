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

// counter sums of each sub-run over its COMPUTE events, CT_SG slots per launch.  A block stages its
// 2048-event tile in shared memory with cp.async -- meta, sub-run ids, pass positions, and for each slot
// the tile's contiguous range of the counter column (events of one gpu take consecutive pass positions,
// D2) -- so every global read is a bulk asynchronous copy.  Lane = event: warp w walks events
// [256w, 256w + 256) 32 at a time; sums within a warp come from a segmented warp scan keyed by the
// sub-run id, and a run still open at the end of a warp is finished by thread 0 from the per-warp edge
// pieces (sub-runs never cross tiles).  Every value read -- the slot's column at every non-MEMOP event,
// i.e. the whole column -- is checked for finiteness (R8), so a counter pass is read once.
constexpr int CT_NT = 256, CT_TILE = 2048, CT_SG = 4, CT_WARPS = CT_NT / 32, CT_WEV = CT_TILE / CT_WARPS;
struct CtSmem {
    uint32_t meta[CT_TILE];
    int32_t rid[CT_TILE];
    int32_t nm[CT_TILE];
    double val[CT_SG][CT_TILE];
    double lead[CT_WARPS][CT_SG], tail[CT_WARPS][CT_SG];
    int32_t tail_id[CT_WARPS], has[CT_WARPS];
};
__device__ __forceinline__ void ct_cp16(void *smem, const void *g) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void ct_cp8(void *smem, const void *g) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g));
}
__global__ void __launch_bounds__(CT_NT, 2) k_counters_tiled(const uint32_t *__restrict__ meta,
                                                             const int32_t *__restrict__ run_id,
                                                             const int32_t *__restrict__ nm_rank,
                                                             const int32_t *__restrict__ gpu_lg,
                                                             const double *const *__restrict__ col, int C, int s0,
                                                             int64_t N, double *__restrict__ out, int64_t cap,
                                                             unsigned int *__restrict__ colbad,
                                                             const int64_t *__restrict__ mg, int vec_ok) {
    extern __shared__ __align__(16) unsigned char ct_dsm[];
    CtSmem &S = *reinterpret_cast<CtSmem *>(ct_dsm);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * CT_TILE;
    const int nt = (int)min((int64_t)CT_TILE, N - base);
    const int ns = min(CT_SG, C - s0);
    // ---- stage the tile ----
    if (vec_ok && nt == CT_TILE) {
        for (int u = tid; u < CT_TILE / 4; u += CT_NT) {
            ct_cp16(&S.meta[4 * u], meta + base + 4 * u);
            ct_cp16(&S.rid[4 * u], run_id + base + 4 * u);
            ct_cp16(&S.nm[4 * u], nm_rank + base + 4 * u);
        }
    } else {
        for (int e = tid; e < CT_TILE; e += CT_NT) {
            const bool ok = e < nt;
            S.meta[e] = ok ? meta[base + e] : (uint32_t)CK_MEMOP;
            S.rid[e] = ok ? run_id[base + e] : -2;
            S.nm[e] = ok ? nm_rank[base + e] : 0;
        }
    }
    // one gpu in the tile (events are grouped by gpu): its pass positions form one contiguous range
    const int lg_a = gpu_lg[gpu_of(meta[base])], lg_b = gpu_lg[gpu_of(meta[base + nt - 1])];
    const bool single = lg_a == lg_b;
    int64_t nm_lo = 0;
    int cnt = 0;
    if (single) {
        nm_lo = nm_rank[base];
        cnt = (int)min((int64_t)CT_TILE, mg[lg_a] - nm_lo);
        for (int q = 0; q < ns; q++) {
            const double *c = col[lg_a * C + s0 + q];
            if (!c) continue;
            for (int k = tid; k < cnt; k += CT_NT) ct_cp8(&S.val[q][k], c + nm_lo + k);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if (lane < CT_SG) { S.lead[w][lane] = 0.0; }
    __syncthreads();
    // ---- per warp: 8 batches of 32 events ----
    const int e0 = w * CT_WEV;
    const int nv_w = max(0, min(CT_WEV, nt - e0));
    double carry[CT_SG];
#pragma unroll
    for (int q = 0; q < CT_SG; q++) carry[q] = 0.0;
    bool open = e0 > 0 && nv_w > 0, open_here = false, seen_head = false;
    int32_t open_id = (e0 > 0 && nv_w > 0) ? S.rid[e0 - 1] : -1;
    for (int b = 0; b < CT_WEV / 32; b++) {
        const int e = e0 + b * 32 + lane;
        const bool valid = b * 32 + lane < nv_w;
        const unsigned vm = __ballot_sync(CH_FULL, valid);
        if (vm == 0) break;
        const uint32_t m = S.meta[e];
        const int32_t rid = valid ? S.rid[e] : -2;
        const int32_t nm = S.nm[e];
        const bool head = valid && (e == 0 || rid != S.rid[e - 1]);
        const int kd = kind_of(m);
        const bool rd = valid && kd != CK_MEMOP;
        double v[CT_SG];
        const int lg = rd ? gpu_lg[gpu_of(m)] : -1;
#pragma unroll
        for (int q = 0; q < CT_SG; q++) {
            v[q] = 0.0;
            if (q < ns && rd) {
                const double *c = col[lg * C + s0 + q];
                if (c) {
                    const double x = (single && nm - nm_lo < cnt) ? S.val[q][nm - nm_lo] : __ldg(c + nm);
                    if (!isfinite(x)) atomicOr(&colbad[lg * C + s0 + q], 1u);
                    if (kd == CK_COMPUTE) v[q] = x;
                }
            }
        }
        const unsigned hm = __ballot_sync(CH_FULL, head);
        bool f = head;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const bool pf = __shfl_up_sync(CH_FULL, f, o);
#pragma unroll
            for (int q = 0; q < CT_SG; q++) {
                const double pv = __shfl_up_sync(CH_FULL, v[q], o);
                if (lane >= o && !f) v[q] = pv + v[q];
            }
            if (lane >= o) f = f || pf;
        }
        const int last_valid = 31 - __clz(vm);
        const int first_head = hm ? __ffs(hm) - 1 : 32;
        if (lane < first_head) {
#pragma unroll
            for (int q = 0; q < CT_SG; q++) v[q] = carry[q] + v[q];
        }
        // 1) the open run ends before first_head (or at the last valid event)
        if (open && (first_head < 32 || last_valid < 31)) {
            const int endl = min(first_head, last_valid + 1) - 1;
            if (lane == (endl >= 0 ? endl : 0)) {
                for (int q = 0; q < ns; q++) {
                    const double t = endl >= 0 ? v[q] : carry[q];
                    if (open_here) out[(int64_t)(s0 + q) * cap + open_id] = t;
                    else S.lead[w][q] = t;
                }
            }
            open = false;
        }
        // 2) runs starting in this batch that end inside it
        const bool nxt_head = lane < 31 && ((hm >> (lane + 1)) & 1u);
        if (valid && lane >= first_head && (nxt_head || (lane == last_valid && last_valid < 31)))
            for (int q = 0; q < ns; q++) out[(int64_t)(s0 + q) * cap + rid] = v[q];
        // 3) the run open at lane 31
        if (last_valid == 31) {
            if (hm) { open_here = true; open_id = __shfl_sync(CH_FULL, rid, 31); }
#pragma unroll
            for (int q = 0; q < CT_SG; q++) carry[q] = __shfl_sync(CH_FULL, v[q], 31);
            open = true;
        }
        seen_head = seen_head || hm != 0;
        if (last_valid < 31) break;
    }
    if (lane == 0) {
        S.has[w] = seen_head;
        S.tail_id[w] = open ? open_id : -1;
#pragma unroll
        for (int q = 0; q < CT_SG; q++) S.tail[w][q] = open ? carry[q] : 0.0;
    }
    __syncthreads();
    if (tid == 0) {
        for (int wa = 0; wa < CT_WARPS; wa++) {
            if (S.tail_id[wa] < 0 || !S.has[wa]) continue;
            const int32_t id = S.tail_id[wa];
            double acc[CT_SG];
            for (int q = 0; q < ns; q++) acc[q] = S.tail[wa][q];
            for (int wb = wa + 1; wb < CT_WARPS; wb++) {
                if (S.has[wb] || S.tail_id[wb] != id) {
                    for (int q = 0; q < ns; q++) acc[q] += S.lead[wb][q];
                    break;
                }
                for (int q = 0; q < ns; q++) acc[q] += S.tail[wb][q];
            }
            for (int q = 0; q < ns; q++) out[(int64_t)(s0 + q) * cap + id] = acc[q];
        }
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
__global__ void k_prefix_check(const unsigned long long *__restrict__ key, const int64_t *__restrict__ starts,
                               int64_t nseg, int sh, unsigned int *__restrict__ bad) {
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
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
    int cbeg[5];
    int unsorted;
    int64_t scan[33];
};
__device__ __forceinline__ int seg_class(unsigned long long k, const KeyLayout &L) {
    if (k == CH_INVALID_KEY) return 3;
    if (comp(k, L.sh_op, L.kb[3]) > 0) return 0;
    if (comp(k, L.sh_ly, L.kb[2]) > 0) return 1;
    if (comp(k, L.sh_ph, L.kb[1]) > 0) return 2;
    return 3;
}
__global__ void __launch_bounds__(SS_NT) k_seg_sort(unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals,
                                                    const int64_t *__restrict__ starts, int64_t nseg, KeyLayout L) {
    extern __shared__ __align__(16) unsigned char ss_dsm[];
    SegSortSmem &S = *reinterpret_cast<SegSortSmem *>(ss_dsm);
    const int64_t lo = starts[blockIdx.x], hi = starts[blockIdx.x + 1];
    const int n = (int)(hi - lo);
    if (n <= 1 || n > SS_MAX) return;
    bool sorted = true;   // fast exit for an already ordered segment
    for (int i = threadIdx.x + 1; i < n; i += blockDim.x)
        if (keys[lo + i] < keys[lo + i - 1]) sorted = false;
    if (__syncthreads_and(sorted)) return;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { S.k[i] = keys[lo + i]; S.v[i] = vals[lo + i]; }
    if (threadIdx.x == 0) { S.unsorted = 0; S.cbeg[0] = 0; }
    __syncthreads();
    // stable partition by class: per-thread chunk counts, one packed block scan (4 x 16-bit counters)
    const int per = (n + SS_NT - 1) / SS_NT;
    const int i0 = threadIdx.x * per, i1 = min(n, i0 + per);
    unsigned long long cnt = 0;
    for (int i = i0; i < i1; i++) cnt += 1ull << (16 * seg_class(S.k[i], L));
    int64_t tot;
    unsigned long long ex = (unsigned long long)block_excl_sum<SS_NT>((int64_t)cnt, &tot, S.scan);
    const unsigned long long t64 = (unsigned long long)tot;
    int cb[4];
    cb[0] = 0;
    cb[1] = (int)(t64 & 0xFFFF);
    cb[2] = cb[1] + (int)((t64 >> 16) & 0xFFFF);
    cb[3] = cb[2] + (int)((t64 >> 32) & 0xFFFF);
    if (threadIdx.x == 0) { S.cbeg[1] = cb[1]; S.cbeg[2] = cb[2]; S.cbeg[3] = cb[3]; S.cbeg[4] = n; }
    int pos[4];
#pragma unroll
    for (int c = 0; c < 4; c++) pos[c] = cb[c] + (int)((ex >> (16 * c)) & 0xFFFF);
    for (int i = i0; i < i1; i++) {
        const int c = seg_class(S.k[i], L);
        const int d = pos[c]++;
        S.ck[d] = S.k[i];
        S.cv[d] = S.v[i];
    }
    __syncthreads();
    // every class ascending?
    for (int c = 0; c < 4; c++)
        for (int d = S.cbeg[c] + 1 + threadIdx.x; d < S.cbeg[c + 1]; d += blockDim.x)
            if (S.ck[d] < S.ck[d - 1]) S.unsorted = 1;
    __syncthreads();
    if (!S.unsorted) {
        for (int d = threadIdx.x; d < n; d += blockDim.x) {
            int c = 0;
            while (d >= S.cbeg[c + 1]) c++;
            const unsigned long long x = S.ck[d];
            int p = d - S.cbeg[c];
            for (int o = 0; o < 4; o++) {
                if (o == c) continue;
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

__global__ void __launch_bounds__(256) k_sum_rows(TabView ch, const uint32_t *__restrict__ perm,
                                                  const int64_t *__restrict__ starts, int64_t ng, int shift, int C,
                                                  TabView pa) {
    const int lane = lane_id();
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
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
            for (int64_t j = lo; j < hi; j++) acc += ch.cnt[(int64_t)s * ch.ccap + (perm ? (int64_t)perm[j] : j)];
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
            for (int64_t j = qlo + lane; j < qhi; j += 32) acc += ch.cnt[(int64_t)s * ch.ccap + (perm ? (int64_t)perm[j] : j)];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(CH_FULL, acc, o);
            if (lane == 0) pa.cnt[(int64_t)s * pa.ccap + q] = acc;
        }
    }
}

// warp per parent (groups averaging several children: layer / phase / iteration / gpu roll-ups and
// points): lanes take consecutive children (coalesced on field-major tables), every field and counter
// in one pass, then a butterfly.
__global__ void __launch_bounds__(256) k_sum_rows_warp(TabView ch, const uint32_t *__restrict__ perm,
                                                       const int64_t *__restrict__ starts, int64_t ng, int shift,
                                                       int C, TabView pa) {
    const int lane = lane_id();
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (q >= ng) return;
    const int64_t qlo = starts[q], qhi = starts[q + 1];
    RowAcc a;
    a.zero();
    constexpr int CMAX = 32;
    double acc[CMAX];
#pragma unroll
    for (int s = 0; s < CMAX; s++) acc[s] = 0.0;
    for (int64_t j = qlo + lane; j < qhi; j += 32) {
        const int64_t c = perm ? (int64_t)perm[j] : j;
        a.add_child(ch, c);
#pragma unroll
        for (int s = 0; s < CMAX; s++)
            if (s < C) acc[s] += ch.cnt[(int64_t)s * ch.ccap + c];
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

// block of RC_NT parents: their children (a contiguous range, or a perm range) are staged RC_CH at a time
// in shared memory -- coalesced column loads for field-major tables, one 128 B row per child for the
// AoS sub-run rows -- and each thread folds its own parent's children from shared memory in order.
constexpr int RC_NT = 256, RC_CH = 256;
__global__ void __launch_bounds__(RC_NT) k_sum_rows_chunked(TabView ch, const uint32_t *__restrict__ perm,
                                                            const int64_t *__restrict__ starts, int64_t ng, int shift,
                                                            int C, TabView pa) {
    extern __shared__ int64_t rsm[];
    const int NF = RF_NFIELDS + C;
    int64_t *vals = rsm;                               // [NF][RC_CH]
    const int tid = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * RC_NT;
    const int64_t pend = min(p0 + RC_NT, ng);
    const int64_t p = p0 + tid;
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
            for (int e = tid; e < NF * RC_CH; e += RC_NT) {
                const int f = e / RC_CH, t = e % RC_CH;
                if (t < m) {
                    const int64_t c = j0 + t;
                    vals[e] = f < RF_NFIELDS ? ch.f[(int64_t)f * ch.cap + c]
                                             : __double_as_longlong(ch.cnt[(int64_t)(f - RF_NFIELDS) * ch.ccap + c]);
                }
            }
        } else {
            for (int t = tid; t < m; t += RC_NT) {
                const int64_t c = perm ? (int64_t)perm[j0 + t] : j0 + t;
                const int64_t *row = ch.f + c * ch.rs;
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) vals[f * RC_CH + t] = row[(int64_t)f * ch.cap];
                for (int s2 = 0; s2 < C; s2++)
                    vals[(RF_NFIELDS + s2) * RC_CH + t] = __double_as_longlong(ch.cnt[(int64_t)s2 * ch.ccap + c]);
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
    if (p >= ng) return;
#pragma unroll
    for (int f = 0; f < RF_NFIELDS; f++) pa.f[(int64_t)f * pa.cap + p] = a.v[f];
#pragma unroll
    for (int s2 = 0; s2 < 8; s2++)
        if (s2 < C) pa.cnt[(int64_t)s2 * pa.ccap + p] = cs[s2];
    const unsigned long long k0 = my_hi > my_lo ? ch.key[perm ? (int64_t)perm[my_lo] : my_lo] : 0ull;
    pa.key[p] = shift >= 64 ? 0ull : ((k0 >> shift) << shift);
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

// points (gpu, iteration, op label) = instances of the iteration with that op label, summed over layers
// in instance order.  One block per iteration group of the sorted instance table:
// chunks of PT_CH instances are loaded coalesced into shared memory, then thread l folds the chunk's
// instances with label l in order.  Results go to a dense [label][lg][rank] grid (compacted afterwards in
// (label, lg, rank) order = point-key order).
constexpr int PT_CH = 256;
__global__ void __launch_bounds__(256) k_points_iter(TabView iv, const int64_t *__restrict__ its, int64_t n_it,
                                                     KeyLayout Lk, const int64_t *__restrict__ list_beg,
                                                     const int32_t *__restrict__ P_label, int nL, int n_lg, int R0,
                                                     int C, int64_t *__restrict__ df, double *__restrict__ dc,
                                                     int64_t *__restrict__ dvalid, unsigned int *__restrict__ ovf) {
    // one instance per thread per chunk; a stable counting sort by label puts each label's instances of
    // the chunk in a contiguous list (instance order), which thread `label` then folds
    extern __shared__ int64_t psm[];
    const int NF = RF_NFIELDS + C;
    int64_t *vals = psm;                                                      // [NF][PT_CH]
    double *cacc = reinterpret_cast<double *>(vals + (int64_t)NF * PT_CH);    // [nL][C]
    int32_t *lab = reinterpret_cast<int32_t *>(cacc + (int64_t)nL * C);       // [PT_CH]
    int32_t *order = lab + PT_CH;                                             // [PT_CH]
    int32_t *wc = order + PT_CH;                                              // [8][nL] per-warp counts
    int32_t *lstart = wc + 8 * nL;                                            // [nL]
    __shared__ int64_t scan_sm[33];
    const int64_t g = blockIdx.x;
    if (g >= n_it) return;
    const int64_t a = its[g], b = its[g + 1];
    const unsigned long long k0 = iv.key[a];
    const int lg = (int)(k0 >> Lk.sh_lg);
    const int rank = (int)comp(k0, Lk.sh_it, Lk.kb[0]) - 1;
    const int64_t opb = list_beg[lg * 4 + 3];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t cells = (int64_t)nL * n_lg * R0;
    RowAcc acc;
    acc.zero();
    int cnt_n = 0;
    for (int q = tid; q < nL * C; q += blockDim.x) cacc[q] = 0.0;
    for (int64_t j0 = a; j0 < b; j0 += PT_CH) {
        const int m = (int)min((int64_t)PT_CH, b - j0);
        for (int e = tid; e < NF * PT_CH; e += blockDim.x) {
            const int f = e / PT_CH, t = e % PT_CH;
            if (t < m) {
                const int64_t j = j0 + t;
                vals[e] = f < RF_NFIELDS ? iv.f[(int64_t)f * iv.cap + j]
                                         : __double_as_longlong(iv.cnt[(int64_t)(f - RF_NFIELDS) * iv.ccap + j]);
            }
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
        if (tid < nL) lstart[tid] = st;
        __syncthreads();
        if (l >= 0) order[lstart[l] + wc[w * nL + l] + inrank] = tid;
        __syncthreads();
        if (tid < nL) {
            for (int k = st; k < st + tot_l; k++) {
                const int t = order[k];
                int64_t x[RF_NFIELDS];
#pragma unroll
                for (int f = 0; f < RF_NFIELDS; f++) x[f] = vals[f * PT_CH + t];
                acc.merge(x);
                for (int s2 = 0; s2 < C; s2++)
                    cacc[tid * C + s2] += __longlong_as_double(vals[(RF_NFIELDS + s2) * PT_CH + t]);
            }
            cnt_n += tot_l;
        }
        __syncthreads();
    }
    if (tid < nL && cnt_n > 0) {
        const int64_t cell = ((int64_t)tid * n_lg + lg) * R0 + rank;
#pragma unroll
        for (int f = 0; f < RF_NFIELDS; f++) df[(int64_t)f * cells + cell] = acc.v[f];
        for (int s2 = 0; s2 < C; s2++) dc[(int64_t)s2 * cells + cell] = cacc[tid * C + s2];
        dvalid[cell] = 1;
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

// parents from n children: warp per parent when groups average >= 4 children (and counters fit the
// warp kernel's register array), else lane per parent with warp help for the few big groups
static chopper_status sum_rows(chopper_ctx *ctx, const TabView &ch, const uint32_t *perm, const int64_t *starts,
                               int64_t ng, int64_t n_children, int shift, int C, const TabView &pa) {
    if (ng <= 0) return CHOPPER_OK;
    const size_t shb = (size_t)(RF_NFIELDS + C) * RC_CH * 8;
    if (n_children >= 16 * ng && C <= 32) {
        // parents with many children (layer -> phase, iteration -> gpu): a warp per parent
        k_sum_rows_warp<<<(unsigned)ceil_div(ng * 32, NT), NT, 0, ctx->st>>>(ch, perm, starts, ng, shift, C, pa);
    } else if (ng >= (int64_t)RC_NT * 148 && shb <= 160 * 1024) {
        // many parents with a few children each (instance -> layer): children staged per block
        static size_t attr = 0;
        if (shb > 48 * 1024 && shb > attr) {
            CH_CUDA(ctx, cudaFuncSetAttribute(k_sum_rows_chunked, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shb));
            attr = shb;
        }
        if (C > 8) CH_CUDA(ctx, cudaMemsetAsync(pa.cnt, 0, 8 * (size_t)C * pa.ccap, ctx->st));
        k_sum_rows_chunked<<<(unsigned)ceil_div(ng, RC_NT), RC_NT, shb, ctx->st>>>(ch, perm, starts, ng, shift, C, pa);
    } else {
        k_sum_rows<<<(unsigned)ceil_div(ng, NT), NT, 0, ctx->st>>>(ch, perm, starts, ng, shift, C, pa);
    }
    CH_LAUNCHED(ctx);
    return CHOPPER_OK;
}

static chopper_status rollup(chopper_ctx *ctx, RowTable &child, RowTable &parent, int shift, int depth,
                             const KeyLayout &L, int32_t *lg_gpu_d) {
    int64_t *starts;
    int64_t ng;
    CH_TRY(group(ctx, child.key, child.n, shift, &starts, &ng));
    CH_TRY(alloc_table(ctx, parent, std::max<int64_t>(ng, 1), ctx->C, true));
    parent.n = ng;
    if (ng > 0) {
        CH_TRY(sum_rows(ctx, view(child), nullptr, starts, ng, child.n, shift, ctx->C, view(parent)));
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
        const int n_lg = ctx->n_lg;
        const int n_passes = (int)ctx->passes.size();
        ctx->d_colbad = CH_ALLOC(ctx, unsigned int, (int64_t)n_lg * C);
        CH_ALLOC_END(ctx);
        for (int round = 0; round < 2; round++) {
            CH_CUDA(ctx, cudaMemsetAsync(ctx->d_colbad, 0, 4 * (size_t)n_lg * C, ctx->st));
            static bool attr = false;
            if (!attr) {
                CH_CUDA(ctx, cudaFuncSetAttribute(k_counters_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)sizeof(CtSmem)));
                attr = true;
            }
            const int vec_ok = (((uintptr_t)ctx->ev.meta | (uintptr_t)ctx->d_run_id | (uintptr_t)ctx->d_nm_rank) & 15u) == 0;
            for (int s0 = 0; s0 < C; s0 += CT_SG) {
                k_counters_tiled<<<(unsigned)ceil_div(ctx->N, CT_TILE), CT_NT, sizeof(CtSmem), ctx->st>>>(
                    ctx->ev.meta, ctx->d_run_id, ctx->d_nm_rank, ctx->d_gpu_lg, ctx->d_col, C, s0, ctx->N, subv.cnt,
                    subv.ccap, ctx->d_colbad, ctx->d_mg, vec_ok);
                CH_LAUNCHED(ctx);
            }
            // finiteness of every name-matching pass (R8): columns feeding a slot were checked just now,
            // the others by k_pass_finite in ch_align
            std::vector<unsigned int> cb((size_t)n_lg * C), pb(std::max(n_passes, 1));
            CH_CUDA(ctx, cudaMemcpyAsync(cb.data(), ctx->d_colbad, 4 * cb.size(), cudaMemcpyDeviceToHost, ctx->st));
            if (n_passes > 0)
                CH_CUDA(ctx, cudaMemcpyAsync(pb.data(), ctx->d_pass_bad, 4 * n_passes, cudaMemcpyDeviceToHost, ctx->st));
            CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
            bool changed = false;
            for (int p = 0; p < n_passes; p++) {
                if (ctx->pass_mismatch[p] >= 0 || ctx->pass_bad[p]) continue;
                bool bad = pb[p] != 0;
                for (size_t q = 0; q < cb.size(); q++)
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
            // (every name-matching pass's finiteness is now known, so one redo settles it)
            CH_TRY(ch_assign_slots(ctx));
            CH_TRY(ch_counters_full(ctx));
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
    {
        // segmented sort inside (gpu, iteration) prefixes; radix sort if the prefixes are not in order
        bool done = false;
        if (R > 1) {
            size_t mk = ctx->used;
            int64_t *hd = CH_ALLOC(ctx, int64_t, R), *ex = CH_ALLOC(ctx, int64_t, R), *st = CH_ALLOC(ctx, int64_t, R + 2);
            int64_t *nseg_d = CH_ALLOC(ctx, int64_t, 1);
            unsigned int *bad = CH_ALLOC(ctx, unsigned int, 1);
            CH_ALLOC_END(ctx);
            k_prefix_heads<<<(unsigned)ceil_div(R, NT), NT, 0, ctx->st>>>(k1, R, L.sh_it, hd);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_scan_excl_i64(ctx, hd, ex, R, nseg_d));
            k_group_starts<<<(unsigned)ceil_div(R, NT), NT, 0, ctx->st>>>(hd, ex, R, st);
            CH_LAUNCHED(ctx);
            int64_t nseg = 0;
            CH_CUDA(ctx, cudaMemcpyAsync(&nseg, nseg_d, 8, cudaMemcpyDeviceToHost, ctx->st));
            CH_CUDA(ctx, cudaMemsetAsync(bad, 0, 4, ctx->st));
            CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
            int64_t rr = R;
            CH_CUDA(ctx, cudaMemcpyAsync(st + nseg, &rr, 8, cudaMemcpyHostToDevice, ctx->st));
            k_prefix_check<<<(unsigned)ceil_div(nseg, NT), NT, 0, ctx->st>>>(k1, st, nseg, L.sh_it, bad);
            CH_LAUNCHED(ctx);
            unsigned int hbad = 0;
            CH_CUDA(ctx, cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, ctx->st));
            CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
            if (!hbad) {
                static bool ss_attr = false;
                if (!ss_attr) {
                    CH_CUDA(ctx, cudaFuncSetAttribute(k_seg_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)sizeof(SegSortSmem)));
                    ss_attr = true;
                }
                k_seg_sort<<<(unsigned)nseg, SS_NT, sizeof(SegSortSmem), ctx->st>>>(k1, v1, st, nseg, L);
                CH_LAUNCHED(ctx);
                k_valid_flags<<<(unsigned)ceil_div(R, NT), NT, 0, ctx->st>>>(k1, R, hd);
                CH_LAUNCHED(ctx);
                CH_TRY(ch_scan_excl_i64(ctx, hd, ex, R, nseg_d));
                k_partition<<<(unsigned)ceil_div(R, NT), NT, 0, ctx->st>>>(k1, v1, R, ex, nseg_d, k2, v2);
                CH_LAUNCHED(ctx);
                alt = true;
                done = true;
            }
            ctx->used = mk;
        }
        if (!done) CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, R, 0, key_bits, &alt));
    }
    unsigned long long *ks = alt ? k2 : k1;
    uint32_t *so = alt ? v2 : v1;
    {
        int64_t *starts;
        int64_t ng;
        CH_TRY(group(ctx, ks, R, 0, &starts, &ng));
        CH_TRY(alloc_table(ctx, ctx->inst, std::max<int64_t>(ng, 1), C, true));
        ctx->inst.n = ng;
        if (ng > 0) {
            CH_TRY(sum_rows(ctx, subv, so, starts, ng, R, 0, C, view(ctx->inst)));
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
    // points (label, gpu, iteration): per-iteration label folds into a dense grid, then compaction
    {
        const int64_t n = ctx->inst.n;
        const int nL = std::max(ctx->cfg.n_labels, 1), n_lg = std::max(ctx->n_lg, 1);
        const int R0 = (int)std::max<int64_t>(ctx->max_it_list, 1);
        const int64_t cells = (int64_t)nL * n_lg * R0;
        int lbits = bits_for((uint64_t)std::max(ctx->cfg.n_labels, 1));
        int pbits = lbits + ctx->kg + L.kb[0];
        if (pbits > 63) return ch_fail(ctx, CHOPPER_E_RANGE, "point key exceeds 63 bits");
        int64_t *its = nullptr, n_it = 0;
        CH_TRY(group(ctx, ctx->inst.key, n, L.sh_it, &its, &n_it));
        int64_t *df = CH_ALLOC(ctx, int64_t, (int64_t)RF_NFIELDS * cells);
        double *dc = CH_ALLOC(ctx, double, (int64_t)std::max(C, 1) * cells);
        int64_t *dvalid = CH_ALLOC(ctx, int64_t, cells), *dex = CH_ALLOC(ctx, int64_t, cells), *np_d = CH_ALLOC(ctx, int64_t, 1);
        unsigned int *ovf = CH_ALLOC(ctx, unsigned int, 1);
        CH_ALLOC_END(ctx);
        CH_CUDA(ctx, cudaMemsetAsync(dvalid, 0, 8 * (size_t)cells, ctx->st));
        CH_CUDA(ctx, cudaMemsetAsync(ovf, 0, 4, ctx->st));
        if (n_it > 0) {
            if (nL > 256) return ch_fail(ctx, CHOPPER_E_RANGE, "more than 256 op labels");
            size_t shb = (size_t)(RF_NFIELDS + C) * PT_CH * 8 + (size_t)nL * C * 8 + 4 * (2 * PT_CH + 9 * (size_t)nL);
            static size_t attr_shb = 0;
            if (shb > 48 * 1024 && shb > attr_shb) {
                CH_CUDA(ctx, cudaFuncSetAttribute(k_points_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shb));
                attr_shb = shb;
            }
            k_points_iter<<<(unsigned)n_it, 256, shb, ctx->st>>>(view(ctx->inst), its, n_it, L, ctx->d_list_beg,
                                                                 ctx->P_label, nL, n_lg, R0, C, df, dc, dvalid, ovf);
            CH_LAUNCHED(ctx);
        }
        CH_TRY(ch_scan_excl_i64(ctx, dvalid, dex, cells, np_d));
        int64_t np = 0;
        unsigned int hovf = 0;
        CH_CUDA(ctx, cudaMemcpyAsync(&np, np_d, 8, cudaMemcpyDeviceToHost, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(&hovf, ovf, 4, cudaMemcpyDeviceToHost, ctx->st));
        CH_CUDA(ctx, cudaStreamSynchronize(ctx->st));
        if (hovf) return ch_fail(ctx, CHOPPER_E_RANGE, "op span label >= n_labels");
        CH_TRY(alloc_table(ctx, ctx->point, std::max<int64_t>(np, 1), C, true));
        ctx->point.n = np;
        if (np > 0) {
            k_points_compact<<<(unsigned)ceil_div(cells, NT), NT, 0, ctx->st>>>(dvalid, dex, cells, df, dc, C, n_lg, R0,
                                                                              ctx->kg, L.kb[0], view(ctx->point));
            CH_LAUNCHED(ctx);
            k_decode_points<<<(unsigned)ceil_div(np, NT), NT, 0, ctx->st>>>(
                ctx->point.key, np, ctx->kg, L.kb[0], lg_gpu_d, ctx->d_list_beg, ctx->P_orig, ctx->point.f,
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
