// compose.cu -- a10 gap decomposition and a11 cross-rank reduce
// (chopper_breakdown part 2, chopper_reduce_ranks).
//
// Per-gpu rows are laid into a fixed-shape dense exchange block (iteration rows
// [max_iters], points [max_iters][n_labels]) so that the cross-rank exchange is
// exactly one ncclAllGather (#2) and every rank composes the global result in
// the same order, re-indexed by gpu id (identical for any rank count).
//
// a10 (Eqs. 4-8; readings D14-D20): one block per gemm / fa
// op label.  Medians by block bitonic sort; the least-squares fallback and the
// final factors are evaluated by one thread in (gpu, iteration) order with the
// same operation order as DESIGN.md O13 (compiled with -fmad=false).
// a11: T(it) = max over gpus of (busy + launch),
// throughput = b*s*R / T, median over sampled iterations.
#include "common.cuh"

namespace {
// exchange block layout (int64 words; doubles bit-cast)
constexpr int HDR = 4;          // gpu, present, has_samples, C
constexpr int IT_W = 8;         // valid, step, busy, prep, call, n, first_ks, last_ke
constexpr int PT_W = 9;         // valid, busy, launch, ovl, phi, cg, fp, un, ud
constexpr int E2E_P = 8, E2E_W = E2E_P * 4;   // per iteration rank: [phase label][vec, gemm, fa, launch] (O16)

struct Layout {
    int64_t MI, L, C, W;
    __host__ __device__ int64_t it_off() const { return HDR + C; }
    __host__ __device__ int64_t pt_off() const { return HDR + C + IT_W * MI; }
    __host__ __device__ int64_t e2e_off() const { return HDR + C + IT_W * MI + PT_W * MI * L; }
};

__device__ __forceinline__ int64_t dbits(double d) { return __double_as_longlong(d); }
__device__ __forceinline__ double bitsd(int64_t v) { return __longlong_as_double(v); }

__global__ void k_dense_header(int64_t *blk, Layout Ly, int n_lg, const int32_t *__restrict__ lg_gpu,
                               const int32_t *__restrict__ has_smp, const int32_t *__restrict__ present) {
    int l = blockIdx.x;
    if (l >= n_lg) return;
    int64_t *b = blk + (int64_t)l * Ly.W;
    if (threadIdx.x == 0) {
        b[0] = lg_gpu[l];
        b[1] = 1;
        b[2] = has_smp[l];
        b[3] = Ly.C;
    }
    for (int s = threadIdx.x; s < Ly.C; s += blockDim.x) b[HDR + s] = present[(int64_t)l * Ly.C + s];
}

__global__ void k_dense_iters(int64_t *blk, Layout Ly, int64_t n, const int32_t *__restrict__ gpu,
                              const int32_t *__restrict__ rank, const int32_t *__restrict__ step,
                              const int64_t *__restrict__ f, int64_t cap, const int32_t *__restrict__ gpu_lg,
                              unsigned int *ovf) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int64_t r = rank[j];
    if (r < 0 || r >= Ly.MI) { atomicOr(ovf, 1u); return; }
    int64_t *b = blk + (int64_t)gpu_lg[gpu[j]] * Ly.W + Ly.it_off() + r * IT_W;
    b[0] = 1;
    b[1] = step[j];
    b[2] = f[(int64_t)RF_BUSY * cap + j];
    b[3] = f[(int64_t)RF_PREP * cap + j];
    b[4] = f[(int64_t)RF_CALL * cap + j];
    b[5] = f[(int64_t)RF_N * cap + j];
    b[6] = f[(int64_t)RF_FIRST_KS * cap + j];
    b[7] = f[(int64_t)RF_LAST_KE * cap + j];
}

__global__ void k_dense_points(int64_t *blk, Layout Ly, int64_t n, const int32_t *__restrict__ gpu,
                               const int32_t *__restrict__ rank, const int32_t *__restrict__ label,
                               const int64_t *__restrict__ f, const double *__restrict__ cnt, int64_t cap,
                               const int32_t *__restrict__ gpu_lg, int s_cyc, int s_fl, int s_un, int s_ud,
                               unsigned int *ovf) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int64_t r = rank[j];
    int lab = label[j];
    if (r < 0 || r >= Ly.MI || lab < 0 || lab >= Ly.L) { atomicOr(ovf, 1u); return; }
    int64_t *b = blk + (int64_t)gpu_lg[gpu[j]] * Ly.W + Ly.pt_off() + (r * Ly.L + lab) * PT_W;
    b[0] = 1;
    b[1] = f[(int64_t)RF_BUSY * cap + j];
    b[2] = f[(int64_t)RF_PREP * cap + j] + f[(int64_t)RF_CALL * cap + j];
    b[3] = f[(int64_t)RF_OVL * cap + j];
    b[4] = f[(int64_t)RF_PHI * cap + j];
    b[5] = dbits(s_cyc >= 0 ? cnt[(int64_t)s_cyc * cap + j] : 0.0);
    b[6] = dbits(s_fl >= 0 ? cnt[(int64_t)s_fl * cap + j] : 0.0);
    b[7] = dbits(s_un >= 0 ? cnt[(int64_t)s_un * cap + j] : 0.0);
    b[8] = dbits(s_ud >= 0 ? cnt[(int64_t)s_ud * cap + j] : 0.0);
}

// O16 cells: instance durations by (phase label, op type) and launch overhead by phase label, summed into
// the gpu's iteration-rank row of the exchange block (integer atomics: exact in any order)
// instances are in key order, so long runs of them share a (gpu, iteration, phase) row: each lane walks K of a
// warp's 32 K instances (stride 32, coalesced) and accumulates per target cell, issuing the atomics only when the
// row changes (integer sums: exact in any order).  K grows with the instance count once the grid is full
// (a small table keeps K = 1: every lane one instance, all in parallel)
constexpr int E2E_KMAX = 16;
__global__ void k_dense_e2e(int64_t *blk, Layout Ly, const int64_t *__restrict__ n_dev, const int32_t *__restrict__ gpu,
                            const int32_t *__restrict__ rank, const int32_t *__restrict__ ph,
                            const int32_t *__restrict__ label, const int64_t *__restrict__ f, int64_t cap,
                            const int32_t *__restrict__ gpu_lg, const int32_t *__restrict__ span_label,
                            const int32_t *__restrict__ op_type, int E2E_K) {
    const int64_t n = *n_dev;
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w0 = wid * 32 * E2E_K; w0 < n; w0 += nw * 32 * E2E_K) {
        int64_t *cur = nullptr;
        unsigned long long acc[4] = {0, 0, 0, 0};
        for (int k = 0; k < E2E_K; k++) {
            const int64_t j = w0 + (int64_t)k * 32 + lane;
            if (j >= n) break;
            const int64_t r = rank[j];
            if (r < 0 || r >= Ly.MI || ph[j] < 0) continue;
            const int P = span_label[ph[j]];
            if (P < 0 || P >= E2E_P) continue;
            const int lab = label[j];
            const int T = lab >= 0 && op_type[lab] == 1 ? 1 : lab >= 0 && op_type[lab] == 2 ? 2 : 0;
            int64_t *b = blk + (int64_t)gpu_lg[gpu[j]] * Ly.W + Ly.e2e_off() + r * E2E_W + P * 4;
            if (b != cur) {
                if (cur)
                    for (int q = 0; q < 4; q++)
                        if (acc[q]) atomicAdd(reinterpret_cast<unsigned long long *>(cur + q), acc[q]);
                cur = b;
                acc[0] = acc[1] = acc[2] = acc[3] = 0;
            }
            acc[T] += (unsigned long long)f[(int64_t)RF_BUSY * cap + j];
            acc[3] += (unsigned long long)(f[(int64_t)RF_PREP * cap + j] + f[(int64_t)RF_CALL * cap + j]);
        }
        if (cur)
            for (int q = 0; q < 4; q++)
                if (acc[q]) atomicAdd(reinterpret_cast<unsigned long long *>(cur + q), acc[q]);
    }
}

// ---- block-level helpers ----
// Bitonic sort of a[0..n2) (n2 a power of two) by the whole block.  Each warp owns a contiguous segment of
// n2 / warps elements, so every stage with partner distance j below the segment length stays inside one warp
// and needs only __syncwarp; block barriers remain for the log2(warps) widest distances of each merge.
template <class T>
__device__ void block_bitonic(T *a, int n2) {
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int seg = n2 / nw;
    const bool local_ok = seg >= 32 && seg * nw == n2;
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (local_ok && j < seg) {
                for (int i = w * seg + l; i < (w + 1) * seg; i += 32) {
                    const int x = i ^ j;
                    if (x > i) {
                        const bool up = (i & k) == 0;
                        const T p = a[i], q = a[x];
                        if ((p > q) == up) { a[i] = q; a[x] = p; }
                    }
                }
                __syncwarp();
                continue;
            }
            __syncthreads();
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int x = i ^ j;
                if (x > i) {
                    const bool up = (i & k) == 0;
                    const T p = a[i], q = a[x];
                    if ((p > q) == up) { a[i] = q; a[x] = p; }
                }
            }
            __syncthreads();
        }
    }
    __syncthreads();
}
// block sum of doubles (all threads get the total); sh holds >= 32 doubles
__device__ __forceinline__ double block_sum_f64(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CH_FULL, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += sh[i];
    return t;
}
__device__ __forceinline__ int pow2ceil(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}
// median of a[0..n) (D21: even count = mean of the two central values).  The values are sorted in
// shared memory when they fit (sh != nullptr), else in place in global memory.
__device__ double med_i64(int64_t *a, int n, int64_t *sh) {
    int n2 = pow2ceil(n);
    int64_t *w = sh ? sh : a;
    for (int i = threadIdx.x; i < n2; i += blockDim.x)
        if (w != a || i >= n) w[i] = i < n ? a[i] : INT64_MAX;
    __syncthreads();
    block_bitonic<int64_t>(w, n2);
    double m = (n % 2) ? (double)w[n / 2] : 0.5 * ((double)w[n / 2 - 1] + (double)w[n / 2]);
    __syncthreads();
    return m;
}
__device__ double med_f64(double *a, int n, double *sh) {
    int n2 = pow2ceil(n);
    double *w = sh ? sh : a;
    for (int i = threadIdx.x; i < n2; i += blockDim.x)
        if (w != a || i >= n) w[i] = i < n ? a[i] : INFINITY;
    __syncthreads();
    block_bitonic<double>(w, n2);
    double m = (n % 2) ? w[n / 2] : 0.5 * (w[n / 2 - 1] + w[n / 2]);
    __syncthreads();
    return m;
}

// medians of up to MED_SM values sorted in a static shared-memory buffer (16 KB) instead of in place in global
// memory (each bitonic stage would otherwise be a global-memory round trip)
constexpr int MED_SM = 2048;
__device__ __forceinline__ int64_t *med_buf() {
    __shared__ __align__(16) int64_t b[MED_SM];
    return b;
}
__device__ __forceinline__ double med_i64_s(int64_t *a, int n) {
    return med_i64(a, n, pow2ceil(n) <= MED_SM ? med_buf() : nullptr);
}
__device__ __forceinline__ double med_f64_s(double *a, int n) {
    return med_f64(a, n, pow2ceil(n) <= MED_SM ? reinterpret_cast<double *>(med_buf()) : nullptr);
}

enum { BD_FIT = 1, BD_NO_FLOPS = 2, BD_NO_UTIL = 4, BD_UTIL_RANGE = 8, BD_D0_ZERO = 16, BD_NO_CYCLES = 32,
       BD_NO_SAMPLES = 64, BD_INSUFFICIENT = 128 };

struct BdArgs {
    const int64_t *blk;
    int nslots;
    Layout Ly;
    const int32_t *slot_order;   // slots sorted by gpu id, -1 terminated
    const int32_t *labels;       // gemm / fa labels, one per block row
    const double *f_gemm;
    double tpt, freq;
    int warmup;
    int s_cyc, s_fl, s_un, s_ud;
    int64_t maxp2;               // capacity per work array (pow2)
    int64_t *wi;                 // [nblocks][BD_TASKS][maxp2] int64 / double work arrays (global fallback)
    double *res;                 // [nblocks][BD_TASKS][4] task results
    double *out;                 // [nblocks][16]
    int use_smem;
};

// one block per (gemm / fa label, task): every median of O13 runs in its own block (the points are few,
// the blocks many); k_bd_compose then evaluates Eqs. 4-8 per label in the fixed order of DESIGN.md O13.
enum { BT_ACT = 0, BT_D0, BT_D50, BT_FP, BT_U, BT_CG, BT_BL, BT_V, BT_FIT, BD_TASKS };

__global__ void __launch_bounds__(512) k_breakdown(BdArgs A) {
    extern __shared__ int64_t bsh[];
    const int task = blockIdx.y;
    const int L = A.labels[blockIdx.x];
    double *res = A.res + ((int64_t)blockIdx.x * BD_TASKS + task) * 4;
    int64_t *w = A.use_smem ? bsh : A.wi + ((int64_t)blockIdx.x * BD_TASKS + task) * 2 * A.maxp2;
    int64_t *w2 = w + A.maxp2;                   // second operand (LS fit)
    double *wd = reinterpret_cast<double *>(w), *wd2 = reinterpret_cast<double *>(w2);
    const Layout Ly = A.Ly;
    __shared__ int64_t scan_sm[33];
    __shared__ int s_count, s_all, s_flags_in;
    if (threadIdx.x == 0) {
        s_count = 0;
        s_all = 0;
        s_flags_in = (A.s_cyc >= 0) | ((A.s_fl >= 0) << 1) | ((A.s_un >= 0 && A.s_ud >= 0) << 2) | (1 << 3);
    }
    __syncthreads();
    // sampled points of L in (gpu, iteration) order (ordered block compaction over the candidate grid);
    // each task keeps the members and the value it needs.  Slot presence is AND-ed over contributing gpus.
    {
        int nq = 0;
        while (nq < A.nslots && A.slot_order[nq] >= 0) nq++;
        const int64_t r0 = A.warmup > 0 ? A.warmup : 0;
        const int64_t nr = Ly.MI > r0 ? Ly.MI - r0 : 0;
        const int64_t total = (int64_t)nq * nr;
        for (int64_t c0 = 0; c0 < total; c0 += blockDim.x) {
            int64_t c = c0 + threadIdx.x;
            bool ok = false, keep = false;
            const int64_t *b = nullptr, *p = nullptr;
            if (c < total) {
                b = A.blk + (int64_t)A.slot_order[c / nr] * Ly.W;
                p = b + Ly.pt_off() + ((r0 + c % nr) * Ly.L + L) * PT_W;
                ok = b[1] != 0 && p[0] != 0 && p[1] > 0;
            }
            int64_t busy = 0, launch = 0, ovl = 0, phi = 0;
            if (ok) {
                busy = p[1]; launch = p[2]; ovl = p[3]; phi = p[4];
                keep = true;
                if (task == BT_D0) keep = 20 * ovl <= busy;                                   // D15 buckets
                if (task == BT_D50) keep = 2 * busy <= 5 * ovl && 5 * ovl <= 3 * busy;
                int drop = 0;
                if (A.s_cyc >= 0 && !b[HDR + A.s_cyc]) drop |= 1;
                if (A.s_fl >= 0 && !b[HDR + A.s_fl]) drop |= 2;
                if (A.s_un >= 0 && A.s_ud >= 0 && !(b[HDR + A.s_un] && b[HDR + A.s_ud])) drop |= 4;
                if (!b[2]) drop |= 8;
                if (drop) atomicAnd(&s_flags_in, ~drop);
            }
            int64_t tot, tall;
            int64_t pos = block_excl_sum<512>(keep ? 1 : 0, &tot, scan_sm) + s_count;
            block_excl_sum<512>(ok ? 1 : 0, &tall, scan_sm);
            if (keep && pos < A.maxp2) {
                switch (task) {
                    case BT_ACT: case BT_D0: case BT_D50: w[pos] = busy; break;
                    case BT_FP: wd[pos] = bitsd(p[6]); break;
                    case BT_U:      // both readings; presence (known after the gather) picks one (D18)
                        wd[pos] = bitsd(p[7]) / bitsd(p[8]);
                        wd2[pos] = (bitsd(p[6]) / bitsd(p[5])) * (A.freq / A.tpt);
                        break;
                    case BT_CG: wd[pos] = bitsd(p[5]); break;
                    case BT_BL: w[pos] = busy + launch; break;
                    case BT_V: wd[pos] = (double)phi / (double)busy * 1e6; break;
                    case BT_FIT: wd[pos] = (double)ovl / (double)busy; wd2[pos] = (double)busy; break;
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) { s_count += (int)tot; s_all += (int)tall; }
            __syncthreads();
        }
    }
    const int n = s_count < A.maxp2 ? s_count : (int)A.maxp2;
    const int n_all = s_all < A.maxp2 ? s_all : (int)A.maxp2;
    const int fin = n_all == 0 ? (s_flags_in & ~8) : s_flags_in;
    const bool has_cyc = fin & 1, has_fl = fin & 2, has_util = fin & 4, has_smp = fin & 8;
    bool run = n_all >= 2 && n > 0;
    if (task == BT_FP) run &= has_fl;
    if (task == BT_U) run &= has_util || (has_fl && has_cyc);
    if (task == BT_CG) run &= has_cyc;
    if (task == BT_V) run &= has_smp;
    if (run && task == BT_U && !has_util) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) wd[i] = wd2[i];
        __syncthreads();
    }
    double m = 0.0;
    if (run && task != BT_FIT) {
        if (task == BT_ACT || task == BT_D0 || task == BT_D50 || task == BT_BL) m = med_i64(w, n, nullptr);
        else m = med_f64(wd, n, nullptr);
    }
    if (run && task == BT_FIT && threadIdx.x == 0) {
        // least-squares busy ~ a + c*r over all points, two sequential passes in (gpu, iteration) order
        double sr = 0.0, sb = 0.0;
        for (int i = 0; i < n; i++) { sr += wd[i]; sb += wd2[i]; }
        double mr = sr / (double)n, mb = sb / (double)n, sxx = 0.0, sxy = 0.0;
        for (int i = 0; i < n; i++) {
            double dr = wd[i] - mr, db = wd2[i] - mb;
            sxx += dr * dr;
            sxy += dr * db;
        }
        if (sxx == 0.0) { res[1] = 0.0; res[2] = 0.0; res[3] = 1.0; }   // all r equal: D0 = D50 = D_act
        else { double c = sxy / sxx, a = mb - c * mr; res[1] = a; res[2] = a + c * 0.5; res[3] = 0.0; }
    }
    if (threadIdx.x == 0) {
        res[0] = m;
        if (task == BT_ACT) { res[1] = n_all; res[2] = fin; }
        if (task == BT_D0 || task == BT_D50) res[1] = n;
    }
}

__global__ void k_bd_compose(BdArgs A, int nb) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nb) return;
    const int L = A.labels[q];
    const double *r = A.res + (int64_t)q * BD_TASKS * 4;
    double *out = A.out + (int64_t)q * 16;
    for (int k = 0; k < 16; k++) out[k] = NAN;
    const int n = (int)r[BT_ACT * 4 + 1], fin = (int)r[BT_ACT * 4 + 2];
    if (n < 2) { out[0] = n; out[1] = 0; out[14] = BD_INSUFFICIENT; out[15] = L; return; }
    const bool has_cyc = fin & 1, has_fl = fin & 2, has_util = fin & 4, has_smp = fin & 8;
    int flags = 0;
    const double d_act = r[BT_ACT * 4];
    const int n0 = (int)r[BT_D0 * 4 + 1], n50 = (int)r[BT_D50 * 4 + 1];
    double d0, d50;
    const bool bucket = n0 > 0 && n50 > 0;
    if (bucket) { d0 = r[BT_D0 * 4]; d50 = r[BT_D50 * 4]; }
    else {
        if (r[BT_FIT * 4 + 3] != 0.0) { d0 = d_act; d50 = d_act; }
        else { d0 = r[BT_FIT * 4 + 1]; d50 = r[BT_FIT * 4 + 2]; }
        flags |= BD_FIT;
    }
    const double med_fp = r[BT_FP * 4], med_u = r[BT_U * 4], med_cg = r[BT_CG * 4], med_bl = r[BT_BL * 4],
                 med_v = r[BT_V * 4];
    out[0] = n;
    out[1] = bucket ? 0 : 1;
    out[2] = d_act * 1e-9;
    out[3] = d0 * 1e-9;
    out[4] = d50 * 1e-9;
    double d_thr = A.f_gemm[L] / A.tpt;                                   // Eq. 4
    out[5] = d_thr;
    double ovr_inst = 1.0;                                               // Eq. 5
    if (has_fl) ovr_inst = med_fp / A.f_gemm[L]; else flags |= BD_NO_FLOPS;
    out[6] = ovr_inst;
    double ovr_util = 1.0;                                               // Eq. 6
    if (has_util || (has_fl && has_cyc)) {
        if (!(med_u > 0.0 && med_u <= 1.0)) flags |= BD_UTIL_RANGE;
        ovr_util = 1.0 / med_u;
    } else flags |= BD_NO_UTIL;
    out[7] = ovr_util;
    double ovr_ovl = d50 / d0;                                           // Eq. 7
    if (!(d0 > 0.0)) flags |= BD_D0_ZERO;
    out[8] = ovr_ovl;
    if (has_cyc) {                                                       // Eq. 8
        double d_peak = med_cg / A.freq;
        out[9] = d_peak;
        out[10] = (d_act * 1e-9 / d_peak) / ovr_ovl;
    } else flags |= BD_NO_CYCLES;
    out[11] = med_bl / d_act;                                            // launch term (D20)
    out[12] = d_act * 1e-9 / (d_thr * ovr_inst * ovr_util * ovr_ovl * out[10]);
    if (has_smp) out[13] = A.freq / med_v; else flags |= BD_NO_SAMPLES;
    out[14] = flags;
    out[15] = L;
}

// ---- report statistics per op label (O14) ----------------
// One block per label over the same points as the breakdown (sampled iterations, busy > 0) in (gpu,
// iteration) order: duration and overlap-ratio quantiles at q = 0, .25, .5, .75, 1 (linear interpolation at
// h = q (n - 1), R9) from block bitonic sorts, and the Pearson correlation of ratio with duration (two
// passes, means then centred sums, each a block reduction; R10).  Row layout as oracle report.rows.
struct RepArgs {
    const int64_t *blk;
    int nslots;
    Layout Ly;
    const int32_t *slot_order;
    int warmup;
    int64_t maxp2;
    double *wk;                  // [L][4][maxp2] global work (when shared memory is too small)
    double *out;                 // [L][16]
    int use_smem;
};
__device__ __forceinline__ double quantile_sorted_dev(const double *x, int n, double q) {
    const double h = q * (double)(n - 1);
    const int lo = (int)floor(h);
    if (lo >= n - 1) return x[n - 1];
    const double fr = h - (double)lo;
    return x[lo] + fr * (x[lo + 1] - x[lo]);
}
__global__ void __launch_bounds__(512) k_report(RepArgs A) {
    extern __shared__ int64_t rsh[];
    const int L = blockIdx.x;
    const Layout Ly = A.Ly;
    double *w = A.use_smem ? reinterpret_cast<double *>(rsh) : A.wk + (int64_t)L * 4 * A.maxp2;
    double *b = w, *r = w + A.maxp2, *sb = w + 2 * A.maxp2, *sr = w + 3 * A.maxp2;
    double *out = A.out + (int64_t)L * 16;
    __shared__ int64_t scan_sm[33];
    __shared__ int s_count;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    int nq = 0;
    while (nq < A.nslots && A.slot_order[nq] >= 0) nq++;
    const int64_t r0 = A.warmup > 0 ? A.warmup : 0;
    const int64_t nr = Ly.MI > r0 ? Ly.MI - r0 : 0;
    const int64_t total = (int64_t)nq * nr;
    for (int64_t c0 = 0; c0 < total; c0 += blockDim.x) {
        const int64_t c = c0 + threadIdx.x;
        bool ok = false;
        const int64_t *p = nullptr;
        if (c < total) {
            const int64_t *bb = A.blk + (int64_t)A.slot_order[c / nr] * Ly.W;
            p = bb + Ly.pt_off() + ((r0 + c % nr) * Ly.L + L) * PT_W;
            ok = bb[1] != 0 && p[0] != 0 && p[1] > 0;
        }
        int64_t tot;
        const int64_t pos = block_excl_sum<512>(ok ? 1 : 0, &tot, scan_sm) + s_count;
        if (ok && pos < A.maxp2) {
            b[pos] = (double)p[1];
            r[pos] = (double)p[3] / (double)p[1];
        }
        __syncthreads();
        if (threadIdx.x == 0) s_count += (int)tot;
        __syncthreads();
    }
    const int n = s_count < A.maxp2 ? s_count : (int)A.maxp2;
    if (threadIdx.x < 16) out[threadIdx.x] = NAN;
    __syncthreads();
    if (threadIdx.x == 0) { out[0] = n; out[12] = L; }
    if (n == 0) return;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { sb[i] = b[i]; sr[i] = r[i]; }
    __syncthreads();
    {
        __shared__ double red[32];
        double pb = 0.0, pr = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) { pb += b[i]; pr += r[i]; }
        const double mb = block_sum_f64(pb, red) / (double)n;
        const double mr = block_sum_f64(pr, red) / (double)n;
        double pxx = 0.0, pyy = 0.0, pxy = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double dx = r[i] - mr, dy = b[i] - mb;
            pxx += dx * dx;
            pyy += dy * dy;
            pxy += dx * dy;
        }
        const double sxx = block_sum_f64(pxx, red), syy = block_sum_f64(pyy, red), sxy = block_sum_f64(pxy, red);
        if (threadIdx.x == 0) {
            out[11] = (sxx > 0.0 && syy > 0.0) ? sxy / sqrt(sxx * syy) : NAN;
            out[13] = mb;
        }
    }
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x)
        if (i >= n) { sb[i] = INFINITY; sr[i] = INFINITY; }
    __syncthreads();
    block_bitonic<double>(sb, n2);
    block_bitonic<double>(sr, n2);
    if (threadIdx.x < 5) {
        const double q = 0.25 * threadIdx.x;
        out[1 + threadIdx.x] = quantile_sorted_dev(sb, n, q);
        out[6 + threadIdx.x] = quantile_sorted_dev(sr, n, q);
    }
}

// ---- per-GPU overlap CDFs (O15; Fig. 7) ----------------------------
// block (label, slot position): the gpu's sampled points of the label; count pass, then a write pass that
// sorts them by (duration, iteration rank) -- one int64 key busy * 4096 + rank -- and emits
// (label, gpu, duration / minimum, overlap ratio, (k + 1) / n) at the scanned offset.
__device__ __forceinline__ bool cdf_point(const int64_t *blk, const Layout &Ly, int sl, int64_t r, int L,
                                          const int64_t **pp) {
    const int64_t *b = blk + (int64_t)sl * Ly.W;
    const int64_t *p = b + Ly.pt_off() + (r * Ly.L + L) * PT_W;
    *pp = p;
    return b[1] != 0 && p[0] != 0 && p[1] > 0;
}
__global__ void k_cdf_count(const int64_t *__restrict__ blk, Layout Ly, const int32_t *__restrict__ order, int nslots,
                            int warmup, int64_t *__restrict__ cnt) {
    const int L = blockIdx.x, q = blockIdx.y;
    const int sl = q < nslots ? order[q] : -1;
    int c = 0;
    if (sl >= 0)
        for (int64_t r = (warmup > 0 ? warmup : 0) + threadIdx.x; r < Ly.MI; r += blockDim.x) {
            const int64_t *p;
            c += cdf_point(blk, Ly, sl, r, L, &p) ? 1 : 0;
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(CH_FULL, c, o);
    __shared__ int sc[32];
    if (lane_id() == 0) sc[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += sc[w];
        cnt[(int64_t)L * gridDim.y + q] = t;
    }
}
__global__ void __launch_bounds__(512) k_cdf_write(const int64_t *__restrict__ blk, Layout Ly,
                                                   const int32_t *__restrict__ order, int nslots, int warmup,
                                                   const int64_t *__restrict__ off, double *__restrict__ out) {
    extern __shared__ int64_t ck[];                   // [pow2 >= MI] sort keys
    const int L = blockIdx.x, q = blockIdx.y;
    const int sl = q < nslots ? order[q] : -1;
    if (sl < 0) return;
    const int64_t *b = blk + (int64_t)sl * Ly.W;
    const int64_t r0 = warmup > 0 ? warmup : 0;
    __shared__ int64_t scan_sm[33];
    __shared__ int s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int64_t c0 = r0; c0 < Ly.MI; c0 += blockDim.x) {          // ordered compaction by rank
        const int64_t r = c0 + threadIdx.x;
        const int64_t *p = nullptr;
        const bool ok = r < Ly.MI && cdf_point(blk, Ly, sl, r, L, &p);
        int64_t tot;
        const int64_t pos = block_excl_sum<512>(ok ? 1 : 0, &tot, scan_sm) + s_n;
        if (ok) ck[pos] = p[1] * 4096 + r;
        __syncthreads();
        if (threadIdx.x == 0) s_n += (int)tot;
        __syncthreads();
    }
    const int n = s_n;
    if (n == 0) return;
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = n + threadIdx.x; i < n2; i += blockDim.x) ck[i] = INT64_MAX;
    __syncthreads();
    block_bitonic<int64_t>(ck, n2);
    const int64_t bmin = ck[0] >> 12;
    const int64_t o0 = off[(int64_t)L * gridDim.y + q];
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const int64_t busy = ck[k] >> 12, r = ck[k] & 4095;
        const int64_t *p = b + Ly.pt_off() + (r * Ly.L + L) * PT_W;
        double *o = out + (o0 + k) * 5;
        o[0] = L;
        o[1] = (double)b[0];
        o[2] = (double)busy / (double)bmin;
        o[3] = (double)p[3] / (double)busy;
        o[4] = (double)(k + 1) / (double)n;
    }
}

// O16 global: one block per cell; its values over the sampled (gpu, iteration) points of all gpus
// (iteration rows present, rank >= warmup; cells without instances are 0), median by bitonic sort
__global__ void __launch_bounds__(512) k_e2e(const int64_t *__restrict__ blk, Layout Ly, const int32_t *__restrict__ order,
                                             int nslots, int warmup, int64_t maxp2, int64_t *__restrict__ wk,
                                             double *__restrict__ out) {
    extern __shared__ int64_t esh[];
    const int k = blockIdx.x;                         // cell = P * 4 + {vec, gemm, fa, launch}
    int64_t *w = wk ? wk + (int64_t)k * maxp2 : esh;
    __shared__ int64_t scan_sm[33];
    __shared__ int s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    int nq = 0;
    while (nq < nslots && order[nq] >= 0) nq++;
    const int64_t r0 = warmup > 0 ? warmup : 0;
    const int64_t nr = Ly.MI > r0 ? Ly.MI - r0 : 0;
    const int64_t total = (int64_t)nq * nr;
    for (int64_t c0 = 0; c0 < total; c0 += blockDim.x) {
        const int64_t c = c0 + threadIdx.x;
        bool ok = false;
        int64_t v = 0;
        if (c < total) {
            const int64_t *b = blk + (int64_t)order[c / nr] * Ly.W;
            const int64_t r = r0 + c % nr;
            ok = b[1] != 0 && b[Ly.it_off() + r * IT_W] != 0;
            v = b[Ly.e2e_off() + r * E2E_W + k];
        }
        int64_t tot;
        const int64_t pos = block_excl_sum<512>(ok ? 1 : 0, &tot, scan_sm) + s_n;
        if (ok && pos < maxp2) w[pos] = v;
        __syncthreads();
        if (threadIdx.x == 0) s_n += (int)tot;
        __syncthreads();
    }
    const int n = s_n < maxp2 ? s_n : (int)maxp2;
    double m = NAN;
    if (n > 0) m = med_i64_s(w, n);
    if (threadIdx.x == 0) {
        out[1 + k] = m;
        if (k == 0) out[0] = n;
    }
}

// global iteration rows (a11): one thread per iteration rank of the reference gpu
struct GlobArgs {
    const int64_t *blk;
    int nslots;
    Layout Ly;
    const int32_t *slot_order;
    const int64_t *delta;
    int64_t tokens;              // b*s*R
    int warmup;
    int32_t *step, *complete, *sampled;
    int64_t *T, *af, *al;
    double *tp;
    int64_t *n_out;
    double *med;
    double *work;                // [pow2(MI)]
};

__global__ void __launch_bounds__(256) k_global(GlobArgs A) {
    const Layout Ly = A.Ly;
    __shared__ int s_ref;
    __shared__ int s_nst;
    if (threadIdx.x == 0) {
        s_ref = A.slot_order[0];
        s_nst = 0;
    }
    __syncthreads();
    const int ref = s_ref;
    if (ref < 0) { if (threadIdx.x == 0) { *A.n_out = 0; *A.med = NAN; } return; }
    const int64_t *rb = A.blk + (int64_t)ref * Ly.W;
    // per slot: are the step labels strictly increasing over its valid ranks?
    __shared__ int s_sorted[CH_MAX_GPUS];
    for (int q = threadIdx.x; q < A.nslots && q < CH_MAX_GPUS; q += blockDim.x) s_sorted[q] = 1;
    __syncthreads();
    for (int q = 0; q < A.nslots && q < CH_MAX_GPUS; q++) {
        int sl = A.slot_order[q];
        if (sl < 0) break;
        const int64_t *b = A.blk + (int64_t)sl * Ly.W + Ly.it_off();
        for (int64_t x = threadIdx.x; x < Ly.MI; x += blockDim.x) {
            if (!b[x * IT_W]) continue;
            int64_t y = x + 1;
            while (y < Ly.MI && !b[y * IT_W]) y++;
            if (y < Ly.MI && b[y * IT_W + 1] <= b[x * IT_W + 1]) s_sorted[q] = 0;
        }
    }
    __syncthreads();
    // reference rows are the valid ranks of the reference gpu in rank order; output index = count before
    __shared__ int widx[4096];
    __shared__ int64_t scan_sm[33];
    __shared__ int64_t s_base;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int64_t r0 = 0; r0 < Ly.MI && r0 < 4096; r0 += blockDim.x) {     // ordered compaction (block scan)
        int64_t r = r0 + threadIdx.x;
        bool v = r < Ly.MI && r < 4096 && rb[Ly.it_off() + r * IT_W] != 0;
        int64_t tot;
        int64_t ex = block_excl_sum<256>(v ? 1 : 0, &tot, scan_sm);
        if (r < Ly.MI && r < 4096) widx[r] = (int)(s_base + ex);
        __syncthreads();
        if (threadIdx.x == 0) s_base += tot;
        __syncthreads();
    }
    const int64_t nref_all = s_base;
    for (int64_t r = threadIdx.x; r < Ly.MI && r < 4096; r += blockDim.x) {
        const int64_t *row = rb + Ly.it_off() + r * IT_W;
        if (!row[0]) continue;
        int64_t w = widx[r];
        int64_t step = row[1];
        bool complete = true, samp = true;
        int64_t T = INT64_MIN, lo = INT64_MAX, hi = INT64_MIN;
        for (int q = 0; q < A.nslots; q++) {
            int sl = A.slot_order[q];
            if (sl < 0) break;
            const int64_t *b = A.blk + (int64_t)sl * Ly.W;
            if (!b[1]) continue;
            int g = (int)b[0];
            int64_t f = -1;
            // first iteration (rank order) of gpu g with the same step label (D5); iterations are
            // normally rank-aligned across gpus, so the scan is entered only when rank r differs
            // or an earlier rank carries the same step
            const int64_t *xr = b + Ly.it_off() + r * IT_W;
            if (q < CH_MAX_GPUS && s_sorted[q] && xr[0] && xr[1] == step) {
                f = r;      // steps strictly increasing over the gpu's ranks: rank r is the first match
            } else {
                for (int64_t x = 0; x < Ly.MI; x++)
                    if (b[Ly.it_off() + x * IT_W] && b[Ly.it_off() + x * IT_W + 1] == step) { f = x; break; }
            }
            if (f < 0) { complete = false; continue; }
            const int64_t *x = b + Ly.it_off() + f * IT_W;
            if (f < A.warmup) samp = false;
            int64_t t = x[2] + x[3] + x[4];
            if (t > T) T = t;
            if (x[5] > 0) {
                int64_t a = x[6] - A.delta[g], c = x[7] - A.delta[g];
                if (a < lo) lo = a;
                if (c > hi) hi = c;
            }
        }
        A.step[w] = (int32_t)step;
        A.complete[w] = complete;
        A.sampled[w] = complete && samp;
        A.T[w] = complete ? T : 0;
        A.af[w] = lo;
        A.al[w] = hi;
        A.tp[w] = complete ? (double)A.tokens / ((double)T * 1e-9) : NAN;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int64_t w0 = 0; w0 < nref_all; w0 += blockDim.x) {                 // sampled throughputs, in order
        int64_t w = w0 + threadIdx.x;
        bool v = w < nref_all && A.sampled[w];
        int64_t tot;
        int64_t ex = block_excl_sum<256>(v ? 1 : 0, &tot, scan_sm);
        if (v) A.work[s_base + ex] = A.tp[w];
        __syncthreads();
        if (threadIdx.x == 0) s_base += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *A.n_out = nref_all;
        s_nst = (int)s_base;
    }
    __syncthreads();
    int nst = s_nst;
    double m = NAN;
    if (nst > 0) m = med_f64_s(A.work, nst);
    if (threadIdx.x == 0) *A.med = m;
}

// ---- CPU utilization (R13) ------------------------------
constexpr int CPU_PHYS_MAX = 4096, CPU_PW = CPU_PHYS_MAX / 32;
struct CpuArgs {
    int64_t n;
    const int64_t *ts;
    const int32_t *core;
    const double *util;
    const int32_t *topo;
    int32_t n_logical;
};
// validation, timestamp heads (int64 flags for the scan) and the number of physical cores
__global__ void k_cpu_check(CpuArgs A, int64_t *__restrict__ head, unsigned int *__restrict__ bad,
                            int *__restrict__ n_phys) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < A.n_logical) {
        const int p = A.topo[k];
        if (p < 0 || p >= CPU_PHYS_MAX) atomicOr(bad, 1u);
        else atomicMax(n_phys, p + 1);
    }
    if (k >= A.n) return;
    const int64_t t = A.ts[k];
    const int c = A.core[k];
    const double u = A.util[k];
    bool ok = c >= 0 && c < A.n_logical && u >= 0.0 && u <= 100.0;
    if (k > 0) {
        const int64_t tp = A.ts[k - 1];
        if (t < tp || (t == tp && c <= A.core[k - 1])) ok = false;
    }
    if (!ok) atomicOr(bad, 1u);
    head[k] = (k == 0 || t != A.ts[k - 1]) ? 1 : 0;
}
__global__ void k_cpu_starts(const int64_t *__restrict__ head, const int64_t *__restrict__ ex, int64_t n,
                             int64_t *__restrict__ starts) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && head[k]) starts[ex[k]] = k;
    if (k == n - 1) starts[ex[k] + head[k]] = n;
}
// a warp per timestamp: C_active, C_min (lane 0, logical-core order), physical-core bitmaps
__global__ void __launch_bounds__(256) k_cpu_ts(CpuArgs A, const int64_t *__restrict__ starts,
                                                const int64_t *__restrict__ n_ts_d, const int *__restrict__ n_phys_d,
                                                int64_t *__restrict__ ca, double *__restrict__ cm,
                                                unsigned int *__restrict__ ever,
                                                unsigned long long *__restrict__ pairs,
                                                const unsigned int *__restrict__ bad) {
    __shared__ unsigned int b1[8][CPU_PW], b2[8][CPU_PW];
    if (*bad) return;                 // invalid samples: nothing is computed
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int nw = (*n_phys_d + 31) >> 5;
    const int64_t n_ts = *n_ts_d;
    for (int64_t q = (int64_t)blockIdx.x * 8 + w; q < n_ts; q += (int64_t)gridDim.x * 8) {
        for (int x = l; x < nw; x += 32) { b1[w][x] = 0u; b2[w][x] = 0u; }
        __syncwarp();
        const int64_t a = starts[q], b = starts[q + 1];
        int64_t act = 0;
        double s = 0.0;
        for (int64_t k0 = a; k0 < b; k0 += 32) {
            const int64_t k = k0 + l;
            const double u = k < b ? A.util[k] : 0.0;
            const bool on = k < b && u > 0.0;
            act += __popc(__ballot_sync(CH_FULL, on));
            // C_min = sum of Util_i / 100: the divisions in parallel, the sum in logical-core
            // order (every lane adds the same terms in the same order, so lane 0 holds the sequential sum)
            const double qd = u / 100.0;
            const int m = (int)min((int64_t)32, b - k0);
            for (int j = 0; j < m; j++) s += __shfl_sync(CH_FULL, qd, j);
            if (on) {
                const int p = A.topo[A.core[k]];
                const unsigned bit = 1u << (p & 31);
                const unsigned old = atomicOr(&b1[w][p >> 5], bit);
                if (old & bit) atomicOr(&b2[w][p >> 5], bit);
            }
        }
        __syncwarp();
        unsigned long long p1 = 0, p2 = 0;
        for (int x = l; x < nw; x += 32) {
            p1 += __popc(b1[w][x]);
            p2 += __popc(b2[w][x]);
            if (b1[w][x]) atomicOr(&ever[x], b1[w][x]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            p1 += __shfl_xor_sync(CH_FULL, p1, o);
            p2 += __shfl_xor_sync(CH_FULL, p2, o);
        }
        if (l == 0) {
            ca[q] = act;
            cm[q] = s;
            if (p1) atomicAdd(&pairs[0], p1);
            if (p2) atomicAdd(&pairs[1], p2);
        }
        __syncwarp();
    }
}
// medians (D21, block bitonic over pow2-padded work arrays), maxima, occupancy, SMT co-activity
__global__ void __launch_bounds__(512) k_cpu_summary(int64_t *__restrict__ ca, double *__restrict__ cm,
                                                     const int64_t *__restrict__ n_ts_d, const int *__restrict__ n_phys_d,
                                                     const unsigned int *__restrict__ ever,
                                                     const unsigned long long *__restrict__ pairs,
                                                     const unsigned int *__restrict__ bad, double *__restrict__ out) {
    __shared__ int64_t s_amax;
    __shared__ double s_mmax;
    __shared__ int s_occ;
    if (*bad) return;
    const int n = (int)*n_ts_d;
    const int n_phys = *n_phys_d;
    if (threadIdx.x == 0) { s_amax = 0; s_mmax = 0.0; s_occ = 0; }
    __syncthreads();
    int64_t am = 0;
    double mm = 0.0;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        am = ca[q] > am ? ca[q] : am;
        mm = cm[q] > mm ? cm[q] : mm;
    }
    atomicMax((unsigned long long *)&s_amax, (unsigned long long)am);
    atomicMax((unsigned long long *)&s_mmax, (unsigned long long)__double_as_longlong(mm));   // non-negative doubles
    for (int x = threadIdx.x; x < (n_phys + 31) / 32; x += blockDim.x) atomicAdd(&s_occ, __popc(ever[x]));
    __syncthreads();
    const double ma = n > 0 ? med_i64_s(ca, n) : NAN;
    const double mc = n > 0 ? med_f64_s(cm, n) : NAN;
    if (threadIdx.x == 0) {
        out[0] = n;
        out[1] = ma;
        out[2] = mc;
        out[3] = (double)s_amax;
        out[4] = n > 0 ? s_mmax : NAN;
        out[5] = n_phys > 0 ? (double)s_occ / (double)n_phys : NAN;
        out[6] = pairs[0] > 0 ? (double)pairs[1] / (double)pairs[0] : NAN;
    }
}
}  // namespace

static Layout layout_of(chopper_ctx *ctx) {
    Layout Ly;
    Ly.MI = std::max(1, ctx->cfg.max_iters);
    Ly.L = std::max(1, ctx->cfg.n_labels);
    Ly.C = ctx->C;
    Ly.W = HDR + Ly.C + IT_W * Ly.MI + PT_W * Ly.MI * Ly.L + E2E_W * Ly.MI;
    return Ly;
}

// dense local exchange blocks [slots][W]
static chopper_status densify(chopper_ctx *ctx, int64_t **blk_out, int *slots_out) {
    const Layout Ly = layout_of(ctx);
    const int slots = (int)ceil_div(ctx->cfg.n_traced_gpus, ctx->nranks);
    if (ctx->n_lg > slots) return ch_fail(ctx, CHOPPER_E_RANGE, "more local gpus than ceil(n_traced_gpus / nranks)");
    CH_ALLOC_BEGIN;
    int64_t *blk = CH_ALLOC(ctx, int64_t, (int64_t)slots * Ly.W);
    int32_t *lgg = CH_ALLOC(ctx, int32_t, ctx->n_lg + 1);
    int32_t *pres = CH_ALLOC(ctx, int32_t, (int64_t)std::max(ctx->n_lg, 1) * std::max(ctx->C, 1));
    unsigned int *ovf = CH_ALLOC(ctx, unsigned int, 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemsetAsync(blk, 0, 8 * (size_t)slots * Ly.W, ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(ovf, 0, 4, ctx->st));
    std::vector<int32_t> h(ctx->lg_gpu, ctx->lg_gpu + ctx->n_lg);
    std::vector<int32_t> hp((size_t)std::max(ctx->n_lg, 1) * std::max(ctx->C, 1), 0);
    for (size_t q = 0; q < ctx->present.size() && q < hp.size(); q++) hp[q] = ctx->present[q];
    if (ctx->n_lg) CH_CUDA(ctx, cudaMemcpyAsync(lgg, h.data(), 4 * ctx->n_lg, cudaMemcpyHostToDevice, ctx->st));
    CH_CUDA(ctx, cudaMemcpyAsync(pres, hp.data(), 4 * hp.size(), cudaMemcpyHostToDevice, ctx->st));
    if (ctx->n_lg > 0) {
        k_dense_header<<<ctx->n_lg, 64, 0, ctx->st>>>(blk, Ly, ctx->n_lg, lgg, ctx->d_has_smp, pres);
        CH_LAUNCHED(ctx);
    }
    if (ctx->iter.n > 0) {
        k_dense_iters<<<(unsigned)ceil_div(ctx->iter.n, 256), 256, 0, ctx->st>>>(
            blk, Ly, ctx->iter.n, ctx->iter.gpu, ctx->iter.rank, ctx->iter_step, ctx->iter.f, ctx->iter.cap,
            ctx->d_gpu_lg, ovf);
        CH_LAUNCHED(ctx);
    }
    if (ctx->point.n > 0) {
        const chopper_bd_params &p = ctx->bd;
        k_dense_points<<<(unsigned)ceil_div(ctx->point.n, 256), 256, 0, ctx->st>>>(
            blk, Ly, ctx->point.n, ctx->point.gpu, ctx->point.rank, ctx->point.label, ctx->point.f, ctx->point.cnt,
            ctx->point.cap, ctx->d_gpu_lg, p.slot_gpu_cycles, p.slot_perf_flops, p.slot_util_num, p.slot_util_den,
            ovf);
        CH_LAUNCHED(ctx);
    }
    if (ctx->inst.n > 0 && ctx->cfg.n_labels > 0) {
        const int64_t slots = (int64_t)148 * 8 * 256;   // threads of a full grid
        const int kk = (int)std::max<int64_t>(1, std::min<int64_t>(E2E_KMAX, ctx->inst.n / slots));
        k_dense_e2e<<<(unsigned)std::min<int64_t>(ceil_div(ctx->inst.n, 256 * kk), 148 * 8), 256, 0, ctx->st>>>(
            blk, Ly, ctx->inst.n_dev, ctx->inst.gpu, ctx->inst.rank, ctx->inst.ph, ctx->inst.label, ctx->inst.f,
            ctx->inst.cap, ctx->d_gpu_lg, ctx->sp.label, ctx->d_op_type, kk);
        CH_LAUNCHED(ctx);
    }
    ctx->d_dense_ovf = ovf;     // checked at chopper_reduce_ranks' read-back (no round trip here)
    *blk_out = blk;
    *slots_out = slots;
    return CHOPPER_OK;
}

static chopper_status run_breakdown(chopper_ctx *ctx, const int64_t *blk, int nslots, const int32_t *slot_order,
                                    double **out_dev, int64_t *n_out) {
    const Layout Ly = layout_of(ctx);
    std::vector<int32_t> labs;
    for (int L = 0; L < (int)ctx->op_type.size(); L++)
        if (ctx->op_type[L] == 1 || ctx->op_type[L] == 2) labs.push_back(L);
    int nb = (int)labs.size();
    *n_out = nb;
    CH_ALLOC_BEGIN;
    double *out = CH_ALLOC(ctx, double, (int64_t)std::max(nb, 1) * 16);
    int32_t *dl = CH_ALLOC(ctx, int32_t, std::max(nb, 1));
    int64_t maxp = (int64_t)Ly.MI * ctx->cfg.n_traced_gpus;
    int64_t maxp2 = 1;
    while (maxp2 < maxp) maxp2 <<= 1;
    size_t shb = (size_t)16 * maxp2;     // work array + second operand of the fit
    bool use_smem = shb <= 64 * 1024;
    int64_t *wi = use_smem ? nullptr : CH_ALLOC(ctx, int64_t, (int64_t)std::max(nb, 1) * BD_TASKS * 2 * maxp2);
    double *res = CH_ALLOC(ctx, double, (int64_t)std::max(nb, 1) * BD_TASKS * 4);
    CH_ALLOC_END(ctx);
    *out_dev = out;
    if (nb == 0) return CHOPPER_OK;
    CH_CUDA(ctx, cudaMemcpyAsync(dl, labs.data(), 4 * nb, cudaMemcpyHostToDevice, ctx->st));
    BdArgs A;
    A.blk = blk;
    A.nslots = nslots;
    A.Ly = Ly;
    A.slot_order = slot_order;
    A.labels = dl;
    A.f_gemm = ctx->d_f_gemm;
    A.tpt = ctx->bd.tpt_peak;
    A.freq = ctx->bd.freq_peak_hz;
    A.warmup = ctx->bd.warmup;
    A.s_cyc = ctx->bd.slot_gpu_cycles;
    A.s_fl = ctx->bd.slot_perf_flops;
    A.s_un = ctx->bd.slot_util_num;
    A.s_ud = ctx->bd.slot_util_den;
    A.maxp2 = maxp2;
    A.wi = wi;
    A.res = res;
    A.out = out;
    A.use_smem = use_smem;
    static bool attr = false;
    if (!attr) {
        CH_CUDA(ctx, cudaFuncSetAttribute(k_breakdown, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        attr = true;
    }
    k_breakdown<<<dim3(nb, BD_TASKS), 512, use_smem ? shb : 0, ctx->st>>>(A);
    CH_LAUNCHED(ctx);
    k_bd_compose<<<(unsigned)ceil_div(nb, 64), 64, 0, ctx->st>>>(A, nb);
    CH_LAUNCHED(ctx);
    return CHOPPER_OK;
}

// slot order by gpu id (host, from the exchange headers)
// slot order by gpu id, on the device: slot b (present) goes to position #{present slots with a smaller
// (gpu, slot)}; the rest of the order array is -1
// (a slot whose gpu field is -1 is a failed rank's block, ch_exchange_poison: *poison is set)
__global__ void k_slot_order(const int64_t *__restrict__ blk, int nslots, int64_t W, int32_t *__restrict__ order,
                             unsigned int *__restrict__ poison) {
    for (int b = threadIdx.x; b <= nslots; b += blockDim.x) order[b] = -1;
    __syncthreads();
    for (int b = threadIdx.x; b < nslots; b += blockDim.x) {
        const int64_t *x = blk + (int64_t)b * W;
        if (poison && x[0] == -1) *poison = 1u;
        if (!x[1]) continue;
        const int64_t g = x[0];
        int r = 0;
        for (int c = 0; c < nslots; c++) {
            const int64_t *y = blk + (int64_t)c * W;
            if (y[1] && (y[0] < g || (y[0] == g && c < b))) r++;
        }
        order[r] = b;
    }
}

static chopper_status slot_order(chopper_ctx *ctx, const int64_t *blk, int nslots, int64_t W, int32_t **out,
                                 unsigned int *poison = nullptr) {
    CH_ALLOC_BEGIN;
    int32_t *d = CH_ALLOC(ctx, int32_t, nslots + 1);
    CH_ALLOC_END(ctx);
    k_slot_order<<<1, 256, 0, ctx->st>>>(blk, nslots, W, d, poison);
    CH_LAUNCHED(ctx);
    *out = d;
    return CHOPPER_OK;
}

int64_t ch_dense_width(chopper_ctx *ctx) { return layout_of(ctx).W; }

chopper_status ch_breakdown_local(chopper_ctx *ctx) {
    int64_t *blk;
    int slots;
    CH_TRY(densify(ctx, &blk, &slots));
    ctx->d_dense = blk;
    ctx->dense_slots = slots;
    int32_t *ord;
    CH_TRY(slot_order(ctx, blk, slots, layout_of(ctx).W, &ord));
    CH_TRY(run_breakdown(ctx, blk, slots, ord, &ctx->d_bd, &ctx->n_bd));
    return CHOPPER_OK;
}

chopper_status ch_reduce_ranks(chopper_ctx *ctx, chopper_global *out) {
    const Layout Ly = layout_of(ctx);
    const int slots = ctx->dense_slots;
    const int nslots = slots * ctx->nranks;
    CH_ALLOC_BEGIN;
    int64_t *all = CH_ALLOC(ctx, int64_t, (int64_t)nslots * Ly.W);
    unsigned int *poison = CH_ALLOC(ctx, unsigned int, 1);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemsetAsync(poison, 0, 4, ctx->st));
    if (ctx->nranks > 1) {
        ctx->d_exchanged = true;
        CH_TRY(ch_nccl_allgather(ctx, ctx->d_dense, all, sizeof(int64_t) * (size_t)slots * Ly.W));
    } else {
        all = ctx->d_dense;                   // one rank: the gathered block is the local one (read only from here)
    }
    int32_t *ord;
    CH_TRY(slot_order(ctx, all, nslots, Ly.W, &ord, poison));
    ctx->d_all = all;
    ctx->d_all_order = ord;
    ctx->all_slots = nslots;
    // global iterations + throughput
    int64_t MI = Ly.MI;
    int64_t mi2 = 1;
    while (mi2 < MI) mi2 <<= 1;
    int32_t *step = CH_ALLOC(ctx, int32_t, MI), *comp = CH_ALLOC(ctx, int32_t, MI), *samp = CH_ALLOC(ctx, int32_t, MI);
    int64_t *T = CH_ALLOC(ctx, int64_t, MI), *af = CH_ALLOC(ctx, int64_t, MI), *al = CH_ALLOC(ctx, int64_t, MI);
    double *tp = CH_ALLOC(ctx, double, MI), *work = CH_ALLOC(ctx, double, mi2), *med = CH_ALLOC(ctx, double, 1);
    int64_t *nref = CH_ALLOC(ctx, int64_t, 1);
    int64_t *dd = CH_ALLOC(ctx, int64_t, ctx->cfg.n_traced_gpus);
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemcpyAsync(dd, ctx->delta.data(), 8 * ctx->cfg.n_traced_gpus, cudaMemcpyHostToDevice, ctx->st));
    GlobArgs G;
    G.blk = all;
    G.nslots = nslots;
    G.Ly = Ly;
    G.slot_order = ord;
    G.delta = dd;
    G.tokens = ctx->bd.batch * ctx->bd.seq * ctx->bd.ranks;
    G.warmup = ctx->bd.warmup;
    G.step = step; G.complete = comp; G.sampled = samp; G.T = T; G.af = af; G.al = al; G.tp = tp;
    G.n_out = nref; G.med = med; G.work = work;
    // the global rows, the report statistics and the end-to-end medians are independent small kernels: they
    // run on side streams, concurrently with the breakdown on the ctx stream (joined before the copies)
    CH_CUDA(ctx, cudaEventRecord(ctx->fork_ev, ctx->st));
    for (int q = 0; q < 3; q++) CH_CUDA(ctx, cudaStreamWaitEvent(ctx->side[q], ctx->fork_ev, 0));
    k_global<<<1, 256, 0, ctx->side[0]>>>(G);
    CH_LAUNCHED(ctx);
    double *bd;
    int64_t nbd;
    if (ctx->nranks == 1 && ctx->d_bd) {
        // one rank: the gathered block is the local one, so the global breakdown is the local one (same kernels on
        // the same block, computed in chopper_breakdown) -- reused, not recomputed
        bd = ctx->d_bd;
        nbd = ctx->n_bd;
    } else {
        CH_TRY(run_breakdown(ctx, all, nslots, ord, &bd, &nbd));
    }
    // report statistics per op label (O14)
    const int nL = ctx->cfg.n_labels;
    double *rep = nullptr;
    if (nL > 0) {
        int64_t maxp = (int64_t)Ly.MI * ctx->cfg.n_traced_gpus, maxp2 = 1;
        while (maxp2 < maxp) maxp2 <<= 1;
        const size_t shb = (size_t)4 * 8 * maxp2;
        const bool use_smem = shb <= 96 * 1024;
        CH_ALLOC_BEGIN;
        rep = CH_ALLOC(ctx, double, (int64_t)nL * 16);
        double *wk = use_smem ? nullptr : CH_ALLOC(ctx, double, (int64_t)nL * 4 * maxp2);
        CH_ALLOC_END(ctx);
        static bool rattr = false;
        if (!rattr) {
            CH_CUDA(ctx, cudaFuncSetAttribute(k_report, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            rattr = true;
        }
        RepArgs RA{all, nslots, Ly, ord, ctx->bd.warmup, maxp2, wk, rep, use_smem ? 1 : 0};
        k_report<<<nL, 512, use_smem ? shb : 0, ctx->side[1]>>>(RA);
        CH_LAUNCHED(ctx);
    }
    // end-to-end phase x op-type medians (O16)
    double *e2e = nullptr;
    {
        int64_t maxp = (int64_t)Ly.MI * ctx->cfg.n_traced_gpus, maxp2 = 1;
        while (maxp2 < maxp) maxp2 <<= 1;
        const bool sm_ok = 8 * maxp2 <= 48 * 1024;
        CH_ALLOC_BEGIN;
        e2e = CH_ALLOC(ctx, double, 1 + E2E_W);
        int64_t *wk = sm_ok ? nullptr : CH_ALLOC(ctx, int64_t, (int64_t)E2E_W * maxp2);
        CH_ALLOC_END(ctx);
        k_e2e<<<E2E_W, 512, sm_ok ? 8 * maxp2 : 0, ctx->side[2]>>>(all, Ly, ord, nslots, ctx->bd.warmup, maxp2, wk, e2e);
        CH_LAUNCHED(ctx);
    }
    for (int q = 0; q < 3; q++) {
        CH_CUDA(ctx, cudaEventRecord(ctx->join_ev[q], ctx->side[q]));
        CH_CUDA(ctx, cudaStreamWaitEvent(ctx->st, ctx->join_ev[q], 0));
    }
    // host copies
    int64_t n = 0;
    unsigned int hovf = 0, hpoison = 0;
    if (ctx->d_dense_ovf) CH_CUDA(ctx, ch_d2h(ctx, &hovf, ctx->d_dense_ovf, 4));
    // one read-back: every array at its capacity (max_iters entries, at most 4096), the counts with it
    if (nbd > 256) return ch_fail(ctx, CHOPPER_E_RANGE, "more than 256 breakdown rows");
    if (nL > 256) return ch_fail(ctx, CHOPPER_E_RANGE, "more than 256 op labels in the report rows");
    const int64_t mc = std::min<int64_t>(MI, 4096);
    CH_CUDA(ctx, ch_d2h(ctx, &n, nref, 8));
    CH_CUDA(ctx, ch_d2h(ctx, &hpoison, poison, 4));
    CH_CUDA(ctx, ch_d2h(ctx, out->step, step, 4 * mc));
    CH_CUDA(ctx, ch_d2h(ctx, out->complete, comp, 4 * mc));
    CH_CUDA(ctx, ch_d2h(ctx, out->sampled, samp, 4 * mc));
    CH_CUDA(ctx, ch_d2h(ctx, out->T, T, 8 * mc));
    CH_CUDA(ctx, ch_d2h(ctx, out->aligned_first, af, 8 * mc));
    CH_CUDA(ctx, ch_d2h(ctx, out->aligned_last, al, 8 * mc));
    CH_CUDA(ctx, ch_d2h(ctx, out->throughput, tp, 8 * mc));
    CH_CUDA(ctx, ch_d2h(ctx, &out->throughput_median, med, 8));
    if (nbd > 0) CH_CUDA(ctx, ch_d2h(ctx, out->bd, bd, 8 * 16 * nbd));
    CH_CUDA(ctx, ch_d2h(ctx, out->e2e, e2e, 8 * (1 + E2E_W)));
    if (nL > 0) CH_CUDA(ctx, ch_d2h(ctx, out->report, rep, 8 * 16 * (size_t)nL));
    CH_CUDA(ctx, ch_sync(ctx));
    if (hpoison) return ch_fail(ctx, CHOPPER_E_STATE, "a peer rank failed earlier in this step (all-gather #2)");
    if (n > mc) return ch_fail(ctx, CHOPPER_E_RANGE, "more iterations than max_iters (or 4096) in chopper_global");
    if (hovf) return ch_fail(ctx, CHOPPER_E_RANGE, "iteration rank >= max_iters or op label >= n_labels");
    out->n_iters = n;
    out->n_bd = nbd;
    out->n_report = nL;
    for (int g = 0; g < ctx->cfg.n_traced_gpus && g < 256; g++) {
        out->delta[g] = ctx->delta[g];
        out->delta_flag[g] = ctx->delta_flag[g];
    }
    out->max_skew_ag = ctx->max_skew[0];
    out->max_skew_rs = ctx->max_skew[1];
    return CHOPPER_OK;
}

chopper_status ch_report_cdf(chopper_ctx *ctx, double *out, int64_t cap, int64_t *n_rows) {
    const Layout Ly = layout_of(ctx);
    const int nL = ctx->cfg.n_labels, nslots = ctx->all_slots;
    *n_rows = 0;
    if (nL <= 0 || nslots <= 0 || !ctx->d_all) return CHOPPER_OK;
    if (Ly.MI > 4096) return ch_fail(ctx, CHOPPER_E_RANGE, "max_iters > 4096 in chopper_report_cdf");
    const int64_t cells = (int64_t)nL * nslots;
    size_t mark = ctx->used;
    CH_ALLOC_BEGIN;
    int64_t *cnt = CH_ALLOC(ctx, int64_t, cells), *off = CH_ALLOC(ctx, int64_t, cells), *tot = CH_ALLOC(ctx, int64_t, 1);
    double *rows = CH_ALLOC(ctx, double, (int64_t)nL * nslots * Ly.MI * 5);
    CH_ALLOC_END(ctx);
    k_cdf_count<<<dim3(nL, nslots), 256, 0, ctx->st>>>(ctx->d_all, Ly, ctx->d_all_order, nslots, ctx->bd.warmup, cnt);
    CH_LAUNCHED(ctx);
    CH_TRY(ch_scan_excl_i64(ctx, cnt, off, cells, tot));
    int64_t mi2 = 1;
    while (mi2 < Ly.MI) mi2 <<= 1;
    static bool attr = false;
    if (!attr) {
        CH_CUDA(ctx, cudaFuncSetAttribute(k_cdf_write, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024));
        attr = true;
    }
    k_cdf_write<<<dim3(nL, nslots), 512, 8 * mi2, ctx->st>>>(ctx->d_all, Ly, ctx->d_all_order, nslots, ctx->bd.warmup,
                                                             off, rows);
    CH_LAUNCHED(ctx);
    int64_t n = 0;
    CH_CUDA(ctx, ch_d2h(ctx, &n, tot, 8));
    CH_CUDA(ctx, ch_sync(ctx));
    const int64_t m = n < cap ? n : cap;
    if (m > 0 && out) CH_CUDA(ctx, cudaMemcpy(out, rows, 8 * 5 * (size_t)m, cudaMemcpyDeviceToHost));
    ctx->used = mark;
    *n_rows = n;
    return CHOPPER_OK;
}

chopper_status ch_cpu_util(chopper_ctx *ctx, const chopper_cpu_samples *S, const int32_t *topology, int32_t n_logical,
                           int64_t *c_active, double *c_min, int64_t cap, chopper_cpu_summary *out) {
    // sizes from the sample count (n_ts <= n): one host synchronization, at the end
    const int64_t n = S->n;
    int64_t p2 = 1;
    while (p2 < std::max<int64_t>(n, 1)) p2 <<= 1;
    if (p2 > (1ll << 30)) return ch_fail(ctx, CHOPPER_E_RANGE, "too many CPU samples");
    const size_t mark = ctx->used;
    CH_ALLOC_BEGIN;
    int64_t *head = CH_ALLOC(ctx, int64_t, n + 1), *ex = CH_ALLOC(ctx, int64_t, n + 1);
    int64_t *starts = CH_ALLOC(ctx, int64_t, n + 2), *n_ts_d = CH_ALLOC(ctx, int64_t, 1);
    int64_t *ca = CH_ALLOC(ctx, int64_t, p2);
    double *cm = CH_ALLOC(ctx, double, p2);
    unsigned int *ever = CH_ALLOC(ctx, unsigned int, CPU_PW);
    unsigned long long *pairs = CH_ALLOC(ctx, unsigned long long, 2);
    double *dsum = CH_ALLOC(ctx, double, 8);
    unsigned int *bad = CH_ALLOC(ctx, unsigned int, 2);      // [0] bad, [1] n_physical
    CH_ALLOC_END(ctx);
    CpuArgs A{n, S->ts_ns, S->logical_core, S->util_pct, topology, n_logical};
    CH_CUDA(ctx, cudaMemsetAsync(bad, 0, 8, ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(ever, 0, 4 * CPU_PW, ctx->st));
    CH_CUDA(ctx, cudaMemsetAsync(pairs, 0, 16, ctx->st));
    int *nph = reinterpret_cast<int *>(bad + 1);
    const int64_t m = std::max<int64_t>(n, n_logical);
    k_cpu_check<<<(unsigned)ceil_div(std::max<int64_t>(m, 1), 256), 256, 0, ctx->st>>>(A, head, bad, nph);
    CH_LAUNCHED(ctx);
    if (n > 0) {
        CH_TRY(ch_scan_excl_i64(ctx, head, ex, n, n_ts_d));
        k_cpu_starts<<<(unsigned)ceil_div(n, 256), 256, 0, ctx->st>>>(head, ex, n, starts);
        CH_LAUNCHED(ctx);
        k_cpu_ts<<<(unsigned)std::min<int64_t>(ceil_div(n, 8), 148 * 8), 256, 0, ctx->st>>>(A, starts, n_ts_d, nph, ca, cm,
                                                                                           ever, pairs, bad);
        CH_LAUNCHED(ctx);
        if (c_active && cap > 0) CH_CUDA(ctx, cudaMemcpyAsync(c_active, ca, 8 * std::min(cap, n), cudaMemcpyDeviceToDevice, ctx->st));
        if (c_min && cap > 0) CH_CUDA(ctx, cudaMemcpyAsync(c_min, cm, 8 * std::min(cap, n), cudaMemcpyDeviceToDevice, ctx->st));
    } else {
        CH_CUDA(ctx, cudaMemsetAsync(n_ts_d, 0, 8, ctx->st));
    }
    k_cpu_summary<<<1, 512, 0, ctx->st>>>(ca, cm, n_ts_d, nph, ever, pairs, bad, dsum);
    CH_LAUNCHED(ctx);
    double h[8];
    unsigned int hb[2];
    CH_CUDA(ctx, ch_d2h(ctx, h, dsum, 8 * 7));
    CH_CUDA(ctx, ch_d2h(ctx, hb, bad, 8));
    CH_CUDA(ctx, ch_sync(ctx));
    ctx->used = mark;
    if (hb[0]) return ch_fail(ctx, CHOPPER_E_VALIDATION, "CPU samples unsorted or out of range, or a bad topology entry");
    out->n_ts = (int64_t)h[0];
    out->n_logical = n_logical;
    out->n_physical = (int32_t)hb[1];
    out->c_active_median = h[1];
    out->c_min_median = h[2];
    out->c_active_max = h[3];
    out->c_min_max = h[4];
    out->physical_occupancy = h[5];
    out->smt_coactive = h[6];
    return CHOPPER_OK;
}
