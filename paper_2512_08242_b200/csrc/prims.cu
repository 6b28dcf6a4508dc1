// prims.cu -- device-wide primitives written for this library: exclusive /
// segmented scans and a stable LSD radix sort (8-bit digits, warp-match
// ranking).  Used by the a2 timestamp sort, span push-order sort, sub-run
// grouping and the union / sample prefix builders.
#include "common.cuh"

namespace {
constexpr int SC_NT = 256, SC_IPT = 8, SC_TILE = SC_NT * SC_IPT;

__global__ void k_tile_sums(const int64_t *__restrict__ in, int64_t n, int64_t *__restrict__ sums) {
    __shared__ int64_t sm[33];
    int64_t base = (int64_t)blockIdx.x * SC_TILE;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < SC_IPT; k++) {
        int64_t i = base + (int64_t)k * SC_NT + threadIdx.x;
        if (i < n) s += in[i];
    }
    int64_t tot;
    block_excl_sum<SC_NT>(s, &tot, sm);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void k_tile_apply(const int64_t *__restrict__ in, int64_t n, const int64_t *__restrict__ offs,
                             int64_t *__restrict__ out, int64_t *total_dev) {
    __shared__ int64_t sm[33];
    int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
    int64_t v[SC_IPT];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < SC_IPT; k++) {
        int64_t i = base + k;
        v[k] = i < n ? in[i] : 0;
        s += v[k];
    }
    int64_t tot;
    int64_t ex = block_excl_sum<SC_NT>(s, &tot, sm) + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
    for (int k = 0; k < SC_IPT; k++) {
        int64_t i = base + k;
        if (i < n) out[i] = ex;
        ex += v[k];
    }
    if (total_dev && blockIdx.x == gridDim.x - 1 && threadIdx.x == SC_NT - 1) *total_dev = ex;
}

// single-pass exclusive scan (chained scan with decoupled look-back): tiles are taken in launch order
// through a ticket, each publishes its aggregate, then its inclusive prefix once the predecessors' are
// known; one launch per scan instead of tile-sums + recursive scan + apply.
constexpr unsigned long long SP_A = 1ull << 62, SP_P = 2ull << 62, SP_MASK = (1ull << 62) - 1;
__global__ void __launch_bounds__(SC_NT) k_scan_1pass(const int64_t *__restrict__ in, int64_t n,
                                                      int64_t *__restrict__ out, int64_t *total_dev,
                                                      unsigned long long *__restrict__ state,
                                                      unsigned int *__restrict__ ticket) {
    __shared__ int64_t sm[33];
    __shared__ int64_t s_tile, s_excl;
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
    int64_t v[SC_IPT];
    int64_t tsum = 0;
#pragma unroll
    for (int k = 0; k < SC_IPT; k++) {
        v[k] = base + k < n ? in[base + k] : 0;
        tsum += v[k];
    }
    int64_t tot;
    int64_t ex = block_excl_sum<SC_NT>(tsum, &tot, sm);
    const int lane = lane_id();
    if (threadIdx.x < 32) {
        int64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&state[0], SP_P | (unsigned long long)tot);
        } else {
            if (lane == 0) atomicExch(&state[tile], SP_A | (unsigned long long)tot);
            int64_t p = tile - 1 - lane;
            while (true) {
                unsigned long long st = SP_P;
                if (p >= 0) st = *((volatile unsigned long long *)&state[p]);
                const unsigned fl = (unsigned)(st >> 62);
                const unsigned pm = __ballot_sync(CH_FULL, fl == 2u), zm = __ballot_sync(CH_FULL, fl == 0u);
                const int fp = pm ? __ffs(pm) - 1 : 32;
                const unsigned need = fp >= 31 ? CH_FULL : ((2u << fp) - 1u);
                if (zm & need) continue;
                int64_t x = lane <= fp ? (int64_t)(st & SP_MASK) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(CH_FULL, x, o);
                excl += x;
                if (fp < 32) break;
                p -= 32;
            }
            if (lane == 0) atomicExch(&state[tile], SP_P | (unsigned long long)(excl + tot));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    ex += s_excl;
#pragma unroll
    for (int k = 0; k < SC_IPT; k++) {
        if (base + k < n) out[base + k] = ex;
        ex += v[k];
    }
    if (total_dev && tile == (int64_t)gridDim.x - 1 && threadIdx.x == SC_NT - 1) *total_dev = ex;
}

// ---- segmented scans: aggregate (head seen, value since last head) ------------------------------
template <int OP>
__device__ __forceinline__ int64_t op_comb(int64_t a, int64_t b) {
    if (OP == 1) return a > b ? a : b;
    return a + b;
}
template <int OP>
__device__ __forceinline__ int64_t op_id() { return OP == 1 ? INT64_MIN : 0; }

// (head, value) pair scan: (h1,v1) (+) (h2,v2) = (h1|h2, h2 ? v2 : v1 op v2)
template <int OP>
__device__ __forceinline__ void pair_comb(uint32_t &h, int64_t &v, uint32_t h2, int64_t v2) {
    v = h2 ? v2 : op_comb<OP>(v, v2);
    h |= h2;
}
// block-wide exclusive pair scan (blockDim = SC_NT); returns the exclusive prefix of this thread,
// *tot_h / *tot_v get the block aggregate
template <int OP>
__device__ __forceinline__ void block_pair_excl(uint32_t h, int64_t v, uint32_t *eh, int64_t *ev, uint32_t *th,
                                                int64_t *tv) {
    __shared__ int64_t wv[SC_NT / 32];
    __shared__ uint32_t wh[SC_NT / 32];
    int l = lane_id(), w = threadIdx.x >> 5;
    uint32_t ih = h;
    int64_t iv = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t yh = __shfl_up_sync(CH_FULL, ih, o);
        int64_t yv = __shfl_up_sync(CH_FULL, iv, o);
        if (l >= o) {   // (y) (+) (this)
            uint32_t nh = yh;
            int64_t nv = yv;
            pair_comb<OP>(nh, nv, ih, iv);
            ih = nh;
            iv = nv;
        }
    }
    if (l == 31) { wh[w] = ih; wv[w] = iv; }
    __syncthreads();
    uint32_t ph = 0;
    int64_t pv = op_id<OP>();
    for (int q = 0; q < w; q++) pair_comb<OP>(ph, pv, wh[q], wv[q]);
    // exclusive of this thread = (warp prefix) (+) (lanes before)
    uint32_t xh = __shfl_up_sync(CH_FULL, ih, 1);
    int64_t xv = __shfl_up_sync(CH_FULL, iv, 1);
    uint32_t eh2 = ph;
    int64_t ev2 = pv;
    if (l > 0) pair_comb<OP>(eh2, ev2, xh, xv);
    *eh = eh2;
    *ev = ev2;
    uint32_t ah = 0;
    int64_t av = op_id<OP>();
    for (int q = 0; q < SC_NT / 32; q++) pair_comb<OP>(ah, av, wh[q], wv[q]);
    *th = ah;
    *tv = av;
    __syncthreads();
}

template <int OP>
__global__ void __launch_bounds__(SC_NT) k_seg_tile_agg(const int64_t *__restrict__ in, const uint8_t *__restrict__ head,
                                                        int64_t n, int64_t *__restrict__ agg_v, uint8_t *__restrict__ agg_h) {
    int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
    int64_t v = op_id<OP>();
    uint32_t h = 0;
    for (int k = 0; k < SC_IPT; k++) {
        int64_t i = base + k;
        if (i >= n) break;
        if (head[i]) { v = op_id<OP>(); h = 1; }
        v = op_comb<OP>(v, in[i]);
    }
    uint32_t eh, th;
    int64_t ev, tv;
    block_pair_excl<OP>(h, v, &eh, &ev, &th, &tv);
    if (threadIdx.x == 0) { agg_v[blockIdx.x] = tv; agg_h[blockIdx.x] = (uint8_t)th; }
}

// carry of tile t = inclusive pair scan of the aggregates up to t-1
__global__ void k_shift_carry(const int64_t *__restrict__ incl, int64_t ntile, int64_t ident, int64_t *__restrict__ carry) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < ntile) carry[t] = t > 0 ? incl[t - 1] : ident;
}

template <int OP, bool EXCL>
__global__ void __launch_bounds__(SC_NT) k_seg_apply(const int64_t *__restrict__ in, const uint8_t *__restrict__ head,
                                                     int64_t n, const int64_t *__restrict__ carry,
                                                     int64_t *__restrict__ out) {
    int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
    int64_t v = op_id<OP>();
    uint32_t h = 0;
    for (int k = 0; k < SC_IPT; k++) {
        int64_t i = base + k;
        if (i >= n) break;
        if (head[i]) { v = op_id<OP>(); h = 1; }
        v = op_comb<OP>(v, in[i]);
    }
    uint32_t eh, th;
    int64_t ev, tv;
    block_pair_excl<OP>(h, v, &eh, &ev, &th, &tv);
    int64_t c = eh ? ev : op_comb<OP>(carry ? carry[blockIdx.x] : op_id<OP>(), ev);
    for (int k = 0; k < SC_IPT; k++) {
        int64_t i = base + k;
        if (i >= n) break;
        if (head[i]) c = op_id<OP>();
        if (EXCL) { out[i] = c; c = op_comb<OP>(c, in[i]); }
        else { c = op_comb<OP>(c, in[i]); out[i] = c; }
    }
}

// ---- radix sort ---------------------------------------------------------------------------------
constexpr int RX_NT = 256, RX_WARPS = RX_NT / 32, RX_ROUNDS = 8, RX_TILE = RX_NT * RX_ROUNDS;

struct KeyArr {
    const unsigned long long *k;
    int shift;
    __device__ __forceinline__ int digit(int64_t i) const { return (int)((k[i] >> shift) & 0xFFu); }
};
struct KeyMeta {  // partition digit: bucket = lg * NG + dense group (a2 fast path)
    const uint32_t *meta;
    const int32_t *gpu_lg;
    int NG, other;
    __device__ __forceinline__ int digit(int64_t i) const {
        uint32_t m = meta[i];
        int k = kind_of(m), g;
        if (is_comm(k)) g = 0;
        else if (k == CK_COMPUTE) g = 1 + stream_of(m);
        else g = other;
        return gpu_lg[gpu_of(m)] * NG + g;
    }
};

template <class KS>
__global__ void __launch_bounds__(RX_NT) k_rx_upsweep(KS ks, int64_t n, int64_t *__restrict__ counts,
                                                      int64_t ntile) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * RX_TILE;
    for (int r = 0; r < RX_ROUNDS; r++) {
        int64_t i = base + (int64_t)r * RX_NT + threadIdx.x;
        if (i < n) atomicAdd(&h[ks.digit(i)], 1u);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * ntile + blockIdx.x] = (int64_t)h[threadIdx.x];   // (int64: scanned directly)
}

template <class KS, bool HAS_KEYS, bool HAS_VALS>
__global__ void __launch_bounds__(RX_NT) k_rx_downsweep(KS ks, const unsigned long long *__restrict__ keys_in,
                                                        const uint32_t *__restrict__ vals_in, int64_t n,
                                                        const int64_t *__restrict__ offs, int64_t ntile,
                                                        unsigned long long *__restrict__ keys_out,
                                                        uint32_t *__restrict__ vals_out) {
    __shared__ unsigned int wh[RX_WARPS][256];
    __shared__ int64_t goff[256];
    int w = threadIdx.x >> 5, l = lane_id();
    for (int d = threadIdx.x; d < 256 * RX_WARPS; d += RX_NT) (&wh[0][0])[d] = 0;
    goff[threadIdx.x] = offs[(int64_t)threadIdx.x * ntile + blockIdx.x];
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * RX_TILE + (int64_t)w * (32 * RX_ROUNDS);
    int dg[RX_ROUNDS];
    unsigned int rk[RX_ROUNDS];
    unsigned lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < RX_ROUNDS; r++) {
        int64_t i = base + r * 32 + l;
        bool valid = i < n;
        int d = valid ? ks.digit(i) : 256 + l;
        unsigned mm = __match_any_sync(CH_FULL, d);
        unsigned int before = valid ? wh[w][d] : 0;
        __syncwarp();
        if (valid && (mm & lt) == 0) wh[w][d] = before + __popc(mm);
        __syncwarp();
        dg[r] = d;
        rk[r] = before + __popc(mm & lt);
    }
    __syncthreads();
    unsigned int run = 0;
    {   // exclusive prefix over warps, per digit (thread = digit)
        for (int q = 0; q < RX_WARPS; q++) {
            unsigned int c = wh[q][threadIdx.x];
            wh[q][threadIdx.x] = run;
            run += c;
        }
    }
    // tile-local start of every digit: exclusive scan of the per-digit tile counts
    __shared__ int64_t sc[33];
    __shared__ int tstart[256];
    int64_t ttot;
    tstart[threadIdx.x] = (int)block_excl_sum<RX_NT>((int64_t)run, &ttot, sc);
    __syncthreads();
    // stage the tile in shared memory in (digit, input) order, then write each digit bucket coalesced
    __shared__ unsigned long long sk[HAS_KEYS ? RX_TILE : 1];
    __shared__ uint32_t sv[RX_TILE];
    __shared__ uint8_t sd[RX_TILE];
#pragma unroll
    for (int r = 0; r < RX_ROUNDS; r++) {
        int64_t i = base + r * 32 + l;
        if (i < n) {
            int d = dg[r];
            int loc = tstart[d] + (int)wh[w][d] + (int)rk[r];
            if (HAS_KEYS) sk[loc] = keys_in[i];
            sv[loc] = HAS_VALS ? vals_in[i] : (uint32_t)i;
            sd[loc] = (uint8_t)d;
        }
    }
    __syncthreads();
    const int tn = (int)ttot;
    for (int j = threadIdx.x; j < tn; j += RX_NT) {
        int d = sd[j];
        int64_t pos = goff[d] + (j - tstart[d]);
        if (HAS_KEYS) keys_out[pos] = sk[j];
        vals_out[pos] = sv[j];
    }
}

// ---- onesweep radix sort (one launch per digit pass) ---------------------------------------------------
// All digit histograms come from one read of the keys (k_rx_hist); each pass is one kernel: tiles are taken in
// ticket order, rank their keys locally (warp match, as the downsweep above), publish their per-digit counts and
// find, per digit, the count of that digit in all earlier tiles by a decoupled look-back (thread d walks back
// over digit d's tile states until an inclusive prefix); the tile is then staged in shared memory in (digit,
// input) order and written bucket by bucket.  Stable.  Tile states carry the pass number, so one zeroing per sort
// serves every pass.
constexpr unsigned long long OS_A = 1ull << 62, OS_P = 2ull << 62, OS_VAL = (1ull << 48) - 1;
constexpr int OS_MAXP = 8;
__global__ void __launch_bounds__(256) k_rx_hist(const unsigned long long *__restrict__ keys, int64_t n, int bit_lo,
                                                 int npass, unsigned int *__restrict__ hist) {
    __shared__ unsigned int h[OS_MAXP][256];
    for (int q = threadIdx.x; q < OS_MAXP * 256; q += 256) (&h[0][0])[q] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
        const unsigned long long k = keys[i] >> bit_lo;
        for (int p = 0; p < npass; p++) atomicAdd(&h[p][(k >> (8 * p)) & 0xFFu], 1u);
    }
    __syncthreads();
    for (int p = 0; p < npass; p++)
        if (h[p][threadIdx.x]) atomicAdd(&hist[p * 256 + threadIdx.x], h[p][threadIdx.x]);
}
// exclusive scan of each pass's 256 digit counts (one block)
__global__ void k_rx_hist_scan(unsigned int *__restrict__ hist, int npass, int64_t *__restrict__ excl) {
    __shared__ int64_t sm[33];
    for (int p = 0; p < npass; p++) {
        int64_t tot;
        excl[p * 256 + threadIdx.x] = block_excl_sum<256>((int64_t)hist[p * 256 + threadIdx.x], &tot, sm);
    }
}
constexpr int OS_ROUNDS = 16, OS_TILE = RX_NT * OS_ROUNDS;     // 4096 keys per tile
struct OsSmem {
    unsigned long long sk[OS_TILE];
    uint32_t sv[OS_TILE];
    uint8_t sd[OS_TILE];
};
__global__ void __launch_bounds__(RX_NT, 2) k_rx_onesweep(const unsigned long long *__restrict__ keys_in,
                                                          const uint32_t *__restrict__ vals_in, int64_t n, int shift,
                                                          int pass, const int64_t *__restrict__ hexcl,
                                                          unsigned long long *__restrict__ state,
                                                          unsigned int *__restrict__ ticket,
                                                          unsigned long long *__restrict__ keys_out,
                                                          uint32_t *__restrict__ vals_out) {
    extern __shared__ __align__(16) unsigned char os_dsm[];
    OsSmem &T = *reinterpret_cast<OsSmem *>(os_dsm);
    __shared__ unsigned int wh[RX_WARPS][256];
    __shared__ int64_t goff[256];
    __shared__ int64_t s_tile;
    __shared__ int64_t sc[33];
    __shared__ int tstart[256];
    const int w = threadIdx.x >> 5, l = lane_id();
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(ticket + pass, 1u);
    for (int d = threadIdx.x; d < 256 * RX_WARPS; d += RX_NT) (&wh[0][0])[d] = 0;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * OS_TILE + (int64_t)w * (32 * OS_ROUNDS);
    unsigned long long kv[OS_ROUNDS];
#pragma unroll
    for (int r = 0; r < OS_ROUNDS; r++) {      // all loads in flight before the ranking
        const int64_t i = base + r * 32 + l;
        kv[r] = i < n ? keys_in[i] : 0ull;
    }
    uint32_t dr[OS_ROUNDS];                    // digit (8 bits) | rank in the warp's digit sequence << 8
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < OS_ROUNDS; r++) {
        const int64_t i = base + r * 32 + l;
        const bool valid = i < n;
        const int d = valid ? (int)((kv[r] >> shift) & 0xFFu) : 256 + l;
        const unsigned mm = __match_any_sync(CH_FULL, d);
        const unsigned int before = valid ? wh[w][d] : 0;
        __syncwarp();
        if (valid && (mm & lt) == 0) wh[w][d] = before + __popc(mm);
        __syncwarp();
        dr[r] = (uint32_t)(d & 0xFF) | ((before + __popc(mm & lt)) << 8);
    }
    __syncthreads();
    unsigned int run = 0;
    for (int q = 0; q < RX_WARPS; q++) {
        const unsigned int c = wh[q][threadIdx.x];
        wh[q][threadIdx.x] = run;
        run += c;
    }
    // publish this tile's count of digit d, then look back over earlier tiles for digit d
    {
        const int d = threadIdx.x;
        const unsigned long long tag = (unsigned long long)(pass + 1) << 48;
        volatile unsigned long long *st = state + tile * 256 + d;
        int64_t excl = 0;
        if (tile == 0) {
            *st = OS_P | tag | (unsigned long long)run;
        } else {
            *st = OS_A | tag | (unsigned long long)run;
            for (int64_t p = tile - 1; p >= 0;) {
                const unsigned long long x = *(const volatile unsigned long long *)(state + p * 256 + d);
                if (((x >> 48) & 0x3FFFull) != (unsigned long long)(pass + 1) || (x >> 62) == 0) continue;
                excl += (int64_t)(x & OS_VAL);
                if ((x >> 62) == 2) break;
                p--;
            }
            *st = OS_P | tag | (unsigned long long)(excl + run);
        }
        goff[d] = hexcl[pass * 256 + d] + excl;
    }
    int64_t ttot;
    tstart[threadIdx.x] = (int)block_excl_sum<RX_NT>((int64_t)run, &ttot, sc);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < OS_ROUNDS; r++) {
        const int64_t i = base + r * 32 + l;
        if (i < n) {
            const int d = (int)(dr[r] & 0xFFu);
            const int loc = tstart[d] + (int)wh[w][d] + (int)(dr[r] >> 8);
            T.sk[loc] = kv[r];
            T.sv[loc] = vals_in[i];
            T.sd[loc] = (uint8_t)d;
        }
    }
    __syncthreads();
    const int tn = (int)ttot;
    for (int j = threadIdx.x; j < tn; j += RX_NT) {
        const int d = T.sd[j];
        const int64_t pos = goff[d] + (j - tstart[d]);
        keys_out[pos] = T.sk[j];
        vals_out[pos] = T.sv[j];
    }
}
}  // namespace

chopper_status ch_scan_excl_i64(chopper_ctx *ctx, const int64_t *in, int64_t *out, int64_t n, int64_t *total_dev) {
    if (n <= 0) {
        if (total_dev) CH_CUDA(ctx, cudaMemsetAsync(total_dev, 0, 8, ctx->st));
        return CHOPPER_OK;
    }
    int64_t ntile = ceil_div(n, SC_TILE);
    if (ntile > 1) {
        // single pass: tile states + ticket, zeroed by one memset
        size_t mark = ctx->used;
        CH_ALLOC_BEGIN;
        unsigned long long *state = CH_ALLOC(ctx, unsigned long long, ntile + 1);
        CH_ALLOC_END(ctx);
        CH_CUDA(ctx, cudaMemsetAsync(state, 0, 8 * (size_t)(ntile + 1), ctx->st));
        k_scan_1pass<<<(unsigned)ntile, SC_NT, 0, ctx->st>>>(in, n, out, total_dev, state,
                                                             reinterpret_cast<unsigned int *>(state + ntile));
        CH_LAUNCHED(ctx);
        if (!ctx->hold_scratch) ctx->used = mark;
        return CHOPPER_OK;
    }
    size_t mark = ctx->used;
    CH_ALLOC_BEGIN;
    int64_t *offs = nullptr;
    if (ntile > 1) {
        int64_t *sums = CH_ALLOC(ctx, int64_t, ntile);
        offs = CH_ALLOC(ctx, int64_t, ntile);
        CH_ALLOC_END(ctx);
        k_tile_sums<<<(unsigned)ntile, SC_NT, 0, ctx->st>>>(in, n, sums);
        CH_LAUNCHED(ctx);
        CH_TRY(ch_scan_excl_i64(ctx, sums, offs, ntile, nullptr));
    }
    k_tile_apply<<<(unsigned)ntile, SC_NT, 0, ctx->st>>>(in, n, offs, out, total_dev);
    CH_LAUNCHED(ctx);
    if (!ctx->hold_scratch) ctx->used = mark;
    return CHOPPER_OK;
}

chopper_status ch_seg_scan_i64(chopper_ctx *ctx, const int64_t *in, const uint8_t *head, int64_t *out, int64_t n,
                               int op) {
    if (n <= 0) return CHOPPER_OK;
    int64_t ntile = ceil_div(n, SC_TILE);
    size_t mark = ctx->used;
    int64_t *carry = nullptr;
    if (ntile > 1) {
        CH_ALLOC_BEGIN;
        int64_t *agg = CH_ALLOC(ctx, int64_t, ntile);
        uint8_t *aggh = CH_ALLOC(ctx, uint8_t, ntile);
        int64_t *incl = CH_ALLOC(ctx, int64_t, ntile);
        carry = CH_ALLOC(ctx, int64_t, ntile);
        CH_ALLOC_END(ctx);
        if (op == 1) k_seg_tile_agg<1><<<(unsigned)ntile, SC_NT, 0, ctx->st>>>(in, head, n, agg, aggh);
        else k_seg_tile_agg<0><<<(unsigned)ntile, SC_NT, 0, ctx->st>>>(in, head, n, agg, aggh);
        CH_LAUNCHED(ctx);
        // inclusive pair scan of the tile aggregates (recursive), then shift by one tile
        CH_TRY(ch_seg_scan_i64(ctx, agg, aggh, incl, ntile, op == 1 ? 1 : 2));
        k_shift_carry<<<(unsigned)ceil_div(ntile, 256), 256, 0, ctx->st>>>(incl, ntile, op == 1 ? INT64_MIN : 0, carry);
        CH_LAUNCHED(ctx);
    }
    if (op == 1) k_seg_apply<1, false><<<(unsigned)ntile, SC_NT, 0, ctx->st>>>(in, head, n, carry, out);
    else if (op == 0) k_seg_apply<0, true><<<(unsigned)ntile, SC_NT, 0, ctx->st>>>(in, head, n, carry, out);
    else k_seg_apply<0, false><<<(unsigned)ntile, SC_NT, 0, ctx->st>>>(in, head, n, carry, out);
    CH_LAUNCHED(ctx);
    if (!ctx->hold_scratch) ctx->used = mark;
    return CHOPPER_OK;
}

// stable LSD radix sort of (key, value) pairs over bits [bit_lo, bit_hi).  Each pass reads
// (keys, vals) and writes (keys_alt, vals_alt), then the roles swap; *result_in_alt tells the
// caller which pair holds the sorted result.
chopper_status ch_radix_sort(chopper_ctx *ctx, unsigned long long *keys, uint32_t *vals, unsigned long long *keys_alt,
                             uint32_t *vals_alt, int64_t n, int bit_lo, int bit_hi, bool *result_in_alt) {
    *result_in_alt = false;
    if (n <= 0 || bit_hi <= bit_lo) return CHOPPER_OK;
    const int64_t ntile = ceil_div(n, OS_TILE);
    const int npass = (bit_hi - bit_lo + 7) / 8;
    if (npass > OS_MAXP) return ch_fail(ctx, CHOPPER_E_RANGE, "radix key wider than 64 bits");
    size_t mark = ctx->used;
    CH_ALLOC_BEGIN;
    // one zeroed block: tile states [ntile][256], digit histograms [npass][256], tickets [npass]
    unsigned long long *state = CH_ALLOC(ctx, unsigned long long, ntile * 256 + 256 * OS_MAXP / 2 + OS_MAXP);
    int64_t *hexcl = CH_ALLOC(ctx, int64_t, 256 * OS_MAXP);
    CH_ALLOC_END(ctx);
    unsigned int *hist = reinterpret_cast<unsigned int *>(state + ntile * 256);
    unsigned int *ticket = hist + 256 * OS_MAXP;
    CH_CUDA(ctx, cudaMemsetAsync(state, 0, 8 * (size_t)(ntile * 256 + 256 * OS_MAXP / 2 + OS_MAXP), ctx->st));
    k_rx_hist<<<(unsigned)std::min<int64_t>(ceil_div(n, 256 * 16), 148 * 8), 256, 0, ctx->st>>>(keys, n, bit_lo, npass,
                                                                                              hist);
    CH_LAUNCHED(ctx);
    k_rx_hist_scan<<<1, 256, 0, ctx->st>>>(hist, npass, hexcl);
    CH_LAUNCHED(ctx);
    unsigned long long *ki = keys, *ko = keys_alt;
    uint32_t *vi = vals, *vo = vals_alt;
    bool alt = false;
    static bool os_attr = false;
    if (!os_attr) {
        CH_CUDA(ctx, cudaFuncSetAttribute(k_rx_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OsSmem)));
        os_attr = true;
    }
    for (int p = 0; p < npass; p++) {
        k_rx_onesweep<<<(unsigned)ntile, RX_NT, sizeof(OsSmem), ctx->st>>>(ki, vi, n, bit_lo + 8 * p, p, hexcl, state,
                                                                           ticket, ko, vo);
        CH_LAUNCHED(ctx);
        std::swap(ki, ko);
        std::swap(vi, vo);
        alt = !alt;
    }
    *result_in_alt = alt;
    if (!ctx->hold_scratch) ctx->used = mark;
    return CHOPPER_OK;
}

// a2 fast path: one stable counting pass keyed by (lg, dense group) straight from meta
chopper_status ch_radix_partition_meta(chopper_ctx *ctx, const uint32_t *meta, const int32_t *gpu_lg, int NG,
                                       int other_group, uint32_t *vals_out, int64_t n) {
    if (n <= 0) return CHOPPER_OK;
    int64_t ntile = ceil_div(n, RX_TILE);
    size_t mark = ctx->used;
    CH_ALLOC_BEGIN;
    int64_t *cnt64 = CH_ALLOC(ctx, int64_t, 256 * ntile);
    int64_t *offs = CH_ALLOC(ctx, int64_t, 256 * ntile);
    CH_ALLOC_END(ctx);
    KeyMeta ks{meta, gpu_lg, NG, other_group};
    k_rx_upsweep<KeyMeta><<<(unsigned)ntile, RX_NT, 0, ctx->st>>>(ks, n, cnt64, ntile);
    CH_LAUNCHED(ctx);
    CH_TRY(ch_scan_excl_i64(ctx, cnt64, offs, 256 * ntile, nullptr));
    k_rx_downsweep<KeyMeta, false, false><<<(unsigned)ntile, RX_NT, 0, ctx->st>>>(ks, nullptr, nullptr, n, offs, ntile,
                                                                                 nullptr, vals_out);
    CH_LAUNCHED(ctx);
    ctx->used = mark;
    return CHOPPER_OK;
}
