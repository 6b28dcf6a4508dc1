// ingest.cu -- device-side ingest of a Chrome-trace JSON runtime timeline into the event / span columns
// (R15).
//
// Supported subset: the "traceEvents" array of the root object; device events = ph "X" with cat
// "kernel" or "gpu_*" (pid = gpu, tid = stream, args.correlation), host launches = flow-start events (ph "s",
// id = correlation, ts = dispatch), spans = ph "X" with cat "user_annotation" (pid = gpu, args.level,
// args.label); every other event is ignored.  Times are decimal microseconds converted exactly to integer
// ns, rounded half to even; end = start + duration (each rounded).
//
// Structure (all on the device, one pass per step over the bytes):
//   1. per 64-byte chunk: unescaped quotes -> scan -> in-string state at every chunk start;
//   2. per chunk: depth change of the structural characters outside strings -> scan -> depth at chunk start;
//   3. per chunk: opening '{' at depth 2, closing '}' back to depth 2, root-level '[' / ']' and the
//      "traceEvents" key at depth 1 -> counted, scanned, written (positions in file order);
//   4. a thread per event object parses its keys sequentially (strings with escapes, nested values skipped
//      by depth, exact decimal times);
//   5. flows sorted by id (first in file order wins), kernels join their correlation by binary search
//      (no launch: dispatch = start, counted); names interned by first appearance (64-bit FNV-1a of the
//      decoded name, sorted twice); kernels sorted stably by (gpu, dispatch) into the output columns.
#include "common.cuh"

namespace {
constexpr int JC = 64;                     // bytes per chunk (one thread)
constexpr int NT = 256;

__device__ __forceinline__ bool is_ws(char c) { return c == ' ' || c == '\n' || c == '\r' || c == '\t'; }

// is byte p escaped (preceded by an odd run of backslashes)?
__device__ __forceinline__ bool escaped(const char *js, int64_t p) {
    int64_t k = p - 1;
    int run = 0;
    while (k >= 0 && js[k] == '\\') { run++; k--; }
    return run & 1;
}

__global__ void k_js_quotes(const char *__restrict__ js, int64_t L, int64_t nch, int64_t *__restrict__ nq) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const int64_t a = c * JC, b = a + JC < L ? a + JC : L;
    bool esc = escaped(js, a);
    int64_t q = 0;
    for (int64_t p = a; p < b; p++) {
        const char ch = js[p];
        if (esc) { esc = false; continue; }
        if (ch == '\\') esc = true;
        else if (ch == '"') q++;
    }
    nq[c] = q;
}

// depth change per chunk, structural characters outside strings
__global__ void k_js_depth(const char *__restrict__ js, int64_t L, int64_t nch, const int64_t *__restrict__ qex,
                           int64_t *__restrict__ dd) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const int64_t a = c * JC, b = a + JC < L ? a + JC : L;
    bool ins = qex[c] & 1, esc = escaped(js, a);
    int64_t d = 0;
    for (int64_t p = a; p < b; p++) {
        const char ch = js[p];
        if (esc) { esc = false; continue; }
        if (ins) {
            if (ch == '\\') esc = true;
            else if (ch == '"') ins = false;
            continue;
        }
        if (ch == '"') ins = true;
        else if (ch == '{' || ch == '[') d++;
        else if (ch == '}' || ch == ']') d--;
    }
    dd[c] = d + JC;                 // biased to be non-negative (|d| <= JC): the chained scan takes values >= 0
}

// structural marks: mode 0 counts, mode 1 writes.  Kinds: 0 '{' opening at depth 2 (depth before = 2),
// 1 '}' closing back to depth 2, 2 root '[' (depth before = 1), 3 root ']' (depth after = 1).
// The "traceEvents" key (a string at depth 1 outside strings) -> atomicMin(*key).
__global__ void k_js_marks(const char *__restrict__ js, int64_t L, int64_t nch, const int64_t *__restrict__ qex,
                           const int64_t *__restrict__ dex, int mode, int64_t *__restrict__ cnt,
                           const int64_t *__restrict__ off, int64_t *__restrict__ pos, int32_t *__restrict__ kind,
                           unsigned long long *__restrict__ key) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const int64_t a = c * JC, b = a + JC < L ? a + JC : L;
    bool ins = qex[c] & 1, esc = escaped(js, a);
    int64_t d = dex[c] - (int64_t)JC * c, k = 0, o = mode ? off[c] : 0;     // undo the bias
    for (int64_t p = a; p < b; p++) {
        const char ch = js[p];
        if (esc) { esc = false; continue; }
        if (ins) {
            if (ch == '\\') esc = true;
            else if (ch == '"') ins = false;
            continue;
        }
        int mk = -1;
        if (ch == '"') {
            ins = true;
            if (mode == 0 && d == 1 && p + 12 < L) {
                const char *t = "traceEvents\"";
                bool eq = true;
                for (int q = 0; q < 12 && eq; q++) eq = js[p + 1 + q] == t[q];
                if (eq) atomicMin(key, (unsigned long long)p);
            }
        } else if (ch == '{' || ch == '[') {
            if (ch == '{' && d == 2) mk = 0;
            if (ch == '[' && d == 1) mk = 2;
            d++;
        } else if (ch == '}' || ch == ']') {
            d--;
            if (ch == '}' && d == 2) mk = 1;
            if (ch == ']' && d == 1) mk = 3;
        }
        if (mk >= 0) {
            if (mode) { pos[o + k] = p; kind[o + k] = mk; }
            k++;
        }
    }
    if (!mode) cnt[c] = k;
}

// ---- per-object parser ----
struct Obj {
    int type;                   // 0 ignore, 1 device event, 2 flow start, 3 span
    int64_t pid, tid, ts, dur, id, corr, level, label;
    unsigned long long hash;
    int kind;
    int bad;
};

struct Cursor {
    const char *js;
    int64_t p, e;
    bool bad;
    __device__ __forceinline__ char peek() const { return p < e ? js[p] : '\0'; }
    __device__ __forceinline__ void ws() { while (p < e && is_ws(js[p])) p++; }
    __device__ __forceinline__ bool eat(char c) {
        ws();
        if (p < e && js[p] == c) { p++; return true; }
        bad = true;
        return false;
    }
};

// decode one string (cursor on the opening quote); calls f(byte) for each decoded UTF-8 byte
template <class F>
__device__ void read_string(Cursor &c, F f) {
    if (!c.eat('"')) return;
    while (c.p < c.e) {
        const char ch = c.js[c.p++];
        if (ch == '"') return;
        if (ch != '\\') { f((unsigned char)ch); continue; }
        if (c.p >= c.e) break;
        const char x = c.js[c.p++];
        if (x == 'u') {
            auto hex4 = [&](unsigned &v) -> bool {
                v = 0;
                for (int q = 0; q < 4; q++) {
                    if (c.p >= c.e) return false;
                    const char h = c.js[c.p++];
                    v <<= 4;
                    if (h >= '0' && h <= '9') v |= (unsigned)(h - '0');
                    else if (h >= 'a' && h <= 'f') v |= (unsigned)(h - 'a' + 10);
                    else if (h >= 'A' && h <= 'F') v |= (unsigned)(h - 'A' + 10);
                    else return false;
                }
                return true;
            };
            unsigned u;
            if (!hex4(u)) { c.bad = true; return; }
            if (u >= 0xD800 && u < 0xDC00 && c.p + 1 < c.e && c.js[c.p] == '\\' && c.js[c.p + 1] == 'u') {
                const int64_t save = c.p;
                c.p += 2;
                unsigned lo;
                if (hex4(lo) && lo >= 0xDC00 && lo < 0xE000) u = 0x10000 + ((u - 0xD800) << 10) + (lo - 0xDC00);
                else c.p = save;
            }
            if (u < 0x80) f(u);
            else if (u < 0x800) { f(0xC0 | (u >> 6)); f(0x80 | (u & 0x3F)); }
            else if (u < 0x10000) { f(0xE0 | (u >> 12)); f(0x80 | ((u >> 6) & 0x3F)); f(0x80 | (u & 0x3F)); }
            else { f(0xF0 | (u >> 18)); f(0x80 | ((u >> 12) & 0x3F)); f(0x80 | ((u >> 6) & 0x3F)); f(0x80 | (u & 0x3F)); }
        } else {
            const unsigned v = x == 'n' ? '\n' : x == 't' ? '\t' : x == 'r' ? '\r' : x == 'b' ? '\b' : x == 'f' ? '\f' : (unsigned char)x;
            f(v);
        }
    }
    c.bad = true;
}

// skip any JSON value (strings respected, containers by depth)
__device__ void skip_value(Cursor &c) {
    c.ws();
    const char ch = c.peek();
    if (ch == '"') { read_string(c, [](unsigned) {}); return; }
    if (ch == '{' || ch == '[') {
        int d = 0;
        bool ins = false, esc = false;
        while (c.p < c.e) {
            const char x = c.js[c.p++];
            if (esc) { esc = false; continue; }
            if (ins) { if (x == '\\') esc = true; else if (x == '"') ins = false; continue; }
            if (x == '"') ins = true;
            else if (x == '{' || x == '[') d++;
            else if (x == '}' || x == ']') { if (--d == 0) return; }
        }
        c.bad = true;
        return;
    }
    while (c.p < c.e && c.js[c.p] != ',' && c.js[c.p] != '}' && c.js[c.p] != ']' && !is_ws(c.js[c.p])) c.p++;
}

// a JSON integer (optionally written with a zero fraction / exponent is rejected: ids and pids are integers)
__device__ bool read_int(Cursor &c, int64_t *out) {
    c.ws();
    bool neg = false;
    if (c.peek() == '-') { neg = true; c.p++; }
    if (!(c.peek() >= '0' && c.peek() <= '9')) return false;
    unsigned long long v = 0;
    while (c.p < c.e && c.js[c.p] >= '0' && c.js[c.p] <= '9') {
        if (v > (unsigned long long)(INT64_MAX / 10)) return false;     // more than 19 digits: out of range
        v = v * 10 + (unsigned long long)(c.js[c.p++] - '0');
    }
    if (v > (unsigned long long)INT64_MAX) return false;
    *out = neg ? -(int64_t)v : (int64_t)v;
    return true;
}

// a decimal number of microseconds -> integer ns, rounded half to even, exactly: value = D * 10^x with D the
// significant digits (the first 36 kept, later ones only as a nonzero "sticky" flag)
__device__ bool read_us_ns(Cursor &c, int64_t *out) {
    c.ws();
    bool neg = false;
    if (c.peek() == '-') { neg = true; c.p++; }
    unsigned __int128 D = 0;
    int nd = 0, x = 0;
    bool sticky = false, any = false;
    while (c.p < c.e && c.js[c.p] >= '0' && c.js[c.p] <= '9') {
        const int v = c.js[c.p++] - '0';
        any = true;
        if (nd < 36) { D = D * 10 + (unsigned)v; if (D) nd++; } else { x++; sticky |= v != 0; }
    }
    if (c.peek() == '.') {
        c.p++;
        while (c.p < c.e && c.js[c.p] >= '0' && c.js[c.p] <= '9') {
            const int v = c.js[c.p++] - '0';
            any = true;
            if (nd < 36) { D = D * 10 + (unsigned)v; if (D) nd++; x--; } else { sticky |= v != 0; }
        }
    }
    if (!any) return false;
    if (c.peek() == 'e' || c.peek() == 'E') {
        c.p++;
        bool en = false;
        if (c.peek() == '+' || c.peek() == '-') { en = c.peek() == '-'; c.p++; }
        int ev = 0;
        bool ed = false;
        while (c.p < c.e && c.js[c.p] >= '0' && c.js[c.p] <= '9') { ev = ev * 10 + (c.js[c.p++] - '0'); ed = true; if (ev > 1000) ev = 1000; }
        if (!ed) return false;
        x += en ? -ev : ev;
    }
    x += 3;                                              // microseconds -> nanoseconds
    unsigned __int128 r;
    if (x >= 0) {
        if (x > 38) return false;
        r = D;
        if (r > (unsigned __int128)INT64_MAX) return false;
        for (int q = 0; q < x; q++) {                    // out of range as soon as it passes INT64_MAX (no wrap)
            if (r > (unsigned __int128)(INT64_MAX / 10)) return false;
            r *= 10;
        }
    } else {
        const int k = -x;
        if (k > 38) { r = 0; sticky |= D != 0; D = 0; }
        unsigned __int128 p10 = 1;
        for (int q = 0; q < k && q < 38; q++) p10 *= 10;
        r = k > 38 ? 0 : D / p10;
        const unsigned __int128 rem = k > 38 ? 0 : D % p10;
        if (k <= 38) {
            const unsigned __int128 half = p10 / 2;
            // half to even: above half, or exactly half (no sticky digits) with an odd quotient
            if (rem > half || (rem == half && (sticky || (r & 1)))) r += 1;
        }
    }
    if (r > (unsigned __int128)INT64_MAX) return false;
    *out = neg ? -(int64_t)r : (int64_t)r;
    return true;
}

struct NameAcc {                 // FNV-1a of the decoded name + the kind rules' substring flags (lowercase)
    unsigned long long h = 0xcbf29ce484222325ull;
    unsigned long long w = 0;    // last 14 lowercase bytes, packed (window for the patterns)
    int n = 0;
    unsigned flags = 0;          // 1 allgather / all_gather, 2 reducescatter / reduce_scatter, 4 nccl / rccl, 8 fsdp_copy
};

__device__ __forceinline__ bool ends_with(const unsigned char *buf, int n, const char *pat) {
    int m = 0;
    while (pat[m]) m++;
    if (n < m) return false;
    for (int q = 0; q < m; q++) if (buf[n - m + q] != (unsigned char)pat[q]) return false;
    return true;
}

__device__ void parse_object(const char *js, int64_t a, int64_t b, Obj &o) {
    o.type = 0; o.pid = o.tid = o.ts = o.dur = o.id = 0; o.corr = -1; o.level = -1; o.label = 0;
    o.hash = 0; o.kind = 0; o.bad = 0;
    Cursor c{js, a, b + 1, false};
    char ph = 0;
    int cat = -1;                // 0 kernel, 1 gpu_memset, 2 gpu_memcpy, 3 other gpu_*, 4 user_annotation, 5 other
    bool has_ts = false, has_dur = false, has_pid = false, has_tid = false, has_id = false;
    NameAcc nm;
    unsigned char win[16];
    int wn = 0;
    if (!c.eat('{')) { o.bad = 1; return; }
    c.ws();
    if (c.peek() == '}') return;
    while (!c.bad) {
        // key
        char kb[16];
        int kn = 0;
        read_string(c, [&](unsigned v) { if (kn < 15) kb[kn] = (char)v; kn++; });
        if (c.bad) break;
        kb[kn < 15 ? kn : 15] = 0;
        if (!c.eat(':')) break;
        c.ws();
        auto is = [&](const char *s) { int q = 0; while (s[q] && q < 15 && kb[q] == s[q]) q++; return !s[q] && q == kn; };
        if (is("ph")) {
            read_string(c, [&](unsigned v) { if (!ph) ph = (char)v; });
        } else if (is("cat")) {
            char cb[20];
            int cn = 0;
            read_string(c, [&](unsigned v) { if (cn < 19) cb[cn] = (char)v; cn++; });
            cb[cn < 19 ? cn : 19] = 0;
            auto eqs = [&](const char *s) { int q = 0; while (s[q] && q < 19 && cb[q] == s[q]) q++; return !s[q] && q == cn; };
            if (eqs("kernel")) cat = 0;
            else if (eqs("gpu_memset")) cat = 1;
            else if (eqs("gpu_memcpy")) cat = 2;
            else if (cn >= 4 && cb[0] == 'g' && cb[1] == 'p' && cb[2] == 'u' && cb[3] == '_') cat = 3;
            else if (eqs("user_annotation")) cat = 4;
            else cat = 5;
        } else if (is("name")) {
            read_string(c, [&](unsigned v) {
                nm.h = (nm.h ^ (unsigned long long)(v & 0xFF)) * 0x100000001b3ull;
                unsigned char lc = (unsigned char)v;
                if (lc >= 'A' && lc <= 'Z') lc = (unsigned char)(lc + 32);
                if (wn == 16) { for (int q = 0; q < 15; q++) win[q] = win[q + 1]; wn = 15; }
                win[wn++] = lc;
                if (ends_with(win, wn, "allgather") || ends_with(win, wn, "all_gather")) nm.flags |= 1;
                if (ends_with(win, wn, "reducescatter") || ends_with(win, wn, "reduce_scatter")) nm.flags |= 2;
                if (ends_with(win, wn, "nccl") || ends_with(win, wn, "rccl")) nm.flags |= 4;
                if (ends_with(win, wn, "fsdp_copy")) nm.flags |= 8;
            });
        } else if (is("pid")) {
            has_pid = read_int(c, &o.pid);
            if (!has_pid) skip_value(c);
        } else if (is("tid")) {
            has_tid = read_int(c, &o.tid);
            if (!has_tid) skip_value(c);
        } else if (is("ts")) {
            has_ts = read_us_ns(c, &o.ts);
            if (!has_ts) skip_value(c);
        } else if (is("dur")) {
            has_dur = read_us_ns(c, &o.dur);
            if (!has_dur) skip_value(c);
        } else if (is("id")) {
            has_id = read_int(c, &o.id);
            if (!has_id) skip_value(c);
        } else if (is("args")) {
            if (!c.eat('{')) break;
            c.ws();
            if (c.peek() == '}') { c.p++; }
            else {
                while (!c.bad) {
                    char ab[16];
                    int an = 0;
                    read_string(c, [&](unsigned v) { if (an < 15) ab[an] = (char)v; an++; });
                    ab[an < 15 ? an : 15] = 0;
                    if (!c.eat(':')) break;
                    auto ais = [&](const char *s) { int q = 0; while (s[q] && q < 15 && ab[q] == s[q]) q++; return !s[q] && q == an; };
                    int64_t v;
                    if (ais("correlation")) { if (read_int(c, &v)) o.corr = v; else skip_value(c); }
                    else if (ais("level")) { if (read_int(c, &v)) o.level = v; else skip_value(c); }
                    else if (ais("label")) { if (read_int(c, &v)) o.label = v; else skip_value(c); }
                    else skip_value(c);
                    c.ws();
                    if (c.peek() == ',') { c.p++; c.ws(); continue; }
                    if (c.peek() == '}') { c.p++; break; }
                    c.bad = true;
                }
            }
        } else {
            skip_value(c);
        }
        c.ws();
        if (c.peek() == ',') { c.p++; c.ws(); continue; }
        if (c.peek() == '}') break;
        c.bad = true;
    }
    if (c.bad) { o.bad = 1; return; }
    o.hash = nm.h;
    if (ph == 's' && has_id && has_ts) {
        o.type = 2;
    } else if (ph == 'X' && cat == 4) {
        if (!has_pid || !has_ts || !has_dur || o.level < 0) { o.bad = 1; return; }
        o.type = 3;
    } else if (ph == 'X' && cat >= 0 && cat <= 3) {
        if (!has_pid || !has_tid || !has_ts || !has_dur || o.pid < 0 || o.pid > 255 || o.tid < 0 || o.tid > 0xFFFF) {
            o.bad = 1;
            return;
        }
        o.type = 1;
        o.kind = cat == 1 ? CK_MEMOP : cat == 2 ? CK_COPY : cat == 3 ? CK_OTHER
               : (nm.flags & 1) ? CK_AG : (nm.flags & 2) ? CK_RS : (nm.flags & 4) ? CK_COMM_OTHER
               : (nm.flags & 8) ? CK_COPY : CK_COMPUTE;
    }
}

struct ObjCols {
    int32_t *type;
    int64_t *pid, *tid, *ts, *end, *id, *corr, *level, *label;
    unsigned long long *hash;
    int32_t *kind;
};

// the traceEvents array: the first root '[' after the key, and the first root ']' after that
__global__ void k_js_bounds(const int64_t *__restrict__ mpos, const int32_t *__restrict__ mkind,
                            const int64_t *__restrict__ nm_d, const unsigned long long *__restrict__ key, int step,
                            unsigned long long *__restrict__ arr) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= *nm_d || *key == ~0ull) return;
    if (step == 0 && mkind[t] == 2 && (unsigned long long)mpos[t] > *key) atomicMin(&arr[0], (unsigned long long)mpos[t]);
    if (step == 1 && mkind[t] == 3 && arr[0] != ~0ull && (unsigned long long)mpos[t] > arr[0])
        atomicMin(&arr[1], (unsigned long long)mpos[t]);
}
__global__ void k_js_open_flags(const int32_t *__restrict__ mkind, const int64_t *__restrict__ nm_d, int64_t cap,
                                int64_t *__restrict__ f) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cap) return;
    f[t] = t < *nm_d && mkind[t] == 0 ? 1 : 0;
}
__global__ void k_scatter_idx(const int64_t *__restrict__ f, const int64_t *__restrict__ ex, int64_t n,
                              int64_t *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n && f[t]) out[ex[t]] = t;
}

// a thread per event object (its opening mark; the closing mark is the next mark: nothing between them is at
// depth 2), inside the traceEvents array only
__global__ void k_js_objects(const char *__restrict__ js, const int64_t *__restrict__ mpos,
                             const int32_t *__restrict__ mkind, const int64_t *__restrict__ nm_d,
                             const unsigned long long *__restrict__ arr, const int64_t *__restrict__ opens,
                             const int64_t *__restrict__ n_open, ObjCols O, unsigned int *__restrict__ bad,
                             unsigned long long *__restrict__ bad_at) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= *n_open) return;
    const int64_t mi = opens[q];
    const int64_t a = mpos[mi];
    O.type[q] = 0;
    if (arr[0] == ~0ull || arr[1] == ~0ull || (unsigned long long)a < arr[0] || (unsigned long long)a > arr[1]) return;
    if (!(mi + 1 < *nm_d && mkind[mi + 1] == 1)) {
        atomicOr(bad, 1u);
        atomicMin(bad_at, (unsigned long long)a);
        return;
    }
    Obj o;
    parse_object(js, a, mpos[mi + 1], o);
    if (o.bad) { atomicOr(bad, 1u); atomicMin(bad_at, (unsigned long long)a); return; }
    O.type[q] = o.type;
    O.pid[q] = o.pid; O.tid[q] = o.tid; O.ts[q] = o.ts; O.end[q] = o.ts + o.dur; O.id[q] = o.id;
    O.corr[q] = o.corr; O.level[q] = o.level; O.label[q] = o.label; O.hash[q] = o.hash; O.kind[q] = o.kind;
}

__global__ void k_type_flags(const int32_t *__restrict__ type, const int64_t *__restrict__ n_d, int64_t cap, int want,
                             int64_t *__restrict__ f) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cap) return;
    f[t] = t < *n_d && type[t] == want ? 1 : 0;
}
// keys for the sorts: flows by id, kernels by name hash (values = ordinal in file order)
__global__ void k_flow_keys(const int64_t *__restrict__ fl, int64_t nf, const int64_t *__restrict__ id,
                            unsigned long long *__restrict__ k, uint32_t *__restrict__ v) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nf) return;
    k[t] = enc_i64(id[fl[t]]);
    v[t] = (uint32_t)t;
}
__global__ void k_hash_keys(const int64_t *__restrict__ kl, int64_t nk, const unsigned long long *__restrict__ h,
                            unsigned long long *__restrict__ k, uint32_t *__restrict__ v) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nk) return;
    k[t] = h[kl[t]];
    v[t] = (uint32_t)t;
}
// unique hashes (runs of the stable sort: the first element is the first appearance) -> (first ordinal, run)
__global__ void k_hash_heads(const unsigned long long *__restrict__ k, const uint32_t *__restrict__ v, int64_t n,
                             int64_t *__restrict__ f) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) f[t] = (t == 0 || k[t] != k[t - 1]) ? 1 : 0;
}
__global__ void k_hash_uniq(const unsigned long long *__restrict__ k, const uint32_t *__restrict__ v, int64_t n,
                            const int64_t *__restrict__ f, const int64_t *__restrict__ ex,
                            unsigned long long *__restrict__ uh, unsigned long long *__restrict__ ufirst,
                            uint32_t *__restrict__ uidx) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n || !f[t]) return;
    const int64_t u = ex[t];
    uh[u] = k[t];
    ufirst[u] = v[t];
    uidx[u] = (uint32_t)u;
}
__global__ void k_hash_rank(const uint32_t *__restrict__ uidx_sorted, int64_t nu, int32_t *__restrict__ uid) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nu) uid[uidx_sorted[r]] = (int32_t)r;
}
// per kernel: dispatch from its launch (first flow with the same id), name id, then the final sort key
__global__ void k_kernel_join(const int64_t *__restrict__ kl, int64_t nk, const int64_t *__restrict__ corr,
                              const int64_t *__restrict__ ts, const unsigned long long *__restrict__ h,
                              const unsigned long long *__restrict__ fid, const uint32_t *__restrict__ ford,
                              int64_t nf, const int64_t *__restrict__ fl, const int64_t *__restrict__ fts_obj,
                              const unsigned long long *__restrict__ uh, const int32_t *__restrict__ uid, int64_t nu,
                              int64_t *__restrict__ tl, int32_t *__restrict__ nid,
                              unsigned long long *__restrict__ missing, unsigned long long *__restrict__ tmm) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nk) return;
    const int64_t o = kl[t];
    int64_t d = ts[o];
    bool found = false;
    if (corr[o] >= 0 && nf > 0) {
        const unsigned long long c = enc_i64(corr[o]);
        int64_t l = 0, hi = nf;
        while (l < hi) { const int64_t m = (l + hi) >> 1; if (fid[m] < c) l = m + 1; else hi = m; }
        if (l < nf && fid[l] == c) { d = fts_obj[fl[ford[l]]]; found = true; }
    }
    if (!found) atomicAdd(missing, 1ull);
    tl[t] = d;
    atomicMin(&tmm[0], enc_i64(d));
    atomicMax(&tmm[1], enc_i64(d));
    const unsigned long long hh = h[o];
    int64_t l = 0, hi = nu;
    while (l < hi) { const int64_t m = (l + hi) >> 1; if (uh[m] < hh) l = m + 1; else hi = m; }
    nid[t] = uid[l];
}
__global__ void k_final_keys(const int64_t *__restrict__ kl, int64_t nk, const int64_t *__restrict__ pid,
                             const int64_t *__restrict__ tl, int64_t tmin, int tsbits,
                             unsigned long long *__restrict__ k, uint32_t *__restrict__ v) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nk) return;
    k[t] = ((unsigned long long)pid[kl[t]] << tsbits) | (unsigned long long)(tl[t] - tmin);
    v[t] = (uint32_t)t;
}
__global__ void k_final_gather(const uint32_t *__restrict__ ord, int64_t nk, const int64_t *__restrict__ kl,
                               const int64_t *__restrict__ tl, const int32_t *__restrict__ nid, ObjCols O,
                               int64_t *__restrict__ o_tl, int64_t *__restrict__ o_ks, int64_t *__restrict__ o_ke,
                               uint32_t *__restrict__ o_meta, int32_t *__restrict__ o_nid) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nk) return;
    const uint32_t t = ord[r];
    const int64_t o = kl[t];
    o_tl[r] = tl[t];
    o_ks[r] = O.ts[o];
    o_ke[r] = O.end[o];
    o_meta[r] = ((uint32_t)O.pid[o] << 24) | ((uint32_t)O.tid[o] << 8) | (uint32_t)O.kind[o];
    o_nid[r] = nid[t];
}
__global__ void k_span_out(const int64_t *__restrict__ sl, int64_t ns, ObjCols O, uint32_t *__restrict__ gl,
                           int64_t *__restrict__ s0, int64_t *__restrict__ s1, int32_t *__restrict__ lab,
                           unsigned int *__restrict__ bad) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= ns) return;
    const int64_t o = sl[r];
    if (O.pid[o] < 0 || O.pid[o] > 255 || O.level[o] > 255) atomicOr(bad, 1u);
    gl[r] = ((uint32_t)O.pid[o] << 8) | (uint32_t)(O.level[o] & 0xFF);
    s0[r] = O.ts[o];
    s1[r] = O.end[o];
    lab[r] = (int32_t)O.label[o];
}
}  // namespace

size_t ch_ingest_scratch_bytes(int64_t n_bytes) {
    // chunk arrays + marks (at most one per 8 bytes: an event object of >= 16 bytes has two) x (mark arrays,
    // object columns, sort buffers); a denser document fails with CHOPPER_E_RANGE (scratch exhausted)
    const int64_t nch = ceil_div(std::max<int64_t>(n_bytes, 1), JC);
    const int64_t nmk = n_bytes / 8 + 64;
    return (size_t)nch * 8 * 6 + (size_t)nmk * 300 + (64u << 20);
}

chopper_status ch_ingest_chrome(chopper_ctx *ctx, const char *js, int64_t L, void *scratch, size_t scratch_bytes,
                                const chopper_ingest_out *out, chopper_ingest_report *rep) {
    // the ingest runs in its own scratch (restored afterwards): it precedes chopper_load_columns
    char *sv_s = ctx->scratch;
    const size_t sv_b = ctx->scratch_bytes, sv_u = ctx->used;
    ctx->scratch = (char *)scratch;
    ctx->scratch_bytes = scratch_bytes;
    ctx->used = 0;
    auto restore = [&]() { ctx->scratch = sv_s; ctx->scratch_bytes = sv_b; ctx->used = sv_u; };
    chopper_status st = [&]() -> chopper_status {
        memset(rep, 0, sizeof(*rep));
        rep->bad_offset = -1;
        const int64_t nch = ceil_div(std::max<int64_t>(L, 1), JC);
        CH_ALLOC_BEGIN;
        int64_t *a1 = CH_ALLOC(ctx, int64_t, nch + 1), *q_ex = CH_ALLOC(ctx, int64_t, nch + 1);
        int64_t *a2 = CH_ALLOC(ctx, int64_t, nch + 1), *d_ex = CH_ALLOC(ctx, int64_t, nch + 1);
        int64_t *a3 = CH_ALLOC(ctx, int64_t, nch + 1), *m_ex = CH_ALLOC(ctx, int64_t, nch + 1);
        int64_t *tot = CH_ALLOC(ctx, int64_t, 8);
        unsigned long long *key = CH_ALLOC(ctx, unsigned long long, 8);   // [0] key [1..2] array [3] bad_at [4] missing [5..6] tmin/max
        unsigned int *bad = CH_ALLOC(ctx, unsigned int, 1);
        CH_ALLOC_END(ctx);
        CH_CUDA(ctx, cudaMemsetAsync(key, 0xFF, 8 * 8, ctx->st));
        CH_CUDA(ctx, cudaMemsetAsync(key + 4, 0, 8, ctx->st));
        CH_CUDA(ctx, cudaMemsetAsync(bad, 0, 4, ctx->st));
        {   // tmin / tmax start values (encoded): min = all ones, max = 0
            unsigned long long init[2] = {~0ull, 0ull};
            CH_CUDA(ctx, cudaMemcpyAsync(key + 5, init, 16, cudaMemcpyHostToDevice, ctx->st));
        }
        const unsigned g = (unsigned)ceil_div(nch, NT);
        if (L > 0) {
            k_js_quotes<<<g, NT, 0, ctx->st>>>(js, L, nch, a1);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_scan_excl_i64(ctx, a1, q_ex, nch, tot + 0));
            k_js_depth<<<g, NT, 0, ctx->st>>>(js, L, nch, q_ex, a2);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_scan_excl_i64(ctx, a2, d_ex, nch, tot + 1));
            k_js_marks<<<g, NT, 0, ctx->st>>>(js, L, nch, q_ex, d_ex, 0, a3, nullptr, nullptr, nullptr, key);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_scan_excl_i64(ctx, a3, m_ex, nch, tot + 2));
        } else {
            CH_CUDA(ctx, cudaMemsetAsync(tot, 0, 64, ctx->st));
        }
        int64_t h3[3];
        CH_CUDA(ctx, cudaMemcpyAsync(h3, tot, 24, cudaMemcpyDeviceToHost, ctx->st));
        CH_CUDA(ctx, ch_sync(ctx));
        h3[1] -= (int64_t)JC * nch;
        if ((h3[0] & 1) || h3[1] != 0)
            return ch_fail(ctx, CHOPPER_E_VALIDATION, "JSON: unbalanced strings or brackets (quotes " +
                                                          std::to_string(h3[0]) + ", depth " + std::to_string(h3[1]) + ")");
        const int64_t nmk = h3[2];
        int64_t *mpos = CH_ALLOC(ctx, int64_t, nmk + 1);
        int32_t *mkind = CH_ALLOC(ctx, int32_t, nmk + 1);
        int64_t *of = CH_ALLOC(ctx, int64_t, nmk + 1), *oex = CH_ALLOC(ctx, int64_t, nmk + 1);
        int64_t *opens = CH_ALLOC(ctx, int64_t, nmk + 1);
        CH_ALLOC_END(ctx);
        if (L > 0) {
            k_js_marks<<<g, NT, 0, ctx->st>>>(js, L, nch, q_ex, d_ex, 1, nullptr, m_ex, mpos, mkind, key);
            CH_LAUNCHED(ctx);
        }
        const unsigned gm = (unsigned)ceil_div(std::max<int64_t>(nmk, 1), NT);
        k_js_bounds<<<gm, NT, 0, ctx->st>>>(mpos, mkind, tot + 2, key, 0, key + 1);
        CH_LAUNCHED(ctx);
        k_js_bounds<<<gm, NT, 0, ctx->st>>>(mpos, mkind, tot + 2, key, 1, key + 1);
        CH_LAUNCHED(ctx);
        k_js_open_flags<<<gm, NT, 0, ctx->st>>>(mkind, tot + 2, std::max<int64_t>(nmk, 1), of);
        CH_LAUNCHED(ctx);
        CH_TRY(ch_scan_excl_i64(ctx, of, oex, std::max<int64_t>(nmk, 1), tot + 3));
        k_scatter_idx<<<gm, NT, 0, ctx->st>>>(of, oex, nmk, opens);
        CH_LAUNCHED(ctx);
        // objects (capacity: every opening mark)
        const int64_t nob = std::max<int64_t>(nmk, 1);
        ObjCols O;
        O.type = CH_ALLOC(ctx, int32_t, nob);
        O.pid = CH_ALLOC(ctx, int64_t, nob); O.tid = CH_ALLOC(ctx, int64_t, nob);
        O.ts = CH_ALLOC(ctx, int64_t, nob); O.end = CH_ALLOC(ctx, int64_t, nob);
        O.id = CH_ALLOC(ctx, int64_t, nob); O.corr = CH_ALLOC(ctx, int64_t, nob);
        O.level = CH_ALLOC(ctx, int64_t, nob); O.label = CH_ALLOC(ctx, int64_t, nob);
        O.hash = CH_ALLOC(ctx, unsigned long long, nob);
        O.kind = CH_ALLOC(ctx, int32_t, nob);
        int64_t *tf = CH_ALLOC(ctx, int64_t, nob), *tex = CH_ALLOC(ctx, int64_t, nob);
        int64_t *kl = CH_ALLOC(ctx, int64_t, nob), *fl = CH_ALLOC(ctx, int64_t, nob), *sl = CH_ALLOC(ctx, int64_t, nob);
        CH_ALLOC_END(ctx);
        const unsigned go = (unsigned)ceil_div(nob, NT);
        k_js_objects<<<go, NT, 0, ctx->st>>>(js, mpos, mkind, tot + 2, key + 1, opens, tot + 3, O, bad, key + 3);
        CH_LAUNCHED(ctx);
        int64_t *lists[3] = {kl, fl, sl};
        for (int ty = 1; ty <= 3; ty++) {
            k_type_flags<<<go, NT, 0, ctx->st>>>(O.type, tot + 3, nob, ty, tf);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_scan_excl_i64(ctx, tf, tex, nob, tot + 3 + ty));
            k_scatter_idx<<<go, NT, 0, ctx->st>>>(tf, tex, nob, lists[ty - 1]);
            CH_LAUNCHED(ctx);
        }
        int64_t h7[7];
        unsigned int hbad = 0;
        unsigned long long hk[4];
        CH_CUDA(ctx, cudaMemcpyAsync(h7, tot, 56, cudaMemcpyDeviceToHost, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(hk, key, 32, cudaMemcpyDeviceToHost, ctx->st));
        CH_CUDA(ctx, ch_sync(ctx));
        const int64_t nk = h7[4], nf = h7[5], ns = h7[6];
        rep->n_objects = h7[3];
        rep->n_kernels = nk;
        rep->n_flows = nf;
        rep->n_spans = ns;
        if (hk[0] == ~0ull || hk[1] == ~0ull || hk[2] == ~0ull)
            return ch_fail(ctx, CHOPPER_E_VALIDATION, "JSON: no \"traceEvents\" array");
        if (hbad) {
            rep->bad_offset = (int64_t)hk[3];
            return ch_fail(ctx, CHOPPER_E_VALIDATION, "JSON: malformed event object at byte " + std::to_string(hk[3]));
        }
        if (nk > out->ev_cap || ns > out->span_cap) return ch_fail(ctx, CHOPPER_E_RANGE, "ingest output capacity");
        // flows sorted by id (stable: the first in file order heads each run)
        unsigned long long *k1 = CH_ALLOC(ctx, unsigned long long, std::max<int64_t>(std::max(nk, nf), 1));
        unsigned long long *k2 = CH_ALLOC(ctx, unsigned long long, std::max<int64_t>(std::max(nk, nf), 1));
        uint32_t *v1 = CH_ALLOC(ctx, uint32_t, std::max<int64_t>(std::max(nk, nf), 1));
        uint32_t *v2 = CH_ALLOC(ctx, uint32_t, std::max<int64_t>(std::max(nk, nf), 1));
        unsigned long long *fid = CH_ALLOC(ctx, unsigned long long, std::max<int64_t>(nf, 1));
        uint32_t *ford = CH_ALLOC(ctx, uint32_t, std::max<int64_t>(nf, 1));
        CH_ALLOC_END(ctx);
        bool alt = false;
        if (nf > 0) {
            k_flow_keys<<<(unsigned)ceil_div(nf, NT), NT, 0, ctx->st>>>(fl, nf, O.id, k1, v1);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, nf, 0, 64, &alt));
            CH_CUDA(ctx, cudaMemcpyAsync(fid, alt ? k2 : k1, 8 * nf, cudaMemcpyDeviceToDevice, ctx->st));
            CH_CUDA(ctx, cudaMemcpyAsync(ford, alt ? v2 : v1, 4 * nf, cudaMemcpyDeviceToDevice, ctx->st));
        }
        // names: kernels by hash (stable), unique hashes with their first appearance, ranked by it
        int64_t *hf = CH_ALLOC(ctx, int64_t, std::max<int64_t>(nk, 1)), *hex = CH_ALLOC(ctx, int64_t, std::max<int64_t>(nk, 1));
        unsigned long long *uh = CH_ALLOC(ctx, unsigned long long, std::max<int64_t>(nk, 1));
        unsigned long long *ufirst = CH_ALLOC(ctx, unsigned long long, std::max<int64_t>(nk, 1));
        unsigned long long *uf2 = CH_ALLOC(ctx, unsigned long long, std::max<int64_t>(nk, 1));
        uint32_t *uidx = CH_ALLOC(ctx, uint32_t, std::max<int64_t>(nk, 1)), *ui2 = CH_ALLOC(ctx, uint32_t, std::max<int64_t>(nk, 1));
        int32_t *uid = CH_ALLOC(ctx, int32_t, std::max<int64_t>(nk, 1));
        int64_t *tl = CH_ALLOC(ctx, int64_t, std::max<int64_t>(nk, 1));
        int32_t *nid = CH_ALLOC(ctx, int32_t, std::max<int64_t>(nk, 1));
        CH_ALLOC_END(ctx);
        int64_t nu = 0;
        if (nk > 0) {
            const unsigned gk = (unsigned)ceil_div(nk, NT);
            k_hash_keys<<<gk, NT, 0, ctx->st>>>(kl, nk, O.hash, k1, v1);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, nk, 0, 64, &alt));
            unsigned long long *hs = alt ? k2 : k1;
            uint32_t *hv = alt ? v2 : v1;
            k_hash_heads<<<gk, NT, 0, ctx->st>>>(hs, hv, nk, hf);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_scan_excl_i64(ctx, hf, hex, nk, tot + 7 - 1));      // tot[6] reused: unique count
            k_hash_uniq<<<gk, NT, 0, ctx->st>>>(hs, hv, nk, hf, hex, uh, ufirst, uidx);
            CH_LAUNCHED(ctx);
            CH_CUDA(ctx, cudaMemcpyAsync(&nu, tot + 6, 8, cudaMemcpyDeviceToHost, ctx->st));
            CH_CUDA(ctx, ch_sync(ctx));
            bool alt2 = false;
            CH_TRY(ch_radix_sort(ctx, ufirst, uidx, uf2, ui2, nu, 0, bits_for((uint64_t)std::max<int64_t>(nk, 1)), &alt2));
            k_hash_rank<<<(unsigned)ceil_div(std::max<int64_t>(nu, 1), NT), NT, 0, ctx->st>>>(alt2 ? ui2 : uidx, nu, uid);
            CH_LAUNCHED(ctx);
            k_kernel_join<<<gk, NT, 0, ctx->st>>>(kl, nk, O.corr, O.ts, O.hash, fid, ford, nf, fl, O.ts, uh, uid, nu, tl,
                                                  nid, key + 4, key + 5);
            CH_LAUNCHED(ctx);
            unsigned long long hm[3];
            CH_CUDA(ctx, cudaMemcpyAsync(hm, key + 4, 24, cudaMemcpyDeviceToHost, ctx->st));
            CH_CUDA(ctx, ch_sync(ctx));
            rep->n_missing = (int64_t)hm[0];
            const int64_t tmin = dec_i64(hm[1]), tmax = dec_i64(hm[2]);
            const int tsbits = bits_for((uint64_t)(tmax - tmin));
            if (tsbits + 8 > 64) return ch_fail(ctx, CHOPPER_E_RANGE, "ingest: dispatch time range too wide");
            k_final_keys<<<gk, NT, 0, ctx->st>>>(kl, nk, O.pid, tl, tmin, tsbits, k1, v1);
            CH_LAUNCHED(ctx);
            CH_TRY(ch_radix_sort(ctx, k1, v1, k2, v2, nk, 0, tsbits + 8, &alt));
            k_final_gather<<<gk, NT, 0, ctx->st>>>(alt ? v2 : v1, nk, kl, tl, nid, O, out->t_l, out->t_ks, out->t_ke,
                                                   out->meta, out->name_id);
            CH_LAUNCHED(ctx);
        }
        rep->n_names = nu;
        if (ns > 0) {
            k_span_out<<<(unsigned)ceil_div(ns, NT), NT, 0, ctx->st>>>(sl, ns, O, out->span_gl, out->span_start,
                                                                       out->span_end, out->span_label, bad);
            CH_LAUNCHED(ctx);
        }
        CH_CUDA(ctx, cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, ctx->st));
        CH_CUDA(ctx, ch_sync(ctx));
        if (hbad) return ch_fail(ctx, CHOPPER_E_VALIDATION, "ingest: span gpu or level out of range");
        return CHOPPER_OK;
    }();
    restore();
    return st;
}
