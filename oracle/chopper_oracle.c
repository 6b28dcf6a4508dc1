/*
 * chopper_oracle.c -- TEST INFRASTRUCTURE ONLY (see chopper_oracle.h).
 *
 * A plain, slow, single-threaded reading of the Chopper analysis path
 * (arXiv 2512.08242).  Each block is labelled with the oracle step of
 * DESIGN.md ("O1".."O15"; O14/O15 are the report statistics of SURVEY §8(f)
 * row 1) and the paper passage it restates.  Methods are
 * deliberately the plain definitions: qsort + sequential loops, an
 * active-set sweep for span containment, explicit piecewise integration for
 * frequency / power, pairwise chain checks.  Nothing here is blocked, fused
 * or reordered for speed.
 *
 * Compile with -O2 -ffp-contract=off (no FMA contraction, D22).
 */
#define _GNU_SOURCE
#include "chopper_oracle.h"
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NONE_TS INT64_MIN

enum { K_COMPUTE = 0, K_AG = 1, K_RS = 2, K_COMM_OTHER = 3, K_COPY = 4, K_MEMOP = 5, K_OTHER = 6 };
enum { E_VALIDATION = 1, E_ALIGNMENT = 3, E_AMBIGUOUS = 4, E_RANGE = 5 };
enum {
    V_START_AFTER_END = 0, V_GPU_NOT_GROUPED, V_DISPATCH_DECREASING, V_BAD_META, V_TS_RANGE,
    V_STREAM_OVERLAP, V_SPAN_BAD, V_SAMPLES_UNSORTED, V_COUNTER_NONFINITE, V_NRULES
};

/* ------------------------------------------------------------------ */
/* result registry                                                      */
/* ------------------------------------------------------------------ */
typedef struct { char name[48]; void *ptr; int64_t n; int32_t dtype; } or_array;
struct or_result { or_array a[512]; int32_t n; };

static void *xcalloc(int64_t n, size_t sz) {
    void *p = calloc((size_t)(n > 0 ? n : 1), sz);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}
static void put(or_result *r, const char *name, void *ptr, int64_t n, int32_t dtype) {
    or_array *a = &r->a[r->n++];
    snprintf(a->name, sizeof a->name, "%s", name);
    a->ptr = ptr; a->n = n; a->dtype = dtype;
}
static int64_t *new_i64(or_result *r, const char *name, int64_t n, int64_t fill) {
    int64_t *p = (int64_t *)xcalloc(n, 8);
    for (int64_t i = 0; i < n; i++) p[i] = fill;
    put(r, name, p, n, 1);
    return p;
}
static int32_t *new_i32(or_result *r, const char *name, int64_t n, int32_t fill) {
    int32_t *p = (int32_t *)xcalloc(n, 4);
    for (int64_t i = 0; i < n; i++) p[i] = fill;
    put(r, name, p, n, 0);
    return p;
}
static double *new_f64(or_result *r, const char *name, int64_t n) {
    double *p = (double *)xcalloc(n, 8);
    put(r, name, p, n, 2);
    return p;
}

int32_t or_get(const or_result *r, const char *name, void **ptr, int64_t *n, int32_t *dtype) {
    for (int32_t i = 0; i < r->n; i++)
        if (strcmp(r->a[i].name, name) == 0) { *ptr = r->a[i].ptr; *n = r->a[i].n; *dtype = r->a[i].dtype; return 0; }
    return -1;
}
int32_t or_count(const or_result *r) { return r->n; }
const char *or_name(const or_result *r, int32_t i) { return (i >= 0 && i < r->n) ? r->a[i].name : NULL; }
void or_free(or_result *r) {
    if (!r) return;
    for (int32_t i = 0; i < r->n; i++) free(r->a[i].ptr);
    free(r);
}

/* ------------------------------------------------------------------ */
/* small helpers                                                        */
/* ------------------------------------------------------------------ */
static int kind_of(uint32_t m) { return (int)(m & 0xFFu); }
static int stream_of(uint32_t m) { return (int)((m >> 8) & 0xFFFFu); }
static int gpu_of(uint32_t m) { return (int)(m >> 24); }
static int is_comm(int k) { return k == K_AG || k == K_RS || k == K_COMM_OTHER; }
static int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}
static int cmp_f64(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}
/* median of a copy; even count = mean of the two central values (D21) */
static double median_i64(const int64_t *v, int64_t n) {
    int64_t *c = (int64_t *)xcalloc(n, 8);
    memcpy(c, v, (size_t)n * 8);
    qsort(c, (size_t)n, 8, cmp_i64);
    double m = (n % 2) ? (double)c[n / 2] : 0.5 * ((double)c[n / 2 - 1] + (double)c[n / 2]);
    free(c);
    return m;
}
static double median_f64(const double *v, int64_t n) {
    double *c = (double *)xcalloc(n, 8);
    memcpy(c, v, (size_t)n * 8);
    qsort(c, (size_t)n, 8, cmp_f64);
    double m = (n % 2) ? c[n / 2] : 0.5 * (c[n / 2 - 1] + c[n / 2]);
    free(c);
    return m;
}

/* quantile of sorted values at q in [0, 1]: linear interpolation between the order statistics at
   h = q (n - 1) (R9; q = 0.5 is the D21 median up to the rounding of the interpolation) */
static double quantile_sorted(const double *x, int64_t n, double q) {
    double h = q * (double)(n - 1);
    int64_t lo = (int64_t)floor(h);
    if (lo >= n - 1) return x[n - 1];
    double fr = h - (double)lo;
    return x[lo] + fr * (x[lo + 1] - x[lo]);
}

/* ------------------------------------------------------------------ */
/* O2: stable sort of events by (gpu, group, t_ks) (D1)                 */
/* ------------------------------------------------------------------ */
static int group_of(uint32_t m) {
    int k = kind_of(m);
    if (is_comm(k)) return 0;
    if (k == K_COMPUTE) return 1 + stream_of(m);
    return 255;
}
typedef struct { const or_input *in; } sort_ctx;
static int cmp_event_sorted(const void *a, const void *b, void *arg) {
    const or_input *in = ((const sort_ctx *)arg)->in;
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    int gi = gpu_of(in->meta[i]), gj = gpu_of(in->meta[j]);
    if (gi != gj) return gi < gj ? -1 : 1;
    int ri = group_of(in->meta[i]), rj = group_of(in->meta[j]);
    if (ri != rj) return ri < rj ? -1 : 1;
    if (in->t_ks[i] != in->t_ks[j]) return in->t_ks[i] < in->t_ks[j] ? -1 : 1;
    return (i > j) - (i < j);  /* ties: input (dispatch) order */
}

/* ------------------------------------------------------------------ */
/* O6/O7: interval unions                                               */
/* ------------------------------------------------------------------ */
typedef struct { int64_t s, e; } ival;
static int cmp_ival(const void *a, const void *b) {
    const ival *x = (const ival *)a, *y = (const ival *)b;
    if (x->s != y->s) return x->s < y->s ? -1 : 1;
    return (x->e > y->e) - (x->e < y->e);
}
/* merge intervals (sorted in place by start); returns merged count */
static int64_t merge_ivals(ival *v, int64_t n) {
    qsort(v, (size_t)n, sizeof(ival), cmp_ival);
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++) {
        if (v[i].e <= v[i].s) continue;                /* empty interval */
        if (m > 0 && v[i].s <= v[m - 1].e) { if (v[i].e > v[m - 1].e) v[m - 1].e = v[i].e; }
        else v[m++] = v[i];
    }
    return m;
}
/* |[a,b) ∩ U| : plain sum over the merged intervals that can touch [a,b) */
static int64_t inter_len(const ival *u, int64_t m, int64_t a, int64_t b) {
    if (b <= a || m == 0) return 0;
    int64_t lo = 0, hi = m;                           /* first interval with e > a */
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (u[mid].e > a) hi = mid; else lo = mid + 1; }
    int64_t tot = 0;
    for (int64_t k = lo; k < m && u[k].s < b; k++) {
        int64_t x = i64max(a, u[k].s), y = i64min(b, u[k].e);
        if (y > x) tot += y - x;
    }
    return tot;
}

/* ------------------------------------------------------------------ */
/* spans: push-order ranks (start asc, end desc, index desc), per (g,l) */
/* ------------------------------------------------------------------ */
static int cmp_span_push(const void *a, const void *b, void *arg) {
    const or_input *in = ((const sort_ctx *)arg)->in;
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    if (in->span_gl[i] != in->span_gl[j]) return in->span_gl[i] < in->span_gl[j] ? -1 : 1;
    if (in->span_start[i] != in->span_start[j]) return in->span_start[i] < in->span_start[j] ? -1 : 1;
    if (in->span_end[i] != in->span_end[j]) return in->span_end[i] > in->span_end[j] ? -1 : 1;
    return (i < j) - (i > j);
}

/* ------------------------------------------------------------------ */
/* table rows (O10/O11)                                                 */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t gpu, it, ph, ly, op, label;     /* caller span indices (-1 none) */
    int64_t r_it, r_ph, r_ly, r_op;         /* push-order rank + 1 (0 none) */
    int64_t n_events, n, busy, first_ks, first_idx, first_pred, last_ke;
    int64_t prep, call, ovl, phi, psi, copy_ns, ag_ns, rs_ns;
    double *cnt;                            /* [C] */
} row_t;

static void row_init(row_t *w, int C) {
    memset(w, 0, sizeof *w);
    w->first_ks = INT64_MAX; w->first_idx = INT64_MAX; w->first_pred = NONE_TS; w->last_ke = INT64_MIN;
    w->cnt = (double *)xcalloc(C, 8);
}
/* parent += child, children visited in ascending key order (D12) */
static void row_add(row_t *p, const row_t *c, int C) {
    p->n_events += c->n_events; p->n += c->n; p->busy += c->busy;
    if (c->first_ks < p->first_ks || (c->first_ks == p->first_ks && c->first_idx < p->first_idx)) {
        p->first_ks = c->first_ks; p->first_idx = c->first_idx; p->first_pred = c->first_pred;
    }
    if (c->last_ke > p->last_ke) p->last_ke = c->last_ke;
    p->prep += c->prep; p->call += c->call; p->ovl += c->ovl; p->phi += c->phi; p->psi += c->psi;
    p->copy_ns += c->copy_ns; p->ag_ns += c->ag_ns; p->rs_ns += c->rs_ns;
    for (int c2 = 0; c2 < C; c2++) p->cnt[c2] += c->cnt[c2];
}

static void emit_rows(or_result *r, const char *pfx, row_t *rows, int64_t n, int C) {
    char nm[48];
#define COL32(field) do { snprintf(nm, sizeof nm, "%s." #field, pfx); int32_t *p = new_i32(r, nm, n, 0); \
        for (int64_t i = 0; i < n; i++) p[i] = rows[i].field; } while (0)
#define COL64(field) do { snprintf(nm, sizeof nm, "%s." #field, pfx); int64_t *p = new_i64(r, nm, n, 0); \
        for (int64_t i = 0; i < n; i++) p[i] = rows[i].field; } while (0)
    COL32(gpu); COL32(it); COL32(ph); COL32(ly); COL32(op); COL32(label);
    COL64(n_events); COL64(n); COL64(busy); COL64(first_ks); COL64(first_idx); COL64(first_pred);
    COL64(last_ke); COL64(prep); COL64(call); COL64(ovl); COL64(phi); COL64(psi);
    COL64(copy_ns); COL64(ag_ns); COL64(rs_ns);
#undef COL32
#undef COL64
    snprintf(nm, sizeof nm, "%s.counters", pfx);
    double *cc = new_f64(r, nm, (int64_t)C * n);
    for (int c = 0; c < C; c++)
        for (int64_t i = 0; i < n; i++) cc[(int64_t)c * n + i] = rows[i].cnt[c];
}

/* rows sorted by key prefix: group consecutive rows with equal prefix of length depth (1..4) */
static int same_prefix(const row_t *a, const row_t *b, int depth) {
    if (a->gpu != b->gpu) return 0;
    if (depth >= 2 && a->r_it != b->r_it) return 0;
    if (depth >= 3 && a->r_ph != b->r_ph) return 0;
    if (depth >= 4 && a->r_ly != b->r_ly) return 0;
    return 1;
}
static row_t *rollup(const row_t *child, int64_t nc, int depth, int C, int64_t *n_out) {
    row_t *out = (row_t *)xcalloc(nc, sizeof(row_t));
    int64_t m = 0;
    for (int64_t i = 0; i < nc; i++) {
        if (m == 0 || !same_prefix(&out[m - 1], &child[i], depth)) {
            row_init(&out[m], C);
            out[m].gpu = child[i].gpu;
            out[m].it = child[i].it; out[m].r_it = child[i].r_it;
            out[m].ph = depth >= 3 ? child[i].ph : -1; out[m].r_ph = depth >= 3 ? child[i].r_ph : 0;
            out[m].ly = depth >= 4 ? child[i].ly : -1; out[m].r_ly = depth >= 4 ? child[i].r_ly : 0;
            if (depth < 2) { out[m].it = -1; out[m].r_it = 0; }
            out[m].op = -1; out[m].label = -1;
            m++;
        }
        row_add(&out[m - 1], &child[i], C);
    }
    *n_out = m;
    return out;
}

/* instance ordering key: (g, rank tuple), ties input index */
typedef struct { int64_t k[5]; int64_t i; } ek_t;
static int cmp_ek(const void *a, const void *b) {
    const ek_t *x = (const ek_t *)a, *y = (const ek_t *)b;
    for (int c = 0; c < 5; c++) if (x->k[c] != y->k[c]) return x->k[c] < y->k[c] ? -1 : 1;
    return (x->i > y->i) - (x->i < y->i);
}
/* point ordering: (label, g, iteration rank), ties instance row order */
static int cmp_pt(const void *a, const void *b, void *arg) {
    const row_t *inst = (const row_t *)arg;
    const row_t *x = &inst[*(const int64_t *)a], *y = &inst[*(const int64_t *)b];
    if (x->label != y->label) return x->label < y->label ? -1 : 1;
    if (x->gpu != y->gpu) return x->gpu < y->gpu ? -1 : 1;
    if (x->r_it != y->r_it) return x->r_it < y->r_it ? -1 : 1;
    int64_t a1 = *(const int64_t *)a, b1 = *(const int64_t *)b;
    return (a1 > b1) - (a1 < b1);
}

/* ------------------------------------------------------------------ */
/* O13: gap decomposition for one op label                              */
/* ------------------------------------------------------------------ */
typedef struct { int64_t busy, launch, ovl, phi; double cg, fp, un, ud; } point_t;
enum { BD_FIT = 1, BD_NO_FLOPS = 2, BD_NO_UTIL = 4, BD_UTIL_RANGE = 8, BD_D0_ZERO = 16, BD_NO_CYCLES = 32,
       BD_NO_SAMPLES = 64, BD_INSUFFICIENT = 128 };
#define N_BD 16
#define N_RS 16
/* out fields: 0 n_points,1 method,2 D_act_s,3 D0_s,4 D50_s,5 D_thr,6 Ovr_inst,7 Ovr_util,8 Ovr_overlap,
   9 D_peak,10 Ovr_freq,11 Ovr_launch,12 residual,13 Ovr_freq_samples,14 flags,15 label */
static void breakdown_label(const or_input *in, int L, const point_t *p, int64_t n, int has_cyc, int has_fl,
                            int has_util, int has_smp, double *out) {
    for (int i = 0; i < N_BD; i++) out[i] = NAN;
    int flags = 0;
    out[0] = (double)n; out[15] = (double)L;
    if (n < 2) { out[14] = BD_INSUFFICIENT; out[1] = 0; return; }
    int64_t *b = (int64_t *)xcalloc(n, 8), *bl = (int64_t *)xcalloc(n, 8);
    int64_t *b0 = (int64_t *)xcalloc(n, 8), *b50 = (int64_t *)xcalloc(n, 8);
    double *v = (double *)xcalloc(n, 8);
    int64_t n0 = 0, n50 = 0;
    for (int64_t i = 0; i < n; i++) {
        b[i] = p[i].busy; bl[i] = p[i].busy + p[i].launch;
        if (20 * p[i].ovl <= p[i].busy) b0[n0++] = p[i].busy;                                   /* r <= 0.05 */
        if (2 * p[i].busy <= 5 * p[i].ovl && 5 * p[i].ovl <= 3 * p[i].busy) b50[n50++] = p[i].busy; /* 0.4<=r<=0.6 */
    }
    double d_act = median_i64(b, n), d0, d50;
    if (n0 > 0 && n50 > 0) {
        d0 = median_i64(b0, n0); d50 = median_i64(b50, n50); out[1] = 0;
    } else {
        /* least-squares busy ~ a + c*r, two-pass means, sequential (g, it) order (D15) */
        double sr = 0.0, sb = 0.0;
        for (int64_t i = 0; i < n; i++) { sr += (double)p[i].ovl / (double)p[i].busy; sb += (double)p[i].busy; }
        double mr = sr / (double)n, mb = sb / (double)n, sxx = 0.0, sxy = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double dr = (double)p[i].ovl / (double)p[i].busy - mr, db = (double)p[i].busy - mb;
            sxx += dr * dr; sxy += dr * db;
        }
        if (sxx == 0.0) { d0 = d_act; d50 = d_act; }
        else { double c = sxy / sxx, a = mb - c * mr; d0 = a; d50 = a + c * 0.5; }
        out[1] = 1; flags |= BD_FIT;
    }
    out[2] = d_act * 1e-9; out[3] = d0 * 1e-9; out[4] = d50 * 1e-9;
    double d_thr = in->f_gemm[L] / in->tpt_peak; out[5] = d_thr;
    double ovr_inst = 1.0;
    if (has_fl) { for (int64_t i = 0; i < n; i++) v[i] = p[i].fp; ovr_inst = median_f64(v, n) / in->f_gemm[L]; }
    else flags |= BD_NO_FLOPS;
    out[6] = ovr_inst;
    double ovr_util = 1.0;
    if (has_util || (has_fl && has_cyc)) {
        for (int64_t i = 0; i < n; i++)
            v[i] = has_util ? p[i].un / p[i].ud : (p[i].fp / p[i].cg) * (in->freq_peak_hz / in->tpt_peak);
        double u = median_f64(v, n);
        if (!(u > 0.0 && u <= 1.0)) flags |= BD_UTIL_RANGE;
        ovr_util = 1.0 / u;
    } else flags |= BD_NO_UTIL;
    out[7] = ovr_util;
    double ovr_ovl = d50 / d0;
    if (!(d0 > 0.0)) flags |= BD_D0_ZERO;
    out[8] = ovr_ovl;
    if (has_cyc) {
        for (int64_t i = 0; i < n; i++) v[i] = p[i].cg;
        double d_peak = median_f64(v, n) / in->freq_peak_hz;
        out[9] = d_peak;
        out[10] = (d_act * 1e-9 / d_peak) / ovr_ovl;
    } else flags |= BD_NO_CYCLES;
    out[11] = median_i64(bl, n) / d_act;
    out[12] = d_act * 1e-9 / (d_thr * ovr_inst * ovr_util * ovr_ovl * out[10]);
    if (has_smp) {
        for (int64_t i = 0; i < n; i++) v[i] = (double)p[i].phi / (double)p[i].busy * 1e6;
        out[13] = in->freq_peak_hz / median_f64(v, n);
    } else flags |= BD_NO_SAMPLES;
    out[14] = (double)flags;
    free(b); free(bl); free(b0); free(b50); free(v);
}

/* ------------------------------------------------------------------ */
/* main                                                                 */
/* ------------------------------------------------------------------ */
or_result *or_run(const or_input *in) {
    or_result *r = (or_result *)xcalloc(1, sizeof(or_result));
    const int64_t N = in->n_events, S = in->n_spans, NS = in->n_samples;
    const int G = in->n_traced_gpus, C = in->n_counters;
    int64_t *vcount = new_i64(r, "val.count", V_NRULES, 0);
    int64_t *vfirst = new_i64(r, "val.first", V_NRULES, -1);
    int64_t *status = new_i64(r, "status", 1, 0);
#define VIOL(rule, idx) do { vcount[rule]++; if (vfirst[rule] < 0 || (idx) < vfirst[rule]) vfirst[rule] = (idx); } while (0)

    /* ---------------- O1 validate ---------------- */
    int64_t tmin = INT64_MAX, tmax = INT64_MIN;
    for (int64_t i = 0; i < N; i++) {
        uint32_t m = in->meta[i];
        if (in->t_ks[i] > in->t_ke[i]) VIOL(V_START_AFTER_END, i);
        if (i > 0 && gpu_of(m) < gpu_of(in->meta[i - 1])) VIOL(V_GPU_NOT_GROUPED, i);
        if (i > 0 && gpu_of(m) == gpu_of(in->meta[i - 1]) && in->t_l[i] < in->t_l[i - 1]) VIOL(V_DISPATCH_DECREASING, i);
        if (kind_of(m) > K_OTHER || gpu_of(m) >= G || (kind_of(m) == K_COMPUTE && stream_of(m) > 253)) VIOL(V_BAD_META, i);
        tmin = i64min(tmin, i64min(in->t_l[i], i64min(in->t_ks[i], in->t_ke[i])));
        tmax = i64max(tmax, i64max(in->t_l[i], i64max(in->t_ks[i], in->t_ke[i])));
    }
    if (N > 0 && (uint64_t)tmax - (uint64_t)tmin >= (1ull << 52)) VIOL(V_TS_RANGE, 0);
    for (int64_t j = 0; j < S; j++)
        if (in->span_end[j] < in->span_start[j] || (in->span_gl[j] & 0xFFu) > 3 || (int)(in->span_gl[j] >> 8) >= G)
            VIOL(V_SPAN_BAD, j);
    for (int64_t k = 0; k < NS; k++) {
        if (in->smp_gpu[k] < 0 || in->smp_gpu[k] >= G) VIOL(V_SAMPLES_UNSORTED, k);
        else if (k > 0 && (in->smp_gpu[k] < in->smp_gpu[k - 1] ||
                           (in->smp_gpu[k] == in->smp_gpu[k - 1] && in->smp_ts[k] < in->smp_ts[k - 1])))
            VIOL(V_SAMPLES_UNSORTED, k);
    }
    for (int rule = 0; rule < V_NRULES; rule++)
        if (vcount[rule]) status[0] |= 1 << E_VALIDATION;
    if (status[0]) return r;   /* fatal load-time violations: nothing else is defined */

    /* per-gpu event ranges (events grouped by gpu) */
    int64_t *gbeg = (int64_t *)xcalloc(G + 1, 8), *gend = (int64_t *)xcalloc(G + 1, 8);
    for (int g = 0; g < G; g++) { gbeg[g] = 0; gend[g] = 0; }
    for (int64_t i = 0; i < N; i++) {
        int g = gpu_of(in->meta[i]);
        if (i == 0 || g != gpu_of(in->meta[i - 1])) gbeg[g] = i;
        gend[g] = i + 1;
    }

    /* ---------------- O2 sort + same-stream disjointness + chain ---------------- */
    int64_t *ord = (int64_t *)xcalloc(N, 8);
    for (int64_t i = 0; i < N; i++) ord[i] = i;
    sort_ctx sc = { in };
    qsort_r(ord, (size_t)N, 8, cmp_event_sorted, &sc);
    int64_t *pred = new_i64(r, "ev.pred", N, -1);      /* O8 predecessor (input index) or -1 */
    for (int64_t j = 1; j < N; j++) {
        int64_t a = ord[j - 1], b = ord[j];
        int ga = group_of(in->meta[a]), gb = group_of(in->meta[b]);
        if (gpu_of(in->meta[a]) == gpu_of(in->meta[b]) && ga == gb && gb >= 1 && gb <= 254) {
            pred[b] = a;
            if (in->t_ks[b] < in->t_ke[a]) VIOL(V_STREAM_OVERLAP, b);
        }
    }
    if (vcount[V_STREAM_OVERLAP]) status[0] |= 1 << E_VALIDATION;

    /* ---------------- O8 launch overhead, Eqs. 1-3, D6 ---------------- */
    int64_t *prep = new_i64(r, "ev.prep", N, 0), *call = new_i64(r, "ev.call", N, 0);
    for (int64_t i = 0; i < N; i++) {
        if (kind_of(in->meta[i]) != K_COMPUTE || pred[i] < 0) continue;
        int64_t pe = in->t_ke[pred[i]];
        int64_t tl = i64min(in->t_l[i], in->t_ks[i]);
        prep[i] = i64max(tl - pe, 0);
        call[i] = i64max(i64min(in->t_ks[i] - tl, in->t_ks[i] - pe), 0);
    }

    /* ---------------- O6/O7 unions and overlap (D9) ---------------- */
    int64_t *ovl = new_i64(r, "ev.ovl", N, 0);
    ival **U = (ival **)xcalloc(G, sizeof(ival *)); int64_t *nU = (int64_t *)xcalloc(G, 8);
    for (int g = 0; g < G; g++) {
        int64_t nb = gend[g] - gbeg[g];
        ival *cu = (ival *)xcalloc(nb, sizeof(ival)), *cv = (ival *)xcalloc(nb, sizeof(ival));
        int64_t nc = 0, nv = 0;
        for (int64_t i = gbeg[g]; i < gend[g]; i++) {
            int k = kind_of(in->meta[i]);
            if (is_comm(k)) { cu[nc].s = in->t_ks[i]; cu[nc].e = in->t_ke[i]; nc++; }
            if (k == K_COMPUTE) { cv[nv].s = in->t_ks[i]; cv[nv].e = in->t_ke[i]; nv++; }
        }
        nc = merge_ivals(cu, nc); nv = merge_ivals(cv, nv);
        for (int64_t i = gbeg[g]; i < gend[g]; i++) {
            int k = kind_of(in->meta[i]);
            if (k == K_COMPUTE) ovl[i] = inter_len(cu, nc, in->t_ks[i], in->t_ke[i]);
            else if (is_comm(k)) ovl[i] = inter_len(cv, nv, in->t_ks[i], in->t_ke[i]);
        }
        U[g] = cu; nU[g] = nc;
        free(cv);
    }

    /* ---------------- O9 frequency / power integrals, zero-order hold (D10) ---------------- */
    int64_t *phi = new_i64(r, "ev.phi", N, 0), *psi = new_i64(r, "ev.psi", N, 0);
    int32_t *has_smp = new_i32(r, "gpu.has_samples", G, 0);
    {
        int64_t k0 = 0;
        for (int g = 0; g < G; g++) {
            int64_t k1 = k0;
            while (k1 < NS && in->smp_gpu[k1] == g) k1++;
            int64_t K = k1 - k0;
            if (K > 0) {
                has_smp[g] = 1;
                for (int64_t i = gbeg[g]; i < gend[g]; i++) {
                    if (kind_of(in->meta[i]) != K_COMPUTE) continue;
                    int64_t a = in->t_ks[i], b = in->t_ke[i], F = 0, P = 0;
                    /* pieces ending at or before a contribute nothing: start at the first piece with hi > a */
                    int64_t kl = 0, kh = K - 1;
                    while (kl < kh) {
                        int64_t m = (kl + kh) / 2;
                        if (in->smp_ts[k0 + m + 1] > a) kh = m; else kl = m + 1;
                    }
                    for (int64_t k = kl; k < K; k++) {  /* piece k: [lo, hi) with value sample k */
                        int64_t lo = (k == 0) ? INT64_MIN : in->smp_ts[k0 + k];
                        int64_t hi = (k == K - 1) ? INT64_MAX : in->smp_ts[k0 + k + 1];
                        int64_t x = i64max(a, lo), y = i64min(b, hi);
                        if (y > x) { F += (int64_t)in->smp_freq_mhz[k0 + k] * (y - x); P += (int64_t)in->smp_power_mw[k0 + k] * (y - x); }
                        if (hi >= b) break;
                    }
                    phi[i] = F; psi[i] = P;
                }
            }
            k0 = k1;
        }
    }

    /* ---------------- O5 attribution: active-set sweep per (g, level) (D3, D4) ---------------- */
    int32_t *aidx = new_i32(r, "ev.span_idx", 4 * N, -1);   /* [4][N] */
    int64_t *rank1 = (int64_t *)xcalloc(S, 8);              /* push-order rank + 1 (0: zero length) */
    {
        int64_t *so = (int64_t *)xcalloc(S, 8); int64_t ns = 0;
        for (int64_t j = 0; j < S; j++) if (in->span_end[j] > in->span_start[j]) so[ns++] = j;
        qsort_r(so, (size_t)ns, 8, cmp_span_push, &sc);
        for (int64_t q = 0; q < ns; q++) {
            int64_t rk = (q > 0 && in->span_gl[so[q - 1]] == in->span_gl[so[q]]) ? rank1[so[q - 1]] + 1 : 1;
            rank1[so[q]] = rk;
        }
        int64_t *act = (int64_t *)xcalloc(S, 8);
        for (int g = 0; g < G; g++) {
            for (int lv = 0; lv < 4; lv++) {
                uint32_t key = ((uint32_t)g << 8) | (uint32_t)lv;
                int64_t b0 = 0; while (b0 < ns && in->span_gl[so[b0]] < key) b0++;
                int64_t b1 = b0; while (b1 < ns && in->span_gl[so[b1]] == key) b1++;
                int64_t nxt = b0, na = 0;
                for (int64_t i = gbeg[g]; i < gend[g]; i++) {
                    int64_t t = in->t_l[i];
                    while (nxt < b1 && in->span_start[so[nxt]] <= t) act[na++] = so[nxt++];
                    int64_t w = 0;
                    for (int64_t q = 0; q < na; q++) if (in->span_end[act[q]] > t) act[w++] = act[q];
                    na = w;
                    if (na == 0) continue;
                    int64_t best = act[0];
                    for (int64_t q = 1; q < na; q++) {
                        int64_t c = act[q];
                        if (in->span_start[c] > in->span_start[best] ||
                            (in->span_start[c] == in->span_start[best] &&
                             (in->span_end[c] < in->span_end[best] || (in->span_end[c] == in->span_end[best] && c < best))))
                            best = c;
                    }
                    int chain = 1;
                    for (int64_t x = 0; x < na && chain; x++)
                        for (int64_t y = x + 1; y < na && chain; y++) {
                            int64_t u = act[x], v = act[y];
                            int nest = (in->span_start[u] <= in->span_start[v] && in->span_end[v] <= in->span_end[u]) ||
                                       (in->span_start[v] <= in->span_start[u] && in->span_end[u] <= in->span_end[v]);
                            if (!nest) chain = 0;
                        }
                    aidx[(int64_t)lv * N + i] = chain ? (int32_t)best : -2;
                    if (!chain) status[0] |= 1 << E_AMBIGUOUS;
                }
            }
        }
        free(act); free(so);
    }

    /* ---------------- O3 counter alignment (D2) ---------------- */
    double *cnt = new_f64(r, "ev.counters", (int64_t)C * N);
    int32_t *present = new_i32(r, "gpu.counter_present", (int64_t)G * (C > 0 ? C : 1), 0);
    int64_t *pass_mis = new_i64(r, "pass.mismatch", in->n_passes, -1);
    int64_t *pass_conf = new_i64(r, "pass.conflict", in->n_passes, -1);
    {
        int64_t *pos = (int64_t *)xcalloc(N, 8);   /* position of the j-th non-MEMOP event of g */
        uint8_t *filled = (uint8_t *)xcalloc((int64_t)C * N, 1);
        for (int p = 0; p < in->n_passes; p++) {
            int g = in->pass_gpu[p];
            if (g < 0 || g >= G) { pass_mis[p] = 0; status[0] |= 1 << E_ALIGNMENT; continue; }
            int64_t m = 0;
            for (int64_t i = gbeg[g]; i < gend[g]; i++) if (kind_of(in->meta[i]) != K_MEMOP) pos[m++] = i;
            int64_t np = in->pass_n[p], lim = np < m ? np : m, mis = -1;
            for (int64_t j = 0; j < lim; j++) if (in->pass_name_id[p][j] != in->name_id[pos[j]]) { mis = j; break; }
            if (mis < 0 && np != m) mis = lim;
            if (mis >= 0) { pass_mis[p] = mis; status[0] |= 1 << E_ALIGNMENT; continue; }
            int finite = 1;
            for (int kk = 0; kk < in->pass_k[p]; kk++)
                for (int64_t j = 0; j < np; j++) if (!isfinite(in->pass_values[p][(int64_t)kk * np + j])) finite = 0;
            if (!finite) { VIOL(V_COUNTER_NONFINITE, p); status[0] |= 1 << E_VALIDATION; continue; }
            int64_t conf = -1;
            for (int kk = 0; kk < in->pass_k[p]; kk++) {
                int sl = in->pass_slot[p][kk];
                if (sl < 0 || sl >= C) { conf = 0; continue; }
                for (int64_t j = 0; j < np; j++) {
                    int64_t i = pos[j];
                    double v = in->pass_values[p][(int64_t)kk * np + j];
                    if (filled[(int64_t)sl * N + i]) {
                        double a = cnt[(int64_t)sl * N + i];
                        if (fabs(a - v) > 1e-9 * fmax(fabs(a), fabs(v)) && (conf < 0 || j < conf)) conf = j;
                    } else { cnt[(int64_t)sl * N + i] = v; filled[(int64_t)sl * N + i] = 1; }
                }
                present[(int64_t)g * C + sl] = 1;
            }
            if (conf >= 0) { pass_conf[p] = conf; status[0] |= 1 << E_ALIGNMENT; }
        }
        free(pos); free(filled);
    }

    /* ---------------- O4 clock offsets: lower median of collective-end differences (D13) ---------------- */
    int64_t *delta = new_i64(r, "gpu.delta", G, 0);
    int32_t *delta_flag = new_i32(r, "gpu.delta_flag", G, 0);
    {
        int64_t *cntk[2] = { (int64_t *)xcalloc(G, 8), (int64_t *)xcalloc(G, 8) };
        int64_t **Ee[2], **Es[2];
        for (int k = 0; k < 2; k++) { Ee[k] = (int64_t **)xcalloc(G, sizeof(int64_t *)); Es[k] = (int64_t **)xcalloc(G, sizeof(int64_t *)); }
        int ref = -1;
        for (int g = 0; g < G; g++) {
            if (gend[g] > gbeg[g] && ref < 0) ref = g;
            for (int k = 0; k < 2; k++) {
                int want = k == 0 ? K_AG : K_RS;
                Ee[k][g] = (int64_t *)xcalloc(gend[g] - gbeg[g], 8); Es[k][g] = (int64_t *)xcalloc(gend[g] - gbeg[g], 8);
                for (int64_t i = gbeg[g]; i < gend[g]; i++)
                    if (kind_of(in->meta[i]) == want) { Es[k][g][cntk[k][g]] = in->t_ks[i]; Ee[k][g][cntk[k][g]++] = in->t_ke[i]; }
            }
        }
        int64_t mk[2] = { 0, 0 };
        for (int k = 0; k < 2; k++) {
            int first = 1;
            for (int g = 0; g < G; g++) {
                if (gend[g] <= gbeg[g]) continue;
                if (first || cntk[k][g] < mk[k]) mk[k] = cntk[k][g];
                first = 0;
            }
        }
        for (int g = 0; g < G; g++) {
            if (ref < 0 || gend[g] <= gbeg[g]) { delta_flag[g] = 1; continue; }
            int64_t nd = mk[0] + mk[1], q = 0;
            if (nd == 0) { delta_flag[g] = 1; continue; }
            int64_t *d = (int64_t *)xcalloc(nd, 8);
            for (int k = 0; k < 2; k++) for (int64_t j = 0; j < mk[k]; j++) d[q++] = Ee[k][g][j] - Ee[k][ref][j];
            qsort(d, (size_t)nd, 8, cmp_i64);
            delta[g] = d[(nd - 1) / 2];
            free(d);
        }
        for (int k = 0; k < 2; k++) {
            int64_t *sk = new_i64(r, k == 0 ? "skew.ag" : "skew.rs", mk[k], 0);
            for (int64_t j = 0; j < mk[k]; j++) {
                int64_t lo = INT64_MAX, hi = INT64_MIN;
                for (int g = 0; g < G; g++) {
                    if (gend[g] <= gbeg[g]) continue;
                    int64_t a = Es[k][g][j] - delta[g];
                    lo = i64min(lo, a); hi = i64max(hi, a);
                }
                sk[j] = hi - lo;
            }
            for (int g = 0; g < G; g++) { free(Ee[k][g]); free(Es[k][g]); }
            free(Ee[k]); free(Es[k]); free(cntk[k]);
        }
    }

    /* ---------------- O10 instance sums, sequential in input order ---------------- */
    int64_t n_inst = 0;
    row_t *inst;
    {
        /* events that belong to a table: A_it >= 0 and no ambiguous level */
        int64_t *sel = (int64_t *)xcalloc(N, 8), ns = 0;
        for (int64_t i = 0; i < N; i++) {
            int ok = aidx[i] >= 0;
            for (int lv = 0; lv < 4; lv++) if (aidx[(int64_t)lv * N + i] == -2) ok = 0;
            if (ok) sel[ns++] = i;
        }
        /* order by (g, rank tuple), ties input index: a plain insertion into key order */
        ek_t *ek = (ek_t *)xcalloc(ns, sizeof(ek_t));
        for (int64_t q = 0; q < ns; q++) {
            int64_t i = sel[q];
            ek[q].k[0] = gpu_of(in->meta[i]);
            for (int lv = 0; lv < 4; lv++) { int32_t a = aidx[(int64_t)lv * N + i]; ek[q].k[1 + lv] = a >= 0 ? rank1[a] : 0; }
            ek[q].i = i;
        }
        qsort(ek, (size_t)ns, sizeof(ek_t), cmp_ek);
        inst = (row_t *)xcalloc(ns, sizeof(row_t));
        for (int64_t q = 0; q < ns; q++) {
            int64_t i = ek[q].i;
            int newrow = q == 0;
            if (!newrow) for (int c = 0; c < 5; c++) if (ek[q].k[c] != ek[q - 1].k[c]) newrow = 1;
            if (newrow) {
                row_t *w = &inst[n_inst++];
                row_init(w, C);
                w->gpu = gpu_of(in->meta[i]);
                w->it = aidx[i]; w->ph = aidx[N + i]; w->ly = aidx[2 * N + i]; w->op = aidx[3 * N + i];
                w->r_it = ek[q].k[1]; w->r_ph = ek[q].k[2]; w->r_ly = ek[q].k[3]; w->r_op = ek[q].k[4];
                w->label = w->op >= 0 ? in->span_label[w->op] : -1;
            }
            row_t *w = &inst[n_inst - 1];
            int k = kind_of(in->meta[i]);
            int64_t dur = in->t_ke[i] - in->t_ks[i];
            w->n_events++;
            if (k == K_COMPUTE) {
                w->n++; w->busy += dur;
                if (in->t_ks[i] < w->first_ks || (in->t_ks[i] == w->first_ks && i < w->first_idx)) {
                    w->first_ks = in->t_ks[i]; w->first_idx = i; w->first_pred = pred[i] >= 0 ? in->t_ke[pred[i]] : NONE_TS;
                }
                if (in->t_ke[i] > w->last_ke) w->last_ke = in->t_ke[i];
                w->prep += prep[i]; w->call += call[i]; w->ovl += ovl[i]; w->phi += phi[i]; w->psi += psi[i];
                for (int c = 0; c < C; c++) w->cnt[c] += cnt[(int64_t)c * N + i];
            } else if (k == K_COPY || k == K_OTHER) w->copy_ns += dur;
            else if (k == K_AG) w->ag_ns += dur;
            else if (k == K_RS) w->rs_ns += dur;
        }
        free(sel); free(ek);
    }
    emit_rows(r, "inst", inst, n_inst, C);

    /* ---------------- O11 roll-ups (D12) ---------------- */
    int64_t n_ly, n_ph, n_itr, n_gpu;
    row_t *ly = rollup(inst, n_inst, 4, C, &n_ly);
    row_t *ph = rollup(ly, n_ly, 3, C, &n_ph);
    row_t *itr = rollup(ph, n_ph, 2, C, &n_itr);
    row_t *gp = rollup(itr, n_itr, 1, C, &n_gpu);
    emit_rows(r, "layer", ly, n_ly, C);
    emit_rows(r, "phase", ph, n_ph, C);
    emit_rows(r, "iter", itr, n_itr, C);
    emit_rows(r, "gpu", gp, n_gpu, C);
    {
        int64_t *w = new_i64(r, "iter.wall", n_itr, 0), *cu = new_i64(r, "iter.comm_union", n_itr, 0);
        int64_t *af = new_i64(r, "iter.aligned_first", n_itr, 0), *al = new_i64(r, "iter.aligned_last", n_itr, 0);
        int32_t *lab = new_i32(r, "iter.step", n_itr, 0), *rk = new_i32(r, "iter.rank", n_itr, 0);
        for (int64_t q = 0; q < n_itr; q++) {
            row_t *x = &itr[q];
            lab[q] = in->span_label[x->it]; rk[q] = (int32_t)(x->r_it - 1);
            if (x->n > 0) {
                w[q] = x->last_ke - (x->first_pred != NONE_TS ? x->first_pred : x->first_ks);
                cu[q] = inter_len(U[x->gpu], nU[x->gpu], x->first_ks, x->last_ke);
                af[q] = x->first_ks - delta[x->gpu]; al[q] = x->last_ke - delta[x->gpu];
            }
        }
        /* derived ratio-of-sums rates per iteration row */
        double *rt = new_f64(r, "iter.rates", (int64_t)in->n_ratios * n_itr);
        for (int q = 0; q < in->n_ratios; q++)
            for (int64_t x = 0; x < n_itr; x++) {
                double num = itr[x].cnt[in->ratio_num[q]];
                double den = in->ratio_den[q] < 0 ? (double)itr[x].busy * 1e-9 : itr[x].cnt[in->ratio_den[q]];
                rt[(int64_t)q * n_itr + x] = num / den * in->ratio_scale[q];
            }
    }

    /* ---------------- points (g, it, label): summed across layers ---------------- */
    int64_t n_pt = 0;
    row_t *pt;
    {
        int64_t *ix = (int64_t *)xcalloc(n_inst, 8), nx = 0;
        for (int64_t q = 0; q < n_inst; q++) if (inst[q].op >= 0) ix[nx++] = q;
        qsort_r(ix, (size_t)nx, 8, cmp_pt, inst);
        pt = (row_t *)xcalloc(nx, sizeof(row_t));
        for (int64_t q = 0; q < nx; q++) {
            const row_t *c = &inst[ix[q]];
            if (n_pt == 0 || pt[n_pt - 1].label != c->label || pt[n_pt - 1].gpu != c->gpu || pt[n_pt - 1].r_it != c->r_it) {
                row_init(&pt[n_pt], C);
                pt[n_pt].gpu = c->gpu; pt[n_pt].it = c->it; pt[n_pt].r_it = c->r_it;
                pt[n_pt].ph = pt[n_pt].ly = pt[n_pt].op = -1; pt[n_pt].label = c->label;
                n_pt++;
            }
            row_add(&pt[n_pt - 1], c, C);
        }
        free(ix);
    }
    emit_rows(r, "point", pt, n_pt, C);
    {
        double *rt = new_f64(r, "point.rates", (int64_t)in->n_ratios * n_pt);
        for (int q = 0; q < in->n_ratios; q++)
            for (int64_t x = 0; x < n_pt; x++) {
                double num = pt[x].cnt[in->ratio_num[q]];
                double den = in->ratio_den[q] < 0 ? (double)pt[x].busy * 1e-9 : pt[x].cnt[in->ratio_den[q]];
                rt[(int64_t)q * n_pt + x] = num / den * in->ratio_scale[q];
            }
        int32_t *rk = new_i32(r, "point.rank", n_pt, 0);
        for (int64_t x = 0; x < n_pt; x++) rk[x] = (int32_t)(pt[x].r_it - 1);
    }

    /* ---------------- O12 global iterations and throughput ---------------- */
    {
        int ref = -1;
        for (int g = 0; g < G && ref < 0; g++) if (gend[g] > gbeg[g]) ref = g;
        int64_t nref = 0;
        for (int64_t q = 0; q < n_itr; q++) if (itr[q].gpu == ref) nref++;
        int32_t *gstep = new_i32(r, "glob.step", nref, 0), *gok = new_i32(r, "glob.complete", nref, 0);
        int32_t *gsamp = new_i32(r, "glob.sampled", nref, 0);
        int64_t *gT = new_i64(r, "glob.T", nref, 0), *gfirst = new_i64(r, "glob.aligned_first", nref, 0);
        int64_t *glast = new_i64(r, "glob.aligned_last", nref, 0);
        double *gtp = new_f64(r, "glob.throughput", nref);
        double *sampled_tp = (double *)xcalloc(nref, 8); int64_t nst = 0;
        int64_t w = 0;
        for (int64_t q = 0; q < n_itr; q++) {
            if (itr[q].gpu != ref) continue;
            int32_t step = in->span_label[itr[q].it];
            int complete = 1, samp = 1;
            int64_t T = INT64_MIN, lo = INT64_MAX, hi = INT64_MIN;
            for (int g = 0; g < G; g++) {
                if (gend[g] <= gbeg[g]) continue;
                int64_t f = -1;
                for (int64_t x = 0; x < n_itr; x++)
                    if (itr[x].gpu == g && in->span_label[itr[x].it] == step) { f = x; break; }
                if (f < 0) { complete = 0; continue; }
                if (itr[f].r_it - 1 < in->warmup) samp = 0;
                T = i64max(T, itr[f].busy + itr[f].prep + itr[f].call);
                if (itr[f].n > 0) { lo = i64min(lo, itr[f].first_ks - delta[g]); hi = i64max(hi, itr[f].last_ke - delta[g]); }
            }
            gstep[w] = step; gok[w] = complete; gsamp[w] = complete && samp;
            gT[w] = complete ? T : 0; gfirst[w] = lo; glast[w] = hi;
            gtp[w] = complete ? (double)(in->b * in->s * in->R) / ((double)T * 1e-9) : NAN;
            if (complete && samp) sampled_tp[nst++] = gtp[w];
            w++;
        }
        double *med = new_f64(r, "glob.throughput_median", 1);
        med[0] = nst > 0 ? median_f64(sampled_tp, nst) : NAN;
        free(sampled_tp);
    }

    /* ---------------- O13 breakdown per gemm / fa label ---------------- */
    {
        int64_t nrow = 0;
        for (int L = 0; L < in->n_labels; L++) if (in->op_type[L] == 1 || in->op_type[L] == 2) nrow++;
        double *bd = new_f64(r, "bd.rows", nrow * N_BD);
        point_t *pp = (point_t *)xcalloc(n_pt, sizeof(point_t));
        int64_t w = 0;
        for (int L = 0; L < in->n_labels; L++) {
            if (!(in->op_type[L] == 1 || in->op_type[L] == 2)) continue;
            int64_t np = 0;
            int cyc = in->slot_cycles >= 0, fl = in->slot_flops >= 0;
            int ut = in->slot_unum >= 0 && in->slot_uden >= 0, sm = 1;
            for (int64_t x = 0; x < n_pt; x++) {
                const row_t *p = &pt[x];
                if (p->label != L || p->r_it - 1 < in->warmup || p->busy <= 0) continue;
                if (!((in->bd_gpu_mask >> p->gpu) & 1ull)) continue;
                point_t *o = &pp[np++];
                o->busy = p->busy; o->launch = p->prep + p->call; o->ovl = p->ovl; o->phi = p->phi;
                o->cg = cyc ? p->cnt[in->slot_cycles] : 0; o->fp = fl ? p->cnt[in->slot_flops] : 0;
                o->un = ut ? p->cnt[in->slot_unum] : 0; o->ud = ut ? p->cnt[in->slot_uden] : 0;
                if (cyc && !present[(int64_t)p->gpu * C + in->slot_cycles]) cyc = 0;
                if (fl && !present[(int64_t)p->gpu * C + in->slot_flops]) fl = 0;
                if (ut && !(present[(int64_t)p->gpu * C + in->slot_unum] && present[(int64_t)p->gpu * C + in->slot_uden])) ut = 0;
                if (!has_smp[p->gpu]) sm = 0;
            }
            breakdown_label(in, L, pp, np, cyc, fl, ut, sm && np > 0, &bd[w * N_BD]);
            w++;
        }
        free(pp);
    }

    /* ---------------- O14 report statistics per op label ----
       Over the same points as O13 (sampled iterations, busy > 0, all op labels), in (gpu, iteration) order:
       duration and overlap-ratio quantiles (min, q25, median, q75, max; R9) -- the fills of Fig. 6 -- and the
       Pearson correlation of overlap ratio with duration (R10; NaN when either is constant, as the paper's
       "low or nan values").  Row: 0 n, 1-5 duration q0..q100 (ns), 6-10 ratio q0..q100, 11 pearson,
       12 label, 13 mean duration (ns), 14-15 NaN. */
    {
        double *rs = new_f64(r, "report.rows", (int64_t)in->n_labels * N_RS);
        double *b = (double *)xcalloc(n_pt > 0 ? n_pt : 1, 8), *rr = (double *)xcalloc(n_pt > 0 ? n_pt : 1, 8);
        double *sb = (double *)xcalloc(n_pt > 0 ? n_pt : 1, 8), *sr = (double *)xcalloc(n_pt > 0 ? n_pt : 1, 8);
        for (int L = 0; L < in->n_labels; L++) {
            double *o = &rs[(int64_t)L * N_RS];
            for (int k = 0; k < N_RS; k++) o[k] = NAN;
            int64_t n = 0;
            for (int64_t x = 0; x < n_pt; x++) {
                const row_t *pr = &pt[x];
                if (pr->label != L || pr->r_it - 1 < in->warmup || pr->busy <= 0) continue;
                if (!((in->bd_gpu_mask >> pr->gpu) & 1ull)) continue;
                b[n] = (double)pr->busy;
                rr[n] = (double)pr->ovl / (double)pr->busy;
                n++;
            }
            o[0] = (double)n;
            o[12] = (double)L;
            if (n == 0) continue;
            memcpy(sb, b, (size_t)n * 8);
            memcpy(sr, rr, (size_t)n * 8);
            qsort(sb, (size_t)n, 8, cmp_f64);
            qsort(sr, (size_t)n, 8, cmp_f64);
            const double qs[5] = {0.0, 0.25, 0.5, 0.75, 1.0};
            for (int k = 0; k < 5; k++) { o[1 + k] = quantile_sorted(sb, n, qs[k]); o[6 + k] = quantile_sorted(sr, n, qs[k]); }
            /* Pearson: two-pass means, sequential sums in (gpu, iteration) order */
            double mb = 0.0, mr = 0.0;
            for (int64_t i = 0; i < n; i++) { mb += b[i]; mr += rr[i]; }
            mb /= (double)n;
            mr /= (double)n;
            double sxx = 0.0, syy = 0.0, sxy = 0.0;
            for (int64_t i = 0; i < n; i++) {
                double dx = rr[i] - mr, dy = b[i] - mb;
                sxx += dx * dx; syy += dy * dy; sxy += dx * dy;
            }
            o[11] = (sxx > 0.0 && syy > 0.0) ? sxy / sqrt(sxx * syy) : NAN;
            o[13] = mb;
        }
        free(b); free(rr); free(sb); free(sr);
    }

    /* ---------------- O15 per-GPU overlap CDF of every op label (Fig. 7) -----
       For label L and traced gpu g: the sampled points of (g, L) (same selection as O13/O14) sorted by duration
       (ties: iteration rank), duration normalized to the gpu's minimum (Fig. 7 caption), overlap ratio, and the
       empirical CDF ordinate (k + 1) / n_g (R11).  Rows in (label, gpu, k) order: label, gpu, dur_norm, ratio,
       cdf. */
    {
        int64_t ncdf = 0;
        for (int64_t x = 0; x < n_pt; x++) {
            const row_t *pr = &pt[x];
            if (pr->r_it - 1 < in->warmup || pr->busy <= 0 || !((in->bd_gpu_mask >> pr->gpu) & 1ull)) continue;
            ncdf++;
        }
        double *cd = new_f64(r, "cdf.rows", ncdf * 5);
        int64_t w = 0;
        int64_t *ord = (int64_t *)xcalloc(n_pt > 0 ? n_pt : 1, 8);
        for (int L = 0; L < in->n_labels; L++) {
            for (int g = 0; g < G; g++) {
                int64_t n = 0;
                for (int64_t x = 0; x < n_pt; x++) {
                    const row_t *pr = &pt[x];
                    if (pr->label != L || pr->gpu != g || pr->r_it - 1 < in->warmup || pr->busy <= 0) continue;
                    if (!((in->bd_gpu_mask >> pr->gpu) & 1ull)) continue;
                    ord[n++] = x;
                }
                /* insertion sort by (duration, iteration rank): points of one gpu and label are few */
                for (int64_t a = 1; a < n; a++) {
                    int64_t v = ord[a], b = a - 1;
                    while (b >= 0 && (pt[ord[b]].busy > pt[v].busy ||
                                      (pt[ord[b]].busy == pt[v].busy && pt[ord[b]].r_it > pt[v].r_it))) {
                        ord[b + 1] = ord[b];
                        b--;
                    }
                    ord[b + 1] = v;
                }
                for (int64_t k = 0; k < n; k++) {
                    const row_t *pr = &pt[ord[k]];
                    double *o = &cd[w * 5];
                    o[0] = (double)L;
                    o[1] = (double)g;
                    o[2] = (double)pr->busy / (double)pt[ord[0]].busy;
                    o[3] = (double)pr->ovl / (double)pr->busy;
                    o[4] = (double)(k + 1) / (double)n;
                    w++;
                }
            }
        }
        free(ord);
    }

    /* ---------------- O16 end-to-end phase x op-type breakdown (Fig. 4) -----
       Per traced gpu and sampled iteration (rank >= warmup, the iteration row exists): for each phase label
       P in [0, 8) (the label of the phase span; instances of other labels are not counted) the summed
       duration of its instances by op type T (0 vector / other incl. the unlabeled pseudo-ops, 1 gemm, 2 fa)
       and the summed launch overhead (prep + call).  Row: 0 n_points, then for P = 0..7: median over the
       points of [vec, gemm, fa, launch] (ns; cells without instances count 0) -- "median values across
       iterations and GPUs" (Fig. 4 caption; R12). */
    {
        const int NP = 8;
        int64_t npt = 0;
        for (int64_t x = 0; x < n_itr; x++)
            if (itr[x].r_it - 1 >= in->warmup && ((in->bd_gpu_mask >> itr[x].gpu) & 1ull)) npt++;
        double *e2 = new_f64(r, "e2e.rows", 1 + NP * 4);
        e2[0] = (double)npt;
        int64_t *cell = (int64_t *)xcalloc((npt > 0 ? npt : 1) * NP * 4, 8);
        int64_t w = 0;
        for (int64_t x = 0; x < n_itr; x++) {
            const row_t *it = &itr[x];
            if (it->r_it - 1 < in->warmup || !((in->bd_gpu_mask >> it->gpu) & 1ull)) continue;
            int64_t *c = &cell[w * NP * 4];
            for (int64_t q = 0; q < n_inst; q++) {
                const row_t *ins = &inst[q];
                if (ins->gpu != it->gpu || ins->r_it != it->r_it || ins->ph < 0) continue;
                const int P = in->span_label[ins->ph];
                if (P < 0 || P >= NP) continue;
                const int T = (ins->label >= 0 && in->op_type[ins->label] == 1) ? 1
                            : (ins->label >= 0 && in->op_type[ins->label] == 2) ? 2 : 0;
                c[P * 4 + T] += ins->busy;
                c[P * 4 + 3] += ins->prep + ins->call;
            }
            w++;
        }
        int64_t *col = (int64_t *)xcalloc(npt > 0 ? npt : 1, 8);
        for (int k = 0; k < NP * 4; k++) {
            for (int64_t q = 0; q < npt; q++) col[q] = cell[q * NP * 4 + k];
            e2[1 + k] = npt > 0 ? median_i64(col, npt) : NAN;
        }
        free(col); free(cell);
    }

    /* per-event span indices are reported as caller indices (already) */
    for (int g = 0; g < G; g++) free(U[g]);
    free(U); free(nU); free(gbeg); free(gend); free(ord); free(rank1);
    row_t *tabs[6] = { inst, ly, ph, itr, gp, pt };
    int64_t ns6[6] = { n_inst, n_ly, n_ph, n_itr, n_gpu, n_pt };
    for (int t = 0; t < 6; t++) { for (int64_t q = 0; q < ns6[t]; q++) free(tabs[t][q].cnt); free(tabs[t]); }
    return r;
#undef VIOL
}

/* ======================================================================================================
 * O17 CPU utilization (Sec. "CPU Utilization").
 *   Logical cores:  C_active = sum_i [Util_i > 0],  C_min = sum_i Util_i / 100,
 *   evaluated per sampling timestamp over the logical cores sampled there (reading R13).
 *   Physical cores (Fig. 9): a physical core is occupied when one or more of its
 *   logical cores is active; physical occupancy = |{phys(i) : Util_i > 0 at any timestamp}| / #physical
 *   (SPEC.md:295).  SMT co-activity (Fig. 9's "yellow" points): among (timestamp, physical core) pairs with
 *   an active logical core, the fraction with two or more.
 *   Samples must be sorted by (ts, logical core) with 0 <= util <= 100 and core < N; anything else sets
 *   *bad (nothing else is computed).  Medians follow D21 (even count: mean of the two central values).
 *   Plain loops in sample order; C_min sums in logical-core order within a timestamp.
 * ====================================================================================================== */
int64_t or_cpu_util(int64_t n, const int64_t *ts, const int32_t *core, const double *util, int32_t n_logical,
                    const int32_t *topology, int64_t *c_active, double *c_min, double *summary, int32_t *bad) {
    /* summary: [0] n_ts [1] median C_active [2] median C_min [3] max C_active [4] max C_min
     *          [5] physical occupancy [6] SMT co-activity fraction [7] #physical cores */
    *bad = 0;
    int32_t n_phys = 0;
    for (int32_t i = 0; i < n_logical; i++) {
        if (topology[i] < 0) { *bad = 1; return 0; }
        if (topology[i] + 1 > n_phys) n_phys = topology[i] + 1;
    }
    for (int64_t k = 0; k < n; k++) {
        if (core[k] < 0 || core[k] >= n_logical || !(util[k] >= 0.0 && util[k] <= 100.0)) { *bad = 1; return 0; }
        if (k > 0 && (ts[k] < ts[k - 1] || (ts[k] == ts[k - 1] && core[k] <= core[k - 1]))) { *bad = 1; return 0; }
    }
    char *ever = (char *)xcalloc(n_phys > 0 ? n_phys : 1, 1);
    int32_t *cnt = (int32_t *)xcalloc(n_phys > 0 ? n_phys : 1, sizeof(int32_t));
    int64_t nts = 0, pairs1 = 0, pairs2 = 0;
    for (int64_t a = 0; a < n;) {
        int64_t b = a;
        while (b < n && ts[b] == ts[a]) b++;
        int64_t act = 0;
        double cm = 0.0;
        for (int32_t p = 0; p < n_phys; p++) cnt[p] = 0;
        for (int64_t k = a; k < b; k++) {
            if (util[k] > 0.0) {
                act++;
                ever[topology[core[k]]] = 1;
                cnt[topology[core[k]]]++;
            }
            cm += util[k] / 100.0;
        }
        for (int32_t p = 0; p < n_phys; p++) {
            if (cnt[p] >= 1) pairs1++;
            if (cnt[p] >= 2) pairs2++;
        }
        c_active[nts] = act;
        c_min[nts] = cm;
        nts++;
        a = b;
    }
    int64_t occ = 0;
    for (int32_t p = 0; p < n_phys; p++) occ += ever[p];
    int64_t amax = 0;
    double mmax = 0.0;
    for (int64_t q = 0; q < nts; q++) {
        if (c_active[q] > amax) amax = c_active[q];
        if (c_min[q] > mmax) mmax = c_min[q];
    }
    summary[0] = (double)nts;
    summary[1] = nts > 0 ? median_i64(c_active, nts) : NAN;
    summary[2] = nts > 0 ? median_f64(c_min, nts) : NAN;
    summary[3] = (double)amax;
    summary[4] = nts > 0 ? mmax : NAN;
    summary[5] = n_phys > 0 ? (double)occ / (double)n_phys : NAN;
    summary[6] = pairs1 > 0 ? (double)pairs2 / (double)pairs1 : NAN;
    summary[7] = (double)n_phys;
    free(ever);
    free(cnt);
    return nts;
}
