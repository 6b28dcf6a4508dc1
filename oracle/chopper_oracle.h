/*
 * chopper_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, single-threaded CPU oracle for the Chopper analysis hot path
 * (arXiv 2512.08242, "Chopper: A Multi-Level GPU Characterization Tool").
 * It is the parity reference for the CUDA library in
 * paper_2512_08242_b200/csrc and shares NO code, header, table or helper with
 * it.  Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load it.  The product path never does.
 *
 * Every step follows DESIGN.md section "Oracle" (O1..O13), which restates the
 * paper passages it implements:
 *   PAPER.md:241-244  trace alignment          (O3)
 *   PAPER.md:100-102  granularity ladder       (O5, O10, O11)
 *   PAPER.md:445-521  overlap ratio            (O6, O7)
 *   PAPER.md:576-594  Eqs. 1-3 launch overhead (O8)
 *   PAPER.md:700-725  frequency / power        (O9)
 *   PAPER.md:337-345  throughput (fig:end_to_end caption) (O12)
 *   PAPER.md:727-791  Eqs. 4-8 breakdown       (O13)
 *
 * Results are exposed as named arrays: or_run() returns a handle, or_get()
 * looks an array up by name, or_free() releases everything.
 */
#ifndef CHOPPER_ORACLE_H
#define CHOPPER_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    /* kernel events, grouped by gpu ascending, dispatch-ordered within a gpu */
    int64_t n_events;
    const int64_t *t_l, *t_ks, *t_ke;     /* dispatch, device start, device end (ns) */
    const uint32_t *meta;                 /* (gpu<<24) | (stream<<8) | kind */
    const int32_t *name_id;
    /* annotation spans, any order, half-open [start, end) on the host timeline */
    int64_t n_spans;
    const uint32_t *span_gl;              /* (gpu<<8) | level ; level 0 it,1 ph,2 ly,3 op */
    const int64_t *span_start, *span_end;
    const int32_t *span_label;
    /* 1 ms frequency / power samples, sorted by (gpu, ts) */
    int64_t n_samples;
    const int32_t *smp_gpu;
    const int64_t *smp_ts;
    const int32_t *smp_freq_mhz, *smp_power_mw;
    /* serialized counter passes */
    int32_t n_passes;
    const int32_t *pass_gpu;
    const int64_t *pass_n;
    const int32_t *pass_k;
    const int32_t *const *pass_name_id;   /* [n_passes] -> [pass_n] */
    const int32_t *const *pass_slot;      /* [n_passes] -> [pass_k] */
    const double *const *pass_values;     /* [n_passes] -> [pass_k][pass_n] */
    int32_t n_counters;
    /* run configuration */
    int32_t n_traced_gpus, n_labels, max_iters;
    /* breakdown parameters */
    double tpt_peak, freq_peak_hz;
    int64_t b, s, R;
    int32_t warmup;
    int32_t slot_cycles, slot_flops, slot_unum, slot_uden;   /* -1 = absent */
    const double *f_gemm;                 /* [n_labels] */
    const int32_t *op_type;               /* [n_labels] 0 other, 1 gemm, 2 fa */
    int32_t n_ratios;
    const int32_t *ratio_num, *ratio_den; /* den -1 = busy seconds */
    const double *ratio_scale;
    uint64_t bd_gpu_mask;                 /* gpus whose points feed the breakdown rows */
} or_input;

typedef struct or_result or_result;

or_result *or_run(const or_input *in);
/* dtype codes: 0 int32, 1 int64, 2 float64, 3 uint8 ; returns 0 if found */
int32_t or_get(const or_result *r, const char *name, void **ptr, int64_t *n, int32_t *dtype);
int32_t or_count(const or_result *r);
const char *or_name(const or_result *r, int32_t i);
void or_free(or_result *r);

#ifdef __cplusplus
}
#endif
#endif
