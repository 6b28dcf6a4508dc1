"""Element-by-element comparison of the CUDA path (through the C ABI) with the oracle."""
import numpy as np

INT_EV = ("ev.span_idx", "ev.ovl", "ev.prep", "ev.call", "ev.phi", "ev.psi")
ROW_INT = ("gpu", "it", "ph", "ly", "op", "label", "n_events", "n", "busy", "first_ks", "first_idx", "first_pred",
           "last_ke", "prep", "call", "ovl", "phi", "psi", "copy_ns", "ag_ns", "rs_ns")
ITER_EXTRA = ("wall", "comm_union", "aligned_first", "aligned_last", "step", "rank")
GLOB_INT = ("glob.step", "glob.complete", "glob.sampled", "glob.T", "glob.aligned_first", "glob.aligned_last")
FP_RTOL = 1e-9   # north_star: fp64 counter-derived rates and breakdown fractions within 1e-9 relative


def run_both(bundle, params=None, max_iters=None, full=True):
    import oracle
    import paper_2512_08242_b200 as ch
    p = oracle.default_params(bundle) if params is None else params
    mi = max_iters or max(8, bundle.cfg.n_iters + 2)
    ref = oracle.run(bundle, p, max_iters=mi)
    kcoll = int(max(16, 4 * _max_coll(bundle)))
    pipe = ch.Pipeline(bundle.cfg.n_gpus, len(bundle.labels), mi, kcoll, device=0)
    pipe.upload(bundle, bundle.n_counters)
    res = pipe.run(p, full=full, check=False)
    got = pipe.to_numpy(res, n_ratios=len(p["ratio_num"])) if res.get("tables") is not None else None
    return ref, got, res, pipe


def _max_coll(b):
    k = b.meta & 0xFF
    g = b.meta >> 24
    best = 0
    for gg in np.unique(g):
        m = g == gg
        best = max(best, int(((k == 1) & m).sum()), int(((k == 2) & m).sum()))
    return best


def assert_parity(ref, got, per_event=True, tables=True, glob=True, bd=True):
    errs = []
    if per_event:
        for k in INT_EV:
            if not np.array_equal(ref[k], got[k]):
                bad = np.nonzero(ref[k] != got[k])[0]
                errs.append(f"{k}: {len(bad)} mismatches, first at {bad[:5]} ref={ref[k][bad[:5]]} got={got[k][bad[:5]]}")
        if "ev.counters" in got and got["ev.counters"].size:
            if not np.array_equal(ref["ev.counters"], got["ev.counters"]):
                errs.append("ev.counters differ")
    if tables:
        for t in ("inst", "layer", "phase", "iter", "gpu", "point"):
            n_ref, n_got = len(ref[f"{t}.gpu"]), len(got[f"{t}.gpu"])
            if n_ref != n_got:
                errs.append(f"{t}: {n_ref} rows (oracle) vs {n_got} (gpu)")
                continue
            for f in ROW_INT:
                if f == "label" and t in ("layer", "phase", "iter", "gpu"):
                    continue
                if f in ("ph", "ly", "op") and t == "point":
                    continue
                a, b = ref[f"{t}.{f}"], got[f"{t}.{f}"]
                if not np.array_equal(a, b):
                    bad = np.nonzero(a != b)[0]
                    errs.append(f"{t}.{f}: {len(bad)} mismatches, first {bad[:3]} ref={a[bad[:3]]} got={b[bad[:3]]}")
            a, b = ref[f"{t}.counters"], got[f"{t}.counters"]
            if a.size and not np.allclose(a, b, rtol=FP_RTOL, atol=0):
                errs.append(f"{t}.counters differ beyond rtol {FP_RTOL}")
            if f"{t}.rates" in ref and ref[f"{t}.rates"].size:
                if not np.allclose(ref[f"{t}.rates"], got[f"{t}.rates"], rtol=FP_RTOL, atol=0, equal_nan=True):
                    errs.append(f"{t}.rates differ")
        for f in ITER_EXTRA:
            if not np.array_equal(ref[f"iter.{f}"], got[f"iter.{f}"]):
                errs.append(f"iter.{f} differs")
        if not np.array_equal(ref["point.rank"], got["point.rank"]):
            errs.append("point.rank differs")
    if glob:
        for k in GLOB_INT:
            if not np.array_equal(ref[k], got[k]):
                errs.append(f"{k} differs: ref {ref[k][:5]} got {got[k][:5]}")
        if not np.array_equal(ref["gpu.delta"], got["gpu.delta"]):
            errs.append(f"gpu.delta differs: {ref['gpu.delta']} vs {got['gpu.delta']}")
        if not np.allclose(ref["glob.throughput"], got["glob.throughput"], rtol=1e-12, equal_nan=True):
            errs.append("glob.throughput differs")
        if not np.allclose(ref["glob.throughput_median"], got["glob.throughput_median"], rtol=1e-12, equal_nan=True):
            errs.append("glob.throughput_median differs")
        for cls, key in (("skew.ag", "skew.max_ag"), ("skew.rs", "skew.max_rs")):
            sk = ref.get(cls, np.zeros(0))
            if sk.size and int(sk.max()) != int(got[key][0]):
                errs.append(f"{key} differs: ref {int(sk.max())} got {int(got[key][0])}")
    if bd:
        a, b = ref["bd.rows"], got["bd.rows"]
        if a.shape != b.shape or not np.allclose(a, b, rtol=FP_RTOL, atol=0, equal_nan=True):
            errs.append(f"bd.rows differ:\nref {a.reshape(-1, 16)[:3]}\ngot {b.reshape(-1, 16)[:3]}")
        # report statistics (O14): quantiles and Pearson per label, fp64 within the same budget
        a, b = ref["report.rows"], got.get("report.rows", np.zeros(0))
        if a.shape != b.shape or not np.allclose(a, b, rtol=FP_RTOL, atol=1e-12, equal_nan=True):
            bad = np.nonzero(~np.isclose(a, b, rtol=FP_RTOL, atol=1e-12, equal_nan=True))[0] if a.shape == b.shape else []
            errs.append(f"report.rows differ at {bad[:8]}: ref {a[bad[:4]] if len(bad) else a.shape} "
                        f"got {b[bad[:4]] if len(bad) else b.shape}")
        a, b = ref["e2e.rows"], got.get("e2e.rows", np.zeros(0))
        if a.shape != b.shape or not np.allclose(a, b, rtol=0, atol=0, equal_nan=True):
            errs.append(f"e2e.rows differ: ref {a[:9]} got {b[:9]}")
        if "cdf.rows" in got:
            a, b = ref["cdf.rows"], got["cdf.rows"]
            if a.shape != b.shape or not np.allclose(a, b, rtol=FP_RTOL, atol=1e-12, equal_nan=True):
                errs.append(f"cdf.rows differ: shapes {a.shape} {b.shape}")
    assert not errs, "\n".join(errs)
