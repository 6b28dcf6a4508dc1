"""GPU parity: the CUDA path through the C ABI vs the oracle, element by element.

Integer outputs (span indices, overlap, launch components, DVFS integrals,
every integer table column, clock offsets, iteration joins) must be bit-exact;
fp64 counter sums, rates and breakdown factors within 1e-9 relative
(BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle
import tracegen
from parity import assert_parity, run_both
from tinytrace import AG, COMPUTE, COPY, MEMOP, OTHER, RS, TinyTrace, params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_08242_b200 as ch
    ch.build()
    ch.load_library()


def _check_status(ref, got):
    assert int(ref["status"][0]) == int(got["status_mask"][0]), (ref["status"], got["status_mask"])


def test_config1_toy_full():
    b = tracegen.generate(tracegen.config(1))
    ref, got, res, pipe = run_both(b)
    _check_status(ref, got)
    assert_parity(ref, got)
    np.testing.assert_array_equal(ref["val.count"], got["val.count"])


def test_small_counters_samples_full():
    cfg = tracegen.config(3)
    cfg.n_iters, cfg.n_layers, cfg.n_gpus, cfg.opt_kernels, cfg.warmup = 3, 4, 3, 600, 1
    b = tracegen.generate(cfg)
    ref, got, res, pipe = run_both(b)
    _check_status(ref, got)
    assert_parity(ref, got)


def test_config2_llama_full():
    """BASELINE configs[1]: Llama 3 8B FSDP-shaped, 8 GPUs x 10 iterations (~0.9M events)."""
    b = tracegen.generate(tracegen.config(2))
    ref, got, res, pipe = run_both(b)
    _check_status(ref, got)
    assert_parity(ref, got)


@pytest.mark.slow
def test_config3_counters_dvfs_full():
    """BASELINE configs[2]: 20 counters per kernel + 1 ms frequency / power samples."""
    b = tracegen.generate(tracegen.config(3))
    ref, got, res, pipe = run_both(b)
    _check_status(ref, got)
    assert_parity(ref, got)


@pytest.mark.slow
def test_config4_long_run_full():
    """BASELINE configs[3] at full size (~17.6M events, 8 counters, samples): the bench workload, same launch path."""
    b = tracegen.generate(tracegen.config(4))
    ref, got, res, pipe = run_both(b, max_iters=256)
    _check_status(ref, got)
    assert_parity(ref, got)


def test_tables_only_mode_matches_full():
    """per-event outputs NULL (the bench path) gives the same tables as full mode."""
    import paper_2512_08242_b200 as ch
    b = tracegen.generate(tracegen.config(1))
    p = oracle.default_params(b)
    pipe = ch.Pipeline(b.cfg.n_gpus, len(b.labels), 16, 4096)
    pipe.upload(b, b.n_counters)
    full = pipe.to_numpy(pipe.run(p, full=True), len(p["ratio_num"]))
    lean = pipe.to_numpy(pipe.run(p, full=False), len(p["ratio_num"]))
    for k in lean:
        if k.startswith("ev."):
            continue
        np.testing.assert_array_equal(np.nan_to_num(full[k]), np.nan_to_num(lean[k]), err_msg=k)


@pytest.mark.parametrize("how", ["shuffled", "reversed_level"])
def test_span_input_order(how):
    """spans in any input order (fully shuffled, or each (gpu, level) list in start order but the lists
    interleaved differently) give the oracle's span table and outputs."""
    b = tracegen.generate(tracegen.config(1))
    rng = np.random.default_rng(7)
    if how == "shuffled":
        perm = rng.permutation(len(b.span_gl))
    else:                                   # lists interleaved in a new order, each still in start order
        lv = (b.span_gl & 0xFF).astype(np.int64)
        perm = np.lexsort((np.arange(len(lv)), -lv))
    b2 = tracegen.dataclasses.replace(b, span_gl=b.span_gl[perm], span_start=b.span_start[perm],
                                      span_end=b.span_end[perm], span_label=b.span_label[perm])
    ref, got, res, pipe = run_both(b2)
    _check_status(ref, got)
    assert_parity(ref, got)


def test_double_buffered_inputs():
    """stage_inputs / use_inputs (the streaming e2e path): a run on the second input set, filled from pinned
    host memory on a copy stream while the first set is clobbered, gives the same tables."""
    import torch
    import paper_2512_08242_b200 as ch
    b = tracegen.generate(tracegen.config(1))
    p = oracle.default_params(b)
    pipe = ch.Pipeline(b.cfg.n_gpus, len(b.labels), 16, 4096)
    pipe.upload(b, b.n_counters)
    want = pipe.to_numpy(pipe.run(p, full=False), len(p["ratio_num"]))
    a, s2 = pipe.input_set(), pipe.new_input_set()
    pinned = {k: v.cpu().pin_memory() for k, v in a["d"].items()}
    pp = [(nm.cpu().pin_memory(), vals.cpu().pin_memory()) for (_, nm, _, vals) in a["passes"]]
    cs = torch.cuda.Stream()
    ready = pipe.stage_inputs(s2, pinned, pp, None, cs)
    for v in a["d"].values():
        v.zero_()
    pipe.use_inputs(s2, ready)
    got = pipe.to_numpy(pipe.run(p, full=False), len(p["ratio_num"]))
    for k in want:
        np.testing.assert_array_equal(np.nan_to_num(want[k]), np.nan_to_num(got[k]), err_msg=k)


# ---------------------------------------------------------------------------
# edge cases
# ---------------------------------------------------------------------------
def _tiny(tt, **kw):
    b = tt.bundle()
    p = params(b, **kw)
    return run_both(b, p)


def test_no_spans_all_unannotated():
    tt = TinyTrace().ev(0, 0, 10, 20).ev(0, 1, 25, 40).ev(0, 2, 5, 50, kind=AG, stream=1)
    ref, got, _, _ = _tiny(tt)
    assert_parity(ref, got)
    assert len(got["inst.gpu"]) == 0


def test_single_event():
    tt = TinyTrace().span(0, 0, 0, 100, 3).span(0, 3, 0, 100, 1).ev(0, 5, 10, 20)
    ref, got, _, _ = _tiny(tt)
    assert_parity(ref, got)


def test_crossing_spans_ambiguous_sweep_path():
    """crossing op spans: exact device sweep path; dispatch in the crossing region -> -2 + E_AMBIGUOUS_SPANS."""
    tt = TinyTrace().span(0, 0, 0, 1000, 7).span(0, 3, 100, 200, 0).span(0, 3, 150, 250, 1)
    for t in (50, 120, 160, 220, 300):
        tt.ev(0, t, t + 1, t + 2)
    ref, got, res, pipe = _tiny(tt)
    _check_status(ref, got)
    assert_parity(ref, got)
    assert res["report"].non_laminar_lists == 1


def test_crossing_without_dispatch_is_harmless():
    tt = TinyTrace().span(0, 0, 0, 1000, 7).span(0, 3, 100, 200, 0).span(0, 3, 150, 250, 1)
    for t in (50, 120, 220, 300):
        tt.ev(0, t, t + 1, t + 2)
    ref, got, _, _ = _tiny(tt)
    _check_status(ref, got)
    assert_parity(ref, got)


def test_deep_nesting_and_identical_spans():
    tt = TinyTrace().span(0, 0, 0, 10_000, 1)
    # depth-8 nest of op spans, identical duplicates, zero-length spans, siblings
    for d in range(8):
        tt.span(0, 3, 100 * d, 9000 - 100 * d, d % 4)
    tt.span(0, 3, 300, 8700, 2)                         # identical to the depth-3 span
    tt.span(0, 3, 5000, 5000, 1)                        # zero length: never contains anything
    for s in range(1000, 8000, 700):
        tt.span(0, 3, s, s + 300, 3)
    for t in range(0, 10_000, 97):
        tt.ev(0, t, t + 10, t + 50)
    ref, got, res, _ = _tiny(tt)
    _check_status(ref, got)
    assert_parity(ref, got)
    assert res["report"].non_laminar_lists == 0


def test_multi_stream_compute_and_comm_order():
    """two compute streams (compute union built explicitly) and comm events whose start order
    differs from dispatch order (full radix sort path)."""
    tt = TinyTrace(n_gpus=2).span(0, 0, 0, 10 ** 6, 1).span(1, 0, 0, 10 ** 6, 1)
    for g in range(2):
        t = 0
        for k in range(60):
            tt.ev(g, 10 * k, 100 + 37 * k, 100 + 37 * k + 30, stream=k % 2)
        tt.ev(g, 5, 3000, 3500, kind=AG, stream=2)
        tt.ev(g, 6, 1000, 1200, kind=RS, stream=3)          # dispatched later, starts earlier
        tt.ev(g, 7, 900, 950, kind=AG, stream=2)
        del t
    b = tt.bundle()
    ref, got, res, _ = run_both(b, params(b))
    _check_status(ref, got)
    assert_parity(ref, got)
    assert res["report"].full_sort_used == 1


def test_same_stream_overlap_is_data():
    tt = TinyTrace().span(0, 0, 0, 1000, 1).ev(0, 0, 10, 50).ev(0, 1, 40, 80).ev(0, 2, 30, 90, kind=AG, stream=1)
    ref, got, _, _ = _tiny(tt)
    _check_status(ref, got)
    np.testing.assert_array_equal(ref["val.count"], got["val.count"])
    np.testing.assert_array_equal(ref["val.first"], got["val.first"])
    assert_parity(ref, got)


@pytest.mark.parametrize("case", ["start_after_end", "not_grouped", "dispatch_dec", "bad_meta", "span_bad"])
def test_fatal_validation(case):
    import paper_2512_08242_b200 as ch
    tt = TinyTrace(n_gpus=2)
    keep = False
    if case == "start_after_end":
        tt.ev(0, 0, 10, 5).ev(0, 1, 20, 30)
    elif case == "not_grouped":
        tt.ev(1, 0, 10, 15).ev(0, 1, 20, 30); keep = True
    elif case == "dispatch_dec":
        tt.ev(0, 5, 10, 15).ev(0, 1, 20, 30); keep = True
    elif case == "bad_meta":
        tt.ev(0, 0, 10, 15).ev(0, 1, 20, 30, kind=9)
    elif case == "span_bad":
        tt.ev(0, 0, 10, 15).span(0, 0, 10, 5)
    b = tt.bundle(keep_order=keep)
    p = params(b)
    ref = oracle.run(b, p)
    pipe = ch.Pipeline(2, len(b.labels), 8, 16)
    pipe.upload(b, 0)
    res = pipe.run(p, check=False)
    assert res["load_status"] == 1
    rep = res["report"]
    np.testing.assert_array_equal(ref["val.count"], np.array(rep.val_count[:]))
    np.testing.assert_array_equal(ref["val.first"], np.array(rep.val_first[:]))


def test_counter_alignment_mismatch_and_conflict():
    tt = TinyTrace(n_counters=2).span(0, 0, 0, 1000, 1).span(0, 3, 0, 1000, 0)
    names = [1, 2, 1]
    for k, nm in enumerate(names):
        tt.ev(0, 10 * k, 10 * k + 1, 10 * k + 5, name=nm)
    tt.ev(0, 100, 101, 102, kind=MEMOP, stream=3, name=9)
    tt.counter_pass(0, names, [0], [[1, 2, 3]]).counter_pass(0, [1, 1], [1], [[5, 6]])
    tt.counter_pass(0, names, [0], [[1, 2.5, 3]])
    b = tt.bundle()
    p = params(b, slot_unum=-1, slot_uden=-1)
    ref, got, res, pipe = run_both(b, p)
    _check_status(ref, got)
    assert_parity(ref, got)
    import paper_2512_08242_b200 as ch
    lib = ch.load_library()
    for q in range(3):
        assert lib.chopper_pass_mismatch(pipe.ctx, q) == ref["pass.mismatch"][q]
        assert lib.chopper_pass_conflict(pipe.ctx, q) == ref["pass.conflict"][q]


@pytest.mark.parametrize("where", ["comm", "compute", "unused_column"])
def test_nonfinite_counter_pass_skipped(where):
    """R8: a pass holding a non-finite value is skipped (CV_COUNTER_NONFINITE, E_VALIDATION) and the next
    valid pass with the slot provides it.  The GPU checks the columns feeding a slot inside the counter
    pass and redoes the slot assignment; a column feeding no slot is checked by k_pass_finite."""
    tt = TinyTrace(n_counters=3).span(0, 0, 0, 10_000, 1).span(0, 3, 0, 10_000, 0)
    names, kinds = [], []
    for k in range(40):
        kind = AG if k % 7 == 3 else COMPUTE
        tt.ev(0, 100 * k, 100 * k + 1, 100 * k + 50, kind=kind, stream=1 if kind == AG else 0, name=k % 3)
        names.append(k % 3)
        kinds.append(kind)
    rng = np.random.default_rng(7)
    a = rng.integers(1, 100, size=(2, len(names))).astype(float)
    b2 = rng.integers(1, 100, size=(2, len(names))).astype(float)
    if where == "comm":
        a[0, kinds.index(AG)] = np.nan          # pass 0 provides slots 0, 1
    elif where == "compute":
        a[1, 5] = np.inf
    b2[0] = a[0] if where != "comm" else b2[0]  # pass 1: slot 0 again (agrees unless pass 0 is skipped) + slot 2
    tt.counter_pass(0, names, [0, 1], a)
    tt.counter_pass(0, names, [0, 2], b2)
    if where == "unused_column":
        bad = rng.integers(1, 100, size=(1, len(names))).astype(float)
        bad[0, 3] = np.nan
        tt.counter_pass(0, names, [1], bad)      # slot 1 already provided: column feeds no slot
    b = tt.bundle()
    p = params(b, slot_unum=-1, slot_uden=-1)
    ref, got, res, pipe = run_both(b, p)
    _check_status(ref, got)
    np.testing.assert_array_equal(ref["val.count"], got["val.count"])
    np.testing.assert_array_equal(ref["val.first"], got["val.first"])
    assert_parity(ref, got)


@pytest.mark.parametrize("seed", range(8))
def test_random_traces(seed):
    """random multi-gpu traces with nested / crossing spans, skewed dispatch, comm on two streams, copies,
    memops, samples and counters."""
    rng = np.random.default_rng(1000 + seed)
    G = int(rng.integers(1, 4))
    C = 4
    tt = TinyTrace(n_gpus=G, n_counters=C, labels=["l%d" % i for i in range(6)])
    for g in range(G):
        T = 200_000
        for it in range(3):
            tt.span(g, 0, it * T, (it + 1) * T, 100 + it)
            tt.span(g, 1, it * T, it * T + T // 2, 0).span(g, 1, it * T + T // 2, (it + 1) * T, 1)
            for ly in range(3):
                tt.span(g, 2, it * T + ly * 50_000, it * T + ly * 50_000 + 40_000, ly)
        for _ in range(int(rng.integers(20, 60))):
            s = int(rng.integers(0, 3 * T))
            e = s + int(rng.integers(0, 30_000))
            tt.span(g, 3, s, e, int(rng.integers(0, 6)))
        t_dev = 0
        t_host = 0
        names = []
        kinds = []
        for k in range(int(rng.integers(200, 600))):
            kind = int(rng.choice([COMPUTE] * 8 + [AG, RS, COPY, MEMOP, OTHER]))
            d = int(rng.integers(0, 3000))
            if kind == COMPUTE:
                t_dev += int(rng.integers(0, 800))
                ks = t_dev
                t_dev += d
                st = 0
            else:
                ks = int(rng.integers(0, 3 * T))
                st = {AG: 1, RS: 2, COPY: 0, MEMOP: 3, OTHER: 4}[kind]
                if kind == COPY:
                    t_dev += int(rng.integers(0, 800)); ks = t_dev; t_dev += d
            t_host += int(rng.integers(1, 1500))
            tl = t_host if rng.random() > 0.05 else t_host
            nm = int(rng.integers(0, 5))
            tt.ev(g, tl, ks, ks + d, kind=kind, stream=st, name=nm)
            if kind != MEMOP:
                names.append(nm)
            kinds.append(kind)
        vals = rng.integers(0, 1000, size=(2, len(names))).astype(float)
        tt.counter_pass(g, names, [0, 1], vals)
        tt.counter_pass(g, names, [2, 3], np.vstack([rng.integers(1, 100, len(names)), rng.random(len(names)) + 1]))
        ts = 0
        while ts < 3 * T:
            tt.sample(g, ts, int(rng.integers(1300, 2100)), int(rng.integers(500, 1000)))
            ts += int(rng.integers(5_000, 20_000))
    b = tt.bundle()
    p = params(b, f_gemm=np.full(6, 1e9), op_type=np.array([1, 2, 0, 1, 1, 2], np.int32), warmup=1)
    ref, got, res, _ = run_both(b, p)
    _check_status(ref, got)
    assert_parity(ref, got)


def test_dense_spans_and_samples_overflow_windows():
    """far more span boundaries and timeline entries per 2048-event tile than the event pass stages in shared
    memory (every query past the staged window reads global memory), tiles straddling two gpus, a comm
    interval and a sample every few kernels."""
    rng = np.random.default_rng(77)
    G = 2
    tt = TinyTrace(n_gpus=G, n_counters=2, labels=["l%d" % i for i in range(4)])
    for g in range(G):
        n = 4500 + 700 * g
        t = 1000
        tt.span(g, 0, 0, 10 ** 9, 7)
        tt.span(g, 1, 0, 10 ** 9, 0)
        names = []
        for k in range(n):
            d = int(rng.integers(50, 400))
            tl = t - int(rng.integers(0, 30))
            ks = t
            tt.ev(g, tl, ks, ks + d, name=k % 3)
            names.append(k % 3)
            # op span around the dispatch plus three empty spans (no dispatch inside) after the kernel
            tt.span(g, 3, tl - 1, tl + 1, k % 4)
            for e in range(3):
                tt.span(g, 3, ks + 2 + 3 * e, ks + 4 + 3 * e, (k + e) % 4)
            if k % 40 == 0:
                tt.span(g, 2, tl, tl + 40 * 300, k % 4)
            if k % 5 == 0:
                tt.ev(g, tl, ks + d // 3, ks + d + 500, kind=AG if k % 10 else RS, stream=1 + (k % 10 == 0), name=3)
                names.append(3)
            tt.sample(g, ks + d // 2, int(rng.integers(1300, 2100)), int(rng.integers(500, 900)))
            t = ks + d + int(rng.integers(5, 60))
        tt.counter_pass(g, names, [0, 1], rng.integers(0, 1000, size=(2, len(names))).astype(float))
    b = tt.bundle()
    p = params(b, f_gemm=np.full(4, 1e9), op_type=np.array([1, 2, 0, 1], np.int32))
    ref, got, res, _ = run_both(b, p)
    _check_status(ref, got)
    assert_parity(ref, got)


def _cpu_both(ts, core, util, topo):
    import torch
    import paper_2512_08242_b200 as ch
    ref = oracle.cpu_util(ts, core, util, topo)
    b = TinyTrace().ev(0, 0, 10, 20).span(0, 0, 0, 100).bundle()
    pipe = ch.Pipeline(1, 4, 4, 16, device=0)
    pipe.upload(b, 0)
    pipe.upload_cpu(ts, core, util, topo)
    res = pipe.run(params(b), check=False)
    got = pipe.to_numpy(res)
    pipe.close()
    return ref, got


def test_cpu_util_golden_and_generated():
    """CPU utilization through chopper_cpu_util vs O17: exact per timestamp (same
    logical-core summation order), medians, maxima, occupancy and SMT co-activity."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cpu_util.json")))
    cases = [g[k] for k in ("spec_one_timestamp", "spec_all_zero", "spec_one_of_eight_physical", "median_even")]
    ts, core, util, topo = tracegen.cpu_samples(7, 1_700_000_000_000_000_000, 1_700_000_000_000_000_000 + 98 * 10 ** 9)
    cases.append({"ts": ts, "core": core, "util": util, "topology": topo})
    for c in cases:
        ref, got = _cpu_both(np.asarray(c["ts"]), np.asarray(c["core"]), np.asarray(c["util"], np.float64),
                             np.asarray(c["topology"]))
        np.testing.assert_array_equal(ref["c_active"], got["cpu.c_active"])
        np.testing.assert_array_equal(ref["c_min"], got["cpu.c_min"])
        np.testing.assert_array_equal(ref["summary"], got["cpu.summary"])


def test_cpu_util_rejects_unsorted():
    import paper_2512_08242_b200 as ch
    with pytest.raises(ch.ChopperError):
        _cpu_both(np.array([2, 1]), np.array([0, 0]), np.array([1.0, 1.0]), np.array([0]))


def test_metric_registry_parity():
    """Derived-metric registry evaluated on the device over point and iteration rows vs the
    oracle's recursive evaluator on the oracle's rows (row counter sums agree to 1e-9; NaN for zero divisors)."""
    import paper_2512_08242_b200 as ch
    b = tracegen.generate(tracegen.config(1))
    C = b.n_counters
    names = [f"c{k}" for k in range(C)]
    exprs = ["c4 / dur_s", "(c1 + c2) * 0.5 - c3 / c0", "c5 / (c6 - c6)", "-c7 * 2 + dur_s", "1e-3 * c0",
             "c0 / 1e-320"]
    p = oracle.default_params(b)
    ref = oracle.run(b, p, max_iters=8)
    pipe = ch.Pipeline(b.cfg.n_gpus, len(b.labels), 8, 4096, device=0)
    pipe.upload(b, C)
    pipe.set_metrics(exprs, names)
    res = pipe.run(p, full=False)
    got = pipe.to_numpy(res, n_ratios=len(p["ratio_num"]))
    for t in ("point", "iter"):
        n = len(ref[f"{t}.busy"])
        cnt = ref[f"{t}.counters"].reshape(C, n)
        for m, e in enumerate(exprs):
            want = oracle.metric_eval(e, names, cnt, ref[f"{t}.busy"])
            np.testing.assert_allclose(got[f"{t}.metrics"][m], want, rtol=1e-9, atol=0, equal_nan=True)
    with pytest.raises(ch.ChopperError, match="MissingCounter"):
        pipe.set_metrics(["c0 / nope"], names)
    with pytest.raises(ch.ChopperError, match="ParseError"):
        pipe.set_metrics(["c0 / (c1"], names)
    pipe.close()


def _ingest_gpu(data: bytes):
    import torch
    import paper_2512_08242_b200 as ch
    b = TinyTrace().ev(0, 0, 10, 20).span(0, 0, 0, 100).bundle()
    pipe = ch.Pipeline(1, 4, 4, 16, device=0)
    pipe.upload(b, 0)
    js = torch.frombuffer(bytearray(data), dtype=torch.uint8).to("cuda:0")
    n = max(data.count(b'"ph"'), 1)
    cols, rep = ch.chopper_ingest_chrome(pipe.ctx, js, n, n)
    out = {k: v.cpu().numpy() for k, v in cols.items()}
    out["meta"] = out["meta"].view(np.uint32)
    out["span_gl"] = out["span_gl"].view(np.uint32)
    pipe.close()
    return out, rep


def test_chrome_ingest_golden():
    """device Chrome-trace ingest vs the oracle's on SPEC.md:104-106's examples, half-to-even rounding,
    escapes and nested / ignored events"""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "chrome.json")))
    for k, c in g.items():
        if k.startswith("_"):
            continue
        ref = oracle.ingest_chrome(c["json"].encode())
        got, rep = _ingest_gpu(c["json"].encode())
        assert rep["n_missing"] == ref["n_missing"], k
        for f in ("t_l", "t_ks", "t_ke", "meta", "name_id", "span_gl", "span_start", "span_end", "span_label"):
            np.testing.assert_array_equal(got[f], ref[f], err_msg=f"{k}.{f}")


@pytest.mark.parametrize("cid", [1, 2])
def test_chrome_ingest_generated(cid):
    """bundle -> Chrome trace (shuffled flows and spans, sub-ns digits) -> device ingest == oracle ingest,
    element by element (and == the bundle's columns)"""
    b = tracegen.generate(tracegen.config(cid))
    data = tracegen.to_chrome(b, seed=cid)
    ref = oracle.ingest_chrome(data)
    got, rep = _ingest_gpu(data)
    assert rep["n_missing"] == ref["n_missing"] == 0
    assert rep["n_names"] == len(ref["names"])
    for f in ("t_l", "t_ks", "t_ke", "meta", "name_id", "span_gl", "span_start", "span_end", "span_label"):
        np.testing.assert_array_equal(got[f], ref[f], err_msg=f)
    np.testing.assert_array_equal(got["t_l"], b.t_l)


def test_chrome_ingest_malformed():
    import paper_2512_08242_b200 as ch
    with pytest.raises(ch.ChopperError):
        _ingest_gpu(b'{"traceEvents": [{"ph": "X", "cat": "kernel", "name": "k", "pid": 0, "tid": 0, "ts": 1, "dur": }]}')
    with pytest.raises(ch.ChopperError):
        _ingest_gpu(b'{"events": []}')


def test_multi_stream_many_tiles():
    """two compute streams per gpu over many tiles: timeline queries go backwards between streams (the event
    pass seeks out of its windows), the compute union is built explicitly, chains per (gpu, stream)"""
    rng = np.random.default_rng(91)
    G = 2
    tt = TinyTrace(n_gpus=G, n_counters=2, labels=["l%d" % i for i in range(4)])
    for g in range(G):
        tt.span(g, 0, 0, 10 ** 9, 5).span(g, 1, 0, 10 ** 9, 0)
        t_host = 0
        t_dev = [1000, 1000]
        names = []
        for k in range(6000):
            st = int(rng.integers(0, 2))
            d = int(rng.integers(20, 300))
            ks = t_dev[st] + int(rng.integers(0, 40))
            t_dev[st] = ks + d
            t_host += int(rng.integers(1, 60))
            tl = min(t_host, ks)
            tt.ev(g, tl, ks, ks + d, stream=st, name=k % 5)
            names.append(k % 5)
            if k % 25 == 0:
                tt.span(g, 3, tl, tl + 2000, k % 4)
            if k % 9 == 0:
                a = ks + int(rng.integers(0, 200))
                tt.ev(g, tl, a, a + int(rng.integers(50, 900)), kind=AG if k % 2 else RS, stream=2 + (k % 2), name=5)
                names.append(5)
            if k % 7 == 0:
                tt.sample(g, ks, int(rng.integers(1300, 2100)), int(rng.integers(500, 900)))
        tt.counter_pass(g, names, [0, 1], rng.integers(0, 1000, size=(2, len(names))).astype(float))
    b = tt.bundle()
    p = params(b, f_gemm=np.full(4, 1e9), op_type=np.array([1, 2, 0, 1], np.int32))
    ref, got, res, _ = run_both(b, p)
    _check_status(ref, got)
    assert_parity(ref, got)


@pytest.mark.slow
def test_config4_tables_only_bench_path():
    """The exact bench path: BASELINE configs[3] at full size in tables-only mode (per-event outputs NULL),
    every table, global row and breakdown against the oracle."""
    b = tracegen.generate(tracegen.config(4))
    ref, got, res, pipe = run_both(b, max_iters=256, full=False)
    _check_status(ref, got)
    assert_parity(ref, got, per_event=False)


def test_hand_worked_skew_and_iteration_bounds(golden):
    """tests/golden/skew.json through the CUDA path: clock offsets, max AG / RS arrival skew, iteration
    comm_union and aligned bounds (the oracle pins of test_oracle_pins_extra)."""
    import test_oracle_pins_extra as pins
    g = golden("skew.json")
    b = pins._skew_trace(g).bundle()
    ref, got, res, pipe = run_both(b, params(b))
    assert_parity(ref, got)
    assert int(got["skew.max_ag"][0]) == max(g["ag"]["skew"]) and int(got["skew.max_rs"][0]) == max(g["rs"]["skew"])
    gi = g["iteration"]
    tt = TinyTrace(n_gpus=2)
    for gpu, key in ((0, "gpu0"), (1, "gpu1_true")):
        d = gi["delta"][gpu]
        evs = [(s + d, e + d, COMPUTE, 0) for s, e in gi[key]["compute"]]
        evs += [(s + d, e + d, AG, 1) for s, e in gi[key]["ag"]] + [(s + d, e + d, RS, 2) for s, e in gi[key]["rs"]]
        for s, e, k, st in sorted(evs):
            tt.ev(gpu, s - 5, s, e, kind=k, stream=st)
        tt.span(gpu, 0, 0, 100_000, 7)
    b = tt.bundle()
    ref, got, res, pipe = run_both(b, params(b))
    assert_parity(ref, got)
    np.testing.assert_array_equal(got["iter.comm_union"], [gi["gpu0"]["comm_union"], gi["gpu1_true"]["comm_union"]])
    np.testing.assert_array_equal(got["glob.aligned_last"], [gi["glob_aligned_last"]])


def test_rates_spec_examples(golden):
    """SPEC.md:305-308 rate examples (bandwidth, counter ratio, ratio of sums) through the CUDA path."""
    import test_oracle_pins_extra as pins
    g = golden("rates.json")
    rs = g["ratio_of_sums"]
    tt = pins._rate_trace(rs["X"], rs["Y"], [500, 700])
    b = tt.bundle()
    p = params(b, ratio_num=np.array([0, 1], np.int32), ratio_den=np.array([1, -1], np.int32),
               ratio_scale=np.array([1.0, 1e-9]), op_type=np.zeros(1, np.int32))
    ref, got, res, pipe = run_both(b, p)
    assert_parity(ref, got)
    assert got["iter.rates"][0] == pytest.approx(rs["expect"], rel=1e-15)
    assert got["point.rates"][0] == pytest.approx(rs["expect"], rel=1e-15)


def test_two_compute_streams_chain():
    """D8 chain per (gpu, stream), three compute streams per GPU (the general a2 path)."""
    rng = np.random.default_rng(11)
    tt = TinyTrace(n_gpus=2)
    evs = []
    for g in range(2):
        tt.span(g, 0, 0, 10 ** 7, 3)
        for st in range(3):
            t = 1000 + 37 * st
            for k in range(300):
                d = int(rng.integers(5, 200))
                evs.append((g, t - int(rng.integers(0, 400)), t, t + d, st))
                t += d + int(rng.integers(0, 50))
    for (g, tl, ks, ke, st) in sorted(evs, key=lambda e: (e[0], e[1])):
        tt.ev(g, tl, ks, ke, stream=st)
    b = tt.bundle()
    ref, got, res, pipe = run_both(b, params(b))
    _check_status(ref, got)
    assert_parity(ref, got)


def test_zero_events():
    """a context with no events at all (a rank whose traced GPUs are empty): every call succeeds with empty
    tables, like the oracle."""
    tt = TinyTrace(n_gpus=2)
    tt.span(0, 0, 0, 100, 1)
    b = tt.bundle()
    ref, got, res, pipe = run_both(b, params(b))
    assert len(got["inst.gpu"]) == 0 and len(ref["inst.gpu"]) == 0
    assert_parity(ref, got)


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_scratch_plan_bounds_high_water(cid):
    """chopper_scratch_plan of the trace's shape (the arena the library is given) bounds the measured
    high-water mark, and the step succeeds in exactly that arena."""
    import paper_2512_08242_b200 as ch
    b = tracegen.generate(tracegen.config(cid))
    p = oracle.default_params(b)
    mi, kc = b.cfg.n_iters + 3, 1 << 15
    pipe = ch.Pipeline(b.cfg.n_gpus, len(b.labels), mi, kc)
    pipe.upload(b, b.n_counters, plan_laminar=True)
    plan = ch.scratch_plan(b.cfg.n_gpus, len(b.labels), mi, kc, b, b.n_counters)
    assert pipe.scratch.numel() == plan["total"]
    for full in (False, True):
        pipe.run(p, full=full)
    used = ch.load_library().chopper_scratch_used(pipe.ctx)
    assert 0 < used <= plan["total"]
    pipe.close()


def test_ctx_reuse_across_steps_with_side_streams():
    """One context over several steps (DESIGN §5 concurrency): the span sort is forked by chopper_load_columns
    onto a side stream and joined by chopper_attribute, chopper_overlap's preparation runs beside the span
    tables, the counter pass beside the event pass.  A load whose step is abandoned before chopper_attribute
    (its sort never joined) and a step with a fatal validation error must leave the next step exact; so must a
    change of trace shape."""
    import paper_2512_08242_b200 as ch
    from paper_2512_08242_b200 import chopper_events, chopper_load_columns, chopper_samples, chopper_spans
    c1 = tracegen.config(1)
    c1.n_gpus = 3
    ba = tracegen.generate(c1)                      # 8 counters
    cfg = tracegen.config(3)
    cfg.n_iters, cfg.n_layers, cfg.n_gpus, cfg.opt_kernels, cfg.warmup = 3, 4, 3, 600, 1
    bb = tracegen.generate(cfg)                     # 20 counters, more spans and iterations
    G = 3
    L = max(len(ba.labels), len(bb.labels))
    mi = max(8, ba.cfg.n_iters + 2, bb.cfg.n_iters + 2)
    from parity import _max_coll
    kc = int(max(16, 4 * max(_max_coll(ba), _max_coll(bb))))
    pipe = ch.Pipeline(G, L, mi, kc, device=0)

    def step(b, bare_load=False):
        pipe.upload(b, b.n_counters)
        p = oracle.default_params(b)
        if bare_load:      # only chopper_load_columns: the side-stream span sort is left unjoined
            d = pipe.d
            ev = chopper_events(n=pipe.N, dispatch_ns=d["t_l"].data_ptr(), start_ns=d["t_ks"].data_ptr(),
                                end_ns=d["t_ke"].data_ptr(), meta=d["meta"].data_ptr(), name_id=d["name_id"].data_ptr())
            sp = chopper_spans(n=pipe.S, gpu_level=d["span_gl"].data_ptr(), start_ns=d["span_start"].data_ptr(),
                               end_ns=d["span_end"].data_ptr(), label=d["span_label"].data_ptr())
            smp = chopper_samples(n=pipe.M, gpu=d["smp_gpu"].data_ptr(), ts_ns=d["smp_ts"].data_ptr(),
                                  freq_mhz=d["smp_freq"].data_ptr(), power_mw=d["smp_power"].data_ptr()) \
                if pipe.M > 0 else None
            assert chopper_load_columns(pipe.ctx, ev, sp, smp) == 0
            return None
        res = pipe.run(p, full=True, check=False)
        got = pipe.to_numpy(res, n_ratios=len(p["ratio_num"]))
        ref = oracle.run(b, p, max_iters=mi)
        assert_parity(ref, got)
        return got

    step(ba)
    step(bb, bare_load=True)           # abandoned after the load
    step(ba)
    ke = bb.t_ke.copy()
    ke[7] = bb.t_ks[7] - 1             # fatal: t_ks > t_ke
    bad = tracegen.dataclasses.replace(bb, t_ke=ke)
    pipe.upload(bad, bad.n_counters)
    res = pipe.run(oracle.default_params(bad), full=False, check=False)
    assert res["load_status"] != 0
    step(bb)
    step(ba)
    pipe.close()


def test_comm_stream_out_of_start_order_lean():
    """Lean a2 (one compute stream) with a communication stream whose starts are not in dispatch order: the
    stream-merge fast path's check fails, which the lean path reads only at chopper_align's read-back; the
    communication buckets are then restored and radix-sorted before chopper_overlap reads them (D1)."""
    tt = TinyTrace(n_gpus=2).span(0, 0, 0, 10_000, 1).span(1, 0, 0, 10_000, 1)
    for g in range(2):
        t = 0
        for k in range(40):
            tt.ev(g, t, t + 5, t + 60)                                        # compute, stream 0
            t += 70
        # all-gathers dispatched in this order, started out of order; reduce-scatters in order
        for k, ks in enumerate([300, 100, 900, 500, 700, 200]):
            tt.ev(g, 50 + 10 * k, ks, ks + 150, kind=AG, stream=1)
        for k in range(5):
            tt.ev(g, 60 + 10 * k, 1000 + 300 * k, 1100 + 300 * k, kind=RS, stream=2)
    ref, got, _, _ = _tiny(tt)
    _check_status(ref, got)
    assert_parity(ref, got)
