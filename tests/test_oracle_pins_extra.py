"""More pins for the CPU oracle (round 2): the outputs the round-1 pins left open.

- O4 arrival skew per collective (D13), hand-worked on 3 GPUs with known clock offsets (golden/skew.json);
- O11 iteration extras (comm_union, aligned first / last) and O12 glob.aligned_* (golden/skew.json);
- ratio-of-sums rates against SPEC.md:305-308's worked examples (golden/rates.json);
- O8 chain per (gpu, stream) with two compute streams against Python sorted() (D8);
- north_star's aggregate check: per GPU, sum of COMPUTE overlap <= min(sum busy, |U_g|), and equal to
  |V_g ∩ U_g| computed here by an independent interval sweep when the compute intervals are disjoint;
- R8: a counter pass holding a non-finite value is skipped (rule CV_COUNTER_NONFINITE), the other passes merge.

Each check compares the oracle with a value written by hand from the paper / SPEC, or with an
independent method (Python sorted(), an event sweep over interval endpoints); none re-types the oracle.
"""
import numpy as np
import pytest

import oracle
import tracegen
from tinytrace import AG, COMPUTE, RS, TinyTrace, params

V_COUNTER_NONFINITE = 8
ST_VALIDATION = 1 << 1


def _skew_trace(g):
    """3 GPUs, GPU g's device clock = true + delta_g; AG on stream 1, RS on stream 2."""
    d = g["delta"]
    tt = TinyTrace(n_gpus=3)
    for gpu in range(3):
        for kind, key in ((AG, "ag"), (RS, "rs")):
            for j, starts in enumerate(g[key]["true_start"]):
                ks = starts[gpu] + d[gpu]
                ke = g[key]["true_end"][j] + d[gpu]
                tt.ev(gpu, ks - 10, ks, ke, kind=kind, stream=1 if kind == AG else 2)
    return tt


def test_arrival_skew_hand_worked(golden):
    g = golden("skew.json")
    b = _skew_trace(g).bundle()
    o = oracle.run(b, params(b))
    np.testing.assert_array_equal(o["gpu.delta"], g["delta"])
    np.testing.assert_array_equal(o["gpu.delta_flag"], [0, 0, 0])
    # a skew from END times would be all zero, one that forgets delta differs by the offsets
    np.testing.assert_array_equal(o["skew.ag"], g["ag"]["skew"])
    np.testing.assert_array_equal(o["skew.rs"], g["rs"]["skew"])


def test_arrival_skew_uses_lowest_gpu_as_reference(golden):
    """Shifting every GPU's clock by the same amount changes no skew and no delta (ref = lowest gpu)."""
    g = golden("skew.json")
    b = _skew_trace(g).bundle()
    sh = tracegen.dataclasses.replace(b, t_l=b.t_l + 12345, t_ks=b.t_ks + 12345, t_ke=b.t_ke + 12345)
    o = oracle.run(sh, params(sh))
    np.testing.assert_array_equal(o["gpu.delta"], g["delta"])
    np.testing.assert_array_equal(o["skew.ag"], g["ag"]["skew"])


def test_iteration_comm_union_and_aligned_bounds(golden):
    g = golden("skew.json")["iteration"]
    tt = TinyTrace(n_gpus=2)
    for gpu, key in ((0, "gpu0"), (1, "gpu1_true")):
        d = g["delta"][gpu]
        evs = [(s + d, e + d, COMPUTE, 0) for s, e in g[key]["compute"]]
        evs += [(s + d, e + d, AG, 1) for s, e in g[key]["ag"]]
        evs += [(s + d, e + d, RS, 2) for s, e in g[key]["rs"]]
        for s, e, k, st in sorted(evs):
            tt.ev(gpu, s - 5, s, e, kind=k, stream=st)
        tt.span(gpu, 0, 0, 100_000, 7)
    b = tt.bundle()
    o = oracle.run(b, params(b))
    np.testing.assert_array_equal(o["gpu.delta"], g["delta"])
    np.testing.assert_array_equal(o["iter.comm_union"], [g["gpu0"]["comm_union"], g["gpu1_true"]["comm_union"]])
    np.testing.assert_array_equal(o["iter.aligned_first"],
                                  [g["gpu0"]["aligned_first"], g["gpu1_true"]["aligned_first"]])
    np.testing.assert_array_equal(o["iter.aligned_last"], [g["gpu0"]["aligned_last"], g["gpu1_true"]["aligned_last"]])
    np.testing.assert_array_equal(o["glob.aligned_first"], [g["glob_aligned_first"]])
    np.testing.assert_array_equal(o["glob.aligned_last"], [g["glob_aligned_last"]])
    np.testing.assert_array_equal(o["iter.step"], [7, 7])


def _rate_trace(x, y, dur):
    """one iteration, one labelled op, len(x) COMPUTE kernels carrying counters X (slot 0), Y (slot 1)"""
    tt = TinyTrace(n_counters=2, labels=["op"])
    tt.span(0, 0, 0, 10 ** 9, 0).span(0, 3, 0, 10 ** 9, 0)
    t = 1000
    for k in range(len(x)):
        tt.ev(0, t - 10, t, t + dur[k], name=k)
        t += dur[k] + 100
    tt.counter_pass(0, list(range(len(x))), [0, 1], [list(x), list(y)])
    return tt


def _rates(tt, num, den, scale):
    b = tt.bundle()
    p = params(b, ratio_num=np.array(num, np.int32), ratio_den=np.array(den, np.int32),
               ratio_scale=np.array(scale, np.float64), op_type=np.zeros(1, np.int32))
    return oracle.run(b, p)


def test_rates_bandwidth_spec(golden):
    g = golden("rates.json")
    bw = g["bandwidth"]
    o = _rates(_rate_trace([bw["bytes"]], [0.0], [bw["dur_ns"]]), [0], [-1], [1.0])
    assert o["iter.rates"][0] == pytest.approx(bw["expect"], rel=1e-15)
    assert o["point.rates"][0] == pytest.approx(bw["expect"], rel=1e-15)
    # scale is applied once: bytes/s -> GB/s
    o = _rates(_rate_trace([bw["bytes"]], [0.0], [bw["dur_ns"]]), [0], [-1], [1e-9])
    assert o["iter.rates"][0] == pytest.approx(bw["expect"] * 1e-9, rel=1e-15)


def test_rates_counter_ratio_spec(golden):
    g = golden("rates.json")
    r = g["ratio"]
    o = _rates(_rate_trace([r["X"]], [r["Y"]], [500]), [0], [1], [1.0])
    assert o["iter.rates"][0] == r["expect"] and o["point.rates"][0] == r["expect"]
    rs = g["ratio_of_sums"]
    o = _rates(_rate_trace(rs["X"], rs["Y"], [500, 700]), [0, 1], [1, 0], [1.0, 1.0])
    np.testing.assert_allclose(o["iter.rates"], [rs["expect"], 1.0 / rs["expect"]], rtol=1e-15)
    np.testing.assert_allclose(o["point.rates"], [rs["expect"], 1.0 / rs["expect"]], rtol=1e-15)


def test_two_compute_streams_chain_against_sorted():
    """D8: the chain is per (gpu, compute stream) in t_ks order, ties input order."""
    rng = np.random.default_rng(11)
    tt = TinyTrace(n_gpus=2)
    evs = []
    for g in range(2):
        for st in range(3):
            t = 1000 + 37 * st
            for k in range(60):
                d = int(rng.integers(5, 200))
                evs.append((g, t - int(rng.integers(0, 400)), t, t + d, st))
                t += d + int(rng.integers(0, 50))
    for (g, tl, ks, ke, st) in sorted(evs, key=lambda e: (e[0], e[1])):
        tt.ev(g, tl, ks, ke, stream=st)
    b = tt.bundle()
    o = oracle.run(b, params(b))
    assert o["status"][0] == 0 and o["val.count"][5] == 0
    stream = (b.meta >> 8) & 0xFFFF
    gpu = b.meta >> 24
    expect = np.full(b.n_events, -1)
    for g in range(2):
        for st in range(3):
            idx = [i for i in range(b.n_events) if gpu[i] == g and stream[i] == st]
            srt = sorted(idx, key=lambda i: (b.t_ks[i], i))
            expect[srt[1:]] = srt[:-1]
    np.testing.assert_array_equal(o["ev.pred"], expect)
    has = expect >= 0
    np.testing.assert_array_equal((o["ev.prep"] + o["ev.call"])[has], (b.t_ks - b.t_ke[np.maximum(expect, 0)])[has])
    assert (o["ev.prep"][~has] == 0).all() and (o["ev.call"][~has] == 0).all()


def _union_len(iv):
    """|union of half-open intervals| by an endpoint sweep (independent of the oracle's merge)."""
    pts = sorted([(s, 1) for s, e in iv if e > s] + [(e, -1) for s, e in iv if e > s])
    tot, depth, last = 0, 0, None
    for t, dlt in pts:
        if depth > 0:
            tot += t - last
        depth += dlt
        last = t
    return tot


def _inter_len(a, b):
    """|union(a) ∩ union(b)| = |A| + |B| - |A ∪ B|"""
    return _union_len(a) + _union_len(b) - _union_len(list(a) + list(b))


@pytest.mark.parametrize("cid", [1, 3])
def test_sum_overlap_bounded_by_comm_and_compute(cid):
    """north_star: overlap <= min(comm, compute) in aggregate, per GPU; on one compute stream the COMPUTE
    intervals are disjoint, so the summed overlap is exactly |V_g ∩ U_g|."""
    cfg = tracegen.config(cid)
    if cid == 3:
        cfg.n_iters, cfg.n_layers, cfg.n_gpus, cfg.opt_kernels, cfg.warmup = 2, 3, 2, 300, 0
    b = tracegen.generate(cfg)
    o = oracle.run(b)
    kind = b.meta & 0xFF
    gpu = b.meta >> 24
    for g in range(cfg.n_gpus):
        comp = (gpu == g) & (kind == COMPUTE)
        comm = (gpu == g) & np.isin(kind, [AG, RS, 3])
        U = list(zip(b.t_ks[comm], b.t_ke[comm]))
        V = list(zip(b.t_ks[comp], b.t_ke[comp]))
        s_ovl = int(o["ev.ovl"][comp].sum())
        busy = int((b.t_ke - b.t_ks)[comp].sum())
        assert s_ovl <= min(busy, _union_len(U))
        assert s_ovl == _inter_len(U, V)
        # comm side: each comm kernel's covl <= its runtime, and the comm union's covered part is |U ∩ V|
        assert (o["ev.ovl"][comm] <= (b.t_ke - b.t_ks)[comm]).all()


def test_nonfinite_counter_pass_skipped():
    """R8: a pass with a NaN / inf value is skipped whole (CV_COUNTER_NONFINITE, index = pass), its slots stay
    absent; the other passes of the GPU merge as usual."""
    tt = TinyTrace(n_counters=3)
    tt.span(0, 0, 0, 10 ** 6, 0)
    for k in range(4):
        tt.ev(0, 100 * k, 100 * k + 1, 100 * k + 50, name=k)
    tt.counter_pass(0, [0, 1, 2, 3], [0], [[1, 2, 3, 4]])
    tt.counter_pass(0, [0, 1, 2, 3], [1, 2], [[5, 6, float("nan"), 8], [9, 10, 11, 12]])
    b = tt.bundle()
    o = oracle.run(b, params(b))
    assert o["val.count"][V_COUNTER_NONFINITE] == 1 and o["val.first"][V_COUNTER_NONFINITE] == 1
    assert o["status"][0] & ST_VALIDATION
    np.testing.assert_array_equal(o["gpu.counter_present"], [1, 0, 0])
    cm = o["ev.counters"].reshape(3, -1)
    np.testing.assert_array_equal(cm[0], [1, 2, 3, 4])
    np.testing.assert_array_equal(cm[1:], 0)
    np.testing.assert_array_equal(o["inst.counters"].reshape(3, -1)[:, 0], [10, 0, 0])
    # an inf in the first pass skips that one instead
    tt.passes[0] = (0, np.arange(4, dtype=np.int32), np.array([0], np.int32), np.array([[1, np.inf, 3, 4]]))
    tt.passes[1] = (0, np.arange(4, dtype=np.int32), np.array([1, 2], np.int32),
                    np.array([[5, 6, 7, 8], [9, 10, 11, 12]], np.float64))
    b = tt.bundle()
    o = oracle.run(b, params(b))
    assert o["val.first"][V_COUNTER_NONFINITE] == 0
    np.testing.assert_array_equal(o["gpu.counter_present"], [0, 1, 1])
