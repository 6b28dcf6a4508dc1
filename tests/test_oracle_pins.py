"""Pins for the CPU oracle: worked examples (tests/golden, cited), closed forms,
brute force on tiny inputs, invariants and closed-form scenarios.

None of these checks re-types the oracle's formula: each compares it to a
value the paper / SPEC prints, to an independent brute-force method (ns
rasters, O(n*S) scans, Python sorted()), or to a mathematical identity.
"""
import itertools

import numpy as np
import pytest

import oracle
import tracegen
from tinytrace import AG, COMPUTE, COPY, MEMOP, RS, TinyTrace, params

V_START_AFTER_END, V_GPU_NOT_GROUPED, V_DISPATCH_DECREASING, V_BAD_META, V_TS_RANGE, V_STREAM_OVERLAP, \
    V_SPAN_BAD, V_SAMPLES_UNSORTED, V_COUNTER_NONFINITE = range(9)
ST_VALIDATION, ST_ALIGNMENT, ST_AMBIGUOUS = 1 << 1, 1 << 3, 1 << 4
BD = dict(n=0, method=1, d_act=2, d0=3, d50=4, d_thr=5, inst=6, util=7, overlap=8, d_peak=9, freq=10, launch=11,
          residual=12, freq_samples=13, flags=14, label=15)


def run(tt, **kw):
    b = tt.bundle()
    return oracle.run(b, params(b, **kw))


def bd_rows(o):
    return o["bd.rows"].reshape(-1, 16)


# ---------------------------------------------------------------------------
# Eqs. 1-3
# ---------------------------------------------------------------------------
def test_launch_triples_spec(golden):
    g = golden("launch_triples.json")
    for prev_end, dispatch, start, prep, call, launch in g["rows"]:
        tt = TinyTrace().ev(0, 0, 50, prev_end).ev(0, dispatch, start, start + 10)
        o = run(tt)
        assert o["ev.prep"][1] == prep and o["ev.call"][1] == call and prep + call == launch
        assert o["ev.prep"][0] == 0 and o["ev.call"][0] == 0   # first kernel: no predecessor


@pytest.mark.parametrize("skewed", [False, True])
def test_launch_identity_random(skewed):
    """10,000 random (prev end, dispatch, start) triples: prep, call >= 0 and prep + call = t_ks - t_ke(p)
    whenever the stream is valid (D6)."""
    rng = np.random.default_rng(7 + skewed)
    n = 10_000
    dur = rng.integers(1, 1000, n)
    bub = rng.integers(0, 1000, n)
    ks = np.cumsum(np.r_[0, (dur + bub)[:-1]]) + 10_000
    ke = ks + dur
    if skewed:
        pe = np.r_[ks[0] - 5, ke[:-1]]
        tl = pe + rng.integers(-500, 2500, n)
    else:
        tl = ks - rng.integers(0, 3000, n)
    tt = TinyTrace()
    for i in range(n):
        tt.ev(0, int(tl[i]), int(ks[i]), int(ke[i]))
    b = tt.bundle()
    o = oracle.run(b, params(b))
    order = np.argsort(b.t_ks, kind="stable")
    prep, call = o["ev.prep"][order], o["ev.call"][order]
    sks, ske = b.t_ks[order], b.t_ke[order]
    assert prep[0] == 0 and call[0] == 0
    assert (prep >= 0).all() and (call >= 0).all()
    np.testing.assert_array_equal(prep[1:] + call[1:], sks[1:] - ske[:-1])
    # telescoping: sum(busy + launch) over the chain = last end - first start
    assert (ske - sks).sum() + prep.sum() + call.sum() == ske[-1] - sks[0]


# ---------------------------------------------------------------------------
# overlap (D9)
# ---------------------------------------------------------------------------
def test_overlap_spec(golden):
    g = golden("overlap.json")
    for case in g["cases"]:
        tt = TinyTrace().ev(0, 0, case["kernel"][0], case["kernel"][1])
        for j, (s, e) in enumerate(case["comm"]):
            tt.ev(0, 1 + j, s, e, kind=AG, stream=1 + j)
        o = run(tt)
        k = [i for i in range(len(o["ev.ovl"])) if o["ev.ovl"] is not None]
        b = tt.bundle()
        ci = int(np.where((b.meta & 0xFF) == COMPUTE)[0][0])
        assert o["ev.ovl"][ci] == case["ovl"]
        assert o["ev.ovl"][ci] / (case["kernel"][1] - case["kernel"][0]) == pytest.approx(case["ratio"], abs=0)
        del k


def test_overlap_weighted_spec(golden):
    """op-level ratio = sum(ovl)/sum(busy)."""
    g = golden("overlap.json")
    for case, comm_end in zip(g["weighted"], (100, 120)):
        (r1, _), (r2, _) = case["kernels"]
        tt = TinyTrace().span(0, 0, 0, 10_000, 100).span(0, 3, 0, 10_000, 0)
        tt.ev(0, 1, 0, r1).ev(0, 2, r1, r1 + r2).ev(0, 3, 0, comm_end, kind=AG, stream=1)
        o = run(tt)
        assert o["inst.ovl"][0] / o["inst.busy"][0] == pytest.approx(case["ratio"], abs=1e-15)


def _raster(ivals, lo, hi):
    m = np.zeros(hi - lo, dtype=bool)
    for s, e in ivals:
        m[max(s, lo) - lo:max(min(e, hi), lo) - lo] = True
    return m


def test_overlap_bruteforce_raster():
    """1,000 random interval sets vs an ns raster; plus monotone / split invariance."""
    rng = np.random.default_rng(11)
    for batch in range(4):
        G = 250
        tt = TinyTrace(n_gpus=G)
        truth = {}
        for gg in range(G):
            comm = []
            for j in range(rng.integers(0, 6)):
                s = int(rng.integers(0, 3000)); e = s + int(rng.integers(0, 800))
                comm.append((s, e, 1 + j % 2))
            t = int(rng.integers(0, 200)); comp = []
            while t < 3000:
                d = int(rng.integers(0, 300)); comp.append((t, t + d)); t += d + int(rng.integers(0, 200))
            tl = 0
            for (s, e) in comp:
                tt.ev(gg, tl, s, e); tl += 1
            for (s, e, st) in comm:
                tt.ev(gg, tl, s, e, kind=AG if st == 1 else RS, stream=st); tl += 1
            truth[gg] = (comp, comm)
        b = tt.bundle()
        o = oracle.run(b, params(b))
        i = 0
        for gg in range(G):
            comp, comm = truth[gg]
            cr = _raster([(s, e) for s, e, _ in comm], 0, 5000)
            vr = _raster(comp, 0, 5000)
            for (s, e) in comp:
                assert o["ev.ovl"][i] == cr[s:e].sum(); i += 1
            for (s, e, _) in comm:
                assert o["ev.ovl"][i] == vr[s:e].sum(); i += 1


def test_overlap_monotone_and_split():
    rng = np.random.default_rng(3)
    for trial in range(50):
        comp = [(100 * k, 100 * k + int(rng.integers(1, 100))) for k in range(10)]
        comm = [(int(s), int(s) + int(rng.integers(1, 400))) for s in rng.integers(0, 1000, 3)]

        def ovl(cm):
            tt = TinyTrace()
            tl = 0
            for s, e in comp:
                tt.ev(0, tl, s, e); tl += 1
            for j, (s, e) in enumerate(cm):
                tt.ev(0, tl, s, e, kind=AG, stream=1 + j); tl += 1
            return run(tt)["ev.ovl"][:len(comp)]
        base = ovl(comm)
        extra = ovl(comm + [(int(rng.integers(0, 1000)), 1200)])
        assert (extra >= base).all()
        s, e = comm[0]
        m = (s + e) // 2
        np.testing.assert_array_equal(ovl([(s, m), (m, e)] + comm[1:]), base)


# ---------------------------------------------------------------------------
# attribution (D3, D4)
# ---------------------------------------------------------------------------
def test_annotation_spec(golden):
    g = golden("annotation.json")
    tt = TinyTrace()
    names = list(g["spans"])
    for nm in names:
        lv, s, e = g["spans"][nm]
        tt.span(0, lv, s, e, 0)
    for c in g["cases"]:
        tt.ev(0, c["dispatch"], c["dispatch"] + 5, c["dispatch"] + 6)
    o = run(tt)
    ai = o["ev.span_idx"].reshape(4, -1)
    for i, c in enumerate(g["cases"]):
        ex = c["expect"]
        assert ai[0, i] == names.index(ex["it"])
        assert ai[1, i] == names.index(ex["ph"])
        assert ai[3, i] == (names.index(ex["op"]) if ex["op"] else -1)
        assert ai[2, i] == -1
    amb = g["ambiguous"]
    for t, expect in ((amb["dispatch"], -2), (120, 0), (220, 1)):
        tt = TinyTrace().span(0, 0, 0, 1000, 0)
        for s, e in amb["spans"]:
            tt.span(0, 3, s, e, 0)
        tt.ev(0, t, t + 1, t + 2)
        o = run(tt)
        got = o["ev.span_idx"].reshape(4, -1)[3, 0]
        assert got == (expect if expect < 0 else expect + 1)
        assert bool(o["status"][0] & ST_AMBIGUOUS) == (expect == -2)


def _brute_attr(spans, t):
    """O(S) scan: innermost containing span (greatest start, then smallest end, then index), -2 if not a chain."""
    cont = [j for j, (s, e) in spans if s <= t < e]
    if not cont:
        return -1
    d = dict(spans)
    for a, b in itertools.combinations(cont, 2):
        (sa, ea), (sb, eb) = d[a], d[b]
        if not ((sa <= sb and eb <= ea) or (sb <= sa and ea <= eb)):
            return -2
    return min(cont, key=lambda j: (-d[j][0], d[j][1], j))


@pytest.mark.parametrize("seed", range(6))
def test_attribution_bruteforce(seed):
    rng = np.random.default_rng(100 + seed)
    G = 3
    tt = TinyTrace(n_gpus=G)
    allspans = []
    for g in range(G):
        for lv in range(4):
            for _ in range(int(rng.integers(0, 12))):
                s = int(rng.integers(0, 2000))
                e = s + int(rng.integers(0, 600 if lv < 3 else 300))
                if seed % 2 == 0 and lv == 3 and rng.random() < 0.7:
                    # nested families (laminar): children inside an existing span of this level
                    par = [x for x in allspans if x[0] == g and x[1] == lv]
                    if par:
                        _, _, ps, pe = par[int(rng.integers(0, len(par)))]
                        if pe - ps >= 2:
                            s = int(rng.integers(ps, pe - 1)); e = int(rng.integers(s + 1, pe + 1))
                allspans.append((g, lv, s, e))
                tt.span(g, lv, s, e, lv)
        for t in sorted(rng.integers(0, 2600, 60)):
            tt.ev(g, int(t), int(t) + 1, int(t) + 2)
    b = tt.bundle()
    o = oracle.run(b, params(b))
    ai = o["ev.span_idx"].reshape(4, -1)
    for i in range(b.n_events):
        g = int(b.meta[i] >> 24)
        for lv in range(4):
            sp = [(j, (int(b.span_start[j]), int(b.span_end[j]))) for j in range(len(b.span_gl))
                  if int(b.span_gl[j]) == (g << 8 | lv)]
            assert ai[lv, i] == _brute_attr(sp, int(b.t_l[i])), (i, lv)


# ---------------------------------------------------------------------------
# counter alignment
# ---------------------------------------------------------------------------
def test_alignment_spec(golden):
    g = golden("alignment.json")
    nid = {"A": 1, "B": 2}
    names = [nid[x] for x in g["runtime"]]

    def trace():
        tt = TinyTrace(n_counters=2)
        for k, nm in enumerate(names):
            tt.ev(0, 10 * k, 10 * k + 1, 10 * k + 5, name=nm)
        tt.ev(0, 100, 101, 102, kind=MEMOP, stream=3, name=9)   # DMA memop: not enumerated by passes (D2)
        return tt
    tt = trace().counter_pass(0, [nid[x] for x in g["merge"]["pass_names"]], [0], [g["merge"]["values"]])
    o = run(tt)
    np.testing.assert_array_equal(o["ev.counters"].reshape(2, -1)[0][:3], g["merge"]["values"])
    assert o["status"][0] == 0
    tt = trace().counter_pass(0, [nid[x] for x in g["mismatch"]["pass_names"]], [0], [[1, 2]])
    o = run(tt)
    assert o["pass.mismatch"][0] == g["mismatch"]["first_divergence"] and o["status"][0] & ST_ALIGNMENT
    # two passes, disjoint counters -> both merged; conflicting slot -> ConflictingCounter
    tt = trace().counter_pass(0, names, [0], [[1, 2, 3]]).counter_pass(0, names, [1], [[4, 5, 6]])
    o = run(tt)
    np.testing.assert_array_equal(o["ev.counters"].reshape(2, -1)[:, :3], [[1, 2, 3], [4, 5, 6]])
    tt = trace().counter_pass(0, names, [0], [[1, 2, 3]]).counter_pass(0, names, [0], [[1, 2.5, 3]])
    o = run(tt)
    assert o["pass.conflict"][1] == 1 and o["status"][0] & ST_ALIGNMENT


# ---------------------------------------------------------------------------
# roll-up and throughput
# ---------------------------------------------------------------------------
def test_rollup_spec(golden):
    g = golden("rollup_throughput.json")["rollup"]
    tt = TinyTrace().span(0, 0, 0, 1000, 100)
    t = 100
    for k, rt in enumerate(g["runtimes"]):
        tt.ev(0, k, t, t + rt)
        t += rt + (g["bubbles"][k] if k < len(g["bubbles"]) else 0)
    o = run(tt)
    assert o["iter.busy"][0] == g["duration"]
    assert o["iter.prep"][0] + o["iter.call"][0] == g["launch"]
    assert o["iter.wall"][0] == g["duration"] + g["launch"]


def test_throughput_spec(golden):
    g = golden("rollup_throughput.json")["throughput"]
    dur = int(g["max_dur_launch_s"] * 1e9)
    tt = TinyTrace(n_gpus=2, b=g["b"], s=g["s"])
    for gg, d in ((0, dur), (1, dur // 2)):
        tt.span(gg, 0, 0, 10 ** 10, 7).ev(gg, 0, 10, 10 + d)
    o = oracle.run(tt.bundle(), params(tt.bundle(), R=g["R"]))
    assert o["glob.throughput"][0] == pytest.approx(g["tok_per_s"], rel=1e-12)
    # one GPU twice as slow -> throughput halves
    tt = TinyTrace(n_gpus=2, b=g["b"], s=g["s"])
    for gg, d in ((0, dur), (1, 2 * dur)):
        tt.span(gg, 0, 0, 10 ** 10, 7).ev(gg, 0, 10, 10 + d)
    o = oracle.run(tt.bundle(), params(tt.bundle(), R=g["R"]))
    assert o["glob.throughput"][0] == pytest.approx(g["tok_per_s"] / 2, rel=1e-12)


def test_throughput_median_even():
    """median of an even count = mean of the two central values."""
    tt = TinyTrace(b=1, s=1)
    t = 0   # back-to-back iterations: the inter-iteration bubble is launch overhead
    for it, d in enumerate((10 ** 9, 2 * 10 ** 9, 4 * 10 ** 9, 8 * 10 ** 9)):
        tt.span(0, 0, it * 10, it * 10 + 10, it).ev(0, it * 10, t, t + d)
        t += d
    o = oracle.run(tt.bundle(), params(tt.bundle(), R=1))
    assert o["glob.throughput_median"][0] == pytest.approx((0.5 + 0.25) / 2, rel=1e-12)


# ---------------------------------------------------------------------------
# Eq. 4 FLOPs
# ---------------------------------------------------------------------------
def test_flops_spec(golden):
    g = golden("breakdown.json")["flops"]
    assert oracle.gemm_flops(*g["gemm_mnk"]) == g["gemm"]
    assert oracle.attention_flops(*g["attn_bhsd"]) == g["attn"]
    # brute-force multiply-add count of S = Q K^T and O = P V for one head
    b, h, s, d = g["attn_bhsd"]
    macs = sum(1 for _ in itertools.product(range(s), range(s), range(d))) * 2
    assert 2 * macs * b * h == g["attn"]
    labels = tracegen.label_vocabulary()
    sh = tracegen.workload_shapes(tracegen.config(2))
    base = oracle.flops_table(labels, sh)
    t2 = oracle.flops_table(labels, dict(sh, b=2 * sh["b"]))
    s2 = oracle.flops_table(labels, dict(sh, s=2 * sh["s"]))
    gemm = [i for i, l in enumerate(labels) if tracegen.op_kind(l) == 1]
    fa = [i for i, l in enumerate(labels) if tracegen.op_kind(l) == 2]
    np.testing.assert_array_equal(t2[gemm], 2 * base[gemm])
    np.testing.assert_array_equal(s2[fa], 4 * base[fa])


# ---------------------------------------------------------------------------
# Eqs. 4-8 breakdown
# ---------------------------------------------------------------------------
def _points_trace(points, n_counters=0, counters=None, samples=None):
    """one GEMM op (label 0) per iteration; point = (ovl, busy); comm interval gives the overlap."""
    tt = TinyTrace(n_counters=n_counters)
    tl = 0
    names = []
    for it, (ovl, busy) in enumerate(points):
        base = it * 10 ** 11
        tt.span(0, 0, base, base + 10 ** 11, it).span(0, 3, base, base + 10 ** 10, 0)
        tt.ev(0, base + 1, base + 1000, base + 1000 + busy, name=5)
        names.append(5)
        if ovl:
            tt.ev(0, base + 2, base + 1000, base + 1000 + ovl, kind=AG, stream=1, name=6)
            names.append(6)
        tl += 1
    if counters is not None:
        vals = []
        for slot in range(n_counters):
            row = []
            for it, (ovl, busy) in enumerate(points):
                row.append(counters[slot][it])
                if ovl:
                    row.append(0.0)
            vals.append(row)
        tt.counter_pass(0, names, list(range(n_counters)), vals)
    for (ts, f) in (samples or []):
        tt.sample(0, ts, f, 1)
    return tt


def test_breakdown_buckets_spec(golden):
    g = golden("breakdown.json")
    pts = [(int(round(r * d)), d) for r, d in g["buckets"]["points"]]
    tt = _points_trace(pts)
    b = tt.bundle()
    o = oracle.run(b, params(b, f_gemm=np.full(4, g["dthr"]["flops"]), tpt_peak=g["dthr"]["peak"]))
    row = bd_rows(o)[0]
    assert row[BD["method"]] == 0
    assert row[BD["d0"]] == pytest.approx(g["buckets"]["d0"] * 1e-9, rel=1e-15)
    assert row[BD["d50"]] == pytest.approx(g["buckets"]["d50"] * 1e-9, rel=1e-15)
    assert row[BD["overlap"]] == pytest.approx(g["buckets"]["ovr_overlap"], rel=1e-15)
    assert row[BD["d_thr"]] == pytest.approx(g["dthr"]["seconds"], rel=1e-15)


def test_breakdown_single_point_insufficient():
    tt = _points_trace([(0, 100)])
    o = oracle.run(tt.bundle(), params(tt.bundle()))
    row = bd_rows(o)[0]
    assert row[BD["n"]] == 1 and int(row[BD["flags"]]) & 128


def test_breakdown_all_zero_overlap_fit():
    """all overlaps 0 -> d0 = median, d50 via slope-0 fit = same median."""
    tt = _points_trace([(0, 100), (0, 110), (0, 130)])
    o = oracle.run(tt.bundle(), params(tt.bundle()))
    row = bd_rows(o)[0]
    assert row[BD["method"]] == 1
    assert row[BD["d0"]] == pytest.approx(110e-9, rel=1e-15) and row[BD["d50"]] == pytest.approx(110e-9, rel=1e-15)
    assert row[BD["overlap"]] == 1.0


def test_ovr_freq_spec(golden):
    g = golden("breakdown.json")["freq"]
    D0, D50 = 1_250_000_000, 1_500_000_000
    pts = [(0, D0), (D50 // 2, D50), (D50 // 2, D50)]
    tt = _points_trace(pts, n_counters=1, counters=[[g["c_gpu"]] * 3])
    b = tt.bundle()
    o = oracle.run(b, params(b, freq_peak_hz=g["freq_peak"]))
    row = bd_rows(o)[0]
    assert row[BD["d_peak"]] == pytest.approx(g["d_peak"], rel=1e-15)
    assert row[BD["d_act"]] == pytest.approx(g["d_act"], rel=1e-15)
    assert row[BD["overlap"]] == pytest.approx(g["ovr_overlap"], rel=1e-15)
    assert row[BD["freq"]] == pytest.approx(g["ovr_freq"], rel=1e-14)


def test_compose_spec(golden):
    g = golden("breakdown.json")["compose"]
    D0, D50 = 2_500_000, 2_750_000
    pts = [(0, D0), (D50 // 2, D50), (D50 // 2, D50)]
    cyc = g["d_act"] / g["ovr_overlap"] / g["ovr_freq"] * 2.1e9   # D_peak * Freq_peak
    cnt = [[cyc] * 3, [1.3e12] * 3, [0.5] * 3, [1.0] * 3]
    tt = _points_trace(pts, n_counters=4, counters=cnt)
    b = tt.bundle()
    o = oracle.run(b, params(b))
    row = bd_rows(o)[0]
    assert row[BD["d_thr"]] == pytest.approx(g["d_thr"], rel=1e-15)
    assert row[BD["inst"]] == pytest.approx(g["ovr_inst"], rel=1e-15)
    assert row[BD["util"]] == pytest.approx(g["ovr_util"], rel=1e-15)
    assert row[BD["overlap"]] == pytest.approx(g["ovr_overlap"], rel=1e-15)
    assert row[BD["freq"]] == pytest.approx(g["ovr_freq"], rel=1e-12)
    assert row[BD["d_act"]] == pytest.approx(g["d_act"], rel=1e-15)
    assert row[BD["residual"]] == pytest.approx(g["residual"], rel=1e-12)


def test_frequency_only_scenario():
    """All r = 0 and clocks held at 0.8 x Freq_peak: Ovr_overlap = 1, Ovr_freq = Ovr_freq_samples = 1.25
    (SPEC.md:401, 569).  Durations are multiples of 25 ns so cycles = dur * 1680 / 1000 is exact."""
    durs = [4_000_000, 4_100_000, 3_900_000, 4_050_000, 3_975_000]
    cyc = [d * 1680 // 1000 for d in durs]
    tt = _points_trace([(0, d) for d in durs], n_counters=1, counters=[cyc],
                       samples=[(0, 1680), (10 ** 12, 1680)])
    o = oracle.run(tt.bundle(), params(tt.bundle()))
    row = bd_rows(o)[0]
    assert row[BD["overlap"]] == 1.0
    assert row[BD["freq"]] == pytest.approx(1.25, rel=1e-12)
    assert row[BD["freq_samples"]] == pytest.approx(1.25, rel=1e-12)


def test_overlap_only_scenario():
    """half the points at r = 0, half at r = 0.5 stretched by (1 + kappa/2): Ovr_overlap = 1 + kappa/2."""
    kappa = 0.2
    base = [1_000_000, 1_000_010, 999_990, 1_000_020]
    pts = [(0, d) for d in base] + [(int(d * (1 + kappa / 2)) // 2, int(d * (1 + kappa / 2))) for d in base]
    tt = _points_trace(pts)
    o = oracle.run(tt.bundle(), params(tt.bundle()))
    row = bd_rows(o)[0]
    assert row[BD["method"]] == 0
    assert row[BD["overlap"]] == pytest.approx(1 + kappa / 2, rel=1e-12)


def test_breakdown_residual_identity_generated():
    """With the self-consistent utilization (D18, no util slots) the residual reduces algebraically to
    TPT*U*Cg/(Fp*Freq_peak) = 1 whenever Fp/Cg is the same for every point of a label, which the
    generator guarantees (flops = cycles * rate_label, exact integers).  SURVEY 8(c) O13 identity."""
    b = tracegen.generate(tracegen.config(1))
    p = oracle.default_params(b)
    p.update(slot_unum=-1, slot_uden=-1)
    o = oracle.run(b, p)
    rows = bd_rows(o)
    ok = rows[rows[:, BD["n"]] >= 2]
    assert len(ok) > 0
    np.testing.assert_allclose(ok[:, BD["residual"]], 1.0, rtol=1e-12)


# ---------------------------------------------------------------------------
# DVFS integrals (D10)
# ---------------------------------------------------------------------------
def test_dvfs_bruteforce():
    rng = np.random.default_rng(5)
    for trial in range(20):
        tt = TinyTrace()
        ts = np.sort(rng.integers(0, 3000, int(rng.integers(1, 8))))
        fs = rng.integers(1300, 2100, len(ts))
        ps = rng.integers(100, 1000, len(ts))
        for t, f, p in zip(ts, fs, ps):
            tt.sample(0, int(t), int(f), int(p))
        t = -500
        kern = []
        for k in range(12):
            d = int(rng.integers(0, 400)); kern.append((t, t + d)); tt.ev(0, t, t, t + d); t += d + int(rng.integers(0, 100))
        o = run(tt)

        def fval(x, vals):
            k = np.searchsorted(ts, x, side="right") - 1
            return vals[max(k, 0)]
        for i, (s, e) in enumerate(kern):
            assert o["ev.phi"][i] == sum(int(fval(x, fs)) for x in range(s, e))
            assert o["ev.psi"][i] == sum(int(fval(x, ps)) for x in range(s, e))


def test_dvfs_constant_frequency():
    tt = TinyTrace().sample(0, 50, 1680, 700).ev(0, 0, 10, 1010).ev(0, 1, 2000, 2500)
    o = run(tt)
    np.testing.assert_array_equal(o["ev.phi"], [1680 * 1000, 1680 * 500])


# ---------------------------------------------------------------------------
# clock offsets (D13): pinned by construction in the generator
# ---------------------------------------------------------------------------
def test_clock_offsets_recovered():
    cfg = tracegen.config(2)
    cfg.n_iters = 2
    b = tracegen.generate(cfg)
    o = oracle.run(b)
    np.testing.assert_array_equal(o["gpu.delta"], b.delta)
    # arrival skew of unjittered collectives is the same true time on every GPU
    assert (o["skew.ag"] >= 0).all()


# ---------------------------------------------------------------------------
# pipeline fill
# ---------------------------------------------------------------------------
def test_pipeline_fill_scenario():
    tt = TinyTrace()
    t = 1000
    firsts = []
    for it in range(4):
        base_host = t + 5_000   # host dispatches the iteration's first kernel after the previous step ended
        tt.span(0, 0, base_host - 10, base_host + 1_000_000, it)
        host = base_host
        for k in range(10):
            ks = max(t + 500, host + 300)
            tt.ev(0, host, ks, ks + 1000)
            if k == 0:
                firsts.append(len(tt.events) - 1)
            t = ks + 1000
            host += 50
        t += 100
    b = tt.bundle()
    o = oracle.run(b, params(b))
    pos = (o["ev.prep"] > 0)
    expect = np.zeros(b.n_events, bool)
    expect[firsts[1:]] = True
    np.testing.assert_array_equal(pos, expect)


# ---------------------------------------------------------------------------
# invariants on generated traces
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def gen_small():
    cfg = tracegen.config(1)
    b1 = tracegen.generate(cfg)
    cfg2 = tracegen.config(3)
    cfg2.n_iters, cfg2.n_layers, cfg2.n_gpus, cfg2.opt_kernels, cfg2.warmup = 3, 4, 3, 600, 1
    b2 = tracegen.generate(cfg2)
    return [(b1, oracle.run(b1)), (b2, oracle.run(b2))]


def test_invariants_generated(gen_small):
    for b, o in gen_small:
        assert o["status"][0] == 0
        kind = b.meta & 0xFF
        dur = b.t_ke - b.t_ks
        comp = kind == COMPUTE
        assert (o["ev.ovl"] >= 0).all() and (o["ev.ovl"] <= dur).all()
        assert (o["ev.ovl"][~comp & ~np.isin(kind, [AG, RS, 3])] == 0).all()
        # sorted chain vs Python sorted()
        for g in range(b.cfg.n_gpus):
            idx = [i for i in range(b.n_events) if (b.meta[i] >> 24) == g and kind[i] == COMPUTE]
            srt = sorted(idx, key=lambda i: (b.t_ks[i], i))
            assert o["ev.pred"][srt[0]] == -1
            np.testing.assert_array_equal(o["ev.pred"][srt[1:]], srt[:-1])
        # telescoping: iteration wall = busy + prep + call on one compute stream (north_star)
        np.testing.assert_array_equal(o["iter.wall"], o["iter.busy"] + o["iter.prep"] + o["iter.call"])
        # children sum to parent at every level
        for child, parent, keys in (("inst", "layer", ("gpu", "it", "ph", "ly")), ("layer", "phase", ("gpu", "it", "ph")),
                                    ("phase", "iter", ("gpu", "it")), ("iter", "gpu", ("gpu",))):
            ck = list(zip(*[o[f"{child}.{k}"] for k in keys]))
            pk = list(zip(*[o[f"{parent}.{k}"] for k in keys]))
            for fld in ("n", "busy", "prep", "call", "ovl", "phi", "psi", "copy_ns", "ag_ns", "rs_ns", "n_events"):
                acc = {}
                for k, v in zip(ck, o[f"{child}.{fld}"]):
                    acc[k] = acc.get(k, 0) + int(v)
                assert [acc[k] for k in pk] == [int(v) for v in o[f"{parent}.{fld}"]]
        # instance partition: every annotated event in exactly one instance
        ai = o["ev.span_idx"].reshape(4, -1)
        assert o["inst.n_events"].sum() == (ai[0] >= 0).sum()
        assert o["inst.n"].sum() == ((ai[0] >= 0) & comp).sum()
        # counter multiset unchanged by alignment
        C = b.n_counters
        cm = o["ev.counters"].reshape(C, -1)
        for (g, names, slots, vals) in b.passes:
            sel = ((b.meta >> 24) == g) & (kind != MEMOP)
            for kk, sl in enumerate(slots):
                np.testing.assert_array_equal(np.sort(cm[sl][sel]), np.sort(vals[kk]))


def test_permutation_invariance(gen_small):
    """span order and event shuffle + dispatch re-sort leave every output unchanged."""
    b, o = gen_small[0]
    rng = np.random.default_rng(1)
    perm = rng.permutation(len(b.span_gl))
    inv = np.argsort(perm)
    b2 = tracegen.dataclasses.replace(b, span_gl=b.span_gl[perm], span_start=b.span_start[perm],
                                      span_end=b.span_end[perm], span_label=b.span_label[perm])
    o2 = oracle.run(b2)
    ai, ai2 = o["ev.span_idx"], o2["ev.span_idx"]
    np.testing.assert_array_equal(np.where(ai2 >= 0, perm[np.maximum(ai2, 0)], ai2), ai)
    for k in o:
        if k.endswith((".it", ".ph", ".ly", ".op")) or k == "ev.span_idx":
            continue
        np.testing.assert_array_equal(o[k], o2[k], err_msg=k)
    del inv
    # shuffle events, restore dispatch order with a stable (gpu, t_l) sort
    ep = rng.permutation(b.n_events)
    sh = tracegen.dataclasses.replace(b, t_l=b.t_l[ep], t_ks=b.t_ks[ep], t_ke=b.t_ke[ep], meta=b.meta[ep],
                                      name_id=b.name_id[ep])
    order = np.lexsort((sh.t_l, sh.meta >> 24))
    rs = tracegen.dataclasses.replace(sh, t_l=sh.t_l[order], t_ks=sh.t_ks[order], t_ke=sh.t_ke[order],
                                      meta=sh.meta[order], name_id=sh.name_id[order])
    o3 = oracle.run(rs)
    for k in o:
        np.testing.assert_array_equal(o[k], o3[k], err_msg=k)


def test_drop_counter_pass_degrades_breakdown_only(gen_small):
    b, o = gen_small[0]
    keep = [p for p in b.passes if not (p[0] == 0 and 0 in p[2])]
    b2 = tracegen.dataclasses.replace(b, passes=keep)
    o2 = oracle.run(b2)
    for k in ("ev.ovl", "ev.prep", "ev.call", "iter.busy", "glob.throughput", "inst.busy", "gpu.delta"):
        np.testing.assert_array_equal(o[k], o2[k], err_msg=k)
    assert o2["gpu.counter_present"].reshape(2, -1)[0, 0] == 0
    flags = bd_rows(o2)[:, BD["flags"]].astype(int)
    assert (flags & 32).any()     # missing GPU_CYCLES on GPU 0 -> rows flagged, Ovr_freq undefined


# ---------------------------------------------------------------------------
# validation
# ---------------------------------------------------------------------------
def test_validation_rules():
    def st(tt, keep_order=False):
        b = tt.bundle(keep_order=keep_order)
        return oracle.run(b, params(b))
    o = st(TinyTrace().ev(0, 0, 10, 5).ev(0, 1, 20, 30))
    assert o["val.count"][V_START_AFTER_END] == 1 and o["val.first"][V_START_AFTER_END] == 0
    assert o["status"][0] & ST_VALIDATION
    o = st(TinyTrace(n_gpus=2).ev(1, 0, 10, 15).ev(0, 1, 20, 30), keep_order=True)
    assert o["val.first"][V_GPU_NOT_GROUPED] == 1
    o = st(TinyTrace().ev(0, 5, 10, 15).ev(0, 1, 20, 30), keep_order=True)
    assert o["val.first"][V_DISPATCH_DECREASING] == 1
    o = st(TinyTrace().ev(0, 0, 10, 15).ev(0, 1, 20, 30, kind=9))
    assert o["val.first"][V_BAD_META] == 1
    o = st(TinyTrace().ev(0, 0, 10, 15).ev(0, 1, 2 ** 53, 2 ** 53 + 1))
    assert o["val.count"][V_TS_RANGE] == 1
    o = st(TinyTrace().ev(0, 0, 10, 15).span(0, 0, 10, 5))
    assert o["val.first"][V_SPAN_BAD] == 0
    o = st(TinyTrace().ev(0, 0, 10, 15).ev(0, 1, 12, 30))     # same-stream overlap: data, not fatal
    assert o["val.count"][V_STREAM_OVERLAP] == 1 and o["val.first"][V_STREAM_OVERLAP] == 1
    assert len(o["ev.prep"]) == 2
    o = st(TinyTrace().ev(0, 0, 10, 15))
    assert o["status"][0] == 0 and (o["val.count"] == 0).all()


# ---------------------------------------------------------------------------
# O14 report statistics: quantile and Pearson rows per label
# ---------------------------------------------------------------------------
REP = dict(n=0, dur=slice(1, 6), ratio=slice(6, 11), pearson=11, label=12, mean=13)


def report_rows(o):
    return o["report.rows"].reshape(-1, 16)


def test_report_aggregate_spec(golden):
    g = golden("report.json")["aggregate"]
    tt = _points_trace([(0, v) for v in g["values"]])
    o = oracle.run(tt.bundle(), params(tt.bundle()))
    assert report_rows(o)[0][REP["dur"]][2] == g["median"]


def test_report_quantiles_worked(golden):
    g = golden("report.json")["quantile"]
    tt = _points_trace([(0, v) for v in g["values"]])
    o = oracle.run(tt.bundle(), params(tt.bundle()))
    row = report_rows(o)[0]
    assert row[REP["n"]] == len(g["values"]) and row[REP["label"]] == 0
    np.testing.assert_allclose(row[REP["dur"]], g["expected"], rtol=1e-15)
    np.testing.assert_array_equal(row[REP["ratio"]], 0.0)


@pytest.mark.parametrize("case", ["linear", "anti", "constant"])
def test_report_pearson_worked(golden, case):
    g = golden("report.json")["pearson"][case]
    pts = [(int(round(r * d)), d) for r, d in zip(g["ratios"], g["durations"])]
    tt = _points_trace(pts)
    o = oracle.run(tt.bundle(), params(tt.bundle()))
    rho = report_rows(o)[0][REP["pearson"]]
    if g["rho"] is None:
        assert np.isnan(rho)
    else:
        assert rho == pytest.approx(g["rho"], abs=1e-15)


def test_report_matches_library_on_generated(gen_small):
    """per label: quantiles == numpy.quantile(linear), Pearson == numpy.corrcoef, over the sampled points of
    the oracle's (already pinned) point table; labels without points have n = 0 and NaN statistics."""
    for b, o in gen_small:
        p = oracle.default_params(b)
        rows = report_rows(o)
        lab, rank = o["point.label"], o["point.rank"]
        busy, ovl = o["point.busy"], o["point.ovl"]
        for L in range(len(b.labels)):
            m = (lab == L) & (rank >= p["warmup"]) & (busy > 0)
            row = rows[L]
            assert row[REP["n"]] == m.sum() and row[REP["label"]] == L
            if not m.any():
                assert np.isnan(row[REP["dur"]]).all()
                continue
            d = busy[m].astype(float)
            r = ovl[m] / busy[m]
            np.testing.assert_allclose(row[REP["dur"]], np.quantile(d, [0, .25, .5, .75, 1]), rtol=1e-12)
            np.testing.assert_allclose(row[REP["ratio"]], np.quantile(r, [0, .25, .5, .75, 1]), rtol=1e-12, atol=1e-15)
            if np.ptp(r) == 0 or np.ptp(d) == 0:
                assert np.isnan(row[REP["pearson"]])
            else:
                assert row[REP["pearson"]] == pytest.approx(np.corrcoef(r, d)[0, 1], rel=1e-9, abs=1e-12)
            assert row[REP["mean"]] == pytest.approx(d.mean(), rel=1e-12)


def cdf_rows(o):
    return o["cdf.rows"].reshape(-1, 5)


@pytest.mark.parametrize("case", ["three", "single"])
def test_cdf_spec(golden, case):
    g = golden("report.json")["cdf"]
    g = g if case == "three" else g["single"]
    # shuffle the iteration order: the CDF sorts by duration
    durs = list(reversed(g["durations"]))
    tt = _points_trace([(0, d) for d in durs])
    o = oracle.run(tt.bundle(), params(tt.bundle()))
    rows = cdf_rows(o)
    rows = rows[rows[:, 0] == 0]
    np.testing.assert_allclose(rows[:, 2], g["normalized"], rtol=1e-15)
    np.testing.assert_allclose(rows[:, 4], g["cdf"], rtol=1e-15)
    np.testing.assert_array_equal(rows[:, 3], 0.0)


def test_cdf_invariants_generated(gen_small):
    """per (label, gpu): CDF ends at 1 and increases by 1/n, durations start at 1 and never decrease,
    ratios in [0, 1]; the rows partition the O14 points of the label (same count)."""
    for b, o in gen_small:
        rows, rep = cdf_rows(o), report_rows(o)
        for L in range(len(b.labels)):
            sel = rows[rows[:, 0] == L]
            assert len(sel) == rep[L][REP["n"]]
            for g in np.unique(sel[:, 1]):
                s = sel[sel[:, 1] == g]
                n = len(s)
                np.testing.assert_allclose(s[:, 4], np.arange(1, n + 1) / n, rtol=1e-15)
                assert s[0, 2] == 1.0 and (np.diff(s[:, 2]) >= 0).all()
                assert ((s[:, 3] >= 0) & (s[:, 3] <= 1)).all()


def test_e2e_phase_optype_worked():
    """O16 (Fig. 4 stacked bars): one gpu, one iteration, two phases; hand-summed cells.
    P0: gemm op (kernels 100 + 50), fa op (70); P1: other op (30) + an unlabeled kernel (20, pseudo-op: vector).
    Launch (Eqs. 1-3): gaps 0 (first kernel: none), 0, 50 in P0; 598730 and 10 in P1."""
    tt = TinyTrace(labels=["g", "f", "v"])
    tt.span(0, 0, 0, 10 ** 6, 0).span(0, 1, 0, 500_000, 0).span(0, 1, 500_000, 10 ** 6, 1)
    tt.span(0, 3, 900, 1160, 0).span(0, 3, 1180, 1300, 1).span(0, 3, 599_000, 600_035, 2)
    for ks, ke in ((1000, 1100), (1100, 1150), (1200, 1270), (600_000, 600_030), (600_040, 600_060)):
        tt.ev(0, ks - 1, ks, ke)
    b = tt.bundle()
    o = oracle.run(b, params(b, op_type=np.array([1, 2, 0], np.int32), f_gemm=np.full(3, 1e9)))
    e = o["e2e.rows"]
    assert e[0] == 1
    cells = e[1:].reshape(8, 4)      # [phase][vec, gemm, fa, launch]
    np.testing.assert_array_equal(cells[0], [0, 150, 70, 50])
    np.testing.assert_array_equal(cells[1], [50, 0, 0, 598_730 + 10])
    np.testing.assert_array_equal(cells[2:], 0)


def test_e2e_partitions_iteration_generated(gen_small):
    """SPEC.md:491 invariant: the stacked segments partition the iteration (sum of vec / gemm / fa over phases
    = iteration busy) -- checked on the single-point case of each gpu / iteration: with one sampled point
    the medians are the point's own cells."""
    for b, o in gen_small:
        p = oracle.default_params(b)
        # restrict to one gpu and the last iteration: warmup = last rank, gpu mask = gpu 0
        last = int(o["iter.rank"][o["iter.gpu"] == 0].max())
        o1 = oracle.run(b, dict(p, warmup=last), gpu_mask=1)
        e = o1["e2e.rows"]
        assert e[0] == 1
        cells = e[1:].reshape(8, 4)
        row = (o1["iter.gpu"] == 0) & (o1["iter.rank"] == last)
        assert cells[:, :3].sum() == o1["iter.busy"][row][0]
        assert cells[:, 3].sum() == o1["iter.prep"][row][0] + o1["iter.call"][row][0]


# ---------------------------------------------------------------------------
# O17 CPU utilization
# ---------------------------------------------------------------------------
def _cpu(g):
    return oracle.cpu_util(g["ts"], g["core"], g["util"], g["topology"])


def test_cpu_util_spec(golden):
    g = golden("cpu_util.json")
    for case in ("spec_one_timestamp", "spec_all_zero"):
        r = _cpu(g[case])
        assert r["bad"] == 0
        np.testing.assert_array_equal(r["c_active"], g[case]["c_active"])
        np.testing.assert_allclose(r["c_min"], g[case]["c_min"], rtol=0, atol=1e-15)
    c = g["spec_one_of_eight_physical"]
    r = _cpu(c)
    assert r["summary"][5] == c["occupancy"]          # 1 of 8 physical cores ever active
    assert r["summary"][6] == c["smt"]                # two active siblings at one of the two timestamps
    np.testing.assert_array_equal(r["c_active"], c["c_active"])
    m = g["median_even"]
    r = _cpu(m)
    np.testing.assert_array_equal(r["c_active"], m["c_active"])
    np.testing.assert_allclose(r["c_min"], m["c_min"], rtol=1e-15)
    assert r["summary"][1] == m["median_c_active"]
    assert abs(r["summary"][2] - m["median_c_min"]) < 1e-15


def test_cpu_util_invariants_random():
    """C_min <= C_active <= N at every timestamp; relabelling physical cores or adding idle
    samples changes nothing; dropping a core's samples removes exactly its activity."""
    rng = np.random.default_rng(17)
    for _ in range(200):
        P, S = int(rng.integers(1, 9)), int(rng.integers(1, 3))
        N = P * S
        topo = (np.arange(N) % P).astype(np.int32)
        n_ts = int(rng.integers(1, 8))
        ts, core, util = [], [], []
        for t in range(n_ts):
            cs = np.sort(rng.choice(N, size=int(rng.integers(1, N + 1)), replace=False))
            for c in cs:
                ts.append(10 * t)
                core.append(int(c))
                util.append(float(rng.choice([0, 0, rng.integers(1, 101), rng.random() * 100])))
        ts, core, util = np.array(ts), np.array(core), np.array(util)
        r = oracle.cpu_util(ts, core, util, topo)
        assert r["bad"] == 0
        assert np.all(r["c_min"] <= r["c_active"] + 1e-12) and np.all(r["c_active"] <= N)
        perm = rng.permutation(P).astype(np.int32)
        r2 = oracle.cpu_util(ts, core, util, perm[topo])
        np.testing.assert_array_equal(r2["c_active"], r["c_active"])
        np.testing.assert_array_equal(r2["summary"], r["summary"])
        # occupancy from the definition: set of physical cores with any active logical core
        act = set(int(topo[c]) for c, u in zip(core, util) if u > 0)
        assert r["summary"][5] == len(act) / P


def test_cpu_util_rejects_unsorted_and_out_of_range():
    assert oracle.cpu_util([2, 1], [0, 0], [1, 1], [0])["bad"] == 1
    assert oracle.cpu_util([1, 1], [1, 0], [1, 1], [0, 0])["bad"] == 1
    assert oracle.cpu_util([1], [0], [101.0], [0])["bad"] == 1
    assert oracle.cpu_util([1], [3], [1.0], [0])["bad"] == 1


# ---------------------------------------------------------------------------
# derived-metric registry
# ---------------------------------------------------------------------------
def test_metric_spec(golden):
    g = golden("metrics.json")
    for k, c in g.items():
        if k.startswith("_"):
            continue
        if "error" in c:
            with pytest.raises(oracle.MetricError, match=r"MissingCounter\(Z\)"):
                oracle.metric_eval(c["expr"], c["names"], [[1.0]] * len(c["names"]), [1])
            continue
        v = oracle.metric_eval(c["expr"], c["names"], c["counters"], c["busy_ns"])
        want = np.array([np.nan if x is None else x for x in c["value"]])
        np.testing.assert_allclose(v, want, rtol=1e-15, equal_nan=True)


def _rand_expr(rng, names, depth=0):
    r = rng.random()
    if depth > 3 or r < 0.3:
        c = rng.integers(0, 3)
        if c == 0:
            return repr(float(rng.integers(1, 100)) / 8.0)
        return str(rng.choice(names))
    if r < 0.4:
        return "-" + _rand_expr(rng, names, depth + 1)
    if r < 0.5:
        return "(" + _rand_expr(rng, names, depth + 1) + ")"
    op = str(rng.choice(["+", "-", "*", "/"]))
    return _rand_expr(rng, names, depth + 1) + " " + op + " " + _rand_expr(rng, names, depth + 1)


def test_metric_random_vs_python_eval():
    """1,000 random expressions vs Python's own evaluator of the same infix text (IEEE doubles, the same
    precedence and left associativity)."""
    rng = np.random.default_rng(2512)
    names = ["A", "B", "C_x", "dur_s"]
    vals = {"A": 3.5, "B": -1.25, "C_x": 1e9, "dur_s": 2e-3}
    for _ in range(1000):
        e = _rand_expr(rng, names)
        got = oracle.metric_eval(e, ["A", "B", "C_x"], [[vals["A"]], [vals["B"]], [vals["C_x"]]], [2e6])[0]
        try:
            want = float(eval(e, {"__builtins__": {}}, dict(vals)))
        except ZeroDivisionError:
            want = float("nan")
        if np.isnan(want):
            assert np.isnan(got), e
        else:
            assert got == want or abs(got - want) <= 1e-12 * abs(want), (e, got, want)


# ---------------------------------------------------------------------------
# Chrome-trace ingest
# ---------------------------------------------------------------------------
def test_chrome_ingest_spec(golden):
    g = golden("chrome.json")
    for k, c in g.items():
        if k.startswith("_"):
            continue
        r = oracle.ingest_chrome(c["json"].encode())
        assert r["n_missing"] == c["n_missing"], k
        for f in ("t_l", "t_ks", "t_ke", "name_id", "span_gl", "span_start", "span_end", "span_label"):
            if f in c:
                np.testing.assert_array_equal(r[f], c[f], err_msg=f"{k}.{f}")
        if "kind" in c:
            np.testing.assert_array_equal(r["meta"] & 0xFF, c["kind"], err_msg=k)
        if "stream" in c:
            np.testing.assert_array_equal((r["meta"] >> 8) & 0xFFFF, c["stream"], err_msg=k)
        if "gpu" in c:
            np.testing.assert_array_equal(r["meta"] >> 24, c["gpu"], err_msg=k)


@pytest.mark.parametrize("cid", [1, 2])
def test_chrome_roundtrip(cid):
    """bundle -> Chrome trace -> ingest gives the bundle's columns back (name ids up to the first-appearance
    relabelling, spans as a multiset): the generator writes exact ns and sub-ns digits that round back."""
    b = tracegen.generate(tracegen.config(cid))
    r = oracle.ingest_chrome(tracegen.to_chrome(b, seed=cid))
    for f in ("t_l", "t_ks", "t_ke", "meta"):
        np.testing.assert_array_equal(r[f], getattr(b, f))
    m = {}
    assert all(m.setdefault(int(x), int(y)) == int(y) for x, y in zip(r["name_id"], b.name_id))
    assert len(set(m.values())) == len(m)
    key = lambda gl, s, e, lab: sorted(zip(gl.tolist(), s.tolist(), e.tolist(), lab.tolist()))
    assert key(r["span_gl"], r["span_start"], r["span_end"], r["span_label"]) == \
        key(b.span_gl, b.span_start, b.span_end, b.span_label)
    assert r["n_missing"] == 0
