"""Multi-rank path of the CUDA library on one GPU: P = 1/2/4/8 contexts, each driven by its own
host thread, exchange through the library's in-process loopback transport (chopper_loopback_allgather) in
place of ncclAllGather.  Rank r owns traced GPUs {g : g mod P = r} (north_star: one trace shard per rank).

Checks: every rank's chopper_global is bit-identical for every P and equal to the oracle run on the whole
trace (the offsets vectors and dense row blocks are re-indexed by gpu, not by rank, so P cannot change a
result); every rank's tables are the oracle's rows of its GPUs; the failure protocol (chopper.h) ends a step
on every rank -- none waits forever -- when one rank fails.
"""
import threading

import numpy as np
import pytest

import tracegen
from parity import FP_RTOL, _max_coll
from tinytrace import AG, COMPUTE, RS, TinyTrace, params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2512_08242_b200 as ch
    ch.build()


GLOB_KEYS = ("glob.step", "glob.complete", "glob.sampled", "glob.T", "glob.aligned_first", "glob.aligned_last",
             "glob.throughput", "glob.throughput_median", "bd.rows", "report.rows", "e2e.rows", "gpu.delta",
             "gpu.delta_flag", "skew.max_ag", "skew.max_rs")


def run_ranks(bundle, P, p, mi, kcoll, shard_hook=None, params_hook=None):
    """Run P loopback ranks in threads; returns (per-rank results or exceptions, shards)."""
    import torch
    import paper_2512_08242_b200 as ch
    group = ch.LoopbackGroup(P)
    G = bundle.cfg.n_gpus
    shards = [bundle.gpu_slice([g for g in range(G) if g % P == r]) for r in range(P)]
    if shard_hook:
        shards = [shard_hook(r, s) for r, s in enumerate(shards)]
    out = [None] * P

    def work(r):
        try:
            stream = torch.cuda.Stream(0)
            pipe = ch.Pipeline(G, len(bundle.labels), mi, kcoll, device=0, stream=stream, loopback=group, rank=r)
            pipe.upload(shards[r], bundle.n_counters)
            pr = params_hook(r, p) if params_hook else p
            res = pipe.run(pr, full=False)
            got = pipe.to_numpy(res, n_ratios=len(p["ratio_num"]))
            torch.cuda.synchronize()
            pipe.close()
            out[r] = got
        except Exception as e:       # noqa: BLE001 -- reported per rank
            out[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "a rank is still waiting (failure protocol broken)"
    group.close()
    return out, shards


def _glob_equal(a, b, what):
    for k in GLOB_KEYS:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.shape == y.shape, f"{what}: {k} shape {x.shape} vs {y.shape}"
        if x.dtype.kind == "f":
            np.testing.assert_array_equal(np.isnan(x), np.isnan(y), err_msg=f"{what}: {k} NaN pattern")
            np.testing.assert_array_equal(x[~np.isnan(x)], y[~np.isnan(y)], err_msg=f"{what}: {k}")
        else:
            np.testing.assert_array_equal(x, y, err_msg=f"{what}: {k}")


def _glob_vs_oracle(ref, got):
    for k in ("glob.step", "glob.complete", "glob.sampled", "glob.T", "glob.aligned_first", "glob.aligned_last",
              "gpu.delta"):
        np.testing.assert_array_equal(ref[k], got[k], err_msg=k)
    np.testing.assert_allclose(ref["glob.throughput"], got["glob.throughput"], rtol=1e-12, equal_nan=True)
    np.testing.assert_allclose(ref["glob.throughput_median"], got["glob.throughput_median"], rtol=1e-12,
                               equal_nan=True)
    np.testing.assert_allclose(ref["bd.rows"], got["bd.rows"], rtol=FP_RTOL, atol=0, equal_nan=True)
    np.testing.assert_allclose(ref["report.rows"], got["report.rows"], rtol=FP_RTOL, atol=1e-12, equal_nan=True)
    np.testing.assert_array_equal(ref["e2e.rows"], got["e2e.rows"])
    for cls, key in (("skew.ag", "skew.max_ag"), ("skew.rs", "skew.max_rs")):
        if ref[cls].size:
            assert int(ref[cls].max()) == int(got[key][0]), key


def _tables_vs_oracle(ref, got, full, shard):
    """the rank's table rows = the oracle's rows of the rank's gpus (span / event indices mapped to the shard)"""
    gset = sorted(set((shard.meta >> 24).astype(int).tolist()))
    em = np.isin((full.meta >> 24).astype(int), gset)
    sm = np.isin((full.span_gl >> 8).astype(int), gset)
    ev_map, sp_map = np.nonzero(em)[0], np.nonzero(sm)[0]
    for t in ("inst", "layer", "phase", "iter", "gpu", "point"):
        sel = np.isin(ref[f"{t}.gpu"], gset)
        assert int(sel.sum()) == len(got[f"{t}.gpu"]), f"{t}: row count"
        for f in ("gpu", "n_events", "n", "busy", "first_ks", "prep", "call", "ovl", "phi", "psi", "copy_ns", "ag_ns",
                  "rs_ns", "last_ke"):
            np.testing.assert_array_equal(ref[f"{t}.{f}"][sel], got[f"{t}.{f}"], err_msg=f"{t}.{f}")
        for f in ("it", "ph", "ly", "op"):
            g = got[f"{t}.{f}"]
            np.testing.assert_array_equal(ref[f"{t}.{f}"][sel], np.where(g >= 0, sp_map[np.maximum(g, 0)], g),
                                          err_msg=f"{t}.{f}")
        fi = got[f"{t}.first_idx"]
        ok = (fi >= 0) & (fi < len(ev_map))        # INT64_MAX: no COMPUTE event in the row
        np.testing.assert_array_equal(ref[f"{t}.first_idx"][sel], np.where(ok, ev_map[np.where(ok, fi, 0)], fi),
                                      err_msg=f"{t}.first_idx")


@pytest.fixture(scope="module")
def llama_small():
    import oracle
    cfg = tracegen.config(3)
    cfg.n_iters, cfg.n_layers, cfg.opt_kernels, cfg.warmup = 4, 4, 400, 1
    b = tracegen.generate(cfg)
    p = oracle.default_params(b)
    mi = cfg.n_iters + 2
    return b, p, mi, oracle.run(b, p, max_iters=mi)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_ranks_bit_identical_and_match_oracle(llama_small, P):
    b, p, mi, ref = llama_small
    kcoll = int(max(16, 4 * _max_coll(b)))
    out, shards = run_ranks(b, P, p, mi, kcoll)
    for r in range(P):
        assert not isinstance(out[r], Exception), f"rank {r}: {out[r]}"
    for r in range(P):
        _glob_vs_oracle(ref, out[r])
        _glob_equal(out[0], out[r], f"P={P} rank {r} vs rank 0")
        _tables_vs_oracle(ref, out[r], b, shards[r])
    # and against a single-rank run of the whole trace
    if P > 1:
        one, _ = run_ranks(b, 1, p, mi, kcoll)
        _glob_equal(one[0], out[0], f"P={P} vs P=1")


def _edge_bundle():
    """3 traced GPUs: GPU 1 has no events; GPU 2 lacks iteration step 1 (its span is missing)."""
    tt = TinyTrace(n_gpus=3, labels=["f_mlp_up", "f_attn_fa"], warmup=0)
    for g in (0, 2):
        t = 10_000 + 50 * g
        for it in range(3):
            if not (g == 2 and it == 1):
                tt.span(g, 0, t - 100, t + 90_000, 100 + it)
            tt.span(g, 3, t - 50, t + 40_000, 0).span(g, 3, t + 40_000, t + 80_000, 1)
            for k in range(12):
                ks = t + 6000 * k
                kind = AG if k == 3 else RS if k == 9 else COMPUTE
                tt.ev(g, ks - 30, ks, ks + 4000 + 100 * g, kind=kind, stream={AG: 1, RS: 2}.get(kind, 0))
            t += 100_000
    b = tt.bundle()
    return b


@pytest.mark.parametrize("P", [1, 2, 3])
def test_empty_gpu_and_missing_iteration(P):
    import oracle
    b = _edge_bundle()
    p = params(b, op_type=np.array([1, 2], np.int32))
    ref = oracle.run(b, p, max_iters=8)
    assert list(ref["glob.complete"]) == [1, 0, 1]
    out, shards = run_ranks(b, P, p, 8, 64)
    errs = [f"rank {r}: {o}" for r, o in enumerate(out) if isinstance(o, Exception)]
    assert not errs, errs
    for r in range(P):
        _glob_vs_oracle(ref, out[r])
        _glob_equal(out[0], out[r], f"P={P} rank {r}")
        _tables_vs_oracle(ref, out[r], b, shards[r])
    if P > 1:
        assert shards[1].n_events == 0       # the rank owning only GPU 1 has no events at all


def test_failure_on_one_rank_ends_the_step_everywhere(llama_small):
    """rank 1's shard violates t_ks <= t_ke (fatal, chopper_load_columns): rank 1 raises E_VALIDATION, rank 0
    E_STATE ('a peer rank failed') from chopper_align -- and nobody hangs."""
    import paper_2512_08242_b200 as ch
    b, p, mi, _ = llama_small
    kcoll = int(max(16, 4 * _max_coll(b)))

    def corrupt(r, s):
        if r != 1:
            return s
        ke = s.t_ke.copy()
        ke[5] = s.t_ks[5] - 1
        return tracegen.dataclasses.replace(s, t_ke=ke)
    out, _ = run_ranks(b, 2, p, mi, kcoll, shard_hook=corrupt)
    assert isinstance(out[1], ch.ChopperError) and out[1].status == 1, out[1]
    assert isinstance(out[0], ch.ChopperError) and out[0].status == 9 and "peer" in str(out[0]), out[0]


def test_breakdown_failure_on_one_rank_reaches_reduce(llama_small):
    """rank 1 passes an out-of-range counter slot to chopper_breakdown: rank 0 learns it in reduce_ranks."""
    import paper_2512_08242_b200 as ch
    b, p, mi, _ = llama_small
    kcoll = int(max(16, 4 * _max_coll(b)))

    def bad(r, q):
        return dict(q, slot_cycles=99) if r == 1 else q
    out, _ = run_ranks(b, 2, p, mi, kcoll, params_hook=bad)
    assert isinstance(out[1], ch.ChopperError) and out[1].status == 2, out[1]
    assert isinstance(out[0], ch.ChopperError) and out[0].status == 9 and "peer" in str(out[0]), out[0]
    # the contexts recover: a clean step afterwards succeeds on both ranks
    out, _ = run_ranks(b, 2, p, mi, kcoll)
    assert not any(isinstance(o, Exception) for o in out)
