"""Config 5 (BASELINE.json configs[4]): "synthetic stress: 1B events sharded across 8 GPUs with deep op/layer
nesting, for HBM-roofline scaling" -- the input recipe.

Like tracegen/__init__.py this draws inputs only (no method arithmetic).  Everything is vectorised per
iteration and counter-seeded per (config seed, iteration) -- plus (traced GPU) for the per-GPU draws -- so
any traced GPU's shard, and any prefix of its iterations, is generated on its own and is byte-identical to
the same rows of the full trace (the config-5 parity test compares a full-size shard with the oracle on a
prefix of it).

Shape of one iteration (per traced GPU, dense events: ~2 us kernels + ~1 us gaps on one compute stream):
  * phases forward / backward / optimizer;
  * forward and backward: 32 layers each, in nested layer groups of 4 (a layer-level span containing four
    layer spans); optimizer: no layers;
  * one op tree per layer (and one for the optimizer) over 16,384 kernels: op spans nested 7 deep with
    fan-out 4, 4, 4, 2, 2, 2, 2 (2,004 op spans per tree); a leaf covers the first 12 of its 16 kernels, so
    the last 4 fall to its parent op (the innermost-span rule, D4, produces an instance per internal op too);
    op labels cycle through the Fig. 1 vocabulary by (depth, position);
  * FSDP collectives on their own streams: an all-gather per layer prefetched one layer ahead (forward and
    backward), a reduce-scatter after every backward layer; they end at the same true time
    on every GPU, start (arrive) with a per-GPU jitter, and every GPU's clock is shifted by delta_g (D13);
  * the host dispatches 30 us ahead of the device (t_l = t_ks - 30 us); a collective is dispatched with the
    compute kernel it is issued next to.
Per traced GPU: 117 iterations x 1,065,056 events = 124.6M events, 15.25M spans; 8 GPUs: 997M events,
122M spans; C = 0 counters, no samples; timestamps span ~2^38.4 ns per GPU.
"""
from __future__ import annotations

import concurrent.futures as cf
from typing import List, Optional

import numpy as np

FAN = (4, 4, 4, 2, 2, 2, 2)          # op-tree fan-out per depth (depth 1..7)
TREE_EVENTS = 16384                  # kernels per op tree (= per layer)
LEAF_EVENTS = 16
LEAF_COVER = 12                      # kernels of a leaf inside its span; the rest fall to the parent op
LAYERS = 32
GROUP = 4
N_TREES = 2 * LAYERS + 1             # forward layers, backward layers, optimizer
DISPATCH_AHEAD_NS = 30_000
ITER_BUBBLE_NS = 200_000
PHASE_BUBBLE_NS = 50_000
GOLDEN = 0x9E3779B97F4A7C15


def _tree_template():
    """op tree nodes in pre-order: (depth 1..7, position within its depth, first kernel, end kernel)"""
    nodes = []

    def rec(depth, lo, hi, pos_at):
        if depth > len(FAN):
            return
        k = FAN[depth - 1]
        w = (hi - lo) // k
        for c in range(k):
            a, b = lo + c * w, lo + (c + 1) * w
            p = pos_at[depth]
            pos_at[depth] += 1
            nodes.append((depth, p, a, b))
            rec(depth + 1, a, b, pos_at)
    rec(1, 0, TREE_EVENTS, [0] * (len(FAN) + 2))
    a = np.array(nodes, dtype=np.int64)
    assert (a[a[:, 0] == len(FAN), 3] - a[a[:, 0] == len(FAN), 2] == LEAF_EVENTS).all()
    return a


_TREE = _tree_template()
SPANS_PER_TREE = len(_TREE)
COMM_PER_ITER = 2 * LAYERS + LAYERS         # AG per forward / backward layer, RS per backward layer
EVENTS_PER_ITER = N_TREES * TREE_EVENTS + COMM_PER_ITER
SPANS_PER_ITER = 1 + 3 + 2 * (LAYERS + LAYERS // GROUP) + N_TREES * SPANS_PER_TREE


def _rng(seed: int, n: int) -> np.ndarray:
    """n splitmix64 outputs of the counter stream `seed`"""
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _unif(seed: int, n: int) -> np.ndarray:
    return (_rng(seed, n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _iter_seed(cfg, it: int, g: Optional[int] = None) -> int:
    s = (cfg.seed * 0x100000001B3 + (it + 1) * GOLDEN) & 0xFFFFFFFFFFFFFFFF
    if g is not None:
        s ^= ((g + 1) * 0xD1B54A32D192ED03) & 0xFFFFFFFFFFFFFFFF
    return s


def deltas(cfg) -> np.ndarray:
    u = _unif(cfg.seed ^ 0xDE17A, cfg.n_gpus)
    d = np.floor(u * (2 * cfg.delta_max_ns + 1)).astype(np.int64) - cfg.delta_max_ns
    d[0] = 0
    return d


def _shared_iteration(cfg, it: int, t0: int):
    """the true-time schedule every GPU shares: compute starts, durations, collective windows"""
    n = N_TREES * TREE_EVENTS
    s = _iter_seed(cfg, it)
    u = _unif(s, 3 * n).reshape(3, n)
    dur = np.floor(2000.0 * np.exp(0.15 * np.sqrt(-2.0 * np.log1p(-u[0])) * np.cos(2.0 * np.pi * u[1])))
    dur = np.maximum(dur, 200.0).astype(np.int64)
    gap = np.floor(-1000.0 * np.log1p(-u[2])).astype(np.int64) + 100
    tree = np.arange(n) // TREE_EVENTS
    # phase bubbles before the first backward tree and before the optimizer tree
    gap[LAYERS * TREE_EVENTS - 1] += PHASE_BUBBLE_NS
    gap[2 * LAYERS * TREE_EVENTS - 1] += PHASE_BUBBLE_NS
    ks = t0 + np.concatenate([[0], np.cumsum(dur + gap)[:-1]])
    end = int(ks[-1] + dur[-1])
    return ks, dur, tree, end


def _gpu_iteration(cfg, it: int, g: int, ks, dur, delta_g: int):
    """one iteration of traced GPU g, device clock = true + delta_g; returns event columns in dispatch order
    and the iteration's spans"""
    n = ks.shape[0]
    ug = _unif(_iter_seed(cfg, it, g), n + 2 * COMM_PER_ITER)
    ke = ks + dur - np.floor(ug[:n] * 150.0).astype(np.int64)          # per-GPU speed variation
    tl = ks - DISPATCH_AHEAD_NS
    # collectives (true-time windows shared by all GPUs; arrival jitter per GPU)
    first = np.arange(N_TREES) * TREE_EVENTS
    last = first + TREE_EVENTS - 1
    fw, bw = np.arange(LAYERS), LAYERS + np.arange(LAYERS)
    # AG of layer l (forward l, backward l) issued with the first kernel of the previous layer's tree
    ag_tree = np.concatenate([fw, bw])
    ag_issue = np.maximum(first[ag_tree] - TREE_EVENTS, 0)
    ag_ks = ks[ag_issue] + 2000
    ag_ke = ag_ks + 300_000
    rs_issue = last[bw]
    rs_ks = ke[rs_issue] + 1000
    rs_ke = rs_ks + 500_000
    cks = np.concatenate([ag_ks, rs_ks])
    cke = np.concatenate([ag_ke, rs_ke])
    cks = cks + np.floor(ug[n:n + COMM_PER_ITER] * 20_000.0).astype(np.int64)   # arrival skew
    cks = np.minimum(cks, cke - 1000)
    ckind = np.concatenate([np.full(2 * LAYERS, 1), np.full(LAYERS, 2)]).astype(np.int64)
    # dispatch order: an AG right before its issuing kernel, an RS right after its kernel
    cpos = np.concatenate([ag_issue, rs_issue + 1])                    # insert before compute index cpos
    ctl = tl[np.minimum(cpos, n - 1)]
    ctl = np.where(cpos >= n, tl[-1], ctl)
    order = np.argsort(cpos, kind="stable")
    cpos, ctl, cks, cke, ckind = cpos[order], ctl[order], cks[order], cke[order], ckind[order]
    N = n + COMM_PER_ITER
    is_c = np.zeros(N, bool)
    cdst = cpos + np.arange(COMM_PER_ITER)
    is_c[cdst] = True
    T_l = np.empty(N, np.int64); T_ks = np.empty(N, np.int64); T_ke = np.empty(N, np.int64)
    kind = np.zeros(N, np.int64)
    T_l[~is_c], T_ks[~is_c], T_ke[~is_c] = tl, ks, ke
    T_l[cdst], T_ks[cdst], T_ke[cdst], kind[cdst] = ctl, cks, cke, ckind
    stream = np.where(kind == 1, 1, np.where(kind == 2, 2, 0))
    meta = ((g << 24) | (stream << 8) | kind).astype(np.uint32)
    name = np.zeros(N, np.int32)
    name[~is_c] = (np.arange(n) % 97).astype(np.int32)
    name[cdst] = np.where(ckind == 1, 1000, 1001).astype(np.int32)

    # spans on the dispatch timeline (compute kernels' t_l; collectives share their issuing kernel's t_l)
    lv, ss, se, lab = [], [], [], []

    def add(level, s, e, label):
        lv.append(np.full(np.shape(s), level, np.int64)); ss.append(np.asarray(s, np.int64))
        se.append(np.asarray(e, np.int64)); lab.append(np.asarray(label, np.int64) * np.ones(np.shape(s), np.int64))
    add(0, [tl[0] - 500], [tl[-1] + 500], [it])                        # iteration: label = step (D5)
    ph_first = np.array([0, LAYERS * TREE_EVENTS, 2 * LAYERS * TREE_EVENTS])
    ph_last = np.array([LAYERS * TREE_EVENTS, 2 * LAYERS * TREE_EVENTS, n]) - 1
    add(1, tl[ph_first] - 200, tl[ph_last] + 200, np.arange(3))
    lay = np.concatenate([fw, bw])
    add(2, tl[first[lay]] - 50, tl[last[lay]] + 50, lay % LAYERS)
    grp = np.concatenate([fw[::GROUP], bw[::GROUP]])
    add(2, tl[first[grp]] - 100, tl[last[grp + GROUP - 1]] + 100, 1000 + grp // GROUP)
    d, p, a, b = _TREE.T
    leaf = d == len(FAN)
    bend = np.where(leaf, a + LEAF_COVER, b) - 1
    nL = 42
    olab = (d * 5 + p) % nL
    for t in range(N_TREES):
        o = t * TREE_EVENTS
        add(3, tl[o + a] - 1, tl[o + bend] + 1, olab)
    span_lv = np.concatenate(lv)
    span = (np.concatenate(ss), np.concatenate(se), np.concatenate(lab), span_lv)
    return (T_l + delta_g, T_ks + delta_g, T_ke + delta_g, meta, name), span


def shard_sizes(cfg, n_iters: Optional[int] = None):
    I = cfg.n_iters if n_iters is None else n_iters
    return I * EVENTS_PER_ITER, I * SPANS_PER_ITER


def generate(cfg, gpus: Optional[List[int]] = None, n_iters: Optional[int] = None, threads: int = 8):
    """Bundle of the traced GPUs `gpus` (default all, ascending) over the first n_iters iterations."""
    import tracegen
    gpus = list(range(cfg.n_gpus)) if gpus is None else sorted(int(g) for g in gpus)
    I = cfg.n_iters if n_iters is None else int(n_iters)
    dl = deltas(cfg)
    ne, nsp = I * EVENTS_PER_ITER, I * SPANS_PER_ITER
    G = len(gpus)
    t_l = np.empty(G * ne, np.int64); t_ks = np.empty(G * ne, np.int64); t_ke = np.empty(G * ne, np.int64)
    meta = np.empty(G * ne, np.uint32); name = np.empty(G * ne, np.int32)
    s_gl = np.empty(G * nsp, np.uint32); s_s = np.empty(G * nsp, np.int64); s_e = np.empty(G * nsp, np.int64)
    s_lab = np.empty(G * nsp, np.int32)
    # iteration start times (true time) are shared: each iteration starts after the previous one ended (its
    # last reduce-scatter, 500 us, ends inside the 600 us after the last kernel) plus the bubble
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        lens = list(ex.map(lambda it: _shared_iteration(cfg, it, 0)[3] + 600_000 + ITER_BUBBLE_NS, range(I)))
    starts = [cfg.epoch_ns + int(x) for x in np.concatenate([[0], np.cumsum(lens)[:-1]])]

    def work(job):
        q, it = job
        g = gpus[q]
        ks, dur, _, _ = _shared_iteration(cfg, it, starts[it])
        (a, b, c, m, nm), (s0, s1, lab, lv) = _gpu_iteration(cfg, it, g, ks, dur, int(dl[g]))
        o = q * ne + it * EVENTS_PER_ITER
        t_l[o:o + EVENTS_PER_ITER] = a; t_ks[o:o + EVENTS_PER_ITER] = b; t_ke[o:o + EVENTS_PER_ITER] = c
        meta[o:o + EVENTS_PER_ITER] = m; name[o:o + EVENTS_PER_ITER] = nm
        so = q * nsp + it * SPANS_PER_ITER
        s_gl[so:so + SPANS_PER_ITER] = ((g << 8) | lv).astype(np.uint32)
        s_s[so:so + SPANS_PER_ITER] = s0 + dl[g]; s_e[so:so + SPANS_PER_ITER] = s1 + dl[g]
        s_lab[so:so + SPANS_PER_ITER] = lab.astype(np.int32)
    jobs = [(q, it) for q in range(G) for it in range(I)]
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, jobs))
    z32, z64 = np.zeros(0, np.int32), np.zeros(0, np.int64)
    return tracegen.Bundle(cfg=cfg, t_l=t_l, t_ks=t_ks, t_ke=t_ke, meta=meta, name_id=name, span_gl=s_gl,
                           span_start=s_s, span_end=s_e, span_label=s_lab, smp_gpu=z32, smp_ts=z64, smp_freq=z32,
                           smp_power=z32, passes=[], n_counters=0, labels=tracegen.label_vocabulary(), delta=dl,
                           freq_ratio=np.ones(cfg.n_gpus))
