"""Seeded synthetic trace generator (input recipe: DESIGN.md "Synthetic inputs").

This module is the ONLY code shared by the oracle side and the CUDA side: it
produces input columns and nothing else.  It contains none of the method's
arithmetic (no overlap, launch, attribution, aggregation or breakdown
computation) -- it only draws a Llama-3-8B-FSDP-shaped schedule
 with a splitmix64 counter generator
 and writes the columns the C ABI consumes.

Shape of a trace (per traced GPU, per iteration):
  * phases F, B, O (forward, backward, optimizer);
  * forward: f_ie, 32 layers of the Fig. 1 ops, f_ln, f_lp; backward mirrored
    with b_ prefixes; optimizer b_ga + opt_step with many small kernels
    (PAPER.md:616-618);
  * FSDP all-gather per layer prefetched one layer ahead on an AG stream,
    reduce-scatter per backward layer on an RS stream;
    collectives complete at the same true time on every GPU except a jittered
    minority, then every GPU's clock is shifted by delta_g;
  * FSDPv2 copy kernels serialized on the compute stream before f_attn_n,
    b_mlp_dp and b_ie, dispatched outside op spans;
  * per-kernel counters in serialized passes of 2-3;
  * 1 ms frequency / power samples.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

# kinds (include/chopper.h)
COMPUTE, AG, RS, COMM_OTHER, COPY, MEMOP, OTHER = range(7)

LAYER_OPS = ["attn_n", "qkv_ip", "qkv_s", "qkv_t", "qkv_re", "qkv_c", "attn_fa", "attn_or", "attn_op",
             "attn_ra", "mlp_n", "mlp_gp", "mlp_gs", "mlp_up", "mlp_gu", "mlp_dp", "mlp_ra"]
GEMM_OPS = {"qkv_ip", "attn_op", "mlp_gp", "mlp_up", "mlp_dp", "lp"}
FA_OPS = {"attn_fa"}
# forward kernels per op (x2 in backward); ~70 forward / ~150 backward per layer incl. copies
FWD_KERNELS = {"attn_n": 6, "qkv_ip": 2, "qkv_s": 3, "qkv_t": 4, "qkv_re": 8, "qkv_c": 3, "attn_fa": 2,
               "attn_or": 4, "attn_op": 2, "attn_ra": 3, "mlp_n": 6, "mlp_gp": 2, "mlp_gs": 4, "mlp_up": 2,
               "mlp_gu": 4, "mlp_dp": 2, "mlp_ra": 3}
# template kernel durations (ns) at b2s4; GEMMs ~60% of fwd+bwd busy time
FWD_DUR_NS = {"attn_n": 30_000, "qkv_ip": 380_000, "qkv_s": 8_000, "qkv_t": 12_000, "qkv_re": 15_000,
              "qkv_c": 20_000, "attn_fa": 420_000, "attn_or": 18_000, "attn_op": 260_000, "attn_ra": 25_000,
              "mlp_n": 30_000, "mlp_gp": 900_000, "mlp_gs": 40_000, "mlp_up": 900_000, "mlp_gu": 40_000,
              "mlp_dp": 900_000, "mlp_ra": 25_000}


def label_vocabulary(n_layers_unused: int = 0) -> List[str]:
    """Fig. 1 labels with f_/b_ prefixes plus b_ga and opt_step."""
    names = ["f_ie"] + ["f_" + o for o in LAYER_OPS] + ["f_ln", "f_lp"]
    names += ["b_lp", "b_ln"] + ["b_" + o for o in LAYER_OPS] + ["b_ie", "b_ga", "opt_step"]
    return names


def op_kind(label: str) -> int:
    """op_type code: 1 gemm, 2 fa, 0 other (vector, copy, optimizer)."""
    base = label[2:] if label[:2] in ("f_", "b_") else label
    if base in GEMM_OPS:
        return 1
    if base in FA_OPS:
        return 2
    return 0


# ---------------------------------------------------------------------------
# splitmix64 counter generator
# ---------------------------------------------------------------------------
class Rng:
    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self.ctr = 0

    def u64(self, n: int) -> np.ndarray:
        k = np.arange(self.ctr + 1, self.ctr + 1 + n, dtype=np.uint64)
        self.ctr += n
        with np.errstate(over="ignore"):
            z = self.state + k * GOLDEN
            z = (z ^ (z >> np.uint64(30))) * M1
            z = (z ^ (z >> np.uint64(27))) * M2
            z = z ^ (z >> np.uint64(31))
        return z

    def uniform(self, n) -> np.ndarray:
        shape = n if isinstance(n, tuple) else (n,)
        cnt = int(np.prod(shape))
        return ((self.u64(cnt) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)).reshape(shape)

    def normal(self, n) -> np.ndarray:
        shape = n if isinstance(n, tuple) else (n,)
        cnt = int(np.prod(shape))
        u1 = self.uniform(cnt)
        u2 = self.uniform(cnt)
        return (np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)).reshape(shape)

    def lognormal(self, n, sigma: float) -> np.ndarray:
        return np.exp(sigma * self.normal(n))

    def expo(self, n, mean: float) -> np.ndarray:
        return -mean * np.log1p(-self.uniform(n))

    def integers(self, n, lo: int, hi: int) -> np.ndarray:
        """uniform integers in [lo, hi)"""
        return lo + np.floor(self.uniform(n) * (hi - lo)).astype(np.int64)


# ---------------------------------------------------------------------------
# config
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class TraceConfig:
    config_id: int = 2
    seed: int = 0x5EED0002
    n_gpus: int = 8
    n_iters: int = 10
    n_layers: int = 32
    warmup: int = 0
    batch: int = 2
    seq: int = 4096
    kernel_scale: float = 1.0          # multiplies kernels per op (sizes N)
    opt_kernels: int = 5000            # optimizer kernels per iteration
    n_counters: int = 0                # C
    counters_per_pass: int = 3
    with_samples: bool = False
    freq_peak_mhz: int = 2100
    delta_max_ns: int = 50_000         # clock offsets U[-50, 50] us
    jitter_frac: float = 0.15          # fraction of collective ends jittered per GPU
    epoch_ns: int = 1_700_000_000_000_000_000
    memops_per_iter: int = 2


def config(cid: int, scale: float = 1.0) -> TraceConfig:
    """BASELINE.json configs[cid-1] (1-based ids as in SURVEY.md section 8(d))."""
    if cid == 1:   # toy: 2 GPUs x 1 iteration x 2 layers, ~5k events, 8 counters
        c = TraceConfig(config_id=1, seed=0x5EED0001, n_gpus=2, n_iters=1, n_layers=2, warmup=0,
                        kernel_scale=1.0, opt_kernels=2000, n_counters=8, with_samples=True)
    elif cid == 2:  # Llama 3 8B FSDP, 8 GPUs x 10 iterations (~1M events)
        c = TraceConfig(config_id=2, seed=0x5EED0002, n_gpus=8, n_iters=10, n_layers=32, warmup=3)
    elif cid == 3:  # + ~20 counters per kernel + 1 ms frequency / power samples
        c = TraceConfig(config_id=3, seed=0x5EED0003, n_gpus=8, n_iters=10, n_layers=32, warmup=3,
                        n_counters=20, with_samples=True)
    elif cid == 4:  # long run, 8 GPUs x 200 iterations (~20M events)
        c = TraceConfig(config_id=4, seed=0x5EED0004, n_gpus=8, n_iters=200, n_layers=32, warmup=10,
                        n_counters=8, with_samples=True)
    elif cid == 5:  # synthetic stress: 1B events over 8 GPUs, deep op / layer nesting (tracegen/stress.py)
        c = TraceConfig(config_id=5, seed=0x5EED0005, n_gpus=8, n_iters=117, n_layers=32, warmup=2)
    else:
        raise ValueError(f"unknown config {cid}")
    if scale != 1.0:
        c.n_iters = max(1, int(round(c.n_iters * scale)))
    return c


# counter slots (fixed vocabulary; first four feed the breakdown)
COUNTER_NAMES = ["GPU_CYCLES", "PERF_FLOPS", "UTIL_NUM", "UTIL_DEN", "BYTES_RD", "BYTES_WR", "AVG_POWER_W",
                 "OCCUPANCY"] + [f"AUX_{i}" for i in range(12)]


@dataclasses.dataclass
class Bundle:
    cfg: TraceConfig
    # events
    t_l: np.ndarray
    t_ks: np.ndarray
    t_ke: np.ndarray
    meta: np.ndarray
    name_id: np.ndarray
    # spans
    span_gl: np.ndarray
    span_start: np.ndarray
    span_end: np.ndarray
    span_label: np.ndarray
    # samples
    smp_gpu: np.ndarray
    smp_ts: np.ndarray
    smp_freq: np.ndarray
    smp_power: np.ndarray
    # counter passes: list of (gpu, name_id[n], slots[k], values[k, n])
    passes: List[tuple]
    n_counters: int
    labels: List[str]
    delta: np.ndarray            # injected clock offsets (ground truth for O4)
    freq_ratio: np.ndarray       # per-GPU freq ratio used for samples

    @property
    def n_events(self) -> int:
        return int(self.t_l.shape[0])

    def gpu_slice(self, gpus) -> "Bundle":
        """events / spans / samples / passes of a subset of traced GPUs (rank shard)."""
        gset = set(int(g) for g in gpus)
        eg = (self.meta >> 24).astype(np.int64)
        em = np.isin(eg, list(gset))
        sg = (self.span_gl >> 8).astype(np.int64)
        sm = np.isin(sg, list(gset))
        pm = np.isin(self.smp_gpu, list(gset))
        return dataclasses.replace(
            self, t_l=self.t_l[em], t_ks=self.t_ks[em], t_ke=self.t_ke[em], meta=self.meta[em],
            name_id=self.name_id[em], span_gl=self.span_gl[sm], span_start=self.span_start[sm],
            span_end=self.span_end[sm], span_label=self.span_label[sm], smp_gpu=self.smp_gpu[pm],
            smp_ts=self.smp_ts[pm], smp_freq=self.smp_freq[pm], smp_power=self.smp_power[pm],
            passes=[p for p in self.passes if p[0] in gset])


    def prefix(self, n: int) -> "Bundle":
        """The first n events of a single-gpu bundle (dispatch order) with the spans that start before the
        last kept dispatch, the samples up to it and each counter pass cut to the kept non-MEMOP events:
        a bounded sample of the same workload (the CPU baseline's sample)."""
        n = min(int(n), self.n_events)
        if n == self.n_events:
            return self
        t_cut = int(self.t_l[n - 1])
        sm = self.span_start <= t_cut
        pm = self.smp_ts <= t_cut
        m = int(np.count_nonzero((self.meta[:n] & 0xFF) != MEMOP))
        return dataclasses.replace(
            self, t_l=self.t_l[:n], t_ks=self.t_ks[:n], t_ke=self.t_ke[:n], meta=self.meta[:n],
            name_id=self.name_id[:n], span_gl=self.span_gl[sm], span_start=self.span_start[sm],
            span_end=self.span_end[sm], span_label=self.span_label[sm], smp_gpu=self.smp_gpu[pm],
            smp_ts=self.smp_ts[pm], smp_freq=self.smp_freq[pm], smp_power=self.smp_power[pm],
            passes=[(g, nm[:m], sl, vals[:, :m]) for (g, nm, sl, vals) in self.passes])


def _meta(gpu: int, stream: int, kind: int) -> np.uint32:
    return np.uint32((gpu << 24) | (stream << 8) | kind)


# ---------------------------------------------------------------------------
# program: the per-iteration op sequence (identical on every GPU)
# ---------------------------------------------------------------------------
def _program(cfg: TraceConfig, labels: List[str]):
    """List of segments; each segment is a list of ops (label id, n kernels, template dur ns,
    layer or -1, phase) plus the collective plan attached to the segment."""
    lid = {n: i for i, n in enumerate(labels)}
    ks = cfg.kernel_scale
    scale_bs = (cfg.batch * cfg.seq) / (2 * 4096.0)

    def nk(n):
        return max(1, int(round(n * ks)))

    def dur(op, bwd):
        d = FWD_DUR_NS[op] * (2.0 if bwd else 1.0)
        if op == "attn_fa":
            d *= scale_bs * (cfg.seq / 4096.0) * (2.5 / 2.0 if bwd else 1.0)
        elif op in GEMM_OPS:
            d *= scale_bs
        return d

    segs = []
    # forward
    segs.append(dict(phase=0, layer=-1, ops=[(lid["f_ie"], nk(3), 20_000.0)], ag=True, rs=False, copy_before=False))
    for l in range(cfg.n_layers):
        ops = [(lid["f_" + o], nk(FWD_KERNELS[o]), dur(o, False) / nk(FWD_KERNELS[o])) for o in LAYER_OPS]
        segs.append(dict(phase=0, layer=l, ops=ops, ag=True, rs=False, copy_before=True))
    segs.append(dict(phase=0, layer=-1, ops=[(lid["f_ln"], nk(4), 30_000.0), (lid["f_lp"], nk(2), 1_500_000.0 * scale_bs)],
                     ag=False, rs=False, copy_before=False))
    # backward (mirror)
    segs.append(dict(phase=1, layer=-1, ops=[(lid["b_lp"], nk(4), 1_500_000.0 * scale_bs), (lid["b_ln"], nk(6), 30_000.0)],
                     ag=True, rs=False, copy_before=False))
    for l in reversed(range(cfg.n_layers)):
        ops = [(lid["b_" + o], nk(2 * FWD_KERNELS[o]), dur(o, True) / nk(2 * FWD_KERNELS[o]))
               for o in reversed(LAYER_OPS)]
        segs.append(dict(phase=1, layer=l, ops=ops, ag=True, rs=True, copy_before=True))
    segs.append(dict(phase=1, layer=-1, ops=[(lid["b_ie"], nk(4), 25_000.0)], ag=False, rs=True, copy_before=True))
    # optimizer
    segs.append(dict(phase=2, layer=-1, ops=[(lid["b_ga"], nk(max(1, cfg.opt_kernels // 5)), 6_000.0),
                                             (lid["opt_step"], nk(cfg.opt_kernels - cfg.opt_kernels // 5), 8_000.0)],
                     ag=False, rs=False, copy_before=False))
    return segs


# ---------------------------------------------------------------------------
# generator
# ---------------------------------------------------------------------------
def generate(cfg: TraceConfig) -> Bundle:
    if cfg.config_id == 5:
        from . import stress
        return stress.generate(cfg)
    labels = label_vocabulary()
    segs = _program(cfg, labels)
    G = cfg.n_gpus
    R = Rng(cfg.seed)                                  # collective plan, clock offsets
    Kr = Rng(cfg.seed ^ 0xA5A5A5A55A5A5A5A)            # kernel-level draws, shape [G, k]
    Rg = [Rng(cfg.seed ^ ((g + 1) * 0x9E3779B97F4A7C15 & 0xFFFFFFFFFFFFFFFF)) for g in range(G)]

    delta = R.integers(G, -cfg.delta_max_ns, cfg.delta_max_ns + 1).astype(np.int64)
    if G > 0:
        delta[0] = 0
    freq_ratio = np.clip(0.70 + 0.25 * R.uniform(G), 0.62, 1.0)

    # per-segment static layout (identical on every GPU)
    pre = []
    for sg in segs:
        ns = np.array([n for (_, n, _) in sg["ops"]], dtype=np.int64)
        labs = np.repeat(np.array([l for (l, _, _) in sg["ops"]], dtype=np.int32), ns)
        dt = np.repeat(np.array([d for (_, _, d) in sg["ops"]], dtype=np.float64), ns)
        opi = np.repeat(np.arange(len(ns)), ns)
        first = np.concatenate([[0], np.cumsum(ns)[:-1]])
        last = np.cumsum(ns) - 1
        within = np.arange(int(ns.sum())) - np.repeat(first, ns)
        pre.append(dict(labs=labs, dt=dt, ramp=100.0 * np.arange(int(ns.sum())) + 200.0 * opi, first=first,
                        last=last, names=(labs.astype(np.int64) * 64 + (within % 8)).astype(np.int32),
                        oplabs=np.array([l for (l, _, _) in sg["ops"]], dtype=np.int32)))

    chunks = []     # (kind, stream, tl[G,k], ks[G,k], ke[G,k], name[k] or scalar, lab[k] or scalar)
    spans = []      # (level, s[G,k], e[G,k], label[k])

    t_host = np.zeros(G)
    t_cmp = np.zeros(G)
    t_ag = np.zeros(G)
    t_rs = np.zeros(G)
    step0 = 100

    def collective(kind, stream, arr, dur, tl):
        E = arr.max() + dur
        jit = R.uniform(G) < cfg.jitter_frac
        Eg = E + np.where(jit, R.integers(G, 1, 5_001).astype(np.float64), 0.0)
        chunks.append((kind, stream, tl[:, None], arr[:, None], Eg[:, None], 1000 if kind == AG else 1001, -1))
        return Eg

    def shift(d):
        return np.concatenate([np.zeros((d.shape[0], 1)), d[:, :-1]], axis=1)

    for it in range(cfg.n_iters):
        it_start = t_host.copy()
        phase_start = t_host.copy()
        cur_phase = 0
        # the iteration's first all-gather is issued at iteration start: pipeline fill
        arr = np.maximum(t_host + 5_000.0, t_ag)
        t_ag = collective(AG, 1, arr, 400_000.0 + 300_000.0 * R.uniform(1)[0], t_host + 1_000.0)
        t_host = t_host + 2_000.0
        pending_ag = t_ag.copy()
        for si, sg in enumerate(segs):
            P = pre[si]
            if sg["phase"] != cur_phase:
                spans.append((1, phase_start[:, None], t_host[:, None], np.array([cur_phase], dtype=np.int32)))
                phase_start = t_host.copy()
                cur_phase = sg["phase"]
            wait_ag = pending_ag if (sg["ag"] or si == 0) else None
            pending_ag = None
            if si + 1 < len(segs) and segs[si + 1]["ag"]:
                # prefetch the next layer's all-gather at this segment's start
                arr = np.maximum(t_host + 3_000.0, t_ag)
                t_ag = collective(AG, 1, arr, 250_000.0 + 500_000.0 * R.uniform(1)[0], t_host + 500.0)
                pending_ag = t_ag.copy()
                t_host = t_host + 1_000.0
            layer_start = t_host.copy()
            tc = t_cmp.copy()
            if wait_ag is not None:
                tc = np.maximum(tc, wait_ag)
            th = t_host.copy()
            if sg["copy_before"]:
                # FSDPv2 copy kernels serialized on the compute stream, outside op spans
                d = 15_000.0 * Kr.lognormal((G, 2), 0.15)
                gap = 1_000.0 + Kr.expo((G, 2), 2_000.0)
                ks = tc[:, None] + np.cumsum(gap + shift(d), axis=1)
                ke = ks + d
                tl = th[:, None] + 200.0 * np.arange(1, 3)[None, :]
                chunks.append((COPY, 0, tl, ks, ke, 1002, -1))
                th = tl[:, -1] + 300.0
                tc = ke[:, -1]
            K = P["dt"].shape[0]
            d = np.maximum(P["dt"][None, :] * Kr.lognormal((G, K), 0.15), 1_000.0)
            gap = Kr.expo((G, K), 3_000.0) + 500.0
            ks = tc[:, None] + np.cumsum(gap + shift(d), axis=1)
            ke = ks + d
            lead = 10_000.0 + 490_000.0 * Kr.uniform((G, K))      # host runs ahead 10-500 us
            tl = np.maximum(np.minimum(ks - lead, ks - 2_000.0), th[:, None] + 100.0)
            ramp = P["ramp"][None, :]
            tl = np.maximum.accumulate(tl - ramp, axis=1) + ramp
            sk = Kr.uniform((G, K)) < 0.01                          # host/device skew: dispatch after start (D6)
            tl = np.where(sk, np.maximum(tl, ks + 50.0), tl)
            tl = np.maximum.accumulate(tl - ramp, axis=1) + ramp
            chunks.append((COMPUTE, 0, tl, ks, ke, P["names"], P["labs"]))
            spans.append((3, tl[:, P["first"]] - 50.0, tl[:, P["last"]] + 50.0, P["oplabs"]))
            t_host = tl[:, -1] + 200.0
            t_cmp = ke[:, -1]
            if sg["layer"] >= 0:
                spans.append((2, layer_start[:, None], t_host[:, None] + 100.0, np.array([sg["layer"]], dtype=np.int32)))
            t_host = t_host + 300.0
            if sg["rs"]:
                arr = np.maximum(np.maximum(t_host, t_cmp) + 2_000.0, t_rs)
                t_rs = collective(RS, 2, arr, 250_000.0 + 400_000.0 * R.uniform(1)[0], t_host + 100.0)
                t_host = t_host + 400.0
            if sg["phase"] == 2 or (si + 1 < len(segs) and segs[si + 1]["phase"] == 2):
                t_cmp = np.maximum(t_cmp, t_rs)                      # optimizer waits for every reduce-scatter
        n = cfg.memops_per_iter
        if n:
            # DMA memops on their own stream at iteration end, outside op spans
            tl = t_host[:, None] + 300.0 * np.arange(1, n + 1)[None, :]
            ks = tl + 5_000.0
            ke = ks + 20_000.0 * Kr.lognormal((G, n), 0.1)
            chunks.append((MEMOP, 3, tl, ks, ke, 1003, -1))
        t_host = t_host + 300.0 * (n + 1)
        spans.append((1, phase_start[:, None], t_host[:, None], np.array([cur_phase], dtype=np.int32)))
        spans.append((0, it_start[:, None], t_host[:, None], np.array([step0 + it], dtype=np.int32)))
        # host waits for the step before the next iteration
        t_host = np.maximum(t_host, np.maximum(t_cmp, np.maximum(t_ag, t_rs))) + 20_000.0

    ev = []
    sp = []
    for g in range(G):
        e = dict(tl=[], ks=[], ke=[], meta=[], name=[], lab=[])
        for (kind, stream, tl, ks, ke, name, lab) in chunks:
            k = tl.shape[1]
            e["tl"].append(tl[g]); e["ks"].append(ks[g]); e["ke"].append(ke[g])
            e["meta"].append(np.full(k, _meta(g, stream, kind), dtype=np.uint32))
            e["name"].append(np.broadcast_to(np.asarray(name, dtype=np.int32), (k,)))
            e["lab"].append(np.broadcast_to(np.asarray(lab, dtype=np.int32), (k,)))
        ev.append(e)
        s = dict(gl=[], s=[], e=[], lab=[])
        for (level, ss, se, lab) in spans:
            k = ss.shape[1]
            s["gl"].append(np.full(k, (g << 8) | level, dtype=np.uint32))
            s["s"].append(ss[g]); s["e"].append(se[g]); s["lab"].append(lab)
        sp.append(s)
    return _finish(cfg, labels, ev, sp, delta, freq_ratio, Rg, R)


def _finish(cfg, labels, ev, sp, delta, freq_ratio, Rg, R) -> Bundle:
    G = cfg.n_gpus
    T_l, T_ks, T_ke, META, NAME, LAB = [], [], [], [], [], []
    for g in range(G):
        tl = np.concatenate(ev[g]["tl"])
        ks = np.concatenate(ev[g]["ks"])
        ke = np.concatenate(ev[g]["ke"])
        meta = np.concatenate(ev[g]["meta"])
        name = np.concatenate(ev[g]["name"])
        lab = np.concatenate(ev[g]["lab"])
        # integer ns, dispatch order = strictly increasing t_l
        tl = np.round(tl).astype(np.int64)
        ks = np.round(ks).astype(np.int64)
        ke = np.round(ke).astype(np.int64)
        ke = np.maximum(ke, ks + 1)
        order = np.argsort(tl, kind="stable")
        tl, ks, ke, meta, name, lab = tl[order], ks[order], ke[order], meta[order], name[order], lab[order]
        tl = np.maximum.accumulate(tl - np.arange(len(tl))) + np.arange(len(tl))
        off = cfg.epoch_ns + int(delta[g])
        T_l.append(tl + off); T_ks.append(ks + off); T_ke.append(ke + off)
        META.append(meta); NAME.append(name); LAB.append(lab)
    t_l = np.concatenate(T_l); t_ks = np.concatenate(T_ks); t_ke = np.concatenate(T_ke)
    meta = np.concatenate(META); name_id = np.concatenate(NAME); lab = np.concatenate(LAB)

    # spans (host timeline of each GPU, same clock shift)
    gl, ss, se, sl = [], [], [], []
    for g in range(G):
        off = cfg.epoch_ns + int(delta[g])
        gl.append(np.concatenate(sp[g]["gl"]))
        ss.append(np.round(np.concatenate(sp[g]["s"])).astype(np.int64) + off)
        se.append(np.round(np.concatenate(sp[g]["e"])).astype(np.int64) + off)
        sl.append(np.concatenate(sp[g]["lab"]).astype(np.int32))
    span_gl = np.concatenate(gl); span_start = np.concatenate(ss); span_end = np.concatenate(se)
    span_label = np.concatenate(sl)
    # deliver spans in a shuffled order (the ABI accepts any order)
    perm = np.argsort(R.u64(len(span_gl)), kind="stable")
    span_gl, span_start, span_end, span_label = span_gl[perm], span_start[perm], span_end[perm], span_label[perm]

    # samples
    smp_gpu, smp_ts, smp_f, smp_p = [], [], [], []
    if cfg.with_samples:
        for g in range(G):
            m = (meta >> 24) == g
            lo, hi = int(t_ks[m].min()) - 1_000_000, int(t_ke[m].max()) + 1_000_000
            n = (hi - lo) // 1_000_000 + 1
            ts = lo + 1_000_000 * np.arange(n, dtype=np.int64) + Rg[g].integers(n, -20_000, 20_001)
            f = np.clip(np.round(freq_ratio[g] * cfg.freq_peak_mhz * (1.0 + 0.03 * Rg[g].normal(n))), 1300, 2100)
            p = np.round(700_000 + 250_000 * Rg[g].uniform(n))
            smp_gpu.append(np.full(n, g, dtype=np.int32)); smp_ts.append(ts)
            smp_f.append(f.astype(np.int32)); smp_p.append(p.astype(np.int32))
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dtype=dt))
    smp_gpu, smp_ts, smp_f, smp_p = cat(smp_gpu, np.int32), cat(smp_ts, np.int64), cat(smp_f, np.int32), cat(smp_p, np.int32)

    # counters: passes of counters_per_pass slots over the non-MEMOP kernels of each GPU
    passes = []
    C = cfg.n_counters
    if C > 0:
        kinds = (meta & 0xFF).astype(np.int64)
        for g in range(G):
            m = ((meta >> 24) == g) & (kinds != MEMOP)
            dur = (t_ke[m] - t_ks[m]).astype(np.float64)
            lab_g = lab[m]
            nm = name_id[m]
            n = int(m.sum())
            rg = Rg[g]
            f_mhz = float(int(round(freq_ratio[g] * cfg.freq_peak_mhz)))
            cyc = np.round(dur * f_mhz / 1000.0)                            # integer-valued
            rate = np.where(lab_g >= 0, 2.0e5 + 1.0e4 * (lab_g % 17), 0.0)  # flops per cycle per label
            flops = np.round(cyc * rate)
            util_den = cyc
            util_num = np.round(cyc * np.where(lab_g >= 0, 0.35 + 0.01 * (lab_g % 23), 0.1))
            vals = [cyc, flops, util_num, util_den,
                    np.round(dur * 3.2e3 * rg.uniform(n)), np.round(dur * 1.1e3 * rg.uniform(n)),
                    600.0 + 300.0 * rg.uniform(n), rg.uniform(n)]
            while len(vals) < C:
                vals.append(np.round(1e3 * rg.uniform(n)))
            vals = vals[:C]
            k = cfg.counters_per_pass
            for p0 in range(0, C, k):
                slots = np.arange(p0, min(C, p0 + k), dtype=np.int32)
                passes.append((g, nm.copy(), slots, np.stack([vals[s] for s in slots]).astype(np.float64)))
    return Bundle(cfg=cfg, t_l=t_l, t_ks=t_ks, t_ke=t_ke, meta=meta, name_id=name_id,
                  span_gl=span_gl, span_start=span_start, span_end=span_end, span_label=span_label,
                  smp_gpu=smp_gpu, smp_ts=smp_ts, smp_freq=smp_f, smp_power=smp_p, passes=passes,
                  n_counters=C, labels=labels, delta=delta, freq_ratio=freq_ratio)


def workload_shapes(cfg: TraceConfig) -> Dict[str, int]:
    """Workload spec (Table 2; vocab / head_dim are assumptions, D19)."""
    return dict(b=cfg.batch, s=cfg.seq, layers=cfg.n_layers, hidden=4096, ffn=14336, heads=32, kv_heads=8,
                head_dim=128, vocab=128256)


# ---------------------------------------------------------------------------
# host CPU utilization samples (Fig. 9)
# ---------------------------------------------------------------------------
def cpu_samples(seed: int, t_start: int, t_end: int, period_ns: int = 100_000_000, n_physical: int = 64, smt: int = 2,
                n_workers: int = 32, p_active: float = 0.85, p_sibling: float = 0.05):
    """Every logical core sampled every `period_ns` over [t_start, t_end): a fixed set of `n_workers` worker
    threads (per-rank main / data-loader / communication threads) pinned to distinct physical cores, each
    active with probability p_active at a sample with an integer utilisation in [5, 60] %, its SMT sibling
    rarely (p_sibling) active too; every other core idle (util 0).  Linux-style topology: logical core i
    belongs to physical core i % n_physical.  Returns (ts, core, util, topology), sorted by (ts, core).
    Contains none of the method's arithmetic."""
    rng = Rng(seed ^ 0xC0FFEE)
    n_logical = n_physical * smt
    topology = (np.arange(n_logical) % n_physical).astype(np.int32)
    workers = np.sort(rng.integers(n_workers, 0, 1 << 30) % n_physical)
    workers = np.unique(np.concatenate([workers, np.arange(n_physical)]))[:n_workers]   # distinct physical cores
    n_ts = max(1, int((t_end - t_start) // period_ns))
    ts = np.repeat(t_start + period_ns * np.arange(n_ts, dtype=np.int64), n_logical)
    core = np.tile(np.arange(n_logical, dtype=np.int32), n_ts)
    util = np.zeros((n_ts, n_logical), dtype=np.float64)
    act = rng.uniform((n_ts, len(workers))) < p_active
    util[:, workers] = np.where(act, rng.integers(n_ts * len(workers), 5, 61).reshape(n_ts, len(workers)), 0)
    sib = rng.uniform((n_ts, len(workers))) < p_sibling
    util[:, workers + n_physical] = np.where(sib, rng.integers(n_ts * len(workers), 5, 31).reshape(n_ts, len(workers)),
                                             0)
    return ts, core, util.reshape(-1), topology


# ---------------------------------------------------------------------------
# Chrome-trace export of a bundle (input of the device ingest)
# ---------------------------------------------------------------------------
_CHROME_KIND = {COMPUTE: ("kernel", "k{}"), AG: ("kernel", "ncclDevKernel_AllGather_k{}"),
                RS: ("kernel", "ncclDevKernel_ReduceScatter_k{}"), COMM_OTHER: ("kernel", "ncclDevKernel_AllReduce_k{}"),
                COPY: ("kernel", "fsdp_copy_k{}"), MEMOP: ("gpu_memset", "Memset_k{}"), OTHER: ("gpu_user", "other_k{}")}


def _us(ns: int, extra: str = "") -> str:
    """integer ns as a decimal microsecond string with exactly three fractional digits (+ optional digits)"""
    s = "-" if ns < 0 else ""
    a = abs(int(ns))
    return f"{s}{a // 1000}.{a % 1000:03d}{extra}"


def to_chrome(b: "Bundle", seed: int = 1) -> bytes:
    """The bundle's kernels (X events, cat / name by kind, pid = gpu, tid = stream, args.correlation), their
    host launches as flow-start events (ph 's', id = correlation, ts = dispatch) and the spans as
    user_annotation X events (args.level, args.label), flows and spans interleaved at random between the
    kernels (kernels keep the bundle order).  Some timestamps carry extra sub-ns digits that round back to the
    same ns (half-to-even never changes them).  Formatting only: none of the method's arithmetic."""
    rng = Rng(seed ^ 0xC4120E)
    n = b.n_events
    kind = (b.meta & 0xFF).astype(np.int64)
    gpu = (b.meta >> 24).astype(np.int64)
    stream = ((b.meta >> 8) & 0xFFFF).astype(np.int64)
    extra = rng.integers(n, 0, 4)
    out = []
    for i in range(n):
        cat, nm = _CHROME_KIND[int(kind[i])]
        ex = ["", "0", "4", "49"][int(extra[i])]
        out.append((0, i, '{"ph": "X", "cat": "%s", "name": "%s", "pid": %d, "tid": %d, "ts": %s, "dur": %s, '
                    '"args": {"correlation": %d, "device": %d, "stream": %d}}'
                    % (cat, nm.format(int(b.name_id[i])), gpu[i], stream[i], _us(int(b.t_ks[i]), ex),
                       _us(int(b.t_ke[i] - b.t_ks[i])), i + 1, gpu[i], stream[i])))
    pos_f = rng.uniform(n)
    for i in range(n):
        out.append((1, i + pos_f[i], '{"ph": "s", "id": %d, "pid": %d, "tid": 1, "ts": %s, "cat": "ac2g", '
                    '"name": "ac2g"}' % (i + 1, 1000 + gpu[i], _us(int(b.t_l[i])))))
    S = len(b.span_start)
    pos_s = rng.uniform(S) * n
    for j in range(S):
        g, lv = int(b.span_gl[j] >> 8), int(b.span_gl[j] & 0xFF)
        out.append((1, pos_s[j], '{"ph": "X", "cat": "user_annotation", "name": "span\\"%d\\"", "pid": %d, '
                    '"tid": "annotations", "ts": %s, "dur": %s, "args": {"level": %d, "label": %d}}'
                    % (int(b.span_label[j]), g, _us(int(b.span_start[j])),
                       _us(int(b.span_end[j] - b.span_start[j])), lv, int(b.span_label[j]))))
    out.sort(key=lambda x: (x[1], x[0]))
    return ('{"schemaVersion": 1, "traceEvents": [\n' + ",\n".join(x[2] for x in out) +
            '\n], "displayTimeUnit": "ms"}\n').encode()
