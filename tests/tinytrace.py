"""Hand-built tiny traces for pins and edge cases (test infrastructure, no method arithmetic).

A TinyTrace collects events / spans / samples / counter passes and produces a
tracegen.Bundle so the oracle and the CUDA path consume exactly the same
columns as for generated traces.
"""
from __future__ import annotations

import dataclasses

import numpy as np

import tracegen
from tracegen import AG, COMM_OTHER, COMPUTE, COPY, MEMOP, OTHER, RS  # noqa: F401


class TinyTrace:
    def __init__(self, n_gpus=1, labels=None, n_counters=0, warmup=0, b=2, s=4096):
        self.n_gpus = n_gpus
        self.events = []       # (gpu, t_l, t_ks, t_ke, stream, kind, name)
        self.spans = []        # (gpu, level, start, end, label)
        self.samples = []      # (gpu, ts, f, p)
        self.passes = []       # (gpu, names, slots, values[k][n])
        self.labels = labels or ["op%d" % i for i in range(4)]
        self.n_counters = n_counters
        self.warmup = warmup
        self.b, self.s = b, s

    def ev(self, gpu, t_l, ks, ke, kind=COMPUTE, stream=0, name=0):
        self.events.append((gpu, t_l, ks, ke, stream, kind, name))
        return self

    def span(self, gpu, level, start, end, label=0):
        self.spans.append((gpu, level, start, end, label))
        return self

    def sample(self, gpu, ts, f, p=0):
        self.samples.append((gpu, ts, f, p))
        return self

    def counter_pass(self, gpu, names, slots, values):
        self.passes.append((gpu, np.asarray(names, np.int32), np.asarray(slots, np.int32),
                            np.asarray(values, np.float64).reshape(len(slots), len(names))))
        return self

    def bundle(self, keep_order=False) -> tracegen.Bundle:
        ev = list(self.events)
        if not keep_order:
            # grouped by gpu, dispatch-ordered within a gpu (stable for equal t_l)
            ev = sorted(ev, key=lambda e: (e[0], e[1]))
        a = np.array([(e[0], e[1], e[2], e[3], e[4], e[5], e[6]) for e in ev], dtype=np.int64).reshape(-1, 7)
        meta = ((a[:, 0] << 24) | (a[:, 4] << 8) | a[:, 5]).astype(np.uint32)
        sp = np.array(self.spans, dtype=np.int64).reshape(-1, 5)
        sm = sorted(self.samples, key=lambda x: (x[0], x[1]))
        smp = np.array(sm, dtype=np.int64).reshape(-1, 4)
        cfg = tracegen.TraceConfig(config_id=0, seed=0, n_gpus=self.n_gpus, n_iters=1, n_layers=1,
                                   warmup=self.warmup, batch=self.b, seq=self.s, n_counters=self.n_counters)
        return tracegen.Bundle(
            cfg=cfg, t_l=a[:, 1].copy(), t_ks=a[:, 2].copy(), t_ke=a[:, 3].copy(), meta=meta,
            name_id=a[:, 6].astype(np.int32),
            span_gl=((sp[:, 0] << 8) | sp[:, 1]).astype(np.uint32), span_start=sp[:, 2].copy(),
            span_end=sp[:, 3].copy(), span_label=sp[:, 4].astype(np.int32),
            smp_gpu=smp[:, 0].astype(np.int32), smp_ts=smp[:, 1].copy(), smp_freq=smp[:, 2].astype(np.int32),
            smp_power=smp[:, 3].astype(np.int32), passes=list(self.passes), n_counters=self.n_counters,
            labels=list(self.labels), delta=np.zeros(self.n_gpus, np.int64), freq_ratio=np.ones(self.n_gpus))


def params(bundle, **kw):
    """Breakdown parameters for a tiny trace; op_type / f_gemm given explicitly by the test."""
    L = len(bundle.labels)
    C = bundle.n_counters
    p = dict(tpt_peak=1.3e15, freq_peak_hz=2.1e9, b=bundle.cfg.batch, s=bundle.cfg.seq, R=bundle.cfg.n_gpus,
             warmup=bundle.cfg.warmup, slot_cycles=0 if C > 0 else -1, slot_flops=1 if C > 1 else -1,
             slot_unum=2 if C > 3 else -1, slot_uden=3 if C > 3 else -1,
             f_gemm=np.full(L, 1.3e12), op_type=np.ones(L, dtype=np.int32),
             ratio_num=np.zeros(0, np.int32), ratio_den=np.zeros(0, np.int32), ratio_scale=np.zeros(0))
    p.update(kw)
    return p


def replace(bundle, **kw):
    return dataclasses.replace(bundle, **kw)
