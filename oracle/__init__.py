"""Python loader for the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`) may import this package.  It shares no code with the CUDA
product path (paper_2512_08242_b200/); the theoretical-FLOP table below is the
oracle's own restatement of Eq. 4's F_gemm (D19).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "chopper_oracle.c")
_LIB = os.path.join(_HERE, "libchopper_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2, no FMA contraction: DESIGN.md D22)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=gnu11", "-fPIC", "-shared", "-o", _LIB, _SRC,
                               "-lm"])
    return _LIB


class _Input(ctypes.Structure):
    _fields_ = [
        ("n_events", ctypes.c_int64), ("t_l", ctypes.c_void_p), ("t_ks", ctypes.c_void_p), ("t_ke", ctypes.c_void_p),
        ("meta", ctypes.c_void_p), ("name_id", ctypes.c_void_p),
        ("n_spans", ctypes.c_int64), ("span_gl", ctypes.c_void_p), ("span_start", ctypes.c_void_p),
        ("span_end", ctypes.c_void_p), ("span_label", ctypes.c_void_p),
        ("n_samples", ctypes.c_int64), ("smp_gpu", ctypes.c_void_p), ("smp_ts", ctypes.c_void_p),
        ("smp_freq_mhz", ctypes.c_void_p), ("smp_power_mw", ctypes.c_void_p),
        ("n_passes", ctypes.c_int32), ("pass_gpu", ctypes.c_void_p), ("pass_n", ctypes.c_void_p),
        ("pass_k", ctypes.c_void_p), ("pass_name_id", ctypes.c_void_p), ("pass_slot", ctypes.c_void_p),
        ("pass_values", ctypes.c_void_p), ("n_counters", ctypes.c_int32),
        ("n_traced_gpus", ctypes.c_int32), ("n_labels", ctypes.c_int32), ("max_iters", ctypes.c_int32),
        ("tpt_peak", ctypes.c_double), ("freq_peak_hz", ctypes.c_double),
        ("b", ctypes.c_int64), ("s", ctypes.c_int64), ("R", ctypes.c_int64), ("warmup", ctypes.c_int32),
        ("slot_cycles", ctypes.c_int32), ("slot_flops", ctypes.c_int32), ("slot_unum", ctypes.c_int32),
        ("slot_uden", ctypes.c_int32), ("f_gemm", ctypes.c_void_p), ("op_type", ctypes.c_void_p),
        ("n_ratios", ctypes.c_int32), ("ratio_num", ctypes.c_void_p), ("ratio_den", ctypes.c_void_p),
        ("ratio_scale", ctypes.c_void_p), ("bd_gpu_mask", ctypes.c_uint64),
    ]


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.or_run.restype = ctypes.c_void_p
        _lib.or_run.argtypes = [ctypes.POINTER(_Input)]
        _lib.or_get.restype = ctypes.c_int32
        _lib.or_get.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)]
        _lib.or_count.restype = ctypes.c_int32
        _lib.or_count.argtypes = [ctypes.c_void_p]
        _lib.or_name.restype = ctypes.c_char_p
        _lib.or_name.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        _lib.or_free.argtypes = [ctypes.c_void_p]
    return _lib


# ---------------------------------------------------------------------------
# Eq. 4 theoretical FLOPs (oracle's own table)
# ---------------------------------------------------------------------------
def gemm_flops(m: int, n: int, k: int) -> float:
    """2*m*n*k multiply-adds counted as 2 flops each."""
    return 2.0 * m * n * k


def attention_flops(b: int, heads: int, s: int, head_dim: int, causal_factor: float = 1.0) -> float:
    """forward attention: QK^T and PV, each 2*s*s*d per head -> 4*b*h*s^2*d."""
    return 4.0 * b * heads * s * s * head_dim * causal_factor


def flops_table(labels, shapes: Dict[str, int], bwd_gemm: float = 2.0, bwd_fa: float = 2.5) -> np.ndarray:
    """F_gemm per op label, summed across layers for the per-layer ops (points are summed across layers)."""
    b, s, H, F = shapes["b"], shapes["s"], shapes["hidden"], shapes["ffn"]
    nh, kvh, hd, V, L = shapes["heads"], shapes["kv_heads"], shapes["head_dim"], shapes["vocab"], shapes["layers"]
    m = b * s
    per = {
        "qkv_ip": gemm_flops(m, H + 2 * kvh * hd, H),
        "attn_op": gemm_flops(m, H, H),
        "mlp_gp": gemm_flops(m, F, H),
        "mlp_up": gemm_flops(m, F, H),
        "mlp_dp": gemm_flops(m, H, F),
        "attn_fa": attention_flops(b, nh, s, hd),
        "lp": gemm_flops(m, V, H),
    }
    out = np.zeros(len(labels), dtype=np.float64)
    for i, lab in enumerate(labels):
        pre, base = (lab[:2], lab[2:]) if lab[:2] in ("f_", "b_") else ("", lab)
        if base not in per:
            continue
        v = per[base] * (L if base != "lp" else 1)
        if pre == "b_":
            v *= bwd_fa if base == "attn_fa" else bwd_gemm
        out[i] = v
    return out


def default_params(bundle, n_ratios_default: bool = True) -> dict:
    """Breakdown parameters for a generated bundle (hardware spec: MI300X as in PAPER.md:197, 303)."""
    import tracegen
    cfg = bundle.cfg
    labels = bundle.labels
    C = bundle.n_counters
    p = dict(tpt_peak=1.3e15, freq_peak_hz=2.1e9, b=cfg.batch, s=cfg.seq, R=cfg.n_gpus, warmup=cfg.warmup,
             slot_cycles=0 if C > 0 else -1, slot_flops=1 if C > 1 else -1,
             slot_unum=2 if C > 3 else -1, slot_uden=3 if C > 3 else -1,
             f_gemm=flops_table(labels, tracegen.workload_shapes(cfg)),
             op_type=np.array([tracegen.op_kind(l) for l in labels], dtype=np.int32))
    if C >= 6 and n_ratios_default:
        # bandwidth = bytes / duration, and a counter/counter ratio
        p.update(ratio_num=np.array([4, 5, 1], dtype=np.int32), ratio_den=np.array([-1, -1, 0], dtype=np.int32),
                 ratio_scale=np.array([1.0, 1.0, 1.0], dtype=np.float64))
    else:
        p.update(ratio_num=np.zeros(0, np.int32), ratio_den=np.zeros(0, np.int32), ratio_scale=np.zeros(0))
    return p


def _ptr(a):
    return a.ctypes.data if a is not None and a.size > 0 else None


def run(bundle, params: Optional[dict] = None, max_iters: int = 4096, gpu_mask: Optional[int] = None) -> Dict[str, np.ndarray]:
    """Run the oracle on a whole (all traced GPUs) bundle; returns named numpy arrays."""
    lib = _load()
    p = default_params(bundle) if params is None else params
    keep = []

    def c(a, dt):
        a = np.ascontiguousarray(np.asarray(a), dtype=dt)
        keep.append(a)
        return a

    ev = [c(bundle.t_l, np.int64), c(bundle.t_ks, np.int64), c(bundle.t_ke, np.int64), c(bundle.meta, np.uint32),
          c(bundle.name_id, np.int32)]
    spn = [c(bundle.span_gl, np.uint32), c(bundle.span_start, np.int64), c(bundle.span_end, np.int64),
           c(bundle.span_label, np.int32)]
    smp = [c(bundle.smp_gpu, np.int32), c(bundle.smp_ts, np.int64), c(bundle.smp_freq, np.int32),
           c(bundle.smp_power, np.int32)]
    P = len(bundle.passes)
    pg = c([q[0] for q in bundle.passes], np.int32)
    pn = c([len(q[1]) for q in bundle.passes], np.int64)
    pk = c([len(q[2]) for q in bundle.passes], np.int32)
    names = [c(q[1], np.int32) for q in bundle.passes]
    slots = [c(q[2], np.int32) for q in bundle.passes]
    vals = [c(q[3], np.float64) for q in bundle.passes]
    pnm = (ctypes.c_void_p * max(P, 1))(*[x.ctypes.data for x in names])
    psl = (ctypes.c_void_p * max(P, 1))(*[x.ctypes.data for x in slots])
    pvl = (ctypes.c_void_p * max(P, 1))(*[x.ctypes.data for x in vals])
    fg = c(p["f_gemm"], np.float64)
    ot = c(p["op_type"], np.int32)
    rn, rd, rs = c(p["ratio_num"], np.int32), c(p["ratio_den"], np.int32), c(p["ratio_scale"], np.float64)
    inp = _Input(
        n_events=len(ev[0]), t_l=_ptr(ev[0]), t_ks=_ptr(ev[1]), t_ke=_ptr(ev[2]), meta=_ptr(ev[3]), name_id=_ptr(ev[4]),
        n_spans=len(spn[0]), span_gl=_ptr(spn[0]), span_start=_ptr(spn[1]), span_end=_ptr(spn[2]),
        span_label=_ptr(spn[3]), n_samples=len(smp[0]), smp_gpu=_ptr(smp[0]), smp_ts=_ptr(smp[1]),
        smp_freq_mhz=_ptr(smp[2]), smp_power_mw=_ptr(smp[3]), n_passes=P, pass_gpu=_ptr(pg), pass_n=_ptr(pn),
        pass_k=_ptr(pk), pass_name_id=ctypes.cast(pnm, ctypes.c_void_p), pass_slot=ctypes.cast(psl, ctypes.c_void_p),
        pass_values=ctypes.cast(pvl, ctypes.c_void_p), n_counters=bundle.n_counters,
        n_traced_gpus=bundle.cfg.n_gpus, n_labels=len(bundle.labels), max_iters=max_iters,
        tpt_peak=p["tpt_peak"], freq_peak_hz=p["freq_peak_hz"], b=p["b"], s=p["s"], R=p["R"], warmup=p["warmup"],
        slot_cycles=p["slot_cycles"], slot_flops=p["slot_flops"], slot_unum=p["slot_unum"], slot_uden=p["slot_uden"],
        f_gemm=_ptr(fg), op_type=_ptr(ot), n_ratios=len(rn), ratio_num=_ptr(rn), ratio_den=_ptr(rd),
        ratio_scale=_ptr(rs), bd_gpu_mask=(gpu_mask if gpu_mask is not None else 0xFFFFFFFFFFFFFFFF))
    h = lib.or_run(ctypes.byref(inp))
    out = {}
    try:
        dts = {0: np.int32, 1: np.int64, 2: np.float64, 3: np.uint8}
        for i in range(lib.or_count(h)):
            nm = lib.or_name(h, i)
            ptr, n, dt = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int32()
            lib.or_get(h, nm, ctypes.byref(ptr), ctypes.byref(n), ctypes.byref(dt))
            t = dts[dt.value]
            if n.value > 0:
                buf = (ctypes.c_char * (n.value * np.dtype(t).itemsize)).from_address(ptr.value)
                out[nm.decode()] = np.frombuffer(buf, dtype=t).copy()
            else:
                out[nm.decode()] = np.zeros(0, dtype=t)
    finally:
        lib.or_free(h)
    return out


def cpu_util(ts, core, util, topology) -> Dict[str, np.ndarray]:
    """O17 CPU utilization: per-timestamp C_active / C_min and the summary row
    [n_ts, median C_active, median C_min, max C_active, max C_min, physical occupancy, SMT co-activity,
    #physical]; 'bad' = 1 when the samples are unsorted, out of range or the topology is invalid."""
    lib = _load()
    f = lib.or_cpu_util
    f.restype = ctypes.c_int64
    f.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32)]
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    core = np.ascontiguousarray(core, dtype=np.int32)
    util = np.ascontiguousarray(util, dtype=np.float64)
    topo = np.ascontiguousarray(topology, dtype=np.int32)
    n = int(ts.shape[0])
    ca = np.zeros(max(n, 1), np.int64)
    cm = np.zeros(max(n, 1), np.float64)
    summ = np.full(8, np.nan)
    bad = ctypes.c_int32(0)
    nts = int(f(n, _ptr(ts), _ptr(core), _ptr(util), int(topo.shape[0]), _ptr(topo), ca.ctypes.data, cm.ctypes.data,
                summ.ctypes.data, ctypes.byref(bad)))
    return {"c_active": ca[:nts].copy(), "c_min": cm[:nts].copy(), "summary": summ, "bad": int(bad.value)}



# ---------------------------------------------------------------------------
# derived-metric registry: a recursive-descent evaluator
#   expr := term (('+' | '-') term)* ; term := unary (('*' | '/') unary)* ; unary := '-' unary | primary
#   primary := number | identifier | '(' expr ')'   (binary operators left-associative)
# identifiers: counter names (the row's summed counter) and dur_s (the row's busy seconds); a zero divisor or
# an infinite quotient gives NaN (reading R14).
# ---------------------------------------------------------------------------
class MetricError(ValueError):
    pass


def _metric_tokens(e: str):
    import re
    toks, i = [], 0
    pat = re.compile(r"\s*(?:(\d+\.?\d*(?:[eE][+-]?\d+)?|\.\d+(?:[eE][+-]?\d+)?)|([A-Za-z_][A-Za-z0-9_.]*)|(.))")
    while i < len(e):
        m = pat.match(e, i)
        if not m or m.end() == i:
            break
        i = m.end()
        if m.group(1):
            toks.append(("num", float(m.group(1))))
        elif m.group(2):
            toks.append(("id", m.group(2)))
        elif m.group(3) and not m.group(3).isspace():
            if m.group(3) not in "+-*/()":
                raise MetricError(f"ParseError: unexpected character {m.group(3)!r}")
            toks.append(("op", m.group(3)))
    return toks


def metric_eval(expr: str, names, counters, busy_ns):
    """Evaluate one registry expression over rows: counters [C][n] (summed per row), busy_ns [n]."""
    toks = _metric_tokens(expr)
    counters = np.asarray(counters, dtype=np.float64)
    dur = np.asarray(busy_ns, dtype=np.float64) * 1e-9
    pos = [0]

    def peek():
        return toks[pos[0]] if pos[0] < len(toks) else (None, None)

    def take():
        t = peek()
        pos[0] += 1
        return t

    def primary():
        k, v = take()
        if k == "num":
            return np.full(dur.shape, v)
        if k == "id":
            if v == "dur_s":
                return dur.copy()
            if v not in names:
                raise MetricError(f"MissingCounter({v})")
            return counters[list(names).index(v)].copy()
        if (k, v) == ("op", "("):
            x = expr_()
            if take() != ("op", ")"):
                raise MetricError("ParseError: missing ')'")
            return x
        raise MetricError("ParseError")

    def unary():
        if peek() == ("op", "-"):
            take()
            return -unary()
        return primary()

    def term():
        x = unary()
        while peek() in (("op", "*"), ("op", "/")):
            _, o = take()
            y = unary()
            if o == "*":
                x = x * y
            else:
                with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
                    q = np.where(y == 0.0, np.nan, x / np.where(y == 0.0, 1.0, y))
                    x = np.where(np.isinf(q), np.nan, q)     # "error, not infinity" (R14)
        return x

    def expr_():
        x = term()
        while peek() in (("op", "+"), ("op", "-")):
            _, o = take()
            y = term()
            x = x + y if o == "+" else x - y
        return x

    out = expr_()
    if pos[0] != len(toks):
        raise MetricError("ParseError: trailing tokens")
    return out


# ---------------------------------------------------------------------------
# Chrome-trace ingest (R15): Python's json with
# exact decimals, plain loops.  Device events: ph X with cat "kernel" or "gpu_*" (pid = gpu, tid = stream,
# args.correlation); host launches: flow-start events (ph "s", id = correlation, ts = dispatch); spans: ph X
# with cat "user_annotation" (pid = gpu, args.level, args.label).  Times: decimal microseconds -> integer ns,
# rounded half to even; end = start + duration, each rounded.  Kinds by the first matching rule
# (R15).  name_id = order of first appearance of the name among device events.  Output grouped by gpu and
# dispatch-ordered (stable: file order); kernels without a launch get dispatch = start and are counted.
# ---------------------------------------------------------------------------
def _kind_rule(cat: str, name: str) -> int:
    n = name.lower()
    if cat == "gpu_memset":
        return 5          # MEMOP
    if cat == "gpu_memcpy":
        return 4          # COPY
    if cat != "kernel":
        return 6          # OTHER
    if "allgather" in n or "all_gather" in n:
        return 1          # AG
    if "reducescatter" in n or "reduce_scatter" in n:
        return 2          # RS
    if "nccl" in n or "rccl" in n:
        return 3          # COMM_OTHER
    if "fsdp_copy" in n:
        return 4          # COPY (D7: FSDP copy kernels are bubbles)
    return 0              # COMPUTE


def ingest_chrome(data: bytes) -> Dict[str, np.ndarray]:
    import decimal
    import json
    D = decimal.Decimal

    def ns(x) -> int:
        return int((D(x) * 1000).quantize(D(1), rounding=decimal.ROUND_HALF_EVEN))

    doc = json.loads(data, parse_float=D)
    evs = doc["traceEvents"]
    flows = {}
    dev, spans = [], []
    for e in evs:
        ph, cat = e.get("ph"), e.get("cat", "")
        if ph == "s" and "id" in e:
            flows.setdefault(int(e["id"]), ns(e["ts"]))
        elif ph == "X" and cat == "user_annotation":
            a = e.get("args", {})
            s = ns(e["ts"])
            spans.append((int(e["pid"]), int(a["level"]), s, s + ns(e["dur"]), int(a["label"])))
        elif ph == "X" and (cat == "kernel" or cat.startswith("gpu_")):
            s = ns(e["ts"])
            corr = e.get("args", {}).get("correlation")
            dev.append((int(e["pid"]), int(e["tid"]), _kind_rule(cat, e["name"]), s, s + ns(e["dur"]), e["name"],
                        None if corr is None else int(corr)))
    names = {}
    for d in dev:
        names.setdefault(d[5], len(names))
    missing = 0
    rows = []
    for q, d in enumerate(dev):
        g, st, k, s, t, nm, c = d
        if c is not None and c in flows:
            tl = flows[c]
        else:
            tl = s
            missing += 1
        rows.append((g, tl, q, s, t, (g << 24) | (st << 8) | k, names[nm]))
    rows.sort(key=lambda r: (r[0], r[1], r[2]))
    a = np.array([(r[1], r[3], r[4], r[5], r[6]) for r in rows], dtype=np.int64).reshape(-1, 5)
    sp = np.array(spans, dtype=np.int64).reshape(-1, 5)
    return {"t_l": a[:, 0], "t_ks": a[:, 1], "t_ke": a[:, 2], "meta": a[:, 3].astype(np.uint32),
            "name_id": a[:, 4].astype(np.int32), "span_gl": ((sp[:, 0] << 8) | sp[:, 1]).astype(np.uint32),
            "span_start": sp[:, 2], "span_end": sp[:, 3], "span_label": sp[:, 4].astype(np.int32),
            "n_missing": missing, "names": list(names)}
