"""Pipeline driver over the C ABI: upload columns into torch CUDA tensors, run
chopper_load_columns -> align -> attribute -> overlap -> breakdown ->
reduce_ranks, and read results back.  Marshalling only -- no analysis here.

flops_table() is the host-side Eq. 4 parameter table (theoretical FLOPs of an
op label from the workload shapes, D19).
"""
from __future__ import annotations

import ctypes
from typing import Dict, Optional

import numpy as np

from . import (PassArray, chopper_set_allgather_loopback, chopper_scratch_plan, chopper_shape, chopper_align, chopper_attribute, chopper_breakdown, chopper_config, chopper_counter_pass,
               chopper_cpu_util, chopper_create, chopper_set_metrics, chopper_destroy, chopper_events, chopper_get_report, chopper_global, chopper_report_cdf,
               chopper_kernel_launches, chopper_load_columns, chopper_overlap, chopper_reduce_ranks,
               chopper_samples, chopper_scratch_bytes, chopper_spans, chopper_status_sync, chopper_tables,
               ChopperError, _check, bd_params, chopper_last_error, dev_to_numpy, load_library, rows_to_numpy)

_GEMM = {"qkv_ip", "attn_op", "mlp_gp", "mlp_up", "mlp_dp", "lp"}


def flops_table(labels, shapes: Dict[str, int], bwd_gemm: float = 2.0, bwd_fa: float = 2.5) -> np.ndarray:
    """F_gemm per op label (Eq. 4): GEMM m x n x k -> 2mnk; attention -> 4*b*h*s^2*d; per-layer ops are
    summed over the layers because a point sums an op across layers."""
    b, s, H, F = shapes["b"], shapes["s"], shapes["hidden"], shapes["ffn"]
    h, kvh, d, V, L = shapes["heads"], shapes["kv_heads"], shapes["head_dim"], shapes["vocab"], shapes["layers"]
    tok = b * s
    shape = {"qkv_ip": (tok, H + 2 * kvh * d, H), "attn_op": (tok, H, H), "mlp_gp": (tok, F, H),
             "mlp_up": (tok, F, H), "mlp_dp": (tok, H, F), "lp": (tok, V, H)}
    out = np.zeros(len(labels))
    for i, lab in enumerate(labels):
        pre, base = (lab[:2], lab[2:]) if lab[:2] in ("f_", "b_") else ("", lab)
        if base in shape:
            m, n, k = shape[base]
            v = 2.0 * m * n * k
            mult = bwd_gemm
        elif base == "attn_fa":
            v = 4.0 * b * h * s * s * d
            mult = bwd_fa
        else:
            continue
        if base != "lp":
            v *= L
        out[i] = v * (mult if pre == "b_" else 1.0)
    return out


def default_params(cols, labels, shapes: Dict[str, int], op_kind) -> dict:
    """Host-side breakdown parameters for a run (chopper_bd_params): the hardware spec (MI300X peak dense
    throughput and clock), the workload (b, s, R, warm-up), the counter-slot layout of
    the trace, the Eq. 4 FLOP table (flops_table) and op types.  Plumbing only."""
    cfg = cols.cfg
    C = cols.n_counters
    p = dict(tpt_peak=1.3e15, freq_peak_hz=2.1e9, b=cfg.batch, s=cfg.seq, R=cfg.n_gpus, warmup=cfg.warmup,
             slot_cycles=0 if C > 0 else -1, slot_flops=1 if C > 1 else -1,
             slot_unum=2 if C > 3 else -1, slot_uden=3 if C > 3 else -1,
             f_gemm=flops_table(labels, shapes), op_type=np.array([op_kind(l) for l in labels], dtype=np.int32))
    if C >= 6:
        # bandwidth = bytes / duration, and a counter/counter ratio
        p.update(ratio_num=np.array([4, 5, 1], dtype=np.int32), ratio_den=np.array([-1, -1, 0], dtype=np.int32),
                 ratio_scale=np.array([1.0, 1.0, 1.0], dtype=np.float64))
    else:
        p.update(ratio_num=np.zeros(0, np.int32), ratio_den=np.zeros(0, np.int32), ratio_scale=np.zeros(0))
    return p


def trace_shape(cols, n_counters: int, laminar: bool = True) -> "chopper_shape":
    """chopper_shape of a trace's columns (counts only: spans per level, communication events, local gpus,
    compute streams) for chopper_scratch_plan.  `laminar` is the caller's statement that no same-level spans
    cross (true for FSDP annotations; False plans the exact sweep's per-event table)."""
    meta = np.asarray(cols.meta, np.uint32)
    kind = meta & 0xFF
    lv = np.asarray(cols.span_gl, np.uint32) & 0xFF
    comp = kind == 0
    streams = int(((meta[comp] >> 8) & 0xFFFF).max()) + 1 if comp.any() else 1
    sh = chopper_shape(n_events=len(meta), n_samples=len(cols.smp_gpu), n_comm=int(np.isin(kind, (1, 2, 3)).sum()),
                       n_counters=n_counters, n_local_gpus=len(np.unique(meta >> 24)),
                       max_compute_streams=streams, laminar=1 if laminar else 0)
    for k in range(4):
        sh.n_spans[k] = int((lv == k).sum())
    return sh


def scratch_plan(n_traced_gpus: int, n_labels: int, max_iters: int, max_coll_per_class: int, cols, n_counters: int,
                 laminar: bool = True) -> Dict[str, int]:
    cfg = chopper_config(n_traced_gpus=n_traced_gpus, n_labels=n_labels, max_iters=max_iters,
                         max_coll_per_class=max_coll_per_class)
    return chopper_scratch_plan(cfg, trace_shape(cols, n_counters, laminar))


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class Pipeline:
    """One rank's chopper context.  `cols` is any object with the column attributes of the ABI
    (t_l, t_ks, t_ke, meta, name_id, span_*, smp_*, passes)."""

    def __init__(self, n_traced_gpus: int, n_labels: int, max_iters: int, max_coll_per_class: int,
                 device: int = 0, pg=None, stream=None, loopback=None, rank: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2512_08242_b200 needs a CUDA device (no CPU fallback)")
        load_library()
        self.torch = torch
        self.device = device
        self.cfg = chopper_config(n_traced_gpus=n_traced_gpus, n_labels=n_labels, max_iters=max_iters,
                                  max_coll_per_class=max_coll_per_class)
        self.stream = stream or torch.cuda.current_stream(device)
        self.pg = pg
        self.rank, self.nranks = 0, 1
        self.comm = 0
        if pg is not None:
            import torch.distributed as dist
            self.rank, self.nranks = dist.get_rank(pg), dist.get_world_size(pg)
            if self.nranks > 1:
                be = pg._get_backend(torch.device("cuda", device))
                self.comm = int(be._comm_ptr())
        self.loopback = loopback
        if loopback is not None:
            # in-process ranks on one device (chopper_loopback_*): rank r of loopback.nranks
            self.rank, self.nranks = rank, loopback.nranks
        self.ctx = None
        self.scratch = None
        self.d = {}
        self.passes_dev = []
        self._mcache = {}
        self.cpu = None

    def set_metrics(self, exprs, names) -> None:
        """Derived-metric registry: infix expressions over counter names and dur_s."""
        chopper_set_metrics(self.ctx, list(exprs), list(names))

    def upload_cpu(self, ts, core, util, topology) -> None:
        """Host CPU utilisation samples (sorted by (ts, logical core)) and the logical -> physical topology."""
        torch = self.torch
        dev = torch.device("cuda", self.device)
        with torch.cuda.stream(self.stream):
            self.cpu = {"ts": torch.from_numpy(_i64(ts)).to(dev),
                        "core": torch.from_numpy(np.ascontiguousarray(core, np.int32)).to(dev),
                        "util": torch.from_numpy(np.ascontiguousarray(util, np.float64)).to(dev),
                        "topo": torch.from_numpy(np.ascontiguousarray(topology, np.int32)).to(dev)}

    # ---- inputs ----
    def upload(self, cols, n_counters: int, pinned_host: Optional[dict] = None, plan_laminar: Optional[bool] = None) -> None:
        """Copy input columns to the device (from pinned host tensors if given).  The scratch arena is sized by
        chopper_scratch_bytes (worst case), or by chopper_scratch_plan of the trace's shape when plan_laminar
        is given (the caller states whether same-level spans may cross)."""
        torch = self.torch
        dev = torch.device("cuda", self.device)
        src = {
            "t_l": _i64(cols.t_l), "t_ks": _i64(cols.t_ks), "t_ke": _i64(cols.t_ke),
            "meta": np.ascontiguousarray(cols.meta, np.uint32).view(np.int32),
            "name_id": np.ascontiguousarray(cols.name_id, np.int32),
            "span_gl": np.ascontiguousarray(cols.span_gl, np.uint32).view(np.int32),
            "span_start": _i64(cols.span_start), "span_end": _i64(cols.span_end),
            "span_label": np.ascontiguousarray(cols.span_label, np.int32),
            "smp_gpu": np.ascontiguousarray(cols.smp_gpu, np.int32), "smp_ts": _i64(cols.smp_ts),
            "smp_freq": np.ascontiguousarray(cols.smp_freq, np.int32),
            "smp_power": np.ascontiguousarray(cols.smp_power, np.int32),
        }
        d = {}
        with torch.cuda.stream(self.stream):
            for k, v in src.items():
                if pinned_host is not None and k in pinned_host:
                    d[k] = pinned_host[k].to(dev, non_blocking=True)
                else:
                    d[k] = torch.from_numpy(v).to(dev, non_blocking=False)
            self.passes_dev = []
            for (g, names, slots, vals) in cols.passes:
                self.passes_dev.append((int(g), torch.from_numpy(np.ascontiguousarray(names, np.int32)).to(dev),
                                        np.ascontiguousarray(slots, np.int32),
                                        torch.from_numpy(np.ascontiguousarray(vals, np.float64)).to(dev)))
        self.d = d
        self._mcache = {}
        self.n_counters = n_counters
        self.N, self.S, self.M = len(src["t_l"]), len(src["span_gl"]), len(src["smp_gpu"])
        if plan_laminar is None:
            need = chopper_scratch_bytes(self.cfg, self.N, self.S, self.M, n_counters)
        else:
            need = chopper_scratch_plan(self.cfg, trace_shape(cols, n_counters, plan_laminar))["total"]
        if self.scratch is None or self.scratch.numel() < need:
            self.scratch = None
            if self.ctx:
                chopper_destroy(self.ctx)
                self.ctx = None
            self.scratch = torch.empty(need, dtype=torch.uint8, device=dev)
        if self.ctx is None:
            self.ctx = chopper_create(self.cfg, self.device, self.stream.cuda_stream, self.comm, self.rank,
                                      self.nranks, self.scratch)
            if self.loopback is not None:
                chopper_set_allgather_loopback(self.ctx, self.loopback)

    # ---- double-buffered streaming inputs ----
    def input_set(self) -> dict:
        """The device input buffers now in use, as a set `use_inputs` / `stage_inputs` accept."""
        return {"d": self.d, "passes": self.passes_dev, "cpu": self.cpu}

    def new_input_set(self) -> dict:
        """A second device copy of the input buffers (same shapes), for streaming trace after trace: the next
        trace's host->device copy runs on a copy stream while `run` computes on the other set."""
        torch = self.torch
        return {"d": {k: torch.empty_like(v) for k, v in self.d.items()},
                "passes": [(g, torch.empty_like(nm), sl, torch.empty_like(v)) for (g, nm, sl, v) in self.passes_dev],
                "cpu": None if self.cpu is None else {k: torch.empty_like(v) for k, v in self.cpu.items()}}

    def stage_inputs(self, s: dict, pinned: dict, pinned_passes, pinned_cpu: Optional[dict], copy_stream):
        """Enqueue the pinned-host -> device copies of one trace into set `s` on `copy_stream`; returns the
        CUDA event that completes with them (pass it to `use_inputs`).  The caller guarantees that no
        queued `run` still reads `s` (run returns after its status read-back, so the set used by the
        previous, returned call is free)."""
        torch = self.torch
        with torch.cuda.stream(copy_stream):
            for k, v in pinned.items():
                s["d"][k].copy_(v, non_blocking=True)
            for q, (nm, vals) in enumerate(pinned_passes):
                s["passes"][q][1].copy_(nm, non_blocking=True)
                s["passes"][q][3].copy_(vals, non_blocking=True)
            if pinned_cpu:
                for k, v in pinned_cpu.items():
                    s["cpu"][k].copy_(v, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        return ev

    def use_inputs(self, s: dict, ready=None) -> None:
        """Make `s` the input set of the next `run`; its compute stream waits for `ready` (a stage_inputs
        event) on the device, the host does not block."""
        if ready is not None:
            self.stream.wait_event(ready)
        self.d, self.passes_dev, self.cpu = s["d"], s["passes"], s["cpu"]

    def _marshal(self):
        """The ABI structs of the current input set: events / spans / samples and the counter-pass array.  Built
        once per input set (upload, or each set `use_inputs` alternates between) -- the set's tensors are kept
        in the cache entry, so an entry's device pointers stay valid while it is cached."""
        key = (id(self.d), id(self.passes_dev), id(self.cpu))
        hit = self._mcache.get(key)
        if hit is not None and hit[0] is self.d and hit[1] is self.passes_dev:
            return hit[2]
        d = self.d
        ev = chopper_events(n=self.N, dispatch_ns=d["t_l"].data_ptr(), start_ns=d["t_ks"].data_ptr(),
                            end_ns=d["t_ke"].data_ptr(), meta=d["meta"].data_ptr(), name_id=d["name_id"].data_ptr())
        sp = chopper_spans(n=self.S, gpu_level=d["span_gl"].data_ptr(), start_ns=d["span_start"].data_ptr(),
                           end_ns=d["span_end"].data_ptr(), label=d["span_label"].data_ptr())
        smp = chopper_samples(n=self.M, gpu=d["smp_gpu"].data_ptr(), ts_ns=d["smp_ts"].data_ptr(),
                              freq_mhz=d["smp_freq"].data_ptr(), power_mw=d["smp_power"].data_ptr()) \
            if self.M > 0 else None
        passes = [chopper_counter_pass(gpu=g, n=names.numel(), name_id=names.data_ptr(), k=len(slots),
                                       slot=slots.ctypes.data, values=vals.data_ptr())
                  for (g, names, slots, vals) in self.passes_dev]
        arr = (chopper_counter_pass * max(len(passes), 1))(*passes)
        m = (ev, sp, smp, PassArray(arr, len(passes)))
        if len(self._mcache) >= 4:
            self._mcache.clear()
        self._mcache[key] = (self.d, self.passes_dev, m)     # (the slots arrays live in passes_dev)
        return m

    # ---- run ----
    def run(self, params: dict, full: bool = False, check: bool = True) -> dict:
        """All six ABI calls.  full=True also writes the per-event outputs (parity mode)."""
        torch = self.torch
        N = self.N
        ev, sp, smp, passes = self._marshal()
        res = {"full": full}
        allow = () if check else tuple(range(1, 10))
        s = chopper_load_columns(self.ctx, ev, sp, smp)
        res["load_status"] = s
        res["report"] = chopper_get_report(self.ctx)
        if s != 0 and self.nranks > 1:
            # failure protocol (chopper.h): the remaining calls still run so every rank's all-gathers match
            self._finish_failed_step()
        if s != 0:
            _check(self.ctx, s, "chopper_load_columns", allow=allow)
            return res
        C = self.n_counters
        dev = torch.device("cuda", self.device)
        out = {}
        if full:
            out["counters"] = torch.zeros((max(C, 1), max(N, 1)), dtype=torch.float64, device=dev)
            out["span_idx"] = torch.empty((4, max(N, 1)), dtype=torch.int32, device=dev)
            for k in ("ovl", "prep", "call", "phi", "psi"):
                out[k] = torch.empty(max(N, 1), dtype=torch.int64, device=dev)
        offs = np.zeros(self.cfg.n_traced_gpus, dtype=np.int64)
        self._bd = bd_params(params)
        tabs = chopper_tables()
        glob = chopper_global()
        calls = [("chopper_align", lambda: chopper_align(self.ctx, passes, C, out.get("counters") if C else None, offs)),
                 ("chopper_attribute", lambda: chopper_attribute(self.ctx, out.get("span_idx"))),
                 ("chopper_overlap", lambda: chopper_overlap(self.ctx, out.get("ovl"), out.get("prep"), out.get("call"),
                                                             out.get("phi"), out.get("psi"))),
                 ("chopper_breakdown", lambda: chopper_breakdown(self.ctx, self._bd, tabs)),
                 ("chopper_reduce_ranks", lambda: chopper_reduce_ranks(self.ctx, glob))]
        first = None
        for name, call in calls:
            st = call()
            if st != 0 and first is None:
                first = (name, st, chopper_last_error(self.ctx))
                if self.nranks == 1:
                    break
            # several ranks: keep calling after a failure (chopper.h failure protocol) so no peer hangs
        if first is not None:
            name, st, msg = first
            raise ChopperError(st, f"{name}: {msg}")
        cdf = chopper_report_cdf(self.ctx) if full else None
        if self.cpu is not None:
            c = self.cpu
            n = max(int(c["ts"].numel()), 1)
            out["cpu_active"] = torch.empty(n, dtype=torch.int64, device=dev)
            out["cpu_min"] = torch.empty(n, dtype=torch.float64, device=dev)
            res["cpu"] = chopper_cpu_util(self.ctx, c["ts"], c["core"], c["util"], c["topo"], out["cpu_active"],
                                          out["cpu_min"])
        st, mask = chopper_status_sync(self.ctx)
        res.update(status=st, mask=mask, offsets=offs, tables=tabs, glob=glob, out=out,
                   report=chopper_get_report(self.ctx), cdf=cdf)
        return res

    def _finish_failed_step(self) -> None:
        """After a failed chopper_load_columns on one of several ranks: make the step's remaining calls (each
        returns CHOPPER_E_STATE; align and reduce_ranks join their all-gathers with a failed block)."""
        dummy = chopper_global()
        chopper_align(self.ctx, [], self.n_counters, None, None)
        chopper_attribute(self.ctx, None)
        chopper_overlap(self.ctx)
        chopper_breakdown(self.ctx, bd_params(self._dummy_params()), chopper_tables())
        chopper_reduce_ranks(self.ctx, dummy)

    def _dummy_params(self) -> dict:
        L = self.cfg.n_labels
        return dict(tpt_peak=1.0, freq_peak_hz=1.0, b=1, s=1, R=1, warmup=0, slot_cycles=-1, slot_flops=-1,
                    slot_unum=-1, slot_uden=-1, f_gemm=np.zeros(max(L, 1)), op_type=np.zeros(max(L, 1), np.int32),
                    ratio_num=np.zeros(0, np.int32), ratio_den=np.zeros(0, np.int32), ratio_scale=np.zeros(0))

    def to_numpy(self, res: dict, n_ratios: int = 0) -> Dict[str, np.ndarray]:
        """Results in the oracle's naming (tests compare these element by element)."""
        o: Dict[str, np.ndarray] = {}
        N, C = self.N, self.n_counters
        if res.get("full"):
            out = res["out"]
            o["ev.span_idx"] = out["span_idx"][:, :N].reshape(-1).cpu().numpy()
            for k in ("ovl", "prep", "call", "phi", "psi"):
                o["ev." + k] = out[k][:N].cpu().numpy()
            o["ev.counters"] = out["counters"][:C, :N].reshape(-1).cpu().numpy() if C else np.zeros(0)
        tabs = res["tables"]
        for name, attr in (("inst", "inst"), ("layer", "layer"), ("phase", "phase"), ("iter", "iter"), ("gpu", "gpu"),
                           ("point", "point")):
            r = rows_to_numpy(getattr(tabs, attr), C, n_ratios, int(tabs.n_metrics))
            for k, v in r.items():
                key = {"n_compute": "n", "step": "step"}.get(k, k)
                if k == "counters":
                    o[f"{name}.counters"] = v.reshape(-1)
                elif k == "rates":
                    o[f"{name}.rates"] = v.reshape(-1)
                elif k == "metrics":
                    o[f"{name}.metrics"] = v
                else:
                    o[f"{name}.{key}"] = v
        nbd = int(tabs.n_bd)
        o["bd.local"] = dev_to_numpy(tabs.bd, nbd * 16, np.float64)
        g = res["glob"]
        n = int(g.n_iters)
        o["glob.step"] = np.array(g.step[:n], np.int32)
        o["glob.complete"] = np.array(g.complete[:n], np.int32)
        o["glob.sampled"] = np.array(g.sampled[:n], np.int32)
        o["glob.T"] = np.array(g.T[:n], np.int64)
        o["glob.aligned_first"] = np.array(g.aligned_first[:n], np.int64)
        o["glob.aligned_last"] = np.array(g.aligned_last[:n], np.int64)
        o["glob.throughput"] = np.array(g.throughput[:n], np.float64)
        o["glob.throughput_median"] = np.array([g.throughput_median])
        o["bd.rows"] = np.array(g.bd[:int(g.n_bd) * 16], np.float64)
        o["report.rows"] = np.array(g.report[:int(g.n_report) * 16], np.float64)
        o["e2e.rows"] = np.array(g.e2e[:33], np.float64)
        if res.get("cdf") is not None:
            o["cdf.rows"] = res["cdf"].reshape(-1)
        if res.get("cpu") is not None:
            c = res["cpu"]
            nts = int(c["n_ts"])
            o["cpu.c_active"] = res["out"]["cpu_active"][:nts].cpu().numpy()
            o["cpu.c_min"] = res["out"]["cpu_min"][:nts].cpu().numpy()
            o["cpu.summary"] = np.array([nts, c["c_active_median"], c["c_min_median"], c["c_active_max"],
                                         c["c_min_max"], c["physical_occupancy"], c["smt_coactive"],
                                         c["n_physical"]], np.float64)
        G = self.cfg.n_traced_gpus
        o["gpu.delta"] = np.array(g.delta[:G], np.int64)
        o["gpu.delta_flag"] = np.array(g.delta_flag[:G], np.int32)
        o["skew.max_ag"] = np.array([g.max_skew_ag])
        o["skew.max_rs"] = np.array([g.max_skew_rs])
        rep = res["report"]
        o["val.count"] = np.array(rep.val_count[:], np.int64)
        o["val.first"] = np.array(rep.val_first[:], np.int64)
        o["status_mask"] = np.array([res.get("mask", 0)], np.int64)
        return o

    def launches(self) -> int:
        return chopper_kernel_launches(self.ctx) if self.ctx else 0

    def host_syncs(self) -> int:
        return int(load_library().chopper_host_syncs(self.ctx)) if self.ctx else 0

    def close(self):
        if self.ctx:
            chopper_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
