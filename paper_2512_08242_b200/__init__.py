"""Thin Python binding of the B200 Chopper library (include/chopper.h).

Argument marshalling only: every step of the analysis runs in the sm_100a
kernels of libchopper.so (csrc/).  PyTorch supplies device memory (input
columns, the scratch arena), the CUDA stream and -- for several ranks -- the
NCCL communicator of a ProcessGroupNCCL.  There is no CPU fallback: importing
this package without the built extension, or calling it without a GPU, raises.
"""
from __future__ import annotations

import ctypes
import glob
import os
import subprocess
from typing import Dict, List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_HERE, "csrc")
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, "libchopper.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]

# ---------------------------------------------------------------------------
# build (nvcc cross-compiles sm_100a without a GPU)
# ---------------------------------------------------------------------------
def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(_CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(_CSRC, "*.cuh"))) + [os.path.join(_ROOT, "include", "chopper.h")]
    newest = max(os.path.getmtime(p) for p in srcs + hdrs)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    bdir = os.path.join(_HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(bdir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        cmd = ["nvcc"] + NVCC_FLAGS + ["-c", s, "-o", o]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + out.decode())
        if verbose and out:
            print(out.decode())
    tmp = LIB_PATH + ".tmp"
    cmd = ["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", "-o", tmp] + objs + \
        ["-ldl", "-lpthread", "-lrt"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


# ---------------------------------------------------------------------------
# ABI structures (mirror include/chopper.h)
# ---------------------------------------------------------------------------
P = ctypes.c_void_p
I32, I64, U32, F64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double
N_RULES = 9
STATUS = {0: "OK", 1: "E_VALIDATION", 2: "E_INVALID_ARG", 3: "E_ALIGNMENT", 4: "E_AMBIGUOUS_SPANS", 5: "E_RANGE",
          6: "E_INSUFFICIENT_DATA", 7: "E_CUDA", 8: "E_NCCL", 9: "E_STATE"}


class chopper_events(ctypes.Structure):
    _fields_ = [("n", I64), ("dispatch_ns", P), ("start_ns", P), ("end_ns", P), ("meta", P), ("name_id", P)]


class chopper_spans(ctypes.Structure):
    _fields_ = [("n", I64), ("gpu_level", P), ("start_ns", P), ("end_ns", P), ("label", P)]


class chopper_samples(ctypes.Structure):
    _fields_ = [("n", I64), ("gpu", P), ("ts_ns", P), ("freq_mhz", P), ("power_mw", P)]


class chopper_shape(ctypes.Structure):
    _fields_ = [("n_events", I64), ("n_spans", I64 * 4), ("n_samples", I64), ("n_comm", I64), ("n_counters", I32),
                ("n_local_gpus", I32), ("max_compute_streams", I32), ("laminar", I32)]


class chopper_scratch_items(ctypes.Structure):
    _fields_ = [(k, ctypes.c_size_t) for k in ("events", "spans", "unions", "subruns", "instances", "rollups",
                                               "points", "exchange", "transient", "total")]


class chopper_counter_pass(ctypes.Structure):
    _fields_ = [("gpu", I32), ("n", I64), ("name_id", P), ("k", I32), ("slot", P), ("values", P)]


class chopper_config(ctypes.Structure):
    _fields_ = [("n_traced_gpus", I32), ("n_labels", I32), ("max_iters", I32), ("max_coll_per_class", I32)]


class chopper_bd_params(ctypes.Structure):
    _fields_ = [("tpt_peak", F64), ("freq_peak_hz", F64), ("batch", I64), ("seq", I64), ("ranks", I64),
                ("warmup", I32), ("slot_gpu_cycles", I32), ("slot_perf_flops", I32), ("slot_util_num", I32),
                ("slot_util_den", I32), ("f_gemm", P), ("op_type", P), ("n_ratios", I32), ("ratio_num", P),
                ("ratio_den", P), ("ratio_scale", P)]


_ROW_I32 = ["gpu", "it", "ph", "ly", "op", "label", "rank"]
_ROW_I64 = ["n_events", "n_compute", "busy", "first_ks", "first_idx", "first_pred", "last_ke", "prep", "call", "ovl",
            "phi", "psi", "copy_ns", "ag_ns", "rs_ns"]


class chopper_rows(ctypes.Structure):
    _fields_ = [("n", I64), ("stride", I64)] + [(k, P) for k in _ROW_I32] + [(k, P) for k in _ROW_I64] + \
        [("counters", P), ("rates", P), ("wall", P), ("comm_union", P), ("aligned_first", P), ("aligned_last", P),
         ("step", P), ("metrics", P)]


class chopper_tables(ctypes.Structure):
    _fields_ = [(k, chopper_rows) for k in ("inst", "layer", "phase", "iter", "gpu", "point")] + \
        [("n_bd", I64), ("n_metrics", I32), ("bd", P)]


class chopper_global(ctypes.Structure):
    _fields_ = [("n_iters", I64), ("step", I32 * 4096), ("complete", I32 * 4096), ("sampled", I32 * 4096),
                ("T", I64 * 4096), ("aligned_first", I64 * 4096), ("aligned_last", I64 * 4096),
                ("throughput", F64 * 4096), ("throughput_median", F64), ("n_bd", I64), ("bd", F64 * (256 * 16)),
                ("delta", I64 * 256), ("delta_flag", I32 * 256), ("max_skew_ag", I64), ("max_skew_rs", I64),
                ("n_report", I64), ("report", F64 * (256 * 16)), ("e2e", F64 * 33)]


class chopper_report(ctypes.Structure):
    _fields_ = [("val_count", I64 * N_RULES), ("val_first", I64 * N_RULES), ("n_local_gpus", I64),
                ("local_gpu", I32 * 256), ("t_min", I64), ("t_max", I64), ("full_sort_used", I32),
                ("non_laminar_lists", I32)]


class chopper_ingest_out(ctypes.Structure):
    _fields_ = [("t_l", P), ("t_ks", P), ("t_ke", P), ("meta", P), ("name_id", P), ("ev_cap", I64), ("span_gl", P),
                ("span_start", P), ("span_end", P), ("span_label", P), ("span_cap", I64)]


class chopper_ingest_report(ctypes.Structure):
    _fields_ = [("n_objects", I64), ("n_kernels", I64), ("n_flows", I64), ("n_spans", I64), ("n_missing", I64),
                ("n_names", I64), ("bad_offset", I64)]


class chopper_cpu_samples(ctypes.Structure):
    _fields_ = [("n", I64), ("ts_ns", P), ("logical_core", P), ("util_pct", P)]


class chopper_cpu_summary(ctypes.Structure):
    _fields_ = [("n_ts", I64), ("n_logical", I32), ("n_physical", I32), ("c_active_median", F64),
                ("c_min_median", F64), ("c_active_max", F64), ("c_min_max", F64), ("physical_occupancy", F64),
                ("smt_coactive", F64)]


# every symbol include/chopper.h declares
EXPORTS = ["chopper_scratch_bytes", "chopper_create", "chopper_load_columns", "chopper_align", "chopper_attribute",
           "chopper_overlap", "chopper_breakdown", "chopper_reduce_ranks", "chopper_get_report",
           "chopper_status_sync", "chopper_last_error", "chopper_destroy", "chopper_kernel_launches",
           "chopper_abi_version", "chopper_pass_mismatch", "chopper_pass_conflict", "chopper_counter_present",
           "chopper_scratch_used", "chopper_set_timing", "chopper_phase_time", "chopper_report_cdf",
           "chopper_cpu_util", "chopper_set_metrics", "chopper_ingest_scratch_bytes", "chopper_ingest_chrome",
           "chopper_set_allgather", "chopper_loopback_create", "chopper_scratch_plan", "chopper_host_syncs", "chopper_loopback_destroy",
           "chopper_loopback_allgather"]

_lib = None


def load_library() -> ctypes.CDLL:
    """Load libchopper.so (fails loudly if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libchopper.so not built ({LIB_PATH}); run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    S = I32
    sig = {
        "chopper_scratch_bytes": (ctypes.c_size_t, [ctypes.POINTER(chopper_config), I64, I64, I64, I32]),
        "chopper_create": (S, [ctypes.POINTER(P), ctypes.POINTER(chopper_config), ctypes.c_int, P, P, ctypes.c_int,
                               ctypes.c_int, P, ctypes.c_size_t]),
        "chopper_load_columns": (S, [P, ctypes.POINTER(chopper_events), ctypes.POINTER(chopper_spans),
                                     ctypes.POINTER(chopper_samples)]),
        "chopper_align": (S, [P, ctypes.POINTER(chopper_counter_pass), I32, I32, P, P]),
        "chopper_attribute": (S, [P, P]),
        "chopper_overlap": (S, [P, P, P, P, P, P]),
        "chopper_breakdown": (S, [P, ctypes.POINTER(chopper_bd_params), ctypes.POINTER(chopper_tables)]),
        "chopper_reduce_ranks": (S, [P, ctypes.POINTER(chopper_global)]),
        "chopper_get_report": (S, [P, ctypes.POINTER(chopper_report)]),
        "chopper_status_sync": (S, [P, ctypes.POINTER(U32)]),
        "chopper_last_error": (ctypes.c_char_p, [P]),
        "chopper_destroy": (None, [P]),
        "chopper_kernel_launches": (I64, [P]),
        "chopper_host_syncs": (I64, [P]),
        "chopper_abi_version": (I32, []),
        "chopper_pass_mismatch": (I64, [P, I32]),
        "chopper_pass_conflict": (I64, [P, I32]),
        "chopper_counter_present": (I32, [P, I32, I32]),
        "chopper_scratch_used": (I64, [P]),
        "chopper_set_timing": (None, [P, I32]),
        "chopper_phase_time": (I32, [P, I32, ctypes.POINTER(ctypes.c_float)]),
        "chopper_report_cdf": (I32, [P, P, I64, ctypes.POINTER(I64)]),
        "chopper_set_metrics": (I32, [P, I32, P, I32, P, ctypes.POINTER(I32)]),
        "chopper_ingest_scratch_bytes": (ctypes.c_size_t, [I64]),
        "chopper_ingest_chrome": (I32, [P, P, I64, P, ctypes.c_size_t, ctypes.POINTER(chopper_ingest_out),
                                        ctypes.POINTER(chopper_ingest_report)]),
        "chopper_cpu_util": (I32, [P, ctypes.POINTER(chopper_cpu_samples), P, I32, P, P, I64,
                                   ctypes.POINTER(chopper_cpu_summary)]),
        "chopper_set_allgather": (I32, [P, P, P]),
        "chopper_scratch_plan": (ctypes.c_size_t, [ctypes.POINTER(chopper_config), ctypes.POINTER(chopper_shape),
                                                   ctypes.POINTER(chopper_scratch_items)]),
        "chopper_loopback_create": (P, [I32]),
        "chopper_loopback_destroy": (None, [P]),
        "chopper_loopback_allgather": (I32, [P, P, P, ctypes.c_size_t, I32, I32, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


# ---------------------------------------------------------------------------
# ABI wrappers (same names as the C entry points; marshalling only)
# ---------------------------------------------------------------------------
def _ptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


class ChopperError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(ctx, s: int, what: str, allow=()):
    if s != 0 and s not in allow:
        msg = load_library().chopper_last_error(ctx).decode() if ctx else ""
        raise ChopperError(s, f"{what}: {msg}")
    return s


def chopper_scratch_bytes(cfg: chopper_config, n_events: int, n_spans: int, n_samples: int, n_counters: int) -> int:
    return int(load_library().chopper_scratch_bytes(ctypes.byref(cfg), n_events, n_spans, n_samples, n_counters))


def chopper_scratch_plan(cfg: chopper_config, shape: chopper_shape) -> Dict[str, int]:
    """itemized scratch plan (bytes) for a trace of the given shape (include/chopper.h)"""
    it = chopper_scratch_items()
    load_library().chopper_scratch_plan(ctypes.byref(cfg), ctypes.byref(shape), ctypes.byref(it))
    return {k: int(getattr(it, k)) for k, _ in chopper_scratch_items._fields_}


def chopper_create(cfg: chopper_config, device: int, stream_ptr: int, nccl_comm: int, rank: int, nranks: int,
                   scratch) -> int:
    ctx = P()
    s = load_library().chopper_create(ctypes.byref(ctx), ctypes.byref(cfg), device, stream_ptr or None,
                                      nccl_comm or None, rank, nranks, _ptr(scratch), scratch.numel())
    _check(None, s, "chopper_create")
    return ctx.value


def chopper_load_columns(ctx, ev: chopper_events, sp: chopper_spans, smp: Optional[chopper_samples]) -> int:
    return load_library().chopper_load_columns(ctx, ctypes.byref(ev), ctypes.byref(sp),
                                               ctypes.byref(smp) if smp is not None else None)


class PassArray:
    """A prebuilt ctypes array of chopper_counter_pass (the Pipeline keeps one per input set)."""
    __slots__ = ("arr", "n")

    def __init__(self, arr, n: int):
        self.arr, self.n = arr, n


def chopper_align(ctx, passes, n_counters: int, counters_out=None, offsets=None) -> int:
    """passes: a list of chopper_counter_pass, or a PassArray"""
    if isinstance(passes, PassArray):
        arr, n = passes.arr, passes.n
    else:
        arr, n = (chopper_counter_pass * max(len(passes), 1))(*passes), len(passes)
    return load_library().chopper_align(ctx, arr, n, n_counters, _ptr(counters_out),
                                        offsets.ctypes.data if offsets is not None else None)


def chopper_attribute(ctx, span_idx=None) -> int:
    return load_library().chopper_attribute(ctx, _ptr(span_idx))


def chopper_overlap(ctx, ovl=None, prep=None, call=None, phi=None, psi=None) -> int:
    return load_library().chopper_overlap(ctx, _ptr(ovl), _ptr(prep), _ptr(call), _ptr(phi), _ptr(psi))


def chopper_breakdown(ctx, p: chopper_bd_params, out: chopper_tables) -> int:
    return load_library().chopper_breakdown(ctx, ctypes.byref(p), ctypes.byref(out))


def chopper_reduce_ranks(ctx, out: chopper_global) -> int:
    return load_library().chopper_reduce_ranks(ctx, ctypes.byref(out))


def chopper_report_cdf(ctx) -> np.ndarray:
    """per-GPU overlap CDF rows (label, gpu, duration / gpu minimum, overlap ratio, cdf) of every op label"""
    lib = load_library()
    n = I64()
    _check(ctx, lib.chopper_report_cdf(ctx, None, 0, ctypes.byref(n)), "chopper_report_cdf")
    out = np.zeros((max(n.value, 1), 5), np.float64)
    if n.value > 0:
        _check(ctx, lib.chopper_report_cdf(ctx, out.ctypes.data, n.value, ctypes.byref(n)), "chopper_report_cdf")
    return out[:n.value]


class LoopbackGroup:
    """In-process all-gather transport for `nranks` contexts on one device (chopper_loopback_*): each rank's
    Pipeline runs in its own host thread; used to run P = 1/2/4/8 ranks on one GPU."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.handle = load_library().chopper_loopback_create(nranks)
        if not self.handle:
            raise ValueError(f"bad loopback group size {nranks}")

    def close(self):
        if self.handle:
            load_library().chopper_loopback_destroy(self.handle)
            self.handle = None


def chopper_set_allgather_loopback(ctx, group: LoopbackGroup) -> None:
    lib = load_library()
    fn = ctypes.cast(lib.chopper_loopback_allgather, P)
    _check(ctx, lib.chopper_set_allgather(ctx, fn, group.handle), "chopper_set_allgather")


def chopper_get_report(ctx) -> chopper_report:
    r = chopper_report()
    load_library().chopper_get_report(ctx, ctypes.byref(r))
    return r


def chopper_status_sync(ctx):
    m = U32()
    s = load_library().chopper_status_sync(ctx, ctypes.byref(m))
    return s, m.value


def chopper_last_error(ctx) -> str:
    return load_library().chopper_last_error(ctx).decode()


def chopper_destroy(ctx) -> None:
    load_library().chopper_destroy(ctx)


def chopper_kernel_launches(ctx) -> int:
    return int(load_library().chopper_kernel_launches(ctx))


def chopper_set_timing(ctx, on: bool) -> None:
    load_library().chopper_set_timing(ctx, 1 if on else 0)


PHASES = ["load", "align", "attribute", "overlap_prep", "event_pass", "tables", "breakdown", "reduce_ranks",
          "event_kernel", "counter_kernel"]


def chopper_phase_time(ctx, phase: int) -> Optional[float]:
    ms = ctypes.c_float()
    s = load_library().chopper_phase_time(ctx, phase, ctypes.byref(ms))
    return float(ms.value) if s == 0 else None


# ---------------------------------------------------------------------------
# device-pointer views (read tables back through torch)
# ---------------------------------------------------------------------------
class _DevArray:
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def dev_to_numpy(ptr: Optional[int], n: int, dtype) -> np.ndarray:
    import torch
    dt = np.dtype(dtype)
    if not ptr or n <= 0:
        return np.zeros(max(n, 0), dtype=dt)
    t = torch.as_tensor(_DevArray(ptr, n, dt.str), device="cuda")
    return t.cpu().numpy().copy()


def rows_to_numpy(r: chopper_rows, n_counters: int, n_ratios: int = 0, n_metrics: int = 0) -> Dict[str, np.ndarray]:
    n = int(r.n)
    out = {}
    for k in _ROW_I32:
        out[k] = dev_to_numpy(getattr(r, k), n, np.int32)
    for k in _ROW_I64:
        out[k] = dev_to_numpy(getattr(r, k), n, np.int64)
    st = int(r.stride) if r.stride else n
    out["counters"] = np.stack([dev_to_numpy((r.counters or 0) + 8 * s * st if r.counters else None, n, np.float64)
                                for s in range(n_counters)]) if n_counters else np.zeros((0, n))
    if r.rates and n_ratios:
        out["rates"] = np.stack([dev_to_numpy(r.rates + 8 * q * st, n, np.float64) for q in range(n_ratios)])
    if r.metrics and n_metrics:
        out["metrics"] = np.stack([dev_to_numpy(r.metrics + 8 * q * st, n, np.float64) for q in range(n_metrics)])
    for k in ("wall", "comm_union", "aligned_first", "aligned_last"):
        if getattr(r, k):
            out[k] = dev_to_numpy(getattr(r, k), n, np.int64)
    if r.step:
        out["step"] = dev_to_numpy(r.step, n, np.int32)
    return out


def bd_params(p: dict) -> chopper_bd_params:
    """chopper_bd_params from a dict; host arrays are kept alive on the returned object."""
    keep = dict(f_gemm=np.ascontiguousarray(p["f_gemm"], np.float64),
                op_type=np.ascontiguousarray(p["op_type"], np.int32),
                rn=np.ascontiguousarray(p["ratio_num"], np.int32), rd=np.ascontiguousarray(p["ratio_den"], np.int32),
                rs=np.ascontiguousarray(p["ratio_scale"], np.float64))
    q = chopper_bd_params(tpt_peak=p["tpt_peak"], freq_peak_hz=p["freq_peak_hz"], batch=p["b"], seq=p["s"],
                          ranks=p["R"], warmup=p["warmup"], slot_gpu_cycles=p["slot_cycles"],
                          slot_perf_flops=p["slot_flops"], slot_util_num=p["slot_unum"],
                          slot_util_den=p["slot_uden"], f_gemm=keep["f_gemm"].ctypes.data,
                          op_type=keep["op_type"].ctypes.data, n_ratios=len(keep["rn"]),
                          ratio_num=keep["rn"].ctypes.data if len(keep["rn"]) else None,
                          ratio_den=keep["rd"].ctypes.data if len(keep["rd"]) else None,
                          ratio_scale=keep["rs"].ctypes.data if len(keep["rs"]) else None)
    q._keep = keep
    return q


def chopper_ingest_chrome(ctx, json_dev, ev_cap: int, span_cap: int, device=0):
    """Chrome-trace JSON (a uint8 CUDA tensor) -> event and span columns (CUDA tensors, trimmed) + report dict."""
    import torch
    lib = load_library()
    dev = json_dev.device
    n = int(json_dev.numel())
    scratch = torch.empty(int(lib.chopper_ingest_scratch_bytes(n)), dtype=torch.uint8, device=dev)
    cols = {"t_l": torch.empty(max(ev_cap, 1), dtype=torch.int64, device=dev),
            "t_ks": torch.empty(max(ev_cap, 1), dtype=torch.int64, device=dev),
            "t_ke": torch.empty(max(ev_cap, 1), dtype=torch.int64, device=dev),
            "meta": torch.empty(max(ev_cap, 1), dtype=torch.int32, device=dev),
            "name_id": torch.empty(max(ev_cap, 1), dtype=torch.int32, device=dev),
            "span_gl": torch.empty(max(span_cap, 1), dtype=torch.int32, device=dev),
            "span_start": torch.empty(max(span_cap, 1), dtype=torch.int64, device=dev),
            "span_end": torch.empty(max(span_cap, 1), dtype=torch.int64, device=dev),
            "span_label": torch.empty(max(span_cap, 1), dtype=torch.int32, device=dev)}
    o = chopper_ingest_out(*(_ptr(cols[k]) for k in ("t_l", "t_ks", "t_ke", "meta", "name_id")), ev_cap,
                           *(_ptr(cols[k]) for k in ("span_gl", "span_start", "span_end", "span_label")), span_cap)
    rep = chopper_ingest_report()
    _check(ctx, lib.chopper_ingest_chrome(ctx, _ptr(json_dev), n, _ptr(scratch), scratch.numel(), ctypes.byref(o),
                                          ctypes.byref(rep)), "chopper_ingest_chrome")
    r = {k: getattr(rep, k) for k, _ in chopper_ingest_report._fields_}
    nk, ns = int(rep.n_kernels), int(rep.n_spans)
    for k in ("t_l", "t_ks", "t_ke", "meta", "name_id"):
        cols[k] = cols[k][:nk]
    for k in ("span_gl", "span_start", "span_end", "span_label"):
        cols[k] = cols[k][:ns]
    return cols, r


def chopper_set_metrics(ctx, exprs, names) -> None:
    """Compile the derived-metric registry on the host side of the library; raises
    ChopperError (MissingCounter / ParseError) naming the failing expression."""
    lib = load_library()
    ex = (ctypes.c_char_p * max(len(exprs), 1))(*[e.encode() for e in exprs])
    nm = (ctypes.c_char_p * max(len(names), 1))(*[n.encode() for n in names])
    bad = I32(-1)
    _check(ctx, lib.chopper_set_metrics(ctx, len(exprs), ex, len(names), nm, ctypes.byref(bad)),
           f"chopper_set_metrics (expression {bad.value})")


def chopper_cpu_util(ctx, ts, core, util, topology, c_active=None, c_min=None):
    """CPU utilization over device tensors (int64 ts, int32 core, float64 util, int32 topology);
    optional device outputs c_active (int64) / c_min (float64) per timestamp.  Returns the summary as a dict."""
    lib = load_library()
    s = chopper_cpu_samples(int(ts.numel()), _ptr(ts), _ptr(core), _ptr(util))
    out = chopper_cpu_summary()
    cap = 0 if c_active is None else int(c_active.numel())
    _check(ctx, lib.chopper_cpu_util(ctx, ctypes.byref(s), _ptr(topology), int(topology.numel()), _ptr(c_active),
                                     _ptr(c_min), cap, ctypes.byref(out)), "chopper_cpu_util")
    return {k: getattr(out, k) for k, _ in chopper_cpu_summary._fields_}


from .pipeline import Pipeline, default_params, flops_table, scratch_plan, trace_shape  # noqa: E402,F401

