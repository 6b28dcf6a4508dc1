"""bench.py -- events/s of the B200 Chopper hot path (BASELINE.json metric).

python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 4]

A step = one pass of the whole hot path (chopper_load_columns -> align ->
attribute -> overlap -> breakdown -> reduce_ranks)
over the resident synthetic trace of BASELINE.json configs[3] (Llama 3 8B FSDP
long run: 8 traced GPUs x 200 iterations, ~17.6M kernel events, 8 counters,
1 ms frequency / power samples).  With N ranks (torchrun, NCCL), rank r owns
traced GPUs {g : g mod N == r} of that same trace (strong scaling).

value  = events processed by all ranks / device time of K steps (max over ranks)
e2e    = same metric with the H2D copy of every input column from pinned host
         memory and the D2H of the results inside the timed region; inputs are
         double-buffered (trace i+1 copies on a copy stream while trace i
         computes), so e2e approaches max(H2D, compute) per step.
roofline: the fused event pass kernel (dominant), algorithmic bytes / its
         CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
--impl reference times the CPU oracle (oracle/, single-threaded C) as it
stands on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace events/sec aligned+attributed+reduced at 1/2/4/8 B200; HBM GB/s vs peak"
WORKLOADS = {
    1: "configs[0]: synthetic toy, 2 GPUs x 1 iteration x 2 layers, ~5k events, 8 counters",
    2: "configs[1]: Llama 3 8B FSDP-shaped trace, 8 GPUs x 10 iterations (~0.9M events)",
    3: "configs[2]: Llama 3 8B FSDP trace + 20 counters/kernel + 1 ms freq/power samples",
    4: "configs[3]: Llama 3 8B FSDP long run, 8 GPUs x 200 iterations (~17.6M events), 8 counters, samples",
}


# cpu_baseline: the whole workload once (~15 s of single-threaded oracle work on the dev host);
# --impl reference: traced GPU 0's shard per step (~1.5 s), so K + W steps finish within a minute or two


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured copy (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def workload(cid: int):
    import tracegen
    import paper_2512_08242_b200 as ch
    b = tracegen.generate(tracegen.config(cid))
    # product-side breakdown parameters (hardware spec, counter slots, Eq. 4 FLOP table); no oracle import here
    p = ch.default_params(b, b.labels, tracegen.workload_shapes(b.cfg), tracegen.op_kind)
    return b, p


def input_bytes(b) -> int:
    n = b.t_l.nbytes + b.t_ks.nbytes + b.t_ke.nbytes + b.meta.nbytes + b.name_id.nbytes
    n += b.span_gl.nbytes + b.span_start.nbytes + b.span_end.nbytes + b.span_label.nbytes
    n += b.smp_gpu.nbytes + b.smp_ts.nbytes + b.smp_freq.nbytes + b.smp_power.nbytes
    for (_, names, _, vals) in b.passes:
        n += names.nbytes + vals.nbytes
    return int(n)


def run_reference(args):
    """The oracle as it stands, single-threaded, on a bounded sample (traced GPU 0's shard) of the workload."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    b, p = workload(args.config)
    sample = b.gpu_slice([0])
    oracle.build()
    for _ in range(args.warmup):
        oracle.run(sample, p, max_iters=256)
    t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.run(sample, p, max_iters=256)
        t.append(time.perf_counter() - t0)
    ev = sample.n_events
    value = ev * args.steps / sum(t)
    line = {"metric": METRIC, "value": value, "unit": "events/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(t) / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOADS[args.config], "sample": f"traced GPU 0 shard ({ev} events)",
                       "n_events": ev},
            "cpu_baseline": {"value": value, "unit": "events/s", "cores": 1, "kind": "oracle",
                             "sample": f"traced GPU 0 shard of {WORKLOADS[args.config]} ({ev} events, its "
                                       f"spans, samples and counter passes) per step"},
            "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2512_08242_b200 as ch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
        dist.barrier()
    ch.build()
    b, p = workload(args.config)
    G = b.cfg.n_gpus
    mine = [g for g in range(G) if g % world == rank]
    shard = b.gpu_slice(mine) if world > 1 else b
    n_ev_local = shard.n_events
    stream = torch.cuda.Stream(dev)
    pipe = ch.Pipeline(G, len(b.labels), 256, 1 << 15, device=local, pg=pg, stream=stream)
    pipe.upload(shard, b.n_counters)
    cpu = None
    if rank == 0:
        # host CPU utilisation samples over the trace: one host trace, processed by rank 0
        import tracegen
        cpu = tracegen.cpu_samples(b.cfg.seed, int(b.t_l.min()), int(b.t_ke.max()))
        pipe.upload_cpu(*cpu)
    ch.chopper_set_timing(pipe.ctx, True)
    # warm-up (W >= 3)
    for _ in range(args.warmup):
        res = pipe.run(p, full=False)
    launches0 = pipe.launches()
    ev_ms = []
    ev_phase_ms = []
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    if pg is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        res = pipe.run(p, full=False)
        ev_ms.append(ch.chopper_phase_time(pipe.ctx, 8))
        ev_phase_ms.append(ch.chopper_phase_time(pipe.ctx, 4))
    t1.record(stream)
    torch.cuda.synchronize(dev)
    if pg is not None:
        dist.barrier()
    clocks.stop()
    launches = pipe.launches() - launches0
    ms = t0.elapsed_time(t1)
    phase_ms = {name: ch.chopper_phase_time(pipe.ctx, i) for i, name in enumerate(ch.PHASES)}
    if pg is not None:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        ntot = torch.tensor([n_ev_local], device=dev, dtype=torch.int64)
        dist.all_reduce(ntot)
        n_events = int(ntot.item())
    else:
        n_events = n_ev_local
    value = n_events * args.steps / (ms * 1e-3)

    # ---- e2e: pinned host columns copied in, results read back, every step ----
    e2e = None
    if not args.no_e2e:
        pinned = {}
        cols = {"t_l": shard.t_l, "t_ks": shard.t_ks, "t_ke": shard.t_ke,
                "meta": np.ascontiguousarray(shard.meta).view(np.int32), "name_id": shard.name_id,
                "span_gl": np.ascontiguousarray(shard.span_gl).view(np.int32), "span_start": shard.span_start,
                "span_end": shard.span_end, "span_label": shard.span_label, "smp_gpu": shard.smp_gpu,
                "smp_ts": shard.smp_ts, "smp_freq": shard.smp_freq, "smp_power": shard.smp_power}
        for k, v in cols.items():
            pinned[k] = torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
        pinned_passes = [(g, torch.from_numpy(np.ascontiguousarray(nm)).pin_memory(), sl,
                          torch.from_numpy(np.ascontiguousarray(vals)).pin_memory())
                         for (g, nm, sl, vals) in shard.passes]
        h2d = input_bytes(shard)
        pinned_cpu = {}
        if cpu is not None:
            for k, v in zip(("ts", "core", "util", "topo"), cpu):
                pinned_cpu[k] = torch.from_numpy(np.ascontiguousarray(v, pipe.cpu[k].cpu().numpy().dtype)).pin_memory()
                h2d += pinned_cpu[k].numel() * pinned_cpu[k].element_size()

        # double-buffered streaming: trace i+1's host->device copy runs on a copy stream while trace i
        # computes on the other device input set (every step still copies its whole input and reads its
        # result back; the first copy is not overlapped)
        copy_stream = torch.cuda.Stream(dev)
        sets = [pipe.input_set(), pipe.new_input_set()]
        pp = [(nm, vals) for (_, nm, _, vals) in pinned_passes]

        def e2e_run(k):
            """k steps; returns the d2h bytes of the last step's result"""
            copy_stream.wait_stream(stream)
            ready = pipe.stage_inputs(sets[0], pinned, pp, pinned_cpu, copy_stream)
            d2h = 0
            for i in range(k):
                pipe.use_inputs(sets[i % 2], ready)
                if i + 1 < k:
                    ready = pipe.stage_inputs(sets[(i + 1) % 2], pinned, pp, pinned_cpu, copy_stream)
                r = pipe.run(p, full=False)
                g = r["glob"]
                d2h = int(g.n_iters) * 44 + int(g.n_bd) * 128 + 8
            stream.wait_stream(copy_stream)
            return d2h

        e2e_run(args.warmup)
        if pg is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0.record(stream)
        d2h = e2e_run(args.steps)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        pipe.use_inputs(sets[0])
        ems = t0.elapsed_time(t1)
        if pg is not None:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": n_events * args.steps / (ems * 1e-3), "unit": "events/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    if rank != 0:
        if pg is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel: fused event pass ----
    peak, peak_src = peaks()
    R = pipe.ctx and int(ch.load_library().chopper_scratch_used(pipe.ctx))
    ev_ms = [x for x in ev_ms if x]
    ev_avg = sum(ev_ms) / len(ev_ms) if ev_ms else None
    ev_phase_ms = [x for x in ev_phase_ms if x]
    ev_phase_avg = sum(ev_phase_ms) / len(ev_phase_ms) if ev_phase_ms else None
    # algorithmic bytes per launch: event columns read by the pass
    # (t_l, t_ks, t_ke 24 B, meta 4 B, pred_end 8 B) + run id written (4 B, counters present)
    # + one 128 B sub-run row per instance run
    n_runs = int(res["tables"].inst.n)   # lower bound on sub-runs; DESIGN.md counts sub-runs ~ instances
    alg = n_ev_local * (24 + 4 + 8 + (4 if b.n_counters else 0)) + 128 * n_runs
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "event_pass_traffic.json")) as f:
            tj = json.load(f)
            if tj.get("config") == args.config:
                traffic = tj.get("dram_bytes_per_launch")
    except Exception:
        pass
    achieved = alg / (ev_avg * 1e-3) / 1e9 if ev_avg else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "kernel": "k_events_w (main event-pass kernel, a5-a9; time = its own CUDA-event bracket)",
            "peak_source": peak_src, "alg_bytes_per_launch": alg, "avg_launch_ms": ev_avg,
            "event_pass_phase_ms": ev_phase_avg,
            "event_pass_phase_frac": (alg / (ev_phase_avg * 1e-3) / 1e9 / peak) if ev_phase_avg else None,
            "phase_ms_last_step": phase_ms}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle
        oracle.build()
        t = time.perf_counter()
        oracle.run(b, p, max_iters=256)
        dt = time.perf_counter() - t
        cpu = {"value": b.n_events / dt, "unit": "events/s", "cores": 1, "kind": "oracle",
               "sample": f"the whole workload ({b.n_events} events, all 8 traced GPUs) once, single-threaded C "
                         f"oracle O1-O13, {dt:.1f} s"}

    line = {"metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "n_events": n_events, "n_counters": b.n_counters,
                       "n_spans": int(len(b.span_gl)), "n_samples": int(len(b.smp_gpu)), "mode": "tables-only",
                       "l2": f"inputs {input_bytes(b) / 1e9:.2f} GB > 126 MB L2 (no flush needed)",
                       "parallelism": f"trace shards: rank r owns traced GPUs g mod {world} == r"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary()}
    print(json.dumps(line))
    pipe.close()
    if pg is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
